"""NEXT-1 parity: rt_predict_mlp against the fp64 oracle (oracle/mlp.py), in
both precisions.

fp32 (default, k_mlp_f32): every multiply-add is one binary32 FMA, chains in
index order.  A chain of K FMAs moves a value by at most ~K unit roundoffs of
the same sum over absolute values, so over the 606 FMAs that feed one output
(6 + 100 + 200 + 200 + 100) |u - u_fp64| <= 1024 * 2^-24 * mlp_abs_pass
(DESIGN.md §7 K7).  On a network without cancellation (non-negative weights,
like a length model whose partial sums all add) that bound is relative, and
north_star's "predicted lengths within 1e-5 relative" is asserted directly.

tf32x3 (k_mlp_tf32): layers 2-4 on tcgen05 kind::tf32 with every operand split
into two tf32 numbers (hi + lo, residual <= 2^-22) and three products per
multiply; per product the error is <= 3 * 2^-22 = 12 unit roundoffs of |a||b|,
so the same 1024 * 2^-24 bound holds with room (606 + 3 * 12 roundoffs).

bf16 (opt-in, k_mlp on tcgen05): layers 2-4 round their weights and input
activations to bf16 (unit roundoff 2^-8): six roundings perturb every partial
sum by at most ~6 * 2^-8 of the same sum over absolute values, so
|u - u_fp64| < 2^-5 * mlp_abs_pass; networks whose values are bf16-exact match
exactly.
"""
import numpy as np
import pytest

import oracle
from oracle.mlp import DIMS, mlp_abs_pass, mlp_predict
from rtgen import configs, mlp_weights

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2309_06619_b200 as rt  # noqa: E402

DEV = torch.device("cuda", 0)
TOL_BF16 = 2.0 ** -5
TOL_FP32 = 1024 * 2.0 ** -24


@pytest.fixture(scope="module")
def ctx():
    return rt.Context(configs.read_lexicon(), 0)


def _feat(n, seed, hi=60):
    rng = np.random.default_rng(seed)
    f = np.zeros((n, 8), np.uint16)
    f[:, :7] = rng.integers(0, hi, (n, 7))
    return f


def _run(ctx, f, ws, bs, precision="fp32"):
    ctx.set_mlp(ws, bs)
    ctx.set_mlp_precision(precision)
    u = ctx.predict_mlp(torch.from_numpy(f.view(np.int16)).to(DEV))
    torch.cuda.synchronize()
    ctx.set_mlp_precision("fp32")
    return u.cpu().numpy()


def _length_model(seed):
    """Non-negative weights scaled by 1/fan_in, positive biases: every partial sum
    adds (no cancellation), outputs of a few tens of tokens."""
    ws, bs = mlp_weights(seed)
    ws = [np.abs(w) / w.shape[1] for w in ws]
    ws[4] = ws[4] * 5000.0  # output scale: tens of tokens
    bs = [np.abs(b) for b in bs]
    return [w.astype(np.float32) for w in ws], [b.astype(np.float32) for b in bs]


FP32_MODES = ["fp32", "tf32x3"]


@pytest.mark.parametrize("mode", FP32_MODES)
@pytest.mark.parametrize("n", [1, 63, 64, 65, 127, 128, 129, 1000, 40000])
def test_mlp_fp32_random_weights(ctx, n, mode):
    ws, bs = mlp_weights(7)
    f = _feat(n, n)
    g = _run(ctx, f, ws, bs, mode)
    want = mlp_predict(f, ws, bs)
    bound = TOL_FP32 * mlp_abs_pass(f, ws, bs)
    err = np.abs(g.astype(np.float64) - want)
    assert (err <= bound).all(), (np.max(err / bound), np.argmax(err / bound))


@pytest.mark.parametrize("mode", FP32_MODES)
@pytest.mark.parametrize("n", [129, 50000])
def test_mlp_fp32_within_1e5_relative(ctx, n, mode):
    ws, bs = _length_model(11)
    f = _feat(n, 5 + n)
    g = _run(ctx, f, ws, bs, mode).astype(np.float64)
    want = mlp_predict(f, ws, bs)
    assert (want > 5.0).all() and (want < 500.0).all()
    rel = np.abs(g - want) / want
    assert rel.max() <= 1e-5, rel.max()


@pytest.mark.parametrize("mode", FP32_MODES)
def test_mlp_fp32_on_rule_features(ctx, mode):
    d = configs.config2(n=3000, gid0=777)
    f = oracle.rule_gen(oracle.Lexicon(configs.read_lexicon()), d["data"], d["offsets"])
    for ws, bs in (mlp_weights(21), _length_model(21)):
        g = _run(ctx, f, ws, bs, mode)
        err = np.abs(g.astype(np.float64) - mlp_predict(f, ws, bs))
        assert (err <= TOL_FP32 * mlp_abs_pass(f, ws, bs)).all()


@pytest.mark.parametrize("n", [1, 127, 128, 129, 1000, 40000])
def test_mlp_bf16_random_weights(ctx, n):
    ws, bs = mlp_weights(7)
    f = _feat(n, n)
    g = _run(ctx, f, ws, bs, "bf16")
    want = mlp_predict(f, ws, bs)
    bound = TOL_BF16 * mlp_abs_pass(f, ws, bs)
    err = np.abs(g.astype(np.float64) - want)
    assert (err <= bound).all(), (np.max(err / bound), np.argmax(err / bound))
    assert np.median(err / np.maximum(np.abs(want), 1e-3)) < 2e-2


def test_mlp_bf16_on_rule_features(ctx):
    # the real pipeline's features (config 2 slice, oracle rule scores)
    d = configs.config2(n=3000, gid0=777)
    f = oracle.rule_gen(oracle.Lexicon(configs.read_lexicon()), d["data"], d["offsets"])
    ws, bs = mlp_weights(21)
    g = _run(ctx, f, ws, bs, "bf16")
    err = np.abs(g.astype(np.float64) - mlp_predict(f, ws, bs))
    assert (err <= TOL_BF16 * mlp_abs_pass(f, ws, bs)).all()


def _zero():
    return ([np.zeros((o, i), np.float32) for i, o in zip(DIMS[:-1], DIMS[1:])],
            [np.zeros(o, np.float32) for o in DIMS[1:]])


@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "bf16"])
def test_mlp_exact_networks(ctx, precision):
    # zero network -> 0; a one-path network routing feature 4 with
    # gain g -> g * f4, exact when every value is a bf16 number (integers < 256: 8 bits)
    f = _feat(5000, 3, hi=60)
    ws, bs = _zero()
    assert (_run(ctx, f, ws, bs, precision) == 0).all()
    g = 2.0
    ws[0][0, 4] = g
    for k in (1, 2, 3, 4):
        ws[k][0, 0] = 1.0
    assert np.array_equal(_run(ctx, f, ws, bs, precision).astype(np.float64), g * f[:, 4])


def test_mlp_api_errors(ctx):
    c = rt.Context(configs.read_lexicon(), 0)
    with pytest.raises(rt.RtlmError):
        c.predict_mlp(torch.zeros((4, 8), dtype=torch.int16, device=DEV))
    ws, bs = mlp_weights(1)
    c.set_mlp(ws, bs)
    assert c.predict_mlp(torch.zeros((0, 8), dtype=torch.int16, device=DEV)).numel() == 0
    with pytest.raises(ValueError):
        c.set_mlp(ws[:4] + [np.zeros((2, 100), np.float32)], bs)
    with pytest.raises(KeyError):
        c.set_mlp_precision("fp16")
    with pytest.raises(rt.RtlmError, match="precision"):
        c._check(c._L.rt_set_mlp_precision(c._h, 7))


@pytest.mark.parametrize("mode", ["fp32", "tf32x3", "bf16"])
def test_mlp_full_config2_sampled(ctx, mode):
    # BASELINE's full size (config 2: 2^20 requests) in the bench's launch configuration (one
    # rt_predict_mlp over the whole queue, all SMs): the features come from the GPU scorer (bit-exact
    # against the oracle in test_gpu_parity), the oracle recomputes 2048 sampled rows one by one
    d = configs.config2()
    data = torch.from_numpy(d["data"]).to(DEV)
    off = torch.from_numpy(d["offsets"].view(np.int32)).to(DEV)
    feat = ctx.score(data, off)
    ws, bs = mlp_weights(12345)
    ctx.set_mlp(ws, bs)
    ctx.set_mlp_precision(mode)
    u = ctx.predict_mlp(feat).cpu().numpy().astype(np.float64)
    ctx.set_mlp_precision("fp32")
    n = feat.shape[0]
    assert u.shape == (n,) and n == 1 << 20
    rng = np.random.default_rng(99)
    idx = np.unique(np.concatenate([rng.integers(0, n, 2040), [0, 1, 127, 128, n - 129, n - 128, n - 2, n - 1]]))
    f = feat.cpu().numpy().view(np.uint16)[idx]
    want, absp = mlp_predict(f, ws, bs), mlp_abs_pass(f, ws, bs)
    tol = TOL_BF16 if mode == "bf16" else TOL_FP32
    assert (np.abs(u[idx] - want) <= tol * absp).all()


# ---------------------------------------------------------------- NEXT-2: rt_train_mlp
from oracle.mlp import mlp_train_adam  # noqa: E402


def _train_case(n=300, seed=21):
    rng = np.random.default_rng(seed)
    f = _feat(n, seed, hi=12)
    y = (5.0 + 2.0 * f[:, 3] + 1.5 * f[:, 1] + rng.normal(0, 1.0, n)).astype(np.float32)
    ws, bs = mlp_weights(seed)
    return f, y, [w.astype(np.float32) for w in ws], [b.astype(np.float32) for b in bs]


def _gpu_train(ctx, f, y, ws, bs, epochs, batch, lr, seed):
    ctx.set_mlp(ws, bs)
    losses = ctx.train_mlp(torch.from_numpy(f.view(np.int16)).to(DEV), torch.from_numpy(y).to(DEV), epochs, batch, lr,
                           seed)
    w2, b2 = ctx.get_mlp()
    return losses, w2, b2


def test_train_matches_the_fp64_oracle(ctx):
    """3 epochs of 300 rows in batches of 64 (the last one partial), lr 1e-3: the
    fp32 training follows the fp64 oracle: per-epoch losses within 1e-4
    relative; the trained networks' predictions within 1e-3 relative; each
    parameter within 1e-3 lr + 1e-5 |w| (Adam moves a parameter by ~lr per step
    whatever the gradient's scale, so fp32 / fp64 differences stay ~lr-relative;
    a parameter whose gradient is at fp32 noise level may differ by up to 2 lr
    per step -- allowed for at most 0.1 % of them)."""
    f, y, ws, bs = _train_case()
    epochs, batch, lr, seed = 3, 64, 1e-3, 11
    losses, w2, b2 = _gpu_train(ctx, f, y, ws, bs, epochs, batch, lr, seed)
    ow, ob, ol = mlp_train_adam(f, y.astype(np.float64), ws, bs, epochs, batch, lr, seed)
    np.testing.assert_allclose(losses, ol, rtol=1e-4)
    pg = mlp_predict(f, [w.astype(np.float64) for w in w2], [b.astype(np.float64) for b in b2])
    po = mlp_predict(f, ow, ob)
    assert np.all(np.abs(pg - po) <= 1e-3 * np.maximum(np.abs(po), 1.0))
    steps = epochs * ((len(y) + batch - 1) // batch)
    d = np.concatenate([np.abs(a - b).ravel() for a, b in zip(w2 + b2, ow + ob)])
    w = np.concatenate([np.abs(b).ravel() for b in ow + ob])
    close = d <= 1e-3 * lr + 1e-5 * w
    assert close.mean() >= 0.999, close.mean()
    assert d.max() <= 2 * lr * steps


def test_train_is_deterministic_and_learns(ctx):
    f, y, ws, bs = _train_case(n=1000, seed=5)
    l1, w1, b1 = _gpu_train(ctx, f, y, ws, bs, 8, 128, 1e-3, 3)
    l2, w2, b2 = _gpu_train(ctx, f, y, ws, bs, 8, 128, 1e-3, 3)
    assert np.array_equal(l1, l2)
    assert all(np.array_equal(a, b) for a, b in zip(w1 + b1, w2 + b2))
    assert l1[-1] < 0.5 * l1[0], l1
    # the trained model serves rt_predict_mlp (all precisions follow the trained weights)
    u = ctx.predict_mlp(torch.from_numpy(f.view(np.int16)).to(DEV)).cpu().numpy()
    ref = mlp_predict(f, [w.astype(np.float64) for w in w1], [b.astype(np.float64) for b in b1])
    assert np.all(np.abs(u - ref) <= TOL_FP32 * mlp_abs_pass(f, w1, b1) + 1e-6)


def test_train_argument_checks(ctx):
    f, y, ws, bs = _train_case(n=10)
    fd, yd = torch.from_numpy(f.view(np.int16)).to(DEV), torch.from_numpy(y).to(DEV)
    fresh = rt.Context(configs.read_lexicon(), 0)
    with pytest.raises(rt.RtlmError, match="no MLP model"):
        fresh.train_mlp(fd, yd, 1, 4, 1e-3)
    ctx.set_mlp(ws, bs)
    with pytest.raises(rt.RtlmError, match="batch"):
        ctx.train_mlp(fd, yd, 1, 0, 1e-3)
    with pytest.raises(rt.RtlmError, match="lr"):
        ctx.train_mlp(fd, yd, 1, 4, 0.0)
    assert len(ctx.train_mlp(fd, yd, 0, 4, 1e-3)) == 0  # zero epochs: no-op
    w2, b2 = ctx.get_mlp()
    assert all(np.array_equal(a, b) for a, b in zip(ws + bs, w2 + b2))


def test_train_tiny_sets(ctx):
    """n = 1 (one row, the identity permutation) and batch > n (one partial batch per
    epoch) against the fp64 oracle."""
    for n, batch in ((1, 4), (7, 64)):
        f, y, ws, bs = _train_case(n=n, seed=40 + n)
        losses, w2, b2 = _gpu_train(ctx, f, y, ws, bs, 4, batch, 1e-3, 9)
        _, _, ol = mlp_train_adam(f, y.astype(np.float64), ws, bs, 4, batch, 1e-3, 9)
        np.testing.assert_allclose(losses, ol, rtol=1e-4)
