"""NEXT-1 parity: rt_predict_mlp (tcgen05, BF16 operands, FP32 accumulation)
against the fp64 oracle (oracle/mlp.py).

Tolerance (DESIGN.md §7 K7): layers 2-4 round their weights and input
activations to bf16 (round-to-nearest, unit roundoff 2^-8): six roundings,
each perturbing a term by at most a relative 2^-8, so every partial sum moves
by at most ~6 * 2^-8 of the same sum taken over absolute values; with
fp32 accumulation this is < 2^-5 * mlp_abs_pass.  Networks whose weights and
activations are exactly representable in bf16 must match exactly.
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
TOL = 2.0 ** -5


@pytest.fixture(scope="module")
def ctx():
    return rt.Context(configs.read_lexicon(), 0)


def _feat(n, seed, hi=60):
    rng = np.random.default_rng(seed)
    f = np.zeros((n, 8), np.uint16)
    f[:, :7] = rng.integers(0, hi, (n, 7))
    return f


def _run(ctx, f, ws, bs):
    ctx.set_mlp(ws, bs)
    u = ctx.predict_mlp(torch.from_numpy(f.view(np.int16)).to(DEV))
    torch.cuda.synchronize()
    return u.cpu().numpy()


@pytest.mark.parametrize("n", [1, 127, 128, 129, 1000, 40000])
def test_mlp_random_weights(ctx, n):
    ws, bs = mlp_weights(7)
    f = _feat(n, n)
    g = _run(ctx, f, ws, bs)
    want = mlp_predict(f, ws, bs)
    bound = TOL * mlp_abs_pass(f, ws, bs)
    err = np.abs(g.astype(np.float64) - want)
    assert (err <= bound).all(), (np.max(err / bound), np.argmax(err / bound))
    assert np.median(err / np.maximum(np.abs(want), 1e-3)) < 2e-2


def test_mlp_on_rule_features(ctx):
    # the real pipeline's features (config 1 prompts + a config 2 slice, oracle rule scores)
    d = configs.config2(n=3000, gid0=777)
    f = oracle.rule_gen(oracle.Lexicon(configs.read_lexicon()), d["data"], d["offsets"])
    ws, bs = mlp_weights(21)
    g = _run(ctx, f, ws, bs)
    err = np.abs(g.astype(np.float64) - mlp_predict(f, ws, bs))
    assert (err <= TOL * mlp_abs_pass(f, ws, bs)).all()


def _zero():
    return ([np.zeros((o, i), np.float32) for i, o in zip(DIMS[:-1], DIMS[1:])],
            [np.zeros(o, np.float32) for o in DIMS[1:]])


def test_mlp_exact_networks(ctx):
    # zero network -> 0; a one-path network routing feature 4 with
    # gain g -> g * f4, exact when every value is a bf16 number (integers < 256: 8 bits)
    f = _feat(5000, 3, hi=60)
    ws, bs = _zero()
    assert (_run(ctx, f, ws, bs) == 0).all()
    g = 2.0
    ws[0][0, 4] = g
    for k in (1, 2, 3, 4):
        ws[k][0, 0] = 1.0
    assert np.array_equal(_run(ctx, f, ws, bs).astype(np.float64), g * f[:, 4])


def test_mlp_api_errors(ctx):
    c = rt.Context(configs.read_lexicon(), 0)
    with pytest.raises(rt.RtlmError):
        c.predict_mlp(torch.zeros((4, 8), dtype=torch.int16, device=DEV))
    ws, bs = mlp_weights(1)
    c.set_mlp(ws, bs)
    assert c.predict_mlp(torch.zeros((0, 8), dtype=torch.int16, device=DEV)).numel() == 0
    with pytest.raises(ValueError):
        c.set_mlp(ws[:4] + [np.zeros((2, 100), np.float32)], bs)
