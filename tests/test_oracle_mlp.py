"""Pins of the NEXT-1 MLP oracle (oracle/mlp.py) against closed forms
(SPEC S:196-198 examples) and properties that hold for any weights."""
import numpy as np

from oracle.mlp import DIMS, mlp_abs_pass, mlp_predict
from rtgen import mlp_weights


def _zero():
    ws = [np.zeros((o, i), np.float32) for i, o in zip(DIMS[:-1], DIMS[1:])]
    bs = [np.zeros(o, np.float32) for o in DIMS[1:]]
    return ws, bs


def _feats(n=64, seed=5):
    rng = np.random.default_rng(seed)
    f = np.zeros((n, 8), np.uint16)
    f[:, :7] = rng.integers(0, 40, (n, 7))
    return f


def test_zero_network_is_zero():
    # S:196 "zero-weight, zero-bias model, any features -> value 0"
    ws, bs = _zero()
    assert (mlp_predict(_feats(), ws, bs) == 0).all()


def test_one_path_network_routes_feature_4():
    # S:197 "identity-like handcrafted 1-path network routing feature 4 with gain g -> g x feature4"
    ws, bs = _zero()
    g = 2.75
    ws[0][0, 4] = g
    for k in (1, 2, 3, 4):
        ws[k][0, 0] = 1.0
    f = _feats()
    assert np.array_equal(mlp_predict(f, ws, bs), g * f[:, 4].astype(np.float64))


def test_rectifier_and_output_clamp():
    # a network computing max(0, f0 - f1) through one hidden path; the output
    # layer then negates: -max(0, f0 - f1) clamps to 0
    ws, bs = _zero()
    ws[0][0, 0], ws[0][0, 1] = 1.0, -1.0
    for k in (1, 2, 3):
        ws[k][0, 0] = 1.0
    ws[4][0, 0] = 1.0
    f = _feats(200, 9)
    want = np.maximum(f[:, 0].astype(np.float64) - f[:, 1], 0.0)
    assert np.array_equal(mlp_predict(f, ws, bs), want)
    ws[4][0, 0] = -1.0
    bs[4][0] = 0.5
    assert np.array_equal(mlp_predict(f, ws, bs), np.maximum(0.5 - want, 0.0))


def test_only_six_rule_scores_feed_the_model():
    # the feature vector is the six scores; ntok and ndropped do not enter
    ws, bs = mlp_weights(3)
    f = _feats()
    g = f.copy()
    g[:, 6] += 17
    g[:, 7] += 3
    assert np.array_equal(mlp_predict(f, ws, bs), mlp_predict(g, ws, bs))


def test_output_layer_homogeneity_and_determinism():
    ws, bs = mlp_weights(11)
    f = _feats(128, 2)
    u = mlp_predict(f, ws, bs)
    assert np.array_equal(u, mlp_predict(f, ws, bs))
    ws2 = [w.copy() for w in ws]
    bs2 = [b.copy() for b in bs]
    ws2[4] *= 4.0
    bs2[4] *= 4.0
    assert np.allclose(mlp_predict(f, ws2, bs2), 4.0 * u, rtol=1e-12, atol=0)


def test_abs_pass_bounds_the_output():
    ws, bs = mlp_weights(4)
    f = _feats(256, 3)
    assert (mlp_predict(f, ws, bs) <= mlp_abs_pass(f, ws, bs) + 1e-9).all()


def test_dims_match_the_paper():
    # P:620 / P:1547 "four layers of hidden size [100, 200, 200, 100]"; S:161 [6, ..., 1]
    assert DIMS == (6, 100, 200, 200, 100, 1)
    ws, bs = mlp_weights(1)
    assert [w.shape for w in ws] == [(100, 6), (200, 100), (200, 200), (100, 200), (1, 100)]


# ---------------------------------------------------------------- NEXT-2: training (oracle/mlp.py)
from oracle.mlp import ADAM_EPS, epoch_perm, mlp_grads, mlp_train_adam  # noqa: E402


def _small_net(seed=3, scale=0.2):
    rng = np.random.default_rng(seed)
    ws = [rng.normal(0, scale, (o, i)) for i, o in zip(DIMS[:-1], DIMS[1:])]
    bs = [rng.normal(0, scale, o) for o in DIMS[1:]]
    return ws, bs


def test_gradients_match_central_differences():
    # analytic gradient vs central finite differences, max relative error < 1e-4
    ws, bs = _small_net()
    f = _feats(8, seed=9)
    x = f[:, :6].astype(np.float64)
    y = np.linspace(3.0, 40.0, 8)
    _, gw, gb = mlp_grads(x, y, ws, bs)
    rng = np.random.default_rng(1)
    h = 1e-6
    worst = 0.0
    for _ in range(60):
        layer = int(rng.integers(0, 5))
        is_w = rng.random() < 0.7
        arr = ws[layer] if is_w else bs[layer]
        idx = tuple(int(rng.integers(0, d)) for d in arr.shape)
        g = (gw if is_w else gb)[layer][idx]
        old = arr[idx]
        arr[idx] = old + h
        lp = mlp_grads(x, y, ws, bs)[0]
        arr[idx] = old - h
        lm = mlp_grads(x, y, ws, bs)[0]
        arr[idx] = old
        fd = (lp - lm) / (2 * h)
        worst = max(worst, abs(fd - g) / max(1e-6, abs(fd), abs(g)))
    assert worst < 1e-4, worst


def test_first_adam_step_is_lr_times_sign():
    # t = 1 from zero moments: m^ = g, v^ = g^2, so the update is -lr * g / (|g| + eps)
    ws, bs = _small_net(seed=4)
    f = _feats(16, seed=2)
    y = np.full(16, 20.0)
    lr = 1e-3
    w1, b1, losses = mlp_train_adam(f, y, ws, bs, epochs=1, batch=16, lr=lr, seed=0)
    _, gw, gb = mlp_grads(f[:, :6].astype(np.float64), y, ws, bs)
    for w0, w, g in list(zip(ws, w1, gw)) + list(zip(bs, b1, gb)):
        np.testing.assert_allclose(w - w0, -lr * g / (np.abs(g) + ADAM_EPS), rtol=1e-9, atol=1e-15)
    assert len(losses) == 1


def test_zero_epochs_leave_the_model_unchanged():
    ws, bs = _small_net()
    w1, b1, losses = mlp_train_adam(_feats(10), np.ones(10), ws, bs, epochs=0, batch=4, lr=1e-4, seed=1)
    assert len(losses) == 0
    assert all(np.array_equal(a, b) for a, b in zip(ws, w1)) and all(np.array_equal(a, b) for a, b in zip(bs, b1))


def test_memorises_one_record():
    # one record repeated; after training |predict - target| shrinks >= 10x
    ws, bs = _small_net(seed=8, scale=0.1)
    f = np.tile(_feats(1, seed=4), (64, 1))
    y = np.full(64, 37.0)
    before = abs(mlp_predict(f[:1], ws, bs)[0] - 37.0)
    w1, b1, losses = mlp_train_adam(f, y, ws, bs, epochs=60, batch=16, lr=1e-3, seed=5)
    after = abs(mlp_predict(f[:1], w1, b1)[0] - 37.0)
    assert after * 10 <= before, (before, after)
    assert losses[-1] < losses[0]


def test_epoch_permutations_are_permutations():
    for n in (1, 2, 7, 64, 100, 1000, 65536):
        for e in range(4):
            a, b = epoch_perm(n, 123, e)
            order = (a * np.arange(n, dtype=np.int64) + b) % n
            assert np.array_equal(np.sort(order), np.arange(n))
