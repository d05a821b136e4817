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
