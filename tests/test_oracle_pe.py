"""Pins of the oracle's positional encoding (reading E1) -m "not gpu":
hand values, the Pythagorean and double-angle identities between bands (a wrong frequency, order or sign
fails them), and the wiring of the features into layer 1 ahead of the latent."""
import math

import numpy as np
import pytest

import synth
from synth.configs import ACT_RELU, MLP_FP32


def test_pe_hand_values(oracle_mod):
    f = oracle_mod.pe(2, [0.0, 0.5, 0.25])
    np.testing.assert_allclose(f[:3], [0.0, 0.5, 0.25], atol=0)
    # band 0: sin(pi p), cos(pi p)
    np.testing.assert_allclose(f[3:6], [0.0, 1.0, math.sqrt(0.5)], atol=1e-15)
    np.testing.assert_allclose(f[6:9], [1.0, 0.0, math.sqrt(0.5)], atol=1e-15)
    # band 1: sin(2 pi p), cos(2 pi p)
    np.testing.assert_allclose(f[9:12], [0.0, 0.0, 1.0], atol=1e-15)
    np.testing.assert_allclose(f[12:15], [1.0, -1.0, 0.0], atol=1e-15)


def test_pe_band_identities(oracle_mod):
    rng = np.random.default_rng(0)
    for _ in range(50):
        p = rng.uniform(-8, 8, 3)
        f = oracle_mod.pe(4, p)
        assert f.shape == (27,)
        for i in range(4):
            s, c = f[3 + 6 * i:6 + 6 * i], f[6 + 6 * i:9 + 6 * i]
            np.testing.assert_allclose(s * s + c * c, 1.0, atol=1e-12)
            if i + 1 < 4:
                s2, c2 = f[9 + 6 * i:12 + 6 * i], f[12 + 6 * i:15 + 6 * i]
                np.testing.assert_allclose(s2, 2 * s * c, atol=1e-11)       # sin 2a = 2 sin a cos a
                np.testing.assert_allclose(c2, c * c - s * s, atol=1e-11)   # cos 2a = cos^2 a - sin^2 a
        # period 2 in p for every band
        np.testing.assert_allclose(oracle_mod.pe(4, p + 2.0)[3:], f[3:], atol=1e-12)


@pytest.mark.parametrize("feat", [0, 2, 3, 8, 14, 26])
def test_pe_features_feed_layer_one_before_the_latent(oracle_mod, feat):
    """A ReLU network that passes feature `feat` of [PE(p) | z] to the output (weight 1, bias +2 so the
    ReLU is the identity, output bias -2) returns that feature: the PE columns come first, in order."""
    cfg = synth.get_config("c1pes").replace(mlp_dtype=MLP_FP32, activation=ACT_RELU, hidden=8, n_hidden=2)
    dims = cfg.layer_dims
    Ws = [np.zeros((o, i), np.float32) for i, o in dims]
    bs = [np.zeros(o, np.float32) for _, o in dims]
    Ws[0][0, feat] = 1.0
    bs[0][0] = 2.0
    Ws[1][0, 0] = 1.0
    Ws[2][0, 0] = 1.0
    bs[2][0] = -2.0
    z = np.ones(cfg.latent_dim, np.float32)
    p = np.array([0.3, -0.7, 1.1])
    s = oracle_mod.mlp(oracle_mod.make_cfg(cfg), Ws, bs, z, p)
    assert s == pytest.approx(oracle_mod.pe(4, p)[feat], abs=1e-12)
    # a weight on the first latent column reads z, not a position feature
    Ws[0][0, :] = 0.0
    Ws[0][0, 27] = 1.0
    assert oracle_mod.mlp(oracle_mod.make_cfg(cfg), Ws, bs, z, p) == pytest.approx(1.0, abs=1e-12)
