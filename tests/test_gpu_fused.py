"""GPU parity of the fused rollout (-m gpu): with FUSE the SDF-MLP kernels (kernel_mlp_h128.cu at H = 128,
kernel_mlp_tc.cu's CTA pairs at H = 256) run the CTBR rollout themselves (rows never reach HBM). It must give the step of the unfused path (k_rollout then the
SDF-MLP kernel on the stored rows): the same noise, partial costs, SDF stage terms, costs and update, and the
oracle's costs and update within the north_star tolerances."""
import numpy as np
import pytest

import oracle
import synth
from tests import gpu_helpers as gh

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_07199_b200 import build
    build.build()
    oracle.build()


def _run(cfg, fused, monkeypatch, noise_mode, step=3, noise=None):
    from paper_2603_07199_b200 import Controller
    monkeypatch.setenv("MPPI_FUSED", "1" if fused else "0")
    Ws, bs = synth.make_weights(cfg)
    c = Controller(cfg, noise_mode=noise_mode)
    assert c.fused_rollout() == fused
    assert c.kernels_per_step() == (2 if fused else 3)
    c.set_sdf_weights(Ws, bs)
    c.set_latent(synth.make_latents(cfg), synth.make_query_transforms(cfg))
    c.set_nominal(synth.make_nominal(cfg))
    if noise is not None:
        c.set_noise(noise)
    c.step(synth.make_x0(cfg), synth.make_goals(cfg), step)
    U, u0 = c.get_controls(allow_nonfinite=True)
    out = dict(U=U, u0=u0, J=c.debug("costs"), noise=c.debug("noise"), terms=c.debug("terms"),
               partial=c.debug("partial"), diag=c.diagnostics())
    if fused:
        from paper_2603_07199_b200 import MppiError
        with pytest.raises(MppiError):
            c.debug("queries")      # the fused step stores no query rows
    c.close()
    return out


@pytest.mark.parametrize("name,over", [("c4s", {}), ("c4s", {"n_ctrl": 5, "K": 128, "T": 7}),
                                       ("c3s", {}), ("c2s", {"n_ctrl": 3, "K": 256, "T": 5})])
@pytest.mark.parametrize("noise_mode", ["device", "external"])
def test_fused_rollout_equals_unfused(monkeypatch, name, over, noise_mode):
    cfg = synth.get_config(name, **over)
    noise = synth.make_noise(cfg) if noise_mode == "external" else None
    a = _run(cfg, False, monkeypatch, noise_mode, noise=noise)
    b = _run(cfg, True, monkeypatch, noise_mode, noise=noise)
    np.testing.assert_array_equal(b["noise"], a["noise"])
    # the same rollout code (rollout_dev.cuh) on the same inputs: equal up to fp32 contraction differences
    np.testing.assert_allclose(b["partial"], a["partial"], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(b["terms"], a["terms"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(b["J"], a["J"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(b["U"], a["U"], atol=1e-5)


@pytest.mark.parametrize("name,over", [("c4s", {"n_ctrl": 4, "K": 128, "T": 6}), ("c3s", {"n_ctrl": 2, "T": 5})])
def test_fused_rollout_matches_oracle(monkeypatch, name, over):
    """Costs and update of the fused step against the oracle on the same external noise (staged where the
    fused path allows: J per sample, then U* by the R26 rule and the softmin property)."""
    cfg = synth.get_config(name, **over)
    inp = dict(z=synth.make_latents(cfg), Tq=synth.make_query_transforms(cfg), x0=synth.make_x0(cfg),
               goal=synth.make_goals(cfg), U=synth.make_nominal(cfg), noise=synth.make_noise(cfg))
    Ws, bs = synth.make_weights(cfg)
    got = _run(cfg, True, monkeypatch, "external", step=0, noise=inp["noise"])
    ref = gh.run_oracle(cfg, Ws, bs, inp)
    tolJ = gh.cost_tol(cfg, ref, gh.ABS_SDF_BF16)
    J = got["J"].astype(np.float64)
    assert np.all(np.abs(J - ref["J"]) <= tolJ), np.abs(J - ref["J"]).max()
    for b in range(cfg.n_ctrl):
        noise_b = np.asarray(inp["noise"])[:, b * cfg.K:(b + 1) * cfg.K]
        prop = gh.softmin_property(cfg, inp["U"][b], noise_b, J[b])
        assert np.abs(got["U"][b] - prop).max() <= gh.ABS_U
        d = np.abs(got["U"][b] - ref["U_new"][b]).max()
        if d > gh.ABS_U:
            order = np.argsort(ref["J"][b])
            assert ref["J"][b][order[1]] - ref["J"][b][order[0]] <= tolJ[b][order[0]] + tolJ[b][order[1]], d


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_fused_full_size_sampled(monkeypatch, name):
    """configs[4] / configs[3] at full size (fused, device noise): sampled rollouts recomputed one by one by the
    oracle (global Philox counters) against the GPU's costs; the update by the softmin property on the GPU's
    own costs."""
    from paper_2603_07199_b200 import Controller
    monkeypatch.setenv("MPPI_FUSED", "1")
    cfg = synth.get_config(name)
    Ws, bs = synth.make_weights(cfg)
    z, Tq, x0, goal, U = (synth.make_latents(cfg), synth.make_query_transforms(cfg), synth.make_x0(cfg),
                          synth.make_goals(cfg), synth.make_nominal(cfg))
    c = Controller(cfg, noise_mode="device")
    assert c.fused_rollout()
    c.set_sdf_weights(Ws, bs)
    c.set_latent(z, Tq)
    c.set_nominal(U)
    c.step(x0, goal, 7)
    Ug, _ = c.get_controls()
    J = c.debug("costs").astype(np.float64)
    noise = c.debug("noise")
    oc = oracle.make_cfg(cfg)
    rng = np.random.default_rng(3)
    for b in rng.choice(cfg.n_ctrl, size=min(cfg.n_ctrl, 3), replace=False):
        for k in rng.choice(cfg.K, size=4, replace=False):
            nz = oracle.noise(cfg.seed, 7, int(b) * cfg.K + int(k), 1, cfg.T)[:, 0]
            r = oracle.rollout(oc, Ws, bs, z[b], Tq[b], x0[b], goal[b], U[b], nz)
            ref = {"queries": r["queries"][None, None], "sdf": r["sdf"][None, None], "stage": r["stage"][None, None]}
            tol = gh.cost_tol(cfg, ref, gh.ABS_SDF_BF16)[0, 0]
            assert abs(J[b, k] - r["J"]) <= tol, (b, k, J[b, k], r["J"], tol)
        prop = gh.softmin_property(cfg, U[b], noise[:, b * cfg.K:(b + 1) * cfg.K].astype(np.float64), J[b])
        assert np.abs(Ug[b] - prop).max() <= gh.ABS_U
    c.close()
