"""Shared setup for the -m gpu parity tests: build a Controller and the oracle on the same seeded
synthetic inputs (synth/), with tolerances from north_star / DESIGN.md §Tolerances."""
from __future__ import annotations

import numpy as np

import oracle
import synth

# north_star: 1e-5 relative on fp32 states and costs (+ abs floor, reading R27), 2e-2 absolute on
# bf16 SDF values, 1e-3 on the updated controls.
REL_STATE, ABS_STATE = 1e-5, 1e-6
ABS_SDF_BF16 = 2e-2
ABS_U = 1e-3


def setup(name, noise_mode="external", step=0, seed=0, weights=None, **over):
    from paper_2603_07199_b200 import Controller
    cfg = synth.get_config(name, seed=seed, **over)
    Ws, bs = weights if weights is not None else synth.make_weights(cfg)
    inp = dict(z=synth.make_latents(cfg), Tq=synth.make_query_transforms(cfg), x0=synth.make_x0(cfg),
               goal=synth.make_goals(cfg), U=synth.make_nominal(cfg))
    ctrl = Controller(cfg, noise_mode=noise_mode, debug_outputs=True)
    ctrl.set_sdf_weights(Ws, bs)
    ctrl.set_latent(inp["z"], inp["Tq"])
    ctrl.set_nominal(inp["U"])
    if noise_mode == "external":
        inp["noise"] = synth.make_noise(cfg, step=step)
        ctrl.set_noise(inp["noise"])
    else:
        inp["noise"] = oracle.noise(cfg.seed, step, 0, cfg.n_ctrl * cfg.K, cfg.T)
    return cfg, Ws, bs, inp, ctrl


def run_oracle(cfg, Ws, bs, inp, **ov):
    oc = oracle.make_cfg(cfg, **ov)
    return oracle.step(oc, Ws, bs, inp["z"], inp["Tq"], inp["x0"], inp["goal"], inp["U"], inp["noise"])


# absolute floor of fp32 rollout states: v_z integrates c/m - g, a cancellation with rounding error
# ~ulp(g)/2 per RK4 stage, i.e. <= 1e-6 m/s over a 1 s horizon
ABS_VEL = 1e-6


def check_queries(cfg, q_gpu, q_ref):
    """Query rows vs the oracle. p_c and |v|: 1e-5 relative + 1e-6 absolute (north_star states).
    FD row p_c + h v/|v|: the direction inherits the velocity's error divided by |v|, so its
    tolerance is h * 2 (1e-5 |v| + ABS_VEL) / |v| (conditioning of the normalisation; exact 0 row
    below |v| = 1e-6 on both sides). Returns (ok, worst excess)."""
    a = np.asarray(q_gpu, np.float64)
    b = np.asarray(q_ref, np.float64)
    d = np.abs(a - b)
    tol = REL_STATE * np.abs(b) + ABS_STATE
    tol[..., 3] = REL_STATE * np.abs(b[..., 3]) + ABS_VEL
    nv = np.maximum(b[..., 3:4], 1e-6)
    dirtol = cfg.fd_h * 2 * (REL_STATE * nv + ABS_VEL) / nv
    tol[..., 4:7] = tol[..., 0:3] + dirtol
    m = 7 if cfg.fd else 4      # without guidance there is no FD row on the GPU
    worst = (d[..., :m] - tol[..., :m]).max()
    return worst <= 0, worst


def sdf_tol(cfg, s_ref):
    if cfg.mlp_dtype == 0:
        # fp32 MLP fed fp32 query positions (rel 1e-5): |grad s| = O(1) -> same order absolute
        return 1e-5 * np.abs(s_ref) + 1e-5
    return np.full_like(s_ref, ABS_SDF_BF16)


def cost_tol(cfg, ref, tol_s):
    """Propagate the SDF tolerance through the stage cost:
    |dJ| <= 1e-5 sum_t |c_t| + sum_t [w_sdf/scale e^{-s/scale} + 2 w_guide |v| / h] tol_s."""
    if getattr(cfg, "model", 0) == 1:
        # paper model: the hinge q_sdf max(0, d_safe - s) is 1-Lipschitz in s
        return 1e-5 * np.abs(ref["stage"]).sum(-1) + (cfg.q_sdf * np.broadcast_to(tol_s, ref["stage"].shape)).sum(-1) + 1e-6
    s0 = ref["sdf"][..., 0]
    nv = ref["queries"][..., 3]
    e = np.exp(np.minimum(-s0 / cfg.sdf_scale, cfg.sdf_exp_max))
    per = cfg.w_sdf / cfg.sdf_scale * e * tol_s + (2 * cfg.w_guide * nv / cfg.fd_h) * tol_s
    return 1e-5 * np.abs(ref["stage"]).sum(-1) + per.sum(-1) + 1e-6


def gpu_queries_like_oracle(q):
    """GPU rows [n][T][K][rps][4] -> oracle layout [n][K][T][8] (p_c, |v|, p_c', 0)."""
    n, T, K, r, _ = q.shape
    out = np.zeros((n, K, T, 8), np.float64)
    qq = q.transpose(0, 2, 1, 3, 4)
    out[..., 0:4] = qq[..., 0, :]
    if r == 2:
        out[..., 4:7] = qq[..., 1, :3]
    return out


def gpu_sdf_like_oracle(s):
    n, T, K, r = s.shape
    out = np.zeros((n, K, T, 2))
    ss = s.transpose(0, 2, 1, 3)
    out[..., 0] = ss[..., 0]
    out[..., 1] = ss[..., 1] if r == 2 else ss[..., 0]
    return out


def softmin_property(cfg, U, noise, J):
    """U + sum_k softmax(-J/lambda)_k (clamp(U + sigma n_k) - U) for one controller, in float64 numpy
    (validity check of the update given the GPU's own costs)."""
    from scipy.special import softmax
    w = softmax(-np.asarray(J, np.float64) / cfg.lam)
    u = np.clip(U[None].astype(np.float64) + np.array(cfg.sigma) * noise.transpose(1, 0, 2), cfg.u_lo, cfg.u_hi)
    return U.astype(np.float64) + np.einsum("k,ktc->tc", w, u - U[None].astype(np.float64))
