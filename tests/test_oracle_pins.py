"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what pins it: a closed form, a library routine, a published known-answer vector, a
worked example (tests/golden/, cited), an invariant, or brute force. A plausible slip anywhere in the
oracle (dropped term, wrong sign/index, transposed operand) should fail at least one of these.
"""
import math
import os

import numpy as np
import pytest
import torch

import synth
from synth.configs import ACT_RELU, ACT_SILU, ACT_SOFTPLUS, MLP_BF16, MLP_FP32

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- RNG (reading R24)

def test_philox_known_answer_vectors(oracle_mod):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    for row in _golden("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row]
        out = oracle_mod.philox(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_noise_is_standard_normal(oracle_mod):
    """Box-Muller output: moments and a KS test against the normal CDF (scipy, library)."""
    from scipy import stats
    n = oracle_mod.noise(seed=1234, step=7, g0=0, nK=8192, T=4)
    flat = n.reshape(-1)
    assert abs(flat.mean()) < 0.01
    assert abs(flat.std() - 1.0) < 0.01
    assert stats.kstest(flat, "norm").pvalue > 1e-3
    # channels independent enough: correlation between channel 0 and 1 (a Box-Muller pair) ~ 0
    c = np.corrcoef(n[..., 0].reshape(-1), n[..., 1].reshape(-1))[0, 1]
    assert abs(c) < 0.02


def test_noise_counter_layout(oracle_mod):
    """Counter = (g, t, step_lo, step_hi): a shard at g0 reproduces the unsharded slice exactly."""
    full = oracle_mod.noise(seed=99, step=3, g0=0, nK=64, T=3)
    part = oracle_mod.noise(seed=99, step=3, g0=40, nK=24, T=3)
    np.testing.assert_array_equal(full[:, 40:], part)
    other = oracle_mod.noise(seed=99, step=4, g0=0, nK=64, T=3)
    assert not np.allclose(full, other)
    x = oracle_mod.philox([5, 2, 3, 0], [99, 0])
    u0 = ((int(x[0]) >> 9) + 0.5) / 2 ** 23
    u1 = ((int(x[1]) >> 9) + 0.5) / 2 ** 23
    g = oracle_mod.noise(seed=99, step=3, g0=5, nK=1, T=3)[2, 0]
    assert g[0] == pytest.approx(math.sqrt(-2 * math.log(u0)) * math.cos(2 * math.pi * u1), rel=1e-15)
    assert g[1] == pytest.approx(math.sqrt(-2 * math.log(u0)) * math.sin(2 * math.pi * u1), rel=1e-15)


# ---------------------------------------------------------------- bf16 rounding (R15)

def test_bf16_round_matches_torch(oracle_mod):
    """RNE to bf16 equals torch's float32 -> bfloat16 conversion (library routine)."""
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(2000) * 10 ** rng.uniform(-4, 4, 2000),
                           [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 0.0, 65504.0, 1e-30]])
    ref = torch.tensor(vals.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([oracle_mod.bf16_round(v) for v in vals.astype(np.float32)])
    np.testing.assert_array_equal(got, ref)


# ---------------------------------------------------------------- dynamics (CTBR per configs[0])

M, G = 1.0, 9.81


def _run(oracle_mod, x, u, dt, n):
    for _ in range(n):
        x = oracle_mod.rk4_step(x, u, dt, M, G)
    return x


def _hover_state():
    x = np.zeros(10)
    x[6] = 1.0
    return x


def test_hover_holds_exactly(oracle_mod):
    """north_star invariant: thrust m*g, zero rates, level attitude holds position exactly."""
    x = _hover_state()
    x[:3] = [0.3, -1.2, 2.0]
    y = _run(oracle_mod, x.copy(), [M * G, 0, 0, 0], 0.02, 500)
    np.testing.assert_array_equal(y, x)


def test_free_fall(oracle_mod):
    """Free fall 1 s from rest drops 4.905 m; RK4 is exact for constant acceleration."""
    y = _run(oracle_mod, _hover_state(), [0, 0, 0, 0], 0.02, 50)
    assert y[2] == pytest.approx(-0.5 * G * 1.0, abs=1e-12)
    assert y[5] == pytest.approx(-G * 1.0, abs=1e-12)


def test_constant_thrust_level(oracle_mod):
    """Level attitude, constant thrust c: z(t) = 1/2 (c/m - g) t^2 (closed form)."""
    c = 14.0
    y = _run(oracle_mod, _hover_state(), [c, 0, 0, 0], 0.01, 73)
    t = 0.73
    assert y[2] == pytest.approx(0.5 * (c / M - G) * t * t, abs=1e-12)
    assert abs(y[0]) < 1e-15 and abs(y[1]) < 1e-15


def test_pure_yaw_rate(oracle_mod):
    """Yaw rate w_z: q = (cos(wt/2), 0, 0, sin(wt/2)) (closed form, O(dt^4)); position held at hover."""
    w = 2.5
    y = _run(oracle_mod, _hover_state(), [M * G, 0, 0, w], 0.02, 60)
    t = 1.2
    np.testing.assert_allclose(y[6:10], [math.cos(w * t / 2), 0, 0, math.sin(w * t / 2)], atol=1e-9)
    np.testing.assert_allclose(y[0:6], 0, atol=1e-12)


def test_roll_rate_closed_form(oracle_mod):
    """Roll rate w_x from rest, thrust c: b3 = (0, -sin wt, cos wt);
    p_y = (c/m)(sin wt / w - t)/w, p_z = (c/m)(1 - cos wt)/w^2 - g t^2/2 (closed form)."""
    c, w = 12.0, 1.5
    y = _run(oracle_mod, _hover_state(), [c, w, 0, 0], 0.01, 100)
    t = 1.0
    py = (c / M) * (math.sin(w * t) / w - t) / w
    pz = (c / M) * (1 - math.cos(w * t)) / w ** 2 - 0.5 * G * t * t
    assert y[1] == pytest.approx(py, abs=1e-8)
    assert y[2] == pytest.approx(pz, abs=1e-8)
    assert y[0] == pytest.approx(0.0, abs=1e-14)
    np.testing.assert_allclose(y[6:10], [math.cos(w * t / 2), math.sin(w * t / 2), 0, 0], atol=1e-9)


def test_pitch_rate_closed_form(oracle_mod):
    """Pitch rate w_y from rest: b3 = (sin wt, 0, cos wt) -> p_x = (c/m)(t - sin wt / w)/w."""
    c, w = 12.0, -0.8
    y = _run(oracle_mod, _hover_state(), [c, 0, w, 0], 0.01, 100)
    t = 1.0
    px = (c / M) * (t - math.sin(w * t) / w) / w
    assert y[0] == pytest.approx(px, abs=1e-8)
    assert y[1] == pytest.approx(0.0, abs=1e-14)


def test_quaternion_norm_random_inputs(oracle_mod):
    rng = np.random.default_rng(1)
    x = _hover_state()
    for _ in range(2000):
        u = [rng.uniform(0, 40), *rng.uniform(-6, 6, 3)]
        x = oracle_mod.rk4_step(x, u, 0.02, M, G)
    assert abs(np.linalg.norm(x[6:10]) - 1.0) < 1e-12


# ---------------------------------------------------------------- SDF providers

def test_analytic_gate_sdf_golden(oracle_mod):
    """PAPER.md:66/:71 (Eqs. 1-2) values from tests/golden/gate_sdf_eq2.txt."""
    for c, ta, x, y, z, s in (map(float, r) for r in _golden("gate_sdf_eq2.txt")):
        assert oracle_mod.sdf_analytic(c, ta, [x, y, z]) == pytest.approx(s, abs=1e-4)
    # symmetry in x (hourglass) and in y <-> z (l_inf radial metric)
    assert oracle_mod.sdf_analytic(0.5, 0.3, [1.3, 0.2, -0.7]) == oracle_mod.sdf_analytic(0.5, 0.3, [-1.3, -0.7, 0.2])


def _torch_mlp(Ws, bs, z, p, act, bf16):
    """Reference forward with torch float64 Linear + torch activations (library routines)."""
    fn = {ACT_SOFTPLUS: torch.nn.functional.softplus, ACT_RELU: torch.relu, ACT_SILU: torch.nn.functional.silu}[act]

    def q(t):
        return t.to(torch.float32).to(torch.bfloat16).to(torch.float64) if bf16 else t

    x = torch.cat([torch.tensor(p, dtype=torch.float64), torch.tensor(z, dtype=torch.float64)])
    h = q(fn(torch.nn.functional.linear(x, torch.tensor(Ws[0], dtype=torch.float64), torch.tensor(bs[0], dtype=torch.float64))))
    for W, b in zip(Ws[1:-1], bs[1:-1]):
        h = q(fn(torch.nn.functional.linear(h, q(torch.tensor(W, dtype=torch.float64)), torch.tensor(b, dtype=torch.float64))))
    out = torch.nn.functional.linear(h, q(torch.tensor(Ws[-1], dtype=torch.float64)), torch.tensor(bs[-1], dtype=torch.float64))
    return float(out[0])


@pytest.mark.parametrize("name", ["c0", "c1s", "c2s"])
def test_mlp_matches_torch_reference(oracle_mod, name):
    """Oracle g_phi equals a torch float64 nn.Linear chain (softplus/relu/silu from torch) incl. bf16 rounding."""
    cfg = synth.get_config(name)
    Ws, bs = synth.make_weights(cfg, seed=5)
    z = synth.make_latents(cfg, seed=5)[0]
    oc = oracle_mod.make_cfg(cfg)
    rng = np.random.default_rng(2)
    for _ in range(8):
        p = rng.uniform(-3, 3, 3)
        got = oracle_mod.mlp(oc, Ws, bs, z, p)
        ref = _torch_mlp(Ws, bs, z, p, cfg.activation, cfg.mlp_dtype == MLP_BF16)
        # bf16 rounding decisions can differ by one ulp where fp64 sums land on a tie boundary:
        tol = 1e-9 if cfg.mlp_dtype == MLP_FP32 else 2e-2
        assert got == pytest.approx(ref, abs=tol)
        if cfg.mlp_dtype == MLP_FP32:
            assert got == pytest.approx(ref, rel=1e-12, abs=1e-12)


def test_constructed_relu_net_equals_eq2(oracle_mod):
    """The constructed exact ReLU network reproduces Eq. 2:
    exactly in fp64 mode, and within (tana+2) * ulp_bf16(max|coord|)/2 in the bf16 contract."""
    cfg = synth.get_config("c1s")
    Ws, bs = synth.constructed_gate_net(cfg, c=0.5, tana=0.375)
    z = np.zeros(cfg.latent_dim, np.float32)
    rng = np.random.default_rng(3)
    for bf16 in (0, 1):
        oc = oracle_mod.make_cfg(cfg.replace(mlp_dtype=MLP_BF16 if bf16 else MLP_FP32))
        for _ in range(200):
            p = rng.uniform(-3.5, 3.5, 3).astype(np.float32).astype(np.float64)
            s = oracle_mod.mlp(oc, Ws, bs, z, p)
            ref = oracle_mod.sdf_analytic(0.5, 0.375, p)
            if not bf16:
                assert s == pytest.approx(ref, abs=1e-12)
            else:
                m = np.max(np.abs(p))
                ulp = 2.0 ** (math.floor(math.log2(m)) - 7) if m > 0 else 0
                assert abs(s - ref) <= (0.375 + 2) * ulp / 2 + 1e-12


def test_latent_fold_identity(oracle_mod):
    """Folding W1[:,3:] z + b1 into a bias (A11) is algebraically the unfolded layer (fp64)."""
    cfg = synth.get_config("c0")
    Ws, bs = synth.make_weights(cfg, seed=8)
    z = synth.make_latents(cfg, seed=8)[0]
    oc = oracle_mod.make_cfg(cfg)
    W1 = Ws[0].astype(np.float64)
    b1f = W1[:, 3:] @ z.astype(np.float64) + bs[0]
    Wf = [np.concatenate([Ws[0][:, :3], np.zeros((cfg.hidden, cfg.latent_dim), np.float32)], 1)] + Ws[1:]
    bf = [b1f.astype(np.float64)] + bs[1:]
    p = np.array([0.4, -1.1, 2.2])
    a = oracle_mod.mlp(oc, Ws, bs, z, p)
    # bias rounded to fp32 by the wrapper: tolerance from that rounding only
    b = oracle_mod.mlp(oc, Wf, [x.astype(np.float32) for x in bf], z, p)
    assert a == pytest.approx(b, abs=1e-5)


# ---------------------------------------------------------------- costs (Eq. 10 structure, configs[0..1])

def _single(cfg, oracle_mod, **ov):
    oc = oracle_mod.make_cfg(cfg, **ov)
    Ws, bs = synth.make_weights(cfg, seed=1)
    return oc, Ws, bs


def test_cost_projections_at_hover(oracle_mod):
    """Zero noise at hover: the state never moves, so each term is a hand computation."""
    # gravity chosen exactly representable in fp32 so hover thrust float32(m*g) is an exact equilibrium
    cfg = synth.get_config("c0").replace(T=10, gravity=float(np.float32(9.81)))
    Ws, bs = synth.make_weights(cfg, seed=1)
    z = synth.make_latents(cfg)[0]
    Tq = synth.camera_transform()
    x0 = synth.make_x0(cfg)[0]
    U = synth.make_nominal(cfg)[0]
    goal = np.array([3.0, -1.0, 0.5], np.float32)
    nz = np.zeros((cfg.T, 4))
    zero = dict(w_goal=0.0, w_sdf=0.0, w_u=0.0, w_guide=0.0)
    r = oracle_mod.rollout(oracle_mod.make_cfg(cfg, **zero), Ws, bs, z, Tq, x0, goal, U, nz)
    assert r["J"] == 0.0
    r = oracle_mod.rollout(oracle_mod.make_cfg(cfg, **{**zero, "w_goal": 1.0}), Ws, bs, z, Tq, x0, goal, U, nz)
    assert r["J"] == pytest.approx(cfg.T * float(np.sum(goal.astype(np.float64) ** 2)), rel=1e-14)
    r = oracle_mod.rollout(oracle_mod.make_cfg(cfg, **{**zero, "w_u": 0.01}), Ws, bs, z, Tq, x0, goal, U, nz)
    assert r["J"] == pytest.approx(cfg.T * 0.01 * float(np.float32(cfg.gravity)) ** 2, rel=1e-14)
    # analytic SDF at the origin of the query frame: s = c -> 50 exp(-c/0.1) per step
    r = oracle_mod.rollout(oracle_mod.make_cfg(cfg, sdf_mode=1, gate_c=0.5, **{**zero, "w_sdf": 50.0}),
                           Ws, bs, z, Tq, x0, goal, U, nz)
    assert r["J"] == pytest.approx(cfg.T * 50.0 * math.exp(-5.0), rel=1e-13)
    # queries are the transformed positions: all at the origin
    np.testing.assert_array_equal(r["queries"][:, :4], 0.0)


def test_guidance_term_sign_and_frame(oracle_mod):
    """-w_guide * grad(s).v via a forward difference along R v/|v| (R11, R12). With the analytic
    Gate-SDF (piecewise linear, no kink within h) the difference is exact: moving along world +x with
    the R13 camera means moving along +z_c, where s = c + |x_c| tana - |z_c| has slope -1 -> cost +3/step."""
    cfg = synth.get_config("c1s").replace(T=1)
    Ws, bs = synth.make_weights(cfg, seed=1)
    z = synth.make_latents(cfg)[0]
    Tq = synth.camera_transform()
    x0 = np.array([1.0, 0.1, 0.05, 3.0, 0, 0, 1, 0, 0, 0], np.float32)
    U = synth.make_nominal(cfg)[0]
    oc = oracle_mod.make_cfg(cfg, sdf_mode=1, gate_c=0.5, gate_tana=0.375, w_goal=0.0, w_sdf=0.0, w_u=0.0,
                             w_guide=1.0)
    r = oracle_mod.rollout(oc, Ws, bs, z, Tq, x0, np.zeros(3, np.float32), U, np.zeros((1, 4)))
    assert r["J"] == pytest.approx(3.0, abs=1e-9)
    q = r["queries"][0]
    np.testing.assert_allclose(q[:3], [-0.1, -0.05, 1.0 + 3.0 * cfg.dt], atol=1e-7)
    assert q[3] == pytest.approx(3.0)
    np.testing.assert_allclose(q[4:7], q[:3] + [0, 0, cfg.fd_h], atol=1e-12)


def test_sdf_exp_clamp(oracle_mod):
    """R9: the exponent is clamped at sdf_exp_max, so deeply negative SDF stays finite."""
    cfg = synth.get_config("c0").replace(T=1)
    Ws, bs = synth.make_weights(cfg, seed=1)
    oc = oracle_mod.make_cfg(cfg, sdf_mode=1, gate_c=-100.0, w_goal=0.0, w_u=0.0)
    r = oracle_mod.rollout(oc, Ws, bs, np.zeros(cfg.latent_dim, np.float32), synth.camera_transform(),
                           synth.make_x0(cfg)[0], np.zeros(3, np.float32), synth.make_nominal(cfg)[0], np.zeros((1, 4)))
    assert r["J"] == pytest.approx(50.0 * math.exp(80.0), rel=1e-14)


def test_input_clamp(oracle_mod):
    """R5: huge noise saturates at the box [0, 4mg] x [-6, 6]^3: with max thrust and max rates the
    first step equals an explicit RK4 step with the clamped input."""
    cfg = synth.get_config("c0").replace(T=1)
    Ws, bs = synth.make_weights(cfg, seed=1)
    oc = oracle_mod.make_cfg(cfg)
    x0 = synth.make_x0(cfg)[0]
    r = oracle_mod.rollout(oc, Ws, bs, synth.make_latents(cfg)[0], synth.camera_transform(), x0,
                           np.zeros(3, np.float32), synth.make_nominal(cfg)[0], np.array([[1e6, 1e6, -1e6, 1e6]]))
    y = oracle_mod.rk4_step(x0, [4 * M * G, 6, -6, 6], cfg.dt, M, G)
    np.testing.assert_array_equal(r["states"][1], y)


# ---------------------------------------------------------------- softmin (Eq. 5)

def test_softmin_golden(oracle_mod):
    """tests/golden/softmin_spec.txt."""
    cfg = synth.get_config("c0").replace(T=2, K=2)
    U = np.zeros((2, 4), np.float32)
    nz = np.zeros((2, 2, 4))
    nz[:, 1, 0] = 1.0   # sample 1 differs in thrust by sigma*1 = 2 N
    U[:, 0] = 10.0
    for j0, j1, lam, w1 in (map(float, r) for r in _golden("softmin_spec.txt")):
        oc = oracle_mod.make_cfg(cfg, lam=lam)
        Un, jm, S, V, ess, flag = oracle_mod.softmin(oc, [j0, j1], U, nz)
        assert flag == 0
        assert V[0, 0] / S / 2.0 == pytest.approx(w1, rel=1e-12, abs=1e-300)
        assert (Un[0, 0] - 10.0) / 2.0 == pytest.approx(w1, abs=1e-15)


def test_softmin_matches_scipy(oracle_mod):
    """w = softmax(-J/lambda) (scipy.special.softmax, library); U_new = U + sum_k w_k (u_k - U); ESS."""
    from scipy.special import softmax
    cfg = synth.get_config("c0").replace(K=50, T=3)
    rng = np.random.default_rng(4)
    J = rng.uniform(0, 5, cfg.K)
    U = synth.make_nominal(cfg)[0] + rng.uniform(-1, 1, (cfg.T, 4)).astype(np.float32)
    nz = rng.standard_normal((cfg.T, cfg.K, 4))
    oc = oracle_mod.make_cfg(cfg, lam=0.7)
    Un, jm, S, V, ess, flag = oracle_mod.softmin(oc, J, U, nz)
    w = softmax(-J / 0.7)
    lo, hi = np.array(cfg.u_lo), np.array(cfg.u_hi)
    u = np.clip(U[None].astype(np.float64) + np.array(cfg.sigma) * nz.transpose(1, 0, 2), lo, hi)
    ref = U.astype(np.float64) + np.einsum("k,ktc->tc", w, u - U[None].astype(np.float64))
    np.testing.assert_allclose(Un, ref, rtol=1e-12, atol=1e-12)
    assert jm == J.min()
    assert ess == pytest.approx(1.0 / np.sum(w ** 2), rel=1e-10)
    # convexity: every channel lies within [min_k u, max_k u]
    assert np.all(Un >= u.min(0) - 1e-12) and np.all(Un <= u.max(0) + 1e-12)
    # shift invariance
    Un2 = oracle_mod.softmin(oc, J + 7.3, U, nz)[0]
    np.testing.assert_allclose(Un2, Un, rtol=1e-12, atol=1e-12)


def test_softmin_lambda_to_zero_selects_argmin(oracle_mod):
    cfg = synth.get_config("c0").replace(K=40, T=2)
    rng = np.random.default_rng(5)
    J = rng.permutation(np.arange(40) * 0.01 + 1.0)
    U = synth.make_nominal(cfg)[0]
    nz = rng.standard_normal((cfg.T, cfg.K, 4)) * 0.1
    oc = oracle_mod.make_cfg(cfg, lam=1e-6)
    Un = oracle_mod.softmin(oc, J, U, nz)[0]
    kb = int(np.argmin(J))
    ub = np.clip(U + np.array(cfg.sigma) * nz[:, kb], cfg.u_lo, cfg.u_hi)
    np.testing.assert_allclose(Un, ub, atol=1e-9)


def test_softmin_all_infinite_flags(oracle_mod):
    cfg = synth.get_config("c0").replace(K=4, T=2)
    U = synth.make_nominal(cfg)[0]
    Un, jm, S, V, ess, flag = oracle_mod.softmin(oracle_mod.make_cfg(cfg), [np.inf] * 4, U, np.ones((2, 4, 4)))
    assert flag == 1
    np.testing.assert_array_equal(Un, U)


def test_zero_noise_reproduces_nominal(oracle_mod):
    """north_star invariant: sigma = 0 -> every rollout is the nominal rollout, weights 1/K, U_new = U."""
    cfg = synth.get_config("c1s").replace(K=16, T=4)
    Ws, bs = synth.make_weights(cfg)
    oc = oracle_mod.make_cfg(cfg)
    for i in range(4):
        oc.sigma[i] = 0.0
    U = synth.make_nominal(cfg)
    U[0, :, 0] += np.float32(1.5)  # climb, so the rollout actually moves
    out = oracle_mod.step(oc, Ws, bs, synth.make_latents(cfg), synth.make_query_transforms(cfg), synth.make_x0(cfg),
                          synth.make_goals(cfg), U, synth.make_noise(cfg))
    assert np.all(out["J"][0] == out["J"][0, 0])
    assert out["ess"][0] == pytest.approx(cfg.K)
    np.testing.assert_array_equal(out["U_new"][0], U[0])


def test_brute_force_enumeration(oracle_mod):
    """north_star invariant: T = 3, zero rates, thrust in {0.5mg, mg, 1.5mg} per step: K = 27 samples
    enumerate every sequence. With only the goal term, the vertical motion is piecewise-constant
    acceleration, so each cost is a closed form evaluated here independently (z += v dt + a dt^2/2).
    lambda = 1e-6 makes U_new equal the brute-force argmin sequence."""
    cfg = synth.get_config("c0").replace(K=27, T=3)
    mg = M * G
    levels = [0.5 * mg, mg, 1.5 * mg]
    seqs = [(a, b, c) for a in levels for b in levels for c in levels]
    U = synth.make_nominal(cfg)[0]
    nz = np.zeros((3, 27, 4))
    for k, s in enumerate(seqs):
        for t in range(3):
            nz[t, k, 0] = (s[t] - float(U[t, 0])) / cfg.sigma[0]
    goal = np.array([0.0, 0.0, 0.01], np.float32)
    dt = cfg.dt
    costs = []
    for s in seqs:
        z = v = 0.0
        J = 0.0
        for t in range(3):
            a = s[t] / M - G
            z, v = z + v * dt + 0.5 * a * dt * dt, v + a * dt
            J += (z - float(goal[2])) ** 2
        costs.append(J)
    best = int(np.argmin(costs))
    oc = oracle_mod.make_cfg(cfg, lam=1e-9, w_sdf=0.0, w_u=0.0)
    Ws, bs = synth.make_weights(cfg)
    out = oracle_mod.step(oc, Ws, bs, synth.make_latents(cfg), synth.make_query_transforms(cfg),
                          synth.make_x0(cfg), goal[None], U[None], nz)
    np.testing.assert_allclose(out["J"][0], costs, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(out["U_new"][0, :, 0], seqs[best], rtol=1e-12)
    np.testing.assert_allclose(out["U_new"][0, :, 1:], 0.0, atol=0)


def test_shard_combine_equals_unsharded(oracle_mod):
    """configs[3] combine (log-sum-exp of per-shard records) equals the single softmin (identity)."""
    cfg = synth.get_config("c0").replace(K=96, T=4)
    rng = np.random.default_rng(6)
    J = rng.uniform(10, 30, cfg.K)
    J[7] = np.inf
    U = synth.make_nominal(cfg)[0]
    nz = rng.standard_normal((cfg.T, cfg.K, 4))
    oc = oracle_mod.make_cfg(cfg, lam=0.5)
    ref = oracle_mod.softmin(oc, J, U, nz)[0]
    for R in (2, 3, 4, 8):
        Kr = cfg.K // R
        recs = np.stack([oracle_mod.shard_record(oc, J[r * Kr:(r + 1) * Kr], U,
                                                 np.ascontiguousarray(nz[:, r * Kr:(r + 1) * Kr]))
                         for r in range(R)])
        got, flag = oracle_mod.combine(oc, recs, U)
        assert flag == 0
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_shift(oracle_mod):
    U = np.arange(2 * 3 * 4, dtype=np.float32).reshape(2, 3, 4)
    S = oracle_mod.shift(U)
    np.testing.assert_array_equal(S[:, 0], U[:, 1])
    np.testing.assert_array_equal(S[:, 1], U[:, 2])
    np.testing.assert_array_equal(S[:, 2], U[:, 2])


def test_step_deterministic(oracle_mod):
    """Parallel (OpenMP) evaluation is bitwise deterministic (SPEC.md:774 criterion)."""
    cfg = synth.get_config("c4s")
    Ws, bs = synth.make_weights(cfg)
    args = (synth.make_latents(cfg), synth.make_query_transforms(cfg), synth.make_x0(cfg), synth.make_goals(cfg),
            synth.make_nominal(cfg), synth.make_noise(cfg))
    oc = oracle_mod.make_cfg(cfg)
    a = oracle_mod.step(oc, Ws, bs, *args)
    b = oracle_mod.step(oc, Ws, bs, *args)
    np.testing.assert_array_equal(a["J"], b["J"])
    np.testing.assert_array_equal(a["U_new"], b["U_new"])


def test_gate_pose_transform_puts_gate_at_origin(oracle_mod):
    """configs[4] (R22): T_q maps each drone's gate centre to the query-frame origin, where the
    analytic Gate-SDF equals c (Eq. 2) and its opening is the gate plane x = 0."""
    cfg = synth.get_config("c4s")
    Tq = synth.make_query_transforms(cfg).astype(np.float64)
    pos = synth.make_goals(cfg).astype(np.float64)
    for i in range(cfg.n_ctrl):
        R = Tq[i, :9].reshape(3, 3)
        pc = R @ pos[i] + Tq[i, 9:]
        np.testing.assert_allclose(pc, 0, atol=1e-5)
        np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-6)
        assert oracle_mod.sdf_analytic(0.5, 0.375, pc) == pytest.approx(0.5, abs=1e-5)
