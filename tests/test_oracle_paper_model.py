"""Pins of the oracle's paper model (model 1: SURVEY.md §8f F1 + F2; readings P1-P7) against
closed forms, conservation laws and hand-evaluated cost values (-m "not gpu").

Dynamics: x = [p, v, q, w, T], u = Tdot. Costs (Eqs. 6-10).
A dropped term, a wrong sign or index (k vs k+1), a transposed mixer row or a missing clamp fails one of these.
"""
import math

import numpy as np
import pytest

import synth

G = 9.81


def _cfg(**over):
    return synth.get_config("c5s").replace(**over)


def _hover(cfg, g=G):
    x = np.zeros(17)
    x[6] = 1.0
    x[13:17] = cfg.mass * g / 4.0          # g/4 is exact in binary: sum T = m g exactly
    return x


def test_rotor_hover_is_an_equilibrium(oracle_mod):
    """SPEC.md:215 'at hover input ... all derivative components are zero'; RK4 then holds it exactly."""
    cfg = _cfg()
    oc = oracle_mod.make_cfg(cfg)
    x = _hover(cfg)
    np.testing.assert_array_equal(oracle_mod.rotor_deriv(oc, x, np.zeros(4)), 0.0)
    y = x
    for _ in range(50):
        y = oracle_mod.rotor_step(oc, y, np.zeros(4))
    np.testing.assert_array_equal(y, x)


def test_rotor_free_fall_closed_form(oracle_mod):
    """T = 0, level: z = -g t^2 / 2, v_z = -g t (RK4 is exact for constant acceleration)."""
    cfg = _cfg(dt=0.03)
    oc = oracle_mod.make_cfg(cfg)
    x = np.zeros(17)
    x[6] = 1.0
    for n in range(1, 34):
        x = oracle_mod.rotor_step(oc, x, np.zeros(4))
        t = n * cfg.dt
        assert x[2] == pytest.approx(-0.5 * G * t * t, abs=1e-12)
        assert x[5] == pytest.approx(-G * t, abs=1e-12)
    np.testing.assert_array_equal(x[[0, 1, 3, 4]], 0.0)


def test_rotor_thrust_ramp_is_cubic(oracle_mod):
    """Equal thrust rates a from T0 (no torque): T(t) = T0 + a t, z'' = 4 T(t)/m - g, so
    z(t) = (4 T0/m - g) t^2/2 + (4 a/m) t^3/6 exactly (RK4 is exact on this polynomial solution)."""
    cfg = _cfg(dt=0.03)
    oc = oracle_mod.make_cfg(cfg)
    T0, a = 2.0, 3.0
    x = np.zeros(17)
    x[6] = 1.0
    x[13:17] = T0
    for n in range(1, 21):
        x = oracle_mod.rotor_step(oc, x, np.full(4, a))
        t = n * cfg.dt
        z = (4 * T0 / cfg.mass - G) * t * t / 2 + 4 * a / cfg.mass * t ** 3 / 6
        assert x[2] == pytest.approx(z, abs=1e-11)
        np.testing.assert_allclose(x[13:17], T0 + a * t, atol=1e-12)
    np.testing.assert_array_equal(x[10:13], 0.0)
    np.testing.assert_array_equal(x[7:10], 0.0)


def test_rotor_mixer_diagonal_pairs_give_pure_yaw(oracle_mod):
    """SPEC.md:218 'diagonal-pair thrust imbalance -> wdot has only a z component' (X layout):
    T1 = T2 = a, T3 = T4 = b -> wdot = (0, 0, 2 kappa (a - b) / Jz); yaw then follows psi = alpha t^2 / 2."""
    cfg = _cfg(dt=0.01)
    oc = oracle_mod.make_cfg(cfg)
    a, b = 3.0, 2.0
    x = np.zeros(17)
    x[6] = 1.0
    x[13:17] = [a, a, b, b]
    xd = oracle_mod.rotor_deriv(oc, x, np.zeros(4))
    alpha = 2 * cfg.kappa * (a - b) / cfg.inertia[2]
    assert xd[10] == 0.0 and xd[11] == 0.0
    assert xd[12] == pytest.approx(alpha, rel=1e-15)
    for n in range(1, 11):
        x = oracle_mod.rotor_step(oc, x, np.zeros(4))
    t = 10 * cfg.dt
    psi = 2 * math.atan2(x[9], x[6])
    assert psi == pytest.approx(alpha * t * t / 2, rel=1e-7)
    np.testing.assert_allclose(x[7:9], 0.0, atol=1e-15)


@pytest.mark.parametrize("axis", [0, 1])
def test_rotor_mixer_roll_and_pitch_pairs(oracle_mod, axis):
    """Side pairs: roll (T2, T3 = b > T1, T4 = a) and pitch (T2, T4 = b > T1, T3 = a) torques
    2 d (b - a) about one body axis only, d = arm / sqrt(2), from the rotor positions of reading P2."""
    cfg = _cfg()
    oc = oracle_mod.make_cfg(cfg)
    a, b = 2.0, 2.5
    x = np.zeros(17)
    x[6] = 1.0
    x[13:17] = [a, b, b, a] if axis == 0 else [a, b, a, b]
    xd = oracle_mod.rotor_deriv(oc, x, np.zeros(4))
    d = cfg.arm / math.sqrt(2.0)
    want = np.zeros(3)
    want[axis] = 2 * d * (b - a) / cfg.inertia[axis]
    np.testing.assert_allclose(xd[10:13], want, rtol=1e-14, atol=1e-15)


def test_rotor_torque_free_rotation_conserves_energy_and_momentum(oracle_mod):
    """Equal thrusts give zero torque: Euler's torque-free equations conserve E = w.Jw / 2 and |J w|."""
    cfg = _cfg(dt=0.002, rate_max=100.0)
    oc = oracle_mod.make_cfg(cfg)
    J = np.array(cfg.inertia)
    x = _hover(cfg)
    x[10:13] = [3.0, -2.0, 4.0]
    E0, L0 = 0.5 * np.dot(x[10:13], J * x[10:13]), np.linalg.norm(J * x[10:13])
    for _ in range(500):
        x = oracle_mod.rotor_step(oc, x, np.zeros(4))
    w = x[10:13]
    assert 0.5 * np.dot(w, J * w) == pytest.approx(E0, rel=1e-8)
    assert np.linalg.norm(J * w) == pytest.approx(L0, rel=1e-8)
    assert abs(np.linalg.norm(x[6:10]) - 1.0) < 1e-14


def test_rotor_clamps(oracle_mod):
    """SPEC.md:234 'T = 9.9 N, Tdot = +10, dt = 0.03 -> T capped at 10.0'; clamps are idempotent; body
    rates are clamped to +-rate_max after the step."""
    cfg = _cfg(dt=0.03)
    oc = oracle_mod.make_cfg(cfg)
    x = _hover(cfg)
    x[13:17] = 9.9
    y = oracle_mod.rotor_step(oc, x, np.full(4, 10.0))
    np.testing.assert_array_equal(y[13:17], 10.0)
    y2 = oracle_mod.rotor_step(oc, y, np.full(4, 10.0))
    np.testing.assert_array_equal(y2[13:17], 10.0)
    x = _hover(cfg)
    x[13:17] = [0.0, 10.0, 10.0, 0.0]           # max roll torque
    x[10] = cfg.rate_max - 1e-3
    y = oracle_mod.rotor_step(oc, x, np.zeros(4))
    assert y[10] == cfg.rate_max
    x = _hover(cfg)
    x[13:17] = 0.05
    y = oracle_mod.rotor_step(oc, x, np.full(4, -10.0))
    np.testing.assert_array_equal(y[13:17], 0.0)


def _rollout(oracle_mod, cfg, x0, goal, U=None, noise=None, Tq=None, **oc_over):
    Ws, bs = synth.make_weights(cfg, seed=1)
    z = synth.make_latents(cfg)[0]
    Tq = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], np.float32) if Tq is None else Tq
    U = np.zeros((cfg.T, 4), np.float32) if U is None else U
    noise = np.zeros((cfg.T, 4)) if noise is None else noise
    oc = oracle_mod.make_cfg(cfg, **oc_over)
    return oracle_mod.rollout(oc, Ws, bs, z, Tq, np.asarray(x0, np.float32), np.asarray(goal, np.float32), U, noise)


def test_gate_progress_telescopes(oracle_mod):
    """Eq. 6 sums |p_{k+1} - p_wp|^2 - |p_k - p_wp|^2 over k = 0..K-1: it telescopes to
    |p_K - p_wp|^2 - |p_0 - p_wp|^2 (closed form; pins the k / k+1 pairing and the sign)."""
    cfg = _cfg(T=8)
    rng = np.random.default_rng(3)
    x0 = _hover(cfg)
    x0[3:6] = [2.0, -1.0, 0.5]
    goal = np.array([4.0, 1.0, -0.5])
    noise = rng.standard_normal((cfg.T, 4))
    r = _rollout(oracle_mod, cfg, x0, goal, noise=noise, q_vis=0.0, q_sdf=0.0, q_gate=1.0)
    st = r["states"]
    g = goal.astype(np.float32).astype(np.float64)
    want = np.sum((st[-1, :3] - g) ** 2) - np.sum((st[0, :3] - g) ** 2)
    assert r["J"] == pytest.approx(want, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("gate,yaw_deg,per_step", [((5, 0, 0), 0, 0.0), ((-5, 0, 0), 0, 2.0), ((0, 5, 0), 0, 1.0),
                                                   ((0, 5, 0), 90, 0.0), ((0, -5, 0), 90, 2.0),
                                                   ((3, 3, 1), 45, 0.0)])
def test_perception_alignment_hand_values(oracle_mod, gate, yaw_deg, per_step):
    """Eq. 7: 1 - cos(psi - psi_gate) at hover (the state never moves): facing the gate 0,
    facing away 2, perpendicular 1; yaw from q, line of sight in the horizontal plane."""
    cfg = _cfg(T=5)
    x0 = _hover(cfg)
    h = math.radians(yaw_deg) / 2
    x0[6], x0[9] = math.cos(h), math.sin(h)
    r = _rollout(oracle_mod, cfg, x0, gate, q_gate=0.0, q_sdf=0.0, q_vis=1.0)
    assert r["J"] == pytest.approx(cfg.T * per_step, abs=1e-6)


@pytest.mark.parametrize("d_safe,c,want", [(1.0, 0.5, 0.5), (0.3, 0.5, 0.0), (1.0, -0.25, 1.25)])
def test_sdf_hinge_on_the_analytic_gate(oracle_mod, d_safe, c, want):
    """Eq. 8 max(0, d_safe - s) with the analytic Gate-SDF substituted (Eq. 2: s = c at
    the gate centre): hovering at the query-frame origin costs Q_sdf (d_safe - c)^+ per step,
    and the queries are the states x_0..x_{K-1} (all at the origin)."""
    cfg = _cfg(T=4)
    x0 = _hover(cfg)
    r = _rollout(oracle_mod, cfg, x0, [5, 0, 0], q_gate=0.0, q_vis=0.0, q_sdf=3.0, d_safe=d_safe,
                 sdf_mode=1, gate_c=c)
    assert r["J"] == pytest.approx(cfg.T * 3.0 * want, abs=1e-7)
    np.testing.assert_allclose(r["sdf"][:, 0], c, atol=1e-7)
    np.testing.assert_allclose(r["queries"][:, :3], 0.0, atol=1e-7)


def test_sdf_queries_are_the_pre_step_states(oracle_mod):
    """The Eq. 8-9 sums run over k = 0..K-1 of the current trajectory: query k is at p_k (so query 0 is
    x0 itself), not at p_{k+1} as in the BASELINE configs (reading R7)."""
    cfg = _cfg(T=6)
    x0 = _hover(cfg)
    x0[0:3] = [0.3, -0.2, 0.1]
    x0[3:6] = [1.0, 0.5, -0.25]
    r = _rollout(oracle_mod, cfg, x0, [5, 0, 0], noise=np.random.default_rng(0).standard_normal((cfg.T, 4)))
    np.testing.assert_allclose(r["queries"][:, :3], r["states"][:-1, :3], atol=1e-6)
    np.testing.assert_allclose(r["queries"][:, 3], np.linalg.norm(r["states"][:-1, 3:6], axis=1), rtol=1e-12)


def test_thrust_rate_input_clamp(oracle_mod):
    """Table I Tdot in [-10, 10]: huge noise saturates u, so T_{k+1} = T_k +- 10 dt
    exactly (no torque: the same sign on all rotors)."""
    cfg = _cfg(T=3, dt=0.03)
    x0 = _hover(cfg)
    noise = np.full((cfg.T, 4), 1e3)
    r = _rollout(oracle_mod, cfg, x0, [5, 0, 0], noise=noise)
    np.testing.assert_allclose(r["states"][1:, 13], x0[13] + 10.0 * cfg.dt * np.arange(1, cfg.T + 1), atol=1e-12)


def test_paper_model_zero_noise_keeps_nominal(oracle_mod):
    """North_star invariant in the paper model: with zero noise every sample is the nominal rollout,
    so the weights are uniform and U* is unchanged."""
    cfg = _cfg()
    Ws, bs = synth.make_weights(cfg)
    inp = dict(z=synth.make_latents(cfg), Tq=synth.make_query_transforms(cfg), x0=synth.make_x0(cfg),
               goal=synth.make_goals(cfg), U=synth.make_nominal(cfg) + 0.5)
    noise = np.zeros((cfg.T, cfg.n_ctrl * cfg.K, 4))
    r = oracle_mod.step(oracle_mod.make_cfg(cfg), Ws, bs, inp["z"], inp["Tq"], inp["x0"], inp["goal"], inp["U"], noise)
    np.testing.assert_allclose(r["U_new"], inp["U"], atol=1e-12)
    assert np.all(r["J"] == r["J"][0, 0])
