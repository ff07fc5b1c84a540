"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/mppi_oracle.c (plain C, fp64, OpenMP over samples). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may import this.
The product path (paper_2603_07199_b200/) never imports it and shares no code with it.

Every function here is marshalling only; the arithmetic and its paper citations live in the C file.
Parity unpinned: oracle_noise against the paper (the paper names no generator; the
C implementation is pinned to the Random123 Philox4x32-10 known-answer vectors instead).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mppi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ACT = {"softplus": 0, "relu": 1, "silu": 2}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OracleCfg(C.Structure):
    _fields_ = [
        ("n_ctrl", C.c_int32), ("K", C.c_int32), ("T", C.c_int32),
        ("dt", C.c_double), ("lam", C.c_double), ("mass", C.c_double), ("gravity", C.c_double),
        ("u_lo", C.c_double * 4), ("u_hi", C.c_double * 4), ("sigma", C.c_double * 4),
        ("w_goal", C.c_double), ("w_sdf", C.c_double), ("sdf_scale", C.c_double),
        ("sdf_exp_max", C.c_double), ("w_u", C.c_double), ("w_guide", C.c_double), ("fd_h", C.c_double),
        ("latent_dim", C.c_int32), ("hidden", C.c_int32), ("n_hidden", C.c_int32),
        ("activation", C.c_int32), ("mlp_bf16", C.c_int32),
        ("sdf_mode", C.c_int32), ("gate_c", C.c_double), ("gate_tana", C.c_double),
        ("model", C.c_int32), ("arm", C.c_double), ("kappa", C.c_double), ("inertia", C.c_double * 3),
        ("thrust_max", C.c_double), ("rate_max", C.c_double),
        ("q_gate", C.c_double), ("q_vis", C.c_double), ("q_sdf", C.c_double), ("d_safe", C.c_double),
        ("pe_bands", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, f, i32, i64, u64 = C.c_double, C.c_float, C.c_int32, C.c_int64, C.c_uint64
        P = C.POINTER
        _lib.oracle_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        _lib.oracle_noise.argtypes = [u64, u64, i64, i32, i32, P(d)]
        _lib.oracle_bf16_round.argtypes = [d]
        _lib.oracle_bf16_round.restype = d
        _lib.oracle_rk4_step.argtypes = [P(d), P(d), d, d, d, P(d)]
        _lib.oracle_mlp.argtypes = [P(OracleCfg), P(f), P(f), P(f), P(d)]
        _lib.oracle_mlp.restype = d
        _lib.oracle_mlp_trace.argtypes = [P(OracleCfg), P(f), P(f), P(f), P(d), P(d)]
        _lib.oracle_mlp_trace.restype = d
        _lib.oracle_sdf_analytic.argtypes = [d, d, P(d)]
        _lib.oracle_sdf_analytic.restype = d
        _lib.oracle_sdf_rows.argtypes = [P(OracleCfg), P(f), P(f), P(f), P(f), i64, P(d)]
        _lib.oracle_rollout.argtypes = [P(OracleCfg), P(f), P(f), P(f), P(f), P(f), P(f), P(f), P(d), i64,
                                        P(d), P(d), P(d), P(d)]
        _lib.oracle_rollout.restype = d
        _lib.oracle_softmin.argtypes = [P(OracleCfg), i32, P(d), P(f), P(d), i64, P(d), P(d), P(d), P(d), P(d)]
        _lib.oracle_softmin.restype = C.c_int
        _lib.oracle_shard_record.argtypes = [P(OracleCfg), i32, P(d), P(f), P(d), i64, P(d)]
        _lib.oracle_shard_record.restype = C.c_int
        _lib.oracle_combine.argtypes = [P(OracleCfg), i32, P(d), P(f), P(d)]
        _lib.oracle_combine.restype = C.c_int
        _lib.oracle_step.argtypes = [P(OracleCfg), P(f), P(f), P(f), P(f), P(f), P(f), P(f), P(d),
                                     P(d), P(d), P(d), P(d), P(d), P(d), P(d), P(d), P(d), P(i32)]
        _lib.oracle_shift.argtypes = [i32, i32, P(f)]
        _lib.oracle_rotor_deriv.argtypes = [P(OracleCfg), P(d), P(d), P(d)]
        _lib.oracle_rotor_step.argtypes = [P(OracleCfg), P(d), P(d), P(d)]
        _lib.oracle_pe.argtypes = [C.c_int, P(d), P(d)]
    return _lib


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def make_cfg(cfg, sdf_mode: int | None = None, gate_c: float | None = None, gate_tana: float | None = None,
             **override) -> OracleCfg:
    """Build the C struct from a synth.MPPIConfig (duck-typed). sdf_mode / gate_c / gate_tana default to
    the config's sdf_provider / gate_c / gate_tana (else the MLP, c = 0.5, tan(alpha) = 0.375)."""
    if sdf_mode is None:
        sdf_mode = getattr(cfg, "sdf_provider", 0)
    if gate_c is None:
        gate_c = getattr(cfg, "gate_c", 0.5)
    if gate_tana is None:
        gate_tana = getattr(cfg, "gate_tana", 0.375) if getattr(cfg, "sdf_provider", 0) == 1 else 0.375
    oc = OracleCfg()
    oc.n_ctrl, oc.K, oc.T = cfg.n_ctrl, cfg.K, cfg.T
    oc.dt, oc.lam, oc.mass, oc.gravity = cfg.dt, cfg.lam, cfg.mass, cfg.gravity
    for i in range(4):
        oc.u_lo[i], oc.u_hi[i], oc.sigma[i] = cfg.u_lo[i], cfg.u_hi[i], cfg.sigma[i]
    oc.w_goal, oc.w_sdf, oc.sdf_scale, oc.sdf_exp_max = cfg.w_goal, cfg.w_sdf, cfg.sdf_scale, cfg.sdf_exp_max
    oc.w_u, oc.w_guide, oc.fd_h = cfg.w_u, cfg.w_guide, cfg.fd_h
    oc.latent_dim, oc.hidden, oc.n_hidden = cfg.latent_dim, cfg.hidden, cfg.n_hidden
    oc.activation, oc.mlp_bf16 = cfg.activation, int(cfg.mlp_dtype == 1)
    oc.sdf_mode, oc.gate_c, oc.gate_tana = sdf_mode, gate_c, gate_tana
    oc.model = getattr(cfg, "model", 0)
    oc.pe_bands = getattr(cfg, "pe_bands", 0)
    if oc.model == 1:
        oc.arm, oc.kappa, oc.thrust_max, oc.rate_max = cfg.arm, cfg.kappa, cfg.thrust_max, cfg.rate_max
        for i in range(3):
            oc.inertia[i] = cfg.inertia[i]
        oc.q_gate, oc.q_vis, oc.q_sdf, oc.d_safe = cfg.q_gate, cfg.q_vis, cfg.q_sdf, cfg.d_safe
    for k, v in override.items():
        setattr(oc, k, v)
    return oc


def flat_weights(Ws, bs):
    return (_f32(np.concatenate([np.asarray(w, np.float32).reshape(-1) for w in Ws])),
            _f32(np.concatenate([np.asarray(b, np.float32).reshape(-1) for b in bs])))


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def noise(seed: int, step: int, g0: int, nK: int, T: int) -> np.ndarray:
    out = np.zeros((T, nK, 4), np.float64)
    lib().oracle_noise(seed, step, g0, nK, T, _p(out, C.c_double))
    return out


def bf16_round(v: float) -> float:
    return lib().oracle_bf16_round(float(v))


def rk4_step(x, u, dt, m, g):
    x = _f64(x)
    u = _f64(u)
    out = np.zeros(10, np.float64)
    lib().oracle_rk4_step(_p(x, C.c_double), _p(u, C.c_double), dt, m, g, _p(out, C.c_double))
    return out


def rotor_deriv(oc: OracleCfg, x, u):
    """Paper model (model 1): xdot for x [17], u [4]."""
    x, u = _f64(x), _f64(u)
    out = np.zeros(17)
    lib().oracle_rotor_deriv(C.byref(oc), _p(x, C.c_double), _p(u, C.c_double), _p(out, C.c_double))
    return out


def rotor_step(oc: OracleCfg, x, u):
    """Paper model (model 1): one RK4 step of oc.dt with the post-step renormalisation and clamps."""
    x, u = _f64(x), _f64(u)
    out = np.zeros(17)
    lib().oracle_rotor_step(C.byref(oc), _p(x, C.c_double), _p(u, C.c_double), _p(out, C.c_double))
    return out


def pe(bands: int, p) -> np.ndarray:
    p = _f64(p)
    out = np.zeros(3 + 6 * bands)
    lib().oracle_pe(bands, _p(p, C.c_double), _p(out, C.c_double))
    return out


def mlp(oc: OracleCfg, Ws, bs, z, p) -> float:
    W, b = flat_weights(Ws, bs)
    z = _f32(z)
    p = _f64(p)
    return lib().oracle_mlp(C.byref(oc), _p(W, C.c_float), _p(b, C.c_float), _p(z, C.c_float), _p(p, C.c_double))


def mlp_trace(oc: OracleCfg, Ws, bs, z, p):
    """(s, acts [n_hidden][H]): the forward of mlp() with every hidden layer's activations (test support)."""
    W, b = flat_weights(Ws, bs)
    z = _f32(z)
    p = _f64(p)
    acts = np.zeros((oc.n_hidden, oc.hidden))
    s = lib().oracle_mlp_trace(C.byref(oc), _p(W, C.c_float), _p(b, C.c_float), _p(z, C.c_float), _p(p, C.c_double),
                               _p(acts, C.c_double))
    return s, acts


def sdf_analytic(c: float, tana: float, p) -> float:
    p = _f64(p)
    return lib().oracle_sdf_analytic(c, tana, _p(p, C.c_double))


def sdf_rows(oc: OracleCfg, Ws, bs, z, rows) -> np.ndarray:
    W, b = flat_weights(Ws, bs)
    z = _f32(z)
    rows = _f32(rows)
    out = np.zeros(rows.shape[0], np.float64)
    lib().oracle_sdf_rows(C.byref(oc), _p(W, C.c_float), _p(b, C.c_float), _p(z, C.c_float),
                          _p(rows, C.c_float), rows.shape[0], _p(out, C.c_double))
    return out


def rollout(oc: OracleCfg, Ws, bs, z, Tq, x0, goal, U, noise_tk4):
    """One sample. noise_tk4: [T][4] standard normals. Returns dict of states/queries/sdf/stage/J."""
    W, b = flat_weights(Ws, bs)
    T = oc.T
    nz = _f64(noise_tk4)
    st = np.zeros((T + 1, 17 if oc.model == 1 else 10))
    q = np.zeros((T, 8))
    s = np.zeros((T, 2))
    c = np.zeros(T)
    J = lib().oracle_rollout(C.byref(oc), _p(W, C.c_float), _p(b, C.c_float), _p(_f32(z), C.c_float),
                             _p(_f32(Tq), C.c_float), _p(_f32(x0), C.c_float), _p(_f32(goal), C.c_float),
                             _p(_f32(U), C.c_float), _p(nz, C.c_double), 4,
                             _p(st, C.c_double), _p(q, C.c_double), _p(s, C.c_double), _p(c, C.c_double))
    return {"states": st, "queries": q, "sdf": s, "stage": c, "J": J}


def softmin(oc: OracleCfg, J, U, noise_tk4):
    """One controller. J [K]; U [T][4]; noise [T][K][4]. Returns (U_new, Jmin, S, V, ess, flag)."""
    J = _f64(J)
    U = _f32(U)
    nz = _f64(noise_tk4)
    K = J.shape[0]
    T = oc.T
    V = np.zeros((T, 4))
    Un = np.zeros((T, 4))
    jm, S, es = C.c_double(), C.c_double(), C.c_double()
    flag = lib().oracle_softmin(C.byref(oc), K, _p(J, C.c_double), _p(U, C.c_float), _p(nz, C.c_double),
                                K * 4, C.byref(jm), C.byref(S), _p(V, C.c_double), _p(Un, C.c_double), C.byref(es))
    return Un, jm.value, S.value, V, es.value, flag


def shard_record(oc: OracleCfg, J, U, noise_tk4):
    J = _f64(J)
    nz = _f64(noise_tk4)
    rec = np.zeros(2 + oc.T * 4)
    lib().oracle_shard_record(C.byref(oc), J.shape[0], _p(J, C.c_double), _p(_f32(U), C.c_float),
                              _p(nz, C.c_double), J.shape[0] * 4, _p(rec, C.c_double))
    return rec


def combine(oc: OracleCfg, recs, U):
    recs = _f64(recs)
    Un = np.zeros((oc.T, 4))
    flag = lib().oracle_combine(C.byref(oc), recs.shape[0], _p(recs, C.c_double), _p(_f32(U), C.c_float),
                                _p(Un, C.c_double))
    return Un, flag


def step(oc: OracleCfg, Ws, bs, z, Tq, x0, goal, U, noise_tkn4, want_queries=True):
    """Full iteration over all controllers. noise: [T][n_ctrl*K][4]. U already shifted."""
    W, b = flat_weights(Ws, bs)
    n, K, T = oc.n_ctrl, oc.K, oc.T
    out = {
        "queries": np.zeros((n, K, T, 8)) if want_queries else None,
        "sdf": np.zeros((n, K, T, 2)) if want_queries else None,
        "stage": np.zeros((n, K, T)) if want_queries else None,
        "J": np.zeros((n, K)), "Jmin": np.zeros(n), "S": np.zeros(n), "ess": np.zeros(n),
        "V": np.zeros((n, T, 4)), "U_new": np.zeros((n, T, 4)), "flags": np.zeros(n, np.int32),
    }
    nz = _f64(noise_tkn4)
    lib().oracle_step(C.byref(oc), _p(W, C.c_float), _p(b, C.c_float), _p(_f32(z), C.c_float),
                      _p(_f32(Tq), C.c_float), _p(_f32(x0), C.c_float), _p(_f32(goal), C.c_float),
                      _p(_f32(U), C.c_float), _p(nz, C.c_double),
                      _p(out["queries"], C.c_double), _p(out["sdf"], C.c_double), _p(out["stage"], C.c_double),
                      _p(out["J"], C.c_double), _p(out["Jmin"], C.c_double), _p(out["S"], C.c_double),
                      _p(out["ess"], C.c_double), _p(out["V"], C.c_double), _p(out["U_new"], C.c_double),
                      _p(out["flags"], C.c_int32))
    return out


def shift(U):
    U = _f32(U).copy()
    n, T = U.shape[0], U.shape[1]
    lib().oracle_shift(n, T, _p(U, C.c_float))
    return U
