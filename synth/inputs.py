"""Seeded input generators (no method arithmetic). See synth/__init__.py for the recipe."""
from __future__ import annotations

import math
import zlib

import numpy as np

from .configs import MPPIConfig

_TAGS = {"weights": 1, "latent": 2, "goal": 3, "gate": 4, "noise": 5, "x0": 6, "rows": 7}


def rng_for(seed: int, tag: str, *extra: int) -> np.random.Generator:
    """Independent numpy stream per (seed, tag, extra...)."""
    t = _TAGS.get(tag, zlib.crc32(tag.encode()))
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed & 0xFFFFFFFF, seed >> 32, t, *extra])))


def make_weights(cfg: MPPIConfig, seed: int | None = None):
    """Kaiming-uniform weights [out][in] (float32) and U(+-1/sqrt(fan_in)) biases, nn.Linear order."""
    rng = rng_for(cfg.seed if seed is None else seed, "weights")
    Ws, bs = [], []
    for fan_in, fan_out in cfg.layer_dims:
        bw = math.sqrt(6.0 / fan_in)
        bb = 1.0 / math.sqrt(fan_in)
        Ws.append(rng.uniform(-bw, bw, size=(fan_out, fan_in)).astype(np.float32))
        bs.append(rng.uniform(-bb, bb, size=(fan_out,)).astype(np.float32))
    return Ws, bs


def make_latents(cfg: MPPIConfig, frame: int = 0, seed: int | None = None) -> np.ndarray:
    """z ~ N(0,1), one per controller: [n_ctrl][latent_dim] float32. `frame` = depth-frame index."""
    rng = rng_for(cfg.seed if seed is None else seed, "latent", frame)
    return rng.standard_normal((cfg.n_ctrl, cfg.latent_dim)).astype(np.float32)


def make_goals(cfg: MPPIConfig, seed: int | None = None) -> np.ndarray:
    """Gate centres g_c ~ U([2,6]x[-2,2]x[-1,1]) (R17): [n_ctrl][3] float32."""
    rng = rng_for(cfg.seed if seed is None else seed, "goal")
    lo = np.array([2.0, -2.0, -1.0])
    hi = np.array([6.0, 2.0, 1.0])
    return rng.uniform(lo, hi, size=(cfg.n_ctrl, 3)).astype(np.float32)


def camera_transform() -> np.ndarray:
    """World->camera T_q (R row-major 3x3, t[3]) for a camera at the origin looking along world +x
    with OpenCV axes: x_c = -y_w, y_c = -z_w, z_c = x_w (reading R13)."""
    R = np.array([[0, -1, 0], [0, 0, -1], [1, 0, 0]], dtype=np.float32)
    return np.concatenate([R.reshape(-1), np.zeros(3, np.float32)])


def make_gate_poses(cfg: MPPIConfig, seed: int | None = None):
    """Per-drone gate pose (configs[4], R22): position ~ R17 box, yaw ~ U(-pi,pi), pitch ~ U(-30,30) deg.
    Returns (positions [n][3], yaw [n], pitch [n])."""
    rng = rng_for(cfg.seed if seed is None else seed, "gate")
    pos = make_goals(cfg, seed)
    yaw = rng.uniform(-math.pi, math.pi, size=cfg.n_ctrl)
    pitch = rng.uniform(-math.radians(30), math.radians(30), size=cfg.n_ctrl)
    return pos, yaw, pitch


def _gate_world_from_local(yaw: float, pitch: float) -> np.ndarray:
    cy, sy, cp, sp = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch)
    Rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
    Ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
    return Rz @ Ry


def make_query_transforms(cfg: MPPIConfig, seed: int | None = None) -> np.ndarray:
    """T_q per controller, [n_ctrl][12] float32 (R row-major, then t).

    Single controller: the fixed camera of R13. Per-drone gates (configs[4]): T_q = inverse of the
    gate pose (world -> gate frame), so the analytic Gate-SDF (Eq. 2) is meaningful.
    Analytic provider (cfg.sdf_provider == 1) without per-drone gates: world -> frame of a gate at the
    goal facing along world x (gate plane x = goal x), the frame Eq. 2 is written in."""
    if not cfg.per_drone_gates and getattr(cfg, "sdf_provider", 0) == 1:
        out = np.zeros((cfg.n_ctrl, 12), np.float32)
        out[:, [0, 4, 8]] = 1.0
        out[:, 9:] = -make_goals(cfg, seed)
        return out
    if not cfg.per_drone_gates:
        return np.tile(camera_transform(), (cfg.n_ctrl, 1)).astype(np.float32)
    pos, yaw, pitch = make_gate_poses(cfg, seed)
    out = np.zeros((cfg.n_ctrl, 12), np.float32)
    for i in range(cfg.n_ctrl):
        Rwg = _gate_world_from_local(float(yaw[i]), float(pitch[i]))
        Rgw = Rwg.T
        out[i, :9] = Rgw.reshape(-1)
        out[i, 9:] = -(Rgw @ pos[i].astype(np.float64))
    return out


def make_x0(cfg: MPPIConfig, jitter: float = 0.0, seed: int | None = None) -> np.ndarray:
    """[n_ctrl][10] float32: p=0, v=0, q=(1,0,0,0) (R18); optional seeded jitter on p, v.
    Paper model (cfg.model == 1): [n_ctrl][17], also w = 0 and hover rotor thrusts T_i = m g / 4 (P7)."""
    x0 = np.zeros((cfg.n_ctrl, cfg.state_dim), np.float32)
    x0[:, 6] = 1.0
    if cfg.model == 1:
        x0[:, 13:17] = np.float32(cfg.mass * cfg.gravity / 4.0)
    if jitter:
        rng = rng_for(cfg.seed if seed is None else seed, "x0")
        x0[:, 0:6] += rng.uniform(-jitter, jitter, size=(cfg.n_ctrl, 6)).astype(np.float32)
    return x0


def make_nominal(cfg: MPPIConfig) -> np.ndarray:
    """[n_ctrl][T][4] float32 hover nominal: thrust m*g, zero body rates (R18). Paper model: zero thrust
    rates (the hover thrusts are in the state)."""
    U = np.zeros((cfg.n_ctrl, cfg.T, 4), np.float32)
    if cfg.model == 0:
        U[:, :, 0] = np.float32(cfg.mass * cfg.gravity)
    return U


def make_noise(cfg: MPPIConfig, step: int = 0, seed: int | None = None) -> np.ndarray:
    """Standard normals, time-major [T][n_ctrl*K][4] float32 (external-noise parity mode)."""
    rng = rng_for(cfg.seed if seed is None else seed, "noise", step)
    return rng.standard_normal((cfg.T, cfg.n_ctrl * cfg.K, 4)).astype(np.float32)


def make_query_rows(n_rows: int, scale: float = 3.0, seed: int = 0) -> np.ndarray:
    """Query-frame points [n_rows][4] float32 (x, y, z, 0) within +-scale m, for MLP-only parity."""
    rng = rng_for(seed, "rows")
    rows = np.zeros((n_rows, 4), np.float32)
    rows[:, :3] = rng.uniform(-scale, scale, size=(n_rows, 3)).astype(np.float32)
    return rows


def constructed_gate_net(cfg: MPPIConfig, c: float = 0.5, tana: float = 0.375):
    """Weights of an exact ReLU network that computes the analytic Gate-SDF of PAPER.md:71 (Eq. 2),
    s = c + |x| tan(alpha) - max(|y|, |z|), zero-padded into cfg's shapes (SURVEY.md §8c pin).

    Layer 1: relu(+-x), relu(+-y), relu(+-z) (latent columns zero).
    Layer 2: |x|, |y|, relu(|z| - |y|).  Later hidden layers: identity on those three units.
    Output:  c + tana*|x| - |y| - relu(|z|-|y|)  ( = c + tana|x| - max(|y|,|z|) ).
    All weights are in {0, +-1, tana} (tana = 0.375 is exact in bf16). Requires ReLU, n_hidden >= 2."""
    assert cfg.n_hidden >= 2 and cfg.hidden >= 6
    dims = cfg.layer_dims
    Ws = [np.zeros((o, i), np.float32) for (i, o) in dims]
    bs = [np.zeros((o,), np.float32) for (i, o) in dims]
    W1 = Ws[0]
    for a in range(3):
        W1[2 * a, a] = 1.0
        W1[2 * a + 1, a] = -1.0
    W2 = Ws[1]
    W2[0, 0] = W2[0, 1] = 1.0                       # |x|
    W2[1, 2] = W2[1, 3] = 1.0                       # |y|
    W2[2, 4] = W2[2, 5] = 1.0                       # |z| - |y|
    W2[2, 2] = W2[2, 3] = -1.0
    for l in range(2, cfg.n_hidden):
        for u in range(3):
            Ws[l][u, u] = 1.0
    Wo = Ws[-1]
    Wo[0, 0] = tana
    Wo[0, 1] = -1.0
    Wo[0, 2] = -1.0
    bs[-1][0] = c
    return Ws, bs
