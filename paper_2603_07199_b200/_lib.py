"""Thin ctypes binding of include/mppi.h (argument marshalling only; every step runs in the CUDA
kernels of libmppi_b200.so). Fails loudly when the library or a CUDA device is missing: there is
no CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmppi_b200.so")

MPPI_ABI_VERSION = 3
REC_HEAD = 8   # softmin record header floats (m, S, S2, SJ, N, 0, 0, 0), then V[T][4]
STATUS = {0: "OK", -1: "INVALID", -2: "CUDA", -3: "NCCL", -4: "NOT_READY", -5: "NONFINITE", -6: "OOM",
          -7: "POISONED", -8: "UNSUPPORTED"}
MPPI_OK, MPPI_ERR_INVALID, MPPI_ERR_NONFINITE, MPPI_ERR_UNSUPPORTED = 0, -1, -5, -8
DBG = {"queries": 0, "sdf": 1, "costs": 2, "noise": 3, "terms": 4, "partial": 5, "record": 6, "weights": 7}

# every symbol include/mppi.h declares (checked by tests/test_boundary.py)
EXPORTS = ["mppi_workspace_bytes", "mppi_create", "mppi_destroy", "mppi_get_nccl_unique_id",
           "mppi_set_sdf_weights", "mppi_set_latent", "mppi_set_latent_frame", "mppi_get_latent_status", "mppi_set_nominal", "mppi_set_noise", "mppi_step",
           "mppi_step_device", "mppi_step_local", "mppi_record_size", "mppi_get_record_device",
           "mppi_step_finish", "mppi_get_controls", "mppi_get_diagnostics", "mppi_debug_copy", "mppi_sdf_eval",
           "mppi_set_profiling", "mppi_set_debug_outputs", "mppi_get_kernel_times", "mppi_kernels_per_step", "mppi_fused_rollout", "mppi_debug_trace",
           "mppi_last_error"]


class MppiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"mppi status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class MppiConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("n_ctrl", C.c_int32), ("K", C.c_int32), ("T", C.c_int32),
        ("K_global", C.c_int32), ("k_offset", C.c_int64),
        ("dt", C.c_float), ("lam", C.c_float), ("mass", C.c_float), ("gravity", C.c_float),
        ("u_lo", C.c_float * 4), ("u_hi", C.c_float * 4), ("sigma", C.c_float * 4),
        ("w_goal", C.c_float), ("w_sdf", C.c_float), ("sdf_scale", C.c_float), ("sdf_exp_max", C.c_float),
        ("w_u", C.c_float), ("w_guide", C.c_float), ("fd_h", C.c_float),
        ("latent_dim", C.c_int32), ("hidden", C.c_int32), ("n_hidden", C.c_int32),
        ("activation", C.c_int32), ("mlp_dtype", C.c_int32), ("noise_mode", C.c_int32),
        ("seed", C.c_uint64), ("world_size", C.c_int32), ("rank", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("device", C.c_int32), ("stream", C.c_void_p),
        # ABI 2
        ("model", C.c_int32), ("arm", C.c_float), ("kappa", C.c_float), ("inertia", C.c_float * 3),
        ("thrust_max", C.c_float), ("rate_max", C.c_float),
        ("q_gate", C.c_float), ("q_vis", C.c_float), ("q_sdf", C.c_float), ("d_safe", C.c_float),
        ("sdf_provider", C.c_int32), ("gate_c", C.c_float), ("gate_tana", C.c_float),
        ("pe_bands", C.c_int32),
        # ABI 3
        ("ctrl_offset", C.c_int64),
    ]


_lib = None


def load(path: str | None = None):
    """Load libmppi_b200.so (raises if it is missing; build with paper_2603_07199_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MPPI_LIB", LIB_PATH)   # MPPI_LIB: e.g. the MPPI_TC_TRACE debug build
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp, i32, i64, u64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
    cfgp = C.POINTER(MppiConfig)
    sig = {
        "mppi_workspace_bytes": ([cfgp], sz),
        "mppi_create": ([cfgp, vp, sz, C.POINTER(vp)], i32),
        "mppi_destroy": ([vp], i32),
        "mppi_get_nccl_unique_id": ([vp], i32),
        "mppi_set_sdf_weights": ([vp, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(vp), C.POINTER(vp)], i32),
        "mppi_set_latent": ([vp, i32, vp, vp], i32),
        "mppi_set_latent_frame": ([vp, i32, vp, vp, C.c_double, i32], i32),
        "mppi_get_latent_status": ([vp, vp, vp, vp], i32),
        "mppi_set_nominal": ([vp, i32, vp], i32),
        "mppi_set_noise": ([vp, vp], i32),
        "mppi_step": ([vp, vp, vp, u64], i32),
        "mppi_step_device": ([vp, vp, vp, u64], i32),
        "mppi_step_local": ([vp, vp, vp, u64], i32),
        "mppi_record_size": ([vp], i32),
        "mppi_get_record_device": ([vp], vp),
        "mppi_step_finish": ([vp, vp, i32], i32),
        "mppi_get_controls": ([vp, vp, vp], i32),
        "mppi_get_diagnostics": ([vp, vp], i32),
        "mppi_debug_copy": ([vp, i32, vp, sz], i32),
        "mppi_sdf_eval": ([vp, i32, vp, i64, vp], i32),
        "mppi_set_profiling": ([vp, i32], i32),
        "mppi_set_debug_outputs": ([vp, i32], i32),
        "mppi_get_kernel_times": ([vp, vp, i32], i32),
        "mppi_kernels_per_step": ([vp], i32),
        "mppi_fused_rollout": ([vp], i32),
        "mppi_debug_trace": ([vp, i32], i32),
        "mppi_last_error": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(st: int):
    if st != MPPI_OK:
        raise MppiError(st, _lib.mppi_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def make_config(cfg, *, device: int = 0, stream: int = 0, noise_mode: str = "device", world_size: int = 1,
                rank: int = 0, K_global: int | None = None, k_offset: int = 0, nccl_id: bytes | None = None,
                seed: int | None = None, ctrl_offset: int = 0) -> MppiConfig:
    """Fill the C config from any object with the synth.MPPIConfig attribute names."""
    c = MppiConfig()
    c.abi_version = MPPI_ABI_VERSION
    c.n_ctrl, c.K, c.T = cfg.n_ctrl, cfg.K, cfg.T
    c.K_global = cfg.K if K_global is None else K_global
    c.k_offset = k_offset
    c.dt, c.lam, c.mass, c.gravity = cfg.dt, cfg.lam, cfg.mass, cfg.gravity
    for i in range(4):
        c.u_lo[i], c.u_hi[i], c.sigma[i] = cfg.u_lo[i], cfg.u_hi[i], cfg.sigma[i]
    c.w_goal, c.w_sdf, c.sdf_scale, c.sdf_exp_max = cfg.w_goal, cfg.w_sdf, cfg.sdf_scale, cfg.sdf_exp_max
    c.w_u, c.w_guide, c.fd_h = cfg.w_u, cfg.w_guide, cfg.fd_h
    c.latent_dim, c.hidden, c.n_hidden = cfg.latent_dim, cfg.hidden, cfg.n_hidden
    c.activation, c.mlp_dtype = cfg.activation, cfg.mlp_dtype
    c.noise_mode = {"device": 0, "external": 1}[noise_mode]
    c.seed = cfg.seed if seed is None else seed
    c.world_size, c.rank = world_size, rank
    c._nccl_buf = None
    if nccl_id is not None:
        c._nccl_buf = C.create_string_buffer(bytes(nccl_id), 128)
        c.nccl_unique_id = C.cast(c._nccl_buf, C.c_void_p)
    c.device = device
    c.stream = stream
    c.model = getattr(cfg, "model", 0)
    if c.model == 1:
        c.arm, c.kappa, c.thrust_max, c.rate_max = cfg.arm, cfg.kappa, cfg.thrust_max, cfg.rate_max
        for i in range(3):
            c.inertia[i] = cfg.inertia[i]
        c.q_gate, c.q_vis, c.q_sdf, c.d_safe = cfg.q_gate, cfg.q_vis, cfg.q_sdf, cfg.d_safe
    c.sdf_provider = getattr(cfg, "sdf_provider", 0)
    c.gate_c, c.gate_tana = getattr(cfg, "gate_c", 0.5), getattr(cfg, "gate_tana", 0.0)
    c.pe_bands = getattr(cfg, "pe_bands", 0)
    c.ctrl_offset = ctrl_offset
    return c
