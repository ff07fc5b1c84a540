"""B200-native (sm_100a) MPPI iteration with a neural Gate-SDF cost (arxiv 2603.07199).

Python surface over the C ABI in include/mppi.h. PyTorch provides device memory (the workspace),
streams and process groups; every step of the MPPI iteration runs in this package's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import DBG, MppiError, load, make_config  # noqa: F401

__all__ = ["Controller", "MppiError", "load", "nccl_unique_id"]


def nccl_unique_id() -> bytes:
    lib = load()
    buf = C.create_string_buffer(128)
    _lib._check(lib.mppi_get_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


class Controller:
    """One mppi_ctx: n_ctrl controllers x K samples x T steps on one GPU (one rank).

    cfg: an object with synth.MPPIConfig's attributes (n_ctrl, K, T, dt, lam, ..., mlp_dtype)."""

    def __init__(self, cfg, *, device: int = 0, stream=None, noise_mode: str = "device", world_size: int = 1,
                 rank: int = 0, K_global: int | None = None, k_offset: int = 0, nccl_id: bytes | None = None,
                 seed: int | None = None, debug_outputs: bool = False, ctrl_offset: int = 0, guard_bytes: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_07199_b200.Controller needs a CUDA device (no CPU fallback)")
        self.lib = load()
        self.cfg = cfg
        self.device = device
        self.torch_device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.torch_device)
        self.stream = stream
        self.c = make_config(cfg, device=device, stream=stream.cuda_stream, noise_mode=noise_mode,
                             world_size=world_size, rank=rank, K_global=K_global, k_offset=k_offset,
                             nccl_id=nccl_id, seed=seed, ctrl_offset=ctrl_offset)
        nbytes = self.lib.mppi_workspace_bytes(C.byref(self.c))
        if nbytes == 0:
            raise MppiError(-1, self.lib.mppi_last_error().decode())
        # guard_bytes (test support): a patterned zone before and after the workspace, checked by guards_intact()
        self._guard = guard_bytes
        self._ws_raw = torch.empty(nbytes + 2048 + 2 * guard_bytes, dtype=torch.uint8, device=self.torch_device)
        if guard_bytes:
            self._ws_raw.fill_(0xA5)
        base = self._ws_raw.data_ptr() + guard_bytes
        off = (-base) % 1024
        self.ws_ptr = base + off
        self._ws_lo = guard_bytes + off
        self._ws_hi = self._ws_lo + nbytes
        self.ctx = C.c_void_p()
        _lib._check(self.lib.mppi_create(C.byref(self.c), C.c_void_p(self.ws_ptr), nbytes, C.byref(self.ctx)))
        self.n, self.K, self.T = cfg.n_ctrl, cfg.K, cfg.T
        self.rps = 2 if cfg.w_guide != 0 else 1
        self.state_dim = 17 if getattr(cfg, "model", 0) == 1 else 10
        if debug_outputs:
            self.set_debug_outputs(True)

    def guards_intact(self) -> bool:
        """Test support (guard_bytes > 0): no kernel wrote into the patterned zones around the workspace."""
        import torch
        torch.cuda.synchronize(self.torch_device)
        lo = self._ws_raw[self._ws_lo - self._guard:self._ws_lo]
        hi = self._ws_raw[self._ws_hi:self._ws_hi + self._guard]
        return bool((lo == 0xA5).all().item()) and bool((hi == 0xA5).all().item())

    def set_debug_outputs(self, on: bool):
        """Test support: also write s per query row in every step (debug("sdf")); off by default."""
        _lib._check(self.lib.mppi_set_debug_outputs(self.ctx, 1 if on else 0))

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.lib.mppi_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- setters
    def set_sdf_weights(self, Ws, bs):
        n = len(Ws)
        Ws = [_f32(w) for w in Ws]
        bs = [_f32(b) for b in bs]
        ind = (C.c_int32 * n)(*[w.shape[1] for w in Ws])
        outd = (C.c_int32 * n)(*[w.shape[0] for w in Ws])
        Wp = (C.c_void_p * n)(*[w.ctypes.data for w in Ws])
        bp = (C.c_void_p * n)(*[b.ctypes.data for b in bs])
        _lib._check(self.lib.mppi_set_sdf_weights(self.ctx, n, ind, outd, Wp, bp))

    def set_latent(self, z, T_q, ctrl: int = -1):
        z = _f32(z)
        T_q = _f32(T_q)
        _lib._check(self.lib.mppi_set_latent(self.ctx, ctrl, _lib._ptr(z), _lib._ptr(T_q)))

    def set_latent_frame(self, z, T_q, t_frame: float, valid: bool = True, ctrl: int = -1):
        """A depth frame for the latent cache: valid frames refresh (z, T_q) and record
        t_frame; invalid (occluded) frames keep the cached pair (z, T_q may be None)."""
        zp = tp = None
        if valid:
            z, T_q = _f32(z), _f32(T_q)
            zp, tp = _lib._ptr(z), _lib._ptr(T_q)
        _lib._check(self.lib.mppi_set_latent_frame(self.ctx, ctrl, zp, tp, float(t_frame), 1 if valid else 0))

    def latent_status(self):
        """(t_frame [n], steps since the cached frame [n], invalid frames since [n])."""
        t = np.zeros(self.n, np.float64)
        st = np.zeros(self.n, np.int64)
        inv = np.zeros(self.n, np.int64)
        _lib._check(self.lib.mppi_get_latent_status(self.ctx, _lib._ptr(t), _lib._ptr(st), _lib._ptr(inv)))
        return t, st, inv

    def set_nominal(self, U, ctrl: int = -1):
        U = _f32(U)
        _lib._check(self.lib.mppi_set_nominal(self.ctx, ctrl, _lib._ptr(U)))

    def set_noise(self, noise):
        """noise: torch CUDA float32 tensor [T][n_ctrl*K][4] of standard normals (or a numpy array)."""
        import torch
        if not isinstance(noise, torch.Tensor):
            noise = torch.from_numpy(_f32(noise)).to(self.torch_device)
        noise = noise.contiguous().to(torch.float32)
        self._noise_keep = noise
        _lib._check(self.lib.mppi_set_noise(self.ctx, C.c_void_p(noise.data_ptr())))

    # ---------------------------------------------------------------- steps
    def _host_inputs(self, x0, goal):
        x0, goal = _f32(x0), _f32(goal)
        if x0.size != self.n * self.state_dim or goal.size != self.n * 3:
            raise ValueError(f"x0 must be [{self.n}][{self.state_dim}] and goal [{self.n}][3]")
        return x0, goal

    def step(self, x0, goal, step_index: int = 0):
        x0, goal = self._host_inputs(x0, goal)
        _lib._check(self.lib.mppi_step(self.ctx, _lib._ptr(x0), _lib._ptr(goal), step_index))

    def step_device(self, x0, goal, step_index: int = 0):
        """x0, goal: torch CUDA float32 tensors [n_ctrl][10] ([n_ctrl][17] for the paper model), [n_ctrl][3]."""
        _lib._check(self.lib.mppi_step_device(self.ctx, C.c_void_p(x0.data_ptr()), C.c_void_p(goal.data_ptr()),
                                              step_index))

    def step_local(self, x0, goal, step_index: int = 0):
        x0, goal = self._host_inputs(x0, goal)
        goal = _f32(goal)
        _lib._check(self.lib.mppi_step_local(self.ctx, _lib._ptr(x0), _lib._ptr(goal), step_index))

    def record_size(self) -> int:
        return self.lib.mppi_record_size(self.ctx)

    def record_ptr(self) -> int:
        return self.lib.mppi_get_record_device(self.ctx)

    def step_finish(self, records):
        """records: torch CUDA float32 [R][n_ctrl][record_size] gathered in rank order."""
        _lib._check(self.lib.mppi_step_finish(self.ctx, C.c_void_p(records.data_ptr()), records.shape[0]))

    # ---------------------------------------------------------------- results
    def get_controls(self, allow_nonfinite: bool = False):
        U = np.zeros((self.n, self.T, 4), np.float32)
        u0 = np.zeros((self.n, 4), np.float32)
        st = self.lib.mppi_get_controls(self.ctx, _lib._ptr(U), _lib._ptr(u0))
        if st == _lib.MPPI_ERR_NONFINITE and allow_nonfinite:
            return U, u0
        _lib._check(st)
        return U, u0

    def diagnostics(self) -> np.ndarray:
        out = np.zeros((self.n, 4), np.float32)
        _lib._check(self.lib.mppi_get_diagnostics(self.ctx, _lib._ptr(out)))
        return out

    def debug(self, what: str) -> np.ndarray:
        n, K, T, r = self.n, self.K, self.T, self.rps
        shapes = {"queries": (n, T, K, r, 4), "sdf": (n, T, K, r), "costs": (n, K), "noise": (T, n * K, 4),
                  "terms": (n, T, K), "partial": (n, K), "record": (n, _lib.REC_HEAD + 4 * T), "weights": (n, K)}
        out = np.zeros(shapes[what], np.float32)
        _lib._check(self.lib.mppi_debug_copy(self.ctx, DBG[what], _lib._ptr(out), out.nbytes))
        return out

    def sdf_eval(self, rows, ctrl: int = 0):
        """Run the production SDF-MLP kernel on query-frame rows [n][4] (torch CUDA or numpy)."""
        import torch
        if not isinstance(rows, torch.Tensor):
            rows = torch.from_numpy(_f32(rows)).to(self.torch_device)
        rows = rows.contiguous()
        out = torch.empty(rows.shape[0], dtype=torch.float32, device=self.torch_device)
        _lib._check(self.lib.mppi_sdf_eval(self.ctx, ctrl, C.c_void_p(rows.data_ptr()), rows.shape[0],
                                           C.c_void_p(out.data_ptr())))
        return out

    def set_profiling(self, level):
        """0 off, 1 events around the SDF-MLP launch, 2 every stage (True -> 2)."""
        level = 2 if level is True else int(level)
        _lib._check(self.lib.mppi_set_profiling(self.ctx, level))

    def kernel_times(self) -> np.ndarray:
        out = np.zeros(5, np.float32)
        _lib._check(self.lib.mppi_get_kernel_times(self.ctx, _lib._ptr(out), 5))
        return out

    def kernels_per_step(self) -> int:
        return self.lib.mppi_kernels_per_step(self.ctx)

    def fused_rollout(self) -> bool:
        """True if the step runs the rollout inside the SDF-MLP kernel (query rows never reach HBM)."""
        return bool(self.lib.mppi_fused_rollout(self.ctx))
