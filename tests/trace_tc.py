"""Debug timeline of the tcgen05 SDF-MLP kernel (not a test). Needs the MPPI_TC_TRACE build:
  python paper_2603_07199_b200/build.py --trace
  MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so python tests/trace_tc.py [c2|c1] [tiles_per_cta]
Prints, for CTA 0, the cycle (clock64, relative) of every MMA-unit issue and epilogue phase."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402

EV = {0: "mma.wait", 1: "mma.issue", 2: "mma.done_issue", 3: "epi.wait", 4: "epi.got", 5: "epi.unit_done",
      6: "L1.start", 7: "L1.end", 8: "tile.out", 9: "epi.ld_done", 10: "epi.dfree_sent", 11: "L1.rows_ready",
      12: "L1.computed"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    tpc = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cfg, Ws, bs, inp, ctrl = gh.setup(name + "s" if name in ("c1", "c2") else name)
    cg = 2 if cfg.hidden == 256 else 1
    n = 148 // cg * cg * 128 * tpc
    rows = synth.make_query_rows(n, seed=3)
    ctrl.sdf_eval(rows)                      # warm-up (module load)
    lib = ctrl.lib
    cap = 4 * 3 * 2048
    buf = np.zeros(cap, np.uint64)
    lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), cap)   # reset
    import torch
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    step_mode = len(sys.argv) > 3 and sys.argv[3] == "step"   # a whole controller step (MPPI_FUSED=1: fused)
    if step_mode:
        from paper_2603_07199_b200 import Controller
        cfg = synth.get_config(name)
        sc = Controller(cfg, noise_mode="device")
        sc.set_sdf_weights(Ws, bs)
        sc.set_latent(synth.make_latents(cfg), synth.make_query_transforms(cfg))
        sc.set_nominal(synth.make_nominal(cfg))
        sc.step(synth.make_x0(cfg), synth.make_goals(cfg), 0)
        sc.get_controls()
        lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), cap)   # reset
        print(f"fused rollout: {sc.fused_rollout()}")
    t0.record()
    if step_mode:
        sc.step(synth.make_x0(cfg), synth.make_goals(cfg), 1)
    else:
        ctrl.sdf_eval(rows)
    t1.record()
    torch.cuda.synchronize()
    print(f"{name}: {n} rows, {t0.elapsed_time(t1) * 1e3:.1f} us (with tracing)")
    lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), cap)
    rec = buf.reshape(4, 3, 2048)
    for blk in range(2):
        ev = []
        for role in range(3):
            r = rec[blk, role]
            r = r[r != 0]
            code = (r >> np.uint64(48)).astype(np.int64)
            clk = (r & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
            ev += [(int(k), role, int(c)) for k, c in zip(clk, code)]
        if not ev:
            continue
        ev.sort()
        base = ev[0][0]
        print(f"--- block {blk}: {len(ev)} events, span {ev[-1][0] - base} cycles")
        for k, role, ci in ev:
            print(f"{k - base:8d} {['MMA', 'EPI0', 'EPI7'][role]:5s} {EV.get((ci >> 8) & 15, '?'):16s} "
                  f"l={(ci >> 6) & 3} q={(ci >> 4) & 3} t={ci & 15}")


if __name__ == "__main__":
    main()
