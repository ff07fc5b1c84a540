"""Debug timeline of the H = 128 tcgen05 SDF-MLP kernel (kernel_mlp_h128.cu; not a test). Needs the trace build:
  python paper_2603_07199_b200/build.py --trace
  MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so MPPI_TRACE_H128=1 python tests/trace_h128.py [c1|c4] [tiles_per_cta]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402

EV = {0: "mma.wait", 1: "mma.issue", 2: "mma.committed", 3: "epi.wait", 4: "epi.got", 5: "epi.done", 6: "A1.start",
      7: "A1.done"}
ROLES = ["MMA", "EPI0", "EPI1", "EPI2", "EPI3"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    tpc = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    cfg, Ws, bs, inp, ctrl = gh.setup(name + "s")
    n = 148 * 128 * tpc
    rows = synth.make_query_rows(n, seed=3)
    ctrl.sdf_eval(rows)
    lib = ctrl.lib
    cap = 2 * 5 * 2048
    buf = np.zeros(cap, np.uint64)
    lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), cap)
    import torch
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    ctrl.sdf_eval(rows)
    t1.record()
    torch.cuda.synchronize()
    print(f"{name}: {n} rows, {t0.elapsed_time(t1) * 1e3:.1f} us (with tracing)")
    lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), cap)
    rec = buf.reshape(2, 5, 2048)
    for blk in range(1):
        ev = []
        for role in range(5):
            r = rec[blk, role]
            r = r[r != 0]
            code = (r >> np.uint64(48)).astype(np.int64)
            clk = (r & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
            ev += [(int(k), role, int(c)) for k, c in zip(clk, code)]
        ev.sort()
        base = ev[0][0]
        print(f"--- block {blk}: {len(ev)} events, span {ev[-1][0] - base} cycles")
        for k, role, ci in ev:
            print(f"{k - base:8d} {ROLES[role]:5s} {EV.get((ci >> 8) & 15, '?'):14s} u={(ci >> 4) & 15} t={ci & 15}")


if __name__ == "__main__":
    main()
