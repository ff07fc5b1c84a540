"""Debug timeline of k_softmin (not a test). Needs the trace build:
  python -m paper_2603_07199_b200.build --trace
  MPPI_LIB=$PWD/paper_2603_07199_b200/libmppi_b200_trace.so MPPI_SKIP_BUILD=1 MPPI_TRACE_SOFTMIN=1 python tests/trace_softmin.py [c3]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402


def main():
    from paper_2603_07199_b200 import Controller
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    cfg = synth.get_config(name)
    Ws, bs = synth.make_weights(cfg)
    c = Controller(cfg, noise_mode="device")
    c.set_sdf_weights(Ws, bs)
    c.set_latent(synth.make_latents(cfg), synth.make_query_transforms(cfg))
    c.set_nominal(synth.make_nominal(cfg))
    for s in range(4):
        c.step(synth.make_x0(cfg), synth.make_goals(cfg), s)
    c.get_controls()
    buf = np.zeros(1024 * 10, np.uint64)
    c.lib.mppi_debug_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    r = buf.reshape(1024, 10).astype(np.int64)
    r = r[r[:, 0] != 0]
    t0 = r[:, 0].min()
    n = len(r)
    print(f"{name}: {n} blocks traced (controller 0, T slice 0); times in us from the first block start")
    st = (r[:, :5] - t0) / 1e3
    for lab, a, b in [("phase 1", 0, 1), ("reductions", 1, 2), ("phase 2", 2, 3)]:
        d = st[:, b] - st[:, a]
        print(f"  {lab:11s} mean {d.mean():7.2f}  min {d.min():7.2f}  max {d.max():7.2f}")
    print(f"  block start: min {st[:, 0].min():.2f} max {st[:, 0].max():.2f}; block end (phase 2 done) max {st[:, 3].max():.2f}")
    last = r[:, 4] != 0
    if last.any():   # stale stamps of earlier steps' last blocks may remain: the latest is this step's
        i = int(np.argmax(np.where(last, r[:, 4], 0)))
        print(f"  last block {i}: phase 2 done {st[i, 3]:.2f}, combine done {st[i, 4]:.2f} (tail {st[i, 4] - st[i, 3]:.2f})")
        print(f"    final ticket won {(r[i, 6] - t0) / 1e3:.2f} (two-level: after this SM's group combine), U* written {st[i, 4]:.2f}")
    sms = r[:, 5]
    print(f"  distinct SMs {len(set(sms.tolist()))}; blocks per SM max {np.bincount(sms).max()}")
    order = np.argsort(st[:, 0])
    for i in order[:: max(1, n // 24)]:
        print(f"   blk {i:4d} sm {sms[i]:3d}  start {st[i,0]:7.2f}  p1 {st[i,1]:7.2f}  red {st[i,2]:7.2f}  p2 {st[i,3]:7.2f}")
    c.close()


if __name__ == "__main__":
    main()
