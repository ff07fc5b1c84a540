"""Diagnostic (not a test): where the end-to-end time of a configs[3] step goes. Times, back to back on one
box: (1) the device step with the bench's L2 flush between steps, (2) the device step back to back, (3) the
public API loop (mppi_step with host buffers + mppi_get_controls), each with the median SM clock sampled by
nvidia-smi during the loop. python tests/diag_e2e.py [config] [steps]"""
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402


def clocks():
    return subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "50"], stdout=subprocess.PIPE, text=True)


def stop(p):
    p.terminate()
    rows = [r.split(",") for r in p.communicate()[0].strip().splitlines() if r.strip()]
    sm = [float(r[0]) for r in rows]
    pw = [float(r[1]) for r in rows]
    return (float(np.median(sm)) if sm else None, float(np.median(pw)) if pw else None)


def main():
    import torch
    from paper_2603_07199_b200 import Controller
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cfg = synth.get_config(name)
    Ws, bs = synth.make_weights(cfg)
    c = Controller(cfg, noise_mode="device")
    c.set_sdf_weights(Ws, bs)
    c.set_latent(synth.make_latents(cfg), synth.make_query_transforms(cfg))
    c.set_nominal(synth.make_nominal(cfg))
    x0, goal = synth.make_x0(cfg), synth.make_goals(cfg)
    x0d, goald = torch.from_numpy(x0).cuda(), torch.from_numpy(goal).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(5):
        c.step_device(x0d, goald, i)
    torch.cuda.synchronize()
    out = {}
    for mode in ("device_flush", "device", "e2e", "device_flush"):
        p = clocks()
        time.sleep(0.3)
        ms = []
        t0 = time.perf_counter()
        for i in range(steps):
            if mode == "e2e":
                c.step(x0, goal, 100 + i)
                c.get_controls()
            else:
                if mode == "device_flush":
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                c.step_device(x0d, goald, 100 + i)
                b.record()
                b.synchronize()
                ms.append(a.elapsed_time(b))
        wall = (time.perf_counter() - t0) / steps * 1e3
        sm, pw = stop(p)
        out.setdefault(mode, []).append(dict(event_ms=float(np.mean(ms)) if ms else None, wall_ms=wall, sm_mhz=sm, watts=pw))
        print(mode, out[mode][-1], flush=True)


if __name__ == "__main__":
    main()
