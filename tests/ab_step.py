"""A/B timing of whole MPPI steps for several library builds (not a test):
python tests/ab_step.py LIB1 LIB2 ... [--cfg=c1]. Each library runs in its own subprocess (A B A B A B);
device-resident inputs, no profiling events in the graph, L2 flushed before every step outside the events."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg_name):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import synth
    from paper_2603_07199_b200 import Controller
    cfg = synth.get_config(cfg_name)
    ctrl = Controller(cfg, noise_mode="device")
    Ws, bs = synth.make_weights(cfg)
    ctrl.set_sdf_weights(Ws, bs)
    ctrl.set_latent(synth.make_latents(cfg), synth.make_query_transforms(cfg))
    ctrl.set_nominal(synth.make_nominal(cfg))
    x0 = torch.from_numpy(synth.make_x0(cfg)).cuda()
    goal = torch.from_numpy(synth.make_goals(cfg)).cuda()
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(40):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctrl.step_device(x0, goal, i)
        b.record()
        b.synchronize()
        if i >= 10:
            ts.append(a.elapsed_time(b))
    print(json.dumps({"ms": float(np.median(ts))}))


def main():
    if sys.argv[1] == "--child":
        return child(sys.argv[2])
    cfg = next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--cfg=")), "c1")
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    res = {l: [] for l in libs}
    for _ in range(3):
        for lib in libs:
            out = subprocess.run([sys.executable, __file__, "--child", cfg], env=dict(os.environ, MPPI_LIB=lib),
                                 capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            res[lib].append(json.loads(line[-1]) if line else {"error": out.stderr[-300:]})
    for lib, rs in res.items():
        print(cfg, os.path.basename(lib), rs)


if __name__ == "__main__":
    main()
