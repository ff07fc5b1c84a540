"""Diagnostic (not a test): rollout / softmin stage times for device vs external noise."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    for mode in ["device", "external"]:
        cfg, Ws, bs, inp, ctrl = gh.setup(name, noise_mode=mode)
        ctrl.set_profiling(2)
        ts = []
        for s in range(12):
            ctrl.step(inp["x0"], inp["goal"], s)
            ctrl.get_controls(allow_nonfinite=True)
            ts.append(ctrl.kernel_times())
        t = np.median(np.array(ts[2:]), axis=0)
        print(name, mode, "stage ms", np.round(t, 4))
