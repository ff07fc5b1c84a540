"""GPU diagnostics (not a test): error statistics of the CUDA path vs the oracle and rough stage
timings, printed as text. Run on a GPU box: python tests/diag_gpu.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402


def stats(name, **over):
    cfg, Ws, bs, inp, ctrl = gh.setup(name, **over)
    ctrl.step(inp["x0"], inp["goal"], 0)
    Ug, _ = ctrl.get_controls(allow_nonfinite=True)
    ref = gh.run_oracle(cfg, Ws, bs, inp)
    q = gh.gpu_queries_like_oracle(ctrl.debug("queries"))
    s = gh.gpu_sdf_like_oracle(ctrl.debug("sdf"))
    J = ctrl.debug("costs")
    qe = np.abs(q[..., :7] - ref["queries"][..., :7]) / (np.abs(ref["queries"][..., :7]) + 1e-6)
    se = np.abs(s - ref["sdf"])
    je = np.abs(J - ref["J"]) / np.abs(ref["J"])
    ue = np.abs(Ug - ref["U_new"]).max()
    print(f"{name} {over}: query relerr max {qe.max():.2e}; sdf abs err max {se.max():.2e} med {np.median(se):.2e};"
          f" J relerr max {je.max():.2e} med {np.median(je):.2e}; U err {ue:.2e};"
          f" Jmin {ref['Jmin']}, ess {ref['ess']}", flush=True)


def timing(name, steps=20):
    import torch
    cfg, Ws, bs, inp, ctrl = gh.setup(name, noise_mode="device")
    ctrl.set_profiling(2)
    for i in range(3):
        ctrl.step(inp["x0"], inp["goal"], i)
    ctrl.get_controls()
    t0 = time.time()
    st = []
    for i in range(steps):
        ctrl.step(inp["x0"], inp["goal"], 3 + i)
        st.append(ctrl.kernel_times())
    torch.cuda.synchronize()
    dt = (time.time() - t0) / steps
    kt = np.median(np.array(st), 0)
    print(f"timing {name}: wall {dt * 1e3:.3f} ms/step; stages ms (noise, rollout, mlp, softmin, exchange) {kt}", flush=True)


if __name__ == "__main__":
    for n in ["c0", "c1s", "c2s", "c3s", "c4s"]:
        try:
            stats(n)
        except Exception as e:  # keep going: this is a diagnostic
            print(f"{n}: FAILED {type(e).__name__}: {e}", flush=True)
    for n in ["c0", "c1", "c2"]:
        try:
            timing(n)
        except Exception as e:
            print(f"timing {n}: FAILED {type(e).__name__}: {e}", flush=True)
