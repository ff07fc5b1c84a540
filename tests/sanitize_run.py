"""Small end-to-end run for compute-sanitizer (not a test): one MPPI iteration each of configs c0 (fp32 SIMT
MLP), c1s (H = 128 tcgen05 kernel), c2s (H = 256 CTA-pair kernel), c1pes (positional encoding) and c4s
(controller batch), with the debug copies, through the C ABI.
  compute-sanitizer --tool memcheck python tests/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402


def main():
    names = sys.argv[1:] or ["c0", "c1s", "c2s", "c1pes", "c4s"]
    for name in names:
        cfg, Ws, bs, inp, ctrl = gh.setup(name)
        ctrl.step(inp["x0"], inp["goal"], 0)
        U, u0 = ctrl.get_controls(allow_nonfinite=True)
        for what in ("queries", "sdf", "costs", "terms", "partial", "weights"):
            ctrl.debug(what)
        if cfg.mlp_dtype == 1:
            ctrl.sdf_eval(synth.make_query_rows(300, seed=1)).cpu()
        ctrl.close()
        print(name, "ok", float(np.abs(U).max()))


if __name__ == "__main__":
    main()
