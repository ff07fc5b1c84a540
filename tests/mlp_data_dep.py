"""Diagnostic (not a test): SDF-MLP kernel time on random query rows vs the rollout's own rows."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


cfg, Ws, bs, inp, ctrl = gh.setup("c2", noise_mode="device")
ctrl.set_profiling(True)
for i in range(3):
    ctrl.step(inp["x0"], inp["goal"], i)
ctrl.get_controls()
print("step stage ms", ctrl.kernel_times())
q = ctrl.debug("queries").reshape(-1, 4)
n = q.shape[0]
rnd = torch.from_numpy(synth.make_query_rows(n, seed=4)).cuda()
qq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
print("rows: rollout |p| mean", np.abs(q[:, :3]).mean(), "max", np.abs(q[:, :3]).max())
print("sdf_eval random rows ms", timeit(lambda: ctrl.sdf_eval(rnd)))
print("sdf_eval rollout rows ms", timeit(lambda: ctrl.sdf_eval(qq)))
z = torch.zeros_like(rnd)
print("sdf_eval zero rows ms", timeit(lambda: ctrl.sdf_eval(z)))
s = ctrl.sdf_eval(qq).cpu().numpy()
print("sdf on rollout rows: mean", s.mean(), "min", s.min(), "max", s.max())
