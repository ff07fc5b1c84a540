"""Profiling driver (not a test): run the production SDF-MLP kernel (mppi_sdf_eval) a few times on a
config's full per-iteration row count, for ncu. python tests/prof_mlp.py c4 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from tests import gpu_helpers as gh  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg0 = synth.get_config(name)
    cfg, Ws, bs, inp, ctrl = gh.setup(name + "s")
    n = cfg0.n_ctrl * cfg0.K * cfg0.T * (2 if cfg0.fd else 1)
    rows = torch.from_numpy(synth.make_query_rows(n, seed=4)).cuda()
    for _ in range(reps):
        ctrl.sdf_eval(rows)
    torch.cuda.synchronize()
    print("done", name, n)


if __name__ == "__main__":
    main()
