"""A/B timing of SDF-MLP kernel builds (not a test): python tests/ab_mlp.py LIB1 LIB2 ... [--cfg c2]
A library argument may carry environment settings: path,VAR=VAL,... (e.g. lib.so,MPPI_H128_LEGACY=1).
Runs each library in its own subprocess, interleaved A B A B (3 rounds), timing mppi_sdf_eval on the
configs' full per-iteration row count with CUDA events and sampling the SM clock with nvidia-smi."""
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
    from tests import gpu_helpers as gh
    cfg0 = synth.get_config(cfg_name)
    cfg, Ws, bs, inp, ctrl = gh.setup(cfg_name + "s")
    n = cfg0.n_ctrl * cfg0.K * cfg0.T * (2 if cfg0.fd else 1)
    rows = torch.from_numpy(synth.make_query_rows(n, seed=4)).cuda()
    for _ in range(3):
        out = ctrl.sdf_eval(rows)
    torch.cuda.synchronize()
    np.save(os.environ["AB_OUT"], out[:1 << 18].float().cpu().numpy())
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "20"],
                           stdout=subprocess.PIPE, text=True)
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctrl.sdf_eval(rows)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    smi.terminate()
    clk = [float(x) for x in smi.communicate()[0].split()]
    H, G = cfg0.hidden, cfg0.n_hidden - 1
    flop = 2 * ((3 + 6 * cfg0.pe_bands) * H + G * H * H + H) * n
    ms = float(np.median(ts))
    print(json.dumps({"ms": ms, "tflops": flop / ms / 1e9, "sm_mhz": float(np.median(clk)) if clk else None}))


def main():
    if sys.argv[1] == "--child":
        return child(sys.argv[2])
    cfg = "c2"
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    for a in sys.argv[1:]:
        if a.startswith("--cfg="):
            cfg = a.split("=")[1]
    res = {l: [] for l in libs}
    for _ in range(3):
        for lib in libs:
            path, *kv = lib.split(",")
            env = dict(os.environ, MPPI_LIB=path, AB_OUT=f"/tmp/ab_{os.path.basename(lib)}_{cfg}.npy", MPPI_SKIP_BUILD="1",
                       **dict(x.split("=", 1) for x in kv))
            out = subprocess.run([sys.executable, __file__, "--child", cfg], env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            res[lib].append(json.loads(line[-1]) if line else {"error": out.stderr[-300:]})
    import numpy as np
    base = np.load(f"/tmp/ab_{os.path.basename(libs[0])}_{cfg}.npy")
    for lib, rs in res.items():
        o = np.load(f"/tmp/ab_{os.path.basename(lib)}_{cfg}.npy")
        print(os.path.basename(lib), rs, "max|d sdf| vs first:", float(np.abs(o - base).max()))


if __name__ == "__main__":
    main()
