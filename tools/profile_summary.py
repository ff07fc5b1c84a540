"""Summarise a round's GPU evidence (gpurun_out/<round>) into the committed profiles/<round>/ files and
profiles/ncu_mlp_summary.json (the `traffic` source of bench.py). Not part of the library.
python tools/profile_summary.py r01 [SRC_DIR DST_DIR]   (default gpurun_out/r01 -> profiles/r01; on the GPU box
run it with DST under gpurun_out/ and delete the .ncu-rep files, so the merged-back output stays small)"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        res.append((name, {k: [r[h.index(k)], u[h.index(k)]] for k in KEYS if k in h}))
    return res


def nbytes(v):
    return float(v[0].replace(",", "")) * SCALE.get(v[1], 1)


def main():
    rnd = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", rnd)
    dst = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    for f in os.listdir(src):
        if f.endswith((".json", ".txt", ".csv")) and not f.startswith("ncu_launch") and os.path.abspath(src) != os.path.abspath(dst):
            shutil.copy(os.path.join(src, f), dst)
    full = {}
    summ_path = os.path.join(dst, "..", "ncu_mlp_summary.json") if len(sys.argv) > 3 else \
        os.path.join(ROOT, "profiles", "ncu_mlp_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for c in ["c3", "c2", "c1", "c4", "c2pe"]:
        rep = os.path.join(src, f"mlp_{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        for name, m in raw(rep):
            full[f"{c}: {name[:60]}"] = m
            rd, wr = nbytes(m["dram__bytes_read.sum"]), nbytes(m["dram__bytes_write.sum"])
            summ[c] = {"kernel": name[:60], "source": f"profiles/{rnd}/ncu_full_metrics.json (ncu --set full, one launch, "
                       f"bench.py --config {c} --steps 3 --warmup 3)", "dram_bytes_per_launch": rd + wr,
                       "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "tensor_pipe_active_pct": float(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][0]),
                       "xu_pipe_pct": float(m["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"][0]),
                       "duration_us_under_ncu": float(m["gpu__time_duration.sum"][0].replace(",", "")) *
                                                 {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
                                                     m["gpu__time_duration.sum"][1], 1.0)}
    for c in ["c3", "c2"]:
        rep = os.path.join(src, f"small_{c}.ncu-rep")
        if os.path.exists(rep):
            for name, m in raw(rep):
                full[f"{c}: {name[:60]}"] = m
    json.dump(full, open(os.path.join(dst, "ncu_full_metrics.json"), "w"), indent=1)
    json.dump(summ, open(summ_path, "w"), indent=1)
    # launch list
    lf = os.path.join(src, "ncu_launches_c3.csv")
    if os.path.exists(lf):
        shutil.copy(lf, dst)
        rows = list(csv.reader(open(lf)))
        start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[start]
        d = defaultdict(list)
        for r in rows[start + 1:]:
            if len(r) > h.index("Metric Value"):
                d[r[h.index("Kernel Name")]].append(float(r[h.index("Metric Value")].replace(",", "")) / 1e3)
        step = {k: v for k, v in d.items() if "mppi" in k or "tc::" in k}
        per_step = sum(sum(v) / len(v) for k, v in step.items() if "k_fold" not in k)
        with open(os.path.join(dst, "ncu_launches_summary.txt"), "w") as f:
            f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none), bench.py --steps 3 --warmup 3, configs[3]\n")
            f.write("# cold-cache, serialised per-launch times: compare SHARES of one step, not absolutes\n")
            f.write(f"{'kernel':60s} launches  mean_us  share_of_step\n")
            for k, v in d.items():
                m = sum(v) / len(v)
                share = f"{m / per_step:.3f}" if k in step and "k_fold" not in k else "  -"
                f.write(f"{k[:60]:60s} {len(v):8d} {m:8.2f}  {share}\n")
    print(open(os.path.join(dst, "ncu_launches_summary.txt")).read() if os.path.exists(lf) else "no launch list")


if __name__ == "__main__":
    main()
