"""Summarise an ncu --set full report: headline pipe metrics and the SASS lines with the most stall samples.
python tools/ncu_hot.py REPORT.ncu-rep [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {v[i]:>14s} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hdr = srows[1]
data = [r for r in srows[2:] if len(r) > 3 and r[2].isdigit()]
tot = sum(int(r[2]) for r in data)
print("stall samples", tot)
for r in sorted(data, key=lambda r: -int(r[2]))[:n]:
    print(f"{int(r[2]):6d} {int(r[3]):6d} {r[0][-5:]} {r[1][:100]}")
