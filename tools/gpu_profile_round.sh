# One GPU session producing the round's committed evidence (profiles/$ROUND): bench lines, the reference
# arm, the ncu launch list of the default bench, and ncu --set full captures of the kernels.
# usage (on the GPU box): ROUND=r02 bash tools/gpu_profile_round.sh
set -x
R=${ROUND:-r02}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > $O/gpu.txt
lscpu | grep -E "^CPU\(s\)|Model name" > $O/cpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err   # the default line (+ c2/c1/c4/c5 keys)
cp gpurun_out/clocks_rank0.csv $O/clocks_last_run.csv
for c in c1pe c2pe; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > $O/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches_c3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > $O/ncu_launch.log 2>&1
for c in c3 c2 c1 c4 c2pe; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp -s 4 -c 1 -o $O/mlp_$c \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_mlp_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout|k_softmin" -s 8 -c 2 -o $O/small_c3 \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_small.log 2>&1
# summarise here (ncu CLI), keep the small outputs, drop the large reports (gpurun merges <= 64 MiB)
mkdir -p gpurun_out/${R}_out
cp profiles/ncu_mlp_summary.json gpurun_out/ncu_mlp_summary.json 2>/dev/null
python tools/profile_summary.py $R $O gpurun_out/${R}_out > gpurun_out/${R}_out/summary.log 2>&1
for f in $O/*.ncu-rep; do ncu -i $f --page source --csv --print-source sass > ${f%.ncu-rep}_source.csv 2>/dev/null; done
ls -la $O gpurun_out/${R}_out
rm -f $O/*.ncu-rep
