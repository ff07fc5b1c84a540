# One GPU session producing the round's committed evidence (profiles/$ROUND): bench lines, the reference
# arm, the ncu launch list of the default bench, and ncu --set full captures of the kernels.
# usage (on the GPU box): ROUND=r01 bash tools/gpu_profile_round.sh
set -x
R=${ROUND:-r01}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > $O/gpu.txt
lscpu | grep -E "^CPU\(s\)|Model name" > $O/cpu.txt
timeout 300 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
cp gpurun_out/clocks_rank0.csv $O/clocks_last_run.csv
for c in c1 c3 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for c in c2 c1 c4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 4 -c 1 -o $O/mlp_$c \
    python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_mlp_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rollout|k_softmin" -s 8 -c 2 -o $O/small_c2 \
  python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_small.log 2>&1
ls -la $O
