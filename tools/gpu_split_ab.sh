# warp-specialised rollout (k_rollout_split) vs the one-thread form: parity tests, then stage times
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
for r in 1 2; do for c in c1 c2; do for v in 0 1; do
  MPPI_ROLLOUT_NOSPLIT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/split_${c}_ns${v}_r$r.json 2>>gpurun_out/split.err
done; done; done
