# rollout / fused A/B on the GPU box: parity of the rollout paths, then c4 and c3 stage times unfused and fused
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "rollout or fused or queries or noise or clamp or closed_loop or full_size" > gpurun_out/pytest_ro.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ro.log
for c in c4 c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/ro_$c.json 2>>gpurun_out/ro.err
  MPPI_FUSED=1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/ro_${c}_fused.json 2>>gpurun_out/ro.err
done
tail -n 3 gpurun_out/pytest_ro.log
