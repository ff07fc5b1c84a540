# GPU: parity tests + bench lines for the configs in $CFGS (default c2 c1), stage breakdown printed.
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && { tail -40 gpurun_out/pytest_gpu.log; exit 1; }
for c in ${CFGS:-c2 c1}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline']
print('$c','ms %.4f'%d['ms_per_step'],'value %.3e'%d['value'],'frac %.3f'%r['frac'],{k:round(v,4) for k,v in r['stage_ms'].items()},d['clocks']['sm_mhz'])"
done
