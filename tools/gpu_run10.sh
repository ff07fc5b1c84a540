# configs[3] step A/B: unfused vs fused (control warpgroup 80 registers) vs fused (64: epilogue 104)
mkdir -p gpurun_out
L=$PWD/paper_2603_07199_b200
for r in 1 2; do
  MPPI_FUSED=0 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fc_u_r$r.json 2>>gpurun_out/fc.err
  MPPI_FUSED=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fc_f80_r$r.json 2>>gpurun_out/fc.err
  MPPI_LIB=$L/libmppi_b200_fc64.so MPPI_SKIP_BUILD=1 MPPI_FUSED=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fc_f64_r$r.json 2>>gpurun_out/fc.err
done
for f in gpurun_out/fc_*_r*.json; do python -c "
import json;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
tail -3 gpurun_out/fc.err
