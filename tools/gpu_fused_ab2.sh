# fused vs unfused step A/B (interleaved, 2 rounds) for configs[4] and configs[1]
mkdir -p gpurun_out
for r in 1 2; do for c in c4 c1; do for f in 0 1; do
  MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fab_${c}_f${f}_r$r.json 2>>gpurun_out/fab.err
done; done; done
for f in gpurun_out/fab_c*_f*_r*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'])"; done
