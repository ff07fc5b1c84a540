# fused vs unfused step A/B (interleaved, 2 rounds) at configs[2] / configs[5] (H = 256, few blocks)
mkdir -p gpurun_out
for r in 1 2; do for c in c2 c5; do for f in 0 1; do
  MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fab3_${c}_f${f}_r$r.json 2>>gpurun_out/fab3.err
done; done; done
for f in gpurun_out/fab3_c*_f*_r*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'], d['roofline']['stage_ms'])"; done
tail -3 gpurun_out/fab3.err
