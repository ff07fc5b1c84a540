# fused vs unfused step A/B (interleaved, 2 rounds) for configs[4] and configs[3]
mkdir -p gpurun_out
for r in 1 2; do for c in c4 c3; do for f in 0 1; do
  MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fab_${c}_f${f}_r$r.json 2>>gpurun_out/fab.err
done; done; done
