# fused vs unfused at the small configurations (configs[1], configs[2])
mkdir -p gpurun_out
for r in 1 2; do for c in c1 c2; do for f in 0 1; do
  MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/fs_${c}_f${f}_r$r.json 2>>gpurun_out/fs.err
done; done; done
