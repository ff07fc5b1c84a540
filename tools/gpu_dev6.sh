set -x
export MPPI_SKIP_BUILD=1
export MPPI_LIB=${DEV_LIB}
for c in c1 c2 c5; do for f in 0 1; do MPPI_SPLIT_NOISE=$f timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${c}_split$f.json 2>&1; done; done
