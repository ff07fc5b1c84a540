set -x
export MPPI_SKIP_BUILD=1
export MPPI_LIB=${DEV_LIB}
timeout 900 python -m pytest tests -m gpu -q -rf -k "${DEV_TESTS}" > gpurun_out/pytest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dev.log
for c in ${BENCH_CFGS}; do for f in 0 1; do MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/bench_${c}_fused$f.json 2>&1; done; done
