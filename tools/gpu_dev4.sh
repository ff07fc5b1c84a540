set -x
export MPPI_SKIP_BUILD=1
L=paper_2603_07199_b200
MPPI_LIB=$DEV_LIB timeout 600 python -m pytest tests -m gpu -q -rf -k "${DEV_TESTS}" > gpurun_out/pytest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dev.log
for c in ${AB_CFGS}; do timeout 400 python tests/ab_mlp.py $AB_LIBS --cfg=$c > gpurun_out/ab_$c.txt 2>&1; done
