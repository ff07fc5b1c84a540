# development GPU check against a dev build (MPPI_LIB=$DEV_LIB): selected parity tests, then A/B timing
set -x
mkdir -p gpurun_out
export MPPI_SKIP_BUILD=1
export MPPI_LIB=${DEV_LIB:-paper_2603_07199_b200/libmppi_b200_dev.so}
timeout 600 python -m pytest tests -m gpu -q -rf -k "${DEV_TESTS:-c1s or c1pes or c4s or c1 or c4 or ragged or single}" > gpurun_out/pytest_dev.log 2>&1; rc=$?
echo "pytest rc=$rc" >> gpurun_out/pytest_dev.log
tail -25 gpurun_out/pytest_dev.log
for cfg in ${AB_CFGS:-c1 c4}; do
  timeout 300 python tests/ab_mlp.py $AB_LIBS --cfg=$cfg > gpurun_out/ab_$cfg.txt 2>&1
  cat gpurun_out/ab_$cfg.txt
done
