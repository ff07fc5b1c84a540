# GPU check of a kernel change: parity tests, then A/B MLP timing of the builds named in $AB_LIBS.
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
for cfg in ${AB_CFGS:-c2 c1 c4}; do
  timeout 250 python tests/ab_mlp.py ${AB_LIBS:-paper_2603_07199_b200/libmppi_b200_old.so paper_2603_07199_b200/libmppi_b200.so} --cfg=$cfg > gpurun_out/ab_$cfg.txt 2>&1
  cat gpurun_out/ab_$cfg.txt
done
