# H = 128 A/B: GEMM descriptors by address-field adds (H128_DESC_ADD)
mkdir -p gpurun_out
L=paper_2603_07199_b200
MPPI_LIB=$PWD/$L/libmppi_b200_desc.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c1 or c4 or h128" > gpurun_out/pytest_desc.log 2>&1; echo "desc pytest rc=$?"; tail -2 gpurun_out/pytest_desc.log
for c in c4 c1; do
  timeout 400 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_desc.so --cfg=$c > gpurun_out/ab_desc_$c.txt 2>&1; cat gpurun_out/ab_desc_$c.txt
done
