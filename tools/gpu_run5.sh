# H = 256 A/B: TS-form B descriptors by address-field adds (MPPI_DESC_ADD); bench stage times at c3
mkdir -p gpurun_out
L=paper_2603_07199_b200
MPPI_LIB=$PWD/$L/libmppi_b200_desc.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c2 or c3 or h256 or c5" > gpurun_out/pytest_desc2.log 2>&1; echo "desc pytest rc=$?"; tail -2 gpurun_out/pytest_desc2.log
for c in c2 c3 c2pe; do
  timeout 400 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_desc.so --cfg=$c > gpurun_out/ab_desc2_$c.txt 2>&1; cat gpurun_out/ab_desc2_$c.txt
done
