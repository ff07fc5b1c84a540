# H = 256 A/B: issuer probes each barrier once before its suspend-hint wait loop (MPPI_WAIT_FIRST)
mkdir -p gpurun_out
L=paper_2603_07199_b200
MPPI_LIB=$PWD/$L/libmppi_b200_wf.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c2 or h256" > gpurun_out/pytest_wf.log 2>&1; echo "wf pytest rc=$?"; tail -1 gpurun_out/pytest_wf.log
for c in c2 c3; do
  timeout 400 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_wf.so --cfg=$c > gpurun_out/ab_wf2_$c.txt 2>&1; cat gpurun_out/ab_wf2_$c.txt | cut -c1-330
done
