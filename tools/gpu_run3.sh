# H = 128 issue-order A/B (H128_L1LAG): parity of the variants, then interleaved MLP timing at configs[4] / [1]
mkdir -p gpurun_out
L=paper_2603_07199_b200
for v in lag2 lag1; do
  MPPI_LIB=$PWD/$L/libmppi_b200_$v.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c1 or c4 or h128 or fused" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"; tail -2 gpurun_out/pytest_$v.log
done
for c in c4 c1 c1pe; do
  timeout 400 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_lag1.so $L/libmppi_b200_lag2.so $L/libmppi_b200_lag3.so --cfg=$c > gpurun_out/ab_lag_$c.txt 2>&1; cat gpurun_out/ab_lag_$c.txt
done
