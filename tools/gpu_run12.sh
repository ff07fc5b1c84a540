# H = 256 PE: compact bias MMA (default) vs biases in the epilogue (MPPI_BIAS_EPI=1 build, the previous PE form)
mkdir -p gpurun_out
L=$PWD/paper_2603_07199_b200
timeout 600 python -m pytest tests -m gpu -q -x -k "pe" > gpurun_out/pytest_cb.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_cb.log
timeout 300 python tests/ab_mlp.py $L/libmppi_b200_oldpe.so $L/libmppi_b200.so --cfg=c2pe > gpurun_out/ab_cb_c2pe.txt 2>&1; cut -c1-300 gpurun_out/ab_cb_c2pe.txt
