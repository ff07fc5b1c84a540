mkdir -p gpurun_out
L=paper_2603_07199_b200
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 250 python tests/ab_mlp.py $L/libmppi_b200_old.so $L/libmppi_b200.so --cfg=c2pe > gpurun_out/ab_c2pe.txt 2>&1; cat gpurun_out/ab_c2pe.txt
timeout 250 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_l1m.so --cfg=c2 > gpurun_out/ab_c2.txt 2>&1; cat gpurun_out/ab_c2.txt
MPPI_LIB=$PWD/$L/libmppi_b200_l1m.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2 or c3" > gpurun_out/pytest_l1m.log 2>&1; echo "l1m pytest rc=$?"; tail -3 gpurun_out/pytest_l1m.log
