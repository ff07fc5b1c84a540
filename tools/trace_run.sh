set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so timeout 300 python tests/trace_tc.py c1 8 > gpurun_out/trace_c1.txt 2>&1
MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so timeout 300 python tests/trace_tc.py c2 4 > gpurun_out/trace_c2.txt 2>&1
tail -3 gpurun_out/trace_c1.txt gpurun_out/trace_c2.txt
