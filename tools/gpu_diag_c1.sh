# Diagnose the H = 128 path (configs[1]): timeline trace + ncu source-level stall attribution of K2.
mkdir -p gpurun_out
MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so timeout 120 python tests/trace_tc.py c1 8 > gpurun_out/tr_c1_now.txt 2>&1
MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so timeout 120 python tests/trace_tc.py c2 8 > gpurun_out/tr_c2_now.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 4 -c 1 -o /tmp/mlp_c1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1_diag.log 2>&1
python tools/ncu_hot.py /tmp/mlp_c1.ncu-rep 60 > gpurun_out/hot_c1.txt 2>&1
ncu -i /tmp/mlp_c1.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_c1_cuda.csv 2>&1
ncu -i /tmp/mlp_c1.ncu-rep --page details --csv > gpurun_out/details_c1.csv 2>&1
ls -la gpurun_out
