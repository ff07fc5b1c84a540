# L1M (H = 256 layer 1 as an MMA) A/B and timeline trace at configs[2]
mkdir -p gpurun_out
L=paper_2603_07199_b200
timeout 300 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_l1m.so $L/libmppi_b200_l1mall.so --cfg=c2 > gpurun_out/ab2_c2.txt 2>&1; cat gpurun_out/ab2_c2.txt
MPPI_LIB=$PWD/$L/libmppi_b200_trace_l1m.so MPPI_SKIP_BUILD=1 timeout 120 python tests/trace_tc.py c2 8 > gpurun_out/trace_l1m_c2.txt 2>&1; tail -3 gpurun_out/trace_l1m_c2.txt
