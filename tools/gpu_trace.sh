# Timeline traces of K2 (MPPI_TC_TRACE build) for the configs in $TR_CFGS.
mkdir -p gpurun_out
for c in ${TR_CFGS:-c1 c2}; do
  MPPI_LIB=paper_2603_07199_b200/libmppi_b200_trace.so timeout 120 python tests/trace_tc.py $c 8 > gpurun_out/tr_${c}_now.txt 2>&1
done
