# Timeline traces of K2 (MPPI_TC_TRACE builds) for the configs in $TR_CFGS and the trace libraries in $TR_LIBS.
mkdir -p gpurun_out
for lib in ${TR_LIBS:-paper_2603_07199_b200/libmppi_b200_trace.so}; do
  for c in ${TR_CFGS:-c1 c2}; do
    MPPI_LIB=$lib timeout 120 python tests/trace_tc.py $c 8 > gpurun_out/tr_${c}_$(basename $lib .so).txt 2>&1
  done
done
