set -x
export MPPI_SKIP_BUILD=1 MPPI_LIB=paper_2603_07199_b200/libmppi_b200_dev.so
python tests/prof_mlp.py c4 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_h128 -s 1 -c 1 -o gpurun_out/h128_c4 python tests/prof_mlp.py c4 3 > gpurun_out/ncu_h128.log 2>&1
MPPI_H128_LEGACY=1 python tests/prof_mlp.py c4 3 > gpurun_out/plain2.log 2>&1 && \
MPPI_H128_LEGACY=1 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 1 -c 1 -o gpurun_out/legacy_c4 python tests/prof_mlp.py c4 3 > gpurun_out/ncu_legacy.log 2>&1
ls -la gpurun_out/*.ncu-rep
