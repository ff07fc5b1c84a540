set -x
export MPPI_SKIP_BUILD=1
L=paper_2603_07199_b200
MPPI_LIB=$L/libmppi_b200_dev.so timeout 600 python -m pytest tests -m gpu -q -rf -k "constructed_relu_net_is_exact or (random_weights_rows and (over0 or over1 or over5)) or bf16_step_parity or multi_controller or tiles_across or ragged or single_sample or full_size_sampled or zero_velocity or softmin_weights" > gpurun_out/pytest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dev.log
for c in c4 c1 c1pe; do timeout 400 python tests/ab_mlp.py $L/libmppi_b200_w4.so $L/libmppi_b200_dev.so --cfg=$c > gpurun_out/abw_$c.txt 2>&1; done
MPPI_LIB=$L/libmppi_b200_trace.so MPPI_TRACE_H128=1 timeout 300 python tests/trace_h128.py c4 12 > gpurun_out/trace_h128_c4.txt 2>&1
