# H = 256 A/B: hidden biases in the epilogue (MPPI_BIAS_EPI=1, pipelined D loads) vs the bias MMA
mkdir -p gpurun_out
L=$PWD/paper_2603_07199_b200
MPPI_LIB=$L/libmppi_b200_be.so MPPI_SKIP_BUILD=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c2s or c3s or h256" > gpurun_out/pytest_be.log 2>&1; echo "be pytest rc=$?"; tail -1 gpurun_out/pytest_be.log
for r in 1 2; do
  timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/be_d_r$r.json 2>>gpurun_out/be.err
  MPPI_LIB=$L/libmppi_b200_be.so MPPI_SKIP_BUILD=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/be_b_r$r.json 2>>gpurun_out/be.err
done
for f in gpurun_out/be_*_r*.json; do python -c "
import json;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],4), round(d['roofline']['stage_ms']['sdf_mlp'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 300 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_be.so --cfg=c2 > gpurun_out/ab_be_c2.txt 2>&1; cut -c1-300 gpurun_out/ab_be_c2.txt
