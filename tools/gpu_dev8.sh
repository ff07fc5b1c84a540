set -x
export MPPI_SKIP_BUILD=1
L=paper_2603_07199_b200
for c in c4 c2 c3; do timeout 400 python tests/ab_mlp.py $L/libmppi_b200_r56.so $L/libmppi_b200_dev.so --cfg=$c > gpurun_out/ab_$c.txt 2>&1; done
export MPPI_LIB=$L/libmppi_b200_dev.so
for c in c3 c4; do for f in 0 1; do MPPI_FUSED=$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/bench_${c}_fused$f.json 2>&1; done; done
