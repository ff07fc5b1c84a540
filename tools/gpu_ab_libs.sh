# A/B of library variants on one box: bench stage times per config. Usage: bash tools/gpu_ab_libs.sh "c4 c3" lib1.so lib2.so ...
mkdir -p gpurun_out
cfgs="$1"; shift
for lib in "$@"; do
  tag=$(basename $lib .so)
  for c in $cfgs; do
    MPPI_LIB=$PWD/paper_2603_07199_b200/$lib MPPI_SKIP_BUILD=1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/ab_${tag}_$c.json 2>>gpurun_out/ab.err
  done
done
