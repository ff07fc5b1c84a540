# ncu of the softmin kernel at configs[2]: duration and hot SASS lines.
mkdir -p gpurun_out
rm -f /tmp/small_c2.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_softmin -s 4 -c 1 -o /tmp/small_c2 \
  python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_small_c2.log 2>&1
python tools/ncu_hot.py /tmp/small_c2.ncu-rep 45 > gpurun_out/hot_softmin_c2.txt 2>&1
