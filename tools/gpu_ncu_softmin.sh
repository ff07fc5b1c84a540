mkdir -p gpurun_out
for c in c3 c4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_softmin -s 3 -c 1 -o gpurun_out/softmin2_$c -f python bench.py --config $c --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ncu_sm_$c.log 2>&1; echo "ncu $c rc=$?"
done
