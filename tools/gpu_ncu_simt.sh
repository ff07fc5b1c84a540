# ncu --set full of the SIMT kernels: k_softmin at configs[3], k_rollout at configs[4]
mkdir -p gpurun_out
timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ns_c3.json 2>/dev/null; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_softmin -s 3 -c 1 -o gpurun_out/softmin_c3 -f python bench.py --config c3 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ncu_sm.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rollout -s 3 -c 1 -o gpurun_out/rollout_c4 -f python bench.py --config c4 --steps 2 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/ncu_ro.log 2>&1; echo "ncu2 rc=$?"
