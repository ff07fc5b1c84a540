# H = 128 A/B: issuer probes each barrier once before its wait loop (H128_WAIT_FIRST)
mkdir -p gpurun_out
L=paper_2603_07199_b200
for c in c4 c1; do
  timeout 400 python tests/ab_mlp.py $L/libmppi_b200.so $L/libmppi_b200_wf.so --cfg=$c > gpurun_out/ab_wf_$c.txt 2>&1; cat gpurun_out/ab_wf_$c.txt
done
