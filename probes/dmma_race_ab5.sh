mkdir -p gpurun_out
for i in $(seq 1 8); do
  STRESS_CFGS=lmax python probes/stress_dmma_phys.py 6 2>&1 | grep -E "disagree|agreement" | sed "s/^/lmax /" >> gpurun_out/race_ab5.txt
done
