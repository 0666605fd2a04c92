mkdir -p gpurun_out
for i in $(seq 1 8); do
  STRESS_WARM=none python probes/stress_dmma_phys.py 4 2>&1 | grep -E "disagreements" >> gpurun_out/race_pad.txt
done
