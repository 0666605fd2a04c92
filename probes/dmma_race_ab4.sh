mkdir -p gpurun_out
for i in $(seq 1 6); do
  for w in none fullpass; do
    STRESS_WARM=$w python probes/stress_dmma_phys.py 6 2>&1 | grep -E "disagree|agreement" | sed "s/^/$w /" >> gpurun_out/race_ab4.txt
  done
done
