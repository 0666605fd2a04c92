mkdir -p gpurun_out
for i in $(seq 1 5); do
  for w in none sleep dmma700 dmma2100once; do
    STRESS_WARM=$w python probes/stress_dmma_phys.py 6 2>&1 | grep -E "disagree|agreement" | sed "s/^/$w /" >> gpurun_out/race_ab3.txt
  done
done
