mkdir -p gpurun_out
for i in $(seq 1 10); do
  python probes/stress_dmma_phys.py 20 2>&1 | grep -E "disagree|agreement" | sed "s/^/base /" >> gpurun_out/race_ab2.txt
  HSB_NO_ZPLANES=1 python probes/stress_dmma_phys.py 20 2>&1 | grep -E "disagree|agreement" | sed "s/^/noplanes /" >> gpurun_out/race_ab2.txt
done
