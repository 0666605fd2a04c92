# DMMA triangle-launch disagreements by variant: 6 fresh processes x 20 reps each
mkdir -p gpurun_out
for v in base HSB_NO_TILE_ORDER HSB_NO_ZPLANES; do
  for i in 1 2 3 4 5 6; do
    if [ $v = base ]; then python probes/stress_dmma_phys.py 20 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/race_ab.txt;
    else env $v=1 python probes/stress_dmma_phys.py 20 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/race_ab.txt; fi
  done
done
