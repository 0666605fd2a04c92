# C4 bench with different INT8 GEMM slab sizes (k bytes per work item): DRAM traffic vs slab epilogues
mkdir -p gpurun_out
for r in 1 2; do for kb in 16 8 4; do
  HSB_OZ_SLAB_KB=$kb python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/slab.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/slab.json').read().strip().splitlines()[-1]);print('$kb', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/slab_c4.txt
done; done
for kb in 16 4; do
  HSB_OZ_SLAB_KB=$kb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ozaki_gemm_kernel -s 1 -c 1 --csv python bench.py --config C4 --steps 1 --warmup 0 --no-compare --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/$kb /" >> gpurun_out/slab_c4.txt
done
