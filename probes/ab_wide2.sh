# wide INT8 GEMM at C4 with different slab sizes
mkdir -p gpurun_out
for r in 1 2; do for v in "HSB_OZ_WIDE=1 HSB_OZ_SLAB_KB=32" "HSB_OZ_WIDE=1" "HSB_OZ_SLAB_KB=32"; do
  env $v python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w2.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/w2.json').read().strip().splitlines()[-1]);print('C4 $v |', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/wide2.txt
done; done
