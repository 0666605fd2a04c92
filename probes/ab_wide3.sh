# wide INT8 GEMM combined with slab size / tile-group shape at C4
mkdir -p gpurun_out
for r in 1 2; do for v in "HSB_OZ_NONE=1" "HSB_OZ_WIDE=1" "HSB_OZ_WIDE=1 HSB_OZ_SLAB_KB=8" "HSB_OZ_WIDE=1 HSB_OZ_GROUP=8" "HSB_OZ_WIDE=1 HSB_OZ_GROUP=12"; do
  env $v python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w3.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/w3.json').read().strip().splitlines()[-1]);print('C4 $v |', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/wide3.txt
done; done
