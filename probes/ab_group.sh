# INT8 GEMM tile-group size (HSB_OZ_GROUP, default 6) at C3 and C4
mkdir -p gpurun_out
for r in 1 2; do for g in 6 4 8 12; do
  HSB_OZ_GROUP=$g python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/grp.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/grp.json').read().strip().splitlines()[-1]);print('C3 $g', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/group.txt
done; done
for g in 6 4 8 12; do
  HSB_OZ_GROUP=$g python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/grp.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/grp.json').read().strip().splitlines()[-1]);print('C4 $g', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/group.txt
done
