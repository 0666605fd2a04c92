# C3 bench vs the SMs the V products leave to the side preparation (HSB_V_RESERVE_SMS)
mkdir -p gpurun_out
for r in 1 2; do for v in 0 20 30 40; do
  HSB_V_RESERVE_SMS=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/res.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/res.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), round(d['sections_ms']['loop1'],3), d['clocks']['sm_mhz'])" >> gpurun_out/reserve.txt
done; done
