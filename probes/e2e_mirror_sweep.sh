# bench e2e (pinned numpy A/B in, host H/S out) vs the host mirror's thread count
mkdir -p gpurun_out
for r in 1 2; do for th in 4 8 12 16; do
HSB_MIRROR_THREADS=$th python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-compare > gpurun_out/b41.json 2>gpurun_out/b41.err
python -c "
import json;d=json.loads(open('gpurun_out/b41.json').read().strip().splitlines()[-1])
print('$th', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), round(d['e2e_physical']['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/sweep41.txt
done; done
