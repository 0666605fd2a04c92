python -m pytest tests/test_gpu_build.py -m gpu -q -x -k "lower_triangle or kpoint or pageable or pinned" > gpurun_out/gt37.log 2>&1
for r in 1 2; do for x in 0 0.2 0.35 0.5; do
HSB_D2H_UPPER=$x python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-compare > gpurun_out/b37.json 2>gpurun_out/b37.err
python -c "
import json;d=json.loads(open('gpurun_out/b37.json').read().strip().splitlines()[-1])
print('$x', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), round(d['e2e_physical']['ms_per_step'],2), d['e2e']['d2h_bytes_per_step'], d['clocks']['sm_mhz'])" >> gpurun_out/sweep37.txt
done; done
