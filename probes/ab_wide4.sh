mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gt112.log 2>&1; tail -1 gpurun_out/gt112.log >> gpurun_out/wide4.txt
for r in 1 2; do for v in "HSB_OZ_NONE=1" "HSB_OZ_WIDE=1"; do
  env $v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w4.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/w4.json').read().strip().splitlines()[-1]);print('C3 $v |', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/wide4.txt
  env $v python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w4.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/w4.json').read().strip().splitlines()[-1]);print('C4 $v |', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/wide4.txt
done; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches112.csv python bench.py --steps 1 --warmup 0 --no-compare --no-e2e --no-cpu-baseline > /dev/null 2>&1
