# A/B of an environment switch on the C3 bench (alternating, 3 rounds): $1 = tag, $2 = VAR=value
mkdir -p gpurun_out
for r in 1 2 3; do for v in base "$2"; do
  if [ "$v" = base ]; then python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/abenv.json 2>&1;
  else env $v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/abenv.json 2>&1; fi
  python -c "
import json;d=json.loads(open('gpurun_out/abenv.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/abenv_$1.txt
done; done
