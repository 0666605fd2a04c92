# GEMM change check: GPU tests, 8-way shard launch lists (C3, C4), C3 bench x2, C3 launch list
mkdir -p gpurun_out
T=${1:-x}
python -m pytest tests -m gpu -q -x > gpurun_out/gt_$T.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shard_c3_$T.csv python probes/shard_launches.py C3 8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shard_c4_$T.csv python probes/shard_launches.py C4 8 > /dev/null 2>&1
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/b_$T.json 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b_$T.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_$T.txt; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 0 --no-compare --no-e2e --no-cpu-baseline > /dev/null 2>&1
