# Round-end evidence on one B200: GPU tests, smoke, bench lines (C3 default
# contract, C4, C5, reference arm), launch list.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/fin_gputests.log 2>&1
python __graft_entry__.py > gpurun_out/fin_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err
python bench.py --config C5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-compare --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu.log 2>&1
