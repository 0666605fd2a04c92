# wide INT8 GEMM work items (HSB_OZ_WIDE): correctness, then C3/C4 time, clock and DRAM traffic
mkdir -p gpurun_out
HSB_OZ_WIDE=1 python -m pytest tests/test_gpu_build.py tests/test_gpu_sweep.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/wide_tests.log 2>&1
tail -1 gpurun_out/wide_tests.log >> gpurun_out/wide.txt
HSB_OZ_WIDE=1 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -x > gpurun_out/wide_tests2.log 2>&1
tail -1 gpurun_out/wide_tests2.log >> gpurun_out/wide.txt
for r in 1 2; do for v in base HSB_OZ_WIDE=1; do
  if [ $v = base ]; then python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w.json 2>&1;
  else env $v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w.json 2>&1; fi
  python -c "
import json;d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1]);print('C3 $v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/wide.txt
done; done
for r in 1 2; do for v in base HSB_OZ_WIDE=1; do
  if [ $v = base ]; then python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w.json 2>&1;
  else env $v python bench.py --config C4 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline --no-compare > gpurun_out/w.json 2>&1; fi
  python -c "
import json;d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1]);print('C4 $v', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/wide.txt
done; done
HSB_OZ_WIDE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ozaki_gemm_kernel -s 1 -c 1 --csv python bench.py --config C4 --steps 1 --warmup 0 --no-compare --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time|xbar|imma|cycles_elapsed" | awk -F'","' '{print "ncu C4 wide", $(NF-2), $NF}' >> gpurun_out/wide.txt
