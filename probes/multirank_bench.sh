# bench.py under torchrun with 2 ranks sharing one GPU (gloo: host-staged collectives), every exchange path
mkdir -p gpurun_out
for rs in nccl tri fused; do
  HSB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config C2 --steps 2 --warmup 3 --rs $rs --no-e2e --no-cpu-baseline --no-compare > gpurun_out/mr_$rs.json 2> gpurun_out/mr_$rs.err
  echo "$rs rc=$?" >> gpurun_out/mr.txt
  tail -1 gpurun_out/mr_$rs.json | cut -c1-200 >> gpurun_out/mr.txt
done
HSB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --impl reference --config C2 --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$?" >> gpurun_out/mr.txt; tail -1 gpurun_out/mr_ref.json | cut -c1-160 >> gpurun_out/mr.txt
