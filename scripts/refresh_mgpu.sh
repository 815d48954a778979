#!/bin/bash
# Multi-GPU evidence refresh on one box of N GPUs (gpurun --gpus N): the N-GPU
# parity test, the driver's default line, C2/C3/C5 with the fused put and with
# NCCL, then the 2-GPU default line and C3/C5 puts on the first two GPUs.
N=${1:-4}
o=gpurun_out/refresh_mgpu; mkdir -p $o
run() {  # nproc tag args...
  local np=$1 tag=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > $o/$tag.json 2> $o/$tag.err
  echo "$tag rc=$?"
}
timeout 600 python -m pytest tests/test_multigpu.py -x -q > $o/test_multigpu_${N}.log 2>&1; echo "multigpu tests rc=$?"
run $N default_${N}gpu
for cfg in C2 C3 C5; do for ex in put nccl; do
  run $N ${cfg}_${ex}_${N}gpu --steps 10 --warmup 3 --config $cfg --exchange $ex
done; done
export CUDA_VISIBLE_DEVICES=0,1
run 2 default_2gpu
for cfg in C3 C5; do run 2 ${cfg}_put_2gpu --steps 10 --warmup 3 --config $cfg; done
run 2 C2_nccl_2gpu --steps 10 --warmup 3 --config C2 --exchange nccl
