#!/bin/bash
# Four-GPU round-2 evidence: NVLink ceilings, the N-GPU parity test and the
# exchange sweep, the driver-style default line at 4 and 2 GPUs, and rank-0
# ncu launch lists of the put and the NCCL exchange.
o=gpurun_out/r02; mkdir -p $o
paper_2503_23830_b200/lib/p2pbench 1024 > gpurun_out/p2p_4gpu.jsonl 2>&1; echo "p2pbench rc=$?"
bash scripts/mgpu_sweep.sh 4 r02f "C2 C3 C5" "put nccl"
for N in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N - 1))) timeout 400 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py \
    --gpus $N > $o/default_${N}gpu.json 2> $o/default_${N}gpu.err; echo "default $N rc=$?"
done
CUDA_VISIBLE_DEVICES=0,1 bash scripts/ncu_mgpu.sh 2 put C2
CUDA_VISIBLE_DEVICES=0,1 bash scripts/ncu_mgpu.sh 2 nccl C2
bash scripts/ncu_mgpu.sh 4 put C2
bash scripts/ncu_mgpu.sh 4 nccl C2
exit 0
