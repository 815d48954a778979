#!/bin/bash
# The driver's own commands at N = 2 (or 4): our arm and the reference arm.
o=gpurun_out/driver_style; mkdir -p $o
N=$(nvidia-smi -L | wc -l)
for impl in b200 reference; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 300)) bench.py --impl $impl --gpus $N --steps 10 --warmup 3 \
    > $o/${N}gpu_$impl.json 2> $o/${N}gpu_$impl.err
  echo "N=$N $impl rc=$? $(tail -1 $o/${N}gpu_$impl.json | cut -c1-300)"
done
