#!/bin/bash
# A/B: windows in NCCL symmetric memory (put-nccl: gather + rows) against CUDA IPC (put)
o=gpurun_out/gather_ab; mkdir -p $o
N=$(nvidia-smi -L | wc -l)
for rep in 1 2 3; do
  for ex in put-nccl put; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 300)) bench.py --gpus $N --exchange $ex \
      > $o/${N}_${ex}_$rep.json 2> $o/${N}_${ex}_$rep.err
    echo "N=$N $ex rep=$rep rc=$? $(tail -1 $o/${N}_${ex}_$rep.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); e=j['e2e']; print(round(j['value']/1e6,1), round(e['value']/1e6,1), round(e['sync_value']/1e6,1), j['windows'])" 2>&1 | tail -1)"
  done
done
