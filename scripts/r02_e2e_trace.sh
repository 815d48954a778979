#!/bin/bash
# per-step host times of the e2e loops at N GPUs (ORCH_BENCH_E2E_TRACE)
o=gpurun_out/e2e_trace; mkdir -p $o
N=$(nvidia-smi -L | wc -l)
for rep in 1 2 3 4; do
  ORCH_BENCH_E2E_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus $N --steps 40 \
    > $o/${N}_$rep.json 2> $o/${N}_$rep.err
  echo "rep=$rep $(tail -1 $o/${N}_$rep.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); e=j['e2e']; print(round(j['value']/1e6,1), round(e['value']/1e6,1), round(e['sync_value']/1e6,1))" 2>&1 | tail -1)"
  grep "\[e2e" $o/${N}_$rep.err
done
