#!/bin/bash
# e2e pipelining depth (ORCH_E2E_DEPTH = steps issued beyond the one waited for)
o=gpurun_out/e2e_depth; mkdir -p $o
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do
  [ $N -gt $NG ] && continue
  for D in 1 2 3; do
    if [ $N = 1 ]; then
      ORCH_E2E_DEPTH=$D timeout 400 python bench.py --no-cpu-baseline > $o/${N}_$D.json 2> $o/${N}_$D.err
    else
      ORCH_E2E_DEPTH=$D CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N - 1))) timeout 400 python -m torch.distributed.run \
        --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) \
        bench.py --gpus $N > $o/${N}_$D.json 2> $o/${N}_$D.err
    fi
    echo "N=$N depth=$D rc=$? $(python -c "import json; j=json.loads(open('$o/${N}_$D.json').read().splitlines()[-1]); e=j['e2e']; print(round(j['value']/1e6,1), round(e['value']/1e6,1), round(e['sync_value']/1e6,1))" 2>&1 | tail -1)"
  done
done
