#!/bin/bash
# The default bench line at 1, 2 and 4 GPUs (e2e with two steps in flight; the
# line carries the synchronous loop's figure as e2e.sync_value).
o=gpurun_out/e2e_pipe; mkdir -p $o
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do
  [ $N -gt $NG ] && continue
  if [ $N = 1 ]; then
    timeout 400 python bench.py > $o/${N}gpu.json 2> $o/${N}gpu.err
  else
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N - 1))) timeout 400 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py \
      --gpus $N > $o/${N}gpu.json 2> $o/${N}gpu.err
  fi
  echo "N=$N rc=$? $(python -c "import json,sys; j=json.loads(open('$o/${N}gpu.json').read().splitlines()[-1]); e=j['e2e']; print(round(j['value']/1e6,1), round(e['value']/1e6,1), round(e['sync_value']/1e6,1))" 2>&1)"
done
