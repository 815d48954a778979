#!/bin/bash
# The fused put into NCCL symmetric-memory windows (orch_window_create_nccl)
# against CUDA IPC windows: the multi-GPU parity test, then bench lines.
o=gpurun_out/nccl_window; mkdir -p $o
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest -q -x tests/test_multigpu.py > $o/pytest_mgpu.log 2>&1; echo "mgpu tests rc=$? $(tail -1 $o/pytest_mgpu.log)"
for cfg in ${CFGS:-C2 C5}; do
  for ex in ${EXS:-put put-nccl nccl}; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 300)) bench.py --gpus $N --config $cfg --exchange $ex \
      > $o/${N}gpu_${cfg}_$ex.json 2> $o/${N}gpu_${cfg}_$ex.err
    echo "N=$N $cfg $ex rc=$? $(python -c "import json; j=json.loads(open('$o/${N}gpu_${cfg}_$ex.json').read().splitlines()[-1]); a=j['a2a']; print(round(j['value']/1e6,1), 'busbw', round(a['busbw_gbs_rank'],1), 'frac nccl', round(a['frac_of_nccl_ceiling'],3), 'e2e', round(j['e2e']['value']/1e6,1))" 2>&1 | tail -1)"
  done
done
