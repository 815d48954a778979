#!/bin/bash
# Multi-GPU exchange sweep on one box of N GPUs (gpurun --gpus N):
#   scripts/mgpu_sweep.sh N tag [configs] [exchanges]
# the N-GPU parity test, then bench.py per (config, exchange) -> gpurun_out/mgpu_<tag>.jsonl
N=$1; tag=$2; CFGS=${3:-"C2 C3 C5"}; EXS=${4:-"put nccl nccl-sync nccl-direct"}
out=gpurun_out/mgpu_${tag}.jsonl; : > $out
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_test_${tag}.log 2>&1; echo "multigpu tests rc=$?"
for cfg in $CFGS; do for ex in $EXS; do
  # an exchange name may carry +reg (--nccl-register) and @VAR=val,VAR=val (environment)
  extra=""; envs=""; e=$ex
  case $e in *@*) envs=$(echo ${e#*@} | tr ',' ' '); e=${e%@*};; esac
  case $e in *+reg) e=${e%+reg}; extra=--nccl-register;; esac
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $N --steps 10 --warmup 3 --config $cfg \
    --exchange $e $extra >> $out 2> gpurun_out/mgpu_${tag}_${cfg}_${ex}.err
  echo "$cfg $ex rc=$?"
done; done
python - <<'PY' $out
import json,sys
for l in open(sys.argv[1]):
    if not l.startswith("{"): continue
    d=json.loads(l); a=d.get("a2a",{})
    print(d["config"]["workload"][:3], d.get("exchange"), d["n_gpus"], f'{d["value"]/1e6:.1f}M tok/s', f'{d["ms_per_step"]:.3f} ms', f'busbw {a.get("busbw_gbs_rank",0):.0f}', f'eg {a.get("max_egress_bytes",0)/1e6:.0f}MB in {a.get("max_ingress_bytes",0)/1e6:.0f}MB', f'e2e {d["e2e"]["value"]/1e6:.1f}M')
PY
