#!/bin/bash
# usage: mgpu.sh N tag
N=$1; tag=$2
out=gpurun_out/mgpu_${tag}.jsonl; : > $out
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_test_${tag}.log 2>&1; echo "multigpu tests rc=$?"
for cfg in C2 C3 C5; do for ex in put nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --config $cfg --exchange $ex >> $out 2> gpurun_out/mgpu_${tag}_${cfg}_${ex}.err
  echo "$cfg $ex rc=$?"
done; done
python - <<'PY' $out
import json,sys
for l in open(sys.argv[1]):
    if not l.startswith("{"): continue
    d=json.loads(l); a=d.get("a2a",{})
    print(d["config"]["workload"][:3], d.get("exchange"), d["n_gpus"], f'{d["value"]/1e6:.1f}M tok/s', f'{d["ms_per_step"]:.3f} ms', f'busbw {a.get("busbw_gbs_rank",0):.0f}', f'eg {a.get("max_egress_bytes",0)/1e6:.0f}MB in {a.get("max_ingress_bytes",0)/1e6:.0f}MB', f'e2e {d["e2e"]["value"]/1e6:.1f}M')
PY
