#!/bin/bash
# A/B of an environment knob on the multi-GPU bench line.
# usage: ab_env.sh N VAR "v1 v2 ..." "C2 C5 ..." tag [extra bench args]
N=$1; VAR=$2; VALS=$3; CFGS=$4; tag=$5; shift 5
out=gpurun_out/ab_${tag}.jsonl; : > $out
for cfg in $CFGS; do for v in $VALS; do
  env $VAR=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 10 --warmup 3 --config $cfg "$@" 2> gpurun_out/ab_${tag}_${cfg}_${v}.err | sed "s/^{/{\"ab\": \"$VAR=$v\", /" >> $out
  echo "$cfg $VAR=$v rc=${PIPESTATUS[0]}"
done; done
python - <<'PY' $out
import json,sys
for l in open(sys.argv[1]):
    if not l.startswith("{"): continue
    d=json.loads(l); a=d.get("a2a",{})
    print(d["ab"], d["config"]["workload"][:3], d["n_gpus"], f'{d["value"]/1e6:.1f}M tok/s', f'{d["ms_per_step"]:.3f} ms', f'busbw {a.get("busbw_gbs_rank",0):.0f}', f'e2e {d["e2e"]["value"]/1e6:.1f}M')
PY
