#!/bin/bash
# A/B of the N-GPU default line: the current tree against the round-1 tree
# checked out at old_r01/ (git worktree, built in place). Alternates 3 times.
N=${1:-2}
o=gpurun_out/ab; mkdir -p $o
for i in 1 2 3; do
  for tree in . old_r01; do
    tag=$(basename $(realpath $tree))
    (cd $tree && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus $N \
      --no-cpu-baseline > $OLDPWD/$o/${tag}_${N}_$i.json 2> $OLDPWD/$o/${tag}_${N}_$i.err)
    python -c "import json; d=json.loads(open('$o/${tag}_${N}_$i.json').read().strip().split(chr(10))[-1]); print('$tag', $i, round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1))"
  done
done
