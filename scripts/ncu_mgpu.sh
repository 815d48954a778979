#!/bin/bash
# Launch lists of the N > 1 exchange with ncu on rank 0 only (one GPU under the
# profiler; the other ranks run plain), 2..N GPUs of one box:
#   scripts/ncu_mgpu.sh N exchange [config]   -> gpurun_out/ncu_<exchange>_<config>_<N>gpu.csv
# The metadata all-gather and the step barrier go through NCCL here, so a rank
# slowed down by the profiler never trips the peer-memory waits' 4 s timeouts.
# gpu__time_duration is a single-pass metric: no kernel replay, so NCCL kernels
# are measured as they run.
N=$1; EX=$2; CFG=${3:-C2}
export MASTER_ADDR=127.0.0.1 MASTER_PORT=$((29600 + RANDOM % 300)) WORLD_SIZE=$N
o=gpurun_out/ncu_${EX}_${CFG}_${N}gpu
for r in $(seq 1 $((N - 1))); do
  RANK=$r LOCAL_RANK=$r timeout 900 python bench.py --gpus $N --steps 5 --warmup 3 --config $CFG \
    --exchange $EX --gather nccl --barrier nccl > $o.r$r.log 2>&1 &
done
RANK=0 LOCAL_RANK=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o.csv python bench.py --gpus $N --steps 5 --warmup 3 --config $CFG --exchange $EX \
  --gather nccl --barrier nccl > $o.r0.log 2>&1
echo "ncu rank0 rc=$?"
wait
