#!/bin/bash
# One-GPU evidence refresh: the driver's bench line, the reference arm, the
# per-config balance evidence, the C3/C5 single-GPU lines, the ncu launch list
# and one ncu --set full capture of the row mover (after each command ran clean).
set -x
o=gpurun_out/refresh; mkdir -p $o
python bench.py > $o/bench_1gpu.json 2> $o/bench_1gpu.err
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err
python bench.py --config C3 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c3.json 2> $o/bench_c3.err
python bench.py --config C5 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c5.json 2> $o/bench_c5.err
python bench_configs.py --sweep --out $o/configs.jsonl > $o/configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $o/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_move_tma -s 8 -c 2 \
    -o $o/k_move_tma_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_balance_small -s 8 -c 1 \
    -o $o/k_balance_small_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_small.log 2>&1
ls -la $o
