#!/bin/bash
# End-of-round one-GPU evidence: C3 / C5 bench lines, the per-config balance sweep,
# the reference arm.
o=gpurun_out/final1; mkdir -p $o
python bench.py --config C3 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c3.json 2> $o/bench_c3.err; echo "c3 rc=$?"
python bench.py --config C5 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c5.json 2> $o/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench_configs.py --sweep --out $o/configs.jsonl > $o/configs.log 2>&1; echo "configs rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err; echo "ref rc=$?"
