#!/bin/bash
# One-GPU evidence refresh for round 2 (each ncu pass after its command ran clean):
# the driver's bench line, the reference arm, C3/C5 lines, the per-config balance
# evidence, the C++ API call for call, stage clocks, the ncu launch list and one
# ncu --set full capture of the row mover, then the bounds-checked suite.
o=gpurun_out/refresh2; mkdir -p $o
python bench.py > $o/bench_1gpu.json 2> $o/bench_1gpu.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err; echo "ref rc=$?"
python bench.py --config C3 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c3.json 2> $o/bench_c3.err; echo "c3 rc=$?"
python bench.py --config C5 --no-cpu-baseline --steps 10 --warmup 3 > $o/bench_c5.json 2> $o/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench_configs.py --sweep --out $o/configs.jsonl > $o/configs.log 2>&1; echo "configs rc=$?"
bash scripts/cpp_api_compare.sh; cp gpurun_out/cpp_api_b200.jsonl gpurun_out/cpp_api_ref.jsonl $o/; echo "cpp api rc=$?"
ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so timeout 300 python scripts/small_prof.py C1 C2 C3 C5 > $o/small_prof.log 2>&1
ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so timeout 300 python scripts/lpt_prof.py > $o/lpt_prof.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $o/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_move_tma -s 8 -c 2 \
    -o $o/k_move_tma_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_full.log 2>&1; echo "ncu full rc=$?"
bash scripts/checked_suite.sh
exit 0
