#!/bin/bash
# Round-2 check of the hand-written radix sort and scans: the balance / dispatch /
# compose / C++-API suites, then the per-kernel launch list of one warm balance
# call per C4 phase (ncu, single process).
o=gpurun_out/r02; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_balance.py tests/test_gpu_dispatch.py tests/test_gpu_compose.py tests/test_composed_golden.py tests/test_reference_suite.py tests/test_gpu_hosting.py -q -p no:cacheprovider > $o/pytest_sort.log 2>&1; echo "pytest rc=$? $(tail -1 $o/pytest_sort.log)"
for c in C4x30 C4x64; do for p in 0 1 2; do
  timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $o/kprof_${c}_$p.csv python scripts/kprof.py $c $p > $o/kprof_${c}_$p.log 2>&1
  echo "kprof $c $p rc=$?"
done; done
