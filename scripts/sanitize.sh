#!/bin/bash
# compute-sanitizer over the single-GPU -m gpu suite (the library's kernels only:
# --kernel-regex kns=orchb). Logs -> gpurun_out/sanitize_<tool>.log; summary lines
# ("ERROR SUMMARY: N errors") are what profiles/r02_sanitizer.md records.
# The 20 GB bench-scale tests and the ~4 s timeout tests are left out (the tool
# slows every kernel 10-100x; the timeouts rely on clock64 spin limits).
set -u
TESTS="tests/test_gpu_balance.py tests/test_gpu_dispatch.py tests/test_gpu_windows.py tests/test_gpu_hosting.py tests/test_gpu_compose.py"
SEL="not timeout and not c5_offsets and not c2_phases_share"
for tool in ${@:-memcheck racecheck synccheck initcheck}; do
  log=gpurun_out/sanitize_${tool}.log
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 3000 compute-sanitizer --tool $tool $extra --kernel-regex kns=orchb --error-exitcode 99 \
    --print-limit 200 python -m pytest $TESTS -q -x -p no:cacheprovider -k "$SEL" > $log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1) $(tail -1 $log)"
done
