#!/bin/bash
# The -m gpu suite against the bounds-checked build (ORCH_BOUNDS_CHECK: device
# asserts on every copy's source / destination range and on the balance and
# layout kernels' indices; a violation prints and traps). compute-sanitizer is
# closed on the GPU pool, so this is the memory-safety evidence
# (profiles/r02_bounds_check.md). The C++-API and reference-suite tests link the
# product library and are left to the normal run.
o=gpurun_out/r02; mkdir -p $o
ORCH_LIB_PATH=paper_2503_23830_b200/lib/checked/liborchsim_b200.so timeout 1800 \
  python -m pytest tests -m gpu -q -p no:cacheprovider --ignore=tests/test_reference_suite.py \
  > $o/pytest_checked.log 2>&1
echo "checked suite rc=$? $(tail -1 $o/pytest_checked.log)"
grep -c "ORCH_DCHECK failed" $o/pytest_checked.log || true
