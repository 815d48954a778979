#!/bin/bash
# One-GPU round-2 evidence pass: -m gpu suite, stage clocks of the small
# balance kernel and of the one-CTA LPT, the driver's bench line, and (with
# "checked") the suite against the bounds-checked build.
o=gpurun_out/r02; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $o/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $o/pytest_gpu.log)"
ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so timeout 300 python scripts/small_prof.py C1 C2 C3 C5 > $o/small_prof.log 2>&1; echo "small_prof rc=$?"
ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so timeout 300 python scripts/lpt_prof.py > $o/lpt_prof.log 2>&1; echo "lpt_prof rc=$?"
timeout 300 python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
[ "${1:-}" = "checked" ] && bash scripts/checked_suite.sh
exit 0
