#!/bin/bash
# Round-2 verification on one GPU: the -m gpu suite, smoke(), the default bench
# line, and the bounds-checked suite (lib/checked, build with ORCH_BOUNDS_CHECK).
o=gpurun_out/verify; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/pytest_gpu.log 2>&1
echo "gpu suite rc=$? $(tail -1 $o/pytest_gpu.log)"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/smoke.log)"
timeout 900 python bench.py > $o/bench_1gpu.json 2> $o/bench_1gpu.err; echo "bench rc=$?"; cat $o/bench_1gpu.json | cut -c1-400
bash scripts/checked_suite.sh
