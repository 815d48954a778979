set -x
timeout 900 python -m pytest -q -x tests/test_gpu_balance.py tests/test_reference_suite.py tests/test_gpu_dispatch.py -s 2>&1 | grep -E "passed|failed|Error|stats_us|C5|\(\(" | tail -30
bash scripts/cpp_api_compare.sh
cat gpurun_out/cpp_api_b200.jsonl
ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so timeout 300 python scripts/small_prof.py C5 C2
