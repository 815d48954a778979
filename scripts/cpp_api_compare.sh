#!/bin/bash
# The reference's C++ API, balance(policy, d, items), timed call for call: the
# B200 drop-in (liborchsim_b200_host.so) against the unmodified reference code,
# on every BASELINE phase. Output: gpurun_out/cpp_api_{b200,ref}.jsonl
python scripts/dump_phases.py > /dev/null
f=$(ls gpurun_out/phases/in_*.bin | sort)
paper_2503_23830_b200/lib/cpp_api_bench_b200 $f > gpurun_out/cpp_api_b200.jsonl
oracle/_ref/cpp_api_bench_ref $f > gpurun_out/cpp_api_ref.jsonl
