#!/bin/bash
# Copy the 1-GPU refresh (scripts/refresh_1gpu.sh + cpp_api_compare.sh output in
# gpurun_out/) into profiles/ and regenerate the summaries.
set -e
R=gpurun_out/refresh
grep '^{' $R/bench_1gpu.json > profiles/r01_bench_1gpu.json
grep '^{' $R/bench_ref.json > profiles/r01_bench_ref.json
grep -h '^{' $R/bench_c3.json $R/bench_c5.json > profiles/r01_bench_c3_c5_1gpu.jsonl
cp $R/configs.jsonl profiles/r01_configs.jsonl
cp $R/launches.csv profiles/r01_launches.csv
python profiles/summarize.py launches profiles/r01_launches.csv profiles/r01_launches.md
python profiles/summarize.py full $R/k_move_tma_full.ncu-rep profiles/r01_k_move_tma_full.md
python profiles/summarize.py full $R/k_balance_small_full.ncu-rep profiles/r01_k_balance_small_full.md
python - <<'PY'
import json
b = [json.loads(l) for l in open("gpurun_out/cpp_api_b200.jsonl")]
r = [json.loads(l) for l in open("gpurun_out/cpp_api_ref.jsonl")]
with open("profiles/r01_cpp_api.jsonl", "w") as f:
    for x, y in zip(b, r):
        f.write(json.dumps({"phase_file": x["file"].split("/")[-1], "n": x["n"], "d": x["d"],
                            "policy": x["kind"], "b200_cpp_api_median_us": x["median_us"],
                            "reference_cpp_api_median_us": y["median_us"],
                            "speedup": round(y["median_us"] / x["median_us"], 2),
                            "identical_result": x["checksum"] == y["checksum"]
                            and x["objective"] == y["objective"],
                            "objective": x["objective"]}) + "\n")
PY
