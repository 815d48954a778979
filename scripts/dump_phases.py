"""Writes the BASELINE phase inputs (bench_configs.CONFIGS) as binary files for
scripts/cpp_api_bench.cpp: n, d, kind, v (int64), lambda (f64), len[n] i64, origin[n] i32."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, bench_configs as bc
os.makedirs(f"{ROOT}/gpurun_out/phases", exist_ok=True)
for cname in ("C1", "C2", "C3", "C4x30", "C4x64", "C5"):
    cfg = bc.CONFIGS[cname]
    for i, (pname, L, O, kind, lam, v) in enumerate(cfg["phases"]()):
        with open(f"{ROOT}/gpurun_out/phases/in_{cname}_{i}.bin", "wb") as f:
            np.array([len(L), cfg["d"], kind, v], np.int64).tofile(f)
            np.array([lam], np.float64).tofile(f)
            L.astype(np.int64).tofile(f); O.astype(np.int32).tofile(f)
        print(cname, i, pname, len(L), kind)
