"""Stage clocks of the single-CTA balance kernel (k_balance_small) on the
BASELINE small phases. Needs the diagnostics build:

    ORCH_NVCC_EXTRA=-DORCH_SMALL_PROFILE python -c "from paper_2503_23830_b200 import build as b; \
        b.build_cuda(force=True, lib_dir='paper_2503_23830_b200/lib/prof')"
    ORCH_LIB_PATH=paper_2503_23830_b200/lib/prof/liborchsim_b200.so python scripts/small_prof.py

Prints, per phase, the cycles between the kernel's stage marks (S1 load and
validate, S2 identity grouping, S3 sort, S4 policy, S5 costs, S6 outputs) and
the event-timed launch duration.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_configs as bc  # noqa: E402
from paper_2503_23830_b200 import capi  # noqa: E402

MARKS = {0: "start", 1: "S1 load+validate", 2: "S2 identity grouping", 3: "S3 sort",
         4: "S4 policy", 5: "S5 assemble", 6: "S6 costs+decide", 7: "S7 outputs"}


def main():
    ctx = capi.Context(0)
    lib = capi.lib()
    buf = (C.c_longlong * 16)()
    for cname in sys.argv[1:] or ("C1", "C2", "C5"):
        cfg = bc.CONFIGS[cname]
        for name, L, O, kind, lam, v in cfg["phases"]():
            Lt = torch.from_numpy(np.ascontiguousarray(L, np.int64)).cuda()
            Ot = torch.from_numpy(np.ascontiguousarray(O, np.int32)).cuda()
            out, lay = ctx.balance_layout1(kind, cfg["d"], Lt, Ot, lam=lam, v=v)
            times = []
            for _ in range(20):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.balance_layout1(kind, cfg["d"], Lt, Ot, lam=lam, v=v, out=out, layout=lay)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3)
            lib.orch_debug_small_profile(buf)
            st = list(buf)
            marks = [k for k in sorted(MARKS) if st[k]]
            seg = ", ".join(f"{MARKS[b]} {st[b] - st[a]}" for a, b in zip(marks, marks[1:]))
            print(f"{cname} {name:7s} n={len(L):5d} d={cfg['d']:3d} kind={kind} "
                  f"us={sorted(times)[len(times) // 2]:.1f} cycles: {seg}, total {st[marks[-1]] - st[0]}",
                  flush=True)


if __name__ == "__main__":
    main()
