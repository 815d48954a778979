"""Stage clocks of the one-CTA exact LPT (k_greedy_lpt) on the C4 phases,
summed over its rounds (diagnostics build, see scripts/small_prof.py):
key build, rank sort, k search, assignment; plus the event-timed balance."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_configs as bc  # noqa: E402
from paper_2503_23830_b200 import capi  # noqa: E402


def main():
    ctx = capi.Context(0)
    lib = capi.lib()
    buf = (C.c_longlong * 16)()
    for cname in sys.argv[1:] or ("C4x30", "C4x64"):
        cfg = bc.CONFIGS[cname]
        for name, L, O, kind, lam, v in cfg["phases"]():
            if kind != 0:
                continue
            Lt = torch.from_numpy(np.ascontiguousarray(L, np.int64)).cuda()
            Ot = torch.from_numpy(np.ascontiguousarray(O, np.int32)).cuda()
            out = ctx.balance(kind, cfg["d"], Lt, Ot)
            torch.cuda.synchronize()
            times = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.balance(kind, cfg["d"], Lt, Ot, out=out)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3)
            lib.orch_debug_small_profile(buf)
            st = list(buf)
            r = max(st[12], 1)
            print(f"{cname} {name} n={len(L)} d={cfg['d']} balance_us={sorted(times)[2]:.1f} "
                  f"rounds={st[12]} cycles/round: start {st[13] / r:.0f} keys {st[8] / r:.0f} "
                  f"sort {st[9] / r:.0f} k {st[10] / r:.0f} assign {st[11] / r:.0f}", flush=True)


if __name__ == "__main__":
    main()
