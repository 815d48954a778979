"""Per-kernel device times of one balance call (the third, warm) under ncu:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file out.csv python scripts/kprof.py C4x30 [phase-index]
Only the third call sits between cudaProfilerStart/Stop."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

import bench_configs as bc  # noqa: E402
from paper_2503_23830_b200.capi import Context  # noqa: E402

cfg = bc.CONFIGS[sys.argv[1]]
only = int(sys.argv[2]) if len(sys.argv) > 2 else None
ctx = Context(0)
for i, (name, L, O, kind, lam, v) in enumerate(cfg["phases"]()):
    if only is not None and i != only:
        continue
    Lt, Ot = torch.from_numpy(L).cuda(), torch.from_numpy(O).cuda()
    bal = ctx.balance(kind, cfg["d"], Lt, Ot, lam=lam, v=v)
    ctx.balance(kind, cfg["d"], Lt, Ot, lam=lam, v=v, out=bal)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ctx.balance(kind, cfg["d"], Lt, Ot, lam=lam, v=v, out=bal)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(sys.argv[1], name, "n", len(L), flush=True)
