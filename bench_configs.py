#!/usr/bin/env python3
"""Per-config evidence for BASELINE.json configs C1..C5 on one B200 (not the
driver's bench line; see bench.py for that). For every config and phase:
GPU balance time (device-resident inputs, CUDA events, median of reps),
host-buffer C-ABI time (orch_balance_host through ctypes, synchronous, median), the reference's own
balance() time on the host (oracle/_ref), bit-exact parity of the assignment
and objective against the reference, and for the dispatched configs the
token-row movement time and HBM GB/s.

    python bench_configs.py [--sweep] [--only C3,C4x30] [--out profiles/r01_configs.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def c1_items():
    """C1: DP=8 text-only, 64 seqs/instance, U[128,4096] from
    std::mt19937_64(0xC1) as lo + rng() % (hi - lo + 1) (tests/helpers.hpp:34-39)."""
    from paper_2503_23830_b200.workload import MT19937_64
    g = MT19937_64(0xC1)
    n = 512
    L = np.array([128 + g() % (4096 - 128 + 1) for _ in range(n)], np.int64)
    return [("text", L, (np.arange(n) % 8).astype(np.int32), 0, 0.0, 0)]


def mci_phases(d, per, seed, mix=3):
    from paper_2503_23830_b200 import workload
    b = workload.make_batch(mix, d, per, seed)
    out = []
    lv, ov, _ = b.phase_items("vision")
    out.append(("vision", lv, ov, 0, 0.0, 0))
    if mix == 3:
        la, oa, _ = b.phase_items("audio")
        out.append(("audio", la, oa, 1, 0.0, 0))
    ll, ol = b.llm_items()
    out.append(("llm", ll, ol, 0, 0.0, 0))
    return out


def c5_phases(P=8):
    rng = np.random.default_rng(5)
    n = 8 * P
    L = rng.integers(8192, 32769, n).astype(np.int64)
    O = (np.arange(n) % P).astype(np.int32)
    lam = 1.0 / (6 * 8192)
    return [("long-ctx greedy", L, O, 0, lam, 0),
            ("long-ctx quadtol", L, O, 2, lam, 2048),
            ("long-ctx fixed32k quadtol", np.full(n, 32768, np.int64), O, 2, lam, 2048)]


CONFIGS = {
    "C1": dict(d=8, R=None, phases=c1_items),
    "C2": dict(d=8, R=8192, phases=lambda: mci_phases(8, 64, 2, mix=2)),
    "C3": dict(d=64, R=16384, phases=lambda: mci_phases(64, 64, 7)),
    "C4x30": dict(d=2560, R=None, phases=lambda: mci_phases(2560, 30, 7)),
    "C4x64": dict(d=2560, R=None, phases=lambda: mci_phases(2560, 64, 7)),
    "C5": dict(d=8, R=16384, phases=c5_phases),
}
# C4's balancer scaling sweep: d in {8, 64, 256, 1024}
# at 30 examples per instance, three modalities (d = 2560 is C4x30 above)
SWEEP = {f"C4sweep_d{d}": dict(d=d, R=None, phases=(lambda d=d: mci_phases(d, 30, 7)))
         for d in (8, 64, 256, 1024)}


def main():
    import torch

    from oracle import RefLib
    from paper_2503_23830_b200.capi import Context
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_configs.jsonl"))
    ap.add_argument("--only", default="")
    ap.add_argument("--sweep", action="store_true",
                    help="also C4's balancer sweep over d in {8, 64, 256, 1024}")
    args = ap.parse_args()
    configs = dict(CONFIGS, **SWEEP) if args.sweep else CONFIGS
    ref = RefLib() if RefLib.available() else None
    ctx = Context(0)
    lines = []
    for cname, cfg in configs.items():
        if args.only and cname not in args.only.split(","):
            continue
        d = cfg["d"]
        for pname, L, O, kind, lam, v in cfg["phases"]():
            n = len(L)
            Lt, Ot = torch.from_numpy(L).cuda(), torch.from_numpy(O).cuda()
            bal = ctx.balance(kind, d, Lt, Ot, lam=lam, v=v)
            torch.cuda.synchronize()
            reps = 20 if n <= 20000 else 5
            times = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.balance(kind, d, Lt, Ot, lam=lam, v=v, out=bal)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3)
            gpu_us = statistics.median(times)
            hr = ctx.balance_host(kind, d, L, O, lam=lam, v=v)  # warm (staging sized)
            hts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                hr = ctx.balance_host(kind, d, L, O, lam=lam, v=v)
                hts.append((time.perf_counter() - t0) * 1e6)
            host_us = statistics.median(hts)
            s = bal.summary()
            rec = dict(config=cname, phase=pname, policy=kind, d=d, n=n, tokens=int(L.sum()),
                       gpu_balance_us=round(gpu_us, 1), host_abi_balance_us=round(host_us, 1),
                       objective=s.objective, used_identity=s.used_identity,
                       pre_max_over_mean=round(s.pre_ratio, 6),
                       post_max_over_mean=round(s.post_ratio, 6), rounds=s.rounds)
            if ref is not None:
                di, ds, obj, _ = ref.balance(kind, d, L, O, lam=lam, v=v)
                rec["parity_vs_reference"] = bool(
                    np.array_equal(bal.dest_inst[:n].cpu().numpy(), di)
                    and np.array_equal(bal.dest_slot[:n].cpu().numpy(), ds)
                    and np.float64(s.objective).tobytes() == np.float64(obj).tobytes()
                    and np.array_equal(hr["dest_inst"], di))
                rt = ref.time_balance(kind, d, L, O, 3 if n > 20000 else 10, lam=lam, v=v)
                rec["reference_balance_us"] = round(float(np.median(rt)) * 1e6, 1)
                rec["speedup_vs_reference"] = round(rec["reference_balance_us"] / gpu_us, 1)
            if cfg["R"]:
                R = cfg["R"]
                lay = ctx.layout(d, 1, Lt, Ot, bal)
                rows = int(L.sum())
                rin = torch.randint(0, 255, (rows * R,), dtype=torch.uint8, device="cuda")
                rout = torch.empty_like(rin)
                for _ in range(3):
                    ctx.dispatch(d, Lt, Ot, bal, lay, R, rin, rout)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    ctx.dispatch(d, Lt, Ot, bal, lay, R, rin, rout)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                rec.update(row_bytes=R, rows=rows, dispatch_ms=round(ms, 4),
                           dispatch_hbm_gbs=round(2 * rows * R / ms / 1e6, 1))
                del rin, rout
                torch.cuda.empty_cache()
            print(json.dumps(rec), flush=True)
            lines.append(rec)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for r in lines:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
