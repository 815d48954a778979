"""tests/golden/ref_hosting.npz from the unmodified reference's solve_hosting
(oracle/_ref): random volume matrices plus C2-shaped ones (DP=8 balanced by the
reference greedy, c = 8/P for P = 2, 4, 8), then larger ones (d <= 32, 2..16
nodes); with the reference's nodes_visited."""
import os
import signal
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Oracle, RefLib  # noqa: E402


def _finishes(d, c, V, secs):
    """True when the reference solves (d, c, V) within secs (in a forked child)."""
    pid = os.fork()
    if pid == 0:
        RefLib().solve_hosting(d, c, V)
        os._exit(0)
    t0 = time.monotonic()
    while time.monotonic() - t0 < secs:
        done, _ = os.waitpid(pid, os.WNOHANG)
        if done:
            return True
        time.sleep(0.01)
    os.kill(pid, signal.SIGKILL)
    os.waitpid(pid, 0)
    return False


def main():
    ref, orc = RefLib(), Oracle()
    rng = np.random.default_rng(2024)
    cases = []
    for _ in range(300):
        c = int(rng.integers(1, 5))
        nodes = int(rng.integers(1, 6))
        d = c * nodes
        if d > 12:
            continue
        V = rng.integers(0, int(rng.choice([3, 100, 10000])), (d, d)) * (rng.random((d, d)) < 0.7)
        cases.append((d, c, V))
    from paper_2503_23830_b200 import workload
    b = workload.make_batch(2, 8, 64, 2)
    for L, O in [b.phase_items("vision")[:2], b.llm_items()]:
        r = orc.balance(0, 8, L, O)
        V = orc.volume_matrix(8, L, O, r.dest_inst)
        for c in (4, 2, 1):
            cases.append((8, c, V))
    # larger ones, kept when the reference's sequential search finishes in 2 s
    rng = np.random.default_rng(2025)
    big = 0
    while big < 40:
        nodes = int(rng.choice([2, 3, 4, 8, 16]))
        c = int(rng.integers(1, max(2, 32 // nodes) + 1))
        d = nodes * c
        if d > 32 or d <= 12:
            continue
        V = rng.integers(0, int(rng.choice([3, 50, 1000])), (d, d)) * (rng.random((d, d)) < 0.5)
        if _finishes(d, c, V, 2.0):
            cases.append((d, c, V))
            big += 1
    D = 32
    Vs = np.zeros((len(cases), D * D), np.int64)
    out_h = np.zeros((len(cases), D), np.int32)
    ds, cs, mx, vis = [], [], [], []
    for k, (d, c, V) in enumerate(cases):
        r = ref.solve_hosting(d, c, V)
        Vs[k, :d * d] = np.asarray(V).reshape(-1)
        out_h[k, :d] = r["hosting"]
        ds.append(d)
        cs.append(c)
        mx.append(r["max_egress"])
        vis.append(r["visited"])
    np.savez_compressed(os.path.join(HERE, "ref_hosting.npz"), d=np.array(ds, np.int32),
                        c=np.array(cs, np.int32), V=Vs, hosting=out_h,
                        max_egress=np.array(mx, np.int64), visited=np.array(vis, np.int64))
    print("cases", len(cases))


if __name__ == "__main__":
    main()
