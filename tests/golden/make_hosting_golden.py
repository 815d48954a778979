"""tests/golden/ref_hosting.npz from the unmodified reference's solve_hosting
(oracle/_ref): random volume matrices plus C2-shaped ones (DP=8 balanced by the
reference greedy, c = 8/P for P = 2, 4, 8)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Oracle, RefLib  # noqa: E402


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
    D = 16
    Vs = np.zeros((len(cases), D * D), np.int64)
    out_h = np.zeros((len(cases), D), np.int32)
    ds, cs, mx = [], [], []
    for k, (d, c, V) in enumerate(cases):
        r = ref.solve_hosting(d, c, V)
        Vs[k, :d * d] = np.asarray(V).reshape(-1)
        out_h[k, :d] = r["hosting"]
        ds.append(d)
        cs.append(c)
        mx.append(r["max_egress"])
    np.savez_compressed(os.path.join(HERE, "ref_hosting.npz"), d=np.array(ds, np.int32),
                        c=np.array(cs, np.int32), V=Vs, hosting=out_h,
                        max_egress=np.array(mx, np.int64))
    print("cases", len(cases))


if __name__ == "__main__":
    main()
