"""tests/golden/ref_hosting_c3.npz from the unmodified reference's solve_hosting
(oracle/_ref): volume matrices of the reference balancer's vision / audio / LLM
phases of the C3 batch (DP=64, 64 examples per instance, generator seed 7),
hosted with c = 32, 16, 8 instances per GPU (2, 4, 8 GPUs)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import RefLib  # noqa: E402


def main():
    from paper_2503_23830_b200 import workload
    ref = RefLib()
    b = workload.make_batch(3, 64, 64, 7)
    Vs, cs, hs, mx, vis = [], [], [], [], []
    for name, kind in (("vision", 0), ("audio", 1), ("llm", 0)):
        L, O = b.llm_items() if name == "llm" else b.phase_items(name)[:2]
        di, _, _, _ = ref.balance(kind, 64, L, O)
        V = np.zeros((64, 64), np.int64)
        np.add.at(V, (O, di), L)  # volume_matrix (topology.cpp:40-53)
        for c in (32, 16, 8):
            r = ref.solve_hosting(64, c, V)
            Vs.append(V.reshape(-1))
            cs.append(c)
            hs.append(r["hosting"])
            mx.append(r["max_egress"])
            vis.append(r["visited"])
    np.savez_compressed(os.path.join(HERE, "ref_hosting_c3.npz"), V=np.array(Vs, np.int64),
                        c=np.array(cs, np.int32), hosting=np.array(hs, np.int32),
                        max_egress=np.array(mx, np.int64), visited=np.array(vis, np.int64))
    print("cases", len(cs))


if __name__ == "__main__":
    main()
