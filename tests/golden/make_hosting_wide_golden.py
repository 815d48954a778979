"""tests/golden/ref_hosting_wide.npz from the unmodified reference's solve_hosting
(oracle/_ref) beyond d = 64: random volume matrices at d = 72..256 (kept when the
reference's sequential search finishes in 5 s), and the C4 (d = 2560) vision
phase's volume matrix -- rebuilt by the test from bench_configs through the
oracle, so only its answers are stored -- on 2, 16 and 32 nodes."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from oracle import Oracle, RefLib  # noqa: E402
from make_hosting_golden import _finishes  # noqa: E402


def c4_vision_volume(orc):
    import bench_configs as bc
    cfg = bc.CONFIGS["C4x30"]
    name, L, O, kind, lam, v = next(iter(cfg["phases"]()))
    r = orc.balance(kind, cfg["d"], L, O, lam=lam, v=v)
    return orc.volume_matrix(cfg["d"], L, O, r.dest_inst)


def main():
    ref, orc = RefLib(), Oracle()
    rng = np.random.default_rng(4096)
    Vs, ds, cs, hs, mx, vis = [], [], [], [], [], []
    D = 256
    while len(ds) < 12:
        d = int(rng.choice([72, 96, 128, 256]))
        nodes = int(rng.choice([2, 3, 4, 8, 16, 32]))
        if d % nodes:
            continue
        c = d // nodes
        V = rng.integers(0, int(rng.choice([50, 1000])), (d, d)) * (rng.random((d, d)) < 0.3)
        if not _finishes(d, c, V, 5.0):
            continue
        r = ref.solve_hosting(d, c, V)
        Vp = np.zeros((D, D), np.int64)
        Vp[:d, :d] = V
        Vs.append(Vp)
        ds.append(d)
        cs.append(c)
        h = np.zeros(D, np.int32)
        h[:d] = r["hosting"]
        hs.append(h)
        mx.append(r["max_egress"])
        vis.append(r["visited"])
    V4 = c4_vision_volume(orc)
    c4c, c4h, c4m, c4v = [], [], [], []
    for c in (1280, 160, 80):
        r = ref.solve_hosting(2560, c, V4)
        c4c.append(c)
        c4h.append(r["hosting"])
        c4m.append(r["max_egress"])
        c4v.append(r["visited"])
    np.savez_compressed(os.path.join(HERE, "ref_hosting_wide.npz"), V=np.array(Vs), d=np.array(ds),
                        c=np.array(cs), hosting=np.array(hs), max_egress=np.array(mx),
                        visited=np.array(vis), c4_c=np.array(c4c), c4_hosting=np.array(c4h),
                        c4_max_egress=np.array(c4m), c4_visited=np.array(c4v))
    print("cases", len(ds), "+ C4", c4c, "visited", vis, c4v)


if __name__ == "__main__":
    main()
