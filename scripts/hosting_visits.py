"""Times orch_solve_hosting_host (hosting + the reference's nodes_visited replay)
on the C3 fixtures and prints the visit counts next to the reference's:

    python scripts/hosting_visits.py [case ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2503_23830_b200.capi import Context  # noqa: E402


def main():
    ctx = Context(0)
    f = np.load(os.path.join(ROOT, "tests", "golden", "ref_hosting_c3.npz"))
    cases = [int(a) for a in sys.argv[1:]] or range(len(f["c"]))
    for k in cases:
        c = int(f["c"][k])
        ctx.solve_hosting(64, c, f["V"][k])
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            a = ctx.solve_hosting(64, c, f["V"][k])
            ts.append(time.perf_counter() - t0)
        tb = []
        for _ in range(5):
            t0 = time.perf_counter()
            ctx.solve_hosting(64, c, f["V"][k], info=False)
            tb.append(time.perf_counter() - t0)
        print(f"C3 case {k} c={c}: visited {a['visited']} (reference {int(f['visited'][k])}), "
              f"{1e3 * min(ts):.2f} ms ({1e3 * min(tb):.2f} ms without the count)", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
