"""Generates tests/golden/ref_fixtures.npz from the UNMODIFIED reference
library (oracle/_ref/liborchsim_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src). Run here (the reference tree is not on GPU boxes):

    python tests/golden/make_golden.py

Each case: policy kind, d, lambda, v, lengths, origins -> the reference's
assignment vectors (dest instance, dest slot), objective (IEEE bits), whether
the identity was returned, and for BinaryPadded the minimal feasible bound.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import RefLib  # noqa: E402


def cases():
    rng = np.random.default_rng(20250330)
    out = []
    # the reference's own test generators (tests/helpers.hpp) + adversarial shapes
    for trial in range(400):
        kind = trial % 4
        d = int(rng.integers(1, 9))
        n = int(rng.integers(1, 60))
        hi = int(rng.choice([2, 5, 50, 4096, 100000]))
        mode = trial % 3
        L = rng.integers(1, hi + 1, n)
        O = (np.zeros(n) if mode == 0 else (np.arange(n) % d if mode == 1 else rng.integers(0, d, n)))
        lam = float(rng.choice([0.0, 0.01, 0.05, 1.0 / (6 * 8192)]))
        v = int(rng.choice([0, 1, 3, 64, 2048]))
        out.append((kind, d, lam, v, L, O))
    for trial in range(40):  # larger d (block greedy) and config-like shapes
        kind = trial % 4
        d = int(rng.choice([33, 64, 128, 300]))
        n = int(rng.integers(d, 4 * d + 50))
        L = np.ceil(np.exp(rng.normal(6.5, 0.8, n))).clip(64, 4096)
        O = np.arange(n) % d
        out.append((kind, d, 2.03e-5, 2048, L, O))
    return out


def main():
    ref = RefLib()
    kinds, ds, lams, vs, offs, lens, orgs = [], [], [], [], [0], [], []
    dest, slot, obj, ident, bound = [], [], [], [], []
    for kind, d, lam, v, L, O in cases():
        L = np.asarray(L, np.int64)
        O = np.asarray(O, np.int32)
        di, dsl, ob, idn = ref.balance(kind, d, L, O, lam=lam, v=v)
        kinds.append(kind), ds.append(d), lams.append(lam), vs.append(v)
        lens.append(L), orgs.append(O), dest.append(di), slot.append(dsl)
        obj.append(ob), ident.append(idn)
        bound.append(ref.min_feasible_padded_bound(d, L, O) if kind == 1 else 0)
        offs.append(offs[-1] + len(L))
    np.savez_compressed(os.path.join(HERE, "ref_fixtures.npz"), kind=np.array(kinds, np.int32),
                        d=np.array(ds, np.int32), lam=np.array(lams, np.float64),
                        v=np.array(vs, np.int64), offset=np.array(offs, np.int64),
                        length=np.concatenate(lens), origin=np.concatenate(orgs),
                        dest_inst=np.concatenate(dest), dest_slot=np.concatenate(slot),
                        objective=np.array(obj, np.float64), is_identity=np.array(ident, np.int32),
                        bound=np.array(bound, np.int64))
    print("cases", len(kinds), "items", offs[-1])


if __name__ == "__main__":
    main()
