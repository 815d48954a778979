"""CPU tests: the oracle (oracle/orchsim_oracle.c) pinned against the
reference's known answers and against fixtures produced by the unmodified
reference library (tests/golden/ref_fixtures.npz, tests/golden/make_golden.py),
plus a live differential against oracle/_ref when it is built here."""
import json
import os

import numpy as np
import pytest

from conftest import random_instance

HERE = os.path.dirname(os.path.abspath(__file__))
KNOWN = json.load(open(os.path.join(HERE, "golden", "reference_known_answers.json")))


def _origin(case):
    return np.zeros(len(case["lengths"]), np.int32)


def test_known_balance_answers(oracle):
    for c in KNOWN["balance"]:
        r = oracle.balance(c["kind"], c["d"], c["lengths"], _origin(c), lam=c.get("lam", 0.0),
                           v=c.get("v", 0))
        assert r.objective == pytest.approx(c["objective"], rel=1e-12), c["cite"]
        if "sorted_batches" in c:
            L = np.asarray(c["lengths"])
            got = sorted(sorted(L[r.dest_inst == b].tolist()) for b in range(c["d"]))
            assert got == c["sorted_batches"], c["cite"]
        if "nonempty" in c:
            assert int((r.bin_count > 0).sum()) == c["nonempty"]
        if "bound" in c:
            assert oracle.min_feasible_padded_bound(c["d"], c["lengths"], _origin(c)) == c["bound"]


def test_known_errors(oracle):
    from oracle import OracleError
    for c in KNOWN["errors"]:
        with pytest.raises(OracleError) as e:
            oracle.balance(c["kind"], c["d"], c["lengths"], _origin(c), lam=c.get("lam", 0.0))
        assert e.value.code == c["code"], c["cite"]


def test_known_costs(oracle):
    for c in KNOWN["cost"]:
        v = oracle.cost(c["alpha"], c["beta"], c["padded"], c["variant"], c["padded"], c["lengths"])
        assert v == pytest.approx(c["value"], rel=1e-12), c["cite"]
    from oracle import OracleError
    with pytest.raises(OracleError):  # test_core.cpp:61-65 padding-mode mismatch
        oracle.cost(1.0, 0.1, 1, 1, 0, [3])
    assert oracle.cost(1.0, 0.1, 1, 1, 1, []) == 0.0


def test_reference_fixtures(oracle):
    f = np.load(os.path.join(HERE, "golden", "ref_fixtures.npz"))
    off = f["offset"]
    for c in range(len(f["kind"])):
        a, b = off[c], off[c + 1]
        L, O = f["length"][a:b], f["origin"][a:b]
        r = oracle.balance(int(f["kind"][c]), int(f["d"][c]), L, O, lam=float(f["lam"][c]),
                           v=int(f["v"][c]))
        np.testing.assert_array_equal(r.dest_inst, f["dest_inst"][a:b])
        np.testing.assert_array_equal(r.dest_slot, f["dest_slot"][a:b])
        assert np.float64(r.objective).tobytes() == np.float64(f["objective"][c]).tobytes()
        if f["kind"][c] == 1:
            assert oracle.min_feasible_padded_bound(int(f["d"][c]), L, O) == f["bound"][c]


def test_live_differential_vs_reference(oracle, reflib):
    rng = np.random.default_rng(7)
    for trial in range(600):
        kind = trial % 4
        d = int(rng.integers(1, 12))
        n = int(rng.integers(1, 80))
        L, O = random_instance(rng, d, n, 1, int(rng.choice([3, 40, 3000])))
        lam, v = float(rng.choice([0.0, 0.02, 2e-5])), int(rng.choice([0, 2, 500]))
        di, ds, obj, _ = reflib.balance(kind, d, L, O, lam=lam, v=v)
        r = oracle.balance(kind, d, L, O, lam=lam, v=v)
        np.testing.assert_array_equal(r.dest_inst, di)
        np.testing.assert_array_equal(r.dest_slot, ds)
        assert np.float64(r.objective).tobytes() == np.float64(obj).tobytes()


def test_oracle_large_shapes_vs_reference(oracle, reflib):
    """C4-like shape (d=2560 x 30) and DP=64 x 64 differential (a few seconds)."""
    rng = np.random.default_rng(11)
    for d, per in [(64, 64), (2560, 30)]:
        n = d * per
        L = rng.integers(128, 4097, n)
        O = np.arange(n) % d
        for kind in (0, 1):
            di, ds, obj, _ = reflib.balance(kind, d, L, O)
            r = oracle.balance(kind, d, L, O)
            np.testing.assert_array_equal(r.dest_inst, di)
            np.testing.assert_array_equal(r.dest_slot, ds)
            assert r.objective == obj


def test_costs_vs_reference(oracle, reflib):
    rng = np.random.default_rng(3)
    for _ in range(300):
        variant = int(rng.integers(0, 3))
        padded = int(rng.integers(0, 2))
        L = rng.integers(1, int(rng.choice([30, 70000, 2 ** 28])), int(rng.integers(0, 9)))
        alpha, beta = float(rng.choice([0.5, 1.0, 2.0])), float(rng.choice([0.0, 0.02, 1e-5]))
        a = oracle.cost(alpha, beta, padded, variant, padded, L)
        b = reflib.cost(alpha, beta, padded, variant, padded, L)
        assert np.float64(a).tobytes() == np.float64(b).tobytes()


def test_layout_and_rows_semantics(oracle):
    """apply() on rows == per-instance batches in destination slot order."""
    rng = np.random.default_rng(5)
    R = 32
    for P in (1, 2, 4):
        d = 4 * P
        L, O = random_instance(rng, d, 60, 1, 9)
        r = oracle.balance(0, d, L, O)
        e = oracle.layout(d, P, L, O, r.dest_inst, r.dest_slot)
        c = d // P
        ins = [np.zeros(int(e["in_tokens"][q]) * R, np.uint8) for q in range(P)]
        for q in range(P):
            sel = np.nonzero(O // c == q)[0]
            oracle.fill_rows(L[sel], sel.astype(np.int64), e["rank_src_off"][sel], R, ins[q])
        outs = [np.zeros(int(e["out_tokens"][q]) * R, np.uint8) for q in range(P)]
        oracle.dispatch_rows(d, P, L, O, r.dest_inst, e["rank_src_off"], e["rank_dst_off"], R,
                             ins, outs, nthreads=3)
        # check: walk destination batches in slot order, rows tagged by input position
        for q in range(P):
            words = outs[q].view(np.int64).reshape(-1, 2)
            row = 0
            for j in range(q * c, (q + 1) * c):
                members = np.nonzero(r.dest_inst == j)[0]
                members = members[np.argsort(r.dest_slot[members])]
                for pos in members:
                    k = int(L[pos]) * R // 16
                    assert (words[row:row + k, 0] == pos).all()
                    assert (words[row:row + k, 1] == np.arange(k)).all()
                    row += k


def test_solve_hosting_vs_reference(oracle, reflib):
    """solve_hosting (topology.cpp:179-265): the C restatement reproduces the
    reference's hosting, max egress and even its branch-and-bound node count."""
    rng = np.random.default_rng(17)
    for _ in range(600):
        c = int(rng.integers(1, 5))
        nodes = int(rng.integers(1, 6))
        d = c * nodes
        if d > 12:
            continue
        V = rng.integers(0, int(rng.choice([3, 100, 10000])), (d, d)) * (rng.random((d, d)) < 0.7)
        a = oracle.solve_hosting(d, c, V)
        b = reflib.solve_hosting(d, c, V)
        np.testing.assert_array_equal(a["hosting"], b["hosting"])
        assert a["max_egress"] == b["max_egress"] and a["visited"] == b["visited"]


def test_hosting_fixtures(oracle):
    f = np.load(os.path.join(HERE, "golden", "ref_hosting.npz"))
    for k in range(len(f["d"])):
        d, c = int(f["d"][k]), int(f["c"][k])
        V = f["V"][k, :d * d].reshape(d, d)
        a = oracle.solve_hosting(d, c, V)
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k, :d])
        assert a["max_egress"] == f["max_egress"][k]
        assert a["visited"] == f["visited"][k]


def test_hosting_wide_fixtures(oracle):
    """d = 72..256 volume matrices (make_hosting_wide_golden.py)."""
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_wide.npz"))
    for k in range(len(f["d"])):
        d, c = int(f["d"][k]), int(f["c"][k])
        a = oracle.solve_hosting(d, c, f["V"][k][:d, :d])
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k][:d])
        assert a["max_egress"] == f["max_egress"][k]
        assert a["visited"] == f["visited"][k]


def test_hosting_c3_fixtures(oracle):
    """DP=64 (C3) phase volume matrices on 2/4/8 GPUs (make_hosting_c3_golden.py)."""
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_c3.npz"))
    for k in range(len(f["c"])):
        a = oracle.solve_hosting(64, int(f["c"][k]), f["V"][k].reshape(64, 64))
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k])
        assert a["max_egress"] == f["max_egress"][k]
        assert a["visited"] == f["visited"][k]
