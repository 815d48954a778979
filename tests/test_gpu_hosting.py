"""GPU node-wise hosting (orch_solve_hosting_host / orch_nodewise) against the
oracle restatement of the reference's branch and bound (exact hosting, the
reference's tie-breaking) and the reference's own fixtures."""
import os

import numpy as np
import pytest
import torch

from conftest import random_instance

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_solve_hosting_random(ctx, oracle):
    rng = np.random.default_rng(5)
    for _ in range(300):
        c = int(rng.integers(1, 5))
        nodes = int(rng.integers(1, 6))
        d = c * nodes
        if d > 12:
            continue
        V = rng.integers(0, int(rng.choice([2, 3, 100, 10000])), (d, d)) * (rng.random((d, d)) < 0.7)
        a = ctx.solve_hosting(d, c, V)
        o = oracle.solve_hosting(d, c, V)
        np.testing.assert_array_equal(a["hosting"], o["hosting"])
        assert a["max_egress"] == o["max_egress"]
        assert a["baseline_max"] == o["baseline_max"]
        assert a["visited"] == o["visited"], (d, c)


def test_solve_hosting_fixtures(ctx):
    f = np.load(os.path.join(HERE, "golden", "ref_hosting.npz"))
    for k in range(len(f["d"])):
        d, c = int(f["d"][k]), int(f["c"][k])
        a = ctx.solve_hosting(d, c, f["V"][k, :d * d])
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k, :d])
        assert a["max_egress"] == f["max_egress"][k]
        assert a["visited"] == f["visited"][k], (k, d, c)  # the reference's nodes_visited


@pytest.mark.parametrize("P", [2, 4, 8])
def test_nodewise_in_place(ctx, oracle, P):
    """balance -> orch_nodewise: dest instances relabelled by batch_to_instance,
    per-batch arrays and CSR permuted, then layout + dispatch still byte-exact."""
    rng = np.random.default_rng(P)
    for kind in (0, 1, 2, 3):
        d = 8
        c = d // P
        n = 300
        L, O = random_instance(rng, d, n, 1, 60)
        o = oracle.balance(kind, d, L, O, lam=0.01, v=3)
        V = oracle.volume_matrix(d, L, O, o.dest_inst)
        h = oracle.solve_hosting(d, c, V)
        b2i = h["batch_to_instance"]
        Lt, Ot = torch.from_numpy(L).cuda(), torch.from_numpy(O).cuda()
        bal = ctx.balance(kind, d, Lt, Ot, lam=0.01, v=3)
        hosting, g_b2i, info = ctx.nodewise(d, c, Lt, Ot, bal)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(hosting.cpu().numpy(), h["hosting"])
        np.testing.assert_array_equal(g_b2i.cpu().numpy(), b2i)
        assert int(info[0]) == h["max_egress"] and int(info[1]) == h["baseline_max"]
        np.testing.assert_array_equal(bal.dest_inst[:n].cpu().numpy(), b2i[o.dest_inst])
        np.testing.assert_array_equal(bal.dest_slot[:n].cpu().numpy(), o.dest_slot)
        inv = np.argsort(b2i)
        np.testing.assert_array_equal(bal.bin_count.cpu().numpy(), o.bin_count[inv])
        assert bal.bin_cost.cpu().numpy().tobytes() == o.bin_cost[inv].tobytes()
        off = bal.bin_offset.cpu().numpy()
        mem = bal.bin_member[:n].cpu().numpy()
        di = b2i[o.dest_inst]
        for j in range(d):
            seg = mem[off[j]:off[j + 1]]
            assert (di[seg] == j).all() and (o.dest_slot[seg] == np.arange(len(seg))).all()
        # the relabelled result still dispatches byte-exactly
        R = 32
        lay = ctx.layout(d, 1, Lt, Ot, bal)
        e = oracle.layout(d, 1, L, O, di, o.dest_slot)
        rows = int(L.sum())
        hin = np.zeros(rows * R, np.uint8)
        oracle.fill_rows(L, np.arange(n, dtype=np.int64), e["rank_src_off"], R, hin)
        hout = np.zeros_like(hin)
        oracle.dispatch_rows(d, 1, L, O, di, e["rank_src_off"], e["rank_dst_off"], R, [hin], [hout])
        rin = torch.from_numpy(hin).cuda()
        rout = torch.zeros_like(rin)
        ctx.dispatch(d, Lt, Ot, bal, lay, R, rin, rout)
        torch.cuda.synchronize()
        assert torch.equal(rout.cpu(), torch.from_numpy(hout))


def test_solve_hosting_c3_shapes(ctx, oracle):
    """DP=64 (C3) volume matrices of the reference balancer's three phases,
    hosted on 2, 4 and 8 GPUs: the branch and bound against the reference's
    own answers (tests/golden/ref_hosting_c3.npz)."""
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_c3.npz"))
    for k in range(len(f["c"])):
        c = int(f["c"][k])
        a = ctx.solve_hosting(64, c, f["V"][k])
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k])
        assert a["max_egress"] == f["max_egress"][k]
        o = oracle.solve_hosting(64, c, f["V"][k])
        np.testing.assert_array_equal(o["hosting"], f["hosting"][k])
        assert a["visited"] == f["visited"][k], (k, a["visited"], int(f["visited"][k]))


def test_solve_hosting_random_larger(ctx, oracle):
    """d up to 32 with 2..16 nodes: leaves beating the incumbents, ties."""
    rng = np.random.default_rng(99)
    for _ in range(60):
        nodes = int(rng.choice([2, 3, 4, 8, 16]))
        c = int(rng.integers(1, max(2, 32 // nodes) + 1))
        d = nodes * c
        if d > 32 or nodes > 32:
            continue
        V = rng.integers(0, int(rng.choice([3, 50, 1000])), (d, d)) * (rng.random((d, d)) < 0.5)
        o = oracle.solve_hosting(d, c, V)
        a = ctx.solve_hosting(d, c, V)
        np.testing.assert_array_equal(a["hosting"], o["hosting"])
        assert a["max_egress"] == o["max_egress"]
        assert a["visited"] == o["visited"], (d, c)


def test_hosting_limits(ctx):
    from paper_2503_23830_b200.capi import OrchError
    with pytest.raises(OrchError) as e:  # 64 nodes: lane = node
        ctx.solve_hosting(64, 1, np.zeros((64, 64), np.int64))
    assert e.value.code == 12
    with pytest.raises(OrchError) as e:
        ctx.solve_hosting(6, 4, np.zeros((6, 6), np.int64))
    assert e.value.code == 1
    # orch_nodewise (the in-place relabelling of a balance) stays at d <= 64
    rng = np.random.default_rng(1)
    L, O = random_instance(rng, 72, 300)
    Lt, Ot = torch.from_numpy(L).cuda(), torch.from_numpy(O).cuda()
    bal = ctx.balance(0, 72, Lt, Ot)
    with pytest.raises(OrchError) as e:
        ctx.nodewise(72, 8, Lt, Ot, bal)
    assert e.value.code == 12


def test_solve_hosting_wide_fixtures(ctx):
    """d = 72..256 (tables and warp stacks in global memory) against the
    reference's answers and visit counts (tests/golden/ref_hosting_wide.npz)."""
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_wide.npz"))
    for k in range(len(f["d"])):
        d, c = int(f["d"][k]), int(f["c"][k])
        a = ctx.solve_hosting(d, c, f["V"][k][:d, :d])
        np.testing.assert_array_equal(a["hosting"], f["hosting"][k][:d])
        assert a["max_egress"] == f["max_egress"][k]
        assert a["visited"] == f["visited"][k], (k, d, c)


def test_solve_hosting_c4(ctx, oracle):
    """C4 (d = 2560): the vision phase's volume matrix (the reference greedy's
    balance, rebuilt here by the oracle) hosted on 2, 16 and 32 nodes -- the
    reference's hosting, egress and nodes_visited."""
    import bench_configs as bc
    cfg = bc.CONFIGS["C4x30"]
    name, L, O, kind, lam, v = next(iter(cfg["phases"]()))
    r = oracle.balance(kind, cfg["d"], L, O, lam=lam, v=v)
    V = oracle.volume_matrix(cfg["d"], L, O, r.dest_inst)
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_wide.npz"))
    for k, c in enumerate(f["c4_c"]):
        a = ctx.solve_hosting(2560, int(c), V)
        np.testing.assert_array_equal(a["hosting"], f["c4_hosting"][k])
        assert a["max_egress"] == f["c4_max_egress"][k]
        assert a["visited"] == f["c4_visited"][k]


def test_solve_hosting_repeated(ctx):
    """The search state lives in the reused workspace: back-to-back searches
    (the pipelined bench re-hosts every phase of every step) must not see
    each other's work-queue entries."""
    f = np.load(os.path.join(HERE, "golden", "ref_hosting_c3.npz"))
    for _ in range(6):
        for k in range(len(f["c"])):
            a = ctx.solve_hosting(64, int(f["c"][k]), f["V"][k])
            np.testing.assert_array_equal(a["hosting"], f["hosting"][k])
            assert a["max_egress"] == f["max_egress"][k]


@pytest.mark.parametrize("d,c", [(8, 1), (8, 2), (8, 4), (6, 2), (9, 3), (10, 5), (16, 8),
                                 (12, 6), (4, 1), (12, 4), (12, 3)])
def test_nodewise_small_path(ctx, oracle, d, c):
    """orch_nodewise's one-CTA path (d <= 32, <= 2^18 leaves; (12, 3) takes the
    multi-CTA path) against the oracle's branch and bound on the volume matrix."""
    rng = np.random.default_rng(d * 100 + c)
    for trial in range(12):
        n = int(rng.integers(d, 400))
        L, O = random_instance(rng, d, n, 1, int(rng.choice([3, 60, 4000])))
        kind = int(rng.integers(0, 4))
        o = oracle.balance(kind, d, L, O, lam=0.01, v=3)
        V = oracle.volume_matrix(d, L, O, o.dest_inst)
        h = oracle.solve_hosting(d, c, V)
        Lt, Ot = torch.from_numpy(L).cuda(), torch.from_numpy(O).cuda()
        bal = ctx.balance(kind, d, Lt, Ot, lam=0.01, v=3)
        hosting, b2i, info = ctx.nodewise(d, c, Lt, Ot, bal)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(hosting.cpu().numpy(), h["hosting"])
        np.testing.assert_array_equal(b2i.cpu().numpy(), h["batch_to_instance"])
        assert int(info[0]) == h["max_egress"] and int(info[1]) == h["baseline_max"]
        di = h["batch_to_instance"][o.dest_inst]
        np.testing.assert_array_equal(bal.dest_inst[:n].cpu().numpy(), di)
        inv = np.argsort(h["batch_to_instance"])
        np.testing.assert_array_equal(bal.bin_count.cpu().numpy(), o.bin_count[inv])
        off = bal.bin_offset.cpu().numpy()
        mem = bal.bin_member[:n].cpu().numpy()
        for j in range(d):
            seg = mem[off[j]:off[j + 1]]
            assert (di[seg] == j).all() and (o.dest_slot[seg] == np.arange(len(seg))).all()


def test_inter_node_egress(ctx, oracle):
    """orch_inter_node_egress_host (topology.cpp:61-89) for any node count
    (c = 1 .. d): the solution's and the identity hosting's egress against the
    oracle's search and a direct sum."""
    rng = np.random.default_rng(61)
    for d, c in [(8, 1), (8, 4), (16, 2), (64, 8), (64, 1), (300, 3), (256, 128)]:
        V = rng.integers(0, 1000, (d, d)) * (rng.random((d, d)) < 0.4)
        nodes = d // c
        for hosting in (np.arange(d) // c, rng.permutation(np.arange(d) // c)):
            e = ctx.inter_node_egress(d, c, V, hosting)
            src_node = np.arange(d) // c
            want = np.array([V[src_node == nd][:, hosting != nd].sum() for nd in range(nodes)])
            np.testing.assert_array_equal(e, want)
        if d <= 12:
            o = oracle.solve_hosting(d, c, V)
            np.testing.assert_array_equal(ctx.inter_node_egress(d, c, V, o["hosting"]),
                                          o["per_node_egress"])


@pytest.mark.parametrize("d,c", [(8, 8), (32, 1), (96, 96), (72, 9), (128, 64)])
def test_solve_hosting_edge_shapes(ctx, oracle, d, c):
    """One node (nothing to choose), 32 nodes of one instance (every lane a
    node), all-zero and single-entry volume matrices, ties everywhere: hosting,
    egress and nodes_visited against the oracle's restatement of the reference."""
    rng = np.random.default_rng(d * 7 + c)
    cases = [np.zeros((d, d), np.int64), np.ones((d, d), np.int64)]
    one = np.zeros((d, d), np.int64)
    one[d - 1, 0] = 5
    cases.append(one)
    if d <= 72:  # (a random matrix on 2 x 64 is beyond the sequential oracle's patience)
        cases.append(rng.integers(0, 3, (d, d)) * (rng.random((d, d)) < 0.2))
    for V in cases:
        o = oracle.solve_hosting(d, c, V)
        a = ctx.solve_hosting(d, c, V)
        np.testing.assert_array_equal(a["hosting"], o["hosting"])
        assert a["max_egress"] == o["max_egress"] and a["visited"] == o["visited"], (d, c)
