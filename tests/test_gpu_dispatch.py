"""GPU parity of the send/recv layout and the token-row movement.

Packed buffers are "parity unpinned" by the reference (it moves no tensor
data); their canonical definition is apply() (core.cpp:120-161)
on token rows, restated by the oracle (orc_layout / orc_dispatch_rows). Row
content is a function of (item, row, chunk) so any misplaced byte is caught.
Multi-rank pack/unpack is exercised on one GPU by emulating the all-to-all
with device copies between per-rank buffers (the NCCL path itself is covered
by tests/test_multigpu.py under gpurun --gpus N).
"""
import numpy as np
import pytest
import torch

from conftest import random_instance

pytestmark = pytest.mark.gpu


def to_dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a, dt)).cuda()


def make_case(rng, d, n, hi=20, kind=0):
    length, origin = random_instance(rng, d, n, 1, hi)
    return length, origin


def expected_layout(oracle, d, P, length, origin, o):
    return oracle.layout(d, P, length, origin, o.dest_inst, o.dest_slot)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_layout_matches_oracle(ctx, oracle, P):
    rng = np.random.default_rng(100 + P)
    for kind in (0, 1, 2, 3):
        for _ in range(8):
            d = P * int(rng.integers(1, 9))
            n = int(rng.integers(1, 400))
            length, origin = make_case(rng, d, n, hi=int(rng.choice([3, 50, 900])))
            o = oracle.balance(kind, d, length, origin, lam=0.01, v=5)
            L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
            bal = ctx.balance(kind, d, L, O, lam=0.01, v=5)
            lay = ctx.layout(d, P, L, O, bal)
            torch.cuda.synchronize()
            e = expected_layout(oracle, d, P, length, origin, o)
            np.testing.assert_array_equal(lay.rank_src_off[:n].cpu().numpy(), e["rank_src_off"])
            np.testing.assert_array_equal(lay.rank_dst_off[:n].cpu().numpy(), e["rank_dst_off"])
            np.testing.assert_array_equal(lay.in_rows.cpu().numpy(), e["in_tokens"])
            np.testing.assert_array_equal(lay.out_rows.cpu().numpy(), e["out_tokens"])
            if P > 1:
                np.testing.assert_array_equal(lay.pair_off[:n].cpu().numpy(), e["pair_off"])
                np.testing.assert_array_equal(lay.send_rows.cpu().numpy().reshape(P, P),
                                              e["send_tokens"])


@pytest.mark.parametrize("P,d,n", [(1, 320, 3000), (4, 64, 20000), (8, 512, 30000),
                                   (2, 256, 16384), (2, 256, 16385), (8, 256, 500), (1, 257, 500)])
def test_layout_multi_kernel_path(ctx, oracle, P, d, n):
    """Either side of the single-CTA layout limits (n <= 16384, d <= 256)."""
    rng = np.random.default_rng(7 * P + d)
    length, origin = make_case(rng, d, n, hi=300)
    o = oracle.balance(0, d, length, origin)
    L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
    bal = ctx.balance(0, d, L, O)
    lay = ctx.layout(d, P, L, O, bal)
    torch.cuda.synchronize()
    e = expected_layout(oracle, d, P, length, origin, o)
    np.testing.assert_array_equal(lay.rank_src_off[:n].cpu().numpy(), e["rank_src_off"])
    np.testing.assert_array_equal(lay.rank_dst_off[:n].cpu().numpy(), e["rank_dst_off"])
    np.testing.assert_array_equal(lay.out_rows.cpu().numpy(), e["out_tokens"])
    if P > 1:
        np.testing.assert_array_equal(lay.pair_off[:n].cpu().numpy(), e["pair_off"])
        np.testing.assert_array_equal(lay.send_rows.cpu().numpy().reshape(P, P), e["send_tokens"])


def test_balance_layout1_matches_the_pair(ctx, oracle):
    """orch_balance_layout1 (balance + single-rank layout in one launch when small,
    else the two calls) equals orch_balance followed by orch_layout(P = 1)."""
    rng = np.random.default_rng(1234)
    cases = [(int(rng.integers(1, 65)), int(rng.integers(1, 4097))) for _ in range(24)]
    cases += [(8, 301), (64, 4096), (65, 500), (8, 4097), (300, 6000)]
    for t, (d, n) in enumerate(cases):
        kind = t % 4
        length, origin = make_case(rng, d, n, hi=int(rng.choice([3, 900, 70000])), kind=kind)
        L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
        for ident in (False, True):
            b1 = ctx.balance(kind, d, L, O, lam=1e-4, v=64, identity_only=ident)
            l1 = ctx.layout(d, 1, L, O, b1)
            b2, l2 = ctx.balance_layout1(kind, d, L, O, lam=1e-4, v=64, identity_only=ident)
            torch.cuda.synchronize()
            for k in ("dest_inst", "dest_slot", "src_off", "dst_off"):
                assert torch.equal(getattr(b1, k)[:n], getattr(b2, k)[:n]), (d, n, kind, k)
            for k in ("rank_src_off", "rank_dst_off", "pair_off"):
                assert torch.equal(getattr(l1, k)[:n], getattr(l2, k)[:n]), (d, n, kind, ident, k)
            for k in ("send_rows", "send_displ", "recv_displ", "in_rows", "out_rows", "status"):
                assert torch.equal(getattr(l1, k), getattr(l2, k)), (d, n, kind, ident, k)


def test_volume_matrix(ctx, oracle):
    rng = np.random.default_rng(3)
    for d in (1, 3, 8, 64, 300):
        n = 2000
        length, origin = make_case(rng, d, n, hi=4096)
        o = oracle.balance(0, d, length, origin)
        L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
        V = ctx.volume_matrix(d, L, O, to_dev(o.dest_inst, np.int32))
        np.testing.assert_array_equal(V.cpu().numpy(), oracle.volume_matrix(d, length, origin,
                                                                            o.dest_inst))


def host_inputs(oracle, d, P, length, origin, o, R):
    e = oracle.layout(d, P, length, origin, o.dest_inst, o.dest_slot)
    c = d // P
    ins = [np.zeros(max(int(e["in_tokens"][r]), 1) * R, np.uint8) for r in range(P)]
    tags = np.arange(len(length), dtype=np.int64) * 1000003 + 17
    for r in range(P):
        sel = np.nonzero(np.asarray(origin) // c == r)[0]
        oracle.fill_rows(length[sel], tags[sel], e["rank_src_off"][sel], R, ins[r])
    outs = [np.zeros(max(int(e["out_tokens"][r]), 1) * R, np.uint8) for r in range(P)]
    oracle.dispatch_rows(d, P, length, origin, o.dest_inst, e["rank_src_off"],
                         e["rank_dst_off"], R, ins, outs, nthreads=2)
    return e, ins, outs


@pytest.mark.parametrize("R", [16, 64, 8192, 16384, 12288])
def test_dispatch_one_rank_bytes(ctx, oracle, R):
    rng = np.random.default_rng(R)
    cases = [(8, 512, 30), (1, 40, 9), (33, 700, 12), (64, 3000, 5)] if R < 8192 else \
        [(8, 256, 40), (1, 3, 1), (16, 400, 3)]
    for d, n, hi in cases:
        for kind in (0, 1, 2, 3):
            length, origin = make_case(rng, d, n, hi)
            o = oracle.balance(kind, d, length, origin, lam=0.002, v=4)
            e, ins, outs = host_inputs(oracle, d, 1, length, origin, o, R)
            L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
            bal = ctx.balance(kind, d, L, O, lam=0.002, v=4)
            lay = ctx.layout(d, 1, L, O, bal)
            rin = torch.from_numpy(ins[0]).cuda()
            rout = torch.zeros_like(rin)
            ctx.dispatch(d, L, O, bal, lay, R, rin, rout)
            torch.cuda.synchronize()
            assert int(lay.status.item()) == 0
            assert torch.equal(rout.cpu(), torch.from_numpy(outs[0]))


@pytest.mark.parametrize("R", [32, 8192, 24576])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_pack_unpack_emulated_ranks(ctx, oracle, P, R):
    """pack on every rank -> emulated all-to-all (device copies of the
    r->q segments at the layout displacements) -> unpack on every rank.
    R >= 8 KiB exercises the TMA bulk-copy movement kernels."""
    rng = np.random.default_rng(7 * P + R)
    for kind in (0, 1, 2, 3):
        for trial in range(3 if R == 32 else 2):
            d = P * int(rng.integers(1, 5))
            n = int(rng.integers(1, 600 if R == 32 else 200))
            length, origin = make_case(rng, d, n, hi=int(rng.choice([4, 40] if R == 32 else [3, 9])))
            o = oracle.balance(kind, d, length, origin, lam=0.01, v=3)
            e, ins, outs = host_inputs(oracle, d, P, length, origin, o, R)
            L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
            bal = ctx.balance(kind, d, L, O, lam=0.01, v=3)
            lay = ctx.layout(d, P, L, O, bal)
            torch.cuda.synchronize()
            S = lay.send_rows.cpu().numpy().reshape(P, P)
            sd = lay.send_displ.cpu().numpy().reshape(P, P)
            rd = lay.recv_displ.cpu().numpy().reshape(P, P)
            np.testing.assert_array_equal(S, e["send_tokens"])
            d_in = [torch.from_numpy(x).cuda() for x in ins]
            d_out = [torch.zeros(len(x), dtype=torch.uint8, device="cuda") for x in outs]
            send_rows = [max(int(S[r].sum() - S[r, r]), 1) for r in range(P)]
            recv_rows = [max(int(S[:, q].sum() - S[q, q]), 1) for q in range(P)]
            d_send = [torch.zeros(x * R, dtype=torch.uint8, device="cuda") for x in send_rows]
            d_recv = [torch.zeros(x * R, dtype=torch.uint8, device="cuda") for x in recv_rows]
            for r in range(P):
                ctx.pack(r, P, d, L, O, bal, lay, R, d_in[r], d_out[r], d_send[r])
            for r in range(P):
                for q in range(P):
                    if q == r or S[r, q] == 0:
                        continue
                    a, b = int(sd[r, q]) * R, int(rd[q, r]) * R
                    k = int(S[r, q]) * R
                    d_recv[q][b:b + k].copy_(d_send[r][a:a + k])
            for q in range(P):
                ctx.unpack(q, P, d, L, O, bal, lay, R, d_recv[q], d_out[q])
            torch.cuda.synchronize()
            assert int(lay.status.item()) == 0
            for q in range(P):
                assert torch.equal(d_out[q].cpu(), torch.from_numpy(outs[q])), (kind, q)


def test_capacity_guard(ctx, oracle):
    """A too-small output buffer moves nothing and flags layout.status."""
    rng = np.random.default_rng(1)
    length, origin = make_case(rng, 4, 100, 10)
    L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
    bal = ctx.balance(0, 4, L, O)
    lay = ctx.layout(4, 1, L, O, bal)
    R = 16
    rin = torch.ones(int(length.sum()) * R, dtype=torch.uint8, device="cuda")
    rout = torch.zeros(int(length.sum()) * R - R, dtype=torch.uint8, device="cuda")
    ctx.dispatch(4, L, O, bal, lay, R, rin, rout)
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 1
    assert int(rout.sum().item()) == 0


def test_group_by_origin_and_costs(ctx, oracle):
    rng = np.random.default_rng(21)
    for variant in (0, 1, 2):
        for padded in (0, 1):
            d, n = 12, 300
            length, origin = make_case(rng, d, n, hi=70000)
            L, O = to_dev(length, np.int64), to_dev(origin, np.int32)
            off, mem = ctx.group_by_origin(d, O)
            np.testing.assert_array_equal(mem.cpu().numpy(), np.argsort(origin, kind="stable"))
            cost, stats = ctx.batch_costs(1.5, 0.003, padded, variant, padded, d, L, off, mem)
            exp = np.array([oracle.cost(1.5, 0.003, padded, variant, padded, length[origin == i])
                            for i in range(d)])
            assert cost.cpu().numpy().tobytes() == exp.tobytes()
            assert tuple(stats.cpu().numpy()) == oracle.stats(exp)


def test_encode_lengths(ctx):
    """encode_lengths / interleaved_length (test_core.cpp:154-201 values)."""
    # examples: {text 8, vision 784, audio 100}, {text 8}, {vision 784, text 12}, {vision 1, vision 5}
    part_offset = to_dev([0, 3, 4, 6, 8], np.int32)
    modality = to_dev([0, 1, 2, 0, 1, 0, 1, 1], np.int32)
    meta = to_dev([8, 784, 100, 8, 784, 12, 1, 5], np.int64)
    enc, inter = ctx.encode_lengths(part_offset, modality, meta, [1, 4, 2])
    assert enc.cpu().tolist() == [8, 196, 50, 8, 196, 12, 1, 2]
    assert inter.cpu().tolist() == [254, 8, 208, 3]
    from paper_2503_23830_b200.capi import OrchError
    with pytest.raises(OrchError) as e:
        ctx.encode_lengths(part_offset, modality, meta, [1, 0, 2])
    assert e.value.code == 2
