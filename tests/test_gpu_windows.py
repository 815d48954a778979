"""The multi-GPU data plane on ONE GPU: P ranks emulated in this process.

Loopback communicators (orch_comm_create_local) and windows
(orch_window_create_local) run the same kernels as across GPUs -- the fused
pack+put k_move_tma<kPut> / k_move<kPut>, the peer-memory k_window_barrier,
the consumer release k_window_release and the gather window's k_gather_put --
with each emulated rank on its own stream. Expected placements come from the
oracle's layout (apply() on rows, core.cpp:120-161); rows are tagged and
compared on the device (tests/rowcheck.py). The NCCL entry points are covered
by tests/test_multigpu.py on 2+ GPUs; the NCCL symmetric-memory window also on
a one-rank communicator here.
"""
import numpy as np
import pytest
import torch

from conftest import random_instance
from rowcheck import fill_tagged, first_mismatch, rows_equal, source_rows

pytestmark = pytest.mark.gpu


class Group:
    """P loopback ranks: communicators, windows of `nbytes`, one stream each."""

    def __init__(self, ctx, P, nbytes):
        from paper_2503_23830_b200.capi import Comm, Context, Window
        self.P = P
        # a context of its own: the ranks' streams get their own workspaces
        # without recycling the session context's (a recycle synchronises the
        # device, which must not happen between two ranks' halves of a barrier)
        self.ctx = Context(0)
        self.comms = Comm.local_group(P)
        self.wins = Window.local_group(self.ctx, self.comms, nbytes)
        self.views = [w.tensor_view(torch.device("cuda", 0)) for w in self.wins]
        self.streams = [torch.cuda.Stream() for _ in range(P)]
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)

    def close(self):
        torch.cuda.synchronize()
        self.views = None
        for w in self.wins:
            w.close()
        for c in self.comms:
            c.close()
        self.ctx.close()


def rank_inputs(e, P, R, seed=0):
    """One device buffer holding every rank's input rows (rank r at in_base[r])."""
    in_rows = np.asarray(e["in_tokens"], np.int64)
    in_base = np.concatenate([[0], np.cumsum(in_rows)[:-1]])
    big = torch.empty(max(int(in_rows.sum()), 1) * R, dtype=torch.uint8, device="cuda")
    fill_tagged(big, R, seed=seed)
    ins = [big[int(in_base[r]) * R:(int(in_base[r]) + max(int(in_rows[r]), 1)) * R]
           for r in range(P)]
    return big, ins, in_base


def put_step(ctx, g, d, L, O, bal, lay, R, ins, offset=0, barrier=True):
    ctx = g.ctx
    for r in range(g.P):
        ctx.put(d, L, O, bal, lay, R, ins[r], g.wins[r], g.comms[r], offset=offset,
                stream=g.streams[r])
    if barrier:
        for r in range(g.P):
            g.ctx.window_barrier(g.wins[r], stream=g.streams[r])


def balance_case(ctx, oracle, kind, d, P, length, origin, lam=0.01, v=3):
    o = oracle.balance(kind, d, length, origin, lam=lam, v=v)
    e = oracle.layout(d, P, length, origin, o.dest_inst, o.dest_slot)
    L = torch.from_numpy(np.ascontiguousarray(length, np.int64)).cuda()
    O = torch.from_numpy(np.ascontiguousarray(origin, np.int32)).cuda()
    bal = ctx.balance(kind, d, L, O, lam=lam, v=v)
    lay = ctx.layout(d, P, L, O, bal)
    return o, e, L, O, bal, lay


@pytest.mark.parametrize("R", [4096, 8192, 16384])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_put_barrier_emulated(ctx, oracle, P, R):
    """put (k_move<kPut> for R < 8 KiB, k_move_tma<kPut> beyond) + window barrier:
    every rank's window holds its destination batches, byte-exact."""
    rng = np.random.default_rng(31 * P + R)
    for kind in (0, 1, 2, 3):
        c = int(rng.integers(1, 4))
        d = P * c
        n = int(rng.integers(P, 400))
        length, origin = random_instance(rng, d, n, 1, int(rng.choice([3, 40])))
        o, e, L, O, bal, lay = balance_case(ctx, oracle, kind, d, P, length, origin)
        big, ins, in_base = rank_inputs(e, P, R, seed=kind)
        idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], c,
                          P, in_base)
        wbytes = max(int(e["out_tokens"].max()), 1) * R
        g = Group(ctx, P, wbytes)
        for step in range(3):  # epochs 1..3: each step waits for the previous release
            put_step(ctx, g, d, L, O, bal, lay, R, ins)
            for r in range(P):
                g.streams[r].synchronize()
                assert rows_equal(g.views[r], big, idx[r], R), \
                    (kind, step, r, first_mismatch(g.views[r], big, idx[r], R))
                g.views[r][:wbytes].zero_()
            torch.cuda.synchronize()
            for r in range(P):
                g.ctx.window_release(g.wins[r], stream=g.streams[r])
        torch.cuda.synchronize()
        assert int(lay.status.item()) == 0
        assert all(w.status() == 0 for w in g.wins)
        g.close()


def test_put_c2_phases_share_one_window(ctx, oracle):
    """The bench's N>1 step at the full C2 size (4.3 GB of rows), 4 emulated ranks:
    both phases put into one window at their offsets, one barrier, one release."""
    from paper_2503_23830_b200 import workload
    P, d, R = 4, 8, 8192
    c = d // P
    b = workload.make_batch(2, d, 64, 2)
    lv, ov, _ = b.phase_items("vision")
    ll, ol = b.llm_items()
    cases, woff = [], 0
    for length, origin in ((lv, ov), (ll, ol)):
        o, e, L, O, bal, lay = balance_case(ctx, oracle, 0, d, P, length, origin)
        big, ins, in_base = rank_inputs(e, P, R, seed=len(cases))
        idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], c,
                          P, in_base)
        wrows = max(int(e["out_tokens"].max()), 1)
        cases.append((L, O, bal, lay, big, ins, idx, woff))
        woff += wrows * R
    g = Group(ctx, P, woff)
    for step in range(2):
        for L, O, bal, lay, big, ins, idx, off in cases:
            put_step(ctx, g, d, L, O, bal, lay, R, ins, offset=off, barrier=False)
        for r in range(P):
            g.ctx.window_barrier(g.wins[r], stream=g.streams[r])
        torch.cuda.synchronize()
        for L, O, bal, lay, big, ins, idx, off in cases:
            assert int(lay.status.item()) == 0
            for r in range(P):
                assert rows_equal(g.views[r][off:], big, idx[r], R), (step, r)
        for r in range(P):
            g.ctx.window_release(g.wins[r], stream=g.streams[r])
    g.close()


def test_put_c5_offsets_beyond_4gib(ctx, oracle):
    """C5 (long context, 16 KiB rows, ~21 GB) through the put on 4 emulated ranks:
    byte offsets in the inputs and windows pass 4 GiB."""
    P, d, R = 4, 8, 16384
    c = d // P
    rng = np.random.default_rng(5)
    length = rng.integers(8192, 32769, d * 8).astype(np.int64)
    origin = (np.arange(d * 8) % d).astype(np.int32)
    o, e, L, O, bal, lay = balance_case(ctx, oracle, 2, d, P, length, origin,
                                        lam=1.0 / (6 * 8192), v=2048)
    assert int(e["in_tokens"].sum()) * R > (1 << 34)
    assert int(e["out_tokens"].max()) * R > (1 << 32)
    big, ins, in_base = rank_inputs(e, P, R, seed=5)
    idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], c, P,
                      in_base)
    g = Group(ctx, P, int(e["out_tokens"].max()) * R)
    put_step(ctx, g, d, L, O, bal, lay, R, ins)
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 0
    for r in range(P):
        assert rows_equal(g.views[r], big, idx[r], R), (r, first_mismatch(g.views[r], big, idx[r], R))
    del big, ins
    g.close()


def test_write_after_read_guard(ctx, oracle):
    """A slow consumer reads each rank's window after step 1's barrier while step 2's
    puts (different rows) are already queued on the ranks' streams. The puts wait on
    the device for every rank's release, so the consumer's snapshot is step 1's rows
    and the window afterwards holds step 2's rows."""
    P, R = 4, 8192
    rng = np.random.default_rng(77)
    d, n = 8, 300
    length, origin = random_instance(rng, d, n, 20, 200)
    c = d // P
    o, e, L, O, bal, lay = balance_case(ctx, oracle, 0, d, P, length, origin)
    big1, ins1, in_base = rank_inputs(e, P, R, seed=1)
    big2, ins2, _ = rank_inputs(e, P, R, seed=2)
    idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], c, P,
                      in_base)
    wbytes = int(e["out_tokens"].max()) * R
    g = Group(ctx, P, wbytes)
    consumers = [torch.cuda.Stream() for _ in range(P)]
    snaps = [torch.empty(wbytes, dtype=torch.uint8, device="cuda") for _ in range(P)]
    put_step(ctx, g, d, L, O, bal, lay, R, ins1)  # step 1 + barrier
    for r in range(P):
        ev = torch.cuda.Event()
        ev.record(g.streams[r])
        consumers[r].wait_event(ev)
        with torch.cuda.stream(consumers[r]):
            torch.cuda._sleep(100_000_000)  # ~50 ms: the consumer is still busy
            snaps[r].copy_(g.views[r][:wbytes])
        g.ctx.window_release(g.wins[r], stream=consumers[r])
    # step 2 is queued at once; nothing on the host waits for the consumers
    put_step(ctx, g, d, L, O, bal, lay, R, ins2)
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 0
    for r in range(P):
        assert rows_equal(snaps[r], big1, idx[r], R), (r, first_mismatch(snaps[r], big1, idx[r], R))
        assert rows_equal(g.views[r], big2, idx[r], R), r
    g.close()


def test_put_without_release_times_out(ctx, oracle):
    """A put issued after a barrier whose rows were never released gives up after
    ~4 s: layout.status = ORCH_CUDA_ERROR and nothing is stored."""
    P, R = 2, 4096
    rng = np.random.default_rng(3)
    d, n = 4, 50
    length, origin = random_instance(rng, d, n, 1, 9)
    o, e, L, O, bal, lay = balance_case(ctx, oracle, 0, d, P, length, origin)
    big, ins, in_base = rank_inputs(e, P, R, seed=9)
    wbytes = int(e["out_tokens"].max()) * R
    g = Group(ctx, P, wbytes)
    put_step(ctx, g, d, L, O, bal, lay, R, ins)
    torch.cuda.synchronize()
    for v in g.views:
        v[:wbytes].fill_(0x5A)
    torch.cuda.synchronize()
    put_step(ctx, g, d, L, O, bal, lay, R, ins, barrier=False)  # no release in between
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 10  # ORCH_CUDA_ERROR
    for v in g.views:
        assert bool((v[:wbytes] == 0x5A).all())
    g.close()


def test_window_barrier_timeout(ctx):
    """A rank whose peer never arrives leaves the barrier after ~4 s with the
    window status set (instead of hanging the stream)."""
    from paper_2503_23830_b200.capi import OrchError
    g = Group(ctx, 2, 4096)
    g.ctx.window_barrier(g.wins[0], stream=g.streams[0])  # rank 1 never calls it
    torch.cuda.synchronize()
    assert g.wins[0].status() == 10
    assert g.wins[1].status() == 0
    with pytest.raises(OrchError):  # nothing was closed on rank 1: nothing to release
        g.ctx.window_release(g.wins[1])
    g.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_gather_put_emulated(ctx, P):
    """gather_lengths through peer memory (k_gather_put): every rank ends with
    the global (length, origin) arrays in input order, over several numbered calls
    (the consumed[] handshake lets call k+1 overwrite call k's window)."""
    from paper_2503_23830_b200.capi import Comm, Context, GatherWindow
    ctx = Context(0)
    comms = Comm.local_group(P)
    max_n = 5000
    gws = GatherWindow.local_group(ctx, comms, max_n)
    streams = [torch.cuda.Stream() for _ in range(P)]
    rng = np.random.default_rng(P)
    for call in range(5):
        d = P * int(rng.integers(1, 5))
        c = d // P
        n = int(rng.integers(1, max_n + 1))
        L = rng.integers(1, 100000, n).astype(np.int64)
        O = rng.integers(0, d, n).astype(np.int32)
        outs = []
        for r in range(P):  # inputs first: a rank's gather waits for every other rank
            mine = np.nonzero(O // c == r)[0]
            outs.append((torch.full((n,), -1, dtype=torch.int64, device="cuda"),
                         torch.full((n,), -1, dtype=torch.int32, device="cuda"),
                         torch.zeros(1, dtype=torch.int32, device="cuda"),
                         torch.from_numpy(mine.astype(np.int64)).cuda(),
                         torch.from_numpy(L[mine]).cuda(), torch.from_numpy(O[mine]).cuda()))
        torch.cuda.synchronize()
        for r, (gl, go, st, pos, ll, lo) in enumerate(outs):
            ctx.allgather_items_put(gws[r], pos, ll, lo, n, gl, go, st, stream=streams[r])
        torch.cuda.synchronize()
        for r, (gl, go, st, *_) in enumerate(outs):
            assert int(st.item()) == 0, (call, r)
            np.testing.assert_array_equal(gl.cpu().numpy(), L)
            np.testing.assert_array_equal(go.cpu().numpy(), O)
    for gw in gws:
        gw.close()
    for cm in comms:
        cm.close()
    ctx.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_bench_chain_emulated(ctx, oracle, P):
    """bench.py's N>1 step, every stage on every emulated rank: gather-put of the
    rank's local lengths -> balance -> node-wise hosting -> layout -> put ->
    window barrier -> release, twice; checked against the oracle (balance,
    solve_hosting, layout) and byte-exact on every rank's window. C2 workload."""
    from paper_2503_23830_b200 import workload
    from paper_2503_23830_b200.capi import Comm, Context, GatherWindow, Window
    ctx = Context(0)
    d, R = 8, 8192
    c = d // P
    b = workload.make_batch(2, d, 64, 2)
    ll, ol = b.llm_items()
    n = len(ll)
    o = oracle.balance(0, d, ll, ol)
    V = oracle.volume_matrix(d, ll, ol, o.dest_inst)
    h = oracle.solve_hosting(d, c, V)
    di = h["batch_to_instance"][o.dest_inst]
    e = oracle.layout(d, P, ll, ol, di, o.dest_slot)
    comms = Comm.local_group(P)
    gws = GatherWindow.local_group(ctx, comms, n)
    wbytes = int(e["out_tokens"].max()) * R
    wins = Window.local_group(ctx, comms, wbytes)
    views = [w.tensor_view(torch.device("cuda", 0)) for w in wins]
    streams = [torch.cuda.Stream() for _ in range(P)]
    big, ins, in_base = rank_inputs(e, P, R, seed=P)
    idx = source_rows(ll, ol, di, e["rank_src_off"], e["rank_dst_off"], c, P, in_base)
    local = []
    for r in range(P):
        mine = np.nonzero(ol // c == r)[0]
        local.append(tuple(torch.from_numpy(x).cuda() for x in
                           (mine.astype(np.int64), ll[mine], ol[mine])))
    torch.cuda.synchronize()
    for step in range(2):
        # One host thread drives every rank, so the collective stages are issued
        # for all ranks before anything that may synchronise a stream (a
        # workspace growth does): gathers, then the local chains, then barriers.
        per_rank = []
        for r in range(P):
            s = streams[r]
            with torch.cuda.stream(s):
                gl = torch.empty(n, dtype=torch.int64, device="cuda")
                go = torch.empty(n, dtype=torch.int32, device="cuda")
            ctx.allgather_items_put(gws[r], *local[r], n, gl, go, stream=s)
            per_rank.append([gl, go])
        for r in range(P):
            s = streams[r]
            gl, go = per_rank[r]
            bal = ctx.balance(0, d, gl, go, stream=s)
            hosting = ctx.nodewise(d, c, gl, go, bal, stream=s)
            lay = ctx.layout(d, P, gl, go, bal, stream=s)
            ctx.put(d, gl, go, bal, lay, R, ins[r], wins[r], comms[r], stream=s)
            per_rank[r] += [bal, lay, hosting]
        for r in range(P):
            ctx.window_barrier(wins[r], stream=streams[r])
        torch.cuda.synchronize()
        for r, (gl, go, bal, lay, _) in enumerate(per_rank):
            assert int(lay.status.item()) == 0
            np.testing.assert_array_equal(bal.dest_inst[:n].cpu().numpy(), di)
            np.testing.assert_array_equal(bal.dest_slot[:n].cpu().numpy(), o.dest_slot)
            np.testing.assert_array_equal(lay.rank_dst_off[:n].cpu().numpy(), e["rank_dst_off"])
            assert rows_equal(views[r], big, idx[r], R), (step, r)
            views[r].zero_()
        torch.cuda.synchronize()
        for r in range(P):
            ctx.window_release(wins[r], stream=streams[r])
    torch.cuda.synchronize()
    views = None
    for w in wins:
        w.close()
    for gw in gws:
        gw.close()
    for cm in comms:
        cm.close()
    ctx.close()


def test_nccl_symmetric_window_one_rank(ctx, oracle):
    """orch_window_create_nccl on a one-rank NCCL communicator (the driver's
    one-GPU run): ncclMemAlloc + ncclCommWindowRegister, the rank's address from
    the device API's ncclGetPeerPointer (NCCL's flat mapping of the window, not
    the allocation's own address), then the put, barrier and release through it,
    byte-exact; two steps."""
    from paper_2503_23830_b200.capi import Comm, Window
    rng = np.random.default_rng(11)
    d, R = 8, 4096
    length, origin = random_instance(rng, d, 400, 1, 40)
    o, e, L, O, bal, lay = balance_case(ctx, oracle, 0, d, 1, length, origin)
    comm = Comm(1, 0, Comm.unique_id())
    big, ins, in_base = rank_inputs(e, 1, R, seed=5)
    win = Window(ctx, comm, max(int(e["out_tokens"][0]), 1) * R, backend="nccl")
    view = win.tensor_view(torch.device("cuda", 0))
    idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], d, 1,
                      in_base)
    for _ in range(2):
        view.zero_()
        ctx.put(d, L, O, bal, lay, R, ins[0], win, comm)
        ctx.window_barrier(win)
        torch.cuda.synchronize()
        assert int(lay.status.item()) == 0 and win.status() == 0
        assert rows_equal(view, big, idx[0], R), first_mismatch(view, big, idx[0], R)
        ctx.window_release(win)
    torch.cuda.synchronize()
    view = None
    win.close()
    comm.close()
