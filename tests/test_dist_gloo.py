"""World-size-2 and -4 gloo tests of the N>1 host logic (CPU): local shards by origin
rank, the length all-gather (records scattered back into input order), and the
rank-level exchange layout (send/recv displacements, pair offsets) realised
with gloo send/recv on host buffers -- the same protocol orch_allgather_items /
orch_pack / orch_exchange / orch_unpack run over NCCL on B200s."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    ok = True
    R = 16
    for seed in range(5):
        for kind in (0, 1, 2, 3):
            rng = np.random.default_rng(seed * 10 + kind)
            c = int(rng.integers(1, 4))
            d = world * c
            n = int(rng.integers(world, 200))
            L = rng.integers(1, 9, n).astype(np.int64)
            O = rng.integers(0, d, n).astype(np.int32)
            mine = np.nonzero(O // c == rank)[0]
            max_local = int(np.bincount(O // c, minlength=world).max())
            rec = np.full((max_local, 3), -1, np.int64)
            rec[:len(mine), 0] = mine
            rec[:len(mine), 1] = L[mine]
            rec[:len(mine), 2] = O[mine]
            got = [torch.empty(max_local, 3, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(got, torch.from_numpy(rec))
            gl = np.zeros(n, np.int64)
            go = np.zeros(n, np.int32)
            for g in got:
                for p, ln, o in g.numpy():
                    if p >= 0:
                        gl[p], go[p] = ln, o
            ok &= np.array_equal(gl, L) and np.array_equal(go, O)
            # replicated balance + layout
            r = orc.balance(kind, d, gl, go, lam=0.01, v=2)
            e = orc.layout(d, world, gl, go, r.dest_inst, r.dest_slot)
            S = e["send_tokens"]
            # this rank's input rows
            inp = np.zeros(max(int(e["in_tokens"][rank]), 1) * R, np.uint8)
            orc.fill_rows(L[mine], mine.astype(np.int64), e["rank_src_off"][mine], R, inp)
            out = np.zeros(max(int(e["out_tokens"][rank]), 1) * R, np.uint8)
            # send displacements: segments q != rank in q order
            sdis, a = {}, 0
            for qq in range(world):
                if qq != rank:
                    sdis[qq] = a
                    a += int(S[rank, qq])
            rdis, b = {}, 0
            for rr in range(world):
                if rr != rank:
                    rdis[rr] = b
                    b += int(S[rr, rank])
            send = np.zeros(max(a, 1) * R, np.uint8)
            recv = np.zeros(max(b, 1) * R, np.uint8)
            for i in mine:  # pack
                qd = r.dest_inst[i] // c
                src = inp[e["rank_src_off"][i] * R:(e["rank_src_off"][i] + L[i]) * R]
                if qd == rank:
                    out[e["rank_dst_off"][i] * R:(e["rank_dst_off"][i] + L[i]) * R] = src
                else:
                    o = (sdis[qd] + e["pair_off"][i]) * R
                    send[o:o + L[i] * R] = src
            reqs = []  # exchange
            for qq in range(world):
                if qq == rank:
                    continue
                if S[rank, qq]:
                    reqs.append(dist.isend(torch.from_numpy(
                        send[sdis[qq] * R:(sdis[qq] + S[rank, qq]) * R].copy()), qq))
            bufs = {}
            for rr in range(world):
                if rr != rank and S[rr, rank]:
                    bufs[rr] = torch.empty(int(S[rr, rank]) * R, dtype=torch.uint8)
                    dist.recv(bufs[rr], rr)
            for w in reqs:
                w.wait()
            for rr, t in bufs.items():
                recv[rdis[rr] * R:(rdis[rr] + S[rr, rank]) * R] = t.numpy()
            for i in np.nonzero(r.dest_inst // c == rank)[0]:  # unpack
                rr = O[i] // c
                if rr == rank:
                    continue
                o = (rdis[rr] + e["pair_off"][i]) * R
                out[e["rank_dst_off"][i] * R:(e["rank_dst_off"][i] + L[i]) * R] = \
                    recv[o:o + L[i] * R]
            # expected: apply() on rows over all ranks
            ins = [np.zeros(max(int(e["in_tokens"][x]), 1) * R, np.uint8) for x in range(world)]
            for x in range(world):
                sel = np.nonzero(O // c == x)[0]
                orc.fill_rows(L[sel], sel.astype(np.int64), e["rank_src_off"][sel], R, ins[x])
            outs = [np.zeros(max(int(e["out_tokens"][x]), 1) * R, np.uint8) for x in range(world)]
            orc.dispatch_rows(d, world, L, O, r.dest_inst, e["rank_src_off"], e["rank_dst_off"],
                              R, ins, outs)
            ok &= np.array_equal(out, outs[rank])
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
