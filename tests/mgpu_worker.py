"""Multi-GPU worker (one process per GPU, launched by tests/test_multigpu.py
through torch.distributed.run). Each rank holds only its origin instances'
items and token rows; the path runs end to end through the C-ABI:
all-gather of lengths (ncclAllGather) -> replicated balance -> layout ->
pack -> grouped ncclSend/ncclRecv -> unpack. Every rank checks its output
buffer byte-for-byte against the oracle's apply() on rows."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle  # noqa: E402
from paper_2503_23830_b200.capi import Comm, Context, GatherWindow, OrchError, Window, XPlan  # noqa: E402


def main():
    # small cases still take the sliced, pipelined staged NCCL path (4 slices)
    os.environ.setdefault("ORCH_NCCL_MIN_SLICE_BYTES", "65536")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    uid = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = Comm(world, rank, uid[0])
    ctx = Context(local)
    orc = Oracle()
    P = world
    failures = 0
    cases = 0
    gwin = GatherWindow(ctx, comm, 300)
    gwin_nccl = GatherWindow(ctx, comm, 300, backend="nccl")  # NCCL symmetric memory
    for seed in range(6):
        for kind in (0, 1, 2, 3):
            for R in (32, 8192):
                rng = np.random.default_rng(1000 * seed + 10 * kind + (R > 32))
                c = int(rng.integers(1, 4))
                d = P * c
                n = int(rng.integers(P, 300))
                hi = 12 if R == 32 else 4
                L = rng.integers(1, hi + 1, n).astype(np.int64)
                O = (rng.integers(0, d, n) if seed % 2 else np.arange(n) % d).astype(np.int32)
                mine = np.nonzero(O // c == rank)[0]
                max_local = int(np.bincount(O // c, minlength=P).max())
                gl = torch.zeros(n, dtype=torch.int64, device="cuda")
                go = torch.zeros(n, dtype=torch.int32, device="cuda")
                ctx.allgather_items(comm, torch.from_numpy(mine.astype(np.int64)).cuda(),
                                    torch.from_numpy(L[mine]).cuda(),
                                    torch.from_numpy(O[mine]).cuda(), max_local, n, gl, go)
                torch.cuda.synchronize()
                ok = np.array_equal(gl.cpu().numpy(), L) and np.array_equal(go.cpu().numpy(), O)
                # the same records through peer memory (one window, numbered calls)
                gl2 = torch.full((n,), -1, dtype=torch.int64, device="cuda")
                go2 = torch.full((n,), -1, dtype=torch.int32, device="cuda")
                gst = torch.zeros(1, dtype=torch.int32, device="cuda")
                ctx.allgather_items_put(gwin, torch.from_numpy(mine.astype(np.int64)).cuda(),
                                        torch.from_numpy(L[mine]).cuda(),
                                        torch.from_numpy(O[mine]).cuda(), n, gl2, go2, gst)
                torch.cuda.synchronize()
                ok = ok and np.array_equal(gl2.cpu().numpy(), L)
                ok = ok and np.array_equal(go2.cpu().numpy(), O) and int(gst.item()) == 0
                gl2.fill_(-1)
                go2.fill_(-1)
                ctx.allgather_items_put(gwin_nccl, torch.from_numpy(mine.astype(np.int64)).cuda(),
                                        torch.from_numpy(L[mine]).cuda(),
                                        torch.from_numpy(O[mine]).cuda(), n, gl2, go2, gst)
                torch.cuda.synchronize()
                ok = ok and np.array_equal(gl2.cpu().numpy(), L)
                ok = ok and np.array_equal(go2.cpu().numpy(), O) and int(gst.item()) == 0
                bal = ctx.balance(kind, d, gl, go, lam=0.01, v=3)
                lay = ctx.layout(d, P, gl, go, bal)
                torch.cuda.synchronize()
                ref = orc.balance(kind, d, L, O, lam=0.01, v=3)
                e = orc.layout(d, P, L, O, ref.dest_inst, ref.dest_slot)
                ins = [np.zeros(max(int(e["in_tokens"][r]), 1) * R, np.uint8) for r in range(P)]
                tags = np.arange(n, dtype=np.int64) * 7919 + 3
                for r in range(P):
                    sel = np.nonzero(O // c == r)[0]
                    orc.fill_rows(L[sel], tags[sel], e["rank_src_off"][sel], R, ins[r])
                outs = [np.zeros(max(int(e["out_tokens"][r]), 1) * R, np.uint8) for r in range(P)]
                orc.dispatch_rows(d, P, L, O, ref.dest_inst, e["rank_src_off"], e["rank_dst_off"],
                                  R, ins, outs)
                S = e["send_tokens"]
                send_rows = max(int(S[rank].sum() - S[rank, rank]), 1)
                recv_rows = max(int(S[:, rank].sum() - S[rank, rank]), 1)
                rin = torch.from_numpy(ins[rank]).cuda()
                rout = torch.zeros(len(outs[rank]), dtype=torch.uint8, device="cuda")
                send = torch.zeros(send_rows * R, dtype=torch.uint8, device="cuda")
                recv = torch.zeros(recv_rows * R, dtype=torch.uint8, device="cuda")
                ctx.dispatch(d, gl, go, bal, lay, R, rin, rout, send, recv, comm)
                torch.cuda.synchronize()
                ok = ok and int(lay.status.item()) == 0
                ok = ok and torch.equal(rout.cpu(), torch.from_numpy(outs[rank]))
                # per-item ncclSend/ncclRecv between the row buffers (no staging)
                xp = XPlan(ctx, n, P)
                ms = torch.cuda.Stream()
                ms.wait_stream(torch.cuda.current_stream())
                ctx.xplan_fetch(xp, d, gl, go, bal, lay, stream=ms)
                rout.zero_()
                ctx.dispatch_nccl(xp, R, rin, rout, comm)
                torch.cuda.synchronize()
                ok = ok and int(lay.status.item()) == 0
                ok = ok and torch.equal(rout.cpu(), torch.from_numpy(outs[rank]))
                # the same plan, staged: pack, one send/recv per peer, unpack
                rout.zero_()
                ctx.dispatch_nccl(xp, R, rin, rout, comm, send=send, recv=recv)
                torch.cuda.synchronize()
                ok = ok and int(lay.status.item()) == 0
                ok = ok and torch.equal(rout.cpu(), torch.from_numpy(outs[rank]))
                xp.close()
                # fused pack + put into IPC windows (one pass over NVLink)
                wbytes = max(int(e["out_tokens"].max()), 1) * R
                win = Window(ctx, comm, wbytes)
                wv = win.tensor_view(torch.device("cuda", local))
                wv.zero_()
                torch.cuda.synchronize()
                dist.barrier()
                ctx.dispatch_put(d, gl, go, bal, lay, R, rin, win, comm)
                torch.cuda.synchronize()
                ok = ok and int(lay.status.item()) == 0
                k = len(outs[rank])
                ok = ok and torch.equal(wv[:k].cpu(), torch.from_numpy(outs[rank]))
                ctx.window_release(win)
                # put + the window's peer-memory barrier, twice (epochs 1, 2): the
                # rows are complete as soon as this rank's barrier returns on its stream
                for _ in range(2):
                    wv.zero_()
                    torch.cuda.synchronize()
                    dist.barrier()
                    ctx.put(d, gl, go, bal, lay, R, rin, win, comm)
                    ctx.window_barrier(win)
                    ok = ok and torch.equal(wv[:k].cpu(), torch.from_numpy(outs[rank]))
                    ctx.window_release(win)
                    torch.cuda.synchronize()
                    ok = ok and int(lay.status.item()) == 0 and win.status() == 0
                    dist.barrier()
                win.close()
                # the same put into NCCL symmetric-memory windows (ncclMemAlloc +
                # ncclCommWindowRegister, peers from ncclGetPeerPointer)
                nwin = Window(ctx, comm, wbytes, backend="nccl")
                nv = nwin.tensor_view(torch.device("cuda", local))
                for _ in range(2):
                    nv.zero_()
                    torch.cuda.synchronize()
                    dist.barrier()
                    ctx.put(d, gl, go, bal, lay, R, rin, nwin, comm)
                    ctx.window_barrier(nwin)
                    ok = ok and torch.equal(nv[:k].cpu(), torch.from_numpy(outs[rank]))
                    ctx.window_release(nwin)
                    torch.cuda.synchronize()
                    ok = ok and int(lay.status.item()) == 0 and nwin.status() == 0
                    dist.barrier()
                nv = None
                nwin.close()
                cases += 1
                if not ok:
                    failures += 1
                    print(f"rank {rank}: MISMATCH seed={seed} kind={kind} R={R} d={d} n={n}",
                          flush=True)
    # windows of different sizes are refused on every rank, before any mapping
    try:
        Window(ctx, comm, 4096 * (1 + rank)).close()
        failures += 1
    except OrchError as e:
        failures += 0 if e.code == 1 else 1
    t = torch.tensor([failures])
    dist.all_reduce(t)
    gwin.close()
    gwin_nccl.close()
    comm.close()
    if rank == 0:
        print(f"MGPU world={world} cases={cases} failures={int(t.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
