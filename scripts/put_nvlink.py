"""The fused put over real NVLink from ONE process (P GPUs, loopback
communicators and windows with one rank per device, peer access): every rank's
C2 LLM-phase rows are put into the destination ranks' windows and checked
byte-exactly against the oracle's placement. One process means ncu can profile
the put kernel while it stores into a peer GPU (a multi-rank ncu run hangs on
the ranks' waits):

    python scripts/put_nvlink.py [P]                    # run + check, print GB/s
    ncu --set full -k regex:k_move_tma -c 1 -o put python scripts/put_nvlink.py 2 --no-barrier
"""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2503_23830_b200 import workload  # noqa: E402
from paper_2503_23830_b200.capi import Comm, Context, Window  # noqa: E402
from rowcheck import fill_tagged, rows_equal, source_rows  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
    barrier = "--no-barrier" not in sys.argv
    d, R = 8, 8192
    c = d // P
    orc = Oracle()
    b = workload.make_batch(2, d, 64, 2)
    L, O = b.llm_items()
    o = orc.balance(0, d, L, O)
    e = orc.layout(d, P, L, O, o.dest_inst, o.dest_slot)
    comms, ctxs, streams, ins, bals = [], [], [], [], []
    for r in range(P):
        torch.cuda.set_device(r)
        comms.append(Comm(P, r, None))
        ctxs.append(Context(r))
        streams.append(torch.cuda.Stream(device=r))
    wbytes = int(e["out_tokens"].max()) * R
    wins = Window.local_group(ctxs[0], comms, wbytes)
    big = []
    for r in range(P):
        torch.cuda.set_device(r)
        dev = torch.device("cuda", r)
        Lt = torch.from_numpy(L).to(dev)
        Ot = torch.from_numpy(O).to(dev)
        bal = ctxs[r].balance(0, d, Lt, Ot)
        lay = ctxs[r].layout(d, P, Lt, Ot, bal)
        rows = max(int(e["in_tokens"][r]), 1)
        x = torch.empty(rows * R, dtype=torch.uint8, device=dev)
        fill_tagged(x, R, seed=r)
        ins.append(x)
        bals.append((Lt, Ot, bal, lay))
    for r in range(P):
        torch.cuda.synchronize(r)
    t0 = time.perf_counter()
    ev = []
    for r in range(P):
        torch.cuda.set_device(r)
        Lt, Ot, bal, lay = bals[r]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[r])
        ctxs[r].put(d, Lt, Ot, bal, lay, R, ins[r], wins[r], comms[r], stream=streams[r])
        e1.record(streams[r])
        ev.append((e0, e1))
    if barrier:
        for r in range(P):
            torch.cuda.set_device(r)
            ctxs[r].window_barrier(wins[r], stream=streams[r])
    for r in range(P):
        torch.cuda.synchronize(r)
    wall = time.perf_counter() - t0
    ms = max(a.elapsed_time(z) for a, z in ev)
    S = e["send_tokens"]
    egress = max(int(S[r].sum() - S[r, r]) for r in range(P)) * R
    print(f"P={P} put max {ms:.3f} ms, bottleneck egress {egress / 1e6:.0f} MB -> "
          f"{egress / ms / 1e6:.0f} GB/s (wall {wall * 1e3:.1f} ms)", flush=True)
    # byte check: all inputs concatenated on one device vs every rank's window
    torch.cuda.set_device(0)
    allin = torch.cat([x.to("cuda:0") for x in ins])
    in_base = np.concatenate([[0], np.cumsum([x.numel() // R for x in ins])[:-1]])
    idx = source_rows(L, O, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], c, P, in_base)
    ok = True
    for r in range(P):
        view = wins[r].tensor_view(torch.device("cuda", r)).to("cuda:0")
        ok = ok and rows_equal(view, allin, idx[r], R)
    for r in range(P):
        assert int(bals[r][3].status.item()) == 0 and wins[r].status() == 0
    print("bytes", "OK" if ok else "MISMATCH", flush=True)
    for w in wins:
        w.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
