#!/usr/bin/env python3
"""Benchmark of the B200 Batch Post-Balancing Dispatcher (BASELINE.json metric).

One step = one iteration's balance + dispatch of the C2 workload
(BASELINE.json configs[1]): DP=8 instances, vision+text batch of 64 examples
per instance from the reference's synthetic MCI generator, per-phase
rebalancing (vision encoder phase on metadata lengths, LLM phase on
interleaved lengths, GreedyUnpadded), bf16 d_model=4096 token rows (8 KiB).
Per phase: [all-gather of lengths] -> cost model + ordering + greedy
assignment + never-worse (one balance call) -> [node-wise hosting] -> send/recv
layout -> row movement. At N GPUs the 8 instances are spread 8/N per GPU
(strong scaling: the job is fixed); the rows move by the fused pack+put into
the peers' windows -- NCCL symmetric-memory windows (ncclCommWindowRegister,
peers from ncclGetPeerPointer) by default, CUDA IPC windows with --exchange put
-- closed by a window barrier + release per step, or, with
--exchange nccl, by pack -> grouped ncclSend/ncclRecv -> unpack.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the data, metadata and per-phase streams each get a hardware queue: a kernel that
# waits for a peer (window barrier, gather) must never sit in front of another
# stream's work in a shared queue (set before CUDA initialises)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "balance+dispatch tokens/s at 1–8 B200; a2a GB/s vs NVLink; max/mean load"
LAM_LONG = 1.0 / (6 * 8192)  # attention vs dense FLOPs per token at d_model 8192
CONFIGS = {
    # the driver's bench line (BASELINE.json configs[1])
    "C2": dict(d=8, per=64, seed=2, mix=2, R=8192,
               workload="C2: DP=8 vision+text MCI batch (64 examples/instance, reference generator "
                        "seed 2), per-phase GreedyUnpadded rebalancing (vision metadata lengths, LLM "
                        "interleaved lengths, vision rate 4), bf16 d=4096 token rows (8 KiB)"),
    # evidence lines (configs[2], configs[4]): python bench.py --config C3|C5
    "C3": dict(d=64, per=64, seed=7, mix=3, R=16384,
               workload="C3: DP=64 vision+audio+text MCI batch (64 examples/instance, seed 7): "
                        "vision GreedyUnpadded, audio BinaryPadded, LLM GreedyUnpadded, bf16 "
                        "d=8192 token rows (16 KiB)"),
    "C5": dict(d=8, per=8, seed=5, mix=0, R=16384,
               workload="C5: DP=8 long-context, 8 sequences/instance, lengths U[8192,32768], "
                        "QuadraticTolerance (lambda=1/(6*8192), v=2048), bf16 d=8192 rows (16 KiB)"),
}
CFG = dict(CONFIGS["C2"], name="C2")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def nvlink_peaks(n_gpus):
    """NVLink ceilings measured by scripts/p2pbench.cu (profiles/nvlink_peaks.json):
    the all-to-all pattern at this GPU count when measured, else at the largest
    measured count below it (e.g. 8 GPUs -> the 4-GPU measurement)."""
    with open(os.path.join(ROOT, "profiles", "nvlink_peaks.json")) as f:
        p = json.load(f)["by_gpus"]
    counts = sorted(int(k) for k in p)
    below = [k for k in counts if k <= n_gpus]
    key = str(below[-1] if below else counts[0])
    a2a = p[key]["a2a"]
    return dict(copy_engine=a2a["ce"], kernel_push=max(a2a["tma"], a2a["stg"]), nccl=a2a["nccl"],
                measured_at_gpus=int(key))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={','.join(map(str, self.gpus))}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                    "sw_power_cap"), f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        except Exception:
            pass
        finally:
            try:
                os.remove(self.path)
            except Exception:
                pass
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


def build_inputs():
    """Phases of one step: (name, lengths, origins, policy kind, lambda, v)."""
    from paper_2503_23830_b200 import workload
    d = CFG["d"]
    if CFG["mix"] == 0:  # long context (C5)
        rng = np.random.default_rng(CFG["seed"])
        n = d * CFG["per"]
        L = rng.integers(8192, 32769, n).astype(np.int64)
        O = (np.arange(n) % d).astype(np.int32)
        return None, [("llm", L, O, 2, LAM_LONG, 2048)]
    b = workload.make_batch(CFG["mix"], d, CFG["per"], CFG["seed"])
    phases = []
    lv, ov, _ = b.phase_items("vision")
    phases.append(("vision", lv, ov, 0, 0.0, 0))
    if CFG["mix"] == 3:
        la, oa, _ = b.phase_items("audio")
        phases.append(("audio", la, oa, 1, 0.0, 0))
    ll, ol = b.llm_items()
    phases.append(("llm", ll, ol, 0, 0.0, 0))
    return b, phases


# --------------------------------------------------------------- reference arm
def cpu_reference_step(phases, nthreads, ref, oracle, bufs):
    """Reference balance() (oracle/_ref: the reference's own code, or the C
    restatement when _ref was not built) + threaded host memcpy dispatch
    restating apply() on token rows."""
    t0 = time.perf_counter()
    d, R = CFG["d"], CFG["R"]
    for (name, L, O, kind, lam, v), (ins, outs) in zip(phases, bufs):
        if ref is not None:
            di, ds, _, _ = ref.balance(kind, d, L, O, lam=lam, v=v)
        else:
            r = oracle.balance(kind, d, L, O, lam=lam, v=v)
            di, ds = r.dest_inst, r.dest_slot
        lay = oracle.layout(d, 1, L, O, di, ds)
        oracle.dispatch_rows(d, 1, L, O, di, lay["rank_src_off"], lay["rank_dst_off"],
                             R, ins, outs, nthreads)
    return time.perf_counter() - t0


def cpu_arm(phases, steps, warmup):
    from oracle import Oracle, RefLib
    oracle = Oracle()
    ref = RefLib() if RefLib.available() else None
    kind = "reference" if ref is not None else "port"
    nthreads = os.cpu_count() or 1
    bufs = []
    for ph in phases:
        rows = int(ph[1].sum())
        bufs.append(([np.ones(rows * CFG["R"], np.uint8)], [np.empty(rows * CFG["R"], np.uint8)]))
    for _ in range(warmup):
        cpu_reference_step(phases, nthreads, ref, oracle, bufs)
    times = [cpu_reference_step(phases, nthreads, ref, oracle, bufs) for _ in range(steps)]
    tokens = sum(int(ph[1].sum()) for ph in phases)
    return times, tokens, kind, nthreads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    _, phases = build_inputs()
    steps = max(1, args.steps)
    times, tokens, kind, nthreads = cpu_arm(phases, steps, max(1, args.warmup))
    total = sum(times)
    value = tokens * steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": CFG["workload"], "global_batch": CFG["d"] * CFG["per"],
                   "dp_instances": CFG["d"], "row_bytes": CFG["R"], "tokens_per_step": tokens},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": nthreads, "kind": kind,
                         "sample": f"full {CFG['name']} step x{steps}: reference balance() per phase "
                                   f"(single thread) + {nthreads}-thread host memcpy dispatch"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_2503_23830_b200.capi import (Balance, Comm, Context, GatherWindow, Layout, OrchError,
                                            Window, XPlan)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    D_INST = CFG["d"]
    if D_INST % world:
        raise SystemExit(f"N must divide the {D_INST} DP instances")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm_meta = comm_data = None
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
        uid = [(Comm.unique_id(), Comm.unique_id()) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        # two communicators: lengths all-gather (metadata stream) and row
        # exchange (data stream) run concurrently, so they must not share one
        comm_meta = Comm(world, rank, uid[0][0])
        comm_data = Comm(world, rank, uid[0][1])
    # one context (workspace arena) per stream
    ctx_data = Context(local)
    P, c, R = world, D_INST // world, CFG["R"]
    batch, phases = build_inputs()
    # The metadata chain (gather, balance, hosting, layout) is latency-bound and
    # runs beside the row movement. Each phase gets its own stream, context and
    # gather window, so the phases' chains overlap one another (ncclAllGather
    # on one communicator needs one stream: --gather nccl keeps a single one).
    per_phase = args.gather == "put" or comm_meta is None
    prio = int(os.environ.get("ORCH_META_PRIO", "-1"))
    ms0 = torch.cuda.Stream(device=dev, priority=prio)
    ctx0 = Context(local)
    meta_ctx = [Context(local) if per_phase and i else ctx0 for i in range(len(phases))]
    meta_streams = [torch.cuda.Stream(device=dev, priority=prio) if per_phase and i else ms0
                    for i in range(len(phases))]
    window_kind = ["nccl" if args.exchange == "put-nccl" else "ipc"]

    def make_gwin(i, n):  # NCCL symmetric memory with --exchange put-nccl (IPC if refused)
        if window_kind[0] == "nccl":
            try:
                return GatherWindow(meta_ctx[i], comm_meta, n, backend="nccl")
            except OrchError as e:
                print(f"[bench] NCCL symmetric window unavailable ({e}); CUDA IPC windows",
                      file=sys.stderr)
                window_kind[0] = "ipc"
        return GatherWindow(meta_ctx[i], comm_meta, n)

    gwins = [make_gwin(i, len(ph[1])) if comm_meta is not None and args.gather == "put" else None
             for i, ph in enumerate(phases)]
    data_stream = torch.cuda.Stream(device=dev)

    # Per phase: local items (global input positions), and two buffer sets of
    # the metadata (global arrays, balance, layout) so step i+1's balance runs
    # on the metadata stream while step i's rows move on the data stream (the
    # paper overlaps the solver with the forward pass).
    st = []
    for i_ph, (name, L, O, kind, lam, v) in enumerate(phases):
        n = len(L)
        mine = np.nonzero(O // c == rank)[0]
        max_local = int(max(np.bincount(O // c, minlength=P)))
        s = dict(name=name, n=n, L=L, O=O, kind=kind, lam=lam, v=v, max_local=max_local,
                 h_pos=torch.from_numpy(mine.astype(np.int64)).pin_memory(),
                 h_len=torch.from_numpy(L[mine]).pin_memory(),
                 h_org=torch.from_numpy(O[mine]).pin_memory(),
                 h_glen=torch.from_numpy(L).pin_memory(),
                 h_gorg=torch.from_numpy(O).pin_memory())
        s["pos"] = s["h_pos"].to(dev)
        s["llen"] = s["h_len"].to(dev)
        s["lorg"] = s["h_org"].to(dev)
        s["buf"] = [dict(glen=torch.from_numpy(L).to(dev), gorg=torch.from_numpy(O).to(dev),
                         bal=Balance.alloc(D_INST, n, dev), lay=Layout.alloc(P, n, dev),
                         meta_done=torch.cuda.Event(), data_done=torch.cuda.Event(),
                         hosting=(torch.empty(D_INST, dtype=torch.int32, device=dev),
                                  torch.empty(D_INST, dtype=torch.int32, device=dev),
                                  torch.empty(4, dtype=torch.int64, device=dev)),
                         xplan=XPlan(ctx_data, n, P)
                         if P > 1 and args.exchange in ("nccl", "nccl-direct") else None)
                    for _ in range(2)]
        s["ctx"], s["ms"], s["gwin"] = meta_ctx[i_ph], meta_streams[i_ph], gwins[i_ph]
        st.append(s)

    meta_marks = []  # ORCH_BENCH_TRACE: events between the metadata sub-steps

    def mark(stream):
        if os.environ.get("ORCH_BENCH_TRACE"):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            meta_marks.append(e)

    probe_x = torch.zeros(1, device=dev)
    probe = []  # ORCH_BENCH_TRACE: one tiny kernel's event-timed latency per phase

    def meta(s, B, stream):
        if os.environ.get("ORCH_BENCH_TRACE"):
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(int(os.environ.get("ORCH_PROBE_CYCLES", "1000")))
            p1.record(stream)
            probe.append((p0, p1))
        mark(stream)
        ctx_meta = s["ctx"]
        if s["gwin"] is not None:  # one single-CTA kernel through peer memory
            ctx_meta.allgather_items_put(s["gwin"], s["pos"], s["llen"], s["lorg"], s["n"],
                                         B["glen"], B["gorg"], stream=stream)
        elif comm_meta is not None:
            ctx_meta.allgather_items(comm_meta, s["pos"], s["llen"], s["lorg"], s["max_local"],
                                     s["n"], B["glen"], B["gorg"], stream=stream)
        mark(stream)
        if P == 1:  # balance + the single-rank layout, one launch for small phases
            ctx_meta.balance_layout1(s["kind"], D_INST, B["glen"], B["gorg"], lam=s["lam"],
                                     v=s["v"], out=B["bal"], layout=B["lay"], stream=stream)
            mark(stream)
            mark(stream)
            mark(stream)
            return
        ctx_meta.balance(s["kind"], D_INST, B["glen"], B["gorg"], lam=s["lam"], v=s["v"],
                         out=B["bal"], stream=stream)
        mark(stream)
        if args.nodewise:  # GPU-wise hosting (orchestrator.cpp:283 with node = GPU)
            ctx_meta.nodewise(D_INST, c, B["glen"], B["gorg"], B["bal"], out=B["hosting"],
                              stream=stream)
        mark(stream)
        ctx_meta.layout(D_INST, P, B["glen"], B["gorg"], B["bal"], out=B["lay"], stream=stream)
        if B["xplan"] is not None:  # the per-item runs for the host's NCCL calls
            ctx_meta.xplan_fetch(B["xplan"], D_INST, B["glen"], B["gorg"], B["bal"], B["lay"],
                                 stream=stream)
        mark(stream)

    # sizing pass (not timed): buffers from this batch's layout
    for s in st:
        for B in s["buf"]:
            meta(s, B, torch.cuda.current_stream())
    torch.cuda.synchronize()
    # Input rows and the NCCL staging buffers are shared by the phases (they
    # run one after another on the data stream); each phase has its own output.
    for s in st:
        lay = s["buf"][0]["lay"]
        s["in_rows"] = int(lay.in_rows[rank].item())
        out_rows = int(lay.out_rows[rank].item())
        S = lay.send_rows.cpu().numpy().reshape(P, P)
        s["moved_rows"] = out_rows  # every row of this rank's output is written once
        s["send_rows"] = int(S[rank].sum() - S[rank, rank])
        s["recv_rows"] = int(S[:, rank].sum() - S[rank, rank])
        s["wrows"] = max(int(lay.out_rows.max().item()), 1)
    # N>1 put: the phases of a step share one window (one barrier, one release),
    # each phase's output at its own offset
    win = None
    if P > 1 and args.exchange in ("put", "put-nccl"):
        off = 0
        for s in st:
            s["win_off"] = off
            off += s["wrows"] * R
        if args.exchange == "put-nccl" and window_kind[0] == "nccl":
            try:
                win = Window(ctx_data, comm_data, off, backend="nccl")
            except OrchError as e:  # NCCL without symmetric memory: the same put, IPC windows
                print(f"[bench] NCCL symmetric window unavailable ({e}); CUDA IPC windows",
                      file=sys.stderr)
                window_kind[0] = "ipc"
        if win is None:
            if args.exchange == "put-nccl":
                args.exchange = "put"
            win = Window(ctx_data, comm_data, off)
        wview = win.tensor_view(dev)
        for s in st:
            s["rout"] = wview[s["win_off"]:s["win_off"] + s["wrows"] * R]
    else:
        for s in st:
            s["rout"] = torch.empty(max(s["buf"][0]["lay"].out_rows[rank].item(), 1) * R,
                                    dtype=torch.uint8, device=dev)
    rin = torch.randint(0, 255, (max(max(s["in_rows"] for s in st), 1) * R,), dtype=torch.uint8,
                        device=dev)
    send = recv = None
    if P > 1 and args.exchange in ("nccl", "nccl-sync"):
        send = torch.empty(max(max(s["send_rows"] for s in st), 1) * R, dtype=torch.uint8,
                           device=dev)
        recv = torch.empty(max(max(s["recv_rows"] for s in st), 1) * R, dtype=torch.uint8,
                           device=dev)
    for s in st:
        s["rin"] = rin[:max(s["in_rows"], 1) * R]
        s["send"], s["recv"] = send, recv
    reg = []
    if P > 1 and args.exchange.startswith("nccl") and args.nccl_register:
        reg = [comm_data.register(rin)] + [comm_data.register(s["rout"]) for s in st]
        reg += [comm_data.register(t) for t in (send, recv) if t is not None]

    disp_events = []
    counter = [0]
    # ORCH_BENCH_TRACE=1: per-phase event timeline of the timed steps (stderr)
    trace = [] if os.environ.get("ORCH_BENCH_TRACE") else None

    def step(record=False, h2d=False):
        b = counter[0] % 2
        counter[0] += 1
        for s in st:
            B = s["buf"][b]
            meta_stream = s["ms"]
            meta_stream.wait_event(B["data_done"])  # rows of step i-2 moved: buffers free
            with torch.cuda.stream(meta_stream):
                if h2d:  # e2e: this step's metadata comes from pinned host memory
                    if comm_meta is None:
                        B["glen"].copy_(s["h_glen"], non_blocking=True)
                        B["gorg"].copy_(s["h_gorg"], non_blocking=True)
                    else:
                        s["pos"].copy_(s["h_pos"], non_blocking=True)
                        s["llen"].copy_(s["h_len"], non_blocking=True)
                        s["lorg"].copy_(s["h_org"], non_blocking=True)
            if trace is not None:
                m0 = torch.cuda.Event(enable_timing=True)
                m0.record(meta_stream)
            meta(s, B, meta_stream)
            B["meta_done"].record(meta_stream)
            if trace is not None:
                m1 = torch.cuda.Event(enable_timing=True)
                m1.record(meta_stream)
                d0 = torch.cuda.Event(enable_timing=True)
                d0.record(data_stream)  # data stream reaches this phase
            data_stream.wait_event(B["meta_done"])
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(data_stream)
            if os.environ.get("ORCH_BENCH_NOMOVE"):  # diagnostics only: metadata alone
                pass
            elif win is not None:  # one barrier per step closes both phases' puts
                ctx_data.put(D_INST, B["glen"], B["gorg"], B["bal"], B["lay"], R, s["rin"],
                             win, comm_data, offset=s["win_off"], stream=data_stream)
                if s is st[-1]:
                    if args.barrier == "window":  # peer-memory flags (one 1-warp kernel)
                        ctx_data.window_barrier(win, stream=data_stream)
                        # the consumer of the rows (the encoder / LLM forward) runs
                        # here; then the window is released, which the next step's
                        # puts on every rank wait for (write-after-read guard)
                        ctx_data.window_release(win, stream=data_stream)
                    elif args.barrier == "nccl":
                        ctx_data.barrier(comm_data, stream=data_stream)
            elif B["xplan"] is not None:  # NCCL with host counts from the metadata stream
                ctx_data.dispatch_nccl(B["xplan"], R, s["rin"], s["rout"], comm_data,
                                       send=s["send"], recv=s["recv"], stream=data_stream)
            else:
                ctx_data.dispatch(D_INST, B["glen"], B["gorg"], B["bal"], B["lay"], R, s["rin"],
                                  s["rout"], s["send"], s["recv"], comm_data, stream=data_stream)
            if record:
                e1.record(data_stream)
                disp_events.append((s["name"], e0, e1))
                if trace is not None:
                    trace.append((counter[0], s["name"], m0, m1, d0, e0, e1))
            B["data_done"].record(data_stream)
        return b

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w0 = time.perf_counter()
    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    # then keep warming for ~0.5 s (untimed): the first few hundred ms of a fresh
    # process move rows up to ~6% slower; every rank runs the same count
    per = (time.perf_counter() - w0) / max(args.warmup, 3)
    extra = int(max_over_ranks(float(min(400, int(0.5 / max(per, 1e-4))))))
    for _ in range(extra):
        step()
    barrier()
    all_ctx = list({id(x): x for x in meta_ctx}.values()) + [ctx_data]
    launches0 = sum(x.launches for x in all_ctx)
    with ClockSampler([local]) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(data_stream)
        for ms in meta_streams:
            ms.wait_event(t0)
        for _ in range(args.steps):
            step(record=True)
        t1.record(data_stream)
        barrier()
    launches = sum(x.launches for x in all_ctx) - launches0
    if trace:
        for gwin in gwins:
            if gwin is None:
                continue
            stm = gwin.stamps().astype(np.int64)
            for row in stm:
                if row[0]:
                    print(f"[trace r{rank}] gather stages us: free {(row[1] - row[0]) / 1e3:.1f} "
                          f"store+fence {(row[2] - row[1]) / 1e3:.1f} wait peers "
                          f"{(row[3] - row[2]) / 1e3:.1f} copy-out {(row[4] - row[3]) / 1e3:.1f}",
                          file=sys.stderr)
        pr = [a.elapsed_time(b) * 1e3 for a, b in probe[-3 * len(st):]]
        print(f"[trace r{rank}] tiny kernel on the metadata stream: "
              + " ".join(f"{x:.1f}" for x in pr) + " us", file=sys.stderr)
        mm = meta_marks[-5 * 3 * len(st):]
        for i in range(0, len(mm), 5):
            g = [mm[i].elapsed_time(mm[i + j]) for j in range(1, 5)]
            print(f"[trace r{rank}] meta allgather {g[0]:.3f} balance {g[1] - g[0]:.3f} "
                  f"nodewise {g[2] - g[1]:.3f} layout {g[3] - g[2]:.3f} ms", file=sys.stderr)
        for it, name, m0, m1, d0, e0, e1 in trace[-3 * len(st):]:
            print(f"[trace r{rank}] step {it} {name:6s} meta {t0.elapsed_time(m0):8.3f}-"
                  f"{t0.elapsed_time(m1):8.3f}  data ready {t0.elapsed_time(d0):8.3f} "
                  f"move {t0.elapsed_time(e0):8.3f}-{t0.elapsed_time(e1):8.3f} ms",
                  file=sys.stderr)
    ms = max_over_ranks(t0.elapsed_time(t1))
    tokens = sum(int(s["L"].sum()) for s in st)
    seqs = sum(s["n"] for s in st)
    value = tokens * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (the row movement; one dispatch per phase)
    disp_ms = sum(e0.elapsed_time(e1) for _, e0, e1 in disp_events)
    moved = sum(s["moved_rows"] for s in st) * R * args.steps  # rows written once, read once
    hbm_bytes = 2 * moved
    if P > 1 and args.exchange in ("nccl", "nccl-sync"):  # staging: pack to send, recv to out
        hbm_bytes += 2 * sum(s["send_rows"] + s["recv_rows"] for s in st) * R * args.steps
    peak, peak_kind = peaks()
    achieved = hbm_bytes / (disp_ms / 1e3) / 1e9 if disp_ms > 0 else None
    traffic = None  # DRAM bytes per launch from the committed ncu --set full capture
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)["per_launch"]
        traffic = sum(x["dram_read_plus_write"] for x in tj) / len(tj)
        traffic_alg = sum(x["algorithmic_bytes"] for x in tj) / len(tj)
    except Exception:
        traffic_alg = None

    # steps the e2e host loop keeps in flight beyond the one it waits for
    E2E_DEPTH = int(os.environ.get("ORCH_E2E_DEPTH", "1"))
    # end-to-end through the C-ABI with host buffers: each step copies its
    # metadata from pinned host memory and reads back its assignment vectors
    # and summaries (its own set of pinned buffers). Steps stay in flight as in
    # a training loop's input pipeline: the host waits for step i's results
    # (on the host) after issuing step i + E2E_DEPTH, so the next steps' copies
    # and metadata overlap step i's rows; --e2e-sync completes every step
    # before the next one starts.
    if comm_meta is None:
        h2d = sum(s["h_glen"].numel() * 8 + s["h_gorg"].numel() * 4 for s in st)
    else:
        h2d = sum(s["h_pos"].numel() * 8 + s["h_len"].numel() * 8 + s["h_org"].numel() * 4
                  for s in st)
    d2h = sum(s["n"] * 8 + 128 for s in st)
    host_out = [[(torch.empty(s["n"], dtype=torch.int32).pin_memory(),
                  torch.empty(s["n"], dtype=torch.int32).pin_memory(),
                  torch.empty(128, dtype=torch.uint8).pin_memory()) for s in st]
                for _ in range(E2E_DEPTH + 1)]  # one set per step in flight
    in_flight = []
    e2e_count = [0]

    def e2e_step(sync):
        b = step(h2d=True)
        hb = e2e_count[0] % len(host_out)
        e2e_count[0] += 1
        done = []
        for s, (hi, hs, hsum) in zip(st, host_out[hb]):
            with torch.cuda.stream(s["ms"]):
                bal = s["buf"][b]["bal"]
                hi.copy_(bal.dest_inst[:s["n"]], non_blocking=True)
                hs.copy_(bal.dest_slot[:s["n"]], non_blocking=True)
                hsum[:bal.summary_raw.numel()].copy_(bal.summary_raw, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s["ms"])
                done.append(ev)
        ev = torch.cuda.Event()
        ev.record(data_stream)
        done.append(ev)
        in_flight.append(done)
        # step i - E2E_DEPTH's results are on the host (step i's when synchronous)
        while len(in_flight) > (0 if sync else E2E_DEPTH):
            for ev in in_flight.pop(0):
                ev.synchronize()

    def e2e_drain():
        while in_flight:
            for ev in in_flight.pop(0):
                ev.synchronize()

    def e2e_run(sync):
        for _ in range(max(args.warmup, 10)):
            e2e_step(sync)
        e2e_drain()
        # the timed host loop runs without the cyclic garbage collector, so a
        # collection pass cannot land inside the K steps; the collection runs
        # before the barrier, so the ranks enter the loop together (a collection
        # after it skewed their starts by a few ms, which the first step paid)
        gc.collect()
        gc.disable()
        barrier()
        w0 = time.perf_counter()
        marks = []
        for _ in range(args.steps):
            e2e_step(sync)
            marks.append(time.perf_counter())
        e2e_drain()
        barrier()
        secs = max_over_ranks(time.perf_counter() - w0)
        gc.enable()
        if os.environ.get("ORCH_BENCH_E2E_TRACE"):  # host time per step (diagnostics)
            gaps = np.diff([w0] + marks) * 1e3
            print(f"[e2e r{rank} sync={sync}] ms/step " + " ".join(f"{g:.2f}" for g in gaps),
                  file=sys.stderr)
        return secs

    # both loops are measured; the line's e2e is the pipelined one unless
    # --e2e-sync, and carries the other as e2e.sync_value / e2e.pipelined_value
    e2e_sync_s = e2e_run(True)
    e2e_pipe_s = e2e_run(False)
    e2e_s = e2e_sync_s if args.e2e_sync else e2e_pipe_s
    if os.environ.get("ORCH_BENCH_TRACE"):  # the metadata sub-steps of the last e2e steps
        mm = meta_marks[-5 * 2 * len(st):]
        for i in range(0, len(mm), 5):
            g = [mm[i].elapsed_time(mm[i + j]) for j in range(1, 5)]
            print(f"[trace r{rank}] e2e meta allgather {g[0]:.3f} balance {g[1] - g[0]:.3f} "
                  f"nodewise {g[2] - g[1]:.3f} layout {g[3] - g[2]:.3f} ms", file=sys.stderr)

    # load balance (stats_of max/mean, orchestrator.cpp:91-102)
    imb = {}
    for s in st:
        sm = s["buf"][0]["bal"].summary()
        imb[s["name"]] = {"pre": round(sm.pre_ratio, 6), "post": round(sm.post_ratio, 6)}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "warmup_extra": extra,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": CFG["workload"], "global_batch": D_INST * CFG["per"],
                   "dp_instances": D_INST, "instances_per_gpu": c, "row_bytes": R,
                   "tokens_per_step": tokens, "seqs_per_step": seqs,
                   "l2": f"row buffers {tokens * R / 1e9:.1f} GB >> 126 MB L2 (no flush needed)"},
        "seqs_per_s": seqs * args.steps / (ms / 1e3),
        "load_imbalance_max_over_mean": imb,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic,
                     "traffic_algorithmic_per_launch": traffic_alg,
                     "kernel": "k_move_tma<kLocal> (orch_dispatch)", "peak_kind": peak_kind,
                     "share_of_step": disp_ms / (t0.elapsed_time(t1) or 1.0)},
        "e2e": {"value": tokens * args.steps / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": ("C-ABI with host metadata buffers, one synchronous step at a time; "
                         if args.e2e_sync else
                         f"C-ABI with host metadata buffers, {E2E_DEPTH + 1} steps in flight "
                         f"(the host waits for step i's results after issuing step "
                         f"i+{E2E_DEPTH}); ") +
                        "token rows are device-resident activations (encoder/embedding "
                        "outputs)",
                "sync_value": tokens * args.steps / e2e_sync_s,
                "pipelined_value": tokens * args.steps / e2e_pipe_s},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if P > 1:
        # NVLink bottleneck: the busiest direction of the busiest rank (egress =
        # rows this rank sends off-rank, ingress = rows it receives)
        egress = max_over_ranks(sum(s["send_rows"] for s in st) * R)
        ingress = max_over_ranks(sum(s["recv_rows"] for s in st) * R)
        a2a_bytes = max(egress, ingress)
        disp_ms = max_over_ranks(disp_ms)
        busbw = a2a_bytes * args.steps / (disp_ms / 1e3) / 1e9
        line["exchange"] = args.exchange
        line["gather"] = args.gather
        line["windows"] = window_kind[0] if (win is not None or any(gwins)) else None
        line["nodewise_hosting"] = bool(args.nodewise)
        nv = nvlink_peaks(world)
        line["a2a"] = {"bytes_per_rank_per_step": a2a_bytes, "max_egress_bytes": egress,
                       "max_ingress_bytes": ingress, "busbw_gbs_rank": busbw,
                       "nvlink_spec_gbs": 900.0, "nvlink_measured": nv,
                       "frac_of_kernel_push": busbw / nv["kernel_push"],
                       "frac_of_nccl_ceiling": busbw / nv["nccl"],
                       "note": "max over ranks of max(off-rank bytes sent, received) / max over "
                               "ranks of the device time of the dispatch calls; ceilings measured "
                               "by scripts/p2pbench.cu (profiles/nvlink_peaks.json)"}
        # at N > 1 the row movement is NVLink-bound: roofline against the best
        # measured per-direction copy (the copy engines, all-to-all pattern)
        hbm_view = line["roofline"]
        line["roofline"] = {"bound": "nvlink", "achieved": busbw, "peak": nv["copy_engine"],
                            "unit": "GB/s", "frac": busbw / nv["copy_engine"], "traffic": None,
                            "kernel": {"put": "k_move_tma<kPut> (orch_put)",
                                       "put-nccl": "k_move_tma<kPut> (orch_put) into NCCL "
                                                   "symmetric-memory windows "
                                                   "(orch_window_create_nccl)",
                                       "nccl": "pack + ncclSend/ncclRecv per peer + unpack, host "
                                               "counts from the metadata stream "
                                               "(orch_dispatch_nccl)",
                                       "nccl-direct": "ncclSend/ncclRecv per item run "
                                                      "(orch_dispatch_nccl)",
                                       "nccl-sync": "pack + ncclSend/ncclRecv + unpack, counts "
                                                    "read on the data stream (orch_dispatch)"
                                       }[args.exchange],
                            "peak_kind": "measured copy-engine peer copy, all-to-all at "
                                         f"{nv['measured_at_gpus']} GPUs (profiles/nvlink_peaks.json)",
                            "share_of_step": hbm_view["share_of_step"],
                            "hbm_view": {k: hbm_view[k] for k in ("achieved", "peak", "frac")}}
    host_bytes = 2 * tokens * R
    if rank == 0 and world == 1 and not args.no_cpu_baseline and host_bytes <= 16e9:
        times, ctoks, kind, nthreads = cpu_arm(phases, 1, 1)
        line["cpu_baseline"] = {"value": ctoks / times[0], "unit": "tokens/s", "cores": nthreads,
                                "kind": kind,
                                "sample": f"one full {CFG['name']} step after one warm-up step: "
                                          f"reference balance() per phase + {nthreads}-thread "
                                          "host memcpy dispatch"}
    elif rank == 0 and world == 1:
        line["cpu_baseline"] = {"value": None, "note": f"skipped: host row buffers of "
                                                       f"{host_bytes / 1e9:.0f} GB"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if win is not None:
        for s in st:
            s["rout"] = None
        wview = None
        win.close()
    for gwin in gwins:
        if gwin is not None:
            gwin.close()
    for h in reg:
        comm_data.deregister(h)
    if comm_meta is not None:
        comm_meta.close()
        comm_data.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS),
                    help="workload: C2 (default, the driver's line) or the C3 / C5 evidence lines")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nodewise", dest="nodewise", action="store_false",
                    help="N>1: skip the GPU-wise hosting of destination batches")
    ap.add_argument("--gather", default="put", choices=["put", "nccl"],
                    help="N>1 lengths all-gather: peer-memory kernel (default) or ncclAllGather")
    ap.add_argument("--barrier", default="window", choices=["window", "nccl", "none"],
                    help="N>1 put: the per-step barrier through the window's peer memory "
                         "(default), a 1-int ncclAllReduce, or none (diagnostics only)")
    ap.add_argument("--exchange", default="put-nccl",
                    choices=["put", "put-nccl", "nccl", "nccl-direct", "nccl-sync"],
                    help="N>1: fused pack+put over NVLink into NCCL symmetric-memory windows "
                         "(put-nccl, default) or CUDA IPC windows (put); NCCL: pack, one send/recv "
                         "per peer, unpack (nccl), one send/recv per item run (nccl-direct), or "
                         "the round-1 path that reads the counts on the data stream (nccl-sync)")
    ap.add_argument("--nccl-register", action="store_true",
                    help="--exchange nccl*: ncclCommRegister the row buffers")
    ap.add_argument("--e2e-sync", action="store_true",
                    help="e2e: complete every step before the next (default: two in flight)")
    args = ap.parse_args()
    CFG.clear()
    CFG.update(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
