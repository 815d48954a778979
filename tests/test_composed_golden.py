"""Composed delivery pinned to the reference
orchestrator: tests/golden/ref_composed.npz holds, for C2 / C3 / a node-wise
hosted C3, the end state of run_iteration's composed delivery
(orchestrator.cpp:390-418) -- every example's LLM destination and, for every
part, the instance and position of the backbone's assembled input
(tests/golden/make_composed_golden.py, the unmodified reference).

The CPU test pins the oracle's restatement (orc_backbone_targets =
backbone_mapping_for, :367-388); the GPU test runs the device path --
balances, orch_nodewise, orch_backbone_targets and the composed row exchange
of tagged encoder outputs -- and decodes the delivered rows."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = np.load(os.path.join(HERE, "golden", "ref_composed.npz"))
CASES = [tuple(int(x) for x in row) for row in FIX["cases"]]
MODALITIES = (0, 1, 2)  # text (passthrough), vision, audio


def batch_of(case):
    from paper_2503_23830_b200 import workload
    mix, d, c, per, seed, nw = case
    return workload.make_batch(mix, d, per, seed)


def interleave_pos(b):
    return np.concatenate([np.arange(b.part_offset[e + 1] - b.part_offset[e])
                           for e in range(len(b.origin))]).astype(np.int32)


def expected(k, b, code):
    """Per instance: the parts of one universe in the reference's assembled order."""
    ai, ap = FIX[f"{k}_asm_inst"], FIX[f"{k}_asm_pos"]
    d = b.d
    out = []
    for i in range(d):
        sel = np.nonzero((ai == i) & (b.modality == code))[0]
        out.append(sel[np.argsort(ap[sel])])
    return out


def delivered(d, parts, ti, ts):
    """Per instance: parts in the order of their destination slots."""
    out = []
    for i in range(d):
        sel = np.nonzero(ti == i)[0]
        out.append(parts[sel[np.argsort(ts[sel])]])
    return out


@pytest.mark.parametrize("k", range(len(CASES)))
def test_oracle_composed_delivery_matches_reference(oracle, k):
    mix, d, c, per, seed, nw = CASES[k]
    b = batch_of(CASES[k])
    ll, ol = b.llm_items()
    o = oracle.balance(0, d, ll, ol)
    di, ds = o.dest_inst, o.dest_slot
    if nw:
        h = oracle.solve_hosting(d, c, oracle.volume_matrix(d, ll, ol, di))
        di = h["batch_to_instance"][di]
    np.testing.assert_array_equal(di, FIX[f"{k}_llm_dest_inst"])
    np.testing.assert_array_equal(ds, FIX[f"{k}_llm_dest_slot"])
    ip = interleave_pos(b)
    for code in MODALITIES:
        parts = np.nonzero(b.modality == code)[0].astype(np.int32)
        if len(parts) == 0:
            continue
        ti, ts = oracle.backbone_targets(d, di, ds, b.part_offset, ip, parts)
        got, want = delivered(d, parts, ti, ts), expected(k, b, code)
        for i in range(d):
            np.testing.assert_array_equal(got[i], want[i], err_msg=f"case {k} modality {code} inst {i}")


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)))
def test_gpu_composed_delivery_matches_reference(ctx, k):
    """Device path end to end: encoder balance (vision GreedyUnpadded, audio
    BinaryPadded) on metadata lengths, LLM balance (+ orch_nodewise when the case
    hosts node-wise), orch_backbone_targets per universe, then the encoder
    outputs (encoded lengths, rows tagged with their part) take ONE exchange from
    the encoder's destination batches to the backbone slots (orch_rearrange +
    orch_layout + orch_dispatch). The delivered buffers are decoded row by row."""
    import torch
    mix, d, c, per, seed, nw = CASES[k]
    b = batch_of(CASES[k])
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).cuda()  # noqa: E731
    ll, ol = b.llm_items()
    Ll, Ol = dev(ll, np.int64), dev(ol, np.int32)
    llm = ctx.balance(0, d, Ll, Ol)
    if nw:
        keep = ctx.nodewise(d, c, Ll, Ol, llm)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(llm.dest_inst[:len(ll)].cpu().numpy(), FIX[f"{k}_llm_dest_inst"])
    np.testing.assert_array_equal(llm.dest_slot[:len(ll)].cpu().numpy(), FIX[f"{k}_llm_dest_slot"])
    ip = dev(interleave_pos(b), np.int32)
    po = dev(b.part_offset, np.int32)
    R = 16
    for code, kind in ((0, None), (1, 0), (2, 1)):
        parts = np.nonzero(b.modality == code)[0].astype(np.int32)
        if len(parts) == 0:
            continue
        n = len(parts)
        ti, ts = ctx.backbone_targets(d, llm, po, ip, dev(parts, np.int32))
        origin = b.origin[np.searchsorted(b.part_offset, parts, side="right") - 1].astype(np.int32)
        enc = b.encoded[parts].astype(np.int64)
        if kind is None:  # passthrough: delivered straight from the origin batches
            src_inst = dev(origin, np.int32)
            src_slot = None
        else:  # the encoder phase's balance on metadata lengths places the outputs
            eb = ctx.balance(kind, d, dev(b.meta[parts], np.int64), dev(origin, np.int32))
            src_inst, src_slot = eb.dest_inst[:n], eb.dest_slot[:n]
        if src_slot is None:
            slot = np.zeros(n, np.int32)
            nxt = np.zeros(d, np.int64)
            for i in range(n):
                slot[i] = nxt[origin[i]]
                nxt[origin[i]] += 1
            src_slot = dev(slot, np.int32)
        L = dev(enc, np.int64)
        re = ctx.rearrange(d, L, src_inst, src_slot, ti, ts)
        lay = ctx.layout(d, 1, L, src_inst, re)
        torch.cuda.synchronize()
        assert re.summary().error == 0
        rows = int(enc.sum())
        # rows of the encoder's output batches, each tagged with its part id
        rso = lay.rank_src_off[:n].cpu().numpy()
        tag = np.zeros(rows, np.int64)
        tag[np.repeat(rso, enc) + (np.arange(rows) - np.repeat(np.cumsum(enc) - enc, enc))] = \
            np.repeat(parts, enc)
        rin = torch.zeros(rows, R // 8, dtype=torch.int64, device="cuda")
        rin[:, 0] = dev(tag, np.int64)
        rin[:, 1] = torch.arange(rows, device="cuda")
        rout = torch.zeros_like(rin)
        ctx.dispatch(d, L, src_inst, re, lay, R, rin.view(torch.uint8).view(-1),
                     rout.view(torch.uint8).view(-1))
        torch.cuda.synchronize()
        assert int(lay.status.item()) == 0
        out_tag = rout[:, 0].cpu().numpy()
        base = np.concatenate([[0], np.cumsum(np.bincount(ti.cpu().numpy(), weights=enc,
                                                          minlength=d))]).astype(np.int64)
        want = expected(k, b, code)
        for i in range(d):
            seq = out_tag[base[i]:base[i + 1]]
            firsts = seq[np.r_[True, seq[1:] != seq[:-1]]] if len(seq) else seq
            np.testing.assert_array_equal(firsts, want[i], err_msg=f"case {k} modality {code} inst {i}")
