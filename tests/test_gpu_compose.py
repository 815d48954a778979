"""Composed delivery on the GPU: orch_rearrange,
orch_backbone_targets and the one-exchange delivery of encoder outputs,
against the oracle and against the reference's two-exchange path
(verify.cpp:219-270 check_composition: apply(compose(B, E), encoded) ==
apply(B, apply(inverse(E), encoded)), here on token rows)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a, dt)).cuda()


def random_re(rng, d, origin):
    """verify.cpp:233-247: shuffle all source slots into dense destinations."""
    n = len(origin)
    src_slot = np.zeros(n, np.int32)
    nxt = np.zeros(d, np.int64)
    for i in range(n):
        src_slot[i] = nxt[origin[i]]
        nxt[origin[i]] += 1
    perm = rng.permutation(n)
    dst_inst = origin[perm].astype(np.int32)  # destinations: a shuffle of the source slots
    dst_slot = np.zeros(n, np.int32)
    nxt = np.zeros(d, np.int64)
    for i in range(n):
        dst_slot[i] = nxt[dst_inst[i]]
        nxt[dst_inst[i]] += 1
    return src_slot, dst_inst, dst_slot


def dispatch_rows(ctx, d, L, src_inst, src_slot, dst_inst, dst_slot, rows_in, R):
    Lt = dev(L, np.int64)
    re = ctx.rearrange(d, Lt, dev(src_inst, np.int32), dev(src_slot, np.int32),
                       dev(dst_inst, np.int32), dev(dst_slot, np.int32))
    torch.cuda.synchronize()
    assert re.summary().error == 0
    si = dev(src_inst, np.int32)
    lay = ctx.layout(d, 1, Lt, si, re)
    out = torch.zeros_like(rows_in)
    ctx.dispatch(d, Lt, si, re, lay, R, rows_in, out)
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 0
    return out, re


def test_rearrange_offsets_match_oracle(ctx, oracle):
    rng = np.random.default_rng(8)
    for _ in range(60):
        d = int(rng.integers(1, 9))
        n = int(rng.integers(1, 300))
        L = rng.integers(1, 50, n).astype(np.int64)
        O = rng.integers(0, d, n).astype(np.int32)
        ss, di, ds = random_re(rng, d, O)
        so, do = oracle.rearrange_offsets(d, L, O, ss, di, ds)
        re = ctx.rearrange(d, dev(L, np.int64), dev(O, np.int32), dev(ss, np.int32),
                           dev(di, np.int32), dev(ds, np.int32))
        torch.cuda.synchronize()
        assert re.summary().error == 0
        np.testing.assert_array_equal(re.src_off[:n].cpu().numpy(), so)
        np.testing.assert_array_equal(re.dst_off[:n].cpu().numpy(), do)
        np.testing.assert_array_equal(re.bin_count.cpu().numpy(), np.bincount(di, minlength=d))


def test_rearrange_rejects_invalid(ctx, oracle):
    from oracle import OracleError
    L = dev(np.array([3, 4, 5], np.int64), np.int64)
    bad = [
        ([0, 0, 1], [0, 1, 0], [0, 0, 1], [0, 0, 0]),  # two items on one destination slot
        ([0, 0, 1], [0, 1, 0], [0, 0, 1], [0, 2, 0]),  # destination slots not dense
        ([0, 0, 1], [0, 0, 0], [0, 0, 1], [0, 1, 0]),  # a source slot twice
        ([0, 0, 1], [0, 1, 0], [0, 0, 5], [0, 1, 0]),  # instance outside [0, d)
    ]
    for si, ss, di, ds in bad:
        re = ctx.rearrange(2, L, dev(si, np.int32), dev(ss, np.int32), dev(di, np.int32),
                           dev(ds, np.int32))
        torch.cuda.synchronize()
        assert re.summary().error == 1
        with pytest.raises(OracleError):
            oracle.rearrange_offsets(2, [3, 4, 5], si, ss, di, ds)


def test_composition_on_rows(ctx, oracle):
    """check_composition on token rows: one composed exchange == inverse then backbone."""
    rng = np.random.default_rng(3)
    R = 32
    for trial in range(20):
        d = 2 + int(rng.integers(0, 4))
        n = 1 + int(rng.integers(0, 60))
        L = rng.integers(1, 12, n).astype(np.int64)
        O = rng.integers(0, d, n).astype(np.int32)
        e_ss, e_di, e_ds = random_re(rng, d, O)  # encoder rearrangement
        b_ss, b_di, b_ds = random_re(rng, d, O)  # backbone mapping (from origin slots)
        assert np.array_equal(e_ss, b_ss)
        so, _ = oracle.rearrange_offsets(d, L, O, e_ss, e_di, e_ds)
        base = np.zeros(d + 1, np.int64)
        np.add.at(base, O + 1, L)
        base = np.cumsum(base)
        rows = int(L.sum())
        h = np.zeros(rows * R, np.uint8)
        oracle.fill_rows(L, np.arange(n, dtype=np.int64) + 100, base[O] + so, R, h)
        batches = dev(h, np.uint8)
        encoded, _ = dispatch_rows(ctx, d, L, O, e_ss, e_di, e_ds, batches, R)
        # composed: from the encoder's destination straight to the backbone slot
        composed, _ = dispatch_rows(ctx, d, L, e_di, e_ds, b_di, b_ds, encoded, R)
        # reference path: reset to origin (inverse), then the backbone mapping
        reset, _ = dispatch_rows(ctx, d, L, e_di, e_ds, O, e_ss, encoded, R)
        assert torch.equal(reset, batches)  # inverse round trip
        two_step, _ = dispatch_rows(ctx, d, L, O, b_ss, b_di, b_ds, reset, R)
        assert torch.equal(composed, two_step), trial


def test_backbone_targets_and_delivery(ctx, oracle):
    """C3-like iteration: vision encoder balance, LLM balance, then each vision
    part delivered from the encoder's batches straight to its backbone slot."""
    from paper_2503_23830_b200 import workload
    d = 16
    b = workload.make_batch(3, d, 16, 11)
    E = len(b.origin)
    interleave_pos = np.concatenate([np.arange(b.part_offset[e + 1] - b.part_offset[e])
                                     for e in range(E)]).astype(np.int32)
    ll, ol = b.llm_items()
    llm = ctx.balance(0, d, dev(ll, np.int64), dev(ol, np.int32))
    ref_llm = oracle.balance(0, d, ll, ol)
    lv, ov, vparts = b.phase_items("vision")
    vis = ctx.balance(0, d, dev(lv, np.int64), dev(ov, np.int32))
    ref_vis = oracle.balance(0, d, lv, ov)
    ti, ts = ctx.backbone_targets(d, llm, dev(b.part_offset, np.int32),
                                  dev(interleave_pos, np.int32), dev(vparts, np.int32))
    torch.cuda.synchronize()
    ei, es = oracle.backbone_targets(d, ref_llm.dest_inst, ref_llm.dest_slot, b.part_offset,
                                     interleave_pos, vparts)
    np.testing.assert_array_equal(ti.cpu().numpy(), ei)
    np.testing.assert_array_equal(ts.cpu().numpy(), es)
    # rows: encoder output batches -> one composed exchange -> backbone layout
    R = 16
    enc_src, enc_dst = oracle.rearrange_offsets(d, lv, ov, ref_vis.src_slot, ref_vis.dest_inst,
                                                ref_vis.dest_slot)
    n = len(lv)
    base = np.zeros(d + 1, np.int64)
    np.add.at(base, ref_vis.dest_inst + 1, lv)
    base = np.cumsum(base)
    h = np.zeros(int(lv.sum()) * R, np.uint8)
    oracle.fill_rows(lv, vparts.astype(np.int64), base[ref_vis.dest_inst] + enc_dst, R, h)
    final, re = dispatch_rows(ctx, d, lv, ref_vis.dest_inst, ref_vis.dest_slot, ei, es,
                              dev(h, np.uint8), R)
    # expected: per backbone instance, vision parts in target-slot order
    _, tgt_off = oracle.rearrange_offsets(d, lv, ref_vis.dest_inst, ref_vis.dest_slot, ei, es)
    tb = np.zeros(d + 1, np.int64)
    np.add.at(tb, ei + 1, lv)
    tb = np.cumsum(tb)
    expect = np.zeros_like(h)
    oracle.fill_rows(lv, vparts.astype(np.int64), tb[ei] + tgt_off, R, expect)
    assert torch.equal(final.cpu(), torch.from_numpy(expect))
