"""Parity at the bench's own sizes on one GPU (the calls bench.py times).

* C2 (BASELINE configs[1]): both phases of the step through
  orch_balance_layout1 + orch_dispatch, 530,243 token rows of 8 KiB
  (4.3 GB), checked row by row on the device.
* C5 (configs[4]): the long-context phase, 16 KiB rows, ~21 GB, so byte
  offsets pass 4 GiB and the buffers 2^34 bytes.

Assignments, slots and offsets are compared with the oracle; the expected
row placement is the oracle's layout (apply() on rows, core.cpp:120-161).
Every input row carries an (input row, item, row-in-item) tag; the rest is
random, so any misplaced or missing byte fails the device compare.
"""
import numpy as np
import pytest
import torch

from rowcheck import fill_tagged, first_mismatch, rows_equal, source_rows

pytestmark = pytest.mark.gpu


def tags_for_input(length, origin, rank_src_off, rows):
    """item position and row-within-item of every row of a one-rank input buffer."""
    length = np.asarray(length, np.int64)
    item = np.zeros(rows, np.int64)
    within = np.zeros(rows, np.int64)
    for_items = np.repeat(np.arange(len(length)), length)
    start = np.repeat(np.asarray(rank_src_off, np.int64), length)
    w = np.arange(len(for_items), dtype=np.int64) - np.repeat(np.cumsum(length) - length, length)
    item[start + w] = for_items
    within[start + w] = w
    return torch.from_numpy(item).cuda(), torch.from_numpy(within).cuda()


def one_rank_phase(ctx, oracle, kind, d, length, origin, R, lam=0.0, v=0, seed=0):
    length = np.ascontiguousarray(length, np.int64)
    origin = np.ascontiguousarray(origin, np.int32)
    n = len(length)
    o = oracle.balance(kind, d, length, origin, lam=lam, v=v)
    e = oracle.layout(d, 1, length, origin, o.dest_inst, o.dest_slot)
    L = torch.from_numpy(length).cuda()
    O = torch.from_numpy(origin).cuda()
    bal, lay = ctx.balance_layout1(kind, d, L, O, lam=lam, v=v)
    rows = int(length.sum())
    rin = torch.empty(rows * R, dtype=torch.uint8, device="cuda")
    item, within = tags_for_input(length, origin, e["rank_src_off"], rows)
    fill_tagged(rin, R, item, within, seed=seed)
    del item, within
    rout = torch.empty_like(rin)
    rout.fill_(0xEE)
    ctx.dispatch(d, L, O, bal, lay, R, rin, rout)
    torch.cuda.synchronize()
    assert int(lay.status.item()) == 0
    np.testing.assert_array_equal(bal.dest_inst[:n].cpu().numpy(), o.dest_inst)
    np.testing.assert_array_equal(bal.dest_slot[:n].cpu().numpy(), o.dest_slot)
    assert bal.summary().objective == o.objective
    np.testing.assert_array_equal(lay.rank_src_off[:n].cpu().numpy(), e["rank_src_off"])
    np.testing.assert_array_equal(lay.rank_dst_off[:n].cpu().numpy(), e["rank_dst_off"])
    idx = source_rows(length, origin, o.dest_inst, e["rank_src_off"], e["rank_dst_off"], d, 1,
                      [0])[0]
    assert len(idx) == rows
    assert rows_equal(rout, rin, idx, R), first_mismatch(rout, rin, idx, R)
    return rows


def test_c2_full_step_bytes(ctx, oracle):
    from paper_2503_23830_b200 import workload
    d, R = 8, 8192
    b = workload.make_batch(2, d, 64, 2)
    lv, ov, _ = b.phase_items("vision")
    ll, ol = b.llm_items()
    rows = one_rank_phase(ctx, oracle, 0, d, lv, ov, R, seed=1)
    rows += one_rank_phase(ctx, oracle, 0, d, ll, ol, R, seed=2)
    assert rows == 530243  # the bench's tokens per step


def test_c5_phase_beyond_4gib(ctx, oracle):
    d, R = 8, 16384
    rng = np.random.default_rng(5)  # bench.py build_inputs() for C5
    length = rng.integers(8192, 32769, d * 8).astype(np.int64)
    origin = (np.arange(d * 8) % d).astype(np.int32)
    assert int(length.sum()) * R > (1 << 34)
    one_rank_phase(ctx, oracle, 2, d, length, origin, R, lam=1.0 / (6 * 8192), v=2048, seed=5)
    # the same rows under the greedy policy (the C5 GreedyUnpadded variant)
    one_rank_phase(ctx, oracle, 0, d, length, origin, R, seed=6)
