"""Device-side row tagging and checking for the bench-scale parity tests.

The expected placement of every token row comes from the oracle's layout
(orc_layout, the restatement of apply() on rows: core.cpp:120-161 with
batches_from_items order, core.cpp:183-199). Buffers of many GB are filled
and compared on the GPU with torch ops (test infrastructure only; the rows
themselves are moved by the library under test):

  * every input row carries a tag in its first 16 bytes: (global input row,
    item input position << 32 | row within the item), the rest is random;
  * rank q's expected output is index_select(all inputs, source row of every
    output row), compared with torch.equal in bounded chunks.
"""
from __future__ import annotations

import numpy as np
import torch

CHUNK_BYTES = 1 << 30


def source_rows(length, origin, dest_inst, rank_src_off, rank_dst_off, c, P, in_base):
    """Per destination rank q: int64 array, for every row of q's output, the
    global input row (in_base[origin rank] + row in that rank's input)."""
    length = np.asarray(length, np.int64)
    origin = np.asarray(origin, np.int64)
    dest = np.asarray(dest_inst, np.int64)
    rs = np.asarray(rank_src_off, np.int64)
    rd = np.asarray(rank_dst_off, np.int64)
    out = []
    for q in range(P):
        sel = np.nonzero(dest // c == q)[0]
        if len(sel) == 0:
            out.append(np.zeros(0, np.int64))
            continue
        L = length[sel]
        tot = int(L.sum())
        item = np.repeat(np.arange(len(sel)), L)
        within = np.arange(tot, dtype=np.int64) - np.repeat(np.cumsum(L) - L, L)
        dst_row = rd[sel][item] + within
        src_row = np.asarray(in_base, np.int64)[origin[sel] // c][item] + rs[sel][item] + within
        idx = np.empty(tot, np.int64)
        idx[dst_row - dst_row.min()] = src_row  # dest rows of rank q are 0..tot-1
        assert dst_row.min() == 0 and dst_row.max() == tot - 1
        out.append(idx)
    return out


def fill_tagged(buf_u8: torch.Tensor, R: int, item_of_row: torch.Tensor | None = None,
                row_in_item: torch.Tensor | None = None, seed: int = 0):
    """Random rows with a 16-byte tag at the start of each row (see module doc)."""
    rows = buf_u8.numel() // R
    g = torch.Generator(device=buf_u8.device)
    g.manual_seed(seed)
    w = buf_u8.view(torch.int64).view(rows, R // 8)
    step = max(1, CHUNK_BYTES // R)
    for a in range(0, rows, step):
        b = min(rows, a + step)
        w[a:b].random_(generator=g)
        w[a:b, 0] = torch.arange(a, b, device=buf_u8.device, dtype=torch.int64)
        if item_of_row is not None:
            w[a:b, 1] = (item_of_row[a:b].to(torch.int64) << 32) | row_in_item[a:b].to(torch.int64)


def rows_equal(out_u8: torch.Tensor, all_in_u8: torch.Tensor, idx: np.ndarray, R: int) -> bool:
    """out row k == input row idx[k] for every k (compared on the device)."""
    rows = len(idx)
    if rows == 0:
        return True
    src = all_in_u8.view(torch.int64).view(-1, R // 8)
    dst = out_u8[:rows * R].view(torch.int64).view(rows, R // 8)
    dev_idx = torch.from_numpy(idx).to(out_u8.device)
    step = max(1, CHUNK_BYTES // R)
    for a in range(0, rows, step):
        b = min(rows, a + step)
        if not torch.equal(dst[a:b], src.index_select(0, dev_idx[a:b])):
            return False
    return True


def first_mismatch(out_u8, all_in_u8, idx, R):
    """Diagnostics: (output row, expected tag, found tag) of the first bad row."""
    src = all_in_u8.view(torch.int64).view(-1, R // 8)
    dst = out_u8[:len(idx) * R].view(torch.int64).view(len(idx), R // 8)
    dev_idx = torch.from_numpy(idx).to(out_u8.device)
    bad = (dst != src.index_select(0, dev_idx)).any(dim=1).nonzero()
    if len(bad) == 0:
        return None
    k = int(bad[0])
    return k, src[int(idx[k]), :2].tolist(), dst[k, :2].tolist()
