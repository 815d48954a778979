"""GPU parity of the balance pipeline against the oracle (bit-exact).

Every comparison is exact: assignment vectors, slots, token offsets, per-batch
counts/lengths/tokens, per-batch costs and the objective compared as IEEE
bits, the identity fallback flag, the CSR outputs. Cases follow the
reference's own test generators (proj/tests/helpers.hpp:15-60,
test_balancers.cpp) plus config-shaped and adversarial inputs.
"""
import numpy as np
import pytest
import torch

from conftest import random_instance

pytestmark = pytest.mark.gpu

KINDS = [0, 1, 2, 3]


def gpu_balance(ctx, kind, d, length, origin, lam=0.0, v=0, identity_only=False):
    L = torch.from_numpy(np.ascontiguousarray(length, np.int64)).cuda()
    O = torch.from_numpy(np.ascontiguousarray(origin, np.int32)).cuda()
    b = ctx.balance(kind, d, L, O, lam=lam, v=v, identity_only=identity_only)
    torch.cuda.synchronize()
    return b


def check_same(b, o, n, d):
    s = b.summary()
    assert s.error == 0, s.error
    np.testing.assert_array_equal(b.dest_inst[:n].cpu().numpy(), o.dest_inst)
    np.testing.assert_array_equal(b.dest_slot[:n].cpu().numpy(), o.dest_slot)
    np.testing.assert_array_equal(b.src_slot[:n].cpu().numpy(), o.src_slot)
    np.testing.assert_array_equal(b.src_off[:n].cpu().numpy(), o.src_off)
    np.testing.assert_array_equal(b.dst_off[:n].cpu().numpy(), o.dst_off)
    np.testing.assert_array_equal(b.bin_count.cpu().numpy(), o.bin_count)
    np.testing.assert_array_equal(b.bin_len.cpu().numpy(), o.bin_len)
    np.testing.assert_array_equal(b.bin_tokens.cpu().numpy(), o.bin_tokens)
    assert b.bin_cost.cpu().numpy().tobytes() == o.bin_cost.tobytes()
    assert np.float64(s.objective).tobytes() == np.float64(o.objective).tobytes()
    assert s.used_identity == o.used_identity
    # CSR consistency: members in (dest, slot) order
    off = b.bin_offset.cpu().numpy()
    mem = b.bin_member[:n].cpu().numpy()
    assert off[0] == 0 and off[-1] == n
    np.testing.assert_array_equal(np.diff(off), o.bin_count)
    if n:
        di, ds = o.dest_inst[mem], o.dest_slot[mem]
        np.testing.assert_array_equal(di, np.repeat(np.arange(d), o.bin_count))
        np.testing.assert_array_equal(ds, np.concatenate([np.arange(c) for c in o.bin_count]))
    soff = b.src_offset.cpu().numpy()
    assert soff[0] == 0 and soff[-1] == n


def run_case(ctx, oracle, kind, d, length, origin, lam=0.0, v=0):
    n = len(length)
    o = oracle.balance(kind, d, length, origin, lam=lam, v=v)
    b = gpu_balance(ctx, kind, d, length, origin, lam=lam, v=v)
    check_same(b, o, n, d)
    # source CSR = origin batches in input order
    if n:
        smem = b.src_member[:n].cpu().numpy()
        np.testing.assert_array_equal(smem, np.argsort(np.asarray(origin), kind="stable"))


@pytest.mark.parametrize("kind", KINDS)
def test_random_small(ctx, oracle, kind):
    rng = np.random.default_rng(1000 + kind)
    for trial in range(150):
        d = int(rng.integers(1, 9))
        n = int(rng.integers(1 if kind in (1, 3) else 0, 40))
        hi = int(rng.choice([3, 10, 50, 5000]))
        length, origin = random_instance(rng, d, n, 1, hi,
                                         rng.choice(["random", "zero", "rr"]))
        lam = float(rng.choice([0.0, 0.01, 0.05, 0.3]))
        v = int(rng.choice([0, 1, 3, 20]))
        run_case(ctx, oracle, kind, d, length, origin, lam, v)


@pytest.mark.parametrize("kind", KINDS)
def test_random_medium_large_d(ctx, oracle, kind):
    """d > 32 exercises the round-batched block greedy."""
    rng = np.random.default_rng(2000 + kind)
    for trial in range(25):
        d = int(rng.choice([33, 64, 100, 256, 511, 600, 1024]))
        n = int(rng.integers(1, 6000))
        hi = int(rng.choice([2, 8, 100, 4096, 100000]))
        length, origin = random_instance(rng, d, n, 1, hi, rng.choice(["random", "zero", "rr"]))
        run_case(ctx, oracle, kind, d, length, origin, lam=1e-4, v=int(rng.choice([0, 64, 2048])))


@pytest.mark.parametrize("kind", KINDS)
def test_random_fused_d33_64(ctx, oracle, kind):
    """33 <= d <= 64, n <= 4096: the single-CTA kernel with two batches per lane
    (greedy, padded; quadtol / conv take the multi-kernel path). Large lengths
    push the phase total past 2^26 (64-bit greedy keys)."""
    rng = np.random.default_rng(2500 + kind)
    for trial in range(40):
        d = int(rng.integers(33, 65))
        n = int(rng.integers(1, 4097))
        hi = int(rng.choice([2, 50, 4096, 1 << 20]))
        length, origin = random_instance(rng, d, n, 1, hi, rng.choice(["random", "zero", "rr"]))
        run_case(ctx, oracle, kind, d, length, origin, lam=1e-4, v=int(rng.choice([0, 64])))


def test_quadtol_warp_scan(ctx, oracle):
    """QuadraticTolerance in the single-CTA kernel (d <= 32): the warp scan with
    cached beat masks and pointer jumping, narrow and wide d."""
    rng = np.random.default_rng(4242)
    for trial in range(60):
        d = int(rng.integers(1, 9)) if trial % 2 else int(rng.integers(9, 33))
        n = int(rng.integers(1, 3000))
        hi = int(rng.choice([4, 300, 40000]))
        length, origin = random_instance(rng, d, n, 1, hi, rng.choice(["random", "zero", "rr"]))
        v = int(rng.choice([0, 1, 8, 2048, 1 << 40]))
        run_case(ctx, oracle, 2, d, length, origin, lam=float(rng.choice([0.0, 1e-5, 0.3])), v=v)


@pytest.mark.parametrize("kind", KINDS)
def test_path_thresholds(ctx, oracle, kind):
    """Either side of every switch between kernels: the single-CTA kernel's
    item-count instantiations (512 / 1024 / 4096 items) and width limits
    (32 for quadtol / conv, 64 otherwise) against the multi-kernel path."""
    rng = np.random.default_rng(31 + kind)
    for n in (512, 513, 1024, 1025, 4096, 4097):
        for d in (8, 32, 33, 64, 65):
            length, origin = random_instance(rng, d, n, 1, 3000, "random")
            run_case(ctx, oracle, kind, d, length, origin, lam=2e-5, v=256)


def test_heavy_ties(ctx, oracle):
    """All-equal lengths: every argmin is a tie broken by the lowest index."""
    for d in (2, 7, 31, 32, 33, 64, 257):
        for n in (1, d - 1, d, d + 1, 5 * d + 3):
            if n < 1:
                continue
            length = np.full(n, 7, np.int64)
            origin = (np.arange(n) % d).astype(np.int32)
            for kind in KINDS:
                run_case(ctx, oracle, kind, d, length, origin, lam=0.01, v=2)


@pytest.mark.parametrize("shape", [(8, 512), (64, 4096), (2560, 76800), (4096, 40000)])
def test_config_shapes_greedy(ctx, oracle, shape):
    """C1 (DP=8x64), DP=64x64, C4 (DP=2560x30), and the d limit."""
    d, n = shape
    rng = np.random.default_rng(0xC1 + d)
    length = rng.integers(128, 4097, n).astype(np.int64)
    origin = (np.arange(n) % d).astype(np.int32)
    run_case(ctx, oracle, 0, d, length, origin)


@pytest.mark.parametrize("kind", [1, 2, 3])
def test_config_shapes_other_policies(ctx, oracle, kind):
    rng = np.random.default_rng(77 + kind)
    for d, n in [(8, 512), (64, 4096), (256, 20000)]:
        length = np.ceil(np.exp(rng.normal(6.5, 0.8, n))).clip(64, 4096).astype(np.int64)
        origin = (np.arange(n) % d).astype(np.int32)
        run_case(ctx, oracle, kind, d, length, origin, lam=1.0 / (6 * 8192), v=2048)


def test_long_context_quadratic(ctx, oracle):
    """C5: 32k-token sequences, quadratic cost, tolerance v=2048."""
    rng = np.random.default_rng(5)
    for P in (2, 4, 8):
        n = 8 * P
        length = rng.integers(8192, 32769, n).astype(np.int64)
        origin = (np.arange(n) % P).astype(np.int32)
        for kind in (0, 2):
            run_case(ctx, oracle, kind, P, length, origin, lam=1.0 / (6 * 8192), v=2048)
        run_case(ctx, oracle, 2, P, np.full(n, 32768, np.int64), origin, lam=2.03e-5, v=2048)


def test_identity_arrangement(ctx, oracle):
    rng = np.random.default_rng(9)
    for kind in KINDS:
        for _ in range(20):
            d = int(rng.integers(1, 40))
            n = int(rng.integers(0, 200))
            length, origin = random_instance(rng, d, n, 1, 300)
            o = oracle.identity(kind, d, length, origin, lam=0.02, v=3)
            b = gpu_balance(ctx, kind, d, length, origin, lam=0.02, v=3, identity_only=True)
            o.used_identity = 1
            check_same(b, o, n, d)


def test_reference_known_answers(ctx):
    """Golden values of proj/tests/test_balancers.cpp."""
    def items_on_zero(ls):
        return np.asarray(ls, np.int64), np.zeros(len(ls), np.int32)

    L, O = items_on_zero([5, 4, 3, 3, 2, 1])
    r = ctx.balance_host(0, 2, L, O)
    assert r["summary"].objective == 9.0                      # :40-46
    L, O = items_on_zero([3, 3, 2, 2, 2])
    assert ctx.balance_host(0, 2, L, O)["summary"].objective == 7.0  # :48-55
    L, O = items_on_zero([7, 5, 3, 2])
    r = ctx.balance_host(1, 2, L, O)
    assert r["summary"].objective == 14.0                     # :71-81
    assert ctx.min_feasible_padded_bound(2, L, O) == 14
    L, O = items_on_zero([8, 8, 4, 4])
    assert abs(ctx.balance_host(2, 2, L, O, lam=0.1, v=1)["summary"].objective - 20.0) < 1e-12
    L, O = items_on_zero([6, 5, 4, 3])
    assert abs(ctx.balance_host(3, 2, L, O, lam=0.05)["summary"].objective - 15.75) < 1e-12
    L, O = items_on_zero([7])
    assert abs(ctx.balance_host(2, 3, L, O, lam=0.2, v=2)["summary"].objective - (7 + 0.2 * 49)) < 1e-12
    L, O = items_on_zero([9])
    assert abs(ctx.balance_host(3, 2, L, O, lam=0.1)["summary"].objective - (9 + 0.1 * 81)) < 1e-12


def test_errors_match_reference_classes(ctx, oracle):
    from oracle import OracleError
    from paper_2503_23830_b200.capi import OrchError
    cases = [
        (0, 0, [1], [0], 0.0, 0),     # d = 0
        (0, 2, [1, 2], [0, 2], 0.0, 0),  # origin outside [0, d)
        (0, 2, [1, 0], [0, 1], 0.0, 0),  # length 0
        (1, 2, [], [], 0.0, 0),       # padded, empty
        (3, 2, [], [], 0.1, 0),       # conv, empty
        (2, 2, [1], [0], -1.0, 0),    # negative lambda
        (2, 2, [1], [0], 0.0, -1),    # negative v
        (3, 2, [1], [0], -0.5, 0),
        (0, 3, [5, -1, 2], [0, 5, 1], 0.0, 0),  # first bad item decides the message
    ]
    for kind, d, L, O, lam, v in cases:
        with pytest.raises(OracleError) as eo:
            oracle.balance(kind, d, L, O, lam=lam, v=v)
        with pytest.raises(OrchError) as eg:
            ctx.balance_host(kind, d, L, O, lam=lam, v=v)
        assert eg.value.code == eo.value.code
        assert eg.value.msg == eo.value.msg


def test_padded_bound_functions(ctx, oracle):
    """test_balancers.cpp:96-110 (minimal feasible bound property), seed 47."""
    rng = np.random.default_rng(47)
    for _ in range(100):
        d = int(rng.integers(1, 4))
        n = int(rng.integers(1, 11))
        L = rng.integers(1, 31, n).astype(np.int64)
        O = (np.arange(n) % d).astype(np.int32)
        b = ctx.min_feasible_padded_bound(d, L, O)
        assert b == oracle.min_feasible_padded_bound(d, L, O)
        assert ctx.padded_bound_feasible(d, L, O, b)
        assert not ctx.padded_bound_feasible(d, L, O, b - 1)
        assert ctx.padded_bound_feasible(d, L, O, int(L.max()) * (n // d + 1))


def test_greedy_wide_loads(ctx, oracle):
    """d > 32 with loads 2^32 and more apart: the LPT's relative 32-bit radix keys
    overflow and the round falls back to 64-bit bitonic keys."""
    rng = np.random.default_rng(4242)
    for d, n in [(40, 300), (300, 2000), (1500, 6000)]:
        length = rng.integers(1, 2 ** 32 - 1, n).astype(np.int64)
        length[: n // 10] = 2 ** 32 - 1
        origin = rng.integers(0, d, n).astype(np.int32)
        for kind in (0, 3):
            run_case(ctx, oracle, kind, d, length, origin, lam=1e-9)


def test_padded_search_paths(ctx, oracle):
    """BinaryPadded on the general path: the successor-table search (n <= 100K),
    groups of >= 65535 items (the table's far marker), and the one-warp-per-
    candidate scan for n > 100K; bounds checked against the oracle's bisection."""
    rng = np.random.default_rng(65535)
    cases = [
        (300, rng.integers(1, 5000, 50000)),           # table path, ~170 items/group
        (1, np.ones(70000, np.int64)),                   # one group of 70000 (far)
        (3, np.concatenate([np.ones(90000, np.int64), rng.integers(1, 9, 50)])),
        (2560, rng.integers(64, 4097, 99999)),           # C4-like, just under the table cap
        (1000, rng.integers(1, 3000, 120001)),           # warp scan, n > 100K
        (2, np.ones(150000, np.int64)),                  # warp scan with huge groups
    ]
    for d, length in cases:
        length = np.asarray(length, np.int64)
        n = len(length)
        origin = (np.arange(n) % d).astype(np.int32)
        run_case(ctx, oracle, 1, d, length, origin)
        if n <= 100000:
            b = ctx.min_feasible_padded_bound(d, length, origin)
            assert b == oracle.min_feasible_padded_bound(d, length, origin)
            assert ctx.padded_bound_feasible(d, length, origin, b)
            assert not ctx.padded_bound_feasible(d, length, origin, b - 1)


def test_pre_post_stats(ctx, oracle):
    rng = np.random.default_rng(13)
    for kind in KINDS:
        d, n = 16, 400
        length, origin = random_instance(rng, d, n, 1, 3000)
        o = oracle.balance(kind, d, length, origin, lam=0.001, v=10)
        oi = oracle.identity(kind, d, length, origin, lam=0.001, v=10)
        s = gpu_balance(ctx, kind, d, length, origin, lam=0.001, v=10).summary()
        assert (s.pre_max, s.pre_mean, s.pre_ratio) == oracle.stats(oi.bin_cost)
        assert (s.post_max, s.post_mean, s.post_ratio) == oracle.stats(o.bin_cost)


def test_reference_library_agrees(ctx, reflib):
    """Direct differential against the unmodified reference (oracle/_ref)."""
    rng = np.random.default_rng(31)
    for kind in KINDS:
        for _ in range(40):
            d = int(rng.integers(1, 70))
            n = int(rng.integers(1, 500))
            length, origin = random_instance(rng, d, n, 1, int(rng.choice([5, 500, 5000])))
            di, ds, obj, _ = reflib.balance(kind, d, length, origin, lam=0.003, v=17)
            b = gpu_balance(ctx, kind, d, length, origin, lam=0.003, v=17)
            np.testing.assert_array_equal(b.dest_inst[:n].cpu().numpy(), di)
            np.testing.assert_array_equal(b.dest_slot[:n].cpu().numpy(), ds)
            assert np.float64(b.summary().objective).tobytes() == np.float64(obj).tobytes()


@pytest.mark.parametrize("kind", KINDS)
def test_radix_passes_and_tiles(ctx, oracle, kind):
    """The hand-written device radix sort (radix.cuh) on the multi-kernel path:
    several 4096-item tiles, lengths needing 2 and 4 passes (below and above
    2^16), heavy ties (stability), origins spanning d up to 4096 (two passes)."""
    rng = np.random.default_rng(4000 + kind)
    for d, n, hi in [(100, 9000, 200), (1500, 20000, 1 << 20), (4096, 12000, 70000),
                     (80, 5000, 3)]:
        length, origin = random_instance(rng, d, n, 1, hi)
        b = gpu_balance(ctx, kind, d, length, origin, lam=1e-6, v=100)
        o = oracle.balance(kind, d, length, origin, lam=1e-6, v=100)
        check_same(b, o, n, d)


def test_group_by_origin_tiles(ctx):
    """orch_group_by_origin: the stable order by origin over many tiles."""
    rng = np.random.default_rng(77)
    for d, n in [(4096, 100000), (7, 50000), (300, 4097)]:
        origin = rng.integers(0, d, n).astype(np.int32)
        off, mem = ctx.group_by_origin(d, torch.from_numpy(origin).cuda())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(mem.cpu().numpy(), np.argsort(origin, kind="stable"))
        np.testing.assert_array_equal(off.cpu().numpy(),
                                      np.concatenate([[0], np.cumsum(np.bincount(origin, minlength=d))]))
