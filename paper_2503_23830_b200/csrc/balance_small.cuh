// Fused single-CTA balance for the common small phase (n <= 4096 items,
// d <= 32 instances: C1, C2, C5): one launch does everything the
// multi-kernel pipeline does -- validation, identity grouping, ordering,
// the policy's packing, costs, never_worse, all outputs -- with every array in
// shared memory. Same outputs, bit for bit, as the multi-kernel path.
//
// Latency is the whole game here (one SM, sequential policies), so:
//  * identity grouping ranks items with __match_any_sync per 32-item chunk
//    instead of a radix sort;
//  * the greedy (distribute_min_sum, balancers.cpp:92-107) runs on one warp
//    as exact round-batched LPT with the bins held in lanes: per round every
//    lane ranks its packed key (load << 5 | bin) against the others (d
//    independent shuffles), k = #lanes whose rank r satisfies
//    load_(r) - load_(0) < x_r (a prefix of ranks), and those k
//    lanes take items next..next+k-1 -- no re-sort between rounds;
//  * the quadratic-tolerance champion scan keeps (sum, square sum) in lanes.
#pragma once


#include "balance_kernels.cuh"

namespace orchb {
namespace {

#ifdef ORCH_SMALL_PROFILE
__device__ long long g_small_prof[16];
#define SMALL_MARK(i) do { __syncthreads(); if (threadIdx.x == 0) g_small_prof[i] = clock64(); } while (0)
#define SMALL_SUB(i) do { if (threadIdx.x == 0) g_small_prof[i] = clock64(); } while (0)
#else
#define SMALL_MARK(i) do { } while (0)
#define SMALL_SUB(i) do { } while (0)
#endif

constexpr int kSmallThreads = 256;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr int kSmallMaxD = 64;       // greedy, padded, identity; quadtol / conv: 32
constexpr int kSmallMaxItems = 4096;

struct SmallArgs {
  int kind;
  int identity_only;
  int d;
  int n;
  int64_t tol_v;
  orch_cost_model model;
  const int64_t* len;
  const int32_t* origin;
  // resolved outputs (never null)
  int32_t* dest_inst;
  int32_t* dest_slot;
  int32_t* src_slot;
  int64_t* src_off;
  int64_t* dst_off;
  int32_t* bin_count;
  int64_t* bin_len;
  int64_t* bin_tokens;
  double* bin_cost;
  int32_t* bin_offset;
  int32_t* bin_member;
  int32_t* src_offset;
  int32_t* src_member;
  orch_summary* s;
  // optional: the single-rank layout (orch_layout with P = 1), fused
  int with_layout;
  orch_layout_out lay;
};

template <int ITEMS>
struct SmallSmem {
  static constexpr int NS = kSmallThreads * ITEMS;
  static constexpr int NCH = NS / 32;  // 32-item chunks of the identity ranking
  int64_t len[NS];
  int64_t pfx[NS + 1];  // exclusive prefix of lengths in identity order, then in policy order
  int32_t org[NS];
  int32_t ord_id[NS];
  int32_t ord[NS];
  uint32_t xs[NS];
  uint16_t a_slot[NS];
  uint16_t id_rank[NS + 1];               // rank inside its chunk among same-origin items
  // origin-major, so a warp scans one origin's chunk counts conflict-free
  uint16_t chunk_base[kSmallMaxD][NCH + 2];  // same-origin items in earlier chunks (rows padded:
  uint8_t chunk_cnt[kSmallMaxD][NCH + 4];    // lanes of one chunk hit different banks)
  uint8_t a_dest[NS];
  uint8_t g_bin[NS + 1];  // greedy: bin per sorted position (g_slot = id_rank, g_off = pfx)
  struct SortTmp {  // block_sort_pairs: the other half of the key / value ping-pong
    uint32_t k[NS];
    int32_t v[NS];
    uint16_t hist[256 * kSmallWarps];  // [digit][warp]
  };
  union {
    SortTmp sort;
    int64_t wsum[kSmallWarps];  // block_exclusive_sum
  } tmp;
  int32_t cnt_id[kSmallMaxD + 1], off_id[kSmallMaxD + 1];
  int32_t cnt_a[kSmallMaxD + 1], off_a[kSmallMaxD + 1];
  int64_t tok_a[kSmallMaxD], seed_load[kSmallMaxD];
  int32_t seed_cnt[kSmallMaxD];
  // per-batch results: [0] algorithm, [1] identity
  int32_t b_cnt[2][kSmallMaxD];
  int64_t b_len[2][kSmallMaxD], b_tok[2][kSmallMaxD];
  double b_cost[2][kSmallMaxD];
  int64_t starts[kSmallMaxD + 2];
  unsigned long long nhi, nlo;  // padded search: min feasible / max infeasible + 1 this round
  unsigned long long maxlen, total;
  int bad, unsup, groups, used_identity, gfirst;
  int64_t lo, hi, bound, rounds;
};

// Warp 0: round-batched LPT over xs[first, n) (descending). Lane b < d holds
// bin b: load (optionally pre-seeded) and item count. kWrite: record, per
// sorted position, the item's bin, slot and token offset (g_bin / g_slot /
// g_off, plain predicated stores off the round's dependency chain);
// greedy_scatter() moves them to input positions with the whole block.
template <bool kWrite, int W, typename Key, int ITEMS>
__device__ void warp_greedy_w(SmallSmem<ITEMS>& S, int d, int first, int n,
                              const int64_t* init_load, const int32_t* init_cnt,
                              int64_t* rounds_out) {
  constexpr Key kKeyMax = ~Key{0};
  const int lane = threadIdx.x & 31;
  int64_t L = 0;
  int32_t cnt = 0;
  if (lane < d) {
    L = init_load ? init_load[lane] : 0;
    cnt = init_cnt ? init_cnt[lane] : 0;
  }
  int next = first;
  int64_t rounds = 0;
  while (next < n) {
    const int m = n - next < d ? n - next : d;
    const Key key = lane < d ? ((static_cast<Key>(L) << 5) | lane) : kKeyMax;
    const uint32_t xv = next + lane < n ? S.xs[next + lane] : 0u;
    int r0 = 0, r1 = 0;  // two partial counts: half the dependent adds
    Key mn;
    if constexpr (sizeof(Key) == 4) {
      mn = __reduce_min_sync(~0u, key);
#pragma unroll
      for (int j = 0; j < W; j += 2) {  // W independent shuffles in flight (keys of lanes >= d are MAX)
        r0 += __shfl_sync(~0u, key, j) < key;
        r1 += __shfl_sync(~0u, key, j + 1) < key;
      }
    } else {
      mn = key;
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        const Key k0 = __shfl_sync(~0u, key, j), k1 = __shfl_sync(~0u, key, j + 1);
        r0 += k0 < key;
        r1 += k1 < key;
        mn = k0 < mn ? k0 : mn;
        mn = k1 < mn ? k1 : mn;
      }
    }
    const int rank = r0 + r1;
    const int64_t L0 = static_cast<int64_t>(mn >> 5);
    const bool live = lane < d && rank < m;
    // x_rank: every lane read xs[next + lane] beside the key shuffles (its
    // address depends on `next` only); one shuffle by rank replaces a
    // dependent shared-memory load
    const uint32_t xr = __shfl_sync(~0u, xv, rank & 31);  // all lanes shuffle
    const int64_t x = live ? static_cast<int64_t>(xr) : 0;
    const bool c = live && (L - L0 < x);
    const int k = __popc(__ballot_sync(~0u, c));  // c holds exactly for ranks 0..k-1
    if (kWrite) {  // unconditional stores (no branch): lanes that take nothing write slot NS
      const int at = c ? next + rank : SmallSmem<ITEMS>::NS;
      S.g_bin[at] = static_cast<uint8_t>(lane);
      S.id_rank[at] = static_cast<uint16_t>(cnt);  // g_slot
      S.pfx[at] = L;                               // g_off
    }
    cnt += c ? 1 : 0;
    L += c ? x : 0;
    next += k;
    ++rounds;
  }
  if (lane < d) {
    S.cnt_a[lane] = cnt;
    S.tok_a[lane] = L;
  }
  __syncwarp();
  if (rounds_out && lane == 0) *rounds_out = rounds;
}

// Warp 0, 32 < d <= 64 (greedy only): the same rounds with two bins per lane,
// b = lane and b = lane + 32; keys (load << 6 | bin).
template <bool kWrite, typename Key, int ITEMS>
__device__ void warp_greedy_w64(SmallSmem<ITEMS>& S, int d, int n, int64_t* rounds_out) {
  constexpr Key kKeyMax = ~Key{0};
  const int lane = threadIdx.x & 31;
  const int b1 = lane + 32;
  int64_t LA = 0, LB = 0;
  int32_t cA = 0, cB = 0;
  int next = 0;
  int64_t rounds = 0;
  while (next < n) {
    const int m = n - next < d ? n - next : d;
    const Key kA = (static_cast<Key>(LA) << 6) | lane;
    const Key kB = b1 < d ? ((static_cast<Key>(LB) << 6) | b1) : kKeyMax;
    const uint32_t xa = next + lane < n ? S.xs[next + lane] : 0u;
    const uint32_t xb = next + b1 < n ? S.xs[next + b1] : 0u;
    int rA = 0, rB = 0, sA = 0, sB = 0;
    Key mn = kA < kB ? kA : kB;
#pragma unroll
    for (int j = 0; j < 32; ++j) {  // all 64 keys against both of mine (keys are distinct)
      const Key ja = __shfl_sync(~0u, kA, j), jb = __shfl_sync(~0u, kB, j);
      rA += ja < kA;
      sA += jb < kA;
      rB += ja < kB;
      sB += jb < kB;
      mn = ja < mn ? ja : mn;
      mn = jb < mn ? jb : mn;
    }
    const int rankA = rA + sA, rankB = rB + sB;
    const int64_t L0 = static_cast<int64_t>(mn >> 6);
    const uint32_t xA0 = __shfl_sync(~0u, xa, rankA & 31), xA1 = __shfl_sync(~0u, xb, rankA & 31);
    const uint32_t xB0 = __shfl_sync(~0u, xa, rankB & 31), xB1 = __shfl_sync(~0u, xb, rankB & 31);
    const bool liveA = rankA < m, liveB = b1 < d && rankB < m;
    const int64_t xA = liveA ? static_cast<int64_t>(rankA < 32 ? xA0 : xA1) : 0;
    const int64_t xB = liveB ? static_cast<int64_t>(rankB < 32 ? xB0 : xB1) : 0;
    const bool tA = liveA && (LA - L0 < xA), tB = liveB && (LB - L0 < xB);
    const int k = __popc(__ballot_sync(~0u, tA)) + __popc(__ballot_sync(~0u, tB));
    if (kWrite) {  // unconditional stores: lanes that take nothing write slot NS
      const int atA = tA ? next + rankA : SmallSmem<ITEMS>::NS;
      S.g_bin[atA] = static_cast<uint8_t>(lane);
      S.id_rank[atA] = static_cast<uint16_t>(cA);
      S.pfx[atA] = LA;
      const int atB = tB ? next + rankB : SmallSmem<ITEMS>::NS;
      S.g_bin[atB] = static_cast<uint8_t>(b1);
      S.id_rank[atB] = static_cast<uint16_t>(cB);
      S.pfx[atB] = LB;
    }
    cA += tA ? 1 : 0;
    LA += tA ? xA : 0;
    cB += tB ? 1 : 0;
    LB += tB ? xB : 0;
    next += k;
    ++rounds;
  }
  S.cnt_a[lane] = cA;
  S.tok_a[lane] = LA;
  if (b1 < d) {
    S.cnt_a[b1] = cB;
    S.tok_a[b1] = LB;
  }
  __syncwarp();
  if (rounds_out && lane == 0) *rounds_out = rounds;
}

// Whole block, after warp_greedy<true>: sorted positions [first, n) to inputs.
template <int ITEMS>
__device__ void greedy_scatter(SmallSmem<ITEMS>& S, int first, int n, int64_t* dst_off) {
  for (int k = first + static_cast<int>(threadIdx.x); k < n; k += kSmallThreads) {
    const int32_t pos = S.ord[k];
    S.a_dest[pos] = S.g_bin[k];
    S.a_slot[pos] = S.id_rank[k];
    dst_off[pos] = S.pfx[k];
  }
}

// Keys (load << 5 | bin) are 32-bit when every load fits 27 bits (loads never
// exceed the phase's total length): half the shuffles of the 64-bit keys.
template <bool kWrite, int ITEMS>
__device__ void warp_greedy(SmallSmem<ITEMS>& S, int d, int first, int n, const int64_t* init_load,
                            const int32_t* init_cnt, int64_t* rounds_out) {
  if (d > 32) {  // greedy only (the caller keeps quadtol / conv at d <= 32)
    if (S.total < (1ull << 26))
      warp_greedy_w64<kWrite, uint32_t>(S, d, n, rounds_out);
    else
      warp_greedy_w64<kWrite, uint64_t>(S, d, n, rounds_out);
    return;
  }
  if (S.total < (1ull << 27)) {
    if (d <= 8)
      warp_greedy_w<kWrite, 8, uint32_t>(S, d, first, n, init_load, init_cnt, rounds_out);
    else if (d <= 16)
      warp_greedy_w<kWrite, 16, uint32_t>(S, d, first, n, init_load, init_cnt, rounds_out);
    else
      warp_greedy_w<kWrite, 32, uint32_t>(S, d, first, n, init_load, init_cnt, rounds_out);
  } else if (d <= 8) {
    warp_greedy_w<kWrite, 8, uint64_t>(S, d, first, n, init_load, init_cnt, rounds_out);
  } else if (d <= 16) {
    warp_greedy_w<kWrite, 16, uint64_t>(S, d, first, n, init_load, init_cnt, rounds_out);
  } else {
    warp_greedy_w<kWrite, 32, uint64_t>(S, d, first, n, init_load, init_cnt, rounds_out);
  }
}

// Warp 0: exclusive scan of cnt[0..d) into off[0..d], off[d] = total (d <= 64:
// lane holds elements lane and lane + 32).
__device__ __forceinline__ void warp_offsets64(const int32_t* cnt, int32_t* off, int d, int total) {
  const int lane = threadIdx.x & 31;
  const int c0 = lane < d ? cnt[lane] : 0;
  const int c1 = lane + 32 < d ? cnt[lane + 32] : 0;
  int i0 = c0, i1 = c1;
  for (int o = 1; o < 32; o <<= 1) {
    const int u0 = __shfl_up_sync(~0u, i0, o), u1 = __shfl_up_sync(~0u, i1, o);
    if (lane >= o) {
      i0 += u0;
      i1 += u1;
    }
  }
  const int half = __shfl_sync(~0u, i0, 31);
  if (lane < d) off[lane] = i0 - c0;
  if (lane + 32 < d) off[lane + 32] = half + i1 - c1;
  if (lane == 0) off[d] = total;
}

template <int ITEMS>
__device__ __forceinline__ void block_max_total(SmallSmem<ITEMS>& S, int64_t mx, int64_t tot) {
  unsigned long long m = static_cast<unsigned long long>(mx), t = static_cast<unsigned long long>(tot);
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long om = __shfl_xor_sync(~0u, m, off);
    m = om > m ? om : m;
    t += __shfl_xor_sync(~0u, t, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&S.maxlen, m);
    atomicAdd(&S.total, t);
  }
}

// Exclusive sum over the block of ITEMS values per thread (blocked order:
// thread t holds elements t * ITEMS + j); agg = the total. Caller syncs before
// reusing wsum.
template <int ITEMS>
__device__ __forceinline__ void block_exclusive_sum(int64_t (&v)[ITEMS], int64_t* wsum,
                                                    int64_t& agg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) s += v[j];
  int64_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t u = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int64_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSmallWarps; ++w) {
    const int64_t x = wsum[w];
    before += w < warp ? x : 0;
    total += x;
  }
  int64_t ex = before + incl - s;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int64_t x = v[j];
    v[j] = ex;
    ex += x;
  }
  agg = total;
}

// Stable block LSD radix sort of the first `ns` slots of (kin, vin), 8-bit
// digits over bits [0, bits): each warp owns 32 * ITEMS consecutive slots,
// ranks its digits with __match_any_sync against per-warp counters, and a
// scan over (digit, warp) gives every slot its position. desc: digit' = 255 -
// digit (descending, equal keys keep their order). The result ends in
// (kout, vout); (kt, vt) is the other half of the ping-pong.
template <int ITEMS>
__device__ void block_sort_pairs(uint32_t* kin, int32_t* vin, uint32_t* kout, int32_t* vout,
                                 uint32_t* kt, int32_t* vt, uint16_t* hist, int bits, bool desc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int passes = bits > 0 ? (bits + 7) / 8 : 1;
  // odd pass count: start in (kin -> kout), even: (kin -> kt -> kout)
  uint32_t* ks = kin;
  int32_t* vs = vin;
  for (int p = 0; p < passes; ++p) {
    const bool last = p == passes - 1;
    uint32_t* kd = last ? kout : ((passes - p) % 2 == 0 ? kt : kout);
    int32_t* vd = last ? vout : ((passes - p) % 2 == 0 ? vt : vout);
    for (int i = threadIdx.x; i < 256 * kSmallWarps; i += kSmallThreads) hist[i] = 0;
    __syncthreads();
    uint32_t key[ITEMS];
    int32_t val[ITEMS];
    int dig[ITEMS], rank[ITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int i = warp * 32 * ITEMS + j * 32 + lane;
      key[j] = ks[i];
      val[j] = vs[i];
      const int dg = static_cast<int>((key[j] >> (8 * p)) & 255u);
      dig[j] = desc ? 255 - dg : dg;
    }
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const unsigned peers = __match_any_sync(~0u, dig[j]);
      const int before = __popc(peers & lt);
      uint16_t* h = hist + dig[j] * kSmallWarps + warp;
      const int run = *h;
      rank[j] = run + before;
      __syncwarp();
      if (before == 0) *h = static_cast<uint16_t>(run + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    {  // exclusive scan over hist[digit][warp], 8 entries per thread
      static_assert(256 * kSmallWarps == 8 * kSmallThreads, "8 counters per thread");
      __shared__ uint32_t ws[kSmallWarps];
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = hist[8 * threadIdx.x + q];
        sum += v[q];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(~0u, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) ws[warp] = incl;
      __syncthreads();
      uint32_t before = 0;
#pragma unroll
      for (int w = 0; w < kSmallWarps; ++w) before += w < warp ? ws[w] : 0u;
      uint32_t ex = before + incl - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        hist[8 * threadIdx.x + q] = static_cast<uint16_t>(ex);
        ex += v[q];
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int pos = hist[dig[j] * kSmallWarps + warp] + rank[j];
      ORCH_DCHECK(pos < kSmallThreads * ITEMS);
      kd[pos] = key[j];
      vd[pos] = val[j];
    }
    __syncthreads();
    ks = kd;
    vs = vd;
  }
}

template <int ITEMS>
__global__ void __launch_bounds__(kSmallThreads, 1) k_balance_small(SmallArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SS = SmallSmem<ITEMS>;
  SS& S = *reinterpret_cast<SS*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  // provably warp-uniform (no WARPSYNC.COLLECTIVE around the warp-level code)
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const int n = a.n, d = a.d;
  const int nch = (n + 31) / 32;
  orch_summary* sum = a.s;

  SMALL_MARK(0);
  // ---- S1: load, validate (index_sources, balancers.cpp:25-37)
  if (tid == 0) {
    S.bad = INT_MAX;
    S.unsup = 0;
    S.maxlen = 0;
    S.total = 0;
  }
  __syncthreads();
  {
    int64_t mx = 0, tot = 0;
    for (int i = tid; i < n; i += kSmallThreads) {
      const int32_t o = a.origin[i];
      const int64_t l = a.len[i];
      S.len[i] = l;
      S.org[i] = o;
      if (o < 0 || o >= d || l < 1) atomicMin(&S.bad, i);
      if (l > ORCH_MAX_LENGTH) S.unsup = 1;
      mx = l > mx ? l : mx;
      tot += l > 0 ? l : 0;
    }
    block_max_total(S, mx, tot);
  }
  __syncthreads();
  if (S.bad < n || S.unsup || S.total >= (1ull << 50)) {
    if (tid == 0) {
      sum->objective = sum->algo_objective = sum->identity_objective = 0.0;
      sum->pre_max = sum->pre_mean = sum->post_max = sum->post_mean = 0.0;
      sum->pre_ratio = sum->post_ratio = 1.0;
      sum->bound = 0;
      sum->used_identity = 0;
      sum->rounds = 0;
      if (S.bad < n) {
        sum->error = ORCH_INVALID_ARGUMENT;
        sum->error_index = S.bad;
      } else {
        sum->error = ORCH_UNSUPPORTED;
        sum->error_index = INT64_MAX;
      }
    }
    return;
  }

  SMALL_MARK(1);
  // ---- S2: identity grouping (batches_from_items, core.cpp:183-199): the
  // source slot of an item is the number of earlier items with its origin.
  // Same-origin lanes of a 32-item chunk by one ballot per origin bit (d <= 64:
  // at most 6), cheaper than __match_any_sync.
  const int obits = d > 1 ? 32 - __clz(d - 1) : 0;
#pragma unroll 2
  for (int c = warp; c < nch; c += kSmallWarps) {
    const int i = c * 32 + lane;
    const int o = i < n ? S.org[i] : 0;
    unsigned peers = __ballot_sync(~0u, i < n);
    for (int bit = 0; bit < obits; ++bit) {
      const bool set = (o >> bit) & 1;
      const unsigned m = __ballot_sync(~0u, set);
      peers &= set ? m : ~m;
    }
    if (i < n) S.id_rank[i] = static_cast<uint16_t>(__popc(peers & ((1u << lane) - 1u)));
    if (lane < d) S.chunk_cnt[lane][c] = 0;
    if (lane + 32 < d) S.chunk_cnt[lane + 32][c] = 0;
    __syncwarp();
    if (i < n && (__ffs(peers) - 1) == lane) S.chunk_cnt[o][c] = static_cast<uint8_t>(__popc(peers));
  }
  __syncthreads();
  SMALL_SUB(10);
  {  // running count of each origin over the chunks: warp per origin, lane per
     // ceil(NCH / 32) consecutive chunks, one warp scan
    constexpr int PER = (SS::NCH + 31) / 32;
    for (int o = warp; o < d; o += kSmallWarps) {
      int c[PER], tot = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int ch = lane * PER + j;
        c[j] = ch < nch ? S.chunk_cnt[o][ch] : 0;
        tot += c[j];
      }
      int incl = tot;
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(~0u, incl, off);
        if (lane >= off) incl += u;
      }
      int run = incl - tot;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int ch = lane * PER + j;
        if (ch < nch) S.chunk_base[o][ch] = static_cast<uint16_t>(run);
        run += c[j];
      }
      if (lane == 31) S.cnt_id[o] = incl;
    }
  }
  __syncthreads();
  SMALL_SUB(11);
  if (warp == 0) warp_offsets64(S.cnt_id, S.off_id, d, n);  // offsets of the origin batches
  __syncthreads();
  SMALL_SUB(12);
  for (int i = tid; i < n; i += kSmallThreads) {
    const int o = S.org[i];
    const int slot = S.chunk_base[o][i >> 5] + S.id_rank[i];
    ORCH_DCHECK(o >= 0 && o < d && S.off_id[o] + slot < S.off_id[o + 1]);
    a.src_slot[i] = slot;
    S.ord_id[S.off_id[o] + slot] = i;
    S.a_slot[i] = static_cast<uint16_t>(S.off_id[o] + slot);  // identity position (a_slot is free here)
  }
  __syncthreads();
  SMALL_SUB(13);
  {
    int64_t v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int k = tid * ITEMS + j;
      v[j] = k < n ? S.len[S.ord_id[k]] : 0;
    }
    int64_t agg;
    block_exclusive_sum<ITEMS>(v, S.tmp.wsum, agg);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) S.pfx[tid * ITEMS + j] = v[j];
    if (tid == 0) S.pfx[SS::NS] = agg;
  }
  __syncthreads();
  SMALL_SUB(14);
  for (int i = tid; i < n; i += kSmallThreads)  // by input position: coalesced org / a_slot reads
    a.src_off[i] = S.pfx[S.a_slot[i]] - S.pfx[S.off_id[S.org[i]]];
  for (int k = tid; k < n; k += kSmallThreads) a.src_member[k] = S.ord_id[k];
  if (tid <= d) a.src_offset[tid] = S.off_id[tid];

  SMALL_MARK(2);
  // ---- S3..S5: the policy's own packing
  if (!a.identity_only) {
    const bool asc = a.kind == ORCH_BINARY_PADDED;
    // key bits of the longest item; ascending padding sorts after equal keys (stable sort)
    const int lbits = 32 - __clz(static_cast<unsigned>(S.maxlen));
    const uint32_t pad_asc = lbits == 32 ? 0xffffffffu : ((1u << lbits) - 1u);
    if (n <= kSmallThreads) {
      // few items (C5: 64): each thread ranks its item against all n keys
      // (broadcast shared-memory reads) -- the stable order of the reference's
      // std::stable_sort by length, without the block radix sort's passes
      if (tid < n) {
        const uint32_t ki = static_cast<uint32_t>(S.len[tid]);
        int r = 0;
#pragma unroll 8
        for (int j = 0; j < n; ++j) {
          const uint32_t kj = static_cast<uint32_t>(S.len[j]);
          r += (asc ? kj < ki : kj > ki) || (kj == ki && j < tid);
        }
        ORCH_DCHECK(r >= 0 && r < n);
        S.ord[r] = tid;
        S.xs[r] = ki;
      }
    } else {
      // stage the keys (padding slots sort last) and sort into (S.xs, S.ord)
      __syncthreads();  // tmp storage reuse
      uint32_t* kst = S.tmp.sort.k;
      int32_t* vst = S.tmp.sort.v;
      for (int i = tid; i < SS::NS; i += kSmallThreads) {
        kst[i] = i < n ? static_cast<uint32_t>(S.len[i]) : (asc ? pad_asc : 0u);
        vst[i] = i;
      }
      __syncthreads();
      block_sort_pairs<ITEMS>(kst, vst, S.xs, S.ord, kst, vst, S.tmp.sort.hist, lbits, !asc);
    }
    __syncthreads();
    SMALL_MARK(3);
    if (a.kind == ORCH_GREEDY_UNPADDED) {
      if (warp == 0) warp_greedy<true>(S, d, 0, n, nullptr, nullptr, &S.rounds);
      __syncthreads();
      greedy_scatter(S, 0, n, a.dst_off);
    } else if (a.kind == ORCH_QUADRATIC_TOLERANCE) {
      if (warp == 0) {
        // Champion scan (balancers.cpp:223-231): best = 0; for i = 1..d-1:
        // if less(s[i], s[best]) best = i, with the non-transitive tolerance
        // comparator less(a, b) = |a.sum - b.sum| < v ? a.sq < b.sq : a.sum < b.sum.
        // Lane j holds batch j and beats_j, bit i set iff less(s[i], s[j]).
        // An item changes one batch b, so only row and column b are redone
        // (one ballot). The scan moves from a champion j to the first later
        // batch that beats it, nxt_j = lowest bit of beats_j above j.
        const int64_t v = a.tol_v;
        const unsigned dmask = d >= 32 ? ~0u : ((1u << d) - 1u);
        const unsigned above = lane >= 31 ? 0u : (dmask & (~0u << (lane + 1)));
        int64_t qs = 0, qq = 0;
        int32_t cnt = 0;
        unsigned beats = 0;  // all sums equal and zero: nothing beats anything
        uint32_t x_next = n > 0 ? S.xs[0] : 0u;  // raw: widened where used
        if (d <= 8) {
          // d <= 8 (C5): the champion chain is walked on a packed word, 4 bits
          // per batch j = nxt_j (15: nothing later beats j), rebuilt by one OR
          // reduction per item, so a step is a 32-bit shift and mask with no
          // shuffle. Both comparisons are evaluated and masked (no divergent
          // branch): ~400 cycles per item against ~530 with the branches
          // (scripts/qt_bench.cu).
          unsigned W = 0xffffffffu;
          for (int k = 0; k < n; ++k) {
            const int64_t x = static_cast<int64_t>(x_next);
            if (k + 1 < n) x_next = S.xs[k + 1];
            const int64_t xx = x * x;
            int best = 0;
            for (;;) {
              const unsigned t = (W >> (4 * best)) & 0xfu;
              if (t == 0xfu) break;
              best = static_cast<int>(t);
            }
            const bool me = lane == best;
            const int at = me ? k : SmallSmem<ITEMS>::NS;  // per sorted position, no branch
            S.g_bin[at] = static_cast<uint8_t>(lane);
            S.id_rank[at] = static_cast<uint16_t>(cnt);
            S.pfx[at] = qs;
            cnt += me ? 1 : 0;
            qs += me ? x : 0;
            qq += me ? xx : 0;
            const int64_t bs = __shfl_sync(~0u, qs, best);
            const int64_t bq = __shfl_sync(~0u, qq, best);
            const int64_t df = qs - bs;
            const bool near = (df < 0 ? -df : df) < v;
            const bool on = lane < d && !me;
            const bool b_beats_me = on & (near ? bq < qq : bs < qs);
            const bool i_beat_b = on & (near ? qq < bq : qs < bs);
            const unsigned row = __ballot_sync(~0u, i_beat_b);
            beats = me ? row : ((beats & ~(1u << best)) | (b_beats_me ? 1u << best : 0u));
            const unsigned m = beats & above;
            const unsigned nx = m ? static_cast<unsigned>(__ffs(m) - 1) : 0xfu;
            W = __reduce_or_sync(~0u, lane < 8 ? nx << (4 * lane) : 0u);
          }
        } else {
        for (int k = 0; k < n; ++k) {
          const int64_t x = static_cast<int64_t>(x_next);
          if (k + 1 < n) x_next = S.xs[k + 1];  // off the critical path
          // the scan's last champion, by pointer jumping along the chain
          // 0 -> nxt_0 -> ... (a batch nothing later beats points to itself):
          // ceil(log2 d) dependent shuffles, no branches
          const int nxt = __ffs(beats & above) - 1;
          int jump = nxt < 0 ? lane : nxt;
          for (int span = 1; span < d; span <<= 1) jump = __shfl_sync(~0u, jump, jump);
          const int best = __shfl_sync(~0u, jump, 0);
          const bool me = lane == best;
          const int at = me ? k : SmallSmem<ITEMS>::NS;  // per sorted position, no branch
          S.g_bin[at] = static_cast<uint8_t>(lane);
          S.id_rank[at] = static_cast<uint16_t>(cnt);
          S.pfx[at] = qs;
          cnt += me ? 1 : 0;
          qs += me ? x : 0;
          qq += me ? x * x : 0;
          const int64_t bs = __shfl_sync(~0u, qs, best);
          const int64_t bq = __shfl_sync(~0u, qq, best);
          // column best: does batch `best` beat me; row best: do I beat it
          const int64_t df = qs - bs;
          const bool near = (df < 0 ? -df : df) < v;
          const bool b_beats_me = !me & (near ? bq < qq : bs < qs);
          const bool i_beat_b = (lane < d) & !me & (near ? qq < bq : qs < bs);
          const unsigned row = __ballot_sync(~0u, i_beat_b);
          beats = lane == best ? row : ((beats & ~(1u << best)) | (b_beats_me ? 1u << best : 0u));
        }
        }
        if (lane < d) {
          S.cnt_a[lane] = cnt;
          S.tok_a[lane] = qs;
        }
        if (lane == 0) S.rounds = n;
      }
      __syncthreads();
      greedy_scatter(S, 0, n, a.dst_off);
    } else if (a.kind == ORCH_CONVTRANSFORMER) {
      if (warp == 0) {
        // bound = greedy objective (balancers.cpp:247-256)
        warp_greedy<false>(S, d, 0, n, nullptr, nullptr, nullptr);
        int64_t bound = lane < d ? S.tok_a[lane] : 0;
        for (int off = 16; off > 0; off >>= 1) {
          const int64_t o = __shfl_xor_sync(~0u, bound, off);
          bound = o > bound ? o : bound;
        }
        if (lane < d) {
          S.seed_load[lane] = 0;
          S.seed_cnt[lane] = 0;
        }
        __syncwarp();
        // seeding (balancers.cpp:258-267), 32 items per ballot
        int g = 0;
        int64_t size = 0, load = 0;
        int k = 0;
        while (k < n) {
          const int t = k + lane;
          const int64_t x = t < n ? static_cast<int64_t>(S.xs[t]) : 0;
          const bool c = t < n && (size + lane + 1) * x > bound;
          const unsigned mv = __ballot_sync(~0u, t < n);
          const unsigned m = __ballot_sync(~0u, c);
          const int take = m ? __ffs(m) - 1 : __popc(mv);
          int64_t incl = lane < take ? x : 0;
          for (int off = 1; off < 32; off <<= 1) {
            const int64_t o = __shfl_up_sync(~0u, incl, off);
            if (lane >= off) incl += o;
          }
          if (lane < take) {
            const int32_t pos = S.ord[t];
            S.a_dest[pos] = static_cast<uint8_t>(g);
            S.a_slot[pos] = static_cast<uint16_t>(size + lane);
            a.dst_off[pos] = load + incl - x;
          }
          load += __shfl_sync(~0u, incl, 31);
          size += take;
          k += take;
          if (m) {
            if (g + 1 == d) break;
            if (lane == 0) {
              S.seed_load[g] = load;
              S.seed_cnt[g] = static_cast<int32_t>(size);
            }
            ++g;
            size = 0;
            load = 0;
          }
        }
        if (lane == 0) {
          S.seed_load[g] = load;
          S.seed_cnt[g] = static_cast<int32_t>(size);
          S.bound = bound;
        }
        __syncwarp();
        warp_greedy<true>(S, d, k, n, S.seed_load, S.seed_cnt, &S.rounds);
        if (lane == 0) S.gfirst = k;
      }
      __syncthreads();
      greedy_scatter(S, S.gfirst, n, a.dst_off);
    } else {  // BinaryPadded: k-ary search over the ascending lengths in smem
      {
        int64_t v[ITEMS];  // prefix of ascending lengths (token offsets in groups)
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
          const int k = tid * ITEMS + j;
          v[j] = k < n ? static_cast<int64_t>(S.xs[k]) : 0;
        }
        int64_t agg;
        __syncthreads();
        block_exclusive_sum<ITEMS>(v, S.tmp.wsum, agg);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) S.pfx[tid * ITEMS + j] = v[j];
        if (tid == 0) S.pfx[n] = agg;
      }
      const int64_t max_len = S.xs[n - 1];
      if (tid == 0) {
        S.lo = max_len;
        S.hi = max_len * (n / d + 1);
      }
      __syncthreads();
#ifdef ORCH_SMALL_PROFILE
      if (tid == 0) g_small_prof[8] = clock64();
#endif
      // k-ary search with one candidate bound per thread (256 per round; the
      // answer is the minimal feasible bound whatever the probe order)
      while (true) {
        const int64_t lo = S.lo, hi = S.hi;
        if (lo >= hi) break;
        const int64_t span = hi - lo;
        const int64_t c = span <= kSmallThreads ? lo + tid : lo + (span * tid) / kSmallThreads;
        __syncthreads();  // every thread has read lo / hi
        if (tid == 0) {
          S.nhi = static_cast<unsigned long long>(hi);
          S.nlo = static_cast<unsigned long long>(lo);
        }
        __syncthreads();
        if (c < hi) {
          if (thread_feasible(S.xs, n, d, c))
            atomicMin(&S.nhi, static_cast<unsigned long long>(c));
          else
            atomicMax(&S.nlo, static_cast<unsigned long long>(c + 1));
        }
        __syncthreads();
        if (tid == 0) {
          const int64_t nhi = static_cast<int64_t>(S.nhi), nlo = static_cast<int64_t>(S.nlo);
          S.hi = nhi;
          S.lo = nlo < nhi ? nlo : nhi;
        }
        __syncthreads();
      }
#ifdef ORCH_SMALL_PROFILE
      if (tid == 0) g_small_prof[9] = clock64();
#endif
      if (warp == 0) {
        const int64_t bound = S.hi;
        int64_t p = 0;
        int g = 0;
        int64_t size = 0;
        while (p < n) {
          if (lane == 0) S.starts[g] = p;
          ++g;
          const int64_t q = warp_next_start_hint(S.xs, n, p, bound, lane, size);
          size = q - p;
          p = q;
        }
        if (lane == 0) {
          S.starts[g] = n;
          S.groups = g;
          S.bound = bound;
          S.rounds = 0;
        }
      }
      __syncthreads();
      const int G = S.groups;
      for (int k = tid; k < n; k += kSmallThreads) {
        int g = 0, hi = G - 1;  // last group whose start is <= k
        while (g < hi) {
          const int mid = (g + hi + 1) >> 1;
          if (S.starts[mid] <= k) g = mid; else hi = mid - 1;
        }
        const int32_t pos = S.ord[k];
        S.a_dest[pos] = static_cast<uint8_t>(g);
        S.a_slot[pos] = static_cast<uint16_t>(k - S.starts[g]);
        a.dst_off[pos] = S.pfx[k] - S.pfx[S.starts[g]];
      }
      if (tid < d) S.cnt_a[tid] = tid < G ? static_cast<int32_t>(S.starts[tid + 1] - S.starts[tid]) : 0;
    }
    __syncthreads();
    SMALL_MARK(4);
    // ---- algorithm CSR (balancers.cpp:43-60 assemble: slot = position in bin)
    if (warp == 0) warp_offsets64(S.cnt_a, S.off_a, d, n);
    __syncthreads();
    for (int i = tid; i < n; i += kSmallThreads) {
      const int b = S.a_dest[i];
      const int sl = S.a_slot[i];
      a.dest_inst[i] = b;
      a.dest_slot[i] = sl;
      ORCH_DCHECK(b >= 0 && b < d && S.off_a[b] + sl < S.off_a[b + 1]);
      S.ord[S.off_a[b] + sl] = i;  // reuse: algorithm members in (batch, slot) order
    }
    __syncthreads();
    for (int k = tid; k < n; k += kSmallThreads) a.bin_member[k] = S.ord[k];
    if (tid <= d) a.bin_offset[tid] = S.off_a[tid];
  }

  SMALL_MARK(5);
  // ---- S6: batch costs (core.cpp:91-118), algorithm batches then identity batches.
  // Integer sums are exact; Sum l^2 is replayed as the reference's sequential
  // double loop when a partial sum could reach 2^53.
  const orch_cost_model& model = a.model;
  auto finish_batch = [&](int side, int b, int beg, int end, int64_t s, int64_t mx, double sqd) {
    const int64_t cnt = end - beg;
    S.b_cnt[side][b] = static_cast<int32_t>(cnt);
    S.b_tok[side][b] = s;
    S.b_len[side][b] = model.padded ? cnt * mx : s;
    S.b_cost[side][b] = batch_cost(model, cnt, s, mx, sqd);
  };
  auto replay_sq = [&](int side, int beg, int end) {
    double acc = 0.0;
    for (int k = beg; k < end; ++k) {
      const double l = static_cast<double>(S.len[side ? S.ord_id[k] : S.ord[k]]);
      acc = rn_add(acc, rn_mul(l, l));
    }
    return acc;
  };
  const bool quad_unpadded = model.variant == ORCH_TRANSFORMER_QUADRATIC && !model.padded;
  if (d >= 32) {  // many short batches: a thread per batch
    for (int task = tid; task < 2 * d; task += kSmallThreads) {
      const int side = task < d ? 0 : 1;  // 0 algorithm, 1 identity
      const int b = side ? task - d : task;
      if (side == 0 && a.identity_only) continue;
      const int beg = side ? S.off_id[b] : S.off_a[b];
      const int end = side ? S.off_id[b + 1] : S.off_a[b + 1];
      int64_t sm = 0, mx = 0;
      unsigned long long sq = 0;
      bool inexact = false;
      for (int k = beg; k < end; ++k) {
        const int64_t l = S.len[side ? S.ord_id[k] : S.ord[k]];
        sm += l;
        mx = l > mx ? l : mx;
        if (l >= (1ll << 26)) inexact = true;
        sq += static_cast<unsigned long long>(l) * static_cast<unsigned long long>(l);
        if (sq >= (1ull << 53)) inexact = true;
      }
      finish_batch(side, b, beg, end, sm, mx,
                   inexact && quad_unpadded ? replay_sq(side, beg, end) : static_cast<double>(sq));
    }
  } else {  // few long batches: a warp per batch
    for (int task = warp; task < 2 * d; task += kSmallWarps) {
      const int side = task < d ? 0 : 1;
      const int b = side ? task - d : task;
      if (side == 0 && a.identity_only) continue;
      const int beg = side ? S.off_id[b] : S.off_a[b];
      const int end = side ? S.off_id[b + 1] : S.off_a[b + 1];
      int64_t sm = 0, mx = 0;
      unsigned long long sq = 0;
      bool inexact = false;
      for (int k = beg + lane; k < end; k += 32) {
        const int64_t l = S.len[side ? S.ord_id[k] : S.ord[k]];
        sm += l;
        mx = l > mx ? l : mx;
        if (l >= (1ll << 26)) inexact = true;
        sq += static_cast<unsigned long long>(l) * static_cast<unsigned long long>(l);
        if (sq >= (1ull << 53)) inexact = true;
      }
      for (int off = 16; off > 0; off >>= 1) {
        sm += __shfl_xor_sync(~0u, sm, off);
        const int64_t om = __shfl_xor_sync(~0u, mx, off);
        mx = om > mx ? om : mx;
        sq += __shfl_xor_sync(~0u, sq, off);
      }
      inexact = __any_sync(~0u, inexact) || sq >= (1ull << 53);
      double sqd = static_cast<double>(sq);
      if (inexact && quad_unpadded) {
        double acc = 0.0;
        if (lane == 0) acc = replay_sq(side, beg, end);
        sqd = __shfl_sync(~0u, acc, 0);
      }
      if (lane == 0) finish_batch(side, b, beg, end, sm, mx, sqd);
    }
  }
  __syncthreads();
  SMALL_MARK(6);
  // ---- never_worse (balancers.cpp:71-76) + stats_of (orchestrator.cpp:91-102)
  if (tid == 0) {
    double stat[2][3];
    for (int side = 0; side < 2; ++side) {
      double M = 0.0, T = 0.0;
      if (side == 0 && a.identity_only) {
        stat[0][0] = stat[0][1] = 0.0;
        stat[0][2] = 1.0;
        continue;
      }
      for (int b = 0; b < d; ++b) {
        const double c = S.b_cost[side][b];
        M = c > M ? c : M;
        T = rn_add(T, c);
      }
      const double mean = rn_div(T, static_cast<double>(d));
      stat[side][0] = M;
      stat[side][1] = mean;
      stat[side][2] = mean > 0.0 ? rn_div(M, mean) : 1.0;
    }
    const bool ident = a.identity_only || stat[1][0] <= stat[0][0];
    S.used_identity = ident ? 1 : 0;
    const int w = ident ? 1 : 0;
    sum->identity_objective = stat[1][0];
    sum->algo_objective = a.identity_only ? stat[1][0] : stat[0][0];
    sum->objective = stat[w][0];
    sum->pre_max = stat[1][0];
    sum->pre_mean = stat[1][1];
    sum->pre_ratio = stat[1][2];
    sum->post_max = stat[w][0];
    sum->post_mean = stat[w][1];
    sum->post_ratio = stat[w][2];
    sum->used_identity = S.used_identity;
    sum->error = 0;
    sum->error_index = INT64_MAX;
    sum->bound = a.identity_only
                     ? 0
                     : ((a.kind == ORCH_BINARY_PADDED || a.kind == ORCH_CONVTRANSFORMER) ? S.bound
                                                                                         : 0);
    sum->rounds = a.identity_only ? 0 : S.rounds;
  }
  __syncthreads();
  const int w = S.used_identity;
  if (tid < d) {
    a.bin_count[tid] = S.b_cnt[w][tid];
    a.bin_len[tid] = S.b_len[w][tid];
    a.bin_tokens[tid] = S.b_tok[w][tid];
    a.bin_cost[tid] = S.b_cost[w][tid];
  }
  if (w) {  // identity arrangement: dest = origin, slot = source slot
    for (int i = tid; i < n; i += kSmallThreads) {
      a.dest_inst[i] = S.org[i];
      a.dest_slot[i] = a.src_slot[i];
      a.dst_off[i] = a.src_off[i];
      a.bin_member[i] = S.ord_id[i];
    }
    if (tid <= d) a.bin_offset[tid] = S.off_id[tid];
  }
  if (a.with_layout) {
    // orch_layout for one rank (k_layout_small with P = 1): every instance on
    // rank 0, origin batches in instance order in the input buffer, destination
    // batches in instance order in the output buffer; the (0 -> 0) segment is
    // the whole output, so pair_off = rank_dst_off.
    __syncthreads();  // the identity epilogue's dst_off stores
    if (warp == 0) {  // instance bases: exclusive scans over d <= 64 batch totals
      for (int side = 0; side < 2; ++side) {
        const int64_t* tok = side ? S.b_tok[w] : S.b_tok[1];
        int64_t* base = side ? S.tok_a : S.seed_load;  // free here
        const int64_t t0 = lane < d ? tok[lane] : 0, t1 = lane + 32 < d ? tok[lane + 32] : 0;
        int64_t i0 = t0, i1 = t1;
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t u0 = __shfl_up_sync(~0u, i0, o), u1 = __shfl_up_sync(~0u, i1, o);
          if (lane >= o) {
            i0 += u0;
            i1 += u1;
          }
        }
        const int64_t half = __shfl_sync(~0u, i0, 31);
        if (lane < d) base[lane] = i0 - t0;
        if (lane + 32 < d) base[lane + 32] = half + i1 - t1;
        if (side == 1 && lane == 0) {
          const int64_t total = static_cast<int64_t>(S.total);
          a.lay.in_rows[0] = total;
          a.lay.out_rows[0] = total;
          a.lay.send_rows[0] = total;
          a.lay.send_displ[0] = 0;
          a.lay.recv_displ[0] = 0;
          *a.lay.status = 0;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += kSmallThreads) {
      const int64_t rd = a.dst_off[i] + S.tok_a[w ? S.org[i] : S.a_dest[i]];
      a.lay.rank_src_off[i] = a.src_off[i] + S.seed_load[S.org[i]];
      a.lay.rank_dst_off[i] = rd;
      a.lay.pair_off[i] = rd;
    }
  }
  SMALL_MARK(7);
}

}  // namespace
}  // namespace orchb
