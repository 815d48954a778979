// Fused single-CTA balance for the common small phase (n <= 4096 items,
// d <= 32 instances: C1, C2, C5): one launch does everything the
// multi-kernel pipeline does -- validation, identity grouping, ordering,
// the policy's packing, costs, never_worse, all outputs -- with every array in
// shared memory. Same outputs, bit for bit, as the multi-kernel path.
//
// The greedy (distribute_min_sum, balancers.cpp:92-107) runs on one warp as
// exact round-batched LPT: lane r holds the bin of rank r (packed key
// load << 5 | bin); per round the first k items go to ranks 0..k-1 where k is
// the first r with load_(r) - load_(0) >= x_r, then a register bitonic sort
// restores the order (proof in DESIGN.md).
#pragma once

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "balance_kernels.cuh"

namespace orchb {
namespace {

#ifdef ORCH_SMALL_PROFILE
__device__ long long g_small_prof[16];
#define SMALL_MARK(i) do { __syncthreads(); if (threadIdx.x == 0) g_small_prof[i] = clock64(); } while (0)
#else
#define SMALL_MARK(i) do { } while (0)
#endif

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxD = 32;

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
};

template <int ITEMS>
struct SmallSmem {
  static constexpr int NS = kSmallThreads * ITEMS;
  using Sort = cub::BlockRadixSort<uint32_t, kSmallThreads, ITEMS, int32_t>;
  using Scan = cub::BlockScan<int64_t, kSmallThreads>;
  int64_t len[NS];
  int64_t pfx[NS + 1];  // exclusive prefix of lengths in identity order, then in policy order
  int32_t org[NS];
  int32_t ord_id[NS];
  int32_t ord[NS];
  uint32_t xs[NS];
  uint16_t a_slot[NS];
  uint8_t a_dest[NS];
  union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  int32_t cnt_id[kSmallMaxD + 1], off_id[kSmallMaxD + 1];
  int32_t cnt_a[kSmallMaxD + 1], off_a[kSmallMaxD + 1];
  int64_t tok_a[kSmallMaxD], seed_load[kSmallMaxD];
  int32_t seed_cnt[kSmallMaxD];
  int64_t qsum[kSmallMaxD], qsq[kSmallMaxD];
  // per-batch results: [0] algorithm, [1] identity
  int32_t b_cnt[2][kSmallMaxD];
  int64_t b_len[2][kSmallMaxD], b_tok[2][kSmallMaxD];
  double b_cost[2][kSmallMaxD];
  int64_t starts[kSmallMaxD + 2];
  int64_t cand[32];
  int feas[32];
  unsigned long long maxlen, total;
  int bad, unsup, k, groups, used_identity;
  int64_t lo, hi, bound, consumed, rounds;
};

__device__ __forceinline__ uint64_t warp_bitonic(uint64_t key, int width) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= width; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t other = __shfl_xor_sync(~0u, key, stride);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      const uint64_t lo = other < key ? other : key;
      const uint64_t hi = other < key ? key : other;
      key = (lower == up) ? lo : hi;
    }
  return key;
}

// Warp 0: round-batched LPT over xs[first, n) (descending), bins optionally
// pre-seeded. kWrite: record each item's bin / slot / token offset.
template <bool kWrite, int ITEMS>
__device__ void warp_greedy(SmallSmem<ITEMS>& S, int d, int first, int n, const int64_t* init_load,
                            const int32_t* init_cnt, int64_t* dst_off, int64_t* rounds_out) {
  const int lane = threadIdx.x & 31;
  int width = 1;
  while (width < d) width <<= 1;
  uint64_t key = kU64Max;
  if (lane < d) {
    key = (static_cast<uint64_t>(init_load ? init_load[lane] : 0) << 5) | lane;
    S.cnt_a[lane] = init_cnt ? init_cnt[lane] : 0;
  }
  __syncwarp();
  if (init_load) key = warp_bitonic(key, width);
  int next = first;
  int64_t rounds = 0;
  while (next < n) {
    const int m = n - next < d ? n - next : d;
    const int64_t L = static_cast<int64_t>(key >> 5);
    const int64_t L0 = __shfl_sync(~0u, L, 0);
    const int64_t x = lane < m ? static_cast<int64_t>(S.xs[next + lane]) : 0;
    const bool c = lane < m && (L - L0 < x);
    const unsigned bal = __ballot_sync(~0u, c);
    const int k = bal == ~0u ? 32 : __ffs(~bal) - 1;
    if (lane < k) {
      const int b = static_cast<int>(key & 31u);
      if (kWrite) {
        const int32_t pos = S.ord[next + lane];
        S.a_dest[pos] = static_cast<uint8_t>(b);
        S.a_slot[pos] = static_cast<uint16_t>(S.cnt_a[b]);
        dst_off[pos] = L;
      }
      S.cnt_a[b] += 1;  // each bin has one rank: no race
      key = (static_cast<uint64_t>(L + x) << 5) | static_cast<uint64_t>(b);
    }
    __syncwarp();
    key = warp_bitonic(key, width);
    next += k;
    ++rounds;
  }
  if (lane < d) S.tok_a[key & 31u] = static_cast<int64_t>(key >> 5);
  __syncwarp();
  if (rounds_out && lane == 0) *rounds_out = rounds;
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

template <int ITEMS>
__global__ void __launch_bounds__(kSmallThreads, 1) k_balance_small(SmallArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SS = SmallSmem<ITEMS>;
  SS& S = *reinterpret_cast<SS*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  // provably warp-uniform (no WARPSYNC.COLLECTIVE around the warp-level greedy)
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const int n = a.n, d = a.d;
  orch_summary* sum = a.s;

  SMALL_MARK(0);
  // ---- S1: load, validate (index_sources, balancers.cpp:25-37)
  if (tid == 0) {
    S.bad = INT_MAX;
    S.unsup = 0;
    S.maxlen = 0;
    S.total = 0;
  }
  if (tid <= kSmallMaxD) S.cnt_id[tid] = 0;
  __syncthreads();
  {
    int64_t mx = 0, tot = 0;
    for (int i = tid; i < n; i += kSmallThreads) {
      const int32_t o = a.origin[i];
      const int64_t l = a.len[i];
      S.len[i] = l;
      S.org[i] = o;
      if (o < 0 || o >= d || l < 1) {
        atomicMin(&S.bad, i);
      } else {
        atomicAdd(&S.cnt_id[o], 1);
      }
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
  // ---- S2: identity grouping: stable sort by origin
  const int obits = 32 - __clz(d);  // covers the padding key d
  {
    uint32_t keys[ITEMS];
    int32_t vals[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int i = tid * ITEMS + j;
      keys[j] = i < n ? static_cast<uint32_t>(S.org[i]) : static_cast<uint32_t>(d);
      vals[j] = i;
    }
    typename SS::Sort(S.tmp.sort).Sort(keys, vals, 0, obits);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) S.ord_id[tid * ITEMS + j] = vals[j];
  }
  if (warp == 0) {  // offsets of the origin batches
    const int c = lane < d ? S.cnt_id[lane] : 0;
    int incl = c;
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(~0u, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane < d) S.off_id[lane] = incl - c;
    if (lane == 0) S.off_id[d] = n;
  }
  __syncthreads();
  {
    int64_t v[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int k = tid * ITEMS + j;
      v[j] = k < n ? S.len[S.ord_id[k]] : 0;
    }
    int64_t agg;
    typename SS::Scan(S.tmp.scan).ExclusiveSum(v, v, agg);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) S.pfx[tid * ITEMS + j] = v[j];
    if (tid == 0) S.pfx[SS::NS] = agg;
  }
  __syncthreads();
  for (int k = tid; k < n; k += kSmallThreads) {
    const int32_t pos = S.ord_id[k];
    const int st = S.off_id[S.org[pos]];
    a.src_slot[pos] = k - st;
    a.src_off[pos] = S.pfx[k] - S.pfx[st];
    a.src_member[k] = pos;
  }
  if (tid <= d) a.src_offset[tid] = S.off_id[tid];

  SMALL_MARK(2);
  // ---- S3..S5: the policy's own packing
  if (!a.identity_only) {
    const bool asc = a.kind == ORCH_BINARY_PADDED;
    // key bits of the longest item; ascending padding sorts after equal keys (stable sort)
    const int lbits = 32 - __clz(static_cast<unsigned>(S.maxlen));
    const uint32_t pad_asc = lbits == 32 ? 0xffffffffu : ((1u << lbits) - 1u);
    {
      uint32_t keys[ITEMS];
      int32_t vals[ITEMS];
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        const int i = tid * ITEMS + j;
        keys[j] = i < n ? static_cast<uint32_t>(S.len[i])
                        : (asc ? pad_asc : 0u);
        vals[j] = i;
      }
      __syncthreads();  // tmp storage reuse
      if (asc)
        typename SS::Sort(S.tmp.sort).Sort(keys, vals, 0, lbits);
      else
        typename SS::Sort(S.tmp.sort).SortDescending(keys, vals, 0, lbits);
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        S.ord[tid * ITEMS + j] = vals[j];
        S.xs[tid * ITEMS + j] = keys[j];
      }
    }
    __syncthreads();
    SMALL_MARK(3);
    if (a.kind == ORCH_GREEDY_UNPADDED) {
      if (warp == 0) warp_greedy<true>(S, d, 0, n, nullptr, nullptr, a.dst_off, &S.rounds);
    } else if (a.kind == ORCH_QUADRATIC_TOLERANCE) {
      if (warp == 0) {  // champion scan (balancers.cpp:223-231), d <= 32: one ballot + restarts
        if (lane < d) {
          S.qsum[lane] = 0;
          S.qsq[lane] = 0;
          S.cnt_a[lane] = 0;
        }
        __syncwarp();
        for (int k = 0; k < n; ++k) {
          int best = 0;
          int64_t bs = S.qsum[0], bq = S.qsq[0];
          int i0 = 1;
          while (i0 < d) {
            const int i = i0 + lane;
            bool c = false;
            if (i < d) {
              const int64_t as = S.qsum[i], aq = S.qsq[i];
              const int64_t df = as - bs;
              c = (df < 0 ? -df : df) < a.tol_v ? (aq < bq) : (as < bs);
            }
            const unsigned m = __ballot_sync(~0u, c);
            if (!m) break;
            best = i0 + __ffs(m) - 1;
            bs = S.qsum[best];
            bq = S.qsq[best];
            i0 = best + 1;
          }
          if (lane == 0) {
            const int64_t x = S.xs[k];
            const int32_t pos = S.ord[k];
            S.a_dest[pos] = static_cast<uint8_t>(best);
            S.a_slot[pos] = static_cast<uint16_t>(S.cnt_a[best]);
            a.dst_off[pos] = S.qsum[best];
            S.cnt_a[best] += 1;
            S.qsum[best] += x;
            S.qsq[best] += x * x;
          }
          __syncwarp();
        }
        if (lane < d) S.tok_a[lane] = S.qsum[lane];
        if (lane == 0) S.rounds = n;
      }
    } else if (a.kind == ORCH_CONVTRANSFORMER) {
      if (warp == 0) {
        // bound = greedy objective (balancers.cpp:247-256)
        warp_greedy<false>(S, d, 0, n, nullptr, nullptr, nullptr, nullptr);
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
        warp_greedy<true>(S, d, k, n, S.seed_load, S.seed_cnt, a.dst_off, &S.rounds);
      }
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
        typename SS::Scan(S.tmp.scan).ExclusiveSum(v, v, agg);
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
      while (true) {
        const int64_t lo = S.lo, hi = S.hi;
        if (lo >= hi) break;
        const int64_t span = hi - lo;
        const int64_t c = span <= 32 ? lo + warp : lo + (span * warp) / 32;
        bool f = true;
        if (c < hi) f = warp_feasible(S.xs, n, d, c, lane);
        if (lane == 0) {
          S.cand[warp] = c;
          S.feas[warp] = f;
        }
        __syncthreads();
        if (tid == 0) {
          int64_t nhi = hi, nlo = lo;
          for (int w = 0; w < 32; ++w) {
            if (S.cand[w] >= hi) continue;
            if (S.feas[w]) {
              if (S.cand[w] < nhi) nhi = S.cand[w];
            } else if (S.cand[w] + 1 > nlo) {
              nlo = S.cand[w] + 1;
            }
          }
          S.hi = nhi;
          S.lo = nlo < nhi ? nlo : nhi;
        }
        __syncthreads();
      }
      if (warp == 0) {
        const int64_t bound = S.hi;
        int64_t p = 0;
        int g = 0;
        while (p < n) {
          if (lane == 0) S.starts[g] = p;
          ++g;
          p = warp_next_start(S.xs, n, p, bound, lane);
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
        int g = 0;
        while (g + 1 < G && S.starts[g + 1] <= k) ++g;
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
    if (warp == 0) {
      const int c = lane < d ? S.cnt_a[lane] : 0;
      int incl = c;
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(~0u, incl, off);
        if (lane >= off) incl += o;
      }
      if (lane < d) S.off_a[lane] = incl - c;
      if (lane == 0) S.off_a[d] = n;
    }
    __syncthreads();
    for (int i = tid; i < n; i += kSmallThreads) {
      const int b = S.a_dest[i];
      const int sl = S.a_slot[i];
      a.dest_inst[i] = b;
      a.dest_slot[i] = sl;
      a.bin_member[S.off_a[b] + sl] = i;
    }
    if (tid <= d) a.bin_offset[tid] = S.off_a[tid];
    __syncthreads();  // bin_member (global) visible to the block
  }

  SMALL_MARK(5);
  // ---- S6: batch costs (core.cpp:91-118): warp w -> algorithm batch w, identity batch w
  for (int task = warp; task < 2 * d; task += 32) {
    const int side = task < d ? 0 : 1;  // 0 algorithm, 1 identity
    const int b = side ? task - d : task;
    if (side == 0 && a.identity_only) continue;
    const int beg = side ? S.off_id[b] : S.off_a[b];
    const int end = side ? S.off_id[b + 1] : S.off_a[b + 1];
    int64_t s = 0, mx = 0;
    unsigned long long sq = 0;
    bool inexact = false;
    for (int k = beg + lane; k < end; k += 32) {
      const int32_t pos = side ? S.ord_id[k] : a.bin_member[k];
      const int64_t l = S.len[pos];
      s += l;
      mx = l > mx ? l : mx;
      if (l >= (1ll << 26)) inexact = true;
      sq += static_cast<unsigned long long>(l) * static_cast<unsigned long long>(l);
      if (sq >= (1ull << 53)) inexact = true;
    }
    for (int off = 16; off > 0; off >>= 1) {
      s += __shfl_xor_sync(~0u, s, off);
      const int64_t om = __shfl_xor_sync(~0u, mx, off);
      mx = om > mx ? om : mx;
      sq += __shfl_xor_sync(~0u, sq, off);
    }
    inexact = __any_sync(~0u, inexact) || sq >= (1ull << 53);
    // the identity side must score under the policy cost model too
    const orch_cost_model& m = a.model;
    double sqd = static_cast<double>(sq);
    if (inexact && m.variant == ORCH_TRANSFORMER_QUADRATIC && !m.padded) {
      double acc = 0.0;
      if (lane == 0)
        for (int k = beg; k < end; ++k) {
          const double l = static_cast<double>(S.len[side ? S.ord_id[k] : a.bin_member[k]]);
          acc = rn_add(acc, rn_mul(l, l));
        }
      sqd = __shfl_sync(~0u, acc, 0);
    }
    if (lane == 0) {
      const int64_t cnt = end - beg;
      S.b_cnt[side][b] = static_cast<int32_t>(cnt);
      S.b_tok[side][b] = s;
      S.b_len[side][b] = m.padded ? cnt * mx : s;
      S.b_cost[side][b] = batch_cost(m, cnt, s, mx, sqd);
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
    sum->bound = a.identity_only ? 0 : ((a.kind == ORCH_BINARY_PADDED || a.kind == ORCH_CONVTRANSFORMER) ? S.bound : 0);
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
  SMALL_MARK(7);
}

}  // namespace
}  // namespace orchb
