// distribute_min_sum (balancers.cpp:92-107) for 32 < d <= ORCH_MAX_INSTANCES on
// one CTA: exact round-batched LPT.
//
// Each round the d bins are ranked by (load, bin index): a stable LSD radix
// sort of the loads relative to the previous round's minimum, fed in bin-index
// order so that equal loads keep the lower index first. In an LPT the loads
// stay within ~2 x_max of each other, so the relative keys take 2 passes of 8
// bits (3 or 4 for long sequences); loads >= 2^32 apart fall back to a 64-bit
// bitonic network on (load << ib | bin). With the bins ranked, the next k
// items go to ranks 0..k-1 where k is the first r with load_(r) - load_(0) >=
// x_r, exactly the choices the sequential heap makes.
//
// One sort pass: each warp owns 128 consecutive slots (4 per lane, striped),
// ranks its digits with __match_any_sync against a per-warp 256-bin histogram,
// a block scan over (digit, warp) turns the histograms into offsets, and the
// slots scatter -- stable by construction.
#pragma once

#include "balance_kernels.cuh"

namespace orchb {
namespace {

template <int kThreads>
struct LptShape {
  static constexpr int kWarps = kThreads / 32;
  static constexpr int kSlots = 4 * kThreads;        // bins + padding slots
  static constexpr int kHist = 256 * kWarps;          // [digit][warp]
};

template <int kThreads>
__host__ __device__ inline size_t lpt_smem_bytes(int d) {
  using Sh = LptShape<kThreads>;
  size_t b = sizeof(int64_t) * d;                            // load
  b += sizeof(int32_t) * d;                                  // count
  b = (b + 15) & ~size_t{15};
  b += 2 * (sizeof(uint32_t) + sizeof(uint16_t)) * Sh::kSlots;  // keys / bins, double-buffered
  b += sizeof(uint16_t) * Sh::kHist;
  b += sizeof(uint32_t) * Sh::kWarps;
  return b;
}

// exclusive scan in place over hist[kHist] (8 entries per thread)
template <int kThreads>
__device__ __forceinline__ void lpt_hist_scan(uint16_t* hist, uint32_t* wsum) {
  using Sh = LptShape<kThreads>;
  static_assert(Sh::kHist == 8 * kThreads, "8 histogram entries per thread");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v[8];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = hist[8 * threadIdx.x + q];
    s += v[q];
  }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < Sh::kWarps ? wsum[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(~0u, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < Sh::kWarps) wsum[lane] = wi - w;
  }
  __syncthreads();
  uint32_t ex = wsum[warp] + incl - s;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    hist[8 * threadIdx.x + q] = static_cast<uint16_t>(ex);
    ex += v[q];
  }
  __syncthreads();
}

// one stable pass on the 8-bit digit at `shift`: (kin, vin) -> (kout, vout)
template <int kThreads>
__device__ __forceinline__ void lpt_sort_pass(const uint32_t* kin, const uint16_t* vin,
                                              uint32_t* kout, uint16_t* vout, uint16_t* hist,
                                              uint32_t* wsum, int shift) {
  using Sh = LptShape<kThreads>;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < Sh::kHist; i += kThreads) hist[i] = 0;
  __syncthreads();
  uint32_t key[4];
  uint16_t val[4];
  int dig[4], rank[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = warp * 128 + j * 32 + lane;
    key[j] = kin[i];
    val[j] = vin[i];
    dig[j] = static_cast<int>((key[j] >> shift) & 255u);
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const unsigned peers = __match_any_sync(~0u, dig[j]);
    const int before = __popc(peers & lt);
    uint16_t* h = hist + dig[j] * Sh::kWarps + warp;
    const int base = *h;
    rank[j] = base + before;
    __syncwarp();
    if (before == 0) *h = static_cast<uint16_t>(base + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  lpt_hist_scan<kThreads>(hist, wsum);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int pos = hist[dig[j] * Sh::kWarps + warp] + rank[j];
    kout[pos] = key[j];
    vout[pos] = val[j];
  }
  __syncthreads();
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads, 1)
    k_greedy_lpt(int d, int64_t n, const int64_t* __restrict__ d_first,
                 const uint32_t* __restrict__ xs, const int32_t* __restrict__ order,
                 const int64_t* __restrict__ init_load, const int32_t* __restrict__ init_count,
                 int32_t* __restrict__ dest_inst, int32_t* __restrict__ dest_slot,
                 int64_t* __restrict__ dst_off, int32_t* __restrict__ bin_count,
                 int64_t* __restrict__ bin_tokens, orch_summary* s,
                 int32_t* __restrict__ s_bin, int32_t* __restrict__ s_slot,
                 int64_t* __restrict__ s_off) {
  // s_bin given: results go out by SORTED position (coalesced stores from the
  // one SM; k_lpt_scatter moves them to input positions on every SM) -- the
  // scattered per-item stores were half of a round's time at d = 2560
  using Sh = LptShape<kThreads>;
  if (pipeline_failed(s)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t* load = reinterpret_cast<int64_t*>(smem_raw);
  int32_t* cnt = reinterpret_cast<int32_t*>(load + d);
  unsigned char* p = smem_raw + ((sizeof(int64_t) * d + sizeof(int32_t) * d + 15) & ~size_t{15});
  uint32_t* kA = reinterpret_cast<uint32_t*>(p);
  uint32_t* kB = kA + Sh::kSlots;
  uint16_t* vA = reinterpret_cast<uint16_t*>(kB + Sh::kSlots);
  uint16_t* vB = vA + Sh::kSlots;
  uint16_t* hist = vB + Sh::kSlots;
  uint32_t* wsum = reinterpret_cast<uint32_t*>(hist + Sh::kHist);
  uint64_t* wide = reinterpret_cast<uint64_t*>(kA);  // fallback keys alias the key buffers
  __shared__ int s_k;
  __shared__ unsigned s_max;
  __shared__ int s_wide;
  __shared__ unsigned long long s_min;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  unsigned ib = 0;
  while ((1u << ib) < static_cast<unsigned>(d)) ++ib;

  if (tid == 0) s_min = ~0ull;
  __syncthreads();
  for (int b = tid; b < d; b += kThreads) {
    load[b] = init_load ? init_load[b] : 0;
    cnt[b] = init_count ? init_count[b] : 0;
    atomicMin(&s_min, static_cast<unsigned long long>(load[b]));
  }
  __syncthreads();
  int64_t base = static_cast<int64_t>(s_min);
  int64_t next = d_first ? *d_first : 0;
  int64_t rounds = 0;
#ifdef ORCH_SMALL_PROFILE
  // diagnostics build: cycles per round stage, summed over the rounds
  long long prof[5] = {0, 0, 0, 0, 0}, t_prev = clock64();
#define LPT_STAGE(i)                       \
  do {                                     \
    const long long t_ = clock64();        \
    prof[i] += t_ - t_prev;                \
    t_prev = t_;                           \
  } while (0)
#else
#define LPT_STAGE(i) \
  do {               \
  } while (0)
#endif
  constexpr int kPer = Sh::kSlots / kThreads;  // round slots r = tid + i * kThreads
  while (next < n) {
    const int m = static_cast<int>(n - next < d ? n - next : d);
    // this round's candidate items, fetched now so the L2 latency hides behind the sort
    // (raw 32-bit registers, predicated loads: nothing consumes them before
    // the k search, so the key build and sort run while they are in flight --
    // a conversion or select here made every round wait ~1.2k cycles for them)
    uint32_t xr[kPer];
    int32_t pr[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int r = tid + i * kThreads;
      xr[i] = 0u;
      pr[i] = 0;
      if (r < m) {
        xr[i] = xs[next + r];
        if (!s_bin) pr[i] = order[next + r];
      }
    }
    // ---- rank the bins by (load, index)
    if (tid == 0) {
      s_max = 0;
      s_wide = 0;
      s_k = m;
    }
    __syncthreads();
    LPT_STAGE(4);
    unsigned mx = 0;
    bool wd = false;
    for (int i = tid; i < Sh::kSlots; i += kThreads) {
      uint32_t key = 0xffffffffu;
      if (i < d) {
        const int64_t rel = load[i] - base;  // >= 0: loads only grow, base was a minimum
        if (rel >= 0xffffffffll) wd = true;
        key = rel >= 0xffffffffll ? 0xfffffffeu : static_cast<uint32_t>(rel);
        mx = key > mx ? key : mx;
      }
      kA[i] = key;
      vA[i] = static_cast<uint16_t>(i);
    }
    mx = __reduce_max_sync(~0u, mx);
    if (__any_sync(~0u, wd) && lane == 0) s_wide = 1;
    if (lane == 0) atomicMax(&s_max, mx);
    __syncthreads();
    LPT_STAGE(0);
    const uint16_t* rank_bin;
    if (!s_wide) {
      const int bits = s_max ? 32 - __clz(s_max) : 1;
      const int passes = (bits + 7) >> 3;
      uint32_t *ki = kA, *ko = kB;
      uint16_t *vi = vA, *vo = vB;
      for (int ps = 0; ps < passes; ++ps) {
        lpt_sort_pass<kThreads>(ki, vi, ko, vo, hist, wsum, 8 * ps);
        uint32_t* tk = ki;
        ki = ko;
        ko = tk;
        uint16_t* tv = vi;
        vi = vo;
        vo = tv;
      }
      rank_bin = vi;
    } else {  // loads 2^32 apart: 64-bit (load << ib | bin) keys, bitonic network
      int p2 = 32;
      while (p2 < d) p2 <<= 1;
      for (int i = tid; i < p2; i += kThreads)
        wide[i] = i < d ? (static_cast<uint64_t>(load[i]) << ib) | static_cast<uint64_t>(i) : kU64Max;
      __syncthreads();
      block_bitonic<kThreads>(wide, p2);
      uint16_t* out = vB;  // vB does not alias wide[0, p2): p2 * 8 <= 2 * 4 * kSlots
      for (int i = tid; i < d; i += kThreads)
        out[i] = static_cast<uint16_t>(wide[i] & ((1ull << ib) - 1));
      __syncthreads();
      rank_bin = out;
    }
    LPT_STAGE(1);
    // ---- k = first rank r with load_(r) - load_(0) >= x_r
    const int64_t L0 = load[rank_bin[0]];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int r0 = warp * 32 + i * kThreads, r = r0 + lane;
      if (r0 >= m) break;
      const bool bad = r < m && !(load[rank_bin[r]] - L0 < static_cast<int64_t>(xr[i]));
      const unsigned bm = __ballot_sync(~0u, bad);
      if (bm) {
        if (lane == 0) atomicMin(&s_k, r0 + __ffs(bm) - 1);
        break;  // later chunks of this warp only hold larger r
      }
    }
    __syncthreads();
    LPT_STAGE(2);
    const int k = s_k;  // >= 1: x_0 >= 1 > 0 = load_(0) - load_(0)
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int r = tid + i * kThreads;
      if (r < k) {
        const int b = rank_bin[r];  // distinct bins within a round
        if (s_bin) {
          const int64_t q = next + r;
          s_bin[q] = b;
          s_slot[q] = cnt[b];
          s_off[q] = load[b];
        } else {
          const int32_t pos = pr[i];
          dest_inst[pos] = b;
          dest_slot[pos] = cnt[b];
          dst_off[pos] = load[b];
        }
        ++cnt[b];
        load[b] += static_cast<int64_t>(xr[i]);
      }
    }
    __syncthreads();
    LPT_STAGE(3);
    base = L0;
    next += k;
    ++rounds;
  }
#ifdef ORCH_SMALL_PROFILE
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) g_small_prof[8 + i] = prof[i];
    g_small_prof[12] = rounds;
    g_small_prof[13] = prof[4];
  }
#endif
#undef LPT_STAGE
  for (int b = tid; b < d; b += kThreads) {
    bin_tokens[b] = load[b];
    bin_count[b] = cnt[b];
  }
  if (tid == 0) s->rounds = rounds;
}

// Sorted-position results of k_greedy_lpt -> input positions.
__global__ void k_lpt_scatter(int64_t n, const int64_t* __restrict__ d_first,
                              const int32_t* __restrict__ order, const int32_t* __restrict__ s_bin,
                              const int32_t* __restrict__ s_slot, const int64_t* __restrict__ s_off,
                              int32_t* __restrict__ dest_inst, int32_t* __restrict__ dest_slot,
                              int64_t* __restrict__ dst_off, orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int64_t f = d_first ? *d_first : 0;
  for (int64_t k = f + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t pos = order[k];
    dest_inst[pos] = s_bin[k];
    dest_slot[pos] = s_slot[k];
    dst_off[pos] = s_off[k];
  }
}

}  // namespace
}  // namespace orchb
