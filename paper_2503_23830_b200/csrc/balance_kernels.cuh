// sm_100a kernels of the Post-Balancing algorithms (balancers.cpp). Integer
// work is exact; double cost arithmetic goes through explicitly rounded
// intrinsics (common.cuh) so results are bit-identical to the reference's
// non-FMA build.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace orchb {
namespace {  // internal linkage: included by several translation units

constexpr uint64_t kU64Max = ~0ull;

// Workspace flags shared by the pipeline kernels of one balance call.
struct Flags {
  unsigned long long first_bad;  // min input position failing index_sources checks
  unsigned int unsupported;      // a device limit was exceeded
  unsigned int pad;
  unsigned long long total_tokens;
};

__device__ __forceinline__ bool pipeline_failed(const orch_summary* s) { return s->error != 0; }

// ---------------------------------------------------------------- K1
// index_sources checks (balancers.cpp:25-37): origin in [0,d), length >= 1,
// reported for the FIRST offending input position. Also emits the radix-sort
// keys (length, origin) and identity values, and the token total.
__global__ void k_validate(int d, int64_t n, const int64_t* __restrict__ len,
                           const int32_t* __restrict__ origin, uint32_t* __restrict__ key_len,
                           uint32_t* __restrict__ key_org, int32_t* __restrict__ iota,
                           Flags* flags) {
  unsigned long long local_tokens = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = origin[i];
    const int64_t l = len[i];
    if (o < 0 || o >= d || l < 1) atomicMin(&flags->first_bad, (unsigned long long)i);
    if (l > ORCH_MAX_LENGTH) atomicOr(&flags->unsupported, 1u);
    key_len[i] = static_cast<uint32_t>(l);
    key_org[i] = static_cast<uint32_t>(o);
    iota[i] = static_cast<int32_t>(i);
    local_tokens += l > 0 ? static_cast<unsigned long long>(l) : 0ull;
  }
  // warp-aggregate the token total, one atomic per warp
  for (int off = 16; off > 0; off >>= 1) local_tokens += __shfl_xor_sync(~0u, local_tokens, off);
  if ((threadIdx.x & 31) == 0 && local_tokens) atomicAdd(&flags->total_tokens, local_tokens);
}

// Turns the flags into the summary's error (reference error first).
__global__ void k_validate_finish(int64_t n, const Flags* flags, orch_summary* s) {
  if (flags->first_bad < static_cast<unsigned long long>(n)) {
    s->error = ORCH_INVALID_ARGUMENT;
    s->error_index = static_cast<int64_t>(flags->first_bad);
  } else if (flags->unsupported || flags->total_tokens >= (1ull << 50)) {
    s->error = ORCH_UNSUPPORTED;
  }
}

// ---------------------------------------------------------------- K2
// Identity grouping (group_by_origin balancers.cpp:62-66 / batches_from_items
// core.cpp:183-199): items sorted stably by origin. Counts per origin and the
// lengths in that order (for the segmented token prefix).
__global__ void k_ident_count(int64_t n, const int32_t* __restrict__ ident_order,
                              const int32_t* __restrict__ origin, const int64_t* __restrict__ len,
                              int32_t* __restrict__ ident_count, int64_t* __restrict__ ident_len,
                              const orch_summary* s) {
  if (pipeline_failed(s)) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pos = ident_order[k];
    ident_len[k] = len[pos];
    // run-length aware: one atomic per run of equal origins inside the warp
    const int32_t o = origin[pos];
    atomicAdd(&ident_count[o], 1);
  }
}

// src_slot / src_off per item from the identity order (index_sources slot =
// running count per origin in input order; token offset = running sum).
__global__ void k_ident_slots(int64_t n, const int32_t* __restrict__ ident_order,
                              const int32_t* __restrict__ origin,
                              const int32_t* __restrict__ ident_offset,
                              const int64_t* __restrict__ ident_prefix,
                              int32_t* __restrict__ src_slot, int64_t* __restrict__ src_off,
                              const orch_summary* s) {
  if (pipeline_failed(s)) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pos = ident_order[k];
    const int32_t start = ident_offset[origin[pos]];
    src_slot[pos] = static_cast<int32_t>(k - start);
    src_off[pos] = ident_prefix[k] - ident_prefix[start];
  }
}

// ---------------------------------------------------------------- K4a
// distribute_min_sum (balancers.cpp:92-107) for d <= 32: one warp, lane b
// owns bin b; per item a butterfly argmin over the packed key
// (load << 5 | lane) == lexicographic (sum, batch index): lowest index wins
// ties exactly like the reference's priority_queue of (sum, idx) pairs.
// Items arrive in descending order (xs/order from the stable radix sort);
// [first, n) is processed, bins may be pre-seeded (init_load/init_count).
__global__ void k_greedy_warp(int d, int64_t n, const int64_t* __restrict__ d_first,
                              const uint32_t* __restrict__ xs, const int32_t* __restrict__ order,
                              const int64_t* __restrict__ init_load,
                              const int32_t* __restrict__ init_count,
                              int32_t* __restrict__ dest_inst, int32_t* __restrict__ dest_slot,
                              int64_t* __restrict__ dst_off, int32_t* __restrict__ bin_count,
                              int64_t* __restrict__ bin_tokens, orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int lane = threadIdx.x;
  int width = 1;
  while (width < d) width <<= 1;
  int64_t load = 0;
  int32_t cnt = 0;
  if (lane < d) {
    load = init_load ? init_load[lane] : 0;
    cnt = init_count ? init_count[lane] : 0;
  }
  const uint64_t mine_valid = lane < d;
  const int64_t first = d_first ? *d_first : 0;
  for (int64_t base = first; base < n; base += 32) {
    const int64_t my = base + lane;
    const int64_t myx = my < n ? static_cast<int64_t>(xs[my]) : 0;
    const int32_t mypos = my < n ? order[my] : 0;
    const int m = static_cast<int>(n - base < 32 ? n - base : 32);
    for (int j = 0; j < m; ++j) {
      const int64_t x = __shfl_sync(~0u, myx, j);
      const int32_t pos = __shfl_sync(~0u, mypos, j);
      uint64_t key = mine_valid ? ((static_cast<uint64_t>(load) << 5) | lane) : kU64Max;
      for (int off = width >> 1; off > 0; off >>= 1) {
        const uint64_t other = __shfl_xor_sync(~0u, key, off);
        key = other < key ? other : key;
      }
      if (mine_valid && static_cast<int>(key & 31u) == lane) {
        dest_inst[pos] = lane;
        dest_slot[pos] = cnt++;
        dst_off[pos] = load;
        load += x;
      }
    }
  }
  if (lane < d) {
    bin_count[lane] = cnt;
    bin_tokens[lane] = load;
  }
  if (lane == 0) s->rounds = n - first;
}

// Block-wide ascending bitonic sort of p (power of two) 64-bit keys in shared
// memory. Stages with stride >= 32 exchange through shared memory (one
// barrier each); the strides 16..1 of every size run in registers with warp
// shuffles, so a 4096-key sort takes 36 barriers instead of 78.
template <int kThreads>
__device__ void block_bitonic(uint64_t* U, int p) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  auto reg_stages = [&](int size_lo, int size_hi) {  // sizes size_lo..size_hi, strides < 32
    for (int blk = warp; blk * 32 < p; blk += kWarps) {
      const int i = blk * 32 + lane;
      uint64_t key = U[i];
      for (int size = size_lo; size <= size_hi; size <<= 1)
        for (int stride = (size > 32 ? 16 : size >> 1); stride > 0; stride >>= 1) {
          const uint64_t other = __shfl_xor_sync(~0u, key, stride);
          const bool up = (i & size) == 0;
          const bool lower = (i & stride) == 0;
          const uint64_t lo = other < key ? other : key;
          const uint64_t hi = other < key ? key : other;
          key = (lower == up) ? lo : hi;
        }
      U[i] = key;
    }
  };
  if (p <= 1) return;
  if (p < 32) {  // tiny: plain shared-memory network
    for (int size = 2; size <= p; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < (p >> 1); i += kThreads) {
          const int lo = 2 * stride * (i / stride) + (i % stride);
          const int hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint64_t a = U[lo], b = U[hi];
          if ((a > b) == up) {
            U[lo] = b;
            U[hi] = a;
          }
        }
        __syncthreads();
      }
    return;
  }
  reg_stages(2, 32);
  __syncthreads();
  for (int size = 64; size <= p; size <<= 1) {
    for (int stride = size >> 1; stride >= 32; stride >>= 1) {
      for (int i = threadIdx.x; i < (p >> 1); i += kThreads) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = U[lo], b = U[hi];
        if ((a > b) == up) {
          U[lo] = b;
          U[hi] = a;
        }
      }
      __syncthreads();
    }
    reg_stages(size, size);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K6
// Quadratic tolerance greedy (balancers.cpp:210-233). The comparator is not
// transitive, so the reference's left-to-right champion scan is reproduced
// exactly: starting from the current champion, a warp tests the next 32
// candidates at once and the FIRST one that beats the champion becomes the
// new champion (what the sequential scan does), continuing after it.
__global__ void k_quadtol(int d, int64_t n, int64_t v, const uint32_t* __restrict__ xs,
                          const int32_t* __restrict__ order, int32_t* __restrict__ dest_inst,
                          int32_t* __restrict__ dest_slot, int64_t* __restrict__ dst_off,
                          int32_t* __restrict__ bin_count, int64_t* __restrict__ bin_tokens,
                          orch_summary* s) {
  if (pipeline_failed(s)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t* sum = reinterpret_cast<int64_t*>(smem_raw);
  int64_t* sq = sum + d;
  int32_t* cnt = reinterpret_cast<int32_t*>(sq + d);
  const int lane = threadIdx.x;
  for (int i = lane; i < d; i += 32) {
    sum[i] = 0;
    sq[i] = 0;
    cnt[i] = 0;
  }
  __syncwarp();
  for (int64_t k = 0; k < n; ++k) {
    int best = 0;
    int64_t bs = sum[0], bq = sq[0];
    int i0 = 1;
    while (i0 < d) {
      const int i = i0 + lane;
      bool c = false;
      if (i < d) {
        const int64_t as = sum[i], aq = sq[i];
        const int64_t diff = as - bs;
        const int64_t ad = diff < 0 ? -diff : diff;
        c = ad < v ? (aq < bq) : (as < bs);  // tolerance_less :151-154
      }
      const unsigned m = __ballot_sync(~0u, c);
      if (m) {
        best = i0 + __ffs(m) - 1;
        bs = sum[best];
        bq = sq[best];
        i0 = best + 1;
      } else {
        i0 += 32;
      }
    }
    if (lane == 0) {
      const int64_t x = xs[k];
      const int32_t pos = order[k];
      dest_inst[pos] = best;
      dest_slot[pos] = cnt[best]++;
      dst_off[pos] = sum[best];
      sum[best] += x;
      sq[best] += x * x;
    }
    __syncwarp();
  }
  for (int i = lane; i < d; i += 32) {
    bin_count[i] = cnt[i];
    bin_tokens[i] = sum[i];
  }
}

// ---------------------------------------------------------------- K5
// BinaryPadded (Alg. 2, balancers.cpp:111-143,194-208). Ascending lengths a[]
// (stable radix sort). next_start(p, b): GetLeastBatches closes the group that
// starts at p at the first idx with (idx - p + 1) * a[idx] > b; both factors
// are nondecreasing in idx, so the predicate is monotone and a warp finds the
// boundary by galloping + 32-ary search.
__device__ __forceinline__ int64_t warp_next_start(const uint32_t* __restrict__ a, int64_t n,
                                                   int64_t p, int64_t b, int lane) {
  // cond(t) = t >= n || (t - p + 1) * a[t] > b ; cond(p) is false (a[p] <= max <= b)
  int64_t lo = p, step = 1;
  int64_t hi = n;
  for (;;) {  // gallop
    const int64_t t = lo + step * (lane + 1);
    const bool c = t >= n || (t - p + 1) * static_cast<int64_t>(a[t]) > b;
    const unsigned m = __ballot_sync(~0u, c);
    if (m) {
      const int f = __ffs(m) - 1;
      hi = lo + step * (f + 1);
      if (hi > n) hi = n;
      lo = lo + step * f;  // the probe before (or lo itself) is false
      break;
    }
    lo = lo + step * 32;
    step *= 32;
  }
  while (hi - lo > 1) {  // invariant: cond(lo) false, cond(hi) true
    const int64_t span = hi - lo;
    const int64_t st = (span + 31) / 32;
    const int64_t t = lo + st * (lane + 1);
    const bool c = t >= hi || (t - p + 1) * static_cast<int64_t>(a[t]) > b;
    const unsigned m = __ballot_sync(~0u, c);
    const int f = __ffs(m) - 1;  // m != 0: lane 31 probes >= hi
    const int64_t nhi = lo + st * (f + 1);
    hi = nhi < hi ? nhi : hi;
    lo = lo + st * f;
  }
  return hi;
}

// One thread: next_start from p with a guess h of the group size. Probe
// t = p + h - 1: if cond(t) is false the boundary is beyond t (gallop from t),
// else it is in (p, t] (bisect). Sizes change slowly along ascending lengths,
// so the guess is usually within a step or two.
__device__ __forceinline__ int64_t thread_next_start_hint(const uint32_t* a, int64_t n, int64_t p,
                                                          int64_t b, int64_t h) {
  auto cond = [&](int64_t t) { return t >= n || (t - p + 1) * static_cast<int64_t>(a[t]) > b; };
  int64_t lo = p, hi;
  const int64_t g = h > 1 ? p + h - 1 : p + 1;
  if (cond(g)) {
    hi = g;
    if (g - 1 > p && !cond(g - 1)) return g;  // the guess was exact
  } else {
    lo = g;
    int64_t k = 1;
    for (;; k <<= 1) {
      const int64_t t = g + k;
      if (cond(t)) {
        hi = t < n ? t : n;
        break;
      }
      lo = t;
    }
  }
  while (hi - lo > 1) {  // cond(lo) false (lo == p or probed), cond(hi) true
    const int64_t t = lo + ((hi - lo) >> 1);
    if (cond(t)) hi = t;
    else lo = t;
  }
  return hi;
}

// One thread: is bound b feasible (at most d groups)?
__device__ __forceinline__ bool thread_feasible(const uint32_t* a, int64_t n, int d, int64_t b) {
  int64_t p = 0, size = 0;
  for (int groups = 0; p < n; ++groups) {
    if (groups == d) return false;
    const int64_t q = thread_next_start_hint(a, n, p, b, size);
    size = q - p;
    p = q;
  }
  return true;
}

// warp_next_start with a guess of the group size (the previous group's: sizes
// change slowly along ascending lengths). One ballot over the 32 starts
// around the guess settles most groups; otherwise the boundary is bracketed by
// the window and finished by 32-ary search (or the plain gallop).
__device__ __forceinline__ int64_t warp_next_start_hint(const uint32_t* __restrict__ a, int64_t n,
                                                        int64_t p, int64_t b, int lane,
                                                        int64_t size_hint) {
  if (size_hint <= 16) return warp_next_start(a, n, p, b, lane);
  const int64_t base = p + size_hint - 16;  // > p
  const int64_t t = base + lane;
  const bool c = t >= n || (t - p + 1) * static_cast<int64_t>(a[t]) > b;
  const unsigned m = __ballot_sync(~0u, c);
  int64_t lo, hi;
  if (m & 1u) {  // boundary in (p, base]: cond(p) false, cond(base) true
    lo = p;
    hi = base;
  } else if (m) {
    return base + (__ffs(m) - 1);  // cond(base + f - 1) false, cond(base + f) true
  } else {  // past the window: gallop from base + 31 (false)
    lo = base + 31;
    int64_t step = 1;
    for (;;) {
      const int64_t tt = lo + step * (lane + 1);
      const bool cc = tt >= n || (tt - p + 1) * static_cast<int64_t>(a[tt]) > b;
      const unsigned mm = __ballot_sync(~0u, cc);
      if (mm) {
        const int f = __ffs(mm) - 1;
        hi = lo + step * (f + 1);
        if (hi > n) hi = n;
        lo = lo + step * f;
        break;
      }
      lo = lo + step * 32;
      step *= 32;
    }
  }
  while (hi - lo > 1) {  // invariant: cond(lo) false, cond(hi) true
    const int64_t span = hi - lo;
    const int64_t st = (span + 31) / 32;
    const int64_t tt = lo + st * (lane + 1);
    const bool cc = tt >= hi || (tt - p + 1) * static_cast<int64_t>(a[tt]) > b;
    const unsigned mm = __ballot_sync(~0u, cc);
    const int f = __ffs(mm) - 1;
    const int64_t nhi = lo + st * (f + 1);
    hi = nhi < hi ? nhi : hi;
    lo = lo + st * f;
  }
  return hi;
}

__device__ __forceinline__ bool warp_feasible(const uint32_t* __restrict__ a, int64_t n, int d,
                                              int64_t b, int lane) {
  int64_t p = 0, size = 0;
  int groups = 0;
  while (p < n) {
    if (++groups > d) return false;
    const int64_t q = warp_next_start_hint(a, n, p, b, lane, size);
    size = q - p;
    p = q;
  }
  return true;
}

// One CTA of 32 warps: k-ary search for the minimal feasible bound in
// [max, max * (n/d + 1)] (feasibility is monotone in b), then the
// group starts at that bound. mode 0: search; mode 1: feasibility of `bound`.
__global__ void __launch_bounds__(1024, 1)
    k_padded_search(int d, int64_t n, const uint32_t* __restrict__ a_global, int mode, int64_t probe,
                    int64_t* __restrict__ starts, int32_t* __restrict__ n_groups,
                    int64_t* __restrict__ out_bound, orch_summary* s, int smem_items) {
  if (pipeline_failed(s)) return;
  __shared__ int64_t cand[32];
  __shared__ int feas[32];
  __shared__ int64_t s_lo, s_hi;
  extern __shared__ __align__(16) uint32_t a_smem[];
  // The galloping group scans probe a[] ~d times per candidate: keep the
  // ascending lengths in shared memory when they fit (L2 latency -> ~30 cycles).
  const uint32_t* a = a_global;
  if (n <= smem_items) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a_smem[i] = a_global[i];
    __syncthreads();
    a = a_smem;
  }
  // warp index through a shuffle: provably warp-uniform, so the warp-collective
  // code below compiles without WARPSYNC.COLLECTIVE divergence handling
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int64_t max_len = a[n - 1];
  if (mode == 1) {
    if (warp == 0) {
      const bool f = probe >= max_len && warp_feasible(a, n, d, probe, lane);
      if (lane == 0) *n_groups = f ? 1 : 0;
    }
    return;
  }
  if (threadIdx.x == 0) {
    s_lo = max_len;
    s_hi = max_len * (n / d + 1);  // always feasible (proof in DESIGN.md)
  }
  __syncthreads();
  while (true) {
    const int64_t lo = s_lo, hi = s_hi;
    if (lo >= hi) break;
    const int64_t span = hi - lo;
    const int64_t c = span <= 32 ? lo + warp : lo + (span * warp) / 32;
    if (lane == 0) cand[warp] = c;
    bool f = true;
    if (c < hi) f = warp_feasible(a, n, d, c, lane);
    if (lane == 0) feas[warp] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t nhi = hi, nlo = lo;
      for (int w = 0; w < 32; ++w) {
        if (cand[w] >= hi) continue;
        if (feas[w]) {
          if (cand[w] < nhi) nhi = cand[w];
        } else if (cand[w] + 1 > nlo) {
          nlo = cand[w] + 1;
        }
      }
      s_hi = nhi;
      s_lo = nlo < nhi ? nlo : nhi;
    }
    __syncthreads();
  }
  const int64_t bound = s_hi;
  if (warp == 0) {  // group starts at the minimal bound
    int64_t p = 0;
    int g = 0;
    while (p < n) {
      if (lane == 0) starts[g] = p;
      ++g;
      p = warp_next_start(a, n, p, bound, lane);
    }
    if (lane == 0) {
      starts[g] = n;
      *n_groups = g;
      *out_bound = bound;
      s->bound = bound;
    }
  }
}

// Multi-SM k-ary search (general path). Every round G = 148 CTAs evaluate G
// candidate bounds, one per SM. A CTA does not walk the group chain warp-
// serially (one galloping search per group, ~300 cycles each): it builds the
// successor table nx[p] = next_start(p) for EVERY p in parallel (1024 threads,
// coalesced gallops over a[]), squares it three times in place into
// nx8 = next^8, and walks nx8 from 0 — d/8 shared-memory hops. Feasibility is
// monotone in the bound, so the last CTA to finish narrows [lo, hi] (hi stays
// feasible); the span shrinks ~G-fold per round and kPadRounds covers any
// 2^56 span. Tables are u16 deltas (kNxFar = group of >= 65535 items: the
// walker falls back to a galloping search there); n > kNxMax uses the
// one-warp-per-candidate scan instead.
constexpr int kPadRounds = 9;
constexpr int kNxMax = 100 * 1024;  // u16 table in 200 KiB of shared memory
constexpr uint16_t kNxFar = 0xFFFF;
struct PadSearch {
  int64_t lo, hi;
  unsigned done;  // CTAs finished this round (last-block-done narrowing)
};

__global__ void k_pad_init(int d, int64_t n, const uint32_t* __restrict__ a, PadSearch* st,
                           const orch_summary* s) {
  if (pipeline_failed(s) || threadIdx.x != 0) return;
  const int64_t max_len = a[n - 1];
  st->lo = max_len;
  st->hi = max_len * (n / d + 1);  // always feasible
  st->done = 0;
}

// next_start for one thread: gallop then bisect on cond(t) = t >= n ||
// (t - p + 1) * a[t] > b (monotone in t), starting after `from` (p <= from,
// cond(from) known false; from = p always qualifies since a[p] <= b).
__device__ __forceinline__ int64_t thread_next_start(const uint32_t* __restrict__ a, int64_t n,
                                                     int64_t p, int64_t b, int64_t from) {
  int64_t lo = from, hi, k = 1;
  for (;; k <<= 1) {
    const int64_t t = from + k;
    if (t >= n || (t - p + 1) * static_cast<int64_t>(__ldg(a + t)) > b) {
      hi = t < n ? t : n;
      break;
    }
    lo = t;
  }
  while (hi - lo > 1) {
    const int64_t t = lo + ((hi - lo) >> 1);
    if ((t - p + 1) * static_cast<int64_t>(__ldg(a + t)) > b) hi = t;
    else lo = t;
  }
  return hi;
}

// nx (and optionally a global copy nx1) then nx8 in place. Phase 2 handles
// ascending chunks of blockDim positions and reads only positions >= the
// chunk start, which the chunk has not overwritten yet.
// Phase 1: next(p) is nondecreasing in p (a later start closes its group no
// earlier), so each thread takes a contiguous block of starts and searches
// each from the previous answer: ~1-2 loads per start instead of a fresh
// gallop + bisect (~10 dependent loads).
__device__ void build_nx8(const uint32_t* __restrict__ a, int64_t n, int64_t b, uint16_t* nx,
                          uint16_t* __restrict__ nx1) {
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t p0 = threadIdx.x * per, p1 = p0 + per < n ? p0 + per : n;
  int64_t e = p0;  // next(p - 1); cond_p(e - 1) is false for every p > p0 (weaker predicate)
  for (int64_t p = p0; p < p1; ++p) {
    e = thread_next_start(a, n, p, b, e - 1 > p ? e - 1 : p);
    const int64_t dl = e - p;
    const uint16_t v = dl < kNxFar ? static_cast<uint16_t>(dl) : kNxFar;
    nx[p] = v;
  }
  __syncthreads();
  if (nx1)  // coalesced copy of the single-step table (the squaring below rewrites nx)
    for (int64_t p = threadIdx.x; p < n; p += blockDim.x) nx1[p] = nx[p];
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const int64_t p = c0 + threadIdx.x;
    uint16_t v = kNxFar;
    if (p < n) {
      int64_t q = p;
      bool far = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (q < n) {
          const uint16_t sv = nx[q];
          if (sv == kNxFar) far = true;
          if (!far) q += sv;
        }
      }
      const int64_t dl = q - p;
      if (!far && dl < kNxFar) v = static_cast<uint16_t>(dl);
    }
    __syncthreads();
    if (p < n) nx[p] = v;
    __syncthreads();
  }
}

// Warp 0: group count at bound b by nx8 hops (8 full groups each) plus single
// galloping steps where a hop is far or would reach n. Stops once > d.
// heads/starts (optional): records each group start and the indices g of the
// 8-hop heads, for the parallel fill in k_pad_starts2.
__device__ int warp_walk_nx8(const uint32_t* __restrict__ a, int64_t n, int d, int64_t b,
                             const uint16_t* nx8, int lane, int64_t* __restrict__ starts,
                             int32_t* heads, int* n_heads) {
  int64_t p = 0;
  int g = 0, m = 0;
  while (p < n) {
    const uint16_t v = nx8[p];
    if (starts && lane == 0) starts[g] = p;
    if (v != kNxFar && p + v < n) {
      if (heads && lane == 0) heads[m] = g;
      ++m;
      g += 8;
      p += v;
    } else {
      g += 1;
      p = warp_next_start(a, n, p, b, lane);
    }
    if (g > d && !starts) return g;
  }
  if (n_heads) *n_heads = m;
  return g;
}

// Last CTA of the round: lanes of warp 0 reduce min feasible / max infeasible.
__device__ void pad_narrow_last(PadSearch* st, const int32_t* feas, const int64_t* cand, int G,
                                int64_t lo, int64_t hi) {
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&st->done, 1u) == static_cast<unsigned>(G - 1);
  }
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  __threadfence();
  int64_t nhi = hi, mx = lo - 1;
  for (int w = threadIdx.x; w < G; w += 32) {
    const int64_t c = __ldcg(cand + w);
    if (c >= hi) continue;
    if (__ldcg(feas + w)) nhi = c < nhi ? c : nhi;
    else mx = c > mx ? c : mx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t h2 = __shfl_xor_sync(~0u, nhi, o), m2 = __shfl_xor_sync(~0u, mx, o);
    nhi = h2 < nhi ? h2 : nhi;
    mx = m2 > mx ? m2 : mx;
  }
  if (threadIdx.x == 0) {
    const int64_t nlo = mx + 1 > lo ? mx + 1 : lo;
    st->hi = nhi;
    st->lo = nlo < nhi ? nlo : nhi;
    st->done = 0;
  }
}

__device__ __forceinline__ int64_t pad_candidate(int64_t lo, int64_t hi, int G, int b) {
  const int64_t span = hi - lo;
  return span <= G ? lo + b : lo + (span / G) * b + ((span % G) * b) / G;
}

// One CTA (1024 threads) per candidate; mode 1 = feasibility of `probe` only.
__global__ void __launch_bounds__(1024, 1)
    k_pad_eval_nx(int d, int64_t n, const uint32_t* __restrict__ a, PadSearch* st,
                  int32_t* __restrict__ feas, int64_t* __restrict__ cand, int mode, int64_t probe,
                  int32_t* __restrict__ probe_out, const orch_summary* s) {
  if (pipeline_failed(s)) return;
  extern __shared__ __align__(16) uint16_t nx[];
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0);
  if (mode == 1) {
    const bool ok = probe >= static_cast<int64_t>(a[n - 1]);
    if (ok) build_nx8(a, n, probe, nx, nullptr);
    if (warp == 0) {
      const bool f = ok && warp_walk_nx8(a, n, d, probe, nx, lane, nullptr, nullptr, nullptr) <= d;
      if (lane == 0) *probe_out = f ? 1 : 0;
    }
    return;
  }
  const int64_t lo = st->lo, hi = st->hi;
  if (lo >= hi) return;
  const int G = gridDim.x;
  const int64_t c = pad_candidate(lo, hi, G, blockIdx.x);
  if (c < hi) {
    build_nx8(a, n, c, nx, nullptr);
    if (warp == 0) {
      const bool f = warp_walk_nx8(a, n, d, c, nx, lane, nullptr, nullptr, nullptr) <= d;
      if (lane == 0) {
        feas[blockIdx.x] = f;
        cand[blockIdx.x] = c;
      }
    }
  } else if (threadIdx.x == 0) {
    cand[blockIdx.x] = hi;  // not a candidate this round
  }
  pad_narrow_last(st, feas, cand, G, lo, hi);
}

// Group starts at the minimal bound: warp 0 walks nx8 recording every start
// it visits and the 8-hop heads; then all threads fill the 7 starts inside
// each hop from the single-step table nx1 in parallel.
__global__ void __launch_bounds__(1024, 1)
    k_pad_starts_nx(int d, int64_t n, const uint32_t* __restrict__ a, const PadSearch* st,
                    uint16_t* __restrict__ nx1, int64_t* __restrict__ starts,
                    int32_t* __restrict__ n_groups, int64_t* __restrict__ out_bound,
                    orch_summary* s) {
  if (pipeline_failed(s)) return;
  extern __shared__ __align__(16) uint16_t nx[];
  __shared__ int32_t heads[ORCH_MAX_INSTANCES / 8 + 2];
  __shared__ int s_m, s_g;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0);
  const int64_t bound = st->hi;
  build_nx8(a, n, bound, nx, nx1);
  __threadfence_block();
  if (warp == 0) {
    int m = 0;
    const int g = warp_walk_nx8(a, n, d, bound, nx, lane, starts, heads, &m);
    if (lane == 0) {
      s_m = m;
      s_g = g;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_m; i += blockDim.x) {
    const int g0 = heads[i];
    int64_t p = starts[g0];
    for (int j = 1; j < 8; ++j) {
      const uint16_t v = nx1[p];
      p = v == kNxFar ? thread_next_start(a, n, p, bound, p) : p + v;
      starts[g0 + j] = p;
    }
  }
  if (threadIdx.x == 0) {
    starts[s_g] = n;
    *n_groups = s_g;
    *out_bound = bound;
    s->bound = bound;
  }
}

// Fallbacks for n > kNxMax: one warp per candidate walks the chain serially.
__global__ void __launch_bounds__(32)
    k_pad_starts_warp(int d, int64_t n, const uint32_t* __restrict__ a, const PadSearch* st,
                      int64_t* __restrict__ starts, int32_t* __restrict__ n_groups,
                      int64_t* __restrict__ out_bound, orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int lane = threadIdx.x;
  const int64_t bound = st->hi;
  int64_t p = 0;
  int g = 0;
  while (p < n) {
    if (lane == 0) starts[g] = p;
    ++g;
    p = warp_next_start(a, n, p, bound, lane);
  }
  if (lane == 0) {
    starts[g] = n;
    *n_groups = g;
    *out_bound = bound;
    s->bound = bound;
  }
}

__global__ void __launch_bounds__(32)
    k_pad_eval_warp(int d, int64_t n, const uint32_t* __restrict__ a, PadSearch* st,
                    int32_t* __restrict__ feas, int64_t* __restrict__ cand,
                    const orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int64_t lo = st->lo, hi = st->hi;
  if (lo >= hi) return;
  const int G = gridDim.x, lane = threadIdx.x;
  const int64_t c = pad_candidate(lo, hi, G, blockIdx.x);
  if (c < hi) {
    const bool f = warp_feasible(a, n, d, c, lane);
    if (lane == 0) {
      feas[blockIdx.x] = f;
      cand[blockIdx.x] = c;
    }
  } else if (lane == 0) {
    cand[blockIdx.x] = hi;
  }
  pad_narrow_last(st, feas, cand, G, lo, hi);
}

// Item placement from group starts: group g -> bin g (balancers.cpp:203-206),
// slot and token offset within the group; empty trailing bins.
__global__ void k_padded_place(int d, int64_t n, const int32_t* __restrict__ asc_order,
                               const int64_t* __restrict__ asc_prefix,
                               const int64_t* __restrict__ starts,
                               const int32_t* __restrict__ n_groups,
                               int32_t* __restrict__ dest_inst, int32_t* __restrict__ dest_slot,
                               int64_t* __restrict__ dst_off, int32_t* __restrict__ bin_offset,
                               int32_t* __restrict__ bin_member, int32_t* __restrict__ bin_count,
                               int64_t* __restrict__ bin_tokens, const orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int G = *n_groups;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = tid; k < n; k += stride) {
    int lo = 0, hi = G;  // last g with starts[g] <= k
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (starts[mid] <= k) lo = mid; else hi = mid;
    }
    const int32_t pos = asc_order[k];
    dest_inst[pos] = lo;
    dest_slot[pos] = static_cast<int32_t>(k - starts[lo]);
    dst_off[pos] = asc_prefix[k] - asc_prefix[starts[lo]];
    bin_member[k] = pos;
  }
  for (int64_t g = tid; g <= d; g += stride) {
    const int64_t st = g < G ? starts[g] : n;
    bin_offset[g] = static_cast<int32_t>(st);
    if (g < d) {
      const int64_t en = g < G ? starts[g + 1] : n;
      bin_count[g] = static_cast<int32_t>(en - st);
      bin_tokens[g] = asc_prefix[en] - asc_prefix[st];
    }
  }
}

// ---------------------------------------------------------------- K5b
// ConvTransformer seeding (balancers.cpp:245-268): descending items fill
// group after group under the greedy bound; a group ends at the first item
// with (size + 1) * len > bound (not monotone: scanned 32 at a time with a
// ballot); when d groups exist the rest is left to distribute_min_sum.
__global__ void k_conv_seed(int d, int64_t n, const uint32_t* __restrict__ xs,
                            const int32_t* __restrict__ order,
                            const int64_t* __restrict__ greedy_tokens, int32_t* __restrict__ dest_inst,
                            int32_t* __restrict__ dest_slot, int64_t* __restrict__ dst_off,
                            int64_t* __restrict__ seed_load, int32_t* __restrict__ seed_count,
                            int64_t* __restrict__ consumed_out, orch_summary* s) {
  if (pipeline_failed(s)) return;
  const int lane = threadIdx.x;
  int64_t bound = 0;
  for (int i = lane; i < d; i += 32) bound = greedy_tokens[i] > bound ? greedy_tokens[i] : bound;
  for (int off = 16; off > 0; off >>= 1) {
    const int64_t o = __shfl_xor_sync(~0u, bound, off);
    bound = o > bound ? o : bound;
  }
  for (int i = lane; i < d; i += 32) {
    seed_load[i] = 0;
    seed_count[i] = 0;
  }
  // items stream through a shared-memory window so the sequential group scan
  // never waits on L2 latency
  constexpr int kWin = 2048;
  __shared__ uint32_t wx[kWin];
  __shared__ int32_t wpos[kWin];
  int64_t wbase = 0, wend = 0;
  int g = 0;
  int64_t size = 0, load = 0, k = 0;
  while (k < n) {
    if (k + 32 > wend && wend < n) {  // refill from k
      __syncwarp();
      wbase = k;
      wend = k + kWin < n ? k + kWin : n;
      for (int64_t j = lane; j < wend - wbase; j += 32) {
        wx[j] = xs[wbase + j];
        wpos[j] = order[wbase + j];
      }
      __syncwarp();
    }
    const int64_t t = k + lane;
    const int64_t x = t < n ? static_cast<int64_t>(wx[t - wbase]) : 0;
    const bool c = t < n && (size + lane + 1) * x > bound;
    const bool valid = t < n;
    const unsigned mv = __ballot_sync(~0u, valid);
    const unsigned m = __ballot_sync(~0u, c);
    const int take = m ? __ffs(m) - 1 : __popc(mv);
    // exclusive prefix of x over lanes < take
    int64_t incl = lane < take ? x : 0;
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t o = __shfl_up_sync(~0u, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane < take) {
      const int32_t pos = wpos[t - wbase];
      dest_inst[pos] = g;
      dest_slot[pos] = static_cast<int32_t>(size + lane);
      dst_off[pos] = load + incl - x;
    }
    load += __shfl_sync(~0u, incl, 31);
    size += take;
    k += take;
    if (m) {
      if (g + 1 == d) break;  // (size+1)*len > bound with d groups open
      if (lane == 0) {
        seed_load[g] = load;
        seed_count[g] = static_cast<int32_t>(size);
      }
      ++g;
      size = 0;
      load = 0;
    }
  }
  if (lane == 0) {
    seed_load[g] = load;
    seed_count[g] = static_cast<int32_t>(size);
    *consumed_out = k;
    s->bound = bound;
  }
}

// ---------------------------------------------------------------- K7
// Per-batch reductions + cost() (core.cpp:70-118), one warp per batch over
// its CSR members (slot order). The TQ-unpadded square sum equals the
// reference's sequential double sum whenever every partial sum is an exact
// integer (< 2^53, lengths < 2^26); otherwise lane 0 replays the sequential
// double accumulation in slot order.
__global__ void k_bin_cost(orch_cost_model m, int d, const int32_t* __restrict__ bin_offset,
                           const int32_t* __restrict__ bin_member,
                           const int64_t* __restrict__ len, int32_t* __restrict__ out_count,
                           int64_t* __restrict__ out_len, int64_t* __restrict__ out_tokens,
                           double* __restrict__ out_cost, const orch_summary* s) {
  if (s && pipeline_failed(s)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < d; b += warps) {
    const int beg = bin_offset[b], end = bin_offset[b + 1];
    int64_t sum = 0, mx = 0;
    unsigned long long sq = 0;
    bool inexact = false;
    for (int k = beg + lane; k < end; k += 32) {
      const int64_t l = len[bin_member[k]];
      sum += l;
      mx = l > mx ? l : mx;
      if (l >= (1ll << 26)) inexact = true;
      sq += static_cast<unsigned long long>(l) * static_cast<unsigned long long>(l);
      if (sq >= (1ull << 53)) inexact = true;  // per-lane partials stay < 2^53 + 2^52
    }
    for (int off = 16; off > 0; off >>= 1) {
      sum += __shfl_xor_sync(~0u, sum, off);
      const int64_t om = __shfl_xor_sync(~0u, mx, off);
      mx = om > mx ? om : mx;
      sq += __shfl_xor_sync(~0u, sq, off);
    }
    inexact = __any_sync(~0u, inexact) || sq >= (1ull << 53);
    double sqd = static_cast<double>(sq);
    if (inexact && m.variant == ORCH_TRANSFORMER_QUADRATIC && !m.padded) {
      if (lane == 0) {
        double acc = 0.0;
        for (int k = beg; k < end; ++k) {
          const double l = static_cast<double>(len[bin_member[k]]);
          acc = rn_add(acc, rn_mul(l, l));
        }
        sqd = acc;
      }
      sqd = __shfl_sync(~0u, sqd, 0);
    }
    if (lane == 0) {
      const int64_t count = end - beg;
      if (out_count) out_count[b] = static_cast<int32_t>(count);
      if (out_tokens) out_tokens[b] = sum;
      if (out_len) out_len[b] = m.padded ? count * mx : sum;
      out_cost[b] = batch_cost(m, count, sum, mx, sqd);
    }
  }
}

// max / mean / ratio of stats_of (orchestrator.cpp:91-102) over d batch
// costs, block-wide. The mean is the reference's sequential left-to-right
// double sum; when every cost is an integer and the total < 2^53 all partial
// sums are exact so a parallel integer sum gives the same bits.
__device__ void block_stats(int d, const double* __restrict__ cost, double* out_max,
                            double* out_mean, double* out_ratio) {
  __shared__ double s_max[32];
  __shared__ int s_int[32];
  __shared__ long long s_sum[32];
  double mx = 0.0;
  long long isum = 0;
  int integral = 1;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double c = cost[i];
    mx = c > mx ? c : mx;
    if (c >= 0.0 && c < 1099511627776.0 && c == floor(c))  // < 2^40: d*2^40 cannot overflow
      isum += static_cast<long long>(c);
    else
      integral = 0;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(~0u, mx, off);
    mx = o > mx ? o : mx;
    isum += __shfl_xor_sync(~0u, isum, off);
    integral &= __shfl_xor_sync(~0u, integral, off);
  }
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_max[w] = mx;
    s_sum[w] = isum;
    s_int[w] = integral;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = 0.0;
    long long T = 0;
    int I = 1;
    for (int i = 0; i < nw; ++i) {
      M = s_max[i] > M ? s_max[i] : M;
      T += s_sum[i];
      I &= s_int[i];
    }
    double total;
    if (I && T < (1ll << 53)) {
      total = static_cast<double>(T);
    } else {
      total = 0.0;
      for (int i = 0; i < d; ++i) total = rn_add(total, cost[i]);
    }
    const double mean = d == 0 ? 0.0 : rn_div(total, static_cast<double>(d));
    *out_max = M;
    *out_mean = mean;
    *out_ratio = mean > 0.0 ? rn_div(M, mean) : 1.0;
  }
  __syncthreads();
}

// never_worse (balancers.cpp:71-76): identity if ident.obj <= algo.obj
// (objective = max over batches starting at 0.0, balancers.cpp:57-58).
__global__ void k_decide(int d, int identity_only, const double* __restrict__ ident_cost,
                         const double* __restrict__ algo_cost, orch_summary* s) {
  if (pipeline_failed(s)) return;
  __shared__ double i_mean, i_ratio, a_mean, a_ratio, i_max, a_max;
  block_stats(d, ident_cost, &i_max, &i_mean, &i_ratio);
  if (!identity_only) block_stats(d, algo_cost, &a_max, &a_mean, &a_ratio);
  if (threadIdx.x == 0) {
    s->identity_objective = i_max;
    s->pre_max = i_max;
    s->pre_mean = i_mean;
    s->pre_ratio = i_ratio;
    const bool ident = identity_only || i_max <= a_max;
    s->algo_objective = identity_only ? i_max : a_max;
    s->used_identity = ident ? 1 : 0;
    s->objective = ident ? i_max : a_max;
    s->post_max = ident ? i_max : a_max;
    s->post_mean = ident ? i_mean : a_mean;
    s->post_ratio = ident ? i_ratio : a_ratio;
  }
}

// Identity fallback: overwrite the algorithm's arrangement with the identity
// (dest = origin, slot = source slot, offsets = source offsets).
__global__ void k_apply_identity(int d, int64_t n, const int32_t* __restrict__ origin,
                                 const int32_t* __restrict__ src_slot,
                                 const int64_t* __restrict__ src_off,
                                 const int32_t* __restrict__ ident_offset,
                                 const int32_t* __restrict__ ident_order,
                                 const int32_t* __restrict__ i_count,
                                 const int64_t* __restrict__ i_len,
                                 const int64_t* __restrict__ i_tokens,
                                 const double* __restrict__ i_cost, int32_t* __restrict__ dest_inst,
                                 int32_t* __restrict__ dest_slot, int64_t* __restrict__ dst_off,
                                 int32_t* __restrict__ bin_offset, int32_t* __restrict__ bin_member,
                                 int32_t* __restrict__ bin_count, int64_t* __restrict__ bin_len,
                                 int64_t* __restrict__ bin_tokens, double* __restrict__ bin_cost,
                                 const orch_summary* s) {
  if (pipeline_failed(s) || !s->used_identity) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) {
    if (dest_inst) dest_inst[i] = origin[i];
    if (dest_slot) dest_slot[i] = src_slot[i];
    if (dst_off) dst_off[i] = src_off[i];
    if (bin_member) bin_member[i] = ident_order[i];
  }
  for (int64_t b = tid; b <= d; b += stride) {
    if (bin_offset) bin_offset[b] = ident_offset[b];
    if (b < d) {
      if (bin_count) bin_count[b] = i_count[b];
      if (bin_len) bin_len[b] = i_len[b];
      if (bin_tokens) bin_tokens[b] = i_tokens[b];
      if (bin_cost) bin_cost[b] = i_cost[b];
    }
  }
}

// CSR members of a packing from (dest_inst, dest_slot).
__global__ void k_scatter_members(int64_t n, const int32_t* __restrict__ dest_inst,
                                  const int32_t* __restrict__ dest_slot,
                                  const int32_t* __restrict__ bin_offset,
                                  int32_t* __restrict__ bin_member, const orch_summary* s) {
  if (pipeline_failed(s)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bin_member[bin_offset[dest_inst[i]] + dest_slot[i]] = static_cast<int32_t>(i);
}

__global__ void k_u32_to_i64(int64_t n, const uint32_t* __restrict__ a, int64_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

}  // namespace
}  // namespace orchb

namespace orchb {
namespace {  // internal linkage: included by several translation units

// stats_of over precomputed batch costs: d_stats = {max, mean, ratio}.
__global__ void k_stats_only(int d, const double* __restrict__ cost, double* __restrict__ stats) {
  __shared__ double mx, mn, ra;
  block_stats(d, cost, &mx, &mn, &ra);
  if (threadIdx.x == 0) {
    stats[0] = mx;
    stats[1] = mn;
    stats[2] = ra;
  }
}

// Sort keys for batches_from_items; origin counts (caller validated origins).
__global__ void k_origin_keys(int d, int64_t n, const int32_t* __restrict__ origin,
                              uint32_t* __restrict__ key, int32_t* __restrict__ iota,
                              int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = origin[i];
    key[i] = static_cast<uint32_t>(o);
    iota[i] = static_cast<int32_t>(i);
    if (o >= 0 && o < d) atomicAdd(&cnt[o], 1);
  }
}

}  // namespace
}  // namespace orchb
