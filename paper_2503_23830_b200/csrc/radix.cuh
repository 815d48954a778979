// Stable LSD radix sort of (u32 key, i32 value) pairs and exclusive scans for
// the multi-kernel balance path -- the ordering steps sorted_descending /
// sorted_ascending (balancers.cpp:78-88) and batches_from_items' grouping by
// origin (core.cpp:183-199). Hand-written for sm_100a; replaces the library
// sort and scan of round 1.
//
// A pass sorts on one 8-bit digit, in two launches:
//   k_rs_hist     tile of 4096 items per CTA: a shared-memory histogram of the
//                 digit -> hist[digit][tile]; pass 0 also finds the largest key
//   k_rs_scatter  every CTA computes its own base offsets from the histograms
//                 (prefix over earlier tiles + the digits' totals), ranks its
//                 items stably (warps own 256 consecutive items, __match_any_sync
//                 per 32, per-warp digit counters) and scatters keys and values.
// Descending order is ascending order on digit' = 255 - digit (every byte of
// ~key), which keeps equal keys in input order -- std::stable_sort by length,
// descending. Passes 2 and 3 run only when the largest key reaches 2^16 (the
// lengths of the BASELINE phases need two passes); they are skipped together
// on the device, so the result always lands in the output buffer:
//   pass 0: in -> tmp, pass 1: tmp -> out, [pass 2: out -> tmp, pass 3: tmp -> out].
#pragma once

#include <cstdint>

#include "common.cuh"

namespace orchb {
namespace {

constexpr int kRsThreads = 512;
constexpr int kRsPer = 8;                          // items per thread
constexpr int kRsTile = kRsThreads * kRsPer;       // 4096 items per CTA
constexpr int kRsWarps = kRsThreads / 32;

struct RsState {
  unsigned max_key;
};

__device__ __forceinline__ int rs_digit(uint32_t key, int shift, bool desc) {
  const int dg = static_cast<int>((key >> shift) & 255u);
  return desc ? 255 - dg : dg;
}

__device__ __forceinline__ bool rs_skip(const RsState* st, int pass) {
  return pass >= 2 && st->max_key < 65536u;
}

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint32_t* __restrict__ keys,
                                                        int64_t n, int pass, bool desc,
                                                        uint32_t* __restrict__ hist, int tiles,
                                                        RsState* st) {
  if (rs_skip(st, pass)) return;
  __shared__ uint32_t h[256];
  __shared__ unsigned smax;
  for (int i = threadIdx.x; i < 256; i += kRsThreads) h[i] = 0;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  unsigned mx = 0;
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    const int64_t i = base + j * kRsThreads + threadIdx.x;
    if (i < n) {
      const uint32_t k = keys[i];
      mx = k > mx ? k : mx;
      atomicAdd(&h[rs_digit(k, 8 * pass, desc)], 1u);
    }
  }
  if (pass == 0) {
    mx = __reduce_max_sync(~0u, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(&smax, mx);
  }
  __syncthreads();
  for (int dg = threadIdx.x; dg < 256; dg += kRsThreads)
    hist[static_cast<int64_t>(dg) * tiles + blockIdx.x] = h[dg];
  if (pass == 0 && threadIdx.x == 0) atomicMax(&st->max_key, smax);
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    int32_t* __restrict__ vout, int64_t n, int pass, bool desc,
    const uint32_t* __restrict__ hist, int tiles, const RsState* st) {
  if (rs_skip(st, pass)) return;
  __shared__ uint32_t base[256];          // this tile's first output slot per digit
  __shared__ uint32_t tot[256];
  __shared__ uint16_t wcnt[kRsWarps][256];  // per-warp digit counts, then warp bases
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tile = blockIdx.x;
  // ---- offsets: digits' totals (exclusive scan over 256) + earlier tiles' counts
  if (t < 256) {
    const uint32_t* row = hist + static_cast<int64_t>(t) * tiles;
    uint32_t before = 0, all = 0;
#pragma unroll 8
    for (int b = 0; b < tiles; ++b) {
      const uint32_t v = row[b];
      before += b < tile ? v : 0u;
      all += v;
    }
    base[t] = before;
    tot[t] = all;
  }
  for (int i = t; i < kRsWarps * 256; i += kRsThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 256 totals, 8 per lane
    uint32_t v[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = tot[lane * 8 + j];
      s += v[j];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += u;
    }
    uint32_t ex = incl - s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      tot[lane * 8 + j] = ex;
      ex += v[j];
    }
  }
  __syncthreads();
  if (t < 256) base[t] += tot[t];
  // ---- stable ranks: warp w owns items [w * 256, (w + 1) * 256) of the tile
  const int64_t first = static_cast<int64_t>(tile) * kRsTile + warp * (32 * kRsPer);
  uint32_t key[kRsPer];
  int32_t val[kRsPer];
  int dig[kRsPer], rank[kRsPer];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    const int64_t i = first + j * 32 + lane;
    const bool ok = i < n;
    key[j] = ok ? kin[i] : 0u;
    val[j] = ok ? vin[i] : 0;
    dig[j] = ok ? rs_digit(key[j], 8 * pass, desc) : 256;  // 256: no item
  }
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    const unsigned peers = __match_any_sync(~0u, dig[j]);
    const int before = __popc(peers & lt);
    int run = 0;
    if (dig[j] < 256) run = wcnt[warp][dig[j]];
    rank[j] = run + before;
    __syncwarp();
    if (dig[j] < 256 && before == 0) wcnt[warp][dig[j]] = static_cast<uint16_t>(run + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  // warp bases per digit: exclusive scan over the warps
  if (t < 256) {
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = wcnt[w][t];
      wcnt[w][t] = static_cast<uint16_t>(acc);
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    if (dig[j] == 256) continue;
    const uint32_t pos = base[dig[j]] + wcnt[warp][dig[j]] + rank[j];
    ORCH_DCHECK(pos < static_cast<uint64_t>(n));
    kout[pos] = key[j];
    vout[pos] = val[j];
  }
}

// The whole sort of n <= kRsTile items in one CTA (shared memory ping-pong):
// one launch instead of a hist / scatter pair per pass.
struct RsTileSmem {
  uint32_t k[2][kRsTile];
  int32_t v[2][kRsTile];
  uint16_t hist[256 * kRsWarps];  // [digit][warp]
  uint32_t ws[kRsWarps];
  unsigned mx;
};

__global__ void __launch_bounds__(kRsThreads, 1)
    k_rs_sort_tile(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                   uint32_t* __restrict__ kout, int32_t* __restrict__ vout, int n, bool desc) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  RsTileSmem& S = *reinterpret_cast<RsTileSmem*>(rs_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) S.mx = 0;
  __syncthreads();
  unsigned mx = 0;
  for (int i = t; i < kRsTile; i += kRsThreads) {
    const uint32_t k = i < n ? kin[i] : 0u;
    S.k[0][i] = k;
    S.v[0][i] = i < n ? vin[i] : 0;
    mx = k > mx ? k : mx;
  }
  mx = __reduce_max_sync(~0u, mx);
  if (lane == 0) atomicMax(&S.mx, mx);
  __syncthreads();
  const unsigned kmax = S.mx;
  const int passes = kmax < 256u ? 1 : kmax < 65536u ? 2 : kmax < (1u << 24) ? 3 : 4;
  const unsigned lt = (1u << lane) - 1u;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    for (int i = t; i < 256 * kRsWarps; i += kRsThreads) S.hist[i] = 0;
    __syncthreads();
    uint32_t key[kRsPer];
    int32_t val[kRsPer];
    int dig[kRsPer], rank[kRsPer];
#pragma unroll
    for (int j = 0; j < kRsPer; ++j) {
      const int i = warp * 32 * kRsPer + j * 32 + lane;
      key[j] = S.k[cur][i];
      val[j] = S.v[cur][i];
      dig[j] = i < n ? rs_digit(key[j], 8 * p, desc) : 256;  // padding sorts last
    }
#pragma unroll
    for (int j = 0; j < kRsPer; ++j) {
      const unsigned peers = __match_any_sync(~0u, dig[j]);
      const int before = __popc(peers & lt);
      int run = 0;
      if (dig[j] < 256) run = S.hist[dig[j] * kRsWarps + warp];
      rank[j] = run + before;
      __syncwarp();
      if (dig[j] < 256 && before == 0)
        S.hist[dig[j] * kRsWarps + warp] = static_cast<uint16_t>(run + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    {  // exclusive scan over hist[digit][warp], 8 counters per thread
      static_assert(256 * kRsWarps == 8 * kRsThreads, "8 counters per thread");
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = S.hist[8 * t + q];
        sum += v[q];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(~0u, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) S.ws[warp] = incl;
      __syncthreads();
      uint32_t before = 0;
#pragma unroll
      for (int w = 0; w < kRsWarps; ++w) before += w < warp ? S.ws[w] : 0u;
      uint32_t ex = before + incl - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        S.hist[8 * t + q] = static_cast<uint16_t>(ex);
        ex += v[q];
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kRsPer; ++j) {
      if (dig[j] == 256) continue;
      const int pos = S.hist[dig[j] * kRsWarps + warp] + rank[j];
      ORCH_DCHECK(pos < n);
      S.k[cur ^ 1][pos] = key[j];
      S.v[cur ^ 1][pos] = val[j];
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int i = t; i < n; i += kRsThreads) {
    kout[i] = S.k[cur][i];
    vout[i] = S.v[cur][i];
  }
}

// Exclusive scan of int32 / int64 counts: out[i] = sum of in[0, i). Tiles of
// 4096 elements: k_scan_partial sums every tile, k_scan_tiles scans each tile
// on top of the sum of the tiles before it (read from the partial sums).
template <class T>
__global__ void __launch_bounds__(kRsThreads) k_scan_partial(const T* __restrict__ in,
                                                             int64_t count, T* __restrict__ part) {
  __shared__ T ws[kRsWarps];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile + static_cast<int64_t>(t) * kRsPer;
  T s = 0;
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) s += base + j < count ? in[base + j] : T(0);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (t == 0) {
    T a = 0;
    for (int w = 0; w < kRsWarps; ++w) a += ws[w];
    part[blockIdx.x] = a;
  }
}

template <class T>
__global__ void __launch_bounds__(kRsThreads) k_scan_tiles(const T* __restrict__ in,
                                                           T* __restrict__ out, int64_t count,
                                                           const T* __restrict__ part) {
  __shared__ T ws[kRsWarps];
  __shared__ T carry;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (warp == 0) {  // the tiles before this one
    T c = 0;
    for (int b = lane; b < static_cast<int>(blockIdx.x); b += 32) c += part[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(~0u, c, o);
    if (lane == 0) carry = c;
  }
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile + static_cast<int64_t>(t) * kRsPer;
  T v[kRsPer], s = 0;
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    v[j] = base + j < count ? in[base + j] : T(0);
    s += v[j];
  }
  T incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < kRsWarps ? ws[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T u = __shfl_up_sync(~0u, wi, o);
      if (lane >= o) wi += u;
    }
    if (lane < kRsWarps) ws[lane] = wi - w;
  }
  __syncthreads();
  T ex = carry + ws[warp] + incl - s;
#pragma unroll
  for (int j = 0; j < kRsPer; ++j) {
    if (base + j < count) out[base + j] = ex;
    ex += v[j];
  }
}

// Scratch of one sort: a key / value pair of temporaries, the tile histograms
// and the state word (Plan::add these; rs_hist_words(n) histogram words).
inline int rs_tiles(int64_t n) { return static_cast<int>((n + kRsTile - 1) / kRsTile); }
inline size_t rs_hist_words(int64_t n) { return 256 * static_cast<size_t>(rs_tiles(n > 0 ? n : 1)); }

// in -> out (stable), temporaries kt / vt; `in` is left unchanged. Key bits
// beyond 16 are sorted only when some key has them (decided on the device).
inline int rs_sort_pairs(orch_ctx* ctx, const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                         int32_t* vout, uint32_t* kt, int32_t* vt, int64_t n, bool desc,
                         uint32_t* hist, RsState* st, cudaStream_t s) {
  if (n <= 0) return ORCH_OK;
  if (n <= kRsTile) {  // one CTA sorts everything in shared memory
    static PerDeviceOnce configured;
    const int rc = configured([&]() -> int {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_rs_sort_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(RsTileSmem))));
      return ORCH_OK;
    });
    if (rc) return rc;
    k_rs_sort_tile<<<1, kRsThreads, sizeof(RsTileSmem), s>>>(kin, vin, kout, vout,
                                                              static_cast<int>(n), desc);
    ctx->launches += 1;
    ORCH_CUDA_TRY(cudaGetLastError());
    return ORCH_OK;
  }
  const int tiles = rs_tiles(n);
  ORCH_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(RsState), s));
  const uint32_t* ki[4] = {kin, kt, kout, kt};
  const int32_t* vi[4] = {vin, vt, vout, vt};
  uint32_t* ko[4] = {kt, kout, kt, kout};
  int32_t* vo[4] = {vt, vout, vt, vout};
  for (int p = 0; p < 4; ++p) {
    k_rs_hist<<<tiles, kRsThreads, 0, s>>>(ki[p], n, p, desc, hist, tiles, st);
    k_rs_scatter<<<tiles, kRsThreads, 0, s>>>(ki[p], vi[p], ko[p], vo[p], n, p, desc, hist, tiles,
                                              st);
  }
  ctx->launches += 8;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

// Scratch: rs_tiles(count) partial sums of T.
template <class T>
inline int rs_exclusive_scan(orch_ctx* ctx, const T* in, T* out, int64_t count, T* part,
                             cudaStream_t s) {
  if (count <= 0) return ORCH_OK;
  const int tiles = rs_tiles(count);
  if (tiles > 1) {  // one tile needs no partial sums (nothing before it)
    k_scan_partial<T><<<tiles, kRsThreads, 0, s>>>(in, count, part);
    ctx->launches += 1;
  }
  k_scan_tiles<T><<<tiles, kRsThreads, 0, s>>>(in, out, count, part);
  ctx->launches += 1;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // namespace
}  // namespace orchb
