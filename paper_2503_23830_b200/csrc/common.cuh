// Shared plumbing of the sm_100a dispatcher library: context/workspace,
// error reporting, launch accounting, exact double arithmetic helpers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "orchsim_capi.h"

// Bounds-checked diagnostics build (ORCH_NVCC_EXTRA=-DORCH_BOUNDS_CHECK): device
// asserts that print the failing condition and trap, so a bad index or an
// out-of-buffer copy kills the run loudly (compute-sanitizer is not available
// on the GPU pool; profiles/r02_bounds_check.md).
#ifdef ORCH_BOUNDS_CHECK
#define ORCH_DCHECK(cond)                                                       \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("ORCH_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define ORCH_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace orchb {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs
constexpr int kMaxCtxStreams = 16;  // distinct streams one orch_ctx serves

// Thread-local message for orch_last_error().
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define ORCH_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return ::orchb::fail(ORCH_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

// Device workspace: one growable arena per (context, stream); carve() hands out
// 256-byte aligned slices that stay valid until the next reset().
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  size_t high = 0;  // high-water mark of the current pass
};

}  // namespace orchb

struct orch_ctx {
  int device = 0;
  // One workspace per stream: calls on different streams never share scratch
  // (calls on one stream are ordered by the stream, so they may reuse it).
  struct StreamArena {
    cudaStream_t stream;
    orchb::Arena arena;
  };
  StreamArena arenas[orchb::kMaxCtxStreams];
  int n_arenas = 0;
  int evict_next = 0;  // slot handed to the next new stream once all 16 are taken
  // Pinned host staging for small device->host reads.
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  // Device staging of the host-buffer (_host) entry points, mirrored in `pinned`.
  void* stage = nullptr;
  size_t stage_cap = 0;
  int64_t launches = 0;
};

namespace orchb {

// The workspace of `stream` (created on first use; beyond kMaxCtxStreams
// streams a slot is recycled after a device synchronisation; nullptr on error).
Arena* arena_for(orch_ctx* ctx, cudaStream_t stream);
// Reserve `bytes` in the arena, growing it (synchronously, outside timed
// steady state) when needed. Returns nullptr on allocation failure.
void* carve(Arena* a, size_t bytes);
// Make sure the arena can hold `bytes` without reallocation.
int arena_reserve(Arena* a, size_t bytes, cudaStream_t stream);
void* pinned(orch_ctx* ctx, size_t bytes);
// Host-buffer (_host) entry points stage through a per-context device buffer
// and its pinned host mirror of the same layout: one copy each way per call.
int host_stage(orch_ctx* ctx, size_t bytes, char** h, char** d);

// Runs f() once per device (function attributes such as the dynamic shared
// memory limit are per-device state; a process may drive several devices).
struct PerDeviceOnce {
  std::atomic<unsigned long long> done{0};
  template <class F>
  int operator()(F&& f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return ORCH_OK;
    const int rc = f();
    if (rc == ORCH_OK) done.fetch_or(bit, std::memory_order_acq_rel);
    return rc;
  }
};

// The SM's shared-memory carveout is fixed while CTAs are resident. The row
// mover and the metadata kernels that run beside it all ask for the maximum,
// so a metadata CTA fits next to a mover CTA instead of waiting for the SM to
// drain (without this the next phase's balance waited out a whole 0.6 ms move).
template <class K>
inline cudaError_t max_carveout(K kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                              cudaSharedmemCarveoutMaxShared);
}

inline unsigned ceil_log2(unsigned long long x) {
  unsigned b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

inline int blocks_for(int64_t n, int threads, int cap = kSMs * 8) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

}  // namespace orchb

// ---- exact IEEE double helpers: the reference compiles cost() without FMA
// (SURVEY.md section 0.6); every product/sum is an explicitly rounded op.
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }

// cost() of one batch (core.cpp:91-118) from its reductions. count = items,
// tokens = sum of lengths, longest = max length, sq = sum of l*l as the
// reference's sequential double accumulation (exact integer when < 2^53).
__device__ __forceinline__ double batch_cost(const orch_cost_model& m, int64_t count,
                                             int64_t tokens, int64_t longest, double sq) {
  if (count == 0) return 0.0;
  const int64_t blen = m.padded ? count * longest : tokens;  // core.cpp:70-89
  const double linear = rn_mul(m.alpha, static_cast<double>(blen));
  switch (m.variant) {
    case ORCH_LINEAR_ONLY:
      return linear;
    case ORCH_TRANSFORMER_QUADRATIC:
      if (!m.padded) return rn_add(linear, rn_mul(m.beta, sq));
      {
        const double p = static_cast<double>(blen);
        return rn_add(linear, rn_mul(rn_mul(rn_div(m.beta, static_cast<double>(count)), p), p));
      }
    default: {
      const double lo = static_cast<double>(longest);
      return rn_add(linear, rn_mul(rn_mul(rn_mul(m.beta, static_cast<double>(count)), lo), lo));
    }
  }
}
