// Context, workspace arena, error plumbing of the C-ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "common.cuh"

namespace orchb {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

void arena_reset(orch_ctx* ctx) {
  ctx->arena.used = 0;
}

int arena_reserve(orch_ctx* ctx, size_t bytes, cudaStream_t stream) {
  Arena& a = ctx->arena;
  if (bytes <= a.cap) return ORCH_OK;
  size_t cap = a.cap ? a.cap : (size_t{1} << 20);
  while (cap < bytes) cap *= 2;
  if (a.base) {
    ORCH_CUDA_TRY(cudaStreamSynchronize(stream));
    ORCH_CUDA_TRY(cudaFree(a.base));
    a.base = nullptr;
    a.cap = 0;
  }
  ORCH_CUDA_TRY(cudaMalloc(&a.base, cap));
  a.cap = cap;
  a.used = 0;
  return ORCH_OK;
}

void* carve(orch_ctx* ctx, size_t bytes) {
  Arena& a = ctx->arena;
  const size_t aligned = (bytes + 255) & ~size_t{255};
  if (a.used + aligned > a.cap) return nullptr;
  void* p = a.base + a.used;
  a.used += aligned;
  return p;
}

void* pinned(orch_ctx* ctx, size_t bytes) {
  if (bytes > ctx->pinned_cap) {
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    size_t cap = 4096;
    while (cap < bytes) cap *= 2;
    if (cudaMallocHost(&ctx->pinned, cap) != cudaSuccess) {
      ctx->pinned = nullptr;
      ctx->pinned_cap = 0;
      return nullptr;
    }
    ctx->pinned_cap = cap;
  }
  return ctx->pinned;
}

}  // namespace orchb

extern "C" {

int orch_version(void) { return 100; }

const char* orch_last_error(void) { return orchb::g_err.c_str(); }

int orch_ctx_create(int device, orch_ctx** out) {
  if (!out) return orchb::fail(ORCH_INVALID_ARGUMENT, "orch_ctx_create: null out");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return orchb::fail(ORCH_CUDA_ERROR, std::string("no CUDA device available: ") +
                                            cudaGetErrorString(e));
  if (device < 0 || device >= count)
    return orchb::fail(ORCH_INVALID_ARGUMENT, "orch_ctx_create: bad device index");
  ORCH_CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  ORCH_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return orchb::fail(ORCH_CUDA_ERROR, std::string("this build targets sm_100a (B200); device is ") +
                                            prop.name);
  auto* ctx = new orch_ctx();
  ctx->device = device;
  *out = ctx;
  return ORCH_OK;
}

void orch_ctx_destroy(orch_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->arena.base) cudaFree(ctx->arena.base);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
}

int64_t orch_ctx_launches(const orch_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
