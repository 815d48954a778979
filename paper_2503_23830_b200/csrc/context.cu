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

Arena* arena_for(orch_ctx* ctx, cudaStream_t stream) {
  for (int i = 0; i < ctx->n_arenas; ++i)
    if (ctx->arenas[i].stream == stream) return &ctx->arenas[i].arena;
  if (ctx->n_arenas == kMaxCtxStreams) {
    // A 17th stream: wait until no kernel can still be using any workspace,
    // then hand the next slot (round robin) with its buffer to the new stream.
    if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
    const int i = ctx->evict_next;
    ctx->evict_next = (i + 1) % kMaxCtxStreams;
    ctx->arenas[i].stream = stream;
    ctx->arenas[i].arena.used = 0;
    return &ctx->arenas[i].arena;
  }
  ctx->arenas[ctx->n_arenas].stream = stream;
  return &ctx->arenas[ctx->n_arenas++].arena;
}

int arena_reserve(Arena* ap, size_t bytes, cudaStream_t stream) {
  Arena& a = *ap;
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

void* carve(Arena* ap, size_t bytes) {
  Arena& a = *ap;
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

int host_stage(orch_ctx* ctx, size_t bytes, char** h, char** d) {
  if (bytes > ctx->stage_cap) {
    if (ctx->stage) cudaFree(ctx->stage);
    ctx->stage = nullptr;
    ctx->stage_cap = 0;
    size_t cap = 1 << 20;
    while (cap < bytes) cap *= 2;
    ORCH_CUDA_TRY(cudaMalloc(&ctx->stage, cap));
    ctx->stage_cap = cap;
  }
  *h = static_cast<char*>(pinned(ctx, bytes));
  if (!*h) return fail(ORCH_CUDA_ERROR, "pinned staging allocation failed");
  *d = static_cast<char*>(ctx->stage);
  return ORCH_OK;
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
  for (int i = 0; i < ctx->n_arenas; ++i)
    if (ctx->arenas[i].arena.base) cudaFree(ctx->arenas[i].arena.base);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
}

int64_t orch_ctx_launches(const orch_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
