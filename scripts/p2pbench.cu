// NVLink ceilings of one B200 box: how fast can a GPU move bytes into (push)
// or out of (pull) a peer's HBM? The roofline denominator of the N > 1
// exchange (bench.py reads profiles/nvlink_peaks.json, written from this
// program's output). One process drives every visible GPU (peer access on).
//
//   method  stg   kernel stores: LDG.128 from local HBM, STG.128 to the peer
//           tma   kernel bulk copies: cp.async.bulk local -> smem -> peer
//                 (the put's mechanism, k_move_tma<kPut>)
//           ldg   kernel pull: LDG.128 from the peer, STG.128 to local HBM
//           ce    copy engine: cudaMemcpyPeerAsync
//           nccl  one grouped ncclSend/ncclRecv per transfer (ncclCommInitAll,
//                 one communicator per GPU in this process)
//   pattern uni   GPU 0 -> GPU 1
//           bidir 0 -> 1 and 1 -> 0 at once
//           a2a   every GPU to every other GPU at once (1/(N-1) of its bytes each)
//
// Prints one JSON line per (pattern, method): GB/s per GPU per direction =
// bytes one GPU sends / time, the max over GPUs of the event-timed durations,
// median of 5 repetitions after 2 warm-ups.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2pbench scripts/p2pbench.cu
//   ./p2pbench [MiB per GPU, default 1024] [method] [pattern]   (one combination only)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

constexpr int kSMs = 148;
constexpr int kChunk = 32768;
constexpr int kStages = 4;

__global__ void __launch_bounds__(512) k_stg(int4* __restrict__ dst, const int4* __restrict__ src,
                                             size_t nvec) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one warp per CTA, lane 0 drives a kStages ring of kChunk-byte stages: the
// loads of kStages-1 chunks in flight while the oldest is stored (k_move_tma)
__global__ void __launch_bounds__(32) k_tma(char* __restrict__ dst, const char* __restrict__ src,
                                            size_t bytes) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ alignas(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t chunks = bytes / kChunk;
  const size_t mine = chunks > blockIdx.x ? (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk_of = [&](size_t j) { return blockIdx.x + j * gridDim.x; };
  uint32_t phase = 0;
  auto retire = [&](size_t j) {
    const int s = static_cast<int>(j % kStages);
    asm volatile(
        "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W%=;\n}" ::"r"(smem_u32(&bar[s])),
        "r"((phase >> s) & 1u));
    phase ^= 1u << s;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     dst + chunk_of(j) * kChunk),
                 "r"(smem_u32(ring + s * kChunk)), "r"(kChunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  for (size_t j = 0; j < mine; ++j) {
    if (j >= kStages - 1) retire(j - (kStages - 1));
    if (j >= kStages) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    const int s = static_cast<int>(j % kStages);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(kChunk)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(ring + s * kChunk)),
        "l"(src + chunk_of(j) * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s]))
        : "memory");
  }
  for (size_t j = mine > kStages - 1 ? mine - (kStages - 1) : 0; j < mine; ++j) retire(j);
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Xfer {
  int dev;          // the GPU that runs the copy
  char* dst;
  const char* src;
  size_t bytes;
};

std::vector<ncclComm_t> g_comms;

double run(const std::vector<Xfer>& xs, const std::string& method, int ngpu,
           std::vector<cudaStream_t>& st, std::vector<cudaEvent_t>& e0, std::vector<cudaEvent_t>& e1) {
  for (int g = 0; g < ngpu; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(e0[g], st[g]));
  }
  if (method == "nccl") {  // x.dev is the sender; the receiver posts the matching recv
    ncclGroupStart();
    for (const Xfer& x : xs) {
      cudaPointerAttributes at;
      CK(cudaPointerGetAttributes(&at, x.dst));
      const int to = at.device;
      ncclSend(x.src, x.bytes, ncclInt8, to, g_comms[x.dev], st[x.dev]);
      ncclRecv(x.dst, x.bytes, ncclInt8, x.dev, g_comms[to], st[to]);
    }
    if (ncclGroupEnd() != ncclSuccess) {
      std::fprintf(stderr, "nccl group failed\n");
      std::exit(1);
    }
  }
  for (const Xfer& x : xs) {
    if (method == "nccl") break;
    CK(cudaSetDevice(x.dev));
    if (method == "stg" || method == "ldg")
      k_stg<<<kSMs * 4, 512, 0, st[x.dev]>>>(reinterpret_cast<int4*>(x.dst),
                                             reinterpret_cast<const int4*>(x.src), x.bytes / 16);
    else if (method == "tma")
      k_tma<<<kSMs, 32, kStages * kChunk, st[x.dev]>>>(x.dst, x.src, x.bytes);
    else
      CK(cudaMemcpyAsync(x.dst, x.src, x.bytes, cudaMemcpyDefault, st[x.dev]));
  }
  for (int g = 0; g < ngpu; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(e1[g], st[g]));
  }
  double worst = 0;
  for (int g = 0; g < ngpu; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventSynchronize(e1[g]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
    worst = std::max(worst, static_cast<double>(ms));
  }
  return worst;
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
  const size_t bytes = mib << 20;
  int ngpu = 0;
  CK(cudaGetDeviceCount(&ngpu));
  if (ngpu < 2) {
    std::printf("{\"error\": \"needs >= 2 GPUs\", \"gpus\": %d}\n", ngpu);
    return 0;
  }
  std::vector<char*> a(ngpu), b(ngpu);
  std::vector<cudaStream_t> st(ngpu);
  std::vector<cudaEvent_t> e0(ngpu), e1(ngpu);
  for (int g = 0; g < ngpu; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ngpu; ++p)
      if (p != g) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, g, p));
        if (ok) cudaDeviceEnablePeerAccess(p, 0);
      }
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kChunk));
    CK(cudaMalloc(&a[g], bytes));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMemset(a[g], g + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  for (int g = 0; g < ngpu; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  g_comms.resize(ngpu);
  if ((argc <= 2 || std::string(argv[2]) == "nccl") &&
      ncclCommInitAll(g_comms.data(), ngpu, nullptr) != ncclSuccess) {
    std::fprintf(stderr, "ncclCommInitAll failed\n");
    return 1;
  }
  const char* methods[] = {"stg", "tma", "ldg", "ce", "nccl"};
  const char* patterns[] = {"uni", "bidir", "a2a"};
  const std::string only_m = argc > 2 ? argv[2] : "", only_p = argc > 3 ? argv[3] : "";
  for (const char* pat : patterns) {
    for (const char* m : methods) {
      const std::string method = m, pattern = pat;
      if ((!only_m.empty() && only_m != method) || (!only_p.empty() && only_p != pattern)) continue;
      std::vector<Xfer> xs;
      size_t sent_per_gpu = bytes;
      auto add = [&](int from, int to, size_t off, size_t len) {
        // push / ce / nccl: the sender runs the copy; ldg: the receiver pulls
        if (method == "ldg")
          xs.push_back({to, b[to] + off, a[from] + off, len});
        else
          xs.push_back({from, b[to] + off, a[from] + off, len});
      };
      if (pattern == "uni") {
        add(0, 1, 0, bytes);
      } else if (pattern == "bidir") {
        add(0, 1, 0, bytes);
        add(1, 0, 0, bytes);
      } else {
        const size_t part = (bytes / (ngpu - 1)) & ~size_t{kChunk - 1};
        sent_per_gpu = part * (ngpu - 1);
        for (int g = 0; g < ngpu; ++g)
          for (int k = 1; k < ngpu; ++k) add(g, (g + k) % ngpu, (k - 1) * part, part);
      }
      std::vector<double> ms;
      for (int r = 0; r < 7; ++r) {
        const double t = run(xs, method, ngpu, st, e0, e1);
        if (r >= 2) ms.push_back(t);
      }
      std::sort(ms.begin(), ms.end());
      const double med = ms[ms.size() / 2];
      std::printf(
          "{\"pattern\": \"%s\", \"method\": \"%s\", \"gpus\": %d, \"bytes_per_gpu\": %zu, "
          "\"ms\": %.4f, \"gbs_per_gpu_per_dir\": %.1f}\n",
          pat, m, pattern == "a2a" ? ngpu : 2, sent_per_gpu, med, sent_per_gpu / (med * 1e-3) / 1e9);
      std::fflush(stdout);
    }
  }
  return 0;
}
