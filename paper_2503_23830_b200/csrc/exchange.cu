// The exchange's cost report (simulate_exchange, exchange.cpp:49-113) and the
// all-gather plan volumes (make_exchange_plan, exchange.cpp:17-28) as device
// reductions over a device-resident volume matrix V[d][d] (src-major, token
// counts; orch_volume_matrix builds it). At d = 2560 V is 6.5 M entries
// (52 MB); the reference walks it twice per instance on the host (a row and a
// strided column), here it is read once by rows and once by 32-column strips.
//
//   k_xr_rows    warp per instance i: inter_i / intra_i (off-diagonal row sum
//                split by node), local_i = V[i][i]
//   k_xr_cols    block per 32-column strip: in_i = off-diagonal column sum
//   k_xr_finish  one CTA: totals, per-node egress, peak resident volume, and
//                the worst instance -- the reference's running `if (t > worst)`
//                over i in order keeps the FIRST i of maximal t, so a
//                max-then-lowest-index reduction is exact; t_i is evaluated
//                with the reference's rounded double ops (div, div, add)
//   k_xr_stale   plan volumes vs the volume matrix of the items (the stale check)
#include <cstring>
#include <string>

#include "common.cuh"
#include "plan.cuh"

namespace orchb {
namespace {

constexpr int kXrThreads = 1024;

__global__ void k_xr_rows(int d, int c, const int64_t* __restrict__ V, int64_t* __restrict__ inter,
                          int64_t* __restrict__ intra, int64_t* __restrict__ local) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < d;
       i += warps) {
    const int64_t* row = V + i * d;
    const int node = static_cast<int>(i) / c;
    int64_t a = 0, b = 0;
    for (int j = lane; j < d; j += 32) {
      const int64_t v = __ldcs(row + j);
      if (j == i) continue;
      if (j / c == node)
        b += v;
      else
        a += v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(~0u, a, o);
      b += __shfl_xor_sync(~0u, b, o);
    }
    if (lane == 0) {
      inter[i] = a;
      intra[i] = b;
      local[i] = row[i];
    }
  }
}

__global__ void __launch_bounds__(kXrThreads) k_xr_cols(int d, const int64_t* __restrict__ V,
                                                        int64_t* __restrict__ in) {
  __shared__ int64_t part[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  int64_t s = 0;
  if (j < d)
    for (int i = w; i < d; i += 32)
      if (i != j) s += __ldcs(V + static_cast<int64_t>(i) * d + j);
  part[w][lane] = s;
  __syncthreads();
  if (w == 0) {
    int64_t t = 0;
    for (int k = 0; k < 32; ++k) t += part[k][lane];
    if (j < d) in[j] = t;
  }
}

struct XrParams {
  int d, c, mode;  // mode 0: AllToAll, 1: AllGather
  double intra_bw, inter_bw, a2a;
};

template <class T, class Op>
__device__ T block_reduce(T v, Op op, T* smem /* [32] */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(~0u, v, o));
  __syncthreads();  // smem may still be read by a previous reduction
  if (lane == 0) smem[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  T r = smem[0];
  for (int k = 1; k < nw; ++k) r = op(r, smem[k]);
  return r;
}

__global__ void __launch_bounds__(kXrThreads, 1)
    k_xr_finish(XrParams p, const int64_t* __restrict__ inter, const int64_t* __restrict__ intra,
                const int64_t* __restrict__ local, const int64_t* __restrict__ in,
                const int64_t* __restrict__ batch_len, int64_t* __restrict__ egress,
                orch_exchange_cost* __restrict__ rep) {
  __shared__ int64_t red[32];
  __shared__ double redt[32];
  __shared__ int redi[32];
  const int t = threadIdx.x, d = p.d, nodes = d / p.c;
  int64_t s_inter = 0, s_intra = 0, s_local = 0, peak = 0, lengths = 0, mx = 0;
  double best_t = 0.0;  // the reference starts from worst_time = 0.0
  int best_i = INT32_MAX;
  for (int i = t; i < d; i += blockDim.x) {
    const int64_t a = inter[i], b = intra[i], l = local[i];
    s_inter += a;
    s_intra += b;
    s_local += l;
    const int64_t out = a + b, inc = in[i];
    const int64_t pk = (inc > out ? inc : out) + l;
    peak = pk > peak ? pk : peak;
    const double ti = __dadd_rn(__ddiv_rn(static_cast<double>(a), p.inter_bw),
                                __ddiv_rn(static_cast<double>(b), p.intra_bw));
    if (ti > best_t) {  // strictly greater: the first i (in order) of the maximum wins
      best_t = ti;
      best_i = i;
    }
    if (batch_len) {
      lengths += batch_len[i];
      mx = batch_len[i] > mx ? batch_len[i] : mx;
    }
  }
  auto add = [](int64_t x, int64_t y) { return x + y; };
  auto maxi = [](int64_t x, int64_t y) { return x > y ? x : y; };
  s_inter = block_reduce<int64_t>(s_inter, add, red);
  s_intra = block_reduce<int64_t>(s_intra, add, red);
  s_local = block_reduce<int64_t>(s_local, add, red);
  peak = block_reduce<int64_t>(peak, maxi, red);
  lengths = block_reduce<int64_t>(lengths, add, red);
  mx = block_reduce<int64_t>(mx, maxi, red);
  // (max t, then lowest i) over the block
  {
    const int lane = t & 31, w = t >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ot = __shfl_xor_sync(~0u, best_t, o);
      const int oi = __shfl_xor_sync(~0u, best_i, o);
      if (ot > best_t || (ot == best_t && oi < best_i)) {
        best_t = ot;
        best_i = oi;
      }
    }
    if (lane == 0) {
      redt[w] = best_t;
      redi[w] = best_i;
    }
    __syncthreads();
    best_t = redt[0];
    best_i = redi[0];
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
      if (redt[k] > best_t || (redt[k] == best_t && redi[k] < best_i)) {
        best_t = redt[k];
        best_i = redi[k];
      }
  }
  // per-node egress: the inter-node volume of the node's c instances
  for (int nd = t; nd < nodes; nd += blockDim.x) {
    int64_t e = 0;
    for (int i = nd * p.c; i < (nd + 1) * p.c; ++i) e += inter[i];
    egress[nd] = e;
  }
  if (t == 0) {
    orch_exchange_cost r{};
    r.total_inter_volume = s_inter;
    r.total_intra_volume = s_intra;
    r.local_volume = s_local;
    if (p.mode == 0) {
      r.modeled_time = __dmul_rn(p.a2a, best_t);
      r.bottleneck = 0;
      if (best_i != INT32_MAX) {  // worst_kind of the first maximal instance
        const double ti = __ddiv_rn(static_cast<double>(inter[best_i]), p.inter_bw);
        const double tb = __ddiv_rn(static_cast<double>(intra[best_i]), p.intra_bw);
        r.bottleneck = ti >= tb ? 2 : 1;
      }
      r.peak_resident_volume = peak;
    } else {
      r.modeled_time = __ddiv_rn(__dmul_rn(static_cast<double>(d - 1), static_cast<double>(mx)),
                                 p.inter_bw);
      r.bottleneck = d > 1 && mx > 0 ? 2 : 0;
      r.peak_resident_volume = lengths;
    }
    r.stale = rep->stale;
    *rep = r;
  }
}

__global__ void k_xr_stale(int64_t count, const int64_t* __restrict__ a,
                           const int64_t* __restrict__ b, orch_exchange_cost* rep) {
  bool diff = false;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    diff |= __ldcs(a + k) != __ldcs(b + k);
  if (__any_sync(~0u, diff) && (threadIdx.x & 31) == 0) rep->stale = 1;
}

__global__ void k_clear_report(orch_exchange_cost* rep) {
  if (threadIdx.x == 0) *rep = orch_exchange_cost{};
}

// make_exchange_plan, AllGather mode (exchange.cpp:17-28): every other
// instance receives instance i's whole batch.
__global__ void k_allgather_volumes(int d, const int64_t* __restrict__ batch_len,
                                    int64_t* __restrict__ V) {
  const int64_t total = static_cast<int64_t>(d) * d;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = k / d, j = k - i * d;
    V[k] = i == j ? 0 : batch_len[i];
  }
}

// validate_topology (topology.cpp:12-22) for (d, c, bandwidths)
int check_topology(int d, int c, double intra_bw, double inter_bw) {
  if (d < 1 || c < 1)
    return fail(ORCH_INVALID_ARGUMENT, "topology needs at least one instance and one per node");
  if (d % c != 0)
    return fail(ORCH_INVALID_ARGUMENT, "instance count must be divisible by instances per node");
  if (!(inter_bw > 0.0) || intra_bw < inter_bw)
    return fail(ORCH_INVALID_ARGUMENT, "bandwidths must satisfy intra >= inter > 0");
  if (d > ORCH_MAX_INSTANCES) return fail(ORCH_UNSUPPORTED, "instance count above ORCH_MAX_INSTANCES");
  return ORCH_OK;
}

}  // namespace
}  // namespace orchb

using namespace orchb;

extern "C" int orch_volume_matrix(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* d_len,
                                  const int32_t* d_origin, const int32_t* d_dest_inst,
                                  int64_t* d_V, void* stream);

extern "C" {

int orch_exchange_report(orch_ctx* ctx, int32_t d, int32_t c, double intra_bw, double inter_bw,
                         double alltoall_constant, int32_t mode, const int64_t* d_V,
                         const int64_t* d_batch_len, int64_t n, const int64_t* d_len,
                         const int32_t* d_src_inst, const int32_t* d_dst_inst,
                         int64_t* d_per_node_egress, orch_exchange_cost* d_report,
                         void* stream) {
  if (!ctx || !d_V || !d_per_node_egress || !d_report)
    return fail(ORCH_INVALID_ARGUMENT, "null argument");
  int rc = check_topology(d, c, intra_bw, inter_bw);
  if (rc) return rc;
  if (mode != 0 && mode != 1) return fail(ORCH_LOGIC_ERROR, "unknown exchange mode");
  if (mode == 1 && !d_batch_len)
    return fail(ORCH_INVALID_ARGUMENT, "the all-gather report needs the batch lengths");
  auto st = static_cast<cudaStream_t>(stream);
  const bool check_stale = d_len && d_src_inst && d_dst_inst && n >= 0;
  Plan plan;
  int64_t *inter, *intra, *local, *in, *fresh = nullptr;
  plan.add(&inter, d);
  plan.add(&intra, d);
  plan.add(&local, d);
  plan.add(&in, d);
  if (check_stale) plan.add(&fresh, static_cast<size_t>(d) * d);
  rc = plan.commit(ctx, st);
  if (rc) return rc;
  ++ctx->launches;
  k_clear_report<<<1, 32, 0, st>>>(d_report);
  if (check_stale) {  // simulate_exchange's stale-plan check (exchange.cpp:57-60)
    rc = orch_volume_matrix(ctx, d, n, d_len, d_src_inst, d_dst_inst, fresh, stream);
    if (rc) return rc;
    ++ctx->launches;
    k_xr_stale<<<blocks_for(static_cast<int64_t>(d) * d, 256), 256, 0, st>>>(
        static_cast<int64_t>(d) * d, d_V, fresh, d_report);
  }
  ctx->launches += 3;
  k_xr_rows<<<blocks_for(static_cast<int64_t>(d) * 32, 256), 256, 0, st>>>(d, c, d_V, inter, intra,
                                                                          local);
  k_xr_cols<<<(d + 31) / 32, kXrThreads, 0, st>>>(d, d_V, in);
  XrParams p{d, c, mode, intra_bw, inter_bw, alltoall_constant};
  k_xr_finish<<<1, kXrThreads, 0, st>>>(p, inter, intra, local, in, d_batch_len,
                                       d_per_node_egress, d_report);
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_exchange_report_host(orch_ctx* ctx, int32_t d, int32_t c, double intra_bw,
                              double inter_bw, double alltoall_constant, int32_t mode,
                              const int64_t* h_V, const int64_t* h_batch_len, int64_t n,
                              const int64_t* h_len, const int32_t* h_src_inst,
                              const int32_t* h_dst_inst, int64_t* h_per_node_egress,
                              orch_exchange_cost* h_report, void* stream) {
  if (!ctx || !h_V || !h_per_node_egress || !h_report)
    return fail(ORCH_INVALID_ARGUMENT, "null argument");
  int rc = check_topology(d, c, intra_bw, inter_bw);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const bool check_stale = h_len && h_src_inst && h_dst_inst && n >= 0;
  const size_t nn = check_stale ? static_cast<size_t>(n) : 0;
  const size_t dd = static_cast<size_t>(d) * d;
  size_t at = 0;
  auto take = [&](size_t b) {
    const size_t r = at;
    at += (b + 255) & ~size_t{255};
    return r;
  };
  const size_t o_V = take(dd * 8), o_bl = take(static_cast<size_t>(d) * 8);
  const size_t o_len = take(nn * 8), o_src = take(nn * 4), o_dst = take(nn * 4);
  const size_t in_bytes = at;
  const size_t o_eg = take(static_cast<size_t>(d / c) * 8), o_rep = take(sizeof(orch_exchange_cost));
  char *hp, *dp;
  rc = host_stage(ctx, at, &hp, &dp);
  if (rc) return rc;
  memcpy(hp + o_V, h_V, dd * 8);
  if (h_batch_len) memcpy(hp + o_bl, h_batch_len, static_cast<size_t>(d) * 8);
  if (nn) {
    memcpy(hp + o_len, h_len, nn * 8);
    memcpy(hp + o_src, h_src_inst, nn * 4);
    memcpy(hp + o_dst, h_dst_inst, nn * 4);
  }
  ORCH_CUDA_TRY(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, st));
  rc = orch_exchange_report(
      ctx, d, c, intra_bw, inter_bw, alltoall_constant, mode,
      reinterpret_cast<const int64_t*>(dp + o_V),
      h_batch_len ? reinterpret_cast<const int64_t*>(dp + o_bl) : nullptr, check_stale ? n : -1,
      check_stale ? reinterpret_cast<const int64_t*>(dp + o_len) : nullptr,
      check_stale ? reinterpret_cast<const int32_t*>(dp + o_src) : nullptr,
      check_stale ? reinterpret_cast<const int32_t*>(dp + o_dst) : nullptr,
      reinterpret_cast<int64_t*>(dp + o_eg), reinterpret_cast<orch_exchange_cost*>(dp + o_rep),
      stream);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(hp + o_eg, dp + o_eg, at - o_eg, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(h_per_node_egress, hp + o_eg, static_cast<size_t>(d / c) * 8);
  memcpy(h_report, hp + o_rep, sizeof(orch_exchange_cost));
  if (h_report->stale)
    return fail(ORCH_INVALID_ARGUMENT, "exchange plan volumes are stale for these batches");
  return ORCH_OK;
}

int orch_allgather_volumes(orch_ctx* ctx, int32_t d, const int64_t* d_batch_len, int64_t* d_V,
                           void* stream) {
  if (!ctx || !d_batch_len || !d_V) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  auto st = static_cast<cudaStream_t>(stream);
  ++ctx->launches;
  k_allgather_volumes<<<blocks_for(static_cast<int64_t>(d) * d, 256), 256, 0, st>>>(d, d_batch_len,
                                                                                   d_V);
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_allgather_volumes_host(orch_ctx* ctx, int32_t d, const int64_t* h_batch_len,
                                int64_t* h_V, void* stream) {
  if (!ctx || !h_batch_len || !h_V) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const size_t o_V = (static_cast<size_t>(d) * 8 + 255) & ~size_t{255};
  const size_t total = o_V + static_cast<size_t>(d) * d * 8;
  char *hp, *dp;
  int rc = host_stage(ctx, total, &hp, &dp);
  if (rc) return rc;
  memcpy(hp, h_batch_len, static_cast<size_t>(d) * 8);
  ORCH_CUDA_TRY(cudaMemcpyAsync(dp, hp, static_cast<size_t>(d) * 8, cudaMemcpyHostToDevice, st));
  rc = orch_allgather_volumes(ctx, d, reinterpret_cast<const int64_t*>(dp),
                              reinterpret_cast<int64_t*>(dp + o_V), stream);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_V, dp + o_V, static_cast<size_t>(d) * d * 8,
                                cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  return ORCH_OK;
}

}  // extern "C"
