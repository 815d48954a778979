// Node-wise ("GPU-wise") hosting: permute which
// instance hosts which destination batch so that the slow links carry as
// little of the rearrangement as possible -- topology.cpp:55-303
// (inter_node_egress, solve_hosting, nodewise_rearrange). On one NVSwitch box
// a "node" is a GPU holding c = d/P logical instances and the slow link is
// NVLink (the fast one is the GPU's own HBM).
//
// solve_hosting is an exact branch and bound in the reference. Here every
// hosting (nodes^d assignments, the balanced ones kept) is scored in
// parallel; the reference's answer is recovered exactly: its incumbents
// (identity, then greedy) win when they are optimal, otherwise the first
// optimal leaf of its depth-first order, whose rank is the mixed-radix number
// of candidate positions (nodes with room, by descending gain, ties by node).
#include <string>

#include "common.cuh"
#include "plan.cuh"

namespace orchb {
namespace {

constexpr int kHostMaxD = 64;

struct HostState {
  int d, c, nodes;
  long long space;                       // balanced hostings: d! / (c!)^nodes
  int64_t gain[kHostMaxD * kHostMaxD];   // [node][batch]
  int64_t node_total[kHostMaxD];
  int32_t order[kHostMaxD];              // branching order (descending regret, stable)
  int32_t incumbent[kHostMaxD];
  int64_t incumbent_value;
  unsigned long long best_value;
  unsigned long long best_key;           // (dfs key << 30) | index
};

__device__ int64_t host_value(const HostState& H, const int32_t* a) {
  int64_t worst = INT64_MIN;
  for (int n = 0; n < H.nodes; ++n) {
    int64_t e = H.node_total[n];
    for (int b = 0; b < H.d; ++b)
      if (a[b] == n) e -= H.gain[n * H.d + b];
    worst = e > worst ? e : worst;
  }
  return worst;
}

// gain, totals, order, incumbents (topology.cpp:195-262): one thread, d <= 64
__global__ void k_host_prep(int d, int c, const int64_t* __restrict__ V, HostState* H) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int nodes = d / c;
  H->d = d;
  H->c = c;
  H->nodes = nodes;
  // multinomial d! / (c!)^nodes built as a product of binomials C(k*c, c)
  long long sp = 1;
  for (int k = 1; k <= nodes; ++k) {
    long long binom = 1;  // C(k*c, c)
    for (int j = 1; j <= c; ++j) binom = binom * ((k - 1) * c + j) / j;
    sp *= binom;
  }
  H->space = sp;
  for (int n = 0; n < nodes; ++n) {
    H->node_total[n] = 0;
    for (int b = 0; b < d; ++b) H->gain[n * d + b] = 0;
  }
  for (int i = 0; i < d; ++i)
    for (int b = 0; b < d; ++b) {
      H->gain[(i / c) * d + b] += V[i * d + b];
      H->node_total[i / c] += V[i * d + b];
    }
  int64_t regret[kHostMaxD];
  for (int b = 0; b < d; ++b) {
    int64_t top = 0, second = 0;
    for (int n = 0; n < nodes; ++n) {
      const int64_t g = H->gain[n * d + b];
      if (g > top) {
        second = top;
        top = g;
      } else if (g > second) {
        second = g;
      }
    }
    regret[b] = top - second;
    H->order[b] = b;
  }
  for (int i = 1; i < d; ++i) {  // stable insertion sort, descending regret
    const int v = H->order[i];
    int j = i - 1;
    while (j >= 0 && regret[H->order[j]] < regret[v]) {
      H->order[j + 1] = H->order[j];
      --j;
    }
    H->order[j + 1] = v;
  }
  int32_t ident[kHostMaxD], greedy[kHostMaxD];
  int room[kHostMaxD];
  for (int b = 0; b < d; ++b) ident[b] = b / c;
  for (int n = 0; n < nodes; ++n) room[n] = c;
  for (int k = 0; k < d; ++k) {
    const int b = H->order[k];
    int pick = -1;
    int64_t pg = -1;
    for (int n = 0; n < nodes; ++n)
      if (room[n] > 0 && H->gain[n * d + b] > pg) {
        pick = n;
        pg = H->gain[n * d + b];
      }
    greedy[b] = pick;
    room[pick] -= 1;
  }
  const int64_t vi = host_value(*H, ident), vg = host_value(*H, greedy);
  const bool g_better = vg < vi;  // offer(greedy) replaces only when strictly better
  for (int b = 0; b < d; ++b) H->incumbent[b] = g_better ? greedy[b] : ident[b];
  H->incumbent_value = g_better ? vg : vi;
  H->best_value = ~0ull;
  H->best_key = ~0ull;
}

// Unrank idx in [0, space) into a balanced hosting (multiset permutation:
// every node exactly c batches). Completions after choosing node n at a
// position = cur * r_n / T (exact), so the counts stay below space.
__device__ __forceinline__ bool decode(const HostState& H, long long idx, int32_t* a) {
  int r[kHostMaxD];
  for (int n = 0; n < H.nodes; ++n) r[n] = H.c;
  long long cur = H.space;
  int T = H.d;
  for (int b = 0; b < H.d; ++b) {
    for (int n = 0; n < H.nodes; ++n) {
      if (r[n] == 0) continue;
      const long long sub = cur * r[n] / T;
      if (idx < sub) {
        a[b] = n;
        cur = sub;
        --r[n];
        --T;
        break;
      }
      idx -= sub;
    }
  }
  return true;
}

__global__ void k_host_min(const HostState* __restrict__ Hp, unsigned long long* best) {
  const HostState& H = *Hp;
  unsigned long long local = ~0ull;
  int32_t a[kHostMaxD];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < H.space;
       i += (long long)gridDim.x * blockDim.x) {
    if (!decode(H, i, a)) continue;
    const unsigned long long v = static_cast<unsigned long long>(host_value(H, a));
    local = v < local ? v : local;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(~0u, local, off);
    local = o < local ? o : local;
  }
  if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(best, local);
}

// rank of an optimal hosting in the reference's depth-first order
__global__ void k_host_first(HostState* __restrict__ Hp) {
  const HostState& H = *Hp;
  const unsigned long long target = H.best_value;
  unsigned long long local = ~0ull;
  int32_t a[kHostMaxD];
  int room[kHostMaxD];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < H.space;
       i += (long long)gridDim.x * blockDim.x) {
    if (!decode(H, i, a)) continue;
    if (static_cast<unsigned long long>(host_value(H, a)) != target) continue;
    for (int n = 0; n < H.nodes; ++n) room[n] = H.c;
    unsigned long long key = 0;
    for (int t = 0; t < H.d; ++t) {
      const int b = H.order[t];
      const int me = a[b];
      const int64_t gm = H.gain[me * H.d + b];
      int pos = 0;  // candidates (room > 0) ahead of `me`: larger gain, or equal gain and lower index
      for (int n = 0; n < H.nodes; ++n) {
        if (n == me || room[n] == 0) continue;
        const int64_t g = H.gain[n * H.d + b];
        pos += (g > gm) || (g == gm && n < me);
      }
      key = key * H.nodes + pos;
      room[me] -= 1;
    }
    const unsigned long long packed = (key << 30) | static_cast<unsigned long long>(i);
    local = packed < local ? packed : local;
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(~0u, local, off);
    local = o < local ? o : local;
  }
  if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(&Hp->best_key, local);
}

// Final hosting, batch -> instance map, egress figures; then the result remap.
__global__ void k_host_finish(const HostState* __restrict__ Hp, const int64_t* __restrict__ V,
                              int32_t* __restrict__ hosting, int32_t* __restrict__ b2i,
                              int64_t* __restrict__ info) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const HostState& H = *Hp;
  int32_t a[kHostMaxD];
  const bool incumbent = static_cast<long long>(H.best_value) >= H.incumbent_value;
  if (incumbent) {
    for (int b = 0; b < H.d; ++b) a[b] = H.incumbent[b];
  } else {
    decode(H, static_cast<long long>(H.best_key & ((1ull << 30) - 1)), a);
  }
  int next[kHostMaxD];
  for (int n = 0; n < H.nodes; ++n) next[n] = n * H.c;
  for (int b = 0; b < H.d; ++b) {  // topology.cpp:283-290: ascending batch order in a node
    hosting[b] = a[b];
    b2i[b] = next[a[b]]++;
  }
  int64_t worst = 0, base = 0;  // inter_node_egress of the solution and of identity hosting
  for (int n = 0; n < H.nodes; ++n) {
    int64_t e = 0, e0 = 0;
    for (int i = n * H.c; i < (n + 1) * H.c; ++i)
      for (int b = 0; b < H.d; ++b) {
        if (a[b] != n) e += V[i * H.d + b];
        if (b / H.c != n) e0 += V[i * H.d + b];
      }
    worst = e > worst ? e : worst;
    base = e0 > base ? e0 : base;
  }
  info[0] = worst;
  info[1] = base;
  info[2] = incumbent ? 0 : 1;
}

// Relabel destination batches: item dest -> b2i[dest]; per-batch arrays and
// the destination CSR permuted accordingly (contents unchanged).
__global__ void k_host_remap(int d, int64_t n, const int32_t* __restrict__ b2i,
                             int32_t* __restrict__ dest_inst, const int32_t* __restrict__ old_cnt,
                             const int64_t* __restrict__ old_len, const int64_t* __restrict__ old_tok,
                             const double* __restrict__ old_cost,
                             const int32_t* __restrict__ old_off,
                             const int32_t* __restrict__ old_mem, int32_t* __restrict__ bin_count,
                             int64_t* __restrict__ bin_len, int64_t* __restrict__ bin_tokens,
                             double* __restrict__ bin_cost, int32_t* __restrict__ bin_offset,
                             int32_t* __restrict__ bin_member) {
  __shared__ int32_t inv[kHostMaxD];
  __shared__ int32_t noff[kHostMaxD + 1];
  if (threadIdx.x < d) inv[b2i[threadIdx.x]] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int j = 0; j < d; ++j) {
      noff[j] = acc;
      acc += old_cnt[inv[j]];
    }
    noff[d] = acc;
  }
  __syncthreads();
  if (threadIdx.x < d) {
    const int j = threadIdx.x, b = inv[j];
    bin_count[j] = old_cnt[b];
    if (bin_len) bin_len[j] = old_len[b];
    if (bin_tokens) bin_tokens[j] = old_tok[b];
    if (bin_cost) bin_cost[j] = old_cost[b];
  }
  if (threadIdx.x <= d) bin_offset[threadIdx.x] = noff[threadIdx.x];
  for (int j = 0; j < d; ++j) {
    const int b = inv[j];
    for (int k = threadIdx.x; k < old_off[b + 1] - old_off[b]; k += blockDim.x)
      bin_member[noff[j] + k] = old_mem[old_off[b] + k];
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dest_inst[i] = b2i[dest_inst[i]];
}

__global__ void k_vol(int d, int64_t n, const int64_t* __restrict__ len,
                      const int32_t* __restrict__ origin, const int32_t* __restrict__ dest,
                      unsigned long long* __restrict__ V) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&V[static_cast<size_t>(origin[i]) * d + dest[i]],
              static_cast<unsigned long long>(len[i]));
}

int check_hosting_args(int d, int c) {
  if (d < 1 || c < 1)
    return fail(ORCH_INVALID_ARGUMENT, "topology needs at least one instance and one per node");
  if (d % c) return fail(ORCH_INVALID_ARGUMENT, "instance count must be divisible by instances per node");
  if (d > kHostMaxD) return fail(ORCH_UNSUPPORTED, "node-wise hosting limited to d <= 64 on the device");
  long double sp = 1;  // d! / (c!)^(d/c)
  for (int i = 1; i <= d; ++i) sp *= i;
  long double cf = 1;
  for (int i = 1; i <= c; ++i) cf *= i;
  for (int k = 0; k < d / c; ++k) sp /= cf;
  if (sp > 1073741824.0L)
    return fail(ORCH_UNSUPPORTED, "node-wise hosting: more than 2^30 balanced hostings (exhaustive device search)");
  return ORCH_OK;
}

}  // namespace
}  // namespace orchb

using namespace orchb;

extern "C" {

int orch_solve_hosting_host(orch_ctx* ctx, int32_t d, int32_t c, const int64_t* h_V,
                            int32_t* h_hosting, int64_t* h_max_egress, int64_t* h_baseline_max,
                            void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  int rc = check_hosting_args(d, c);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  int64_t *V, *info;
  int32_t *hosting, *b2i;
  HostState* H;
  Plan all;
  all.add(&V, static_cast<size_t>(d) * d);
  all.add(&info, 4);
  all.add(&hosting, d);
  all.add(&b2i, d);
  all.add(&H, 1);
  rc = all.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(V, h_V, sizeof(int64_t) * d * d, cudaMemcpyHostToDevice, st));
  k_host_prep<<<1, 32, 0, st>>>(d, c, V, H);
  k_host_min<<<kSMs * 8, 256, 0, st>>>(H, &H->best_value);
  k_host_first<<<kSMs * 8, 256, 0, st>>>(H);
  k_host_finish<<<1, 32, 0, st>>>(H, V, hosting, b2i, info);
  ctx->launches += 4;
  ORCH_CUDA_TRY(cudaGetLastError());
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_hosting, hosting, sizeof(int32_t) * d, cudaMemcpyDeviceToHost, st));
  int64_t hinfo[4];
  ORCH_CUDA_TRY(cudaMemcpyAsync(hinfo, info, sizeof hinfo, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_max_egress) *h_max_egress = hinfo[0];
  if (h_baseline_max) *h_baseline_max = hinfo[1];
  return ORCH_OK;
}

int orch_nodewise(orch_ctx* ctx, int32_t d, int32_t c, int64_t n, const int64_t* d_len,
                  const int32_t* d_origin, const orch_balance_out* bal, int32_t* d_hosting,
                  int32_t* d_batch_to_instance, int64_t* d_info, void* stream) {
  if (!ctx || !bal) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  int rc = check_hosting_args(d, c);
  if (rc) return rc;
  if (!bal->dest_inst || !bal->bin_count || !bal->bin_offset || !bal->bin_member)
    return fail(ORCH_INVALID_ARGUMENT, "orch_nodewise needs dest_inst, bin_count and the CSR");
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  Plan plan;
  unsigned long long* V;
  HostState* H;
  int32_t *hosting, *b2i, *ocnt, *ooff, *omem;
  int64_t *olen, *otok, *info;
  double* ocost;
  plan.add(&V, static_cast<size_t>(d) * d);
  plan.add(&H, 1);
  plan.add_or(&hosting, d_hosting, d);
  plan.add_or(&b2i, d_batch_to_instance, d);
  plan.add_or(&info, d_info, 4);
  plan.add(&ocnt, d);
  plan.add(&ooff, d + 1);
  plan.add(&omem, nn);
  plan.add(&olen, d);
  plan.add(&otok, d);
  plan.add(&ocost, d);
  rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemsetAsync(V, 0, sizeof(uint64_t) * d * d, st));
  if (n > 0)
    k_vol<<<blocks_for(n, 256), 256, 0, st>>>(d, n, d_len, d_origin, bal->dest_inst, V);
  const int64_t* dV = reinterpret_cast<const int64_t*>(V);
  k_host_prep<<<1, 32, 0, st>>>(d, c, dV, H);
  k_host_min<<<kSMs * 8, 256, 0, st>>>(H, &H->best_value);
  k_host_first<<<kSMs * 8, 256, 0, st>>>(H);
  k_host_finish<<<1, 32, 0, st>>>(H, dV, hosting, b2i, info);
  // snapshot the per-batch arrays, then write them back relabelled
  ORCH_CUDA_TRY(cudaMemcpyAsync(ocnt, bal->bin_count, 4 * d, cudaMemcpyDeviceToDevice, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(ooff, bal->bin_offset, 4 * (d + 1), cudaMemcpyDeviceToDevice, st));
  if (n > 0)
    ORCH_CUDA_TRY(cudaMemcpyAsync(omem, bal->bin_member, 4 * n, cudaMemcpyDeviceToDevice, st));
  if (bal->bin_len)
    ORCH_CUDA_TRY(cudaMemcpyAsync(olen, bal->bin_len, 8 * d, cudaMemcpyDeviceToDevice, st));
  if (bal->bin_tokens)
    ORCH_CUDA_TRY(cudaMemcpyAsync(otok, bal->bin_tokens, 8 * d, cudaMemcpyDeviceToDevice, st));
  if (bal->bin_cost)
    ORCH_CUDA_TRY(cudaMemcpyAsync(ocost, bal->bin_cost, 8 * d, cudaMemcpyDeviceToDevice, st));
  k_host_remap<<<1, 256, 0, st>>>(d, n, b2i, bal->dest_inst, ocnt, olen, otok, ocost, ooff, omem,
                                  bal->bin_count, bal->bin_len, bal->bin_tokens, bal->bin_cost,
                                  bal->bin_offset, bal->bin_member);
  ctx->launches += 6;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"
