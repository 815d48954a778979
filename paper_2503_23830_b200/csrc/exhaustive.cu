// oracle_optimal (balancers.cpp:309-413) as a brute-force sm_100a kernel:
// every assignment of the descending-sorted items to d batches is one index
// of a base-d number (item 0 most significant); canonical assignments (item k
// may only open batch max_so_far + 1, the reference's symmetry pruning) are
// scored with the cost model, the minimum objective is found, and among the
// optimal ones the smallest index -- the first leaf the reference's
// depth-first search reaches with that value -- is returned.
#include <string>

#include "common.cuh"
#include "plan.cuh"

namespace orchb {
namespace {

constexpr int kMaxOracleItems = 24;

// Total order on doubles as unsigned integers.
__device__ __forceinline__ unsigned long long order_key(double x) {
  const unsigned long long b = __double_as_longlong(x);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

struct Sorted {
  int n;
  int d;
  long long total;  // d^n
  int64_t len[kMaxOracleItems];
  int order[kMaxOracleItems];
};

// Stable descending sort of <= 24 lengths (balancers.cpp:393-396).
__global__ void k_sort_small(int n, int d, const int64_t* __restrict__ len, Sorted* s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  s->n = n;
  s->d = d;
  long long t = 1;
  for (int i = 0; i < n; ++i) t *= d;
  s->total = t;
  for (int i = 0; i < n; ++i) s->order[i] = i;
  for (int i = 1; i < n; ++i) {  // insertion sort keeps ties in input order
    const int o = s->order[i];
    int j = i - 1;
    while (j >= 0 && len[s->order[j]] < len[o]) {
      s->order[j + 1] = s->order[j];
      --j;
    }
    s->order[j + 1] = o;
  }
  for (int i = 0; i < n; ++i) s->len[i] = len[s->order[i]];
}

__device__ __forceinline__ bool score(const Sorted& s, const orch_cost_model& m, long long idx,
                                      double* obj) {
  int64_t cnt[4] = {0, 0, 0, 0}, sum[4] = {0, 0, 0, 0}, sq[4] = {0, 0, 0, 0},
          mx[4] = {0, 0, 0, 0};
  long long rest = idx;
  long long place = s.total / s.d;
  int hi = -1;
  for (int k = 0; k < s.n; ++k) {
    const int a = static_cast<int>(rest / place);
    rest -= a * place;
    if (k + 1 < s.n) place /= s.d;
    if (a > hi + 1) return false;  // not canonical
    hi = a > hi ? a : hi;
    const int64_t l = s.len[k];
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b == a) {
        cnt[b] += 1;
        sum[b] += l;
        sq[b] += l * l;
        mx[b] = l > mx[b] ? l : mx[b];
      }
  }
  double best = 0.0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (b >= s.d) break;
    // cost_of (balancers.cpp:325-345): square sum as an int64 cast to double
    const double c = batch_cost(m, cnt[b], sum[b], mx[b], static_cast<double>(sq[b]));
    best = c > best ? c : best;
  }
  *obj = best;
  return true;
}

__global__ void k_exhaustive_min(const Sorted* __restrict__ sp, orch_cost_model m,
                                 unsigned long long* __restrict__ best) {
  const Sorted s = *sp;
  unsigned long long local = ~0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < s.total;
       i += (long long)gridDim.x * blockDim.x) {
    double obj;
    if (score(s, m, i, &obj)) {
      const unsigned long long k = order_key(obj);
      local = k < local ? k : local;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(~0u, local, off);
    local = o < local ? o : local;
  }
  if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(best, local);
}

__global__ void k_exhaustive_first(const Sorted* __restrict__ sp, orch_cost_model m,
                                   const unsigned long long* __restrict__ best,
                                   unsigned long long* __restrict__ first) {
  const Sorted s = *sp;
  const unsigned long long target = *best;
  unsigned long long local = ~0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < s.total;
       i += (long long)gridDim.x * blockDim.x) {
    double obj;
    if (score(s, m, i, &obj) && order_key(obj) == target) {
      local = static_cast<unsigned long long>(i);
      break;  // grid-stride order: later i of this thread are larger
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(~0u, local, off);
    local = o < local ? o : local;
  }
  if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(first, local);
}

__global__ void k_exhaustive_emit(const Sorted* __restrict__ sp,
                                  const unsigned long long* __restrict__ best,
                                  const unsigned long long* __restrict__ first,
                                  int32_t* __restrict__ assignment, double* __restrict__ objective) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Sorted& s = *sp;
  long long rest = static_cast<long long>(*first);
  long long place = s.total / s.d;
  for (int k = 0; k < s.n; ++k) {
    const int a = static_cast<int>(rest / place);
    rest -= a * place;
    if (k + 1 < s.n) place /= s.d;
    assignment[s.order[k]] = a;
  }
  const unsigned long long key = *best;
  const unsigned long long b = (key >> 63) ? (key & ~(1ull << 63)) : ~key;
  *objective = __longlong_as_double(static_cast<long long>(b));
}

}  // namespace
}  // namespace orchb

using namespace orchb;

extern "C" int orch_oracle_optimal_host(orch_ctx* ctx, const orch_cost_model* model, int32_t d,
                                        int64_t n, const int64_t* h_len, int32_t max_items,
                                        int32_t max_instances, int32_t* h_assignment,
                                        double* h_objective, void* stream) {
  if (!ctx || !model) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  if (n > max_items || d > max_instances)
    return fail(ORCH_SIZE_CAP, "oracle instance exceeds caps (n <= " + std::to_string(max_items) +
                                   ", d <= " + std::to_string(max_instances) + ")");
  if (n == 0) {
    *h_objective = 0.0;
    return ORCH_OK;
  }
  long double space = 1;
  for (int i = 0; i < n; ++i) space *= d;
  if (d > 4 || n > kMaxOracleItems || space > 68719476736.0L)
    return fail(ORCH_UNSUPPORTED, "exhaustive oracle limited to d <= 4 and d^n <= 2^36 on the device");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  Plan plan;
  Sorted* s;
  int64_t* len;
  unsigned long long* keys;
  int32_t* assign;
  double* obj;
  plan.add(&s, 1);
  plan.add(&len, static_cast<size_t>(n));
  plan.add(&keys, 2);
  plan.add(&assign, static_cast<size_t>(n));
  plan.add(&obj, 1);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(len, h_len, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(keys, 0xff, 2 * sizeof(unsigned long long), st));
  k_sort_small<<<1, 32, 0, st>>>(static_cast<int>(n), d, len, s);
  const int grid = kSMs * 16;
  k_exhaustive_min<<<grid, 256, 0, st>>>(s, *model, keys);
  k_exhaustive_first<<<grid, 256, 0, st>>>(s, *model, keys, keys + 1);
  k_exhaustive_emit<<<1, 32, 0, st>>>(s, keys, keys + 1, assign, obj);
  ctx->launches += 4;
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_assignment, assign, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_objective, obj, sizeof(double), cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  return ORCH_OK;
}
