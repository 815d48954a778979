// Micro-benchmark of the quadratic-tolerance champion scan for d <= 8 (the C5
// shape): cycles per item of the in-kernel variants, all checked against a
// host restatement of balancers.cpp:223-231. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o paper_2503_23830_b200/lib/qt_bench scripts/qt_bench.cu && paper_2503_23830_b200/lib/qt_bench
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

__device__ __forceinline__ bool less_t(int64_t as, int64_t aq, int64_t bs, int64_t bq, int64_t v) {
  const int64_t df = as - bs;
  return (df < 0 ? -df : df) < v ? aq < bq : as < bs;
}

// A: the current kernel's scheme (lane = batch, beats matrix M in registers,
// shuffles for the champion's state, bit-by-bit spread)
__global__ void qt_a(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  int64_t qs = 0, qq = 0;
  uint64_t M = 0;
  const unsigned dm8 = (1u << d) - 1u;
  __syncwarp();
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const int64_t x = x_next;
    if (k + 1 < n) x_next = xs[k + 1];
    const int64_t xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned m = static_cast<unsigned>(M >> (8 * best)) & dm8 & (0xffu << (best + 1));
      if (!m) break;
      best = __ffs(m) - 1;
    }
    const bool me = lane == best;
    if (me) out[k] = static_cast<uint8_t>(lane);
    qs += me ? x : 0;
    qq += me ? xx : 0;
    const int64_t bs = __shfl_sync(~0u, qs, best);
    const int64_t bq = __shfl_sync(~0u, qq, best);
    const bool b_beats_me = lane < d && lane != best && less_t(bs, bq, qs, qq, v);
    const bool i_beat_b = lane < d && lane != best && less_t(qs, qq, bs, bq, v);
    const unsigned col = __ballot_sync(~0u, b_beats_me);
    const unsigned row = __ballot_sync(~0u, i_beat_b);
    uint64_t spread = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) spread |= static_cast<uint64_t>((col >> j) & 1u) << (8 * j);
    M = (M & ~(0x0101010101010101ull << best)) | (spread << best);
    M = (M & ~(0xffull << (8 * best))) | (static_cast<uint64_t>(row) << (8 * best));
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

__device__ __forceinline__ uint64_t spread8(unsigned col) {  // bit j -> bit 8j
  const unsigned lo = ((col & 0xfu) * 0x204081u) & 0x01010101u;
  const unsigned hi = (((col >> 4) & 0xfu) * 0x204081u) & 0x01010101u;
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// B: as A, but every lane keeps all d states (no shuffles: the champion's
// state is a local select), multiply spread
__global__ void qt_b(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  int64_t s[8], q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] = q[j] = 0;
  uint64_t M = 0;
  const unsigned dm8 = (1u << d) - 1u;
  __syncwarp();
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const int64_t x = x_next;
    if (k + 1 < n) x_next = xs[k + 1];
    const int64_t xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned m = static_cast<unsigned>(M >> (8 * best)) & dm8 & (0xffu << (best + 1));
      if (!m) break;
      best = __ffs(m) - 1;
    }
    if (lane == 0) out[k] = static_cast<uint8_t>(best);
    int64_t bs = s[0], bq = q[0], ms = s[0], mq = q[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      if (best == j) { bs = s[j]; bq = q[j]; }
      if (lane == j) { ms = s[j]; mq = q[j]; }
    }
    bs += x;
    bq += xx;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (best == j) { s[j] = bs; q[j] = bq; }
    if (lane == best) { ms = bs; mq = bq; }
    const bool b_beats_me = lane < d && lane != best && less_t(bs, bq, ms, mq, v);
    const bool i_beat_b = lane < d && lane != best && less_t(ms, mq, bs, bq, v);
    const unsigned col = __ballot_sync(~0u, b_beats_me);
    const unsigned row = __ballot_sync(~0u, i_beat_b);
    M = (M & ~(0x0101010101010101ull << best)) | (spread8(col) << best);
    M = (M & ~(0xffull << (8 * best))) | (static_cast<uint64_t>(row) << (8 * best));
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// D: lane = batch keeps its row beats_j; the champion chain is walked on a
// packed next-champion word (4 bits per batch, 15 = none) built by one OR
// reduction, so a walk step is a 32-bit shift and mask
__global__ void qt_d(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  int64_t qs = 0, qq = 0;
  unsigned beats = 0;
  const unsigned dmask = (1u << d) - 1u;
  const unsigned above = lane >= 31 ? 0u : (dmask & (~0u << (lane + 1)));
  unsigned W = 0xffffffffu;  // every batch: no later batch beats it
  __syncwarp();
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const int64_t x = x_next;
    if (k + 1 < n) x_next = xs[k + 1];
    const int64_t xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned t = (W >> (4 * best)) & 0xfu;
      if (t == 0xfu) break;
      best = static_cast<int>(t);
    }
    const bool me = lane == best;
    if (me) out[k] = static_cast<uint8_t>(lane);
    qs += me ? x : 0;
    qq += me ? xx : 0;
    const int64_t bs = __shfl_sync(~0u, qs, best);
    const int64_t bq = __shfl_sync(~0u, qq, best);
    const bool b_beats_me = lane < d && lane != best && less_t(bs, bq, qs, qq, v);
    const bool i_beat_b = lane < d && lane != best && less_t(qs, qq, bs, bq, v);
    const unsigned row = __ballot_sync(~0u, i_beat_b);
    beats = me ? row : ((beats & ~(1u << best)) | (b_beats_me ? 1u << best : 0u));
    const unsigned m = beats & above;
    const unsigned nx = m ? static_cast<unsigned>(__ffs(m) - 1) : 0xfu;
    W = __reduce_or_sync(~0u, lane < 8 ? nx << (4 * lane) : 0u);
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// E: D without divergent branches (every comparison evaluated, results masked)
// lane = batch keeps its row beats_j; the champion chain is walked on a
// packed next-champion word (4 bits per batch, 15 = none) built by one OR
// reduction, so a walk step is a 32-bit shift and mask
__global__ void qt_e(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  int64_t qs = 0, qq = 0;
  unsigned beats = 0;
  const unsigned dmask = (1u << d) - 1u;
  const unsigned above = lane >= 31 ? 0u : (dmask & (~0u << (lane + 1)));
  unsigned W = 0xffffffffu;  // every batch: no later batch beats it
  __syncwarp();
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const int64_t x = x_next;
    if (k + 1 < n) x_next = xs[k + 1];
    const int64_t xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned t = (W >> (4 * best)) & 0xfu;
      if (t == 0xfu) break;
      best = static_cast<int>(t);
    }
    const bool me = lane == best;
    if (lane == 0) out[k] = static_cast<uint8_t>(best);
    qs += me ? x : 0;
    qq += me ? xx : 0;
    const int64_t bs = __shfl_sync(~0u, qs, best);
    const int64_t bq = __shfl_sync(~0u, qq, best);
    const int64_t df = qs - bs;
    const bool near = (df < 0 ? -df : df) < v;
    const bool on = lane < d && !me;
    const bool b_beats_me = on & (near ? bq < qq : bs < qs);
    const bool i_beat_b = on & (near ? qq < bq : qs < bs);
    const unsigned row = __ballot_sync(~0u, i_beat_b);
    beats = me ? row : ((beats & ~(1u << best)) | (b_beats_me ? 1u << best : 0u));
    const unsigned m = beats & above;
    const unsigned nx = m ? static_cast<unsigned>(__ffs(m) - 1) : 0xfu;
    W = __reduce_or_sync(~0u, lane < 8 ? nx << (4 * lane) : 0u);
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// F: E with the sums and square sums in doubles (exact while n * max_len^2 < 2^53)
// lane = batch keeps its row beats_j; the champion chain is walked on a
// packed next-champion word (4 bits per batch, 15 = none) built by one OR
// reduction, so a walk step is a 32-bit shift and mask
__global__ void qt_f(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  const int lane = threadIdx.x;
  double qs = 0, qq = 0;
  unsigned beats = 0;
  const unsigned dmask = (1u << d) - 1u;
  const unsigned above = lane >= 31 ? 0u : (dmask & (~0u << (lane + 1)));
  unsigned W = 0xffffffffu;  // every batch: no later batch beats it
  const double vd = static_cast<double>(v);
  __syncwarp();
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const double x = static_cast<double>(x_next);
    if (k + 1 < n) x_next = xs[k + 1];
    const double xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned t = (W >> (4 * best)) & 0xfu;
      if (t == 0xfu) break;
      best = static_cast<int>(t);
    }
    const bool me = lane == best;
    if (lane == 0) out[k] = static_cast<uint8_t>(best);
    qs += me ? x : 0.0;
    qq += me ? xx : 0.0;
    const double bs = __shfl_sync(~0u, qs, best);
    const double bq = __shfl_sync(~0u, qq, best);
    const bool near = fabs(qs - bs) < vd;
    const bool on = lane < d && !me;
    const bool b_beats_me = on & (near ? bq < qq : bs < qs);
    const bool i_beat_b = on & (near ? qq < bq : qs < bs);
    const unsigned row = __ballot_sync(~0u, i_beat_b);
    beats = me ? row : ((beats & ~(1u << best)) | (b_beats_me ? 1u << best : 0u));
    const unsigned m = beats & above;
    const unsigned nx = m ? static_cast<unsigned>(__ffs(m) - 1) : 0xfu;
    W = __reduce_or_sync(~0u, lane < 8 ? nx << (4 * lane) : 0u);
  }
  const long long t1 = clock64();
  if (lane == 0) *cyc = t1 - t0;
}

// C: one thread, all states in registers, 16 independent comparisons per item
__global__ void qt_c(const int64_t* gxs, int n, int d, int64_t v, uint8_t* out, long long* cyc) {
  __shared__ int64_t xs[512];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = gxs[i];
  __syncthreads();
  if (threadIdx.x) return;
  int64_t s[8], q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] = q[j] = 0;
  uint64_t M = 0;
  const unsigned dm8 = (1u << d) - 1u;
  const long long t0 = clock64();
  int64_t x_next = xs[0];
  for (int k = 0; k < n; ++k) {
    const int64_t x = x_next;
    if (k + 1 < n) x_next = xs[k + 1];
    const int64_t xx = x * x;
    int best = 0;
    for (;;) {
      const unsigned m = static_cast<unsigned>(M >> (8 * best)) & dm8 & (0xffu << (best + 1));
      if (!m) break;
      best = __ffs(m) - 1;
    }
    out[k] = static_cast<uint8_t>(best);
    int64_t bs = s[0], bq = q[0];
#pragma unroll
    for (int j = 1; j < 8; ++j)
      if (best == j) { bs = s[j]; bq = q[j]; }
    bs += x;
    bq += xx;
    unsigned col = 0, row = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (best == j) { s[j] = bs; q[j] = bq; }
      const bool on = j < d && j != best;
      col |= (on && less_t(bs, bq, s[j], q[j], v)) ? 1u << j : 0u;
      row |= (on && less_t(s[j], q[j], bs, bq, v)) ? 1u << j : 0u;
    }
    M = (M & ~(0x0101010101010101ull << best)) | (spread8(col) << best);
    M = (M & ~(0xffull << (8 * best))) | (static_cast<uint64_t>(row) << (8 * best));
  }
  const long long t1 = clock64();
  *cyc = t1 - t0;
}

static bool less_h(int64_t as, int64_t aq, int64_t bs, int64_t bq, int64_t v) {
  return llabs(as - bs) < v ? aq < bq : as < bs;
}

int main() {
  const int d = 8;
  const int64_t v = 2048;
  srand(5);
  for (int n : {64, 128, 512}) {
    std::vector<int64_t> xs(n);
    for (auto& x : xs) x = 8192 + rand() % 24577;
    std::sort(xs.begin(), xs.end(), [](int64_t a, int64_t b) { return a > b; });
    std::vector<uint8_t> ref(n);
    std::vector<int64_t> S(d, 0), Q(d, 0);
    for (int k = 0; k < n; ++k) {
      int best = 0;
      for (int i = 1; i < d; ++i)
        if (less_h(S[i], Q[i], S[best], Q[best], v)) best = i;
      ref[k] = best;
      S[best] += xs[k];
      Q[best] += xs[k] * xs[k];
    }
    int64_t* dx;
    uint8_t* dout;
    long long* dc;
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dout, n);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dx, xs.data(), n * 8, cudaMemcpyHostToDevice);
    const char* names[6] = {"A current", "B replicated", "C one thread", "D packed next",
                            "E branch-free", "F doubles"};
    for (int var = 0; var < 6; ++var) {
      long long best_c = 1ll << 60;
      for (int r = 0; r < 5; ++r) {
        cudaMemset(dout, 0xff, n);
        if (var == 0) qt_a<<<1, 32>>>(dx, n, d, v, dout, dc);
        if (var == 1) qt_b<<<1, 32>>>(dx, n, d, v, dout, dc);
        if (var == 2) qt_c<<<1, 32>>>(dx, n, d, v, dout, dc);
        if (var == 3) qt_d<<<1, 32>>>(dx, n, d, v, dout, dc);
        if (var == 4) qt_e<<<1, 32>>>(dx, n, d, v, dout, dc);
        if (var == 5) qt_f<<<1, 32>>>(dx, n, d, v, dout, dc);
        long long c = -1;
        const cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) printf("variant %d: %s\n", var, cudaGetErrorString(err));
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        cudaMemset(dc, 0, 8);
        best_c = c < best_c ? c : best_c;
      }
      std::vector<uint8_t> got(n);
      cudaMemcpy(got.data(), dout, n, cudaMemcpyDeviceToHost);
      printf("n=%4d %-14s %7lld cycles, %6.1f per item, %s\n", n, names[var], best_c,
             double(best_c) / n, got == ref ? "match" : "MISMATCH");
    }
    cudaFree(dx);
    cudaFree(dout);
    cudaFree(dc);
  }
  return 0;
}
