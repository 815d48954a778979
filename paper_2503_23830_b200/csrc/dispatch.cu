// Send/recv layout and token-row movement of the exchange (C-ABI
// orch_volume_matrix / orch_layout / orch_dispatch), cost model entry points
// and the NCCL communicator. Row movement realises apply() (core.cpp:120-161)
// on bf16 token rows: every item is a contiguous run of len rows in its origin
// rank's input buffer and lands as a contiguous run in its destination rank's
// output buffer; off-rank runs travel through one grouped NCCL send/recv.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "balance_kernels.cuh"
#include "plan.cuh"
#include "radix.cuh"

struct orch_comm {
  ncclComm_t comm = nullptr;
  int rank = 0;
  int size = 1;
  int device = 0;
  int32_t* barrier_buf = nullptr;  // 1 int on the device (ncclAllReduce barrier)
  bool loopback = false;           // orch_comm_create_local: P ranks emulated in one process
};

// A row buffer every rank of the communicator can store into (CUDA IPC over
// NVLink): the fused pack+put exchange writes rows straight into the
// destination rank's output, one pass, no staging buffers.
// Flag area after the rows, at flags_off (256 bytes):
//   arrive[8] u64 : arrive[q] = the last barrier rank q has published here
//   free[8]   u64 : free[q]   = the last step whose rows rank q has consumed
//                                from ITS window (so this rank may put again)
//   status    i32 : this rank's barrier / put-wait timeout (ORCH_CUDA_ERROR)
struct orch_window {
  orch_comm* comm = nullptr;
  char* base = nullptr;
  size_t bytes = 0;
  size_t flags_off = 0;           // the flag area (IPC-shared with the rows)
  uint64_t epoch = 0;             // orch_window_barrier calls so far (equal on every rank)
  uint64_t released = 0;          // orch_window_release calls so far
  uint64_t acq_epoch = 0;         // the step the last k_window_acquire waited for ...
  void* acq_stream = nullptr;     // ... and its stream
  std::vector<char*> peers;       // host copy, peers[rank] == base
  char** peers_dev = nullptr;     // device copy [P]
  bool loopback = false;          // peers are other windows of this process (no IPC)
  ncclWindow_t nccl_win = nullptr;  // orch_window_create_nccl: NCCL symmetric memory
};

struct orch_gather_window {
  orch_window* w = nullptr;
  uint64_t* stamps = nullptr;  // device [8][8]
  int64_t max_n = 0;
  uint64_t epoch = 0;  // calls made so far (the same count on every rank)
};

namespace orchb {

// nccl_window.cu: every rank's address of an NCCL symmetric window (the device
// API's ncclGetPeerPointer lives in its own translation unit)
cudaError_t nccl_window_peers(ncclWindow_t win, int P, char** peers_dev);

namespace {

constexpr int kThreads = 256;
constexpr int kMoveThreads = 256;
constexpr int kUnitRows = 8;  // rows per work unit of the movement kernels

template <class F>
void launch(orch_ctx* ctx, F&& f) {
  f();
  ++ctx->launches;
}

#define ORCH_NCCL_TRY(expr)                                                          \
  do {                                                                              \
    ncclResult_t r_ = (expr);                                                       \
    if (r_ != ncclSuccess)                                                          \
      return ::orchb::fail(ORCH_NCCL_ERROR, std::string(#expr ": ") + ncclGetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------ volume matrix
// topology.cpp:40-53: V[src][dst] += length. Integer atomics: exact and
// order-independent.
__global__ void k_volume(int d, int64_t n, const int64_t* __restrict__ len,
                         const int32_t* __restrict__ origin, const int32_t* __restrict__ dest,
                         unsigned long long* __restrict__ V) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
  {
    ORCH_DCHECK(origin[i] >= 0 && origin[i] < d && dest[i] >= 0 && dest[i] < d);
    atomicAdd(&V[static_cast<size_t>(origin[i]) * d + dest[i]],
              static_cast<unsigned long long>(len[i]));
  }
}

// ------------------------------------------------------------------ layout
// Per-instance token totals of the origin and destination batches.
__global__ void k_inst_rows(int64_t n, const int64_t* __restrict__ len,
                            const int32_t* __restrict__ origin, const int32_t* __restrict__ dest,
                            unsigned long long* __restrict__ inst_in,
                            unsigned long long* __restrict__ inst_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&inst_in[origin[i]], static_cast<unsigned long long>(len[i]));
    atomicAdd(&inst_out[dest[i]], static_cast<unsigned long long>(len[i]));
  }
}

// Instance bases inside their rank buffers (instances of a rank are
// consecutive): one thread per rank.
__global__ void k_inst_bases(int d, int P, const unsigned long long* __restrict__ inst_in,
                             const unsigned long long* __restrict__ inst_out,
                             int64_t* __restrict__ base_in, int64_t* __restrict__ base_out,
                             int64_t* __restrict__ in_rows, int64_t* __restrict__ out_rows) {
  const int c = d / P;
  for (int r = threadIdx.x; r < P; r += blockDim.x) {
    int64_t a = 0, b = 0;
    for (int i = r * c; i < (r + 1) * c; ++i) {
      base_in[i] = a;
      base_out[i] = b;
      a += static_cast<int64_t>(inst_in[i]);
      b += static_cast<int64_t>(inst_out[i]);
    }
    in_rows[r] = a;
    out_rows[r] = b;
  }
}

__global__ void k_rank_offsets(int64_t n, const int32_t* __restrict__ origin,
                               const int32_t* __restrict__ dest, const int64_t* __restrict__ src_off,
                               const int64_t* __restrict__ dst_off,
                               const int64_t* __restrict__ base_in,
                               const int64_t* __restrict__ base_out,
                               int64_t* __restrict__ rank_src_off,
                               int64_t* __restrict__ rank_dst_off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    rank_src_off[i] = base_in[origin[i]] + src_off[i];
    rank_dst_off[i] = base_out[dest[i]] + dst_off[i];
  }
}

// Within destination batch j (slot order), the running row offset of each
// item among items from the same ORIGIN RANK (P <= 8 lanes of warp scans per
// 32 items), plus the per-(batch, origin rank) totals W[j*P + q]. One warp.
__device__ __forceinline__ void pair_within_batch(int j, int P, int c,
                                                  const int32_t* __restrict__ bin_offset,
                                                  const int32_t* __restrict__ bin_member,
                                                  const int64_t* __restrict__ len,
                                                  const int32_t* __restrict__ origin,
                                                  int64_t* __restrict__ pair_off, int64_t* W) {
  const int lane = threadIdx.x & 31;
  int64_t run[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int beg = bin_offset[j], end = bin_offset[j + 1];
  for (int base = beg; base < end; base += 32) {
    const int k = base + lane;
    int32_t pos = 0, r = -1;
    int64_t l = 0;
    if (k < end) {
      pos = bin_member[k];
      l = len[pos];
      r = origin[pos] / c;
    }
    int64_t mine = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q >= P) break;
      int64_t v = r == q ? l : 0;
      int64_t incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t o = __shfl_up_sync(~0u, incl, off);
        if (lane >= off) incl += o;
      }
      if (r == q) mine = run[q] + incl - v;
      run[q] += __shfl_sync(~0u, incl, 31);
    }
    if (k < end) pair_off[pos] = mine;
  }
  if (lane < P) {
    int64_t v = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == lane) v = run[q];
    W[j * P + lane] = v;
  }
}

__global__ void k_pair_within(int d, int P, const int32_t* __restrict__ bin_offset,
                              const int32_t* __restrict__ bin_member,
                              const int64_t* __restrict__ len, const int32_t* __restrict__ origin,
                              int64_t* __restrict__ pair_off, int64_t* __restrict__ W) {
  const int c = d / P;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < d; j += warps)
    pair_within_batch(static_cast<int>(j), P, c, bin_offset, bin_member, len, origin, pair_off, W);
}

// Segment bases: for dest rank q and origin rank r, the rows from r into the
// batches of q before batch j; per-pair send counts and NCCL displacements.
__global__ void k_pair_bases(int d, int P, const int64_t* __restrict__ W,
                             int64_t* __restrict__ Wbase, int64_t* __restrict__ send_rows,
                             int64_t* __restrict__ send_displ, int64_t* __restrict__ recv_displ) {
  const int c = d / P;
  const int t = threadIdx.x;
  if (t < P * P) {
    const int q = t / P, r = t % P;
    int64_t acc = 0;
    for (int j = q * c; j < (q + 1) * c; ++j) {
      Wbase[j * P + r] = acc;
      acc += W[j * P + r];
    }
    send_rows[r * P + q] = acc;
  }
  __syncthreads();
  if (t < P) {  // rank t's send buffer: segments q != t in q order
    int64_t a = 0;
    for (int q = 0; q < P; ++q) {
      send_displ[t * P + q] = q == t ? 0 : a;
      if (q != t) a += send_rows[t * P + q];
    }
    int64_t b = 0;  // rank t's recv buffer: segments r != t in r order
    for (int r = 0; r < P; ++r) {
      recv_displ[t * P + r] = r == t ? 0 : b;
      if (r != t) b += send_rows[r * P + t];
    }
  }
}

__global__ void k_pair_apply(int64_t n, int d, int P, const int32_t* __restrict__ origin,
                             const int32_t* __restrict__ dest, const int64_t* __restrict__ Wbase,
                             int64_t* __restrict__ pair_off) {
  const int c = d / P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pair_off[i] += Wbase[static_cast<int64_t>(dest[i]) * P + origin[i] / c];
}

// The whole layout of a small phase in one CTA (n <= kLayoutSmallItems,
// d <= kLayoutSmallD): the six kernels above with their intermediates in
// shared memory. The metadata chain of C1-C3 and C5 is latency-bound; this
// saves five launches and the three memsets.
constexpr int kLayoutSmallItems = 16384;
constexpr int kLayoutSmallD = 256;
constexpr int kLayoutSmallThreads = 1024;

__global__ void __launch_bounds__(kLayoutSmallThreads, 1)
    k_layout_small(int n, int d, int P, const int64_t* __restrict__ len,
                   const int32_t* __restrict__ origin, orch_balance_out bal, orch_layout_out L) {
  __shared__ unsigned long long inst_in[kLayoutSmallD], inst_out[kLayoutSmallD];
  __shared__ int64_t base_in[kLayoutSmallD], base_out[kLayoutSmallD];
  __shared__ int64_t W[kLayoutSmallD * 8], Wbase[kLayoutSmallD * 8];
  const int t = threadIdx.x, c = d / P;
  if (t == 0) *L.status = 0;
  for (int i = t; i < d; i += blockDim.x) inst_in[i] = inst_out[i] = 0;
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) {  // k_inst_rows
    ORCH_DCHECK(origin[i] >= 0 && origin[i] < d && bal.dest_inst[i] >= 0 && bal.dest_inst[i] < d);
    const unsigned long long l = static_cast<unsigned long long>(len[i]);
    atomicAdd(&inst_in[origin[i]], l);
    atomicAdd(&inst_out[bal.dest_inst[i]], l);
  }
  __syncthreads();
  if (t < P) {  // k_inst_bases
    int64_t a = 0, b = 0;
    for (int i = t * c; i < (t + 1) * c; ++i) {
      base_in[i] = a;
      base_out[i] = b;
      a += static_cast<int64_t>(inst_in[i]);
      b += static_cast<int64_t>(inst_out[i]);
    }
    L.in_rows[t] = a;
    L.out_rows[t] = b;
  }
  // k_pair_within: warp per destination batch (reads only the balance outputs)
  for (int j = t >> 5; j < d; j += blockDim.x >> 5)
    pair_within_batch(j, P, c, bal.bin_offset, bal.bin_member, len, origin, L.pair_off, W);
  __syncthreads();
  if (t < P * P) {  // k_pair_bases
    const int q = t / P, r = t % P;
    int64_t acc = 0;
    for (int j = q * c; j < (q + 1) * c; ++j) {
      Wbase[j * P + r] = acc;
      acc += W[j * P + r];
    }
    L.send_rows[r * P + q] = acc;
  }
  __syncthreads();
  if (t < P) {
    int64_t a = 0;
    for (int q = 0; q < P; ++q) {
      L.send_displ[t * P + q] = q == t ? 0 : a;
      if (q != t) a += L.send_rows[t * P + q];
    }
    int64_t b = 0;
    for (int r = 0; r < P; ++r) {
      L.recv_displ[t * P + r] = r == t ? 0 : b;
      if (r != t) b += L.send_rows[r * P + t];
    }
  }
  for (int i = t; i < n; i += blockDim.x) {  // k_rank_offsets + k_pair_apply
    const int o = origin[i], de = bal.dest_inst[i];
    L.rank_src_off[i] = base_in[o] + bal.src_off[i];
    L.rank_dst_off[i] = base_out[de] + bal.dst_off[i];
    L.pair_off[i] += Wbase[de * P + o / c];
  }
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// spin until *p >= want; false after ~4 s (a peer that never arrives)
__device__ bool wait_at_least(const uint64_t* p, uint64_t want) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < want) {
    __nanosleep(64);
    if (clock64() - t0 > 8000000000ll) return false;
  }
  return true;
}

constexpr size_t kFlagFree = 64;     // byte offset of free[] in the flag area
constexpr size_t kFlagStatus = 128;  // byte offset of the status word
constexpr size_t kFlagAcquired = 136;  // byte offset of the acquired step (u64)
constexpr size_t kFlagBytes = 256;

// Window barrier: lane q publishes this rank's epoch in rank q's arrive[me]
// (release, system scope: the stream's earlier kernels -- the puts into the
// peers' windows -- are complete, and the fence orders them before the flag),
// then waits until rank q's epoch is in this rank's arrive[q] (acquire). A
// peer that never arrives (~4 s) sets the window's status instead of hanging.
__global__ void k_window_barrier(char* const* __restrict__ peers, size_t flags_off, int me, int P,
                                 uint64_t epoch, int32_t* status) {
  const int q = threadIdx.x;
  if (q < P) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint64_t*>(peers[q] + flags_off) + me, epoch);
    if (!wait_at_least(reinterpret_cast<const uint64_t*>(peers[me] + flags_off) + q, epoch))
      atomicExch(status, ORCH_CUDA_ERROR);
  }
  __syncwarp();
}

// Window acquire (before the first put of a step on a stream): one warp waits
// until every rank q has released `need` steps (free[q] >= need), then records
// `need` as acquired. The puts that follow on the stream store only when the
// acquired step has reached their own `need` (a timed-out acquire, ~4 s, sets
// the window status and leaves it behind, so they store nothing). The wait
// occupies one warp, not the put kernel's CTAs, so a consumer kernel of any
// size can still run and release.
__global__ void k_window_acquire(const uint64_t* __restrict__ free_flags, int P, uint64_t need,
                                 uint64_t* acquired, int32_t* status) {
  const int q = threadIdx.x;
  const bool ok = q >= P || wait_at_least(free_flags + q, need);
  if (__all_sync(~0u, ok)) {
    if (q == 0) *acquired = need;
  } else if (q == 0) {
    atomicExch(status, ORCH_CUDA_ERROR);
  }
}

// Window release: the rows of step `released` have been consumed on this rank
// (every earlier kernel of the stream has finished reading them); lane q
// tells rank q by storing the count into rank q's free[me]. A put issued
// after barrier e waits for free[q] >= e on every rank q before it stores.
__global__ void k_window_release(char* const* __restrict__ peers, size_t flags_off, int me, int P,
                                 uint64_t released) {
  const int q = threadIdx.x;
  if (q < P)
    st_release_sys(reinterpret_cast<uint64_t*>(peers[q] + flags_off + kFlagFree) + me, released);
}

// ---------------------------------------------------------------- movement
// Work units of kUnitRows rows along an iteration buffer (a rank's input or
// output buffer). unit_first[u] = slice index of the item holding row
// u*kUnitRows. Items are >= 1 row, so a unit touches at most kUnitRows items.
// The slice [offs[lo], offs[hi]) of a CSR is read on the device.
__global__ void k_unit_map(const int32_t* __restrict__ offs, int lo_idx, int hi_idx,
                           const int32_t* __restrict__ members,
                           const int64_t* __restrict__ iter_off,
                           const int64_t* __restrict__ iter_rows, int me, int64_t unit_bytes,
                           int64_t R, int32_t* __restrict__ unit_first, int64_t cap_units,
                           unsigned long long* __restrict__ chunk_counter) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && chunk_counter) *chunk_counter = 0;
  const int64_t beg = offs[lo_idx], end = offs[hi_idx];
  int64_t units = (iter_rows[me] * R + unit_bytes - 1) / unit_bytes;
  units = units < cap_units ? units : cap_units;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = u * unit_bytes / R;  // the row holding the unit's first byte
    int64_t lo = beg, hi = end - 1;  // last k with iter_off[members[k]] <= row
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (iter_off[members[mid]] <= row) lo = mid; else hi = mid - 1;
    }
    unit_first[u] = static_cast<int32_t>(lo - beg);
  }
}

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

#ifdef ORCH_BOUNDS_CHECK
// [p, p + bytes) inside [base, base + cap_bytes) (bounds-checked builds)
__device__ __forceinline__ bool within(const void* p, int64_t bytes, const void* base,
                                       int64_t cap_bytes) {
  const char* c = static_cast<const char*>(p);
  const char* b = static_cast<const char*>(base);
  return bytes >= 0 && c >= b && c + bytes <= b + cap_bytes;
}

// Rows this rank receives from its peers (the recv buffer's extent).
__device__ __forceinline__ int64_t recv_rows_of(const int64_t* send_rows, int P, int me) {
  int64_t t = 0;
  for (int r = 0; r < P; ++r)
    if (r != me) t += send_rows[r * P + me];
  return t;
}
#endif

// Clips the segment run [p0, p0 + cnt) to [lo, hi); false when nothing is left.
// shift = how far the run's start moved (the same shift applies to the other side).
__device__ __forceinline__ bool clip_run(int64_t& p0, int64_t& cnt, int64_t lo, int64_t hi,
                                         int64_t& shift) {
  const int64_t a0 = p0 > lo ? p0 : lo, a1 = p0 + cnt < hi ? p0 + cnt : hi;
  if (a1 <= a0) return false;
  shift = a0 - p0;
  p0 = a0;
  cnt = a1 - a0;
  return true;
}

// Block-wide copy of nvec 16-byte vectors, 4 loads in flight per thread.
__device__ __forceinline__ void block_copy(int4* __restrict__ dst, const int4* __restrict__ src,
                                           int64_t nvec) {
  constexpr int U = 4;
  int64_t v = threadIdx.x;
  for (; v + (U - 1) * kMoveThreads < nvec; v += U * kMoveThreads) {
    int4 t[U];
#pragma unroll
    for (int j = 0; j < U; ++j) t[j] = ld_stream(src + v + j * kMoveThreads);
#pragma unroll
    for (int j = 0; j < U; ++j) st_stream(dst + v + j * kMoveThreads, t[j]);
  }
  for (; v < nvec; v += kMoveThreads) st_stream(dst + v, ld_stream(src + v));
}

enum MoveMode { kLocal = 0, kPack = 1, kUnpack = 2, kPut = 3 };

struct MoveArgs {
  int me, P, c;
  const int32_t* offs;  // CSR offsets of the iteration order
  int lo_idx, hi_idx;
  const int32_t* members;
  const int64_t* iter_rows;  // [P] rows of the iterated buffer per rank
  int64_t iter_cap;          // capacity of the iterated buffer (rows)
  int64_t out_cap;           // capacity of the output buffer (rows)
  const int64_t* out_rows;   // [P]
  const int64_t* in_rows;    // [P]
  int64_t in_cap;            // capacity of the input buffer (rows)
  const int64_t* send_rows;  // [P*P]
  int64_t send_cap;
  const int64_t* len;
  const int32_t* origin;
  const int32_t* dest;
  const int64_t* rank_src_off;
  const int64_t* rank_dst_off;
  const int64_t* pair_off;
  const int64_t* displ;  // send_displ row of me (pack) / recv_displ row of me (unpack)
  const int32_t* unit_first;
  char* const* peer_out;  // kPut: output buffer of every rank (IPC-mapped), [P]
  size_t win_off;         // kPut: byte offset of this exchange's output in every window
  const uint64_t* acquired;    // kPut: the window's acquired step (k_window_acquire)
  uint64_t need_free;          // kPut: ... must have reached this, else nothing is stored
  unsigned long long* chunk_counter;  // TMA path: next unclaimed chunk (zeroed by k_unit_map)
  int scramble;                       // kPut: claim chunk batches in a scrambled order
  // Sliced NCCL exchange (orch_dispatch_nccl): move only the rows whose
  // position in their (origin rank -> dest rank) segment lies in
  // [slo[peer], shi[peer]) -- peer = dest rank (kPack) / origin rank (kUnpack);
  // skip_local leaves the rows that stay on the rank to another round.
  int clip, skip_local;
  int64_t slo[8], shi[8];
  int32_t* status;
  size_t R;
  const char* in;
  char* out;
  char* send;
  const char* recv;
};

// Persistent movement kernel. Iterates the units of one rank buffer:
//   kLocal : output buffer order, in -> out                     (one rank)
//   kPack  : input buffer order, in -> out (item stays on rank) or -> send
//   kUnpack: output buffer order, recv -> out (off-rank items only)
template <int MODE>
__global__ void __launch_bounds__(kMoveThreads) k_move(MoveArgs a) {
  const int64_t total = a.iter_rows[a.me];
  bool over = total > a.iter_cap || a.out_rows[a.me] > a.out_cap;
  if (MODE != kUnpack) over = over || a.in_rows[a.me] > a.in_cap;
  if (MODE == kPut)  // every rank's window has the same capacity
    for (int q = 0; q < a.P; ++q) over = over || a.out_rows[q] > a.out_cap;
  if (MODE == kPack && a.send) {
    int64_t st = 0;
    for (int q = 0; q < a.P; ++q)
      if (q != a.me) st += a.send_rows[a.me * a.P + q];
    over = over || st > a.send_cap;
  }
  if (over) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = ORCH_INVALID_ARGUMENT;
    return;
  }
  if (MODE == kPut && *a.acquired < a.need_free) {  // k_window_acquire timed out
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(a.status, ORCH_CUDA_ERROR);
    return;
  }
  const int64_t beg = a.offs[a.lo_idx], end = a.offs[a.hi_idx];
  const int64_t units = (total + kUnitRows - 1) / kUnitRows;
  const int64_t vrow = static_cast<int64_t>(a.R / 16);
  const size_t R = a.R;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t row0 = u * kUnitRows;
    const int64_t row1 = row0 + kUnitRows < total ? row0 + kUnitRows : total;
    for (int64_t k = beg + a.unit_first[u]; k < end; ++k) {
      const int32_t pos = a.members[k];
      const int64_t off =
          (MODE == kPack || MODE == kPut) ? a.rank_src_off[pos] : a.rank_dst_off[pos];
      if (off >= row1) break;
      const int64_t l = a.len[pos];
      const int64_t lo = off > row0 ? off : row0;
      const int64_t hi = off + l < row1 ? off + l : row1;
      const int64_t skip = lo - off;
      const char* s;
      char* t;
      int64_t cnt = hi - lo;
      if (MODE == kLocal) {
        s = a.in + (a.rank_src_off[pos] + skip) * R;
        t = a.out + lo * R;
      } else if (MODE == kPack) {
        s = a.in + lo * R;
        const int q = a.dest[pos] / a.c;
        if (q == a.me) {
          if (a.skip_local) continue;
          t = a.out + (a.rank_dst_off[pos] + skip) * R;
        } else {
          if (!a.send) continue;  // local rows only (orch_dispatch_nccl, direct)
          int64_t p0 = a.pair_off[pos] + skip, sh = 0;
          if (a.clip && !clip_run(p0, cnt, a.slo[q], a.shi[q], sh)) continue;
          s += sh * R;
          t = a.send + (a.displ[q] + p0) * R;
        }
      } else if (MODE == kPut) {  // straight into the destination rank's output (NVLink)
        s = a.in + lo * R;
        t = a.peer_out[a.dest[pos] / a.c] + a.win_off + (a.rank_dst_off[pos] + skip) * R;
      } else {
        const int r = a.origin[pos] / a.c;
        if (r == a.me) continue;  // moved by the pack kernel
        int64_t p0 = a.pair_off[pos] + skip, sh = 0;
        if (a.clip && !clip_run(p0, cnt, a.slo[r], a.shi[r], sh)) continue;
        s = a.recv + (a.displ[r] + p0) * R;
        t = a.out + (lo + sh) * R;
      }
#ifdef ORCH_BOUNDS_CHECK
      {
        const int64_t nb = cnt * static_cast<int64_t>(R);
        const int64_t Rr = static_cast<int64_t>(R);
        if (MODE == kUnpack)
          ORCH_DCHECK(within(s, nb, a.recv, recv_rows_of(a.send_rows, a.P, a.me) * Rr));
        else
          ORCH_DCHECK(within(s, nb, a.in, a.in_cap * Rr));
        if (MODE == kPut) {
          const char* pb = a.peer_out[a.dest[pos] / a.c] + a.win_off;
          ORCH_DCHECK(within(t, nb, pb, a.out_cap * Rr));
        } else if (MODE == kPack && a.dest[pos] / a.c != a.me) {
          ORCH_DCHECK(within(t, nb, a.send, a.send_cap * Rr));
        } else {
          ORCH_DCHECK(within(t, nb, a.out, a.out_cap * Rr));
        }
      }
#endif
      block_copy(reinterpret_cast<int4*>(t), reinterpret_cast<const int4*>(s), cnt * vrow);
    }
  }
  if (MODE == kPut) __threadfence_system();
}

// ------------------------------------------------------------ TMA movement
// Rows of >= 8 KiB move with bulk async copies (cp.async.bulk, SASS UBLKCP):
// global -> shared stage -> global, one warp per SM. The iteration buffer is
// cut into 32 KiB chunks claimed 32 at a time; each chunk is at most
// kTmaMaxPieces contiguous item pieces. The 32 lanes decode 32 chunks' pieces
// in parallel into a shared table, lane 0 streams them through a 4-stage ring:
// loads of three chunks in flight while the oldest chunk is stored (4 stages
// beat 3 by ~1% on one GPU; 6 stages and 48 KiB chunks gain nothing more).
#ifndef ORCH_TMA_STAGES
#define ORCH_TMA_STAGES 4
#endif
#ifndef ORCH_TMA_PUT_STAGES
#define ORCH_TMA_PUT_STAGES 3
#endif
#ifndef ORCH_TMA_CHUNK
#define ORCH_TMA_CHUNK 32768
#endif
// HBM moves use 4 stages; the NVLink put keeps 3 (it is at the push ceiling
// either way, and the smaller ring leaves shared memory for the next step's
// metadata kernels that run beside it: C3 / C5 on 4 GPUs lose ~2% with 4)
constexpr int kTmaStages = ORCH_TMA_STAGES;
constexpr int kTmaPutStages = ORCH_TMA_PUT_STAGES;
static_assert(kTmaPutStages <= kTmaStages, "TmaTable is sized by kTmaStages");
template <int MODE>
__host__ __device__ constexpr int tma_stages() { return MODE == kPut ? kTmaPutStages : kTmaStages; }
constexpr int kTmaChunk = ORCH_TMA_CHUNK;
constexpr int kTmaMaxPieces = 6;
constexpr int64_t kTmaMinRow = 8192;

struct TmaTable {
  const char* src[32][kTmaMaxPieces];
  char* dst[32][kTmaMaxPieces];
  uint32_t bytes[32][kTmaMaxPieces];
  int np[32];
  char* st_dst[kTmaStages][kTmaMaxPieces];
  uint32_t st_bytes[kTmaStages][kTmaMaxPieces];
  int st_np[kTmaStages];
  alignas(8) uint64_t bar[kTmaStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(32) k_move_tma(MoveArgs a) {
  constexpr int kS = tma_stages<MODE>();
  extern __shared__ __align__(128) unsigned char ring[];  // kS * kTmaChunk
  __shared__ TmaTable T;
  const int lane = threadIdx.x;
  const int64_t total = a.iter_rows[a.me];
  bool over = total > a.iter_cap || a.out_rows[a.me] > a.out_cap;
  if (MODE != kUnpack) over = over || a.in_rows[a.me] > a.in_cap;
  if (MODE == kPut)  // every rank's window has the same capacity
    for (int q = 0; q < a.P; ++q) over = over || a.out_rows[q] > a.out_cap;
  if (MODE == kPack && a.send) {
    int64_t st = 0;
    for (int q = 0; q < a.P; ++q)
      if (q != a.me) st += a.send_rows[a.me * a.P + q];
    over = over || st > a.send_cap;
  }
  if (over) {
    if (blockIdx.x == 0 && lane == 0) *a.status = ORCH_INVALID_ARGUMENT;
    return;
  }
  if (MODE == kPut && *a.acquired < a.need_free) {  // k_window_acquire timed out
    if (blockIdx.x == 0 && lane == 0) atomicExch(a.status, ORCH_CUDA_ERROR);
    return;
  }
  const int64_t R = static_cast<int64_t>(a.R);
  const int64_t total_b = total * R;
  const int64_t chunks = (total_b + kTmaChunk - 1) / kTmaChunk;
  // dynamic scheduling: CTAs claim 32 consecutive chunks at a time, so a CTA
  // sharing its SM with other work (the next step's balance) is no straggler
  unsigned long long* claim = a.chunk_counter;
  const int64_t beg = a.offs[a.lo_idx], end = a.offs[a.hi_idx];
  if (lane == 0) {
    for (int s = 0; s < kS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&T.bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phases = 0;  // lane 0: parity bit per stage
  int64_t fed = 0;      // lane 0: chunks issued so far (stage = fed % kS)

  auto retire = [&](int64_t r) {  // lane 0: wait chunk r's loads, store its pieces
    const int s = static_cast<int>(r % kS);
    const uint32_t ph = (phases >> s) & 1u;
    asm volatile(
        "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W%=;\n}" ::"r"(smem_u32(&T.bar[s])),
        "r"(ph));
    phases ^= 1u << s;
    uint32_t off = 0;
    for (int p = 0; p < T.st_np[s]; ++p) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(T.st_dst[s][p]),
                   "r"(smem_u32(ring + s * kTmaChunk + off)), "r"(T.st_bytes[s][p])
                   : "memory");
      off += T.st_bytes[s][p];
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };

  // kPut: batches of 32 chunks are claimed in a scrambled order (batch b ->
  // b * stride mod nb, stride coprime with nb, near nb / golden ratio), so the
  // CTAs in flight are spread over the whole input buffer and every peer
  // receives at a rate proportional to its share of the step. In input order,
  // long items (C5: 128-512 MB each) would send to one peer at a time while the
  // other ranks may pick the same peer: ingress collisions on that peer's links.
  const int64_t nb = (chunks + 31) / 32;
  int64_t stride = 1;
  if (MODE == kPut && a.scramble && nb > 2) {
    stride = static_cast<int64_t>(static_cast<double>(nb) * 0.6180339887) | 1;
    for (;; ++stride) {
      int64_t x = stride, y = nb;
      while (y) {
        const int64_t t = x % y;
        x = y;
        y = t;
      }
      if (x == 1) break;
    }
  }
  for (;;) {
    int64_t base = 0;
    if (lane == 0) base = static_cast<int64_t>(atomicAdd(claim, 32ull));
    base = __shfl_sync(~0u, base, 0);
    if (base >= chunks) break;
    if (stride != 1) base = ((base / 32) * stride % nb) * 32;
    // ---- decode: lane j -> this CTA's chunk (base + j)
    const int64_t c = base + lane;
    int np = 0;
    if (c < chunks) {
      const int64_t b0 = c * kTmaChunk;
      const int64_t b1 = b0 + kTmaChunk < total_b ? b0 + kTmaChunk : total_b;
      for (int64_t k = beg + a.unit_first[c]; k < end && np < kTmaMaxPieces; ++k) {
        const int32_t pos = a.members[k];
        const int64_t ob =
            ((MODE == kPack || MODE == kPut) ? a.rank_src_off[pos] : a.rank_dst_off[pos]) * R;
        if (ob >= b1) break;
        const int64_t ib = ob + a.len[pos] * R;
        const int64_t lo = ob > b0 ? ob : b0;
        const int64_t hi = ib < b1 ? ib : b1;
        const int64_t skip = lo - ob;
        const char* s = nullptr;
        char* d = nullptr;
        int64_t cnt = hi - lo;
        if (MODE == kLocal) {
          s = a.in + a.rank_src_off[pos] * R + skip;
          d = a.out + lo;
        } else if (MODE == kPack) {
          const int q = a.dest[pos] / a.c;
          if (q == a.me) {
            if (!a.skip_local) {
              s = a.in + lo;
              d = a.out + a.rank_dst_off[pos] * R + skip;
            }
          } else if (a.send) {  // no send buffer: local rows only (orch_dispatch_nccl, direct)
            int64_t p0 = a.pair_off[pos] * R + skip, sh = 0;
            if (!a.clip || clip_run(p0, cnt, a.slo[q] * R, a.shi[q] * R, sh)) {
              s = a.in + lo + sh;
              d = a.send + a.displ[q] * R + p0;
            }
          }
        } else if (MODE == kPut) {
          s = a.in + lo;
          d = a.peer_out[a.dest[pos] / a.c] + a.win_off + a.rank_dst_off[pos] * R + skip;
        } else {
          const int r = a.origin[pos] / a.c;
          if (r != a.me) {
            int64_t p0 = a.pair_off[pos] * R + skip, sh = 0;
            if (!a.clip || clip_run(p0, cnt, a.slo[r] * R, a.shi[r] * R, sh)) {
              s = a.recv + a.displ[r] * R + p0;
              d = a.out + lo + sh;
            }
          }
        }
        if (s) {
#ifdef ORCH_BOUNDS_CHECK
          if (MODE == kUnpack)
            ORCH_DCHECK(within(s, cnt, a.recv, recv_rows_of(a.send_rows, a.P, a.me) * R));
          else
            ORCH_DCHECK(within(s, cnt, a.in, a.in_cap * R));
          if (MODE == kPut)
            ORCH_DCHECK(within(d, cnt, a.peer_out[a.dest[pos] / a.c] + a.win_off, a.out_cap * R));
          else if (MODE == kPack && a.dest[pos] / a.c != a.me)
            ORCH_DCHECK(within(d, cnt, a.send, a.send_cap * R));
          else
            ORCH_DCHECK(within(d, cnt, a.out, a.out_cap * R));
          ORCH_DCHECK(cnt > 0 && cnt % 16 == 0);
#endif
          T.src[lane][np] = s;
          T.dst[lane][np] = d;
          T.bytes[lane][np] = static_cast<uint32_t>(cnt);
          ++np;
        }
        if (ib >= b1) break;
      }
    }
    T.np[lane] = np;
    __syncwarp();
    // ---- feed (lane 0)
    if (lane == 0) {
      const int cnt = chunks - base < 32 ? static_cast<int>(chunks - base) : 32;
      for (int j = 0; j < cnt; ++j) {
        const int pn = T.np[j];
        if (pn == 0) continue;  // nothing to move in this chunk
        if (fed >= kS - 1) retire(fed - (kS - 1));
        if (fed >= kS)  // stage of chunk fed-3 is free once its store has read smem
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        const int s = static_cast<int>(fed % kS);
        uint32_t tot = 0;
        for (int p = 0; p < pn; ++p) tot += T.bytes[j][p];
        const uint32_t bar = smem_u32(&T.bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tot)
                     : "memory");
        uint32_t off = 0;
        for (int p = 0; p < pn; ++p) {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(smem_u32(ring + s * kTmaChunk + off)), "l"(T.src[j][p]), "r"(T.bytes[j][p]),
              "r"(bar)
              : "memory");
          T.st_dst[s][p] = T.dst[j][p];
          T.st_bytes[s][p] = T.bytes[j][p];
          off += T.bytes[j][p];
        }
        T.st_np[s] = pn;
        ++fed;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    for (int64_t r = fed - (kS - 1) > 0 ? fed - (kS - 1) : 0; r < fed; ++r)
      retire(r);
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (MODE == kPut) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence_system();
    }
  }
}

// ----------------------------------------------------- all-gather scatter
__global__ void k_pack_records(int64_t local_n, int64_t max_local, const int64_t* __restrict__ pos,
                               const int64_t* __restrict__ len, const int32_t* __restrict__ org,
                               int64_t* __restrict__ rec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < max_local;
       i += (int64_t)gridDim.x * blockDim.x) {
    rec[3 * i] = i < local_n ? pos[i] : -1;
    rec[3 * i + 1] = i < local_n ? len[i] : 0;
    rec[3 * i + 2] = i < local_n ? org[i] : 0;
  }
}

__global__ void k_scatter_records(int64_t total, int64_t n, const int64_t* __restrict__ rec,
                                  int64_t* __restrict__ len, int32_t* __restrict__ org,
                                  unsigned int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = rec[3 * i];
    if (p < 0) continue;
    if (p >= n) {
      atomicOr(bad, 1u);
      continue;
    }
    len[p] = rec[3 * i + 1];
    org[p] = static_cast<int32_t>(rec[3 * i + 2]);
  }
}

// ------------------------------------------- gather_lengths over NVLink
// One-shot all-gather of the (length, origin) records through peer memory
// (gather_lengths, exchange.cpp:34-47). Gather window layout per rank:
//   len[max_n] i64 | origin[max_n] i32 | arrived[P] u64 | consumed[P] u64
// arrived[q] = the last call whose records rank q has fully stored here;
// consumed[q] = the last call whose records rank q has copied out of ITS
// window (so this rank may overwrite them). Calls are numbered 1, 2, ... in
// the same order on every rank.
struct GatherArgs {
  char* const* peers;  // [P] gather windows
  int me, P;
  uint64_t epoch;
  int64_t max_n, n, local_n;
  const int64_t* pos;
  const int64_t* len;
  const int32_t* org;
  int64_t* out_len;
  int32_t* out_org;
  int32_t* status;  // optional: ORCH_INVALID_ARGUMENT on a bad position, ORCH_CUDA_ERROR on timeout
  uint64_t* stamps;  // [8][8] %globaltimer at the kernel's stages, slot epoch % 8 (diagnostics)
};

__host__ __device__ inline size_t gather_flags_off(int64_t max_n) {
  return (static_cast<size_t>(max_n) * 12 + 15) & ~size_t{15};
}

__global__ void __launch_bounds__(1024) k_gather_put(GatherArgs a) {
  __shared__ int bad;
  const int t = threadIdx.x;
  const size_t fo = gather_flags_off(a.max_n);
  auto len_of = [&](int q) { return reinterpret_cast<int64_t*>(a.peers[q]); };
  auto org_of = [&](int q) { return reinterpret_cast<int32_t*>(a.peers[q] + 8 * a.max_n); };
  auto arrived = [&](int q) { return reinterpret_cast<uint64_t*>(a.peers[q] + fo); };
  auto consumed = [&](int q) { return reinterpret_cast<uint64_t*>(a.peers[q] + fo) + a.P; };
  uint64_t* stamp = a.stamps + (a.epoch % 8) * 8;
  if (t == 0) {
    bad = 0;
    stamp[0] = gtimer();
  }
  // 1. every peer has copied out our previous call's records
  if (t < a.P && !wait_at_least(consumed(a.me) + t, a.epoch - 1)) bad = 2;
  __syncthreads();
  if (t == 0) stamp[1] = gtimer();
  // 2. our records, at their global input positions, into every window
  for (int64_t i = t; i < a.local_n && !bad; i += blockDim.x) {
    const int64_t p = a.pos[i];
    if (p < 0 || p >= a.n) {
      bad = 1;
      break;
    }
    const int64_t l = a.len[i];
    const int32_t o = a.org[i];
    ORCH_DCHECK(p < a.max_n);
    for (int q = 0; q < a.P; ++q) {
      len_of(q)[p] = l;
      org_of(q)[p] = o;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (t == 0) stamp[2] = gtimer();
  if (t < a.P) st_release_sys(arrived(t) + a.me, a.epoch);  // this rank's records are in
  // 3. every rank's records are here
  if (t < a.P && !wait_at_least(arrived(a.me) + t, a.epoch)) bad = 2;
  __syncthreads();
  if (t == 0) stamp[3] = gtimer();
  const int64_t* wl = len_of(a.me);
  const int32_t* wo = org_of(a.me);
  for (int64_t i = t; i < a.n; i += blockDim.x) {  // L2 (the coherence point of peer stores)
    a.out_len[i] = __ldcg(wl + i);
    a.out_org[i] = __ldcg(wo + i);
  }
  __syncthreads();
  // 4. the window may be overwritten by the next call
  if (t < a.P) st_release_sys(consumed(t) + a.me, a.epoch);
  if (t == 0 && bad && a.status) *a.status = bad == 1 ? ORCH_INVALID_ARGUMENT : ORCH_CUDA_ERROR;
  if (t == 0) stamp[4] = gtimer();
}

// ------------------------------------------------------- encode_lengths
__global__ void k_encode(int64_t E, const int32_t* __restrict__ part_offset,
                         const int32_t* __restrict__ modality, const int64_t* __restrict__ meta,
                         int32_t M, const int64_t* __restrict__ rates,
                         int64_t* __restrict__ encoded, int64_t* __restrict__ inter) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t sum = 0;
    for (int p = part_offset[e]; p < part_offset[e + 1]; ++p) {
      const int32_t m = modality[p];
      const int64_t rate = (m >= 0 && m < M) ? rates[m] : 1;  // unknown modality: rate 1
      const int64_t enc = (meta[p] + rate - 1) / rate;         // core.cpp:176-179
      if (encoded) encoded[p] = enc;
      sum += enc;
    }
    if (inter) inter[e] = sum;  // interleaved_length, core.cpp:163-169
  }
}

}  // namespace

}  // namespace orchb

using namespace orchb;

extern "C" {

int orch_volume_matrix(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* d_len,
                       const int32_t* d_origin, const int32_t* d_dest_inst, int64_t* d_V,
                       void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  auto st = static_cast<cudaStream_t>(stream);
  ORCH_CUDA_TRY(cudaMemsetAsync(d_V, 0, sizeof(int64_t) * static_cast<size_t>(d) * d, st));
  if (n > 0)
    launch(ctx, [&] {
      k_volume<<<blocks_for(n, kThreads), kThreads, 0, st>>>(
          d, n, d_len, d_origin, d_dest_inst, reinterpret_cast<unsigned long long*>(d_V));
    });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_layout(orch_ctx* ctx, int32_t d, int32_t P, int64_t n, const int64_t* d_len,
                const int32_t* d_origin, const orch_balance_out* bal,
                const orch_layout_out* L, void* stream) {
  if (!ctx || !bal || !L) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (P < 1 || P > 8 || d % P != 0)
    return fail(ORCH_INVALID_ARGUMENT, "rank count must be in [1, 8] and divide the instance count");
  if (!bal->dest_inst || !bal->src_off || !bal->dst_off || !bal->bin_offset || !bal->bin_member)
    return fail(ORCH_INVALID_ARGUMENT, "orch_layout needs dest_inst, src_off, dst_off, bin_offset, bin_member");
  auto st = static_cast<cudaStream_t>(stream);
  if (!L->status) return fail(ORCH_INVALID_ARGUMENT, "layout->status is required");
  if (n <= kLayoutSmallItems && d <= kLayoutSmallD) {
    static PerDeviceOnce configured;
    const int rc_attr = configured([&]() -> int {
      ORCH_CUDA_TRY(max_carveout(k_layout_small));
      return ORCH_OK;
    });
    if (rc_attr) return rc_attr;
    launch(ctx, [&] {
      k_layout_small<<<1, kLayoutSmallThreads, 0, st>>>(static_cast<int>(n), d, P, d_len, d_origin,
                                                        *bal, *L);
    });
    ORCH_CUDA_TRY(cudaGetLastError());
    return ORCH_OK;
  }
  Plan plan;
  unsigned long long *inst_in, *inst_out;
  int64_t *base_in, *base_out, *W, *Wbase;
  plan.add(&inst_in, d);
  plan.add(&inst_out, d);
  plan.add(&base_in, d);
  plan.add(&base_out, d);
  plan.add(&W, static_cast<size_t>(d) * P);
  plan.add(&Wbase, static_cast<size_t>(d) * P);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  if (!L->status) return fail(ORCH_INVALID_ARGUMENT, "layout->status is required");
  ORCH_CUDA_TRY(cudaMemsetAsync(L->status, 0, sizeof(int32_t), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(inst_in, 0, sizeof(uint64_t) * d, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(inst_out, 0, sizeof(uint64_t) * d, st));
  const int gb = blocks_for(n, kThreads);
  if (n > 0)
    launch(ctx, [&] {
      k_inst_rows<<<gb, kThreads, 0, st>>>(n, d_len, d_origin, bal->dest_inst, inst_in, inst_out);
    });
  launch(ctx, [&] {
    k_inst_bases<<<1, 32, 0, st>>>(d, P, inst_in, inst_out, base_in, base_out, L->in_rows,
                                   L->out_rows);
  });
  if (n > 0)
    launch(ctx, [&] {
      k_rank_offsets<<<gb, kThreads, 0, st>>>(n, d_origin, bal->dest_inst, bal->src_off,
                                              bal->dst_off, base_in, base_out, L->rank_src_off,
                                              L->rank_dst_off);
    });
  launch(ctx, [&] {
    k_pair_within<<<blocks_for(static_cast<int64_t>(d) * 32, kThreads), kThreads, 0, st>>>(
        d, P, bal->bin_offset, bal->bin_member, d_len, d_origin, L->pair_off, W);
  });
  launch(ctx, [&] {
    k_pair_bases<<<1, 64, 0, st>>>(d, P, W, Wbase, L->send_rows, L->send_displ, L->recv_displ);
  });
  if (n > 0)
    launch(ctx, [&] {
      k_pair_apply<<<gb, kThreads, 0, st>>>(n, d, P, d_origin, bal->dest_inst, Wbase, L->pair_off);
    });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"

namespace {

int check_move_args(orch_ctx* ctx, int P, int me, int d, const orch_balance_out* bal,
                    const orch_layout_out* L, size_t R) {
  if (!ctx || !bal || !L) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (R == 0 || R % 16 != 0)
    return fail(ORCH_INVALID_ARGUMENT, "row_bytes must be a positive multiple of 16");
  if (P < 1 || P > 8 || me < 0 || me >= P || d % P != 0)
    return fail(ORCH_INVALID_ARGUMENT, "bad rank / rank count (must divide the instance count, <= 8)");
  if (!bal->src_offset || !bal->src_member || !bal->bin_offset || !bal->bin_member ||
      !bal->dest_inst || !L->status)
    return fail(ORCH_INVALID_ARGUMENT, "movement needs the CSR outputs of orch_balance and layout->status");
  return ORCH_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

MoveArgs make_args(int P, int me, int d, const int64_t* len, const int32_t* origin,
                   const orch_balance_out* bal, const orch_layout_out* L, size_t R) {
  MoveArgs a{};
  a.me = me;
  a.P = P;
  a.c = d / P;
  a.lo_idx = me * a.c;
  a.hi_idx = (me + 1) * a.c;
  a.out_rows = L->out_rows;
  a.in_rows = L->in_rows;
  a.send_rows = L->send_rows;
  a.len = len;
  a.origin = origin;
  a.dest = bal->dest_inst;
  a.rank_src_off = L->rank_src_off;
  a.rank_dst_off = L->rank_dst_off;
  a.pair_off = L->pair_off;
  a.status = L->status;
  a.R = R;
  return a;
}

constexpr int kMoveGrid = kSMs * 8;

// grid_cap > 0: at most that many CTAs (leaves SMs to a concurrent NCCL kernel)
int run_move(orch_ctx* ctx, int mode, MoveArgs a, int64_t n, const int64_t* iter_off,
             cudaStream_t st, int grid_cap = 0) {
  const bool tma = static_cast<int64_t>(a.R) >= kTmaMinRow;
  const int64_t unit_bytes = tma ? kTmaChunk : kUnitRows * static_cast<int64_t>(a.R);
  const int64_t cap_units = (a.iter_cap * static_cast<int64_t>(a.R)) / unit_bytes + 2;
  Plan plan;
  int32_t* unit_first;
  unsigned long long* counter;
  plan.add(&unit_first, static_cast<size_t>(cap_units));
  plan.add(&counter, 1);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  a.unit_first = unit_first;
  a.chunk_counter = counter;
  launch(ctx, [&] {
    k_unit_map<<<blocks_for(cap_units, kThreads, kSMs * 4), kThreads, 0, st>>>(
        a.offs, a.lo_idx, a.hi_idx, a.members, iter_off, a.iter_rows, a.me, unit_bytes,
        static_cast<int64_t>(a.R), unit_first, cap_units, counter);
  });
  if (tma) {
    const int sm = kTmaStages * kTmaChunk;
    static const int ctas_per_sm = [] {
      const char* e = getenv("ORCH_TMA_CTAS_PER_SM");
      const int v = e ? atoi(e) : 1;
      return v >= 1 && v <= 2 ? v : 1;
    }();
    // experiment knobs: ORCH_PUT_FREE_SMS=k leaves k SMs to other streams and
    // makes each put CTA claim a whole SM's shared memory (no co-residence)
    static const int free_sms = [] {
      const char* e = getenv("ORCH_PUT_FREE_SMS");
      const int v = e ? atoi(e) : 0;
      return v >= 0 && v < kSMs ? v : 0;
    }();
    const bool fat = mode == kPut && free_sms > 0;
    int tma_grid = fat ? kSMs - free_sms : kSMs * ctas_per_sm;
    if (grid_cap > 0 && tma_grid > grid_cap) tma_grid = grid_cap;
    const int sm_put = kTmaPutStages * kTmaChunk;
    const int sm_req = fat ? 227 * 1024 - static_cast<int>(sizeof(TmaTable)) - 64 : sm_put;
    static PerDeviceOnce attr_done;
    const int rc_attr = attr_done([&]() -> int {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_move_tma<kLocal>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_move_tma<kPack>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_move_tma<kUnpack>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_move_tma<kPut>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sm_req));
      ORCH_CUDA_TRY(max_carveout(k_move_tma<kLocal>));
      ORCH_CUDA_TRY(max_carveout(k_move_tma<kPack>));
      ORCH_CUDA_TRY(max_carveout(k_move_tma<kUnpack>));
      ORCH_CUDA_TRY(max_carveout(k_move_tma<kPut>));
      return ORCH_OK;
    });
    if (rc_attr) return rc_attr;
    launch(ctx, [&] {
      if (mode == kLocal)
        k_move_tma<kLocal><<<tma_grid, 32, sm, st>>>(a);
      else if (mode == kPack)
        k_move_tma<kPack><<<tma_grid, 32, sm, st>>>(a);
      else if (mode == kPut)
        k_move_tma<kPut><<<tma_grid, 32, sm_req, st>>>(a);
      else
        k_move_tma<kUnpack><<<tma_grid, 32, sm, st>>>(a);
    });
  } else {
    launch(ctx, [&] {
      if (mode == kLocal)
        k_move<kLocal><<<grid_cap > 0 ? grid_cap * 8 : kMoveGrid, kMoveThreads, 0, st>>>(a);
      else if (mode == kPack)
        k_move<kPack><<<grid_cap > 0 ? grid_cap * 8 : kMoveGrid, kMoveThreads, 0, st>>>(a);
      else if (mode == kPut)
        k_move<kPut><<<grid_cap > 0 ? grid_cap * 8 : kMoveGrid, kMoveThreads, 0, st>>>(a);
      else
        k_move<kUnpack><<<grid_cap > 0 ? grid_cap * 8 : kMoveGrid, kMoveThreads, 0, st>>>(a);
    });
  }
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // namespace

extern "C" {

int orch_pack(orch_ctx* ctx, int32_t rank, int32_t nranks, int32_t d, int64_t n,
              const int64_t* d_len, const int32_t* d_origin, const orch_balance_out* bal,
              const orch_layout_out* L, size_t R, const void* d_in, int64_t in_cap, void* d_out,
              int64_t out_cap, void* d_send, int64_t send_cap, void* stream) {
  int rc = check_move_args(ctx, nranks, rank, d, bal, L, R);
  if (rc) return rc;
  if (!aligned16(d_in) || !aligned16(d_out) || !aligned16(d_send))
    return fail(ORCH_INVALID_ARGUMENT, "row buffers must be 16-byte aligned");
  if (n == 0) return ORCH_OK;
  MoveArgs a = make_args(nranks, rank, d, d_len, d_origin, bal, L, R);
  a.offs = bal->src_offset;
  a.members = bal->src_member;
  a.iter_rows = L->in_rows;
  a.iter_cap = in_cap;
  a.in_cap = in_cap;
  a.out_cap = out_cap;
  a.send_cap = send_cap;
  a.displ = L->send_displ + rank * nranks;
  a.in = static_cast<const char*>(d_in);
  a.out = static_cast<char*>(d_out);
  a.send = static_cast<char*>(d_send);
  return run_move(ctx, kPack, a, n, L->rank_src_off, static_cast<cudaStream_t>(stream));
}

int orch_unpack(orch_ctx* ctx, int32_t rank, int32_t nranks, int32_t d, int64_t n,
                const int64_t* d_len, const int32_t* d_origin, const orch_balance_out* bal,
                const orch_layout_out* L, size_t R, const void* d_recv, void* d_out,
                int64_t out_cap, void* stream) {
  int rc = check_move_args(ctx, nranks, rank, d, bal, L, R);
  if (rc) return rc;
  if (!aligned16(d_recv) || !aligned16(d_out))
    return fail(ORCH_INVALID_ARGUMENT, "row buffers must be 16-byte aligned");
  if (n == 0) return ORCH_OK;
  MoveArgs a = make_args(nranks, rank, d, d_len, d_origin, bal, L, R);
  a.offs = bal->bin_offset;
  a.members = bal->bin_member;
  a.iter_rows = L->out_rows;
  a.iter_cap = out_cap;
  a.out_cap = out_cap;
  a.displ = L->recv_displ + rank * nranks;
  a.recv = static_cast<const char*>(d_recv);
  a.out = static_cast<char*>(d_out);
  return run_move(ctx, kUnpack, a, n, L->rank_dst_off, static_cast<cudaStream_t>(stream));
}

int orch_exchange(orch_ctx* ctx, orch_comm* comm, const orch_layout_out* L, size_t R,
                  const void* d_send, void* d_recv, int64_t recv_cap, void* stream) {
  if (!ctx || !comm || !L) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (!comm->comm) return fail(ORCH_INVALID_ARGUMENT, "loopback communicator has no NCCL");
  const int P = comm->size, me = comm->rank;
  auto st = static_cast<cudaStream_t>(stream);
  int64_t* h = static_cast<int64_t*>(pinned(ctx, sizeof(int64_t) * 3 * P * P));
  if (!h) return fail(ORCH_CUDA_ERROR, "pinned staging allocation failed");
  int64_t *h_send = h, *h_sdis = h + P * P, *h_rdis = h + 2 * P * P;
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_send, L->send_rows, sizeof(int64_t) * P * P,
                                cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_sdis, L->send_displ, sizeof(int64_t) * P * P,
                                cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_rdis, L->recv_displ, sizeof(int64_t) * P * P,
                                cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));  // NCCL takes host-side counts
  int64_t recv_total = 0;
  for (int r = 0; r < P; ++r)
    if (r != me) recv_total += h_send[r * P + me];
  if (recv_total > recv_cap)
    return fail(ORCH_INVALID_ARGUMENT, "receive buffer smaller than the incoming rows");
  const char* send = static_cast<const char*>(d_send);
  char* recv = static_cast<char*>(d_recv);
  ORCH_NCCL_TRY(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const int64_t s_rows = h_send[me * P + q];
    const int64_t r_rows = h_send[q * P + me];
    if (s_rows > 0)
      ORCH_NCCL_TRY(ncclSend(send + h_sdis[me * P + q] * R, static_cast<size_t>(s_rows) * R,
                             ncclInt8, q, comm->comm, st));
    if (r_rows > 0)
      ORCH_NCCL_TRY(ncclRecv(recv + h_rdis[me * P + q] * R, static_cast<size_t>(r_rows) * R,
                             ncclInt8, q, comm->comm, st));
  }
  ORCH_NCCL_TRY(ncclGroupEnd());
  return ORCH_OK;
}

int orch_dispatch(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                  const int32_t* d_origin, const orch_balance_out* bal,
                  const orch_layout_out* L, size_t R, const void* d_in, int64_t in_cap,
                  void* d_out, int64_t out_cap, void* d_send, int64_t send_cap, void* d_recv,
                  int64_t recv_cap, void* stream) {
  const int P = comm ? comm->size : 1;
  const int me = comm ? comm->rank : 0;
  int rc = check_move_args(ctx, P, me, d, bal, L, R);
  if (rc) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  if (P == 1) {
    if (!aligned16(d_in) || !aligned16(d_out))
      return fail(ORCH_INVALID_ARGUMENT, "row buffers must be 16-byte aligned");
    if (n == 0) return ORCH_OK;
    MoveArgs a = make_args(1, 0, d, d_len, d_origin, bal, L, R);
    a.offs = bal->bin_offset;
    a.members = bal->bin_member;
    a.iter_rows = L->out_rows;
    a.iter_cap = out_cap;
    a.out_cap = out_cap;
    a.in_cap = in_cap;
    a.in = static_cast<const char*>(d_in);
    a.out = static_cast<char*>(d_out);
    return run_move(ctx, kLocal, a, n, L->rank_dst_off, st);
  }
  rc = orch_pack(ctx, me, P, d, n, d_len, d_origin, bal, L, R, d_in, in_cap, d_out, out_cap,
                 d_send, send_cap, stream);
  if (rc) return rc;
  rc = orch_exchange(ctx, comm, L, R, d_send, d_recv, recv_cap, stream);
  if (rc) return rc;
  return orch_unpack(ctx, me, P, d, n, d_len, d_origin, bal, L, R, d_recv, d_out, out_cap,
                     stream);
}

// -------------------------------------------- NCCL exchange, per item run
}  // extern "C"

struct orch_xplan {
  int64_t max_n = 0;
  int P = 1;
  char* pinned = nullptr;  // h_len | h_rso | h_rdo | in/out rows | send rows, displs | h_org | h_dst
  int64_t *h_len = nullptr, *h_rso = nullptr, *h_rdo = nullptr, *h_in = nullptr, *h_out = nullptr;
  int64_t *h_send = nullptr, *h_sdis = nullptr, *h_rdis = nullptr;  // [P*P] each
  int32_t *h_org = nullptr, *h_dst = nullptr;
  cudaEvent_t ready = nullptr;
  // the device-side view of the same layout (for the local-rows kernel)
  int d = 0;
  int64_t n = 0;
  const int64_t* d_len = nullptr;
  const int32_t* d_origin = nullptr;
  orch_balance_out bal{};
  orch_layout_out lay{};
  bool fetched = false;
  std::vector<int64_t> order;  // host scratch: per-peer item lists
  // sliced staged exchange: pack (caller's stream) -> NCCL (s_comm) -> unpack (s_unpack)
  static constexpr int kMaxSlices = 16;
  int dev = -1;
  cudaStream_t s_comm = nullptr, s_unpack = nullptr;
  cudaEvent_t ev_entry = nullptr, ev_done = nullptr;
  cudaEvent_t ev_pack[kMaxSlices] = {}, ev_comm[kMaxSlices] = {};
};

extern "C" {

int orch_xplan_create(orch_ctx* ctx, int64_t max_n, int32_t P, orch_xplan** out) {
  if (!ctx || !out || max_n < 0 || P < 1 || P > 8) return fail(ORCH_INVALID_ARGUMENT, "bad plan arguments");
  auto* x = new orch_xplan();
  x->max_n = max_n;
  x->P = P;
  const size_t nn = static_cast<size_t>(max_n > 0 ? max_n : 1);
  const size_t bytes = nn * (8 * 3 + 4 * 2) + 16 * static_cast<size_t>(P) + 24 * P * P;
  if (cudaMallocHost(&x->pinned, bytes) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->ready, cudaEventDisableTiming) != cudaSuccess) {
    if (x->pinned) cudaFreeHost(x->pinned);
    delete x;
    return fail(ORCH_CUDA_ERROR, "exchange plan allocation failed");
  }
  char* p = x->pinned;
  x->h_len = reinterpret_cast<int64_t*>(p);
  x->h_rso = x->h_len + nn;
  x->h_rdo = x->h_rso + nn;
  x->h_in = x->h_rdo + nn;
  x->h_out = x->h_in + P;
  x->h_send = x->h_out + P;
  x->h_sdis = x->h_send + P * P;
  x->h_rdis = x->h_sdis + P * P;
  x->h_org = reinterpret_cast<int32_t*>(x->h_rdis + P * P);
  x->h_dst = x->h_org + nn;
  x->order.reserve(nn);
  *out = x;
  return ORCH_OK;
}

void orch_xplan_destroy(orch_xplan* x) {
  if (!x) return;
  if (x->ready) cudaEventDestroy(x->ready);
  if (x->s_comm) {
    cudaStreamSynchronize(x->s_comm);
    cudaStreamSynchronize(x->s_unpack);
    cudaStreamDestroy(x->s_comm);
    cudaStreamDestroy(x->s_unpack);
    cudaEventDestroy(x->ev_entry);
    cudaEventDestroy(x->ev_done);
    for (int k = 0; k < orch_xplan::kMaxSlices; ++k) {
      cudaEventDestroy(x->ev_pack[k]);
      cudaEventDestroy(x->ev_comm[k]);
    }
  }

  if (x->pinned) cudaFreeHost(x->pinned);
  delete x;
}

int orch_xplan_fetch(orch_ctx* ctx, orch_xplan* x, int32_t d, int64_t n, const int64_t* d_len,
                     const int32_t* d_origin, const orch_balance_out* bal,
                     const orch_layout_out* L, void* stream) {
  if (!ctx || !x || !bal || !L) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (n < 0 || n > x->max_n) return fail(ORCH_INVALID_ARGUMENT, "plan holds fewer items than n");
  if (d % x->P != 0) return fail(ORCH_INVALID_ARGUMENT, "rank count must divide the instance count");
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n);
  if (nn) {
    ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_len, d_len, nn * 8, cudaMemcpyDeviceToHost, st));
    ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_org, d_origin, nn * 4, cudaMemcpyDeviceToHost, st));
    ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_dst, bal->dest_inst, nn * 4, cudaMemcpyDeviceToHost, st));
    ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_rso, L->rank_src_off, nn * 8, cudaMemcpyDeviceToHost, st));
    ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_rdo, L->rank_dst_off, nn * 8, cudaMemcpyDeviceToHost, st));
  }
  ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_in, L->in_rows, 8 * x->P, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_out, L->out_rows, 8 * x->P, cudaMemcpyDeviceToHost, st));
  const size_t pp = 8 * static_cast<size_t>(x->P) * x->P;
  ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_send, L->send_rows, pp, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_sdis, L->send_displ, pp, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(x->h_rdis, L->recv_displ, pp, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaEventRecord(x->ready, st));
  x->d = d;
  x->n = n;
  x->d_len = d_len;
  x->d_origin = d_origin;
  x->bal = *bal;
  x->lay = *L;
  x->fetched = true;
  return ORCH_OK;
}

}  // extern "C"

namespace {

// The staged exchange in K slices (K = 1 by default), over three streams: slice
// k of every (this rank -> peer) segment is packed on the caller's stream, sent
// by one NCCL group on s_comm while slice k+1 is packed, and the slices
// received are unpacked on s_unpack while the next ones travel. The rows that
// stay on the rank move last on the caller's stream, beside the transfer (HBM
// only, no NVLink). Segment slicing is a function of the segment size only, so
// sender and receiver agree without communicating.
int staged_rounds(orch_ctx* ctx, orch_comm* comm, orch_xplan* x, size_t R, const void* d_in,
                  int64_t in_cap, void* d_out, int64_t out_cap, void* d_send, int64_t send_cap,
                  void* d_recv, int64_t recv_cap, cudaStream_t st) {
  const int P = comm->size, me = comm->rank;
  static const int env_slices = [] {
    // 1 by default: on 2 B200s, overlapping the pack / unpack kernels with
    // NCCL's made the exchange slower (C2: 351 -> 250 GB/s at 4 slices;
    // profiles/r02_nccl.md), so the slicing stays an option
    const char* e = getenv("ORCH_NCCL_SLICES");
    const int v = e ? atoi(e) : 1;
    return v >= 1 && v <= orch_xplan::kMaxSlices ? v : 1;
  }();
  // Slices of at least ~8 MB (ORCH_NCCL_MIN_SLICE_BYTES): fewer for small
  // exchanges. Every rank must cut the same slices, so K comes from a quantity
  // all ranks agree on: the largest off-rank segment of the replicated layout.
  static const int64_t min_slice_bytes = [] {
    const char* e = getenv("ORCH_NCCL_MIN_SLICE_BYTES");
    const long long v = e ? atoll(e) : (8ll << 20);
    return static_cast<int64_t>(v > 0 ? v : (8ll << 20));
  }();
  const int64_t min_slice_rows = (min_slice_bytes + static_cast<int64_t>(R) - 1) / static_cast<int64_t>(R);
  int64_t glob = 0;
  for (int k = 0; k < P * P; ++k)
    if (k / P != k % P) glob = std::max(glob, x->h_send[k]);
  const int Kg = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(env_slices, (glob + min_slice_rows - 1) / min_slice_rows)));
  int dev = 0;
  ORCH_CUDA_TRY(cudaGetDevice(&dev));
  if (!x->s_comm || x->dev != dev) {
    int lo = 0, hi = 0;
    ORCH_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ORCH_CUDA_TRY(cudaStreamCreateWithPriority(&x->s_comm, cudaStreamNonBlocking, hi));
    ORCH_CUDA_TRY(cudaStreamCreateWithFlags(&x->s_unpack, cudaStreamNonBlocking));
    ORCH_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_entry, cudaEventDisableTiming));
    ORCH_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_done, cudaEventDisableTiming));
    for (int k = 0; k < orch_xplan::kMaxSlices; ++k) {
      ORCH_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_pack[k], cudaEventDisableTiming));
      ORCH_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_comm[k], cudaEventDisableTiming));
    }
    x->dev = dev;
  }
  ORCH_CUDA_TRY(cudaEventRecord(x->ev_entry, st));
  ORCH_CUDA_TRY(cudaStreamWaitEvent(x->s_comm, x->ev_entry, 0));
  ORCH_CUDA_TRY(cudaStreamWaitEvent(x->s_unpack, x->ev_entry, 0));
  auto slice = [&](int64_t rows, int k) { return rows * k / Kg; };
  // sliced: the pack / unpack kernels leave SMs to NCCL's kernel running beside them
  static const int mover_sms = [] {
    const char* e = getenv("ORCH_NCCL_MOVER_SMS");
    const int v = e ? atoi(e) : 96;
    return v >= 8 && v <= kSMs ? v : 96;
  }();
  const int cap = Kg > 1 ? mover_sms : 0;
  const char* send = static_cast<const char*>(d_send);
  char* recv = static_cast<char*>(d_recv);
  for (int k = 0; k < Kg; ++k) {
    int rc;
    if (x->n > 0) {  // pack slice k of every off-rank segment
      MoveArgs a = make_args(P, me, x->d, x->d_len, x->d_origin, &x->bal, &x->lay, R);
      a.offs = x->bal.src_offset;
      a.members = x->bal.src_member;
      a.iter_rows = x->lay.in_rows;
      a.iter_cap = in_cap;
      a.in_cap = in_cap;
      a.out_cap = out_cap;
      a.send_cap = send_cap;
      a.displ = x->lay.send_displ + me * P;
      a.in = static_cast<const char*>(d_in);
      a.out = static_cast<char*>(d_out);
      a.send = static_cast<char*>(d_send);
      a.clip = 1;
      a.skip_local = 1;  // the rows that stay move below, beside the transfer
      for (int q = 0; q < P; ++q) {
        const int64_t S = q == me ? 0 : x->h_send[me * P + q];
        a.slo[q] = slice(S, k);
        a.shi[q] = slice(S, k + 1);
      }
      rc = run_move(ctx, kPack, a, x->n, x->lay.rank_src_off, st, cap);
      if (rc) return rc;
    }
    ORCH_CUDA_TRY(cudaEventRecord(x->ev_pack[k], st));
    ORCH_CUDA_TRY(cudaStreamWaitEvent(x->s_comm, x->ev_pack[k], 0));
    ORCH_NCCL_TRY(ncclGroupStart());
    for (int j = 1; j < P; ++j) {
      const int q = (me + j) % P, r = (me + P - j) % P;
      const int64_t S = x->h_send[me * P + q], Sr = x->h_send[r * P + me];
      const int64_t s0 = slice(S, k), s1 = slice(S, k + 1);
      const int64_t r0 = slice(Sr, k), r1 = slice(Sr, k + 1);
      if (s1 > s0)
        ORCH_NCCL_TRY(ncclSend(send + (x->h_sdis[me * P + q] + s0) * R,
                               static_cast<size_t>(s1 - s0) * R, ncclInt8, q, comm->comm,
                               x->s_comm));
      if (r1 > r0)
        ORCH_NCCL_TRY(ncclRecv(recv + (x->h_rdis[me * P + r] + r0) * R,
                               static_cast<size_t>(r1 - r0) * R, ncclInt8, r, comm->comm,
                               x->s_comm));
    }
    ORCH_NCCL_TRY(ncclGroupEnd());
    ORCH_CUDA_TRY(cudaEventRecord(x->ev_comm[k], x->s_comm));
    ORCH_CUDA_TRY(cudaStreamWaitEvent(x->s_unpack, x->ev_comm[k], 0));
    if (x->n > 0) {  // unpack the slices that arrived
      MoveArgs a = make_args(P, me, x->d, x->d_len, x->d_origin, &x->bal, &x->lay, R);
      a.offs = x->bal.bin_offset;
      a.members = x->bal.bin_member;
      a.iter_rows = x->lay.out_rows;
      a.iter_cap = out_cap;
      a.out_cap = out_cap;
      a.displ = x->lay.recv_displ + me * P;
      a.recv = static_cast<const char*>(d_recv);
      a.out = static_cast<char*>(d_out);
      a.clip = 1;
      for (int r = 0; r < P; ++r) {
        const int64_t S = r == me ? 0 : x->h_send[r * P + me];
        a.slo[r] = slice(S, k);
        a.shi[r] = slice(S, k + 1);
      }
      rc = run_move(ctx, kUnpack, a, x->n, x->lay.rank_dst_off, x->s_unpack, cap);
      if (rc) return rc;
    }
  }
  // the rows that stay on this rank: HBM only, while NCCL moves the rest
  if (x->n > 0) {
    MoveArgs a = make_args(P, me, x->d, x->d_len, x->d_origin, &x->bal, &x->lay, R);
    a.offs = x->bal.src_offset;
    a.members = x->bal.src_member;
    a.iter_rows = x->lay.in_rows;
    a.iter_cap = in_cap;
    a.in_cap = in_cap;
    a.out_cap = out_cap;
    a.in = static_cast<const char*>(d_in);
    a.out = static_cast<char*>(d_out);
    a.send = nullptr;
    const int rc = run_move(ctx, kPack, a, x->n, x->lay.rank_src_off, st, cap);
    if (rc) return rc;
  }
  (void)recv_cap;
  ORCH_CUDA_TRY(cudaEventRecord(x->ev_done, x->s_unpack));
  ORCH_CUDA_TRY(cudaStreamWaitEvent(st, x->ev_done, 0));
  return ORCH_OK;
}

}  // namespace

extern "C" {

int orch_dispatch_nccl(orch_ctx* ctx, orch_comm* comm, orch_xplan* x, size_t R, const void* d_in,
                       int64_t in_cap, void* d_out, int64_t out_cap, void* d_send,
                       int64_t send_cap, void* d_recv, int64_t recv_cap, void* stream) {
  if (!ctx || !comm || !x) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (!comm->comm) return fail(ORCH_INVALID_ARGUMENT, "loopback communicator has no NCCL");
  if (!x->fetched) return fail(ORCH_INVALID_ARGUMENT, "orch_xplan_fetch has not been called");
  const int P = comm->size, me = comm->rank;
  if (P != x->P) return fail(ORCH_INVALID_ARGUMENT, "plan and communicator rank counts differ");
  int rc = check_move_args(ctx, P, me, x->d, &x->bal, &x->lay, R);
  if (rc) return rc;
  const bool staged = d_send != nullptr;
  if (!aligned16(d_in) || !aligned16(d_out) || !aligned16(d_send) || !aligned16(d_recv))
    return fail(ORCH_INVALID_ARGUMENT, "row buffers must be 16-byte aligned");
  if (staged && !d_recv) return fail(ORCH_INVALID_ARGUMENT, "staged exchange needs a receive buffer");
  auto st = static_cast<cudaStream_t>(stream);
  // direct: the rows that stay move with one copy kernel, the rest item by item
  if (!staged && x->n > 0) {
    MoveArgs a = make_args(P, me, x->d, x->d_len, x->d_origin, &x->bal, &x->lay, R);
    a.offs = x->bal.src_offset;
    a.members = x->bal.src_member;
    a.iter_rows = x->lay.in_rows;
    a.iter_cap = in_cap;
    a.in_cap = in_cap;
    a.out_cap = out_cap;
    a.send_cap = send_cap;
    a.displ = x->lay.send_displ + me * P;
    a.in = static_cast<const char*>(d_in);
    a.out = static_cast<char*>(d_out);
    a.send = static_cast<char*>(d_send);  // NULL: off-rank rows go item by item below
    rc = run_move(ctx, kPack, a, x->n, x->lay.rank_src_off, st);
    if (rc) return rc;
  }
  // the layout's host mirror: waits for the metadata stream's copy only, never
  // for this stream
  ORCH_CUDA_TRY(cudaEventSynchronize(x->ready));
  if (x->h_in[me] > in_cap || x->h_out[me] > out_cap)
    return fail(ORCH_INVALID_ARGUMENT, "row buffer smaller than the layout");
  const char* in = static_cast<const char*>(d_in);
  char* out = static_cast<char*>(d_out);
  if (staged) {  // one send and one receive per peer and slice
    int64_t stot = 0, rtot = 0;
    for (int q = 0; q < P; ++q)
      if (q != me) {
        stot += x->h_send[me * P + q];
        rtot += x->h_send[q * P + me];
      }
    if (stot > send_cap || rtot > recv_cap)
      return fail(ORCH_INVALID_ARGUMENT, "send / receive buffer smaller than the off-rank rows");
    return staged_rounds(ctx, comm, x, R, d_in, in_cap, d_out, out_cap, d_send, send_cap, d_recv,
                         recv_cap, st);
  }
  const int c = x->d / P;
  ORCH_NCCL_TRY(ncclGroupStart());
  for (int k = 1; k < P; ++k) {  // peers in ring order from this rank
    const int q = (me + k) % P;
    for (int64_t i = 0; i < x->n; ++i) {
      const int r = x->h_org[i] / c, t = x->h_dst[i] / c;
      const size_t bytes = static_cast<size_t>(x->h_len[i]) * R;
      if (r == me && t == q)
        ORCH_NCCL_TRY(ncclSend(in + x->h_rso[i] * R, bytes, ncclInt8, q, comm->comm, st));
      else if (r == q && t == me)
        ORCH_NCCL_TRY(ncclRecv(out + x->h_rdo[i] * R, bytes, ncclInt8, q, comm->comm, st));
    }
  }
  ORCH_NCCL_TRY(ncclGroupEnd());
  return ORCH_OK;
}

int orch_comm_register(orch_comm* comm, void* ptr, size_t bytes, void** handle) {
  if (!comm || !ptr || !handle) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (!comm->comm) return fail(ORCH_INVALID_ARGUMENT, "loopback communicator has no NCCL");
  ORCH_NCCL_TRY(ncclCommRegister(comm->comm, ptr, bytes, handle));
  return ORCH_OK;
}

int orch_comm_deregister(orch_comm* comm, void* handle) {
  if (!comm || !comm->comm) return fail(ORCH_INVALID_ARGUMENT, "null communicator");
  ORCH_NCCL_TRY(ncclCommDeregister(comm->comm, handle));
  return ORCH_OK;
}

// ------------------------------------------------------------- cost model
int orch_batch_costs(orch_ctx* ctx, const orch_cost_model* model, int32_t batch_padded, int32_t d,
                     int64_t n, const int64_t* d_len, const int32_t* d_bin_offset,
                     const int32_t* d_bin_member, double* d_cost, double* d_stats, void* stream) {
  (void)n;
  if (!ctx || !model) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if ((model->padded != 0) != (batch_padded != 0))
    return fail(ORCH_INVALID_ARGUMENT, "cost model padding mode does not match batch padding mode");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  auto st = static_cast<cudaStream_t>(stream);
  launch(ctx, [&] {
    k_bin_cost<<<blocks_for(static_cast<int64_t>(d) * 32, kThreads), kThreads, 0, st>>>(
        *model, d, d_bin_offset, d_bin_member, d_len, nullptr, nullptr, nullptr, d_cost, nullptr);
  });
  if (d_stats) {
    launch(ctx, [&] { k_stats_only<<<1, 1024, 0, st>>>(d, d_cost, d_stats); });
  }
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_group_by_origin(orch_ctx* ctx, int32_t d, int64_t n, const int32_t* d_origin,
                         int32_t* d_bin_offset, int32_t* d_bin_member, void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  Plan plan;
  uint32_t *k_in, *k_out, *rs_kt, *rs_hist;
  int32_t *iota, *cnt, *rs_vt, *part;
  RsState* rs_state;
  plan.add(&k_in, nn);
  plan.add(&k_out, nn);
  plan.add(&iota, nn);
  plan.add(&cnt, d + 1);
  plan.add(&rs_kt, nn);
  plan.add(&rs_vt, nn);
  plan.add(&rs_hist, rs_hist_words(static_cast<int64_t>(nn)));
  plan.add(&rs_state, 1);
  plan.add(&part, static_cast<size_t>(rs_tiles(static_cast<int64_t>(d) + 1)));
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (d + 1), st));
  if (n > 0) {
    launch(ctx, [&] {
      k_origin_keys<<<blocks_for(n, kThreads), kThreads, 0, st>>>(d, n, d_origin, k_in, iota, cnt);
    });
    rc = rs_sort_pairs(ctx, k_in, iota, k_out, d_bin_member, rs_kt, rs_vt, n, false, rs_hist,
                       rs_state, st);
    if (rc) return rc;
  }
  rc = rs_exclusive_scan<int32_t>(ctx, cnt, d_bin_offset, d + 1, part, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_encode_lengths(orch_ctx* ctx, int64_t E, const int32_t* d_part_offset,
                        const int32_t* d_modality, const int64_t* d_meta_len, int32_t M,
                        const int64_t* h_rates, int64_t* d_encoded, int64_t* d_interleaved,
                        void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  if (M < 0 || M > 64) return fail(ORCH_INVALID_ARGUMENT, "modality count must be in [0, 64]");
  for (int m = 0; m < M; ++m)
    if (h_rates[m] < 1) return fail(ORCH_CONFIG_ERROR, "downsample rate must be >= 1");
  auto st = static_cast<cudaStream_t>(stream);
  Plan plan;
  int64_t* rates;
  plan.add(&rates, M > 0 ? M : 1);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  if (M > 0)
    ORCH_CUDA_TRY(cudaMemcpyAsync(rates, h_rates, sizeof(int64_t) * M, cudaMemcpyHostToDevice, st));
  if (E > 0)
    launch(ctx, [&] {
      k_encode<<<blocks_for(E, kThreads), kThreads, 0, st>>>(E, d_part_offset, d_modality,
                                                             d_meta_len, M, rates, d_encoded,
                                                             d_interleaved);
    });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

// Host-buffer variants (synchronous): inputs and outputs staged through the
// context's pinned mirror of a device buffer, one copy each way per call.
namespace {
struct StageLayout {
  size_t at = 0;
  size_t take(size_t b) {
    const size_t r = at;
    at += (b + 255) & ~size_t{255};
    return r;
  }
};
}  // namespace

constexpr size_t kZeroCopyBytes = 16384;

int orch_batch_costs_host(orch_ctx* ctx, const orch_cost_model* model, int32_t batch_padded,
                          int32_t d, int64_t n, const int64_t* h_len, const int32_t* h_bin_offset,
                          const int32_t* h_bin_member, double* h_cost, double* h_stats,
                          void* stream) {
  if (!ctx || !model) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if ((model->padded != 0) != (batch_padded != 0))
    return fail(ORCH_INVALID_ARGUMENT, "cost model padding mode does not match batch padding mode");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 0);
  StageLayout sl;
  const size_t o_len = sl.take(nn * 8), o_mem = sl.take(nn * 4);
  const size_t o_off = sl.take(static_cast<size_t>(d + 1) * 4);
  const size_t in_bytes = sl.at;
  const size_t o_cost = sl.take(static_cast<size_t>(d) * 8), o_stats = sl.take(24);
  char *hp, *dp;
  int rc = host_stage(ctx, sl.at, &hp, &dp);
  if (rc) return rc;
  if (nn) {
    memcpy(hp + o_len, h_len, nn * 8);
    memcpy(hp + o_mem, h_bin_member, nn * 4);
  }
  memcpy(hp + o_off, h_bin_offset, static_cast<size_t>(d + 1) * 4);
  // The costs (d doubles) and stats go straight to the pinned mirror (mapped
  // into the device's address space under UVA): no device-to-host copy call,
  // which is a third of a one-batch cost() round trip. Small inputs (one
  // batch: the per-batch cost() of stats_of) are read through the mapping too,
  // so such a call is one launch and one synchronize.
  const char* in = in_bytes <= kZeroCopyBytes ? hp : dp;
  if (in == dp) ORCH_CUDA_TRY(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, st));
  double* cost = reinterpret_cast<double*>(hp + o_cost);
  launch(ctx, [&] {
    k_bin_cost<<<blocks_for(static_cast<int64_t>(d) * 32, kThreads), kThreads, 0, st>>>(
        *model, d, reinterpret_cast<const int32_t*>(in + o_off),
        reinterpret_cast<const int32_t*>(in + o_mem), reinterpret_cast<const int64_t*>(in + o_len),
        nullptr, nullptr, nullptr, cost, nullptr);
  });
  if (h_stats)
    launch(ctx, [&] {
      k_stats_only<<<1, 1024, 0, st>>>(d, cost, reinterpret_cast<double*>(hp + o_stats));
    });
  ORCH_CUDA_TRY(cudaGetLastError());
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(h_cost, hp + o_cost, static_cast<size_t>(d) * 8);
  if (h_stats) memcpy(h_stats, hp + o_stats, 24);
  return ORCH_OK;
}

int orch_volume_matrix_host(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* h_len,
                            const int32_t* h_origin, const int32_t* h_dest_inst, int64_t* h_V,
                            void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 0);
  StageLayout sl;
  const size_t o_len = sl.take(nn * 8), o_org = sl.take(nn * 4), o_dst = sl.take(nn * 4);
  const size_t in_bytes = sl.at;
  const size_t o_V = sl.take(sizeof(int64_t) * d * d);
  char *hp, *dp;
  int rc = host_stage(ctx, sl.at, &hp, &dp);
  if (rc) return rc;
  if (nn) {
    memcpy(hp + o_len, h_len, nn * 8);
    memcpy(hp + o_org, h_origin, nn * 4);
    memcpy(hp + o_dst, h_dest_inst, nn * 4);
    ORCH_CUDA_TRY(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, st));
  }
  rc = orch_volume_matrix(ctx, d, n, reinterpret_cast<const int64_t*>(dp + o_len),
                          reinterpret_cast<const int32_t*>(dp + o_org),
                          reinterpret_cast<const int32_t*>(dp + o_dst),
                          reinterpret_cast<int64_t*>(dp + o_V), stream);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(hp + o_V, dp + o_V, sizeof(int64_t) * d * d,
                                cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(h_V, hp + o_V, sizeof(int64_t) * d * d);
  return ORCH_OK;
}

// ---------------------------------------------------------------- NCCL
int orch_comm_unique_id(unsigned char* h_id128) {
  ncclUniqueId id;
  ORCH_NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(h_id128, &id, sizeof id);
  return ORCH_OK;
}

int orch_comm_create(int32_t nranks, int32_t rank, const unsigned char* h_id128,
                     orch_comm** out) {
  if (!out || !h_id128) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ORCH_INVALID_ARGUMENT, "bad rank");
  ncclUniqueId id;
  memcpy(&id, h_id128, sizeof id);
  auto* c = new orch_comm();
  ORCH_CUDA_TRY(cudaGetDevice(&c->device));
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(ORCH_NCCL_ERROR, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  c->rank = rank;
  c->size = nranks;
  if (cudaMalloc(&c->barrier_buf, sizeof(int32_t)) != cudaSuccess) {
    ncclCommDestroy(c->comm);
    delete c;
    return fail(ORCH_CUDA_ERROR, "barrier buffer allocation failed");
  }
  cudaMemset(c->barrier_buf, 0, sizeof(int32_t));
  *out = c;
  return ORCH_OK;
}

void orch_comm_destroy(orch_comm* comm) {
  if (!comm) return;
  if (comm->comm) ncclCommDestroy(comm->comm);
  if (comm->barrier_buf) cudaFree(comm->barrier_buf);
  delete comm;
}

int32_t orch_comm_rank(const orch_comm* comm) { return comm ? comm->rank : 0; }
int32_t orch_comm_size(const orch_comm* comm) { return comm ? comm->size : 1; }

int orch_allgather_items(orch_ctx* ctx, orch_comm* comm, int64_t local_n, int64_t max_local,
                         const int64_t* d_local_pos, const int64_t* d_local_len,
                         const int32_t* d_local_origin, int64_t n, int64_t* d_len,
                         int32_t* d_origin, void* stream) {
  if (!ctx || !comm) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (!comm->comm) return fail(ORCH_INVALID_ARGUMENT, "loopback communicator has no NCCL");
  if (local_n > max_local || max_local < 0) return fail(ORCH_INVALID_ARGUMENT, "local_n > max_local");
  auto st = static_cast<cudaStream_t>(stream);
  const int P = comm->size;
  Plan plan;
  int64_t *sendrec, *recvrec;
  unsigned int* bad;
  plan.add(&sendrec, static_cast<size_t>(3 * (max_local > 0 ? max_local : 1)));
  plan.add(&recvrec, static_cast<size_t>(3 * (max_local > 0 ? max_local : 1) * P));
  plan.add(&bad, 1);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned int), st));
  if (max_local > 0) {
    launch(ctx, [&] {
      k_pack_records<<<blocks_for(max_local, kThreads), kThreads, 0, st>>>(
          local_n, max_local, d_local_pos, d_local_len, d_local_origin, sendrec);
    });
    ORCH_NCCL_TRY(ncclAllGather(sendrec, recvrec, static_cast<size_t>(3 * max_local), ncclInt64,
                                comm->comm, st));
    launch(ctx, [&] {
      k_scatter_records<<<blocks_for(max_local * P, kThreads), kThreads, 0, st>>>(
          max_local * P, n, recvrec, d_len, d_origin, bad);
    });
  }
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}


// ------------------------------------------------------------ windows / put
int orch_barrier(orch_comm* comm, void* stream) {
  if (!comm) return fail(ORCH_INVALID_ARGUMENT, "null communicator");
  if (!comm->comm) return fail(ORCH_INVALID_ARGUMENT, "loopback communicator has no NCCL");
  ORCH_NCCL_TRY(ncclAllReduce(comm->barrier_buf, comm->barrier_buf, 1, ncclInt32, ncclSum,
                              comm->comm, static_cast<cudaStream_t>(stream)));
  return ORCH_OK;
}

int orch_comm_create_local(int32_t nranks, int32_t rank, orch_comm** out) {
  if (!out) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks)
    return fail(ORCH_INVALID_ARGUMENT, "bad rank (loopback communicators hold 1..8 ranks)");
  auto* c = new orch_comm();
  ORCH_CUDA_TRY(cudaGetDevice(&c->device));
  c->rank = rank;
  c->size = nranks;
  c->loopback = true;
  *out = c;
  return ORCH_OK;
}

}  // extern "C"

namespace {

// Allocates the rows + flag area of one window (flags zeroed).
int window_alloc(orch_comm* comm, size_t bytes, orch_window** out) {
  auto* w = new orch_window();
  w->comm = comm;
  w->bytes = bytes;
  w->peers.assign(comm->size, nullptr);
  w->flags_off = (bytes + 255) & ~size_t{255};
  cudaError_t e = cudaMalloc(&w->base, w->flags_off + kFlagBytes);
  if (e != cudaSuccess) {
    delete w;
    return fail(ORCH_CUDA_ERROR, std::string("window allocation: ") + cudaGetErrorString(e));
  }
  e = cudaMemset(w->base + w->flags_off, 0, kFlagBytes);
  if (e != cudaSuccess) {
    cudaFree(w->base);
    delete w;
    return fail(ORCH_CUDA_ERROR, std::string("window flags: ") + cudaGetErrorString(e));
  }
  *out = w;
  return ORCH_OK;
}

int window_publish_peers(orch_window* w) {
  const int P = w->comm->size;
  ORCH_CUDA_TRY(cudaMalloc(&w->peers_dev, sizeof(char*) * P));
  ORCH_CUDA_TRY(cudaMemcpy(w->peers_dev, w->peers.data(), sizeof(char*) * P,
                           cudaMemcpyHostToDevice));
  return ORCH_OK;
}

void window_free(orch_window* w) {
  int dev0 = 0;
  cudaGetDevice(&dev0);
  cudaSetDevice(w->comm->device);
  if (w->nccl_win) {  // collective, like the registration
    cudaDeviceSynchronize();
    ncclCommWindowDeregister(w->comm->comm, w->nccl_win);
  } else if (!w->loopback) {
    for (int q = 0; q < static_cast<int>(w->peers.size()); ++q)
      if (q != w->comm->rank && w->peers[q]) cudaIpcCloseMemHandle(w->peers[q]);
  }
  if (w->peers_dev) cudaFree(w->peers_dev);
  if (w->base) {
    if (w->comm->comm && w->nccl_win) ncclMemFree(w->base);
    else cudaFree(w->base);
  }
  delete w;
  cudaSetDevice(dev0);
}


// What every rank contributes to the window set-up all-gather.
struct WindowCard {
  cudaIpcMemHandle_t handle;
  uint64_t bytes;
  uint64_t pad[7];
};

}  // namespace

extern "C" {

int orch_window_create(orch_ctx* ctx, orch_comm* comm, size_t bytes, orch_window** out) {
  if (!ctx || !comm || !out || bytes == 0) return fail(ORCH_INVALID_ARGUMENT, "bad window arguments");
  if (comm->loopback || !comm->comm)
    return fail(ORCH_INVALID_ARGUMENT, "loopback communicator: use orch_window_create_local");
  const int P = comm->size;
  orch_window* w = nullptr;
  int rc = window_alloc(comm, bytes, &w);
  if (rc) return rc;
  WindowCard mine{};
  mine.bytes = bytes;
  cudaError_t e = cudaIpcGetMemHandle(&mine.handle, w->base);
  // every rank's handle and size (the puts and barriers address peers with
  // this rank's flags offset and capacity, so all sizes must agree)
  char* dev = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&dev, sizeof(WindowCard) * (P + 1));
  if (e == cudaSuccess) e = cudaMemcpy(dev, &mine, sizeof mine, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (dev) cudaFree(dev);
    window_free(w);
    return fail(ORCH_CUDA_ERROR, std::string("window set-up: ") + cudaGetErrorString(e));
  }
  ncclResult_t nr = ncclAllGather(dev, dev + sizeof(WindowCard), sizeof(WindowCard), ncclChar,
                                  comm->comm, 0);
  std::vector<WindowCard> all(P);
  if (nr == ncclSuccess)
    e = cudaMemcpy(all.data(), dev + sizeof(WindowCard), sizeof(WindowCard) * P,
                   cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (nr != ncclSuccess || e != cudaSuccess) {
    window_free(w);
    return fail(nr != ncclSuccess ? ORCH_NCCL_ERROR : ORCH_CUDA_ERROR,
                std::string("window handle exchange: ") +
                    (nr != ncclSuccess ? ncclGetErrorString(nr) : cudaGetErrorString(e)));
  }
  for (int q = 0; q < P; ++q)
    if (all[q].bytes != bytes) {  // every rank sees the same cards, so every rank fails here
      window_free(w);
      return fail(ORCH_INVALID_ARGUMENT,
                  "orch_window_create: ranks passed different window sizes (rank " +
                      std::to_string(q) + ": " + std::to_string(all[q].bytes) + " bytes, rank " +
                      std::to_string(comm->rank) + ": " + std::to_string(bytes) + ")");
    }
  for (int q = 0; q < P; ++q) {
    if (q == comm->rank) {
      w->peers[q] = w->base;
      continue;
    }
    void* p = nullptr;
    e = cudaIpcOpenMemHandle(&p, all[q].handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      window_free(w);
      return fail(ORCH_CUDA_ERROR, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    w->peers[q] = static_cast<char*>(p);
  }
  rc = window_publish_peers(w);
  if (rc) {
    window_free(w);
    return rc;
  }
  *out = w;
  return ORCH_OK;
}

int orch_window_create_nccl(orch_ctx* ctx, orch_comm* comm, size_t bytes, orch_window** out) {
  if (!ctx || !comm || !out || bytes == 0) return fail(ORCH_INVALID_ARGUMENT, "bad window arguments");
  if (comm->loopback || !comm->comm)
    return fail(ORCH_INVALID_ARGUMENT, "loopback communicator: use orch_window_create_local");
  ORCH_CUDA_TRY(cudaSetDevice(comm->device));
  const int P = comm->size;
  // every rank's size first (the puts and barriers address peers with this
  // rank's flags offset and capacity, so all sizes must agree)
  uint64_t* sz = nullptr;
  ORCH_CUDA_TRY(cudaMalloc(&sz, sizeof(uint64_t) * (P + 1)));
  const uint64_t mine = bytes;
  cudaError_t e = cudaMemcpy(sz, &mine, sizeof mine, cudaMemcpyHostToDevice);
  ncclResult_t nr = e == cudaSuccess ? ncclAllGather(sz, sz + 1, 1, ncclUint64, comm->comm, 0)
                                     : ncclSuccess;
  std::vector<uint64_t> all(P);
  if (e == cudaSuccess && nr == ncclSuccess)
    e = cudaMemcpy(all.data(), sz + 1, sizeof(uint64_t) * P, cudaMemcpyDeviceToHost);
  cudaFree(sz);
  if (e != cudaSuccess) return fail(ORCH_CUDA_ERROR, std::string("window sizes: ") + cudaGetErrorString(e));
  if (nr != ncclSuccess) return fail(ORCH_NCCL_ERROR, std::string("window sizes: ") + ncclGetErrorString(nr));
  for (int q = 0; q < P; ++q)
    if (all[q] != bytes)
      return fail(ORCH_INVALID_ARGUMENT,
                  "orch_window_create_nccl: ranks passed different window sizes (rank " +
                      std::to_string(q) + ": " + std::to_string(all[q]) + " bytes, rank " +
                      std::to_string(comm->rank) + ": " + std::to_string(bytes) + ")");
  auto* w = new orch_window();
  w->comm = comm;
  w->bytes = bytes;
  w->peers.assign(P, nullptr);
  w->flags_off = (bytes + 255) & ~size_t{255};
  const size_t total = (w->flags_off + kFlagBytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) &
                       ~size_t{NCCL_WIN_REQUIRED_ALIGNMENT - 1};
  void* base = nullptr;
  nr = ncclMemAlloc(&base, total);
  if (nr != ncclSuccess) {
    delete w;
    return fail(ORCH_NCCL_ERROR, std::string("ncclMemAlloc: ") + ncclGetErrorString(nr));
  }
  w->base = static_cast<char*>(base);
  e = cudaMemset(w->base + w->flags_off, 0, kFlagBytes);
  if (e != cudaSuccess) {
    ncclMemFree(base);
    w->base = nullptr;
    delete w;
    return fail(ORCH_CUDA_ERROR, std::string("window flags: ") + cudaGetErrorString(e));
  }
  nr = ncclCommWindowRegister(comm->comm, base, total, &w->nccl_win, NCCL_WIN_COLL_SYMMETRIC);
  if (nr != ncclSuccess) {
    ncclMemFree(base);
    w->base = nullptr;
    w->nccl_win = nullptr;
    delete w;
    return fail(ORCH_NCCL_ERROR, std::string("ncclCommWindowRegister: ") + ncclGetErrorString(nr));
  }
  e = cudaMalloc(&w->peers_dev, sizeof(char*) * P);
  if (e == cudaSuccess) e = nccl_window_peers(w->nccl_win, P, w->peers_dev);
  if (e == cudaSuccess)
    e = cudaMemcpy(w->peers.data(), w->peers_dev, sizeof(char*) * P, cudaMemcpyDeviceToHost);
  // (this rank's own entry is its address in NCCL's flat mapping of the
  // window: another virtual address of the same memory as base)
  if (e != cudaSuccess) {
    window_free(w);
    return fail(ORCH_CUDA_ERROR, std::string("NCCL window peers: ") + cudaGetErrorString(e));
  }
  *out = w;
  return ORCH_OK;
}

int orch_window_create_local(orch_ctx* ctx, orch_comm* const* comms, int32_t P, size_t bytes,
                             orch_window** out) {
  if (!ctx || !comms || !out || bytes == 0 || P < 1 || P > 8)
    return fail(ORCH_INVALID_ARGUMENT, "bad window arguments");
  for (int r = 0; r < P; ++r)
    if (!comms[r] || !comms[r]->loopback || comms[r]->size != P || comms[r]->rank != r)
      return fail(ORCH_INVALID_ARGUMENT,
                  "orch_window_create_local needs loopback communicators of ranks 0..P-1");
  // Each rank's window lives on the device its loopback communicator was made
  // on: one device (all ranks on one GPU) or one per rank (several GPUs driven
  // by one process, peers reached over NVLink through peer access).
  int dev0 = 0;
  ORCH_CUDA_TRY(cudaGetDevice(&dev0));
  std::vector<orch_window*> ws(P, nullptr);
  int rc = ORCH_OK;
  for (int r = 0; r < P && !rc; ++r) {
    ORCH_CUDA_TRY(cudaSetDevice(comms[r]->device));
    rc = window_alloc(comms[r], bytes, &ws[r]);
    if (!rc) ws[r]->loopback = true;
  }
  for (int r = 0; r < P && !rc; ++r) {
    ORCH_CUDA_TRY(cudaSetDevice(comms[r]->device));
    for (int q = 0; q < P; ++q) {
      ws[r]->peers[q] = ws[q]->base;
      if (comms[q]->device != comms[r]->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(comms[q]->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          rc = fail(ORCH_CUDA_ERROR, std::string("peer access: ") + cudaGetErrorString(e));
        cudaGetLastError();  // clear "already enabled"
      }
    }
    if (!rc) rc = window_publish_peers(ws[r]);
  }
  for (int r = 0; r < P && !rc; ++r) {
    ORCH_CUDA_TRY(cudaSetDevice(comms[r]->device));
    ORCH_CUDA_TRY(cudaDeviceSynchronize());
  }
  cudaSetDevice(dev0);
  if (rc) {
    for (int q = 0; q < P; ++q)
      if (ws[q]) window_free(ws[q]);
    return rc;
  }
  for (int r = 0; r < P; ++r) out[r] = ws[r];
  return ORCH_OK;
}

int orch_window_barrier(orch_ctx* ctx, orch_window* w, void* stream) {
  if (!ctx || !w) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  const int P = w->comm->size;
  ++w->epoch;
  launch(ctx, [&] {
    k_window_barrier<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        w->peers_dev, w->flags_off, w->comm->rank, P, w->epoch,
        reinterpret_cast<int32_t*>(w->base + w->flags_off + kFlagStatus));
  });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_window_release(orch_ctx* ctx, orch_window* w, void* stream) {
  if (!ctx || !w) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (w->released >= w->epoch)
    return fail(ORCH_INVALID_ARGUMENT,
                "orch_window_release: no barrier-closed step left to release");
  ++w->released;
  launch(ctx, [&] {
    k_window_release<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        w->peers_dev, w->flags_off, w->comm->rank, w->comm->size, w->released);
  });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_window_status(const orch_window* w, int32_t* h_status) {
  if (!w || !h_status) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  ORCH_CUDA_TRY(cudaMemcpy(h_status, w->base + w->flags_off + kFlagStatus, sizeof(int32_t),
                           cudaMemcpyDeviceToHost));
  return ORCH_OK;
}

void* orch_window_ptr(const orch_window* w) { return w ? w->base : nullptr; }
size_t orch_window_bytes(const orch_window* w) { return w ? w->bytes : 0; }

int orch_window_destroy(orch_window* w) {
  if (!w) return ORCH_OK;
  int rc = ORCH_OK;
  // every rank must be done writing into / reading from the windows
  if (!w->loopback) rc = orch_barrier(w->comm, nullptr);
  int dev0 = 0;
  cudaGetDevice(&dev0);
  cudaSetDevice(w->comm->device);
  cudaDeviceSynchronize();
  cudaSetDevice(dev0);
  window_free(w);
  return rc;
}

}  // extern "C"

namespace {

// The first put after a barrier on a stream: k_window_acquire waits until
// every rank released the steps closed so far (see orch_window_release).
int window_acquire(orch_ctx* ctx, orch_window* w, void* stream) {
  if (w->epoch == 0 || (w->acq_epoch == w->epoch && w->acq_stream == stream)) return ORCH_OK;
  char* flags = w->base + w->flags_off;
  auto st = static_cast<cudaStream_t>(stream);
  launch(ctx, [&] {
    k_window_acquire<<<1, 32, 0, st>>>(reinterpret_cast<const uint64_t*>(flags + kFlagFree),
                                       w->comm->size, w->epoch,
                                       reinterpret_cast<uint64_t*>(flags + kFlagAcquired),
                                       reinterpret_cast<int32_t*>(flags + kFlagStatus));
  });
  ORCH_CUDA_TRY(cudaGetLastError());
  w->acq_epoch = w->epoch;
  w->acq_stream = stream;
  return ORCH_OK;
}

}  // namespace

extern "C" {

int orch_put_at(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                const int32_t* d_origin, const orch_balance_out* bal, const orch_layout_out* L,
                size_t R, const void* d_in, int64_t in_cap, orch_window* out_win,
                size_t win_offset, void* stream) {
  if (!comm || !out_win) return fail(ORCH_INVALID_ARGUMENT, "put needs a communicator and a window");
  if (out_win->comm != comm) return fail(ORCH_INVALID_ARGUMENT, "window belongs to another communicator");
  const int P = comm->size, me = comm->rank;
  int rc = check_move_args(ctx, P, me, d, bal, L, R);
  if (rc) return rc;
  if (!aligned16(d_in)) return fail(ORCH_INVALID_ARGUMENT, "row buffers must be 16-byte aligned");
  if (win_offset % 16 != 0 || win_offset > out_win->bytes)
    return fail(ORCH_INVALID_ARGUMENT, "window offset must be a multiple of 16 inside the window");
  if (n > 0) {
    MoveArgs a = make_args(P, me, d, d_len, d_origin, bal, L, R);
    a.offs = bal->src_offset;
    a.members = bal->src_member;
    a.iter_rows = L->in_rows;
    a.iter_cap = in_cap;
    a.in_cap = in_cap;
    a.out_cap = static_cast<int64_t>((out_win->bytes - win_offset) / R);
    a.in = static_cast<const char*>(d_in);
    a.out = out_win->base + win_offset;
    a.peer_out = out_win->peers_dev;
    a.win_off = win_offset;
    char* flags = out_win->base + out_win->flags_off;
    a.acquired = reinterpret_cast<const uint64_t*>(flags + kFlagAcquired);
    a.need_free = out_win->epoch;  // the steps closed so far must all be consumed
    rc = window_acquire(ctx, out_win, stream);
    if (rc) return rc;
    static const int scramble = [] {
      const char* e = getenv("ORCH_PUT_SCRAMBLE");
      return e ? atoi(e) : 1;
    }();
    a.scramble = scramble;
    rc = run_move(ctx, kPut, a, n, L->rank_src_off, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
  }
  return ORCH_OK;
}

int orch_put(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
             const int32_t* d_origin, const orch_balance_out* bal, const orch_layout_out* L,
             size_t R, const void* d_in, int64_t in_cap, orch_window* out_win, void* stream) {
  return orch_put_at(ctx, comm, d, n, d_len, d_origin, bal, L, R, d_in, in_cap, out_win, 0,
                     stream);
}

int orch_dispatch_put(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                      const int32_t* d_origin, const orch_balance_out* bal,
                      const orch_layout_out* L, size_t R, const void* d_in, int64_t in_cap,
                      orch_window* out_win, void* stream) {
  int rc = orch_put(ctx, comm, d, n, d_len, d_origin, bal, L, R, d_in, in_cap, out_win, stream);
  if (rc) return rc;
  // rows from every peer have landed once every rank passed its put kernel
  return orch_window_barrier(ctx, out_win, stream);
}

}  // extern "C"

namespace {

int gather_window_wrap(orch_window* w, int64_t max_n, orch_gather_window** out) {
  auto* g = new orch_gather_window();
  g->max_n = max_n;
  g->w = w;
  ORCH_CUDA_TRY(cudaMalloc(&g->stamps, 64 * sizeof(uint64_t)));
  ORCH_CUDA_TRY(cudaMemset(g->stamps, 0, 64 * sizeof(uint64_t)));
  // flags start at 0 on every rank before any peer can store into them
  ORCH_CUDA_TRY(cudaMemset(w->base, 0, w->bytes));
  *out = g;
  return ORCH_OK;
}

size_t gather_window_bytes(int64_t max_n, int P) {
  return gather_flags_off(max_n) + 16 * static_cast<size_t>(P);
}

}  // namespace

extern "C" {

int orch_gather_window_create(orch_ctx* ctx, orch_comm* comm, int64_t max_n,
                              orch_gather_window** out) {
  if (!ctx || !comm || !out || max_n < 1) return fail(ORCH_INVALID_ARGUMENT, "bad gather window arguments");
  orch_window* w = nullptr;
  int rc = orch_window_create(ctx, comm, gather_window_bytes(max_n, comm->size), &w);
  if (rc) return rc;
  rc = gather_window_wrap(w, max_n, out);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaDeviceSynchronize());
  rc = orch_barrier(comm, nullptr);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaDeviceSynchronize());
  return ORCH_OK;
}

int orch_gather_window_create_nccl(orch_ctx* ctx, orch_comm* comm, int64_t max_n,
                                   orch_gather_window** out) {
  if (!ctx || !comm || !out || max_n < 1) return fail(ORCH_INVALID_ARGUMENT, "bad gather window arguments");
  orch_window* w = nullptr;
  int rc = orch_window_create_nccl(ctx, comm, gather_window_bytes(max_n, comm->size), &w);
  if (rc) return rc;
  rc = gather_window_wrap(w, max_n, out);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaDeviceSynchronize());
  rc = orch_barrier(comm, nullptr);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaDeviceSynchronize());
  return ORCH_OK;
}

int orch_gather_window_create_local(orch_ctx* ctx, orch_comm* const* comms, int32_t P,
                                    int64_t max_n, orch_gather_window** out) {
  if (!ctx || !comms || !out || max_n < 1 || P < 1 || P > 8)
    return fail(ORCH_INVALID_ARGUMENT, "bad gather window arguments");
  std::vector<orch_window*> ws(P, nullptr);
  int rc = orch_window_create_local(ctx, comms, P, gather_window_bytes(max_n, P), ws.data());
  if (rc) return rc;
  int dev0 = 0;
  ORCH_CUDA_TRY(cudaGetDevice(&dev0));
  for (int r = 0; r < P; ++r) {
    ORCH_CUDA_TRY(cudaSetDevice(comms[r]->device));
    rc = gather_window_wrap(ws[r], max_n, &out[r]);
    if (rc) return rc;
    ORCH_CUDA_TRY(cudaDeviceSynchronize());
  }
  ORCH_CUDA_TRY(cudaSetDevice(dev0));
  return ORCH_OK;
}

int orch_gather_window_destroy(orch_gather_window* g) {
  if (!g) return ORCH_OK;
  const int rc = orch_window_destroy(g->w);
  cudaFree(g->stamps);
  delete g;
  return rc;
}

int orch_gather_window_stamps(const orch_gather_window* g, uint64_t* h_out) {
  if (!g || !h_out) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  ORCH_CUDA_TRY(cudaMemcpy(h_out, g->stamps, 64 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return ORCH_OK;
}

int orch_allgather_items_put(orch_ctx* ctx, orch_gather_window* g, int64_t local_n,
                             const int64_t* d_local_pos, const int64_t* d_local_len,
                             const int32_t* d_local_origin, int64_t n, int64_t* d_len,
                             int32_t* d_origin, int32_t* d_status, void* stream) {
  if (!ctx || !g) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (n > g->max_n || local_n < 0 || local_n > n)
    return fail(ORCH_INVALID_ARGUMENT, "gather window holds fewer items than n");
  GatherArgs a{};
  a.peers = g->w->peers_dev;
  a.me = g->w->comm->rank;
  a.P = g->w->comm->size;
  a.epoch = ++g->epoch;
  a.max_n = g->max_n;
  a.n = n;
  a.local_n = local_n;
  a.pos = d_local_pos;
  a.len = d_local_len;
  a.org = d_local_origin;
  a.out_len = d_len;
  a.out_org = d_origin;
  a.status = d_status;
  a.stamps = g->stamps;
  auto st = static_cast<cudaStream_t>(stream);
  static PerDeviceOnce configured;
  const int rc_attr = configured([&]() -> int {
    ORCH_CUDA_TRY(max_carveout(k_gather_put));
    return ORCH_OK;
  });
  if (rc_attr) return rc_attr;
  launch(ctx, [&] { k_gather_put<<<1, 1024, 0, st>>>(a); });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"
