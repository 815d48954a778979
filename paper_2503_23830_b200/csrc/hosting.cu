// Node-wise ("GPU-wise") hosting: permute which
// instance hosts which destination batch so that the slow links carry as
// little of the rearrangement as possible -- topology.cpp:55-303
// (inter_node_egress, solve_hosting, nodewise_rearrange). On one NVSwitch box
// a "node" is a GPU holding c = d/P logical instances and the slow link is
// NVLink (the fast one is the GPU's own HBM).
//
// solve_hosting is an exact depth-first branch and bound in the reference
// (topology.cpp:87-262). Its answer is fixed by the search order: the
// incumbents (identity, then greedy if strictly better) unless some leaf is
// strictly better, in which case the FIRST optimal leaf in DFS order. That is
// independent of how hard the search prunes, so the device search is free to
// be parallel as long as its bounds are valid:
//   pass 1  optimum value V*, pruning on lb >= best (a global atomic incumbent);
//   pass 2  (only if V* beats the incumbents) the first leaf of value V* in DFS
//           order, pruning on lb > V* and on paths that already sort after the
//           best V*-leaf found so far.
// The reference also reports how many nodes its sequential DFS entered
// (nodes_visited); orch_solve_hosting_host replays that count exactly:
//   pass 3  (one launch per link) the reference's chain of improving leaves:
//           the first leaf after the previous link, in DFS order, of value
//           below it -- pass 2 with a threshold and a lower end;
//   pass 4  a DFS that cuts each node on lb >= the incumbent the reference held
//           when it reached it (set by the chain leaves that sort before it),
//           and counts.
// Work: the DFS tree cut at depth k0 into <= 8192 prefixes, then work stealing:
// one warp runs a subtree depth-first (lane = node); when warps are idle, a busy
// warp donates the shallowest untried sibling of its current path to a global
// queue. A subtree is identified by its path of candidate positions, and DFS
// order is the lexicographic order of paths, so pass 2 stays exact.
// d <= 64 keeps the tables and the warps' DFS stacks in shared memory; beyond
// (orch_solve_hosting_host up to ORCH_MAX_INSTANCES, e.g. C4's d = 2560) they
// stay in global memory and grid-wide kernels build the tables (k_hw_*).
// The bound is the reference's lower_bound -- max over nodes of
// (total - gained - optimistic gain) -- read in O(1): the unassigned batches
// at depth k are exactly order[k..d), so the optimistic gain of node n with r
// slots left is a table og[k][n][r] built once.
#include <algorithm>
#include <cstring>
#include <climits>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "plan.cuh"

namespace orchb {
namespace {

constexpr int kHostMaxD = 64;
constexpr int kHostMaxNodes = 32;                  // lane = node
constexpr int kHostWarps = 8;
constexpr long long kHostTasks = 8192;
constexpr int kHostGrid = 148;
constexpr int kHostQueue = 16384;  // donated subtrees waiting for a warp
constexpr int kHostQueueWide = 4096;  // d > kHostMaxD: paths are d bytes
constexpr int kHostChainMax = 1024;  // improving leaves of the reference's sequential search
constexpr unsigned long long kHostVisitBudget = 1ull << 31;
#ifndef ORCH_HOST_SLEEP
#define ORCH_HOST_SLEEP 2000
#endif
#ifndef ORCH_HOST_CHECK
#define ORCH_HOST_CHECK 63
#endif

// Per-call buffers of the multi-CTA search, sized for this d (workspace): the
// search tables, the stored paths (d candidate positions each) and the work
// queue; with d > kHostMaxD also the warps' DFS stacks.
struct HostBufs {
  int32_t* order;       // branching order (descending regret, stable)
  int32_t* incumbent;
  // search tables by depth k (the batch order[k])
  int64_t* g2;          // [k][node] gain of node for order[k]
  uint8_t* no;          // [k][j] j-th candidate: descending gain, ties by node
  uint8_t* pos;         // [k][node] inverse of no
  int64_t* og;          // [k][node][r] sum of the top r gains over order[k..d)
  uint8_t* best_path;   // passes 2, 3: candidate position per depth
  uint8_t* after_path;  // pass 3
  uint8_t* chain_path;  // pass 4: [kHostChainMax][d]
  unsigned* q_ready;    // pass tag | (index + 1) once published, 0 once read
  uint16_t* q_depth;
  uint8_t* q_path;      // [q_cap][d]
  uint8_t* stacks;      // wide: [kHostGrid * kHostWarps][wide_stack_bytes(d)]
};

struct HostState {
  int d, c, nodes, k0;
  long long tasks;                       // nodes^k0 prefixes, numbered in DFS order
  int wide;                              // d > kHostMaxD: tables and stacks in global memory
  unsigned q_cap;                        // work-queue slots
  HostBufs b;
  int64_t node_total[kHostMaxNodes];
  int64_t incumbent_value;
  unsigned long long best_value;            // pass 1 incumbent value (starts at the incumbents')
  unsigned long long visits;
  int overflow;
  // work distribution, reset before each pass
  unsigned long long task_counter;          // initial prefixes handed out
  unsigned q_head, q_tail;                  // donated subtrees
  int pending;                              // tasks queued or running
  int idle;                                 // warps waiting for work
  int lock;
  int done_ctas;                            // pass 1 CTAs finished (the last one resets for pass 2)
  int have_best;                            // pass 2: b.best_path holds a V*-leaf
  unsigned long long best_key;              // passes 2, 3: least path_key of a found leaf
  int64_t best_leaf;                        // passes 2, 3: the recorded leaf's value
  // pass 3 (one link of the reference's chain of improving leaves): the first
  // leaf after b.after_path (when after_depth == d) with value <= thresh
  int64_t thresh;
  int after_depth;
  // pass 4 (the reference's visit count): chain_bound[i] is the reference's
  // incumbent value once the first i chain leaves have been offered
  int chain_len;
  int chain_done;                           // 1: complete, 2: beyond the budget or kHostChainMax
  int64_t chain_last;                       // chain_bound[chain_len]
  int64_t chain_bound[kHostChainMax + 1];
#ifdef ORCH_HOST_DEBUG
  unsigned long long dbg_t0, dbg_found, dbg_end, dbg_task_max, dbg_donated, dbg_first_end;
  unsigned long long dbg_visits0, dbg_visits_max;
#endif
};

// ----------------------------------------------------------- preparation
// gains, node totals, branching order, incumbents and search tables
// (topology.cpp:195-262), block-wide in shared memory: every global round trip
// of this latency-bound chain costs microseconds while the row exchange loads
// the memory system, so nothing here touches global memory.
template <int MD>
struct Prep {
  unsigned long long V[MD * MD];                // [src instance][dest batch]
  int64_t gain[kHostMaxNodes * MD];             // [node][batch]
  int64_t g2[MD * kHostMaxNodes];               // [k][node] gain of node for order[k]
  int64_t og[(MD + 1) * (MD + kHostMaxNodes)];  // [k][node][r], (d+1)*nodes*(c+1) entries
  int64_t node_total[kHostMaxNodes];
  int64_t regret[MD];
  int64_t vals[2];          // host_value of identity, greedy
  int64_t incumbent_value;
  int64_t root_lb;          // the bound at the root: no leaf is below it
  int32_t order[MD], ident[MD], greedy[MD], incumbent[MD];
  uint8_t no[MD * kHostMaxNodes];   // [k][j] j-th candidate: descending gain, ties by node
  uint8_t pos[MD * kHostMaxNodes];  // [k][node] inverse of no
};

// argmax over lanes of v (v >= -1), lowest lane on ties
__device__ __forceinline__ int warp_argmax_first(int64_t v) {
  int bl = threadIdx.x & 31;
  int64_t bv = v;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(~0u, bv, o);
    const int ol = __shfl_xor_sync(~0u, bl, o);
    if (ov > bv || (ov == bv && ol < bl)) {
      bv = ov;
      bl = ol;
    }
  }
  return bl;
}

// S.V must be filled (and a __syncthreads() passed); blockDim.x >= 96 and >= d.
template <int MD>
__device__ void prep_run(Prep<MD>& S, int d, int c) {
  const int nodes = d / c, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < nodes * d; i += blockDim.x) {
    const int nd = i / d, b = i % d;
    int64_t g = 0;
    for (int r = nd * c; r < (nd + 1) * c; ++r) g += static_cast<int64_t>(S.V[r * d + b]);
    S.gain[i] = g;
  }
  __syncthreads();
  if (t < nodes) {
    int64_t tot = 0;
    for (int b = 0; b < d; ++b) tot += S.gain[t * d + b];
    S.node_total[t] = tot;
  }
  if (t < d) {  // top - second gain over the nodes
    int64_t top = 0, second = 0;
    for (int nd = 0; nd < nodes; ++nd) {
      const int64_t g = S.gain[nd * d + t];
      if (g > top) {
        second = top;
        top = g;
      } else if (g > second) {
        second = g;
      }
    }
    S.regret[t] = top - second;
  }
  __syncthreads();
  if (t < d) {  // stable order by descending regret (the reference's insertion sort)
    int r = 0;
    for (int b = 0; b < d; ++b) r += S.regret[b] > S.regret[t] || (S.regret[b] == S.regret[t] && b < t);
    S.order[r] = t;
    S.ident[t] = t / c;
  }
  __syncthreads();
  if (warp == 0) {  // greedy incumbent: each batch in order to the best node with room
    int room = lane < nodes ? c : 0;
    for (int k = 0; k < d; ++k) {
      const int b = S.order[k];
      const int pick = warp_argmax_first(room > 0 ? S.gain[lane * d + b] : -1);
      if (lane == pick) {
        --room;
        S.greedy[b] = pick;
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // per depth: candidate nodes by descending gain, ties by node
    for (int k = lane; k < d; k += 32) {
      const int b = S.order[k];
      uint8_t* no = S.no + k * nodes;
      for (int nd = 0; nd < nodes; ++nd) {
        S.g2[k * nodes + nd] = S.gain[nd * d + b];
        int j = nd - 1;
        while (j >= 0 && S.gain[no[j] * d + b] < S.gain[nd * d + b]) {
          no[j + 1] = no[j];
          --j;
        }
        no[j + 1] = static_cast<uint8_t>(nd);
      }
      for (int j = 0; j < nodes; ++j) S.pos[k * nodes + no[j]] = static_cast<uint8_t>(j);
    }
  } else if (warp == 2 && lane < nodes) {  // og[k][node][r], deepest level first
    int64_t top[MD];
    int have = 0;
    for (int k = d; k >= 0; --k) {
      if (k < d) {
        const int64_t g = S.gain[lane * d + S.order[k]];
        int j = -1;
        if (have < c) j = have++;
        else if (top[c - 1] < g) j = c - 1;  // else not in the top c (sums unchanged on ties)
        if (j >= 0) {
          while (j > 0 && top[j - 1] < g) {
            top[j] = top[j - 1];
            --j;
          }
          top[j] = g;
        }
      }
      int64_t* og = S.og + (static_cast<size_t>(k) * nodes + lane) * (c + 1);
      int64_t acc = 0;
      og[0] = 0;
      for (int r = 1; r <= c; ++r) {
        if (r <= have) acc += top[r - 1];
        og[r] = acc;
      }
    }
  }
  __syncthreads();
  if (warp < 2) {  // host_value: worst node egress of identity (warp 0) and greedy (warp 1)
    const int32_t* asg = warp == 0 ? S.ident : S.greedy;
    int64_t e = INT64_MIN;
    if (lane < nodes) {
      e = S.node_total[lane];
      for (int b = 0; b < d; ++b)
        if (asg[b] == lane) e -= S.gain[lane * d + b];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int64_t x = __shfl_xor_sync(~0u, e, o);
      e = x > e ? x : e;
    }
    if (lane == 0) S.vals[warp] = e;
  } else if (warp == 2) {  // lower bound at the root
    int64_t e = lane < nodes ? S.node_total[lane] - S.og[static_cast<size_t>(lane) * (c + 1) + c] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int64_t x = __shfl_xor_sync(~0u, e, o);
      e = x > e ? x : e;
    }
    if (lane == 0) S.root_lb = e > 0 ? e : 0;
  }
  __syncthreads();
  const bool g_better = S.vals[1] < S.vals[0];  // offer(greedy) replaces only when strictly better
  if (t < d) S.incumbent[t] = g_better ? S.greedy[t] : S.ident[t];
  if (t == 0) S.incumbent_value = g_better ? S.vals[1] : S.vals[0];
  __syncthreads();
}

// volume matrix (topology.cpp:40-53) into S.V: from the items, or a given d x d
template <int MD>
__device__ void prep_volume(Prep<MD>& S, int d, int64_t n, const int64_t* len, const int32_t* origin,
                            const int32_t* dest, const int64_t* Vin) {
  for (int i = threadIdx.x; i < d * d; i += blockDim.x)
    S.V[i] = Vin ? static_cast<unsigned long long>(Vin[i]) : 0ull;
  __syncthreads();
  if (!Vin)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      atomicAdd(&S.V[origin[i] * d + dest[i]], static_cast<unsigned long long>(len[i]));
  __syncthreads();
}

// per warp, for depths up to md: choice stack ch[md] (u8), then avail[md] and
// donated[md] (u32 masks), then lo[md+1] and hi[md+1] (u16, pass 4: the chain
// leaves below the path). In shared memory (md = kHostMaxD) unless wide.
__host__ __device__ inline size_t warp_stack_bytes(int md) {
  return ((static_cast<size_t>(md + 3) & ~size_t{3}) + 8 * static_cast<size_t>(md) +
          4 * static_cast<size_t>(md + 1) + 15) & ~size_t{15};
}

struct HostSmem {
  const int64_t* g2;
  const int64_t* og;
  const uint8_t* no;
  const uint8_t* pos;
};

__host__ __device__ inline size_t host_table_bytes(int d, int c) {  // 16-byte aligned
  const int nodes = d / c;
  const size_t b = sizeof(int64_t) * (static_cast<size_t>(d) * nodes +
                                      static_cast<size_t>(d + 1) * nodes * (c + 1)) +
                   2 * static_cast<size_t>(d) * nodes;
  return (b + 15) & ~size_t{15};
}
__host__ __device__ inline size_t host_smem_bytes(int d, int c) {
  if (d > kHostMaxD) return 0;  // wide: tables and stacks stay in global memory
  return host_table_bytes(d, c) + kHostWarps * warp_stack_bytes(kHostMaxD);
}

// kWide: the tables stay in global memory. A template, so that the narrow
// search's table and stack pointers are known to be shared-memory ones (LDS/STS
// instead of generic loads and stores in the DFS loop).
template <bool kWide>
__device__ __forceinline__ HostSmem host_load_tables(const HostState& H, unsigned char* raw) {
  const int d = H.d, c = H.c, nodes = H.nodes;
  if constexpr (kWide) return HostSmem{H.b.g2, H.b.og, H.b.no, H.b.pos};
  int64_t* g2 = reinterpret_cast<int64_t*>(raw);
  int64_t* og = g2 + d * nodes;
  uint8_t* no = reinterpret_cast<uint8_t*>(og + (d + 1) * nodes * (c + 1));
  uint8_t* pos = no + d * nodes;
  for (int i = threadIdx.x; i < d * nodes; i += blockDim.x) {
    g2[i] = H.b.g2[i];
    no[i] = H.b.no[i];
    pos[i] = H.b.pos[i];
  }
  for (int i = threadIdx.x; i < (d + 1) * nodes * (c + 1); i += blockDim.x) og[i] = H.b.og[i];
  __syncthreads();
  return HostSmem{g2, og, no, pos};
}

// max over the warp of nonnegative 64-bit values: two 32-bit REDUX steps
__device__ __forceinline__ int64_t warp_max_nonneg(int64_t v) {
  const uint64_t u = v > 0 ? static_cast<uint64_t>(v) : 0ull;
  const unsigned hi = static_cast<unsigned>(u >> 32), lo = static_cast<unsigned>(u);
  const unsigned mh = __reduce_max_sync(~0u, hi);
  const unsigned ml = __reduce_max_sync(~0u, hi == mh ? lo : 0u);
  return static_cast<int64_t>((static_cast<uint64_t>(mh) << 32) | ml);
}

__device__ __forceinline__ unsigned long long volatile_load(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ unsigned volatile_u32(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}
__device__ __forceinline__ int volatile_i32(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}

// Lane-parallel lexicographic compare of path a[0, k) with b[0, k): -1, 0, 1.
__device__ __forceinline__ int path_cmp(const uint8_t* a, const volatile uint8_t* b, int k,
                                        int lane) {
  for (int l0 = 0; l0 < k; l0 += 32) {
    const int l = l0 + lane;
    const int x = l < k ? a[l] : 0, y = l < k ? b[l] : 0;
    const unsigned diff = __ballot_sync(~0u, x != y);
    if (diff) {
      const int f = __ffs(diff) - 1;
      const int xf = __shfl_sync(~0u, x, f), yf = __shfl_sync(~0u, y, f);
      return xf < yf ? -1 : 1;
    }
  }
  return 0;
}

#ifdef ORCH_HOST_DEBUG
__device__ __forceinline__ unsigned long long dbg_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// The first km positions of a path packed kb bits each, most significant
// first (kb = bits of a node index): keys order as paths do, so a path whose
// key (missing positions as 0: the least leaf below it) exceeds a found leaf's
// key sorts after that leaf, and one atomicMin keeps the least key found.
__device__ __forceinline__ unsigned long long path_key(const uint8_t* ch, int k, int kb, int km,
                                                       int lane) {
  const int m = k < km ? k : km;
  unsigned hi = 0, lo = 0;
  for (int l0 = 0; l0 < m; l0 += 32) {
    const int l = l0 + lane;
    if (l < m) {
      const unsigned long long v = static_cast<unsigned long long>(ch[l]) << (64 - kb * (l + 1));
      hi |= static_cast<unsigned>(v >> 32);
      lo |= static_cast<unsigned>(v);
    }
  }
  hi = __reduce_or_sync(~0u, hi);
  lo = __reduce_or_sync(~0u, lo);
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

struct WarpStack {
  uint8_t* ch;        // candidate position chosen per depth
  unsigned* avail;    // positions with room per depth (as of choosing there)
  unsigned* donated;  // positions given away per depth (current path only)
  uint16_t* lo;       // pass 4, per depth k: chain leaves [lo, hi) share the path's
  uint16_t* hi;       //   first k positions; those below lo sort before the node
};

// Pass 4: the chain leaves below the node at depth k + 1 reached by position
// j, from those [lo, hi) below its parent (sorted: ascending position at k).
__device__ __forceinline__ void chain_step(const HostState& H, int k, int j, int lo, int hi,
                                           int lane, int& nlo, int& nhi) {
  int less = 0, same = 0;
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const int i = i0 + lane;
    const int x = i < hi ? H.b.chain_path[static_cast<size_t>(i) * H.d + k] : 256;
    less += __popc(__ballot_sync(~0u, x < j));
    same += __popc(__ballot_sync(~0u, x == j));
  }
  nlo = lo + less;
  nhi = nlo + same;
}

// the work queue's publication word for a subtree: launch tag, slot + 1 (never 0)
__device__ __forceinline__ unsigned q_tag(int pass, unsigned slot) {
  return (static_cast<unsigned>(pass & 3) << 30) | (slot + 1);
}

// Depth-first search of the subtree below the path ch[0, root) (state: this
// lane's room / gained). pass 1 prunes lb >= best and lowers the global
// incumbent at leaves; pass 2 prunes lb > vstar and paths after the best
// V*-leaf, and records a V*-leaf if it sorts first; pass 3 is pass 2 restricted
// to leaves after H.after_path; pass 4 prunes a node on lb >= the incumbent the
// reference holds when it gets there (chain_bound[lo]) and only counts.
// Donates siblings to idle warps. Returns when the subtree is exhausted (or cut).
__device__ __forceinline__ unsigned long long host_dfs(HostState& H, const HostSmem& T, int pass, int64_t vstar, WarpStack W,
                         int root, int room, int64_t gained) {
  const int d = H.d, c = H.c, nodes = H.nodes, lane = threadIdx.x & 31;
  const bool active = lane < nodes;
  const int64_t total = active ? H.node_total[lane] : 0;
  int64_t best = static_cast<int64_t>(
      __shfl_sync(~0u, (threadIdx.x & 31) == 0 ? volatile_load(&H.best_value) : 0ull, 0));
  unsigned long long visits = 0;
  int k = root, jstart = 0;
  bool descend = true;
  W.donated[root] = 0;
  const int after = pass == 3 ? H.after_depth : 0;
  const int kb = nodes > 1 ? 32 - __clz(nodes - 1) : 1, km = d < 64 / kb ? d : 64 / kb;
  if (pass == 4) {  // the chain leaves below the subtree's root
    int lo = 0, hi = H.chain_len;
    for (int l = 0; l < root; ++l) chain_step(H, l, W.ch[l], lo, hi, lane, lo, hi);
    if (lane == 0) {
      W.lo[root] = static_cast<uint16_t>(lo);
      W.hi[root] = static_cast<uint16_t>(hi);
    }
    __syncwarp();
  }
  for (;;) {
    if (descend) {
      ++visits;
      if ((visits & ORCH_HOST_CHECK) == 0) {
        // shared flags are read by lane 0 and broadcast: every branch below
        // must be warp-uniform (the warp-collective ops need all 32 lanes)
        if (__shfl_sync(~0u, lane == 0 ? volatile_i32(&H.overflow) : 0, 0)) break;
        if ((visits & 65535) == 0 && lane == 0 &&
            atomicAdd(&H.visits, 65536ull) > kHostVisitBudget)
          H.overflow = 1;
        if (pass == 1) {
          best = static_cast<int64_t>(
              __shfl_sync(~0u, lane == 0 ? volatile_load(&H.best_value) : 0ull, 0));
        } else if ((pass == 2 || pass == 3) &&
                   path_key(W.ch, k, kb, km, lane) >
                       __shfl_sync(~0u, lane == 0 ? volatile_load(&H.best_key) : 0ull, 0)) {
          break;  // everything left in this subtree sorts after the best V*-leaf
        }
        // donate the shallowest untried sibling when warps wait for work
        int want = 0;
        if (lane == 0) {
          const unsigned queued = volatile_u32(&H.q_tail) - volatile_u32(&H.q_head);
          want = volatile_i32(&H.idle) > static_cast<int>(queued) && queued < H.q_cap - H.q_cap / 8;
        }
        if (__shfl_sync(~0u, want, 0)) {
          int lvl = -1;
          unsigned untried = 0;
          for (int l0 = root; l0 < k && lvl < 0; l0 += 32) {
            const int l = l0 + lane;
            unsigned u = 0;
            if (l < k) {
              const int j = W.ch[l];
              u = W.avail[l] & ~W.donated[l] & (j >= 31 ? 0u : (~0u << (j + 1)));
            }
            const unsigned has = __ballot_sync(~0u, u != 0);
            if (has) {
              const int f = __ffs(has) - 1;
              lvl = l0 + f;
              untried = __shfl_sync(~0u, u, f);
            }
          }
          if (lvl >= 0) {
            const int q = __ffs(untried) - 1;
            unsigned slot = 0;
            if (lane == 0) {
              atomicAdd(&H.pending, 1);
              slot = atomicAdd(&H.q_tail, 1u);
            }
            slot = __shfl_sync(~0u, slot, 0);
            const unsigned qi = slot % H.q_cap;
            if (lane == 0)  // the slot's previous subtree must have been read out
              while (volatile_u32(&H.b.q_ready[qi]) != 0u) {
              }
            __syncwarp();
            uint8_t* dst = H.b.q_path + static_cast<size_t>(qi) * d;
            for (int l = lane; l < lvl; l += 32) dst[l] = W.ch[l];
            if (lane == 0) {
              dst[lvl] = static_cast<uint8_t>(q);
              H.b.q_depth[qi] = static_cast<uint16_t>(lvl + 1);
            }
            __syncwarp();
            __threadfence();
            __syncwarp();
            if (lane == 0)
              *reinterpret_cast<volatile unsigned*>(&H.b.q_ready[qi]) = q_tag(pass, slot);
            W.donated[lvl] |= 1u << q;
#ifdef ORCH_HOST_DEBUG
            if (lane == 0) atomicAdd(&H.dbg_donated, 1ull);
#endif
            __syncwarp();
          }
        }
      }
      const int64_t term =
          active ? total - gained - T.og[(static_cast<size_t>(k) * nodes + lane) * (c + 1) + room]
                 : 0;
      const int64_t lb = warp_max_nonneg(term);  // egress >= 0: clamping keeps the bound valid
      bool prune;
      if (pass == 1) {
        prune = lb >= best;
      } else if (pass == 4) {
        prune = k == d || lb >= H.chain_bound[W.lo[k]];
      } else {
        prune = lb > vstar;
        if (!prune && after) {  // pass 3: only what sorts after the previous chain leaf
          const int cmp = path_cmp(W.ch, H.b.after_path, k, lane);
          prune = cmp < 0 || (cmp == 0 && k == d);
        }
      }
      if (!prune && k == d) {  // leaf: value == lb
        if (pass == 1) {
          if (lane == 0) atomicMin(&H.best_value, static_cast<unsigned long long>(lb));
          best = lb;
          prune = true;
        } else {  // a V*-leaf: keep it if it is the first in DFS order so far
          // lock-free filter first: only a leaf whose key is not above every
          // key found so far can be the first (keys tie on paths that share
          // their first km positions: those compare in full under the lock)
          const unsigned long long key = path_key(W.ch, d, kb, km, lane);
          unsigned long long least = 0;
          if (lane == 0) least = atomicMin(&H.best_key, key);
          if (key > __shfl_sync(~0u, least, 0)) break;
          if (lane == 0)
            while (atomicCAS(&H.lock, 0, 1) != 0) {
            }
          __syncwarp();
          __threadfence();
          const bool first = !__shfl_sync(~0u, lane == 0 ? volatile_i32(&H.have_best) : 0, 0) ||
                             path_cmp(W.ch, H.b.best_path, d, lane) < 0;
#ifdef ORCH_HOST_DEBUG
          if (lane == 0) atomicMax(&H.dbg_found, dbg_now());
#endif
          if (first) {
            volatile uint8_t* bp = H.b.best_path;
            for (int l = lane; l < d; l += 32) bp[l] = W.ch[l];
            if (lane == 0) *reinterpret_cast<volatile int64_t*>(&H.best_leaf) = lb;
            __threadfence();
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile int*>(&H.have_best) = 1;
          }
          __syncwarp();
          __threadfence();
          if (lane == 0) atomicExch(&H.lock, 0);
          break;  // the rest of this subtree sorts after this leaf
        }
      }
      if (prune) {
        descend = false;
      } else {
        jstart = 0;
      }
    }
    if (!descend) {  // back up one level and move to the next candidate there
      if (k == root) break;
      --k;
      const int j = W.ch[k];
      const int m = T.no[k * nodes + j];
      if (lane == m) {
        ++room;
        gained -= T.g2[k * nodes + m];
      }
      jstart = j + 1;
    }
    const unsigned av =
        __reduce_or_sync(~0u, (active && room > 0) ? (1u << T.pos[k * nodes + lane]) : 0u);
    W.avail[k] = av;
    unsigned pm = av & ~W.donated[k];
    pm = jstart >= 32 ? 0u : pm & (~0u << jstart);
    if (!pm) {
      descend = false;
      continue;
    }
    const int j = __ffs(pm) - 1;
    W.ch[k] = static_cast<uint8_t>(j);
    const int m = T.no[k * nodes + j];
    if (lane == m) {
      --room;
      gained += T.g2[k * nodes + m];
    }
    if (pass == 4) {
      int lo, hi;
      chain_step(H, k, j, W.lo[k], W.hi[k], lane, lo, hi);
      __syncwarp();
      if (lane == 0) {
        W.lo[k + 1] = static_cast<uint16_t>(lo);
        W.hi[k + 1] = static_cast<uint16_t>(hi);
      }
      __syncwarp();
    }
    ++k;
    if (k < d) W.donated[k] = 0;
    descend = true;
  }
  if (lane == 0) atomicAdd(&H.visits, visits & 65535);
  return visits;
}


// The search state after the tables are built (one thread).
__device__ void host_init_search(HostState* H, const HostBufs& b, int d, int c, int wide,
                                 unsigned q_cap, int64_t incumbent_value, int64_t root_lb) {
  const int nodes = d / c;
  H->d = d;
  H->c = c;
  H->nodes = nodes;
  H->wide = wide;
  H->q_cap = q_cap;
  H->b = b;
  H->incumbent_value = incumbent_value;
  H->best_value = static_cast<unsigned long long>(incumbent_value);
  H->visits = 0;
  H->overflow = 0;
  H->have_best = 0;
  H->best_key = ~0ull;
  int k0 = 0;
  long long tasks = 1;
  while (k0 < d && tasks * nodes <= kHostTasks) {
    tasks *= nodes;
    ++k0;
  }
  if (root_lb >= incumbent_value) tasks = 0;  // no leaf can beat the incumbents
  H->k0 = k0;
  H->tasks = tasks;
  H->task_counter = 0;
  H->q_head = H->q_tail = 0;
  H->pending = static_cast<int>(tasks);
  H->idle = 0;
  H->lock = 0;
  H->done_ctas = 0;
}

// One CTA: volume matrix, preparation, search state of both passes.
__global__ void __launch_bounds__(1024, 1) k_host_setup(int d, int c, int64_t n,
                                                        const int64_t* __restrict__ len,
                                                        const int32_t* __restrict__ origin,
                                                        const int32_t* __restrict__ dest,
                                                        const int64_t* __restrict__ Vin,
                                                        int64_t* __restrict__ Vout, HostState* H,
                                                        HostBufs b) {
  extern __shared__ __align__(16) unsigned char setup_raw[];
  Prep<kHostMaxD>& S = *reinterpret_cast<Prep<kHostMaxD>*>(setup_raw);
  const int nodes = d / c, t = threadIdx.x;
  prep_volume(S, d, n, len, origin, dest, Vin);
  if (Vout)
    for (int i = t; i < d * d; i += blockDim.x) Vout[i] = static_cast<int64_t>(S.V[i]);
  prep_run(S, d, c);
  for (int i = t; i < nodes * d; i += blockDim.x) {
    b.g2[i] = S.g2[i];
    b.no[i] = S.no[i];
    b.pos[i] = S.pos[i];
  }
  for (int i = t; i < (d + 1) * nodes * (c + 1); i += blockDim.x) b.og[i] = S.og[i];
  if (t < nodes) H->node_total[t] = S.node_total[t];
  if (t < d) {
    b.order[t] = S.order[t];
    b.incumbent[t] = S.incumbent[t];
  }
  for (int i = t; i < kHostQueue; i += blockDim.x) b.q_ready[i] = 0u;
  if (t == 0) host_init_search(H, b, d, c, 0, kHostQueue, S.incumbent_value, S.root_lb);
}

template <bool kWide>
__global__ void __launch_bounds__(kHostWarps * 32) k_host_bb(HostState* __restrict__ Hp, int pass) {
  extern __shared__ __align__(16) unsigned char host_raw[];
  HostState& H = *Hp;
  // pass 1 CTAs never leave early: the last one to finish resets the queue
  if (pass == 2 && (H.overflow || static_cast<long long>(H.best_value) >= H.incumbent_value)) return;
  if (pass == 3 && H.chain_done) return;
#ifdef ORCH_HOST_DEBUG
  if (threadIdx.x == 0) atomicMin(&H.dbg_t0, dbg_now());
#endif
  const HostSmem T = host_load_tables<kWide>(H, host_raw);
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int md = kWide ? H.d : kHostMaxD;
  unsigned char* ws;
  if constexpr (kWide)
    ws = H.b.stacks + (static_cast<size_t>(blockIdx.x) * kHostWarps + warp) * warp_stack_bytes(md);
  else
    ws = host_raw + host_table_bytes(H.d, H.c) + warp * warp_stack_bytes(md);
  unsigned* masks = reinterpret_cast<unsigned*>(ws + ((md + 3) & ~3));
  uint16_t* ranges = reinterpret_cast<uint16_t*>(masks + 2 * md);
  WarpStack W{ws, masks, masks + md, ranges, ranges + md + 1};
  const int64_t vstar = pass == 3 ? H.thresh : static_cast<int64_t>(H.best_value);
  const int c = H.c, nodes = H.nodes, k0 = H.k0;
  const int kb = nodes > 1 ? 32 - __clz(nodes - 1) : 1, km = H.d < 64 / kb ? H.d : 64 / kb;
  const bool active = lane < nodes;
  bool waiting = false;
  for (;;) {
    long long t = -1;
    long long qs = -1;
    if (lane == 0) {
      if (volatile_load(&H.task_counter) < static_cast<unsigned long long>(H.tasks)) {
        const unsigned long long x = atomicAdd(&H.task_counter, 1ull);
        if (x < static_cast<unsigned long long>(H.tasks)) t = static_cast<long long>(x);
      }
      while (t < 0) {
        if (volatile_i32(&H.overflow)) break;
        const unsigned h = volatile_u32(&H.q_head), tl = volatile_u32(&H.q_tail);
        if (h < tl) {
          if (atomicCAS(&H.q_head, h, h + 1) == h) {
            qs = h;
            break;
          }
          continue;
        }
        if (volatile_i32(&H.pending) == 0) break;  // nothing queued, nothing running: done
        if (!waiting) {
          atomicAdd(&H.idle, 1);
          waiting = true;
        }
        __nanosleep(ORCH_HOST_SLEEP);
      }
      if (waiting && (t >= 0 || qs >= 0)) {
        atomicSub(&H.idle, 1);
        waiting = false;
      }
    }
    t = __shfl_sync(~0u, t, 0);
    qs = __shfl_sync(~0u, qs, 0);
    if (t < 0 && qs < 0) break;
    int room = active ? c : 0;
    int64_t gained = 0;
    int root = 0;
    bool ok = true;
    if (t >= 0) {  // initial prefix: digit k = candidate position among nodes with room
      const int ti = static_cast<int>(t);
      int div = static_cast<int>(H.tasks) / nodes;
      int lo = 0, hi = pass == 4 ? H.chain_len : 0;
      for (int k = 0; k < k0; ++k) {
        if (pass == 4) {
          // the prefix node at depth k, entered by the reference (its ancestors
          // were not cut): counted once, by the task whose later digits are all
          // 0, then cut as the reference cuts it
          if (lane == 0 && ti % ((div > 0 ? div : 1) * nodes) == 0) atomicAdd(&H.visits, 1ull);
          const int64_t term =
              active ? H.node_total[lane] - gained -
                           T.og[(static_cast<size_t>(k) * nodes + lane) * (c + 1) + room]
                     : 0;
          if (warp_max_nonneg(term) >= H.chain_bound[lo]) {
            ok = false;
            break;
          }
        }
        const int p = (ti / (div > 0 ? div : 1)) % nodes;
        div /= nodes;
        const unsigned pm =
            __reduce_or_sync(~0u, (active && room > 0) ? (1u << T.pos[k * nodes + lane]) : 0u);
        if (__popc(pm) <= p) {
          ok = false;  // no such prefix
          break;
        }
        unsigned rest = pm;
        for (int q = 0; q < p; ++q) rest &= rest - 1;  // drop the p lowest candidates
        const int j = __ffs(rest) - 1;
        W.ch[k] = static_cast<uint8_t>(j);
        const int m = T.no[k * nodes + j];
        if (lane == m) {
          --room;
          gained += T.g2[k * nodes + m];
        }
        if (pass == 4) chain_step(H, k, j, lo, hi, lane, lo, hi);
      }
      root = k0;
    } else {  // donated subtree: wait until published, then replay its path
      const unsigned slot = static_cast<unsigned>(qs) % H.q_cap;
      const unsigned want = q_tag(pass, static_cast<unsigned>(qs));
      if (lane == 0)
        while (volatile_u32(&H.b.q_ready[slot]) != want) {
        }
      __syncwarp();
      __threadfence();
      root = *reinterpret_cast<volatile uint16_t*>(&H.b.q_depth[slot]);
      const volatile uint8_t* src = H.b.q_path + static_cast<size_t>(slot) * H.d;
      for (int k = 0; k < root; ++k) {
        const int j = src[k];
        W.ch[k] = static_cast<uint8_t>(j);
        const int m = T.no[k * nodes + j];
        if (lane == m) {
          --room;
          gained += T.g2[k * nodes + m];
        }
      }
      __syncwarp();
      __threadfence();
      if (lane == 0)  // path copied out: the slot may be reused
        *reinterpret_cast<volatile unsigned*>(&H.b.q_ready[slot]) = 0u;
    }
    __syncwarp();
    if (ok && (pass == 2 || pass == 3) &&
        path_key(W.ch, root, kb, km, lane) >
            __shfl_sync(~0u, lane == 0 ? volatile_load(&H.best_key) : 0ull, 0))
      ok = false;  // the whole subtree sorts after the best V*-leaf
#ifdef ORCH_HOST_DEBUG
    const unsigned long long ts = dbg_now();
#endif
#ifdef ORCH_HOST_DEBUG
    const unsigned long long tv = ok ? host_dfs(H, T, pass, vstar, W, root, room, gained) : 0;
    if (lane == 0) {
      atomicMax(&H.dbg_task_max, dbg_now() - ts);
      atomicMax(&H.dbg_visits_max, tv);
      if (t == 0) {
        H.dbg_first_end = dbg_now();
        H.dbg_visits0 = tv;
      }
    }
#else
    if (ok) host_dfs(H, T, pass, vstar, W, root, room, gained);
#endif
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicSub(&H.pending, 1);
    }
  }
#ifdef ORCH_HOST_DEBUG
  if (threadIdx.x == 0) atomicMax(&H.dbg_end, dbg_now());
#endif
  if (pass == 1) {  // the last CTA out resets the work distribution for pass 2
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&H.done_ctas, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      H.task_counter = 0;
      H.q_head = H.q_tail = 0;
      H.pending = static_cast<int>(H.tasks);
      H.idle = 0;
      H.lock = 0;
      H.done_ctas = 0;
      __threadfence();
    }
  }
}

// Before a pass 3 or pass 4 launch: the work distribution as after setup and a
// fresh visit budget. mode 3: the chain's first link (leaves below the
// incumbents' value); mode 5: the next link, after appending the last pass 3's
// leaf to the chain (or closing the chain: no leaf, or the budget hit), so that
// links run back to back without the host; mode 4: the counting pass (a root
// the incumbents already cut is the reference's single visit; otherwise each
// task walks its prefix nodes as the reference would: k_host_bb).
__global__ void k_host_reset(HostState* H, int mode) {
#ifdef ORCH_HOST_DEBUG
  if (!H->chain_done || mode != 5)
    printf("reset mode %d: chain %d have %d leaf %lld thresh %lld visits %llu overflow %d | "
           "found +%llu us, task0 end +%llu us, end +%llu us, longest task %llu us, donated %llu\n",
           mode, H->chain_len, H->have_best, (long long)H->best_leaf, (long long)H->thresh,
           H->visits, H->overflow, (H->dbg_found - H->dbg_t0) / 1000,
           (H->dbg_first_end - H->dbg_t0) / 1000, (H->dbg_end - H->dbg_t0) / 1000,
           H->dbg_task_max / 1000, H->dbg_donated);
  printf("   task 0 visits %llu, most visits in a task %llu\n", H->dbg_visits0, H->dbg_visits_max);
  H->dbg_visits0 = H->dbg_visits_max = 0;
  H->dbg_t0 = ~0ull;
  H->dbg_found = H->dbg_end = H->dbg_task_max = H->dbg_donated = H->dbg_first_end = 0;
#endif
  if (mode == 3) {
    H->chain_len = 0;
    // no leaf beats the incumbents (pass 1's optimum is theirs): an empty chain
    H->chain_done = static_cast<long long>(H->best_value) >= H->incumbent_value ? 1 : 0;
    H->chain_bound[0] = H->chain_last = H->incumbent_value;
    H->thresh = H->incumbent_value - 1;
    H->after_depth = 0;
  } else if (mode == 5) {
    if (H->chain_done) return;
    if (H->overflow || H->chain_len == kHostChainMax) {
      H->chain_done = 2;
      return;
    }
    if (!H->have_best) {
      H->chain_done = 1;
      return;
    }
    const int i = H->chain_len, d = H->d;
    for (int l = 0; l < d; ++l)
      H->b.chain_path[static_cast<size_t>(i) * d + l] = H->b.after_path[l] = H->b.best_path[l];
    H->chain_bound[i + 1] = H->chain_last = H->best_leaf;
    H->chain_len = i + 1;
    // a link at pass 1's optimum is the last: nothing after it can be lower
    if (static_cast<unsigned long long>(H->best_leaf) == H->best_value) H->chain_done = 1;
    H->thresh = H->best_leaf - 1;
    H->after_depth = d;
  }
  H->task_counter = 0;
  H->q_head = H->q_tail = 0;
  H->idle = 0;
  H->lock = 0;
  H->done_ctas = 0;
  H->have_best = 0;
  H->best_key = ~0ull;
  H->overflow = 0;
  H->visits = 0;
  if (mode == 4 && H->tasks == 0) H->visits = 1;  // the incumbents cut the root
  H->pending = static_cast<int>(H->tasks);
}

// Final hosting, batch -> instance map (topology.cpp:283-290), egress figures;
// with a balance result, its relabelling (batch b becomes instance b2i[b]).
constexpr int kFinMaxItems = 10240;  // destination CSR members kept in shared memory (static, < 48 KB)
struct FinSmem {
  unsigned long long e[kHostMaxNodes], e0[kHostMaxNodes];
  int32_t a[kHostMaxD], b2i[kHostMaxD], inv[kHostMaxD], noff[kHostMaxD + 1];
  int32_t ocnt[kHostMaxD], ooff[kHostMaxD + 1];
  int64_t olen[kHostMaxD], otok[kHostMaxD];
  double ocost[kHostMaxD];
  int32_t members[kFinMaxItems];
};

struct RemapArgs {
  int64_t n;
  int32_t* dest_inst;
  int32_t* bin_count;
  int64_t* bin_len;
  int64_t* bin_tokens;
  double* bin_cost;
  int32_t* bin_offset;
  int32_t* bin_member;
  int32_t* scratch;  // n members when n > kFinMaxItems
};

__global__ void __launch_bounds__(1024, 1) k_host_finish(const HostState* __restrict__ Hp,
                                                         const int64_t* __restrict__ V,
                                                         int32_t* __restrict__ hosting,
                                                         int32_t* __restrict__ b2i_out,
                                                         int64_t* __restrict__ info, RemapArgs r) {
  __shared__ FinSmem F;
  const HostState& H = *Hp;
  const int d = H.d, c = H.c, nodes = H.nodes, t = threadIdx.x;
  const bool incumbent = static_cast<long long>(H.best_value) >= H.incumbent_value || H.overflow ||
                         !H.have_best;
  const bool remap = r.dest_inst != nullptr;
  int32_t* mem = r.n > kFinMaxItems ? r.scratch : F.members;
  if (remap) {  // the old per-batch arrays and CSR, before anything is overwritten
    if (t < d) {
      F.ocnt[t] = r.bin_count[t];
      if (r.bin_len) F.olen[t] = r.bin_len[t];
      if (r.bin_tokens) F.otok[t] = r.bin_tokens[t];
      if (r.bin_cost) F.ocost[t] = r.bin_cost[t];
    }
    if (t <= d) F.ooff[t] = r.bin_offset[t];
    for (int64_t i = t; i < r.n; i += blockDim.x) mem[i] = r.bin_member[i];
  }
  if (t < d) F.a[t] = H.b.incumbent[t];
  if (t < nodes) F.e[t] = F.e0[t] = 0;
  __syncthreads();
  if (!incumbent && t < d) F.a[H.b.order[t]] = H.b.no[t * nodes + H.b.best_path[t]];
  __syncthreads();
  if (t == 0) {
    int next[kHostMaxNodes];
    for (int nd = 0; nd < nodes; ++nd) next[nd] = nd * c;
    for (int b = 0; b < d; ++b) {
      const int nb = next[F.a[b]]++;
      F.b2i[b] = nb;
      F.inv[nb] = b;
    }
  }
  for (int i = t; i < d * d; i += blockDim.x) {  // inter_node_egress of the solution and identity
    const int src = i / d, b = i % d, nd = src / c;
    const unsigned long long v = static_cast<unsigned long long>(V[i]);
    if (v) {
      if (F.a[b] != nd) atomicAdd(&F.e[nd], v);
      if (b / c != nd) atomicAdd(&F.e0[nd], v);
    }
  }
  __syncthreads();
  if (t < d) {
    hosting[t] = F.a[t];
    b2i_out[t] = F.b2i[t];
  }
  if (t == 0) {
    unsigned long long worst = 0, base = 0;
    for (int nd = 0; nd < nodes; ++nd) {
      worst = F.e[nd] > worst ? F.e[nd] : worst;
      base = F.e0[nd] > base ? F.e0[nd] : base;
    }
    info[0] = static_cast<int64_t>(worst);
    info[1] = static_cast<int64_t>(base);
    info[2] = H.overflow ? -1 : (incumbent ? 0 : 1);  // -1: visit budget hit, incumbent kept
    info[3] = static_cast<int64_t>(H.visits);
    if (remap) {
      int acc = 0;
      for (int j = 0; j < d; ++j) {
        F.noff[j] = acc;
        acc += F.ocnt[F.inv[j]];
      }
      F.noff[d] = acc;
    }
  }
#ifdef ORCH_HOST_DEBUG
  if (t == 0)
    printf("hosting: best %llu inc %lld visits %llu overflow %d k0 %d tasks %lld queued %u\n",
           H.best_value, (long long)H.incumbent_value, H.visits, H.overflow, H.k0, H.tasks, H.q_tail);
#endif
  if (!remap) return;
  __syncthreads();
  if (t < d) {
    const int b = F.inv[t];
    r.bin_count[t] = F.ocnt[b];
    if (r.bin_len) r.bin_len[t] = F.olen[b];
    if (r.bin_tokens) r.bin_tokens[t] = F.otok[b];
    if (r.bin_cost) r.bin_cost[t] = F.ocost[b];
  }
  if (t <= d) r.bin_offset[t] = F.noff[t];
  for (int j = 0; j < d; ++j) {
    const int b = F.inv[j];
    const int cnt = F.ooff[b + 1] - F.ooff[b];
    for (int k = t; k < cnt; k += blockDim.x) r.bin_member[F.noff[j] + k] = mem[F.ooff[b] + k];
  }
  for (int64_t i = t; i < r.n; i += blockDim.x) r.dest_inst[i] = F.b2i[r.dest_inst[i]];
}

// ------------------------------------------------ one-CTA node-wise path
// For small searches (d <= 32, <= 2^18 leaves, n <= 12288: every C2 shape on
// 2/4/8 GPUs) the whole of orch_nodewise is ONE kernel in shared memory:
// volume matrix -> preparation -> two-pass branch and bound (32 warps, lane =
// node, prefix tasks claimed in DFS order) -> hosting, batch_to_instance,
// egress figures -> relabelling of the balance result. Same answer as the
// multi-CTA path (first optimal leaf in DFS order, else the incumbents).
constexpr int kNwThreads = 1024;
constexpr int kNwWarps = kNwThreads / 32;
constexpr int kNwMaxD = 32;
constexpr int kNwMaxItems = 12288;
constexpr int kNwTasks = 64;  // at least two prefix tasks per warp
constexpr double kNwMaxLeaves = 262144.0;

struct NwSmem {
  Prep<kNwMaxD> p;
  int64_t node_e[kNwMaxD], node_e0[kNwMaxD];
  unsigned long long best;  // pass 1: best value so far
  unsigned long long visits;
  int tasks, k0, best_task, lock;
  unsigned task_ctr;
  int32_t a[kNwMaxD], b2i[kNwMaxD], inv[kNwMaxD], noff[kNwMaxD + 1];
  int32_t ocnt[kNwMaxD], ooff[kNwMaxD + 1];
  int64_t olen[kNwMaxD], otok[kNwMaxD];
  double ocost[kNwMaxD];
  uint8_t ch[kNwWarps][kNwMaxD];  // per-warp DFS path (candidate positions)
  uint8_t best_path[kNwMaxD];
  int32_t members[kNwMaxItems];
};

struct NwArgs {
  int d, c, n;
  const int64_t* len;
  const int32_t* origin;
  int32_t* dest_inst;
  int32_t* bin_count;
  int64_t* bin_len;
  int64_t* bin_tokens;
  double* bin_cost;
  int32_t* bin_offset;
  int32_t* bin_member;
  int32_t* hosting;
  int32_t* b2i;
  int64_t* info;
};

// DFS of the subtree below ch[0, root) for one warp (lane = node): the
// prune rules and visiting order of host_dfs, without donation.
__device__ void nw_dfs(NwSmem& S, int pass, int64_t vstar, int task, int root, int room,
                       int64_t gained, int d, int c, int nodes, uint8_t* ch) {
  const Prep<kNwMaxD>& T = S.p;
  const int lane = threadIdx.x & 31;
  const bool active = lane < nodes;
  const int64_t total = active ? T.node_total[lane] : 0;
  unsigned long long visits = 0;
  int k = root, jstart = 0;
  bool descend = true;
  for (;;) {
    if (descend) {
      ++visits;
      if (pass == 2 &&
          __shfl_sync(~0u, lane == 0 ? *reinterpret_cast<volatile int*>(&S.best_task) : 0, 0) < task)
        break;  // an earlier task already holds a V*-leaf
      const int64_t term =
          active ? total - gained - T.og[(static_cast<size_t>(k) * nodes + lane) * (c + 1) + room] : 0;
      const int64_t lb = warp_max_nonneg(term);
      bool prune;
      if (pass == 1) {
        const int64_t best = static_cast<int64_t>(__shfl_sync(
            ~0u, lane == 0 ? *reinterpret_cast<volatile unsigned long long*>(&S.best) : 0ull, 0));
        prune = lb >= best;
      } else {
        prune = lb > vstar;
      }
      if (!prune && k == d) {  // leaf: value == lb
        if (pass == 1) {
          if (lane == 0) atomicMin(&S.best, static_cast<unsigned long long>(lb));
          prune = true;
        } else {  // the first V*-leaf of this task in DFS order
          if (lane == 0)
            while (atomicCAS(&S.lock, 0, 1) != 0) {
            }
          __syncwarp();
          __threadfence_block();
          const int won = __shfl_sync(
              ~0u, lane == 0 ? (task < *reinterpret_cast<volatile int*>(&S.best_task)) : 0, 0);
          if (won) {
            for (int l = lane; l < d; l += 32) S.best_path[l] = ch[l];
            __threadfence_block();
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile int*>(&S.best_task) = task;
          }
          __syncwarp();
          __threadfence_block();
          if (lane == 0) atomicExch(&S.lock, 0);
          break;
        }
      }
      if (prune) {
        descend = false;
      } else {
        jstart = 0;
      }
    }
    if (!descend) {
      if (k == root) break;
      --k;
      const int j = ch[k];
      const int m = T.no[k * nodes + j];
      if (lane == m) {
        ++room;
        gained -= T.g2[k * nodes + m];
      }
      jstart = j + 1;
    }
    const unsigned av =
        __reduce_or_sync(~0u, (active && room > 0) ? (1u << T.pos[k * nodes + lane]) : 0u);
    const unsigned pm = jstart >= 32 ? 0u : av & (~0u << jstart);
    if (!pm) {
      descend = false;
      continue;
    }
    const int j = __ffs(pm) - 1;
    __syncwarp();
    if (lane == 0) ch[k] = static_cast<uint8_t>(j);
    __syncwarp();
    const int m = T.no[k * nodes + j];
    if (lane == m) {
      --room;
      gained += T.g2[k * nodes + m];
    }
    ++k;
    descend = true;
  }
  if (lane == 0) atomicAdd(&S.visits, visits);
}

// one pass over the prefix tasks, claimed in DFS order
__device__ void nw_pass(NwSmem& S, int pass, int64_t vstar, int d, int c, int nodes) {
  const Prep<kNwMaxD>& T = S.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = lane < nodes;
  uint8_t* ch = S.ch[warp];
  for (;;) {
    int t = 0;
    if (lane == 0) t = static_cast<int>(atomicAdd(&S.task_ctr, 1u));
    t = __shfl_sync(~0u, t, 0);
    if (t >= S.tasks) break;
    if (pass == 2 &&
        __shfl_sync(~0u, lane == 0 ? *reinterpret_cast<volatile int*>(&S.best_task) : 0, 0) < t)
      break;  // the remaining tasks sort after the best leaf
    int room = active ? c : 0;
    int64_t gained = 0;
    bool ok = true;
    int div = S.tasks / nodes;
    for (int k = 0; k < S.k0; ++k) {
      const int p = (t / (div > 0 ? div : 1)) % nodes;
      div /= nodes;
      const unsigned pm =
          __reduce_or_sync(~0u, (active && room > 0) ? (1u << T.pos[k * nodes + lane]) : 0u);
      if (__popc(pm) <= p) {
        ok = false;
        break;
      }
      unsigned rest = pm;
      for (int q = 0; q < p; ++q) rest &= rest - 1;
      const int j = __ffs(rest) - 1;
      __syncwarp();
      if (lane == 0) ch[k] = static_cast<uint8_t>(j);
      __syncwarp();
      const int m = T.no[k * nodes + j];
      if (lane == m) {
        --room;
        gained += T.g2[k * nodes + m];
      }
    }
    if (ok) nw_dfs(S, pass, vstar, t, S.k0, room, gained, d, c, nodes, ch);
  }
}

__global__ void __launch_bounds__(kNwThreads, 1) k_nodewise_small(NwArgs a) {
  extern __shared__ __align__(16) unsigned char nw_raw[];
  NwSmem& S = *reinterpret_cast<NwSmem*>(nw_raw);
  Prep<kNwMaxD>& T = S.p;
  const int d = a.d, c = a.c, nodes = d / c, n = a.n, t = threadIdx.x;
  // the old per-batch arrays and CSR, before anything is overwritten
  if (t < d) {
    S.ocnt[t] = a.bin_count[t];
    if (a.bin_len) S.olen[t] = a.bin_len[t];
    if (a.bin_tokens) S.otok[t] = a.bin_tokens[t];
    if (a.bin_cost) S.ocost[t] = a.bin_cost[t];
  }
  if (t <= d) S.ooff[t] = a.bin_offset[t];
  for (int i = t; i < n; i += kNwThreads) S.members[i] = a.bin_member[i];
  if (t == 0) {
    S.visits = 0;
    S.task_ctr = 0;
    S.best_task = INT_MAX;
    S.lock = 0;
  }
  prep_volume(T, d, n, a.len, a.origin, a.dest_inst, nullptr);
  prep_run(T, d, c);
  if (t == 0) {
    S.best = static_cast<unsigned long long>(T.incumbent_value);
    int k0 = 0, tasks = 1;  // a few prefix tasks per warp: these trees are small
    while (k0 < d && tasks < kNwTasks) {
      tasks *= nodes;
      ++k0;
    }
    S.k0 = k0;
    S.tasks = T.root_lb >= T.incumbent_value ? 0 : tasks;  // no leaf can beat the incumbents
  }
  __syncthreads();
  // ---- search: pass 1 finds V*, pass 2 the first V*-leaf in DFS order
  nw_pass(S, 1, 0, d, c, nodes);
  __syncthreads();
  const int64_t vstar = static_cast<int64_t>(S.best);
  const bool search2 = vstar < T.incumbent_value;
  if (t == 0) S.task_ctr = 0;
  __syncthreads();
  if (search2) nw_pass(S, 2, vstar, d, c, nodes);
  __syncthreads();
  // ---- hosting, batch -> instance (topology.cpp:283-290), egress figures
  const bool incumbent = !search2 || S.best_task == INT_MAX;
  if (t < d) S.a[t] = T.incumbent[t];
  __syncthreads();
  if (!incumbent && t < d) S.a[T.order[t]] = T.no[t * nodes + S.best_path[t]];
  __syncthreads();
  if (t == 0) {
    int next[kNwMaxD];
    for (int nd = 0; nd < nodes; ++nd) next[nd] = nd * c;
    for (int b = 0; b < d; ++b) {
      const int nb = next[S.a[b]]++;
      S.b2i[b] = nb;
      S.inv[nb] = b;
    }
  }
  __syncthreads();
  if (t < nodes) {
    int64_t e = 0, e0 = 0;
    for (int i = t * c; i < (t + 1) * c; ++i)
      for (int b = 0; b < d; ++b) {
        const int64_t v = static_cast<int64_t>(T.V[i * d + b]);
        if (S.a[b] != t) e += v;
        if (b / c != t) e0 += v;
      }
    S.node_e[t] = e;
    S.node_e0[t] = e0;
  }
  if (t < d) {
    a.hosting[t] = S.a[t];
    a.b2i[t] = S.b2i[t];
  }
  if (t == 0) {
    int acc = 0;
    for (int j = 0; j < d; ++j) {
      S.noff[j] = acc;
      acc += S.ocnt[S.inv[j]];
    }
    S.noff[d] = acc;
  }
  __syncthreads();
  if (t == 0 && a.info) {
    int64_t worst = 0, base = 0;
    for (int nd = 0; nd < nodes; ++nd) {
      worst = S.node_e[nd] > worst ? S.node_e[nd] : worst;
      base = S.node_e0[nd] > base ? S.node_e0[nd] : base;
    }
    a.info[0] = worst;
    a.info[1] = base;
    a.info[2] = incumbent ? 0 : 1;
    a.info[3] = static_cast<int64_t>(S.visits);
  }
  // ---- relabel the balance result: batch b becomes instance b2i[b]
  if (t < d) {
    const int b = S.inv[t];
    a.bin_count[t] = S.ocnt[b];
    if (a.bin_len) a.bin_len[t] = S.olen[b];
    if (a.bin_tokens) a.bin_tokens[t] = S.otok[b];
    if (a.bin_cost) a.bin_cost[t] = S.ocost[b];
  }
  if (t <= d) a.bin_offset[t] = S.noff[t];
  for (int j = 0; j < d; ++j) {
    const int b = S.inv[j];
    const int cnt = S.ooff[b + 1] - S.ooff[b];
    for (int k = t; k < cnt; k += kNwThreads) a.bin_member[S.noff[j] + k] = S.members[S.ooff[b] + k];
  }
  for (int i = t; i < n; i += kNwThreads) a.dest_inst[i] = S.b2i[a.dest_inst[i]];
}

bool nodewise_small_fits(int d, int c, int64_t n) {
  const int nodes = d / c;
  if (d > kNwMaxD || nodes > kNwMaxD || n > kNwMaxItems) return false;
  double leaves = 1.0;  // d! / (c!)^nodes
  for (int i = 2; i <= d; ++i) leaves *= i;
  double cf = 1.0;
  for (int i = 2; i <= c; ++i) cf *= i;
  for (int nd = 0; nd < nodes; ++nd) leaves /= cf;
  return leaves <= kNwMaxLeaves;
}

// ------------------------------------------------- wide setup and finish
// d > kHostMaxD (up to ORCH_MAX_INSTANCES, e.g. C4's 2560): the same tables as
// prep_run, built by grid-wide kernels in global memory (V alone is d^2 words),
// for orch_solve_hosting_host. Scratch per call:
struct WideScratch {
  int64_t* gain;           // [node][batch]
  int64_t* regret;         // [batch]
  int32_t* at;             // [batch] position in the branching order
  int32_t* srt_at;         // [node][rank]: order position of the node's rank-th largest gain
  int64_t* srt_g;          // [node][rank]: that gain
  int32_t* greedy;         // [batch]
  unsigned long long* sub; // [4][nodes]: identity, greedy gains kept; solution, identity egress
  int32_t* a;              // [batch] final node
};

__global__ void k_hw_gain(const int64_t* __restrict__ V, int d, int c, int64_t* __restrict__ gain) {
  const int nodes = d / c;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<int64_t>(nodes) * d; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int nd = static_cast<int>(i / d), b = static_cast<int>(i % d);
    int64_t g = 0;
    for (int r = nd * c; r < (nd + 1) * c; ++r) g += V[static_cast<size_t>(r) * d + b];
    gain[i] = g;
  }
}

// regret per batch (top - second gain over the nodes); node totals (block 0)
__global__ void k_hw_regret(const int64_t* __restrict__ gain, int d, int nodes,
                            int64_t* __restrict__ regret, HostState* H) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < d) {
    int64_t top = 0, second = 0;
    for (int nd = 0; nd < nodes; ++nd) {
      const int64_t g = gain[static_cast<size_t>(nd) * d + b];
      if (g > top) {
        second = top;
        top = g;
      } else if (g > second) {
        second = g;
      }
    }
    regret[b] = top - second;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // node totals: one warp per node, in turn
    for (int nd = 0; nd < nodes; ++nd) {
      int64_t t = 0;
      for (int x = threadIdx.x; x < d; x += 32) t += gain[static_cast<size_t>(nd) * d + x];
#pragma unroll
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
      if (threadIdx.x == 0) H->node_total[nd] = t;
    }
  }
}

// stable order by descending regret (topology.cpp:212-228): rank by counting
__global__ void k_hw_order(const int64_t* __restrict__ regret, int d, int32_t* __restrict__ order,
                           int32_t* __restrict__ at) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d) return;
  const int64_t mine = regret[b];
  int r = 0;
  for (int x = 0; x < d; ++x) {
    const int64_t o = regret[x];
    r += o > mine || (o == mine && x < b);
  }
  order[r] = b;
  at[b] = r;
}

// per depth k: candidate nodes by descending gain for order[k], ties by node
__global__ void k_hw_tables(const int64_t* __restrict__ gain, const int32_t* __restrict__ order,
                            int d, int nodes, int64_t* __restrict__ g2, uint8_t* __restrict__ no,
                            uint8_t* __restrict__ pos) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
  const int b = order[k];
  int64_t g[kHostMaxNodes];
  uint8_t srt[kHostMaxNodes];
  for (int nd = 0; nd < nodes; ++nd) {
    g[nd] = gain[static_cast<size_t>(nd) * d + b];
    g2[static_cast<size_t>(k) * nodes + nd] = g[nd];
    int j = nd - 1;
    while (j >= 0 && g[srt[j]] < g[nd]) {
      srt[j + 1] = srt[j];
      --j;
    }
    srt[j + 1] = static_cast<uint8_t>(nd);
  }
  for (int j = 0; j < nodes; ++j) {
    no[static_cast<size_t>(k) * nodes + j] = srt[j];
    pos[static_cast<size_t>(k) * nodes + srt[j]] = static_cast<uint8_t>(j);
  }
}

// per node: its gains in descending order (ties by batch) with their order positions
__global__ void k_hw_sorted(const int64_t* __restrict__ gain, const int32_t* __restrict__ at, int d,
                            int nodes, int32_t* __restrict__ srt_at, int64_t* __restrict__ srt_g) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<int64_t>(nodes) * d; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int nd = static_cast<int>(i / d), b = static_cast<int>(i % d);
    const int64_t* row = gain + static_cast<size_t>(nd) * d;
    const int64_t mine = row[b];
    int r = 0;
    for (int x = 0; x < d; ++x) r += row[x] > mine || (row[x] == mine && x < b);
    srt_at[static_cast<size_t>(nd) * d + r] = at[b];
    srt_g[static_cast<size_t>(nd) * d + r] = mine;
  }
}

// og[k][node][r]: the node's r largest gains among order[k..d) (r <= c)
__global__ void k_hw_og(const int32_t* __restrict__ srt_at, const int64_t* __restrict__ srt_g, int d,
                        int nodes, int c, int64_t* __restrict__ og) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<int64_t>(nodes) * (d + 1); i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int nd = static_cast<int>(i / (d + 1)), k = static_cast<int>(i % (d + 1));
    int64_t* out = og + (static_cast<size_t>(k) * nodes + nd) * (c + 1);
    const int32_t* sa = srt_at + static_cast<size_t>(nd) * d;
    const int64_t* sg = srt_g + static_cast<size_t>(nd) * d;
    int64_t acc = 0;
    int r = 0;
    out[0] = 0;
    for (int x = 0; x < d && r < c; ++x)
      if (sa[x] >= k) {
        acc += sg[x];
        out[++r] = acc;
      }
    while (r < c) out[++r] = acc;
  }
}

// greedy incumbent (topology.cpp:238-254), one warp: the gains of 32 depths at
// a time staged in shared memory, then the sequential picks
__global__ void k_hw_greedy(const int64_t* __restrict__ g2, const int32_t* __restrict__ order, int d,
                            int nodes, int c, int32_t* __restrict__ greedy) {
  __shared__ int64_t tile[32 * kHostMaxNodes];
  const int lane = threadIdx.x;
  int room = lane < nodes ? c : 0;
  for (int k0 = 0; k0 < d; k0 += 32) {
    const int kn = d - k0 < 32 ? d - k0 : 32;
    for (int i = lane; i < kn * nodes; i += 32) tile[i] = g2[static_cast<size_t>(k0) * nodes + i];
    __syncwarp();
    for (int k = 0; k < kn; ++k) {
      const int pick = warp_argmax_first(room > 0 ? tile[k * nodes + lane] : -1);
      if (lane == pick) {
        --room;
        greedy[order[k0 + k]] = pick;
      }
    }
    __syncwarp();
  }
}

// kept gains of the identity (sub[0]) and greedy (sub[1]) hostings
__global__ void k_hw_values(const int64_t* __restrict__ gain, const int32_t* __restrict__ greedy,
                            int d, int c, unsigned long long* __restrict__ sub) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d) return;
  const int nodes = d / c, ni = b / c, ng = greedy[b];
  atomicAdd(&sub[ni], static_cast<unsigned long long>(gain[static_cast<size_t>(ni) * d + b]));
  atomicAdd(&sub[nodes + ng], static_cast<unsigned long long>(gain[static_cast<size_t>(ng) * d + b]));
}

// incumbent values, the bound at the root, the search state (one thread)
__global__ void k_hw_init(HostState* H, HostBufs b, int d, int c,
                          const unsigned long long* __restrict__ sub, int* __restrict__ g_better) {
  const int nodes = d / c;
  int64_t vi = INT64_MIN, vg = INT64_MIN, root = 0;
  for (int nd = 0; nd < nodes; ++nd) {
    const int64_t t = H->node_total[nd];
    const int64_t ei = t - static_cast<int64_t>(sub[nd]), eg = t - static_cast<int64_t>(sub[nodes + nd]);
    vi = ei > vi ? ei : vi;
    vg = eg > vg ? eg : vg;
    const int64_t e = t - b.og[static_cast<size_t>(nd) * (c + 1) + c];
    root = e > root ? e : root;
  }
  *g_better = vg < vi;  // offer(greedy) replaces only when strictly better
  host_init_search(H, b, d, c, 1, kHostQueueWide, vg < vi ? vg : vi, root);
}

__global__ void k_hw_incumbent(const int32_t* __restrict__ greedy, const int* __restrict__ g_better,
                               int d, int c, int32_t* __restrict__ incumbent,
                               unsigned* __restrict__ q_ready) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) incumbent[i] = *g_better ? greedy[i] : i / c;
  if (i < kHostQueueWide) q_ready[i] = 0u;
}

// final hosting and batch -> instance map (topology.cpp:283-290), one CTA
__global__ void k_hw_assign(const HostState* __restrict__ Hp, int32_t* __restrict__ a,
                            int32_t* __restrict__ hosting, int32_t* __restrict__ b2i,
                            unsigned long long* __restrict__ e) {
  const HostState& H = *Hp;
  const int d = H.d, c = H.c, nodes = H.nodes;
  const bool incumbent = static_cast<long long>(H.best_value) >= H.incumbent_value || H.overflow ||
                         !H.have_best;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    const int v = incumbent ? H.b.incumbent[t]
                            : H.b.no[static_cast<size_t>(t) * nodes + H.b.best_path[t]];
    a[incumbent ? t : H.b.order[t]] = v;
  }
  if (threadIdx.x < 2 * nodes) e[threadIdx.x] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < d; t += blockDim.x) hosting[t] = a[t];
  if (threadIdx.x == 0) {
    int next[kHostMaxNodes];
    for (int nd = 0; nd < nodes; ++nd) next[nd] = nd * c;
    for (int x = 0; x < d; ++x) b2i[x] = next[a[x]]++;
  }
}

// inter_node_egress of the solution (e[0..nodes)) and of the identity (e[nodes..))
__global__ void k_hw_egress(const int64_t* __restrict__ V, const int32_t* __restrict__ a, int d,
                            int c, unsigned long long* __restrict__ e) {
  const int nodes = d / c;
  __shared__ unsigned long long acc[2 * kHostMaxNodes];
  if (threadIdx.x < 2 * kHostMaxNodes) acc[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<int64_t>(d) * d; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int src = static_cast<int>(i / d), b = static_cast<int>(i % d), nd = src / c;
    const unsigned long long v = static_cast<unsigned long long>(V[i]);
    if (v) {
      if (a[b] != nd) atomicAdd(&acc[nd], v);
      if (b / c != nd) atomicAdd(&acc[nodes + nd], v);
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * nodes && acc[threadIdx.x]) atomicAdd(&e[threadIdx.x], acc[threadIdx.x]);
}

__global__ void k_hw_info(const HostState* __restrict__ Hp, const unsigned long long* __restrict__ e,
                          int64_t* __restrict__ info) {
  const HostState& H = *Hp;
  const int nodes = H.nodes;
  const bool incumbent = static_cast<long long>(H.best_value) >= H.incumbent_value || H.overflow ||
                         !H.have_best;
  unsigned long long worst = 0, base = 0;
  for (int nd = 0; nd < nodes; ++nd) {
    worst = e[nd] > worst ? e[nd] : worst;
    base = e[nodes + nd] > base ? e[nodes + nd] : base;
  }
  info[0] = static_cast<int64_t>(worst);
  info[1] = static_cast<int64_t>(base);
  info[2] = H.overflow ? -1 : (incumbent ? 0 : 1);
  info[3] = static_cast<int64_t>(H.visits);
}

// inter_node_egress of one hosting for any node count: per-CTA node totals in
// shared memory, one atomic per node and CTA
__global__ void k_node_egress(const int64_t* __restrict__ V, const int32_t* __restrict__ hosting,
                              int d, int c, unsigned long long* __restrict__ e) {
  extern __shared__ unsigned long long eg_acc[];
  const int nodes = d / c;
  for (int i = threadIdx.x; i < nodes; i += blockDim.x) eg_acc[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<int64_t>(d) * d; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int src = static_cast<int>(i / d), b = static_cast<int>(i % d), nd = src / c;
    const int64_t v = V[i];
    if (v && hosting[b] != nd) atomicAdd(&eg_acc[nd], static_cast<unsigned long long>(v));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nodes; i += blockDim.x)
    if (eg_acc[i]) atomicAdd(&e[i], eg_acc[i]);
}

// setup, both passes and the finish of the wide search; V on the device
int run_wide_hosting(orch_ctx* ctx, int d, int c, const int64_t* V, HostState* H, const HostBufs& hb,
                     const WideScratch& w, int32_t* hosting, int32_t* b2i, int64_t* info,
                     int* g_better, cudaStream_t st) {
  const int nodes = d / c, T = 256;
  const int nb = (d + T - 1) / T;
  const int grid = kSMs * 8;
  ORCH_CUDA_TRY(cudaMemsetAsync(w.sub, 0, sizeof(unsigned long long) * 4 * kHostMaxNodes, st));
  k_hw_gain<<<grid, T, 0, st>>>(V, d, c, w.gain);
  k_hw_regret<<<nb, T, 0, st>>>(w.gain, d, nodes, w.regret, H);
  k_hw_order<<<nb, T, 0, st>>>(w.regret, d, hb.order, w.at);
  k_hw_tables<<<nb, T, 0, st>>>(w.gain, hb.order, d, nodes, hb.g2, hb.no, hb.pos);
  k_hw_sorted<<<grid, T, 0, st>>>(w.gain, w.at, d, nodes, w.srt_at, w.srt_g);
  k_hw_og<<<grid, T, 0, st>>>(w.srt_at, w.srt_g, d, nodes, c, hb.og);
  k_hw_greedy<<<1, 32, 0, st>>>(hb.g2, hb.order, d, nodes, c, w.greedy);
  k_hw_values<<<nb, T, 0, st>>>(w.gain, w.greedy, d, c, w.sub);
  k_hw_init<<<1, 1, 0, st>>>(H, hb, d, c, w.sub, g_better);
  k_hw_incumbent<<<(kHostQueueWide > d ? kHostQueueWide + T - 1 : d + T - 1) / T, T, 0, st>>>(
      w.greedy, g_better, d, c, hb.incumbent, hb.q_ready);
  k_host_bb<true><<<kHostGrid, kHostWarps * 32, 0, st>>>(H, 1);
  k_host_bb<true><<<kHostGrid, kHostWarps * 32, 0, st>>>(H, 2);
  k_hw_assign<<<1, 1024, 0, st>>>(H, w.a, hosting, b2i, w.sub + 2 * kHostMaxNodes);
  k_hw_egress<<<grid, T, 0, st>>>(V, w.a, d, c, w.sub + 2 * kHostMaxNodes);
  k_hw_info<<<1, 1, 0, st>>>(H, w.sub + 2 * kHostMaxNodes, info);
  ctx->launches += 15;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

// max_d: kHostMaxD for orch_nodewise (its finish remaps the balance in shared
// memory), ORCH_MAX_INSTANCES for orch_solve_hosting_host
int check_hosting_args(int d, int c, int max_d = kHostMaxD) {
  if (d < 1 || c < 1)
    return fail(ORCH_INVALID_ARGUMENT, "topology needs at least one instance and one per node");
  if (d % c) return fail(ORCH_INVALID_ARGUMENT, "instance count must be divisible by instances per node");
  if (d > max_d)
    return fail(ORCH_UNSUPPORTED, max_d == kHostMaxD
                                      ? "orch_nodewise limited to d <= 64 on the device"
                                      : "node-wise hosting limited to d <= 4096 on the device");
  if (d / c > kHostMaxNodes)
    return fail(ORCH_UNSUPPORTED, "node-wise hosting limited to 32 nodes on the device");
  return ORCH_OK;
}

// the search state and its per-call buffers (tables, paths, queue; wide: stacks)
void plan_host_search(Plan& p, int d, int c, HostState** H, HostBufs* b) {
  const size_t nodes = static_cast<size_t>(d / c), dd = static_cast<size_t>(d);
  const bool wide = d > kHostMaxD;
  const size_t q_cap = wide ? kHostQueueWide : kHostQueue;
  p.add(H, 1);
  p.add(&b->order, dd);
  p.add(&b->incumbent, dd);
  p.add(&b->g2, dd * nodes);
  p.add(&b->no, dd * nodes);
  p.add(&b->pos, dd * nodes);
  p.add(&b->og, (dd + 1) * nodes * static_cast<size_t>(c + 1));
  p.add(&b->best_path, dd);
  p.add(&b->after_path, dd);
  p.add(&b->chain_path, static_cast<size_t>(kHostChainMax) * dd);
  p.add(&b->q_ready, q_cap);
  p.add(&b->q_depth, q_cap);
  p.add(&b->q_path, q_cap * dd);
  b->stacks = nullptr;
  if (wide) p.add(&b->stacks, static_cast<size_t>(kHostGrid) * kHostWarps * warp_stack_bytes(d));
}

// setup + both passes of the multi-CTA search (V from the items, or given)
int launch_hosting_search(orch_ctx* ctx, int d, int c, int64_t n, const int64_t* len,
                          const int32_t* origin, const int32_t* dest, const int64_t* Vin,
                          int64_t* Vout, HostState* H, const HostBufs& b, cudaStream_t st) {
  const int sm = static_cast<int>(host_smem_bytes(d, c));
  static PerDeviceOnce configured;
  const int rc_attr = configured([&]() -> int {
    const int mx = static_cast<int>(host_smem_bytes(kHostMaxD, 2));  // the largest table set
    ORCH_CUDA_TRY(cudaFuncSetAttribute(k_host_bb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    ORCH_CUDA_TRY(cudaFuncSetAttribute(k_host_setup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(Prep<kHostMaxD>))));
    ORCH_CUDA_TRY(max_carveout(k_host_bb<false>));
    ORCH_CUDA_TRY(max_carveout(k_host_setup));
    return ORCH_OK;
  });
  if (rc_attr) return rc_attr;
  k_host_setup<<<1, 1024, sizeof(Prep<kHostMaxD>), st>>>(d, c, n, len, origin, dest, Vin, Vout, H,
                                                          b);
  k_host_bb<false><<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 1);
  k_host_bb<false><<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 2);
  ctx->launches += 3;
  return ORCH_OK;
}

// The reference's nodes_visited (topology.cpp:150-151, 263). Its sequential DFS
// enters a node iff the parent was not cut by lb >= the incumbent it held at
// that moment, and that incumbent changes only at its chain of strictly
// improving leaves: each the first leaf in DFS order after the previous one
// whose value is below it, starting from the incumbents' value. The chain is
// found link by link (pass 3, launched in batches that the device chains
// itself), then one pass replays the reference's cuts node by node and counts
// (pass 4). Runs after the hosting search (its pass 1/2 state is consumed).
// *visits = -1 when a pass exceeds the visit budget or the chain kHostChainMax
// links.
int reference_visits(orch_ctx* ctx, HostState* H, int d, int c, cudaStream_t st, int64_t* visits) {
  const int sm = static_cast<int>(host_smem_bytes(d, c));
  auto* bb = d > kHostMaxD ? k_host_bb<true> : k_host_bb<false>;
  int links = 2;  // links launched per host check: 2, 4, 8, 8, ...
  *visits = -1;
  k_host_reset<<<1, 1, 0, st>>>(H, 3);
  bb<<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 3);
  ctx->launches += 2;
  int done = 0;
  while (!done) {
    for (int i = 0; i < links; ++i) {
      k_host_reset<<<1, 1, 0, st>>>(H, 5);
      bb<<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 3);
    }
    ctx->launches += 2 * links;
    links = links < 8 ? 2 * links : 8;
    ORCH_CUDA_TRY(cudaGetLastError());
    ORCH_CUDA_TRY(cudaMemcpyAsync(&done, &H->chain_done, sizeof done, cudaMemcpyDeviceToHost, st));
    ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (done != 1) return ORCH_OK;
  // the chain ends at the optimum pass 1 found (or is empty: the incumbents stand)
  int64_t last = 0;
  unsigned long long vstar = 0;
  ORCH_CUDA_TRY(cudaMemcpyAsync(&last, &H->chain_last, sizeof last, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(&vstar, &H->best_value, sizeof vstar, cudaMemcpyDeviceToHost, st));
  k_host_reset<<<1, 1, 0, st>>>(H, 4);
  bb<<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 4);
  ctx->launches += 2;
  ORCH_CUDA_TRY(cudaGetLastError());
  unsigned long long count = 0;
  int overflow = 0;
  ORCH_CUDA_TRY(cudaMemcpyAsync(&count, &H->visits, sizeof count, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(&overflow, &H->overflow, sizeof overflow, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  if (static_cast<unsigned long long>(last) != vstar)
    return fail(ORCH_LOGIC_ERROR, "solve_hosting: the improving-leaf chain misses the optimum");
  if (!overflow) *visits = static_cast<int64_t>(count);
  return ORCH_OK;
}

}  // namespace
}  // namespace orchb

using namespace orchb;

extern "C" {

int orch_solve_hosting_host(orch_ctx* ctx, int32_t d, int32_t c, const int64_t* h_V,
                            int32_t* h_hosting, int64_t* h_info, void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  int rc = check_hosting_args(d, c, ORCH_MAX_INSTANCES);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const bool wide = d > kHostMaxD;
  const size_t dd = static_cast<size_t>(d), nodes = static_cast<size_t>(d / c);
  int64_t *V, *info;
  int32_t *hosting, *b2i;
  int* g_better = nullptr;
  HostState* H;
  HostBufs hb;
  WideScratch w{};
  Plan all;
  all.add(&V, dd * dd);
  all.add(&info, 4);
  all.add(&hosting, dd);
  all.add(&b2i, dd);
  plan_host_search(all, d, c, &H, &hb);
  if (wide) {
    all.add(&w.gain, nodes * dd);
    all.add(&w.regret, dd);
    all.add(&w.at, dd);
    all.add(&w.srt_at, nodes * dd);
    all.add(&w.srt_g, nodes * dd);
    all.add(&w.greedy, dd);
    all.add(&w.sub, 4 * static_cast<size_t>(kHostMaxNodes));
    all.add(&w.a, dd);
    all.add(&g_better, 1);
  }
  rc = all.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(V, h_V, sizeof(int64_t) * dd * dd, cudaMemcpyHostToDevice, st));
  if (wide) {
    rc = run_wide_hosting(ctx, d, c, V, H, hb, w, hosting, b2i, info, g_better, st);
    if (rc) return rc;
  } else {
    rc = launch_hosting_search(ctx, d, c, 0, nullptr, nullptr, nullptr, V, nullptr, H, hb, st);
    if (rc) return rc;
    k_host_finish<<<1, 1024, 0, st>>>(H, V, hosting, b2i, info, RemapArgs{});
    ctx->launches += 1;
  }
  ORCH_CUDA_TRY(cudaGetLastError());
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_hosting, hosting, sizeof(int32_t) * d, cudaMemcpyDeviceToHost, st));
  int64_t hinfo[4];
  ORCH_CUDA_TRY(cudaMemcpyAsync(hinfo, info, sizeof hinfo, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  if (hinfo[2] == -1) {  // the exact answer is unknown: never return the incumbent silently
    if (h_info) memcpy(h_info, hinfo, sizeof hinfo);
    return fail(ORCH_UNSUPPORTED,
                "solve_hosting: the exact search exceeded its budget of 2^31 visited nodes");
  }
  if (h_info) {
    rc = reference_visits(ctx, H, d, c, st, &hinfo[3]);
    if (rc) return rc;
    memcpy(h_info, hinfo, sizeof hinfo);
  }
  return ORCH_OK;
}

int orch_inter_node_egress_host(orch_ctx* ctx, int32_t d, int32_t c, const int64_t* h_V,
                                const int32_t* h_hosting, int64_t* h_egress, void* stream) {
  if (!ctx || !h_V || !h_hosting || !h_egress) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (d < 1 || c < 1 || d % c)
    return fail(ORCH_INVALID_ARGUMENT, "instance count must be divisible by instances per node");
  if (d > ORCH_MAX_INSTANCES)
    return fail(ORCH_UNSUPPORTED, "inter_node_egress limited to d <= 4096 on the device");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  auto st = static_cast<cudaStream_t>(stream);
  const size_t dd = static_cast<size_t>(d), nodes = static_cast<size_t>(d / c);
  int64_t* V;
  int32_t* hosting;
  unsigned long long* e;
  Plan plan;
  plan.add(&V, dd * dd);
  plan.add(&hosting, dd);
  plan.add(&e, nodes);
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemcpyAsync(V, h_V, sizeof(int64_t) * dd * dd, cudaMemcpyHostToDevice, st));
  ORCH_CUDA_TRY(cudaMemcpyAsync(hosting, h_hosting, sizeof(int32_t) * dd, cudaMemcpyHostToDevice, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(e, 0, sizeof(unsigned long long) * nodes, st));
  const int grid = static_cast<int>(std::min<int64_t>((static_cast<int64_t>(dd * dd) + 255) / 256, kSMs * 4));
  k_node_egress<<<grid, 256, sizeof(unsigned long long) * nodes, st>>>(V, hosting, d, c, e);
  ctx->launches += 1;
  ORCH_CUDA_TRY(cudaGetLastError());
  ORCH_CUDA_TRY(cudaMemcpyAsync(h_egress, e, sizeof(int64_t) * nodes, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
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
  static const bool small_off = getenv("ORCH_NODEWISE_SMALL") && atoi(getenv("ORCH_NODEWISE_SMALL")) == 0;
  if (!small_off && nodewise_small_fits(d, c, n)) {
    Plan sp;
    int32_t *hosting, *b2i;
    sp.add_or(&hosting, d_hosting, d);
    sp.add_or(&b2i, d_batch_to_instance, d);
    rc = sp.commit(ctx, st);
    if (rc) return rc;
    NwArgs a{};
    a.d = d;
    a.c = c;
    a.n = static_cast<int>(n);
    a.len = d_len;
    a.origin = d_origin;
    a.dest_inst = bal->dest_inst;
    a.bin_count = bal->bin_count;
    a.bin_len = bal->bin_len;
    a.bin_tokens = bal->bin_tokens;
    a.bin_cost = bal->bin_cost;
    a.bin_offset = bal->bin_offset;
    a.bin_member = bal->bin_member;
    a.hosting = hosting;
    a.b2i = b2i;
    a.info = d_info;
    static PerDeviceOnce configured;
    const int rc_attr = configured([&]() -> int {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_nodewise_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(NwSmem))));
      ORCH_CUDA_TRY(max_carveout(k_nodewise_small));
      return ORCH_OK;
    });
    if (rc_attr) return rc_attr;
    k_nodewise_small<<<1, kNwThreads, sizeof(NwSmem), st>>>(a);
    ctx->launches += 1;
    ORCH_CUDA_TRY(cudaGetLastError());
    return ORCH_OK;
  }
  Plan plan;
  int64_t* V;
  HostState* H;
  HostBufs hb;
  int32_t *hosting, *b2i, *scratch = nullptr;
  int64_t* info;
  plan.add(&V, static_cast<size_t>(d) * d);
  plan_host_search(plan, d, c, &H, &hb);
  plan.add_or(&hosting, d_hosting, d);
  plan.add_or(&b2i, d_batch_to_instance, d);
  plan.add_or(&info, d_info, 4);
  if (n > kFinMaxItems) plan.add(&scratch, static_cast<size_t>(n));
  rc = plan.commit(ctx, st);
  if (rc) return rc;
  rc = launch_hosting_search(ctx, d, c, n, d_len, d_origin, bal->dest_inst, nullptr, V, H, hb, st);
  if (rc) return rc;
  RemapArgs r{n, bal->dest_inst, bal->bin_count, bal->bin_len, bal->bin_tokens, bal->bin_cost,
              bal->bin_offset, bal->bin_member, scratch};
  k_host_finish<<<1, 1024, 0, st>>>(H, V, hosting, b2i, info, r);
  ctx->launches += 1;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"
