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
// Work: the DFS tree cut at depth k0 into <= 8192 prefixes, then work stealing:
// one warp runs a subtree depth-first (lane = node); when warps are idle, a busy
// warp donates the shallowest untried sibling of its current path to a global
// queue. A subtree is identified by its path of candidate positions, and DFS
// order is the lexicographic order of paths, so pass 2 stays exact.
// The bound is the reference's lower_bound -- max over nodes of
// (total - gained - optimistic gain) -- read in O(1): the unassigned batches
// at depth k are exactly order[k..d), so the optimistic gain of node n with r
// slots left is a table og[k][n][r] built once.
#include <climits>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "plan.cuh"

namespace orchb {
namespace {

constexpr int kHostMaxD = 64;
constexpr int kHostMaxNodes = 32;                  // lane = node
constexpr int kOgMax = (kHostMaxD + 1) * (kHostMaxD + kHostMaxNodes);
constexpr int kHostWarps = 8;
constexpr long long kHostTasks = 8192;
constexpr int kHostGrid = 148;
constexpr int kHostQueue = 16384;  // donated subtrees waiting for a warp
constexpr unsigned long long kHostVisitBudget = 1ull << 31;
#ifndef ORCH_HOST_SLEEP
#define ORCH_HOST_SLEEP 2000
#endif
#ifndef ORCH_HOST_CHECK
#define ORCH_HOST_CHECK 63
#endif

struct HostState {
  int d, c, nodes, k0;
  long long tasks;                       // nodes^k0 prefixes, numbered in DFS order
  int64_t gain[kHostMaxD * kHostMaxD];   // [node][batch]
  int64_t node_total[kHostMaxD];
  int32_t order[kHostMaxD];              // branching order (descending regret, stable)
  int32_t incumbent[kHostMaxD];
  int64_t incumbent_value;
  // search tables by depth k (the batch order[k])
  int64_t g2[kHostMaxD * kHostMaxNodes];    // [k][node] gain of node for order[k]
  uint8_t no[kHostMaxD * kHostMaxNodes];    // [k][j] j-th candidate: descending gain, ties by node
  uint8_t pos[kHostMaxD * kHostMaxNodes];   // [k][node] inverse of no
  int64_t og[kOgMax];                       // [k][node][r] sum of the top r gains over order[k..d)
  unsigned long long best_value;            // pass 1 incumbent value (starts at the incumbents')
  unsigned long long visits;
  int overflow;
  // work distribution, reset before each pass
  unsigned long long task_counter;          // initial prefixes handed out
  unsigned q_head, q_tail;                  // donated subtrees
  int pending;                              // tasks queued or running
  int idle;                                 // warps waiting for work
  int lock;
  int have_best;                            // pass 2: best_path holds a V*-leaf
  uint8_t best_path[kHostMaxD];             // candidate position per depth
  unsigned q_ready[kHostQueue];             // pass << 30 | (index + 1) once published, 0 once read
  uint8_t q_depth[kHostQueue];
  uint8_t q_path[kHostQueue][kHostMaxD];
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
  H->best_value = static_cast<unsigned long long>(H->incumbent_value);
  H->visits = 0;
  H->overflow = 0;
  H->have_best = 0;
  int k0 = 0;
  long long tasks = 1;
  while (k0 < d && tasks * nodes <= kHostTasks) {
    tasks *= nodes;
    ++k0;
  }
  H->k0 = k0;
  H->tasks = tasks;
}

// Search tables: thread k < d builds depth k's candidate order (stable sort of
// the nodes by descending gain for batch order[k]); thread n < nodes builds
// og[.][n][.] from the deepest level up, keeping its top-c gains sorted.
__global__ void k_host_tables(HostState* __restrict__ H) {
  const int d = H->d, c = H->c, nodes = H->nodes, t = threadIdx.x;
  if (t < d) {
    const int b = H->order[t];
    uint8_t* no = H->no + t * nodes;
    for (int n = 0; n < nodes; ++n) {
      H->g2[t * nodes + n] = H->gain[n * d + b];
      int j = n - 1;  // insertion: strictly larger gains first, ties keep node order
      while (j >= 0 && H->gain[no[j] * d + b] < H->gain[n * d + b]) {
        no[j + 1] = no[j];
        --j;
      }
      no[j + 1] = static_cast<uint8_t>(n);
    }
    for (int j = 0; j < nodes; ++j) H->pos[t * nodes + no[j]] = static_cast<uint8_t>(j);
  }
  if (t < nodes) {
    int64_t top[kHostMaxD];
    int have = 0;
    for (int k = d; k >= 0; --k) {
      if (k < d) {  // insert gain of order[k]
        const int64_t g = H->gain[t * d + H->order[k]];
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
      int64_t* og = H->og + (static_cast<size_t>(k) * nodes + t) * (c + 1);
      int64_t acc = 0;
      og[0] = 0;
      for (int r = 1; r <= c; ++r) {
        if (r <= have) acc += top[r - 1];
        og[r] = acc;
      }
    }
  }
}

// per warp: choice stack ch[64] (u8), then avail[64] and donated[64] (u32 masks)
constexpr int kWarpStack = kHostMaxD + 2 * 4 * kHostMaxD;

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
  return host_table_bytes(d, c) + kHostWarps * kWarpStack;
}

__device__ HostSmem host_load_tables(const HostState& H, unsigned char* raw) {
  const int d = H.d, c = H.c, nodes = H.nodes;
  int64_t* g2 = reinterpret_cast<int64_t*>(raw);
  int64_t* og = g2 + d * nodes;
  uint8_t* no = reinterpret_cast<uint8_t*>(og + (d + 1) * nodes * (c + 1));
  uint8_t* pos = no + d * nodes;
  for (int i = threadIdx.x; i < d * nodes; i += blockDim.x) {
    g2[i] = H.g2[i];
    no[i] = H.no[i];
    pos[i] = H.pos[i];
  }
  for (int i = threadIdx.x; i < (d + 1) * nodes * (c + 1); i += blockDim.x) og[i] = H.og[i];
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

struct WarpStack {
  uint8_t* ch;        // candidate position chosen per depth
  unsigned* avail;    // positions with room per depth (as of choosing there)
  unsigned* donated;  // positions given away per depth (current path only)
};

// Depth-first search of the subtree below the path ch[0, root) (state: this
// lane's room / gained). pass 1 prunes lb >= best and lowers the global
// incumbent at leaves; pass 2 prunes lb > vstar and paths after the best
// V*-leaf, and records a V*-leaf if it sorts first. Donates siblings to idle
// warps. Returns when the subtree is exhausted (or cut).
__device__ void host_dfs(HostState& H, const HostSmem& T, int pass, int64_t vstar, WarpStack W,
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
        } else if (__shfl_sync(~0u, lane == 0 ? volatile_i32(&H.have_best) : 0, 0) &&
                   path_cmp(W.ch, H.best_path, k, lane) > 0) {
          break;  // everything left in this subtree sorts after the best V*-leaf
        }
        // donate the shallowest untried sibling when warps wait for work
        int want = 0;
        if (lane == 0) {
          const unsigned queued = volatile_u32(&H.q_tail) - volatile_u32(&H.q_head);
          want = volatile_i32(&H.idle) > static_cast<int>(queued) && queued < kHostQueue - 2048;
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
            if (lane == 0)  // the slot's previous subtree must have been read out
              while (volatile_u32(&H.q_ready[slot % kHostQueue]) != 0u) {
              }
            __syncwarp();
            uint8_t* dst = H.q_path[slot % kHostQueue];
            for (int l = lane; l < lvl; l += 32) dst[l] = W.ch[l];
            if (lane == 0) {
              dst[lvl] = static_cast<uint8_t>(q);
              H.q_depth[slot % kHostQueue] = static_cast<uint8_t>(lvl + 1);
            }
            __syncwarp();
            __threadfence();
            __syncwarp();
            if (lane == 0)
              *reinterpret_cast<volatile unsigned*>(&H.q_ready[slot % kHostQueue]) =
                  (static_cast<unsigned>(pass) << 30) | (slot + 1);
            W.donated[lvl] |= 1u << q;
            __syncwarp();
          }
        }
      }
      const int64_t term =
          active ? total - gained - T.og[(static_cast<size_t>(k) * nodes + lane) * (c + 1) + room]
                 : 0;
      const int64_t lb = warp_max_nonneg(term);  // egress >= 0: clamping keeps the bound valid
      bool prune = pass == 1 ? lb >= best : lb > vstar;
      if (!prune && k == d) {  // leaf: value == lb
        if (pass == 1) {
          if (lane == 0) atomicMin(&H.best_value, static_cast<unsigned long long>(lb));
          best = lb;
          prune = true;
        } else {  // a V*-leaf: keep it if it is the first in DFS order so far
          if (lane == 0)
            while (atomicCAS(&H.lock, 0, 1) != 0) {
            }
          __syncwarp();
          __threadfence();
          const bool first = !__shfl_sync(~0u, lane == 0 ? volatile_i32(&H.have_best) : 0, 0) ||
                             path_cmp(W.ch, H.best_path, d, lane) < 0;
          if (first) {
            volatile uint8_t* bp = H.best_path;
            for (int l = lane; l < d; l += 32) bp[l] = W.ch[l];
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
    ++k;
    if (k < d) W.donated[k] = 0;
    descend = true;
  }
  if (lane == 0) atomicAdd(&H.visits, visits & 65535);
}

// Before each pass. The queue's publish flags are cleared too: the state lives
// in the reused workspace arena, and a flag left over from an earlier search
// (same pass, same slot) would let a reader take a path before it is written.
__global__ void k_host_reset(HostState* __restrict__ H) {
  for (int i = threadIdx.x; i < kHostQueue; i += blockDim.x) H->q_ready[i] = 0u;
  if (threadIdx.x == 0) {
    H->task_counter = 0;
    H->q_head = H->q_tail = 0;
    H->pending = static_cast<int>(H->tasks);
    H->idle = 0;
    H->lock = 0;
  }
}

__global__ void __launch_bounds__(kHostWarps * 32) k_host_bb(HostState* __restrict__ Hp, int pass) {
  extern __shared__ __align__(16) unsigned char host_raw[];
  HostState& H = *Hp;
  if (H.overflow) return;
  if (pass == 2 && static_cast<long long>(H.best_value) >= H.incumbent_value) return;
  const HostSmem T = host_load_tables(H, host_raw);
  const int warp = __shfl_sync(~0u, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  unsigned char* ws = host_raw + host_table_bytes(H.d, H.c) + warp * kWarpStack;
  WarpStack W{ws, reinterpret_cast<unsigned*>(ws + kHostMaxD),
              reinterpret_cast<unsigned*>(ws + kHostMaxD) + kHostMaxD};
  const int64_t vstar = static_cast<int64_t>(H.best_value);
  const int c = H.c, nodes = H.nodes, k0 = H.k0;
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
      long long div = H.tasks / nodes;
      for (int k = 0; k < k0; ++k) {
        const int p = static_cast<int>((t / (div > 0 ? div : 1)) % nodes);
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
      }
      root = k0;
    } else {  // donated subtree: wait until published, then replay its path
      const unsigned slot = static_cast<unsigned>(qs) % kHostQueue;
      const unsigned want = (static_cast<unsigned>(pass) << 30) | (static_cast<unsigned>(qs) + 1);
      if (lane == 0)
        while (volatile_u32(&H.q_ready[slot]) != want) {
        }
      __syncwarp();
      __threadfence();
      root = *reinterpret_cast<volatile uint8_t*>(&H.q_depth[slot]);
      const volatile uint8_t* src = H.q_path[slot];
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
        *reinterpret_cast<volatile unsigned*>(&H.q_ready[slot]) = 0u;
    }
    __syncwarp();
    if (ok && pass == 2 && __shfl_sync(~0u, lane == 0 ? volatile_i32(&H.have_best) : 0, 0) &&
        path_cmp(W.ch, H.best_path, root, lane) > 0)
      ok = false;  // the whole subtree sorts after the best V*-leaf
    if (ok) host_dfs(H, T, pass, vstar, W, root, room, gained);
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicSub(&H.pending, 1);
    }
  }
}

// Final hosting, batch -> instance map, egress figures; then the result remap.
__global__ void k_host_finish(const HostState* __restrict__ Hp, const int64_t* __restrict__ V,
                              int32_t* __restrict__ hosting, int32_t* __restrict__ b2i,
                              int64_t* __restrict__ info) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const HostState& H = *Hp;
  int32_t a[kHostMaxD];
  const bool incumbent = static_cast<long long>(H.best_value) >= H.incumbent_value ||
                         H.overflow || !H.have_best;
  for (int b = 0; b < H.d; ++b) a[b] = H.incumbent[b];
  if (!incumbent)
    for (int l = 0; l < H.d; ++l) a[H.order[l]] = H.no[l * H.nodes + H.best_path[l]];
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
  info[2] = H.overflow ? -1 : (incumbent ? 0 : 1);  // -1: visit budget hit, incumbent kept
  info[3] = static_cast<int64_t>(H.visits);
#ifdef ORCH_HOST_DEBUG
  printf("hosting: best %llu inc %lld visits %llu overflow %d k0 %d tasks %lld queued %u\n",
         H.best_value, (long long)H.incumbent_value, H.visits, H.overflow, H.k0, H.tasks,
         H.q_tail);
#endif
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

// ------------------------------------------------ one-CTA node-wise path
// For small searches (d <= 32, <= 2^18 leaves, n <= 12288: every C2 shape on
// 2/4/8 GPUs) the whole of orch_nodewise runs in ONE kernel, in shared memory:
// volume matrix -> gains, regret order, incumbents, search tables -> two-pass
// branch and bound (32 warps, lane = node, DFS-ordered prefix tasks) -> hosting,
// batch_to_instance, egress figures -> relabelling of the balance result.
// The metadata chain runs beside the NVLink row exchange, where every global
// round trip costs several microseconds; this path pays about four of them
// instead of a dozen launches and copies. Same answer as the multi-CTA path
// (first optimal leaf in DFS order, the incumbents otherwise).
constexpr int kNwThreads = 1024;
constexpr int kNwWarps = kNwThreads / 32;
constexpr int kNwMaxD = 32;
constexpr int kNwMaxItems = 12288;
constexpr int kNwTasks = 64;  // at least two prefix tasks per warp
constexpr double kNwMaxLeaves = 262144.0;

struct NwSmem {
  unsigned long long V[kNwMaxD * kNwMaxD];  // [src instance][dest batch]
  int64_t gain[kNwMaxD * kNwMaxD];          // [node][batch]
  int64_t g2[kNwMaxD * kNwMaxD];            // [k][node]
  int64_t og[(kNwMaxD + 1) * 2 * kNwMaxD];  // [k][node][r], (d+1)*nodes*(c+1) <= (d+1)*2d
  int64_t node_total[kNwMaxD];
  int64_t regret[kNwMaxD];
  int64_t node_e[kNwMaxD], node_e0[kNwMaxD];
  int64_t incumbent_value;
  unsigned long long best;  // pass 1: best value so far
  unsigned long long visits;
  int32_t order[kNwMaxD];
  int32_t ident[kNwMaxD], greedy[kNwMaxD], incumbent[kNwMaxD], a[kNwMaxD];
  int32_t b2i[kNwMaxD], inv[kNwMaxD], noff[kNwMaxD + 1];
  int32_t ocnt[kNwMaxD], ooff[kNwMaxD + 1];
  int64_t olen[kNwMaxD], otok[kNwMaxD];
  double ocost[kNwMaxD];
  uint8_t no[kNwMaxD * kNwMaxD];   // [k][j] j-th candidate node of depth k
  uint8_t pos[kNwMaxD * kNwMaxD];  // [k][node]
  uint8_t ch[kNwWarps][kNwMaxD];   // per-warp DFS path (candidate positions)
  uint8_t best_path[kNwMaxD];
  int64_t vals[2];
  int tasks, k0, best_task, lock;
  unsigned task_ctr;
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

// argmax over lanes of v (v >= -1), lowest lane on ties
__device__ __forceinline__ int warp_argmax_first(int64_t v) {
  int lane = threadIdx.x & 31;
  int64_t bv = v;
  int bl = lane;
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

// DFS of the subtree below ch[0, root) for one warp (lane = node); the
// prune rules and visiting order of host_dfs, without donation.
__device__ void nw_dfs(NwSmem& S, int pass, int64_t vstar, int task, int root, int room,
                       int64_t gained, int d, int c, int nodes, uint8_t* ch) {
  const int lane = threadIdx.x & 31;
  const bool active = lane < nodes;
  const int64_t total = active ? S.node_total[lane] : 0;
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
          active ? total - gained - S.og[(static_cast<size_t>(k) * nodes + lane) * (c + 1) + room] : 0;
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
          const int won = __shfl_sync(~0u, lane == 0 ? (task < *reinterpret_cast<volatile int*>(&S.best_task)) : 0, 0);
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
      const int m = S.no[k * nodes + j];
      if (lane == m) {
        ++room;
        gained -= S.g2[k * nodes + m];
      }
      jstart = j + 1;
    }
    const unsigned av =
        __reduce_or_sync(~0u, (active && room > 0) ? (1u << S.pos[k * nodes + lane]) : 0u);
    const unsigned pm = jstart >= 32 ? 0u : av & (~0u << jstart);
    if (!pm) {
      descend = false;
      continue;
    }
    const int j = __ffs(pm) - 1;
    __syncwarp();
    if (lane == 0) ch[k] = static_cast<uint8_t>(j);
    __syncwarp();
    const int m = S.no[k * nodes + j];
    if (lane == m) {
      --room;
      gained += S.g2[k * nodes + m];
    }
    ++k;
    descend = true;
  }
  if (lane == 0) atomicAdd(&S.visits, visits);
}

// one pass over the prefix tasks (DFS order), dynamic claiming
__device__ void nw_pass(NwSmem& S, int pass, int64_t vstar, int d, int c, int nodes) {
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
      break;  // tasks are claimed in DFS order: the rest sort after the best leaf
    int room = active ? c : 0;
    int64_t gained = 0;
    bool ok = true;
    int div = S.tasks / nodes;
    for (int k = 0; k < S.k0; ++k) {
      const int p = (t / (div > 0 ? div : 1)) % nodes;
      div /= nodes;
      const unsigned pm =
          __reduce_or_sync(~0u, (active && room > 0) ? (1u << S.pos[k * nodes + lane]) : 0u);
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
      const int m = S.no[k * nodes + j];
      if (lane == m) {
        --room;
        gained += S.g2[k * nodes + m];
      }
    }
    if (ok) nw_dfs(S, pass, vstar, t, S.k0, room, gained, d, c, nodes, ch);
  }
}

__global__ void __launch_bounds__(kNwThreads, 1) k_nodewise_small(NwArgs a) {
  extern __shared__ __align__(16) unsigned char nw_raw[];
  NwSmem& S = *reinterpret_cast<NwSmem*>(nw_raw);
  const int d = a.d, c = a.c, nodes = d / c, n = a.n, t = threadIdx.x;
#ifdef ORCH_NW_STAMPS
  uint64_t ts[8];
  int nts = 0;
  auto stamp = [&] { if (t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[nts++])); };
  stamp();
#else
  auto stamp = [] {};
#endif
  const int lane = t & 31, warp = t >> 5;
  // ---- volume matrix (topology.cpp:40-53) and the old per-batch arrays
  for (int i = t; i < d * d; i += kNwThreads) S.V[i] = 0;
  if (t < d) {
    S.ocnt[t] = a.bin_count[t];
    if (a.bin_len) S.olen[t] = a.bin_len[t];
    if (a.bin_tokens) S.otok[t] = a.bin_tokens[t];
    if (a.bin_cost) S.ocost[t] = a.bin_cost[t];
  }
  if (t <= d) S.ooff[t] = a.bin_offset[t];
  if (t == 0) {
    S.visits = 0;
    S.task_ctr = 0;
    S.best_task = INT_MAX;
    S.lock = 0;
  }
  __syncthreads();
  for (int i = t; i < n; i += kNwThreads) {
    S.members[i] = a.bin_member[i];
    atomicAdd(&S.V[a.origin[i] * d + a.dest_inst[i]], static_cast<unsigned long long>(a.len[i]));
  }
  __syncthreads();
  stamp();
  // ---- gains, node totals (topology.cpp:195-262)
  for (int i = t; i < nodes * d; i += kNwThreads) {
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
  if (t < d) {
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
    for (int b = 0; b < d; ++b)
      r += S.regret[b] > S.regret[t] || (S.regret[b] == S.regret[t] && b < t);
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
  } else if (warp == 1) {  // search tables, candidate order per depth
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
    int64_t top[kNwMaxD];
    int have = 0;
    for (int k = d; k >= 0; --k) {
      if (k < d) {
        const int64_t g = S.gain[lane * d + S.order[k]];
        int j = -1;
        if (have < c) j = have++;
        else if (top[c - 1] < g) j = c - 1;
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
  if (warp < 2) {  // host_value of identity (warp 0) and greedy (warp 1)
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
  }
  __syncthreads();
  if (t < d) {
    const bool g_better = S.vals[1] < S.vals[0];  // offer(greedy) only when strictly better
    S.incumbent[t] = g_better ? S.greedy[t] : S.ident[t];
  }
  if (t == 0) {
    const bool g_better = S.vals[1] < S.vals[0];
    S.incumbent_value = g_better ? S.vals[1] : S.vals[0];
    S.best = static_cast<unsigned long long>(S.incumbent_value);
    // a few prefix tasks per warp: the trees here are small, and a task costs
    // its prefix decode even when the bound cuts it at once
    int k0 = 0, tasks = 1;
    while (k0 < d && tasks < kNwTasks) {
      tasks *= nodes;
      ++k0;
    }
    S.k0 = k0;
    S.tasks = tasks;
    // no leaf can beat the incumbents when the root bound already reaches them
    int64_t lb = 0;
    for (int nd = 0; nd < nodes; ++nd) {
      const int64_t e = S.node_total[nd] - S.og[static_cast<size_t>(nd) * (c + 1) + c];
      lb = e > lb ? e : lb;
    }
    if (lb >= S.incumbent_value) S.tasks = 0;
  }
  __syncthreads();
  stamp();
  // ---- search: pass 1 finds V*, pass 2 the first V*-leaf in DFS order
  nw_pass(S, 1, 0, d, c, nodes);
  __syncthreads();
  stamp();
  const int64_t vstar = static_cast<int64_t>(S.best);
  const bool search2 = vstar < S.incumbent_value;
  if (t == 0) S.task_ctr = 0;
  __syncthreads();
  if (search2) nw_pass(S, 2, vstar, d, c, nodes);
  __syncthreads();
  stamp();
  // ---- hosting, batch -> instance (topology.cpp:283-290), egress figures
  const bool incumbent = !search2 || S.best_task == INT_MAX;
  if (t < d) S.a[t] = S.incumbent[t];
  __syncthreads();
  if (!incumbent && t < d) S.a[S.order[t]] = S.no[t * nodes + S.best_path[t]];
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
        const int64_t v = static_cast<int64_t>(S.V[i * d + b]);
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
#ifdef ORCH_NW_STAMPS
  __syncthreads();
  stamp();
  if (t == 0) {
    static __device__ unsigned calls = 0;
    if ((atomicAdd(&calls, 1u) % 16) == 15)
      printf("NWSTAMP d=%d c=%d load %.1f prep %.1f pass1 %.1f pass2 %.1f out %.1f us visits %llu tasks %d\n", d, c,
             (ts[1] - ts[0]) / 1e3, (ts[2] - ts[1]) / 1e3, (ts[3] - ts[2]) / 1e3, (ts[4] - ts[3]) / 1e3,
             (ts[5] - ts[4]) / 1e3, S.visits, S.tasks);
  }
#endif
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

int check_hosting_args(int d, int c) {
  if (d < 1 || c < 1)
    return fail(ORCH_INVALID_ARGUMENT, "topology needs at least one instance and one per node");
  if (d % c) return fail(ORCH_INVALID_ARGUMENT, "instance count must be divisible by instances per node");
  if (d > kHostMaxD) return fail(ORCH_UNSUPPORTED, "node-wise hosting limited to d <= 64 on the device");
  if (d / c > kHostMaxNodes)
    return fail(ORCH_UNSUPPORTED, "node-wise hosting limited to 32 nodes on the device");
  return ORCH_OK;
}

int launch_hosting_search(orch_ctx* ctx, int d, int c, const int64_t* V, HostState* H,
                          cudaStream_t st) {
  const int sm = static_cast<int>(host_smem_bytes(d, c));
  static bool configured = false;
  if (!configured) {
    const int mx = static_cast<int>(host_smem_bytes(kHostMaxD, 2));  // the largest table set
    ORCH_CUDA_TRY(cudaFuncSetAttribute(k_host_bb, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    configured = true;
  }
  k_host_prep<<<1, 32, 0, st>>>(d, c, V, H);
  k_host_tables<<<1, kHostMaxD, 0, st>>>(H);
  k_host_reset<<<1, 1024, 0, st>>>(H);
  k_host_bb<<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 1);
  k_host_reset<<<1, 1024, 0, st>>>(H);
  k_host_bb<<<kHostGrid, kHostWarps * 32, sm, st>>>(H, 2);
  ctx->launches += 6;
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
  rc = launch_hosting_search(ctx, d, c, V, H, st);
  if (rc) return rc;
  k_host_finish<<<1, 32, 0, st>>>(H, V, hosting, b2i, info);
  ctx->launches += 1;
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
    static bool configured = false;
    if (!configured) {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_nodewise_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(NwSmem))));
      configured = true;
    }
    k_nodewise_small<<<1, kNwThreads, sizeof(NwSmem), st>>>(a);
    ctx->launches += 1;
    ORCH_CUDA_TRY(cudaGetLastError());
    return ORCH_OK;
  }
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
  rc = launch_hosting_search(ctx, d, c, dV, H, st);
  if (rc) return rc;
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
  ctx->launches += 3;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"
