/*
 * orchsim_oracle.c -- plain-C restatement of the reference Batch
 * Post-Balancing Dispatcher. TEST INFRASTRUCTURE ONLY (see orchsim_oracle.h):
 * the checker for the B200 library, never linked into it.
 *
 * Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj).
 */
#include "orchsim_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ cost */

/* core.cpp:91-118. Evaluation order kept exactly (left-associative double
 * products, no contraction: compiled with -ffp-contract=off). `lens` is the
 * batch in slot order. */
static double batch_cost(double alpha, double beta, int padded, int variant, int64_t count,
                         const int64_t* lens_in_order, const int32_t* members,
                         const int64_t* len_by_pos) {
  if (count == 0) return 0.0;
  int64_t sum = 0, mx = 0;
  for (int64_t s = 0; s < count; ++s) {
    const int64_t l = lens_in_order ? lens_in_order[s] : len_by_pos[members[s]];
    sum += l;
    if (l > mx) mx = l;
  }
  const int64_t blen = padded ? count * mx : sum; /* core.cpp:70-89 */
  const double linear = alpha * (double)blen;
  switch (variant) {
    case ORC_LINEAR_ONLY:
      return linear;
    case ORC_TRANSFORMER_QUADRATIC: {
      if (!padded) {
        double square_sum = 0.0; /* sequential, slot order: core.cpp:101-104 */
        for (int64_t s = 0; s < count; ++s) {
          const int64_t l = lens_in_order ? lens_in_order[s] : len_by_pos[members[s]];
          square_sum += (double)l * (double)l;
        }
        return linear + beta * square_sum;
      }
      const double p = (double)blen;
      return linear + beta / (double)count * p * p; /* core.cpp:108-109 */
    }
    case ORC_CONV_TRANSFORMER_PADDED: {
      const double longest = (double)mx;
      return linear + beta * (double)count * longest * longest; /* core.cpp:112-114 */
    }
  }
  return linear;
}

int orc_cost(double alpha, double beta, int model_padded, int variant, int batch_padded,
             int64_t n, const int64_t* len, double* out) {
  if (model_padded != batch_padded)
    return fail(1, "cost model padding mode does not match batch padding mode");
  *out = batch_cost(alpha, beta, batch_padded, variant, n, len, NULL, NULL);
  return 0;
}

/* orchestrator.cpp:91-102 */
void orc_stats(int d, const double* costs, double* max, double* mean, double* ratio) {
  double mx = 0.0, total = 0.0;
  for (int i = 0; i < d; ++i) {
    if (costs[i] > mx) mx = costs[i];
    total += costs[i];
  }
  const double mn = d == 0 ? 0.0 : total / (double)d;
  if (max) *max = mx;
  if (mean) *mean = mn;
  if (ratio) *ratio = mn > 0.0 ? mx / mn : 1.0;
}

/* ------------------------------------------------------- policy plumbing */

/* policy_cost_model: balancers.cpp:162-176; native_mode: :39-41 */
static void policy_model(int kind, double lambda, double* beta, int* padded, int* variant) {
  *padded = kind == ORC_BINARY_PADDED;
  switch (kind) {
    case ORC_GREEDY_UNPADDED:
    case ORC_BINARY_PADDED:
      *beta = 0.0;
      *variant = ORC_LINEAR_ONLY;
      break;
    case ORC_QUADRATIC_TOLERANCE:
      *beta = lambda;
      *variant = ORC_TRANSFORMER_QUADRATIC;
      break;
    default:
      *beta = lambda;
      *variant = ORC_CONV_TRANSFORMER_PADDED;
      break;
  }
}

/* Packing under construction: bins as growable arrays of input positions. */
typedef struct {
  int d;
  int32_t** items;
  int64_t* count;
  int64_t* cap;
} packing;

static void pk_init(packing* p, int d) {
  p->d = d;
  p->items = calloc((size_t)d, sizeof(int32_t*));
  p->count = calloc((size_t)d, sizeof(int64_t));
  p->cap = calloc((size_t)d, sizeof(int64_t));
}
static void pk_push(packing* p, int b, int32_t pos) {
  if (p->count[b] == p->cap[b]) {
    p->cap[b] = p->cap[b] ? 2 * p->cap[b] : 8;
    p->items[b] = realloc(p->items[b], (size_t)p->cap[b] * sizeof(int32_t));
  }
  p->items[b][p->count[b]++] = pos;
}
static void pk_free(packing* p) {
  for (int b = 0; b < p->d; ++b) free(p->items[b]);
  free(p->items);
  free(p->count);
  free(p->cap);
}

/* index_sources: balancers.cpp:25-37 -- validation in input order, source
 * slot = running count per origin. */
static int index_sources(int d, int64_t n, const int64_t* len, const int32_t* origin,
                         int32_t* src_slot) {
  int32_t* next = calloc((size_t)d, sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) {
    if (origin[i] < 0 || origin[i] >= d) {
      free(next);
      return fail(1, "item origin instance outside [0, d)");
    }
    if (len[i] < 1) {
      free(next);
      return fail(1, "item length must be >= 1");
    }
    src_slot[i] = next[origin[i]]++;
  }
  free(next);
  return 0;
}

/* sorted_descending / sorted_ascending: balancers.cpp:78-88 (stable_sort by
 * length only). The composite key (length, input position) is unique, so any
 * correct sort on it reproduces the stable sort. */
static const int64_t* g_sort_len;
static int cmp_desc(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  if (g_sort_len[x] != g_sort_len[y]) return g_sort_len[x] > g_sort_len[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}
static int cmp_asc(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  if (g_sort_len[x] != g_sort_len[y]) return g_sort_len[x] < g_sort_len[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}
static int32_t* sorted_order(int64_t n, const int64_t* len, int descending) {
  int32_t* order = malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
  g_sort_len = len;
  qsort(order, (size_t)n, sizeof(int32_t), descending ? cmp_desc : cmp_asc);
  return order;
}

/* distribute_min_sum: balancers.cpp:92-107. std::priority_queue over
 * (sum, batch index) with std::greater: pops the lexicographic minimum. A
 * binary min-heap on the same unique keys pops the same sequence. */
typedef struct {
  int64_t sum;
  int idx;
} hentry;
static int hless(hentry a, hentry b) { return a.sum < b.sum || (a.sum == b.sum && a.idx < b.idx); }
static void heap_push(hentry* h, int* sz, hentry e) {
  int i = (*sz)++;
  h[i] = e;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!hless(h[i], h[p])) break;
    hentry t = h[i];
    h[i] = h[p];
    h[p] = t;
    i = p;
  }
}
static hentry heap_pop(hentry* h, int* sz) {
  hentry top = h[0];
  h[0] = h[--(*sz)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < *sz && hless(h[l], h[m])) m = l;
    if (r < *sz && hless(h[r], h[m])) m = r;
    if (m == i) break;
    hentry t = h[i];
    h[i] = h[m];
    h[m] = t;
    i = m;
  }
  return top;
}
static void distribute_min_sum(const int32_t* desc, int64_t cnt, const int64_t* len,
                               packing* pk) {
  hentry* h = malloc((size_t)pk->d * sizeof(hentry));
  int sz = 0;
  for (int b = 0; b < pk->d; ++b) {
    int64_t s = 0;
    for (int64_t k = 0; k < pk->count[b]; ++k) s += len[pk->items[b][k]];
    heap_push(h, &sz, (hentry){s, b});
  }
  for (int64_t k = 0; k < cnt; ++k) {
    hentry e = heap_pop(h, &sz);
    pk_push(pk, e.idx, desc[k]);
    e.sum += len[desc[k]];
    heap_push(h, &sz, e);
  }
  free(h);
}

/* get_least_batches: balancers.cpp:111-123 -- returns group count, and if
 * `start` is non-NULL the start index of every group (ascending positions). */
static int64_t least_batches(const int32_t* asc, int64_t n, const int64_t* len, int64_t bound,
                             int64_t* start) {
  int64_t groups = 1, size = 0;
  if (start) start[0] = 0;
  for (int64_t idx = 0; idx < n; ++idx) {
    const int64_t l = len[asc[idx]];
    if ((size + 1) * l > bound) {
      if (start) start[groups] = idx;
      ++groups;
      size = 0;
    }
    ++size;
  }
  return groups;
}

/* padded_binary_search: balancers.cpp:130-143 */
static int64_t padded_search(int d, const int32_t* asc, int64_t n, const int64_t* len) {
  const int64_t max_len = len[asc[n - 1]];
  int64_t left = max_len, right = max_len * (n / d + 1);
  while (left < right) {
    const int64_t mid = (left + right) / 2;
    if (least_batches(asc, n, len, mid, NULL) <= d)
      right = mid;
    else
      left = mid + 1;
  }
  return left;
}

/* tolerance_less: balancers.cpp:151-154 */
static int tolerance_less(int64_t as, int64_t aq, int64_t bs, int64_t bq, int64_t v) {
  const int64_t diff = as - bs;
  if ((diff < 0 ? -diff : diff) < v) return aq < bq;
  return as < bs;
}

/* assemble: balancers.cpp:43-60 -- evaluates a packing and fills the outputs.
 * Returns the objective (max over batches of cost(), starting at 0.0). */
static double assemble_objective(const packing* pk, int kind, double lambda, const int64_t* len) {
  double beta;
  int padded, variant;
  policy_model(kind, lambda, &beta, &padded, &variant);
  double obj = 0.0;
  for (int b = 0; b < pk->d; ++b) {
    const double c = batch_cost(1.0, beta, padded, variant, pk->count[b], NULL, pk->items[b], len);
    if (c > obj) obj = c; /* std::max(objective, cost) */
  }
  return obj;
}

static void export_packing(const packing* pk, int kind, double lambda, const int64_t* len,
                           orc_balance_out* out) {
  double beta;
  int padded, variant;
  policy_model(kind, lambda, &beta, &padded, &variant);
  for (int b = 0; b < pk->d; ++b) {
    int64_t off = 0, mx = 0;
    for (int64_t s = 0; s < pk->count[b]; ++s) {
      const int32_t pos = pk->items[b][s];
      if (out->dest_inst) out->dest_inst[pos] = b;
      if (out->dest_slot) out->dest_slot[pos] = (int32_t)s;
      if (out->dst_off) out->dst_off[pos] = off;
      off += len[pos];
      if (len[pos] > mx) mx = len[pos];
    }
    if (out->bin_count) out->bin_count[b] = (int32_t)pk->count[b];
    if (out->bin_tokens) out->bin_tokens[b] = off;
    if (out->bin_len) out->bin_len[b] = padded ? pk->count[b] * mx : off;
    if (out->bin_cost)
      out->bin_cost[b] = batch_cost(1.0, beta, padded, variant, pk->count[b], NULL, pk->items[b], len);
  }
}

/* group_by_origin: balancers.cpp:62-66 */
static void group_by_origin(int64_t n, const int32_t* origin, packing* pk) {
  for (int64_t i = 0; i < n; ++i) pk_push(pk, origin[i], (int32_t)i);
}

static void export_sources(int d, int64_t n, const int64_t* len, const int32_t* origin,
                           const int32_t* src_slot, orc_balance_out* out) {
  if (out->src_slot) memcpy(out->src_slot, src_slot, (size_t)n * sizeof(int32_t));
  if (out->src_off) {
    int64_t* run = calloc((size_t)d, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
      out->src_off[i] = run[origin[i]];
      run[origin[i]] += len[i];
    }
    free(run);
  }
}

static orc_balance_out g_null_out;

int orc_balance(int kind, double lambda, int64_t tolerance_v, int d, int64_t n,
                const int64_t* len, const int32_t* origin, orc_balance_out* out,
                double* objective, int32_t* used_identity) {
  if (!out) out = &g_null_out;
  if (kind < 0 || kind > 3) return fail(4, "unknown policy kind");
  if (d < 1) return fail(1, "instance count must be >= 1"); /* require_valid_d :156-158 */
  if ((kind == ORC_BINARY_PADDED || kind == ORC_CONVTRANSFORMER) && n == 0)
    return fail(1, kind == ORC_BINARY_PADDED ? "padded balancing needs at least one item"
                                             : "convtransformer balancing needs at least one item");
  if (kind == ORC_QUADRATIC_TOLERANCE && (lambda < 0.0 || tolerance_v < 0))
    return fail(1, "lambda and tolerance_v must be nonnegative");
  if (kind == ORC_CONVTRANSFORMER && lambda < 0.0) return fail(1, "lambda must be nonnegative");

  int32_t* src_slot = malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  int rc = index_sources(d, n, len, origin, src_slot);
  if (rc) {
    free(src_slot);
    return rc;
  }
  packing pk;
  pk_init(&pk, d);

  if (kind == ORC_GREEDY_UNPADDED) { /* :185-192 */
    int32_t* desc = sorted_order(n, len, 1);
    distribute_min_sum(desc, n, len, &pk);
    free(desc);
  } else if (kind == ORC_BINARY_PADDED) { /* :194-208 */
    int32_t* asc = sorted_order(n, len, 0);
    const int64_t bound = padded_search(d, asc, n, len);
    int64_t* start = malloc((size_t)(n + 2) * sizeof(int64_t));
    const int64_t groups = least_batches(asc, n, len, bound, start);
    start[groups] = n;
    for (int64_t g = 0; g < groups; ++g)
      for (int64_t k = start[g]; k < start[g + 1]; ++k) pk_push(&pk, (int)g, asc[k]);
    free(start);
    free(asc);
  } else if (kind == ORC_QUADRATIC_TOLERANCE) { /* :210-233 */
    int32_t* desc = sorted_order(n, len, 1);
    int64_t* sum = calloc((size_t)d, sizeof(int64_t));
    int64_t* sq = calloc((size_t)d, sizeof(int64_t));
    for (int64_t k = 0; k < n; ++k) {
      int best = 0;
      for (int i = 1; i < d; ++i)
        if (tolerance_less(sum[i], sq[i], sum[best], sq[best], tolerance_v)) best = i;
      const int64_t l = len[desc[k]];
      pk_push(&pk, best, desc[k]);
      sum[best] += l;
      sq[best] += l * l;
    }
    free(sum);
    free(sq);
    free(desc);
  } else { /* ConvTransformer :235-271 */
    int32_t* desc = sorted_order(n, len, 1);
    int64_t bound = 0;
    {
      packing g;
      pk_init(&g, d);
      distribute_min_sum(desc, n, len, &g);
      for (int b = 0; b < d; ++b) {
        int64_t s = 0;
        for (int64_t k = 0; k < g.count[b]; ++k) s += len[g.items[b][k]];
        if (s > bound) bound = s;
      }
      pk_free(&g);
    }
    int open = 1;
    int64_t consumed = 0;
    for (; consumed < n; ++consumed) {
      const int64_t l = len[desc[consumed]];
      if ((pk.count[open - 1] + 1) * l > bound) {
        if (open == d) break;
        ++open;
      }
      pk_push(&pk, open - 1, desc[consumed]);
    }
    distribute_min_sum(desc + consumed, n - consumed, len, &pk);
    free(desc);
  }

  /* never_worse: balancers.cpp:71-76 */
  const double algo = assemble_objective(&pk, kind, lambda, len);
  packing id;
  pk_init(&id, d);
  group_by_origin(n, origin, &id);
  const double ident = assemble_objective(&id, kind, lambda, len);
  const int take_identity = ident <= algo;
  export_packing(take_identity ? &id : &pk, kind, lambda, len, out);
  export_sources(d, n, len, origin, src_slot, out);
  if (objective) *objective = take_identity ? ident : algo;
  if (used_identity) *used_identity = take_identity;
  pk_free(&id);
  pk_free(&pk);
  free(src_slot);
  return 0;
}

int orc_identity(int kind, double lambda, int64_t tolerance_v, int d, int64_t n,
                 const int64_t* len, const int32_t* origin, orc_balance_out* out,
                 double* objective) {
  (void)tolerance_v;
  if (!out) out = &g_null_out;
  if (kind < 0 || kind > 3) return fail(4, "unknown policy kind");
  if (d < 1) return fail(1, "instance count must be >= 1");
  int32_t* src_slot = malloc((size_t)(n ? n : 1) * sizeof(int32_t));
  int rc = index_sources(d, n, len, origin, src_slot);
  if (rc) {
    free(src_slot);
    return rc;
  }
  packing id;
  pk_init(&id, d);
  group_by_origin(n, origin, &id);
  if (objective) *objective = assemble_objective(&id, kind, lambda, len);
  export_packing(&id, kind, lambda, len, out);
  export_sources(d, n, len, origin, src_slot, out);
  pk_free(&id);
  free(src_slot);
  return 0;
}

int orc_min_feasible_padded_bound(int d, int64_t n, const int64_t* len, const int32_t* origin,
                                  int64_t* bound) {
  if (d < 1) return fail(1, "instance count must be >= 1");
  if (n == 0) return fail(1, "padded balancing needs at least one item");
  int32_t* slot = malloc((size_t)n * sizeof(int32_t));
  int rc = index_sources(d, n, len, origin, slot);
  free(slot);
  if (rc) return rc;
  int32_t* asc = sorted_order(n, len, 0);
  *bound = padded_search(d, asc, n, len);
  free(asc);
  return 0;
}

int orc_padded_bound_feasible(int d, int64_t n, const int64_t* len, const int32_t* origin,
                              int64_t bound, int32_t* feasible) {
  if (d < 1) return fail(1, "instance count must be >= 1");
  if (n == 0) return fail(1, "padded balancing needs at least one item");
  int32_t* slot = malloc((size_t)n * sizeof(int32_t));
  int rc = index_sources(d, n, len, origin, slot);
  free(slot);
  if (rc) return rc;
  int32_t* asc = sorted_order(n, len, 0);
  if (bound < len[asc[n - 1]])
    *feasible = 0;
  else
    *feasible = least_batches(asc, n, len, bound, NULL) <= d;
  free(asc);
  return 0;
}

/* ---------------------------------------------------------- data movement */

void orc_volume_matrix(int d, int64_t n, const int64_t* len, const int32_t* origin,
                       const int32_t* dest_inst, int64_t* V) {
  memset(V, 0, (size_t)d * (size_t)d * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) V[(size_t)origin[i] * (size_t)d + dest_inst[i]] += len[i];
}

typedef struct {
  int64_t key; /* dest_inst * 2^31 + dest_slot */
  int32_t pos;
} dkey;
static int cmp_dkey(const void* a, const void* b) {
  const dkey* x = a;
  const dkey* y = b;
  return x->key < y->key ? -1 : (x->key > y->key);
}

int orc_layout(int d, int P, int64_t n, const int64_t* len, const int32_t* origin,
               const int32_t* dest_inst, const int32_t* dest_slot, int64_t* rank_src_off,
               int64_t* rank_dst_off, int64_t* pair_off, int64_t* send_tokens,
               int64_t* in_tokens, int64_t* out_tokens) {
  if (P < 1 || d % P != 0) return fail(1, "instance count must be divisible by rank count");
  const int c = d / P;
  int64_t* inst_in = calloc((size_t)d, sizeof(int64_t));
  int64_t* inst_out = calloc((size_t)d, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    inst_in[origin[i]] += len[i];
    inst_out[dest_inst[i]] += len[i];
  }
  /* per-instance base inside its rank buffer */
  int64_t* base_in = calloc((size_t)d, sizeof(int64_t));
  int64_t* base_out = calloc((size_t)d, sizeof(int64_t));
  for (int r = 0; r < P; ++r) {
    int64_t a = 0, b = 0;
    for (int i = r * c; i < (r + 1) * c; ++i) {
      base_in[i] = a;
      base_out[i] = b;
      a += inst_in[i];
      b += inst_out[i];
    }
    if (in_tokens) in_tokens[r] = a;
    if (out_tokens) out_tokens[r] = b;
  }
  /* source offsets: input order within origin */
  int64_t* run = calloc((size_t)d, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    rank_src_off[i] = base_in[origin[i]] + run[origin[i]];
    run[origin[i]] += len[i];
  }
  /* dest offsets + pair offsets: walk items in (dest_inst, dest_slot) order */
  dkey* keys = malloc((size_t)(n ? n : 1) * sizeof(dkey));
  for (int64_t i = 0; i < n; ++i) {
    keys[i].key = (int64_t)dest_inst[i] * 2147483648LL + dest_slot[i];
    keys[i].pos = (int32_t)i;
  }
  qsort(keys, (size_t)n, sizeof(dkey), cmp_dkey);
  memset(run, 0, (size_t)d * sizeof(int64_t));
  int64_t* pair_run = calloc((size_t)P * (size_t)P, sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) {
    const int32_t i = keys[k].pos;
    const int j = dest_inst[i];
    rank_dst_off[i] = base_out[j] + run[j];
    run[j] += len[i];
    const int r = origin[i] / c, q = j / c;
    pair_off[i] = pair_run[r * P + q];
    pair_run[r * P + q] += len[i];
  }
  if (send_tokens) memcpy(send_tokens, pair_run, (size_t)P * (size_t)P * sizeof(int64_t));
  free(pair_run);
  free(keys);
  free(run);
  free(base_in);
  free(base_out);
  free(inst_in);
  free(inst_out);
  return 0;
}

typedef struct {
  int64_t lo, hi;
  int c;
  const int64_t* len;
  const int32_t* origin;
  const int32_t* dest_inst;
  const int64_t* src;
  const int64_t* dst;
  size_t R;
  const uint8_t* const* in;
  uint8_t* const* out;
} copy_job;

static void* copy_worker(void* arg) {
  const copy_job* j = arg;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    const int r = j->origin[i] / j->c, q = j->dest_inst[i] / j->c;
    memcpy(j->out[q] + (size_t)j->dst[i] * j->R, j->in[r] + (size_t)j->src[i] * j->R,
           (size_t)j->len[i] * j->R);
  }
  return NULL;
}

int orc_dispatch_rows(int d, int P, int64_t n, const int64_t* len, const int32_t* origin,
                      const int32_t* dest_inst, const int64_t* rank_src_off,
                      const int64_t* rank_dst_off, size_t row_bytes,
                      const uint8_t* const* in_bufs, uint8_t* const* out_bufs, int nthreads) {
  if (P < 1 || d % P != 0) return fail(1, "instance count must be divisible by rank count");
  if (nthreads < 1) nthreads = 1;
  /* split items into nthreads ranges of roughly equal bytes */
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) total += len[i];
  pthread_t* th = malloc((size_t)nthreads * sizeof(pthread_t));
  copy_job* jobs = malloc((size_t)nthreads * sizeof(copy_job));
  int64_t i = 0, acc = 0;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t target = total * (t + 1) / nthreads;
    jobs[t] = (copy_job){i, i, d / P, len, origin, dest_inst, rank_src_off, rank_dst_off,
                         row_bytes, in_bufs, out_bufs};
    while (i < n && (acc < target || t == nthreads - 1)) acc += len[i++];
    jobs[t].hi = i;
  }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, copy_worker, &jobs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* Row content: each 16-byte chunk k of row t of an item = {tag, t*(R/16)+k}. */
void orc_fill_rows(int64_t n, const int64_t* len, const int64_t* tag, const int64_t* row_off,
                   size_t row_bytes, uint8_t* buf) {
  const int64_t W = (int64_t)(row_bytes / 16);
  for (int64_t i = 0; i < n; ++i) {
    int64_t* p = (int64_t*)(buf + (size_t)row_off[i] * row_bytes);
    for (int64_t w = 0; w < len[i] * W; ++w) {
      p[2 * w] = tag[i];
      p[2 * w + 1] = w;
    }
  }
}

/* ------------------------------------------------------- node-wise hosting */

/* inter_node_egress: topology.cpp:61-89 */
static void egress_of(int d, int c, const int64_t* V, const int32_t* hosting, int64_t* egress) {
  const int nodes = d / c;
  for (int n = 0; n < nodes; ++n) egress[n] = 0;
  for (int i = 0; i < d; ++i) {
    const int src = i / c;
    for (int b = 0; b < d; ++b)
      if (hosting[b] != src) egress[src] += V[(size_t)i * d + b];
  }
}

typedef struct {
  int nodes, d;
  int64_t* gain;       /* [nodes][d] */
  int64_t* node_total; /* [nodes] */
  int32_t* preferred;  /* [nodes][d] batches by descending gain (stable) */
  int32_t* order;      /* [d] branching order */
  int32_t* assignment; /* [d] */
  int32_t* remaining;  /* [nodes] */
  int64_t* gained;     /* [nodes] */
  int64_t best;
  int32_t* best_assignment;
  int64_t visited;
} hsearch;

static int64_t hs_optimistic(const hsearch* h, int n) { /* topology.cpp:114-126 */
  int64_t total = 0;
  int taken = 0;
  for (int k = 0; k < h->d; ++k) {
    if (taken == h->remaining[n]) break;
    const int b = h->preferred[(size_t)n * h->d + k];
    if (h->assignment[b] == -1) {
      total += h->gain[(size_t)n * h->d + b];
      ++taken;
    }
  }
  return total;
}

static int64_t hs_lower_bound(const hsearch* h) { /* :128-134 */
  int64_t bound = 0;
  for (int n = 0; n < h->nodes; ++n) {
    const int64_t v = h->node_total[n] - h->gained[n] - hs_optimistic(h, n);
    if (v > bound) bound = v;
  }
  return bound;
}

static int64_t hs_evaluate(const hsearch* h, const int32_t* hosting) { /* :136-141 */
  int64_t worst = INT64_MIN;
  for (int n = 0; n < h->nodes; ++n) {
    int64_t e = h->node_total[n];
    for (int b = 0; b < h->d; ++b)
      if (hosting[b] == n) e -= h->gain[(size_t)n * h->d + b];
    if (e > worst) worst = e;
  }
  return worst;
}

static void hs_offer(hsearch* h, const int32_t* hosting) { /* :143-149 */
  const int64_t v = hs_evaluate(h, hosting);
  if (v < h->best) {
    h->best = v;
    memcpy(h->best_assignment, hosting, (size_t)h->d * sizeof(int32_t));
  }
}

static const int64_t* g_cmp_gain;
static int cmp_gain_desc(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  if (g_cmp_gain[x] != g_cmp_gain[y]) return g_cmp_gain[x] > g_cmp_gain[y] ? -1 : 1;
  return x < y ? -1 : (x > y); /* stable: ties keep ascending index */
}

static void hs_dfs(hsearch* h, int depth) { /* :151-172 */
  ++h->visited;
  if (hs_lower_bound(h) >= h->best) return;
  if (depth == h->d) {
    hs_offer(h, h->assignment);
    return;
  }
  const int b = h->order[depth];
  int32_t cand[64];
  int nc = 0;
  for (int n = 0; n < h->nodes; ++n)
    if (h->remaining[n] > 0) cand[nc++] = n;
  /* stable sort of candidate nodes by descending gain for batch b */
  for (int i = 1; i < nc; ++i) { /* insertion sort = stable */
    const int32_t v = cand[i];
    int j = i - 1;
    while (j >= 0 && h->gain[(size_t)cand[j] * h->d + b] < h->gain[(size_t)v * h->d + b]) {
      cand[j + 1] = cand[j];
      --j;
    }
    cand[j + 1] = v;
  }
  for (int k = 0; k < nc; ++k) {
    const int n = cand[k];
    h->assignment[b] = n;
    h->remaining[n] -= 1;
    h->gained[n] += h->gain[(size_t)n * h->d + b];
    hs_dfs(h, depth + 1);
    h->gained[n] -= h->gain[(size_t)n * h->d + b];
    h->remaining[n] += 1;
    h->assignment[b] = -1;
  }
}

int orc_solve_hosting(int d, int c, const int64_t* V, int32_t* hosting, int64_t* per_node_egress,
                      int64_t* max_egress, int64_t* baseline_max, int64_t* nodes_visited) {
  if (d < 1 || c < 1) return fail(1, "topology needs at least one instance and one per node");
  if (d % c) return fail(1, "instance count must be divisible by instances per node");
  const int nodes = d / c;
  if (nodes > 64) return fail(1, "oracle hosting search limited to 64 nodes");
  hsearch h;
  memset(&h, 0, sizeof h);
  h.nodes = nodes;
  h.d = d;
  h.gain = calloc((size_t)nodes * d, sizeof(int64_t));
  h.node_total = calloc((size_t)nodes, sizeof(int64_t));
  for (int i = 0; i < d; ++i) {
    const int n = i / c;
    for (int b = 0; b < d; ++b) {
      h.gain[(size_t)n * d + b] += V[(size_t)i * d + b];
      h.node_total[n] += V[(size_t)i * d + b];
    }
  }
  h.preferred = malloc((size_t)nodes * d * sizeof(int32_t));
  for (int n = 0; n < nodes; ++n) {
    int32_t* list = h.preferred + (size_t)n * d;
    for (int b = 0; b < d; ++b) list[b] = b;
    g_cmp_gain = h.gain + (size_t)n * d;
    qsort(list, (size_t)d, sizeof(int32_t), cmp_gain_desc);
  }
  /* branching order: descending regret (top - second gain), stable (:219-238) */
  int64_t* regret = malloc((size_t)d * sizeof(int64_t));
  h.order = malloc((size_t)d * sizeof(int32_t));
  for (int b = 0; b < d; ++b) {
    int64_t top = 0, second = 0;
    for (int n = 0; n < nodes; ++n) {
      const int64_t g = h.gain[(size_t)n * d + b];
      if (g > top) {
        second = top;
        top = g;
      } else if (g > second) {
        second = g;
      }
    }
    regret[b] = top - second;
    h.order[b] = b;
  }
  g_cmp_gain = regret;
  qsort(h.order, (size_t)d, sizeof(int32_t), cmp_gain_desc);
  h.assignment = malloc((size_t)d * sizeof(int32_t));
  for (int b = 0; b < d; ++b) h.assignment[b] = -1;
  h.remaining = malloc((size_t)nodes * sizeof(int32_t));
  for (int n = 0; n < nodes; ++n) h.remaining[n] = c;
  h.gained = calloc((size_t)nodes, sizeof(int64_t));
  h.best = INT64_MAX;
  h.best_assignment = malloc((size_t)d * sizeof(int32_t));
  /* incumbents: identity, then greedy (:243-262) */
  int32_t* tmp = malloc((size_t)d * sizeof(int32_t));
  for (int b = 0; b < d; ++b) tmp[b] = b / c;
  hs_offer(&h, tmp);
  int32_t* room = malloc((size_t)nodes * sizeof(int32_t));
  for (int n = 0; n < nodes; ++n) room[n] = c;
  for (int k = 0; k < d; ++k) {
    const int b = h.order[k];
    int pick = -1;
    int64_t pick_gain = -1;
    for (int n = 0; n < nodes; ++n)
      if (room[n] > 0 && h.gain[(size_t)n * d + b] > pick_gain) {
        pick = n;
        pick_gain = h.gain[(size_t)n * d + b];
      }
    tmp[b] = pick;
    room[pick] -= 1;
  }
  hs_offer(&h, tmp);
  hs_dfs(&h, 0);
  memcpy(hosting, h.best_assignment, (size_t)d * sizeof(int32_t));
  int64_t* eg = per_node_egress ? per_node_egress : malloc((size_t)nodes * sizeof(int64_t));
  egress_of(d, c, V, hosting, eg);
  int64_t mx = INT64_MIN;
  for (int n = 0; n < nodes; ++n)
    if (eg[n] > mx) mx = eg[n];
  if (max_egress) *max_egress = mx;
  for (int b = 0; b < d; ++b) tmp[b] = b / c;
  egress_of(d, c, V, tmp, eg);
  int64_t bm = INT64_MIN;
  for (int n = 0; n < nodes; ++n)
    if (eg[n] > bm) bm = eg[n];
  if (baseline_max) *baseline_max = bm;
  if (nodes_visited) *nodes_visited = h.visited;
  if (!per_node_egress) free(eg);
  else egress_of(d, c, V, hosting, per_node_egress);
  free(room);
  free(tmp);
  free(regret);
  free(h.gain);
  free(h.node_total);
  free(h.preferred);
  free(h.order);
  free(h.assignment);
  free(h.remaining);
  free(h.gained);
  free(h.best_assignment);
  return 0;
}

/* topology.cpp:281-290: within a node, batches take instances in ascending batch order */
void orc_batch_to_instance(int d, int c, const int32_t* hosting, int32_t* batch_to_instance) {
  const int nodes = d / c;
  int32_t* next = malloc((size_t)nodes * sizeof(int32_t));
  for (int n = 0; n < nodes; ++n) next[n] = n * c;
  for (int b = 0; b < d; ++b) batch_to_instance[b] = next[hosting[b]]++;
  free(next);
}

/* ------------------------------------------------------- composed delivery */

typedef struct {
  int32_t slot;
  int32_t ex;
} arrival;
static int cmp_arrival(const void* a, const void* b) {
  const arrival* x = a;
  const arrival* y = b;
  return x->slot < y->slot ? -1 : (x->slot > y->slot);
}

void orc_backbone_targets(int d, int64_t E, const int32_t* llm_dest_inst,
                          const int32_t* llm_dest_slot, const int32_t* part_offset,
                          const int32_t* interleave_pos, int64_t n, const int32_t* item_part,
                          int32_t* dst_inst, int32_t* dst_slot) {
  /* part -> universe item */
  const int64_t parts = part_offset[E];
  int64_t* item_of = malloc((size_t)(parts ? parts : 1) * sizeof(int64_t));
  for (int64_t p = 0; p < parts; ++p) item_of[p] = -1;
  for (int64_t k = 0; k < n; ++k) item_of[item_part[k]] = k;
  /* per instance: examples by LLM slot (orchestrator.cpp:370-378) */
  arrival* arr = malloc((size_t)(E ? E : 1) * sizeof(arrival));
  for (int inst = 0; inst < d; ++inst) {
    int64_t m = 0;
    for (int64_t e = 0; e < E; ++e)
      if (llm_dest_inst[e] == inst) arr[m++] = (arrival){llm_dest_slot[e], (int32_t)e};
    qsort(arr, (size_t)m, sizeof(arrival), cmp_arrival);
    int slot = 0;
    for (int64_t k = 0; k < m; ++k) {
      const int32_t e = arr[k].ex;
      const int np = part_offset[e + 1] - part_offset[e];
      for (int q = 0; q < np; ++q) { /* parts in interleave order (:380-384) */
        for (int p = part_offset[e]; p < part_offset[e + 1]; ++p) {
          if (interleave_pos[p] != q) continue;
          const int64_t it = item_of[p];
          if (it >= 0) {
            dst_inst[it] = inst;
            dst_slot[it] = slot++;
          }
        }
      }
    }
  }
  free(arr);
  free(item_of);
}

typedef struct {
  int64_t key; /* inst * 2^31 + slot */
  int32_t pos;
} skey;
static int cmp_skey(const void* a, const void* b) {
  const skey* x = a;
  const skey* y = b;
  return x->key < y->key ? -1 : (x->key > y->key);
}

static int slot_offsets(int d, int64_t n, const int64_t* len, const int32_t* inst,
                        const int32_t* slot, int64_t* off, const char* what) {
  skey* k = malloc((size_t)(n ? n : 1) * sizeof(skey));
  for (int64_t i = 0; i < n; ++i) {
    if (inst[i] < 0 || inst[i] >= d) {
      free(k);
      return fail(1, "rearrangement references instance outside [0, d)");
    }
    k[i].key = (int64_t)inst[i] * 2147483648LL + slot[i];
    k[i].pos = (int32_t)i;
  }
  qsort(k, (size_t)n, sizeof(skey), cmp_skey);
  int64_t run = 0;
  for (int64_t j = 0; j < n; ++j) {
    const int32_t i = k[j].pos;
    const int new_inst = j == 0 || inst[k[j - 1].pos] != inst[i];
    if (!new_inst && k[j].key == k[j - 1].key) {
      free(k);
      return fail(1, what[0] == 'd' ? "rearrangement maps two items to one destination slot"
                                    : "rearrangement covers a slot twice");
    }
    const int expect = new_inst ? 0 : slot[k[j - 1].pos] + 1;
    if (slot[i] != expect) {
      free(k);
      return fail(1, what[0] == 'd' ? "destination slots are not dense"
                                    : "rearrangement covers a slot absent from the input batches");
    }
    if (new_inst) run = 0;
    off[i] = run;
    run += len[i];
  }
  free(k);
  return 0;
}

int orc_rearrange_offsets(int d, int64_t n, const int64_t* len, const int32_t* src_inst,
                          const int32_t* src_slot, const int32_t* dst_inst,
                          const int32_t* dst_slot, int64_t* src_off, int64_t* dst_off) {
  int rc = slot_offsets(d, n, len, dst_inst, dst_slot, dst_off, "dst");
  if (rc) return rc;
  return slot_offsets(d, n, len, src_inst, src_slot, src_off, "src");
}
