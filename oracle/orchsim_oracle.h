/*
 * orchsim_oracle.h -- CPU restatement of the reference Batch Post-Balancing
 * Dispatcher (OrchMLLM, arXiv 2503.23830; reference /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. The product path (paper_2503_23830_b200) never
 * links or calls it and fails loudly when its CUDA library is missing.
 *
 * Parity pinning: every function is checked against (a) the known answers in
 * the reference's own tests (proj/tests/test_balancers.cpp, test_core.cpp,
 * committed as tests/golden/reference_known_answers.json) and (b) the
 * reference library itself compiled unmodified into oracle/_ref (oracle/Makefile),
 * via committed fixtures tests/golden/ref_fixtures.npz (tests/golden/make_golden.py).
 *
 * Item arrays are indexed by INPUT POSITION (the order of the reference's
 * std::vector<SeqItem>); bins/instances by index in [0, d).
 *
 * Return codes (mirroring the reference's exception types):
 *   0 ok, 1 std::invalid_argument, 2 ConfigError, 4 std::logic_error.
 */
#ifndef ORCHSIM_ORACLE_H
#define ORCHSIM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_GREEDY_UNPADDED = 0, ORC_BINARY_PADDED = 1, ORC_QUADRATIC_TOLERANCE = 2,
       ORC_CONVTRANSFORMER = 3 };
enum { ORC_LINEAR_ONLY = 0, ORC_TRANSFORMER_QUADRATIC = 1, ORC_CONV_TRANSFORMER_PADDED = 2 };

typedef struct {
  int32_t* dest_inst;  /* [n] destination instance per input item        */
  int32_t* dest_slot;  /* [n] destination slot (position within dest bin) */
  int32_t* src_slot;   /* [n] source slot (position within origin batch)  */
  int64_t* src_off;    /* [n] token offset within origin batch            */
  int64_t* dst_off;    /* [n] token offset within destination batch       */
  int32_t* bin_count;  /* [d] items per destination batch                 */
  int64_t* bin_len;    /* [d] batch_length under the policy padding mode  */
  int64_t* bin_tokens; /* [d] unpadded token sum per destination batch    */
  double* bin_cost;    /* [d] cost() of each destination batch            */
} orc_balance_out;     /* every pointer may be NULL                        */

const char* orc_last_error(void);

/* balance() -- balancers.cpp:273-287 dispatching to :185-192 (greedy),
 * :194-208 (binary padded), :210-233 (quadratic tolerance), :235-271 (conv). */
int orc_balance(int kind, double lambda, int64_t tolerance_v, int d, int64_t n,
                const int64_t* len, const int32_t* origin, orc_balance_out* out,
                double* objective, int32_t* used_identity);

/* identity_arrangement() -- balancers.cpp:178-183 */
int orc_identity(int kind, double lambda, int64_t tolerance_v, int d, int64_t n,
                 const int64_t* len, const int32_t* origin, orc_balance_out* out,
                 double* objective);

/* balancers.cpp:289-307 */
int orc_min_feasible_padded_bound(int d, int64_t n, const int64_t* len, const int32_t* origin,
                                  int64_t* bound);
int orc_padded_bound_feasible(int d, int64_t n, const int64_t* len, const int32_t* origin,
                              int64_t bound, int32_t* feasible);

/* cost() of one batch -- core.cpp:91-118 */
int orc_cost(double alpha, double beta, int model_padded, int variant, int batch_padded,
             int64_t n, const int64_t* len, double* out);

/* stats_of() -- orchestrator.cpp:91-102 (max, sequential mean, max/mean) */
void orc_stats(int d, const double* costs, double* max, double* mean, double* ratio);

/* volume_matrix() -- topology.cpp:40-53: V[src_inst*d + dst_inst] += length */
void orc_volume_matrix(int d, int64_t n, const int64_t* len, const int32_t* origin,
                       const int32_t* dest_inst, int64_t* V);

/* Dispatch layout over P ranks, instances blocked c = d/P per rank
 * (instance i on rank i / c). Definitions:
 *  rank input buffer  = instances of the rank in order, each in source-slot order;
 *  rank output buffer = instances of the rank in order, each in dest-slot order;
 *  send segment r->q  = items with origin rank r, dest rank q, ordered by
 *                       (dest_inst, dest_slot); pair_off = token offset inside it.
 * Outputs: rank_src_off[n], rank_dst_off[n], pair_off[n] (tokens),
 *          send_tokens[P*P] (r-major), in_tokens[P], out_tokens[P]. */
int orc_layout(int d, int P, int64_t n, const int64_t* len, const int32_t* origin,
               const int32_t* dest_inst, const int32_t* dest_slot, int64_t* rank_src_off,
               int64_t* rank_dst_off, int64_t* pair_off, int64_t* send_tokens,
               int64_t* in_tokens, int64_t* out_tokens);

/* apply() (core.cpp:120-161) realised on token rows: for every item copy its
 * len*row_bytes bytes from in_bufs[origin rank] + rank_src_off*row_bytes to
 * out_bufs[dest rank] + rank_dst_off*row_bytes. Multi-threaded host memcpy
 * (the CPU dispatch baseline of BASELINE.md section 2). */
int orc_dispatch_rows(int d, int P, int64_t n, const int64_t* len, const int32_t* origin,
                      const int32_t* dest_inst, const int64_t* rank_src_off,
                      const int64_t* rank_dst_off, size_t row_bytes,
                      const uint8_t* const* in_bufs, uint8_t* const* out_bufs, int nthreads);

/* Deterministic token-row content: byte k of row t of item (example_id, part)
 * (used to fill input buffers so any misplaced row is detectable). */
void orc_fill_rows(int64_t n, const int64_t* len, const int64_t* tag, const int64_t* row_off,
                   size_t row_bytes, uint8_t* buf);

#ifdef __cplusplus
}
#endif
#endif
