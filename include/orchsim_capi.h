/*
 * orchsim_capi.h -- the drop-in C-ABI of the B200-native Batch Post-Balancing
 * Dispatcher (OrchMLLM, arXiv 2503.23830). This is the ONLY boundary between
 * host code and the sm_100a kernels: plain pointers and sizes, no C++ or
 * torch types. Implemented in paper_2503_23830_b200/csrc and exported by
 * paper_2503_23830_b200/lib/liborchsim_b200.so.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj). The C++ API of the reference
 * (the headers under include/orchsim in this repo, same names/signatures/exceptions) is
 * implemented on top of these calls in liborchsim_b200_host.so.
 *
 * Conventions
 *  - Item arrays are indexed by INPUT POSITION (the position of the SeqItem in
 *    the reference's std::vector<SeqItem>); instance/bin arrays by instance.
 *  - "d_" pointers are device memory (cudaMalloc / torch CUDA tensors),
 *    "h_" pointers are host memory. Streams are cudaStream_t passed as void*.
 *  - Device-pointer entry points are asynchronous on the given stream unless
 *    stated; validation errors found on the device are reported through the
 *    device-resident orch_summary (error, error_index) and make every later
 *    kernel of the same pipeline a no-op. Host-pointer entry points (_host)
 *    synchronise and return the reference's error class as a return code.
 *  - Return codes mirror the reference's exception types.
 */
#ifndef ORCHSIM_CAPI_H
#define ORCHSIM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORCH_OK 0
#define ORCH_INVALID_ARGUMENT 1 /* std::invalid_argument (balancers.cpp:30-33,157,196-241) */
#define ORCH_CONFIG_ERROR 2     /* orchsim::ConfigError  (core.cpp:178)                    */
#define ORCH_SIZE_CAP 3         /* orchsim::SizeCapError (balancers.cpp:383-387)           */
#define ORCH_LOGIC_ERROR 4      /* std::logic_error      (balancers.cpp:175,286)           */
#define ORCH_CUDA_ERROR 10      /* -> std::runtime_error                                   */
#define ORCH_NCCL_ERROR 11      /* -> std::runtime_error                                   */
#define ORCH_UNSUPPORTED 12     /* input beyond a documented device limit      */

/* PolicyKind (balancers.hpp:12), same numbering. */
#define ORCH_GREEDY_UNPADDED 0
#define ORCH_BINARY_PADDED 1
#define ORCH_QUADRATIC_TOLERANCE 2
#define ORCH_CONVTRANSFORMER 3
/* CostVariant (core.hpp:21), same numbering. */
#define ORCH_LINEAR_ONLY 0
#define ORCH_TRANSFORMER_QUADRATIC 1
#define ORCH_CONV_TRANSFORMER_PADDED 2

/* Device limits of this build (checked; ORCH_UNSUPPORTED beyond them). */
#define ORCH_MAX_INSTANCES 4096        /* d: bins live in one CTA's shared memory */
#define ORCH_MAX_ITEMS 16777215        /* n < 2^24                                */
#define ORCH_MAX_LENGTH 4294967295LL   /* per-item length < 2^32                  */

/* Per-device context. Device-pointer calls on different streams get separate
 * workspaces, so one context may feed several streams (16 at a time; a call on
 * a 17th stream first synchronises the device and recycles a workspace). A
 * context is used by one host thread at a time (not thread-safe). */
typedef struct orch_ctx orch_ctx;
typedef struct orch_comm orch_comm; /* NCCL communicator over the ranks of one box               */
typedef struct orch_window orch_window; /* a row buffer every rank can store into (below)    */

/* BalancePolicy (balancers.hpp:14-18). */
typedef struct {
  int32_t kind;
  int32_t reserved;
  int64_t tolerance_v;
  double lambda;
} orch_policy;

/* CostModel (core.hpp:63-68). padded: PaddingMode::Padded == 1. */
typedef struct {
  double alpha;
  double beta;
  int32_t padded;
  int32_t variant;
} orch_cost_model;

/* Device-resident result summary of one balance call. */
typedef struct {
  double objective;          /* BalanceResult::objective_value                     */
  double algo_objective;     /* objective of the balancer's own packing             */
  double identity_objective; /* objective of the identity arrangement               */
  double pre_max, pre_mean, pre_ratio;    /* stats_of (orchestrator.cpp:91-102) of the  */
  double post_max, post_mean, post_ratio; /* origin / destination batches, policy model */
  int64_t bound;             /* BinaryPadded: the minimal feasible bound; Conv: seeding bound */
  int64_t error_index;       /* first offending input position, or INT64_MAX       */
  int32_t error;             /* 0 or an ORCH_* code raised on the device           */
  int32_t used_identity;     /* never_worse (balancers.cpp:71-76) took the identity */
  int64_t rounds;            /* greedy rounds executed (diagnostic)                 */
} orch_summary;

/* Flat BalanceResult (balancers.hpp:20-24): every pointer is device memory,
 * caller-owned; any may be NULL except where a later call needs it. */
typedef struct {
  int32_t* dest_inst;  /* [n] Rearrangement dest instance      */
  int32_t* dest_slot;  /* [n] Rearrangement dest slot          */
  int32_t* src_slot;   /* [n] source slot (index_sources)      */
  int64_t* src_off;    /* [n] token offset in origin batch     */
  int64_t* dst_off;    /* [n] token offset in dest batch       */
  int32_t* bin_count;  /* [d] new_batches[i].items.size()      */
  int64_t* bin_len;    /* [d] batch_length(new_batches[i])     */
  int64_t* bin_tokens; /* [d] unpadded_length(new_batches[i])  */
  double* bin_cost;    /* [d] cost(policy model, new_batches[i]) */
  int32_t* bin_offset; /* [d+1] CSR of new_batches              */
  int32_t* bin_member; /* [n] input positions, (dest_inst, dest_slot) order */
  int32_t* src_offset; /* [d+1] CSR of the origin batches (batches_from_items)     */
  int32_t* src_member; /* [n] input positions, (origin, src_slot) order            */
  orch_summary* summary; /* device, required */
} orch_balance_out;

/* Rank-level dispatch layout: P ranks, instance i
 * on rank i / (d/P). All device memory. */
typedef struct {
  int64_t* rank_src_off; /* [n] row offset of the item in its origin rank's input buffer */
  int64_t* rank_dst_off; /* [n] row offset of the item in its dest rank's output buffer   */
  int64_t* pair_off;     /* [n] row offset inside the (origin rank -> dest rank) segment  */
  int64_t* send_rows;    /* [P*P] rows from rank r to rank q (r-major)                    */
  int64_t* send_displ;   /* [P*P] row offset of segment r->q in rank r's send buffer      */
  int64_t* recv_displ;   /* [P*P] row offset of segment r->q in rank q's recv buffer (q-major) */
  int64_t* in_rows;      /* [P] rows of each rank's input buffer                           */
  int64_t* out_rows;     /* [P] rows of each rank's output buffer                          */
  int32_t* status;       /* [1] 0, or ORCH_INVALID_ARGUMENT when a buffer capacity was short */
} orch_layout_out;

/* ------------------------------------------------------------- context */
int orch_ctx_create(int device, orch_ctx** out);
void orch_ctx_destroy(orch_ctx* ctx);
/* Message of the last failing call on this host thread. */
const char* orch_last_error(void);
int orch_version(void);
/* Number of kernels this library launched so far on ctx (for launch accounting). */
int64_t orch_ctx_launches(const orch_ctx* ctx);

/* ------------------------------------------------------------- balance */
/* balance(policy, d, items)             balancers.hpp:53  (balancers.cpp:273-287)
 * identity_arrangement(policy, d, items) balancers.hpp:59 (balancers.cpp:178-183)
 * when identity_only != 0.                                                     */
int orch_balance(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                 const int64_t* d_len, const int32_t* d_origin, int32_t identity_only,
                 const orch_balance_out* out, void* stream);

/* orch_balance followed by orch_layout for one rank (P = 1), in one launch when
 * the phase fits the single-CTA balance kernel (n <= 4096, d <= 64), else the
 * two calls. Same outputs as the pair. Every layout array is required. */
int orch_balance_layout1(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                         const int64_t* d_len, const int32_t* d_origin, int32_t identity_only,
                         const orch_balance_out* out, const orch_layout_out* layout,
                         void* stream);

/* Host-buffer variant: copies h_len/h_origin in, runs orch_balance, copies
 * the flat result out (any h_ output may be NULL) and synchronises. Returns
 * the reference's error class. */
int orch_balance_host(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                      const int64_t* h_len, const int32_t* h_origin, int32_t identity_only,
                      int32_t* h_dest_inst, int32_t* h_dest_slot, int64_t* h_dst_off,
                      int32_t* h_bin_count, double* h_bin_cost, orch_summary* h_summary,
                      void* stream);

/* min_feasible_padded_bound  balancers.hpp:64 (balancers.cpp:289-296)
 * padded_bound_feasible      balancers.hpp:68 (balancers.cpp:298-307)
 * Host buffers, synchronous. */
int orch_min_feasible_padded_bound_host(orch_ctx* ctx, int32_t d, int64_t n,
                                        const int64_t* h_len, const int32_t* h_origin,
                                        int64_t* h_bound, void* stream);
int orch_padded_bound_feasible_host(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* h_len,
                                    const int32_t* h_origin, int64_t bound, int32_t* h_feasible,
                                    void* stream);

/* oracle_optimal (balancers.hpp:84, balancers.cpp:380-413): exhaustive
 * minimum of the max batch cost over canonical assignments, brute force on
 * the device; returns the first optimum in the reference's depth-first order.
 * ORCH_SIZE_CAP above the caller's caps, ORCH_UNSUPPORTED above d <= 4,
 * d^n <= 2^36. Host buffers, synchronous. */
int orch_oracle_optimal_host(orch_ctx* ctx, const orch_cost_model* model, int32_t d, int64_t n,
                             const int64_t* h_len, int32_t max_items, int32_t max_instances,
                             int32_t* h_assignment, double* h_objective, void* stream);

/* ---------------------------------------------------------- cost model */
/* cost(model, batch) over many batches at once (core.cpp:91-118) plus
 * stats_of (orchestrator.cpp:91-102): batches given as CSR over input
 * positions. d_stats = {max, mean, ratio}. Requires model->padded == batch
 * padding (the caller's MiniBatch mode), else ORCH_INVALID_ARGUMENT. */
int orch_batch_costs(orch_ctx* ctx, const orch_cost_model* model, int32_t batch_padded,
                     int32_t d, int64_t n, const int64_t* d_len, const int32_t* d_bin_offset,
                     const int32_t* d_bin_member, double* d_cost, double* d_stats, void* stream);

/* Host-buffer variant of orch_batch_costs (synchronous); h_stats may be NULL. */
int orch_batch_costs_host(orch_ctx* ctx, const orch_cost_model* model, int32_t batch_padded,
                          int32_t d, int64_t n, const int64_t* h_len,
                          const int32_t* h_bin_offset, const int32_t* h_bin_member,
                          double* h_cost, double* h_stats, void* stream);

/* batches_from_items (core.cpp:183-199): CSR of the origin batches. */
int orch_group_by_origin(orch_ctx* ctx, int32_t d, int64_t n, const int32_t* d_origin,
                         int32_t* d_bin_offset, int32_t* d_bin_member, void* stream);

/* encode_lengths + interleaved_length (core.cpp:163-181), vectorised: parts
 * of example e are [part_offset[e], part_offset[e+1]); encoded = ceil(meta /
 * rate[modality]) with rate >= 1 (else ORCH_CONFIG_ERROR, host-checked);
 * d_interleaved[e] = sum of encoded parts. */
int orch_encode_lengths(orch_ctx* ctx, int64_t num_examples, const int32_t* d_part_offset,
                        const int32_t* d_modality, const int64_t* d_meta_len,
                        int32_t num_modalities, const int64_t* h_rates, int64_t* d_encoded,
                        int64_t* d_interleaved, void* stream);

/* ------------------------------------------------ node-wise hosting */
/* solve_hosting (topology.hpp:71, topology.cpp:179-265) on a host volume
 * matrix h_V[d*d] with c instances per node: exact (the reference's answer,
 * including its tie-breaking) by a parallel two-pass branch and bound on the
 * device; ORCH_UNSUPPORTED when d > ORCH_MAX_INSTANCES or d/c > 32 nodes (d > 64:
 * search tables and DFS stacks in global memory). h_info (optional,
 * [4]) as orch_nodewise's d_info below, except h_info[3]: the reference's own
 * nodes_visited (topology.cpp:150,263), replayed on the device from its chain of
 * improving leaves (-1 if that replay exceeds 2^31 nodes; h_info == NULL skips
 * it). A search that exceeds 2^31 visited nodes returns ORCH_UNSUPPORTED
 * (h_hosting then holds the incumbent). */
int orch_solve_hosting_host(orch_ctx* ctx, int32_t d, int32_t c, const int64_t* h_V,
                            int32_t* h_hosting, int64_t* h_info, void* stream);

/* inter_node_egress (topology.hpp:68, topology.cpp:61-89) of a given hosting on
 * the device: h_egress[n] = sum of V[i][b] over source instances i on node n
 * (= i / c) and batches b hosted elsewhere (h_hosting[b] != n), for any node
 * count d / c. The caller validates the hosting (the C++ adapter throws as the
 * reference does); hosting entries are taken as node indices in [0, d / c). */
int orch_inter_node_egress_host(orch_ctx* ctx, int32_t d, int32_t c, const int64_t* h_V,
                                const int32_t* h_hosting, int64_t* h_egress, void* stream);

/* nodewise_rearrange (topology.hpp:87, topology.cpp:267-303) applied in place
 * to a balance result: volume matrix of the result, optimal hosting, then
 * destination batch b is relabelled batch_to_instance[b] (dest_inst and the
 * per-batch arrays / CSR permuted; slots and offsets unchanged). With one
 * rank per node this is the GPU-wise hosting that cuts NVLink egress.
 * d_info = {max_egress, baseline_max_egress (identity hosting), leaf_used
 * (1: a search leaf beat the identity/greedy incumbents, 0: incumbent,
 * -1: visit budget exhausted, incumbent kept), nodes visited by the device
 * search (its parallel order prunes differently from the reference's
 * sequential DFS, so this is not the reference's count)}. */
int orch_nodewise(orch_ctx* ctx, int32_t d, int32_t c, int64_t n, const int64_t* d_len,
                  const int32_t* d_origin, const orch_balance_out* bal, int32_t* d_hosting,
                  int32_t* d_batch_to_instance, int64_t* d_info, void* stream);

/* -------------------------------------------------- composed delivery */
/* Any rearrangement of n items, given per item as (src_inst, src_slot) ->
 * (dst_inst, dst_slot), laid out as a flat balance result (dest arrays,
 * token offsets, both CSRs, bin_count/bin_tokens) so orch_layout and
 * orch_dispatch / orch_put move its rows, with d_src_inst as the origin array.
 * Validated like Rearrangement + apply (core.cpp:14-43, 120-161): instances in
 * range, source and destination slots dense and unique per instance; a
 * violation sets out->summary->error = ORCH_INVALID_ARGUMENT.
 * compose(outer, inner) (exchange.cpp:125-137) of flat rearrangements is this
 * call with inner's destination as the source and outer's destination as the
 * target; inverse (exchange.cpp:115-123) swaps the two sides. */
int orch_rearrange(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* d_len,
                   const int32_t* d_src_inst, const int32_t* d_src_slot,
                   const int32_t* d_dst_inst, const int32_t* d_dst_slot,
                   const orch_balance_out* out, void* stream);

/* backbone_mapping_for (orchestrator.cpp:367-388): the backbone destination of
 * every item of an encoder universe. Examples e in [0, E) with LLM result
 * (d_llm_dest_inst, CSR d_llm_bin_offset / d_llm_bin_member from orch_balance);
 * parts of example e are [part_offset[e], part_offset[e+1]) with interleave
 * position d_interleave_pos[part]; universe items are the global part indices
 * d_item_part[n]. Out: d_dst_inst[n], d_dst_slot[n]. */
int orch_backbone_targets(orch_ctx* ctx, int32_t d, int64_t E, const int32_t* d_llm_dest_inst,
                          const int32_t* d_llm_bin_offset, const int32_t* d_llm_bin_member,
                          const int32_t* d_part_offset, const int32_t* d_interleave_pos,
                          int64_t num_parts, int64_t n, const int32_t* d_item_part,
                          int32_t* d_dst_inst, int32_t* d_dst_slot, void* stream);

/* ------------------------------------------------------ layout / movement */
/* volume_matrix (topology.cpp:40-53): d_V[d*d] (src-major) token volumes. */
int orch_volume_matrix(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* d_len,
                       const int32_t* d_origin, const int32_t* d_dest_inst, int64_t* d_V,
                       void* stream);

/* Host-buffer variant of orch_volume_matrix (synchronous). */
int orch_volume_matrix_host(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* h_len,
                            const int32_t* h_origin, const int32_t* h_dest_inst, int64_t* h_V,
                            void* stream);

/* ExchangeCostReport (exchange.hpp:27-35) without its per-node vector. */
typedef struct {
  double modeled_time;
  int64_t total_inter_volume;
  int64_t total_intra_volume;
  int64_t local_volume;
  int64_t peak_resident_volume;
  int32_t bottleneck; /* Bottleneck (exchange.hpp:25): 0 None, 1 IntraNode, 2 InterNode */
  int32_t stale;      /* 1: d_V is not the volume matrix of the given items */
} orch_exchange_cost;

/* simulate_exchange's cost report (exchange.cpp:64-111) as one device
 * reduction over the volume matrix d_V[d*d] (src-major; the plan's
 * per_pair_volumes) for c instances per node: inter / intra / local volume,
 * per-node egress (d_per_node_egress[d/c]), peak resident volume, modeled time
 * (alltoall_constant x the slowest instance's inter/inter_bw + intra/intra_bw,
 * mode 0 = AllToAll) or the ring bound (d-1) max L / inter_bw (mode 1 =
 * AllGather, needs d_batch_len[d] = batch_length of the input batches) and
 * the bottleneck, bit-identical to the reference. With items (n >= 0, d_len,
 * d_src_inst, d_dst_inst: the plan's rearrangement) the plan is also checked
 * against their volume matrix (exchange.cpp:57-60): d_report->stale.
 * Topology errors as validate_topology (topology.cpp:12-22). */
int orch_exchange_report(orch_ctx* ctx, int32_t d, int32_t c, double intra_bw, double inter_bw,
                         double alltoall_constant, int32_t mode, const int64_t* d_V,
                         const int64_t* d_batch_len, int64_t n, const int64_t* d_len,
                         const int32_t* d_src_inst, const int32_t* d_dst_inst,
                         int64_t* d_per_node_egress, orch_exchange_cost* d_report, void* stream);
/* Host-buffer variant (synchronous): a stale plan returns ORCH_INVALID_ARGUMENT
 * with the reference's message. */
int orch_exchange_report_host(orch_ctx* ctx, int32_t d, int32_t c, double intra_bw,
                              double inter_bw, double alltoall_constant, int32_t mode,
                              const int64_t* h_V, const int64_t* h_batch_len, int64_t n,
                              const int64_t* h_len, const int32_t* h_src_inst,
                              const int32_t* h_dst_inst, int64_t* h_per_node_egress,
                              orch_exchange_cost* h_report, void* stream);
/* make_exchange_plan's AllGather volumes (exchange.cpp:17-28):
 * V[i][j] = batch_len[i] for j != i, 0 on the diagonal. */
int orch_allgather_volumes(orch_ctx* ctx, int32_t d, const int64_t* d_batch_len, int64_t* d_V,
                           void* stream);
int orch_allgather_volumes_host(orch_ctx* ctx, int32_t d, const int64_t* h_batch_len,
                                int64_t* h_V, void* stream);

/* Send/recv layout of the exchange (make_exchange_plan, exchange.cpp:10-32,
 * realised on ranks): offsets, per-pair counts. Needs the balance result's
 * dest_inst, src_off, dst_off, bin_offset, bin_member. */
int orch_layout(orch_ctx* ctx, int32_t d, int32_t nranks, int64_t n, const int64_t* d_len,
                const int32_t* d_origin, const orch_balance_out* bal,
                const orch_layout_out* layout, void* stream);

/* The data movement of simulate_exchange (exchange.cpp:62 = apply,
 * core.cpp:120-161) realised on token rows of row_bytes bytes (a multiple of
 * 16; bf16 d_model=4096 -> 8192). Buffers are this rank's:
 *   d_in   [in_cap rows]   origin batches of the rank's instances, in order
 *   d_out  [out_cap rows]  destination batches of the rank's instances
 *   d_send / d_recv        off-rank segments (layout send_displ / recv_displ)
 * A rank buffer larger than its capacity sets layout->status and moves
 * nothing. Split into the three stages of the exchange: */

/* pack: rows of this rank's items -> d_out (staying on the rank) or d_send. */
int orch_pack(orch_ctx* ctx, int32_t rank, int32_t nranks, int32_t d, int64_t n,
              const int64_t* d_len, const int32_t* d_origin, const orch_balance_out* bal,
              const orch_layout_out* layout, size_t row_bytes, const void* d_in, int64_t in_cap,
              void* d_out, int64_t out_cap, void* d_send, int64_t send_cap, void* stream);
/* exchange: one grouped ncclSend/ncclRecv over all peers (reads the per-peer
 * counts on the host: one stream synchronisation). */
int orch_exchange(orch_ctx* ctx, orch_comm* comm, const orch_layout_out* layout,
                  size_t row_bytes, const void* d_send, void* d_recv, int64_t recv_cap,
                  void* stream);
/* unpack: received rows -> their destination slots in d_out. */
int orch_unpack(orch_ctx* ctx, int32_t rank, int32_t nranks, int32_t d, int64_t n,
                const int64_t* d_len, const int32_t* d_origin, const orch_balance_out* bal,
                const orch_layout_out* layout, size_t row_bytes, const void* d_recv,
                void* d_out, int64_t out_cap, void* stream);
/* pack + exchange + unpack. comm == NULL: one rank, every item moves in one
 * fused pass d_in -> d_out (no send/recv buffers, no synchronisation). */
int orch_dispatch(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                  const int32_t* d_origin, const orch_balance_out* bal,
                  const orch_layout_out* layout, size_t row_bytes, const void* d_in,
                  int64_t in_cap, void* d_out, int64_t out_cap, void* d_send, int64_t send_cap,
                  void* d_recv, int64_t recv_cap, void* stream);

/* The NCCL exchange with its counts read from a pinned host mirror of the
 * layout (orch_xplan), filled on the METADATA stream right after orch_layout:
 * orch_dispatch_nccl waits for that copy only (an event), never for the data
 * stream, so the host issues step k+1's exchange while step k's rows still
 * move. Two forms:
 *  - staged (d_send, d_recv given): one pass packs the rows that stay into
 *    d_out and the off-rank rows into per-peer segments of d_send; one grouped
 *    ncclSend/ncclRecv per peer; one pass unpacks d_recv into d_out;
 *  - direct (d_send == NULL): every off-rank item is one ncclSend from its run
 *    in d_in to its run in the peer's d_out (no staging passes; NCCL pairs a
 *    peer's sends and receives in issue order, item order on both sides), the
 *    rows that stay move with one copy kernel. Fast only for few, large items
 *    (every NCCL operation has a fixed cost). */
typedef struct orch_xplan orch_xplan;
int orch_xplan_create(orch_ctx* ctx, int64_t max_n, int32_t nranks, orch_xplan** out);
void orch_xplan_destroy(orch_xplan* x);
/* Enqueue on `stream` the copy of the layout into the plan's pinned mirror
 * (the arrays must stay valid until orch_dispatch_nccl has run). */
int orch_xplan_fetch(orch_ctx* ctx, orch_xplan* x, int32_t d, int64_t n, const int64_t* d_len,
                     const int32_t* d_origin, const orch_balance_out* bal,
                     const orch_layout_out* layout, void* stream);
int orch_dispatch_nccl(orch_ctx* ctx, orch_comm* comm, orch_xplan* x, size_t row_bytes,
                       const void* d_in, int64_t in_cap, void* d_out, int64_t out_cap,
                       void* d_send, int64_t send_cap, void* d_recv, int64_t recv_cap,
                       void* stream);
/* ncclCommRegister / ncclCommDeregister of a row buffer (zero-copy transfers
 * where NCCL supports them for send/recv). */
int orch_comm_register(orch_comm* comm, void* ptr, size_t bytes, void** handle);
int orch_comm_deregister(orch_comm* comm, void* handle);

/* ----------------------------------------------------------- NCCL comm */
/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the caller. */
int orch_comm_unique_id(unsigned char* h_id128);
int orch_comm_create(int32_t nranks, int32_t rank, const unsigned char* h_id128,
                     orch_comm** out);
void orch_comm_destroy(orch_comm* comm);
int32_t orch_comm_rank(const orch_comm* comm);
int32_t orch_comm_size(const orch_comm* comm);

/* Barrier over the communicator on a stream (a 1-int ncclAllReduce). */
int orch_barrier(orch_comm* comm, void* stream);

/* A row buffer every rank can store into over NVLink (cudaMalloc + CUDA IPC
 * handles exchanged over the communicator). Collective: every rank calls it
 * with the same size; the sizes are exchanged with the handles and a mismatch
 * fails on every rank (ORCH_INVALID_ARGUMENT) before any peer is mapped.
 *
 * One step of a put exchange, on every rank (the protocol INTEGRATION.md 2
 * spells out):
 *   orch_put / orch_put_at      (any number, into disjoint window ranges)
 *   orch_window_barrier         every rank's puts of the step have landed here
 *   ... consumers read this rank's window ...
 *   orch_window_release         after the last consumer kernel (stream order)
 * The first put after the e-th barrier (per stream) is preceded by a one-warp
 * kernel that waits, on the device, until every rank has released e steps, so
 * the next step's puts never overwrite rows a peer is still reading
 * (write-after-read); the wait holds one warp, not the put's CTAs, so the
 * consumers keep the SMs they need. Waits give up after ~4 s: the barrier or
 * the acquire sets the window status, and a put whose acquire timed out sets
 * layout->status to ORCH_CUDA_ERROR and stores nothing. */
int orch_window_create(orch_ctx* ctx, orch_comm* comm, size_t bytes, orch_window** out);
/* The same window in NCCL symmetric memory instead of CUDA IPC: ncclMemAlloc +
 * ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC) (NCCL >= 2.28), the peers'
 * addresses from the device API's ncclGetPeerPointer. Puts, barrier, release
 * and destroy are unchanged. Collective over the communicator. */
int orch_window_create_nccl(orch_ctx* ctx, orch_comm* comm, size_t bytes, orch_window** out);
void* orch_window_ptr(const orch_window* w);
size_t orch_window_bytes(const orch_window* w);
int orch_window_destroy(orch_window* w); /* collective */
/* Barrier through the window's peer memory (one 1-warp kernel, no NCCL):
 * lane q stores this rank's call count into rank q's arrival slot with a
 * system-scope release, then waits for every rank's store into its own slots
 * (acquire). Everything earlier on `stream` (e.g. this step's puts) is visible
 * to every rank once its barrier returns. Collective: every rank calls it the
 * same number of times on the same window. */
int orch_window_barrier(orch_ctx* ctx, orch_window* w, void* stream);
/* The rows of the oldest unreleased barrier-closed step have been consumed on
 * this rank (everything earlier on `stream` is done reading the window): one
 * 1-warp kernel stores the release count into every rank's window. */
int orch_window_release(orch_ctx* ctx, orch_window* w, void* stream);
/* 0, or ORCH_CUDA_ERROR when a barrier on this window timed out (synchronous
 * read; call after the streams that used the window have been synchronised). */
int orch_window_status(const orch_window* w, int32_t* h_status);

/* Fused pack + put exchange: every item's rows are
 * read once from this rank's d_in and stored directly at their final
 * destination-slot offset in the destination rank's window (TMA bulk stores
 * over NVLink to peer memory); orch_window_barrier on the stream then
 * publishes the windows. Same result bytes as orch_dispatch. The caller
 * releases the window (orch_window_release) once the rows are consumed. */
int orch_dispatch_put(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                      const int32_t* d_origin, const orch_balance_out* bal,
                      const orch_layout_out* layout, size_t row_bytes, const void* d_in,
                      int64_t in_cap, orch_window* out_win, void* stream);
/* The put alone (no barrier): several exchanges (e.g. the phases of one
 * iteration) can share one window barrier. orch_put_at stores this exchange's
 * output at byte offset win_offset (a multiple of 16) of every rank's window,
 * so the phases of a step share one window, one barrier and one release. */
int orch_put(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
             const int32_t* d_origin, const orch_balance_out* bal,
             const orch_layout_out* layout, size_t row_bytes, const void* d_in, int64_t in_cap,
             orch_window* out_win, void* stream);
int orch_put_at(orch_ctx* ctx, orch_comm* comm, int32_t d, int64_t n, const int64_t* d_len,
                const int32_t* d_origin, const orch_balance_out* bal,
                const orch_layout_out* layout, size_t row_bytes, const void* d_in,
                int64_t in_cap, orch_window* out_win, size_t win_offset, void* stream);

/* ------------------------------------------ single-process rank emulation */
/* P ranks in one process on one device (tests and single-GPU integration
 * checks): a loopback communicator carries rank and size but no NCCL (the
 * NCCL entry points refuse it), and orch_window_create_local makes the P
 * windows of such communicators at once, each rank's peers being the other
 * windows' device buffers. Puts, window barriers, releases and the gather
 * window then run the same kernels as across GPUs; each emulated rank needs
 * its own stream (a barrier waits for the other ranks' kernels). A rank's
 * window lives on the device current when its loopback communicator was
 * created, so one process can also drive P GPUs (peer access over NVLink). */
int orch_comm_create_local(int32_t nranks, int32_t rank, orch_comm** out);
int orch_window_create_local(orch_ctx* ctx, orch_comm* const* comms, int32_t nranks, size_t bytes,
                             orch_window** out /* [nranks] */);

/* gather_lengths (exchange.cpp:34-47) realised as ncclAllGather: every rank
 * contributes its local items (global input position, length, origin) and
 * receives the global arrays scattered into input order. Local counts are
 * padded to max_local (>= every rank's local_n). */
int orch_allgather_items(orch_ctx* ctx, orch_comm* comm, int64_t local_n, int64_t max_local,
                         const int64_t* d_local_pos, const int64_t* d_local_len,
                         const int32_t* d_local_origin, int64_t n, int64_t* d_len,
                         int32_t* d_origin, void* stream);

/* gather_lengths (exchange.cpp:34-47) over NVLink peer memory, for the
 * metadata path of a pipelined step: one single-CTA kernel per call stores
 * this rank's records (length, origin) at their global input positions in
 * every rank's gather window, raises this rank's arrival flag there, waits for
 * all P flags, copies the window into d_len / d_origin and acknowledges, so
 * the next call may overwrite the window. Same result as
 * orch_allgather_items; no NCCL kernel, no ring. Calls are collective and
 * numbered: every rank makes them in the same order. A position outside
 * [0, n) sets *d_status = ORCH_INVALID_ARGUMENT (d_status optional); a peer
 * that does not arrive within ~4 s sets ORCH_CUDA_ERROR instead of hanging. */
typedef struct orch_gather_window orch_gather_window;
int orch_gather_window_create(orch_ctx* ctx, orch_comm* comm, int64_t max_n,
                              orch_gather_window** out);
/* The same in NCCL symmetric memory (orch_window_create_nccl). Collective. */
int orch_gather_window_create_nccl(orch_ctx* ctx, orch_comm* comm, int64_t max_n,
                                   orch_gather_window** out); /* collective */
int orch_gather_window_destroy(orch_gather_window* g);   /* collective */
/* P gather windows of loopback communicators (see orch_window_create_local). */
int orch_gather_window_create_local(orch_ctx* ctx, orch_comm* const* comms, int32_t nranks,
                                    int64_t max_n, orch_gather_window** out /* [nranks] */);
/* Diagnostics: %globaltimer (ns) at the stages of the last 8 calls, [epoch % 8][k]:
 * k = 0 start, 1 window free, 2 records stored + fenced, 3 all ranks arrived, 4 end. */
int orch_gather_window_stamps(const orch_gather_window* g, uint64_t* h_out64);
int orch_allgather_items_put(orch_ctx* ctx, orch_gather_window* g, int64_t local_n,
                             const int64_t* d_local_pos, const int64_t* d_local_len,
                             const int32_t* d_local_origin, int64_t n, int64_t* d_len,
                             int32_t* d_origin, int32_t* d_status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ORCHSIM_CAPI_H */
