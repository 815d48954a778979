// Host orchestration of the balance pipeline (C-ABI orch_balance*): a short
// chain of sm_100a kernels on one stream, no host synchronisation.
//
//   K1 k_validate          index_sources checks + sort keys   (balancers.cpp:25-37)
//   radix sort by origin   -> identity order (batches_from_items, core.cpp:183-199)
//   K2 k_ident_*           source slots / offsets, origin batches
//   radix sort by length   -> descending (stable) order        (balancers.cpp:78-88)
//   K4 greedy              distribute_min_sum                  (balancers.cpp:92-107)
//   K5 padded search       Alg.2 GetLeastBatches + search      (balancers.cpp:111-143)
//   K6 quadratic tolerance champion scan                       (balancers.cpp:210-233)
//   K7 k_bin_cost/k_decide cost(), objective, never_worse      (balancers.cpp:43-76)

#include <algorithm>
#include <cstring>
#include <string>

#include "balance_kernels.cuh"
#include "balance_small.cuh"
#include "greedy_lpt.cuh"
#include "plan.cuh"
#include "radix.cuh"

namespace orchb {

namespace {

constexpr int kThreads = 256;

template <class F>
void launch(orch_ctx* ctx, F&& f) {
  f();
  ++ctx->launches;
}

__global__ void k_init(orch_summary* s, Flags* f) {
  s->objective = s->algo_objective = s->identity_objective = 0.0;
  s->pre_max = s->pre_mean = s->post_max = s->post_mean = 0.0;
  s->pre_ratio = s->post_ratio = 1.0;
  s->bound = 0;
  s->error_index = INT64_MAX;
  s->error = 0;
  s->used_identity = 0;
  s->rounds = 0;
  f->first_bad = ~0ull;
  f->unsupported = 0;
  f->total_tokens = 0;
}

orch_cost_model policy_model(const orch_policy& p) {  // balancers.cpp:162-176
  orch_cost_model m{1.0, 0.0, 0, ORCH_LINEAR_ONLY};
  switch (p.kind) {
    case ORCH_BINARY_PADDED:
      m.padded = 1;
      break;
    case ORCH_QUADRATIC_TOLERANCE:
      m.beta = p.lambda;
      m.variant = ORCH_TRANSFORMER_QUADRATIC;
      break;
    case ORCH_CONVTRANSFORMER:
      m.beta = p.lambda;
      m.variant = ORCH_CONV_TRANSFORMER_PADDED;
      break;
    default:
      break;
  }
  return m;
}

// distribute_min_sum on [first, n) of the descending order.
// lpt_*: n-sized scratch for the one-CTA LPT's sorted-position results (d > 32).
int launch_greedy(orch_ctx* ctx, int d, int64_t n, const int64_t* first, const uint32_t* xs,
                  const int32_t* order, const int64_t* init_load, const int32_t* init_count,
                  int32_t* di, int32_t* ds, int64_t* doff, int32_t* bc, int64_t* bt,
                  orch_summary* s, cudaStream_t st, int32_t* lpt_bin, int32_t* lpt_slot,
                  int64_t* lpt_off) {
  if (d <= 32) {
    launch(ctx, [&] {
      k_greedy_warp<<<1, 32, 0, st>>>(d, n, first, xs, order, init_load, init_count, di, ds, doff,
                                      bc, bt, s);
    });
  } else {
    auto run = [&](auto kern, size_t sm, int threads) -> int {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm)));
      launch(ctx, [&] {
        kern<<<1, threads, sm, st>>>(d, n, first, xs, order, init_load, init_count, di, ds, doff,
                                     bc, bt, s, lpt_bin, lpt_slot, lpt_off);
      });
      if (lpt_bin && n > 0)
        launch(ctx, [&] {
          k_lpt_scatter<<<blocks_for(n, kThreads), kThreads, 0, st>>>(
              n, first, order, lpt_bin, lpt_slot, lpt_off, di, ds, doff, s);
        });
      return ORCH_OK;
    };
    int rc;
    if (d <= LptShape<64>::kSlots)
      rc = run(k_greedy_lpt<64>, lpt_smem_bytes<64>(d), 64);
    else if (d <= LptShape<256>::kSlots)
      rc = run(k_greedy_lpt<256>, lpt_smem_bytes<256>(d), 256);
    else
      rc = run(k_greedy_lpt<1024>, lpt_smem_bytes<1024>(d), 1024);
    if (rc) return rc;
  }
  return ORCH_OK;
}

}  // namespace

// Host-side argument checks in the reference's order (require_valid_d, then
// the policy's own checks; index_sources is checked on the device).
int check_policy_args(const orch_policy* p, int d, int64_t n, int identity_only) {
  if (!p) return fail(ORCH_INVALID_ARGUMENT, "null policy");
  if (p->kind < 0 || p->kind > 3) return fail(ORCH_LOGIC_ERROR, "unknown policy kind");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  if (d > ORCH_MAX_INSTANCES)
    return fail(ORCH_UNSUPPORTED, "instance count exceeds ORCH_MAX_INSTANCES (" +
                                      std::to_string(ORCH_MAX_INSTANCES) + ")");
  if (n < 0 || n > ORCH_MAX_ITEMS) return fail(ORCH_UNSUPPORTED, "item count exceeds ORCH_MAX_ITEMS");
  if (identity_only) return ORCH_OK;
  switch (p->kind) {
    case ORCH_BINARY_PADDED:
      if (n == 0) return fail(ORCH_INVALID_ARGUMENT, "padded balancing needs at least one item");
      break;
    case ORCH_QUADRATIC_TOLERANCE:
      if (p->lambda < 0.0 || p->tolerance_v < 0)
        return fail(ORCH_INVALID_ARGUMENT, "lambda and tolerance_v must be nonnegative");
      break;
    case ORCH_CONVTRANSFORMER:
      if (n == 0)
        return fail(ORCH_INVALID_ARGUMENT, "convtransformer balancing needs at least one item");
      if (p->lambda < 0.0) return fail(ORCH_INVALID_ARGUMENT, "lambda must be nonnegative");
      break;
    default:
      break;
  }
  return ORCH_OK;
}

// The single-CTA kernel serves the call (k_balance_small): it reads each input
// once and writes each output once.
bool takes_small_path(const orch_policy* pol, int d, int64_t n, int mode) {
  const bool one_lane_per_batch = mode == 0 && (pol->kind == ORCH_QUADRATIC_TOLERANCE ||
                                                pol->kind == ORCH_CONVTRANSFORMER);
  return mode <= 1 && d <= (one_lane_per_batch ? 32 : kSmallMaxD) && n <= kSmallMaxItems;
}

// mode: 0 balance, 1 identity only, 2 padded search only, 3 padded feasibility probe
int run_balance(orch_ctx* ctx, const orch_policy* pol, int d, int64_t n, const int64_t* len,
                const int32_t* origin, int mode, int64_t probe, const orch_balance_out* out,
                int64_t* d_bound_out, int32_t* d_probe_out, cudaStream_t st,
                const orch_layout_out* lay1 = nullptr, bool* lay1_done = nullptr) {
  if (lay1_done) *lay1_done = false;
  const int identity_only = mode == 1;
  if (!out || !out->summary) return fail(ORCH_INVALID_ARGUMENT, "orch_balance: summary required");
  orch_summary* S = out->summary;
  const orch_cost_model model = policy_model(*pol);
  const int kind = pol->kind;
  const bool padded_only = mode >= 2;
  const bool needs_desc = !identity_only && !padded_only && kind != ORCH_BINARY_PADDED;
  const bool needs_asc = padded_only || (!identity_only && kind == ORCH_BINARY_PADDED);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);

  // quadratic tolerance and ConvTransformer keep one batch per lane (d <= 32)
  if (takes_small_path(pol, d, n, mode)) {
    Plan sp;
    SmallArgs a{};
    const size_t nn1 = static_cast<size_t>(n > 0 ? n : 1);
    sp.add_or(&a.dest_inst, out->dest_inst, nn1);
    sp.add_or(&a.dest_slot, out->dest_slot, nn1);
    sp.add_or(&a.src_slot, out->src_slot, nn1);
    sp.add_or(&a.src_off, out->src_off, nn1);
    sp.add_or(&a.dst_off, out->dst_off, nn1);
    sp.add_or(&a.bin_count, out->bin_count, d);
    sp.add_or(&a.bin_len, out->bin_len, d);
    sp.add_or(&a.bin_tokens, out->bin_tokens, d);
    sp.add_or(&a.bin_cost, out->bin_cost, d);
    sp.add_or(&a.bin_offset, out->bin_offset, d + 1);
    sp.add_or(&a.bin_member, out->bin_member, nn1);
    sp.add_or(&a.src_offset, out->src_offset, d + 1);
    sp.add_or(&a.src_member, out->src_member, nn1);
    int rc0 = sp.commit(ctx, st);
    if (rc0) return rc0;
    a.kind = kind;
    a.identity_only = identity_only;
    a.d = d;
    a.n = static_cast<int>(n);
    a.tol_v = pol->tolerance_v;
    a.model = model;
    a.len = len;
    a.origin = origin;
    a.s = S;
    if (lay1) {  // the single-rank layout in the same launch
      a.with_layout = 1;
      a.lay = *lay1;
      if (lay1_done) *lay1_done = true;
    }
    auto run_small = [&](auto kern, int sm) -> int {
      static PerDeviceOnce configured[3];  // per instantiation
      const int slot = sm == static_cast<int>(sizeof(SmallSmem<2>)) ? 0
                       : sm == static_cast<int>(sizeof(SmallSmem<4>)) ? 1 : 2;
      const int rc_attr = configured[slot]([&]() -> int {
        ORCH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        ORCH_CUDA_TRY(max_carveout(kern));
        return ORCH_OK;
      });
      if (rc_attr) return rc_attr;
      launch(ctx, [&] { kern<<<1, kSmallThreads, sm, st>>>(a); });
      return ORCH_OK;
    };
    int rc1;
    if (n <= 2 * kSmallThreads)
      rc1 = run_small(k_balance_small<2>, static_cast<int>(sizeof(SmallSmem<2>)));
    else if (n <= 4 * kSmallThreads)
      rc1 = run_small(k_balance_small<4>, static_cast<int>(sizeof(SmallSmem<4>)));
    else
      rc1 = run_small(k_balance_small<16>, static_cast<int>(sizeof(SmallSmem<16>)));
    if (rc1) return rc1;
    ORCH_CUDA_TRY(cudaGetLastError());
    return ORCH_OK;
  }

  // ---- workspace plan
  Plan plan;
  Flags* flags;
  uint32_t *key_len, *key_org, *sorted_org, *xs;
  int32_t *iota, *ident_order, *order, *ident_count, *ident_offset;
  int64_t *ident_len, *ident_prefix;
  int32_t* i_count;
  int64_t *i_len, *i_tokens;
  double* i_cost;
  int32_t *dest_inst, *dest_slot, *src_slot, *bin_count, *bin_offset, *bin_member, *a_count;
  int64_t *src_off, *dst_off, *bin_len, *bin_tokens, *a_tokens;
  double* bin_cost;
  plan.add(&flags, 1);
  plan.add(&key_len, nn);
  plan.add(&key_org, nn);
  plan.add(&sorted_org, nn);
  plan.add(&xs, nn);
  plan.add(&iota, nn);
  plan.add_or(&ident_order, out->src_member, nn);
  plan.add(&order, nn);
  plan.add(&ident_count, d + 1);
  plan.add_or(&ident_offset, out->src_offset, d + 1);
  plan.add(&ident_len, nn + 1);
  plan.add(&ident_prefix, nn + 1);
  plan.add(&i_count, d);
  plan.add(&i_len, d);
  plan.add(&i_tokens, d);
  plan.add(&i_cost, d);
  plan.add(&a_count, d + 1);
  plan.add(&a_tokens, d);
  plan.add_or(&dest_inst, out->dest_inst, nn);
  plan.add_or(&dest_slot, out->dest_slot, nn);
  plan.add_or(&src_slot, out->src_slot, nn);
  plan.add_or(&src_off, out->src_off, nn);
  plan.add_or(&dst_off, out->dst_off, nn);
  plan.add_or(&bin_count, out->bin_count, d);
  plan.add_or(&bin_len, out->bin_len, d);
  plan.add_or(&bin_tokens, out->bin_tokens, d);
  plan.add_or(&bin_cost, out->bin_cost, d);
  plan.add_or(&bin_offset, out->bin_offset, d + 1);
  plan.add_or(&bin_member, out->bin_member, nn);
  // ConvTransformer / BinaryPadded extras
  int32_t *g_di, *g_ds, *seed_count, *n_groups;
  int64_t *g_doff, *seed_load, *consumed, *asc_len, *asc_prefix, *starts, *bound;
  const bool conv = !identity_only && !padded_only && kind == ORCH_CONVTRANSFORMER;
  plan.add(&g_di, conv ? nn : 1);
  plan.add(&g_ds, conv ? nn : 1);
  plan.add(&g_doff, conv ? nn : 1);
  plan.add(&seed_load, d);
  plan.add(&seed_count, d);
  plan.add(&consumed, 1);
  plan.add(&asc_len, needs_asc ? nn + 1 : 1);
  plan.add(&asc_prefix, needs_asc ? nn + 1 : 1);
  plan.add(&starts, d + 2);
  plan.add(&n_groups, 1);
  plan.add(&bound, 1);
  PadSearch* pads;
  int32_t* pad_feas;
  int64_t* pad_cand;
  plan.add(&pads, 1);
  plan.add(&pad_feas, kSMs);
  plan.add(&pad_cand, kSMs);
  uint16_t* pad_nx1;
  plan.add(&pad_nx1, n <= kNxMax ? n : 1);
  // sorted-position results of the one-CTA LPT (greedy / conv, d > 32)
  int32_t *lpt_bin, *lpt_slot;
  int64_t* lpt_off;
  const bool lpt = !identity_only && !padded_only && d > 32 &&
                   (kind == ORCH_GREEDY_UNPADDED || kind == ORCH_CONVTRANSFORMER);
  plan.add(&lpt_bin, lpt ? nn : 1);
  plan.add(&lpt_slot, lpt ? nn : 1);
  plan.add(&lpt_off, lpt ? nn : 1);
  // radix sort / scan scratch (radix.cuh)
  uint32_t *rs_kt, *rs_hist;
  int32_t *rs_vt, *scan32_part;
  int64_t* scan64_part;
  RsState* rs_state;
  plan.add(&rs_kt, nn);
  plan.add(&rs_vt, nn);
  plan.add(&rs_hist, rs_hist_words(static_cast<int64_t>(nn)));
  plan.add(&rs_state, 1);
  plan.add(&scan64_part, static_cast<size_t>(rs_tiles(static_cast<int64_t>(nn) + 1)));
  plan.add(&scan32_part, static_cast<size_t>(rs_tiles(static_cast<int64_t>(d) + 1)));
  int rc = plan.commit(ctx, st);
  if (rc) return rc;

  const int gb = blocks_for(n, kThreads);
  launch(ctx, [&] { k_init<<<1, 1, 0, st>>>(S, flags); });
  ORCH_CUDA_TRY(cudaMemsetAsync(ident_count, 0, sizeof(int32_t) * (d + 1), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(a_count + d, 0, sizeof(int32_t), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(ident_len + n, 0, sizeof(int64_t), st));
  if (n > 0)
    launch(ctx, [&] {
      k_validate<<<gb, kThreads, 0, st>>>(d, n, len, origin, key_len, key_org, iota, flags);
    });
  launch(ctx, [&] { k_validate_finish<<<1, 1, 0, st>>>(n, flags, S); });

  // ---- identity (origin) batches: always needed (never_worse)
  if (n > 0) {
    rc = rs_sort_pairs(ctx, key_org, iota, sorted_org, ident_order, rs_kt, rs_vt, n, false,
                       rs_hist, rs_state, st);
    if (rc) return rc;
    launch(ctx, [&] {
      k_ident_count<<<gb, kThreads, 0, st>>>(n, ident_order, origin, len, ident_count, ident_len, S);
    });
  }
  {
    rc = rs_exclusive_scan<int32_t>(ctx, ident_count, ident_offset, d + 1, scan32_part, st);
    if (rc) return rc;
  }
  if (n > 0) {
    rc = rs_exclusive_scan<int64_t>(ctx, ident_len, ident_prefix, n + 1, scan64_part, st);
    if (rc) return rc;
    launch(ctx, [&] {
      k_ident_slots<<<gb, kThreads, 0, st>>>(n, ident_order, origin, ident_offset, ident_prefix,
                                             src_slot, src_off, S);
    });
  }
  const int cb = blocks_for(static_cast<int64_t>(d) * 32, kThreads);
  launch(ctx, [&] {
    k_bin_cost<<<cb, kThreads, 0, st>>>(model, d, ident_offset, ident_order, len, i_count, i_len,
                                        i_tokens, i_cost, S);
  });

  // ---- the balancer's own packing
  if (needs_desc && n > 0) {
    rc = rs_sort_pairs(ctx, key_len, iota, xs, order, rs_kt, rs_vt, n, true, rs_hist, rs_state, st);
    if (rc) return rc;
  }
  if (needs_asc) {
    rc = rs_sort_pairs(ctx, key_len, iota, xs, order, rs_kt, rs_vt, n, false, rs_hist, rs_state,
                       st);
    if (rc) return rc;
    launch(ctx, [&] { k_u32_to_i64<<<gb, kThreads, 0, st>>>(n, xs, asc_len); });
    ORCH_CUDA_TRY(cudaMemsetAsync(asc_len + n, 0, sizeof(int64_t), st));
    rc = rs_exclusive_scan<int64_t>(ctx, asc_len, asc_prefix, n + 1, scan64_part, st);
    if (rc) return rc;
    const bool use_nx = n <= kNxMax;
    const int nx_smem = static_cast<int>(n) * 2;
    static PerDeviceOnce pad_configured;
    const int rc_attr = pad_configured([&]() -> int {
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_pad_eval_nx, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kNxMax * 2));
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_pad_starts_nx,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kNxMax * 2));
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_padded_search,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      return ORCH_OK;
    });
    if (rc_attr) return rc_attr;
    if (mode == 3) {  // one feasibility probe
      if (use_nx) {
        launch(ctx, [&] {
          k_pad_eval_nx<<<1, 1024, nx_smem, st>>>(d, n, xs, pads, pad_feas, pad_cand, 1, probe,
                                                  n_groups, S);
        });
      } else {
        launch(ctx, [&] {
          k_padded_search<<<1, 1024, 0, st>>>(d, n, xs, 1, probe, starts, n_groups, bound, S, 0);
        });
      }
    } else {
      launch(ctx, [&] { k_pad_init<<<1, 32, 0, st>>>(d, n, xs, pads, S); });
      for (int r = 0; r < kPadRounds; ++r) {
        launch(ctx, [&] {
          if (use_nx)
            k_pad_eval_nx<<<kSMs, 1024, nx_smem, st>>>(d, n, xs, pads, pad_feas, pad_cand, 0, 0,
                                                       nullptr, S);
          else
            k_pad_eval_warp<<<kSMs, 32, 0, st>>>(d, n, xs, pads, pad_feas, pad_cand, S);
        });
      }
      launch(ctx, [&] {
        if (use_nx)
          k_pad_starts_nx<<<1, 1024, nx_smem, st>>>(d, n, xs, pads, pad_nx1, starts, n_groups,
                                                    bound, S);
        else
          k_pad_starts_warp<<<1, 32, 0, st>>>(d, n, xs, pads, starts, n_groups, bound, S);
      });
    }
    if (padded_only) {
      if (mode == 2 && d_bound_out)
        ORCH_CUDA_TRY(cudaMemcpyAsync(d_bound_out, bound, sizeof(int64_t),
                                      cudaMemcpyDeviceToDevice, st));
      if (mode == 3 && d_probe_out)
        ORCH_CUDA_TRY(cudaMemcpyAsync(d_probe_out, n_groups, sizeof(int32_t),
                                      cudaMemcpyDeviceToDevice, st));
      return ORCH_OK;
    }
    launch(ctx, [&] {
      k_padded_place<<<gb, kThreads, 0, st>>>(d, n, order, asc_prefix, starts, n_groups, dest_inst,
                                              dest_slot, dst_off, bin_offset, bin_member, a_count,
                                              a_tokens, S);
    });
  }
  if (!identity_only && kind != ORCH_BINARY_PADDED) {
    if (kind == ORCH_GREEDY_UNPADDED) {
      rc = launch_greedy(ctx, d, n, nullptr, xs, order, nullptr, nullptr, dest_inst, dest_slot,
                         dst_off, a_count, a_tokens, S, st, lpt ? lpt_bin : nullptr, lpt_slot,
                         lpt_off);
      if (rc) return rc;
    } else if (kind == ORCH_QUADRATIC_TOLERANCE) {
      const size_t sm = (2 * sizeof(int64_t) + sizeof(int32_t)) * d;
      ORCH_CUDA_TRY(cudaFuncSetAttribute(k_quadtol, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm));
      launch(ctx, [&] {
        k_quadtol<<<1, 32, sm, st>>>(d, n, pol->tolerance_v, xs, order, dest_inst, dest_slot,
                                     dst_off, a_count, a_tokens, S);
      });
    } else {  // ConvTransformer
      rc = launch_greedy(ctx, d, n, nullptr, xs, order, nullptr, nullptr, g_di, g_ds, g_doff,
                         a_count, a_tokens, S, st, lpt ? lpt_bin : nullptr, lpt_slot, lpt_off);
      if (rc) return rc;
      launch(ctx, [&] {
        k_conv_seed<<<1, 32, 0, st>>>(d, n, xs, order, a_tokens, dest_inst, dest_slot, dst_off,
                                      seed_load, seed_count, consumed, S);
      });
      rc = launch_greedy(ctx, d, n, consumed, xs, order, seed_load, seed_count, dest_inst,
                         dest_slot, dst_off, a_count, a_tokens, S, st, lpt ? lpt_bin : nullptr,
                         lpt_slot, lpt_off);
      if (rc) return rc;
    }
    rc = rs_exclusive_scan<int32_t>(ctx, a_count, bin_offset, d + 1, scan32_part, st);
    if (rc) return rc;
    if (n > 0)
      launch(ctx, [&] {
        k_scatter_members<<<gb, kThreads, 0, st>>>(n, dest_inst, dest_slot, bin_offset,
                                                   bin_member, S);
      });
  }
  if (!identity_only)
    launch(ctx, [&] {
      k_bin_cost<<<cb, kThreads, 0, st>>>(model, d, bin_offset, bin_member, len, bin_count,
                                          bin_len, bin_tokens, bin_cost, S);
    });
  launch(ctx, [&] {
    k_decide<<<1, 1024, 0, st>>>(d, identity_only, i_cost, identity_only ? i_cost : bin_cost, S);
  });
  const int fb = blocks_for(std::max<int64_t>(n, d + 1), kThreads);
  launch(ctx, [&] {
    k_apply_identity<<<fb, kThreads, 0, st>>>(
        d, n, origin, src_slot, src_off, ident_offset, ident_order, i_count, i_len, i_tokens,
        i_cost, dest_inst, dest_slot, dst_off, bin_offset, bin_member, bin_count, bin_len,
        bin_tokens, bin_cost, S);
  });
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // namespace orchb

namespace {

int device_error_message(int code, int64_t idx, int d, const int64_t* h_len,
                         const int32_t* h_origin) {
  if (code == ORCH_INVALID_ARGUMENT && h_len && h_origin) {
    if (h_origin[idx] < 0 || h_origin[idx] >= d)
      return orchb::fail(code, "item origin instance outside [0, d)");
    return orchb::fail(code, "item length must be >= 1");
  }
  if (code == ORCH_INVALID_ARGUMENT) return orchb::fail(code, "invalid item at input position " + std::to_string(idx));
  return orchb::fail(code, "input exceeds the device limits (length < 2^32, total tokens < 2^50)");
}

struct HostStage {
  int64_t* len;
  int32_t* origin;
  orch_balance_out out;
  orch_summary* summary;
};

}  // namespace

extern "C" {

int orch_balance(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                 const int64_t* d_len, const int32_t* d_origin, int32_t identity_only,
                 const orch_balance_out* out, void* stream) {
  if (!ctx) return orchb::fail(ORCH_INVALID_ARGUMENT, "null context");
  int rc = orchb::check_policy_args(policy, d, n, identity_only);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  return orchb::run_balance(ctx, policy, d, n, d_len, d_origin, identity_only ? 1 : 0, 0, out,
                            nullptr, nullptr, static_cast<cudaStream_t>(stream));
}

int orch_balance_layout1(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                         const int64_t* d_len, const int32_t* d_origin, int32_t identity_only,
                         const orch_balance_out* out, const orch_layout_out* layout,
                         void* stream) {
  if (!ctx) return orchb::fail(ORCH_INVALID_ARGUMENT, "null context");
  if (!layout || !layout->status || !layout->rank_src_off || !layout->rank_dst_off ||
      !layout->pair_off || !layout->send_rows || !layout->send_displ || !layout->recv_displ ||
      !layout->in_rows || !layout->out_rows)
    return orchb::fail(ORCH_INVALID_ARGUMENT, "orch_balance_layout1: every layout array is required");
  if (!out || !out->dest_inst || !out->src_off || !out->dst_off || !out->bin_offset ||
      !out->bin_member)
    return orchb::fail(ORCH_INVALID_ARGUMENT,
                       "orch_balance_layout1 needs dest_inst, src_off, dst_off, bin_offset, bin_member");
  int rc = orchb::check_policy_args(policy, d, n, identity_only);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  bool fused = false;
  rc = orchb::run_balance(ctx, policy, d, n, d_len, d_origin, identity_only ? 1 : 0, 0, out,
                          nullptr, nullptr, static_cast<cudaStream_t>(stream), layout, &fused);
  if (rc || fused) return rc;
  return orch_layout(ctx, d, 1, n, d_len, d_origin, out, layout, stream);
}

}  // extern "C"

// Host-buffer variants stage through a per-context device buffer and its
// pinned host mirror with the same layout: inputs | outputs. One H2D copy of
// the inputs, the pipeline, one D2H copy of the outputs, one synchronize
// (pageable cudaMemcpyAsync calls cost ~10 us each; a call used to make eight).
namespace {

constexpr int64_t kZeroCopyItems = 4096;

int host_pipeline(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                  const int64_t* h_len, const int32_t* h_origin, int mode, int64_t probe,
                  int32_t* h_dest_inst, int32_t* h_dest_slot, int64_t* h_dst_off,
                  int32_t* h_bin_count, double* h_bin_cost, orch_summary* h_summary,
                  int64_t* h_bound, int32_t* h_probe, cudaStream_t st) {
  if (!ctx) return orchb::fail(ORCH_INVALID_ARGUMENT, "null context");
  ORCH_CUDA_TRY(cudaSetDevice(ctx->device));
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  auto al = [](size_t b) { return (b + 255) & ~size_t{255}; };
  // byte offsets of the staged arrays (device buffer and pinned mirror alike)
  size_t at = 0;
  auto take = [&](size_t b) {
    const size_t r = at;
    at += al(b);
    return r;
  };
  const size_t o_len = take(nn * 8), o_org = take(nn * 4);
  const size_t in_bytes = at;
  const size_t o_di = take(nn * 4), o_ds = take(nn * 4), o_doff = take(nn * 8);
  const size_t o_bc = take(static_cast<size_t>(d) * 4), o_cost = take(static_cast<size_t>(d) * 8);
  const size_t o_sum = take(sizeof(orch_summary)), o_bound = take(8), o_probe = take(8);
  const size_t total = at;
  char *hp, *dp;
  int rc = orchb::host_stage(ctx, total, &hp, &dp);
  if (rc) return rc;
  orch_balance_out out{};
  // only the outputs this mode reads back are written by the pipeline
  const bool rows = n > 0 && mode < 2;
  // Zero copy when the single-CTA kernel serves the call and the phase is small
  // (C5: 64 items): it reads the pinned staging through the host mapping and
  // writes its outputs back the same way, so a call is one launch and one
  // synchronize with no copy operations.
  const bool zero_copy = n <= kZeroCopyItems && orchb::takes_small_path(policy, d, n, mode);
  char* base = zero_copy ? hp : dp;
  out.dest_inst = reinterpret_cast<int32_t*>(base + o_di);
  out.dest_slot = reinterpret_cast<int32_t*>(base + o_ds);
  out.dst_off = reinterpret_cast<int64_t*>(base + o_doff);
  out.bin_count = reinterpret_cast<int32_t*>(base + o_bc);
  out.bin_cost = reinterpret_cast<double*>(base + o_cost);
  out.summary = reinterpret_cast<orch_summary*>(base + o_sum);
  if (n > 0) {
    std::memcpy(hp + o_len, h_len, static_cast<size_t>(n) * 8);
    std::memcpy(hp + o_org, h_origin, static_cast<size_t>(n) * 4);
    if (!zero_copy) ORCH_CUDA_TRY(cudaMemcpyAsync(dp, hp, in_bytes, cudaMemcpyHostToDevice, st));
  }
  rc = orchb::run_balance(ctx, policy, d, n, reinterpret_cast<int64_t*>(base + o_len),
                          reinterpret_cast<int32_t*>(base + o_org), mode, probe, &out,
                          reinterpret_cast<int64_t*>(base + o_bound),
                          reinterpret_cast<int32_t*>(base + o_probe), st);
  if (rc) return rc;
  // one read-back: the per-item outputs (balance modes) through the probe word
  const size_t back = rows ? o_di : o_bc;
  if (!zero_copy)
    ORCH_CUDA_TRY(cudaMemcpyAsync(hp + back, dp + back, total - back, cudaMemcpyDeviceToHost, st));
  ORCH_CUDA_TRY(cudaStreamSynchronize(st));
  orch_summary sum;
  std::memcpy(&sum, hp + o_sum, sizeof sum);
  if (rows) {
    if (h_dest_inst) std::memcpy(h_dest_inst, hp + o_di, static_cast<size_t>(n) * 4);
    if (h_dest_slot) std::memcpy(h_dest_slot, hp + o_ds, static_cast<size_t>(n) * 4);
    if (h_dst_off) std::memcpy(h_dst_off, hp + o_doff, static_cast<size_t>(n) * 8);
  }
  if (mode < 2) {
    if (h_bin_count) std::memcpy(h_bin_count, hp + o_bc, static_cast<size_t>(d) * 4);
    if (h_bin_cost) std::memcpy(h_bin_cost, hp + o_cost, static_cast<size_t>(d) * 8);
  }
  if (mode == 2 && h_bound) std::memcpy(h_bound, hp + o_bound, 8);
  if (mode == 3 && h_probe) std::memcpy(h_probe, hp + o_probe, 4);
  if (h_summary) *h_summary = sum;
  if (sum.error) return device_error_message(sum.error, sum.error_index, d, h_len, h_origin);
  return ORCH_OK;
}

}  // namespace

extern "C" {

int orch_balance_host(orch_ctx* ctx, const orch_policy* policy, int32_t d, int64_t n,
                      const int64_t* h_len, const int32_t* h_origin, int32_t identity_only,
                      int32_t* h_dest_inst, int32_t* h_dest_slot, int64_t* h_dst_off,
                      int32_t* h_bin_count, double* h_bin_cost, orch_summary* h_summary,
                      void* stream) {
  int rc = orchb::check_policy_args(policy, d, n, identity_only);
  if (rc) return rc;
  return host_pipeline(ctx, policy, d, n, h_len, h_origin, identity_only ? 1 : 0, 0, h_dest_inst,
                       h_dest_slot, h_dst_off, h_bin_count, h_bin_cost, h_summary, nullptr,
                       nullptr, static_cast<cudaStream_t>(stream));
}

int orch_min_feasible_padded_bound_host(orch_ctx* ctx, int32_t d, int64_t n,
                                        const int64_t* h_len, const int32_t* h_origin,
                                        int64_t* h_bound, void* stream) {
  orch_policy p{ORCH_BINARY_PADDED, 0, 0, 0.0};
  int rc = orchb::check_policy_args(&p, d, n, 0);
  if (rc) return rc;
  return host_pipeline(ctx, &p, d, n, h_len, h_origin, 2, 0, nullptr, nullptr, nullptr, nullptr,
                       nullptr, nullptr, h_bound, nullptr, static_cast<cudaStream_t>(stream));
}

int orch_padded_bound_feasible_host(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* h_len,
                                    const int32_t* h_origin, int64_t bound, int32_t* h_feasible,
                                    void* stream) {
  orch_policy p{ORCH_BINARY_PADDED, 0, 0, 0.0};
  int rc = orchb::check_policy_args(&p, d, n, 0);
  if (rc) return rc;
  return host_pipeline(ctx, &p, d, n, h_len, h_origin, 3, bound, nullptr, nullptr, nullptr,
                       nullptr, nullptr, nullptr, nullptr, h_feasible,
                       static_cast<cudaStream_t>(stream));
}

}  // extern "C"

#ifdef ORCH_SMALL_PROFILE
// Diagnostics build only (ORCH_NVCC_EXTRA=-DORCH_SMALL_PROFILE): clock64 stamps
// of the last k_balance_small launch at its stage boundaries (SMALL_MARK/SUB).
extern "C" int orch_debug_small_profile(long long* h_out16) {
  ORCH_CUDA_TRY(cudaDeviceSynchronize());
  ORCH_CUDA_TRY(cudaMemcpyFromSymbol(h_out16, orchb::g_small_prof, 16 * sizeof(long long)));
  return ORCH_OK;
}
#endif
