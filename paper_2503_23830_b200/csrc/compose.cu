// Composed delivery: encoder outputs go from where
// the encoder phase left them straight to their backbone (LLM) slots in ONE
// exchange, compose(to_backbone, encoder) = to_backbone o encoder^-1
// (exchange.cpp:115-137, orchestrator.cpp:390-418), instead of resetting to
// the origin first.
//
//   orch_backbone_targets  backbone_mapping_for (orchestrator.cpp:367-388):
//                          each universe item's (instance, slot) in the LLM
//                          layout -- examples on their LLM instance in LLM
//                          slot order, parts in interleave order.
//   orch_rearrange         any rearrangement given per item as
//                          (src_inst, src_slot) -> (dst_inst, dst_slot),
//                          validated like Rearrangement/apply (core.cpp:14-43,
//                          120-161) and laid out as a flat balance result, so
//                          orch_layout / orch_dispatch / orch_put move its rows.
// Composition and inversion of flat rearrangements are argument swaps: the
// encoder result's (dest_inst, dest_slot) is the composed move's source.

#include <string>

#include "common.cuh"
#include "plan.cuh"
#include "radix.cuh"

namespace orchb {
namespace {

constexpr int kT = 256;

struct RrFlags {
  unsigned int bad_range;  // an instance outside [0, d)
  unsigned int dup_dst;    // two items on one destination slot / non-dense
  unsigned int dup_src;    // a source slot twice / absent
};

__global__ void k_rr_count(int d, int64_t n, const int32_t* __restrict__ si,
                           const int32_t* __restrict__ di, int32_t* __restrict__ scnt,
                           int32_t* __restrict__ dcnt, RrFlags* f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int a = si[i], b = di[i];
    if (a < 0 || a >= d || b < 0 || b >= d) {
      atomicOr(&f->bad_range, 1u);
      continue;
    }
    atomicAdd(&scnt[a], 1);
    atomicAdd(&dcnt[b], 1);
  }
}

// Slots in [0, count) and no slot twice <=> dense (Rearrangement's checks).
__global__ void k_rr_scatter(int d, int64_t n, const int32_t* __restrict__ inst,
                             const int32_t* __restrict__ slot, const int32_t* __restrict__ off,
                             int32_t* __restrict__ member, unsigned int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int a = inst[i], s = slot[i];
    if (a < 0 || a >= d) continue;
    const int cnt = off[a + 1] - off[a];
    if (s < 0 || s >= cnt || atomicCAS(&member[off[a] + s], -1, static_cast<int32_t>(i)) != -1)
      atomicOr(flag, 1u);
  }
}

__global__ void k_rr_gather_len(int64_t n, const int32_t* __restrict__ member,
                                const int64_t* __restrict__ len, int64_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = member[k];
    out[k] = i >= 0 ? len[i] : 0;  // -1: slot left empty by an invalid rearrangement
  }
}

__global__ void k_rr_offsets(int64_t n, const int32_t* __restrict__ member,
                             const int32_t* __restrict__ inst, const int32_t* __restrict__ off,
                             const int64_t* __restrict__ pfx, int64_t* __restrict__ tok_off) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = member[k];
    if (i >= 0) tok_off[i] = pfx[k] - pfx[off[inst[i]]];
  }
}

__global__ void k_rr_finish(int d, int64_t n, const RrFlags* f, const int32_t* __restrict__ doff,
                            const int64_t* __restrict__ dpfx, const int32_t* __restrict__ di,
                            const int32_t* __restrict__ ds, const int32_t* __restrict__ ss,
                            int32_t* __restrict__ dest_inst, int32_t* __restrict__ dest_slot,
                            int32_t* __restrict__ src_slot, int32_t* __restrict__ bin_count,
                            int64_t* __restrict__ bin_tokens, orch_summary* s) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    s->error = (f->bad_range || f->dup_dst || f->dup_src) ? ORCH_INVALID_ARGUMENT : 0;
    s->error_index = f->bad_range ? 0 : (f->dup_dst ? 1 : (f->dup_src ? 2 : INT64_MAX));
    s->used_identity = 0;
    s->rounds = 0;
    s->bound = 0;
  }
  for (int64_t i = tid; i < n; i += stride) {
    if (dest_inst) dest_inst[i] = di[i];
    if (dest_slot) dest_slot[i] = ds[i];
    if (src_slot) src_slot[i] = ss[i];
  }
  for (int64_t b = tid; b < d; b += stride) {
    if (bin_count) bin_count[b] = doff[b + 1] - doff[b];
    if (bin_tokens) bin_tokens[b] = dpfx[doff[b + 1]] - dpfx[doff[b]];
  }
}

// ---- backbone targets
__global__ void k_bt_parts(int64_t E, const int32_t* __restrict__ part_offset,
                           int32_t* __restrict__ part_example) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    for (int p = part_offset[e]; p < part_offset[e + 1]; ++p) part_example[p] = static_cast<int32_t>(e);
}

__global__ void k_bt_mark(int64_t n, const int32_t* __restrict__ item_part,
                          uint8_t* __restrict__ in_u) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    in_u[item_part[k]] = 1;
}

// universe parts per example, listed in LLM (instance, slot) order
__global__ void k_bt_count(int64_t E, const int32_t* __restrict__ llm_member,
                           const int32_t* __restrict__ part_offset,
                           const uint8_t* __restrict__ in_u, int64_t* __restrict__ cnt_in_order) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = llm_member[k];
    int64_t c = 0;
    for (int p = part_offset[e]; p < part_offset[e + 1]; ++p) c += in_u[p];
    cnt_in_order[k] = c;
  }
}

__global__ void k_bt_base(int64_t E, const int32_t* __restrict__ llm_member,
                          const int32_t* __restrict__ llm_offset,
                          const int32_t* __restrict__ llm_dest_inst,
                          const int64_t* __restrict__ pfx, int64_t* __restrict__ base) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = llm_member[k];
    base[e] = pfx[k] - pfx[llm_offset[llm_dest_inst[e]]];
  }
}

__global__ void k_bt_target(int64_t n, const int32_t* __restrict__ item_part,
                            const int32_t* __restrict__ part_example,
                            const int32_t* __restrict__ part_offset,
                            const int32_t* __restrict__ interleave_pos,
                            const uint8_t* __restrict__ in_u,
                            const int32_t* __restrict__ llm_dest_inst,
                            const int64_t* __restrict__ base, int32_t* __restrict__ dst_inst,
                            int32_t* __restrict__ dst_slot) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = item_part[k];
    const int32_t e = part_example[p];
    const int32_t q = interleave_pos[p];
    int rank = 0;  // universe parts of e ahead in interleave order
    for (int p2 = part_offset[e]; p2 < part_offset[e + 1]; ++p2)
      rank += (in_u[p2] && interleave_pos[p2] < q);
    dst_inst[k] = llm_dest_inst[e];
    dst_slot[k] = static_cast<int32_t>(base[e] + rank);
  }
}

}  // namespace
}  // namespace orchb

using namespace orchb;

extern "C" {

int orch_rearrange(orch_ctx* ctx, int32_t d, int64_t n, const int64_t* d_len,
                   const int32_t* d_src_inst, const int32_t* d_src_slot,
                   const int32_t* d_dst_inst, const int32_t* d_dst_slot,
                   const orch_balance_out* out, void* stream) {
  if (!ctx || !out || !out->summary) return fail(ORCH_INVALID_ARGUMENT, "null argument");
  if (d < 1) return fail(ORCH_INVALID_ARGUMENT, "instance count must be >= 1");
  if (!out->src_off || !out->dst_off || !out->bin_offset || !out->bin_member ||
      !out->src_offset || !out->src_member)
    return fail(ORCH_INVALID_ARGUMENT, "orch_rearrange needs the offset and CSR outputs");
  auto st = static_cast<cudaStream_t>(stream);
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  Plan plan;
  RrFlags* f;
  int32_t *scnt, *dcnt;
  int64_t *glen, *spfx, *dpfx, *part64;
  int32_t* part32;
  plan.add(&f, 1);
  plan.add(&scnt, d + 1);
  plan.add(&dcnt, d + 1);
  plan.add(&glen, nn + 1);
  plan.add(&spfx, nn + 1);
  plan.add(&dpfx, nn + 1);
  plan.add(&part64, static_cast<size_t>(rs_tiles(static_cast<int64_t>(nn) + 1)));
  plan.add(&part32, static_cast<size_t>(rs_tiles(static_cast<int64_t>(d) + 1)));
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemsetAsync(f, 0, sizeof(RrFlags), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(scnt, 0, 4 * (d + 1), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(dcnt, 0, 4 * (d + 1), st));
  ORCH_CUDA_TRY(cudaMemsetAsync(out->bin_member, 0xff, 4 * nn, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(out->src_member, 0xff, 4 * nn, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(glen + n, 0, 8, st));
  const int gb = blocks_for(n, kT);
  if (n > 0) k_rr_count<<<gb, kT, 0, st>>>(d, n, d_src_inst, d_dst_inst, scnt, dcnt, f);
  rc = rs_exclusive_scan<int32_t>(ctx, scnt, out->src_offset, d + 1, part32, st);
  if (rc) return rc;
  rc = rs_exclusive_scan<int32_t>(ctx, dcnt, out->bin_offset, d + 1, part32, st);
  if (rc) return rc;
  if (n > 0) {
    k_rr_scatter<<<gb, kT, 0, st>>>(d, n, d_dst_inst, d_dst_slot, out->bin_offset,
                                    out->bin_member, &f->dup_dst);
    k_rr_scatter<<<gb, kT, 0, st>>>(d, n, d_src_inst, d_src_slot, out->src_offset,
                                    out->src_member, &f->dup_src);
  }
  // token offsets inside each batch, destination then source side
  const int32_t* mem[2] = {out->bin_member, out->src_member};
  const int32_t* ins[2] = {d_dst_inst, d_src_inst};
  const int32_t* offs[2] = {out->bin_offset, out->src_offset};
  int64_t* pfx[2] = {dpfx, spfx};
  int64_t* tok[2] = {out->dst_off, out->src_off};
  for (int side = 0; side < 2; ++side) {
    if (n > 0)
      k_rr_gather_len<<<gb, kT, 0, st>>>(n, mem[side], d_len, glen);
    rc = rs_exclusive_scan<int64_t>(ctx, glen, pfx[side], n + 1, part64, st);
    if (rc) return rc;
    if (n > 0) k_rr_offsets<<<gb, kT, 0, st>>>(n, mem[side], ins[side], offs[side], pfx[side], tok[side]);
  }
  k_rr_finish<<<blocks_for(n > d ? n : d, kT), kT, 0, st>>>(
      d, n, f, out->bin_offset, dpfx, d_dst_inst, d_dst_slot, d_src_slot, out->dest_inst,
      out->dest_slot, out->src_slot, out->bin_count, out->bin_tokens, out->summary);
  ctx->launches += 9;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

int orch_backbone_targets(orch_ctx* ctx, int32_t d, int64_t E, const int32_t* d_llm_dest_inst,
                          const int32_t* d_llm_bin_offset, const int32_t* d_llm_bin_member,
                          const int32_t* d_part_offset, const int32_t* d_interleave_pos,
                          int64_t num_parts, int64_t n, const int32_t* d_item_part,
                          int32_t* d_dst_inst, int32_t* d_dst_slot, void* stream) {
  if (!ctx) return fail(ORCH_INVALID_ARGUMENT, "null context");
  if (d < 1 || E < 0 || n < 0) return fail(ORCH_INVALID_ARGUMENT, "bad sizes");
  auto st = static_cast<cudaStream_t>(stream);
  const size_t ee = static_cast<size_t>(E > 0 ? E : 1), pp = static_cast<size_t>(num_parts > 0 ? num_parts : 1);
  Plan plan;
  int32_t* part_example;
  uint8_t* in_u;
  int64_t *cnt, *pfx, *base, *part;
  plan.add(&part_example, pp);
  plan.add(&in_u, pp);
  plan.add(&cnt, ee + 1);
  plan.add(&pfx, ee + 1);
  plan.add(&base, ee);
  plan.add(&part, static_cast<size_t>(rs_tiles(static_cast<int64_t>(ee) + 1)));
  int rc = plan.commit(ctx, st);
  if (rc) return rc;
  ORCH_CUDA_TRY(cudaMemsetAsync(in_u, 0, pp, st));
  ORCH_CUDA_TRY(cudaMemsetAsync(cnt + E, 0, 8, st));
  if (E > 0) k_bt_parts<<<blocks_for(E, kT), kT, 0, st>>>(E, d_part_offset, part_example);
  if (n > 0) k_bt_mark<<<blocks_for(n, kT), kT, 0, st>>>(n, d_item_part, in_u);
  if (E > 0)
    k_bt_count<<<blocks_for(E, kT), kT, 0, st>>>(E, d_llm_bin_member, d_part_offset, in_u, cnt);
  rc = rs_exclusive_scan<int64_t>(ctx, cnt, pfx, E + 1, part, st);
  if (rc) return rc;
  if (E > 0)
    k_bt_base<<<blocks_for(E, kT), kT, 0, st>>>(E, d_llm_bin_member, d_llm_bin_offset,
                                                d_llm_dest_inst, pfx, base);
  if (n > 0)
    k_bt_target<<<blocks_for(n, kT), kT, 0, st>>>(n, d_item_part, part_example, d_part_offset,
                                                  d_interleave_pos, in_u, d_llm_dest_inst, base,
                                                  d_dst_inst, d_dst_slot);
  ctx->launches += 5;
  ORCH_CUDA_TRY(cudaGetLastError());
  return ORCH_OK;
}

}  // extern "C"
