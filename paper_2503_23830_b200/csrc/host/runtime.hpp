// Host adapter runtime: per-thread C-ABI context on the current CUDA device
// and the mapping of C-ABI return codes onto the reference's exceptions.
#pragma once

#include <cstdint>
#include <vector>

#include "orchsim/core.hpp"
#include "orchsim_capi.h"

namespace orchsim::b200 {

// The calling thread's context on its current CUDA device (created lazily).
orch_ctx* context();

// Throws the exception class the reference raises for `code` (errors.hpp /
// <stdexcept>) with the library's message; no-op for ORCH_OK.
void check(int code);

// cost(model, b) of many batches in one device call (orch_batch_costs_host);
// throws like cost() on the first batch (in order) whose padding mode differs.
std::vector<double> batch_costs(const CostModel& model, const std::vector<const MiniBatch*>& batches);

inline orch_cost_model to_abi(const CostModel& m) {
  return orch_cost_model{m.alpha, m.beta, m.padding_mode == PaddingMode::Padded ? 1 : 0,
                         static_cast<int32_t>(m.variant)};
}

}  // namespace orchsim::b200
