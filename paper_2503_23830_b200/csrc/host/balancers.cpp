// orchsim balancers over the B200 C-ABI: items are flattened to (length,
// origin) arrays, balanced by the sm_100a pipeline (orch_balance_host), and the
// flat result is materialised into the reference's BalanceResult
// (balancers.cpp:43-60 assemble(): moves map, new_batches in slot order,
// objective).
#include <string>

#include "orchsim/balancers.hpp"
#include "runtime.hpp"

namespace orchsim {

namespace {

PaddingMode native_mode(PolicyKind k) {  // balancers.cpp:39-41
  return k == PolicyKind::BinaryPadded ? PaddingMode::Padded : PaddingMode::Unpadded;
}

BalanceResult run(const BalancePolicy& policy, int d, const std::vector<SeqItem>& items,
                  bool identity_only) {
  const std::int64_t n = static_cast<std::int64_t>(items.size());
  std::vector<std::int64_t> len(items.size());
  std::vector<int32_t> origin(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) {
    len[i] = items[i].length;
    origin[i] = items[i].origin_instance;
  }
  std::vector<int32_t> dest(items.size()), slot(items.size());
  std::vector<int32_t> count(static_cast<std::size_t>(d > 0 ? d : 1));
  orch_summary summary{};
  const orch_policy p{static_cast<int32_t>(policy.kind), 0, policy.tolerance_v, policy.lambda};
  b200::check(orch_balance_host(b200::context(), &p, d, n, len.data(), origin.data(),
                                identity_only ? 1 : 0, dest.data(), slot.data(), nullptr,
                                count.data(), nullptr, &summary, nullptr));
  BalanceResult r;
  r.objective_value = summary.objective;
  r.new_batches.resize(static_cast<std::size_t>(d));
  for (int i = 0; i < d; ++i) {
    r.new_batches[i].instance = i;
    r.new_batches[i].padding_mode = native_mode(policy.kind);
    r.new_batches[i].items.resize(static_cast<std::size_t>(count[i]));
  }
  // moves keyed by (origin, source slot): inserted in key order (a stable
  // counting sort by origin) so every insert is a hinted append
  std::vector<std::size_t> obase(static_cast<std::size_t>(d) + 1, 0);
  for (std::size_t i = 0; i < items.size(); ++i) {
    r.new_batches[dest[i]].items[slot[i]] = items[i];
    ++obase[static_cast<std::size_t>(origin[i]) + 1];
  }
  for (int i = 0; i < d; ++i) obase[i + 1] += obase[i];
  std::vector<int32_t> by_src(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) by_src[obase[origin[i]]++] = static_cast<int32_t>(i);
  std::map<SlotRef, SlotRef> moves;
  std::vector<int> next(static_cast<std::size_t>(d), 0);  // source slots (index_sources)
  for (const int32_t i : by_src)
    moves.emplace_hint(moves.end(), SlotRef{origin[i], next[origin[i]]++}, SlotRef{dest[i], slot[i]});
  r.rearrangement = Rearrangement(d, std::move(moves));
  return r;
}

}  // namespace

CostModel policy_cost_model(const BalancePolicy& p) {  // balancers.cpp:162-176
  switch (p.kind) {
    case PolicyKind::GreedyUnpadded:
      return CostModel{1.0, 0.0, PaddingMode::Unpadded, CostVariant::LinearOnly};
    case PolicyKind::BinaryPadded:
      return CostModel{1.0, 0.0, PaddingMode::Padded, CostVariant::LinearOnly};
    case PolicyKind::QuadraticTolerance:
      return CostModel{1.0, p.lambda, PaddingMode::Unpadded, CostVariant::TransformerQuadratic};
    case PolicyKind::ConvTransformer:
      return CostModel{1.0, p.lambda, PaddingMode::Unpadded, CostVariant::ConvTransformerPadded};
  }
  throw std::logic_error("unknown policy kind");
}

BalanceResult balance_greedy_unpadded(int d, const std::vector<SeqItem>& items) {
  return run(BalancePolicy{PolicyKind::GreedyUnpadded, 0, 0.0}, d, items, false);
}

BalanceResult balance_binary_padded(int d, const std::vector<SeqItem>& items) {
  return run(BalancePolicy{PolicyKind::BinaryPadded, 0, 0.0}, d, items, false);
}

BalanceResult balance_quadratic_tolerance(int d, const std::vector<SeqItem>& items, double lambda,
                                          std::int64_t tolerance_v) {
  return run(BalancePolicy{PolicyKind::QuadraticTolerance, tolerance_v, lambda}, d, items, false);
}

BalanceResult balance_convtransformer(int d, const std::vector<SeqItem>& items, double lambda) {
  return run(BalancePolicy{PolicyKind::ConvTransformer, 0, lambda}, d, items, false);
}

BalanceResult balance(const BalancePolicy& policy, int d, const std::vector<SeqItem>& items) {
  switch (policy.kind) {  // balancers.cpp:273-287: the per-kind entry points ignore
    case PolicyKind::GreedyUnpadded:  // the parameters they do not use
      return balance_greedy_unpadded(d, items);
    case PolicyKind::BinaryPadded:
      return balance_binary_padded(d, items);
    case PolicyKind::QuadraticTolerance:
      return balance_quadratic_tolerance(d, items, policy.lambda, policy.tolerance_v);
    case PolicyKind::ConvTransformer:
      return balance_convtransformer(d, items, policy.lambda);
  }
  throw std::logic_error("unknown policy kind");
}

BalanceResult identity_arrangement(const BalancePolicy& policy, int d,
                                   const std::vector<SeqItem>& items) {
  return run(policy, d, items, true);
}

std::int64_t min_feasible_padded_bound(int d, const std::vector<SeqItem>& items) {
  std::vector<std::int64_t> len(items.size());
  std::vector<int32_t> origin(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) {
    len[i] = items[i].length;
    origin[i] = items[i].origin_instance;
  }
  std::int64_t bound = 0;
  b200::check(orch_min_feasible_padded_bound_host(b200::context(), d,
                                                  static_cast<std::int64_t>(items.size()),
                                                  len.data(), origin.data(), &bound, nullptr));
  return bound;
}

bool padded_bound_feasible(int d, const std::vector<SeqItem>& items, std::int64_t bound) {
  std::vector<std::int64_t> len(items.size());
  std::vector<int32_t> origin(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) {
    len[i] = items[i].length;
    origin[i] = items[i].origin_instance;
  }
  int32_t ok = 0;
  b200::check(orch_padded_bound_feasible_host(b200::context(), d,
                                              static_cast<std::int64_t>(items.size()),
                                              len.data(), origin.data(), bound, &ok, nullptr));
  return ok != 0;
}

OracleResult oracle_optimal(int d, const std::vector<SeqItem>& items, const CostModel& model,
                            const OracleLimits& limits) {
  if (d < 1) throw std::invalid_argument("instance count must be >= 1");
  std::vector<std::int64_t> len(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) len[i] = items[i].length;
  OracleResult r;
  r.assignment.assign(items.size(), 0);
  std::vector<int32_t> a(items.size() ? items.size() : 1);
  const orch_cost_model m = b200::to_abi(model);
  b200::check(orch_oracle_optimal_host(b200::context(), &m, d,
                                       static_cast<std::int64_t>(items.size()), len.data(),
                                       limits.max_items, limits.max_instances, a.data(),
                                       &r.objective, nullptr));
  for (std::size_t i = 0; i < items.size(); ++i) r.assignment[i] = a[i];
  return r;
}

}  // namespace orchsim
