// extern "C" driver around the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Test and
// baseline infrastructure only: tests/ use it to pin the C restatement
// (oracle/orchsim_oracle.c) and to generate golden fixtures; bench.py's
// reference arm uses it to time the reference's own balance() on host cores.
//
// Bound reference entry points:
//   balance / identity_arrangement      proj/include/orchsim/balancers.hpp:53-60
//   min_feasible_padded_bound / padded_bound_feasible  balancers.hpp:64-69
//   cost                                proj/include/orchsim/core.hpp:115
//   volume_matrix                       proj/include/orchsim/topology.hpp:49
//   generate (synthetic MCI workload)   proj/include/orchsim/workload.hpp:48-51
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "orchsim/balancers.hpp"
#include "orchsim/core.hpp"
#include "orchsim/errors.hpp"
#include "orchsim/topology.hpp"
#include "orchsim/workload.hpp"

using namespace orchsim;

namespace {

thread_local std::string g_err;

int classify(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const SizeCapError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
  return 9;
}

std::vector<SeqItem> make_items(int64_t n, const int64_t* len, const int32_t* origin) {
  std::vector<SeqItem> items;
  items.reserve(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    items.push_back({i, "m", 0, len[i], origin[i]});
  }
  return items;
}

void export_result(const BalanceResult& r, int d, int64_t n, const int32_t* origin,
                   int32_t* dest_inst, int32_t* dest_slot, double* objective,
                   int32_t* is_identity) {
  std::vector<int> next(static_cast<std::size_t>(d), 0);
  for (int64_t i = 0; i < n; ++i) {
    const SlotRef src{origin[i], next[origin[i]]++};
    const SlotRef dst = r.rearrangement.dest_of(src);
    if (dest_inst) dest_inst[i] = dst.instance;
    if (dest_slot) dest_slot[i] = dst.slot;
  }
  if (objective) *objective = r.objective_value;
  if (is_identity) *is_identity = r.rearrangement.is_identity() ? 1 : 0;
}

BalancePolicy make_policy(int kind, double lambda, int64_t v) {
  BalancePolicy p;
  p.kind = static_cast<PolicyKind>(kind);
  p.lambda = lambda;
  p.tolerance_v = v;
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_balance(int kind, double lambda, int64_t v, int d, int64_t n, const int64_t* len,
                const int32_t* origin, int32_t* dest_inst, int32_t* dest_slot, double* objective,
                int32_t* is_identity) {
  try {
    const auto items = make_items(n, len, origin);
    const BalanceResult r = balance(make_policy(kind, lambda, v), d, items);
    export_result(r, d, n, origin, dest_inst, dest_slot, objective, is_identity);
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_identity(int kind, double lambda, int64_t v, int d, int64_t n, const int64_t* len,
                 const int32_t* origin, int32_t* dest_inst, int32_t* dest_slot,
                 double* objective) {
  try {
    const auto items = make_items(n, len, origin);
    const BalanceResult r = identity_arrangement(make_policy(kind, lambda, v), d, items);
    export_result(r, d, n, origin, dest_inst, dest_slot, objective, nullptr);
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_min_feasible_padded_bound(int d, int64_t n, const int64_t* len, const int32_t* origin,
                                  int64_t* out) {
  try {
    *out = min_feasible_padded_bound(d, make_items(n, len, origin));
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_padded_bound_feasible(int d, int64_t n, const int64_t* len, const int32_t* origin,
                              int64_t bound, int32_t* out) {
  try {
    *out = padded_bound_feasible(d, make_items(n, len, origin), bound) ? 1 : 0;
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_cost(double alpha, double beta, int padded, int variant, int64_t n, const int64_t* len,
             int batch_padded, double* out) {
  try {
    CostModel m{alpha, beta, padded ? PaddingMode::Padded : PaddingMode::Unpadded,
                static_cast<CostVariant>(variant)};
    MiniBatch b;
    b.padding_mode = batch_padded ? PaddingMode::Padded : PaddingMode::Unpadded;
    for (int64_t i = 0; i < n; ++i) b.items.push_back({i, "m", 0, len[i], 0});
    *out = cost(m, b);
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// solve_hosting (topology.hpp:71) on a d*d volume matrix (src-major) with
// instances_per_node = c (bandwidths 1: only the hosting matters).
int ref_solve_hosting(int d, int c, const int64_t* V, int32_t* hosting, int64_t* max_egress,
                      int64_t* nodes_visited) {
  try {
    VolumeMatrix vm(d);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) vm.at(i, j) = V[static_cast<size_t>(i) * d + j];
    ClusterTopology topo{d, c, 2.0, 1.0};
    const HostingSolution sol = solve_hosting(vm, topo);
    for (int b = 0; b < d; ++b) hosting[b] = sol.hosting[static_cast<size_t>(b)];
    *max_egress = sol.max_egress;
    *nodes_visited = sol.nodes_visited;
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// Times `reps` back-to-back calls of the reference balance() on prebuilt
// items (the reference's own operator, stock code path). Writes per-call
// seconds into secs[reps].
int ref_time_balance(int kind, double lambda, int64_t v, int d, int64_t n, const int64_t* len,
                     const int32_t* origin, int reps, double* secs) {
  try {
    const auto items = make_items(n, len, origin);
    const BalancePolicy p = make_policy(kind, lambda, v);
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      BalanceResult res = balance(p, d, items);
      const auto t1 = std::chrono::steady_clock::now();
      secs[r] = std::chrono::duration<double>(t1 - t0).count();
      if (res.new_batches.size() != static_cast<std::size_t>(d)) return 9;
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// Reference synthetic generator (workload.cpp:107-161) with the survey's
// profile sets. mix: 2 = C2 (vision-instruct 0.6,
// text-only 0.4); 3 = C3 MCI (vision 0.4, ASR 0.2, speech-QA 0.2, text 0.2).
// Output: per example, up to 3 parts as (modality code, metadata length);
// modality codes 0 text, 1 vision, 2 audio; parts_per_example[n] and
// flattened part arrays sized 3*n.
int ref_generate(int mix, int n, uint64_t seed, int32_t* parts_per_example, int32_t* modality,
                 int64_t* meta_len) {
  try {
    auto lognormal = [](double mu, double sigma, int64_t lo, int64_t hi) {
      LengthDist d;
      d.kind = DistKind::LogNormal;
      d.mu = mu;
      d.sigma = sigma;
      d.clip_min = lo;
      d.clip_max = hi;
      return d;
    };
    TaskProfile vision{"vision-instruct",
                       {{"vision", lognormal(6.5, 0.8, 64, 4096)},
                        {"text", lognormal(5.0, 1.0, 8, 2048)}},
                       0.0, "", ""};
    TaskProfile text{"text-only", {{"text", lognormal(6.0, 1.0, 16, 8192)}}, 0.0, "", ""};
    TaskProfile asr{"asr",
                    {{"audio", lognormal(6.8, 0.6, 50, 3000)},
                     {"text", lognormal(4.0, 0.6, 4, 512)}},
                    0.9, "audio", "text"};
    TaskProfile sqa{"speech-qa",
                    {{"audio", lognormal(6.5, 0.7, 50, 3000)},
                     {"text", lognormal(3.0, 1.2, 2, 1024)}},
                    0.0, "", ""};
    std::vector<TaskProfile> profiles;
    std::vector<double> weights;
    if (mix == 2) {
      profiles = {vision, text};
      weights = {0.6, 0.4};
    } else if (mix == 3) {
      profiles = {vision, asr, sqa, text};
      weights = {0.4, 0.2, 0.2, 0.2};
    } else {
      g_err = "unknown mix";
      return 1;
    }
    const auto examples = generate(profiles, weights, n, seed);
    for (int j = 0; j < n; ++j) {
      const auto& ex = examples[static_cast<std::size_t>(j)];
      parts_per_example[j] = static_cast<int32_t>(ex.parts.size());
      for (std::size_t p = 0; p < ex.parts.size(); ++p) {
        const auto& m = ex.parts[p].modality;
        modality[3 * j + p] = m == "text" ? 0 : (m == "vision" ? 1 : 2);
        meta_len[3 * j + p] = ex.parts[p].metadata_length;
      }
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

}  // extern "C"
