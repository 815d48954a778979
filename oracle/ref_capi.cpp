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
//   run_iteration (composed delivery)   proj/include/orchsim/orchestrator.hpp:131-135
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
#include "orchsim/orchestrator.hpp"
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


// The survey's profile sets through the reference
// generator (workload.cpp:107-161). mix 2 = C2 (vision-instruct 0.6, text-only
// 0.4); mix 3 = C3 MCI (vision 0.4, ASR 0.2, speech-QA 0.2, text 0.2).
bool mix_examples(int mix, int n, uint64_t seed, std::vector<Example>* out) {
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
    return false;
  }
  *out = generate(profiles, weights, n, seed);
  return true;
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
    std::vector<Example> examples;
    if (!mix_examples(mix, n, seed, &examples)) return 1;
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

// One training iteration of the reference orchestrator (run_iteration,
// orchestrator.cpp:563-569) on the mix's examples (ids 0..E-1, origins j % d):
// encoder phases vision (GreedyUnpadded) and, for mix 3, audio (BinaryPadded),
// both rate 4, then the LLM phase (GreedyUnpadded) and the composed delivery
// of the encoder outputs (compose_exchanges on; node-wise hosting as given,
// on d/c nodes). Out, with parts numbered example-major (global part g):
//   llm_dest_inst / llm_dest_slot [E]   the LLM rearrangement of each example
//   asm_inst / asm_pos [parts]          where the backbone's assembled input
//                                       holds the part (outcome.assembled)
//   flags[0] assembly_ok, [1] composed exchanges, [2] delivery exchanges of
//   the vision universe
int ref_run_iteration(int mix, int d, int c, int per_instance, uint64_t seed, int nodewise,
                      int32_t* llm_dest_inst, int32_t* llm_dest_slot, int32_t* asm_inst,
                      int32_t* asm_pos, int32_t* flags) {
  try {
    const int E = d * per_instance;
    std::vector<Example> examples;
    if (!mix_examples(mix, E, seed, &examples)) return 1;
    std::vector<int> origins(static_cast<std::size_t>(E));
    for (int j = 0; j < E; ++j) origins[j] = j % d;
    auto phase = [](const char* name, const char* modality, PolicyKind kind, int64_t rate) {
      PhaseSpec p;
      p.name = name;
      if (modality) p.modality = ModalityId(modality);
      p.policy.kind = kind;
      p.cost_model = policy_cost_model(p.policy);
      p.downsample_rate = rate;
      return p;
    };
    std::vector<PhaseSpec> phases{phase("vision", "vision", PolicyKind::GreedyUnpadded, 4)};
    if (mix == 3) phases.push_back(phase("audio", "audio", PolicyKind::BinaryPadded, 4));
    phases.push_back(phase("llm", nullptr, PolicyKind::GreedyUnpadded, 1));
    ClusterTopology topo{d, c, 2.0, 1.0};
    OrchestratorOptions opt;
    opt.nodewise = nodewise != 0;
    opt.compose_exchanges = true;
    const IterationOutcome out = run_iteration(examples, origins, phases, topo, opt);
    std::vector<int> next(static_cast<std::size_t>(d), 0);
    std::vector<int64_t> part_base(static_cast<std::size_t>(E) + 1, 0);
    for (int j = 0; j < E; ++j) {
      const SlotRef dst = out.llm_rearrangement.dest_of(SlotRef{origins[j], next[origins[j]]++});
      llm_dest_inst[j] = dst.instance;
      llm_dest_slot[j] = dst.slot;
      part_base[j + 1] = part_base[j] + static_cast<int64_t>(examples[j].parts.size());
    }
    for (int64_t g = 0; g < part_base[E]; ++g) asm_inst[g] = asm_pos[g] = -1;
    for (int i = 0; i < d; ++i)
      for (std::size_t k = 0; k < out.assembled[i].size(); ++k) {
        const PlacedPart& pp = out.assembled[i][k];
        const int64_t g = part_base[pp.example_id] + pp.part_index;
        asm_inst[g] = i;
        asm_pos[g] = static_cast<int32_t>(k);
      }
    flags[0] = out.report.assembly_ok ? 1 : 0;
    flags[1] = out.report.composed_exchange_count;
    const auto it = out.report.delivery_exchanges_per_encoder.find("vision");
    flags[2] = it == out.report.delivery_exchanges_per_encoder.end() ? -1 : it->second;
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

}  // extern "C"
