// The exchange side of the reference's C++ API on the BASELINE phase inputs,
// built twice from this one source: against the B200 host adapter
// (liborchsim_b200_host.so) and against the unmodified reference objects
// (oracle/_ref). For every phase file (format of scripts/cpp_api_bench.cpp)
// it balances once, then times and prints:
//   * stats_of (orchestrator.cpp:91-102) of the origin and new batches,
//     restated over the public cost() exactly as the orchestrator calls it
//     (one cost() per batch);
//   * make_exchange_plan (AllToAll, AllGather) and simulate_exchange
//     (exchange.cpp:49-113) on a topology of `c` instances per node;
//   * gather_lengths' metadata volume and a stale-plan rejection;
//   * permutation_invariance_check (topology.cpp:305-316);
//   * d <= 64: nodewise_rearrange on 2 and 8 nodes (topology.cpp:267-303) --
//     hosting, egress, the identity baseline, nodes_visited, the relabelled
//     moves -- and inter_node_egress of the identity hosting.
// Doubles are printed as IEEE bit patterns so the two builds compare exactly.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "orchsim/balancers.hpp"
#include "orchsim/exchange.hpp"
#include "orchsim/topology.hpp"

using namespace orchsim;

namespace {

uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}

struct Stats {
  double max = 0.0, mean = 0.0, ratio = 1.0;
};

Stats stats_of(const std::vector<MiniBatch>& batches, const CostModel& model) {
  Stats s;  // orchestrator.cpp:91-102, through the public cost()
  double total = 0.0;
  for (const MiniBatch& b : batches) {
    const double c = cost(model, b);
    s.max = std::max(s.max, c);
    total += c;
  }
  s.mean = batches.empty() ? 0.0 : total / static_cast<double>(batches.size());
  s.ratio = s.mean > 0.0 ? s.max / s.mean : 1.0;
  return s;
}

template <class F>
double median_us(int reps, F&& f) {
  std::vector<double> us;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    f();
    const auto t1 = std::chrono::steady_clock::now();
    us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  std::sort(us.begin(), us.end());
  return us[us.size() / 2];
}

}  // namespace

int main(int argc, char** argv) {
  for (int f = 1; f < argc; ++f) {
    FILE* fp = std::fopen(argv[f], "rb");
    if (!fp) return 2;
    int64_t hdr[4];
    double lam = 0.0;
    if (std::fread(hdr, 8, 4, fp) != 4 || std::fread(&lam, 8, 1, fp) != 1) return 2;
    const int64_t n = hdr[0];
    const int d = static_cast<int>(hdr[1]);
    std::vector<int64_t> len(n);
    std::vector<int32_t> org(n);
    if (std::fread(len.data(), 8, n, fp) != static_cast<size_t>(n) ||
        std::fread(org.data(), 4, n, fp) != static_cast<size_t>(n))
      return 2;
    std::fclose(fp);
    std::vector<SeqItem> items(n);
    for (int64_t i = 0; i < n; ++i) {
      items[i].example_id = i;
      items[i].modality = "text";
      items[i].part_index = 0;
      items[i].length = len[i];
      items[i].origin_instance = org[i];
    }
    BalancePolicy pol;
    pol.kind = static_cast<PolicyKind>(hdr[2]);
    pol.tolerance_v = hdr[3];
    pol.lambda = lam;
    const BalanceResult res = balance(pol, d, items);
    const CostModel model = policy_cost_model(pol);
    const std::vector<MiniBatch> in = batches_from_items(d, items, model.padding_mode);
    const int reps = d >= 1024 ? 5 : 20;

    Stats pre, post;
    const double t_stats = median_us(reps, [&] {
      pre = stats_of(in, model);
      post = stats_of(res.new_batches, model);
    });

    ClusterTopology topo;
    topo.instance_count = d;
    topo.instances_per_node = d >= 8 ? d / 8 : 1;  // 8 nodes (GPUs) where d allows
    topo.intra_bandwidth = 900.0;
    topo.inter_bandwidth = 50.0;
    ExchangePlan a2a, ag;
    const double t_plan = median_us(reps, [&] {
      a2a = make_exchange_plan(in, res.rearrangement, ExchangeMode::AllToAll);
    });
    ag = make_exchange_plan(in, res.rearrangement, ExchangeMode::AllGather);
    std::pair<std::vector<MiniBatch>, ExchangeCostReport> xa, xg;
    const double t_sim = median_us(reps, [&] { xa = simulate_exchange(a2a, in, topo, 1.37); });
    xg = simulate_exchange(ag, in, topo, 1.0);
    bool stale_rejected = false;
    {
      ExchangePlan bad = a2a;
      bad.per_pair_volumes.at(0, d - 1) += 1;
      try {
        simulate_exchange(bad, in, topo);
      } catch (const std::invalid_argument&) {
        stale_rejected = true;
      }
    }
    // every instance gets a copy of the table: d copies of n records (skipped at d = 2560)
    const GatheredLengths g = d <= 256 ? gather_lengths(in) : GatheredLengths{};
    bool perm_ok = false;
    const double t_perm =
        median_us(reps, [&] { perm_ok = permutation_invariance_check(in, in, model); });
    const bool perm_changed = permutation_invariance_check(in, res.new_batches, model);

    // node-wise hosting on 2 and 8 nodes (d <= 64: the reference's search is
    // exponential beyond)
    std::string hosting = "[";
    double t_host = 0.0;
    for (int nodes : {2, 8}) {
      if (d > 64 || d % nodes || nodes > d) continue;
      ClusterTopology tn = topo;
      tn.instances_per_node = d / nodes;
      NodewiseResult nw;
      const double t = median_us(d >= 64 ? 3 : reps, [&] { nw = nodewise_rearrange(in, res.rearrangement, tn); });
      if (nodes == 8) t_host = t;
      const VolumeMatrix vm = volume_matrix(in, res.rearrangement);
      const std::vector<int64_t> base = inter_node_egress(vm, tn, identity_hosting(tn));
      uint64_t h = 1469598103934665603ull;
      for (int b = 0; b < d; ++b) {
        h = (h ^ static_cast<uint64_t>(nw.hosting[b])) * 1099511628211ull;
        h = (h ^ static_cast<uint64_t>(nw.batch_to_instance[b])) * 1099511628211ull;
      }
      for (const auto& kv : nw.rearrangement.moves()) {
        h = (h ^ static_cast<uint64_t>(kv.second.instance)) * 1099511628211ull;
        h = (h ^ static_cast<uint64_t>(kv.second.slot)) * 1099511628211ull;
      }
      std::string eg, be;
      for (size_t k = 0; k < nw.per_node_egress.size(); ++k)
        eg += (k ? ", " : "") + std::to_string(nw.per_node_egress[k]);
      for (size_t k = 0; k < base.size(); ++k) be += (k ? ", " : "") + std::to_string(base[k]);
      hosting += std::string(hosting.size() > 1 ? ", " : "") + "{\"nodes\": " +
                 std::to_string(nodes) + ", \"max\": " + std::to_string(nw.max_egress) +
                 ", \"baseline\": " + std::to_string(nw.baseline_max_egress) +
                 ", \"visited\": " + std::to_string(nw.nodes_visited) + ", \"egress\": [" + eg +
                 "], \"identity_egress\": [" + be + "], \"hash\": \"" + std::to_string(h) + "\"}";
    }
    hosting += "]";

    uint64_t moved_sum = 1469598103934665603ull;
    for (const auto& b : xa.first)
      for (const auto& it : b.items) moved_sum = (moved_sum ^ static_cast<uint64_t>(it.example_id)) * 1099511628211ull;
    uint64_t vsum = 1469598103934665603ull;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        vsum = (vsum ^ static_cast<uint64_t>(a2a.per_pair_volumes.at(i, j))) * 1099511628211ull;
        vsum = (vsum ^ static_cast<uint64_t>(ag.per_pair_volumes.at(i, j))) * 1099511628211ull;
      }
    auto report = [](const ExchangeCostReport& r) {
      std::string s = "{\"t\": \"" + std::to_string(bits(r.modeled_time)) +
                      "\", \"bottleneck\": " + std::to_string(static_cast<int>(r.bottleneck)) +
                      ", \"inter\": " + std::to_string(r.total_inter_volume) +
                      ", \"intra\": " + std::to_string(r.total_intra_volume) +
                      ", \"local\": " + std::to_string(r.local_volume) +
                      ", \"peak\": " + std::to_string(r.peak_resident_volume) + ", \"egress\": [";
      for (size_t k = 0; k < r.per_node_egress.size(); ++k)
        s += (k ? ", " : "") + std::to_string(r.per_node_egress[k]);
      return s + "]}";
    };
    std::printf(
        "{\"file\": \"%s\", \"n\": %lld, \"d\": %d, \"stats_us\": %.1f, \"plan_us\": %.1f, "
        "\"simulate_us\": %.1f, \"perm_check_us\": %.1f, \"pre\": [\"%llu\", \"%llu\", \"%llu\"], "
        "\"post\": [\"%llu\", \"%llu\", \"%llu\"], \"volumes\": \"%016llx\", \"moved\": "
        "\"%016llx\", \"a2a\": %s, \"ag\": %s, \"stale_rejected\": %d, \"metadata_volume\": %lld, "
        "\"views\": %zu, \"perm_same\": %d, \"perm_new\": %d, \"hosting_us\": %.1f, "
        "\"hosting\": %s}\n",
        argv[f], static_cast<long long>(n), d, t_stats, t_plan, t_sim, t_perm,
        static_cast<unsigned long long>(bits(pre.max)), static_cast<unsigned long long>(bits(pre.mean)),
        static_cast<unsigned long long>(bits(pre.ratio)), static_cast<unsigned long long>(bits(post.max)),
        static_cast<unsigned long long>(bits(post.mean)),
        static_cast<unsigned long long>(bits(post.ratio)), static_cast<unsigned long long>(vsum),
        static_cast<unsigned long long>(moved_sum), report(xa.second).c_str(),
        report(xg.second).c_str(), stale_rejected ? 1 : 0,
        static_cast<long long>(g.metadata_volume), g.views.size(), perm_ok ? 1 : 0,
        perm_changed ? 1 : 0, t_host, hosting.c_str());
    std::fflush(stdout);
  }
  return 0;
}
