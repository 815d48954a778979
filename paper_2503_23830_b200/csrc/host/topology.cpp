// orchsim topology over the B200 C-ABI: the volume matrix of a rearrangement
// (orch_volume_matrix), node egress (orch_inter_node_egress_host) and the
// hosting search (orch_solve_hosting_host) run on the device; semantics of
// /root/reference/proj/src/topology.cpp:12-316.
#include <algorithm>
#include <numeric>

#include "orchsim/topology.hpp"
#include "runtime.hpp"

namespace orchsim {

void validate_topology(const ClusterTopology& t) {  // topology.cpp:12-22
  if (t.instance_count < 1 || t.instances_per_node < 1)
    throw std::invalid_argument("topology needs at least one instance and one per node");
  if (t.instance_count % t.instances_per_node != 0)
    throw std::invalid_argument("instance count must be divisible by instances per node");
  if (t.inter_bandwidth <= 0.0 || t.intra_bandwidth < t.inter_bandwidth)
    throw std::invalid_argument("bandwidths must satisfy intra >= inter > 0");
}

std::int64_t VolumeMatrix::row_sum(int i) const {
  std::int64_t s = 0;
  for (int j = 0; j < d_; ++j) s += at(i, j);
  return s;
}

std::int64_t VolumeMatrix::column_sum(int j) const {
  std::int64_t s = 0;
  for (int i = 0; i < d_; ++i) s += at(i, j);
  return s;
}

std::int64_t VolumeMatrix::total() const {
  return std::accumulate(v_.begin(), v_.end(), std::int64_t{0});
}

VolumeMatrix volume_matrix(const std::vector<MiniBatch>& batches, const Rearrangement& re) {
  const int d = re.instance_count();
  if (static_cast<int>(batches.size()) != d)
    throw std::invalid_argument("rearrangement instance count does not match batch count");
  std::vector<std::int64_t> len;
  std::vector<int32_t> src, dst;
  len.reserve(re.size());
  src.reserve(re.size());
  dst.reserve(re.size());
  for (const auto& kv : re.moves()) {
    const SlotRef& s = kv.first;
    if (s.instance >= d || s.slot >= static_cast<int>(batches[s.instance].items.size()))
      throw std::invalid_argument("rearrangement covers a slot absent from the input batches");
    len.push_back(batches[s.instance].items[s.slot].length);
    src.push_back(s.instance);
    dst.push_back(kv.second.instance);
  }
  VolumeMatrix V(d);
  if (d > 0)
    b200::check(orch_volume_matrix_host(b200::context(), d, static_cast<std::int64_t>(len.size()),
                                        len.data(), src.data(), dst.data(), V.data(), nullptr));
  return V;
}

std::vector<int> identity_hosting(const ClusterTopology& topo) {  // topology.cpp:55-59
  std::vector<int> h(static_cast<std::size_t>(topo.instance_count));
  for (int b = 0; b < topo.instance_count; ++b) h[b] = topo.node_of(b);
  return h;
}

namespace {

// A hosting must name a node for every batch and give each node exactly c
// batches (topology.cpp:61-80); the egress itself is summed on the device.
void require_balanced_hosting(const ClusterTopology& topo, const std::vector<int>& hosting) {
  std::vector<int> load(static_cast<std::size_t>(topo.node_count()), 0);
  for (int node : hosting) {
    if (node < 0 || node >= topo.node_count())
      throw std::invalid_argument("hosting references unknown node");
    ++load[static_cast<std::size_t>(node)];
  }
  if (std::any_of(load.begin(), load.end(), [&](int k) { return k != topo.instances_per_node; }))
    throw std::invalid_argument("hosting must place exactly c batches per node");
}

std::vector<std::int64_t> device_egress(const VolumeMatrix& v, const ClusterTopology& topo,
                                        const std::vector<int>& hosting) {
  const std::vector<int32_t> h(hosting.begin(), hosting.end());
  std::vector<std::int64_t> e(static_cast<std::size_t>(topo.node_count()));
  b200::check(orch_inter_node_egress_host(b200::context(), topo.instance_count,
                                          topo.instances_per_node, v.data(), h.data(), e.data(),
                                          nullptr));
  return e;
}

// solve_hosting's search on the device; info = {max egress, identity hosting's
// max egress, leaf used, the reference's nodes_visited}
HostingSolution search(const VolumeMatrix& v, const ClusterTopology& topo, std::int64_t info[4]) {
  validate_topology(topo);
  if (v.dimension() != topo.instance_count)
    throw std::invalid_argument("volume matrix dimension does not match topology");
  std::vector<int32_t> h(static_cast<std::size_t>(topo.instance_count));
  b200::check(orch_solve_hosting_host(b200::context(), topo.instance_count,
                                      topo.instances_per_node, v.data(), h.data(), info, nullptr));
  HostingSolution sol;
  sol.hosting.assign(h.begin(), h.end());
  sol.per_node_egress = device_egress(v, topo, sol.hosting);
  sol.max_egress = info[0];
  sol.nodes_visited = info[3];
  return sol;
}

}  // namespace

std::vector<std::int64_t> inter_node_egress(const VolumeMatrix& v, const ClusterTopology& topo,
                                            const std::vector<int>& hosting) {  // :61-89
  validate_topology(topo);
  if (v.dimension() != topo.instance_count ||
      static_cast<int>(hosting.size()) != topo.instance_count)
    throw std::invalid_argument("volume matrix / hosting size does not match topology");
  require_balanced_hosting(topo, hosting);
  return device_egress(v, topo, hosting);
}

HostingSolution solve_hosting(const VolumeMatrix& volumes, const ClusterTopology& topo) {
  std::int64_t info[4] = {0, 0, 0, 0};  // topology.cpp:179-265
  return search(volumes, topo, info);
}

NodewiseResult nodewise_rearrange(const std::vector<MiniBatch>& batches, const Rearrangement& re,
                                  const ClusterTopology& topo) {  // topology.cpp:267-303
  validate_topology(topo);
  if (re.instance_count() != topo.instance_count)
    throw std::invalid_argument("rearrangement instance count does not match topology");
  std::int64_t info[4] = {0, 0, 0, 0};
  HostingSolution sol = search(volume_matrix(batches, re), topo, info);
  // within a node, its batches take its instances in ascending batch order
  std::vector<int> seat(static_cast<std::size_t>(topo.node_count()), 0);
  NodewiseResult r;
  r.batch_to_instance.resize(sol.hosting.size());
  for (std::size_t b = 0; b < sol.hosting.size(); ++b)
    r.batch_to_instance[b] = sol.hosting[b] * topo.instances_per_node + seat[sol.hosting[b]]++;
  std::map<SlotRef, SlotRef> moves;
  for (const auto& kv : re.moves())
    moves.emplace(kv.first, SlotRef{r.batch_to_instance[kv.second.instance], kv.second.slot});
  r.rearrangement = Rearrangement(topo.instance_count, std::move(moves));
  r.hosting = std::move(sol.hosting);
  r.max_egress = sol.max_egress;
  r.per_node_egress = std::move(sol.per_node_egress);
  r.baseline_max_egress = info[1];  // the identity hosting's, from the same device pass
  r.nodes_visited = sol.nodes_visited;
  return r;
}

bool permutation_invariance_check(const std::vector<MiniBatch>& before,
                                  const std::vector<MiniBatch>& after, const CostModel& model) {
  // topology.cpp:305-316
  if (before.size() != after.size()) return false;
  std::vector<const MiniBatch*> all;
  all.reserve(before.size() + after.size());
  for (const MiniBatch& b : before) all.push_back(&b);
  for (const MiniBatch& b : after) all.push_back(&b);
  std::vector<double> c = b200::batch_costs(model, all);
  const auto mid = c.begin() + static_cast<std::ptrdiff_t>(before.size());
  std::sort(c.begin(), mid);
  std::sort(mid, c.end());
  return std::equal(c.begin(), mid, mid, c.end());
}

}  // namespace orchsim
