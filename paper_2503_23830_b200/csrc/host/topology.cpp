// orchsim topology subset over the B200 C-ABI: the volume matrix of a
// rearrangement is accumulated by the sm_100a kernel (orch_volume_matrix);
// semantics of /root/reference/proj/src/topology.cpp:12-53.
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

}  // namespace orchsim
