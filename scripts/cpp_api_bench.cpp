// Latency of the reference's C++ API, orchsim::balance(policy, d, items), on the
// BASELINE phase inputs: built twice from this one source, against the B200
// host adapter (liborchsim_b200_host.so) and against the unmodified reference
// objects (oracle/_ref), so the drop-in is timed call for call. Inputs are the
// phase files written by scripts/dump_phases.py (n, d, kind, v, lambda, len[n],
// origin[n]). Prints one JSON line per file: median and min microseconds over
// the repetitions after one warm-up call, objective and a checksum of the
// rearrangement (dest instance, dest slot per source slot).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "orchsim/balancers.hpp"

int main(int argc, char** argv) {
  const int reps = 20;
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
    std::vector<orchsim::SeqItem> items(n);
    for (int64_t i = 0; i < n; ++i) {
      items[i].example_id = i;
      items[i].modality = "text";
      items[i].part_index = 0;
      items[i].length = len[i];
      items[i].origin_instance = org[i];
    }
    orchsim::BalancePolicy pol;
    pol.kind = static_cast<orchsim::PolicyKind>(hdr[2]);
    pol.tolerance_v = hdr[3];
    pol.lambda = lam;
    auto res = orchsim::balance(pol, d, items);  // warm-up (device context, staging)
    std::vector<double> us;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      res = orchsim::balance(pol, d, items);
      const auto t1 = std::chrono::steady_clock::now();
      us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    std::sort(us.begin(), us.end());
    uint64_t sum = 1469598103934665603ull;  // FNV-1a over dest (instance, slot) per batch slot
    for (const auto& b : res.new_batches)
      for (const auto& it : b.items) {
        sum = (sum ^ static_cast<uint64_t>(it.example_id)) * 1099511628211ull;
        sum = (sum ^ static_cast<uint64_t>(it.origin_instance)) * 1099511628211ull;
      }
    std::printf("{\"file\": \"%s\", \"n\": %lld, \"d\": %d, \"kind\": %lld, \"median_us\": %.1f, "
                "\"min_us\": %.1f, \"objective\": %.17g, \"checksum\": \"%016llx\"}\n",
                argv[f], static_cast<long long>(n), d, static_cast<long long>(hdr[2]),
                us[us.size() / 2], us[0], res.objective_value, static_cast<unsigned long long>(sum));
  }
  return 0;
}
