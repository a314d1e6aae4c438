// Test driver (test infrastructure): the shim's schedule_decode_batch — the
// reference's signature (decode_alloc.h:70-72) running on the B200 through
// sbs_decode_schedule_batch — on batches read from a file, printing what the
// reference's caller and observer would see.  tests/test_gpu_alloc.py
// compares it with the reference's own function.
//   input : per batch "k M U", then M lines "id sort_len kv_len", U lines "B K"
//   output: per batch one line: placements, thresholds, fallbacks, units after
#include <cstdio>
#include <vector>

#include "sbsim/decode_alloc.h"

using namespace sbsim;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  FILE* f = std::fopen(argv[1], "r");
  if (!f) return 2;
  double k;
  long m, u;
  while (std::fscanf(f, "%lf %ld %ld", &k, &m, &u) == 3) {
    std::vector<DecodeCandidate> c((size_t)m);
    for (auto& x : c) {
      unsigned long long id;
      long long sl, kl;
      if (std::fscanf(f, "%llu %lld %lld", &id, &sl, &kl) != 3) return 2;
      x = DecodeCandidate{id, sl, kl};
    }
    std::vector<DecodeUnitPlan> units((size_t)u);
    for (long i = 0; i < u; ++i) {
      long long b, kv;
      if (std::fscanf(f, "%lld %lld", &b, &kv) != 2) return 2;
      units[(size_t)i] = DecodeUnitPlan{(int)i, (int)b, kv};
    }
    std::vector<double> th;
    std::vector<int> fb;
    auto pl = schedule_decode_batch(c, units, k, [&](const DecodePlacementInfo& info) {
      th.push_back(info.threshold);
      fb.push_back(info.fallback ? 1 : 0);
    });
    std::printf("P");
    for (auto& p : pl) std::printf(" %llu %d", (unsigned long long)p.first, p.second);
    std::printf(" T");
    for (double t : th) std::printf(" %.17g", t);
    std::printf(" F");
    for (int x : fb) std::printf(" %d", x);
    std::printf(" U");
    for (auto& x : units) std::printf(" %d %lld", x.batch, (long long)x.kv);
    std::printf("\n");
  }
  return 0;
}
