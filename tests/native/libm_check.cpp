// CPU check (test infrastructure): glibc_libm.cuh's restatement of glibc's
// FMA-path exp/log/cos against the host libm, on the generator's own input
// domains (1 - u01, 2*pi*u01, mu + sigma*normal, workload.cpp:19-28, 58) and
// on wide random ranges.  Built by tests/test_libm.py with
//   g++ -O2 -mfma -ffp-contract=off  (fma() inlines to one vfmadd, nothing else fuses)
// Usage: libm_check <draws per domain> <seed>; prints one JSON line.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../../paper_2512_16134_b200/csrc/glibc_libm.cuh"

namespace g = sbs::glibc;

static uint64_t bits(double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; }
static double from_bits(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }

struct Tally {
  const char* name;
  uint64_t n = 0, bad = 0;
  double first_x = 0;
  void check(double x, double want, double got) {
    ++n;
    if (bits(want) != bits(got) && !(std::isnan(want) && std::isnan(got))) {
      if (bad == 0) first_x = x;
      ++bad;
    }
  }
};

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  const uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
  std::mt19937_64 rng(seed);
  auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  Tally t[9] = {{"log_gen"}, {"log_wide"}, {"log_near1"}, {"cos_gen"}, {"cos_wide"},
                {"cos_small"}, {"exp_gen"}, {"exp_wide"}, {"exp_edge"}};
  volatile double sink = 0;
  for (uint64_t i = 0; i < n; ++i) {
    // generator domains
    double a = u01(), b = u01();
    double x = 1.0 - a;
    t[0].check(x, std::log(x), g::log(x));
    double c = kTwoPi * b;
    t[3].check(c, std::cos(c), g::cos(c));
    double r = std::sqrt(-2.0 * std::log(1.0 - u01()));
    double z = r * std::cos(kTwoPi * u01());
    double mu = 10.0 * u01() - 2.0, sg = 2.0 * u01();
    double e = mu + sg * z;
    t[6].check(e, std::exp(e), g::exp(e));
    // wide ranges: any positive finite double for log
    double w = from_bits(rng() & 0x7fefffffffffffffull);
    t[1].check(w, std::log(w), g::log(w));
    double w1 = 1.0 + (u01() - 0.5) * 0.14;
    t[2].check(w1, std::log(w1), g::log(w1));
    // cos: log-uniform magnitude up to 1e8, both signs
    double m = std::ldexp(1.0 + u01(), (int)(rng() % 56) - 30) * ((rng() & 1) ? 1 : -1);
    if (std::fabs(m) < 105414350.0) t[4].check(m, std::cos(m), g::cos(m));
    double sm = (u01() - 0.5) * 6.0;
    t[5].check(sm, std::cos(sm), g::cos(sm));
    // exp: the whole finite range incl. the subnormal / overflow specialcases
    double ew = (u01() - 0.5) * 1500.0;
    t[7].check(ew, std::exp(ew), g::exp(ew));
    double ed = std::ldexp((u01() - 0.5), -(int)(rng() % 70));
    t[8].check(ed, std::exp(ed), g::exp(ed));
    sink = sink + x;
  }
  // exact boundaries
  const double edges[] = {0.0, -0.0, 1.0, 0x1p-53, 0x1p-27, -0x1p-27, 0.85546875, -0.85546875,
                          0.8554687499999999, 2.426265, 2.4262650000000003, 1.5707963267948966,
                          3.141592653589793, 6.283185307179586, 512.0, -512.0, 709.7, -708.0,
                          -745.0, 0x1p-54, 0x1p-55, 1e-300, 0.9375, 1.064697265625};
  for (double x : edges) {
    t[8].check(x, std::exp(x), g::exp(x));
    if (x > 0) t[1].check(x, std::log(x), g::log(x));
    t[5].check(x, std::cos(x), g::cos(x));
  }
  std::printf("{");
  for (int k = 0; k < 9; ++k)
    std::printf("%s\"%s\": [%llu, %llu, %.17g]", k ? ", " : "", t[k].name,
                (unsigned long long)t[k].n, (unsigned long long)t[k].bad, t[k].first_x);
  std::printf("}\n");
  return 0;
}
