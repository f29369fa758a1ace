// det_sincos (oracle/oracle.cpp, the portable sin/cos that the oracle and the
// EXACT kernels share) against glibc's std::sin / std::cos, the functions the
// reference calls (proj/src/geometry.cpp:9-28). Prints the histogram of the
// distance in ulps over N arguments per range and exits 1 if any exceeds 1.
//   g++ -O2 -ffp-contract=off -std=c++20 -I oracle sincos_vs_glibc.cpp oracle/oracle.cpp
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "oracle.hpp"

static int64_t ordinal(double x) {
  int64_t b;
  std::memcpy(&b, &x, 8);
  return b < 0 ? (int64_t)0x8000000000000000ULL - b : b;  // monotone over all finite doubles
}
static int64_t ulps(double a, double b) {
  const int64_t d = ordinal(a) - ordinal(b);
  return d < 0 ? -d : d;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 100000000;
  struct Range {
    const char* name;
    double lo, hi;
    bool log;
    double share;
  } ranges[] = {{"[-pi,pi] (scene Euler angles)", -M_PI, M_PI, false, 0.7},
                {"[-100,100] (drifting copies)", -100.0, 100.0, false, 0.2},
                {"+-[1e-8,1] log-uniform (small angles)", 1e-8, 1.0, true, 0.1}};
  std::mt19937_64 rng(12345);
  int64_t worst_all = 0;
  for (const Range& r : ranges) {
    const int64_t m = (int64_t)(n * r.share);
    int64_t hist[4] = {0, 0, 0, 0};  // 0, 1, 2, >2 ulps (sin and cos counted separately)
    int64_t worst = 0;
    double worst_x = 0;
    for (int64_t i = 0; i < m; ++i) {
      const double u = (double)(rng() >> 11) * 0x1p-53;
      double x;
      if (r.log) {
        x = std::exp(std::log(r.lo) + u * (std::log(r.hi) - std::log(r.lo)));
        if (rng() & 1) x = -x;
      } else {
        x = r.lo + u * (r.hi - r.lo);
      }
      double s, c;
      orc::det_sincos(x, &s, &c);
      const int64_t ds = ulps(s, std::sin(x)), dc = ulps(c, std::cos(x));
      for (int64_t d : {ds, dc}) {
        ++hist[d > 2 ? 3 : d];
        if (d > worst) {
          worst = d;
          worst_x = x;
        }
      }
    }
    std::printf("%-40s n=%lld  0ulp %.6f  1ulp %.6f  2ulp %lld  >2ulp %lld  max %lld (x=%.17g)\n",
                r.name, (long long)m, hist[0] / (2.0 * m), hist[1] / (2.0 * m), (long long)hist[2],
                (long long)hist[3], (long long)worst, worst_x);
    if (worst > worst_all) worst_all = worst;
  }
  std::printf("max ulps %lld\n", (long long)worst_all);
  return worst_all <= 1 ? 0 : 1;
}
