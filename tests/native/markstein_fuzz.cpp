// Fuzz: Markstein division with a correctly rounded reciprocal equals IEEE
// division (round-to-nearest) on random, adversarial and LDLT-like operands.
// Built with -mfma -ffp-contract=off so std::fma is the hardware instruction.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

static inline bool safe(double a, double b) {  // same guard as the device code
  const double aa = std::fabs(a), ab = std::fabs(b);
  return aa >= 0x1p-400 && aa < 0x1p+400 && ab >= 0x1p-400 && ab < 0x1p+400;
}
static inline double mdiv(double a, double b, double y) {
  // dbag_exact.cu ldlt_col (MD): zeros, denormals, huge values, NaN and inf
  // leave the guarded exponent band and take IEEE '/' (the out-of-line solve)
  if (!safe(a, b)) return a / b;
  const double q0 = a * y;
  const double r = std::fma(-q0, b, a);
  return std::fma(r, y, q0);
}
static inline double bits(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }

int main(int argc, char** argv) {
  const long long N = argc > 1 ? atoll(argv[1]) : 20000000;
  std::mt19937_64 g(12345);
  long long bad = 0, tested = 0;
  auto check = [&](double a, double b) {
    const volatile double y = 1.0 / b;  // correctly rounded reciprocal
    const double q = mdiv(a, b, y), e = a / b;
    ++tested;
    if (std::memcmp(&q, &e, 8) != 0 && !(std::isnan(q) && std::isnan(e))) {  // sign of 0 too
      if (bad < 10) std::printf("MISMATCH a=%a b=%a q=%a e=%a\n", a, b, q, e);
      ++bad;
    }
  };
  for (long long i = 0; i < N; ++i) {
    // random bit patterns in a wide exponent band
    // the whole guarded band [2^-400, 2^400] and a little beyond it
    const uint64_t ea = 1023 - 410 + g() % 821, eb = 1023 - 410 + g() % 821;
    const uint64_t ma = g() & ((1ull << 52) - 1), mb = g() & ((1ull << 52) - 1);
    double a = bits((ea << 52) | ma), b = bits((eb << 52) | mb);
    if (g() & 1) a = -a;
    if (g() & 1) b = -b;
    check(a, b);
    // adversarial divisors: significand all ones / nearly one / powers of two
    const uint64_t specials[] = {(1ull << 52) - 1, (1ull << 52) - 2, 0, 1, 2, (1ull << 51),
                                 (1ull << 51) - 1};
    check(a, bits((eb << 52) | specials[g() % 7]));
    // adversarial numerators near b * k
    const double bb = bits((eb << 52) | mb);
    check(std::nextafter(bb * 3.0, 0.0), bb);
    check(std::nextafter(bb * 7.0, 1e300), bb);
    // LDLT-like: numerator a sum of products, divisor a pivot
    check(a * 0.5 + b * 1e-3, std::fabs(b) + 0.5);
    // signed zero numerators
    check(0.0, b);
    check(-0.0, b);
  }
  std::printf("tested %lld mismatches %lld\n", tested, bad);
  return bad != 0;
}
