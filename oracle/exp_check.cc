// TEST INFRASTRUCTURE ONLY: the device exp restatement (csrc/libm_exp.cuh)
// compiled for the host, compared with the host's std::exp (the reference's
// map exp, ops.cc:24) on random and edge-case doubles.
//   g++ -O2 -ffp-contract=off oracle/exp_check.cc -o /tmp/exp_check && /tmp/exp_check 100000000
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#define __device__
#define __constant__
#define __forceinline__ inline
static inline double __fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
static inline double __dadd_rn(double a, double b) { return a + b; }
static inline double __dsub_rn(double a, double b) { return a - b; }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline long long __double_as_longlong(double d) { long long u; std::memcpy(&u, &d, 8); return u; }
static inline double __longlong_as_double(long long u) { double d; std::memcpy(&d, &u, 8); return d; }
#include "../paper_2410_02682_b200/csrc/libm_exp.cuh"

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 10000000;
  std::mt19937_64 g(7);
  long long bad = 0, total = 0;
  auto check = [&](double x) {
    const double a = ed::libm_exp(x), b = std::exp(x);
    ++total;
    if (std::memcmp(&a, &b, 8) != 0 && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 10) std::printf("x=%a dev=%a host=%a\n", x, a, b);
      ++bad;
    }
  };
  std::uniform_real_distribution<double> wide(-750.0, 720.0), mid(-40.0, 40.0), small(-1.0, 1.0);
  for (long long i = 0; i < n; ++i) {
    check(wide(g));
    check(mid(g));
    check(small(g));
    uint64_t u = g();  // any bit pattern
    double x;
    std::memcpy(&x, &u, 8);
    check(x);
  }
  const double edge[] = {0.0, -0.0, 1e-300, -1e-300, 0x1p-54, -0x1p-54, 0x1p-55, 512.0, -512.0, 709.782712893384,
                         709.79, -708.39641853226408, -708.4, -745.13321910194110, -745.2, 1024.0, -1024.0,
                         INFINITY, -INFINITY, NAN, 7.0978271289338397e+02, -7.4513321910194122e+02};
  for (double x : edge) check(x);
  std::printf("%lld / %lld differ\n", bad, total);
  return bad != 0;
}
