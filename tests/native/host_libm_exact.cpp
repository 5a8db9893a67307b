// Host build of paper_2408_12057_b200/csrc/libm_exact.cuh for the CPU test suite
// (tests/test_libm_exact.py): the device source itself, with its CUDA intrinsics mapped
// to the IEEE operations they denote, compiled -ffp-contract=off so nothing is fused
// except the explicit fma()s.  Checks the table and constants without a GPU.
#include <cmath>
#include <cstdint>
#include <cstring>

#define __device__
#define __forceinline__ inline
#define __noinline__
static inline double __dadd_rn(double a, double b) { return a + b; }
static inline double __dsub_rn(double a, double b) { return a - b; }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline double __ddiv_rn(double a, double b) { return a / b; }
static inline double __fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
static inline long long __double_as_longlong(double x) {
  long long r;
  std::memcpy(&r, &x, 8);
  return r;
}
static inline double __longlong_as_double(long long x) {
  double r;
  std::memcpy(&r, &x, 8);
  return r;
}

#include "libm_exact.cuh"

extern "C" void host_gexp(const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = asmcdev::gexp(x[i]);
}
extern "C" void host_crlog(const double* x, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = asmcdev::crlog(x[i]);
}
// mismatch counts against the host libm over n pseudo-random arguments of each kind
extern "C" void host_sweep(uint64_t n, uint64_t seed, uint64_t* exp_bad, uint64_t* log_bad) {
  uint64_t s = seed | 1, eb = 0, lb = 0;
  for (uint64_t i = 0; i < n; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    const double u = (double)(s >> 11) * 0x1p-53;
    double x;
    switch (i & 3) {
      case 0: x = -745.2 * u; break;
      case 1: x = -40.0 * u; break;
      case 2: x = -u; break;
      default: x = 1420.0 * u - 720.0; break;
    }
    const double a = asmcdev::gexp(x), b = std::exp(x);
    eb += std::memcmp(&a, &b, 8) != 0;
    const double y = 1.0 + u * 4194303.0;
    const double c = asmcdev::crlog(y), d = std::log(y);
    lb += std::memcmp(&c, &d, 8) != 0;
  }
  *exp_bad = eb;
  *log_bad = lb;
}
