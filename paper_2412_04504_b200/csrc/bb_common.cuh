// bb_common.cuh -- shared device/host helpers for the B200 binbatch engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math_constants.h>

#include "binbatch_b200.h"

#define BB_HD __host__ __device__ __forceinline__
// std::numeric_limits<double>::quiet_NaN() bit pattern (CUDART_NAN has the sign bit set)
#define BB_QNAN __longlong_as_double(0x7ff8000000000000LL)

namespace bb {

// host-side launch accounting (bb_launch_count)
void note_launch(unsigned n = 1);
// kernels this thread has noted so far (a captured graph's launch count)
unsigned long long launches_noted_here();

// ----------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11).  Replaces the reference's sequential
// std::mt19937_64 streams (rng.hpp:28-53) with a counter-based generator so
// any (request, stream, replica seed) draw is computable independently.
// Constants and KATs: SURVEY App. C; curand_philox4x32_x.h:88-91.
constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;
// The engine's fixed key; streams are separated through the counter
// (c1 = stream id, c2:c3 = whitened replica seed), so the key can be a
// compile-time constant folded into every round.
constexpr uint32_t kKey0 = 0xA4093822u, kKey1 = 0x299F31D0u;

BB_HD uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(kPhiloxM0, c.x), lo0 = kPhiloxM0 * c.x;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c.z), lo1 = kPhiloxM1 * c.z;
#else
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c.x, p1 = (uint64_t)kPhiloxM1 * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
}

BB_HD uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  return philox4x32_10(make_uint4(c0, c1, c2, c3), kKey0, kKey1);
}

// 53-bit integer from two 32-bit words; u = x * 2^-53 is the reference's
// uniform01 resolution (rng.hpp:38).
BB_HD uint64_t bits53(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 21) | (lo >> 11); }

constexpr uint64_t kKeyDomain53 = 1ull << 53;

// detail::splitmix64, rng.hpp:16-21
BB_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// replication_seed, experiment.hpp:90-92
BB_HD uint64_t replication_seed(uint64_t master, uint64_t rep) {
  return splitmix64(master ^ splitmix64(rep + 0x51ED2701A7B4E5D3ull));
}

// Stream ids (Philox counter word c1).
enum : uint32_t { kStreamArrivalService = 0, kStreamError = 1 };

// ------------------------------------------------------ exponential variate
__constant__ const double kAtanhC[10] = {1.0 / 21, 1.0 / 19, 1.0 / 17, 1.0 / 15, 1.0 / 13,
                                         1.0 / 11, 1.0 / 9,  1.0 / 7,  1.0 / 5,  1.0 / 3};

// E = -log1p(-u) with u = x * 2^-53 (the reference's draw, rng.hpp:43).
// 1 - u = (2^53 - x) * 2^-53 is exact, so E = -log(y) + 53 ln2 with the
// integer y = 2^53 - x in [1, 2^53].  Branch-free: exponent split, reduction
// to m in [sqrt(1/2), sqrt(2)), log(m) = 2 atanh(s), s = (m-1)/(m+1) via a
// fp32 reciprocal seed + two Newton steps, and the atanh series to s^21
// (|s| <= 0.1716: truncation < 2^-54).  About 30 instructions and no
// divergence, against CUDA's two-path log1p (~125 issue slots per warp when
// lanes take both paths).  Error <= 3 ulp: a different rounding of the same
// exponential variate, not a different distribution.
template <class Coef>
__device__ __forceinline__ double exp1_from_bits53_c(uint64_t x, const Coef& C) {
  const double y = (double)(kKeyDomain53 - x);  // exact: 1 <= y <= 2^53
  int hi = __double2hiint(y);
  const int lo = __double2loint(y);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000FFFFF) | 0x3FF00000;  // m in [1, 2)
  const int big = hi >= 0x3FF6A09F;      // m >= sqrt(2): halve it
  hi -= big << 20;
  e += big;
  const double m = __hiloint2double(hi, lo);
  const double num = m - 1.0, den = m + 1.0;
  float rf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)den));  // den in [1.7, 2.5]
  double r = (double)rf;
  r = fma(fma(-den, r, 1.0), r, r);
  r = fma(fma(-den, r, 1.0), r, r);
  double s = num * r;
  s = fma(fma(-den, s, num), r, s);
  const double s2 = s * s;
  double p = C[0];
#pragma unroll
  for (int j = 1; j < 10; ++j) p = fma(p, s2, C[j]);
  const double logm = fma(2.0 * s * s2, p, 2.0 * s);
  constexpr double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  const double k = (double)(53 - e);  // E = (53 - e) ln2 - log(m)
  return fma(k, kLn2Hi, fma(k, kLn2Lo, -logm));
}

__device__ __forceinline__ double exp1_from_bits53(uint64_t x) { return exp1_from_bits53_c(x, kAtanhC); }

// Table-driven variant for the inter-arrival gaps (the per-request hot op).
// y = 2^53 - x = 2^k z with z in [0.6875, 1.375) from a bit-pattern split;
// 256 subintervals by the top 8 bits of bits(y) - bits(0.6875), each with
// invc ~ 1/c and logc = -log(invc) (shared-memory table, init_log_table);
// r = fl(z invc - 1) with |r| <= 2^-8 and log1p(r) by its Taylor series to r^7
// (truncation < 2^-59 |r|).  The two subintervals next to 1 use c = 1, so small
// gaps keep full relative accuracy.  ~12 fp64 + 10 integer instructions and
// one shared-memory load, against ~24 fp64 + 3 XU for exp1_from_bits53.  The
// gaps need no monotonicity in x (service keys keep exp1_from_bits53).
constexpr uint32_t kLogTab = 256;
__device__ __forceinline__ void init_log_table(double2* tab) {  // all threads; then sync
  for (uint32_t i = threadIdx.x; i < kLogTab; i += blockDim.x) {
    const double zlo = __longlong_as_double(0x3fe6000000000000ll + ((long long)i << 44));
    const double zhi = __longlong_as_double(0x3fe6000000000000ll + ((long long)(i + 1) << 44));
    double invc = 1.0, logc = 0.0;
    if (zlo != 1.0 && zhi != 1.0) {
      invc = 1.0 / (0.5 * (zlo + zhi));
      logc = -log(invc);
    }
    tab[i] = make_double2(invc, logc);
  }
}
__device__ __forceinline__ double exp1_tab(uint64_t x, const double2* __restrict__ tab) {
  const double y = (double)(kKeyDomain53 - x);  // exact: 1 <= y <= 2^53
  const int hi = __double2hiint(y), lo = __double2loint(y);
  const int th = hi - 0x3fe60000;  // bits(y) - bits(0.6875), high word (low word is 0)
  const uint32_t idx = ((uint32_t)th >> 12) & (kLogTab - 1);
  const int kk = 53 - (th >> 20);  // E = (53 - k) ln2 - log(z)
  const double z = __hiloint2double(hi - (th & 0xfff00000), lo);
  const double2 t = tab[idx];
  const double r = fma(z, t.x, -1.0);
  double p = fma(1.0 / 7.0, r, -1.0 / 6.0);
  p = fma(p, r, 0.2);
  p = fma(p, r, -0.25);
  p = fma(p, r, 1.0 / 3.0);
  p = fma(p, r, -0.5);
  const double lp = fma(r * r, p, r);  // log1p(r)
  const double kd = __hiloint2double(0x43300000, kk) - 0x1.0p52;  // kk in [0, 53]
  constexpr double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  return fma(kd, kLn2Hi, -t.y) + fma(kd, kLn2Lo, -lp);
}

// the atanh coefficients as kernel-parameter (constant bank 0) operands
struct AtanhCoef {
  double c[10];
  __device__ __forceinline__ double operator[](int j) const { return c[j]; }
};
inline AtanhCoef make_atanh_coef() {
  AtanhCoef a;
  for (int j = 0; j < 10; ++j) a.c[j] = 1.0 / (double)(21 - 2 * j);
  return a;
}

// --------------------------------------------------------- service in key space
// Generated mode draws a 53-bit key x per request and the service time is a
// monotone non-decreasing function s(x).  Bins are therefore thresholds on x
// (found by bisection on the same device function), and a batch's service
// max_i s(x_i) == s(max_i x_i): the transcendental runs once per batch.
enum SvcKind : int32_t {
  kSvcUniform = 0,   // lo + (hi-lo)*u                 (rng.hpp:40)
  kSvcExponential,   // -log1p(-u)/rate                (rng.hpp:43)
  kSvcLogNormal,     // exp(mu + sigma*Phi^-1(u'))     u' = (x+1/2)*2^-53
  kSvcTable,         // sorted[floor(u*n)]             (service_dist.hpp:98)
  kSvcLinear,        // b*(lo + (hi-lo)*u) + a         (workload.hpp:167-170)
  kSvcCyclic         // sorted[x], x = rank of lengths[id % n] (simulator.hpp:350)
};

struct SvcParams {
  int32_t kind;
  uint32_t n_table;
  double lo, hi, rate, mu, sigma, lin_a, lin_b;
  const double* table;   // sorted ascending (device)
  uint64_t key_domain;   // 2^53, or n_table for cyclic
};

__device__ __forceinline__ double svc_of_key(const SvcParams& p, uint64_t x) {
  switch (p.kind) {
    case kSvcUniform: {
      const double u = (double)x * 0x1.0p-53;
      return __dadd_rn(p.lo, __dmul_rn(__dsub_rn(p.hi, p.lo), u));
    }
    case kSvcLinear: {
      const double u = (double)x * 0x1.0p-53;
      const double len = __dadd_rn(p.lo, __dmul_rn(__dsub_rn(p.hi, p.lo), u));
      return __dadd_rn(__dmul_rn(p.lin_b, len), p.lin_a);
    }
    case kSvcExponential:
      return exp1_from_bits53(x) / p.rate;
    case kSvcLogNormal: {
      const double u = ((double)x + 0.5) * 0x1.0p-53;
      return exp(p.mu + p.sigma * normcdfinv(u));
    }
    case kSvcTable: {
      const uint64_t idx = __umul64hi(x << 11, (uint64_t)p.n_table);
      return p.table[idx];
    }
    default:  // kSvcCyclic
      return p.table[x];
  }
}

// Same, with the kind fixed at compile time (the fused kernel's closures).
template <int KIND>
__device__ __forceinline__ double svc_of_key_t(const SvcParams& p, uint64_t x) {
  if (KIND == kSvcUniform) {
    const double u = (double)x * 0x1.0p-53;
    return __dadd_rn(p.lo, __dmul_rn(__dsub_rn(p.hi, p.lo), u));
  } else if (KIND == kSvcLinear) {
    const double u = (double)x * 0x1.0p-53;
    const double len = __dadd_rn(p.lo, __dmul_rn(__dsub_rn(p.hi, p.lo), u));
    return __dadd_rn(__dmul_rn(p.lin_b, len), p.lin_a);
  } else if (KIND == kSvcExponential) {
    return exp1_from_bits53(x) / p.rate;
  } else if (KIND == kSvcLogNormal) {
    const double u = ((double)x + 0.5) * 0x1.0p-53;
    return exp(p.mu + p.sigma * normcdfinv(u));
  } else if (KIND == kSvcTable) {
    return p.table[__umul64hi(x << 11, (uint64_t)p.n_table)];
  } else {
    return p.table[x];
  }
}

// ------------------------------------------------------------- errors
// First failing request wins (the reference throws at the first offending
// arrival in event order): packed (index << 8 | code) via atomicMin.
struct DevError {
  unsigned long long packed;  // UINT64_MAX == no error
  double value;               // offending value (for the message)
  unsigned long long aux;     // replica / extra
};

__device__ __forceinline__ void raise_error(DevError* e, uint64_t index, int code, double value,
                                            uint64_t aux = 0) {
  const unsigned long long p = ((unsigned long long)index << 8) | (unsigned)code;
  const unsigned long long old = atomicMin(&e->packed, p);
  if (p < old) {
    e->value = value;  // best effort (racy only among failing threads)
    e->aux = aux;
  }
}

// ------------------------------------------------------ fast 32-bit divider
// n / d for runtime d via one mul-hi (Granlund-Montgomery); exact for all
// 32-bit n.
struct FastDiv {
  uint32_t d, m, s;
  BB_HD FastDiv() : d(1), m(0), s(0) {}
  BB_HD explicit FastDiv(uint32_t dv) : d(dv) {
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < dv) ++l;
    s = l;
    m = (uint32_t)((((1ull << 32) * ((1ull << l) - dv)) / dv) + 1);
  }
  BB_HD uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    const uint64_t t = (uint64_t)__umulhi(n, m) + n;
#else
    const uint64_t t = (((uint64_t)n * m) >> 32) + n;
#endif
    return (uint32_t)(t >> s);
  }
};

}  // namespace bb
