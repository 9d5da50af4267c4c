// tg_synth.cuh — counter-based synthetic batches, identical bits on the host
// and on the GPU (the on-device input pipeline).
//
// The mt19937_64 stream of tg_synth_batch (tg_models.hpp, the reference's
// TestRng, testing_support.hpp:49-58) is one sequential recurrence: a GPU
// cannot start sample s without the 312-word state after s's predecessors.
// This generator keeps its draw definitions — unit() = top 53 bits * 2^-53,
// below(n) = high 64 bits of u64 * n, Box-Muller on two unit() draws, Zipf by
// inverse CDF over the fp64 table p_k ∝ k^-s with a binary search — but takes
// draw j of sample s from Philox4x32-10 keyed by the seed at counter
// (s, j / 2): any sample, on any rank, is generated independently, so a batch
// [s0, s0 + b) is the same bits whichever device or chunking produced it.
//
// Transcendentals (cos/sin of the moons arc, log/cos of Box-Muller) are this
// file's own polynomials written with explicit roundings (tg_add / tg_mul /
// tg_fma map to __dadd_rn / __dmul_rn / __fma_rn on the device, so nvcc never
// contracts them, and to plain IEEE operations plus std::fma on the host), so
// host and device agree bit for bit; division and sqrt are IEEE-correctly
// rounded on both.  Accuracy: < 2 ulp against libm over the used ranges
// (tests/test_abi.py::test_counter_synth_math_accuracy).
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define TG_SHD __host__ __device__ __forceinline__
#define TG_SUNROLL _Pragma("unroll")
#else
#include <cmath>
#define TG_SHD inline
#define TG_SUNROLL
#endif

namespace tgs {

TG_SHD double tg_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
TG_SHD double tg_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
TG_SHD double tg_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
TG_SHD std::uint64_t mulhi64(std::uint64_t a, std::uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return static_cast<std::uint64_t>((static_cast<__uint128_t>(a) * b) >> 64);
#endif
}
TG_SHD std::uint32_t mulhi32(std::uint32_t a, std::uint32_t b) {
  return static_cast<std::uint32_t>((static_cast<std::uint64_t>(a) * b) >> 32);
}
TG_SHD std::uint64_t dbits(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<std::uint64_t>(__double_as_longlong(x));
#else
  std::uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
TG_SHD double bitsd(std::uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of two 32x32->64 products
// and key bumps by the Weyl constants.
struct U64x2 { std::uint64_t a, b; };
TG_SHD U64x2 philox(std::uint64_t seed, std::uint64_t ctr_lo, std::uint64_t ctr_hi) {
  std::uint32_t c0 = static_cast<std::uint32_t>(ctr_lo), c1 = static_cast<std::uint32_t>(ctr_lo >> 32);
  std::uint32_t c2 = static_cast<std::uint32_t>(ctr_hi), c3 = static_cast<std::uint32_t>(ctr_hi >> 32);
  std::uint32_t k0 = static_cast<std::uint32_t>(seed), k1 = static_cast<std::uint32_t>(seed >> 32);
TG_SUNROLL
  for (int r = 0; r < 10; ++r) {
    const std::uint32_t h0 = mulhi32(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
    const std::uint32_t h1 = mulhi32(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
    const std::uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
    c0 = n0; c1 = l1; c2 = n2; c3 = l0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {static_cast<std::uint64_t>(c0) | (static_cast<std::uint64_t>(c1) << 32),
          static_cast<std::uint64_t>(c2) | (static_cast<std::uint64_t>(c3) << 32)};
}

// Draws of one sample: draw j from counter (sample, j / 2), word j % 2.
struct SampleRng {
  std::uint64_t seed, sample, j = 0;
  U64x2 buf{0, 0};
  TG_SHD SampleRng(std::uint64_t seed_, std::uint64_t sample_) : seed(seed_), sample(sample_) {}
  TG_SHD std::uint64_t next() {
    if ((j & 1) == 0) buf = philox(seed, sample, j >> 1);
    const std::uint64_t v = (j & 1) ? buf.b : buf.a;
    ++j;
    return v;
  }
  TG_SHD double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  TG_SHD double uniform(double lo, double hi) { return tg_fma(hi - lo, unit(), lo); }
  TG_SHD std::uint64_t below(std::uint64_t n) { return mulhi64(next(), n); }
};

// sin and cos of x in [0, 8): quadrant k = nearest multiple of pi/2, two-part
// Cody-Waite reduction, Taylor polynomials on |r| <= pi/4 (truncation < 1e-19).
TG_SHD void sincos_small(double x, double* s, double* c) {
  const double kPio2Hi = 1.5707963267948966, kPio2Lo = 6.123233995736766e-17, k2OverPi = 0.6366197723675814;
  const double kd = static_cast<double>(static_cast<int>(tg_fma(x, k2OverPi, 0.5)));
  double r = tg_fma(-kd, kPio2Hi, x);
  r = tg_fma(-kd, kPio2Lo, r);
  const double r2 = tg_mul(r, r);
  // sin r = r + r^3 P(r^2), cos r = 1 + r^2 Q(r^2): Taylor coefficients (-1)^n / (2n+1)!, (-1)^n / (2n)!
  const double S[8] = {-1.6666666666666666e-01, 8.3333333333333332e-03, -1.9841269841269841e-04, 2.7557319223985893e-06,
                       -2.5052108385441720e-08, 1.6059043836821613e-10, -7.6471637318198164e-13, 2.8114572543455206e-15};
  const double C[9] = {-5.0000000000000000e-01, 4.1666666666666664e-02, -1.3888888888888889e-03, 2.4801587301587302e-05,
                       -2.7557319223985888e-07, 2.0876756987868100e-09, -1.1470745597729725e-11, 4.7794773323873853e-14,
                       -1.5619206968586225e-16};
  double p = S[7];
TG_SUNROLL
  for (int i = 6; i >= 0; --i) p = tg_fma(p, r2, S[i]);
  const double sr = tg_fma(tg_mul(r, r2), p, r);
  double q = C[8];
TG_SUNROLL
  for (int i = 7; i >= 0; --i) q = tg_fma(q, r2, C[i]);
  const double cr = tg_fma(r2, q, 1.0);
  switch (static_cast<int>(kd) & 3) {
    case 0: *s = sr; *c = cr; break;
    case 1: *s = cr; *c = -sr; break;
    case 2: *s = -sr; *c = -cr; break;
    default: *s = -cr; *c = sr; break;
  }
}

// Natural log of y in (0, 1] (normal numbers): y = m 2^e with m in
// [sqrt(1/2), sqrt(2)), log m = 2 atanh(f), f = (m - 1) / (m + 1), |f| < 0.172.
TG_SHD double log_pos(double y) {
  const std::uint64_t u = dbits(y);
  int e = static_cast<int>((u >> 52) & 0x7ff) - 1023;
  double m = bitsd((u & 0x000fffffffffffffull) | 0x3ff0000000000000ull);   // [1, 2)
  if (m > 1.4142135623730951) { m = tg_mul(m, 0.5); e += 1; }
  const double f = (m - 1.0) / (m + 1.0);
  const double f2 = tg_mul(f, f);
  // atanh f / f - 1 = sum_{n>=1} f^(2n) / (2n + 1), |f|^2 < 0.0295: 13 terms
  double p = 1.0 / 27.0;
TG_SUNROLL
  for (int n = 12; n >= 1; --n) p = tg_fma(p, f2, 1.0 / (2 * n + 1));
  const double lm = tg_fma(tg_mul(2.0 * f, f2), p, 2.0 * f);
  const double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  const double ed = static_cast<double>(e);
  return tg_add(tg_fma(ed, kLn2Hi, 0.0), tg_fma(ed, kLn2Lo, lm));
}

TG_SHD double normal(SampleRng& r, double mean, double sd) {
  const double u1 = r.unit(), u2 = r.unit();
  const double rad = sqrt(tg_mul(-2.0, log_pos(1.0 - u1)));
  double s, c;
  sincos_small(tg_mul(6.283185307179586, u2), &s, &c);
  return tg_fma(tg_mul(sd, rad), c, mean);
}

TG_SHD std::int32_t zipf_draw(SampleRng& r, const double* cdf, std::uint32_t V) {
  const double u = r.unit();
  std::uint32_t lo = 0, hi = V - 1;
  while (lo < hi) {
    const std::uint32_t mid = (lo + hi) / 2;
    if (u < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return static_cast<std::int32_t>(lo);
}

// Models of tg_models.hpp (same numbering) and their per-sample columns.
enum : int { kFig1 = 1, kListing1 = 2, kMoons = 3, kCharMlp = 4, kGpt = 5, kWideMlp = 6 };

struct SynthArgs {
  int model;
  int f64;                        // inputs are double (else float)
  std::uint32_t n_inputs, n_index; // columns
  std::uint32_t n_classes;         // wide MLP labels
  std::uint32_t V;                 // Zipf table size
  std::uint64_t seed, first;       // sample ids [first, first + batch)
  std::size_t batch;
  void* x;                         // [n_inputs][batch]
  std::int32_t* idx;               // [n_index][batch]
  const double* cdf;               // Zipf CDF (V entries)
};

template <class Scalar>
TG_SHD void put(void* x, std::size_t at, double v) { static_cast<Scalar*>(x)[at] = static_cast<Scalar>(v); }

// Sample i of the batch (global id first + i): the same draw order as
// tgm::synth (tg_models.hpp:116-160) with counter-based draws.
template <class Scalar>
TG_SHD void synth_sample(const SynthArgs& a, std::size_t i) {
  SampleRng r(a.seed, a.first + i);
  const std::size_t b = a.batch;
  switch (a.model) {
    case kFig1: case kListing1:
      put<Scalar>(a.x, i, r.uniform(-4.0, 4.0));
      put<Scalar>(a.x, b + i, r.uniform(-4.0, 4.0));
      break;
    case kMoons: {
      const bool second = r.below(2) == 1;
      const double th = r.uniform(0.0, 3.141592653589793);
      double s, c;
      sincos_small(th, &s, &c);
      double x0 = c, x1 = s;
      if (second) { x0 = 1.0 - x0; x1 = 0.5 - x1; }
      x0 = tg_add(x0, normal(r, 0.0, 0.1));
      x1 = tg_add(x1, normal(r, 0.0, 0.1));
      put<Scalar>(a.x, i, x0);
      put<Scalar>(a.x, b + i, x1);
      put<Scalar>(a.x, 2 * b + i, second ? 1.0 : -1.0);
      break;
    }
    case kCharMlp: case kGpt:
      for (std::uint32_t c = 0; c < a.n_index; ++c) a.idx[c * b + i] = zipf_draw(r, a.cdf, a.V);
      break;
    case kWideMlp:
      for (std::uint32_t c = 0; c < a.n_inputs; ++c) put<Scalar>(a.x, c * b + i, r.unit());
      a.idx[i] = static_cast<std::int32_t>(r.below(a.n_classes));
      break;
    default: break;
  }
}

}  // namespace tgs
