// tg_math.cuh — branch-free fp64 transcendental used on the tape hot path.
//
// This file is compiled by nvcc into the interpreter kernels AND embedded
// verbatim (Makefile -> build/tg_math.inc) into every NVRTC-specialised
// kernel, so both tiers run the same instructions.  No preprocessor lines
// below this comment block.
//
// tg_tanh(x): the libdevice tanh(double) costs ~80 SASS instructions per call
// with sample-dependent branches (warp divergence); tanh dominates cfg2's
// instruction count.  Here, branch-free:
//   tanh|x| = -u / (2 + u),  u = expm1(-2|x|)   (no cancellation for small x)
//   expm1(t) = 2^k * p(r) + (2^k - 1),  t = k ln2 + r,  |r| <= ln2/2,
//   p(r) = r + r^2 Q(r), Q the degree-11 Taylor tail (trunc. error < 2e-17),
//   exact for k = 0 (fma(1, p, 0) = p); then the quotient by d = 2 + u in
//   (1, 2], refined by Newton steps and one residual correction.
// Two variants of the reduction and the reciprocal seed:
//   tg_tanh       rint / float reciprocal seed (XU unit) + 2 Newton steps;
//                 fewest FP64 instructions (one-thread-per-sample kernels);
//   tg_tanh_fp64  k by the 1.5 * 2^52 shift inside one FMA (k = low word),
//                 2^k from its exponent bits, linear seed 24/17 - 8/17 d
//                 (error <= 1/17) + 4 Newton steps: FP64 pipe only, for the
//                 DMMA kernel, whose XU queue (1/4 rate) throttled issue.
// Accuracy vs correctly rounded tanh: a few ulp (tested against numpy).
// The polynomial coefficients sit in the constant bank: a DFMA takes a
// c[bank][offset] / uniform-register operand, whereas 64-bit immediates cost
// two uniform-register moves per use (measured: 17% of the DMMA kernel's issue).
static __constant__ double tg_tanh_q[12] = {
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
    1.0 / 5040.0,       1.0 / 720.0,       1.0 / 120.0,      1.0 / 24.0,      1.0 / 6.0,      0.5};
static __constant__ double tg_tanh_k[6] = {1.4426950408889634, -6.93147180369123816490e-01,
                                           -1.90821492927058770002e-10, 6755399441055744.0,
                                           -0.47058823529411764706, 1.41176470588235294118};
__device__ __forceinline__ double tg_expm1_core(double r) {
  double q = tg_tanh_q[0];   // 1/13!, 1/12!, ..., 1/2
#pragma unroll
  for (int i = 1; i < 12; ++i) q = fma(q, r, tg_tanh_q[i]);
  return fma(r * r, q, r);
}
__device__ __forceinline__ double tg_tanh(double x) {
  const double a = fmin(fabs(x), 20.0);  // tanh(20) = 1 - 8.5e-18 rounds to 1
  const double t = -2.0 * a;
  const double kf = rint(t * tg_tanh_k[0]);
  double r = fma(kf, tg_tanh_k[1], t);
  r = fma(kf, tg_tanh_k[2], r);
  const double em = tg_expm1_core(r);
  const double sc = __longlong_as_double(static_cast<long long>(static_cast<int>(kf) + 1023) << 52);
  const double u = fma(sc, em, sc - 1.0);
  const double d = 2.0 + u;
  const double n = -u;
  double rc = static_cast<double>(__frcp_rn(static_cast<float>(d)));
  rc = fma(rc, fma(-d, rc, 1.0), rc);
  rc = fma(rc, fma(-d, rc, 1.0), rc);
  const double q0 = n * rc;
  const double res = fma(-d, q0, n);
  return copysign(fma(res, rc, q0), x);
}
__device__ __forceinline__ double tg_tanh_fp64(double x) {
  const double a = fmin(fabs(x), 20.0);
  const double t = -2.0 * a;
  const double sh = fma(t, tg_tanh_k[0], tg_tanh_k[3]);   // 1.5 * 2^52 + round(t / ln2)
  const double kf = sh - tg_tanh_k[3];
  const int k = __double2loint(sh);
  double r = fma(kf, tg_tanh_k[1], t);
  r = fma(kf, tg_tanh_k[2], r);
  const double em = tg_expm1_core(r);
  const double sc = __hiloint2double((k + 1023) << 20, 0);
  const double u = fma(sc, em, sc - 1.0);
  const double d = 2.0 + u;
  const double n = -u;
  double rc = fma(tg_tanh_k[4], d, tg_tanh_k[5]);
#pragma unroll
  for (int i = 0; i < 4; ++i) rc = fma(rc, fma(-d, rc, 1.0), rc);
  const double q0 = n * rc;
  const double res = fma(-d, q0, n);
  return copysign(fma(res, rc, q0), x);
}
