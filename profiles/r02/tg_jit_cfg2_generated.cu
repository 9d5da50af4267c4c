typedef double T;
// tg_math.cuh — branch-free fp64 transcendental used on the tape hot path.
//
// This file is compiled by nvcc into the interpreter kernels AND embedded
// verbatim (Makefile -> build/tg_math.inc) into every NVRTC-specialised
// kernel, so both tiers run the same instructions.  No preprocessor lines
// below this comment block.
//
// tg_tanh(x): the libdevice tanh(double) costs ~80 SASS instructions per call
// with sample-dependent branches (warp divergence); tanh dominates cfg2's
// instruction count.  Here, branch-free, ~33 instructions:
//   tanh|x| = -u / (2 + u),  u = expm1(-2|x|)   (no cancellation for small x)
//   expm1(t) = 2^k * p(r) + (2^k - 1),  t = k ln2 + r,  |r| <= ln2/2,
//   p(r) = r + r^2 Q(r), Q the degree-11 Taylor tail (trunc. error < 2e-17),
//   exact for k = 0 (fma(1, p, 0) = p); quotient by a float reciprocal seed,
//   two Newton steps and one residual correction.
// Accuracy vs correctly rounded tanh: a few ulp (tested against numpy).
// The polynomial coefficients sit in the constant bank: a DFMA takes a
// c[bank][offset] operand directly, whereas 64-bit immediates cost two
// uniform-register moves per use (measured: 17% of the DMMA kernel's issue).
static __constant__ double tg_tanh_q[12] = {
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
    1.0 / 5040.0,       1.0 / 720.0,       1.0 / 120.0,      1.0 / 24.0,      1.0 / 6.0,      0.5};
static __constant__ double tg_tanh_k[3] = {1.4426950408889634, -6.93147180369123816490e-01,
                                           -1.90821492927058770002e-10};
__device__ __forceinline__ double tg_tanh(double x) {
  const double a = fmin(fabs(x), 20.0);  // tanh(20) = 1 - 8.5e-18 rounds to 1
  const double t = -2.0 * a;
  const double kf = rint(t * tg_tanh_k[0]);
  double r = fma(kf, tg_tanh_k[1], t);
  r = fma(kf, tg_tanh_k[2], r);
  double q = tg_tanh_q[0];   // 1/13!, 1/12!, ..., 1/2
#pragma unroll
  for (int i = 1; i < 12; ++i) q = fma(q, r, tg_tanh_q[i]);
  const double em = fma(r * r, q, r);
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

struct TermC { unsigned a; unsigned f; int row; unsigned kind; double coef; };
__device__ __forceinline__ void tg_err(unsigned long long* key, unsigned long long s, unsigned node) {
  atomicMin(key, (s << 32) | node);
}
__device__ __forceinline__ int tg_ix(const int* __restrict__ idx, unsigned long long at, unsigned n) {
  const int r = idx[at];
  return (unsigned)r < n ? r : 0;
}
// kernel argument block; host mirror: tgj::JitArgs<T> (tg_jit.hpp), same field order
struct JitArgs {
  const T* in; const int* idx; unsigned long long batch;
  T* loss; T* igrad; T* partial; unsigned grid_rows; unsigned n_groups;
  unsigned long long* err_key; double* err_val; unsigned* err_op;
  const T* UVg; const unsigned* cand; const unsigned* toff; const TermC* terms;
  const T* params; const T* consts; T* UVw;
  unsigned* tickets; T* partial2;
  T* grad_sum; T* gd_params; T gamma; T gd_batch;
};
__constant__ unsigned cDU[338] = {0u, 1u, 2u, 3u, 4u, 5u, 6u, 7u, 8u, 9u, 10u, 11u, 12u, 13u, 14u, 15u, 16u, 17u, 18u, 19u, 20u, 21u, 22u, 23u, 24u, 25u, 26u, 27u, 28u, 29u, 30u, 31u, 32u, 33u, 34u, 35u, 36u, 37u, 38u, 39u, 40u, 41u, 42u, 43u, 44u, 45u, 46u, 47u, 48u, 49u, 50u, 51u, 52u, 53u, 54u, 55u, 56u, 57u, 58u, 59u, 60u, 61u, 62u, 63u, 64u, 65u, 66u, 67u, 68u, 69u, 70u, 71u, 72u, 73u, 74u, 75u, 76u, 77u, 78u, 79u, 80u, 81u, 82u, 83u, 84u, 85u, 86u, 87u, 88u, 89u, 90u, 91u, 92u, 93u, 94u, 95u, 96u, 97u, 98u, 99u, 100u, 101u, 102u, 103u, 104u, 105u, 106u, 107u, 108u, 109u, 110u, 111u, 112u, 113u, 114u, 115u, 116u, 117u, 118u, 119u, 120u, 121u, 122u, 123u, 124u, 125u, 126u, 127u, 128u, 129u, 130u, 131u, 132u, 133u, 134u, 135u, 136u, 137u, 138u, 139u, 140u, 141u, 142u, 143u, 144u, 145u, 146u, 147u, 148u, 149u, 150u, 151u, 152u, 153u, 154u, 155u, 156u, 157u, 158u, 159u, 160u, 161u, 162u, 163u, 164u, 165u, 166u, 167u, 168u, 169u, 170u, 171u, 172u, 173u, 174u, 175u, 176u, 177u, 178u, 179u, 180u, 181u, 182u, 183u, 184u, 185u, 186u, 187u, 188u, 189u, 190u, 191u, 192u, 193u, 194u, 195u, 196u, 197u, 198u, 199u, 200u, 201u, 202u, 203u, 204u, 205u, 206u, 207u, 208u, 209u, 210u, 211u, 212u, 213u, 214u, 215u, 216u, 217u, 218u, 219u, 220u, 221u, 222u, 223u, 224u, 225u, 226u, 227u, 228u, 229u, 230u, 231u, 232u, 233u, 234u, 235u, 236u, 237u, 238u, 239u, 240u, 241u, 242u, 243u, 244u, 245u, 246u, 247u, 248u, 249u, 250u, 251u, 252u, 253u, 254u, 255u, 256u, 257u, 258u, 259u, 260u, 261u, 262u, 263u, 264u, 265u, 266u, 267u, 268u, 269u, 270u, 271u, 272u, 273u, 274u, 275u, 276u, 277u, 278u, 279u, 280u, 281u, 282u, 283u, 284u, 285u, 286u, 287u, 288u, 289u, 290u, 291u, 292u, 293u, 294u, 295u, 296u, 297u, 298u, 299u, 300u, 301u, 302u, 303u, 304u, 305u, 306u, 307u, 308u, 309u, 310u, 311u, 312u, 313u, 314u, 315u, 316u, 317u, 318u, 319u, 320u, 321u, 322u, 323u, 324u, 325u, 326u, 327u, 328u, 329u, 330u, 331u, 332u, 333u, 334u, 335u, 336u, 338u};
__constant__ unsigned cUO[674] = {0u, 1u, 2u, 3u, 4u, 5u, 6u, 7u, 8u, 9u, 10u, 11u, 12u, 13u, 14u, 15u, 16u, 17u, 18u, 19u, 20u, 21u, 22u, 23u, 24u, 25u, 26u, 27u, 28u, 29u, 30u, 31u, 32u, 33u, 34u, 35u, 36u, 37u, 38u, 39u, 40u, 41u, 42u, 43u, 44u, 45u, 46u, 47u, 48u, 49u, 50u, 51u, 52u, 53u, 54u, 55u, 56u, 57u, 58u, 59u, 60u, 61u, 62u, 63u, 64u, 65u, 66u, 67u, 68u, 69u, 70u, 71u, 72u, 73u, 74u, 75u, 76u, 77u, 78u, 79u, 80u, 81u, 82u, 83u, 84u, 85u, 86u, 87u, 88u, 89u, 90u, 91u, 92u, 93u, 94u, 95u, 96u, 97u, 98u, 99u, 100u, 101u, 102u, 103u, 104u, 105u, 106u, 107u, 108u, 109u, 110u, 111u, 112u, 113u, 114u, 115u, 116u, 117u, 118u, 119u, 120u, 121u, 122u, 123u, 124u, 125u, 126u, 127u, 128u, 129u, 130u, 131u, 132u, 133u, 134u, 135u, 136u, 137u, 138u, 139u, 140u, 141u, 142u, 143u, 144u, 145u, 146u, 147u, 148u, 149u, 150u, 151u, 152u, 153u, 154u, 155u, 156u, 157u, 158u, 159u, 160u, 161u, 162u, 163u, 164u, 165u, 166u, 167u, 168u, 169u, 170u, 171u, 172u, 173u, 174u, 175u, 176u, 177u, 178u, 179u, 180u, 181u, 182u, 183u, 184u, 185u, 186u, 187u, 188u, 189u, 190u, 191u, 192u, 193u, 194u, 195u, 196u, 197u, 198u, 199u, 200u, 201u, 202u, 203u, 204u, 205u, 206u, 207u, 208u, 209u, 210u, 211u, 212u, 213u, 214u, 215u, 216u, 217u, 218u, 219u, 220u, 221u, 222u, 223u, 224u, 225u, 226u, 227u, 228u, 229u, 230u, 231u, 232u, 233u, 234u, 235u, 236u, 237u, 238u, 239u, 240u, 241u, 242u, 243u, 244u, 245u, 246u, 247u, 248u, 249u, 250u, 251u, 252u, 253u, 254u, 255u, 256u, 257u, 258u, 259u, 260u, 261u, 262u, 263u, 264u, 265u, 266u, 267u, 268u, 269u, 270u, 271u, 272u, 273u, 274u, 275u, 276u, 277u, 278u, 279u, 280u, 281u, 282u, 283u, 284u, 285u, 286u, 287u, 288u, 289u, 290u, 291u, 292u, 293u, 294u, 295u, 296u, 297u, 298u, 299u, 300u, 301u, 302u, 303u, 304u, 305u, 306u, 307u, 308u, 309u, 310u, 311u, 312u, 313u, 314u, 315u, 316u, 317u, 318u, 319u, 320u, 321u, 322u, 323u, 324u, 325u, 326u, 327u, 328u, 329u, 330u, 331u, 332u, 333u, 334u, 335u, 336u, 0u, 1u, 2u, 3u, 4u, 5u, 6u, 7u, 8u, 9u, 10u, 11u, 12u, 13u, 14u, 15u, 16u, 17u, 18u, 19u, 20u, 21u, 22u, 23u, 24u, 25u, 26u, 27u, 28u, 29u, 30u, 31u, 32u, 33u, 34u, 35u, 36u, 37u, 38u, 39u, 40u, 41u, 42u, 43u, 44u, 45u, 46u, 47u, 48u, 49u, 50u, 51u, 52u, 53u, 54u, 55u, 56u, 57u, 58u, 59u, 60u, 61u, 62u, 63u, 64u, 65u, 66u, 67u, 68u, 69u, 70u, 71u, 72u, 73u, 74u, 75u, 76u, 77u, 78u, 79u, 80u, 81u, 82u, 83u, 84u, 85u, 86u, 87u, 88u, 89u, 90u, 91u, 92u, 93u, 94u, 95u, 96u, 97u, 98u, 99u, 100u, 101u, 102u, 103u, 104u, 105u, 106u, 107u, 108u, 109u, 110u, 111u, 112u, 113u, 114u, 115u, 116u, 117u, 118u, 119u, 120u, 121u, 122u, 123u, 124u, 125u, 126u, 127u, 128u, 129u, 130u, 131u, 132u, 133u, 134u, 135u, 136u, 137u, 138u, 139u, 140u, 141u, 142u, 143u, 144u, 145u, 146u, 147u, 148u, 149u, 150u, 151u, 152u, 153u, 154u, 155u, 156u, 157u, 158u, 159u, 160u, 161u, 162u, 163u, 164u, 165u, 166u, 167u, 168u, 169u, 170u, 171u, 172u, 173u, 174u, 175u, 176u, 177u, 178u, 179u, 180u, 181u, 182u, 183u, 184u, 185u, 186u, 187u, 188u, 189u, 190u, 191u, 192u, 193u, 194u, 195u, 196u, 197u, 198u, 199u, 200u, 201u, 202u, 203u, 204u, 205u, 206u, 207u, 208u, 209u, 210u, 211u, 212u, 213u, 214u, 215u, 216u, 217u, 218u, 219u, 220u, 221u, 222u, 223u, 224u, 225u, 226u, 227u, 228u, 229u, 230u, 231u, 232u, 233u, 234u, 235u, 236u, 237u, 238u, 239u, 240u, 241u, 242u, 243u, 244u, 245u, 246u, 247u, 248u, 249u, 250u, 251u, 252u, 253u, 254u, 255u, 256u, 257u, 258u, 259u, 260u, 261u, 262u, 263u, 264u, 265u, 266u, 267u, 268u, 269u, 270u, 271u, 272u, 273u, 274u, 275u, 276u, 277u, 278u, 279u, 280u, 281u, 282u, 283u, 284u, 285u, 286u, 287u, 288u, 289u, 290u, 291u, 292u, 293u, 294u, 295u, 296u, 297u, 298u, 299u, 300u, 301u, 302u, 303u, 304u, 305u, 306u, 307u, 308u, 309u, 310u, 311u, 312u, 313u, 314u, 315u, 316u, 317u, 318u, 319u, 320u, 321u, 322u, 323u, 324u, 325u, 326u, 327u, 328u, 329u, 330u, 331u, 332u, 333u, 334u, 335u, 336u};
__device__ __forceinline__ T tg_block_sum(T v, T* red) {  // fixed order; result in thread 0
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  __syncthreads();
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T t = (T)0;
  if (threadIdx.x == 0) for (unsigned i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
  return t;
}
__device__ __forceinline__ void tg_dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__constant__ unsigned cBD0[16] = {32u, 33u, 34u, 35u, 36u, 37u, 38u, 39u, 40u, 41u, 42u, 43u, 44u, 45u, 46u, 47u};
__constant__ unsigned cBD1[16] = {304u, 305u, 306u, 307u, 308u, 309u, 310u, 311u, 312u, 313u, 314u, 315u, 316u, 317u, 318u, 319u};
__constant__ unsigned cBD2[1] = {336u};
extern "C" __global__ void __launch_bounds__(128) tg_jit_tape(const JitArgs A) {
  const T* __restrict__ in = A.in; const int* __restrict__ idx = A.idx; const unsigned long long batch = A.batch;
  T* __restrict__ loss = A.loss; T* __restrict__ igrad = A.igrad; T* __restrict__ partial = A.partial;
  const unsigned grid_rows = A.grid_rows; unsigned long long* err_key = A.err_key;
  const T* __restrict__ UVg = A.UVg; const unsigned* __restrict__ cand = A.cand;
  const unsigned* __restrict__ toff = A.toff; const TermC* __restrict__ terms = A.terms;
  (void)in; (void)idx; (void)loss; (void)igrad; (void)UVg; (void)cand; (void)toff; (void)terms; (void)err_key;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // params of the previous step
  __shared__ T sU[340];
  __shared__ T sRed_[32];
  for (unsigned i = threadIdx.x; i < 337u; i += 128u) sU[i] = A.params[i];
  for (unsigned i = threadIdx.x; i < 1u; i += 128u) sU[339u + i] = A.consts[i];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const unsigned g = lane >> 2, c = lane & 3u;
  T* gzb = sm + 1000u + warp * 448u;
  T* xb = gzb + 160u;
  T* sRed = sm + 2792u;
  (void)toff; (void)terms; (void)cand; (void)idx; (void)in; (void)err_key; (void)gzb; (void)xb;
  for (unsigned e = tid; e < 64u; e += 128u) {
    const unsigned t = e / 64u, u = (e >> 5) % 2u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), cc = L & 3u;
    const unsigned k = 4u * t + cc;
    T w = (T)0;
    if (n < 16u) { if (k < 2u) w = A.params[0u + n * 2u + k]; else if (k == 2u) w = A.params[32u + n]; }
    sm[0u + e] = w;
  }
  for (unsigned e = tid; e < 128u; e += 128u) {
    const unsigned t = e / 32u, u = (e >> 5) % 1u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), k = 8u * (t >> 1) + 2u * (L & 3u) + (t & 1u);
    sm[64u + e] = (k < 16u && n < 2u) ? A.params[0u + k * 2u + n] : (T)0;
  }
  for (unsigned e = tid; e < 256u; e += 128u) {
    const unsigned t = e / 64u, u = (e >> 5) % 2u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), cc = L & 3u;
    const unsigned k = 8u * (t >> 1) + 2u * cc + (t & 1u);
    sm[208u + e] = (n < 16u && k < 16u) ? A.params[48u + n * 16u + k] : (T)0;
  }
  for (unsigned e = tid; e < 256u; e += 128u) {
    const unsigned t = e / 64u, u = (e >> 5) % 2u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), k = 8u * (t >> 1) + 2u * (L & 3u) + (t & 1u);
    sm[464u + e] = (k < 16u && n < 16u) ? A.params[48u + k * 16u + n] : (T)0;
  }
  for (unsigned e = tid; e < 16u; e += 128u) sm[720u + e] = e < 16u ? A.params[304u + e] : (T)0;
  for (unsigned e = tid; e < 128u; e += 128u) {
    const unsigned t = e / 32u, u = (e >> 5) % 1u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), cc = L & 3u;
    const unsigned k = 8u * (t >> 1) + 2u * cc + (t & 1u);
    sm[736u + e] = (n < 1u && k < 16u) ? A.params[320u + n * 16u + k] : (T)0;
  }
  for (unsigned e = tid; e < 128u; e += 128u) {
    const unsigned t = e / 64u, u = (e >> 5) % 2u, L = e & 31u;
    const unsigned n = 8u * u + (L >> 2), k = 8u * (t >> 1) + 2u * (L & 3u) + (t & 1u);
    sm[864u + e] = (k < 1u && n < 16u) ? A.params[320u + k * 16u + n] : (T)0;
  }
  for (unsigned e = tid; e < 8u; e += 128u) sm[992u + e] = e < 1u ? A.params[336u + e] : (T)0;
  for (unsigned e = tid; e < 1352u; e += 128u) sRed[e] = (T)0;
  __syncthreads();
  __syncthreads();
  {
    { T part = (T)0;
      for (unsigned j = threadIdx.x; j < 337u; j += 128u) { const T v = sU[cUO[0u + j]]; part += v * v; }
      part = tg_block_sum(part, sRed_);
      if (threadIdx.x == 0) { T r = part; sU[337] = r; }
      __syncthreads(); }
    if (threadIdx.x == 0) {
      const T v338 = sU[337] * (T)0.0001;
      sU[338] = v338;
    }
    __syncthreads();
    if (blockIdx.x == 0)  // UV for the epilogue and for diagnostics
      for (unsigned i = threadIdx.x; i < 340u; i += 128u) A.UVw[i] = sU[i];
  }
  T aw0_0_0_0 = (T)0, aw0_0_0_1 = (T)0;
  T aw0_1_0_0 = (T)0, aw0_1_0_1 = (T)0;
  T aw1_0_0_0 = (T)0, aw1_0_0_1 = (T)0;
  T aw1_0_1_0 = (T)0, aw1_0_1_1 = (T)0;
  T aw1_0_2_0 = (T)0, aw1_0_2_1 = (T)0;
  T aw1_1_0_0 = (T)0, aw1_1_0_1 = (T)0;
  T aw1_1_1_0 = (T)0, aw1_1_1_1 = (T)0;
  T aw1_1_2_0 = (T)0, aw1_1_2_1 = (T)0;
  T aw2_0_0_0 = (T)0, aw2_0_0_1 = (T)0;
  T aw2_0_1_0 = (T)0, aw2_0_1_1 = (T)0;
  T aw2_0_2_0 = (T)0, aw2_0_2_1 = (T)0;
  T as0 = (T)0;
  const unsigned long long TW = (unsigned long long)gridDim.x * 4u;
  unsigned long long base = ((unsigned long long)blockIdx.x * 4u + warp) * 8u;
  const unsigned long long s0 = base + g < batch ? base + g : batch - 1;
  T pf0 = in[0ull * batch + s0];
  T pf1 = in[1ull * batch + s0];
  T pf2 = in[2ull * batch + s0];
  for (; base < batch; base += TW * 8u) {
    const unsigned long long sa = base + g;
    const bool active = sa < batch;
    const unsigned long long s = active ? sa : batch - 1;
    const T in0 = pf0;
    const T in1 = pf1;
    const T in2 = pf2;
    {
      const unsigned long long sn = base + TW * 8u + g < batch ? base + TW * 8u + g : batch - 1;
      pf0 = in[0ull * batch + sn];
      pf1 = in[1ull * batch + sn];
      pf2 = in[2ull * batch + sn];
    }
    {
      const T v0 = in0;
      const T v1 = in1;
      const T v2 = in2;
      // dense 0: 16 x 2 on DMMA
      T dz0_0_0 = (T)0;
      T dz0_0_1 = (T)0;
      T dz0_1_0 = (T)0;
      T dz0_1_1 = (T)0;
      T da0 = (T)0; da0 = c == 2u ? (T)1 : da0; da0 = c == 1u ? v1 : da0; da0 = c == 0u ? v0 : da0;
      tg_dmma(dz0_0_0, dz0_0_1, da0, sm[0u + lane]);
      tg_dmma(dz0_1_0, dz0_1_1, da0, sm[32u + lane]);
      const T dh0_0_0 = tg_tanh(dz0_0_0);
      const T dh0_0_1 = tg_tanh(dz0_0_1);
      const T dh0_1_0 = tg_tanh(dz0_1_0);
      const T dh0_1_1 = tg_tanh(dz0_1_1);
      // dense 1: 16 x 16 on DMMA
      T dz1_0_0 = sm[720u + 2u * c];
      T dz1_0_1 = sm[721u + 2u * c];
      T dz1_1_0 = sm[728u + 2u * c];
      T dz1_1_1 = sm[729u + 2u * c];
      tg_dmma(dz1_0_0, dz1_0_1, dh0_0_0, sm[208u + lane]);
      tg_dmma(dz1_1_0, dz1_1_1, dh0_0_0, sm[240u + lane]);
      tg_dmma(dz1_0_0, dz1_0_1, dh0_0_1, sm[272u + lane]);
      tg_dmma(dz1_1_0, dz1_1_1, dh0_0_1, sm[304u + lane]);
      tg_dmma(dz1_0_0, dz1_0_1, dh0_1_0, sm[336u + lane]);
      tg_dmma(dz1_1_0, dz1_1_1, dh0_1_0, sm[368u + lane]);
      tg_dmma(dz1_0_0, dz1_0_1, dh0_1_1, sm[400u + lane]);
      tg_dmma(dz1_1_0, dz1_1_1, dh0_1_1, sm[432u + lane]);
      const T dh1_0_0 = tg_tanh(dz1_0_0);
      const T dh1_0_1 = tg_tanh(dz1_0_1);
      const T dh1_1_0 = tg_tanh(dz1_1_0);
      const T dh1_1_1 = tg_tanh(dz1_1_1);
      // dense 2: 1 x 16 on DMMA
      T dz2_0_0 = sm[992u + 2u * c];
      T dz2_0_1 = sm[993u + 2u * c];
      tg_dmma(dz2_0_0, dz2_0_1, dh1_0_0, sm[736u + lane]);
      tg_dmma(dz2_0_0, dz2_0_1, dh1_0_1, sm[768u + lane]);
      tg_dmma(dz2_0_0, dz2_0_1, dh1_1_0, sm[800u + lane]);
      tg_dmma(dz2_0_0, dz2_0_1, dh1_1_1, sm[832u + lane]);
      const T bv67 = __shfl_sync(0xffffffffu, dz2_0_0, (lane & ~3u) | 0u);
      const T v68 = v2 * bv67;
      const T v69 = sU[339] - v68;
      const T v70 = v69 > (T)0 ? v69 : (T)0;
      const T v71 = v70 + sU[338];
      if (loss && active && c == 0u) loss[s] = v71;
      T gh0_0_0 = (T)0, gh0_0_1 = (T)0;
      T gh0_1_0 = (T)0, gh0_1_1 = (T)0;
      T gh1_0_0 = (T)0, gh1_0_1 = (T)0;
      T gh1_1_0 = (T)0, gh1_1_1 = (T)0;
      T gh2_0_0 = (T)0, gh2_0_1 = (T)0;
      T g71 = (T)1;
      T g70 = g71;
      T g69 = (v69 > (T)0 ? g70 : (T)0);
      T g68 = -g69;
      T g2 = g68 * bv67;
      if (c == 0u) gh2_0_0 += g68 * v2;
      // dense 2 reverse
      T gz2_0_0 = gh2_0_0;
      if (0u + 2u * c >= 1u) gz2_0_0 = (T)0;
      T gz2_0_1 = gh2_0_1;
      if (1u + 2u * c >= 1u) gz2_0_1 = (T)0;
      tg_dmma(gh1_0_0, gh1_0_1, gz2_0_0, sm[864u + lane]);
      tg_dmma(gh1_1_0, gh1_1_1, gz2_0_0, sm[896u + lane]);
      tg_dmma(gh1_0_0, gh1_0_1, gz2_0_1, sm[928u + lane]);
      tg_dmma(gh1_1_0, gh1_1_1, gz2_0_1, sm[960u + lane]);
      gzb[g * 20u + 0u + 2u * c] = active ? gz2_0_0 : (T)0;
      gzb[g * 20u + 1u + 2u * c] = active ? gz2_0_1 : (T)0;
      xb[g * 36u + 0u + 2u * c] = active ? dh1_0_0 : (T)0;
      xb[g * 36u + 1u + 2u * c] = active ? dh1_0_1 : (T)0;
      xb[g * 36u + 8u + 2u * c] = active ? dh1_1_0 : (T)0;
      xb[g * 36u + 9u + 2u * c] = active ? dh1_1_1 : (T)0;
      if (c == 0u) xb[g * 36u + 16u] = active ? (T)1 : (T)0;
      __syncwarp();
      const T qa2_0_0 = gzb[(0u + c) * 20u + 0u + g];
      const T qb2_0_0 = xb[(0u + c) * 36u + 0u + g];
      const T qb2_0_1 = xb[(0u + c) * 36u + 8u + g];
      const T qb2_0_2 = xb[(0u + c) * 36u + 16u + g];
      tg_dmma(aw2_0_0_0, aw2_0_0_1, qa2_0_0, qb2_0_0);
      tg_dmma(aw2_0_1_0, aw2_0_1_1, qa2_0_0, qb2_0_1);
      tg_dmma(aw2_0_2_0, aw2_0_2_1, qa2_0_0, qb2_0_2);
      const T qa2_1_0 = gzb[(4u + c) * 20u + 0u + g];
      const T qb2_1_0 = xb[(4u + c) * 36u + 0u + g];
      const T qb2_1_1 = xb[(4u + c) * 36u + 8u + g];
      const T qb2_1_2 = xb[(4u + c) * 36u + 16u + g];
      tg_dmma(aw2_0_0_0, aw2_0_0_1, qa2_1_0, qb2_1_0);
      tg_dmma(aw2_0_1_0, aw2_0_1_1, qa2_1_0, qb2_1_1);
      tg_dmma(aw2_0_2_0, aw2_0_2_1, qa2_1_0, qb2_1_2);
      __syncwarp();
      // dense 1 reverse
      T gz1_0_0 = gh1_0_0 * ((T)1 - dh1_0_0 * dh1_0_0);
      T gz1_0_1 = gh1_0_1 * ((T)1 - dh1_0_1 * dh1_0_1);
      T gz1_1_0 = gh1_1_0 * ((T)1 - dh1_1_0 * dh1_1_0);
      T gz1_1_1 = gh1_1_1 * ((T)1 - dh1_1_1 * dh1_1_1);
      tg_dmma(gh0_0_0, gh0_0_1, gz1_0_0, sm[464u + lane]);
      tg_dmma(gh0_1_0, gh0_1_1, gz1_0_0, sm[496u + lane]);
      tg_dmma(gh0_0_0, gh0_0_1, gz1_0_1, sm[528u + lane]);
      tg_dmma(gh0_1_0, gh0_1_1, gz1_0_1, sm[560u + lane]);
      tg_dmma(gh0_0_0, gh0_0_1, gz1_1_0, sm[592u + lane]);
      tg_dmma(gh0_1_0, gh0_1_1, gz1_1_0, sm[624u + lane]);
      tg_dmma(gh0_0_0, gh0_0_1, gz1_1_1, sm[656u + lane]);
      tg_dmma(gh0_1_0, gh0_1_1, gz1_1_1, sm[688u + lane]);
      gzb[g * 20u + 0u + 2u * c] = active ? gz1_0_0 : (T)0;
      gzb[g * 20u + 1u + 2u * c] = active ? gz1_0_1 : (T)0;
      gzb[g * 20u + 8u + 2u * c] = active ? gz1_1_0 : (T)0;
      gzb[g * 20u + 9u + 2u * c] = active ? gz1_1_1 : (T)0;
      xb[g * 36u + 0u + 2u * c] = active ? dh0_0_0 : (T)0;
      xb[g * 36u + 1u + 2u * c] = active ? dh0_0_1 : (T)0;
      xb[g * 36u + 8u + 2u * c] = active ? dh0_1_0 : (T)0;
      xb[g * 36u + 9u + 2u * c] = active ? dh0_1_1 : (T)0;
      if (c == 0u) xb[g * 36u + 16u] = active ? (T)1 : (T)0;
      __syncwarp();
      const T qa1_0_0 = gzb[(0u + c) * 20u + 0u + g];
      const T qa1_0_1 = gzb[(0u + c) * 20u + 8u + g];
      const T qb1_0_0 = xb[(0u + c) * 36u + 0u + g];
      const T qb1_0_1 = xb[(0u + c) * 36u + 8u + g];
      const T qb1_0_2 = xb[(0u + c) * 36u + 16u + g];
      tg_dmma(aw1_0_0_0, aw1_0_0_1, qa1_0_0, qb1_0_0);
      tg_dmma(aw1_0_1_0, aw1_0_1_1, qa1_0_0, qb1_0_1);
      tg_dmma(aw1_0_2_0, aw1_0_2_1, qa1_0_0, qb1_0_2);
      tg_dmma(aw1_1_0_0, aw1_1_0_1, qa1_0_1, qb1_0_0);
      tg_dmma(aw1_1_1_0, aw1_1_1_1, qa1_0_1, qb1_0_1);
      tg_dmma(aw1_1_2_0, aw1_1_2_1, qa1_0_1, qb1_0_2);
      const T qa1_1_0 = gzb[(4u + c) * 20u + 0u + g];
      const T qa1_1_1 = gzb[(4u + c) * 20u + 8u + g];
      const T qb1_1_0 = xb[(4u + c) * 36u + 0u + g];
      const T qb1_1_1 = xb[(4u + c) * 36u + 8u + g];
      const T qb1_1_2 = xb[(4u + c) * 36u + 16u + g];
      tg_dmma(aw1_0_0_0, aw1_0_0_1, qa1_1_0, qb1_1_0);
      tg_dmma(aw1_0_1_0, aw1_0_1_1, qa1_1_0, qb1_1_1);
      tg_dmma(aw1_0_2_0, aw1_0_2_1, qa1_1_0, qb1_1_2);
      tg_dmma(aw1_1_0_0, aw1_1_0_1, qa1_1_1, qb1_1_0);
      tg_dmma(aw1_1_1_0, aw1_1_1_1, qa1_1_1, qb1_1_1);
      tg_dmma(aw1_1_2_0, aw1_1_2_1, qa1_1_1, qb1_1_2);
      __syncwarp();
      // dense 0 reverse
      T gz0_0_0 = gh0_0_0 * ((T)1 - dh0_0_0 * dh0_0_0);
      T gz0_0_1 = gh0_0_1 * ((T)1 - dh0_0_1 * dh0_0_1);
      T gz0_1_0 = gh0_1_0 * ((T)1 - dh0_1_0 * dh0_1_0);
      T gz0_1_1 = gh0_1_1 * ((T)1 - dh0_1_1 * dh0_1_1);
      T dx0_0_0 = (T)0, dx0_0_1 = (T)0;
      tg_dmma(dx0_0_0, dx0_0_1, gz0_0_0, sm[64u + lane]);
      tg_dmma(dx0_0_0, dx0_0_1, gz0_0_1, sm[96u + lane]);
      tg_dmma(dx0_0_0, dx0_0_1, gz0_1_0, sm[128u + lane]);
      tg_dmma(dx0_0_0, dx0_0_1, gz0_1_1, sm[160u + lane]);
      const T px1 = __shfl_sync(0xffffffffu, dx0_0_0, (lane & ~3u) | 0u);
      T g0 = px1;
      const T px2 = __shfl_sync(0xffffffffu, dx0_0_1, (lane & ~3u) | 0u);
      T g1 = px2;
      gzb[g * 20u + 0u + 2u * c] = active ? gz0_0_0 : (T)0;
      gzb[g * 20u + 1u + 2u * c] = active ? gz0_0_1 : (T)0;
      gzb[g * 20u + 8u + 2u * c] = active ? gz0_1_0 : (T)0;
      gzb[g * 20u + 9u + 2u * c] = active ? gz0_1_1 : (T)0;
      if (c == 0u) xb[g * 36u + 0u] = active ? v0 : (T)0;
      if (c == 1u) xb[g * 36u + 1u] = active ? v1 : (T)0;
      if (c == 0u) xb[g * 36u + 2u] = active ? (T)1 : (T)0;
      __syncwarp();
      const T qa0_0_0 = gzb[(0u + c) * 20u + 0u + g];
      const T qa0_0_1 = gzb[(0u + c) * 20u + 8u + g];
      const T qb0_0_0 = xb[(0u + c) * 36u + 0u + g];
      tg_dmma(aw0_0_0_0, aw0_0_0_1, qa0_0_0, qb0_0_0);
      tg_dmma(aw0_1_0_0, aw0_1_0_1, qa0_0_1, qb0_0_0);
      const T qa0_1_0 = gzb[(4u + c) * 20u + 0u + g];
      const T qa0_1_1 = gzb[(4u + c) * 20u + 8u + g];
      const T qb0_1_0 = xb[(4u + c) * 36u + 0u + g];
      tg_dmma(aw0_0_0_0, aw0_0_0_1, qa0_1_0, qb0_1_0);
      tg_dmma(aw0_1_0_0, aw0_1_0_1, qa0_1_1, qb0_1_0);
      __syncwarp();
      if (igrad && active && c == 0u) igrad[0ull * batch + s] = g0;
      if (igrad && active && c == 0u) igrad[1ull * batch + s] = g1;
      if (igrad && active && c == 0u) igrad[2ull * batch + s] = g2;
      if (active && c == 0u) {
        as0 += (T)1.0 * g71;
      }
    }
    __syncwarp();
  }
  as0 += __shfl_xor_sync(0xffffffffu, as0, 4);
  as0 += __shfl_xor_sync(0xffffffffu, as0, 8);
  as0 += __shfl_xor_sync(0xffffffffu, as0, 16);
  {
    T* red = sRed + warp * 338u;
    { const unsigned n = 0u + g, k = 0u + 2u * c; if (n < 16u) { if (k < 2u) red[0u + n * 2u + k] = aw0_0_0_0; if (k == 2u && cBD0[n] != 0xffffffffu) red[cBD0[n]] = aw0_0_0_0; } }
    { const unsigned n = 0u + g, k = 1u + 2u * c; if (n < 16u) { if (k < 2u) red[0u + n * 2u + k] = aw0_0_0_1; if (k == 2u && cBD0[n] != 0xffffffffu) red[cBD0[n]] = aw0_0_0_1; } }
    { const unsigned n = 8u + g, k = 0u + 2u * c; if (n < 16u) { if (k < 2u) red[0u + n * 2u + k] = aw0_1_0_0; if (k == 2u && cBD0[n] != 0xffffffffu) red[cBD0[n]] = aw0_1_0_0; } }
    { const unsigned n = 8u + g, k = 1u + 2u * c; if (n < 16u) { if (k < 2u) red[0u + n * 2u + k] = aw0_1_0_1; if (k == 2u && cBD0[n] != 0xffffffffu) red[cBD0[n]] = aw0_1_0_1; } }
    { const unsigned n = 0u + g, k = 0u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_0_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_0_0; } }
    { const unsigned n = 0u + g, k = 1u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_0_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_0_1; } }
    { const unsigned n = 0u + g, k = 8u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_1_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_1_0; } }
    { const unsigned n = 0u + g, k = 9u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_1_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_1_1; } }
    { const unsigned n = 0u + g, k = 16u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_2_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_2_0; } }
    { const unsigned n = 0u + g, k = 17u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_0_2_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_0_2_1; } }
    { const unsigned n = 8u + g, k = 0u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_0_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_0_0; } }
    { const unsigned n = 8u + g, k = 1u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_0_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_0_1; } }
    { const unsigned n = 8u + g, k = 8u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_1_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_1_0; } }
    { const unsigned n = 8u + g, k = 9u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_1_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_1_1; } }
    { const unsigned n = 8u + g, k = 16u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_2_0; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_2_0; } }
    { const unsigned n = 8u + g, k = 17u + 2u * c; if (n < 16u) { if (k < 16u) red[48u + n * 16u + k] = aw1_1_2_1; if (k == 16u && cBD1[n] != 0xffffffffu) red[cBD1[n]] = aw1_1_2_1; } }
    { const unsigned n = 0u + g, k = 0u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_0_0; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_0_0; } }
    { const unsigned n = 0u + g, k = 1u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_0_1; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_0_1; } }
    { const unsigned n = 0u + g, k = 8u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_1_0; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_1_0; } }
    { const unsigned n = 0u + g, k = 9u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_1_1; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_1_1; } }
    { const unsigned n = 0u + g, k = 16u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_2_0; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_2_0; } }
    { const unsigned n = 0u + g, k = 17u + 2u * c; if (n < 1u) { if (k < 16u) red[320u + n * 16u + k] = aw2_0_2_1; if (k == 16u && cBD2[n] != 0xffffffffu) red[cBD2[n]] = aw2_0_2_1; } }
    if (lane == 0u) red[337u] = as0;
  }
  __syncthreads();
  for (unsigned d = tid; d < 338u; d += 128u) {
    T t = (T)0;
    for (unsigned w = 0; w < 4u; ++w) t += sRed[w * 338u + d];
    partial[(unsigned long long)d * grid_rows + blockIdx.x] = t;
  }
}
extern "C" __global__ void __launch_bounds__(256) tg_jit_epi(const JitArgs A) {
  __shared__ T sU[340];
  __shared__ T sG[340];
  __shared__ unsigned last;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // tg_jit_tape's partials / UV
  const unsigned warp = (blockIdx.x * 256u + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  if (warp < 338u) {
    const T* row = A.partial + (unsigned long long)warp * A.grid_rows;
    T t = (T)0;
    unsigned c = lane;
    for (; c + 224u < A.grid_rows; c += 256u) {  // 8 loads in flight, added in sequential order
      T x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(row + c + 32u * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) t += x[u];
    }
    for (; c < A.grid_rows; c += 32u) t += __ldcg(row + c);
    for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
    if (lane == 0) A.partial2[warp] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(A.tickets, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (unsigned i = threadIdx.x; i < 340u; i += 256u) { sU[i] = __ldcg(A.UVw + i); sG[i] = (T)0; }
  __syncthreads();
  for (unsigned d = threadIdx.x; d < 338u; d += 256u) sG[cDU[d]] = __ldcg(A.partial2 + d);
  if (threadIdx.x == 0) A.tickets[0] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
      sG[337] += sG[338] * (T)0.0001;
  }
  __syncthreads();
  { const T g = sG[337];
    for (unsigned j = threadIdx.x; j < 337u; j += 256u) {
      const unsigned u = cUO[337u + j];
      T c;
      c = g * (T)2 * sU[u];
      if (u < 339u) sG[u] += c;
    }
    __syncthreads(); }
  for (unsigned i = threadIdx.x; i < 337u; i += 256u) {
    const T gs = sG[i];
    if (A.grad_sum) A.grad_sum[i] = gs;
    if (A.gd_params) A.gd_params[i] = A.gd_params[i] - A.gamma * gs / A.gd_batch;
  }
}
