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
__device__ __forceinline__ double tg_tanh(double x) {
  const double a = fmin(fabs(x), 20.0);  // tanh(20) = 1 - 8.5e-18 rounds to 1
  const double t = -2.0 * a;
  const double kf = rint(t * 1.4426950408889634);
  double r = fma(kf, -6.93147180369123816490e-01, t);
  r = fma(kf, -1.90821492927058770002e-10, r);
  double q = 1.0 / 6227020800.0;   // 1/13!
  q = fma(q, r, 1.0 / 479001600.0);
  q = fma(q, r, 1.0 / 39916800.0);
  q = fma(q, r, 1.0 / 3628800.0);
  q = fma(q, r, 1.0 / 362880.0);
  q = fma(q, r, 1.0 / 40320.0);
  q = fma(q, r, 1.0 / 5040.0);
  q = fma(q, r, 1.0 / 720.0);
  q = fma(q, r, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
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
__constant__ T cUV[340];
__constant__ unsigned cDG0[18] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 0, 1};
__constant__ unsigned cDG1[32] = {16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17};
__constant__ unsigned cDG2[17] = {32, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33};
extern "C" __global__ void __launch_bounds__(128) tg_jit_tape(
    const T* __restrict__ in, const int* __restrict__ idx, unsigned long long batch,
    T* __restrict__ loss, T* __restrict__ igrad, T* __restrict__ partial, unsigned grid_rows,
    unsigned long long* err_key, const T* __restrict__ UVg, const unsigned* __restrict__ cand,
    const unsigned* __restrict__ toff, const TermC* __restrict__ terms) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sG = reinterpret_cast<T*>(smem_raw);
  T* sV = sG + 34 * 129;
  T* sDW = sV + 34 * 129;
  T* sS = sDW + 338;
  (void)sG; (void)sV; (void)sDW; (void)sS;
  const unsigned tid = threadIdx.x;
  for (unsigned q = tid; q < 338u; q += 128u) sDW[q] = (T)0;
  T acc[3]; for (int q = 0; q < 3; ++q) acc[q] = 0;
  for (unsigned long long tile = blockIdx.x; tile * 128ull < batch; tile += gridDim.x) {
    const unsigned long long base = tile * 128ull;
#pragma unroll
    for (unsigned jj = 0; jj < 1u; ++jj) {
    const unsigned long long s = base + jj * 128u + tid;
    const unsigned col = jj * 128u + tid;
    (void)col;
    if (s < batch) {
      const T v0 = in[0ull * batch + s];
      const T v1 = in[1ull * batch + s];
      const T v2 = in[2ull * batch + s];
      const T dx0 = v0;
      const T dx1 = v1;
      T a2 = cUV[32]; a2 += dx0 * cUV[0]; a2 += dx1 * cUV[1];
      const T v3 = a2;
      const T v19 = tg_tanh(v3);
      T a3 = cUV[33]; a3 += dx0 * cUV[2]; a3 += dx1 * cUV[3];
      const T v4 = a3;
      const T v20 = tg_tanh(v4);
      T a4 = cUV[34]; a4 += dx0 * cUV[4]; a4 += dx1 * cUV[5];
      const T v5 = a4;
      const T v21 = tg_tanh(v5);
      T a5 = cUV[35]; a5 += dx0 * cUV[6]; a5 += dx1 * cUV[7];
      const T v6 = a5;
      const T v22 = tg_tanh(v6);
      T a6 = cUV[36]; a6 += dx0 * cUV[8]; a6 += dx1 * cUV[9];
      const T v7 = a6;
      const T v23 = tg_tanh(v7);
      T a7 = cUV[37]; a7 += dx0 * cUV[10]; a7 += dx1 * cUV[11];
      const T v8 = a7;
      const T v24 = tg_tanh(v8);
      T a8 = cUV[38]; a8 += dx0 * cUV[12]; a8 += dx1 * cUV[13];
      const T v9 = a8;
      const T v25 = tg_tanh(v9);
      T a9 = cUV[39]; a9 += dx0 * cUV[14]; a9 += dx1 * cUV[15];
      const T v10 = a9;
      const T v26 = tg_tanh(v10);
      T a10 = cUV[40]; a10 += dx0 * cUV[16]; a10 += dx1 * cUV[17];
      const T v11 = a10;
      const T v27 = tg_tanh(v11);
      T a11 = cUV[41]; a11 += dx0 * cUV[18]; a11 += dx1 * cUV[19];
      const T v12 = a11;
      const T v28 = tg_tanh(v12);
      T a12 = cUV[42]; a12 += dx0 * cUV[20]; a12 += dx1 * cUV[21];
      const T v13 = a12;
      const T v29 = tg_tanh(v13);
      T a13 = cUV[43]; a13 += dx0 * cUV[22]; a13 += dx1 * cUV[23];
      const T v14 = a13;
      const T v30 = tg_tanh(v14);
      T a14 = cUV[44]; a14 += dx0 * cUV[24]; a14 += dx1 * cUV[25];
      const T v15 = a14;
      const T v31 = tg_tanh(v15);
      T a15 = cUV[45]; a15 += dx0 * cUV[26]; a15 += dx1 * cUV[27];
      const T v16 = a15;
      const T v32 = tg_tanh(v16);
      T a16 = cUV[46]; a16 += dx0 * cUV[28]; a16 += dx1 * cUV[29];
      const T v17 = a16;
      const T v33 = tg_tanh(v17);
      T a17 = cUV[47]; a17 += dx0 * cUV[30]; a17 += dx1 * cUV[31];
      const T v18 = a17;
      const T v34 = tg_tanh(v18);
      const T dx18 = v19;
      const T dx19 = v20;
      const T dx20 = v21;
      const T dx21 = v22;
      const T dx22 = v23;
      const T dx23 = v24;
      const T dx24 = v25;
      const T dx25 = v26;
      const T dx26 = v27;
      const T dx27 = v28;
      const T dx28 = v29;
      const T dx29 = v30;
      const T dx30 = v31;
      const T dx31 = v32;
      const T dx32 = v33;
      const T dx33 = v34;
      T a34 = cUV[304]; a34 += dx18 * cUV[48]; a34 += dx19 * cUV[49]; a34 += dx20 * cUV[50]; a34 += dx21 * cUV[51]; a34 += dx22 * cUV[52]; a34 += dx23 * cUV[53]; a34 += dx24 * cUV[54]; a34 += dx25 * cUV[55]; a34 += dx26 * cUV[56]; a34 += dx27 * cUV[57]; a34 += dx28 * cUV[58]; a34 += dx29 * cUV[59]; a34 += dx30 * cUV[60]; a34 += dx31 * cUV[61]; a34 += dx32 * cUV[62]; a34 += dx33 * cUV[63];
      const T v35 = a34;
      const T v51 = tg_tanh(v35);
      T a35 = cUV[305]; a35 += dx18 * cUV[64]; a35 += dx19 * cUV[65]; a35 += dx20 * cUV[66]; a35 += dx21 * cUV[67]; a35 += dx22 * cUV[68]; a35 += dx23 * cUV[69]; a35 += dx24 * cUV[70]; a35 += dx25 * cUV[71]; a35 += dx26 * cUV[72]; a35 += dx27 * cUV[73]; a35 += dx28 * cUV[74]; a35 += dx29 * cUV[75]; a35 += dx30 * cUV[76]; a35 += dx31 * cUV[77]; a35 += dx32 * cUV[78]; a35 += dx33 * cUV[79];
      const T v36 = a35;
      const T v52 = tg_tanh(v36);
      T a36 = cUV[306]; a36 += dx18 * cUV[80]; a36 += dx19 * cUV[81]; a36 += dx20 * cUV[82]; a36 += dx21 * cUV[83]; a36 += dx22 * cUV[84]; a36 += dx23 * cUV[85]; a36 += dx24 * cUV[86]; a36 += dx25 * cUV[87]; a36 += dx26 * cUV[88]; a36 += dx27 * cUV[89]; a36 += dx28 * cUV[90]; a36 += dx29 * cUV[91]; a36 += dx30 * cUV[92]; a36 += dx31 * cUV[93]; a36 += dx32 * cUV[94]; a36 += dx33 * cUV[95];
      const T v37 = a36;
      const T v53 = tg_tanh(v37);
      T a37 = cUV[307]; a37 += dx18 * cUV[96]; a37 += dx19 * cUV[97]; a37 += dx20 * cUV[98]; a37 += dx21 * cUV[99]; a37 += dx22 * cUV[100]; a37 += dx23 * cUV[101]; a37 += dx24 * cUV[102]; a37 += dx25 * cUV[103]; a37 += dx26 * cUV[104]; a37 += dx27 * cUV[105]; a37 += dx28 * cUV[106]; a37 += dx29 * cUV[107]; a37 += dx30 * cUV[108]; a37 += dx31 * cUV[109]; a37 += dx32 * cUV[110]; a37 += dx33 * cUV[111];
      const T v38 = a37;
      const T v54 = tg_tanh(v38);
      T a38 = cUV[308]; a38 += dx18 * cUV[112]; a38 += dx19 * cUV[113]; a38 += dx20 * cUV[114]; a38 += dx21 * cUV[115]; a38 += dx22 * cUV[116]; a38 += dx23 * cUV[117]; a38 += dx24 * cUV[118]; a38 += dx25 * cUV[119]; a38 += dx26 * cUV[120]; a38 += dx27 * cUV[121]; a38 += dx28 * cUV[122]; a38 += dx29 * cUV[123]; a38 += dx30 * cUV[124]; a38 += dx31 * cUV[125]; a38 += dx32 * cUV[126]; a38 += dx33 * cUV[127];
      const T v39 = a38;
      const T v55 = tg_tanh(v39);
      T a39 = cUV[309]; a39 += dx18 * cUV[128]; a39 += dx19 * cUV[129]; a39 += dx20 * cUV[130]; a39 += dx21 * cUV[131]; a39 += dx22 * cUV[132]; a39 += dx23 * cUV[133]; a39 += dx24 * cUV[134]; a39 += dx25 * cUV[135]; a39 += dx26 * cUV[136]; a39 += dx27 * cUV[137]; a39 += dx28 * cUV[138]; a39 += dx29 * cUV[139]; a39 += dx30 * cUV[140]; a39 += dx31 * cUV[141]; a39 += dx32 * cUV[142]; a39 += dx33 * cUV[143];
      const T v40 = a39;
      const T v56 = tg_tanh(v40);
      T a40 = cUV[310]; a40 += dx18 * cUV[144]; a40 += dx19 * cUV[145]; a40 += dx20 * cUV[146]; a40 += dx21 * cUV[147]; a40 += dx22 * cUV[148]; a40 += dx23 * cUV[149]; a40 += dx24 * cUV[150]; a40 += dx25 * cUV[151]; a40 += dx26 * cUV[152]; a40 += dx27 * cUV[153]; a40 += dx28 * cUV[154]; a40 += dx29 * cUV[155]; a40 += dx30 * cUV[156]; a40 += dx31 * cUV[157]; a40 += dx32 * cUV[158]; a40 += dx33 * cUV[159];
      const T v41 = a40;
      const T v57 = tg_tanh(v41);
      T a41 = cUV[311]; a41 += dx18 * cUV[160]; a41 += dx19 * cUV[161]; a41 += dx20 * cUV[162]; a41 += dx21 * cUV[163]; a41 += dx22 * cUV[164]; a41 += dx23 * cUV[165]; a41 += dx24 * cUV[166]; a41 += dx25 * cUV[167]; a41 += dx26 * cUV[168]; a41 += dx27 * cUV[169]; a41 += dx28 * cUV[170]; a41 += dx29 * cUV[171]; a41 += dx30 * cUV[172]; a41 += dx31 * cUV[173]; a41 += dx32 * cUV[174]; a41 += dx33 * cUV[175];
      const T v42 = a41;
      const T v58 = tg_tanh(v42);
      T a42 = cUV[312]; a42 += dx18 * cUV[176]; a42 += dx19 * cUV[177]; a42 += dx20 * cUV[178]; a42 += dx21 * cUV[179]; a42 += dx22 * cUV[180]; a42 += dx23 * cUV[181]; a42 += dx24 * cUV[182]; a42 += dx25 * cUV[183]; a42 += dx26 * cUV[184]; a42 += dx27 * cUV[185]; a42 += dx28 * cUV[186]; a42 += dx29 * cUV[187]; a42 += dx30 * cUV[188]; a42 += dx31 * cUV[189]; a42 += dx32 * cUV[190]; a42 += dx33 * cUV[191];
      const T v43 = a42;
      const T v59 = tg_tanh(v43);
      T a43 = cUV[313]; a43 += dx18 * cUV[192]; a43 += dx19 * cUV[193]; a43 += dx20 * cUV[194]; a43 += dx21 * cUV[195]; a43 += dx22 * cUV[196]; a43 += dx23 * cUV[197]; a43 += dx24 * cUV[198]; a43 += dx25 * cUV[199]; a43 += dx26 * cUV[200]; a43 += dx27 * cUV[201]; a43 += dx28 * cUV[202]; a43 += dx29 * cUV[203]; a43 += dx30 * cUV[204]; a43 += dx31 * cUV[205]; a43 += dx32 * cUV[206]; a43 += dx33 * cUV[207];
      const T v44 = a43;
      const T v60 = tg_tanh(v44);
      T a44 = cUV[314]; a44 += dx18 * cUV[208]; a44 += dx19 * cUV[209]; a44 += dx20 * cUV[210]; a44 += dx21 * cUV[211]; a44 += dx22 * cUV[212]; a44 += dx23 * cUV[213]; a44 += dx24 * cUV[214]; a44 += dx25 * cUV[215]; a44 += dx26 * cUV[216]; a44 += dx27 * cUV[217]; a44 += dx28 * cUV[218]; a44 += dx29 * cUV[219]; a44 += dx30 * cUV[220]; a44 += dx31 * cUV[221]; a44 += dx32 * cUV[222]; a44 += dx33 * cUV[223];
      const T v45 = a44;
      const T v61 = tg_tanh(v45);
      T a45 = cUV[315]; a45 += dx18 * cUV[224]; a45 += dx19 * cUV[225]; a45 += dx20 * cUV[226]; a45 += dx21 * cUV[227]; a45 += dx22 * cUV[228]; a45 += dx23 * cUV[229]; a45 += dx24 * cUV[230]; a45 += dx25 * cUV[231]; a45 += dx26 * cUV[232]; a45 += dx27 * cUV[233]; a45 += dx28 * cUV[234]; a45 += dx29 * cUV[235]; a45 += dx30 * cUV[236]; a45 += dx31 * cUV[237]; a45 += dx32 * cUV[238]; a45 += dx33 * cUV[239];
      const T v46 = a45;
      const T v62 = tg_tanh(v46);
      T a46 = cUV[316]; a46 += dx18 * cUV[240]; a46 += dx19 * cUV[241]; a46 += dx20 * cUV[242]; a46 += dx21 * cUV[243]; a46 += dx22 * cUV[244]; a46 += dx23 * cUV[245]; a46 += dx24 * cUV[246]; a46 += dx25 * cUV[247]; a46 += dx26 * cUV[248]; a46 += dx27 * cUV[249]; a46 += dx28 * cUV[250]; a46 += dx29 * cUV[251]; a46 += dx30 * cUV[252]; a46 += dx31 * cUV[253]; a46 += dx32 * cUV[254]; a46 += dx33 * cUV[255];
      const T v47 = a46;
      const T v63 = tg_tanh(v47);
      T a47 = cUV[317]; a47 += dx18 * cUV[256]; a47 += dx19 * cUV[257]; a47 += dx20 * cUV[258]; a47 += dx21 * cUV[259]; a47 += dx22 * cUV[260]; a47 += dx23 * cUV[261]; a47 += dx24 * cUV[262]; a47 += dx25 * cUV[263]; a47 += dx26 * cUV[264]; a47 += dx27 * cUV[265]; a47 += dx28 * cUV[266]; a47 += dx29 * cUV[267]; a47 += dx30 * cUV[268]; a47 += dx31 * cUV[269]; a47 += dx32 * cUV[270]; a47 += dx33 * cUV[271];
      const T v48 = a47;
      const T v64 = tg_tanh(v48);
      T a48 = cUV[318]; a48 += dx18 * cUV[272]; a48 += dx19 * cUV[273]; a48 += dx20 * cUV[274]; a48 += dx21 * cUV[275]; a48 += dx22 * cUV[276]; a48 += dx23 * cUV[277]; a48 += dx24 * cUV[278]; a48 += dx25 * cUV[279]; a48 += dx26 * cUV[280]; a48 += dx27 * cUV[281]; a48 += dx28 * cUV[282]; a48 += dx29 * cUV[283]; a48 += dx30 * cUV[284]; a48 += dx31 * cUV[285]; a48 += dx32 * cUV[286]; a48 += dx33 * cUV[287];
      const T v49 = a48;
      const T v65 = tg_tanh(v49);
      T a49 = cUV[319]; a49 += dx18 * cUV[288]; a49 += dx19 * cUV[289]; a49 += dx20 * cUV[290]; a49 += dx21 * cUV[291]; a49 += dx22 * cUV[292]; a49 += dx23 * cUV[293]; a49 += dx24 * cUV[294]; a49 += dx25 * cUV[295]; a49 += dx26 * cUV[296]; a49 += dx27 * cUV[297]; a49 += dx28 * cUV[298]; a49 += dx29 * cUV[299]; a49 += dx30 * cUV[300]; a49 += dx31 * cUV[301]; a49 += dx32 * cUV[302]; a49 += dx33 * cUV[303];
      const T v50 = a49;
      const T v66 = tg_tanh(v50);
      const T dx50 = v51;
      const T dx51 = v52;
      const T dx52 = v53;
      const T dx53 = v54;
      const T dx54 = v55;
      const T dx55 = v56;
      const T dx56 = v57;
      const T dx57 = v58;
      const T dx58 = v59;
      const T dx59 = v60;
      const T dx60 = v61;
      const T dx61 = v62;
      const T dx62 = v63;
      const T dx63 = v64;
      const T dx64 = v65;
      const T dx65 = v66;
      T a66 = cUV[336]; a66 += dx50 * cUV[320]; a66 += dx51 * cUV[321]; a66 += dx52 * cUV[322]; a66 += dx53 * cUV[323]; a66 += dx54 * cUV[324]; a66 += dx55 * cUV[325]; a66 += dx56 * cUV[326]; a66 += dx57 * cUV[327]; a66 += dx58 * cUV[328]; a66 += dx59 * cUV[329]; a66 += dx60 * cUV[330]; a66 += dx61 * cUV[331]; a66 += dx62 * cUV[332]; a66 += dx63 * cUV[333]; a66 += dx64 * cUV[334]; a66 += dx65 * cUV[335];
      const T v67 = a66;
      const T v68 = v2 * v67;
      const T v69 = cUV[339] - v68;
      const T v70 = v69 > (T)0 ? v69 : (T)0;
      const T v71 = v70 + cUV[338];
      if (loss) loss[s] = v71;
      T g71 = (T)1;
      T g70 = g71;
      T g69 = (v69 > (T)0 ? g70 : (T)0);
      T g68 = -g69;
      T g2 = g68 * v67;
      T g67 = g68 * v2;
      T gx67 = (T)0;
      T gx68 = (T)0;
      T gx69 = (T)0;
      T gx70 = (T)0;
      T gx71 = (T)0;
      T gx72 = (T)0;
      T gx73 = (T)0;
      T gx74 = (T)0;
      T gx75 = (T)0;
      T gx76 = (T)0;
      T gx77 = (T)0;
      T gx78 = (T)0;
      T gx79 = (T)0;
      T gx80 = (T)0;
      T gx81 = (T)0;
      T gx82 = (T)0;
      gx67 += g67 * cUV[320]; gx68 += g67 * cUV[321]; gx69 += g67 * cUV[322]; gx70 += g67 * cUV[323]; gx71 += g67 * cUV[324]; gx72 += g67 * cUV[325]; gx73 += g67 * cUV[326]; gx74 += g67 * cUV[327]; gx75 += g67 * cUV[328]; gx76 += g67 * cUV[329]; gx77 += g67 * cUV[330]; gx78 += g67 * cUV[331]; gx79 += g67 * cUV[332]; gx80 += g67 * cUV[333]; gx81 += g67 * cUV[334]; gx82 += g67 * cUV[335];
      T g51 = gx67;
      T g52 = gx68;
      T g53 = gx69;
      T g54 = gx70;
      T g55 = gx71;
      T g56 = gx72;
      T g57 = gx73;
      T g58 = gx74;
      T g59 = gx75;
      T g60 = gx76;
      T g61 = gx77;
      T g62 = gx78;
      T g63 = gx79;
      T g64 = gx80;
      T g65 = gx81;
      T g66 = gx82;
      T gx83 = (T)0;
      T gx84 = (T)0;
      T gx85 = (T)0;
      T gx86 = (T)0;
      T gx87 = (T)0;
      T gx88 = (T)0;
      T gx89 = (T)0;
      T gx90 = (T)0;
      T gx91 = (T)0;
      T gx92 = (T)0;
      T gx93 = (T)0;
      T gx94 = (T)0;
      T gx95 = (T)0;
      T gx96 = (T)0;
      T gx97 = (T)0;
      T gx98 = (T)0;
      T g35 = g51 * ((T)1 - v51 * v51);
      gx83 += g35 * cUV[48]; gx84 += g35 * cUV[49]; gx85 += g35 * cUV[50]; gx86 += g35 * cUV[51]; gx87 += g35 * cUV[52]; gx88 += g35 * cUV[53]; gx89 += g35 * cUV[54]; gx90 += g35 * cUV[55]; gx91 += g35 * cUV[56]; gx92 += g35 * cUV[57]; gx93 += g35 * cUV[58]; gx94 += g35 * cUV[59]; gx95 += g35 * cUV[60]; gx96 += g35 * cUV[61]; gx97 += g35 * cUV[62]; gx98 += g35 * cUV[63];
      T g36 = g52 * ((T)1 - v52 * v52);
      gx83 += g36 * cUV[64]; gx84 += g36 * cUV[65]; gx85 += g36 * cUV[66]; gx86 += g36 * cUV[67]; gx87 += g36 * cUV[68]; gx88 += g36 * cUV[69]; gx89 += g36 * cUV[70]; gx90 += g36 * cUV[71]; gx91 += g36 * cUV[72]; gx92 += g36 * cUV[73]; gx93 += g36 * cUV[74]; gx94 += g36 * cUV[75]; gx95 += g36 * cUV[76]; gx96 += g36 * cUV[77]; gx97 += g36 * cUV[78]; gx98 += g36 * cUV[79];
      T g37 = g53 * ((T)1 - v53 * v53);
      gx83 += g37 * cUV[80]; gx84 += g37 * cUV[81]; gx85 += g37 * cUV[82]; gx86 += g37 * cUV[83]; gx87 += g37 * cUV[84]; gx88 += g37 * cUV[85]; gx89 += g37 * cUV[86]; gx90 += g37 * cUV[87]; gx91 += g37 * cUV[88]; gx92 += g37 * cUV[89]; gx93 += g37 * cUV[90]; gx94 += g37 * cUV[91]; gx95 += g37 * cUV[92]; gx96 += g37 * cUV[93]; gx97 += g37 * cUV[94]; gx98 += g37 * cUV[95];
      T g38 = g54 * ((T)1 - v54 * v54);
      gx83 += g38 * cUV[96]; gx84 += g38 * cUV[97]; gx85 += g38 * cUV[98]; gx86 += g38 * cUV[99]; gx87 += g38 * cUV[100]; gx88 += g38 * cUV[101]; gx89 += g38 * cUV[102]; gx90 += g38 * cUV[103]; gx91 += g38 * cUV[104]; gx92 += g38 * cUV[105]; gx93 += g38 * cUV[106]; gx94 += g38 * cUV[107]; gx95 += g38 * cUV[108]; gx96 += g38 * cUV[109]; gx97 += g38 * cUV[110]; gx98 += g38 * cUV[111];
      T g39 = g55 * ((T)1 - v55 * v55);
      gx83 += g39 * cUV[112]; gx84 += g39 * cUV[113]; gx85 += g39 * cUV[114]; gx86 += g39 * cUV[115]; gx87 += g39 * cUV[116]; gx88 += g39 * cUV[117]; gx89 += g39 * cUV[118]; gx90 += g39 * cUV[119]; gx91 += g39 * cUV[120]; gx92 += g39 * cUV[121]; gx93 += g39 * cUV[122]; gx94 += g39 * cUV[123]; gx95 += g39 * cUV[124]; gx96 += g39 * cUV[125]; gx97 += g39 * cUV[126]; gx98 += g39 * cUV[127];
      T g40 = g56 * ((T)1 - v56 * v56);
      gx83 += g40 * cUV[128]; gx84 += g40 * cUV[129]; gx85 += g40 * cUV[130]; gx86 += g40 * cUV[131]; gx87 += g40 * cUV[132]; gx88 += g40 * cUV[133]; gx89 += g40 * cUV[134]; gx90 += g40 * cUV[135]; gx91 += g40 * cUV[136]; gx92 += g40 * cUV[137]; gx93 += g40 * cUV[138]; gx94 += g40 * cUV[139]; gx95 += g40 * cUV[140]; gx96 += g40 * cUV[141]; gx97 += g40 * cUV[142]; gx98 += g40 * cUV[143];
      T g41 = g57 * ((T)1 - v57 * v57);
      gx83 += g41 * cUV[144]; gx84 += g41 * cUV[145]; gx85 += g41 * cUV[146]; gx86 += g41 * cUV[147]; gx87 += g41 * cUV[148]; gx88 += g41 * cUV[149]; gx89 += g41 * cUV[150]; gx90 += g41 * cUV[151]; gx91 += g41 * cUV[152]; gx92 += g41 * cUV[153]; gx93 += g41 * cUV[154]; gx94 += g41 * cUV[155]; gx95 += g41 * cUV[156]; gx96 += g41 * cUV[157]; gx97 += g41 * cUV[158]; gx98 += g41 * cUV[159];
      T g42 = g58 * ((T)1 - v58 * v58);
      gx83 += g42 * cUV[160]; gx84 += g42 * cUV[161]; gx85 += g42 * cUV[162]; gx86 += g42 * cUV[163]; gx87 += g42 * cUV[164]; gx88 += g42 * cUV[165]; gx89 += g42 * cUV[166]; gx90 += g42 * cUV[167]; gx91 += g42 * cUV[168]; gx92 += g42 * cUV[169]; gx93 += g42 * cUV[170]; gx94 += g42 * cUV[171]; gx95 += g42 * cUV[172]; gx96 += g42 * cUV[173]; gx97 += g42 * cUV[174]; gx98 += g42 * cUV[175];
      T g43 = g59 * ((T)1 - v59 * v59);
      gx83 += g43 * cUV[176]; gx84 += g43 * cUV[177]; gx85 += g43 * cUV[178]; gx86 += g43 * cUV[179]; gx87 += g43 * cUV[180]; gx88 += g43 * cUV[181]; gx89 += g43 * cUV[182]; gx90 += g43 * cUV[183]; gx91 += g43 * cUV[184]; gx92 += g43 * cUV[185]; gx93 += g43 * cUV[186]; gx94 += g43 * cUV[187]; gx95 += g43 * cUV[188]; gx96 += g43 * cUV[189]; gx97 += g43 * cUV[190]; gx98 += g43 * cUV[191];
      T g44 = g60 * ((T)1 - v60 * v60);
      gx83 += g44 * cUV[192]; gx84 += g44 * cUV[193]; gx85 += g44 * cUV[194]; gx86 += g44 * cUV[195]; gx87 += g44 * cUV[196]; gx88 += g44 * cUV[197]; gx89 += g44 * cUV[198]; gx90 += g44 * cUV[199]; gx91 += g44 * cUV[200]; gx92 += g44 * cUV[201]; gx93 += g44 * cUV[202]; gx94 += g44 * cUV[203]; gx95 += g44 * cUV[204]; gx96 += g44 * cUV[205]; gx97 += g44 * cUV[206]; gx98 += g44 * cUV[207];
      T g45 = g61 * ((T)1 - v61 * v61);
      gx83 += g45 * cUV[208]; gx84 += g45 * cUV[209]; gx85 += g45 * cUV[210]; gx86 += g45 * cUV[211]; gx87 += g45 * cUV[212]; gx88 += g45 * cUV[213]; gx89 += g45 * cUV[214]; gx90 += g45 * cUV[215]; gx91 += g45 * cUV[216]; gx92 += g45 * cUV[217]; gx93 += g45 * cUV[218]; gx94 += g45 * cUV[219]; gx95 += g45 * cUV[220]; gx96 += g45 * cUV[221]; gx97 += g45 * cUV[222]; gx98 += g45 * cUV[223];
      T g46 = g62 * ((T)1 - v62 * v62);
      gx83 += g46 * cUV[224]; gx84 += g46 * cUV[225]; gx85 += g46 * cUV[226]; gx86 += g46 * cUV[227]; gx87 += g46 * cUV[228]; gx88 += g46 * cUV[229]; gx89 += g46 * cUV[230]; gx90 += g46 * cUV[231]; gx91 += g46 * cUV[232]; gx92 += g46 * cUV[233]; gx93 += g46 * cUV[234]; gx94 += g46 * cUV[235]; gx95 += g46 * cUV[236]; gx96 += g46 * cUV[237]; gx97 += g46 * cUV[238]; gx98 += g46 * cUV[239];
      T g47 = g63 * ((T)1 - v63 * v63);
      gx83 += g47 * cUV[240]; gx84 += g47 * cUV[241]; gx85 += g47 * cUV[242]; gx86 += g47 * cUV[243]; gx87 += g47 * cUV[244]; gx88 += g47 * cUV[245]; gx89 += g47 * cUV[246]; gx90 += g47 * cUV[247]; gx91 += g47 * cUV[248]; gx92 += g47 * cUV[249]; gx93 += g47 * cUV[250]; gx94 += g47 * cUV[251]; gx95 += g47 * cUV[252]; gx96 += g47 * cUV[253]; gx97 += g47 * cUV[254]; gx98 += g47 * cUV[255];
      T g48 = g64 * ((T)1 - v64 * v64);
      gx83 += g48 * cUV[256]; gx84 += g48 * cUV[257]; gx85 += g48 * cUV[258]; gx86 += g48 * cUV[259]; gx87 += g48 * cUV[260]; gx88 += g48 * cUV[261]; gx89 += g48 * cUV[262]; gx90 += g48 * cUV[263]; gx91 += g48 * cUV[264]; gx92 += g48 * cUV[265]; gx93 += g48 * cUV[266]; gx94 += g48 * cUV[267]; gx95 += g48 * cUV[268]; gx96 += g48 * cUV[269]; gx97 += g48 * cUV[270]; gx98 += g48 * cUV[271];
      T g49 = g65 * ((T)1 - v65 * v65);
      gx83 += g49 * cUV[272]; gx84 += g49 * cUV[273]; gx85 += g49 * cUV[274]; gx86 += g49 * cUV[275]; gx87 += g49 * cUV[276]; gx88 += g49 * cUV[277]; gx89 += g49 * cUV[278]; gx90 += g49 * cUV[279]; gx91 += g49 * cUV[280]; gx92 += g49 * cUV[281]; gx93 += g49 * cUV[282]; gx94 += g49 * cUV[283]; gx95 += g49 * cUV[284]; gx96 += g49 * cUV[285]; gx97 += g49 * cUV[286]; gx98 += g49 * cUV[287];
      T g50 = g66 * ((T)1 - v66 * v66);
      gx83 += g50 * cUV[288]; gx84 += g50 * cUV[289]; gx85 += g50 * cUV[290]; gx86 += g50 * cUV[291]; gx87 += g50 * cUV[292]; gx88 += g50 * cUV[293]; gx89 += g50 * cUV[294]; gx90 += g50 * cUV[295]; gx91 += g50 * cUV[296]; gx92 += g50 * cUV[297]; gx93 += g50 * cUV[298]; gx94 += g50 * cUV[299]; gx95 += g50 * cUV[300]; gx96 += g50 * cUV[301]; gx97 += g50 * cUV[302]; gx98 += g50 * cUV[303];
      T g19 = gx83;
      T g20 = gx84;
      T g21 = gx85;
      T g22 = gx86;
      T g23 = gx87;
      T g24 = gx88;
      T g25 = gx89;
      T g26 = gx90;
      T g27 = gx91;
      T g28 = gx92;
      T g29 = gx93;
      T g30 = gx94;
      T g31 = gx95;
      T g32 = gx96;
      T g33 = gx97;
      T g34 = gx98;
      T gx99 = (T)0;
      T gx100 = (T)0;
      T g3 = g19 * ((T)1 - v19 * v19);
      gx99 += g3 * cUV[0]; gx100 += g3 * cUV[1];
      T g4 = g20 * ((T)1 - v20 * v20);
      gx99 += g4 * cUV[2]; gx100 += g4 * cUV[3];
      T g5 = g21 * ((T)1 - v21 * v21);
      gx99 += g5 * cUV[4]; gx100 += g5 * cUV[5];
      T g6 = g22 * ((T)1 - v22 * v22);
      gx99 += g6 * cUV[6]; gx100 += g6 * cUV[7];
      T g7 = g23 * ((T)1 - v23 * v23);
      gx99 += g7 * cUV[8]; gx100 += g7 * cUV[9];
      T g8 = g24 * ((T)1 - v24 * v24);
      gx99 += g8 * cUV[10]; gx100 += g8 * cUV[11];
      T g9 = g25 * ((T)1 - v25 * v25);
      gx99 += g9 * cUV[12]; gx100 += g9 * cUV[13];
      T g10 = g26 * ((T)1 - v26 * v26);
      gx99 += g10 * cUV[14]; gx100 += g10 * cUV[15];
      T g11 = g27 * ((T)1 - v27 * v27);
      gx99 += g11 * cUV[16]; gx100 += g11 * cUV[17];
      T g12 = g28 * ((T)1 - v28 * v28);
      gx99 += g12 * cUV[18]; gx100 += g12 * cUV[19];
      T g13 = g29 * ((T)1 - v29 * v29);
      gx99 += g13 * cUV[20]; gx100 += g13 * cUV[21];
      T g14 = g30 * ((T)1 - v30 * v30);
      gx99 += g14 * cUV[22]; gx100 += g14 * cUV[23];
      T g15 = g31 * ((T)1 - v31 * v31);
      gx99 += g15 * cUV[24]; gx100 += g15 * cUV[25];
      T g16 = g32 * ((T)1 - v32 * v32);
      gx99 += g16 * cUV[26]; gx100 += g16 * cUV[27];
      T g17 = g33 * ((T)1 - v33 * v33);
      gx99 += g17 * cUV[28]; gx100 += g17 * cUV[29];
      T g18 = g34 * ((T)1 - v34 * v34);
      gx99 += g18 * cUV[30]; gx100 += g18 * cUV[31];
      T g0 = gx99;
      T g1 = gx100;
      if (igrad) igrad[0ull * batch + s] = g0;
      if (igrad) igrad[1ull * batch + s] = g1;
      if (igrad) igrad[2ull * batch + s] = g2;
      sV[0u + col] = v0;
      sV[129u + col] = v1;
      sG[0u + col] = g3;
      sG[129u + col] = g4;
      sG[258u + col] = g5;
      sG[387u + col] = g6;
      sG[516u + col] = g7;
      sG[645u + col] = g8;
      sG[774u + col] = g9;
      sG[903u + col] = g10;
      sG[1032u + col] = g11;
      sG[1161u + col] = g12;
      sG[1290u + col] = g13;
      sG[1419u + col] = g14;
      sG[1548u + col] = g15;
      sG[1677u + col] = g16;
      sG[1806u + col] = g17;
      sG[1935u + col] = g18;
      sV[258u + col] = v19;
      sV[387u + col] = v20;
      sV[516u + col] = v21;
      sV[645u + col] = v22;
      sV[774u + col] = v23;
      sV[903u + col] = v24;
      sV[1032u + col] = v25;
      sV[1161u + col] = v26;
      sV[1290u + col] = v27;
      sV[1419u + col] = v28;
      sV[1548u + col] = v29;
      sV[1677u + col] = v30;
      sV[1806u + col] = v31;
      sV[1935u + col] = v32;
      sV[2064u + col] = v33;
      sV[2193u + col] = v34;
      sG[2064u + col] = g35;
      sG[2193u + col] = g36;
      sG[2322u + col] = g37;
      sG[2451u + col] = g38;
      sG[2580u + col] = g39;
      sG[2709u + col] = g40;
      sG[2838u + col] = g41;
      sG[2967u + col] = g42;
      sG[3096u + col] = g43;
      sG[3225u + col] = g44;
      sG[3354u + col] = g45;
      sG[3483u + col] = g46;
      sG[3612u + col] = g47;
      sG[3741u + col] = g48;
      sG[3870u + col] = g49;
      sG[3999u + col] = g50;
      sV[2322u + col] = v51;
      sV[2451u + col] = v52;
      sV[2580u + col] = v53;
      sV[2709u + col] = v54;
      sV[2838u + col] = v55;
      sV[2967u + col] = v56;
      sV[3096u + col] = v57;
      sV[3225u + col] = v58;
      sV[3354u + col] = v59;
      sV[3483u + col] = v60;
      sV[3612u + col] = v61;
      sV[3741u + col] = v62;
      sV[3870u + col] = v63;
      sV[3999u + col] = v64;
      sV[4128u + col] = v65;
      sV[4257u + col] = v66;
      sG[4128u + col] = g67;
      sG[4257u + col] = g71;
    }
    }
    __syncthreads();
    const unsigned valid = (unsigned)((batch - base) < 128ull ? (batch - base) : 128ull);
    T totq[3];
#pragma unroll 1
    for (unsigned q = 0; q < 3u; ++q) {
      const unsigned d = q * 128u + tid;
      T tot = 0;
      if (d < 338u)
      for (unsigned t = toff[d]; t < toff[d + 1]; ++t) {
        const TermC tm = terms[t];
        const T* ga = sG + tm.a * 129u;
        T p0 = 0, p1 = 0, p2 = 0, p3 = 0;
        unsigned j = 0;
        if (tm.kind == 0) {
          if (tm.f == 0xffffffffu) {
            for (; j + 4 <= valid; j += 4) { p0 += ga[j]; p1 += ga[j + 1]; p2 += ga[j + 2]; p3 += ga[j + 3]; }
            for (; j < valid; ++j) p0 += ga[j];
          } else {
            const T* vf = sV + tm.f * 129u;
            for (; j + 4 <= valid; j += 4) { p0 += ga[j] * vf[j]; p1 += ga[j + 1] * vf[j + 1]; p2 += ga[j + 2] * vf[j + 2]; p3 += ga[j + 3] * vf[j + 3]; }
            for (; j < valid; ++j) p0 += ga[j] * vf[j];
          }
        } else {
          const int* ix = idx + (unsigned long long)tm.f * batch + base;
          for (; j < valid; ++j) p0 += ix[j] == tm.row ? ga[j] : (T)0;
        }
        tot += (T)tm.coef * ((p0 + p1) + (p2 + p3));
      }
      totq[q] = tot;
    }
    // dense weight gradient 16x2: register-tiled outer products over samples
    if (tid < 64u) {
      const unsigned bb = tid % 4u, c = tid / 4u;
      const unsigned j0 = (bb / 1u) * 4u, k0 = (bb % 1u) * 4u;
      const unsigned s0 = c * valid / 16u, s1 = (c + 1u) * valid / 16u;
      unsigned ar[4], fr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ar[u] = cDG0[min(j0 + u, 15u)] * 129u;
        fr[u] = cDG0[16u + min(k0 + u, 1u)] * 129u;
      }
      T a4[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a4[u][v] = 0;
      for (unsigned j = s0; j < s1; ++j) {
        T av[4], fv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { av[u] = sG[ar[u] + j]; fv[u] = sV[fr[u] + j]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a4[u][v] += av[u] * fv[v];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (j0 + u < 16u && k0 + v < 2u)
            sS[c * 32u + (j0 + u) * 2u + k0 + v] = a4[u][v];
    }
    __syncthreads();
    for (unsigned q = tid; q < 32u; q += 128u) {
      T t = 0;
      for (unsigned c = 0; c < 16u; ++c) t += sS[c * 32u + q];
      sDW[0u + q] = t;
    }
    __syncthreads();
    // dense weight gradient 16x16: register-tiled outer products over samples
    if (tid < 32u) {
      const unsigned bb = tid % 16u, c = tid / 16u;
      const unsigned j0 = (bb / 4u) * 4u, k0 = (bb % 4u) * 4u;
      const unsigned s0 = c * valid / 2u, s1 = (c + 1u) * valid / 2u;
      unsigned ar[4], fr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ar[u] = cDG1[min(j0 + u, 15u)] * 129u;
        fr[u] = cDG1[16u + min(k0 + u, 15u)] * 129u;
      }
      T a4[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a4[u][v] = 0;
      for (unsigned j = s0; j < s1; ++j) {
        T av[4], fv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { av[u] = sG[ar[u] + j]; fv[u] = sV[fr[u] + j]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a4[u][v] += av[u] * fv[v];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (j0 + u < 16u && k0 + v < 16u)
            sS[c * 256u + (j0 + u) * 16u + k0 + v] = a4[u][v];
    }
    __syncthreads();
    for (unsigned q = tid; q < 256u; q += 128u) {
      T t = 0;
      for (unsigned c = 0; c < 2u; ++c) t += sS[c * 256u + q];
      sDW[48u + q] = t;
    }
    __syncthreads();
    // dense weight gradient 1x16: register-tiled outer products over samples
    if (tid < 64u) {
      const unsigned bb = tid % 4u, c = tid / 4u;
      const unsigned j0 = (bb / 4u) * 4u, k0 = (bb % 4u) * 4u;
      const unsigned s0 = c * valid / 16u, s1 = (c + 1u) * valid / 16u;
      unsigned ar[4], fr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ar[u] = cDG2[min(j0 + u, 0u)] * 129u;
        fr[u] = cDG2[1u + min(k0 + u, 15u)] * 129u;
      }
      T a4[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a4[u][v] = 0;
      for (unsigned j = s0; j < s1; ++j) {
        T av[4], fv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { av[u] = sG[ar[u] + j]; fv[u] = sV[fr[u] + j]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a4[u][v] += av[u] * fv[v];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (j0 + u < 1u && k0 + v < 16u)
            sS[c * 16u + (j0 + u) * 16u + k0 + v] = a4[u][v];
    }
    __syncthreads();
    for (unsigned q = tid; q < 16u; q += 128u) {
      T t = 0;
      for (unsigned c = 0; c < 16u; ++c) t += sS[c * 16u + q];
      sDW[320u + q] = t;
    }
    __syncthreads();
#pragma unroll 1
    for (unsigned q = 0; q < 3u; ++q) {
      const unsigned d = q * 128u + tid;
      if (d >= 338u) break;
      const T tot = totq[q] + sDW[d];
      acc[q] += tot;
    }
    __syncthreads();
  }
  for (int q = 0; q < 3; ++q) { const unsigned d = q * 128u + tid;
    if (d < 338u) partial[(unsigned long long)d * grid_rows + blockIdx.x] = acc[q]; }
}
