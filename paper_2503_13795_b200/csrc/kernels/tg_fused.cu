// tg_fused.cu — the embedding-MLP / softmax-CE tape as one kernel (staged tier,
// fp32): SURVEY.md §8d cfg3, the Bengio character MLP
//   x = [E[tok_0] .. E[tok_{C-1}]],  h = act(W1 x + b1),  z = W2 h + b2,
//   loss = log(sum_j exp(z_j - m)) - (z_t - m),  m = stop-gradient max z
// recognised in the recorded scalar graph by tg_abi.cpp (fused_mlp_plan).
//
// The staged chain runs this as 31 launches over HBM rows (1.43 ms for
// b = 262,144: every 200-wide activation written and re-read).  Here a CTA
// keeps the 47.6 KB of weights and the same-sized gradient accumulators in
// shared memory and walks tiles of kS samples: gather, two products, the CE
// and its adjoint, the two weight-gradient products, the input adjoints and
// the embedding scatter all stay on chip.  Each product is a register-tiled
// FP32 loop over shared-memory operands in a fixed k order; the per-CTA sums
// are written once, as partials [cta][q], and reduced over CTAs in a fixed
// order (k_fused_reduce) into the step's gradient accumulator — the same
// deterministic contract as the rest of the staged tier.
// Measured 1.90 ms on cfg3 (r07f: issue 49%, a quarter of the stall samples at
// barriers between phases whose products leave most threads idle: 27 x 32 and
// 30 x 32 outputs over K = 200), so it is opt-in (TG_FUSED_MLP=1); warp-level
// tensor-core tiles for the six products are what it needs to beat the chain.
#include <cuda_runtime.h>

#include <cstdint>

#include "tg_devcache.cuh"
#include "tg_ops.cuh"
#include "tg_staged.cuh"

namespace tgk {
namespace {

constexpr int kS = 32;            // samples per tile
constexpr int kLd = kS + 1;       // activation row stride (bank-conflict free column walks)
constexpr int kThreads = 512;

// C[m][n] = sum_k a(m, k) b(k, n) over a TM x TN register tile per thread;
// n is the fast thread index (B reads along n are consecutive, A reads broadcast).
template <int TM, int TN, class FA, class FB, class FE>
__device__ __forceinline__ void tile_gemm(int M, int N, int K, FA a, FB b, FE epi) {
  const int tm = (M + TM - 1) / TM, tn = (N + TN - 1) / TN;
  for (int t = threadIdx.x; t < tm * tn; t += kThreads) {
    const int m0 = (t / tn) * TM, n0 = (t % tn) * TN;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    for (int k = 0; k < K; ++k) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = m0 + i < M ? a(m0 + i, k) : 0.f;
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = n0 + j < N ? b(k, n0 + j) : 0.f;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        if (m0 + i < M && n0 + j < N) epi(m0 + i, n0 + j, acc[i][j]);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_fused_mlp_ce(FusedMlpArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = a.C, E = a.E, V = a.V, H = a.H, O = a.O, NI = C * E;
  // weights [W1 | b1 | W2 | b2 | E] and their gradient sums, both in q order
  float* sW1 = sm;
  float* sb1 = sW1 + H * NI;
  float* sW2 = sb1 + H;
  float* sb2 = sW2 + O * H;
  float* sE = sb2 + O;
  float* gq = sE + V * E;
  float* gW1 = gq;
  float* gb1 = gW1 + H * NI;
  float* gW2 = gb1 + H;
  float* gb2 = gW2 + O * H;
  float* gE = gb2 + O;
  float* X = gE + V * E;        // [NI][kLd]   inputs, later their adjoints
  float* Hh = X + NI * kLd;     // [H][kLd]    hidden activations
  float* Z = Hh + H * kLd;      // [O][kLd]    logits, then their adjoints
  float* D = Z + O * kLd;       // [H][kLd]    hidden pre-activation adjoints
  float* XT = D + H * kLd;      // [kS][NI + 1]  x transposed (weight-gradient products read rows of samples)
  float* HT = XT + kS * (NI + 1);   // [kS][H + 1]
  int* tok = reinterpret_cast<int*>(HT + kS * (H + 1));   // [C + 1][kS]: context tokens, target

  const std::uint32_t nq = a.nq;
  for (std::uint32_t q = threadIdx.x; q < nq; q += kThreads) {
    std::uint32_t u;
    if (q < std::uint32_t(H * NI)) u = a.uv_W1 + q;
    else if (q < std::uint32_t(H * NI + H)) u = a.uv_b1 == tgc::kNone ? tgc::kNone : a.uv_b1 + (q - H * NI);
    else if (q < std::uint32_t(H * NI + H + O * H)) u = a.uv_W2 + (q - H * NI - H);
    else if (q < std::uint32_t(H * NI + H + O * H + O)) u = a.uv_b2 == tgc::kNone ? tgc::kNone : a.uv_b2 + (q - H * NI - H - O * H);
    else u = a.uv_E + (q - H * NI - H - O * H - O);
    sm[q] = u == tgc::kNone ? 0.f : a.UV[u];
    gq[q] = 0.f;
  }
  __syncthreads();

  const std::size_t n_tiles = (a.batch + kS - 1) / kS;
  for (std::size_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const std::size_t s0 = tile * kS;
    const int ns = static_cast<int>(a.batch - s0 < std::size_t(kS) ? a.batch - s0 : kS);
    // ---- tokens and the gathered inputs ----
    for (int i = threadIdx.x; i < (C + 1) * kS; i += kThreads) {
      const int c = i / kS, s = i % kS;
      const std::uint32_t col = c < C ? a.ctx_col[c] : a.tgt_col;
      tok[i] = s < ns ? a.idx[std::size_t(col) * a.batch + s0 + s] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NI * kS; i += kThreads) {
      const int q = i / kS, s = i % kS;
      const float v = s < ns ? sE[tok[(q / E) * kS + s] * E + q % E] : 0.f;
      X[q * kLd + s] = v;
      XT[s * (NI + 1) + q] = v;
    }
    __syncthreads();
    // ---- h = act(W1 x + b1) ----
    tile_gemm<4, 4>(
        H, kS, NI, [&](int j, int k) { return sW1[j * NI + k]; }, [&](int k, int s) { return X[k * kLd + s]; },
        [&](int j, int s, float v) {
          const float h = act_fwd<float>(a.act, v + sb1[j]);
          Hh[j * kLd + s] = h;
          HT[s * (H + 1) + j] = h;
        });
    __syncthreads();
    // ---- z = W2 h + b2 ----
    tile_gemm<2, 2>(
        O, kS, H, [&](int c, int j) { return sW2[c * H + j]; }, [&](int j, int s) { return Hh[j * kLd + s]; },
        [&](int c, int s, float v) { Z[c * kLd + s] = v + sb2[c]; });
    __syncthreads();
    // ---- softmax CE (stop-gradient max shift) and its adjoint dz_c = softmax_c - [c == t] ----
    if (threadIdx.x < kS) {
      const int s = threadIdx.x;
      if (s < ns) {
        float m = Z[s];
        for (int c = 1; c < O; ++c) m = fmaxf(m, Z[c * kLd + s]);
        float tot = 0.f;
        for (int c = 0; c < O; ++c) tot += d_exp(Z[c * kLd + s] - m);
        const int t = tok[C * kS + s];
        a.loss[s0 + s] = d_log(tot) - (Z[t * kLd + s] - m);
        const float inv = 1.f / tot;
        for (int c = 0; c < O; ++c) {
          const float e = d_exp(Z[c * kLd + s] - m);
          Z[c * kLd + s] = inv * e - (c == t ? 1.f : 0.f);
        }
      } else {
        for (int c = 0; c < O; ++c) Z[c * kLd + s] = 0.f;   // padding samples contribute nothing
      }
    }
    __syncthreads();
    // ---- gW2 += dz h^T, gb2 += sum_s dz ----
    tile_gemm<2, 4>(
        O, H, kS, [&](int c, int s) { return Z[c * kLd + s]; }, [&](int s, int j) { return HT[s * (H + 1) + j]; },
        [&](int c, int j, float v) { gW2[c * H + j] += v; });
    if (threadIdx.x < O) {
      float t = 0.f;
      for (int s = 0; s < kS; ++s) t += Z[threadIdx.x * kLd + s];
      gb2[threadIdx.x] += t;
    }
    // ---- dz1 = act'(h) * W2^T dz ----
    tile_gemm<4, 4>(
        H, kS, O, [&](int j, int c) { return sW2[c * H + j]; }, [&](int c, int s) { return Z[c * kLd + s]; },
        [&](int j, int s, float v) { D[j * kLd + s] = act_bwd_h<float>(a.act, v, Hh[j * kLd + s]); });
    __syncthreads();
    // ---- gW1 += dz1 x^T, gb1 += sum_s dz1 ----
    tile_gemm<4, 2>(
        H, NI, kS, [&](int j, int s) { return D[j * kLd + s]; }, [&](int s, int k) { return XT[s * (NI + 1) + k]; },
        [&](int j, int k, float v) { gW1[j * NI + k] += v; });
    for (int j = threadIdx.x; j < H; j += kThreads) {
      float t = 0.f;
      for (int s = 0; s < kS; ++s) t += D[j * kLd + s];
      gb1[j] += t;
    }
    __syncthreads();
    // ---- dx = W1^T dz1 (into X) ----
    tile_gemm<2, 2>(
        NI, kS, H, [&](int k, int j) { return sW1[j * NI + k]; }, [&](int j, int s) { return D[j * kLd + s]; },
        [&](int k, int s, float v) { X[k * kLd + s] = v; });
    __syncthreads();
    // ---- embedding scatter: gE[v][e] += dx[c E + e][s] over tok[c][s] == v, in (c, s) order ----
    for (int i = threadIdx.x; i < V * E; i += kThreads) {
      const int v = i / E, e = i % E;
      float t = 0.f;
      for (int c = 0; c < C; ++c)
        for (int s = 0; s < ns; ++s)
          if (tok[c * kS + s] == v) t += X[(c * E + e) * kLd + s];
      gE[i] += t;
    }
    __syncthreads();
  }
  for (std::uint32_t q = threadIdx.x; q < nq; q += kThreads) a.part[std::size_t(blockIdx.x) * nq + q] = gq[q];
}

// acc[dmap[q]] += sum over CTAs of part[cta][q], in CTA order.
__global__ void k_fused_reduce(const float* __restrict__ part, std::uint32_t nq, std::uint32_t n_cta,
                               const std::uint32_t* __restrict__ dmap, float* __restrict__ acc) {
  const std::uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq || dmap[q] == tgc::kNone) return;
  float t = 0.f;
  for (std::uint32_t c = 0; c < n_cta; ++c) t += part[std::size_t(c) * nq + q];
  acc[dmap[q]] += t;
}

}  // namespace

std::size_t fused_mlp_smem(const FusedMlpArgs& a) {
  const std::size_t NI = std::size_t(a.C) * a.E;
  return (2 * std::size_t(a.nq) + (NI + 2 * a.H + a.O) * kLd + kS * (NI + 1 + a.H + 1)) * sizeof(float) +
         (a.C + 1) * kS * sizeof(int);
}

unsigned fused_mlp_grid(std::size_t batch, int nsm) {
  const std::size_t tiles = (batch + kS - 1) / kS;
  return static_cast<unsigned>(tiles < std::size_t(nsm) ? tiles : std::size_t(nsm));
}

cudaError_t launch_fused_mlp(const FusedMlpArgs& a, unsigned grid, const std::uint32_t* dmap, float* acc,
                             cudaStream_t st) {
  const std::size_t smem = fused_mlp_smem(a);
  static PerDeviceMax attr;
  if (const cudaError_t e = attr.raise_to(static_cast<int>(smem), [](int bytes) {
        return cudaFuncSetAttribute(k_fused_mlp_ce, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      }); e != cudaSuccess)
    return e;
  k_fused_mlp_ce<<<grid, kThreads, smem, st>>>(a);
  if (const cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
  k_fused_reduce<<<(a.nq + 255) / 256, 256, 0, st>>>(a.part, a.nq, grid, dmap, acc);
  return cudaGetLastError();
}

}  // namespace tgk
