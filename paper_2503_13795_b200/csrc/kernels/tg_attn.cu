// tg_attn.cu — fused softmax attention heads (kAttn) of the staged tier.
//
// A head (tg_program.hpp Attn) is the scalar subgraph the reference ops build
// for softmax(scale q K^T) V, one query unit per position.  In the staged tier
// its rows live in HBM as [row][sample]; the interpreter form
// (attn_fwd_sample / attn_bwd_sample in tg_ops.cuh) walks one sample per
// thread through every unit and recomputes the scores several times.  Here a
// CTA takes one head and a tile of kS samples:
//   * the head's key and value rows for the tile are staged once in shared
//     memory as [key][dim][sample] (kS consecutive samples of a row are one
//     32-byte sector in HBM);
//   * thread (sample s, slot t) runs units t and U-1-t, so every slot does
//     about the same number of (unit, key) steps under a causal key prefix;
//     the four slots of a warp walk the same key index, so their shared
//     reads are broadcasts of one word per sample (no bank conflicts);
//   * forward: one pass per unit with a running max / sum (the max shift is a
//     constant of the reference graph; rescaling by exp(m_old - m_new) gives
//     the same value up to rounding);
//   * reverse, with D_u = dO_u . o_u (= sum_j a_j dA_j, the normaliser's
//     adjoint term of the div / reduceSum / exp chain):
//       phase A (query-owned): dq_u = scale sum_j a_j (dO_u.v_j - D_u) k_j,
//       phase B (key-owned, q and dO of every unit staged in shared memory):
//       dk_j = scale sum_u a_uj (dO_u.v_j - D_u) q_u,  dv_j = sum_u a_uj dO_u.
//     The head is the only pusher into its q / k / v rows: it stores them.
#include <cuda_runtime.h>

#include <cstdint>

#include "tg_ops.cuh"
#include "tg_devcache.cuh"
#include "tg_staged.cuh"

namespace tgk {
namespace {

constexpr int kS = 8;          // samples per CTA
constexpr int kSlots = 32;     // unit / key slots per sample
constexpr int kThreads = kS * kSlots;
constexpr int kHDMax = 16;     // fast-path limit on the key / value width (padded to HD = 4, 8 or 16)
constexpr int kMaxKeys = 64;   // fast-path limit on keys and units

struct AttnStage {
  const tgc::Instr* list;
  const tgc::Attn* attn;
  const std::uint32_t* arows;
  float* V;
  float* G;
  std::size_t ld, n;
  std::uint32_t begin;
};

__device__ __forceinline__ void unit_rows(const tgc::Attn& A, const std::uint32_t* ar, std::uint32_t u, std::uint32_t& q,
                                          std::uint32_t& o, std::uint32_t& n) {
  q = ar[A.unit_off + 3 * u];
  o = ar[A.unit_off + 3 * u + 1];
  n = ar[A.unit_off + 3 * u + 2];
}

// stage rows {row_of(j) + i : j < nk, i < w} of X for the tile into dst[j][i][s],
// zero-padded to HD columns (padded products contribute exact zeros)
template <int HD, class RowOf>
__device__ __forceinline__ void stage_rows(float* dst, const float* X, std::size_t ld, std::size_t c0, std::size_t n,
                                           std::uint32_t nk, std::uint32_t w, RowOf row_of) {
  const std::uint32_t total = nk * HD * kS;
  for (std::uint32_t e = threadIdx.x; e < total; e += kThreads) {
    const std::uint32_t s = e % kS, ji = e / kS, j = ji / HD, i = ji % HD;
    const std::size_t col = c0 + s;
    dst[e] = (col < n && i < w) ? X[std::size_t(row_of(j) + i) * ld + col] : 0.f;
  }
}

template <int HD> __host__ __device__ constexpr std::size_t tile_floats() { return std::size_t(kMaxKeys) * HD * kS; }
template <int HD> constexpr std::size_t fwd_smem() { return 2 * tile_floats<HD>() * sizeof(float); }
template <int HD> constexpr std::size_t bwd_smem() {
  return 2 * tile_floats<HD>() * sizeof(float) + 3 * kMaxKeys * kS * sizeof(float) + kMaxKeys * 4;
}

template <int HD>
__global__ void __launch_bounds__(kThreads) k_attn_fwd(AttnStage a) {
  constexpr std::size_t kTile = tile_floats<HD>();
  extern __shared__ __align__(16) float smf[];
  float* Ks = smf;
  float* Vs = smf + kTile;
  const tgc::Attn A = a.attn[a.list[a.begin + blockIdx.x].aux];
  const std::uint32_t* K = a.arows + A.key_off;
  const std::size_t c0 = std::size_t(blockIdx.y) * kS;
  const std::uint32_t hd = A.hd, dv = A.dv, U = A.n_units;
  stage_rows<HD>(Ks, a.V, a.ld, c0, a.n, A.n_keys, hd, [&](std::uint32_t j) { return K[2 * j]; });
  stage_rows<HD>(Vs, a.V, a.ld, c0, a.n, A.n_keys, dv, [&](std::uint32_t j) { return K[2 * j + 1]; });
  __syncthreads();
  const std::uint32_t s = threadIdx.x % kS, slot = threadIdx.x / kS;
  const std::size_t col = c0 + s;
  if (col >= a.n) return;
  const float scale = static_cast<float>(A.scale);
  for (std::uint32_t u0 = slot; u0 < (U + 1) / 2; u0 += kSlots)
    for (int pass = 0; pass < 2; ++pass) {
      const std::uint32_t u = pass ? U - 1 - u0 : u0;
      if (pass && u == u0) break;
      std::uint32_t qr, orow, n;
      unit_rows(A, a.arows, u, qr, orow, n);
      float q[HD], acc[HD];
#pragma unroll
      for (int i = 0; i < HD; ++i) {
        q[i] = i < static_cast<int>(hd) ? a.V[std::size_t(qr + i) * a.ld + col] : 0.f;
        acc[i] = 0.f;
      }
      float m = -INFINITY, l = 0.f;
      for (std::uint32_t j = 0; j < n; ++j) {
        const float* kj = Ks + j * HD * kS + s;
        float c = 0.f;
#pragma unroll
        for (int i = 0; i < HD; ++i)
          c += q[i] * kj[i * kS];
        c *= scale;
        if (c > m) {
          const float r = expf(m - c);
          l *= r;
#pragma unroll
          for (int i = 0; i < HD; ++i) acc[i] *= r;
          m = c;
        }
        const float p = expf(c - m);
        l += p;
        const float* vj = Vs + j * HD * kS + s;
#pragma unroll
        for (int i = 0; i < HD; ++i)
          acc[i] += p * vj[i * kS];
      }
      const float inv = 1.f / l;
#pragma unroll
      for (int i = 0; i < HD; ++i)
        if (i < static_cast<int>(dv)) a.V[std::size_t(orow + i) * a.ld + col] = acc[i] * inv;
      a.V[std::size_t(A.stat_row + 2 * u) * a.ld + col] = m;        // for the reverse kernel
      a.V[std::size_t(A.stat_row + 2 * u + 1) * a.ld + col] = inv;
    }
}

template <int HD>
__global__ void __launch_bounds__(kThreads) k_attn_bwd(AttnStage a) {
  constexpr std::size_t kTile = tile_floats<HD>();
  extern __shared__ __align__(16) float smb[];
  float* S0 = smb;               // phase A: keys;   phase B: queries
  float* S1 = smb + kTile;       // phase A: values; phase B: output adjoints
  float* st_m = smb + 2 * kTile;
  float* st_l = st_m + kMaxKeys * kS;
  float* st_d = st_l + kMaxKeys * kS;
  std::uint32_t* st_n = reinterpret_cast<std::uint32_t*>(st_d + kMaxKeys * kS);
  const tgc::Attn A = a.attn[a.list[a.begin + blockIdx.x].aux];
  const std::uint32_t* K = a.arows + A.key_off;
  const std::size_t c0 = std::size_t(blockIdx.y) * kS;
  const std::uint32_t hd = A.hd, dv = A.dv, U = A.n_units, T = A.n_keys;
  const float scale = static_cast<float>(A.scale);
  stage_rows<HD>(S0, a.V, a.ld, c0, a.n, T, hd, [&](std::uint32_t j) { return K[2 * j]; });
  stage_rows<HD>(S1, a.V, a.ld, c0, a.n, T, dv, [&](std::uint32_t j) { return K[2 * j + 1]; });
  for (std::uint32_t u = threadIdx.x; u < U; u += kThreads) st_n[u] = a.arows[A.unit_off + 3 * u + 2];
  __syncthreads();
  const std::uint32_t s = threadIdx.x % kS, slot = threadIdx.x / kS;
  const std::size_t col = c0 + s;
  const bool live = col < a.n;
  // ---- phase A: query-owned (dq, softmax statistics) ----
  if (live)
    for (std::uint32_t u0 = slot; u0 < (U + 1) / 2; u0 += kSlots)
      for (int pass = 0; pass < 2; ++pass) {
        const std::uint32_t u = pass ? U - 1 - u0 : u0;
        if (pass && u == u0) break;
        std::uint32_t qr, orow, n;
        unit_rows(A, a.arows, u, qr, orow, n);
        float q[HD], dO[HD], dq[HD];
        float D = 0.f;
#pragma unroll
        for (int i = 0; i < HD; ++i) {
          q[i] = i < static_cast<int>(hd) ? a.V[std::size_t(qr + i) * a.ld + col] : 0.f;
          dO[i] = i < static_cast<int>(dv) ? a.G[std::size_t(orow + i) * a.ld + col] : 0.f;
          if (i < static_cast<int>(dv)) D += dO[i] * a.V[std::size_t(orow + i) * a.ld + col];
          dq[i] = 0.f;
        }
        // softmax statistics of the forward pass (stat rows)
        const float m = a.V[std::size_t(A.stat_row + 2 * u) * a.ld + col];
        const float inv = a.V[std::size_t(A.stat_row + 2 * u + 1) * a.ld + col];
        for (std::uint32_t j = 0; j < n; ++j) {
          const float* kj = S0 + j * HD * kS + s;
          const float* vj = S1 + j * HD * kS + s;
          float c = 0.f, dA = 0.f;
#pragma unroll
          for (int i = 0; i < HD; ++i) {
            c += q[i] * kj[i * kS];
            if (i < static_cast<int>(dv)) dA += dO[i] * vj[i * kS];
          }
          const float p = expf(c * scale - m) * inv;
          const float ds = scale * p * (dA - D);
#pragma unroll
          for (int i = 0; i < HD; ++i)
            dq[i] += ds * kj[i * kS];
        }
#pragma unroll
        for (int i = 0; i < HD; ++i)
          if (i < static_cast<int>(hd)) a.G[std::size_t(qr + i) * a.ld + col] = dq[i];
        st_m[u * kS + s] = m;
        st_l[u * kS + s] = inv;
        st_d[u * kS + s] = D;
      }
  __syncthreads();
  // ---- phase B: key-owned (dk, dv) with queries and output adjoints staged ----
  stage_rows<HD>(S0, a.V, a.ld, c0, a.n, U, hd, [&](std::uint32_t u) { return a.arows[A.unit_off + 3 * u]; });
  stage_rows<HD>(S1, a.G, a.ld, c0, a.n, U, dv, [&](std::uint32_t u) { return a.arows[A.unit_off + 3 * u + 1]; });
  __syncthreads();
  if (!live) return;
  for (std::uint32_t j0 = slot; j0 < (T + 1) / 2; j0 += kSlots)
    for (int pass = 0; pass < 2; ++pass) {
      const std::uint32_t j = pass ? T - 1 - j0 : j0;
      if (pass && j == j0) break;
      const std::uint32_t kr = K[2 * j], vr = K[2 * j + 1];
      float k[HD], v[HD], dk[HD], dvv[HD];
#pragma unroll
      for (int i = 0; i < HD; ++i) {
        k[i] = i < static_cast<int>(hd) ? a.V[std::size_t(kr + i) * a.ld + col] : 0.f;
        v[i] = i < static_cast<int>(dv) ? a.V[std::size_t(vr + i) * a.ld + col] : 0.f;
        dk[i] = 0.f;
        dvv[i] = 0.f;
      }
      for (std::uint32_t u = 0; u < U; ++u) {
        if (st_n[u] <= j) continue;
        const float* qu = S0 + u * HD * kS + s;
        const float* du = S1 + u * HD * kS + s;
        float c = 0.f, dA = 0.f;
#pragma unroll
        for (int i = 0; i < HD; ++i) {
          c += qu[i * kS] * k[i];
          dA += du[i * kS] * v[i];
        }
        const float p = expf(c * scale - st_m[u * kS + s]) * st_l[u * kS + s];
        const float ds = scale * p * (dA - st_d[u * kS + s]);
#pragma unroll
        for (int i = 0; i < HD; ++i) {
          dk[i] += ds * qu[i * kS];
          dvv[i] += p * du[i * kS];
        }
      }
#pragma unroll
      for (int i = 0; i < HD; ++i) {
        if (i < static_cast<int>(hd)) a.G[std::size_t(kr + i) * a.ld + col] = dk[i];
        if (i < static_cast<int>(dv)) a.G[std::size_t(vr + i) * a.ld + col] = dvv[i];
      }
    }
}

}  // namespace

bool attn_fast_ok(const tgc::Attn& A) {
  return A.hd <= static_cast<std::uint32_t>(kHDMax) && A.dv <= static_cast<std::uint32_t>(kHDMax) &&
         A.n_keys <= static_cast<std::uint32_t>(kMaxKeys) && A.n_units <= static_cast<std::uint32_t>(kMaxKeys) &&
         A.hd > 0 && A.dv > 0 && A.n_keys > 0;
}

namespace {
template <int HD>
cudaError_t launch_attn_hd(bool fwd, const AttnStage& a, dim3 grid, cudaStream_t st) {
  static PerDeviceOnce attr;
  if (const cudaError_t e0 = attr.ensure([] {
        for (cudaError_t e : {cudaFuncSetAttribute(k_attn_fwd<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fwd_smem<HD>())),
                              cudaFuncSetAttribute(k_attn_bwd<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bwd_smem<HD>()))})
          if (e != cudaSuccess) return e;
        return cudaSuccess;
      }); e0 != cudaSuccess)
    return e0;
  if (fwd) k_attn_fwd<HD><<<grid, kThreads, fwd_smem<HD>(), st>>>(a);
  else k_attn_bwd<HD><<<grid, kThreads, bwd_smem<HD>(), st>>>(a);
  return cudaGetLastError();
}
}  // namespace

// hd_max: the widest head of the stage (the kernels pad every head to HD)
cudaError_t launch_attn(bool fwd, const tgc::Instr* list, std::uint32_t begin, std::uint32_t count, const tgc::Attn* attn,
                        const std::uint32_t* arows, float* V, float* G, std::size_t n, std::size_t ld, std::uint32_t hd_max,
                        cudaStream_t st) {
  if (!count || !n) return cudaSuccess;
  AttnStage a{list, attn, arows, V, G, ld, n, begin};
  const dim3 grid(count, static_cast<unsigned>((n + kS - 1) / kS));
  if (hd_max <= 4) return launch_attn_hd<4>(fwd, a, grid, st);
  if (hd_max <= 8) return launch_attn_hd<8>(fwd, a, grid, st);
  return launch_attn_hd<16>(fwd, a, grid, st);
}

}  // namespace tgk
