// tg_umma.cu — 5th-generation tensor-core GEMM (tcgen05 / TMEM) for the dense
// layers of the staged path, fp32 accuracy via 3xTF32.
//
// D[m][n] = sum_k A(m, k) B(k, n) with fp32 operands split into TF32 pairs
// a = a_hi + a_lo (cvt.rna.tf32): D = A_lo B_hi + A_hi B_lo + A_hi B_hi,
// relative error ~2^-21 per product (plain TF32, 2^-11, would miss the 1e-5
// parity bar).  Accumulators live in TMEM (128 lanes x 128 fp32 columns),
// operands in shared memory as canonical K-major no-swizzle core matrices
// (8 rows x 16 B), described by tcgen05 shared-memory descriptors:
//   byte(m, k) = (k / 4) * (BM * 16) + m * 16 + (k % 4) * 4
//   LBO (next core matrix along K) = BM * 16,  SBO (next 8 rows) = 128.
// CTA: 128 threads.  All threads stage a k-tile (LDG -> hi/lo -> STS) into a
// 2-deep ring; one thread issues 4 k-steps x 3 tcgen05.mma.kind::tf32 and
// tcgen05.commit's them to the stage's mbarrier; the ring slot is refilled
// only after that mbarrier completes, so loads of tile t+1 overlap the MMAs
// of tile t.  Epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes 32w..32w+31
// = output rows), bias / activation / accumulate / split-K partial store.
#include <cuda_runtime.h>

#include <cstdint>

#include "tg_ops.cuh"
#include "tg_staged.cuh"

namespace tgk {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr std::uint32_t kTileA = BM * BK * 4, kTileB = BN * BK * 4;   // 16 KB each
constexpr std::uint32_t kStage = 2 * kTileA + 2 * kTileB;             // hi + lo of A and B
constexpr std::uint32_t kSmem = 2 * kStage + 64;

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// Nearest TF32 (10 explicit mantissa bits) with the low 13 bits cleared, so
// that x - tf32(x) is the exact remainder the tensor core would otherwise
// truncate away (cvt.rna.tf32.f32 leaves those bits in the register).
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

__device__ __forceinline__ std::uint64_t umma_desc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<std::uint64_t>(lbo >> 4) << 16) |
         (static_cast<std::uint64_t>(sbo >> 4) << 32) | (1ull << 46);   // version 1 (sm_100), SWIZZLE_NONE
}

__device__ __forceinline__ void mma_tf32(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                         std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_wait(std::uint32_t mbar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TG_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TG_DONE;\n\t"
      "bra TG_WAIT;\n"
      "TG_DONE:\n\t}\n" ::"r"(mbar),
      "r"(parity));
}

// Stage rows [0, R) x k [0, BK) of an operand view into hi / lo tiles.
// kcontig: element (r, k) at P[r * ld + k], else at P[k * ld + r].
__device__ __forceinline__ void stage_operand(const float* __restrict__ P, std::size_t ld, bool kcontig, std::uint32_t r0,
                                              std::uint32_t R, std::uint32_t k0, std::uint32_t kend, unsigned char* hi,
                                              unsigned char* lo, int rows_tile) {
  const int r = threadIdx.x;  // one row per thread (128 threads, 128 rows)
  const std::uint32_t gr = r0 + r;
#pragma unroll 2
  for (int kc = 0; kc < BK / 4; ++kc) {
    float v[4];
    const std::uint32_t gk = k0 + kc * 4;
    if (kcontig) {
      const float* src = P + std::size_t(gr) * ld + gk;
      if (gr < R && gk + 3 < kend && (reinterpret_cast<std::uintptr_t>(src) & 15) == 0) {
        const float4 q = *reinterpret_cast<const float4*>(src);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (gr < R && gk + e < kend) ? src[e] : 0.f;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = (gr < R && gk + e < kend) ? P[std::size_t(gk + e) * ld + gr] : 0.f;
    }
    float4 h, l;
    h.x = tf32_rna(v[0]); l.x = tf32_rna(v[0] - h.x);
    h.y = tf32_rna(v[1]); l.y = tf32_rna(v[1] - h.y);
    h.z = tf32_rna(v[2]); l.z = tf32_rna(v[2] - h.z);
    h.w = tf32_rna(v[3]); l.w = tf32_rna(v[3] - h.w);
    const std::uint32_t off = kc * (rows_tile * 16) + r * 16;
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

__global__ void __launch_bounds__(128, 1) k_umma_tf32x3(GemmArgs<float> g) {
  extern __shared__ __align__(1024) unsigned char smem[];
  std::uint64_t* mbar = reinterpret_cast<std::uint64_t*>(smem + 2 * kStage);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(smem + 2 * kStage + 32);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const std::uint32_t tmem = *tmem_slot;

  const std::uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  std::uint32_t k_begin = 0, k_end = g.K;
  if (g.epi == kEpiSplitK) {
    k_begin = blockIdx.z * g.k_chunk;
    k_end = min(g.K, k_begin + g.k_chunk);
  }
  const std::uint32_t T = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
  // kind::tf32: D F32 (bit 4), A/B TF32 (bits 7, 10), K-major A/B, N >> 3 at 17, M >> 4 at 24
  const std::uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

  for (std::uint32_t t = 0; t < T; ++t) {
    const std::uint32_t st = t & 1;
    if (t >= 2) mbar_wait(smem_u32(&mbar[st]), ((t - 2) >> 1) & 1);   // ring slot free again
    unsigned char* base = smem + st * kStage;
    const std::uint32_t k0 = k_begin + t * BK;
    stage_operand(g.A, g.lda, g.a_kmaj, m0, g.M, k0, k_end, base, base + kTileA, BM);
    stage_operand(g.B, g.ldb, !g.b_nmaj, n0, g.N, k0, k_end, base + 2 * kTileA, base + 2 * kTileA + kTileB, BN);
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy stores -> tensor-core reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const std::uint32_t a_hi = smem_u32(base), a_lo = a_hi + kTileA;
      const std::uint32_t b_hi = a_hi + 2 * kTileA, b_lo = b_hi + kTileB;
#pragma unroll
      for (int s = 0; s < BK / 8; ++s) {   // K = 8 per tf32 MMA = 2 core matrices
        const std::uint32_t ka = s * 2 * (BM * 16), kb = s * 2 * (BN * 16);
        const std::uint64_t dAh = umma_desc(a_hi + ka, BM * 16, 128), dAl = umma_desc(a_lo + ka, BM * 16, 128);
        const std::uint64_t dBh = umma_desc(b_hi + kb, BN * 16, 128), dBl = umma_desc(b_lo + kb, BN * 16, 128);
        mma_tf32(tmem, dAl, dBh, idesc, (t | s) != 0 ? 1u : 0u);
        mma_tf32(tmem, dAh, dBl, idesc, 1u);
        mma_tf32(tmem, dAh, dBh, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar[st])));
    }
  }
  if (T > 0) mbar_wait(smem_u32(&mbar[(T - 1) & 1]), ((T - 1) >> 1) & 1);  // MMAs retire in issue order
  asm volatile("tcgen05.fence::after_thread_sync;");

  // ---- epilogue: TMEM lane (32 warp + lane) = output row ----
  const std::uint32_t m = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    std::uint32_t r[16];
    const std::uint32_t taddr = tmem + (static_cast<std::uint32_t>(warp * 32) << 16) + c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const std::uint32_t n = n0 + c + j;
      if (n >= g.N) continue;
      const float acc = T > 0 ? __uint_as_float(r[j]) : 0.f;
      if (g.epi == kEpiBiasAct) {
        const float z = (g.bias ? g.bias[m] : 0.f) + acc;
        g.C[std::size_t(m) * g.ldc + n] = z;
        if (g.act) g.C2[std::size_t(m) * g.ldc + n] = act_fwd<float>(g.act, z);
      } else if (g.epi == kEpiAccum) {
        float* p = &g.C[std::size_t(m) * g.ldc + n];
        *p = g.beta ? *p + acc : acc;
      } else {
        g.C[(std::size_t(blockIdx.z) * g.M + m) * g.N + n] = acc;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

}  // namespace

cudaError_t launch_gemm_umma(const GemmArgs<float>& g, std::uint32_t splits, cudaStream_t st) {
  if (g.M == 0 || g.N == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_umma_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.epi == kEpiSplitK ? splits : 1);
  k_umma_tf32x3<<<grid, 128, kSmem, st>>>(g);
  return cudaGetLastError();
}

}  // namespace tgk
