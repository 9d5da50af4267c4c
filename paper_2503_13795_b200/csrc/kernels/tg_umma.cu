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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "tg_ops.cuh"
#include "tg_devcache.cuh"
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
        if (!(g.no_z && g.act)) g.C[std::size_t(m) * g.ldc + n] = z;
        if (g.act) g.C2[std::size_t(m) * g.ldc + n] = act_fwd<float>(g.act, z);
      } else if (g.epi == kEpiAccum) {
        float* p = &g.C[std::size_t(m) * g.ldc + n];
        if (g.dact) *p = act_bwd_h<float>(g.dact, acc, g.C2[std::size_t(m) * g.ldc + n]);
        else *p = g.beta ? *p + acc : acc;
      } else {
        g.C[(std::size_t(blockIdx.z) * g.M + m) * g.N + n] = acc;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}


// ---------------------------------------------------------------------------
// TMA-fed, warp-specialised variant (k_umma_tma).
//
// Operand tiles travel HBM -> shared memory by TMA (cp.async.bulk.tensor,
// SWIZZLE_128B) straight into the canonical UMMA layouts, whichever way the
// operand is stored:
//   K-major  (k contiguous):  one box {32 k, 128 rows}: rows of 128 B,
//            8-row swizzle atoms (SBO = 1024 B); a K = 8 step advances the
//            descriptor start address by 32 B inside the atom;
//   MN-major (m/n contiguous): four boxes {32 mn, 32 k} (4 KB each, LBO =
//            4 KB between them, SBO = 1024 B); a K = 8 step is +1024 B.
// The 3xTF32 split is elementwise and therefore layout-agnostic: converter
// warps round each landed fp32 tile in place to hi = tf32_rna(x) and write
// lo = x - hi at the same offset of a parallel buffer.
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (one
// lane), warps 2..5 converters and, after the K loop, the TMEM epilogue
// (warp w reads TMEM lanes 32 (w % 4) ..).  A 3-stage ring of mbarriers:
// full (TMA bytes landed) -> conv (128 converter threads done) -> empty
// (tcgen05.commit: the MMAs that read the stage retired).
constexpr int kTStagesMax = 3;
constexpr std::uint32_t kTTile = BM * BK * 4;                   // 16 KB: one operand tile
constexpr std::uint32_t kTStage = 4 * kTTile;                   // A hi, A lo, B hi, B lo
// dynamic shared memory of a STAGES-deep ring (at least the staged-epilogue tile)
__host__ __device__ constexpr std::uint32_t tma_smem(int stages) {
  return (stages * kTStage > BM * (BN + 4) * 4 ? stages * kTStage : BM * (BN + 4) * 4) + 1024 + 512;
}

struct TmaOperand {
  bool mn;   // MN-major (m / n contiguous) vs K-major
};

__device__ __forceinline__ void mbar_init(std::uint32_t mbar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(std::uint32_t mbar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(mbar));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint32_t mbar, std::uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(mbar), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait2(std::uint32_t mbar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TG_WAIT2:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TG_DONE2;\n\t"
      "bra TG_WAIT2;\n"
      "TG_DONE2:\n\t}\n" ::"r"(mbar),
      "r"(parity));
}
__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const CUtensorMap* map, int c0, int c1, std::uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
// SWIZZLE_128B smem descriptor (sm_100 version 1).
__device__ __forceinline__ std::uint64_t umma_desc_sw128(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<std::uint64_t>(lbo >> 4) << 16) |
         (static_cast<std::uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Issue the TMA loads of one operand's k-tile (rows r0.., k0..) into dst.
// `off` shifts the map's outer (row) coordinate: the k rows of an MN-major
// operand, the m / n rows of a K-major one (batched products).
__device__ __forceinline__ void tma_operand(const CUtensorMap* map, bool mn, std::uint32_t dst, int r0, int k0, int off,
                                            std::uint32_t mbar) {
  if (mn) {
#pragma unroll
    for (int c = 0; c < 4; ++c) tma_load_2d(dst + c * 4096, map, r0 + 32 * c, k0 + off, mbar);
  } else {
    tma_load_2d(dst, map, k0, r0 + off, mbar);
  }
}
// MN-major 32-bit operands: the only UMMA layout is SWIZZLE_128B_BASE32B
// (layout type 1; Swizzle<2,5,2>: 32-byte granules XOR row % 4, 4-row atoms of
// 512 B), written by TMA's SWIZZLE_128B_ATOM_32B mode.  LBO = 4 KB between the
// 32-wide MN chunks, SBO = 512 B between 4-row K groups.
__device__ __forceinline__ std::uint64_t umma_desc_b32(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<std::uint64_t>(lbo >> 4) << 16) |
         (static_cast<std::uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (1ull << 61);
}
__device__ __forceinline__ std::uint64_t operand_desc(std::uint32_t base, bool mn, int ks) {
  if (!mn) return umma_desc_sw128(base + ks * 32, 16, 1024);
  return umma_desc_b32(base + ks * 1024, 4096, 512);
}

// Accumulation.  tcgen05's fp32 accumulation is biased (measured: mean
// relative error -1.1e-8 x K on positive data, 1.4e-5 normwise at K = 2048),
// so no TMEM accumulator sums more than kFlush k-tiles (12 x kFlush MMAs):
// the issuer alternates between two TMEM buffers, and the converter warps
// drain each finished buffer into fp32 round-to-nearest register sums (one
// output row per thread) while the tensor core fills the other one.
constexpr int kFlush = 4;   // K 128 per TMEM accumulation window (as the CTA pairs, r07g)
// float4 epilogue stores need 16-byte aligned C / C2 bases (tg_gemm accepts any
// device pointer: a view offset by one float must take the scalar stores)
__device__ __forceinline__ bool c_aligned16(const GemmArgs<float>& g) {
  return ((reinterpret_cast<std::uintptr_t>(g.C) | reinterpret_cast<std::uintptr_t>(g.C2)) & 15u) == 0;
}
#ifdef TG_PROFILING
__device__ int g_umma_exp = 0;   // TG_UMMA_EXP (profiling build only) ablations (wrong results): 1 skip conversion, 2 one MMA per k-step, 3 TMA ring
                                 // only, 4 one MMA on the raw fp32 tiles (how kind::tf32 reads fp32 bits)
#else
constexpr int g_umma_exp = 0;    // product build: no setting can make a kernel skip work
#endif
constexpr int kConvThreads = 256;                 // 8 converter / drain warps
constexpr int kTThreads = 64 + kConvThreads;      // + TMA producer + MMA issuer

template <int kTStages>
__global__ void __launch_bounds__(kTThreads, 1) k_umma_tma(GemmArgs<float> g, const __grid_constant__ CUtensorMap tmA,
                                                     const __grid_constant__ CUtensorMap tmB, int a_mn, int b_mn) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzle atoms, by pointer arithmetic on the
  // shared array (an integer round trip would turn every converter access
  // into a generic LD/ST instead of LDS/STS)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // barriers after the ring (or after the epilogue tile, whichever is larger)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + tma_smem(kTStages) - 1024 - 512);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 3 * kTStages + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto conv = [&](int s) { return smem_u32(&bars[kTStages + s]); };
  auto empty = [&](int s) { return smem_u32(&bars[2 * kTStages + s]); };
  auto tfull = [&](int b) { return smem_u32(&bars[3 * kTStages + b]); };
  auto tempty = [&](int b) { return smem_u32(&bars[3 * kTStages + 2 + b]); };

  if (tid == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(conv(s), kConvThreads);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), kConvThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const std::uint32_t tmem = *tmem_slot;

  // M tiles are the fast grid index: the CTAs that read the same B tile (the
  // sample-axis operand, too large for L2) run together and share it in L2
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  std::uint32_t slice = blockIdx.z;
  int a_off = 0, b_off = 0;
  std::size_t c_off = 0, c2_off = 0;
  if (g.mem) {   // batch member blockIdx.z / zs
    const uint4 e = g.mem[blockIdx.z / g.zs];
    slice = blockIdx.z % g.zs;
    a_off = static_cast<int>(e.x);
    b_off = static_cast<int>(e.y);
    c_off = e.z;
    c2_off = e.w;
  }
  std::uint32_t k_begin = 0, k_end = g.K;
  if (g.epi == kEpiSplitK) {
    k_begin = slice * g.k_chunk;
    k_end = min(g.K, k_begin + g.k_chunk);
  }
  const std::uint32_t T = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
  const std::uint32_t NG = (T + kFlush - 1) / kFlush;   // accumulation groups

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0)
      for (std::uint32_t t = 0; t < T; ++t) {
        const int s = t % kTStages;
        if (t >= kTStages) mbar_wait2(empty(s), ((t / kTStages) - 1) & 1);
        const std::uint32_t base = smem_u32(smem + s * kTStage);
        mbar_expect_tx(full(s), 2 * kTTile);
        const int k0 = static_cast<int>(k_begin + t * BK);
        tma_operand(&tmA, a_mn, base, m0, k0, a_off, full(s));
        tma_operand(&tmB, b_mn, base + 2 * kTTile, n0, k0, b_off, full(s));
      }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    // kind::tf32: D F32 (bit 4), A/B TF32 (bits 7, 10), majors (bits 15, 16), N >> 3 at 17, M >> 4 at 24
    const std::uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (std::uint32_t(a_mn) << 15) |
                                (std::uint32_t(b_mn) << 16) | ((BN >> 3) << 17) | ((BM >> 4) << 24);
    for (std::uint32_t t = 0; t < T; ++t) {
      const int s = t % kTStages;
      const std::uint32_t grp = t / kFlush;
      const int buf = grp & 1;
      if (t % kFlush == 0 && grp >= 2) mbar_wait2(tempty(buf), ((grp >> 1) - 1) & 1);   // buffer drained
      mbar_wait2(conv(s), (t / kTStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const std::uint32_t a_hi = smem_u32(smem + s * kTStage), a_lo = a_hi + kTTile;
        const std::uint32_t b_hi = a_hi + 2 * kTTile, b_lo = a_hi + 3 * kTTile;
        const std::uint32_t td = tmem + buf * BN;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const std::uint64_t dAh = operand_desc(a_hi, a_mn, ks), dAl = operand_desc(a_lo, a_mn, ks);
          const std::uint64_t dBh = operand_desc(b_hi, b_mn, ks), dBl = operand_desc(b_lo, b_mn, ks);
          if (g_umma_exp == 3) continue;   // no MMAs at all: the TMA ring alone
          if (g_umma_exp == 2 || g_umma_exp == 4) {
            mma_tf32(td, dAh, dBh, idesc, (t % kFlush != 0 || ks != 0) ? 1u : 0u);
            continue;
          }
          mma_tf32(td, dAl, dBh, idesc, (t % kFlush != 0 || ks != 0) ? 1u : 0u);
          mma_tf32(td, dAh, dBl, idesc, 1u);
          mma_tf32(td, dAh, dBh, idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty(s)));
        if (t % kFlush == kFlush - 1 || t == T - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tfull(buf)));
      }
      __syncwarp();
    }
  } else {
    // ===== converters (hi = tf32_rna(x) in place, lo = x - hi) + accumulation drain =====
    // 8 warps, two per SMSP; for the drain, warps w and w + 4 share TMEM lane
    // quarter w % 4 (32 rows) and take column halves [0, 64) / [64, 128)
    const int ct = tid - 64;                    // 0..255
    const int wq = warp & 3;                    // TMEM lane quarter
    const int c0 = ((warp - 2) >> 2) * (BN / 2);  // column half
    constexpr int kCols = BN / 2;
    float acc[kCols];
#pragma unroll
    for (int j = 0; j < kCols; ++j) acc[j] = 0.f;
    auto drain = [&](std::uint32_t grp) {
      const int buf = grp & 1;
      mbar_wait2(tfull(buf), (grp >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c = 0; c < kCols; c += 16) {
        std::uint32_t r[16];
        const std::uint32_t taddr = tmem + buf * BN + (static_cast<std::uint32_t>(wq * 32) << 16) + c0 + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(tempty(buf));
    };
    for (std::uint32_t t = 0; t < T; ++t) {
      const int s = t % kTStages;
      mbar_wait2(full(s), (t / kTStages) & 1);
      unsigned char* base = smem + s * kTStage;
      const int nop = (g_umma_exp == 1 || g_umma_exp == 3 || g_umma_exp == 4) ? 0 : 2;
#pragma unroll
      for (int op = 0; op < nop; ++op) {
        float4* hi = reinterpret_cast<float4*>(base + op * 2 * kTTile);
        float4* lo = reinterpret_cast<float4*>(base + op * 2 * kTTile + kTTile);
#pragma unroll 4
        for (int i = ct; i < static_cast<int>(kTTile / 16); i += kConvThreads) {
          const float4 x = hi[i];
          float4 h, l;
          h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
          h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
          h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
          h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
          hi[i] = h;
          lo[i] = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy stores -> tensor-core reads
      mbar_arrive(conv(s));
      // drain two groups back: its MMAs retired before the previous group's
      // began, so the converters never wait on the tensor core here (draining
      // the previous group stalled the next conversion until those MMAs were
      // done, a bubble in front of every group's MMAs)
      if (t % kFlush == 0 && t / kFlush >= 2) drain(t / kFlush - 2);
    }
    for (std::uint32_t q = NG >= 2 ? NG - 2 : 0; q < NG; ++q) drain(q);
    // ===== epilogue: through shared memory, then whole 512-byte rows per warp =====
    // (one row per thread straight to global made every store touch 32 rows:
    // ~14 us of fixed cost per CTA, measured by scripts/gemm_ksweep.py)
    constexpr int kLd = BN + 4;   // row stride in floats: 16-byte aligned, conflict-free float4 stores
    float* tile = reinterpret_cast<float*>(smem);   // the pipeline stages are idle now
    asm volatile("bar.sync 1, %0;" ::"n"(kConvThreads));   // every stage consumed, every drain done
    {
      const int r = wq * 32 + lane;
#pragma unroll
      for (int j = 0; j < kCols; j += 4)
        *reinterpret_cast<float4*>(tile + r * kLd + c0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConvThreads));
    const int cw = (tid - 64) >> 5;   // converter warp 0..7
    const std::uint32_t n = n0 + 4 * lane;
    const bool vec = (g.ldc % 4 == 0) && (g.epi != kEpiSplitK || g.N % 4 == 0) && c_aligned16(g);
    for (int r = cw; r < BM && g_umma_exp != 5; r += kConvThreads / 32) {   // (ablation 5: no output stores)
      const std::uint32_t m = m0 + r;
      if (m >= g.M || n >= g.N) continue;
      const float4 v = *reinterpret_cast<const float4*>(tile + r * kLd + 4 * lane);
      float a4[4] = {v.x, v.y, v.z, v.w};
      float* dst = g.epi == kEpiSplitK ? g.C + (std::size_t(blockIdx.z) * g.M + m) * g.N + n
                                       : g.C + (c_off + m) * g.ldc + n;
      const int cnt = min(4u, g.N - n);
      if (g.epi == kEpiBiasAct) {
        const float bv = g.bias ? g.bias[m] : 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) a4[e] += bv;
        if (g.act) {
          float h4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) h4[e] = act_fwd<float>(g.act, a4[e]);
          float* d2 = g.C2 + (c2_off + m) * g.ldc + n;
          if (vec && cnt == 4) *reinterpret_cast<float4*>(d2) = make_float4(h4[0], h4[1], h4[2], h4[3]);
          else for (int e = 0; e < cnt; ++e) d2[e] = h4[e];
        }
      } else if (g.epi == kEpiAccum && g.dact) {
        const float* hp = g.C2 + (c2_off + m) * g.ldc + n;
        float h4[4] = {0.f, 0.f, 0.f, 0.f};
        if (vec && cnt == 4) {
          const float4 o = *reinterpret_cast<const float4*>(hp);
          h4[0] = o.x; h4[1] = o.y; h4[2] = o.z; h4[3] = o.w;
        } else {
          for (int e = 0; e < cnt; ++e) h4[e] = hp[e];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) a4[e] = act_bwd_h<float>(g.dact, a4[e], h4[e]);
      } else if (g.epi == kEpiAccum && g.beta) {
        if (vec && cnt == 4) {
          const float4 o = *reinterpret_cast<const float4*>(dst);
          a4[0] += o.x; a4[1] += o.y; a4[2] += o.z; a4[3] += o.w;
        } else {
          for (int e = 0; e < cnt; ++e) a4[e] += dst[e];
        }
      }
      if (g.no_z && g.act && g.epi == kEpiBiasAct) continue;   // z has no reader
      if (vec && cnt == 4) *reinterpret_cast<float4*>(dst) = make_float4(a4[0], a4[1], a4[2], a4[3]);
      else for (int e = 0; e < cnt; ++e) dst[e] = a4[e];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

// ---------------------------------------------------------------------------
// Persistent variant (k_umma_tma_p) for short reductions.  With K <= 256 a
// 128 x 128 tile is 2-8 k-tiles: measured on cfg4's shapes, a CTA spent
// ~6 us per tile of which the MMAs were well under one (prologue, first TMA
// round trip, drain, epilogue; ablations in scripts/gemm_bench.py).  Here a
// CTA per SM walks tiles L = blockIdx.x, + gridDim.x, ... (M fastest, then
// N, then the z slice / batch member); the k-tile and accumulation-group
// counters run on across tiles, so the TMA producer prefetches the next
// tile's operands while the converter warps drain and store the current one,
// and the prologue is paid once.  The epilogue tile has its own shared
// memory (two ring stages + epilogue tile).
constexpr int kPStages = 2;
__host__ __device__ constexpr std::uint32_t persist_smem() {
  return kPStages * kTStage + BM * (BN + 4) * 4 + 1024 + 512;
}

__global__ void __launch_bounds__(kTThreads, 1) k_umma_tma_p(GemmArgs<float> g, const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB, int a_mn, int b_mn,
                                                      std::uint32_t mt, std::uint32_t nt, std::uint32_t n_tiles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* etile = reinterpret_cast<float*>(smem + kPStages * kTStage);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + persist_smem() - 1024 - 512);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 3 * kPStages + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto conv = [&](int s) { return smem_u32(&bars[kPStages + s]); };
  auto empty = [&](int s) { return smem_u32(&bars[2 * kPStages + s]); };
  auto tfull = [&](int b) { return smem_u32(&bars[3 * kPStages + b]); };
  auto tempty = [&](int b) { return smem_u32(&bars[3 * kPStages + 2 + b]); };
  if (tid == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(conv(s), kConvThreads);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), kConvThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const std::uint32_t tmem = *tmem_slot;

  struct Tile {
    int m0, n0, a_off, b_off;
    std::size_t c_off, c2_off;
    std::uint32_t z, k_begin, T;
  };
  auto tile_of = [&](std::uint32_t L) {
    Tile t;
    const std::uint32_t mi = L % mt, ni = (L / mt) % nt, z = L / (mt * nt);
    t.m0 = static_cast<int>(mi) * BM;
    t.n0 = static_cast<int>(ni) * BN;
    t.z = z;
    std::uint32_t slice = z;
    t.a_off = t.b_off = 0;
    t.c_off = t.c2_off = 0;
    if (g.mem) {
      const uint4 e = g.mem[z / g.zs];
      slice = z % g.zs;
      t.a_off = static_cast<int>(e.x);
      t.b_off = static_cast<int>(e.y);
      t.c_off = e.z;
      t.c2_off = e.w;
    }
    std::uint32_t k_end = g.K;
    t.k_begin = 0;
    if (g.epi == kEpiSplitK) {
      t.k_begin = slice * g.k_chunk;
      k_end = min(g.K, t.k_begin + g.k_chunk);
    }
    t.T = k_end > t.k_begin ? (k_end - t.k_begin + BK - 1) / BK : 0;
    return t;
  };

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      std::uint32_t gt = 0;
      for (std::uint32_t L = blockIdx.x; L < n_tiles; L += gridDim.x) {
        const Tile tl = tile_of(L);
        for (std::uint32_t t = 0; t < tl.T; ++t, ++gt) {
          const int s = gt % kPStages;
          if (gt >= static_cast<std::uint32_t>(kPStages)) mbar_wait2(empty(s), ((gt / kPStages) - 1) & 1);
          const std::uint32_t base = smem_u32(smem + s * kTStage);
          mbar_expect_tx(full(s), 2 * kTTile);
          const int k0 = static_cast<int>(tl.k_begin + t * BK);
          tma_operand(&tmA, a_mn, base, tl.m0, k0, tl.a_off, full(s));
          tma_operand(&tmB, b_mn, base + 2 * kTTile, tl.n0, k0, tl.b_off, full(s));
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one accumulation group per k-tile) =====
    const std::uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (std::uint32_t(a_mn) << 15) |
                                (std::uint32_t(b_mn) << 16) | ((BN >> 3) << 17) | ((BM >> 4) << 24);
    std::uint32_t gt = 0;
    for (std::uint32_t L = blockIdx.x; L < n_tiles; L += gridDim.x) {
      const Tile tl = tile_of(L);
      for (std::uint32_t t = 0; t < tl.T; ++t, ++gt) {
        const int s = gt % kPStages;
        const int buf = gt & 1;
        if (gt >= 2) mbar_wait2(tempty(buf), ((gt >> 1) - 1) & 1);
        mbar_wait2(conv(s), (gt / kPStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const std::uint32_t a_hi = smem_u32(smem + s * kTStage), a_lo = a_hi + kTTile;
          const std::uint32_t b_hi = a_hi + 2 * kTTile, b_lo = a_hi + 3 * kTTile;
          const std::uint32_t td = tmem + buf * BN;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const std::uint64_t dAh = operand_desc(a_hi, a_mn, ks), dAl = operand_desc(a_lo, a_mn, ks);
            const std::uint64_t dBh = operand_desc(b_hi, b_mn, ks), dBl = operand_desc(b_lo, b_mn, ks);
            mma_tf32(td, dAl, dBh, idesc, ks != 0 ? 1u : 0u);
            mma_tf32(td, dAh, dBl, idesc, 1u);
            mma_tf32(td, dAh, dBh, idesc, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty(s)));
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tfull(buf)));
        }
        __syncwarp();
      }
    }
  } else {
    // ===== converters + drain + epilogue =====
    const int ct = tid - 64;
    const int wq = warp & 3;
    const int c0 = ((warp - 2) >> 2) * (BN / 2);
    constexpr int kCols = BN / 2;
    constexpr int kLd = BN + 4;
    const int cw = (tid - 64) >> 5;
    float acc[kCols];
    auto drain = [&](std::uint32_t grp) {
      const int buf = grp & 1;
      mbar_wait2(tfull(buf), (grp >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c = 0; c < kCols; c += 16) {
        std::uint32_t r[16];
        const std::uint32_t taddr = tmem + buf * BN + (static_cast<std::uint32_t>(wq * 32) << 16) + c0 + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(tempty(buf));
    };
    std::uint32_t gt = 0;
    for (std::uint32_t L = blockIdx.x; L < n_tiles; L += gridDim.x) {
      const Tile tl = tile_of(L);
#pragma unroll
      for (int j = 0; j < kCols; ++j) acc[j] = 0.f;
      for (std::uint32_t t = 0; t < tl.T; ++t, ++gt) {
        const int s = gt % kPStages;
        mbar_wait2(full(s), (gt / kPStages) & 1);
        unsigned char* base = smem + s * kTStage;
#pragma unroll
        for (int op = 0; op < 2; ++op) {
          float4* hi = reinterpret_cast<float4*>(base + op * 2 * kTTile);
          float4* lo = reinterpret_cast<float4*>(base + op * 2 * kTTile + kTTile);
#pragma unroll 4
          for (int i = ct; i < static_cast<int>(kTTile / 16); i += kConvThreads) {
            const float4 x = hi[i];
            float4 h, l;
            h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
            h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
            h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
            h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
            hi[i] = h;
            lo[i] = l;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;");
        mbar_arrive(conv(s));
        if (t > 0) drain(gt - 1);
      }
      if (tl.T > 0) drain(gt - 1);
      // epilogue through the dedicated tile (the previous tile's row stores are done)
      asm volatile("bar.sync 1, %0;" ::"n"(kConvThreads));
      {
        const int r = wq * 32 + lane;
#pragma unroll
        for (int j = 0; j < kCols; j += 4)
          *reinterpret_cast<float4*>(etile + r * kLd + c0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kConvThreads));
      const std::uint32_t n = tl.n0 + 4 * lane;
      const bool vec = (g.ldc % 4 == 0) && (g.epi != kEpiSplitK || g.N % 4 == 0) && c_aligned16(g);
      constexpr int kRS = kConvThreads / 32;   // rows between a warp's consecutive rows
      const int rows = static_cast<std::uint32_t>(tl.m0) < g.M
                           ? static_cast<int>(min(static_cast<std::uint32_t>(BM), g.M - static_cast<std::uint32_t>(tl.m0))) : 0;
      if (vec && g.N % 4 == 0 && !(g.epi == kEpiAccum && (g.dact || g.beta))) {
        // store-only epilogues with 16-byte row segments: one rolled loop with hoisted addressing and kind
        // tests, the next row's bias loaded while this row is stored (as the CTA pairs; the general loop
        // below waits for a global load and re-derives addresses on every one of the warp's 32 rows)
        if (n < g.N) {
          const bool ba = g.epi == kEpiBiasAct, wh = ba && g.act != 0, wz = !(wh && g.no_z);
          const std::size_t rstride = g.epi == kEpiSplitK ? g.N : g.ldc;
          float* d = (g.epi == kEpiSplitK ? g.C + (std::size_t(tl.z) * g.M + tl.m0 + cw) * g.N
                                          : g.C + (tl.c_off + tl.m0 + cw) * g.ldc) + n;
          float* d2 = wh ? g.C2 + (tl.c2_off + tl.m0 + cw) * g.ldc + n : nullptr;
          const float* tp = etile + cw * kLd + 4 * lane;
          const float* bp = (ba && g.bias) ? g.bias + tl.m0 + cw : nullptr;
          float bnext = (bp && cw < rows) ? bp[0] : 0.f;
          for (int r = cw; r < rows; r += kRS, d += kRS * rstride, d2 += kRS * g.ldc, tp += kRS * kLd) {
            const float bv = bnext;
            if (bp && r + kRS < rows) bnext = bp[r + kRS - cw];
            float4 v = *reinterpret_cast<const float4*>(tp);
            v.x += bv; v.y += bv; v.z += bv; v.w += bv;
            if (wh)
              *reinterpret_cast<float4*>(d2) = make_float4(act_fwd<float>(g.act, v.x), act_fwd<float>(g.act, v.y),
                                                           act_fwd<float>(g.act, v.z), act_fwd<float>(g.act, v.w));
            if (wz) *reinterpret_cast<float4*>(d) = v;
          }
        }
      } else if (vec && g.N % 4 == 0 && g.epi == kEpiAccum && g.dact) {
        // input adjoint through act': h of the warp's next eight rows is in flight while eight rows are consumed
        if (n < g.N) {
          constexpr int kCh = 8;
          const float* hrow = g.C2 + (tl.c2_off + tl.m0 + cw) * g.ldc + n;
          float* d = g.C + (tl.c_off + tl.m0 + cw) * g.ldc + n;
          const float* tp = etile + cw * kLd + 4 * lane;
          float4 hn[kCh];
          auto load_h = [&](int r0) {
#pragma unroll
            for (int j = 0; j < kCh; ++j)
              if (r0 + j * kRS < rows) hn[j] = *reinterpret_cast<const float4*>(hrow + std::size_t(r0 + j * kRS - cw) * g.ldc);
          };
          load_h(cw);
          for (int r0 = cw; r0 < rows; r0 += kCh * kRS) {
            float4 h[kCh];
#pragma unroll
            for (int j = 0; j < kCh; ++j) h[j] = hn[j];
            load_h(r0 + kCh * kRS);
#pragma unroll
            for (int j = 0; j < kCh; ++j) {
              const int r = r0 + j * kRS;
              if (r >= rows) break;
              float4 v = *reinterpret_cast<const float4*>(tp + std::size_t(r - cw) * kLd);
              v.x = act_bwd_h<float>(g.dact, v.x, h[j].x);
              v.y = act_bwd_h<float>(g.dact, v.y, h[j].y);
              v.z = act_bwd_h<float>(g.dact, v.z, h[j].z);
              v.w = act_bwd_h<float>(g.dact, v.w, h[j].w);
              *reinterpret_cast<float4*>(d + std::size_t(r - cw) * g.ldc) = v;
            }
          }
        }
      } else
      for (int r = cw; r < BM; r += kConvThreads / 32) {
        const std::uint32_t m = tl.m0 + r;
        if (m >= g.M || n >= g.N) continue;
        const float4 v = *reinterpret_cast<const float4*>(etile + r * kLd + 4 * lane);
        float a4[4] = {v.x, v.y, v.z, v.w};
        float* dst = g.epi == kEpiSplitK ? g.C + (std::size_t(tl.z) * g.M + m) * g.N + n : g.C + (tl.c_off + m) * g.ldc + n;
        const int cnt = min(4u, g.N - n);
        if (g.epi == kEpiBiasAct) {
          const float bv = g.bias ? g.bias[m] : 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) a4[e] += bv;
          if (g.act) {
            float h4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) h4[e] = act_fwd<float>(g.act, a4[e]);
            float* d2 = g.C2 + (tl.c2_off + m) * g.ldc + n;
            if (vec && cnt == 4) *reinterpret_cast<float4*>(d2) = make_float4(h4[0], h4[1], h4[2], h4[3]);
            else for (int e = 0; e < cnt; ++e) d2[e] = h4[e];
          }
        } else if (g.epi == kEpiAccum && g.dact) {
          const float* hp = g.C2 + (tl.c2_off + m) * g.ldc + n;
          float h4[4] = {0.f, 0.f, 0.f, 0.f};
          if (vec && cnt == 4) {
            const float4 o = *reinterpret_cast<const float4*>(hp);
            h4[0] = o.x; h4[1] = o.y; h4[2] = o.z; h4[3] = o.w;
          } else {
            for (int e = 0; e < cnt; ++e) h4[e] = hp[e];
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) a4[e] = act_bwd_h<float>(g.dact, a4[e], h4[e]);
        } else if (g.epi == kEpiAccum && g.beta) {
          if (vec && cnt == 4) {
            const float4 o = *reinterpret_cast<const float4*>(dst);
            a4[0] += o.x; a4[1] += o.y; a4[2] += o.z; a4[3] += o.w;
          } else {
            for (int e = 0; e < cnt; ++e) a4[e] += dst[e];
          }
        }
        if (g.no_z && g.act && g.epi == kEpiBiasAct) continue;   // z has no reader
        if (vec && cnt == 4) *reinterpret_cast<float4*>(dst) = make_float4(a4[0], a4[1], a4[2], a4[3]);
        else for (int e = 0; e < cnt; ++e) dst[e] = a4[e];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

// ---------------------------------------------------------------------------
// CTA-pair variant (k_umma_pair): two CTAs of a (2,1,1) cluster on one TPC run
// one 256 x 256 output tile with tcgen05.mma.cta_group::2 (M = 256, N = 256).
// CTA r holds A rows [128 r, 128 r + 128) and B columns [128 r, 128 r + 128)
// of the pair's tile in its own shared memory (the same per-CTA layout as
// k_umma_tma), and TMEM lanes of its 128 output rows x all 256 columns.
// Per k-tile a CTA lands and converts 32 KB as before but feeds twice the
// MMA work, which halves the L2 -> SM traffic and the shared-memory traffic
// per flop: in k_umma_tma (one CTA, N = 128) the MMAs' own operand reads
// (8 KB per 64-cycle MMA) already fill the 128 B/cycle shared-memory port,
// so TMA writes and the converter's hi/lo pass could only queue behind them.
//
// Roles per CTA are those of k_umma_tma with 16 converter / drain warps (the
// 128 x 256 fp32 running sum is 64 registers per thread); only the leader's
// warp 1 issues MMAs.
// Cross-CTA signalling:
//   full[s]   local: this CTA's TMA bytes landed;
//   conv[s]   leader: one arrive per converter warp of both CTAs (32);
//   empty[s]  both: tcgen05.commit multicast (the MMAs reading stage s retired);
//   tfull[b]  both: commit multicast (accumulator buffer b complete);
//   tempty[b] leader: one arrive per drain warp of both CTAs (32).
// The accumulator is drained every kPFlush k-tiles (TMEM reads per k-tile
// double with N = 256; 4 tiles = K 128 keeps the tensor core's biased fp32
// accumulation at ~9e-7 relative: 1.06e-6 worst over scripts/gemm_shapes_err.py's
// 160 cases; K 64 gave 4.7e-7 at 2.5% less throughput, r07g).
constexpr int kPN = 256;
constexpr int kPFlush = 4;
constexpr int kPConv = 512;                 // 16 converter / drain warps: 64 accumulator columns per thread
constexpr int kPThreads = 64 + kPConv;
__host__ __device__ constexpr std::uint32_t pair_smem(int stages) {
  return (stages * kTStage > BM * (kPN + 4) * 4 ? stages * kTStage : BM * (kPN + 4) * 4) + 1024 + 512;
}

__device__ __forceinline__ std::uint32_t cluster_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of a local shared::cta address in CTA `rank`
__device__ __forceinline__ std::uint32_t peer_addr(std::uint32_t local, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(std::uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq(std::uint32_t mbar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TG_WAITC:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TG_DONEC;\n\t"
      "bra TG_WAITC;\n"
      "TG_DONEC:\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_tf32_pair(std::uint32_t tmem_d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                              std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_pair(std::uint32_t mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(mbar),
      "h"(static_cast<unsigned short>(3)));
}

#ifdef TG_PROFILING
// k-tile timeline of one CTA pair's leader (profiling build only, scripts/pair_trace.py): SM clock stamps of
// 0 TMA issue, 1 `full` seen by converter warp 2, 2 that warp's conv arrive, 3 `conv` seen by the MMA warp,
// 4 MMAs issued + committed, 5 drain of the group two back finished (converter warp 2)
constexpr int kTraceT = 96;
__device__ long long g_pair_trace[7][kTraceT];   // row 6: 0 kernel entry, 1 set-up done, 2 last drain done, 3 tile staged, 4 stores issued, 5 exit
#define TG_TRACE(ev, t)                                                                        \
  do {                                                                                         \
    if (traced && (t) < static_cast<std::uint32_t>(kTraceT)) g_pair_trace[ev][t] = clock64();  \
  } while (0)
#else
#define TG_TRACE(ev, t) do { } while (0)
#endif
template <int kTStages>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    k_umma_pair(GemmArgs<float> g, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int a_mn, int b_mn, int n_tile) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + pair_smem(kTStages) - 1024 - 512);
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 3 * kTStages + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const std::uint32_t rank = cluster_rank();
#ifdef TG_PROFILING
  const bool traced = rank == 0 && lane == 0 && blockIdx.x < 2 && blockIdx.y == gridDim.y / 2 && blockIdx.z == 0;
  if (warp == 2) TG_TRACE(6, 0u);
#endif
  auto full = [&](int s) { return smem_u32(&bars[s]); };
  auto conv = [&](int s) { return smem_u32(&bars[kTStages + s]); };
  auto empty = [&](int s) { return smem_u32(&bars[2 * kTStages + s]); };
  auto tfull = [&](int b) { return smem_u32(&bars[3 * kTStages + b]); };
  auto tempty = [&](int b) { return smem_u32(&bars[3 * kTStages + 2 + b]); };
  constexpr std::uint32_t kArrivals = 2 * (kPConv / 32);   // converter / drain warps of both CTAs

  if (tid == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(conv(s), kArrivals);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), kArrivals);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(2 * kPN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;");
  const std::uint32_t tmem = *tmem_slot;
  if (warp == 2) TG_TRACE(6, 1u);

  const int m0 = static_cast<int>(blockIdx.x >> 1) * (2 * BM) + static_cast<int>(rank) * BM;
  // n_tile <= 256 output columns per pair (a multiple of 16: N spread evenly over its tiles, so a
  // 784-column product runs four tiles of 208 instead of three full ones and one of 16)
  const int n0 = static_cast<int>(blockIdx.y) * n_tile;
  const int nb = n0 + static_cast<int>(rank) * (n_tile >> 1);   // this CTA's B rows (the MMA reads n_tile / 2 of the 128 landed)
  std::uint32_t slice = blockIdx.z;
  int a_off = 0, b_off = 0;
  std::size_t c_off = 0, c2_off = 0;
  if (g.mem) {
    const uint4 e = g.mem[blockIdx.z / g.zs];
    slice = blockIdx.z % g.zs;
    a_off = static_cast<int>(e.x);
    b_off = static_cast<int>(e.y);
    c_off = e.z;
    c2_off = e.w;
  }
  std::uint32_t k_begin = 0, k_end = g.K;
  if (g.epi == kEpiSplitK) {
    k_begin = slice * g.k_chunk;
    k_end = min(g.K, k_begin + g.k_chunk);
  }
  const std::uint32_t T = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
  const std::uint32_t NG = (T + kPFlush - 1) / kPFlush;

  if (warp == 0) {
    // ===== TMA producer (each CTA loads its own A rows and B columns) =====
    if (lane == 0)
      for (std::uint32_t t = 0; t < T; ++t) {
        const int s = t % kTStages;
        if (t >= kTStages) mbar_wait2(empty(s), ((t / kTStages) - 1) & 1);
        const std::uint32_t base = smem_u32(smem + s * kTStage);
        TG_TRACE(0, t);
        mbar_expect_tx(full(s), 2 * kTTile);
        const int k0 = static_cast<int>(k_begin + t * BK);
        tma_operand(&tmA, a_mn, base, m0, k0, a_off, full(s));
        tma_operand(&tmB, b_mn, base + 2 * kTTile, nb, k0, b_off, full(s));
      }
  } else if (warp == 1) {
    // ===== MMA issuer: the leader CTA only =====
    if (rank == 0) {
      const std::uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (std::uint32_t(a_mn) << 15) |
                                  (std::uint32_t(b_mn) << 16) | ((std::uint32_t(n_tile) >> 3) << 17) | (((2 * BM) >> 4) << 24);
      for (std::uint32_t t = 0; t < T; ++t) {
        const int s = t % kTStages;
        const std::uint32_t grp = t / kPFlush;
        const int buf = grp & 1;
        if (t % kPFlush == 0 && grp >= 2) mbar_wait_acq(tempty(buf), ((grp >> 1) - 1) & 1);
        mbar_wait_acq(conv(s), (t / kTStages) & 1);
        TG_TRACE(3, t);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const std::uint32_t a_hi = smem_u32(smem + s * kTStage), a_lo = a_hi + kTTile;
          const std::uint32_t b_hi = a_hi + 2 * kTTile, b_lo = a_hi + 3 * kTTile;
          const std::uint32_t td = tmem + buf * kPN;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const std::uint64_t dAh = operand_desc(a_hi, a_mn, ks), dAl = operand_desc(a_lo, a_mn, ks);
            const std::uint64_t dBh = operand_desc(b_hi, b_mn, ks), dBl = operand_desc(b_lo, b_mn, ks);
            if (g_umma_exp == 3) continue;
            if (g_umma_exp == 2 || g_umma_exp == 4) {
              mma_tf32_pair(td, dAh, dBh, idesc, (t % kPFlush != 0 || ks != 0) ? 1u : 0u);
              continue;
            }
            mma_tf32_pair(td, dAl, dBh, idesc, (t % kPFlush != 0 || ks != 0) ? 1u : 0u);
            mma_tf32_pair(td, dAh, dBl, idesc, 1u);
            mma_tf32_pair(td, dAh, dBh, idesc, 1u);
          }
          commit_pair(empty(s));
          if (t % kPFlush == kPFlush - 1 || t == T - 1) commit_pair(tfull(buf));
          TG_TRACE(4, t);
        }
        __syncwarp();
      }
    }
  } else {
    // ===== converters + accumulation drain (16 warps: TMEM lane quarter w % 4, column quarter) =====
    const int ct = tid - 64;
    const int wq = warp & 3;
    const int c0 = ((warp - 2) >> 2) * (kPN / 4);
    constexpr int kCols = kPN / 4;
    const std::uint32_t leader_conv0 = peer_addr(conv(0), 0);
    const std::uint32_t leader_tempty0 = peer_addr(tempty(0), 0);
    float acc[kCols];
#pragma unroll
    for (int j = 0; j < kCols; ++j) acc[j] = 0.f;
    // fused bias row sums of a K-major A (weight-gradient products, g.rowsum):
    // thread ct holds A rows ct / 8 and ct / 8 + 64 of every k-tile (one
    // 16-byte chunk of each: row r is float4s [8r, 8r + 8) whatever the
    // swizzle); the N-tile-0 CTAs of each split sum them in k order
    const bool rs_on = g.rowsum && !a_mn && blockIdx.y == 0;
    float rs[static_cast<int>(kTTile / 16) / kPConv] = {};
    auto drain = [&](std::uint32_t grp) {
      const int buf = grp & 1;
      mbar_wait2(tfull(buf), (grp >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int c = 0; c < kCols; c += 16) {
        std::uint32_t r[16];
        const std::uint32_t taddr = tmem + buf * kPN + (static_cast<std::uint32_t>(wq * 32) << 16) + c0 + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_tempty0 + buf * 8);
    };
    for (std::uint32_t t = 0; t < T; ++t) {
      const int s = t % kTStages;
      mbar_wait2(full(s), (t / kTStages) & 1);
      if (warp == 2) TG_TRACE(1, t);
      unsigned char* base = smem + s * kTStage;
      const int nop = (g_umma_exp == 1 || g_umma_exp == 3 || g_umma_exp == 4) ? 0 : 2;
#pragma unroll
      for (int op = 0; op < nop; ++op) {
        float4* hi = reinterpret_cast<float4*>(base + op * 2 * kTTile);
        float4* lo = reinterpret_cast<float4*>(base + op * 2 * kTTile + kTTile);
#pragma unroll
        for (int it = 0; it < static_cast<int>(kTTile / 16) / kPConv; ++it) {
          const int i = ct + it * kPConv;
          const float4 x = hi[i];
          if (op == 0 && rs_on) rs[it] += (x.x + x.y) + (x.z + x.w);   // A row (i / 8), four consecutive k
          float4 h, l;
          h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
          h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
          h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
          h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
          hi[i] = h;
          lo[i] = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy stores -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_conv0 + s * 8);
      if (warp == 2) TG_TRACE(2, t);
      // two groups back (see k_umma_tma): no converter stall on the tensor core
      if (t % kPFlush == 0 && t / kPFlush >= 2) {
        drain(t / kPFlush - 2);
        if (warp == 2) TG_TRACE(5, t);
      }
    }
    for (std::uint32_t q = NG >= 2 ? NG - 2 : 0; q < NG; ++q) drain(q);
    if (warp == 2) TG_TRACE(6, 2u);
    if (rs_on) {   // eight threads per row (consecutive lanes): fixed-order tree, one store per row
#pragma unroll
      for (int it = 0; it < static_cast<int>(kTTile / 16) / kPConv; ++it) {
        float v = rs[it];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        const std::uint32_t m = static_cast<std::uint32_t>(m0 + (ct + it * kPConv) / 8);
        if ((ct & 7) == 0 && m < g.M) g.rowsum[std::size_t(blockIdx.z) * g.M + m] = v;
      }
    }
    // ===== epilogue: this CTA's 128 rows x 256 columns through shared memory =====
    constexpr int kLd = kPN + 4;
    float* tile = reinterpret_cast<float*>(smem);
    asm volatile("bar.sync 1, %0;" ::"n"(kPConv));
    {
      const int r = wq * 32 + lane;
#pragma unroll
      for (int j = 0; j < kCols; j += 4)
        *reinterpret_cast<float4*>(tile + r * kLd + c0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kPConv));
    if (warp == 2) TG_TRACE(6, 3u);
    const int cw = (tid - 64) >> 5;
    const bool vec = (g.ldc % 4 == 0) && (g.epi != kEpiSplitK || g.N % 4 == 0) && c_aligned16(g);
    if (g.epi == kEpiAccum && g.dact && vec && g.N % 4 == 0) {
      // input adjoint through act': the 16 h segments of this warp's rows are all in
      // flight before the first is consumed (the running sums are dead by now, so the
      // registers are there); the general loop below waits for one row's h at a time
      float4 hp[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = (i & 1) * 128 + 4 * lane;
        const std::uint32_t m = static_cast<std::uint32_t>(m0 + cw + (i >> 1) * (kPConv / 32));
        const std::uint32_t n = static_cast<std::uint32_t>(n0 + col);
        if (m < g.M && n < g.N && col < n_tile) hp[i] = *reinterpret_cast<const float4*>(g.C2 + (c2_off + m) * g.ldc + n);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = cw + (i >> 1) * (kPConv / 32), col = (i & 1) * 128 + 4 * lane;
        const std::uint32_t m = static_cast<std::uint32_t>(m0 + r), n = static_cast<std::uint32_t>(n0 + col);
        if (m >= g.M || n >= g.N || col >= n_tile) continue;
        float4 v = *reinterpret_cast<const float4*>(tile + r * kLd + col);
        v.x = act_bwd_h<float>(g.dact, v.x, hp[i].x);
        v.y = act_bwd_h<float>(g.dact, v.y, hp[i].y);
        v.z = act_bwd_h<float>(g.dact, v.z, hp[i].z);
        v.w = act_bwd_h<float>(g.dact, v.w, hp[i].w);
        *reinterpret_cast<float4*>(g.C + (c_off + m) * g.ldc + n) = v;
      }
    } else if (vec && g.N % 4 == 0 && !(g.epi == kEpiAccum && (g.dact || g.beta))) {
      // store-only epilogues (forward bias / activation, plain products, split-K partials) with 16-byte row
      // segments: one rolled loop over the warp's 8 rows whose pointers advance by a fixed stride and whose
      // kind tests are hoisted (the general loop below re-derives addresses and kinds per segment, and a
      // tile's store phase was bound by issuing those instructions: 2.7 us for 128 KB, profiles/r08/trace)
      const int col = 4 * lane;
      const bool in0 = static_cast<std::uint32_t>(n0 + col) < g.N && col < n_tile;
      const bool in1 = static_cast<std::uint32_t>(n0 + 128 + col) < g.N && 128 + col < n_tile;
      const bool ba = g.epi == kEpiBiasAct, wh = ba && g.act != 0, wz = !(wh && g.no_z);
      const std::size_t rstride = g.epi == kEpiSplitK ? g.N : g.ldc;
      float* d = (g.epi == kEpiSplitK ? g.C + (std::size_t(blockIdx.z) * g.M + m0 + cw) * g.N
                                      : g.C + (c_off + m0 + cw) * g.ldc) + n0 + col;
      float* d2 = wh ? g.C2 + (c2_off + m0 + cw) * g.ldc + n0 + col : nullptr;
      const float* tp = tile + cw * kLd + col;
      const float* bp = (ba && g.bias) ? g.bias + m0 + cw : nullptr;
      const int rows = static_cast<std::uint32_t>(m0) < g.M ? static_cast<int>(min(static_cast<std::uint32_t>(BM), g.M - static_cast<std::uint32_t>(m0))) : 0;   // (the pair's second CTA may lie wholly past M)
      float bnext = (bp && cw < rows) ? bp[0] : 0.f;   // the next row's bias is loaded while this row is stored
      for (int r = cw; r < rows; r += kPConv / 32, d += (kPConv / 32) * rstride, d2 += (kPConv / 32) * g.ldc,
               tp += (kPConv / 32) * kLd) {
        const float bv = bnext;
        if (bp && r + kPConv / 32 < rows) bnext = bp[r + kPConv / 32 - cw];
        float4 v0 = *reinterpret_cast<const float4*>(tp), v1 = *reinterpret_cast<const float4*>(tp + 128);
        v0.x += bv; v0.y += bv; v0.z += bv; v0.w += bv;
        v1.x += bv; v1.y += bv; v1.z += bv; v1.w += bv;
        if (wh) {
          if (in0)
            *reinterpret_cast<float4*>(d2) = make_float4(act_fwd<float>(g.act, v0.x), act_fwd<float>(g.act, v0.y),
                                                         act_fwd<float>(g.act, v0.z), act_fwd<float>(g.act, v0.w));
          if (in1)
            *reinterpret_cast<float4*>(d2 + 128) = make_float4(act_fwd<float>(g.act, v1.x), act_fwd<float>(g.act, v1.y),
                                                               act_fwd<float>(g.act, v1.z), act_fwd<float>(g.act, v1.w));
        }
        if (wz) {
          if (in0) *reinterpret_cast<float4*>(d) = v0;
          if (in1) *reinterpret_cast<float4*>(d + 128) = v1;
        }
      }
    } else
    for (int r = cw; r < BM; r += kPConv / 32) {
      const std::uint32_t m = static_cast<std::uint32_t>(m0 + r);
      if (m >= g.M) continue;
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const std::uint32_t n = static_cast<std::uint32_t>(n0 + hlf * 128) + 4 * lane;
        if (n >= g.N || hlf * 128 + 4 * lane >= n_tile) continue;
        const float4 v = *reinterpret_cast<const float4*>(tile + r * kLd + hlf * 128 + 4 * lane);
        float a4[4] = {v.x, v.y, v.z, v.w};
        float* dst = g.epi == kEpiSplitK ? g.C + (std::size_t(blockIdx.z) * g.M + m) * g.N + n
                                         : g.C + (c_off + m) * g.ldc + n;
        const int cnt = min(4u, g.N - n);
        if (g.epi == kEpiBiasAct) {
          const float bv = g.bias ? g.bias[m] : 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) a4[e] += bv;
          if (g.act) {
            float h4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) h4[e] = act_fwd<float>(g.act, a4[e]);
            float* d2 = g.C2 + (c2_off + m) * g.ldc + n;
            if (vec && cnt == 4) *reinterpret_cast<float4*>(d2) = make_float4(h4[0], h4[1], h4[2], h4[3]);
            else for (int e = 0; e < cnt; ++e) d2[e] = h4[e];
          }
        } else if (g.epi == kEpiAccum && g.dact) {
          const float* hp = g.C2 + (c2_off + m) * g.ldc + n;
          float h4[4] = {0.f, 0.f, 0.f, 0.f};
          if (vec && cnt == 4) {
            const float4 o = *reinterpret_cast<const float4*>(hp);
            h4[0] = o.x; h4[1] = o.y; h4[2] = o.z; h4[3] = o.w;
          } else {
            for (int e = 0; e < cnt; ++e) h4[e] = hp[e];
          }
  #pragma unroll
          for (int e = 0; e < 4; ++e) a4[e] = act_bwd_h<float>(g.dact, a4[e], h4[e]);
        } else if (g.epi == kEpiAccum && g.beta) {
          if (vec && cnt == 4) {
            const float4 o = *reinterpret_cast<const float4*>(dst);
            a4[0] += o.x; a4[1] += o.y; a4[2] += o.z; a4[3] += o.w;
          } else {
            for (int e = 0; e < cnt; ++e) a4[e] += dst[e];
          }
        }
        if (g.no_z && g.act && g.epi == kEpiBiasAct) continue;   // z has no reader
        if (vec && cnt == 4) *reinterpret_cast<float4*>(dst) = make_float4(a4[0], a4[1], a4[2], a4[3]);
        else for (int e = 0; e < cnt; ++e) dst[e] = a4[e];
      }
    }
  }
  if (warp == 2) TG_TRACE(6, 4u);
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();   // no CTA leaves while its peer may still signal its barriers or read its tiles
  if (warp == 2) TG_TRACE(6, 5u);
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * kPN));
}

// Host: 2D tensor map of an operand view for TMA (SWIZZLE_128B, zero OOB fill).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time lookup
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
    return f;
  }();
  return fn;
}

// rows x k operand; mn: element (r, k) at P[k * ld + r], else at P[r * ld + k]
bool make_operand_map(CUtensorMap* map, const float* P, std::size_t ld, bool mn, std::uint32_t rows, std::uint32_t K) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  if ((reinterpret_cast<std::uintptr_t>(P) & 15) || ((ld * 4) & 15) || ld * 4 >= (1ull << 40)) return false;
  cuuint64_t dims[2], strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (mn) {
    dims[0] = rows; dims[1] = K;
    box[0] = 32; box[1] = 32;
  } else {
    dims[0] = K; dims[1] = rows;
    box[0] = 32; box[1] = BM;
  }
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(P), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// CTA pairs for products with more than one 128-row M tile (TG_UMMA_PAIR=0: single CTAs)
bool use_pair(std::uint32_t M) {
  static const bool on = !(std::getenv("TG_UMMA_PAIR") && std::getenv("TG_UMMA_PAIR")[0] == '0');
  return on && M > static_cast<std::uint32_t>(BM);
}

cudaError_t launch_tma_kernel(const GemmArgs<float>& g, std::uint32_t z, const CUtensorMap& ta, const CUtensorMap& tb,
                              bool a_mn, bool b_mn, cudaStream_t st) {
  static PerDeviceOnce attr;
  if (const cudaError_t e0 = attr.ensure([] {
        for (cudaError_t e : {cudaFuncSetAttribute(k_umma_tma<kTStagesMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(tma_smem(kTStagesMax))),
                              cudaFuncSetAttribute(k_umma_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(tma_smem(1))),
                              cudaFuncSetAttribute(k_umma_pair<kTStagesMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(pair_smem(kTStagesMax)))})
          if (e != cudaSuccess) return e;
        return cudaSuccess;
      }); e0 != cudaSuccess)
    return e0;
  // (routing short-K products with M > 128 to the persistent single-CTA tiles
  // instead was measured slower end to end: cfg3 1.61 -> 1.83 ms, cfg4 34.6 -> 37.0 ms)
  if (use_pair(g.M) && !g.no_pair) {
    const std::uint32_t nt = (g.N + kPN - 1) / kPN;
    const int n_tile = static_cast<int>(((g.N + nt - 1) / nt + 15) / 16 * 16);
    const dim3 grid(2 * ((g.M + 2 * BM - 1) / (2 * BM)), nt, z);
    k_umma_pair<kTStagesMax><<<grid, kPThreads, pair_smem(kTStagesMax), st>>>(g, ta, tb, a_mn ? 1 : 0, b_mn ? 1 : 0, n_tile);
    return cudaGetLastError();
  }
  static const bool persist = !(std::getenv("TG_UMMA_PERSIST") && std::getenv("TG_UMMA_PERSIST")[0] == '0');
  const std::uint32_t kspan0 = g.epi == kEpiSplitK ? g.k_chunk : g.K;
  if (persist && kspan0 <= 256) {
    static PerDeviceOnce pattr;
    if (const cudaError_t e = pattr.ensure([] {
          return cudaFuncSetAttribute(k_umma_tma_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(persist_smem()));
        }); e != cudaSuccess)
      return e;
    const std::uint32_t mt = (g.M + BM - 1) / BM, nt = (g.N + BN - 1) / BN;
    const std::uint32_t tiles = mt * nt * z;
    const int nsm = sm_count();
    const std::uint32_t grid = std::min<std::uint32_t>(tiles, static_cast<std::uint32_t>(nsm));
    if (grid == 0) return cudaSuccess;
    k_umma_tma_p<<<grid, kTThreads, persist_smem(), st>>>(g, ta, tb, a_mn ? 1 : 0, b_mn ? 1 : 0, mt, nt, tiles);
    return cudaGetLastError();
  }
  const dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN, z);
  // one k-tile per CTA (K <= 32): a 1-stage ring, so two CTAs share an SM
  // and one's TMA / epilogue latency hides behind the other's work
  const std::uint32_t kspan = g.epi == kEpiSplitK ? g.k_chunk : g.K;
  static const std::uint32_t k1max = std::getenv("TG_UMMA_K1") ? std::atoi(std::getenv("TG_UMMA_K1")) : BK;
  if (kspan <= k1max)
    k_umma_tma<1><<<grid, kTThreads, tma_smem(1), st>>>(g, ta, tb, a_mn ? 1 : 0, b_mn ? 1 : 0);
  else
    k_umma_tma<kTStagesMax><<<grid, kTThreads, tma_smem(kTStagesMax), st>>>(g, ta, tb, a_mn ? 1 : 0, b_mn ? 1 : 0);
  return cudaGetLastError();
}
}  // namespace

std::uint32_t umma_ctas_per_slice(std::uint32_t M, std::uint32_t N) {
  if (use_pair(M)) return 2 * ((M + 2 * BM - 1) / (2 * BM)) * ((N + kPN - 1) / kPN);
  return ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
}

// ---------------------------------------------------------------------------
// Short reductions (K <= 32) on the FP32 pipe: k_gemm_shortk.  With one
// k-tile per output tile the tensor-core kernels are bound by their per-tile
// fixed cost (TMA round trip, hi/lo split, TMEM drain, staged epilogue: cfg3's
// 200 x 30 layer ran at 275 us for 210 MB of output).  Here a CTA owns 64
// rows x 256 samples: the A tile sits in shared memory (warp-uniform
// broadcast reads), each thread keeps 4 k-rows of its 4 samples (float4 loads
// straight from HBM, 512 B per warp) in registers and accumulates 16 rows x 4
// samples with FFMA; the epilogue stores whole 512-byte row segments.  fp32
// FMA over K <= 32 is as accurate as the 3xTF32 split (no TF32 rounding).
// The same kernel with one 16-row group and 1024 samples per CTA serves
// skinny forward products (M <= 16: a classifier head) whose tensor-core
// tiles would be 128 rows for 10 real ones (cfg5's 10 x 1024 head: 2.05 ms
// on k_umma_tma).  Routed for forward products only (bias + activation
// epilogue): cfg3's 200 x 30 layer 275 -> 220 us.  Input-adjoint products read h for act' in
// the epilogue and measured slower here than on the CTA pairs (cfg3 dX
// 221 -> 274 us, cfg5's 1024 x 10 dX ~2 -> 3.3 ms, r05d), so they stay there.
constexpr int kSkRows = 16;

// MG row groups of kSkRows rows per CTA (MG = 4: 64 rows x 256 samples, the
// short-K shape; MG = 1: 16 rows x 1024 samples, the skinny-M shape of a
// classifier head such as cfg5's 10 x 1024 layer, whose A tile is 16 x K).
// A lives in dynamic shared memory as [row][kp] (kp = K rounded up to 4, + 4).
template <bool AK, int MG>
__global__ void __launch_bounds__(256, 2) k_gemm_shortk(GemmArgs<float> g, int kp) {
  extern __shared__ __align__(16) float As[];
  constexpr int kTpg = 256 / MG, kMT = MG * kSkRows;
  const int tid = threadIdx.x;
  const std::uint32_t m0 = blockIdx.y * kMT;
  const std::uint32_t k4 = (g.K + 3) & ~3u;
  for (std::uint32_t i = tid; i < kMT * k4; i += 256) {
    std::uint32_t mm, kk;
    if (AK) { mm = i / k4; kk = i % k4; } else { kk = i / kMT; mm = i % kMT; }
    const std::uint32_t gm = m0 + mm;
    float v = 0.f;
    if (gm < g.M && kk < g.K) v = AK ? g.A[std::size_t(gm) * g.lda + kk] : g.A[std::size_t(kk) * g.lda + gm];
    As[mm * kp + kk] = v;
  }
  __syncthreads();
  const int mg = tid / kTpg;
  const std::size_t n = std::size_t(blockIdx.x) * (4 * kTpg) + 4 * (tid % kTpg);
  if (n >= g.N) return;
  const float* Ar = As + mg * kSkRows * kp;
  float acc[kSkRows][4];
#pragma unroll
  for (int r = 0; r < kSkRows; ++r)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[r][e] = 0.f;
  // the next four k-rows' loads are in flight while the current four are consumed
  float4 bn[4];
  auto load_b = [&](std::uint32_t k0) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      bn[kk] = k0 + kk < g.K ? __ldg(reinterpret_cast<const float4*>(g.B + std::size_t(k0 + kk) * g.ldb + n))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  load_b(0);
  for (std::uint32_t k0 = 0; k0 < g.K; k0 += 4) {
    float4 b[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) b[kk] = bn[kk];
    if (k0 + 4 < g.K) load_b(k0 + 4);
#pragma unroll
    for (int r = 0; r < kSkRows; ++r) {
      const float4 a0 = *reinterpret_cast<const float4*>(Ar + r * kp + k0);
      const float av[4] = {a0.x, a0.y, a0.z, a0.w};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        acc[r][0] = fmaf(av[kk], b[kk].x, acc[r][0]);
        acc[r][1] = fmaf(av[kk], b[kk].y, acc[r][1]);
        acc[r][2] = fmaf(av[kk], b[kk].z, acc[r][2]);
        acc[r][3] = fmaf(av[kk], b[kk].w, acc[r][3]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kSkRows; ++r) {
    const std::uint32_t m = m0 + mg * kSkRows + r;
    if (m >= g.M) break;
    float a4[4] = {acc[r][0], acc[r][1], acc[r][2], acc[r][3]};
    float* dst = g.C + std::size_t(m) * g.ldc + n;
    if (g.epi == kEpiBiasAct) {
      const float bv = g.bias ? g.bias[m] : 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) a4[e] += bv;
      if (g.act) {
        float h4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) h4[e] = act_fwd<float>(g.act, a4[e]);
        *reinterpret_cast<float4*>(g.C2 + std::size_t(m) * g.ldc + n) = make_float4(h4[0], h4[1], h4[2], h4[3]);
        if (g.no_z) continue;   // z has no reader
      }
    } else if (g.dact) {
      const float4 o = *reinterpret_cast<const float4*>(g.C2 + std::size_t(m) * g.ldc + n);
      const float h4[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) a4[e] = act_bwd_h<float>(g.dact, a4[e], h4[e]);
    } else if (g.beta) {
      const float4 o = *reinterpret_cast<const float4*>(dst);
      a4[0] += o.x; a4[1] += o.y; a4[2] += o.z; a4[3] += o.w;
    }
    *reinterpret_cast<float4*>(dst) = make_float4(a4[0], a4[1], a4[2], a4[3]);
  }
}

template <bool AK, int MG>
cudaError_t launch_shortk(const GemmArgs<float>& g, cudaStream_t st) {
  const int kp = static_cast<int>(((g.K + 3) & ~3u) + 4);
  const std::size_t smem = std::size_t(MG * kSkRows) * kp * sizeof(float);
  static PerDeviceMax attr;
  if (smem > 48 * 1024)
    if (const cudaError_t e = attr.raise_to(static_cast<int>(smem), [](int v) {
          return cudaFuncSetAttribute(k_gemm_shortk<AK, MG>, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
        }); e != cudaSuccess)
      return e;
  const dim3 grid(static_cast<unsigned>((g.N + 4 * (256 / MG) - 1) / (4 * (256 / MG))), (g.M + MG * kSkRows - 1) / (MG * kSkRows));
  k_gemm_shortk<AK, MG><<<grid, 256, smem, st>>>(g, kp);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Skinny weight gradients on the FP32 pipe: dW = dZ X^T with M <= 16 output
// rows (a classifier head: cfg5's 10 x 1024 weight over 1M samples) is a
// 16x-padded tile on the tensor core (k_umma_tma: 1.73 ms for 20 GFLOP) and
// an HBM stream of X here.  CTA (n-block, split z): 8 warps x 4 rows n of
// B(k, n) = X[n][k] (K-major: every row is contiguous in k), lane l takes k =
// kb + l of each 512-wide sub-chunk whose A(m, k) = dZ[m][k] columns the CTA
// stages in shared memory; per 4 k: 4 coalesced 16-byte row loads, M shared
// loads, 16 M FMAs (M exact: one instantiation per even row count).  Each lane sums its k in order, the warp folds lanes in a fixed tree,
// and the split partials [z][M][N] take the split-K reduce (deterministic).
constexpr int kSwRows = 16, kSwK = 512, kSwWarps = 8, kSwN = 4;
__device__ __forceinline__ void cp_async4_zfill(float* dst, const float* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
template <int MR>
__global__ void __launch_bounds__(256, 2) k_dw_skinny(GemmArgs<float> g) {
  // the dZ chunk of the next 512 k lands (cp.async, zero-filled past M / the
  // split's end) while the current one is consumed: one barrier per chunk and
  // no exposed global round trip in front of it
  extern __shared__ __align__(16) float Ab[];   // [2][MR][kSwK]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t z = blockIdx.y;
  const std::uint32_t k_begin = min(g.K, z * g.k_chunk);
  const std::uint32_t k_end = min(g.K, k_begin + g.k_chunk);
  const std::uint32_t n0 = (blockIdx.x * kSwWarps + warp) * kSwN;
  float acc[kSwN][MR];
#pragma unroll
  for (int j = 0; j < kSwN; ++j)
#pragma unroll
    for (int m = 0; m < MR; ++m) acc[j][m] = 0.f;
  auto stage = [&](int buf, std::uint32_t kb) {
    for (std::uint32_t i = threadIdx.x; i < MR * kSwK; i += 256) {
      const std::uint32_t m = i / kSwK, k = i % kSwK;
      const bool ok = m < g.M && kb + k < k_end;
      cp_async4_zfill(Ab + (std::size_t(buf) * MR + m) * kSwK + k, ok ? g.A + std::size_t(m) * g.lda + kb + k : g.A, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (k_begin < k_end) stage(0, k_begin);
  int buf = 0;
  for (std::uint32_t kb = k_begin; kb < k_end; kb += kSwK, buf ^= 1) {
    const std::uint32_t kn = min(static_cast<std::uint32_t>(kSwK), k_end - kb);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();   // this chunk landed for every thread; the other buffer's readers are done
    if (kb + kSwK < k_end) stage(buf ^ 1, kb + kSwK);
    const float* As = Ab + std::size_t(buf) * MR * kSwK;
    const float* rows[kSwN];
#pragma unroll
    for (int j = 0; j < kSwN; ++j) rows[j] = g.B + std::size_t(min(n0 + j, g.N - 1)) * g.ldb + kb;
    // four consecutive k per lane (16-byte loads: 512 bytes per row per warp in flight)
#pragma unroll 4
    for (std::uint32_t k = 4 * lane; k < kn; k += 128) {
      float4 b[kSwN];
      if (k + 3 < kn) {
#pragma unroll
        for (int j = 0; j < kSwN; ++j) b[j] = __ldg(reinterpret_cast<const float4*>(rows[j] + k));
      } else {
#pragma unroll
        for (int j = 0; j < kSwN; ++j)
          b[j] = make_float4(rows[j][k], k + 1 < kn ? rows[j][k + 1] : 0.f, k + 2 < kn ? rows[j][k + 2] : 0.f, 0.f);
      }
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        const float4 a = *reinterpret_cast<const float4*>(As + m * kSwK + k);
#pragma unroll
        for (int j = 0; j < kSwN; ++j) {
          float t = acc[j][m];
          t = fmaf(a.x, b[j].x, t);
          t = fmaf(a.y, b[j].y, t);
          t = fmaf(a.z, b[j].z, t);
          t = fmaf(a.w, b[j].w, t);
          acc[j][m] = t;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kSwN; ++j)
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      float v = acc[j][m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[j][m] = v;
    }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < kSwN; ++j)
#pragma unroll
      for (int m = 0; m < MR; ++m)
        if (m < static_cast<int>(g.M) && n0 + j < g.N) g.C[(std::size_t(z) * g.M + m) * g.N + n0 + j] = acc[j][m];
}

cudaError_t launch_dw_skinny(const GemmArgs<float>& g0, std::uint32_t splits, cudaStream_t st) {
  // split ranges on sub-chunk boundaries (16-byte aligned loads); trailing splits may be empty (zero partials)
  GemmArgs<float> g = g0;
  g.k_chunk = (g.K + splits - 1) / splits;
  g.k_chunk = (g.k_chunk + kSwK - 1) / kSwK * kSwK;
  const dim3 grid((g.N + kSwWarps * kSwN - 1) / (kSwWarps * kSwN), splits);
  auto go = [&](auto mr) -> cudaError_t {
    constexpr int MR = decltype(mr)::value;
    constexpr int smem = 2 * MR * kSwK * static_cast<int>(sizeof(float));
    if constexpr (smem > 48 * 1024) {
      static PerDeviceOnce attr;
      if (const cudaError_t e = attr.ensure([] {
            return cudaFuncSetAttribute(k_dw_skinny<MR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          }); e != cudaSuccess)
        return e;
    }
    k_dw_skinny<MR><<<grid, 256, smem, st>>>(g);
    return cudaGetLastError();
  };
  switch ((g.M + 1) / 2) {
    case 1: return go(std::integral_constant<int, 2>{});
    case 2: return go(std::integral_constant<int, 4>{});
    case 3: return go(std::integral_constant<int, 6>{});
    case 4: return go(std::integral_constant<int, 8>{});
    case 5: return go(std::integral_constant<int, 10>{});
    case 6: return go(std::integral_constant<int, 12>{});
    case 7: return go(std::integral_constant<int, 14>{});
    default: return go(std::integral_constant<int, 16>{});
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Skinny input adjoints on the FP32 pipe: dX = W^T dZ with K <= 16 (the layer
// below a classifier head: cfg5's 1024 x 1M product over 10 classes) is an
// HBM stream: 4 B written per output, 4 B of h read for act', 20 flop.  On
// the CTA pairs it is one padded k-tile per 256 x 256 tile (3.9 ms for 8.6 GB);
// on k_gemm_shortk each thread's h loads sat one at a time behind its stores
// (3.3 ms, r05d).  Here a thread owns 4 consecutive samples: its K values of
// dZ stay in registers (KR float4), the CTA's 64 x K block of W sits in shared
// memory (warp-uniform broadcast reads), and the rows are walked four at a
// time with the next four rows' h loads in flight before the current four are
// computed and stored, so every warp keeps 2 KB of reads outstanding.
constexpr int kDxRows = 64, kDxChunk = 4;
template <int KR>
__global__ void __launch_bounds__(256, 2) k_dx_skinny(GemmArgs<float> g) {
  __shared__ __align__(16) float As[kDxRows][KR];
  const int tid = threadIdx.x;
  const std::uint32_t m0 = blockIdx.y * kDxRows;
  for (int i = tid; i < kDxRows * KR; i += 256) {
    const std::uint32_t mm = i / KR, kk = i % KR, gm = m0 + mm;
    float v = 0.f;
    if (gm < g.M && kk < g.K) v = g.a_kmaj ? g.A[std::size_t(gm) * g.lda + kk] : g.A[std::size_t(kk) * g.lda + gm];
    As[mm][kk] = v;
  }
  __syncthreads();
  const std::size_t n = (std::size_t(blockIdx.x) * 256 + tid) * 4;
  if (n >= g.N) return;
  float4 b[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k)
    b[k] = k < static_cast<int>(g.K) ? __ldg(reinterpret_cast<const float4*>(g.B + std::size_t(k) * g.ldb + n))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
  const std::uint32_t rows = min(static_cast<std::uint32_t>(kDxRows), g.M - m0);
  const float* hp = g.dact ? g.C2 + std::size_t(m0) * g.ldc + n : nullptr;
  float* cp = g.C + std::size_t(m0) * g.ldc + n;
  float4 hn[kDxChunk];
  auto load_h = [&](std::uint32_t r0) {
#pragma unroll
    for (int j = 0; j < kDxChunk; ++j)
      if (hp && r0 + j < rows) hn[j] = __ldcs(reinterpret_cast<const float4*>(hp + std::size_t(r0 + j) * g.ldc));
  };
  load_h(0);
#pragma unroll 2
  for (std::uint32_t r0 = 0; r0 < rows; r0 += kDxChunk) {
    float4 h[kDxChunk];
#pragma unroll
    for (int j = 0; j < kDxChunk; ++j) h[j] = hn[j];
    load_h(r0 + kDxChunk);
#pragma unroll
    for (int j = 0; j < kDxChunk; ++j) {
      if (r0 + j >= rows) break;
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k4 = 0; k4 < KR; k4 += 4) {
        const float4 a = *reinterpret_cast<const float4*>(&As[r0 + j][k4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          a4[0] = fmaf(av[kk], b[k4 + kk].x, a4[0]);
          a4[1] = fmaf(av[kk], b[k4 + kk].y, a4[1]);
          a4[2] = fmaf(av[kk], b[k4 + kk].z, a4[2]);
          a4[3] = fmaf(av[kk], b[k4 + kk].w, a4[3]);
        }
      }
      float* dst = cp + std::size_t(r0 + j) * g.ldc;
      if (g.dact) {
        const float h4[4] = {h[j].x, h[j].y, h[j].z, h[j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) a4[e] = act_bwd_h<float>(g.dact, a4[e], h4[e]);
      } else if (g.beta) {
        const float4 o = *reinterpret_cast<const float4*>(dst);
        a4[0] += o.x; a4[1] += o.y; a4[2] += o.z; a4[3] += o.w;
      }
      *reinterpret_cast<float4*>(dst) = make_float4(a4[0], a4[1], a4[2], a4[3]);
    }
  }
}

cudaError_t launch_dx_skinny(const GemmArgs<float>& g, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>((g.N + 1023) / 1024), (g.M + kDxRows - 1) / kDxRows);
  switch ((g.K + 3) / 4) {
    case 1: k_dx_skinny<4><<<grid, 256, 0, st>>>(g); break;
    case 2: k_dx_skinny<8><<<grid, 256, 0, st>>>(g); break;
    case 3: k_dx_skinny<12><<<grid, 256, 0, st>>>(g); break;
    default: k_dx_skinny<16><<<grid, 256, 0, st>>>(g); break;
  }
  return cudaGetLastError();
}

int simt_route(const GemmArgs<float>& g);
// A batched weight-gradient product that runs on the CTA pairs can also leave
// the row sums of its K-major A (the bias gradient) in g.rowsum: partials
// [z][M] for the caller's split reduce.
bool umma_rowsum_fusable(const GemmArgs<float>& g) {
  static const bool use_tma = !(std::getenv("TG_UMMA_TMA") && std::getenv("TG_UMMA_TMA")[0] == '0');
  if (!use_tma || g.epi != kEpiSplitK || !g.a_kmaj || !use_pair(g.M) || g.no_pair || simt_route(g) != 0) return false;
  if (g.mem) return true;   // batched products always take the TMA maps
  // unbatched: the pair path runs exactly when both operand maps encode as given
  CUtensorMap ta, tb;
  return make_operand_map(&ta, g.A, g.lda, false, g.M, g.K) && make_operand_map(&tb, g.B, g.ldb, g.b_nmaj, g.N, g.K);
}

// 0: tensor cores; 4: short K (K <= 32); 1: skinny M (M <= 16, K <= 2048);
// 2: skinny weight gradient (M <= 16 split-K over >= 65,536 samples);
// 3: skinny input adjoint (K <= 16 over >= 4,096 samples)
int simt_route(const GemmArgs<float>& g) {
  static const bool on = !(std::getenv("TG_SHORTK") && std::getenv("TG_SHORTK")[0] == '0');
  static const bool skinny = !(std::getenv("TG_SKINNY") && std::getenv("TG_SKINNY")[0] == '0');
  auto al = [](const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; };
  if (skinny && !g.mem && !g.no_pair && g.epi == kEpiSplitK && g.a_kmaj && !g.b_nmaj && g.M <= kSwRows &&
      g.K >= 65536 && g.ldb % 4 == 0 && al(g.B))
    return 2;
  if (skinny && !g.mem && !g.no_pair && g.epi == kEpiAccum && g.b_nmaj && g.K <= 16 && g.N >= 4096 && g.N % 4 == 0 &&
      g.ldb % 4 == 0 && g.ldc % 4 == 0 && al(g.B) && al(g.C) && (!g.dact || al(g.C2)))
    return 3;
  if (!on || g.mem || g.no_pair || g.epi != kEpiBiasAct || !g.b_nmaj || g.N % 4 || g.ldb % 4 || g.ldc % 4 || !al(g.B) ||
      !al(g.C) || (g.C2 && !al(g.C2)))
    return 0;
  if (g.K <= 32) return 4;
  if (skinny && g.M <= kSkRows && g.K <= 2048 && g.N >= 4096) return 1;
  return 0;
}

cudaError_t launch_gemm_umma(const GemmArgs<float>& g0, std::uint32_t splits, cudaStream_t st) {
  if (g0.M == 0 || g0.N == 0) return cudaSuccess;
  switch (simt_route(g0)) {
    case 2: return launch_dw_skinny(g0, splits, st);
    case 3: return launch_dx_skinny(g0, st);
    case 4: return g0.a_kmaj ? launch_shortk<true, 4>(g0, st) : launch_shortk<false, 4>(g0, st);
    case 1: return g0.a_kmaj ? launch_shortk<true, 1>(g0, st) : launch_shortk<false, 1>(g0, st);
    default: break;
  }
  // TMA-fed path: operands that satisfy the tensor-map rules (16-byte aligned
  // base and row stride); split-K slices start on 32-element k boundaries so a
  // k-tile never reads into the next slice (TMA zero-fills only past K).
  static const bool use_tma = !(std::getenv("TG_UMMA_TMA") && std::getenv("TG_UMMA_TMA")[0] == '0');
#ifdef TG_PROFILING
  static bool exp_set = false;
  if (!exp_set) {
    exp_set = true;
    if (const char* e = std::getenv("TG_UMMA_EXP")) {
      const int v = std::atoi(e);
      cudaMemcpyToSymbol(g_umma_exp, &v, sizeof(int));
    }
  }
#endif
  if (use_tma) {
    GemmArgs<float> g = g0;
    if (g.epi == kEpiSplitK) g.k_chunk = (g.k_chunk + BK - 1) / BK * BK;
    CUtensorMap ta, tb;
    const bool a_mn = !g.a_kmaj, b_mn = g.b_nmaj;
    // An operand TMA cannot describe (row stride not a multiple of 16 bytes,
    // e.g. cfg3's 200 x 30 weight) is copied to a padded scratch first when it
    // is small: one strided device copy (stream-ordered, graph-capturable)
    // instead of the register-staged kernel, whose per-tile fixed cost
    // dominated those products (880 us per call at K = 30, measured).
    float* pad_a = nullptr;
    float* pad_b = nullptr;
    auto pad = [&](const float* P, std::size_t ld, bool mn, std::uint32_t rows, float*& buf, std::size_t& ldp) {
      const std::size_t inner = mn ? rows : g.K, outer = mn ? g.K : rows;
      if (inner * outer > (std::size_t(1) << 22)) return P;
      ldp = (inner + 3) / 4 * 4;
      if (cudaMallocAsync(reinterpret_cast<void**>(&buf), ldp * outer * sizeof(float), st) != cudaSuccess ||
          cudaMemcpy2DAsync(buf, ldp * sizeof(float), P, ld * sizeof(float), inner * sizeof(float), outer,
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        cudaGetLastError();
        return P;
      }
      return static_cast<const float*>(buf);
    };
    if (g.mem) {
      // batched: one map per operand over its whole row span (rows are shifted
      // per member in the kernel); every operand is row-aligned, no padding
      if (!g.zs || (g.epi != kEpiSplitK && g.zs != 1)) return cudaErrorInvalidValue;
      auto span_map = [&](CUtensorMap* m, const float* P, std::size_t ld, bool mn, std::uint32_t rows, std::uint32_t span) {
        if (!span) return make_operand_map(m, P, ld, mn, rows, g.K);
        return mn ? make_operand_map(m, P, ld, true, rows, span) : make_operand_map(m, P, ld, false, span, g.K);
      };
      if (!span_map(&ta, g.A, g.lda, a_mn, g.M, g.a_span) || !span_map(&tb, g.B, g.ldb, b_mn, g.N, g.b_span))
        return cudaErrorInvalidValue;
      return launch_tma_kernel(g, splits, ta, tb, a_mn, b_mn, st);   // splits = members x zs
    }
    if (!make_operand_map(&ta, g.A, g.lda, a_mn, g.M, g.K)) {
      std::size_t ldp = g.lda;
      g.A = pad(g.A, g.lda, a_mn, g.M, pad_a, ldp);
      g.lda = ldp;
    }
    if (!make_operand_map(&tb, g.B, g.ldb, b_mn, g.N, g.K)) {
      std::size_t ldp = g.ldb;
      g.B = pad(g.B, g.ldb, b_mn, g.N, pad_b, ldp);
      g.ldb = ldp;
    }
    auto release = [&] {
      if (pad_a) cudaFreeAsync(pad_a, st);
      if (pad_b) cudaFreeAsync(pad_b, st);
    };
    if (make_operand_map(&ta, g.A, g.lda, a_mn, g.M, g.K) && make_operand_map(&tb, g.B, g.ldb, b_mn, g.N, g.K)) {
      const cudaError_t e = launch_tma_kernel(g, g.epi == kEpiSplitK ? splits : 1, ta, tb, a_mn, b_mn, st);
      release();
      return e;
    }
    release();
  }
  if (g0.mem) return cudaErrorInvalidValue;   // batched products need the TMA path
  const GemmArgs<float>& g = g0;
  // register-staged fallback (operands TMA cannot describe): its accumulator
  // is never drained, so its bias grows with K; beyond K = 1024 per launch the
  // SIMT GEMM is the more accurate engine
  {
    const std::uint32_t keff = g.epi == kEpiSplitK ? g.k_chunk : g.K;
    if (keff > 1024) return launch_gemm<float>(g, splits, st);
  }
  static PerDeviceOnce attr;
  if (const cudaError_t e = attr.ensure([] {
        return cudaFuncSetAttribute(k_umma_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
      }); e != cudaSuccess)
    return e;
  const dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.epi == kEpiSplitK ? splits : 1);
  k_umma_tf32x3<<<grid, 128, kSmem, st>>>(g);
  return cudaGetLastError();
}

#ifdef TG_PROFILING
cudaError_t read_pair_trace(long long* out) { return cudaMemcpyFromSymbol(out, g_pair_trace, sizeof(g_pair_trace)); }
#endif

}  // namespace tgk
#ifdef TG_PROFILING
extern "C" int tg_debug_pair_trace(long long* out) { return static_cast<int>(tgk::read_pair_trace(out)); }
#endif
