// mma_peak.cu — measured tcgen05 tensor-core throughput of this GPU for the
// kinds the dense-layer products use: kind::tf32 (the 3xTF32 fp32 emulation
// issues three of these per fp32 product) and kind::f16 with bf16 operands
// (the MEASURED_PEAKS.json bf16 figure, for comparison).  The roofline
// denominator of the tensor-bound configs (cfg4, cfg5) is tf32 / 3.
//
// One CTA per SM; one elected thread issues M=128 x N=256 MMAs (K = 8 tf32 /
// 16 bf16 per instruction) from shared-memory operands into one TMEM
// accumulator back to back, commits once, waits.  Burst = best of 5 short
// launches; sustained = the mean over ~4 s of back-to-back launches.
// Writes profiles/mma_peaks.json.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ std::uint64_t desc_none(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
  return static_cast<std::uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<std::uint64_t>(lbo >> 4) << 16) |
         (static_cast<std::uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}

constexpr int M = 128, N = 256;

template <int KIND>   // 0: tf32 (K 8), 1: bf16 (K 16)
__global__ void __launch_bounds__(128, 1) k_mma_peak(int iters, float* sink) {
  __shared__ __align__(1024) unsigned char sA[M * 32];
  __shared__ __align__(1024) unsigned char sB[N * 32];
  __shared__ std::uint64_t mbar;
  __shared__ std::uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * 32 / 4; i += 128) reinterpret_cast<std::uint32_t*>(sA)[i] = 0x3f800000u ^ (i * 2654435761u & 0x007fe000u);
  for (int i = tid; i < N * 32 / 4; i += 128) reinterpret_cast<std::uint32_t*>(sB)[i] = 0x3f000000u ^ (i * 2246822519u & 0x007fe000u);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const std::uint32_t tmem = tslot;
  if (tid == 0) {
    const std::uint32_t idesc = KIND == 0 ? (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24)
                                          : (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
    const std::uint64_t da = desc_none(smem_u32(sA), M * 16, 128), db = desc_none(smem_u32(sB), N * 16, 128);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const std::uint32_t acc = (i | u) ? 1u : 0u;
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                       "l"(da), "l"(db), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                       "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}\n" ::"r"(
            smem_u32(&mbar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  std::uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + (static_cast<std::uint32_t>(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (tid == 0) sink[blockIdx.x] = __uint_as_float(r);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N));
}

template <int KIND>
void measure(int nsm, double& burst, double& sustained) {
  float* sink;
  cudaMalloc(&sink, 4096 * sizeof(float));
  const double flop_per_instr = 2.0 * M * N * (KIND == 0 ? 8 : 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mma_peak<KIND><<<nsm, 128>>>(64, sink);
  cudaDeviceSynchronize();
  const int iters = 20000;   // ~3-6 ms per launch
  burst = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_mma_peak<KIND><<<nsm, 128>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = flop_per_instr * 8.0 * iters * nsm / (ms * 1e-3) / 1e12;
    if (tf > burst) burst = tf;
  }
  // sustained: back-to-back for ~4 s
  const auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0);
  long launches = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 4.0) {
    for (int j = 0; j < 50; ++j) k_mma_peak<KIND><<<nsm, 128>>>(iters, sink);
    launches += 50;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  sustained = flop_per_instr * 8.0 * iters * nsm * double(launches) / (ms * 1e-3) / 1e12;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) std::printf("CUDA error: %s\n", cudaGetErrorString(e));
  cudaFree(sink);
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double tb, ts, bb, bs;
  measure<0>(nsm, tb, ts);
  measure<1>(nsm, bb, bs);
  std::printf("tcgen05 kind::tf32  burst %.1f TFLOP/s  sustained %.1f TFLOP/s\n", tb, ts);
  std::printf("tcgen05 kind::f16 (bf16)  burst %.1f TFLOP/s  sustained %.1f TFLOP/s\n", bb, bs);
  const char* path = argc > 1 ? argv[1] : "profiles/mma_peaks.json";
  if (FILE* f = std::fopen(path, "w")) {
    std::fprintf(f,
                 "{\"tf32_tcgen05_tflops\": %.1f, \"tf32_tcgen05_tflops_sustained\": %.1f, \"bf16_tcgen05_tflops\": %.1f, "
                 "\"bf16_tcgen05_tflops_sustained\": %.1f, \"sms\": %d, \"how\": \"tools/mma_peak.cu: 1 CTA/SM, M128 N256 "
                 "tcgen05.mma cta_group::1 back to back from smem into one TMEM accumulator; burst = best of 5 launches, "
                 "sustained = mean over 4 s back to back\"}\n",
                 tb, ts, bb, bs, nsm);
    std::fclose(f);
  }
  return 0;
}
