// fp_peak.cu — measures the SIMT FMA throughput ceiling (FP64 DFMA, FP32 FFMA)
// of this GPU: the roofline denominator for the scalar-tape kernels, which
// MEASURED_PEAKS.json (HBM copy, bf16 GEMM) does not cover.  Writes
// profiles/fp_peaks.json.  8 independent FMA chains per thread, full grid.
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <class T>
double run(int nsm) {
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  T* out;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_loop<T><<<blocks, threads>>>(out, 16, T(0.999), T(0.001));
  double best = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    best = flops / (ms * 1e-3) / 1e12 > best ? flops / (ms * 1e-3) / 1e12 : best;
  }
  cudaFree(out);
  return best;
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const double f64 = run<double>(nsm), f32 = run<float>(nsm);
  const char* path = argc > 1 ? argv[1] : "profiles/fp_peaks.json";
  FILE* f = fopen(path, "w");
  fprintf(f, "{\"fp64_tflops\": %.3f, \"fp32_tflops\": %.3f, \"sms\": %d, \"how\": \"8 independent FMA chains x 256 threads x 8 CTAs/SM, best of 5, CUDA events\"}\n", f64, f32, nsm);
  fclose(f);
  printf("fp64 %.2f TFLOP/s  fp32 %.2f TFLOP/s  (%d SMs)\n", f64, f32, nsm);
  return 0;
}
