// tg_synth.cu — on-device synthetic batches: the same
// bits as the host generator tgs::synth_sample (tg_synth.cuh), written
// straight into the step's device input arrays, so a training loop over
// generated data moves no input bytes over PCIe.
//
// One thread per sample; every column store of a warp is 32 consecutive
// samples of one column (128 B fp32 / 256 B fp64 / 128 B int32 rows), so the
// [col][batch] SoA layout is written with full-sector coalesced stores.  The
// Zipf CDF (<= 1024 fp64 entries) travels in the kernel parameters.
#include <cuda_runtime.h>

#include <cstdint>

#include "tg_synth.cuh"

namespace tgk {
namespace {

constexpr std::uint32_t kMaxV = 1024;
struct CdfTable { double v[kMaxV]; };

template <class Scalar>
__global__ void __launch_bounds__(256) k_synth(tgs::SynthArgs a, const __grid_constant__ CdfTable t) {
  a.cdf = t.v;
  for (std::size_t i = blockIdx.x * std::size_t(blockDim.x) + threadIdx.x; i < a.batch;
       i += std::size_t(gridDim.x) * blockDim.x)
    tgs::synth_sample<Scalar>(a, i);
}

}  // namespace

// Returns cudaErrorInvalidValue when the Zipf table exceeds kMaxV entries.
cudaError_t launch_synth(const tgs::SynthArgs& a, const double* cdf_host, cudaStream_t st) {
  if (a.batch == 0) return cudaSuccess;
  CdfTable t{};
  if (a.V > kMaxV) return cudaErrorInvalidValue;
  for (std::uint32_t i = 0; i < a.V; ++i) t.v[i] = cdf_host[i];
  const std::size_t blocks = (a.batch + 255) / 256;
  const unsigned grid = static_cast<unsigned>(blocks < 148 * 32 ? blocks : 148 * 32);
  if (a.f64) k_synth<double><<<grid, 256, 0, st>>>(a, t);
  else k_synth<float><<<grid, 256, 0, st>>>(a, t);
  return cudaGetLastError();
}

}  // namespace tgk
