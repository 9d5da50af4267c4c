// tg_epilogue.cu — sample-invariant prologue and the batch-reduction epilogue.
//
// Prologue (one CTA): UV <- [params | uniform nodes | constants], evaluated
// once per launch instead of once per sample; wide reductions (e.g. the
// 1e-4 * sum p^2 regulariser over all 337 parameters of cfg2) run
// block-parallel with a fixed-order tree.
//
// Epilogue (grid): one warp per reduction destination sums its per-CTA
// partials in a fixed order (deterministic); the last CTA to finish then runs
// the uniform reverse sweep (propagate_node semantics, ops.hpp:316-454, in the
// reference processing order), writes grad_sum (= the accumulator of
// train_step) and, for tg_train_step, applies the GD update
// x -= gamma * g / b (sgd_step).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "tg_epilogue.cuh"
#include "tg_ops.cuh"

namespace tgk {

using tgc::Instr;
using tgc::kIndexMask;

namespace {

constexpr unsigned kBlock = 256;

// Block-wide sum with a fixed reduction tree (deterministic).
template <class T>
__device__ T block_sum(T v, T* red) {
  const unsigned t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (unsigned s = kBlock / 2; s > 0; s >>= 1) {
    if (t < s) red[t] += red[t + s];
    __syncthreads();
  }
  const T r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ bool wide_reducible(std::uint8_t op) {
  return op == AddVarying || op == MeanVarying || op == NegativeMeanVarying || op == SumOfSquaresVarying ||
         op == MeanSquaresVarying || op == InnerProductNoBias || op == InnerProductWithBias;
}

// Contribution of one node to its child j (ops whose per-child rule needs no
// other child's running state).  Returns false for rules that are serial.
template <class T>
__device__ __forceinline__ bool child_rule(std::uint8_t op, std::uint32_t n, std::uint32_t j, const std::uint32_t* o,
                                           const T* UV, T g, T& out) {
  switch (op) {
    case AddVarying: out = g; return true;
    case SubVarying: out = j == 0 ? g : -g; return true;
    case MeanVarying: out = g / static_cast<T>(n); return true;
    case NegativeMeanVarying: out = -g / static_cast<T>(n); return true;
    case SumOfSquaresVarying: out = g * T(2) * UV[o[j] & kIndexMask]; return true;
    case MeanSquaresVarying: out = (g * T(2) / static_cast<T>(n)) * UV[o[j] & kIndexMask]; return true;
    case InnerProductNoBias: {
      const std::uint32_t m = n / 2;
      out = g * UV[o[j < m ? j + m : j - m] & kIndexMask];
      return true;
    }
    case InnerProductWithBias: {
      const std::uint32_t m = (n - 1) / 2;
      out = j == n - 1 ? g : g * UV[o[j < m ? j + m : j - m] & kIndexMask];
      return true;
    }
    default: return false;
  }
}

}  // namespace

// Grid-wide part of the prologue for large parameter vectors (cfg5: 1.86 M).
template <class T>
__global__ void __launch_bounds__(kBlock) k_uv_init(UniformArgs<T> a) {
  const std::uint32_t stride = gridDim.x * kBlock;
  for (std::uint32_t i = blockIdx.x * kBlock + threadIdx.x; i < a.n_uv; i += stride) {
    a.UG[i] = T(0);
    if (i < a.n_params) a.UV[i] = a.params[i];
    else if (i >= a.const_base) a.UV[i] = a.consts[i - a.const_base];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.done) *a.done = 0u;
}

// Grid-wide grad_sum copy (+ fused GD) for large parameter vectors.
template <class T>
__global__ void __launch_bounds__(kBlock) k_finalize(UniformArgs<T> a) {
  const std::uint32_t stride = gridDim.x * kBlock;
  for (std::uint32_t i = blockIdx.x * kBlock + threadIdx.x; i < a.n_params; i += stride) {
    const T gsum = a.UG[i];
    if (a.grad_sum) a.grad_sum[i] = gsum;
    if (a.gd_params) a.gd_params[i] = a.gd_params[i] - a.gamma * gsum / a.gd_batch;
  }
}

template <class T>
__global__ void __launch_bounds__(kBlock) k_uniform_fwd(UniformArgs<T> a) {
  __shared__ T red[kBlock];
  // small tables (a.smem): the uniform program runs on a shared-memory copy of
  // UV (each instruction is a few shared-memory round trips, not global ones)
  extern __shared__ __align__(16) unsigned char dyn[];
  T* V = a.smem ? reinterpret_cast<T*>(dyn) : a.UV;
  if (a.copy) {
    for (std::uint32_t i = threadIdx.x; i < a.n_params; i += kBlock) V[i] = a.params[i];
    for (std::uint32_t i = threadIdx.x; i < a.n_const; i += kBlock) V[a.const_base + i] = a.consts[i];
    if (!a.smem)  // the smem epilogue reads only the reduced entries of UG
      for (std::uint32_t i = threadIdx.x; i < a.n_uv; i += kBlock) a.UG[i] = T(0);
    if (threadIdx.x == 0 && a.done) *a.done = 0u;
  }
  __syncthreads();
  UvAcc<T> acc{V, a.UG, nullptr, a.const_base};
  for (std::uint32_t k = 0; k < a.n_instr; ++k) {
    const Instr in = a.instr[k];
    const std::uint32_t* o = a.opnd + in.opnd;
    if (in.nops >= 64 && wide_reducible(in.op)) {
      const std::uint32_t n = in.nops;
      const bool ip = in.op == InnerProductNoBias || in.op == InnerProductWithBias;
      const std::uint32_t m = in.op == InnerProductWithBias ? (n - 1) / 2 : (ip ? n / 2 : n);
      T part = 0;
      for (std::uint32_t j = threadIdx.x; j < m; j += kBlock) {
        const T v = V[o[j] & kIndexMask];
        if (ip) part += v * V[o[m + j] & kIndexMask];
        else if (in.op == SumOfSquaresVarying || in.op == MeanSquaresVarying) part += v * v;
        else part += v;
      }
      T s = block_sum(part, red);
      if (threadIdx.x == 0) {
        if (in.op == InnerProductWithBias) s = V[o[n - 1] & kIndexMask] + s;
        if (in.op == MeanVarying || in.op == MeanSquaresVarying) s /= static_cast<T>(n);
        if (in.op == NegativeMeanVarying) s = -s / static_cast<T>(n);
        V[in.out] = s;
      }
    } else if (threadIdx.x == 0) {
      acc.o = o;
      bool bad = false;
      T badv = 0;
      V[in.out] = eval_node<T>(in.op, in.nops, o, in.cst, acc, bad, badv);
      if (bad) {
        record_error(a.err_key, 0, in.node);
        if (*a.err_op == 0xffffffffu) { *a.err_op = in.op; *a.err_val = static_cast<double>(badv); }
      }
    }
    __syncthreads();
  }
  if (a.smem || a.UVc)
    for (std::uint32_t i = threadIdx.x; i < a.n_uv; i += kBlock) {
      const T v = V[i];
      if (a.smem) a.UV[i] = v;
      if (a.UVc) a.UVc[i] = v;   // mirror into the specialised kernel's __constant__ table
    }
}

template <class T>
__global__ void __launch_bounds__(kBlock) k_reduce_epilogue(ReduceArgs<T> r, UniformArgs<T> a) {
  __shared__ unsigned last;
  // ---- fixed-order reduction of the per-CTA partials ----
  const std::uint32_t warp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const std::uint32_t lane = threadIdx.x & 31;
  if (r.n_rows == 1) {
    // one partial row (the staged tier's chunk accumulator): a grid-stride
    // copy, not a warp per destination (cfg5: 1.86M destinations had made
    // this launch 232,962 CTAs and 0.56 ms)
    for (std::size_t d = std::size_t(blockIdx.x) * kBlock + threadIdx.x; d < r.n_dest;
         d += std::size_t(gridDim.x) * kBlock)
      a.UG[r.dest_uv[d]] = r.partial[d];
  } else if (warp < r.n_dest) {
    const T* row = r.partial + std::size_t(warp) * r.n_rows;
    T tot = 0;
    for (std::uint32_t c = lane; c < r.n_rows; c += 32) tot += row[c];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, s);
    if (lane == 0) a.UG[r.dest_uv[warp]] = tot;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // ---- uniform reverse sweep (last CTA) ----
  // small tables (a.smem): on shared-memory copies of UV / UG; UG starts from
  // the reduced destinations only (the prologue does not zero it)
  extern __shared__ __align__(16) unsigned char dyn[];
  T* V = a.UV;
  T* G = a.UG;
  if (a.smem) {
    V = reinterpret_cast<T*>(dyn);
    G = V + a.n_uv;
    for (std::uint32_t i = threadIdx.x; i < a.n_uv; i += kBlock) {
      V[i] = a.UV[i];
      G[i] = T(0);
    }
    __syncthreads();
    for (std::uint32_t d = threadIdx.x; d < r.n_dest; d += kBlock) G[r.dest_uv[d]] = a.UG[r.dest_uv[d]];
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.root_uv != tgc::kNone) G[a.root_uv] += static_cast<T>(a.batch);
  __syncthreads();
  UvAcc<T> acc{V, G, nullptr, a.const_base};
  for (std::uint32_t k = 0; k < a.n_instr; ++k) {
    const Instr in = a.instr[k];
    const std::uint32_t* o = a.opnd + in.opnd;
    const T g = G[in.out];
    const T y = V[in.out];
    T dummy;
    const bool parallel = (in.pad & 1) && in.nops >= 32 && child_rule<T>(in.op, in.nops, 0, o, V, g, dummy);
    if (parallel) {  // distinct children: one thread per child
      for (std::uint32_t j = threadIdx.x; j < in.nops; j += kBlock) {
        T c;
        child_rule<T>(in.op, in.nops, j, o, V, g, c);
        const std::uint32_t u = o[j] & kIndexMask;
        if (u < a.const_base) G[u] += c;
      }
    } else if (threadIdx.x == 0) {
      acc.o = o;
      propagate<T>(in.op, in.nops, o, in.cst, g, y, acc);
    }
    __syncthreads();
  }
  // ---- grad_sum and the fused GD update (large vectors: k_finalize) ----
  if (!a.copy) return;
  for (std::uint32_t i = threadIdx.x; i < a.n_params; i += kBlock) {
    const T gsum = G[i];
    if (a.grad_sum) a.grad_sum[i] = gsum;
    if (a.gd_params) a.gd_params[i] = a.gd_params[i] - a.gamma * gsum / a.gd_batch;
  }
}

constexpr std::uint32_t kGridCopy = 1u << 16;   // above this many entries, copies run grid-wide
constexpr std::uint32_t kSmemUV = 3072;         // up to this many entries, UV / UG are staged in shared memory

template <class T>
cudaError_t launch_uniform_fwd(const UniformArgs<T>& a, cudaStream_t st, std::uint64_t& launches) {
  UniformArgs<T> b = a;
  b.copy = a.n_uv <= kGridCopy;
  b.smem = a.n_uv <= kSmemUV;
  if (!b.copy) {
    k_uv_init<T><<<std::min<std::uint32_t>(592, (a.n_uv + kBlock - 1) / kBlock), kBlock, 0, st>>>(a);
    ++launches;
    if (a.n_instr == 0 && !a.UVc) return cudaGetLastError();
  }
  k_uniform_fwd<T><<<1, kBlock, b.smem ? a.n_uv * sizeof(T) : 0, st>>>(b);
  ++launches;
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_reduce_epilogue(const ReduceArgs<T>& r, const UniformArgs<T>& a, cudaStream_t st,
                                   std::uint64_t& launches) {
  const unsigned warps_per_block = kBlock / 32;
  unsigned grid = r.n_dest ? (r.n_dest + warps_per_block - 1) / warps_per_block : 1;
  if (r.n_rows == 1) grid = std::max(1u, std::min<unsigned>(1184u, (r.n_dest + kBlock - 1) / kBlock));
  UniformArgs<T> b = a;
  b.copy = a.n_params <= kGridCopy;
  b.smem = a.n_uv <= kSmemUV;
  k_reduce_epilogue<T><<<grid, kBlock, b.smem ? 2 * a.n_uv * sizeof(T) : 0, st>>>(r, b);
  ++launches;
  if (!b.copy) {
    k_finalize<T><<<std::min<std::uint32_t>(592, (a.n_params + kBlock - 1) / kBlock), kBlock, 0, st>>>(b);
    ++launches;
  }
  return cudaGetLastError();
}

template cudaError_t launch_uniform_fwd<double>(const UniformArgs<double>&, cudaStream_t, std::uint64_t&);
template cudaError_t launch_uniform_fwd<float>(const UniformArgs<float>&, cudaStream_t, std::uint64_t&);
template cudaError_t launch_reduce_epilogue<double>(const ReduceArgs<double>&, const UniformArgs<double>&, cudaStream_t,
                                                    std::uint64_t&);
template cudaError_t launch_reduce_epilogue<float>(const ReduceArgs<float>&, const UniformArgs<float>&, cudaStream_t,
                                                   std::uint64_t&);

}  // namespace tgk
