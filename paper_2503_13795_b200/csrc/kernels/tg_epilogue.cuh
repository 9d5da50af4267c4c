// tg_epilogue.cuh — argument blocks of the uniform prologue / reduction epilogue.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../host/tg_program.hpp"

namespace tgk {

template <class T>
struct UniformArgs {
  const tgc::Instr* instr;   // ufwd (prologue) or ubwd (epilogue)
  const std::uint32_t* opnd;
  const T* params;
  const T* consts;
  T* UV;
  T* UVc;                    // optional __constant__ mirror (specialised kernels)
  T* UG;
  T* grad_sum;
  T* gd_params;              // non-null: fused GD update in the epilogue
  T gamma;
  T gd_batch;
  unsigned* done;            // last-CTA ticket (zeroed by the prologue)
  unsigned long long* err_key;
  double* err_val;
  std::uint32_t* err_op;
  std::size_t batch;
  std::uint32_t n_instr, n_params, n_const, const_base, n_uv, root_uv;
  int copy;                  // set by the launchers: copies done inside the single-CTA kernels
  int smem;                  // set by the launchers: UV / UG staged in shared memory (small tables)
};

template <class T>
struct ReduceArgs {
  const T* partial;          // [dest][n_rows]
  const std::uint32_t* dest_uv;
  std::uint32_t n_dest, n_rows;
};

template <class T> cudaError_t launch_uniform_fwd(const UniformArgs<T>& a, cudaStream_t st, std::uint64_t& launches);
template <class T>
cudaError_t launch_reduce_epilogue(const ReduceArgs<T>& r, const UniformArgs<T>& a, cudaStream_t st,
                                   std::uint64_t& launches);

}  // namespace tgk
