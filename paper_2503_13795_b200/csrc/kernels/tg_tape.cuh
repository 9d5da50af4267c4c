// tg_tape.cuh — kernel argument blocks and launchers of the tape engine.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../host/tg_program.hpp"
#include "tg_epilogue.cuh"

namespace tgk {

template <class T>
struct MainArgs {
  const tgc::Instr* fwd;
  const tgc::Instr* bwd;
  const std::uint32_t* opnd;
  const std::uint8_t* oflag;
  const std::uint32_t* oaux;
  const std::uint32_t* zero_rows;
  const std::uint32_t* input_rows;
  const tgc::GatherTable* ug;
  const tgc::GatherTable* sg;
  const std::uint32_t* cand;
  const std::uint32_t* term_off;
  const tgc::Term* terms;
  const tgc::Dense* dense;
  const tgc::Attn* attn;
  const std::uint32_t* arows;
  const tgc::LNorm* lnorm;
  const std::uint32_t* lnrows;
  const std::uint8_t* lnflag;
  const T* UV;
  const T* inputs;
  const std::int32_t* idx;
  T* loss;
  T* igrad;
  T* partial;
  T* gV;
  T* gG;
  unsigned long long* err_key;
  double* err_val;
  std::uint32_t* err_op;
  std::size_t batch;
  std::size_t ld;          // row stride: S+pad (shared) or grid*S (HBM)
  long long diag_sample;   // >= 0: re-run one sample to recover a domain error
  std::uint32_t n_fwd, n_bwd, n_zero, n_inputs, n_dest;
  std::uint32_t n_rows, S, root_row;
};
template <class T>
cudaError_t launch_tape(const MainArgs<T>& a, bool smem, unsigned grid, unsigned block, std::size_t smem_bytes,
                        cudaStream_t st);
template <class T> int tape_occupancy(bool smem, unsigned block, std::size_t smem_bytes);
template <class T>
cudaError_t launch_gd(T* params, const T* g, std::uint32_t n, double gamma, double b, cudaStream_t st);

}  // namespace tgk
