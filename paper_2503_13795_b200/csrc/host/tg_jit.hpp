// tg_jit.hpp — register-resident specialisation of short tapes.
//
// The interpreter (kernels/tg_tape.cu) keeps per-sample values in shared
// memory because an instruction stream cannot index registers.  For short
// tapes (cfg1, cfg2, fuzz graphs) the compiler instead emits the program as
// straight-line CUDA C++ — every node value and adjoint a register, every
// sample-invariant operand a constant-bank operand — and compiles it with
// NVRTC for sm_100a at tg_compile time.  Semantics are those of the
// interpreter, instruction by instruction (same forward formulas, same
// reverse processing order, same first-write analysis, same contraction).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tg_program.hpp"

namespace tgj {

struct JitConfig {
  unsigned block = 128;          // threads per CTA
  unsigned spt = 1;              // samples per thread per tile
  bool const_uv = true;          // sample-invariant table in __constant__
  unsigned ndpt = 0;             // reduction destinations per thread (registers)
  unsigned min_blocks = 0;       // __launch_bounds__ minBlocksPerSM (0 = unset)
  unsigned unroll_j = 4;         // dense-layer output loop unroll (independent chains)
  bool dense_loop = false;       // dense layers as loops (rows in smem) vs unrolled (rows in registers)
  bool fuse = false;             // prologue in the kernel + generated epilogue kernel (tg_jit_epi)
  bool coop = false;             // fused epilogue inside the tape kernel (cooperative launch, grid barriers)
};

// Kernel argument block of tg_jit_tape, passed by value; the generated code
// declares the same struct (tg_jit.cpp kPrelude), field for field.
template <class T>
struct JitArgs {
  const T* in; const int* idx; unsigned long long batch;
  T* loss; T* igrad; T* partial; unsigned grid_rows; unsigned n_groups;
  unsigned long long* err_key; double* err_val; unsigned* err_op;
  const T* UVg; const unsigned* cand; const unsigned* toff; const void* terms;
  const T* params; const T* consts; T* UVw;      // fused prologue: each CTA evaluates the uniform program
  unsigned* tickets; T* partial2;                // fused epilogue: two-level last-CTA reduction
  T* grad_sum; T* gd_params; T gamma; T gd_batch;
};

struct JitKernel {
  bool ok = false;
  std::string log;               // NVRTC log / failure reason
  std::string source;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  cudaKernel_t fn_epi = nullptr;  // generated epilogue (fused programs)
  void* cuv = nullptr;           // __constant__ table address (const_uv)
  std::size_t cuv_bytes = 0;
  JitConfig cfg;
  unsigned tile = 128;           // samples per tile = block * spt (grouped: per block iteration)
  unsigned group = 0;            // lanes per sample (grouped form), 0 = one thread per sample
  std::string group_log;         // why the dmma / grouped form was not used
  std::string form;              // "dmma" | "group" | "classic"
  bool fused = false;            // prologue + epilogue (+ GD) inside the kernel: one launch per step
  bool balanced = false;         // CTAs take contiguous shares of the batch (grid sized by 32-sample units)
  bool coop = false;             // one cooperative launch per step (no tg_jit_epi)
  std::size_t smem_bytes = 0;    // contraction rows
  unsigned n_crow_g = 0, n_crow_v = 0;
  int occ = 0;
  void* d_terms = nullptr;       // remapped terms
  void* d_toff = nullptr;
  double compile_ms = 0;
  std::size_t cubin_bytes = 0;
};

/// Whether the program is small enough to specialise.
bool eligible(const tgc::Program& P);
/// Emits the CUDA source for P (exposed for tests / inspection).
std::string generate(const tgc::Program& P, const JitConfig& cfg, unsigned& n_crow_g, unsigned& n_crow_v,
                     std::vector<tgc::Term>& terms_out, std::vector<std::uint32_t>& toff_out,
                     std::size_t& smem_elems);
/// Generates, compiles (NVRTC, sm_100a) and loads; requires a device.
JitKernel build(const tgc::Program& P);
void release(JitKernel& k);

}  // namespace tgj
