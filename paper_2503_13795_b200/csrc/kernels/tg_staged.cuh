// tg_staged.cuh — staged execution of large tapes over an HBM SoA workspace.
//
// Tapes whose per-sample rows do not fit a shared-memory tile (cfg3/4/5) run
// stage by stage over a chunk of the batch: per-sample segments of the
// instruction stream on the interpreter (one thread per sample, rows in HBM
// [row][sample]), dense layers (kDense) as matrix products over the chunk.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../host/tg_program.hpp"

namespace tgk {

enum RangeFlags : std::uint32_t {
  kRFwd = 1,      // forward instructions [fwd_begin, fwd_end)
  kRSeed = 2,     // zero_rows <- 0, loss out, root adjoint <- 1
  kRBwd = 4,      // reverse instructions [bwd_begin, bwd_end)
  kROut = 8,      // input gradients out
};

template <class T>
struct RangeArgs {
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
  T* V;
  T* G;
  unsigned long long* err_key;
  std::size_t batch;      // global batch (leading dim of inputs / idx / outputs)
  std::size_t s0;         // first sample of the chunk
  std::size_t n;          // samples in the chunk
  std::size_t ld;         // row stride of V / G (chunk capacity)
  std::uint32_t fwd_begin, fwd_end, bwd_begin, bwd_end;
  std::uint32_t n_zero, n_inputs, root_row, flags;
  std::uint32_t per_sample;   // level stages of macro-instructions (layer norms ...): one sample per thread
};

// C(m, n) = sum_k A(m, k) B(k, n) over an operand view:
//   A(m, k) = A[m * lda + k]  (a_kmaj)   or  A[k * lda + m]
//   B(k, n) = B[k * ldb + n]  (b_nmaj)   or  B[n * ldb + k]
enum GemmEpi : int {
  kEpiBiasAct = 0,   // C = acc (+ bias[m]); C2 = act(C) if act
  kEpiAccum = 1,     // C = beta ? C + acc : acc
  kEpiSplitK = 2,    // part[kz][m][n] = acc over this CTA's K slice
};

template <class T>
struct GemmArgs {
  const T* A;
  const T* B;
  T* C;
  T* C2;
  const T* bias;
  std::size_t lda, ldb, ldc;
  std::uint32_t M, N, K;
  std::uint32_t k_chunk;   // split-K slice (kEpiSplitK)
  std::uint32_t act;
  int beta;
  bool a_kmaj, b_nmaj;
  int epi;
  // Batched products (tcgen05 path only): blockIdx.z / zs selects a member
  // whose row offsets {a, b, c, c2} shift the operands' outer (row)
  // coordinate and the output rows; a_span / b_span are the row extents of
  // the operand maps (0: the operand is shared, no offset).  Split-K partials
  // are indexed by blockIdx.z = member * zs + slice.
  const uint4* mem;
  std::uint32_t zs;
  std::uint32_t a_span, b_span;
  bool no_pair;            // tcgen05 path: single-CTA tiles even when M > 128 (tg_gemm engine 2)
  // kEpiAccum with dact != 0 (beta = 0): C = act'(H) * acc, the derivative
  // taken from the activation output H at C2 (+ member row offset c2), i.e.
  // the input adjoint product writes dz of the layer below directly
  std::uint32_t dact;
  // kEpiBiasAct with act: store only H (C2); the pre-activation Z has no reader
  bool no_z;
  // kEpiSplitK, K-major A on the CTA pairs (umma_rowsum_fusable): also write
  // the row sums of A over this split's k range to rowsum[z * M + m]
  T* rowsum;
};

// Table-scatter (kind-1) batch terms grouped by (adjoint row a, index column f).
struct ScatterGroup {
  std::uint32_t a, f, rows, pad;
};
struct ScatterUse {          // dest += coef * H_g[r]
  std::uint32_t g, r;
  double coef;
};
template <class T>
cudaError_t launch_scatter(const ScatterGroup* groups, std::uint32_t n_groups, std::uint32_t r_max, const ScatterUse* uses,
                           const std::uint32_t* use_off, const std::uint32_t* dests, std::uint32_t n_dests, const T* G,
                           const std::int32_t* idx, std::size_t batch, std::size_t s0, std::size_t n, std::size_t ld,
                           T* part, std::uint32_t n_chunks, T* acc, cudaStream_t st);

template <class T> cudaError_t launch_tape_range(const RangeArgs<T>& a, cudaStream_t st);
// One dependency level (fwd_begin/fwd_end with kRFwd, else bwd_begin/bwd_end):
// one instruction per CTA column, 128 samples per CTA.
template <class T> cudaError_t launch_level_range(const RangeArgs<T>& a, cudaStream_t st);
template <class T> cudaError_t launch_gemm(const GemmArgs<T>& g, std::uint32_t splits, cudaStream_t st);
// fp32 GEMM on the 5th-gen tensor cores (tcgen05.mma kind::tf32, 3xTF32 split), tg_umma.cu
cudaError_t launch_gemm_umma(const GemmArgs<float>& g, std::uint32_t splits, cudaStream_t st);
// Fused softmax attention heads (kAttn) of one stage: instructions list[begin, begin + count),
// one CTA per head and 8 samples (tg_attn.cu); fp32, hd / dv <= 16, <= 64 keys and units.
bool attn_fast_ok(const tgc::Attn& A);
cudaError_t launch_attn(bool fwd, const tgc::Instr* list, std::uint32_t begin, std::uint32_t count, const tgc::Attn* attn,
                        const std::uint32_t* arows, float* V, float* G, std::size_t n, std::size_t ld, std::uint32_t hd_max,
                        cudaStream_t st);
// CTAs one split-K slice / batch member of a tcgen05 product launches (CTA pairs when M > 128)
std::uint32_t umma_ctas_per_slice(std::uint32_t M, std::uint32_t N);
bool umma_rowsum_fusable(const GemmArgs<float>& g);
// dst[m * N + n] += sum_kz part[kz][m][n]   (fixed order)
template <class T> cudaError_t launch_splitk_reduce(const T* part, T* dst, std::uint32_t MN, std::uint32_t splits, cudaStream_t st);
// G[z rows] = act'(G[h rows], V[h rows], V[z rows]) for n_out consecutive rows
template <class T> cudaError_t launch_act_bwd(T* G, const T* V, std::uint32_t z_row, std::uint32_t h_row, std::uint32_t n_out,
                                              std::size_t n, std::size_t ld, std::uint32_t act, cudaStream_t st);
// dst[j] += sum_s G[(row0 + j) * ld + s]   (fixed-order block tree per row)
template <class T> cudaError_t launch_rowsum(const T* G, std::uint32_t row0, std::uint32_t rows, std::size_t n, std::size_t ld,
                                             T* dst, cudaStream_t st);
// Batched forms over the members of a dense batch (mem[p].z = z row, .w = h row):
// activation derivative for every member, and dst[j] += sum_p sum_s G[mem[p].z + j]
// (members in order, then the fixed-order tree over samples).
template <class T> cudaError_t launch_act_bwd_batched(T* G, const T* V, const uint4* mem, std::uint32_t n_mem, std::uint32_t n_out,
                                                      std::size_t n, std::size_t ld, std::uint32_t act, cudaStream_t st);
template <class T> cudaError_t launch_rowsum_batched(const T* G, const uint4* mem, std::uint32_t n_mem, std::uint32_t rows,
                                                     std::size_t n, std::size_t ld, T* dst, T* scratch,
                                                     std::size_t scratch_elems, cudaStream_t st);
// Contended adjoint rows at the end of a reverse level, e = {row, assign, t0, count}:
// G[row] = (assign ? 0 : G[row]) + G[t0] + ... + G[t0 + count - 1]   (in order)
template <class T> cudaError_t launch_row_sums(const uint4* ent, std::uint32_t n_ent, T* G, std::size_t n, std::size_t ld,
                                               cudaStream_t st);
// zero `count` rows of X starting at row0 (first n columns)
template <class T> cudaError_t launch_zero_rows(T* X, const std::uint32_t* rows, std::uint32_t count, std::size_t n, std::size_t ld, cudaStream_t st);
// generic batch terms of the listed destinations over the chunk: acc[d] += ...
template <class T>
cudaError_t launch_contract(const std::uint32_t* dests, std::uint32_t n_dests, const std::uint32_t* term_off, const tgc::Term* terms,
                            const T* G, const T* V, const std::int32_t* idx, std::size_t batch, std::size_t s0, std::size_t n,
                            std::size_t ld, T* acc, cudaStream_t st);

// Embedding-MLP / softmax-CE tape as one kernel (tg_fused.cu): C contexts of an
// E-wide table of V rows -> H units (act) -> O logits -> CE against the target
// column.  Parameter UV offsets; gradients as partials [cta][q] in q order
// [W1 (H x C E) | b1 (H) | W2 (O x H) | b2 (O) | E (V x E)], reduced into
// acc[dmap[q]] (dmap[q] == kNone: no destination).
struct FusedMlpArgs {
  const float* UV;
  const std::int32_t* idx;   // [n_index_inputs][batch]
  std::size_t batch;
  std::uint32_t C, E, V, H, O, act;
  std::uint32_t ctx_col[8], tgt_col;
  std::uint32_t uv_E, uv_W1, uv_b1, uv_W2, uv_b2;   // b: kNone when absent
  std::uint32_t nq;
  float* loss;
  float* part;               // [grid][nq]
};
std::size_t fused_mlp_smem(const FusedMlpArgs& a);
unsigned fused_mlp_grid(std::size_t batch, int nsm);
cudaError_t launch_fused_mlp(const FusedMlpArgs& a, unsigned grid, const std::uint32_t* dmap, float* acc,
                             cudaStream_t st);

}  // namespace tgk
