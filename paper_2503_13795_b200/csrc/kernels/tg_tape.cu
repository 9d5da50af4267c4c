// tg_tape.cu — batched forward / reverse tape kernels for sm_100a.
//
// One CTA processes a tile of S samples, one sample per thread, and walks the
// compiled program: a warp-uniform instruction stream (every lane executes
// the same node), per-sample values and adjoints stored [row][sample] so each
// node access is a unit-stride shared-memory (or HBM) transaction.  At the end
// of a tile the CTA contracts over its samples the per-sample contributions
// to sample-invariant operands (parameter gradients, uniform-node adjoints),
// accumulating a per-CTA partial row; a second kernel reduces the partial rows
// in a fixed order (deterministic), then the uniform reverse sweep and the GD
// update run.
//
// Replaces, per sample, the reference's eager build (ops.hpp:38-307),
// zero_grads (backprop.hpp:100-109), backward_with_scratch
// (backprop.hpp:139-184) and the accumulator add of train_step.
#include <cuda_runtime.h>

#include <cstdint>

#include "tg_ops.cuh"
#include "tg_tape.cuh"

namespace tgk {

using tgc::Instr;
using tgc::Term;
using tgc::GatherTable;
using tgc::kIndexMask;
using tgc::kModeShift;

// ---------------------------------------------------------------------------
// accessors
// ---------------------------------------------------------------------------

template <class T>
struct RowAcc {
  T* V;
  T* G;
  std::size_t ld;
  std::size_t col;
  const T* __restrict__ UV;
  const std::int32_t* __restrict__ idx;
  std::size_t batch;
  std::size_t s;
  const GatherTable* __restrict__ sg;
  const std::uint32_t* __restrict__ cand;
  const std::uint32_t* o;
  const std::uint8_t* fl;
  const std::uint32_t* ax;
  unsigned long long* err_key;

  __device__ __forceinline__ std::uint32_t sg_row(std::uint32_t i) const {
    const GatherTable t = sg[i];
    std::int32_t r = idx[std::size_t(t.col) * batch + s];
    if (r < 0 || static_cast<std::uint32_t>(r) >= t.n_rows) r = 0;
    return cand[t.cand_off + r];
  }
  __device__ __forceinline__ T val(std::uint32_t op) const {
    const std::uint32_t m = op >> kModeShift, i = op & kIndexMask;
    if (m == tgc::kSlot) return V[i * ld + col];
    if (m == tgc::kUv) return UV[i];
    return V[sg_row(i) * ld + col];
  }
  __device__ __forceinline__ void push(std::uint32_t k, T v) {
    const std::uint32_t op = o[k];
    const std::uint32_t m = op >> kModeShift, i = op & kIndexMask;
    const std::uint8_t f = fl[k];
    if (f & tgc::kToAux) {   // sample-invariant operand, or (staged levels) a contended row's temporary
      G[std::size_t(ax[k]) * ld + col] = v;
    } else if (m == tgc::kSlot) {
      T* p = &G[i * ld + col];
      *p = (f & tgc::kAssign) ? v : *p + v;
    } else if (m == tgc::kSGather) {
      G[sg_row(i) * ld + col] += v;
    }
  }
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

template <class T, bool kSmem>
__global__ void __launch_bounds__(256) k_tape(MainArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const std::uint32_t tid = threadIdx.x;
  const std::uint32_t S = a.S;
  T* V;
  T* G;
  std::size_t ld, col0;
  if (kSmem) {
    V = reinterpret_cast<T*>(smem_raw);
    G = V + std::size_t(a.n_rows) * a.ld;
    ld = a.ld;
    col0 = 0;
  } else {
    V = a.gV;
    G = a.gG;
    ld = a.ld;
    col0 = std::size_t(blockIdx.x) * S;
  }
  const std::size_t n_tiles = (a.batch + S - 1) / S;
  const bool diag = a.diag_sample >= 0;
  for (std::size_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const std::size_t s = diag ? static_cast<std::size_t>(a.diag_sample) : tile * S + tid;
    const bool active = diag ? tid == 0 : s < a.batch;
    const std::size_t col = col0 + tid;
    if (active) {
      RowAcc<T> acc{V, G, ld, col, a.UV, a.idx, a.batch, s, a.sg, a.cand, nullptr, nullptr, nullptr, a.err_key};
      for (std::uint32_t z = 0; z < a.n_zero; ++z) G[std::size_t(a.zero_rows[z]) * ld + col] = T(0);
      bool seen_bad = false;
      // ---- forward sweep (topological) ----
      for (std::uint32_t k = 0; k < a.n_fwd; ++k) {
        const Instr in = a.fwd[k];
        T v;
        if (in.kind == tgc::kNode) {
          acc.o = a.opnd + in.opnd;
          bool bad = false;
          T badv = 0;
          v = eval_node<T>(in.op, in.nops, acc.o, in.cst, acc, bad, badv);
          if (bad) {
            record_error(a.err_key, s, in.node);
            if (diag && !seen_bad) { seen_bad = true; *a.err_op = in.op; *a.err_val = static_cast<double>(badv); }
          }
        } else if (in.kind == tgc::kInputLoad) {
          v = a.inputs[std::size_t(in.aux) * a.batch + s];
        } else if (in.kind == tgc::kAttn) {
          attn_fwd_sample<T>(a.attn[in.aux], a.arows, V, ld, col);
          continue;
        } else if (in.kind == tgc::kLNorm) {
          const tgc::LNorm L = a.lnorm[in.aux];
          if (ln_fwd_sample<T>(L, a.lnrows, a.UV, V, ld, col)) {
            record_error(a.err_key, s, L.rstd_node);
            if (diag && !seen_bad) {
              seen_bad = true;
              *a.err_op = 11;   // invSqrt
              T mu, ve;
              ln_stats<T>(L, a.lnrows, V, ld, col, mu, ve);
              *a.err_val = static_cast<double>(ve);
            }
          }
          continue;
        } else if (in.kind == tgc::kDense) {  // dense layer: z_j = b_j + <x, W[j]>, h_j = act(z_j)
          const tgc::Dense D = a.dense[in.aux];
          const std::uint32_t* xo = a.opnd + D.x_opnd;
          for (std::uint32_t j = 0; j < D.n_out; ++j) {
            T z = D.b_uv != tgc::kNone ? a.UV[D.b_uv + j] : T(0);
            const T* w = a.UV + D.w_uv + std::size_t(j) * D.n_in;
            for (std::uint32_t q = 0; q < D.n_in; ++q) z += V[std::size_t(xo[q] & kIndexMask) * ld + col] * w[q];
            V[std::size_t(D.out_row + j) * ld + col] = z;
            if (D.act_op) V[std::size_t(D.act_row + j) * ld + col] = act_fwd<T>(D.act_op, z);
          }
          continue;
        } else {  // kGatherLoad: embedding row element selected by a token id
          const GatherTable t = a.ug[in.aux];
          std::int32_t r = a.idx[std::size_t(t.col) * a.batch + s];
          if (r < 0 || static_cast<std::uint32_t>(r) >= t.n_rows) { record_error(a.err_key, s, 0xfffffffeu); r = 0; }
          v = a.UV[a.cand[t.cand_off + r]];
        }
        V[std::size_t(in.out) * ld + col] = v;
      }
      if (a.root_row != tgc::kNone) {
        if (a.loss) a.loss[s] = V[std::size_t(a.root_row) * ld + col];
        G[std::size_t(a.root_row) * ld + col] = T(1);  // seed overwrites (backprop.hpp:178)
      }
      // ---- reverse sweep (reference processing order) ----
      for (std::uint32_t k = 0; k < a.n_bwd; ++k) {
        const Instr in = a.bwd[k];
        if (in.kind == tgc::kAttn) {
          attn_bwd_sample<T>(a.attn[in.aux], a.arows, V, G, ld, col);
          continue;
        }
        if (in.kind == tgc::kLNorm) {
          ln_bwd_sample<T>(a.lnorm[in.aux], a.lnrows, a.lnflag, a.UV, V, G, ld, col);
          continue;
        }
        if (in.kind == tgc::kDense) {
          const tgc::Dense D = a.dense[in.aux];
          if (D.act_op)
            for (std::uint32_t j = 0; j < D.n_out; ++j) {
              const std::size_t hr = std::size_t(D.act_row + j) * ld + col, zr = std::size_t(D.out_row + j) * ld + col;
              G[zr] = act_bwd<T>(D.act_op, G[hr], V[hr], V[zr]);
            }
          const std::uint32_t* xo = a.opnd + D.x_opnd;
          const std::uint8_t* xf = a.oflag + D.x_opnd;
          for (std::uint32_t q = 0; q < D.n_in; ++q) {
            T dx = 0;
            for (std::uint32_t j = 0; j < D.n_out; ++j)
              dx += G[std::size_t(D.out_row + j) * ld + col] * a.UV[D.w_uv + std::size_t(j) * D.n_in + q];
            T* p = &G[std::size_t(xo[q] & kIndexMask) * ld + col];
            *p = (xf[q] & tgc::kAssign) ? dx : *p + dx;
          }
          continue;
        }
        acc.o = a.opnd + in.opnd;
        acc.fl = a.oflag + in.opnd;
        acc.ax = a.oaux + in.opnd;
        const T g = G[std::size_t(in.out) * ld + col];
        const T y = V[std::size_t(in.out) * ld + col];
        propagate<T>(in.op, in.nops, acc.o, in.cst, g, y, acc);
      }
      if (a.igrad)
        for (std::uint32_t c = 0; c < a.n_inputs; ++c) {
          const std::uint32_t r = a.input_rows[c];
          if (r != tgc::kNone) a.igrad[std::size_t(c) * a.batch + s] = G[std::size_t(r) * ld + col];
        }
    }
    if (diag) return;
    __syncthreads();
    // ---- per-tile contraction over the sample axis ----
    const std::size_t valid = min(static_cast<std::size_t>(S), a.batch - tile * S);
    for (std::uint32_t d = tid; d < a.n_dest; d += blockDim.x) {
      T tot = 0;
      for (std::uint32_t q = a.term_off[d]; q < a.term_off[d + 1]; ++q) {
        const Term t = a.terms[q];
        const T* ga = G + std::size_t(t.a) * ld + col0;
        T part = 0;
        if (t.kind == 0) {
          if (t.f == tgc::kNone) {
            for (std::size_t j = 0; j < valid; ++j) part += ga[j];
          } else {
            const T* vf = V + std::size_t(t.f) * ld + col0;
            for (std::size_t j = 0; j < valid; ++j) part += ga[j] * vf[j];
          }
        } else {
          const std::int32_t* ix = a.idx + std::size_t(t.f) * a.batch + tile * S;
          for (std::size_t j = 0; j < valid; ++j) part += ix[j] == t.row ? ga[j] : T(0);
        }
        tot += static_cast<T>(t.coef) * part;
      }
      T* dst = a.partial + std::size_t(d) * gridDim.x + blockIdx.x;   // [dest][cta]
      *dst = (tile == blockIdx.x) ? tot : *dst + tot;
    }
    __syncthreads();
  }
}

// sgd_step: x -= gamma * g / b, in the tape's scalar type.
template <class T>
__global__ void k_gd(T* __restrict__ params, const T* __restrict__ g, std::uint32_t n, T gamma, T b) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) params[i] = params[i] - gamma * g[i] / b;
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------

template <class T>
cudaError_t launch_tape(const MainArgs<T>& a, bool smem, unsigned grid, unsigned block, std::size_t smem_bytes,
                        cudaStream_t st) {
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute(k_tape<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes));
    if (e != cudaSuccess) return e;
    k_tape<T, true><<<grid, block, smem_bytes, st>>>(a);
  } else {
    k_tape<T, false><<<grid, block, 0, st>>>(a);
  }
  return cudaGetLastError();
}
template <class T>
int tape_occupancy(bool smem, unsigned block, std::size_t smem_bytes) {
  int occ = 0;
  if (smem) {
    cudaFuncSetAttribute(k_tape<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tape<T, true>, static_cast<int>(block), smem_bytes);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tape<T, false>, static_cast<int>(block), 0);
  }
  return occ;
}
template <class T>
cudaError_t launch_gd(T* params, const T* g, std::uint32_t n, double gamma, double b, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_gd<T><<<(n + 255) / 256, 256, 0, st>>>(params, g, n, static_cast<T>(gamma), static_cast<T>(b));
  return cudaGetLastError();
}

#define TG_INSTANTIATE(T)                                                                              \
  template cudaError_t launch_tape<T>(const MainArgs<T>&, bool, unsigned, unsigned, std::size_t,       \
                                      cudaStream_t);                                                   \
  template int tape_occupancy<T>(bool, unsigned, std::size_t);                                         \
  template cudaError_t launch_gd<T>(T*, const T*, std::uint32_t, double, double, cudaStream_t);
TG_INSTANTIATE(double)
TG_INSTANTIATE(float)

}  // namespace tgk
