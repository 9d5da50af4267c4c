// tg_staged.cu — kernels of the staged (HBM SoA) execution of large tapes.
//
// * k_tape_range: the tape interpreter over a range of the instruction stream,
//   one thread per sample of the chunk, rows persistent in HBM [row][sample]
//   between stages (same per-node semantics as k_tape, ops.hpp / propagate_node).
// * k_gemm: register-tiled SIMT matrix product for dense layers (kDense):
//     forward  Z = W X + b, H = act(Z)       (bias + activation epilogue)
//     reverse  dX (+)= W^T dZ                 (adjoints of the layer inputs)
//              dW  = dZ X^T  (split-K over the sample axis, fixed-order reduce)
//   inner-product order per output matches the reference's left-to-right sum
//   up to the K-tiling of the contraction.
// * deterministic row sums (bias gradients) and generic batch-term contraction.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "tg_ops.cuh"
#include "tg_devcache.cuh"
#include "tg_staged.cuh"

namespace tgk {

using tgc::GatherTable;
using tgc::Instr;
using tgc::kIndexMask;
using tgc::kModeShift;
using tgc::Term;

namespace {

template <class T>
struct RowAccS {
  T* V;
  T* G;
  std::size_t ld, col;
  const T* __restrict__ UV;
  const std::int32_t* __restrict__ idx;
  std::size_t batch, s;
  const GatherTable* __restrict__ sg;
  const std::uint32_t* __restrict__ cand;
  const std::uint32_t* o;
  const std::uint8_t* fl;
  const std::uint32_t* ax;

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

// One forward instruction for sample s (column col of the chunk rows).
template <class T>
__device__ __forceinline__ void fwd_instr(const RangeArgs<T>& a, RowAccS<T>& acc, std::uint32_t k, std::size_t s,
                                          std::size_t col) {
  T* V = a.V;
  const std::size_t ld = a.ld;
  const Instr in = a.fwd[k];
  T v;
  if (in.kind == tgc::kNode) {
    acc.o = a.opnd + in.opnd;
    bool bad = false;
    T badv = 0;
    v = eval_node<T>(in.op, in.nops, acc.o, in.cst, acc, bad, badv);
    if (bad) record_error(a.err_key, s, in.node);
  } else if (in.kind == tgc::kInputLoad) {
    v = a.inputs[std::size_t(in.aux) * a.batch + s];
  } else if (in.kind == tgc::kAttn) {
    attn_fwd_sample<T>(a.attn[in.aux], a.arows, V, ld, col);
    return;
  } else if (in.kind == tgc::kLNorm) {
    const tgc::LNorm L = a.lnorm[in.aux];
    if (ln_fwd_sample<T>(L, a.lnrows, a.UV, V, ld, col)) record_error(a.err_key, s, L.rstd_node);
    return;
  } else if (in.kind == tgc::kDense) {
    const tgc::Dense D = a.dense[in.aux];
    const std::uint32_t* xo = a.opnd + D.x_opnd;
    for (std::uint32_t j = 0; j < D.n_out; ++j) {
      T z = D.b_uv != tgc::kNone ? a.UV[D.b_uv + j] : T(0);
      const T* w = a.UV + D.w_uv + std::size_t(j) * D.n_in;
      for (std::uint32_t q = 0; q < D.n_in; ++q) z += V[std::size_t(xo[q] & kIndexMask) * ld + col] * w[q];
      V[std::size_t(D.out_row + j) * ld + col] = z;
      if (D.act_op) V[std::size_t(D.act_row + j) * ld + col] = act_fwd<T>(D.act_op, z);
    }
    return;
  } else {
    const GatherTable t = a.ug[in.aux];
    std::int32_t r = a.idx[std::size_t(t.col) * a.batch + s];
    if (r < 0 || static_cast<std::uint32_t>(r) >= t.n_rows) { record_error(a.err_key, s, 0xfffffffeu); r = 0; }
    v = a.UV[a.cand[t.cand_off + r]];
  }
  V[std::size_t(in.out) * ld + col] = v;
}

// One reverse instruction for column col.
template <class T>
__device__ __forceinline__ void bwd_instr(const RangeArgs<T>& a, RowAccS<T>& acc, std::uint32_t k, std::size_t col) {
  T* V = a.V;
  T* G = a.G;
  const std::size_t ld = a.ld;
  const Instr in = a.bwd[k];
  if (in.kind == tgc::kAttn) {
    attn_bwd_sample<T>(a.attn[in.aux], a.arows, V, G, ld, col);
    return;
  }
  if (in.kind == tgc::kLNorm) {
    ln_bwd_sample<T>(a.lnorm[in.aux], a.lnrows, a.lnflag, a.UV, V, G, ld, col);
    return;
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
    return;
  }
  acc.o = a.opnd + in.opnd;
  acc.fl = a.oflag + in.opnd;
  acc.ax = a.oaux + in.opnd;
  const T g = G[std::size_t(in.out) * ld + col];
  const T y = V[std::size_t(in.out) * ld + col];
  propagate<T>(in.op, in.nops, acc.o, in.cst, g, y, acc);
}

template <class T>
__global__ void __launch_bounds__(128) k_tape_range(RangeArgs<T> a) {
  const std::size_t col = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (col >= a.n) return;
  const std::size_t s = a.s0 + col;
  T* V = a.V;
  T* G = a.G;
  const std::size_t ld = a.ld;
  RowAccS<T> acc{V, G, ld, col, a.UV, a.idx, a.batch, s, a.sg, a.cand, nullptr, nullptr, nullptr};
  if (a.flags & kRFwd)
    for (std::uint32_t k = a.fwd_begin; k < a.fwd_end; ++k) fwd_instr(a, acc, k, s, col);
  if (a.flags & kRSeed) {
    for (std::uint32_t z = 0; z < a.n_zero; ++z) G[std::size_t(a.zero_rows[z]) * ld + col] = T(0);
    if (a.loss) a.loss[s] = V[std::size_t(a.root_row) * ld + col];
    G[std::size_t(a.root_row) * ld + col] = T(1);
  }
  if (a.flags & kRBwd)
    for (std::uint32_t k = a.bwd_begin; k < a.bwd_end; ++k) bwd_instr(a, acc, k, col);
  if ((a.flags & kROut) && a.igrad)
    for (std::uint32_t c = 0; c < a.n_inputs; ++c) {
      const std::uint32_t r = a.input_rows[c];
      if (r != tgc::kNone) a.igrad[std::size_t(c) * a.batch + s] = G[std::size_t(r) * ld + col];
    }
}

// One dependency level: instruction begin + blockIdx.x for the 128 samples of
// blockIdx.y (instructions of a level are independent; in the reverse sweep no
// two of them push into the same adjoint row).
template <class T>
__global__ void __launch_bounds__(128) k_level_range(RangeArgs<T> a) {
  const std::size_t col = std::size_t(blockIdx.y) * blockDim.x + threadIdx.x;
  if (col >= a.n) return;
  const std::size_t s = a.s0 + col;
  RowAccS<T> acc{a.V, a.G, a.ld, col, a.UV, a.idx, a.batch, s, a.sg, a.cand, nullptr, nullptr, nullptr};
  if (a.flags & kRFwd) fwd_instr(a, acc, a.fwd_begin + blockIdx.x, s, col);
  else bwd_instr(a, acc, a.bwd_begin + blockIdx.x, col);
}

// ---- fp32 levels, four consecutive samples per thread ------------------------
// The scalar level kernel keeps one 4-byte load in flight per thread behind
// the operand decode, and launches one 128-thread CTA per instruction and 128
// samples: at ~8k samples a level of 4k elementwise nodes ran at a third of the
// HBM bandwidth (ncu: long-scoreboard bound, 500 instructions per thread).
// Here a thread moves float4s (4 samples) for every slot operand and a CTA
// walks kLvInstr instructions; the node math stays the scalar eval_node /
// propagate per lane (same operations, same order, same domain checks), or an
// explicit lane loop for the many-operand sums and inner products.  Partial
// groups of four (chunk tail) take the scalar path.
constexpr int kLvInstr = 4;   // instructions per CTA on large levels

struct L4 {
  float v[4];
};
__device__ __forceinline__ L4 ld4(const float* p) {
  const float4 q = *reinterpret_cast<const float4*>(p);
  return L4{{q.x, q.y, q.z, q.w}};
}
__device__ __forceinline__ void st4(float* p, const L4& x) {
  *reinterpret_cast<float4*>(p) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
}

// operand accessor of one lane for nodes of at most two operands
struct Pre2 {
  std::uint32_t o0, o1;
  float v0, v1;
  float pv[2];
  bool pushed[2];
  __device__ __forceinline__ float val(std::uint32_t op) const { return op == o0 ? v0 : v1; }
  __device__ __forceinline__ void push(std::uint32_t k, float v) {
    pv[k] = v;
    pushed[k] = true;
  }
};

struct Lv4 {
  const RangeArgs<float>& a;
  std::size_t col, s;
  __device__ __forceinline__ std::uint32_t sg_row(std::uint32_t i, int l) const {
    const GatherTable t = a.sg[i];
    std::int32_t r = a.idx[std::size_t(t.col) * a.batch + s + l];
    if (r < 0 || static_cast<std::uint32_t>(r) >= t.n_rows) r = 0;
    return a.cand[t.cand_off + r];
  }
  __device__ __forceinline__ L4 val(std::uint32_t op) const {
    const std::uint32_t m = op >> kModeShift, i = op & kIndexMask;
    if (m == tgc::kSlot) return ld4(a.V + std::size_t(i) * a.ld + col);
    if (m == tgc::kUv) {
      const float u = a.UV[i];
      return L4{{u, u, u, u}};
    }
    L4 r;
#pragma unroll
    for (int l = 0; l < 4; ++l) r.v[l] = a.V[std::size_t(sg_row(i, l)) * a.ld + col + l];
    return r;
  }
  // reverse push of operand position pos (operand code, flags and aux row of the instruction)
  __device__ __forceinline__ void push(std::uint32_t pos, const L4& x) const {
    const std::uint32_t op = a.opnd[pos], m = op >> kModeShift, i = op & kIndexMask;
    const std::uint8_t f = a.oflag[pos];
    if (f & tgc::kToAux) {
      st4(a.G + std::size_t(a.oaux[pos]) * a.ld + col, x);
    } else if (m == tgc::kSlot) {
      float* p = a.G + std::size_t(i) * a.ld + col;
      if (f & tgc::kAssign) {
        st4(p, x);
      } else {
        L4 c = ld4(p);
#pragma unroll
        for (int l = 0; l < 4; ++l) c.v[l] += x.v[l];
        st4(p, c);
      }
    } else if (m == tgc::kSGather) {
#pragma unroll
      for (int l = 0; l < 4; ++l) a.G[std::size_t(sg_row(i, l)) * a.ld + col + l] += x.v[l];
    }
  }
};

// Layer norm of four consecutive samples (ln_fwd_sample / ln_bwd_sample, one float4 per row).
__device__ void ln_fwd4(const RangeArgs<float>& a, const tgc::LNorm& L, std::size_t col, std::size_t s,
                        std::uint32_t node_err) {
  const std::uint32_t* lr = a.lnrows;
  L4 s1{{0.f, 0.f, 0.f, 0.f}}, s2{{0.f, 0.f, 0.f, 0.f}};
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const L4 x = ld4(a.V + std::size_t(lr[L.off + i]) * a.ld + col);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      s1.v[l] += x.v[l];
      s2.v[l] += x.v[l] * x.v[l];
    }
  }
  L4 mu, rstd;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    mu.v[l] = s1.v[l] / static_cast<float>(L.n);
    const float ve = (s2.v[l] / static_cast<float>(L.n) - mu.v[l] * mu.v[l]) + static_cast<float>(L.eps);
    if (!(ve > 0.f)) record_error(a.err_key, s + l, node_err);
    rstd.v[l] = 1.f / d_sqrt(ve);
  }
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const L4 x = ld4(a.V + std::size_t(lr[L.off + i]) * a.ld + col);
    const float gm = a.UV[lr[L.off + 3 * L.n + i]], bt = a.UV[lr[L.off + 4 * L.n + i]];
    L4 nv, y;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      nv.v[l] = (x.v[l] - mu.v[l]) * rstd.v[l];
      y.v[l] = nv.v[l] * gm + bt;
    }
    st4(a.V + std::size_t(lr[L.off + L.n + i]) * a.ld + col, nv);
    st4(a.V + std::size_t(lr[L.off + 2 * L.n + i]) * a.ld + col, y);
  }
}

__device__ void ln_bwd4(const RangeArgs<float>& a, const tgc::LNorm& L, std::size_t col) {
  const std::uint32_t* lr = a.lnrows;
  L4 s1{{0.f, 0.f, 0.f, 0.f}}, s2{{0.f, 0.f, 0.f, 0.f}};
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const L4 x = ld4(a.V + std::size_t(lr[L.off + i]) * a.ld + col);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      s1.v[l] += x.v[l];
      s2.v[l] += x.v[l] * x.v[l];
    }
  }
  L4 mu, ve, rstd, drstd{{0.f, 0.f, 0.f, 0.f}}, sdc{{0.f, 0.f, 0.f, 0.f}};
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    mu.v[l] = s1.v[l] / static_cast<float>(L.n);
    ve.v[l] = (s2.v[l] / static_cast<float>(L.n) - mu.v[l] * mu.v[l]) + static_cast<float>(L.eps);
    rstd.v[l] = 1.f / d_sqrt(ve.v[l]);
  }
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const L4 dy = ld4(a.G + std::size_t(lr[L.off + 2 * L.n + i]) * a.ld + col);
    const L4 x = ld4(a.V + std::size_t(lr[L.off + i]) * a.ld + col);
    const float gm = a.UV[lr[L.off + 3 * L.n + i]];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const float dn = dy.v[l] * gm;
      drstd.v[l] += dn * (x.v[l] - mu.v[l]);
      sdc.v[l] += dn * rstd.v[l];
    }
  }
  L4 cx, cm;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const float dve = -drstd.v[l] * rstd.v[l] / (2.f * ve.v[l]);
    const float dmu = -sdc.v[l] + (-dve) * 2.f * mu.v[l];
    cx.v[l] = dve * 2.f / static_cast<float>(L.n);
    cm.v[l] = dmu / static_cast<float>(L.n);
  }
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const L4 dy = ld4(a.G + std::size_t(lr[L.off + 2 * L.n + i]) * a.ld + col);
    const L4 x = ld4(a.V + std::size_t(lr[L.off + i]) * a.ld + col);
    const float gm = a.UV[lr[L.off + 3 * L.n + i]];
    float* p = a.G + std::size_t(lr[L.off + i]) * a.ld + col;
    L4 dx;
#pragma unroll
    for (int l = 0; l < 4; ++l) dx.v[l] = dy.v[l] * gm * rstd.v[l] + cx.v[l] * x.v[l] + cm.v[l];
    if (!(a.lnflag[L.flag_off + i] & tgc::kAssign)) {
      const L4 c = ld4(p);
#pragma unroll
      for (int l = 0; l < 4; ++l) dx.v[l] += c.v[l];
    }
    st4(p, dx);
  }
}

__device__ __forceinline__ bool many_operand_op(std::uint8_t op) {
  return op == AddVarying || op == MeanVarying || op == NegativeMeanVarying || op == SubVarying ||
         op == SumOfSquaresVarying || op == MeanSquaresVarying || op == InnerProductNoBias ||
         op == InnerProductWithBias || op == StopGradMax;
}

__device__ void fwd_instr4(const RangeArgs<float>& a, std::uint32_t k, std::size_t col, std::size_t s) {
  const Instr in = a.fwd[k];
  Lv4 L{a, col, s};
  L4 out;
  if (in.kind == tgc::kLNorm) {
    ln_fwd4(a, a.lnorm[in.aux], col, s, a.lnorm[in.aux].rstd_node);
    return;
  }
  if (in.kind == tgc::kInputLoad) {
    const float* src = a.inputs + std::size_t(in.aux) * a.batch + s;
    if ((reinterpret_cast<std::uintptr_t>(src) & 15) == 0) {
      out = ld4(src);
    } else {
#pragma unroll
      for (int l = 0; l < 4; ++l) out.v[l] = src[l];
    }
  } else if (in.kind == tgc::kNode && in.nops <= 2 && !many_operand_op(in.op)) {
    const std::uint32_t* o = a.opnd + in.opnd;
    const std::uint32_t o1 = in.nops > 1 ? o[1] : o[0];
    const L4 x0 = L.val(o[0]), x1 = in.nops > 1 ? L.val(o1) : x0;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      Pre2 p{o[0], o1, x0.v[l], x1.v[l], {0.f, 0.f}, {false, false}};
      bool bad = false;
      float badv = 0;
      out.v[l] = eval_node<float>(in.op, in.nops, o, in.cst, p, bad, badv);
      if (bad) record_error(a.err_key, s + l, in.node);
    }
  } else if (in.kind == tgc::kNode && many_operand_op(in.op)) {
    const std::uint32_t* o = a.opnd + in.opnd;
    const std::uint32_t n = in.nops;
    const std::uint8_t op = in.op;
    if (op == InnerProductNoBias || op == InnerProductWithBias) {
      const std::uint32_t m = op == InnerProductWithBias ? (n - 1) / 2 : n / 2;
      L4 acc = op == InnerProductWithBias ? L.val(o[n - 1]) : L4{{0.f, 0.f, 0.f, 0.f}};
      for (std::uint32_t j = 0; j < m; ++j) {
        const L4 x = L.val(o[j]), y = L.val(o[m + j]);
#pragma unroll
        for (int l = 0; l < 4; ++l) acc.v[l] += x.v[l] * y.v[l];
      }
      out = acc;
    } else if (op == StopGradMax) {
      out = L.val(o[0]);
      for (std::uint32_t j = 1; j < n; ++j) {
        const L4 x = L.val(o[j]);
#pragma unroll
        for (int l = 0; l < 4; ++l) out.v[l] = x.v[l] > out.v[l] ? x.v[l] : out.v[l];
      }
    } else if (op == SubVarying) {
      out = L.val(o[0]);
      for (std::uint32_t j = 1; j < n; ++j) {
        const L4 x = L.val(o[j]);
#pragma unroll
        for (int l = 0; l < 4; ++l) out.v[l] -= x.v[l];
      }
    } else {   // sums (of squares), left to right, then the mean scaling of eval_node
      const bool sq = op == SumOfSquaresVarying || op == MeanSquaresVarying;
      L4 acc{{0.f, 0.f, 0.f, 0.f}};
      std::uint32_t j = 0;
      for (; j + 4 <= n; j += 4) {
        L4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = L.val(o[j + u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int l = 0; l < 4; ++l) acc.v[l] += sq ? x[u].v[l] * x[u].v[l] : x[u].v[l];
      }
      for (; j < n; ++j) {
        const L4 x = L.val(o[j]);
#pragma unroll
        for (int l = 0; l < 4; ++l) acc.v[l] += sq ? x.v[l] * x.v[l] : x.v[l];
      }
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if (op == MeanVarying || op == MeanSquaresVarying) acc.v[l] /= static_cast<float>(n);
        if (op == NegativeMeanVarying) acc.v[l] = -acc.v[l] / static_cast<float>(n);
      }
      out = acc;
    }
  } else {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      RowAccS<float> acc{a.V, a.G, a.ld, col + l, a.UV, a.idx, a.batch, s + l, a.sg, a.cand, nullptr, nullptr, nullptr};
      fwd_instr(a, acc, k, s + l, col + l);
    }
    return;
  }
  st4(a.V + std::size_t(in.out) * a.ld + col, out);
}

__device__ void bwd_instr4(const RangeArgs<float>& a, std::uint32_t k, std::size_t col, std::size_t s) {
  const Instr in = a.bwd[k];
  if (in.kind == tgc::kLNorm) {
    ln_bwd4(a, a.lnorm[in.aux], col);
    return;
  }
  if (in.kind != tgc::kNode || !(many_operand_op(in.op) || in.nops <= 2) || in.op == StopGradMax) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      RowAccS<float> acc{a.V, a.G, a.ld, col + l, a.UV, a.idx, a.batch, s + l, a.sg, a.cand, nullptr, nullptr, nullptr};
      bwd_instr(a, acc, k, col + l);
    }
    return;
  }
  Lv4 L{a, col, s};
  const std::uint32_t* o = a.opnd + in.opnd;
  const std::uint32_t n = in.nops, p0 = in.opnd;
  const std::uint8_t op = in.op;
  const L4 g = ld4(a.G + std::size_t(in.out) * a.ld + col);
  if (!many_operand_op(op)) {
    const L4 y = ld4(a.V + std::size_t(in.out) * a.ld + col);
    const std::uint32_t o1 = n > 1 ? o[1] : o[0];
    const L4 x0 = L.val(o[0]), x1 = n > 1 ? L.val(o1) : x0;
    L4 pv[2];
    bool any[2] = {false, false};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      Pre2 p{o[0], o1, x0.v[l], x1.v[l], {0.f, 0.f}, {false, false}};
      propagate<float>(op, n, o, in.cst, g.v[l], y.v[l], p);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        pv[q].v[l] = p.pv[q];
        any[q] = any[q] || p.pushed[q];
      }
    }
    if (any[0]) L.push(p0, pv[0]);
    if (n > 1 && any[1]) L.push(p0 + 1, pv[1]);
    return;
  }
  auto scaled = [&](float c) {
    L4 r;
#pragma unroll
    for (int l = 0; l < 4; ++l) r.v[l] = g.v[l] * c;
    return r;
  };
  if (op == AddVarying) {
    for (std::uint32_t j = 0; j < n; ++j) L.push(p0 + j, g);
  } else if (op == SubVarying) {
    L.push(p0, g);
    const L4 ng = scaled(-1.f);
    for (std::uint32_t j = 1; j < n; ++j) L.push(p0 + j, ng);
  } else if (op == MeanVarying || op == NegativeMeanVarying) {
    L4 dd;
#pragma unroll
    for (int l = 0; l < 4; ++l) dd.v[l] = (op == MeanVarying ? g.v[l] : -g.v[l]) / static_cast<float>(n);
    for (std::uint32_t j = 0; j < n; ++j) L.push(p0 + j, dd);
  } else if (op == SumOfSquaresVarying || op == MeanSquaresVarying) {
    L4 sc;
#pragma unroll
    for (int l = 0; l < 4; ++l)
      sc.v[l] = op == SumOfSquaresVarying ? g.v[l] * 2.f : g.v[l] * 2.f / static_cast<float>(n);
    for (std::uint32_t j = 0; j < n; ++j) {
      const L4 x = L.val(o[j]);
      L4 r;
#pragma unroll
      for (int l = 0; l < 4; ++l) r.v[l] = op == SumOfSquaresVarying ? g.v[l] * 2.f * x.v[l] : sc.v[l] * x.v[l];
      L.push(p0 + j, r);
    }
  } else {   // inner products: x and y adjoints interleaved as in propagate (ops.hpp:436-452)
    const std::uint32_t m = op == InnerProductWithBias ? (n - 1) / 2 : n / 2;
    for (std::uint32_t j = 0; j < m; ++j) {
      const L4 x = L.val(o[j]), y = L.val(o[m + j]);
      L4 gx, gy;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        gx.v[l] = g.v[l] * y.v[l];
        gy.v[l] = g.v[l] * x.v[l];
      }
      L.push(p0 + j, gx);
      L.push(p0 + m + j, gy);
    }
    if (op == InnerProductWithBias) L.push(p0 + n - 1, g);
  }
}

__device__ void level_instr1(const RangeArgs<float>& a, bool fwd, std::uint32_t k, std::size_t c) {
  RowAccS<float> acc{a.V, a.G, a.ld, c, a.UV, a.idx, a.batch, a.s0 + c, a.sg, a.cand, nullptr, nullptr, nullptr};
  if (fwd) fwd_instr(a, acc, k, a.s0 + c, c);
  else bwd_instr(a, acc, k, c);
}

__global__ void __launch_bounds__(128) k_level_range4(RangeArgs<float> a, std::uint32_t ipc) {
  const std::size_t col = (std::size_t(blockIdx.y) * blockDim.x + threadIdx.x) * 4;
  if (col >= a.n) return;
  const std::size_t s = a.s0 + col;
  const bool fwd = a.flags & kRFwd;
  const std::uint32_t begin = fwd ? a.fwd_begin : a.bwd_begin, end = fwd ? a.fwd_end : a.bwd_end;
  const std::uint32_t k0 = begin + blockIdx.x * ipc, k1 = min(end, k0 + ipc);
  if (col + 4 <= a.n) {
    for (std::uint32_t k = k0; k < k1; ++k) {
      if (fwd) fwd_instr4(a, k, col, s);
      else bwd_instr4(a, k, col, s);
    }
    return;
  }
  for (std::size_t c = col; c < a.n; ++c)   // chunk tail
    for (std::uint32_t k = k0; k < k1; ++k) level_instr1(a, fwd, k, c);
}

// Sums of the contended rows of one reverse level (entry blockIdx.x, 128
// samples per CTA row): the temporaries in execution order after the row's
// earlier value, so the result does not depend on scheduling.
template <class T>
__global__ void __launch_bounds__(128) k_row_sums(const uint4* __restrict__ ent, T* G, std::size_t n, std::size_t ld) {
  const std::size_t col = std::size_t(blockIdx.y) * blockDim.x + threadIdx.x;
  if (col >= n) return;
  const uint4 e = ent[blockIdx.x];
  T v = (e.y & 1u) ? T(0) : G[std::size_t(e.x) * ld + col];
  std::uint32_t i = 0;
  for (; i + 4 <= e.w; i += 4) {
    T x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = G[std::size_t(e.z + i + u) * ld + col];
#pragma unroll
    for (int u = 0; u < 4; ++u) v += x[u];
  }
  for (; i < e.w; ++i) v += G[std::size_t(e.z + i) * ld + col];
  G[std::size_t(e.x) * ld + col] = v;
}

// ---- register-tiled SIMT GEMM ------------------------------------------------
template <class T> struct GemmTile;
template <> struct GemmTile<float> { static constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8; };
template <> struct GemmTile<double> { static constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4; };

template <class T, bool AK, bool BN_>
__global__ void __launch_bounds__(256) k_gemm(GemmArgs<T> g) {
  constexpr int BM = GemmTile<T>::BM, BN = GemmTile<T>::BN, BK = GemmTile<T>::BK;
  constexpr int TM = GemmTile<T>::TM, TN = GemmTile<T>::TN;
  __shared__ T As[2][BK][BM + 4];
  __shared__ T Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const std::uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  std::uint32_t k_begin = 0, k_end = g.K;
  if (g.epi == kEpiSplitK) {
    k_begin = blockIdx.z * g.k_chunk;
    k_end = min(g.K, k_begin + g.k_chunk);
  }
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  constexpr int A_PER = BM * BK / 256, B_PER = BN * BK / 256;
  T ra[A_PER], rb[B_PER];
  auto load = [&](std::uint32_t k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int li = tid + e * 256;
      int mm, kk;
      if (AK) { kk = li % BK; mm = li / BK; } else { mm = li % BM; kk = li / BM; }
      const std::uint32_t gm = m0 + mm, gk = k0 + kk;
      ra[e] = (gm < g.M && gk < k_end) ? (AK ? g.A[std::size_t(gm) * g.lda + gk] : g.A[std::size_t(gk) * g.lda + gm]) : T(0);
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int li = tid + e * 256;
      int nn, kk;
      if (BN_) { nn = li % BN; kk = li / BN; } else { kk = li % BK; nn = li / BK; }
      const std::uint32_t gn = n0 + nn, gk = k0 + kk;
      rb[e] = (gn < g.N && gk < k_end) ? (BN_ ? g.B[std::size_t(gk) * g.ldb + gn] : g.B[std::size_t(gn) * g.ldb + gk]) : T(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int li = tid + e * 256;
      int mm, kk;
      if (AK) { kk = li % BK; mm = li / BK; } else { mm = li % BM; kk = li / BM; }
      As[buf][kk][mm] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int li = tid + e * 256;
      int nn, kk;
      if (BN_) { nn = li % BN; kk = li / BN; } else { kk = li % BK; nn = li / BK; }
      Bs[buf][kk][nn] = rb[e];
    }
  };
  int buf = 0;
  load(k_begin);
  store(0);
  __syncthreads();
  for (std::uint32_t k0 = k_begin; k0 < k_end; k0 += BK) {
    const bool more = k0 + BK < k_end;
    if (more) load(k0 + BK);   // next tile in flight while this one is consumed
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] += a[i] * b[j];
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const std::uint32_t m = m0 + ty * TM + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const std::uint32_t n = n0 + tx * TN + j;
      if (n >= g.N) continue;
      if (g.epi == kEpiBiasAct) {
        const T z = (g.bias ? g.bias[m] : T(0)) + acc[i][j];
        if (!(g.no_z && g.act)) g.C[std::size_t(m) * g.ldc + n] = z;
        if (g.act) g.C2[std::size_t(m) * g.ldc + n] = act_fwd<T>(g.act, z);
      } else if (g.epi == kEpiAccum) {
        T* p = &g.C[std::size_t(m) * g.ldc + n];
        if (g.dact) *p = act_bwd_h<T>(g.dact, acc[i][j], g.C2[std::size_t(m) * g.ldc + n]);
        else *p = g.beta ? *p + acc[i][j] : acc[i][j];
      } else {
        g.C[(std::size_t(blockIdx.z) * g.M + m) * g.N + n] = acc[i][j];
      }
    }
  }
}

template <class T>
__global__ void k_splitk_reduce(const T* __restrict__ part, T* __restrict__ dst, std::uint32_t MN, std::uint32_t splits) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MN) return;
  // 8 partials in flight (batched weight gradients sum hundreds), summed in slice order
  T t = 0;
  std::uint32_t z = 0;
  for (; z + 8 <= splits; z += 8) {
    T x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = part[std::size_t(z + u) * MN + i];
#pragma unroll
    for (int u = 0; u < 8; ++u) t += x[u];
  }
  for (; z < splits; ++z) t += part[std::size_t(z) * MN + i];
  dst[i] += t;
}

template <class T>
__global__ void k_act_bwd(T* G, const T* V, std::uint32_t z_row, std::uint32_t h_row, std::size_t n, std::size_t ld,
                          std::uint32_t act, const uint4* mem) {
  const std::size_t s = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if (mem) {   // batch member blockIdx.z
    const uint4 e = mem[blockIdx.z];
    z_row = e.z;
    h_row = e.w;
  }
  const std::size_t zr = std::size_t(z_row + blockIdx.y) * ld + s, hr = std::size_t(h_row + blockIdx.y) * ld + s;
  // tanh / sigmoid / exp derivatives use the output only: skip the z read (a quarter of the bytes)
  // relu: z > 0 exactly when h = relu(z) > 0 (NaN z gives h = 0), so the mask comes from h
  const bool need_z = act == Sqr || act == Cub;
  const T h = V[hr];
  G[zr] = act == Relu ? (h > T(0) ? G[hr] : T(0)) : act_bwd<T>(act, G[hr], h, need_z ? V[zr] : T(0));
}

template <class T>
__global__ void __launch_bounds__(256) k_rowsum(const T* G, std::uint32_t row0, std::size_t n, std::size_t ld, T* dst,
                                                const uint4* mem, std::uint32_t n_mem) {
  __shared__ T red[256];
  // 8 loads in flight per thread, summed in sequential order (deterministic);
  // batched: the members' rows one after another
  T t = 0;
  for (std::uint32_t p = 0; p < n_mem; ++p) {
    const T* row = G + std::size_t((mem ? mem[p].z : row0) + blockIdx.x) * ld;
    std::size_t s = threadIdx.x;
    for (; s + 7 * 256 < n; s += 8 * 256) {
      T x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = row[s + u * 256];
#pragma unroll
      for (int u = 0; u < 8; ++u) t += x[u];
    }
    for (; s < n; s += 256) t += row[s];
  }
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) dst[blockIdx.x] += red[0];
}

// Two-pass form of the bias row sums for many samples: CTA (row, chunk c) sums
// the c-th contiguous share of the (member, sample) sequence of a row, then
// k_rowsum_fin adds the shares in chunk order (deterministic; one CTA per row
// had left most SMs idle when a layer has 64 rows).
template <class T>
__global__ void __launch_bounds__(256) k_rowsum_part(const T* G, std::size_t n, std::size_t ld, const uint4* mem,
                                                     std::uint32_t n_mem, std::size_t per, T* part) {
  __shared__ T red[256];
  const std::size_t total = std::size_t(n_mem) * n;
  const std::size_t b = std::size_t(blockIdx.y) * per, e = min(total, b + per);
  T t = 0;
  std::size_t q = b;
  while (q < e) {   // runs of one member's row
    const std::uint32_t p = static_cast<std::uint32_t>(q / n);
    const std::size_t s0 = q % n, s1 = min(n, s0 + (e - q));
    const T* row = G + std::size_t(mem[p].z + blockIdx.x) * ld;
    std::size_t s = s0 + threadIdx.x;
    for (; s + 7 * 256 < s1; s += 8 * 256) {
      T x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = row[s + u * 256];
#pragma unroll
      for (int u = 0; u < 8; ++u) t += x[u];
    }
    for (; s < s1; s += 256) t += row[s];
    q += s1 - s0;
  }
  red[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[std::size_t(blockIdx.x) * gridDim.y + blockIdx.y] = red[0];
}

template <class T>
__global__ void k_rowsum_fin(const T* part, std::uint32_t rows, std::uint32_t chunks, T* dst) {
  const std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  T t = 0;
  for (std::uint32_t c = 0; c < chunks; ++c) t += part[std::size_t(j) * chunks + c];
  dst[j] += t;
}

template <class T>
__global__ void k_zero_rows(T* X, const std::uint32_t* rows, std::size_t n, std::size_t ld) {
  const std::size_t s = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) X[std::size_t(rows[blockIdx.y]) * ld + s] = T(0);
}

template <class T>
__global__ void __launch_bounds__(256) k_contract(const std::uint32_t* dests, const std::uint32_t* term_off, const Term* terms,
                                                  const T* G, const T* V, const std::int32_t* idx, std::size_t batch,
                                                  std::size_t s0, std::size_t n, std::size_t ld, T* acc) {
  __shared__ T red[256];
  const std::uint32_t d = dests[blockIdx.x];
  T tot = 0;
  for (std::uint32_t q = term_off[d]; q < term_off[d + 1]; ++q) {
    const Term t = terms[q];
    const T* ga = G + std::size_t(t.a) * ld;
    T part = 0;
    if (t.kind == 0) {
      if (t.f == tgc::kNone) {
        for (std::size_t s = threadIdx.x; s < n; s += 256) part += ga[s];
      } else {
        const T* vf = V + std::size_t(t.f) * ld;
        for (std::size_t s = threadIdx.x; s < n; s += 256) part += ga[s] * vf[s];
      }
    } else {
      const std::int32_t* ix = idx + std::size_t(t.f) * batch + s0;
      for (std::size_t s = threadIdx.x; s < n; s += 256) part += ix[s] == t.row ? ga[s] : T(0);
    }
    tot += static_cast<T>(t.coef) * part;
  }
  red[threadIdx.x] = tot;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[d] += red[0];
}

// Table-scatter contraction as histograms (cfg3 / cfg4 embedding gradients).
// Group g = (adjoint row a, index column f, rows R): H_g[r] = sum_s [idx[f][s]
// == r] G[a][s].  Every thread accumulates its samples (in order) into its own
// shared-memory column bins[r][thread]; each bin row is then reduced in a
// fixed order, giving per-chunk partials part[g][chunk][r].  k_contract's
// one-CTA-per-destination scan read every G row once per table row.
template <class T>
__global__ void __launch_bounds__(128) k_scatter_hist(const ScatterGroup* groups, const T* G, const std::int32_t* idx,
                                                       std::size_t batch, std::size_t s0, std::size_t n, std::size_t ld,
                                                       std::uint32_t n_chunks, std::uint32_t r_max, T* part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* bins = reinterpret_cast<T*>(smem_raw);
  const ScatterGroup gp = groups[blockIdx.x];
  const std::uint32_t tid = threadIdx.x, chunk = blockIdx.y;
  for (std::uint32_t r = 0; r < gp.rows; ++r) bins[r * 128 + tid] = T(0);
  const std::size_t lo = n * chunk / n_chunks, hi = n * (chunk + 1) / n_chunks;
  const T* ga = G + std::size_t(gp.a) * ld;
  const std::int32_t* ix = idx + std::size_t(gp.f) * batch + s0;
  for (std::size_t s = lo + tid; s < hi; s += 128) {
    const std::int32_t r = ix[s];
    if (static_cast<std::uint32_t>(r) < gp.rows) bins[r * 128 + tid] += ga[s];
  }
  __syncthreads();
  const std::uint32_t warp = tid >> 5, lane = tid & 31;
  for (std::uint32_t r = warp; r < gp.rows; r += 4) {
    const T* b = bins + r * 128;
    T t = ((b[lane] + b[lane + 32]) + (b[lane + 64] + b[lane + 96]));
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
    if (lane == 0) part[(std::size_t(blockIdx.x) * n_chunks + chunk) * r_max + r] = t;
  }
}

// acc[dest] += sum over the dest's uses (g, r, coef) of coef * sum_chunks part[g][chunk][r]   (fixed order)
template <class T>
__global__ void k_scatter_apply(const ScatterUse* uses, const std::uint32_t* use_off, const std::uint32_t* dests,
                                std::uint32_t n_dests, const T* part, std::uint32_t n_chunks, std::uint32_t r_max, T* acc) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_dests) return;
  T tot = 0;
  for (std::uint32_t u = use_off[i]; u < use_off[i + 1]; ++u) {
    const ScatterUse su = uses[u];
    T h = 0;
    for (std::uint32_t c = 0; c < n_chunks; ++c) h += part[(std::size_t(su.g) * n_chunks + c) * r_max + su.r];
    tot += static_cast<T>(su.coef) * h;
  }
  acc[dests[i]] += tot;
}

}  // namespace

template <class T>
cudaError_t launch_scatter(const ScatterGroup* groups, std::uint32_t n_groups, std::uint32_t r_max, const ScatterUse* uses,
                           const std::uint32_t* use_off, const std::uint32_t* dests, std::uint32_t n_dests, const T* G,
                           const std::int32_t* idx, std::size_t batch, std::size_t s0, std::size_t n, std::size_t ld,
                           T* part, std::uint32_t n_chunks, T* acc, cudaStream_t st) {
  if (n_groups == 0 || n == 0) return cudaSuccess;
  const std::size_t smem = std::size_t(r_max) * 128 * sizeof(T);
  static PerDeviceOnce attr;
  if (smem > 48 * 1024)
    if (const cudaError_t e = attr.ensure([] {
          return cudaFuncSetAttribute(k_scatter_hist<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        }); e != cudaSuccess)
      return e;
  k_scatter_hist<T><<<dim3(n_groups, n_chunks), 128, smem, st>>>(groups, G, idx, batch, s0, n, ld, n_chunks, r_max, part);
  k_scatter_apply<T><<<(n_dests + 127) / 128, 128, 0, st>>>(uses, use_off, dests, n_dests, part, n_chunks, r_max, acc);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_tape_range(const RangeArgs<T>& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  k_tape_range<T><<<static_cast<unsigned>((a.n + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_level_range(const RangeArgs<T>& a, cudaStream_t st) {
  const std::uint32_t count = (a.flags & kRFwd) ? a.fwd_end - a.fwd_begin : a.bwd_end - a.bwd_begin;
  if (a.n == 0 || count == 0) return cudaSuccess;
  if constexpr (std::is_same_v<T, float>) {
    static const bool vec = !(std::getenv("TG_LEVEL4") && std::getenv("TG_LEVEL4")[0] == '0');
    if (vec && !a.per_sample && a.ld % 4 == 0 && (reinterpret_cast<std::uintptr_t>(a.V) & 15) == 0 &&
        (reinterpret_cast<std::uintptr_t>(a.G) & 15) == 0) {
      // instructions per CTA: kLvInstr (one load group) while the launch keeps
      // >= ~16 CTAs per SM, else one (few-instruction levels, e.g. the
      // layer-norm statistics, need the CTAs more than the grouping)
      const std::uint32_t ys = static_cast<std::uint32_t>((a.n + 511) / 512);
      const std::uint32_t ipc = std::uint64_t(count) * ys >= 4ull * 148 * 16 ? kLvInstr : 1;
      k_level_range4<<<dim3((count + ipc - 1) / ipc, ys), 128, 0, st>>>(a, ipc);
      return cudaGetLastError();
    }
  }
  k_level_range<T><<<dim3(count, static_cast<unsigned>((a.n + 127) / 128)), 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_gemm(const GemmArgs<T>& g, std::uint32_t splits, cudaStream_t st) {
  constexpr int BM = GemmTile<T>::BM, BN = GemmTile<T>::BN;
  if (g.M == 0 || g.N == 0) return cudaSuccess;
  const dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, g.epi == kEpiSplitK ? splits : 1);
  if (g.a_kmaj && g.b_nmaj) k_gemm<T, true, true><<<grid, 256, 0, st>>>(g);
  else if (g.a_kmaj && !g.b_nmaj) k_gemm<T, true, false><<<grid, 256, 0, st>>>(g);
  else if (!g.a_kmaj && g.b_nmaj) k_gemm<T, false, true><<<grid, 256, 0, st>>>(g);
  else k_gemm<T, false, false><<<grid, 256, 0, st>>>(g);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_splitk_reduce(const T* part, T* dst, std::uint32_t MN, std::uint32_t splits, cudaStream_t st) {
  k_splitk_reduce<T><<<(MN + 255) / 256, 256, 0, st>>>(part, dst, MN, splits);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_act_bwd(T* G, const T* V, std::uint32_t z_row, std::uint32_t h_row, std::uint32_t n_out, std::size_t n,
                           std::size_t ld, std::uint32_t act, cudaStream_t st) {
  if (n == 0 || n_out == 0) return cudaSuccess;
  k_act_bwd<T><<<dim3(static_cast<unsigned>((n + 255) / 256), n_out), 256, 0, st>>>(G, V, z_row, h_row, n, ld, act, nullptr);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_row_sums(const uint4* ent, std::uint32_t n_ent, T* G, std::size_t n, std::size_t ld, cudaStream_t st) {
  if (n == 0 || n_ent == 0) return cudaSuccess;
  k_row_sums<T><<<dim3(n_ent, static_cast<unsigned>((n + 127) / 128)), 128, 0, st>>>(ent, G, n, ld);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_act_bwd_batched(T* G, const T* V, const uint4* mem, std::uint32_t n_mem, std::uint32_t n_out, std::size_t n,
                                   std::size_t ld, std::uint32_t act, cudaStream_t st) {
  if (n == 0 || n_out == 0 || n_mem == 0) return cudaSuccess;
  k_act_bwd<T><<<dim3(static_cast<unsigned>((n + 255) / 256), n_out, n_mem), 256, 0, st>>>(G, V, 0, 0, n, ld, act, mem);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_rowsum(const T* G, std::uint32_t row0, std::uint32_t rows, std::size_t n, std::size_t ld, T* dst,
                          cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  k_rowsum<T><<<rows, 256, 0, st>>>(G, row0, n, ld, dst, nullptr, 1);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_rowsum_batched(const T* G, const uint4* mem, std::uint32_t n_mem, std::uint32_t rows, std::size_t n,
                                  std::size_t ld, T* dst, T* scratch, std::size_t scratch_elems, cudaStream_t st) {
  if (rows == 0 || n_mem == 0) return cudaSuccess;
  // about four CTAs per SM over all rows, shares of >= 8k elements
  const std::size_t total = std::size_t(n_mem) * n;
  std::size_t chunks = std::max<std::size_t>(1, (592 + rows - 1) / rows);
  chunks = std::min<std::size_t>(chunks, std::max<std::size_t>(1, total / 8192));
  if (scratch) chunks = std::min<std::size_t>(chunks, std::max<std::size_t>(1, scratch_elems / rows));
  if (!scratch || chunks <= 1) {
    k_rowsum<T><<<rows, 256, 0, st>>>(G, 0, n, ld, dst, mem, n_mem);
    return cudaGetLastError();
  }
  const std::size_t per = (total + chunks - 1) / chunks;
  k_rowsum_part<T><<<dim3(rows, static_cast<unsigned>(chunks)), 256, 0, st>>>(G, n, ld, mem, n_mem, per, scratch);
  k_rowsum_fin<T><<<(rows + 127) / 128, 128, 0, st>>>(scratch, rows, static_cast<std::uint32_t>(chunks), dst);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_zero_rows(T* X, const std::uint32_t* rows, std::uint32_t count, std::size_t n, std::size_t ld,
                             cudaStream_t st) {
  if (count == 0 || n == 0) return cudaSuccess;
  k_zero_rows<T><<<dim3(static_cast<unsigned>((n + 255) / 256), count), 256, 0, st>>>(X, rows, n, ld);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_contract(const std::uint32_t* dests, std::uint32_t n_dests, const std::uint32_t* term_off,
                            const Term* terms, const T* G, const T* V, const std::int32_t* idx, std::size_t batch,
                            std::size_t s0, std::size_t n, std::size_t ld, T* acc, cudaStream_t st) {
  if (n_dests == 0) return cudaSuccess;
  k_contract<T><<<n_dests, 256, 0, st>>>(dests, term_off, terms, G, V, idx, batch, s0, n, ld, acc);
  return cudaGetLastError();
}

#define TG_STAGED_INST(T)                                                                                                  \
  template cudaError_t launch_tape_range<T>(const RangeArgs<T>&, cudaStream_t);                                            \
  template cudaError_t launch_level_range<T>(const RangeArgs<T>&, cudaStream_t);                                           \
  template cudaError_t launch_gemm<T>(const GemmArgs<T>&, std::uint32_t, cudaStream_t);                                    \
  template cudaError_t launch_splitk_reduce<T>(const T*, T*, std::uint32_t, std::uint32_t, cudaStream_t);                  \
  template cudaError_t launch_act_bwd<T>(T*, const T*, std::uint32_t, std::uint32_t, std::uint32_t, std::size_t,           \
                                         std::size_t, std::uint32_t, cudaStream_t);                                        \
  template cudaError_t launch_rowsum<T>(const T*, std::uint32_t, std::uint32_t, std::size_t, std::size_t, T*,              \
                                        cudaStream_t);                                                                     \
  template cudaError_t launch_row_sums<T>(const uint4*, std::uint32_t, T*, std::size_t, std::size_t, cudaStream_t);       \
  template cudaError_t launch_act_bwd_batched<T>(T*, const T*, const uint4*, std::uint32_t, std::uint32_t, std::size_t,   \
                                                 std::size_t, std::uint32_t, cudaStream_t);                                \
  template cudaError_t launch_rowsum_batched<T>(const T*, const uint4*, std::uint32_t, std::uint32_t, std::size_t,          \
                                                std::size_t, T*, T*, std::size_t, cudaStream_t);                           \
  template cudaError_t launch_zero_rows<T>(T*, const std::uint32_t*, std::uint32_t, std::size_t, std::size_t,              \
                                           cudaStream_t);                                                                  \
  template cudaError_t launch_contract<T>(const std::uint32_t*, std::uint32_t, const std::uint32_t*, const Term*,          \
                                          const T*, const T*, const std::int32_t*, std::size_t, std::size_t, std::size_t,  \
                                          std::size_t, T*, cudaStream_t);                                                   \
  template cudaError_t launch_scatter<T>(const ScatterGroup*, std::uint32_t, std::uint32_t, const ScatterUse*,             \
                                         const std::uint32_t*, const std::uint32_t*, std::uint32_t, const T*,               \
                                         const std::int32_t*, std::size_t, std::size_t, std::size_t, std::size_t, T*,      \
                                         std::uint32_t, T*, cudaStream_t);
TG_STAGED_INST(float)
TG_STAGED_INST(double)

}  // namespace tgk
