// tg_ops.cuh — per-node forward values and reverse rules on the device.
//
// Forward formulas restate reference ops.hpp:38-307 (same expression shapes:
// bias first then left-to-right products for inner products, division by the
// arity for means); reverse rules restate detail::propagate_node
// (ops.hpp:316-454), including the zero-safe prefix/suffix product of
// reduceMul (ops.hpp:403-417).  The accessor `A` abstracts where operands
// live (per-sample rows in shared memory / HBM, or the sample-invariant table).
#pragma once

#include <cstdint>

#include "../host/tg_program.hpp"
#include "tg_math.cuh"

namespace tgk {

template <class T> __device__ __forceinline__ T d_tanh(T x);
template <> __device__ __forceinline__ double d_tanh(double x) { return tg_tanh(x); }
template <> __device__ __forceinline__ float d_tanh(float x) { return tanhf(x); }
template <class T> __device__ __forceinline__ T d_exp(T x);
template <> __device__ __forceinline__ double d_exp(double x) { return exp(x); }
template <> __device__ __forceinline__ float d_exp(float x) { return expf(x); }
template <class T> __device__ __forceinline__ T d_log(T x);
template <> __device__ __forceinline__ double d_log(double x) { return log(x); }
template <> __device__ __forceinline__ float d_log(float x) { return logf(x); }
template <class T> __device__ __forceinline__ T d_sqrt(T x);
template <> __device__ __forceinline__ double d_sqrt(double x) { return sqrt(x); }
template <> __device__ __forceinline__ float d_sqrt(float x) { return sqrtf(x); }

enum : std::uint8_t {
  Leaf = 0, Relu, Tanh, Exp, NegLog, Sigmoid, Inv, Sqr, Cub, Log, Sqrt, InvSqrt,
  Add, Sub, Mul, MulByConst, Div, Mean, AddSquares, MeanSquares, NegativeMean,
  AddVarying, SubVarying, MulVarying, MeanVarying, SumOfSquaresVarying, MeanSquaresVarying,
  NegativeMeanVarying, InnerProductNoBias, InnerProductWithBias,
  StopGradMax = TG_OP_STOPGRAD_MAX,
};

// Forward value of one node.  `bad` is set (and `badv` records the offending
// input) on a domain violation; the reference throws std::domain_error there
// (ops.hpp:16-32), the device records the first offender per launch.
template <class T, class A>
__device__ __forceinline__ T eval_node(std::uint8_t op, std::uint32_t n, const std::uint32_t* o, double cst,
                                       A& a, bool& bad, T& badv) {
  switch (op) {
    case Relu: { const T v = a.val(o[0]); return v > T(0) ? v : T(0); }
    case Tanh: return d_tanh(a.val(o[0]));
    case Exp: return d_exp(a.val(o[0]));
    case NegLog: { const T v = a.val(o[0]); if (!(v > T(0))) { bad = true; badv = v; } return -d_log(v); }
    case Sigmoid: return T(1) / (T(1) + d_exp(-a.val(o[0])));
    case Inv: { const T v = a.val(o[0]); if (v == T(0)) { bad = true; badv = v; } return T(1) / v; }
    case Sqr: { const T v = a.val(o[0]); return v * v; }
    case Cub: { const T v = a.val(o[0]); return v * v * v; }
    case Log: { const T v = a.val(o[0]); if (!(v > T(0))) { bad = true; badv = v; } return d_log(v); }
    case Sqrt: { const T v = a.val(o[0]); if (!(v > T(0))) { bad = true; badv = v; } return d_sqrt(v); }
    case InvSqrt: { const T v = a.val(o[0]); if (!(v > T(0))) { bad = true; badv = v; } return T(1) / d_sqrt(v); }
    case MulByConst: return a.val(o[0]) * static_cast<T>(cst);
    case Add: return a.val(o[0]) + a.val(o[1]);
    case Sub: return a.val(o[0]) - a.val(o[1]);
    case Mul: return a.val(o[0]) * a.val(o[1]);
    case Div: { const T b = a.val(o[1]); if (b == T(0)) { bad = true; badv = b; } return a.val(o[0]) / b; }
    case Mean: return (a.val(o[0]) + a.val(o[1])) / T(2);
    case AddSquares: { const T x = a.val(o[0]), y = a.val(o[1]); return x * x + y * y; }
    case MeanSquares: { const T x = a.val(o[0]), y = a.val(o[1]); return (x * x + y * y) / T(2); }
    case NegativeMean: return -(a.val(o[0]) + a.val(o[1])) / T(2);
    case AddVarying: case MeanVarying: case NegativeMeanVarying: {
      T acc = 0;
      for (std::uint32_t j = 0; j < n; ++j) acc += a.val(o[j]);
      if (op == MeanVarying) acc /= static_cast<T>(n);
      if (op == NegativeMeanVarying) acc = -acc / static_cast<T>(n);
      return acc;
    }
    case SubVarying: {
      T acc = a.val(o[0]);
      for (std::uint32_t j = 1; j < n; ++j) acc -= a.val(o[j]);
      return acc;
    }
    case MulVarying: {
      T acc = T(1);
      for (std::uint32_t j = 0; j < n; ++j) acc *= a.val(o[j]);
      return acc;
    }
    case SumOfSquaresVarying: case MeanSquaresVarying: {
      T acc = 0;
      for (std::uint32_t j = 0; j < n; ++j) { const T v = a.val(o[j]); acc += v * v; }
      if (op == MeanSquaresVarying) acc /= static_cast<T>(n);
      return acc;
    }
    case InnerProductNoBias: {
      const std::uint32_t m = n / 2;
      T acc = 0;
      for (std::uint32_t j = 0; j < m; ++j) acc += a.val(o[j]) * a.val(o[m + j]);
      return acc;
    }
    case InnerProductWithBias: {
      const std::uint32_t m = (n - 1) / 2;
      T acc = a.val(o[n - 1]);
      for (std::uint32_t j = 0; j < m; ++j) acc += a.val(o[j]) * a.val(o[m + j]);
      return acc;
    }
    case StopGradMax: {
      T m = a.val(o[0]);
      for (std::uint32_t j = 1; j < n; ++j) { const T v = a.val(o[j]); m = v > m ? v : m; }
      return m;
    }
    default: return T(0);
  }
}

// Reverse rule of one node: pushes d(root)/d(child) contributions.
// a.push(k, v) routes contribution v of operand k (by its mode/flags).
template <class T, class A>
__device__ __forceinline__ void propagate(std::uint8_t op, std::uint32_t n, const std::uint32_t* o, double cst,
                                          T g, T y, A& a) {
  switch (op) {
    case Relu: a.push(0, a.val(o[0]) > T(0) ? g : T(0)); break;
    case Tanh: a.push(0, g * (T(1) - y * y)); break;
    case Exp: a.push(0, g * y); break;
    case NegLog: a.push(0, -g / a.val(o[0])); break;
    case Sigmoid: a.push(0, g * y * (T(1) - y)); break;
    case Inv: a.push(0, -g * y * y); break;
    case Sqr: a.push(0, g * T(2) * a.val(o[0])); break;
    case Cub: { const T x = a.val(o[0]); a.push(0, g * T(3) * x * x); break; }
    case Log: a.push(0, g / a.val(o[0])); break;
    case Sqrt: a.push(0, g / (T(2) * y)); break;
    case InvSqrt: a.push(0, -g * y / (T(2) * a.val(o[0]))); break;
    case MulByConst: a.push(0, g * static_cast<T>(cst)); break;
    case Add: a.push(0, g); a.push(1, g); break;
    case Sub: a.push(0, g); a.push(1, -g); break;
    case Mul: { const T x0 = a.val(o[0]), x1 = a.val(o[1]); a.push(0, g * x1); a.push(1, g * x0); break; }
    case Div: {
      const T b = a.val(o[1]), x = a.val(o[0]);
      a.push(0, g / b);
      a.push(1, -g * x / (b * b));
      break;
    }
    case Mean: a.push(0, g / T(2)); a.push(1, g / T(2)); break;
    case AddSquares: { const T x0 = a.val(o[0]), x1 = a.val(o[1]); a.push(0, g * T(2) * x0); a.push(1, g * T(2) * x1); break; }
    case MeanSquares: { const T x0 = a.val(o[0]), x1 = a.val(o[1]); a.push(0, g * x0); a.push(1, g * x1); break; }
    case NegativeMean: a.push(0, -g / T(2)); a.push(1, -g / T(2)); break;
    case AddVarying: for (std::uint32_t j = 0; j < n; ++j) a.push(j, g); break;
    case SubVarying: a.push(0, g); for (std::uint32_t j = 1; j < n; ++j) a.push(j, -g); break;
    case MulVarying: {
      // d/dx_k = prefix(k) * suffix(k+1), multiplied in the reference's order.
      T prefix = T(1);
      for (std::uint32_t k = 0; k < n; ++k) {
        T suffix = T(1);
        for (std::uint32_t j = n - 1; j > k; --j) suffix *= a.val(o[j]);
        a.push(k, g * prefix * suffix);
        prefix *= a.val(o[k]);
      }
      break;
    }
    case MeanVarying: { const T dd = g / static_cast<T>(n); for (std::uint32_t j = 0; j < n; ++j) a.push(j, dd); break; }
    case SumOfSquaresVarying: for (std::uint32_t j = 0; j < n; ++j) a.push(j, g * T(2) * a.val(o[j])); break;
    case MeanSquaresVarying: {
      const T sc = g * T(2) / static_cast<T>(n);
      for (std::uint32_t j = 0; j < n; ++j) a.push(j, sc * a.val(o[j]));
      break;
    }
    case NegativeMeanVarying: { const T dd = -g / static_cast<T>(n); for (std::uint32_t j = 0; j < n; ++j) a.push(j, dd); break; }
    case InnerProductNoBias: {
      const std::uint32_t m = n / 2;
      for (std::uint32_t k = 0; k < m; ++k) {
        const T xk = a.val(o[k]), yk = a.val(o[m + k]);
        a.push(k, g * yk);
        a.push(m + k, g * xk);
      }
      break;
    }
    case InnerProductWithBias: {
      const std::uint32_t m = (n - 1) / 2;
      for (std::uint32_t k = 0; k < m; ++k) {
        const T xk = a.val(o[k]), yk = a.val(o[m + k]);
        a.push(k, g * yk);
        a.push(m + k, g * xk);
      }
      a.push(n - 1, g);
      break;
    }
    default: break;
  }
}

// ---- fused softmax attention head (kAttn, tg_program.hpp Attn), per sample ----
// The interpreter form: one thread walks the head's units with the same
// operations, in the same order, as the scalar nodes it replaces (eval_node /
// propagate above): c_j = <q, k_j> * scale, m = max_j c_j, e_j = exp(c_j - m),
// Z = sum_j e_j (left to right), a_j = e_j / Z, o_i = sum_j a_j v_j[i].
// Reverse, node by node: dA_j = sum_i dO_i v_j[i] and dv_j[i] += dO_i a_j
// (innerProduct), de_j = dA_j / Z and dZ = -sum_j dA_j e_j / Z^2 (div),
// de_j += dZ (reduceSum), dc_j = de_j e_j (exp), the shift takes no gradient,
// ds_j = dc_j scale (mulByConstant), dq += ds_j k_j and dk_j += ds_j q
// (innerProduct).  Scores are recomputed: interior nodes have no rows.  The
// head is the only pusher into its q / k / v rows, so it clears them first.
template <class T>
__device__ __forceinline__ T attn_score(const tgc::Attn& A, const T* V, std::size_t ld, std::size_t col,
                                        std::uint32_t q, std::uint32_t kr) {
  T acc = 0;
  for (std::uint32_t i = 0; i < A.hd; ++i) acc += V[std::size_t(q + i) * ld + col] * V[std::size_t(kr + i) * ld + col];
  return acc * static_cast<T>(A.scale);
}

template <class T>
__device__ void attn_fwd_sample(const tgc::Attn A, const std::uint32_t* __restrict__ ar, T* V, std::size_t ld,
                                std::size_t col) {
  const std::uint32_t* K = ar + A.key_off;
  for (std::uint32_t u = 0; u < A.n_units; ++u) {
    const std::uint32_t q = ar[A.unit_off + 3 * u], o = ar[A.unit_off + 3 * u + 1], n = ar[A.unit_off + 3 * u + 2];
    T m = attn_score<T>(A, V, ld, col, q, K[0]);
    for (std::uint32_t j = 1; j < n; ++j) {
      const T c = attn_score<T>(A, V, ld, col, q, K[2 * j]);
      m = c > m ? c : m;
    }
    T Z = 0;
    for (std::uint32_t j = 0; j < n; ++j) Z += d_exp(attn_score<T>(A, V, ld, col, q, K[2 * j]) - m);
    for (std::uint32_t i = 0; i < A.dv; ++i) V[std::size_t(o + i) * ld + col] = T(0);
    for (std::uint32_t j = 0; j < n; ++j) {
      const T a = d_exp(attn_score<T>(A, V, ld, col, q, K[2 * j]) - m) / Z;
      const std::uint32_t vr = K[2 * j + 1];
      for (std::uint32_t i = 0; i < A.dv; ++i) V[std::size_t(o + i) * ld + col] += a * V[std::size_t(vr + i) * ld + col];
    }
  }
}

template <class T>
__device__ void attn_bwd_sample(const tgc::Attn A, const std::uint32_t* __restrict__ ar, const T* V, T* G,
                                std::size_t ld, std::size_t col) {
  const std::uint32_t* K = ar + A.key_off;
  const T scale = static_cast<T>(A.scale);
  for (std::uint32_t j = 0; j < A.n_keys; ++j) {
    for (std::uint32_t i = 0; i < A.hd; ++i) G[std::size_t(K[2 * j] + i) * ld + col] = T(0);
    for (std::uint32_t i = 0; i < A.dv; ++i) G[std::size_t(K[2 * j + 1] + i) * ld + col] = T(0);
  }
  for (std::uint32_t u = 0; u < A.n_units; ++u) {
    const std::uint32_t q = ar[A.unit_off + 3 * u], o = ar[A.unit_off + 3 * u + 1], n = ar[A.unit_off + 3 * u + 2];
    for (std::uint32_t i = 0; i < A.hd; ++i) G[std::size_t(q + i) * ld + col] = T(0);
    T m = attn_score<T>(A, V, ld, col, q, K[0]);
    for (std::uint32_t j = 1; j < n; ++j) {
      const T c = attn_score<T>(A, V, ld, col, q, K[2 * j]);
      m = c > m ? c : m;
    }
    T Z = 0;
    for (std::uint32_t j = 0; j < n; ++j) Z += d_exp(attn_score<T>(A, V, ld, col, q, K[2 * j]) - m);
    auto dA = [&](std::uint32_t j) {
      const std::uint32_t vr = K[2 * j + 1];
      T acc = 0;
      for (std::uint32_t i = 0; i < A.dv; ++i) acc += G[std::size_t(o + i) * ld + col] * V[std::size_t(vr + i) * ld + col];
      return acc;
    };
    T dZ = 0;
    for (std::uint32_t j = 0; j < n; ++j) {
      const T e = d_exp(attn_score<T>(A, V, ld, col, q, K[2 * j]) - m);
      dZ += -dA(j) * e / (Z * Z);
    }
    for (std::uint32_t j = 0; j < n; ++j) {
      const std::uint32_t kr = K[2 * j], vr = K[2 * j + 1];
      const T e = d_exp(attn_score<T>(A, V, ld, col, q, kr) - m);
      const T a = e / Z;
      const T da = dA(j);
      for (std::uint32_t i = 0; i < A.dv; ++i) G[std::size_t(vr + i) * ld + col] += G[std::size_t(o + i) * ld + col] * a;
      const T ds = (da / Z + dZ) * e * scale;
      for (std::uint32_t i = 0; i < A.hd; ++i) {
        G[std::size_t(q + i) * ld + col] += ds * V[std::size_t(kr + i) * ld + col];
        G[std::size_t(kr + i) * ld + col] += ds * V[std::size_t(q + i) * ld + col];
      }
    }
  }
}

// ---- fused layer normalisation (kLNorm, tg_program.hpp LNorm), per sample ----
// Forward as the nodes it replaces: mu = sum(x)/n, ms = sum(x^2)/n,
// var = ms - mu*mu, rstd = 1/sqrt(var + eps) (invSqrt domain check: the
// reference's std::domain_error), n_i = (x_i - mu) * rstd, y_i = n_i g_i + b_i.
// Reverse, node by node: dn_i = dy_i g_i, dc_i = dn_i rstd,
// drstd = sum_i dn_i c_i, dve = -drstd rstd / (2 ve), dms = dve, dmu2 = -dve,
// dmu = -sum_i dc_i + 2 mu dmu2, dx_i += dc_i + (2 dms / n) x_i + dmu / n.
// The gamma / beta gradients are batch terms over dy and n (compiler).
template <class T>
__device__ __forceinline__ void ln_stats(const tgc::LNorm& L, const std::uint32_t* __restrict__ lr, const T* V,
                                         std::size_t ld, std::size_t col, T& mu, T& ve) {
  T s1 = 0, s2 = 0;
#pragma unroll 8
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const T x = V[std::size_t(lr[L.off + i]) * ld + col];
    s1 += x;
    s2 += x * x;
  }
  mu = s1 / static_cast<T>(L.n);
  const T ms = s2 / static_cast<T>(L.n);
  ve = (ms - mu * mu) + static_cast<T>(L.eps);
}

template <class T>
__device__ bool ln_fwd_sample(const tgc::LNorm L, const std::uint32_t* __restrict__ lr, const T* __restrict__ UV, T* V,
                              std::size_t ld, std::size_t col) {
  T mu, ve;
  ln_stats<T>(L, lr, V, ld, col, mu, ve);
  const bool bad = !(ve > T(0));
  const T rstd = T(1) / d_sqrt(ve);
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const T x = V[std::size_t(lr[L.off + i]) * ld + col];
    const T nv = (x - mu) * rstd;
    V[std::size_t(lr[L.off + L.n + i]) * ld + col] = nv;
    V[std::size_t(lr[L.off + 2 * L.n + i]) * ld + col] = nv * UV[lr[L.off + 3 * L.n + i]] + UV[lr[L.off + 4 * L.n + i]];
  }
  return bad;
}

template <class T>
__device__ void ln_bwd_sample(const tgc::LNorm L, const std::uint32_t* __restrict__ lr, const std::uint8_t* __restrict__ lf,
                              const T* __restrict__ UV, const T* V, T* G, std::size_t ld, std::size_t col) {
  T mu, ve;
  ln_stats<T>(L, lr, V, ld, col, mu, ve);
  const T rstd = T(1) / d_sqrt(ve);
  T drstd = 0, sdc = 0;
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const T dn = G[std::size_t(lr[L.off + 2 * L.n + i]) * ld + col] * UV[lr[L.off + 3 * L.n + i]];
    const T cval = V[std::size_t(lr[L.off + i]) * ld + col] - mu;
    drstd += dn * cval;
    sdc += dn * rstd;
  }
  const T dve = -drstd * rstd / (T(2) * ve);
  const T dms = dve;
  const T dmu = -sdc + (-dve) * T(2) * mu;
  const T cx = dms * T(2) / static_cast<T>(L.n), cm = dmu / static_cast<T>(L.n);
#pragma unroll 4
  for (std::uint32_t i = 0; i < L.n; ++i) {
    const T dc = G[std::size_t(lr[L.off + 2 * L.n + i]) * ld + col] * UV[lr[L.off + 3 * L.n + i]] * rstd;
    const T x = V[std::size_t(lr[L.off + i]) * ld + col];
    const T dx = dc + cx * x + cm;
    T* p = &G[std::size_t(lr[L.off + i]) * ld + col];
    *p = (lf[L.flag_off + i] & tgc::kAssign) ? dx : *p + dx;
  }
}

// Fused activations of kDense groups (domain-free unary ops only); same
// formulas as eval_node / propagate above.
template <class T>
__device__ __forceinline__ T act_fwd(std::uint32_t op, T z) {
  switch (op) {
    case Relu: return z > T(0) ? z : T(0);
    case Tanh: return d_tanh(z);
    case Exp: return d_exp(z);
    case Sigmoid: return T(1) / (T(1) + d_exp(-z));
    case Sqr: return z * z;
    case Cub: return z * z * z;
    default: return z;
  }
}
template <class T>
__device__ __forceinline__ T act_bwd(std::uint32_t op, T g, T y, T z) {
  switch (op) {
    case Relu: return z > T(0) ? g : T(0);
    case Tanh: return g * (T(1) - y * y);
    case Exp: return g * y;
    case Sigmoid: return g * y * (T(1) - y);
    case Sqr: return g * T(2) * z;
    case Cub: return g * T(3) * z * z;
    default: return g;
  }
}

// Derivative of an activation from its output alone (dz = g * act'(z) with
// act'(z) written in h = act(z)), for the activations whose derivative needs
// no z: relu masks on h > 0 (z > 0 exactly when relu(z) > 0), tanh 1 - h^2,
// exp h, sigmoid h (1 - h).  Used where a dense layer's input adjoint product
// writes dz of the layer below directly (act_bwd_from_h_ok).
__host__ __device__ __forceinline__ bool act_bwd_from_h_ok(std::uint32_t op) {
  return op == Relu || op == Tanh || op == Exp || op == Sigmoid;
}
template <class T>
__device__ __forceinline__ T act_bwd_h(std::uint32_t op, T g, T h) {
  switch (op) {
    case Relu: return h > T(0) ? g : T(0);
    case Tanh: return g * (T(1) - h * h);
    case Exp: return g * h;
    case Sigmoid: return g * h * (T(1) - h);
    default: return g;
  }
}

// Accessor over the sample-invariant table (uniform forward / reverse sweeps).
template <class T>
struct UvAcc {
  T* UV;
  T* UG;
  const std::uint32_t* o;
  std::uint32_t const_base;
  __device__ __forceinline__ T val(std::uint32_t op) const { return UV[op & tgc::kIndexMask]; }
  __device__ __forceinline__ void push(std::uint32_t k, T v) {
    const std::uint32_t i = o[k] & tgc::kIndexMask;
    if (i < const_base) UG[i] += v;
  }
};

// First domain violation of a launch: min over (sample << 32 | node).
__device__ __forceinline__ void record_error(unsigned long long* key, std::size_t s, std::uint32_t node) {
  atomicMin(key, (static_cast<unsigned long long>(s) << 32) | node);
}

}  // namespace tgk
