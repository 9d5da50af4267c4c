// tg_models.hpp — the BASELINE.json workloads composed from reference ops.
//
// The reference has no nn/models code (SPEC.md:257-407 is spec only), so the
// compositions here are this build's choices, written once against a
// "builder" interface so the identical op sequence can be recorded
//   * on the reference tapegrad::Tape (oracle/_ref, oracle/ref_driver.cpp), and
//   * on tg::Tape (this package) for compilation to the GPU.
// Topology parity between the two is then a byte comparison of the recorded
// opcode and child arrays (SURVEY.md §3.1 topology hazard: every operand is
// sequenced through a named temporary, never through argument evaluation order).
//
// Builder interface (B):
//   using Scalar, VR;
//   VR param(Scalar) / input(col, Scalar) / constant(Scalar)
//   VR gather(VR first, stride, n_rows, col, offset, int idx)   // data-dependent child
//   VR stopgrad_max(span)                                        // softmax shift
//   VR unary(op,x) / binary(op,x,y) / mul_by_constant(x,c) / varying(op,span)
//   VR ip(span,span) / ipwb(span,span,VR)
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

namespace tgm {

// OpKind numbering of reference op_kind.hpp:10-44.
enum Op : std::uint8_t {
  kLeaf = 0, kRelu, kTanh, kExp, kNegLog, kSigmoid, kInv, kSqr, kCub, kLog, kSqrt, kInvSqrt,
  kAdd, kSub, kMul, kMulByConst, kDiv, kMean, kAddSquares, kMeanSquares, kNegativeMean,
  kAddVarying, kSubVarying, kMulVarying, kMeanVarying, kSumOfSquaresVarying, kMeanSquaresVarying,
  kNegativeMeanVarying, kInnerProductNoBias, kInnerProductWithBias,
};

/// Deterministic generator of the reference test suite: mt19937_64 with a
/// 53-bit unit() and a 128-bit multiply below(n) (testing_support.hpp:49-58).
struct Rng {
  std::mt19937_64 gen;
  explicit Rng(std::uint64_t seed) : gen(seed) {}
  double unit() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
  std::uint64_t below(std::uint64_t n) {
    return static_cast<std::uint64_t>((static_cast<__uint128_t>(gen()) * n) >> 64);
  }
  /// Box-Muller on two unit() draws.
  double normal(double mean, double sd) {
    const double u1 = unit(), u2 = unit();
    const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
    return mean + sd * r * std::cos(6.283185307179586 * u2);
  }
};

/// Zipf(s) over ids 0..V-1 by inverse CDF with p_k ∝ k^-s.
struct Zipf {
  std::vector<double> cdf;
  Zipf(std::uint32_t V, double s) : cdf(V) {
    double acc = 0;
    for (std::uint32_t k = 1; k <= V; ++k) { acc += std::pow(static_cast<double>(k), -s); cdf[k - 1] = acc; }
    for (double& c : cdf) c /= acc;
  }
  std::int32_t draw(Rng& r) const {
    const double u = r.unit();
    std::uint32_t lo = 0, hi = static_cast<std::uint32_t>(cdf.size()) - 1;
    while (lo < hi) { const std::uint32_t mid = (lo + hi) / 2; if (u < cdf[mid]) hi = mid; else lo = mid + 1; }
    return static_cast<std::int32_t>(lo);
  }
};

enum Model : int { kFig1 = 1, kListing1 = 2, kMoons = 3, kCharMlp = 4, kGpt = 5, kWideMlp = 6 };

/// Model dimensions; zeros in the ABI args select these BASELINE.json sizes.
struct Dims {
  std::uint32_t d[8]{};
  static Dims defaults(int model) {
    Dims x;
    switch (model) {
      case kMoons: x.d[0] = 16; x.d[1] = 16; break;                                   // 2-16-16-1
      case kCharMlp: x.d[0] = 27; x.d[1] = 3; x.d[2] = 10; x.d[3] = 200; break;        // V ctx emb hid
      case kGpt: x.d[0] = 65; x.d[1] = 64; x.d[2] = 64; x.d[3] = 4; x.d[4] = 4; x.d[5] = 256; break;
      case kWideMlp: x.d[0] = 784; x.d[1] = 1024; x.d[2] = 1024; x.d[3] = 10; break;
      default: break;
    }
    return x;
  }
  static Dims resolve(int model, const std::uint32_t* user) {
    Dims x = defaults(model);
    if (user) for (int i = 0; i < 8; ++i) if (user[i]) x.d[i] = user[i];
    return x;
  }
};

/// Per-sample data columns of a model.
inline void io_shape(int model, const Dims& D, std::uint32_t& n_inputs, std::uint32_t& n_index) {
  switch (model) {
    case kFig1: case kListing1: n_inputs = 2; n_index = 0; break;
    case kMoons: n_inputs = 3; n_index = 0; break;                 // x0, x1, y
    case kCharMlp: n_inputs = 0; n_index = D.d[1] + 1; break;     // ctx ids + target
    case kGpt: n_inputs = 0; n_index = D.d[1] + 1; break;         // T+1 token ids
    case kWideMlp: n_inputs = D.d[0]; n_index = 1; break;         // pixels + label
    default: throw std::invalid_argument("unknown model");
  }
}

/// One sample's data: x[col], idx[col].
struct Sample {
  const double* x;
  const std::int32_t* idx;
};

/// Synthetic batch, sample-major draws (so a batch is a prefix of any larger
/// batch with the same seed), stored SoA [col][batch].
template <class Scalar>
void synth(int model, const Dims& D, std::uint64_t seed, std::size_t batch, Scalar* x,
           std::int32_t* idx) {
  Rng r(seed);
  std::uint32_t ni = 0, nk = 0;
  io_shape(model, D, ni, nk);
  switch (model) {
    case kFig1: case kListing1:
      for (std::size_t s = 0; s < batch; ++s) {
        x[s] = static_cast<Scalar>(r.uniform(-4.0, 4.0));
        x[batch + s] = static_cast<Scalar>(r.uniform(-4.0, 4.0));
      }
      break;
    case kMoons:
      // Two interleaved half-circles: theta ~ U[0, pi], radius 1; the second
      // arc is the first reflected and offset by (1, -0.5); N(0, 0.1) noise.
      for (std::size_t s = 0; s < batch; ++s) {
        const bool second = r.below(2) == 1;
        const double th = r.uniform(0.0, 3.141592653589793);
        double a = std::cos(th), b = std::sin(th);
        if (second) { a = 1.0 - a; b = 0.5 - b; }
        a += r.normal(0.0, 0.1);
        b += r.normal(0.0, 0.1);
        x[s] = static_cast<Scalar>(a);
        x[batch + s] = static_cast<Scalar>(b);
        x[2 * batch + s] = static_cast<Scalar>(second ? 1.0 : -1.0);
      }
      break;
    case kCharMlp: {
      const Zipf z(D.d[0], 1.1);
      for (std::size_t s = 0; s < batch; ++s)
        for (std::uint32_t c = 0; c < nk; ++c) idx[c * batch + s] = z.draw(r);
      break;
    }
    case kGpt: {
      const Zipf z(D.d[0], 1.0);
      for (std::size_t s = 0; s < batch; ++s)
        for (std::uint32_t c = 0; c < nk; ++c) idx[c * batch + s] = z.draw(r);
      break;
    }
    case kWideMlp:
      for (std::size_t s = 0; s < batch; ++s) {
        for (std::uint32_t c = 0; c < ni; ++c) x[c * batch + s] = static_cast<Scalar>(r.unit());
        idx[s] = static_cast<std::int32_t>(r.below(D.d[3]));
      }
      break;
    default: throw std::invalid_argument("unknown model");
  }
}

// ---------------------------------------------------------------------------
// nn helpers (SPEC.md nn module) over a builder
// ---------------------------------------------------------------------------

template <class B> using VRs = std::vector<typename B::VR>;

/// Contiguous param block, row-major [rows][cols].
template <class B>
struct Block {
  VRs<B> v;
  std::uint32_t rows{0}, cols{0};
  typename B::VR at(std::uint32_t r, std::uint32_t c) const { return v[r * cols + c]; }
  std::span<const typename B::VR> row(std::uint32_t r) const { return {v.data() + std::size_t(r) * cols, cols}; }
};

template <class B, class Init>
Block<B> param_block(B& b, std::uint32_t rows, std::uint32_t cols, Init&& init) {
  Block<B> blk;
  blk.rows = rows;
  blk.cols = cols;
  blk.v.reserve(std::size_t(rows) * cols);
  for (std::size_t i = 0; i < std::size_t(rows) * cols; ++i) blk.v.push_back(b.param(static_cast<typename B::Scalar>(init())));
  return blk;
}

/// linear: out_j = innerProductWithBias(x, W[j], b[j]),
/// optionally followed by one activation node per output.
template <class B>
VRs<B> linear(B& b, std::span<const typename B::VR> x, const Block<B>& W, const Block<B>& bias,
              std::uint8_t act) {
  if (x.size() != W.cols) throw std::invalid_argument("linear: dimension mismatch");
  VRs<B> out;
  out.reserve(W.rows);
  for (std::uint32_t j = 0; j < W.rows; ++j) out.push_back(b.ipwb(x, W.row(j), bias.v[j]));
  if (act != kLeaf)
    for (auto& o : out) o = b.unary(act, o);
  return out;
}

/// Softmax cross-entropy with a stop-gradient max shift:
/// loss = log(sum_j exp(z_j - m)) - (z_t - m), target selected by idx[col].
template <class B>
typename B::VR softmax_ce(B& b, std::span<const typename B::VR> z, std::uint32_t col, std::int32_t target) {
  using VR = typename B::VR;
  const VR m = b.stopgrad_max(z);
  VRs<B> sh, e;
  sh.reserve(z.size());
  e.reserve(z.size());
  for (const VR& zj : z) sh.push_back(b.binary(kSub, zj, m));
  for (const VR& s : sh) e.push_back(b.unary(kExp, s));
  const VR tot = b.varying(kAddVarying, e);
  const VR l = b.unary(kLog, tot);
  const VR zt = b.gather(sh[0], 1, static_cast<std::uint32_t>(z.size()), col, 0, target);
  return b.binary(kSub, l, zt);
}

/// layer_norm: mean / mean-of-squares in one pass, biased
/// variance identity, y_i = gamma_i * (x_i - mu) * invSqrt(var + eps) + beta_i.
template <class B>
VRs<B> layer_norm(B& b, std::span<const typename B::VR> x, const Block<B>& gamma, const Block<B>& beta,
                  double eps) {
  using VR = typename B::VR;
  const VR mu = b.varying(kMeanVarying, x);
  const VR ms = b.varying(kMeanSquaresVarying, x);
  const VR mu2 = b.unary(kSqr, mu);
  const VR var = b.binary(kSub, ms, mu2);
  const VR e = b.constant(static_cast<typename B::Scalar>(eps));
  const VR ve = b.binary(kAdd, var, e);
  const VR rstd = b.unary(kInvSqrt, ve);
  VRs<B> y;
  y.reserve(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) {
    const VR c = b.binary(kSub, x[i], mu);
    const VR n = b.binary(kMul, c, rstd);
    const VR g = b.binary(kMul, n, gamma.v[i]);
    y.push_back(b.binary(kAdd, g, beta.v[i]));
  }
  return y;
}

// ---------------------------------------------------------------------------
// Models: params(b, rng) once, then sample(b, params, data) per sample.
// ---------------------------------------------------------------------------

template <class B>
struct Params {
  std::vector<Block<B>> blocks;  // in creation order
};

template <class B>
Params<B> make_params(B& b, int model, const Dims& D, std::uint64_t seed) {
  Params<B> P;
  Rng r(seed);
  auto unif = [&](double a) { return [&r, a] { return r.uniform(-a, a); }; };
  auto normal = [&](double sd) { return [&r, sd] { return r.normal(0.0, sd); }; };
  auto zero = [] { return 0.0; };
  auto one = [] { return 1.0; };
  switch (model) {
    case kFig1: case kListing1: break;
    case kMoons: {
      const std::uint32_t h1 = D.d[0], h2 = D.d[1];
      // SPEC.md init_params: Uniform(±1/sqrt(in)) weights, zero biases.
      P.blocks.push_back(param_block(b, h1, 2, unif(1.0 / std::sqrt(2.0))));
      P.blocks.push_back(param_block(b, 1, h1, zero));
      P.blocks.push_back(param_block(b, h2, h1, unif(1.0 / std::sqrt(double(h1)))));
      P.blocks.push_back(param_block(b, 1, h2, zero));
      P.blocks.push_back(param_block(b, 1, h2, unif(1.0 / std::sqrt(double(h2)))));
      P.blocks.push_back(param_block(b, 1, 1, zero));
      break;
    }
    case kCharMlp: {
      const std::uint32_t V = D.d[0], C = D.d[1], E = D.d[2], H = D.d[3];
      P.blocks.push_back(param_block(b, V, E, normal(0.1)));      // embedding table
      P.blocks.push_back(param_block(b, H, C * E, normal(0.1)));  // W1
      P.blocks.push_back(param_block(b, 1, H, normal(0.1)));      // b1
      P.blocks.push_back(param_block(b, V, H, normal(0.1)));      // W2
      P.blocks.push_back(param_block(b, 1, V, normal(0.1)));      // b2
      break;
    }
    case kGpt: {
      const std::uint32_t V = D.d[0], T = D.d[1], d = D.d[2], L = D.d[4], F = D.d[5];
      P.blocks.push_back(param_block(b, V, d, normal(0.02)));  // wte
      P.blocks.push_back(param_block(b, T, d, normal(0.02)));  // wpe
      for (std::uint32_t l = 0; l < L; ++l) {
        P.blocks.push_back(param_block(b, 1, d, one));           // ln1 gamma
        P.blocks.push_back(param_block(b, 1, d, zero));          // ln1 beta
        P.blocks.push_back(param_block(b, 3 * d, d, normal(0.02)));  // Wqkv
        P.blocks.push_back(param_block(b, 1, 3 * d, zero));      // bqkv
        P.blocks.push_back(param_block(b, d, d, normal(0.02)));  // Wo
        P.blocks.push_back(param_block(b, 1, d, zero));          // bo
        P.blocks.push_back(param_block(b, 1, d, one));           // ln2 gamma
        P.blocks.push_back(param_block(b, 1, d, zero));          // ln2 beta
        P.blocks.push_back(param_block(b, F, d, normal(0.02)));  // W1
        P.blocks.push_back(param_block(b, 1, F, zero));          // b1
        P.blocks.push_back(param_block(b, d, F, normal(0.02)));  // W2
        P.blocks.push_back(param_block(b, 1, d, zero));          // b2
      }
      P.blocks.push_back(param_block(b, 1, d, one));             // lnf gamma
      P.blocks.push_back(param_block(b, 1, d, zero));            // lnf beta
      P.blocks.push_back(param_block(b, V, d, normal(0.02)));    // head W
      P.blocks.push_back(param_block(b, 1, V, zero));            // head b
      break;
    }
    case kWideMlp: {
      const std::uint32_t I = D.d[0], H1 = D.d[1], H2 = D.d[2], O = D.d[3];
      // He init: N(0, sqrt(2 / fan_in)), zero biases.
      P.blocks.push_back(param_block(b, H1, I, normal(std::sqrt(2.0 / I))));
      P.blocks.push_back(param_block(b, 1, H1, zero));
      P.blocks.push_back(param_block(b, H2, H1, normal(std::sqrt(2.0 / H1))));
      P.blocks.push_back(param_block(b, 1, H2, zero));
      P.blocks.push_back(param_block(b, O, H2, normal(std::sqrt(2.0 / H2))));
      P.blocks.push_back(param_block(b, 1, O, zero));
      break;
    }
    default: throw std::invalid_argument("unknown model");
  }
  return P;
}

/// Records one sample's graph and returns the loss (backward root).
template <class B>
typename B::VR build_sample(B& b, int model, const Dims& D, const Params<B>& P, const Sample& s) {
  using VR = typename B::VR;
  using S = typename B::Scalar;
  switch (model) {
    case kFig1: {
      // g = f/2, f = e^2, e = c - d, d = ab + b^3, c = a + b
      const VR a = b.input(0, static_cast<S>(s.x[0]));
      const VR bb = b.input(1, static_cast<S>(s.x[1]));
      const VR c = b.binary(kAdd, a, bb);
      const VR ab = b.binary(kMul, a, bb);
      const VR b3 = b.unary(kCub, bb);
      const VR d = b.binary(kAdd, ab, b3);
      const VR e = b.binary(kSub, c, d);
      const VR f = b.unary(kSqr, e);
      const VR two = b.constant(S(2));
      return b.binary(kDiv, f, two);
    }
    case kListing1: {
      // PAPER.md:1286-1304 (BurTorch column), operands sequenced explicitly.
      const VR a = b.input(0, static_cast<S>(s.x[0]));
      const VR bb = b.input(1, static_cast<S>(s.x[1]));
      VR c = b.binary(kAdd, a, bb);
      const VR ab = b.binary(kMul, a, bb);
      const VR b3 = b.unary(kCub, bb);
      VR d = b.binary(kAdd, ab, b3);
      const VR one = b.constant(S(1));
      const VR t0 = b.binary(kAdd, c, one);
      c = b.binary(kAdd, c, t0);                  // c += c + 1
      const VR one2 = b.constant(S(1));
      const VR t1 = b.binary(kAdd, one2, c);
      const VR t2 = b.binary(kSub, t1, a);
      c = b.binary(kAdd, c, t2);                  // c += 1 + c - a
      const VR two = b.constant(S(2));
      const VR t3 = b.binary(kMul, d, two);
      const VR ba = b.binary(kAdd, bb, a);
      const VR r1 = b.unary(kRelu, ba);
      const VR t4 = b.binary(kAdd, t3, r1);
      d = b.binary(kAdd, d, t4);                  // d += d*2 + relu(b+a)
      const VR three = b.constant(S(3));
      const VR t5 = b.binary(kMul, three, d);
      const VR bma = b.binary(kSub, bb, a);
      const VR r2 = b.unary(kRelu, bma);
      const VR t6 = b.binary(kAdd, t5, r2);
      d = b.binary(kAdd, d, t6);                  // d += 3*d + relu(b-a)
      const VR e = b.binary(kSub, c, d);
      const VR f = b.unary(kSqr, e);
      const VR two2 = b.constant(S(2));
      VR g = b.binary(kDiv, f, two2);
      const VR ten = b.constant(S(10));
      const VR t7 = b.binary(kDiv, ten, f);
      g = b.binary(kAdd, g, t7);                  // g += 10 / f
      return g;
    }
    case kMoons: {
      const VR x0 = b.input(0, static_cast<S>(s.x[0]));
      const VR x1 = b.input(1, static_cast<S>(s.x[1]));
      const VR y = b.input(2, static_cast<S>(s.x[2]));
      const VRs<B> x{x0, x1};
      const VRs<B> h1 = linear(b, std::span<const VR>(x), P.blocks[0], P.blocks[1], kTanh);
      const VRs<B> h2 = linear(b, std::span<const VR>(h1), P.blocks[2], P.blocks[3], kTanh);
      const VRs<B> out = linear(b, std::span<const VR>(h2), P.blocks[4], P.blocks[5], kLeaf);
      // SVM hinge relu(1 - y * score) plus 1e-4 * sum of squared parameters.
      const VR ys = b.binary(kMul, y, out[0]);
      const VR one = b.constant(S(1));
      const VR margin = b.binary(kSub, one, ys);
      const VR hinge = b.unary(kRelu, margin);
      VRs<B> all;
      for (const auto& blk : P.blocks) all.insert(all.end(), blk.v.begin(), blk.v.end());
      const VR sq = b.varying(kSumOfSquaresVarying, all);
      const VR reg = b.mul_by_constant(sq, S(1e-4));
      return b.binary(kAdd, hinge, reg);
    }
    case kCharMlp: {
      const std::uint32_t V = D.d[0], C = D.d[1], E = D.d[2];
      const Block<B>& emb = P.blocks[0];
      VRs<B> x;
      x.reserve(C * E);
      for (std::uint32_t c = 0; c < C; ++c)
        for (std::uint32_t e = 0; e < E; ++e) x.push_back(b.gather(emb.v[0], E, V, c, e, s.idx[c]));
      const VRs<B> h = linear(b, std::span<const VR>(x), P.blocks[1], P.blocks[2], kTanh);
      const VRs<B> z = linear(b, std::span<const VR>(h), P.blocks[3], P.blocks[4], kLeaf);
      return softmax_ce(b, std::span<const VR>(z), C, s.idx[C]);
    }
    case kWideMlp: {
      const std::uint32_t I = D.d[0];
      VRs<B> x;
      x.reserve(I);
      for (std::uint32_t i = 0; i < I; ++i) x.push_back(b.input(i, static_cast<S>(s.x[i])));
      const VRs<B> h1 = linear(b, std::span<const VR>(x), P.blocks[0], P.blocks[1], kRelu);
      const VRs<B> h2 = linear(b, std::span<const VR>(h1), P.blocks[2], P.blocks[3], kRelu);
      const VRs<B> z = linear(b, std::span<const VR>(h2), P.blocks[4], P.blocks[5], kLeaf);
      return softmax_ce(b, std::span<const VR>(z), 0, s.idx[0]);
    }
    case kGpt: {
      const std::uint32_t V = D.d[0], T = D.d[1], d = D.d[2], H = D.d[3], L = D.d[4];
      const std::uint32_t hd = d / H;
      const Block<B>& wte = P.blocks[0];
      const Block<B>& wpe = P.blocks[1];
      std::vector<VRs<B>> x(T);
      for (std::uint32_t p = 0; p < T; ++p)
        for (std::uint32_t e = 0; e < d; ++e) {
          const VR tok = b.gather(wte.v[0], d, V, p, e, s.idx[p]);
          x[p].push_back(b.binary(kAdd, tok, wpe.at(p, e)));
        }
      const S scale = static_cast<S>(1.0 / std::sqrt(static_cast<double>(hd)));
      for (std::uint32_t l = 0; l < L; ++l) {
        const std::size_t o = 2 + std::size_t(l) * 12;
        const auto &g1 = P.blocks[o + 0], &be1 = P.blocks[o + 1], &Wqkv = P.blocks[o + 2],
                   &bqkv = P.blocks[o + 3], &Wo = P.blocks[o + 4], &bo = P.blocks[o + 5],
                   &g2 = P.blocks[o + 6], &be2 = P.blocks[o + 7], &W1 = P.blocks[o + 8],
                   &b1 = P.blocks[o + 9], &W2 = P.blocks[o + 10], &b2 = P.blocks[o + 11];
        std::vector<VRs<B>> qkv(T);
        for (std::uint32_t p = 0; p < T; ++p) {
          const VRs<B> ln = layer_norm(b, std::span<const VR>(x[p]), g1, be1, 1e-5);
          qkv[p] = linear(b, std::span<const VR>(ln), Wqkv, bqkv, kLeaf);
        }
        std::vector<VRs<B>> att(T, VRs<B>(d));
        for (std::uint32_t h = 0; h < H; ++h) {
          for (std::uint32_t p = 0; p < T; ++p) {
            // causal: scores for j > p are never built
            const std::span<const VR> q(qkv[p].data() + h * hd, hd);
            VRs<B> sc;
            for (std::uint32_t j = 0; j <= p; ++j) {
              const std::span<const VR> k(qkv[j].data() + d + h * hd, hd);
              const VR dot = b.ip(q, k);
              sc.push_back(b.mul_by_constant(dot, scale));
            }
            const VR m = b.stopgrad_max(std::span<const VR>(sc));
            VRs<B> ex;
            for (const VR& v : sc) { const VR sh = b.binary(kSub, v, m); ex.push_back(b.unary(kExp, sh)); }
            const VR Z = b.varying(kAddVarying, ex);
            VRs<B> a;
            for (const VR& v : ex) a.push_back(b.binary(kDiv, v, Z));
            for (std::uint32_t i = 0; i < hd; ++i) {
              VRs<B> vcol;
              for (std::uint32_t j = 0; j <= p; ++j) vcol.push_back(qkv[j][2 * d + h * hd + i]);
              att[p][h * hd + i] = b.ip(std::span<const VR>(a), std::span<const VR>(vcol));
            }
          }
        }
        for (std::uint32_t p = 0; p < T; ++p) {
          const VRs<B> proj = linear(b, std::span<const VR>(att[p]), Wo, bo, kLeaf);
          for (std::uint32_t e = 0; e < d; ++e) x[p][e] = b.binary(kAdd, x[p][e], proj[e]);
          const VRs<B> ln = layer_norm(b, std::span<const VR>(x[p]), g2, be2, 1e-5);
          const VRs<B> f1 = linear(b, std::span<const VR>(ln), W1, b1, kRelu);
          const VRs<B> f2 = linear(b, std::span<const VR>(f1), W2, b2, kLeaf);
          for (std::uint32_t e = 0; e < d; ++e) x[p][e] = b.binary(kAdd, x[p][e], f2[e]);
        }
      }
      const std::size_t o = 2 + std::size_t(L) * 12;
      VRs<B> losses;
      for (std::uint32_t p = 0; p < T; ++p) {
        const VRs<B> ln = layer_norm(b, std::span<const VR>(x[p]), P.blocks[o], P.blocks[o + 1], 1e-5);
        const VRs<B> z = linear(b, std::span<const VR>(ln), P.blocks[o + 2], P.blocks[o + 3], kLeaf);
        losses.push_back(softmax_ce(b, std::span<const VR>(z), p + 1, s.idx[p + 1]));
      }
      return b.varying(kMeanVarying, losses);  // per-sequence loss: mean over T positions
    }
    default: throw std::invalid_argument("unknown model");
  }
}

}  // namespace tgm
