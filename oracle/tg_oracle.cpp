// tg_oracle.cpp — CPU restatement of the reference gradient-oracle path.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, imports or
// executes this file; tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it (as liboracle.so) as the
// checker.  It restates, over a recorded tape description (tg_tape_desc), what
// the reference does per sample inside train_step:
//   1. eager forward of every node in construction order with the formulas of
//      ops.hpp:38-307 (construction order is topological, tape.hpp:55-57);
//   2. zero_grads + backward_with_scratch: iterative DFS post-order from the
//      root with children expanded in stored order, zero-child nodes routed to
//      the leaf list, root seeded to 1, propagate_node in reverse post-order
//      (backprop.hpp:139-184, ops.hpp:316-454);
//   3. GradAccumulator: acc[p] += grad(param p) in sample order;
//   4. sgd_step: x -= gamma * acc / b.
// Gathers are resolved per sample, exactly as re-recording the sample with its
// token ids would wire the children (SPEC.md:266-269 views).  The stop-gradient
// max is a Leaf on a reference tape: it is evaluated from its
// children but has no children for the DFS.
//
// Arithmetic follows the reference's expression shapes operation by operation
// and is compiled with -ffp-contract=off, so it is bit-identical to the
// reference headers built the same way (oracle/_ref, checked in tests).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tg_abi.h"

namespace {

enum : std::uint8_t {
  Leaf = 0, Relu, Tanh, Exp, NegLog, Sigmoid, Inv, Sqr, Cub, Log, Sqrt, InvSqrt,
  Add, Sub, Mul, MulByConst, Div, Mean, AddSquares, MeanSquares, NegativeMean,
  AddVarying, SubVarying, MulVarying, MeanVarying, SumOfSquaresVarying, MeanSquaresVarying,
  NegativeMeanVarying, InnerProductNoBias, InnerProductWithBias,
  StopGradMax = TG_OP_STOPGRAD_MAX,
};

// Mnemonics of reference op_kind.hpp:89-123.
const char* name_of(std::uint8_t op) {
  static const char* const names[] = {
      "leaf", "relu", "tanh", "exp", "negativeLog", "sigmoid", "inv", "sqr", "pow3", "logarithm",
      "sqrt", "invSqrt", "add", "sub", "mul", "mulByConstant", "div", "mean", "addSquares",
      "meanSquares", "negativeMean", "reduceSum", "reduceSub", "reduceMul", "reduceMean",
      "reduceSumOfSquares", "reduceMeanSquares", "reduceNegativeMean", "innerProduct",
      "innerProductWithBias"};
  if (op < sizeof(names) / sizeof(names[0])) return names[op];
  return op == StopGradMax ? "stopGradMax" : "?";
}

struct DomainHit {
  bool hit = false;
  std::int64_t sample = -1;
  std::uint32_t node = 0;
  std::uint8_t op = 0;
  double value = 0;
};

template <class S>
struct Worker {
  const tg_tape_desc& d;
  std::vector<S> val, grad, scratch;
  std::vector<std::uint32_t> kids_buf;      // resolved children of all nodes
  std::vector<std::uint32_t> order, stack_node, stack_cur, visited;
  std::uint32_t epoch = 0;

  explicit Worker(const tg_tape_desc& desc) : d(desc) {
    val.resize(d.n_nodes);
    grad.resize(d.n_nodes);
    kids_buf.resize(d.child_offset[d.n_nodes]);
    visited.assign(d.n_nodes, 0);
    std::uint64_t max_ar = 0;
    for (std::uint32_t i = 0; i < d.n_nodes; ++i)
      max_ar = std::max<std::uint64_t>(max_ar, d.child_offset[i + 1] - d.child_offset[i]);
    scratch.resize(max_ar + 1);
    for (std::uint64_t e = 0; e < kids_buf.size(); ++e) kids_buf[e] = d.child[e];
  }

  const std::uint32_t* kids(std::uint32_t i) const { return kids_buf.data() + d.child_offset[i]; }
  std::uint32_t nk(std::uint32_t i) const {
    return static_cast<std::uint32_t>(d.child_offset[i + 1] - d.child_offset[i]);
  }
  // Children the reverse sweep sees: a stop-gradient max is a Leaf.
  std::uint32_t nk_bwd(std::uint32_t i) const { return d.op[i] == StopGradMax ? 0 : nk(i); }

  void resolve(const std::int32_t* idx, std::size_t ld, std::size_t s) {
    const std::uint64_t E = d.child_offset[d.n_nodes];
    for (std::uint64_t e = 0; e < E; ++e) {
      const std::uint32_t c = d.child[e];
      if (c & TG_GATHER_FLAG) {
        const tg_gather& g = d.gathers[c & ~TG_GATHER_FLAG];
        const std::int32_t r = idx[std::size_t(g.index_col) * ld + s];
        kids_buf[e] = g.first_node + g.stride * static_cast<std::uint32_t>(r) + g.offset;
      } else {
        kids_buf[e] = c;
      }
    }
  }

  // Eager forward of one node (ops.hpp:38-307).  Returns false on a domain
  // violation (the reference throws std::domain_error at construction).
  bool forward_node(std::uint32_t i, DomainHit& dh, std::int64_t s) {
    const std::uint8_t op = d.op[i];
    const std::uint32_t* k = kids(i);
    const std::uint32_t n = nk(i);
    auto bad = [&](double v) {
      if (!dh.hit) { dh.hit = true; dh.sample = s; dh.node = i; dh.op = op; dh.value = v; }
      return false;
    };
    S y = 0;
    switch (op) {
      case Relu: { const S v = val[k[0]]; y = v > S(0) ? v : S(0); break; }
      case Tanh: y = std::tanh(val[k[0]]); break;
      case Exp: y = std::exp(val[k[0]]); break;
      case NegLog: { const S v = val[k[0]]; if (!(v > S(0))) return bad(v); y = -std::log(v); break; }
      case Sigmoid: y = S(1) / (S(1) + std::exp(-val[k[0]])); break;
      case Inv: { const S v = val[k[0]]; if (v == S(0)) return bad(v); y = S(1) / v; break; }
      case Sqr: { const S v = val[k[0]]; y = v * v; break; }
      case Cub: { const S v = val[k[0]]; y = v * v * v; break; }
      case Log: { const S v = val[k[0]]; if (!(v > S(0))) return bad(v); y = std::log(v); break; }
      case Sqrt: { const S v = val[k[0]]; if (!(v > S(0))) return bad(v); y = std::sqrt(v); break; }
      case InvSqrt: { const S v = val[k[0]]; if (!(v > S(0))) return bad(v); y = S(1) / std::sqrt(v); break; }
      case MulByConst: y = val[k[0]] * static_cast<S>(d.constant[i]); break;
      case Add: y = val[k[0]] + val[k[1]]; break;
      case Sub: y = val[k[0]] - val[k[1]]; break;
      case Mul: y = val[k[0]] * val[k[1]]; break;
      case Div: { const S b = val[k[1]]; if (b == S(0)) return bad(b); y = val[k[0]] / b; break; }
      case Mean: y = (val[k[0]] + val[k[1]]) / S(2); break;
      case AddSquares: { const S a = val[k[0]], b = val[k[1]]; y = a * a + b * b; break; }
      case MeanSquares: { const S a = val[k[0]], b = val[k[1]]; y = (a * a + b * b) / S(2); break; }
      case NegativeMean: y = -(val[k[0]] + val[k[1]]) / S(2); break;
      case AddVarying: case MeanVarying: case NegativeMeanVarying: {
        S acc = 0;
        for (std::uint32_t j = 0; j < n; ++j) acc += val[k[j]];
        const S nn = static_cast<S>(n);
        if (op == MeanVarying) acc /= nn;
        if (op == NegativeMeanVarying) acc = -acc / nn;
        y = acc;
        break;
      }
      case SubVarying: {
        S acc = val[k[0]];
        for (std::uint32_t j = 1; j < n; ++j) acc -= val[k[j]];
        y = acc;
        break;
      }
      case MulVarying: {
        S acc = S(1);
        for (std::uint32_t j = 0; j < n; ++j) acc *= val[k[j]];
        y = acc;
        break;
      }
      case SumOfSquaresVarying: case MeanSquaresVarying: {
        S acc = 0;
        for (std::uint32_t j = 0; j < n; ++j) { const S v = val[k[j]]; acc += v * v; }
        if (op == MeanSquaresVarying) acc /= static_cast<S>(n);
        y = acc;
        break;
      }
      case InnerProductNoBias: {
        const std::uint32_t m = n / 2;
        S acc = 0;
        for (std::uint32_t j = 0; j < m; ++j) acc += val[k[j]] * val[k[m + j]];
        y = acc;
        break;
      }
      case InnerProductWithBias: {
        const std::uint32_t m = (n - 1) / 2;
        S acc = val[k[n - 1]];
        for (std::uint32_t j = 0; j < m; ++j) acc += val[k[j]] * val[k[m + j]];
        y = acc;
        break;
      }
      case StopGradMax: {
        S m = val[k[0]];
        for (std::uint32_t j = 1; j < n; ++j) m = std::max(m, val[k[j]]);
        y = m;
        break;
      }
      default: break;
    }
    val[i] = y;
    return true;
  }

  // propagate_node (ops.hpp:316-454).
  void propagate(std::uint32_t i) {
    const S g = grad[i];
    const S y = val[i];
    const std::uint32_t* k = kids(i);
    const std::uint32_t n = nk(i);
    auto addg = [&](std::uint32_t c, S v) { grad[c] += v; };
    switch (d.op[i]) {
      case Relu: addg(k[0], val[k[0]] > S(0) ? g : S(0)); break;
      case Tanh: addg(k[0], g * (S(1) - y * y)); break;
      case Exp: addg(k[0], g * y); break;
      case NegLog: addg(k[0], -g / val[k[0]]); break;
      case Sigmoid: addg(k[0], g * y * (S(1) - y)); break;
      case Inv: addg(k[0], -g * y * y); break;
      case Sqr: addg(k[0], g * S(2) * val[k[0]]); break;
      case Cub: { const S x = val[k[0]]; addg(k[0], g * S(3) * x * x); break; }
      case Log: addg(k[0], g / val[k[0]]); break;
      case Sqrt: addg(k[0], g / (S(2) * y)); break;
      case InvSqrt: addg(k[0], -g * y / (S(2) * val[k[0]])); break;
      case MulByConst: addg(k[0], g * static_cast<S>(d.constant[i])); break;
      case Add: addg(k[0], g); addg(k[1], g); break;
      case Sub: addg(k[0], g); addg(k[1], -g); break;
      case Mul: addg(k[0], g * val[k[1]]); addg(k[1], g * val[k[0]]); break;
      case Div: {
        const S b = val[k[1]];
        addg(k[0], g / b);
        addg(k[1], -g * val[k[0]] / (b * b));
        break;
      }
      case Mean: addg(k[0], g / S(2)); addg(k[1], g / S(2)); break;
      case AddSquares: addg(k[0], g * S(2) * val[k[0]]); addg(k[1], g * S(2) * val[k[1]]); break;
      case MeanSquares: addg(k[0], g * val[k[0]]); addg(k[1], g * val[k[1]]); break;
      case NegativeMean: addg(k[0], -g / S(2)); addg(k[1], -g / S(2)); break;
      case AddVarying: for (std::uint32_t j = 0; j < n; ++j) addg(k[j], g); break;
      case SubVarying:
        addg(k[0], g);
        for (std::uint32_t j = 1; j < n; ++j) addg(k[j], -g);
        break;
      case MulVarying: {
        S suffix = S(1);
        for (std::uint32_t j = n; j-- > 0;) { scratch[j] = suffix; suffix *= val[k[j]]; }
        S prefix = S(1);
        for (std::uint32_t j = 0; j < n; ++j) { addg(k[j], g * prefix * scratch[j]); prefix *= val[k[j]]; }
        break;
      }
      case MeanVarying: { const S dd = g / static_cast<S>(n); for (std::uint32_t j = 0; j < n; ++j) addg(k[j], dd); break; }
      case SumOfSquaresVarying: for (std::uint32_t j = 0; j < n; ++j) addg(k[j], g * S(2) * val[k[j]]); break;
      case MeanSquaresVarying: {
        const S sc = g * S(2) / static_cast<S>(n);
        for (std::uint32_t j = 0; j < n; ++j) addg(k[j], sc * val[k[j]]);
        break;
      }
      case NegativeMeanVarying: { const S dd = -g / static_cast<S>(n); for (std::uint32_t j = 0; j < n; ++j) addg(k[j], dd); break; }
      case InnerProductNoBias: {
        const std::uint32_t m = n / 2;
        for (std::uint32_t j = 0; j < m; ++j) { addg(k[j], g * val[k[m + j]]); addg(k[m + j], g * val[k[j]]); }
        break;
      }
      case InnerProductWithBias: {
        const std::uint32_t m = (n - 1) / 2;
        for (std::uint32_t j = 0; j < m; ++j) { addg(k[j], g * val[k[m + j]]); addg(k[m + j], g * val[k[j]]); }
        addg(k[n - 1], g);
        break;
      }
      default: break;  // Leaf, StopGradMax
    }
  }

  // backward_with_scratch order (backprop.hpp:150-183): iterative DFS.
  void dfs_order(std::uint32_t root) {
    if (++epoch == 0) { std::fill(visited.begin(), visited.end(), 0u); epoch = 1; }
    order.clear();
    stack_node.clear();
    stack_cur.clear();
    visited[root] = epoch;
    if (nk_bwd(root) != 0) { stack_node.push_back(root); stack_cur.push_back(0); }
    while (!stack_node.empty()) {
      const std::uint32_t node = stack_node.back();
      const std::uint32_t cur = stack_cur.back();
      if (cur < nk_bwd(node)) {
        stack_cur.back() = cur + 1;
        const std::uint32_t c = kids(node)[cur];
        if (visited[c] != epoch) {
          visited[c] = epoch;
          if (nk_bwd(c) != 0) { stack_node.push_back(c); stack_cur.push_back(0); }
        }
      } else {
        order.push_back(node);
        stack_node.pop_back();
        stack_cur.pop_back();
      }
    }
  }

  // One sample of train_step: returns false on a domain error.
  bool sample(const double* x, const std::int32_t* idx, std::size_t ld, std::size_t s,
              const S* params, DomainHit& dh) {
    if (d.n_gathers) resolve(idx, ld, s);
    for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
      if (d.op[i] == Leaf) {
        switch (d.leaf_class[i]) {
          case TG_LEAF_PARAM: val[i] = params[d.leaf_index[i]]; break;
          case TG_LEAF_INPUT: val[i] = static_cast<S>(x[std::size_t(d.leaf_index[i]) * ld + s]); break;
          default: val[i] = static_cast<S>(d.leaf_value[i]); break;
        }
      } else if (!forward_node(i, dh, static_cast<std::int64_t>(s))) {
        return false;
      }
    }
    std::fill(grad.begin(), grad.end(), S(0));  // zero_grads over the whole tape
    dfs_order(d.root);
    grad[d.root] = S(1);
    for (std::size_t j = order.size(); j-- > 0;) propagate(order[j]);
    return true;
  }
};

thread_local std::string g_err;

template <class S>
int run_impl(const tg_tape_desc* d, const double* x, const std::int32_t* idx, std::size_t batch,
             const double* params_d, double* loss, double* igrad, double* gsum, int threads,
             std::int64_t* bad_sample, std::uint32_t* bad_node) {
  std::vector<S> params(d->n_params);
  for (std::uint32_t p = 0; p < d->n_params; ++p) params[p] = static_cast<S>(params_d[p]);
  std::vector<std::uint32_t> param_node(d->n_params, 0xffffffffu);
  for (std::uint32_t i = 0; i < d->n_nodes; ++i)
    if (d->op[i] == Leaf && d->leaf_class[i] == TG_LEAF_PARAM) param_node[d->leaf_index[i]] = i;

  if (threads < 1) threads = 1;
  if (static_cast<std::size_t>(threads) > batch) threads = static_cast<int>(std::max<std::size_t>(batch, 1));
  std::vector<std::vector<S>> acc(threads, std::vector<S>(d->n_params, S(0)));
  std::vector<DomainHit> hits(threads);
  auto body = [&](int t) {
    Worker<S> w(*d);
    const std::size_t lo = batch * t / threads, hi = batch * (t + 1) / threads;
    for (std::size_t s = lo; s < hi; ++s) {
      if (!w.sample(x, idx, batch, s, params.data(), hits[t])) return;
      if (loss) loss[s] = static_cast<double>(w.val[d->root]);
      if (igrad)
        for (std::uint32_t i = 0; i < d->n_nodes; ++i)
          if (d->op[i] == Leaf && d->leaf_class[i] == TG_LEAF_INPUT)
            igrad[std::size_t(d->leaf_index[i]) * batch + s] = static_cast<double>(w.grad[i]);
      // GradAccumulator: acc += grads over the parameter range
      for (std::uint32_t p = 0; p < d->n_params; ++p)
        if (param_node[p] != 0xffffffffu) acc[t][p] += w.grad[param_node[p]];
    }
  };
  if (threads == 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(body, t);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < threads; ++t)
    if (hits[t].hit) {
      const DomainHit& h = hits[t];
      g_err = std::string(name_of(h.op)) + ": input " + std::to_string(h.value) +
              " is outside the operator domain";
      if (bad_sample) *bad_sample = h.sample;
      if (bad_node) *bad_node = h.node;
      return TG_DOMAIN;
    }
  if (gsum) {
    for (std::uint32_t p = 0; p < d->n_params; ++p) {
      S tot = acc[0][p];
      for (int t = 1; t < threads; ++t) tot += acc[t][p];  // thread order
      gsum[p] = static_cast<double>(tot);
    }
  }
  return TG_OK;
}

}  // namespace

extern "C" {

/// Per-sample forward + backward + accumulation over a batch.
int oracle_run(const tg_tape_desc* d, const double* inputs, const std::int32_t* index_inputs,
               std::size_t batch, const double* params, double* loss_out, double* input_grad_out,
               double* grad_sum, int threads, std::int64_t* bad_sample, std::uint32_t* bad_node) {
  try {
    if (d->dtype == TG_F64)
      return run_impl<double>(d, inputs, index_inputs, batch, params, loss_out, input_grad_out,
                              grad_sum, threads, bad_sample, bad_node);
    return run_impl<float>(d, inputs, index_inputs, batch, params, loss_out, input_grad_out,
                           grad_sum, threads, bad_sample, bad_node);
  } catch (const std::exception& e) {
    g_err = e.what();
    return TG_INVALID_ARGUMENT;
  }
}

/// sgd_step in the tape's scalar type: x -= gamma * acc / b.
void oracle_sgd(int dtype, double* params, const double* grad_sum, std::size_t n, double gamma,
                std::size_t batch) {
  if (dtype == TG_F64) {
    for (std::size_t p = 0; p < n; ++p)
      params[p] = params[p] - gamma * grad_sum[p] / static_cast<double>(batch);
  } else {
    for (std::size_t p = 0; p < n; ++p) {
      const float x = static_cast<float>(params[p]);
      const float g = static_cast<float>(grad_sum[p]);
      params[p] = static_cast<double>(x - static_cast<float>(gamma) * g / static_cast<float>(batch));
    }
  }
}

/// Reference processing order (backward_with_scratch's scratch.order after
/// the final std::reverse, backprop.hpp:183) for sample `s`.
int oracle_order(const tg_tape_desc* d, const std::int32_t* index_inputs, std::size_t ld,
                 std::size_t s, std::uint32_t* order_out, std::uint32_t* n_out) {
  try {
    if (d->dtype == TG_F64) {
      Worker<double> w(*d);
      w.resolve(index_inputs, ld, s);
      w.dfs_order(d->root);
      for (std::size_t j = 0; j < w.order.size(); ++j) order_out[j] = w.order[w.order.size() - 1 - j];
      *n_out = static_cast<std::uint32_t>(w.order.size());
    } else {
      Worker<float> w(*d);
      w.resolve(index_inputs, ld, s);
      w.dfs_order(d->root);
      for (std::size_t j = 0; j < w.order.size(); ++j) order_out[j] = w.order[w.order.size() - 1 - j];
      *n_out = static_cast<std::uint32_t>(w.order.size());
    }
    return TG_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TG_INVALID_ARGUMENT;
  }
}

const char* oracle_last_error(void) { return g_err.c_str(); }

}  // extern "C"
