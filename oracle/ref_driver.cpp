// ref_driver.cpp — drives the UNMODIFIED reference tapegrad headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/
// libtgref.so with -I/root/reference/proj/include (the reference sources are
// compiled where they lie, never copied).  It gives the tests and the bench's
// reference arm the reference's own per-sample path:
//   per sample: rewind to the post-parameter checkpoint (tape.hpp:235-242),
//   re-record the sample with the reference ops (ops.hpp), zero_grads
//   (backprop.hpp:100-109), backward_with_scratch (backprop.hpp:139-184),
//   accumulate parameter grads.
// It also exports the reference's random-graph fuzzer (testing_support.hpp:
// 206-302) so recipes can be replayed on the GPU recorder.
//
// Tape::leaf does not compile as shipped (tape.hpp:169, ambiguous emplace
// overload); the explicit specialisations below are the documented shim
// and must precede any instantiation of leaf().
#include "tapegrad/tape.hpp"
template <> tapegrad::ValueRef tapegrad::Tape<double>::leaf(double v) {
  return emplace_with(OpKind::Leaf, v, 0, [](NodeIndex*) {});
}
template <> tapegrad::ValueRef tapegrad::Tape<float>::leaf(float v) {
  return emplace_with(OpKind::Leaf, v, 0, [](NodeIndex*) {});
}
#include "tapegrad/backprop.hpp"
#include "tapegrad/ops.hpp"
#include "../tests/testing_support.hpp"  // resolved via -I/root/reference/proj/tests/..

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>

#include "tg_from_tapegrad.hpp"
#include "tg_models.hpp"

namespace testsupport {
std::uint64_t allocation_count() { return 0; }  // alloc_probe.cpp is absent from the reference
}

namespace {

thread_local std::string g_err;

template <class S>
struct RefBuilder {
  using Scalar = S;
  using VR = tapegrad::ValueRef;
  tapegrad::Tape<S>& t;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> inputs;  // (col, node)
  tgadapt::Recording* rec = nullptr;   // drop-in description (tg_from_tapegrad.hpp)

  VR param(S v) { return t.leaf(v); }
  VR constant(S v) { return t.leaf(v); }
  VR input(std::uint32_t col, S v) {
    VR r = t.leaf(v);
    inputs.emplace_back(col, r.index);
    return r;
  }
  // A re-recorded sample wires the selected node directly.
  VR gather(VR first, std::uint32_t stride, std::uint32_t n_rows, std::uint32_t col, std::uint32_t off,
            std::int32_t idx) {
    if (rec) return rec->select(t, first, stride, n_rows, col, off, idx);
    return VR{first.index + stride * static_cast<std::uint32_t>(idx) + off};
  }
  // Softmax shift: a non-differentiable constant leaf.
  VR stopgrad_max(std::span<const VR> xs) {
    if (rec) return rec->stopgrad_max(t, xs);
    S m = t.value_of(xs[0]);
    for (std::size_t i = 1; i < xs.size(); ++i) m = std::max(m, t.value_of(xs[i]));
    return t.leaf(m);
  }
  VR unary(std::uint8_t op, VR x) { return tapegrad::unary(t, static_cast<tapegrad::OpKind>(op), x); }
  VR binary(std::uint8_t op, VR x, VR y) { return tapegrad::binary(t, static_cast<tapegrad::OpKind>(op), x, y); }
  VR mul_by_constant(VR x, S c) { return tapegrad::mul_by_constant(t, x, c); }
  VR varying(std::uint8_t op, std::span<const VR> xs) {
    return tapegrad::varying(t, static_cast<tapegrad::OpKind>(op), xs);
  }
  VR ip(std::span<const VR> x, std::span<const VR> y) { return tapegrad::inner_product(t, x, y); }
  VR ipwb(std::span<const VR> x, std::span<const VR> y, VR b) {
    return tapegrad::inner_product_with_bias(t, x, y, b);
  }
};

template <class S>
int run_model(int model, const std::uint32_t* dims, const double* params, const double* x,
              const std::int32_t* idx, std::size_t batch, double* loss, double* igrad,
              double* gsum, int threads) {
  const tgm::Dims D = tgm::Dims::resolve(model, dims);
  std::uint32_t ni = 0, nk = 0;
  tgm::io_shape(model, D, ni, nk);
  if (threads < 1) threads = 1;
  if (static_cast<std::size_t>(threads) > batch) threads = static_cast<int>(std::max<std::size_t>(batch, 1));
  std::vector<std::vector<S>> acc(threads);
  std::vector<std::string> errs(threads);
  std::uint32_t n_params = 0;
  auto body = [&](int th) {
    try {
      tapegrad::Tape<S> tape(tapegrad::TapeConfig{.capacity = 1 << 16});
      RefBuilder<S> b{tape, {}};
      const auto P = tgm::make_params(b, model, D, 0);
      std::vector<std::uint32_t> pnodes;
      for (const auto& blk : P.blocks) for (auto v : blk.v) pnodes.push_back(v.index);
      for (std::size_t p = 0; p < pnodes.size(); ++p) tape.set_value(tapegrad::ValueRef{pnodes[p]}, static_cast<S>(params[p]));
      if (th == 0) n_params = static_cast<std::uint32_t>(pnodes.size());
      acc[th].assign(pnodes.size(), S(0));
      const tapegrad::Checkpoint cp = tape.checkpoint();
      tapegrad::ScratchBuffers<S> scratch;
      std::vector<double> xs(ni);
      std::vector<std::int32_t> ks(nk);
      const std::size_t lo = batch * th / threads, hi = batch * (th + 1) / threads;
      for (std::size_t s = lo; s < hi; ++s) {
        tape.rewind(cp);
        b.inputs.clear();
        for (std::uint32_t c = 0; c < ni; ++c) xs[c] = x[std::size_t(c) * batch + s];
        for (std::uint32_t c = 0; c < nk; ++c) ks[c] = idx[std::size_t(c) * batch + s];
        const tgm::Sample smp{xs.data(), ks.data()};
        const auto root = tgm::build_sample(b, model, D, P, smp);
        tapegrad::zero_grads(tape, 0, tape.size());
        tapegrad::backward_with_scratch(tape, root, scratch);
        if (loss) loss[s] = static_cast<double>(tape.value_of(root));
        if (igrad) for (auto [c, node] : b.inputs) igrad[std::size_t(c) * batch + s] = static_cast<double>(tape.grad_at(node));
        for (std::size_t p = 0; p < pnodes.size(); ++p) acc[th][p] += tape.grad_at(pnodes[p]);
      }
    } catch (const std::exception& e) {
      errs[th] = e.what();
    }
  };
  if (threads == 1) body(0);
  else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(body, t);
    for (auto& t : pool) t.join();
  }
  for (int t = 0; t < threads; ++t)
    if (!errs[t].empty()) { g_err = errs[t]; return 5; }
  if (gsum)
    for (std::uint32_t p = 0; p < n_params; ++p) {
      S tot = acc[0][p];
      for (int t = 1; t < threads; ++t) tot += acc[t][p];
      gsum[p] = static_cast<double>(tot);
    }
  return 0;
}

struct RecipeBuf {
  std::vector<double> leaves;
  std::vector<std::uint8_t> ops;
  std::vector<std::uint32_t> arg_off, args;
  std::vector<double> consts;
};
thread_local RecipeBuf g_recipe;

testsupport::GraphRecipe unpack(std::uint32_t n_leaves, std::uint32_t n_steps, const std::uint8_t* ops,
                                const std::uint32_t* arg_off, const std::uint32_t* args, const double* consts) {
  testsupport::GraphRecipe r;
  r.leaf_count = n_leaves;
  for (std::uint32_t i = 0; i < n_steps; ++i) {
    testsupport::GraphRecipe::Step st;
    st.op = static_cast<tapegrad::OpKind>(ops[i]);
    st.args.assign(args + arg_off[i], args + arg_off[i + 1]);
    st.constant = consts[i];
    r.steps.push_back(std::move(st));
  }
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

/// Records params + one sample of `model` on a reference tape and copies out
/// the topology.  Call with null buffers first to get the sizes.
int ref_build(int model, const std::uint32_t* dims, std::uint64_t seed, int dtype, const double* x1,
              const std::int32_t* idx1, std::uint32_t* n_nodes, std::uint64_t* n_edges, std::uint8_t* ops,
              std::uint64_t* child_off, std::uint32_t* child, double* consts, double* values,
              std::uint32_t* root_out) {
  try {
    auto go = [&](auto tag) -> int {
      using S = decltype(tag);
      const tgm::Dims D = tgm::Dims::resolve(model, dims);
      tapegrad::Tape<S> tape(tapegrad::TapeConfig{.capacity = 1 << 16});
      RefBuilder<S> b{tape, {}};
      const auto P = tgm::make_params(b, model, D, seed);
      const tgm::Sample smp{x1, idx1};
      const auto root = tgm::build_sample(b, model, D, P, smp);
      *n_nodes = tape.size();
      *n_edges = tape.child_pool_size();
      if (root_out) *root_out = root.index;
      if (ops) {
        std::uint64_t off = 0;
        for (std::uint32_t i = 0; i < tape.size(); ++i) {
          ops[i] = static_cast<std::uint8_t>(tape.op_at(i));
          child_off[i] = off;
          for (auto c : tape.children_at(i)) child[off++] = c;
          if (consts) consts[i] = static_cast<double>(tape.constant_at(i));
          if (values) values[i] = static_cast<double>(tape.value_at(i));
        }
        child_off[tape.size()] = off;
      }
      return 0;
    };
    return dtype == 0 ? go(double{}) : go(float{});
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// Initial parameter values of `model` recorded on a reference tape
/// (make_params over tapegrad::Tape<S>, values read back as S).  Call with
/// out = NULL to get the count.  The bench's reference arm takes its
/// parameters from here, never from the product library.
int ref_params(int model, const std::uint32_t* dims, std::uint64_t seed, int dtype, double* out,
               std::uint32_t* n_out) {
  try {
    auto go = [&](auto tag) -> int {
      using S = decltype(tag);
      const tgm::Dims D = tgm::Dims::resolve(model, dims);
      tapegrad::Tape<S> tape(tapegrad::TapeConfig{.capacity = 1 << 16});
      RefBuilder<S> b{tape, {}};
      const auto P = tgm::make_params(b, model, D, seed);
      std::uint32_t n = 0;
      for (const auto& blk : P.blocks)
        for (auto v : blk.v) {
          if (out) out[n] = static_cast<double>(tape.value_of(v));
          ++n;
        }
      *n_out = n;
      return 0;
    };
    return dtype == 0 ? go(double{}) : go(float{});
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// Synthetic batch of `model` (tgm::synth, the SURVEY.md §8d generators) in
/// the tape's scalar type, widened to double: x [n_inputs][batch], idx
/// [n_index][batch].  Same bits as the product's tg_synth_batch for the same
/// seed, so both bench arms see identical samples.
int ref_synth(int model, const std::uint32_t* dims, int dtype, std::uint64_t seed, std::size_t batch, double* x,
              std::int32_t* idx, std::uint32_t* n_inputs, std::uint32_t* n_index) {
  try {
    const tgm::Dims D = tgm::Dims::resolve(model, dims);
    std::uint32_t ni = 0, nk = 0;
    tgm::io_shape(model, D, ni, nk);
    *n_inputs = ni;
    *n_index = nk;
    if (!x && !idx) return 0;
    auto go = [&](auto tag) {
      using S = decltype(tag);
      std::vector<S> xs(std::max<std::size_t>(std::size_t(ni) * batch, 1));
      tgm::synth<S>(model, D, seed, batch, xs.data(), idx);
      for (std::size_t i = 0; i < std::size_t(ni) * batch; ++i) x[i] = static_cast<double>(xs[i]);
    };
    if (dtype == 0) go(double{}); else go(float{});
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// A template sample of `model` recorded on the UNMODIFIED reference tape with
/// the drop-in adapter's side record (tgadapt::Recording: selections and max
/// shifts), described by tgadapt::describe into *out (arrays valid until the
/// next call on this thread).  Template index inputs are idx[c] = c mod rows
/// (distinct rows per table); template inputs x[c] = x1[c] when given.
int ref_describe(int model, const std::uint32_t* dims, std::uint64_t seed, int dtype, const double* x1,
                 tg_tape_desc* out) {
  thread_local tgadapt::DescArrays keep;
  try {
    auto go = [&](auto tag) -> int {
      using S = decltype(tag);
      const tgm::Dims D = tgm::Dims::resolve(model, dims);
      std::uint32_t ni = 0, nk = 0;
      tgm::io_shape(model, D, ni, nk);
      std::vector<double> xs(std::max<std::uint32_t>(ni, 1), 0.5);
      if (x1) std::copy(x1, x1 + ni, xs.begin());
      std::vector<std::int32_t> ks(std::max<std::uint32_t>(nk, 1));
      for (std::uint32_t c = 0; c < nk; ++c) ks[c] = static_cast<std::int32_t>(c);
      const std::uint32_t rows = model == tgm::kWideMlp ? D.d[3] : D.d[0];   // classes / vocabulary
      for (std::uint32_t c = 0; c < nk; ++c) ks[c] %= static_cast<std::int32_t>(rows);
      tapegrad::Tape<S> tape(tapegrad::TapeConfig{.capacity = 1 << 24});
      tgadapt::Recording rec;
      RefBuilder<S> b{tape, {}, &rec};
      const auto P = tgm::make_params(b, model, D, seed);
      std::vector<std::pair<std::uint32_t, tgadapt::LeafRole>> roles;
      std::uint32_t pid = 0;
      for (const auto& blk : P.blocks)
        for (auto v : blk.v) roles.push_back({v.index, {TG_LEAF_PARAM, pid++}});
      const tgm::Sample smp{xs.data(), ks.data()};
      const auto root = tgm::build_sample(b, model, D, P, smp);
      for (auto [col, node] : b.inputs) roles.push_back({node, {TG_LEAF_INPUT, col}});
      keep = tgadapt::describe(tape, root.index, roles, &rec);
      *out = keep.desc;
      return 0;
    };
    return dtype == 0 ? go(double{}) : go(float{});
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// The reference per-sample training-step path over a batch (params given).
int ref_run(int model, const std::uint32_t* dims, int dtype, const double* params, const double* x,
            const std::int32_t* idx, std::size_t batch, double* loss, double* igrad, double* gsum,
            int threads) {
  if (dtype == 0) return run_model<double>(model, dims, params, x, idx, batch, loss, igrad, gsum, threads);
  return run_model<float>(model, dims, params, x, idx, batch, loss, igrad, gsum, threads);
}

/// testsupport::random_recipe (testing_support.hpp:206-302) serialised.
int ref_recipe(std::uint64_t seed, std::size_t max_nodes, std::uint32_t* n_leaves, std::uint32_t* n_steps,
               std::uint32_t* n_args) {
  testsupport::TestRng rng(seed);
  std::vector<double> leaf_values;
  const testsupport::GraphRecipe r = testsupport::random_recipe(rng, max_nodes, leaf_values);
  RecipeBuf& B = g_recipe;
  B = RecipeBuf{};
  B.leaves = leaf_values;
  B.arg_off.push_back(0);
  for (const auto& st : r.steps) {
    B.ops.push_back(static_cast<std::uint8_t>(st.op));
    B.args.insert(B.args.end(), st.args.begin(), st.args.end());
    B.arg_off.push_back(static_cast<std::uint32_t>(B.args.size()));
    B.consts.push_back(st.constant);
  }
  *n_leaves = static_cast<std::uint32_t>(r.leaf_count);
  *n_steps = static_cast<std::uint32_t>(r.steps.size());
  *n_args = static_cast<std::uint32_t>(B.args.size());
  return 0;
}

/// Copies out the recipe produced by the last ref_recipe call on this thread.
void ref_recipe_fetch(double* leaves, std::uint8_t* ops, std::uint32_t* arg_off, std::uint32_t* args,
                      double* consts) {
  const RecipeBuf& B = g_recipe;
  std::copy(B.leaves.begin(), B.leaves.end(), leaves);
  std::copy(B.ops.begin(), B.ops.end(), ops);
  std::copy(B.arg_off.begin(), B.arg_off.end(), arg_off);
  std::copy(B.args.begin(), B.args.end(), args);
  std::copy(B.consts.begin(), B.consts.end(), consts);
}

/// Per sample: GraphRecipe::build on a fresh reference tape, then backward
/// (variant 0) or backward_with_scratch (variant 1).  leaf_values [leaf][batch].
/// Also GraphRecipe::eval (the independent interpreter) into eval_out.
int ref_recipe_eval(std::uint32_t n_leaves, std::uint32_t n_steps, const std::uint8_t* ops,
                    const std::uint32_t* arg_off, const std::uint32_t* args, const double* consts, int dtype,
                    int variant, const double* leaf_values, std::size_t batch, double* root_out,
                    double* leaf_grad_out, double* eval_out, std::uint32_t* n_nodes_out,
                    std::uint64_t* n_edges_out) {
  try {
    const testsupport::GraphRecipe r = unpack(n_leaves, n_steps, ops, arg_off, args, consts);
    auto go = [&](auto tag) -> int {
      using S = decltype(tag);
      std::vector<double> lv(n_leaves);
      tapegrad::ScratchBuffers<S> scratch;
      for (std::size_t s = 0; s < batch; ++s) {
        for (std::uint32_t l = 0; l < n_leaves; ++l) lv[l] = leaf_values[std::size_t(l) * batch + s];
        tapegrad::Tape<S> tape(std::size_t(256));
        const auto refs = r.build(tape, std::span<const double>(lv));
        const tapegrad::ValueRef root = refs.back();
        if (variant == 0) tapegrad::backward(tape, root);
        else tapegrad::backward_with_scratch(tape, root, scratch);
        if (root_out) root_out[s] = static_cast<double>(tape.value_of(root));
        if (leaf_grad_out)
          for (std::uint32_t l = 0; l < n_leaves; ++l) leaf_grad_out[std::size_t(l) * batch + s] = static_cast<double>(tape.grad_of(refs[l]));
        if (eval_out) eval_out[s] = r.eval(std::span<const double>(lv));
        if (s == 0 && n_nodes_out) { *n_nodes_out = tape.size(); *n_edges_out = tape.child_pool_size(); }
      }
      return 0;
    };
    return dtype == 0 ? go(double{}) : go(float{});
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // extern "C"
