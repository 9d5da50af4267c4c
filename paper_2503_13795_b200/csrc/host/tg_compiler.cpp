// tg_compiler.cpp — lowers a recorded tape to the device program.
//
// What the reference does per sample, this does once per tape:
//   * the reverse processing order of backward_with_scratch (iterative DFS
//     post-order from the root, children in stored order, zero-child nodes
//     skipped, backprop.hpp:150-183) depends only on topology, which is
//     sample-invariant, so it is computed here a single time;
//   * zero_grads (backprop.hpp:100-109) becomes "first contribution stores":
//     the compiler knows which reverse-sweep write reaches each adjoint row
//     first;
//   * accumulator adds of the parameter range become
//     batch-reduction terms: for an inner product the contribution of weight
//     y_k is g * x_k (ops.hpp:436-452), so its batch sum is sum_s g(s) x_k(s),
//     a contraction over the sample axis evaluated per CTA tile.
#include <algorithm>
#include <map>
#include <queue>
#include <tuple>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "tg_program.hpp"

namespace tgc {
namespace {

enum Cls : std::uint8_t { cParam, cInput, cConst, cUniform, cSample };

constexpr std::uint8_t ExpOp = 3, DivOp = 16;
constexpr std::uint8_t Leaf = 0, MulByConst = 15, Add = 12, Sub = 13, Mul = 14, Mean = 17,
                       NegativeMean = 20, AddVarying = 21, SubVarying = 22, MeanVarying = 24,
                       NegativeMeanVarying = 27, IPNoBias = 28, IPWithBias = 29,
                       StopGradMax = TG_OP_STOPGRAD_MAX;

bool valid_op(std::uint8_t op) { return op <= 29 || op == StopGradMax; }

std::uint32_t arity_min(std::uint8_t op) {
  if (op == Leaf) return 0;
  if (op <= 11 || op == MulByConst) return 1;
  if (op <= 20) return 2;
  return 1;
}

struct Ctx {
  const tg_tape_desc& d;
  Program& P;
  std::vector<std::uint8_t> cls;
  std::vector<std::uint32_t> row, uv;         // per node
  std::vector<std::uint32_t> grow;            // per gather: materialised row (uniform tables)
  std::vector<std::uint32_t> sg_of;           // per gather: slot-gather table id
  std::vector<std::uint8_t> gkind;            // 0 unused, 1 uniform table, 2 slot table

  std::uint32_t nkids(std::uint32_t i) const {
    return static_cast<std::uint32_t>(d.child_offset[i + 1] - d.child_offset[i]);
  }
  const std::uint32_t* kids(std::uint32_t i) const { return d.child + d.child_offset[i]; }
  std::uint32_t cand(std::uint32_t g, std::uint32_t r) const {
    const tg_gather& G = d.gathers[g];
    return G.first_node + G.stride * r + G.offset;
  }
};

void validate(const tg_tape_desc& d) {
  if (d.n_nodes == 0) throw std::invalid_argument("tg_compile: empty tape");
  if (d.root >= d.n_nodes)
    throw std::invalid_argument("backward: stale root index " + std::to_string(d.root));
  if (d.child_offset[0] != 0) throw std::invalid_argument("tg_compile: child_offset[0] != 0");
  for (std::uint32_t g = 0; g < d.n_gathers; ++g) {
    const tg_gather& G = d.gathers[g];
    if (G.n_rows == 0) throw std::invalid_argument("tg_compile: gather with zero rows");
    const std::uint64_t last = std::uint64_t(G.first_node) + std::uint64_t(G.stride) * (G.n_rows - 1) + G.offset;
    if (last >= d.n_nodes) throw std::invalid_argument("tg_compile: gather table past tape end");
    if (G.index_col >= d.n_index_inputs) throw std::invalid_argument("tg_compile: gather index column out of range");
  }
  for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
    const std::uint8_t op = d.op[i];
    if (!valid_op(op)) throw std::invalid_argument("tg_compile: bad opcode " + std::to_string(op) + " at node " + std::to_string(i));
    const std::uint64_t n = d.child_offset[i + 1] - d.child_offset[i];
    if (d.child_offset[i + 1] < d.child_offset[i]) throw std::invalid_argument("tg_compile: child offsets not monotone");
    if (op == Leaf) {
      if (n != 0) throw std::invalid_argument("tg_compile: leaf with children");
      const std::uint8_t c = d.leaf_class[i];
      if (c == TG_LEAF_PARAM && d.leaf_index[i] >= d.n_params) throw std::invalid_argument("tg_compile: param index out of range");
      if (c == TG_LEAF_INPUT && d.leaf_index[i] >= d.n_inputs) throw std::invalid_argument("tg_compile: input column out of range");
      if (c != TG_LEAF_PARAM && c != TG_LEAF_INPUT && c != TG_LEAF_CONST) throw std::invalid_argument("tg_compile: leaf without a class");
      continue;
    }
    if (n < arity_min(op)) throw std::invalid_argument(std::string(tg_op_name(op)) + ": empty input sequence");
    if (op <= 11 || op == MulByConst) { if (n != 1) throw std::invalid_argument(std::string("unary: op ") + tg_op_name(op) + " needs 1 child"); }
    else if (op <= 20) { if (n != 2) throw std::invalid_argument(std::string("binary: op ") + tg_op_name(op) + " needs 2 children"); }
    else if (op == IPNoBias && (n % 2) != 0) throw std::invalid_argument("innerProduct: odd child count");
    else if (op == IPWithBias && (n % 2) != 1) throw std::invalid_argument("innerProductWithBias: even child count");
    const std::uint32_t* k = d.child + d.child_offset[i];
    for (std::uint64_t j = 0; j < n; ++j) {
      const std::uint32_t c = k[j];
      if (c & TG_GATHER_FLAG) {
        if ((c & ~TG_GATHER_FLAG) >= d.n_gathers) throw std::invalid_argument("tg_compile: bad gather id");
        const tg_gather& G = d.gathers[c & ~TG_GATHER_FLAG];
        if (std::uint64_t(G.first_node) + std::uint64_t(G.stride) * (G.n_rows - 1) + G.offset >= i)
          throw std::invalid_argument("tg_compile: gather table not built before its consumer");
      } else if (c >= i) {
        throw std::invalid_argument("tg_compile: child " + std::to_string(c) + " of node " + std::to_string(i) + " is not earlier (topological order violated)");
      }
    }
  }
}

void classify(Ctx& c) {
  const tg_tape_desc& d = c.d;
  c.cls.assign(d.n_nodes, cConst);
  c.gkind.assign(d.n_gathers, 0);
  auto gather_class = [&](std::uint32_t g) -> std::uint8_t {
    bool any_sample = false, any_uniform = false;
    for (std::uint32_t r = 0; r < d.gathers[g].n_rows; ++r) {
      const std::uint8_t k = c.cls[c.cand(g, r)];
      if (k == cSample || k == cInput) any_sample = true; else any_uniform = true;
    }
    if (any_sample && any_uniform)
      throw std::invalid_argument("tg_compile: gather mixes per-sample and sample-invariant nodes");
    return any_sample ? 2 : 1;
  };
  for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
    if (d.op[i] == Leaf) {
      c.cls[i] = d.leaf_class[i] == TG_LEAF_PARAM ? cParam : d.leaf_class[i] == TG_LEAF_INPUT ? cInput : cConst;
      continue;
    }
    bool sample = false;
    const std::uint32_t* k = c.kids(i);
    for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
      if (k[j] & TG_GATHER_FLAG) {
        const std::uint32_t g = k[j] & ~TG_GATHER_FLAG;
        if (!c.gkind[g]) c.gkind[g] = gather_class(g);
        sample = true;  // a token-selected value differs per sample
      } else if (c.cls[k[j]] == cSample || c.cls[k[j]] == cInput) {
        sample = true;
      }
    }
    c.cls[i] = sample ? cSample : cUniform;
  }
}

// Processing order of backward_with_scratch (backprop.hpp:150-183) over the
// union of all per-sample wirings (a gather visits its candidates in row
// order; for model tapes this coincides with every concrete sample's order).
std::vector<std::uint32_t> processing_order(const Ctx& c) {
  const tg_tape_desc& d = c.d;
  std::vector<std::uint8_t> seen(d.n_nodes, 0);
  std::vector<std::uint32_t> post;
  auto bwd_kids = [&](std::uint32_t i, std::vector<std::uint32_t>& out) {
    out.clear();
    if (d.op[i] == StopGradMax || d.op[i] == Leaf) return;
    const std::uint32_t* k = c.kids(i);
    for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
      if (k[j] & TG_GATHER_FLAG) {
        const std::uint32_t g = k[j] & ~TG_GATHER_FLAG;
        for (std::uint32_t r = 0; r < d.gathers[g].n_rows; ++r) out.push_back(c.cand(g, r));
      } else {
        out.push_back(k[j]);
      }
    }
  };
  struct Frame { std::uint32_t node; std::uint32_t cur; std::vector<std::uint32_t> kids; };
  std::vector<Frame> st;
  seen[d.root] = 1;
  Frame f0{d.root, 0, {}};
  bwd_kids(d.root, f0.kids);
  if (!f0.kids.empty()) st.push_back(std::move(f0));
  while (!st.empty()) {
    Frame& top = st.back();
    if (top.cur < top.kids.size()) {
      const std::uint32_t ch = top.kids[top.cur++];
      if (!seen[ch]) {
        seen[ch] = 1;
        Frame f{ch, 0, {}};
        bwd_kids(ch, f.kids);
        if (!f.kids.empty()) st.push_back(std::move(f));
      }
    } else {
      post.push_back(top.node);
      st.pop_back();
    }
  }
  std::reverse(post.begin(), post.end());
  return post;  // processing order (children after parents)
}

// ---- softmax attention heads in the recorded graph (kAttn) -------------------
// One query unit of a head is the node pattern the reference ops produce for
// softmax(scale * q K^T) V:
//   s_j = innerProduct(q, k_j)      c_j = mulByConstant(s_j, scale)
//   m   = stopGradMax(c_0..c_{n-1}) sh_j = c_j - m      e_j = exp(sh_j)
//   Z   = reduceSum(e_0..e_{n-1})   a_j = e_j / Z
//   o_i = innerProduct(a_0..a_{n-1}, v_0[i]..v_{n-1}[i])
// with q, k_j, v_j blocks of consecutive nodes.  Matching is structural and
// exact (op, children in order, consumer counts), so a fused head computes
// the same function; anything that does not match stays scalar.
struct AttnUnit {
  std::uint32_t q0 = 0, n = 0;
  std::vector<std::uint32_t> kb, vb, o, interior;
};
struct AttnGroup {
  std::uint32_t hd = 0, dv = 0;
  double scale = 0;
  std::vector<AttnUnit> units;
  std::vector<std::uint32_t> kb, vb;   // longest key list
  std::uint32_t last_o = 0, first_node = 0;
  bool ok = true;
};

std::vector<AttnGroup> find_attention(const Ctx& c, const std::vector<std::uint32_t>& order) {
  const tg_tape_desc& d = c.d;
  const std::uint32_t N = d.n_nodes;
  std::vector<AttnGroup> groups;
  if (!d.constant) return groups;
  std::vector<std::uint8_t> pinned(N, 0), reach(N, 0);
  pinned[d.root] = 1;
  for (std::uint32_t g = 0; g < d.n_gathers; ++g)
    for (std::uint32_t r = 0; r < d.gathers[g].n_rows; ++r) pinned[c.cand(g, r)] = 1;
  for (std::uint32_t nd : order) reach[nd] = 1;
  std::vector<std::uint32_t> ccount(N, 0), cfirst(N, kNone), cmin(N, kNone);
  std::vector<std::uint32_t> coff(N + 1, 0), cons;
  for (std::uint32_t i = 0; i < N; ++i)
    for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
      const std::uint32_t k = c.kids(i)[j];
      if (k & TG_GATHER_FLAG) continue;
      ++ccount[k];
      ++coff[k + 1];
      cmin[k] = std::min(cmin[k], i);
    }
  for (std::uint32_t i = 0; i < N; ++i) coff[i + 1] += coff[i];
  cons.resize(coff[N]);
  {
    std::vector<std::uint32_t> fill(coff.begin(), coff.end() - 1);
    for (std::uint32_t i = 0; i < N; ++i)
      for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
        const std::uint32_t k = c.kids(i)[j];
        if (!(k & TG_GATHER_FLAG)) cons[fill[k]++] = i;
      }
  }
  auto plain = [&](std::uint32_t x) { return !(x & TG_GATHER_FLAG) && x < N; };
  auto free_node = [&](std::uint32_t x) { return plain(x) && c.cls[x] == cSample && !pinned[x] && reach[x]; };
  std::map<std::tuple<std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t, double>, std::uint32_t> gid;
  for (std::uint32_t Z = 0; Z < N; ++Z) {
    if (d.op[Z] != AddVarying || !free_node(Z)) continue;
    const std::uint32_t n = c.nkids(Z);
    const std::uint32_t* e = c.kids(Z);
    AttnUnit U;
    U.n = n;
    bool ok = n >= 1 && ccount[Z] == n;
    std::uint32_t m = kNone, hd = 0;
    double scale = 0;
    std::vector<std::uint32_t> cj(n), aj(n);
    for (std::uint32_t j = 0; ok && j < n; ++j) {
      const std::uint32_t ej = e[j];
      ok = free_node(ej) && d.op[ej] == ExpOp && c.nkids(ej) == 1 && ccount[ej] == 2;
      if (!ok) break;
      const std::uint32_t sh = c.kids(ej)[0];
      ok = free_node(sh) && d.op[sh] == Sub && ccount[sh] == 1;
      if (!ok) break;
      const std::uint32_t cc = c.kids(sh)[0], mm = c.kids(sh)[1];
      if (j == 0) m = mm;
      ok = free_node(cc) && plain(mm) && mm == m && d.op[cc] == MulByConst && ccount[cc] == 2;
      if (!ok) break;
      if (j == 0) scale = d.constant[cc];
      ok = d.constant[cc] == scale;
      const std::uint32_t sj = c.kids(cc)[0];
      ok = ok && free_node(sj) && d.op[sj] == IPNoBias && ccount[sj] == 1 && c.nkids(sj) >= 2 && c.nkids(sj) % 2 == 0;
      if (!ok) break;
      const std::uint32_t h = c.nkids(sj) / 2;
      if (j == 0) { hd = h; U.q0 = c.kids(sj)[0]; }
      ok = h == hd;
      const std::uint32_t* sk = c.kids(sj);
      for (std::uint32_t i = 0; ok && i < hd; ++i)
        ok = plain(sk[i]) && plain(sk[hd + i]) && sk[i] == U.q0 + i && sk[hd + i] == sk[hd] + i;
      if (!ok) break;
      U.kb.push_back(sk[hd]);
      cj[j] = cc;
      // a_j: the consumer of e_j other than Z, a_j = e_j / Z
      std::uint32_t a = kNone;
      for (std::uint32_t q = coff[ej]; q < coff[ej + 1]; ++q)
        if (cons[q] != Z) a = cons[q];
      ok = a != kNone && free_node(a) && d.op[a] == DivOp && c.kids(a)[0] == ej && c.kids(a)[1] == Z;
      aj[j] = a;
      U.interior.insert(U.interior.end(), {ej, sh, cc, sj});
    }
    // (the shift has no reverse children, so it is absent from the processing order)
    ok = ok && m != kNone && plain(m) && c.cls[m] == cSample && !pinned[m] && d.op[m] == StopGradMax && c.nkids(m) == n && ccount[m] == n;
    for (std::uint32_t j = 0; ok && j < n; ++j) ok = c.kids(m)[j] == cj[j];
    if (!ok) continue;
    // outputs: the consumers of a_0, each o_i = innerProduct(a_0..a_{n-1}, v_0[i]..v_{n-1}[i])
    for (std::uint32_t q = coff[aj[0]]; q < coff[aj[0] + 1]; ++q) U.o.push_back(cons[q]);
    std::sort(U.o.begin(), U.o.end());
    const std::uint32_t dv = static_cast<std::uint32_t>(U.o.size());
    ok = dv >= 1;
    for (std::uint32_t j = 0; ok && j < n; ++j) ok = ccount[aj[j]] == dv;
    for (std::uint32_t i = 0; ok && i < dv; ++i) {
      const std::uint32_t o = U.o[i];
      ok = plain(o) && c.cls[o] == cSample && reach[o] && d.op[o] == IPNoBias && c.nkids(o) == 2 * n;
      for (std::uint32_t j = 0; ok && j < n; ++j) ok = c.kids(o)[j] == aj[j] && plain(c.kids(o)[n + j]);
      if (ok && i > 0) ok = U.o[i] == U.o[0] + i;
    }
    for (std::uint32_t j = 0; ok && j < n; ++j) {
      const std::uint32_t v0 = c.kids(U.o[0])[n + j];
      U.vb.push_back(v0);
      for (std::uint32_t i = 1; ok && i < dv; ++i) ok = c.kids(U.o[i])[n + j] == v0 + i;
    }
    if (!ok) continue;
    U.interior.push_back(m);
    U.interior.push_back(Z);
    U.interior.insert(U.interior.end(), aj.begin(), aj.end());
    const auto key = std::make_tuple(U.kb[0], U.vb[0], hd, dv, scale);
    auto it = gid.find(key);
    if (it == gid.end()) {
      it = gid.emplace(key, static_cast<std::uint32_t>(groups.size())).first;
      groups.emplace_back();
      groups.back().hd = hd;
      groups.back().dv = dv;
      groups.back().scale = scale;
    }
    groups[it->second].units.push_back(std::move(U));
  }
  // group checks: prefix key lists, disjoint q / k / v / o blocks whose every
  // consumer is inside the group, outputs consumed only after the last one
  for (AttnGroup& G : groups) {
    for (const AttnUnit& U : G.units)
      if (U.kb.size() > G.kb.size()) { G.kb = U.kb; G.vb = U.vb; }
    const std::uint32_t T = static_cast<std::uint32_t>(G.kb.size());
    std::vector<std::uint32_t> users(T, 0);
    std::unordered_map<std::uint32_t, std::uint32_t> owner;   // node -> role
    auto claim = [&](std::uint32_t x, std::uint32_t role) {
      if (!plain(x) || pinned[x] || (c.cls[x] != cSample && c.cls[x] != cInput) || owner.count(x)) return false;
      owner[x] = role;
      return true;
    };
    G.first_node = kNone;
    for (const AttnUnit& U : G.units) {
      for (std::uint32_t j = 0; G.ok && j < U.n; ++j) G.ok = U.kb[j] == G.kb[j] && U.vb[j] == G.vb[j];
      for (std::uint32_t j = 0; j < U.n && j < T; ++j) ++users[j];
      for (std::uint32_t i = 0; G.ok && i < G.hd; ++i) G.ok = claim(U.q0 + i, 0) && ccount[U.q0 + i] == U.n;
      for (std::uint32_t x : U.o) G.last_o = std::max(G.last_o, x);
      for (std::uint32_t x : U.interior) G.first_node = std::min(G.first_node, x);
    }
    for (std::uint32_t j = 0; G.ok && j < T; ++j) {
      for (std::uint32_t i = 0; G.ok && i < G.hd; ++i) G.ok = claim(G.kb[j] + i, 1) && ccount[G.kb[j] + i] == users[j];
      for (std::uint32_t i = 0; G.ok && i < G.dv; ++i) G.ok = claim(G.vb[j] + i, 2) && ccount[G.vb[j] + i] == users[j];
    }
    for (const AttnUnit& U : G.units)
      for (std::uint32_t x : U.o) G.ok = G.ok && (cmin[x] == kNone || cmin[x] > G.last_o) && !owner.count(x);
  }
  groups.erase(std::remove_if(groups.begin(), groups.end(), [](const AttnGroup& G) { return !G.ok; }), groups.end());
  return groups;
}

// ---- layer normalisations in the recorded graph (kLNorm) ----------------------
// The node pattern of SPEC.md:288-296 built from reference ops (tg_models.hpp
// layer_norm): mu = meanVarying(x), ms = meanSquaresVarying(x), mu2 = mu^2,
// var = ms - mu2, ve = var + eps, rstd = invSqrt(ve), and per element
// c_i = x_i - mu, n_i = c_i * rstd, g_i = n_i * gamma_i, y_i = g_i + beta_i
// (gamma, beta parameters).  Exact structural match with consumer counts.
struct LnMatch {
  std::vector<std::uint32_t> x, nn, y, gamma, beta, interior;
  std::uint32_t rstd = 0, last_y = 0, first_node = 0;
  double eps = 0;
};

std::vector<LnMatch> find_layernorm(const Ctx& c, const std::vector<std::uint32_t>& order) {
  const tg_tape_desc& d = c.d;
  const std::uint32_t N = d.n_nodes;
  std::vector<LnMatch> out;
  if (!d.leaf_value) return out;
  constexpr std::uint8_t SqrOp = 7, InvSqrtOp = 11, MeanVaryingOp = 24, MeanSquaresVaryingOp = 26;
  std::vector<std::uint8_t> pinned(N, 0), reach(N, 0);
  pinned[d.root] = 1;
  for (std::uint32_t g = 0; g < d.n_gathers; ++g)
    for (std::uint32_t r = 0; r < d.gathers[g].n_rows; ++r) pinned[c.cand(g, r)] = 1;
  for (std::uint32_t nd : order) reach[nd] = 1;
  std::vector<std::uint32_t> ccount(N, 0), cmin(N, kNone), coff(N + 1, 0), cons;
  for (std::uint32_t i = 0; i < N; ++i)
    for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
      const std::uint32_t k = c.kids(i)[j];
      if (k & TG_GATHER_FLAG) continue;
      ++ccount[k];
      ++coff[k + 1];
      cmin[k] = std::min(cmin[k], i);
    }
  for (std::uint32_t i = 0; i < N; ++i) coff[i + 1] += coff[i];
  cons.resize(coff[N]);
  {
    std::vector<std::uint32_t> fill(coff.begin(), coff.end() - 1);
    for (std::uint32_t i = 0; i < N; ++i)
      for (std::uint32_t j = 0; j < c.nkids(i); ++j) {
        const std::uint32_t k = c.kids(i)[j];
        if (!(k & TG_GATHER_FLAG)) cons[fill[k]++] = i;
      }
  }
  auto plain = [&](std::uint32_t x) { return !(x & TG_GATHER_FLAG) && x < N; };
  auto interior_ok = [&](std::uint32_t x) { return plain(x) && c.cls[x] == cSample && !pinned[x]; };
  auto kid = [&](std::uint32_t i, std::uint32_t j) { return c.kids(i)[j]; };
  std::vector<std::uint8_t> used(N, 0);
  for (std::uint32_t mu = 0; mu < N; ++mu) {
    if (d.op[mu] != MeanVaryingOp || !interior_ok(mu) || used[mu]) continue;
    const std::uint32_t n = c.nkids(mu);
    if (n < 2 || ccount[mu] != n + 1) continue;
    LnMatch M;
    bool ok = true;
    for (std::uint32_t i = 0; ok && i < n; ++i) {
      const std::uint32_t xi = kid(mu, i);
      ok = plain(xi) && (c.cls[xi] == cSample || c.cls[xi] == cInput);
      for (std::uint32_t j = 0; ok && j < i; ++j) ok = kid(mu, j) != xi;
      M.x.push_back(xi);
    }
    if (!ok) continue;
    std::uint32_t ms = kNone, mu2 = kNone;
    for (std::uint32_t q = coff[M.x[0]]; q < coff[M.x[0] + 1]; ++q) {
      const std::uint32_t cand = cons[q];
      if (d.op[cand] != MeanSquaresVaryingOp || c.nkids(cand) != n) continue;
      bool same = true;
      for (std::uint32_t i = 0; same && i < n; ++i) same = kid(cand, i) == M.x[i];
      if (same) ms = cand;
    }
    ok = ms != kNone && interior_ok(ms) && ccount[ms] == 1;
    // consumers of mu: mu^2 and the n centred values (x_i - mu)
    std::vector<std::uint32_t> cidx(n, kNone);
    for (std::uint32_t q = coff[mu]; ok && q < coff[mu + 1]; ++q) {
      const std::uint32_t u = cons[q];
      if (d.op[u] == SqrOp && c.nkids(u) == 1) {
        ok = mu2 == kNone;
        mu2 = u;
        continue;
      }
      ok = d.op[u] == Sub && c.nkids(u) == 2 && kid(u, 1) == mu;
      std::uint32_t i = 0;
      while (ok && i < n && M.x[i] != kid(u, 0)) ++i;
      ok = ok && i < n && cidx[i] == kNone;
      if (ok) cidx[i] = u;
    }
    ok = ok && mu2 != kNone && interior_ok(mu2) && ccount[mu2] == 1;
    if (!ok) continue;
    const std::uint32_t var = cons[coff[mu2]];
    ok = interior_ok(var) && d.op[var] == Sub && kid(var, 0) == ms && kid(var, 1) == mu2 && ccount[var] == 1 &&
         cons[coff[ms]] == var;
    if (!ok) continue;
    const std::uint32_t ve = cons[coff[var]];
    ok = interior_ok(ve) && d.op[ve] == Add && kid(ve, 0) == var && plain(kid(ve, 1)) && c.cls[kid(ve, 1)] == cConst &&
         d.op[kid(ve, 1)] == Leaf && ccount[ve] == 1;
    if (!ok) continue;
    M.eps = d.leaf_value[kid(ve, 1)];
    const std::uint32_t rstd = cons[coff[ve]];
    ok = interior_ok(rstd) && d.op[rstd] == InvSqrtOp && ccount[rstd] == n;
    for (std::uint32_t i = 0; ok && i < n; ++i) {
      const std::uint32_t ci = cidx[i];
      ok = ci != kNone && interior_ok(ci) && ccount[ci] == 1;
      if (!ok) break;
      const std::uint32_t ni = cons[coff[ci]];
      ok = interior_ok(ni) && reach[ni] && d.op[ni] == Mul && kid(ni, 0) == ci && kid(ni, 1) == rstd && ccount[ni] == 1;
      if (!ok) break;
      const std::uint32_t gi = cons[coff[ni]];
      ok = interior_ok(gi) && d.op[gi] == Mul && kid(gi, 0) == ni && plain(kid(gi, 1)) && c.cls[kid(gi, 1)] == cParam &&
           ccount[gi] == 1;
      if (!ok) break;
      const std::uint32_t yi = cons[coff[gi]];
      ok = plain(yi) && c.cls[yi] == cSample && !pinned[yi] && reach[yi] && d.op[yi] == Add && kid(yi, 0) == gi &&
           plain(kid(yi, 1)) && c.cls[kid(yi, 1)] == cParam;
      if (!ok) break;
      M.nn.push_back(ni);
      M.y.push_back(yi);
      M.gamma.push_back(d.leaf_index[kid(gi, 1)]);
      M.beta.push_back(d.leaf_index[kid(yi, 1)]);
      M.interior.push_back(ci);
      M.interior.push_back(gi);
      M.last_y = std::max(M.last_y, yi);
    }
    for (std::uint32_t i = 0; ok && i < n; ++i) ok = cmin[M.y[i]] == kNone || cmin[M.y[i]] > M.last_y;
    if (!ok) continue;
    M.rstd = rstd;
    M.interior.insert(M.interior.end(), {mu, ms, mu2, var, ve, rstd});
    M.first_node = *std::min_element(M.interior.begin(), M.interior.end());
    for (std::uint32_t x : M.interior) used[x] = 1;
    out.push_back(std::move(M));
  }
  return out;
}

}  // namespace

Program compile(const tg_tape_desc& d) {
  validate(d);
  Program P;
  P.dtype = d.dtype;
  P.n_nodes = d.n_nodes;
  P.n_params = d.n_params;
  P.n_inputs = d.n_inputs;
  P.n_index_inputs = d.n_index_inputs;
  P.n_edges = d.child_offset[d.n_nodes];
  Ctx c{d, P, {}, {}, {}, {}, {}, {}};
  classify(c);

  // ---- uniform value table: [params | uniform nodes | constants] ----------
  c.uv.assign(d.n_nodes, kNone);
  P.uv_uniform_base = d.n_params;
  std::uint32_t nu = 0, nc = 0;
  for (std::uint32_t i = 0; i < d.n_nodes; ++i) if (c.cls[i] == cUniform) ++nu; else if (c.cls[i] == cConst) ++nc;
  P.uv_const_base = d.n_params + nu;
  P.n_uv = d.n_params + nu + nc;
  P.uv_init.assign(P.n_uv, 0.0);
  {
    std::uint32_t ku = 0, kc = 0;
    for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
      switch (c.cls[i]) {
        case cParam: c.uv[i] = d.leaf_index[i]; P.uv_init[c.uv[i]] = d.leaf_value ? d.leaf_value[i] : 0.0; break;
        case cUniform: c.uv[i] = P.uv_uniform_base + ku++; break;
        case cConst: c.uv[i] = P.uv_const_base + kc; P.uv_init[c.uv[i]] = d.leaf_value ? d.leaf_value[i] : 0.0; ++kc; break;
        default: break;
      }
    }
  }
  P.n_uniform_nodes = nu;

  // ---- softmax attention heads (kAttn): interior nodes get no rows ------------
  std::vector<AttnGroup> agroups = find_attention(c, processing_order(c));
  std::vector<std::int32_t> attn_of(d.n_nodes, -1);      // interior and output nodes -> group
  std::vector<std::uint8_t> attn_interior(d.n_nodes, 0);
  for (std::size_t g = 0; g < agroups.size(); ++g)
    for (const AttnUnit& U : agroups[g].units) {
      for (std::uint32_t x : U.interior) { attn_of[x] = static_cast<std::int32_t>(g); attn_interior[x] = 1; }
      for (std::uint32_t x : U.o) attn_of[x] = static_cast<std::int32_t>(g);
    }

  std::vector<LnMatch> lns = find_layernorm(c, processing_order(c));
  std::vector<std::int32_t> ln_of(d.n_nodes, -1);        // interior, n_i and y_i nodes -> instance
  for (std::size_t g = 0; g < lns.size(); ++g) {
    bool clash = false;   // an attention head already owns one of its nodes
    for (std::uint32_t x : lns[g].interior) clash = clash || attn_of[x] >= 0;
    for (std::uint32_t x : lns[g].y) clash = clash || attn_of[x] >= 0;
    if (clash) { lns[g].x.clear(); continue; }
    for (std::uint32_t x : lns[g].interior) { ln_of[x] = static_cast<std::int32_t>(g); attn_interior[x] = 1; }
    for (std::uint32_t x : lns[g].nn) ln_of[x] = static_cast<std::int32_t>(g);
    for (std::uint32_t x : lns[g].y) ln_of[x] = static_cast<std::int32_t>(g);
  }

  // ---- per-sample rows -------------------------------------------------------
  c.row.assign(d.n_nodes, kNone);
  std::uint32_t nrow = 0;
  P.input_rows.assign(d.n_inputs, kNone);
  for (std::uint32_t i = 0; i < d.n_nodes; ++i)
    if (c.cls[i] == cInput) {
      const std::uint32_t col = d.leaf_index[i];
      if (P.input_rows[col] != kNone)
        throw std::invalid_argument("tg_compile: input column " + std::to_string(col) + " bound to two leaves");
      c.row[i] = nrow++;
      P.input_rows[col] = c.row[i];
      Instr in{kInputLoad, Leaf, 0, c.row[i], 0, 0, col, i, 0.0};
      P.fwd.push_back(in);
    }
  c.grow.assign(d.n_gathers, kNone);
  c.sg_of.assign(d.n_gathers, kNone);
  for (std::uint32_t g = 0; g < d.n_gathers; ++g) {
    if (!c.gkind[g]) continue;
    GatherTable T{d.gathers[g].index_col, d.gathers[g].n_rows, static_cast<std::uint32_t>(P.cand.size()), 0};
    if (c.gkind[g] == 1) {
      for (std::uint32_t r = 0; r < T.n_rows; ++r) P.cand.push_back(c.uv[c.cand(g, r)]);
      c.grow[g] = nrow++;
      const std::uint32_t id = static_cast<std::uint32_t>(P.ugather.size());
      P.ugather.push_back(T);
      Instr gl{kGatherLoad, Leaf, 0, c.grow[g], 0, 0, id, d.gathers[g].first_node, 0.0};
      P.fwd.push_back(gl);
    }
  }
  // x-row blocks: the x operands of an inner product over a parameter row
  // (a dense-layer candidate) get consecutive rows in operand order, so the
  // staged tier can run the layer as one GEMM over a row block even when the
  // producer interleaves them (layer-norm outputs, attention heads).  A block
  // is placed where its first member appears; every other node keeps its
  // order.  Rows are storage slots only: the numbering does not change any
  // result.
  std::vector<std::uint32_t> blk_of(d.n_nodes, kNone);
  std::vector<std::vector<std::uint32_t>> blocks;
  {
    std::vector<std::uint8_t> mark(d.n_nodes, 0);
    auto param_ip = [&](std::uint32_t i) {   // IP over a consecutive parameter row
      if (c.cls[i] != cSample || (d.op[i] != IPNoBias && d.op[i] != IPWithBias)) return 0u;
      const std::uint32_t n = c.nkids(i), m = d.op[i] == IPWithBias ? (n - 1) / 2 : n / 2;
      const std::uint32_t* k = c.kids(i);
      for (std::uint32_t j = 0; j < m; ++j) {
        const std::uint32_t y = k[m + j];
        if ((y & TG_GATHER_FLAG) || c.cls[y] != cParam || d.leaf_index[y] != d.leaf_index[k[m]] + j) return 0u;
      }
      return m;
    };
    for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
      const std::uint32_t m = param_ip(i);
      if (m < 8) continue;
      const std::uint32_t* k = c.kids(i);
      bool ok = true, increasing = true;
      for (std::uint32_t j = 0; ok && j < m; ++j) {
        const std::uint32_t x = k[j];
        ok = !(x & TG_GATHER_FLAG) && c.cls[x] == cSample && blk_of[x] == kNone && !mark[x];
        if (ok) mark[x] = 1;
        if (j && x <= k[j - 1]) increasing = false;
      }
      for (std::uint32_t j = 0; j < m; ++j) if (!(k[j] & TG_GATHER_FLAG)) mark[k[j]] = 0;
      if (!ok) continue;   // shared with another block (or the same x list again)
      // members that are themselves dense outputs keep their node order
      if (!increasing)
        for (std::uint32_t j = 0; ok && j < m; ++j) ok = param_ip(k[j]) == 0;
      if (!ok) continue;
      const std::uint32_t id = static_cast<std::uint32_t>(blocks.size());
      blocks.emplace_back(k, k + m);
      for (std::uint32_t j = 0; j < m; ++j) blk_of[k[j]] = id;
    }
  }
  for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
    if (c.cls[i] != cSample || c.row[i] != kNone || attn_interior[i]) continue;
    if (blk_of[i] != kNone) {
      for (std::uint32_t x : blocks[blk_of[i]]) { c.row[x] = nrow++; ++P.n_sample_nodes; }
    } else {
      c.row[i] = nrow++;
      ++P.n_sample_nodes;
    }
  }
  // attention blocks must be consecutive rows; a head whose blocks are not
  // falls back to scalar nodes (its interior rows appended here)
  for (std::size_t g = 0; g < agroups.size(); ++g) {
    AttnGroup& G = agroups[g];
    auto consec = [&](std::uint32_t x0, std::uint32_t n) {
      for (std::uint32_t i = 0; i < n; ++i)
        if (c.row[x0 + i] == kNone || c.row[x0 + i] != c.row[x0] + i) return false;
      return true;
    };
    bool ok = true;
    for (const AttnUnit& U : G.units) ok = ok && consec(U.q0, G.hd) && consec(U.o[0], G.dv);
    for (std::size_t j = 0; ok && j < G.kb.size(); ++j) ok = consec(G.kb[j], G.hd) && consec(G.vb[j], G.dv);
    if (ok) {
      for (const AttnUnit& U : G.units) P.n_sample_nodes += static_cast<std::uint32_t>(U.interior.size());
      continue;
    }
    G.ok = false;
    for (const AttnUnit& U : G.units) {
      for (std::uint32_t x : U.interior) { attn_of[x] = -1; attn_interior[x] = 0; c.row[x] = nrow++; ++P.n_sample_nodes; }
      for (std::uint32_t x : U.o) attn_of[x] = -1;
    }
  }
  std::vector<std::uint32_t> ln_id(lns.size(), kNone);
  for (std::size_t g = 0; g < lns.size(); ++g) {
    const LnMatch& M = lns[g];
    if (M.x.empty()) continue;
    LNorm L{};
    L.n = static_cast<std::uint32_t>(M.x.size());
    L.off = static_cast<std::uint32_t>(P.lnrows.size());
    for (std::uint32_t x : M.x) P.lnrows.push_back(c.row[x]);
    for (std::uint32_t x : M.nn) P.lnrows.push_back(c.row[x]);
    for (std::uint32_t x : M.y) P.lnrows.push_back(c.row[x]);
    P.lnrows.insert(P.lnrows.end(), M.gamma.begin(), M.gamma.end());
    P.lnrows.insert(P.lnrows.end(), M.beta.begin(), M.beta.end());
    L.flag_off = static_cast<std::uint32_t>(P.lnflag.size());
    P.lnflag.resize(P.lnflag.size() + L.n, 0);
    L.rstd_node = M.rstd;
    L.first_node = M.first_node;
    L.n_nodes = static_cast<std::uint32_t>(M.interior.size() + 2 * M.x.size());
    L.eps = M.eps;
    ln_id[g] = static_cast<std::uint32_t>(P.lnorm.size());
    P.lnorm.push_back(L);
    P.n_sample_nodes += static_cast<std::uint32_t>(M.interior.size());
  }
  std::vector<std::uint32_t> attn_id(agroups.size(), kNone);
  for (std::size_t g = 0; g < agroups.size(); ++g) {
    const AttnGroup& G = agroups[g];
    if (!G.ok) continue;
    Attn A{};
    A.n_units = static_cast<std::uint32_t>(G.units.size());
    A.n_keys = static_cast<std::uint32_t>(G.kb.size());
    A.hd = G.hd;
    A.dv = G.dv;
    A.unit_off = static_cast<std::uint32_t>(P.arows.size());
    for (const AttnUnit& U : G.units) P.arows.insert(P.arows.end(), {c.row[U.q0], c.row[U.o[0]], U.n});
    A.key_off = static_cast<std::uint32_t>(P.arows.size());
    for (std::size_t j = 0; j < G.kb.size(); ++j) P.arows.insert(P.arows.end(), {c.row[G.kb[j]], c.row[G.vb[j]]});
    A.first_node = G.first_node;
    A.n_nodes = 0;
    for (const AttnUnit& U : G.units) A.n_nodes += static_cast<std::uint32_t>(U.interior.size() + U.o.size());
    A.scale = G.scale;
    A.stat_row = nrow;
    nrow += 2 * A.n_units;
    attn_id[g] = static_cast<std::uint32_t>(P.attn.size());
    P.attn.push_back(A);
  }

  // slot-gather candidate tables (rows are known now)
  for (std::uint32_t g = 0; g < d.n_gathers; ++g) {
    if (c.gkind[g] != 2) continue;
    GatherTable T{d.gathers[g].index_col, d.gathers[g].n_rows, static_cast<std::uint32_t>(P.cand.size()), 0};
    for (std::uint32_t r = 0; r < T.n_rows; ++r) P.cand.push_back(c.row[c.cand(g, r)]);
    c.sg_of[g] = static_cast<std::uint32_t>(P.sgather.size());
    P.sgather.push_back(T);
  }

  auto operand = [&](std::uint32_t ch) -> std::uint32_t {
    if (ch & TG_GATHER_FLAG) {
      const std::uint32_t g = ch & ~TG_GATHER_FLAG;
      return c.gkind[g] == 1 ? enc(kSlot, c.grow[g]) : enc(kSGather, c.sg_of[g]);
    }
    const std::uint8_t k = c.cls[ch];
    if (k == cSample || k == cInput) return enc(kSlot, c.row[ch]);
    return enc(kUv, c.uv[ch]);
  };

  // ---- forward streams -------------------------------------------------------
  std::vector<std::uint32_t> instr_of(d.n_nodes, kNone);   // per-sample node -> fwd index
  std::vector<std::uint32_t> uinstr_of(d.n_nodes, kNone);  // uniform node -> ufwd index
  for (std::uint32_t i = 0; i < d.n_nodes; ++i) {
    if (c.cls[i] != cSample && c.cls[i] != cUniform) continue;
    if (ln_of[i] >= 0) {     // fused layer norm: one instruction where its last output stood
      const LnMatch& M = lns[ln_of[i]];
      if (i == M.last_y) {
        const LNorm& L = P.lnorm[ln_id[ln_of[i]]];
        P.fwd.push_back(Instr{kLNorm, 0, 0, P.lnrows[L.off + 2 * L.n], 0, 0, ln_id[ln_of[i]], L.first_node, L.eps});
      }
      continue;
    }
    if (attn_of[i] >= 0) {   // fused head: one instruction where its last output node stood
      const AttnGroup& G = agroups[attn_of[i]];
      if (i == G.last_o) {
        const Attn& A = P.attn[attn_id[attn_of[i]]];
        P.fwd.push_back(Instr{kAttn, 0, 0, P.arows[A.unit_off + 1], 0, 0, attn_id[attn_of[i]], A.first_node, 0.0});
      }
      continue;
    }
    Instr in{};
    in.kind = kNode;
    in.op = d.op[i];
    in.nops = c.nkids(i);
    in.opnd = static_cast<std::uint32_t>(P.opnd.size());
    in.node = i;
    in.cst = d.constant ? d.constant[i] : 0.0;
    for (std::uint32_t j = 0; j < in.nops; ++j) {
      P.opnd.push_back(operand(c.kids(i)[j]));
      P.oflag.push_back(0);
      P.oaux.push_back(kNone);
    }
    if (c.cls[i] == cSample) {
      in.out = c.row[i];
      instr_of[i] = static_cast<std::uint32_t>(P.fwd.size());
      P.fwd.push_back(in);
    } else {
      in.out = c.uv[i];
      uinstr_of[i] = static_cast<std::uint32_t>(P.ufwd.size());
      P.ufwd.push_back(in);
    }
  }

  P.order = processing_order(c);

  // ---- dense layers (kDense) -----------------------------------------------------
  // A run of consecutive per-sample inner products over the same x rows whose
  // y operands walk a row-major parameter block, plus (when each output's only
  // consumer is one) the elementwise activation run that follows, becomes one
  // macro-instruction: forward = loop over outputs, reverse = activation
  // derivative + x-adjoint accumulation, weight gradients = outer products.
  std::vector<std::int32_t> dense_of(d.n_nodes, -1);
  const std::vector<Instr> nodefwd = P.fwd;
  {
    std::vector<std::uint32_t> uses(nrow + 1, 0);
    std::vector<std::uint8_t> reach(d.n_nodes, 0);
    for (std::uint32_t nd : P.order) reach[nd] = 1;
    for (const Instr& in : nodefwd) {
      if (in.kind != kNode) continue;
      for (std::uint32_t j = 0; j < in.nops; ++j) {
        const std::uint32_t o = P.opnd[in.opnd + j];
        if ((o >> kModeShift) == kSlot) ++uses[o & kIndexMask];
        else if ((o >> kModeShift) == kSGather) {
          const GatherTable& T = P.sgather[o & kIndexMask];
          for (std::uint32_t r = 0; r < T.n_rows; ++r) uses[P.cand[T.cand_off + r]] += 2;
        }
      }
    }
    if (c.cls[d.root] == cSample) uses[c.row[d.root]] += 2;
    for (const LNorm& L : P.lnorm)   // rows read by fused layer norms
      for (std::uint32_t i = 0; i < L.n; ++i) uses[P.lnrows[L.off + i]] += 2;
    for (const Attn& A : P.attn) {   // rows read by fused heads
      for (std::uint32_t u = 0; u < A.n_units; ++u)
        for (std::uint32_t i = 0; i < A.hd; ++i) uses[P.arows[A.unit_off + 3 * u] + i] += 2;
      for (std::uint32_t j = 0; j < A.n_keys; ++j) {
        for (std::uint32_t i = 0; i < A.hd; ++i) uses[P.arows[A.key_off + 2 * j] + i] += 2;
        for (std::uint32_t i = 0; i < A.dv; ++i) uses[P.arows[A.key_off + 2 * j + 1] + i] += 2;
      }
    }
    auto ip_shape = [&](std::uint32_t node, std::uint32_t& xo, std::uint32_t& m, std::uint32_t& w, std::uint32_t& b) -> bool {
      if (node >= d.n_nodes || c.cls[node] != cSample || !reach[node] || (d.op[node] != IPNoBias && d.op[node] != IPWithBias) ||
          attn_of[node] >= 0)
        return false;
      const Instr& in = nodefwd[instr_of[node]];
      const bool bias = d.op[node] == IPWithBias;
      m = bias ? (in.nops - 1) / 2 : in.nops / 2;
      xo = in.opnd;
      for (std::uint32_t k = 0; k < m; ++k) {
        const std::uint32_t xk = P.opnd[in.opnd + k], yk = P.opnd[in.opnd + m + k];
        if ((xk >> kModeShift) != kSlot || (yk >> kModeShift) != kUv) return false;
        if (k == 0) w = yk & kIndexMask;
        if ((yk & kIndexMask) != w + k || w + k >= d.n_params) return false;
      }
      b = kNone;
      if (bias) {
        const std::uint32_t bo = P.opnd[in.opnd + in.nops - 1];
        if ((bo >> kModeShift) != kUv || (bo & kIndexMask) >= d.n_params) return false;
        b = bo & kIndexMask;
      }
      return m > 0;
    };
    auto same_x = [&](std::uint32_t o1, std::uint32_t o2, std::uint32_t m) {
      for (std::uint32_t k = 0; k < m; ++k) if (P.opnd[o1 + k] != P.opnd[o2 + k]) return false;
      return true;
    };
    std::uint32_t i = 0;
    while (i < d.n_nodes) {
      std::uint32_t xo, m, w0, b0;
      if (!ip_shape(i, xo, m, w0, b0)) { ++i; continue; }
      std::uint32_t n_out = 1;
      for (;;) {
        std::uint32_t xo1, m1, w1, b1;
        const std::uint32_t nx = i + n_out;
        if (!ip_shape(nx, xo1, m1, w1, b1) || m1 != m || d.op[nx] != d.op[i] || !same_x(xo, xo1, m) ||
            w1 != w0 + n_out * m || (b0 == kNone) != (b1 == kNone) || (b0 != kNone && b1 != b0 + n_out) ||
            c.row[nx] != c.row[i] + n_out)
          break;
        ++n_out;
      }
      const std::uint32_t first = i;
      i += n_out;
      if (std::uint64_t(n_out) * m < 8) continue;
      // fused activation: the next n_out nodes apply one domain-free unary op to z_j,
      // the only consumer of z_j
      std::uint32_t act = 0, act_row = kNone;
      {
        const std::uint8_t op0 = i < d.n_nodes ? d.op[i] : 0;
        bool ok = op0 == 1 /*Relu*/ || op0 == 2 /*Tanh*/ || op0 == 3 /*Exp*/ || op0 == 5 /*Sigmoid*/ ||
                  op0 == 7 /*Sqr*/ || op0 == 8 /*Cub*/;
        for (std::uint32_t j = 0; ok && j < n_out; ++j) {
          const std::uint32_t an = i + j;
          ok = an < d.n_nodes && c.cls[an] == cSample && reach[an] && d.op[an] == op0 &&
               P.opnd[nodefwd[instr_of[an]].opnd] == enc(kSlot, c.row[first + j]) &&
               uses[c.row[first + j]] == 1 && c.row[an] == c.row[i] + j;
        }
        if (ok) { act = op0; act_row = c.row[i]; }
      }
      const std::uint32_t id = static_cast<std::uint32_t>(P.dense.size());
      P.dense.push_back(Dense{c.row[first], n_out, m, xo, w0, b0, first, act, act_row, 0});
      for (std::uint32_t j = 0; j < n_out; ++j) dense_of[first + j] = static_cast<std::int32_t>(id);
      if (act) {
        for (std::uint32_t j = 0; j < n_out; ++j) dense_of[i + j] = static_cast<std::int32_t>(id);
        i += n_out;
      }
      P.n_dense_nodes += n_out * (act ? 2 : 1);
    }
    // forward stream: the group at its first member, members / activations dropped
    P.fwd.clear();
    for (const Instr& in : nodefwd) {
      if (in.kind == kNode && dense_of[in.node] >= 0) {
        const std::uint32_t id = static_cast<std::uint32_t>(dense_of[in.node]);
        const Dense& D = P.dense[id];
        if (in.node == D.first_node)
          P.fwd.push_back(Instr{kDense, static_cast<std::uint8_t>(D.act_op), 0, D.out_row, D.n_in, D.x_opnd, id, D.first_node, 0.0});
        continue;
      }
      P.fwd.push_back(in);
    }
  }

  // ---- reverse sweep -----------------------------------------------------------
  std::vector<std::uint32_t> dense_seen(P.dense.size(), 0);
  std::vector<std::uint8_t> written(nrow + 1, 0);
  std::vector<std::uint8_t> needs_zero(nrow + 1, 0);
  const std::uint8_t rc = c.cls[d.root];
  if (rc == cSample || rc == cInput) { P.root_row = c.row[d.root]; written[P.root_row] = 1; }
  else P.root_uv = c.uv[d.root];

  struct PendingTerm { std::uint32_t dest; Term t; };
  std::vector<PendingTerm> pend;
  auto new_aux_row = [&]() { const std::uint32_t r = nrow++; written.push_back(0); needs_zero.push_back(0); return r; };

  // fused heads: the reverse instruction runs where the head's last node in
  // processing order stood (every output adjoint is final there; the q / k / v
  // producers, children of head nodes, all come later); it is the only pusher
  // into its q / k / v rows and stores them
  std::vector<std::uint32_t> attn_left(agroups.size(), 0), ln_left(lns.size(), 0);
  for (std::uint32_t node : P.order) {
    if (attn_of[node] >= 0) ++attn_left[attn_of[node]];
    if (ln_of[node] >= 0) ++ln_left[ln_of[node]];
  }
  for (std::uint32_t node : P.order) {
    if (c.cls[node] == cUniform) { P.ubwd.push_back(P.ufwd[uinstr_of[node]]); continue; }
    if (c.cls[node] != cSample) continue;
    if (ln_of[node] >= 0) {
      if (--ln_left[ln_of[node]] > 0) continue;
      const std::uint32_t id = ln_id[ln_of[node]];
      const LNorm& L = P.lnorm[id];
      P.bwd.push_back(Instr{kLNorm, 0, 0, P.lnrows[L.off + 2 * L.n], 0, 0, id, L.first_node, L.eps});
      for (std::uint32_t i = 0; i < L.n; ++i) {
        const std::uint32_t xr = P.lnrows[L.off + i];
        if (!written[xr]) { P.lnflag[L.flag_off + i] |= kAssign; written[xr] = 1; }
        // gamma_i: sum_s dy_i n_i (the adjoint of n_i * gamma_i equals dy_i); beta_i: sum_s dy_i
        const std::uint32_t yr = P.lnrows[L.off + 2 * L.n + i], nr = P.lnrows[L.off + L.n + i];
        const std::uint32_t gu = P.lnrows[L.off + 3 * L.n + i], bu = P.lnrows[L.off + 4 * L.n + i];
        pend.push_back({gu, Term{yr, nr, -1, 0, 1.0}});
        pend.push_back({bu, Term{yr, kNone, -1, 0, 1.0}});
      }
      continue;
    }
    if (attn_of[node] >= 0) {
      if (--attn_left[attn_of[node]] > 0) continue;
      const std::uint32_t id = attn_id[attn_of[node]];
      const Attn& A = P.attn[id];
      P.bwd.push_back(Instr{kAttn, 0, 0, P.arows[A.unit_off + 1], 0, 0, id, A.first_node, 0.0});
      for (std::uint32_t u = 0; u < A.n_units; ++u)
        for (std::uint32_t i = 0; i < A.hd; ++i) written[P.arows[A.unit_off + 3 * u] + i] = 1;
      for (std::uint32_t j = 0; j < A.n_keys; ++j) {
        for (std::uint32_t i = 0; i < A.hd; ++i) written[P.arows[A.key_off + 2 * j] + i] = 1;
        for (std::uint32_t i = 0; i < A.dv; ++i) written[P.arows[A.key_off + 2 * j + 1] + i] = 1;
      }
      continue;
    }
    if (dense_of[node] >= 0) {
      // the fused group runs where its last member would: every member's
      // adjoint is final there (parents precede children in this order)
      const std::uint32_t id = static_cast<std::uint32_t>(dense_of[node]);
      const Dense& D = P.dense[id];
      if (++dense_seen[id] < D.n_out * (D.act_op ? 2u : 1u)) continue;
      P.bwd.push_back(Instr{kDense, static_cast<std::uint8_t>(D.act_op), 0, D.out_row, D.n_in, D.x_opnd, id,
                            D.first_node, 0.0});
      for (std::uint32_t j = 0; j < D.n_out; ++j) written[D.out_row + j] = 1;
      for (std::uint32_t k = 0; k < D.n_in; ++k) {
        const std::uint32_t xr = P.opnd[D.x_opnd + k] & kIndexMask;
        if (!written[xr]) { P.oflag[D.x_opnd + k] |= kAssign; written[xr] = 1; }
      }
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        for (std::uint32_t k = 0; k < D.n_in; ++k)
          pend.push_back({D.w_uv + j * D.n_in + k, Term{D.out_row + j, P.opnd[D.x_opnd + k] & kIndexMask, -1, 0, 1.0}});
        if (D.b_uv != kNone) pend.push_back({D.b_uv + j, Term{D.out_row + j, kNone, -1, 0, 1.0}});
      }
      continue;
    }
    const Instr in = nodefwd[instr_of[node]];
    if (in.op == StopGradMax) continue;  // no gradient flows through the shift
    P.bwd.push_back(in);
    const std::uint32_t n = in.nops;
    for (std::uint32_t j = 0; j < n; ++j) {
      const std::uint32_t o = P.opnd[in.opnd + j];
      const std::uint32_t mode = o >> kModeShift, idx = o & kIndexMask;
      if (mode == kSlot) {
        if (!written[idx]) { P.oflag[in.opnd + j] |= kAssign; written[idx] = 1; }
      } else if (mode == kSGather) {
        const GatherTable& T = P.sgather[idx];
        for (std::uint32_t r = 0; r < T.n_rows; ++r) {
          const std::uint32_t rr = P.cand[T.cand_off + r];
          if (!written[rr]) { needs_zero[rr] = 1; written[rr] = 1; }
        }
      } else {  // sample-invariant operand: batch-reduction term
        if (idx >= P.uv_const_base) continue;  // constants take no gradient
        const std::uint8_t op = in.op;
        double coef = 0.0;
        std::uint32_t f = kNone;
        bool direct = true;
        auto partner_row = [&](std::uint32_t k) -> bool {
          const std::uint32_t po = P.opnd[in.opnd + k];
          if ((po >> kModeShift) != kSlot) return false;
          f = po & kIndexMask;
          return true;
        };
        switch (op) {
          case Add: case AddVarying: coef = 1.0; break;
          case Sub: case SubVarying: coef = j == 0 ? 1.0 : -1.0; break;
          case Mean: coef = 0.5; break;
          case NegativeMean: coef = -0.5; break;
          case MeanVarying: coef = 1.0 / n; break;
          case NegativeMeanVarying: coef = -1.0 / n; break;
          case Mul: coef = 1.0; direct = partner_row(1 - j); break;
          case IPNoBias: { const std::uint32_t m = n / 2; coef = 1.0; direct = partner_row(j < m ? j + m : j - m); break; }
          case IPWithBias: {
            const std::uint32_t m = (n - 1) / 2;
            coef = 1.0;
            if (j == n - 1) break;
            direct = partner_row(j < m ? j + m : j - m);
            break;
          }
          default: direct = false; break;
        }
        Term t{};
        if (direct) {
          t = Term{in.out, f, -1, 0, coef};
        } else {
          const std::uint32_t ar = new_aux_row();
          P.oflag[in.opnd + j] |= kToAux;
          P.oaux[in.opnd + j] = ar;
          written[ar] = 1;
          t = Term{ar, kNone, -1, 0, 1.0};
        }
        pend.push_back({idx, t});
      }
    }
  }
  // scatter terms of materialised sample-invariant gathers (embedding rows)
  for (std::uint32_t g = 0; g < d.n_gathers; ++g) {
    if (c.gkind[g] != 1 || !written[c.grow[g]]) continue;
    for (std::uint32_t r = 0; r < d.gathers[g].n_rows; ++r) {
      const std::uint32_t u = c.uv[c.cand(g, r)];
      if (u >= P.uv_const_base) continue;
      pend.push_back({u, Term{c.grow[g], d.gathers[g].index_col, static_cast<std::int32_t>(r), 1, 1.0}});
    }
  }
  // With fused heads the reference processing order is not always a valid
  // order of the reverse instructions: a head's reverse runs once every output
  // adjoint is final, but the processing order may reach a q / k / v producer
  // (e.g. position 0's projection) before the last head node.  Re-sort the
  // reverse list topologically over "pushes into a row -> reads that row's
  // adjoint", keeping the original order wherever it is valid (Kahn's
  // algorithm, smallest original index first), then recompute the first-write
  // (assign) flags and the rows that must start at zero for the new order.
  if (!P.attn.empty() || !P.lnorm.empty()) {
    const std::size_t NB = P.bwd.size();
    std::vector<std::uint32_t> reader(nrow, kNone);   // reverse instruction reading each row's adjoint
    std::vector<std::vector<std::uint32_t>> pushes(NB);
    std::vector<std::uint32_t> rows;
    for (std::uint32_t k = 0; k < NB; ++k) {
      const Instr& in = P.bwd[k];
      rows.clear();
      if (in.kind == kLNorm) {
        const LNorm& L = P.lnorm[in.aux];
        for (std::uint32_t i = 0; i < L.n; ++i) {
          reader[P.lnrows[L.off + 2 * L.n + i]] = k;
          rows.push_back(P.lnrows[L.off + i]);
        }
      } else if (in.kind == kAttn) {
        const Attn& A = P.attn[in.aux];
        for (std::uint32_t u = 0; u < A.n_units; ++u) {
          for (std::uint32_t i = 0; i < A.dv; ++i) reader[P.arows[A.unit_off + 3 * u + 1] + i] = k;
          for (std::uint32_t i = 0; i < A.hd; ++i) rows.push_back(P.arows[A.unit_off + 3 * u] + i);
        }
        for (std::uint32_t j = 0; j < A.n_keys; ++j) {
          for (std::uint32_t i = 0; i < A.hd; ++i) rows.push_back(P.arows[A.key_off + 2 * j] + i);
          for (std::uint32_t i = 0; i < A.dv; ++i) rows.push_back(P.arows[A.key_off + 2 * j + 1] + i);
        }
      } else if (in.kind == kDense) {
        const Dense& D = P.dense[in.aux];
        for (std::uint32_t j = 0; j < D.n_out; ++j) {
          reader[D.out_row + j] = k;
          if (D.act_op) reader[D.act_row + j] = k;
        }
        for (std::uint32_t q = 0; q < D.n_in; ++q) rows.push_back(P.opnd[D.x_opnd + q] & kIndexMask);
      } else {
        reader[in.out] = k;
        for (std::uint32_t j = 0; j < in.nops; ++j) {
          const std::uint32_t o = P.opnd[in.opnd + j], mode = o >> kModeShift, idx = o & kIndexMask;
          if (mode == kSlot) rows.push_back(idx);
          else if (mode == kSGather) {
            const GatherTable& T = P.sgather[idx];
            for (std::uint32_t r = 0; r < T.n_rows; ++r) rows.push_back(P.cand[T.cand_off + r]);
          }
        }
      }
      pushes[k] = rows;
    }
    std::vector<std::uint32_t> indeg(NB, 0);
    std::vector<std::vector<std::uint32_t>> succ(NB);
    for (std::uint32_t k = 0; k < NB; ++k) {
      std::sort(pushes[k].begin(), pushes[k].end());
      pushes[k].erase(std::unique(pushes[k].begin(), pushes[k].end()), pushes[k].end());
      for (std::uint32_t r : pushes[k])
        if (reader[r] != kNone && reader[r] != k) { succ[k].push_back(reader[r]); ++indeg[reader[r]]; }
    }
    std::priority_queue<std::uint32_t, std::vector<std::uint32_t>, std::greater<std::uint32_t>> ready;
    for (std::uint32_t k = 0; k < NB; ++k) if (!indeg[k]) ready.push(k);
    std::vector<Instr> nb;
    nb.reserve(NB);
    while (!ready.empty()) {
      const std::uint32_t k = ready.top();
      ready.pop();
      nb.push_back(P.bwd[k]);
      for (std::uint32_t t : succ[k]) if (--indeg[t] == 0) ready.push(t);
    }
    if (nb.size() != NB) throw std::runtime_error("tg_compile: cyclic reverse order around a fused attention head");
    P.bwd.swap(nb);
    // first-write flags and zero-start rows for the new order
    std::fill(written.begin(), written.end(), 0);
    std::fill(needs_zero.begin(), needs_zero.end(), 0);
    if (P.root_row != kNone) written[P.root_row] = 1;
    for (std::size_t q = 0; q < P.oflag.size(); ++q)
      if (P.oflag[q] & kToAux) written[P.oaux[q]] = 1;
    for (const Instr& in : P.bwd) {
      auto flag = [&](std::uint32_t pos) {
        const std::uint32_t r = P.opnd[pos] & kIndexMask;
        if (!written[r]) { P.oflag[pos] |= kAssign; written[r] = 1; }
        else P.oflag[pos] &= static_cast<std::uint8_t>(~kAssign);
      };
      if (in.kind == kLNorm) {
        const LNorm& L = P.lnorm[in.aux];
        for (std::uint32_t i = 0; i < L.n; ++i) {
          const std::uint32_t r = P.lnrows[L.off + i];
          if (!written[r]) { P.lnflag[L.flag_off + i] |= kAssign; written[r] = 1; }
          else P.lnflag[L.flag_off + i] &= static_cast<std::uint8_t>(~kAssign);
        }
      } else if (in.kind == kAttn) {
        std::vector<std::uint32_t> rr;
        const Attn& A = P.attn[in.aux];
        for (std::uint32_t u = 0; u < A.n_units; ++u)
          for (std::uint32_t i = 0; i < A.hd; ++i) written[P.arows[A.unit_off + 3 * u] + i] = 1;
        for (std::uint32_t j = 0; j < A.n_keys; ++j) {
          for (std::uint32_t i = 0; i < A.hd; ++i) written[P.arows[A.key_off + 2 * j] + i] = 1;
          for (std::uint32_t i = 0; i < A.dv; ++i) written[P.arows[A.key_off + 2 * j + 1] + i] = 1;
        }
      } else if (in.kind == kDense) {
        const Dense& D = P.dense[in.aux];
        for (std::uint32_t j = 0; j < D.n_out; ++j) written[D.out_row + j] = 1;
        for (std::uint32_t q = 0; q < D.n_in; ++q) flag(D.x_opnd + q);
      } else {
        for (std::uint32_t j = 0; j < in.nops; ++j) {
          const std::uint32_t o = P.opnd[in.opnd + j], mode = o >> kModeShift, idx = o & kIndexMask;
          if (mode == kSlot) flag(in.opnd + j);
          else if (mode == kSGather) {
            const GatherTable& T = P.sgather[idx];
            for (std::uint32_t r = 0; r < T.n_rows; ++r) {
              const std::uint32_t rr = P.cand[T.cand_off + r];
              if (!written[rr]) { needs_zero[rr] = 1; written[rr] = 1; }
            }
          }
        }
      }
    }
  }
  // input rows never reached still report a zero input gradient
  for (std::uint32_t col = 0; col < d.n_inputs; ++col) {
    const std::uint32_t r = P.input_rows[col];
    if (r != kNone && !written[r]) { needs_zero[r] = 1; written[r] = 1; }
  }
  for (std::uint32_t r = 0; r < nrow; ++r) if (needs_zero[r]) P.zero_rows.push_back(r);
  P.n_rows = nrow;

  // group terms by destination (stable: keeps reverse-sweep order per dest)
  std::stable_sort(pend.begin(), pend.end(), [](const PendingTerm& a, const PendingTerm& b) { return a.dest < b.dest; });
  P.term_off.push_back(0);
  for (std::size_t k = 0; k < pend.size(); ++k) {
    if (k == 0 || pend[k].dest != pend[k - 1].dest) {
      if (k) P.term_off.push_back(static_cast<std::uint32_t>(P.terms.size()));
      P.dest_uv.push_back(pend[k].dest);
    }
    P.terms.push_back(pend[k].t);
  }
  if (!pend.empty()) P.term_off.push_back(static_cast<std::uint32_t>(P.terms.size()));

  // ---- weight gradients of dense layers: outer-product contractions -----------
  P.dest_dense.assign(P.dest_uv.size(), 0);
  {
    std::unordered_map<std::uint32_t, std::uint32_t> dest_of_uv;
    for (std::uint32_t dd = 0; dd < P.dest_uv.size(); ++dd) dest_of_uv[P.dest_uv[dd]] = dd;
    for (const Dense& D : P.dense) {
      auto it = dest_of_uv.find(D.w_uv);
      if (it == dest_of_uv.end()) continue;
      const std::uint32_t d0 = it->second;
      bool ok = d0 + D.n_out * D.n_in <= P.dest_uv.size();
      for (std::uint32_t q = 0; ok && q < D.n_out * D.n_in; ++q)  // each W dest fed by this layer only
        ok = P.dest_uv[d0 + q] == D.w_uv + q && P.term_off[d0 + q + 1] - P.term_off[d0 + q] == 1;
      if (!ok) continue;
      DenseGrad g{D.n_out, D.n_in, static_cast<std::uint32_t>(P.dg_rows.size()), d0};
      for (std::uint32_t j = 0; j < D.n_out; ++j) P.dg_rows.push_back(D.out_row + j);
      for (std::uint32_t k = 0; k < D.n_in; ++k) P.dg_rows.push_back(P.opnd[D.x_opnd + k] & kIndexMask);
      for (std::uint32_t q = 0; q < D.n_out * D.n_in; ++q) P.dest_dense[d0 + q] = 1;
      P.dgrad.push_back(g);
    }
  }
  // uniform reverse sweep: children pairwise distinct -> pushes may run in parallel
  for (Instr& in : P.ubwd) {
    std::vector<std::uint32_t> ch(P.opnd.begin() + in.opnd, P.opnd.begin() + in.opnd + in.nops);
    std::sort(ch.begin(), ch.end());
    in.pad = std::adjacent_find(ch.begin(), ch.end()) == ch.end() ? 1 : 0;
  }
  return P;
}

}  // namespace tgc
