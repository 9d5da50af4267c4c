// tg_recorder.hpp — recording surface of the B200 gradient oracle.
//
// A from-scratch recorder that keeps the reference's C++ graph-building API
// (tapegrad, /root/reference/proj/include/tapegrad) so that model code written
// against Tape / ValueRef / ops.hpp free functions records the same tape here:
//   * Tape<Scalar>: node arena, eager values, checkpoint/rewind
//     (reference tape.hpp:68-353);
//   * unary / binary / mul_by_constant / varying / inner_product[_with_bias] /
//     *_inplace / variance helpers with the reference's eager formulas and
//     domain checks (ops.hpp:38-307);
//   * OpKind numbering and mnemonics (op_kind.hpp:10-123).
// What it adds is what the GPU compiler needs and the reference leaves
// implicit in user code: leaf roles (param / per-sample input / constant),
// data-dependent gathers (embedding rows and softmax targets selected by
// token ids) and the stop-gradient max used for the softmax shift.
//
// The recorder never runs a backward pass on the CPU: the batch backward is
// the device program built by tg_compile.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tg_abi.h"

namespace tg {

using NodeIndex = std::uint32_t;
constexpr std::uint32_t kGatherFlag = TG_GATHER_FLAG;

/// Handle into one tape (reference tape.hpp:23-27).  Plain data.  When the
/// kGatherFlag bit is set the handle names a gather reference instead of a
/// node: its value depends on the sample's token ids.
struct ValueRef {
  NodeIndex index{0};
  friend constexpr bool operator==(ValueRef, ValueRef) = default;
};

/// Same numbering as reference op_kind.hpp:10-44, plus one extension.
enum class OpKind : std::uint8_t {
  Leaf, Relu, Tanh, Exp, NegLog, Sigmoid, Inv, Sqr, Cub, Log, Sqrt, InvSqrt,
  Add, Sub, Mul, MulByConst, Div, Mean, AddSquares, MeanSquares, NegativeMean,
  AddVarying, SubVarying, MulVarying, MeanVarying, SumOfSquaresVarying,
  MeanSquaresVarying, NegativeMeanVarying, InnerProductNoBias, InnerProductWithBias,
  StopGradMax = TG_OP_STOPGRAD_MAX,
};

enum class OpArity : std::uint8_t { Leaf, Unary, Binary, Varying };

constexpr OpArity arity_of(OpKind k) noexcept {
  const auto v = static_cast<unsigned>(k);
  if (k == OpKind::Leaf) return OpArity::Leaf;
  if (v >= 1 && v <= 11) return OpArity::Unary;
  if (k == OpKind::MulByConst) return OpArity::Unary;
  if (v >= 12 && v <= 20) return OpArity::Binary;
  return OpArity::Varying;  // 21..29 and StopGradMax
}

inline const char* op_name(OpKind k) noexcept { return tg_op_name(static_cast<std::uint8_t>(k)); }

struct TapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : TapeError { using TapeError::TapeError; };
struct InvalidHandle : TapeError { using TapeError::TapeError; };
struct InvalidCheckpoint : TapeError { using TapeError::TapeError; };

struct Checkpoint {
  NodeIndex mark{0};
  std::size_t child_mark{0};
  std::uint32_t params{0};
  std::uint32_t gathers{0};
};

struct TapeConfig {
  std::size_t capacity{0};
  bool fixed_capacity{false};
  bool names_enabled{false};     // accepted for API parity; names are not stored
  std::size_t child_capacity{0};
};

namespace detail {
template <class Scalar>
[[noreturn]] inline void throw_domain(OpKind kind, Scalar offending) {
  // Message text of reference ops.hpp:17-19.
  throw std::domain_error(std::string(op_name(kind)) + ": input " +
                          std::to_string(static_cast<double>(offending)) +
                          " is outside the operator domain");
}
template <class Scalar> Scalar require_positive(OpKind k, Scalar x) {
  if (!(x > Scalar(0))) throw_domain(k, x);
  return x;
}
template <class Scalar> Scalar require_nonzero(OpKind k, Scalar x) {
  if (x == Scalar(0)) throw_domain(k, x);
  return x;
}
}  // namespace detail

template <class Scalar>
class Tape {
 public:
  using scalar_type = Scalar;

  explicit Tape(const TapeConfig& cfg) : fixed_(cfg.fixed_capacity), capacity_(cfg.capacity) {
    if (cfg.capacity == 0) throw std::invalid_argument("Tape: capacity must be >= 1");
    child_capacity_ = cfg.child_capacity ? cfg.child_capacity : cfg.capacity * 8;
    values_.reserve(capacity_);
    ops_.reserve(capacity_);
    consts_.reserve(capacity_);
    child_off_.reserve(capacity_ + 1);
    leaf_class_.reserve(capacity_);
    leaf_index_.reserve(capacity_);
    child_pool_.reserve(child_capacity_);
    child_off_.push_back(0);
  }
  explicit Tape(std::size_t capacity) : Tape(TapeConfig{.capacity = capacity}) {}
  Tape(const Tape&) = delete;
  Tape& operator=(const Tape&) = delete;

  NodeIndex size() const noexcept { return static_cast<NodeIndex>(ops_.size()); }
  bool empty() const noexcept { return ops_.empty(); }
  std::size_t capacity() const noexcept { return capacity_; }
  NodeIndex peak_nodes() const noexcept { return peak_nodes_; }
  std::size_t child_pool_size() const noexcept { return child_pool_.size(); }
  std::uint32_t max_arity() const noexcept { return max_arity_; }
  /// High-water mark of the child-pool cursor (reference Tape::peak_children).
  std::size_t peak_children() const noexcept { return peak_children_; }
  /// Bytes of recorder storage touched at the high-water marks, accounted from
  /// this recorder's own per-node buffers (value, op, constant, child offset,
  /// leaf class and index) and the child pool, as the reference's
  /// peak_arena_bytes (tape.hpp:118-125) accounts from its arenas.
  std::size_t peak_arena_bytes() const noexcept {
    constexpr std::size_t per_node = 2 * sizeof(Scalar) + 1 + sizeof(std::uint64_t) + 1 + sizeof(std::uint32_t);
    return static_cast<std::size_t>(peak_nodes_) * per_node + peak_children_ * sizeof(std::uint32_t);
  }
  bool fixed_capacity() const noexcept { return fixed_; }

  // ---- leaves -----------------------------------------------------------
  /// Reference Tape::leaf (tape.hpp:169).  A bare leaf is a constant: its
  /// value is the same for every sample and it is not trained.
  ValueRef leaf(Scalar v) { return push_leaf(TG_LEAF_CONST, 0, v); }
  ValueRef constant(Scalar v) { return push_leaf(TG_LEAF_CONST, 0, v); }
  /// Trainable parameter leaf (one entry of a ParamRange).
  ValueRef param(Scalar v) { return push_leaf(TG_LEAF_PARAM, n_params_++, v); }
  /// Per-sample input leaf; `v` is this template sample's value.
  ValueRef input(std::uint32_t col, Scalar v) {
    n_inputs_ = std::max(n_inputs_, col + 1);
    return push_leaf(TG_LEAF_INPUT, col, v);
  }
  /// Data-dependent reference: first + stride * idx[col] + offset.
  ValueRef gather(ValueRef first, std::uint32_t stride, std::uint32_t n_rows, std::uint32_t col,
                  std::uint32_t offset, std::int32_t template_index) {
    check_live(first);
    if (n_rows == 0 || template_index < 0 || static_cast<std::uint32_t>(template_index) >= n_rows)
      throw std::invalid_argument("gather: template index " + std::to_string(template_index) +
                                  " outside [0, " + std::to_string(n_rows) + ")");
    const std::uint64_t last = std::uint64_t(first.index) + std::uint64_t(stride) * (n_rows - 1) + offset;
    if (last >= size()) throw InvalidHandle("gather: table extends past live node count");
    gathers_.push_back(tg_gather{first.index, stride, n_rows, col, offset});
    gather_tidx_.push_back(template_index);
    n_index_inputs_ = std::max(n_index_inputs_, col + 1);
    return ValueRef{kGatherFlag | static_cast<std::uint32_t>(gathers_.size() - 1)};
  }

  // ---- reads ------------------------------------------------------------
  NodeIndex resolve(ValueRef v) const {
    if (v.index & kGatherFlag) {
      const std::uint32_t g = v.index & ~kGatherFlag;
      if (g >= gathers_.size()) throw InvalidHandle("stale gather handle " + std::to_string(g));
      const tg_gather& G = gathers_[g];
      return G.first_node + G.stride * static_cast<std::uint32_t>(gather_tidx_[g]) + G.offset;
    }
    check_live(v);
    return v.index;
  }
  Scalar value_of(ValueRef v) const { return values_[resolve(v)]; }
  OpKind op_of(ValueRef v) const { return static_cast<OpKind>(ops_[resolve(v)]); }
  Scalar constant_of(ValueRef v) const { return consts_[resolve(v)]; }
  std::span<const NodeIndex> children_of(ValueRef v) const { return children_at(resolve(v)); }
  Scalar value_at(NodeIndex i) const noexcept { return values_[i]; }
  OpKind op_at(NodeIndex i) const noexcept { return static_cast<OpKind>(ops_[i]); }
  Scalar constant_at(NodeIndex i) const noexcept { return consts_[i]; }
  std::span<const NodeIndex> children_at(NodeIndex i) const noexcept {
    return {child_pool_.data() + child_off_[i], child_off_[i + 1] - child_off_[i]};
  }
  void set_value(ValueRef v, Scalar value) { values_[resolve(v)] = value; }

  // ---- checkpoint / rewind (tape.hpp:228-242) -------------------------------
  Checkpoint checkpoint() const noexcept {
    return Checkpoint{size(), child_pool_.size(), n_params_, static_cast<std::uint32_t>(gathers_.size())};
  }
  void rewind(Checkpoint cp) {
    if (cp.mark > size())
      throw InvalidCheckpoint("rewind: checkpoint mark " + std::to_string(cp.mark) +
                              " is ahead of tape size " + std::to_string(size()));
    if (cp.child_mark > child_pool_.size() || cp.params > n_params_ || cp.gathers > gathers_.size())
      throw InvalidCheckpoint("rewind: checkpoint child mark " + std::to_string(cp.child_mark) +
                              " is ahead of child pool cursor " + std::to_string(child_pool_.size()));
    values_.resize(cp.mark);
    ops_.resize(cp.mark);
    consts_.resize(cp.mark);
    leaf_class_.resize(cp.mark);
    leaf_index_.resize(cp.mark);
    child_off_.resize(cp.mark + 1);
    child_pool_.resize(cp.child_mark);
    n_params_ = cp.params;
    gathers_.resize(cp.gathers);
    gather_tidx_.resize(cp.gathers);
    if (root_ >= cp.mark) root_ = 0;
  }

  // ---- node construction (tape.hpp:132-167) ---------------------------------
  ValueRef emplace(OpKind op, Scalar value, std::span<const ValueRef> kids, Scalar c = Scalar(0)) {
    const std::size_t off = child_pool_.size();
    if (fixed_ && off + kids.size() > child_capacity_)
      throw CapacityError("tape child pool capacity exceeded: " + std::to_string(child_capacity_) +
                          " entries");
    if (fixed_ && size() >= capacity_)
      throw CapacityError("tape capacity exceeded: " + std::to_string(capacity_) + " nodes");
    for (ValueRef k : kids) child_pool_.push_back(k.index);
    values_.push_back(value);
    ops_.push_back(static_cast<std::uint8_t>(op));
    consts_.push_back(c);
    leaf_class_.push_back(TG_NODE_OP);
    leaf_index_.push_back(0);
    child_off_.push_back(child_pool_.size());
    peak_nodes_ = std::max(peak_nodes_, size());
    peak_children_ = std::max(peak_children_, child_pool_.size());
    max_arity_ = std::max<std::uint32_t>(max_arity_, static_cast<std::uint32_t>(kids.size()));
    return ValueRef{size() - 1};
  }

  void set_root(ValueRef r) { root_ = resolve(r); }
  NodeIndex root() const noexcept { return root_; }

  /// Plain-array view for tg_compile (valid until the next mutation).
  tg_tape_desc describe() const {
    tg_tape_desc d{};
    d.n_nodes = size();
    d.dtype = sizeof(Scalar) == 8 ? TG_F64 : TG_F32;
    d.op = ops_.data();
    d.child_offset = child_off_.data();
    d.child = child_pool_.data();
    consts64_.assign(consts_.begin(), consts_.end());
    values64_.assign(values_.begin(), values_.end());
    d.constant = consts64_.data();
    d.leaf_class = leaf_class_.data();
    d.leaf_index = leaf_index_.data();
    d.leaf_value = values64_.data();
    d.n_gathers = static_cast<std::uint32_t>(gathers_.size());
    d.gathers = gathers_.data();
    d.root = root_;
    d.n_params = n_params_;
    d.n_inputs = n_inputs_;
    d.n_index_inputs = n_index_inputs_;
    return d;
  }

  std::span<const std::uint8_t> leaf_classes() const noexcept { return leaf_class_; }
  std::span<const std::uint32_t> leaf_indices() const noexcept { return leaf_index_; }
  const std::vector<tg_gather>& gathers() const noexcept { return gathers_; }
  const std::vector<std::int32_t>& gather_template_indices() const noexcept { return gather_tidx_; }
  std::uint32_t n_params() const noexcept { return n_params_; }
  std::uint32_t n_inputs() const noexcept { return n_inputs_; }
  std::uint32_t n_index_inputs() const noexcept { return n_index_inputs_; }

 private:
  ValueRef push_leaf(std::uint8_t cls, std::uint32_t idx, Scalar v) {
    ValueRef r = emplace(OpKind::Leaf, v, {}, Scalar(0));
    leaf_class_.back() = cls;
    leaf_index_.back() = idx;
    return r;
  }
  void check_live(ValueRef v) const {
    if (v.index >= size())
      throw InvalidHandle("stale handle: node index " + std::to_string(v.index) +
                          " >= live count " + std::to_string(size()));
  }

  bool fixed_;
  std::size_t capacity_;
  std::size_t child_capacity_{0};
  std::vector<Scalar> values_;
  std::vector<std::uint8_t> ops_;
  std::vector<Scalar> consts_;
  std::vector<std::uint64_t> child_off_;
  std::vector<std::uint32_t> child_pool_;
  std::vector<std::uint8_t> leaf_class_;
  std::vector<std::uint32_t> leaf_index_;
  std::vector<tg_gather> gathers_;
  std::vector<std::int32_t> gather_tidx_;
  mutable std::vector<double> consts64_, values64_;
  std::uint32_t n_params_{0}, n_inputs_{0}, n_index_inputs_{0};
  NodeIndex root_{0};
  NodeIndex peak_nodes_{0};
  std::size_t peak_children_{0};
  std::uint32_t max_arity_{0};
};

// ---------------------------------------------------------------------------
// Operators: eager forward values with the reference's formulas (ops.hpp).
// ---------------------------------------------------------------------------

template <class Scalar>
ValueRef unary(Tape<Scalar>& t, OpKind kind, ValueRef x) {
  if (arity_of(kind) != OpArity::Unary || kind == OpKind::MulByConst)
    throw std::invalid_argument(std::string("unary: op ") + op_name(kind) +
                                " is not a plain unary operator");
  const Scalar v = t.value_of(x);
  Scalar y = 0;
  switch (kind) {
    case OpKind::Relu: y = v > Scalar(0) ? v : Scalar(0); break;
    case OpKind::Tanh: y = std::tanh(v); break;
    case OpKind::Exp: y = std::exp(v); break;
    case OpKind::NegLog: y = -std::log(detail::require_positive(kind, v)); break;
    case OpKind::Sigmoid: y = Scalar(1) / (Scalar(1) + std::exp(-v)); break;
    case OpKind::Inv: y = Scalar(1) / detail::require_nonzero(kind, v); break;
    case OpKind::Sqr: y = v * v; break;
    case OpKind::Cub: y = v * v * v; break;
    case OpKind::Log: y = std::log(detail::require_positive(kind, v)); break;
    case OpKind::Sqrt: y = std::sqrt(detail::require_positive(kind, v)); break;
    case OpKind::InvSqrt: y = Scalar(1) / std::sqrt(detail::require_positive(kind, v)); break;
    default: break;
  }
  const ValueRef kids[1] = {x};
  return t.emplace(kind, y, kids);
}

template <class S> ValueRef relu(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Relu, x); }
template <class S> ValueRef tanh(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Tanh, x); }
template <class S> ValueRef exp(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Exp, x); }
template <class S> ValueRef negative_log(Tape<S>& t, ValueRef x) { return unary(t, OpKind::NegLog, x); }
template <class S> ValueRef sigmoid(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Sigmoid, x); }
template <class S> ValueRef inv(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Inv, x); }
template <class S> ValueRef sqr(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Sqr, x); }
template <class S> ValueRef pow3(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Cub, x); }
template <class S> ValueRef log(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Log, x); }
template <class S> ValueRef sqrt(Tape<S>& t, ValueRef x) { return unary(t, OpKind::Sqrt, x); }
template <class S> ValueRef inv_sqrt(Tape<S>& t, ValueRef x) { return unary(t, OpKind::InvSqrt, x); }

template <class Scalar>
ValueRef binary(Tape<Scalar>& t, OpKind kind, ValueRef x, ValueRef y) {
  if (arity_of(kind) != OpArity::Binary)
    throw std::invalid_argument(std::string("binary: op ") + op_name(kind) +
                                " is not a binary operator");
  const Scalar a = t.value_of(x), b = t.value_of(y);
  Scalar r = 0;
  switch (kind) {
    case OpKind::Add: r = a + b; break;
    case OpKind::Sub: r = a - b; break;
    case OpKind::Mul: r = a * b; break;
    case OpKind::Div: r = a / detail::require_nonzero(kind, b); break;
    case OpKind::Mean: r = (a + b) / Scalar(2); break;
    case OpKind::AddSquares: r = a * a + b * b; break;
    case OpKind::MeanSquares: r = (a * a + b * b) / Scalar(2); break;
    case OpKind::NegativeMean: r = -(a + b) / Scalar(2); break;
    default: break;
  }
  const ValueRef kids[2] = {x, y};
  return t.emplace(kind, r, kids);
}

template <class S> ValueRef add(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::Add, x, y); }
template <class S> ValueRef sub(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::Sub, x, y); }
template <class S> ValueRef mul(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::Mul, x, y); }
template <class S> ValueRef div(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::Div, x, y); }
template <class S> ValueRef mean(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::Mean, x, y); }
template <class S> ValueRef add_squares(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::AddSquares, x, y); }
template <class S> ValueRef mean_squares(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::MeanSquares, x, y); }
template <class S> ValueRef negative_mean(Tape<S>& t, ValueRef x, ValueRef y) { return binary(t, OpKind::NegativeMean, x, y); }

/// x * c; c lives in the node's constant slot (ops.hpp:138-142).
template <class Scalar>
ValueRef mul_by_constant(Tape<Scalar>& t, ValueRef x, Scalar c) {
  const ValueRef kids[1] = {x};
  return t.emplace(OpKind::MulByConst, t.value_of(x) * c, kids, c);
}

template <class Scalar>
ValueRef varying(Tape<Scalar>& t, OpKind kind, std::span<const ValueRef> xs) {
  if (arity_of(kind) != OpArity::Varying || kind == OpKind::StopGradMax)
    throw std::invalid_argument(std::string("varying: op ") + op_name(kind) +
                                " is not a varying-arity operator");
  if (kind == OpKind::InnerProductNoBias || kind == OpKind::InnerProductWithBias)
    throw std::invalid_argument("varying: inner products take two sequences; "
                                "use inner_product / inner_product_with_bias");
  if (xs.empty()) throw std::invalid_argument(std::string(op_name(kind)) + ": empty input sequence");
  const auto n = static_cast<Scalar>(xs.size());
  Scalar acc = 0;
  switch (kind) {
    case OpKind::AddVarying:
    case OpKind::MeanVarying:
    case OpKind::NegativeMeanVarying:
      for (ValueRef x : xs) acc += t.value_of(x);
      if (kind == OpKind::MeanVarying) acc /= n;
      if (kind == OpKind::NegativeMeanVarying) acc = -acc / n;
      break;
    case OpKind::SubVarying:
      acc = t.value_of(xs[0]);
      for (std::size_t i = 1; i < xs.size(); ++i) acc -= t.value_of(xs[i]);
      break;
    case OpKind::MulVarying:
      acc = Scalar(1);
      for (ValueRef x : xs) acc *= t.value_of(x);
      break;
    case OpKind::SumOfSquaresVarying:
    case OpKind::MeanSquaresVarying:
      for (ValueRef x : xs) { const Scalar v = t.value_of(x); acc += v * v; }
      if (kind == OpKind::MeanSquaresVarying) acc /= n;
      break;
    default: break;
  }
  return t.emplace(kind, acc, xs);
}

template <class S> ValueRef reduce_sum(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::AddVarying, xs); }
template <class S> ValueRef reduce_sub(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::SubVarying, xs); }
template <class S> ValueRef reduce_mul(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::MulVarying, xs); }
template <class S> ValueRef reduce_mean(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::MeanVarying, xs); }
template <class S> ValueRef reduce_sum_of_squares(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::SumOfSquaresVarying, xs); }
template <class S> ValueRef reduce_mean_squares(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::MeanSquaresVarying, xs); }
template <class S> ValueRef reduce_negative_mean(Tape<S>& t, std::span<const ValueRef> xs) { return varying(t, OpKind::NegativeMeanVarying, xs); }

namespace detail {
template <class Scalar>
ValueRef ip_common(Tape<Scalar>& t, std::span<const ValueRef> xs, std::span<const ValueRef> ys,
                   const ValueRef* bias, const char* name) {
  if (xs.empty()) throw std::invalid_argument(std::string(name) + ": empty input sequence");
  if (xs.size() != ys.size())
    throw std::invalid_argument(std::string(name) + ": sequence lengths differ (" +
                                std::to_string(xs.size()) + " vs " + std::to_string(ys.size()) + ")");
  // bias first, then x_i * y_i left to right (ops.hpp:230-233, :253-256)
  Scalar acc = bias ? t.value_of(*bias) : Scalar(0);
  for (std::size_t i = 0; i < xs.size(); ++i) acc += t.value_of(xs[i]) * t.value_of(ys[i]);
  std::vector<ValueRef> kids;
  kids.reserve(2 * xs.size() + (bias ? 1 : 0));
  kids.insert(kids.end(), xs.begin(), xs.end());
  kids.insert(kids.end(), ys.begin(), ys.end());
  if (bias) kids.push_back(*bias);
  return t.emplace(bias ? OpKind::InnerProductWithBias : OpKind::InnerProductNoBias, acc, kids);
}
}  // namespace detail

template <class Scalar>
ValueRef inner_product(Tape<Scalar>& t, std::span<const ValueRef> xs, std::span<const ValueRef> ys) {
  return detail::ip_common(t, xs, ys, nullptr, "innerProduct");
}
template <class Scalar>
ValueRef inner_product_with_bias(Tape<Scalar>& t, std::span<const ValueRef> xs,
                                 std::span<const ValueRef> ys, ValueRef bias) {
  return detail::ip_common(t, xs, ys, &bias, "innerProductWithBias");
}

template <class S> ValueRef add_inplace(Tape<S>& t, ValueRef& x, ValueRef y) { return x = add(t, x, y); }
template <class S> ValueRef sub_inplace(Tape<S>& t, ValueRef& x, ValueRef y) { return x = sub(t, x, y); }
template <class S> ValueRef mul_inplace(Tape<S>& t, ValueRef& x, ValueRef y) { return x = mul(t, x, y); }
template <class S> ValueRef div_inplace(Tape<S>& t, ValueRef& x, ValueRef y) { return x = div(t, x, y); }

template <class S>
std::pair<ValueRef, ValueRef> reduce_mean_and_mean_squares(Tape<S>& t, std::span<const ValueRef> xs) {
  ValueRef m = reduce_mean(t, xs);
  ValueRef ms = reduce_mean_squares(t, xs);
  return {m, ms};
}
template <class S>
ValueRef variance_biased(Tape<S>& t, std::span<const ValueRef> xs) {
  auto [m, ms] = reduce_mean_and_mean_squares(t, xs);
  ValueRef m2 = sqr(t, m);
  return sub(t, ms, m2);
}
template <class S>
ValueRef variance(Tape<S>& t, std::span<const ValueRef> xs) {
  if (xs.size() < 2)
    throw std::invalid_argument("variance: needs at least 2 inputs, got " + std::to_string(xs.size()));
  const auto n = static_cast<S>(xs.size());
  return mul_by_constant(t, variance_biased(t, xs), n / (n - S(1)));
}

/// Non-differentiable max over xs: the softmax shift constant.
template <class Scalar>
ValueRef stopgrad_max(Tape<Scalar>& t, std::span<const ValueRef> xs) {
  if (xs.empty()) throw std::invalid_argument("stopGradMax: empty input sequence");
  Scalar m = t.value_of(xs[0]);
  for (std::size_t i = 1; i < xs.size(); ++i) m = std::max(m, t.value_of(xs[i]));
  return t.emplace(OpKind::StopGradMax, m, xs);
}

}  // namespace tg
