// tg_from_tapegrad.hpp — describe a tape recorded with the reference API.
//
// Drop-in adapter for code that records with tapegrad::Tape (reference
// tape.hpp:68-353): reads ops() / children_at() / constant_at() / value_at()
// (tape.hpp:250-260) and the caller's leaf roles, and fills the plain arrays
// of tg_tape_desc for tg_compile.  Header-only, works with any tape type that
// exposes those members (tapegrad::Tape<float|double>, tg::Tape).
//
// A reference user re-records every sample, so data-dependent choices are
// plain wiring on the reference tape: an embedding row or a softmax target is
// selected by wiring the chosen node directly, and
// the softmax max shift is a constant leaf holding that sample's max
// (SPEC.md:297-305).  Compiled once for the whole batch, those choices must be
// per-sample instead.  A `Recording` kept beside the tape while the template
// sample is recorded says where they are:
//   * rec.select(tape, first, stride, n_rows, col, offset, idx) returns the
//     node the reference would wire (first + stride * idx + offset, the same
//     eager value) and logs a gather: in the description, every child entry
//     of a node recorded after the select that names that node becomes a
//     gather reference (TG_GATHER_FLAG | id) resolved per sample from int32
//     index input `col`;
//   * rec.stopgrad_max(tape, xs) records the reference's constant leaf and
//     logs it: the description turns that leaf into the stop-gradient max over
//     xs (TG_OP_STOPGRAD_MAX), evaluated per sample.
// Gather ids follow the select order, so a model recorded this way describes
// to exactly the arrays tg::Tape records for it (tests/test_oracle.py).  A
// node selected twice (two columns choosing the same row of one table in the
// template sample) is ambiguous and rejected: record the template sample with
// distinct rows per table, e.g. idx[c] = c.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "tg_abi.h"

namespace tgadapt {

struct LeafRole {
  std::uint8_t cls;     // TG_LEAF_PARAM / TG_LEAF_INPUT / TG_LEAF_CONST
  std::uint32_t index;  // param id or input column
};

/// Data-dependent selections and max-shift leaves of a reference recording.
class Recording {
 public:
  struct Select {
    std::uint32_t node;  // the node the template sample wired
    std::uint32_t at;    // tape size when selected: consumers at or after it
    tg_gather g;
  };
  struct Shift {
    std::uint32_t leaf;
    std::vector<std::uint32_t> over;
  };

  template <class TapeT, class VR>
  VR select(const TapeT& t, VR first, std::uint32_t stride, std::uint32_t n_rows, std::uint32_t col,
            std::uint32_t offset, std::int32_t idx) {
    if (n_rows == 0 || idx < 0 || static_cast<std::uint32_t>(idx) >= n_rows)
      throw std::invalid_argument("select: index " + std::to_string(idx) + " outside [0, " + std::to_string(n_rows) + ")");
    const std::uint64_t node = std::uint64_t(first.index) + std::uint64_t(stride) * std::uint32_t(idx) + offset;
    const std::uint64_t last = std::uint64_t(first.index) + std::uint64_t(stride) * (n_rows - 1) + offset;
    if (last >= t.size()) throw std::invalid_argument("select: table extends past the recorded nodes");
    selects.push_back({static_cast<std::uint32_t>(node), static_cast<std::uint32_t>(t.size()),
                       tg_gather{first.index, stride, n_rows, col, offset}});
    return VR{static_cast<std::uint32_t>(node)};
  }

  template <class TapeT, class VR>
  VR stopgrad_max(TapeT& t, std::span<const VR> xs) {
    if (xs.empty()) throw std::invalid_argument("stopgrad_max: empty input");
    auto m = t.value_of(xs[0]);
    for (std::size_t i = 1; i < xs.size(); ++i) m = std::max(m, t.value_of(xs[i]));
    const VR leaf = t.leaf(m);
    Shift s{leaf.index, {}};
    s.over.reserve(xs.size());
    for (const VR& x : xs) s.over.push_back(x.index);
    shifts.push_back(std::move(s));
    return leaf;
  }

  std::vector<Select> selects;
  std::vector<Shift> shifts;
};

/// Owns the arrays behind a tg_tape_desc.
struct DescArrays {
  std::vector<std::uint8_t> op, leaf_class;
  std::vector<std::uint64_t> child_offset;
  std::vector<std::uint32_t> child, leaf_index;
  std::vector<double> constant, leaf_value;
  std::vector<tg_gather> gathers;
  tg_tape_desc desc{};
};

/// roles: (leaf node, role) for the params and per-sample inputs; leaves
/// without a role are constants.  rec: the side record of selections and
/// max shifts (nullable: a tape without data-dependent choices).
template <class TapeT>
DescArrays describe(const TapeT& tape, std::uint32_t root, const std::vector<std::pair<std::uint32_t, LeafRole>>& roles,
                    const Recording* rec = nullptr) {
  using S = typename TapeT::scalar_type;
  DescArrays a;
  const std::uint32_t n = static_cast<std::uint32_t>(tape.size());
  a.op.resize(n);
  a.leaf_class.assign(n, TG_NODE_OP);
  a.leaf_index.assign(n, 0);
  a.constant.resize(n);
  a.leaf_value.resize(n);
  a.child_offset.reserve(n + 1);
  a.child_offset.push_back(0);
  // node -> (select id) and leaf -> (shift id)
  std::unordered_map<std::uint32_t, std::uint32_t> sel, shift;
  std::uint32_t n_index = 0;
  if (rec) {
    for (std::uint32_t g = 0; g < rec->selects.size(); ++g) {
      const auto& s = rec->selects[g];
      if (!sel.emplace(s.node, g).second)
        throw std::invalid_argument("tgadapt::describe: node " + std::to_string(s.node) +
                                    " selected twice (record the template sample with distinct rows per table)");
      a.gathers.push_back(s.g);
      n_index = std::max(n_index, s.g.index_col + 1);
    }
    for (std::uint32_t k = 0; k < rec->shifts.size(); ++k) {
      const auto& s = rec->shifts[k];
      if (s.leaf >= n || static_cast<int>(tape.op_at(s.leaf)) != 0) throw std::invalid_argument("tgadapt::describe: max-shift node is not a leaf");
      shift.emplace(s.leaf, k);
    }
  }
  std::uint32_t n_params = 0, n_inputs = 0;
  for (std::uint32_t i = 0; i < n; ++i) {
    a.op[i] = static_cast<std::uint8_t>(tape.op_at(i));
    a.constant[i] = static_cast<double>(tape.constant_at(i));
    a.leaf_value[i] = static_cast<double>(tape.value_at(i));
    if (const auto it = shift.find(i); it != shift.end()) {   // the per-sample stop-gradient max
      a.op[i] = static_cast<std::uint8_t>(TG_OP_STOPGRAD_MAX);
      a.constant[i] = 0.0;
      for (std::uint32_t c : rec->shifts[it->second].over) a.child.push_back(c);
      a.child_offset.push_back(a.child.size());
      continue;
    }
    if (a.op[i] == 0) a.leaf_class[i] = TG_LEAF_CONST;
    for (auto c : tape.children_at(i)) {
      const auto it = sel.find(c);
      if (it != sel.end() && rec->selects[it->second].at <= i) a.child.push_back(TG_GATHER_FLAG | it->second);
      else a.child.push_back(c);
    }
    a.child_offset.push_back(a.child.size());
  }
  for (const auto& [node, role] : roles) {
    if (node >= n || a.op[node] != 0) throw std::invalid_argument("tgadapt::describe: role on a non-leaf node");
    a.leaf_class[node] = role.cls;
    a.leaf_index[node] = role.index;
    if (role.cls == TG_LEAF_PARAM) n_params = std::max(n_params, role.index + 1);
    if (role.cls == TG_LEAF_INPUT) n_inputs = std::max(n_inputs, role.index + 1);
  }
  tg_tape_desc& d = a.desc;
  d.n_nodes = n;
  d.dtype = sizeof(S) == 8 ? TG_F64 : TG_F32;
  d.op = a.op.data();
  d.child_offset = a.child_offset.data();
  d.child = a.child.data();
  d.constant = a.constant.data();
  d.leaf_class = a.leaf_class.data();
  d.leaf_index = a.leaf_index.data();
  d.leaf_value = a.leaf_value.data();
  d.n_gathers = static_cast<std::uint32_t>(a.gathers.size());
  d.gathers = a.gathers.empty() ? nullptr : a.gathers.data();
  d.root = root;
  d.n_params = n_params;
  d.n_inputs = n_inputs;
  d.n_index_inputs = n_index;
  return a;
}

}  // namespace tgadapt
