// tg_from_tapegrad.hpp — describe a tape recorded with the reference API.
//
// Drop-in adapter for code that records with tapegrad::Tape (reference
// tape.hpp:68-353): reads ops() / children_at() / constant_at() / value_at()
// (tape.hpp:250-260) and the caller's leaf roles, and fills the plain arrays
// of tg_tape_desc for tg_compile.  Header-only, works with any tape type that
// exposes those members (tapegrad::Tape<float|double>, tg::Tape).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "tg_abi.h"

namespace tgadapt {

struct LeafRole {
  std::uint8_t cls;     // TG_LEAF_PARAM / TG_LEAF_INPUT / TG_LEAF_CONST
  std::uint32_t index;  // param id or input column
};

/// Owns the arrays behind a tg_tape_desc.
struct DescArrays {
  std::vector<std::uint8_t> op, leaf_class;
  std::vector<std::uint64_t> child_offset;
  std::vector<std::uint32_t> child, leaf_index;
  std::vector<double> constant, leaf_value;
  tg_tape_desc desc{};
};

/// roles: one entry per leaf node in index order (params, per-sample inputs,
/// constants).  Leaves without a role are constants.
template <class TapeT>
DescArrays describe(const TapeT& tape, std::uint32_t root, const std::vector<std::pair<std::uint32_t, LeafRole>>& roles) {
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
  std::uint32_t n_params = 0, n_inputs = 0;
  for (std::uint32_t i = 0; i < n; ++i) {
    a.op[i] = static_cast<std::uint8_t>(tape.op_at(i));
    a.constant[i] = static_cast<double>(tape.constant_at(i));
    a.leaf_value[i] = static_cast<double>(tape.value_at(i));
    if (a.op[i] == 0) a.leaf_class[i] = TG_LEAF_CONST;
    for (auto c : tape.children_at(i)) a.child.push_back(c);
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
  d.n_gathers = 0;
  d.gathers = nullptr;
  d.root = root;
  d.n_params = n_params;
  d.n_inputs = n_inputs;
  d.n_index_inputs = 0;
  return a;
}

}  // namespace tgadapt
