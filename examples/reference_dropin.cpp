// examples/reference_dropin.cpp — the integration a reference user writes.
//
// Records the Fig. 1 graph with the UNMODIFIED reference API
// (tapegrad::Tape + ops.hpp), describes it with include/tg_from_tapegrad.hpp
// and compiles it with tg_compile.  Prints the compiled program and the
// reference's own backward_with_scratch order next to the compiler's order.
// Build (tests/test_integration.py does this):
//   g++ -std=c++20 -I/root/reference/proj/include -Iinclude examples/reference_dropin.cpp \
//       -Lpaper_2503_13795_b200 -ltg -Wl,-rpath,$PWD/paper_2503_13795_b200
#include "tapegrad/tape.hpp"
template <> tapegrad::ValueRef tapegrad::Tape<double>::leaf(double v) {   // SURVEY.md §0 shim
  return emplace_with(OpKind::Leaf, v, 0, [](NodeIndex*) {});
}
#include "tapegrad/backprop.hpp"

#include <cstdio>

#include "tg_abi.h"
#include "tg_from_tapegrad.hpp"

int main() {
  using namespace tapegrad;
  Tape<double> t(64);
  const ValueRef a = t.leaf(-41.0), b = t.leaf(2.0);
  const ValueRef c = add(t, a, b);
  const ValueRef ab = mul(t, a, b);
  const ValueRef b3 = pow3(t, b);
  const ValueRef d = add(t, ab, b3);
  const ValueRef e = sub(t, c, d);
  const ValueRef f = sqr(t, e);
  const ValueRef two = t.leaf(2.0);
  const ValueRef g = div(t, f, two);
  ScratchBuffers<double> s;
  backward_with_scratch(t, g, s);   // reference order, for comparison

  // a and b are per-sample inputs 0 and 1; "2" stays a constant
  auto arrays = tgadapt::describe(t, g.index, {{a.index, {TG_LEAF_INPUT, 0}}, {b.index, {TG_LEAF_INPUT, 1}}});
  tg_program_t prog = nullptr;
  if (tg_compile(&arrays.desc, &prog) != TG_OK) { std::printf("compile failed: %s\n", tg_last_error()); return 1; }
  tg_program_info info{};
  tg_program_info_get(prog, &info);
  const uint32_t* order = nullptr;
  uint32_t n = 0;
  tg_program_order(prog, &order, &n);
  std::printf("nodes %u sample_nodes %u inputs %u fwd %u bwd %u\n", t.size(), info.n_sample_nodes, info.n_inputs,
              info.n_fwd_instr, info.n_bwd_instr);
  std::printf("reference order:");
  for (auto i : s.order) std::printf(" %u", i);
  std::printf("\ncompiled order: ");
  for (uint32_t i = 0; i < n; ++i) std::printf(" %u", order[i]);
  std::printf("\n");
  bool same = n == s.order.size();
  for (uint32_t i = 0; same && i < n; ++i) same = order[i] == s.order[i];
  std::printf("%s\n", same ? "ORDER_MATCH" : "ORDER_MISMATCH");
  tg_program_free(prog);
  return same ? 0 : 2;
}
