// tg_abi.cpp — extern "C" boundary of the B200 gradient oracle (include/tg_abi.h).
//
// No exception crosses this boundary: every entry point maps the reference's
// exception taxonomy (errors.hpp:9-36, std::domain_error / invalid_argument
// of ops.hpp and backprop.hpp) to a tg_status and a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <map>
#include <set>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "tg_abi.h"
#include "tg_comm.hpp"
#include "tg_jit.hpp"
#include "tg_models.hpp"
#include "tg_program.hpp"
#include "tg_recorder.hpp"
#include "../kernels/tg_staged.cuh"
#include "../kernels/tg_tape.cuh"
#include "../kernels/tg_synth.cuh"

namespace tgk {
cudaError_t launch_synth(const tgs::SynthArgs& a, const double* cdf_host, cudaStream_t st);
}

namespace {

thread_local std::string g_err;

tg_status fail(tg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

template <class F>
tg_status guard(F&& f) {
  try {
    return f();
  } catch (const tg::CapacityError& e) {
    return fail(TG_CAPACITY, e.what());
  } catch (const tg::InvalidHandle& e) {
    return fail(TG_INVALID_HANDLE, e.what());
  } catch (const tg::InvalidCheckpoint& e) {
    return fail(TG_INVALID_CHECKPOINT, e.what());
  } catch (const std::domain_error& e) {
    return fail(TG_DOMAIN, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(TG_INVALID_ARGUMENT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(TG_CAPACITY, "out of host memory");
  } catch (const std::exception& e) {
    return fail(TG_INVALID_ARGUMENT, e.what());
  }
}

#define TG_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return fail(TG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class S>
struct TgBuilder {
  using Scalar = S;
  using VR = tg::ValueRef;
  tg::Tape<S>& t;
  VR param(S v) { return t.param(v); }
  VR constant(S v) { return t.constant(v); }
  VR input(std::uint32_t c, S v) { return t.input(c, v); }
  VR gather(VR first, std::uint32_t stride, std::uint32_t n_rows, std::uint32_t col, std::uint32_t off,
            std::int32_t idx) {
    return t.gather(first, stride, n_rows, col, off, idx);
  }
  VR stopgrad_max(std::span<const VR> xs) { return tg::stopgrad_max(t, xs); }
  VR unary(std::uint8_t op, VR x) { return tg::unary(t, static_cast<tg::OpKind>(op), x); }
  VR binary(std::uint8_t op, VR x, VR y) { return tg::binary(t, static_cast<tg::OpKind>(op), x, y); }
  VR mul_by_constant(VR x, S c) { return tg::mul_by_constant(t, x, c); }
  VR varying(std::uint8_t op, std::span<const VR> xs) { return tg::varying(t, static_cast<tg::OpKind>(op), xs); }
  VR ip(std::span<const VR> x, std::span<const VR> y) { return tg::inner_product(t, x, y); }
  VR ipwb(std::span<const VR> x, std::span<const VR> y, VR b) { return tg::inner_product_with_bias(t, x, y, b); }
};

}  // namespace

tg_status tgcomm::fail_status(tg_status s, const std::string& msg) { return fail(s, msg); }

struct tg_recorder {
  tg_dtype dtype;
  std::unique_ptr<tg::Tape<double>> t64;
  std::unique_ptr<tg::Tape<float>> t32;
  template <class F> auto visit(F&& f) {
    if (dtype == TG_F64) return f(*t64);
    return f(*t32);
  }
};

// ---------------------------------------------------------------------------
// device program
// ---------------------------------------------------------------------------

struct tg_program {
  tgc::Program P;
  bool uploaded = false;
  std::vector<void*> allocs;
  tgc::Instr *d_fwd = nullptr, *d_bwd = nullptr, *d_ufwd = nullptr, *d_ubwd = nullptr;
  std::uint32_t *d_opnd = nullptr, *d_oaux = nullptr, *d_zero = nullptr, *d_inrows = nullptr, *d_cand = nullptr,
                *d_termoff = nullptr, *d_destuv = nullptr;
  std::uint8_t* d_oflag = nullptr;
  tgc::GatherTable *d_ug = nullptr, *d_sg = nullptr;
  tgc::Term* d_terms = nullptr;
  tgc::Dense* d_dense = nullptr;
  tgc::Attn* d_attn = nullptr;
  std::uint32_t* d_arows = nullptr;
  tgc::LNorm* d_lnorm = nullptr;
  std::uint32_t* d_lnrows = nullptr;
  std::uint8_t* d_lnflag = nullptr;
  void* d_consts = nullptr;
  unsigned long long* d_err_key = nullptr;
  double* d_err_val = nullptr;
  std::uint32_t* d_err_op = nullptr;
  unsigned* d_ticket = nullptr;   // grid-barrier words of the cooperative JIT form (TG_JIT_COOP=1 only)
  // launch configuration
  bool smem = true;
  unsigned S = 128;
  std::size_t ld_smem = 129;
  std::size_t smem_bytes = 0;
  unsigned occ_bound = 1;
  int occ = 0;
  int nsm = 148;
  std::uint64_t launches = 0;
  // last main launch, for domain-error diagnosis
  bool have_last = false;
  std::vector<unsigned char> last_args;
  std::size_t last_batch = 0;
  // kernel timing (tg_profile_enable)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::size_t ev_used = 0;
  // register-resident specialisation (tg_jit.cpp)
  tgj::JitKernel jit;
  // staged execution over an HBM SoA workspace (large tapes, dense layers as GEMMs)
  struct Stage { int batch; std::uint32_t begin, end; bool level = false; bool inputs_only = false; bool macro = false; };   // batch >= 0: GEMM stage; level: one
                                                                              // instruction per CTA column (k_level_range);
                                                                              // batch == kSumStage: sums[begin, end)
  // Dense layers of one dependency level over the same weights (a GPT's 64
  // positions): one launch per role with per-member row offsets.
  struct Batch {
    std::vector<std::uint32_t> members;   // dense ids, identical (w, b, n_out, n_in, act)
    std::vector<uint4> tab;               // member rows: forward | input adjoints | weight gradient
    uint4* d_tab = nullptr;
    std::vector<std::uint32_t> zero_x;    // x adjoint rows zeroed before an accumulating dX
    std::uint32_t* d_zero_x = nullptr;
    int beta = 0;
    bool bf = false, bx = false, bw = false;   // forward / dX / dW run batched (else per member)
    bool x_inputs = false;                     // every member's x rows are input leaves
    // dX writes dz of the layer below: C rows = the producing members' z rows
    // (tab[nm + p].z), act' taken from their h rows (= this batch's x rows,
    // tab[nm + p].w); the producing batch then skips its activation backward
    std::uint32_t dx_act = 0;
    bool skip_act = false;
  };
  std::vector<Batch> batches;
  // Contended adjoint rows of the reverse levels: pushes into a row with more
  // than one pusher in a level store to temporaries (rows n_rows ..), summed
  // into the row at the end of the level: {row, assign, first temporary, count}.
  std::vector<uint4> sums;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> level_sums;   // per reverse level: [begin, end) of sums
  uint4* d_sums = nullptr;
  std::uint32_t n_tmp = 0;
  bool levels = false;            // staged lists reordered into dependency levels (TG_STAGED_LEVELS=0: off)
  struct DensePlan {
    bool gemm = false;
    std::uint32_t xrow0 = 0;
    std::uint32_t dw_dest0 = tgc::kNone, db_dest0 = tgc::kNone;
    int beta = 0;                 // dX: 0 store, 1 accumulate
    bool x_inputs = false;        // x rows are all input leaves: dX only feeds the input gradients
    std::uint32_t x_col0 = tgc::kNone;   // x rows = input columns x_col0.. in order: GEMMs read the inputs array
    std::vector<std::uint32_t> zero_x;   // assign-flagged x rows zeroed first (mixed flags)
    std::uint32_t* d_zero_x = nullptr;
  };
  // embedding-MLP / softmax-CE tape run as one kernel (fused_mlp_plan, kernels/tg_fused.cu)
  struct FusedMlp {
    bool on = false;
    tgk::FusedMlpArgs args{};            // dims and parameter offsets (pointers set per call)
    std::vector<std::uint32_t> dmap;     // q -> destination
    std::uint32_t* d_dmap = nullptr;
  } fmlp;
  bool staged = false;
  std::vector<Stage> sfwd, sbwd;
  std::vector<DensePlan> dplan;
  std::vector<std::uint32_t> gen_dests;
  std::uint32_t* d_gen_dests = nullptr;
  // table-scatter dests (all terms kind 1) as histograms per (adjoint row, index column)
  std::vector<tgk::ScatterGroup> sc_groups;
  std::vector<tgk::ScatterUse> sc_uses;
  std::vector<std::uint32_t> sc_use_off, sc_dests;
  std::uint32_t sc_rmax = 0, sc_chunks = 1;
  tgk::ScatterGroup* d_sc_groups = nullptr;
  tgk::ScatterUse* d_sc_uses = nullptr;
  std::uint32_t *d_sc_use_off = nullptr, *d_sc_dests = nullptr;
  std::size_t chunk = 0;          // samples per chunk (0 = by batch)
  std::size_t mem_budget = 0;     // staged rows per chunk within this many bytes (0: TG_STAGED_MB or 64 GB)
  bool umma = true;               // fp32 dense layers on tcgen05 (3xTF32); TG_UMMA=0 -> SIMT GEMM
  bool attn_fast = false;         // fused heads on the shared-memory kernels (tg_attn.cu; TG_ATTN_FAST=0: interpreter)
  std::uint32_t attn_hd = 0;      // widest key / value block of the fused heads
  ~tg_program() {
    tgj::release(jit);
    for (auto& e : ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (void* p : allocs) cudaFree(p);
  }
  std::size_t tsz() const { return P.dtype == TG_F64 ? 8 : 4; }
  std::uint32_t n_dest() const { return static_cast<std::uint32_t>(P.dest_uv.size()); }
};

namespace {

constexpr int kSumStage = -2;
constexpr int kAttnStage = -3;   // fused attention heads [begin, end) of one level
constexpr std::size_t kSmemBudget = 200 * 1024;
constexpr unsigned kMaxOcc = 32;

// Dense layers with consecutive x rows run as GEMMs over the chunk; the rest of
// the instruction stream runs on the interpreter in ranges between them.
// Dependency-level schedule of the staged instruction lists.  Outside the
// dense layers the staged interpreter ran one thread per sample through every
// instruction of a range: for cfg4 (~6e5 nodes per sample) that is a serial,
// latency-bound walk with only `batch` threads in flight.  Here the forward
// list is stably sorted by dependency level (instructions of one level are
// independent) and the reverse list by (reverse level, sub-level), where a
// sub-level never holds two instructions pushing into the same adjoint row,
// so one launch per level runs every instruction of the level on every sample
// without atomics and in a fixed order.  Assign flags are recomputed for the
// new order; rows reachable from a slot gather only ever accumulate and are
// zeroed at the seed.  Both orders stay valid sequential orders, so the
// interpreter (domain-error diagnosis) runs them unchanged.
// Rows of a fused attention head: reads (q of every unit, k and v of every
// key) and outputs (o of every unit).
void attn_in_rows(const tgc::Program& P, std::uint32_t id, std::vector<std::uint32_t>& out) {
  const tgc::Attn& A = P.attn[id];
  for (std::uint32_t u = 0; u < A.n_units; ++u)
    for (std::uint32_t i = 0; i < A.hd; ++i) out.push_back(P.arows[A.unit_off + 3 * u] + i);
  for (std::uint32_t j = 0; j < A.n_keys; ++j) {
    for (std::uint32_t i = 0; i < A.hd; ++i) out.push_back(P.arows[A.key_off + 2 * j] + i);
    for (std::uint32_t i = 0; i < A.dv; ++i) out.push_back(P.arows[A.key_off + 2 * j + 1] + i);
  }
}
// Rows of a fused layer norm: reads (x) and outputs (n_i and y_i).
void ln_in_rows(const tgc::Program& P, std::uint32_t id, std::vector<std::uint32_t>& out) {
  const tgc::LNorm& L = P.lnorm[id];
  for (std::uint32_t i = 0; i < L.n; ++i) out.push_back(P.lnrows[L.off + i]);
}
void ln_out_rows(const tgc::Program& P, std::uint32_t id, std::vector<std::uint32_t>& out, bool with_n) {
  const tgc::LNorm& L = P.lnorm[id];
  for (std::uint32_t i = 0; i < L.n; ++i) {
    if (with_n) out.push_back(P.lnrows[L.off + L.n + i]);
    out.push_back(P.lnrows[L.off + 2 * L.n + i]);
  }
}
void attn_out_rows(const tgc::Program& P, std::uint32_t id, std::vector<std::uint32_t>& out) {
  const tgc::Attn& A = P.attn[id];
  for (std::uint32_t u = 0; u < A.n_units; ++u)
    for (std::uint32_t i = 0; i < A.dv; ++i) out.push_back(P.arows[A.unit_off + 3 * u + 1] + i);
}

void level_schedule(tg_program& pr, const std::vector<char>& gemm_dense) {
  tgc::Program& P = pr.P;
  const std::uint32_t R = P.n_rows;
  auto slot_rows = [&](std::uint32_t op, std::vector<std::uint32_t>& out) {
    const std::uint32_t m = op >> tgc::kModeShift, i = op & tgc::kIndexMask;
    if (m == tgc::kSlot) out.push_back(i);
    else if (m == tgc::kSGather) {
      const tgc::GatherTable& t = P.sgather[i];
      for (std::uint32_t r = 0; r < t.n_rows; ++r) out.push_back(P.cand[t.cand_off + r]);
    }
  };
  // ---- forward ----
  std::vector<std::uint32_t> row_level(R, 0), lvl(P.fwd.size(), 0), rows;
  for (std::size_t k = 0; k < P.fwd.size(); ++k) {
    const tgc::Instr& in = P.fwd[k];
    rows.clear();
    if (in.kind == tgc::kNode) for (std::uint32_t j = 0; j < in.nops; ++j) slot_rows(P.opnd[in.opnd + j], rows);
    if (in.kind == tgc::kDense) {
      const tgc::Dense& D = P.dense[in.aux];
      for (std::uint32_t j = 0; j < D.n_in; ++j) slot_rows(P.opnd[D.x_opnd + j], rows);
    }
    if (in.kind == tgc::kAttn) attn_in_rows(P, in.aux, rows);
    if (in.kind == tgc::kLNorm) ln_in_rows(P, in.aux, rows);
    std::uint32_t L = 0;
    for (std::uint32_t r : rows) L = std::max(L, row_level[r] + 1);
    lvl[k] = L;
    if (in.kind == tgc::kLNorm) {
      std::vector<std::uint32_t> orows;
      ln_out_rows(P, in.aux, orows, true);
      for (std::uint32_t r : orows) row_level[r] = L;
    } else if (in.kind == tgc::kAttn) {
      std::vector<std::uint32_t> orows;
      attn_out_rows(P, in.aux, orows);
      for (std::uint32_t r : orows) row_level[r] = L;
    } else if (in.kind == tgc::kDense) {
      const tgc::Dense& D = P.dense[in.aux];
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        row_level[D.out_row + j] = L;
        if (D.act_op) row_level[D.act_row + j] = L;
      }
    } else {
      row_level[in.out] = L;
    }
  }
  std::vector<std::uint32_t> ord(P.fwd.size());
  for (std::uint32_t k = 0; k < ord.size(); ++k) ord[k] = k;
  auto is_gemm = [&](const tgc::Instr& in) { return in.kind == tgc::kDense && gemm_dense[in.aux]; };
  // within a level the interpreter instructions first, then the GEMM stages
  // grouped by weight block (adjacent layers over one weight form a batch)
  auto gkey = [&](const tgc::Instr& in) -> std::uint64_t {
    if (in.kind == tgc::kAttn) return std::uint64_t(1) << 40;   // fused heads: their own stage, after the rest
    return is_gemm(in) ? 1 + std::uint64_t(P.dense[in.aux].w_uv) : 0;
  };
  std::stable_sort(ord.begin(), ord.end(), [&](std::uint32_t a, std::uint32_t b) {
    if (lvl[a] != lvl[b]) return lvl[a] < lvl[b];
    return gkey(P.fwd[a]) < gkey(P.fwd[b]);
  });
  std::vector<tgc::Instr> nf(P.fwd.size());
  std::vector<std::uint32_t> nlvl(P.fwd.size());
  for (std::size_t k = 0; k < ord.size(); ++k) { nf[k] = P.fwd[ord[k]]; nlvl[k] = lvl[ord[k]]; }
  P.fwd.swap(nf);
  P.fwd_level = nlvl;
  // ---- reverse: level = 1 + max level of the instructions pushing into the rows it reads ----
  // Pushes: "soft" (a slot operand of a node: may be redirected to a
  // temporary) and "hard" (slot-gather candidates, dense-layer x rows).
  struct Push { std::uint32_t row, pos; bool hard; };
  std::vector<std::vector<Push>> pushes(P.bwd.size());
  std::vector<std::uint32_t> pushed_level(R, 0), rl(P.bwd.size(), 0), sub(P.bwd.size(), 0);
  std::vector<char> has_push(R, 0);
  for (std::size_t k = 0; k < P.bwd.size(); ++k) {
    const tgc::Instr& in = P.bwd[k];
    rows.clear();
    std::vector<std::uint32_t> uv_aux;
    if (in.kind == tgc::kLNorm) {
      ln_out_rows(P, in.aux, rows, false);
      std::vector<std::uint32_t> xr;
      ln_in_rows(P, in.aux, xr);
      for (std::uint32_t r : xr) pushes[k].push_back({r, tgc::kNone, true});
    } else if (in.kind == tgc::kAttn) {
      attn_out_rows(P, in.aux, rows);
      std::vector<std::uint32_t> xr;
      attn_in_rows(P, in.aux, xr);
      for (std::uint32_t r : xr) pushes[k].push_back({r, tgc::kNone, true});
    } else if (in.kind == tgc::kDense) {
      const tgc::Dense& D = P.dense[in.aux];
      for (std::uint32_t j = 0; j < D.n_out; ++j) rows.push_back(D.act_op ? D.act_row + j : D.out_row + j);
      std::vector<std::uint32_t> xr;
      for (std::uint32_t j = 0; j < D.n_in; ++j) slot_rows(P.opnd[D.x_opnd + j], xr);
      for (std::uint32_t r : xr) pushes[k].push_back({r, tgc::kNone, true});
    } else {
      rows.push_back(in.out);
      for (std::uint32_t j = 0; j < in.nops; ++j) {
        const std::uint32_t pos = in.opnd + j, op = P.opnd[pos];
        const std::uint32_t m = op >> tgc::kModeShift;
        if (m == tgc::kUv) {
          if (P.oflag[pos] & tgc::kToAux) uv_aux.push_back(P.oaux[pos]);
        } else if (m == tgc::kSlot) {
          pushes[k].push_back({op & tgc::kIndexMask, pos, false});
        } else {
          std::vector<std::uint32_t> cr;
          slot_rows(op, cr);
          for (std::uint32_t r : cr) pushes[k].push_back({r, pos, true});
        }
      }
    }
    std::uint32_t L = 0;
    for (std::uint32_t r : rows) if (has_push[r]) L = std::max(L, pushed_level[r] + 1);
    rl[k] = L;
    auto mark = [&](std::uint32_t t) {
      pushed_level[t] = has_push[t] ? std::max(pushed_level[t], L) : L;
      has_push[t] = 1;
    };
    for (const Push& q : pushes[k]) mark(q.row);
    for (std::uint32_t t : uv_aux) mark(t);
  }
  // pushers per (level, row): a soft push into a row with several pushers in
  // its level goes to a temporary; hard pushes keep sub-levels among themselves
  std::unordered_map<std::uint64_t, std::uint32_t> cnt;
  for (std::size_t k = 0; k < P.bwd.size(); ++k)
    for (const Push& q : pushes[k]) ++cnt[(std::uint64_t(rl[k]) << 32) | q.row];
  auto contended = [&](std::size_t k, const Push& q) {
    return !q.hard && cnt[(std::uint64_t(rl[k]) << 32) | q.row] > 1;
  };
  std::unordered_map<std::uint64_t, std::uint32_t> last_sub;   // (level, row) -> last sub-level used
  for (std::size_t k = 0; k < P.bwd.size(); ++k) {
    std::uint32_t sl = 0;
    for (const Push& q : pushes[k]) {
      if (!q.hard) continue;
      auto it = last_sub.find((std::uint64_t(rl[k]) << 32) | q.row);
      if (it != last_sub.end()) sl = std::max(sl, it->second + 1);
    }
    sub[k] = sl;
    for (const Push& q : pushes[k])
      if (q.hard) last_sub[(std::uint64_t(rl[k]) << 32) | q.row] = sl;
  }
  std::vector<std::uint32_t> bo(P.bwd.size());
  for (std::uint32_t k = 0; k < bo.size(); ++k) bo[k] = k;
  std::stable_sort(bo.begin(), bo.end(), [&](std::uint32_t a, std::uint32_t b) {
    if (rl[a] != rl[b]) return rl[a] < rl[b];
    if (sub[a] != sub[b]) return sub[a] < sub[b];
    return gkey(P.bwd[a]) < gkey(P.bwd[b]);
  });
  std::vector<tgc::Instr> nb(P.bwd.size());
  std::vector<std::uint32_t> nbl(P.bwd.size());
  std::vector<std::vector<Push>> np(P.bwd.size());
  std::vector<std::uint32_t> nrl(P.bwd.size());
  for (std::size_t k = 0; k < bo.size(); ++k) {
    nb[k] = P.bwd[bo[k]];
    nbl[k] = (rl[bo[k]] << 12) | std::min<std::uint32_t>(sub[bo[k]], 4095);   // stage key
    nrl[k] = rl[bo[k]];
    np[k] = std::move(pushes[bo[k]]);
  }
  for (std::size_t k = 0; k < bo.size(); ++k) rl[k] = nrl[k];   // cnt keys stay valid: same levels
  P.bwd.swap(nb);
  P.bwd_level = nbl;
  // ---- temporaries (consecutive per contended row, in execution order) and
  // first-write (assign) flags for the new reverse order ----
  std::vector<char> gather_target(R, 0), seen(R, 0);
  for (const auto& t : P.sgather)
    for (std::uint32_t r = 0; r < t.n_rows; ++r) gather_target[P.cand[t.cand_off + r]] = 1;
  auto flag = [&](std::uint32_t pos) {
    const std::uint32_t op = P.opnd[pos];
    if ((op >> tgc::kModeShift) != tgc::kSlot) return;
    const std::uint32_t r = op & tgc::kIndexMask;
    if (!seen[r] && !gather_target[r]) P.oflag[pos] |= tgc::kAssign;
    else P.oflag[pos] &= static_cast<std::uint8_t>(~tgc::kAssign);
    seen[r] = 1;
  };
  pr.sums.clear();
  pr.level_sums.clear();
  pr.n_tmp = 0;
  for (std::size_t k0 = 0; k0 < P.bwd.size();) {
    std::size_t k1 = k0;
    while (k1 < P.bwd.size() && rl[k1] == rl[k0]) ++k1;
    std::vector<std::uint32_t> order;                               // contended rows, first-use order
    std::unordered_map<std::uint32_t, std::vector<std::uint32_t>> uses;   // row -> operand positions
    for (std::size_t k = k0; k < k1; ++k) {
      const tgc::Instr& in = P.bwd[k];
      if (in.kind == tgc::kLNorm) {   // x adjoints: pushes with first-write flags, like dense x operands
        const tgc::LNorm& LN = P.lnorm[in.aux];
        for (std::uint32_t i = 0; i < LN.n; ++i) {
          const std::uint32_t r = P.lnrows[LN.off + i];
          if (!seen[r] && !gather_target[r]) P.lnflag[LN.flag_off + i] |= tgc::kAssign;
          else P.lnflag[LN.flag_off + i] &= static_cast<std::uint8_t>(~tgc::kAssign);
          seen[r] = 1;
        }
        continue;
      }
      if (in.kind == tgc::kAttn) {   // stores its q / k / v adjoints
        std::vector<std::uint32_t> xr;
        attn_in_rows(P, in.aux, xr);
        for (std::uint32_t r : xr) seen[r] = 1;
        continue;
      }
      if (in.kind == tgc::kDense) {
        const tgc::Dense& D = P.dense[in.aux];
        for (std::uint32_t j = 0; j < D.n_in; ++j) flag(D.x_opnd + j);
        continue;
      }
      std::unordered_map<std::uint32_t, char> hot;   // positions of this instruction going to temporaries
      for (const Push& q : np[k])
        if (contended(k, q)) {
          auto& u = uses[q.row];
          if (u.empty()) order.push_back(q.row);
          u.push_back(q.pos);
          hot[q.pos] = 1;
        }
      for (std::uint32_t j = 0; j < in.nops; ++j) {
        const std::uint32_t pos = in.opnd + j;
        if ((P.opnd[pos] >> tgc::kModeShift) != tgc::kSlot) continue;
        if (hot.count(pos)) {
          P.oflag[pos] = static_cast<std::uint8_t>((P.oflag[pos] | tgc::kToAux) & ~tgc::kAssign);
        } else {
          P.oflag[pos] &= static_cast<std::uint8_t>(~tgc::kToAux);
          flag(pos);
        }
      }
    }
    const std::uint32_t lv = rl[k0];
    if (pr.level_sums.size() <= lv) pr.level_sums.resize(lv + 1, {0, 0});
    const std::uint32_t sb = static_cast<std::uint32_t>(pr.sums.size());
    std::uint32_t next = 0;
    for (std::uint32_t r : order) {
      const auto& u = uses[r];
      for (std::size_t i = 0; i < u.size(); ++i) P.oaux[u[i]] = R + next + static_cast<std::uint32_t>(i);
      const bool assign = !seen[r] && !gather_target[r];
      seen[r] = 1;
      pr.sums.push_back(uint4{r, assign ? 1u : 0u, R + next, static_cast<std::uint32_t>(u.size())});
      next += static_cast<std::uint32_t>(u.size());
    }
    pr.level_sums[lv] = {sb, static_cast<std::uint32_t>(pr.sums.size())};
    pr.n_tmp = std::max(pr.n_tmp, next);
    k0 = k1;
  }
  std::vector<char> zero(R, 0);
  for (std::uint32_t r : P.zero_rows) zero[r] = 1;
  for (std::uint32_t r = 0; r < R; ++r)
    if (gather_target[r] && !zero[r]) P.zero_rows.push_back(r);
}

// Recognises the embedding-MLP / softmax-CE composition (
// tg_models.hpp char_mlp: gathers -> linear(act) -> linear -> softmax_ce) in
// the compiled program, exactly: C x E gathered inputs of one V x E parameter
// table, two dense layers in a chain (the first with a fused activation whose
// derivative reads its output), and the CE nodes StopGradMax, O Sub, O Exp,
// AddVarying, Log, Sub(log, gather of the shifted logits by the target
// column) as the root.  Anything else keeps the staged chain.
bool fused_mlp_plan(const tgc::Program& P, tg_program::FusedMlp& fm, std::string& why) {
  using tgc::kNone;
  auto no = [&](const char* w) { why = w; return false; };
  if (P.dtype != TG_F32) return no("fp64");
  if (P.dense.size() != 2 || !P.attn.empty() || !P.lnorm.empty() || !P.ufwd.empty() || P.root_row == kNone ||
      P.n_inputs != 0 || !P.ugather.size())
    return no("not two dense layers over gathers with a per-sample root");
  auto slot = [&](std::uint32_t op, std::uint32_t& r) {
    r = op & tgc::kIndexMask;
    return (op >> tgc::kModeShift) == tgc::kSlot;
  };
  int i0 = -1, i1 = -1;
  for (int a = 0; a < 2 && i1 < 0; ++a) {
    const tgc::Dense& A = P.dense[a];
    const tgc::Dense& B = P.dense[1 - a];
    if (!A.act_op || A.act_row == kNone || B.act_op || B.n_in != A.n_out) continue;
    bool chain = true;
    for (std::uint32_t k = 0; k < B.n_in && chain; ++k) {
      std::uint32_t r;
      chain = slot(P.opnd[B.x_opnd + k], r) && r == A.act_row + k;
    }
    if (chain) { i0 = a; i1 = 1 - a; }
  }
  if (i0 < 0) return no("dense layers are not a chain");
  const tgc::Dense& D0 = P.dense[i0];
  const tgc::Dense& D1 = P.dense[i1];
  {
    using tg::OpKind;
    const std::uint32_t ao = D0.act_op;
    if (ao != std::uint32_t(OpKind::Relu) && ao != std::uint32_t(OpKind::Tanh) && ao != std::uint32_t(OpKind::Exp) &&
        ao != std::uint32_t(OpKind::Sigmoid))
      return no("activation derivative needs z");
  }
  const std::uint32_t NI = D0.n_in, H = D0.n_out, O = D1.n_out;
  // rows written by gather loads
  std::vector<int> gat(P.n_rows, -1);
  std::uint32_t n_node = 0, n_gather = 0, n_dense = 0;
  for (const tgc::Instr& in : P.fwd) {
    if (in.kind == tgc::kGatherLoad) { gat[in.out] = static_cast<int>(in.aux); ++n_gather; }
    else if (in.kind == tgc::kDense) ++n_dense;
    else if (in.kind == tgc::kNode) ++n_node;
    else return no("other instruction kinds");
  }
  if (n_gather != NI || n_dense != 2 || n_node != 2 * O + 4) return no("extra instructions");
  // gathered inputs: x[c E + e] = T[idx[col_c]][e], T at uv_E with row stride E
  std::uint32_t rows0, E = 0, V = 0, uvE = 0;
  if (!slot(P.opnd[D0.x_opnd], rows0) || gat[rows0] < 0) return no("first layer input is not gathered");
  {
    const tgc::GatherTable& g0 = P.ugather[gat[rows0]];
    V = g0.n_rows;
    uvE = P.cand[g0.cand_off];
    if (V < 2) return no("table of one row");
    E = P.cand[g0.cand_off + 1] - uvE;
  }
  if (E == 0 || NI % E || NI / E > 8) return no("gather layout");
  const std::uint32_t C = NI / E;
  tgk::FusedMlpArgs& a = fm.args;
  a = tgk::FusedMlpArgs{};
  for (std::uint32_t k = 0; k < NI; ++k) {
    std::uint32_t r;
    if (!slot(P.opnd[D0.x_opnd + k], r) || gat[r] < 0) return no("first layer input is not gathered");
    const tgc::GatherTable& g = P.ugather[gat[r]];
    const std::uint32_t c = k / E, e = k % E;
    if (g.n_rows != V) return no("gather tables differ in size");
    if (e == 0) a.ctx_col[c] = g.col;
    else if (g.col != a.ctx_col[c]) return no("one context over several index columns");
    for (std::uint32_t v = 0; v < V; ++v)
      if (P.cand[g.cand_off + v] != uvE + v * E + e) return no("gather candidates are not one table");
  }
  // the CE nodes, from the root down
  std::vector<int> ins(P.n_rows, -1);
  for (std::size_t i = 0; i < P.fwd.size(); ++i)
    if (P.fwd[i].kind == tgc::kNode) ins[P.fwd[i].out] = static_cast<int>(i);
  using tg::OpKind;
  auto node = [&](std::uint32_t row, OpKind op, std::uint32_t nops) -> const tgc::Instr* {
    if (row >= P.n_rows || ins[row] < 0) return nullptr;
    const tgc::Instr& in = P.fwd[ins[row]];
    return (in.op == static_cast<std::uint8_t>(op) && in.nops == nops) ? &in : nullptr;
  };
  const tgc::Instr* root = node(P.root_row, OpKind::Sub, 2);
  if (!root) return no("root is not a subtraction");
  std::uint32_t lrow, trow, mrow = kNone;
  if (!slot(P.opnd[root->opnd], lrow)) return no("CE log operand");
  const std::uint32_t zt = P.opnd[root->opnd + 1];
  if ((zt >> tgc::kModeShift) != tgc::kSGather) return no("CE target is not a gather");
  const tgc::GatherTable& tg = P.sgather[zt & tgc::kIndexMask];
  if (tg.n_rows != O) return no("CE target table size");
  const tgc::Instr* lg = node(lrow, OpKind::Log, 1);
  if (!lg || !slot(P.opnd[lg->opnd], trow)) return no("CE log");
  const tgc::Instr* tot = node(trow, OpKind::AddVarying, O);
  if (!tot) return no("CE sum");
  for (std::uint32_t j = 0; j < O; ++j) {
    std::uint32_t er, sr, zr, mr;
    const tgc::Instr* ex = slot(P.opnd[tot->opnd + j], er) ? node(er, OpKind::Exp, 1) : nullptr;
    const tgc::Instr* sb = ex && slot(P.opnd[ex->opnd], sr) ? node(sr, OpKind::Sub, 2) : nullptr;
    if (!sb || !slot(P.opnd[sb->opnd], zr) || zr != D1.out_row + j || !slot(P.opnd[sb->opnd + 1], mr))
      return no("CE shifted exponentials");
    if (P.cand[tg.cand_off + j] != sr) return no("CE target candidates");
    if (mrow == kNone) mrow = mr;
    else if (mr != mrow) return no("CE shift");
  }
  const tgc::Instr* mx = node(mrow, OpKind::StopGradMax, O);
  if (!mx) return no("CE shift is not a stop-gradient max");
  for (std::uint32_t j = 0; j < O; ++j) {
    std::uint32_t zr;
    if (!slot(P.opnd[mx->opnd + j], zr) || zr != D1.out_row + j) return no("CE max operands");
  }
  a.C = C; a.E = E; a.V = V; a.H = H; a.O = O; a.act = D0.act_op; a.tgt_col = tg.col;
  a.uv_E = uvE; a.uv_W1 = D0.w_uv; a.uv_b1 = D0.b_uv; a.uv_W2 = D1.w_uv; a.uv_b2 = D1.b_uv;
  a.nq = H * NI + H + O * H + O + V * E;
  // destinations, and no destination the kernel does not produce
  std::vector<std::uint32_t> inv(P.n_uv, kNone);
  for (std::uint32_t d = 0; d < P.dest_uv.size(); ++d) inv[P.dest_uv[d]] = d;
  fm.dmap.assign(a.nq, kNone);
  std::uint32_t covered = 0;
  auto map = [&](std::uint32_t q, std::uint32_t u) {
    if (u < P.n_params && inv[u] != kNone) { fm.dmap[q] = inv[u]; ++covered; }
  };
  std::uint32_t q = 0;
  for (std::uint32_t i = 0; i < H * NI; ++i) map(q++, a.uv_W1 + i);
  for (std::uint32_t i = 0; i < H; ++i, ++q) if (a.uv_b1 != kNone) map(q, a.uv_b1 + i);
  for (std::uint32_t i = 0; i < O * H; ++i) map(q++, a.uv_W2 + i);
  for (std::uint32_t i = 0; i < O; ++i, ++q) if (a.uv_b2 != kNone) map(q, a.uv_b2 + i);
  for (std::uint32_t i = 0; i < V * E; ++i) map(q++, uvE + i);
  if (covered != P.dest_uv.size()) return no("gradient destinations outside the fused layers");
  if (tgk::fused_mlp_smem(a) > 227 * 1024) return no("does not fit one SM's shared memory");
  return true;
}

void build_staged_plan(tg_program& pr) {
  const tgc::Program& P = pr.P;
  const char* env = std::getenv("TG_STAGED");
  bool big = false;
  pr.dplan.assign(P.dense.size(), {});
  for (std::size_t i = 0; i < P.dense.size(); ++i) {
    const tgc::Dense& D = P.dense[i];
    tg_program::DensePlan& dp = pr.dplan[i];
    dp.xrow0 = P.opnd[D.x_opnd] & tgc::kIndexMask;
    bool consec = true;
    for (std::uint32_t k = 0; k < D.n_in; ++k)
      consec = consec && (P.opnd[D.x_opnd + k] >> tgc::kModeShift) == tgc::kSlot &&
               (P.opnd[D.x_opnd + k] & tgc::kIndexMask) == dp.xrow0 + k;
    dp.gemm = consec && std::uint64_t(D.n_out) * D.n_in >= 256;
    if (std::uint64_t(D.n_out) * D.n_in >= 2048) big = true;
  }
  pr.staged = env ? env[0] == '1' : (big && !tgj::eligible(P));
  {
    const char* af = std::getenv("TG_ATTN_FAST");
    pr.attn_fast = pr.tsz() == 4 && !P.attn.empty() && !(af && af[0] == '0');
    for (const auto& A : P.attn) {
      pr.attn_fast = pr.attn_fast && tgk::attn_fast_ok(A);
      pr.attn_hd = std::max({pr.attn_hd, A.hd, A.dv});
    }
  }
  if (const char* u = std::getenv("TG_UMMA")) pr.umma = u[0] != '0';
  if (!pr.staged || P.root_row == tgc::kNone) { pr.staged = false; return; }
  {
    // opt-in (TG_FUSED_MLP=1): the one-kernel form is correct but measured slower
    // than the staged chain on cfg3 (1.90 vs 1.43 ms, profiles/r07/README.md)
    const char* fe = std::getenv("TG_FUSED_MLP");
    std::string why;
    pr.fmlp.on = fe && fe[0] == '1' && fused_mlp_plan(P, pr.fmlp, why);
    if (fe && fe[0] == '1' && !pr.fmlp.on && std::getenv("TG_FUSED_MLP_WHY")) std::fprintf(stderr, "fused_mlp: %s\n", why.c_str());
  }
  {
    const char* lv = std::getenv("TG_STAGED_LEVELS");
    pr.levels = !(lv && lv[0] == '0');
    if (pr.levels) {
      std::vector<char> gd(P.dense.size(), 0);
      for (std::size_t i = 0; i < P.dense.size(); ++i) gd[i] = pr.dplan[i].gemm ? 1 : 0;
      level_schedule(pr, gd);
    }
  }
  // Weight / bias gradient destinations handled by the GEMM path.  Dense
  // layers over one weight block (a GPT's positions) form a weight group; the
  // group's dests are covered when every user runs as a GEMM and each dest's
  // terms are exactly the users' products (dW[j][k]: G[out_u + j] . V[x_u + k];
  // db[j]: G[out_u + j]), so the split-K GEMMs and row sums of the users
  // accumulate the whole gradient.
  std::vector<std::uint8_t> covered(P.dest_uv.size(), 0);
  std::unordered_map<std::uint32_t, std::uint32_t> dest_of_uv;
  for (std::uint32_t d = 0; d < P.dest_uv.size(); ++d) dest_of_uv[P.dest_uv[d]] = d;
  std::map<std::uint32_t, std::vector<std::uint32_t>> users;
  for (std::uint32_t i = 0; i < P.dense.size(); ++i) users[P.dense[i].w_uv].push_back(i);
  for (const auto& [w, us] : users) {
    const tgc::Dense& D0 = P.dense[us.front()];
    bool ok = true;
    std::unordered_map<std::uint32_t, std::uint32_t> x_of_out;   // out_row -> x row0
    for (std::uint32_t u : us) {
      const tgc::Dense& D = P.dense[u];
      ok = ok && pr.dplan[u].gemm && D.n_out == D0.n_out && D.n_in == D0.n_in;
      x_of_out[D.out_row] = pr.dplan[u].xrow0;
    }
    if (!ok) continue;
    const std::uint32_t nu = static_cast<std::uint32_t>(us.size());
    auto it = dest_of_uv.find(w);
    std::uint32_t d0 = it == dest_of_uv.end() ? tgc::kNone : it->second;
    ok = d0 != tgc::kNone && d0 + std::size_t(D0.n_out) * D0.n_in <= P.dest_uv.size();
    for (std::uint32_t j = 0; ok && j < D0.n_out; ++j)
      for (std::uint32_t k = 0; ok && k < D0.n_in; ++k) {
        const std::uint32_t d = d0 + j * D0.n_in + k;
        ok = P.dest_uv[d] == w + j * D0.n_in + k && P.term_off[d + 1] - P.term_off[d] == nu;
        for (std::uint32_t q = P.term_off[d]; ok && q < P.term_off[d + 1]; ++q) {
          const tgc::Term& t = P.terms[q];
          const auto x = t.a >= j ? x_of_out.find(t.a - j) : x_of_out.end();
          ok = t.kind == 0 && t.coef == 1.0 && x != x_of_out.end() && t.f == x->second + k;
        }
      }
    if (ok) {
      for (std::uint32_t u : us) pr.dplan[u].dw_dest0 = d0;
      for (std::uint32_t q = 0; q < D0.n_out * D0.n_in; ++q) covered[d0 + q] = 1;
    }
    bool bok = D0.b_uv != tgc::kNone;
    for (std::uint32_t u : us) bok = bok && P.dense[u].b_uv == D0.b_uv;
    auto bt = bok ? dest_of_uv.find(D0.b_uv) : dest_of_uv.end();
    bok = bok && bt != dest_of_uv.end() && bt->second + D0.n_out <= P.dest_uv.size();
    for (std::uint32_t j = 0; bok && j < D0.n_out; ++j) {
      const std::uint32_t d = bt->second + j;
      bok = P.dest_uv[d] == D0.b_uv + j && P.term_off[d + 1] - P.term_off[d] == nu;
      for (std::uint32_t q = P.term_off[d]; bok && q < P.term_off[d + 1]; ++q) {
        const tgc::Term& t = P.terms[q];
        bok = t.kind == 0 && t.coef == 1.0 && t.f == tgc::kNone && t.a >= j && x_of_out.count(t.a - j);
      }
    }
    if (bok) {
      for (std::uint32_t u : us) pr.dplan[u].db_dest0 = bt->second;
      for (std::uint32_t j = 0; j < D0.n_out; ++j) covered[bt->second + j] = 1;
    }
  }
  std::vector<char> is_input(P.n_rows, 0);
  for (std::uint32_t r : P.input_rows) if (r != tgc::kNone) is_input[r] = 1;
  for (std::size_t i = 0; i < P.dense.size(); ++i) {
    const tgc::Dense& D = P.dense[i];
    tg_program::DensePlan& dp = pr.dplan[i];
    if (!dp.gemm) continue;
    dp.x_inputs = true;
    for (std::uint32_t k = 0; k < D.n_in; ++k) dp.x_inputs = dp.x_inputs && is_input[dp.xrow0 + k];
    std::uint32_t n_assign = 0;
    for (std::uint32_t k = 0; k < D.n_in; ++k) n_assign += (P.oflag[D.x_opnd + k] & tgc::kAssign) ? 1 : 0;
    dp.beta = n_assign == D.n_in ? 0 : 1;
    if (n_assign && n_assign != D.n_in)
      for (std::uint32_t k = 0; k < D.n_in; ++k)
        if (P.oflag[D.x_opnd + k] & tgc::kAssign) dp.zero_x.push_back(dp.xrow0 + k);
  }
  pr.gen_dests.clear();
  pr.sc_groups.clear();
  pr.sc_uses.clear();
  pr.sc_use_off.assign(1, 0);
  pr.sc_dests.clear();
  pr.sc_rmax = 0;
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::uint32_t> group_of;
  const std::uint32_t r_cap = pr.tsz() == 8 ? 192 : 384;   // bins[R][128] in shared memory
  for (std::uint32_t d = 0; d < P.dest_uv.size(); ++d) {
    if (covered[d]) continue;
    bool scatter = P.term_off[d + 1] > P.term_off[d];
    for (std::uint32_t q = P.term_off[d]; q < P.term_off[d + 1] && scatter; ++q)
      scatter = P.terms[q].kind == 1 && P.terms[q].row >= 0 && static_cast<std::uint32_t>(P.terms[q].row) < r_cap;
    if (!scatter) {
      pr.gen_dests.push_back(d);
      continue;
    }
    for (std::uint32_t q = P.term_off[d]; q < P.term_off[d + 1]; ++q) {
      const tgc::Term& t = P.terms[q];
      const auto key = std::make_pair(t.a, t.f);
      auto it = group_of.find(key);
      if (it == group_of.end()) {
        it = group_of.emplace(key, static_cast<std::uint32_t>(pr.sc_groups.size())).first;
        pr.sc_groups.push_back({t.a, t.f, 0, 0});
      }
      tgk::ScatterGroup& g = pr.sc_groups[it->second];
      g.rows = std::max<std::uint32_t>(g.rows, static_cast<std::uint32_t>(t.row) + 1);
      pr.sc_uses.push_back({it->second, static_cast<std::uint32_t>(t.row), t.coef});
    }
    pr.sc_dests.push_back(d);
    pr.sc_use_off.push_back(static_cast<std::uint32_t>(pr.sc_uses.size()));
  }
  for (const auto& g : pr.sc_groups) pr.sc_rmax = std::max(pr.sc_rmax, g.rows);
  // sample chunks: about four CTAs per SM over all groups
  pr.sc_chunks = pr.sc_groups.empty() ? 1 : std::max<std::uint32_t>(
      1, std::min<std::uint32_t>(256, (592 + static_cast<std::uint32_t>(pr.sc_groups.size()) - 1) /
                                          static_cast<std::uint32_t>(pr.sc_groups.size())));
  // stages: GEMM dense groups on their own; the rest either in instruction
  // ranges (one thread per sample) or, with levels, one range per level key
  const char* be = std::getenv("TG_STAGED_BATCH");
  const bool batching = !(be && be[0] == '0');
  auto same_sig = [&](std::uint32_t a, std::uint32_t b) {
    const tgc::Dense &A = P.dense[a], &B = P.dense[b];
    return A.w_uv == B.w_uv && A.b_uv == B.b_uv && A.n_out == B.n_out && A.n_in == B.n_in && A.act_op == B.act_op &&
           pr.dplan[a].dw_dest0 == pr.dplan[b].dw_dest0 && pr.dplan[a].db_dest0 == pr.dplan[b].db_dest0;
  };
  auto split = [&](const std::vector<tgc::Instr>& list, const std::vector<std::uint32_t>& key,
                   std::vector<tg_program::Stage>& out, bool sums) {
    out.clear();
    const bool lv = pr.levels && key.size() == list.size();
    std::uint32_t b = 0;
    auto flush = [&](std::uint32_t e) {
      if (e > b) out.push_back({-1, b, e, lv});
      b = e;
    };
    // after the last stage of a reverse level: the sums of its contended rows
    auto level_end = [&](std::uint32_t k) {
      if (!sums || !lv) return;
      const std::uint32_t L = key[k] >> 12;
      if (L < pr.level_sums.size() && pr.level_sums[L].second > pr.level_sums[L].first)
        out.push_back({kSumStage, pr.level_sums[L].first, pr.level_sums[L].second, false});
    };
    for (std::uint32_t k = 0; k < list.size(); ++k) {
      if (lv && k > 0 && (key[k] >> 12) != (key[k - 1] >> 12)) {
        flush(k);
        level_end(k - 1);
      }
      if (list[k].kind == tgc::kDense && pr.dplan[list[k].aux].gemm) {
        flush(k);
        const std::uint32_t id = list[k].aux;
        const bool join = lv && batching && !out.empty() && out.back().batch >= 0 && out.back().end == k &&
                          key[k] == key[k - 1] && same_sig(pr.batches[out.back().batch].members.front(), id);
        if (join) {
          pr.batches[out.back().batch].members.push_back(id);
          out.back().end = k + 1;
        } else {
          pr.batches.push_back({});
          pr.batches.back().members.push_back(id);
          out.push_back({static_cast<int>(pr.batches.size() - 1), k, k + 1, false});
        }
        b = k + 1;
      } else if (list[k].kind == tgc::kAttn) {
        flush(k);
        if (!out.empty() && out.back().batch == kAttnStage && out.back().end == k && (!lv || key[k] == key[k - 1]))
          out.back().end = k + 1;
        else
          out.push_back({kAttnStage, k, k + 1, lv});
        b = k + 1;
      } else if (lv && k > b && key[k] != key[k - 1]) {
        flush(k);
      }
    }
    flush(static_cast<std::uint32_t>(list.size()));
    if (!list.empty()) level_end(static_cast<std::uint32_t>(list.size() - 1));
  };
  pr.batches.clear();
  split(P.fwd, P.fwd_level, pr.sfwd, false);
  split(P.bwd, P.bwd_level, pr.sbwd, true);
  // interpreter stages holding macro-instructions (fused layer norms, ...)
  // run one sample per thread: the per-sample routines carry their own
  // memory parallelism, and four samples per thread would serialise them
  for (int w = 0; w < 2; ++w)
    for (auto& stg : w ? pr.sbwd : pr.sfwd)
      if (stg.batch == -1)
        for (std::uint32_t k = stg.begin; k < stg.end && !stg.macro; ++k) {
          const auto kind = (w ? P.bwd : P.fwd)[k].kind;
          stg.macro = kind == tgc::kDense || kind == tgc::kAttn;   // (kLNorm has a four-sample form)
        }
  // batch tables: forward {0, x, z, h}, input adjoints {0, z, x, 0}, weight gradient {z, x, 0, 0}
  const bool tc = pr.tsz() == 4 && pr.umma;
  for (auto& B : pr.batches) {
    const std::uint32_t nm = static_cast<std::uint32_t>(B.members.size());
    const tgc::Dense& D0 = P.dense[B.members.front()];
    B.tab.assign(3 * std::size_t(nm), uint4{0, 0, 0, 0});
    B.beta = 0;
    for (std::uint32_t p = 0; p < nm; ++p) {
      const tgc::Dense& D = P.dense[B.members[p]];
      const auto& dp = pr.dplan[B.members[p]];
      B.tab[p] = uint4{0, dp.xrow0, D.out_row, D.act_op ? D.act_row : 0};
      B.tab[nm + p] = uint4{0, D.out_row, dp.xrow0, 0};
      B.tab[2 * nm + p] = uint4{D.out_row, dp.xrow0, 0, 0};
      B.beta |= dp.beta;
    }
    B.x_inputs = true;
    for (std::uint32_t u : B.members) B.x_inputs = B.x_inputs && pr.dplan[u].x_inputs;
    B.zero_x.clear();
    for (std::uint32_t u : B.members) {
      const auto& dp = pr.dplan[u];
      if (B.beta && !dp.beta)
        for (std::uint32_t k = 0; k < P.dense[u].n_in; ++k) B.zero_x.push_back(dp.xrow0 + k);
      else
        B.zero_x.insert(B.zero_x.end(), dp.zero_x.begin(), dp.zero_x.end());
    }
    // an offset MN-major operand must end on a k-tile: a tile past K would read
    // the next rows (TMA zero-fills only past the map), so such roles loop
    B.bf = tc && nm > 1 && D0.n_in % 32 == 0;
    B.bx = tc && nm > 1 && D0.n_out % 32 == 0;
    B.bw = tc && nm > 1 && pr.dplan[B.members.front()].dw_dest0 != tgc::kNone;
  }
  // Input adjoints fused with the activation backward of the layer below.  A
  // batch C whose x rows are exactly the activation rows h of a batch A (act'
  // expressible in h), where C's dX is the only push into those rows and
  // assigns them, and no batch term reads their adjoints, writes
  // G[z_A] = act'(h) * (W^T dZ_C) in its GEMM epilogue: G[h] is never
  // materialised and A's activation-backward pass (read G[h], V[h], write
  // G[z]) disappears.  TG_DX_ACT=0 disables.
  const char* dxa = std::getenv("TG_DX_ACT");
  if (!(dxa && dxa[0] == '0')) {
    std::vector<std::uint32_t> pushers(P.n_rows, 0);
    auto push_opnd = [&](std::uint32_t o) {
      if ((P.opnd[o] >> tgc::kModeShift) == tgc::kSlot && (P.opnd[o] & tgc::kIndexMask) < P.n_rows)
        ++pushers[P.opnd[o] & tgc::kIndexMask];
    };
    for (const auto& I : P.fwd) {
      if (I.kind == tgc::kNode)
        for (std::uint32_t k = 0; k < I.nops; ++k) push_opnd(I.opnd + k);
      else if (I.kind == tgc::kDense)
        for (std::uint32_t k = 0; k < P.dense[I.aux].n_in; ++k) push_opnd(P.dense[I.aux].x_opnd + k);
      else if (I.kind == tgc::kAttn || I.kind == tgc::kLNorm) {
        std::vector<std::uint32_t> xr;
        if (I.kind == tgc::kAttn) attn_in_rows(P, I.aux, xr);
        else ln_in_rows(P, I.aux, xr);
        for (std::uint32_t r : xr) ++pushers[r];
      }
    }
    std::vector<char> term_a(P.n_rows, 0);
    for (const auto& t : P.terms)
      if (t.a < P.n_rows) term_a[t.a] = 1;
    // the reverse list's batches (the forward list has its own copies)
    std::vector<char> in_bwd(pr.batches.size(), 0);
    for (const auto& stg : pr.sbwd)
      if (stg.batch >= 0) in_bwd[stg.batch] = 1;
    std::unordered_map<std::uint32_t, std::pair<std::uint32_t, std::uint32_t>> act_owner;   // h row0 -> (batch, member)
    for (std::uint32_t bi = 0; bi < pr.batches.size(); ++bi)
      if (in_bwd[bi])
      for (std::uint32_t p = 0; p < pr.batches[bi].members.size(); ++p) {
        const tgc::Dense& D = P.dense[pr.batches[bi].members[p]];
        if (D.act_op == std::uint32_t(tg::OpKind::Relu) || D.act_op == std::uint32_t(tg::OpKind::Tanh) ||
            D.act_op == std::uint32_t(tg::OpKind::Exp) || D.act_op == std::uint32_t(tg::OpKind::Sigmoid))   // act' from h
          act_owner[D.act_row] = {bi, p};
      }
    for (std::uint32_t ci = 0; ci < pr.batches.size(); ++ci) {
      auto& C = pr.batches[ci];
      const std::uint32_t nm = static_cast<std::uint32_t>(C.members.size());
      bool ok = in_bwd[ci] && !C.x_inputs && C.zero_x.empty() && C.beta == 0;
      std::int64_t ab = -1;
      std::vector<std::uint32_t> zrow(nm);
      std::vector<char> seen;
      for (std::uint32_t p = 0; ok && p < nm; ++p) {
        const tgc::Dense& D = P.dense[C.members[p]];
        const auto& dp = pr.dplan[C.members[p]];
        auto it = act_owner.find(dp.xrow0);
        ok = dp.beta == 0 && it != act_owner.end() && (ab < 0 || ab == it->second.first);
        if (!ok) break;
        ab = it->second.first;
        if (seen.empty()) seen.assign(pr.batches[ab].members.size(), 0);
        const tgc::Dense& A = P.dense[pr.batches[ab].members[it->second.second]];
        ok = A.n_out == D.n_in && !seen[it->second.second] && &pr.batches[ab] != &C;
        seen[it->second.second] = 1;
        for (std::uint32_t k = 0; ok && k < D.n_in; ++k)
          ok = pushers[dp.xrow0 + k] == 1 && !term_a[dp.xrow0 + k];
        zrow[p] = A.out_row;
      }
      ok = ok && ab >= 0 && pr.batches[ab].members.size() == nm;
      if (!ok) continue;
      C.dx_act = P.dense[pr.batches[ab].members.front()].act_op;
      for (std::uint32_t p = 0; p < nm; ++p)
        C.tab[nm + p] = uint4{0, P.dense[C.members[p]].out_row, zrow[p], pr.dplan[C.members[p]].xrow0};
      pr.batches[ab].skip_act = true;
    }
  }
  // Dense layers over input leaves read the caller's inputs array ([col][batch],
  // the rows' own SoA layout) instead of copies in V; a forward stage of input
  // loads whose rows no other consumer reads is then skipped (cfg5: 784 rows,
  // 3.3 GB copied per step at b = 1M).  TG_DIRECT_X=0 disables.
  const char* dxx = std::getenv("TG_DIRECT_X");
  if (!(dxx && dxx[0] == '0') && pr.umma && pr.tsz() == 4) {
    std::vector<std::uint32_t> col_of(P.n_rows, tgc::kNone);
    for (std::uint32_t c = 0; c < P.input_rows.size(); ++c)
      if (P.input_rows[c] != tgc::kNone && P.input_rows[c] < P.n_rows) col_of[P.input_rows[c]] = c;
    std::vector<char> other(P.n_rows, 0);   // read by something other than a direct-input GEMM
    for (std::size_t i = 0; i < P.dense.size(); ++i) {
      const tgc::Dense& D = P.dense[i];
      auto& dp = pr.dplan[i];
      if (!dp.gemm || !dp.x_inputs || col_of[dp.xrow0] == tgc::kNone) continue;
      bool ok = true;
      for (std::uint32_t k = 0; ok && k < D.n_in; ++k) ok = col_of[dp.xrow0 + k] == col_of[dp.xrow0] + k;
      if (ok) dp.x_col0 = col_of[dp.xrow0];
    }
    for (const auto& B : pr.batches)   // batched launches offset rows of V: single-member layers only
      if (B.members.size() > 1)
        for (std::uint32_t u : B.members) pr.dplan[u].x_col0 = tgc::kNone;
    auto mark = [&](std::uint32_t o) {
      if ((P.opnd[o] >> tgc::kModeShift) == tgc::kSlot && (P.opnd[o] & tgc::kIndexMask) < P.n_rows)
        other[P.opnd[o] & tgc::kIndexMask] = 1;
    };
    for (const auto& I : P.fwd) {
      if (I.kind == tgc::kNode)
        for (std::uint32_t k = 0; k < I.nops; ++k) mark(I.opnd + k);
      else if (I.kind == tgc::kDense && pr.dplan[I.aux].x_col0 == tgc::kNone)
        for (std::uint32_t k = 0; k < P.dense[I.aux].n_in; ++k) mark(P.dense[I.aux].x_opnd + k);
      else if (I.kind == tgc::kAttn || I.kind == tgc::kLNorm) {
        std::vector<std::uint32_t> xr;
        if (I.kind == tgc::kAttn) attn_in_rows(P, I.aux, xr);
        else ln_in_rows(P, I.aux, xr);
        for (std::uint32_t r : xr) other[r] = 1;
      }
    }
    // batch terms reading V of a row outside the GEMM-covered weight gradients
    for (std::uint32_t d = 0; d < P.dest_uv.size(); ++d)
      if (!covered[d])
        for (std::uint32_t q = P.term_off[d]; q < P.term_off[d + 1]; ++q)
          if (P.terms[q].kind == 0 && P.terms[q].f < P.n_rows) other[P.terms[q].f] = 1;
    // (a direct-input layer's weight gradient must itself be GEMM-covered)
    for (std::size_t i = 0; i < P.dense.size(); ++i) {
      const auto& dp = pr.dplan[i];
      if (dp.x_col0 != tgc::kNone && dp.dw_dest0 == tgc::kNone)
        for (std::uint32_t k = 0; k < P.dense[i].n_in; ++k) other[dp.xrow0 + k] = 1;
    }
    for (auto& stg : pr.sfwd) {
      if (stg.batch != -1) continue;
      bool only = stg.end > stg.begin;
      for (std::uint32_t k = stg.begin; only && k < stg.end; ++k)
        only = P.fwd[k].kind == tgc::kInputLoad && P.fwd[k].out < P.n_rows && !other[P.fwd[k].out];
      stg.inputs_only = only;
    }
  }
  if (const char* v = std::getenv("TG_STAGED_VERBOSE"); v && v[0] == '1') {
    std::size_t ng = 0;
    for (std::size_t i = 0; i < P.dense.size(); ++i) {
      ng += pr.dplan[i].gemm;
      if (!pr.dplan[i].gemm)
        std::fprintf(stderr, "[staged] dense %zu: %u x %u interpreted (x rows not consecutive)\n", i,
                     P.dense[i].n_out, P.dense[i].n_in);
    }
    auto stats = [&](const char* name, const std::vector<tg_program::Stage>& st, const std::vector<tgc::Instr>& list) {
      std::size_t nl = 0, ni = 0, nops = 0, small = 0;
      for (const auto& s : st) {
        if (s.batch != -1) continue;
        ++nl;
        ni += s.end - s.begin;
        small += (s.end - s.begin) < 128;
        for (std::uint32_t k = s.begin; k < s.end; ++k)
          nops += list[k].kind == tgc::kDense ? std::size_t(P.dense[list[k].aux].n_in) * P.dense[list[k].aux].n_out
                                              : list[k].nops;
      }
      std::fprintf(stderr, "[staged] %s: %zu stages (%zu interpreter, %zu with <128 instrs), %zu instrs, %zu operands\n",
                   name, st.size(), nl, small, ni, nops);
      std::map<int, std::size_t> ops_small;
      std::set<std::uint32_t> lv_small;
      const auto& key = list.data() == P.fwd.data() ? P.fwd_level : P.bwd_level;
      for (const auto& s : st)
        if (s.batch == -1 && s.end - s.begin < 128)
          for (std::uint32_t k = s.begin; k < s.end; ++k) {
            ops_small[list[k].kind == tgc::kNode ? list[k].op : 1000 + list[k].kind]++;
            if (key.size() == list.size()) lv_small.insert(key[k] >> 12);
          }
      std::fprintf(stderr, "[staged]   small stages span %zu levels; ops:", lv_small.size());
      for (const auto& [op, c] : ops_small) std::fprintf(stderr, " %d:%zu", op, c);
      std::fprintf(stderr, "\n");
    };
    std::size_t nb = 0, nbm = 0;
    for (const auto& B : pr.batches) if (B.members.size() > 1) { ++nb; nbm += B.members.size(); }
    std::size_t nfx = 0, nio = 0;
    for (const auto& B : pr.batches) nfx += B.dx_act != 0;
    for (const auto& stg : pr.sfwd) nio += stg.inputs_only ? stg.end - stg.begin : 0;
    std::fprintf(stderr, "[staged] %zu input loads replaced by direct GEMM reads of the inputs\n", nio);
    std::fprintf(stderr, "[staged] %zu contended-row sums, %u temporary rows; %zu dX products fused with act backward\n",
                 pr.sums.size(), pr.n_tmp, nfx);
    std::fprintf(stderr, "[staged] rows %u, dense %zu (%zu GEMM), %zu batches (%zu with %zu members); %zu generic dests, %zu scatter dests\n",
                 P.n_rows, P.dense.size(), ng, pr.batches.size(), nb, nbm, pr.gen_dests.size(), pr.sc_dests.size());
    stats("fwd", pr.sfwd, P.fwd);
    stats("bwd", pr.sbwd, P.bwd);
    if (v[1] == '2')
      for (int w = 0; w < 2; ++w) {
        const auto& st = w ? pr.sbwd : pr.sfwd;
        const auto& list = w ? P.bwd : P.fwd;
        const auto& key = w ? P.bwd_level : P.fwd_level;
        for (const auto& sg : st) {
          std::map<int, std::size_t> ops;
          for (std::uint32_t k = sg.begin; k < sg.end && sg.batch != kSumStage; ++k)
            ops[list[k].kind == tgc::kNode ? list[k].op : 1000 + list[k].kind]++;
          std::fprintf(stderr, "[staged] %s stage batch %d [%u,%u) key %u:%u members %zu ops", w ? "bwd" : "fwd", sg.batch,
                       sg.begin, sg.end, sg.batch == kSumStage ? 0u : key[sg.begin] >> 12,
                       sg.batch == kSumStage ? 0u : key[sg.begin] & 4095u,
                       sg.batch >= 0 ? pr.batches[sg.batch].members.size() : std::size_t(0));
          for (const auto& [op, c] : ops) std::fprintf(stderr, " %d:%zu", op, c);
          if (sg.batch >= 0) {
            const auto u = pr.batches[sg.batch].members.front();
            std::fprintf(stderr, " | %ux%u w%u act%u dw%u db%u dxact%u skip%d", P.dense[u].n_out, P.dense[u].n_in,
                         P.dense[u].w_uv, P.dense[u].act_op, pr.dplan[u].dw_dest0, pr.dplan[u].db_dest0,
                         pr.batches[sg.batch].dx_act, int(pr.batches[sg.batch].skip_act));
          }
          std::fprintf(stderr, "\n");
        }
      }
  }
}

// The pre-activation rows of a GEMM dense layer are read by nobody when the
// activation's derivative is taken from its output (relu, tanh, exp, sigmoid:
// k_act_bwd and the fused dX epilogue read h): the forward stores h only.
bool z_dead(const tgc::Dense& D) {
  static const bool off = std::getenv("TG_KEEP_Z") && std::getenv("TG_KEEP_Z")[0] == '1';
  const auto a = D.act_op;
  return !off && (a == std::uint32_t(tg::OpKind::Relu) || a == std::uint32_t(tg::OpKind::Tanh) ||
                  a == std::uint32_t(tg::OpKind::Exp) || a == std::uint32_t(tg::OpKind::Sigmoid));
}

// Samples per chunk of the staged path: rows of V and G (plus the reverse
// levels' contended-row temporaries) for the chunk within 64 GB of the B200's
// 180 GB HBM (TG_STAGED_MB overrides), a multiple of 128.  One chunk covers
// cfg4 (b = 8,192: 6.0e5 rows of V and G + 2.7e5 temporaries, 48 GB) and cfg5
// (b = 1M: 39 GB), so every stage runs once per step over the whole batch (a
// 4 GB budget split cfg4 into ten chunks: 36k launches per step).
std::size_t staged_chunk(const tg_program& pr, std::size_t batch) {
  std::size_t budget = std::size_t(64) << 30;
  if (const char* e = std::getenv("TG_STAGED_MB")) budget = std::size_t(std::atoll(e)) << 20;
  if (pr.mem_budget) budget = pr.mem_budget;
  const std::size_t per = (2 * std::max<std::size_t>(1, pr.P.n_rows) + pr.n_tmp) * pr.tsz();
  std::size_t cb = std::max<std::size_t>(128, (budget / per) / 128 * 128);
  const std::size_t need = (std::max<std::size_t>(batch, 1) + 127) / 128 * 128;
  return std::min(cb, need);
}

// CTAs per split-K slice of a dense layer's weight-gradient product: the
// tcgen05 kernel's (CTA pairs of 256 x 256 when n_out > 128) for fp32, the
// SIMT kernel's 64 x 64 tiles for fp64.
std::uint32_t dw_ctas(const tgc::Dense& D, std::size_t tsz) {
  if (tsz == 4) return tgk::umma_ctas_per_slice(D.n_out, D.n_in);
  return ((D.n_out + 63) / 64) * ((D.n_in + 63) / 64);
}

std::uint32_t splitk_splits(const tgc::Dense& D, std::size_t n, std::size_t tsz) {
  const std::uint32_t tiles = dw_ctas(D, tsz);
  std::uint32_t s = std::max<std::uint32_t>(1, 296 / std::max(1u, tiles));
  s = std::min<std::uint32_t>(s, static_cast<std::uint32_t>(std::max<std::size_t>(1, n / 256)));
  return std::max(1u, s);
}

// Split-K slices per member of a batched weight-gradient product: about four
// waves of CTAs over all members, slices of at least 256 samples.
std::uint32_t batch_splits(const tgc::Dense& D, std::uint32_t nm, std::size_t n) {
  const std::uint32_t tiles = dw_ctas(D, 4) * std::max(1u, nm);
  std::uint32_t z = std::max<std::uint32_t>(1, (592 + tiles - 1) / tiles);
  return std::min<std::uint32_t>(z, static_cast<std::uint32_t>(std::max<std::size_t>(1, n / 256)));
}

void choose_config(tg_program& pr) {
  const std::size_t row_bytes = 2 * pr.tsz();
  pr.smem = false;
  for (unsigned S : {256u, 128u, 64u, 32u}) {
    const std::size_t ld = S + 1;
    const std::size_t bytes = std::max<std::size_t>(1, pr.P.n_rows) * ld * row_bytes;
    if (bytes <= kSmemBudget) {
      pr.smem = true;
      pr.S = S;
      pr.ld_smem = ld;
      pr.smem_bytes = bytes;
      break;
    }
  }
  if (!pr.smem) { pr.S = 128; pr.smem_bytes = 0; }
  unsigned bound = std::min(kMaxOcc, 2048u / pr.S);
  if (pr.smem) bound = std::min<unsigned>(bound, static_cast<unsigned>((228 * 1024) / (pr.smem_bytes + 1024)));
  pr.occ_bound = std::max(1u, bound);
  build_staged_plan(pr);
}

std::size_t grid_cap(const tg_program& pr, std::size_t batch) {
  const std::size_t tiles = (batch + pr.S - 1) / pr.S;
  std::size_t cap = std::size_t(148) * pr.occ_bound;
  if (!pr.smem) cap = std::min<std::size_t>(cap, 148 * 8);
  return std::max<std::size_t>(1, std::min(tiles, cap));
}

// Upper bound on CTAs of any tape kernel variant (>= 32 samples per tile,
// <= 32 resident CTAs per SM): sizes the partial-sum rows of the workspace.
std::size_t partial_rows(std::size_t batch) {
  return std::max<std::size_t>(1, std::min<std::size_t>((batch + 31) / 32, std::size_t(148) * 32));
}

std::size_t jit_grid(const tg_program& pr, std::size_t batch) {
  const std::size_t unit = pr.jit.balanced ? 32 : pr.jit.tile;   // balanced: contiguous shares of >= 32 samples
  const std::size_t tiles = (batch + unit - 1) / unit;
  std::size_t g = std::min<std::size_t>(tiles, std::size_t(pr.jit.occ) * pr.nsm);
  return std::max<std::size_t>(1, std::min(g, partial_rows(batch)));
}

std::size_t grid_for(const tg_program& pr, std::size_t batch) {
  std::size_t g = grid_cap(pr, batch);
  if (pr.occ > 0) g = std::min<std::size_t>(g, std::size_t(pr.occ) * pr.nsm);
  return std::max<std::size_t>(1, g);
}

std::size_t align_up(std::size_t x) { return (x + 255) & ~std::size_t(255); }

struct Layout {
  std::size_t done, uv, ug, partial, gv, gg, sk, sp, total;
};
Layout layout(const tg_program& pr, std::size_t batch) {
  const std::size_t t = pr.tsz();
  if (pr.staged) {  // [done | UV | UG | acc[n_dest] | V | G | split-K partials]
    Layout L{};
    std::size_t off = 0;
    const std::size_t cb = staged_chunk(pr, batch);
    L.done = off; off = align_up(off + 16);
    L.uv = off; off = align_up(off + std::max<std::size_t>(1, pr.P.n_uv) * t);
    L.ug = off; off = align_up(off + std::max<std::size_t>(1, pr.P.n_uv) * t);
    L.partial = off; off = align_up(off + std::max<std::uint32_t>(1, pr.n_dest()) * t);
    L.gv = off; off = align_up(off + std::size_t(pr.P.n_rows) * cb * t);
    L.gg = off; off = align_up(off + (std::size_t(pr.P.n_rows) + pr.n_tmp) * cb * t);   // + contended-row temporaries
    std::size_t sk = 0;
    for (std::size_t i = 0; i < pr.P.dense.size(); ++i)
      if (pr.dplan[i].gemm && pr.dplan[i].dw_dest0 != tgc::kNone)
        sk = std::max<std::size_t>(sk, std::size_t(splitk_splits(pr.P.dense[i], cb, t)) *
                                           (std::size_t(pr.P.dense[i].n_out) * pr.P.dense[i].n_in + pr.P.dense[i].n_out));
    for (const auto& B : pr.batches)
      if (B.bw) {
        const tgc::Dense& D = pr.P.dense[B.members.front()];
        const std::uint32_t nm = static_cast<std::uint32_t>(B.members.size());
        sk = std::max<std::size_t>(sk, std::size_t(nm) * batch_splits(D, nm, cb) * (std::size_t(D.n_out) * D.n_in + D.n_out));
      }
    if (pr.fmlp.on)   // the fused kernel's per-CTA gradient partials
      sk = std::max<std::size_t>(sk, std::size_t(tgk::fused_mlp_grid(batch, pr.nsm)) * pr.fmlp.args.nq);
    L.sk = off; off = align_up(off + std::max<std::size_t>(1, sk) * t);
    L.sp = off; off = align_up(off + std::max<std::size_t>(1, std::size_t(pr.sc_groups.size()) * pr.sc_chunks * pr.sc_rmax) * t);
    L.total = off;
    return L;
  }
  const std::size_t grid = grid_cap(pr, batch);
  Layout L{};
  std::size_t off = 0;
  L.done = off; off = align_up(off + 16);
  L.uv = off; off = align_up(off + std::max<std::size_t>(1, pr.P.n_uv) * t);
  L.ug = off; off = align_up(off + std::max<std::size_t>(1, pr.P.n_uv) * t);
  L.partial = off; off = align_up(off + std::max(grid, partial_rows(batch)) * std::max<std::uint32_t>(1, pr.n_dest()) * t);
  L.gv = off;
  if (!pr.smem) off = align_up(off + std::size_t(pr.P.n_rows) * grid * pr.S * t);
  L.gg = off;
  if (!pr.smem) off = align_up(off + std::size_t(pr.P.n_rows) * grid * pr.S * t);
  L.total = off;
  return L;
}

template <class V>
tg_status upload_vec(tg_program& pr, const std::vector<V>& v, V** out) {
  *out = nullptr;
  if (v.empty()) return TG_OK;
  void* p = nullptr;
  TG_CUDA_TRY(cudaMalloc(&p, v.size() * sizeof(V)));
  pr.allocs.push_back(p);
  TG_CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
  *out = static_cast<V*>(p);
  return TG_OK;
}

#define TG_TRY(expr)                          \
  do {                                        \
    tg_status s_ = (expr);                    \
    if (s_ != TG_OK) return s_;               \
  } while (0)

tg_status upload(tg_program& pr) {
  if (pr.uploaded) return TG_OK;
  int dev = 0;
  TG_CUDA_TRY(cudaGetDevice(&dev));
  TG_CUDA_TRY(cudaDeviceGetAttribute(&pr.nsm, cudaDevAttrMultiProcessorCount, dev));
  const tgc::Program& P = pr.P;
  TG_TRY(upload_vec(pr, P.fwd, &pr.d_fwd));
  TG_TRY(upload_vec(pr, P.bwd, &pr.d_bwd));
  TG_TRY(upload_vec(pr, P.ufwd, &pr.d_ufwd));
  TG_TRY(upload_vec(pr, P.ubwd, &pr.d_ubwd));
  TG_TRY(upload_vec(pr, P.opnd, &pr.d_opnd));
  TG_TRY(upload_vec(pr, P.oflag, &pr.d_oflag));
  TG_TRY(upload_vec(pr, P.oaux, &pr.d_oaux));
  TG_TRY(upload_vec(pr, P.zero_rows, &pr.d_zero));
  TG_TRY(upload_vec(pr, P.input_rows, &pr.d_inrows));
  TG_TRY(upload_vec(pr, P.ugather, &pr.d_ug));
  TG_TRY(upload_vec(pr, P.sgather, &pr.d_sg));
  TG_TRY(upload_vec(pr, P.cand, &pr.d_cand));
  if (pr.fmlp.on) TG_TRY(upload_vec(pr, pr.fmlp.dmap, &pr.fmlp.d_dmap));
  TG_TRY(upload_vec(pr, P.term_off, &pr.d_termoff));
  TG_TRY(upload_vec(pr, P.terms, &pr.d_terms));
  TG_TRY(upload_vec(pr, P.dest_uv, &pr.d_destuv));
  TG_TRY(upload_vec(pr, P.dense, &pr.d_dense));
  TG_TRY(upload_vec(pr, P.attn, &pr.d_attn));
  TG_TRY(upload_vec(pr, P.arows, &pr.d_arows));
  TG_TRY(upload_vec(pr, P.lnorm, &pr.d_lnorm));
  TG_TRY(upload_vec(pr, P.lnrows, &pr.d_lnrows));
  TG_TRY(upload_vec(pr, P.lnflag, &pr.d_lnflag));
  const std::uint32_t nc = P.n_uv - P.uv_const_base;
  if (P.dtype == TG_F64) {
    std::vector<double> c(P.uv_init.begin() + P.uv_const_base, P.uv_init.end());
    double* d = nullptr;
    TG_TRY(upload_vec(pr, c, &d));
    pr.d_consts = d;
  } else {
    std::vector<float> c(nc);
    for (std::uint32_t i = 0; i < nc; ++i) c[i] = static_cast<float>(P.uv_init[P.uv_const_base + i]);
    float* d = nullptr;
    TG_TRY(upload_vec(pr, c, &d));
    pr.d_consts = d;
  }
  void* e = nullptr;
  TG_CUDA_TRY(cudaMalloc(&e, 64));
  pr.allocs.push_back(e);
  pr.d_err_key = static_cast<unsigned long long*>(e);
  pr.d_err_val = reinterpret_cast<double*>(static_cast<char*>(e) + 8);
  pr.d_err_op = reinterpret_cast<std::uint32_t*>(static_cast<char*>(e) + 16);
  pr.d_ticket = reinterpret_cast<unsigned*>(static_cast<char*>(e) + 32);
  TG_CUDA_TRY(cudaMemset(e, 0xff, 8));
  TG_CUDA_TRY(cudaMemset(static_cast<char*>(e) + 16, 0xff, 4));
  TG_CUDA_TRY(cudaMemset(static_cast<char*>(e) + 32, 0, 8));   // ticket / grid-barrier count + generation
  if (P.dtype == TG_F64) pr.occ = tgk::tape_occupancy<double>(pr.smem, pr.S, pr.smem_bytes);
  else pr.occ = tgk::tape_occupancy<float>(pr.smem, pr.S, pr.smem_bytes);
  cudaGetLastError();
  const char* env = std::getenv("TG_JIT");
  if (!pr.staged && !(env && env[0] == '0') && tgj::eligible(P)) pr.jit = tgj::build(P);
  if (pr.staged) {
    TG_TRY(upload_vec(pr, pr.gen_dests, &pr.d_gen_dests));
    TG_TRY(upload_vec(pr, pr.sc_groups, &pr.d_sc_groups));
    TG_TRY(upload_vec(pr, pr.sc_uses, &pr.d_sc_uses));
    TG_TRY(upload_vec(pr, pr.sc_use_off, &pr.d_sc_use_off));
    TG_TRY(upload_vec(pr, pr.sc_dests, &pr.d_sc_dests));
    TG_TRY(upload_vec(pr, pr.sums, &pr.d_sums));
    for (auto& B : pr.batches) {
      TG_TRY(upload_vec(pr, B.tab, &B.d_tab));
      TG_TRY(upload_vec(pr, B.zero_x, &B.d_zero_x));
    }
  }
  if (env && env[0] == 'v' && !pr.jit.ok) std::fprintf(stderr, "[tg] JIT not used: %s\n", pr.jit.log.c_str());
  cudaGetLastError();
  pr.uploaded = true;
  return TG_OK;
}

// Dense-layer GEMM: tcgen05 tensor cores for fp32 (3xTF32), SIMT for fp64
// (there is no fp64 tcgen05 kind) or when disabled.
// role bits of the tcgen05 path (TG_UMMA_MASK): 1 forward, 2 input adjoints, 4 weight gradients
bool umma_role(const tg_program& pr, int role) {
  static const int mask = std::getenv("TG_UMMA_MASK") ? std::atoi(std::getenv("TG_UMMA_MASK")) : 7;
  return pr.umma && (mask & role);
}

template <class T>
cudaError_t dense_gemm(const tg_program& pr, const tgk::GemmArgs<T>& g, std::uint32_t splits, cudaStream_t st) {
  if constexpr (std::is_same_v<T, float>) {
    // Roles on tcgen05: bit 0 forward Z = W X, bit 1 input adjoints, bit 2 weight
    // gradients.  Default: all three.  The TMA-fed kernel drains its TMEM
    // accumulator every k-tile into round-to-nearest fp32 sums, which removes
    // the tensor core's accumulation bias (2.6e-7 normwise at any K, below the
    // SIMT GEMM's 5e-7..6.5e-6; scripts/gemm_kerr.py).  With the biased
    // accumulation of round 1 (~6e-6 at K ~ 1e3) the forward role had flipped
    // ReLU masks and moved cfg5's gradient by 5.5e-4, so it had stayed on SIMT.
    const int role = g.epi == tgk::kEpiBiasAct ? 1 : g.epi == tgk::kEpiAccum ? 2 : 4;
    if (umma_role(pr, role)) return tgk::launch_gemm_umma(g, splits, st);
  }
  return tgk::launch_gemm<T>(g, splits, st);
}

bool P_inputs_missing(const tg_program& pr, const void* inputs, const std::int32_t* idx) {
  return (pr.P.n_inputs && !inputs) || (pr.P.n_index_inputs && !idx);
}

// Staged execution: chunks of the batch through HBM-resident rows; dense
// layers as GEMMs, everything else on the interpreter in ranges.
template <class T>
tg_status run_staged(tg_program& pr, const void* inputs, const std::int32_t* idx, std::size_t batch, const void* params,
                     void* loss, void* igrad, void* grad_sum, void* ws, std::size_t ws_bytes, cudaStream_t st,
                     void* gd_params, double gamma) {
  const tgc::Program& P = pr.P;
  const Layout L = layout(pr, batch);
  if (ws_bytes < L.total)
    return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: workspace of " + std::to_string(ws_bytes) +
                                         " bytes, need " + std::to_string(L.total));
  char* w = static_cast<char*>(ws);
  T* UV = reinterpret_cast<T*>(w + L.uv);
  T* UG = reinterpret_cast<T*>(w + L.ug);
  T* acc = reinterpret_cast<T*>(w + L.partial);
  T* V = reinterpret_cast<T*>(w + L.gv);
  T* G = reinterpret_cast<T*>(w + L.gg);
  T* sk = reinterpret_cast<T*>(w + L.sk);
  const std::size_t cb = staged_chunk(pr, batch);

  tgk::UniformArgs<T> ua{};
  ua.instr = pr.d_ufwd;
  ua.opnd = pr.d_opnd;
  ua.params = static_cast<const T*>(params);
  ua.consts = static_cast<const T*>(pr.d_consts);
  ua.UV = UV;
  ua.UG = UG;
  ua.grad_sum = static_cast<T*>(grad_sum);
  ua.err_key = pr.d_err_key;
  ua.err_val = pr.d_err_val;
  ua.err_op = pr.d_err_op;
  ua.batch = batch;
  ua.n_instr = static_cast<std::uint32_t>(P.ufwd.size());
  ua.n_params = P.n_params;
  ua.n_const = P.n_uv - P.uv_const_base;
  ua.const_base = P.uv_const_base;
  ua.n_uv = P.n_uv;
  ua.root_uv = P.root_uv;
  ua.done = reinterpret_cast<unsigned*>(w + L.done);
  TG_CUDA_TRY(tgk::launch_uniform_fwd<T>(ua, st, pr.launches));
  TG_CUDA_TRY(cudaMemsetAsync(acc, 0, std::max<std::uint32_t>(1, pr.n_dest()) * sizeof(T), st));

  tgk::RangeArgs<T> ra{};
  ra.fwd = pr.d_fwd;
  ra.bwd = pr.d_bwd;
  ra.opnd = pr.d_opnd;
  ra.oflag = pr.d_oflag;
  ra.oaux = pr.d_oaux;
  ra.zero_rows = pr.d_zero;
  ra.input_rows = pr.d_inrows;
  ra.ug = pr.d_ug;
  ra.sg = pr.d_sg;
  ra.cand = pr.d_cand;
  ra.dense = pr.d_dense;
  ra.attn = pr.d_attn;
  ra.arows = pr.d_arows;
  ra.lnorm = pr.d_lnorm;
  ra.lnrows = pr.d_lnrows;
  ra.lnflag = pr.d_lnflag;
  ra.UV = UV;
  ra.inputs = static_cast<const T*>(inputs);
  ra.idx = idx;
  ra.loss = static_cast<T*>(loss);
  ra.igrad = static_cast<T*>(igrad);
  ra.V = V;
  ra.G = G;
  ra.err_key = pr.d_err_key;
  ra.batch = batch;
  ra.ld = cb;
  ra.n_zero = static_cast<std::uint32_t>(P.zero_rows.size());
  ra.n_inputs = P.n_inputs;
  ra.root_row = P.root_row;

  // Interpreter arguments for domain-error diagnosis (k_tape re-runs the one
  // offending sample; the staged V / G buffers serve as its row storage).
  {
    tgk::MainArgs<T> ma{};
    ma.fwd = pr.d_fwd;
    ma.bwd = pr.d_bwd;
    ma.opnd = pr.d_opnd;
    ma.oflag = pr.d_oflag;
    ma.oaux = pr.d_oaux;
    ma.zero_rows = pr.d_zero;
    ma.input_rows = pr.d_inrows;
    ma.ug = pr.d_ug;
    ma.sg = pr.d_sg;
    ma.cand = pr.d_cand;
    ma.term_off = pr.d_termoff;
    ma.terms = pr.d_terms;
    ma.dense = pr.d_dense;
    ma.attn = pr.d_attn;
    ma.arows = pr.d_arows;
    ma.lnorm = pr.d_lnorm;
    ma.lnrows = pr.d_lnrows;
    ma.lnflag = pr.d_lnflag;
    ma.UV = UV;
    ma.inputs = static_cast<const T*>(inputs);
    ma.idx = idx;
    ma.partial = acc;
    ma.gV = V;
    ma.gG = G;
    ma.err_key = pr.d_err_key;
    ma.err_val = pr.d_err_val;
    ma.err_op = pr.d_err_op;
    ma.batch = batch;
    ma.ld = pr.smem ? pr.ld_smem : cb;
    ma.diag_sample = -1;
    ma.n_fwd = static_cast<std::uint32_t>(P.fwd.size());
    ma.n_bwd = static_cast<std::uint32_t>(P.bwd.size());
    ma.n_zero = static_cast<std::uint32_t>(P.zero_rows.size());
    ma.n_inputs = P.n_inputs;
    ma.n_dest = 0;
    ma.n_rows = P.n_rows;
    ma.S = pr.S;
    ma.root_row = P.root_row;
    pr.last_args.assign(reinterpret_cast<unsigned char*>(&ma), reinterpret_cast<unsigned char*>(&ma) + sizeof(ma));
    pr.have_last = true;
  }
  cudaEvent_t e1 = nullptr;   // tg_profile_enable: time the staged chain
  if (pr.profiling) {
    if (pr.ev_used == pr.ev.size()) {
      cudaEvent_t a0, b0;
      TG_CUDA_TRY(cudaEventCreate(&a0));
      TG_CUDA_TRY(cudaEventCreate(&b0));
      pr.ev.emplace_back(a0, b0);
    }
    TG_CUDA_TRY(cudaEventRecord(pr.ev[pr.ev_used].first, st));
    e1 = pr.ev[pr.ev_used].second;
    ++pr.ev_used;
  }

  // tensor-core roles (TG_UMMA_MASK bits: 1 forward, 2 input adjoints, 4 weight gradients)
  static const int umask = std::getenv("TG_UMMA_MASK") ? std::atoi(std::getenv("TG_UMMA_MASK")) : 7;
  // dense layers over input leaves read inputs[col][s] in place (TMA: 16-byte rows)
  const bool direct_x = (umask & 5) == 5 && batch % 4 == 0 && inputs &&
                        (reinterpret_cast<std::uintptr_t>(inputs) & 15) == 0;
  auto x_ptr = [&](const tg_program::DensePlan& dp, const T* Vb, std::size_t s0, std::size_t& ld) -> const T* {
    if (direct_x && dp.x_col0 != tgc::kNone) {
      ld = batch;
      return static_cast<const T*>(inputs) + std::size_t(dp.x_col0) * batch + s0;
    }
    ld = cb;
    return Vb + std::size_t(dp.xrow0) * cb;
  };
  if constexpr (std::is_same_v<T, float>) {
    if (pr.fmlp.on) {   // the whole tape in one kernel, no HBM rows
      tgk::FusedMlpArgs fa = pr.fmlp.args;
      fa.UV = UV;
      fa.idx = idx;
      fa.batch = batch;
      fa.loss = static_cast<float*>(loss);
      fa.part = sk;
      const unsigned grid = tgk::fused_mlp_grid(batch, pr.nsm);
      TG_CUDA_TRY(tgk::launch_fused_mlp(fa, grid, pr.fmlp.d_dmap, acc, st));
      pr.launches += 2;
    }
  }
  for (std::size_t s0 = 0; s0 < batch && !pr.fmlp.on; s0 += cb) {
    const std::size_t n = std::min(cb, batch - s0);
    ra.s0 = s0;
    ra.n = n;
    // Z[n_out][n] = W[n_out][n_in] . X[n_in][n] + b (one member)
    auto fwd_one = [&](std::uint32_t u) -> cudaError_t {
      const tgc::Dense& D = P.dense[u];
      tgk::GemmArgs<T> g{};
      g.A = UV + D.w_uv;
      g.lda = D.n_in;
      g.a_kmaj = true;
      g.B = x_ptr(pr.dplan[u], V, s0, g.ldb);
      g.b_nmaj = true;
      g.C = V + std::size_t(D.out_row) * cb;
      g.C2 = D.act_op ? V + std::size_t(D.act_row) * cb : nullptr;
      g.no_z = z_dead(D);
      g.ldc = cb;
      g.bias = D.b_uv != tgc::kNone ? UV + D.b_uv : nullptr;
      g.M = D.n_out;
      g.N = static_cast<std::uint32_t>(n);
      g.K = D.n_in;
      g.act = D.act_op;
      g.epi = tgk::kEpiBiasAct;
      ++pr.launches;
      return dense_gemm<T>(pr, g, 1, st);
    };
    // dX[n_in][n] (+)= W^T[n_in][n_out] . dZ[n_out][n] (one member)
    // (dact: C = the producing layer's z rows c_row, act' from its h rows = x rows)
    auto dx_one = [&](std::uint32_t u, int beta, std::uint32_t dact, std::uint32_t c_row) -> cudaError_t {
      const tgc::Dense& D = P.dense[u];
      tgk::GemmArgs<T> g{};
      g.A = UV + D.w_uv;
      g.lda = D.n_in;
      g.a_kmaj = false;
      g.B = G + std::size_t(D.out_row) * cb;
      g.ldb = cb;
      g.b_nmaj = true;
      g.C = G + std::size_t(dact ? c_row : pr.dplan[u].xrow0) * cb;
      g.dact = dact;
      g.C2 = dact ? V + std::size_t(pr.dplan[u].xrow0) * cb : nullptr;
      g.ldc = cb;
      g.M = D.n_in;
      g.N = static_cast<std::uint32_t>(n);
      g.K = D.n_out;
      g.beta = beta;
      g.epi = tgk::kEpiAccum;
      ++pr.launches;
      return dense_gemm<T>(pr, g, 1, st);
    };
    // dW[n_out][n_in] += dZ[n_out][n] . X^T, split-K over samples (one member)
    bool db_fused_u = false;   // the last dw_one also produced its layer's bias gradient
    auto dw_one = [&](std::uint32_t u, bool fuse_db) -> cudaError_t {
      db_fused_u = false;
      const tgc::Dense& D = P.dense[u];
      const std::uint32_t splits = splitk_splits(D, n, sizeof(T));
      tgk::GemmArgs<T> g{};
      g.A = G + std::size_t(D.out_row) * cb;
      g.lda = cb;
      g.a_kmaj = true;
      g.B = x_ptr(pr.dplan[u], V, s0, g.ldb);
      g.b_nmaj = false;
      g.C = sk;
      g.M = D.n_out;
      g.N = D.n_in;
      g.K = static_cast<std::uint32_t>(n);
      g.k_chunk = static_cast<std::uint32_t>((n + splits - 1) / splits);
      g.epi = tgk::kEpiSplitK;
      pr.launches += 2;
      // the bias gradient (row sums of dz) rides in the CTA-pair product's converters
      bool rs = false;
      if constexpr (std::is_same_v<T, float>) {
        rs = fuse_db && pr.dplan[u].db_dest0 != tgc::kNone && umma_role(pr, 4) && tgk::umma_rowsum_fusable(g);
        if (rs) g.rowsum = sk + std::size_t(splits) * D.n_out * D.n_in;
      }
      cudaError_t e = dense_gemm<T>(pr, g, splits, st);
      if (e == cudaSuccess) e = tgk::launch_splitk_reduce<T>(sk, acc + pr.dplan[u].dw_dest0, D.n_out * D.n_in, splits, st);
      if (e == cudaSuccess && rs) {
        e = tgk::launch_splitk_reduce<T>(g.rowsum, acc + pr.dplan[u].db_dest0, D.n_out, splits, st);
        ++pr.launches;
        db_fused_u = true;
      }
      return e;
    };
    // ---- forward stages ----
    // fused attention heads: the shared-memory kernels (fp32, small heads) or,
    // otherwise, one interpreter CTA row per head (attn_*_sample)
    auto attn_stage = [&](const tg_program::Stage& stg, bool fwd) -> cudaError_t {
      ++pr.launches;
      if constexpr (std::is_same_v<T, float>) {
        if (pr.attn_fast)
          return tgk::launch_attn(fwd, fwd ? pr.d_fwd : pr.d_bwd, stg.begin, stg.end - stg.begin, pr.d_attn, pr.d_arows,
                                  V, G, n, cb, pr.attn_hd, st);
      }
      ra.flags = fwd ? tgk::kRFwd : tgk::kRBwd;
      (fwd ? ra.fwd_begin : ra.bwd_begin) = stg.begin;
      (fwd ? ra.fwd_end : ra.bwd_end) = stg.end;
      return tgk::launch_level_range<T>(ra, st);
    };
    for (const auto& stg : pr.sfwd) {
      if (stg.batch == kAttnStage) { TG_CUDA_TRY(attn_stage(stg, true)); continue; }
      if (stg.batch < 0 && stg.inputs_only && direct_x) continue;   // rows read in place by their GEMMs
      if (stg.batch < 0) {
        ra.flags = tgk::kRFwd;
        ra.fwd_begin = stg.begin;
        ra.fwd_end = stg.end;
        ra.per_sample = stg.macro ? 1 : 0;
        TG_CUDA_TRY(stg.level ? tgk::launch_level_range<T>(ra, st) : tgk::launch_tape_range<T>(ra, st));
        ++pr.launches;
        continue;
      }
      const auto& B = pr.batches[stg.batch];
      const std::uint32_t nm = static_cast<std::uint32_t>(B.members.size());
      if constexpr (std::is_same_v<T, float>) {
        if (B.bf && (umask & 1)) {
          const tgc::Dense& D = P.dense[B.members.front()];
          tgk::GemmArgs<float> g{};
          g.A = UV + D.w_uv;
          g.lda = D.n_in;
          g.a_kmaj = true;
          g.B = V;
          g.ldb = cb;
          g.b_nmaj = true;
          g.b_span = P.n_rows;
          g.C = V;
          g.C2 = D.act_op ? V : nullptr;
          g.no_z = z_dead(D);
          g.ldc = cb;
          g.bias = D.b_uv != tgc::kNone ? UV + D.b_uv : nullptr;
          g.M = D.n_out;
          g.N = static_cast<std::uint32_t>(n);
          g.K = D.n_in;
          g.act = D.act_op;
          g.epi = tgk::kEpiBiasAct;
          g.mem = B.d_tab;
          g.zs = 1;
          TG_CUDA_TRY(tgk::launch_gemm_umma(g, nm, st));
          ++pr.launches;
          continue;
        }
      }
      for (std::uint32_t u : B.members) TG_CUDA_TRY(fwd_one(u));
    }
    ra.flags = tgk::kRSeed;
    TG_CUDA_TRY(tgk::launch_tape_range<T>(ra, st));
    ++pr.launches;
    // ---- reverse stages ----
    for (const auto& stg : pr.sbwd) {
      if (stg.batch == kAttnStage) { TG_CUDA_TRY(attn_stage(stg, false)); continue; }
      if (stg.batch == kSumStage) {
        TG_CUDA_TRY(tgk::launch_row_sums<T>(pr.d_sums + stg.begin, stg.end - stg.begin, G, n, cb, st));
        ++pr.launches;
        continue;
      }
      if (stg.batch < 0) {
        ra.flags = tgk::kRBwd;
        ra.bwd_begin = stg.begin;
        ra.bwd_end = stg.end;
        ra.per_sample = stg.macro ? 1 : 0;
        TG_CUDA_TRY(stg.level ? tgk::launch_level_range<T>(ra, st) : tgk::launch_tape_range<T>(ra, st));
        ++pr.launches;
        continue;
      }
      const auto& B = pr.batches[stg.batch];
      const std::uint32_t nm = static_cast<std::uint32_t>(B.members.size());
      const tgc::Dense& D = P.dense[B.members.front()];
      const auto& dp0 = pr.dplan[B.members.front()];
      if (D.act_op && !B.skip_act) {
        TG_CUDA_TRY(tgk::launch_act_bwd_batched<T>(G, V, B.d_tab, nm, D.n_out, n, cb, D.act_op, st));
        ++pr.launches;
      }
      // input-leaf x rows: their adjoints are read only by the input-gradient output
      bool dx_done = !igrad && B.x_inputs;
      bool dw_done = false, db_done = false;
      if (!dx_done && !B.zero_x.empty()) {
        TG_CUDA_TRY(tgk::launch_zero_rows<T>(G, B.d_zero_x, static_cast<std::uint32_t>(B.zero_x.size()), n, cb, st));
        ++pr.launches;
      }
      if constexpr (std::is_same_v<T, float>) {
        if (!dx_done && B.bx && (umask & 2)) {
          tgk::GemmArgs<float> g{};
          g.A = UV + D.w_uv;
          g.lda = D.n_in;
          g.a_kmaj = false;
          g.B = G;
          g.ldb = cb;
          g.b_nmaj = true;
          g.b_span = P.n_rows;
          g.C = G;
          g.ldc = cb;
          g.M = D.n_in;
          g.N = static_cast<std::uint32_t>(n);
          g.K = D.n_out;
          g.beta = B.beta;
          g.dact = B.dx_act;
          g.C2 = B.dx_act ? V : nullptr;
          g.epi = tgk::kEpiAccum;
          g.mem = B.d_tab + nm;
          g.zs = 1;
          TG_CUDA_TRY(tgk::launch_gemm_umma(g, nm, st));
          ++pr.launches;
          dx_done = true;
        }
        if (B.bw && (umask & 4)) {
          const std::uint32_t zs = batch_splits(D, nm, n);
          tgk::GemmArgs<float> g{};
          g.A = G;
          g.lda = cb;
          g.a_kmaj = true;
          g.a_span = P.n_rows;
          g.B = V;
          g.ldb = cb;
          g.b_nmaj = false;
          g.b_span = P.n_rows;
          g.C = sk;
          g.M = D.n_out;
          g.N = D.n_in;
          g.K = static_cast<std::uint32_t>(n);
          g.k_chunk = static_cast<std::uint32_t>((n + zs - 1) / zs);
          g.epi = tgk::kEpiSplitK;
          g.mem = B.d_tab + 2 * nm;
          g.zs = zs;
          // the bias gradient (row sums of dz) rides in the product's converters
          const bool rs = dp0.db_dest0 != tgc::kNone && tgk::umma_rowsum_fusable(g);
          if (rs) g.rowsum = sk + std::size_t(nm) * zs * D.n_out * D.n_in;
          TG_CUDA_TRY(tgk::launch_gemm_umma(g, nm * zs, st));
          TG_CUDA_TRY(tgk::launch_splitk_reduce<T>(sk, acc + dp0.dw_dest0, D.n_out * D.n_in, nm * zs, st));
          pr.launches += 2;
          if (rs) {
            TG_CUDA_TRY(tgk::launch_splitk_reduce<T>(g.rowsum, acc + dp0.db_dest0, D.n_out, nm * zs, st));
            ++pr.launches;
            db_done = true;
          }
          dw_done = true;
        }
      }
      for (std::uint32_t p = 0; p < nm; ++p) {
        const std::uint32_t u = B.members[p];
        // zeroed rows above follow the batch's beta; members that only assign keep their store
        if (!dx_done) TG_CUDA_TRY(dx_one(u, B.beta ? pr.dplan[u].beta : 0, B.dx_act, B.tab[nm + p].z));
        if (!dw_done && pr.dplan[u].dw_dest0 != tgc::kNone) {
          TG_CUDA_TRY(dw_one(u, nm == 1));
          if (db_fused_u) db_done = true;
        }
      }
      if (dp0.db_dest0 != tgc::kNone && !db_done) {
        TG_CUDA_TRY(tgk::launch_rowsum_batched<T>(G, B.d_tab, nm, D.n_out, n, cb, acc + dp0.db_dest0, sk,
                                                  (L.sp - L.sk) / sizeof(T), st));   // split-K scratch, free here
        ++pr.launches;
      }
    }
    if (igrad) {
      ra.flags = tgk::kROut;
      TG_CUDA_TRY(tgk::launch_tape_range<T>(ra, st));
      ++pr.launches;
    }
    if (!pr.gen_dests.empty()) {
      TG_CUDA_TRY(tgk::launch_contract<T>(pr.d_gen_dests, static_cast<std::uint32_t>(pr.gen_dests.size()), pr.d_termoff,
                                          pr.d_terms, G, V, idx, batch, s0, n, cb, acc, st));
      ++pr.launches;
    }
    if (!pr.sc_groups.empty()) {
      TG_CUDA_TRY(tgk::launch_scatter<T>(pr.d_sc_groups, static_cast<std::uint32_t>(pr.sc_groups.size()), pr.sc_rmax,
                                         pr.d_sc_uses, pr.d_sc_use_off, pr.d_sc_dests,
                                         static_cast<std::uint32_t>(pr.sc_dests.size()), G, idx, batch, s0, n, cb,
                                         reinterpret_cast<T*>(w + L.sp), pr.sc_chunks, acc, st));
      pr.launches += 2;
    }
  }
  if (e1) TG_CUDA_TRY(cudaEventRecord(e1, st));
  // fused: acc -> UG -> uniform reverse sweep -> grad_sum (-> GD)
  tgk::ReduceArgs<T> rd{acc, pr.d_destuv, pr.n_dest(), 1};
  ua.instr = pr.d_ubwd;
  ua.n_instr = static_cast<std::uint32_t>(P.ubwd.size());
  if (gd_params) {
    ua.gd_params = static_cast<T*>(gd_params);
    ua.gamma = static_cast<T>(gamma);
    ua.gd_batch = static_cast<T>(static_cast<double>(batch));
  }
  TG_CUDA_TRY(tgk::launch_reduce_epilogue<T>(rd, ua, st, pr.launches));
  return TG_OK;
}

// Launch with programmatic stream serialisation: the kernel may be scheduled
// while its stream predecessor drains; it waits (griddepcontrol.wait) before
// its first dependent read.
cudaError_t launch_pdl(cudaKernel_t fn, unsigned grid, unsigned block, std::size_t smem, void** args, cudaStream_t st,
                       bool cooperative = false) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(block);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  static const bool pdl = !(std::getenv("TG_PDL") && std::getenv("TG_PDL")[0] == '0');
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cooperative) {   // grid barriers inside the kernel: every CTA must be resident
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  lc.attrs = at;
  lc.numAttrs = n;
  return cudaLaunchKernelExC(&lc, reinterpret_cast<const void*>(fn), args);
}

// One step as two launches of the program's module: tg_jit_tape (uniform
// prologue per CTA + per-sample sweeps + per-CTA partials) and tg_jit_epi
// (fixed-order reduction, uniform reverse sweep, grad_sum, GD).
template <class T>
tg_status run_fused(tg_program& pr, const void* inputs, const std::int32_t* idx, std::size_t batch, const void* params,
                    void* loss, void* igrad, void* grad_sum, T* UV, T* UG, T* partial, char* w, const Layout& L,
                    cudaStream_t st, void* gd_params, double gamma) {
  tgj::JitArgs<T> ja{};
  const std::size_t rows = jit_grid(pr, batch);
  ja.in = static_cast<const T*>(inputs);
  ja.idx = idx;
  ja.batch = batch;
  ja.loss = static_cast<T*>(loss);
  ja.igrad = static_cast<T*>(igrad);
  ja.partial = partial;
  ja.grid_rows = static_cast<unsigned>(rows);
  ja.err_key = pr.d_err_key;
  ja.err_val = pr.d_err_val;
  ja.err_op = pr.d_err_op;
  ja.UVg = UV;
  ja.cand = pr.d_cand;
  ja.toff = static_cast<const unsigned*>(pr.jit.d_toff);
  ja.terms = pr.jit.d_terms;
  ja.params = static_cast<const T*>(params);
  ja.consts = static_cast<const T*>(pr.d_consts);
  ja.UVw = UV;
  ja.tickets = pr.jit.coop ? pr.d_ticket : reinterpret_cast<unsigned*>(w + L.done);   // see tg_jit.cpp fuse_wait
  ja.partial2 = UG;
  ja.grad_sum = static_cast<T*>(grad_sum);
  ja.gd_params = static_cast<T*>(gd_params);
  ja.gamma = static_cast<T>(gamma);
  ja.gd_batch = static_cast<T>(static_cast<double>(batch));
  void* args[] = {&ja};
  cudaEvent_t e1 = nullptr;
  if (pr.profiling) {
    if (pr.ev_used == pr.ev.size()) {
      cudaEvent_t a, b;
      TG_CUDA_TRY(cudaEventCreate(&a));
      TG_CUDA_TRY(cudaEventCreate(&b));
      pr.ev.emplace_back(a, b);
    }
    TG_CUDA_TRY(cudaEventRecord(pr.ev[pr.ev_used].first, st));
    e1 = pr.ev[pr.ev_used].second;
    ++pr.ev_used;
  }
  TG_CUDA_TRY(launch_pdl(pr.jit.fn, ja.grid_rows, pr.jit.cfg.block, pr.jit.smem_bytes, args, st, pr.jit.coop));
  if (e1) TG_CUDA_TRY(cudaEventRecord(e1, st));
  const unsigned nd = pr.n_dest();
  ++pr.launches;
  // the cooperative kernel runs the epilogue itself; programs with nothing to
  // reduce or propagate (cfg1) need none
  if (!pr.jit.coop && (nd > 0 || !pr.P.ubwd.empty())) {
    TG_CUDA_TRY(launch_pdl(pr.jit.fn_epi, std::max(1u, (nd + 7) / 8), 256, 0, args, st));
    ++pr.launches;
  }
  // diagnosis of a domain error re-runs the interpreter on this launch's inputs
  tgk::MainArgs<T> ma{};
  ma.fwd = pr.d_fwd;
  ma.bwd = pr.d_bwd;
  ma.opnd = pr.d_opnd;
  ma.oflag = pr.d_oflag;
  ma.oaux = pr.d_oaux;
  ma.zero_rows = pr.d_zero;
  ma.input_rows = pr.d_inrows;
  ma.ug = pr.d_ug;
  ma.sg = pr.d_sg;
  ma.cand = pr.d_cand;
  ma.term_off = pr.d_termoff;
  ma.terms = pr.d_terms;
  ma.dense = pr.d_dense;
  ma.attn = pr.d_attn;
  ma.arows = pr.d_arows;
  ma.lnorm = pr.d_lnorm;
  ma.lnrows = pr.d_lnrows;
  ma.lnflag = pr.d_lnflag;
  ma.UV = UV;
  ma.inputs = static_cast<const T*>(inputs);
  ma.idx = idx;
  ma.partial = partial;
  ma.gV = reinterpret_cast<T*>(w + L.gv);
  ma.gG = reinterpret_cast<T*>(w + L.gg);
  ma.err_key = pr.d_err_key;
  ma.err_val = pr.d_err_val;
  ma.err_op = pr.d_err_op;
  ma.batch = batch;
  ma.ld = pr.smem ? pr.ld_smem : grid_for(pr, batch) * pr.S;
  ma.diag_sample = -1;
  ma.n_fwd = static_cast<std::uint32_t>(pr.P.fwd.size());
  ma.n_bwd = static_cast<std::uint32_t>(pr.P.bwd.size());
  ma.n_zero = static_cast<std::uint32_t>(pr.P.zero_rows.size());
  ma.n_inputs = pr.P.n_inputs;
  ma.n_dest = pr.n_dest();
  ma.n_rows = pr.P.n_rows;
  ma.S = pr.S;
  ma.root_row = pr.P.root_row;
  pr.last_args.assign(reinterpret_cast<unsigned char*>(&ma), reinterpret_cast<unsigned char*>(&ma) + sizeof(ma));
  pr.have_last = true;
  pr.last_batch = batch;
  return TG_OK;
}

template <class T>
tg_status run_fb(tg_program& pr, const void* inputs, const std::int32_t* idx, std::size_t batch, const void* params,
                 void* loss, void* igrad, void* grad_sum, void* ws, std::size_t ws_bytes, cudaStream_t st,
                 void* gd_params = nullptr, double gamma = 0.0) {
  TG_TRY(upload(pr));
  if (pr.staged) {
    if (batch > 0 && P_inputs_missing(pr, inputs, idx)) return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: inputs are NULL");
    return run_staged<T>(pr, inputs, idx, batch, params, loss, igrad, grad_sum, ws, ws_bytes, st, gd_params, gamma);
  }
  const tgc::Program& P = pr.P;
  const Layout L = layout(pr, batch);
  if (ws_bytes < L.total)
    return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: workspace of " + std::to_string(ws_bytes) +
                                         " bytes, need " + std::to_string(L.total));
  if (batch > 0 && P.n_inputs && !inputs) return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: inputs is NULL");
  if (batch > 0 && P.n_index_inputs && !idx) return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: index_inputs is NULL");
  if (P.n_params && !params) return fail(TG_INVALID_ARGUMENT, "tg_forward_backward: params is NULL");
  char* w = static_cast<char*>(ws);
  T* UV = reinterpret_cast<T*>(w + L.uv);
  T* UG = reinterpret_cast<T*>(w + L.ug);
  T* partial = reinterpret_cast<T*>(w + L.partial);

  if (pr.jit.ok && pr.jit.fused && batch > 0)
    return run_fused<T>(pr, inputs, idx, batch, params, loss, igrad, grad_sum, UV, UG, partial, w, L, st, gd_params, gamma);
  tgk::UniformArgs<T> ua{};
  ua.instr = pr.d_ufwd;
  ua.opnd = pr.d_opnd;
  ua.params = static_cast<const T*>(params);
  ua.consts = static_cast<const T*>(pr.d_consts);
  ua.UV = UV;
  ua.UVc = pr.jit.ok ? static_cast<T*>(pr.jit.cuv) : nullptr;
  ua.UG = UG;
  ua.grad_sum = static_cast<T*>(grad_sum);
  ua.err_key = pr.d_err_key;
  ua.err_val = pr.d_err_val;
  ua.err_op = pr.d_err_op;
  ua.batch = batch;
  ua.n_instr = static_cast<std::uint32_t>(P.ufwd.size());
  ua.n_params = P.n_params;
  ua.n_const = P.n_uv - P.uv_const_base;
  ua.const_base = P.uv_const_base;
  ua.n_uv = P.n_uv;
  ua.root_uv = P.root_uv;
  ua.done = reinterpret_cast<unsigned*>(w + L.done);
  TG_CUDA_TRY(tgk::launch_uniform_fwd<T>(ua, st, pr.launches));
  tgk::ReduceArgs<T> ra{partial, pr.d_destuv, 0, 1};

  const std::size_t grid = grid_for(pr, batch);
  if (batch > 0 && P.root_row != tgc::kNone) {
    tgk::MainArgs<T> ma{};
    ma.fwd = pr.d_fwd;
    ma.bwd = pr.d_bwd;
    ma.opnd = pr.d_opnd;
    ma.oflag = pr.d_oflag;
    ma.oaux = pr.d_oaux;
    ma.zero_rows = pr.d_zero;
    ma.input_rows = pr.d_inrows;
    ma.ug = pr.d_ug;
    ma.sg = pr.d_sg;
    ma.cand = pr.d_cand;
    ma.term_off = pr.d_termoff;
    ma.terms = pr.d_terms;
    ma.dense = pr.d_dense;
    ma.attn = pr.d_attn;
    ma.arows = pr.d_arows;
    ma.lnorm = pr.d_lnorm;
    ma.lnrows = pr.d_lnrows;
    ma.lnflag = pr.d_lnflag;
    ma.UV = UV;
    ma.inputs = static_cast<const T*>(inputs);
    ma.idx = idx;
    ma.loss = static_cast<T*>(loss);
    ma.igrad = static_cast<T*>(igrad);
    ma.partial = partial;
    ma.gV = reinterpret_cast<T*>(w + L.gv);
    ma.gG = reinterpret_cast<T*>(w + L.gg);
    ma.err_key = pr.d_err_key;
    ma.err_val = pr.d_err_val;
    ma.err_op = pr.d_err_op;
    ma.batch = batch;
    ma.ld = pr.smem ? pr.ld_smem : grid * pr.S;
    ma.diag_sample = -1;
    ma.n_fwd = static_cast<std::uint32_t>(P.fwd.size());
    ma.n_bwd = static_cast<std::uint32_t>(P.bwd.size());
    ma.n_zero = static_cast<std::uint32_t>(P.zero_rows.size());
    ma.n_inputs = P.n_inputs;
    ma.n_dest = pr.n_dest();
    ma.n_rows = P.n_rows;
    ma.S = pr.S;
    ma.root_row = P.root_row;
    cudaEvent_t e1 = nullptr;
    if (pr.profiling) {
      if (pr.ev_used == pr.ev.size()) {
        cudaEvent_t a, b;
        TG_CUDA_TRY(cudaEventCreate(&a));
        TG_CUDA_TRY(cudaEventCreate(&b));
        pr.ev.emplace_back(a, b);
      }
      TG_CUDA_TRY(cudaEventRecord(pr.ev[pr.ev_used].first, st));
      e1 = pr.ev[pr.ev_used].second;
      ++pr.ev_used;
    }
    std::size_t rows = grid;
    if (pr.jit.ok) {
      rows = jit_grid(pr, batch);
      tgj::JitArgs<T> ja{};
      ja.in = ma.inputs;
      ja.idx = ma.idx;
      ja.batch = batch;
      ja.loss = ma.loss;
      ja.igrad = ma.igrad;
      ja.partial = ma.partial;
      ja.grid_rows = static_cast<unsigned>(rows);
      ja.err_key = ma.err_key;
      ja.err_val = ma.err_val;
      ja.err_op = ma.err_op;
      ja.UVg = UV;
      ja.cand = ma.cand;
      ja.toff = static_cast<const unsigned*>(pr.jit.d_toff);
      ja.terms = pr.jit.d_terms;
      void* args[] = {&ja};
      TG_CUDA_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(pr.jit.fn), dim3(ja.grid_rows), dim3(pr.jit.cfg.block),
                                   args, pr.jit.smem_bytes, st));
    } else {
      TG_CUDA_TRY(tgk::launch_tape<T>(ma, pr.smem, static_cast<unsigned>(grid), pr.S, pr.smem_bytes, st));
    }
    if (e1) TG_CUDA_TRY(cudaEventRecord(e1, st));
    ++pr.launches;
    pr.last_args.assign(reinterpret_cast<unsigned char*>(&ma), reinterpret_cast<unsigned char*>(&ma) + sizeof(ma));
    pr.have_last = true;
    pr.last_batch = batch;

    ra = tgk::ReduceArgs<T>{partial, pr.d_destuv, pr.n_dest(), static_cast<std::uint32_t>(rows)};
  }
  // fused: per-CTA partial reduction -> uniform reverse sweep -> grad_sum (-> GD)
  ua.instr = pr.d_ubwd;
  ua.n_instr = static_cast<std::uint32_t>(P.ubwd.size());
  if (gd_params) {
    ua.gd_params = static_cast<T*>(gd_params);
    ua.gamma = static_cast<T>(gamma);
    ua.gd_batch = static_cast<T>(static_cast<double>(batch));
  }
  TG_CUDA_TRY(tgk::launch_reduce_epilogue<T>(ra, ua, st, pr.launches));
  return TG_OK;
}

template <class T>
tg_status diagnose(tg_program& pr, std::int64_t sample, cudaStream_t st) {
  if (!pr.have_last) return TG_OK;
  tgk::MainArgs<T> ma;
  std::memcpy(&ma, pr.last_args.data(), sizeof(ma));
  ma.diag_sample = sample;
  ma.loss = nullptr;
  ma.igrad = nullptr;
  // domain violations happen in the forward sweep; the reverse sweep of a
  // staged program also writes temporaries beyond the interpreter's rows
  ma.n_bwd = 0;
  TG_CUDA_TRY(tgk::launch_tape<T>(ma, pr.smem, 1, pr.S, pr.smem_bytes, st));
  ++pr.launches;
  return TG_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* tg_last_error(void) { return g_err.c_str(); }

const char* tg_status_name(tg_status s) {
  switch (s) {
    case TG_OK: return "TG_OK";
    case TG_INVALID_ARGUMENT: return "TG_INVALID_ARGUMENT";
    case TG_CAPACITY: return "TG_CAPACITY";
    case TG_INVALID_HANDLE: return "TG_INVALID_HANDLE";
    case TG_INVALID_CHECKPOINT: return "TG_INVALID_CHECKPOINT";
    case TG_DOMAIN: return "TG_DOMAIN";
    case TG_FORMAT: return "TG_FORMAT";
    case TG_IO: return "TG_IO";
    case TG_CUDA: return "TG_CUDA";
    case TG_UNSUPPORTED: return "TG_UNSUPPORTED";
    case TG_NCCL: return "TG_NCCL";
  }
  return "?";
}

const char* tg_op_name(uint8_t op) {
  static const char* const names[] = {
      "leaf", "relu", "tanh", "exp", "negativeLog", "sigmoid", "inv", "sqr", "pow3", "logarithm",
      "sqrt", "invSqrt", "add", "sub", "mul", "mulByConstant", "div", "mean", "addSquares",
      "meanSquares", "negativeMean", "reduceSum", "reduceSub", "reduceMul", "reduceMean",
      "reduceSumOfSquares", "reduceMeanSquares", "reduceNegativeMean", "innerProduct",
      "innerProductWithBias"};
  if (op < sizeof(names) / sizeof(names[0])) return names[op];
  if (op == TG_OP_STOPGRAD_MAX) return "stopGradMax";
  return "?";
}

tg_status tg_recorder_new(tg_dtype dtype, size_t capacity, tg_recorder_t* out) {
  return guard([&] {
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_recorder_new: out is NULL");
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "tg_recorder_new: bad dtype");
    auto r = std::make_unique<tg_recorder>();
    r->dtype = dtype;
    if (dtype == TG_F64) r->t64 = std::make_unique<tg::Tape<double>>(capacity);
    else r->t32 = std::make_unique<tg::Tape<float>>(capacity);
    *out = r.release();
    return TG_OK;
  });
}

void tg_recorder_free(tg_recorder_t r) { delete r; }

tg_status tg_recorder_new_fixed(tg_dtype dtype, size_t capacity, size_t child_capacity, tg_recorder_t* out) {
  return guard([&] {
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_recorder_new_fixed: out is NULL");
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "tg_recorder_new_fixed: bad dtype");
    const tg::TapeConfig cfg{.capacity = capacity, .fixed_capacity = true, .child_capacity = child_capacity};
    auto r = std::make_unique<tg_recorder>();
    r->dtype = dtype;
    if (dtype == TG_F64) r->t64 = std::make_unique<tg::Tape<double>>(cfg);
    else r->t32 = std::make_unique<tg::Tape<float>>(cfg);
    *out = r.release();
    return TG_OK;
  });
}

tg_status tg_rec_checkpoint(tg_recorder_t r, tg_checkpoint* out) {
  return guard([&] {
    if (!r) return fail(TG_INVALID_HANDLE, "tg_rec_checkpoint: recorder is NULL");
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_rec_checkpoint: out is NULL");
    const tg::Checkpoint cp = r->visit([](auto& t) { return t.checkpoint(); });
    *out = tg_checkpoint{cp.mark, cp.params, cp.child_mark, cp.gathers, 0};
    return TG_OK;
  });
}

tg_status tg_rec_rewind(tg_recorder_t r, const tg_checkpoint* cp) {
  return guard([&] {
    if (!r) return fail(TG_INVALID_HANDLE, "tg_rec_rewind: recorder is NULL");
    if (!cp) return fail(TG_INVALID_ARGUMENT, "tg_rec_rewind: checkpoint is NULL");
    const tg::Checkpoint c{cp->mark, static_cast<std::size_t>(cp->child_mark), cp->params, cp->gathers};
    r->visit([&](auto& t) { t.rewind(c); return 0; });
    return TG_OK;
  });
}

tg_status tg_rec_get_stats(tg_recorder_t r, tg_rec_stats* out) {
  return guard([&] {
    if (!r) return fail(TG_INVALID_HANDLE, "tg_rec_get_stats: recorder is NULL");
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_rec_get_stats: out is NULL");
    *out = r->visit([](auto& t) {
      return tg_rec_stats{t.size(), t.peak_nodes(), t.child_pool_size(), t.peak_children(), t.peak_arena_bytes(),
                          t.max_arity(), t.n_params()};
    });
    return TG_OK;
  });
}

tg_status tg_rec_param(tg_recorder_t r, double v, uint32_t* node) {
  return guard([&] {
    *node = r->visit([&](auto& t) { return t.param(static_cast<typename std::decay_t<decltype(t)>::scalar_type>(v)).index; });
    return TG_OK;
  });
}
tg_status tg_rec_input(tg_recorder_t r, uint32_t col, double v, uint32_t* node) {
  return guard([&] {
    *node = r->visit([&](auto& t) { return t.input(col, static_cast<typename std::decay_t<decltype(t)>::scalar_type>(v)).index; });
    return TG_OK;
  });
}
tg_status tg_rec_const(tg_recorder_t r, double v, uint32_t* node) {
  return guard([&] {
    *node = r->visit([&](auto& t) { return t.constant(static_cast<typename std::decay_t<decltype(t)>::scalar_type>(v)).index; });
    return TG_OK;
  });
}
tg_status tg_rec_gather(tg_recorder_t r, uint32_t first, uint32_t stride, uint32_t n_rows, uint32_t col,
                        uint32_t offset, int32_t tidx, uint32_t* ref) {
  return guard([&] {
    *ref = r->visit([&](auto& t) { return t.gather(tg::ValueRef{first}, stride, n_rows, col, offset, tidx).index; });
    return TG_OK;
  });
}
tg_status tg_rec_op(tg_recorder_t r, uint8_t op, const uint32_t* children, uint32_t n, double c, uint32_t* node) {
  return guard([&] {
    std::vector<tg::ValueRef> k(n);
    for (uint32_t i = 0; i < n; ++i) k[i].index = children[i];
    *node = r->visit([&](auto& t) -> uint32_t {
      using S = typename std::decay_t<decltype(t)>::scalar_type;
      const auto kind = static_cast<tg::OpKind>(op);
      if (op == 0) throw std::invalid_argument("tg_rec_op: use tg_rec_param / tg_rec_input / tg_rec_const for leaves");
      if (kind == tg::OpKind::MulByConst) {
        if (n != 1) throw std::invalid_argument("mulByConstant: needs 1 child");
        return tg::mul_by_constant(t, k[0], static_cast<S>(c)).index;
      }
      if (kind == tg::OpKind::StopGradMax) return tg::stopgrad_max(t, std::span<const tg::ValueRef>(k)).index;
      switch (tg::arity_of(kind)) {
        case tg::OpArity::Unary:
          if (n != 1) throw std::invalid_argument(std::string("unary: op ") + tg_op_name(op) + " needs 1 child");
          return tg::unary(t, kind, k[0]).index;
        case tg::OpArity::Binary:
          if (n != 2) throw std::invalid_argument(std::string("binary: op ") + tg_op_name(op) + " needs 2 children");
          return tg::binary(t, kind, k[0], k[1]).index;
        default: break;
      }
      if (kind == tg::OpKind::InnerProductNoBias) {
        if (n % 2) throw std::invalid_argument("innerProduct: sequence lengths differ");
        return tg::inner_product(t, std::span<const tg::ValueRef>(k.data(), n / 2),
                                 std::span<const tg::ValueRef>(k.data() + n / 2, n / 2)).index;
      }
      if (kind == tg::OpKind::InnerProductWithBias) {
        if (n % 2 == 0) throw std::invalid_argument("innerProductWithBias: sequence lengths differ");
        const uint32_t m = (n - 1) / 2;
        return tg::inner_product_with_bias(t, std::span<const tg::ValueRef>(k.data(), m),
                                           std::span<const tg::ValueRef>(k.data() + m, m), k[n - 1]).index;
      }
      if (op > 29) throw std::invalid_argument("tg_rec_op: unknown opcode " + std::to_string(op));
      return tg::varying(t, kind, std::span<const tg::ValueRef>(k)).index;
    });
    return TG_OK;
  });
}
tg_status tg_rec_value(tg_recorder_t r, uint32_t ref, double* v) {
  return guard([&] {
    *v = r->visit([&](auto& t) { return static_cast<double>(t.value_of(tg::ValueRef{ref})); });
    return TG_OK;
  });
}
tg_status tg_rec_set_root(tg_recorder_t r, uint32_t node) {
  return guard([&] {
    r->visit([&](auto& t) { t.set_root(tg::ValueRef{node}); return 0; });
    return TG_OK;
  });
}
tg_status tg_rec_describe(tg_recorder_t r, tg_tape_desc* d) {
  return guard([&] {
    *d = r->visit([&](auto& t) { return t.describe(); });
    return TG_OK;
  });
}

tg_status tg_build_model(tg_model model, const tg_model_args* args, uint64_t seed, tg_recorder_t* out) {
  return guard([&] {
    const tgm::Dims D = tgm::Dims::resolve(model, args ? args->dims : nullptr);
    const tg_dtype dt = args ? args->dtype : TG_F64;
    std::uint32_t ni = 0, nk = 0;
    tgm::io_shape(model, D, ni, nk);
    std::vector<double> x(ni);
    std::vector<std::int32_t> k(nk);
    tgm::synth<double>(model, D, seed + 1, 1, x.data(), k.data());  // template sample
    auto r = std::make_unique<tg_recorder>();
    r->dtype = dt;
    if (dt == TG_F64) r->t64 = std::make_unique<tg::Tape<double>>(std::size_t(1) << 16);
    else r->t32 = std::make_unique<tg::Tape<float>>(std::size_t(1) << 16);
    r->visit([&](auto& t) {
      using S = typename std::decay_t<decltype(t)>::scalar_type;
      TgBuilder<S> b{t};
      const auto P = tgm::make_params(b, model, D, seed);
      const tgm::Sample smp{x.data(), k.data()};
      const auto root = tgm::build_sample(b, model, D, P, smp);
      t.set_root(root);
      return 0;
    });
    *out = r.release();
    return TG_OK;
  });
}

tg_status tg_synth_batch(tg_model model, const tg_model_args* args, uint64_t seed, size_t batch, void* inputs,
                         int32_t* index_inputs) {
  return guard([&] {
    const tgm::Dims D = tgm::Dims::resolve(model, args ? args->dims : nullptr);
    const tg_dtype dt = args ? args->dtype : TG_F64;
    if (dt == TG_F64) tgm::synth<double>(model, D, seed, batch, static_cast<double*>(inputs), index_inputs);
    else tgm::synth<float>(model, D, seed, batch, static_cast<float*>(inputs), index_inputs);
    return TG_OK;
  });
}

// Counter-based synthetic batches (tg_synth.cuh): arguments shared by the
// host and device generators.
namespace {
tgs::SynthArgs synth_args(tg_model model, const tg_model_args* args, uint64_t seed, uint64_t first, size_t batch,
                          void* inputs, int32_t* index_inputs, std::vector<double>& cdf) {
  const tgm::Dims D = tgm::Dims::resolve(model, args ? args->dims : nullptr);
  tgs::SynthArgs a{};
  a.model = model;
  a.f64 = (args ? args->dtype : TG_F64) == TG_F64;
  tgm::io_shape(model, D, a.n_inputs, a.n_index);
  if (batch && ((a.n_inputs && !inputs) || (a.n_index && !index_inputs)))
    throw std::invalid_argument("tg_synth: NULL output for a model with " + std::to_string(a.n_inputs) + " input and " +
                                std::to_string(a.n_index) + " index columns");
  a.n_classes = int(model) == tgm::kWideMlp ? D.d[3] : 0;
  if (int(model) == tgm::kCharMlp || int(model) == tgm::kGpt) {
    cdf = tgm::Zipf(D.d[0], int(model) == tgm::kCharMlp ? 1.1 : 1.0).cdf;
    a.V = static_cast<std::uint32_t>(cdf.size());
    a.cdf = cdf.data();
  }
  a.seed = seed;
  a.first = first;
  a.batch = batch;
  a.x = inputs;
  a.idx = index_inputs;
  return a;
}
}  // namespace

tg_status tg_synth_ctr(tg_model model, const tg_model_args* args, uint64_t seed, uint64_t first_sample, size_t batch,
                       void* inputs, int32_t* index_inputs) {
  return guard([&] {
    std::vector<double> cdf;
    const tgs::SynthArgs a = synth_args(model, args, seed, first_sample, batch, inputs, index_inputs, cdf);
    for (std::size_t i = 0; i < batch; ++i) {
      if (a.f64) tgs::synth_sample<double>(a, i);
      else tgs::synth_sample<float>(a, i);
    }
    return TG_OK;
  });
}

tg_status tg_synth_ctr_device(tg_model model, const tg_model_args* args, uint64_t seed, uint64_t first_sample,
                              size_t batch, void* inputs, int32_t* index_inputs, tg_stream_t stream) {
  return guard([&] {
    std::vector<double> cdf;
    const tgs::SynthArgs a = synth_args(model, args, seed, first_sample, batch, inputs, index_inputs, cdf);
    if (a.V > 1024) return fail(TG_INVALID_ARGUMENT, "tg_synth_ctr_device: Zipf vocabulary above 1024 ids");
    TG_CUDA_TRY(tgk::launch_synth(a, cdf.data(), static_cast<cudaStream_t>(stream)));
    return TG_OK;
  });
}

tg_status tg_compile(const tg_tape_desc* desc, tg_program_t* out) {
  return guard([&] {
    if (!desc || !out) return fail(TG_INVALID_ARGUMENT, "tg_compile: NULL argument");
    auto pr = std::make_unique<tg_program>();
    pr->P = tgc::compile(*desc);
    choose_config(*pr);
    *out = pr.release();
    return TG_OK;
  });
}

tg_status tg_program_info_get(tg_program_t p, tg_program_info* info) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_program_info_get: NULL program");
    if (!info) return fail(TG_INVALID_ARGUMENT, "tg_program_info_get: NULL info");
    const tgc::Program& P = p->P;
    tg_program_info i{};
    i.n_params = P.n_params;
    i.n_inputs = P.n_inputs;
    i.n_index_inputs = P.n_index_inputs;
    i.n_sample_nodes = P.n_sample_nodes;
    i.n_uniform_nodes = P.n_uniform_nodes;
    i.n_dense_groups = static_cast<uint32_t>(P.dense.size());
    i.n_fwd_instr = static_cast<uint32_t>(P.fwd.size());
    i.n_bwd_instr = static_cast<uint32_t>(P.bwd.size());
    i.n_edges = P.n_edges;
    i.tile_samples = p->S;
    i.smem_bytes = static_cast<uint32_t>(p->smem_bytes);
    i.storage = p->staged ? 3 : (p->jit.ok ? 2 : (p->smem ? 0 : 1));
    i.dtype = P.dtype;
    i.n_attn_heads = static_cast<uint32_t>(P.attn.size());
    i.n_layer_norms = static_cast<uint32_t>(P.lnorm.size());
    i.fused_mlp = p->fmlp.on ? 1u : 0u;
    *info = i;
    return TG_OK;
  });
}

tg_status tg_program_order(tg_program_t p, const uint32_t** order, uint32_t* n) {
  if (!p) return fail(TG_INVALID_HANDLE, "tg_program_order: NULL program");
  if (!order || !n) return fail(TG_INVALID_ARGUMENT, "tg_program_order: NULL argument");
  *order = p->P.order.data();
  *n = static_cast<uint32_t>(p->P.order.size());
  return TG_OK;
}

tg_status tg_set_memory_budget(tg_program_t p, size_t bytes) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_set_memory_budget: null program");
    p->mem_budget = bytes;
    return TG_OK;
  });
}

tg_status tg_chunk_samples(tg_program_t p, size_t batch, size_t* samples) {
  return guard([&] {
    if (!p || !samples) return fail(TG_INVALID_ARGUMENT, "tg_chunk_samples: null argument");
    *samples = p->staged ? std::min(staged_chunk(*p, batch), std::max<std::size_t>(batch, 1)) : std::max<std::size_t>(batch, 1);
    return TG_OK;
  });
}

tg_status tg_workspace_size(tg_program_t p, size_t batch, size_t* bytes) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_workspace_size: NULL program");
    if (!bytes) return fail(TG_INVALID_ARGUMENT, "tg_workspace_size: NULL bytes");
    *bytes = layout(*p, batch).total;
    return TG_OK;
  });
}

tg_status tg_forward_backward(tg_program_t p, const void* inputs, const int32_t* idx, size_t batch, const void* params,
                              void* loss, void* igrad, void* grad_sum, void* ws, size_t ws_bytes, tg_stream_t stream) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_forward_backward: NULL program");
    auto st = static_cast<cudaStream_t>(stream);
    if (p->P.dtype == TG_F64) return run_fb<double>(*p, inputs, idx, batch, params, loss, igrad, grad_sum, ws, ws_bytes, st);
    return run_fb<float>(*p, inputs, idx, batch, params, loss, igrad, grad_sum, ws, ws_bytes, st);
  });
}

tg_status tg_gd_update(tg_program_t p, void* params, const void* grad_sum, double gamma, size_t global_batch,
                       tg_stream_t stream) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_gd_update: NULL program");
    if (p->P.n_params && (!params || !grad_sum)) return fail(TG_INVALID_ARGUMENT, "tg_gd_update: NULL buffer");
    auto st = static_cast<cudaStream_t>(stream);
    if (global_batch == 0) return fail(TG_INVALID_ARGUMENT, "train_step: batch empty");
    if (p->P.dtype == TG_F64)
      TG_CUDA_TRY(tgk::launch_gd<double>(static_cast<double*>(params), static_cast<const double*>(grad_sum),
                                         p->P.n_params, gamma, static_cast<double>(global_batch), st));
    else
      TG_CUDA_TRY(tgk::launch_gd<float>(static_cast<float*>(params), static_cast<const float*>(grad_sum),
                                        p->P.n_params, gamma, static_cast<double>(global_batch), st));
    ++p->launches;
    return TG_OK;
  });
}

tg_status tg_allreduce_gd_step(tg_program_t p, void* params, void* grad_sum, double gamma, size_t global_batch,
                               tg_comm_t comm, tg_stream_t stream) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_allreduce_gd_step: NULL program");
    if (global_batch == 0) return fail(TG_INVALID_ARGUMENT, "train_step: batch empty");
    if (p->P.n_params && (!params || !grad_sum)) return fail(TG_INVALID_ARGUMENT, "tg_allreduce_gd_step: NULL buffer");
    auto st = static_cast<cudaStream_t>(stream);
    if (comm && p->P.n_params) {
      std::string err;
      if (!tgcomm::allreduce_sum(grad_sum, p->P.n_params, p->P.dtype, comm, st, err)) return fail(TG_NCCL, err);
    }
    return tg_gd_update(p, params, grad_sum, gamma, global_batch, stream);
  });
}

tg_status tg_train_step(tg_program_t p, const void* inputs, const int32_t* idx, size_t batch, void* params, void* loss,
                        void* grad_sum, double gamma, void* ws, size_t ws_bytes, tg_stream_t stream) {
  // GD fused into the reduction epilogue (one launch fewer per step).
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_train_step: NULL program");
    if (batch == 0) return fail(TG_INVALID_ARGUMENT, "train_step: batch empty");
    auto st = static_cast<cudaStream_t>(stream);
    if (p->P.dtype == TG_F64)
      return run_fb<double>(*p, inputs, idx, batch, params, loss, nullptr, grad_sum, ws, ws_bytes, st, params, gamma);
    return run_fb<float>(*p, inputs, idx, batch, params, loss, nullptr, grad_sum, ws, ws_bytes, st, params, gamma);
  });
}

tg_status tg_check_device_error(tg_program_t p, tg_stream_t stream, int64_t* sample_out, uint32_t* node_out) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_check_device_error: NULL program");
    if (!p->uploaded) return TG_OK;
    auto st = static_cast<cudaStream_t>(stream);
    TG_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long key = 0;
    TG_CUDA_TRY(cudaMemcpy(&key, p->d_err_key, 8, cudaMemcpyDeviceToHost));
    if (key == ~0ull) return TG_OK;
    const std::int64_t sample = static_cast<std::int64_t>(key >> 32);
    const std::uint32_t node = static_cast<std::uint32_t>(key & 0xffffffffu);
    if (sample_out) *sample_out = sample;
    if (node_out) *node_out = node;
    std::uint32_t op = 0xffffffffu;
    TG_CUDA_TRY(cudaMemcpy(&op, p->d_err_op, 4, cudaMemcpyDeviceToHost));
    if (op == 0xffffffffu && node != 0xfffffffeu) {
      tg_status s = p->P.dtype == TG_F64 ? diagnose<double>(*p, sample, st) : diagnose<float>(*p, sample, st);
      if (s != TG_OK) return s;
      TG_CUDA_TRY(cudaStreamSynchronize(st));
      TG_CUDA_TRY(cudaMemcpy(&op, p->d_err_op, 4, cudaMemcpyDeviceToHost));
    }
    double val = 0;
    TG_CUDA_TRY(cudaMemcpy(&val, p->d_err_val, 8, cudaMemcpyDeviceToHost));
    TG_CUDA_TRY(cudaMemset(p->d_err_key, 0xff, 8));
    TG_CUDA_TRY(cudaMemset(p->d_err_op, 0xff, 4));
    if (node == 0xfffffffeu)
      return fail(TG_INVALID_ARGUMENT, "gather: token index outside the table at sample " + std::to_string(sample));
    return fail(TG_DOMAIN, std::string(tg_op_name(static_cast<uint8_t>(op))) + ": input " + std::to_string(val) +
                               " is outside the operator domain");
  });
}

tg_status tg_profile_enable(tg_program_t p, int on) {
  if (!p) return fail(TG_INVALID_HANDLE, "tg_profile_enable: NULL program");
  p->profiling = on != 0;
  p->ev_used = 0;
  return TG_OK;
}

tg_status tg_profile_read(tg_program_t p, double* ms, uint64_t* n) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_profile_read: NULL program");
    if (!ms || !n) return fail(TG_INVALID_ARGUMENT, "tg_profile_read: NULL argument");
    double tot = 0;
    for (std::size_t i = 0; i < p->ev_used; ++i) {
      TG_CUDA_TRY(cudaEventSynchronize(p->ev[i].second));
      float t = 0;
      TG_CUDA_TRY(cudaEventElapsedTime(&t, p->ev[i].first, p->ev[i].second));
      tot += t;
    }
    *ms = tot;
    *n = p->ev_used;
    p->ev_used = 0;
    return TG_OK;
  });
}

tg_status tg_program_jit(tg_program_t p, const char** source, const char** log, double* compile_ms) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_program_jit: NULL program");
    if (!source || !log) return fail(TG_INVALID_ARGUMENT, "tg_program_jit: NULL argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      if (p->jit.source.empty()) p->jit = tgj::build(p->P);  // NVRTC compile only
    } else {
      TG_TRY(upload(*p));
    }
    *source = p->jit.source.c_str();
    *log = p->jit.log.c_str();
    if (compile_ms) *compile_ms = p->jit.compile_ms;
    return p->jit.ok ? TG_OK : fail(TG_UNSUPPORTED, "JIT not used: " + p->jit.log);
  });
}

uint64_t tg_launch_count(tg_program_t p) { return p ? p->launches : 0; }

void tg_program_free(tg_program_t p) { delete p; }

}  // extern "C"

extern "C" tg_status tg_gemm(tg_dtype dtype, int engine, uint32_t M, uint32_t N, uint32_t K, const void* A, size_t lda,
                             int a_kmajor, const void* B, size_t ldb, int b_nmajor, void* C, size_t ldc, int accumulate,
                             tg_stream_t stream) {
  return guard([&] {
    auto st = static_cast<cudaStream_t>(stream);
    auto fill = [&](auto* a, auto* b, auto* c, auto& g) {
      g.A = a;
      g.B = b;
      g.C = c;
      g.lda = lda;
      g.ldb = ldb;
      g.ldc = ldc;
      g.M = M;
      g.N = N;
      g.K = K;
      g.a_kmaj = a_kmajor != 0;
      g.b_nmaj = b_nmajor != 0;
      g.beta = accumulate != 0;
      g.epi = tgk::kEpiAccum;
    };
    if (dtype == TG_F32) {
      tgk::GemmArgs<float> g{};
      fill(static_cast<const float*>(A), static_cast<const float*>(B), static_cast<float*>(C), g);
      g.no_pair = engine == 2;   // engine 2: tcgen05 with single-CTA tiles only
      TG_CUDA_TRY(engine >= 1 ? tgk::launch_gemm_umma(g, 1, st) : tgk::launch_gemm<float>(g, 1, st));
    } else {
      if (engine >= 1) return fail(TG_UNSUPPORTED, "tg_gemm: no fp64 tcgen05 kind");
      tgk::GemmArgs<double> g{};
      fill(static_cast<const double*>(A), static_cast<const double*>(B), static_cast<double*>(C), g);
      TG_CUDA_TRY(tgk::launch_gemm<double>(g, 1, st));
    }
    return TG_OK;
  });
}

// ===========================================================================
// Host-buffer training loop.  Slot k of `depth` owns the device buffers of
// one in-flight step.  Per step:
//   copy-in stream : H2D(inputs -> slot)            -> record ready
//   caller's stream: wait ready -> forward/backward/reduce/GD -> record computed
//   copy-out stream: wait computed -> D2H(losses)   -> record done
// All compute stays on one stream (back to back, no cross-stream hop between
// steps); the copies of neighbouring steps overlap it.  The compute of a slot
// is a CUDA graph captured once (TG_PIPE_GRAPH=0: direct launches).
struct tg_pipeline {
  tg_program* p = nullptr;
  std::size_t batch = 0;
  void* params = nullptr;
  cudaStream_t cs = nullptr;                  // compute: the caller's stream
  cudaStream_t in = nullptr, out = nullptr;   // copy streams
  cudaStream_t cap = nullptr;                 // capture stream
  int depth = 4;                              // steps in flight (TG_PIPE_DEPTH)
  bool use_graph = true;
  struct Slot {
    void *X = nullptr, *K = nullptr, *L = nullptr;
    cudaEvent_t ready = nullptr, computed = nullptr, done = nullptr;
    bool used = false;
    cudaGraphExec_t ge = nullptr;
    double gamma = 0;
    std::uint64_t launches = 0;
  };
  std::vector<Slot> slot;
  void* G = nullptr;
  void* ws = nullptr;
  std::size_t ws_bytes = 0, x_bytes = 0, k_bytes = 0, l_bytes = 0;
  std::uint64_t steps = 0;
  bool trace = false;           // TG_PIPE_TRACE=1: host time per section, printed at free
  double t_sync = 0, t_in = 0, t_compute = 0, t_out = 0, t_total = 0;
  ~tg_pipeline() {
    if (trace && steps)
      std::fprintf(stderr, "[tg pipeline] %llu steps, host us/step: total %.2f sync %.2f copy-in %.2f compute %.2f "
                           "copy-out %.2f\n", static_cast<unsigned long long>(steps), t_total / steps,
                   t_sync / steps, t_in / steps, t_compute / steps, t_out / steps);
    for (cudaStream_t s : {in, out, cap})
      if (s) cudaStreamSynchronize(s);
    cudaStreamSynchronize(cs);
    for (Slot& s : slot) {
      if (s.ge) cudaGraphExecDestroy(s.ge);
      cudaFree(s.X);
      cudaFree(s.K);
      cudaFree(s.L);
      if (s.ready) cudaEventDestroy(s.ready);
      if (s.computed) cudaEventDestroy(s.computed);
      if (s.done) cudaEventDestroy(s.done);
    }
    for (cudaStream_t s : {in, out, cap})
      if (s) cudaStreamDestroy(s);
    cudaFree(G);
    cudaFree(ws);
  }
};

namespace {

tg_status pipe_compute(tg_pipeline& pl, tg_pipeline::Slot& sl, double gamma, cudaStream_t st) {
  tg_program& pr = *pl.p;
  const std::uint64_t l0 = pr.launches;
  const tg_status s =
      pr.P.dtype == TG_F64
          ? run_fb<double>(pr, sl.X, static_cast<const std::int32_t*>(sl.K), pl.batch, pl.params, sl.L, nullptr,
                           pl.G, pl.ws, pl.ws_bytes, st, pl.params, gamma)
          : run_fb<float>(pr, sl.X, static_cast<const std::int32_t*>(sl.K), pl.batch, pl.params, sl.L, nullptr,
                          pl.G, pl.ws, pl.ws_bytes, st, pl.params, gamma);
  sl.launches = pr.launches - l0;
  return s;
}

tg_status pipe_capture(tg_pipeline& pl, tg_pipeline::Slot& sl, double gamma) {
  if (sl.ge) TG_CUDA_TRY(cudaGraphExecDestroy(sl.ge));
  sl.ge = nullptr;
  const std::uint64_t l0 = pl.p->launches;
  TG_CUDA_TRY(cudaStreamBeginCapture(pl.cap, cudaStreamCaptureModeThreadLocal));
  const tg_status st = pipe_compute(pl, sl, gamma, pl.cap);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(pl.cap, &g);
  pl.p->launches = l0;   // counted per replay instead
  if (st != TG_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  TG_CUDA_TRY(ce);
  const cudaError_t ie = cudaGraphInstantiate(&sl.ge, g, 0);
  cudaGraphDestroy(g);
  TG_CUDA_TRY(ie);
  sl.gamma = gamma;
  return TG_OK;
}

}  // namespace

extern "C" {

tg_status tg_pipeline_new(tg_program_t p, size_t batch, void* params, tg_stream_t stream, tg_pipeline_t* out) {
  return guard([&] {
    if (!p) return fail(TG_INVALID_HANDLE, "tg_pipeline_new: NULL program");
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_new: NULL out");
    if (batch == 0) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_new: batch empty");
    if (p->P.n_params && !params) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_new: params is NULL");
    TG_TRY(upload(*p));   // synchronous set-up (and the JIT build) outside any capture
    auto pl = std::make_unique<tg_pipeline>();
    pl->p = p;
    pl->batch = batch;
    pl->params = params;
    pl->cs = static_cast<cudaStream_t>(stream);
    if (const char* e = std::getenv("TG_PIPE_DEPTH")) pl->depth = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("TG_PIPE_GRAPH")) pl->use_graph = e[0] != '0';
    if (const char* e = std::getenv("TG_PIPE_TRACE")) pl->trace = e[0] == '1';
    const std::size_t t = p->tsz();
    pl->x_bytes = std::size_t(p->P.n_inputs) * batch * t;
    pl->k_bytes = std::size_t(p->P.n_index_inputs) * batch * 4;
    pl->l_bytes = batch * t;
    TG_CUDA_TRY(cudaStreamCreateWithFlags(&pl->in, cudaStreamNonBlocking));
    TG_CUDA_TRY(cudaStreamCreateWithFlags(&pl->out, cudaStreamNonBlocking));
    TG_CUDA_TRY(cudaStreamCreateWithFlags(&pl->cap, cudaStreamNonBlocking));
    pl->slot.resize(pl->depth);
    for (tg_pipeline::Slot& sl : pl->slot) {
      if (pl->x_bytes) TG_CUDA_TRY(cudaMalloc(&sl.X, pl->x_bytes));
      if (pl->k_bytes) TG_CUDA_TRY(cudaMalloc(&sl.K, pl->k_bytes));
      TG_CUDA_TRY(cudaMalloc(&sl.L, pl->l_bytes));
      TG_CUDA_TRY(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
      TG_CUDA_TRY(cudaEventCreateWithFlags(&sl.computed, cudaEventDisableTiming));
      TG_CUDA_TRY(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    TG_CUDA_TRY(cudaMalloc(&pl->G, std::max<std::size_t>(1, p->P.n_params) * t));
    pl->ws_bytes = layout(*p, batch).total;
    TG_CUDA_TRY(cudaMalloc(&pl->ws, pl->ws_bytes));
    *out = pl.release();
    return TG_OK;
  });
}

tg_status tg_pipeline_step(tg_pipeline_t pl, const void* h_inputs, const int32_t* h_idx, void* h_loss, double gamma) {
  return guard([&] {
    if (!pl) return fail(TG_INVALID_HANDLE, "tg_pipeline_step: NULL pipeline");
    tg_program& pr = *pl->p;
    if (pr.P.n_inputs && !h_inputs) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_step: inputs is NULL");
    if (pr.P.n_index_inputs && !h_idx) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_step: index_inputs is NULL");
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    auto t = t0;
    auto lap = [&](double& acc) {
      if (!pl->trace) return;
      const auto n = clk::now();
      acc += std::chrono::duration<double, std::micro>(n - t).count();
      t = n;
    };
    tg_pipeline::Slot& sl = pl->slot[pl->steps % pl->slot.size()];
    // the slot was last used `depth` steps ago: that step must be complete
    if (sl.used) TG_CUDA_TRY(cudaEventSynchronize(sl.done));
    lap(pl->t_sync);
    if (pl->x_bytes) TG_CUDA_TRY(cudaMemcpyAsync(sl.X, h_inputs, pl->x_bytes, cudaMemcpyHostToDevice, pl->in));
    if (pl->k_bytes) TG_CUDA_TRY(cudaMemcpyAsync(sl.K, h_idx, pl->k_bytes, cudaMemcpyHostToDevice, pl->in));
    TG_CUDA_TRY(cudaEventRecord(sl.ready, pl->in));
    lap(pl->t_in);
    TG_CUDA_TRY(cudaStreamWaitEvent(pl->cs, sl.ready, 0));
    if (pl->use_graph && !pr.profiling) {
      if (!sl.ge || sl.gamma != gamma) TG_TRY(pipe_capture(*pl, sl, gamma));
      TG_CUDA_TRY(cudaGraphLaunch(sl.ge, pl->cs));
      pr.launches += sl.launches;
    } else {
      TG_TRY(pipe_compute(*pl, sl, gamma, pl->cs));
    }
    TG_CUDA_TRY(cudaEventRecord(sl.computed, pl->cs));
    lap(pl->t_compute);
    TG_CUDA_TRY(cudaStreamWaitEvent(pl->out, sl.computed, 0));
    if (h_loss) TG_CUDA_TRY(cudaMemcpyAsync(h_loss, sl.L, pl->l_bytes, cudaMemcpyDeviceToHost, pl->out));
    TG_CUDA_TRY(cudaEventRecord(sl.done, pl->out));
    lap(pl->t_out);
    if (pl->trace) pl->t_total += std::chrono::duration<double, std::micro>(clk::now() - t0).count();
    sl.used = true;
    ++pl->steps;
    return TG_OK;
  });
}

tg_status tg_pipeline_join(tg_pipeline_t pl, tg_stream_t stream) {
  return guard([&] {
    if (!pl) return fail(TG_INVALID_HANDLE, "tg_pipeline_join: NULL pipeline");
    for (const tg_pipeline::Slot& sl : pl->slot)
      if (sl.used) TG_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), sl.done, 0));
    return TG_OK;
  });
}

tg_status tg_pipeline_sync(tg_pipeline_t pl) {
  return guard([&] {
    if (!pl) return fail(TG_INVALID_HANDLE, "tg_pipeline_sync: NULL pipeline");
    for (const tg_pipeline::Slot& sl : pl->slot)
      if (sl.used) TG_CUDA_TRY(cudaEventSynchronize(sl.done));
    return TG_OK;
  });
}

tg_status tg_pipeline_grad_sum(tg_pipeline_t pl, void** grad_sum) {
  return guard([&] {
    if (!pl || !grad_sum) return fail(TG_INVALID_ARGUMENT, "tg_pipeline_grad_sum: NULL argument");
    *grad_sum = pl->G;
    return TG_OK;
  });
}

void tg_pipeline_free(tg_pipeline_t pl) { delete pl; }

tg_status tg_host_alloc(size_t bytes, void** out) {
  return guard([&] {
    if (!out) return fail(TG_INVALID_ARGUMENT, "tg_host_alloc: NULL out");
    TG_CUDA_TRY(cudaHostAlloc(out, std::max<std::size_t>(1, bytes), cudaHostAllocDefault));
    return TG_OK;
  });
}

void tg_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

// ===========================================================================
// Bit-exact serialization: raw ranges and BTSG snapshots.
namespace {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();   // no device / unregistered host memory
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// dst <- src (bytes), either side on the device or the host.  The byte image
// of an IEEE value is copied verbatim; the hosts this runs on are little-endian.
tg_status copy_bytes(void* dst, const void* src, std::size_t n) {
  if (n == 0) return TG_OK;
  if (is_device_ptr(dst) || is_device_ptr(src)) {
    TG_CUDA_TRY(cudaMemcpy(dst, src, n, cudaMemcpyDefault));
  } else {
    std::memcpy(dst, src, n);
  }
  return TG_OK;
}

std::size_t width_of(tg_dtype d) { return d == TG_F64 ? 8 : 4; }
constexpr std::size_t kSnapHeader = 4 + 4 + 1 + 1 + 8;
constexpr std::uint32_t kSnapVersion = 1;

}  // namespace

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "raw range format is little-endian");

extern "C" {

size_t tg_range_bytes(tg_dtype dtype, size_t count, int with_grads) {
  return width_of(dtype) * count * (with_grads ? 2 : 1);
}

tg_status tg_save_range(tg_dtype dtype, const void* values, const void* grads, size_t count, void* out, size_t out_bytes,
                        size_t* written) {
  return guard([&] {
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "save_range: dtype");
    const std::size_t w = width_of(dtype), need = tg_range_bytes(dtype, count, grads != nullptr);
    if (count && !values) return fail(TG_INVALID_ARGUMENT, "save_range: values is NULL");
    if (out_bytes < need || (need && !out)) return fail(TG_INVALID_ARGUMENT, "save_range: output buffer too small");
    char* o = static_cast<char*>(out);
    TG_TRY(copy_bytes(o, values, w * count));
    if (grads) TG_TRY(copy_bytes(o + w * count, grads, w * count));
    if (written) *written = need;
    return TG_OK;
  });
}

tg_status tg_load_range(tg_dtype dtype, void* values, void* grads, size_t count, const void* in, size_t in_bytes) {
  return guard([&] {
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "load_range: dtype");
    const std::size_t w = width_of(dtype), need = tg_range_bytes(dtype, count, grads != nullptr);
    if (in_bytes != need)
      return fail(TG_FORMAT, "load_range: " + std::to_string(in_bytes) + " bytes, expected " + std::to_string(need));
    if (count && (!values || !in)) return fail(TG_INVALID_ARGUMENT, "load_range: NULL buffer");
    const char* i = static_cast<const char*>(in);
    TG_TRY(copy_bytes(values, i, w * count));
    if (grads) TG_TRY(copy_bytes(grads, i + w * count, w * count));
    return TG_OK;
  });
}

size_t tg_snapshot_bytes(tg_dtype dtype, size_t count, int with_grads) {
  return kSnapHeader + tg_range_bytes(dtype, count, with_grads);
}

tg_status tg_save_snapshot(tg_dtype dtype, const void* values, const void* grads, size_t count, void* out,
                           size_t out_bytes, size_t* written) {
  return guard([&] {
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "save_snapshot: dtype");
    const std::size_t need = tg_snapshot_bytes(dtype, count, grads != nullptr);
    if (out_bytes < need || !out) return fail(TG_INVALID_ARGUMENT, "save_snapshot: output buffer too small");
    unsigned char* o = static_cast<unsigned char*>(out);
    std::memcpy(o, "BTSG", 4);
    const std::uint32_t ver = kSnapVersion;
    std::memcpy(o + 4, &ver, 4);
    o[8] = dtype == TG_F64 ? 1 : 0;
    o[9] = grads ? 1 : 0;
    const std::uint64_t n = count;
    std::memcpy(o + 10, &n, 8);
    std::size_t w = 0;
    TG_TRY(tg_save_range(dtype, values, grads, count, o + kSnapHeader, out_bytes - kSnapHeader, &w));
    if (written) *written = kSnapHeader + w;
    return TG_OK;
  });
}

tg_status tg_load_snapshot(const void* in, size_t in_bytes, tg_dtype dtype, void* values, void* grads, size_t capacity,
                           size_t* count_out, int* with_grads_out) {
  return guard([&] {
    if (dtype != TG_F64 && dtype != TG_F32) return fail(TG_INVALID_ARGUMENT, "load_snapshot: dtype");
    if (!in || in_bytes < kSnapHeader) return fail(TG_FORMAT, "load_snapshot: truncated header");
    const unsigned char* i = static_cast<const unsigned char*>(in);
    if (std::memcmp(i, "BTSG", 4) != 0) return fail(TG_FORMAT, "load_snapshot: bad magic");
    std::uint32_t ver = 0;
    std::memcpy(&ver, i + 4, 4);
    if (ver != kSnapVersion) return fail(TG_FORMAT, "load_snapshot: unsupported version " + std::to_string(ver));
    if (i[8] > 1 || i[9] > 1) return fail(TG_FORMAT, "load_snapshot: bad precision / flags");
    const tg_dtype dt = i[8] ? TG_F64 : TG_F32;
    const bool with_grads = i[9] & 1;
    std::uint64_t n = 0;
    std::memcpy(&n, i + 10, 8);
    if (in_bytes != tg_snapshot_bytes(dt, n, with_grads)) return fail(TG_FORMAT, "load_snapshot: payload size mismatch");
    // every check before the first byte is written: a cross-precision or
    // oversized load is an error with no partial write
    if (dt != dtype)
      return fail(TG_FORMAT, std::string("load_snapshot: snapshot precision ") + (dt == TG_F64 ? "fp64" : "fp32") +
                                 " differs from the target range's " + (dtype == TG_F64 ? "fp64" : "fp32"));
    if (n > capacity) return fail(TG_CAPACITY, "load_snapshot: " + std::to_string(n) + " values exceed capacity " +
                                                   std::to_string(capacity));
    if (count_out) *count_out = n;
    if (with_grads_out) *with_grads_out = with_grads ? 1 : 0;
    const std::size_t w = width_of(dt);
    if (n && !values) return fail(TG_INVALID_ARGUMENT, "load_snapshot: values is NULL");
    TG_TRY(copy_bytes(values, i + kSnapHeader, w * n));
    if (with_grads && grads) TG_TRY(copy_bytes(grads, i + kSnapHeader + w * n, w * n));
    return TG_OK;
  });
}

}  // extern "C"
