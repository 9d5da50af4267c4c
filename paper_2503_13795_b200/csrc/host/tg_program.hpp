// tg_program.hpp — compiled device program of a recorded tape.
//
// The compiler (tg_compiler.cpp) lowers a tg_tape_desc into the instruction
// streams below.  They are shared verbatim between host and device code.
//
// Storage model (per CTA tile of S samples, one sample per thread):
//   V[row][S+pad]  per-sample values   (shared memory, or HBM SoA workspace)
//   G[row][S+pad]  per-sample adjoints
// Rows hold: input leaves, per-sample op nodes, materialised gathers of
// sample-invariant tables (embedding rows), and AUX rows that carry
// per-sample contributions to sample-invariant operands.
//   UV[u]  sample-invariant values: [params | uniform op nodes | constants]
//   UG[u]  their batch-summed adjoints
// A sample-invariant ("uniform") op node — all children params / constants —
// is evaluated once per launch, not once per sample (e.g. the 1e-4 * sum p^2
// regulariser of cfg2).  Its adjoint is linear in the per-sample adjoints, so
// it is summed over the batch first and propagated once afterwards.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tg_abi.h"

namespace tgc {

// Operand encoding: mode in the top 3 bits.
constexpr std::uint32_t kModeShift = 29;
constexpr std::uint32_t kIndexMask = (1u << kModeShift) - 1;
enum OperandMode : std::uint32_t {
  kSlot = 0,     // per-sample row
  kUv = 1,       // sample-invariant value table entry
  kSGather = 2,  // per-sample row selected by a token id (slot gather table)
};
constexpr std::uint32_t enc(OperandMode m, std::uint32_t i) { return (std::uint32_t(m) << kModeShift) | i; }
constexpr std::uint32_t kNone = 0xffffffffu;

// Instruction kinds.
enum InstrKind : std::uint8_t {
  kNode = 0,        // evaluate op over operands into row `out`
  kInputLoad = 1,   // V[out] = inputs[aux][s]
  kGatherLoad = 2,  // V[out] = UV[table[idx[col][s]]]   (aux = uniform gather id)
  kDense = 3,       // rows [out, out+n_out) = W x + b   (aux = dense id)
  kAttn = 4,        // softmax attention head over per-sample rows (aux = attn id)
  kLNorm = 5,       // layer normalisation of n per-sample rows (aux = lnorm id)
};

// Operand flags for the reverse sweep.
enum OperandFlag : std::uint8_t {
  kAssign = 1,   // first contribution to this row: store instead of add
  kToAux = 2,    // contribution to a sample-invariant operand goes to aux row oaux[k]
};

struct Instr {
  std::uint8_t kind;
  std::uint8_t op;       // OpKind
  std::uint16_t pad;
  std::uint32_t out;     // row (per-sample) or uv index (uniform program)
  std::uint32_t nops;
  std::uint32_t opnd;    // offset into operand arrays
  std::uint32_t aux;     // input column / gather id / dense id / node id
  std::uint32_t node;    // recorded node index (diagnostics)
  double cst;            // constant slot (MulByConst)
};
static_assert(sizeof(Instr) == 32, "Instr layout");

// Per-sample contribution summed into a sample-invariant adjoint:
//   kind 0: coef * sum_s G[a][s] * (f == kNone ? 1 : V[f][s])
//   kind 1: coef * sum_s [idx[col][s] == row] * G[a][s]        (table scatter)
struct Term {
  std::uint32_t a;
  std::uint32_t f;       // factor row, or index column for kind 1
  std::int32_t row;      // -1 for kind 0
  std::uint32_t kind;
  double coef;
};
static_assert(sizeof(Term) == 24, "Term layout");

// A run of inner-product nodes that share their x operands and read a
// contiguous row-major weight block (a dense layer),
// optionally followed by the elementwise activation node of each output.
// Executed as one macro-instruction (kDense) forward and backward.
struct Dense {
  std::uint32_t out_row;   // rows of z_j = <x, W[j]> (+ b_j): out_row .. out_row+n_out-1
  std::uint32_t n_out;
  std::uint32_t n_in;
  std::uint32_t x_opnd;    // offset of the n_in shared x operands (kSlot)
  std::uint32_t w_uv;      // UV index of W[0][0]; W[j][k] = w_uv + j*n_in + k
  std::uint32_t b_uv;      // UV index of b[0] (b_j = b_uv + j), or kNone
  std::uint32_t first_node;
  std::uint32_t act_op;    // fused activation opcode (0 = none)
  std::uint32_t act_row;   // rows of act(z_j), or kNone
  std::uint32_t pad;
};

// Weight-gradient block of a dense layer: dest (j, k) = dest0 + j * n_in + k
// receives sum_s G[arow[j]][s] * V[frow[k]][s] — an outer-product
// contraction over the sample axis, evaluated register-tiled.
struct DenseGrad {
  std::uint32_t n_out, n_in;
  std::uint32_t arow_off;  // offset into dg_rows: n_out adjoint rows, then n_in value rows
  std::uint32_t dest0;
};

// A softmax attention head recognised in the recorded scalar graph (the
// composition of SPEC.md:306-312 out of reference ops): query unit u reads
// keys 0 .. n_u-1 of the head's key list and computes
//   c_j = scale * <q_u, k_j>        (innerProduct + mulByConstant)
//   m   = max_j c_j                 (stop-gradient shift)
//   a_j = exp(c_j - m) / sum_l exp(c_l - m)   (sub, exp, reduceSum, div)
//   o_u[i] = sum_j a_j v_j[i]       (innerProduct over the values' column i)
// One macro-instruction runs every unit; the interior nodes (scores, shifts,
// exponentials, normaliser, weights) get no rows.  Rows are hd (dv)
// consecutive rows per block: arows[unit_off + 3u] = {q_row, o_row, n_keys},
// arows[key_off + 2j] = {k_row, v_row}.
struct Attn {
  std::uint32_t n_units, n_keys, hd, dv;
  std::uint32_t unit_off, key_off;
  std::uint32_t first_node, n_nodes;   // recorded nodes covered (diagnostics, node-eval counts)
  std::uint32_t stat_row;              // rows stat_row + 2u, + 2u + 1: softmax max and 1 / sum of unit u
                                       // (written by the staged forward kernel for its reverse)
  double scale;
};

// Layer normalisation recognised in the recorded graph (the SPEC.md:288-296
// composition out of reference ops):
//   mu = mean(x), ms = meanSquares(x), var = ms - mu^2, rstd = invSqrt(var + eps),
//   n_i = (x_i - mu) * rstd,  y_i = n_i * gamma_i + beta_i.
// One macro-instruction; the scalar statistics and c_i, n_i * gamma_i get no
// rows; n_i keeps its row (the gamma gradient term reads it).  lnrows[off ..]
// holds five lists of n: x rows, n rows, y rows, gamma uv, beta uv.  The x
// adjoints are pushes like a dense layer's: lnflag[flag_off + i] & kAssign.
struct LNorm {
  std::uint32_t n, off, flag_off;
  std::uint32_t rstd_node, first_node, n_nodes;
  double eps;
};

struct GatherTable {          // candidate list of one gather
  std::uint32_t col;          // index column
  std::uint32_t n_rows;
  std::uint32_t cand_off;     // offset into cand[]
  std::uint32_t pad;
};

struct Program {
  tg_dtype dtype = TG_F64;
  std::uint32_t n_nodes = 0, n_params = 0, n_inputs = 0, n_index_inputs = 0;
  std::uint32_t n_rows = 0;               // per-sample rows
  std::uint32_t n_uv = 0;                 // params + uniform nodes + constants
  std::uint32_t uv_uniform_base = 0, uv_const_base = 0;
  std::uint32_t root_row = kNone;         // per-sample root row (kNone if root is uniform)
  std::uint32_t root_uv = kNone;
  std::uint64_t n_edges = 0;

  // per-sample program
  std::vector<Instr> fwd;                 // forward, topological
  std::vector<Instr> bwd;                 // reverse, processing order
  std::vector<std::uint32_t> opnd;        // operands
  std::vector<std::uint8_t> oflag;        // reverse-sweep flags per operand
  std::vector<std::uint32_t> oaux;        // aux row per operand (kToAux)
  std::vector<std::uint32_t> zero_rows;   // adjoint rows that must start at 0
  std::vector<std::uint32_t> input_rows;  // row of input column c (kNone if unused)
  std::vector<Dense> dense;
  std::vector<Attn> attn;
  std::vector<std::uint32_t> arows;
  std::vector<LNorm> lnorm;
  std::vector<std::uint32_t> lnrows;
  std::vector<std::uint8_t> lnflag;

  // gathers
  std::vector<GatherTable> ugather;       // sample-invariant tables (materialised)
  std::vector<GatherTable> sgather;       // per-sample row tables
  std::vector<std::uint32_t> cand;        // candidates (uv index or row)

  // batch reduction into sample-invariant adjoints
  std::vector<std::uint32_t> dest_uv;     // destination uv of each dest
  std::vector<std::uint32_t> term_off;    // CSR over terms, size n_dest+1
  std::vector<Term> terms;
  std::vector<DenseGrad> dgrad;           // register-tiled weight-gradient blocks
  std::vector<std::uint32_t> dg_rows;
  std::vector<std::uint8_t> dest_dense;   // 1 if the dest is produced by a DenseGrad block

  // uniform (sample-invariant) program
  std::vector<Instr> ufwd;                // evaluated once per launch
  std::vector<Instr> ubwd;                // processing order
  std::vector<double> uv_init;            // constants (and initial params)

  // processing order of the reference backward (recorded node ids)
  std::vector<std::uint32_t> order;

  // staged tier with dependency levels (tg_abi.cpp level_schedule): stage key
  // of each fwd / bwd instruction (level; reverse level << 12 | sub-level)
  std::vector<std::uint32_t> fwd_level, bwd_level;

  std::uint32_t n_dense_nodes = 0;
  std::uint32_t n_sample_nodes = 0, n_uniform_nodes = 0;
};

// Lowers desc; throws std::invalid_argument / std::runtime_error.
Program compile(const tg_tape_desc& desc);

}  // namespace tgc
