// tg_jit.cpp — straight-line CUDA emission + NVRTC build of short tapes.
//
// The emitted kernel follows the interpreter instruction by instruction:
//   forward  : reference ops.hpp:38-307 formulas (bias first, left to right);
//   reverse  : detail::propagate_node (ops.hpp:316-454) in the processing order
//              of backward_with_scratch (backprop.hpp:150-183), first write
//              of each adjoint a store (zero_grads folded away);
//   reduction: the compiler's batch terms, contracted over the CTA tile.
#include "tg_jit.hpp"

#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <cstdio>
#include <sstream>
#include <unordered_map>
#include <vector>

namespace tgj {
namespace {
// TG_JIT_SKIP=bwd|contract|tanh: work-skipping ablations (wrong results) that
// exist only in a -DTG_PROFILING build; the product library ignores the variable.
const char* profiling_skip() {
#ifdef TG_PROFILING
  return std::getenv("TG_JIT_SKIP");
#else
  return nullptr;
#endif
}
}  // namespace

namespace {

using tgc::Instr;
using tgc::kIndexMask;
using tgc::kModeShift;
using tgc::kNone;

constexpr std::uint64_t kMaxEdges = 6000;      // straight-line code budget
constexpr std::size_t kMaxConstBytes = 60 * 1024;

enum : std::uint8_t {
  Leaf = 0, Relu, Tanh, Exp, NegLog, Sigmoid, Inv, Sqr, Cub, Log, Sqrt, InvSqrt,
  Add, Sub, Mul, MulByConst, Div, Mean, AddSquares, MeanSquares, NegativeMean,
  AddVarying, SubVarying, MulVarying, MeanVarying, SumOfSquaresVarying, MeanSquaresVarying,
  NegativeMeanVarying, InnerProductNoBias, InnerProductWithBias,
  StopGradMax = TG_OP_STOPGRAD_MAX,
};

std::string lit(double c, bool f64) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", c);
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  if (s == "inf") s = f64 ? "__longlong_as_double(0x7ff0000000000000LL)" : "__int_as_float(0x7f800000)";
  else if (s == "-inf") s = f64 ? "__longlong_as_double(0xfff0000000000000LL)" : "__int_as_float(0xff800000)";
  else if (s == "nan" || s == "-nan") s = f64 ? "__longlong_as_double(0x7ff8000000000000LL)" : "__int_as_float(0x7fc00000)";
  return f64 ? "(T)" + s : "(T)" + s + "f";
}

struct Gen {
  const tgc::Program& P;
  const JitConfig& cfg;
  bool f64;
  std::ostringstream o;
  int tmp = 0;
  std::vector<int> vslot, gslot;     // row -> shared-memory slot of its value / adjoint (or -1)
  std::vector<char> vsm, gsm;        // value / adjoint lives in shared memory (written in place)
  unsigned ld = 0;                   // shared-memory row stride (tile + 1)
  std::vector<char> vstored, gstored;  // register-homed contraction rows already stored

  // Rows read by the batch-reduction terms are stored to shared memory as soon
  // as they are final, so their registers die early (register pressure sets
  // the occupancy of this kernel).
  void vstore(std::uint32_t r) {
    if (vslot[r] >= 0 && !vsm[r] && !vstored[r]) { o << "      " << sv(r) << " = " << v(r) << ";\n"; vstored[r] = 1; }
  }
  void gstore(std::uint32_t r) {
    if (gslot[r] >= 0 && !gsm[r] && !gstored[r]) { o << "      " << sg_(r) << " = " << g(r) << ";\n"; gstored[r] = 1; }
  }

  Gen(const tgc::Program& p, const JitConfig& c) : P(p), cfg(c), f64(p.dtype == TG_F64) {
    if (const char* e = std::getenv("TG_TANH")) tanh_fn = std::string(e) == "fp64" ? "tg_tanh_fp64" : "tg_tanh";
  }

  std::string fn(const char* d, const char* f) const { return f64 ? d : f; }
  std::string v(std::uint32_t r) const { return "v" + std::to_string(r); }
  std::string g(std::uint32_t r) const { return "g" + std::to_string(r); }
  std::string sv(std::uint32_t r) const { return "sV[" + std::to_string(std::size_t(vslot[r]) * ld) + "u + col]"; }
  std::string sg_(std::uint32_t r) const { return "sG[" + std::to_string(std::size_t(gslot[r]) * ld) + "u + col]"; }
  // value of row r: once a register-homed row has been stored for the
  // contraction, later reads (the reverse sweep) reload it from shared memory
  // so the register dies at the store (TG_JIT_RELOAD=0 keeps registers)
  std::string V(std::uint32_t r) const {
    if (umode) return "sU[" + std::to_string(r) + "]";
    if (!vov.empty() && !vov[r].empty()) return vov[r];
    return vsm[r] || (reload && !vstored.empty() && vstored[r]) ? sv(r) : v(r);
  }
  // grouped mode (generate_grouped): a dense-layer output row lives in lane j
  // of the sample's lane group; its value is read from the group's exchange
  // buffer (vov) and contributions to its adjoint go to the owner lane (gov).
  std::vector<std::string> vov, gov, gcond;
  std::vector<int> gj;
  bool reload = true;
  std::string Gx(std::uint32_t r) const {  // adjoint of row r
    if (umode) return "sG[" + std::to_string(r) + "]";
    return gsm[r] ? sg_(r) : g(r);
  }
  std::string uv(std::uint32_t i) const {
    // tape constants are known when the program is compiled: literals (x / 2
    // becomes an exact multiply, domain checks on constants fold away)
    if (i >= P.uv_const_base && i < P.n_uv) return lit(P.uv_init[i], f64);
    if (su) return "sU[" + std::to_string(i) + "]";
    return cfg.const_uv ? "cUV[" + std::to_string(i) + "]" : "UVg[" + std::to_string(i) + "]";
  }
  // fused kernels: the sample-invariant table lives in shared memory (sU),
  // evaluated by each CTA; umode emits the uniform program itself (values
  // sU[u], adjoints sG[u]).
  bool su = false, umode = false;
  std::string tanh_fn = "tg_tanh";   // fp64 tanh variant (kernels/tg_math.cuh)
  std::string ix_expr(const tgc::GatherTable& t) const {
    return "tg_ix(idx, " + std::to_string(t.col) + "ull * batch + s, " + std::to_string(t.n_rows) + "u)";
  }

  // Operand value expression; slot gathers are materialised into a temp.
  std::string val(std::uint32_t op) {
    const std::uint32_t m = op >> kModeShift, i = op & kIndexMask;
    if (m == tgc::kSlot) return V(i);
    if (m == tgc::kUv) return uv(i);
    const tgc::GatherTable& t = P.sgather[i];
    const std::string name = "sg" + std::to_string(tmp++);
    o << "      T " << name << "; { const int ix = " << ix_expr(t) << "; switch (ix) {";
    for (std::uint32_t r = 0; r < t.n_rows; ++r)
      o << " case " << r << ": " << name << " = " << V(P.cand[t.cand_off + r]) << "; break;";
    o << " default: " << name << " = " << V(P.cand[t.cand_off]) << "; } }\n";
    return name;
  }

  void push(const Instr& in, std::uint32_t k, const std::string& expr) {
    const std::uint32_t op = P.opnd[in.opnd + k];
    const std::uint32_t m = op >> kModeShift, i = op & kIndexMask;
    const std::uint8_t fl = P.oflag[in.opnd + k];
    if (umode) {
      if (m == tgc::kUv && i < P.uv_const_base) o << "      sG[" << i << "] += " << expr << ";\n";
      return;
    }
    if (m == tgc::kSlot && !gov.empty() && !gov[i].empty()) {
      const std::string cond = gcond.empty() ? "q == " + std::to_string(gj[i]) + "u" : gcond[i];
      o << "      if (" << cond << ") " << gov[i] << " += " << expr << ";\n";
    } else if (m == tgc::kSlot) {
      if (gsm[i]) o << "      " << sg_(i) << (fl & tgc::kAssign ? " = " : " += ") << expr << ";\n";
      else if (fl & tgc::kAssign) o << "      T " << g(i) << " = " << expr << ";\n";
      else o << "      " << g(i) << " += " << expr << ";\n";
    } else if (m == tgc::kSGather) {
      const tgc::GatherTable& t = P.sgather[i];
      o << "      { const T c_ = " << expr << "; const int ix = " << ix_expr(t) << "; switch (ix) {";
      for (std::uint32_t r = 0; r < t.n_rows; ++r)
        o << " case " << r << ": " << Gx(P.cand[t.cand_off + r]) << " += c_; break;";
      o << " default: " << Gx(P.cand[t.cand_off]) << " += c_; } }\n";
    } else if (fl & tgc::kToAux) {
      o << "      T " << g(P.oaux[in.opnd + k]) << " = " << expr << ";\n";
    }
  }

  void check(const std::string& cond, const Instr& in, const std::string& bad) {
    if (umode) {  // sample-invariant node: CTA 0 reports it like the interpreter's prologue
      o << "      if (blockIdx.x == 0u && (" << cond << ")) { tg_err(err_key, 0ull, " << in.node
        << "u); if (atomicCAS(A.err_op, 0xffffffffu, " << unsigned(in.op) << "u) == 0xffffffffu) *A.err_val = (double)("
        << bad << "); }\n";
      return;
    }
    o << "      if (" << cond << ") tg_err(err_key, s, " << in.node << "u);\n";
  }

  void forward(const Instr& in) {
    if (in.kind == tgc::kInputLoad) {
      o << "      const T " << v(in.out) << " = in[" << in.aux << "ull * batch + s];\n";
      return;
    }
    if (in.kind == tgc::kDense) { dense_fwd(P.dense[in.aux]); return; }
    if (in.kind == tgc::kGatherLoad) {
      const tgc::GatherTable& t = P.ugather[in.aux];
      o << "      const T " << v(in.out) << " = UVt[cand[" << t.cand_off << "u + " << ix_expr(t) << "]];\n";
      return;
    }
    const std::uint32_t n = in.nops;
    std::vector<std::string> a(n);
    for (std::uint32_t j = 0; j < n; ++j) a[j] = val(P.opnd[in.opnd + j]);
    const std::string out = "      const T " + v(in.out) + " = ";
    const std::string Z = "(T)0", ONE = "(T)1", TWO = "(T)2";
    switch (in.op) {
      case Relu: o << out << a[0] << " > " << Z << " ? " << a[0] << " : " << Z << ";\n"; break;
      case Tanh: o << out << fn(tanh_fn.c_str(), "tanhf") << "(" << a[0] << ");\n"; break;
      case Exp: o << out << fn("exp", "expf") << "(" << a[0] << ");\n"; break;
      case NegLog: check("!(" + a[0] + " > (T)0)", in, a[0]); o << out << "-" << fn("log", "logf") << "(" << a[0] << ");\n"; break;
      case Sigmoid: o << out << ONE << " / (" << ONE << " + " << fn("exp", "expf") << "(-" << a[0] << "));\n"; break;
      case Inv: check(a[0] + " == (T)0", in, a[0]); o << out << ONE << " / " << a[0] << ";\n"; break;
      case Sqr: o << out << a[0] << " * " << a[0] << ";\n"; break;
      case Cub: o << out << a[0] << " * " << a[0] << " * " << a[0] << ";\n"; break;
      case Log: check("!(" + a[0] + " > (T)0)", in, a[0]); o << out << fn("log", "logf") << "(" << a[0] << ");\n"; break;
      case Sqrt: check("!(" + a[0] + " > (T)0)", in, a[0]); o << out << fn("sqrt", "sqrtf") << "(" << a[0] << ");\n"; break;
      case InvSqrt: check("!(" + a[0] + " > (T)0)", in, a[0]); o << out << ONE << " / " << fn("sqrt", "sqrtf") << "(" << a[0] << ");\n"; break;
      case MulByConst: o << out << a[0] << " * " << lit(in.cst, f64) << ";\n"; break;
      case Add: o << out << a[0] << " + " << a[1] << ";\n"; break;
      case Sub: o << out << a[0] << " - " << a[1] << ";\n"; break;
      case Mul: o << out << a[0] << " * " << a[1] << ";\n"; break;
      case Div: check(a[1] + " == (T)0", in, a[1]); o << out << a[0] << " / " << a[1] << ";\n"; break;
      case Mean: o << out << "(" << a[0] << " + " << a[1] << ") / " << TWO << ";\n"; break;
      case AddSquares: o << out << a[0] << " * " << a[0] << " + " << a[1] << " * " << a[1] << ";\n"; break;
      case MeanSquares: o << out << "(" << a[0] << " * " << a[0] << " + " << a[1] << " * " << a[1] << ") / " << TWO << ";\n"; break;
      case NegativeMean: o << out << "-(" << a[0] << " + " << a[1] << ") / " << TWO << ";\n"; break;
      case AddVarying: case MeanVarying: case NegativeMeanVarying: {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = 0;";
        for (auto& x : a) o << " " << acc << " += " << x << ";";
        o << "\n";
        if (in.op == MeanVarying) o << "      " << acc << " /= (T)" << n << ";\n";
        if (in.op == NegativeMeanVarying) o << "      " << acc << " = -" << acc << " / (T)" << n << ";\n";
        o << out << acc << ";\n";
        break;
      }
      case SubVarying: {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = " << a[0] << ";";
        for (std::uint32_t j = 1; j < n; ++j) o << " " << acc << " -= " << a[j] << ";";
        o << "\n" << out << acc << ";\n";
        break;
      }
      case MulVarying: {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = " << ONE << ";";
        for (auto& x : a) o << " " << acc << " *= " << x << ";";
        o << "\n" << out << acc << ";\n";
        break;
      }
      case SumOfSquaresVarying: case MeanSquaresVarying: {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = 0;";
        for (auto& x : a) o << " " << acc << " += " << x << " * " << x << ";";
        o << "\n";
        if (in.op == MeanSquaresVarying) o << "      " << acc << " /= (T)" << n << ";\n";
        o << out << acc << ";\n";
        break;
      }
      case InnerProductNoBias: case InnerProductWithBias: {
        const bool bias = in.op == InnerProductWithBias;
        const std::uint32_t m = bias ? (n - 1) / 2 : n / 2;
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = " << (bias ? a[n - 1] : std::string("(T)0")) << ";";
        for (std::uint32_t j = 0; j < m; ++j) o << " " << acc << " += " << a[j] << " * " << a[m + j] << ";";
        o << "\n" << out << acc << ";\n";
        break;
      }
      case StopGradMax: {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = " << a[0] << ";";
        for (std::uint32_t j = 1; j < n; ++j) o << " " << acc << " = " << a[j] << " > " << acc << " ? " << a[j] << " : " << acc << ";";
        o << "\n" << out << acc << ";\n";
        break;
      }
      default: o << out << "(T)0;\n"; break;
    }
  }

  std::string act_f(std::uint32_t op, const std::string& z) const {
    switch (op) {
      case Relu: return "(" + z + " > (T)0 ? " + z + " : (T)0)";
      case Tanh: {
        const char* sk = profiling_skip();
        if (sk && std::string(sk) == "tanh") return "(" + z + ")";
        return fn(tanh_fn.c_str(), "tanhf") + "(" + z + ")";
      }
      case Exp: return fn("exp", "expf") + "(" + z + ")";
      case Sigmoid: return "((T)1 / ((T)1 + " + fn("exp", "expf") + "(-" + z + ")))";
      case Sqr: return "(" + z + " * " + z + ")";
      case Cub: return "(" + z + " * " + z + " * " + z + ")";
      default: return z;
    }
  }
  std::string act_b(std::uint32_t op, const std::string& g, const std::string& y, const std::string& z) const {
    switch (op) {
      case Relu: return "(" + z + " > (T)0 ? " + g + " : (T)0)";
      case Tanh: return g + " * ((T)1 - " + y + " * " + y + ")";
      case Exp: return g + " * " + y;
      case Sigmoid: return g + " * " + y + " * ((T)1 - " + y + ")";
      case Sqr: return g + " * (T)2 * " + z;
      case Cub: return g + " * (T)3 * " + z + " * " + z;
      default: return g;
    }
  }
  std::string wexpr(const tgc::Dense& D, std::uint32_t k) const {
    const std::string idx = std::to_string(D.w_uv) + "u + j * " + std::to_string(D.n_in) + "u + " + std::to_string(k) + "u";
    if (su) return "sU[" + idx + "]";
    return cfg.const_uv ? "cUV[" + idx + "]" : "UVg[" + idx + "]";
  }
  // Dense layer forward: loop over the outputs (static code O(n_in)),
  // x operands held in registers, weights from the constant bank.
  std::string wconst(const tgc::Dense& D, std::uint32_t j, std::uint32_t k) const {
    return uv(D.w_uv + j * D.n_in + k);
  }
  void dense_fwd(const tgc::Dense& D) {
    std::vector<std::string> x(D.n_in);
    for (std::uint32_t k = 0; k < D.n_in; ++k) {
      x[k] = "dx" + std::to_string(tmp++);
      o << "      const T " << x[k] << " = " << val(P.opnd[D.x_opnd + k]) << ";\n";
    }
    if (!cfg.dense_loop) {  // unrolled: every output a register, weights constant-bank operands
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        const std::string acc = "a" + std::to_string(tmp++);
        o << "      T " << acc << " = " << (D.b_uv != kNone ? uv(D.b_uv + j) : std::string("(T)0")) << ";";
        for (std::uint32_t k = 0; k < D.n_in; ++k) o << " " << acc << " += " << x[k] << " * " << wconst(D, j, k) << ";";
        o << "\n      const T " << v(D.out_row + j) << " = " << acc << ";\n";
        if (D.act_op) o << "      const T " << v(D.act_row + j) << " = " << act_f(D.act_op, v(D.out_row + j)) << ";\n";
      }
      return;
    }
    o << "#pragma unroll " << cfg.unroll_j << "\n      for (unsigned j = 0; j < " << D.n_out << "u; ++j) {\n";
    if (D.b_uv != kNone) o << "        T z = " << (su ? "sU[" : cfg.const_uv ? "cUV[" : "UVg[") << D.b_uv << "u + j];\n";
    else o << "        T z = (T)0;\n";
    for (std::uint32_t k = 0; k < D.n_in; ++k) o << "        z += " << x[k] << " * " << wexpr(D, k) << ";\n";
    if (vslot[D.out_row] >= 0) o << "        sV[(" << vslot[D.out_row] << "u + j) * " << ld << "u + col] = z;\n";
    if (D.act_op) o << "        sV[(" << vslot[D.act_row] << "u + j) * " << ld << "u + col] = " << act_f(D.act_op, "z") << ";\n";
    o << "      }\n";
  }
  // Dense layer reverse: activation derivative, adjoint of z (kept for the
  // weight-gradient contraction), x adjoints accumulated in registers.
  void dense_bwd(const tgc::Dense& D) {
    std::vector<std::string> dx(D.n_in);
    for (std::uint32_t k = 0; k < D.n_in; ++k) {
      dx[k] = "gx" + std::to_string(tmp++);
      o << "      T " << dx[k] << " = (T)0;\n";
    }
    if (!cfg.dense_loop) {
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        const std::uint32_t zr = D.out_row + j;
        if (D.act_op) {
          const std::uint32_t hr = D.act_row + j;
          o << "      T " << g(zr) << " = " << act_b(D.act_op, Gx(hr), V(hr), V(zr)) << ";\n";
        }
        o << "     ";
        for (std::uint32_t k = 0; k < D.n_in; ++k) o << " " << dx[k] << " += " << g(zr) << " * " << wconst(D, j, k) << ";";
        o << "\n";
      }
      Instr pseudo{};
      pseudo.opnd = D.x_opnd;
      for (std::uint32_t k = 0; k < D.n_in; ++k) push(pseudo, k, dx[k]);
      return;
    }
    o << "#pragma unroll " << cfg.unroll_j << "\n      for (unsigned j = 0; j < " << D.n_out << "u; ++j) {\n";
    const std::string gz = "sG[(" + std::to_string(gslot[D.out_row]) + "u + j) * " + std::to_string(ld) + "u + col]";
    if (D.act_op) {
      const std::string gh = "sG[(" + std::to_string(gslot[D.act_row]) + "u + j) * " + std::to_string(ld) + "u + col]";
      const std::string y = "sV[(" + std::to_string(vslot[D.act_row]) + "u + j) * " + std::to_string(ld) + "u + col]";
      const std::string z = vslot[D.out_row] >= 0
          ? "sV[(" + std::to_string(vslot[D.out_row]) + "u + j) * " + std::to_string(ld) + "u + col]" : std::string("(T)0");
      o << "        const T gz = " << act_b(D.act_op, gh, y, z) << ";\n        " << gz << " = gz;\n";
    } else {
      o << "        const T gz = " << gz << ";\n";
    }
    for (std::uint32_t k = 0; k < D.n_in; ++k) o << "        " << dx[k] << " += gz * " << wexpr(D, k) << ";\n";
    o << "      }\n";
    Instr pseudo{};
    pseudo.opnd = D.x_opnd;
    for (std::uint32_t k = 0; k < D.n_in; ++k) push(pseudo, k, dx[k]);
  }

  void reverse(const Instr& in) {
    if (in.kind == tgc::kDense) { dense_bwd(P.dense[in.aux]); return; }
    const std::uint32_t n = in.nops;
    std::vector<std::string> a(n);
    auto A = [&](std::uint32_t j) -> const std::string& {
      if (a[j].empty()) a[j] = val(P.opnd[in.opnd + j]);
      return a[j];
    };
    const std::string G = Gx(in.out), Y = V(in.out);
    const std::string ONE = "(T)1", TWO = "(T)2";
    switch (in.op) {
      case Relu: push(in, 0, "(" + A(0) + " > (T)0 ? " + G + " : (T)0)"); break;
      case Tanh: push(in, 0, G + " * (" + ONE + " - " + Y + " * " + Y + ")"); break;
      case Exp: push(in, 0, G + " * " + Y); break;
      case NegLog: push(in, 0, "-" + G + " / " + A(0)); break;
      case Sigmoid: push(in, 0, G + " * " + Y + " * (" + ONE + " - " + Y + ")"); break;
      case Inv: push(in, 0, "-" + G + " * " + Y + " * " + Y); break;
      case Sqr: push(in, 0, G + " * " + TWO + " * " + A(0)); break;
      case Cub: push(in, 0, G + " * (T)3 * " + A(0) + " * " + A(0)); break;
      case Log: push(in, 0, G + " / " + A(0)); break;
      case Sqrt: push(in, 0, G + " / (" + TWO + " * " + Y + ")"); break;
      case InvSqrt: push(in, 0, "-" + G + " * " + Y + " / (" + TWO + " * " + A(0) + ")"); break;
      case MulByConst: push(in, 0, G + " * " + lit(in.cst, f64)); break;
      case Add: push(in, 0, G); push(in, 1, G); break;
      case Sub: push(in, 0, G); push(in, 1, "-" + G); break;
      case Mul: A(0); A(1); push(in, 0, G + " * " + a[1]); push(in, 1, G + " * " + a[0]); break;
      case Div: A(0); A(1); push(in, 0, G + " / " + a[1]); push(in, 1, "-" + G + " * " + a[0] + " / (" + a[1] + " * " + a[1] + ")"); break;
      case Mean: push(in, 0, G + " / " + TWO); push(in, 1, G + " / " + TWO); break;
      case AddSquares: A(0); A(1); push(in, 0, G + " * " + TWO + " * " + a[0]); push(in, 1, G + " * " + TWO + " * " + a[1]); break;
      case MeanSquares: A(0); A(1); push(in, 0, G + " * " + a[0]); push(in, 1, G + " * " + a[1]); break;
      case NegativeMean: push(in, 0, "-" + G + " / " + TWO); push(in, 1, "-" + G + " / " + TWO); break;
      case AddVarying: for (std::uint32_t j = 0; j < n; ++j) push(in, j, G); break;
      case SubVarying: push(in, 0, G); for (std::uint32_t j = 1; j < n; ++j) push(in, j, "-" + G); break;
      case MulVarying: {
        for (std::uint32_t j = 0; j < n; ++j) A(j);
        for (std::uint32_t k = 0; k < n; ++k) {
          std::string prefix = ONE, suffix = ONE;
          for (std::uint32_t j = 0; j < k; ++j) prefix = "(" + prefix + " * " + a[j] + ")";
          for (std::uint32_t j = n - 1; j > k; --j) suffix = "(" + suffix + " * " + a[j] + ")";
          push(in, k, G + " * " + prefix + " * " + suffix);
        }
        break;
      }
      case MeanVarying: for (std::uint32_t j = 0; j < n; ++j) push(in, j, G + " / (T)" + std::to_string(n)); break;
      case SumOfSquaresVarying: for (std::uint32_t j = 0; j < n; ++j) push(in, j, G + " * " + TWO + " * " + A(j)); break;
      case MeanSquaresVarying: {
        const std::string sc = "(" + G + " * " + TWO + " / (T)" + std::to_string(n) + ")";
        for (std::uint32_t j = 0; j < n; ++j) push(in, j, sc + " * " + A(j));
        break;
      }
      case NegativeMeanVarying: for (std::uint32_t j = 0; j < n; ++j) push(in, j, "-" + G + " / (T)" + std::to_string(n)); break;
      case InnerProductNoBias: case InnerProductWithBias: {
        const bool bias = in.op == InnerProductWithBias;
        const std::uint32_t m = bias ? (n - 1) / 2 : n / 2;
        for (std::uint32_t k = 0; k < m; ++k) {
          A(k);
          A(m + k);
          push(in, k, G + " * " + a[m + k]);
          push(in, m + k, G + " * " + a[k]);
        }
        if (bias) push(in, n - 1, G);
        break;
      }
      default: break;
    }
  }
};

const char* kMath =
#include "tg_math.inc"
    ;

const char* kPrelude = R"(
struct TermC { unsigned a; unsigned f; int row; unsigned kind; double coef; };
__device__ __forceinline__ void tg_err(unsigned long long* key, unsigned long long s, unsigned node) {
  atomicMin(key, (s << 32) | node);
}
__device__ __forceinline__ int tg_ix(const int* __restrict__ idx, unsigned long long at, unsigned n) {
  const int r = idx[at];
  return (unsigned)r < n ? r : 0;
}
// kernel argument block; host mirror: tgj::JitArgs<T> (tg_jit.hpp), same field order
struct JitArgs {
  const T* in; const int* idx; unsigned long long batch;
  T* loss; T* igrad; T* partial; unsigned grid_rows; unsigned n_groups;
  unsigned long long* err_key; double* err_val; unsigned* err_op;
  const T* UVg; const unsigned* cand; const unsigned* toff; const TermC* terms;
  const T* params; const T* consts; T* UVw;
  unsigned* tickets; T* partial2;
  T* grad_sum; T* gd_params; T gamma; T gd_batch;
};
)";

const char* kArgAliases =
    "  const T* __restrict__ in = A.in; const int* __restrict__ idx = A.idx; const unsigned long long batch = A.batch;\n"
    "  T* __restrict__ loss = A.loss; T* __restrict__ igrad = A.igrad; T* __restrict__ partial = A.partial;\n"
    "  const unsigned grid_rows = A.grid_rows; unsigned long long* err_key = A.err_key;\n"
    "  const T* __restrict__ UVg = A.UVg; const unsigned* __restrict__ cand = A.cand;\n"
    "  const unsigned* __restrict__ toff = A.toff; const TermC* __restrict__ terms = A.terms;\n"
    "  (void)in; (void)idx; (void)loss; (void)igrad; (void)UVg; (void)cand; (void)toff; (void)terms; (void)err_key;\n";

// Prologue of a fused tg_jit_tape: wait for the previous kernel on the stream
// (PDL), then CTA 0 resets the generated epilogue's last-CTA ticket, which
// lives in the caller's workspace (tickets == workspace + Layout::done), so
// launches of one program on several streams / workspaces never share it.
// The previous launch's epilogue has completed once griddepcontrol.wait
// returns, and this launch's epilogue only counts after this kernel is done.
// The cooperative form keeps its grid-barrier words in the program instead.
std::string fuse_wait(bool coop) {
  std::string s = "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");   // params of the previous step\n";
  if (!coop) s += "  if (blockIdx.x == 0 && threadIdx.x == 0) A.tickets[0] = 0u;   // epilogue ticket (workspace)\n";
  return s;
}

}  // namespace

// ---------------------------------------------------------------------------
// Fused prologue / generated epilogue (one module per program).
//
// Prologue: every CTA of tg_jit_tape stages UV = [params | uniform nodes |
// consts] in shared memory (sU) and evaluates the uniform program there, as
// straight-line code (block-parallel fixed-order sums for wide reductions).
// That replaces the separate single-CTA k_uniform_fwd launch and its chain of
// global round trips; the per-sample code reads uniform operands from sU.
//
// Epilogue (tg_jit_epi, same module): one warp per reduction destination sums
// the per-CTA partials in a fixed order; the last CTA to finish runs the
// uniform reverse sweep as straight-line code on shared memory, writes
// grad_sum and applies GD.  Both kernels are launched with programmatic
// stream serialisation, so each one's launch overlaps the tail of the kernel
// before it (griddepcontrol.wait before the first dependent read).
constexpr std::uint32_t kFuseMaxUv = 2048;

bool wide_op(std::uint8_t op) {
  return op == AddVarying || op == MeanVarying || op == NegativeMeanVarying || op == SumOfSquaresVarying ||
         op == MeanSquaresVarying || op == InnerProductNoBias || op == InnerProductWithBias;
}

bool fusable(const tgc::Program& P, std::string& why) {
  if (P.n_uv > kFuseMaxUv) { why = "uniform table too large to fuse"; return false; }
  for (const auto* list : {&P.ufwd, &P.ubwd})
    for (const Instr& in : *list) {
      if (in.kind != tgc::kNode) { why = "uniform instruction kind"; return false; }
      for (std::uint32_t j = 0; j < in.nops; ++j)
        if ((P.opnd[in.opnd + j] >> kModeShift) != tgc::kUv) { why = "uniform operand mode"; return false; }
    }
  return true;
}

struct FuseCode {
  std::string tail;       // inside tg_jit_tape, at its end (cooperative grid-wide epilogue)
  std::string decl;       // file scope: operand lists, helpers
  std::string pro_load;   // inside tg_jit_tape: params / consts -> sU (loads in flight, no barrier)
  std::string pro_prog;   // barrier, then the uniform program on sU
  std::string pro;        // pro_load + pro_prog
  std::string epi;        // the tg_jit_epi kernel
};

FuseCode fuse_code(const tgc::Program& P, const JitConfig& cfg, const std::string& launch_bounds) {
  const bool f64 = P.dtype == TG_F64;
  FuseCode fc;
  // operand uv lists of the wide uniform instructions, read one per thread: a
  // contiguous run is indexed directly, anything else comes from a __device__
  // table (coalesced; a __constant__ table would serialise divergent reads)
  std::vector<std::uint32_t> ops;
  auto opx = [&](const Instr& in, const std::string& j) -> std::string {
    const std::uint32_t o0 = P.opnd[in.opnd] & kIndexMask;
    bool run = true;
    for (std::uint32_t k = 1; k < in.nops && run; ++k) run = (P.opnd[in.opnd + k] & kIndexMask) == o0 + k;
    if (run) return "(" + std::to_string(o0) + "u + (" + j + "))";
    const std::size_t off = ops.size();
    for (std::uint32_t k = 0; k < in.nops; ++k) ops.push_back(P.opnd[in.opnd + k] & kIndexMask);
    return "gUO[" + std::to_string(off) + "u + (" + j + ")]";
  };
  const unsigned B = cfg.block;
  const std::string NUV = std::to_string(std::max<std::uint32_t>(1, P.n_uv));
  // ---- prologue ----
  {
    Gen U(P, cfg);
    U.umode = true;
    U.su = true;
    std::ostringstream& o = U.o;
    fc.pro_load = "  __shared__ T sU[" + NUV + "];\n  __shared__ T sRed_[32];\n"
      "  for (unsigned i = threadIdx.x; i < " + std::to_string(P.n_params) + "u; i += " + std::to_string(B) +
      "u) sU[i] = A.params[i];\n"
      "  for (unsigned i = threadIdx.x; i < " + std::to_string(P.n_uv - P.uv_const_base) + "u; i += " +
      std::to_string(B) + "u) sU[" + std::to_string(P.uv_const_base) + "u + i] = A.consts[i];\n";
    o << "  __syncthreads();\n  {\n";
    for (const Instr& in : P.ufwd) {
      if (in.nops >= 64 && wide_op(in.op)) {
        const std::uint32_t n = in.nops;
        const bool ip = in.op == InnerProductNoBias || in.op == InnerProductWithBias;
        const std::uint32_t m = in.op == InnerProductWithBias ? (n - 1) / 2 : (ip ? n / 2 : n);
        const std::string xo = opx(in, "j"), yo = ip ? opx(in, std::to_string(m) + "u + j") : std::string();
        o << "    { T part = (T)0;\n"
          << "      for (unsigned j = threadIdx.x; j < " << m << "u; j += " << B << "u) { const T v = sU[" << xo
          << "]; part += ";
        if (ip) o << "v * sU[" << yo << "]";
        else if (in.op == SumOfSquaresVarying || in.op == MeanSquaresVarying) o << "v * v";
        else o << "v";
        o << "; }\n      part = tg_block_sum(part, sRed_);\n"
          << "      if (threadIdx.x == 0) { T r = part;";
        if (in.op == InnerProductWithBias) o << " r = sU[" << (P.opnd[in.opnd + n - 1] & kIndexMask) << "] + r;";
        if (in.op == MeanVarying || in.op == MeanSquaresVarying) o << " r /= (T)" << n << ";";
        if (in.op == NegativeMeanVarying) o << " r = -r / (T)" << n << ";";
        o << " sU[" << in.out << "] = r; }\n      __syncthreads(); }\n";
      } else {
        o << "    if (threadIdx.x == 0) {\n";
        U.forward(in);
        o << "      sU[" << in.out << "] = " << U.v(in.out) << ";\n    }\n    __syncthreads();\n";
      }
    }
    o << "    if (blockIdx.x == 0)  // UV for the epilogue and for diagnostics\n"
      << "      for (unsigned i = threadIdx.x; i < " << P.n_uv << "u; i += " << B << "u) A.UVw[i] = sU[i];\n  }\n";
    fc.pro_prog = o.str();
    fc.pro = fc.pro_load + fc.pro_prog;
  }
  // ---- epilogue: fixed-order reduction of the per-CTA partials, then the
  // uniform reverse sweep, grad_sum and GD on one CTA ----
  const unsigned nd = static_cast<unsigned>(P.dest_uv.size());
  // The reverse sweep from the reduced totals (in A.partial2) on one CTA of
  // `nt` threads; sU holds the uniform table; pp(r) the parameter values.
  auto tail = [&](std::ostringstream& o, Gen& U, unsigned nt, const std::function<std::string(unsigned)>& pp) {
    const std::string NT = std::to_string(nt) + "u";
    o << "  for (unsigned i = threadIdx.x; i < " << P.n_uv << "u; i += " << NT << ") sG[i] = (T)0;\n"
      << "  __syncthreads();\n"
      << "  for (unsigned d = threadIdx.x; d < " << nd << "u; d += " << NT << ") sG[gDU[d]] = __ldcg(A.partial2 + d);\n"
      << "  __syncthreads();\n";
    if (P.root_uv != kNone) o << "  if (threadIdx.x == 0) sG[" << P.root_uv << "] += (T)A.batch;\n  __syncthreads();\n";
    for (const Instr& in : P.ubwd) {
      const bool par = (in.pad & 1) && in.nops >= 32 &&
                       (in.op == AddVarying || in.op == SubVarying || in.op == MeanVarying || in.op == NegativeMeanVarying ||
                        in.op == SumOfSquaresVarying || in.op == MeanSquaresVarying || in.op == InnerProductNoBias ||
                        in.op == InnerProductWithBias);
      if (par) {  // distinct children: one thread per child
        const std::uint32_t n = in.nops;
        const std::string uo = opx(in, "j");
        o << "  { const T g = sG[" << in.out << "];\n"
          << "    for (unsigned j = threadIdx.x; j < " << n << "u; j += " << NT << ") {\n"
          << "      const unsigned u = " << uo << ";\n      T c;\n";
        switch (in.op) {
          case AddVarying: o << "      c = g;\n"; break;
          case SubVarying: o << "      c = j == 0u ? g : -g;\n"; break;
          case MeanVarying: o << "      c = g / (T)" << n << ";\n"; break;
          case NegativeMeanVarying: o << "      c = -g / (T)" << n << ";\n"; break;
          case SumOfSquaresVarying: o << "      c = g * (T)2 * sU[u];\n"; break;
          case MeanSquaresVarying: o << "      c = (g * (T)2 / (T)" << n << ") * sU[u];\n"; break;
          case InnerProductNoBias:
            o << "      c = g * sU[" << opx(in, "j < " + std::to_string(n / 2) + "u ? j + " + std::to_string(n / 2) + "u : j - " +
                                       std::to_string(n / 2) + "u") << "];\n";
            break;
          default: {
            const std::uint32_t m = (n - 1) / 2;
            o << "      c = j == " << n - 1 << "u ? g : g * sU[" << opx(in, "j < " + std::to_string(m) + "u ? j + " +
                                                                           std::to_string(m) + "u : j - " + std::to_string(m) + "u")
              << "];\n";
          }
        }
        o << "      if (u < " << P.uv_const_base << "u) sG[u] += c;\n    }\n    __syncthreads(); }\n";
      } else {
        o << "  if (threadIdx.x == 0) {\n";
        U.reverse(in);
        o << "  }\n  __syncthreads();\n";
      }
    }
    const unsigned rounds = (P.n_params + nt - 1) / nt;
    o << "#pragma unroll\n"
      << "  for (int r = 0; r < " << rounds << "; ++r) {\n"
      << "    const unsigned i = threadIdx.x + " << NT << " * r;\n"
      << "    if (i < " << P.n_params << "u) {\n"
      << "      const T gs = sG[i];\n"
      << "      if (A.grad_sum) A.grad_sum[i] = gs;\n"
      << "      if (A.gd_params) A.gd_params[i] = " << pp(rounds) << " - A.gamma * gs / A.gd_batch;\n    }\n  }\n";
  };
  // warp-per-destination reduction of partial rows: destinations d0, d0 + dstride, ...
  auto reduce = [&](std::ostringstream& o, const std::string& d0, const std::string& dstride) {
    o << "  for (unsigned d = " << d0 << "; d < " << nd << "u; d += " << dstride << ") {\n"
      << "    const T* row = A.partial + (unsigned long long)d * A.grid_rows;\n"
      << "    const unsigned lane = threadIdx.x & 31u;\n"
      << "    T t = (T)0;\n"
      << "    for (unsigned c = lane; c < A.grid_rows; c += 512u) {  // 16 loads in flight, added in sequential order\n"
      << "      T x[16];\n"
      << "#pragma unroll\n"
      << "      for (int u = 0; u < 16; ++u) x[u] = c + 32u * u < A.grid_rows ? __ldcg(row + c + 32u * u) : (T)0;\n"
      << "#pragma unroll\n"
      << "      for (int u = 0; u < 16; ++u) if (c + 32u * u < A.grid_rows) t += x[u];\n"
      << "    }\n"
      << "    for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);\n"
      << "    if (lane == 0) A.partial2[d] = t;\n  }\n";
  };
  if (cfg.coop) {
    // in the tape kernel itself (cooperative launch: every CTA is resident):
    // grid barrier, reduction spread over all warps, grid barrier, tail on CTA 0
    Gen U(P, cfg);
    U.umode = true;
    U.su = true;
    std::ostringstream& o = U.o;
    const std::string W = std::to_string(cfg.block / 32) + "u";
    o << "  // ---- grid-wide epilogue (cooperative launch) ----\n"
      << "  tg_grid_barrier(A.tickets);\n";
    reduce(o, "blockIdx.x * " + W + " + (threadIdx.x >> 5)", "gridDim.x * " + W);
    o << "  tg_grid_barrier(A.tickets);\n"
      << "  if (blockIdx.x == 0) {\n"
      << "  __shared__ T sG[" << NUV << "];\n";
    tail(o, U, cfg.block, [&](unsigned) { return std::string("A.gd_params[i]"); });
    o << "  }\n";
    fc.tail = o.str();
  } else if (nd > 0 || !P.ubwd.empty()) {   // nothing to reduce or propagate (cfg1): no epilogue
    Gen U(P, cfg);
    U.umode = true;
    U.su = true;
    std::ostringstream& o = U.o;
    o << "extern \"C\" __global__ void __launch_bounds__(256) tg_jit_epi(const JitArgs A) {\n"
      << "  __shared__ T sU[" << NUV << "];\n  __shared__ T sG[" << NUV << "];\n  __shared__ unsigned last;\n"
      << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");   // tg_jit_tape's partials / UV\n"
      << "  // UV and the parameters are final: fetched now, so the last CTA's serial\n"
      << "  // tail only waits for the reduced totals\n"
      << "  T uvp[" << std::max(1u, (P.n_uv + 255) / 256) << "], pp[" << std::max(1u, (P.n_params + 255) / 256) << "];\n"
      << "#pragma unroll\n"
      << "  for (int r = 0; r < " << (P.n_uv + 255) / 256 << "; ++r) { const unsigned i = threadIdx.x + 256u * r; uvp[r] = i < "
      << P.n_uv << "u ? __ldcg(A.UVw + i) : (T)0; }\n"
      << "#pragma unroll\n"
      << "  for (int r = 0; r < " << (P.n_params + 255) / 256 << "; ++r) { const unsigned i = threadIdx.x + 256u * r; pp[r] = (A.gd_params && i < "
      << P.n_params << "u) ? A.gd_params[i] : (T)0; }\n";
    reduce(o, "(blockIdx.x * 256u + threadIdx.x) >> 5", "gridDim.x * 8u");
    o << "  __threadfence();\n  __syncthreads();\n"
      << "  if (threadIdx.x == 0) last = atomicAdd(A.tickets, 1u) == gridDim.x - 1u;\n"
      << "  __syncthreads();\n  if (!last) return;\n  __threadfence();\n"
      << "  if (threadIdx.x == 0) A.tickets[0] = 0u;\n"
      << "#pragma unroll\n"
      << "  for (int r = 0; r < " << (P.n_uv + 255) / 256 << "; ++r) { const unsigned i = threadIdx.x + 256u * r; if (i < " << P.n_uv
      << "u) sU[i] = uvp[r]; }\n";
    tail(o, U, 256, [&](unsigned) { return std::string("pp[r]"); });
    o << "}\n";
    fc.epi = o.str();
  }
  {
    std::ostringstream d;
    d << "__device__ const unsigned gDU[" << std::max(1u, nd) << "] = {";
    for (unsigned i = 0; i < nd; ++i) d << (i ? ", " : "") << P.dest_uv[i] << "u";
    d << "};\n"
      << "// grid-wide barrier of a cooperative launch: bar[0] arrivals, bar[1] generation;\n"
      << "// the last arrival resets the count and opens the next generation\n"
      << "__device__ __forceinline__ void tg_grid_barrier(unsigned* bar) {\n"
      << "  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n"
      << "    volatile unsigned* gen = bar + 1;\n"
      << "    const unsigned g = *gen;\n"
      << "    __threadfence();\n"
      << "    if (atomicAdd(bar, 1u) == gridDim.x - 1u) {\n"
      << "      bar[0] = 0u;\n"
      << "      __threadfence();\n"
      << "      atomicAdd(bar + 1, 1u);\n"
      << "    } else {\n"
      << "      while (*gen == g) __nanosleep(32);\n"
      << "    }\n"
      << "    __threadfence();\n"
      << "  }\n"
      << "  __syncthreads();\n"
      << "}\n";
    fc.decl += d.str();
  }
  std::ostringstream d;
  d << "__device__ const unsigned gUO[" << std::max<std::size_t>(1, ops.size()) << "] = {";
  for (std::size_t i = 0; i < ops.size(); ++i) d << (i ? ", " : "") << ops[i] << "u";
  d << "};\n"
    << "__device__ __forceinline__ T tg_block_sum(T v, T* red) {  // fixed order; result in thread 0\n"
    << "  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);\n"
    << "  __syncthreads();\n"
    << "  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;\n"
    << "  __syncthreads();\n"
    << "  T t = (T)0;\n"
    << "  if (threadIdx.x == 0) for (unsigned i = 0; i < (blockDim.x >> 5); ++i) t += red[i];\n"
    << "  return t;\n}\n";
  fc.decl += d.str();
  (void)launch_bounds;
  (void)f64;
  return fc;
}

bool eligible(const tgc::Program& P) {
  return P.root_row != kNone && P.n_edges <= kMaxEdges && P.n_rows <= 4096 && P.attn.empty() && P.lnorm.empty();   // no kAttn / kLNorm codegen
}

std::string generate(const tgc::Program& P, const JitConfig& cfg, unsigned& n_crow_g, unsigned& n_crow_v,
                     std::vector<tgc::Term>& terms_out, std::vector<std::uint32_t>& toff_out,
                     std::size_t& smem_elems) {
  Gen G(P, cfg);
  G.su = cfg.fuse;
  const FuseCode fc = cfg.fuse ? fuse_code(P, cfg, "") : FuseCode{};
  const bool f64 = P.dtype == TG_F64;
  const unsigned tile = cfg.block * cfg.spt;
  G.ld = tile + 1;
  // shared-memory slots: rows produced inside dense loops live there (written
  // in place); rows read by the batch-reduction terms get a slot too and are
  // stored from registers at the end of the sample.
  G.vslot.assign(P.n_rows, -1);
  G.gslot.assign(P.n_rows, -1);
  G.vsm.assign(P.n_rows, 0);
  G.gsm.assign(P.n_rows, 0);
  n_crow_g = n_crow_v = 0;
  auto vrange = [&](std::uint32_t r0, std::uint32_t n) {
    for (std::uint32_t j = 0; j < n; ++j) { G.vslot[r0 + j] = static_cast<int>(n_crow_v++); G.vsm[r0 + j] = 1; }
  };
  auto grange = [&](std::uint32_t r0, std::uint32_t n) {
    for (std::uint32_t j = 0; j < n; ++j) { G.gslot[r0 + j] = static_cast<int>(n_crow_g++); G.gsm[r0 + j] = 1; }
  };
  for (const auto& D : P.dense) {
    if (!cfg.dense_loop) break;  // unrolled dense layers keep their rows in registers
    // z values are kept only when something reads them: the activation's
    // derivative (relu / sqr / cub) or, without a fused activation, the consumers
    const bool need_z = !D.act_op || D.act_op == Relu || D.act_op == Sqr || D.act_op == Cub;
    if (need_z) vrange(D.out_row, D.n_out);
    grange(D.out_row, D.n_out);
    if (D.act_op) { vrange(D.act_row, D.n_out); grange(D.act_row, D.n_out); }
  }
  for (const auto& t : P.terms) {
    if (G.gslot[t.a] < 0) G.gslot[t.a] = static_cast<int>(n_crow_g++);
    if (t.kind == 0 && t.f != kNone && G.vslot[t.f] < 0) G.vslot[t.f] = static_cast<int>(n_crow_v++);
  }
  // generic terms (dense-block destinations are produced by the register-tiled blocks)
  const unsigned nd = static_cast<unsigned>(P.dest_uv.size());
  terms_out.clear();
  toff_out.assign(1, 0);
  for (unsigned d = 0; d < nd; ++d) {
    if (!P.dest_dense[d])
      for (std::uint32_t q = P.term_off[d]; q < P.term_off[d + 1]; ++q) {
        tgc::Term t = P.terms[q];
        t.a = static_cast<std::uint32_t>(G.gslot[t.a]);
        if (t.kind == 0 && t.f != kNone) t.f = static_cast<std::uint32_t>(G.vslot[t.f]);
        terms_out.push_back(t);
      }
    toff_out.push_back(static_cast<std::uint32_t>(terms_out.size()));
  }
  const unsigned ld = G.ld;
  const unsigned ndpt = (nd + cfg.block - 1) / cfg.block;
  const bool reg_acc = ndpt <= 8;
  const bool dense = !P.dgrad.empty();
  // dense-block thread mapping: 4x4 register tiles x sample chunks
  struct DB { unsigned nj, nk, bj, bk, nb, c, dest0, off; };
  std::vector<DB> dbs;
  std::size_t scratch = 0;
  for (const auto& dg : P.dgrad) {
    DB b{dg.n_out, dg.n_in, (dg.n_out + 3) / 4, (dg.n_in + 3) / 4, 0, 0, dg.dest0, dg.arow_off};
    b.nb = b.bj * b.bk;
    // sample chunks per 4x4 tile: enough threads busy, scratch <= 512 partials
    // (keeps shared memory from limiting occupancy below the register limit)
    b.c = std::max(1u, std::min({cfg.block / b.nb, tile / 8, 512u / std::max(1u, b.nj * b.nk)}));
    if (b.nb > cfg.block) b.c = 1;
    scratch = std::max<std::size_t>(scratch, std::size_t(b.c) * b.nj * b.nk);
    dbs.push_back(b);
  }
  smem_elems = std::size_t(n_crow_g + n_crow_v) * ld + (dense ? nd + scratch : 0);

  std::ostringstream& o = G.o;
  o << "typedef " << (f64 ? "double" : "float") << " T;\n" << kMath << kPrelude << fc.decl;
  if (cfg.const_uv && !cfg.fuse) o << "__constant__ T cUV[" << std::max<std::uint32_t>(1, P.n_uv) << "];\n";
  for (std::size_t bi = 0; bi < dbs.size(); ++bi) {
    const DB& b = dbs[bi];
    o << "__constant__ unsigned cDG" << bi << "[" << b.nj + b.nk << "] = {";
    for (unsigned j = 0; j < b.nj; ++j) o << (j ? ", " : "") << G.gslot[P.dg_rows[b.off + j]];
    for (unsigned k = 0; k < b.nk; ++k) o << ", " << G.vslot[P.dg_rows[b.off + b.nj + k]];
    o << "};\n";
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << cfg.block;
  if (cfg.min_blocks) o << ", " << cfg.min_blocks;
  o << ") tg_jit_tape(const JitArgs A) {\n" << kArgAliases
    << (cfg.fuse ? fuse_wait(cfg.coop) : std::string())
    << fc.pro
    << (cfg.fuse ? "  const T* __restrict__ UVt = sU;\n" : "  const T* __restrict__ UVt = UVg;\n") << "  (void)UVt;\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  T* sG = reinterpret_cast<T*>(smem_raw);\n"
    << "  T* sV = sG + " << n_crow_g << " * " << ld << ";\n"
    << "  T* sDW = sV + " << n_crow_v << " * " << ld << ";\n"
    << "  T* sS = sDW + " << (dense ? nd : 0) << ";\n"
    << "  (void)sG; (void)sV; (void)sDW; (void)sS;\n"
    << "  const unsigned tid = threadIdx.x;\n";
  if (dense) o << "  for (unsigned q = tid; q < " << nd << "u; q += " << cfg.block << "u) sDW[q] = (T)0;\n";
  if (reg_acc && nd) o << "  T acc[" << ndpt << "]; for (int q = 0; q < " << ndpt << "; ++q) acc[q] = 0;\n";
  // each CTA owns a contiguous share of the batch (a multiple of 32 samples),
  // walked in tiles; a partial last tile instead of a whole extra tile on a
  // few CTAs (cfg1: 1,954 tiles on 1,776 resident CTAs left the GPU 40% idle)
  o << "  const unsigned long long per = ((batch + gridDim.x - 1) / gridDim.x + 31ull) / 32ull * 32ull;\n"
    << "  const unsigned long long lo = (unsigned long long)blockIdx.x * per;\n"
    << "  const unsigned long long hi = lo + per < batch ? lo + per : batch;\n";
  if (nd && !reg_acc)
    o << "  if (lo >= hi)\n    for (unsigned d = tid; d < " << nd << "u; d += " << cfg.block
      << "u) partial[(unsigned long long)d * grid_rows + blockIdx.x] = (T)0;\n";
  // the tile's inputs are loaded before any per-sample code, so every load of
  // the thread is in flight at once (stores of one sample would otherwise sit
  // between the loads of the next)
  std::vector<std::uint32_t> incols;
  for (const Instr& in : P.fwd)
    if (in.kind == tgc::kInputLoad) incols.push_back(in.aux);
  o << "  for (unsigned long long base = lo; base < hi; base += " << tile << "ull) {\n";
  for (std::uint32_t c : incols)
    o << "    T pin" << c << "[" << cfg.spt << "];\n";
  if (!incols.empty()) {
    o << "#pragma unroll\n    for (unsigned jj = 0; jj < " << cfg.spt << "u; ++jj) {\n"
      << "      const unsigned long long sp = base + jj * " << cfg.block << "u + tid;\n";
    for (std::uint32_t c : incols)
      o << "      pin" << c << "[jj] = sp < hi ? in[" << c << "ull * batch + sp] : (T)0;\n";
    o << "    }\n";
  }
  o << "#pragma unroll\n"
    << "    for (unsigned jj = 0; jj < " << cfg.spt << "u; ++jj) {\n"
    << "    const unsigned long long s = base + jj * " << cfg.block << "u + tid;\n"
    << "    const unsigned col = jj * " << cfg.block << "u + tid;\n"
    << "    (void)col;\n"
    << "    if (s < hi) {\n";
  G.vstored.assign(P.n_rows, 0);
  if (const char* e = std::getenv("TG_JIT_RELOAD")) G.reload = std::atoi(e) != 0;
  G.gstored.assign(P.n_rows, 0);
  for (const Instr& in : P.fwd) {
    if (in.kind == tgc::kInputLoad) o << "      const T " << G.v(in.out) << " = pin" << in.aux << "[jj];\n";
    else G.forward(in);
    if (in.kind == tgc::kDense) {
      const tgc::Dense& D = P.dense[in.aux];
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        G.vstore(D.out_row + j);
        if (D.act_op) G.vstore(D.act_row + j);
      }
    } else {
      G.vstore(in.out);
    }
  }
  o << "      if (loss) loss[s] = " << G.V(P.root_row) << ";\n";
  for (std::uint32_t r : P.zero_rows) {
    if (G.gsm[r]) o << "      " << G.sg_(r) << " = (T)0;\n";
    else o << "      T " << G.g(r) << " = (T)0;\n";
  }
  if (G.gsm[P.root_row]) o << "      " << G.sg_(P.root_row) << " = (T)1;\n";
  else o << "      T " << G.g(P.root_row) << " = (T)1;\n";
  // profiling-only ablations (wrong results): TG_JIT_SKIP=bwd|contract
  const char* skip = profiling_skip();
  const bool skip_bwd = skip && std::string(skip) == "bwd", skip_con = skip && std::string(skip) == "contract";
  if (!skip_bwd)
    for (const Instr& in : P.bwd) {
      if (in.kind == tgc::kNode) G.gstore(in.out);   // adjoint final when its node is processed
      G.reverse(in);
      if (in.kind == tgc::kDense)
        for (std::uint32_t j = 0; j < P.dense[in.aux].n_out; ++j) G.gstore(P.dense[in.aux].out_row + j);
    }
  else
    for (std::uint32_t r = 0; r < P.n_rows; ++r)
      if (!G.gsm[r] && r != P.root_row && std::find(P.zero_rows.begin(), P.zero_rows.end(), r) == P.zero_rows.end())
        o << "      T " << G.g(r) << " = " << G.V(r) << ";\n";
  for (std::uint32_t c = 0; c < P.n_inputs; ++c) {
    const std::uint32_t r = P.input_rows[c];
    if (r != kNone) o << "      if (igrad) igrad[" << c << "ull * batch + s] = " << G.Gx(r) << ";\n";
  }
  for (std::uint32_t r = 0; r < P.n_rows; ++r) {
    G.gstore(r);
    G.vstore(r);
  }
  o << "    }\n    }\n";
  if (nd && !skip_con) {
    o << "    __syncthreads();\n"
      << "    const unsigned valid = (unsigned)((hi - base) < " << tile << "ull ? (hi - base) : " << tile << "ull);\n"
      << "    T totq[" << ndpt << "];\n"
      << "#pragma unroll 1\n"
      << "    for (unsigned q = 0; q < " << ndpt << "u; ++q) {\n"
      << "      const unsigned d = q * " << cfg.block << "u + tid;\n"
      << "      T tot = 0;\n"
      << "      if (d < " << nd << "u)\n"
      << "      for (unsigned t = toff[d]; t < toff[d + 1]; ++t) {\n"
      << "        const TermC tm = terms[t];\n"
      << "        const T* ga = sG + tm.a * " << ld << "u;\n"
      << "        T p0 = 0, p1 = 0, p2 = 0, p3 = 0;\n"
      << "        unsigned j = 0;\n"
      << "        if (tm.kind == 0) {\n"
      << "          if (tm.f == 0xffffffffu) {\n"
      << "            for (; j + 4 <= valid; j += 4) { p0 += ga[j]; p1 += ga[j + 1]; p2 += ga[j + 2]; p3 += ga[j + 3]; }\n"
      << "            for (; j < valid; ++j) p0 += ga[j];\n"
      << "          } else {\n"
      << "            const T* vf = sV + tm.f * " << ld << "u;\n"
      << "            for (; j + 4 <= valid; j += 4) { p0 += ga[j] * vf[j]; p1 += ga[j + 1] * vf[j + 1]; p2 += ga[j + 2] * vf[j + 2]; p3 += ga[j + 3] * vf[j + 3]; }\n"
      << "            for (; j < valid; ++j) p0 += ga[j] * vf[j];\n"
      << "          }\n"
      << "        } else {\n"
      << "          const int* ix = idx + (unsigned long long)tm.f * batch + base;\n"
      << "          for (; j < valid; ++j) p0 += ix[j] == tm.row ? ga[j] : (T)0;\n"
      << "        }\n"
      << "        tot += (T)tm.coef * ((p0 + p1) + (p2 + p3));\n"
      << "      }\n"
      << "      totq[q] = tot;\n"
      << "    }\n";
    for (std::size_t bi = 0; bi < dbs.size(); ++bi) {
      const DB& b = dbs[bi];
      const std::string A = "cDG" + std::to_string(bi);
      o << "    // dense weight gradient " << b.nj << "x" << b.nk << ": register-tiled outer products over samples\n"
        << "    if (tid < " << b.nb * b.c << "u) {\n"
        << "      const unsigned bb = tid % " << b.nb << "u, c = tid / " << b.nb << "u;\n"
        << "      const unsigned j0 = (bb / " << b.bk << "u) * 4u, k0 = (bb % " << b.bk << "u) * 4u;\n"
        << "      const unsigned s0 = c * valid / " << b.c << "u, s1 = (c + 1u) * valid / " << b.c << "u;\n"
        << "      unsigned ar[4], fr[4];\n"
        << "#pragma unroll\n"
        << "      for (int u = 0; u < 4; ++u) {\n"
        << "        ar[u] = " << A << "[min(j0 + u, " << b.nj - 1 << "u)] * " << ld << "u;\n"
        << "        fr[u] = " << A << "[" << b.nj << "u + min(k0 + u, " << b.nk - 1 << "u)] * " << ld << "u;\n"
        << "      }\n"
        << "      T a4[4][4];\n"
        << "#pragma unroll\n"
        << "      for (int u = 0; u < 4; ++u)\n"
        << "#pragma unroll\n"
        << "        for (int v = 0; v < 4; ++v) a4[u][v] = 0;\n"
        << "      for (unsigned j = s0; j < s1; ++j) {\n"
        << "        T av[4], fv[4];\n"
        << "#pragma unroll\n"
        << "        for (int u = 0; u < 4; ++u) { av[u] = sG[ar[u] + j]; fv[u] = sV[fr[u] + j]; }\n"
        << "#pragma unroll\n"
        << "        for (int u = 0; u < 4; ++u)\n"
        << "#pragma unroll\n"
        << "          for (int v = 0; v < 4; ++v) a4[u][v] += av[u] * fv[v];\n"
        << "      }\n"
        << "#pragma unroll\n"
        << "      for (int u = 0; u < 4; ++u)\n"
        << "#pragma unroll\n"
        << "        for (int v = 0; v < 4; ++v)\n"
        << "          if (j0 + u < " << b.nj << "u && k0 + v < " << b.nk << "u)\n"
        << "            sS[c * " << b.nj * b.nk << "u + (j0 + u) * " << b.nk << "u + k0 + v] = a4[u][v];\n"
        << "    }\n"
        << "    __syncthreads();\n"
        << "    for (unsigned q = tid; q < " << b.nj * b.nk << "u; q += " << cfg.block << "u) {\n"
        << "      T t = 0;\n"
        << "      for (unsigned c = 0; c < " << b.c << "u; ++c) t += sS[c * " << b.nj * b.nk << "u + q];\n"
        << "      sDW[" << b.dest0 << "u + q] = t;\n"
        << "    }\n"
        << "    __syncthreads();\n";
    }
    o << "#pragma unroll 1\n"
      << "    for (unsigned q = 0; q < " << ndpt << "u; ++q) {\n"
      << "      const unsigned d = q * " << cfg.block << "u + tid;\n"
      << "      if (d >= " << nd << "u) break;\n"
      << "      const T tot = totq[q]" << (dense ? " + sDW[d]" : "") << ";\n";
    if (reg_acc) o << "      acc[q] += tot;\n";
    else o << "      T* dst = partial + (unsigned long long)d * grid_rows + blockIdx.x;\n"
           << "      *dst = (base == lo) ? tot : *dst + tot;\n";
    o << "    }\n    __syncthreads();\n";
  }
  o << "  }\n";
  if (reg_acc && nd)
    o << "  for (int q = 0; q < " << ndpt << "; ++q) { const unsigned d = q * " << cfg.block << "u + tid;\n"
      << "    if (d < " << nd << "u) partial[(unsigned long long)d * grid_rows + blockIdx.x] = acc[q]; }\n";
  o << fc.tail << "}\n" << fc.epi;
  return o.str();
}

// ---------------------------------------------------------------------------
// Grouped specialisation: G lanes (8 / 16 / 32) per sample.  Lane q of the
// group owns neuron q of every dense layer (forward value, activation,
// adjoint), so one sample's layers run G-wide instead of serially in one
// thread; per-lane state is a handful of registers, which raises the number
// of resident warps.  Layer vectors are exchanged through a per-sample
// shared-memory buffer (broadcast reads); weights sit in shared memory in
// both orientations so every lane access is conflict-free.  Weight and bias
// gradients accumulate in the owner lanes' registers across all samples the
// warp processes (no per-tile contraction), then a fixed-order block
// reduction writes the per-CTA partials.  Everything that is not a dense
// layer (inputs, loss glue) is emitted exactly as in generate(), replicated
// across the group's lanes.
// Dense-chain analysis shared by the grouped and the DMMA forms: every
// dense layer reads either per-sample scalar rows or exactly the outputs of
// one earlier layer; the loss glue reads layer outputs but never a
// pre-activation of a fused layer; every batch term is a layer's weight
// block, a layer's bias (sum of its z adjoint) or a product of scalar rows.
struct DenseGroup {
  const tgc::Dense* D = nullptr;
  bool xvec = false;               // x = outputs of dense[src]
  int src = -1;
  std::vector<std::uint32_t> xr;   // x rows
  std::uint32_t crow = 0;          // consumed output rows (act rows if fused, else z rows)
  std::uint32_t dw0 = kNone;       // weight-gradient dest block
  std::vector<std::uint32_t> bdest;  // bias dest per output (or kNone)
  std::vector<double> bcoef;
  unsigned wf = 0, wb = 0, bb = 0, xo = 0, xg = 0;   // generator scratch (shared-memory offsets)
  bool has_bias() const {
    for (auto d : bdest) if (d != kNone) return true;
    return false;
  }
  bool unit_bias() const {
    for (auto c : bcoef) if (c != 1.0) return false;
    return true;
  }
};
struct DensePlan {
  std::vector<DenseGroup> gr;
  std::vector<int> rg, rj, zg, zj;  // row -> (group, output) for consumed rows / z rows
  std::vector<char> internal;       // pre-activation of a fused layer
  std::vector<unsigned> sdests;     // dests over scalar rows only
};

bool plan_dense(const tgc::Program& P, DensePlan& pl, std::string& why) {
  auto no = [&](const std::string& w) { why = w; return false; };
  if (P.root_row == kNone) return no("root is sample-invariant");
  if (P.dense.empty()) return no("no dense layers");
  if (!P.sgather.empty()) return no("slot gathers");
  const unsigned nd = static_cast<unsigned>(P.dest_uv.size());
  const std::size_t ng = P.dense.size();
  auto& gr = pl.gr;
  auto& rg = pl.rg;
  auto& rj = pl.rj;
  auto& zg = pl.zg;
  auto& zj = pl.zj;
  auto& internal = pl.internal;
  gr.assign(ng, {});
  rg.assign(P.n_rows, -1);
  rj.assign(P.n_rows, -1);
  zg.assign(P.n_rows, -1);
  zj.assign(P.n_rows, -1);
  internal.assign(P.n_rows, 0);
  for (std::size_t i = 0; i < ng; ++i) {
    const tgc::Dense& D = P.dense[i];
    gr[i].D = &D;
    gr[i].crow = D.act_op ? D.act_row : D.out_row;
    gr[i].bdest.assign(D.n_out, kNone);
    gr[i].bcoef.assign(D.n_out, 1.0);
    for (std::uint32_t j = 0; j < D.n_out; ++j) {
      rg[gr[i].crow + j] = static_cast<int>(i);
      rj[gr[i].crow + j] = static_cast<int>(j);
      zg[D.out_row + j] = static_cast<int>(i);
      zj[D.out_row + j] = static_cast<int>(j);
      if (D.act_op) internal[D.out_row + j] = 1;
    }
  }
  for (std::size_t i = 0; i < ng; ++i) {
    const tgc::Dense& D = *gr[i].D;
    bool any = false;
    for (std::uint32_t k = 0; k < D.n_in; ++k) {
      const std::uint32_t op = P.opnd[D.x_opnd + k];
      if ((op >> kModeShift) != tgc::kSlot) return no("dense x operand is not a per-sample row");
      const std::uint32_t r = op & kIndexMask;
      if (internal[r]) return no("pre-activation read by another layer");
      gr[i].xr.push_back(r);
      any = any || rg[r] >= 0;
    }
    if (any) {
      const int src = rg[gr[i].xr[0]];
      if (P.dense[src].n_out != D.n_in) return no("dense x is part of a layer");
      for (std::uint32_t k = 0; k < D.n_in; ++k)
        if (rg[gr[i].xr[k]] != src || rj[gr[i].xr[k]] != static_cast<int>(k)) return no("dense x mixes rows");
      gr[i].xvec = true;
      gr[i].src = src;
    } else if (D.n_in > 32) {
      return no("too many scalar inputs to one dense layer");
    }
  }
  for (const Instr& in : P.fwd) {
    if (in.kind != tgc::kNode) continue;
    for (std::uint32_t j = 0; j < in.nops; ++j) {
      const std::uint32_t op = P.opnd[in.opnd + j];
      if ((op >> kModeShift) == tgc::kSlot && internal[op & kIndexMask]) return no("pre-activation read outside its layer");
    }
  }
  if (rg[P.root_row] >= 0 || internal[P.root_row]) return no("root is a dense-layer row");
  for (std::size_t b = 0; b < P.dgrad.size(); ++b) {
    const tgc::DenseGrad& dg = P.dgrad[b];
    const std::uint32_t a0 = P.dg_rows[dg.arow_off];
    bool found = false;
    for (std::size_t i = 0; i < ng && !found; ++i)
      if (gr[i].D->out_row == a0 && gr[i].D->n_out == dg.n_out && gr[i].D->n_in == dg.n_in) {
        gr[i].dw0 = dg.dest0;
        found = true;
      }
    if (!found) return no("weight-gradient block without its layer");
  }
  std::vector<char> covered(nd, 0);
  for (const auto& g : gr)
    if (g.dw0 != kNone)
      for (std::uint32_t q = 0; q < g.D->n_out * g.D->n_in; ++q) covered[g.dw0 + q] = 1;
  pl.sdests.clear();
  auto scalar_row = [&](std::uint32_t r) { return rg[r] < 0 && zg[r] < 0; };
  for (unsigned d = 0; d < nd; ++d) {
    if (covered[d]) continue;
    if (P.dest_dense[d]) return no("dense gradient dest outside its block");
    const std::uint32_t t0 = P.term_off[d], t1 = P.term_off[d + 1];
    const tgc::Term& t = P.terms[t0];
    if (t1 - t0 == 1 && t.kind == 0 && t.f == kNone && zg[t.a] >= 0) {
      DenseGroup& g = gr[zg[t.a]];
      if (g.bdest[zj[t.a]] != kNone) return no("two bias dests on one neuron");
      g.bdest[zj[t.a]] = d;
      g.bcoef[zj[t.a]] = t.coef;
      continue;
    }
    for (std::uint32_t u = t0; u < t1; ++u) {
      const tgc::Term& tu = P.terms[u];
      if (tu.kind != 0 || !scalar_row(tu.a) || (tu.f != kNone && !scalar_row(tu.f)))
        return no("batch term over a dense-layer row");
    }
    pl.sdests.push_back(d);
  }
  if (pl.sdests.size() > 32) return no("too many scalar gradient destinations");
  return true;
}

std::string generate_grouped(const tgc::Program& P, const JitConfig& cfg, unsigned& G_out, unsigned& spb,
                             std::size_t& smem_bytes, std::string& why) {
  const bool f64 = P.dtype == TG_F64;
  const std::size_t ts = f64 ? 8 : 4;
  auto no = [&](const std::string& w) { why = w; return std::string(); };
  DensePlan plan;
  if (!plan_dense(P, plan, why)) return std::string();
  const unsigned nd = static_cast<unsigned>(P.dest_uv.size());
  unsigned maxw = 1;
  for (const auto& D : P.dense) maxw = std::max(maxw, D.n_out);
  if (maxw > 32) return no("dense layer wider than a warp");
  const unsigned G = maxw <= 8 ? 8 : maxw <= 16 ? 16 : 32;
  const unsigned SPW = 32 / G, WPB = cfg.block / 32;
  using Grp = DenseGroup;
  const std::size_t ng = P.dense.size();
  auto& gr = plan.gr;
  auto& rg = plan.rg;
  auto& zg = plan.zg;
  auto& sdests = plan.sdests;

  // shared memory (elements): weights, per-sample exchange buffers, block reduction
  unsigned off = 0, xs = 0;
  for (auto& g : gr) {
    g.wf = off;
    off += g.D->n_in * G;
    if (g.xvec) { g.wb = off; off += g.D->n_out * G; }
    g.bb = off;
    off += G;
    g.xo = xs;
    xs += G;
    if (g.xvec) { g.xg = xs; xs += G; }
  }
  const std::size_t elems = std::size_t(off) + std::size_t(WPB) * SPW * xs + std::size_t(WPB) * nd;
  if (elems * ts > 160 * 1024) return no("shared memory");
  smem_bytes = elems * ts;
  G_out = G;
  spb = WPB * SPW;

  Gen Gn(P, cfg);
  Gn.su = cfg.fuse;
  const FuseCode fc = cfg.fuse ? fuse_code(P, cfg, "") : FuseCode{};
  // where the layer tables are staged from: params / consts straight from
  // global (those loads overlap sU's), uniform nodes from sU after the program
  auto tsrc = [&](std::uint32_t uv0, std::uint32_t cnt) -> std::string {
    if (!cfg.fuse) return "UVg[";
    if (uv0 + cnt <= P.n_params) return "A.params[";
    if (uv0 >= P.uv_const_base) return "(A.consts - " + std::to_string(P.uv_const_base) + ")[";
    return "sU[";
  };
  bool late = false;
  for (const auto& D : P.dense) {
    late = late || tsrc(D.w_uv, D.n_out * D.n_in) == "sU[";
    if (D.b_uv != kNone) late = late || tsrc(D.b_uv, D.n_out) == "sU[";
  }

  Gn.vslot.assign(P.n_rows, -1);
  Gn.gslot.assign(P.n_rows, -1);
  Gn.vsm.assign(P.n_rows, 0);
  Gn.gsm.assign(P.n_rows, 0);
  Gn.vov.assign(P.n_rows, "");
  Gn.gov.assign(P.n_rows, "");
  Gn.gj.assign(P.n_rows, -1);
  for (std::size_t i = 0; i < ng; ++i)
    for (std::uint32_t j = 0; j < gr[i].D->n_out; ++j) {
      const std::uint32_t r = gr[i].crow + j;
      Gn.vov[r] = "sX[" + std::to_string(gr[i].xo + j) + "u]";
      Gn.gov[r] = "gh" + std::to_string(i);
      Gn.gj[r] = static_cast<int>(j);
    }
  std::ostringstream& o = Gn.o;
  const std::string Gs = std::to_string(G) + "u";
  o << "typedef " << (f64 ? "double" : "float") << " T;\n" << kMath << kPrelude << fc.decl;
  if (cfg.const_uv && !cfg.fuse) o << "__constant__ T cUV[" << std::max<std::uint32_t>(1, P.n_uv) << "];\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << cfg.block;
  if (cfg.min_blocks) o << ", " << cfg.min_blocks;
  o << ") tg_jit_tape(const JitArgs A) {\n" << kArgAliases
    << (cfg.fuse ? fuse_wait(cfg.coop) : std::string())
    << (late ? fc.pro : fc.pro_load)
    << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  T* sm = reinterpret_cast<T*>(smem_raw);\n"
    << "  T* sRed = sm + " << off + WPB * SPW * xs << "u;\n"
    << "  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;\n"
    << "  const unsigned q = lane & " << G - 1 << "u, slot = lane / " << Gs << ";\n"
    << "  T* sX = sm + " << off << "u + (warp * " << SPW << "u + slot) * " << xs << "u;\n"
    << "  (void)toff; (void)terms; (void)cand; (void)idx; (void)in; (void)err_key;\n";
  // weights: forward / scalar-x layout [k][j] (lane j), vector-x backward layout [j][k] (lane k)
  for (const auto& g : gr) {
    const tgc::Dense& D = *g.D;
    o << "  for (unsigned e = tid; e < " << D.n_in * G << "u; e += " << cfg.block << "u) { const unsigned k = e / " << Gs
      << ", j = e % " << Gs << "; sm[" << g.wf << "u + e] = j < " << D.n_out << "u ? " << tsrc(D.w_uv, D.n_out * D.n_in) << D.w_uv << "u + j * "
      << D.n_in << "u + k] : (T)0; }\n";
    if (g.xvec)
      o << "  for (unsigned e = tid; e < " << D.n_out * G << "u; e += " << cfg.block << "u) { const unsigned j = e / "
        << Gs << ", k = e % " << Gs << "; sm[" << g.wb << "u + e] = k < " << D.n_in << "u ? " << tsrc(D.w_uv, D.n_out * D.n_in) << D.w_uv
        << "u + j * " << D.n_in << "u + k] : (T)0; }\n";
    o << "  for (unsigned e = tid; e < " << Gs << "; e += " << cfg.block << "u) sm[" << g.bb << "u + e] = ";
    if (D.b_uv != kNone) o << "e < " << D.n_out << "u ? " << tsrc(D.b_uv, D.n_out) << D.b_uv << "u + e] : (T)0;\n";
    else o << "(T)0;\n";
  }
  o << "  for (unsigned e = tid; e < " << WPB * nd << "u; e += " << cfg.block << "u) sRed[e] = (T)0;\n"
    << "  __syncthreads();\n" << (late ? std::string() : fc.pro_prog);
  // accumulators
  for (std::size_t i = 0; i < ng; ++i) {
    const Grp& g = gr[i];
    if (g.dw0 != kNone) {
      const unsigned na = g.xvec ? g.D->n_out : g.D->n_in;
      for (unsigned c = 0; c < na; ++c) o << "  T aw" << i << "_" << c << " = (T)0;\n";
    }
    bool anyb = false, unit = true;
    for (std::uint32_t j = 0; j < g.D->n_out; ++j) {
      anyb = anyb || g.bdest[j] != kNone;
      unit = unit && g.bcoef[j] == 1.0;
    }
    if (anyb) {
      o << "  T ab" << i << " = (T)0;\n";
      if (!unit) {
        o << "  T bc" << i << " = (T)0;\n";
        for (std::uint32_t j = 0; j < g.D->n_out; ++j)
          o << "  if (q == " << j << "u) bc" << i << " = " << lit(g.bcoef[j], f64) << ";\n";
      }
    }
  }
  for (std::size_t e = 0; e < sdests.size(); ++e) o << "  T as" << e << " = (T)0;\n";

  o << "  const unsigned long long TW = (unsigned long long)gridDim.x * " << WPB << "u;\n"
    << "  for (unsigned long long base = ((unsigned long long)blockIdx.x * " << WPB << "u + warp) * " << SPW
    << "u; base < batch; base += TW * " << SPW << "u) {\n"
    << "    const unsigned long long sa = base + slot;\n"
    << "    const bool active = sa < batch;\n"
    << "    const unsigned long long s = active ? sa : batch - 1;\n"
    << "    {\n";
  auto group_fwd = [&](std::size_t i) {
    const Grp& g = gr[i];
    const tgc::Dense& D = *g.D;
    const std::string I = std::to_string(i);
    o << "      // dense " << I << ": " << D.n_out << " x " << D.n_in << (g.xvec ? " (x from dense " + std::to_string(g.src) + ")" : " (scalar x)") << "\n";
    std::vector<std::string> x(D.n_in);
    for (std::uint32_t k = 0; k < D.n_in; ++k)
      x[k] = g.xvec ? "sX[" + std::to_string(gr[g.src].xo + k) + "u]" : Gn.V(g.xr[k]);
    o << "      T zz" << I << " = sm[" << g.bb << "u + q];";
    for (std::uint32_t k = 0; k < D.n_in; ++k)
      o << " zz" << I << " += " << x[k] << " * sm[" << g.wf + k * G << "u + q];";
    o << "\n";
    if (D.act_op) o << "      const T hh" << I << " = " << Gn.act_f(D.act_op, "zz" + I) << ";\n";
    o << "      sX[" << g.xo << "u + q] = " << (D.act_op ? "hh" : "zz") << I << ";\n      __syncwarp();\n";
  };
  auto group_bwd = [&](std::size_t i) {
    const Grp& g = gr[i];
    const tgc::Dense& D = *g.D;
    const std::string I = std::to_string(i);
    o << "      // dense " << I << " reverse\n";
    o << "      T gz" << I << " = " << (D.act_op ? Gn.act_b(D.act_op, "gh" + I, "hh" + I, "zz" + I) : "gh" + I) << ";\n";
    if (D.n_out < G) o << "      if (q >= " << D.n_out << "u) gz" << I << " = (T)0;\n";
    bool anyb = false, unit = true;
    for (std::uint32_t j = 0; j < D.n_out; ++j) {
      anyb = anyb || g.bdest[j] != kNone;
      unit = unit && g.bcoef[j] == 1.0;
    }
    if (anyb) o << "      if (active) ab" << I << " += " << (unit ? "gz" + I : "bc" + I + " * gz" + I) << ";\n";
    if (g.xvec) {
      const Grp& sg = gr[g.src];
      const std::string xk = sg.D->act_op ? "hh" + std::to_string(g.src) : "zz" + std::to_string(g.src);
      o << "      sX[" << g.xg << "u + q] = gz" << I << ";\n      __syncwarp();\n"
        << "      { T dx = (T)0;\n";
      for (std::uint32_t j = 0; j < D.n_out; ++j) {
        o << "        { const T gj = sX[" << g.xg + j << "u]; dx += gj * sm[" << g.wb + j * G << "u + q];";
        if (g.dw0 != kNone) o << " if (active) aw" << I << "_" << j << " += gj * " << xk << ";";
        o << " }\n";
      }
      o << "        gh" << g.src << " += dx; }\n";
    } else {
      Instr pseudo{};
      pseudo.opnd = D.x_opnd;
      for (std::uint32_t k = 0; k < D.n_in; ++k) {
        const std::string pk = "px" + std::to_string(Gn.tmp++);
        o << "      T " << pk << " = gz" << I << " * sm[" << g.wf + k * G << "u + q];";
        for (unsigned m = G / 2; m >= 1; m /= 2)
          o << " " << pk << " += __shfl_xor_sync(0xffffffffu, " << pk << ", " << m << ");";
        o << "\n";
        if (g.dw0 != kNone) o << "      if (active) aw" << I << "_" << k << " += gz" << I << " * " << Gn.V(g.xr[k]) << ";\n";
        Gn.push(pseudo, k, pk);
      }
    }
  };
  for (const Instr& in : P.fwd) {
    if (in.kind == tgc::kDense) group_fwd(in.aux);
    else Gn.forward(in);
  }
  o << "      if (loss && active && q == 0u) loss[s] = " << Gn.V(P.root_row) << ";\n";
  for (std::size_t i = 0; i < ng; ++i) o << "      T gh" << i << " = (T)0;\n";
  for (std::uint32_t r : P.zero_rows)
    if (rg[r] < 0 && zg[r] < 0) o << "      T " << Gn.g(r) << " = (T)0;\n";
  o << "      T " << Gn.g(P.root_row) << " = (T)1;\n";
  for (const Instr& in : P.bwd) {
    if (in.kind == tgc::kDense) group_bwd(in.aux);
    else Gn.reverse(in);
  }
  for (std::uint32_t c = 0; c < P.n_inputs; ++c) {
    const std::uint32_t r = P.input_rows[c];
    if (r != kNone) o << "      if (igrad && active && q == 0u) igrad[" << c << "ull * batch + s] = " << Gn.Gx(r) << ";\n";
  }
  if (!sdests.empty()) {
    o << "      if (active) {\n";
    for (std::size_t e = 0; e < sdests.size(); ++e) {
      const unsigned d = sdests[e];
      for (std::uint32_t u = P.term_off[d]; u < P.term_off[d + 1]; ++u) {
        const tgc::Term& t = P.terms[u];
        o << "        as" << e << " += " << lit(t.coef, f64) << " * " << Gn.Gx(t.a);
        if (t.f != kNone) o << " * " << Gn.V(t.f);
        o << ";\n";
      }
    }
    o << "      }\n";
  }
  o << "    }\n    __syncwarp();\n  }\n";
  // reduction: sample slots of a warp (lanes q, q+G, ...), then warps in fixed order
  auto slot_sum = [&](const std::string& a) {
    for (unsigned m = G; m < 32; m *= 2) o << "  " << a << " += __shfl_xor_sync(0xffffffffu, " << a << ", " << m << ");\n";
  };
  for (std::size_t i = 0; i < ng; ++i) {
    const Grp& g = gr[i];
    const std::string I = std::to_string(i);
    if (g.dw0 != kNone) {
      const unsigned na = g.xvec ? g.D->n_out : g.D->n_in;
      for (unsigned c = 0; c < na; ++c) slot_sum("aw" + I + "_" + std::to_string(c));
    }
    bool anyb = false;
    for (auto d : g.bdest) anyb = anyb || d != kNone;
    if (anyb) slot_sum("ab" + I);
  }
  for (std::size_t e = 0; e < sdests.size(); ++e) slot_sum("as" + std::to_string(e));
  o << "  if (slot == 0u) {\n    T* red = sRed + warp * " << nd << "u;\n";
  for (std::size_t i = 0; i < ng; ++i) {
    const Grp& g = gr[i];
    const tgc::Dense& D = *g.D;
    const std::string I = std::to_string(i);
    if (g.dw0 != kNone) {
      if (g.xvec) {
        o << "    if (q < " << D.n_in << "u) {";
        for (std::uint32_t j = 0; j < D.n_out; ++j)
          o << " red[" << g.dw0 + j * D.n_in << "u + q] = aw" << I << "_" << j << ";";
        o << " }\n";
      } else {
        o << "    if (q < " << D.n_out << "u) {";
        for (std::uint32_t k = 0; k < D.n_in; ++k)
          o << " red[" << g.dw0 + k << "u + q * " << D.n_in << "u] = aw" << I << "_" << k << ";";
        o << " }\n";
      }
    }
    for (std::uint32_t j = 0; j < D.n_out; ++j)
      if (g.bdest[j] != kNone) o << "    if (q == " << j << "u) red[" << g.bdest[j] << "u] = ab" << I << ";\n";
  }
  for (std::size_t e = 0; e < sdests.size(); ++e) o << "    if (q == 0u) red[" << sdests[e] << "u] = as" << e << ";\n";
  o << "  }\n  __syncthreads();\n"
    << "  for (unsigned d = tid; d < " << nd << "u; d += " << cfg.block << "u) {\n"
    << "    T t = (T)0;\n"
    << "    for (unsigned w = 0; w < " << WPB << "u; ++w) t += sRed[w * " << nd << "u + d];\n"
    << "    partial[(unsigned long long)d * grid_rows + blockIdx.x] = t;\n  }\n" << fc.tail << "}\n" << fc.epi;
  return o.str();
}

// ---------------------------------------------------------------------------
// FP64 tensor-core form: mma.sync m8n8k4 f64 (DMMA).  A warp runs 8 samples
// at a time; lane (g, c) = (lane / 4, lane % 4) belongs to sample g.  The
// outputs of a dense layer live in the accumulator (D) layout: lane (g, c)
// holds neurons 8u + 2c + {0, 1} of sample g for every 8-wide tile u.  The
// next layer's A operand is read straight from those registers by ordering
// its k axis as k = 8 (t / 2) + 2c + (t % 2) for k-step t; the weights'
// B fragments are staged in shared memory in the same order, so activations
// never move between layers.  Biases of scalar-input layers ride in A as a
// ones column; those of chained layers initialise the accumulator.  Weight
// and bias gradients are a DMMA contraction over the samples of each step
// through a per-warp transpose buffer, accumulated in registers across the
// warp's samples, then reduced over the block in a fixed order.  The loss
// glue runs replicated on the 4 lanes of each sample, as in generate().
std::string generate_dmma(const tgc::Program& P, const JitConfig& cfg, unsigned& spb, std::size_t& smem_bytes,
                          std::string& why) {
  auto no = [&](const std::string& w) { why = w; return std::string(); };
  if (P.dtype != TG_F64) return no("DMMA form is fp64 only");
  DensePlan plan;
  if (!plan_dense(P, plan, why)) return std::string();
  const unsigned nd = static_cast<unsigned>(P.dest_uv.size());
  const unsigned WPB = cfg.block / 32;
  auto& gr = plan.gr;
  auto& rg = plan.rg;
  auto& zg = plan.zg;
  auto& sdests = plan.sdests;
  const std::size_t ng = gr.size();
  for (const auto& g : gr)
    if (g.D->n_out > 64 || g.D->n_in > 64) return no("dense layer wider than 64");
  auto tiles = [](unsigned n) { return (n + 7) / 8; };
  auto ld16 = [](unsigned n) { unsigned l = n; while (l % 16 != 4) ++l; return l; };   // conflict-free fragment loads
  struct Geo { unsigned ntO = 0, ks = 0, ntX = 0, ntK = 0, kin = 0; bool fb = false, contract = false; unsigned bf = 0, bk = 0, bb = 0; };
  std::vector<Geo> ge(ng);
  unsigned off = 0, maxg = 0, maxx = 0;
  for (std::size_t i = 0; i < ng; ++i) {
    const tgc::Dense& D = *gr[i].D;
    Geo& q = ge[i];
    q.ntO = tiles(D.n_out);
    q.fb = D.b_uv != kNone;
    q.ks = gr[i].xvec ? 2 * tiles(D.n_in) : (D.n_in + (q.fb ? 1 : 0) + 3) / 4;
    q.ntX = tiles(D.n_in);
    q.contract = gr[i].dw0 != kNone || gr[i].has_bias();
    q.kin = D.n_in + (gr[i].has_bias() ? 1 : 0);
    q.ntK = tiles(q.kin);
    q.bf = off;
    off += q.ks * q.ntO * 32;
    q.bk = off;
    off += 2 * q.ntO * q.ntX * 32;
    q.bb = off;
    off += 8 * q.ntO;
    if (q.contract) {
      maxg = std::max(maxg, 8 * q.ntO);
      maxx = std::max(maxx, 8 * q.ntK);
    }
  }
  const unsigned ldg = maxg ? ld16(maxg) : 0, ldx = maxx ? ld16(maxx) : 0;
  const unsigned per_warp = 8 * (ldg + ldx);
  const std::size_t elems = std::size_t(off) + std::size_t(WPB) * per_warp + std::size_t(WPB) * nd;
  if (elems * 8 > 160 * 1024) return no("shared memory");
  smem_bytes = elems * 8;
  spb = WPB * 8;

  // glue reads of layer outputs are materialised once (lane shuffle from the owner)
  std::vector<char> needv(P.n_rows, 0);
  for (const Instr& in : P.fwd) {
    if (in.kind != tgc::kNode) continue;
    for (std::uint32_t j = 0; j < in.nops; ++j) {
      const std::uint32_t op = P.opnd[in.opnd + j];
      if ((op >> kModeShift) == tgc::kSlot && rg[op & kIndexMask] >= 0) needv[op & kIndexMask] = 1;
    }
  }
  for (unsigned d : sdests)
    for (std::uint32_t u = P.term_off[d]; u < P.term_off[d + 1]; ++u)
      if (P.terms[u].f != kNone && rg[P.terms[u].f] >= 0) needv[P.terms[u].f] = 1;

  Gen Gn(P, cfg);
  Gn.su = cfg.fuse;
  const FuseCode fc = cfg.fuse ? fuse_code(P, cfg, "") : FuseCode{};
  // where the layer tables are staged from: params / consts straight from
  // global (those loads overlap sU's), uniform nodes from sU after the program
  auto tsrc = [&](std::uint32_t uv0, std::uint32_t cnt) -> std::string {
    if (!cfg.fuse) return "UVg[";
    if (uv0 + cnt <= P.n_params) return "A.params[";
    if (uv0 >= P.uv_const_base) return "(A.consts - " + std::to_string(P.uv_const_base) + ")[";
    return "sU[";
  };
  bool late = false;
  for (const auto& D : P.dense) {
    late = late || tsrc(D.w_uv, D.n_out * D.n_in) == "sU[";
    if (D.b_uv != kNone) late = late || tsrc(D.b_uv, D.n_out) == "sU[";
  }

  Gn.vslot.assign(P.n_rows, -1);
  Gn.gslot.assign(P.n_rows, -1);
  Gn.vsm.assign(P.n_rows, 0);
  Gn.gsm.assign(P.n_rows, 0);
  Gn.vov.assign(P.n_rows, "");
  Gn.gov.assign(P.n_rows, "");
  Gn.gcond.assign(P.n_rows, "");
  if (!std::getenv("TG_TANH")) Gn.tanh_fn = "tg_tanh_fp64";   // keeps the XU queue off the DMMA kernel's path
  Gn.gj.assign(P.n_rows, -1);
  auto nm = [](const char* p, std::size_t i, unsigned u, unsigned e) {
    return std::string(p) + std::to_string(i) + "_" + std::to_string(u) + "_" + std::to_string(e);
  };
  auto outn = [&](std::size_t i, unsigned u, unsigned e) { return nm(gr[i].D->act_op ? "dh" : "dz", i, u, e); };
  for (std::size_t i = 0; i < ng; ++i)
    for (std::uint32_t j = 0; j < gr[i].D->n_out; ++j) {
      const std::uint32_t r = gr[i].crow + j;
      Gn.vov[r] = "bv" + std::to_string(r);
      Gn.gov[r] = nm("gh", i, j / 8, j % 2);
      Gn.gcond[r] = "c == " + std::to_string((j % 8) / 2) + "u";
    }
  std::ostringstream& o = Gn.o;
  o << "typedef double T;\n" << kMath << kPrelude << fc.decl
    << "__device__ __forceinline__ void tg_dmma(double& d0, double& d1, double a, double b) {\n"
    << "  asm(\"mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\"\n"
    << "      : \"+d\"(d0), \"+d\"(d1) : \"d\"(a), \"d\"(b));\n}\n";
  if (cfg.const_uv && !cfg.fuse) o << "__constant__ T cUV[" << std::max<std::uint32_t>(1, P.n_uv) << "];\n";
  for (std::size_t i = 0; i < ng; ++i) {
    if (!gr[i].has_bias()) continue;
    o << "__constant__ unsigned cBD" << i << "[" << gr[i].D->n_out << "] = {";
    for (std::uint32_t j = 0; j < gr[i].D->n_out; ++j) o << (j ? ", " : "") << gr[i].bdest[j] << "u";
    o << "};\n";
    if (!gr[i].unit_bias()) {
      o << "__constant__ T cBC" << i << "[" << gr[i].D->n_out << "] = {";
      for (std::uint32_t j = 0; j < gr[i].D->n_out; ++j) o << (j ? ", " : "") << lit(gr[i].bcoef[j], true);
      o << "};\n";
    }
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << cfg.block;
  if (cfg.min_blocks) o << ", " << cfg.min_blocks;
  o << ") tg_jit_tape(const JitArgs A) {\n" << kArgAliases
    << (cfg.fuse ? fuse_wait(cfg.coop) : std::string())
    << (late ? fc.pro : fc.pro_load)
    << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  T* sm = reinterpret_cast<T*>(smem_raw);\n"
    << "  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;\n"
    << "  const unsigned g = lane >> 2, c = lane & 3u;\n"
    << "  T* gzb = sm + " << off << "u + warp * " << per_warp << "u;\n"
    << "  T* xb = gzb + " << 8 * ldg << "u;\n"
    << "  T* sRed = sm + " << off + WPB * per_warp << "u;\n"
    << "  (void)toff; (void)terms; (void)cand; (void)idx; (void)in; (void)err_key; (void)gzb; (void)xb;\n";
  // B fragments of every layer, in the lane order of mma.sync m8n8k4 (b0 = B[lane % 4][lane / 4])
  for (std::size_t i = 0; i < ng; ++i) {
    const tgc::Dense& D = *gr[i].D;
    const Geo& q = ge[i];
    const std::string W = std::to_string(D.w_uv) + "u", NI = std::to_string(D.n_in) + "u",
                      NO = std::to_string(D.n_out) + "u";
    o << "  for (unsigned e = tid; e < " << q.ks * q.ntO * 32 << "u; e += " << cfg.block << "u) {\n"
      << "    const unsigned t = e / " << q.ntO * 32 << "u, u = (e >> 5) % " << q.ntO << "u, L = e & 31u;\n"
      << "    const unsigned n = 8u * u + (L >> 2), cc = L & 3u;\n";
    if (gr[i].xvec)
      o << "    const unsigned k = 8u * (t >> 1) + 2u * cc + (t & 1u);\n"
        << "    sm[" << q.bf << "u + e] = (n < " << NO << " && k < " << NI << ") ? " << tsrc(D.w_uv, D.n_out * D.n_in) << W << " + n * " << NI << " + k] : (T)0;\n";
    else {
      o << "    const unsigned k = 4u * t + cc;\n"
        << "    T w = (T)0;\n"
        << "    if (n < " << NO << ") { if (k < " << NI << ") w = " << tsrc(D.w_uv, D.n_out * D.n_in) << W << " + n * " << NI << " + k];";
      if (q.fb) o << " else if (k == " << NI << ") w = " << tsrc(D.b_uv, D.n_out) << D.b_uv << "u + n];";
      o << " }\n    sm[" << q.bf << "u + e] = w;\n";
    }
    o << "  }\n"
      << "  for (unsigned e = tid; e < " << 2 * q.ntO * q.ntX * 32 << "u; e += " << cfg.block << "u) {\n"
      << "    const unsigned t = e / " << q.ntX * 32 << "u, u = (e >> 5) % " << q.ntX << "u, L = e & 31u;\n"
      << "    const unsigned n = 8u * u + (L >> 2), k = 8u * (t >> 1) + 2u * (L & 3u) + (t & 1u);\n"
      << "    sm[" << q.bk << "u + e] = (k < " << NO << " && n < " << NI << ") ? " << tsrc(D.w_uv, D.n_out * D.n_in) << W << " + k * " << NI << " + n] : (T)0;\n"
      << "  }\n";
    if (gr[i].xvec && q.fb)
      o << "  for (unsigned e = tid; e < " << 8 * q.ntO << "u; e += " << cfg.block << "u) sm[" << q.bb << "u + e] = e < "
        << NO << " ? " << tsrc(D.b_uv, D.n_out) << D.b_uv << "u + e] : (T)0;\n";
  }
  o << "  for (unsigned e = tid; e < " << WPB * nd << "u; e += " << cfg.block << "u) sRed[e] = (T)0;\n"
    << "  __syncthreads();\n" << (late ? std::string() : fc.pro_prog);
  for (std::size_t i = 0; i < ng; ++i)
    if (ge[i].contract)
      for (unsigned u = 0; u < ge[i].ntO; ++u)
        for (unsigned v = 0; v < ge[i].ntK; ++v)
          o << "  T aw" << i << "_" << u << "_" << v << "_0 = (T)0, aw" << i << "_" << u << "_" << v << "_1 = (T)0;\n";
  for (std::size_t e = 0; e < sdests.size(); ++e) o << "  T as" << e << " = (T)0;\n";
  // inputs of the next 8-sample step are loaded at the top of the current one
  // (register double buffer), so their latency hides behind a whole step
  std::vector<std::uint32_t> incols;
  for (const Instr& in : P.fwd)
    if (in.kind == tgc::kInputLoad) incols.push_back(in.aux);
  o << "  const unsigned long long TW = (unsigned long long)gridDim.x * " << WPB << "u;\n"
    << "  unsigned long long base = ((unsigned long long)blockIdx.x * " << WPB << "u + warp) * 8u;\n"
    << "  const unsigned long long s0 = base + g < batch ? base + g : batch - 1;\n";
  for (std::uint32_t col : incols) o << "  T pf" << col << " = in[" << col << "ull * batch + s0];\n";
  o << "  for (; base < batch; base += TW * 8u) {\n"
    << "    const unsigned long long sa = base + g;\n"
    << "    const bool active = sa < batch;\n"
    << "    const unsigned long long s = active ? sa : batch - 1;\n";
  for (std::uint32_t col : incols) o << "    const T in" << col << " = pf" << col << ";\n";
  o << "    {\n      const unsigned long long sn = base + TW * 8u + g < batch ? base + TW * 8u + g : batch - 1;\n";
  for (std::uint32_t col : incols) o << "      pf" << col << " = in[" << col << "ull * batch + sn];\n";
  o << "    }\n    {\n";
  auto group_fwd = [&](std::size_t i) {
    const DenseGroup& G = gr[i];
    const tgc::Dense& D = *G.D;
    const Geo& q = ge[i];
    const std::string I = std::to_string(i);
    o << "      // dense " << I << ": " << D.n_out << " x " << D.n_in << " on DMMA\n";
    for (unsigned u = 0; u < q.ntO; ++u)
      for (unsigned e = 0; e < 2; ++e) {
        o << "      T " << nm("dz", i, u, e) << " = ";
        if (G.xvec && q.fb) o << "sm[" << q.bb + 8 * u + e << "u + 2u * c];\n";
        else o << "(T)0;\n";
      }
    for (unsigned t = 0; t < q.ks; ++t) {
      std::string a;
      if (G.xvec) {
        a = outn(G.src, t / 2, t % 2);
      } else {
        auto X = [&](unsigned k) -> std::string {
          if (k < D.n_in) return Gn.V(G.xr[k]);
          return (k == D.n_in && q.fb) ? "(T)1" : "(T)0";
        };
        // lane c takes x[4t + c]: a chain of selects (a nested ?: becomes a jump table)
        a = "da" + std::to_string(Gn.tmp++);
        o << "      T " << a << " = " << X(4 * t + 3) << "; " << a << " = c == 2u ? " << X(4 * t + 2) << " : " << a << "; "
          << a << " = c == 1u ? " << X(4 * t + 1) << " : " << a << "; " << a << " = c == 0u ? " << X(4 * t) << " : " << a
          << ";\n";
      }
      for (unsigned u = 0; u < q.ntO; ++u)
        o << "      tg_dmma(" << nm("dz", i, u, 0) << ", " << nm("dz", i, u, 1) << ", " << a << ", sm["
          << q.bf + (t * q.ntO + u) * 32 << "u + lane]);\n";
    }
    if (D.act_op)
      for (unsigned u = 0; u < q.ntO; ++u)
        for (unsigned e = 0; e < 2; ++e)
          o << "      const T " << nm("dh", i, u, e) << " = " << Gn.act_f(D.act_op, nm("dz", i, u, e)) << ";\n";
    for (std::uint32_t j = 0; j < D.n_out; ++j) {
      const std::uint32_t r = G.crow + j;
      if (needv[r])
        o << "      const T bv" << r << " = __shfl_sync(0xffffffffu, " << outn(i, j / 8, j % 2) << ", (lane & ~3u) | "
          << (j % 8) / 2 << "u);\n";
    }
  };
  auto group_bwd = [&](std::size_t i) {
    const DenseGroup& G = gr[i];
    const tgc::Dense& D = *G.D;
    const Geo& q = ge[i];
    const std::string I = std::to_string(i);
    o << "      // dense " << I << " reverse\n";
    for (unsigned u = 0; u < q.ntO; ++u)
      for (unsigned e = 0; e < 2; ++e) {
        const std::string gz = nm("gz", i, u, e);
        o << "      T " << gz << " = "
          << (D.act_op ? Gn.act_b(D.act_op, nm("gh", i, u, e), nm("dh", i, u, e), nm("dz", i, u, e)) : nm("gh", i, u, e)) << ";\n";
        if (8 * u + 8 > D.n_out)
          o << "      if (" << 8 * u + e << "u + 2u * c >= " << D.n_out << "u) " << gz << " = (T)0;\n";
      }
    // input adjoints: dX = gz . W (k axis = this layer's outputs in D-layout order)
    if (G.xvec) {
      for (unsigned t = 0; t < 2 * q.ntO; ++t)
        for (unsigned u = 0; u < q.ntX; ++u)
          o << "      tg_dmma(" << nm("gh", G.src, u, 0) << ", " << nm("gh", G.src, u, 1) << ", " << nm("gz", i, t / 2, t % 2)
            << ", sm[" << q.bk + (t * q.ntX + u) * 32 << "u + lane]);\n";
    } else {
      for (unsigned u = 0; u < q.ntX; ++u)
        o << "      T " << nm("dx", i, u, 0) << " = (T)0, " << nm("dx", i, u, 1) << " = (T)0;\n";
      for (unsigned t = 0; t < 2 * q.ntO; ++t)
        for (unsigned u = 0; u < q.ntX; ++u)
          o << "      tg_dmma(" << nm("dx", i, u, 0) << ", " << nm("dx", i, u, 1) << ", " << nm("gz", i, t / 2, t % 2)
            << ", sm[" << q.bk + (t * q.ntX + u) * 32 << "u + lane]);\n";
      Instr pseudo{};
      pseudo.opnd = D.x_opnd;
      for (std::uint32_t k = 0; k < D.n_in; ++k) {
        const std::string px = "px" + std::to_string(Gn.tmp++);
        o << "      const T " << px << " = __shfl_sync(0xffffffffu, " << nm("dx", i, k / 8, k % 2) << ", (lane & ~3u) | "
          << (k % 8) / 2 << "u);\n";
        Gn.push(pseudo, k, px);
      }
    }
    if (!q.contract) return;
    // weight / bias gradients: Acc[n][k] += sum over this step's 8 samples of gz[s][n] x[s][k]
    for (unsigned u = 0; u < q.ntO; ++u)
      for (unsigned e = 0; e < 2; ++e)
        o << "      gzb[g * " << ldg << "u + " << 8 * u + e << "u + 2u * c] = active ? " << nm("gz", i, u, e) << " : (T)0;\n";
    if (G.xvec) {
      const unsigned nts = ge[G.src].ntO;
      for (unsigned u = 0; u < nts; ++u)
        for (unsigned e = 0; e < 2; ++e) {
          o << "      ";
          if (8 * u + 8 > D.n_in) o << "if (" << 8 * u + e << "u + 2u * c < " << D.n_in << "u) ";
          o << "xb[g * " << ldx << "u + " << 8 * u + e << "u + 2u * c] = active ? " << outn(G.src, u, e) << " : (T)0;\n";
        }
    } else {
      for (std::uint32_t k = 0; k < D.n_in; ++k)
        o << "      if (c == " << k % 4 << "u) xb[g * " << ldx << "u + " << k << "u] = active ? " << Gn.V(G.xr[k]) << " : (T)0;\n";
    }
    if (G.has_bias()) o << "      if (c == 0u) xb[g * " << ldx << "u + " << D.n_in << "u] = active ? (T)1 : (T)0;\n";
    o << "      __syncwarp();\n";
    for (unsigned t = 0; t < 2; ++t) {
      for (unsigned u = 0; u < q.ntO; ++u)
        o << "      const T qa" << i << "_" << t << "_" << u << " = gzb[(" << 4 * t << "u + c) * " << ldg << "u + " << 8 * u << "u + g];\n";
      for (unsigned v = 0; v < q.ntK; ++v)
        o << "      const T qb" << i << "_" << t << "_" << v << " = xb[(" << 4 * t << "u + c) * " << ldx << "u + " << 8 * v << "u + g];\n";
      for (unsigned u = 0; u < q.ntO; ++u)
        for (unsigned v = 0; v < q.ntK; ++v)
          o << "      tg_dmma(aw" << i << "_" << u << "_" << v << "_0, aw" << i << "_" << u << "_" << v << "_1, qa" << i << "_"
            << t << "_" << u << ", qb" << i << "_" << t << "_" << v << ");\n";
    }
    o << "      __syncwarp();\n";
  };
  for (const Instr& in : P.fwd) {
    if (in.kind == tgc::kDense) group_fwd(in.aux);
    else if (in.kind == tgc::kInputLoad) o << "      const T " << Gn.v(in.out) << " = in" << in.aux << ";\n";
    else Gn.forward(in);
  }
  o << "      if (loss && active && c == 0u) loss[s] = " << Gn.V(P.root_row) << ";\n";
  for (std::size_t i = 0; i < ng; ++i)
    for (unsigned u = 0; u < ge[i].ntO; ++u)
      o << "      T " << nm("gh", i, u, 0) << " = (T)0, " << nm("gh", i, u, 1) << " = (T)0;\n";
  for (std::uint32_t r : P.zero_rows)
    if (rg[r] < 0 && zg[r] < 0) o << "      T " << Gn.g(r) << " = (T)0;\n";
  o << "      T " << Gn.g(P.root_row) << " = (T)1;\n";
  for (const Instr& in : P.bwd) {
    if (in.kind == tgc::kDense) group_bwd(in.aux);
    else Gn.reverse(in);
  }
  for (std::uint32_t cI = 0; cI < P.n_inputs; ++cI) {
    const std::uint32_t r = P.input_rows[cI];
    if (r != kNone) o << "      if (igrad && active && c == 0u) igrad[" << cI << "ull * batch + s] = " << Gn.Gx(r) << ";\n";
  }
  if (!sdests.empty()) {
    o << "      if (active && c == 0u) {\n";
    for (std::size_t e = 0; e < sdests.size(); ++e) {
      const unsigned d = sdests[e];
      for (std::uint32_t u = P.term_off[d]; u < P.term_off[d + 1]; ++u) {
        const tgc::Term& t = P.terms[u];
        o << "        as" << e << " += " << lit(t.coef, true) << " * " << Gn.Gx(t.a);
        if (t.f != kNone) o << " * " << Gn.V(t.f);
        o << ";\n";
      }
    }
    o << "      }\n";
  }
  o << "    }\n    __syncwarp();\n  }\n";
  for (std::size_t e = 0; e < sdests.size(); ++e)
    for (unsigned m = 4; m < 32; m *= 2)
      o << "  as" << e << " += __shfl_xor_sync(0xffffffffu, as" << e << ", " << m << ");\n";
  o << "  {\n    T* red = sRed + warp * " << nd << "u;\n";
  for (std::size_t i = 0; i < ng; ++i) {
    const DenseGroup& G = gr[i];
    const Geo& q = ge[i];
    if (!q.contract) continue;
    const unsigned no_ = G.D->n_out, ni = G.D->n_in;
    for (unsigned u = 0; u < q.ntO; ++u)
      for (unsigned v = 0; v < q.ntK; ++v)
        for (unsigned e = 0; e < 2; ++e) {
          o << "    { const unsigned n = " << 8 * u << "u + g, k = " << 8 * v + e << "u + 2u * c; if (n < " << no_ << "u) {";
          if (G.dw0 != kNone) o << " if (k < " << ni << "u) red[" << G.dw0 << "u + n * " << ni << "u + k] = aw" << i << "_" << u << "_" << v << "_" << e << ";";
          if (G.has_bias()) {
            o << " if (k == " << ni << "u && cBD" << i << "[n] != 0xffffffffu) red[cBD" << i << "[n]] = ";
            if (!G.unit_bias()) o << "cBC" << i << "[n] * ";
            o << "aw" << i << "_" << u << "_" << v << "_" << e << ";";
          }
          o << " } }\n";
        }
  }
  for (std::size_t e = 0; e < sdests.size(); ++e) o << "    if (lane == 0u) red[" << sdests[e] << "u] = as" << e << ";\n";
  o << "  }\n  __syncthreads();\n"
    << "  for (unsigned d = tid; d < " << nd << "u; d += " << cfg.block << "u) {\n"
    << "    T t = (T)0;\n"
    << "    for (unsigned w = 0; w < " << WPB << "u; ++w) t += sRed[w * " << nd << "u + d];\n"
    << "    partial[(unsigned long long)d * grid_rows + blockIdx.x] = t;\n  }\n" << fc.tail << "}\n" << fc.epi;
  return o.str();
}

JitKernel build(const tgc::Program& P) {
  JitKernel k;
  if (!eligible(P)) { k.log = "not eligible"; return k; }
  const auto t0 = std::chrono::steady_clock::now();
  JitConfig cfg;
  const std::size_t ts = P.dtype == TG_F64 ? 8 : 4;
  cfg.const_uv = std::size_t(std::max<std::uint32_t>(1, P.n_uv)) * ts <= kMaxConstBytes;
  if (const char* e = std::getenv("TG_JIT_CONST")) cfg.const_uv = cfg.const_uv && std::atoi(e) != 0;
  cfg.block = 128;
  // samples per thread for dest-free tapes (cfg1 with L2 flushed between
  // steps: 4 -> 11.2 us, 8 -> 11.4 us; L2-warm 8 was faster, 10.2 vs 10.6)
  cfg.spt = P.dest_uv.empty() ? (P.n_rows <= 32 ? 4 : 2) : 1;
  // tuning overrides (profiling sweeps): TG_JIT_BLOCK, TG_JIT_SPT, TG_JIT_MINB
  if (const char* e = std::getenv("TG_JIT_BLOCK")) cfg.block = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_SPT")) cfg.spt = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_MINB")) cfg.min_blocks = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_UJ")) cfg.unroll_j = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_DLOOP")) cfg.dense_loop = std::atoi(e) != 0;
  std::vector<tgc::Term> terms;
  std::vector<std::uint32_t> toff;
  // TG_JIT_FUSE=0 keeps the separate prologue / epilogue kernels
  {
    const char* fu = std::getenv("TG_JIT_FUSE");
    std::string why;
    cfg.fuse = !(fu && fu[0] == '0') && fusable(P, why);
    if (cfg.fuse) cfg.const_uv = false;
    // TG_JIT_COOP=1: epilogue inside the tape kernel behind two grid barriers
    // (cooperative launch).  Off by default: on cfg2 the barriers over 444 CTAs
    // cost more than the PDL-overlapped epilogue launch (37.8 vs 30.7 us/step,
    // 29.0 vs 23.3 us back to back, measured)
    const char* co = std::getenv("TG_JIT_COOP");
    cfg.coop = cfg.fuse && (co && co[0] == '1') && (!P.dest_uv.empty() || !P.ubwd.empty());
  }
  // specialised forms for dense-layer chains before the one-thread-per-sample form
  // form: TG_JIT_FORM = dmma | group | classic (default: first that applies, in that order)
  const char* fe = std::getenv("TG_JIT_FORM");
  const std::string form = fe ? fe : "";
  if (form.empty() || form == "dmma") {
    JitConfig dc = cfg;
    dc.block = 128;
    dc.min_blocks = 0;
    if (const char* e = std::getenv("TG_JIT_GBLOCK")) dc.block = static_cast<unsigned>(std::atoi(e));
    if (const char* e = std::getenv("TG_JIT_GMINB")) dc.min_blocks = static_cast<unsigned>(std::atoi(e));
    unsigned spb = 0;
    std::size_t sb = 0;
    std::string src = generate_dmma(P, dc, spb, sb, k.group_log);
    if (!src.empty()) {
      k.source = std::move(src);
      k.cfg = dc;
      k.tile = spb;
      k.smem_bytes = sb;
      k.group = 4;
      k.form = "dmma";
    }
  }
  if (!k.group && (form.empty() || form == "group")) {
    JitConfig gc = cfg;
    gc.block = 256;
    gc.min_blocks = 0;
    if (const char* e = std::getenv("TG_JIT_GBLOCK")) gc.block = static_cast<unsigned>(std::atoi(e));
    if (const char* e = std::getenv("TG_JIT_GMINB")) gc.min_blocks = static_cast<unsigned>(std::atoi(e));
    unsigned G = 0, spb = 0;
    std::size_t sb = 0;
    std::string src = generate_grouped(P, gc, G, spb, sb, k.group_log);
    if (!src.empty()) {
      k.source = std::move(src);
      k.cfg = gc;
      k.tile = spb;
      k.smem_bytes = sb;
      k.group = G;
      k.form = "group";
    }
  }
  if (!k.group) {
    k.form = "classic";
    k.balanced = true;
    // the one-thread-per-sample form reads dense weights as constant-bank
    // operands; fused, they would be shared-memory loads (42 -> 66 us on cfg2,
    // measured), so it fuses only tapes without dense layers (cfg1: 49 -> 61 G/s)
    if (cfg.fuse && !P.dense.empty()) {
      cfg.fuse = false;
      cfg.coop = false;
      cfg.const_uv = std::size_t(std::max<std::uint32_t>(1, P.n_uv)) * ts <= kMaxConstBytes;
    }
    std::size_t smem_elems = 0;
    k.source = generate(P, cfg, k.n_crow_g, k.n_crow_v, terms, toff, smem_elems);
    k.cfg = cfg;
    k.tile = cfg.block * cfg.spt;
    k.smem_bytes = smem_elems * ts;
    if (k.smem_bytes > 200 * 1024) { k.log = "contraction rows exceed shared memory"; return k; }
  }

  nvrtcProgram prog;
  // TG_JIT_DUMP=<dir>: write the source there and name it so -lineinfo maps to it (ncu source page)
  std::string src_name = "tg_jit.cu";
  if (const char* dir = std::getenv("TG_JIT_DUMP")) {
    src_name = std::string(dir) + "/tg_jit_" + std::to_string(std::hash<std::string>{}(k.source) & 0xffffff) + ".cu";
    if (FILE* f = std::fopen(src_name.c_str(), "w")) { std::fputs(k.source.c_str(), f); std::fclose(f); }
  }
  if (nvrtcCreateProgram(&prog, k.source.c_str(), src_name.c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    k.log = "nvrtcCreateProgram failed";
    return k;
  }
  // TG_JIT_VERBOSE=1: ptxas register / spill report in the compile log
  const bool verbose = std::getenv("TG_JIT_VERBOSE") && std::getenv("TG_JIT_VERBOSE")[0] == '1';
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true",
                        "--diag-suppress=550,177", "--ptxas-options=-v"};
  const nvrtcResult rc = nvrtcCompileProgram(prog, verbose ? 6 : 5, opts);
  std::size_t logn = 0;
  nvrtcGetProgramLogSize(prog, &logn);
  if (logn > 1) {
    k.log.resize(logn);
    nvrtcGetProgramLog(prog, k.log.data());
    k.log.resize(std::strlen(k.log.c_str()));   // drop the terminating NUL before appending
  }
  if (rc != NVRTC_SUCCESS) { nvrtcDestroyProgram(&prog); k.log = "NVRTC: " + k.log; return k; }
  std::size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);

  k.cubin_bytes = cubin.size();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {  // compile-only (no GPU here)
    cudaGetLastError();
    k.log += "compiled (" + std::to_string(cubin.size()) + " bytes cubin); no device to load it";
    return k;
  }
  if (cudaLibraryLoadData(&k.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&k.fn, k.lib, "tg_jit_tape") != cudaSuccess) {
    k.log = std::string("library load failed: ") + cudaGetErrorString(cudaGetLastError());
    return k;
  }
  k.coop = k.cfg.fuse && k.cfg.coop;
  const bool has_epi = k.cfg.fuse && !k.coop && (!P.dest_uv.empty() || !P.ubwd.empty());   // see fuse_code
  if (has_epi && cudaLibraryGetKernel(&k.fn_epi, k.lib, "tg_jit_epi") != cudaSuccess) {
    k.log = "tg_jit_epi lookup failed";
    return k;
  }
  k.fused = k.cfg.fuse;
  if (k.cfg.const_uv && cudaLibraryGetGlobal(&k.cuv, &k.cuv_bytes, k.lib, "cUV") != cudaSuccess) {
    k.log = "cUV lookup failed";
    return k;
  }
  const void* f = reinterpret_cast<const void*>(k.fn);
  if (k.smem_bytes > 48 * 1024 &&
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem_bytes)) != cudaSuccess) {
    k.log = "smem attribute failed";
    return k;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.occ, f, static_cast<int>(k.cfg.block), k.smem_bytes);
  if (!P.dest_uv.empty() && !k.group) {
    cudaMalloc(&k.d_terms, std::max<std::size_t>(1, terms.size()) * sizeof(tgc::Term));
    if (!terms.empty()) cudaMemcpy(k.d_terms, terms.data(), terms.size() * sizeof(tgc::Term), cudaMemcpyHostToDevice);
    cudaMalloc(&k.d_toff, toff.size() * sizeof(std::uint32_t));
    cudaMemcpy(k.d_toff, toff.data(), toff.size() * sizeof(std::uint32_t), cudaMemcpyHostToDevice);
  }
  cudaGetLastError();
  k.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  k.ok = k.occ > 0;
  if (!k.ok) k.log = "zero occupancy";
  return k;
}

void release(JitKernel& k) {
  if (k.d_terms) cudaFree(k.d_terms);
  if (k.d_toff) cudaFree(k.d_toff);
  if (k.lib) cudaLibraryUnload(k.lib);
  k = JitKernel{};
}

}  // namespace tgj
