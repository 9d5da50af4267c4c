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
#include <functional>
#include <cstdio>
#include <sstream>
#include <unordered_map>
#include <vector>

namespace tgj {
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

  Gen(const tgc::Program& p, const JitConfig& c) : P(p), cfg(c), f64(p.dtype == TG_F64) {}

  std::string fn(const char* d, const char* f) const { return f64 ? d : f; }
  std::string v(std::uint32_t r) const { return "v" + std::to_string(r); }
  std::string g(std::uint32_t r) const { return "g" + std::to_string(r); }
  std::string sv(std::uint32_t r) const { return "sV[" + std::to_string(std::size_t(vslot[r]) * ld) + "u + col]"; }
  std::string sg_(std::uint32_t r) const { return "sG[" + std::to_string(std::size_t(gslot[r]) * ld) + "u + col]"; }
  // value of row r: once a register-homed row has been stored for the
  // contraction, later reads (the reverse sweep) reload it from shared memory
  // so the register dies at the store (TG_JIT_RELOAD=0 keeps registers)
  std::string V(std::uint32_t r) const { return vsm[r] || (reload && !vstored.empty() && vstored[r]) ? sv(r) : v(r); }
  bool reload = true;
  std::string Gx(std::uint32_t r) const { return gsm[r] ? sg_(r) : g(r); } // adjoint of row r
  std::string uv(std::uint32_t i) const {
    return cfg.const_uv ? "cUV[" + std::to_string(i) + "]" : "UVg[" + std::to_string(i) + "]";
  }
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
    if (m == tgc::kSlot) {
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

  void check(const std::string& cond, const Instr& in) {
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
      o << "      const T " << v(in.out) << " = UVg[cand[" << t.cand_off << "u + " << ix_expr(t) << "]];\n";
      return;
    }
    const std::uint32_t n = in.nops;
    std::vector<std::string> a(n);
    for (std::uint32_t j = 0; j < n; ++j) a[j] = val(P.opnd[in.opnd + j]);
    const std::string out = "      const T " + v(in.out) + " = ";
    const std::string Z = "(T)0", ONE = "(T)1", TWO = "(T)2";
    switch (in.op) {
      case Relu: o << out << a[0] << " > " << Z << " ? " << a[0] << " : " << Z << ";\n"; break;
      case Tanh: o << out << fn("tg_tanh", "tanhf") << "(" << a[0] << ");\n"; break;
      case Exp: o << out << fn("exp", "expf") << "(" << a[0] << ");\n"; break;
      case NegLog: check("!(" + a[0] + " > (T)0)", in); o << out << "-" << fn("log", "logf") << "(" << a[0] << ");\n"; break;
      case Sigmoid: o << out << ONE << " / (" << ONE << " + " << fn("exp", "expf") << "(-" << a[0] << "));\n"; break;
      case Inv: check(a[0] + " == (T)0", in); o << out << ONE << " / " << a[0] << ";\n"; break;
      case Sqr: o << out << a[0] << " * " << a[0] << ";\n"; break;
      case Cub: o << out << a[0] << " * " << a[0] << " * " << a[0] << ";\n"; break;
      case Log: check("!(" + a[0] + " > (T)0)", in); o << out << fn("log", "logf") << "(" << a[0] << ");\n"; break;
      case Sqrt: check("!(" + a[0] + " > (T)0)", in); o << out << fn("sqrt", "sqrtf") << "(" << a[0] << ");\n"; break;
      case InvSqrt: check("!(" + a[0] + " > (T)0)", in); o << out << ONE << " / " << fn("sqrt", "sqrtf") << "(" << a[0] << ");\n"; break;
      case MulByConst: o << out << a[0] << " * " << lit(in.cst, f64) << ";\n"; break;
      case Add: o << out << a[0] << " + " << a[1] << ";\n"; break;
      case Sub: o << out << a[0] << " - " << a[1] << ";\n"; break;
      case Mul: o << out << a[0] << " * " << a[1] << ";\n"; break;
      case Div: check(a[1] + " == (T)0", in); o << out << a[0] << " / " << a[1] << ";\n"; break;
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
        const char* sk = std::getenv("TG_JIT_SKIP");  // profiling-only ablation
        if (sk && std::string(sk) == "tanh") return "(" + z + ")";
        return fn("tg_tanh", "tanhf") + "(" + z + ")";
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
    if (D.b_uv != kNone) o << "        T z = " << (cfg.const_uv ? "cUV[" : "UVg[") << D.b_uv << "u + j];\n";
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
)";

}  // namespace

bool eligible(const tgc::Program& P) {
  return P.root_row != kNone && P.n_edges <= kMaxEdges && P.n_rows <= 4096;
}

std::string generate(const tgc::Program& P, const JitConfig& cfg, unsigned& n_crow_g, unsigned& n_crow_v,
                     std::vector<tgc::Term>& terms_out, std::vector<std::uint32_t>& toff_out,
                     std::size_t& smem_elems) {
  Gen G(P, cfg);
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
  o << "typedef " << (f64 ? "double" : "float") << " T;\n" << kMath << kPrelude;
  if (cfg.const_uv) o << "__constant__ T cUV[" << std::max<std::uint32_t>(1, P.n_uv) << "];\n";
  for (std::size_t bi = 0; bi < dbs.size(); ++bi) {
    const DB& b = dbs[bi];
    o << "__constant__ unsigned cDG" << bi << "[" << b.nj + b.nk << "] = {";
    for (unsigned j = 0; j < b.nj; ++j) o << (j ? ", " : "") << G.gslot[P.dg_rows[b.off + j]];
    for (unsigned k = 0; k < b.nk; ++k) o << ", " << G.vslot[P.dg_rows[b.off + b.nj + k]];
    o << "};\n";
  }
  o << "extern \"C\" __global__ void __launch_bounds__(" << cfg.block;
  if (cfg.min_blocks) o << ", " << cfg.min_blocks;
  o << ") tg_jit_tape(\n"
    << "    const T* __restrict__ in, const int* __restrict__ idx, unsigned long long batch,\n"
    << "    T* __restrict__ loss, T* __restrict__ igrad, T* __restrict__ partial, unsigned grid_rows,\n"
    << "    unsigned long long* err_key, const T* __restrict__ UVg, const unsigned* __restrict__ cand,\n"
    << "    const unsigned* __restrict__ toff, const TermC* __restrict__ terms) {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  T* sG = reinterpret_cast<T*>(smem_raw);\n"
    << "  T* sV = sG + " << n_crow_g << " * " << ld << ";\n"
    << "  T* sDW = sV + " << n_crow_v << " * " << ld << ";\n"
    << "  T* sS = sDW + " << (dense ? nd : 0) << ";\n"
    << "  (void)sG; (void)sV; (void)sDW; (void)sS;\n"
    << "  const unsigned tid = threadIdx.x;\n";
  if (dense) o << "  for (unsigned q = tid; q < " << nd << "u; q += " << cfg.block << "u) sDW[q] = (T)0;\n";
  if (reg_acc && nd) o << "  T acc[" << ndpt << "]; for (int q = 0; q < " << ndpt << "; ++q) acc[q] = 0;\n";
  o << "  for (unsigned long long tile = blockIdx.x; tile * " << tile << "ull < batch; tile += gridDim.x) {\n"
    << "    const unsigned long long base = tile * " << tile << "ull;\n"
    << "#pragma unroll\n"
    << "    for (unsigned jj = 0; jj < " << cfg.spt << "u; ++jj) {\n"
    << "    const unsigned long long s = base + jj * " << cfg.block << "u + tid;\n"
    << "    const unsigned col = jj * " << cfg.block << "u + tid;\n"
    << "    (void)col;\n"
    << "    if (s < batch) {\n";
  G.vstored.assign(P.n_rows, 0);
  if (const char* e = std::getenv("TG_JIT_RELOAD")) G.reload = std::atoi(e) != 0;
  G.gstored.assign(P.n_rows, 0);
  for (const Instr& in : P.fwd) {
    G.forward(in);
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
  const char* skip = std::getenv("TG_JIT_SKIP");
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
      << "    const unsigned valid = (unsigned)((batch - base) < " << tile << "ull ? (batch - base) : " << tile << "ull);\n"
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
           << "      *dst = (tile == blockIdx.x) ? tot : *dst + tot;\n";
    o << "    }\n    __syncthreads();\n";
  }
  o << "  }\n";
  if (reg_acc && nd)
    o << "  for (int q = 0; q < " << ndpt << "; ++q) { const unsigned d = q * " << cfg.block << "u + tid;\n"
      << "    if (d < " << nd << "u) partial[(unsigned long long)d * grid_rows + blockIdx.x] = acc[q]; }\n";
  o << "}\n";
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
  cfg.spt = P.dest_uv.empty() ? (P.n_rows <= 32 ? 4 : 2) : 1;
  // tuning overrides (profiling sweeps): TG_JIT_BLOCK, TG_JIT_SPT, TG_JIT_MINB
  if (const char* e = std::getenv("TG_JIT_BLOCK")) cfg.block = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_SPT")) cfg.spt = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_MINB")) cfg.min_blocks = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_UJ")) cfg.unroll_j = static_cast<unsigned>(std::atoi(e));
  if (const char* e = std::getenv("TG_JIT_DLOOP")) cfg.dense_loop = std::atoi(e) != 0;
  std::vector<tgc::Term> terms;
  std::vector<std::uint32_t> toff;
  std::size_t smem_elems = 0;
  k.source = generate(P, cfg, k.n_crow_g, k.n_crow_v, terms, toff, smem_elems);
  k.cfg = cfg;
  k.tile = cfg.block * cfg.spt;
  k.smem_bytes = smem_elems * ts;
  if (k.smem_bytes > 200 * 1024) { k.log = "contraction rows exceed shared memory"; return k; }

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
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true"};
  const nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  std::size_t logn = 0;
  nvrtcGetProgramLogSize(prog, &logn);
  if (logn > 1) { k.log.resize(logn); nvrtcGetProgramLog(prog, k.log.data()); }
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
    k.log = "compiled (" + std::to_string(cubin.size()) + " bytes cubin); no device to load it";
    return k;
  }
  if (cudaLibraryLoadData(&k.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
      cudaLibraryGetKernel(&k.fn, k.lib, "tg_jit_tape") != cudaSuccess) {
    k.log = std::string("library load failed: ") + cudaGetErrorString(cudaGetLastError());
    return k;
  }
  if (cfg.const_uv && cudaLibraryGetGlobal(&k.cuv, &k.cuv_bytes, k.lib, "cUV") != cudaSuccess) {
    k.log = "cUV lookup failed";
    return k;
  }
  const void* f = reinterpret_cast<const void*>(k.fn);
  if (k.smem_bytes > 48 * 1024 &&
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem_bytes)) != cudaSuccess) {
    k.log = "smem attribute failed";
    return k;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.occ, f, static_cast<int>(cfg.block), k.smem_bytes);
  if (!P.dest_uv.empty()) {
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
