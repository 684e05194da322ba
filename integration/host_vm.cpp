// See host_vm.hpp.  Every rule below cites the reference interpreter
// (/root/reference/proj/src/interp.cpp) line it restates.
#include "host_vm.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace liftc::gpu {

using namespace minilang;
using interp::ExecMode;
using interp::ExecStatus;

namespace {

constexpr int kMaxCallDepth = 1024;       // interp.cpp:10
constexpr size_t kTraceCap = 1u << 20;    // interp.cpp:11

// ------------------------------------------------------------------ IR --
enum class EK : uint8_t {
  IntLit, FloatLit, Var, Index, Neg, Not, And, Or, Min, Max, ToI64, ToF64, Fabs, Sqrt, Dispatch, Call,
  Add, Sub, Mul, Div, Mod, Lt, Le, Gt, Ge, Eq, Ne
};

// Static type of an expression: the resolver (minilang.cpp:680-1000) types every
// variable and operator, so an expression without calls is int or float for certain;
// a call's value is dynamic (a float function that falls off its end yields int 0,
// interp.cpp:521) and takes the generic, tagged path.
enum : int8_t { TY_INT = 0, TY_FLT = 1, TY_DYN = 2 };

struct CExpr {
  EK k = EK::IntLit;
  int8_t ty = TY_DYN;
  int slot = -1;            // Var / Index (pointer slot)
  int a0 = -1, a1 = -1;     // children (unary: a0; binary: a0, a1)
  int fn = -1;              // Call: callee index
  int argb = 0, argn = 0;   // Call: arguments F.args[argb, argb + argn) (pointer params are Var)
  long long i = 0;
  double f = 0.0;
};

enum class SK : uint8_t {
  Let, Assign, Store, For, While, If, Call, Return, VLoad, VStore, VSplat, VAdd, VMul, VFma, VReduce
};

struct CStmt {
  SK k = SK::Let;
  LocalType lt = LocalType::I64;
  int slot = -1;             // Let / Assign / For var / VReduce target / vec dst
  int ptr = -1;              // Store / VLoad / VStore pointer slot
  int e0 = -1, e1 = -1, e2 = -1;  // Let init | Assign value | Store index,value | For lo,hi,step | cond | call | ret
  int va = -1, vb = -1;      // vector operand slots
  int width = 4;
  std::vector<int> body, els;
};

struct CFunc {
  const FunctionIR* ir = nullptr;
  int n_slots = 0;
  std::vector<int8_t> slot_ty;  // TY_INT / TY_FLT, TY_DYN for pointers and vectors
  std::vector<CExpr> ex;
  std::vector<int> args;
  std::vector<CStmt> st;
  std::vector<int> body;
};

}  // namespace

struct VmProgram {
  std::vector<CFunc> fns;
  std::map<std::string, int> index;
};

namespace {

// --------------------------------------------------------- compilation --
struct Compiler {
  VmProgram& P;
  CFunc& F;
  std::vector<std::map<std::string, int>> scopes;

  int declare(const std::string& name, int8_t ty = TY_DYN) {
    const int s = F.n_slots++;
    scopes.back()[name] = s;
    F.slot_ty.push_back(ty);
    return s;
  }
  static int8_t arith(int8_t a, int8_t b) {
    return a == TY_DYN || b == TY_DYN ? TY_DYN : a == TY_INT && b == TY_INT ? TY_INT : TY_FLT;
  }
  int lookup(const std::string& name) {
    for (auto it = scopes.rbegin(); it != scopes.rend(); ++it) {
      auto f = it->find(name);
      if (f != it->end()) return f->second;
    }
    throw std::runtime_error("host_vm: unbound identifier '" + name + "'");
  }

  int expr(const Expr& e) {
    CExpr c;
    switch (e.kind) {
      case Expr::Kind::IntLit:
        c.k = EK::IntLit;
        c.i = e.int_val;
        break;
      case Expr::Kind::FloatLit:
        c.k = EK::FloatLit;
        c.f = e.float_val;
        break;
      case Expr::Kind::Var:
        c.k = EK::Var;
        c.slot = lookup(e.name);
        break;
      case Expr::Kind::Index:
        c.k = EK::Index;
        c.slot = lookup(e.name);
        c.a0 = expr(*e.args[0]);
        break;
      case Expr::Kind::Unary:
        c.k = e.uop == UnOp::Not ? EK::Not : EK::Neg;
        c.a0 = expr(*e.args[0]);
        break;
      case Expr::Kind::Binary: {
        static const EK kinds[] = {EK::Add, EK::Sub, EK::Mul, EK::Div, EK::Mod, EK::Lt, EK::Le,
                                   EK::Gt,  EK::Ge,  EK::Eq,  EK::Ne,  EK::And, EK::Or};
        c.k = kinds[(int)e.bop];
        c.a0 = expr(*e.args[0]);
        c.a1 = expr(*e.args[1]);
        break;
      }
      case Expr::Kind::Call: {
        const std::string& n = e.name;
        if (n == "min" || n == "max") c.k = n == "min" ? EK::Min : EK::Max;
        else if (n == "to_i64") c.k = EK::ToI64;
        else if (n == "to_f64") c.k = EK::ToF64;
        else if (n == "fabs") c.k = EK::Fabs;
        else if (n == "sqrt") c.k = EK::Sqrt;
        else if (is_dispatch_builtin(n)) {
          c.k = EK::Dispatch;  // no handler: a no-op whose arguments are never evaluated (interp.cpp:506)
          break;
        } else {
          c.k = EK::Call;
          auto it = P.index.find(n);
          c.fn = it == P.index.end() ? -1 : it->second;  // -1: "call to unknown function" at run time
        }
        std::vector<int> args;
        if (c.k == EK::Call && c.fn >= 0) {
          const FunctionIR* callee = P.fns[c.fn].ir;
          for (size_t i = 0; i < e.args.size(); ++i) {
            if (i < callee->params.size() && callee->params[i].kind == ParamKind::Pointer) {
              CExpr v;
              v.k = EK::Var;
              v.slot = lookup(e.args[i]->name);
              F.ex.push_back(v);
              args.push_back((int)F.ex.size() - 1);
            } else {
              args.push_back(expr(*e.args[i]));
            }
          }
        } else if (c.k != EK::Call) {
          for (const auto& a : e.args) args.push_back(expr(*a));
        }
        if (!args.empty()) c.a0 = args[0];
        if (args.size() > 1) c.a1 = args[1];
        c.argb = (int)F.args.size();
        c.argn = (int)args.size();
        F.args.insert(F.args.end(), args.begin(), args.end());
        break;
      }
    }
    c.ty = type_of(c);
    F.ex.push_back(std::move(c));
    return (int)F.ex.size() - 1;
  }

  int8_t type_of(const CExpr& c) const {
    auto ty = [&](int i) { return i >= 0 ? F.ex[i].ty : TY_DYN; };
    switch (c.k) {
      case EK::IntLit: return TY_INT;
      case EK::FloatLit: return TY_FLT;
      case EK::Var: return F.slot_ty[c.slot];
      case EK::Index: return TY_FLT;
      case EK::Neg: return ty(c.a0);
      case EK::Not: case EK::And: case EK::Or: case EK::Lt: case EK::Le: case EK::Gt: case EK::Ge: case EK::Eq:
      case EK::Ne: case EK::Dispatch: case EK::ToI64: return TY_INT;
      case EK::Add: case EK::Sub: case EK::Mul: case EK::Div: return arith(ty(c.a0), ty(c.a1));
      case EK::Mod: case EK::Min: case EK::Max: return ty(c.a0) == TY_INT && ty(c.a1) == TY_INT ? TY_INT : TY_DYN;
      case EK::ToF64: case EK::Fabs: case EK::Sqrt: return TY_FLT;
      case EK::Call: return TY_DYN;
    }
    return TY_DYN;
  }

  std::vector<int> block(const std::vector<StmtPtr>& body, bool new_scope) {
    if (new_scope) scopes.emplace_back();
    std::vector<int> out;
    for (const auto& s : body) out.push_back(stmt(*s));
    if (new_scope) scopes.pop_back();
    return out;
  }

  int stmt(const Stmt& s) {
    CStmt c;
    switch (s.kind) {
      case Stmt::Kind::Let:
        c.k = SK::Let;
        c.lt = s.let_type;
        c.e0 = s.let_init ? expr(*s.let_init) : -1;  // evaluated before the declaration
        c.slot = declare(s.let_name, s.let_type == LocalType::I64   ? TY_INT
                                     : s.let_type == LocalType::F32 || s.let_type == LocalType::F64 ? TY_FLT
                                                                                                     : TY_DYN);
        break;
      case Stmt::Kind::Assign:
        c.k = SK::Assign;
        c.e0 = expr(*s.value);
        c.slot = lookup(s.target);
        break;
      case Stmt::Kind::Store:
        c.k = SK::Store;
        c.e0 = expr(*s.index);
        c.e1 = expr(*s.value);
        c.ptr = lookup(s.target);
        break;
      case Stmt::Kind::For:
        c.k = SK::For;
        c.e0 = expr(*s.lo);
        c.e1 = expr(*s.hi);
        c.e2 = s.step ? expr(*s.step) : -1;
        scopes.emplace_back();  // the iteration scope: loop var + body (interp.cpp:304-311)
        c.slot = declare(s.loop_var, TY_INT);
        c.body = block(s.body, false);
        scopes.pop_back();
        break;
      case Stmt::Kind::While:
        c.k = SK::While;
        c.e0 = expr(*s.cond);
        c.body = block(s.body, true);
        break;
      case Stmt::Kind::If:
        c.k = SK::If;
        c.e0 = expr(*s.cond);
        c.body = block(s.body, true);
        c.els = block(s.else_body, true);
        break;
      case Stmt::Kind::CallStmt:
        c.k = SK::Call;
        c.e0 = expr(*s.call);
        break;
      case Stmt::Kind::Return:
        c.k = SK::Return;
        c.e0 = s.value ? expr(*s.value) : -1;
        break;
      case Stmt::Kind::Vec:
        c.width = s.vec_width;
        switch (s.vec_op) {
          case VecOp::Load:
            c.k = SK::VLoad;
            c.e0 = expr(*s.index);
            c.slot = lookup(s.vec_dst);
            c.ptr = lookup(s.target);
            break;
          case VecOp::Store:
            c.k = SK::VStore;
            c.e0 = expr(*s.index);
            c.va = lookup(s.vec_a);
            c.ptr = lookup(s.target);
            break;
          case VecOp::Splat:
            c.k = SK::VSplat;
            c.e0 = expr(*s.value);
            c.slot = lookup(s.vec_dst);
            break;
          case VecOp::Add:
          case VecOp::Mul:
          case VecOp::Fma:
            c.k = s.vec_op == VecOp::Add ? SK::VAdd : s.vec_op == VecOp::Mul ? SK::VMul : SK::VFma;
            c.va = lookup(s.vec_a);
            c.vb = lookup(s.vec_b);
            c.slot = lookup(s.vec_dst);
            break;
          case VecOp::Reduce:
            c.k = SK::VReduce;
            c.va = lookup(s.vec_a);
            c.slot = lookup(s.target);
            break;
        }
        break;
    }
    F.st.push_back(std::move(c));
    return (int)F.st.size() - 1;
  }
};

// ------------------------------------------------------------ runtime --
struct Fault {
  ExecStatus status;
  std::string msg;
};

// interp.cpp:20-29.  16 bytes (returned in registers): the int and float payloads
// share storage, so iv() / fv() give the reference's view of the other field — a float
// Value reads as int 0 (make_float leaves i == 0), an int Value as float 0.0.
struct Val {
  union {
    long long i;
    double f;
  };
  bool is_int;
  static Val I(long long v) {
    Val r;
    r.i = v;
    r.is_int = true;
    return r;
  }
  static Val F(double v) {
    Val r;
    r.f = v;
    r.is_int = false;
    return r;
  }
  long long iv() const { return is_int ? i : 0; }
  double fv() const { return is_int ? 0.0 : f; }
  double d() const { return is_int ? (double)i : f; }
  bool truthy() const { return is_int ? i != 0 : f != 0.0; }
};

struct Slot {  // interp.cpp:31-39
  Val v = Val::I(0);
  bool round_f32 = false;
  int region = -1;
  double lanes[8] = {};
};

enum class Flow { Next, Ret };

struct Run {
  const VmProgram& P;
  ExecMode mode;
  unsigned long long limit, steps = 0;
  // regions: index = position among the root's pointer params
  std::vector<std::string> keys;
  std::vector<interp::Region*> reg;  // Plain: the region in the output image
  std::vector<std::vector<bool>*> wr;  // Plain + track_writes
  // DimProbe: target region index (-2: every region — the survey), extent, scratch
  int target = -1;
  long long extent = 0;
  double scratch = 1.0;
  bool record = false;
  std::vector<std::vector<long long>> trace;
  std::vector<long long> maxoff;
  std::vector<char> dead;  // survey: this region's own run has ended (OutOfBounds)
  std::vector<std::string> dead_msg;
  std::vector<Slot> stack;
  size_t base = 0;
  int depth = 0;
  Val ret;
  bool has_ret = false;

  Run(const VmProgram& p, ExecMode m, unsigned long long lim) : P(p), mode(m), limit(lim) {}

  Slot& S(int s) { return stack[base + (size_t)s]; }

  void step() {  // interp.cpp:282-285
    if (++steps > limit) throw Fault{ExecStatus::StepLimit, "statement budget exhausted"};
  }

  void note(int r, long long off) {  // interp.cpp:213-216
    if (record && trace[r].size() < kTraceCap) trace[r].push_back(off);
    if (off > maxoff[r]) maxoff[r] = off;
  }

  double load(int r, long long off) {
    if (mode == ExecMode::DimProbe) {  // interp.cpp:219-227
      if (target == -2) {
        if (r < 0 || dead[r]) return scratch;
        note(r, off);
        if (off < 0 || off >= extent) {
          dead[r] = 1;
          dead_msg[r] = "load offset " + std::to_string(off) + " outside extent " + std::to_string(extent);
        }
        return scratch;
      }
      if (r != target) return scratch;
      note(r, off);
      if (off < 0 || off >= extent)
        throw Fault{ExecStatus::OutOfBounds,
                    "load offset " + std::to_string(off) + " outside extent " + std::to_string(extent)};
      return scratch;
    }
    interp::Region& R = *reg[r];  // interp.cpp:228-232
    if (off < 0 || off >= (long long)R.data.size())
      throw Fault{ExecStatus::RuntimeFault, "load offset " + std::to_string(off) + " outside region '" + keys[r] + "'"};
    return R.data[(size_t)off];
  }

  void store(int r, long long off, double v) {
    if (mode == ExecMode::DimProbe) {  // interp.cpp:235-244
      if (target == -2) {
        if (r < 0 || dead[r]) return;
        note(r, off);
        if (off < 0 || off >= extent) {
          dead[r] = 1;
          dead_msg[r] = "store offset " + std::to_string(off) + " outside extent " + std::to_string(extent);
        }
        return;
      }
      if (r != target) return;
      note(r, off);
      if (off < 0 || off >= extent)
        throw Fault{ExecStatus::OutOfBounds,
                    "store offset " + std::to_string(off) + " outside extent " + std::to_string(extent)};
      return;
    }
    interp::Region& R = *reg[r];  // interp.cpp:245-251
    if (off < 0 || off >= (long long)R.data.size())
      throw Fault{ExecStatus::RuntimeFault,
                  "store offset " + std::to_string(off) + " outside region '" + keys[r] + "'"};
    R.data[(size_t)off] = R.elem == ScalarType::F32 ? (double)(float)v : v;
    if (wr[r]) (*wr[r])[(size_t)off] = true;
  }

  // ----------------------------------------------------------- calls --
  // interp.cpp:145-170: frame, parameters, body, return rounding.  Frames live on
  // one slot stack that only grows (a callee's slots above `top`); slots need no
  // initialisation — the resolver guarantees a write before every read.
  size_t top = 0;

  Val call(int fi, const Slot* args, int nargs, bool& has) {
    const CFunc& F = P.fns[fi];
    if (depth >= kMaxCallDepth)
      throw Fault{ExecStatus::RuntimeFault, "call depth limit exceeded in '" + F.ir->name + "'"};
    const size_t saved = base, nb = top;
    if (stack.size() < nb + (size_t)F.n_slots) stack.resize(std::max(stack.size() * 2, nb + (size_t)F.n_slots + 64));
    for (int i = 0; i < nargs; ++i) stack[nb + i] = args[i];
    base = nb;
    top = nb + (size_t)F.n_slots;
    ++depth;
    has_ret = false;
    exec_list(F, F.body);
    Val r = ret;
    has = has_ret;
    has_ret = false;
    --depth;
    base = saved;
    top = nb;
    if (has) {
      if (F.ir->ret == RetType::F32)
        r = Val::F((double)(float)r.d());
      else if (F.ir->ret == RetType::F64)
        r = Val::F(r.d());
      else if (F.ir->ret == RetType::I64 && !r.is_int)
        throw Fault{ExecStatus::RuntimeFault, "float returned from i64 function"};
    }
    return r;
  }

  // ------------------------------------------------ typed expressions --
  // Statically int / float subtrees (CExpr::ty) evaluate without tags: the same
  // operations in the same order as eval(), on plain int64 / double.
  long long ival(const CFunc& F, int ei) {  // eval(F, ei).iv()
    return F.ex[ei].ty == TY_INT ? ileaf(F, ei) : eval(F, ei).iv();
  }
  double dval(const CFunc& F, int ei) {  // eval(F, ei).d()
    const CExpr& e = F.ex[ei];
    if (e.k == EK::Var && e.ty != TY_DYN) {
      const Val& v = S(e.slot).v;
      return e.ty == TY_INT ? (double)v.i : v.f;
    }
    return e.ty == TY_INT ? (double)ieval(F, ei) : e.ty == TY_FLT ? feval(F, ei) : eval(F, ei).d();
  }
  bool truth(const CFunc& F, int ei) {  // eval(F, ei).truthy()
    const int8_t t = F.ex[ei].ty;
    return t == TY_INT ? ieval(F, ei) != 0 : t == TY_FLT ? feval(F, ei) != 0.0 : eval(F, ei).truthy();
  }
  // a comparison: int compare when both sides are ints, else on doubles (interp.cpp:446)
  template <class Op>
  long long cmp(const CFunc& F, const CExpr& e, Op op) {
    const int8_t ta = F.ex[e.a0].ty, tb = F.ex[e.a1].ty;
    if (ta == TY_INT && tb == TY_INT) {
      const long long a = ieval(F, e.a0);
      const long long b = ieval(F, e.a1);
      return op(a, b) ? 1 : 0;
    }
    if (ta != TY_DYN && tb != TY_DYN) {  // at least one float: doubles
      const double a = dval(F, e.a0);
      const double b = dval(F, e.a1);
      return op(a, b) ? 1 : 0;
    }
    const Val a = eval(F, e.a0), b = eval(F, e.a1);
    return (a.is_int && b.is_int ? op(a.i, b.i) : op(a.d(), b.d())) ? 1 : 0;
  }

  // leaves read in place (no call): most operands of index arithmetic are variables
  // and literals
  long long ileaf(const CFunc& F, int ei) {
    const CExpr& e = F.ex[ei];
    if (e.k == EK::Var) return S(e.slot).v.i;
    if (e.k == EK::IntLit) return e.i;
    return ieval(F, ei);
  }

  long long ieval(const CFunc& F, int ei) {  // CExpr::ty == TY_INT
    const CExpr& e = F.ex[ei];
    switch (e.k) {
      case EK::IntLit:
        return e.i;
      case EK::Var:
        return S(e.slot).v.i;
      case EK::Add: {
        const long long a = ileaf(F, e.a0);
        return a + ileaf(F, e.a1);
      }
      case EK::Sub: {
        const long long a = ileaf(F, e.a0);
        return a - ileaf(F, e.a1);
      }
      case EK::Mul: {
        const long long a = ileaf(F, e.a0);
        return a * ileaf(F, e.a1);
      }
      case EK::Div: {
        const long long a = ieval(F, e.a0);
        const long long b = ieval(F, e.a1);
        if (b == 0) throw Fault{ExecStatus::RuntimeFault, "integer division by zero"};
        return a / b;
      }
      case EK::Mod: {
        const long long a = ieval(F, e.a0);
        const long long b = ieval(F, e.a1);
        if (b == 0) throw Fault{ExecStatus::RuntimeFault, "integer modulo by zero"};
        return a % b;
      }
      case EK::Lt: return cmp(F, e, [](auto a, auto b) { return a < b; });
      case EK::Le: return cmp(F, e, [](auto a, auto b) { return a <= b; });
      case EK::Gt: return cmp(F, e, [](auto a, auto b) { return a > b; });
      case EK::Ge: return cmp(F, e, [](auto a, auto b) { return a >= b; });
      case EK::Eq: return cmp(F, e, [](auto a, auto b) { return a == b; });
      case EK::Ne: return cmp(F, e, [](auto a, auto b) { return a != b; });
      case EK::Not:
        return truth(F, e.a0) ? 0 : 1;
      case EK::And:
        if (!truth(F, e.a0)) return 0;
        return truth(F, e.a1) ? 1 : 0;
      case EK::Or:
        if (truth(F, e.a0)) return 1;
        return truth(F, e.a1) ? 1 : 0;
      case EK::Neg:
        return -ieval(F, e.a0);
      case EK::Min:
      case EK::Max: {
        const long long a = ieval(F, e.a0);
        const long long b = ieval(F, e.a1);
        const bool lt = a < b;
        return e.k == EK::Min ? (lt ? a : b) : (lt ? b : a);
      }
      case EK::ToI64: {
        const int8_t t = F.ex[e.a0].ty;
        if (t == TY_INT) return ieval(F, e.a0);
        if (t == TY_FLT) return (long long)feval(F, e.a0);
        return eval(F, ei).iv();
      }
      default:
        return eval(F, ei).iv();
    }
  }

  double feval(const CFunc& F, int ei) {  // CExpr::ty == TY_FLT
    const CExpr& e = F.ex[ei];
    switch (e.k) {
      case EK::FloatLit:
        return e.f;
      case EK::Var:
        return S(e.slot).v.f;
      case EK::Index: {  // interp.cpp:416-419
        const long long off = ival(F, e.a0);
        return load(S(e.slot).region, off);
      }
      case EK::Add: {
        const double a = dval(F, e.a0);
        return a + dval(F, e.a1);
      }
      case EK::Sub: {
        const double a = dval(F, e.a0);
        return a - dval(F, e.a1);
      }
      case EK::Mul: {
        const double a = dval(F, e.a0);
        return a * dval(F, e.a1);
      }
      case EK::Div: {
        const double a = dval(F, e.a0);
        const double b = dval(F, e.a1);
        if (b == 0.0) throw Fault{ExecStatus::RuntimeFault, "float division by zero"};
        return a / b;
      }
      case EK::Neg:
        return -feval(F, e.a0);
      case EK::ToF64:
        return dval(F, e.a0);
      case EK::Fabs:
        return std::fabs(dval(F, e.a0));
      case EK::Sqrt: {
        const double v = dval(F, e.a0);
        if (v < 0.0) throw Fault{ExecStatus::RuntimeFault, "sqrt of a negative value"};
        return std::sqrt(v);
      }
      default:
        return eval(F, ei).d();
    }
  }

  // ----------------------------------------------------- expressions --
  Val eval(const CFunc& F, int ei) {
    const CExpr& e = F.ex[ei];
    switch (e.k) {
      case EK::IntLit:
        return Val::I(e.i);
      case EK::FloatLit:
        return Val::F(e.f);
      case EK::Var:
        return S(e.slot).v;
      case EK::Index: {  // interp.cpp:416-419
        const long long off = eval(F, e.a0).iv();
        return Val::F(load(S(e.slot).region, off));
      }
      case EK::Not:
        return Val::I(eval(F, e.a0).truthy() ? 0 : 1);
      case EK::Neg: {
        const Val v = eval(F, e.a0);
        return v.is_int ? Val::I(-v.i) : Val::F(-v.f);
      }
      case EK::And:  // interp.cpp:434-441
        if (!eval(F, e.a0).truthy()) return Val::I(0);
        return Val::I(eval(F, e.a1).truthy() ? 1 : 0);
      case EK::Or:
        if (eval(F, e.a0).truthy()) return Val::I(1);
        return Val::I(eval(F, e.a1).truthy() ? 1 : 0);
      // interp.cpp:443-477: float arithmetic as soon as one operand is a float
      case EK::Add: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return a.is_int && b.is_int ? Val::I(a.i + b.i) : Val::F(a.d() + b.d());
      }
      case EK::Sub: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return a.is_int && b.is_int ? Val::I(a.i - b.i) : Val::F(a.d() - b.d());
      }
      case EK::Mul: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return a.is_int && b.is_int ? Val::I(a.i * b.i) : Val::F(a.d() * b.d());
      }
      case EK::Div: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        if (!a.is_int || !b.is_int) {
          if (b.d() == 0.0) throw Fault{ExecStatus::RuntimeFault, "float division by zero"};
          return Val::F(a.d() / b.d());
        }
        if (b.i == 0) throw Fault{ExecStatus::RuntimeFault, "integer division by zero"};
        return Val::I(a.i / b.i);
      }
      case EK::Mod: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        if (b.iv() == 0) throw Fault{ExecStatus::RuntimeFault, "integer modulo by zero"};
        return Val::I(a.iv() % b.iv());
      }
      case EK::Lt: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i < b.i : a.d() < b.d());
      }
      case EK::Le: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i <= b.i : a.d() <= b.d());
      }
      case EK::Gt: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i > b.i : a.d() > b.d());
      }
      case EK::Ge: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i >= b.i : a.d() >= b.d());
      }
      case EK::Eq: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i == b.i : a.d() == b.d());
      }
      case EK::Ne: {
        const Val a = eval(F, e.a0), b = eval(F, e.a1);
        return Val::I(a.is_int && b.is_int ? a.i != b.i : a.d() != b.d());
      }
      case EK::Min:
      case EK::Max: {  // interp.cpp:483-488
        const long long a = eval(F, e.a0).iv();
        const long long b = eval(F, e.a1).iv();
        const bool lt = a < b;
        return Val::I(e.k == EK::Min ? (lt ? a : b) : (lt ? b : a));
      }
      case EK::ToI64: {
        const Val v = eval(F, e.a0);
        return v.is_int ? v : Val::I((long long)v.f);
      }
      case EK::ToF64:
        return Val::F(eval(F, e.a0).d());
      case EK::Fabs:
        return Val::F(std::fabs(eval(F, e.a0).d()));
      case EK::Sqrt: {
        const double v = eval(F, e.a0).d();
        if (v < 0.0) throw Fault{ExecStatus::RuntimeFault, "sqrt of a negative value"};
        return Val::F(std::sqrt(v));
      }
      case EK::Dispatch:
        return Val::I(0);
      case EK::Call: {  // interp.cpp:503-524
        if (e.fn < 0) throw Fault{ExecStatus::RuntimeFault, "call to unknown function"};
        const FunctionIR* callee = P.fns[e.fn].ir;
        constexpr int kInline = 16;
        Slot small[kInline];
        std::vector<Slot> big;
        Slot* args = small;
        if (e.argn > kInline) {
          big.resize(e.argn);
          args = big.data();
        }
        for (int i = 0; i < e.argn; ++i) {
          const Param& p = callee->params[i];
          Slot& s = args[i];
          s = Slot{};
          const int ai = F.args[e.argb + i];
          if (p.kind == ParamKind::Pointer) {
            s.region = S(F.ex[ai].slot).region;
          } else {
            const Val v = eval(F, ai);
            if (p.kind == ParamKind::FloatScalar) {
              s.round_f32 = p.elem == ScalarType::F32;
              s.v = Val::F(s.round_f32 ? (double)(float)v.d() : v.d());
            } else {
              s.v = v;
            }
          }
        }
        bool has = false;
        const Val r = call(e.fn, args, e.argn, has);
        return has ? r : Val::I(0);
      }
    }
    return Val::I(0);
  }

  // ------------------------------------------------------ statements --
  Flow exec_list(const CFunc& F, const std::vector<int>& body) {
    for (int si : body)
      if (exec(F, F.st[si]) == Flow::Ret) return Flow::Ret;
    return Flow::Next;
  }

  Flow exec(const CFunc& F, const CStmt& s) {
    step();
    switch (s.k) {
      case SK::Let: {  // interp.cpp:290-321
        if (s.lt == LocalType::Vec4 || s.lt == LocalType::Vec8) {  // zero lanes
          Slot& d = S(s.slot);
          d = Slot{};
          return Flow::Next;
        }
        const bool r32 = s.lt == LocalType::F32;
        Val v = s.lt == LocalType::I64 ? Val::I(0) : Val::F(0.0);
        if (s.e0 >= 0) {
          if (s.lt == LocalType::I64) {
            v = F.ex[s.e0].ty == TY_INT ? Val::I(ieval(F, s.e0)) : eval(F, s.e0);
          } else {
            const double x = dval(F, s.e0);
            v = Val::F(r32 ? (double)(float)x : x);
          }
        }
        Slot& d = S(s.slot);
        d.v = v;
        d.round_f32 = r32;
        return Flow::Next;
      }
      case SK::Assign: {  // interp.cpp:323-331
        const int8_t t = F.ex[s.e0].ty;
        if (F.slot_ty[s.slot] == TY_FLT && t != TY_DYN) {  // a float variable: the value as a double
          const double x = dval(F, s.e0);
          Slot& slot = S(s.slot);
          slot.v = Val::F(slot.round_f32 ? (double)(float)x : x);
          return Flow::Next;
        }
        if (F.slot_ty[s.slot] == TY_INT && t == TY_INT) {
          const long long x = ieval(F, s.e0);
          S(s.slot).v = Val::I(x);
          return Flow::Next;
        }
        const Val v = eval(F, s.e0);
        Slot& slot = S(s.slot);
        if (slot.v.is_int)
          slot.v = v;
        else
          slot.v = Val::F(slot.round_f32 ? (double)(float)v.d() : v.d());
        return Flow::Next;
      }
      case SK::Store: {  // interp.cpp:333-337
        const long long off = ival(F, s.e0);
        const double v = dval(F, s.e1);
        store(S(s.ptr).region, off, v);
        return Flow::Next;
      }
      case SK::For: {  // interp.cpp:339-353
        const long long lo = ival(F, s.e0);
        const long long hi = ival(F, s.e1);
        const long long st = s.e2 >= 0 ? ival(F, s.e2) : 1;
        if (st <= 0) throw Fault{ExecStatus::RuntimeFault, "loop step must be positive"};
        for (long long iv = lo; iv < hi; iv += st) {
          Slot& lv = S(s.slot);  // a fresh int scalar every iteration (interp.cpp:344-347)
          lv.v = Val::I(iv);
          lv.round_f32 = false;
          if (exec_list(F, s.body) == Flow::Ret) return Flow::Ret;
        }
        return Flow::Next;
      }
      case SK::While:  // interp.cpp:354-359
        while (truth(F, s.e0)) {
          step();
          if (exec_list(F, s.body) == Flow::Ret) return Flow::Ret;
        }
        return Flow::Next;
      case SK::If:
        return exec_list(F, truth(F, s.e0) ? s.body : s.els);
      case SK::Call:
        eval(F, s.e0);
        return Flow::Next;
      case SK::Return:  // interp.cpp:368-375
        has_ret = false;
        if (s.e0 >= 0) {
          ret = eval(F, s.e0);
          has_ret = true;
        }
        return Flow::Ret;
      case SK::VLoad: {  // interp.cpp:385-391
        const long long b = ival(F, s.e0);
        const int r = S(s.ptr).region;
        for (int l = 0; l < s.width; ++l) {
          const double x = load(r, b + l);
          S(s.slot).lanes[l] = x;
        }
        return Flow::Next;
      }
      case SK::VStore: {
        const long long b = ival(F, s.e0);
        const int r = S(s.ptr).region;
        for (int l = 0; l < s.width; ++l) store(r, b + l, S(s.va).lanes[l]);
        return Flow::Next;
      }
      case SK::VSplat: {
        const double v = dval(F, s.e0);
        for (int l = 0; l < s.width; ++l) S(s.slot).lanes[l] = v;
        return Flow::Next;
      }
      case SK::VAdd:
      case SK::VMul:
      case SK::VFma: {  // interp.cpp:405-420
        for (int l = 0; l < s.width; ++l) {
          const double a = S(s.va).lanes[l], b = S(s.vb).lanes[l];
          double& d = S(s.slot).lanes[l];
          if (s.k == SK::VAdd)
            d = a + b;
          else if (s.k == SK::VMul)
            d = a * b;
          else
            d += a * b;
        }
        return Flow::Next;
      }
      case SK::VReduce: {  // interp.cpp:421-428
        double sum = 0.0;
        for (int l = 0; l < s.width; ++l) sum += S(s.va).lanes[l];
        Slot& d = S(s.slot);
        d.v = Val::F(d.round_f32 ? (double)(float)sum : sum);
        return Flow::Next;
      }
    }
    return Flow::Next;
  }
};

// Root arguments (interp.cpp:98-135) in parameter order: ints, floats, pointers.
std::vector<Slot> root_args(Run& R, const FunctionIR& f, const interp::MemoryImage& mem) {
  std::vector<Slot> args;
  for (const auto& p : f.params) {
    Slot s;
    switch (p.kind) {
      case ParamKind::IntScalar: {
        auto it = mem.int_args.find(p.name);
        if (it == mem.int_args.end())
          throw Fault{ExecStatus::RuntimeFault, "missing integer argument '" + p.name + "'"};
        s.v = Val::I(it->second);
        break;
      }
      case ParamKind::FloatScalar: {
        auto it = mem.float_args.find(p.name);
        if (it == mem.float_args.end())
          throw Fault{ExecStatus::RuntimeFault, "missing float argument '" + p.name + "'"};
        s.round_f32 = p.elem == ScalarType::F32;
        s.v = Val::F(s.round_f32 ? (double)(float)it->second : it->second);
        break;
      }
      case ParamKind::Pointer: {
        if (R.mode == ExecMode::Plain && !mem.regions.count(p.name))
          throw Fault{ExecStatus::RuntimeFault, "missing region '" + p.name + "'"};
        s.region = (int)R.keys.size();
        R.keys.push_back(p.name);
        break;
      }
    }
    args.push_back(s);
  }
  return args;
}

}  // namespace

HostVm::HostVm(const Program& prog) : prog_(std::make_unique<VmProgram>()) {
  VmProgram& P = *prog_;
  P.fns.resize(prog.functions.size());
  for (size_t i = 0; i < prog.functions.size(); ++i) {
    P.fns[i].ir = &prog.functions[i];
    P.index.emplace(prog.functions[i].name, (int)i);
  }
  for (auto& F : P.fns) {
    Compiler c{P, F, {}};
    c.scopes.emplace_back();
    for (const auto& p : F.ir->params)
      c.declare(p.name, p.kind == ParamKind::IntScalar ? TY_INT : p.kind == ParamKind::FloatScalar ? TY_FLT : TY_DYN);
    F.body = c.block(F.ir->body, true);
  }
}

HostVm::~HostVm() = default;

interp::ExecutionOutcome HostVm::execute(const std::string& function, const interp::MemoryImage& input,
                                         const interp::InstrumentationPolicy& policy,
                                         unsigned long long step_limit) const {
  if (policy.dispatch && policy.dispatch->handler)
    throw std::logic_error("HostVm: dispatch handlers run on the reference interpreter");
  interp::ExecutionOutcome out;
  Run R(*prog_, policy.mode, step_limit);
  interp::MemoryImage mem = input;
  std::map<std::string, std::vector<bool>> writes;
  if (policy.mode == ExecMode::Plain && policy.track_writes)
    for (const auto& [name, r] : mem.regions) writes[name].assign(r.data.size(), false);
  R.scratch = policy.scratch_value;
  R.extent = policy.target_extent;
  R.record = policy.record_trace;
  auto fit = prog_->index.find(function);
  try {
    if (fit == prog_->index.end())
      throw Fault{ExecStatus::RuntimeFault, "no function named '" + function + "'"};
    const FunctionIR& f = *prog_->fns[fit->second].ir;
    std::vector<Slot> args = root_args(R, f, mem);
    const size_t nr = R.keys.size();
    R.trace.assign(nr, {});
    R.maxoff.assign(nr, -1);
    for (size_t r = 0; r < nr; ++r) {
      if (policy.mode == ExecMode::DimProbe && R.keys[r] == policy.target) R.target = (int)r;
      auto it = mem.regions.find(R.keys[r]);
      R.reg.push_back(it == mem.regions.end() ? nullptr : &it->second);
      auto w = writes.find(R.keys[r]);
      R.wr.push_back(w == writes.end() ? nullptr : &w->second);
    }
    bool has = false;
    const Val rv = R.call(fit->second, args.data(), (int)args.size(), has);
    out.status = ExecStatus::Normal;
    out.has_ret = has;
    if (has) {
      out.ret_is_int = rv.is_int;
      out.ret_int = rv.iv();
      out.ret_float = rv.fv();
    }
    out.final = std::move(mem);
    out.writes = std::move(writes);
    if (R.target >= 0) out.trace = std::move(R.trace[R.target]);
  } catch (const Fault& flt) {
    out.status = flt.status;
    out.fault_msg = flt.msg;
  }
  out.steps = R.steps;
  out.max_target_offset = R.target >= 0 && (size_t)R.target < R.maxoff.size() ? R.maxoff[R.target] : -1;
  return out;
}

std::map<std::string, HostVm::Survey> HostVm::dim_survey(const std::string& function,
                                                         const interp::MemoryImage& input,
                                                         unsigned long long step_limit) const {
  std::map<std::string, Survey> out;
  Run R(*prog_, ExecMode::DimProbe, step_limit);
  R.target = -2;
  R.extent = interp::kUnboundedExtent;
  R.scratch = 1.0;  // InstrumentationPolicy::scratch_value default
  R.record = true;
  auto fit = prog_->index.find(function);
  if (fit == prog_->index.end()) return out;
  const FunctionIR& f = *prog_->fns[fit->second].ir;
  ExecStatus status = ExecStatus::Normal;
  std::string msg;
  try {
    std::vector<Slot> args = root_args(R, f, input);
    const size_t nr = R.keys.size();
    R.trace.assign(nr, {});
    R.maxoff.assign(nr, -1);
    R.dead.assign(nr, 0);
    R.dead_msg.assign(nr, {});
    bool has = false;
    R.call(fit->second, args.data(), (int)args.size(), has);
  } catch (const Fault& flt) {
    status = flt.status;
    msg = flt.msg;
  }
  for (size_t r = 0; r < R.keys.size(); ++r) {
    Survey s;
    s.max_target_offset = r < R.maxoff.size() ? R.maxoff[r] : -1;
    if (r < R.dead.size() && R.dead[r]) {
      s.status = ExecStatus::OutOfBounds;
      s.fault_msg = R.dead_msg[r];
    } else {
      s.status = status;
      s.fault_msg = msg;
      if (status == ExecStatus::Normal && r < R.trace.size()) s.trace = std::move(R.trace[r]);
    }
    out[R.keys[r]] = std::move(s);
  }
  return out;
}

}  // namespace liftc::gpu
