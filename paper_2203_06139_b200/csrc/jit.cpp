// Generic lowering: any Listing-style `global` kernel
// of a DSL module — together with the generated gradients it calls, exactly as
// the reference prints them (adc::print(Module), printer.cpp:60-242) — is
// translated to CUDA C++ and compiled for sm_100a with NVRTC.  This replaces
// the hand-transcribed registry for gradients that have no hand-written
// kernel: the corpus gradients with branches, loops and value/control tapes
// (reverse.cpp:331-676) become launchable.
//
// Semantics follow the reference interpreter (proj/src/eval.cpp:339-703):
//  * every real operation is one IEEE double op in source order (__dadd_rn,
//    __dmul_rn, ... and -fmad=false), integers are int64;
//  * an expression is integer-valued when the interpreter says so
//    (eval.cpp:170-202): integer literals and variables, negation and
//    + - * of integer operands, __pop_ctl(); an integer expression in a real
//    context is converted to double;
//  * slots accumulate (+=), a[i] in an array-parameter position is a length-1
//    slice (eval.cpp:485-499);
//  * domain errors of the interpreter (division by zero, log of a non-positive
//    value, sqrt of a negative value, an index out of range, tape underflow)
//    are detected per thread and reported as ADC_E_EVAL after the launch;
//  * the value / control tapes (__push, __pop, __push_ctl, __pop_ctl) are
//    per call frame, as in the interpreter (eval.cpp:312-319), held in a
//    thread-private array of the chosen capacity.
//  * int64 overflow of + - * (binary, unary minus, +=) raises the
//    interpreter's 'integer overflow' Eval error (eval.cpp:601-628).
//
// Hazards: a whole real[] kernel parameter that is written (directly at an
// index other than the thread index, or through a callee's writes) is a
// shared-write hazard (launch.cpp:112-240); compiling such a kernel is refused
// with the reference's message unless `unsafe`, in which case every indexed
// += into an array compiles to an atomic add (the reference's forced
// parallel mode, eval.cpp:414-423: race-free, order unspecified).
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"

using namespace adcb;

namespace {

// ---- NVRTC, bound at first use (a process may already hold another copy) ------
struct Nvrtc {
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*error_string)(nvrtcResult) = nullptr;
  bool ok = false;
};

const Nvrtc* nvrtc() {
  static Nvrtc N;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    N.ok = sym(N.create, "nvrtcCreateProgram") && sym(N.compile, "nvrtcCompileProgram") &&
           sym(N.log_size, "nvrtcGetProgramLogSize") && sym(N.log, "nvrtcGetProgramLog") &&
           sym(N.cubin_size, "nvrtcGetCUBINSize") && sym(N.cubin, "nvrtcGetCUBIN") &&
           sym(N.destroy, "nvrtcDestroyProgram") && sym(N.error_string, "nvrtcGetErrorString");
  });
  return N.ok ? &N : nullptr;
}

// ---- AST ---------------------------------------------------------------------
enum class VT { Real, RealArray, Integer };

struct Ex;
using ExP = std::unique_ptr<Ex>;
struct Ex {
  enum K { Num, Var, Neg, Bin, Cmp, Call, Index } k = Num;
  double v = 0;
  bool int_lit = false, pi = false;
  std::string name;  // Var / Call (intrinsic) / Index
  char op = 0;       // Bin: + - * /
  std::string cmp;   // Cmp: < <= > >= == !=
  std::vector<ExP> a;
  bool is_int = false;
};

struct St;
using StP = std::unique_ptr<St>;
using Blk = std::vector<StP>;
struct St {
  enum K { Decl, Assign, Return, If, For, Call } k = Decl;
  VT type = VT::Real;
  std::string target;
  bool indexed = false, compound = false;
  ExP index, expr;
  Blk then_b, else_b;
  std::string loop_var;
  ExP lo, hi;
  std::string callee;
  std::vector<ExP> args;
  int line = 0;
};

struct Prm {
  std::string name;
  VT type;
};

struct Fn {
  std::string name;
  bool global = false, returns_void = false;
  std::vector<Prm> params;
  Blk body;
  bool uses_tape = false, uses_ctl = false;
};

struct ParseError {
  std::string msg;
};

// ---- lexer / parser ------------------------------------------------------------
struct Tok {
  enum K { Id, Num, Punct, End } k = End;
  std::string s;
  int line = 0;
};

std::vector<Tok> lex(const std::string& src) {
  std::vector<Tok> t;
  size_t i = 0;
  int line = 1;
  while (i < src.size()) {
    const char c = src[i];
    if (c == '\n') {
      ++line;
      ++i;
    } else if (std::isspace((unsigned char)c)) {
      ++i;
    } else if (c == '/' && i + 1 < src.size() && src[i + 1] == '/') {
      while (i < src.size() && src[i] != '\n') ++i;
    } else if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < src.size() && (std::isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      t.push_back({Tok::Id, src.substr(i, j - i), line});
      i = j;
    } else if (std::isdigit((unsigned char)c) ||
               (c == '.' && i + 1 < src.size() && std::isdigit((unsigned char)src[i + 1]))) {
      size_t j = i;
      while (j < src.size() && (std::isdigit((unsigned char)src[j]) || src[j] == '.')) ++j;
      if (j < src.size() && (src[j] == 'e' || src[j] == 'E')) {
        size_t k = j + 1;
        if (k < src.size() && (src[k] == '+' || src[k] == '-')) ++k;
        if (k < src.size() && std::isdigit((unsigned char)src[k])) {
          j = k;
          while (j < src.size() && std::isdigit((unsigned char)src[j])) ++j;
        }
      }
      t.push_back({Tok::Num, src.substr(i, j - i), line});
      i = j;
    } else {
      static const char* two[] = {"<=", ">=", "==", "!=", "+="};
      std::string p(1, c);
      for (const char* tw : two)
        if (src.compare(i, 2, tw) == 0) p = tw;
      if (std::strchr("(){}[],;+-*/<>=", c) == nullptr)
        throw ParseError{"line " + std::to_string(line) + ": unexpected character '" + p + "'"};
      t.push_back({Tok::Punct, p, line});
      i += p.size();
    }
  }
  t.push_back({Tok::End, "", line});
  return t;
}

struct Parser {
  std::vector<Tok> t;
  size_t i = 0;
  const Tok& peek(size_t k = 0) const { return t[std::min(i + k, t.size() - 1)]; }
  bool is(const char* s, size_t k = 0) const { return peek(k).s == s && peek(k).k != Tok::End; }
  [[noreturn]] void error(const std::string& m) const {
    throw ParseError{"line " + std::to_string(peek().line) + ": " + m};
  }
  void expect(const char* s) {
    if (!is(s)) error(std::string("expected '") + s + "', got '" + peek().s + "'");
    ++i;
  }
  std::string ident() {
    if (peek().k != Tok::Id) error("expected identifier, got '" + peek().s + "'");
    return t[i++].s;
  }

  VT type() {
    const std::string n = ident();
    if (n == "integer") return VT::Integer;
    if (n != "real") error("unknown type '" + n + "'");
    if (is("[")) {
      expect("[");
      expect("]");
      return VT::RealArray;
    }
    return VT::Real;
  }

  ExP primary() {
    auto e = std::make_unique<Ex>();
    if (peek().k == Tok::Num) {
      const std::string s = t[i++].s;
      e->k = Ex::Num;
      e->v = std::strtod(s.c_str(), nullptr);
      e->int_lit = s.find_first_of(".eE") == std::string::npos;
      return e;
    }
    if (is("(")) {
      expect("(");
      ExP in = expr();
      expect(")");
      return in;
    }
    const std::string n = ident();
    if (n == "PI") {
      e->k = Ex::Num;
      e->pi = true;
      e->v = 3.14159265358979323846;  // ast.cpp:119-123
      return e;
    }
    if (is("(")) {
      expect("(");
      e->k = Ex::Call;
      e->name = n;
      if (!is(")")) {
        e->a.push_back(expr());
        while (is(",")) {
          expect(",");
          e->a.push_back(expr());
        }
      }
      expect(")");
      return e;
    }
    if (is("[")) {
      expect("[");
      e->k = Ex::Index;
      e->name = n;
      e->a.push_back(expr());
      expect("]");
      return e;
    }
    e->k = Ex::Var;
    e->name = n;
    return e;
  }
  ExP unary() {
    if (is("-")) {
      expect("-");
      ExP in = unary();
      // a negated literal is a signed constant (parser.cpp:482-487; PI stays
      // a negation) — no unary-minus op at run time, as in the interpreter
      if (in->k == Ex::Num && !in->pi) {
        in->v = -in->v;
        return in;
      }
      auto e = std::make_unique<Ex>();
      e->k = Ex::Neg;
      e->a.push_back(std::move(in));
      return e;
    }
    return primary();
  }
  ExP term() {
    ExP l = unary();
    while (is("*") || is("/")) {
      auto e = std::make_unique<Ex>();
      e->k = Ex::Bin;
      e->op = t[i++].s[0];
      e->a.push_back(std::move(l));
      e->a.push_back(unary());
      l = std::move(e);
    }
    return l;
  }
  ExP arith() {
    ExP l = term();
    while (is("+") || is("-")) {
      auto e = std::make_unique<Ex>();
      e->k = Ex::Bin;
      e->op = t[i++].s[0];
      e->a.push_back(std::move(l));
      e->a.push_back(term());
      l = std::move(e);
    }
    return l;
  }
  ExP expr() {
    ExP l = arith();
    for (const char* c : {"<", "<=", ">", ">=", "==", "!="}) {
      if (is(c)) {
        auto e = std::make_unique<Ex>();
        e->k = Ex::Cmp;
        e->cmp = t[i++].s;
        e->a.push_back(std::move(l));
        e->a.push_back(arith());
        return e;
      }
    }
    return l;
  }

  Blk block() {
    expect("{");
    Blk b;
    while (!is("}")) {
      if (peek().k == Tok::End) error("unterminated block");
      b.push_back(stmt());
    }
    expect("}");
    return b;
  }

  StP stmt() {
    auto s = std::make_unique<St>();
    s->line = peek().line;
    if (is("real") || is("integer")) {
      s->k = St::Decl;
      s->type = type();
      s->target = ident();
      expect("=");
      s->expr = expr();
      expect(";");
      return s;
    }
    if (is("return")) {
      ++i;
      s->k = St::Return;
      s->expr = expr();
      expect(";");
      return s;
    }
    if (is("if")) {
      ++i;
      s->k = St::If;
      expect("(");
      s->expr = expr();
      expect(")");
      s->then_b = block();
      if (is("else")) {
        ++i;
        if (is("if")) s->else_b.push_back(stmt());
        else s->else_b = block();
      }
      return s;
    }
    if (is("for")) {
      ++i;
      s->k = St::For;
      expect("(");
      if (ident() != "integer") error("for loop variable must be integer");
      s->loop_var = ident();
      expect("=");
      s->lo = expr();
      expect(";");
      if (ident() != s->loop_var) error("for condition must test the loop variable");
      expect("<");
      s->hi = expr();
      expect(";");
      if (ident() != s->loop_var) error("for step must advance the loop variable");
      expect("+=");
      if (peek().s != "1") error("for step must be += 1");
      ++i;
      expect(")");
      s->then_b = block();
      return s;
    }
    const std::string n = ident();
    if (is("(")) {
      s->k = St::Call;
      s->callee = n;
      expect("(");
      if (!is(")")) {
        s->args.push_back(expr());
        while (is(",")) {
          expect(",");
          s->args.push_back(expr());
        }
      }
      expect(")");
      expect(";");
      return s;
    }
    s->k = St::Assign;
    s->target = n;
    if (is("[")) {
      expect("[");
      s->indexed = true;
      s->index = expr();
      expect("]");
    }
    if (is("+=")) {
      s->compound = true;
      ++i;
    } else {
      expect("=");
    }
    s->expr = expr();
    expect(";");
    return s;
  }

  Fn function() {
    Fn f;
    while (is("device") || is("host") || is("global")) {
      if (is("global")) f.global = true;
      ++i;
    }
    if (is("void")) {
      ++i;
      f.returns_void = true;
    } else if (ident() != "real") {
      error("functions return real or void");
    }
    f.name = ident();
    expect("(");
    if (!is(")")) {
      for (;;) {
        Prm p;
        p.type = type();
        p.name = ident();
        f.params.push_back(p);
        if (!is(",")) break;
        expect(",");
      }
    }
    expect(")");
    f.body = block();
    return f;
  }
};

// ---- typing --------------------------------------------------------------------
const std::set<std::string> kIntrinsics = {"sin", "cos", "tan", "exp", "log",
                                           "sqrt", "pow", "fabs", "__pop", "__pop_ctl"};
const std::set<std::string> kKernelBuiltins = {"blockIdx", "blockDim", "threadIdx", "N"};

struct Scope {
  std::vector<std::map<std::string, VT>> frames;
  bool global = false;
  void push() { frames.emplace_back(); }
  void pop() { frames.pop_back(); }
  void add(const std::string& n, VT t) { frames.back()[n] = t; }
  bool find(const std::string& n, VT& t) const {
    for (auto it = frames.rbegin(); it != frames.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) {
        t = f->second;
        return true;
      }
    }
    if (global && kKernelBuiltins.count(n)) {
      t = VT::Integer;
      return true;
    }
    return false;
  }
};

void type_expr(Ex& e, const Scope& sc, Fn& f) {
  for (auto& c : e.a) type_expr(*c, sc, f);
  VT t;
  switch (e.k) {
    case Ex::Num: e.is_int = e.int_lit; break;
    case Ex::Var:
      if (!sc.find(e.name, t)) throw ParseError{"unknown variable '" + e.name + "' in " + f.name};
      if (t == VT::RealArray)
        throw ParseError{"array '" + e.name + "' used as a value in " + f.name};
      e.is_int = t == VT::Integer;
      break;
    case Ex::Neg: e.is_int = e.a[0]->is_int; break;
    case Ex::Bin: e.is_int = e.op != '/' && e.a[0]->is_int && e.a[1]->is_int; break;
    case Ex::Cmp: e.is_int = false; break;
    case Ex::Call:
      if (!kIntrinsics.count(e.name))
        throw ParseError{"unknown function '" + e.name + "' in an expression of " + f.name};
      if (e.name == "__pop") f.uses_tape = true;
      if (e.name == "__pop_ctl") f.uses_ctl = true;
      e.is_int = e.name == "__pop_ctl";
      break;
    case Ex::Index:
      if (!sc.find(e.name, t) || t != VT::RealArray)
        throw ParseError{"'" + e.name + "' is not an array in " + f.name};
      e.is_int = false;
      break;
  }
}

void type_block(Blk& b, Scope& sc, Fn& f) {
  sc.push();
  for (auto& sp : b) {
    St& s = *sp;
    switch (s.k) {
      case St::Decl:
        type_expr(*s.expr, sc, f);
        sc.add(s.target, s.type);
        break;
      case St::Assign: {
        VT t;
        if (!sc.find(s.target, t)) throw ParseError{"unknown variable '" + s.target + "'"};
        if (s.indexed) type_expr(*s.index, sc, f);
        type_expr(*s.expr, sc, f);
        break;
      }
      case St::Return: type_expr(*s.expr, sc, f); break;
      case St::If:
        type_expr(*s.expr, sc, f);
        type_block(s.then_b, sc, f);
        type_block(s.else_b, sc, f);
        break;
      case St::For:
        type_expr(*s.lo, sc, f);
        type_expr(*s.hi, sc, f);
        sc.push();
        sc.add(s.loop_var, VT::Integer);
        type_block(s.then_b, sc, f);
        sc.pop();
        break;
      case St::Call:
        if (s.callee == "__push") f.uses_tape = true;
        if (s.callee == "__push_ctl") f.uses_ctl = true;
        for (auto& a : s.args) {
          VT t;
          if (a->k == Ex::Var && sc.find(a->name, t) && t == VT::RealArray) continue;  // whole array
          type_expr(*a, sc, f);
        }
        break;
    }
  }
  sc.pop();
}

// ---- hazard analysis (launch.cpp:112-240, conservatively) -------------------------
// Which array parameters a function writes (directly or through callees).
struct Module {
  std::vector<Fn> fns;
  const Fn* find(const std::string& n) const {
    for (auto& f : fns)
      if (f.name == n) return &f;
    return nullptr;
  }
};

void collect_writes(const Module& m, const Fn& f, std::set<std::string>& written,
                    std::set<std::string>& visiting);

void block_writes(const Module& m, const Blk& b, std::set<std::string>& w,
                  std::set<std::string>& visiting) {
  for (auto& sp : b) {
    const St& s = *sp;
    if (s.k == St::Assign && s.indexed) w.insert(s.target);
    if (s.k == St::If) {
      block_writes(m, s.then_b, w, visiting);
      block_writes(m, s.else_b, w, visiting);
    }
    if (s.k == St::For) block_writes(m, s.then_b, w, visiting);
    if (s.k == St::Call) {
      const Fn* c = m.find(s.callee);
      if (c == nullptr) continue;
      std::set<std::string> cw;
      collect_writes(m, *c, cw, visiting);
      for (size_t a = 0; a < s.args.size() && a < c->params.size(); ++a)
        if (cw.count(c->params[a].name) &&
            (s.args[a]->k == Ex::Var || s.args[a]->k == Ex::Index))
          w.insert(s.args[a]->name);
    }
  }
}

void collect_writes(const Module& m, const Fn& f, std::set<std::string>& written,
                    std::set<std::string>& visiting) {
  if (visiting.count(f.name)) return;
  visiting.insert(f.name);
  block_writes(m, f.body, written, visiting);
  visiting.erase(f.name);
}

// Shared-write hazards of a global kernel: array params written other than
// through the thread-indexed slice `a[i]` of `integer i = blockIdx*blockDim+threadIdx`.
bool is_thread_index_decl(const St& s) {
  if (s.k != St::Decl || s.type != VT::Integer) return false;
  const Ex& e = *s.expr;
  if (e.k != Ex::Bin || e.op != '+') return false;
  const Ex& m = *e.a[0];
  return m.k == Ex::Bin && m.op == '*' && m.a[0]->k == Ex::Var && m.a[0]->name == "blockIdx" &&
         m.a[1]->k == Ex::Var && m.a[1]->name == "blockDim" && e.a[1]->k == Ex::Var &&
         e.a[1]->name == "threadIdx";
}

void kernel_hazards(const Module& m, const Blk& b, const std::string& tid,
                    const std::set<std::string>& arrays, std::map<std::string, std::string>& haz,
                    std::string& tvar) {
  for (auto& sp : b) {
    const St& s = *sp;
    if (is_thread_index_decl(s)) tvar = s.target;
    if (s.k == St::Assign && s.indexed && arrays.count(s.target)) {
      if (!(s.index->k == Ex::Var && s.index->name == tvar && !tvar.empty()))
        haz[s.target] = "written at an index other than the thread index";
    }
    if (s.k == St::If) {
      kernel_hazards(m, s.then_b, tid, arrays, haz, tvar);
      kernel_hazards(m, s.else_b, tid, arrays, haz, tvar);
    }
    if (s.k == St::For) kernel_hazards(m, s.then_b, tid, arrays, haz, tvar);
    if (s.k == St::Call) {
      const Fn* c = m.find(s.callee);
      if (c == nullptr) continue;
      std::set<std::string> cw, vis;
      collect_writes(m, *c, cw, vis);
      for (size_t a = 0; a < s.args.size() && a < c->params.size(); ++a) {
        const Ex& arg = *s.args[a];
        if (!cw.count(c->params[a].name) || !arrays.count(arg.name)) continue;
        if (arg.k == Ex::Var)
          haz[arg.name] = "whole array shared with a writing callee across threads";
        else if (arg.k == Ex::Index && !(arg.a[0]->k == Ex::Var && arg.a[0]->name == tvar))
          haz[arg.name] = "slice at an index other than the thread index written by a callee";
      }
    }
  }
}

// ---- CUDA emission ---------------------------------------------------------------
// Static tape (tape elimination by SSA renaming).  The
// value / control tapes of the generated code (reverse.cpp:335-382 pushes in
// the forward sweep, 432-466 pops in the reversed loops) are LIFO per call
// frame, so wherever the tape depth at a push or pop is a compile-time
// constant, the entry is a plain local variable: push at depth d writes
// _tv<d>, the matching pop reads it back — registers instead of a
// thread-private array in local memory.  The depth is static through
//  * straight-line code;
//  * if/else whose branches move the depth by different amounts: forward
//    branches (net pushes) all start at the same depth and the depth after the
//    statement is padded to the largest branch; reverse branches (net pops)
//    start where their forward branch ended (depth - max + own), so each
//    reverse branch reads back exactly the slots its forward branch wrote;
//  * loops whose body leaves both depths unchanged (slots reused every
//    iteration);
//  * loops with a compile-time trip count (integer kernel arguments are
//    specialised per launch, integer locals, loop variables and control-tape
//    entries folded), fully unrolled;
// otherwise (data-dependent trip counts that push, deep unrolling) the
// function keeps the dynamic tape.  Pops and pushes happen at the same points
// in the same order with the same values, so results are the same bits.
struct Dynamic {};

struct Emitter {
  const Module& m;
  bool unsafe;
  int tape_cap;
  bool prefetch = true;
  // static-tape state of the function frame being emitted
  struct Frame {
    bool stat = false;
    int dv = 0, dc = 0, maxv = 0, maxc = 0;
    std::map<std::string, long long> ienv;  // integer variables holding a known constant
    std::map<int, long long> ctlval;        // control-tape slots holding a known constant
    std::set<int> wide;  // control slots that may hold a value beyond int32 (others: int)
  };
  Frame fr;
  long long unrolled_stmts = 0;  // emission budget of the unrolled code (per module)
  static constexpr long long kUnrollBudget = 20000;
  static constexpr long long kMaxTrip = 512;
  // specialisations: key (function, cached, integer constants) -> emitted name
  std::map<std::string, std::string> spec;
  std::set<std::string> spec_active;
  bool all_static = true;  // every callee specialisation got a static tape
  std::ostringstream spec_decls, spec_defs;
  int spec_count = 0;
  // Counting variant (LaunchStats): every interpreter-counted operation of
  // eval.cpp increments the thread's counter (adds: +, -, unary -, compound
  // +=; muls; divs; intrinsics; comparisons: each if condition; tape pushes
  // and pops) and every kernel-frame statement increments `st`.
  bool count = false;
  std::string C(const char* field, const std::string& e) const {
    return count ? "(++ctx.cnt->" + std::string(field) + ", " + e + ")" : e;
  }
  void Cst(const char* field, int d) {
    if (count) o << ind(d) << "++ctx.cnt->" << field << ";\n";
  }
  // Slot caching: a void function whose array parameters are only ever
  // accessed at the literal index 0 (the length-1 slices of Listing-1 slots)
  // gets a second variant fn_<name>_c that keeps each such slot in a
  // register for the whole call (one load at entry, one store at exit if
  // written) instead of a global read-modify-write per `+=` statement.  Used
  // only where the call's array arguments are pairwise distinct kernel arrays
  // (no aliasing; BufferSet arrays are distinct) and never when unsafe.
  std::map<std::string, std::vector<int>> cacheable;  // fn -> per param: 0 no, 1 read, 2 written
  const std::set<std::string>* cached = nullptr;      // params cached in the variant being emitted
  std::ostringstream o;
  int tmp = 0;

  // DSL identifiers get a prefix so they can never clash with C++/CUDA names
  // or the emitter's own (tape, ctx, N, ...).
  static std::string V(const std::string& n) { return "v_" + n; }

  static std::string dbl(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    std::string s = b;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    if (s == "inf") return "__longlong_as_double(0x7ff0000000000000LL)";
    return s;
  }
  std::string ind(int d) { return std::string(2 * d, ' '); }

  // Compile-time value of an integer expression in the current frame (static
  // tape mode), or nothing; overflow is left to the run-time check.
  bool fold(const Ex& e, long long& v) const {
    if (!fr.stat || !e.is_int) return false;
    long long a, b;
    switch (e.k) {
      case Ex::Num: v = (long long)e.v; return true;
      case Ex::Var: {
        auto it = fr.ienv.find(e.name);
        if (it == fr.ienv.end()) return false;
        v = it->second;
        return true;
      }
      case Ex::Neg:
        if (!fold(*e.a[0], a) || a == (-9223372036854775807LL - 1)) return false;
        v = -a;
        return true;
      case Ex::Bin:
        if (!fold(*e.a[0], a) || !fold(*e.a[1], b)) return false;
        if (e.op == '+') return !__builtin_add_overflow(a, b, &v);
        if (e.op == '-') return !__builtin_sub_overflow(a, b, &v);
        if (e.op == '*') return !__builtin_mul_overflow(a, b, &v);
        return false;
      case Ex::Call: {
        if (e.name != "__pop_ctl" || fr.dc <= 0) return false;
        auto it = fr.ctlval.find(fr.dc - 1);
        if (it == fr.ctlval.end()) return false;
        v = it->second;
        return true;
      }
      default: return false;
    }
  }
  static int count_pops(const Ex& e) {
    int n = e.k == Ex::Call && (e.name == "__pop" || e.name == "__pop_ctl");
    for (auto& c : e.a) n += count_pops(*c);
    return n;
  }
  // beyond this many live entries per frame the registers would spill to
  // local memory anyway: keep the dynamic tape
  static constexpr int kMaxStaticSlots = 64;
  void note_push_v() {
    fr.maxv = std::max(fr.maxv, ++fr.dv);
    if (fr.maxv > kMaxStaticSlots) throw Dynamic{};
  }
  void note_push_c() {
    fr.maxc = std::max(fr.maxc, ++fr.dc);
    if (fr.maxc > kMaxStaticSlots) throw Dynamic{};
  }

  // integer-valued expression (only called when e.is_int)
  std::string ie(const Ex& e) {
    switch (e.k) {
      case Ex::Num: return "(long long)" + std::to_string((long long)e.v);
      case Ex::Var:
        if (e.name == "blockIdx") return "(long long)blockIdx.x";
        if (e.name == "blockDim") return "(long long)blockDim.x";
        if (e.name == "threadIdx") return "(long long)threadIdx.x";
        if (e.name == "N") return "N";
        if (fr.stat && fr.ienv.count(e.name))
          return "(long long)" + std::to_string(fr.ienv.at(e.name)) + "LL";
        return V(e.name);
      // int64 arithmetic with the interpreter's overflow errors (eval.cpp:601-628)
      case Ex::Neg: return C("a", "adc_ineg(" + ie(*e.a[0]) + ", ctx)");
      case Ex::Bin:
        return C(e.op == '*' ? "m" : "a",
                 std::string(e.op == '+' ? "adc_iadd(" : e.op == '-' ? "adc_isub(" : "adc_imul(") +
                     ie(*e.a[0]) + ", " + ie(*e.a[1]) + ", ctx)");
      case Ex::Call:
        if (fr.stat) {
          if (fr.dc <= 0) throw Dynamic{};  // underflow: the dynamic tape reports it
          return "_tc" + std::to_string(--fr.dc);
        }
        return C("po", "adc_pop_ctl(ctl, cp, ctx)");
      default: return "0";
    }
  }
  // real-valued expression (an integer expression is converted, eval.cpp:526)
  std::string re(const Ex& e) {
    if (e.is_int) return "(double)" + ie(e);
    switch (e.k) {
      case Ex::Num: return dbl(e.v);
      case Ex::Var: return V(e.name);
      case Ex::Neg: return C("a", "(-" + re(*e.a[0]) + ")");
      case Ex::Bin: {
        const std::string a = re(*e.a[0]), b = re(*e.a[1]);
        switch (e.op) {
          case '+': return C("a", "__dadd_rn(" + a + ", " + b + ")");
          case '-': return C("a", "__dsub_rn(" + a + ", " + b + ")");
          case '*': return C("m", "__dmul_rn(" + a + ", " + b + ")");
          default: {
            // x / 2^k == x * 2^-k exactly (both are the correctly rounded
            // quotient, subnormals included), and the divisor is not 0
            const Ex& d = *e.a[1];
            int ex = 0;
            if (d.k == Ex::Num && !d.pi && d.v != 0.0 && std::isfinite(d.v) &&
                std::fabs(std::frexp(d.v, &ex)) == 0.5 && ex >= -1020 && ex <= 1020)
              return C("d", "__dmul_rn(" + a + ", " + dbl(1.0 / d.v) + ")");
            return C("d", "adc_div(" + a + ", " + b + ", ctx)");
          }
        }
      }
      case Ex::Call: {
        if (e.name == "__pop") {
          if (fr.stat) {
            if (fr.dv <= 0) throw Dynamic{};
            return "_tv" + std::to_string(--fr.dv);
          }
          return C("po", "adc_pop(tape, tp, ctx)");
        }
        std::vector<std::string> a;
        for (auto& c : e.a) a.push_back(re(*c));
        if (e.name == "log") return C("i", "adc_log(" + a[0] + ", ctx)");
        if (e.name == "sqrt") return C("i", "adc_sqrt(" + a[0] + ", ctx)");
        if (e.name == "pow") return C("i", "pow(" + a[0] + ", " + a[1] + ")");
        return C("i", e.name + "(" + a[0] + ")");
      }
      case Ex::Index:
        if (cached != nullptr && cached->count(e.name)) return "c_" + V(e.name);
        return "adc_ld(" + V(e.name) + ", " + ie_any(*e.a[0]) + ", ctx)";
      default: return "0.0";
    }
  }
  // an index: the interpreter evaluates it with eval_int (must be integer)
  std::string ie_any(const Ex& e) {
    if (!e.is_int) throw ParseError{"array index is not an integer expression"};
    return ie(e);
  }
  std::string cond(const Ex& e) {
    if (e.k != Ex::Cmp) throw ParseError{"condition must be a comparison"};
    const bool ints = e.a[0]->is_int && e.a[1]->is_int;
    const std::string a = ints ? ie(*e.a[0]) : re(*e.a[0]);
    const std::string b = ints ? ie(*e.a[1]) : re(*e.a[1]);
    return "(" + a + " " + e.cmp + " " + b + ")";
  }

  void block(const Blk& b, const Fn& f, Scope& sc, int d) {
    sc.push();
    for (auto& sp : b) stmt(*sp, f, sc, d);
    sc.pop();
  }

  // Integer variables a block may assign (their constants are forgotten
  // around code that may run a data-dependent number of times).
  static void assigned_ints(const Blk& b, std::set<std::string>& out) {
    for (auto& sp : b) {
      const St& s = *sp;
      if ((s.k == St::Decl || (s.k == St::Assign && !s.indexed)) && !s.target.empty())
        out.insert(s.target);
      if (s.k == St::For) out.insert(s.loop_var);
      assigned_ints(s.then_b, out);
      assigned_ints(s.else_b, out);
    }
  }

  // Emits `b` into a scratch stream and returns the frame state after it (the
  // emitter's own state is restored): the depth a block leaves behind.
  Frame dry_block(const Blk& b, const Fn& f, Scope& sc, int d) {
    const Frame saved = fr;
    const int saved_tmp = tmp;
    const long long saved_budget = unrolled_stmts;
    std::ostringstream scratch;
    std::swap(o, scratch);
    Frame out;
    try {
      block(b, f, sc, d);
      out = fr;
    } catch (...) {
      std::swap(o, scratch);
      fr = saved;
      tmp = saved_tmp;
      unrolled_stmts = saved_budget;
      throw;
    }
    std::swap(o, scratch);
    fr = saved;
    tmp = saved_tmp;
    unrolled_stmts = saved_budget;
    return out;
  }

  // Start depth of each branch of an if (static tape; see the Dynamic note).
  static void branch_starts(int d0, int e1, int e2, int& s1, int& s2, int& after) {
    const int a = e1 - d0, b = e2 - d0;
    if (a == b) {
      s1 = s2 = d0;
      after = e1;
    } else if (a >= 0 && b >= 0) {  // forward: pad to the larger branch
      s1 = s2 = d0;
      after = d0 + std::max(a, b);
    } else if (a <= 0 && b <= 0) {  // reverse: each branch reads its forward branch's slots
      const int mn = std::min(a, b);
      s1 = d0 + mn - a;
      s2 = d0 + mn - b;
      after = d0 + mn;
    } else {
      throw Dynamic{};
    }
  }

  void stmt(const St& s, const Fn& f, Scope& sc, int d) {
    VT t;
    if (f.global) Cst("st", d);  // eval.cpp:402, the kernel frame's statements
    if (s.k == St::Assign && s.compound) Cst("a", d);  // eval.cpp:420-447
    if (s.k == St::If) Cst("c", d);                    // eval.cpp:647
    if (s.k == St::Call && (s.callee == "__push" || s.callee == "__push_ctl")) Cst("pu", d);
    if (fr.stat) {
      int pops = (s.expr ? count_pops(*s.expr) : 0) + (s.index ? count_pops(*s.index) : 0);
      for (auto& a : s.args) pops += count_pops(*a);
      if (pops > 1) throw Dynamic{};  // several pops in one statement: keep the dynamic tape
      if (++unrolled_stmts > kUnrollBudget) throw Dynamic{};
    }
    switch (s.k) {
      case St::Decl: {
        long long cv = 0;
        const bool known = s.type == VT::Integer && fold(*s.expr, cv);
        if (s.type == VT::Integer)
          o << ind(d) << "long long " << V(s.target) << " = " << ie_any(*s.expr) << ";\n";
        else
          o << ind(d) << "double " << V(s.target) << " = " << re(*s.expr) << ";\n";
        if (f.global && prefetch && is_thread_index_decl(s)) {
          // Every array the kernel touches at the thread index: start its DRAM
          // read now (L2 prefetch), so a thread's loads of x[i], ... and of
          // the slots' read-modify-writes are in flight together.
          std::set<std::string> seen;
          prefetch_scan(f.body, s.target, seen);
          for (const auto& a : seen)
            o << ind(d) << "if (" << V(s.target) << " >= 0 && " << V(s.target) << " < " << V(a)
              << ".len) asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(" << V(a)
              << ".p + " << V(s.target) << "));\n";
        }
        sc.add(s.target, s.type);
        if (known) fr.ienv[s.target] = cv;
        else fr.ienv.erase(s.target);
        break;
      }
      case St::Assign:
        sc.find(s.target, t);
        if (s.indexed && cached != nullptr && cached->count(s.target)) {
          const std::string v = re(*s.expr);
          const std::string c = "c_" + V(s.target);
          if (s.compound) o << ind(d) << c << " = __dadd_rn(" << c << ", " << v << ");\n";
          else o << ind(d) << c << " = " << v << ";\n";
        } else if (s.indexed) {
          const std::string idx = ie_any(*s.index), v = re(*s.expr);
          if (s.compound)
            o << ind(d) << (unsafe ? "adc_st_add_atomic(" : "adc_st_add(") << V(s.target) << ", "
              << idx << ", " << v << ", ctx);\n";
          else
            o << ind(d) << "adc_st(" << V(s.target) << ", " << idx << ", " << v << ", ctx);\n";
        } else if (t == VT::Integer) {
          long long cv = 0, ev = 0;
          bool known = fold(*s.expr, ev);
          if (known && s.compound) {
            auto it = fr.ienv.find(s.target);
            known = it != fr.ienv.end() && !__builtin_add_overflow(it->second, ev, &cv);
          } else {
            cv = ev;
          }
          const std::string v = ie_any(*s.expr);
          if (s.compound)
            o << ind(d) << V(s.target) << " = adc_iadd(" << V(s.target) << ", " << v << ", ctx);\n";
          else o << ind(d) << V(s.target) << " = " << v << ";\n";
          if (known) fr.ienv[s.target] = cv;
          else fr.ienv.erase(s.target);
        } else {
          const std::string v = re(*s.expr);
          if (s.compound)
            o << ind(d) << V(s.target) << " = __dadd_rn(" << V(s.target) << ", " << v << ");\n";
          else
            o << ind(d) << V(s.target) << " = " << v << ";\n";
        }
        break;
      case St::Return:
        o << ind(d) << "return " << re(*s.expr) << ";\n";
        break;
      case St::If: {
        if (!fr.stat) {
          o << ind(d) << "if " << cond(*s.expr) << " {\n";
          block(s.then_b, f, sc, d + 1);
          o << ind(d) << "}";
          if (!s.else_b.empty()) {
            o << " else {\n";
            block(s.else_b, f, sc, d + 1);
            o << ind(d) << "}";
          }
          o << "\n";
          break;
        }
        o << ind(d) << "if " << cond(*s.expr) << " {\n";  // (a condition never pops)
        const Frame f1 = dry_block(s.then_b, f, sc, d + 1);
        const Frame f2 = dry_block(s.else_b, f, sc, d + 1);
        int v1, v2, va, c1, c2, ca;
        branch_starts(fr.dv, f1.dv, f2.dv, v1, v2, va);
        branch_starts(fr.dc, f1.dc, f2.dc, c1, c2, ca);
        const Frame base = fr;
        fr.dv = v1;
        fr.dc = c1;
        block(s.then_b, f, sc, d + 1);
        const Frame t1 = fr;
        fr = base;
        fr.maxv = std::max(fr.maxv, t1.maxv);
        fr.maxc = std::max(fr.maxc, t1.maxc);
        fr.wide = t1.wide;
        fr.dv = v2;
        fr.dc = c2;
        o << ind(d) << "} else {\n";
        block(s.else_b, f, sc, d + 1);
        o << ind(d) << "}\n";
        const Frame t2 = fr;
        fr = base;
        fr.wide = t2.wide;  // (t2 started from t1's: the union)
        fr.maxv = std::max({fr.maxv, t1.maxv, t2.maxv, va});
        fr.maxc = std::max({fr.maxc, t1.maxc, t2.maxc, ca});
        if (fr.maxv > kMaxStaticSlots || fr.maxc > kMaxStaticSlots) throw Dynamic{};
        fr.dv = va;
        fr.dc = ca;
        // constants that both branches agree on survive the statement
        fr.ienv.clear();
        for (auto& kv : t1.ienv) {
          auto it = t2.ienv.find(kv.first);
          if (it != t2.ienv.end() && it->second == kv.second) fr.ienv.insert(kv);
        }
        // control slots written in a branch hold a data-dependent value
        for (int k = std::min(base.dc, ca); k < std::max({base.dc, t1.maxc, t2.maxc, ca}); ++k)
          fr.ctlval.erase(k);
        for (auto& kv : t1.ctlval) {
          auto it = t2.ctlval.find(kv.first);
          if (kv.first < std::min(base.dc, ca) && it != t2.ctlval.end() && it->second == kv.second)
            fr.ctlval[kv.first] = kv.second;
        }
        break;
      }
      case St::For: {
        long long lo = 0, hi = 0;
        const bool const_trip = fold(*s.lo, lo) && fold(*s.hi, hi);
        if (fr.stat) {
          // does the body move the tape depths?
          std::set<std::string> asg;
          assigned_ints(s.then_b, asg);
          Frame probe_base = fr;
          for (auto& v : asg) fr.ienv.erase(v);
          fr.ctlval.clear();
          bool balanced = false;
          sc.push();
          sc.add(s.loop_var, VT::Integer);
          try {
            const Frame body_end = dry_block(s.then_b, f, sc, d + 2);
            balanced = body_end.dv == fr.dv && body_end.dc == fr.dc;
          } catch (Dynamic&) {
            balanced = false;  // e.g. an inner trip count that needs this loop's variable
          }
          sc.pop();
          fr = probe_base;
          if (!balanced) {
            if (!const_trip || hi - lo > kMaxTrip) throw Dynamic{};
            // unrolled: one copy of the body per iteration, the loop variable a constant
            const int k = tmp++;
            o << ind(d) << "{  // unrolled: " << std::max(0LL, hi - lo) << " iterations\n";
            (void)k;
            for (long long it = lo; it < hi; ++it) {
              o << ind(d + 1) << "{\n";
              o << ind(d + 2) << "const long long " << V(s.loop_var) << " = " << it << "LL;\n";
              sc.push();
              sc.add(s.loop_var, VT::Integer);
              fr.ienv[s.loop_var] = it;
              block(s.then_b, f, sc, d + 2);
              fr.ienv.erase(s.loop_var);
              sc.pop();
              o << ind(d + 1) << "}\n";
            }
            o << ind(d) << "}\n";
            break;
          }
          for (auto& v : asg) fr.ienv.erase(v);
          fr.ctlval.clear();  // a body may pop and re-push slots below its start depth
        }
        const int k = tmp++;
        o << ind(d) << "{\n";
        o << ind(d + 1) << "const long long _adc_lo" << k << " = " << ie_any(*s.lo) << ";\n";
        o << ind(d + 1) << "const long long _adc_hi" << k << " = " << ie_any(*s.hi) << ";\n";
        o << ind(d + 1) << "for (long long " << V(s.loop_var) << " = _adc_lo" << k << "; "
          << V(s.loop_var) << " < _adc_hi" << k << "; ++" << V(s.loop_var) << ") {\n";
        sc.push();
        sc.add(s.loop_var, VT::Integer);
        const int cbase = fr.dc;
        block(s.then_b, f, sc, d + 2);
        sc.pop();
        o << ind(d + 1) << "}\n" << ind(d) << "}\n";
        if (fr.stat) {
          std::set<std::string> asg;
          assigned_ints(s.then_b, asg);
          for (auto& v : asg) fr.ienv.erase(v);
          fr.ctlval.clear();
          (void)cbase;
        }
        break;
      }
      case St::Call: {
        if (s.callee == "__push") {
          if (fr.stat) {
            o << ind(d) << "_tv" << fr.dv << " = " << re(*s.args[0]) << ";\n";
            note_push_v();
          } else {
            o << ind(d) << "adc_push(tape, tp, " << re(*s.args[0]) << ", ctx);\n";
          }
          break;
        }
        if (s.callee == "__push_ctl") {
          if (fr.stat) {
            long long cv = 0;
            const bool known = fold(*s.args[0], cv);
            o << ind(d) << "_tc" << fr.dc << " = " << ie_any(*s.args[0]) << ";\n";
            if (known) fr.ctlval[fr.dc] = cv;
            else fr.ctlval.erase(fr.dc);
            if (!known || cv != (long long)(int)cv) fr.wide.insert(fr.dc);
            note_push_c();
          } else {
            o << ind(d) << "adc_push_ctl(ctl, cp, " << ie_any(*s.args[0]) << ", ctx);\n";
          }
          break;
        }
        const Fn* c = m.find(s.callee);
        if (c == nullptr) throw ParseError{"unknown callee '" + s.callee + "'"};
        if (c->global) throw ParseError{"a kernel cannot call a global function"};
        if (c->params.size() != s.args.size())
          throw ParseError{"wrong argument count calling '" + s.callee + "'"};
        bool use_cached = false;
        if (!unsafe && cacheable.count(c->name)) {
          std::set<std::string> arrays_seen;
          use_cached = true;
          for (size_t a = 0; a < s.args.size() && a < c->params.size(); ++a) {
            if (c->params[a].type != VT::RealArray) continue;
            const Ex& arg = *s.args[a];
            if (!arrays_seen.insert(arg.name).second) use_cached = false;  // aliasing
          }
        }
        std::string callee = "fn_" + c->name + (use_cached ? "_c" : "");
        if (fr.stat) callee = specialised(*c, s, use_cached, callee);
        o << ind(d) << callee << "(";
        for (size_t a = 0; a < s.args.size(); ++a) {
          const Ex& arg = *s.args[a];
          const VT pt = c->params[a].type;
          if (a) o << ", ";
          if (pt == VT::RealArray) {
            if (arg.k == Ex::Var) o << V(arg.name);  // whole array
            else if (arg.k == Ex::Index)             // length-1 slice (eval.cpp:485-499)
              o << "adc_slice(" << V(arg.name) << ", " << ie_any(*arg.a[0]) << ", ctx)";
            else throw ParseError{"argument of '" + s.callee + "' must be an array or slice"};
          } else if (pt == VT::Integer) {
            o << ie_any(arg);
          } else {
            o << re(arg);
          }
        }
        o << ", ctx);\n";
        break;
      }
    }
  }

  // The static-tape definition of callee c for this call's integer constants
  // (emitted once per distinct key into spec_defs); the generic name when the
  // callee needs the dynamic tape or is already being specialised (recursion).
  std::string specialised(const Fn& c, const St& call, bool cached_variant,
                          const std::string& generic) {
    std::map<std::string, long long> consts;
    std::string key = c.name + (cached_variant ? "|c" : "|g");
    for (size_t a = 0; a < call.args.size() && a < c.params.size(); ++a) {
      long long v = 0;
      if (c.params[a].type == VT::Integer && fold(*call.args[a], v)) {
        consts[c.params[a].name] = v;
        key += "|" + c.params[a].name + "=" + std::to_string(v);
      }
    }
    auto it = spec.find(key);
    if (it != spec.end()) return it->second;
    if (spec_active.count(key)) {
      all_static = false;
      return generic;
    }
    spec_active.insert(key);
    const std::string name = "fn_" + c.name + "_s" + std::to_string(spec_count++);
    std::string text;
    const bool ok = function_text(c, name, cached_variant, &consts, text);
    spec_active.erase(key);
    const std::string use = ok ? name : generic;
    if (!ok) all_static = false;
    spec[key] = use;
    if (ok) {
      spec_decls << signature(c, name) << ";\n";
      spec_defs << text;
    }
    return use;
  }

  // arrays of the kernel indexed exactly by the thread-index variable
  void prefetch_scan_expr(const Ex& e, const std::string& tv, std::set<std::string>& out) {
    if (e.k == Ex::Index && e.a[0]->k == Ex::Var && e.a[0]->name == tv) out.insert(e.name);
    for (auto& c : e.a) prefetch_scan_expr(*c, tv, out);
  }
  void prefetch_scan(const Blk& b, const std::string& tv, std::set<std::string>& out) {
    for (auto& sp : b) {
      const St& s = *sp;
      if (s.expr) prefetch_scan_expr(*s.expr, tv, out);
      if (s.indexed && s.index->k == Ex::Var && s.index->name == tv) out.insert(s.target);
      for (auto& a : s.args) prefetch_scan_expr(*a, tv, out);
      prefetch_scan(s.then_b, tv, out);
      prefetch_scan(s.else_b, tv, out);
    }
  }

  static std::string ptype(VT t) {
    return t == VT::RealArray ? "AdcArr" : t == VT::Integer ? "long long" : "double";
  }

  void prelude() {
    o << R"(// Generated by libadc_b200 (csrc/jit.cpp) from a DSL module; sm_100a, -fmad=false.
struct AdcArr { double* p; long long len; };
struct AdcErr { unsigned long long code; long long thread; long long aux; };
)";
    if (count)
      o << "struct AdcCnt { unsigned long long a, m, d, i, c, pu, po, st; };\n"
           "struct AdcCtx { AdcErr* err; long long tid; AdcCnt* cnt; };\n";
    else
      o << "struct AdcCtx { AdcErr* err; long long tid; };\n";
    o << R"(
enum { ADC_JE_DIV0 = 1, ADC_JE_LOG = 2, ADC_JE_SQRT = 3, ADC_JE_INDEX = 4, ADC_JE_TAPE_FULL = 5,
       ADC_JE_TAPE_EMPTY = 6, ADC_JE_CTL_EMPTY = 7, ADC_JE_IOVF = 8 };
__device__ __noinline__ void adc_fail(const AdcCtx& c, unsigned code, long long aux) {
  if (atomicCAS(&c.err->code, 0ull, (unsigned long long)code) == 0ull) {
    c.err->thread = c.tid;
    c.err->aux = aux;
  }
}
__device__ __forceinline__ double adc_div(double a, double b, const AdcCtx& c) {
  if (b == 0.0) adc_fail(c, ADC_JE_DIV0, 0);
  return __ddiv_rn(a, b);
}
__device__ __forceinline__ double adc_log(double a, const AdcCtx& c) {
  if (a <= 0.0) adc_fail(c, ADC_JE_LOG, 0);
  return log(a);
}
__device__ __forceinline__ double adc_sqrt(double a, const AdcCtx& c) {
  if (a < 0.0) adc_fail(c, ADC_JE_SQRT, 0);
  return __dsqrt_rn(a);
}
__device__ __forceinline__ long long adc_iadd(long long a, long long b, const AdcCtx& c) {
  const long long r = (long long)((unsigned long long)a + (unsigned long long)b);
  if (((a ^ r) & (b ^ r)) < 0) adc_fail(c, ADC_JE_IOVF, 0);
  return r;
}
__device__ __forceinline__ long long adc_isub(long long a, long long b, const AdcCtx& c) {
  const long long r = (long long)((unsigned long long)a - (unsigned long long)b);
  if (((a ^ b) & (a ^ r)) < 0) adc_fail(c, ADC_JE_IOVF, 0);
  return r;
}
__device__ __forceinline__ long long adc_imul(long long a, long long b, const AdcCtx& c) {
  const long long r = (long long)((unsigned long long)a * (unsigned long long)b);
  const long long mn = -9223372036854775807LL - 1;
  bool ovf;
  if (a == -1) ovf = b == mn;  // (r / a would itself overflow)
  else if (b == -1) ovf = a == mn;
  else ovf = a != 0 && r / a != b;
  if (ovf) adc_fail(c, ADC_JE_IOVF, 0);
  return r;
}
__device__ __forceinline__ long long adc_ineg(long long a, const AdcCtx& c) {
  if (a == (-9223372036854775807LL - 1)) adc_fail(c, ADC_JE_IOVF, 0);
  return (long long)(0ull - (unsigned long long)a);
}
__device__ __forceinline__ bool adc_ok(const AdcArr& a, long long i, const AdcCtx& c) {
  if (i < 0 || i >= a.len) { adc_fail(c, ADC_JE_INDEX, i); return false; }
  return true;
}
__device__ __forceinline__ double adc_ld(const AdcArr& a, long long i, const AdcCtx& c) {
  return adc_ok(a, i, c) ? a.p[i] : __longlong_as_double(0x7ff8000000000000LL);
}
__device__ __forceinline__ void adc_st(const AdcArr& a, long long i, double v, const AdcCtx& c) {
  if (adc_ok(a, i, c)) a.p[i] = v;
}
__device__ __forceinline__ void adc_st_add(const AdcArr& a, long long i, double v, const AdcCtx& c) {
  if (adc_ok(a, i, c)) a.p[i] = __dadd_rn(a.p[i], v);
}
__device__ __forceinline__ void adc_st_add_atomic(const AdcArr& a, long long i, double v,
                                                  const AdcCtx& c) {
  if (adc_ok(a, i, c)) atomicAdd(a.p + i, v);
}
__device__ __forceinline__ AdcArr adc_slice(const AdcArr& a, long long i, const AdcCtx& c) {
  AdcArr s{a.p, 0};
  if (adc_ok(a, i, c)) { s.p = a.p + i; s.len = 1; }
  return s;
}
)";
    o << "#define ADC_TAPE " << tape_cap << "\n";
    o << R"(__device__ __forceinline__ void adc_push(double* t, int& tp, double v, const AdcCtx& c) {
  if (tp >= ADC_TAPE) { adc_fail(c, ADC_JE_TAPE_FULL, tp); return; }
  t[tp++] = v;
}
__device__ __forceinline__ double adc_pop(double* t, int& tp, const AdcCtx& c) {
  if (tp <= 0) { adc_fail(c, ADC_JE_TAPE_EMPTY, 0); return 0.0; }
  return t[--tp];
}
__device__ __forceinline__ void adc_push_ctl(long long* t, int& cp, long long v, const AdcCtx& c) {
  if (cp >= ADC_TAPE) { adc_fail(c, ADC_JE_TAPE_FULL, cp); return; }
  t[cp++] = v;
}
__device__ __forceinline__ long long adc_pop_ctl(long long* t, int& cp, const AdcCtx& c) {
  if (cp <= 0) { adc_fail(c, ADC_JE_CTL_EMPTY, 0); return 0; }
  return t[--cp];
}
)";
  }

  // 0: not cacheable, 1: only read at [0], 2: read/written at [0] only
  static void slot_uses(const Blk& b, const std::string& n, bool& ok, bool& written) {
    std::function<void(const Ex&)> ex = [&](const Ex& e) {
      if ((e.k == Ex::Index && e.name == n) &&
          !(e.a[0]->k == Ex::Num && e.a[0]->int_lit && e.a[0]->v == 0.0))
        ok = false;
      if (e.k == Ex::Var && e.name == n) ok = false;  // whole-array use (a call argument)
      for (auto& c : e.a) ex(*c);
    };
    for (auto& sp : b) {
      const St& s = *sp;
      if (s.k == St::Assign && s.indexed && s.target == n) {
        written = true;
        if (!(s.index->k == Ex::Num && s.index->int_lit && s.index->v == 0.0)) ok = false;
      }
      if (s.expr) ex(*s.expr);
      if (s.index) ex(*s.index);
      if (s.lo) ex(*s.lo);
      if (s.hi) ex(*s.hi);
      for (auto& a : s.args) {
        if ((a->k == Ex::Var || a->k == Ex::Index) && a->name == n && s.callee != "__push")
          ok = false;  // passed on to a callee
        ex(*a);
      }
      slot_uses(s.then_b, n, ok, written);
      slot_uses(s.else_b, n, ok, written);
    }
  }

  void analyse_cacheable(const Fn& f) {
    if (f.global || !f.returns_void) return;
    std::vector<int> v(f.params.size(), 0);
    bool any = false;
    for (size_t i = 0; i < f.params.size(); ++i) {
      if (f.params[i].type != VT::RealArray) continue;
      bool ok = true, written = false;
      slot_uses(f.body, f.params[i].name, ok, written);
      if (ok) {
        v[i] = written ? 2 : 1;
        any = true;
      }
    }
    if (any) cacheable[f.name] = v;
  }

  // The register-slot form (vector kernels): every slot parameter is the
  // caller's register, by reference.
  std::string signature_ref(const Fn& f, const std::string& name,
                            const std::vector<int>& v) const {
    std::string sig = std::string("__device__ ") + (f.returns_void ? "void " : "double ") + name + "(";
    for (size_t i = 0; i < f.params.size(); ++i)
      sig += (i ? ", " : "") +
             (v[i] ? "double& c_" + V(f.params[i].name)
                   : ptype(f.params[i].type) + " " + V(f.params[i].name));
    return sig + (f.params.empty() ? "" : ", ") + "const AdcCtx& ctx)";
  }

  std::string signature(const Fn& f, const std::string& name) const {
    std::string sig = std::string("__device__ ") + (f.returns_void ? "void " : "double ") + name + "(";
    for (size_t i = 0; i < f.params.size(); ++i)
      sig += (i ? ", " : "") + ptype(f.params[i].type) + " " + V(f.params[i].name);
    return sig + (f.params.empty() ? "" : ", ") + "const AdcCtx& ctx)";
  }

  // The definition of a device function under `name`: slot-cached or not;
  // with `consts` (static tape) its integer parameters bound to constants.
  // Returns false (and no text) when the static tape is not possible.
  bool function_text(const Fn& f, const std::string& name, bool cached_variant,
                     const std::map<std::string, long long>* consts, std::string& text,
                     bool ref = false) {
    const Frame saved_fr = fr;
    const std::set<std::string>* saved_cached = cached;
    std::ostringstream body;
    std::swap(o, body);
    std::set<std::string> names;
    const std::vector<int>* v = cached_variant ? &cacheable.at(f.name) : nullptr;
    fr = Frame{};
    fr.stat = consts != nullptr;
    if (consts) fr.ienv = *consts;
    bool ok = true;
    try {
      if (v)
        for (size_t i = 0; i < f.params.size(); ++i) {
          if (!(*v)[i]) continue;
          const std::string n = V(f.params[i].name);
          names.insert(f.params[i].name);
          if (!ref)
            o << "  double c_" << n << " = adc_ok(" << n << ", 0, ctx) ? " << n << ".p[0] : 0.0;\n";
        }
      Scope sc;
      sc.push();
      for (auto& p : f.params) sc.add(p.name, p.type);
      cached = v ? &names : nullptr;
      block(f.body, f, sc, 1);
      cached = saved_cached;
      if (v && !ref)
        for (size_t i = 0; i < f.params.size(); ++i)
          if ((*v)[i] == 2) {
            const std::string n = V(f.params[i].name);
            o << "  if (" << n << ".len > 0) " << n << ".p[0] = c_" << n << ";\n";
          }
      if (!f.returns_void) o << "  return __longlong_as_double(0x7ff8000000000000LL);\n";
    } catch (Dynamic&) {
      ok = false;
    } catch (...) {
      std::swap(o, body);
      fr = saved_fr;
      cached = saved_cached;
      throw;
    }
    std::swap(o, body);
    const Frame done = fr;
    fr = saved_fr;
    cached = saved_cached;
    if (!ok) return false;
    std::ostringstream t;
    t << (ref ? signature_ref(f, name, *v) : signature(f, name)) << " {\n";
    if (done.stat) {
      for (int k = 0; k < done.maxv; ++k) t << "  double _tv" << k << " = 0.0;\n";
      for (int k = 0; k < done.maxc; ++k)
        t << (done.wide.count(k) ? "  long long _tc" : "  int _tc") << k << " = 0;\n";
    } else {
      if (f.uses_tape) t << "  double tape[ADC_TAPE]; int tp = 0;\n";
      if (f.uses_ctl) t << "  long long ctl[ADC_TAPE]; int cp = 0;\n";
    }
    t << body.str() << "}\n\n";
    text = t.str();
    return true;
  }

  // Generic (dynamic-tape) definitions of a device function: fn_<f> and,
  // when cacheable, fn_<f>_c.
  void function(const Fn& f) {
    std::string text;
    if (cacheable.count(f.name)) {
      function_text(f, "fn_" + f.name + "_c", true, nullptr, text);
      o << text;
    }
    function_text(f, "fn_" + f.name, false, nullptr, text);
    o << text;
  }

  // Vector form of a Listing-1 kernel (static-tape variants only): when the
  // kernel is exactly `integer i = blockIdx*blockDim+threadIdx; if (i < N) {
  // f(..) }` with every argument of f a slice a[i] of a kernel array (the
  // slots; pairwise distinct), a by-value a[i], a kernel scalar or a literal,
  // and f's array parameters all length-1 slots, `adc_kernel_<k>_v2` runs
  // points 2t and 2t+1 on thread t with 16-byte loads and stores, through a
  // register-slot variant of f (the same statements in the same order per
  // point, so the same bits).  The launch picks it when every array is
  // 16-byte aligned and covers N (no index error can occur), never for the
  // counting variant or forced (unsafe) launches.
  bool kernel_v2(const Fn& f, const std::map<std::string, long long>& kconst) {
    if (unsafe || count || f.body.size() != 2) return false;
    const St& d = *f.body[0];
    const St& g = *f.body[1];
    if (!is_thread_index_decl(d) || g.k != St::If || !g.else_b.empty() || g.then_b.size() != 1)
      return false;
    const std::string iv = d.target;
    const Ex& ce = *g.expr;
    if (ce.k != Ex::Cmp || ce.cmp != "<" || ce.a[0]->k != Ex::Var || ce.a[0]->name != iv ||
        ce.a[1]->k != Ex::Var || ce.a[1]->name != "N")
      return false;
    const St& call = *g.then_b[0];
    if (call.k != St::Call) return false;
    const Fn* c = m.find(call.callee);
    if (c == nullptr || c->global || c->params.size() != call.args.size() ||
        !cacheable.count(c->name))
      return false;
    const std::vector<int>& cv = cacheable.at(c->name);
    std::map<std::string, VT> kp;
    for (auto& p : f.params) kp[p.name] = p.type;
    std::set<std::string> slots, loads;
    std::map<std::string, long long> consts;
    std::string key = c->name + "|r";
    for (size_t a = 0; a < call.args.size(); ++a) {
      const Ex& e = *call.args[a];
      const VT pt = c->params[a].type;
      const bool at_i = e.k == Ex::Index && e.a[0]->k == Ex::Var && e.a[0]->name == iv &&
                        kp.count(e.name) && kp[e.name] == VT::RealArray;
      if (pt == VT::RealArray) {
        if (!at_i || !cv[a] || !slots.insert(e.name).second) return false;
      } else if (pt == VT::Real) {
        if (at_i) loads.insert(e.name);
        else if (!(e.k == Ex::Num || (e.k == Ex::Var && kp.count(e.name) && kp[e.name] != VT::RealArray)))
          return false;
      } else {
        if (e.k == Ex::Var && kconst.count(e.name)) {
          consts[c->params[a].name] = kconst.at(e.name);
          key += "|" + c->params[a].name + "=" + std::to_string(kconst.at(e.name));
        } else if (e.k == Ex::Num && e.int_lit) {
          consts[c->params[a].name] = (long long)e.v;
          key += "|" + c->params[a].name + "=" + std::to_string((long long)e.v);
        } else {
          return false;
        }
      }
    }
    for (auto& l : loads)
      if (slots.count(l)) return false;  // read by value and written through a slot
    std::string name;
    auto it = spec.find(key);
    if (it != spec.end()) {
      name = it->second;
    } else {
      name = "fn_" + c->name + "_r" + std::to_string(spec_count++);
      std::string text;
      if (!function_text(*c, name, true, &consts, text, true)) return false;
      spec[key] = name;
      spec_decls << signature_ref(*c, name, cv) << ";\n";
      spec_defs << text;
    }
    // the kernel
    o << "extern \"C\" __global__ void adc_kernel_" << f.name << "_v2(";
    for (size_t i = 0; i < f.params.size(); ++i) {
      const Prm& p = f.params[i];
      if (i) o << ", ";
      if (p.type == VT::RealArray)
        o << "double* " << V(p.name) << "_p, long long " << V(p.name) << "_n";
      else
        o << ptype(p.type) << " " << V(p.name);
    }
    o << (f.params.empty() ? "" : ", ") << "long long N, AdcErr* adc_err) {\n";
    o << "  const long long i0 = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);\n";
    o << "  if (i0 >= N) return;\n";
    auto arg_expr = [&](const Ex& e, int lane) -> std::string {
      if (e.k == Ex::Index) return "L_" + V(e.name) + (lane ? ".y" : ".x");
      if (e.k == Ex::Num) return dbl(e.v);
      return V(e.name);
    };
    auto emit_call = [&](int lane, bool pair) {
      o << "    {\n      const AdcCtx ctx{adc_err, i0 + " << lane << "};\n      " << name << "(";
      for (size_t a = 0; a < call.args.size(); ++a) {
        const Ex& e = *call.args[a];
        const VT pt = c->params[a].type;
        if (a) o << ", ";
        if (pt == VT::RealArray) o << "S_" << V(e.name) << (pair ? (lane ? ".y" : ".x") : "");
        else if (pt == VT::Integer) o << "(long long)" << consts[c->params[a].name] << "LL";
        else if (e.k == Ex::Index) o << (pair ? arg_expr(e, lane) : V(e.name) + "_p[i0]");
        else o << arg_expr(e, lane);
      }
      o << ", ctx);\n    }\n";
    };
    o << "  if (i0 + 1 < N) {\n";
    for (auto& l : loads)
      o << "    const double2 L_" << V(l) << " = __ldcs(reinterpret_cast<const double2*>(" << V(l)
        << "_p + i0));\n";
    for (auto& sl : slots)
      o << "    double2 S_" << V(sl) << " = __ldcs(reinterpret_cast<const double2*>(" << V(sl)
        << "_p + i0));\n";
    emit_call(0, true);
    emit_call(1, true);
    for (auto& sl : slots)
      o << "    __stcs(reinterpret_cast<double2*>(" << V(sl) << "_p + i0), S_" << V(sl) << ");\n";
    o << "  } else {\n";
    for (auto& sl : slots) o << "    double S_" << V(sl) << " = " << V(sl) << "_p[i0];\n";
    emit_call(0, false);
    for (auto& sl : slots) o << "    " << V(sl) << "_p[i0] = S_" << V(sl) << ";\n";
    o << "  }\n}\n\n";
    return true;
  }

  // The kernel.  kconst: integer kernel parameters bound to constants (the
  // static tape specialisation; nullptr = the generic dynamic-tape kernel).
  // Throws Dynamic if the kernel frame itself cannot use a static tape.
  void kernel(const Fn& f, const std::map<std::string, long long>* kconst) {
    Scope sc;
    sc.push();
    sc.global = true;
    for (auto& p : f.params) sc.add(p.name, p.type);
    o << "extern \"C\" __global__ void adc_kernel_" << f.name << "(";
    for (size_t i = 0; i < f.params.size(); ++i) {
      const Prm& p = f.params[i];
      if (i) o << ", ";
      if (p.type == VT::RealArray)
        o << "double* " << V(p.name) << "_p, long long " << V(p.name) << "_n";
      else
        o << ptype(p.type) << " " << V(p.name);
    }
    o << (f.params.empty() ? "" : ", ") << "long long N, AdcErr* adc_err"
      << (count ? ", unsigned long long* adc_cnt_out, unsigned* adc_stm" : "") << ") {\n";
    if (count)
      o << "  AdcCnt adc_cnt{};\n"
           "  const AdcCtx ctx{adc_err, (long long)blockIdx.x * blockDim.x + threadIdx.x, "
           "&adc_cnt};\n";
    else
      o << "  const AdcCtx ctx{adc_err, (long long)blockIdx.x * blockDim.x + threadIdx.x};\n";
    for (auto& p : f.params)
      if (p.type == VT::RealArray)
        o << "  const AdcArr " << V(p.name) << "{" << V(p.name) << "_p, " << V(p.name) << "_n};\n";
    fr = Frame{};
    fr.stat = kconst != nullptr;
    if (kconst) fr.ienv = *kconst;
    std::ostringstream body;
    std::swap(o, body);
    try {
      block(f.body, f, sc, 1);
    } catch (...) {
      std::swap(o, body);
      throw;
    }
    std::swap(o, body);
    if (fr.stat) {
      for (int k = 0; k < fr.maxv; ++k) o << "  double _tv" << k << " = 0.0;\n";
      for (int k = 0; k < fr.maxc; ++k)
        o << (fr.wide.count(k) ? "  long long _tc" : "  int _tc") << k << " = 0;\n";
    } else {
      if (f.uses_tape) o << "  double tape[ADC_TAPE]; int tp = 0;\n";
      if (f.uses_ctl) o << "  long long ctl[ADC_TAPE]; int cp = 0;\n";
    }
    o << body.str();
    if (count)  // per-block sums of the counters, one atomic per counter per block
      o << R"(  __shared__ unsigned long long adc_bs[7];
  if (threadIdx.x < 7) adc_bs[threadIdx.x] = 0ull;
  __syncthreads();
  atomicAdd(&adc_bs[0], adc_cnt.a);
  atomicAdd(&adc_bs[1], adc_cnt.m);
  atomicAdd(&adc_bs[2], adc_cnt.d);
  atomicAdd(&adc_bs[3], adc_cnt.i);
  atomicAdd(&adc_bs[4], adc_cnt.c);
  atomicAdd(&adc_bs[5], adc_cnt.pu);
  atomicAdd(&adc_bs[6], adc_cnt.po);
  __syncthreads();
  if (threadIdx.x < 7 && adc_bs[threadIdx.x] != 0ull) atomicAdd(adc_cnt_out + threadIdx.x, adc_bs[threadIdx.x]);
  if (adc_stm != nullptr) adc_stm[ctx.tid] = (unsigned)adc_cnt.st;
)";
    o << "}\n\n";
  }
};

std::string hazard_message(const std::map<std::string, std::string>& haz) {
  std::string msg = "launch refused, hazardous parameter(s):";
  for (auto& h : haz) msg += " " + h.first + " (" + h.second + ")";
  return msg + "; pass the unsafe flag to force";
}

}  // namespace

// ---- the module object ------------------------------------------------------------
struct ErrWordT {
  unsigned long long code;
  long long thread, aux;
};

struct adc_jit_module {
  std::map<int, ErrWordT*> derr;  // per device, reset before every launch
  ErrWordT* herr = nullptr;       // pinned
  std::string kernel;
  std::string source;  // the module text (the counting variant is built from it on demand)
  bool unsafe = false;
  int tape_capacity = 256;
  // counting variant (adc_cuda_jit_launch_counted): built on first use
  std::string cuda_counted;
  std::vector<char> cubin_counted;
  std::map<int, cudaLibrary_t> libs_counted;
  std::map<int, cudaKernel_t> fns_counted;
  unsigned long long* dcnt = nullptr;  // [7] device counters (the device of the last counted launch)
  int dcnt_dev = -1;
  std::vector<int32_t> kinds;  // 0 real[], 1 real, 2 integer
  std::vector<std::string> names;
  std::string cuda;
  std::vector<char> cubin;
  std::map<int, cudaLibrary_t> libs;  // per device
  std::map<int, cudaKernel_t> fns;
  // static-tape variants (jit.cpp, "Static tape"): one for every launch when
  // the kernel needs no integer constants (key "*"), else one per tuple of
  // integer kernel arguments (built on first use, at most kMaxStaticVariants)
  struct Variant {
    bool ok = false;  // false: this key runs the dynamic-tape kernel
    bool has_v2 = false;  // the vector Listing-1 kernel adc_kernel_<k>_v2 is in the image
    std::string cuda;
    std::vector<char> cubin;
    std::map<int, cudaLibrary_t> libs;
    std::map<int, cudaKernel_t> fns;
    std::map<int, cudaKernel_t> fns_v2;
  };
  std::map<std::string, Variant> statics;
  bool static_any = false;  // statics["*"] serves every launch
  std::mutex mu;
};

namespace {
int parse_module(const std::string& src, Module& m) {
  try {
    Parser p;
    p.t = lex(src);
    while (p.peek().k != Tok::End) m.fns.push_back(p.function());
    for (auto& f : m.fns) {
      Scope sc;
      sc.global = f.global;
      sc.push();
      for (auto& prm : f.params) sc.add(prm.name, prm.type);
      type_block(f.body, sc, f);
    }
  } catch (const ParseError& e) {
    return fail(ADC_E_SEMANTIC, "jit: " + e.msg);
  }
  return ADC_OK;
}
}  // namespace

namespace {
// Emission (plain or counting variant) and NVRTC compilation of kernel k of m.
// kconst != nullptr: the static-tape variant with the kernel's integer
// parameters bound as given (possibly none); returns kStaticImpossible when it
// cannot be built (the caller keeps the dynamic-tape kernel).
constexpr int kStaticImpossible = -1000;

int emit_and_compile(const Module& m, const Fn* k, const std::string& kernel, bool unsafe,
                     int tape_capacity, bool count, std::string& cuda, std::vector<char>& cubin,
                     const std::map<std::string, long long>* kconst = nullptr,
                     bool* fully_static = nullptr, bool* has_v2 = nullptr) {
  Emitter em{m, unsafe, tape_capacity};
  em.count = count;
  try {
    em.prelude();
    for (auto& f : m.fns)
      if (!f.global && f.name != "") em.o << "__device__ " << (f.returns_void ? "void" : "double") << " fn_"
                          << f.name << "(" << [&] {
                               std::string s;
                               for (size_t i = 0; i < f.params.size(); ++i)
                                 s += (i ? ", " : "") + Emitter::ptype(f.params[i].type) + " " +
                                      Emitter::V(f.params[i].name);
                               return s + (f.params.empty() ? "" : ", ") + "const AdcCtx& ctx);\n";
                             }();
    em.o << "\n";
    // only what the kernel reaches through call statements
    std::set<std::string> reach{kernel};
    std::vector<const Fn*> work{k};
    std::function<void(const Blk&)> scan = [&](const Blk& b) {
      for (auto& sp : b) {
        if (sp->k == St::Call && !reach.count(sp->callee)) {
          if (const Fn* c = m.find(sp->callee)) {
            reach.insert(c->name);
            work.push_back(c);
          }
        }
        scan(sp->then_b);
        scan(sp->else_b);
      }
    };
    for (size_t w = 0; w < work.size(); ++w) scan(work[w]->body);
    for (auto& f : m.fns)
      if (reach.count(f.name)) em.analyse_cacheable(f);
    // callees first, so a cached variant is declared before its call sites
    for (auto& f : m.fns)
      if (reach.count(f.name) && !f.global) em.function(f);
    // the kernel (its static-tape specialisations of the callees before it)
    std::ostringstream ko;
    std::swap(em.o, ko);
    try {
      em.kernel(*k, kconst);
      if (kconst != nullptr && has_v2 != nullptr) *has_v2 = em.kernel_v2(*k, *kconst);
    } catch (Dynamic&) {
      return kStaticImpossible;
    } catch (...) {
      std::swap(em.o, ko);
      throw;
    }
    std::swap(em.o, ko);
    em.o << em.spec_decls.str() << "\n" << em.spec_defs.str() << ko.str();
    if (fully_static) *fully_static = em.all_static;
  } catch (const ParseError& e) {
    return fail(ADC_E_SEMANTIC, "jit: " + e.msg);
  }
  const Nvrtc* N = nvrtc();
  if (N == nullptr) return fail(ADC_E_CUDA, "jit: libnvrtc.so.12 could not be loaded");
  cuda = em.o.str();
  nvrtcProgram prog = nullptr;
  nvrtcResult r = N->create(&prog, cuda.c_str(), "adc_jit.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail(ADC_E_CUDA, std::string("nvrtcCreateProgram: ") + N->error_string(r));
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17",
                        "-default-device", "--extra-device-vectorization"};
  r = N->compile(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    N->log_size(prog, &n);
    std::string log(n, '\0');
    if (n) N->log(prog, &log[0]);
    N->destroy(&prog);
    return fail(ADC_E_CUDA, "jit: NVRTC failed: " + log);
  }
  size_t n = 0;
  N->cubin_size(prog, &n);
  cubin.resize(n);
  N->cubin(prog, cubin.data());
  N->destroy(&prog);
  return ADC_OK;
}
}  // namespace

extern "C" int adc_jit_compile(const char* source, const char* kernel, int32_t unsafe,
                               int32_t tape_capacity, adc_jit_module** out) {
  clear_error();
  if (source == nullptr || kernel == nullptr || out == nullptr)
    return fail(ADC_E_ARG, "null argument");
  *out = nullptr;
  if (tape_capacity <= 0) tape_capacity = 256;
  Module m;
  if (int rc = parse_module(source, m)) return rc;
  const Fn* k = m.find(kernel);
  if (k == nullptr) return fail(ADC_E_LAUNCH, std::string("unknown kernel '") + kernel + "'");
  if (!k->global) return fail(ADC_E_LAUNCH, std::string("'") + kernel + "' is not a global kernel");
  // race_check (launch.cpp:261-267): same refusal message
  std::set<std::string> arrays;
  for (auto& p : k->params)
    if (p.type == VT::RealArray) arrays.insert(p.name);
  std::map<std::string, std::string> haz;
  std::string tvar;
  kernel_hazards(m, k->body, "", arrays, haz, tvar);
  if (!haz.empty() && !unsafe) return fail(ADC_E_LAUNCH, hazard_message(haz));
  auto* J = new (std::nothrow) adc_jit_module();
  if (J == nullptr) return fail(ADC_E_ARG, "out of host memory");
  J->kernel = kernel;
  J->source = source;
  J->unsafe = unsafe != 0;
  J->tape_capacity = tape_capacity;
  for (auto& p : k->params) {
    J->kinds.push_back(p.type == VT::RealArray ? 0 : p.type == VT::Real ? 1 : 2);
    J->names.push_back(p.name);
  }
  if (int rc = emit_and_compile(m, k, kernel, unsafe != 0, tape_capacity, false, J->cuda,
                                J->cubin)) {
    delete J;
    return rc;
  }
  // the static-tape kernel that needs no integer constants, when there is one
  {
    const std::map<std::string, long long> none;
    adc_jit_module::Variant v;
    bool full = false;
    const int rc = emit_and_compile(m, k, kernel, unsafe != 0, tape_capacity, false, v.cuda,
                                    v.cubin, &none, &full, &v.has_v2);
    bool has_ints = false;
    for (auto& p : k->params) has_ints = has_ints || p.type == VT::Integer;
    if (rc == ADC_OK && (full || !has_ints)) {
      v.ok = true;
      J->statics["*"] = std::move(v);
      J->static_any = true;
    } else if (rc != ADC_OK && rc != kStaticImpossible) {
      delete J;
      return rc;
    }
  }
  *out = J;
  return ADC_OK;
}

extern "C" int adc_jit_destroy(adc_jit_module* J) {
  if (J == nullptr) return ADC_OK;
  for (auto& l : J->libs) cudaLibraryUnload(l.second);
  for (auto& l : J->libs_counted) cudaLibraryUnload(l.second);
  for (auto& v : J->statics)
    for (auto& l : v.second.libs) cudaLibraryUnload(l.second);
  if (J->dcnt) cudaFree(J->dcnt);
  for (auto& e : J->derr) cudaFree(e.second);
  if (J->herr) cudaFreeHost(J->herr);
  delete J;
  return ADC_OK;
}

extern "C" int adc_jit_kernel_params(const adc_jit_module* J, int32_t* nparams, int32_t* kinds,
                                     int32_t cap) {
  clear_error();
  if (J == nullptr || nparams == nullptr) return fail(ADC_E_ARG, "null argument");
  *nparams = (int32_t)J->kinds.size();
  for (int32_t i = 0; kinds != nullptr && i < cap && i < *nparams; ++i) kinds[i] = J->kinds[i];
  return ADC_OK;
}

extern "C" const char* adc_jit_kernel_param_name(const adc_jit_module* J, int32_t i) {
  return J && i >= 0 && i < (int32_t)J->names.size() ? J->names[i].c_str() : nullptr;
}

extern "C" const char* adc_jit_cuda_source(const adc_jit_module* J) {
  return J ? J->cuda.c_str() : nullptr;
}

namespace {
constexpr size_t kMaxStaticVariants = 32;

// The static-tape variant a launch with these arguments uses (built on first
// use); nullptr = the dynamic-tape kernel.  Caller holds J->mu.
adc_jit_module::Variant* static_variant(adc_jit_module* J, const adc_jit_arg* args, int& rc) {
  rc = ADC_OK;
  if (J->static_any) return &J->statics["*"];
  std::map<std::string, long long> consts;
  std::string key;
  for (size_t i = 0; i < J->kinds.size(); ++i)
    if (J->kinds[i] == 2) {
      consts[J->names[i]] = args[i].int_value;
      key += std::to_string(args[i].int_value) + ",";
    }
  if (consts.empty()) return nullptr;  // no constants to specialise on
  auto it = J->statics.find(key);
  if (it != J->statics.end()) return it->second.ok ? &it->second : nullptr;
  if (J->statics.size() >= kMaxStaticVariants) return nullptr;
  Module m;
  if ((rc = parse_module(J->source, m))) return nullptr;
  adc_jit_module::Variant v;
  bool full = false;
  rc = emit_and_compile(m, m.find(J->kernel), J->kernel, J->unsafe, J->tape_capacity, false,
                        v.cuda, v.cubin, &consts, &full, &v.has_v2);
  if (rc == kStaticImpossible) rc = ADC_OK;
  else if (rc != ADC_OK) return nullptr;
  else v.ok = full;  // a partly static variant buys nothing over the dynamic kernel
  auto& slot = J->statics[key] = std::move(v);
  return slot.ok ? &slot : nullptr;
}
}  // namespace

extern "C" int adc_jit_static_variant(adc_jit_module* J, const int64_t* int_args, int32_t nint,
                                      const char** cuda_source) {
  clear_error();
  if (J == nullptr || cuda_source == nullptr) return fail(ADC_E_ARG, "null argument");
  std::vector<adc_jit_arg> args(J->kinds.size());
  int32_t k = 0;
  for (size_t i = 0; i < J->kinds.size(); ++i)
    if (J->kinds[i] == 2) {
      if (k >= nint || int_args == nullptr) return fail(ADC_E_ARG, "missing integer argument");
      args[i].int_value = int_args[k++];
    }
  std::lock_guard<std::mutex> lock(J->mu);
  int rc = ADC_OK;
  adc_jit_module::Variant* v = static_variant(J, args.data(), rc);
  if (rc != ADC_OK) return rc;
  *cuda_source = v ? v->cuda.c_str() : nullptr;
  return ADC_OK;
}

extern "C" size_t adc_jit_cubin_size(const adc_jit_module* J) { return J ? J->cubin.size() : 0; }

namespace {
const char* jit_error_text(unsigned long long code) {
  switch (code) {
    case 1: return "division by zero";
    case 2: return "log of non-positive value";
    case 3: return "sqrt of negative value";
    case 4: return "index out of range";
    case 5: return "tape capacity exceeded (raise tape_capacity)";
    case 6: return "__pop on empty tape";
    case 7: return "__pop_ctl on empty control tape";
    case 8: return "integer overflow";
    default: return "device error";
  }
}

}  // namespace

namespace {
// counted: the counting variant (built on first use); counts[7] (host) gets
// the OpCounters summed over all threads, stm (device, grid*block) every
// thread's kernel-frame statement count when non-null.
int jit_launch(adc_jit_module* J, int64_t grid, int64_t block, int64_t n, const adc_jit_arg* args,
               int32_t nargs, void* stream, bool counted, uint64_t* counts, uint32_t* stm) {
  if (J == nullptr || (nargs > 0 && args == nullptr)) return fail(ADC_E_ARG, "null argument");
  if (grid <= 0 || block <= 0 || n <= 0)
    return fail(ADC_E_LAUNCH, "launch configuration must be positive (grid " +
                                  std::to_string(grid) + ", block " + std::to_string(block) +
                                  ", n " + std::to_string(n) + ")");
  if (grid > INT64_MAX / block || grid * block < n)
    return fail(ADC_E_LAUNCH, "grid " + std::to_string(grid) + " x block " + std::to_string(block) +
                                  " does not cover problem size " + std::to_string(n));
  if (block > 1024 || grid > 0x7fffffff)
    return fail(ADC_E_LAUNCH, "block must be <= 1024 and grid < 2^31 on the device");
  if (nargs != (int32_t)J->kinds.size())
    return fail(ADC_E_LAUNCH, "kernel '" + J->kernel + "' takes " +
                                  std::to_string(J->kinds.size()) + " parameters");
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  int dev = 0;
  ADCB_CUDA(cudaGetDevice(&dev));
  cudaKernel_t fn = nullptr;
  ErrWordT* derr = nullptr;
  std::unique_lock<std::mutex> lock(J->mu);  // one launch of a module at a time (shared error word)
  {
    if (J->herr == nullptr) ADCB_CUDA(cudaMallocHost(&J->herr, sizeof(ErrWordT)));
    if (J->derr.count(dev) == 0) {
      ErrWordT* d = nullptr;
      ADCB_CUDA(cudaMalloc(&d, sizeof(ErrWordT)));
      J->derr[dev] = d;
    }
    derr = J->derr[dev];
    if (counted && J->cubin_counted.empty()) {
      Module m;
      if (int rc = parse_module(J->source, m)) return rc;
      if (int rc = emit_and_compile(m, m.find(J->kernel), J->kernel, J->unsafe, J->tape_capacity,
                                    true, J->cuda_counted, J->cubin_counted))
        return rc;
    }
    if (counted && (J->dcnt == nullptr || J->dcnt_dev != dev)) {
      if (J->dcnt) cudaFree(J->dcnt);
      J->dcnt = nullptr;
      ADCB_CUDA(cudaMalloc(&J->dcnt, 7 * sizeof(unsigned long long)));
      J->dcnt_dev = dev;
    }
    adc_jit_module::Variant* sv = nullptr;
    if (!counted) {
      int rc = ADC_OK;
      sv = static_variant(J, args, rc);
      if (rc != ADC_OK) return rc;
    }
    auto& fns = sv ? sv->fns : counted ? J->fns_counted : J->fns;
    auto& libs = sv ? sv->libs : counted ? J->libs_counted : J->libs;
    const std::vector<char>& cubin = sv ? sv->cubin : counted ? J->cubin_counted : J->cubin;
    auto it = fns.find(dev);
    if (it == fns.end()) {
      cudaLibrary_t lib = nullptr;
      ADCB_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
      const std::string name = "adc_kernel_" + J->kernel;
      cudaError_t e = cudaLibraryGetKernel(&fn, lib, name.c_str());
      if (e == cudaSuccess && sv && sv->has_v2) {
        cudaKernel_t f2 = nullptr;
        e = cudaLibraryGetKernel(&f2, lib, (name + "_v2").c_str());
        sv->fns_v2[dev] = f2;
      }
      if (e != cudaSuccess) {
        cudaLibraryUnload(lib);
        return cuda_fail(e, "cudaLibraryGetKernel");
      }
      libs[dev] = lib;
      fns[dev] = fn;
    } else {
      fn = it->second;
    }
    // the vector form: every array 16-byte aligned and covering N
    if (sv && sv->has_v2) {
      bool ok = true;
      for (int32_t i = 0; i < nargs && ok; ++i)
        if (J->kinds[i] == 0)
          ok = (reinterpret_cast<uintptr_t>(args[i].ptr) & 15) == 0 && args[i].len >= n;
      if (ok) {
        fn = sv->fns_v2[dev];
        block = 256;
        grid = ((n + 1) / 2 + block - 1) / block;
      }
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ADCB_CUDA(cudaMemsetAsync(derr, 0, sizeof(ErrWordT), s));
  // kernel arguments: real[] -> (double*, long long len), real -> double, integer -> long long
  std::vector<double*> ptrs(nargs);
  std::vector<long long> lens(nargs), ints(nargs);
  std::vector<double> reals(nargs);
  std::vector<void*> kp;
  for (int32_t i = 0; i < nargs; ++i) {
    switch (J->kinds[i]) {
      case 0:
        if (args[i].ptr == nullptr && args[i].len > 0)
          return fail(ADC_E_LAUNCH, "missing buffer for parameter " + std::to_string(i));
        ptrs[i] = args[i].ptr;
        lens[i] = args[i].len;
        kp.push_back(&ptrs[i]);
        kp.push_back(&lens[i]);
        break;
      case 1:
        reals[i] = args[i].real_value;
        kp.push_back(&reals[i]);
        break;
      default:
        ints[i] = args[i].int_value;
        kp.push_back(&ints[i]);
        break;
    }
  }
  long long nn = n;
  kp.push_back(&nn);
  kp.push_back(&derr);
  unsigned long long* dcnt = J->dcnt;
  uint32_t* dstm = stm;
  if (counted) {
    ADCB_CUDA(cudaMemsetAsync(dcnt, 0, 7 * sizeof(unsigned long long), s));
    kp.push_back(&dcnt);
    kp.push_back(&dstm);
  }
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3((unsigned)grid),
                                   dim3((unsigned)block), kp.data(), 0, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel (jit)");
  ADCB_CUDA(cudaMemcpyAsync(J->herr, derr, sizeof(ErrWordT), cudaMemcpyDeviceToHost, s));
  if (counted) {
    unsigned long long h[7];
    ADCB_CUDA(cudaMemcpyAsync(h, dcnt, sizeof h, cudaMemcpyDeviceToHost, s));
    ADCB_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 7; ++i) counts[i] = h[i];
  }
  ADCB_CUDA(cudaStreamSynchronize(s));
  const ErrWordT herr = *J->herr;
  if (herr.code != 0) {
    std::string msg = jit_error_text(herr.code);
    if (herr.code == 4) msg = "index " + std::to_string(herr.aux) + " out of range";
    return fail(ADC_E_EVAL, msg + " (thread " + std::to_string(herr.thread) + ")");
  }
  return ADC_OK;
}
}  // namespace

extern "C" int adc_cuda_jit_launch(adc_jit_module* J, int64_t grid, int64_t block, int64_t n,
                                   const adc_jit_arg* args, int32_t nargs, void* stream) {
  clear_error();
  return jit_launch(J, grid, block, n, args, nargs, stream, false, nullptr, nullptr);
}

extern "C" int adc_cuda_jit_launch_counted(adc_jit_module* J, int64_t grid, int64_t block,
                                           int64_t n, const adc_jit_arg* args, int32_t nargs,
                                           void* stream, uint64_t* counts,
                                           uint32_t* thread_statements) {
  clear_error();
  if (counts == nullptr) return fail(ADC_E_ARG, "null argument");
  return jit_launch(J, grid, block, n, args, nargs, stream, true, counts, thread_statements);
}

namespace {
// A larger tape: the module is re-emitted and recompiled with `cap` entries
// per frame tape (both variants; the loaded images are dropped).
int jit_grow_tape(adc_jit_module* J, int cap) {
  std::lock_guard<std::mutex> lock(J->mu);
  if (J->tape_capacity >= cap) return ADC_OK;
  Module m;
  if (int rc = parse_module(J->source, m)) return rc;
  std::string cuda;
  std::vector<char> cubin;
  if (int rc = emit_and_compile(m, m.find(J->kernel), J->kernel, J->unsafe, cap, false, cuda, cubin))
    return rc;
  for (auto& l : J->libs) cudaLibraryUnload(l.second);
  for (auto& l : J->libs_counted) cudaLibraryUnload(l.second);
  J->libs.clear();
  J->fns.clear();
  J->libs_counted.clear();
  J->fns_counted.clear();
  J->cuda = std::move(cuda);
  J->cubin = std::move(cubin);
  J->cuda_counted.clear();
  J->cubin_counted.clear();
  J->tape_capacity = cap;
  return ADC_OK;
}

// Host buffers stay untouched until the copy-back, so a launch that ran out
// of tape (the reference's tapes are unbounded vectors) is redone from the
// caller's data with a larger tape, up to kMaxTape entries per frame tape.
constexpr int kMaxTape = 4096;

int jit_launch_host(adc_jit_module* J, int64_t grid, int64_t block, int64_t n,
                    const adc_jit_arg* args, int32_t nargs, bool counted, uint64_t* counts,
                    uint32_t* thread_statements) {
  if (J == nullptr || (nargs > 0 && args == nullptr)) return fail(ADC_E_ARG, "null argument");
  if (nargs != (int32_t)J->kinds.size())
    return fail(ADC_E_LAUNCH, "kernel '" + J->kernel + "' takes " +
                                  std::to_string(J->kinds.size()) + " parameters");
  if (!device_present()) return fail(ADC_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  std::vector<adc_jit_arg> dargs(args, args + nargs);
  std::vector<double*> owned;
  auto release = [&] {
    for (double* p : owned) cudaFree(p);
  };
  for (int32_t i = 0; i < nargs; ++i) {
    if (J->kinds[i] != 0 || args[i].len <= 0) continue;
    double* d = nullptr;
    const size_t bytes = (size_t)args[i].len * sizeof(double);
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(d, args[i].ptr, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "jit host staging");
    }
    owned.push_back(d);
    dargs[i].ptr = d;
  }
  uint32_t* dstm = nullptr;
  const size_t total = grid > 0 && block > 0 ? (size_t)grid * (size_t)block : 0;
  if (counted && thread_statements != nullptr && total > 0) {
    cudaError_t e = cudaMalloc(&dstm, total * sizeof(uint32_t));
    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "jit statement counts");
    }
  }
  int rc = jit_launch(J, grid, block, n, dargs.data(), nargs, nullptr, counted, counts, dstm);
  while (rc == ADC_E_EVAL && J->herr != nullptr && J->herr->code == 5 &&
         J->tape_capacity < kMaxTape) {  // tape capacity exceeded
    if (int g = jit_grow_tape(J, std::min(kMaxTape, J->tape_capacity * 4))) {
      rc = g;
      break;
    }
    for (int32_t i = 0; i < nargs; ++i)  // the caller's data again
      if (J->kinds[i] == 0 && args[i].len > 0)
        cudaMemcpy(dargs[i].ptr, args[i].ptr, (size_t)args[i].len * sizeof(double),
                   cudaMemcpyHostToDevice);
    clear_error();
    rc = jit_launch(J, grid, block, n, dargs.data(), nargs, nullptr, counted, counts, dstm);
  }
  if (dstm != nullptr) {
    if (rc == ADC_OK)
      cudaMemcpy(thread_statements, dstm, total * sizeof(uint32_t), cudaMemcpyDeviceToHost);
    cudaFree(dstm);
  }
  // buffers are written in place even when a thread reported an error, as in
  // the reference (a throwing launch leaves the other threads' writes)
  for (int32_t i = 0, k = 0; i < nargs; ++i) {
    if (J->kinds[i] != 0 || args[i].len <= 0) continue;
    cudaMemcpy(args[i].ptr, dargs[i].ptr, (size_t)args[i].len * sizeof(double),
               cudaMemcpyDeviceToHost);
    ++k;
  }
  release();
  return rc;
}
}  // namespace

extern "C" int adc_cuda_jit_launch_host(adc_jit_module* J, int64_t grid, int64_t block, int64_t n,
                                        const adc_jit_arg* args, int32_t nargs) {
  clear_error();
  return jit_launch_host(J, grid, block, n, args, nargs, false, nullptr, nullptr);
}

extern "C" int adc_cuda_jit_launch_counted_host(adc_jit_module* J, int64_t grid, int64_t block,
                                                int64_t n, const adc_jit_arg* args, int32_t nargs,
                                                uint64_t* counts, uint32_t* thread_statements) {
  clear_error();
  if (counts == nullptr) return fail(ADC_E_ARG, "null argument");
  return jit_launch_host(J, grid, block, n, args, nargs, true, counts, thread_statements);
}
