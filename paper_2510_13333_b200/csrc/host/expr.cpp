#include "expr.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <unordered_map>

#include "sparse.hpp"  // Error

namespace nclb {

namespace {
XRef mknode(int op, XRef a, XRef b, double v, int slot) {
  auto n = std::make_shared<XNode>();
  n->op = op;
  n->a = std::move(a);
  n->b = std::move(b);
  n->value = v;
  n->slot = slot;
  return n;
}
bool is_c(const XRef& n, double v) { return n && n->op == NCL_OP_CONST && n->value == v; }
}  // namespace

X X::constant(double v) { return X(mknode(NCL_OP_CONST, nullptr, nullptr, v, -1)); }
X X::var(int slot) {
  if (slot < 0) throw Error{NCL_E_INVALID, "Expr::var: negative slot"};
  return X(mknode(NCL_OP_VAR, nullptr, nullptr, 0.0, slot));
}
X X::param(int slot) {
  if (slot < 0) throw Error{NCL_E_INVALID, "Expr::param: negative slot"};
  return X(mknode(NCL_OP_PARAM, nullptr, nullptr, 0.0, slot));
}
bool X::is_constant(double v) const { return is_c(n_, v); }

// Folding rules of Expr::make (expr.cpp:38-84).
X X::make(int op, const X& a, const X& b, double v) {
  const bool ca = a.n_ && a.n_->op == NCL_OP_CONST;
  const bool cb = b.n_ && b.n_->op == NCL_OP_CONST;
  switch (op) {
    case NCL_OP_ADD:
      if (ca && cb) return constant(a.n_->value + b.n_->value);
      if (a.is_zero()) return b;
      if (b.is_zero()) return a;
      break;
    case NCL_OP_SUB:
      if (ca && cb) return constant(a.n_->value - b.n_->value);
      if (b.is_zero()) return a;
      if (a.is_zero()) return X(mknode(NCL_OP_NEG, b.n_, nullptr, 0.0, -1));
      break;
    case NCL_OP_MUL:
      if (ca && cb) return constant(a.n_->value * b.n_->value);
      if (a.is_zero() || b.is_zero()) return constant(0.0);
      if (a.is_constant(1.0)) return b;
      if (b.is_constant(1.0)) return a;
      if (a.is_constant(-1.0)) return -b;
      if (b.is_constant(-1.0)) return -a;
      break;
    case NCL_OP_DIV:
      if (a.is_zero()) return constant(0.0);
      if (b.is_constant(1.0)) return a;
      if (ca && cb && b.n_->value != 0.0) return constant(a.n_->value / b.n_->value);
      break;
    case NCL_OP_POW:
      if (v == 0.0) return constant(1.0);
      if (v == 1.0) return a;
      if (ca) return constant(std::pow(a.n_->value, v));
      break;
    case NCL_OP_NEG:
      if (ca) return constant(-a.n_->value);
      if (a.n_ && a.n_->op == NCL_OP_NEG) return X(a.n_->a);
      break;
    case NCL_OP_SIN:
      if (ca) return constant(std::sin(a.n_->value));
      break;
    case NCL_OP_COS:
      if (ca) return constant(std::cos(a.n_->value));
      break;
    default:
      break;
  }
  return X(mknode(op, a.n_, b.n_, v, -1));
}

X operator+(const X& a, const X& b) { return X::make(NCL_OP_ADD, a, b); }
X operator-(const X& a, const X& b) { return X::make(NCL_OP_SUB, a, b); }
X operator*(const X& a, const X& b) { return X::make(NCL_OP_MUL, a, b); }
X operator/(const X& a, const X& b) { return X::make(NCL_OP_DIV, a, b); }
X operator-(const X& a) { return X::make(NCL_OP_NEG, a, X()); }
X xpow(const X& a, double e) { return X::make(NCL_OP_POW, a, X(), e); }
X xsin(const X& a) { return X::make(NCL_OP_SIN, a, X()); }
X xcos(const X& a) { return X::make(NCL_OP_COS, a, X()); }

// Differentiation rules of Expr::diff (expr.cpp:95-127).
X X::diff(int s) const {
  if (!n_) throw Error{NCL_E_LOGIC, "Expr::diff: empty expression"};
  const XNode& n = *n_;
  const X a = n.a ? X(n.a) : X();
  const X b = n.b ? X(n.b) : X();
  switch (n.op) {
    case NCL_OP_CONST:
    case NCL_OP_PARAM:
      return constant(0.0);
    case NCL_OP_VAR:
      return constant(n.slot == s ? 1.0 : 0.0);
    case NCL_OP_ADD:
      return a.diff(s) + b.diff(s);
    case NCL_OP_SUB:
      return a.diff(s) - b.diff(s);
    case NCL_OP_MUL:
      return a.diff(s) * b + a * b.diff(s);
    case NCL_OP_DIV: {
      const X da = a.diff(s), db = b.diff(s);
      return da / b - (a * db) / (b * b);
    }
    case NCL_OP_POW:
      return constant(n.value) * xpow(a, n.value - 1.0) * a.diff(s);
    case NCL_OP_NEG:
      return -a.diff(s);
    case NCL_OP_SIN:
      return xcos(a) * a.diff(s);
    case NCL_OP_COS:
      return -xsin(a) * a.diff(s);
  }
  throw Error{NCL_E_LOGIC, "Expr::diff: unknown op"};
}

X build_from_program(int nn, const ncl_expr_node* nodes) {
  if (nn <= 0) throw Error{NCL_E_INVALID, "expression program is empty"};
  std::vector<X> e(nn);
  for (int k = 0; k < nn; ++k) {
    const ncl_expr_node& q = nodes[k];
    auto arg = [&](int i) -> const X& {
      if (i < 0 || i >= k) throw Error{NCL_E_INVALID, "expression program: operand out of order"};
      return e[i];
    };
    switch (q.op) {
      case NCL_OP_CONST: e[k] = X::constant(q.value); break;
      case NCL_OP_VAR: e[k] = X::var(q.slot); break;
      case NCL_OP_PARAM: e[k] = X::param(q.slot); break;
      case NCL_OP_ADD: e[k] = arg(q.a) + arg(q.b); break;
      case NCL_OP_SUB: e[k] = arg(q.a) - arg(q.b); break;
      case NCL_OP_MUL: e[k] = arg(q.a) * arg(q.b); break;
      case NCL_OP_DIV: e[k] = arg(q.a) / arg(q.b); break;
      case NCL_OP_POW: e[k] = xpow(arg(q.a), q.value); break;
      case NCL_OP_NEG: e[k] = -arg(q.a); break;
      case NCL_OP_SIN: e[k] = xsin(arg(q.a)); break;
      case NCL_OP_COS: e[k] = xcos(arg(q.a)); break;
      default: throw Error{NCL_E_INVALID, "expression program: bad op"};
    }
  }
  return e[nn - 1];
}

namespace {
struct Key {
  int op, slot, a, b;
  uint64_t vbits;
  bool operator==(const Key& o) const {
    return op == o.op && slot == o.slot && a == o.a && b == o.b && vbits == o.vbits;
  }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = k.vbits * 0x9e3779b97f4a7c15ull;
    h ^= (static_cast<uint64_t>(k.op) << 48) ^ (static_cast<uint64_t>(k.slot + 1) << 32) ^
         (static_cast<uint64_t>(k.a + 1) << 16) ^ static_cast<uint64_t>(k.b + 1) * 0x85ebca6bull;
    return static_cast<size_t>(h ^ (h >> 29));
  }
};
}  // namespace

Program compile(const std::vector<X>& roots) {
  Program P;
  std::unordered_map<const XNode*, int> reg_of;
  std::unordered_map<Key, int, KeyHash> cse;
  struct Frame {
    const XNode* n;
    bool expanded;
  };
  for (const X& r : roots) {
    if (!r.node()) throw Error{NCL_E_LOGIC, "compile: empty expression"};
    std::vector<Frame> st{{r.node().get(), false}};
    while (!st.empty()) {
      Frame fr = st.back();
      st.pop_back();
      if (reg_of.count(fr.n)) continue;
      if (!fr.expanded) {
        st.push_back({fr.n, true});
        if (fr.n->a) st.push_back({fr.n->a.get(), false});
        if (fr.n->b) st.push_back({fr.n->b.get(), false});
        continue;
      }
      Key k{fr.n->op, fr.n->slot, fr.n->a ? reg_of.at(fr.n->a.get()) : -1,
            fr.n->b ? reg_of.at(fr.n->b.get()) : -1, 0};
      std::memcpy(&k.vbits, &fr.n->value, sizeof(double));
      if (fr.n->op != NCL_OP_CONST && fr.n->op != NCL_OP_POW) k.vbits = 0;
      auto it = cse.find(k);
      if (it != cse.end()) {
        reg_of[fr.n] = it->second;
        continue;
      }
      CInstr ins{};
      ins.op = fr.n->op;
      ins.a = k.a;
      ins.b = k.b;
      ins.slot = fr.n->slot;
      ins.value = fr.n->value;
      const int reg = static_cast<int>(P.code.size());
      if (reg >= 32000) throw Error{NCL_E_INVALID, "template program too long"};
      P.code.push_back(ins);
      cse.emplace(k, reg);
      reg_of[fr.n] = reg;
    }
    P.out.push_back(reg_of.at(r.node().get()));
  }
  return P;
}

std::vector<Instr> encode(const Program& p) {
  std::vector<Instr> out(p.code.size());
  for (size_t i = 0; i < p.code.size(); ++i) {
    const CInstr& c = p.code[i];
    Instr& d = out[i];
    d.op = static_cast<int8_t>(c.op);
    d.pad = 0;
    d.dst = static_cast<int16_t>(c.dst);
    const bool leaf = c.op == NCL_OP_VAR || c.op == NCL_OP_PARAM;
    d.a = static_cast<int16_t>(leaf ? c.slot : c.a);
    d.b = static_cast<int16_t>(c.b);
    d.value = c.value;
  }
  return out;
}

Template::Template(X fx, int ns, std::string nm) : name(std::move(nm)), nslots(ns), f(std::move(fx)) {
  std::vector<X> first(ns);
  for (int i = 0; i < ns; ++i) {
    first[i] = f.diff(i);
    if (!first[i].is_zero()) {
      grad_slot.push_back(i);
      grad.push_back(first[i]);
    }
  }
  for (int i = 0; i < ns; ++i) {
    if (first[i].is_zero()) continue;
    for (int j = 0; j <= i; ++j) {
      X second = first[i].diff(j);
      if (!second.is_zero()) {
        hess_slot.emplace_back(i, j);
        hess.push_back(second);
      }
    }
  }
}

}  // namespace nclb
