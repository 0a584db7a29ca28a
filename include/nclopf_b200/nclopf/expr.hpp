// Drop-in façade for /root/reference/proj/include/nclopf/expr.hpp over the
// B200 library's C-ABI (include/nclopf_b200.h). Same namespace, names and
// value semantics, so a reference caller compiles unchanged with
// -I include/nclopf_b200 and links libnclopf_b200.so instead of the reference.
//
// An Expr here RECORDS the DAG a caller builds (ExprNode is the reference's
// node struct); the library replays it through its copy of the reference's
// smart constructors (expr.cpp:38-93), so folding, derivatives and therefore
// every Jacobian / Hessian entry are the reference's. Differences: folding
// happens in the library, so is_constant / is_zero see only literal
// constants, and Expr::diff / Tape (internal to the reference's evaluator)
// are not exposed — templates are differentiated inside the library.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "nclopf_expr_program.h"

namespace nclopf {

/// expr.hpp:15-17
struct DomainError : std::runtime_error {
  explicit DomainError(const std::string& what) : std::runtime_error(what) {}
};

/// expr.hpp:19-31 (same order as ncl_expr_op)
enum class ExprOp : std::uint8_t { constant, var, param, add, sub, mul, div, pow, neg, sin_, cos_ };

struct ExprNode;
using ExprRef = std::shared_ptr<const ExprNode>;

/// expr.hpp:36-42
struct ExprNode {
  ExprOp op;
  double value = 0.0;
  int slot = -1;
  ExprRef a, b;
};

class Expr {
 public:
  Expr() : node_(nullptr) {}
  static Expr constant(double v) { return Expr(ExprOp::constant, {}, {}, v); }
  static Expr var(int slot) { return Expr(ExprOp::var, {}, {}, 0.0, slot); }
  static Expr param(int slot) { return Expr(ExprOp::param, {}, {}, 0.0, slot); }

  bool is_constant(double v) const { return node_ && node_->op == ExprOp::constant && node_->value == v; }
  bool is_zero() const { return is_constant(0.0); }
  const ExprRef& node() const { return node_; }

  friend Expr operator+(const Expr& x, const Expr& y) { return Expr(ExprOp::add, x, y); }
  friend Expr operator-(const Expr& x, const Expr& y) { return Expr(ExprOp::sub, x, y); }
  friend Expr operator*(const Expr& x, const Expr& y) { return Expr(ExprOp::mul, x, y); }
  friend Expr operator/(const Expr& x, const Expr& y) { return Expr(ExprOp::div, x, y); }
  friend Expr operator-(const Expr& x) { return Expr(ExprOp::neg, x, {}); }
  friend Expr pow(const Expr& x, double e) { return Expr(ExprOp::pow, x, {}, e); }
  friend Expr sin(const Expr& x) { return Expr(ExprOp::sin_, x, {}); }
  friend Expr cos(const Expr& x) { return Expr(ExprOp::cos_, x, {}); }

  friend Expr operator+(const Expr& x, double c) { return x + Expr::constant(c); }
  friend Expr operator+(double c, const Expr& x) { return Expr::constant(c) + x; }
  friend Expr operator-(const Expr& x, double c) { return x - Expr::constant(c); }
  friend Expr operator-(double c, const Expr& x) { return Expr::constant(c) - x; }
  friend Expr operator*(const Expr& x, double c) { return x * Expr::constant(c); }
  friend Expr operator*(double c, const Expr& x) { return Expr::constant(c) * x; }
  friend Expr operator/(const Expr& x, double c) { return x / Expr::constant(c); }

  /// the node program the C-ABI takes (topological order, root last)
  std::vector<ncl_expr_node> program() const {
    std::vector<ncl_expr_node> out;
    std::unordered_map<const ExprNode*, int> id;
    encode(node_.get(), out, id);
    return out;
  }

 private:
  Expr(ExprOp op, const Expr& a, const Expr& b, double v = 0.0, int slot = -1) {
    if ((op != ExprOp::constant && op != ExprOp::var && op != ExprOp::param && !a.node_) ||
        ((op == ExprOp::add || op == ExprOp::sub || op == ExprOp::mul || op == ExprOp::div) && !b.node_))
      throw std::invalid_argument("Expr: empty operand");
    node_ = std::make_shared<const ExprNode>(ExprNode{op, v, slot, a.node_, b.node_});
  }
  static int encode(const ExprNode* n, std::vector<ncl_expr_node>& out, std::unordered_map<const ExprNode*, int>& id) {
    if (!n) return -1;
    auto it = id.find(n);
    if (it != id.end()) return it->second;
    const int a = encode(n->a.get(), out, id), b = encode(n->b.get(), out, id);
    out.push_back(ncl_expr_node{static_cast<int32_t>(n->op), a, b, n->slot, n->value});
    return id[n] = static_cast<int>(out.size()) - 1;
  }
  ExprRef node_;
};

/// expr.hpp:108-135 (value() interprets the recorded DAG on the host; the
/// compiled derivative tapes live in the library)
class ExpressionTemplate {
 public:
  ExpressionTemplate() = default;
  ExpressionTemplate(Expr f, int num_var_slots, std::string name)
      : f_(std::move(f)), num_var_slots_(num_var_slots), name_(std::move(name)) {
    if (!f_.node()) throw std::invalid_argument("ExpressionTemplate: empty expression");
  }
  const std::string& name() const { return name_; }
  int num_var_slots() const { return num_var_slots_; }
  const Expr& expr() const { return f_; }
  double value(std::span<const double> v, std::span<const double> p) const { return eval(f_.node().get(), v, p); }

 private:
  static double eval(const ExprNode* n, std::span<const double> v, std::span<const double> p) {
    switch (n->op) {
      case ExprOp::constant: return n->value;
      case ExprOp::var: return v[n->slot];
      case ExprOp::param: return p[n->slot];
      case ExprOp::add: return eval(n->a.get(), v, p) + eval(n->b.get(), v, p);
      case ExprOp::sub: return eval(n->a.get(), v, p) - eval(n->b.get(), v, p);
      case ExprOp::mul: return eval(n->a.get(), v, p) * eval(n->b.get(), v, p);
      case ExprOp::div: return eval(n->a.get(), v, p) / eval(n->b.get(), v, p);
      case ExprOp::pow: return std::pow(eval(n->a.get(), v, p), n->value);
      case ExprOp::neg: return -eval(n->a.get(), v, p);
      case ExprOp::sin_: return std::sin(eval(n->a.get(), v, p));
      case ExprOp::cos_: return std::cos(eval(n->a.get(), v, p));
    }
    return 0.0;
  }
  Expr f_;
  int num_var_slots_ = 0;
  std::string name_;
};

}  // namespace nclopf
