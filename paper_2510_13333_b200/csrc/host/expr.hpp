// Clean-room symbolic expressions with the reference's semantics
// (/root/reference/proj/include/nclopf/expr.hpp:19-135,
//  /root/reference/proj/src/expr.cpp:26-240): same smart-constructor folding,
// same differentiation rules, same choice of nonzero gradient / lower-Hessian
// entries, so derivative values are computed by the same operation sequence.
//
// The B200 path does not interpret one tape per entry (expr.cpp:168-220).
// Instead all outputs a GPU kernel needs (value, gradient entries, Hessian
// entries) are compiled into ONE straight-line register program with
// hash-consed common-subexpression elimination across outputs; structurally
// identical nodes compute bit-identical values, so CSE never changes a result.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/nclopf_expr_program.h"

namespace nclb {

struct XNode;
using XRef = std::shared_ptr<const XNode>;
struct XNode {
  int op;  // ncl_expr_op
  double value = 0.0;
  int slot = -1;
  XRef a, b;
};

class X {
 public:
  X() = default;
  explicit X(XRef n) : n_(std::move(n)) {}
  static X constant(double v);
  static X var(int slot);
  static X param(int slot);
  bool is_constant(double v) const;
  bool is_zero() const { return is_constant(0.0); }
  const XRef& node() const { return n_; }
  X diff(int slot) const;
  static X make(int op, const X& a, const X& b, double v = 0.0);

 private:
  XRef n_;
};

X operator+(const X& a, const X& b);
X operator-(const X& a, const X& b);
X operator*(const X& a, const X& b);
X operator/(const X& a, const X& b);
X operator-(const X& a);
X xpow(const X& a, double e);
X xsin(const X& a);
X xcos(const X& a);

// Replay a C-ABI node program through the smart constructors.
X build_from_program(int nn, const ncl_expr_node* nodes);

// Compiler-side instruction: operands a/b are instruction indices before
// register allocation and physical registers after; dst is the physical
// destination register.
struct CInstr {
  int op = 0;
  int a = -1, b = -1, slot = -1;
  double value = 0.0;
  int dst = -1;
};

struct Program {
  std::vector<CInstr> code;
  std::vector<int> out;  // register of each requested root
};

// Device instruction (16 bytes): a holds the slot for var/param.
struct Instr {
  int8_t op;
  int8_t pad;
  int16_t dst;
  int16_t a;
  int16_t b;
  double value;
};
static_assert(sizeof(Instr) == 16, "Instr layout");
std::vector<Instr> encode(const Program& p);

// Kinds of program a family carries (value, gradient, Hessian, all three).
enum ProgKind { PK_V = 0, PK_G = 1, PK_H = 2, PK_VGH = 3, PK_N = 4 };

// CSE-compiled program computing every expression in `roots`.
Program compile(const std::vector<X>& roots);

// ExpressionTemplate (expr.hpp:108-135): grad entries for every slot with a
// nonzero first derivative, lower-Hessian entries (i>=j) for nonzero seconds
// of those, in the reference's loop order (expr.cpp:224-235).
struct Template {
  std::string name;
  int nslots = 0;
  X f;
  std::vector<int> grad_slot;
  std::vector<X> grad;
  std::vector<std::pair<int, int>> hess_slot;  // (hi, lo)
  std::vector<X> hess;
  Template(X f, int nslots, std::string name);
};

}  // namespace nclb
