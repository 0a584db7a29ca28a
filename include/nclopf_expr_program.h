/* nclopf_expr_program.h — plain-C encoding of an nclopf::Expr DAG and the
 * shared status codes of the C-ABI.
 *
 * The reference builds templates from nclopf::Expr values
 * (/root/reference/proj/include/nclopf/expr.hpp:46-81). A C-ABI cannot carry
 * shared_ptr DAGs, so a template crosses the boundary as a topologically
 * ordered node array: node k = op(node a, node b). Replaying the array through
 * the smart constructors (expr.cpp:38-93) reproduces the same folded DAG, so
 * derivatives, tapes and therefore floating-point results are identical on
 * both sides of the boundary. The root is the last node.
 */
#ifndef NCLOPF_EXPR_PROGRAM_H
#define NCLOPF_EXPR_PROGRAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same order as nclopf::ExprOp (expr.hpp:19-31). */
enum ncl_expr_op {
  NCL_OP_CONST = 0,
  NCL_OP_VAR = 1,
  NCL_OP_PARAM = 2,
  NCL_OP_ADD = 3,
  NCL_OP_SUB = 4,
  NCL_OP_MUL = 5,
  NCL_OP_DIV = 6,
  NCL_OP_POW = 7, /* a ^ value (constant exponent) */
  NCL_OP_NEG = 8,
  NCL_OP_SIN = 9,
  NCL_OP_COS = 10
};

typedef struct ncl_expr_node {
  int32_t op;    /* enum ncl_expr_op */
  int32_t a, b;  /* operand node indices (< k) or -1 */
  int32_t slot;  /* var/param slot or -1 */
  double value;  /* constant value or pow exponent */
} ncl_expr_node;

/* Status codes. Exceptions of the reference C++ API map 1:1:
 *   std::invalid_argument -> NCL_E_INVALID, std::logic_error -> NCL_E_LOGIC,
 *   nclopf::DomainError -> NCL_E_DOMAIN (sparse_sym.cpp:13-23, expr.hpp:15-17). */
enum ncl_status {
  NCL_OK = 0,
  NCL_E_INVALID = -1,
  NCL_E_LOGIC = -2,
  NCL_E_DOMAIN = -3,
  NCL_E_CUDA = -4,
  NCL_E_INTERNAL = -5,
  NCL_E_NOMEM = -6
};

#ifdef __cplusplus
}
#endif
#endif
