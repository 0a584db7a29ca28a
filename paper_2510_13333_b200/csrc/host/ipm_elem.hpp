// Element-wise formulas and fixed-order reductions of the NCL/IPM iteration
// (north_star step (4): the IPM vector kernels), shared VERBATIM by the GPU
// kernels (csrc/cuda/ipm.cu, compiled with --fmad=false) and by the CPU
// oracle backend (oracle/ref_ipm.cpp, -ffp-contract=off): the same source
// expression per element on both sides, and the same reduction tree
// (kRedBlocks x kRedThreads partials, block-local halving tree, then the
// kRedBlocks block partials folded to kRedThreads and the same halving tree
// again), so sums/maxima are bit-identical on both backends given
// bit-identical inputs.
//
// The subproblem for the generic NLP
//   min f(x)  s.t.  gl <= c(x) <= gu,  xl <= x <= xu
// in NCL form with a free regularisation r (m) and slacks s (m; s == gl on
// equality rows):
//   min  sf f(x) + lamN'r + rho/2 |r|^2
//   s.t. c(x) - r - s = 0,  xl <= x <= xu,  gl <= s <= gu.
// Lagrangian  L = sf f + lamN'r + rho/2 r'r + y'(c - r - s) - zl'(x-xl)
//                 - zu'(xu-x) - vl'(s-gl) - vu'(gu-s),
// so y = lamN + rho r at a stationary point (the NCL multiplier
// update lamN <- y) and the complementarity rows W1 W2 e <= t of PAPER.md:323
// are rows with gu = 0 whose r plays the role of t.
//
// Newton system (primal-dual, bound duals eliminated), with
//   Sx = zl/(x-xl) + zu/(xu-x),  Ss = vl/(s-gl) + vu/(gu-s),
//   gx = sf grad + J'y - mu/(x-xl) + mu/(xu-x),  gr = lamN + rho r - y,
//   gs = -y - mu/(s-gl) + mu/(gu-s),             gy = c - r - s:
//   (W + Sx + dw) dx + J'dy = -gx;  rho dr - dy = -gr;  Ss ds - dy = -gs;
//   J dx - dr - ds - dc dy = -gy.
// Eliminating dr, ds (block C = 1/rho + 1/Ss) gives
//   dy = D (J dx + q),  D = 1/(1/rho + [ineq] 1/Ss + dc),
//   q  = gy + gr/rho + [ineq] gs/Ss,
//   (W + Sx + dw + J'DJ) dx = -(gx + J'(D q))        (the condensed K),
// and the recovery dr = (dy - gr)/rho, ds = (dy - gs)/Ss,
//   dzl = mu/(x-xl) - zl - zl/(x-xl) dx, dzu = mu/(xu-x) - zu + zu/(xu-x) dx
// (and the same for vl, vu with s, ds) — derived from the full Newton
// linearisation as SURVEY.md §8(a) row a16 requires, not from the printed
// recovery formulas of PAPER.md:424-426 (sign caveat).
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define NCL_HD __host__ __device__ __forceinline__
#else
#define NCL_HD inline
#endif

namespace nclb::ipm {

constexpr double kBig = 1e20;  // |bound| >= kBig means "no bound" (Ipopt's nlp_lower/upper_bound_inf)
constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kRedThreads = 256;

NCL_HD bool has_lo(double b) { return b > -kBig; }
NCL_HD bool has_up(double b) { return b < kBig; }

// All vectors of one solver instance (device pointers on the GPU backend,
// host pointers on the oracle backend). Sizes: x-part n, row-part m.
struct Vecs {
  int n = 0, m = 0;
  const double *xl = nullptr, *xu = nullptr, *gl = nullptr, *gu = nullptr;
  double *x = nullptr, *zl = nullptr, *zu = nullptr;
  double *r = nullptr, *s = nullptr, *y = nullptr, *vl = nullptr, *vu = nullptr, *lamN = nullptr;
  double *c = nullptr, *grad = nullptr, *jty = nullptr;
  double *sigx = nullptr, *gx = nullptr, *rhs = nullptr, *jtdq = nullptr;
  double *D = nullptr, *q = nullptr, *dq = nullptr;
  double *dx = nullptr, *dzl = nullptr, *dzu = nullptr;
  double *dr = nullptr, *ds = nullptr, *dy = nullptr, *dvl = nullptr, *dvu = nullptr, *jdx = nullptr;
  double *xt = nullptr, *rt = nullptr, *st = nullptr, *ct = nullptr;
};

struct Scal {
  double sf = 1.0;     // objective scale
  double mu = 0.1;     // barrier
  double rho = 100.0;  // NCL penalty
  double dc = 0.0;     // dual regularisation
  double alpha = 1.0, alpha_dual = 1.0;
  double tau = 0.99;
  double kappa_sigma = 1e10;
  double push = 1e-2, frac = 1e-2;
};

// ---------------------------------------------------------------- initial point
// Ipopt-style bound push of x0 (bound_push = bound_frac = 1e-2) and unit bound duals.
NCL_HD double push_into(double v, double lo, double up, double push, double frac) {
  const bool hl = has_lo(lo), hu = has_up(up);
  if (hl && hu) {
    const double w = up - lo;
    const double pl = fmin(push * fmax(1.0, fabs(lo)), frac * w);
    const double pu = fmin(push * fmax(1.0, fabs(up)), frac * w);
    return fmin(fmax(v, lo + pl), up - pu);
  }
  if (hl) return fmax(v, lo + push * fmax(1.0, fabs(lo)));
  if (hu) return fmin(v, up - push * fmax(1.0, fabs(up)));
  return v;
}
NCL_HD void init_x(const Vecs& V, int i, const Scal& S) {
  V.x[i] = push_into(V.x[i], V.xl[i], V.xu[i], S.push, S.frac);
  V.zl[i] = has_lo(V.xl[i]) ? 1.0 : 0.0;
  V.zu[i] = has_up(V.xu[i]) ? 1.0 : 0.0;
}
// after c(x) is known
NCL_HD void init_row(const Vecs& V, int i, const Scal& S) {
  const double lo = V.gl[i], up = V.gu[i];
  const bool eq = lo == up;
  V.s[i] = eq ? lo : push_into(V.c[i], lo, up, S.push, S.frac);
  V.r[i] = 0.0;
  V.y[i] = 0.0;
  V.lamN[i] = 0.0;
  V.vl[i] = (!eq && has_lo(lo)) ? 1.0 : 0.0;
  V.vu[i] = (!eq && has_up(up)) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- Newton system
NCL_HD void newton_x(const Vecs& V, int i, const Scal& S) {
  const double x = V.x[i], lo = V.xl[i], up = V.xu[i];
  double sig = 0.0, g = S.sf * V.grad[i] + V.jty[i];
  if (has_lo(lo)) {
    const double sl = x - lo;
    sig += V.zl[i] / sl;
    g -= S.mu / sl;
  }
  if (has_up(up)) {
    const double su = up - x;
    sig += V.zu[i] / su;
    g += S.mu / su;
  }
  V.sigx[i] = sig;
  V.gx[i] = g;
}
// gr, gy, and for inequality rows Ss and gs
NCL_HD void row_terms(const Vecs& V, int i, const Scal& S, double& gr, double& gy, double& ss, double& gs,
                      bool& ineq) {
  const double lo = V.gl[i], up = V.gu[i], s = V.s[i], y = V.y[i];
  gr = V.lamN[i] + S.rho * V.r[i] - y;
  gy = V.c[i] - V.r[i] - s;
  ineq = lo != up;
  ss = 0.0;
  gs = -y;
  if (ineq) {
    if (has_lo(lo)) {
      const double sl = s - lo;
      ss += V.vl[i] / sl;
      gs -= S.mu / sl;
    }
    if (has_up(up)) {
      const double su = up - s;
      ss += V.vu[i] / su;
      gs += S.mu / su;
    }
  }
}
NCL_HD void newton_row(const Vecs& V, int i, const Scal& S) {
  double gr, gy, ss, gs;
  bool ineq;
  row_terms(V, i, S, gr, gy, ss, gs, ineq);
  double cc = 1.0 / S.rho, qq = gy + gr / S.rho;
  if (ineq) {
    cc += 1.0 / ss;
    qq += gs / ss;
  }
  cc += S.dc;
  const double d = 1.0 / cc;
  V.D[i] = d;
  V.q[i] = qq;
  V.dq[i] = d * qq;
}
// rhs of the condensed system, after jtdq = J'(D q)
NCL_HD void rhs_x(const Vecs& V, int i) { V.rhs[i] = -(V.gx[i] + V.jtdq[i]); }

// ---------------------------------------------------------------- recovery
NCL_HD void recover_x(const Vecs& V, int i, const Scal& S) {
  const double x = V.x[i], lo = V.xl[i], up = V.xu[i], d = V.dx[i];
  if (has_lo(lo)) {
    const double sl = x - lo;
    V.dzl[i] = S.mu / sl - V.zl[i] - (V.zl[i] / sl) * d;
  } else {
    V.dzl[i] = 0.0;
  }
  if (has_up(up)) {
    const double su = up - x;
    V.dzu[i] = S.mu / su - V.zu[i] + (V.zu[i] / su) * d;
  } else {
    V.dzu[i] = 0.0;
  }
}
// after jdx = J dx
NCL_HD void recover_row(const Vecs& V, int i, const Scal& S) {
  double gr, gy, ss, gs;
  bool ineq;
  row_terms(V, i, S, gr, gy, ss, gs, ineq);
  const double dy = V.D[i] * (V.jdx[i] + V.q[i]);
  V.dy[i] = dy;
  V.dr[i] = (dy - gr) / S.rho;
  double ds = 0.0, dvl = 0.0, dvu = 0.0;
  if (ineq) {
    ds = (dy - gs) / ss;
    const double s = V.s[i], lo = V.gl[i], up = V.gu[i];
    if (has_lo(lo)) {
      const double sl = s - lo;
      dvl = S.mu / sl - V.vl[i] - (V.vl[i] / sl) * ds;
    }
    if (has_up(up)) {
      const double su = up - s;
      dvu = S.mu / su - V.vu[i] + (V.vu[i] / su) * ds;
    }
  }
  V.ds[i] = ds;
  V.dvl[i] = dvl;
  V.dvu[i] = dvu;
}

// ---------------------------------------------------------------- trial / accept
NCL_HD void trial_x(const Vecs& V, int i, const Scal& S) { V.xt[i] = V.x[i] + S.alpha * V.dx[i]; }
NCL_HD void trial_row(const Vecs& V, int i, const Scal& S) {
  V.rt[i] = V.r[i] + S.alpha * V.dr[i];
  V.st[i] = V.gl[i] == V.gu[i] ? V.s[i] : V.s[i] + S.alpha * V.ds[i];
}
NCL_HD double safeguard(double z, double slack, const Scal& S) {
  // Ipopt's kappa_sigma reset of the bound duals
  return fmax(fmin(z, S.kappa_sigma * S.mu / slack), S.mu / (S.kappa_sigma * slack));
}
NCL_HD void accept_x(const Vecs& V, int i, const Scal& S) {
  const double x = V.xt[i];
  V.x[i] = x;
  if (has_lo(V.xl[i])) V.zl[i] = safeguard(V.zl[i] + S.alpha_dual * V.dzl[i], x - V.xl[i], S);
  if (has_up(V.xu[i])) V.zu[i] = safeguard(V.zu[i] + S.alpha_dual * V.dzu[i], V.xu[i] - x, S);
}
NCL_HD void accept_row(const Vecs& V, int i, const Scal& S) {
  const double s = V.st[i];
  V.r[i] = V.rt[i];
  V.s[i] = s;
  V.c[i] = V.ct[i];
  V.y[i] = V.y[i] + S.alpha * V.dy[i];
  if (V.gl[i] != V.gu[i]) {
    if (has_lo(V.gl[i])) V.vl[i] = safeguard(V.vl[i] + S.alpha_dual * V.dvl[i], s - V.gl[i], S);
    if (has_up(V.gu[i])) V.vu[i] = safeguard(V.vu[i] + S.alpha_dual * V.dvu[i], V.gu[i] - s, S);
  }
}
// restoration shortcut: the NCL subproblem is always feasible,
// r := c - s zeroes the constraint violation exactly.
NCL_HD void restore_row(const Vecs& V, int i) { V.r[i] = V.c[i] - V.s[i]; }
NCL_HD void update_multiplier_row(const Vecs& V, int i) { V.lamN[i] = V.y[i]; }

// ---------------------------------------------------------------- reductions
enum Comb : int { kSum = 0, kMax = 1, kMin = 2 };
NCL_HD double comb(int k, double a, double b) {
  return k == kSum ? a + b : (k == kMax ? fmax(a, b) : fmin(a, b));
}
NCL_HD double comb_init(int k) { return k == kSum ? 0.0 : (k == kMax ? 0.0 : 1e300); }

// Each reduction kind: NV accumulators with fixed combine kinds; index space
// [0, n) = x-part, [n, n+m) = row-part.
// R_KKT: max|dual_x|, max|primal|, max|dual_r,s|, max|compl-mu|, max|compl|, sum|y|, sum|z|
struct RedKkt {
  static constexpr int NV = 7;
  NCL_HD static int kind(int k) { return k < 5 ? kMax : kSum; }
  NCL_HD static void elem(const Vecs& V, int64_t j, const Scal& S, double* a) {
    if (j < V.n) {
      const int i = static_cast<int>(j);
      const double x = V.x[i], lo = V.xl[i], up = V.xu[i];
      double d = S.sf * V.grad[i] + V.jty[i];
      if (has_lo(lo)) {
        const double z = V.zl[i], p = (x - lo) * z;
        d -= z;
        a[3] = fmax(a[3], fabs(p - S.mu));
        a[4] = fmax(a[4], fabs(p));
        a[6] += fabs(z);
      }
      if (has_up(up)) {
        const double z = V.zu[i], p = (up - x) * z;
        d += z;
        a[3] = fmax(a[3], fabs(p - S.mu));
        a[4] = fmax(a[4], fabs(p));
        a[6] += fabs(z);
      }
      a[0] = fmax(a[0], fabs(d));
    } else {
      const int i = static_cast<int>(j - V.n);
      const double lo = V.gl[i], up = V.gu[i], s = V.s[i], y = V.y[i];
      a[1] = fmax(a[1], fabs(V.c[i] - V.r[i] - s));
      a[2] = fmax(a[2], fabs(V.lamN[i] + S.rho * V.r[i] - y));
      a[5] += fabs(y);
      if (lo != up) {
        double d = -y;
        if (has_lo(lo)) {
          const double z = V.vl[i], p = (s - lo) * z;
          d -= z;
          a[3] = fmax(a[3], fabs(p - S.mu));
          a[4] = fmax(a[4], fabs(p));
          a[6] += fabs(z);
        }
        if (has_up(up)) {
          const double z = V.vu[i], p = (up - s) * z;
          d += z;
          a[3] = fmax(a[3], fabs(p - S.mu));
          a[4] = fmax(a[4], fabs(p));
          a[6] += fabs(z);
        }
        a[2] = fmax(a[2], fabs(d));
      }
    }
  }
};

// fraction to the boundary: min alpha_primal, min alpha_dual
struct RedFtb {
  static constexpr int NV = 2;
  NCL_HD static int kind(int) { return kMin; }
  NCL_HD static void step(double v, double dv, double tau, double& a) {
    if (dv < 0.0) a = fmin(a, -tau * v / dv);
  }
  NCL_HD static void elem(const Vecs& V, int64_t j, const Scal& S, double* a) {
    if (j < V.n) {
      const int i = static_cast<int>(j);
      const double x = V.x[i], d = V.dx[i];
      if (has_lo(V.xl[i])) {
        step(x - V.xl[i], d, S.tau, a[0]);
        step(V.zl[i], V.dzl[i], S.tau, a[1]);
      }
      if (has_up(V.xu[i])) {
        step(V.xu[i] - x, -d, S.tau, a[0]);
        step(V.zu[i], V.dzu[i], S.tau, a[1]);
      }
    } else {
      const int i = static_cast<int>(j - V.n);
      if (V.gl[i] == V.gu[i]) return;
      const double s = V.s[i], d = V.ds[i];
      if (has_lo(V.gl[i])) {
        step(s - V.gl[i], d, S.tau, a[0]);
        step(V.vl[i], V.dvl[i], S.tau, a[1]);
      }
      if (has_up(V.gu[i])) {
        step(V.gu[i] - s, -d, S.tau, a[0]);
        step(V.vu[i], V.dvu[i], S.tau, a[1]);
      }
    }
  }
};

// merit at the trial point (xt, rt, st, ct): sum theta (l1 violation),
// sum (lamN r + rho/2 r^2), sum of -log barrier terms, count of non-interior
struct RedMerit {
  static constexpr int NV = 4;
  NCL_HD static int kind(int) { return kSum; }
  NCL_HD static void elem(const Vecs& V, int64_t j, const Scal& S, double* a) {
    if (j < V.n) {
      const int i = static_cast<int>(j);
      const double x = V.xt[i];
      if (has_lo(V.xl[i])) {
        const double sl = x - V.xl[i];
        if (sl > 0.0) a[2] -= log(sl);
        else a[3] += 1.0;
      }
      if (has_up(V.xu[i])) {
        const double su = V.xu[i] - x;
        if (su > 0.0) a[2] -= log(su);
        else a[3] += 1.0;
      }
    } else {
      const int i = static_cast<int>(j - V.n);
      const double r = V.rt[i], s = V.st[i];
      a[0] += fabs(V.ct[i] - r - s);
      a[1] += V.lamN[i] * r + 0.5 * S.rho * (r * r);
      if (V.gl[i] != V.gu[i]) {
        if (has_lo(V.gl[i])) {
          const double sl = s - V.gl[i];
          if (sl > 0.0) a[2] -= log(sl);
          else a[3] += 1.0;
        }
        if (has_up(V.gu[i])) {
          const double su = V.gu[i] - s;
          if (su > 0.0) a[2] -= log(su);
          else a[3] += 1.0;
        }
      }
    }
  }
};

// directional derivative of the barrier objective along (dx, dr, ds)
struct RedDphi {
  static constexpr int NV = 1;
  NCL_HD static int kind(int) { return kSum; }
  NCL_HD static void elem(const Vecs& V, int64_t j, const Scal& S, double* a) {
    if (j < V.n) {
      const int i = static_cast<int>(j);
      const double x = V.x[i];
      double g = S.sf * V.grad[i];
      if (has_lo(V.xl[i])) g -= S.mu / (x - V.xl[i]);
      if (has_up(V.xu[i])) g += S.mu / (V.xu[i] - x);
      a[0] += g * V.dx[i];
    } else {
      const int i = static_cast<int>(j - V.n);
      double t = (V.lamN[i] + S.rho * V.r[i]) * V.dr[i];
      if (V.gl[i] != V.gu[i]) {
        const double s = V.s[i];
        double g = 0.0;
        if (has_lo(V.gl[i])) g -= S.mu / (s - V.gl[i]);
        if (has_up(V.gu[i])) g += S.mu / (V.gu[i] - s);
        t += g * V.ds[i];
      }
      a[0] += t;
    }
  }
};

// max|r| (NCL outer test) and max|dx| / max|x| (tiny-step test)
struct RedRinf {
  static constexpr int NV = 3;
  NCL_HD static int kind(int) { return kMax; }
  NCL_HD static void elem(const Vecs& V, int64_t j, const Scal&, double* a) {
    if (j < V.n) {
      a[1] = fmax(a[1], fabs(V.dx[j]));
      a[2] = fmax(a[2], fabs(V.x[j]));
    } else {
      a[0] = fmax(a[0], fabs(V.r[j - V.n]));
    }
  }
};

// CPU emulation of the GPU reduction order: thread t of block b visits
// j = b*T + t, j += B*T; block-local halving tree (pairs (t, t+h), h = T/2..1);
// then the B block partials: p[t] (+) p[t+T] for t + T < B, and the same
// halving tree over T (csrc/cuda/ipm.cu, last block to finish).
template <class R>
void reduce_host(const Vecs& V, const Scal& S, double* out) {
  const int64_t N = static_cast<int64_t>(V.n) + V.m;
  constexpr int B = kRedBlocks, T = kRedThreads, NV = R::NV;
  static_assert(B > T && B <= 2 * T, "final fold assumes T < B <= 2T");
  static thread_local double part[B * T * 8];
  static thread_local double fin[T * 8];
  static_assert(NV <= 8, "too many accumulators");
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < T; ++t) {
      double* a = part + (static_cast<int64_t>(b) * T + t) * NV;
      for (int k = 0; k < NV; ++k) a[k] = comb_init(R::kind(k));
      for (int64_t j = static_cast<int64_t>(b) * T + t; j < N; j += static_cast<int64_t>(B) * T) R::elem(V, j, S, a);
    }
  auto tree = [](double* blk) {
    for (int h = T / 2; h > 0; h >>= 1)
      for (int t = 0; t < h; ++t)
        for (int k = 0; k < NV; ++k) blk[t * NV + k] = comb(R::kind(k), blk[t * NV + k], blk[(t + h) * NV + k]);
  };
  for (int b = 0; b < B; ++b) tree(part + static_cast<int64_t>(b) * T * NV);
  auto blockp = [&](int b, int k) { return part[static_cast<int64_t>(b) * T * NV + k]; };
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < NV; ++k)
      fin[t * NV + k] = t + T < B ? comb(R::kind(k), blockp(t, k), blockp(t + T, k)) : blockp(t, k);
  tree(fin);
  for (int k = 0; k < NV; ++k) out[k] = fin[k];
}

}  // namespace nclb::ipm
