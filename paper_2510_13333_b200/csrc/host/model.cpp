#include "model.hpp"

#include <algorithm>
#include <limits>
#include <stdexcept>

#include "sparse.hpp"

namespace nclb {

int allocate_registers(Program& p) {
  const int n = static_cast<int>(p.code.size());
  std::vector<int> last(n, -1);
  for (int i = 0; i < n; ++i) {
    if (p.code[i].a >= 0) last[p.code[i].a] = i;
    if (p.code[i].b >= 0) last[p.code[i].b] = i;
  }
  for (int o : p.out) last[o] = std::numeric_limits<int>::max();
  std::vector<int> phys(n, -1), freelist;
  int nphys = 0;
  for (int i = 0; i < n; ++i) {
    CInstr& ins = p.code[i];
    const int a = ins.a, b = ins.b;
    if (a >= 0) ins.a = phys[a];
    if (b >= 0) ins.b = phys[b];
    if (a >= 0 && last[a] == i) freelist.push_back(phys[a]);
    if (b >= 0 && b != a && last[b] == i) freelist.push_back(phys[b]);
    int r;
    if (!freelist.empty()) {
      r = freelist.back();
      freelist.pop_back();
    } else {
      r = nphys++;
    }
    phys[i] = r;
    // results nobody reads are dead immediately (never happens for roots)
    if (last[i] < 0) freelist.push_back(r);
    ins.dst = r;
  }
  for (int& o : p.out) o = phys[o];
  return nphys;
}

int HostBuilder::add_template(Template t) {
  if (t.nslots > kMaxSlots) throw Error{NCL_E_INVALID, "ModelBuilder: template has too many variable slots"};
  fams_.emplace_back(std::move(t));
  return static_cast<int>(fams_.size()) - 1;
}

int HostBuilder::add_rows(int count) {
  const int first = m_;
  m_ += count;
  return first;
}

// add_objective_term / add_constraint_term + check_instance (model.cpp:43-73)
void HostBuilder::add_terms(int tid, bool objective, int64_t count, const int* rows, int nv, const int* vars, int np,
                            const double* params) {
  if (tid < 0 || tid >= static_cast<int>(fams_.size()))
    throw Error{NCL_E_LOGIC, "vector::_M_range_check: template id out of range"};
  HFamily& f = fams_[tid];
  for (int64_t k = 0; k < count; ++k) {
    if (objective) {
      if (f.used && !f.objective) throw Error{NCL_E_LOGIC, "ModelBuilder: template already used for constraints"};
      f.objective = true;
    } else {
      if (f.used && f.objective) throw Error{NCL_E_LOGIC, "ModelBuilder: template already used for the objective"};
      if (rows[k] < 0 || rows[k] >= m_) throw Error{NCL_E_INVALID, "ModelBuilder: row out of range"};
    }
    if (nv != f.tmpl.nslots)
      throw Error{NCL_E_INVALID, "ModelBuilder: instance variable count mismatch for template " + f.tmpl.name};
    const int* v = vars + k * nv;
    for (int s = 0; s < nv; ++s)
      if (v[s] < 0 || v[s] >= n_)
        throw Error{NCL_E_INVALID, "ModelBuilder: variable index out of range in template " + f.tmpl.name};
    f.vars.insert(f.vars.end(), v, v + nv);
    if (f.pstart.empty()) f.pstart.push_back(0);
    if (np > 0) f.params.insert(f.params.end(), params + k * np, params + (k + 1) * np);
    f.pstart.push_back(static_cast<int64_t>(f.params.size()));
    f.np = std::max(f.np, np);
    f.rows.push_back(objective ? -1 : rows[k]);
    f.ninst++;
    f.used = true;
  }
}

namespace {
inline uint64_t key2(int a, int b) { return (static_cast<uint64_t>(static_cast<uint32_t>(a)) << 32) | static_cast<uint32_t>(b); }

// counting-sort gather builder: entries appended in canonical order
struct GatherBuilder {
  std::vector<int64_t> ptr;
  std::vector<int64_t> idx;
  std::vector<int64_t> fill;
  void init(int64_t nslots) { ptr.assign(nslots + 1, 0); }
  void count(int64_t slot) { ptr[slot + 1]++; }
  void finish_count() {
    for (size_t s = 0; s + 1 < ptr.size(); ++s) ptr[s + 1] += ptr[s];
    idx.resize(ptr.back());
    fill.assign(ptr.begin(), ptr.end() - 1);
  }
  void put(int64_t slot, int64_t c) { idx[fill[slot]++] = c; }
};
}  // namespace

BuiltModel HostBuilder::build() {
  BuiltModel M;
  M.n = n_;
  M.m = m_;
  // --- Jacobian / Hessian patterns (model.cpp:81-108): sorted unique keys
  std::vector<uint64_t> jk, hk;
  for (auto& f : fams_) {
    const int nv = f.tmpl.nslots;
    for (int64_t i = 0; i < f.ninst; ++i) {
      const int* v = f.vars.data() + i * nv;
      if (!f.objective)
        for (int s : f.tmpl.grad_slot) jk.push_back(key2(f.rows[i], v[s]));
      for (auto [hi, lo] : f.tmpl.hess_slot) {
        const int gi = v[hi], gj = v[lo];
        hk.push_back(gi >= gj ? key2(gi, gj) : key2(gj, gi));
      }
    }
  }
  std::sort(jk.begin(), jk.end());
  jk.erase(std::unique(jk.begin(), jk.end()), jk.end());
  std::sort(hk.begin(), hk.end());
  hk.erase(std::unique(hk.begin(), hk.end()), hk.end());
  M.jac_coords.resize(jk.size());
  for (size_t k = 0; k < jk.size(); ++k)
    M.jac_coords[k] = {static_cast<int>(jk[k] >> 32), static_cast<int>(jk[k] & 0xffffffffu)};
  M.hess_coords.resize(hk.size());
  for (size_t k = 0; k < hk.size(); ++k)
    M.hess_coords[k] = {static_cast<int>(hk[k] >> 32), static_cast<int>(hk[k] & 0xffffffffu)};
  auto jslot = [&](int r, int c) {
    return static_cast<int64_t>(std::lower_bound(jk.begin(), jk.end(), key2(r, c)) - jk.begin());
  };
  auto hslot = [&](int gi, int gj) {
    const uint64_t k = gi >= gj ? key2(gi, gj) : key2(gj, gi);
    return static_cast<int64_t>(std::lower_bound(hk.begin(), hk.end(), k) - hk.begin());
  };

  // --- per-family SoA tables, programs, contribution layout
  int64_t base = 0;
  M.f.resize(fams_.size());
  for (size_t fi = 0; fi < fams_.size(); ++fi) {
    HFamily& h = fams_[fi];
    BuiltModel::F& F = M.f[fi];
    F.ninst = h.ninst;
    F.nv = h.tmpl.nslots;
    F.np = h.np;
    F.G = static_cast<int>(h.tmpl.grad.size());
    F.H = static_cast<int>(h.tmpl.hess.size());
    F.objective = h.objective;
    F.vars.resize(static_cast<size_t>(F.nv) * F.ninst);
    for (int64_t i = 0; i < F.ninst; ++i)
      for (int s = 0; s < F.nv; ++s) F.vars[s * F.ninst + i] = h.vars[i * F.nv + s];
    F.params.assign(static_cast<size_t>(F.np) * F.ninst, 0.0);
    for (int64_t i = 0; i < F.ninst; ++i)
      for (int64_t q = h.pstart[i]; q < h.pstart[i + 1]; ++q) F.params[(q - h.pstart[i]) * F.ninst + i] = h.params[q];
    F.rows = h.rows;
    for (auto [hi, lo] : h.tmpl.hess_slot) {
      F.hess_hi.push_back(hi);
      F.hess_lo.push_back(lo);
    }
    std::vector<X> roots;
    F.prog[PK_V] = compile({h.tmpl.f});
    F.prog[PK_G] = compile(h.tmpl.grad.empty() ? std::vector<X>{X::constant(0.0)} : h.tmpl.grad);
    F.prog[PK_H] = compile(h.tmpl.hess.empty() ? std::vector<X>{X::constant(0.0)} : h.tmpl.hess);
    roots.push_back(h.tmpl.f);
    roots.insert(roots.end(), h.tmpl.grad.begin(), h.tmpl.grad.end());
    roots.insert(roots.end(), h.tmpl.hess.begin(), h.tmpl.hess.end());
    F.prog[PK_VGH] = compile(roots);
    for (int k = 0; k < PK_N; ++k) F.nregs[k] = allocate_registers(F.prog[k]);
    F.base = base;
    base += static_cast<int64_t>(1 + F.G + F.H) * F.ninst;
  }
  M.ncontrib = base;

  // --- reference-order gather lists
  GatherBuilder gc, gj, gh, gg, go;
  gc.init(m_);
  gj.init(static_cast<int64_t>(jk.size()));
  gh.init(static_cast<int64_t>(hk.size()));
  gg.init(n_);
  go.init(1);
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t fi = 0; fi < fams_.size(); ++fi) {
      const HFamily& h = fams_[fi];
      const BuiltModel::F& F = M.f[fi];
      const int nv = F.nv;
      for (int64_t i = 0; i < F.ninst; ++i) {
        const int* v = h.vars.data() + i * nv;
        const int64_t cval = F.base + i;
        if (F.objective) {
          pass == 0 ? go.count(0) : go.put(0, cval);
          for (int g = 0; g < F.G; ++g) {
            const int64_t c = F.base + (1 + g) * F.ninst + i;
            const int var = v[h.tmpl.grad_slot[g]];
            pass == 0 ? gg.count(var) : gg.put(var, c);
          }
        } else {
          pass == 0 ? gc.count(h.rows[i]) : gc.put(h.rows[i], cval);
          for (int g = 0; g < F.G; ++g) {
            const int64_t c = F.base + (1 + g) * F.ninst + i;
            const int64_t s = jslot(h.rows[i], v[h.tmpl.grad_slot[g]]);
            pass == 0 ? gj.count(s) : gj.put(s, c);
          }
        }
        for (int hh = 0; hh < F.H; ++hh) {
          const int64_t c = F.base + (1 + F.G + hh) * F.ninst + i;
          const int64_t s = hslot(v[h.tmpl.hess_slot[hh].first], v[h.tmpl.hess_slot[hh].second]);
          pass == 0 ? gh.count(s) : gh.put(s, c);
        }
      }
    }
    if (pass == 0) {
      gc.finish_count();
      gj.finish_count();
      gh.finish_count();
      gg.finish_count();
      go.finish_count();
    }
  }
  M.c_ptr = std::move(gc.ptr);
  M.c_idx = std::move(gc.idx);
  M.j_ptr = std::move(gj.ptr);
  M.j_idx = std::move(gj.idx);
  M.h_ptr = std::move(gh.ptr);
  M.h_idx = std::move(gh.idx);
  M.g_ptr = std::move(gg.ptr);
  M.g_idx = std::move(gg.idx);
  M.o_ptr = std::move(go.ptr);
  M.o_idx = std::move(go.idx);
  // jac_times (row ranges) and jac_trans_times (by column, k ascending)
  const int64_t nj = static_cast<int64_t>(M.jac_coords.size());
  M.jr_ptr.assign(m_ + 1, 0);
  M.jcol.resize(nj);
  M.jrow.resize(nj);
  std::vector<int64_t> cc(n_ + 1, 0);
  for (int64_t k = 0; k < nj; ++k) {
    M.jr_ptr[M.jac_coords[k].first + 1]++;
    cc[M.jac_coords[k].second + 1]++;
    M.jrow[k] = M.jac_coords[k].first;
    M.jcol[k] = M.jac_coords[k].second;
  }
  for (int r = 0; r < m_; ++r) M.jr_ptr[r + 1] += M.jr_ptr[r];
  for (int c = 0; c < n_; ++c) cc[c + 1] += cc[c];
  M.jt_ptr = cc;
  M.jt_idx.resize(nj);
  {
    std::vector<int64_t> fp(cc.begin(), cc.end() - 1);
    for (int64_t k = 0; k < nj; ++k) M.jt_idx[fp[M.jac_coords[k].second]++] = static_cast<int>(k);
  }
  M.fams = std::move(fams_);
  fams_.clear();
  return M;
}

}  // namespace nclb
