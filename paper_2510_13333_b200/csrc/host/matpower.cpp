// matpower_io; see matpower.hpp.
#include "host/matpower.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <sstream>

namespace nclb::matpower {

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Block {
  int line = 0;                          // line of "mpc.X = ["
  std::vector<std::vector<double>> rows;
  std::vector<int> row_line;
};

double number(const std::string& tok, int line) {
  if (tok == "Inf" || tok == "inf") return std::numeric_limits<double>::infinity();
  if (tok == "-Inf" || tok == "-inf") return -std::numeric_limits<double>::infinity();
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || *end != '\0') throw ParseError(line, "not a number: '" + tok + "'");
  return v;
}

// the numeric blocks (mpc.bus / gen / branch / gencost) and scalars
// (mpc.baseMVA) of the text; comments (% ...) and MATLAB decoration skipped
void scan(const std::string& text, std::map<std::string, Block>& blocks, std::map<std::string, double>& scalars,
          std::string& name) {
  std::istringstream in(text);
  std::string raw;
  int line = 0;
  Block* cur = nullptr;
  std::string curname;
  std::vector<double> row;
  auto flush_row = [&](int ln) {
    if (!row.empty()) {
      cur->rows.push_back(row);
      cur->row_line.push_back(ln);
      row.clear();
    }
  };
  while (std::getline(in, raw)) {
    ++line;
    const size_t pc = raw.find('%');
    std::string s = pc == std::string::npos ? raw : raw.substr(0, pc);
    if (!cur) {
      const size_t fn = s.find("function");
      if (fn != std::string::npos) {
        const size_t eq = s.find('=');
        if (eq != std::string::npos) {
          std::string nm = s.substr(eq + 1);
          nm.erase(0, nm.find_first_not_of(" \t"));
          nm.erase(nm.find_last_not_of(" \t;\r") + 1);
          name = nm;
        }
        continue;
      }
      const size_t mp = s.find("mpc.");
      if (mp == std::string::npos) continue;
      const size_t eq = s.find('=', mp);
      if (eq == std::string::npos) throw ParseError(line, "expected '=' after " + s.substr(mp));
      std::string key = s.substr(mp + 4, eq - mp - 4);
      key.erase(key.find_last_not_of(" \t") + 1);
      std::string rhs = s.substr(eq + 1);
      const size_t lb = rhs.find('[');
      if (lb == std::string::npos) {  // scalar (or a string such as version = '2')
        rhs.erase(0, rhs.find_first_not_of(" \t"));
        rhs.erase(rhs.find_last_not_of(" \t;\r") + 1);
        if (!rhs.empty() && rhs[0] != '\'') scalars[key] = number(rhs, line);
        continue;
      }
      if (blocks.count(key)) throw ParseError(line, "duplicate block mpc." + key);
      cur = &blocks[key];
      cur->line = line;
      curname = key;
      s = rhs.substr(lb + 1);
    }
    // inside a block: numbers, ';' ends a row, ']' ends the block
    std::string tok;
    bool done = false;
    for (size_t i = 0; i <= s.size() && !done; ++i) {
      const char c = i < s.size() ? s[i] : '\n';
      if (c == ' ' || c == '\t' || c == ',' || c == '\r' || c == '\n' || c == ';' || c == ']') {
        if (!tok.empty()) {
          row.push_back(number(tok, line));
          tok.clear();
        }
        if (c == ';') flush_row(line);
        if (c == ']') {
          flush_row(line);
          cur = nullptr;
          done = true;
        }
      } else {
        tok += c;
      }
    }
    if (cur) flush_row(line);  // a row ends at the end of its line as well
  }
  if (cur) throw ParseError(line, "unterminated block mpc." + curname);
}

double col(const std::vector<double>& r, size_t k, double dflt, int line, size_t need) {
  if (r.size() < need) throw ParseError(line, "row has " + std::to_string(r.size()) + " columns, need " + std::to_string(need));
  return k < r.size() ? r[k] : dflt;
}

}  // namespace

PowerNetwork parse_case(const std::string& text) {
  std::map<std::string, Block> blocks;
  std::map<std::string, double> scalars;
  PowerNetwork net;
  scan(text, blocks, scalars, net.name);
  if (!scalars.count("baseMVA")) throw ParseError(0, "missing mpc.baseMVA");
  net.base_mva = scalars["baseMVA"];
  if (!(net.base_mva > 0)) throw ValidationError("baseMVA must be positive");
  for (const char* k : {"bus", "gen", "branch"})
    if (!blocks.count(k)) throw ParseError(0, std::string("missing mpc.") + k);
  const double B = net.base_mva;
  std::map<int, int> idx;
  const Block& bb = blocks["bus"];
  for (size_t i = 0; i < bb.rows.size(); ++i) {
    const auto& r = bb.rows[i];
    const int ln = bb.row_line[i];
    Bus u;
    u.id = static_cast<int>(col(r, 0, 0, ln, 13));
    u.type = static_cast<int>(r[1]);
    u.pd = r[2] / B, u.qd = r[3] / B, u.gs = r[4] / B, u.bs = r[5] / B;
    u.area = static_cast<int>(r[6]), u.vm = r[7], u.va = r[8], u.base_kv = r[9], u.zone = static_cast<int>(r[10]);
    u.vmax = r[11], u.vmin = r[12];
    if (idx.count(u.id)) throw ParseError(ln, "duplicate bus id " + std::to_string(u.id));
    idx[u.id] = static_cast<int>(net.bus.size());
    if (u.type == 3) {
      if (net.ref >= 0) throw ValidationError("more than one reference bus");
      net.ref = static_cast<int>(net.bus.size());
    }
    net.bus.push_back(u);
  }
  if (net.ref < 0) throw ValidationError("no reference bus");
  const Block& gb = blocks["gen"];
  for (size_t i = 0; i < gb.rows.size(); ++i) {
    const auto& r = gb.rows[i];
    const int ln = gb.row_line[i];
    Gen g;
    g.bus = static_cast<int>(col(r, 0, 0, ln, 10));
    g.pg = r[1] / B, g.qg = r[2] / B, g.qmax = r[3] / B, g.qmin = r[4] / B, g.vg = r[5], g.mbase = r[6];
    g.status = r[7] > 0 ? 1 : 0;
    g.pmax = r[8] / B, g.pmin = r[9] / B;
    if (!idx.count(g.bus)) throw ValidationError("generator " + std::to_string(i) + " at unknown bus " + std::to_string(g.bus));
    if (g.status && (g.pmin > g.pmax || g.qmin > g.qmax))
      throw ValidationError("generator " + std::to_string(i) + " has inverted limits");
    net.gen.push_back(g);
  }
  const Block& lb = blocks["branch"];
  for (size_t i = 0; i < lb.rows.size(); ++i) {
    const auto& r = lb.rows[i];
    const int ln = lb.row_line[i];
    Branch e;
    e.f = static_cast<int>(col(r, 0, 0, ln, 11));
    e.t = static_cast<int>(r[1]);
    e.r = r[2], e.x = r[3], e.b = r[4];
    e.rate_a = r[5] / B, e.rate_b = r[6] / B, e.rate_c = r[7] / B;
    e.tap = r[8], e.shift = r[9];
    e.status = r[10] > 0 ? 1 : 0;
    e.angmin = col(r, 11, -360, ln, 11), e.angmax = col(r, 12, 360, ln, 11);
    if (!idx.count(e.f) || !idx.count(e.t)) throw ValidationError("branch " + std::to_string(i) + " is dangling");
    net.branch.push_back(e);
  }
  if (blocks.count("gencost")) {
    const Block& cb = blocks["gencost"];
    for (size_t i = 0; i < cb.rows.size() && i < net.gen.size(); ++i) {
      const auto& r = cb.rows[i];
      const int ln = cb.row_line[i];
      const int model = static_cast<int>(col(r, 0, 0, ln, 4));
      if (model != 2) throw ParseError(ln, "piecewise-linear cost (model 1) is not supported");
      const int nc = static_cast<int>(r[3]);
      if (nc < 0 || nc > 3) throw ParseError(ln, "polynomial cost of degree > 2 is not supported");
      if (static_cast<int>(r.size()) < 4 + nc) throw ParseError(ln, "gencost row too short");
      Gen& g = net.gen[i];
      g.ncost = nc;
      double c[3] = {0, 0, 0};  // c2, c1, c0
      for (int k = 0; k < nc; ++k) c[3 - nc + k] = r[4 + k];
      g.c2 = c[0], g.c1 = c[1], g.c0 = c[2];
    }
  }
  return net;
}

std::vector<TwoPort> branch_admittances(const PowerNetwork& net) {
  std::vector<TwoPort> out;
  out.reserve(net.branch.size());
  for (size_t l = 0; l < net.branch.size(); ++l) {
    const Branch& e = net.branch[l];
    if (e.r == 0.0 && e.x == 0.0) throw ValidationError("DegenerateBranch " + std::to_string(l) + ": r = x = 0");
    const std::complex<double> ys = 1.0 / std::complex<double>(e.r, e.x);
    const double tap = e.tap == 0.0 ? 1.0 : e.tap;
    const std::complex<double> t = std::polar(tap, e.shift * kPi / 180.0);
    const std::complex<double> bc(0.0, e.b / 2.0);
    TwoPort y;
    y.yff = (ys + bc) / (tap * tap);
    y.yft = -ys / std::conj(t);
    y.ytf = -ys / t;
    y.ytt = ys + bc;
    out.push_back(y);
  }
  return out;
}

namespace {
std::string fmt(double v) {
  if (std::isinf(v)) return v > 0 ? "Inf" : "-Inf";
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
}  // namespace

std::string serialize(const PowerNetwork& net) {
  const double B = net.base_mva;
  std::ostringstream o;
  o << "function mpc = " << (net.name.empty() ? "case" : net.name) << "\n";
  o << "mpc.version = '2';\nmpc.baseMVA = " << fmt(B) << ";\n";
  o << "%% bus data\nmpc.bus = [\n";
  for (const Bus& u : net.bus)
    o << "\t" << u.id << "\t" << u.type << "\t" << fmt(u.pd * B) << "\t" << fmt(u.qd * B) << "\t" << fmt(u.gs * B)
      << "\t" << fmt(u.bs * B) << "\t" << u.area << "\t" << fmt(u.vm) << "\t" << fmt(u.va) << "\t" << fmt(u.base_kv)
      << "\t" << u.zone << "\t" << fmt(u.vmax) << "\t" << fmt(u.vmin) << ";\n";
  o << "];\n%% generator data\nmpc.gen = [\n";
  for (const Gen& g : net.gen)
    o << "\t" << g.bus << "\t" << fmt(g.pg * B) << "\t" << fmt(g.qg * B) << "\t" << fmt(g.qmax * B) << "\t"
      << fmt(g.qmin * B) << "\t" << fmt(g.vg) << "\t" << fmt(g.mbase) << "\t" << g.status << "\t" << fmt(g.pmax * B)
      << "\t" << fmt(g.pmin * B) << ";\n";
  o << "];\n%% branch data\nmpc.branch = [\n";
  for (const Branch& e : net.branch)
    o << "\t" << e.f << "\t" << e.t << "\t" << fmt(e.r) << "\t" << fmt(e.x) << "\t" << fmt(e.b) << "\t"
      << fmt(e.rate_a * B) << "\t" << fmt(e.rate_b * B) << "\t" << fmt(e.rate_c * B) << "\t" << fmt(e.tap) << "\t"
      << fmt(e.shift) << "\t" << e.status << "\t" << fmt(e.angmin) << "\t" << fmt(e.angmax) << ";\n";
  o << "];\n%% generator cost data\nmpc.gencost = [\n";
  for (const Gen& g : net.gen) {
    o << "\t2\t0\t0\t3\t" << fmt(g.c2) << "\t" << fmt(g.c1) << "\t" << fmt(g.c0) << ";\n";
  }
  o << "];\n";
  return o.str();
}

std::string to_json(const PowerNetwork& net) {
  std::ostringstream o;
  o << "{\"name\": \"" << net.name << "\", \"baseMVA\": " << fmt(net.base_mva) << ", \"ref\": " << net.ref
    << ",\n \"bus\": [";
  for (size_t i = 0; i < net.bus.size(); ++i) {
    const Bus& u = net.bus[i];
    o << (i ? ", " : "") << "[" << u.id << ", " << u.type << ", " << fmt(u.pd) << ", " << fmt(u.qd) << ", "
      << fmt(u.gs) << ", " << fmt(u.bs) << ", " << fmt(u.vmin) << ", " << fmt(u.vmax) << "]";
  }
  o << "],\n \"branch\": [";
  for (size_t i = 0; i < net.branch.size(); ++i) {
    const Branch& e = net.branch[i];
    o << (i ? ", " : "") << "[" << e.f << ", " << e.t << ", " << fmt(e.r) << ", " << fmt(e.x) << ", " << fmt(e.b)
      << ", " << fmt(e.rate_a) << ", " << fmt(e.tap) << ", " << fmt(e.shift) << ", " << e.status << "]";
  }
  o << "],\n \"gen\": [";
  for (size_t i = 0; i < net.gen.size(); ++i) {
    const Gen& g = net.gen[i];
    o << (i ? ", " : "") << "[" << g.bus << ", " << fmt(g.pmin) << ", " << fmt(g.pmax) << ", " << fmt(g.qmin)
      << ", " << fmt(g.qmax) << ", " << g.status << ", " << fmt(g.c2) << ", " << fmt(g.c1) << ", " << fmt(g.c0)
      << "]";
  }
  o << "]}\n";
  return o.str();
}

Grid to_grid(const PowerNetwork& net) {
  Grid g;
  g.name = net.name;
  g.base_mva = net.base_mva;
  const double B = net.base_mva;
  std::map<int, int> idx;
  for (size_t i = 0; i < net.bus.size(); ++i) {
    const Bus& u = net.bus[i];
    idx[u.id] = static_cast<int>(i);
    g.pd.push_back(u.pd), g.qd.push_back(u.qd), g.gs.push_back(u.gs), g.bs.push_back(u.bs);
    g.vmin.push_back(u.vmin), g.vmax.push_back(u.vmax);
  }
  g.nb = static_cast<int>(net.bus.size());
  g.ref = net.ref;
  for (const Branch& e : net.branch) {
    if (!e.status) continue;  // out-of-service elements stay in the data model only
    g.f.push_back(idx.at(e.f)), g.t.push_back(idx.at(e.t));
    g.r.push_back(e.r), g.x.push_back(e.x), g.b.push_back(e.b);
    g.rate.push_back(e.rate_a > 0 ? e.rate_a : std::numeric_limits<double>::infinity());  // 0: unconstrained
    g.tap.push_back(e.tap == 0.0 ? 1.0 : e.tap);
    g.shift.push_back(e.shift * kPi / 180.0);
  }
  g.nl = static_cast<int>(g.f.size());
  for (const Gen& k : net.gen) {
    if (!k.status) continue;
    g.gbus.push_back(idx.at(k.bus));
    g.pmin.push_back(k.pmin), g.pmax.push_back(k.pmax), g.qmin.push_back(k.qmin), g.qmax.push_back(k.qmax);
    g.c2.push_back(k.c2 * B * B), g.c1.push_back(k.c1 * B), g.c0.push_back(k.c0);  // $/h of p in pu
  }
  g.ng = static_cast<int>(g.gbus.size());
  return g;
}

}  // namespace nclb::matpower
