// matpower_io: MATPOWER case text -> validated per-unit
// PowerNetwork, the standard branch two-port admittances, a canonical
// serializer (round trip) and the conversion to the SCOPF builder's Grid
// (in-service elements). Host code, setup only.
#pragma once

#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/scopf.hpp"

namespace nclb::matpower {

struct ParseError : std::invalid_argument {
  ParseError(int line, const std::string& why)
      : std::invalid_argument("ParseError(line " + std::to_string(line) + "): " + why), line(line) {}
  int line;
};
struct ValidationError : std::invalid_argument {
  explicit ValidationError(const std::string& why) : std::invalid_argument("ValidationError: " + why) {}
};

struct Bus {
  int id = 0, type = 1;                // 1 PQ, 2 PV, 3 ref, 4 isolated
  double pd = 0, qd = 0, gs = 0, bs = 0;  // pu
  double vm = 1, va = 0, base_kv = 0, vmax = 1.1, vmin = 0.9;
  int area = 1, zone = 1;
};
struct Branch {
  int f = 0, t = 0;                 // bus ids
  double r = 0, x = 0, b = 0;       // pu
  double rate_a = 0, rate_b = 0, rate_c = 0;  // pu MVA (0 = unconstrained)
  double tap = 0, shift = 0;        // MATPOWER ratio (0 = 1) and angle (degrees)
  int status = 1;
  double angmin = -360, angmax = 360;
};
struct Gen {
  int bus = 0;
  double pg = 0, qg = 0, qmax = 0, qmin = 0, vg = 1, mbase = 100;  // pu
  int status = 1;
  double pmax = 0, pmin = 0;  // pu
  // polynomial cost in $/h of p in MW (MATPOWER gencost model 2, degree <= 2)
  double c2 = 0, c1 = 0, c0 = 0;
  int ncost = 0;
};
struct PowerNetwork {
  std::string name;
  double base_mva = 100.0;
  std::vector<Bus> bus;
  std::vector<Branch> branch;
  std::vector<Gen> gen;
  int ref = -1;  // index of the reference bus
};

PowerNetwork parse_case(const std::string& text);

struct TwoPort {
  std::complex<double> yff, yft, ytf, ytt;
};
// standard MATPOWER pi model with tap and phase shift
std::vector<TwoPort> branch_admittances(const PowerNetwork& net);

// canonical MATPOWER text (parse(serialize(net)) == net)
std::string serialize(const PowerNetwork& net);
// canonical JSON dump
std::string to_json(const PowerNetwork& net);

// the SCOPF builder's Grid over the in-service elements (buses renumbered
// in file order, costs converted to p in pu)
Grid to_grid(const PowerNetwork& net);

}  // namespace nclb::matpower
