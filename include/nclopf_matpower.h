/* nclopf_matpower.h — matpower_io C-ABI.
 *
 * The reference has no code for this module (SPEC only): a MATPOWER case
 * parser into a validated per-unit network (out-of-service elements kept and
 * flagged), the standard branch two-port admittances, a canonical serializer
 * (parse(serialize(net)) == net), a JSON dump, and the corrective SCOPF of a
 * parsed network (scopf_builder input). Host code, setup only. */
#ifndef NCLOPF_MATPOWER_H
#define NCLOPF_MATPOWER_H

#include <stdint.h>

#include "nclopf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ncl_network* ncl_network_t;
typedef struct ncl_network_info {
  double base_mva;
  int nbus, nbranch, ngen, ref; /* all elements; ref = index of the reference bus */
  int nbranch_in, ngen_in;      /* in service */
} ncl_network_info;

/* parse_case(text): NCL_E_INVALID with "ParseError(line N): ..." or
 * "ValidationError: ..." (no / several reference buses, dangling branch,
 * inverted generator limits, piecewise-linear costs) in ncl_last_error */
int ncl_matpower_parse(const char* text, ncl_network_t* out);
void ncl_network_destroy(ncl_network_t N);
int ncl_network_info_get(ncl_network_t N, ncl_network_info* info);
/* per bus (file order): id, type, Pd, Qd (pu), Vmin, Vmax; any may be NULL */
int ncl_network_buses(ncl_network_t N, int* id, int* type, double* pd, double* qd, double* vmin, double* vmax);
/* branch_admittances: y[8 l .. 8 l + 7] = re/im of y_ff, y_ft, y_tf, y_tt
 * (pi model, tap, phase shift, half charging); NCL_E_INVALID on r = x = 0 */
int ncl_network_branch_admittances(ncl_network_t N, double* y);
int ncl_network_serialize(ncl_network_t N, char* buf, int64_t cap, int64_t* len);
int ncl_network_json(ncl_network_t N, char* buf, int64_t cap, int64_t* len);
/* the corrective SCOPF of the in-service network: K non-islanding outages
 * (or the listed ids, as ncl_scopf_create_list) */
int ncl_scopf_create_network(ncl_network_t N, int K, const int* branch_ids, ncl_scopf_t* out);

#ifdef __cplusplus
}
#endif
#endif
