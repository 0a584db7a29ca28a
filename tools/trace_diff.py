"""Diff two full-precision NCL/IPM traces (tools/gpu_solve.py --trace,
tools/oracle_solve.py) iteration by iteration: where the continuous iterates
first separate beyond a relative threshold, and the first DISCRETE
divergence (a different line-search count, factorization count, refinement
sweep count or accept/reject), with the relative differences that preceded it.

  python tools/trace_diff.py A.json B.json [OUT.json]
"""
import json
import math
import sys

CONT = ["mu", "inf_pr", "inf_du", "e0", "obj", "theta", "phi", "g", "dw", "dc", "alpha_pr", "alpha_du"]
DISC = ["outer", "ls", "factorizations", "sweeps", "accepted"]


def rel(a, b):
    if a == b:
        return 0.0
    if not (math.isfinite(a) and math.isfinite(b)):
        return math.inf
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def load(p):
    d = json.load(open(p))
    return d, [t for t in d["trace"] if "iter" in t]


def diff(pa, pb):
    da, ta = load(pa)
    db, tb = load(pb)
    rows, first = [], {}
    disc = None
    for i, (a, b) in enumerate(zip(ta, tb)):
        r = {k: rel(float(a[k]), float(b[k])) for k in CONT}
        worst = max(r, key=r.get)
        row = {"iter": a["iter"], "max_rel": r[worst], "field": worst}
        rows.append(row)
        for thr in (1e-14, 1e-12, 1e-10, 1e-8, 1e-6):
            if r[worst] > thr and thr not in first:
                first[thr] = row
        d = [k for k in DISC if a[k] != b[k]]
        if d and disc is None:
            disc = {"iter": a["iter"], "fields": {k: [a[k], b[k]] for k in d},
                    "a": {k: a[k] for k in CONT + DISC}, "b": {k: b[k] for k in CONT + DISC},
                    "max_rel_before": max((x["max_rel"] for x in rows[:-1]), default=0.0),
                    "max_rel_at": row}
            break
    return {"a": pa, "b": pb,
            "a_summary": {k: da["result"].get(k) for k in ("outer_iters", "inner_iters", "factorizations",
                                                          "objective", "r_inf")} | {"variant": da.get("variant")},
            "b_summary": {k: db["result"].get(k) for k in ("outer_iters", "inner_iters", "factorizations",
                                                          "objective", "r_inf")} | {"variant": db.get("variant")},
            "iterations_compared": len(rows),
            "first_above": {f"{k:.0e}": v for k, v in sorted(first.items())},
            "first_discrete_divergence": disc,
            "max_rel_by_iter": [[x["iter"], x["max_rel"], x["field"]] for x in rows]}


if __name__ == "__main__":
    out = diff(sys.argv[1], sys.argv[2])
    s = {k: v for k, v in out.items() if k != "max_rel_by_iter"}
    print(json.dumps(s, indent=1))
    if len(sys.argv) > 3:
        json.dump(out, open(sys.argv[3], "w"), indent=1)
