"""Parity record at a full-size configuration: the B200 NCL solve's trace
against the reference (oracle/_ref) trace, next to the SAME reference built
with FMA contraction (oracle/_ref_fma) against itself — how far two equally
valid builds of the reference drift apart under ulp-level rounding changes.

  python tools/parity_record.py GPU.json REF.json REF_FMA.json OUT.json
"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from tools.trace_diff import diff  # noqa: E402

gpu, ref, fma, out = sys.argv[1:5]
a = diff(gpu, ref)
b = diff(fma, ref)


def brief(d):
    x = d["first_discrete_divergence"]
    return {"first_above": {k: [v["iter"], v["max_rel"], v["field"]] for k, v in d["first_above"].items()},
            "first_discrete_divergence": None if x is None else
            {"iter": x["iter"], "fields": x["fields"], "max_rel_before": x["max_rel_before"]},
            "max_rel_at_iter": {str(i): r for i, r, _ in d["max_rel_by_iter"]
                                if i in (1, 2, 5, 10, 20, 30, 50, 80, 100, 120, 130)}}


rec = {"what": "NCL/IPM iterate traces at full size: B200 vs reference, and reference-with-FMA vs reference "
               "(same unmodified reference sources, -ffp-contract=fast -march=x86-64-v3)",
       "runs": {"b200": a["a_summary"], "reference": a["b_summary"], "reference_fma": b["a_summary"]},
       "b200_vs_reference": brief(a), "reference_fma_vs_reference": brief(b)}
json.dump(rec, open(out, "w"), indent=1)
print(json.dumps(rec, indent=1))
