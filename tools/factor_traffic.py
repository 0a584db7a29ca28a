"""Sum ncu per-launch DRAM bytes and durations of the kernels of ONE
refactorization (the bench's dominant step) from a --metrics csv, and write
profiles/factor_traffic_<grid>x<K>.json (read by bench.py for roofline.traffic
of that configuration only).

usage: python tools/factor_traffic.py gpurun_out/traffic.csv activsg500x256
"""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (int(d["ID"]), re.sub(r"\(.*", "", d["Kernel Name"]).replace("nclb::", "").replace("<unnamed>::", ""))
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
    per.setdefault(key, {})[d["Metric Name"]] = v * scale
# one refactorization = the launches from a maxdiag_kernel up to (excluding) the next one, take the last complete
ids = list(per.keys())
starts = [i for i, k in enumerate(ids) if "maxdiag" in k[1]]
seg = ids[starts[-2]:starts[-1]] if len(starts) >= 2 else ids
# the factorization only: maxdiag .. inertia (drop the solve and the L2 flush)
end = max(i for i, k in enumerate(seg) if "inertia" in k[1])
seg = seg[:end + 1]
tot_b = sum(per[k].get("dram__bytes_read.sum", 0) + per[k].get("dram__bytes_write.sum", 0) for k in seg)
tot_t = sum(per[k].get("gpu__time_duration.sum", 0) for k in seg)
by = collections.defaultdict(lambda: [0.0, 0.0, 0])
for k in seg:
    b = per[k].get("dram__bytes_read.sum", 0) + per[k].get("dram__bytes_write.sum", 0)
    by[k[1]][0] += b
    by[k[1]][1] += per[k].get("gpu__time_duration.sum", 0)
    by[k[1]][2] += 1
out = {"bytes_per_launch": tot_b, "seconds_serialised": tot_t, "launches": len(seg),
       "what": "dram__bytes_read.sum + dram__bytes_write.sum over every kernel of one refactorization "
               "(maxdiag .. inertia, solve excluded), ncu --metrics, serialised / cold-cache",
       "by_kernel": {k: {"bytes": v[0], "seconds": v[1], "launches": v[2]} for k, v in by.items()}}
cfg = sys.argv[2] if len(sys.argv) > 2 else "activsg500x256"
out["config"] = cfg
json.dump(out, open(f"profiles/factor_traffic_{cfg}.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in ("bytes_per_launch", "seconds_serialised", "launches")}))
