"""Per-source-line warp-stall samples and executed instructions of one kernel
from an ncu report (ncu -i R --page source --print-source cuda,sass --csv),
the hottest lines first (profiling helper, not part of the library).

  python tools/ncu_lines.py gpurun_out/X.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samp = collections.Counter()
inst = collections.Counter()
text = {}
fname = "?"
hdr = None
line = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row
        line = (fname, int(r[0]))
        text[line] = r[1]
    if line is None or not r[2]:
        continue
    try:
        samp[line] += float(r[4] or 0)
        inst[line] += float(r[7] or 0)
    except ValueError:
        pass
ts, ti = sum(samp.values()), sum(inst.values())
print(f"samples {ts:.0f}  warp instructions {ti:.0f}")
for k, v in samp.most_common(top):
    print(f"{k[0]}:{k[1]:<5} {100 * v / ts:5.1f}% samp {100 * inst[k] / ti:5.1f}% inst  {text.get(k, '').strip()[:100]}")
