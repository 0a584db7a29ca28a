"""Per-kernel roofline table of the per-iteration kernels (north_star: achieved
HBM GB/s for evaluation, assembly and solves; FP64 tensor-pipe utilisation
for the supernodal updates) from ncu --set full reports (tools/gpu_r02a.sh).

  python tools/kernel_table.py gpurun_out/a_prof_<kernel>.ncu-rep ... > profiles/r02_kernels.md

For each launch: duration, DRAM bytes (read + write) and their rate against
MEASURED_PEAKS.json hbm_gbs, and for DMMA kernels the tensor (DMMA) pipe
utilisation. Algorithmic bytes per launch are given where the
kernel has a closed form at 500x256 (sizes from bench.py's config line).
"""
import csv
import re
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# 500x256 paper-layout sizes (bench config / tools output)
N, M, NNZH, NNZJ, NNZK, NNZL = 957100, 1263335, 1668284, 4662337, 5305003, 10330784
ALG = {
    # K2: read H, J, D, sigma_x; write K; + the 12 B/slot map
    "kkt_assemble_kernel": 8 * (NNZH + NNZJ + N + M) + 12 * NNZK,
    # compact form: the same values in/out; its maps (slot, term start, term
    # J position + byte offset) are counted at the per-slot form's 12 B/slot
    "kkt_assemble_compact": 8 * (NNZH + NNZJ + N + M) + 12 * NNZK,
}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def rows_of(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, unit = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, unit))

        def num(k, scale_units=True):
            v = d.get(k)
            if v in (None, ""):
                return None
            v = float(v.replace(",", ""))
            un = u.get(k, "")
            if scale_units:
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
                      "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(un, 1)
            return v
        name = d.get("Kernel Name", "?").replace("(anonymous namespace)::", "")
        name = re.sub(r"^.*::", "", name.split("(")[0].replace("void ", "").strip())
        res.append({"kernel": name, "us": num("gpu__time_duration.sum"),
                    "dram": (num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0),
                    "dmma": num("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", False),
                    "fp64": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", False),
                    "dram_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", False)})
    return res


def main(paths):
    pk, src = peak()
    print(f"# Per-kernel roofline evidence (ncu --set full, one capture per kernel, cold cache)\n")
    print(f"HBM peak {pk:.1f} GB/s ({src}, MEASURED_PEAKS.json). DRAM bytes = dram__bytes_read.sum + "
          "dram__bytes_write.sum of the launch. Algorithmic bytes per DESIGN.md §3 where the kernel has a "
          "closed form at 500x256.\n")
    print("K4 solves: a forward (or backward) sweep is two launches (`<32>` warp part, `<256>` CTA part); "
          f"together they read L once: (24 nnzL + 32 N) / 2 = {(24 * NNZL + 32 * N) / 2e6:.1f} MB per sweep.\n")
    print("| kernel | report | us | DRAM MB | DRAM GB/s | frac of HBM | algorithmic MB | alg GB/s | DMMA pipe % | FP64 pipe % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        for r in rows_of(p):
            base = r["kernel"].split("<")[0]
            alg = ALG.get(base)
            gbs = r["dram"] / (r["us"] * 1e-6) / 1e9 if r["us"] else 0
            ag = f"{alg / 1e6:.1f}" if alg else "-"
            agbs = f"{alg / (r['us'] * 1e-6) / 1e9:.0f}" if alg and r["us"] else "-"
            print(f"| `{r['kernel']}` | {os.path.basename(p)} | {r['us']:.1f} | {r['dram'] / 1e6:.1f} | {gbs:.0f} | "
                  f"{gbs / pk:.3f} | {ag} | {agbs} | "
                  f"{'-' if r['dmma'] is None else f'{r[chr(100)+chr(109)+chr(109)+chr(97)]:.1f}'} | "
                  f"{'-' if r['fp64'] is None else f'{r[chr(102)+chr(112)+chr(54)+chr(52)]:.1f}'} |")


if __name__ == "__main__":
    main(sys.argv[1:])
