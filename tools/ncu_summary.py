"""Summarise ncu outputs for profiles/ (run here, on the CPU side).

  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
  python tools/ncu_summary.py report gpurun_out/prof_factor.ncu-rep > profiles/rNN_factor_full.md
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct"]


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("nclb::", "").replace("<unnamed>::", "").replace("void ", "")
    return name.strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "ns":
            v /= 1e3
        elif d["Metric Unit"] == "ms":
            v *= 1e3
        k = short(d["Kernel Name"])
        per.setdefault(k, []).append(v)
        order.append((k, v))
    tot = sum(sum(v) for v in per.values())
    print(f"# ncu launch list ({len(order)} launches, {tot:.1f} us total, cold-cache / serialised)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print("empty report")
        return
    hdr, unit = rows[0], rows[1]
    print(f"# ncu --set full: {path}\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## `{short(name)}`\n")
        print("| metric | unit | value |")
        print("|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {unit[i]} | {r[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
