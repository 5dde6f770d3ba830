"""Summarise ncu outputs into profiles/ (launch shares + top-kernel metrics + dynamic SASS mix).

    python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <out_dir> [--key cfg3_spl1]
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.per_cycle_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__grid_size",
    "launch__block_size", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[re.sub(r"\(.*", "", r[ki])[:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "total_ms": sum(v) / 1e6, "share": sum(v) / tot,
                    "avg_us": sum(v) / len(v) / 1e3})
    return out


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                d[m] = v[h.index(m)] + " " + u[h.index(m)]
        stalls = {}
        for i, x in enumerate(h):
            if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio"):
                try:
                    val = float(v[i])
                except ValueError:
                    continue
                if val > 0.05:
                    stalls[x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = val
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(d)
    return res


def sass_mix(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    ops = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9]+)", r[si].strip())
        if m and r[ie]:
            ops[m.group(2)] += int(r[ie])
    return ops


def main():
    lp, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
    key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
    os.makedirs(out, exist_ok=True)
    L = launches(lp)
    R = raw(rep)
    ops = sass_mix(rep)
    with open(os.path.join(out, "launches_summary.json"), "w") as f:
        json.dump(L, f, indent=1)
    with open(os.path.join(out, "top_kernel_metrics.json"), "w") as f:
        json.dump(R, f, indent=1)
    warps = None
    for r in R:
        g = float(r["launch__grid_size"].split()[0]); b = float(r["launch__block_size"].split()[0])
        warps = g * b / 32
    tot = sum(ops.values())
    mix = {op: {"per_warp": n / warps, "share": n / tot} for op, n in ops.most_common(40)}
    with open(os.path.join(out, "sass_dynamic_mix.json"), "w") as f:
        json.dump({"instructions_per_warp": tot / warps, "ops": mix}, f, indent=1)
    if key and R:
        r = R[0]
        rd = float(r["dram__bytes_read.sum"].split()[0]); wr = float(r["dram__bytes_write.sum"].split()[0])
        unit = r["dram__bytes_read.sum"].split()[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        tp = os.path.join(os.path.dirname(out.rstrip("/")), "traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        tj[key] = {"dram_bytes_per_launch": (rd + wr) * scale, "source": os.path.join(out, "top_kernel_metrics.json")}
        json.dump(tj, open(tp, "w"), indent=1)
    print(json.dumps(L[:5], indent=1))
    print(json.dumps(R, indent=1)[:3000])
    print("instructions/warp", tot / warps)


if __name__ == "__main__":
    main()
