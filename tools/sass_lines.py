"""Join an ncu SASS source page with nvdisasm line info: stall samples and instruction counts
per CUDA source line, plus the dynamic opcode mix.
    python tools/sass_lines.py <prof.ncu-rep> <kernel-mangled-name> <warp-units> [topN]"""
import collections, csv, io, re, subprocess, sys, os
rep, fn, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.environ.get("ER_LIB", os.path.join(ROOT, "paper_2605_13766_b200", "lib", "libelasticarod.so"))
tmp = "/tmp/_cubins"
os.makedirs(tmp, exist_ok=True)
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith(os.environ.get("CUBIN", "er_kernels")) and f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
i0 = [i for i, l in enumerate(dis) if l.startswith(fn + ":")][0]
seq, cur, curf = [], None, None
for l in dis[i0 + 1:]:
    if l.startswith(".section") or (l.startswith("_Z") and l.endswith(":")):
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', l)
    if m:
        curf, cur = os.path.basename(m.group(1)), int(m.group(2))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        seq.append((curf, cur))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
si, ie, ss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > ie]
assert len(body) == len(seq), (len(body), len(seq))
files = {}
for f in ("er_kernels.cu", "er_math.cuh", "er_warp.cu", "er_tma.cuh"):
    files[f] = open(os.path.join(ROOT, "paper_2605_13766_b200", "csrc", f)).read().split("\n")
agg, inst, ops = collections.Counter(), collections.Counter(), collections.Counter()
tots = sum(int(r[ss] or 0) for r in body)
tot = sum(int(r[ie] or 0) for r in body)
for (f, ln), r in zip(seq, body):
    agg[(f, ln)] += int(r[ss] or 0)
    inst[(f, ln)] += int(r[ie] or 0)
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9]+)", r[si].strip())
    if m:
        ops[m.group(2)] += int(r[ie] or 0)
print(f"instructions per unit: {tot / units:.1f}")
print("opcode mix per unit:", ", ".join(f"{o} {n / units:.1f}" for o, n in ops.most_common(24)))
for (f, ln), sv in agg.most_common(top):
    src = files.get(f, [""] * 10000)[ln - 1].strip() if ln else ""
    print(f"{100 * sv / tots:5.1f}%  {inst[(f, ln)] / units:6.1f}/u  {f}:{ln}: {src[:85]}")
