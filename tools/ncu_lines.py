"""Dynamic instruction counts per CUDA source line: joins ncu's SASS page
(instructions executed per PC) with nvdisasm line info of the same cubin.
usage: ncu_lines.py REPORT OBJ KERNEL_SUBSTR ITEMS [TOP]"""
import collections, csv, re, subprocess, sys, tempfile, os, glob

rep, obj, ksub, items = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iA, iS, iE = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
metric = os.environ.get("NCU_LINES_METRIC", "exec")  # exec | stall | wave | excess
iX = {"wave": "L1 Wavefronts Shared", "excess": "L1 Wavefronts Shared Excessive"}.get(metric)
iX = h.index(iX) if iX else None
execs = []
for r in rows[2:]:
    if len(r) > iE and r[iA].startswith("0x"):
        col = iE if metric == "exec" else iW if metric == "stall" else iX
        val = int(float(r[col] or 0))
        execs.append((int(r[iA], 16), r[iS].strip(), val))
base = execs[0][0]
sys.path.insert(0, os.path.dirname(__file__))
from sassmap import line_map, func_of
line_of = line_map(obj, ksub)
cnt = collections.Counter()
miss = 0
for addr, src, n in execs:
    key = line_of.get(addr - base)
    if key is None:
        miss += n
        continue
    cnt[key] += n
tot = sum(cnt.values()) + miss
print(f"total per item {tot / items:.0f} (unmapped {miss / items:.0f})")
srcs = {}
for (f, l), n in cnt.most_common(top):
    if f not in srcs:
        p = [q for q in glob.glob("/root/repo/**/" + f, recursive=True)]
        srcs[f] = open(p[0]).read().split("\n") if p else []
    txt = srcs[f][l - 1].strip()[:80] if srcs[f] and l <= len(srcs[f]) else ""
    print(f"{n / items:7.1f}  {f}:{l}  {txt}")

fcnt = collections.Counter()
for (f, l), n in cnt.items():
    fcnt[func_of(f, l)] += n
print("-- by enclosing function")
for nm, n in fcnt.most_common(top):
    print(f"{n / items:7.1f}  {nm}")
