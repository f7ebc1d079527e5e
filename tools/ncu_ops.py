"""Per source line, dynamic count of one SASS opcode family (e.g. IMAD) per work item.
usage: ncu_ops.py REPORT OBJ KERNEL_SUBSTR ITEMS OPCODE_PREFIX [TOP]"""
import collections, csv, subprocess, sys, os, glob
rep, obj, ksub, items, opx = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5]
top = int(sys.argv[6]) if len(sys.argv) > 6 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iA, iS, iE = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
sys.path.insert(0, os.path.dirname(__file__))
from sassmap import line_map
line_of = line_map(obj, ksub)
execs = [(int(r[iA], 16), r[iS].strip(), int(float(r[iE] or 0))) for r in rows[2:] if len(r) > iE and r[iA].startswith("0x")]
base = execs[0][0]
cnt = collections.Counter(); full = collections.Counter()
for a, src, n in execs:
    t = src.split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    if op.startswith(opx):
        cnt[line_of.get(a - base)] += n
        full[op] += n
print("variants:", {k: round(v / items, 1) for k, v in full.most_common(8)})
srcs = {}
for key, n in cnt.most_common(top):
    if key is None: print(f"{n/items:7.1f} ?"); continue
    f, l = key
    if f not in srcs:
        p = glob.glob("/root/repo/**/" + f, recursive=True)
        srcs[f] = open(p[0]).read().split("\n") if p else []
    print(f"{n/items:7.1f}  {f}:{l}  {srcs[f][l-1].strip()[:90] if srcs[f] else ''}")
