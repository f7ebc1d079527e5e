"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix per work item."""
import csv, collections, subprocess, sys

rep = sys.argv[1]
items = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0


def csv_rows(args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


rows = csv_rows(["--page", "details"])
h = rows[0]
want = {"Duration", "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy",
        "Theoretical Occupancy", "L1/TEX Hit Rate", "Mem Busy", "DRAM Throughput", "Compute (SM) Throughput",
        "Shared Memory Configuration Size", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"}
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:34s} {d['Metric Value']} {d['Metric Unit']}")
raw = csv_rows(["--page", "raw"])
d = dict(zip(raw[0], raw[2]))
st = [(k, v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
tot = sum(float(v) for k, v in st if v.replace(".", "").isdigit()) or 1
print("stall reasons:")
for k, v in sorted(st, key=lambda kv: -float(kv[1]) if kv[1].replace(".", "").isdigit() else 0)[:8]:
    print(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * float(v) / tot:5.1f}%")
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"):
    if k in d:
        print(f"{k:48s} {d[k]}")
src = csv_rows(["--page", "source", "--print-source=sass"])
hh = src[1]
iS, iE = hh.index("Source"), hh.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for r in src[2:]:
    if len(r) <= iE:
        continue
    t = r[iS].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    n = int(r[iE] or 0)
    cnt[op] += n
    tot += n
print(f"instructions per item: {tot / items:.0f}")
print("   " + "  ".join(f"{op}:{n / items:.0f}" for op, n in cnt.most_common(16)))
