"""Per decoding-tree node instruction budget of decode_kernel2: joins ncu's
SASS page (instructions executed per PC) with the full inline call-site
chain of every SASS instruction (nvdisasm -gi) and walks the chain through
the node recursion (root_node / node2 left and right calls, fht_node /
spc_node leaves), so that each instruction is charged to one tree node.
usage: ncu_nodes.py REPORT OBJ KERNEL_SUBSTR ITEMS [MM]"""
import collections, csv, os, re, subprocess, sys

sys.path.insert(0, os.path.dirname(__file__))
from sassmap import cubin_of, func_of, source  # noqa: E402

SRC = "rmfht_fast.cuh"


def call_lines():
    """line numbers of the recursion's call sites in rmfht_fast.cuh"""
    roles = {}
    for i, t in enumerate(source(SRC), 1):
        s = t.strip()
        if "node2<R, MM, L, RR - 1, SS - 1, SPINE>(cx, xl, l1)" in s or "node2<R, MM, L, R - 1, MM - 1, true>(cx, xl, l1)" in s:
            roles[i] = "L"
        elif "node2<R, MM, L, RR, SS - 1, false>(cx, xr, l2)" in s or "node2<R, MM, L, R, MM - 1, false>(cx, xr, l2)" in s:
            roles[i] = "R"
        elif "bits = node2<R, MM, L, R, MM, true>(cx, x, rlin)" in s:
            roles[i] = "root"
        elif s.startswith("bits = root_node("):
            roles[i] = "root"
        elif s.startswith("return fht_node<"):
            roles[i] = "FHT"
        elif s.startswith("return spc_node<"):
            roles[i] = "SPC"
        elif "perm_ext_root2(cx);" in s:
            roles[i] = "permext"
        elif "perm_ext_inner2<R, MM, L, SS>(cx, x)" in s:
            roles[i] = "permext_inner"
    return roles


def chains(obj, ksub):
    """{addr: [call-site (file, line) outermost first]}"""
    dis = subprocess.run(["nvdisasm", "-gi", cubin_of(obj)], capture_output=True, text=True).stdout
    out, fn, pend, fresh = {}, None, [], True
    cur, own, nown = [], None, None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            if fresh:
                pend = []
                nown = (os.path.basename(m.group(1)), int(m.group(2)))
            fresh = False
            if m.group(3):
                pend.append((os.path.basename(m.group(3)), int(m.group(4))))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", ln)
        if m:
            if not fresh:
                cur = list(reversed(pend))  # innermost-first listing -> outermost first
                own = nown
            fresh = True
            if fn and ksub in fn and "$" not in fn:  # the kernel's own section
                out[int(m.group(1), 16)] = (cur, own)
    return out


def label(co, roles, mm):
    chain, own = co
    if not chain:  # the kernel body itself, or an out-of-line (cold) helper
        fn = func_of(*own) if own else "?"
        return "cold: " + fn.split(":")[-1].split("@")[0] if ("fht_exact" in fn or "fht_fallback" in fn) else "item loop"
    path, n, leaf = [], mm, None
    for f, l in chain:
        if f != SRC:
            continue
        r = roles.get(l)
        if r == "root":
            path = ["root"]
        elif r in ("L", "R"):
            path.append(r)
            n -= 1
        elif r in ("FHT", "SPC"):
            leaf = r
        elif r in ("permext", "permext_inner"):
            leaf = r
    if not path:
        return "item prologue/epilogue" if leaf != "permext" else "root perm-ext"
    nm = "/".join(path) + f" n={1 << n}"
    return nm + (f" {leaf}" if leaf else " glue")


def main():
    rep, obj, ksub, items = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    mm = int(sys.argv[5]) if len(sys.argv) > 5 else 9
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
    iW = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    execs = [(int(r[iA], 16), int(float(r[iE] or 0)), int(float(r[iW] or 0)) if iW is not None else 0, r[iS])
             for r in rows[2:] if len(r) > iE and r[iA].startswith("0x")]
    base = execs[0][0]
    ch = chains(obj, ksub)
    roles = call_lines()
    cnt, wav = collections.Counter(), collections.Counter()
    cls = collections.defaultdict(collections.Counter)
    for a, n, w, sass in execs:
        c = ch.get(a - base)
        key = label(c, roles, mm) if c is not None else "unmapped"
        cnt[key] += n
        wav[key] += w
        cls[key][opclass(sass)] += n
    tot = sum(cnt.values())
    print(f"warp instructions per item: {tot / items:.0f}; shared wavefronts per item: {sum(wav.values()) / items:.0f}")
    print("classes: fp = FADD/FADD2/FFMA/FFMA2/FMUL/FMUL2/FMNMX/FMNMX3 (the ledger's additions and comparisons; a "
          "packed instruction counts once), fpsel = FSETP/FSEL (candidate tests and selects), mio = LDS/STS/SHFL/"
          "LDGSTS/LDG/STG/ATOM, ctl = everything else (integer, logic, moves, predicates, branches, votes)")
    print("ledger: the reference ledger's operations of the node (n log2 n per FHT, n/2 per f and g, per path; "
          "LM of the 2L root trials) / 32 lanes = the instructions an ideal scalar-per-lane kernel would issue")
    print(f"{'node':34s} {'instr/item':>10s} {'share':>6s} {'fp':>6s} {'fpsel':>6s} {'mio':>6s} {'ctl':>6s} {'wavefr':>7s} {'ledger':>7s}")
    for k in sorted(cnt, key=lambda k: (-cnt[k])):
        c = cls[k]
        led = ledger_floor(k, mm)
        print(f"{k:34s} {cnt[k] / items:10.1f} {100 * cnt[k] / tot:5.1f}% {c['fp'] / items:6.0f} {c['fpsel'] / items:6.0f} "
              f"{c['mio'] / items:6.0f} {c['ctl'] / items:6.0f} {wav[k] / items:7.1f} {led if led is not None else '':>7}")
    c = collections.Counter()
    for k in cls:
        c.update(cls[k])
    print(f"{'total':34s} {tot / items:10.1f} {'':6s} {c['fp'] / items:6.0f} {c['fpsel'] / items:6.0f} {c['mio'] / items:6.0f} "
          f"{c['ctl'] / items:6.0f} {sum(wav.values()) / items:7.1f}")


FP = ("FADD", "FFMA", "FMUL", "FMNMX")
MIO = ("LDS", "STS", "SHFL", "LDGSTS", "LDG", "STG", "ATOM", "RED", "LDL", "STL", "LD.", "ST.")


def opclass(sass):
    t = sass.split()
    if not t:
        return "ctl"
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    if op.startswith(FP):
        return "fp"
    if op.startswith(("FSETP", "FSEL", "FSET")):
        return "fpsel"
    if op.startswith(MIO):
        return "mio"
    return "ctl"


def ledger_floor(name, mm, L=4):
    """the reference ledger's operation count of a tree node (accounting.py:136-152: n log2 n per
    FHT, n/2 per f and per g, per path) in warp instructions (/ 32)"""
    m = re.search(r"n=(\d+)", name)
    if name == "root perm-ext":
        n = 1 << mm
        return round(2 * L * n / 32)  # 2L trials x (n/2 minima + n/2 additions)
    if not m:
        return None
    n = int(m.group(1))
    if name.endswith("FHT"):
        return round(L * n * (n.bit_length() - 1) / 32)
    if name.endswith("glue"):
        return round(L * n / 32)  # f and g: n/2 each
    if name.endswith("SPC"):
        return round(L * 2 * n / 32)
    return None


if __name__ == "__main__":
    main()


def lines_of(rep, obj, ksub, items, mm, want, top=40):
    """top source lines (innermost frame) of the instructions charged to node `want`"""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
    execs = [(int(r[iA], 16), int(float(r[iE] or 0)), r[iS].strip()) for r in rows[2:] if len(r) > iE and r[iA].startswith("0x")]
    base = execs[0][0]
    ch, roles = chains(obj, ksub), call_lines()
    cnt, ops = collections.Counter(), collections.Counter()
    for a, n, sass in execs:
        c = ch.get(a - base)
        if c is None or label(c, roles, mm) != want:
            continue
        chain, own = c
        key = (own, chain[-1][1] if chain else 0)
        cnt[key] += n
        t = sass.split()
        if t:
            ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += n
    print("opcodes:", {k: round(v / items) for k, v in ops.most_common(16)})
    for (own, site), n in cnt.most_common(top):
        src = source(own[0]) if own else []
        txt = src[own[1] - 1].strip()[:90] if own and 0 < own[1] <= len(src) else "?"
        print(f"{n / items:7.1f}  {own[0]}:{own[1]} (via {site})  {txt}")
