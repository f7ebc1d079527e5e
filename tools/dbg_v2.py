import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden
from oracle import oracle
from paper_2108_12550_b200.decoder import Plan
for name in sys.argv[1:]:
    g = load_golden(name)
    p = Plan(g["r"], g["m"], g["L"], g["M"], True, "f32")
    o = p.decode(g["llr"], raw_maps=g["raw"], diag=True)
    c = oracle.decode(g["r"], g["m"], g["L"], g["M"], g["llr"], g["raw"], dtype=np.float32, order="v2", nthreads=8)
    cr = oracle.decode(g["r"], g["m"], g["L"], g["M"], g["llr"], g["raw"], dtype=np.float32, order="reference", nthreads=8)
    bad = np.argwhere(o["att_pm"] != c["att_pm"])
    print(name, "kernel", p.kernel, "attempt mismatches", len(bad), "of", o["att_pm"].size)
    for f, a in bad[:8]:
        print(f"  f={f} a={a} gpu={o['att_pm'][f,a]!r} v2={c['att_pm'][f,a]!r} ref32={cr['att_pm'][f,a]!r} ref64={g['att_pm'][f,a]!r} cw_eq={np.array_equal(o['att_cw'][f,a], c['att_cw'][f,a])}")
