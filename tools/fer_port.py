"""Reference FER counts at the BASELINE.json Eb/N0 points from the float64
C port (oracle/, cross-checked bit-exact against the unmodified Python
reference on 10^4 frames per config: profiles/r2_xcheck_port_vs_reference.json),
decoding the reference's own harness stream (harness.py:103-107:
frame_rng(777, q, k), float64 LLRs) under the product's counter-based
permutation table (uniform GL(m,2) x F2^m like the reference sampler,
decoder 0's root maps = identity; seed fixed per point).  Frame errors and
the ML lower bound are counted as harness.py:79-84,109-112 does.

VERDICT r1 "next" 2: the GPU test (tests/test_gpu_fer_points.py) decodes
the same frames (rounded to float32) under the same table and must land in
the 95% Clopper-Pearson interval of these counts; the error frame indices
are stored so the two error sets can be compared frame by frame.

Also pins the reference's own golden FER file (pkg/data/golden_fer.csv:1-5,
RM(2,6) L=4, 30,000 frames per point): FHT-FSCL needs no permutations, and
p-FHT-FSCL with M = 1 draws its maps from the frame's generator after the
channel draws, which top_decoders._attempt_maps replays — so the port must
reproduce those rows exactly.

Usage: python tools/fer_port.py [--only NAME] [--scale 1.0]
Writes tests/golden/fer_points.json (merged per config).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "fer_points.json")

# name: (r, m, L, M, algorithm, points, frames per point, table)
#   table: "counter" (product sampler, seed per point) or "reference" (the
#   frame generator's own draws replayed: p-FHT-FSCL, M = 1) or None
JOBS = {
    "rm29_L4_M20": (2, 9, 4, 20, "p-FHT-FSCL", (2.5, 3.0, 3.5), 1000000, "counter"),
    "rm27_L2_M4": (2, 7, 2, 4, "p-FHT-FSCL", (2.0, 3.0, 4.0), 1000000, "counter"),
    "rm37_L8_M32": (3, 7, 8, 32, "p-FHT-FSCL", (4.0,), 1000000, "counter"),
    "rm29_L1_M512": (2, 9, 1, 512, "p-FHT-FSCL", (3.0,), 100000, "counter"),
    "rm25_fhtfsc": (2, 5, 1, 1, "FHT-FSC", (3.0,), 100000, None),
    "golden_rm26_fhtfscl_L4": (2, 6, 4, 1, "FHT-FSCL", (2.0, 2.5), 30000, None),
    "golden_rm26_pfhtfscl_L4": (2, 6, 4, 1, "p-FHT-FSCL", (2.0, 2.5), 30000, "reference"),
}
SEED = 777
CHUNK = 4000


def table_seed(name, q):
    """Counter-sampler seed of point q (the GPU test uses the same)."""
    return 0x5EED0000 + 131 * q + sum(map(ord, name))


def _chunk(a):
    name, q, k0, n, threads = a
    from oracle import oracle
    from paper_2108_12550_b200.automorphism import maps_to_raw
    from paper_2108_12550_b200.channel_model import harness_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    from paper_2108_12550_b200.top_decoders import _attempt_maps
    r, m, L, M, algo, pts, _, table = JOBS[name]
    spec = build_code(r, m)
    x, llr, rngs = harness_frames(spec, pts[q], SEED, q, k0, n)
    perms = algo == "p-FHT-FSCL"
    raw = None
    if table == "counter":
        raw, _ = Plan(r, m, L, M, True, "f32").sample(n, table_seed(name, q), frame0=k0, identity_root=True,
                                                       want_records=False)
    elif table == "reference":
        raw = np.stack([maps_to_raw(_attempt_maps(spec, L, g, None), m) for g in rngs])[:, None]
    o = oracle.decode(r, m, L, M, llr, raw, perms=perms, dtype=np.float64, nthreads=threads, want_attempts=False)
    wrong = np.flatnonzero(np.any(o["cw"] != x, axis=1))
    ml = 0
    for i in wrong:  # harness.ml_lower_bound: corr(x_hat) >= corr(x)
        c_hat = np.sum((1.0 - 2.0 * o["cw"][i]) * llr[i])
        c_tx = np.sum((1.0 - 2.0 * x[i]) * llr[i])
        ml += int(c_hat >= c_tx)
    return [int(k0 + i) for i in wrong], ml


def clopper_pearson(k, n, alpha=0.05):
    from scipy.stats import beta
    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the frame counts (smoke runs)")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["_about"] = ("reference FER counts: float64 C port of the reference (oracle/) on the reference harness "
                     "stream frame_rng(777, q, k); tables from the counter sampler with table_seed(name, q) "
                     "(tools/fer_port.py), or the reference's own draws replayed (golden rows)")
    for name, (r, m, L, M, algo, pts, frames, table) in JOBS.items():
        if args.only and name not in args.only.split(","):
            continue
        F = max(1, int(frames * args.scale))
        rec = dict(r=r, m=m, L=L, M=M, algorithm=algo, table=table, seed=SEED, points=[])
        for q, eb in enumerate(pts):
            t0 = time.time()
            # many processes x 1 thread: frame generation is Python, decode is C
            tasks = [(name, q, k0, min(CHUNK, F - k0), 1) for k0 in range(0, F, CHUNK)]
            with Pool(args.workers) as pool:
                parts = pool.map(_chunk, tasks, chunksize=1)
            errs = sorted(i for p in parts for i in p[0])
            ml = sum(p[1] for p in parts)
            lo, hi = clopper_pearson(len(errs), F)
            pt = dict(ebn0=eb, q=q, frames=F, errors=len(errs), ml_errors=ml, fer=len(errs) / F,
                      ci95=[lo, hi], table_seed=table_seed(name, q) if table == "counter" else None,
                      error_frames=errs, wall_s=round(time.time() - t0, 1))
            rec["points"].append(pt)
            print(name, eb, {k: v for k, v in pt.items() if k != "error_frames"}, flush=True)
        out[name] = rec
        with open(OUT, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
