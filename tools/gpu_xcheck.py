"""GPU float32 throughput kernel vs the float64 CPU port at volume, with the
tie accounting of oracle/ties.py (VERDICT r1 "next" 1b).  GPU box only.

For each BASELINE config and Eb/N0 point: frames 0..F-1 of the reference
harness stream (channel_model.harness_frames = frame_rng(777, q, k),
harness.py:103-107), LLRs rounded to float32 and fed to both sides; one
permutation table from the product's counter-based sampler (seed fixed per
point, decoder 0's root maps = identity) fed to both sides.  The port (the
f64 restatement, itself cross-checked bit-exact against the unmodified
Python reference on 10^4 frames per config: profiles/r2_xcheck_port_vs_reference.json)
runs on all host cores.

Usage: python tools/gpu_xcheck.py [--frames 100000] [--only rm29_L4_M20] [--out FILE]
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

# name: (r, m, L, M, permutations, points)
CONFIGS = {
    "rm29_L4_M20": (2, 9, 4, 20, True, (2.5, 3.0, 3.5)),
    "rm27_L2_M4": (2, 7, 2, 4, True, (2.0, 3.0, 4.0)),
    "rm37_L8_M32": (3, 7, 8, 32, True, (4.0,)),
    "rm29_L1_M512": (2, 9, 1, 512, True, (3.0,)),
    "rm25_fhtfsc": (2, 5, 1, 1, False, (3.0,)),
}
SEED = 777


def table_seed(name, q):
    return 0x7AB1E000 + 97 * q + sum(map(ord, name))


def _frames(args):
    r, m, eb, q, k0, n = args
    from paper_2108_12550_b200.channel_model import harness_frames
    from paper_2108_12550_b200.rm_core import build_code
    x, llr, _ = harness_frames(build_code(r, m), eb, SEED, q, k0, n)
    return x, llr.astype(np.float32)


def stream_frames(r, m, eb, q, F, pool, chunk=2000):
    parts = pool.map(_frames, [(r, m, eb, q, k0, min(chunk, F - k0)) for k0 in range(0, F, chunk)])
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def run_point(name, q, F, pool, threads):
    import torch
    from oracle import oracle, ties
    from paper_2108_12550_b200.decoder import Plan
    r, m, L, M, perms, pts = CONFIGS[name]
    eb = pts[q]
    t0 = time.time()
    x, llr = stream_frames(r, m, eb, q, F, pool)
    t_gen = time.time() - t0
    plan = Plan(r, m, L, M, perms, "f32")
    seed = table_seed(name, q)
    parts = []
    t_gpu = t_cpu = 0.0
    G = 32768 if M <= 32 else 2048
    C = max(64, min(4000, 200000 // max(1, M * (1 << m) // 64)))  # port chunk (bounds att_cw memory)
    for g0 in range(0, F, G):
        g1 = min(F, g0 + G)
        raw, rec = plan.sample(g1 - g0, seed, frame0=g0, identity_root=True) if perms else (None, None)
        t = time.time()
        o = plan.decode(llr[g0:g1], records=rec)
        torch.cuda.synchronize()
        t_gpu += time.time() - t
        for c0 in range(g0, g1, C):
            c1 = min(g1, c0 + C)
            t = time.time()
            p = oracle.decode(r, m, L, M, llr[c0:c1].astype(np.float64),
                              raw[c0 - g0:c1 - g0] if perms else None, perms=perms, dtype=np.float64,
                              nthreads=threads, want_attempts=True)
            t_cpu += time.time() - t
            parts.append(ties.classify(o["cw"][c0 - g0:c1 - g0], o["pm"][c0 - g0:c1 - g0],
                                       o["attempt"][c0 - g0:c1 - g0], p, x=x[c0:c1]))
    res = ties.merge(parts)
    res.update(ebn0=eb, q=q, table_seed=seed, ok=ties.ok(res), gen_s=round(t_gen, 1), gpu_s=round(t_gpu, 2),
               port_s=round(t_cpu, 1), port_threads=threads)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=100000)
    ap.add_argument("--only", default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gpu_xcheck.json"))
    args = ap.parse_args()
    threads = os.cpu_count() or 1
    out = {"_about": "GPU float32 throughput kernel vs float64 CPU port (oracle/) on the reference harness "
                     "stream frame_rng(777, q, k) rounded to float32, identical permutation tables; tie "
                     "accounting per oracle/ties.py (tools/gpu_xcheck.py)", "frames_per_point": args.frames}
    with Pool(threads) as pool:
        for name in CONFIGS:
            if args.only and name not in args.only.split(","):
                continue
            pts = CONFIGS[name][5]
            F = args.frames if name != "rm29_L1_M512" else max(1, args.frames // 4) * 4
            out[name] = [run_point(name, q, F, pool, threads) for q in range(len(pts))]
            for p in out[name]:
                print(name, json.dumps(p), flush=True)
            os.makedirs(os.path.dirname(args.out), exist_ok=True)
            with open(args.out, "w") as fh:
                json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
