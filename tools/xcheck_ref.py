"""Cross-check the float64 C port (oracle/) against the UNMODIFIED Python
reference at volume (VERDICT r1 "next" 1a; SURVEY §8(c) last row: the CPU
restatement must match the reference on >= 10^4 frames per config before
it stands in for it).

Build container only (imports /root/reference/pkg/src).  For every frame k
of SNR point q it does exactly what the reference harness does
(harness.py:103-108): g = frame_rng(777, q, k), message, polar transform,
BPSK/AWGN, float64 LLR, then ``decode(spec, alpha, cfg, g)`` — the
reference's own permutation stream.  A deep copy of g taken before the
decode is replayed through ``top_decoders._attempt_maps`` (the product's
reference-stream replay of automorphism.py:144-161, pinned by
tests/golden/sampler_stream.npz) into the raw permutation table the port
consumes, so both sides decode identical float64 LLRs under identical maps.

Compared per frame: codeword (bit-exact), pm (bit-exact float64).  On every
8th frame the reference is additionally run attempt by attempt
(``p_fht_fscl`` with a replay sampler, as ensemble_decode does,
top_decoders.py:190-202) so that every attempt's pm and codeword and the
selected attempt are compared too.  The reference's frame-error and
ML-lower-bound counts (harness.py:79-84,109-112) are recorded as well: they
are the unmodified reference's FER on its own harness stream.

Usage: python tools/xcheck_ref.py [--frames 10000] [--only NAME] [--workers 8]
Writes profiles/r2_xcheck_port_vs_reference.json (merged per config).
"""

from __future__ import annotations

import argparse
import copy
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = os.environ.get("RMFHT_REFERENCE", "/root/reference/pkg/src")
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from rmworkbench import rm_core as ref_core  # noqa: E402
from rmworkbench.automorphism import AffinePermutation  # noqa: E402
from rmworkbench.channel_model import ChannelConfig, frame_rng, llr, transmit  # noqa: E402
from rmworkbench.harness import ml_lower_bound  # noqa: E402
from rmworkbench.top_decoders import DecoderConfig, decode, p_fht_fscl  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2108_12550_b200 import automorphism as host_aut  # noqa: E402
from paper_2108_12550_b200.plan import map_sizes  # noqa: E402
from paper_2108_12550_b200.top_decoders import _attempt_maps  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "r2_xcheck_port_vs_reference.json")

# name: (r, m, algorithm, L, M, ebn0 points) — BASELINE.json configs, plus the
# reference's golden-FER family (pkg/data/golden_fer.csv: RM(2,6) L4)
CONFIGS = {
    "rm25_fhtfsc": (2, 5, "FHT-FSC", 1, 1, (3.0,)),
    "rm27_L2_M4": (2, 7, "p-FHT-FSCL", 2, 4, (2.0, 3.0, 4.0)),
    "rm29_L4_M20": (2, 9, "p-FHT-FSCL", 4, 20, (2.5, 3.0, 3.5)),
    "rm37_L8_M32": (3, 7, "p-FHT-FSCL", 8, 32, (4.0,)),
    "rm29_L1_M512": (2, 9, "p-FHT-FSCL", 1, 512, (3.0,)),
    "rm26_fhtfscl_L4": (2, 6, "FHT-FSCL", 4, 1, (2.0, 2.5)),
    "rm26_pfhtfscl_L4_M1": (2, 6, "p-FHT-FSCL", 4, 1, (2.0, 2.5)),
}
SEED = 777
CHUNK = 125


def _replay_table(spec, L, M, g):
    """The raw table [M, S, m+1] that decode(spec, alpha, cfg, g) consumes."""
    maps = []
    if M > 1:
        seeds = g.integers(0, 2 ** 63 - 1, size=M, dtype=np.int64)  # top_decoders.py:196
        for a in range(M):
            maps += _attempt_maps(spec, L, np.random.default_rng(int(seeds[a])), None)
    else:
        maps += _attempt_maps(spec, L, g, None)
    S = len(map_sizes(spec.r, spec.m, L, True))
    return host_aut.maps_to_raw(maps, spec.m).reshape(M, S, spec.m + 1), maps


def _chunk(args):
    name, q, k0, n = args
    r, m, algo, L, M, pts = CONFIGS[name]
    spec = ref_core.build_code(r, m)
    cfg = DecoderConfig(algo, L=L, M=M)
    chan = ChannelConfig.for_rate(pts[q], spec.rate, SEED)
    perms = algo == "p-FHT-FSCL"
    N = spec.N
    S = len(map_sizes(r, m, L, True)) if perms else 0
    llrs = np.zeros((n, N))
    xs = np.zeros((n, N), dtype=np.uint8)
    raw = np.zeros((n, M, S, m + 1), dtype=np.uint16) if perms else None
    ref_cw = np.zeros((n, N), dtype=np.uint8)
    ref_pm = np.zeros(n)
    ref_err = ref_ml = 0
    att_checks = []
    for i in range(n):
        k = k0 + i
        g = frame_rng(SEED, q, k)
        u = ref_core.random_message(spec, g)
        x = ref_core.polar_transform(u)
        alpha = llr(transmit(x, chan, g), chan)
        g2 = copy.deepcopy(g)
        res = decode(spec, alpha, cfg, g)
        llrs[i], xs[i], ref_cw[i], ref_pm[i] = alpha, x, res.codeword, res.pm
        if not np.array_equal(res.codeword, x):
            ref_err += 1
            ref_ml += int(ml_lower_bound(alpha, x, res.codeword))
        if perms:
            raw[i], maps = _replay_table(spec, L, M, g2)
            if M > 1 and k % 8 == 0:
                # per attempt, as ensemble_decode runs them (top_decoders.py:197-201)
                pms, cws = [], []
                for a in range(M):
                    it = iter([AffinePermutation(p.a, p.b) for p in maps[a * S:(a + 1) * S]])
                    ra = p_fht_fscl(spec, alpha, L, None, sampler=lambda it=it: next(it))
                    pms.append(ra.pm)
                    cws.append(ra.codeword)
                att_checks.append((i, np.array(pms), np.array(cws)))
    o = oracle.decode(r, m, 1 if algo == "FHT-FSC" else L, M, llrs, raw, perms=perms, dtype=np.float64,
                      want_attempts=True)
    port_err = int(np.sum(np.any(o["cw"] != xs, axis=1)))
    cw_diff = np.flatnonzero(np.any(o["cw"] != ref_cw, axis=1))
    pm_diff = np.flatnonzero(o["pm"] != ref_pm)
    rel = np.abs(o["pm"] - ref_pm) / np.maximum(np.abs(ref_pm), 1e-300)
    att_frames = att_ok_pm = att_ok_cw = att_ok_sel = 0
    for i, pms, cws in att_checks:
        att_frames += 1
        att_ok_pm += int(np.array_equal(o["att_pm"][i], pms))
        att_ok_cw += int(np.array_equal(o["att_cw"][i], cws))
        best = 0
        for a in range(1, M):
            if pms[a] < pms[best]:
                best = a
        att_ok_sel += int(o["attempt"][i] == best)
    return dict(frames=n, cw_mismatch=[int(k0 + j) for j in cw_diff], pm_mismatch=[int(k0 + j) for j in pm_diff],
                pm_max_rel=float(rel.max()) if n else 0.0, ref_errors=ref_err, ref_ml=ref_ml, port_errors=port_err,
                att_frames=att_frames, att_pm_equal=att_ok_pm, att_cw_equal=att_ok_cw, att_sel_equal=att_ok_sel)


def run(name, frames, workers):
    r, m, algo, L, M, pts = CONFIGS[name]
    res = dict(r=r, m=m, algorithm=algo, L=L, M=M, seed=SEED, points=[])
    for q, eb in enumerate(pts):
        t0 = time.time()
        tasks = [(name, q, k0, min(CHUNK, frames - k0)) for k0 in range(0, frames, CHUNK)]
        with Pool(workers) as pool:
            parts = pool.map(_chunk, tasks, chunksize=1)
        agg = dict(ebn0=eb, q=q, frames=0, cw_mismatch=[], pm_mismatch=[], pm_max_rel=0.0, ref_errors=0, ref_ml=0,
                   port_errors=0, att_frames=0, att_pm_equal=0, att_cw_equal=0, att_sel_equal=0)
        for p in parts:
            for key in ("frames", "ref_errors", "ref_ml", "port_errors", "att_frames", "att_pm_equal",
                        "att_cw_equal", "att_sel_equal"):
                agg[key] += p[key]
            agg["cw_mismatch"] += p["cw_mismatch"]
            agg["pm_mismatch"] += p["pm_mismatch"]
            agg["pm_max_rel"] = max(agg["pm_max_rel"], p["pm_max_rel"])
        agg["wall_s"] = round(time.time() - t0, 1)
        agg["bit_exact"] = not agg["cw_mismatch"] and not agg["pm_mismatch"] and \
            agg["att_pm_equal"] == agg["att_frames"] and agg["att_cw_equal"] == agg["att_frames"] and \
            agg["att_sel_equal"] == agg["att_frames"]
        res["points"].append(agg)
        print(name, eb, {k: (len(v) if isinstance(v, list) else v) for k, v in agg.items()}, flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=10000)
    ap.add_argument("--only", default=None)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out.setdefault("_about", "f64 C port (oracle/) vs the unmodified Python reference on the reference's own "
                   "harness stream (frame_rng(777, q, k), its own permutation draws replayed into the port); "
                   "tools/xcheck_ref.py")
    for name in CONFIGS:
        if args.only and name not in args.only.split(","):
            continue
        out[name] = run(name, args.frames, args.workers)
        out[name]["frames_per_point"] = args.frames
        with open(OUT, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
