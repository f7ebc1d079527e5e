"""Generate golden parity fixtures by running the UNMODIFIED Python reference.

Runs only in the build container (it imports /root/reference/pkg/src); the
outputs, tests/golden/*.npz, travel with the repo and pin both the CPU
oracle (tests/test_oracle_pins.py) and the CUDA decoder (tests/test_gpu_*).

Each fixture holds identical inputs for both sides — LLRs and one raw
permutation table replayed into the reference through its ``sampler=`` hook
in the reference's consumption order — and the reference's
outputs: per-attempt (codeword, pm), the ensemble pick (first strict
minimum, top_decoders.py:200) and the final (codeword, pm).

Two input modes:
  exact   — integer LLRs (|alpha| <= 31 or <= 1024): every f/g/FHT/LM/PM value
            is an exact float32 number, so fp32 and fp64 must agree bit-for-bit
            and exact ties exercise every stable-sort rule.
  channel — BPSK/AWGN LLRs from the harness stream frame_rng(777, q, k)
            (harness.py:103-107), rounded to float32 and fed to the reference
            as float64.

Usage:  python tools/gen_golden.py [--only NAME]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
import zlib

import numpy as np

REF = os.environ.get("RMFHT_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from rmworkbench import rm_core as ref_core  # noqa: E402
from rmworkbench.automorphism import AffinePermutation, sample_affine_batch  # noqa: E402
from rmworkbench.channel_model import ChannelConfig, frame_rng, llr, transmit  # noqa: E402
from rmworkbench.top_decoders import (aut_ssc, correlation, ensemble_decode,  # noqa: E402
                                      fht_fsc_decode, fht_fscl_decode, p_fht_fscl,
                                      ssc_decode)
from rmworkbench.automorphism import apply_perm, apply_perm_inverse, sample_affine  # noqa: E402

from paper_2108_12550_b200 import automorphism as host_aut  # noqa: E402
from paper_2108_12550_b200.plan import map_sizes  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

# name: (r, m, L, M, perms, frames, mode, ebn0, identity_root, extra)
CASES = {
    "rm25_fhtfsc_channel": (2, 5, 1, 1, False, 96, "channel", 3.0, 0, {}),
    "rm25_fhtfsc_exact": (2, 5, 1, 1, False, 96, "exact31", 3.0, 0, {}),
    "rm27_L2_M4_channel": (2, 7, 2, 4, True, 200, "channel", 2.0, 2, {}),
    "rm27_L2_M4_exact": (2, 7, 2, 4, True, 48, "exact31", 2.0, 2, {}),
    "rm29_L4_M20_channel": (2, 9, 4, 20, True, 64, "channel", 2.5, 4, {}),
    "rm29_L4_M20_exact": (2, 9, 4, 20, True, 32, "exact31", 2.5, 4, {}),
    "rm29_L4_M20_exact1024": (2, 9, 4, 20, True, 8, "exact1024", 2.5, 4, {}),
    "rm37_L8_M32_channel": (3, 7, 8, 32, True, 24, "channel", 4.0, 8, {}),
    "rm37_L8_M32_exact": (3, 7, 8, 32, True, 16, "exact31", 4.0, 8, {}),
    "rm29_L1_M512_channel": (2, 9, 1, 512, True, 8, "channel", 3.0, 1, {}),
    "rm29_L1_M512_exact": (2, 9, 1, 512, True, 6, "exact31", 3.0, 1, {}),
    "rm26_L4_M1_channel": (2, 6, 4, 1, True, 64, "channel", 2.0, 0, {}),
    "rm26_fhtfscl_L4_channel": (2, 6, 4, 1, False, 64, "channel", 2.0, 0, {}),
    "rm26_fhtfscl_L4_exact": (2, 6, 4, 1, False, 64, "exact31", 2.0, 0, {}),
    "rm36_L2_M3_exact": (3, 6, 2, 3, True, 24, "exact31", 2.0, 0, {}),
    "rm24_L2_M2_exact": (2, 4, 2, 2, True, 48, "exact31", 2.0, 0, {}),
    "rm15_L4_M3_channel": (1, 5, 4, 3, True, 32, "channel", 1.0, 0, {}),
    "rm34_L4_M2_channel": (3, 4, 4, 2, True, 32, "channel", 2.0, 0, {}),
    "rm12_L4_M2_exact": (1, 2, 4, 2, True, 32, "exact31", 2.0, 0, {}),
    "rm25_L4_M2_zero": (2, 5, 4, 2, True, 24, "zero", 3.0, 0, {}),
    "rm28_L8_M4_channel": (2, 8, 8, 4, True, 8, "channel", 2.0, 0, {}),
    "rm38_L4_M4_exact": (3, 8, 4, 4, True, 6, "exact31", 2.0, 4, {}),
    "rm29_L2_M8_channel": (2, 9, 2, 8, True, 8, "channel", 2.5, 2, {}),
}


# Aut-SSC (top_decoders.py:235-249): name: (r, m, P, frames, mode, ebn0)
AUT_CASES = {
    "autssc_rm12_P4_exact": (1, 2, 4, 32, "exact31", 2.0),
    "autssc_rm15_P3_zero": (1, 5, 3, 24, "zero", 3.0),
    "autssc_rm25_P8_exact": (2, 5, 8, 48, "exact31", 2.0),
    "autssc_rm27_P16_channel": (2, 7, 16, 256, "channel", 2.0),
    "autssc_rm28_P64_channel": (2, 8, 64, 64, "channel", 2.0),
    "autssc_rm38_P32_exact": (3, 8, 32, 48, "exact31", 2.5),
    "autssc_rm48_P16_channel": (4, 8, 16, 48, "channel", 3.0),
    "autssc_rm29_P32_channel": (2, 9, 32, 32, "channel", 2.0),
    "autssc_rm310_P8_channel": (3, 10, 8, 16, "channel", 3.0),
}


def run_aut_case(name, r, m, P, frames, mode, ebn0):
    """The reference's aut_ssc on a replayed table, plus its per-decode scores
    (ssc_decode / apply_perm / correlation, the same calls aut_ssc makes)."""
    spec = ref_core.build_code(r, m)
    llrs, xs = make_llrs(spec, frames, mode, ebn0)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    raw = host_aut.random_raw_table(rng, (frames, P), [m], m).reshape(frames, P, m + 1)
    cw = np.zeros((frames, spec.N), dtype=np.uint8)
    score = np.zeros(frames)
    winner = np.zeros(frames, dtype=np.int32)
    scores = np.zeros((frames, P))
    for f in range(frames):
        alpha = llrs[f].astype(np.float64)
        maps = [to_ref_perm(p) for p in host_aut.raw_to_maps(raw[f], [m] * P)]
        res = aut_ssc(spec, alpha, P, None, sampler=replay_sampler(maps))
        best, bs = -1, -np.inf
        for p, perm in enumerate(maps):
            cand = apply_perm_inverse(perm, ssc_decode(spec, apply_perm(perm, alpha)).codeword)
            scores[f, p] = correlation(cand, alpha)
            if scores[f, p] > bs:
                best, bs = p, scores[f, p]
        assert np.array_equal(res.codeword, apply_perm_inverse(
            maps[best], ssc_decode(spec, apply_perm(maps[best], alpha)).codeword)), name
        cw[f], score[f], winner[f] = res.codeword, bs, best
    return dict(r=r, m=m, P=P, mode=mode, ebn0=ebn0, llr=llrs, x=xs, raw=raw, scores=scores,
                cw=np.packbits(cw, axis=-1, bitorder="little"), score=score, winner=winner)


def make_llrs(spec, frames, mode, ebn0, seed=777, q=0):
    chan = ChannelConfig.for_rate(ebn0, spec.rate, seed)
    out = np.zeros((frames, spec.N), dtype=np.float32)
    xs = np.zeros((frames, spec.N), dtype=np.uint8)
    for k in range(frames):
        rng = frame_rng(seed, q, k)
        u = ref_core.random_message(spec, rng)
        x = ref_core.polar_transform(u)
        y = transmit(x, chan, rng, zero_noise=(mode == "zero"))
        a = llr(y, chan)
        if mode == "exact31":
            a = np.clip(np.round(3.0 * a), -31, 31)
        elif mode == "exact1024":
            a = np.clip(np.round(64.0 * a), -1024, 1024)
        elif mode == "zero":
            a = (1.0 - 2.0 * x) * 4.0
        out[k] = a.astype(np.float32)
        xs[k] = x
    return out, xs


def replay_sampler(maps):
    it = iter(maps)
    return lambda: next(it)


def to_ref_perm(p):
    return AffinePermutation(p.a, p.b)


def run_case(name, r, m, L, M, perms, frames, mode, ebn0, identity_root):
    spec = ref_core.build_code(r, m)
    llrs, xs = make_llrs(spec, frames, mode, ebn0)
    sizes = map_sizes(r, m, L, perms)
    S = len(sizes)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    N = spec.N
    Meff = M if perms else 1
    att_pm = np.zeros((frames, Meff))
    att_cw = np.zeros((frames, Meff, N), dtype=np.uint8)
    pm = np.zeros(frames)
    cw = np.zeros((frames, N), dtype=np.uint8)
    attempt = np.zeros(frames, dtype=np.int32)
    if perms:
        raw = host_aut.random_raw_table(rng, (frames, M), sizes, m, identity_root=identity_root)
    else:
        raw = np.zeros((frames, 1, 0, m + 1), dtype=np.uint16)
    for f in range(frames):
        alpha = llrs[f].astype(np.float64)
        if not perms:
            res = fht_fsc_decode(spec, alpha) if L == 1 else fht_fscl_decode(spec, alpha, L)
            att_pm[f, 0] = res.pm
            att_cw[f, 0] = res.codeword
            pm[f], cw[f], attempt[f] = res.pm, res.codeword, 0
            continue
        maps = [to_ref_perm(p) for p in host_aut.raw_to_maps(raw[f], sizes * M)]
        for a in range(M):
            sub = maps[a * S:(a + 1) * S]
            res = p_fht_fscl(spec, alpha, L, None, sampler=replay_sampler(sub))
            att_pm[f, a] = res.pm
            att_cw[f, a] = res.codeword
        # the reference's own ensemble over the same table
        ens = ensemble_decode(spec, alpha, L, M, np.random.default_rng(0),
                              sampler=replay_sampler(maps))
        best = 0
        for a in range(1, M):
            if att_pm[f, a] < att_pm[f, best]:
                best = a
        assert ens.pm == att_pm[f, best] and np.array_equal(ens.codeword, att_cw[f, best]), name
        pm[f], cw[f], attempt[f] = ens.pm, ens.codeword, best
    return dict(r=r, m=m, L=L, M=M, perms=int(perms), mode=mode, ebn0=ebn0, llr=llrs, x=xs,
                raw=raw, sizes=np.asarray(sizes, dtype=np.int32), att_pm=att_pm,
                att_cw=np.packbits(att_cw, axis=-1, bitorder="little"), pm=pm,
                cw=np.packbits(cw, axis=-1, bitorder="little"), attempt=attempt)


def sampler_stream_fixture():
    """The reference sampler's own draws (to pin host-side stream replay)."""
    out = {}
    for m, count, seed in [(9, 4, 1), (9, 8, 2), (7, 16, 3), (6, 16, 4), (5, 3, 5), (2, 7, 6)]:
        g = np.random.default_rng(seed)
        maps = sample_affine_batch(m, count, g)
        raw = host_aut.maps_to_raw(maps, m)
        out[f"m{m}_c{count}_s{seed}"] = raw
        out[f"m{m}_c{count}_s{seed}_next"] = g.integers(0, 2 ** 31, size=4)
        out[f"m{m}_c{count}_s{seed}_perm0"] = maps[0].perm
    # single draws (sample_affine, automorphism.py:127-141), as aut_ssc makes them
    for m, count, seed in [(9, 6, 7), (5, 10, 8), (2, 12, 9), (8, 5, 10)]:
        g = np.random.default_rng(seed)
        maps = [sample_affine(m, g) for _ in range(count)]
        out[f"single_m{m}_c{count}_s{seed}"] = host_aut.maps_to_raw(maps, m)
        out[f"single_m{m}_c{count}_s{seed}_next"] = g.integers(0, 2 ** 31, size=4)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for name, (r, m, L, M, perms, frames, mode, ebn0, ident, _extra) in CASES.items():
        if args.only and args.only != name:
            continue
        t0 = time.time()
        d = run_case(name, r, m, L, M, perms, frames, mode, ebn0, ident)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
        print(f"{name}: {frames} frames in {time.time() - t0:.1f}s", flush=True)
    for name, (r, m, P, frames, mode, ebn0) in AUT_CASES.items():
        if args.only and args.only not in (name, "aut"):
            continue
        t0 = time.time()
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **run_aut_case(name, r, m, P, frames, mode, ebn0))
        print(f"{name}: {frames} frames in {time.time() - t0:.1f}s", flush=True)
    if not args.only or args.only == "sampler":
        np.savez_compressed(os.path.join(OUT, "sampler_stream.npz"), **sampler_stream_fixture())
        print("sampler_stream done")


if __name__ == "__main__":
    main()
