"""TEST INFRASTRUCTURE ONLY — tie accounting of the float32 GPU decoder
against the float64 CPU port (the reference restated; SURVEY §8(c)
"Channel-LLR mode").  Used by tests/, tools/gpu_xcheck.py and bench.py's
CPU-baseline leg; the product package never imports it.

BASELINE.json north_star: "Decoded codewords and selected path indices must
be bit-exact except on exact path-metric ties, which are counted and
reported.  Path metrics must agree within 1e-5 relative in fp32."

Per frame, with the port run on the same float32 LLRs (upcast exactly) and
the same permutation table:

* ``ens_exact_ties``: two or more attempts reach the port's minimum pm
  exactly (top_decoders.py:200 keeps the first, strict <).
* ``ens_near_ties``: no exact tie, but another attempt's pm is within
  ``rel`` of the minimum (fp32 rounding can reorder them).
* ``sel_exact_ties`` / ``sel_near_ties``: the port's instrumented minimum
  selection gap over every ranking inside every attempt (extension LM cut,
  FHT per-path top-k and pool cut, SPC order; ``margin``) is exactly 0 /
  within ``rel``.
* ``cw_mismatch``: GPU codeword != port codeword; ``_excused`` when the
  frame has a near or exact tie at some selection (margin <= rel), else
  ``_unexcused`` (must be 0).
* ``attempt_mismatch``: GPU attempt != port attempt; ``_pm_equivalent``
  when the port's own pm for the GPU's attempt is within ``rel`` of its
  minimum and that attempt's codeword equals the port's answer (the same
  decision reached by another attempt), else ``_other``; ``_unexcused``
  counts the ones that are neither pm-equivalent nor on a near-tie frame;
  ``_on_exact_ties`` the ones where the GPU picked another attempt of the
  port's exactly tied minimum (same codeword, bit-identical float64 pm): the
  "exact path-metric ties" of the north star.
* ``pm_max_rel``: max |pm_gpu - pm_port| / max(|pm_port|, 1).
"""

from __future__ import annotations

import numpy as np

REL = 1e-5


def classify(gpu_cw, gpu_pm, gpu_att, port, rel: float = REL, x=None) -> dict:
    """gpu_cw uint8 [B, N]; gpu_pm [B]; gpu_att int [B]; port = oracle.decode(...,
    dtype=float64, want_attempts=True) on the same inputs.  x: transmitted
    codewords (optional) for frame-error counts on both sides."""
    B = gpu_cw.shape[0]
    pcw, ppm, patt = port["cw"], port["pm"].astype(np.float64), port["attempt"]
    att_pm = port["att_pm"].astype(np.float64)
    margin = port["margin"]
    idx = np.arange(B)
    scale = np.maximum(np.abs(ppm), 1.0)
    n_at_min = np.sum(att_pm == ppm[:, None], axis=1)
    ens_exact = n_at_min >= 2
    near_mask = (np.abs(att_pm - ppm[:, None]) <= rel * scale[:, None]) & (att_pm != ppm[:, None])
    ens_near = ~ens_exact & np.any(near_mask, axis=1)
    sel_exact = margin == 0.0
    sel_near = (margin > 0.0) & (margin <= rel)
    tie_frame = margin <= rel
    cw_diff = np.any(gpu_cw != pcw, axis=1)
    att_diff = gpu_att != patt
    ga = np.clip(gpu_att, 0, att_pm.shape[1] - 1)
    pm_equiv = np.abs(att_pm[idx, ga] - ppm) <= rel * scale
    if port.get("att_cw") is not None:
        same_cw = np.all(port["att_cw"][idx, ga] == pcw, axis=1)
    else:
        same_cw = np.ones(B, dtype=bool)
    att_equiv = att_diff & pm_equiv & same_cw
    # the GPU's attempt is one of the port's exactly tied minimum attempts
    on_exact = att_diff & (att_pm[idx, ga] == ppm) & same_cw
    pm_rel = np.abs(gpu_pm.astype(np.float64) - ppm) / scale
    out = dict(
        frames=int(B),
        ens_exact_ties=int(ens_exact.sum()), ens_near_ties=int(ens_near.sum()),
        sel_exact_ties=int(sel_exact.sum()), sel_near_ties=int(sel_near.sum()),
        cw_mismatch=int(cw_diff.sum()), cw_mismatch_excused=int((cw_diff & tie_frame).sum()),
        cw_mismatch_unexcused=int((cw_diff & ~tie_frame).sum()),
        attempt_mismatch=int(att_diff.sum()), attempt_mismatch_pm_equivalent=int(att_equiv.sum()),
        attempt_mismatch_on_exact_ties=int(on_exact.sum()),
        attempt_mismatch_unexcused=int((att_diff & ~att_equiv & ~tie_frame).sum()),
        pm_max_rel=float(pm_rel.max()) if B else 0.0,
        pm_over_tol=int((pm_rel > rel).sum()),
        rel_tolerance=rel,
    )
    if x is not None:
        out["gpu_frame_errors"] = int(np.sum(np.any(gpu_cw != x, axis=1)))
        out["port_frame_errors"] = int(np.sum(np.any(pcw != x, axis=1)))
    return out


def merge(parts) -> dict:
    """Sum the counters of several classify() results (max for pm_max_rel)."""
    out: dict = {}
    for p in parts:
        for k, v in p.items():
            if k == "pm_max_rel":
                out[k] = max(out.get(k, 0.0), v)
            elif k == "rel_tolerance":
                out[k] = v
            else:
                out[k] = out.get(k, 0) + v
    return out


def ok(c: dict) -> bool:
    """The north-star bar: every mismatch excused by a tie, pm within rel."""
    return c["cw_mismatch_unexcused"] == 0 and c["attempt_mismatch_unexcused"] == 0 and c["pm_over_tol"] == 0
