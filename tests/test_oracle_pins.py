"""Pin the CPU oracle against the unmodified Python reference.

tests/golden/*.npz were produced by tools/gen_golden.py, which ran the
reference's own p_fht_fscl / ensemble_decode / fht_fsc(l)_decode on these
exact LLRs and permutation tables.  The float64 oracle must match every
field bit-for-bit; the float32 restatement must match exactly on
exact-arithmetic fixtures and stay within the fp32 tolerance on channel
fixtures.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, aut_names, golden_names, load_aut, load_golden

NAMES = golden_names()
AUT = aut_names()


def _run(oracle_mod, g, dtype):
    return oracle_mod.decode(g["r"], g["m"], g["L"], g["M"], g["llr"],
                             g["raw"] if g["perms"] else None, perms=bool(g["perms"]),
                             dtype=dtype, nthreads=4)


@pytest.mark.parametrize("name", NAMES)
def test_f64_oracle_is_bit_exact_with_reference(oracle_mod, name):
    g = load_golden(name)
    o = _run(oracle_mod, g, np.float64)
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["pm"], g["pm"])
    assert np.array_equal(o["attempt"], g["attempt"])
    assert np.array_equal(o["att_pm"], g["att_pm"])
    assert np.array_equal(o["att_cw"], g["att_cw_bits"])


@pytest.mark.parametrize("name", NAMES)
def test_f32_oracle_against_reference(oracle_mod, name):
    g = load_golden(name)
    o = _run(oracle_mod, g, np.float32)
    if g["mode"] != "channel":
        # integer LLRs: every intermediate is exact in float32
        assert np.array_equal(o["cw"], g["cw_bits"])
        assert np.array_equal(o["pm"].astype(np.float64), g["pm"])
        assert np.array_equal(o["attempt"], g["attempt"])
        assert np.array_equal(o["att_pm"].astype(np.float64), g["att_pm"])
    else:
        # PM within 1e-5 relative (absolute 1e-5 near zero), codewords equal
        # except frames the f64 oracle marks as near-ties
        pm = o["pm"].astype(np.float64)
        assert np.all(np.abs(pm - g["pm"]) <= 1e-5 * np.maximum(np.abs(g["pm"]), 1.0))
        o64 = _run(oracle_mod, g, np.float64)
        differ = ~np.all(o["cw"] == g["cw_bits"], axis=1)
        assert np.all(o64["margin"][differ] <= 1e-5)


@pytest.mark.parametrize("name", AUT)
def test_aut_ssc_oracle_is_bit_exact_with_reference(oracle_mod, name):
    """aut_ssc (top_decoders.py:235-249): codeword, winning correlation and
    the winning permutation (first strictly largest score)."""
    g = load_aut(name)
    o = oracle_mod.aut_ssc(g["r"], g["m"], g["P"], g["llr"].astype(np.float64), g["raw"], nthreads=4)
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["score"], g["score"])
    assert np.array_equal(o["winner"], g["winner"])
    assert np.array_equal(o["score"], g["scores"].max(axis=1))


@pytest.mark.parametrize("name", AUT)
def test_aut_ssc_f32_oracle(oracle_mod, name):
    """float32 restatement: exact on integer-LLR fixtures; on channel LLRs the
    winner may only move between candidates whose float64 scores are within
    float32 rounding."""
    g = load_aut(name)
    o = oracle_mod.aut_ssc(g["r"], g["m"], g["P"], g["llr"].astype(np.float32), g["raw"], dtype=np.float32)
    if g["mode"] in ("exact31", "zero"):
        assert np.array_equal(o["cw"], g["cw_bits"])
        assert np.array_equal(o["winner"], g["winner"])
        assert np.array_equal(o["score"].astype(np.float64), g["score"])
    else:
        sc = g["scores"]
        picked = sc[np.arange(len(sc)), o["winner"]]
        assert np.all(picked >= g["score"] - 1e-5 * np.abs(g["score"]) - 1e-4)
        assert np.mean(o["winner"] == g["winner"]) > 0.9


def test_golden_fer_rows_pinned_by_port():
    """The reference's own golden FER file (pkg/data/golden_fer.csv:1-5,
    copied to tests/golden/ref_golden_fer.csv by tools/copy_ref_golden.sh):
    the float64 port on the reference harness stream (tools/fer_port.py,
    tests/golden/fer_points.json "golden_*") reproduces frames, frame errors
    and the ML bound of every row exactly — FHT-FSCL needs no table, and
    p-FHT-FSCL (M = 1) the frame generator's own draws, replayed."""
    import csv
    import json
    pts = json.load(open(os.path.join(GOLDEN, "fer_points.json")))
    rows = list(csv.DictReader(open(os.path.join(GOLDEN, "ref_golden_fer.csv"))))
    assert len(rows) == 4
    for row in rows:
        name = "golden_rm26_fhtfscl_L4" if row["decoder"] == "FHT-FSCL" else "golden_rm26_pfhtfscl_L4"
        pt = next(p for p in pts[name]["points"] if p["ebn0"] == float(row["ebn0_db"]))
        assert pt["frames"] == int(row["frames"])
        assert pt["errors"] == int(row["frame_errors"]), (name, row)
        assert pt["ml_errors"] == round(float(row["ml_lb_fer"]) * int(row["frames"])), (name, row)
