"""Host-side logic: code shapes, schedule, map tables, sampler stream replay."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2108_12550_b200 import automorphism as aut
from paper_2108_12550_b200.plan import map_sizes, plan_visits
from paper_2108_12550_b200.rm_core import (ConfigurationError, build_code, is_codeword,
                                           polar_transform, random_message)


def test_build_code_shapes_and_errors():
    s = build_code(2, 9)
    assert (s.N, s.K, s.d) == (512, 46, 128)
    assert build_code(3, 7).K == 64 and build_code(2, 7).K == 29 and build_code(2, 5).K == 16
    for r, m in [(0, 5), (5, 5), (1, 1), (1, 15)]:
        with pytest.raises(ConfigurationError):
            build_code(r, m)


def test_schedules_match_survey():
    # SURVEY §3.3 probed schedules (accounting.plan_visits)
    v = plan_visits(2, 9)
    assert v[:3] == [("perm", 9), ("f", 9), ("fht", 8)]
    assert v[-1] == ("spc", 3)
    assert sum(1 for k, _ in v if k == "perm") == 1
    v37 = plan_visits(3, 7)
    assert [m for k, m in v37 if k == "perm"] == [7, 6]
    assert sum(1 for k, _ in v37 if k == "fht") == 6 and sum(1 for k, _ in v37 if k == "spc") == 4
    assert map_sizes(2, 9, 4) == [9] * 12
    assert map_sizes(3, 7, 8) == [7] * 24 + [6] * 16
    assert map_sizes(2, 9, 1) == [9] * 3
    assert map_sizes(2, 5, 1, permutations=False) == []


def test_polar_codewords():
    rng = np.random.default_rng(0)
    spec = build_code(2, 6)
    for _ in range(20):
        x = polar_transform(random_message(spec, rng))
        assert is_codeword(spec, x)
    x[3] ^= 1
    assert not is_codeword(spec, x)


def test_sampler_replays_reference_stream():
    d = np.load(os.path.join(GOLDEN, "sampler_stream.npz"))
    for key in [k for k in d.files if not k.endswith(("_next", "_perm0")) and not k.startswith("single_")]:
        m, count, seed = (int(t[1:]) for t in key.split("_"))
        g = np.random.default_rng(seed)
        maps = aut.sample_affine_batch(m, count, g)
        assert np.array_equal(aut.maps_to_raw(maps, m), d[key])
        assert np.array_equal(g.integers(0, 2 ** 31, size=4), d[key + "_next"])  # same draws consumed
        assert np.array_equal(maps[0].perm, d[key + "_perm0"])


def test_single_sampler_replays_reference_stream():
    """sample_affine (automorphism.py:127-141), the per-decode draw of aut_ssc."""
    d = np.load(os.path.join(GOLDEN, "sampler_stream.npz"))
    keys = [k for k in d.files if k.startswith("single_") and not k.endswith("_next")]
    assert keys
    for key in keys:
        m, count, seed = (int(t[1:]) for t in key.split("_")[1:])
        g = np.random.default_rng(seed)
        maps = [aut.sample_affine(m, g) for _ in range(count)]
        assert np.array_equal(aut.maps_to_raw(maps, m), d[key])
        assert np.array_equal(g.integers(0, 2 ** 31, size=4), d[key + "_next"])


def test_random_table_is_invertible_and_uniform_shape():
    rng = np.random.default_rng(1)
    sizes = map_sizes(3, 7, 8)
    raw = aut.random_raw_table(rng, (5, 3), sizes, 7, identity_root=8)
    assert raw.shape == (5, 3, len(sizes), 8)
    for f in range(5):
        for a in range(3):
            for s, mn in enumerate(sizes):
                masks = raw[f, a, s, :mn].astype(np.int64)
                assert aut.gf2_invertible_masks(masks[None, :], mn)[0]
                assert not raw[f, a, s, mn:7].any()
    assert np.all(raw[:, 0, :8, :7] == (1 << np.arange(7)))
    assert np.all(raw[:, 0, :8, 7] == 0)


def test_affine_map_inverse_and_identity():
    rng = np.random.default_rng(2)
    for m in (3, 6, 9):
        p = aut.sample_affine_batch(m, 1, rng)[0]
        assert np.array_equal(p.perm[p.inv], np.arange(1 << m))
    assert np.array_equal(aut.AffineMap.identity(4).perm, np.arange(16))


def test_counter_sampler_uniform_over_gl3():
    """rmfht_sample_maps draws A uniformly from GL(3,2) (168 elements) and b
    uniformly from F_2^3 — the reference's distribution (automorphism.py:127-161)."""
    from paper_2108_12550_b200.decoder import Plan
    from scipy.stats import chisquare
    plan = Plan(1, 3, 4, 8, True, "f32")       # RM(1,3): L root maps of 3 variables per attempt
    assert plan.S == 4 and list(plan.sizes) == [3, 3, 3, 3]
    raw, _ = plan.sample(420, seed=3, identity_root=False)
    A = raw[..., :3].reshape(-1, 3).astype(np.int64)
    assert aut.gf2_invertible_masks(A, 3).all()
    code = A[:, 0] | (A[:, 1] << 3) | (A[:, 2] << 6)
    uniq, counts = np.unique(code, return_counts=True)
    assert len(uniq) == 168 and counts.sum() == 420 * 8 * 4
    assert chisquare(counts).pvalue > 1e-4
    b = raw[..., 3].ravel()
    assert chisquare(np.bincount(b, minlength=8)).pvalue > 1e-4
    # A and b independent: contingency of (A[0,0], b)
    from scipy.stats import chi2_contingency
    joint = np.bincount(((A[:, 0] & 1) * 8 + b).astype(np.int64), minlength=16).reshape(2, 8)
    assert chi2_contingency(joint).pvalue > 1e-4


def test_counter_sampler_uniform_over_gl9_projection():
    """For m = 9 (the headline's root maps), the image of a fixed nonzero
    vector under A is uniform over the 511 nonzero vectors."""
    from paper_2108_12550_b200.decoder import Plan
    from scipy.stats import chisquare
    plan = Plan(2, 9, 4, 20, True, "f32")
    raw, _ = plan.sample(300, seed=11, identity_root=False)
    A = raw[..., :9].reshape(-1, 9).astype(np.int64)
    img = np.zeros(len(A), dtype=np.int64)
    for r in range(9):  # A @ (1,0,...,0, 1): columns 0 and 8
        img |= (((A[:, r] >> 0) ^ (A[:, r] >> 8)) & 1) << r
    counts = np.bincount(img, minlength=512)
    assert counts[0] == 0
    assert chisquare(counts[1:]).pvalue > 1e-4


def test_counter_sampler_batch_independent_and_identity_root():
    from paper_2108_12550_b200.decoder import Plan
    plan = Plan(2, 9, 4, 20, True, "f32")
    raw, rec = plan.sample(10, seed=5, frame0=0)
    raw2, rec2 = plan.sample(4, seed=5, frame0=6)
    assert np.array_equal(raw[6:], raw2) and np.array_equal(rec[6:], rec2)
    ident = np.zeros(10, dtype=np.uint16)
    ident[:9] = 1 << np.arange(9)
    assert np.all(raw[:, 0, :4, :] == ident)
    assert not np.any(np.all(raw[:, 1:, :, :] == ident, axis=-1))
    raw3, _ = plan.sample(10, seed=6, frame0=0)
    assert not np.array_equal(raw3[:, 1:], raw[:, 1:])


def test_counter_sampler_records_hold_the_inverse():
    """The sampler reads A^-1 off its reduced echelon basis (no Gauss-Jordan):
    every record's inverse columns, and c = A^-1 b, must invert (A, b); the
    raw rows must be the transpose of the record's columns.  Every map size
    of RM(3,7) L=8 (7 and 6 variables) and RM(2,9)."""
    from paper_2108_12550_b200.decoder import Plan

    def gf2_mul(cols_a, cols_b, m):  # columns of A.B
        out = []
        for cb in cols_b:
            v = 0
            for k in range(m):
                if (cb >> k) & 1:
                    v ^= cols_a[k]
            out.append(v)
        return out

    for (r, m, L, M) in [(3, 7, 8, 3), (2, 9, 4, 3)]:
        plan = Plan(r, m, L, M, True, "f32")
        raw, rec = plan.sample(6, seed=13, identity_root=False)
        for f in range(6):
            for a in range(M):
                for s, mn in enumerate(plan.sizes):
                    rr = [int(x) for x in rec[f, a, s]]
                    cols, b, icols, c = rr[:m], rr[m], rr[m + 1:2 * m + 1], rr[2 * m + 1]
                    assert not any(cols[mn:]) and not any(icols[mn:])
                    assert gf2_mul(cols[:mn], icols[:mn], mn) == [1 << k for k in range(mn)]
                    assert gf2_mul(icols[:mn], [b], mn)[0] == c
                    rows = [sum(((cols[k] >> i) & 1) << k for k in range(mn)) for i in range(mn)]
                    assert [int(x) for x in raw[f, a, s, :mn]] == rows and int(raw[f, a, s, m]) == b
