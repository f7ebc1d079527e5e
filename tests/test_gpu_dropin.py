"""The single-frame drop-in API (paper_2108_12550_b200.top_decoders) against
the oracle on the maps the reference would draw from the same rng (the
stream replay itself is pinned by tests/test_host.py against the
reference's own sampler)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _frame(spec, seed, ebn0=2.0):
    from paper_2108_12550_b200.channel_model import harness_frames
    x, llr, rngs = harness_frames(spec, ebn0, seed, 0, 0, 1)
    return x[0], llr[0].astype(np.float32).astype(np.float64), rngs[0]


def _oracle_attempts(oracle_mod, spec, alpha, L, maps_per_attempt):
    from paper_2108_12550_b200.automorphism import maps_to_raw
    M = len(maps_per_attempt)
    raw = np.stack([maps_to_raw(m, spec.m) for m in maps_per_attempt])[None]
    return oracle_mod.decode(spec.r, spec.m, L, M, alpha[None], raw, dtype=np.float64)


@pytest.mark.parametrize("r,m,L,M", [(2, 7, 2, 4), (2, 9, 4, 20), (3, 7, 8, 4), (2, 6, 3, 2)])
def test_ensemble_decode_consumes_rng_like_reference(r, m, L, M, oracle_mod):
    from paper_2108_12550_b200 import top_decoders as td
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(r, m)
    x, alpha, rng = _frame(spec, 5)
    state = rng.bit_generator.state
    res = td.ensemble_decode(spec, alpha, L, M, rng)
    after = rng.integers(0, 2 ** 31)
    # replay: M seeds from rng, then each attempt's maps from default_rng(seed)
    g = np.random.default_rng()
    g.bit_generator.state = state
    seeds = g.integers(0, 2 ** 63 - 1, size=M, dtype=np.int64)
    assert g.integers(0, 2 ** 31) == after
    maps = [td._attempt_maps(spec, L, np.random.default_rng(int(s)), None) for s in seeds]
    o = _oracle_attempts(oracle_mod, spec, alpha, L, maps)
    assert np.array_equal(res.codeword, o["cw"][0]) and res.pm == o["pm"][0]
    assert res.attempt == o["attempt"][0]


def test_p_fht_fscl_with_sampler_and_trace(oracle_mod):
    from paper_2108_12550_b200 import top_decoders as td
    from paper_2108_12550_b200.automorphism import sample_affine_batch
    from paper_2108_12550_b200.plan import map_sizes
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(3, 7)
    x, alpha, rng = _frame(spec, 9, 3.0)
    maps = [sample_affine_batch(mn, 1, np.random.default_rng(100 + i))[0] for i, mn in enumerate(map_sizes(3, 7, 8))]
    it = iter(maps)
    trace = []
    res = td.p_fht_fscl(spec, alpha, 8, None, sampler=lambda: next(it), trace=trace)
    o = _oracle_attempts(oracle_mod, spec, alpha, 8, [maps])
    assert np.array_equal(res.codeword, o["cw"][0]) and res.pm == o["pm"][0]
    assert [t[0] for t in trace][:4] == ["perm", "f", "perm", "f"]


def test_fht_fsc_and_fscl_and_dispatch(oracle_mod):
    from paper_2108_12550_b200 import top_decoders as td
    from paper_2108_12550_b200.rm_core import ConfigurationError, build_code
    spec = build_code(2, 6)
    x, alpha, rng = _frame(spec, 13)
    a = td.fht_fsc_decode(spec, alpha)
    o = oracle_mod.decode(2, 6, 1, 1, alpha[None], None, perms=False, dtype=np.float64)
    assert np.array_equal(a.codeword, o["cw"][0]) and a.pm == o["pm"][0]
    b = td.decode(spec, alpha, td.DecoderConfig("FHT-FSCL", L=4), rng)
    o = oracle_mod.decode(2, 6, 4, 1, alpha[None], None, perms=False, dtype=np.float64)
    assert np.array_equal(b.codeword, o["cw"][0]) and b.pm == o["pm"][0]
    c = td.decode(spec, alpha, td.DecoderConfig("p-FHT-FSCL", L=4, permutations_enabled=False), rng)
    assert np.array_equal(c.codeword, b.codeword) and c.pm == b.pm
    with pytest.raises(ConfigurationError):
        td.decode(spec, alpha, td.DecoderConfig("SCL", L=2), rng)
    with pytest.raises(ValueError):
        td.fht_fsc_decode(spec, alpha[:10])
    with pytest.raises(ConfigurationError):
        td.p_fht_fscl(spec, alpha, 2, None)


def test_zero_noise_and_degenerate_roots():
    # test_top_decoders.py:175-187: r = 1 and r = m-1 roots keep their root maps
    from paper_2108_12550_b200 import top_decoders as td
    from paper_2108_12550_b200.rm_core import build_code, polar_transform, random_message
    rng = np.random.default_rng(23)
    for (r, m) in [(1, 5), (3, 4), (1, 2), (2, 5)]:
        spec = build_code(r, m)
        for _ in range(5):
            x = polar_transform(random_message(spec, rng))
            res = td.p_fht_fscl(spec, (1.0 - 2.0 * x) * 8.0, 4, rng)
            assert np.array_equal(res.codeword, x) and res.pm == 0.0
