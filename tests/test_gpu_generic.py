"""The generic (runtime-shaped) kernel: bit-exact with the reference fixtures
(float64) and with the float32 oracle on every fixture, and on shapes that
have no compile-time specialisation."""
import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu
NAMES = golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_generic_f64_bit_exact_with_reference(name):
    from paper_2108_12550_b200.decoder import Plan
    g = load_golden(name)
    p = Plan(g["r"], g["m"], g["L"], g["M"], bool(g["perms"]), "f64", generic=True)
    assert p.kernel == 3
    o = p.decode(g["llr"], raw_maps=g["raw"] if g["perms"] else None, diag=True)
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["pm"], g["pm"])
    assert np.array_equal(o["attempt"], g["attempt"])
    assert np.array_equal(o["att_pm"], g["att_pm"])


@pytest.mark.parametrize("name", NAMES)
def test_generic_f32_bit_exact_with_oracle(name, oracle_mod):
    from paper_2108_12550_b200.decoder import Plan
    g = load_golden(name)
    p = Plan(g["r"], g["m"], g["L"], g["M"], bool(g["perms"]), "f32", generic=True)
    o = p.decode(g["llr"], raw_maps=g["raw"] if g["perms"] else None)
    c = oracle_mod.decode(g["r"], g["m"], g["L"], g["M"], g["llr"], g["raw"] if g["perms"] else None,
                          perms=bool(g["perms"]), dtype=np.float32, nthreads=8)
    assert np.array_equal(o["cw"], c["cw"]) and np.array_equal(o["pm"], c["pm"])
    assert np.array_equal(o["attempt"], c["attempt"])


UNCOMPILED = [(2, 8, 2, 3), (4, 8, 2, 2), (1, 6, 8, 2), (5, 6, 4, 2), (2, 10, 2, 2), (3, 9, 4, 2), (2, 3, 2, 2),
              (3, 5, 16, 2), (2, 6, 3, 3)]


@pytest.mark.parametrize("r,m,L,M", UNCOMPILED)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_uncompiled_shapes(r, m, L, M, dtype, oracle_mod):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code, is_codeword
    spec = build_code(r, m)
    p = Plan(r, m, L, M, True, dtype)
    assert p.kernel in (1, 2, 3)
    x, llr = synthetic_frames(spec, 1.5, 24, seed=r * 100 + m * 10 + L)
    raw, _ = p.sample(24, seed=3)
    dt = np.float64 if dtype == "f64" else np.float32
    o = p.decode(llr.astype(dt), raw_maps=raw)
    c = oracle_mod.decode(r, m, L, M, llr.astype(dt), raw, dtype=dt, nthreads=8,
                          order="v2" if p.kernel in (2, 7) else "reference")
    assert np.array_equal(o["cw"], c["cw"]) and np.array_equal(o["pm"], c["pm"])
    assert np.array_equal(o["attempt"], c["attempt"])
    for f in range(0, 24, 6):
        assert is_codeword(spec, o["cw"][f])
