"""Aut-SSC on the GPU (aut_ssc, top_decoders.py:235-249)
against the reference's own outputs (tests/golden/autssc_*.npz, made by
tools/gen_golden.py running the unmodified aut_ssc on replayed tables) and
the CPU oracle (oracle/rmo_impl.h FN(rmo_aut_ssc)).  float64 is bit-exact
with the reference, including every one of the P decodes' correlations;
float32 is bit-exact with the oracle's float32 restatement."""
import numpy as np
import pytest

from conftest import aut_names, load_aut

pytestmark = pytest.mark.gpu
AUT = aut_names()


def _plan(g, dtype):
    from paper_2108_12550_b200.decoder import Plan
    return Plan(g["r"], g["m"], 1, g["P"], True, dtype, aut_ssc=True)


@pytest.mark.parametrize("name", AUT)
def test_f64_bit_exact_with_reference(name):
    g = load_aut(name)
    plan = _plan(g, "f64")
    assert plan.kernel == 4 and plan.S == 1
    o = plan.decode(g["llr"].astype(np.float64), raw_maps=g["raw"][:, :, None, :], diag=True)
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["pm"], g["score"])
    assert np.array_equal(o["attempt"], g["winner"])
    assert np.array_equal(o["att_pm"], g["scores"])          # every decode's correlation


@pytest.mark.parametrize("name", AUT)
def test_f32_bit_exact_with_oracle(oracle_mod, name):
    g = load_aut(name)
    llr = g["llr"].astype(np.float32)
    o = _plan(g, "f32").decode(llr, raw_maps=g["raw"][:, :, None, :])
    ref = oracle_mod.aut_ssc(g["r"], g["m"], g["P"], llr, g["raw"], dtype=np.float32)
    assert np.array_equal(o["cw"], ref["cw"])
    assert np.array_equal(o["pm"], ref["score"])
    assert np.array_equal(o["attempt"], ref["winner"])


def test_drop_in_api_with_sampler_and_rng(oracle_mod):
    from paper_2108_12550_b200 import automorphism as aut
    from paper_2108_12550_b200.rm_core import build_code
    from paper_2108_12550_b200.top_decoders import DecoderConfig, aut_ssc, decode
    g = load_aut("autssc_rm27_P16_channel")
    spec = build_code(g["r"], g["m"])
    for f in range(8):
        maps = aut.raw_to_maps(g["raw"][f], [g["m"]] * g["P"])
        it = iter(maps)
        res = aut_ssc(spec, g["llr"][f], g["P"], None, sampler=lambda: next(it))
        assert np.array_equal(res.codeword, g["cw_bits"][f]) and np.isnan(res.pm)
    # rng path: the reference's draws (sample_affine once per decode)
    alpha = g["llr"][0].astype(np.float64)
    res = decode(spec, alpha, DecoderConfig("Aut-SSC", P=16), np.random.default_rng(5))
    rng = np.random.default_rng(5)
    raw = aut.maps_to_raw([aut.sample_affine(spec.m, rng) for _ in range(16)], spec.m)
    ref = oracle_mod.aut_ssc(spec.r, spec.m, 16, alpha[None, :], raw[None])
    assert np.array_equal(res.codeword, ref["cw"][0]) and res.attempt == ref["winner"][0]


def test_sampled_matches_table_and_zero_noise():
    import torch
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    x, llr = synthetic_frames(spec, 2.5, 200, seed=3)
    plan = Plan(2, 9, 1, 64, True, "f32", aut_ssc=True)
    _, rec = plan.sample(200, seed=9, frame0=7, identity_root=False)
    a = plan.decode(llr, records=rec)
    out = plan.alloc_outputs(200)
    plan.launch_sampled(torch.from_numpy(llr).cuda(), 9, out, frame0=7, identity_root=False)
    torch.cuda.synchronize()
    assert np.array_equal(out["cw"].cpu().numpy().view(np.uint32), a["cw_packed"])
    assert np.array_equal(out["attempt"].cpu().numpy(), a["attempt"])
    z = plan.decode(((1.0 - 2.0 * x) * 3.0).astype(np.float32), records=rec)
    assert np.array_equal(z["cw"], x)


@pytest.mark.parametrize("P", [1, 3, 8, 17])
def test_odd_P_and_warp_counts(oracle_mod, P):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(3, 7)
    _, llr = synthetic_frames(spec, 2.0, 64, seed=P)
    plan = Plan(3, 7, 1, P, True, "f64", aut_ssc=True)
    raw, rec = plan.sample(64, seed=P, identity_root=False)
    o = plan.decode(llr.astype(np.float64), records=rec)
    ref = oracle_mod.aut_ssc(3, 7, P, llr.astype(np.float64), raw[:, :, 0, :])
    assert np.array_equal(o["cw"], ref["cw"]) and np.array_equal(o["attempt"], ref["winner"])


@pytest.mark.parametrize("r,m,P", [(2, 9, 40), (3, 8, 24), (4, 8, 16), (2, 10, 8), (2, 6, 33), (2, 5, 7)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_register_kernel_matches_shared_memory_kernel(r, m, P, dtype):
    """The compiled register-resident kernel (rmfht_ssc_reg.cuh) and the
    runtime-shaped shared-memory walk give identical results, every decode."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(r, m)
    _, llr = synthetic_frames(spec, 2.0, 48, seed=r * 100 + m)
    llr = llr.astype(np.float64 if dtype == "f64" else np.float32)
    reg = Plan(r, m, 1, P, True, dtype, aut_ssc=True)
    gen = Plan(r, m, 1, P, True, dtype, aut_ssc=True, generic=True)
    _, rec = reg.sample(48, seed=P, identity_root=False)
    a = reg.decode(llr, records=rec, diag=True)
    b = gen.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "att_pm", "att_cw"):
        assert np.array_equal(a[k], b[k]), k
