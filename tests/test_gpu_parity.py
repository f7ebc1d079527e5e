"""CUDA decoder parity (needs a B200).

* float64 kernel vs the reference (golden fixtures): bit-exact on every field.
* float32 kernels vs the float32 oracle restatement of the same operation
  order: bit-exact on every field (the throughput kernel "v2" sums LM and
  llr_abs in its own order, restated by oracle order="v2"; the
  reference-order float32 kernel against oracle order="reference").
* float32 kernel vs the reference: bit-exact on exact-arithmetic fixtures;
  on channel fixtures PM within 1e-5 relative and codewords equal except on
  frames the float64 oracle flags as near-ties (counted, and must be rare).
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden

NAMES = golden_names()
pytestmark = pytest.mark.gpu


def _plan(g, dtype, reference_order=False):
    from paper_2108_12550_b200.decoder import Plan
    return Plan(g["r"], g["m"], g["L"], g["M"], bool(g["perms"]), dtype, reference_order=reference_order)


def _gpu(g, dtype, reference_order=False):
    p = _plan(g, dtype, reference_order)
    out = p.decode(g["llr"], raw_maps=g["raw"] if g["perms"] else None, diag=True)
    out["kernel"] = p.kernel
    return out


def _order(kernel):
    return "v2" if kernel in (2, 7) else "reference"  # 7: lane-group kernel, the throughput kernel's L = 1 order


@pytest.mark.parametrize("name", NAMES)
def test_f64_kernel_bit_exact_with_reference(name):
    g = load_golden(name)
    o = _gpu(g, "f64")
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["pm"], g["pm"])
    assert np.array_equal(o["attempt"], g["attempt"])
    assert np.array_equal(o["att_pm"], g["att_pm"])
    assert np.array_equal(o["att_cw"], g["att_cw_bits"])


@pytest.mark.parametrize("reference_order", [False, True])
@pytest.mark.parametrize("name", NAMES)
def test_f32_kernel_bit_exact_with_f32_oracle(name, reference_order, oracle_mod):
    g = load_golden(name)
    o = _gpu(g, "f32", reference_order)
    c = oracle_mod.decode(g["r"], g["m"], g["L"], g["M"], g["llr"], g["raw"] if g["perms"] else None,
                          perms=bool(g["perms"]), dtype=np.float32, nthreads=8, order=_order(o["kernel"]))
    assert np.array_equal(o["cw"], c["cw"])
    assert np.array_equal(o["pm"], c["pm"])
    assert np.array_equal(o["attempt"], c["attempt"])
    assert np.array_equal(o["path"], c["path"])
    assert np.array_equal(o["att_pm"], c["att_pm"])
    assert np.array_equal(o["att_cw"], c["att_cw"])


@pytest.mark.parametrize("name", NAMES)
def test_f32_kernel_against_reference(name, oracle_mod):
    g = load_golden(name)
    o = _gpu(g, "f32")
    if g["mode"] != "channel":
        assert np.array_equal(o["cw"], g["cw_bits"])
        assert np.array_equal(o["pm"].astype(np.float64), g["pm"])
        assert np.array_equal(o["attempt"], g["attempt"])
        return
    pm = o["pm"].astype(np.float64)
    assert np.all(np.abs(pm - g["pm"]) <= 1e-5 * np.maximum(np.abs(g["pm"]), 1.0))
    c64 = oracle_mod.decode(g["r"], g["m"], g["L"], g["M"], g["llr"], g["raw"] if g["perms"] else None,
                            perms=bool(g["perms"]), dtype=np.float64, nthreads=8)
    differ = ~np.all(o["cw"] == g["cw_bits"], axis=1)
    assert np.all(c64["margin"][differ] <= 1e-5), "codeword mismatch on a frame without a near-tie"
    # selected attempt: same codeword and PM-equivalent in the reference
    a = o["attempt"]
    same = np.all(g["att_cw_bits"][np.arange(len(a)), a] == g["cw_bits"], axis=1)
    near = np.abs(g["att_pm"][np.arange(len(a)), a] - g["pm"]) <= 1e-5 * np.maximum(np.abs(g["pm"]), 1.0)
    assert np.all((same & near) | differ)


# ------------------------------------------------ larger batches, headline shapes
SHAPES = [(2, 9, 4, 20, 2.5, 512), (2, 7, 2, 4, 2.0, 4096), (3, 7, 8, 32, 4.0, 256), (2, 9, 1, 512, 3.0, 48),
          (2, 9, 4, 20, 1.0, 256)]


@pytest.mark.parametrize("r,m,L,M,ebn0,B", SHAPES)
def test_batch_f32_bit_exact_with_oracle(r, m, L, M, ebn0, B, oracle_mod):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code, is_codeword
    spec = build_code(r, m)
    x, llr = synthetic_frames(spec, ebn0, B, seed=11 + r + m)
    plan = Plan(r, m, L, M, True, "f32")
    raw, rec = plan.sample(B, seed=5, identity_root=True)
    o = plan.decode(llr, records=rec)
    c = oracle_mod.decode(r, m, L, M, llr, raw, dtype=np.float32, nthreads=16, order=_order(plan.kernel),
                          want_attempts=False)
    assert np.array_equal(o["cw"], c["cw"])
    assert np.array_equal(o["pm"], c["pm"])
    assert np.array_equal(o["attempt"], c["attempt"])
    assert np.array_equal(o["path"], c["path"])
    for f in range(0, B, max(1, B // 16)):
        assert is_codeword(spec, o["cw"][f])


@pytest.mark.parametrize("r,m,L,M,ebn0,B", SHAPES[:3])
def test_batch_f64_bit_exact_with_oracle(r, m, L, M, ebn0, B, oracle_mod):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(r, m)
    x, llr = synthetic_frames(spec, ebn0, B // 2, seed=3)
    plan = Plan(r, m, L, M, True, "f64")
    raw, rec = plan.sample(B // 2, seed=9, identity_root=True)
    o = plan.decode(llr.astype(np.float64), records=rec)
    c = oracle_mod.decode(r, m, L, M, llr.astype(np.float64), raw, dtype=np.float64, nthreads=16,
                          want_attempts=False)
    assert np.array_equal(o["cw"], c["cw"]) and np.array_equal(o["pm"], c["pm"])
    assert np.array_equal(o["attempt"], c["attempt"])


def test_zero_noise_round_trip():
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code, polar_transform, random_message
    spec = build_code(2, 9)
    rng = np.random.default_rng(4)
    x = np.stack([polar_transform(random_message(spec, rng)) for _ in range(64)])
    plan = Plan(2, 9, 4, 20, True, "f32")
    _, rec = plan.sample(64, seed=2)
    o = plan.decode(((1.0 - 2.0 * x) * 4.0).astype(np.float32), records=rec)
    assert np.array_equal(o["cw"], x) and np.all(o["pm"] == 0)


@pytest.mark.parametrize("r,m,L,M", [(2, 9, 4, 20), (3, 7, 8, 32), (2, 7, 2, 4), (4, 9, 2, 3), (5, 8, 2, 3)])
def test_device_sampler_matches_host(r, m, L, M):
    import torch
    from paper_2108_12550_b200.decoder import Plan
    plan = Plan(r, m, L, M, True, "f32")
    raw, rec = plan.sample(37, seed=123, frame0=1000, identity_root=True)
    d = plan.sample_device(37, seed=123, frame0=1000, identity_root=True)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy().view(np.uint16), rec)


def test_sampled_decode_matches_table_decode():
    import torch
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    _, llr = synthetic_frames(spec, 2.5, 300, seed=8)
    plan = Plan(2, 9, 4, 20, True, "f32")
    _, rec = plan.sample(300, seed=77, frame0=5)
    a = plan.decode(llr, records=rec)
    d_llr = torch.from_numpy(llr).cuda()
    out = plan.alloc_outputs(300)
    plan.launch_sampled(d_llr, 77, out, frame0=5)
    torch.cuda.synchronize()
    assert np.array_equal(out["cw"].cpu().numpy().view(np.uint32), a["cw_packed"])
    assert np.array_equal(out["pm"].cpu().numpy(), a["pm"])
    assert np.array_equal(out["attempt"].cpu().numpy(), a["attempt"])


def test_stream_decoder_matches_direct_launch():
    import torch
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan, StreamDecoder
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 7)
    plan = Plan(2, 7, 2, 4, True, "f32")
    batches = [synthetic_frames(spec, 2.0, 1000, seed=s)[1] for s in range(5)]
    sd = StreamDecoder(plan, 1000, seed=31)
    got = []
    for llr in batches:
        r = sd.submit(torch.from_numpy(llr).pin_memory())
        if r is not None:
            got.append({k: v.clone() for k, v in r.items()})
    got += [{k: v.clone() for k, v in r.items()} for r in sd.drain()]
    assert len(got) == 5
    for i, llr in enumerate(batches):
        _, rec = plan.sample(1000, seed=31, frame0=1000 * i)
        ref = plan.decode(llr, records=rec)
        assert np.array_equal(got[i]["cw"].numpy().view(np.uint32), ref["cw_packed"])
        assert np.array_equal(got[i]["pm"].numpy(), ref["pm"])
        assert np.array_equal(got[i]["attempt"].numpy(), ref["attempt"])


def test_chunked_launch_matches_single_launch(monkeypatch):
    """Batches above the per-launch item limit go in frame chunks
    (launch_fast); a tiny limit (RMFHT_MAX_ITEMS, read when the plan binds)
    must reproduce the single-launch result on every field, diag included."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    _, llr = synthetic_frames(spec, 2.5, 77, seed=21)
    one = Plan(2, 9, 4, 20, True, "f32")
    _, rec = one.sample(77, seed=4)
    a = one.decode(llr, records=rec, diag=True)
    monkeypatch.setenv("RMFHT_MAX_ITEMS", "200")  # 10 frames (200 items) per launch: 8 chunks
    many = Plan(2, 9, 4, 20, True, "f32")
    b = many.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        if k in a:
            assert np.array_equal(a[k], b[k]), k
