"""Lane-per-frame FHT-FSC kernel (rmfht_lane.cuh, plan kernel 5): bit-exact
with the float32 oracle (codeword, reported pm, attempt, path) on batches
of every compiled short shape, and equal to the float64 reference port's
codewords except on float32 near-ties."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("r,m", [(2, 5), (2, 6)])
@pytest.mark.parametrize("ebn0", [1.0, 3.0, 6.0])
def test_lane_kernel_matches_oracle(r, m, ebn0, oracle_mod):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code, is_codeword
    spec = build_code(r, m)
    x, llr = synthetic_frames(spec, ebn0, 20000, seed=7 + m)
    plan = Plan(r, m, 1, 1, False, "f32")
    assert plan.kernel == 5
    o = plan.decode(llr, diag=True)
    c = oracle_mod.decode(r, m, 1, 1, llr, None, perms=False, dtype=np.float32, nthreads=16)
    assert np.array_equal(o["cw"], c["cw"])
    assert np.array_equal(o["pm"], c["pm"])
    assert not o["attempt"].any() and not o["path"].any()
    assert np.array_equal(o["att_pm"][:, 0], o["pm"]) and np.array_equal(o["att_cw"][:, 0], o["cw"])
    # the float64 reference port: the same codewords except on float32 near-ties
    # of the FHT bin / SPC order (selection margin <= 1e-5, oracle/ties.py)
    c64 = oracle_mod.decode(r, m, 1, 1, llr.astype(np.float64), None, perms=False, dtype=np.float64, nthreads=16)
    differ = np.any(o["cw"] != c64["cw"], axis=1)
    assert np.all(c64["margin"][differ] <= 1e-5) and differ.sum() <= 20
    for f in range(0, 20000, 2000):
        assert is_codeword(spec, o["cw"][f])


def test_lane_kernel_exact_ties_fixture():
    """Integer LLRs: every FHT bin / SPC magnitude tie resolves like the
    reference (golden fixture made by the unmodified reference)."""
    from conftest import load_golden
    from paper_2108_12550_b200.decoder import Plan
    g = load_golden("rm25_fhtfsc_exact")
    plan = Plan(2, 5, 1, 1, False, "f32")
    o = plan.decode(g["llr"])
    assert np.array_equal(o["cw"], g["cw_bits"])
    assert np.array_equal(o["pm"].astype(np.float64), g["pm"])


# ---------------------------------------------------------------- pair kernel
@pytest.mark.parametrize("m,M", [(7, 4), (7, 1), (7, 2), (7, 8), (7, 16), (4, 4)])
def test_pair_kernel_matches_reference_order_kernel(m, M, oracle_mod):
    """Pair kernel (plan kernel 6: r = 2, L = 2, two threads per item) vs the
    reference-order float32 kernel and the float32 oracle (order
    "reference"): every output bit-exact, every attempt's pm and codeword
    included; M not dividing 16 binds the warp-per-item kernel instead."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, m)
    B = 1000 + 37
    _, llr = synthetic_frames(spec, 1.5, B, seed=m * 31 + M)
    plan = Plan(2, m, 2, M, True, "f32")
    assert plan.kernel == 6
    ref = Plan(2, m, 2, M, True, "f32", reference_order=True)
    assert ref.kernel == 1
    raw, rec = plan.sample(B, seed=9 + M)
    a = plan.decode(llr, records=rec, diag=True)
    b = ref.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        assert np.array_equal(a[k], b[k]), k
    c = oracle_mod.decode(2, m, 2, M, llr, raw, dtype=np.float32, nthreads=16)
    assert np.array_equal(a["cw"], c["cw"]) and np.array_equal(a["pm"], c["pm"])
    assert np.array_equal(a["attempt"], c["attempt"])


def test_pair_kernel_not_for_m_not_dividing_16():
    from paper_2108_12550_b200.decoder import Plan
    assert Plan(2, 7, 2, 3, True, "f32").kernel == 2
    assert Plan(2, 7, 2, 4, True, "f64").kernel == 1


def test_pair_kernel_honours_no_tie_fix(oracle_mod):
    """tie_fix=False (RMFHT_NO_TIE_FIX) on the pair kernel equals the
    reference-order kernel and the oracle without the tie fix."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    _, llr = synthetic_frames(build_code(2, 7), 2.0, 800, seed=5)
    a_plan = Plan(2, 7, 2, 4, True, "f32", tie_fix=False)
    assert a_plan.kernel == 6
    raw, rec = a_plan.sample(800, seed=3)
    a = a_plan.decode(llr, records=rec, diag=True)
    b = Plan(2, 7, 2, 4, True, "f32", tie_fix=False, reference_order=True).decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "att_pm"):
        assert np.array_equal(a[k], b[k]), k
    c = oracle_mod.decode(2, 7, 2, 4, llr, raw, dtype=np.float32, tie_fix=False, nthreads=16)
    assert np.array_equal(a["cw"], c["cw"]) and np.array_equal(a["pm"], c["pm"])
