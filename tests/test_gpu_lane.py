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
