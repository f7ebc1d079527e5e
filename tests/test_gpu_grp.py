"""Lane-group kernel (rmfht_grp.cuh, plan kernel 7: p-FHT-FSCL with r = 2,
L = 1, four attempts of a frame per warp) against the throughput kernel
(plan kernel 2, bound when RMFHT_NO_GRP is set) and the float32 oracle in
the throughput kernel's summation order: every output bit-exact, every
attempt's reported pm and codeword included."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _throughput_plan(*a):
    from paper_2108_12550_b200.decoder import Plan
    os.environ["RMFHT_NO_GRP"] = "1"
    try:
        return Plan(*a)
    finally:
        del os.environ["RMFHT_NO_GRP"]


@pytest.mark.parametrize("M,B,ebn0", [(4, 3001, 1.0), (8, 1500, 2.0), (20, 700, 0.0), (512, 40, 3.0), (64, 257, 4.0)])
def test_grp_kernel_matches_throughput_kernel_and_oracle(M, B, ebn0, oracle_mod):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code, is_codeword
    spec = build_code(2, 9)
    _, llr = synthetic_frames(spec, ebn0, B, seed=100 + M)
    plan = Plan(2, 9, 1, M, True, "f32")
    assert plan.kernel == 7
    ref = _throughput_plan(2, 9, 1, M, True, "f32")
    assert ref.kernel == 2
    raw, rec = plan.sample(B, seed=3 + M, identity_root=(M % 8 == 0))
    a = plan.decode(llr, records=rec, diag=True)
    b = ref.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        assert np.array_equal(a[k], b[k]), k
    n = min(B, 400)
    c = oracle_mod.decode(2, 9, 1, M, llr[:n], raw[:n], dtype=np.float32, nthreads=16, order="v2")
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        assert np.array_equal(a[k][:n], c[k]), k
    for f in range(0, B, max(1, B // 8)):
        assert is_codeword(spec, a["cw"][f])


def test_grp_kernel_sampled_launch_matches_table_launch():
    """The device-drawn table path (rmfht_decode_launch_sampled) through the
    lane-group kernel equals decoding the same table drawn explicitly."""
    import torch
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    B = 96
    _, llr = synthetic_frames(spec, 3.0, B, seed=5)
    plan = Plan(2, 9, 1, 512, True, "f32")
    assert plan.kernel == 7
    out = plan.alloc_outputs(B)
    plan.launch_sampled(torch.from_numpy(llr).cuda(), 77, out)
    torch.cuda.synchronize()
    _, rec = plan.sample(B, seed=77)
    o = plan.decode(llr, records=rec)
    assert np.array_equal(out["cw"].cpu().numpy().view(np.uint32), o["cw_packed"])
    assert np.array_equal(out["attempt"].cpu().numpy(), o["attempt"])


def test_grp_kernel_only_when_attempts_divide():
    from paper_2108_12550_b200.decoder import Plan
    assert Plan(2, 9, 1, 6, True, "f32").kernel == 2
    assert Plan(2, 9, 1, 512, True, "f64").kernel == 1
    assert Plan(2, 9, 1, 1, False, "f32").kernel == 2  # FHT-FSC: no permutations


@pytest.mark.parametrize("M,B", [(4, 2000), (16, 600)])
def test_grp_kernel_rm28(M, B, oracle_mod):
    """The m = 8 instantiation (N = 256): against the throughput kernel and the oracle."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 8)
    _, llr = synthetic_frames(spec, 2.0, B, seed=40 + M)
    plan = Plan(2, 8, 1, M, True, "f32")
    assert plan.kernel == 7
    ref = _throughput_plan(2, 8, 1, M, True, "f32")
    assert ref.kernel == 2
    raw, rec = plan.sample(B, seed=M)
    a = plan.decode(llr, records=rec, diag=True)
    b = ref.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        assert np.array_equal(a[k], b[k]), k
    c = oracle_mod.decode(2, 8, 1, M, llr[:300], raw[:300], dtype=np.float32, nthreads=16, order="v2")
    for k in ("cw", "pm", "attempt", "att_pm"):
        assert np.array_equal(a[k][:300], c[k]), k


@pytest.mark.parametrize("B", [1, 2, 3, 33])
def test_grp_kernel_small_and_ragged_batches(B):
    """Batches smaller than a CTA round and not a multiple of anything: every
    frame still gets its own answer (against the throughput kernel)."""
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    _, llr = synthetic_frames(spec, 1.0, B, seed=B)
    for M in (4, 512):
        plan = Plan(2, 9, 1, M, True, "f32")
        ref = _throughput_plan(2, 9, 1, M, True, "f32")
        assert (plan.kernel, ref.kernel) == (7, 2)
        _, rec = plan.sample(B, seed=B + M)
        a = plan.decode(llr, records=rec, diag=True)
        b = ref.decode(llr, records=rec, diag=True)
        for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
            assert np.array_equal(a[k], b[k]), (k, M)
