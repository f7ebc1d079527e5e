"""C-ABI contract on the GPU (include/rmfht.h conventions; VERDICT r1 /
ADVICE r1): caller-owned workspace, no plan-owned device state, so one plan
launched concurrently on two streams with different batches gives results
bit-identical to serial launches; workspace errors are ValueError-class."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _frames(r, m, ebn0, B, seed):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.rm_core import build_code
    return synthetic_frames(build_code(r, m), ebn0, B, seed)[1]


@pytest.mark.parametrize("r,m,L,M", [(2, 9, 4, 20), (2, 7, 2, 4), (3, 7, 8, 32)])
def test_one_plan_two_streams_concurrently(r, m, L, M):
    import torch
    from paper_2108_12550_b200.decoder import Plan
    plan = Plan(r, m, L, M, True, "f32")
    sizes = (3000, 1700)
    llrs = [torch.from_numpy(_frames(r, m, 2.5, n, 40 + i)).cuda() for i, n in enumerate(sizes)]
    seeds = (11, 12)
    # serial reference results
    ref = []
    for llr, sd in zip(llrs, seeds):
        o = plan.alloc_outputs(llr.shape[0])
        plan.launch_sampled(llr, sd, o, frame0=0)
        torch.cuda.synchronize()
        ref.append({k: v.cpu().clone() for k, v in o.items()})
    # the same plan on two streams at once, repeatedly, each with its own workspace
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    works = [plan.alloc_workspace(llr.shape[0], sampled=True, stream=st) for llr, st in zip(llrs, streams)]
    outs = [plan.alloc_outputs(llr.shape[0]) for llr in llrs]
    torch.cuda.synchronize()
    for _ in range(4):
        for llr, sd, o, st, w in zip(llrs, seeds, outs, streams, works):
            plan.launch_sampled(llr, sd, o, frame0=0, stream=st, work=w)
    torch.cuda.synchronize()
    for o, rf in zip(outs, ref):
        for k in ("cw", "pm", "attempt", "path"):
            assert torch.equal(o[k].cpu(), rf[k]), k


def test_workspace_too_small_is_value_error():
    import torch
    from paper_2108_12550_b200.decoder import Plan
    plan = Plan(2, 9, 4, 20, True, "f32")
    llr = torch.from_numpy(_frames(2, 9, 2.5, 64, 3)).cuda()
    out = plan.alloc_outputs(64)
    small = torch.empty(plan.workspace_bytes(64, sampled=True) - 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="workspace"):
        plan.launch_sampled(llr, 1, out, work=small)
    # NULL workspace through the raw ABI
    lib = plan._lib
    rc = lib.rmfht_decode_launch_sampled(plan._h, llr.data_ptr(), ctypes.c_uint64(1), 0, 1,
                                         out["cw"].data_ptr(), out["pm"].data_ptr(), out["attempt"].data_ptr(),
                                         out["path"].data_ptr(), 64, None, 0, None)
    assert rc == -2


def test_att_cw_without_att_pm():
    """att_cw is written even when att_pm is NULL."""
    import torch
    from paper_2108_12550_b200.decoder import Plan
    plan = Plan(2, 9, 4, 20, True, "f32")
    B = 50
    llr = _frames(2, 9, 2.5, B, 5)
    _, rec = plan.sample(B, seed=9)
    full = plan.decode(llr, records=rec, diag=True)
    d_llr = torch.from_numpy(llr).cuda()
    d_rec = torch.from_numpy(rec.view(np.int16)).cuda()
    out = plan.alloc_outputs(B, diag=True)
    out["att_cw"].fill_(-1)
    w = plan.alloc_workspace(B)
    st = torch.cuda.current_stream()
    rc = plan._lib.rmfht_decode_launch_diag(
        plan._h, d_llr.data_ptr(), d_rec.data_ptr(), out["cw"].data_ptr(), out["pm"].data_ptr(),
        out["attempt"].data_ptr(), out["path"].data_ptr(), None, out["att_cw"].data_ptr(), B, w.data_ptr(),
        w.numel(), st.cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert np.array_equal(out["att_cw"].cpu().numpy().view(np.uint32), full["att_cw_packed"])


def test_free_running_warps_decode_the_same():
    """RMFHT_LOCKSTEP_GROUP=0 (A/B hook: no round barrier in the throughput
    kernel) changes the schedule, not the results."""
    import os
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    _, llr = synthetic_frames(spec, 2.0, 700, seed=21)
    plan = Plan(2, 9, 4, 20, True, "f32")
    os.environ["RMFHT_LOCKSTEP_GROUP"] = "0"
    try:
        free = Plan(2, 9, 4, 20, True, "f32")
    finally:
        del os.environ["RMFHT_LOCKSTEP_GROUP"]
    _, rec = plan.sample(700, seed=8)
    a = plan.decode(llr, records=rec, diag=True)
    b = free.decode(llr, records=rec, diag=True)
    for k in ("cw", "pm", "attempt", "path", "att_pm", "att_cw"):
        assert np.array_equal(a[k], b[k]), k
