"""FER parity on the GPU: the batched harness against the reference's own
Monte Carlo (tests/golden/ref_fer.json, made by tools/ref_fer.py running the
unmodified rmworkbench.harness.run_job).  Frames and permutations are drawn
from different (equally distributed) streams, so the comparison is
statistical: Fisher's exact test on the two error counts must not reject at
the 1e-3 level, and the GPU FER must lie in the reference's 99.9%
Clopper-Pearson interval widened by the GPU's own."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
REF = json.load(open(os.path.join(GOLDEN, "ref_fer.json"))) if os.path.exists(os.path.join(GOLDEN, "ref_fer.json")) else None


@pytest.mark.skipif(REF is None, reason="reference FER fixture missing")
@pytest.mark.parametrize("name", sorted(REF["jobs"]) if REF else [])
def test_fer_matches_reference_monte_carlo(name):
    from scipy.stats import fisher_exact
    from paper_2108_12550_b200 import harness
    from paper_2108_12550_b200.top_decoders import DecoderConfig
    job = REF["jobs"][name]
    cfg = DecoderConfig(job["algorithm"], L=job["L"], M=job["M"], P=job.get("P", 1))
    pts = tuple(p["ebn0"] for p in job["points"])
    frames = max(200000, 4 * max(p["frames"] for p in job["points"]))
    recs = harness.run_job(harness.SimJob(r=job["r"], m=job["m"], decoder=cfg, ebn0_points=pts, max_frames=frames,
                                          min_frame_errors=10 ** 9, seed=2024, batch=65536))
    for rec, ref in zip(recs, job["points"]):
        p = fisher_exact([[rec.frame_errors, rec.frames - rec.frame_errors],
                          [ref["errors"], ref["frames"] - ref["errors"]]]).pvalue
        assert p > 1e-3, (name, rec.ebn0_db, rec.frame_errors, rec.frames, ref["errors"], ref["frames"])
        lo, hi = harness.clopper_pearson(ref["errors"], ref["frames"], alpha=1e-3)
        glo, ghi = harness.clopper_pearson(rec.frame_errors, rec.frames, alpha=1e-3)
        assert ghi >= lo and glo <= hi
        # ML lower bound (harness.py:79-84): same test on its counts
        ml, ref_ml = round(rec.ml_lb_fer * rec.frames), round(ref["ml_lb_fer"] * ref["frames"])
        p = fisher_exact([[ml, rec.frames - ml], [ref_ml, ref["frames"] - ref_ml]]).pvalue
        assert p > 1e-3, (name, rec.ebn0_db, ml, rec.frames, ref_ml, ref["frames"])


def test_gpu_harness_zero_noise_and_rank_invariance():
    from paper_2108_12550_b200 import harness
    from paper_2108_12550_b200.top_decoders import DecoderConfig
    cfg = DecoderConfig("p-FHT-FSCL", L=4, M=20)
    rec = harness.run_job(harness.SimJob(r=2, m=9, decoder=cfg, ebn0_points=(3.0,), max_frames=5000,
                                         zero_noise=True, batch=2048))[0]
    assert rec.frame_errors == 0 and rec.frames == 5000
    # the same frames split into other batch rounds give the same counts
    a = harness.run_job(harness.SimJob(r=2, m=7, decoder=DecoderConfig("p-FHT-FSCL", L=2, M=4), ebn0_points=(2.0,),
                                       max_frames=20000, min_frame_errors=10 ** 9, batch=4000))[0]
    b = harness.run_job(harness.SimJob(r=2, m=7, decoder=DecoderConfig("p-FHT-FSCL", L=2, M=4), ebn0_points=(2.0,),
                                       max_frames=20000, min_frame_errors=10 ** 9, batch=2500))[0]
    assert (a.frames, a.frame_errors, a.ml_lb_fer) == (b.frames, b.frame_errors, b.ml_lb_fer)
    # (frames and permutation tables are keyed by the frame index, not by the batch that draws them)
    c = harness.run_job(harness.SimJob(r=2, m=9, decoder=DecoderConfig("p-FHT-FSCL", L=1, M=512), ebn0_points=(2.0,),
                                       max_frames=3000, min_frame_errors=10 ** 9, batch=1000))[0]
    d = harness.run_job(harness.SimJob(r=2, m=9, decoder=DecoderConfig("p-FHT-FSCL", L=1, M=512), ebn0_points=(2.0,),
                                       max_frames=3000, min_frame_errors=10 ** 9, batch=768))[0]
    assert (c.frames, c.frame_errors, c.ml_lb_fer) == (d.frames, d.frame_errors, d.ml_lb_fer)
