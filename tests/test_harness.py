"""Harness on the CPU: validation, cost model, CSV, and the
multi-rank path on gloo (world size 2 == world size 1, byte for byte).
The decode function here is the CPU oracle (test infrastructure); the
product harness uses the CUDA decoder (tests/test_gpu_fer.py)."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2108_12550_b200 import harness
from paper_2108_12550_b200.rm_core import ConfigurationError, build_code
from paper_2108_12550_b200.top_decoders import DecoderConfig


class OracleDecode:
    def __init__(self, spec, cfg):
        from oracle import oracle
        from paper_2108_12550_b200.decoder import Plan
        self.oracle = oracle
        self.spec, self.cfg = spec, cfg
        self.perms = cfg.algorithm == "p-FHT-FSCL" and cfg.permutations_enabled
        self.L = 1 if cfg.algorithm == "FHT-FSC" else cfg.L
        self.M = cfg.M if self.perms else 1
        self.plan = Plan(spec.r, spec.m, self.L, self.M, self.perms, "f32")

    def __call__(self, llr, table_seed, frame0):
        raw = None
        if self.perms:
            raw, _ = self.plan.sample(llr.shape[0], table_seed, frame0=frame0, identity_root=True,
                                      want_records=False)
        o = self.oracle.decode(self.spec.r, self.spec.m, self.L, self.M, llr, raw, perms=self.perms,
                               dtype=np.float32, order="v2" if self.perms and self.spec.m >= 5 else "reference",
                               nthreads=4, want_attempts=False)
        return o["cw"]


def _job(**kw):
    base = dict(r=2, m=5, decoder=DecoderConfig("p-FHT-FSCL", L=4, M=2), ebn0_points=(1.0, 2.0),
                max_frames=600, min_frame_errors=10 ** 9, seed=11, batch=100)
    base.update(kw)
    return harness.SimJob(**base)


def test_job_validation():
    for kw in (dict(ebn0_points=()), dict(ebn0_points=(2.0, 1.0)), dict(max_frames=0), dict(r=0),
               dict(decoder=DecoderConfig("SC"))):
        with pytest.raises(ConfigurationError):
            _job(**kw)


def test_frames_mode_validation():
    spec = build_code(2, 5)
    cfg = DecoderConfig("p-FHT-FSCL", L=4, M=2)
    with pytest.raises(ConfigurationError):
        harness.run_job(_job(), decode_fn=OracleDecode(spec, cfg), frames="device")
    with pytest.raises(ConfigurationError):
        harness.run_job(_job(), decode_fn=OracleDecode(spec, cfg), frames="disk")


def test_modeled_costs_match_reference():
    path = os.path.join(GOLDEN, "ref_fer.json")
    if not os.path.exists(path):
        pytest.skip("reference FER fixture not generated")
    ref = json.load(open(path))
    for name, job in ref["jobs"].items():
        cfg = DecoderConfig(job["algorithm"], L=job["L"], M=job["M"], P=job.get("P", 1))
        ops, steps, mem = harness.modeled_cost(job["r"], job["m"], cfg)
        c = ref["costs"][name]
        assert (ops, steps, mem) == (c["ops"], c["steps"], c["mem"]), name
        assert harness.split_ops(job["r"], job["m"], cfg, ops) == (c["adds"], c["comps"]), name


def test_zero_noise_gives_zero_fer():
    spec = build_code(2, 5)
    for cfg in (DecoderConfig("p-FHT-FSCL", L=4, M=2), DecoderConfig("FHT-FSCL", L=4), DecoderConfig("FHT-FSC")):
        job = _job(decoder=cfg, zero_noise=True, ebn0_points=(3.0,), max_frames=250)
        rec = harness.run_job(job, decode_fn=OracleDecode(spec, cfg))[0]
        assert rec.frames == 250 and rec.frame_errors == 0 and rec.fer == 0.0


def test_stopping_rule_and_csv_round_trip(tmp_path):
    spec = build_code(2, 5)
    job = _job(ebn0_points=(-1.0,), max_frames=5000, min_frame_errors=5)
    recs = harness.run_job(job, decode_fn=OracleDecode(spec, job.decoder))
    assert recs[0].frame_errors >= 5 and recs[0].frames < 5000
    text = harness.records_to_csv(recs)
    assert text.splitlines()[0] == ",".join(harness.CSV_HEADER)
    assert harness.parse_csv(text) == recs
    json.loads(harness.records_to_json(recs))


def test_clopper_pearson():
    lo, hi = harness.clopper_pearson(1, 80000)
    assert abs(lo - 3.16e-7) < 1e-8 and abs(hi - 6.96e-5) < 1e-6
    assert harness.clopper_pearson(0, 100)[0] == 0.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = _job()
    recs = harness.run_job(job, decode_fn=OracleDecode(build_code(job.r, job.m), job.decoder), rank=rank, world=world)
    out_q.put((rank, [r.__dict__ | {"wall_seconds": 0.0} for r in recs]))
    dist.destroy_process_group()


def test_two_ranks_gloo_equal_one_rank():
    import torch.multiprocessing as mp
    job = _job()
    one = [r.__dict__ | {"wall_seconds": 0.0}
           for r in harness.run_job(job, decode_fn=OracleDecode(build_code(job.r, job.m), job.decoder))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got[0] == one and got[1] == one


# ------------------------------------------------ job files and persistence
# the reference's documented job file (pkg/README.md "Command line"), the
# golden_fer.csv acceptance run
JOB_JSON = {"code": [2, 6], "decoder": {"algorithm": "p-FHT-FSCL", "L": 4}, "ebn0_points": [2.0, 2.5],
            "max_frames": 30000, "min_frame_errors": 1000000000, "seed": 777, "workers": 2}


def test_job_from_dict_reference_schema():
    """harness.py:248-262 field by field."""
    job = harness.job_from_dict(JOB_JSON)
    assert (job.r, job.m) == (2, 6)
    assert job.decoder == DecoderConfig("p-FHT-FSCL", L=4, M=1, P=1, permutations_enabled=True, seed=777)
    assert job.ebn0_points == (2.0, 2.5) and job.max_frames == 30000
    assert job.min_frame_errors == 10 ** 9 and job.seed == 777 and job.workers == 2 and not job.zero_noise
    j2 = harness.job_from_dict({"code": [2, 9], "decoder": {"algorithm": "p-FHT-FSCL", "L": 4, "M": 20,
                                                             "permutations_enabled": False},
                                "ebn0_points": [3.0], "batch": 4096})
    assert j2.decoder.M == 20 and not j2.decoder.permutations_enabled and j2.batch == 4096
    assert j2.max_frames == 10000 and j2.min_frame_errors == 100 and j2.seed == 0
    with pytest.raises(ConfigurationError):
        harness.job_from_dict({"code": [2, 9], "decoder": {"algorithm": "p-FHT-FSCL", "L": 0},
                               "ebn0_points": [3.0]})
    with pytest.raises(ConfigurationError):
        harness.job_from_dict({"code": [2, 9], "decoder": {"algorithm": "p-FHT-FSCL"}, "ebn0_points": [3.0, 2.0]})


def test_emit_csv_json_roundtrip(tmp_path):
    """harness.py:198-229: emit writes what records_to_csv / _json return;
    the CSV parses back to the same records; unknown formats raise."""
    recs = [harness.FerRecord(r=2, m=6, decoder="p-FHT-FSCL", L=4, M=1, P=1, ebn0_db=2.0, frames=30000,
                              frame_errors=748, fer=748 / 30000, ml_lb_fer=629 / 30000, avg_additions=1252.0,
                              avg_comparisons=832.0, time_steps=46, mem_bits=11008, wall_seconds=0.25, seed=777)]
    p = tmp_path / "r.csv"
    harness.emit(recs, str(p), "csv")
    text = p.read_text()
    assert text == harness.records_to_csv(recs)
    assert text.splitlines()[0] == ",".join(harness.CSV_HEADER)
    assert harness.parse_csv(text) == recs
    q = tmp_path / "r.json"
    harness.emit(recs, str(q), "json")
    assert json.loads(q.read_text())[0]["frame_errors"] == 748
    with pytest.raises(ConfigurationError):
        harness.emit(recs, str(tmp_path / "r.txt"), "xml")
