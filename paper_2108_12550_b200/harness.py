"""Batched Monte Carlo FER harness on the GPU.

A drop-in for the reference's ``harness.run_job`` on the p-FHT-FSCL family
(``harness.py:116-165``): the same ``SimJob`` / ``FerRecord`` fields and CSV
schema (``harness.py:26-29,198-262``), the same stopping rule (after each
round of batches, stop once ``min_frame_errors`` is reached), the same
ML-lower-bound rule (``harness.py:79-84``).  Differences, by design:

* frames are decoded in GPU batches instead of 250-frame CPU chunks;
* frames are drawn per batch from counter-keyed generators (seed, point,
  batch) and permutation tables per frame from (seed, point, frame), so a
  run is identical for any number of ranks (the reference's
  worker-determinism property, ``test_acceptance.py:306-318``);
* ranks shard the batches (round-robin); the only collective is one sum
  of three counters per round (``torch.distributed``; NCCL or gloo).

``decode_fn`` is injectable for tests (e.g. the CPU oracle on gloo ranks);
the default is the CUDA decoder.
"""

from __future__ import annotations

import csv
import io
import json
import time
from dataclasses import asdict, dataclass
from math import ceil, log2

import numpy as np

from .channel_model import ChannelConfig
from .plan import complexity_ops, plan_visits, ssc_ops, ssc_steps
from .rm_core import ConfigurationError, build_code, polar_transform
from .top_decoders import SUPPORTED, DecoderConfig

CSV_HEADER = ["r", "m", "decoder", "L", "M", "P", "ebn0_db", "frames",
              "frame_errors", "fer", "ml_lb_fer", "avg_additions",
              "avg_comparisons", "time_steps", "mem_bits", "wall_seconds",
              "seed"]


@dataclass(frozen=True)
class SimJob:
    """harness.py:34-56 (plus the GPU batch size)."""
    r: int
    m: int
    decoder: DecoderConfig
    ebn0_points: tuple
    max_frames: int = 10000
    min_frame_errors: int = 100
    seed: int = 0
    workers: int = 1
    zero_noise: bool = False
    batch: int = 65536

    def __post_init__(self):
        if self.max_frames < 1:
            raise ConfigurationError("max_frames must be >= 1")
        pts = tuple(float(p) for p in self.ebn0_points)
        if not pts or any(b <= a for a, b in zip(pts, pts[1:])):
            raise ConfigurationError("ebn0_points must be nonempty and strictly increasing")
        object.__setattr__(self, "ebn0_points", pts)
        build_code(self.r, self.m)
        if self.decoder.algorithm not in SUPPORTED:
            raise ConfigurationError(f"algorithm {self.decoder.algorithm!r} is not part of this decoder "
                                     f"(supported: {', '.join(SUPPORTED)})")
        if self.batch < 1:
            raise ConfigurationError("batch must be >= 1")


@dataclass
class FerRecord:
    """harness.py:58-76"""
    r: int
    m: int
    decoder: str
    L: int
    M: int
    P: int
    ebn0_db: float
    frames: int
    frame_errors: int
    fer: float
    ml_lb_fer: float
    avg_additions: float
    avg_comparisons: float
    time_steps: int
    mem_bits: int
    wall_seconds: float
    seed: int


# --------------------------------------------------------------- cost model
# Restated from accounting.py for the supported family: the modeled figures
# the reference writes into every FerRecord.

def modeled_cost(r: int, m: int, cfg: DecoderConfig):
    """(ops, time_steps, mem_bits): complexity_model, latency_total,
    memory_model (accounting.py:189-227, 323-347)."""
    algo = cfg.algorithm
    if algo == "Aut-SSC":
        # accounting.py:195-197, 214-216, 338-339
        N, P = 1 << m, cfg.P
        steps = ssc_steps(r, m) + (int(ceil(log2(P))) if P > 1 else 0)
        return P * (ssc_ops(r, m) + N) + (P - 1), steps, (P + 1) * N * 32 + P * N
    perms = algo == "p-FHT-FSCL"
    ops = complexity_ops(r, m, cfg.L if algo != "FHT-FSC" else 1, cfg.M if perms else 1, perms,
                         include_perm=False, fsc=algo == "FHT-FSC")
    eff_l = 1 if algo == "FHT-FSC" else cfg.L

    def msteps(n):
        return int(ceil(log2(n))) if n > 1 else 0

    steps = 0
    for kind, mm in plan_visits(r, m, perms):
        n = 1 << mm
        if kind in ("f", "g"):
            steps += 1
        elif kind == "fht":
            steps += mm + msteps(eff_l * min(eff_l, n))
        elif kind == "spc":
            steps += mm if eff_l == 1 else mm + (min(eff_l, n) - 1) + msteps(2 * eff_l)
        elif kind == "perm":
            steps += 2 + msteps(2 * eff_l)
    steps += msteps(eff_l)
    if perms and cfg.M > 1:
        steps += msteps(cfg.M)
    N, Q, L, M = 1 << m, 32, cfg.L, cfg.M
    if algo == "FHT-FSC":
        mem = (2 * N - 1) * Q + N
    elif not perms:
        mem = N * (L + 1) * Q + 2 * L * Q + 2 * N * L
    elif L == 1 and M == 1:
        mem = (2 * N + 1) * Q + N
    elif L == 1:
        mem = (N + M * (N + 1)) * Q + M * N
    elif M == 1:
        mem = N * (L + 1) * Q + 2 * L * Q + 2 * N * L
    else:
        mem = N * (L * M + 1) * Q + 2 * M * L * Q + 2 * M * N * L
    return ops, steps, mem


def split_ops(r: int, m: int, cfg: DecoderConfig, total: int):
    """harness._split_ops (harness.py:172-195): additions vs comparisons."""
    if cfg.algorithm == "Aut-SSC":
        return total, 0  # no _ALGO_FLAGS entry: everything counts as additions
    perms = cfg.algorithm == "p-FHT-FSCL"  # the model follows the algorithm's flags (accounting._ALGO_FLAGS)
    eff_l = 1 if cfg.algorithm == "FHT-FSC" else cfg.L
    comps = 0
    for kind, mm in plan_visits(r, m, perms):
        if kind == "f":
            comps += eff_l * (1 << (mm - 1))
        elif kind == "fht":
            comps += eff_l * (1 << mm) + int(2 * eff_l * eff_l * np.log2(eff_l))
        elif kind == "spc":
            n = 1 << mm
            if eff_l == 1:
                comps += n
            else:
                tau = min(eff_l, n)
                comps += min(eff_l * mm * n, eff_l * eff_l * n) + int(2 * tau * eff_l * (1 + log2(eff_l)))
    comps = min(comps, total)
    return total - comps, comps


# ----------------------------------------------------------------- frames

def batch_frames(spec, chan: ChannelConfig, seed: int, point: int, batch_index: int, size: int,
                 zero_noise: bool = False):
    """Frames of one batch, keyed by (seed, point, batch): uniform info
    bits, polar encoding, BPSK + AWGN, float32 LLR = 2y/sigma^2."""
    rng = np.random.default_rng(np.random.SeedSequence((int(seed), int(point), int(batch_index), 0x4D43)))
    u = np.zeros((size, spec.N), dtype=np.uint8)
    u[:, list(spec.info_set)] = rng.integers(0, 2, size=(size, spec.K), dtype=np.uint8)
    x = polar_transform(u)
    y = 1.0 - 2.0 * x
    if not zero_noise:
        y = y + chan.sigma * rng.standard_normal((size, spec.N))
    return x, (2.0 * y / chan.sigma ** 2).astype(np.float32)


def _table_seed(seed: int, point: int) -> int:
    return (int(seed) * 1000003 + int(point) * 7919 + 0x5EED) & ((1 << 63) - 1)


class GpuDecoder:
    """Default decode_fn: the CUDA decoder with on-device permutation tables."""

    def __init__(self, spec, cfg: DecoderConfig, device=None):
        import torch
        from .decoder import Plan
        self.torch = torch
        if cfg.algorithm == "Aut-SSC":
            # P permutations drawn on the device, none of them the identity
            self.plan = Plan(spec.r, spec.m, 1, cfg.P, True, "f32", aut_ssc=True)
            self.perms, self.ident = True, False
        else:
            perms = cfg.algorithm == "p-FHT-FSCL" and cfg.permutations_enabled
            L = 1 if cfg.algorithm == "FHT-FSC" else cfg.L
            self.plan = Plan(spec.r, spec.m, L, cfg.M if perms else 1, perms, "f32")
            self.perms, self.ident = perms, True
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def __call__(self, llr: np.ndarray, table_seed: int, frame0: int):
        torch = self.torch
        d_llr = torch.from_numpy(llr).to(self.device)
        out = self.plan.alloc_outputs(llr.shape[0], self.device)
        if self.perms:
            self.plan.launch_sampled(d_llr, table_seed, out, frame0=frame0, identity_root=self.ident)
        else:
            self.plan.launch(d_llr, None, out)
        words = out["cw"].cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little")[:, :llr.shape[1]]
        return bits


def _allreduce(vals, group):
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group) if group is not None else dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(vals, dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return [int(v) for v in t.cpu().tolist()]


class DeviceSimulator:
    """The GPU pipeline of one job, with no host frames: per batch,
    rmfht_gen_frames -> decode (on-device permutation tables) ->
    rmfht_count_errors into a device counter."""

    def __init__(self, spec, cfg: DecoderConfig, batch: int, device=None):
        import torch
        self.torch, self.spec = torch, spec
        self.dec = GpuDecoder(spec, cfg, device)
        dev = self.dec.device
        self.llr = torch.empty((batch, spec.N), dtype=torch.float32, device=dev)
        self.tx = torch.empty((batch, self.dec.plan.words), dtype=torch.int32, device=dev)
        self.out = self.dec.plan.alloc_outputs(batch, dev)
        self.counts = torch.zeros(2, dtype=torch.int64, device=dev)
        self.work = self.dec.plan.alloc_workspace(batch, sampled=self.dec.perms, device=dev)

    def run_batch(self, chan: ChannelConfig, point: int, frame0: int, size: int, table_seed: int,
                  zero_noise: bool = False) -> None:
        """Queue one batch (stream-ordered; counts accumulate on the device)."""
        from .channel_model import count_errors_device, gen_frames_device
        llr, tx = self.llr[:size], self.tx[:size]
        out = {k: v[:size] for k, v in self.out.items()}
        gen_frames_device(self.spec, chan, point, frame0, llr, tx, zero_noise)
        if self.dec.perms:
            self.dec.plan.launch_sampled(llr, table_seed, out, frame0=frame0, identity_root=self.dec.ident,
                                         work=self.work)
        else:
            self.dec.plan.launch(llr, None, out, work=self.work)
        count_errors_device(self.spec, llr, tx, out["cw"], self.counts)

    def take_counts(self):
        """[frame errors, ML errors] since the last call (synchronises)."""
        c = [int(v) for v in self.counts.cpu().tolist()]
        self.counts.zero_()
        return c


def run_job(job: SimJob, decode_fn=None, rank: int = 0, world: int = 1, group=None,
            frames: str = "auto") -> list:
    """Simulate every SNR point; returns one FerRecord each (harness.py:116-165).

    frames="host": batches drawn on the host (batch_frames) and decoded by
    `decode_fn` (default: the CUDA decoder), errors counted on the host.
    frames="device": frames generated, decoded and counted on the GPU
    (DeviceSimulator; decode_fn must be None).  "auto" = device when
    decode_fn is None.  Batches are dealt round-robin over `world` ranks and
    the counts all-reduced after every round (early stop on
    min_frame_errors is then identical on every rank)."""
    spec = build_code(job.r, job.m)
    cfg = job.decoder
    ops, steps, mem = modeled_cost(job.r, job.m, cfg)
    adds, comps = split_ops(job.r, job.m, cfg, ops)
    if frames == "auto":
        frames = "device" if decode_fn is None else "host"
    if frames not in ("host", "device"):
        raise ConfigurationError(f"frames must be 'host', 'device' or 'auto', not {frames!r}")
    if frames == "device" and decode_fn is not None:
        raise ConfigurationError("frames='device' runs the CUDA decoder; decode_fn must be None")
    sim = None
    if frames == "device":
        sim = DeviceSimulator(spec, cfg, job.batch)
    elif decode_fn is None:
        decode_fn = GpuDecoder(spec, cfg)
    nb_total = -(-job.max_frames // job.batch)
    records = []
    for q, ebn0 in enumerate(job.ebn0_points):
        chan = ChannelConfig.for_rate(ebn0, spec.rate, job.seed)
        tseed = _table_seed(job.seed, q)
        t0 = time.monotonic()
        frames_n = errors = ml_errors = 0
        b = 0
        while b < nb_total:
            my = [bi for bi in range(b, min(b + world, nb_total)) if bi % world == rank]
            loc = [0, 0, 0]
            for bi in my:
                size = min(job.batch, job.max_frames - bi * job.batch)
                if sim is not None:
                    sim.run_batch(chan, q, bi * job.batch, size, tseed, job.zero_noise)
                    loc[0] += size
                    continue
                x, llr = batch_frames(spec, chan, job.seed, q, bi, size, job.zero_noise)
                xhat = decode_fn(llr, tseed, bi * job.batch)
                wrong = np.any(xhat != x, axis=1)
                if wrong.any():
                    a = llr[wrong].astype(np.float64)
                    c_hat = np.sum((1.0 - 2.0 * xhat[wrong]) * a, axis=1)   # correlation (top_decoders.py:231)
                    c_tx = np.sum((1.0 - 2.0 * x[wrong]) * a, axis=1)
                    ml = int(np.sum(c_hat >= c_tx))
                else:
                    ml = 0
                loc[0] += size
                loc[1] += int(wrong.sum())
                loc[2] += ml
            if sim is not None:
                e, ml = sim.take_counts()
                loc[1] += e
                loc[2] += ml
            if world > 1:
                loc = _allreduce(loc, group)
            frames_n += loc[0]
            errors += loc[1]
            ml_errors += loc[2]
            b += world
            if errors >= job.min_frame_errors:
                break
        wall = time.monotonic() - t0
        records.append(FerRecord(
            r=job.r, m=job.m, decoder=cfg.algorithm, L=cfg.L, M=cfg.M, P=cfg.P, ebn0_db=float(ebn0),
            frames=frames_n, frame_errors=errors, fer=errors / frames_n, ml_lb_fer=ml_errors / frames_n,
            avg_additions=float(adds), avg_comparisons=float(comps), time_steps=steps, mem_bits=mem,
            wall_seconds=wall, seed=job.seed))
    return records


# ------------------------------------------------------------ persistence
def _fmt(value):
    return repr(value) if isinstance(value, float) else value


def records_to_csv(records) -> str:
    """harness.py:198-206"""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for rec in records:
        row = asdict(rec)
        w.writerow([_fmt(row[k]) for k in CSV_HEADER])
    return buf.getvalue()


def records_to_json(records) -> str:
    return json.dumps([asdict(r) for r in records], indent=1)


def emit(records, path: str, fmt: str = "csv") -> None:
    """harness.py:220-229: write the records as CSV or JSON."""
    if fmt == "csv":
        text = records_to_csv(records)
    elif fmt == "json":
        text = records_to_json(records)
    else:
        raise ConfigurationError(f"unknown output format {fmt!r}")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)


def job_from_dict(cfg: dict) -> SimJob:
    """harness.py:248-262: a SimJob from the reference's job-file schema
    ({"code": [r, m], "decoder": {"algorithm", "L", "M", "P",
    "permutations_enabled"}, "ebn0_points", "max_frames",
    "min_frame_errors", "seed", "workers", "zero_noise"}), plus the optional
    GPU batch size "batch"."""
    dec = cfg["decoder"]
    decoder = DecoderConfig(algorithm=dec["algorithm"], L=int(dec.get("L", 1)), M=int(dec.get("M", 1)),
                            P=int(dec.get("P", 1)),
                            permutations_enabled=bool(dec.get("permutations_enabled", True)),
                            seed=int(cfg.get("seed", 0)))
    code = cfg["code"]
    extra = {"batch": int(cfg["batch"])} if "batch" in cfg else {}
    return SimJob(r=int(code[0]), m=int(code[1]), decoder=decoder, ebn0_points=tuple(cfg["ebn0_points"]),
                  max_frames=int(cfg.get("max_frames", 10000)),
                  min_frame_errors=int(cfg.get("min_frame_errors", 100)), seed=int(cfg.get("seed", 0)),
                  workers=int(cfg.get("workers", 1)), zero_noise=bool(cfg.get("zero_noise", False)), **extra)


def simulate(config_path: str, out: str | None = None, fmt: str = "csv", seed: int | None = None,
             workers: int | None = None, zero_noise: bool = False, rank: int = 0, world: int = 1,
             group=None) -> str:
    """The drop-in for ``rmwb simulate --config job.json`` (cli.py:46-63):
    read the reference-format job file, apply the same overrides, run the
    job on the GPU (run_job) and either write the records to ``out``
    (``emit``) or return them as CSV / JSON text.  ``workers`` is accepted
    and recorded for schema parity; the GPU decodes in batches instead."""
    with open(config_path, "r", encoding="utf-8") as fh:
        cfg = json.load(fh)
    if seed is not None:
        cfg["seed"] = seed
    if workers is not None:
        cfg["workers"] = workers
    if zero_noise:
        cfg["zero_noise"] = True
    records = run_job(job_from_dict(cfg), rank=rank, world=world, group=group)
    if out:
        if rank == 0:
            emit(records, out, fmt)
        return ""
    return records_to_csv(records) if fmt == "csv" else records_to_json(records)


def parse_csv(text: str) -> list:
    out = []
    for row in csv.DictReader(io.StringIO(text)):
        out.append(FerRecord(
            r=int(row["r"]), m=int(row["m"]), decoder=row["decoder"], L=int(row["L"]), M=int(row["M"]),
            P=int(row["P"]), ebn0_db=float(row["ebn0_db"]), frames=int(row["frames"]),
            frame_errors=int(row["frame_errors"]), fer=float(row["fer"]), ml_lb_fer=float(row["ml_lb_fer"]),
            avg_additions=float(row["avg_additions"]), avg_comparisons=float(row["avg_comparisons"]),
            time_steps=int(row["time_steps"]), mem_bits=int(row["mem_bits"]),
            wall_seconds=float(row["wall_seconds"]), seed=int(row["seed"])))
    return out


def clopper_pearson(k: int, n: int, alpha: float = 0.05):
    """Exact binomial interval (FER interval)."""
    from scipy.stats import beta
    lo = 0.0 if k == 0 else float(beta.ppf(alpha / 2, k, n - k + 1))
    hi = 1.0 if k == n else float(beta.ppf(1 - alpha / 2, k + 1, n - k))
    return lo, hi
