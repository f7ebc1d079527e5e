"""Throughput of the batched p-FHT-FSCL-L-M decoder on B200.

Workload (BASELINE.json headline): RM(2,9), M=20 affine automorphisms
(decoder 0's root maps = identity), L=4, BPSK/AWGN float32 LLRs at
Eb/N0 = 2.5 dB.  One step = one pass of the hot path over a batch of
frames resident in HBM (larger than the 126 MB L2, so no flush is needed
between steps): on-device permutation sampling + decode + per-frame pick.

  value     decoded frames/s of the whole job (sum over ranks / max time)
  e2e       same metric through the public API with host buffers
            (decoder.StreamDecoder -> rmfht_decode_launch_sampled): pinned
            host LLRs copied in and codewords / PM / attempt copied out
            every step; permutations are drawn on the device, so no table
            crosses the host link
  roofline  reference op ledger (accounting.complexity_model, include_perm)
            per frame x frames/s against the FP32 issue peak
            (SMs x 128 lanes x max SM clock); HBM bound alongside
  cpu_baseline  the float64 C port of the reference (oracle/) on this host's
            cores over a bounded sample: the first frames of the GPU's own
            batch under the same permutation table, so the same sample also
            yields ``ties`` — the tie accounting of the GPU's answers against
            the port (oracle/ties.py)
  cpu_baseline_reference  the UNMODIFIED Python reference
            (baseline/_ref: rmworkbench.harness._simulate_chunk, its stock
            per-frame path) on all host cores, bounded sample

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, frames sharded, seeds
distinct per rank, no data-path collective).  --dry-run runs the same
launch/timing plumbing on CPU ranks (gloo) with a stand-in step (tests).

--impl reference times the CPU restatement of the reference decoder (the
reference is pure Python with no native path; the float64 C port is its CPU
implementation here) on the same config, rank 0 only, and reports the
unmodified Python reference beside it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configurations: name -> (r, m, L, M, permutations, Eb/N0, frames per step)
CONFIGS = {
    "rm29_L4_M20": (2, 9, 4, 20, True, 2.5, 32768),   # headline
    "rm27_L2_M4": (2, 7, 2, 4, True, 2.0, 262144),
    "rm37_L8_M32": (3, 7, 8, 32, True, 4.0, 16384),
    "rm29_L1_M512": (2, 9, 1, 512, True, 3.0, 1024),
    "rm25_fhtfsc": (2, 5, 1, 1, False, 3.0, 4194304),
    # the paper's Table IV comparator, Aut-SSC with P = 512 (M = P here)
    "rm29_autssc_P512": (2, 9, 1, 512, "aut", 2.5, 2048),
}
R, M_VARS, L, M = 2, 9, 4, 20
PERMS = True
AUT = False
EBN0 = 2.5
WORKLOAD = "RM(2,9) p-FHT-FSCL L=4 M=20 (decoder 0 = identity), Eb/N0 2.5 dB"
METRIC = "decoded frames/s, RM(2,9) M=20 L=4, 1 B200; % of roofline; vs host CPU"


CURRENT = "rm29_L4_M20"


def select_config(name):
    global R, M_VARS, L, M, PERMS, AUT, EBN0, WORKLOAD, CURRENT
    CURRENT = name
    r, m, l, mm, perms, ebn0, frames = CONFIGS[name]
    AUT = perms == "aut"
    R, M_VARS, L, M, PERMS, EBN0 = r, m, l, mm, bool(perms), ebn0
    algo = "Aut-SSC" if AUT else "p-FHT-FSCL" if perms else ("FHT-FSC" if l == 1 else "FHT-FSCL")
    if AUT:
        WORKLOAD = f"RM({r},{m}) Aut-SSC P={mm}, Eb/N0 {ebn0} dB"
    else:
        WORKLOAD = (f"RM({r},{m}) {algo} L={l} M={mm}" + (" (decoder 0 = identity)" if perms else "") +
                    f", Eb/N0 {ebn0} dB")
    global METRIC
    if name != "rm29_L4_M20":
        METRIC = (f"decoded frames/s, RM({r},{m}) Aut-SSC P={mm}, 1 B200" if AUT else
                  f"decoded frames/s, RM({r},{m}) {algo} L={l} M={mm}, 1 B200")
    return frames


def _capture(config):
    """The dominant kernel's ncu figures for this config (profiles/r2_traffic.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as fh:
            return json.load(fh)[config]
    except Exception:
        return {}


def _traffic(config, frames):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture
    (scaled from the captured launch's frame count to this launch's), or None."""
    d = _capture(config)
    if "dram_read_bytes" not in d:
        return None
    return (d["dram_read_bytes"] + d["dram_write_bytes"]) * frames / d["frames_per_launch"]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6536.4)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def wait_first(self, timeout: float = 3.0):
        """Block until nvidia-smi has delivered its first row (its start-up
        takes longer than a short timed region)."""
        t0 = time.time()
        while self.proc is not None and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8
                          for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _relaunch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run with N
    ranks on 127.0.0.1 (the driver's own launch line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def make_inputs(plan, spec, B, seed):
    """Frames and permutation records for one batch (host)."""
    from paper_2108_12550_b200.channel_model import synthetic_frames

    x, llr = synthetic_frames(spec, EBN0, B, seed)
    recs = None
    if plan.permutations:
        _, recs = plan.sample(B, seed, identity_root=not AUT, want_raw=False)
    return x, llr, recs


def _cpu_batches(B, count, seed0):
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.plan import map_sizes
    from paper_2108_12550_b200.automorphism import random_raw_table
    from paper_2108_12550_b200.rm_core import build_code

    spec = build_code(R, M_VARS)
    out = []
    for s in range(count):
        _, llr = synthetic_frames(spec, EBN0, B, seed0 + s)
        sizes = [M_VARS] if AUT else map_sizes(R, M_VARS, L)
        raw = (random_raw_table(np.random.default_rng(seed0 + s), (B, M), sizes, M_VARS,
                                identity_root=0 if AUT else L) if PERMS else None)
        out.append((llr, raw))
    return out


def _cpu_decode(llr, raw, cores, want_attempts=False):
    from oracle import oracle
    if AUT:
        return oracle.aut_ssc(R, M_VARS, M, llr, raw[:, :, 0, :], dtype=np.float64, nthreads=cores)
    return oracle.decode(R, M_VARS, L, M if PERMS else 1, llr.astype(np.float64), raw, perms=PERMS,
                         dtype=np.float64, nthreads=cores, want_attempts=want_attempts)


def cpu_baseline(plan, llr, x, gpu, seed, seconds: float = 12.0):
    """The float64 C port (oracle/) on all host cores over a bounded sample:
    the first frames of the GPU's batch with the same permutation table
    (plan.sample(seed) = the table the device drew), so the same decodes give
    the tie accounting of the GPU's answers against the port (oracle/ties.py).
    Returns (cpu_baseline, ties)."""
    from oracle import ties as T
    cores = os.cpu_count() or 1
    B = llr.shape[0]
    cmax = max(16, (1 << 26) // max(1, M * (1 << M_VARS)))  # bounds the per-attempt outputs of a chunk
    C = min(cmax, 4 * cores)  # the first chunk calibrates the rest to ~1/6 of the budget each
    frames, t_used, parts, c0 = 0, 0.0, [], 0
    while c0 < B and t_used < seconds:
        c1 = min(B, c0 + C)
        raw = None
        if PERMS:
            raw, _ = plan.sample(c1 - c0, seed, frame0=c0, identity_root=not AUT, want_records=False)
        t0 = time.perf_counter()
        p = _cpu_decode(llr[c0:c1], raw, cores, want_attempts=not AUT)
        t_used += time.perf_counter() - t0
        if not AUT:
            parts.append(T.classify(gpu["cw"][c0:c1], gpu["pm"][c0:c1], gpu["attempt"][c0:c1], p, x=x[c0:c1]))
        frames += c1 - c0
        c0 = c1
        C = max(16, min(cmax, int(frames * (seconds / 6) / max(t_used, 1e-6))))
    base = {"value": frames / t_used, "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"frames 0..{frames - 1} of the GPU's batch under the same permutation table, float64 "
                      f"C port of the reference (oracle/), {cores} threads, {t_used:.1f} s"}
    tie = None
    if parts:
        tie = T.merge(parts)
        tie["ok"] = T.ok(tie)
        tie["note"] = ("GPU float32 vs float64 port on the same float32 LLRs and table (oracle/ties.py): "
                       "codeword mismatches must sit on frames with a selection margin <= rel, attempt "
                       "mismatches must be pm-equivalent (same codeword, pm within rel) or on such frames; "
                       "ens_exact_ties = frames whose minimum pm is reached by >= 2 attempts")
    return base, tie


def _ref_cfg():
    from rmworkbench.top_decoders import DecoderConfig
    if AUT:
        return DecoderConfig("Aut-SSC", P=M)
    if not PERMS:
        return DecoderConfig("FHT-FSC" if L == 1 else "FHT-FSCL", L=L)
    return DecoderConfig("p-FHT-FSCL", L=L, M=M)


def _ref_chunk(a):
    sys.path.insert(0, a[0])
    from rmworkbench import rm_core
    from rmworkbench.channel_model import ChannelConfig
    from rmworkbench.harness import SimJob, _simulate_chunk
    job = SimJob(r=R, m=M_VARS, decoder=_ref_cfg(), ebn0_points=(EBN0,), max_frames=a[2], seed=777)
    spec = rm_core.build_code(R, M_VARS)
    chan = ChannelConfig.for_rate(EBN0, spec.rate, 777)
    t0 = time.perf_counter()
    err, ml = _simulate_chunk(job, spec, chan, 0, a[1], a[2])
    return err, ml, time.perf_counter() - t0


def cpu_baseline_reference(seconds: float = 12.0):
    """The UNMODIFIED Python reference (baseline/_ref, installed from
    /root/reference) on all host cores: its stock per-frame harness path
    rmworkbench.harness._simulate_chunk (frame generation, decode, error
    count; harness.py:94-113) over a bounded sample, one chunk per core."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "rmworkbench")):
        return {"unavailable": "baseline/_ref is not installed (pip install --target baseline/_ref, DESIGN.md)"}
    from concurrent.futures import ProcessPoolExecutor
    cores = os.cpu_count() or 1
    try:
        e, ml, dt = _ref_chunk((ref, 0, 1))  # calibration: one frame in-process (also warms the imports)
    except Exception as ex:  # noqa: BLE001
        return {"unavailable": f"reference import failed: {ex!r}"}
    per = max(1, int(seconds / max(dt, 1e-4)))
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores, initializer=_select_in_worker, initargs=(CURRENT,)) as ex:
        res = list(ex.map(_ref_chunk, [(ref, 1 + c * per, per) for c in range(cores)]))
    wall = time.perf_counter() - t0
    frames = per * cores
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except Exception:  # noqa: BLE001
        pass
    return {"value": frames / wall, "unit": "frames/s", "cores": cores, "kind": "reference", "cpu": cpu,
            "sample": f"{frames} frames ({cores} processes x {per}) of the reference harness stream "
                      f"frame_rng(777, 0, k) through the unmodified Python reference "
                      f"(baseline/_ref rmworkbench.harness._simulate_chunk), wall {wall:.1f} s incl. process "
                      f"start; frame errors {sum(r[0] for r in res)}"}


def _select_in_worker(name):
    select_config(name)


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # bounded per-step sample: ~1.5 s of CPU work per step
    (llr, raw), = _cpu_batches(16 * cores, 1, 400)
    t0 = time.perf_counter()
    _cpu_decode(llr, raw, cores)
    B = max(16 * cores, int(16 * cores * 1.5 / max(time.perf_counter() - t0, 1e-3)))
    batches = _cpu_batches(B, args.steps + args.warmup, 500)
    for llr, raw in batches[:args.warmup]:
        _cpu_decode(llr, raw, cores)
    t0 = time.perf_counter()
    for llr, raw in batches[args.warmup:]:
        _cpu_decode(llr, raw, cores)
    dt = time.perf_counter() - t0
    v = B * args.steps / dt
    line = {"metric": METRIC, "value": v, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "frames_per_step": B},
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "port",
                             "sample": f"{B} frames per step x {args.steps} steps, float64 CPU restatement "
                                       f"of the reference decoder (oracle/), {cores} threads"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_cpu:
        line["reference_python"] = cpu_baseline_reference(args.cpu_seconds)
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    comm = 1
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = dist.get_world_size()
        if rank == 0:
            print(f"bench: NCCL communicator of {comm} ranks", file=sys.stderr, flush=True)
    from paper_2108_12550_b200.decoder import Plan
    from paper_2108_12550_b200.plan import complexity_ops
    from paper_2108_12550_b200.rm_core import build_code

    spec = build_code(R, M_VARS)
    plan = Plan(R, M_VARS, L, M, PERMS, "f32", lockstep=0 if args.no_lockstep else args.lockstep, aut_ssc=AUT)
    B = args.frames
    x, llr, recs = make_inputs(plan, spec, B, seed=1 + rank)  # host table: decode-only timing
    dev = torch.device("cuda", local)
    d_llr = torch.from_numpy(llr).to(dev)
    d_rec = torch.from_numpy(recs.view(np.int16)).to(dev) if recs is not None else None
    out = plan.alloc_outputs(B, dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    SEED = 1 + rank
    # caller-owned workspaces (rmfht_workspace_bytes), allocated once
    work_s = plan.alloc_workspace(B, sampled=True, device=dev, stream=stream)
    work_d = plan.alloc_workspace(B, sampled=False, device=dev, stream=stream)

    def step():
        # one pass of the hot path: draw the batch's permutations on the device
        # (the reference samples them inside decode) and decode
        plan.launch_sampled(d_llr, SEED, out, frame0=0, identity_root=not AUT, stream=stream, work=work_s)

    for _ in range(args.warmup):
        step()
    barrier()
    # correctness spot check of the warm-up output (not timed)
    cw = out["cw"].cpu().numpy().view(np.uint32)
    bits = np.unpackbits(cw.view(np.uint8), axis=-1, bitorder="little")[:, :spec.N]
    fer_warm = float(np.mean(np.any(bits != x, axis=1)))

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        clk.wait_first()
        time.sleep(0.1)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = ws * B * args.steps / (ms / 1e3)
    # the timed steps' answers (every step decodes the same batch and table)
    gpu_host = {"cw": np.unpackbits(out["cw"].cpu().numpy().view(np.uint32).view(np.uint8), axis=-1,
                                    bitorder="little")[:, :spec.N],
                "pm": out["pm"].cpu().numpy(), "attempt": out["attempt"].cpu().numpy()}

    # decode only, permutation table resident in HBM (explains value)
    for _ in range(2):
        plan.launch(d_llr, d_rec, out, stream, work=work_d)
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        plan.launch(d_llr, d_rec, out, stream, work=work_d)
    ev1.record(stream)
    barrier()
    ms_dec = ev0.elapsed_time(ev1)

    # e2e through the public streaming API with host buffers, every step:
    # pinned host LLRs in, codewords / PM / attempt out; permutations drawn on
    # the device; H2D of batch k+1 and D2H of batch k-1 overlap decode of k
    from paper_2108_12550_b200.decoder import StreamDecoder
    h_llr = torch.from_numpy(llr).pin_memory()
    sd = StreamDecoder(plan, B, seed=SEED, identity_root=not AUT)
    e_steps = max(3, 2 * args.steps)  # host-path jitter averages out over more steps
    for _ in range(2):
        sd.submit(h_llr)
    sd.drain()
    barrier()
    ev0.record(sd.h2d)
    for _ in range(e_steps):
        sd.submit(h_llr)
    ev1.record(sd.d2h)  # after the last D2H (the D2H stream orders it)
    sd.drain()
    barrier()
    ms_e = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_e], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_e = float(t.item())
    e2e = ws * B * e_steps / (ms_e / 1e3)
    h2d = llr.nbytes
    d2h = B * (plan.words * 4 + 4 + 4)

    if rank == 0:
        hbm, sm_mhz, src = _peaks()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        if AUT:  # accounting.complexity_model("Aut-SSC"): P (SSC ops + N) + P - 1
            from paper_2108_12550_b200.plan import ssc_ops
            ops = M * (ssc_ops(R, M_VARS) + spec.N) + M - 1
        else:
            ops = complexity_ops(R, M_VARS, L, M, PERMS, include_perm=True, fsc=not PERMS and L == 1)
        peak_gops = sms * 128 * sm_mhz * 1e6 / 1e9
        per_gpu = value / ws
        # the dominant kernel's own rate: decode_kernel (+ its 1% reduce) timed
        # with CUDA events on the launching stream, permutation table resident
        kern_fps = B * args.steps / (ms_dec / 1e3)
        ach_gops = ops * kern_fps / 1e9
        # decode kernel's algorithmic HBM bytes per frame: LLRs + its permutation records + codeword
        bytes_frame = 4 * spec.N + spec.N // 8
        rec_bytes_frame = plan.M * plan.S * plan.rec_u16 * 2
        clk = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "nccl_world": comm,
            "config": {"workload": WORKLOAD, "frames_per_step": B, "parallelism": f"replicas{ws}",
                       "l2": f"inputs {(llr.nbytes + (recs.nbytes if recs is not None else 0)) / 2**20:.0f} MiB/step > 126 MB L2, no flush",
                       "fer_check": fer_warm},
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e_steps},
            # sampler kernel + decode (+ reduce) per step; plans without
            # permutations launch the decoder alone
            "gpu_launches": args.steps * (plan.launches_per_call + (1 if PERMS else 0)),
            "decode_only": {"value": ws * B * args.steps / (ms_dec / 1e3), "ms_per_step": ms_dec / args.steps,
                            "note": "same batch, permutation table already resident in HBM"},
            "roofline_fp32": {"bound": "fp32", "achieved": ach_gops, "peak": peak_gops, "unit": "Gop/s",
                              "frac": ach_gops / peak_gops, "traffic": _traffic(args.config, B),
                              "ops_per_frame": ops,
                              "kernel_ms": ms_dec / args.steps,
                              "note": f"reference op ledger per frame x frames per launch / decode-kernel time "
                                      f"(CUDA events) vs {sms} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz ({src} "
                                      f"sm_max_mhz)"},
            "roofline_hbm": {"bound": "hbm", "achieved": bytes_frame * kern_fps / 1e9,
                             "peak": hbm, "unit": "GB/s", "frac": bytes_frame * kern_fps / 1e9 / hbm,
                             "bytes_per_frame": bytes_frame, "traffic": _traffic(args.config, B),
                             "note": "LLR-in / codeword-out bytes per frame (4N + N/8) x frames per launch / "
                                     "decode-kernel time vs MEASURED_PEAKS hbm_gbs; with a host table the kernel "
                                     f"also reads {rec_bytes_frame} B/frame of map records"},
            "clocks": clk,
        }
        # the roofline that bounds this config: the slower of the ledger ops at
        # the FP32 issue peak and the LLR-in / codeword-out bytes at HBM
        # bandwidth (BASELINE.json north_star)
        fp32_fps = peak_gops * 1e9 / ops
        hbm_fps = hbm * 1e9 / bytes_frame
        line["roofline"] = dict(line["roofline_fp32"] if fp32_fps <= hbm_fps else line["roofline_hbm"])
        line["roofline"]["bound_frames_per_s"] = min(fp32_fps, hbm_fps)
        cap = _capture(args.config)
        if "warp_instructions" in cap:
            # issue view of the same kernel: warp instructions per frame (ncu,
            # committed capture) x the live frame rate vs 4 issue slots/clk/SM
            ipf = cap["warp_instructions"] / cap["frames_per_launch"]
            peak_i = sms * 4 * sm_mhz * 1e6 / 1e9
            line["roofline_issue"] = {"bound": "issue", "achieved": ipf * kern_fps / 1e9, "peak": peak_i,
                                      "unit": "G warp-inst/s", "frac": ipf * kern_fps / 1e9 / peak_i,
                                      "inst_per_frame": ipf}
        if not args.no_cpu and ws == 1:
            base, tie = cpu_baseline(plan, llr, x, gpu_host, SEED, args.cpu_seconds)
            line["cpu_baseline"] = base
            if tie is not None:
                line["ties"] = tie
            line["cpu_baseline_reference"] = cpu_baseline_reference(args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_dry(args):
    """The launch / timing / reduction plumbing on CPU ranks (gloo), with a
    stand-in step (hard decisions of the rank's own frames, no decoder):
    rank count, per-rank seeds, barrier + max-over-ranks time, rank-summed
    frames.  Tests only."""
    import torch
    import torch.distributed as dist
    from paper_2108_12550_b200.channel_model import synthetic_frames
    from paper_2108_12550_b200.rm_core import build_code
    ws, rank, _ = _dist()
    if ws > 1:
        dist.init_process_group("gloo")
    _, llr = synthetic_frames(build_code(R, M_VARS), EBN0, args.frames, seed=1 + rank)
    for _ in range(args.warmup):
        np.signbit(llr).sum()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    done = 0
    for _ in range(args.steps):
        done += int(np.signbit(llr).any(axis=1).shape[0])
    if ws > 1:
        dist.barrier()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    n = torch.tensor([done], dtype=torch.int64)
    firsts = [None] * ws
    if ws > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        dist.all_gather_object(firsts, float(llr[0, 0]))
    else:
        firsts = [float(llr[0, 0])]
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": ws, "steps": args.steps,
                          "warmup": args.warmup, "frames_total": int(n[0]), "value": int(n[0]) / float(dt),
                          "unit": "frames/s", "rank_first_llr": firsts,
                          "config": {"workload": WORKLOAD, "frames_per_step": args.frames}}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--frames", type=int, default=None)
    ap.add_argument("--config", default="rm29_L4_M20", choices=sorted(CONFIGS),
                    help="BASELINE.json configuration (default: the headline)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-lockstep", action="store_true", help="throughput kernel without per-round barriers")
    ap.add_argument("--lockstep", type=int, default=16, choices=[4, 8, 16], help="warps per lock-step group")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--dry-run", action="store_true", help="CPU ranks (gloo), stand-in step: plumbing tests only")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _relaunch(args)  # does not return
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or omit WORLD_SIZE to let bench.py spawn them")
    if args.warmup < 3:
        args.warmup = 3
    frames = select_config(args.config)
    if args.frames is None:
        args.frames = frames
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
