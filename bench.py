"""Throughput of the batched p-FHT-FSCL-L-M decoder on B200.

Workload (BASELINE.json headline): RM(2,9), M=20 affine automorphisms
(decoder 0's root maps = identity), L=4, BPSK/AWGN float32 LLRs at
Eb/N0 = 2.5 dB.  One step = one decode launch over a batch of frames whose
LLRs and permutation tables are resident in HBM (together larger than the
126 MB L2, so no flush is needed between steps).

  value     decoded frames/s of the whole job (sum over ranks / max time)
  e2e       same metric through the public C-ABI path with host buffers:
            pinned host LLRs + map records copied in, codewords/PM/attempt
            copied out, every step
  roofline  reference op ledger (accounting.complexity_model, include_perm)
            per frame x frames/s against the FP32 issue peak
            (SMs x 128 lanes x max SM clock); HBM bound alongside
  cpu_baseline  the CPU oracle port (float64 restatement of the reference)
            on this host's cores, bounded sample

--impl reference times the CPU restatement of the reference decoder (the
reference is pure Python with no native path; the oracle port is its CPU
implementation here) on the same config, rank 0 only.
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
    "rm25_fhtfsc": (2, 5, 1, 1, False, 3.0, 1048576),
    # the paper's Table IV comparator, Aut-SSC with P = 512 (M = P here)
    "rm29_autssc_P512": (2, 9, 1, 512, "aut", 2.5, 2048),
}
R, M_VARS, L, M = 2, 9, 4, 20
PERMS = True
AUT = False
EBN0 = 2.5
WORKLOAD = "RM(2,9) p-FHT-FSCL L=4 M=20 (decoder 0 = identity), Eb/N0 2.5 dB"
METRIC = "decoded frames/s, RM(2,9) M=20 L=4, 1 B200; % of roofline; vs host CPU"


def select_config(name):
    global R, M_VARS, L, M, PERMS, AUT, EBN0, WORKLOAD
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
    """The dominant kernel's ncu figures for this config (profiles/r1_traffic.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

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


def _cpu_decode(llr, raw, cores):
    from oracle import oracle
    if AUT:
        oracle.aut_ssc(R, M_VARS, M, llr, raw[:, :, 0, :], dtype=np.float64, nthreads=cores)
        return
    oracle.decode(R, M_VARS, L, M if PERMS else 1, llr, raw, perms=PERMS, dtype=np.float64, nthreads=cores,
                  want_attempts=False)


def cpu_baseline(seconds: float = 12.0):
    """Oracle port (float64 restatement) on all host cores over a bounded sample."""
    cores = os.cpu_count() or 1
    done, t_used, frames = 0, 0.0, 0
    B = 16 * cores
    # calibrate the batch so one call is ~1/8 of the budget
    (llr, raw), = _cpu_batches(B, 1, 1000)
    t0 = time.perf_counter()
    _cpu_decode(llr, raw, cores)
    dt = time.perf_counter() - t0
    B = max(B, int(B * (seconds / 8) / max(dt, 1e-3)))
    while t_used < seconds and done < 64:
        (llr, raw), = _cpu_batches(B, 1, 1001 + done)
        t0 = time.perf_counter()
        _cpu_decode(llr, raw, cores)
        t_used += time.perf_counter() - t0
        frames += B
        done += 1
    return {"value": frames / t_used, "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{frames} frames of the workload ({done} batches of {B}), float64 oracle port, "
                      f"{cores} threads, {t_used:.1f} s"}


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
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
        time.sleep(0.3)
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
            "config": {"workload": WORKLOAD, "frames_per_step": B, "parallelism": f"replicas{ws}",
                       "l2": f"inputs {(llr.nbytes + (recs.nbytes if recs is not None else 0)) / 2**20:.0f} MiB/step > 126 MB L2, no flush",
                       "fer_check": fer_warm},
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e_steps},
            "gpu_launches": args.steps * (plan.launches_per_call + 1),
            "decode_only": {"value": ws * B * args.steps / (ms_dec / 1e3), "ms_per_step": ms_dec / args.steps,
                            "note": "same batch, permutation table already resident in HBM"},
            "roofline": {"bound": "fp32", "achieved": ach_gops, "peak": peak_gops, "unit": "Gop/s",
                         "frac": ach_gops / peak_gops, "traffic": _traffic(args.config, B),
                         "ops_per_frame": ops,
                         "kernel_ms": ms_dec / args.steps,
                         "note": f"reference op ledger per frame x frames per launch / decode-kernel time (CUDA "
                                 f"events) vs {sms} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz ({src} sm_max_mhz)"},
            "roofline_hbm": {"bound": "hbm", "achieved": (bytes_frame + rec_bytes_frame) * kern_fps / 1e9,
                             "peak": hbm, "unit": "GB/s",
                             "frac": (bytes_frame + rec_bytes_frame) * kern_fps / 1e9 / hbm,
                             "bytes_per_frame": bytes_frame + rec_bytes_frame},
            "clocks": clk,
        }
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
            line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        print(json.dumps(line), flush=True)
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    frames = select_config(args.config)
    if args.frames is None:
        args.frames = frames
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
