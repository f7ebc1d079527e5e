"""Batched decoding on the GPU through the C ABI.

``Plan`` owns one ``rmfht_plan`` (code shape, list size, ensemble size,
dtype) and launches the decoder on torch device buffers (torch is only the
allocator and stream provider here).  ``decode_batch`` is the batched
counterpart of the reference's per-frame ``ensemble_decode`` loop.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native
from .automorphism import random_raw_table
from .rm_core import ConfigurationError, UnsupportedShape, build_code

_ERRS = {
    _native.RMFHT_ECONFIG: ConfigurationError,
    _native.RMFHT_EVALUE: ValueError,
    _native.RMFHT_EUNSUPPORTED: UnsupportedShape,
}


def _check(rc: int):
    if rc != 0:
        raise _ERRS.get(rc, RuntimeError)(_native.last_error())


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the p-FHT-FSCL decoder runs only on the GPU")
    return torch


class Plan:
    """An immutable decode plan bound to a compiled kernel specialisation."""

    def __init__(self, r: int, m: int, L: int, M: int = 1, permutations: bool = True,
                 dtype: str = "f32", tie_fix: bool | None = None, reference_order: bool = False,
                 lockstep: int = 16, generic: bool = False, aut_ssc: bool = False):
        build_code(r, m)
        if L < 1 or M < 1:
            raise ConfigurationError("L, M and P must all be >= 1")
        self.r, self.m, self.L = r, m, L
        self.permutations = bool(permutations)
        self.M = M if self.permutations else 1
        self.N = 1 << m
        self.dtype = np.dtype(np.float64 if dtype in ("f64", np.float64, "float64") else np.float32)
        flags = _native.RMFHT_PERMUTATIONS if self.permutations else 0
        if tie_fix is True:
            flags |= _native.RMFHT_TIE_FIX
        elif tie_fix is False:
            flags |= _native.RMFHT_NO_TIE_FIX
        if reference_order:
            flags |= _native.RMFHT_REFERENCE_ORDER
        if not lockstep:
            flags |= _native.RMFHT_NO_LOCKSTEP
        elif lockstep == 4:
            flags |= _native.RMFHT_LOCKSTEP_4
        elif lockstep == 8:
            flags |= _native.RMFHT_LOCKSTEP_8
        if generic:
            flags |= _native.RMFHT_GENERIC
        if aut_ssc:
            # Aut-SSC: M = P single-map SSC decodes per frame (RMFHT_AUT_SSC)
            if L != 1 or not self.permutations:
                raise ConfigurationError("Aut-SSC plans take L = 1 with permutations (P = M decodes)")
            flags |= _native.RMFHT_AUT_SSC
        self.aut_ssc = bool(aut_ssc)
        lib = _native.lib()
        h = ctypes.c_void_p()
        _check(lib.rmfht_plan_create(r, m, L, M, flags,
                                     _native.RMFHT_F64 if self.dtype == np.float64 else _native.RMFHT_F32,
                                     ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.S = lib.rmfht_plan_maps_per_attempt(h)
        sizes = (ctypes.c_int * max(1, self.S))()
        lib.rmfht_plan_map_sizes(h, sizes)
        self.sizes = [int(sizes[i]) for i in range(self.S)]
        self.rec_u16 = lib.rmfht_plan_record_u16(h)
        self.words = max(1, self.N // 32)
        self.launches_per_call = lib.rmfht_plan_launches_per_call(h)
        self.kernel = lib.rmfht_plan_kernel(h)  # 1 reference-order, 2 float32 throughput, 3 generic, 4 Aut-SSC, 5 lane, 6 pair, 7 lane-group

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.rmfht_plan_destroy(h)
            self._h = None

    # ------------------------------------------------------------ maps ----
    def expand(self, raw: np.ndarray) -> np.ndarray:
        """Raw reference-format maps [..., S, m+1] -> device records [..., S, 2m+2]."""
        raw = np.ascontiguousarray(raw, dtype=np.uint16)
        if raw.shape[-2:] != (self.S, self.m + 1):
            raise ValueError(f"raw maps must end in {(self.S, self.m + 1)}, got {raw.shape}")
        rec = np.empty(raw.shape[:-1] + (self.rec_u16,), dtype=np.uint16)
        count = int(np.prod(raw.shape[:-1]))
        _check(self._lib.rmfht_expand_maps(self._h, raw.ctypes.data_as(ctypes.c_void_p),
                                           rec.ctypes.data_as(ctypes.c_void_p), count))
        return rec

    def random_raw(self, B: int, seed: int, identity_root: bool = True) -> np.ndarray:
        """Seeded numpy table (vectorised rejection sampler)."""
        rng = np.random.default_rng(seed)
        return random_raw_table(rng, (B, self.M), self.sizes, self.m,
                                identity_root=self.L if identity_root else 0)

    def sample(self, B: int, seed: int, frame0: int = 0, identity_root: bool = True,
               want_raw: bool = True, want_records: bool = True):
        """Counter-based C sampler (rmfht_sample_maps): (raw, records)."""
        raw = np.empty((B, self.M, self.S, self.m + 1), dtype=np.uint16) if want_raw else None
        rec = np.empty((B, self.M, self.S, self.rec_u16), dtype=np.uint16) if want_records else None
        if self.S == 0:
            return raw, rec
        _check(self._lib.rmfht_sample_maps(
            self._h, ctypes.c_uint64(seed), frame0, B, int(identity_root),
            None if raw is None else raw.ctypes.data_as(ctypes.c_void_p),
            None if rec is None else rec.ctypes.data_as(ctypes.c_void_p)))
        return raw, rec

    def sample_device(self, B: int, seed: int, frame0: int = 0, identity_root: bool = True, stream=None):
        """Device map records drawn on the GPU (bit-identical to ``sample``)."""
        torch = _torch()
        rec = torch.empty((B, self.M, self.S, self.rec_u16), dtype=torch.int16, device="cuda")
        st = stream if stream is not None else torch.cuda.current_stream()
        _check(self._lib.rmfht_sample_maps_device(self._h, ctypes.c_uint64(seed), frame0, B, int(identity_root),
                                                  rec.data_ptr(), st.cuda_stream))
        return rec

    # ------------------------------------------------------- workspace ----
    def workspace_bytes(self, B: int, sampled: bool = False) -> int:
        """rmfht_workspace_bytes: device scratch a launch of B frames needs."""
        n = self._lib.rmfht_workspace_bytes(self._h, B, int(sampled))
        if n < 0:
            _check(int(n))
        return int(n)

    def alloc_workspace(self, B: int, sampled: bool = False, device=None, stream=None):
        """A caller-owned workspace for launches of up to B frames (None if
        the plan's kernel needs none).  Allocated on `stream` so torch's
        caching allocator orders its reuse with that stream."""
        n = self.workspace_bytes(B, sampled)
        if n == 0:
            return None
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            return torch.empty(n, dtype=torch.uint8, device=device or torch.device("cuda"))

    def _work(self, B: int, sampled: bool, work, stream):
        """(tensor kept alive by the caller until the launch is queued, ptr, bytes)"""
        if work is None:
            work = self.alloc_workspace(B, sampled, stream=stream)
        if work is None:
            return None, None, 0
        return work, work.data_ptr(), work.numel() * work.element_size()

    def launch_sampled(self, llr, seed: int, out: dict, frame0: int = 0, identity_root: bool = True,
                       stream=None, work=None) -> None:
        """Stream-ordered decode with on-device permutation sampling.
        `work`: a workspace from alloc_workspace(B, sampled=True), else one is
        allocated for this call."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream()
        _keep, wp, wn = self._work(llr.shape[0], True, work, st)
        _check(self._lib.rmfht_decode_launch_sampled(
            self._h, llr.data_ptr(), ctypes.c_uint64(seed), frame0, int(identity_root), out["cw"].data_ptr(),
            out["pm"].data_ptr(), out["attempt"].data_ptr(), out["path"].data_ptr(), llr.shape[0], wp, wn,
            st.cuda_stream))

    # ---------------------------------------------------------- launch ----
    def alloc_outputs(self, B: int, device=None, diag: bool = False):
        torch = _torch()
        tdt = torch.float64 if self.dtype == np.float64 else torch.float32
        dev = device or torch.device("cuda")
        out = dict(
            cw=torch.empty((B, self.words), dtype=torch.int32, device=dev),
            pm=torch.empty(B, dtype=tdt, device=dev),
            attempt=torch.empty(B, dtype=torch.int32, device=dev),
            path=torch.empty(B, dtype=torch.int32, device=dev),
        )
        if diag:
            out["att_pm"] = torch.empty((B, self.M), dtype=tdt, device=dev)
            out["att_cw"] = torch.empty((B, self.M, self.words), dtype=torch.int32, device=dev)
        return out

    def launch(self, llr, rec, out: dict, stream=None, work=None) -> None:
        """Stream-ordered launch on device tensors (no host synchronisation).
        `work`: a workspace from alloc_workspace(B), else one is allocated."""
        torch = _torch()
        B = llr.shape[0]
        if llr.shape[-1] != self.N:
            raise ValueError(f"LLR length {llr.shape[-1]} != ({self.N},)")
        if llr.dtype != (torch.float64 if self.dtype == np.float64 else torch.float32):
            raise ValueError("LLR dtype does not match the plan dtype")
        if not llr.is_cuda or not llr.is_contiguous():
            raise ValueError("llr must be a contiguous CUDA tensor")
        if self.permutations:
            if rec is None or tuple(rec.shape) != (B, self.M, self.S, self.rec_u16):
                raise ValueError(f"map records must have shape {(B, self.M, self.S, self.rec_u16)}")
            rec_ptr = rec.data_ptr()
        else:
            rec_ptr = None
        st = stream if stream is not None else torch.cuda.current_stream()
        _keep, wp, wn = self._work(B, False, work, st)
        diag = "att_pm" in out
        args = [self._h, llr.data_ptr(), rec_ptr, out["cw"].data_ptr(), out["pm"].data_ptr(),
                out["attempt"].data_ptr(), out["path"].data_ptr()]
        if diag:
            rc = self._lib.rmfht_decode_launch_diag(*args, out["att_pm"].data_ptr(),
                                                    out["att_cw"].data_ptr(), B, wp, wn, st.cuda_stream)
        else:
            rc = self._lib.rmfht_decode_launch(*args, B, wp, wn, st.cuda_stream)
        _check(rc)

    def decode(self, llr, raw_maps=None, records=None, diag: bool = False) -> dict:
        """Host arrays in, host arrays out (synchronises).  For tests and the drop-in API."""
        torch = _torch()
        llr = np.ascontiguousarray(llr, dtype=self.dtype)
        if llr.ndim == 1:
            llr = llr[None, :]
        B = llr.shape[0]
        d_llr = torch.from_numpy(llr).cuda()
        d_rec = None
        if self.permutations:
            if records is None:
                records = self.expand(raw_maps)
            d_rec = torch.from_numpy(np.ascontiguousarray(records).view(np.int16)).cuda()
        out = self.alloc_outputs(B, diag=diag)
        self.launch(d_llr, d_rec, out)
        torch.cuda.synchronize()
        res = {k: v.cpu().numpy() for k, v in out.items()}
        words = res["cw"].view(np.uint32)
        res["cw_packed"] = words
        res["cw"] = unpack_bits(words, self.N)
        if diag:
            res["att_cw_packed"] = res["att_cw"].view(np.uint32)
            res["att_cw"] = unpack_bits(res["att_cw_packed"], self.N)
        return res


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
    return bits[..., :n]


@lru_cache(maxsize=64)
def get_plan(r: int, m: int, L: int, M: int, permutations: bool = True, dtype: str = "f32",
             aut_ssc: bool = False) -> Plan:
    return Plan(r, m, L, M, permutations, dtype, aut_ssc=aut_ssc)


@dataclass
class BatchResult:
    codewords: np.ndarray  # uint8 [B, N]
    pm: np.ndarray         # [B]
    attempt: np.ndarray    # int32 [B]
    path: np.ndarray       # int32 [B]


def decode_batch(spec, alphas, L: int, M: int = 1, maps=None, seed: int | None = None,
                 permutations: bool = True, dtype: str = "f32") -> BatchResult:
    """Decode B frames at once.  ``maps``: raw table [B, M, S, m+1] (reference
    format); otherwise one is drawn from ``seed`` (decoder 0's root maps = I)."""
    plan = get_plan(spec.r, spec.m, L, M, permutations, dtype)
    alphas = np.asarray(alphas)
    if alphas.ndim != 2 or alphas.shape[1] != spec.N:
        raise ValueError(f"alphas must be [B, {spec.N}]")
    if plan.permutations and maps is None:
        maps = plan.random_raw(alphas.shape[0], 0 if seed is None else seed)
    res = plan.decode(alphas, raw_maps=maps)
    return BatchResult(res["cw"], res["pm"], res["attempt"], res["path"])


class StreamDecoder:
    """Double-buffered host-to-host decoding: while batch k decodes on the
    compute stream, batch k+1's LLRs copy in on a copy stream and batch k-1's
    results copy out.  Permutation tables are drawn on the device from
    (seed, frame offset), so only LLRs cross PCIe.

        sd = StreamDecoder(plan, batch=16384, seed=777)
        for llr in host_batches:            # pinned float32 [batch, N]
            done = sd.submit(llr)           # results of an older batch, or None
        rest = sd.drain()                   # results of the batches still in flight

    Result dicts hold host tensors (cw words, pm, attempt) owned by the caller.
    """

    def __init__(self, plan: Plan, batch: int, seed: int = 0, identity_root: bool = True, depth: int = 2):
        torch = _torch()
        self.torch, self.plan, self.batch, self.seed, self.ident = torch, plan, batch, seed, identity_root
        dev = torch.device("cuda")
        self.compute = torch.cuda.Stream()
        # one stream per direction: an H2D queued behind the previous batch's
        # D2H (which waits for that decode) would serialise copy and decode
        self.h2d = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self.depth = depth
        self.d_llr = [torch.empty((batch, plan.N), dtype=torch.float32, device=dev) for _ in range(depth)]
        self.out = [plan.alloc_outputs(batch, dev) for _ in range(depth)]
        self.work = [plan.alloc_workspace(batch, sampled=True, stream=self.compute) for _ in range(depth)]
        self.h_out = [dict(cw=torch.empty((batch, plan.words), dtype=torch.int32).pin_memory(),
                           pm=torch.empty(batch, dtype=torch.float32).pin_memory(),
                           attempt=torch.empty(batch, dtype=torch.int32).pin_memory()) for _ in range(depth)]
        self.in_ready = [torch.cuda.Event() for _ in range(depth)]
        self.done = [torch.cuda.Event() for _ in range(depth)]
        self.out_ready = [torch.cuda.Event() for _ in range(depth)]
        self.pending = []
        self.k = 0
        self.frame0 = 0

    def submit(self, h_llr):
        """Queue one pinned host batch (torch tensor [n <= batch, N])."""
        torch = self.torch
        i = self.k % self.depth
        n = h_llr.shape[0]
        ready = None
        if len(self.pending) >= self.depth:
            j, ev, nj = self.pending.pop(0)
            ev.synchronize()
            # buffer j is reused right below: hand out a snapshot
            ready = {k: v[:nj].clone() for k, v in self.h_out[j].items()}
        with torch.cuda.stream(self.h2d):
            self.h2d.wait_event(self.done[i])  # buffer i free (its previous decode finished)
            self.d_llr[i][:n].copy_(h_llr, non_blocking=True)
            self.in_ready[i].record(self.h2d)
        with torch.cuda.stream(self.compute):
            self.compute.wait_event(self.in_ready[i])
            self.compute.wait_event(self.out_ready[i])  # previous results of buffer i copied out
            out = {k: v[:n] for k, v in self.out[i].items()}
            self.plan.launch_sampled(self.d_llr[i][:n], self.seed, out, frame0=self.frame0,
                                     identity_root=self.ident, stream=self.compute, work=self.work[i])
            self.done[i].record(self.compute)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.done[i])
            for key in ("cw", "pm", "attempt"):
                self.h_out[i][key][:n].copy_(self.out[i][key][:n], non_blocking=True)
            self.out_ready[i].record(self.d2h)
        self.pending.append((i, self.out_ready[i], n))
        self.k += 1
        self.frame0 += n
        return ready

    def drain(self):
        """Wait for all queued batches; returns the last `depth` batches' host results."""
        res = []
        for i, ev, n in self.pending:
            ev.synchronize()
            res.append({k: v[:n].clone() for k, v in self.h_out[i].items()})
        self.pending = []
        return res
