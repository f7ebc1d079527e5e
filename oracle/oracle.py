"""TEST INFRASTRUCTURE ONLY — Python handle on the CPU oracle.

Loads ``oracle/librmfht_oracle.so`` (built by ``oracle/Makefile``; a plain-C
restatement of the reference hot path, see ``rmfht_oracle.c``).  Imported
only by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline
legs; the product package never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librmfht_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()  # make: a no-op when up to date, loud when the sources do not compile
        _lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        for sfx in ("f64", "f32"):
            fn = getattr(_lib, f"rmo_decode_{sfx}")
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_int] * 6 + [P, ctypes.c_long, P, ctypes.c_int] + [P] * 7
            fa = getattr(_lib, f"rmo_aut_ssc_{sfx}")
            fa.restype = ctypes.c_int
            fa.argtypes = [ctypes.c_int] * 3 + [P, ctypes.c_long, P, ctypes.c_int, P, P, P]
        _lib.rmo_maps_per_attempt.restype = ctypes.c_int
        _lib.rmo_maps_per_attempt.argtypes = [ctypes.c_int] * 4 + [P]
        _lib.rmo_expand_table.restype = ctypes.c_int
        _lib.rmo_expand_table.argtypes = [P, ctypes.c_long, ctypes.c_int, P, ctypes.c_int, P]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def maps_per_attempt(r, m, L, perms=True):
    return lib().rmo_maps_per_attempt(r, m, L, int(perms), None)


RMO_TIE_FIX, RMO_ORDER_V2 = 1, 2


def decode(r, m, L, M, llr, raw_maps=None, perms=True, dtype=np.float64, tie_fix=None,
           nthreads=1, want_attempts=True, order="reference"):
    """Decode a batch on the CPU oracle.

    llr: (B, N) array; raw_maps: (B, M, S, m+1) uint16 or None when perms is
    False.  dtype float64 restates the reference bit-for-bit; float32 runs
    the same operation order in float32 (the GPU fp32 kernel's arithmetic).
    tie_fix defaults to on for float32 (equal pairing directions keep equal
    LM) and off for float64 (pure reference behaviour).
    order="v2" restates the float32 throughput kernel's summation orders
    (llr_abs and LM; canonical LM order makes the tie fix implicit).
    """
    dtype = np.dtype(dtype)
    if tie_fix is None:
        tie_fix = dtype == np.float32 and order != "v2"
    flags = (RMO_TIE_FIX if tie_fix else 0) | (RMO_ORDER_V2 if order == "v2" else 0)
    llr = np.ascontiguousarray(llr, dtype=dtype)
    B, N = llr.shape
    if N != 1 << m:
        raise ValueError(f"LLR length {N} != {1 << m}")
    Meff = M if perms else 1
    S = maps_per_attempt(r, m, L, perms)
    if perms:
        raw_maps = np.ascontiguousarray(raw_maps, dtype=np.uint16)
        if raw_maps.shape != (B, M, S, m + 1):
            raise ValueError(f"raw_maps shape {raw_maps.shape} != {(B, M, S, m + 1)}")
    cw = np.zeros((B, N), dtype=np.uint8)
    pm = np.zeros(B, dtype=dtype)
    att = np.zeros(B, dtype=np.int32)
    path = np.zeros(B, dtype=np.int32)
    att_pm = np.zeros((B, Meff), dtype=dtype) if want_attempts else None
    att_cw = np.zeros((B, Meff, N), dtype=np.uint8) if want_attempts else None
    margin = np.zeros(B, dtype=np.float64)
    fn = lib().rmo_decode_f64 if dtype == np.float64 else lib().rmo_decode_f32
    rc = fn(r, m, L, M, int(perms), flags, _ptr(llr), B,
            _ptr(raw_maps) if perms else None, int(nthreads), _ptr(cw), _ptr(pm), _ptr(att),
            _ptr(path), _ptr(att_pm), _ptr(att_cw), _ptr(margin))
    if rc != 0:
        raise RuntimeError(f"oracle decode failed rc={rc}")
    return dict(cw=cw, pm=pm, attempt=att, path=path, att_pm=att_pm, att_cw=att_cw,
                margin=margin)


def aut_ssc(r, m, P, llr, raw_maps, dtype=np.float64, nthreads=1):
    """Aut-SSC (top_decoders.py:235-249) on the CPU oracle: P SSC decodes per
    frame under the maps raw_maps (B, P, m+1); returns dict(cw, score, winner)."""
    dtype = np.dtype(dtype)
    llr = np.ascontiguousarray(llr, dtype=dtype)
    B, N = llr.shape
    if N != 1 << m:
        raise ValueError(f"LLR length {N} != {1 << m}")
    raw_maps = np.ascontiguousarray(raw_maps, dtype=np.uint16)
    if raw_maps.shape != (B, P, m + 1):
        raise ValueError(f"raw_maps shape {raw_maps.shape} != {(B, P, m + 1)}")
    cw = np.zeros((B, N), dtype=np.uint8)
    score = np.zeros(B, dtype=dtype)
    win = np.zeros(B, dtype=np.int32)
    fn = lib().rmo_aut_ssc_f64 if dtype == np.float64 else lib().rmo_aut_ssc_f32
    rc = fn(r, m, P, _ptr(llr), B, _ptr(raw_maps), int(nthreads), _ptr(cw), _ptr(score), _ptr(win))
    if rc != 0:
        raise RuntimeError(f"oracle aut_ssc failed rc={rc}")
    return dict(cw=cw, score=score, winner=win)
