"""ctypes binding of librmfht.so (the C ABI in include/rmfht.h).

The CUDA library is the product path: there is no CPU fallback.  If the
library is missing or no GPU is visible, decoding raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMFHT_LIB_OVERRIDE") or os.path.join(_HERE, "librmfht.so")  # override: A/B experiments only
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

RMFHT_F32, RMFHT_F64 = 0, 1
RMFHT_PERMUTATIONS, RMFHT_TIE_FIX, RMFHT_NO_TIE_FIX, RMFHT_REFERENCE_ORDER, RMFHT_NO_LOCKSTEP = 1, 2, 4, 8, 16
RMFHT_LOCKSTEP_4, RMFHT_LOCKSTEP_8, RMFHT_GENERIC, RMFHT_AUT_SSC = 32, 64, 128, 256
RMFHT_OK, RMFHT_ECONFIG, RMFHT_EVALUE, RMFHT_EUNSUPPORTED, RMFHT_ECUDA = 0, -1, -2, -3, -4

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp", "-shared", "-lgomp"]

EXPORTS = [
    "rmfht_plan_create", "rmfht_plan_destroy", "rmfht_plan_maps_per_attempt",
    "rmfht_plan_map_sizes", "rmfht_plan_record_u16", "rmfht_expand_maps",
    "rmfht_decode_launch", "rmfht_decode_launch_diag", "rmfht_plan_launches_per_call",
    "rmfht_last_error", "rmfht_version", "rmfht_sample_maps", "rmfht_plan_kernel",
    "rmfht_sample_maps_device", "rmfht_decode_launch_sampled", "rmfht_gen_frames", "rmfht_count_errors",
    "rmfht_workspace_bytes",
]

_lib = None


def build(verbose: bool = False, jobs: int | None = None) -> str:
    """Compile librmfht.so in-tree for sm_100a (nvcc cross-compiles without a
    GPU).  The kernel specialisations are split into dtype x chunk units that
    compile in parallel."""
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    units = [("rmfht_capi", os.path.join(CSRC, "rmfht_capi.cu"), []),
             ("rmfht_gen", os.path.join(CSRC, "rmfht_gen.cu"), []),
             ("rmfht_chan", os.path.join(CSRC, "rmfht_chan.cu"), []),
             ("rmfht_ssc", os.path.join(CSRC, "rmfht_ssc.cu"), [])]
    for t in ("float", "double"):
        for c in range(4):
            units.append((f"rmfht_bind_{t}_{c}", os.path.join(CSRC, "rmfht_bind.cu"),
                          [f"-DRMFHT_T={t}", f"-DRMFHT_CHUNK={c}"]))
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-lgomp")]

    def one(u):
        name, src, defs = u
        obj = os.path.join(objdir, name + ".o")
        cmd = ["nvcc", *compile_flags, *defs, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=jobs or min(len(units), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, units))
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fopenmp",
           "-o", LIB_PATH, *objs, "-lgomp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                           "(the decoder has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
    L.rmfht_plan_create.argtypes = [I, I, I, I, I, I, ctypes.POINTER(P)]
    L.rmfht_plan_create.restype = I
    L.rmfht_plan_destroy.argtypes = [P]
    L.rmfht_plan_destroy.restype = None
    L.rmfht_plan_maps_per_attempt.argtypes = [P]
    L.rmfht_plan_maps_per_attempt.restype = I
    L.rmfht_plan_map_sizes.argtypes = [P, P]
    L.rmfht_plan_map_sizes.restype = I
    L.rmfht_plan_record_u16.argtypes = [P]
    L.rmfht_plan_record_u16.restype = I
    L.rmfht_plan_launches_per_call.argtypes = [P]
    L.rmfht_plan_launches_per_call.restype = I
    L.rmfht_plan_kernel.argtypes = [P]
    L.rmfht_plan_kernel.restype = I
    L.rmfht_expand_maps.argtypes = [P, P, P, LL]
    L.rmfht_expand_maps.restype = I
    L.rmfht_workspace_bytes.argtypes = [P, LL, I]
    L.rmfht_workspace_bytes.restype = LL
    L.rmfht_decode_launch.argtypes = [P, P, P, P, P, P, P, LL, P, LL, P]
    L.rmfht_decode_launch.restype = I
    L.rmfht_decode_launch_diag.argtypes = [P, P, P, P, P, P, P, P, P, LL, P, LL, P]
    L.rmfht_decode_launch_diag.restype = I
    L.rmfht_sample_maps.argtypes = [P, ctypes.c_uint64, LL, LL, I, P, P]
    L.rmfht_sample_maps.restype = I
    L.rmfht_sample_maps_device.argtypes = [P, ctypes.c_uint64, LL, LL, I, P, P]
    L.rmfht_sample_maps_device.restype = I
    L.rmfht_decode_launch_sampled.argtypes = [P, P, ctypes.c_uint64, LL, I, P, P, P, P, LL, P, LL, P]
    L.rmfht_decode_launch_sampled.restype = I
    L.rmfht_gen_frames.argtypes = [I, I, ctypes.c_uint64, LL, LL, LL, ctypes.c_double, I, P, P, P]
    L.rmfht_gen_frames.restype = I
    L.rmfht_count_errors.argtypes = [I, P, P, P, LL, P, P]
    L.rmfht_count_errors.restype = I
    L.rmfht_last_error.argtypes = []
    L.rmfht_last_error.restype = ctypes.c_char_p
    L.rmfht_version.argtypes = []
    L.rmfht_version.restype = I
    _lib = L
    return L


def last_error() -> str:
    return lib().rmfht_last_error().decode()
