"""Build an A/B variant of librmfht.so with extra nvcc flags into tools/_ab/
(git-ignored, travels to the GPU box).  usage: build_variant.py NAME FLAG..."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_12550_b200 import _native
name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join("/tmp", "rmfht_ab", name)  # objects stay here; only the .so travels
os.makedirs(os.path.join(ROOT, "tools", "_ab"), exist_ok=True)
os.makedirs(out, exist_ok=True)
flags = [f for f in _native.NVCC_FLAGS if f not in ("-shared", "-lgomp")] + extra
units = [("capi", "rmfht_capi.cu", []), ("gen", "rmfht_gen.cu", []), ("chan", "rmfht_chan.cu", []),
         ("ssc", "rmfht_ssc.cu", [])] + \
        [(f"b{t}{c}", "rmfht_bind.cu", [f"-DRMFHT_T={t}", f"-DRMFHT_CHUNK={c}"]) for t in ("float", "double")
         for c in range(4)]

def one(u):
    n, src, defs = u
    o = os.path.join(out, n + ".o")
    subprocess.run(["nvcc", *flags, *defs, "-c", os.path.join(_native.CSRC, src), "-o", o], check=True)
    return o

with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, units))
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fopenmp",
                "-o", os.path.join(ROOT, "tools", "_ab", f"librmfht_{name}.so"), *objs, "-lgomp"], check=True)
print("built", f"tools/_ab/librmfht_{name}.so")
