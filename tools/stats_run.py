"""Diagnostic build + run: node-path counters and per-item cycle histogram of
the throughput kernel (RMFHT_STATS).  Builds librmfht_stats.so from the same
sources into /tmp, runs one headline batch, prints the counters.
usage: python tools/stats_run.py [frames]   (needs a GPU)"""
import ctypes, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_12550_b200 import _native

out = os.path.join(ROOT, "tools", "_stats")  # git-ignored; built here, travels to the GPU box
os.makedirs(out, exist_ok=True)
lib = os.path.join(out, "librmfht.so")
if not os.path.exists(lib):
    flags = [f for f in _native.NVCC_FLAGS if f not in ("-shared", "-lgomp")] + ["-DRMFHT_STATS"]
    from concurrent.futures import ThreadPoolExecutor
    units = [("capi", "rmfht_capi.cu", []), ("gen", "rmfht_gen.cu", []), ("chan", "rmfht_chan.cu", []),
             ("ssc", "rmfht_ssc.cu", [])] + \
            [(f"b{t}{c}", "rmfht_bind.cu", [f"-DRMFHT_T={t}", f"-DRMFHT_CHUNK={c}"]) for t in ("float", "double")
             for c in range(4)]

    def one(u):
        name, src, defs = u
        o = os.path.join(out, name + ".o")
        subprocess.run(["nvcc", *flags, *defs, "-c", os.path.join(_native.CSRC, src), "-o", o], check=True)
        return o

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, units))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fopenmp",
                    "-o", lib, *objs, "-lgomp"], check=True)
_native.LIB_PATH = lib
if len(sys.argv) > 1 and sys.argv[1] == "build":
    sys.exit(0)
import torch
from paper_2108_12550_b200.decoder import Plan
from paper_2108_12550_b200.channel_model import synthetic_frames
from paper_2108_12550_b200.rm_core import build_code
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
spec = build_code(2, 9)
_, llr = synthetic_frames(spec, 2.5, B, seed=1)
plan = Plan(2, 9, 4, 20, True, "f32")
out_t = plan.alloc_outputs(B)
plan.launch_sampled(torch.from_numpy(llr).cuda(), 1, out_t)
torch.cuda.synchronize()
L = ctypes.CDLL(lib)
fn = L.rmfht_stats_read_float_0
fn.argtypes = [ctypes.c_void_p]
st = np.zeros(256, dtype=np.uint64)
assert fn(st.ctypes.data_as(ctypes.c_void_p)) == 0
items = B * 20
print(f"items {items}")
for ss in range(3, 9):
    n, common, gen, fb, tot, over, greedy, exact = (int(st[ss * 8 + k]) for k in range(8))
    if n:
        print(f"FHT 2^{ss}: {n / items:.2f}/item  common {common / n:.3f}  greedy {greedy / n:.3f} "
              f"(collision -> exact list {exact / n:.3f}; over {over / n:.3f})  fallback {fb / n:.4f}  "
              f"mean cand {tot / n:.1f}  off-common with every lane <= 1 cand {int(st[100 + ss]) / max(1, n - common):.3f}"
              f"  <= 2 cand {int(st[110 + ss]) / max(1, n - common):.3f}")
cnt, s1, s2, mx = int(st[202]), int(st[200]), int(st[201]) * 1024, int(st[203])
if cnt:
    mean = s1 / cnt
    print(f"item cycles: mean {mean:.0f}  sd {max(0.0, s2 / cnt - mean * mean) ** 0.5:.0f}  max {mx}")
    hist = st[210:244]
    print("hist (2048-cycle buckets from 2048):", " ".join(str(int(h)) for h in hist))
    for ng in range(8):
        c = int(st[160 + ng])
        if c:
            print(f"items with {ng} FHT nodes off the common case: {c / cnt:.3f}  mean cycles {int(st[150 + ng]) / c:.0f}")
    g1, g2, gm = int(st[244]), int(st[245]) * 1024, int(st[246])
    gmean = g1 / cnt
    print(f"root f gathers: mean {gmean:.0f} cycles  sd {max(0.0, g2 / cnt - gmean * gmean) ** 0.5:.0f}  max {gm}")
