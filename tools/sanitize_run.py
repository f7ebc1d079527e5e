"""Small decode workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family of the product path on a few frames.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Test tooling: checks the f64 kernel against the golden fixtures (made by
running the reference, tools/gen_golden.py) so a sanitizer run that
perturbs nothing also shows the results unchanged.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_12550_b200.decoder import Plan  # noqa: E402

CASES = [  # (fixture, r, m, L, M)
    ("rm29_L4_M20_channel", 2, 9, 4, 20),
    ("rm37_L8_M32_channel", 3, 7, 8, 32),
    ("rm29_L1_M512_channel", 2, 9, 1, 512),
    ("rm27_L2_M4_channel", 2, 7, 2, 4),
    ("rm28_L8_M4_channel", 2, 8, 8, 4),
]
B = int(os.environ.get("SAN_FRAMES", "4"))


def main():
    torch.cuda.set_device(0)
    for name, r, m, L, M in CASES:
        g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
        llr, raw = g["llr"][:B], g["raw"][:B]
        N = 1 << m
        ref_cw = np.unpackbits(g["cw"][:B], axis=-1, bitorder="little")[:, :N]
        for dt in ("f64", "f32"):
            p = Plan(r, m, L, M, True, dt)
            o = p.decode(llr.astype(p.dtype), raw_maps=raw)
            if dt == "f64":
                assert np.array_equal(o["cw"], ref_cw), name
                assert np.array_equal(o["pm"], g["pm"][:B]), name
            print(f"{name} {dt} kernel={p.kernel} ok", flush=True)
        # device sampler + decode + reduce (the bench's launch sequence)
        p = Plan(r, m, L, M, True, "f32")
        d_llr = torch.from_numpy(np.ascontiguousarray(llr, dtype=np.float32)).cuda()
        out = p.alloc_outputs(B)
        p.launch_sampled(d_llr, 1234, out)
        torch.cuda.synchronize()
        print(f"{name} sampled ok", flush=True)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
