"""FER curves on the GPU for the BASELINE.json configurations (10^6 frames per
point by default) with Clopper-Pearson 95% intervals, next to the reference's
own Monte Carlo counts where available (tests/golden/ref_fer.json,
BASELINE.md §3).  Frames are generated, decoded and counted on the GPU (harness frames="device").
Writes a JSON report (default profiles/r1_fer.json)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_12550_b200 import harness
from paper_2108_12550_b200.top_decoders import DecoderConfig

CONFIGS = {
    "RM(2,5) FHT-FSC": (2, 5, DecoderConfig("FHT-FSC"), (3.0,)),
    "RM(2,7) L2 M4": (2, 7, DecoderConfig("p-FHT-FSCL", L=2, M=4), (2.0, 3.0, 4.0)),
    "RM(2,9) L4 M20": (2, 9, DecoderConfig("p-FHT-FSCL", L=4, M=20), (2.0, 2.5, 3.0, 3.5)),
    "RM(3,7) L8 M32": (3, 7, DecoderConfig("p-FHT-FSCL", L=8, M=32), (4.0,)),
    "RM(2,9) L1 M512": (2, 9, DecoderConfig("p-FHT-FSCL", L=1, M=512), (3.0,)),
    # the paper's Table IV comparators
    "RM(2,8) Aut-SSC P64": (2, 8, DecoderConfig("Aut-SSC", P=64), (2.0, 2.5, 3.0)),
    "RM(2,9) Aut-SSC P512": (2, 9, DecoderConfig("Aut-SSC", P=512), (2.0, 2.5, 3.0)),
}
ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=1000000)
ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "profiles", "r1_fer.json"))
ap.add_argument("--only", default=None)
ap.add_argument("--frames-headline", type=int, default=None, help="frames per point for RM(2,9) L4 M20")
args = ap.parse_args()
out = {}
for name, (r, m, cfg, pts) in CONFIGS.items():
    if args.only and args.only not in name:
        continue
    t = time.time()
    nf = args.frames_headline if (args.frames_headline and name == "RM(2,9) L4 M20") else args.frames
    recs = harness.run_job(harness.SimJob(r=r, m=m, decoder=cfg, ebn0_points=pts, max_frames=nf,
                                          min_frame_errors=10 ** 9, seed=777, batch=65536))
    out[name] = [dict(ebn0=rc.ebn0_db, frames=rc.frames, errors=rc.frame_errors, fer=rc.fer, ml_lb_fer=rc.ml_lb_fer,
                      ci95=harness.clopper_pearson(rc.frame_errors, rc.frames), wall_s=rc.wall_seconds,
                      frames_per_s=rc.frames / rc.wall_seconds) for rc in recs]
    print(name, [(p["ebn0"], p["errors"], p["frames"]) for p in out[name]], f"{time.time() - t:.1f}s", flush=True)
json.dump(out, open(args.out, "w"), indent=1)
