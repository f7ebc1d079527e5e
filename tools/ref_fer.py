"""Reference FER and modeled-cost fixtures: runs the UNMODIFIED reference
harness (rmworkbench.harness.run_job, all host cores) here in the build
container and stores tests/golden/ref_fer.json.  The GPU harness is compared
with these counts through Clopper-Pearson intervals (tests/test_gpu_fer.py)."""
import json, os, sys, time
sys.path.insert(0, os.environ.get("RMFHT_REFERENCE", "/root/reference/pkg/src"))
from rmworkbench.harness import SimJob, run_job, _modeled_cost
from rmworkbench.top_decoders import DecoderConfig

JOBS = [
    ("rm27_L2_M4", 2, 7, DecoderConfig("p-FHT-FSCL", L=2, M=4), (2.0, 3.0), 24000),
    ("rm25_fhtfsc", 2, 5, DecoderConfig("FHT-FSC"), (2.0, 3.0), 40000),
    ("rm26_fhtfscl_L4", 2, 6, DecoderConfig("FHT-FSCL", L=4), (2.0, 2.5), 40000),
    ("rm26_pfhtfscl_L4", 2, 6, DecoderConfig("p-FHT-FSCL", L=4), (2.0, 2.5), 40000),
    ("rm29_L4_M20", 2, 9, DecoderConfig("p-FHT-FSCL", L=4, M=20), (1.0, 1.5), 6000),
    ("rm27_autssc_P16", 2, 7, DecoderConfig("Aut-SSC", P=16), (2.0, 3.0), 16000),
    ("rm28_autssc_P64", 2, 8, DecoderConfig("Aut-SSC", P=64), (2.0, 2.5), 4000),
]
OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "ref_fer.json")
only = sys.argv[1] if len(sys.argv) > 1 else None
out = json.load(open(OUT)) if (only and os.path.exists(OUT)) else {"jobs": {}, "costs": {}}
for name, r, m, cfg, pts, frames in JOBS:
    if only and name != only:
        continue
    job = SimJob(r=r, m=m, decoder=cfg, ebn0_points=pts, max_frames=frames, min_frame_errors=10 ** 9,
                 seed=777, workers=os.cpu_count())
    t = time.time()
    recs = run_job(job)
    out["jobs"][name] = dict(r=r, m=m, algorithm=cfg.algorithm, L=cfg.L, M=cfg.M, P=cfg.P,
                             points=[dict(ebn0=rc.ebn0_db, frames=rc.frames, errors=rc.frame_errors,
                                          ml_lb_fer=rc.ml_lb_fer, wall=rc.wall_seconds) for rc in recs])
    ops, steps, mem = _modeled_cost(job)
    out["costs"][name] = dict(ops=ops, steps=steps, mem=mem, adds=recs[0].avg_additions,
                              comps=recs[0].avg_comparisons)
    print(name, [(p["ebn0"], p["errors"], p["frames"]) for p in out["jobs"][name]["points"]], f"{time.time()-t:.0f}s",
          flush=True)
json.dump(out, open(OUT, "w"), indent=1)
