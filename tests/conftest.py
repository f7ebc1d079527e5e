import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "rm*.npz")))


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {k: d[k] for k in d.files}
    for k in ("r", "m", "L", "M", "perms"):
        out[k] = int(out[k])
    out["mode"] = str(out["mode"])
    N = 1 << out["m"]
    out["cw_bits"] = np.unpackbits(out["cw"], axis=-1, bitorder="little")[..., :N]
    out["att_cw_bits"] = np.unpackbits(out["att_cw"], axis=-1, bitorder="little")[..., :N]
    return out


def aut_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "autssc_*.npz")))


def load_aut(name):
    """Aut-SSC fixture (tools/gen_golden.py run_aut_case)."""
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {k: d[k] for k in d.files}
    for k in ("r", "m", "P"):
        out[k] = int(out[k])
    out["mode"] = str(out["mode"])
    out["cw_bits"] = np.unpackbits(out["cw"], axis=-1, bitorder="little")[..., :1 << out["m"]]
    return out


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.lib()
    return oracle
