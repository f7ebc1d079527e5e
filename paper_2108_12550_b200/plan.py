"""Static decode schedule of p-FHT-FSCL / FHT-FSCL.

The reference walks the decoding tree recursively (``_decode_node``,
``top_decoders.py:72-113``); its visit order is a pure function of
(r, m, permutations) and is written out by ``accounting.plan_visits``
(``accounting.py:96-123``).  The GPU kernel is specialised on exactly this
schedule at compile time; this module restates it for the host (table
layout, validation, tracing).
"""

from __future__ import annotations

from .rm_core import ConfigurationError, build_code


def plan_visits(r: int, m: int, permutations: bool = True) -> list:
    """Node visits in decode order as (kind, m_node) — FHT and SPC nodes on."""
    build_code(r, m)
    visits: list = []
    state = {"perm": permutations}

    def rec(rr: int, mm: int):
        if rr == 1:
            state["perm"] = False
            visits.append(("fht", mm))
            return
        if mm >= 1 and rr == mm - 1:
            visits.append(("spc", mm))
            return
        if permutations and state["perm"] and 1 < rr < mm - 1:
            visits.append(("perm", mm))
        visits.append(("f", mm))
        rec(rr - 1, mm - 1)
        visits.append(("g", mm))
        rec(rr, mm - 1)

    rec(r, m)
    return visits


def map_sizes(r: int, m: int, L: int, permutations: bool = True) -> list:
    """Variable count of every map one attempt consumes, in consumption order:
    L root maps (top_decoders.py:129-132), then 2L per permutation node
    (automorphism.py:224-228) in visit order."""
    if not permutations:
        return []
    sizes = [m] * L
    for kind, mm in plan_visits(r, m, True):
        if kind == "perm":
            sizes += [mm] * (2 * L)
    return sizes


def validate(r: int, m: int, L: int, M: int) -> None:
    build_code(r, m)
    if L < 1 or M < 1:
        raise ConfigurationError("L, M and P must all be >= 1")


# ----------------------------------------------------------------------
# The reference's operation ledger (accounting.py:48-80, 136-152, 189-205),
# restated for the p-FHT-FSCL family.  It defines the roofline op count.

def _spc_charge(m: int, L: int) -> int:
    from math import log2
    n = 1 << m
    if L == 1:
        return n
    tau = min(L, n)
    lg = log2(L)
    adds = L * (1 + 2 * tau)
    comps = min(L * m * n, L * L * n) + int(2 * tau * L * (1 + lg))
    return adds + comps


def _perm_charge(m: int, L: int) -> int:
    from math import log2
    half = (1 << m) >> 1
    return 2 * L * half + 2 * L * half + int(2 * (2 * L) * log2(2 * L))


def complexity_ops(r: int, m: int, L: int, M: int, permutations: bool = True,
                   include_perm: bool = True, fsc: bool = False) -> int:
    """Operations (additions + comparisons) per decoded frame, as
    accounting.complexity_model(algo, r, m, L, M, include_perm) counts them."""
    from math import log2
    eff_l = 1 if fsc else L
    total = 0
    for kind, mm in plan_visits(r, m, permutations):
        n = 1 << mm
        if kind in ("f", "g"):
            total += eff_l * (n >> 1)
        elif kind == "fht":
            total += eff_l * n * (mm + 1) + int(2 * eff_l * eff_l * log2(eff_l))
        elif kind == "spc":
            total += _spc_charge(mm, eff_l)
        elif kind == "perm" and include_perm:
            total += _perm_charge(mm, eff_l)
    return (M if permutations else 1) * total


def ssc_walk(r: int, m: int) -> list:
    """Node visits of ssc_decode (accounting._ssc_walk, accounting.py:232-252):
    rate0 / rate1 / rep / spc1 leaves, f and g at internal nodes."""
    visits = []

    def rec(rr: int, mm: int):
        if rr < 0 or rr == mm or rr == 0 or (mm >= 1 and rr == mm - 1):
            visits.append(("rate0" if rr < 0 else "rate1" if rr == mm else "rep" if rr == 0 else "spc1", mm))
            return
        visits.append(("f", mm))
        rec(rr - 1, mm - 1)
        visits.append(("g", mm))
        rec(rr, mm - 1)

    rec(r, m)
    return visits


def ssc_ops(r: int, m: int) -> int:
    """accounting._ssc_operations (accounting.py:255-265)."""
    ops = 0
    for kind, mm in ssc_walk(r, m):
        n = 1 << mm
        if kind in ("f", "g"):
            ops += n >> 1
        elif kind == "rep":
            ops += n - 1
        elif kind == "spc1":
            ops += n
    return ops


def ssc_steps(r: int, m: int) -> int:
    """accounting._ssc_steps (accounting.py:268-273)."""
    return sum(1 for kind, _ in ssc_walk(r, m) if kind in ("f", "g", "rep", "spc1"))
