"""Drop-in mirror of the reference decoder entry points (top_decoders.py).

Same names, arguments, error types and random-number consumption as
``/root/reference/pkg/src/rmworkbench/top_decoders.py`` for the
p-FHT-FSCL family and Aut-SSC; decoding itself runs in the CUDA library.  Permutations
are drawn on the host exactly as the reference draws them (or taken from a
``sampler`` plugin, called in the reference's order) and handed to the GPU
as a table.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .automorphism import maps_to_raw, sample_affine, sample_affine_batch
from .decoder import get_plan
from .plan import map_sizes, plan_visits
from .rm_core import CodeSpec, ConfigurationError, UnsupportedShape  # noqa: F401 (re-exported)

ALGORITHMS = ("SC", "SCL", "FSCL", "FHT-FSC", "FHT-FSCL", "p-FHT-FSCL",
              "Aut-SSC", "RPA", "SRPA")
SUPPORTED = ("FHT-FSC", "FHT-FSCL", "p-FHT-FSCL", "Aut-SSC")


@dataclass(frozen=True)
class DecoderConfig:
    """top_decoders.py:29-42"""
    algorithm: str
    L: int = 1
    M: int = 1
    P: int = 1
    permutations_enabled: bool = True
    seed: int = 0

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ConfigurationError(f"unknown algorithm {self.algorithm!r}")
        if self.L < 1 or self.M < 1 or self.P < 1:
            raise ConfigurationError("L, M and P must all be >= 1")


@dataclass
class DecodeResult:
    """top_decoders.py:45-48 (plus the selected attempt and path)."""
    codeword: np.ndarray
    pm: float
    attempt: int = 0
    path: int = 0


def _alpha(spec: CodeSpec, alpha) -> np.ndarray:
    a = np.asarray(alpha, dtype=np.float64)
    if a.shape != (spec.N,):
        raise ValueError(f"LLR length {a.shape} != ({spec.N},)")
    return a


def _attempt_maps(spec: CodeSpec, L: int, rng, sampler) -> list:
    """Maps of one attempt in consumption order: L root maps (top_decoders.py:
    129-132), then one batch of 2L per permutation node (automorphism.py:224-228)."""
    if sampler is not None:
        return [sampler() for _ in map_sizes(spec.r, spec.m, L, True)]
    maps = list(sample_affine_batch(spec.m, L, rng))
    for kind, mm in plan_visits(spec.r, spec.m, True):
        if kind == "perm":
            maps += sample_affine_batch(mm, 2 * L, rng)
    return maps


def _trace(spec: CodeSpec, L: int, permutations: bool, trace: list) -> None:
    """The reference's node trace (kind, m, alive) (top_decoders.py:67-69,
    76-105): the schedule is static and so are the path counts."""
    state = {"perm": permutations, "p": L if permutations else 1}

    def rec(r, m):
        p = state["p"]
        if r == 1:
            state["perm"] = False
            trace.append(("fht", m, p))
            state["p"] = min(L, p * min(L, 1 << m))
            return
        if m >= 1 and r == m - 1:
            trace.append(("spc", m, p))
            for _ in range(min(L, (1 << m) - 1)):
                p = min(L, 2 * p)
            state["p"] = p
            return
        if state["perm"] and 1 < r < m - 1:
            trace.append(("perm", m, p))
            state["p"] = min(L, 2 * p)
        trace.append(("f", m, state["p"]))
        rec(r - 1, m - 1)
        trace.append(("g", m, state["p"]))
        rec(r, m - 1)

    rec(spec.r, spec.m)


# The single-frame drop-in API decodes in float64, which reproduces the
# float64 reference bit-for-bit; batched throughput runs use float32
# (decoder.decode_batch / Plan).
DEFAULT_DTYPE = "f64"


def _run(spec, alpha, L, M, maps, permutations) -> DecodeResult:
    plan = get_plan(spec.r, spec.m, L, M, permutations, DEFAULT_DTYPE)
    raw = None
    if permutations:
        raw = maps_to_raw(maps, spec.m).reshape(1, M, plan.S, spec.m + 1)
    res = plan.decode(alpha[None, :], raw_maps=raw)
    return DecodeResult(codeword=res["cw"][0].astype(np.uint8), pm=float(res["pm"][0]),
                        attempt=int(res["attempt"][0]), path=int(res["path"][0]))


def p_fht_fscl(spec: CodeSpec, alpha, L: int, rng, sampler=None, trace=None) -> DecodeResult:
    """Permuted FHT-FSCL, one attempt (top_decoders.py:178-187)."""
    alpha = _alpha(spec, alpha)
    if rng is None and sampler is None:
        raise ConfigurationError("permuted decoding needs an rng")
    if trace is not None:
        _trace(spec, L, True, trace)
    maps = _attempt_maps(spec, L, rng, sampler)
    return _run(spec, alpha, L, 1, maps, True)


def ensemble_decode(spec: CodeSpec, alpha, L: int, M: int, rng, sampler=None) -> DecodeResult:
    """M independent permuted attempts; strictly smallest pm wins, the first
    attempt keeping the lead on ties (top_decoders.py:190-202)."""
    if M < 1:
        raise ConfigurationError("M must be >= 1")
    alpha = _alpha(spec, alpha)
    seeds = rng.integers(0, 2 ** 63 - 1, size=M, dtype=np.int64)
    maps: list = []
    for i in range(M):
        g = np.random.default_rng(int(seeds[i])) if sampler is None else None
        maps += _attempt_maps(spec, L, g, sampler)
    return _run(spec, alpha, L, M, maps, True)


def fht_fscl_decode(spec: CodeSpec, alpha, L: int, trace=None) -> DecodeResult:
    """FHT-FSCL, permutations off (top_decoders.py:170-171)."""
    alpha = _alpha(spec, alpha)
    if trace is not None:
        _trace(spec, L, False, trace)
    return _run(spec, alpha, L, 1, None, False)


def fht_fsc_decode(spec: CodeSpec, alpha, trace=None) -> DecodeResult:
    """FHT-FSC: L = 1, permutations off (top_decoders.py:174-175)."""
    return fht_fscl_decode(spec, alpha, 1, trace=trace)


def aut_ssc(spec: CodeSpec, alpha, P: int, rng, sampler=None) -> DecodeResult:
    """P SSC decodes under random permutations; the candidate with the
    largest correlation wins, the first on ties (top_decoders.py:235-249).
    Maps are drawn one per decode like the reference (sample_affine, or the
    ``sampler`` plugin).  ``pm`` is NaN as in the reference; ``attempt`` is
    the winning decode."""
    if P < 1:
        raise ConfigurationError("P must be >= 1")
    alpha = _alpha(spec, alpha)
    if rng is None and sampler is None:
        raise ConfigurationError("Aut-SSC needs an rng")
    maps = [sampler() if sampler is not None else sample_affine(spec.m, rng) for _ in range(P)]
    plan = get_plan(spec.r, spec.m, 1, P, True, DEFAULT_DTYPE, aut_ssc=True)
    res = plan.decode(alpha[None, :], raw_maps=maps_to_raw(maps, spec.m).reshape(1, P, 1, spec.m + 1))
    return DecodeResult(codeword=res["cw"][0].astype(np.uint8), pm=float("nan"),
                        attempt=int(res["attempt"][0]), path=0)


def decode(spec: CodeSpec, alpha, cfg: DecoderConfig, rng) -> DecodeResult:
    """Dispatch one frame (top_decoders.py:252-271) for the p-FHT-FSCL family
    and Aut-SSC."""
    algo = cfg.algorithm
    if algo == "FHT-FSC":
        return fht_fsc_decode(spec, alpha)
    if algo == "FHT-FSCL":
        return fht_fscl_decode(spec, alpha, cfg.L)
    if algo == "p-FHT-FSCL":
        if not cfg.permutations_enabled:
            return fht_fscl_decode(spec, alpha, cfg.L)
        if cfg.M > 1:
            return ensemble_decode(spec, alpha, cfg.L, cfg.M, rng)
        return p_fht_fscl(spec, alpha, cfg.L, rng)
    if algo == "Aut-SSC":
        return aut_ssc(spec, alpha, cfg.P, rng)
    raise ConfigurationError(f"algorithm {algo!r} is not part of this decoder "
                             f"(supported: {', '.join(SUPPORTED)})")
