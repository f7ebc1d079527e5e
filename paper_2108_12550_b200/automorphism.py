"""Affine automorphisms x -> A x + b of RM codes, on the host.

The decoder consumes permutations as a *table* (one record per map, in the
reference's consumption order).  This module produces those tables:

* ``sample_affine_batch`` replays the reference sampler's random-number
  stream exactly (``automorphism.py:144-161``): the same ``rng.integers``
  calls with the same sizes, accepting invertible candidates in order.  The
  drop-in single-frame API uses it so that ``decode(spec, alpha, cfg, rng)``
  consumes ``rng`` exactly like the reference.
* ``random_raw_table`` is a bulk, vectorised sampler (uniform over
  GL(m,2) x F_2^m, seeded) for batched decoding where reference-stream
  replay is not required.

Raw map format (shared with the C-ABI, ``include/rmfht.h``): ``m_root + 1``
uint16 per map — row masks of A in ``[0, m_node)`` (bit j of row r is
A[r, j]), zeros up to ``m_root``, and the shift b at index ``m_root``.
"""

from __future__ import annotations

import numpy as np

from .rm_core import ConfigurationError


class AffineMap:
    """Element (A, b) acting on indices by i -> A bits(i) xor b, LSB-first.

    Duck-compatible with the reference's ``AffinePermutation`` (``.a``,
    ``.b``, ``.m``, ``.perm``, ``.inv``), so reference samplers can be passed
    to the drop-in API and vice versa.
    """

    __slots__ = ("a", "b", "m", "_perm", "_inv")

    def __init__(self, a, b):
        self.a = np.asarray(a, dtype=np.uint8)
        self.b = np.asarray(b, dtype=np.uint8)
        self.m = self.a.shape[0]
        if self.a.shape != (self.m, self.m) or self.b.shape != (self.m,):
            raise ValueError("shape mismatch between A and b")
        self._perm = None
        self._inv = None

    @classmethod
    def identity(cls, m: int) -> "AffineMap":
        return cls(np.eye(m, dtype=np.uint8), np.zeros(m, dtype=np.uint8))

    @classmethod
    def from_masks(cls, masks, shift: int, m: int) -> "AffineMap":
        masks = np.asarray(masks, dtype=np.int64)
        a = ((masks[:, None] >> np.arange(m)) & 1).astype(np.uint8)
        b = ((int(shift) >> np.arange(m)) & 1).astype(np.uint8)
        return cls(a, b)

    def masks(self) -> np.ndarray:
        return (self.a.astype(np.int64) << np.arange(self.m)).sum(axis=1)

    def shift(self) -> int:
        return int((self.b.astype(np.int64) << np.arange(self.m)).sum())

    @property
    def perm(self) -> np.ndarray:
        if self._perm is None:
            n = 1 << self.m
            bits = (np.arange(n)[:, None] >> np.arange(self.m)) & 1
            out = (bits @ self.a.T.astype(np.int64)) & 1
            self._perm = (out << np.arange(self.m)).sum(axis=1) ^ self.shift()
        return self._perm

    @property
    def inv(self) -> np.ndarray:
        if self._inv is None:
            inv = np.empty_like(self.perm)
            inv[self.perm] = np.arange(self.perm.shape[0])
            self._inv = inv
        return self._inv


def gf2_invertible_masks(masks: np.ndarray, m: int) -> np.ndarray:
    """Vectorised GF(2) invertibility of row-mask matrices, shape (..., m)."""
    rows = np.array(masks, dtype=np.int64).reshape(-1, m)
    count = rows.shape[0]
    basis = np.zeros((count, m), dtype=np.int64)  # basis[:, bit] = vector with leading bit
    ok = np.ones(count, dtype=bool)
    for r in range(m):
        x = rows[:, r].copy()
        placed = np.zeros(count, dtype=bool)
        for bit in range(m - 1, -1, -1):
            has = ((x >> bit) & 1).astype(bool)
            b = basis[:, bit]
            red = has & (b != 0)
            x[red] ^= b[red]
            place = has & (b == 0)
            basis[place, bit] = x[place]
            x[place] = 0
            placed |= place
        ok &= placed  # a row that reduced to zero is dependent
    return ok.reshape(np.shape(masks)[:-1])


def sample_affine(m: int, rng: np.random.Generator) -> AffineMap:
    """Reference-stream replay of ``sample_affine`` (automorphism.py:127-141):
    m row masks per candidate until invertible, then b — the draws aut_ssc
    makes once per decode."""
    if m < 1:
        raise ValueError("m must be >= 1")
    while True:
        masks = rng.integers(0, 1 << m, size=m, dtype=np.int64)
        if gf2_invertible_masks(masks[None, :], m)[0]:
            break
    b = int(rng.integers(0, 1 << m))
    return AffineMap.from_masks(masks, b, m)


def sample_affine_batch(m: int, count: int, rng: np.random.Generator) -> list:
    """Reference-stream replay of ``sample_affine_batch`` (automorphism.py:144-161)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    out: list = []
    while len(out) < count:
        todo = count - len(out)
        attempts = 4 * todo + 4
        masks = rng.integers(0, 1 << m, size=(attempts, m), dtype=np.int64)
        shifts = rng.integers(0, 1 << m, size=attempts, dtype=np.int64)
        good = gf2_invertible_masks(masks, m)
        for t in np.flatnonzero(good):
            out.append(AffineMap.from_masks(masks[t], int(shifts[t]), m))
            if len(out) == count:
                break
    return out


def maps_to_raw(maps, m_root: int) -> np.ndarray:
    """Pack AffineMap-like objects (``.a``, ``.b``) into raw records."""
    raw = np.zeros((len(maps), m_root + 1), dtype=np.uint16)
    for i, p in enumerate(maps):
        a = np.asarray(p.a, dtype=np.int64)
        mn = a.shape[0]
        if mn > m_root:
            raise ConfigurationError("map larger than the code")
        raw[i, :mn] = (a << np.arange(mn)).sum(axis=1)
        raw[i, m_root] = int((np.asarray(p.b, dtype=np.int64) << np.arange(mn)).sum())
    return raw


def raw_to_maps(raw: np.ndarray, sizes) -> list:
    raw = np.asarray(raw)
    m_root = raw.shape[-1] - 1
    flat = raw.reshape(-1, m_root + 1)
    return [AffineMap.from_masks(flat[i, :mn], int(flat[i, m_root]), mn)
            for i, mn in zip(range(flat.shape[0]), np.resize(np.asarray(sizes), flat.shape[0]))]


def random_raw_table(rng: np.random.Generator, lead_shape: tuple, sizes, m_root: int,
                     identity_root: int = 0) -> np.ndarray:
    """Bulk sampler: uniform maps for every slot of a ``lead_shape + (S,)`` table.

    ``sizes[s]`` is the variable count of slot s (from ``plan.map_sizes``).
    ``identity_root`` > 0 makes the first ``identity_root`` slots of attempt 0
    (the L root maps) the identity — BASELINE's "decoder 0 = identity".
    The attempt axis is ``lead_shape[-1]``.
    """
    sizes = np.asarray(sizes, dtype=np.int64)
    S = sizes.shape[0]
    total = int(np.prod(lead_shape)) * S
    raw = np.zeros((total, m_root + 1), dtype=np.uint16)
    slot_size = np.resize(sizes, total)
    for mn in np.unique(sizes):
        idx = np.flatnonzero(slot_size == mn)
        need = idx.shape[0]
        got = np.zeros((0, int(mn)), dtype=np.int64)
        while got.shape[0] < need:
            cand = rng.integers(0, 1 << int(mn), size=(int((need - got.shape[0]) * 3.6) + 64, int(mn)),
                                dtype=np.int64)
            got = np.concatenate([got, cand[gf2_invertible_masks(cand, int(mn))]])
        raw[idx, :mn] = got[:need]
        raw[idx, m_root] = rng.integers(0, 1 << int(mn), size=need, dtype=np.int64)
    raw = raw.reshape(tuple(lead_shape) + (S, m_root + 1))
    if identity_root:
        ident = np.zeros(m_root + 1, dtype=np.uint16)
        ident[:m_root] = 1 << np.arange(m_root)
        raw[..., 0, :identity_root, :] = ident
    return raw
