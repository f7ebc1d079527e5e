"""BPSK/AWGN frames for the decoder (host-side input generation).

``harness_frames`` replays the reference harness stream frame by frame
(``harness.py:103-107``: ``frame_rng(seed, q, k)`` → info bits → polar
transform → BPSK + inverse-CDF AWGN → LLR = 2y/sigma^2), so a GPU run can
decode exactly the frames the reference's ``run_job`` would.
``synthetic_frames`` draws the same distribution vectorised over a batch
(seeded, not stream-identical) for throughput runs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import ndtri

from .rm_core import CodeSpec, ConfigurationError, polar_transform, random_message

_U53 = float(1 << 53)


@dataclass(frozen=True)
class ChannelConfig:
    """channel_model.py:21-33"""
    ebn0_db: float
    rate: float
    sigma: float
    seed: int = 0

    @classmethod
    def for_rate(cls, ebn0_db: float, rate: float, seed: int = 0) -> "ChannelConfig":
        if rate <= 0 or rate > 1:
            raise ConfigurationError(f"rate {rate} outside (0, 1]")
        sigma = 1.0 / np.sqrt(2.0 * rate * 10.0 ** (ebn0_db / 10.0))
        return cls(ebn0_db=ebn0_db, rate=rate, sigma=float(sigma), seed=seed)


def frame_rng(seed: int, *key: int) -> np.random.Generator:
    """Per-frame substream (channel_model.py:36-38)."""
    return np.random.default_rng(np.random.SeedSequence((int(seed),) + tuple(int(k) for k in key)))


def gaussian(rng: np.random.Generator, size: int) -> np.ndarray:
    u = (rng.integers(0, 1 << 53, size=size).astype(np.float64) + 0.5) / _U53
    return ndtri(u)


def transmit(x, cfg: ChannelConfig, rng, zero_noise: bool = False) -> np.ndarray:
    symbols = 1.0 - 2.0 * np.asarray(x).astype(np.float64)
    if zero_noise:
        return symbols
    return symbols + cfg.sigma * gaussian(rng, symbols.shape[-1])


def llr(y, cfg: ChannelConfig) -> np.ndarray:
    if cfg.sigma <= 0:
        raise ConfigurationError("sigma must be positive")
    return 2.0 * np.asarray(y, dtype=np.float64) / (cfg.sigma ** 2)


def harness_frames(spec: CodeSpec, ebn0_db: float, seed: int, point: int, start: int, count: int,
                   zero_noise: bool = False):
    """Frames start..start+count of SNR point `point`, exactly as the reference
    harness draws them.  Returns (x uint8 [count, N], llr float64 [count, N],
    rngs) — the per-frame generators continue where the decoder would."""
    chan = ChannelConfig.for_rate(ebn0_db, spec.rate, seed)
    xs = np.zeros((count, spec.N), dtype=np.uint8)
    ls = np.zeros((count, spec.N), dtype=np.float64)
    rngs = []
    for i, k in enumerate(range(start, start + count)):
        g = frame_rng(seed, point, k)
        x = polar_transform(random_message(spec, g))
        xs[i] = x
        ls[i] = llr(transmit(x, chan, g, zero_noise), chan)
        rngs.append(g)
    return xs, ls, rngs


def synthetic_frames(spec: CodeSpec, ebn0_db: float, B: int, seed: int, dtype=np.float32):
    """B frames with uniform info bits, BPSK over AWGN, vectorised."""
    rng = np.random.default_rng(seed)
    chan = ChannelConfig.for_rate(ebn0_db, spec.rate)
    u = np.zeros((B, spec.N), dtype=np.uint8)
    u[:, list(spec.info_set)] = rng.integers(0, 2, size=(B, spec.K), dtype=np.uint8)
    x = polar_transform(u)
    y = (1.0 - 2.0 * x) + chan.sigma * rng.standard_normal((B, spec.N))
    return x, (2.0 * y / chan.sigma ** 2).astype(dtype)


# ------------------------------------------------- on-device generation
def gen_frames_device(spec: CodeSpec, chan: ChannelConfig, point: int, frame0: int, llr, tx,
                      zero_noise: bool = False, stream=None) -> None:
    """Frames frame0 .. frame0+B-1 of SNR point `point` generated on the GPU
    (rmfht_gen_frames: uniform info bits, polar transform, BPSK + inverse-CDF
    AWGN, float32 LLR = 2y/sigma^2).  `llr` float32 [B, N] and `tx` int32
    [B, max(1, N/32)] are CUDA tensors; stream-ordered, no host sync."""
    from . import _native
    from .decoder import _check, _torch
    torch = _torch()
    st = stream if stream is not None else torch.cuda.current_stream()
    B = llr.shape[0]
    if tuple(llr.shape) != (B, spec.N) or llr.dtype != torch.float32 or tx.shape[0] != B:
        raise ValueError("llr must be float32 [B, N] and tx int32 [B, words]")
    _check(_native.lib().rmfht_gen_frames(spec.r, spec.m, chan.seed & ((1 << 64) - 1), point, frame0, B,
                                          chan.sigma, int(zero_noise), llr.data_ptr(), tx.data_ptr(),
                                          st.cuda_stream))


def count_errors_device(spec: CodeSpec, llr, tx, cw, counts, stream=None) -> None:
    """Accumulate [frame errors, ML-lower-bound errors] of decoded words `cw`
    against transmitted `tx` into the int64[2] CUDA tensor `counts`
    (harness.py:79-84,109-112)."""
    from . import _native
    from .decoder import _check, _torch
    torch = _torch()
    st = stream if stream is not None else torch.cuda.current_stream()
    _check(_native.lib().rmfht_count_errors(spec.m, llr.data_ptr(), tx.data_ptr(), cw.data_ptr(), llr.shape[0],
                                            counts.data_ptr(), st.cuda_stream))
