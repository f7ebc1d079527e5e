"""On-device frame generation and error counting (rmfht_gen_frames /
rmfht_count_errors) against a numpy restatement of the
same counter-based streams and the reference's frame pipeline
(rm_core.polar_transform, channel_model.transmit/llr, harness.ml_lower_bound).
Messages and codewords are bit-exact; LLRs agree to float32 rounding of the
inverse normal CDF (CUDA normcdfinv vs scipy ndtri)."""
import numpy as np
import pytest
from scipy.special import ndtri

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def frame_key(seed, point, frame):
    with np.errstate(over="ignore"):
        a = mix64(np.uint64((seed * 0xD1B54A32D192ED03) & M64) ^ np.uint64((point * 0xABC98388FB8FAC03) & M64))
        return mix64(a + np.uint64((frame * GAMMA) & M64))


def stream(key, n):
    with np.errstate(over="ignore"):
        j = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(GAMMA)
        return mix64(np.uint64(key) + j)


def host_frame(spec, seed, point, frame, sigma, zero_noise=False):
    """The device's frame, restated: (u, x, llr float32)."""
    from paper_2108_12550_b200.rm_core import polar_transform
    k = frame_key(seed, point, frame)
    kmsg, knoise = mix64(k ^ np.uint64(1)), mix64(k ^ np.uint64(2))
    nw = max(1, spec.N // 32)
    words = (stream(kmsg, nw) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:spec.N]
    u = np.zeros(spec.N, dtype=np.uint8)
    info = list(spec.info_set)
    u[info] = bits[info]
    x = polar_transform(u)
    y = 1.0 - 2.0 * x.astype(np.float64)
    if not zero_noise:
        uu = ((stream(knoise, spec.N) >> np.uint64(11)).astype(np.float64) + 0.5) / float(1 << 53)
        y = y + sigma * ndtri(uu)
    return u, x, (2.0 * y / sigma ** 2).astype(np.float32)


def run_gen(spec, seed, point, frame0, B, sigma, zero_noise=False):
    import torch
    from paper_2108_12550_b200.channel_model import ChannelConfig, gen_frames_device
    chan = ChannelConfig(ebn0_db=0.0, rate=spec.rate, sigma=sigma, seed=seed)
    llr = torch.empty((B, spec.N), dtype=torch.float32, device="cuda")
    tx = torch.empty((B, max(1, spec.N // 32)), dtype=torch.int32, device="cuda")
    gen_frames_device(spec, chan, point, frame0, llr, tx, zero_noise)
    torch.cuda.synchronize()
    words = tx.cpu().numpy().view(np.uint32)
    x = np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little")[:, :spec.N]
    return llr.cpu().numpy(), x


@pytest.mark.parametrize("r,m", [(2, 9), (1, 3), (2, 4), (3, 7), (2, 5), (4, 10)])
def test_frames_match_restated_stream(r, m):
    from paper_2108_12550_b200.channel_model import ChannelConfig
    from paper_2108_12550_b200.rm_core import build_code, is_codeword
    spec = build_code(r, m)
    sigma = ChannelConfig.for_rate(2.0, spec.rate).sigma
    seed, point, frame0, B = 2024, 3, 1000, 67
    llr, x = run_gen(spec, seed, point, frame0, B, sigma)
    for i in (0, 1, 33, B - 1):
        u, xh, lh = host_frame(spec, seed, point, frame0 + i, sigma)
        assert np.array_equal(x[i], xh)                     # bit-exact message + polar transform
        assert is_codeword(spec, x[i])
        np.testing.assert_allclose(llr[i], lh, rtol=4e-7, atol=1e-6)
    # a frame does not depend on the batch that generates it
    llr2, x2 = run_gen(spec, seed, point, frame0 + 33, 5, sigma)
    assert np.array_equal(x2, x[33:38]) and np.array_equal(llr2, llr[33:38])


def test_zero_noise_frames_are_scaled_bpsk():
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    llr, x = run_gen(spec, 5, 0, 0, 100, 0.8, zero_noise=True)
    np.testing.assert_array_equal(llr, ((1.0 - 2.0 * x) * 2.0 / 0.64).astype(np.float32))


def test_noise_statistics():
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 9)
    sigma = 0.75
    llr, x = run_gen(spec, 9, 1, 0, 8192, sigma)
    z = (llr.astype(np.float64) * sigma ** 2 / 2.0 - (1.0 - 2.0 * x)) / sigma
    assert abs(z.mean()) < 5e-3 and abs(z.std() - 1.0) < 5e-3
    # info bits uniform: half of the transmitted bits are ones
    assert abs(x.mean() - 0.5) < 5e-3


def test_count_errors_matches_host():
    import torch
    from paper_2108_12550_b200.channel_model import count_errors_device
    from paper_2108_12550_b200.rm_core import build_code
    spec = build_code(2, 7)
    rng = np.random.default_rng(3)
    B = 3000
    llr = rng.normal(size=(B, spec.N)).astype(np.float32)
    x = rng.integers(0, 2, size=(B, spec.N)).astype(np.uint8)
    xh = x.copy()
    flip = rng.random(B) < 0.3
    for i in np.flatnonzero(flip):
        xh[i, rng.integers(0, spec.N, size=rng.integers(1, 6))] ^= 1
    pack = lambda b: torch.from_numpy(np.packbits(b, axis=-1, bitorder="little").view(np.int32).copy()).cuda()
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    count_errors_device(spec, torch.from_numpy(llr).cuda(), pack(x), pack(xh), counts)
    count_errors_device(spec, torch.from_numpy(llr).cuda(), pack(x), pack(xh), counts)  # accumulates
    wrong = np.any(xh != x, axis=1)
    a = llr.astype(np.float64)
    ml = wrong & (np.sum((1.0 - 2.0 * xh) * a, axis=1) >= np.sum((1.0 - 2.0 * x) * a, axis=1))
    assert counts.cpu().tolist() == [2 * int(wrong.sum()), 2 * int(ml.sum())]


def test_device_harness_matches_host_harness_statistically():
    """frames='device' and frames='host' simulate the same channel: their
    FER at one point agree (Fisher), and the device run is deterministic."""
    from scipy.stats import fisher_exact
    from paper_2108_12550_b200 import harness
    from paper_2108_12550_b200.top_decoders import DecoderConfig
    cfg = DecoderConfig("p-FHT-FSCL", L=2, M=4)
    job = harness.SimJob(r=2, m=7, decoder=cfg, ebn0_points=(2.0,), max_frames=100000,
                         min_frame_errors=10 ** 9, batch=16384)
    d = harness.run_job(job, frames="device")[0]
    d2 = harness.run_job(job, frames="device")[0]
    h = harness.run_job(job, frames="host")[0]
    assert (d.frames, d.frame_errors, d.ml_lb_fer) == (d2.frames, d2.frame_errors, d2.ml_lb_fer)
    assert d.frames == h.frames == 100000
    p = fisher_exact([[d.frame_errors, d.frames - d.frame_errors], [h.frame_errors, h.frames - h.frame_errors]]).pvalue
    assert p > 1e-3, (d.frame_errors, h.frame_errors)
