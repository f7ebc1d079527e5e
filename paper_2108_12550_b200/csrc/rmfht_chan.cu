// On-device frame generation and error counting: the
// reference harness's per-frame pipeline (harness.py:103-112) — uniform info
// bits at the RM info set (rm_core.py:66-95, random_message :182-186),
// polar transform (:102-118), BPSK + AWGN by the inverse-CDF method and
// LLR = 2y/sigma^2 (channel_model.py:41-61) — and its error / ML-lower-bound
// counting (harness.py:79-84,109-112), so a simulation needs no host frames.
//
// Random streams are counter-based (splitmix64 finalizer over (key + (j+1)
// gamma)), keyed by (seed, point, frame): a frame's bits and noise do not
// depend on the batch that generates it.  tests/test_gpu_chan.py restates
// the streams in numpy.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/rmfht.h"
#include "rmfht_plan.h"

using rmfht_internal::fail;

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// frame key and its two substreams (message bits, noise)
__device__ __forceinline__ uint64_t frame_key(uint64_t seed, long long point, long long frame) {
    return mix64(mix64(seed * 0xD1B54A32D192ED03ull ^ (uint64_t)point * 0xABC98388FB8FAC03ull) +
                 (uint64_t)frame * kGamma);
}
__device__ __forceinline__ uint64_t stream_at(uint64_t key, uint64_t j) { return mix64(key + (j + 1) * kGamma); }

// info position of RM(r, m): row weight 2^popcount(i) >= d = 2^(m-r)
__device__ __forceinline__ uint32_t info_word(int m, int r, int w) {
    uint32_t v = 0;
    const int n = 1 << m;
    for (int b = 0; b < 32 && 32 * w + b < n; b++)
        if (__popc(32 * w + b) >= m - r) v |= 1u << b;
    return v;
}

// one warp per frame; the codeword words live in the warp's shared slice
__global__ void __launch_bounds__(256) gen_frames_kernel(int r, int m, uint64_t seed, long long point,
                                                         long long frame0, long long B, double sigma,
                                                         int zero_noise, float* llr, uint32_t* tx) {
    extern __shared__ uint32_t sw[];
    const int n = 1 << m, nw = n >= 32 ? n / 32 : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* w = sw + warp * nw;
    const long long f = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    if (f >= B) return;
    const uint64_t key = frame_key(seed, point, frame0 + f);
    const uint64_t kmsg = mix64(key ^ 1ull), knoise = mix64(key ^ 2ull);
    // message: uniform bits at the info positions, zeros elsewhere
    for (int j = lane; j < nw; j += 32) w[j] = (uint32_t)stream_at(kmsg, j) & info_word(m, r, j);
    __syncwarp();
    // polar transform: for t < m, x[i] ^= x[i + 2^t] where bit t of i is clear
    const uint32_t inword[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    for (int j = lane; j < nw; j += 32) {
        uint32_t v = w[j];
        for (int t = 0; t < 5 && t < m; t++) v ^= (v >> (1 << t)) & inword[t];
        w[j] = v;
    }
    __syncwarp();
    for (int t = 5; t < m; t++) {
        const int d = 1 << (t - 5);
        for (int j = lane; j < nw; j += 32)
            if (!(j & d)) w[j] ^= w[j + d];
        __syncwarp();
    }
    for (int j = lane; j < nw; j += 32) tx[f * nw + j] = w[j];
    // BPSK + AWGN (inverse CDF of a centred 53-bit uniform), LLR = 2y/sigma^2
    const double s2 = sigma * sigma;
    for (int i = lane; i < n; i += 32) {
        const int x = (w[i >> 5] >> (i & 31)) & 1;
        double y = 1.0 - 2.0 * (double)x;
        if (!zero_noise) {
            const double u = ((double)(stream_at(knoise, (uint64_t)i) >> 11) + 0.5) * 0x1p-53;
            y += sigma * normcdfinv(u);
        }
        llr[f * n + i] = (float)(2.0 * y / s2);
    }
}

// one warp per frame: frame error if the decoded word differs; ML lower
// bound if, in addition, corr(x_hat) >= corr(x_tx), corr(c) = sum (1-2c) alpha
__global__ void __launch_bounds__(256) count_errors_kernel(int m, const float* llr, const uint32_t* tx,
                                                           const uint32_t* cw, long long B,
                                                           unsigned long long* counts) {
    const int n = 1 << m, nw = n >= 32 ? n / 32 : 1;
    const uint32_t last = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long f = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    if (f >= B) return;
    uint32_t diff = 0;
    for (int j = lane; j < nw; j += 32) diff |= (cw[f * nw + j] ^ tx[f * nw + j]) & last;
    if (!__any_sync(0xffffffffu, diff != 0)) return;
    double ch = 0.0, ct = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double a = (double)llr[f * n + i];
        const int xh = (cw[f * nw + (i >> 5)] >> (i & 31)) & 1, xt = (tx[f * nw + (i >> 5)] >> (i & 31)) & 1;
        ch += xh ? -a : a;
        ct += xt ? -a : a;
    }
    for (int off = 16; off >= 1; off >>= 1) {
        ch += __shfl_xor_sync(0xffffffffu, ch, off);
        ct += __shfl_xor_sync(0xffffffffu, ct, off);
    }
    if (lane == 0) {
        atomicAdd(&counts[0], 1ull);
        if (ch >= ct) atomicAdd(&counts[1], 1ull);
    }
}

}  // namespace

extern "C" {

int rmfht_gen_frames(int r, int m, uint64_t seed, long long point, long long frame0, long long B, double sigma,
                     int zero_noise, float* d_llr, uint32_t* d_tx, void* stream) {
    if (m < 2 || m > 14 || r < 1 || r > m - 1) return fail(RMFHT_ECONFIG, "RM(r, m) outside 1 <= r <= m-1, 2 <= m <= 14");
    if (B < 0 || !(sigma > 0.0)) return fail(RMFHT_EVALUE, "B must be >= 0 and sigma > 0");
    if (B == 0) return 0;
    if (!d_llr || !d_tx) return fail(RMFHT_EVALUE, "output pointer is NULL");
    const int nw = m >= 5 ? (1 << m) / 32 : 1;
    const int wpb = 8;
    const long long blocks = (B + wpb - 1) / wpb;
    gen_frames_kernel<<<(unsigned)blocks, wpb * 32, wpb * nw * sizeof(uint32_t), static_cast<cudaStream_t>(stream)>>>(
        r, m, seed, point, frame0, B, sigma, zero_noise, d_llr, d_tx);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("gen_frames launch: ") + cudaGetErrorString(e));
    return 0;
}

int rmfht_count_errors(int m, const float* d_llr, const uint32_t* d_tx, const uint32_t* d_cw, long long B,
                       unsigned long long* d_counts, void* stream) {
    if (m < 2 || m > 14) return fail(RMFHT_ECONFIG, "m outside [2, 14]");
    if (B < 0) return fail(RMFHT_EVALUE, "negative batch");
    if (B == 0) return 0;
    if (!d_llr || !d_tx || !d_cw || !d_counts) return fail(RMFHT_EVALUE, "pointer is NULL");
    const int wpb = 8;
    const long long blocks = (B + wpb - 1) / wpb;
    count_errors_kernel<<<(unsigned)blocks, wpb * 32, 0, static_cast<cudaStream_t>(stream)>>>(m, d_llr, d_tx, d_cw,
                                                                                             B, d_counts);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("count_errors launch: ") + cudaGetErrorString(e));
    return 0;
}

}  // extern "C"
