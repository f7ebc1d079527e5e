// Lane-per-frame float32 kernel for single-path decoding without
// permutations — FHT-FSC (fht_fsc_decode, top_decoders.py:174-175: L = 1,
// M = 1) on short codes (N <= 64).  BASELINE config 1 (RM(2,5), N = 32).
//
// The warp-per-(frame, attempt) throughput kernel (rmfht_fast.cuh) spends a
// whole warp on a 32-element frame whose tree is a handful of tiny nodes; it
// ran at 2% of the HBM bound.  Here each thread decodes one frame with the
// node vectors in registers: the compile-time recursion of _decode_node
// (top_decoders.py:72-113) with
//   f (list_engine.py:15-20) as one min.xorsign.abs per pair,
//   g (:23-27) as hi + (1 - 2c) lo,
//   the FHT node (fht_decode.py:28-48,101-126) with L = 1: butterflies in the
//     reference's stage order, the first bin of maximal |w| (stable argsort
//     of -|w|), codeword bit j = parity(~b & ~j & (n-1)) ^ [w_b < 0],
//   the SPC node (list_engine.py:68-119) with L = 1: hard decisions, and on
//     odd parity the first least reliable position flipped (the single
//     split j = 1 never keeps the flip: its metric is >= the keep's),
//   propagate_hard (:30-36) as bit-field XORs.
// With one path no decision depends on the accumulated metric, so the
// kernel does not accumulate it; it reports the decided codeword's metric
// from the channel LLRs exactly as the other float32 kernels do
// (rmfht::CorrPm: positions i = 32 t + l summed per l in double in
// ascending t, then the xor tree 16 .. 1, rounded once), so its outputs are
// bit-identical with theirs and with the float32 oracle.
//
// Memory: 4N bytes of LLRs in (8 x LDG.128 per thread for N = 32), one
// codeword word, pm, attempt and path out per frame.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "rmfht_kernels.cuh"

namespace rmfht_lane {

using u32 = uint32_t;
using u64 = unsigned long long;

__device__ __forceinline__ float f_op(float a, float b) {
    float r;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// bits of a node of size n = 2^SS: bit j = hard decision of element j
template <int SS>
using BitsT = typename std::conditional<(SS > 5), u64, u32>::type;

// fhtl, L = 1
template <int SS>
__device__ __forceinline__ BitsT<SS> fht1(const float (&x)[1 << SS]) {
    constexpr int n = 1 << SS;
    float w[n];
#pragma unroll
    for (int k = 0; k < n; k++) w[k] = x[k];
    // stage t: half = 2^(s - t - 1); lo' = hi - lo, hi' = hi + lo
#pragma unroll
    for (int t = 0; t < SS; t++) {
        const int half = n >> (t + 1);
#pragma unroll
        for (int lo = 0; lo < n; lo++) {
            if (lo & half) continue;
            const float a = w[lo], b = w[lo + half];
            w[lo] = b - a;
            w[lo + half] = b + a;
        }
    }
    // first bin of maximal |w| (ties -> lower bin)
    float best = fabsf(w[0]);
    int bin = 0;
    float wb = w[0];
#pragma unroll
    for (int k = 1; k < n; k++) {
        const float a = fabsf(w[k]);
        if (a > best) { best = a; bin = k; wb = w[k]; }
    }
    // codeword: bit j = parity(~b & ~j & (n-1)) ^ sign; as a bit pattern over j,
    // parity(B & ~j) = parity(B) ^ parity(B & j) with B = ~b & (n-1)
    const u32 B = (u32)(~bin) & (u32)(n - 1);
    using BT = BitsT<SS>;
    BT P = 0;
    constexpr u64 pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                            0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
#pragma unroll
    for (int k = 0; k < SS; k++)
        if ((B >> k) & 1u) P ^= (BT)pat[k];
    const int c0 = (__popc(B) & 1) ^ (wb < 0.f ? 1 : 0);
    constexpr BT VM = (n >= 8 * (int)sizeof(BT)) ? (BT)~(BT)0 : (BT)(((BT)1 << n) - 1);
    return (c0 ? ~P : P) & VM;
}

// spc_decode_list, L = 1
template <int SS>
__device__ __forceinline__ BitsT<SS> spc1(const float (&x)[1 << SS]) {
    constexpr int n = 1 << SS;
    using BT = BitsT<SS>;
    BT bits = 0;
    float amin = fabsf(x[0]);
    int imin = 0;
#pragma unroll
    for (int k = 0; k < n; k++) {
        bits |= (BT)(x[k] < 0.f ? 1 : 0) << k;
        const float a = fabsf(x[k]);
        if (k > 0 && a < amin) { amin = a; imin = k; }  // first minimum (stable argsort)
    }
    int par;
    if constexpr (sizeof(BT) == 8) par = __popcll(bits) & 1;
    else par = __popc(bits) & 1;
    return bits ^ ((BT)par << imin);
}

template <int RR, int SS>
__device__ __forceinline__ BitsT<SS> node(const float (&x)[1 << SS]) {
    constexpr int n = 1 << SS, h = n / 2;
    if constexpr (RR == 1) {
        return fht1<SS>(x);
    } else if constexpr (RR == SS - 1) {
        return spc1<SS>(x);
    } else {
        float xl[h];
#pragma unroll
        for (int k = 0; k < h; k++) xl[k] = f_op(x[k], x[k + h]);
        const BitsT<SS - 1> bl = node<RR - 1, SS - 1>(xl);
        float xr[h];
#pragma unroll
        for (int k = 0; k < h; k++) xr[k] = ((bl >> k) & 1) ? x[k + h] - x[k] : x[k + h] + x[k];
        const BitsT<SS - 1> br = node<RR, SS - 1>(xr);
        return ((BitsT<SS>)br << h) | (BitsT<SS>)(bl ^ br);
    }
}

template <int R, int MM>
__global__ void __launch_bounds__(256) lane_kernel(rmfht::Params<float> prm) {
    constexpr int N = 1 << MM, NW = N >= 32 ? N / 32 : 1;
    static_assert(N >= 4 && N <= 64, "lane kernel: 4 <= N <= 64");
    const long long stride = (long long)gridDim.x * blockDim.x;
    // software pipeline: the next frame's LLRs are in flight while this one
    // decodes (the kernel is bound by HBM latency: two frames per thread in
    // flight double the memory-level parallelism)
    float4 nxt[N / 4];
    auto load = [&](long long f) {
        const float4* src = reinterpret_cast<const float4*>(prm.llr + f * N);
#pragma unroll
        for (int k = 0; k < N / 4; k++) nxt[k] = __ldg(src + k);
    };
    long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (f < prm.B) load(f);
    for (; f < prm.B; f += stride) {
        float x[N];
#pragma unroll
        for (int k = 0; k < N / 4; k++) {
            x[4 * k] = nxt[k].x; x[4 * k + 1] = nxt[k].y; x[4 * k + 2] = nxt[k].z; x[4 * k + 3] = nxt[k].w;
        }
        if (f + stride < prm.B) load(f + stride);
        const BitsT<MM> bits = node<R, MM>(x);
        // reported pm: rmfht::CorrPm's order, lane l's positions l, l + 32
        double q[32];
#pragma unroll
        for (int l = 0; l < 32; l++) {
            double acc = 0.0;
#pragma unroll
            for (int i = l; i < N; i += 32) {
                const int c = (int)((bits >> i) & 1);
                if ((x[i] < 0.f) != (c != 0)) acc += fabs((double)x[i]);
            }
            q[l] = acc;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
            for (int l = 0; l < off; l++) q[l] = q[l] + q[l + off];
        const float pm = (float)q[0];
#pragma unroll
        for (int t = 0; t < NW; t++) {
            const u32 word = (u32)(bits >> (32 * t));
            prm.cw[f * NW + t] = word;
            if (prm.att_cw) prm.att_cw[f * NW + t] = word;
        }
        prm.pm[f] = pm;
        prm.attempt[f] = 0;
        prm.path[f] = 0;
        if (prm.att_pm) prm.att_pm[f] = pm;
    }
}

}  // namespace rmfht_lane
