// Aut-SSC, register-resident variant for compiled (r, m) shapes (rmfht_ssc.cu
// dispatches to it when the shape is in RMFHT_SSC_SHAPES).  One warp = one
// SSC decode; a node vector of n = 2^s elements lives in "channel layout":
// element e = k*32 + lane is register k of lane `lane` (n >= 32), or lane e
// of register 0 (n < 32, lanes >= n idle).  The tree (ssc_decode,
// top_decoders.py:205-230) is unrolled at compile time: f / g of a node whose
// halves differ in a register bit are lane-local, in a lane bit one shuffle;
// a node's hard decisions come back as one packed word per lane (bit k =
// element k*32 + lane).  Sums keep numpy's pairwise order (repetition leaves,
// the correlation score), so results are bit-identical to the shared-memory
// kernel, the oracle and — in float64 — the reference.
#pragma once

namespace rmfht_ssc {

template <int S>
struct NodeL {
    static constexpr int n = 1 << S;
    static constexpr int V = S >= 5 ? (1 << (S - 5)) : 1;  // registers per lane
};

// numpy pairwise sum of the node vector (n = 2^S elements, channel layout);
// the result in every lane
template <typename T, int S>
__device__ __forceinline__ T node_pw_sum(const T (&x)[NodeL<S>::V], int lane) {
    constexpr int n = 1 << S;
    if constexpr (n < 8) {
        T res = 0;
#pragma unroll
        for (int e = 0; e < n; e++) res += __shfl_sync(kFull, x[0], e);
        return res;
    } else {
        // blocks of up to 128: accumulator j (lane j < 8) sums elements
        // 8t + j of the block in t order, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7));
        // blocks combine as a balanced tree (pairwise halving)
        constexpr int BL = n < 128 ? n : 128, NB = n / BL;
        T blk[NB];
        const int j = lane & 7;
#pragma unroll
        for (int b = 0; b < NB; b++) {
            T r = 0;
#pragma unroll
            for (int t = 0; t < BL / 8; t++) {
                const int e0 = b * BL + 8 * t;  // element of accumulator 0
                const T v = __shfl_sync(kFull, x[e0 >> 5], (e0 & 31) + j);
                r = t == 0 ? v : r + v;
            }
            r += __shfl_xor_sync(kFull, r, 1);
            r += __shfl_xor_sync(kFull, r, 2);
            r += __shfl_xor_sync(kFull, r, 4);
            blk[b] = __shfl_sync(kFull, r, 0);
        }
#pragma unroll
        for (int w = 1; w < NB; w <<= 1)
#pragma unroll
            for (int b = 0; b + w < NB; b += 2 * w) blk[b] = blk[b] + blk[b + w];
        return blk[0];
    }
}

// SSC of one node; returns the packed hard decisions of this lane
template <typename T, int R, int S>
__device__ __forceinline__ uint32_t ssc_node(const T (&x)[NodeL<S>::V], int lane) {
    using NL = NodeL<S>;
    constexpr int n = NL::n, V = NL::V;
    if constexpr (R < 0) {
        return 0u;
    } else if constexpr (R == S) {
        uint32_t w = 0;
#pragma unroll
        for (int k = 0; k < V; k++) w |= (x[k] < T(0) ? 1u : 0u) << k;
        return w;
    } else if constexpr (R == 0) {
        const T sum = node_pw_sum<T, S>(x, lane);
        return sum < T(0) ? (V >= 32 ? 0xffffffffu : ((1u << V) - 1u)) : 0u;
    } else if constexpr (R == S - 1) {
        // SPC: hard decisions; odd parity flips the first minimum of |x|
        const bool act = n >= 32 || lane < n;
        uint32_t w = 0;
        T bv = 0;
        int be = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < V; k++) {
            w |= (act && x[k] < T(0) ? 1u : 0u) << k;
            const T v = x[k] < T(0) ? -x[k] : x[k];
            if (act && (be == 0x7fffffff || v < bv)) { bv = v; be = k * 32 + lane; }
        }
        // argmin over the node's lanes only (log2(min(n, 32)) steps; every
        // participating lane holds a candidate)
#pragma unroll
        for (int off = (n < 32 ? n : 32) / 2; off >= 1; off >>= 1) {
            const T ov = __shfl_xor_sync(kFull, bv, off);
            const int oe = __shfl_xor_sync(kFull, be, off);
            if (ov < bv || (ov == bv && oe < be)) {
                bv = ov;
                be = oe;
            }
        }
        const int odd = __popc(__ballot_sync(kFull, __popc(w) & 1)) & 1;
        if (odd && (be & 31) == lane) w ^= 1u << (be >> 5);
        return w;
    } else {
        using CL = NodeL<S - 1>;
        T y[CL::V];
        if constexpr (S >= 6) {
            constexpr int H = V / 2;  // halves differ in register bit S-6
#pragma unroll
            for (int k = 0; k < H; k++) y[k] = f_op(x[k], x[k + H]);
            const uint32_t lw = ssc_node<T, R - 1, S - 1>(y, lane);
#pragma unroll
            for (int k = 0; k < H; k++) y[k] = g_op(x[k], x[k + H], (int)((lw >> k) & 1u));
            const uint32_t rw = ssc_node<T, R, S - 1>(y, lane);
            return (lw ^ rw) | (rw << H);  // propagate_hard, list_engine.py:30-36
        } else {
            constexpr int h = n / 2;  // halves differ in lane bit S-1
            const T o = __shfl_xor_sync(kFull, x[0], h);
            y[0] = f_op(x[0], o);  // meaningful in lanes < h
            const uint32_t lw = ssc_node<T, R - 1, S - 1>(y, lane);
            y[0] = g_op(x[0], o, (int)(lw & 1u));
            const uint32_t rw = ssc_node<T, R, S - 1>(y, lane);
            const uint32_t up = __shfl_xor_sync(kFull, rw, h);  // lanes h..n-1: the right child's bit
            return (lane & h) ? (up & 1u) : ((lw ^ rw) & 1u);
        }
    }
}

// linear part of an affine map from its columns (held in registers)
template <int MM>
__device__ __forceinline__ unsigned rec_lin(const unsigned* cols, unsigned x) {
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < MM; k++) v ^= ((x >> k) & 1u) ? (unsigned)cols[k] : 0u;
    return v;
}

template <typename T, int R, int MM>
__global__ void __launch_bounds__(256) aut_ssc_reg_kernel(rmfht::Params<T> prm) {
    constexpr int N = 1 << MM, V = NodeL<MM>::V, REC = 2 * MM + 2;
    static_assert(MM >= 5 && MM <= 10, "register Aut-SSC: 32 <= N <= 1024");
    extern __shared__ __align__(16) unsigned char smem[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* alpha = reinterpret_cast<T*>(smem);
    uint32_t* cww = reinterpret_cast<uint32_t*>(smem + sizeof(T) * N) + 32 * warp;  // codeword words of the warp
    uint16_t* recw = reinterpret_cast<uint16_t*>(smem + sizeof(T) * N + 128 * nw) + 32 * warp;
    T* red_score = reinterpret_cast<T*>(smem + sizeof(T) * N + 128 * nw + 64 * nw);
    int* red_p = reinterpret_cast<int*>(red_score + nw);
    const int P = prm.M;
    for (long long f = blockIdx.x; f < prm.B; f += gridDim.x) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = prm.llr[f * N + i];
        __syncthreads();
        T best = 0;
        int bestp = -1;
        uint32_t bestword = 0;
        for (int p = warp; p < P; p += nw) {
            const uint16_t* g = prm.maps + ((size_t)f * P + p) * REC;
            if (lane < REC) recw[lane] = g[lane];
            __syncwarp();
            // the map's columns in registers (every index below is an XOR of them)
            unsigned cols[MM], icols[MM];
#pragma unroll
            for (int k = 0; k < MM; k++) {
                cols[k] = recw[k];
                icols[k] = recw[MM + 1 + k];
            }
            // apply_perm (automorphism.py:164-170): x[j] = alpha[sigma^-1(j)],
            // j = k*32 + lane
            T x[V];
            const unsigned sil = rec_lin<MM>(icols, (unsigned)lane) ^ recw[2 * MM + 1];
#pragma unroll
            for (int k = 0; k < V; k++) x[k] = alpha[sil ^ rec_lin<MM>(icols, 32u * k)];
            const uint32_t w = ssc_node<T, R, MM>(x, lane);
            cww[lane] = w;
            __syncwarp();
            // un-permute + correlation (top_decoders.py:231, 245-247) in
            // numpy's pairwise order over the original index i: lane
            // 8 (b % 4) + j accumulates elements 128 b + 8 t + j of block b
            constexpr int BL = N < 128 ? N : 128, NB = N / BL;
            const int j = lane & 7;
            const unsigned bsh = recw[MM];
            T pass_sum = 0;
#pragma unroll
            for (int q = 0; q < NB; q += 4) {
                const int b = q + (lane >> 3);
                T r = 0;
                if (b < NB) {
                    const unsigned base = rec_lin<MM>(cols, (unsigned)(b * BL + j)) ^ bsh;
#pragma unroll
                    for (int t = 0; t < BL / 8; t++) {
                        const int i = b * BL + 8 * t + j;
                        const unsigned s = base ^ rec_lin<MM>(cols, 8u * t);
                        const int c = (cww[s & 31u] >> (s >> 5)) & 1;
                        const T a = alpha[i];
                        const T v = c ? -a : a;
                        r = t == 0 ? v : r + v;
                    }
                }
                r += __shfl_xor_sync(kFull, r, 1);
                r += __shfl_xor_sync(kFull, r, 2);
                r += __shfl_xor_sync(kFull, r, 4);
                if (NB - q >= 2) r += __shfl_xor_sync(kFull, r, 8);
                if (NB - q >= 4) r += __shfl_xor_sync(kFull, r, 16);
                const T s = __shfl_sync(kFull, r, 0);
                pass_sum = q == 0 ? s : pass_sum + s;
            }
            const T score = pass_sum;
            const bool better = bestp < 0 || score > best;  // first strictly largest (warp-uniform)
            if (better || prm.att_cw) {
                // the un-permuted codeword, bit-packed: word k of lane k (only
                // for a new best, or when every decode's codeword is wanted)
                uint32_t myword = 0;
                const unsigned sl = rec_lin<MM>(cols, (unsigned)lane) ^ bsh;
#pragma unroll
                for (int k = 0; k < V; k++) {
                    const unsigned s = sl ^ rec_lin<MM>(cols, 32u * k);
                    const uint32_t wv = __ballot_sync(kFull, (cww[s & 31u] >> (s >> 5)) & 1u);
                    if (lane == k) myword = wv;
                }
                if (prm.att_cw && lane < V) prm.att_cw[((size_t)f * P + p) * V + lane] = myword;
                if (better) bestword = myword;
            }
            if (prm.att_pm && lane == 0) prm.att_pm[(size_t)f * P + p] = score;
            if (better) {
                best = score;
                bestp = p;
            }
            __syncwarp();
        }
        if (lane == 0) {
            red_score[warp] = best;
            red_p[warp] = bestp;
        }
        __syncthreads();
        int ww = -1;
        for (int w2 = 0; w2 < nw; w2++) {
            if (red_p[w2] < 0) continue;
            if (ww < 0 || red_score[w2] > red_score[ww] ||
                (red_score[w2] == red_score[ww] && red_p[w2] < red_p[ww]))
                ww = w2;
        }
        if (warp == ww) {
            if (lane < V) prm.cw[f * V + lane] = bestword;
            if (lane == 0) {
                prm.pm[f] = best;
                prm.attempt[f] = bestp;
                prm.path[f] = 0;
            }
        }
        __syncthreads();
    }
}

template <typename T, int MM>
constexpr size_t reg_smem_bytes(int nw) {
    return sizeof(T) * (size_t(1) << MM) + 128 * size_t(nw) + 64 * size_t(nw) + 16 * size_t(nw);
}

}  // namespace rmfht_ssc
