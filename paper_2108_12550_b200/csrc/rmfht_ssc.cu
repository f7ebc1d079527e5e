// Aut-SSC (the paper's Table IV comparator): P simplified
// SC decodes per frame, each on the frame permuted by its own affine map,
// un-permuted and scored by correlation; the first strictly largest score
// wins (aut_ssc, top_decoders.py:235-249; ssc_decode :205-230).
//
// One CTA per frame (grid-stride): the frame's LLRs are staged once in shared
// memory, each warp runs whole SSC decodes (permutation p = warp, warp + nw,
// ...) on its shared-memory workspace, keeps its best (score, p, codeword)
// in registers, and the CTA picks the winner at the end of the frame.  The
// SSC tree is walked with an explicit stack (runtime r, m <= 10); node
// vectors live in per-level shared buffers, leaf decisions in a byte array.
// Every sum (repetition leaves, the correlation score) is numpy's pairwise
// order, as in the oracle (oracle/rmo_impl.h FN(ssc), FN(rmo_aut_ssc)), so
// float64 results are bit-identical to the reference.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "rmfht_kernels.cuh"
#include "rmfht_plan.h"

using rmfht_internal::fail;

namespace rmfht_ssc {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxM = 10;

// f_op, list_engine.py:15-20: min(|a|,|b|) sgn(a) sgn(b).  The sign comes from
// sign(a) ^ sign(b) (one FMNMX.XORSIGN, the sign bit of a*b); it differs from
// sgn(a)sgn(b) (sgn(0) = +1) only on a zero result, where it yields
// -0.0 == +0.0 — every downstream use is a comparison with 0 or a sum, so
// results are unchanged.
__device__ __forceinline__ float f_op(float a, float b) {
    float r;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ double f_op(double a, double b) {
    const double m = fmin(fabs(a), fabs(b));
    return __longlong_as_double(__double_as_longlong(m) | (__double_as_longlong(a * b) & (long long)0x8000000000000000ull));
}

// g_op, list_engine.py:23-27: b + (1 - 2c) a, one rounding (exactly b - a or b + a)
__device__ __forceinline__ float g_op(float a, float b, int c) { return __fmaf_rn(c ? -1.f : 1.f, a, b); }
__device__ __forceinline__ double g_op(double a, double b, int c) { return __fma_rn(c ? -1.0 : 1.0, a, b); }

__device__ __forceinline__ unsigned lin(const uint16_t* cols, int m, unsigned x) {
    unsigned v = 0;
    for (int k = 0; k < m; k++) v ^= ((x >> k) & 1u) ? (unsigned)cols[k] : 0u;
    return v;
}

// numpy pairwise sum (loops_utils.h.src pairwise_sum) of a[0..n), n a power
// of two <= 1024, by one warp; the result in every lane.  Blocks of 128 use
// 8 accumulators of stride 8 (lanes 8 blk + j), combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); larger n halve recursively, i.e. a
// balanced tree over the blocks.
template <typename T>
__device__ T warp_pw_sum(const T* a, int n, int lane) {
    if (n < 8) {
        T res = 0;
        if (lane == 0)
            for (int i = 0; i < n; i++) res += a[i];
        return __shfl_sync(kFull, res, 0);
    }
    const int j = lane & 7;
    if (n <= 128) {
        T r = 0;
        if (lane < 8) {
            r = a[j];
            for (int i = 8; i < n; i += 8) r += a[i + j];
        }
        r += __shfl_xor_sync(kFull, r, 1);
        r += __shfl_xor_sync(kFull, r, 2);
        r += __shfl_xor_sync(kFull, r, 4);
        return __shfl_sync(kFull, r, 0);
    }
    const int nb = n >> 7;
    T total = 0;
    for (int q = 0; q < nb; q += 4) {
        const int blk = q + (lane >> 3);
        T r = 0;
        if (blk < nb) {
            const T* b = a + 128 * blk;
            r = b[j];
#pragma unroll
            for (int i = 8; i < 128; i += 8) r += b[i + j];
        }
        r += __shfl_xor_sync(kFull, r, 1);
        r += __shfl_xor_sync(kFull, r, 2);
        r += __shfl_xor_sync(kFull, r, 4);
        r += __shfl_xor_sync(kFull, r, 8);
        if (nb >= 4) r += __shfl_xor_sync(kFull, r, 16);
        const T s = __shfl_sync(kFull, r, 0);
        total = q == 0 ? s : total + s;
    }
    return total;
}

struct Frame {
    int r, s, base, in, ph;
};

template <typename T>
struct Layout {
    int N, words;
    size_t warp_bytes, cta_bytes;
    __host__ __device__ Layout(int m, int nw) {
        N = 1 << m;
        words = N >= 32 ? N / 32 : 1;
        // per warp: x0 [N] + level buffers / score summands [N] (T), bits [N],
        // map tables A32, Ai32 [words] (u16), record [2m+2] (u16)
        warp_bytes = ((size_t)2 * N * sizeof(T) + N + 4 * words + 2 * (2 * kMaxM + 2) + 15) & ~(size_t)15;
        cta_bytes = (((size_t)N * sizeof(T) + 15) & ~(size_t)15) + warp_bytes * nw + 16 * (size_t)nw;
    }
};

template <typename T>
__global__ void __launch_bounds__(256) aut_ssc_kernel(rmfht::Params<T> prm, int r, int m) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Layout<T> lay(m, nw);
    const int N = lay.N, words = lay.words, P = prm.M, REC = 2 * m + 2;
    T* alpha = reinterpret_cast<T*>(smem);
    unsigned char* wbase = smem + (((size_t)N * sizeof(T) + 15) & ~(size_t)15) + lay.warp_bytes * warp;
    T* x0 = reinterpret_cast<T*>(wbase);
    T* lvl = x0 + N;  // level buffers during the walk, score summands after it
    uint8_t* bits = reinterpret_cast<uint8_t*>(lvl + N);
    uint16_t* a32 = reinterpret_cast<uint16_t*>(bits + N);
    uint16_t* ai32 = a32 + words;
    uint16_t* rec = ai32 + words;
    T* red_score = reinterpret_cast<T*>(smem + (((size_t)N * sizeof(T) + 15) & ~(size_t)15) + lay.warp_bytes * nw);
    int* red_p = reinterpret_cast<int*>(red_score + nw);
    // level buffer of a node of 2^s elements (s < m): disjoint, sizes N/2, N/4, ...
    auto lvl_off = [&](int s) { return N + (N - (2 << s)); };

    for (long long f = blockIdx.x; f < prm.B; f += gridDim.x) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = prm.llr[f * N + i];
        __syncthreads();
        T best = 0;
        int bestp = -1;
        uint32_t bestword = 0;
        for (int p = warp; p < P; p += nw) {
            const uint16_t* g = prm.maps + ((size_t)f * P + p) * REC;
            for (int k = lane; k < REC; k += 32) rec[k] = g[k];
            __syncwarp();
            const uint16_t* cols = rec;
            const uint16_t* icols = rec + m + 1;
            const unsigned b = rec[m], c = rec[2 * m + 1];
            if (lane < words) {
                a32[lane] = (uint16_t)lin(cols, m, 32u * lane);
                ai32[lane] = (uint16_t)lin(icols, m, 32u * lane);
            }
            const unsigned sl = lin(cols, m, (unsigned)lane) ^ b, sil = lin(icols, m, (unsigned)lane) ^ c;
            __syncwarp();
            // apply_perm (automorphism.py:164-170): x0[sigma(i)] = alpha[i],
            // i.e. x0[j] = alpha[sigma^-1(j)]
            for (int k = 0; k < words; k++) {
                const int j = lane + 32 * k;
                if (j < N) x0[j] = alpha[sil ^ ai32[k]];
            }
            __syncwarp();
            // SSC walk (top_decoders.py:205-230)
            Frame st[kMaxM + 1];
            int sp = 0;
            st[0] = Frame{r, m, 0, 0, 0};
            while (sp >= 0) {
                Frame& fr = st[sp];
                const int s = fr.s, n = 1 << s, h = n >> 1, rr = fr.r;
                const T* in = x0 + fr.in;
                uint8_t* ob = bits + fr.base;
                if (rr < 0 || rr == s || rr == 0 || rr == s - 1) {
                    if (rr < 0) {
                        for (int i = lane; i < n; i += 32) ob[i] = 0;
                    } else if (rr == s) {
                        for (int i = lane; i < n; i += 32) ob[i] = in[i] < T(0);
                    } else if (rr == 0) {
                        const T sum = warp_pw_sum(in, n, lane);
                        const uint8_t v = sum < T(0);
                        for (int i = lane; i < n; i += 32) ob[i] = v;
                    } else {
                        // SPC: hard decisions; odd parity flips the first minimum of |a|
                        int par = 0, bi = 0x7fffffff;
                        T bv = 0;
                        for (int i = lane; i < n; i += 32) {
                            const T a = in[i];
                            const uint8_t hd = a < T(0);
                            ob[i] = hd;
                            par ^= hd;
                            const T v = a < T(0) ? -a : a;
                            if (bi == 0x7fffffff || v < bv) { bv = v; bi = i; }
                        }
#pragma unroll
                        for (int off = 16; off >= 1; off >>= 1) {
                            const T ov = __shfl_xor_sync(kFull, bv, off);
                            const int oi = __shfl_xor_sync(kFull, bi, off);
                            if (oi != 0x7fffffff && (bi == 0x7fffffff || ov < bv || (ov == bv && oi < bi))) {
                                bv = ov;
                                bi = oi;
                            }
                        }
                        const int odd = __popc(__ballot_sync(kFull, par)) & 1;
                        __syncwarp();
                        if (odd && lane == 0) ob[bi] ^= 1;
                    }
                    __syncwarp();
                    sp--;
                    continue;
                }
                T* child = x0 + lvl_off(s - 1);
                if (fr.ph == 0) {
                    for (int i = lane; i < h; i += 32) child[i] = f_op(in[i], in[h + i]);
                    __syncwarp();
                    fr.ph = 1;
                    st[sp + 1] = Frame{rr - 1, s - 1, fr.base, lvl_off(s - 1), 0};
                    sp++;
                } else if (fr.ph == 1) {
                    for (int i = lane; i < h; i += 32) child[i] = g_op(in[i], in[h + i], (int)ob[i]);
                    __syncwarp();
                    fr.ph = 2;
                    st[sp + 1] = Frame{rr, s - 1, fr.base + h, lvl_off(s - 1), 0};
                    sp++;
                } else {
                    for (int i = lane; i < h; i += 32) ob[i] ^= ob[h + i];  // propagate_hard
                    __syncwarp();
                    sp--;
                }
            }
            // un-permute (apply_perm_inverse: cand[i] = c[sigma(i)]) and score
            // (correlation, top_decoders.py:231: sum (1 - 2 cand) alpha)
            uint32_t myword = 0;
            T* sv = lvl;
            for (int k = 0; k < words; k++) {
                const int i = lane + 32 * k;
                int cb = 0;
                if (i < N) {
                    cb = bits[sl ^ a32[k]];
                    sv[i] = cb ? -alpha[i] : alpha[i];
                }
                const uint32_t wv = __ballot_sync(kFull, cb);
                if (lane == k) myword = wv;
            }
            __syncwarp();
            const T score = warp_pw_sum(sv, N, lane);
            if (prm.att_pm && lane == 0) prm.att_pm[(size_t)f * P + p] = score;
            if (prm.att_cw && lane < words) prm.att_cw[((size_t)f * P + p) * words + lane] = myword;
            if (bestp < 0 || score > best) {  // first strictly largest
                best = score;
                bestp = p;
                bestword = myword;
            }
            __syncwarp();
        }
        if (lane == 0) {
            red_score[warp] = best;
            red_p[warp] = bestp;
        }
        __syncthreads();
        // winner: largest score, lowest permutation index among equals
        int ww = -1;
        for (int w = 0; w < nw; w++) {
            if (red_p[w] < 0) continue;
            if (ww < 0 || red_score[w] > red_score[ww] || (red_score[w] == red_score[ww] && red_p[w] < red_p[ww]))
                ww = w;
        }
        if (warp == ww) {
            if (lane < words) prm.cw[f * words + lane] = bestword;
            if (lane == 0) {
                prm.pm[f] = best;
                prm.attempt[f] = bestp;
                prm.path[f] = 0;
            }
        }
        __syncthreads();
    }
}

}  // namespace rmfht_ssc

#include "rmfht_ssc_reg.cuh"

// compiled register-resident shapes (r, m): the paper's Table IV comparators
// (RM(2,8), (3,8), (4,8), (2,9)) and the FER / bench shapes
#define RMFHT_SSC_SHAPES(X) X(2, 9) X(2, 8) X(3, 8) X(4, 8) X(2, 7) X(3, 7) X(2, 6) X(2, 10) X(3, 10) X(2, 5)

namespace rmfht_ssc {

template <typename T, int R, int MM>
int prepare_reg(rmfht_plan* p) {
    int nw = 8;
    const size_t smem = reg_smem_bytes<T, MM>(nw);
    auto kern = aut_ssc_reg_kernel<T, R, MM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "Aut-SSC kernel does not fit an SM");
    p->nwarps = nw;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

template <typename T, int R, int MM>
int launch_reg(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
               int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/, cudaStream_t st) {
    rmfht::Params<T> prm;
    prm.llr = static_cast<const T*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = 1;
    prm.tie_fix = 0;
    prm.cw = cw;
    prm.pm = static_cast<T*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<T*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const long long grid = B < p->grid ? B : p->grid;
    aut_ssc_reg_kernel<T, R, MM><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(prm);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("Aut-SSC launch: ") + cudaGetErrorString(e));
    return 0;
}

template <typename T>
int prepare(rmfht_plan* p) {
    int nw = p->M < 8 ? p->M : 8;
    while (nw > 1 && Layout<T>(p->m, nw).cta_bytes > 200 * 1024) nw--;
    const size_t smem = Layout<T>(p->m, nw).cta_bytes;
    auto kern = aut_ssc_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "Aut-SSC kernel does not fit an SM");
    p->nwarps = nw;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

template <typename T>
int launch(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
           int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/, cudaStream_t st) {
    rmfht::Params<T> prm;
    prm.llr = static_cast<const T*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = 1;
    prm.tie_fix = 0;
    prm.cw = cw;
    prm.pm = static_cast<T*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<T*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const long long grid = B < p->grid ? B : p->grid;
    aut_ssc_kernel<T><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(prm, p->r, p->m);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("Aut-SSC launch: ") + cudaGetErrorString(e));
    return 0;
}

}  // namespace rmfht_ssc

// Binds the Aut-SSC kernels (plan created with RMFHT_AUT_SSC: M = P maps of
// m variables per frame, one per decode).
int rmfht_bind_aut_ssc(rmfht_plan* p) {
    if (p->m > rmfht_ssc::kMaxM) return RMFHT_EUNSUPPORTED;
    p->fast = 0;
    p->generic = 0;
    if (!p->force_generic) {
        const bool f64 = p->dtype == RMFHT_F64;
#define X(R_, M_)                                                                              \
        if (p->r == R_ && p->m == M_) {                                                         \
            p->launch = f64 ? &rmfht_ssc::launch_reg<double, R_, M_> : &rmfht_ssc::launch_reg<float, R_, M_>; \
            p->prepare = f64 ? &rmfht_ssc::prepare_reg<double, R_, M_> : &rmfht_ssc::prepare_reg<float, R_, M_>; \
            return 0;                                                                           \
        }
        RMFHT_SSC_SHAPES(X)
#undef X
    }
    p->generic = 1;  // runtime-shaped shared-memory walk
    if (p->dtype == RMFHT_F64) {
        p->launch = &rmfht_ssc::launch<double>;
        p->prepare = &rmfht_ssc::prepare<double>;
    } else {
        p->launch = &rmfht_ssc::launch<float>;
        p->prepare = &rmfht_ssc::prepare<float>;
    }
    return 0;
}
