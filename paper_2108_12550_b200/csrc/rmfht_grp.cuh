// Lane-group float32 kernel for p-FHT-FSCL with ONE list path (L = 1), r = 2:
// the Aut-style ensemble of BASELINE config 4 (RM(2,9), L = 1, M = 512).
//
// With L = 1 the throughput kernel (rmfht_fast.cuh) gives a whole warp to one
// (frame, attempt): 32 lanes on one path, sub-warp activity below n = 32 and
// the per-node control (shuffles, ballots, scalar round trips) paid per item
// — 1,860 warp-instructions per item, 8% of the ledger bound.  Here a warp
// decodes FOUR consecutive attempts of one frame, 8 lanes each ("lane
// group"), in the throughput kernel's own register layout for L = 4 (element
// e = k * 8 + u in slot k of lane u), so every warp-level instruction serves
// four items and every lane is active down to the n = 8 leaves.  One path
// has no list: the FHT node keeps the first bin of maximal |w|
// (fht_decode.py:101-126 with L = 1), the SPC node is the hard decision with
// the single split (list_engine.py:68-119 with tau = 1), there is no lineage.
//
// Arithmetic is the throughput kernel's for L = 1, bit for bit (checked
// against it and against the float32 oracle, order v2): the LM sums of the
// root permutation extension in the canonical channel-domain order
// (lm_partial_root, multi_tree), llr_abs as the 32-lane partials of the
// L = 1 layout (element e in lane e % 32, ascending e / 32, then the xor tree
// 1 .. 16), the accumulated metric pm + 0.5 (llr_abs - max|w|) per FHT leaf and
// the SPC split in the reference's order.  The attempt records go to the same
// workspace as the throughput kernel's and reduce_kernel2 picks the attempt.
#pragma once

#include "rmfht_fast.cuh"

namespace rmfht_grp {

using rmfht::kFull;
using rmfht2::AttHdr;
using rmfht2::MapR;
using rmfht2::add2;
using rmfht2::clog2;
using rmfht2::cp_async16;
using rmfht2::cp_async4;
using rmfht2::cp_async_commit;
using rmfht2::cp_async_wait_all;
using rmfht2::f_op;
using rmfht2::fma2;
using rmfht2::lds_addr;
using rmfht2::mul2;
using rmfht2::phi;
using rmfht2::pk;
using rmfht2::plo;
using rmfht2::sub2;
using u32 = uint32_t;
using u64 = unsigned long long;

constexpr int kLpp = 8;    // lanes per item
constexpr int kItems = 4;  // items per warp
constexpr int kMaps = 3;   // maps per attempt: the root map and two trials (r = 2, L = 1)

#ifndef RMFHT_GRP_WARPS
#define RMFHT_GRP_WARPS 24
#endif
constexpr int kGrpWarps = RMFHT_GRP_WARPS;

template <int MM>
struct alignas(16) GWS {
    static constexpr int REC = 2 * MM + 2;
    static constexpr int RECW = kItems * kMaps * REC;  // uint16 of a warp round's records
    alignas(16) uint16_t recs[(RECW + 7) & ~7];
    MapR<MM> comp[kItems];  // composite root map of each item (init, then the winning trial)
    float lm[2 * kItems];
    int dir[2 * kItems];
    // the transforms' transpose rows (fht_leaf, V >= 8); the LM lane partials
    // of the root permutation extension are dead by then and share the space
    union alignas(16) {
        float wsp[32][32];
        float lmp[2 * kItems][32];
    };
};

template <int MM>
__host__ __device__ constexpr size_t smem_bytes(int nwarps) {
    return 2048 + (size_t(4) << MM) * nwarps + sizeof(GWS<MM>) * size_t(nwarps);
}

__device__ __forceinline__ float group_max8(float v) {
#pragma unroll
    for (int off = 1; off < kLpp; off <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, off));
    return v;
}

// llr_abs (fht_decode.py:114) of a node held as x[k] = element k * 8 + u, in
// the summation order of the L = 1 throughput kernel: element e belongs to
// "lane" e % 32 and is added in ascending e / 32, then the xor tree over the
// lane bits 1, 2, 4, 8, 16.  Here lane bits 0..2 are u and bits 3, 4 are the
// low bits of k, so a lane carries up to four partials.
template <int V>
__device__ __forceinline__ float llr_abs(const float (&x)[V]) {
    constexpr int J = V >= 4 ? 4 : V;
    float P[J];
#pragma unroll
    for (int j = 0; j < J; j++) P[j] = fabsf(x[j]);
#pragma unroll
    for (int k = J; k < V; k++) P[k & (J - 1)] += fabsf(x[k]);
    // The xor tree over the lane bits 1, 2, 4 of every partial, transposed:
    // at each level a lane keeps half of its partials and hands the other
    // half to its partner, so the same sums (operands swapped at most: the
    // addition commutes) take 6 shuffles instead of 12.  u: lane in the group.
    const int u = threadIdx.x & 7;
    if constexpr (J == 4) {
        const bool b0 = u & 1, b1 = u & 2;
        const float A = (b0 ? P[2] : P[0]) + __shfl_xor_sync(kFull, b0 ? P[0] : P[2], 1);
        const float Bv = (b0 ? P[3] : P[1]) + __shfl_xor_sync(kFull, b0 ? P[1] : P[3], 1);
        float C = (b1 ? Bv : A) + __shfl_xor_sync(kFull, b1 ? A : Bv, 2);  // partial 2 b0 + b1
        C = C + __shfl_xor_sync(kFull, C, 4);
        const float D = C + __shfl_xor_sync(kFull, C, 2);  // P0 + P1 (b0 = 0) or P2 + P3
        return D + __shfl_xor_sync(kFull, D, 1);           // (P0 + P1) + (P2 + P3)
    } else if constexpr (J == 2) {
        const bool b0 = u & 1;
        float A = (b0 ? P[1] : P[0]) + __shfl_xor_sync(kFull, b0 ? P[0] : P[1], 1);
        A = A + __shfl_xor_sync(kFull, A, 2);
        A = A + __shfl_xor_sync(kFull, A, 4);
        return A + __shfl_xor_sync(kFull, A, 1);
    } else {
#pragma unroll
        for (int off = 1; off < kLpp; off <<= 1) P[0] = P[0] + __shfl_xor_sync(kFull, P[0], off);
        return P[0];
    }
}

// fhtl with one path (fht_decode.py:101-126): transform in the reference's
// stage order, first bin of maximal |w|, metric and codeword bits.  bits:
// bit k = hard decision of element k * 8 + u.
template <int V>
__device__ __forceinline__ u32 fht_leaf(const float (&x)[V], float (*wsp)[32], int lane, float& pm, int& bin,
                                        int& sgn) {
    constexpr int n = V * kLpp;
    const int g = lane >> 3, u = lane & 7;
    const float la = llr_abs<V>(x);
    float w[V];
#pragma unroll
    for (int k = 0; k < V; k++) w[k] = x[k];
    // register stages (high index bits first): lo' = hi - lo, hi' = hi + lo
    auto reg_stage = [&](const int hr) {
        if (hr >= 2) {
#pragma unroll
            for (int k = 0; k < V; k += 2)
                if (!(k & hr)) {
                    const u64 lo = pk(w[k], w[k + 1]), hi = pk(w[k + hr], w[k + hr + 1]);
                    const u64 d = sub2(hi, lo), e = add2(hi, lo);
                    w[k] = plo(d);
                    w[k + 1] = phi(d);
                    w[k + hr] = plo(e);
                    w[k + hr + 1] = phi(e);
                }
        } else {
#pragma unroll
            for (int k = 0; k < V; k += 2) {
                const float lo = w[k], hi = w[k + 1];
                w[k] = hi - lo;
                w[k + 1] = hi + lo;
            }
        }
    };
#pragma unroll
    for (int st = 0; st < clog2(V); st++) reg_stage(V >> (st + 1));
    // TR (V >= 8): the vector is transposed through the warp's rows so that
    // the lane-bit stages are register stages too — 16 wide shared accesses
    // instead of 3 V shuffles (as rmfht2::FhtLayout::TR).  Afterwards slot
    // j * G + q of lane u holds element (u * G + q) * 8 + j, G = V / 8.
    constexpr bool TR = V >= 8;
    constexpr int G = TR ? V / 8 : 1;
    if constexpr (TR) {
        // rows are lane-major, 16-byte chunks XOR-swizzled by the lane (and a
        // per-group twist for V < 32): conflict-free STS.128 and transposed reads
        const int tw = V == 16 ? 4 * (g & 1) : V == 8 ? 2 * g : 0;
        auto at = [&](int row, int k) -> float& { return wsp[row][k ^ (((row & 7) ^ tw) << 2)]; };
#pragma unroll
        for (int k = 0; k < V; k += 4) *reinterpret_cast<float4*>(&at(lane, k)) = make_float4(w[k], w[k + 1], w[k + 2], w[k + 3]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const float* src = &at(g * 8 + j, u * G);
            if constexpr (G == 4) {
                const float4 v = *reinterpret_cast<const float4*>(src);
                w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
            } else if constexpr (G == 2) {
                const float2 v = *reinterpret_cast<const float2*>(src);
                w[2 * j] = v.x; w[2 * j + 1] = v.y;
            } else {
                w[j] = *src;
            }
        }
        __syncwarp();  // every row read before the next node stores
        reg_stage(4 * G);
        reg_stage(2 * G);
        reg_stage(G);
    } else {
    // lane stages (index bits 2, 1, 0)
#pragma unroll
    for (int half = kLpp / 2; half >= 1; half >>= 1) {
        const float sg = (u & half) ? 1.f : -1.f;
        if constexpr (V >= 2) {
            const u64 sg2 = pk(sg, sg);
#pragma unroll
            for (int k = 0; k < V; k += 2) {
                const float o0 = __shfl_xor_sync(kFull, w[k], half), o1 = __shfl_xor_sync(kFull, w[k + 1], half);
                const u64 r = fma2(sg2, pk(w[k], w[k + 1]), pk(o0, o1));  // hi lane: w + o, lo lane: o - w
                w[k] = plo(r);
                w[k + 1] = phi(r);
            }
        } else {
            const float o = __shfl_xor_sync(kFull, w[0], half);
            w[0] = __fmaf_rn(sg, w[0], o);
        }
    }
    }
    float mx;
    {
        float t[V];
#pragma unroll
        for (int k = 0; k < V; k++) t[k] = fabsf(w[k]);
#pragma unroll
        for (int sd = 1; sd < V; sd <<= 1)
#pragma unroll
            for (int k = 0; k + sd < V; k += 2 * sd) t[k] = fmaxf(t[k], t[k + sd]);
        mx = t[0];
    }
    const float M1 = group_max8(mx);
    pm = pm + 0.5f * (la - M1);  // :119
    // first bin of maximal |w| (stable argsort of -|w|, :116), with its sign
    // (el: the lane's elements in ascending bin order; default layout: slot
    // el is bin el * 8 + u, transposed: slot (el & 7) * G + (el >> 3) is bin
    // u * V + el)
    int kk = V;
    float wv = 0.f;
#pragma unroll
    for (int el = V - 1; el >= 0; el--) {
        const int s = TR ? (el & 7) * G + (el >> 3) : el;
        if (fabsf(w[s]) == M1) {
            kk = el;
            wv = w[s];
        }
    }
    const int mybin = TR ? u * V + kk : ((kk << 3) | u);
    u32 key = kk < V ? (u32)((mybin << 1) | (wv < 0.f ? 1 : 0)) : 0xffffffffu;
#pragma unroll
    for (int off = 1; off < kLpp; off <<= 1) key = min(key, __shfl_xor_sync(kFull, key, off));
    bin = (int)(key >> 1);
    sgn = (int)(key & 1u);
    // bit k = parity(~b & ~e & (n-1)) ^ sign for e = k * 8 + u (_bin_codewords, :58-62)
    const u32 B = (u32)(~bin) & (u32)(n - 1);
    const u32 Bh = B >> 3;
    const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)u & 7u) & 1);
    constexpr u32 VM = V >= 32 ? ~0u : ((1u << V) - 1u);
    u32 P = 0;
    if (Bh & 1u) P ^= 0xAAAAAAAAu;
    if (Bh & 2u) P ^= 0xCCCCCCCCu;
    if (Bh & 4u) P ^= 0xF0F0F0F0u;
    if (Bh & 8u) P ^= 0xFF00FF00u;
    if (Bh & 16u) P ^= 0xFFFF0000u;
    return (c0 ? ~P : P) & VM;
}

// g (list_engine.py:23-27) after an FHT left child of V slots per lane: the
// hard decisions are bit_k = c0 ^ parity(Bh & k), so the +-1 factors follow a
// Gray-code walk over the slot pairs (as rmfht2::g_fht_child)
template <int V>
__device__ __forceinline__ void g_after_fht(int bin, int sgn, int u, const float* a, const float* b, float* out) {
    constexpr int n = V * kLpp;
    const u32 B = (u32)(~bin) & (u32)(n - 1);
    const u32 Bh = B >> 3;
    const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)u & 7u) & 1);
    const float base = c0 ? -1.f : 1.f;
    if constexpr (V >= 2) {
        const float col0 = (Bh & 1u) ? -1.f : 1.f;
        u64 s2 = pk(base, base * col0);
#pragma unroll
        for (int i = 0; i < V / 2; i++) {
            if (i > 0) {
                const int j = __ffs(i);
                const float cj = ((Bh >> j) & 1u) ? -1.f : 1.f;
                s2 = mul2(s2, pk(cj, cj));
            }
            const int k = 2 * (i ^ (i >> 1));
            const u64 r = fma2(s2, pk(a[k], a[k + 1]), pk(b[k], b[k + 1]));
            out[k] = plo(r);
            out[k + 1] = phi(r);
        }
    } else {
        out[0] = __fmaf_rn(base, a[0], b[0]);
    }
}

// The root's g from its gathers parked in tensor memory (rmfht2::tmem_park):
// column k holds the lower half's slot k, column V + k the upper half's; the
// Gray-code steps 4 c .. 4 c + 3 stay inside the 8-slot chunk c ^ (c >> 1).
template <int V>
__device__ __forceinline__ void g_after_fht_tmem(int bin, int sgn, int u, u32 taddr, float* out) {
    static_assert(V >= 8 && V % 8 == 0, "8-column chunks");
    constexpr int n = V * kLpp;
    const u32 B = (u32)(~bin) & (u32)(n - 1);
    const u32 Bh = B >> 3;
    const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)u & 7u) & 1);
    const float base = c0 ? -1.f : 1.f;
    const float col0 = (Bh & 1u) ? -1.f : 1.f;
    u64 s2 = pk(base, base * col0);
#pragma unroll
    for (int c = 0; c < V / 8; c++) {
        const int k0 = 8 * (c ^ (c >> 1));
        u32 ra[8], rb[8];
        rmfht2::tmem_ld8(taddr + k0, ra);
        rmfht2::tmem_ld8(taddr + V + k0, rb);
        rmfht2::tmem_wait_ld16(ra, rb);
#pragma unroll
        for (int i = 4 * c; i < 4 * c + 4; i++) {
            if (i > 0) {
                const int j = __ffs(i);
                const float cj = ((Bh >> j) & 1u) ? -1.f : 1.f;
                s2 = mul2(s2, pk(cj, cj));
            }
            const int k = 2 * (i ^ (i >> 1)), q = k - k0;
            const u64 r = fma2(s2, pk(__uint_as_float(ra[q]), __uint_as_float(ra[q + 1])),
                               pk(__uint_as_float(rb[q]), __uint_as_float(rb[q + 1])));
            out[k] = plo(r);
            out[k + 1] = phi(r);
        }
    }
}

// spc_decode_list (list_engine.py:68-119) with one path on n = 8 (one element
// per lane): tau = 1, i.e. the hard decision (:84-88) and one split (:97-112)
// between keeping it and flipping the second least reliable position.
__device__ __forceinline__ u32 spc_leaf8(float xv, int g, int u, float& pm) {
    const float mag = fabsf(xv);
    const int sb = xv < 0.f ? 1 : 0;
    const u32 gs = (__ballot_sync(kFull, sb) >> (g * kLpp)) & 0xffu;
    const int par0 = __popc(gs) & 1;
    float a0 = mag;
#pragma unroll
    for (int off = 1; off < kLpp; off <<= 1) a0 = fminf(a0, __shfl_xor_sync(kFull, a0, off));
    const int i0 = __ffs((__ballot_sync(kFull, mag == a0) >> (g * kLpp)) & 0xffu) - 1;  // stable order (:83)
    const float mag2 = u == i0 ? __int_as_float(0x7f800000) : mag;
    float a1 = mag2;
#pragma unroll
    for (int off = 1; off < kLpp; off <<= 1) a1 = fminf(a1, __shfl_xor_sync(kFull, a1, off));
    const int i1 = __ffs((__ballot_sync(kFull, mag2 == a1) >> (g * kLpp)) & 0xffu) - 1;
    const float spm = pm + (par0 ? a0 : 0.f);  // :88
    const float t = spm + a1;
    const float flip = par0 ? t - a0 : t + a0;  // pms + a_j + (1 - 2 par) a_m
    const bool take = flip < spm;               // stable order of (keep, flip) (:104)
    pm = take ? flip : spm;
    const int tot = par0 ^ (take ? 1 : 0);
    return (u32)(sb ^ ((take && u == i1) ? 1 : 0) ^ ((tot && u == i0) ? 1 : 0));
}

// _decode_node (top_decoders.py:72-113) below the root: RM(RR, SS) on x[k] =
// element k * 8 + u of this item's vector
template <int RR, int SS>
__device__ __forceinline__ u32 node(float (&x)[(1 << SS) / kLpp], float (*wsp)[32], int lane, float& pm, int& bin,
                                    int& sgn) {
    constexpr int V = (1 << SS) / kLpp;
    const int g = lane >> 3, u = lane & 7;
    if constexpr (RR == 1) {
        return fht_leaf<V>(x, wsp, lane, pm, bin, sgn);
    } else if constexpr (RR == SS - 1) {
        static_assert(V == 1, "SPC leaf of r = 2 is RM(2, 3)");
        return spc_leaf8(x[0], g, u, pm);
    } else {
        constexpr int VC = V / 2;
        float xl[VC];
#pragma unroll
        for (int k = 0; k < VC; k++) xl[k] = f_op(x[k], x[k + VC]);
        int cb, cs;
        const u32 bl = node<RR - 1, SS - 1>(xl, wsp, lane, pm, cb, cs);
        float xr[VC];
        static_assert(RR - 1 == 1, "r = 2: the left child is an FHT leaf");
        g_after_fht<VC>(cb, cs, u, x, x + VC, xr);
        const u32 br = node<RR, SS - 1>(xr, wsp, lane, pm, bin, sgn);
        return (br << VC) | (bl ^ br);
    }
}

template <int MM>
__global__ void __launch_bounds__(32 * kGrpWarps, 1) grp_kernel(rmfht::Params<float> prm, AttHdr* hdr, u64* bitsout) {
    constexpr int N = 1 << MM, NS = N / 32, REC = 2 * MM + 2, V = N / kLpp, VC = V / 2;
    static_assert(MM >= 8 && MM <= 9, "lane-group kernel: RM(2, 8) and RM(2, 9)");
    using WS = GWS<MM>;
    extern __shared__ __align__(16) unsigned char graw[];
    const int lane = threadIdx.x & 31, wib = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0);
    const int g = lane >> 3, u = lane & 7;
    WS& ws = reinterpret_cast<WS*>(graw)[wib];
    const u32 raw_saddr = (u32)__cvta_generic_to_shared(graw) + (u32)(kGrpWarps * sizeof(WS));
    const u32 pad = ((raw_saddr + 2047u) & ~2047u) - raw_saddr;
    float* const alpha_w = reinterpret_cast<float*>(graw + kGrpWarps * sizeof(WS) + pad + (size_t)wib * (4u << MM));
    const u32 asa = (u32)__cvta_generic_to_shared(alpha_w);
    // tensor memory for the root's parked gathers: warp w owns lanes
    // 32 (w % 4) .. + 31 and columns V (w / 4) .. + V - 1 of the CTA's 512
    constexpr bool TPARK = RMFHT_TMEM_PARK != 0;
    __shared__ u32 tmem_slot;
    u32 tmem = 0;
    if constexpr (TPARK) {
        static_assert((kGrpWarps + 3) / 4 * V <= 512, "tensor-memory columns");
        if (wib == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             (u32)__cvta_generic_to_shared(&tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem = tmem_slot + ((u32)(32 * (wib & 3)) << 16) + (u32)(V * (wib >> 2));
    }
    const int M = prm.M;
    const long long rounds = prm.B * (long long)M / kItems;  // M % 4 == 0 (bind_one)
    const long long stride = (long long)gridDim.x * kGrpWarps;
    const MapR<MM>* maps = reinterpret_cast<const MapR<MM>*>(ws.recs);
    auto prefetch_recs = [&](long long r) {
        if (r >= rounds) return;
        const u32 rsa = (u32)__cvta_generic_to_shared(ws.recs);
        const char* gr = reinterpret_cast<const char*>(prm.maps + (size_t)r * WS::RECW);
        constexpr int RB = WS::RECW * 2;
        if (RB % 16 == 0 && (reinterpret_cast<uintptr_t>(prm.maps) & 15u) == 0) {
            for (int i = lane; i < RB / 16; i += 32) cp_async16(rsa + 16u * i, gr + 16 * i);
        } else {
            for (int i = lane; i < RB / 4; i += 32) cp_async4(rsa + 4u * i, gr + 4 * i);
        }
        cp_async_commit();
    };
    auto prefetch_alpha = [&](long long frame) {
        const char* ga = reinterpret_cast<const char*>(prm.llr + (size_t)frame * N);
        for (int i = lane; i < N / 4; i += 32) cp_async16(asa + 16u * i, ga + 16 * i);
        cp_async_commit();
    };
    const int lockstep = prm.tie_fix >> 8 & 0xff;
    long long have = -1;  // frame whose LLRs the warp's buffer holds (or is loading)
    {
        const long long r = (long long)blockIdx.x * kGrpWarps + wib;
        prefetch_recs(r);
        if (r < rounds) {
            have = r * kItems / M;
            prefetch_alpha(have);
        }
    }
    for (long long r0 = (long long)blockIdx.x * kGrpWarps; r0 < rounds; r0 += stride) {
        const long long r = r0 + wib;
        if (r < rounds) {
            const long long item0 = r * kItems, item = item0 + g;
            cp_async_wait_all();
            __syncwarp();
            float ach[NS];
#pragma unroll
            for (int s = 0; s < NS; s++) ach[s] = alpha_w[lane + 32 * s];
            // root permutation extension (automorphism.py:207-237) of the four
            // items: trial t of item i pairs direction A_init^-1 (A_t^-1 e_{m-1})
            if (lane < 2 * kItems) {
                const int i = lane >> 1, t = lane & 1;
                ws.dir[lane] = (int)rmfht2::icol_apply<MM>(maps[i * kMaps], (u32)maps[i * kMaps + 1 + t].icol[MM - 1]);
            }
            __syncwarp();
            {
                float part[2 * kItems];
                if constexpr (TPARK) {
                    // the lane partials wait in the warp's tensor-memory columns (idle until the root's f)
#pragma unroll 1
                    for (int t = 0; t < 2 * kItems; t++)
                        rmfht2::tmem_st1(tmem + t, rmfht2::lm_partial_root<NS>(ach, (u32)ws.dir[t], lane, asa));
                    rmfht2::tmem_wait_st();
                    u32 r8[8];
                    rmfht2::tmem_ld8(tmem, r8);
                    rmfht2::tmem_wait_ld8(r8);
#pragma unroll
                    for (int t = 0; t < 8; t++) part[t] = __uint_as_float(r8[t]);
                } else {
#pragma unroll 1
                    for (int t = 0; t < 2 * kItems; t++)
                        ws.lmp[t][lane] = rmfht2::lm_partial_root<NS>(ach, (u32)ws.dir[t], lane, asa);
                    __syncwarp();
#pragma unroll
                    for (int t = 0; t < 2 * kItems; t++) part[t] = ws.lmp[t][lane];
                }
                int tri;
                const float tot = rmfht2::multi_tree<2 * kItems>(part, lane, &tri);
                if ((lane & (32 / (2 * kItems) - 1)) == 0) ws.lm[tri] = tot;
            }
            __syncwarp();
            // the winning trial (LM descending, lower trial first, :234) and the
            // composite's inverse (one column per lane task)
            int win[kItems];
#pragma unroll
            for (int i = 0; i < kItems; i++) win[i] = ws.lm[2 * i + 1] > ws.lm[2 * i] ? 1 : 0;
            constexpr int NT = (kItems * (MM + 1) + 31) / 32;
#pragma unroll
            for (int q = 0; q < NT; q++) {
                const int task = lane + 32 * q;
                if (task < kItems * (MM + 1)) {
                    const int i = task / (MM + 1), k = task % (MM + 1);
                    int wi = win[0];
#pragma unroll
                    for (int j = 1; j < kItems; j++) wi = i == j ? win[j] : wi;
                    const MapR<MM>& tm = maps[i * kMaps + 1 + wi];
                    const MapR<MM>& im = maps[i * kMaps];
                    const u32 v = rmfht2::icol_apply<MM>(im, (u32)(k < MM ? tm.icol[k] : tm.c));
                    if (k < MM) ws.comp[i].icol[k] = (uint16_t)v;
                    else ws.comp[i].c = (uint16_t)(v ^ im.c);
                }
            }
            int mywin = win[0];
#pragma unroll
            for (int j = 1; j < kItems; j++) mywin = g == j ? win[j] : mywin;
            __syncwarp();
            prefetch_recs(r + stride);  // the records are dead: the composites carry the maps
            float pm = 0.f;
            // root (2, m): never held; f (:100) and g (:104) gather through the composite
            float xl[VC];
            {
                rmfht2::RootIdx<MM, kLpp, V> ri;
                ri.build(ws.comp[g], u, asa);
                if constexpr (TPARK) {
#pragma unroll
                    for (int k0 = 0; k0 < VC; k0 += 8) {
                        float a[8], b[8];
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            a[i] = lds_addr(ri.off(k0 + i));
                            b[i] = lds_addr(ri.off(k0 + i + VC));
                        }
                        rmfht2::tmem_st8(tmem + k0, a);
                        rmfht2::tmem_st8(tmem + VC + k0, b);
#pragma unroll
                        for (int i = 0; i < 8; i++) xl[k0 + i] = f_op(a[i], b[i]);
                    }
                    rmfht2::tmem_wait_st();
                } else {
#pragma unroll
                    for (int k = 0; k < VC; k++) xl[k] = f_op(lds_addr(ri.off(k)), lds_addr(ri.off(k + VC)));
                }
            }
            // the frame LLRs may be dead for this round: fetch the next round's if it is another frame
            auto next_alpha = [&] {
                const long long rn = r + stride;
                if (rn < rounds) {
                    const long long fn = rn * kItems / M;
                    if (fn != have) {
                        __syncwarp();
                        have = fn;
                        prefetch_alpha(fn);
                    }
                }
            };
            if constexpr (TPARK) next_alpha();
            int cb, cs;
            const u32 bl = node<1, MM - 1>(xl, ws.wsp, lane, pm, cb, cs);
            float xr[VC];
            if constexpr (TPARK) {
                g_after_fht_tmem<VC>(cb, cs, u, tmem, xr);
            } else {
                rmfht2::RootIdx<MM, kLpp, V> ri;
                ri.build(ws.comp[g], u, asa);
                float ga[VC], gb[VC];
#pragma unroll
                for (int k = 0; k < VC; k++) {
                    ga[k] = lds_addr(ri.off(k));
                    gb[k] = lds_addr(ri.off(k + VC));
                }
                next_alpha();
                g_after_fht<VC>(cb, cs, u, ga, gb, xr);
            }
            int db, ds;
            const u32 br = node<2, MM - 1>(xr, ws.wsp, lane, pm, db, ds);
            const u64 out = ((u64)br << VC) | (u64)(bl ^ br);
            if (u == 0) {
                AttHdr h;
                h.pm = pm;
                h.path = 0;
                h.init_map = 0;
                h.trial_map = 1 + mywin;
                hdr[item] = h;
            }
            bitsout[(size_t)item * kLpp + u] = out;
            __syncwarp();
        }
        if (lockstep) __syncthreads();
    }
    if constexpr (TPARK) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (wib == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_slot) : "memory");
    }
}

constexpr size_t work_bytes() { return sizeof(AttHdr) + sizeof(u64) * size_t(kLpp); }

}  // namespace rmfht_grp
