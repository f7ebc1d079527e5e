// Pair kernel: p-FHT-FSCL with L = 2 on short RM(2, m) codes (m <= 7) —
// BASELINE config 2 (RM(2,7), L = 2, M = 4).  Two threads per
// (frame, attempt) work item, one per list path, 16 items per warp.
//
// The warp-per-item throughput kernel (rmfht_fast.cuh) gives an RM(2,7)
// L = 2 item 16 lanes per path and 8 elements per lane at the root: the
// per-node selection and lineage logic (warp collectives, shared-memory
// scalars) is fixed cost that the tiny nodes cannot amortise — 1,475 warp
// instructions per item, 3.7% of the ledger roofline.  Here each thread
// holds its path's node vector in registers and runs the node arithmetic
// alone; the list steps exchange a few scalars with the partner thread
// (lane ^ 1) by shuffles.
//
// Semantics and summation order are the reference's (top_decoders.py:72-153,
// fht_decode.py:28-48,101-126, list_engine.py:15-36,68-119,
// automorphism.py:207-237), exactly as the reference-order kernel
// (rmfht_kernels.cuh, decode_kernel<float>) computes them: numpy's pairwise
// order for the LM and llr_abs sums, the tie fix for equal pairing
// directions, the reference's stage order for the butterflies, every
// stable-sort tie rule — so its outputs equal that kernel's and the float32
// oracle's (order "reference") bit for bit.  The reported pm is the decided
// codeword's metric recomputed from the channel LLRs (rmfht::CorrPm order).
//
// The M attempts of a frame sit in consecutive items of one warp (M divides
// 16), so the ensemble pick (first strict minimum, top_decoders.py:200) is a
// shuffle reduction: no workspace, no second kernel.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "rmfht_kernels.cuh"
#include "rmfht_fast.cuh"  // tensor-memory parking helpers

namespace rmfht_pair {

using u32 = uint32_t;
using u64 = unsigned long long;
using rmfht::kFull;
constexpr int L = 2;  // list size (paths per item)
#ifndef RMFHT_PAIR_WARPS
#define RMFHT_PAIR_WARPS 16  // lock-stepped warps per CTA (128 registers, one CTA per SM)
#endif
constexpr int kPairWarps = RMFHT_PAIR_WARPS;
#ifndef RMFHT_PAIR_PREFETCH
#define RMFHT_PAIR_PREFETCH 1
#endif

// |x| as an operand modifier.  It differs from the reference's x < 0 ? -x : x
// only in the sign of a zero, which no comparison, sum or decision sees.
__device__ __forceinline__ float tabs(float x) { return fabsf(x); }
// f_op (list_engine.py:15-20): one FMNMX.XORSIGN — min(|a|,|b|) with the
// sign bit of a*b; equal to the reference's min(|a|,|b|) sgn(a) sgn(b)
// (sgn(0) = +1) up to the sign of a zero result (rmfht_fast.cuh f_op)
__device__ __forceinline__ float f_op(float a, float b) {
    float r;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float g_op(float a, float b, int c) { return c ? b - a : b + a; }

// numpy pairwise sum of v(0 .. NV-1) (rmfht_kernels.cuh pairwise_groups, one group)
template <int NV, typename F>
__device__ __forceinline__ float pw_sum(F v) {
    static_assert(NV <= 128, "pair kernel: rows of at most 128");
    if constexpr (NV < 8) {
        float s = v(0);
#pragma unroll
        for (int i = 1; i < NV; i++) s += v(i);
        return s;
    } else {
        constexpr int LEN = NV / 8;
        float r[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            float s = v(q);
#pragma unroll
            for (int i = 1; i < LEN; i++) s += v(q + 8 * i);
            r[q] = s;
        }
        return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    }
}

// an affine map by columns (rmfht::MapS restricted to MM variables)
template <int MM>
struct Map {
    u32 icol[MM], c, col[MM], b;
    __device__ __forceinline__ u32 inv(u32 j) const {
        u32 v = c;
#pragma unroll
        for (int k = 0; k < MM; k++) v ^= ((j >> k) & 1u) ? icol[k] : 0u;
        return v;
    }
    __device__ __forceinline__ u32 fwd(u32 i) const {
        u32 v = b;
#pragma unroll
        for (int k = 0; k < MM; k++) v ^= ((i >> k) & 1u) ? col[k] : 0u;
        return v;
    }
    __device__ __forceinline__ void load(const uint16_t* rec) {  // record: col, b, icol, c
#pragma unroll
        for (int k = 0; k < MM; k++) {
            col[k] = rec[k];
            icol[k] = rec[MM + 1 + k];
        }
        b = rec[MM];
        c = rec[2 * MM + 1];
    }
};

// composite "apply first, then t" (rmfht_kernels.cuh compose)
template <int MM>
__device__ __forceinline__ Map<MM> compose(const Map<MM>& t, const Map<MM>& first) {
    auto lin = [](const u32* cols, u32 x) {
        u32 v = 0;
#pragma unroll
        for (int k = 0; k < MM; k++) v ^= ((x >> k) & 1u) ? cols[k] : 0u;
        return v;
    };
    Map<MM> out;
#pragma unroll
    for (int k = 0; k < MM; k++) {
        out.icol[k] = lin(first.icol, t.icol[k]);
        out.col[k] = lin(t.col, first.col[k]);
    }
    out.c = lin(first.icol, t.c) ^ first.c;
    out.b = lin(t.col, first.b) ^ t.b;
    return out;
}

// index tables of a map's inverse for j = lo3 | mid << 3 | top << (MM-1)
template <int MM>
struct InvTab {
    static constexpr int NA = MM - 1 >= 3 ? 8 : (1 << (MM - 1));
    static constexpr int NB = (MM - 1) > 3 ? (1 << (MM - 4)) : 1;
    u32 A[NA], B[NB], top;
    __device__ __forceinline__ void build(const Map<MM>& mp) {
#pragma unroll
        for (int q = 0; q < NA; q++) {
            u32 v = mp.c;
#pragma unroll
            for (int k = 0; k < 3 && k < MM - 1; k++) v ^= ((q >> k) & 1) ? mp.icol[k] : 0u;
            A[q] = v;
        }
#pragma unroll
        for (int q = 0; q < NB; q++) {
            u32 v = 0;
#pragma unroll
            for (int k = 3; k < MM - 1; k++) v ^= ((q >> (k - 3)) & 1) ? mp.icol[k] : 0u;
            B[q] = v;
        }
        top = mp.icol[MM - 1];
    }
    // sigma^-1(j) for a compile-time j (unrolled loops)
    __device__ __forceinline__ u32 at(int j) const {
        const u32 v = A[j % NA] ^ B[(j / NA) % NB];
        return ((j >> (MM - 1)) & 1) ? v ^ top : v;
    }
    // the same as byte offsets OR-ed into a shared-window base aligned to 4N
    // bytes: one LOP3 per gather address (rmfht_fast.cuh RootIdx)
    __device__ __forceinline__ void rebase(u32 base) {
#pragma unroll
        for (int q = 0; q < NA; q++) A[q] = base | (A[q] << 2);
#pragma unroll
        for (int q = 0; q < NB; q++) B[q] <<= 2;
        top <<= 2;
    }
};

__device__ __forceinline__ float lds(u32 saddr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
    return v;
}

template <int SS>
using BitsT = typename std::conditional<(SS > 5), u64, u32>::type;

// packed float32x2 (sm_100 FADD2): one instruction, two lanes of work (rmfht_fast.cuh)
__device__ __forceinline__ u64 pk(float lo, float hi) {
    return ((u64)__float_as_uint(hi) << 32) | (u64)__float_as_uint(lo);
}
__device__ __forceinline__ float plo(u64 v) { return __uint_as_float((u32)v); }
__device__ __forceinline__ float phi(u64 v) { return __uint_as_float((u32)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// exchange with the partner thread (the other path of the item)
template <typename X>
__device__ __forceinline__ X other(X v) {
    if constexpr (sizeof(X) == 8) {
        u64 u;
        memcpy(&u, &v, 8);
        const u32 lo = __shfl_xor_sync(kFull, (u32)u, 1), hi = __shfl_xor_sync(kFull, (u32)(u >> 32), 1);
        u = ((u64)hi << 32) | lo;
        X r;
        memcpy(&r, &u, 8);
        return r;
    } else {
        return __shfl_xor_sync(kFull, v, 1);
    }
}
// value of path slot s of this item (s = 0 or 1; q = my slot)
template <typename X>
__device__ __forceinline__ X from_slot(X mine, int q, int s) {
    const X o = other(mine);
    return s == q ? mine : o;
}

struct Node {  // per-thread list state of its path slot
    float pm;
};

// fhtl with L = 2 (fht_decode.py:101-126): P = 2 paths, K = 2 bins each,
// keep 2 of the pool of 4 by (pm, source, bin).  Returns this slot's
// survivor codeword bits; *lin = its source slot.
// (x is consumed: the transform runs in place)
template <int SS>
__device__ __forceinline__ BitsT<SS> fhtl2(float (&x)[1 << SS], Node& nd, int q, int* lin) {
    constexpr int n = 1 << SS;
    const float llr = pw_sum<n>([&](int j) { return tabs(x[j]); });  // :114
    float (&w)[n] = x;
    // :28-48, two butterflies per packed f32x2 instruction (FADD2): pairs
    // (lo, lo + half) and (lo + d, lo + half + d), d = 1 for half >= 2, else 2
#pragma unroll
    for (int t = 0; t < SS; t++) {
        const int half = n >> (t + 1);
        const int d = half >= 2 ? 1 : 2;
#pragma unroll
        for (int lo = 0; lo < n; lo++) {
            if ((lo & half) || (lo & d)) continue;
            const u64 a = pk(w[lo], w[lo + d]), b = pk(w[lo + half], w[lo + half + d]);
            const u64 dd = sub2(b, a), ee = add2(b, a);
            w[lo] = plo(dd);
            w[lo + d] = phi(dd);
            w[lo + half] = plo(ee);
            w[lo + half + d] = phi(ee);
        }
    }
    // top-2 bins by |w| descending, ties to the lower bin (:116)
    float a1 = -1.f, a2 = -1.f, w1 = 0.f, w2 = 0.f;
    int b1 = 0, b2 = 1;
#pragma unroll
    for (int k = 0; k < n; k++) {  // branch-free (selects)
        const float a = tabs(w[k]);
        const bool g1 = a > a1, g2 = a > a2;
        a2 = g1 ? a1 : (g2 ? a : a2);
        w2 = g1 ? w1 : (g2 ? w[k] : w2);
        b2 = g1 ? b1 : (g2 ? k : b2);
        a1 = g1 ? a : a1;
        w1 = g1 ? w[k] : w1;
        b1 = g1 ? k : b1;
    }
    // pool (:119-120): candidate c = slot * 2 + k
    float cpm[4], cw[4];
    int cb[4];
    {
        const float p0 = nd.pm + 0.5f * (llr - a1), p1 = nd.pm + 0.5f * (llr - a2);
        const float o0 = other(p0), o1 = other(p1), ow1 = other(w1), ow2 = other(w2);
        const int ob1 = other(b1), ob2 = other(b2);
        if (q == 0) {
            cpm[0] = p0; cw[0] = w1; cb[0] = b1; cpm[1] = p1; cw[1] = w2; cb[1] = b2;
            cpm[2] = o0; cw[2] = ow1; cb[2] = ob1; cpm[3] = o1; cw[3] = ow2; cb[3] = ob2;
        } else {
            cpm[0] = o0; cw[0] = ow1; cb[0] = ob1; cpm[1] = o1; cw[1] = ow2; cb[1] = ob2;
            cpm[2] = p0; cw[2] = w1; cb[2] = b1; cpm[3] = p1; cw[3] = w2; cb[3] = b2;
        }
    }
    // the candidate ranked q (lexsort (pm, source, bin); stable)
    int sel = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        int rank = 0;
#pragma unroll
        for (int d = 0; d < 4; d++)
            rank += (cpm[d] < cpm[c]) || (cpm[d] == cpm[c] && ((d >> 1) < (c >> 1) || ((d >> 1) == (c >> 1) && cb[d] < cb[c])));
        if (rank == q) sel = c;
    }
    float spm = cpm[0], sw = cw[0];
    int sb = cb[0];
#pragma unroll
    for (int c = 1; c < 4; c++)
        if (sel == c) { spm = cpm[c]; sw = cw[c]; sb = cb[c]; }
    nd.pm = spm;
    *lin = sel >> 1;
    // codeword bits: bit j = parity(~b & ~j & (n-1)) ^ [w_b < 0] (:58-62, :123-125)
    using BT = BitsT<SS>;
    const u32 B = (u32)(~sb) & (u32)(n - 1);
    constexpr u64 pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                            0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
    BT P = 0;
#pragma unroll
    for (int k = 0; k < SS; k++)
        if ((B >> k) & 1u) P ^= (BT)pat[k];
    const int c0 = (__popc(B) & 1) ^ (sw < 0.f ? 1 : 0);
    constexpr BT VM = (n >= 8 * (int)sizeof(BT)) ? (BT)~(BT)0 : (BT)(((BT)1 << n) - 1);
    return (c0 ? ~P : P) & VM;
}

// spc_decode_list with L = 2 (list_engine.py:68-119), n = 2^SS
template <int SS>
__device__ __forceinline__ BitsT<SS> spc2(const float (&x)[1 << SS], Node& nd, int q, int* lin) {
    constexpr int n = 1 << SS;
    constexpr int TAU = (L < n ? L : n) < n - 1 ? (L < n ? L : n) : n - 1;
    using BT = BitsT<SS>;
    // stable ascending order of |alpha| (:83): rank of each element
    int ordpos[TAU + 1];  // positions of ranks 0 .. TAU
    float amag[TAU + 1];
#pragma unroll
    for (int r = 0; r <= TAU; r++) { ordpos[r] = 0; amag[r] = 0.f; }
    BT sg = 0;
#pragma unroll
    for (int j = 0; j < n; j++) {
        const float mj = tabs(x[j]);
        int rank = 0;
#pragma unroll
        for (int i = 0; i < n; i++) {
            const float mi = tabs(x[i]);
            rank += (mi < mj) || (mi == mj && i < j);
        }
#pragma unroll
        for (int r = 0; r <= TAU; r++)
            if (rank == r) { ordpos[r] = j; amag[r] = mj; }
        sg |= (BT)(x[j] < 0.f ? 1 : 0) << j;
    }
    int par;
    if constexpr (sizeof(BT) == 8) par = __popcll(sg) & 1;
    else par = __popc(sg) & 1;
    // per-path state (:84-88), then the TAU splits (:97-112), computed the
    // same on both threads; path slots 0 / 1 held in explicit pairs (no
    // dynamically indexed local arrays)
    const float mypm = nd.pm + (par ? amag[0] : 0.f);
    const float opm = other(mypm);
    const int opar = other(par);
    float a0[TAU + 1], a1[TAU + 1];  // sorted magnitudes of input paths 0 and 1
#pragma unroll
    for (int r = 0; r <= TAU; r++) {
        const float oa = other(amag[r]);
        a0[r] = q == 0 ? amag[r] : oa;
        a1[r] = q == 0 ? oa : amag[r];
    }
    float pm0 = q == 0 ? mypm : opm, pm1 = q == 0 ? opm : mypm;
    float pr0 = (float)(q == 0 ? par : opar), pr1 = (float)(q == 0 ? opar : par);
    int pa0 = 0, pa1 = 1;
    u32 fl0 = 0u, fl1 = 0u;
#pragma unroll
    for (int j = 1; j <= TAU; j++) {
        const float aj0 = pa0 ? a1[j] : a0[j], am0 = pa0 ? a1[0] : a0[0];
        const float aj1 = pa1 ? a1[j] : a0[j], am1 = pa1 ? a1[0] : a0[0];
        float cand[4];
        cand[0] = pm0;
        cand[1] = pr0 != 0.f ? (pm0 + aj0) - am0 : (pm0 + aj0) + am0;
        cand[2] = pm1;
        cand[3] = pr1 != 0.f ? (pm1 + aj1) - am1 : (pm1 + aj1) + am1;
        int s0 = 0, s1 = 1;  // the two lowest candidates, stable (argsort, :104)
#pragma unroll
        for (int c = 0; c < 4; c++) {
            int rank = 0;
#pragma unroll
            for (int d = 0; d < 4; d++) rank += (cand[d] < cand[c]) || (cand[d] == cand[c] && d < c);
            if (rank == 0) s0 = c;
            if (rank == 1) s1 = c;
        }
        auto pick = [&](int sc, float& npm, float& npr, int& npa, u32& nfl) {
            const int which = sc & 1, src = sc >> 1;
            float cv = cand[0];
#pragma unroll
            for (int c = 1; c < 4; c++)
                if (sc == c) cv = cand[c];
            npm = cv;
            const u32 fs = src ? fl1 : fl0;
            const float ps = src ? pr1 : pr0;
            nfl = fs | (which ? (1u << j) : 0u);
            npr = which ? 1.f - ps : ps;
            npa = src ? pa1 : pa0;
        };
        float n0pm, n0pr, n1pm, n1pr;
        int n0pa, n1pa;
        u32 n0fl, n1fl;
        pick(s0, n0pm, n0pr, n0pa, n0fl);
        pick(s1, n1pm, n1pr, n1pa, n1fl);
        pm0 = n0pm; pr0 = n0pr; pa0 = n0pa; fl0 = n0fl;
        pm1 = n1pm; pr1 = n1pr; pa1 = n1pa; fl1 = n1fl;
    }
    // my slot's survivor: sign xor flips, least reliable fixes even parity (:114-118)
    const int par_q = q == 0 ? pa0 : pa1;
    const u32 flq = q == 0 ? fl0 : fl1;
    nd.pm = q == 0 ? pm0 : pm1;
    *lin = par_q;
    const BT psg = from_slot(sg, q, par_q);
    int pos[TAU + 1];
#pragma unroll
    for (int r = 0; r <= TAU; r++) pos[r] = from_slot(ordpos[r], q, par_q);
    BT bits = psg;
#pragma unroll
    for (int j = 1; j <= TAU; j++)
        if ((flq >> j) & 1u) bits ^= (BT)1 << pos[j];
    int tot;
    if constexpr (sizeof(BT) == 8) tot = __popcll(bits) & 1;
    else tot = __popc(bits) & 1;
    bits ^= (BT)tot << pos[0];
    return bits;
}

// _decode_node without permutations (RR >= 2, below the root)
template <int RR, int SS>
__device__ __forceinline__ BitsT<SS> node(float (&x)[1 << SS], Node& nd, int q, int* lin) {
    constexpr int n = 1 << SS, h = n / 2;
    if constexpr (RR == 1) {
        return fhtl2<SS>(x, nd, q, lin);
    } else if constexpr (RR == SS - 1) {
        return spc2<SS>(x, nd, q, lin);
    } else {
        float xl[h];
#pragma unroll
        for (int k = 0; k < h; k++) xl[k] = f_op(x[k], x[k + h]);  // :100
        int l1;
        const BitsT<SS - 1> bl = node<RR - 1, SS - 1>(xl, nd, q, &l1);  // :101
        float xr[h];
        // alphas = alphas[lin1] (:102), then g (:104)
        const bool moved = __any_sync(kFull, l1 != q);
#pragma unroll
        for (int k = 0; k < h; k++) {
            float lo = x[k], hi = x[k + h];
            if (moved) {
                lo = from_slot(lo, q, l1);
                hi = from_slot(hi, q, l1);
            }
            xr[k] = g_op(lo, hi, (int)((bl >> k) & 1));
        }
        int l2;
        const BitsT<SS - 1> br = node<RR, SS - 1>(xr, nd, q, &l2);  // :105
        // combine (:106-107) and lineage (:113: lineage0 is the identity here)
        const BitsT<SS - 1> blm = from_slot(bl, q, l2);
        *lin = from_slot(l1, q, l2);
        return ((BitsT<SS>)br << h) | (BitsT<SS>)(blm ^ br);
    }
}

template <int MM>
struct Out2 {  // root-domain bits of a path, N = 2^MM <= 128
    u64 w[(1 << MM) > 64 ? 2 : 1];
};

template <int MM>
__global__ void __launch_bounds__(32 * kPairWarps, 1) pair_kernel(rmfht::Params<float> prm) {
    constexpr int N = 1 << MM, H = N / 2, NW = N >= 32 ? N / 32 : 1, S = L + 2 * L;
    static_assert(MM >= 4 && MM <= 7, "pair kernel: RM(2, m), 4 <= m <= 7");
    constexpr int REC = 2 * MM + 2;
    extern __shared__ __align__(16) unsigned char fraw[];  // per warp: the frames of its 16 items
    // frames start 4N-byte aligned in the shared window (gather offsets are OR-ed in)
    const u32 rs = (u32)__cvta_generic_to_shared(fraw);
    float* const fr = reinterpret_cast<float*>(fraw + ((((rs + 4 * N - 1) / (4 * N)) * (4 * N)) - rs));
    const int lane = threadIdx.x & 31, wib = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // provably warp-uniform
    const int M = prm.M, FPW = 16 / M;  // frames per warp (M divides 16)
    // PREF: the next round's frames and map records are in flight (cp.async,
    // double buffers) while this round decodes; needs 16-byte aligned sources
    // and whole 16-byte records per item (m = 7)
    constexpr int RECB = S * REC * 2;  // record bytes per item
    constexpr bool PREFC = RMFHT_PAIR_PREFETCH != 0 && RECB % 16 == 0;
    // (M >= 4: at most four frames per warp, so the double buffers fit; prepare_pair sizes them)
    const bool pref = PREFC && prm.M >= 4 && (reinterpret_cast<uintptr_t>(prm.llr) & 15u) == 0 &&
                      (reinterpret_cast<uintptr_t>(prm.maps) & 15u) == 0;
    const size_t fbuf = (size_t)kPairWarps * FPW * N;  // floats of one frame buffer (all warps)
    float* const fw0 = fr + (size_t)wib * FPW * N;  // the warp's frames in buffer 0
    float* fw = fw0;
    uint16_t* const recs0 = reinterpret_cast<uint16_t*>(fr + 2 * fbuf) + (size_t)wib * 16 * S * REC;
    const size_t rbuf = (size_t)kPairWarps * 16 * S * REC;  // uint16 of one record buffer (all warps)
    // tensor memory for the root's gathers between f and g (rmfht2::tmem_park):
    // N columns per thread, warp w in lanes 32 (w % 4) .. + 31, columns N (w / 4) ..
    constexpr bool TPARK = RMFHT_TMEM_PARK != 0 && H % 8 == 0 && (kPairWarps + 3) / 4 * N <= 512;
    __shared__ u32 tmem_slot;
    u32 tmem = 0;
    if constexpr (TPARK) {
        if (wib == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             (u32)__cvta_generic_to_shared(&tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem = tmem_slot + ((u32)(32 * (wib & 3)) << 16) + (u32)(N * (wib >> 2));
    }
    const int q = lane & 1, it = lane >> 1;
    const long long items = prm.B * (long long)M;
    const long long warps_total = (items + 15) / 16;
    // lock-stepped rounds (a CTA barrier per round): the warps of the CTA run
    // the same ~4K-instruction body together and share one instruction-fetch
    // stream (free-running warps thrashed the instruction caches: 39%
    // no_instructions stalls at 12 warps per SM)
    const int nwb = blockDim.x >> 5;
    auto prefetch = [&](long long wgn, int buf) {
        if (wgn >= warps_total) return;
        const long long i0 = wgn * 16, fn = i0 / M;
        const u32 fsa = (u32)__cvta_generic_to_shared(fw0 + buf * fbuf);
        for (int i = lane; i < FPW * N / 4; i += 32) {
            const long long f = fn + (i * 4) / N;
            if (f < prm.B) rmfht2::cp_async16(fsa + 16u * i, reinterpret_cast<const float4*>(prm.llr + f * N) + (i % (N / 4)));
        }
        const long long left = items - i0;
        const int nb = (int)(left < 16 ? left : 16) * RECB / 16;  // 16-byte chunks of the round's records
        const u32 rsa = (u32)__cvta_generic_to_shared(recs0 + buf * rbuf);
        const char* gr = reinterpret_cast<const char*>(prm.maps + (size_t)i0 * S * REC);
        for (int i = lane; i < nb; i += 32) rmfht2::cp_async16(rsa + 16u * i, gr + 16 * i);
        rmfht2::cp_async_commit();
    };
    int cur = 0;
    if (pref) prefetch((long long)blockIdx.x * nwb + wib, 0);
    for (long long r0 = (long long)blockIdx.x * nwb; r0 < warps_total; r0 += (long long)gridDim.x * nwb) {
        const long long wg = r0 + wib;
        if (wg >= warps_total) {
            __syncthreads();
            continue;
        }
        const long long item0 = wg * 16, f0 = item0 / M;
        if (pref) {
            rmfht2::cp_async_wait_all();
            __syncwarp();
            fw = fw0 + cur * fbuf;
            prefetch(wg + (long long)gridDim.x * nwb, cur ^ 1);
        } else {
        // the warp's frames into shared memory (coalesced)
        __syncwarp();
        for (int i = lane; i < FPW * N / 4; i += 32) {
            const long long f = f0 + (i * 4) / N;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (f < prm.B) v = __ldg(reinterpret_cast<const float4*>(prm.llr + f * N) + (i % (N / 4)));
            reinterpret_cast<float4*>(fw)[i] = v;
        }
        __syncwarp();
        }
        const long long item = item0 + it;
        const bool live = item < items;
        const long long fidx = live ? item / M : f0;
        const int at = live ? (int)(item - fidx * M) : 0;
        const float* alpha = fw + (fidx - f0) * N;
        const u32 abase = (u32)__cvta_generic_to_shared(alpha);
        // this thread's maps: root map q, trial maps q and q + 2 (both permute path q)
        const uint16_t* rec = pref ? recs0 + cur * rbuf + (size_t)(live ? it : 0) * S * REC
                                   : prm.maps + (size_t)(live ? item : item0) * S * REC;
        Map<MM> root, t0, t1;
        root.load(rec + q * REC);
        t0.load(rec + (L + q) * REC);
        t1.load(rec + (L + q + 2) * REC);
        const Map<MM> c0 = compose<MM>(t0, root), c1 = compose<MM>(t1, root);
        // ---- root permutation extension (automorphism.py:207-237): LM of trials q, q+2
        InvTab<MM> tb0, tb1;
        tb0.build(c0);
        tb1.build(c1);
        tb0.rebase(abase);
        tb1.rebase(abase);
        float lmv[2];
#pragma unroll 1
        for (int tt = 0; tt < 2; tt++) {  // one copy of the 64-pair body (instruction cache)
            InvTab<MM> tb;
#pragma unroll
            for (int v = 0; v < InvTab<MM>::NA; v++) tb.A[v] = tt ? tb1.A[v] : tb0.A[v];
#pragma unroll
            for (int v = 0; v < InvTab<MM>::NB; v++) tb.B[v] = tt ? tb1.B[v] : tb0.B[v];
            tb.top = tt ? tb1.top : tb0.top;
            const float v = pw_sum<H>([&](int j) {
                return fminf(fabsf(lds(tb.at(j))), fabsf(lds(tb.at(j + H))));
            });
            if (tt) lmv[1] = v;
            else lmv[0] = v;
        }
        const float lm0 = lmv[0], lm1 = lmv[1];
        // all four trials: t = 0 (slot 0), 1 (slot 1), 2 (slot 0), 3 (slot 1)
        float lm[4];
        u32 key[4];
        {
            const float o0 = other(lm0), o1 = other(lm1);
            const u32 k0 = c0.icol[MM - 1], k1 = c1.icol[MM - 1];
            const u32 ok0 = other(k0), ok1 = other(k1);
            lm[q] = lm0; lm[q + 2] = lm1; lm[1 - q] = o0; lm[3 - q] = o1;
            key[q] = k0; key[q + 2] = k1; key[1 - q] = ok0; key[3 - q] = ok1;
        }
        // tie fix: equal pairing directions keep equal LM (select_trials;
        // on by default for float32, RMFHT_NO_TIE_FIX turns it off)
#pragma unroll
        for (int t = 1; t < 4 && prm.tie_fix; t++) {
            bool done = false;
#pragma unroll
            for (int s = 0; s < t; s++)
                if (!done && key[s] == key[t]) { lm[t] = lm[s]; done = true; }
        }
        // keep 2 by LM descending, ties to the lower trial (:234)
        int sel[2] = {0, 1};
#pragma unroll
        for (int t = 0; t < 4; t++) {
            int rank = 0;
#pragma unroll
            for (int s = 0; s < 4; s++) rank += (lm[s] > lm[t]) || (lm[s] == lm[t] && s < t);
            if (rank < 2) sel[rank] = t;
        }
        // my slot q takes trial sel[q]: its composite lives on the thread of
        // slot sel[q] % 2 as that thread's c0 (t < 2) or c1
        const int tq = sel[q];
        Map<MM> comp;
        {
            // owner = tq & 1; which = tq >> 1
#pragma unroll
            for (int k = 0; k < MM; k++) {
                const u32 i0 = other(c0.icol[k]), i1 = other(c1.icol[k]);
                const u32 o0 = other(c0.col[k]), o1 = other(c1.col[k]);
                const bool mine = (tq & 1) == q;
                comp.icol[k] = (tq >> 1) ? (mine ? c1.icol[k] : i1) : (mine ? c0.icol[k] : i0);
                comp.col[k] = (tq >> 1) ? (mine ? c1.col[k] : o1) : (mine ? c0.col[k] : o0);
            }
            const u32 cc0 = other(c0.c), cc1 = other(c1.c), bb0 = other(c0.b), bb1 = other(c1.b);
            const bool mine = (tq & 1) == q;
            comp.c = (tq >> 1) ? (mine ? c1.c : cc1) : (mine ? c0.c : cc0);
            comp.b = (tq >> 1) ? (mine ? c1.b : bb1) : (mine ? c0.b : bb0);
        }
        Node nd{0.f};  // pms stay 0 through the extension (pms[t % P] = 0)
        // ---- root: f from the frame through my composite (:100)
        InvTab<MM> tc;
        tc.build(comp);
        tc.rebase(abase);
        float xl[H];
        if constexpr (TPARK) {
            // the gathered halves wait in tensor memory for g (column j: lower half, H + j: upper)
#pragma unroll
            for (int j0 = 0; j0 < H; j0 += 8) {
                float a[8], b[8];
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    a[i] = lds(tc.at(j0 + i));
                    b[i] = lds(tc.at(j0 + i + H));
                }
                rmfht2::tmem_st8(tmem + j0, a);
                rmfht2::tmem_st8(tmem + H + j0, b);
#pragma unroll
                for (int i = 0; i < 8; i++) xl[j0 + i] = f_op(a[i], b[i]);
            }
            rmfht2::tmem_wait_st();
        } else {
#pragma unroll
            for (int j = 0; j < H; j++) xl[j] = f_op(lds(tc.at(j)), lds(tc.at(j + H)));
        }
        int l1;
        const BitsT<MM - 1> bl = node<1, MM - 1>(xl, nd, q, &l1);  // :101 (RM(1, m-1): FHT)
        float xr[H];
        if constexpr (TPARK) {
            // g on the parked gathers of slot l1 (:102-104): mine, or the partner thread's
#pragma unroll
            for (int j0 = 0; j0 < H; j0 += 8) {
                u32 ra[8], rb[8];
                rmfht2::tmem_ld8(tmem + j0, ra);
                rmfht2::tmem_ld8(tmem + H + j0, rb);
                rmfht2::tmem_wait_ld16(ra, rb);
#pragma unroll
                for (int i = 0; i < 8; i++)
                    xr[j0 + i] = g_op(__uint_as_float(from_slot(ra[i], q, l1)), __uint_as_float(from_slot(rb[i], q, l1)),
                                      (int)((bl >> (j0 + i)) & 1));
            }
        } else {
        // g through the composite of slot l1 (:102-104)
        InvTab<MM> tg;
        {
            Map<MM> cs;
#pragma unroll
            for (int k = 0; k < MM; k++) cs.icol[k] = from_slot(comp.icol[k], q, l1);
            cs.c = from_slot(comp.c, q, l1);
            tg.build(cs);
            tg.rebase(abase);
        }
#pragma unroll
        for (int j = 0; j < H; j++) xr[j] = g_op(lds(tg.at(j)), lds(tg.at(j + H)), (int)((bl >> j) & 1));
        }
        int l2;
        const BitsT<MM - 1> br = node<2, MM - 1>(xr, nd, q, &l2);  // :105
        const BitsT<MM - 1> blm = from_slot(bl, q, l2);
        const int chain = from_slot(l1, q, l2);  // :109 root chain of my slot
        // root-domain bits of my slot: [bl[lin2] ^ br, br] (:106-107)
        Out2<MM> ob;
        if constexpr (N > 64) {
            ob.w[0] = (u64)(blm ^ br);
            ob.w[1] = (u64)br;
        } else {
            ob.w[0] = ((u64)br << H) | (u64)(blm ^ br);
        }
        // best path: first minimum (:152)
        const float opm = other(nd.pm);
        const float pm0 = q == 0 ? nd.pm : opm, pm1 = q == 0 ? opm : nd.pm;
        const int best = pm1 < pm0 ? 1 : 0;
        const float bpm = best ? pm1 : pm0;
        // un-permute the best path by the composite of its root chain (:147-150):
        // codeword bit i = beta[sigma(i)]; thread q takes words q, q + 2, ...
        const int bchain = from_slot(chain, q, best);
        Map<MM> cf;
        {
            // composite of slot bchain (forward columns)
#pragma unroll
            for (int k = 0; k < MM; k++) cf.col[k] = from_slot(comp.col[k], q, bchain);
            cf.b = from_slot(comp.b, q, bchain);
        }
        Out2<MM> bb;
#pragma unroll
        for (int w = 0; w < (N > 64 ? 2 : 1); w++) bb.w[w] = from_slot(ob.w[w], q, best);
        // sigma(32 t + i) = (b ^ A 32t) ^ (A i): per-word base, tables over i
        constexpr int PB = N < 32 ? MM : 5;  // bits of i within a word
        u32 tlo[8], thi[PB > 3 ? 1 << (PB - 3) : 1];
#pragma unroll
        for (int v = 0; v < 8; v++) {
            u32 e = 0;
#pragma unroll
            for (int k = 0; k < 3 && k < PB; k++) e ^= ((v >> k) & 1) ? cf.col[k] : 0u;
            tlo[v] = e;
        }
#pragma unroll
        for (int v = 0; v < (PB > 3 ? 1 << (PB - 3) : 1); v++) {
            u32 e = 0;
#pragma unroll
            for (int k = 3; k < PB; k++) e ^= ((v >> (k - 3)) & 1) ? cf.col[k] : 0u;
            thi[v] = e;
        }
        constexpr int WPT = NW > 1 ? NW / 2 : 1;  // words per thread: t = 2 j + q
        u32 mine[WPT];
#pragma unroll
        for (int j = 0; j < WPT; j++) {
            const int t = NW > 1 ? 2 * j + q : 0;
            const u32 base = cf.fwd((u32)(t * 32));
            u32 word = 0;
#pragma unroll
            for (int i = 0; i < (N < 32 ? N : 32); i++) {
                const u32 e = base ^ tlo[i & 7] ^ thi[(i >> 3) & ((PB > 3 ? 1 << (PB - 3) : 1) - 1)];
                u64 src = bb.w[0];
                if constexpr (N > 64) src = (e & 64) ? bb.w[1] : bb.w[0];
                word |= (u32)((src >> (e & 63)) & 1ull) << i;
            }
            mine[j] = word;
        }
        // exchange halves: both threads of the item hold the whole codeword
        u32 cw[NW];
#pragma unroll
        for (int j = 0; j < WPT; j++) {
            const u32 o = other(mine[j]);
            if (NW > 1) {
                cw[2 * j] = q == 0 ? mine[j] : o;
                cw[2 * j + 1] = q == 0 ? o : mine[j];
            } else {
                cw[0] = mine[0];
            }
        }
        // reported pm of this attempt (rmfht::CorrPm order: "lane" l sums
        // positions l + 32 t in double, then the xor tree 16 .. 1)
        auto corr = [&]() {
            double qv[16];  // thread q holds "lanes" 16 q .. 16 q + 15
#pragma unroll
            for (int l = 0; l < 16; l++) {
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < (N + 31) / 32; t++) {
                    const int i = t * 32 + 16 * q + l;
                    if (i < N) {
                        const float a = alpha[i];
                        const int c = (int)((cw[i / 32] >> (i % 32)) & 1u);
                        if ((a < 0.f) != (c != 0)) acc += fabs((double)a);
                    }
                }
                qv[l] = acc;
            }
            // off 16: lane l (< 16) + lane l + 16 (the partner's qv[l])
#pragma unroll
            for (int l = 0; l < 16; l++) {
                const double o = other(qv[l]);
                qv[l] = q == 0 ? qv[l] + o : o + qv[l];
            }
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1)
#pragma unroll
                for (int l = 0; l < off; l++) qv[l] = qv[l] + qv[l + off];
            return (float)qv[0];
        };
        // every attempt's reported pm (one inlined copy: the winners' come from it)
        const float rep = corr();
        if (live && q == 0) {
            if (prm.att_pm) prm.att_pm[item] = rep;
            if (prm.att_cw)
                for (int t = 0; t < NW; t++) prm.att_cw[item * NW + t] = cw[t];
        }
        // ensemble pick over the frame's M attempts (items it - at .. + M - 1):
        // first strict minimum of the accumulated pm (top_decoders.py:200)
        float vpm = live ? bpm : __int_as_float(0x7f800000);
        int vat = live ? at : 0x7fffffff;
#pragma unroll
        for (int off = 2; off < 32; off <<= 1) {
            if (off >= 2 * M) break;
            const float opv = __shfl_xor_sync(kFull, vpm, off);
            const int oat = __shfl_xor_sync(kFull, vat, off);
            if (opv < vpm || (opv == vpm && oat < vat)) { vpm = opv; vat = oat; }
        }
        const bool winner = live && vat == at;
        if (winner && q == 0) {
            for (int t = 0; t < NW; t++) prm.cw[fidx * NW + t] = cw[t];
            prm.pm[fidx] = rep;
            prm.attempt[fidx] = at;
            prm.path[fidx] = best;
        }
        cur ^= 1;
        __syncthreads();
    }
    if constexpr (TPARK) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (wib == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_slot) : "memory");
    }
}

}  // namespace rmfht_pair
