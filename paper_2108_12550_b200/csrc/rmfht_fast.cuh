// B200 (sm_100a) float32 throughput kernel for p-FHT-FSCL-L-M ("v2").
//
// Same decoder as rmfht_kernels.cuh (the float64 reference-exact kernel),
// re-laid out for throughput:
//   * one warp = one (frame, attempt); the L list paths own 32/L lanes each
//     ("lane group"); a node vector of size n lives in REGISTERS, element
//     e = k*LPP + u in register slot k of lane u of its path's group, so f/g
//     are register-local and an FHT needs log2(LPP) shuffle stages only;
//   * the channel LLRs of the frame sit in shared memory (root gathers) and
//     in registers in "channel layout" (lane l holds alpha[l + 32 s]) for the
//     permutation-extension reliabilities;
//   * root gathers cost one 3-input XOR and one LDS per element (affine index
//     tables), no per-element bit loops;
//   * LM (automorphism.py:232-233) is summed in a canonical channel-domain
//     order, so trials that pair the same channel entries get bit-identical
//     LM (the structural ties of SURVEY §8(c) stay exact without a tie fix);
//   * the FHT top-k / pool step (fht_decode.py:116-120) filters candidates
//     with an exact path-metric threshold before any sorting.
// The summation orders are restated by the oracle's float32 mode
// (oracle/rmo_impl.h, RMO_ORDER_V2), which is how bit-exact parity of this
// kernel is checked.  FHT butterflies run in the reference's stage order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "rmfht_kernels.cuh"  // MapS, Params, maps_per_attempt, helpers

namespace rmfht2 {

using rmfht::MapS;
using rmfht::kFull;
using u32 = uint32_t;
using u64 = unsigned long long;

__host__ __device__ constexpr int clog2(int x) { return x <= 1 ? 0 : 1 + clog2(x >> 1); }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// f_op (list_engine.py:15-20): min(|a|,|b|) with the sign of a*b
// (sgn(0) = +1 only changes the sign of a zero result, which never matters).
// One FMNMX.XORSIGN: min(|a|,|b|) with sign(a) ^ sign(b) — bit-identical to
// min(|a|,|b|) | (sign bit of a*b), which it replaces (3 instructions)
__device__ __forceinline__ float f_op(float a, float b) {
    float r;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

constexpr int kCap = 64;  // FHT candidate list capacity (two per lane)

// packed float32x2 (sm_100 FADD2 / FFMA2): one instruction, two lanes of work
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
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int R, int MM, int L>
struct Cfg {
    static constexpr int N = 1 << MM;
    static constexpr int LPP = 32 / L;
    static constexpr int LB = clog2(LPP);
    static constexpr int S = rmfht::maps_per_attempt(R, MM, L);
    static constexpr int NS = N / 32;  // channel slots per lane
    static constexpr int SPCMAX = 1 << cmin(R + 1, MM);
};

template <int SS, int LPP>
struct Lv {
    static constexpr int n = 1 << SS;
    static constexpr bool full = n >= LPP;       // every lane of the group active
    static constexpr int V = full ? n / LPP : 1;  // register slots per lane
    static constexpr int act = full ? LPP : n;    // active lanes of the group
};

// an affine map in device-record layout (rmfht.h): columns of A, b, columns
// of A^-1, A^-1 b — read in place from the item's record buffer
template <int MM>
struct alignas(4) MapR {
    uint16_t col[MM];
    uint16_t b;
    uint16_t icol[MM];
    uint16_t c;
};

// A^-1 x of a record (x: m-bit): the columns come in as 32-bit words (half
// word MM + 1 + k of the record is icol[k]) and every set bit of x XORs a
// whole word into the low- or high-half accumulator
template <int MM>
__device__ __forceinline__ uint32_t icol_apply(const MapR<MM>& mp, uint32_t x) {
    constexpr int W0 = (MM + 1) >> 1, W1 = (2 * MM) >> 1;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(&mp);
    uint32_t wv[W1 - W0 + 1];
#pragma unroll
    for (int i = 0; i <= W1 - W0; i++) wv[i] = wp[W0 + i];
    uint32_t lo = 0u, hi = 0u;
#pragma unroll
    for (int k = 0; k < MM; k++) {
        const int h = MM + 1 + k;
        if ((x >> k) & 1u) {
            if (h & 1) hi ^= wv[(h >> 1) - W0];
            else lo ^= wv[(h >> 1) - W0];
        }
    }
    return (lo ^ (hi >> 16)) & 0xffffu;
}

// per-warp shared scratch
template <int R, int MM, int L>
struct alignas(16) WS2 {
    using C = Cfg<R, MM, L>;
    static constexpr int RECW = (C::S > 0 ? C::S : 1) * (2 * MM + 2);  // uint16 per item's map records
    // inner permutation nodes (r >= 3) read the item's records deep in the
    // tree: double-buffered (the next item's are prefetched at item start);
    // otherwise the records are dead after the root's permutation extension
    // and one buffer is refilled from there
    static constexpr bool INNER = R >= 3 && MM - R >= 2;
    static constexpr int RB = INNER ? 2 : 1;
    alignas(16) uint16_t recs[RB][(RECW + 7) & ~7];  // cp.async prefetch; the item's maps
    MapR<MM> comp[L];  // composite map of each root path (root perm-ext winners)
    float pm[L], llrabs[L];
    alignas(16) float lm[2 * L];
    static constexpr int CA = kCap > L * L ? kCap : L * L;  // candidate list (and the exact fallback)
    static constexpr int CB = L * L > 2 * L ? L * L : 2 * L;  // per path / per split / fallback pool
    float cw[CA], cpm[CB];  // candidate values (|w| = fabsf(cw)), pool pms
    int16_t cb[CB], cp[CB], celig[CB];
    alignas(16) u64 ckey[kCap + 4];
    // FHT outputs spilled for candidate extraction: lane-major, padded (conflict-free STS.128)
    // largest FHT node: RM(1, m-r+1), the first left descendant (the root when r == 1).
    // The LM lane partials of the root permutation extension share the space
    // (they are dead before the first FHT node).
    static constexpr int VMAX = cmax(4, (R == 1 ? C::N : (C::N >> (R - 1))) / C::LPP);
    // The inner permutation nodes' vectors (vbuf, at the node's start) and
    // output bits (ubits, at its end) are dead whenever an FHT node runs, so
    // they share the space too; the largest inner node has N/2 elements.
    // The SPC nodes' scratch (magnitudes, signs, order of the tau+1 least
    // reliable positions) is dead whenever any of the others is live: SPC
    // nodes are leaves that run after an FHT node's spill rows died and
    // between an inner permutation node's vbuf (its start) and ubits (its end).
    union alignas(16) {
        float wsp[32][VMAX];  // 16-byte chunks XOR-swizzled per lane (wsp_idx): conflict-free STS.128
        float lmp[2 * L][32];
        float vbuf[R >= 3 ? L * C::N / 2 : 1];
        uint8_t ubits[R >= 3 ? L * C::N / 2 : 1];
        struct {
            float smag[L * (C::SPCMAX > 16 ? C::SPCMAX : 16)];
            uint8_t ssgn[L * C::SPCMAX];
            uint16_t sord[L * 16];
        };
    };
    // element k of lane `lane`'s row
    // t: extra per-node chunk twist (FhtLayout::twist) for the transposed FHT reads
    __device__ __forceinline__ static int wsp_idx(int lane, int k, int t = 0) {
        constexpr int G = VMAX / 4;  // 16-byte chunks per row
        const int swz = G >= 8 ? (lane & 7) : ((lane / (8 / G)) & (G - 1));
        return k ^ ((swz ^ t) << 2);  // chunk (k >> 2) ^ swz ^ t, word k & 3
    }
    __device__ __forceinline__ float& wspk(int lane, int k, int t = 0) { return wsp[lane][wsp_idx(lane, k, t)]; }
    int sel_src[2 * L], sel_bin[2 * L];
    float sel_w[2 * L], sel_pm[2 * L];
    int8_t l0[MM + 1][L], l1[MM + 1][L], l2[MM + 1][L], rootchain[L], ord[2 * L];
    int16_t nmap[MM + 1][L];
    int next_map;
};

template <int R, int MM, int L>
struct Ctx2 {
    using C = Cfg<R, MM, L>;
    WS2<R, MM, L>& ws;
    const float* alpha;        // frame LLRs (shared memory)
    const MapR<MM>* maps;      // the item's map records (shared memory); unused without permutations
    int perms;                 // p-FHT-FSCL (else FHT-FSCL / FHT-FSC: identity maps, no permutation nodes)
    float ach[C::NS];          // channel layout: ach[s] = alpha[lane + 32 s]
    int lane, p, u;
    u32 alpha_saddr;           // shared-window address of alpha (2 KB aligned)
    int ngen;                  // RMFHT_STATS only: FHT nodes of this item off the common case
    u32 tmem;                  // this warp's tensor-memory block (tmem_park), lane quadrant and first column
};

// ------------------------------------------------------------ helpers ----
template <int MN>
__device__ __forceinline__ u32 lin_apply(const u32* cols, u32 x) {
    u32 v = 0;
#pragma unroll
    for (int k = 0; k < MN; k++) v ^= (x >> k & 1u) ? cols[k] : 0u;
    return v;
}

// order-preserving float <-> uint32 keys (any sign; no NaN)
__device__ __forceinline__ u32 float_key(float f) {
    const u32 b = __float_as_uint(f);
    return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float key_float(u32 k) {
    return __uint_as_float(k ^ ((k >> 31) ? 0x80000000u : 0xffffffffu));
}

template <int MN>
__device__ __forceinline__ u32 lin_apply(const uint16_t* cols, u32 x) {
    u32 v = 0;
#pragma unroll
    for (int k = 0; k < MN; k++) v ^= (x >> k & 1u) ? (u32)cols[k] : 0u;
    return v;
}

// group-local xor reduce / broadcast helpers
template <int LPP, int ACT>
__device__ __forceinline__ float group_sum_tree(float v) {
    // ascending offsets 1, 2, 4 ... (mirrored by the oracle, RMO_ORDER_V2)
#pragma unroll
    for (int off = 1; off < ACT; off <<= 1) v = v + __shfl_xor_sync(kFull, v, off);
    return v;
}
template <int ACT>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
    for (int off = 1; off < ACT; off <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, off));
    return v;
}

// gather tables of one root path: element k*LPP+u of the permuted vector is
// alpha[base ^ A[k & 7] ^ B[k >> 3]] (byte offsets)
template <int MM, int LPP, int V>
struct RootIdx {
    static constexpr int NA = V < 8 ? V : 8;
    static constexpr int NB = V / NA;
    u32 base, A[NA], B[NB];
    // alpha_saddr: shared-window address of the frame LLRs, aligned to 2 KB so
    // that XOR-ing byte offsets (< 2 KB) into it forms the address directly
    template <typename Map>
    __device__ __forceinline__ void build(const Map& mp, int u, u32 alpha_saddr) {
        constexpr int LB = clog2(LPP);
        u32 bse = mp.c;
#pragma unroll
        for (int b = 0; b < LB; b++) bse ^= (u >> b & 1) ? (u32)mp.icol[b] : 0u;
        base = alpha_saddr | (bse << 2);
        A[0] = 0;
#pragma unroll
        for (int i = 1; i < NA; i++) {
            const int b = __ffs(i) - 1;  // lowest set bit: A[i] = A[i & (i-1)] ^ col
            A[i] = A[i & (i - 1)] ^ ((u32)mp.icol[LB + b] << 2);
        }
        B[0] = 0;
#pragma unroll
        for (int i = 1; i < NB; i++) {
            const int b = __ffs(i) - 1;
            B[i] = B[i & (i - 1)] ^ ((u32)mp.icol[LB + clog2(NA) + b] << 2);
        }
    }
    __device__ __forceinline__ u32 off(int k) const { return base ^ A[k % NA] ^ B[k / NA]; }
};

// the same tables for an inner node of size 2^SS: element k*LPP+u maps to
// index shift ^ cols(e) = base ^ A[k % NA] ^ B[k / NA] (one XOR per element
// instead of an SS-term GF(2) product)
template <int SS, int LPP, int V>
struct NodeIdx {
    static constexpr int NA = V < 8 ? V : 8;
    static constexpr int NB = V / NA;
    u32 base, A[NA], B[NB];
    __device__ __forceinline__ void build(const uint16_t* cols, u32 shift, int u) {
        constexpr int LB = clog2(LPP);
        u32 bse = shift;
#pragma unroll
        for (int b = 0; b < LB; b++) bse ^= (u >> b & 1) ? (u32)cols[b] : 0u;
        base = bse;
        A[0] = 0;
#pragma unroll
        for (int i = 1; i < NA; i++) A[i] = A[i & (i - 1)] ^ (u32)cols[LB + __ffs(i) - 1];
        B[0] = 0;
#pragma unroll
        for (int i = 1; i < NB; i++) B[i] = B[i & (i - 1)] ^ (u32)cols[LB + clog2(NA) + __ffs(i) - 1];
    }
    __device__ __forceinline__ u32 at(int k) const { return base ^ A[k % NA] ^ B[k / NA]; }
};

__device__ __forceinline__ float lds_byte(const float* base, u32 byteoff) {
    return *reinterpret_cast<const float*>(reinterpret_cast<const char*>(base) + byteoff);
}
// asynchronous global -> shared copies (LDGSTS), used to prefetch the next
// work item's LLRs and map records while the current item decodes
__device__ __forceinline__ void cp_async16(u32 saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(u32 saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// load from a 32-bit shared-window address (the gather tables carry the base)
__device__ __forceinline__ float lds_addr(u32 saddr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(saddr));
    return v;
}

// ------------------------------------------------- tensor-memory parking ----
// The root's g (:104) needs the same 2 VC channel LLRs per lane that its f
// (:100) gathered a whole left subtree earlier; there are no registers to
// keep them and no shared memory left, so the kernel gathered them twice —
// VC * 2 bank-conflicted LDS per lane, a fifth of the kernel's shared-memory
// wavefronts.  Blackwell's tensor memory (256 KB per SM, unused by a kernel
// without MMAs) holds them instead: f's gathers are stored with tcgen05.st
// (32 lanes x 32-bit columns, a warp's own lane quadrant, its own column
// block) and g reads them back with tcgen05.ld; when the left child re-ordered
// the paths, the values come from the source path's lanes by shuffles.
#ifndef RMFHT_XPARK
#define RMFHT_XPARK 1
#endif
#ifndef RMFHT_XPARK_MINV
#define RMFHT_XPARK_MINV 32
#endif
#ifndef RMFHT_NO_TMEM
#define RMFHT_TMEM_PARK 1
#else
#define RMFHT_TMEM_PARK 0
#endif
template <int R, int MM, int L>
__host__ __device__ constexpr bool tmem_park() {
    // an internal root whose halves have a multiple of 8 slots per lane (the
    // parked columns move in chunks of 8); 2 VC columns per warp, 7 warps per
    // lane quadrant at most
    constexpr int LPP = 32 / L, VC = (1 << (MM - 1)) / (LPP > 0 ? LPP : 1);
    return RMFHT_TMEM_PARK && R > 1 && R < MM - 1 && L <= 32 && VC >= 8 && VC % 8 == 0 && 2 * VC * 8 <= 512;
}
__device__ __forceinline__ void tmem_st8(u32 taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_st1(u32 taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(u32 taddr, u32* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
}
// the loaded registers may only be read after the wait: they pass through it
__device__ __forceinline__ void tmem_wait_ld16(u32* a, u32* b) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                   "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld8(u32* a) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#ifdef RMFHT_STATS
// diagnostic counters (tools/stats_run.py builds a separate library with them)
__device__ unsigned long long g_stats[256];
#define RMFHT_STAT(i) do { if (lane_id() == 0) atomicAdd(&g_stats[(i)], 1ull); } while (0)
#define RMFHT_STAT_ADD(i, v) do { if (lane_id() == 0) atomicAdd(&g_stats[(i)], (unsigned long long)(v)); } while (0)
#else
#define RMFHT_STAT(i) do { } while (0)
#define RMFHT_STAT_ADD(i, v) do { } while (0)
#endif

// Where an FHT node's transform values live after the butterflies.
// Default: element (bin) e = k * LPP + u sits in register slot k of lane u.
// TR ("transposed lane stages", 8 lanes per path, V >= 8): the register
// stages run in the default layout, the vector is then transposed through
// the spill rows so that the last three stages (the lane bits of e) are
// register stages too — no shuffles.  Afterwards lane u holds, in slot
// k = j * G + g, element e = (u * G + g) * 8 + j (G = V / 8), so each
// transposed LDS.128 / LDS.64 fills consecutive slots (register pairs for
// the packed butterflies).
template <int R, int MM, int L, int SS>
struct FhtLayout {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    static constexpr int V = LV::V;
    static constexpr bool TSHAPE = C::LPP == 8 && WS2<R, MM, L>::VMAX == 32;
    static constexpr bool TR = TSHAPE && LV::full && V >= 8;
    static constexpr int G = TR ? V / 8 : 1;
    __device__ __forceinline__ static int bin(int k, int u) {
        if constexpr (TR) return ((u * G + k % G) << 3) | (k / G);
        else return LV::full ? k * C::LPP + u : u;
    }
    __device__ __forceinline__ static int owner(int b) {  // lane of the group holding bin b
        if constexpr (TR) return (b >> 3) / G;
        else return LV::full ? b % C::LPP : b;
    }
    __device__ __forceinline__ static int slot(int b) {
        if constexpr (TR) return (b & 7) * G + (b >> 3) % G;
        else return LV::full ? b / C::LPP : 0;
    }
    // chunk twist of the spill rows (XOR-ed into the lane swizzle) so that the
    // transposed reads are conflict-free: LDS.128 (V = 32) phases are one
    // path, LDS.64 (V = 16) phases two paths, LDS.32 (V = 8) all four
    __device__ __forceinline__ static int twist(int p) {
        if constexpr (TSHAPE && V == 16) return 4 * (p & 1);
        else if constexpr (TSHAPE && V == 8) return 2 * p;
        else return 0;
    }
};

// Rare path of fht_node (more candidates than kCap): exact K-round selection
// per path, then the pool — as the reference-order kernel does it.
template <int R, int MM, int L, int SS>
__device__ __noinline__ void fht_fallback(WS2<R, MM, L>* wsp_, int lane, float llrabs) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    using FL = FhtLayout<R, MM, L, SS>;
    constexpr int n = LV::n, V = LV::V, K = cmin(L, n);
    auto& ws = *wsp_;
    const int p = lane / C::LPP, u = lane % C::LPP;
    const int tw = FL::twist(p);
    const bool act = LV::full || u < n;
        // rare: exact K-round selection per path, then the pool (as rmfht_kernels.cuh)
        {
            const float la = __shfl_sync(kFull, llrabs, (lane % L) * C::LPP);
            if (lane < L) ws.llrabs[lane] = la;
        }
        u64 taken = 0ull;
#pragma unroll 1
        for (int rr = 0; rr < K; rr++) {
            float bv = -1.f, bw = 0.f;
            int bb = 0x7fffffff;
#pragma unroll
            for (int k = 0; k < V; k++) {
                const int e = FL::bin(k, u);
                const float wk = ws.wspk(lane, k, tw);
                const float a = fabsf(wk);
                if (act && !((taken >> k) & 1ull) && (a > bv || (a == bv && e < bb))) { bv = a; bb = e; bw = wk; }
            }
#pragma unroll
            for (int off = 1; off < LV::act; off <<= 1) {
                const float ov = __shfl_xor_sync(kFull, bv, off), ow = __shfl_xor_sync(kFull, bw, off);
                const int ob = __shfl_xor_sync(kFull, bb, off);
                if (ov > bv || (ov == bv && ob < bb)) { bv = ov; bb = ob; bw = ow; }
            }
            if (act && FL::owner(bb) == u) taken |= 1ull << FL::slot(bb);
            if (u == 0) {
                ws.cb[p * K + rr] = bb;
                ws.cw[p * K + rr] = bw;
                ws.cp[p * K + rr] = p;
            }
        }
        __syncwarp();
        constexpr int PK = L * K;
        for (int c = lane; c < PK; c += 32) ws.cpm[c] = ws.pm[c / K] + 0.5f * (ws.llrabs[c / K] - fabsf(ws.cw[c]));
        __syncwarp();
#pragma unroll 1
        for (int c = lane; c < PK; c += 32) {
            const float pc = ws.cpm[c];
            const int sc = c / K, bc = ws.cb[c];
            int rank = 0;
#pragma unroll 1
            for (int d = 0; d < PK; d++) {
                const float pd = ws.cpm[d];
                const int sd = d / K;
                rank += (pd < pc) || (pd == pc && (sd < sc || (sd == sc && ws.cb[d] < bc)));
            }
            if (rank < L) {
                ws.sel_src[rank] = sc;
                ws.sel_bin[rank] = bc;
                ws.sel_w[rank] = ws.cw[c];
                ws.sel_pm[rank] = pc;
            }
        }
        __syncwarp();
    }

// Exact list path of fht_node (cold: a same-path pm collision among the
// pool's top L, or more than kCap candidates): per-path top-K by (|w| desc,
// bin asc) (fht_decode.py:116), then the pool ranked by the 64-bit key
// (pm, source path, bin) (:120).  Out of line so the hot node code stays
// compact in the instruction cache.
template <int R, int MM, int L, int SS>
__device__ __noinline__ void fht_exact(WS2<R, MM, L>* wsp_, int lane, u64 mask64, int cnt, int total, float pmp,
                                       float llrabs) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    using FL = FhtLayout<R, MM, L, SS>;
    constexpr int n = LV::n, V = LV::V, K = cmin(L, n);
    using MaskT = typename std::conditional<(V > 32), u64, u32>::type;
    auto& ws = *wsp_;
    const int p = lane / C::LPP, u = lane % C::LPP;
    const int tw = FL::twist(p);
    const MaskT mask = (MaskT)mask64;
    (void)n;
    // candidates per path (for the per-path top-K rule, fht_decode.py:116) and
    // each lane's position in the warp list (inclusive prefix sum)
    int pcnt = cnt;
#pragma unroll
    for (int off = 1; off < LV::act; off <<= 1) pcnt += __shfl_xor_sync(kFull, pcnt, off);
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += t;
    }
    if (total <= kCap) {
        const bool over = __any_sync(kFull, pcnt > K);
        RMFHT_STAT(SS * 8 + 2);
        if (over) RMFHT_STAT(SS * 8 + 5);
        int pos = incl - cnt;
        // this path's candidates occupy [pstart, pstart + pcnt) (lane order)
        const int pstart = __shfl_sync(kFull, incl - cnt, p * C::LPP);
        if (u == 0) {
            ws.cp[p] = (int16_t)pstart;
            ws.celig[p] = (int16_t)pcnt;
        }
        MaskT mk = mask;
        while (mk) {
            const int k = sizeof(MaskT) == 8 ? __ffsll((long long)mk) - 1 : __ffs((int)mk) - 1;
            mk &= mk - 1;
            const float v = ws.wspk(lane, k, tw);
            const float a = fabsf(v);
            const int bin = FL::bin(k, u);
            const float pmc = pmp + 0.5f * (llrabs - a);  // :119
            u32 kb = __float_as_uint(pmc);
            kb ^= (kb >> 31) ? 0xffffffffu : 0x80000000u;  // order-preserving for any sign
            ws.ckey[pos] = ((u64)kb << 32) | ((u32)p << 16) | (u32)bin;
            ws.cw[pos] = v;
            pos++;
        }
        if (lane < 4 && total + lane < ((total + 3) & ~3)) ws.ckey[total + lane] = ~0ull;  // pad to 4
        __syncwarp();
        if (over) {
            // a path with more than K candidates: keep only its top-K by
            // (|w| desc, bin asc); the rest leave the pool
            bool kill[2] = {false, false};
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int i = lane + 32 * h;
                if (i < total) {
                    const u64 ki = ws.ckey[i];
                    const int pi = (int)((ki >> 16) & 0xffff), bi = (int)(ki & 0xffff);
                    const int j0 = ws.cp[pi], j1 = j0 + ws.celig[pi];
                    if (j1 - j0 > K) {
                        const float ai = fabsf(ws.cw[i]);
                        int rp = 0;
#pragma unroll 1
                        for (int j = j0; j < j1; j++) {
                            const float aj = fabsf(ws.cw[j]);
                            rp += aj > ai || (aj == ai && (int)(ws.ckey[j] & 0xffff) < bi);
                        }
                        kill[h] = rp >= K;
                    }
                }
            }
            __syncwarp();
            if (kill[0]) ws.ckey[lane] = ~0ull;
            if (kill[1]) ws.ckey[lane + 32] = ~0ull;
            __syncwarp();
        }
        // pool: rank by (pm, source path, bin) (:120)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int i = lane + 32 * h;
            if (h == 1 && total <= 32) break;
            const u64 ki = i < total ? ws.ckey[i] : ~0ull;
            if (ki != ~0ull) {
                int rank = 0;
                const int tot4 = (total + 3) & ~3;
#pragma unroll 1
                for (int j = 0; j < tot4; j += 4) {
                    const ulonglong2 k01 = *reinterpret_cast<const ulonglong2*>(&ws.ckey[j]);
                    const ulonglong2 k23 = *reinterpret_cast<const ulonglong2*>(&ws.ckey[j + 2]);
                    rank += (k01.x < ki) + (k01.y < ki) + (k23.x < ki) + (k23.y < ki);
                }
                if (rank < L) {
                    u32 kb = (u32)(ki >> 32);
                    kb ^= (kb >> 31) ? 0x80000000u : 0xffffffffu;
                    ws.sel_src[rank] = (int)((ki >> 16) & 0xffff);
                    ws.sel_bin[rank] = (int)(ki & 0xffff);
                    ws.sel_w[rank] = ws.cw[i];
                    ws.sel_pm[rank] = __uint_as_float(kb);
                }
            }
        }
        __syncwarp();
    } else {
        RMFHT_STAT(SS * 8 + 3);
        fht_fallback<R, MM, L, SS>(&ws, lane, llrabs);
    }
}

// ------------------------------------------- FHT node (RR == 1) ---------
// fhtl (fht_decode.py:101-126) on all L paths (P == L invariant of
// p-FHT-FSCL).  x[] is this lane's part of its path's node vector.
// Writes the survivors (pool order) into ws.sel_*; returns packed bits of
// this lane group's survivor codeword; lineage into lin[].
template <int R, int MM, int L, int SS>
__device__ __forceinline__ u64 fht_node(Ctx2<R, MM, L>& cx, float (&x)[Lv<SS, 32 / L>::V], int8_t* lin) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    constexpr int n = LV::n, V = LV::V, K = cmin(L, n);
    auto& ws = cx.ws;
    const int lane = cx.lane, p = cx.p, u = cx.u;
    const bool act = LV::full || u < n;
    // llr_abs (:114): lane partial in slot order, then the group tree
    float part = act ? fabsf(x[0]) : 0.f;
#pragma unroll
    for (int k = 1; k < V; k++) part += fabsf(x[k]);
    const float llrabs = group_sum_tree<C::LPP, LV::act>(part);
    // butterflies (:28-48): register bits (high) first, then lane bits
    using FL = FhtLayout<R, MM, L, SS>;
    const int tw = FL::twist(p);
    float w[V];
#pragma unroll
    for (int k = 0; k < V; k++) w[k] = act ? x[k] : 0.f;
    // stages on register-slot bit hr (lo = slot k, hi = slot k + hr)
    auto reg_stage = [&](const int hr) {
        if (hr >= 2) {
            // two butterflies per instruction: (k, k+1) against (k+hr, k+hr+1)
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
    constexpr int LOGV = clog2(V);
#pragma unroll
    for (int st = 0; st < LOGV; st++) reg_stage(V >> (st + 1));
    if constexpr (FL::TR) {
        // transpose through the spill rows: lane u of path p gathers, for
        // every j < 8, slots u*G .. u*G+G-1 of row p*8 + j (element
        // (u*G + g)*8 + j) into slot j*G + g; then the lane-bit stages
        // (half = 4, 2, 1 on e) are register stages on slot bits 4G, 2G, G
        constexpr int G = FL::G;
#pragma unroll
        for (int k = 0; k < V; k += 4)
            *reinterpret_cast<float4*>(&ws.wspk(lane, k, tw)) = make_float4(w[k], w[k + 1], w[k + 2], w[k + 3]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int row = p * 8 + j;
            const float* src = &ws.wspk(row, u * G, tw);
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
        __syncwarp();  // every row read before the transform is spilled again
        reg_stage(4 * G);
        reg_stage(2 * G);
        reg_stage(G);
    } else {
    constexpr int LOGA = clog2(LV::act);
#pragma unroll
    for (int st = 0; st < LOGA; st++) {
        const int half = LV::act >> (st + 1);
        const float sg = (u & half) ? 1.f : -1.f;
        if constexpr (V >= 2) {
            const u64 sg2 = pk(sg, sg);
#pragma unroll
            for (int k = 0; k < V; k += 2) {
                const float o0 = __shfl_xor_sync(kFull, w[k], half), o1 = __shfl_xor_sync(kFull, w[k + 1], half);
                // hi lane: w + o = hi + lo; lo lane: o - w = hi - lo
                const u64 r = fma2(sg2, pk(w[k], w[k + 1]), pk(o0, o1));
                w[k] = plo(r);
                w[k + 1] = phi(r);
            }
        } else {
            const float o = __shfl_xor_sync(kFull, w[0], half);
            w[0] = __fmaf_rn(sg, w[0], o);
        }
    }
    }
    // path maximum and the pool threshold tau = L-th smallest path-best pm
    // (a warp-wide maximum: one REDUX on order-preserving integer keys; cbest
    // can be a rounding error below zero, llrabs and M1 being summed in
    // different orders)
    // (maxima and masks as trees, not V-long dependency chains)
    float mx;
    {
        float t[V];
#pragma unroll
        for (int k = 0; k < V; k++) t[k] = fabsf(w[k]);
#pragma unroll
        for (int sd = 1; sd < V; sd <<= 1)
#pragma unroll
            for (int k = 0; k + sd < V; k += 2 * sd) t[k] = fmaxf(t[k], t[k + sd]);
        mx = act ? t[0] : -1.f;
    }
    constexpr u32 GBITS = (LV::act >= 32) ? 0xffffffffu : ((1u << LV::act) - 1u);  // active lanes of a group
    const float M1 = group_max<LV::act>(mx);
    const float pmp = ws.pm[p];
    const float cbest = pmp + 0.5f * (llrabs - M1);
    const float tau = key_float(__reduce_max_sync(kFull, float_key(cbest)));
    // |w| >= theta is implied by pm(|w|) <= tau (with slack for rounding)
    const float th0 = llrabs - 2.f * (tau - pmp);
    const float theta = th0 - (fabsf(th0) + llrabs + fabsf(tau) + fabsf(pmp)) * 9.5367431640625e-07f - 1e-30f;
    using MaskT = typename std::conditional<(V > 32), u64, u32>::type;
    MaskT mask;
    // LAZY: the spill of the transform (for candidate extraction) is only
    // needed off the common case; there the lane's single candidate value
    // (wsel, its last candidate) comes from the mask pass
    constexpr bool LAZY = sizeof(MaskT) == 4;
    float wsel = 0.f;
    if constexpr (sizeof(MaskT) == 4) {
        // one compare and one predicated OR (and move) per element
        u32 m0 = 0u, m1 = 0u;
#pragma unroll
        for (int k = 0; k < V; k++) {
            if (fabsf(w[k]) >= theta) {
                if (k & 1) m1 |= 1u << k;
                else m0 |= 1u << k;
                wsel = w[k];
            }
        }
        mask = act ? (m0 | m1) : 0u;
    } else {
        MaskT t[V];
#pragma unroll
        for (int k = 0; k < V; k++) t[k] = fabsf(w[k]) >= theta ? ((MaskT)1 << k) : (MaskT)0;
#pragma unroll
        for (int sd = 1; sd < V; sd <<= 1)
#pragma unroll
            for (int k = 0; k + sd < V; k += 2 * sd) t[k] |= t[k + sd];
        mask = act ? t[0] : (MaskT)0;
    }
    const int cnt = sizeof(MaskT) == 8 ? __popcll((u64)mask) : __popc((u32)mask);
    const int total = __reduce_add_sync(kFull, cnt);
    // spill the transform for candidate extraction (conflict-free STS.128)
    auto spill = [&] {
        if constexpr (V >= 4) {
#pragma unroll
            for (int k = 0; k < V; k += 4)
                *reinterpret_cast<float4*>(&ws.wspk(lane, k, tw)) = make_float4(w[k], w[k + 1], w[k + 2], w[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < V; k++) ws.wspk(lane, k, tw) = w[k];
        }
        __syncwarp();
    };
    if constexpr (!LAZY) spill();
    RMFHT_STAT(SS * 8 + 0);
#ifdef RMFHT_STATS
    cx.ngen++;
#endif
    RMFHT_STAT_ADD(SS * 8 + 4, total);
    // common case: L candidates in all and every path has one (its maximum is
    // always a candidate), i.e. every path's only candidate is its maximum
    const u32 bal = __ballot_sync(kFull, cnt > 0);
    if (total == L && __all_sync(kFull, ((bal >> (p * C::LPP)) & GBITS) != 0u)) {
        RMFHT_STAT(SS * 8 + 1);
#ifdef RMFHT_STATS
        cx.ngen--;  // (counted below for every node, undone here)
#endif
        // the pool is the L path maxima ordered by (pm, source slot) (:116-120)
        int rank = 0;
        if constexpr (C::LPP >= L) {
            // lane u < L of every group compares its path with path u: one
            // shuffle and one ballot give each path its rank
            const float cq = __shfl_sync(kFull, cbest, (u < L ? u : 0) * C::LPP);
            const bool before = u < L && ((cq < cbest) || (cq == cbest && u < p));
            rank = __popc((__ballot_sync(kFull, before) >> (p * C::LPP)) & ((1u << L) - 1u));
        } else {
            // fewer lanes per path than paths: L / LPP passes, lane u of every
            // group comparing its path with path u + t LPP
            static_assert(L % C::LPP == 0, "paths per pass");
#pragma unroll
            for (int t = 0; t < L / C::LPP; t++) {
                const int q = u + t * C::LPP;
                const float cq = __shfl_sync(kFull, cbest, q * C::LPP);
                const bool before = (cq < cbest) || (cq == cbest && q < p);
                rank += __popc((__ballot_sync(kFull, before) >> (p * C::LPP)) & ((1u << C::LPP) - 1u));
            }
        }
        // the one lane of each path holding a candidate (its maximum) records it
        if (cnt > 0) {
            const int k = (sizeof(MaskT) == 8 ? __ffsll((long long)mask) : __ffs((int)mask)) - 1;
            ws.sel_src[rank] = p;
            ws.sel_bin[rank] = FL::bin(k, u);
            ws.sel_w[rank] = LAZY ? wsel : ws.wspk(lane, k, tw);
            ws.sel_pm[rank] = cbest;
        }
        __syncwarp();
    } else {
#ifdef RMFHT_STATS
    if (__all_sync(kFull, cnt <= 1)) RMFHT_STAT(100 + SS);  // no lane holds two candidates
    if (__all_sync(kFull, cnt <= 2)) RMFHT_STAT(110 + SS);
#endif
    if constexpr (LAZY) spill();
    // General case, more than 32 candidates: L rounds of warp-wide minimum
    // selection over the pool key (pm, source path, bin) (:120), each lane
    // offering its best remaining candidate.  The per-path top-K cut (:116, K = L here) can only exclude
    // a pool top-L candidate X when a candidate Z of the same path has the
    // same pm but a larger |w| and a larger bin (a pm rounding collision);
    // every pick therefore checks that no other remaining candidate of its
    // path has its exact pm, and a collision hands the node to the exact
    // list path below.
    bool exact_needed = true;
    if (K == L && total <= 32) {
        // At most 32 candidates: list them (warp prefix sum of the counts),
        // one per lane, and rank each by its 64-bit pool key (pm, source
        // path, bin) (:120) against the whole list.  The per-path top-K cut
        // (:116, K = L) can only remove a pool top-L candidate through a
        // same-path pm collision at the L-th pick's pm (see the greedy
        // selection below): checked after the ranks.
        int pos;
        if (__all_sync(kFull, cnt <= 1)) {
            // at most one candidate per lane: positions from one ballot
            pos = __popc(__ballot_sync(kFull, cnt > 0) & ((1u << lane) - 1u));
        } else {
            int incl = cnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += t;
            }
            pos = incl - cnt;
        }
        MaskT mk = mask;
        while (mk) {
            const int k = (sizeof(MaskT) == 8 ? __ffsll((long long)mk) : __ffs((int)mk)) - 1;
            mk &= mk - 1;
            const float pmc = pmp + 0.5f * (llrabs - fabsf(ws.wspk(lane, k, tw)));  // :119
            ws.ckey[pos++] = ((u64)float_key(pmc) << 32) | ((u32)p << 16) | (u32)FL::bin(k, u);
        }
        if (lane < 4 && total + lane < ((total + 3) & ~3)) ws.ckey[total + lane] = ~0ull;  // pad to 4
        __syncwarp();
        const bool mine = lane < total;
        const u64 ki = mine ? ws.ckey[lane] : ~0ull;
        int rank = 0;
        const int tot4 = (total + 3) & ~3;
#pragma unroll 1
        for (int j = 0; j < tot4; j += 4) {
            const ulonglong2 k01 = *reinterpret_cast<const ulonglong2*>(&ws.ckey[j]);
            const ulonglong2 k23 = *reinterpret_cast<const ulonglong2*>(&ws.ckey[j + 2]);
            rank += (k01.x < ki) + (k01.y < ki) + (k23.x < ki) + (k23.y < ki);
        }
        const u32 hk = (u32)(ki >> 32);
        const int src = (int)((ki >> 16) & 0xffffu), bin = (int)(ki & 0xffffu);
        const bool sel = mine && rank < L;
        if (sel) {
            ws.sel_src[rank] = src;
            ws.sel_bin[rank] = bin;
            ws.sel_w[rank] = ws.wspk(src * C::LPP + FL::owner(bin), FL::slot(bin), FL::twist(src));
            ws.sel_pm[rank] = key_float(hk);
        }
        const int lastl = __ffs(__ballot_sync(kFull, mine && rank == L - 1)) - 1;
        const u32 hlast = __shfl_sync(kFull, hk, lastl);
        const u32 lastp = __reduce_or_sync(kFull, sel && hk == hlast ? 1u << src : 0u);
        exact_needed = __any_sync(kFull, mine && rank >= L && hk == hlast && ((lastp >> src) & 1u));
        __syncwarp();
    } else if constexpr (K == L) {
        const u32 pkey = (u32)p << 16;
        auto lane_best = [&](MaskT m, u32& hi, u32& lo) {
            hi = 0xffffffffu;
            lo = 0xffffffffu;
            while (m) {
                const int k = (sizeof(MaskT) == 8 ? __ffsll((long long)m) : __ffs((int)m)) - 1;
                m &= m - 1;
                const float pmc = pmp + 0.5f * (llrabs - fabsf(ws.wspk(lane, k, tw)));  // :119
                const u32 h = float_key(pmc), l = pkey | (u32)FL::bin(k, u);
                if (h < hi || (h == hi && l < lo)) { hi = h; lo = l; }
            }
        };
        MaskT rem = mask;
        u32 hi, lo;
        lane_best(rem, hi, lo);
        // picks come in ascending pm order, so a same-path pm collision that
        // matters (a remaining candidate with the pm of a pick) can only be at
        // the last pick's pm: each lane remembers the key of its own latest
        // pick, and the paths picked at the last pm are one ballot after the
        // rounds
        u32 hlast = 0xffffffffu, mine = 0xffffffffu;
#pragma unroll 1
        for (int r = 0; r < L; r++) {
            const u32 hmin = __reduce_min_sync(kFull, hi);
            const u32 eq = __ballot_sync(kFull, hi == hmin);
            int wl = __ffs(eq) - 1;
            if (eq & (eq - 1)) {  // several lanes at this pm: the lowest (path, bin)
                const u32 lmin = __reduce_min_sync(kFull, hi == hmin ? lo : 0xffffffffu);
                wl = __ffs(__ballot_sync(kFull, hi == hmin && lo == lmin)) - 1;
            }
            hlast = hmin;
            if (lane == wl) {
                const int bin = (int)(lo & 0xffffu);
                const int k = FL::slot(bin);
                ws.sel_src[r] = p;
                ws.sel_bin[r] = bin;
                ws.sel_w[r] = ws.wspk(lane, k, tw);
                ws.sel_pm[r] = key_float(hmin);
                mine = hmin;
                rem &= ~((MaskT)1 << k);
                lane_best(rem, hi, lo);
            }
        }
        const u32 lastb = __ballot_sync(kFull, mine == hlast);  // lanes that picked at the last pm
        const bool path_last = ((lastb >> (p * C::LPP)) & GBITS) != 0u;
        exact_needed = __any_sync(kFull, hi == hlast && path_last);
        __syncwarp();
        RMFHT_STAT(SS * 8 + 6);
        if (exact_needed) RMFHT_STAT(SS * 8 + 7);
    }
    if (exact_needed) fht_exact<R, MM, L, SS>(&cx.ws, lane, (u64)mask, cnt, total, pmp, llrabs);
    }
    // survivors: pm, lineage; my group's codeword bits
    if (lane < L) {
        ws.pm[lane] = ws.sel_pm[lane];
        lin[lane] = (int8_t)ws.sel_src[lane];
    }
    const int b = ws.sel_bin[p];
    const int sgn = ws.sel_w[p] < 0.f;
    __syncwarp();
    // bit k of the packed word = codeword bit of element e = k*LPP+u
    // (_bin_codewords, fht_decode.py:58-62): parity(~b & ~e & (n-1)) ^ sign
    //   = c0 ^ parity(Bh & k),  B = ~b & (n-1), Bh = B >> log2(LPP),
    //   c0 = sign ^ parity(B) ^ parity(B & u & (LPP-1))
    u64 bits;
    if constexpr (LV::full) {
        const u32 B = (u32)(~b) & (u32)(n - 1);
        const u32 Bh = B >> C::LB;
        const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)u & (u32)(C::LPP - 1)) & 1);
        if constexpr (V <= 32) {  // 32-bit patterns
            constexpr u32 VM = V >= 32 ? ~0u : ((1u << V) - 1u);
            u32 P = 0;
            if (Bh & 1u) P ^= 0xAAAAAAAAu;
            if (Bh & 2u) P ^= 0xCCCCCCCCu;
            if (Bh & 4u) P ^= 0xF0F0F0F0u;
            if (Bh & 8u) P ^= 0xFF00FF00u;
            if (Bh & 16u) P ^= 0xFFFF0000u;
            bits = (u64)((c0 ? ~P : P) & VM);
        } else {
            constexpr u64 VM = V >= 64 ? ~0ull : ((1ull << V) - 1ull);
            u64 P = 0;
            if (Bh & 1u) P ^= 0xAAAAAAAAAAAAAAAAull;
            if (Bh & 2u) P ^= 0xCCCCCCCCCCCCCCCCull;
            if (Bh & 4u) P ^= 0xF0F0F0F0F0F0F0F0ull;
            if (Bh & 8u) P ^= 0xFF00FF00FF00FF00ull;
            if (Bh & 16u) P ^= 0xFFFF0000FFFF0000ull;
            if (Bh & 32u) P ^= 0xFFFFFFFF00000000ull;
            bits = (c0 ? ~P : P) & VM;
        }
    } else {
        bits = (u64)((__popc((unsigned)(~(b | u)) & (unsigned)(n - 1)) & 1) ^ sgn);
    }
    return act ? bits : 0ull;
}

// spc_decode_list (list_engine.py:68-119) for nodes with one element per
// lane (n <= lanes per path): list state in lanes (slot i in lane i), ranks
// by shuffles, signs by ballot.
template <int R, int MM, int L, int SS>
__device__ __forceinline__ u64 spc_node_v1(Ctx2<R, MM, L>& cx, float xv, int8_t* lin) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    constexpr int n = LV::n;
    constexpr int TAU = cmin(cmin(L, n), n - 1);
    static_assert(LV::V == 1 && n <= 32, "one element per lane");
    auto& ws = cx.ws;
    const int lane = cx.lane, p = cx.p, u = cx.u;
    const bool act = u < n;
    const float mag = act ? fabsf(xv) : 0.f;
    const u32 sbal = __ballot_sync(kFull, act && xv < 0.f);  // hard decisions (:84)
    constexpr u32 AM = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
    // stable ascending rank of |alpha| inside the path (:83)
    int rank = 0;
#pragma unroll
    for (int v = 1; v < n; v++) {
        const int w = (u + v) % n;
        const float mw = __shfl_sync(kFull, mag, p * C::LPP + w);
        rank += (mw < mag) || (mw == mag && w < u);
    }
    if (act && rank <= TAU) ws.smag[p * 16 + rank] = mag;
    __syncwarp();
    // slot state (lane i < L holds slot i): metric, running parity, parent path, flips
    float spm = 0.f, spar = 0.f;
    int sparent = 0, sfl = 0;
    if (lane < L) {
        const int par0 = __popc((sbal >> (lane * C::LPP)) & AM) & 1;
        spm = ws.pm[lane] + (par0 ? ws.smag[lane * 16] : 0.f);  // :88
        spar = (float)par0;
        sparent = lane;
    }
#pragma unroll 1
    for (int j = 1; j <= TAU; j++) {  // :97-112
        const int i = lane >> 1;
        const float ipm = __shfl_sync(kFull, spm, i);
        const float ipar = __shfl_sync(kFull, spar, i);
        const int ipa = __shfl_sync(kFull, sparent, i);
        const int ifl = __shfl_sync(kFull, sfl, i);
        float cand = 3.4e38f;
        if (lane < 2 * L) {
            if (lane & 1) {
                const float t = ipm + ws.smag[ipa * 16 + j];
                const float am = ws.smag[ipa * 16];
                cand = ipar != 0.f ? t - am : t + am;  // pms + a_j + (1 - 2 par) a_m
            } else {
                cand = ipm;
            }
        }
        int r2 = 0;
        if constexpr (2 * L == 8) {
            // the four quarter warps rank a copy of each candidate against two candidates each
            const int ci = lane & 7, q2 = (lane >> 3) * 2;
            const float mine = __shfl_sync(kFull, cand, ci);
            const float c0 = __shfl_sync(kFull, cand, q2), c1 = __shfl_sync(kFull, cand, q2 + 1);
            r2 = ((c0 < mine) || (c0 == mine && q2 < ci)) + ((c1 < mine) || (c1 == mine && q2 + 1 < ci));
            r2 += __shfl_xor_sync(kFull, r2, 8);
            r2 += __shfl_xor_sync(kFull, r2, 16);
        } else {
#pragma unroll
            for (int c = 0; c < 2 * L; c++) {
                const float cc = __shfl_sync(kFull, cand, c);
                r2 += (cc < cand) || (cc == cand && c < lane);
            }
        }
        // no flip survives and the keeps are already in slot order: the state
        // is unchanged, and since the later positions are at least as
        // unreliable (a_{j+1} >= a_j), every later split keeps it too
        if (__all_sync(kFull, lane >= 2 * L || ((lane & 1) ? r2 >= L : r2 == (lane >> 1)))) break;
        if (lane < 2 * L && r2 < L) {
            const int flip = lane & 1;
            ws.cpm[r2] = cand;
            ws.cw[r2] = flip ? 1.f - ipar : ipar;
            ws.cb[r2] = ipa;
            ws.cp[r2] = ifl | (flip << j);
        }
        __syncwarp();
        if (lane < L) {
            spm = ws.cpm[lane];
            spar = ws.cw[lane];
            sparent = ws.cb[lane];
            sfl = ws.cp[lane];
        }
        __syncwarp();
    }
    // beta = sign xor flips; the least reliable bit makes the parity even (:114-118)
    const int parent = __shfl_sync(kFull, sparent, p);
    const int fl = __shfl_sync(kFull, sfl, p);
    const u32 psg = (sbal >> (parent * C::LPP)) & AM;
    int b = (int)((psg >> u) & 1u);
    // split j flipped the parent's element of rank j (fl bit j): look up this
    // element's rank in the parent path
    const int pr = __shfl_sync(kFull, rank, parent * C::LPP + u);
    b ^= (fl >> pr) & 1;
    const int tot = (__popc(psg) + __popc(fl)) & 1;
    if (pr == 0) b ^= tot;
    if (lane < L) {
        ws.pm[lane] = spm;
        lin[lane] = (int8_t)sparent;
    }
    __syncwarp();
    return act ? (u64)b : 0ull;
}

// ---------------------------------------------------- SPC node ----------
// spc_decode_list (list_engine.py:68-119) on L paths of size n = 2^SS.
template <int R, int MM, int L, int SS>
__device__ __forceinline__ u64 spc_node(Ctx2<R, MM, L>& cx, float (&x)[Lv<SS, 32 / L>::V], int8_t* lin) {
    if constexpr (Lv<SS, 32 / L>::V == 1 && (1 << SS) <= 16) return spc_node_v1<R, MM, L, SS>(cx, x[0], lin);
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    constexpr int n = LV::n, V = LV::V;
    constexpr int TAU = cmin(cmin(L, n), n - 1);
    auto& ws = cx.ws;
    const int lane = cx.lane, p = cx.p, u = cx.u;
    const bool act = LV::full || u < n;
    // magnitudes and signs to shared memory, parity by ballot
    int par = 0;
#pragma unroll
    for (int k = 0; k < V; k++) {
        const int e = LV::full ? k * C::LPP + u : u;
        if (act) ws.smag[p * n + e] = fabsf(x[k]);
        const u32 bal = __ballot_sync(kFull, act && x[k] < 0.f);
        par ^= __popc(bal & (((1u << (LV::act - 1)) << 1) - 1u) << (p * C::LPP)) & 1;
    }
    __syncwarp();
    // rank of each element in the stable ascending |alpha| order (:83); the
    // TAU+1 least reliable positions go to sord
    // (full nodes of up to 16 elements: the path's magnitudes come in once as
    // float4, and the index tie-break j < e is static except inside the
    // element's own slot block — one compare per pair instead of three)
    constexpr bool FASTRANK = LV::full && n <= 16 && n % 4 == 0;
    float mg[FASTRANK ? n : 1];
    if constexpr (FASTRANK) {
#pragma unroll
        for (int j = 0; j < n; j += 4) {
            const float4 v = *reinterpret_cast<const float4*>(&ws.smag[p * n + j]);
            mg[j] = v.x; mg[j + 1] = v.y; mg[j + 2] = v.z; mg[j + 3] = v.w;
        }
    }
#pragma unroll
    for (int k = 0; k < V; k++) {
        const int e = LV::full ? k * C::LPP + u : u;
        if (act) {
            int rank = 0;
            if constexpr (FASTRANK) {
                const float me = fabsf(x[k]);
#pragma unroll
                for (int j = 0; j < n; j++) {
                    const int jb = j / C::LPP, ju = j % C::LPP;
                    if (jb < k) rank += mg[j] <= me;
                    else if (jb > k) rank += mg[j] < me;
                    else rank += (mg[j] < me) || (mg[j] == me && ju < u);
                }
            } else {
            const float me = ws.smag[p * n + e];
            for (int j = 0; j < n; j++) {
                const float mj = ws.smag[p * n + j];
                rank += (mj < me) || (mj == me && j < e);
            }
            }
            if (rank <= TAU) ws.sord[p * 16 + rank] = (uint16_t)e;
            // sign bit and the rank (capped at TAU + 1: only ranks 0..TAU are
            // ever flipped or fixed) for the output bits
            ws.ssgn[p * n + e] = (uint8_t)((x[k] < 0.f) | ((rank <= TAU ? rank : TAU + 1) << 1));
        }
    }
    __syncwarp();
    // the TAU splits (:97-112): one lane per candidate
    // path parity for each path (lane group uniform) -> smem
    if (u == 0) ws.sel_bin[p] = par;
    __syncwarp();
    if (lane < L) {
        const int pp = lane;
        const float amin = ws.smag[pp * n + ws.sord[pp * 16]];
        ws.pm[pp] = ws.pm[pp] + (ws.sel_bin[pp] ? amin : 0.f);  // :88
        ws.sel_w[pp] = (float)ws.sel_bin[pp];                   // running parity
        ws.sel_src[pp] = pp;                                     // parent path
        ws.cb[pp] = 0;                                           // flip mask over j
    }
    __syncwarp();
#pragma unroll 1
    for (int j = 1; j <= TAU; j++) {
        // candidates: 2i = keep, 2i+1 = flip (interleaved, :101-104)
        float cand = 0.f;
        int csrc = 0;
        if (lane < 2 * L) {
            const int i = lane >> 1;
            const int par_i = ws.sel_src[i];
            const float pmi = ws.pm[i];
            if (lane & 1) {
                const float aj = ws.smag[par_i * n + ws.sord[par_i * 16 + j]];
                const float am = ws.smag[par_i * n + ws.sord[par_i * 16]];
                const float t = pmi + aj;
                cand = ws.sel_w[i] != 0.f ? t - am : t + am;
            } else {
                cand = pmi;
            }
            csrc = i;
        }
        // stable rank among the 2L candidates (:104), by shuffles
        int rank = 0;
        if constexpr (2 * L == 16) {
            // the upper half warp ranks a copy of each candidate against the
            // candidates 8 .. 15 while the lower half takes 0 .. 7
            const int ci = lane & 15, h8 = (lane >> 4) * 8;
            const float mine = __shfl_sync(kFull, cand, ci);
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const float pc = __shfl_sync(kFull, cand, h8 + c);
                rank += (pc < mine) || (pc == mine && h8 + c < ci);
            }
            rank += __shfl_xor_sync(kFull, rank, 16);
        } else {
#pragma unroll
            for (int c = 0; c < 2 * L; c++) {
                const float pc = __shfl_sync(kFull, cand, c);
                rank += (pc < cand) || (pc == cand && c < lane);
            }
        }
        // no flip survives and the keeps are already in slot order: the state
        // is unchanged, and since the later positions are at least as
        // unreliable (a_{j+1} >= a_j: every flip metric can only grow while
        // the keeps stay), every later split keeps it too (as spc_node_v1)
        if (__all_sync(kFull, lane >= 2 * L || ((lane & 1) ? rank >= L : rank == (lane >> 1)))) break;
        // new state (read old state before the sync, write after)
        float npar = 0.f;
        int npa = 0, nfl = 0;
        if (lane < 2 * L && rank < L) {
            const int which = lane & 1;
            npar = which ? 1.f - ws.sel_w[csrc] : ws.sel_w[csrc];
            npa = ws.sel_src[csrc];
            nfl = ws.cb[csrc] | (which << j);
        }
        __syncwarp();
        if (lane < 2 * L && rank < L) {
            ws.pm[rank] = cand;
            ws.sel_w[rank] = npar;
            ws.sel_src[rank] = npa;
            ws.cb[rank] = nfl;
        }
        __syncwarp();
    }
    // beta = sign xor flips, least reliable fixes even parity (:114-118);
    // my group's output path is slot p
    const int parent = ws.sel_src[p];
    const int fl = ws.cb[p];
    // parity of the parent's sign bits (its ballot parity, sel_bin) and of the flips
    const int tot = (ws.sel_bin[parent] ^ __popc(fl)) & 1;
    u64 bits = 0;
#pragma unroll
    for (int k = 0; k < V; k++) {
        const int e = LV::full ? k * C::LPP + u : u;
        // split j flipped the parent's element of rank j (fl bit j); rank 0
        // is the least reliable element, which fixes the parity
        const int sr = act ? ws.ssgn[parent * n + e] : 0;
        const int r = sr >> 1;
        int b = (sr & 1) ^ ((fl >> r) & 1);
        if (r == 0) b ^= tot;
        bits |= (u64)b << k;
    }
    if (lane < L) lin[lane] = (int8_t)ws.sel_src[lane];
    __syncwarp();
    return act ? bits : 0ull;
}


// ------------------------------------------- lane-transposed reduction ----
// Sum T per-lane partials (one per trial) over the 32 lanes with the tree
// offsets 16, 8, 4, 2, 1; every trial gets the same tree.  Lane l ends with
// the total of trial t(l); returns t(l) via *tri.
template <int T>
__device__ __forceinline__ float multi_tree(float (&v)[T], int lane, int* tri) {
    int base = 0;
    int cnt = T;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        if (cnt > 1) {
            const int half = cnt / 2;
            const bool upper = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < T / 2; i++) {
                if (i < half) {
                    const float send = upper ? v[i] : v[i + half];
                    const float keep = upper ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(kFull, send, off);
                }
            }
            if (upper) base += half;
            cnt = half;
        } else {
            v[0] = v[0] + __shfl_xor_sync(kFull, v[0], off);
        }
    }
    *tri = base;
    return v[0];
}

// c != 0 with highest set bit HB: own slots are the static s with bit HB
// clear, ascending (the canonical order); the partner alpha[(l ^ delta) + 32 (s ^ c)]
// comes from the warp's frame copy in shared memory (conflict-free: lane
// l ^ delta), so only HB selects the code, not c
template <int NS, int HB>
__device__ __forceinline__ float lm_hb(const float (&ach)[NS], u32 pc) {
    float acc = 0.f;
    bool first = true;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        if (s >> HB & 1) continue;
        const float partner = lds_addr(pc ^ ((u32)s << 7));
        const float m = fminf(fabsf(ach[s]), fabsf(partner));
        acc = first ? m : acc + m;
        first = false;
    }
    return acc;
}

// LM of trial direction d at the root, canonical channel-domain order
template <int NS>
__device__ __forceinline__ float lm_partial_root(const float (&ach)[NS], u32 d, int lane, u32 alpha_saddr) {
    const int delta = d & 31, c = d >> 5;
    if (c != 0) {
        // partner address with the slot bits of c folded in: (l ^ delta) * 4 + (s ^ c) * 128
        const u32 pc = (alpha_saddr | ((u32)(lane ^ delta) << 2)) ^ ((u32)c << 7);
        const int hb = 31 - __clz(c);
        if (hb < 0 || hb > 3) __builtin_unreachable();
        if constexpr (NS >= 16) {
            if (hb == 3) return lm_hb<NS, 3>(ach, pc);
        }
        if constexpr (NS >= 8) {
            if (hb == 2) return lm_hb<NS, (NS >= 8 ? 2 : 0)>(ach, pc);
        }
        if constexpr (NS >= 4) {
            if (hb == 1) return lm_hb<NS, (NS >= 4 ? 1 : 0)>(ach, pc);
        }
        return lm_hb<NS, 0>(ach, pc);
    }
    // d < 32: pairs inside a slot across lanes l, l ^ d; lanes with bit h clear own them
    const int h = 31 - __clz(delta);
    const bool own = !((lane >> h) & 1);
    float acc = 0.f;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const float partner = __shfl_xor_sync(kFull, ach[s], delta);
        const float m = fminf(fabsf(ach[s]), fabsf(partner));
        acc = (s == 0) ? m : acc + m;
    }
    return own ? acc : 0.f;
}

// top-L of 2L trials by LM descending, lower trial first (automorphism.py:234)
template <int R, int MM, int L>
__device__ __forceinline__ void select_trials2(Ctx2<R, MM, L>& cx) {
    auto& ws = cx.ws;
    const int lane = cx.lane;
    if constexpr (2 * L == 16) {
        // both half warps rank a copy of each trial, against 8 trials each
        // (two LDS.128 per lane instead of 16 scalar loads)
        const int ci = lane & 15, h8 = (lane >> 4) * 8;
        const float v = ws.lm[ci];
        const float4 a = *reinterpret_cast<const float4*>(&ws.lm[h8]), b = *reinterpret_cast<const float4*>(&ws.lm[h8 + 4]);
        const float o[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        int rank = 0;
#pragma unroll
        for (int s = 0; s < 8; s++) rank += (o[s] > v) || (o[s] == v && h8 + s < ci);
        rank += __shfl_xor_sync(kFull, rank, 16);
        if (lane < 16 && rank < L) ws.ord[rank] = (int8_t)lane;
    } else if constexpr (2 * L == 8) {
        // the four quarter warps rank a copy of each trial against two trials each
        const int ci = lane & 7, q2 = (lane >> 3) * 2;
        const float v = ws.lm[ci];
        const float2 o = *reinterpret_cast<const float2*>(&ws.lm[q2]);
        int rank = ((o.x > v) || (o.x == v && q2 < ci)) + ((o.y > v) || (o.y == v && q2 + 1 < ci));
        rank += __shfl_xor_sync(kFull, rank, 8);
        rank += __shfl_xor_sync(kFull, rank, 16);
        if (lane < 8 && rank < L) ws.ord[rank] = (int8_t)lane;
    } else if (lane < 2 * L) {
        const float v = ws.lm[lane];
        int rank = 0;
#pragma unroll
        for (int s = 0; s < 2 * L; s++) rank += (ws.lm[s] > v) || (ws.lm[s] == v && s < lane);
        if (rank < L) ws.ord[rank] = (int8_t)lane;
    }
    __syncwarp();
}

// root permutation extension (automorphism.py:207-237) with the composite
// maps (init then trial); the winners' composites replace ws.comp
template <int R, int MM, int L>
__device__ __forceinline__ void perm_ext_root2(Ctx2<R, MM, L>& cx) {
    using C = Cfg<R, MM, L>;
    auto& ws = cx.ws;
    const int lane = cx.lane, base = ws.next_map;
    // pairing direction of each trial's composite: A_init^-1 (A_t^-1 e_{m-1})
    if (lane < 2 * L) {
        const u32 d = icol_apply<MM>(ws.comp[lane % L], (u32)cx.maps[base + lane].icol[MM - 1]);
        ws.cb[lane] = (int)d;
    }
    __syncwarp();
    float part[2 * L];
    if constexpr (tmem_park<R, MM, L>() && (2 * L) % 8 == 0 && 2 * L <= 2 * Lv<MM - 1, C::LPP>::V) {
        // the trials' lane partials wait in the warp's tensor-memory columns
        // (idle until the root's f) instead of shared memory: the loop over
        // the trials is not unrolled, a column address may be dynamic
#pragma unroll 1
        for (int t = 0; t < 2 * L; t++)
            tmem_st1(cx.tmem + t, lm_partial_root<C::NS>(cx.ach, (u32)ws.cb[t], lane, cx.alpha_saddr));
        tmem_wait_st();
#pragma unroll
        for (int t0 = 0; t0 < 2 * L; t0 += 8) {
            u32 r8[8];
            tmem_ld8(cx.tmem + t0, r8);
            tmem_wait_ld8(r8);
#pragma unroll
            for (int t = 0; t < 8; t++) part[t0 + t] = __uint_as_float(r8[t]);
        }
    } else {
#pragma unroll 1
        for (int t = 0; t < 2 * L; t++)
            ws.lmp[t][lane] = lm_partial_root<C::NS>(cx.ach, (u32)ws.cb[t], lane, cx.alpha_saddr);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2 * L; t++) part[t] = ws.lmp[t][lane];
    }
    int tri;
    const float tot = multi_tree<2 * L>(part, lane, &tri);
    if ((lane & (32 / (2 * L) - 1)) == 0) ws.lm[tri] = tot;
    __syncwarp();
    select_trials2(cx);
    // composites of the winners (inverse direction), one column per lane task
    // (computed into registers, written after every lane has read the old ones)
    constexpr int NT = (L * (MM + 1) + 31) / 32;
    uint16_t nv[NT];
#pragma unroll
    for (int q = 0; q < NT; q++) {
        const int task = lane + 32 * q;
        nv[q] = 0;
        if (task < L * (MM + 1)) {
            const int o = task / (MM + 1), k = task % (MM + 1);
            const int t = ws.ord[o];
            const MapR<MM>& tm = cx.maps[base + t];
            const MapR<MM>& im = ws.comp[t % L];
            // column k of the composite's inverse, or (k == MM) its shift
            const u32 v = icol_apply<MM>(im, (u32)(k < MM ? tm.icol[k] : tm.c));
            nv[q] = (uint16_t)(k < MM ? v : v ^ im.c);
        }
    }
    float npm = 0.f;
    if (lane < L) npm = ws.pm[ws.ord[lane] % L];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < NT; q++) {
        const int task = lane + 32 * q;
        if (task < L * (MM + 1)) {
            const int o = task / (MM + 1), k = task % (MM + 1);
            if (k < MM) ws.comp[o].icol[k] = nv[q];
            else ws.comp[o].c = nv[q];
        }
    }
    if (lane < L) {
        ws.pm[lane] = npm;
        ws.l0[MM][lane] = (int8_t)(ws.ord[lane] % L);
        ws.nmap[MM][lane] = (int16_t)(base + ws.ord[lane]);  // trial map of each root slot
    }
    ws.next_map = base + 2 * L;
    __syncwarp();
}

// inner permutation node: vectors through shared memory
template <int R, int MM, int L, int SS>
__device__ __forceinline__ void perm_ext_inner2(Ctx2<R, MM, L>& cx, float (&x)[Lv<SS, 32 / L>::V]) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    constexpr int n = LV::n, V = LV::V, H = n / 2;
    auto& ws = cx.ws;
    const int lane = cx.lane, p = cx.p, u = cx.u, base = ws.next_map;
#pragma unroll
    for (int k = 0; k < V; k++) {
        const int e = LV::full ? k * C::LPP + u : u;
        if (LV::full || u < n) ws.vbuf[p * n + e] = x[k];
    }
    if (lane < 2 * L) ws.cb[lane] = (int)cx.maps[base + lane].icol[SS - 1];
    __syncwarp();
    float part[2 * L];
#pragma unroll
    for (int t = 0; t < 2 * L; t++) {
        const u32 d = (u32)ws.cb[t];
        const int h = 31 - __clz(d);
        const int src = t % L;
        float acc = 0.f;
        // canonical pairs q = lane + 32 r: i = q with a zero inserted at bit h
        for (int q = lane, r = 0; q < H; q += 32, r++) {
            const int i = ((q >> h) << (h + 1)) | (q & ((1 << h) - 1));
            const float m = fminf(fabsf(ws.vbuf[src * n + i]), fabsf(ws.vbuf[src * n + (i ^ (int)d)]));
            acc = (r == 0) ? m : acc + m;
        }
        part[t] = acc;
    }
    int tri;
    const float tot = multi_tree<2 * L>(part, lane, &tri);
    if ((lane & (32 / (2 * L) - 1)) == 0) ws.lm[tri] = tot;
    __syncwarp();
    select_trials2(cx);
    // winners: permuted vectors x'[j] = x_src[sigma^-1(j)]
    const int t = ws.ord[p];
    const int src = t % L;
    const MapR<MM>& mp = cx.maps[base + t];
    if constexpr (LV::full) {
        NodeIdx<SS, C::LPP, V> ni;
        ni.build(mp.icol, (u32)mp.c, u);
        const float* vs = &ws.vbuf[src * n];
#pragma unroll
        for (int k = 0; k < V; k++) x[k] = vs[ni.at(k)];
    } else {
        const u32 j = (u32)mp.c ^ lin_apply<SS>(mp.icol, (u32)u);
        x[0] = u < n ? ws.vbuf[src * n + j] : 0.f;
    }
    float npm = 0.f;
    if (lane < L) npm = ws.pm[ws.ord[lane] % L];
    __syncwarp();
    if (lane < L) {
        ws.pm[lane] = npm;
        ws.l0[SS][lane] = (int8_t)(ws.ord[lane] % L);
        ws.nmap[SS][lane] = (int16_t)(base + ws.ord[lane]);
    }
    ws.next_map = base + 2 * L;
    __syncwarp();
}


// g (list_engine.py:23-27) when the left child is an FHT node: its hard
// decisions for this lane are bit_k = c0 ^ parity(Bh & k) (fht_node), so
// the +-1 factors follow a Gray-code walk: one FMUL2 + one FFMA2 per pair.
template <int R, int MM, int L, int SS>
__device__ __forceinline__ void g_fht_child(const Ctx2<R, MM, L>& cx, int slot, const float* a, const float* b,
                                            float* out) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;  // the left child's level
    constexpr int V = LV::V, n = LV::n;
    static_assert(LV::full && V >= 2, "paired walk");
    const int bin = cx.ws.sel_bin[slot];
    const int sgn = cx.ws.sel_w[slot] < 0.f;
    const u32 B = (u32)(~bin) & (u32)(n - 1);
    const u32 Bh = B >> C::LB;
    const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)cx.u & (u32)(C::LPP - 1)) & 1);
    const float base = c0 ? -1.f : 1.f;
    const float col0 = (Bh & 1u) ? -1.f : 1.f;
    u64 s2 = pk(base, base * col0);  // factors of slots (k, k+1), k = 2 * gray(i)
#pragma unroll
    for (int i = 0; i < V / 2; i++) {
        if (i > 0) {
            const int j = __ffs(i);  // bit of k flipped by this Gray step (>= 1)
            const float cj = ((Bh >> j) & 1u) ? -1.f : 1.f;
            s2 = mul2(s2, pk(cj, cj));
        }
        const int k = 2 * (i ^ (i >> 1));
        const u64 r = fma2(s2, pk(a[k], a[k + 1]), pk(b[k], b[k + 1]));
        out[k] = plo(r);
        out[k + 1] = phi(r);
    }
}

// ------------------------------------------------------- tree recursion ----
template <int R, int MM, int L, int RR, int SS, bool SPINE>
__device__ __forceinline__ u64 node2(Ctx2<R, MM, L>& cx, float (&x)[Lv<SS, 32 / L>::V], int8_t* lin) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<SS, C::LPP>;
    if constexpr (RR == 1) {
        return fht_node<R, MM, L, SS>(cx, x, lin);
    } else if constexpr (RR == SS - 1) {
        return spc_node<R, MM, L, SS>(cx, x, lin);
    } else {
        using LC = Lv<SS - 1, C::LPP>;
        constexpr int V = LV::V, VC = LC::V, n = LV::n, h = n / 2;
        constexpr bool INNER_PERM = SPINE && RR >= 2 && SS - RR >= 2 && SS < MM;
        auto& ws = cx.ws;
        const int lane = cx.lane, p = cx.p, u = cx.u;
        int8_t* l0 = ws.l0[SS];
        int8_t* l1 = ws.l1[SS];
        int8_t* l2 = ws.l2[SS];
        if (INNER_PERM && cx.perms) {
            if constexpr (INNER_PERM) perm_ext_inner2<R, MM, L, SS>(cx, x);
        } else if constexpr (SS < MM) {
            if (lane < L) l0[lane] = (int8_t)lane;
            __syncwarp();
        }
        // f (:100)
        float xl[VC];
        if constexpr (LC::full) {
#pragma unroll
            for (int k = 0; k < VC; k++) xl[k] = f_op(x[k], x[k + VC]);
        } else {
            const float o = __shfl_down_sync(kFull, x[0], h);
            xl[0] = (u < h) ? f_op(x[0], o) : 0.f;
        }
        // An internal node's own vector waits in the warp's tensor-memory block
        // (free after the root's g: for R == 2 every left child is a leaf and
        // these nodes all lie in the root's right subtree) while its left
        // child runs: the FHT leaf then has the registers to itself.
        constexpr bool XPARK = RMFHT_XPARK && tmem_park<R, MM, L>() && R == 2 && SS < MM && LV::full && V % 8 == 0 &&
                               V >= RMFHT_XPARK_MINV;
        if constexpr (XPARK) {
#pragma unroll
            for (int k0 = 0; k0 < V; k0 += 8) tmem_st8(cx.tmem + k0, &x[k0]);
            tmem_wait_st();
        }
        const u64 bl = node2<R, MM, L, RR - 1, SS - 1, SPINE>(cx, xl, l1);   // :101
        if constexpr (XPARK) {
            if constexpr (V == 8) {
                u32 ra[8];
                tmem_ld8(cx.tmem, ra);
                tmem_wait_ld8(ra);
#pragma unroll
                for (int i = 0; i < 8; i++) x[i] = __uint_as_float(ra[i]);
            } else {
#pragma unroll
                for (int k0 = 0; k0 < V; k0 += 16) {
                    u32 ra[8], rb[8];
                    tmem_ld8(cx.tmem + k0, ra);
                    tmem_ld8(cx.tmem + k0 + 8, rb);
                    tmem_wait_ld16(ra, rb);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        x[k0 + i] = __uint_as_float(ra[i]);
                        x[k0 + 8 + i] = __uint_as_float(rb[i]);
                    }
                }
            }
        }
        // alphas = alphas[lin1] (:102)
        const int src1 = l1[p];
        const bool moved = __any_sync(kFull, src1 != p);
        if (moved) {
#pragma unroll
            for (int k = 0; k < V; k++) x[k] = __shfl_sync(kFull, x[k], src1 * C::LPP + u);
        }
        // g (:104) with the left child's hard decisions
        float xr[VC];
        if constexpr (RR - 1 == 1 && LC::full && VC >= 2) {
            g_fht_child<R, MM, L, SS - 1>(cx, p, x, x + VC, xr);
        } else if constexpr (LC::full) {
#pragma unroll
            for (int k = 0; k < VC; k++) {
                const float sg = ((bl >> k) & 1ull) ? -1.f : 1.f;
                xr[k] = __fmaf_rn(sg, x[k], x[k + VC]);
            }
        } else {
            const float o = __shfl_down_sync(kFull, x[0], h);
            const float sg = (bl & 1ull) ? -1.f : 1.f;
            xr[0] = (u < h) ? __fmaf_rn(sg, x[0], o) : 0.f;
        }
        const u64 br = node2<R, MM, L, RR, SS - 1, false>(cx, xr, l2);      // :105
        // combine (:106-107): beta = [beta_l[lin2] ^ beta_r, beta_r]
        const int src2 = l2[p];
        const u64 blm = __shfl_sync(kFull, bl, src2 * C::LPP + u);
        u64 out;
        if constexpr (LC::full) {
            out = (br << VC) | (blm ^ br);
        } else {
            const u64 brup = __shfl_up_sync(kFull, br, h);
            out = (u < h) ? ((blm ^ br) & 1ull) : (brup & 1ull);
            if (!(LV::full || u < n)) out = 0;
        }
        const int chain = l1[src2];
        if (INNER_PERM && cx.perms) {
            // un-permute by this node's trial map (:109-112): out[i] = beta[sigma(i)]
#pragma unroll
            for (int k = 0; k < V; k++) {
                const int e = LV::full ? k * C::LPP + u : u;
                if (LV::full || u < n) ws.ubits[p * n + e] = (uint8_t)((out >> k) & 1ull);
            }
            __syncwarp();
            const MapR<MM>& mp = cx.maps[ws.nmap[SS][chain]];
            u64 o2 = 0;
            if constexpr (LV::full) {
                NodeIdx<SS, C::LPP, V> ni;
                ni.build(mp.col, (u32)mp.b, u);
                const uint8_t* ub = &ws.ubits[p * n];
#pragma unroll
                for (int k = 0; k < V; k++) o2 |= (u64)ub[ni.at(k)] << k;
            } else {
                const u32 sidx = (u32)mp.b ^ lin_apply<SS>(mp.col, (u32)u);
                if (u < n) o2 = (u64)ws.ubits[p * n + sidx];
            }
            out = o2;
            __syncwarp();
        }
        if (lane < L) {
            const int ch = l1[l2[lane]];
            lin[lane] = l0[ch];
            if (SS == MM) ws.rootchain[lane] = (int8_t)ch;
        }
        __syncwarp();
        return out;
    }
}

// ------------------------------------------------------------ root node ----
// Internal root (1 < r < m-1): the root vectors are never held; f (:100) and
// g (:104) read them straight from the frame LLRs through each path's
// composite map, g after the left child's lineage (:102) re-selects the maps.
// `alpha_dead` runs once the frame LLRs have been read for the last time.
template <int R, int MM, int L, typename F>
__device__ __forceinline__ u64 root_node(Ctx2<R, MM, L>& cx, int8_t* lin, F&& alpha_dead) {
    using C = Cfg<R, MM, L>;
    using LV = Lv<MM, C::LPP>;
    using LC = Lv<MM - 1, C::LPP>;
    constexpr int VC = LC::V;
    static_assert(LC::full, "root children span the lane group");
    auto& ws = cx.ws;
    const int lane = cx.lane, p = cx.p, u = cx.u;
    int8_t* l0 = ws.l0[MM];
    int8_t* l1 = ws.l1[MM];
    int8_t* l2 = ws.l2[MM];
    float xl[VC];
    {
#ifdef RMFHT_STATS
        const long long tg = clock64();
#endif
        RootIdx<MM, C::LPP, LV::V> ri;
        ri.build(ws.comp[p], u, cx.alpha_saddr);
        if constexpr (tmem_park<R, MM, L>()) {
            // gather, park both halves in tensor memory (column k: the lower
            // half's slot k, column VC + k the upper half's), then f
#pragma unroll
            for (int k0 = 0; k0 < VC; k0 += 8) {
                float a[8], b[8];
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    a[i] = lds_addr(ri.off(k0 + i));
                    b[i] = lds_addr(ri.off(k0 + i + VC));
                }
                tmem_st8(cx.tmem + k0, a);
                tmem_st8(cx.tmem + VC + k0, b);
#pragma unroll
                for (int i = 0; i < 8; i++) xl[k0 + i] = f_op(a[i], b[i]);
            }
            tmem_wait_st();
            alpha_dead();  // the frame LLRs are not read again
        } else {
#pragma unroll
            for (int k = 0; k < VC; k++) xl[k] = f_op(lds_addr(ri.off(k)), lds_addr(ri.off(k + VC)));
        }
#ifdef RMFHT_STATS
        {
            float z = 0.f;
#pragma unroll
            for (int k = 0; k < VC; k++) z += xl[k];
            __syncwarp();
            const long long dg = clock64() - tg + (z == 1e30f ? 1 : 0);
            RMFHT_STAT_ADD(244, dg);
            RMFHT_STAT_ADD(245, dg * dg / 1024);
            if (lane_id() == 0) atomicMax(&g_stats[246], (unsigned long long)dg);
        }
#endif
    }
    const u64 bl = node2<R, MM, L, R - 1, MM - 1, true>(cx, xl, l1);
    float xr[VC];
    if constexpr (tmem_park<R, MM, L>()) {
        // g (:104) from the parked values of the source path (:102); the
        // factors follow g_fht_child's Gray-code walk, whose steps 4 c .. 4 c + 3
        // stay inside the 8-slot chunk c ^ (c >> 1)
        const int src1 = l1[p];
        const bool moved = __any_sync(kFull, src1 != p);
        const int from = src1 * C::LPP + u;
        if constexpr (R - 1 != 1) {
            // general left child: its hard decisions are the bits of bl
#pragma unroll
            for (int k0 = 0; k0 < VC; k0 += 8) {
                u32 ra[8], rb[8];
                tmem_ld8(cx.tmem + k0, ra);
                tmem_ld8(cx.tmem + VC + k0, rb);
                tmem_wait_ld16(ra, rb);
                if (moved) {
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        ra[i] = __shfl_sync(kFull, ra[i], from);
                        rb[i] = __shfl_sync(kFull, rb[i], from);
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const float sg = ((bl >> (k0 + i)) & 1ull) ? -1.f : 1.f;
                    xr[k0 + i] = __fmaf_rn(sg, __uint_as_float(ra[i]), __uint_as_float(rb[i]));
                }
            }
        } else {
        constexpr int n = 1 << (MM - 1);
        const int bin = ws.sel_bin[p];
        const int sgn = ws.sel_w[p] < 0.f;
        const u32 B = (u32)(~bin) & (u32)(n - 1);
        const u32 Bh = B >> C::LB;
        const int c0 = sgn ^ (__popc(B) & 1) ^ (__popc(B & (u32)u & (u32)(C::LPP - 1)) & 1);
        const float base = c0 ? -1.f : 1.f;
        const float col0 = (Bh & 1u) ? -1.f : 1.f;
        u64 s2 = pk(base, base * col0);
#pragma unroll
        for (int c = 0; c < VC / 8; c++) {
            const int k0 = 8 * (c ^ (c >> 1));
            u32 ra[8], rb[8];
            tmem_ld8(cx.tmem + k0, ra);
            tmem_ld8(cx.tmem + VC + k0, rb);
            tmem_wait_ld16(ra, rb);
            if (moved) {
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    ra[i] = __shfl_sync(kFull, ra[i], from);
                    rb[i] = __shfl_sync(kFull, rb[i], from);
                }
            }
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
                xr[k] = plo(r);
                xr[k + 1] = phi(r);
            }
        }
        }
    } else {
        RootIdx<MM, C::LPP, LV::V> ri;
        ri.build(ws.comp[l1[p]], u, cx.alpha_saddr);
        if constexpr (R - 1 == 1 && VC >= 2) {
            float ga[VC], gb[VC];
#pragma unroll
            for (int k = 0; k < VC; k++) {
                ga[k] = lds_addr(ri.off(k));
                gb[k] = lds_addr(ri.off(k + VC));
            }
            alpha_dead();
            g_fht_child<R, MM, L, MM - 1>(cx, p, ga, gb, xr);
        } else {
#pragma unroll
            for (int k = 0; k < VC; k++) {
                const float sg = ((bl >> k) & 1ull) ? -1.f : 1.f;
                xr[k] = __fmaf_rn(sg, lds_addr(ri.off(k)), lds_addr(ri.off(k + VC)));
            }
            alpha_dead();
        }
    }
    const u64 br = node2<R, MM, L, R, MM - 1, false>(cx, xr, l2);
    const int src2 = l2[p];
    const u64 blm = __shfl_sync(kFull, bl, src2 * C::LPP + u);
    const u64 out = (br << VC) | (blm ^ br);
    if (lane < L) {
        const int ch = l1[l2[lane]];
        lin[lane] = l0[ch];
        ws.rootchain[lane] = (int8_t)ch;
    }
    __syncwarp();
    return out;
}

// per-attempt record written by decode_kernel2, reduced by reduce_kernel2
struct AttHdr {
    float pm;
    int path, init_map, trial_map;
};

template <int R, int MM, int L>
__host__ __device__ constexpr size_t smem_bytes2(int nwarps) {
    // 2 KB alignment pad + per-warp LLR copy (N floats, N-aligned) + per-warp scratch
    return 2048 + size_t(1 << MM) * 4 * size_t(nwarps) + sizeof(WS2<R, MM, L>) * size_t(nwarps);
}

// warps per CTA: the largest multiple of 4 (at most 32, i.e. a 64-register
// cap) whose LLR copies and scratch fit in 227 KB of shared memory
template <int R, int MM, int L>
__host__ __device__ constexpr int fast_warps() {
#ifdef RMFHT_FAST_WARPS_MAX
    int w = RMFHT_FAST_WARPS_MAX;  // A/B builds only (tools/build_variant.py)
#else
    int w = 32;
#endif
    while (w > 4 && smem_bytes2<R, MM, L>(w) > 227 * 1024) w -= 4;
    return w;
}

// ------------------------------------------------------------- kernel ----
// Work item = (frame, attempt); warps of a CTA take consecutive items in
// lock-stepped rounds (they run the same code path, so they share the
// instruction stream).
// PM: permutations (p-FHT-FSCL); false = FHT-FSC (L = 1, identity maps)
template <int R, int MM, int L, bool PM = true>
#ifdef RMFHT_FAST_LB_WARPS
#define RMFHT_KERNEL2_LB (32 * RMFHT_FAST_LB_WARPS)  // A/B builds only: register cap of a larger CTA
#else
#define RMFHT_KERNEL2_LB (32 * fast_warps<R, MM, L>())
#endif
__global__ void __launch_bounds__(RMFHT_KERNEL2_LB, 1) decode_kernel2(rmfht::Params<float> prm, AttHdr* hdr, u64* bitsout) {
    using C = Cfg<R, MM, L>;
    using WS = WS2<R, MM, L>;
    using LV = Lv<MM, C::LPP>;
    constexpr int N = C::N, S = C::S, REC = 2 * MM + 2, V = LV::V;
    static_assert(N >= 32 && L <= 8 && N <= 512, "fast kernel: 32 <= N <= 512, L <= 8");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // the launch always uses fast_warps() warps (prepare_fast): a compile-time
    // count keeps the per-warp scratch addresses cheap to rematerialise
    constexpr int nwarps = fast_warps<R, MM, L>();
    // (warp index through a shuffle: provably warp-uniform, so the per-warp
    // scratch addresses live in uniform registers instead of being
    // rematerialised from threadIdx under register pressure)
    const int warp = __shfl_sync(kFull, (int)(threadIdx.x >> 5), 0), lane = lane_id();
    // per-warp frame LLRs, each 2 KB aligned in the shared window, then the scratch
    // (the scratch first: its addresses need no alignment arithmetic; the
    // compiler rematerialises them all over the kernel)
    static_assert(sizeof(WS) % 16 == 0, "scratch stride");
    WS& ws = reinterpret_cast<WS*>(smem_raw)[warp];
    const u32 raw_saddr = (u32)__cvta_generic_to_shared(smem_raw) + (u32)(nwarps * sizeof(WS));
    const u32 pad = ((raw_saddr + 2047u) & ~2047u) - raw_saddr;
    constexpr u32 ASTRIDE = (u32)N * 4u;  // N-aligned: gather offsets (< 4N bytes) are OR-ed into the base
    float* const alpha_w = reinterpret_cast<float*>(smem_raw + nwarps * sizeof(WS) + pad + (size_t)warp * ASTRIDE);
    const u32 asa = (u32)__cvta_generic_to_shared(alpha_w);
    Ctx2<R, MM, L> cx{ws, alpha_w, nullptr, PM ? 1 : 0, {}, lane, lane / C::LPP, lane % C::LPP, asa};
    static_assert(sizeof(MapR<MM>) == 2 * (2 * MM + 2), "record layout");
    constexpr bool ROOT_INTERNAL = !(R == 1 || R == MM - 1);
    // tensor memory for the root's parked gathers (tmem_park): the whole 512
    // columns (one CTA per SM); warp w owns lanes 32 (w % 4) .. + 31 (the
    // quadrant a warp may access) and 2 VC columns from 2 VC (w / 4)
    constexpr bool TPARK = PM && ROOT_INTERNAL && tmem_park<R, MM, L>();
    __shared__ u32 tmem_slot;
    cx.tmem = 0;
    if constexpr (TPARK) {
        constexpr int TCOLS = 2 * Lv<MM - 1, C::LPP>::V;  // columns per warp
        static_assert((nwarps + 3) / 4 * TCOLS <= 512, "tensor-memory columns");
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             (u32)__cvta_generic_to_shared(&tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        cx.tmem = tmem_slot + ((u32)(32 * (warp & 3)) << 16) + (u32)(TCOLS * (warp >> 2));
    }
    // items < 2^31 per launch (launch_fast splits larger batches)
    const int items = (int)prm.B * prm.M;
    const int stride = (int)gridDim.x * nwarps;
    // Prefetch (LDGSTS) of the warp's next work item: its map records into the
    // idle half of ws.recs at item start, its LLRs into the single LLR buffer
    // as soon as the current item has read the frame LLRs for the last time
    // (after the root's g, i.e. before the right half of the tree).
    auto prefetch_recs = [&](int it, int buf) {
        if (it >= items || !PM) return;
        const u32 rsa = (u32)__cvta_generic_to_shared(ws.recs[buf]);
        const char* gr = reinterpret_cast<const char*>(prm.maps + (size_t)it * S * REC);
        constexpr int RB = S * REC * 2;  // record bytes per item
        if (RB % 16 == 0 && (reinterpret_cast<uintptr_t>(prm.maps) & 15u) == 0) {
            for (int i = lane; i < RB / 16; i += 32) cp_async16(rsa + 16u * i, gr + 16 * i);
        } else {
            for (int i = lane; i < WS::RECW / 2; i += 32) cp_async4(rsa + 4u * i, gr + 4 * i);
        }
        cp_async_commit();
    };
    auto prefetch_alpha = [&](int it) {
        if (it >= items) return;
        __syncwarp();  // every lane is past its last read of the current LLRs
        const char* ga = reinterpret_cast<const char*>(prm.llr + (size_t)((u32)it / (u32)prm.M) * N);
        for (int i = lane; i < N / 4; i += 32) cp_async16(asa + 16u * i, ga + 16 * i);
        cp_async_commit();
    };
    int cur = 0;
    prefetch_recs((int)blockIdx.x * nwarps + warp, 0);
    prefetch_alpha((int)blockIdx.x * nwarps + warp);
    for (int base = (int)blockIdx.x * nwarps; base < items; base += stride) {
        const int item = base + warp;
        if (item < items) {
#ifdef RMFHT_STATS
            const long long t_item = clock64();
            cx.ngen = 0;
#endif
            cp_async_wait_all();
            __syncwarp();
            if constexpr (WS::RB == 2) prefetch_recs(item + stride, cur ^ 1);
#pragma unroll
            for (int s = 0; s < C::NS; s++) cx.ach[s] = alpha_w[lane + 32 * s];
            cx.maps = reinterpret_cast<const MapR<MM>*>(ws.recs[cur]);
            if (lane < L) {
                if constexpr (PM) {
                    ws.comp[lane] = cx.maps[lane];  // L root maps (:129-139)
                } else {
#pragma unroll
                    for (int k = 0; k < MM; k++) ws.comp[lane].col[k] = ws.comp[lane].icol[k] = (uint16_t)(1u << k);
                    ws.comp[lane].b = ws.comp[lane].c = 0;
                }
                ws.pm[lane] = 0.f;
                ws.l0[MM][lane] = (int8_t)lane;
                ws.nmap[MM][lane] = -1;
            }
            ws.next_map = L;
            __syncwarp();
            int8_t* rlin = ws.l2[0];  // root lineage (level-0 slot is unused by nodes)
            u64 bits;
            if constexpr (ROOT_INTERNAL) {
                if constexpr (PM) perm_ext_root2(cx);
            }
            // single record buffer: the records are dead from here on (the root
            // maps live on in ws.comp); refill it with the next item's
            if constexpr (WS::RB == 1) prefetch_recs(item + stride, 0);
            if constexpr (ROOT_INTERNAL && Lv<MM - 1, C::LPP>::full) {
                bits = root_node(cx, rlin, [&] { prefetch_alpha(item + stride); });
            } else {
                float x[V];
                RootIdx<MM, C::LPP, V> ri;
                ri.build(ws.comp[cx.p], cx.u, cx.alpha_saddr);
#pragma unroll
                for (int k = 0; k < V; k++) x[k] = lds_addr(ri.off(k));
                prefetch_alpha(item + stride);
                bits = node2<R, MM, L, R, MM, true>(cx, x, rlin);
            }
            // best path: first minimum (:152)
            int best = 0;
#pragma unroll
            for (int i = 1; i < L; i++)
                if (ws.pm[i] < ws.pm[best]) best = i;
            const int rslot = ROOT_INTERNAL ? ws.rootchain[best] : rlin[best];
            if (lane == 0) {
                AttHdr h;
                h.pm = ws.pm[best];
                h.path = best;
                h.init_map = !PM ? -1 : ROOT_INTERNAL ? ws.l0[MM][rslot] : rslot;
                h.trial_map = !PM ? -1 : ROOT_INTERNAL ? ws.nmap[MM][rslot] : -1;
                hdr[item] = h;
            }
            if (cx.p == best) bitsout[(size_t)item * C::LPP + cx.u] = bits;
            __syncwarp();
            if constexpr (WS::RB == 2) cur ^= 1;
#ifdef RMFHT_STATS
            {
                const long long dt = clock64() - t_item;
                RMFHT_STAT_ADD(200, dt);
                RMFHT_STAT_ADD(201, dt * dt / 1024);
                RMFHT_STAT(202);
                if (lane_id() == 0) atomicMax(&g_stats[203], (unsigned long long)dt);
                const int bucket = dt < 2048 ? 0 : dt < 65536 ? 1 + (int)((dt - 2048) / 2048) : 33;
                RMFHT_STAT(210 + bucket);
                const int ng = cx.ngen < 7 ? cx.ngen : 7;
                RMFHT_STAT_ADD(150 + ng, dt);
                RMFHT_STAT(160 + ng);
            }
#endif
        }
        // lock-step rounds: warps share the instruction stream (named barrier per group)
        const int grp = (prm.tie_fix >> 8) & 0xff;  // warps per lock-step group, 0 = none
        if (grp == 0) {
            // free-running warps
        } else if (grp >= nwarps || nwarps % grp != 0) {
            __syncthreads();
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + warp / grp), "r"(grp * 32) : "memory");
        }
    }
    if constexpr (TPARK) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_slot) : "memory");
    }
}

// Per frame: first strict minimum over attempts (top_decoders.py:200), then
// un-permute the winner's root-domain bits by its composite root map
// (:147-150): codeword bit i = beta[sigma(i)], sigma = trial o init.
// LPPX: lanes per path of the kernel that wrote the records (bit k of lane
// u's word = element k * LPPX + u); the lane-group kernel (rmfht_grp.cuh)
// writes 8-lane records for L = 1
template <int R, int MM, int L, int LPPX = Cfg<R, MM, L>::LPP>
__global__ void __launch_bounds__(256) reduce_kernel2(rmfht::Params<float> prm, const AttHdr* hdr, const u64* bitsin) {
    using C = Cfg<R, MM, L>;
    constexpr int N = C::N, NW = N / 32, S = C::S, REC = 2 * MM + 2, LPP = LPPX;
    __shared__ u64 sbits[8][LPP];
    __shared__ MapS smap[8];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const long long f = (long long)blockIdx.x * 8 + warp;
    if (f >= prm.B) return;
    const int M = prm.M;
    // the frame's LLRs (for the reported pm) do not depend on the winner:
    // in flight while the attempt records are reduced
    float fll[NW];
    {
        const float* fl0 = prm.llr + (size_t)f * N;
#pragma unroll
        for (int t = 0; t < NW; t++) fll[t] = __ldg(fl0 + t * 32 + lane);
    }
    // first minimum over (pm, attempt)
    float bp = 0.f;
    int ba = -1;
    for (int a = lane; a < M; a += 32) {
        const float v = hdr[f * M + a].pm;
        if (ba < 0 || v < bp) { bp = v; ba = a; }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const float ov = __shfl_xor_sync(kFull, bp, off);
        const int oa = __shfl_xor_sync(kFull, ba, off);
        if (oa >= 0 && (ba < 0 || ov < bp || (ov == bp && oa < ba))) { bp = ov; ba = oa; }
    }
    const bool diag = prm.att_pm || prm.att_cw;  // either may be NULL (rmfht.h)
    const int a0 = diag ? 0 : ba, a1 = diag ? M : ba + 1;
    for (int a = a0; a < a1; a++) {
        const long long item = f * M + a;
        const AttHdr h = hdr[item];
        if (lane < LPP) sbits[warp][lane] = bitsin[(size_t)item * LPP + lane];
        // the winner's composite sigma = trial o init (columns of A and the
        // shift), one column per lane: lane k < MM takes column k, lane MM the
        // shift — A_t (A_i e_k) and A_t b_i ^ b_t
        if (lane <= MM) {
            u32 x;
            if (h.init_map < 0) {  // no permutations: identity
                x = lane < MM ? (1u << lane) : 0u;
            } else {
                x = prm.maps[((size_t)item * S + h.init_map) * REC + lane];  // col[lane] or b (half word MM)
            }
            if (h.trial_map >= 0) {
                const uint16_t* tr = prm.maps + ((size_t)item * S + h.trial_map) * REC;
                u32 v = lane == MM ? (u32)tr[MM] : 0u;
#pragma unroll
                for (int j = 0; j < MM; j++)
                    if ((x >> j) & 1u) v ^= tr[j];
                x = v;
            }
            if (lane < MM) smap[warp].col[lane] = x;
            else smap[warp].b = x;
        }
        __syncwarp();
        const MapS& fm = smap[warp];
        u32 myword = 0;
        // reported pm: the decided codeword's metric from the channel LLRs
        // (rmfht::CorrPm); the accumulated h.pm selected the attempt
        rmfht::CorrPm corr;
#pragma unroll
        for (int t = 0; t < NW; t++) {
            const u32 i = (u32)(t * 32 + lane);
            const u32 e = fm.b ^ lin_apply<MM>(fm.col, i);
            const int bit = (int)((sbits[warp][e % LPP] >> (e / LPP)) & 1ull);
            corr.add(fll[t], bit);
            const u32 word = __ballot_sync(kFull, bit);
            if (lane == t) myword = word;
        }
        const float rep = corr.total();
        if (prm.att_pm && lane == 0) prm.att_pm[item] = rep;
        if (prm.att_cw && lane < NW) prm.att_cw[item * NW + lane] = myword;
        if (a == ba) {
            if (lane < NW) prm.cw[f * NW + lane] = myword;
            if (lane == 0) {
                prm.pm[f] = rep;
                prm.attempt[f] = ba;
                prm.path[f] = h.path;
            }
        }
        __syncwarp();
    }
}


template <int R, int MM, int L>
constexpr size_t work_bytes2() {
    return sizeof(AttHdr) + sizeof(u64) * size_t(Cfg<R, MM, L>::LPP);
}

}  // namespace rmfht2
