// Affine-map tables shared by the host (C ABI) and the device sampler:
// one source of truth, so a table drawn on the GPU is bit-identical to the
// one rmfht_sample_maps draws on the host.
//
// Raw map (m+1 uint16): row masks of A (bit j of row r = A[r, j],
// automorphism.py:122-124), b at index m.  Device record (2m+2 uint16):
// columns of A, b, columns of A^-1, A^-1 b (automorphism.py:92-108).
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define RMFHT_HD __host__ __device__ __forceinline__
#else
#define RMFHT_HD inline
#endif

namespace rmfht_maps {

RMFHT_HD uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// raw (row masks, b) -> record; -1 for a singular A (Gauss-Jordan on [A | I],
// gf2_inverse, automorphism.py:58-71)
RMFHT_HD int expand_one(const uint16_t* raw, int mn, int mg, uint16_t* rec) {
    unsigned rows[16], inv[16];
    for (int r = 0; r < mn; r++) {
        rows[r] = raw[r];
        inv[r] = 1u << r;
        if (raw[r] >> mn) return -1;
    }
    for (int r = mn; r < mg; r++)
        if (raw[r]) return -1;
    const unsigned b = raw[mg];
    if (b >> mn) return -1;
    for (int c = 0; c < mn; c++) {
        int piv = -1;
        for (int r = c; r < mn; r++)
            if (rows[r] >> c & 1u) {
                piv = r;
                break;
            }
        if (piv < 0) return -1;
        unsigned t = rows[c];
        rows[c] = rows[piv];
        rows[piv] = t;
        t = inv[c];
        inv[c] = inv[piv];
        inv[piv] = t;
        for (int r = 0; r < mn; r++)
            if (r != c && (rows[r] >> c & 1u)) {
                rows[r] ^= rows[c];
                inv[r] ^= inv[c];
            }
    }
    for (int k = 0; k < 2 * mg + 2; k++) rec[k] = 0;
    unsigned cinv = 0;
    for (int k = 0; k < mn; k++) {
        unsigned col = 0, icol = 0;
        for (int r = 0; r < mn; r++) {
            col |= (unsigned)((raw[r] >> k) & 1u) << r;
            icol |= ((inv[r] >> k) & 1u) << r;
        }
        rec[k] = (uint16_t)col;
        rec[mg + 1 + k] = (uint16_t)icol;
        if (b >> k & 1u) cinv ^= icol;
    }
    rec[mg] = (uint16_t)b;
    rec[2 * mg + 1] = (uint16_t)cinv;
    return 0;
}

// Table semantics (host and device): slot s of (frame f, attempt a) holds a
// map drawn from its own counter-based stream keyed by (seed, f, a, s), so a
// frame's maps do not depend on the batch or the thread that draws them.
// With identity_root, attempt 0's L root slots are the identity ("decoder 0 =
// identity") and are not drawn.
RMFHT_HD uint64_t slot_key(uint64_t seed, long long f, int a, int s) {
    uint64_t st = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull);
    st += ((uint64_t)a << 24) + ((uint64_t)s << 8);
    uint64_t k = splitmix64(st);
    k ^= 0xC2B2AE3D27D4EB4Full;
    return splitmix64(k);
}

// 16-bit words of a splitmix64 stream
struct Word16 {
    uint64_t st, w;
    int left;
    RMFHT_HD explicit Word16(uint64_t key) : st(key), w(0), left(0) {}
    RMFHT_HD unsigned next() {
        if (left == 0) {
            w = splitmix64(st);
            left = 4;
        }
        const unsigned v = (unsigned)w & 0xffffu;
        w >>= 16;
        left--;
        return v;
    }
};

// The same word stream with its first four splitmix64 outputs drawn up front
// (device sampler): the lanes of a warp fall out of step after a redraw, and
// Word16's refill — a whole splitmix64 behind a divergent branch at every call
// site — then ran at nearly every call of every warp; here the refill picks
// one of the four prepared words (a fifth, after more than six redraws in one
// map, is drawn on the spot).
struct Word16p {
    uint64_t st, w, w1, w2, w3;
    int left, fills;
    RMFHT_HD explicit Word16p(uint64_t key) : st(key), left(4), fills(1) {
        w = splitmix64(st);
        w1 = splitmix64(st);
        w2 = splitmix64(st);
        w3 = splitmix64(st);
    }
    RMFHT_HD unsigned next() {
        if (left == 0) {
            w = fills == 1 ? w1 : fills == 2 ? w2 : fills == 3 ? w3 : splitmix64(st);
            fills++;
            left = 4;
        }
        const unsigned v = (unsigned)w & 0xffffu;
        w >>= 16;
        left--;
        return v;
    }
};

// t ^= u when (v & m) != 0
RMFHT_HD void xor_if(unsigned& t, unsigned v, unsigned m, unsigned u) {
#ifdef __CUDA_ARCH__
    // a predicated XOR (two instructions; the compiler's own choice was test,
    // select, XOR — the sampler kernel is issue-bound on exactly these)
    asm("{\n\t.reg .pred p;\n\t.reg .b32 q;\n\tand.b32 q, %1, %2;\n\tsetp.ne.u32 p, q, 0;\n\t@p xor.b32 %0, %0, %3;\n\t}"
        : "+r"(t)
        : "r"(v), "r"(m), "r"(u));
#else
    if (v & m) t ^= u;
#endif
}

// Uniform (A, b) in GL(MN,2) x F_2^MN — the distribution of the reference's
// rejection sampler (automorphism.py:127-161) — drawn column by column, each
// column uniform over the vectors outside the span of the previous ones, so
// every invertible A has probability 1/|GL|.
//
// The span is kept as a REDUCED echelon basis u_j (pivot coordinate p_j:
// u_j has bit p_j set and every other pivot bit clear).  A vector x is
// written uniquely as x = r ^ sum_{j: s_j} u_j with r supported on the free
// (non-pivot) coordinates and s_j = bit p_j of x, so x is outside the span
// iff r != 0, and a uniform m-bit v gives a uniform column outside the span
// as r = v & free (redrawn while 0; the last column's single free bit is
// forced), s = the pivot bits of v.  The redraw loop is a mask test, so
// lanes that redraw do not hold the warp in a reduction loop.
//
// Each basis word also carries, in bits 16.., its coefficients over the
// columns drawn so far (A * coef_j = u_j): the new u_i = r has coef
// e_i ^ sum_{j: s_j} coef_j, and eliminating p_i from the earlier u_j XORs
// both halves.  After MN columns the u_j are the unit vectors e_{p_j}, so
// A^-1 e_{p_j} = coef_j: the columns of A^-1 without a Gauss-Jordan pass.
template <int MN, typename Words = Word16>
RMFHT_HD void draw_map_basis(uint64_t key, unsigned (&cols)[MN], unsigned (&ub)[MN], unsigned (&pv)[MN], unsigned& b) {
    constexpr unsigned mask = (1u << MN) - 1u;
    Words rs(key);
    // ub: basis word (u | coef << 16), pv: its pivot bit
    unsigned pivm = 0u;
#pragma unroll
    for (int i = 0; i < MN; i++) {
        unsigned v, r;
        do {
            v = rs.next() & mask;
            r = (i == MN - 1) ? (mask & ~pivm) : (v & ~pivm);
        } while (r == 0u);
        unsigned t = 0u;
#pragma unroll
        for (int j = 0; j < i; j++) xor_if(t, v, pv[j], ub[j]);
        cols[i] = r ^ (t & 0xffffu);
        ub[i] = (r | (1u << (16 + i))) ^ (t & 0xffff0000u);
        pv[i] = r & (0u - r);
        pivm |= pv[i];
#pragma unroll
        for (int j = 0; j < i; j++) xor_if(ub[j], ub[j], pv[i], ub[i]);
    }
    b = rs.next() & mask;
}

// After draw_map_basis the basis words are e_{p_j} | coef_j << 16 with
// A coef_j = e_{p_j}, i.e. column p_j of A^-1 is coef_j
template <int MN>
RMFHT_HD void draw_map(uint64_t key, unsigned (&cols)[MN], unsigned (&icols)[MN], unsigned& b) {
    unsigned ub[MN], pv[MN];
    draw_map_basis<MN>(key, cols, ub, pv, b);
#pragma unroll
    for (int k = 0; k < MN; k++) {
        unsigned c = 0u;
#pragma unroll
        for (int j = 0; j < MN; j++)
            if ((ub[j] >> k) & 1u) c = ub[j] >> 16;
        icols[k] = c;
    }
}

// runtime-size draw_map (rare slots: map sizes below m-2); same draws
RMFHT_HD void draw_map_rt(uint64_t key, int mn, unsigned* cols, unsigned* icols, unsigned& b) {
    const unsigned mask = (1u << mn) - 1u;
    Word16 rs(key);
    unsigned ub[16], pv[16];
    unsigned pivm = 0u;
    for (int i = 0; i < mn; i++) {
        unsigned v, r;
        do {
            v = rs.next() & mask;
            r = (i == mn - 1) ? (mask & ~pivm) : (v & ~pivm);
        } while (r == 0u);
        unsigned t = 0u;
        for (int j = 0; j < i; j++)
            if (v & pv[j]) t ^= ub[j];
        cols[i] = r ^ (t & 0xffffu);
        ub[i] = (r | (1u << (16 + i))) ^ (t & 0xffff0000u);
        pv[i] = r & (0u - r);
        pivm |= pv[i];
        for (int j = 0; j < i; j++)
            if (ub[j] & pv[i]) ub[j] ^= ub[i];
    }
    b = rs.next() & mask;
    for (int k = 0; k < mn; k++) {
        unsigned c = 0u;
        for (int j = 0; j < mn; j++)
            if ((ub[j] >> k) & 1u) c = ub[j] >> 16;
        icols[k] = c;
    }
}

template <int MN>
RMFHT_HD unsigned inv_shift(const unsigned (&icols)[MN], unsigned b) {
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < MN; k++) v ^= ((b >> k) & 1u) ? icols[k] : 0u;
    return v;
}

// raw map (row masks of A, b) and/or device record from an accepted candidate
template <int MN>
RMFHT_HD void write_map(const unsigned (&cols)[MN], const unsigned (&icols)[MN], unsigned b, int mg, uint16_t* raw,
                        uint16_t* rec) {
    if (raw) {
        for (int k = 0; k <= mg; k++) raw[k] = 0;
#pragma unroll
        for (int r = 0; r < MN; r++) {
            unsigned row = 0;
#pragma unroll
            for (int k = 0; k < MN; k++) row |= ((cols[k] >> r) & 1u) << k;
            raw[r] = (uint16_t)row;
        }
        raw[mg] = (uint16_t)b;
    }
    if (rec) {
        for (int k = 0; k < 2 * mg + 2; k++) rec[k] = 0;
#pragma unroll
        for (int k = 0; k < MN; k++) {
            rec[k] = (uint16_t)cols[k];
            rec[mg + 1 + k] = (uint16_t)icols[k];
        }
        rec[mg] = (uint16_t)b;
        rec[2 * mg + 1] = (uint16_t)inv_shift<MN>(icols, b);
    }
}

RMFHT_HD void write_identity(int mn, int mg, uint16_t* raw, uint16_t* rec) {
    if (raw) {
        for (int k = 0; k <= mg; k++) raw[k] = 0;
        for (int k = 0; k < mn; k++) raw[k] = (uint16_t)(1u << k);
    }
    if (rec) {
        for (int k = 0; k < 2 * mg + 2; k++) rec[k] = 0;
        for (int k = 0; k < mn; k++) {
            rec[k] = (uint16_t)(1u << k);
            rec[mg + 1 + k] = (uint16_t)(1u << k);
        }
    }
}

// host: one drawn slot (raw and/or record)
template <int MN>
inline void fill_slot_host(uint64_t key, int mg, uint16_t* raw, uint16_t* rec) {
    unsigned cols[MN], icols[MN], b;
    draw_map<MN>(key, cols, icols, b);
    write_map<MN>(cols, icols, b, mg, raw, rec);
}

inline void fill_slot_host_any(int mn, uint64_t key, int mg, uint16_t* raw, uint16_t* rec) {
    switch (mn) {
#define RMFHT_FC(K)                                   \
    case K:                                           \
        fill_slot_host<K>(key, mg, raw, rec); \
        break;
        RMFHT_FC(1) RMFHT_FC(2) RMFHT_FC(3) RMFHT_FC(4) RMFHT_FC(5) RMFHT_FC(6) RMFHT_FC(7)
        RMFHT_FC(8) RMFHT_FC(9) RMFHT_FC(10) RMFHT_FC(11) RMFHT_FC(12) RMFHT_FC(13) RMFHT_FC(14)
#undef RMFHT_FC
        default:
            break;
    }
}

}  // namespace rmfht_maps
