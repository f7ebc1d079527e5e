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

// Gauss-Jordan over GF(2) with compile-time size on augmented rows: t[r]
// holds row r of T in bits 0..15 and row r of the identity in bits 16..31, so
// one XOR is one row operation on [T | I].  Swap-free: a missing pivot is
// repaired by adding a later row that has it.  On success t[r] >> 16 is row r
// of T^-1.
template <int MN>
RMFHT_HD bool gj_inverse_aug(unsigned (&t)[MN]) {
#pragma unroll
    for (int c = 0; c < MN; c++) {
        const unsigned bit = 1u << c;
#pragma unroll
        for (int r = c + 1; r < MN; r++)
            if (~t[c] & t[r] & bit) t[c] ^= t[r];
        if (!(t[c] & bit)) return false;
#pragma unroll
        for (int r = 0; r < MN; r++)
            if (r != c && (t[r] & bit)) t[r] ^= t[c];
    }
    return true;
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

// Uniform (A, b) in GL(MN,2) x F_2^MN — the distribution of the reference's
// rejection sampler (automorphism.py:127-161) — drawn column by column: each
// column is uniform over the vectors outside the span of the previous ones
// (redrawn while inside it), so every invertible A has probability 1/|GL|.
// The span test reduces the candidate against a semi-echelon basis (u_j with
// distinct pivot bits p_j, each later u free of earlier pivots).  Columns are
// drawn directly because the device record stores columns; Gauss-Jordan on
// T = A^T then gives the rows of (A^T)^-1 = the columns of A^-1.
template <int MN>
RMFHT_HD void draw_map(uint64_t key, unsigned (&cols)[MN], unsigned (&icols)[MN], unsigned& b) {
    constexpr unsigned mask = (1u << MN) - 1u;
    Word16 rs(key);
    unsigned u[MN], piv[MN];
#pragma unroll
    for (int i = 0; i < MN; i++) {
        for (;;) {
            const unsigned v = rs.next() & mask;
            unsigned x = v;
#pragma unroll
            for (int j = 0; j < i; j++)
                if (x & piv[j]) x ^= u[j];
            if (x) {
                cols[i] = v;
                u[i] = x;
                piv[i] = x & (0u - x);
                break;
            }
        }
    }
    b = rs.next() & mask;
    unsigned t[MN];
#pragma unroll
    for (int k = 0; k < MN; k++) t[k] = cols[k] | (1u << (16 + k));
    gj_inverse_aug<MN>(t);  // A is invertible by construction
#pragma unroll
    for (int k = 0; k < MN; k++) icols[k] = t[k] >> 16;
}

// runtime-size draw_map (rare slots: map sizes below m-2)
RMFHT_HD void draw_map_rt(uint64_t key, int mn, unsigned* cols, unsigned* icols, unsigned& b) {
    const unsigned mask = (1u << mn) - 1u;
    Word16 rs(key);
    unsigned u[16], piv[16], t[16];
    for (int i = 0; i < mn; i++) {
        for (;;) {
            const unsigned v = rs.next() & mask;
            unsigned x = v;
            for (int j = 0; j < i; j++)
                if (x & piv[j]) x ^= u[j];
            if (x) {
                cols[i] = v;
                u[i] = x;
                piv[i] = x & (0u - x);
                break;
            }
        }
    }
    b = rs.next() & mask;
    for (int k = 0; k < mn; k++) t[k] = cols[k] | (1u << (16 + k));
    for (int c = 0; c < mn; c++) {
        const unsigned bit = 1u << c;
        for (int r = c + 1; r < mn; r++)
            if (~t[c] & t[r] & bit) t[c] ^= t[r];
        for (int r = 0; r < mn; r++)
            if (r != c && (t[r] & bit)) t[r] ^= t[c];
    }
    for (int k = 0; k < mn; k++) icols[k] = t[k] >> 16;
}

// A^-1 b = XOR of the columns of A^-1 selected by b
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
