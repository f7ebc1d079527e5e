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

// Gauss-Jordan on [A | I] over GF(2) with compile-time size: rows[] are the
// row masks of A; on success inv[] holds the row masks of A^-1.
template <int MN>
RMFHT_HD bool gj_inverse(const unsigned (&rows_in)[MN], unsigned (&inv)[MN]) {
    unsigned rows[MN];
#pragma unroll
    for (int r = 0; r < MN; r++) {
        rows[r] = rows_in[r];
        inv[r] = 1u << r;
    }
#pragma unroll
    for (int c = 0; c < MN; c++) {
        // pivot: first row >= c with bit c set, swapped into row c
        bool found = false;
#pragma unroll
        for (int r = c; r < MN; r++) {
            const bool take = !found && ((rows[r] >> c) & 1u);
            if (take) {
                const unsigned t = rows[c];
                rows[c] = rows[r];
                rows[r] = t;
                const unsigned ti = inv[c];
                inv[c] = inv[r];
                inv[r] = ti;
            }
            found = found || take;
        }
        if (!found) return false;
#pragma unroll
        for (int r = 0; r < MN; r++)
            if (r != c && ((rows[r] >> c) & 1u)) {
                rows[r] ^= rows[c];
                inv[r] ^= inv[c];
            }
    }
    return true;
}

// uniform (A, b) in GL(MN,2) x F_2^MN by rejection on random row masks
// (the reference's rule, automorphism.py:127-161), from a counter-based
// stream; writes the raw map and its device record
template <int MN>
RMFHT_HD void sample_map(uint64_t key, int mg, uint16_t* raw, uint16_t* rec) {
    uint64_t st = key;
    constexpr unsigned mask = (1u << MN) - 1u;
    unsigned rows[MN], inv[MN];
    for (;;) {
        uint64_t w = 0;
#pragma unroll
        for (int r = 0; r < MN; r++) {
            if (r % 4 == 0) w = splitmix64(st);
            rows[r] = (unsigned)(w >> (16 * (r % 4))) & mask;
        }
        if (gj_inverse<MN>(rows, inv)) break;
    }
    const unsigned b = (unsigned)(splitmix64(st) & mask);
    if (raw) {
        for (int k = 0; k <= mg; k++) raw[k] = 0;
#pragma unroll
        for (int r = 0; r < MN; r++) raw[r] = (uint16_t)rows[r];
        raw[mg] = (uint16_t)b;
    }
    if (rec) {
        for (int k = 0; k < 2 * mg + 2; k++) rec[k] = 0;
        unsigned cinv = 0;
#pragma unroll
        for (int k = 0; k < MN; k++) {
            unsigned col = 0, icol = 0;
#pragma unroll
            for (int r = 0; r < MN; r++) {
                col |= ((rows[r] >> k) & 1u) << r;
                icol |= ((inv[r] >> k) & 1u) << r;
            }
            rec[k] = (uint16_t)col;
            rec[mg + 1 + k] = (uint16_t)icol;
            if ((b >> k) & 1u) cinv ^= icol;
        }
        rec[mg] = (uint16_t)b;
        rec[2 * mg + 1] = (uint16_t)cinv;
    }
}

// entry (frame f, attempt a, slot s) of a table: the identity for attempt
// 0's L root maps when identity_root ("decoder 0 = identity"), else a fresh
// draw keyed by (seed, f, a, s).  raw and/or rec may be null.
template <int MN>
RMFHT_HD void table_entry_t(uint64_t seed, long long f, int a, int s, int L, int mg, int identity_root, uint16_t* raw,
                            uint16_t* rec) {
    if (identity_root && a == 0 && s < L) {
        if (raw) {
            for (int k = 0; k <= mg; k++) raw[k] = 0;
            for (int k = 0; k < MN; k++) raw[k] = (uint16_t)(1u << k);
        }
        if (rec) {
            for (int k = 0; k < 2 * mg + 2; k++) rec[k] = 0;
            for (int k = 0; k < MN; k++) {
                rec[k] = (uint16_t)(1u << k);
                rec[mg + 1 + k] = (uint16_t)(1u << k);
            }
        }
        return;
    }
    const uint64_t key = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull);
    uint64_t st = key + ((uint64_t)a << 20) + (uint64_t)s;
    sample_map<MN>(splitmix64(st), mg, raw, rec);
}

RMFHT_HD void table_entry(uint64_t seed, long long f, int a, int s, int L, int mn, int mg, int identity_root,
                          uint16_t* raw, uint16_t* rec) {
    switch (mn) {
#define RMFHT_TE(K)                                                              \
    case K:                                                                      \
        table_entry_t<K>(seed, f, a, s, L, mg, identity_root, raw, rec); \
        break;
        RMFHT_TE(1) RMFHT_TE(2) RMFHT_TE(3) RMFHT_TE(4) RMFHT_TE(5) RMFHT_TE(6) RMFHT_TE(7)
        RMFHT_TE(8) RMFHT_TE(9) RMFHT_TE(10) RMFHT_TE(11) RMFHT_TE(12) RMFHT_TE(13) RMFHT_TE(14)
#undef RMFHT_TE
        default:
            break;
    }
}

}  // namespace rmfht_maps
