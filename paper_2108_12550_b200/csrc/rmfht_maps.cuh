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

// uniform (A, b) in GL(mn,2) x F_2^mn by rejection on random row masks
// (the reference's rule, automorphism.py:127-161), from a counter-based stream
RMFHT_HD void sample_raw(uint64_t key, int mn, int mg, uint16_t* raw) {
    uint64_t st = key;
    const unsigned mask = (1u << mn) - 1u;
    for (;;) {
        unsigned rows[16];
        uint64_t w = 0;
        for (int r = 0; r < mn; r++) {
            if (r % 4 == 0) w = splitmix64(st);
            rows[r] = (unsigned)(w >> (16 * (r % 4))) & mask;
        }
        unsigned t[16];
        for (int r = 0; r < mn; r++) t[r] = rows[r];
        bool ok = true;
        for (int c = 0; c < mn && ok; c++) {
            int piv = -1;
            for (int r = c; r < mn; r++)
                if (t[r] >> c & 1u) {
                    piv = r;
                    break;
                }
            if (piv < 0) {
                ok = false;
                break;
            }
            const unsigned x = t[c];
            t[c] = t[piv];
            t[piv] = x;
            for (int r = c + 1; r < mn; r++)
                if (t[r] >> c & 1u) t[r] ^= t[c];
        }
        if (!ok) continue;
        for (int k = 0; k <= mg; k++) raw[k] = 0;
        for (int r = 0; r < mn; r++) raw[r] = (uint16_t)rows[r];
        raw[mg] = (uint16_t)(splitmix64(st) & mask);
        return;
    }
}

// map of (frame f, attempt a, slot s): the identity for attempt 0's L root
// maps when identity_root ("decoder 0 = identity"), else a fresh draw keyed
// by (seed, f, a, s)
RMFHT_HD void table_entry(uint64_t seed, long long f, int a, int s, int L, int mn, int mg, int identity_root,
                          uint16_t* raw) {
    if (identity_root && a == 0 && s < L) {
        for (int k = 0; k < mg; k++) raw[k] = (uint16_t)(1u << k);
        raw[mg] = 0;
        return;
    }
    const uint64_t key = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull);
    uint64_t st = key + ((uint64_t)a << 20) + (uint64_t)s;
    sample_raw(splitmix64(st), mn, mg, raw);
}

}  // namespace rmfht_maps
