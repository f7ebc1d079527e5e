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

// Table semantics (host and device): for each (frame f, attempt a), the
// slots are filled class by class (a class = a run of slots with the same
// map size, SURVEY §8(c) consumption order).  Candidate j of class c is
// drawn from a counter-based stream keyed by (seed, f, a, c, j); invertible
// candidates fill the class's slots in candidate order — the reference's own
// rule (sample_affine_batch, automorphism.py:144-161: draw a batch, keep the
// invertible ones in order).  With identity_root, attempt 0's L root slots
// are the identity ("decoder 0 = identity") and are not drawn.
RMFHT_HD uint64_t cand_key(uint64_t seed, long long f, int a, int c, long long j) {
    uint64_t st = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull);
    st += ((uint64_t)a << 24) + ((uint64_t)c << 16);
    uint64_t k = splitmix64(st);
    k ^= (uint64_t)j * 0xC2B2AE3D27D4EB4Full;
    return splitmix64(k);
}

// candidate j: row masks and shift; true if A is invertible (then inv holds A^-1)
template <int MN>
RMFHT_HD bool candidate(uint64_t key, unsigned (&rows)[MN], unsigned (&inv)[MN], unsigned& b) {
    uint64_t st = key;
    constexpr unsigned mask = (1u << MN) - 1u;
    uint64_t w = 0;
#pragma unroll
    for (int r = 0; r < MN; r++) {
        if (r % 4 == 0) w = splitmix64(st);
        rows[r] = (unsigned)(w >> (16 * (r % 4))) & mask;
    }
    b = (unsigned)(splitmix64(st) & mask);
    return gj_inverse<MN>(rows, inv);
}

template <int MN>
RMFHT_HD void write_map(const unsigned (&rows)[MN], const unsigned (&inv)[MN], unsigned b, int mg, uint16_t* raw,
                        uint16_t* rec) {
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

// host: one class of one (frame, attempt), sequential candidate order
template <int MN>
inline void fill_class_host(uint64_t seed, long long f, int a, int c, int s0, int cnt, int mg, uint16_t* raw,
                            uint16_t* rec) {
    int filled = 0;
    for (long long j = 0; filled < cnt; j++) {
        unsigned rows[MN], inv[MN], b;
        if (!candidate<MN>(cand_key(seed, f, a, c, j), rows, inv, b)) continue;
        const int s = s0 + filled++;
        write_map<MN>(rows, inv, b, mg, raw ? raw + (size_t)s * (mg + 1) : nullptr,
                      rec ? rec + (size_t)s * (2 * mg + 2) : nullptr);
    }
}

inline void fill_class_host_any(int mn, uint64_t seed, long long f, int a, int c, int s0, int cnt, int mg,
                                uint16_t* raw, uint16_t* rec) {
    switch (mn) {
#define RMFHT_FC(K)                                                   \
    case K:                                                           \
        fill_class_host<K>(seed, f, a, c, s0, cnt, mg, raw, rec); \
        break;
        RMFHT_FC(1) RMFHT_FC(2) RMFHT_FC(3) RMFHT_FC(4) RMFHT_FC(5) RMFHT_FC(6) RMFHT_FC(7)
        RMFHT_FC(8) RMFHT_FC(9) RMFHT_FC(10) RMFHT_FC(11) RMFHT_FC(12) RMFHT_FC(13) RMFHT_FC(14)
#undef RMFHT_FC
        default:
            break;
    }
}

}  // namespace rmfht_maps
