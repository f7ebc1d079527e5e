// C ABI of the decoder (include/rmfht.h): plans bound to compile-time
// specialised kernels, host-side map expansion, stream-ordered launches.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rmfht_plan.h"

namespace rmfht_internal {
thread_local std::string g_err;
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace rmfht_internal

using rmfht_internal::fail;
using rmfht_internal::g_err;

namespace {

int bind_any(rmfht_plan* p) {
    using Binder = int (*)(rmfht_plan*);
    static const Binder f32[] = {rmfht_bind_float_0, rmfht_bind_float_1, rmfht_bind_float_2, rmfht_bind_float_3};
    static const Binder f64[] = {rmfht_bind_double_0, rmfht_bind_double_1, rmfht_bind_double_2,
                                 rmfht_bind_double_3};
    const Binder* tab = p->dtype == RMFHT_F64 ? f64 : f32;
    for (int c = 0; c < RMFHT_NCHUNKS; c++)
        if (tab[c](p) == 0) return 0;
    char buf[160];
    snprintf(buf, sizeof buf, "no kernel compiled for RM(%d,%d) L=%d", p->r, p->m, p->L);
    return fail(RMFHT_EUNSUPPORTED, buf);
}

// raw (row masks, b) -> record (columns, b, inverse columns, A^-1 b)
int expand_one(const uint16_t* raw, int mn, int mg, uint16_t* rec) {
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
    for (int c = 0; c < mn; c++) {  // Gauss-Jordan over GF(2)
        int piv = -1;
        for (int r = c; r < mn; r++)
            if (rows[r] >> c & 1u) { piv = r; break; }
        if (piv < 0) return -1;
        std::swap(rows[c], rows[piv]);
        std::swap(inv[c], inv[piv]);
        for (int r = 0; r < mn; r++)
            if (r != c && (rows[r] >> c & 1u)) { rows[r] ^= rows[c]; inv[r] ^= inv[c]; }
    }
    std::memset(rec, 0, sizeof(uint16_t) * (2 * mg + 2));
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


// counter-based generator: one independent stream per (seed, frame, attempt, slot)
inline uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// uniform (A, b) in GL(mn,2) x F_2^mn by rejection on random row masks
// (the reference's rule, automorphism.py:127-161), written as a raw record
void sample_raw(uint64_t key, int mn, int mg, uint16_t* raw) {
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
                if (t[r] >> c & 1u) { piv = r; break; }
            if (piv < 0) { ok = false; break; }
            std::swap(t[c], t[piv]);
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
}  // namespace

extern "C" {

int rmfht_version(void) { return 1; }

const char* rmfht_last_error(void) { return g_err.c_str(); }

int rmfht_plan_create(int r, int m, int L, int M, int flags, int dtype, rmfht_plan** out) {
    if (!out) return fail(RMFHT_EVALUE, "out is NULL");
    *out = nullptr;
    if (m < 2 || m > 14) return fail(RMFHT_ECONFIG, "m=" + std::to_string(m) + " outside supported range [2, 14]");
    if (r < 1 || r > m - 1) return fail(RMFHT_ECONFIG, "r=" + std::to_string(r) + " must satisfy 1 <= r <= m-1");
    if (L < 1 || M < 1) return fail(RMFHT_ECONFIG, "L, M and P must all be >= 1");
    if (dtype != RMFHT_F32 && dtype != RMFHT_F64) return fail(RMFHT_ECONFIG, "dtype must be RMFHT_F32 or RMFHT_F64");
    auto* p = new rmfht_plan();
    p->r = r;
    p->m = m;
    p->L = L;
    p->perms = (flags & RMFHT_PERMUTATIONS) ? 1 : 0;
    p->M = p->perms ? M : 1;
    p->dtype = dtype;
    p->tie_fix = dtype == RMFHT_F32 ? 1 : 0;
    p->fast = (dtype == RMFHT_F32 && !(flags & RMFHT_REFERENCE_ORDER)) ? 1 : 0;
    p->lockstep = (flags & RMFHT_NO_LOCKSTEP) ? 0 : 16;
    if (flags & RMFHT_LOCKSTEP_4) p->lockstep = 4;
    if (flags & RMFHT_LOCKSTEP_8) p->lockstep = 8;
    if (flags & RMFHT_TIE_FIX) p->tie_fix = 1;
    if (flags & RMFHT_NO_TIE_FIX) p->tie_fix = 0;
    if (p->perms) {
        for (int l = 0; l < L; l++) p->sizes.push_back(m);
        if (m - r >= 2)
            for (int i = 0; i <= r - 2; i++)
                for (int t = 0; t < 2 * L; t++) p->sizes.push_back(m - i);
    }
    p->S = (int)p->sizes.size();
    const int rc = bind_any(p);
    if (rc != 0) {
        delete p;
        return rc;
    }
    *out = p;
    return 0;
}

void rmfht_plan_destroy(rmfht_plan* plan) { delete plan; }

int rmfht_plan_maps_per_attempt(const rmfht_plan* p) { return p ? p->S : fail(RMFHT_EVALUE, "plan is NULL"); }

int rmfht_plan_map_sizes(const rmfht_plan* p, int* sizes) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    for (int s = 0; s < p->S; s++) sizes[s] = p->sizes[s];
    return p->S;
}

int rmfht_plan_record_u16(const rmfht_plan* p) { return p ? 2 * p->m + 2 : fail(RMFHT_EVALUE, "plan is NULL"); }

int rmfht_plan_launches_per_call(const rmfht_plan* p) { return p ? (p->fast ? 2 : 1) : 0; }

int rmfht_plan_kernel(const rmfht_plan* p) { return p ? (p->fast ? 2 : 1) : 0; }

int rmfht_expand_maps(const rmfht_plan* p, const uint16_t* raw, uint16_t* rec, long long count) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (p->S == 0) return count == 0 ? 0 : fail(RMFHT_EVALUE, "plan consumes no maps");
    const int mg = p->m;
    for (long long i = 0; i < count; i++) {
        const int mn = p->sizes[i % p->S];
        if (expand_one(raw + i * (mg + 1), mn, mg, rec + i * (2 * mg + 2)) != 0) {
            char buf[160];
            snprintf(buf, sizeof buf, "map %lld (slot %lld, %d variables) is not an invertible affine map", i,
                     i % p->S, mn);
            return fail(RMFHT_EVALUE, buf);
        }
    }
    return 0;
}


int rmfht_sample_maps(const rmfht_plan* p, uint64_t seed, long long frame0, long long B, int identity_root,
                      uint16_t* raw, uint16_t* rec) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (B < 0) return fail(RMFHT_EVALUE, "negative batch");
    const int mg = p->m, S = p->S, M = p->M;
    const long long total = B * (long long)M * S;
    int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (long long i = 0; i < total; i++) {
        const long long f = frame0 + i / ((long long)M * S);
        const int a = (int)((i / S) % M), s = (int)(i % S);
        uint16_t tmp[16], rtmp[32];
        uint16_t* r = raw ? raw + i * (mg + 1) : tmp;
        if (identity_root && a == 0 && s < p->L) {
            for (int k = 0; k < mg; k++) r[k] = (uint16_t)(1u << k);
            r[mg] = 0;
        } else {
            uint64_t key = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)f * 0x9E3779B97F4A7C15ull);
            uint64_t st = key + ((uint64_t)a << 20) + (uint64_t)s;
            const uint64_t k2 = splitmix64(st);
            sample_raw(k2, p->sizes[s], mg, r);
        }
        if (rec && expand_one(r, p->sizes[s], mg, rec ? rec + i * (2 * mg + 2) : rtmp) != 0) err |= 1;
    }
    if (err) return fail(RMFHT_EVALUE, "internal: sampled a singular map");
    return 0;
}

int rmfht_decode_launch_diag(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm,
                             int32_t* att, int32_t* path, void* att_pm, uint32_t* att_cw, long long B,
                             void* stream) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (B < 0) return fail(RMFHT_EVALUE, "negative batch");
    if (B > 0 && (!llr || !cw || !pm || !att || !path || (p->perms && !maps)))
        return fail(RMFHT_EVALUE, "NULL buffer");
    return p->launch(p, llr, maps, cw, pm, att, path, att_pm, att_cw, B, static_cast<cudaStream_t>(stream));
}

int rmfht_decode_launch(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm,
                        int32_t* att, int32_t* path, long long B, void* stream) {
    return rmfht_decode_launch_diag(p, llr, maps, cw, pm, att, path, nullptr, nullptr, B, stream);
}

}  // extern "C"
