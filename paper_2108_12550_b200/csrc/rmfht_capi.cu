// C ABI of the decoder (include/rmfht.h): plans bound to compile-time
// specialised kernels, host-side map expansion, stream-ordered launches.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rmfht_maps.cuh"
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
    if (p->force_generic) {
        if (rmfht_bind_generic(p) == 0) return 0;
        return fail(RMFHT_EUNSUPPORTED, "shape outside the generic kernel's limits (m <= 10, L <= 16)");
    }
    for (int c = 0; c < RMFHT_NCHUNKS; c++)
        if (tab[c](p) == 0) return 0;
    if (rmfht_bind_generic(p) == 0) return 0;
    char buf[160];
    snprintf(buf, sizeof buf, "RM(%d,%d) L=%d is outside the compiled shapes and the generic kernel's limits "
             "(m <= 10, L <= 16, workspace <= 220 KB)", p->r, p->m, p->L);
    return fail(RMFHT_EUNSUPPORTED, buf);
}

using rmfht_maps::expand_one;

struct SampleArgs {
    unsigned long long seed;
    long long frame0, B;
    int M, S, L, m, identity_root;
    signed char sizes[128];
};

// one record (2MG+2 uint16 = MG+1 words) built in registers
template <int MN, int MG>
__device__ __forceinline__ void draw_store(uint64_t key, uint32_t* o) {
    unsigned cols[MN], icols[MN], b;
    rmfht_maps::draw_map<MN>(key, cols, icols, b);
    // record halves: cols of A (MG), b, cols of A^-1 (MG), A^-1 b
    unsigned h[2 * MG + 2];
#pragma unroll
    for (int k = 0; k < MG; k++) {
        h[k] = k < MN ? cols[k < MN ? k : 0] : 0u;
        h[MG + 1 + k] = k < MN ? icols[k < MN ? k : 0] : 0u;
    }
    h[MG] = b;
    h[2 * MG + 1] = rmfht_maps::inv_shift<MN>(icols, b);
#pragma unroll
    for (int w = 0; w <= MG; w++) o[w] = h[2 * w] | (h[2 * w + 1] << 16);
}

// slots below MG-2 variables (r >= 5)
template <int MG>
__device__ __noinline__ void draw_store_rt(uint64_t key, int mn, uint16_t* o) {
    unsigned cols[16], icols[16], b;
    rmfht_maps::draw_map_rt(key, mn, cols, icols, b);
    unsigned cinv = 0;
    for (int k = 0; k < MG; k++) {
        o[k] = (uint16_t)(k < mn ? cols[k] : 0u);
        o[MG + 1 + k] = (uint16_t)(k < mn ? icols[k] : 0u);
        if (k < mn && ((b >> k) & 1u)) cinv ^= icols[k];
    }
    o[MG] = (uint16_t)b;
    o[2 * MG + 1] = (uint16_t)cinv;
}

// One thread per (frame, attempt, slot); a warp takes one slot of 32
// consecutive (frame, attempt) items, so its lanes draw maps of one size.
template <int MG>
__global__ void __launch_bounds__(256) sample_kernel(SampleArgs a, uint16_t* rec) {
    const long long items = a.B * (long long)a.M;
    const long long groups = (items + 31) / 32;
    const int lane = threadIdx.x & 31;
    auto one = [&](int s, long long item, long long f, int at) {
        uint16_t* o = rec + ((size_t)item * a.S + s) * (2 * MG + 2);
        const int mn = a.sizes[s];
        if (a.identity_root && at == 0 && s < a.L) {
            rmfht_maps::write_identity(mn, MG, nullptr, o);
            return;
        }
        const uint64_t key = rmfht_maps::slot_key(a.seed, f, at, s);
        uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
        if (mn == MG) draw_store<MG, MG>(key, o32);
        else if (mn == MG - 1 && MG > 1) draw_store<(MG > 1 ? MG - 1 : 1), MG>(key, o32);
        else if (mn == MG - 2 && MG > 2) draw_store<(MG > 2 ? MG - 2 : 1), MG>(key, o32);
        else draw_store_rt<MG>(key, mn, o);
    };
    if (groups * a.S < (1LL << 31)) {
        // 32-bit index arithmetic (the 64-bit divisions cost as much as a map's RNG)
        const unsigned total = (unsigned)(groups * a.S), S = (unsigned)a.S, M = (unsigned)a.M;
        const unsigned nw = gridDim.x * blockDim.x / 32;
        for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) / 32; w < total; w += nw) {
            const unsigned g = w / S, s = w - g * S;
            const unsigned item = g * 32 + lane;
            if (item >= (unsigned)items) continue;
            const unsigned fr = item / M;
            one((int)s, (long long)item, a.frame0 + fr, (int)(item - fr * M));
        }
        return;
    }
    const long long nwarps = (long long)gridDim.x * blockDim.x / 32;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; w < groups * a.S; w += nwarps) {
        const int s = (int)(w % a.S);
        const long long item = (w / a.S) * 32 + lane;
        if (item >= items) continue;
        one(s, item, a.frame0 + item / a.M, (int)(item % a.M));
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
    p->lockstep = (flags & RMFHT_NO_LOCKSTEP) ? 0 : 255;  // 255: one barrier for the whole CTA
    p->force_generic = (flags & RMFHT_GENERIC) ? 1 : 0;
    if (flags & RMFHT_LOCKSTEP_4) p->lockstep = 4;
    if (flags & RMFHT_LOCKSTEP_8) p->lockstep = 8;
    if (flags & RMFHT_TIE_FIX) p->tie_fix = 1;
    if (flags & RMFHT_NO_TIE_FIX) p->tie_fix = 0;
    if (flags & RMFHT_AUT_SSC) {
        // Aut-SSC (top_decoders.py:235-249): P = M SSC decodes, one map of m variables each
        if (L != 1 || !(flags & RMFHT_PERMUTATIONS)) {
            delete p;
            return fail(RMFHT_ECONFIG, "Aut-SSC plans take L = 1 and RMFHT_PERMUTATIONS (P = M decodes)");
        }
        p->aut = 1;
        p->fast = 0;
        p->sizes.assign(1, m);
        p->S = 1;
        const int rc = rmfht_bind_aut_ssc(p);
        if (rc != 0) {
            delete p;
            return fail(RMFHT_EUNSUPPORTED, "Aut-SSC supports m <= 10");
        }
        *out = p;
        return 0;
    }
    if (flags & RMFHT_AUT_SSC) {
        // Aut-SSC (top_decoders.py:235-249): P = M SSC decodes, one map of m variables each
        if (L != 1 || !(flags & RMFHT_PERMUTATIONS)) {
            delete p;
            return fail(RMFHT_ECONFIG, "Aut-SSC plans take L = 1 and RMFHT_PERMUTATIONS (P = M decodes)");
        }
        p->aut = 1;
        p->fast = 0;
        p->sizes.assign(1, m);
        p->S = 1;
        if (rmfht_bind_aut_ssc(p) != 0) {
            delete p;
            return fail(RMFHT_EUNSUPPORTED, "Aut-SSC supports m <= 10");
        }
        *out = p;
        return 0;
    }
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

int rmfht_plan_launches_per_call(const rmfht_plan* p) { return p ? (p->fast ? 2 : 1) : 0; }  // + 1 when sampled

int rmfht_plan_kernel(const rmfht_plan* p) { return p ? (p->aut ? 4 : p->fast ? 2 : (p->generic ? 3 : 1)) : 0; }

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
    const long long items = B * (long long)M;
#pragma omp parallel for schedule(static)
    for (long long item = 0; item < items; item++) {
        const long long f = frame0 + item / M;
        const int at = (int)(item % M);
        uint16_t* raw_i = raw ? raw + (size_t)item * S * (mg + 1) : nullptr;
        uint16_t* rec_i = rec ? rec + (size_t)item * S * (2 * mg + 2) : nullptr;
        for (int s = 0; s < S; s++) {
            const int mn = p->sizes[s];
            uint16_t* raw_s = raw_i ? raw_i + (size_t)s * (mg + 1) : nullptr;
            uint16_t* rec_s = rec_i ? rec_i + (size_t)s * (2 * mg + 2) : nullptr;
            if (identity_root && at == 0 && s < p->L)
                rmfht_maps::write_identity(mn, mg, raw_s, rec_s);
            else
                rmfht_maps::fill_slot_host_any(mn, rmfht_maps::slot_key(seed, f, at, s), mg, raw_s, rec_s);
        }
    }
    return 0;
}

int rmfht_sample_maps_device(const rmfht_plan* p, uint64_t seed, long long frame0, long long B, int identity_root,
                             uint16_t* d_rec, void* stream) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (B < 0 || !d_rec) return fail(RMFHT_EVALUE, "bad arguments");
    if (p->S > 128) return fail(RMFHT_EUNSUPPORTED, "more than 128 maps per attempt");
    if (B == 0 || p->S == 0) return 0;
    SampleArgs a;
    a.seed = seed;
    a.frame0 = frame0;
    a.B = B;
    a.M = p->M;
    a.S = p->S;
    a.L = p->L;
    a.m = p->m;
    a.identity_root = identity_root;
    for (int s = 0; s < p->S; s++) a.sizes[s] = (signed char)p->sizes[s];
    const long long warps = (B * (long long)p->M + 31) / 32 * p->S;
    long long blocks = (warps * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (p->m) {
#define RMFHT_SK(K) \
    case K:         \
        sample_kernel<K><<<(unsigned)blocks, 256, 0, st>>>(a, d_rec); \
        break;
        RMFHT_SK(2) RMFHT_SK(3) RMFHT_SK(4) RMFHT_SK(5) RMFHT_SK(6) RMFHT_SK(7) RMFHT_SK(8) RMFHT_SK(9)
        RMFHT_SK(10) RMFHT_SK(11) RMFHT_SK(12) RMFHT_SK(13) RMFHT_SK(14)
#undef RMFHT_SK
        default:
            return fail(RMFHT_EUNSUPPORTED, "map size");
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("sample launch: ") + cudaGetErrorString(e));
    return 0;
}

int rmfht_decode_launch_sampled(const rmfht_plan* p, const void* d_llr, uint64_t seed, long long frame0,
                                int identity_root, uint32_t* d_cw, void* d_pm, int32_t* d_attempt, int32_t* d_path,
                                long long B, void* stream) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (!p->perms) return rmfht_decode_launch(p, d_llr, nullptr, d_cw, d_pm, d_attempt, d_path, B, stream);
    auto* mp = const_cast<rmfht_plan*>(p);
    const size_t need = (size_t)B * p->M * p->S * (2 * p->m + 2) * sizeof(uint16_t);
    uint16_t* rec;
    {
        std::lock_guard<std::mutex> g(mp->work_mu);
        if (need > mp->maps_cap) {
            if (mp->maps_buf) cudaFree(mp->maps_buf);
            mp->maps_buf = nullptr;
            mp->maps_cap = 0;
            if (cudaMalloc(&mp->maps_buf, need) != cudaSuccess) return fail(RMFHT_ECUDA, "map table allocation failed");
            mp->maps_cap = need;
        }
        rec = static_cast<uint16_t*>(mp->maps_buf);
    }
    int rc = rmfht_sample_maps_device(p, seed, frame0, B, identity_root, rec, stream);
    if (rc) return rc;
    return rmfht_decode_launch(p, d_llr, rec, d_cw, d_pm, d_attempt, d_path, B, stream);
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
