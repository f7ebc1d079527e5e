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
    for (int c = 0; c < RMFHT_NCHUNKS; c++)
        if (tab[c](p) == 0) return 0;
    char buf[160];
    snprintf(buf, sizeof buf, "no kernel compiled for RM(%d,%d) L=%d", p->r, p->m, p->L);
    return fail(RMFHT_EUNSUPPORTED, buf);
}

using rmfht_maps::expand_one;

struct SampleArgs {
    unsigned long long seed;
    long long frame0, B;
    int M, S, L, m, identity_root;
    signed char sizes[128];
};

// one thread per (frame, attempt, slot): the same draw as rmfht_sample_maps
template <int MG>
__global__ void __launch_bounds__(256) sample_kernel(SampleArgs a, uint16_t* rec) {
    const long long total = a.B * (long long)a.M * a.S;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long f = a.frame0 + i / ((long long)a.M * a.S);
        const int at = (int)((i / a.S) % a.M), sl = (int)(i % a.S);
        uint16_t r[2 * MG + 2];
        const int mn = a.sizes[sl];
        if (mn == MG)
            rmfht_maps::table_entry_t<MG>(a.seed, f, at, sl, a.L, MG, a.identity_root, nullptr, r);
        else
            rmfht_maps::table_entry(a.seed, f, at, sl, a.L, mn, MG, a.identity_root, nullptr, r);
        uint32_t* o = reinterpret_cast<uint32_t*>(rec + i * (2 * MG + 2));  // 2*MG+2 is even: 4-byte aligned
#pragma unroll
        for (int k = 0; k < MG + 1; k++) o[k] = (uint32_t)r[2 * k] | ((uint32_t)r[2 * k + 1] << 16);
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

int rmfht_plan_launches_per_call(const rmfht_plan* p) { return p ? (p->fast ? 2 : 1) : 0; }  // + 1 when sampled

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
        rmfht_maps::table_entry(seed, f, a, s, p->L, p->sizes[s], mg, identity_root, raw ? raw + i * (mg + 1) : nullptr,
                                rec ? rec + i * (2 * mg + 2) : nullptr);
    }
    (void)err;
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
    const long long total = B * (long long)p->M * p->S;
    long long blocks = (total + 255) / 256;
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
