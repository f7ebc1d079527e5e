// C ABI of the decoder (include/rmfht.h): plans bound to compile-time
// specialised kernels, host-side map expansion, stream-ordered launches.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
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

// one record (2MG+2 uint16 = MG+1 words): word w handed to put(w, value),
// then the columns of A^-1 and A^-1 b as half words put16(half, value) — a
// basis word's pivot names the column it holds (draw_map_basis), so the
// columns land at their half-word slots with no register permutation
template <int MN, int MG, typename Put, typename Put16>
__device__ __forceinline__ void draw_store(uint64_t key, Put&& put, Put16&& put16) {
    unsigned cols[MN], ub[MN], pv[MN], b;
    rmfht_maps::draw_map_basis<MN, rmfht_maps::Word16p>(key, cols, ub, pv, b);
    // record halves: cols of A (MG), b, cols of A^-1 (MG), A^-1 b; whole
    // words up to half MG, half words after (never both on one location)
    unsigned h[MG + 2];
#pragma unroll
    for (int k = 0; k < MG + 2; k++) h[k] = 0u;
#pragma unroll
    for (int k = 0; k < MN; k++) h[k] = cols[k];
    h[MG] = b;
    constexpr int WF = (MG + 1) / 2;  // words made of halves 0 .. 2 WF - 1 <= MG
#pragma unroll
    for (int w = 0; w < WF; w++) put(w, h[2 * w] | (h[2 * w + 1] << 16));
    if constexpr (2 * WF == MG) put16(MG, b);
#pragma unroll
    for (int k = MN; k < MG; k++) put16(MG + 1 + k, 0u);
    unsigned c = 0u;
#pragma unroll
    for (int j = 0; j < MN; j++) {
        const unsigned coef = ub[j] >> 16;
        put16(MG + 1 + (__ffs(pv[j]) - 1), coef);
        rmfht_maps::xor_if(c, b, pv[j], coef);  // A^-1 b = sum over the set bits k of b of column k
    }
    put16(2 * MG + 1, c);
}

// slots below MG-2 variables (r >= 5)
template <int MG>
__device__ __noinline__ void draw_store_rt(uint64_t key, int mn, uint32_t* o) {
    unsigned cols[16], icols[16], b;
    rmfht_maps::draw_map_rt(key, mn, cols, icols, b);
    unsigned cinv = 0, h[2 * MG + 2];
    for (int k = 0; k < MG; k++) {
        h[k] = k < mn ? cols[k] : 0u;
        h[MG + 1 + k] = k < mn ? icols[k] : 0u;
        if (k < mn && ((b >> k) & 1u)) cinv ^= icols[k];
    }
    h[MG] = b;
    h[2 * MG + 1] = cinv;
    for (int w = 0; w <= MG; w++) o[w] = h[2 * w] | (h[2 * w + 1] << 16);
}

// A CTA draws the records of G consecutive (frame, attempt) items: warp w
// takes slots w, w + 8, ... with one lane per item (a warp's lanes draw maps
// of one size), the records are staged in shared memory in their global
// order (one pad word per 32 against bank conflicts) and leave in contiguous
// 32-bit stores — the item-major record layout made per-lane stores
// S x 40 B apart, which throttled the store pipe.
template <int MG>
__global__ void __launch_bounds__(256) sample_kernel(SampleArgs a, uint32_t* rec, int G) {
    extern __shared__ uint32_t stage[];
    constexpr int W = MG + 1;  // words per record
    const long long items = a.B * (long long)a.M;
    const int S = a.S, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long groups = (items + G - 1) / G;
    for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
        const long long item0 = g * G;
        const int nit = (int)(items - item0 < G ? items - item0 : G);
        if (lane < nit) {
            const long long item = item0 + lane;
            long long f;
            int at;
            if (item < (1LL << 31)) {
                const unsigned q = (unsigned)item / (unsigned)a.M;
                f = q;
                at = (int)((unsigned)item - q * (unsigned)a.M);
            } else {
                f = item / a.M;
                at = (int)(item % a.M);
            }
            f += a.frame0;
            for (int s = warp; s < S; s += nw) {
                const unsigned o0 = (unsigned)(lane * S + s) * W;
                auto put = [&](int w, unsigned v) {
                    const unsigned o = o0 + w;
                    stage[o + (o >> 5)] = v;
                };
                auto put16 = [&](int hw, unsigned v) {
                    const unsigned o = o0 + (unsigned)(hw >> 1);
                    reinterpret_cast<uint16_t*>(stage)[2 * (o + (o >> 5)) + (hw & 1)] = (uint16_t)v;
                };
                const int mn = a.sizes[s];
                if (a.identity_root && at == 0 && s < a.L) {
                    unsigned h[2 * MG + 2];
#pragma unroll
                    for (int k = 0; k < 2 * MG + 2; k++) h[k] = 0u;
                    for (int k = 0; k < mn; k++) h[k] = h[MG + 1 + k] = 1u << k;
#pragma unroll
                    for (int w = 0; w < W; w++) put(w, h[2 * w] | (h[2 * w + 1] << 16));
                    continue;
                }
                const uint64_t key = rmfht_maps::slot_key(a.seed, f, at, s);
                if (mn == MG) draw_store<MG, MG>(key, put, put16);
                else if (mn == MG - 1 && MG > 1) draw_store<(MG > 1 ? MG - 1 : 1), MG>(key, put, put16);
                else if (mn == MG - 2 && MG > 2) draw_store<(MG > 2 ? MG - 2 : 1), MG>(key, put, put16);
                else {
                    uint32_t t[W];
                    draw_store_rt<MG>(key, mn, t);
#pragma unroll
                    for (int w = 0; w < W; w++) put(w, t[w]);
                }
            }
        }
        __syncthreads();
        uint32_t* dst = rec + (size_t)item0 * S * W;
        const int T = nit * S * W;
        for (int o = threadIdx.x; o < T; o += blockDim.x) dst[o] = stage[o + (o >> 5)];
        __syncthreads();
    }
}

// One thread per map: thread t of the launch draws task t = (item, slot)
// = (t / S, t % S) of the table (item-major, the record order in memory), so
// the 32 lanes of a warp draw 32 consecutive records and every thread has
// exactly one draw — no idle warps, no CTA barrier.  A warp stages its 32
// records in its own shared-memory row in memory order (record stride W
// words: the per-lane stores take a two-way bank conflict for even W, the
// write-out needs no index arithmetic) and writes them out as 32 x W
// contiguous words (coalesced 32-bit stores).  Same draws as sample_kernel (draw_store: bit-identical
// tables).
template <int MG>
__global__ void __launch_bounds__(256) sample_kernel_flat(SampleArgs a, uint32_t* rec) {
    constexpr int W = MG + 1;
    __shared__ uint32_t stage[8][32 * W];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long tasks = a.B * (long long)a.M * a.S;
    uint32_t* st = stage[warp];
    for (long long t0 = ((long long)blockIdx.x * 8 + warp) * 32; t0 < tasks; t0 += (long long)gridDim.x * 256) {
        const long long t = t0 + lane;
        if (t < tasks) {
            long long item;
            int s;
            if (t < (1LL << 31)) {
                const unsigned q = (unsigned)t / (unsigned)a.S;
                item = q;
                s = (int)((unsigned)t - q * (unsigned)a.S);
            } else {
                item = t / a.S;
                s = (int)(t % a.S);
            }
            long long f;
            int at;
            if (item < (1LL << 31)) {
                const unsigned q = (unsigned)item / (unsigned)a.M;
                f = q;
                at = (int)((unsigned)item - q * (unsigned)a.M);
            } else {
                f = item / a.M;
                at = (int)(item % a.M);
            }
            f += a.frame0;
            uint32_t* dst = st + lane * W;
            auto put = [&](int w, unsigned v) { dst[w] = v; };
            auto put16 = [&](int hw, unsigned v) { reinterpret_cast<uint16_t*>(dst)[hw] = (uint16_t)v; };
            const int mn = a.sizes[s];
            if (a.identity_root && at == 0 && s < a.L) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    const unsigned lo = (2 * w < mn) ? 1u << (2 * w) : 0u;
                    const unsigned hi = (2 * w + 1 < mn) ? 1u << (2 * w + 1) : 0u;
                    dst[w] = (2 * w < MG ? lo : 0u) | ((2 * w + 1 < MG ? hi : 0u) << 16);
                }
                for (int k = 0; k < MG; k++) put16(MG + 1 + k, k < mn ? 1u << k : 0u);
                put16(2 * MG + 1, 0u);
                if (MG % 2 == 0) put16(MG, 0u);
            } else {
                const uint64_t key = rmfht_maps::slot_key(a.seed, f, at, s);
                if (mn == MG) draw_store<MG, MG>(key, put, put16);
                else if (mn == MG - 1 && MG > 1) draw_store<(MG > 1 ? MG - 1 : 1), MG>(key, put, put16);
                else if (mn == MG - 2 && MG > 2) draw_store<(MG > 2 ? MG - 2 : 1), MG>(key, put, put16);
                else {
                    uint32_t tt[W];
                    draw_store_rt<MG>(key, mn, tt);
#pragma unroll
                    for (int w = 0; w < W; w++) put(w, tt[w]);
                }
            }
        }
        __syncwarp();
        const long long n = tasks - t0 < 32 ? tasks - t0 : 32;  // records of this warp
        uint32_t* out = rec + t0 * W;
#pragma unroll
        for (int j = 0; j < W; j++) {
            const int o = j * 32 + lane;  // word o of the warp's n * W words
            if (o < n * W) out[o] = st[o];
        }
        __syncwarp();
    }
}

}  // namespace

extern "C" {

int rmfht_version(void) { return 2; }  // 2: caller-owned workspace (rmfht_workspace_bytes)

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
    // A/B experiments only: warps per lock-step group of the throughput kernel
    if (const char* env = std::getenv("RMFHT_LOCKSTEP_GROUP")) p->lockstep = std::atoi(env) & 0xff;
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
    if (p->perms) {
        for (int l = 0; l < L; l++) p->sizes.push_back(m);
        if (m - r >= 2)
            for (int i = 0; i <= r - 2; i++)
                for (int t = 0; t < 2 * L; t++) p->sizes.push_back(m - i);
    }
    p->S = (int)p->sizes.size();
    // tests only: a smaller per-launch item limit exercises the chunked launch path
    if (const char* env = std::getenv("RMFHT_MAX_ITEMS")) {
        const long long v = std::atoll(env);
        if (v > 0 && v < p->max_items) p->max_items = v;
    }
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

int rmfht_plan_launches_per_call(const rmfht_plan* p) { return p ? (p->fast && !p->lane && !p->pair ? 2 : 1) : 0; }  // + 1 when sampled

int rmfht_plan_kernel(const rmfht_plan* p) {
    return p ? (p->aut ? 4 : p->lane ? 5 : p->pair ? 6 : p->grp ? 7 : p->fast ? 2 : (p->generic ? 3 : 1)) : 0;
}

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
    if (reinterpret_cast<uintptr_t>(d_rec) & 3u) return fail(RMFHT_EVALUE, "d_rec must be 4-byte aligned");
    // items per CTA group: 32 (one per lane) unless the staged records exceed 48 KB
    const int W = p->m + 1;
    int G = 32;
    auto stage_bytes = [&](int g) { const size_t t = (size_t)g * p->S * W; return (t + t / 32 + 1) * 4; };
    while (G > 1 && stage_bytes(G) > 48 * 1024) G /= 2;
    // warps per CTA: the largest divisor of S up to 8, so every warp draws
    // the same number of slots (S = 12 on 8 warps left 4 warps idle half the time)
    int nw = 1;
    for (int d = 8; d >= 1; d--)
        if (p->S % d == 0) { nw = d; break; }
    const long long groups = (B * (long long)p->M + G - 1) / G;
    long long blocks = groups < 148 * 16 ? groups : 148 * 16;
    const size_t smem = stage_bytes(G);
    // one thread per map (sample_kernel_flat) when every slot has m variables:
    // consecutive lanes draw consecutive slots, so mixed slot sizes (r >= 3)
    // would diverge within a warp — those keep the slot-per-warp kernel.
    // Measured (ncu launch lists): RM(2,9) L4 M20 0.321 -> 0.286 ms, M = 512
    // L = 1 0.091 -> 0.064 ms, Aut-SSC P512 0.120 -> 0.045 ms; RM(3,7) L8 M32
    // 0.568 ms slot-per-warp vs 0.899 ms flat.  RMFHT_SAMPLER=group|flat
    // forces one (A/B only).
    bool flat = true;
    for (int s = 0; s < p->S; s++) flat = flat && p->sizes[s] == p->m;
    if (const char* sv = std::getenv("RMFHT_SAMPLER")) flat = sv[0] == 'f';
    const long long warps_needed = (B * (long long)p->M * p->S + 31) / 32;
    const long long fblocks_all = (warps_needed + 7) / 8;
    const long long fblocks = fblocks_all < (long long)148 * 32 ? fblocks_all : (long long)148 * 32;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t* d_rec32 = reinterpret_cast<uint32_t*>(d_rec);
    switch (p->m) {
#define RMFHT_SK(K) \
    case K:         \
        if (flat) sample_kernel_flat<K><<<(unsigned)fblocks, 256, 0, st>>>(a, d_rec32); \
        else sample_kernel<K><<<(unsigned)blocks, 32 * nw, smem, st>>>(a, d_rec32, G); \
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

// caller-owned workspace: [map table (sampled launches)][per-attempt records of the throughput kernel]
static size_t table_bytes(const rmfht_plan* p, long long B) {
    return rmfht_align256((size_t)B * p->M * p->S * (2 * p->m + 2) * sizeof(uint16_t));
}
static size_t kernel_work_bytes(const rmfht_plan* p, long long B) {
    if (!p->work_per_item || B <= 0) return 0;
    const long long chunk = rmfht_chunk_frames(p);
    const long long B0 = B < chunk ? B : chunk;
    return rmfht_align256((size_t)B0 * p->M * p->work_per_item);
}

long long rmfht_workspace_bytes(const rmfht_plan* p, long long B, int sampled) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (B < 0) return fail(RMFHT_EVALUE, "negative batch");
    if (B > (1LL << 40) / ((long long)p->M * (p->S + 1))) return fail(RMFHT_EVALUE, "batch too large");
    size_t t = kernel_work_bytes(p, B);
    if (sampled && p->perms) t += table_bytes(p, B);
    return (long long)t;
}

static int check_work(const rmfht_plan* p, long long B, int sampled, const void* work, long long work_bytes) {
    const long long need = rmfht_workspace_bytes(p, B, sampled);
    if (need < 0) return (int)need;
    if (need > 0 && (!work || work_bytes < need)) {
        char buf[160];
        snprintf(buf, sizeof buf, "workspace of %lld bytes required (rmfht_workspace_bytes), %lld given%s", need,
                 work_bytes, work ? "" : " (NULL)");
        return fail(RMFHT_EVALUE, buf);
    }
    if (need > 0 && (reinterpret_cast<uintptr_t>(work) & 255u)) return fail(RMFHT_EVALUE, "d_work must be 256-byte aligned");
    return 0;
}

static int check_io(const rmfht_plan* p, const void* llr, const uint16_t* maps, const uint32_t* cw, const void* pm,
                    const int32_t* att, const int32_t* path, long long B, int sampled) {
    if (!p) return fail(RMFHT_EVALUE, "plan is NULL");
    if (B < 0) return fail(RMFHT_EVALUE, "negative batch");
    if (B > 0 && (!llr || !cw || !pm || !att || !path || (p->perms && !sampled && !maps)))
        return fail(RMFHT_EVALUE, "NULL buffer");
    return 0;
}

int rmfht_decode_launch_sampled(const rmfht_plan* p, const void* d_llr, uint64_t seed, long long frame0,
                                int identity_root, uint32_t* d_cw, void* d_pm, int32_t* d_attempt, int32_t* d_path,
                                long long B, void* d_work, long long work_bytes, void* stream) {
    int rc = check_io(p, d_llr, nullptr, d_cw, d_pm, d_attempt, d_path, B, 1);
    if (rc) return rc;
    if ((rc = check_work(p, B, 1, d_work, work_bytes))) return rc;
    if (B == 0) return 0;
    if (!p->perms)
        return p->launch(p, d_llr, nullptr, d_cw, d_pm, d_attempt, d_path, nullptr, nullptr, B, d_work,
                         static_cast<cudaStream_t>(stream));
    // the table takes the head of the workspace, the kernel's records the rest
    uint16_t* rec = static_cast<uint16_t*>(d_work);
    void* kwork = static_cast<char*>(d_work) + table_bytes(p, B);
    rc = rmfht_sample_maps_device(p, seed, frame0, B, identity_root, rec, stream);
    if (rc) return rc;
    return p->launch(p, d_llr, rec, d_cw, d_pm, d_attempt, d_path, nullptr, nullptr, B, kwork,
                     static_cast<cudaStream_t>(stream));
}

int rmfht_decode_launch_diag(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm,
                             int32_t* att, int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* d_work,
                             long long work_bytes, void* stream) {
    int rc = check_io(p, llr, maps, cw, pm, att, path, B, 0);
    if (rc) return rc;
    if ((rc = check_work(p, B, 0, d_work, work_bytes))) return rc;
    if (B == 0) return 0;
    return p->launch(p, llr, maps, cw, pm, att, path, att_pm, att_cw, B, d_work, static_cast<cudaStream_t>(stream));
}

int rmfht_decode_launch(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm,
                        int32_t* att, int32_t* path, long long B, void* d_work, long long work_bytes, void* stream) {
    return rmfht_decode_launch_diag(p, llr, maps, cw, pm, att, path, nullptr, nullptr, B, d_work, work_bytes,
                                    stream);
}

}  // extern "C"
