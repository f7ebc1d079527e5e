// Kernel-binding unit: instantiates decode_kernel<T, r, m, L> for one dtype
// and one chunk of RMFHT_CONFIGS; built once per (RMFHT_T, RMFHT_CHUNK).
#include <cstdlib>

#include "rmfht_fast.cuh"
#include "rmfht_grp.cuh"
#include "rmfht_kernels.cuh"
#include "rmfht_lane.cuh"
#include "rmfht_pair.cuh"
#include "rmfht_plan.h"

#ifndef RMFHT_T
#define RMFHT_T float
#endif
#ifndef RMFHT_CHUNK
#define RMFHT_CHUNK 0
#endif

#define CHUNK_MACRO_(n) RMFHT_CHUNK##n
#define CHUNK_MACRO(n) CHUNK_MACRO_(n)
#define BINDER_(t, n) rmfht_bind_##t##_##n
#define BINDER(t, n) BINDER_(t, n)

using rmfht_internal::fail;

namespace {

template <typename T, int R, int MM, int L>
int launch_impl(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm,
                int32_t* att, int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/,
                cudaStream_t st) {
    rmfht::Params<T> prm;
    prm.llr = static_cast<const T*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = p->perms;
    prm.tie_fix = p->tie_fix;
    prm.cw = cw;
    prm.pm = static_cast<T*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<T*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const long long grid = B < p->grid ? B : p->grid;
    rmfht::decode_kernel<T, R, MM, L><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    return 0;
}

template <typename T, int R, int MM, int L>
int prepare(rmfht_plan* p) {
    const int Meff = p->perms ? p->M : 1;
    int nw = Meff < 8 ? Meff : 8;
    if (nw < 1) nw = 1;
    // keep a CTA's shared memory under ~110 KB so two CTAs fit an SM
    while (nw > 1 && rmfht::smem_bytes<T, R, MM, L>(nw) > 110 * 1024) nw--;
    const size_t smem = rmfht::smem_bytes<T, R, MM, L>(nw);
    auto kern = rmfht::decode_kernel<T, R, MM, L>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "kernel does not fit an SM");
    p->nwarps = nw;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

template <int R, int MM, int L>
int launch_fast(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
                int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* work, cudaStream_t st) {
    rmfht::Params<float> prm;
    prm.llr = static_cast<const float*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = p->perms;
    prm.tie_fix = (p->lockstep & 0xff) << 8;  // warps per lock-step group (the fast kernel has no tie fix)
    prm.cw = cw;
    prm.pm = static_cast<float*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<float*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    // the kernel indexes work items with 32-bit integers: at most 2^30 items
    // (frames x attempts) per launch, larger batches go in frame chunks; the
    // per-attempt records live in the caller's workspace (sized by
    // rmfht_workspace_bytes for one chunk), reused chunk after chunk in
    // stream order
    const long long chunk = rmfht_chunk_frames(p);
    constexpr int N = 1 << MM, NW = N / 32, S = rmfht::maps_per_attempt(R, MM, L), REC = 2 * MM + 2;
    for (long long f0 = 0; f0 < B; f0 += chunk) {
        const long long Bc = B - f0 < chunk ? B - f0 : chunk;
        rmfht::Params<float> q = prm;
        q.B = Bc;
        q.llr = prm.llr + f0 * N;
        if (prm.maps) q.maps = prm.maps + (size_t)f0 * p->M * S * REC;
        q.cw = prm.cw + f0 * NW;
        q.pm = prm.pm + f0;
        q.attempt = prm.attempt + f0;
        q.path = prm.path + f0;
        if (prm.att_pm) q.att_pm = prm.att_pm + f0 * p->M;
        if (prm.att_cw) q.att_cw = prm.att_cw + (size_t)f0 * p->M * NW;
        const size_t items = (size_t)Bc * p->M;
        auto* hdr = static_cast<rmfht2::AttHdr*>(work);
        auto* bits = reinterpret_cast<unsigned long long*>(static_cast<char*>(work) + items * sizeof(rmfht2::AttHdr));
        const long long blocks_needed = ((long long)items + p->nwarps - 1) / p->nwarps;
        const long long grid = blocks_needed < p->grid ? blocks_needed : p->grid;
        if (p->perms) {
            rmfht2::decode_kernel2<R, MM, L, true><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(q, hdr, bits);
        } else if constexpr (L == 1) {
            rmfht2::decode_kernel2<R, MM, L, false><<<(unsigned)grid, p->nwarps * 32, p->smem, st>>>(q, hdr, bits);
        }
        rmfht2::reduce_kernel2<R, MM, L><<<(unsigned)((Bc + 7) / 8), 256, 0, st>>>(q, hdr, bits);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    return 0;
}

template <int R, int MM, int L>
int prepare_fast(rmfht_plan* p) {
    int nw = rmfht2::fast_warps<R, MM, L>();
    while (nw > 4 && rmfht2::smem_bytes2<R, MM, L>(nw) > 227 * 1024) nw -= 4;  // 227 KB: the sm_100 opt-in maximum
    const size_t smem = rmfht2::smem_bytes2<R, MM, L>(nw);
    auto kern = rmfht2::decode_kernel2<R, MM, L, true>;
    if constexpr (L == 1) {
        if (!p->perms) kern = rmfht2::decode_kernel2<R, MM, L, false>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "kernel does not fit an SM");
    p->nwarps = nw;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

// lane-per-frame kernel (rmfht_lane.cuh): FHT-FSC on short codes
template <int R, int MM>
int launch_lane(const rmfht_plan* p, const void* llr, const uint16_t* /*maps*/, uint32_t* cw, void* pm, int32_t* att,
                int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/, cudaStream_t st) {
    rmfht::Params<float> prm;
    prm.llr = static_cast<const float*>(llr);
    prm.maps = nullptr;
    prm.B = B;
    prm.M = 1;
    prm.perms = 0;
    prm.tie_fix = 0;
    prm.cw = cw;
    prm.pm = static_cast<float*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<float*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const long long blocks = (B + 255) / 256;
    const long long grid = blocks < p->grid ? blocks : p->grid;
    rmfht_lane::lane_kernel<R, MM><<<(unsigned)grid, 256, 0, st>>>(prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("lane kernel launch: ") + cudaGetErrorString(e));
    return 0;
}

template <int R, int MM>
int prepare_lane(rmfht_plan* p) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rmfht_lane::lane_kernel<R, MM>, 256, 0);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "lane kernel does not fit an SM");
    p->nwarps = 8;
    p->smem = 0;
    p->grid = sms * per_sm;
    return 0;
}

// pair kernel (rmfht_pair.cuh): p-FHT-FSCL, r = 2, L = 2, short codes
template <int MM>
int launch_pair(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
                int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* /*work: none*/, cudaStream_t st) {
    rmfht::Params<float> prm;
    prm.llr = static_cast<const float*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = 1;
    prm.tie_fix = p->tie_fix;
    prm.cw = cw;
    prm.pm = static_cast<float*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<float*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    const long long warps = (B * p->M + 15) / 16;
    constexpr int PW = rmfht_pair::kPairWarps;  // lock-stepped warps per CTA, one CTA per SM
    const long long blocks = (warps + PW - 1) / PW;
    const long long grid = blocks < p->grid ? blocks : p->grid;
    rmfht_pair::pair_kernel<MM><<<(unsigned)grid, 32 * PW, p->smem, st>>>(prm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("pair kernel launch: ") + cudaGetErrorString(e));
    return 0;
}

template <int MM>
int prepare_pair(rmfht_plan* p) {
    // M >= 4: two frame buffers and two record buffers per warp (the next round's are prefetched)
    const size_t frames = (size_t)rmfht_pair::kPairWarps * (16 / p->M) * (1u << MM) * sizeof(float);
    const size_t records = (size_t)rmfht_pair::kPairWarps * 16 * 6 * (2 * MM + 2) * sizeof(uint16_t);
    const size_t smem = (p->M >= 4 ? 2 * frames + 2 * records : frames) +
                        (size_t)(4u << MM);  // alignment pad of the frame buffers
    cudaError_t a = cudaFuncSetAttribute(rmfht_pair::pair_kernel<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (a != cudaSuccess) return fail(RMFHT_ECUDA, std::string("pair smem attribute: ") + cudaGetErrorString(a));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rmfht_pair::pair_kernel<MM>,
                                                                  32 * rmfht_pair::kPairWarps, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "pair kernel does not fit an SM");
    p->nwarps = rmfht_pair::kPairWarps;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

// lane-group kernel (rmfht_grp.cuh): p-FHT-FSCL, r = 2, L = 1, four attempts of a frame per warp
template <int MM>
int launch_grp(const rmfht_plan* p, const void* llr, const uint16_t* maps, uint32_t* cw, void* pm, int32_t* att,
               int32_t* path, void* att_pm, uint32_t* att_cw, long long B, void* work, cudaStream_t st) {
    rmfht::Params<float> prm;
    prm.llr = static_cast<const float*>(llr);
    prm.maps = maps;
    prm.B = B;
    prm.M = p->M;
    prm.perms = 1;
    // free-running warps: the body is small enough for the instruction caches
    // (measured 2.03 M frames/s against 1.85 M with a CTA barrier per round)
    prm.tie_fix = std::getenv("RMFHT_GRP_LOCKSTEP") ? 1 << 8 : 0;
    prm.cw = cw;
    prm.pm = static_cast<float*>(pm);
    prm.attempt = att;
    prm.path = path;
    prm.att_pm = static_cast<float*>(att_pm);
    prm.att_cw = att_cw;
    if (B <= 0) return 0;
    auto* mp = const_cast<rmfht_plan*>(p);
    std::call_once(mp->once, [mp] { mp->prepared_rc = mp->prepare(mp); });
    if (p->prepared_rc != 0) return p->prepared_rc;
    // frame chunks as launch_fast (32-bit item counts in the reduce kernel's grid)
    const long long chunk = rmfht_chunk_frames(p);
    constexpr int N = 1 << MM, NW = N / 32, S = rmfht_grp::kMaps, REC = 2 * MM + 2;
    constexpr int PW = rmfht_grp::kGrpWarps;
    for (long long f0 = 0; f0 < B; f0 += chunk) {
        const long long Bc = B - f0 < chunk ? B - f0 : chunk;
        rmfht::Params<float> q = prm;
        q.B = Bc;
        q.llr = prm.llr + f0 * N;
        q.maps = prm.maps + (size_t)f0 * p->M * S * REC;
        q.cw = prm.cw + f0 * NW;
        q.pm = prm.pm + f0;
        q.attempt = prm.attempt + f0;
        q.path = prm.path + f0;
        if (prm.att_pm) q.att_pm = prm.att_pm + f0 * p->M;
        if (prm.att_cw) q.att_cw = prm.att_cw + (size_t)f0 * p->M * NW;
        const size_t items = (size_t)Bc * p->M;
        auto* hdr = static_cast<rmfht2::AttHdr*>(work);
        auto* bits = reinterpret_cast<unsigned long long*>(static_cast<char*>(work) + items * sizeof(rmfht2::AttHdr));
        const long long rounds = (long long)items / rmfht_grp::kItems;
        const long long blocks_needed = (rounds + PW - 1) / PW;
        const long long grid = blocks_needed < p->grid ? blocks_needed : p->grid;
        rmfht_grp::grp_kernel<MM><<<(unsigned)grid, 32 * PW, p->smem, st>>>(q, hdr, bits);
        rmfht2::reduce_kernel2<2, MM, 1, rmfht_grp::kLpp><<<(unsigned)((Bc + 7) / 8), 256, 0, st>>>(q, hdr, bits);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(RMFHT_ECUDA, std::string("lane-group kernel launch: ") + cudaGetErrorString(e));
    return 0;
}

template <int MM>
int prepare_grp(rmfht_plan* p) {
    const size_t smem = rmfht_grp::smem_bytes<MM>(rmfht_grp::kGrpWarps);
    auto kern = rmfht_grp::grp_kernel<MM>;
    cudaError_t a = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (a != cudaSuccess) return fail(RMFHT_ECUDA, std::string("lane-group smem attribute: ") + cudaGetErrorString(a));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * rmfht_grp::kGrpWarps, smem);
    if (e != cudaSuccess || per_sm < 1) return fail(RMFHT_ECUDA, "lane-group kernel does not fit an SM");
    p->nwarps = rmfht_grp::kGrpWarps;
    p->smem = smem;
    p->grid = sms * per_sm;
    return 0;
}

template <typename T, int R, int MM, int L>
int bind_one(rmfht_plan* p) {
    if constexpr (sizeof(T) == 4 && R == 2 && L == 1 && MM >= 8 && MM <= 9) {
        // p-FHT-FSCL with one path: four attempts of a frame per warp
        // (RMFHT_NO_GRP: A/B and cross-check against the throughput kernel)
        if (p->fast && p->perms && p->M % rmfht_grp::kItems == 0 && !std::getenv("RMFHT_NO_GRP")) {
            p->grp = 1;
            p->work_per_item = rmfht_grp::work_bytes();
            p->launch = &launch_grp<MM>;
            p->prepare = &prepare_grp<MM>;
            return 0;
        }
    }
    if constexpr (sizeof(T) == 4 && R == 2 && L == 2 && MM >= 4 && MM <= 7) {
        // p-FHT-FSCL, L = 2, short code, the M attempts of a frame within a
        // warp's 16 items: two threads per item (RMFHT_NO_PAIR: A/B only)
        if (p->fast && p->perms && 16 % p->M == 0 && !std::getenv("RMFHT_NO_PAIR")) {
            p->pair = 1;
            p->launch = &launch_pair<MM>;
            p->prepare = &prepare_pair<MM>;
            return 0;
        }
    }
    if constexpr (sizeof(T) == 4 && L == 1 && (1 << MM) <= 64 && (1 << MM) >= 4) {
        // FHT-FSC (L = 1, no permutations) on a short code: one thread per frame
        if (p->fast && !p->perms) {
            p->lane = 1;
            p->launch = &launch_lane<R, MM>;
            p->prepare = &prepare_lane<R, MM>;
            return 0;
        }
    }
    if constexpr (sizeof(T) == 4 && (1 << MM) >= 32 && L <= 8) {
        // without permutations the list starts from one path and grows, which
        // the throughput kernel (P == L at every node) does not model: FHT-FSC
        // (L = 1) only
        if (p->fast && (p->perms || L == 1)) {
            p->work_per_item = rmfht2::work_bytes2<R, MM, L>();
            p->launch = &launch_fast<R, MM, L>;
            p->prepare = &prepare_fast<R, MM, L>;
            return 0;
        }
    }
    p->fast = 0;
    p->launch = &launch_impl<T, R, MM, L>;
    p->prepare = &prepare<T, R, MM, L>;
    return 0;
}

}  // namespace

int BINDER(RMFHT_T, RMFHT_CHUNK)(rmfht_plan* p) {
#define X(R_, M_, L_)                                          \
    if (p->r == R_ && p->m == M_ && p->L == L_) return bind_one<RMFHT_T, R_, M_, L_>(p);
    CHUNK_MACRO(RMFHT_CHUNK)(X)
#undef X
    return RMFHT_EUNSUPPORTED;
}

#ifdef RMFHT_STATS
// diagnostic build only (tools/stats_run.py): read and clear this unit's counters
#define STATS_(t, n) rmfht_stats_read_##t##_##n
#define STATS(t, n) STATS_(t, n)
extern "C" int STATS(RMFHT_T, RMFHT_CHUNK)(unsigned long long* host) {
    if (cudaMemcpyFromSymbol(host, rmfht2::g_stats, sizeof(rmfht2::g_stats)) != cudaSuccess) return -1;
    static const unsigned long long zero[256] = {};
    return cudaMemcpyToSymbol(rmfht2::g_stats, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
#endif
