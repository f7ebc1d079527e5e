// Internal plan object shared by the C-ABI unit and the kernel-binding units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rmfht.h"

// the last pointer is the caller-owned device workspace (rmfht_workspace_bytes)
using LaunchFn = int (*)(const rmfht_plan*, const void*, const uint16_t*, uint32_t*, void*, int32_t*,
                         int32_t*, void*, uint32_t*, long long, void*, cudaStream_t);
using PrepareFn = int (*)(rmfht_plan*);

struct rmfht_plan {
    int r, m, L, M, perms, tie_fix, dtype;
    int lockstep = 255;  // throughput kernel: warps per lock-step group (0 = none, >= CTA warps = whole CTA)
    int fast;  // float32 throughput kernel (rmfht_fast.cuh) instead of the reference-order one
    int generic = 0;  // runtime-shaped interpreter kernel (rmfht_generic.cuh)
    int lane = 0;     // lane-per-frame kernel (rmfht_lane.cuh): FHT-FSC on N <= 64
    int pair = 0;     // pair kernel (rmfht_pair.cuh): r = 2, L = 2, N <= 128
    int grp = 0;      // lane-group kernel (rmfht_grp.cuh): r = 2, L = 1, m = 8, 9, M % 4 == 0
    int force_generic = 0;
    int aut = 0;  // Aut-SSC plan (RMFHT_AUT_SSC): M = P single-map SSC decodes per frame
    int S, nwarps, grid;
    long long max_items = 1LL << 30;  // throughput kernel: work items per launch (env RMFHT_MAX_ITEMS, tests)
    size_t smem;
    std::vector<int> sizes;
    LaunchFn launch;
    PrepareFn prepare;  // CUDA-side binding (shared memory, occupancy), once at the first launch
    std::once_flag once;  // prepare() runs once (function attributes, occupancy); nothing else mutates a plan
    int prepared_rc;
    // throughput kernel: per-(frame, attempt) bytes of the caller-owned
    // workspace (rmfht_workspace_bytes); 0 for kernels that need none
    size_t work_per_item = 0;
};

// workspace helpers shared by the C-ABI unit and the binding units
inline size_t rmfht_align256(size_t x) { return (x + 255) & ~size_t(255); }
// items the throughput kernel decodes per launch chunk (32-bit item indices)
inline long long rmfht_chunk_frames(const rmfht_plan* p) { return p->max_items / p->M > 0 ? p->max_items / p->M : 1; }

namespace rmfht_internal {
int fail(int code, const std::string& msg);
}

// Specialisations compiled into this library: (r, m, L), each for float and
// double.  BASELINE.json's configurations plus the shapes the reference's
// tests exercise.  Split into chunks that compile in
// parallel (rmfht_bind.cu is built once per dtype x chunk).
#define RMFHT_CHUNK0(X) X(2, 9, 4) X(2, 5, 1) X(1, 2, 4) X(3, 4, 4)
#define RMFHT_CHUNK1(X) X(3, 7, 8) X(2, 4, 2) X(1, 5, 4) X(2, 8, 1)
#define RMFHT_CHUNK2(X) X(2, 9, 1) X(2, 7, 2) X(2, 6, 4) X(2, 6, 1)
#define RMFHT_CHUNK3(X) X(2, 8, 8) X(3, 8, 4) X(2, 9, 2) X(3, 6, 2) X(2, 5, 4)
#define RMFHT_NCHUNKS 4

// one binder per (dtype, chunk): returns RMFHT_EUNSUPPORTED when no match
#define RMFHT_DECL_BINDERS(T)              \
    int rmfht_bind_##T##_0(rmfht_plan* p); \
    int rmfht_bind_##T##_1(rmfht_plan* p); \
    int rmfht_bind_##T##_2(rmfht_plan* p); \
    int rmfht_bind_##T##_3(rmfht_plan* p);
RMFHT_DECL_BINDERS(float)
RMFHT_DECL_BINDERS(double)
int rmfht_bind_generic(rmfht_plan* p);
int rmfht_bind_aut_ssc(rmfht_plan* p);
