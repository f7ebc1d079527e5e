// Dependent-chain latency of warp primitives on one warp (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned* out, float* fo, int iters) {
    __shared__ float sm[64];
    const int lane = threadIdx.x;
    sm[lane] = lane; sm[lane + 32] = lane;
    __syncwarp();
    float f = lane * 1.0f; unsigned u = lane; long long t0, t1;
    // shfl_xor chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) f = __shfl_xor_sync(0xffffffffu, f, 1) + 1.0f;
    t1 = clock64(); if (lane == 0) out[0] = (unsigned)((t1 - t0) / iters);
    // redux max chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) u = __reduce_max_sync(0xffffffffu, u) + lane;
    t1 = clock64(); if (lane == 0) out[1] = (unsigned)((t1 - t0) / iters);
    // redux add chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) u = __reduce_add_sync(0xffffffffu, u) & 31u;
    t1 = clock64(); if (lane == 0) out[2] = (unsigned)((t1 - t0) / iters);
    // ballot chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) u = __ballot_sync(0xffffffffu, (u >> lane) & 1u) ^ lane;
    t1 = clock64(); if (lane == 0) out[3] = (unsigned)((t1 - t0) / iters);
    // LDS chain (pointer chase)
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < iters; i++) idx = (int)sm[idx] ;
    t1 = clock64(); if (lane == 0) out[4] = (unsigned)((t1 - t0) / iters);
    // FADD chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) f = f * 1.0001f + 0.5f;
    t1 = clock64(); if (lane == 0) out[5] = (unsigned)((t1 - t0) / iters);
    // shfl idx chain (u32)
    t0 = clock64();
    for (int i = 0; i < iters; i++) u = __shfl_sync(0xffffffffu, u, (int)(u & 31u)) + 1u;
    t1 = clock64(); if (lane == 0) out[6] = (unsigned)((t1 - t0) / iters);
    // vote.all chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) u = __all_sync(0xffffffffu, u != 12345u) + u;
    t1 = clock64(); if (lane == 0) out[7] = (unsigned)((t1 - t0) / iters);
    fo[lane] = f + idx + u;
}
int main() {
    unsigned* d; float* fo; cudaMalloc(&d, 64); cudaMalloc(&fo, 128);
    k<<<1, 32>>>(d, fo, 1000); k<<<1, 32>>>(d, fo, 1000);
    unsigned h[8]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    const char* n[8] = {"shfl_xor+fadd", "redux.max+iadd", "redux.add+and", "ballot+xor", "lds chase", "ffma", "shfl_idx+iadd", "vote.all+iadd"};
    for (int i = 0; i < 8; i++) printf("%-16s %u cycles\n", n[i], h[i]);
}
