// A/B for the north star's tensor-core question (BASELINE.json: "Tensor
// cores are used only if ncu shows that a batched Hadamard contraction on a
// constituent node beats the shuffle butterfly"): the n = 256 FHT node of
// the headline (fht_decode.py:28-55; 4 paths x 655,360 (frame, attempt)
// items per 32,768-frame step), V vectors of 256 floats.
//
//  A  butterfly: the decoder's layout — 8 lanes per vector, 32 elements per
//     lane in registers, 5 register stages as packed f32x2 (FADD2) and 3
//     lane stages by shuffles, then |w| max per vector (the node's first
//     selection step); fp32, bit-exact with the reference's stage order.
//  B  tensor cores: W = X H with H the node's +-1 matrix
//     (H[i,j] = (-1)^popcount(~i & ~j & 255), exact in bf16) through
//     cuBLAS bf16 GEMM with fp32 accumulation (cublasGemmEx, tensor-op
//     kernels on sm_100), one pass = bf16 inputs; fp32-faithful w needs the
//     input split into 3 bf16 parts (3 passes) and still is not bit-exact
//     with the butterfly's rounding, which the tie rules require.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcublas fht_ab.cu
// Prints vectors/s for A and B (one pass) with CUDA events; run under
// `ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,...`
// for the per-kernel counters (profiles/r2_tc_fht_ab.txt).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

using u64 = unsigned long long;
__device__ __forceinline__ u64 pk(float lo, float hi) {
    return ((u64)__float_as_uint(hi) << 32) | (u64)__float_as_uint(lo);
}
__device__ __forceinline__ float plo(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float phi(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

// A: element e = k * 8 + u of a vector in slot k of lane u (u = lane % 8)
// REPS transforms per loaded vector: REPS = 1 is the memory-bound pass,
// REPS = 16 the in-register (compute) rate that the decoder's node sees
template <int REPS>
__global__ void __launch_bounds__(256) fht_butterfly(const float* __restrict__ x, float* __restrict__ best, long long V) {
    const int lane = threadIdx.x & 31, u = lane & 7;
    const long long nvw = (long long)gridDim.x * (blockDim.x / 32) * 4;
    for (long long v0 = ((long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 4; v0 < V; v0 += nvw) {
        const long long vec = v0 + (lane >> 3);
        float w[32];
        const float* src = x + vec * 256;
#pragma unroll
        for (int k = 0; k < 32; k++) w[k] = vec < V ? __ldg(src + k * 8 + u) : 0.f;
#pragma unroll 1
        for (int rep = 0; rep < REPS; rep++) {
        if (rep) {
#pragma unroll
            for (int k = 0; k < 32; k++) w[k] *= 0.0625f;  // keep the magnitudes (H H = 256 I)
        }
        // register stages: slot bits 4..0 (element bits 7..3), halves 16, 8, 4, 2 packed; 1 scalar
#pragma unroll
        for (int hr = 16; hr >= 2; hr >>= 1) {
#pragma unroll
            for (int k = 0; k < 32; k += 2)
                if (!(k & hr)) {
                    const u64 lo = pk(w[k], w[k + 1]), hi = pk(w[k + hr], w[k + hr + 1]);
                    const u64 d = sub2(hi, lo), e = add2(hi, lo);
                    w[k] = plo(d); w[k + 1] = phi(d); w[k + hr] = plo(e); w[k + hr + 1] = phi(e);
                }
        }
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
            const float lo = w[k], hi = w[k + 1];
            w[k] = hi - lo;
            w[k + 1] = hi + lo;
        }
        // lane stages: element bits 2..0 (lane bits), halves 4, 2, 1
#pragma unroll
        for (int half = 4; half >= 1; half >>= 1) {
            const float sg = (u & half) ? 1.f : -1.f;
            const u64 sg2 = pk(sg, sg);
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
                const float o0 = __shfl_xor_sync(0xffffffffu, w[k], half), o1 = __shfl_xor_sync(0xffffffffu, w[k + 1], half);
                const u64 r = fma2(sg2, pk(w[k], w[k + 1]), pk(o0, o1));
                w[k] = plo(r); w[k + 1] = phi(r);
            }
        }
        }
        float m = fabsf(w[0]);
#pragma unroll
        for (int k = 1; k < 32; k++) m = fmaxf(m, fabsf(w[k]));
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (u == 0 && vec < V) best[vec] = m;
    }
}

__global__ void fill(float* x, __nv_bfloat16* xb, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned h = (unsigned)(i * 2654435761u) ^ (unsigned)(i >> 7);
        const float v = ((h & 0xffff) / 32768.f - 1.f) * 3.f;
        x[i] = v;
        xb[i] = __float2bfloat16(v);
    }
}

int main() {
    const long long V = 1 << 20;  // vectors of 256 (1 GiB fp32): > L2
    const int n = 256, reps = 10;
    float *x, *best, *w;
    __nv_bfloat16 *xb, *hb;
    cudaMalloc(&x, V * n * 4);
    cudaMalloc(&best, V * 4);
    cudaMalloc(&xb, V * n * 2);
    cudaMalloc(&w, V * n * 4);
    cudaMalloc(&hb, n * n * 2);
    fill<<<4096, 256>>>(x, xb, V * n);
    std::vector<__nv_bfloat16> h(n * n);
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) h[i * n + j] = __float2bfloat16((__builtin_popcount(~i & ~j & 255) & 1) ? -1.f : 1.f);
    cudaMemcpy(hb, h.data(), n * n * 2, cudaMemcpyHostToDevice);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // A: memory pass (1 transform per load) and in-register rate (16 per load)
    float ms_a, ms_a16;
    for (int i = 0; i < 3; i++) fht_butterfly<1><<<sms * 8, 256>>>(x, best, V);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) fht_butterfly<1><<<sms * 8, 256>>>(x, best, V);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms_a, e0, e1);
    ms_a /= reps;
    for (int i = 0; i < 3; i++) fht_butterfly<16><<<sms * 8, 256>>>(x, best, V);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) fht_butterfly<16><<<sms * 8, 256>>>(x, best, V);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms_a16, e0, e1);
    ms_a16 /= reps * 16;
    // B: W[V x 256] = X[V x 256] H (column-major: W^T = H^T X^T, H symmetric)
    cublasHandle_t hd;
    cublasCreate(&hd);
    const float one = 1.f, zero = 0.f;
    auto gemm = [&] {
        return cublasGemmEx(hd, CUBLAS_OP_N, CUBLAS_OP_N, n, (int)V, n, &one, hb, CUDA_R_16BF, n, xb, CUDA_R_16BF, n,
                            &zero, w, CUDA_R_32F, n, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    };
    for (int i = 0; i < 3; i++) gemm();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) gemm();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms_b;
    cudaEventElapsedTime(&ms_b, e0, e1);
    ms_b /= reps;
    const double flops_b = 2.0 * n * n * (double)V;
    printf("{\"vectors\": %lld, \"n\": %d, \"butterfly_mem_ms\": %.4f, \"butterfly_mem_vectors_per_s\": %.4g, "
           "\"butterfly_inreg_vectors_per_s\": %.4g, "
           "\"tc_bf16_1pass_ms\": %.4f, \"tc_bf16_1pass_vectors_per_s\": %.4g, \"tc_tflops\": %.1f, "
           "\"tc_3pass_vectors_per_s\": %.4g, \"inreg_butterfly_over_tc_1pass\": %.2f, "
           "\"inreg_butterfly_over_tc_3pass\": %.2f}\n",
           V, n, ms_a, V / (ms_a * 1e-3), V / (ms_a16 * 1e-3), ms_b, V / (ms_b * 1e-3),
           flops_b / (ms_b * 1e-3) / 1e12, V / (3 * ms_b * 1e-3), ms_b / ms_a16, 3 * ms_b / ms_a16);
    return 0;
}
