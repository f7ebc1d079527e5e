// Shared-memory bandwidth and packed f32x2 throughput on B200 (kernel-time based).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define U 16
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

template <int OP>
__global__ void kern(float* out) {
  __shared__ __align__(16) float sm[8192];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  float acc[U]; u64 p[U];
  for (int i = 0; i < U; i++) { acc[i] = i; float2 f = make_float2(i, lane); p[i] = *(u64*)&f; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < U; i++) {
      const int j = (it * U + i + w * 5) & 63;
      if (OP == 0) acc[i] += sm[lane + 32 * (j & 255)];                               // LDS.32 conflict-free (+FADD)
      if (OP == 1) { float4 v = reinterpret_cast<const float4*>(sm)[(lane + 32 * (j & 63)) & 2047]; acc[i] += v.x + v.w; } // LDS.128 (+2 FADD)
      if (OP == 2) sm[(lane + 32 * ((j + w * 16) & 255))] = acc[i] + it;              // STS.32 (+FADD)
      if (OP == 3) reinterpret_cast<float4*>(sm)[(lane + 32 * ((j + w * 8) & 63)) & 2047] = make_float4(acc[i], it, i, w); // STS.128
      if (OP == 4) p[i] = add2(p[i], p[(i + 1) % U]);                                   // FADD2
      if (OP == 5) p[i] = fma2(p[i], p[(i + 1) % U], p[(i + 2) % U]);                  // FFMA2
      if (OP == 6) { p[i] = add2(p[i], p[(i + 1) % U]); acc[i] = fminf(fabsf(acc[i]), fabsf(acc[(i+1)%U])); } // FADD2 || FMNMX
      if (OP == 7) acc[i] = acc[i] + acc[(i + 1) % U];                                  // FADD
      if (OP == 8) acc[i] += sm[(lane * 33 + 32 * (j & 127)) & 8191];                   // LDS.32 w/ stride 33
    }
  }
  float s = 0;
  for (int i = 0; i < U; i++) { float2 f = *(float2*)&p[i]; s += acc[i] + f.x + f.y; }
  __syncthreads();
  s += sm[threadIdx.x];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP> void run(const char* name, int wps, double instr_per_iter, double bytes_per_instr) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int nb = sms * (wps / 8), nt = 256;
  float* out; cudaMalloc(&out, nb * nt * 4);
  kern<OP><<<nb, nt>>>(out); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<OP><<<nb, nt>>>(out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;  // at max clock
  double wi = (double)wps * ITERS * U * instr_per_iter;  // per SM
  printf("%-26s warps/SM=%2d  %.3f warp-instr/clk/SM  %.1f B/clk/SM  (%.3f ms)\n", name, wps, wi / cycles,
         wi * bytes_per_instr / cycles, ms);
  cudaFree(out);
}

int main() {
  for (int w : {16, 32}) {
    run<7>("FADD", w, 1, 0);
    run<4>("FADD2", w, 1, 0);
    run<5>("FFMA2", w, 1, 0);
    run<6>("FADD2 + FMNMX", w, 2, 0);
    run<0>("LDS.32 (+FADD)", w, 1, 128);
    run<8>("LDS.32 stride33 (+FADD)", w, 1, 128);
    run<1>("LDS.128 (+2FADD)", w, 1, 512);
    run<2>("STS.32", w, 1, 128);
    run<3>("STS.128", w, 1, 512);
  }
  return 0;
}
