// Per-SM instruction throughput on B200 for the ops the decoder is built from.
// Each kernel runs W warps/SM; reports warp-instructions per SM-clock (clock64).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define U 16
__device__ float sink_f; __device__ unsigned sink_u;

template <int OP>
__global__ void kern(float* out, unsigned long long* cycles) {
  __shared__ float sm[8192];
  float a[U]; unsigned b[U];
  for (int i = 0; i < U; i++) { a[i] = threadIdx.x * 0.001f + i; b[i] = threadIdx.x * 7 + i; }
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < U; i++) {
      if (OP == 0) a[i] = a[i] + a[(i + 1) % U];                                   // FADD
      if (OP == 1) { float2 x = make_float2(a[i], a[(i+1)%U]); float2 y = make_float2(a[(i+2)%U], a[(i+3)%U]);
                     unsigned long long r, xx = *(unsigned long long*)&x, yy = *(unsigned long long*)&y;
                     asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(xx), "l"(yy));
                     float2 z = *(float2*)&r; a[i] = z.x; a[(i+1)%U] = z.y; }            // FADD2
      if (OP == 2) a[i] = fminf(fabsf(a[i]), fabsf(a[(i + 3) % U]));               // FMNMX |.|
      if (OP == 3) b[i] = b[i] ^ b[(i + 1) % U] ^ (b[(i+5)%U] & 0x55);              // LOP3
      if (OP == 4) a[i] = __shfl_xor_sync(0xffffffffu, a[i], (i & 7) + 1);          // SHFL
      if (OP == 5) a[i] = sm[((b[i] + it * 32) & 8191)];                             // LDS.32
      if (OP == 6) { float4 v = reinterpret_cast<float4*>(sm)[((b[i] + it) & 2047)]; a[i] += v.x; }  // LDS.128 (+FADD)
      if (OP == 7) b[i] = min(b[i], b[(i + 1) % U]);                                  // IMNMX
      if (OP == 8) a[i] = (a[i] > a[(i+1)%U]) ? a[(i+2)%U] : a[i];                   // FSETP+FSEL
      if (OP == 9) { a[i] = a[i] + a[(i + 1) % U]; b[i] = min(b[i], b[(i+1)%U]); } // FADD || IMNMX
      if (OP == 10) sm[(b[i] + it * 32 + i) & 8191] = a[i];                           // STS.32
    }
  }
  unsigned long long t1 = clock64();
  float s = 0; unsigned t = 0;
  for (int i = 0; i < U; i++) { s += a[i]; t ^= b[i]; }
  if (s == 12345.f) sink_f = s;
  if (t == 12345u) sink_u = t;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + t;
}

template <int OP> void run(const char* name, int warps_per_block, int blocks_per_sm, float instr_per_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int nb = sms * blocks_per_sm, nt = warps_per_block * 32;
  float* out; unsigned long long* cyc; cudaMalloc(&out, nb * nt * 4); cudaMalloc(&cyc, nb * 8);
  kern<OP><<<nb, nt>>>(out, cyc); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kern<OP><<<nb, nt>>>(out, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[4096]; cudaMemcpy(h, cyc, nb * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < nb; i++) avg += h[i]; avg /= nb;
  double warp_instrs_per_sm = (double)warps_per_block * blocks_per_sm * ITERS * U * instr_per_iter;
  printf("%-22s warps/SM=%3d  %.3f warp-instr/clk/SM (by clock64)  kernel %.3f ms\n", name,
         warps_per_block * blocks_per_sm, warp_instrs_per_sm / avg, ms);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    int bps = w / 8;
    run<0>("FADD", 8, bps, 1);
    run<1>("FADD2 (f32x2)", 8, bps, 0.5f);
    run<2>("FMNMX |a|,|b|", 8, bps, 1);
    run<3>("LOP3 (2 per)", 8, bps, 2);
    run<4>("SHFL.BFLY", 8, bps, 1);
    run<5>("LDS.32 (+addr)", 8, bps, 1);
    run<6>("LDS.128 (+FADD)", 8, bps, 1);
    run<7>("IMNMX", 8, bps, 1);
    run<8>("FSETP+FSEL", 8, bps, 1);
    run<9>("FADD+IMNMX pair", 8, bps, 2);
    run<10>("STS.32 (+addr)", 8, bps, 1);
  }
  return 0;
}
