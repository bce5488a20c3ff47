// Microbenchmark: scalar FFMA/FADD vs packed FFMA2/FADD2 issue + FLOP throughput on sm_100a.
// Also checks the 2-instruction complex multiply form folds as expected.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 upk(u64 v) { float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }

template <int MODE>
__global__ void probe(float* out, int iters, float s) {
  float a[16]; u64 p[16];
  for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-3f + i; p[i] = pk(a[i], a[i] + 0.5f); }
  const u64 c = pk(s, s * 0.5f), d = pk(0.999f, 0.998f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], s, 0.999f);                       // FFMA (imm)
      if (MODE == 1) a[i] = fmaf(a[i], s, a[(i + 1) & 15]);              // FFMA 3-reg
      if (MODE == 2) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(c), "l"(d));   // FFMA2
      if (MODE == 3) a[i] = a[i] + a[(i + 3) & 15];                      // FADD
      if (MODE == 4) asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(p[(i + 3) & 15]));  // FADD2
    }
  }
  float r = 0.f;
  for (int i = 0; i < 16; ++i) { float2 q = upk(p[i]); r += a[i] + q.x + q.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * 148 * 8 * 1024);
  const char* names[] = {"FFMA imm", "FFMA 3reg", "FFMA2", "FADD", "FADD2"};
  const int flops[] = {2, 2, 4, 1, 2};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 5; ++mode) {
    for (int warps = 4; warps <= 32; warps *= 2) {
      const int iters = 4096, blocks = sms * 2, threads = warps * 16;  // 2 blocks/SM -> `warps` warps/SM
      auto launch = [&]() {
        switch (mode) { case 0: probe<0><<<blocks, threads>>>(out, iters, 1.0001f); break;
                        case 1: probe<1><<<blocks, threads>>>(out, iters, 1.0001f); break;
                        case 2: probe<2><<<blocks, threads>>>(out, iters, 1.0001f); break;
                        case 3: probe<3><<<blocks, threads>>>(out, iters, 1.0001f); break;
                        default: probe<4><<<blocks, threads>>>(out, iters, 1.0001f); }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double instr = (double)blocks * threads / 32 * iters * 16;     // warp instructions
      double cyc = ms * 1e-3 * clk * 1e3;                             // at max clock
      printf("%-10s warps/SM=%2d  %.3f ms  warp-instr/clk/SM=%.2f  TFLOP/s=%.1f\n", names[mode], warps, ms,
             instr / sms / cyc, instr * 32 * flops[mode] / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
