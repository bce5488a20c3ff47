// FFMA2 issue-rate probe for the operand patterns of the DFT codelets: accumulate
// 16 packed accumulators from 8 packed inputs with (a) immediate broadcast coefficients,
// (b) register broadcast coefficients (scalar register .F32 operand), (c) register pairs.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
template <int MODE>
__global__ void probe(float* out, int iters, float s) {
  u64 acc[16], x[8];
  for (int i = 0; i < 16; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, i);
  for (int i = 0; i < 8; ++i) x[i] = pk(s * i, s + i);
  float cr[8]; for (int i = 0; i < 8; ++i) cr[i] = s * (i + 1) * 0.01f;
  u64 cp[8]; for (int i = 0; i < 8; ++i) cp[i] = pk(cr[i], cr[i] * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (MODE == 0) acc[k] = fma2(x[j], pk(0.125f * (k + 1) + 0.01f * j, 0.125f * (k + 1) + 0.01f * j), acc[k]);
        if (MODE == 1) acc[k] = fma2(x[j], pk(cr[(j + k) & 7], cr[(j + k) & 7]), acc[k]);
        if (MODE == 2) acc[k] = fma2(x[j], cp[(j + k) & 7], acc[k]);
      }
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = acc[j] ^ (u64)(it & 1);
  }
  u64 r = 0; for (int i = 0; i < 16; ++i) r ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(r & 0xffff);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
  const char* names[] = {"imm bcast", "reg bcast", "reg pair"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int warps = 8; warps <= 16; warps *= 2) {
      const int iters = 2048, blocks = sms * 2, threads = warps * 16;
      auto launch = [&]() { if (mode == 0) probe<0><<<blocks, threads>>>(out, iters, 1.0001f);
                            else if (mode == 1) probe<1><<<blocks, threads>>>(out, iters, 1.0001f);
                            else probe<2><<<blocks, threads>>>(out, iters, 1.0001f); };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double instr = (double)blocks * threads / 32 * iters * 128;
      printf("%-10s warps/SM=%2d FFMA2/clk/SM=%.2f  TFLOP/s=%.1f\n", names[mode], warps,
             instr / sms / (ms * 1e-3 * clk * 1e3), instr * 32 * 4 / (ms * 1e-3) / 1e12);
    }
  return 0;
}
