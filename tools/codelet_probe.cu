// FMA-pipe utilisation of the K2 codelets in isolation (no memory, no syncs): each thread runs
// MODE 0: the 31-point inverse Rader DFT + |.|^2 accumulation, MODE 1: the 33-point DFT (3 x 11),
// MODE 2: the 31-point real-symmetric form, repeatedly on its own registers.  Reports executed
// FMA-pipe cycles per second against 4 SMSPs x clock.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1309_0052_b200/csrc tools/codelet_probe.cu -o tools/codelet_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "pfa.cuh"
#include "rader31.cuh"
using namespace gacq;

template <int MODE>
__global__ void __maxnreg__(168) probe(float* out, int iters, float s) {
    cx x[33];
#pragma unroll
    for (int i = 0; i < 33; ++i) x[i] = pk(s * (i + threadIdx.x), s - i);
    float acc[33];
#pragma unroll
    for (int i = 0; i < 33; ++i) acc[i] = 0.f;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            cx y[31];
            dft31_rader_inv([&](int k) { return x[k]; }, [&](int q, cx v) { y[q] = v; acc[q] = fmaf(im(v), im(v), fmaf(re(v), re(v), acc[q])); });
#pragma unroll
            for (int i = 0; i < 31; ++i) x[i] = mul2(y[i], bc(0.0322f));
        } else if (MODE == 1) {
            cx y[33];
            dft33<1>(x, [&](int q, cx v) { y[q] = v; });
#pragma unroll
            for (int i = 0; i < 33; ++i) x[i] = mul2(y[i], bc(0.0303f));
        } else {
            cx y[31], t[31];
#pragma unroll
            for (int i = 0; i < 31; ++i) t[i] = x[i];
            dft_odd<1, 31, 5>(t, [&](int q, cx v) { y[q] = v; acc[q] = fmaf(im(v), im(v), fmaf(re(v), re(v), acc[q])); });
#pragma unroll
            for (int i = 0; i < 31; ++i) x[i] = mul2(y[i], bc(0.0322f));
        }
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 33; ++i) r += re(x[i]) + acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, int pipe_cycles_per_iter, int sms, int clk_khz, float* out) {
    const int iters = 2000, blocks = sms * 3;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE><<<blocks, 128>>>(out, 10, 1.0001f);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    probe<MODE><<<blocks, 128>>>(out, iters, 1.0001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_iters = (double)blocks * 4 * iters;
    const double cycles = ms * 1e-3 * clk_khz * 1e3;
    printf("%-12s %.3f ms  %.1f warp-iters/SMSP-kcycle  pipe util %.3f (at %d cycles/iter)\n", name, ms,
           warp_iters / (sms * 4) / cycles * 1e3, warp_iters / (sms * 4) * pipe_cycles_per_iter / cycles,
           pipe_cycles_per_iter);
}

int main(int argc, char** argv) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 3 * 128);
    // packed-op counts per iteration from the SASS (cuobjdump) are printed by the caller script
    // FMA-pipe cycles per iteration (2 per packed op, 1 per scalar) counted from the SASS loop
    // bodies by tools/codelet_probe.sh
    const int c0 = argc > 3 ? atoi(argv[1]) : 1, c1 = argc > 3 ? atoi(argv[2]) : 1, c2 = argc > 3 ? atoi(argv[3]) : 1;
    run<0>("rader31", c0, sms, clk, out);
    run<1>("dft33", c1, sms, clk, out);
    run<2>("symm31", c2, sms, clk, out);
    return 0;
}
