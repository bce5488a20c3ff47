// Probe: device float32(cos/sin(float64 angle)) of the 48-bit carrier NCO vs the host values
// (reads p0, step, n from argv; writes float32 pairs to stdout as binary).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(uint64_t p0, uint64_t step, int n, float2* out, int mode) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t p = (p0 + (uint64_t)i * step) & ((1ull << 48) - 1);
    double th = (double)p * (6.283185307179586 / 281474976710656.0);
    double s, c;
    if (mode == 0) sincos(th, &s, &c);
    else { c = cos(th); s = sin(th); }
    out[i] = make_float2((float)c, (float)(-s));
}
int main(int argc, char** argv) {
    uint64_t p0 = strtoull(argv[1], 0, 10), step = strtoull(argv[2], 0, 10);
    int n = atoi(argv[3]), mode = atoi(argv[4]);
    float2* d; cudaMalloc(&d, n * 8);
    k<<<(n + 255) / 256, 256>>>(p0, step, n, d, mode);
    float2* h = (float2*)malloc(n * 8);
    cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
    fwrite(h, 8, n, stdout);
    return 0;
}
