// tc_probe.cu -- validate the tcgen05 kind::tf32 building blocks used by the tensor-core K2:
// A (128 x 64 fp32) written to TMEM with tcgen05.st, B (64 x 64, K-major, no swizzle) in shared
// memory, D = A.B (and the 3xTF32 split D = A.Bhi + A.Blo + Alo.Bhi) accumulated in TMEM and
// read back with tcgen05.ld. Compared with a float64 host product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tools/tc_probe.cu && ./tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1309_0052_b200/csrc/tc_util.cuh"

using namespace gacq::tc;

// B stored K-major, core matrices of 8 (n) x 4 (k) fp32: addr(n, k) = (n/8)*2048 + (k/4)*128 +
// (n%8)*16 + (k%4)*4 bytes (LBO = 128 B between K-adjacent core matrices, SBO = 2048 B between
// N-adjacent 8-row groups).
__host__ __device__ inline int b_off(int n, int k) { return (n >> 3) * 512 + (k >> 2) * 32 + (n & 7) * 4 + (k & 3); }

template <int MODE>  // 0: one pass A.Bhi, 1: three passes
__global__ void __launch_bounds__(128) probe(const float* A, const float* Bhi, const float* Blo, float* D, int reps,
                                             long long* cycles) {
    __shared__ __align__(1024) float sB[2][64 * 64];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long mbar;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 64; i += 128) {
        const int n = i / 64, k = i % 64;
        sB[0][b_off(n, k)] = Bhi[i];
        sB[1][b_off(n, k)] = Blo[i];
    }
    if (w == 0) tmem_alloc<128>(&s_tmem);
    if (threadIdx.x == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t ta = tmem + ((uint32_t)(32 * w) << 16);
    const int m = 32 * w + lane;
    uint32_t v[64], lo[64];
    for (int k = 0; k < 64; ++k) {
        v[k] = __float_as_uint(A[m * 64 + k]);
        const float t = __uint_as_float(v[k] & 0xffffe000u);
        lo[k] = __float_as_uint(__uint_as_float(v[k]) - t);
    }
    const uint32_t idesc = idesc_tf32(128, 64);
    const uint64_t dB0 = sdesc(smem_u32(sB[0]), 128, 2048), dB1 = sdesc(smem_u32(sB[1]), 128, 2048);
    unsigned phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        tmem_st64(ta, v);
        tmem_st_wait();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (threadIdx.x == 0) {
            for (int s = 0; s < 8; ++s) mma_tf32_ts(tmem + 64, tmem + 8 * s, dB0 + 16 * s, idesc, s > 0);
            if (MODE == 1)
                for (int s = 0; s < 8; ++s) mma_tf32_ts(tmem + 64, tmem + 8 * s, dB1 + 16 * s, idesc, true);
            mma_commit(&mbar);
        }
        mbar_wait(&mbar, phase);
        phase ^= 1;
        tc_fence_after();
        if (MODE == 1) {
            tmem_st64(ta, lo);
            tmem_st_wait();
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
            if (threadIdx.x == 0) {
                for (int s = 0; s < 8; ++s) mma_tf32_ts(tmem + 64, tmem + 8 * s, dB0 + 16 * s, idesc, true);
                mma_commit(&mbar);
            }
            mbar_wait(&mbar, phase);
            phase ^= 1;
            tc_fence_after();
        }
    }
    long long t1 = clock64();
    uint32_t d[64];
    tmem_ld64(ta + 64, d);
    tmem_ld_wait();
    for (int k = 0; k < 64; ++k) D[m * 64 + k] = __uint_as_float(d[k]);
    if (threadIdx.x == 0) *cycles = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc<128>(tmem);
}


// throughput: `reps` x (24 MMAs) back to back with one commit; st/ld loops per warp
__global__ void __launch_bounds__(128) tput(const float* Bhi, int reps, long long* cyc) {
    __shared__ __align__(1024) float sB[2][64 * 64];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long mbar;
    const int w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 64; i += 128) { sB[0][i] = Bhi[i]; sB[1][i] = Bhi[i]; }
    if (w == 0) tmem_alloc<128>(&s_tmem);
    if (threadIdx.x == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_proxy_async();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = s_tmem, ta = tmem + ((uint32_t)(32 * w) << 16);
    uint32_t v[64];
    for (int k = 0; k < 64; ++k) v[k] = __float_as_uint(1.0f + k);
    const uint32_t idesc = idesc_tf32(128, 64);
    const uint64_t dB0 = sdesc(smem_u32(sB[0]), 128, 2048);
    // MMA
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int r = 0; r < reps; ++r)
            for (int s = 0; s < 24; ++s) mma_tf32_ts(tmem + 64, tmem + 8 * (s & 7), dB0 + 16 * (s & 7), idesc, true);
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    long long t1 = clock64();
    // st
    for (int r = 0; r < reps; ++r) tmem_st64(ta, v);
    tmem_st_wait();
    __syncthreads();
    long long t2 = clock64();
    uint32_t acc = 0;
    for (int r = 0; r < reps; ++r) { tmem_ld64(ta + 64, v); tmem_ld_wait(); acc += v[r & 63]; }
    __syncthreads();
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = acc; }
    tc_fence_before(); __syncthreads();
    if (w == 0) tmem_dealloc<128>(tmem);
}

int main() {
    std::vector<float> A(128 * 64), Bhi(64 * 64), Blo(64 * 64), B(64 * 64), D(128 * 64);
    srand(1);
    for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 2 - 1) * 1000.f;
    for (int n = 0; n < 64; ++n)
        for (int k = 0; k < 64; ++k) {
            const float b = (float)std::cos(0.1 * n * k + 0.3 * k);
            B[n * 64 + k] = b;
            uint32_t u;
            memcpy(&u, &b, 4);
            u &= 0xffffe000u;
            float h;
            memcpy(&h, &u, 4);
            Bhi[n * 64 + k] = h;
            Blo[n * 64 + k] = b - h;
        }
    float *dA, *dBh, *dBl, *dD;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dBh, B.size() * 4);
    cudaMalloc(&dBl, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBh, Bhi.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBl, Blo.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int fails = 0;
    for (int mode = 0; mode < 2; ++mode) {
        for (int reps : {1, 64}) {
            cudaMemset(dD, 0, D.size() * 4);
            if (mode == 0) probe<0><<<1, 128>>>(dA, dBh, dBl, dD, reps, dc);
            else probe<1><<<1, 128>>>(dA, dBh, dBl, dD, reps, dc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            long long cyc;
            cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            double max_rel = 0, max_abs = 0, ref_max = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 64; ++k) ref += (double)A[m * 64 + k] * (mode ? B[n * 64 + k] : Bhi[n * 64 + k]);
                    max_abs = std::fmax(max_abs, std::fabs(ref - D[m * 64 + n]));
                    ref_max = std::fmax(ref_max, std::fabs(ref));
                }
            max_rel = max_abs / ref_max;
            printf("mode %d (%s) reps %d: max |err| / max |ref| = %.3e   %.1f cycles/rep\n", mode,
                   mode ? "3xTF32 vs fp64 A.B" : "1xTF32 vs fp64 A.Bhi", reps, max_rel, (double)cyc / reps);
            if (max_rel > (mode ? 1e-5 : 2e-3)) ++fails;
        }
    }
    {
        long long c[4];
        long long* dcy;
        cudaMalloc(&dcy, 32);
        for (int reps : {16, 256}) {
            tput<<<1, 128>>>(dBh, reps, dcy);
            cudaDeviceSynchronize();
            cudaMemcpy(c, dcy, 32, cudaMemcpyDeviceToHost);
            printf("reps %d: MMA 128x64x8 tf32 %.1f cyc each; tcgen05.st 4 warps x 8 KB %.1f cyc; ld %.1f cyc\n", reps,
                   (double)c[0] / (24.0 * reps), (double)c[1] / reps, (double)c[2] / reps);
        }
    }
    printf(fails ? "FAIL\n" : "PASS\n");
    return fails;
}
