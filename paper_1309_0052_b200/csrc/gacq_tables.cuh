// gacq_tables.cuh -- on-device construction of a plan's tables.
//
//   gacq_ca_chips_kernel     : C/A Gold codes, cacode.py:41-58 (G1 taps 3,10; G2 phase select),
//                              one thread per PRN running the two 10-stage LFSRs.
//   gacq_carrier_kernel      : wipe-off replicas of every Doppler bin at phase 0,
//                              kernels.py:106-114 / 175-185 (48-bit NCO, float64 angle,
//                              cos/-sin rounded to complex64) -- bit-identical to the reference
//                              (tests/test_gpu_tables.py compares all bins with the oracle).
//   gacq_code_spectrum_kernel: conj(DFT_1023(chips)) / 1023 in float64 (acquisition.py:84-105
//                              restated for the chip domain, see gacq_pfa.cuh), Hermitian half.
#pragma once
#include <cstdint>

#include "gacq_pfa.cuh"

namespace gacq {

// G2 output taps per PRN (cacode.py:22-29), 1-based
__constant__ int8_t c_g2_select[32][2] = {{2, 6},  {3, 7},  {4, 8},  {5, 9},  {1, 9},  {2, 10}, {1, 8},  {2, 9},
                                          {3, 10}, {2, 3},  {3, 4},  {5, 6},  {6, 7},  {7, 8},  {8, 9},  {9, 10},
                                          {1, 4},  {2, 5},  {3, 6},  {4, 7},  {5, 8},  {6, 9},  {1, 3},  {4, 6},
                                          {5, 7},  {6, 8},  {7, 9},  {8, 10}, {1, 6},  {2, 7},  {3, 8},  {4, 9}};

// chips[i][0..1022] = +1 / -1 for prns[i] (bit 1 -> +1, cacode.py:56-57)
__global__ void gacq_ca_chips_kernel(const int32_t* __restrict__ prns, int n_prn, int8_t* __restrict__ chips) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_prn) return;
    const int s1 = c_g2_select[prns[i] - 1][0] - 1, s2 = c_g2_select[prns[i] - 1][1] - 1;
    unsigned g1 = 0x3ffu, g2 = 0x3ffu;  // bit j = register stage j+1, all ones
    for (int n = 0; n < kChips; ++n) {
        const unsigned out = ((g1 >> 9) ^ (g2 >> s1) ^ (g2 >> s2)) & 1u;
        chips[i * kChips + n] = out ? 1 : -1;
        const unsigned f1 = ((g1 >> 2) ^ (g1 >> 9)) & 1u;
        const unsigned f2 = ((g2 >> 1) ^ (g2 >> 2) ^ (g2 >> 5) ^ (g2 >> 7) ^ (g2 >> 8) ^ (g2 >> 9)) & 1u;
        g1 = ((g1 << 1) | f1) & 0x3ffu;
        g2 = ((g2 << 1) | f2) & 0x3ffu;
    }
}

// out[b][k] = complex64(cos th, -sin th), th = float64((k * step_b) mod 2^48) * inv,
// inv = 2 pi / 2^48 as the host computes it (kernels.py:106-114)
__global__ void gacq_carrier_kernel(const uint64_t* __restrict__ steps, int B, int n_coh, double inv,
                                    float2* __restrict__ out) {
    const int64_t total = (int64_t)B * n_coh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(i / n_coh);
        const uint64_t k = (uint64_t)(i - (int64_t)b * n_coh);
        const uint64_t ph = (k * steps[b]) & ((1ull << 48) - 1);
        const double th = __dmul_rn((double)ph, inv);
        double s, c;
        sincos(th, &s, &c);
        out[i] = make_float2((float)c, (float)(-s));
    }
}

// Hermitian half [n_prn][17][32] of Cc[k] = conj(DFT_1023(chip))[k] / 1023 at [k mod 33][k mod 31],
// k2 = k mod 33 <= 16 (gacq_pfa.cuh layout; column 31 stays zero). One warp per (prn, k):
// lanes stride the 1023 chips, float64 partial sums combined by shuffles.
__global__ void gacq_code_spectrum_kernel(const int8_t* __restrict__ chips, int n_prn, float2* __restrict__ ccp) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n_prn * kChips) return;
    const int i = warp / kChips, k = warp % kChips;
    if (k % 33 > 16) return;
    double re = 0.0, im = 0.0;
    for (int j = lane; j < kChips; j += 32) {
        const int m = (int)(((int64_t)j * k) % kChips);
        double s, c;
        sincospi(2.0 * m / kChips, &s, &c);
        const double x = chips[i * kChips + j];
        re += x * c;
        im -= x * s;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) ccp[(size_t)i * kCcHalf + (k % 33) * 32 + k % 31] = make_float2((float)(re / kChips), (float)(-im / kChips));
}

}  // namespace gacq
