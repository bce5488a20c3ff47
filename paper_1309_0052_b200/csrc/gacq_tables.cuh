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

// Hermitian half [n_prn][17][kCcRow] (column 31 repeats column 0) of Cc[k] = conj(DFT_1023(chip))[k] / 1023 at
// [k mod 33][k mod 31], k2 = k mod 33 <= 16 (gacq_pfa.cuh layout). One warp per (prn, k):
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
    if (lane == 0) {
        const float2 v = make_float2((float)(re / kChips), (float)(-im / kChips));
        float2* row = ccp + (size_t)i * kCcHalf + (k % 33) * kCcRow;
        row[k % 31] = v;
        if (k % 31 == 0) row[31] = v;  // column 31 repeats column 0 (gacq_pfa.cuh kCcRow)
    }
}

}  // namespace gacq

namespace gacq {

// ---- on-device synthetic snapshots (perf inputs, never parity) ----
// One satellite of one snapshot with the reference's fixed-point NCO words (gnss_signal.py:157-186
// with kernels.py:56-70): code_p0 = code_phase_to_fixed((-code_phase * 1.023e6/fs) mod 1023),
// carrier_p0 = carrier_phase_to_fixed((-carrier_phase) mod 1), carrier_step for -doppler.
struct SynthSat {
    uint64_t code_p0, carrier_p0, carrier_step;
    int32_t prn_index;  // 0..31
    float amp;          // float32 scale (10^((cn0 - cn0_ref)/20))
};

// Philox4x32-10 (counter-based; the reference's PCG64 stream is not reproduced)
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
        const unsigned hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += 0x9E3779B9u;
        key.y += 0xBB67AE85u;
    }
    return ctr;
}

// out[s][k] = sum over the snapshot's satellites, in order, of amp * code(k) * carrier(k)
// (complex64, as the reference sums them), plus sigma * (N(0,1) + i N(0,1)) rounded to complex64
// when sigma > 0 (Box-Muller in float64 on Philox uniforms, gnss_signal.py:136-154).
__global__ void gacq_synth_kernel(const SynthSat* __restrict__ sats, int n_sat, int64_t n_snap, int64_t n,
                                  uint64_t code_step, const int8_t* __restrict__ chips, double inv, double sigma,
                                  uint64_t seed, float2* __restrict__ out) {
    const int64_t total = n_snap * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / n;
        const uint64_t k = (uint64_t)(i - s * n);
        float re = 0.f, im = 0.f;
        for (int j = 0; j < n_sat; ++j) {
            const SynthSat st = sats[s * n_sat + j];
            const uint64_t cph = (st.code_p0 + k * code_step) % (1023ull << 42);
            const float chip = (float)chips[st.prn_index * kChips + (int)(cph >> 42)];
            const uint64_t ph = (st.carrier_p0 + k * st.carrier_step) & ((1ull << 48) - 1);
            double sn, cs;
            sincos(__dmul_rn((double)ph, inv), &sn, &cs);
            // code (+-1, 0) x carrier (cos, -sin): exact; then x amp; summed in draw order
            re = __fadd_rn(re, __fmul_rn(chip * (float)cs, st.amp));
            im = __fadd_rn(im, __fmul_rn(chip * (float)(-sn), st.amp));
        }
        if (sigma > 0.0) {
            const uint4 r = philox(make_uint4((unsigned)i, (unsigned)(i >> 32), 0x5851F42Du, 0x14057B7Eu),
                                   make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
            const double u1 = 1.0 - ((double)(((uint64_t)r.x << 21) ^ r.y) * 0x1p-53);  // (0, 1]
            const double u2 = (double)(((uint64_t)r.z << 21) ^ r.w) * 0x1p-53;
            const double rad = sqrt(-2.0 * log(u1));
            double s2, c2;
            sincospi(2.0 * u2, &s2, &c2);
            re = __fadd_rn(re, (float)(sigma * (rad * c2)));
            im = __fadd_rn(im, (float)(sigma * (rad * s2)));
        }
        out[i] = make_float2(re, im);
    }
}

}  // namespace gacq
