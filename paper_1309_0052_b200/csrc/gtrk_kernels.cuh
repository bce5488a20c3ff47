// gtrk_kernels.cuh -- tracking E/P/L correlators (tracking.py:126-165) on sm_100a.
//
// One CTA per channel, bit-identical to the reference:
//   (A) all threads: exact fixed-point NCO stepping (48-bit carrier mask, 42-bit code
//       modulus 1023*2^42), the carrier replica float32(cos), float32(-sin) of the float64
//       angle (kernels.py:106-114), the bit-exact complex64 wipe product (kernels.py:78-86)
//       into shared memory, plus the E/P/L chip of every sample (kernels.py:116-128);
//   (B) six lanes: the documented left-to-right complex64 running sums of the dot products
//       (kernels.py:93-95, dsp.py:186-201) -- chip x sample is exact, so each lane adds
//       +/-re or +/-im of the wiped samples in sample order, exactly as the reference.
#pragma once
#include <cstdint>

#include "codelets.cuh"
#include "../../include/gacq.h"

namespace gacq {

constexpr int kTrkThreads = 256;
constexpr uint64_t kCarrierMask = (1ull << 48) - 1;
constexpr uint64_t kCodeMod = 1023ull << 42;
constexpr int kTrkMaxSmem = 227 * 1024;

// dynamic smem: n complex64 wiped samples + 3*n int8 chips
__global__ void __launch_bounds__(kTrkThreads) gacq_epl_kernel(const cx* __restrict__ blocks, int n,
                                                               const gacq_epl_chan* __restrict__ chans,
                                                               const int8_t* __restrict__ chips,
                                                               float* __restrict__ out) {
    extern __shared__ cx trk_smem[];
    cx* w = trk_smem;
    int8_t* sgn = reinterpret_cast<int8_t*>(trk_smem + n);  // [3][n]
    const int t = threadIdx.x;
    const gacq_epl_chan ch = chans[blockIdx.x];
    const cx* x = blocks + ch.block_offset;
    const int8_t* code = chips + (ch.prn - 1) * 1024;
    const double inv = 6.283185307179586 / 281474976710656.0;  // TWO_PI / 2^48 (kernels.py:110)

    uint64_t pc = (ch.carrier_p0 + (uint64_t)t * ch.carrier_step) & kCarrierMask;
    const uint64_t dpc = ((uint64_t)kTrkThreads * ch.carrier_step) & kCarrierMask;
    uint64_t pcode[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) pcode[i] = (ch.code_p0[i] + (uint64_t)t * ch.code_step) % kCodeMod;
    const uint64_t dcode = ((uint64_t)kTrkThreads * ch.code_step) % kCodeMod;
    for (int k = t; k < n; k += kTrkThreads) {
        double s, c;
        sincos((double)pc * inv, &s, &c);
        w[k] = cmul_exact(__ldg(&x[k]), pk((float)c, (float)(-s)));
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            sgn[i * n + k] = __ldg(&code[pcode[i] >> 42]);
            pcode[i] += dcode;
            if (pcode[i] >= kCodeMod) pcode[i] -= kCodeMod;
        }
        pc = (pc + dpc) & kCarrierMask;
    }
    __syncthreads();
    if (t < 6) {
        const int corr = t >> 1, comp = t & 1;
        const float* wf = reinterpret_cast<const float*>(w) + comp;
        const int8_t* sg = sgn + corr * n;
        float acc = 0.f;
        for (int k = 0; k < n; ++k) acc = __fadd_rn(acc, sg[k] > 0 ? wf[2 * k] : -wf[2 * k]);
        out[(int64_t)blockIdx.x * 6 + 2 * corr + comp] = acc;
    }
}

}  // namespace gacq
