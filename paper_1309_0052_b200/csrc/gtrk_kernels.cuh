// gtrk_kernels.cuh -- tracking E/P/L correlators (tracking.py:126-165) on sm_100a.
//
// Each of a channel's six correlator components (ie, qe, ip, qp, il, ql) is a complex64 running
// sum taken left to right over the block (kernels.py:93-95, dsp.py:186-201): a serial chain of
// n float32 additions whose order is fixed by bit-exactness. The kernel is built around those
// chains: one CTA serves kEplChans = 32 channels, and
//   - six consumer warps run the chains: warp j = 2 corr + comp, lane = channel, so every
//     chain is one lane and a warp advances 32 of them per instruction;
//   - kEplProducers (16) producer warps stream the block through shared memory in chunks of
//     kEplChunk samples (double-buffered, named barriers), writing for every (channel,
//     sample) the six signed terms +-re / +-im of the wiped sample. The wipe is bit-exact:
//     exact fixed-point NCOs (48-bit carrier mask, 42-bit code modulus 1023 * 2^42) evaluated
//     statelessly at sample k as p0 + k step, the carrier replica float32(cos), float32(-sin)
//     of the float64 angle (kernels.py:106-114), the complex64 product of kernels.py:78-86,
//     and the E/P/L chips (kernels.py:116-128); chip x sample is exact, so each term is the
//     value the reference adds.
// Shared memory no longer grows with n (a chain needs one chunk at a time), so 384 chains
// run per SM instead of the 30 of a CTA-per-channel layout.
#pragma once
#include <cstdint>

#include "codelets.cuh"
#include "../../include/gacq.h"

namespace gacq {

constexpr uint64_t kCarrierMask = (1ull << 48) - 1;
constexpr uint64_t kCodeMod = 1023ull << 42;
constexpr int kEplChans = 32;                       // channels per CTA: one per chain lane
constexpr int kEplChunk = 64;                       // samples per chunk
#ifndef GACQ_EPL_PRODUCERS
#define GACQ_EPL_PRODUCERS 16
#endif
constexpr int kEplProducers = GACQ_EPL_PRODUCERS;   // producer warps (a divisor of 32)
constexpr int kEplThreads = 32 * (6 + kEplProducers);
constexpr int kEplRow = kEplChans + 1;              // padded: producers write along k, lanes = samples
constexpr int kEplSmem = 2 * 6 * kEplChunk * kEplRow * (int)sizeof(float);  // 101,376 B

// named barriers with immediate ids (a register id makes ptxas reserve all 16)
template <int kId>
__device__ __forceinline__ void epl_bar_sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(kId), "n"(kEplThreads) : "memory");
}
template <int kId>
__device__ __forceinline__ void epl_bar_arrive() {
    asm volatile("bar.arrive %0, %1;" ::"n"(kId), "n"(kEplThreads) : "memory");
}
// buffer b's full (1 + b) / empty (3 + b) barrier
__device__ __forceinline__ void epl_full_sync(int b) { if (b) epl_bar_sync<2>(); else epl_bar_sync<1>(); }
__device__ __forceinline__ void epl_full_arrive(int b) { if (b) epl_bar_arrive<2>(); else epl_bar_arrive<1>(); }
__device__ __forceinline__ void epl_empty_sync(int b) { if (b) epl_bar_sync<4>(); else epl_bar_sync<3>(); }
__device__ __forceinline__ void epl_empty_arrive(int b) { if (b) epl_bar_arrive<4>(); else epl_bar_arrive<3>(); }

// grid: ceil(n_chan / 32) CTAs of kEplThreads; dynamic smem kEplSmem.
// Barrier ids: 1 + b = chunk buffer b full (producers arrive, consumers wait),
//              3 + b = buffer b empty (consumers arrive, producers wait).
// out[c * 6 + 2 corr + comp]. Host guarantees code_p0 + (n - 1) code_step < 2^64.
__global__ void __launch_bounds__(kEplThreads, 2) gacq_epl_kernel(const cx* __restrict__ blocks, int n,
                                                                  const gacq_epl_chan* __restrict__ chans,
                                                                  int64_t n_chan, const int8_t* __restrict__ chips,
                                                                  float* __restrict__ out) {
    extern __shared__ float sv[];  // [2][6][kEplChunk][kEplRow]
    __shared__ gacq_epl_chan sch[kEplChans];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * kEplChans;
    const int nc = (int)min((int64_t)kEplChans, n_chan - c0);
    const int n_chunks = (n + kEplChunk - 1) / kEplChunk;
    if (threadIdx.x < nc) sch[threadIdx.x] = chans[c0 + threadIdx.x];
    __syncthreads();

    if (warp < 6) {
        // consumer: chain (corr = warp / 2, comp = warp % 2) of channel c0 + lane
        float acc = 0.f;
        for (int c = 0; c < n_chunks; ++c) {
            const int b = c & 1;
            epl_full_sync(b);
            const float* r = sv + ((b * 6 + warp) * kEplChunk) * kEplRow + lane;
            const int kn = min(kEplChunk, n - c * kEplChunk);
            if (kn == kEplChunk) {
#pragma unroll 16
                for (int k = 0; k < kEplChunk; ++k) acc = __fadd_rn(acc, r[k * kEplRow]);
            } else {
                for (int k = 0; k < kn; ++k) acc = __fadd_rn(acc, r[k * kEplRow]);
            }
            epl_empty_arrive(b);
        }
        if (lane < nc) out[(c0 + lane) * 6 + warp] = acc;
        return;
    }
    // producers: warp pw owns channels pw + kEplProducers j; lane = sample in a half chunk
    const int pw = warp - 6;
    const double inv = 6.283185307179586 / 281474976710656.0;  // TWO_PI / 2^48 (kernels.py:110)
    for (int c = 0; c < n_chunks; ++c) {
        const int b = c & 1;
        if (c >= 2) epl_empty_sync(b);  // chunk c - 2 consumed
        float* base = sv + (b * 6) * kEplChunk * kEplRow;
#pragma unroll 1
        for (int j = 0; j < kEplChans / kEplProducers; ++j) {
            const int cl = pw + kEplProducers * j;
            if (cl >= nc) break;  // warp-uniform
            const gacq_epl_chan& d = sch[cl];
            const int8_t* code = chips + (d.prn - 1) * 1024;
#pragma unroll
            for (int h = 0; h < kEplChunk / 32; ++h) {
                const int kl = 32 * h + lane;
                const int k = c * kEplChunk + kl;
                float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (k < n) {
                    const uint64_t pc = (d.carrier_p0 + (uint64_t)k * d.carrier_step) & kCarrierMask;
                    double s, co;
                    sincos((double)pc * inv, &s, &co);
                    const cx w = cmul_exact(__ldg(&blocks[d.block_offset + k]), pk((float)co, (float)(-s)));
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        // ((p0 + k step) mod 1023 2^42) >> 42 = ((p0 + k step) >> 42) mod 1023
                        const unsigned q = (unsigned)((d.code_p0[i] + (uint64_t)k * d.code_step) >> 42);
                        const bool pos = __ldg(&code[q % 1023u]) > 0;
                        v[2 * i] = pos ? re(w) : -re(w);
                        v[2 * i + 1] = pos ? im(w) : -im(w);
                    }
                }
#pragma unroll
                for (int i = 0; i < 6; ++i) base[(i * kEplChunk + kl) * kEplRow + cl] = v[i];
            }
        }
        epl_full_arrive(b);
    }
    // drain: match the consumers' arrivals on the last two buffers' empty barriers
    for (int c = max(n_chunks, 2); c < n_chunks + 2; ++c) epl_empty_sync(c & 1);
}

}  // namespace gacq
