// gacq_kernels.cuh -- shared pieces of the acquisition hot path (sm_100a).
//
// Reference path: gnssperf/acquisition.py:128-159 (hot loop 138-149).
//
//   wipe_fold           : bit-exact carrier wipe-off (kernels.py:78-86) of one coherent block,
//                         folded over its K code periods into the transposed table K1 reads.
//   gacq_reduce_kernel  : K3, per (snapshot, prn): merge the bin rows (peak desc, bin asc).
//   cp.async helpers.
// The 1023-point prime-factor K1/K2 are in gacq_pfa.cuh, the generic power-of-two path in
// gacq_generic.cuh (DESIGN.md sections 3-5, 14).
#pragma once
#include <cstdint>

#include "codelets.cuh"
#include "../../include/gacq.h"

namespace gacq {

constexpr int kChips = 1023;
constexpr int kRow = 1024;      // row stride of the transposed wiped block (floats / float2)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Non-finite detection on the samples K1 loads: fin = min over 32-bit words of
// (~word & exponent mask), which is 0 iff some word is a NaN or an infinity (all exponent bits
// set). Two ALU operations per word, off the FP32 pipe.
__device__ __forceinline__ unsigned fin_word(unsigned long long v, unsigned fin) {
    return min(fin, min(~(unsigned)v & 0x7f800000u, ~(unsigned)(v >> 32) & 0x7f800000u));
}
__device__ __forceinline__ unsigned fin_word(ulonglong2 v, unsigned fin) { return fin_word(v.x, fin_word(v.y, fin)); }

// Row stride of the transposed wiped block wt[k][m] = wbar[D m + k]: the +16/D pad makes
// both the wipe stores (consecutive n) and the chip-sum loads (consecutive m) conflict-free.
__host__ __device__ constexpr int fwd_ws(int D) { return kRow + (D <= 16 ? 16 / D : 0); }

// Sample sources of the wipe: complex64, or integer I/Q dequantized in registers exactly as
// read_if_file does (iffile.py:95-98): float32(float64(q) * s), s = scale / limit from the host.
// ld2(i, a, b) returns samples 2i and 2i+1 of the block (one load), ld1(n) sample n.
struct SrcC64 {
    const cx* x;
    __device__ __forceinline__ void ld2(int64_t i, cx& a, cx& b) const {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(x) + i);
        a = v.x;
        b = v.y;
    }
    __device__ __forceinline__ cx ld1(int64_t n) const { return __ldg(x + n); }
    __device__ __forceinline__ SrcC64 at(int64_t n) const { return {x + n}; }
    __device__ __forceinline__ bool aligned() const { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; }
};
__device__ __forceinline__ float deq(int q, double s) { return __double2float_rn(__dmul_rn((double)q, s)); }
// int8: the 256 possible values come from a per-CTA shared-memory table of the same products
// (lut[q + 128] = deq(q, s)), so the wipe load does no float64 work
struct SrcI8 {
    const signed char* q;  // interleaved I/Q bytes
    const float* lut;      // shared memory, 256 entries
    __device__ __forceinline__ float v(int b) const { return lut[b + 128]; }
    __device__ __forceinline__ void ld2(int64_t i, cx& a, cx& b) const {
        const int w = __ldg(reinterpret_cast<const int*>(q) + i);
        a = pk(v((signed char)(w & 0xff)), v((signed char)((w >> 8) & 0xff)));
        b = pk(v((signed char)((w >> 16) & 0xff)), v(w >> 24));
    }
    __device__ __forceinline__ cx ld1(int64_t n) const { return pk(v(__ldg(q + 2 * n)), v(__ldg(q + 2 * n + 1))); }
    __device__ __forceinline__ SrcI8 at(int64_t n) const { return {q + 2 * n, lut}; }
    __device__ __forceinline__ bool aligned() const { return (reinterpret_cast<uintptr_t>(q) & 3) == 0; }
};
struct SrcI16 {
    const short* q;
    double s;
    __device__ __forceinline__ void ld2(int64_t i, cx& a, cx& b) const {
        const int2 w = __ldg(reinterpret_cast<const int2*>(q) + i);
        a = pk(deq((short)(w.x & 0xffff), s), deq(w.x >> 16, s));
        b = pk(deq((short)(w.y & 0xffff), s), deq(w.y >> 16, s));
    }
    __device__ __forceinline__ cx ld1(int64_t n) const { return pk(deq(__ldg(q + 2 * n), s), deq(__ldg(q + 2 * n + 1), s)); }
    __device__ __forceinline__ SrcI16 at(int64_t n) const { return {q + 2 * n, s}; }
    __device__ __forceinline__ bool aligned() const { return (reinterpret_cast<uintptr_t>(q) & 7) == 0; }
};

// Wipe-off (bit-exact, acquisition.py:141) of one coherent block x (K code periods) with the
// carrier replica c, folded over the K periods into the transposed table
// wt[k][m] = wbar[D m + k]; wt[k][1023] repeats wt[k][0] (circular chip m+1). Coalesced,
// two samples per load. All NT threads of the CTA take part; ends with a barrier whose
// result is true when any sample of x (after dequantization) is a NaN or an infinity.
template <int D, int NT, class Src>
__device__ __forceinline__ bool wipe_fold(const Src x, const cx* __restrict__ c, int P, int K,
                                          cx* __restrict__ wt) {
    constexpr int WS = fwd_ws(D);
    auto put = [&](int n, cx w) {
        const int m = n / D, k = n - m * D;
        wt[k * WS + m] = w;
        if (m == 0) wt[k * WS + kChips] = w;
    };
    const bool vec = x.aligned() && (reinterpret_cast<uintptr_t>(c) & 15) == 0 && (P & 1) == 0;
    unsigned fin = 0x7f800000u;
    if (vec) {
        const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(c);
        const int np = P / 2;
#ifndef GACQ_WIPE_U
#define GACQ_WIPE_U 4
#endif
        constexpr int U = GACQ_WIPE_U;  // load pairs in flight per thread
        if (K == 1) {  // one code period per block (coherent_ms = 1): no fold, twice the loads in flight
            constexpr int U1 = 2 * U;
            for (int base = threadIdx.x; base < np; base += U1 * NT) {
                cx xa[U1], xb[U1];
                ulonglong2 cv[U1];
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        x.ld2(i, xa[u], xb[u]);
                        cv[u] = __ldg(c2 + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        fin = fin_word(xa[u], fin_word(xb[u], fin));
                        put(2 * i, cmul_exact(xa[u], cv[u].x));
                        put(2 * i + 1, cmul_exact(xb[u], cv[u].y));
                    }
                }
            }
            return __syncthreads_or(fin == 0u);
        }
        for (int base = threadIdx.x; base < np; base += U * NT) {
            cx w[U][2];
            for (int k = 0; k < K; ++k) {
                cx xa[U], xb[U];
                ulonglong2 cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        x.ld2((int64_t)k * np + i, xa[u], xb[u]);
                        cv[u] = __ldg(c2 + k * np + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (base + u * NT < np) fin = fin_word(xa[u], fin_word(xb[u], fin));
                    const cx p0 = cmul_exact(xa[u], cv[u].x), p1 = cmul_exact(xb[u], cv[u].y);
                    w[u][0] = k ? add2(w[u][0], p0) : p0;
                    w[u][1] = k ? add2(w[u][1], p1) : p1;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = base + u * NT;
                if (i < np) {
                    put(2 * i, w[u][0]);
                    put(2 * i + 1, w[u][1]);
                }
            }
        }
    } else {
        for (int n = threadIdx.x; n < P; n += NT) {
            const cx x0 = x.ld1(n);
            fin = fin_word(x0, fin);
            cx acc = cmul_exact(x0, __ldg(&c[n]));
            for (int k = 1; k < K; ++k) {
                const cx xk = x.ld1((int64_t)k * P + n);
                fin = fin_word(xk, fin);
                acc = add2(acc, cmul_exact(xk, __ldg(&c[k * P + n])));
            }
            put(n, acc);
        }
    }
    return __syncthreads_or(fin == 0u);
}

// Integer I/Q -> complex64, bit-identical to read_if_file (iffile.py:95-98):
// float32(float64(q) * s) per component with s = scale / limit computed on the host.
// n = snapshots * span samples; snapshot j's sample k sits at src[2 (j*src_stride + k)].
template <typename T>
__global__ void gacq_dequant_kernel(const T* __restrict__ src, int64_t src_stride, cx* __restrict__ dst,
                                    int64_t span, int64_t n, double s) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / span, k = i - j * span;
        const T* q = src + 2 * (j * src_stride + k);
        dst[i] = pk((float)((double)q[0] * s), (float)((double)q[1] * s));
    }
}

// one warp per (snapshot, prn): merge bin rows -- np.argmax order (acquisition.py:151):
// highest peak, ties -> lowest bin (the row's own first lag is already the lowest)
__global__ void gacq_reduce_kernel(const gacq_row* __restrict__ rows_bin, gacq_row* __restrict__ rows,
                                   int64_t n_rows, int B) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_rows) return;
    const gacq_row* src = rows_bin + w * B;
    float best = -1.f;
    int bb = 0x7fffffff;  // stays when every peak is NaN (non-finite input, flagged by K1)
    for (int b = lane; b < B; b += 32) {
        const float p = src[b].peak;
        if (p > best) { best = p; bb = b; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int ob = __shfl_xor_sync(0xffffffffu, bb, off);
        if (ov > best || (ov == best && ob < bb)) { best = ov; bb = ob; }
    }
    if (lane == 0) rows[w] = src[bb < B ? bb : 0];
}

}  // namespace gacq
