// gacq_tc.cuh -- K2 of the 1023-point prime-factor path with the 31-point stage on the
// tensor cores (tcgen05, kind::tf32, split into three TF32 products for FP32 accuracy).
//
// Reference path: gnssperf/acquisition.py:138-159 (IFFT, |.|^2, noncoherent sum, argmax/floor).
//
// Same algorithm and item scheduling as gacq_corr_pfa_kernel (gacq_pfa.cuh); the difference is
// where the 31-point inverse DFT over k1 runs. For each (round, phase) the 4 warps of a CTA each
// hold one transform; after the 33-point stage (FP32 pipe, lanes k1 < 31), rows q2 = 0..31 of
// the 4 transforms form a 128 x 64 real matrix A (row = 32 w + q2, column 2 k1 + {re, im}), and
//     D = A . B,   B[2 k1 + c][2 q1 + c'] = the real form of exp(+2 pi i k1 q1 / 31)
// is one M = 128, N = 64, K = 64 tensor-core product. FP32 accuracy comes from the split
//     A.B ~= A.Bhi + A.Blo + Alo.Bhi,   x = hi(x) + lo(x), hi = top 19 bits (what TF32 reads)
// (max error 1.6e-6 of the row scale vs float64, tools/tc_probe.cu). A lives in TMEM (written
// with tcgen05.st from the warp that owns its 32 lanes), B in shared memory (K-major core
// matrices, tc_util.cuh), D in TMEM; the warps read D back with tcgen05.ld and accumulate
// |D|^2 over rounds in registers. Row q2 = 32 stays on the FP32 pipe (coop31), overlapping the
// tensor-core work. Used when 4 | D (4.092 / 8.184 / 16.368 MHz), gacq.cu.
#pragma once
#include "gacq_pfa.cuh"
#include "tc_util.cuh"

namespace gacq {

constexpr int kTcWarps = 4;
constexpr int kTcB = 64 * 64;  // floats per B matrix
constexpr int kTcScr = 34;     // coop31 scratch per warp (cx)
// dynamic smem: B hi | B lo | Z buffer per warp | coop31 scratch per warp | Cc half | Z mbarriers
__host__ __device__ constexpr int corr_tc_smem() {
    return 2 * kTcB * 4 + kTcWarps * (kBuf + kTcScr) * 8 + kCcHalf * 8 + kTcWarps * 8;
}
// float index of B[n][k] in the K-major no-swizzle core-matrix layout (LBO 128 B, SBO 2048 B)
__host__ __device__ constexpr int tc_b_off(int n, int k) { return (n >> 3) * 512 + (k >> 2) * 32 + (n & 7) * 4 + (k & 3); }

// Persistent like gacq_corr_pfa_kernel; 4 warps, warp w owns phases [w PW, (w+1) PW), PW = D/4.
// tcB: [2][kTcB] floats, B hi then B lo, already in tc_b_off order.
template <bool kRegs>
__global__ void __launch_bounds__(32 * kTcWarps, 3) gacq_corr_tc_kernel(CorrPfaArgs a, const float4* __restrict__ tcB) {
    __shared__ float red_v[kTcWarps], red_f[kTcWarps];
    __shared__ int red_i[kTcWarps];
    __shared__ long long s_claim, s_claim0;  // s_claim0: the first claim (read before the item loop)
    __shared__ float s_coef[15][32];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_mma_bar;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* sB = reinterpret_cast<float*>(smem_raw);
    cx* zbuf = reinterpret_cast<cx*>(smem_raw + 2 * kTcB * 4);
    cx* scrb = zbuf + kTcWarps * kBuf;
    cx* ccs = scrb + kTcWarps * kTcScr;
    unsigned long long* zbar = reinterpret_cast<unsigned long long*>(ccs + kCcHalf);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t item = blockIdx.x;
    if (item >= a.n_items) return;

    for (int i = threadIdx.x; i < 2 * kTcB / 4; i += blockDim.x) reinterpret_cast<float4*>(sB)[i] = tcB[i];
    for (int i = threadIdx.x; i < 15 * 32; i += blockDim.x) s_coef[i >> 5][i & 31] = coop31_coef(i & 31, (i >> 5) + 1);
    if (w == 0) tc::tmem_alloc<128>(&s_tmem);
    if (lane == 0) {
        mbar_init(&zbar[w], 1);
        if (w == 0) mbar_init(&s_mma_bar, 1);
        fence_mbar_init();
    }
    tc::fence_proxy_async();  // sB -> tensor core
    auto load_cc = [&](int64_t it) {
        const char* g = reinterpret_cast<const char*>(a.Cc + (it % a.n_prn) * kCcHalf);
        for (int i = threadIdx.x; i < kCcHalf / 2; i += blockDim.x) cp_async16(ccs + 2 * i, g + 16 * i);
        cp_async_commit();
    };
    if (threadIdx.x == 0) s_claim0 = (long long)gridDim.x + (long long)atomicAdd(a.counter, 1ull);
    load_cc(item);
    const int rho0 = w * a.PW;
    const int nph = a.PW;
    const int64_t pair_span = (int64_t)a.R * a.D * kBuf;
    auto zbase = [&](int64_t it) { return a.Z + (it / a.n_prn) * pair_span + rho0 * kBuf; };
    cx* buf = zbuf + w * kBuf;
    cx* scr = scrb + w * kTcScr;
    tc::tc_fence_before();
    __syncthreads();  // mbarrier inits, TMEM address, sB, s_coef
    tc::tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t tA = tmem + ((uint32_t)(32 * w) << 16);  // this warp's lanes, A at columns [0, 64)
    const uint32_t tD = tA + 64;                             // D at columns [64, 128)
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    const uint64_t dBh = tc::sdesc(tc::smem_u32(sB), 128, 2048);
    const uint64_t dBl = tc::sdesc(tc::smem_u32(sB + kTcB), 128, 2048);
    unsigned mma_phase = 0;
    unsigned t = 0;  // this warp's transform count = Z mbarrier phase
    __syncwarp();
    if (lane == 0) bulk_load(buf, zbase(item), kSpecBytes, &zbar[w]);
    float* rows = a.row_scratch + (int64_t)blockIdx.x * a.D * kChips;
    const int pl = lane == 0 ? 0 : 31 - lane;
    cp_async_wait_all();
    __syncthreads();
    int64_t next = s_claim0;  // s_claim itself is rewritten by thread 0 at the end of the first item

    for (;;) {
        long long claim = 0;
        if (threadIdx.x == 0 && next < a.n_items) claim = (long long)gridDim.x + (long long)atomicAdd(a.counter, 1ull);
        const int64_t lp = item / a.n_prn;
        const int pi = (int)(item % a.n_prn);
        const cx* zb = zbase(item);
        const cx* zn = next < a.n_items ? zbase(next) : nullptr;

        float best = -1.f;
        int bidx = 0x7fffffff;
        float acc[31], accx[2];
        int rd = 0, ph = 0;
#pragma unroll 1
        for (;; ++t) {
            if (rd == 0) {
#pragma unroll
                for (int i = 0; i < 31; ++i) acc[i] = 0.f;
                accx[0] = accx[1] = 0.f;
            }
            const bool last_rd = rd + 1 == a.R;
            const bool last = last_rd && ph + 1 == nph;
            mbar_wait(&zbar[w], t & 1);
            cx* E = buf;
            // Z * Cc and the 33-point stage over k2 (FP32 pipe); E[q2][k1] written in place
            if (lane < 31) {
                const cx* Ec = E + lane;
                dft33_stream<1>(
                    [&](int k2, int dep) {
                        return k2 <= 16 ? cmul(Ec[k2 * 32 + dep], ccs[k2 * 32 + lane + dep])
                                        : cmul_conj(Ec[k2 * 32 + dep], ccs[(33 - k2) * 32 + pl + dep]);
                    },
                    a.zero, [&](int q2, cx v) {
                        if (q2 == 0) __syncwarp(0x7fffffffu);
                        E[q2 * 31 + lane] = v;
                    });
            }
            __syncwarp();
            // this lane's row q2 = lane -> the A operand; row 32 element of column k1 = lane
            uint32_t v[64];
            {
                const cx* Er = E + lane * 31;
#pragma unroll
                for (int k1 = 0; k1 < 31; ++k1) {
                    const cx x = Er[k1];
                    v[2 * k1] = (uint32_t)x;
                    v[2 * k1 + 1] = (uint32_t)(x >> 32);
                }
                v[62] = v[63] = 0u;
            }
            const cx e = lane < 31 ? E[32 * 31 + lane] : czero();
            __syncwarp();
            if (lane == 0) {  // the buffer is free: prefetch this warp's next spectrum
                const cx* nsrc = !last ? zb + ((last_rd ? 0 : rd + 1) * a.D + (last_rd ? ph + 1 : ph)) * kBuf : zn;
                if (nsrc) bulk_load(buf, nsrc, kSpecBytes, &zbar[w]);
            }
            // pass 1: A = x (the tensor core reads hi(x)); D = A.Bhi + A.Blo
            tc::tmem_st64(tA, v);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            __syncthreads();
            if (threadIdx.x == 0) {
                tc::tc_fence_after();
#pragma unroll
                for (int s = 0; s < 8; ++s) tc::mma_tf32_ts(tmem + 64, tmem + 8 * s, dBh + 16 * s, idesc, s > 0);
#pragma unroll
                for (int s = 0; s < 8; ++s) tc::mma_tf32_ts(tmem + 64, tmem + 8 * s, dBl + 16 * s, idesc, true);
                tc::mma_commit(&s_mma_bar);
            }
            // row 32 on the FP32 pipe meanwhile
            coop31<1>(e, lane, [&](int j) { return s_coef[j - 1][lane]; }, scr,
                      [&](int sl, int, cx val) { accx[sl] = pow_acc(val, accx[sl]); });
#pragma unroll
            for (int k = 0; k < 62; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) - __uint_as_float(v[k] & 0xffffe000u));
            tc::mbar_wait(&s_mma_bar, mma_phase);
            mma_phase ^= 1;
            tc::tc_fence_after();
            // pass 2: A = lo(x); D += A.Bhi
            tc::tmem_st64(tA, v);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            __syncthreads();
            if (threadIdx.x == 0) {
                tc::tc_fence_after();
#pragma unroll
                for (int s = 0; s < 8; ++s) tc::mma_tf32_ts(tmem + 64, tmem + 8 * s, dBh + 16 * s, idesc, true);
                tc::mma_commit(&s_mma_bar);
            }
            tc::mbar_wait(&s_mma_bar, mma_phase);
            mma_phase ^= 1;
            tc::tc_fence_after();
            tc::tmem_ld64(tD, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int q1 = 0; q1 < 31; ++q1) {
                const float re = __uint_as_float(v[2 * q1]), im = __uint_as_float(v[2 * q1 + 1]);
                acc[q1] = fmaf(im, im, fmaf(re, re, acc[q1]));
            }

            if (!kRegs && last_rd) {  // phase done: spill to the row, track the argmax
                const int rho = rho0 + ph;
                float* row = rows + rho * kChips;
#pragma unroll
                for (int q1 = 0; q1 < 31; ++q1) {
                    row[q1 * 33 + lane] = acc[q1];
                    const int lag = a.D * cell_q(q1, lane) + rho;
                    if (better(acc[q1], lag, best, bidx)) { best = acc[q1]; bidx = lag; }
                }
                if (lane >= 1 && lane <= 16) {
#pragma unroll
                    for (int sl = 0; sl < 2; ++sl) {
                        if (lane == 16 && sl == 1) break;
                        const int q1 = lane == 16 ? 0 : sl ? 31 - lane : lane;
                        row[q1 * 33 + 32] = accx[sl];
                        const int lag = a.D * cell_q(q1, 32) + rho;
                        if (better(accx[sl], lag, best, bidx)) { best = accx[sl]; bidx = lag; }
                    }
                }
            }
            if (last) { ++t; break; }
            if (last_rd) { rd = 0; ++ph; } else { ++rd; }
        }
        auto for_cells = [&](auto&& f) {
#pragma unroll
            for (int q1 = 0; q1 < 31; ++q1) f(acc[q1], a.D * cell_q(q1, lane) + rho0);
            if (lane >= 1 && lane <= 15) {
                f(accx[0], a.D * cell_q(lane, 32) + rho0);
                f(accx[1], a.D * cell_q(31 - lane, 32) + rho0);
            } else if (lane == 16) {
                f(accx[0], a.D * cell_q(0, 32) + rho0);
            }
        };
        if (kRegs) for_cells([&](float val, int lag) { if (better(val, lag, best, bidx)) { best = val; bidx = lag; } });
        // first argmax of the item (acquisition.py:151): ties -> lowest lag
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
            if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
        }
        if (lane == 0) { red_v[w] = best; red_i[w] = bidx; }
        if (threadIdx.x == 0) s_claim = claim;
        __syncthreads();
        const int64_t after = s_claim;
        if (next < a.n_items) load_cc(next);
        best = red_v[0];
        bidx = red_i[0];
        for (int i = 1; i < kTcWarps; ++i)
            if (better(red_v[i], red_i[i], best, bidx)) { best = red_v[i]; bidx = red_i[i]; }
        const int peak = bidx;
        // exclusion floor (acquisition.py:155-159)
        const int64_t pair = a.pair0 + lp;
        const int64_t s = pair / a.B;
        const int b = (int)(pair % a.B);
        float* pm = a.pmap ? a.pmap + ((int64_t)pi * a.B + b) * a.P : nullptr;
        float fl = -1.f;
        if (kRegs) {
            for_cells([&](float val, int lag) {
                if (!excluded(lag, peak, a.P, a.radius)) fl = fmaxf(fl, val);
                if (pm) pm[lag] = val;
            });
        } else {
            for (int i = threadIdx.x; i < a.D * kChips; i += blockDim.x) {
                const int rho = i / kChips, r = i - rho * kChips, q1 = r / 33, q2 = r - q1 * 33;
                const int lag = a.D * cell_q(q1, q2) + rho;
                const float val = rows[i];
                if (!excluded(lag, peak, a.P, a.radius)) fl = fmaxf(fl, val);
                if (pm) pm[lag] = val;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
        if (lane == 0) red_f[w] = fl;
        cp_async_wait_all();
        __syncthreads();
        if (threadIdx.x == 0) {
            float f = red_f[0];
            for (int i = 1; i < kTcWarps; ++i) f = fmaxf(f, red_f[i]);
            gacq_row out;
            out.bin = b;
            out.lag = peak;
            out.peak = best;
            out.floor = f < 0.f ? 0.f : f;
            a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
        }
        item = next;
        next = after;
        if (item >= a.n_items) break;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_dealloc<128>(tmem);
}

}  // namespace gacq
