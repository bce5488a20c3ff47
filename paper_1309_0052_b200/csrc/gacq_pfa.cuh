// gacq_pfa.cuh -- K1/K2 of the acquisition hot path on the 1023-point prime-factor transform.
//
// Reference path: gnssperf/acquisition.py:128-159 (hot loop 138-149).
//
// The chip-polyphase reduction is the one of gacq_kernels.cuh: lag tau = D q + rho of the
// reference's circular correlation over P = 1023 D samples equals the 1023-chip circular
// correlation of z_rho[m] = sum_{i<D} wbar[(D m + rho + i) mod P] with the chips. Here that
// correlation is evaluated with no zero padding:
//   g_rho = IDFT_1023( DFT_1023(z_rho) * Cc ),  Cc = conj(DFT_1023(chip)) / 1023,
// using the 31 x 33 Good-Thomas transform of pfa.cuh (no twiddles), one warp per transform:
//   K1 forward:  31-point stage over n1 (lane = n2, row 32 spread over the warp), exchange,
//                33-point stage over n2 (lane = k1 < 31), spectrum stored as Z[k2][32 lanes].
//   K2 inverse:  Z * Cc on load, 33-point stage over k2 (lane = k1 < 31), exchange in place,
//                31-point stage over k1 (lane = q2, row 32 spread), |.|^2 accumulated over rounds
//                in registers for the cells (q1, q2), q = (33 q1 + 31 q2) mod 1023.
// The spectrum of a transform is 33 x 32 complex64 = 8448 B; K2 streams each one into shared
// memory with a bulk async copy (cp.async.bulk + mbarrier), double-buffered per warp.
#pragma once
#include "gacq_kernels.cuh"
#include "pfa.cuh"
#include "rader31.cuh"

namespace gacq {

constexpr int kBuf = 33 * 32;                    // spectrum [k2][32]; column 31 is padding
constexpr int kScr = 34;                         // K1 coop31 scratch (33 used; keeps 16 B alignment)
constexpr unsigned kSpecBytes = kBuf * sizeof(cx);
constexpr int kCorrMaxWarps = 6;
constexpr int kCorrWarpCx = 2 * kBuf;            // per-warp shared memory (cx): two spectra
constexpr int kCcHalf = 17 * 32;                 // Hermitian half of a conj code spectrum (cx)
#ifndef GACQ_RADER31
#define GACQ_RADER31 1                           // K2's 31-point stage by Rader's algorithm (rader31.cuh)
#endif
#ifndef GACQ_PFA_MAXNREG
#define GACQ_PFA_MAXNREG 168                     // 3 CTAs x 4 warps per SM; no spills (streamed stages)
#endif

__host__ __device__ constexpr int corr_pfa_smem(int W) { return W * (kCorrWarpCx * 8 + 16) + kCcHalf * 8; }
// K1 with one phase per warp (W == D) computes every chip sum before any warp writes its
// exchange tile, so the exchange tiles alias the wiped-block table (one barrier in between)
__host__ __device__ constexpr bool fwd_pfa_alias(int D, int W) { return W == D; }
__host__ __device__ constexpr int fwd_pfa_smem(int D, int W) {
    return fwd_pfa_alias(D, W) ? 8 * (D * fwd_ws(D) > W * (kBuf + kScr) ? D * fwd_ws(D) : W * (kBuf + kScr))
                               : 8 * (D * fwd_ws(D) + W * (kBuf + kScr));
}

// ---- bulk async copy + mbarrier (SASS UBLKCP / SYNCS) ------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// `bytes` from global `src` into shared `dst`; completion is signalled on `bar`. Issued by one
// lane after the warp's generic accesses of `dst` (ordered by a __syncwarp before the call).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ float pow_acc(cx v, float acc) { return fmaf(im(v), im(v), fmaf(re(v), re(v), acc)); }

// ---- K1 ---------------------------------------------------------------------------------
#ifndef GACQ_FWD_MINB
// <= 128 registers (16 warps per SM) where shared memory allows several CTAs; the D >= 13
// variants (131 KB wiped-block table) run one CTA per SM and get the full register file
#define GACQ_FWD_MINB(D, W) ((D) >= 13 ? 1 : 16 / (W) > 0 ? 16 / (W) : 1)
#endif
struct FwdPfaArgs {
    const float2* snaps;   // batch base (device), snapshot s at snaps + s*stride
    int64_t stride;        // complex samples between snapshots
    const float2* carrier; // [B][n_coh] wipe-off replicas
    cx* Z;                 // [pairs][R][D][kBuf] spectra
    int* bad;              // atomicMin'd to the index of a snapshot holding a non-finite sample
    int64_t pair0;         // first (snapshot, bin) pair of this chunk, pair = s*B + b
    int B, R, n_coh, P, K;
};

// grid: pairs_in_chunk * R CTAs (one per (pair, round)) of 32 W threads. Warp w transforms
// phases rho in [w PWF, (w+1) PWF), PWF = ceil(D/W), sliding the chip sums by one sample per
// phase. dynamic smem: fwd_pfa_smem(D, W).
template <int D, int W>
__global__ void __launch_bounds__(32 * W, GACQ_FWD_MINB(D, W)) gacq_fwd_pfa_kernel(FwdPfaArgs a) {
    constexpr int WS = fwd_ws(D);
    constexpr int PWF = (D + W - 1) / W;
    extern __shared__ __align__(16) cx smem[];
    cx* wt = smem;
    const int lp = blockIdx.x / a.R, rd = blockIdx.x % a.R;
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    const cx* xs = reinterpret_cast<const cx*>(a.snaps) + s * a.stride + (int64_t)rd * a.n_coh;
    const cx* cs = reinterpret_cast<const cx*>(a.carrier) + (int64_t)b * a.n_coh;
    // D = 4, K = 1 (C1-C3): chip sums computed in the wipe (wipe_chips4), wt then holds z[rho][m]
    if (wipe_fold<D, 32 * W>(xs, cs, a.P, a.K, wt) && threadIdx.x == 0) atomicMin(a.bad, (int)s);
    // One phase per warp (W = D >= 4: C1-C3 at D = 4, the 8.184 MHz default at D = 8): the chip
    // sums once per chip, in place. Thread t takes chips m = 32 W j + t, reads wt[k][m] and
    // wt[k][m + 1] (row 1023 repeats chip 0), and after a barrier overwrites wt[rho][m] =
    // z_rho[m], summed in chip_sum's order (identical values); each warp then reads its z row
    // instead of summing D entries per element.
    constexpr bool zsum = W == D && D >= 4;
    if constexpr (zsum) {
        constexpr int kIt = (kChips + 32 * W - 1) / (32 * W);
        cx z[kIt][D];
#pragma unroll
        for (int j = 0; j < kIt; ++j) {
            const int m = j * 32 * W + threadIdx.x;
            if (m < kChips) {
                cx v[2 * D - 1];
#pragma unroll
                for (int k = 0; k < 2 * D - 1; ++k) v[k] = k < D ? wt[k * WS + m] : wt[(k - D) * WS + m + 1];
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    cx acc = czero();
#pragma unroll
                    for (int i = 0; i < D; ++i) acc = add2(acc, v[r + i]);
                    z[j][r] = acc;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kIt; ++j) {
            const int m = j * 32 * W + threadIdx.x;
            if (m < kChips) {
#pragma unroll
                for (int r = 0; r < D; ++r) wt[r * WS + m] = z[j][r];
            }
        }
        __syncthreads();
    }
    // Several phases per warp (W < D: D = 13, 14, 16): all D chip sums per chip, in place,
    // z_0 in full and z_rho by the one-sample slide the warps used for their later phases.
    // Chips go in two batches of contiguous ranges, [0, 32 W kB) then the rest: a batch reads
    // columns m and m + 1 of its own range (the first batch's last chip reads the second's first
    // column, before the second writes), and column 1023 (the copy of chip 0) is never written.
    constexpr bool zslide = W < D;
    if constexpr (zslide) {
        constexpr int kIt = (kChips + 32 * W - 1) / (32 * W);
        constexpr int kB = (kIt + 1) / 2;
#pragma unroll 1
        for (int j0 = 0; j0 < kIt; j0 += kB) {
            cx z[kB][D];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int m = (j0 + u) * 32 * W + threadIdx.x;
                if (j0 + u < kIt && m < kChips) {
                    cx acc = czero();
#pragma unroll
                    for (int i = 0; i < D; ++i) acc = add2(acc, wt[i * WS + m]);
                    z[u][0] = acc;
#pragma unroll
                    for (int r = 1; r < D; ++r) {
                        acc = add2(sub2(acc, wt[(r - 1) * WS + m]), wt[(r - 1) * WS + m + 1]);
                        z[u][r] = acc;
                    }
                }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int m = (j0 + u) * 32 * W + threadIdx.x;
                if (j0 + u < kIt && m < kChips) {
#pragma unroll
                    for (int r = 0; r < D; ++r) wt[r * WS + m] = z[u][r];
                }
            }
            __syncthreads();
        }
    }

    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool kAlias = fwd_pfa_alias(D, W);
    cx* T = smem + (kAlias ? 0 : D * WS) + w * (kBuf + kScr);  // exchange [k1][33]
    cx* scr = T + kBuf;
    // lane n2 holds z at m = (33 n1 + 31 n2) mod 1023, n1 < 31; lane L < 31 also holds row
    // n2 = 32 at m = (33 L + 992) mod 1023
    const int mb = 31 * lane, me = (33 * lane + 992) % kChips;
    auto chip_sum = [&](int rho, int m) {
        cx acc = czero();
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int k = rho + i;
            acc = add2(acc, k < D ? wt[k * WS + m] : wt[(k - D) * WS + m + 1]);
        }
        return acc;
    };
    cx zr[31], ze;
    const int rho0 = w * PWF;
#pragma unroll 1
    for (int ph = 0; ph < PWF; ++ph) {
        const int rho = rho0 + ph;
        if (rho >= D) break;
        if (zsum || zslide) {  // the chip sums are in wt
#pragma unroll
            for (int n1 = 0; n1 < 31; ++n1) {
                int m = mb + 33 * n1;
                m -= m >= kChips ? kChips : 0;
                zr[n1] = wt[rho * WS + m];
            }
            ze = lane < 31 ? wt[rho * WS + me] : czero();
            if (kAlias && ph == 0) __syncthreads();  // every warp's chip sums are read before T overwrites wt
        } else if (ph == 0) {
#pragma unroll
            for (int n1 = 0; n1 < 31; ++n1) {
                int m = mb + 33 * n1;
                m -= m >= kChips ? kChips : 0;
                zr[n1] = chip_sum(rho, m);
            }
            ze = lane < 31 ? chip_sum(rho, me) : czero();
            if (kAlias) __syncthreads();  // every warp's chip sums are read before T overwrites wt
        } else {  // window [rho-1, rho-1+D) -> [rho, rho+D): drop wbar[D m + rho-1], add wbar[D (m+1) + rho-1]
            const cx* r = wt + (rho - 1) * WS;
#pragma unroll
            for (int n1 = 0; n1 < 31; ++n1) {
                int m = mb + 33 * n1;
                m -= m >= kChips ? kChips : 0;
                zr[n1] = add2(sub2(zr[n1], r[m]), r[m + 1]);
            }
            if (lane < 31) ze = add2(sub2(ze, r[me]), r[me + 1]);
        }
        // 31-point stage over n1 -> T[k1][n2]
        {
            cx x[31];
#pragma unroll
            for (int n1 = 0; n1 < 31; ++n1) x[n1] = zr[n1];
            dft_odd<-1, 31, 5>(x, [&](int k1, cx v) { T[k1 * 33 + lane] = v; });  // (Rader measured slower here)
            coop31<-1>(ze, lane, [&](int j) { return __ldg(&kCoop31Coef[j - 1][lane]); }, scr,
                       [&](int, int k1, cx v) { T[k1 * 33 + 32] = v; });
        }
        __syncwarp();
        // 33-point stage over n2 -> Z[k2][k1], coalesced 256 B stores
        if (lane < 31) {
            cx y[33];
#pragma unroll
            for (int n2 = 0; n2 < 33; ++n2) y[n2] = T[lane * 33 + n2];
            cx* dst = a.Z + (((int64_t)lp * a.R + rd) * D + rho) * kBuf + lane;
            dft33<-1>(y, [&](int k2, cx v) { dst[k2 * 32] = v; });
        }
        __syncwarp();
    }
}

// ---- K2 ---------------------------------------------------------------------------------
struct CorrPfaArgs {
    const cx* Z;           // spectra of this chunk, [pairs][R][D][kBuf]
    const cx* Cc;          // [n_prn][kCcHalf] conj code spectra / 1023, rows k2 <= 16 of [k2][32]
    gacq_row* rows_bin;    // [n_snap][n_prn][B]
    float* pmap;           // optional [n_prn][B][P] power map (single snapshot), else null
    float* row_scratch;    // [gridDim][D][1023] native-order power rows when PW > 1
    int64_t pair0;
    int64_t n_items;       // pairs_in_chunk * n_prn, item = lp * n_prn + pi
    unsigned long long* counter;  // zeroed before the launch
    int B, R, D, P, n_prn, radius, PW;
    int zero;              // 0 (an opaque runtime zero, see dft31_stream)
    unsigned dmagic;       // ceil(2^32 / D): x / D == umulhi(x, dmagic) for x < 2^32 / D
};

// chip lag of cell (q1, q2)
__device__ __forceinline__ int cell_q(int q1, int q2) {
    const int q = 33 * q1 + 31 * q2;
    return q >= 2 * kChips ? q - 2 * kChips : q >= kChips ? q - kChips : q;
}
__device__ __forceinline__ bool better(float v, int l, float bv, int bl) { return v > bv || (v == bv && l < bl); }
// (power >= 0, lag >= 0) as one unsigned key ordered like better(): the bits of a non-negative
// float order like its value, and the low word inverts the lag so ties go to the lowest lag
__device__ __forceinline__ unsigned long long peak_key(float v, int lag) {
    return ((unsigned long long)__float_as_uint(v) << 32) | (0xffffffffu - (unsigned)lag);
}
__device__ __forceinline__ bool excluded(int lag, int peak, int P, int radius) {
    int d = abs(lag - peak);
    d = min(d, P - d);
    return d <= radius;
}

// Persistent: gridDim.x = resident CTA slots of 32 W threads; CTA c starts with item c and
// claims the following items in order from a global counter (two items ahead, so the atomic
// never stalls), so the CTAs sharing a pair's spectra run together and hit them in L2.
// Warp w owns phases [w PW, w PW + PW) of the item. The item's conjugate code spectrum sits in
// shared memory as the Hermitian half [17][32] (rows k2 > 16 are conj of row 33 - k2, lane
// (31 - k1) mod 31), refilled with cp.async between items.
// kRegs (PW == 1): the powers stay in registers through the argmax and the floor.
// dynamic smem: corr_pfa_smem(W).
template <bool kRegs>
__global__ void __maxnreg__(GACQ_PFA_MAXNREG) gacq_corr_pfa_kernel(CorrPfaArgs a) {
    __shared__ unsigned long long red_k[kCorrMaxWarps];  // per-warp (peak, lag) keys, see peak_key
    __shared__ float red_f[kCorrMaxWarps];
    __shared__ long long s_claim, s_claim0;  // s_claim0: the first claim (read before the item loop)
    __shared__ float s_coef[15][32];  // coop31 columns, read conflict-free as s_coef[j-1][lane]
    extern __shared__ __align__(16) cx smem[];
    const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 15 * 32; i += blockDim.x) s_coef[i >> 5][i & 31] = coop31_coef(i & 31, (i >> 5) + 1);
    cx* buf = smem + w * kCorrWarpCx;  // buf[0..kBuf), buf[kBuf..2kBuf)
    cx* ccs = smem + W * kCorrWarpCx;  // [17][32] conj code spectrum half of the current item
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(ccs + kCcHalf) + 2 * w;
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    // item indices fit 32 bits (launch_corr_pfa checks): unsigned 32-bit divisions per item
    const int n_items = (int)a.n_items;
    const unsigned n_prn = (unsigned)a.n_prn;
    int item = blockIdx.x;
    if (item >= n_items) return;
    auto load_cc = [&](int it) {  // cp.async of the half spectrum of item `it`'s PRN
        const char* g = reinterpret_cast<const char*>(a.Cc + ((unsigned)it % n_prn) * kCcHalf);
        for (int i = threadIdx.x; i < kCcHalf / 2; i += blockDim.x) cp_async16(ccs + 2 * i, g + 16 * i);
        cp_async_commit();
    };
    if (threadIdx.x == 0) s_claim0 = (long long)gridDim.x + (long long)atomicAdd(a.counter, 1ull);
    load_cc(item);

    const int rho0 = w * a.PW;
    const int nph = min(a.PW, a.D - rho0);  // phases of this warp
    const int64_t pair_span = (int64_t)a.R * a.D * kBuf;
    auto zbase = [&](int it) { return a.Z + (int64_t)((unsigned)it / n_prn) * pair_span + rho0 * kBuf; };
    unsigned t = 0;  // this warp's transform count: buffer t & 1, mbarrier parity (t >> 1) & 1
    __syncwarp();
    if (lane == 0) bulk_load(buf, zbase(item), kSpecBytes, &mbar[0]);
    float* rows = a.row_scratch + (int64_t)blockIdx.x * a.D * kChips;
    const int pl = lane == 0 ? 0 : 31 - lane;  // Hermitian partner column of k1 = lane
    cp_async_wait_all();
    __syncthreads();
    int next = (int)s_claim0;  // s_claim itself is rewritten by thread 0 at the end of the first item

    for (;;) {
        long long claim = 0;
        if (threadIdx.x == 0 && next < n_items) claim = (long long)gridDim.x + (long long)atomicAdd(a.counter, 1ull);
        const unsigned lp = (unsigned)item / n_prn;
        const int pi = (int)((unsigned)item - lp * n_prn);
        const cx* zb = a.Z + (int64_t)lp * pair_span + rho0 * kBuf;
        const cx* zn = next < n_items ? zbase(next) : nullptr;

        float best = -1.f;
        int bidx = 0x7fffffff;
        float acc[31], accx[2];
        int rd = 0, ph = 0;  // round and phase of the current transform
#pragma unroll 1
        for (;; ++t) {
            if (rd == 0) {
#pragma unroll
                for (int i = 0; i < 31; ++i) acc[i] = 0.f;
                accx[0] = accx[1] = 0.f;
            }
            const bool last_rd = rd + 1 == a.R;
            const bool last = last_rd && ph + 1 == nph;
            if (lane == 0) {  // prefetch the warp's next spectrum into the other buffer
                const cx* nsrc = !last ? zb + ((last_rd ? 0 : rd + 1) * a.D + (last_rd ? ph + 1 : ph)) * kBuf : zn;
                if (nsrc) bulk_load(buf + ((t + 1) & 1) * kBuf, nsrc, kSpecBytes, &mbar[(t + 1) & 1]);
            }
            mbar_wait(&mbar[t & 1], (t >> 1) & 1);
            cx* E = buf + (t & 1) * kBuf;
            // Z * Cc and the 33-point stage over k2; results E[q2][k1] written in place
            // (the 33-point stage reads all of E before the __syncwarp and writes after it)
            if (lane < 31) {
                const cx* Ec = E + lane;
                dft33_stream<1>(
                    [&](int k2, int dep) {
                        // k2 is a compile-time constant here: the branch folds away
                        return k2 <= 16 ? cmul(Ec[k2 * 32 + dep], ccs[k2 * 32 + lane + dep])
                                        : cmul_conj(Ec[k2 * 32 + dep], ccs[(33 - k2) * 32 + pl + dep]);
                    },
                    a.zero, [&](int q2, cx v) {
                        if (q2 == 0) __syncwarp(0x7fffffffu);
                        E[q2 * 31 + lane] = v;
                    });
            }
            __syncwarp();
            // 31-point stage over k1 for row q2 = lane (+ row 32 spread over the warp, with its
            // scratch in the buffer's unused tail E[1023..1055])
            const cx e = lane < 31 ? E[32 * 31 + lane] : czero();
            const cx* Er = E + lane * 31;
#if GACQ_RADER31
            dft31_rader_inv([&](int k1) { return Er[k1]; }, [&](int q1, cx v) { acc[q1] = pow_acc(v, acc[q1]); });
#else
            dft31_stream<1>([&](int k1, int dep) { return Er[k1 + dep]; }, a.zero,
                            [&](int q1, cx v) { acc[q1] = pow_acc(v, acc[q1]); });
#endif
            coop31<1>(e, lane, [&](int j) { return s_coef[j - 1][lane]; }, E + kChips,
                      [&](int sl, int, cx v) { accx[sl] = pow_acc(v, accx[sl]); });
            __syncwarp();  // E is free for the prefetch issued at the next transform

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
        // cells of this lane (kRegs): (q1, lane) for q1 < 31, and coop cells
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
        // first argmax of the item (acquisition.py:151): ties -> lowest lag
        const bool x0 = lane >= 1 && lane <= 16, x1 = lane >= 1 && lane <= 15;  // lanes owning coop cells
        float lane_max = 0.f;
        if (kRegs) {
            // warp max of the values, then the lowest lag holding it (searched only by the lanes
            // whose own max equals it). Lanes without coop cells keep accx = 0, which is <= every
            // power and never a lag candidate.
            float m = acc[0];
#pragma unroll
            for (int q1 = 1; q1 < 31; ++q1) m = fmaxf(m, acc[q1]);
            m = fmaxf(m, fmaxf(accx[0], accx[1]));
            lane_max = m;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            int bl = 0x7fffffff;
            if (lane_max == m) {  // cells equal to the max as a mask; lags only for its set bits
                unsigned mk = 0u;
#pragma unroll
                for (int q1 = 0; q1 < 31; ++q1) mk |= (acc[q1] == m ? 1u : 0u) << q1;
                while (mk) {
                    const int q1 = __ffs(mk) - 1;
                    mk &= mk - 1u;
                    bl = min(bl, a.D * cell_q(q1, lane) + rho0);
                }
                if (x0 && accx[0] == m) bl = min(bl, a.D * cell_q(lane == 16 ? 0 : lane, 32) + rho0);
                if (x1 && accx[1] == m) bl = min(bl, a.D * cell_q(31 - lane, 32) + rho0);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) bl = min(bl, __shfl_xor_sync(0xffffffffu, bl, off));
            best = m;
            bidx = bl == 0x7fffffff ? rho0 : bl;  // all-NaN powers (non-finite input, flagged by K1)
        } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
            }
            if (bidx == 0x7fffffff) { best = 0.f; bidx = rho0; }  // all-NaN powers (flagged by K1)
        }
        if (lane == 0) red_k[w] = peak_key(best, bidx);
        if (threadIdx.x == 0) s_claim = claim;
        __syncthreads();  // every warp is done with this item's spectra, Cc and row spills
        const int after = (int)s_claim;
        if (next < n_items) load_cc(next);  // lands while the floor is computed
        unsigned long long kb = red_k[0];
        for (int i = 1; i < W; ++i) kb = max(kb, red_k[i]);
        best = __uint_as_float((unsigned)(kb >> 32));
        const int peak = (int)(0xffffffffu - (unsigned)kb);
        // exclusion floor (acquisition.py:155-159)
        float* pm = a.pmap ? a.pmap + ((int64_t)pi * a.B + (a.pair0 + lp) % a.B) * a.P : nullptr;
        float fl = -1.f;
        if (kRegs && !pm) {
            // Only the cells within `radius` of the peak are excluded: lags D q + rho0 for q in
            // [ceil((peak - r - rho0)/D), floor((peak + r - rho0)/D)] (mod 1023), at most 2r/D + 1
            // of them. Cell q lives at (q1, q2) = (16 q mod 31, 16 q mod 33) (inverse of cell_q).
            // A lane with none of them takes its plain max.
            if (2 * a.radius + 1 < a.P) {
                // offset by D * 1023 (> radius + rho0) so both bounds divide as unsigned
                const unsigned off = (unsigned)(a.D * kChips), D = (unsigned)a.D;
                const unsigned lo = (unsigned)(peak - a.radius - rho0) + off, hi = (unsigned)(peak + a.radius - rho0) + off;
                const int qa = (int)__umulhi(lo + D - 1u, a.dmagic) - kChips, qb = (int)__umulhi(hi, a.dmagic) - kChips;
                unsigned m31 = 0u, mx = 0u;
                for (int q = qa; q <= qb; ++q) {
                    const int qq = q < 0 ? q + kChips : q >= kChips ? q - kChips : q;
                    const int q1 = (16 * qq) % 31, q2 = (16 * qq) % 33;
                    if (q2 == lane) m31 |= 1u << q1;
                    if (q2 == 32) {
                        if (lane == 16 && q1 == 0) mx |= 1u;
                        if (x1 && q1 == lane) mx |= 1u;
                        if (x1 && q1 == 31 - lane) mx |= 2u;
                    }
                }
                if ((m31 | mx) == 0u) {
                    fl = lane_max;  // the fake 0 of lanes without coop cells never raises the floor
                } else {
#pragma unroll
                    for (int q1 = 0; q1 < 31; ++q1)
                        if (!((m31 >> q1) & 1u)) fl = fmaxf(fl, acc[q1]);
                    if (x0 && !(mx & 1u)) fl = fmaxf(fl, accx[0]);
                    if (x1 && !(mx & 2u)) fl = fmaxf(fl, accx[1]);
                }
            }
        } else if (kRegs) {
            for_cells([&](float v, int lag) {
                if (!excluded(lag, peak, a.P, a.radius)) fl = fmaxf(fl, v);
                if (pm) pm[lag] = v;
            });
        } else {
            for (int i = threadIdx.x; i < a.D * kChips; i += blockDim.x) {
                const int rho = i / kChips, r = i - rho * kChips, q1 = r / 33, q2 = r - q1 * 33;
                const int lag = a.D * cell_q(q1, q2) + rho;
                const float v = rows[i];
                if (!excluded(lag, peak, a.P, a.radius)) fl = fmaxf(fl, v);
                if (pm) pm[lag] = v;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
        if (lane == 0) red_f[w] = fl;
        cp_async_wait_all();
        __syncthreads();  // publishes red_f and the next item's Cc
        if (threadIdx.x == 0) {
            float f = red_f[0];
            for (int i = 1; i < W; ++i) f = fmaxf(f, red_f[i]);
            const int64_t pair = a.pair0 + lp;
            const int64_t s = pair / a.B;
            const int b = (int)(pair - s * a.B);
            gacq_row out;
            out.bin = b;
            out.lag = peak;
            out.peak = best;
            out.floor = f < 0.f ? 0.f : f;
            a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
        }
        item = next;
        next = after;
        if (item >= n_items) break;
    }
}

}  // namespace gacq
