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

constexpr int kBuf = 33 * 32;                    // K1 exchange tile [k1][33] (+ padding)
constexpr int kScr = 34;                         // K1 coop31 scratch (33 used; keeps 16 B alignment)
constexpr int kSpec = 1024;                      // one spectrum in HBM and in K2's buffer: [k2][31] + 1 pad
constexpr unsigned kSpecBytes = kSpec * sizeof(cx);
constexpr int kXch = 1023 + 33;                  // K2 exchange [q2][31] + coop31 scratch
// Hermitian half [k2 <= 16][kCcRow] of a conj code spectrum: columns k1 < 31, and column 31 a copy
// of column 0. Lane k1 reads the conjugate partner column 31 - k1 of rows k2 > 16 (k1 = 0 is its
// own partner: column 31), so a half-warp's 16 reads are 16 consecutive slots: one bank wavefront
// (with column 0 itself, lanes 0 and 1..15 hit banks 0-1 twice: 3 wavefronts instead of 2)
constexpr int kCcRow = 32;
constexpr int kCcHalf = 17 * kCcRow;
constexpr int kCorrWarps = 4;                    // K2 warps per CTA (one item each)
constexpr int kPhaseRow = 33 * 32;               // K2 scratch row of one phase: [q1 or coop slot][lane] floats
constexpr int kTop2Row = 5 * 32;                 // K2 (kTop2) phase summary: [max, 2nd max, max index, coop 0, coop 1][lane]
#ifndef GACQ_R1_IPW
#define GACQ_R1_IPW 2
#endif
constexpr int kR1PairsPerWarp = GACQ_R1_IPW;     // K2 at R = 1: pairs per warp per unit (kIPW)
#ifndef GACQ_PFA_MAXNREG
#define GACQ_PFA_MAXNREG 168                     // 3 CTAs x 4 warps per SM; no spills (streamed stages)
#endif

// K2 dynamic smem: per warp a spectrum buffer and an exchange buffer, two code-spectrum slots
// per CTA, one mbarrier per warp (3 CTAs per SM fit the 228 KB)
__host__ __device__ constexpr int corr_pfa_smem() { return kCorrWarps * (kSpec + kXch) * 8 + 2 * kCcHalf * 8 + kCorrWarps * 8; }
// K1 with one phase per warp (W == D) computes every chip sum before any warp writes its
// exchange tile, so the exchange tiles alias the wiped-block table (one barrier in between)
__host__ __device__ constexpr bool fwd_pfa_alias(int D, int W) { return W == D; }
__host__ __device__ constexpr int fwd_pfa_main(int D, int W) {
    return fwd_pfa_alias(D, W) ? 8 * (D * fwd_ws(D) > W * (kBuf + kScr) ? D * fwd_ws(D) : W * (kBuf + kScr))
                               : 8 * (D * fwd_ws(D) + W * (kBuf + kScr));
}
// + the int8 dequantization table (256 floats) behind the main region
__host__ __device__ constexpr int fwd_pfa_smem(int D, int W) { return fwd_pfa_main(D, W) + 256 * 4; }

// ---- bulk async copy + mbarrier (SASS UBLKCP / SYNCS) ------------------------------------

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
// the same copy into a buffer that only the async proxy ever writes and the generic proxy only
// reads (reads already consumed, ordered by a __syncwarp): no proxy fence needed
__device__ __forceinline__ void bulk_load_nofence(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
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



__device__ __forceinline__ float pow_acc(cx v, float acc) { return fmaf(im(v), im(v), fmaf(re(v), re(v), acc)); }

// ---- K1 ---------------------------------------------------------------------------------
#ifndef GACQ_FWD_MINB
// <= 128 registers (16 warps per SM) where shared memory allows several CTAs; the D >= 13
// variants (131 KB wiped-block table) run one CTA per SM and get the full register file
#define GACQ_FWD_MINB(D, W) ((D) >= 13 ? 1 : 16 / (W) > 0 ? 16 / (W) : 1)
#endif
struct FwdPfaArgs {
    const void* snaps;     // batch base (device), snapshot s at sample s*stride
    int64_t stride;        // samples between snapshots
    int fmt;               // kSrcC64 (complex64) or GACQ_FMT_INT8 / GACQ_FMT_INT16 interleaved I/Q
    double qs;             // integer formats: scale / limit (iffile.py:95-98)
    const float2* carrier; // [B][n_coh] wipe-off replicas
    cx* Z;                 // [pairs][R][D][kSpec] spectra
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
    const int64_t x0 = s * a.stride + (int64_t)rd * a.n_coh;  // first sample of the block
    const cx* cs = reinterpret_cast<const cx*>(a.carrier) + (int64_t)b * a.n_coh;
    // integer I/Q is dequantized in the wipe's registers (no complex64 staging copy)
    bool bad;
    if (a.fmt == GACQ_FMT_INT8) {
        float* lut = reinterpret_cast<float*>(reinterpret_cast<char*>(smem) + fwd_pfa_main(D, W));
        for (int i = threadIdx.x; i < 256; i += 32 * W) lut[i] = deq(i - 128, a.qs);
        __syncthreads();
        bad = wipe_fold<D, 32 * W>(SrcI8{static_cast<const signed char*>(a.snaps), lut}.at(x0), cs, a.P, a.K, wt);
    }
    else if (a.fmt == GACQ_FMT_INT16)
        bad = wipe_fold<D, 32 * W>(SrcI16{static_cast<const short*>(a.snaps), a.qs}.at(x0), cs, a.P, a.K, wt);
    else
        bad = wipe_fold<D, 32 * W>(SrcC64{static_cast<const cx*>(a.snaps)}.at(x0), cs, a.P, a.K, wt);
    if (bad && threadIdx.x == 0) atomicMin(a.bad, (int)s);
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
        // 33-point stage over n2 -> Z[k2][k1] (rows of 31, the spectrum dense in 8184 B)
        if (lane < 31) {
            cx y[33];
#pragma unroll
            for (int n2 = 0; n2 < 33; ++n2) y[n2] = T[lane * 33 + n2];
            cx* dst = a.Z + (((int64_t)lp * a.R + rd) * D + rho) * kSpec + lane;
            dft33<-1>(y, [&](int k2, cx v) { dst[k2 * 31] = v; });
        }
        __syncwarp();
    }
}

// ---- K2 ---------------------------------------------------------------------------------
struct CorrPfaArgs {
    const cx* Z;           // spectra of this chunk, [pairs][R][D][kSpec]
    const cx* Cc;          // [n_prn][kCcHalf] conj code spectra / 1023, rows k2 <= 16 of [k2][kCcRow]
    gacq_row* rows_bin;    // [n_snap][n_prn][B]
    float* pmap;           // optional [n_prn][B][P] power map (single snapshot), else null
    float* rows;           // [gridDim][kCorrWarps][D][kPhaseRow] per-phase power rows of the warp's item
    int64_t pair0;
    int n_pairs;           // pairs in this chunk
    int n_units;           // ceil(n_pairs / kCorrWarps) * n_prn; unit = group * n_prn + prn index
    unsigned long long* counter;  // zeroed before the launch
    int B, R, D, P, n_prn, radius;
    int zero;              // 0 (an opaque runtime zero, see dft31_stream)
    unsigned dmagic;       // ceil(2^32 / D) for D > 1: x / D == umulhi(x, dmagic) for x < 2^32 / D
                           // (D = 1 has no 32-bit magic: divD returns x itself)
};

// chip lag of cell (q1, q2)
__device__ __forceinline__ int cell_q(int q1, int q2) {
    const int q = 33 * q1 + 31 * q2;
    return q >= 2 * kChips ? q - 2 * kChips : q >= kChips ? q - kChips : q;
}
__device__ __forceinline__ bool better(float v, int l, float bv, int bl) { return v > bv || (v == bv && l < bl); }
__device__ __forceinline__ bool excluded(int lag, int peak, int P, int radius) {
    int d = abs(lag - peak);
    d = min(d, P - d);
    return d <= radius;
}

// Persistent, one item per warp: a CTA of kCorrWarps warps takes a unit = (group of kCorrWarps
// consecutive (snapshot, bin) pairs, PRN) and warp w searches pair w of the group for that PRN
// over all D phases and R rounds; the CTA's warps share the PRN's conjugate code spectrum in
// shared memory (two slots: the next unit's lands with cp.async while this one runs). Units are
// claimed in order from a global counter one ahead, so the n_prn CTAs sharing a group's spectra
// run together and read them from L2.
//
// Per transform (phase rho, round r) of a warp: the spectrum Z (8184 B) sits in the warp's buffer
// (cp.async.bulk + mbarrier); every lane k1 < 31 loads its column and the code spectrum at once,
// Y = Z * Cc, the 3-point layer of the 33-point stage -- after which the buffer is free and lane 0
// issues the bulk copy of the warp's next spectrum into it (no generic-proxy write ever touches
// that buffer, so it needs no proxy fence) -- then the 11-point layers write the exchange buffer
// E[q2][31], the 31-point stage over k1 (lane = q2, Rader) and the spread row q2 = 32 (coop31),
// and |g|^2 accumulated in registers over the rounds.
// After the R rounds of a phase its powers go to the warp's scratch row in global memory (L2)
// and its first argmax (value desc, lag asc) into a running per-lane best. After the last phase
// the warp reduces the peak and takes the exclusion floor from the scratch rows: only cells within
// `radius` of the peak are excluded, and every lane owns at most one q per window (its q values
// are congruent mod 33), found directly by the inverse map (q1, q2) = (16 q mod 31, 16 q mod 33).
// acquisition.py:151-159.
// kTop2 (every window of the exclusion radius holds at most 33 consecutive chip lags, 2 r < 33 D:
// the default one-chip radius and any r < 16.5 chips): each lane owns at most one excluded cell of
// its 31 per phase (its q values are congruent mod 33) and at most one of the spread row's, so a
// phase keeps only the lane's (max, its first index, second max) and the two spread-row cells: 5
// words per lane instead of the 33-float row, and the floor reads them back with no window loop.
// kR1 (one noncoherent round, C1): the phase summary is tracked inside the round's |g|^2 emit
// (ALU work interleaved with the Rader stage's FMAs) instead of a pass over the 31 powers after it.
template <bool kTop2, bool kR1>
__global__ void __maxnreg__(GACQ_PFA_MAXNREG) gacq_corr_pfa_kernel(CorrPfaArgs a) {
    __shared__ int s_unit[2];
    extern __shared__ __align__(16) cx smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cx* zbuf = smem + w * (kSpec + kXch);   // the warp's spectrum buffer (async proxy only)
    cx* E = zbuf + kSpec;                   // exchange [q2][31] + coop31 scratch at E[1023..1055]
    cx* ccs0 = smem + kCorrWarps * (kSpec + kXch);
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(ccs0 + 2 * kCcHalf) + w;
    if (lane == 0) {
        mbar_init(mbar, 1);
        fence_mbar_init();
    }
    const unsigned n_prn = (unsigned)a.n_prn;
    const int D = a.D, R = a.R;
    auto divD = [&](unsigned x) { return D == 1 ? x : __umulhi(x, a.dmagic); };  // x / D
    int unit = blockIdx.x;
    if (unit >= a.n_units) return;
    const int64_t pair_span = (int64_t)R * D * kSpec;
    auto load_cc = [&](int u, int slot) {  // cp.async of the half spectrum of unit u's PRN
        const char* g = reinterpret_cast<const char*>(a.Cc + ((unsigned)u % n_prn) * kCcHalf);
        cx* dst = ccs0 + slot * kCcHalf;
        for (int i = threadIdx.x; i < kCcHalf / 2; i += blockDim.x) cp_async16(dst + 2 * i, g + 16 * i);
        cp_async_commit();
    };
    // R = 1: a unit spans kIPW pairs per warp (one unit barrier and code-spectrum swap per two
    // items: at one transform per phase the per-unit work is a large share of the item)
    constexpr int kIPW = kR1 ? kR1PairsPerWarp : 1;
    auto pair_of = [&](int u, int it) {  // this warp's it-th pair of unit u
        return (int)((unsigned)u / n_prn) * (kCorrWarps * kIPW) + it * kCorrWarps + w;
    };
    if (threadIdx.x == 0) s_unit[1] = (int)(gridDim.x + atomicAdd(a.counter, 1ull));
    load_cc(unit, 0);
    {
        const int lp = pair_of(unit, 0);
        __syncwarp();
        if (lane == 0 && lp < a.n_pairs) bulk_load(zbuf, a.Z + lp * pair_span, kSpecBytes, mbar);
    }
    cp_async_wait_all();
    __syncthreads();
    float* rows = a.rows + ((int64_t)blockIdx.x * kCorrWarps + w) * D * kPhaseRow;
    const int pl = 31 - lane;  // Hermitian partner column of k1 = lane (31: the copy of column 0)
    const bool x0 = lane >= 1 && lane <= 16, x1 = lane >= 1 && lane <= 15;  // lanes owning coop cells
    unsigned t = 0;  // transforms of this warp: mbarrier parity t & 1

    for (int k = 0;; ++k) {
        const int nxt = s_unit[(k + 1) & 1];
        if (nxt < a.n_units) load_cc(nxt, (k + 1) & 1);  // its slot was last read in unit k - 1
        if (threadIdx.x == 0) s_unit[k & 1] = nxt < a.n_units ? (int)(gridDim.x + atomicAdd(a.counter, 1ull)) : a.n_units;
        const cx* ccs = ccs0 + (k & 1) * kCcHalf;
        const int pi = (int)((unsigned)unit % n_prn);
#pragma unroll 1
        for (int it = 0; it < kIPW; ++it) {
        const int lp = pair_of(unit, it);
        // the warp's next item: its next pair in this unit, else its first pair of the next unit
        const int lpn = it + 1 < kIPW ? pair_of(unit, it + 1) : nxt < a.n_units ? pair_of(nxt, 0) : a.n_pairs;
        const cx* znext = lpn < a.n_pairs ? a.Z + lpn * pair_span : nullptr;
        if (lp < a.n_pairs) {
            const cx* zb = a.Z + lp * pair_span;
            const int64_t pair = a.pair0 + lp;
            const int b = (int)(pair % a.B);
            float* pm = a.pmap ? a.pmap + ((int64_t)pi * a.B + b) * a.P : nullptr;
            float best = -1.f;
            int bidx = 0x7fffffff;
            const int64_t rstep = (int64_t)D * kSpec;  // next round, same phase
#pragma unroll 1
            for (int rho = 0; rho < D; ++rho) {
                const cx* cur = zb + rho * kSpec;
                float acc[31], accx[2];
#pragma unroll
                for (int i = 0; i < 31; ++i) acc[i] = 0.f;
                accx[0] = accx[1] = 0.f;
                float v1 = -1.f, v2 = -1.f;  // kTop2: the lane's first max, second max (ties twice), index
                int i1 = 0;
#pragma unroll 1
                for (int rd = 0; rd < R; ++rd, ++t) {
                    // the warp's next spectrum: next round, else the next phase's first round, else
                    // the first spectrum of its next item
                    const cx* nsrc = rd + 1 < R ? cur + rstep : rho + 1 < D ? zb + (rho + 1) * kSpec : znext;
                    cur += rstep;
#ifndef GACQ_ABL_NOWAIT
                    mbar_wait(mbar, t & 1);
#endif
                    // Z * Cc and the 33-point stage over k2 (lanes k1 < 31); results E[q2][k1]
                    if (lane < 31) {
                        const cx* Ec = zbuf + lane;
                        dft33_stream<1>(
                            [&](int k2, int dep) {
                                // k2 is a compile-time constant here: the branch folds away
                                return k2 <= 16 ? cmul(Ec[k2 * 31 + dep], ccs[k2 * kCcRow + lane + dep])
                                                : cmul_conj(Ec[k2 * 31 + dep], ccs[(33 - k2) * kCcRow + pl + dep]);
                            },
                            a.zero,
                            [&]() {  // every input consumed: the buffer takes the next spectrum
                                __syncwarp(0x7fffffffu);
                                if (lane == 0 && nsrc) bulk_load_nofence(zbuf, nsrc, kSpecBytes, mbar);
                            },
                            [&](int q2, cx v) { E[q2 * 31 + lane] = v; });
                    }
                    __syncwarp();
                    // 31-point stage over k1 for row q2 = lane (+ row 32 spread over the warp, its
                    // scratch in E[1023..1055])
                    const cx e = lane < 31 ? E[32 * 31 + lane] : czero();
                    const cx* Er = E + lane * 31;
                    // R > 1: the row's 31 loads issued first and the spread row's FMA chain run under
                    // their latency, then the Rader stage on registers (C3 -1%; at R = 1 the old
                    // order measured 0.9% faster)
                    cx xr[31];
                    if constexpr (!kR1) {
#pragma unroll
                        for (int k1 = 0; k1 < 31; ++k1) xr[k1] = Er[k1];
                        coop31<1>(e, lane, [&](int j) { return __ldg(&kCoop31Coef[j - 1][lane]); }, E + kChips,
                                  [&](int sl, int, cx v) { accx[sl] = pow_acc(v, accx[sl]); });
                    }
                    dft31_rader_inv([&](int k1) { return kR1 ? Er[k1] : xr[k1]; }, [&](int q1, cx v) {
                        const float pw = pow_acc(v, acc[q1]);
                        acc[q1] = pw;
                        if constexpr (kTop2 && kR1) {  // first max in emission order
                            const bool gt = pw > v1;
                            v2 = gt ? v1 : fmaxf(v2, pw);
                            i1 = gt ? q1 : i1;
                            v1 = gt ? pw : v1;
                        }
                    });
                    if constexpr (kR1)
                        coop31<1>(e, lane, [&](int j) { return __ldg(&kCoop31Coef[j - 1][lane]); }, E + kChips,
                                  [&](int sl, int, cx v) { accx[sl] = pow_acc(v, accx[sl]); });
                    __syncwarp();  // E is free for the next transform
                }
                // phase done: the row to scratch (and the parity power map), the running first argmax
                float m;
                if constexpr (kTop2) {
                    if constexpr (!kR1) {
#pragma unroll
                        for (int q1 = 0; q1 < 31; ++q1) {  // first max, and the second max (ties count twice)
                            const float v = acc[q1];
                            const bool gt = v > v1;
                            v2 = gt ? v1 : fmaxf(v2, v);
                            i1 = gt ? q1 : i1;
                            v1 = gt ? v : v1;
                        }
                    }
                    float* row = rows + rho * kTop2Row + lane;
                    row[0] = v1;
                    row[32] = v2;
                    row[64] = __int_as_float(i1);
                    row[96] = accx[0];
                    row[128] = accx[1];
                    m = v1;
                } else {
                    float* row = rows + rho * kPhaseRow + lane;
#pragma unroll
                    for (int q1 = 0; q1 < 31; ++q1) row[q1 * 32] = acc[q1];
                    row[31 * 32] = accx[0];
                    row[32 * 32] = accx[1];
                    m = acc[0];
#pragma unroll
                    for (int q1 = 1; q1 < 31; ++q1) m = fmaxf(m, acc[q1]);
                }
                if (pm) {
#pragma unroll
                    for (int q1 = 0; q1 < 31; ++q1) pm[D * cell_q(q1, lane) + rho] = acc[q1];
                    if (x0) pm[D * cell_q(lane == 16 ? 0 : lane, 32) + rho] = accx[0];
                    if (x1) pm[D * cell_q(31 - lane, 32) + rho] = accx[1];
                }
                // lane max (lanes without coop cells keep accx = 0, <= every power, never a lag
                // candidate), then the lowest lag holding it, searched only when it can win
                m = fmaxf(m, fmaxf(accx[0], accx[1]));
                if (m >= best) {
                    int bl = 0x7fffffff;
                    if (kTop2 && v1 == m && v2 < v1) {  // one main cell holds the lane max: its lag
                        bl = D * cell_q(i1, lane) + rho;
                    } else {  // ties (or a spread-row max): the lowest lag among the cells equal to it
                        unsigned mk = 0u;
#pragma unroll
                        for (int q1 = 0; q1 < 31; ++q1) mk |= (acc[q1] == m ? 1u : 0u) << q1;
                        while (mk) {
                            const int q1 = __ffs(mk) - 1;
                            mk &= mk - 1u;
                            bl = min(bl, D * cell_q(q1, lane) + rho);
                        }
                    }
                    if (x0 && accx[0] == m) bl = min(bl, D * cell_q(lane == 16 ? 0 : lane, 32) + rho);
                    if (x1 && accx[1] == m) bl = min(bl, D * cell_q(31 - lane, 32) + rho);
                    if (bl != 0x7fffffff && better(m, bl, best, bidx)) {
                        best = m;
                        bidx = bl;
                    }
                }
            }
            // the item's first argmax (acquisition.py:151): value desc, lag asc, over the warp
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
            }
            const int peak = bidx == 0x7fffffff ? 0 : bidx;  // all-NaN powers (non-finite input, flagged by K1)
            // exclusion floor (acquisition.py:155-159) from the scratch rows
            float fl = -1.f;
#ifdef GACQ_ABL_NOFLOOR
            if (false) {
#else
            if (2 * a.radius + 1 < a.P) {
#endif
                if constexpr (kTop2) {
                    const int cl = (31 * lane) % 33;  // the residue mod 33 of this lane's q values
#pragma unroll 4
                    for (int rho = 0; rho < D; ++rho) {
                        const unsigned off = (unsigned)(D * kChips), uD = (unsigned)D;
                        const unsigned lo = (unsigned)(peak - a.radius - rho) + off, hi = (unsigned)(peak + a.radius - rho) + off;
                        const int qa = (int)divD(lo + uD - 1u) - kChips, qb = (int)divD(hi) - kChips;
                        const float* row = rows + rho * kTop2Row + lane;
                        const float v1 = row[0], v2 = row[32], c0 = row[96], c1 = row[128];
                        const int i1 = __float_as_int(row[64]);
                        // the window's one lag of residue cl (this lane's cells) and of residue 2 (row 32)
                        const int qm = qa + ((cl - qa) % 33 + 33) % 33, qc = qa + ((2 - qa) % 33 + 33) % 33;
                        const auto wrap = [](int q) { return q < 0 ? q + kChips : q >= kChips ? q - kChips : q; };
                        const int q1m = qm <= qb ? (16 * wrap(qm)) % 31 : -1;
                        const int q1c = qc <= qb ? (16 * wrap(qc)) % 31 : -1;
                        fl = fmaxf(fl, q1m == i1 ? v2 : v1);
                        // lanes without spread-row cells hold 0 there: never above a real power
                        if (!(q1c >= 0 && x0 && q1c == (lane == 16 ? 0 : lane))) fl = fmaxf(fl, c0);
                        if (!(q1c >= 0 && x1 && q1c == 31 - lane)) fl = fmaxf(fl, c1);
                    }
                } else {
#pragma unroll 1
                for (int rho = 0; rho < D; ++rho) {
                    // excluded cells of phase rho: lags D q + rho for q in
                    // [ceil((peak - r - rho)/D), floor((peak + r - rho)/D)] (mod 1023), offset by
                    // D * 1023 (> r + rho) so both bounds divide as unsigned
                    const unsigned off = (unsigned)(D * kChips), uD = (unsigned)D;
                    const unsigned lo = (unsigned)(peak - a.radius - rho) + off, hi = (unsigned)(peak + a.radius - rho) + off;
                    const int qa = (int)divD(lo + uD - 1u) - kChips, qb = (int)divD(hi) - kChips;
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
                    const float* row = rows + rho * kPhaseRow + lane;
#pragma unroll
                    for (int q1 = 0; q1 < 31; ++q1)
                        if (!((m31 >> q1) & 1u)) fl = fmaxf(fl, row[q1 * 32]);
                    // fake 0 of lanes without coop cells: never raises the floor above a real power
                    if (!(mx & 1u)) fl = fmaxf(fl, row[31 * 32]);
                    if (!(mx & 2u)) fl = fmaxf(fl, row[32 * 32]);
                }
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
            if (lane == 0) {
                const int64_t s = pair / a.B;
                gacq_row out;
                out.bin = b;
                out.lag = peak;
                out.peak = best;
                out.floor = fl < 0.f ? 0.f : fl;
                a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
            }
        } else if (znext) {  // idle in this unit: start the next item's first spectrum now
            __syncwarp();
            if (lane == 0) bulk_load_nofence(zbuf, znext, kSpecBytes, mbar);
        }
        }  // items of the unit
        cp_async_wait_all();
        __syncthreads();  // the next unit's code spectrum and claim are visible; this unit's slot is free
        unit = nxt;
        if (unit >= a.n_units) break;
    }
}

}  // namespace gacq
