// gacq_generic.cuh -- the acquisition hot path at sample rates that are NOT chip-aligned
// (fs != D * 1.023 MHz, e.g. 2.5 / 5 / 6 / 8.192 / 20 MHz front ends).
//
// Reference path: gnssperf/acquisition.py:112-159 with its native transform length
// N = n_coh = round(fs * coherent_ms * 1e-3) and P = round(fs * 1023 / 1.023e6) lags.
// Without chip alignment the polyphase reduction of gacq_pfa.cuh does not apply. The
// reference's N-point circular correlation
//   r[tau] = IDFT_N( DFT_N(w) . conj(DFT_N(c)) )[tau],  tau < P   (dsp.py:108-119: 1/N in the ifft)
// is evaluated with one transform of M points:
//   - native (M = N), when N = 2^a 3^b 5^c: mixed-radix (16/8/4/2, 5, 3) transforms at the
//     reference's own length, no padding (5 MHz: 5000 points, 20 MHz: 20000);
//   - otherwise linear (M = 2^k >= N + P - 1): r[tau] = sum_n c[n] w_ext[n + tau] with
//     w_ext[j] = w[j mod N] (j < N + P - 1), zero beyond, so no lag wraps for tau < P.
// The code table carries conj(DFT_M(c)) / M, so no rescale is needed in either form.
//
//   K1 gacq_gen_fwd_kernel : per (snapshot, bin, round): bit-exact wipe-off (kernels.py:78-86),
//                            periodic extension / zero padding (linear form), forward FFT -> Z.
//   K2 gacq_gen_corr_kernel: per (snapshot, bin, PRN): for every round Z . Cg on load, inverse
//                            FFT, |.|^2 of the P lags accumulated; first argmax and exclusion
//                            floor (acquisition.py:151-159).
// Both transforms are Stockham passes in shared memory (below), the radix schedule planned on
// the host (GenArgs.radix). A CTA transforms at most 8192 points (7680 with radix 3 or 5
// passes: 16 values per thread across a pass's barrier); a larger M is split by one radix-L
// step over a cluster of L CTAs (L in {2, 4, 8}, L | M, Ms = M / L):
//   forward, CTA l < L:  X[L k' + l] = DFT_Ms( sum_m x[n + m Ms] W_L^(-l m) W_M^(-l n) )
//   inverse, CTA l:      E_l = IDFT_Ms(Y[L k' + l]), then each CTA takes a contiguous share of the
//                        lags and combines r[tau] = sum_l W_M^(l tau) E_l[tau mod Ms], reading the
//                        other CTAs' E_l straight from their shared memory (distributed shared
//                        memory of the thread-block cluster)
// and spectra / code tables are stored residue-major: slot l Ms + k' holds frequency L k' + l.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "gacq_kernels.cuh"
#include "rader31.cuh"  // r_dft5
#include "pfa.cuh"      // dft3_fma

namespace gacq {

constexpr int kGenMaxMs = 8192;          // points per CTA transform (power-of-two schedules)
constexpr int kGenMaxMsOdd = 7680;       // ... with a radix-3 or radix-5 pass (5 x 3 values per thread)
constexpr int kGenMaxL = 8;              // CTAs per cluster (portable cluster size)
constexpr int kGenMaxM = kGenMaxL * kGenMaxMs;
// Threads per CTA: 256 (32 values per thread per pass, two CTAs per SM) when two CTAs' shared
// memory fits an SM, else 512 (16 values per thread, one CTA per SM). A CTA's share of the lags
// is <= Ms, so each thread owns at most kGenMaxMs / T of them.
__host__ __device__ constexpr int gen_vpt(int T) { return kGenMaxMs / T; }
constexpr int kGenMaxPasses = 16;  // 4-bit radix codes in a 64-bit schedule

// padded transform buffer: gpad(i) < Ms + Ms / 16; the warp-split layout (gen_ws_base) needs
// at most Ms + Ms / 16 + 16 slots
__host__ __device__ constexpr int gen_buf(int Ms) { return Ms + Ms / 16 + 16; }
// dynamic smem of both generic kernels: one padded CTA transform (gpad), the power accumulators
// of the CTA's lags (<= Ms floats; shared memory rather than registers, where they would stay
// live across the transform and spill), and the CTA transform's twiddles W_Ms^e, e < Ms, copied
// from the plan's W_M table once per CTA (global-table reads were the top stall)
__host__ __device__ constexpr int gen_smem(int Ms) {
    return (int)sizeof(float2) * gen_buf(Ms) + (int)sizeof(float) * Ms + (int)sizeof(float2) * Ms;
}

// (cos, S sin)(2 pi e / T) from a full table of T entries
template <int S>
__device__ __forceinline__ cx gen_tw(const float2* __restrict__ tw, int e) {
    const float2 t = tw[e];  // shared-memory table in the passes, the global W_M table otherwise
    return pk(t.x, S < 0 ? -t.y : t.y);
}

// 25-point DFT as 5 x 5 (n = 5 n1 + n2, k = k1 + 5 k2): five 5-point DFTs over n1, the
// twiddles W_25^(S n2 k1) as constants, five 5-point DFTs over n2; natural order in and out
template <int S>
__device__ __forceinline__ void dft25(cx (&v)[25]) {
#pragma unroll
    for (int n2 = 0; n2 < 5; ++n2) r_dft5<S>(v[n2], v[5 + n2], v[10 + n2], v[15 + n2], v[20 + n2]);
    // v[5 k1 + n2] now holds Y[n2][k1]
    // (cos, sin)(2 pi n2 k1 / 25), float32-rounded, at [(k1 - 1) 4 + n2 - 1]
    constexpr float kC[16] = {0.9685831665992737f, 0.8763066530227661f, 0.728968620300293f, 0.5358268022537231f, 0.8763066530227661f, 0.5358268022537231f, 0.06279052048921585f, -0.4257792830467224f, 0.728968620300293f, 0.06279052048921585f, -0.6374239921569824f, -0.9921147227287292f, 0.5358268022537231f, -0.4257792830467224f, -0.9921147227287292f, -0.6374239921569824f};
    constexpr float kS[16] = {0.24868988990783691f, 0.4817536771297455f, 0.6845471262931824f, 0.8443279266357422f, 0.4817536771297455f, 0.8443279266357422f, 0.9980267286300659f, 0.9048270583152771f, 0.6845471262931824f, 0.9980267286300659f, 0.7705132365226746f, 0.12533323466777802f, 0.8443279266357422f, 0.9048270583152771f, 0.12533323466777802f, -0.7705132365226746f};
#pragma unroll
    for (int k1 = 1; k1 < 5; ++k1)
#pragma unroll
        for (int n2 = 1; n2 < 5; ++n2) {
            const int t = (k1 - 1) * 4 + n2 - 1;
            v[5 * k1 + n2] = cmul(v[5 * k1 + n2], pk(kC[t], S < 0 ? -kS[t] : kS[t]));
        }
    cx o[25];
#pragma unroll
    for (int k1 = 0; k1 < 5; ++k1) {
        r_dft5<S>(v[5 * k1], v[5 * k1 + 1], v[5 * k1 + 2], v[5 * k1 + 3], v[5 * k1 + 4]);
#pragma unroll
        for (int k2 = 0; k2 < 5; ++k2) o[k1 + 5 * k2] = v[5 * k1 + k2];
    }
#pragma unroll
    for (int i = 0; i < 25; ++i) v[i] = o[i];
}

template <int S, int R>
__device__ __forceinline__ void gen_dft(cx (&v)[R]) {
    if constexpr (R == 25) {
        dft25<S>(v);
    } else if constexpr (R == 16) {
        dft16<S>(v);
    } else if constexpr (R == 8) {
        dft8<S>(v);
    } else if constexpr (R == 5) {
        r_dft5<S>(v[0], v[1], v[2], v[3], v[4]);
    } else if constexpr (R == 4) {
        dft4<S>(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 3) {
        dft3_fma<S>(v);
    } else {
        const cx a = v[0];
        v[0] = add2(a, v[1]);
        v[1] = sub2(a, v[1]);
    }
}

// Stockham buffers are padded: element i lives at i + i/16 (the radix-16 write pattern
// x[16 j' + r] would otherwise put a warp's 32 stores into one bank group)
__device__ __forceinline__ int gpad(int i) { return i + (i >> 4); }

// One Stockham autosort pass of radix R over x[0, Ms) (natural order in, natural order out
// after the last pass), in place: every thread reads and transforms its groups, the CTA
// synchronises, then every thread writes. Group j < Ms/R reads x[j + r Ms/R], applies
// W_(Ns R)^(S k r), k = j mod Ns (Ns = product of the earlier radices), and writes
// x[(j / Ns) Ns R + k + r Ns]. `tw` is the W_Ms table (W_(Ns R)^e = W_Ms^(e Ms / (Ns R))).
// kLoad: the first pass (Ns = 1, no twiddles) takes its inputs from load(i) instead of x[i].
// kWarp: one warp transforms x alone (lanes for threads, __syncwarp for the CTA barrier).
// kPad: element i at i + (i >> kPad); 4 (gpad) suits the power-of-two strides, 6 the odd
// strides of radix-25/5/3 schedules (at 625 points: 2.5x fewer excess bank wavefronts than 4;
// no padding at all measured 6% slower, its passes spill).
// kPtw: the twiddle powers come from the pass's own table ptw[ci][Ns] (gen_ptw_c), read at unit stride
template <int S, int R, int VPT, bool kLoad = false, bool kWarp = false, int kPad = 4, bool kPtw = false,
          class Load = int>
__device__ __forceinline__ void gen_stockham_pass(cx* __restrict__ x, int Ms, int Ns, const float2* __restrict__ tw,
                                                  Load&& load = 0, const float2* __restrict__ ptw = nullptr) {
    constexpr int kGroups = VPT / R;  // groups per thread (Ms <= R kGroups blockDim)
    const int tid = kWarp ? (int)(threadIdx.x & 31) : (int)threadIdx.x, nth = kWarp ? 32 : (int)blockDim.x;
    auto sync = [] {
        if constexpr (kWarp) __syncwarp();
        else __syncthreads();
    };
    const int ng = Ms / R, tw_step = Ms / (Ns * R);
    auto pad = [](int i) { return kPad ? i + (i >> kPad) : i; };
    const bool pow2 = (Ns & (Ns - 1)) == 0;  // shifts, not divisions, while only radix-2^k passes preceded
    // j mod Ns otherwise by a multiply-high: floor(j m / 2^32) = floor(j / Ns) with
    // m = ceil(2^32 / Ns), exact here since j Ns < 2^26
    const unsigned magic = pow2 ? 0u : (unsigned)((0xffffffffull + Ns) / (unsigned)Ns);
    auto jmod = [&](int j) { return pow2 ? j & (Ns - 1) : j - (int)__umulhi((unsigned)j, magic) * Ns; };
    cx v[kGroups][R];
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
        const int j = tid + g * nth;
        if (j < ng) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if constexpr (kLoad)
                    v[g][r] = load(j + r * ng);
                else
                    v[g][r] = x[pad(j + r * ng)];
            }
            if (!kLoad && Ns > 1) {
                const int kj = jmod(j), e1 = kj * tw_step;
                // W^(c e1), c = gen_ptw_c(R, ci): the W_Ms table at stride c tw_step, or the pass's
                // own table at unit stride (the same values)
                auto twc = [&](int ci, int c) {
                    if constexpr (kPtw) {
                        const float2 t = ptw[ci * Ns + kj];
                        return pk(t.x, S < 0 ? -t.y : t.y);
                    } else {
                        return gen_tw<S>(tw, c * e1);
                    }
                };
                // W^r from the table powers W^1, W^2, W^4, W^8 and at most two products each
                // (<= 3 roundings per twiddle): 4 loads instead of R - 1
                cx w[R];
                if constexpr (R == 25) {
                    // W^(5a + b) = W^(5a) W^b from the loaded 1, 2, 4, 5, 10, 20 (<= 3 roundings)
                    w[1] = twc(0, 1);
                    w[2] = twc(1, 2);
                    w[4] = twc(2, 4);
                    w[5] = twc(3, 5);
                    w[10] = twc(4, 10);
                    w[20] = twc(5, 20);
                    w[3] = cmul(w[1], w[2]);
                    w[15] = cmul(w[5], w[10]);
#pragma unroll
                    for (int a5 = 5; a5 < 25; a5 += 5)
#pragma unroll
                        for (int b = 1; b < 5; ++b)
                            if (a5 + b != 5 && a5 + b != 10 && a5 + b != 20) w[a5 + b] = cmul(w[a5], w[b]);
#pragma unroll
                    for (int r = 1; r < R; ++r) v[g][r] = cmul(v[g][r], w[r]);
                    gen_dft<S, R>(v[g]);
                    continue;
                }
                w[1] = twc(0, 1);
                if (R > 2) w[2] = twc(1, 2);
                if (R > 4 && R != 5) w[4] = twc(2, 4);
                if (R > 8) w[8] = twc(3, 8);
#pragma unroll
                for (int r = 3; r < R; ++r) {
                    if (R == 5) {  // W^3 = W^1 W^2, W^4 = W^2 W^2
                        w[r] = r == 3 ? cmul(w[1], w[2]) : cmul(w[2], w[2]);
                        continue;
                    }
                    if ((r & (r - 1)) == 0) continue;  // powers of two are loaded
                    const int hb = r & 8 ? 8 : r & 4 ? 4 : 2;  // highest loaded power below r
                    const int rest = r - hb;
                    const int hb2 = rest & 4 ? 4 : rest & 2 ? 2 : 1;
                    w[r] = rest == hb2 ? cmul(w[hb], w[rest]) : cmul(cmul(w[hb], w[hb2]), w[rest - hb2]);
                }
#pragma unroll
                for (int r = 1; r < R; ++r) v[g][r] = cmul(v[g][r], w[r]);
            }
            gen_dft<S, R>(v[g]);
        }
    }
    sync();
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
        const int j = tid + g * nth;
        if (j < ng) {
            const int k = jmod(j);
            const int d = (j - k) * R + k;  // (j / Ns) Ns R + k
#pragma unroll
            for (int r = 0; r < R; ++r) x[pad(d + r * Ns)] = v[g][r];
        }
    }
    sync();
}

// Power-of-two CTA transforms (Ms = 2^logMs): the same pass with shifts for every index, radix 16
// and one 8/4/2 tail, the first (radix-16, twiddle-free) pass reading load(i) for x[i]. Inlined
// with compile-time radices this measured 19% faster than the general schedule at 8192 points.
template <int S, int R, int VPT, bool kLoad = false, class Load = int>
__device__ __forceinline__ void gen_p2_pass(cx* __restrict__ x, int logMs, int logNs, const float2* __restrict__ tw,
                                            Load&& load = 0) {
    constexpr int kGroups = VPT / R;
    constexpr int kLogR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int ng = (1 << logMs) >> kLogR, Ns = 1 << logNs;
    const int tw_step = 1 << (logMs - logNs - kLogR);  // W_(Ns R) in units of W_Ms
    cx v[kGroups][R];
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
        const int j = threadIdx.x + g * blockDim.x;
        if (j < ng) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if constexpr (kLoad)
                    v[g][r] = load(j + r * ng);
                else
                    v[g][r] = x[gpad(j + r * ng)];
            }
            if (!kLoad && logNs > 0) {
                const int e1 = (j & (Ns - 1)) * tw_step;
                cx w[R];
                w[1] = gen_tw<S>(tw, e1);
                if (R > 2) w[2] = gen_tw<S>(tw, 2 * e1);
                if (R > 4) w[4] = gen_tw<S>(tw, 4 * e1);
                if (R > 8) w[8] = gen_tw<S>(tw, 8 * e1);
#pragma unroll
                for (int r = 3; r < R; ++r) {
                    if ((r & (r - 1)) == 0) continue;
                    const int hb = r & 8 ? 8 : r & 4 ? 4 : 2;
                    const int rest = r - hb;
                    const int hb2 = rest & 4 ? 4 : rest & 2 ? 2 : 1;
                    w[r] = rest == hb2 ? cmul(w[hb], w[rest]) : cmul(cmul(w[hb], w[hb2]), w[rest - hb2]);
                }
#pragma unroll
                for (int r = 1; r < R; ++r) v[g][r] = cmul(v[g][r], w[r]);
            }
            gen_dft<S, R>(v[g]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
        const int j = threadIdx.x + g * blockDim.x;
        if (j < ng) {
            const int k = j & (Ns - 1);
            const int d = ((j >> logNs) << (logNs + kLogR)) + k;
#pragma unroll
            for (int r = 0; r < R; ++r) x[gpad(d + (r << logNs))] = v[g][r];
        }
    }
    __syncthreads();
}
template <int S, int VPT, class Load>
__device__ __forceinline__ void gen_p2_fft_ld(cx* __restrict__ x, int logMs, const float2* __restrict__ tw, Load&& load) {
    gen_p2_pass<S, 16, VPT, true>(x, logMs, 0, tw, load);
    int logNs = 4;
    for (; logNs + 4 <= logMs; logNs += 4) gen_p2_pass<S, 16, VPT>(x, logMs, logNs, tw);
    const int rem = logMs - logNs;
    if (rem == 3) gen_p2_pass<S, 8, VPT>(x, logMs, logNs, tw);
    else if (rem == 2) gen_p2_pass<S, 4, VPT>(x, logMs, logNs, tw);
    else if (rem == 1) gen_p2_pass<S, 2, VPT>(x, logMs, logNs, tw);
}

struct GenArgs {
    const float2* snaps;    // batch base (device), snapshot s at snaps + s*stride
    int64_t stride;         // complex samples between snapshots
    const float2* carrier;  // [B][n_coh] wipe-off replicas
    const float2* tw;       // [M] (cos, sin)(2 pi e / M)
    const cx* Cg;           // [n_prn][M] conj(DFT_M(code replica)) / M, residue-major
    cx* Z;                  // [pairs_in_chunk][R][M] spectra, residue-major
    gacq_row* rows_bin;     // [n_snap][n_prn][B]
    float* pmap;            // optional [n_prn][B][P] (single snapshot), else null
    int* bad;               // atomicMin'd to the index of a snapshot holding a non-finite sample
    int64_t pair0;          // first (snapshot, bin) pair of this chunk
    int B, R, n_coh, P, n_prn, radius;
    int M, Ms;              // transform length, points per CTA (M = L Ms)
    int n_pass;             // Stockham passes of the Ms-point CTA transform
    unsigned long long sched;  // their radices, 4 bits each from bit 0: gen_radix_code
    // warp split (W > 1, gacq_gen_corr_ws_kernel): Ms = W Q, one Q-point transform per warp
    // (W = warps per CTA) in n_wpass warp-local passes (wsched), then one radix-W step
    int W, Q, n_wpass;
    unsigned long long wsched;
    unsigned qmagic;        // ceil(2^32 / Q): e / Q = umulhi(e, qmagic) for e < Ms
};

// 4-bit codes of the pass radices in GenArgs.sched
__host__ __device__ constexpr int gen_radix_code(int R) {
    return R == 25 ? 7 : R == 16 ? 6 : R == 8 ? 5 : R == 5 ? 4 : R == 4 ? 3 : R == 3 ? 2 : 1;
}
__host__ __device__ constexpr int gen_code_radix(int c) {
    return c == 7 ? 25 : c == 6 ? 16 : c == 5 ? 8 : c == 4 ? 5 : c == 3 ? 4 : c == 2 ? 3 : 2;
}

// Every pass as an out-of-line function: each gets its own register allocation (inlined into
// the runtime radix switch, the kernels spilled the values a pass holds across its barrier)
template <int S, int R, int VPT>
__device__ __noinline__ void gen_pass_call(cx* __restrict__ x, int Ms, int Ns, const float2* __restrict__ tw) {
    gen_stockham_pass<S, R, VPT>(x, Ms, Ns, tw);
}
// first pass of the correlation kernel: inputs Z . Cg straight from global memory
template <int R, int VPT>
__device__ __noinline__ void gen_first_pass_zc(cx* __restrict__ x, int Ms, const cx* __restrict__ z,
                                               const cx* __restrict__ cg) {
    gen_stockham_pass<1, R, VPT, true>(x, Ms, 1, nullptr, [&](int k) { return cmul(__ldg(&z[k]), __ldg(&cg[k])); });
}

// In-place natural-order DFT of x[0, Ms) (sign S, unnormalised) by the plan's Stockham passes,
// starting at pass p0 with Ns = the product of the radices before it (mixed-radix schedules;
// power-of-two ones take gen_p2_fft_ld).
template <int S, int VPT>
__device__ __forceinline__ void gen_fft_from(cx* __restrict__ x, const GenArgs& a, int Ms, const float2* __restrict__ tw,
                                             int p0, int Ns) {
    for (int p = p0; p < a.n_pass; ++p) {
        const int R = gen_code_radix((int)((a.sched >> (4 * p)) & 15));
        switch (R) {
            case 25:
                if constexpr (VPT >= 25) gen_pass_call<S, 25, VPT>(x, Ms, Ns, tw);  // planned only when VPT >= 25
                break;
            case 16: gen_pass_call<S, 16, VPT>(x, Ms, Ns, tw); break;
            case 8: gen_pass_call<S, 8, VPT>(x, Ms, Ns, tw); break;
            case 5: gen_pass_call<S, 5, VPT>(x, Ms, Ns, tw); break;
            case 4: gen_pass_call<S, 4, VPT>(x, Ms, Ns, tw); break;
            case 3: gen_pass_call<S, 3, VPT>(x, Ms, Ns, tw); break;
            default: gen_pass_call<S, 2, VPT>(x, Ms, Ns, tw); break;
        }
        Ns *= R;
    }
}

// ---- warp split (gacq_gen_corr_ws_kernel) ------------------------------------------------
// Ms = W Q: warp w transforms the Q frequencies w + W q (stored contiguously, slot w Q + q, by
// the forward kernel and the host's code table) in its own padded sub-buffer with __syncwarp
// only; one radix-W step across the sub-buffers then yields the Ms-point transform.
#ifndef GACQ_GEN_XTW
#define GACQ_GEN_XTW 1
#endif
#ifndef GACQ_GEN_PTW
#define GACQ_GEN_PTW 1
#endif
#if GACQ_GEN_PTW && !GACQ_GEN_XTW
#error "GACQ_GEN_PTW keeps its tables in the W_Ms region GACQ_GEN_XTW leaves free"
#endif
constexpr int kGenWarpVpt = 32;  // values per lane in a warp pass (Q <= 1024)
// Per-pass twiddle tables of the warp passes (GACQ_GEN_PTW): a pass of radix R after Ns points
// loads the powers W^(c e1), e1 = (j mod Ns) tw_step, c = gen_ptw_c(R, ci), ci < gen_ptw_nc(R)
// (gen_stockham_pass). Read from the W_Q table they stride c tw_step entries across a warp's
// lanes: 2- to 16-way bank conflicts whenever that is even (8.192 MHz, Q = 512 as 16, 8, 4: the
// radix-8 pass strides 4, 8, 16 entries). The pass's table ptw[ci][k] = W_Q^(c k tw_step), k < Ns, holds the same
// values at unit stride. All passes after the first together take sum nc(R) Ns <= Q entries
// (checked on the host: gen_ptw_size), kept in the W_Ms region the radix-W step leaves free.
// Radix-25 passes keep the W_Q table (nc = 0). Measured: 8.192 MHz (16, 8, 4 passes) 56.3 ->
// 54.2 ms correlation; 5 MHz (25, 25) 24.9 -> 26.5 ms with a table for its second pass.
__host__ __device__ constexpr int gen_ptw_nc(int R) {
    return R == 25 ? 0 : R == 16 ? 4 : R == 8 ? 3 : (R == 4 || R == 5 || R == 3) ? 2 : 1;
}
__host__ __device__ constexpr int gen_ptw_c(int, int ci) { return 1 << ci; }  // W^1, W^2, W^4, W^8
// the tables serve the 512-thread warp-split kernels only (8.192 MHz: 16 warps of 512 points,
// passes 16, 8, 4). In the 256-thread ones (5 MHz: passes 25, 25, no table) the mere option
// changed ptxas's register allocation of the shared pass functions: 6% slower
__host__ __device__ constexpr bool gen_ws_ptw(int T) { return GACQ_GEN_PTW && T == 512; }
// staged first-pass batch (gen_wfft_zc kU): 10 at 256 threads (20 spill: 5 MHz 25.0 -> 33.2 ms);
// 20 at 512 threads, where ptxas's allocation of the whole kernel came out better with it (8.192
// MHz 53.8 -> 51.4 ms, although its power-of-two first pass never runs the staged loop)
__host__ __device__ constexpr int gen_ws_ku(int T) { return T == 512 ? 20 : 10; }
// entries of all the tables of a warp schedule (passes 1 .. n - 1)
__host__ __device__ inline int gen_ptw_size(const signed char* radix, int n) {
    int Ns = n > 0 ? radix[0] : 1, t = 0;
    for (int p = 1; p < n; ++p) {
        t += gen_ptw_nc(radix[p]) * Ns;
        Ns *= radix[p];
    }
    return t;
}
__host__ __device__ constexpr int gen_ws_base(int w, int Q) { return w * (Q + Q / 16 + 1); }
// smem of the warp-split correlation: gen_smem(Ms) and the warp transforms' own W_Q table (read
// at unit stride in their last pass; W_Ms entries e W would conflict W-fold on the banks)
__host__ __device__ constexpr int gen_smem_ws(int Ms, int Q) { return gen_smem(Ms) + (int)sizeof(float2) * Q; }

// the warp transforms' padding shift (gen_stockham_pass kPad, 0 = none): 4 for even Q, 6 for odd
// Q. At 625 points no padding at all is bank-conflict-free on every access of the 25 x 25 schedule
// (odd store stride, unit-stride loads), yet measured 5% slower than 6 (26.2 against 24.9 ms)
#ifndef GACQ_WS_ODD_PAD
#define GACQ_WS_ODD_PAD 6
#endif
__host__ __device__ constexpr int gen_ws_pad(int Q) { return (Q & 1) ? GACQ_WS_ODD_PAD : 4; }
__device__ __forceinline__ int gen_ws_at(int i, int shift) { return shift ? i + (i >> shift) : i; }

template <int S, int R, bool kLoad, int kPad, bool kPtw = false>
__device__ __noinline__ void gen_wpass_call(cx* __restrict__ x, int Q, int Ns, const float2* __restrict__ tw,
                                            const cx* __restrict__ z, const cx* __restrict__ cg) {
    // (not kLoad) tw: the pass's own twiddle table with kPtw, else the W_Q table
    if constexpr (kLoad)
        gen_stockham_pass<S, R, kGenWarpVpt, true, true, kPad>(
            x, Q, 1, tw, [&](int k) { return cmul(__ldg(&z[k]), __ldg(&cg[k])); });
    else
        gen_stockham_pass<S, R, kGenWarpVpt, false, true, kPad, kPtw>(x, Q, Ns, tw, 0, tw);
}
template <int S, bool kLoad, int kPad, bool kPtw = false>
__device__ __forceinline__ void gen_wpass_r(int R, cx* __restrict__ x, int Q, int Ns, const float2* __restrict__ tw,
                                            const cx* __restrict__ z, const cx* __restrict__ cg) {
    switch (R) {
        case 25: gen_wpass_call<S, 25, kLoad, kPad, (kPtw && gen_ptw_nc(25) > 0)>(x, Q, Ns, tw, z, cg); break;
        case 16: gen_wpass_call<S, 16, kLoad, kPad, (kPtw && gen_ptw_nc(16) > 0)>(x, Q, Ns, tw, z, cg); break;
        case 8: gen_wpass_call<S, 8, kLoad, kPad, (kPtw && gen_ptw_nc(8) > 0)>(x, Q, Ns, tw, z, cg); break;
        case 5: gen_wpass_call<S, 5, kLoad, kPad, (kPtw && gen_ptw_nc(5) > 0)>(x, Q, Ns, tw, z, cg); break;
        case 4: gen_wpass_call<S, 4, kLoad, kPad, (kPtw && gen_ptw_nc(4) > 0)>(x, Q, Ns, tw, z, cg); break;
        case 3: gen_wpass_call<S, 3, kLoad, kPad, (kPtw && gen_ptw_nc(3) > 0)>(x, Q, Ns, tw, z, cg); break;
        default: gen_wpass_call<S, 2, kLoad, kPad, kPtw>(x, Q, Ns, tw, z, cg); break;
    }
}
template <int S, bool kLoad, bool kPtw = false>
__device__ __forceinline__ void gen_wpass(int R, cx* __restrict__ x, int Q, int Ns, const float2* __restrict__ tw,
                                          const cx* __restrict__ z, const cx* __restrict__ cg) {
    if (gen_ws_pad(Q) == 4) gen_wpass_r<S, kLoad, 4, kPtw>(R, x, Q, Ns, tw, z, cg);
    else if constexpr (!kLoad) gen_wpass_r<S, false, GACQ_WS_ODD_PAD, kPtw>(R, x, Q, Ns, tw, z, cg);  // odd Q: staged first pass
}

// one warp: x = IDFT_Q(z . cg) (unnormalised). A power-of-two first pass reads z . cg straight
// from global memory; a radix-25/5/3 one reads it staged through x in batches of 10 + 10 loads
// per lane (read straight into the radix-25 pass, its 25 x 2 loads in flight spill: 5 MHz
// correlation 15.9 ms against 12.9 staged; 8.192 MHz prefers the direct read, 28.8 against 32.1).
// kPtw: the passes after the first read their twiddles from the tables at ptw (gen_load_ptw);
// kU: loads per lane in flight per batch of the staged first pass (gen_ws_ku)
template <bool kPtw, int kU>
__device__ __forceinline__ void gen_wfft_zc(cx* __restrict__ x, const GenArgs& a, const float2* __restrict__ tw,
                                            const float2* __restrict__ ptw, const cx* __restrict__ z,
                                            const cx* __restrict__ cg) {
    int R = gen_code_radix((int)(a.wsched & 15)), Ns = 1, p = 0;
    if ((R & (R - 1)) == 0) {
        gen_wpass<1, true>(R, x, a.Q, 1, tw, z, cg);
        Ns = R;
        p = 1;
    } else {
        // batches of kU loads per lane in flight (one L2 round trip per batch, not per element)

        for (int i0 = threadIdx.x & 31; i0 < a.Q; i0 += 32 * kU) {
            cx zz[kU], cc[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {  // unconditional (clamped) loads: the arrays stay in registers
                const int i = min(i0 + 32 * u, a.Q - 1);
                zz[u] = __ldg(&z[i]);
                cc[u] = __ldg(&cg[i]);
            }
            __syncwarp();  // a scheduling fence: ptxas would otherwise pair each load with its multiply
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (i0 + 32 * u < a.Q) x[gen_ws_at(i0 + 32 * u, gen_ws_pad(a.Q))] = cmul(zz[u], cc[u]);
        }
        __syncwarp();
    }
    if constexpr (kPtw) {
        const float2* pt = ptw;
        for (; p < a.n_wpass; ++p) {
            R = gen_code_radix((int)((a.wsched >> (4 * p)) & 15));
            gen_wpass<1, false, true>(R, x, a.Q, Ns, gen_ptw_nc(R) > 0 ? pt : tw, nullptr, nullptr);
            if (p > 0) pt += gen_ptw_nc(R) * Ns;  // pass 0 (Ns = 1) has no twiddles and no table
            Ns *= R;
        }
    } else {
        for (; p < a.n_wpass; ++p) {
            R = gen_code_radix((int)((a.wsched >> (4 * p)) & 15));
            gen_wpass<1, false>(R, x, a.Q, Ns, tw, nullptr, nullptr);
            Ns *= R;
        }
    }
}

// the warp passes' twiddle tables (GACQ_GEN_PTW) from the plan's W_M table: W_Q^e = W_M^(e W L)
__device__ __forceinline__ void gen_load_ptw(float2* ptw, const GenArgs& a, int WL) {
    int Ns = gen_code_radix((int)(a.wsched & 15));
    for (int p = 1; p < a.n_wpass; ++p) {
        const int R = gen_code_radix((int)((a.wsched >> (4 * p)) & 15)), tw_step = a.Q / (Ns * R);
        const int n = gen_ptw_nc(R) * Ns;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int ci = i / Ns, k = i - ci * Ns;
            ptw[i] = __ldg(&a.tw[(int64_t)gen_ptw_c(R, ci) * k * tw_step * WL]);
        }
        ptw += n;
        Ns *= R;
    }
}

// shared-memory layout of both kernels: [transform (gpad)][Ms float accumulators][Ms twiddles]
__device__ __forceinline__ float* gen_acc(cx* sm, int Ms) { return reinterpret_cast<float*>(sm + gen_buf(Ms)); }
__device__ __forceinline__ float2* gen_tws(cx* sm, int Ms) { return reinterpret_cast<float2*>(gen_acc(sm, Ms) + Ms); }
// W_Ms^e = W_M^(e L), e < Ms, into shared memory
__device__ __forceinline__ void gen_load_tws(float2* tws, const float2* __restrict__ tw, int Ms, int L) {
    for (int e = threadIdx.x; e < Ms; e += blockDim.x) tws[e] = __ldg(&tw[e * L]);
}

// grid: pairs_in_chunk * R * L CTAs of T threads (part l = blockIdx.x % L); dynamic smem gen_smem(Ms)
template <int L, bool kP2, int T>
__global__ void __launch_bounds__(T, T == 256 ? 2 : 1) gacq_gen_fwd_kernel(GenArgs a) {
    constexpr int VPT = gen_vpt(T);
    extern __shared__ __align__(16) cx sm[];
    const int M = a.M, Ms = a.Ms, N = a.n_coh;
    const int part = blockIdx.x % L, lr = blockIdx.x / L;
    const int lp = lr / a.R, rd = lr % a.R;
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    const cx* x = reinterpret_cast<const cx*>(a.snaps) + s * a.stride + (int64_t)rd * N;
    const cx* c = reinterpret_cast<const cx*>(a.carrier) + (int64_t)b * N;
    const int ext = N + a.P - 1;
    unsigned fin = 0x7f800000u;  // see fin_word
    auto wext = [&](int j) {  // wiped block; periodically extended and zero-padded in the linear form
        if (j >= ext) return czero();
        const int n = j < N ? j : j - N;
        const cx xv = __ldg(&x[n]);
        fin = fin_word(xv, fin);
        return cmul_exact(xv, __ldg(&c[n]));  // acquisition.py:141, kernels.py:78-86
    };
    auto input = [&](int j) {  // transform input j: the radix-L split step folded in
        cx y = wext(j);
        if constexpr (L > 1) {
#pragma unroll
            for (int m = 1; m < L; ++m) y = add2(y, cmul(wext(j + m * Ms), gen_tw<-1>(a.tw, ((part * m) % L) * Ms)));
            if (part) y = cmul(y, gen_tw<-1>(a.tw, part * j));
        }
        return y;
    };
    float2* tws = gen_tws(sm, Ms);
    gen_load_tws(tws, a.tw, Ms, L);
    __syncthreads();
    if constexpr (kP2) {
        gen_p2_fft_ld<-1, VPT>(sm, 31 - __clz(Ms), tws, input);  // read straight into the first pass
    } else {
        for (int i = threadIdx.x; i < Ms; i += blockDim.x) sm[gpad(i)] = input(i);  // staged (wipe, split)
        __syncthreads();
        gen_fft_from<-1, VPT>(sm, a, Ms, tws, 0, 1);
    }
    if (__syncthreads_or(fin == 0u) && threadIdx.x == 0) atomicMin(a.bad, (int)s);
    cx* dst = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
    if (a.W > 1) {  // warp-split order: slot w Q + q holds frequency w + W q (gacq_gen_corr_ws_kernel)
        for (int d = threadIdx.x; d < Ms; d += blockDim.x) {
            const int w = (int)__umulhi((unsigned)d, a.qmagic);
            dst[d] = sm[gpad((d - w * a.Q) * a.W + w)];
        }
    } else {
        for (int k = threadIdx.x; k < Ms; k += blockDim.x) dst[k] = sm[gpad(k)];
    }
}

// first argmax (value desc, lag asc) over the cluster, then the exclusion floor
// (acquisition.py:151-159), from the lags' accumulators accb[t - t0], t in [t0, t1); row out
template <int L, int T>
__device__ __forceinline__ void gen_corr_finish(const GenArgs& a, const float* accb, int t0, int t1, int lp, int pi,
                                                int part) {
    constexpr int kLags = kGenMaxMs / T;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ float red_v[T / 32], red_f[T / 32];
    __shared__ int red_i[T / 32];
    __shared__ float s_best, s_floor;
    __shared__ int s_bidx;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    auto better = [](float v, int l, float bv, int bl) { return v > bv || (v == bv && l < bl); };
    float best = -1.f;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kLags; ++i) {
        const int t = t0 + threadIdx.x + i * T;
        if (t < t1 && better(accb[t - t0], t, best, bidx)) { best = accb[t - t0]; bidx = t; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
    }
    if (lane == 0) { red_v[w] = best; red_i[w] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        best = red_v[0];
        bidx = red_i[0];
        for (int i = 1; i < nw; ++i)
            if (better(red_v[i], red_i[i], best, bidx)) { best = red_v[i]; bidx = red_i[i]; }
        s_best = best;
        s_bidx = bidx;
    }
    if constexpr (L > 1) cl.sync(); else __syncthreads();
    best = s_best;
    bidx = s_bidx;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        if (l == part) continue;
        const float ov = *cl.map_shared_rank(&s_best, l);
        const int oi = *cl.map_shared_rank(&s_bidx, l);
        if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
    }
    if (bidx == 0x7fffffff) { best = 0.f; bidx = 0; }  // all-NaN powers (non-finite input, flagged by K1)
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    float* pm = a.pmap ? a.pmap + ((int64_t)pi * a.B + b) * a.P : nullptr;
    float fl = -1.f;
#pragma unroll
    for (int i = 0; i < kLags; ++i) {
        const int t = t0 + threadIdx.x + i * T;
        if (t < t1) {
            int d = abs(t - bidx);
            d = min(d, a.P - d);
            if (d > a.radius) fl = fmaxf(fl, accb[t - t0]);  // acquisition.py:155-159
            if (pm) pm[t] = accb[t - t0];
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
    if (lane == 0) red_f[w] = fl;
    __syncthreads();
    if (threadIdx.x == 0) {
        float f = red_f[0];
        for (int i = 1; i < nw; ++i) f = fmaxf(f, red_f[i]);
        s_floor = f;
    }
    if constexpr (L > 1) cl.sync(); else __syncthreads();
    if (part == 0 && threadIdx.x == 0) {
        float f = s_floor;
#pragma unroll
        for (int l = 1; l < L; ++l) f = fmaxf(f, *cl.map_shared_rank(&s_floor, l));
        gacq_row out;
        out.bin = b;
        out.lag = bidx;
        out.peak = best;
        out.floor = f < 0.f ? 0.f : f;
        a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
    }
    if constexpr (L > 1) cl.sync();  // rank 0 has read every CTA's shared memory
}

// grid: pairs_in_chunk * n_prn * L CTAs of T threads, clusters of L along x (item =
// blockIdx.x / L = lp * n_prn + pi, part = cluster rank); dynamic smem gen_smem(Ms). CTA `part`
// owns lags [part Pc, (part + 1) Pc), Pc = ceil(P / L), and their power accumulators.
template <int L, bool kP2, int T>
__global__ void __launch_bounds__(T, T == 256 ? 2 : 1) gacq_gen_corr_kernel(GenArgs a) {
    constexpr int VPT = gen_vpt(T), kLags = kGenMaxMs / T;
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) cx sm[];
    const int M = a.M, Ms = a.Ms;
    const int item = blockIdx.x / L, part = blockIdx.x % L;
    const int lp = item / a.n_prn, pi = item % a.n_prn;
    const cx* cgt = a.Cg + (int64_t)pi * M + (int64_t)part * Ms;
    const int Pc = (a.P + L - 1) / L, t0 = part * Pc, t1 = min(a.P, t0 + Pc);
    cg::cluster_group cl = cg::this_cluster();
    float* acc = gen_acc(sm, Ms) + threadIdx.x;  // lag t0 + tid + i*512 at acc[i*512]
    float2* tws = gen_tws(sm, Ms);
    gen_load_tws(tws, a.tw, Ms, L);
#pragma unroll
    for (int i = 0; i < kLags; ++i)
        if ((int)threadIdx.x + i * T < Ms) acc[i * T] = 0.f;  // the region holds Ms floats
    __syncthreads();
    for (int rd = 0; rd < a.R; ++rd) {
        const cx* z = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
        // Z . Cg read straight into the first pass
        const int R0 = gen_code_radix((int)(a.sched & 15));
        if constexpr (kP2) {  // Z . Cg read straight into the first pass
            gen_p2_fft_ld<1, VPT>(sm, 31 - __clz(Ms), tws, [&](int k) { return cmul(__ldg(&z[k]), __ldg(&cgt[k])); });
        } else if (R0 == 16 || R0 == 8) {  // ... out of line
            if (R0 == 16) gen_first_pass_zc<16, VPT>(sm, Ms, z, cgt);
            else gen_first_pass_zc<8, VPT>(sm, Ms, z, cgt);
            gen_fft_from<1, VPT>(sm, a, Ms, tws, 1, R0);
        } else {
            for (int i = threadIdx.x; i < Ms; i += blockDim.x) sm[gpad(i)] = cmul(__ldg(&z[i]), __ldg(&cgt[i]));
            __syncthreads();
            gen_fft_from<1, VPT>(sm, a, Ms, tws, 0, 1);
        }
        if constexpr (L > 1) cl.sync();  // every E_l complete
#pragma unroll 2
        for (int i = 0; i < kLags; ++i) {
            const int t = t0 + threadIdx.x + i * T;
            if (t < t1) {
                const int e = gpad(L == 1 ? t : t % Ms);
                cx v;
                if constexpr (L == 1) {
                    v = sm[e];
                } else {  // E_l of every CTA of the cluster (distributed shared memory)
                    v = *cl.map_shared_rank(sm + e, 0);
#pragma unroll
                    for (int l = 1; l < L; ++l)
                        v = add2(v, cmul(*cl.map_shared_rank(sm + e, l), gen_tw<1>(a.tw, (int)(((int64_t)l * t) % M))));
                }
                float& A = acc[i * T];
                A = fmaf(im(v), im(v), fmaf(re(v), re(v), A));  // acquisition.py:149
            }
        }
        if constexpr (L > 1) cl.sync();  // every CTA has read E_l before the next round overwrites it
        else __syncthreads();
        // (measured: alternating two buffers to drop this barrier was no faster, at 2x the smem)
    }
    gen_corr_finish<L, T>(a, gen_acc(sm, Ms), t0, t1, lp, pi, part);
}

// Warp-split correlation: the grid, clusters, lag ownership and result of gacq_gen_corr_kernel,
// with the CTA transform taken as Ms = W Q (W = T / 32 warps):
//   F_w = IDFT_Q(Y[w + W q]) per warp (no CTA barrier inside), then for tau = t1 + Q t2
//   E[tau] = sum_w W_W^(w t2) (W_Ms^(w t1) F_w[t1]), one radix-W step per t1 (in place: the W
//   inputs of t1 and its W outputs share the slots (w, t1)).
// Two CTA barriers per round instead of two per Stockham pass, and each warp's loads overlap
// the other warps' arithmetic.
template <int L, int T>
__global__ void __launch_bounds__(T, T == 256 ? 2 : 1) gacq_gen_corr_ws_kernel(GenArgs a) {
    constexpr int W = T / 32;
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) cx sm[];
    const int M = a.M, Ms = a.Ms, Q = a.Q;
    const int wpad = gen_ws_pad(Q);
    const int item = blockIdx.x / L, part = blockIdx.x % L, warp = threadIdx.x >> 5;
    const int lp = item / a.n_prn, pi = item % a.n_prn;
    const cx* cgt = a.Cg + (int64_t)pi * M + (int64_t)part * Ms;
    const int Pc = (a.P + L - 1) / L, t0 = part * Pc, t1 = min(a.P, t0 + Pc);
    cg::cluster_group cl = cg::this_cluster();
    float* accb = gen_acc(sm, Ms);  // lag t at accb[t - t0]
    float2* tws = gen_tws(sm, Ms);
    float2* twq = tws + Ms;  // W_Q^e = W_M^(e W L)
#if GACQ_GEN_XTW
    // the radix-W step's twiddles W_Ms^(k q) as a [k - 1][q] table (k < W, q < Q: (W - 1) Q < Ms
    // entries): a warp's 32 consecutive q read it at unit stride (W_Ms^(k q) straight from the
    // W_Ms table strided k entries: up to k-way bank conflicts for each of the W - 1 loads)
    for (int i = threadIdx.x; i < (W - 1) * Q; i += T) {
        const int k1 = (int)__umulhi((unsigned)i, a.qmagic), q = i - k1 * Q;
        tws[i] = __ldg(&a.tw[(int64_t)(k1 + 1) * q * L]);
    }
    float2* ptw = tws + (W - 1) * Q;  // the warp passes' twiddle tables (<= Q entries, gen_ws_ptw)
    if (gen_ws_ptw(T)) gen_load_ptw(ptw, a, L * W);
#else
    float2* ptw = nullptr;
    gen_load_tws(tws, a.tw, Ms, L);
#endif
    gen_load_tws(twq, a.tw, Q, L * W);
    for (int i = threadIdx.x; i < Ms; i += T) accb[i] = 0.f;
    __syncthreads();
    for (int rd = 0; rd < a.R; ++rd) {
        const cx* z = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
        gen_wfft_zc<gen_ws_ptw(T), gen_ws_ku(T)>(sm + gen_ws_base(warp, Q), a, twq, ptw, z + warp * Q, cgt + warp * Q);
        __syncthreads();  // every F_w complete
        for (int q = threadIdx.x; q < Q; q += T) {
            cx v[W];
#pragma unroll
            for (int k = 0; k < W; ++k) v[k] = sm[gen_ws_base(k, Q) + gen_ws_at(q, wpad)];
#pragma unroll
            for (int k = 1; k < W; ++k) v[k] = cmul(v[k], gen_tw<1>(tws, GACQ_GEN_XTW ? (k - 1) * Q + q : k * q));
            gen_dft<1, W>(v);
#pragma unroll
            for (int k = 0; k < W; ++k) {
                if constexpr (L == 1) {
                    const int t = q + k * Q;
                    if (t < t1) accb[t] = fmaf(im(v[k]), im(v[k]), fmaf(re(v[k]), re(v[k]), accb[t]));  // acquisition.py:149
                } else {
                    sm[gen_ws_base(k, Q) + gen_ws_at(q, wpad)] = v[k];
                }
            }
        }
        if constexpr (L == 1) {
            __syncthreads();  // the sub-buffers are read before the next round's warps overwrite them
        } else {
            cl.sync();  // every E_l complete
            for (int t = t0 + threadIdx.x; t < t1; t += T) {
                const int ee = t % Ms, qq = (int)__umulhi((unsigned)ee, a.qmagic);
                const int e = gen_ws_base(qq, Q) + gen_ws_at(ee - qq * Q, wpad);
                cx v = *cl.map_shared_rank(sm + e, 0);
#pragma unroll
                for (int l = 1; l < L; ++l)
                    v = add2(v, cmul(*cl.map_shared_rank(sm + e, l), gen_tw<1>(a.tw, (int)(((int64_t)l * t) % M))));
                accb[t - t0] = fmaf(im(v), im(v), fmaf(re(v), re(v), accb[t - t0]));
            }
            cl.sync();  // every CTA has read E_l before the next round overwrites it
        }
    }
    gen_corr_finish<L, T>(a, accb, t0, t1, lp, pi, part);
}

}  // namespace gacq
