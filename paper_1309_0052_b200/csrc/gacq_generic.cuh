// gacq_generic.cuh -- the acquisition hot path at sample rates that are NOT chip-aligned
// (fs != D * 1.023 MHz, e.g. 2.5 / 5 / 6 / 8.192 MHz front ends).
//
// Reference path: gnssperf/acquisition.py:112-159 with its native transform length
// N = n_coh = round(fs * coherent_ms * 1e-3) and P = round(fs * 1023 / 1.023e6) lags.
// Without chip alignment the polyphase reduction of gacq_pfa.cuh does not apply, so the
// reference's N-point circular correlation is evaluated exactly as a linear correlation with
// one power-of-two transform of M >= N + P - 1 points:
//   r[tau] = sum_{n<N} c[n] w[(n + tau) mod N] = sum_n c[n] w_ext[n + tau],  tau < P,
//   w_ext[j] = w[j mod N] (j < N + P - 1), zero beyond,   c = the sampled code replica
//   r = IDFT_M( DFT_M(w_ext) . conj(DFT_M(c)) / M )[0, P)      (no index wrap for tau < P)
// so no rescale is needed (the reference's ifft carries 1/N, the table carries 1/M).
// When N is itself a power of two (e.g. 8.192 MHz) the plan takes M = N: the transform is then
// the reference's circular correlation directly (j < M = N never reaches the extension), as
// long as P fits the correlation kernel's lag capacity L kGenMaxM / 2.
//
//   K1 gacq_gen_fwd_kernel : per (snapshot, bin, round): bit-exact wipe-off (kernels.py:78-86),
//                            periodic extension, zero padding, forward M-point FFT -> Z.
//   K2 gacq_gen_corr_kernel: per (snapshot, bin, PRN): for every round Z . Cg on load, inverse
//                            FFT, |.|^2 of the first P lags accumulated in registers; first
//                            argmax and exclusion floor (acquisition.py:151-159).
// Both transforms are in place in shared memory: bit-reversed load, then radix-4
// decimation-in-time passes (two radix-2 stages fused, one barrier per pass). A CTA holds at
// most kGenMaxM points; for M = 2 kGenMaxM (L = 2) the transform is split by one radix-2 step
// outside shared memory:
//   forward, CTA l in {0, 1}: X[2k' + l] = DFT_{M/2}( (x[n] + (-1)^l x[n + M/2]) W_M^(-l n) )
//   inverse, one CTA:         r[tau] = E_0[tau] + W_M^(tau) E_1[tau],  E_l = IDFT_{M/2}(Y[2k' + l])
// and spectra / code tables are stored residue-major: slot l (M/L) + k' holds frequency L k' + l.
#pragma once
#include <cstdint>

#include "gacq_kernels.cuh"

namespace gacq {

constexpr int kGenMaxLogM = 14;
constexpr int kGenMaxM = 1 << kGenMaxLogM;  // points per CTA: 128 KB of complex64 in shared memory
constexpr int kGenMaxLogMTotal = kGenMaxLogM + 1;  // M <= 2 kGenMaxM (L = 2)
constexpr int kGenThreads = 512;  // kGenMaxM = 32 * kGenThreads (gen_fft_stockham)
#ifndef GACQ_GEN_STOCKHAM
#define GACQ_GEN_STOCKHAM 1  // register-radix Stockham passes (0: in-place radix-4 DIT from bit-reversed input)
#endif
// corr kernel dynamic smem: padded transform buffer of M / L points, plus P floats when L = 1
inline int gen_corr_smem(int logM, int P) {
    const int L = logM > kGenMaxLogM ? 2 : 1, pts = (1 << logM) / L;
    return (int)sizeof(float2) * (GACQ_GEN_STOCKHAM ? pts + pts / 16 : pts) + (L == 1 ? 4 * P : 0);
}

// In-place DFT of x[0, 2^logM) held in bit-reversed order, natural order out.
// tw[e * tw_stride] = (cos, sin)(2 pi e / 2^logM), e < 2^logM / 2; S = -1 forward, +1 inverse
// (unnormalised).
template <int S>
__device__ __forceinline__ void gen_fft_inplace(cx* __restrict__ x, int logM, const float2* __restrict__ tw,
                                                int tw_stride) {
    const int M = 1 << logM;
    auto wtab = [&](int e) {
        const float2 t = __ldg(&tw[e * tw_stride]);
        return pk(t.x, S < 0 ? -t.y : t.y);
    };
    int s = 0;
    if (logM & 1) {  // one radix-2 stage of half-size 1
        for (int i = threadIdx.x; i < M / 2; i += blockDim.x) {
            const cx a = x[2 * i], b = x[2 * i + 1];
            x[2 * i] = add2(a, b);
            x[2 * i + 1] = sub2(a, b);
        }
        __syncthreads();
        s = 1;
    }
    for (; s < logM; s += 2) {
        // stages s (half-size h) and s+1 (half-size 2h) over blocks of 4h
        const int h = 1 << s;
        for (int q = threadIdx.x; q < M / 4; q += blockDim.x) {
            const int j = q & (h - 1);
            const int base = ((q >> s) << (s + 2)) + j;
            cx a0 = x[base], a1 = x[base + h], a2 = x[base + 2 * h], a3 = x[base + 3 * h];
            const cx w1 = wtab(j << (logM - s - 1));  // W_{2h}^j
            const cx w2 = wtab(j << (logM - s - 2));  // W_{4h}^j
            const cx t1 = cmul(a1, w1), t3 = cmul(a3, w1);
            const cx b0 = add2(a0, t1), b1 = sub2(a0, t1), b2 = add2(a2, t3), b3 = sub2(a2, t3);
            const cx u2 = cmul(b2, w2), u3 = rot<S>(cmul(b3, w2));  // W_{4h}^{j+h} = W_{4h}^j (S i)
            x[base] = add2(b0, u2);
            x[base + 2 * h] = sub2(b0, u2);
            x[base + h] = add2(b1, u3);
            x[base + 3 * h] = sub2(b1, u3);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int bitrev(int j, int logM) { return (int)(__brev((unsigned)j) >> (32 - logM)); }

// (cos, S sin)(2 pi e / M) for any e in [0, M) from the half table (W^(e + M/2) = -W^e)
template <int S>
__device__ __forceinline__ cx gen_tw(const float2* __restrict__ tw, int e, int M) {
    const bool hi = e >= (M >> 1);
    const float2 t = __ldg(&tw[hi ? e - (M >> 1) : e]);
    const float c = hi ? -t.x : t.x, sn = hi ? -t.y : t.y;
    return pk(c, S < 0 ? -sn : sn);
}

template <int S, int R>
__device__ __forceinline__ void gen_dft(cx (&v)[R]) {
    if constexpr (R == 16) {
        dft16<S>(v);
    } else if constexpr (R == 8) {
        dft8<S>(v);
    } else if constexpr (R == 4) {
        dft4<S>(v[0], v[1], v[2], v[3]);
    } else {
        const cx a = v[0];
        v[0] = add2(a, v[1]);
        v[1] = sub2(a, v[1]);
    }
}

// One Stockham autosort pass of radix R over x[0, Ms) (natural order in, natural order out
// after the last pass), in place: every thread reads and transforms its groups, the CTA
// synchronises, then every thread writes. Group j < Ms/R reads x[j + r Ms/R], applies
// W_(Ns R)^(S k r), k = j mod Ns, and writes x[(j / Ns) Ns R + k + r Ns]. The twiddle table
// is the plan's W_M half table, M = L Ms (W_(Ns R)^e = W_M^(e L Ms / (Ns R))).
// Stockham buffers are padded: element i lives at i + i/16 (the radix-16 write pattern
// x[16 j' + r] would otherwise put a warp's 32 stores into one bank group)
__device__ __forceinline__ int gpad(int i) { return i + (i >> 4); }

// kLoad: the first pass (logNs = 0, no twiddles) takes its inputs from load(i) instead of x[i]
template <int S, int R, int VPT, bool kLoad = false, class Load = int>
__device__ __forceinline__ void gen_stockham_pass(cx* __restrict__ x, int logMs, int logNs,
                                                  const float2* __restrict__ tw, int L, Load&& load = 0) {
    constexpr int kGroups = VPT / R;  // VPT values per thread (Ms <= VPT * blockDim)
    constexpr int kLogR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int Ms = 1 << logMs, ng = Ms >> kLogR, Ns = 1 << logNs;
    const int tw_step = L << (logMs - logNs - kLogR);  // W_(Ns R) in units of W_M
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
            const int k = j & (Ns - 1);
            if (logNs > 0) {
                // W^r from the table powers W^1, W^2, W^4, W^8 and at most two products each
                // (<= 3 roundings per twiddle): 4 loads instead of R - 1
                const int Mt = L << logMs, e1 = k * tw_step;
                cx w[R];
                w[1] = gen_tw<S>(tw, e1, Mt);
                if (R > 2) w[2] = gen_tw<S>(tw, 2 * e1, Mt);
                if (R > 4) w[4] = gen_tw<S>(tw, 4 * e1, Mt);
                if (R > 8) w[8] = gen_tw<S>(tw, 8 * e1, Mt);
#pragma unroll
                for (int r = 3; r < R; ++r) {
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

// In-place natural-order DFT of x[0, 2^logMs) (sign S, unnormalised): radix-16 passes, then
// one radix-8/4/2 pass for the remaining bits. Needs 2^logMs <= VPT * blockDim; VPT = 16 halves
// the values each thread holds across a pass's barrier (no spills at 128 registers).
template <int S, int VPT>
__device__ __forceinline__ void gen_fft_stockham(cx* __restrict__ x, int logMs, const float2* __restrict__ tw, int L) {
    int logNs = 0;
    for (; logNs + 4 <= logMs; logNs += 4) gen_stockham_pass<S, 16, VPT>(x, logMs, logNs, tw, L);
    const int rem = logMs - logNs;
    if (rem == 3) gen_stockham_pass<S, 8, VPT>(x, logMs, logNs, tw, L);
    else if (rem == 2) gen_stockham_pass<S, 4, VPT>(x, logMs, logNs, tw, L);
    else if (rem == 1) gen_stockham_pass<S, 2, VPT>(x, logMs, logNs, tw, L);
}
// As gen_fft_stockham, with the first (radix-16, twiddle-free) pass reading load(i) for x[i]:
// the inputs come straight from global memory, saving one shared-memory round trip and a barrier.
template <int S, int VPT, class Load>
__device__ __forceinline__ void gen_fft_stockham_ld(cx* __restrict__ x, int logMs, const float2* __restrict__ tw, int L,
                                                    Load&& load) {
    gen_stockham_pass<S, 16, VPT, true>(x, logMs, 0, tw, L, load);
    int logNs = 4;
    for (; logNs + 4 <= logMs; logNs += 4) gen_stockham_pass<S, 16, VPT>(x, logMs, logNs, tw, L);
    const int rem = logMs - logNs;
    if (rem == 3) gen_stockham_pass<S, 8, VPT>(x, logMs, logNs, tw, L);
    else if (rem == 2) gen_stockham_pass<S, 4, VPT>(x, logMs, logNs, tw, L);
    else if (rem == 1) gen_stockham_pass<S, 2, VPT>(x, logMs, logNs, tw, L);
}
// values per thread of a transform of 2^logMs points on kGenThreads threads
constexpr int gen_vpt(int logMs) { return (1 << logMs) <= 16 * 512 ? 16 : 32; }



struct GenArgs {
    const float2* snaps;    // batch base (device), snapshot s at snaps + s*stride
    int64_t stride;         // complex samples between snapshots
    const float2* carrier;  // [B][n_coh] wipe-off replicas
    const float2* tw;       // [M/2] (cos, sin)(2 pi e / M)
    const cx* Cg;           // [n_prn][M] conj(DFT_M(code replica)) / M, residue-major
    cx* Z;                  // [pairs_in_chunk][R][M] spectra, residue-major
    gacq_row* rows_bin;     // [n_snap][n_prn][B]
    float* pmap;            // optional [n_prn][B][P] (single snapshot), else null
    int* bad;               // atomicMin'd to the index of a snapshot holding a non-finite sample
    int64_t pair0;          // first (snapshot, bin) pair of this chunk
    int B, R, n_coh, P, logM, n_prn, radius;  // M = 2^logM in total, L = 1 or 2 CTA-sized parts
};


// grid: pairs_in_chunk * R * L CTAs of kGenThreads; dynamic smem (M / L) * 8 bytes;
// VPT = gen_vpt(logM - (L == 2))
template <int L, int VPT>
__global__ void __launch_bounds__(kGenThreads, 1) gacq_gen_fwd_kernel(GenArgs a) {
    extern __shared__ __align__(16) cx sm[];
    const int M = 1 << a.logM, Ms = M / L, logMs = a.logM - (L == 2), N = a.n_coh;
    const int part = blockIdx.x % L, lr = blockIdx.x / L;
    const int lp = lr / a.R, rd = lr % a.R;
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    const cx* x = reinterpret_cast<const cx*>(a.snaps) + s * a.stride + (int64_t)rd * N;
    const cx* c = reinterpret_cast<const cx*>(a.carrier) + (int64_t)b * N;
    const int ext = N + a.P - 1;
    unsigned fin = 0x7f800000u;  // see fin_word
    auto wext = [&](int j) {  // periodically extended, zero-padded wiped block
        if (j >= ext) return czero();
        const int n = j < N ? j : j - N;
        const cx xv = __ldg(&x[n]);
        fin = fin_word(xv, fin);
        return cmul_exact(xv, __ldg(&c[n]));  // acquisition.py:141, kernels.py:78-86
    };
    auto input = [&](int j) {  // transform input j (the L = 2 split folds in its radix-2 step)
        cx y = wext(j);
        if (L == 2) {
            const cx u = wext(j + Ms);
            y = part == 0 ? add2(y, u) : cmul(sub2(y, u), gen_tw<-1>(a.tw, j, M));
        }
        return y;
    };
#if GACQ_GEN_STOCKHAM
    gen_fft_stockham_ld<-1, VPT>(sm, logMs, a.tw, L, input);  // read straight into the first pass
#else
#pragma unroll 4
    for (int j = threadIdx.x; j < Ms; j += blockDim.x) sm[bitrev(j, logMs)] = input(j);
    __syncthreads();
    gen_fft_inplace<-1>(sm, logMs, a.tw, L);
#endif
    if (__syncthreads_or(fin == 0u) && threadIdx.x == 0) atomicMin(a.bad, (int)s);
    cx* dst = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
    for (int k = threadIdx.x; k < Ms; k += blockDim.x) dst[k] = sm[GACQ_GEN_STOCKHAM ? gpad(k) : k];
}

// grid: pairs_in_chunk * n_prn CTAs of kGenThreads (item = lp * n_prn + pi);
// dynamic smem: the transform buffer (M / L) * 8 bytes (padded), then for L = 1 the P float
// power accumulators (shared memory rather than registers: live across the transform they
// would push the 512-thread CTA past its 128 registers -- gen_corr_smem)
template <int L, int VPT>
__global__ void __launch_bounds__(kGenThreads, 1) gacq_gen_corr_kernel(GenArgs a) {
    extern __shared__ __align__(16) cx sm[];
    __shared__ float red_v[kGenThreads / 32], red_f[kGenThreads / 32];
    __shared__ int red_i[kGenThreads / 32];
    constexpr int kPer = L * kGenMaxM / 2 / kGenThreads;  // lags per thread (P <= M/2)
    const int M = 1 << a.logM, Ms = M / L, logMs = a.logM - (L == 2);
    const int lp = blockIdx.x / a.n_prn, pi = blockIdx.x % a.n_prn;
    const cx* cg = a.Cg + (int64_t)pi * M;
    constexpr bool kSmemAcc = L == 1;
    float acc[kSmemAcc ? 1 : kPer];
    float* accs = reinterpret_cast<float*>(sm + (GACQ_GEN_STOCKHAM ? Ms + Ms / 16 : Ms));
    // power accumulator of this thread's lag i (t = threadIdx.x + i kGenThreads < P)
    auto A = [&](int i) -> float& { return kSmemAcc ? accs[threadIdx.x + i * kGenThreads] : acc[i]; };
    cx e0[L == 2 ? kPer : 1];  // E_0 of this thread's lags while E_1 is computed
#pragma unroll
    for (int i = 0; i < kPer; ++i)
        if (!kSmemAcc || threadIdx.x + i * kGenThreads < a.P) A(i) = 0.f;
    for (int rd = 0; rd < a.R; ++rd) {
        const cx* z = a.Z + ((int64_t)lp * a.R + rd) * M;
#pragma unroll
        for (int part = 0; part < L; ++part) {
#if GACQ_GEN_STOCKHAM
            // Z . Cg read straight into the first pass (logMs >= 4 on this path)
            gen_fft_stockham_ld<1, VPT>(sm, logMs, a.tw, L, [&](int k) {
                return cmul(__ldg(&z[part * Ms + k]), __ldg(&cg[part * Ms + k]));
            });
#else
#pragma unroll 8  // keep 16 L2 loads in flight per thread
            for (int k = threadIdx.x; k < Ms; k += blockDim.x)
                sm[bitrev(k, logMs)] = cmul(__ldg(&z[part * Ms + k]), __ldg(&cg[part * Ms + k]));
            __syncthreads();
            gen_fft_inplace<1>(sm, logMs, a.tw, L);
#endif
            if constexpr (kSmemAcc) {
                // lag t = tid + i kGenThreads sits at sb[i kSt] (gpad(tid + 512 i) = gpad(tid) + 544 i):
                // one base address instead of kPer, which would stay live across the transform
                constexpr int kSt = GACQ_GEN_STOCKHAM ? kGenThreads + kGenThreads / 16 : kGenThreads;
                const cx* sb = sm + (GACQ_GEN_STOCKHAM ? gpad(threadIdx.x) : threadIdx.x);
                float* ab = accs + threadIdx.x;
                const int nl = (a.P - (int)threadIdx.x + kGenThreads - 1) / kGenThreads;
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    if (i < nl) {
                        const cx v = sb[i * kSt];
                        ab[i * kGenThreads] = fmaf(im(v), im(v), fmaf(re(v), re(v), ab[i * kGenThreads]));
                    }
                }
            } else {
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int t = threadIdx.x + i * kGenThreads;
                if (t < a.P) {
                    cx v = sm[GACQ_GEN_STOCKHAM ? gpad(t) : t];
                    if (L == 2 && part == 0) {
                        e0[i] = v;
                        continue;
                    }
                    if (L == 2) v = add2(e0[i], cmul(v, gen_tw<1>(a.tw, t, M)));  // E_0 + W_M^t E_1
                    A(i) = fmaf(im(v), im(v), fmaf(re(v), re(v), A(i)));  // acquisition.py:149
                }
            }
            }
            __syncthreads();
        }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    auto better = [](float v, int l, float bv, int bl) { return v > bv || (v == bv && l < bl); };
    float best = -1.f;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int t = threadIdx.x + i * kGenThreads;
        if (t < a.P && better(A(i), t, best, bidx)) { best = A(i); bidx = t; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (better(ov, oi, best, bidx)) { best = ov; bidx = oi; }
    }
    if (lane == 0) { red_v[w] = best; red_i[w] = bidx; }
    __syncthreads();
    best = red_v[0];
    bidx = red_i[0];
    for (int i = 1; i < nw; ++i)
        if (better(red_v[i], red_i[i], best, bidx)) { best = red_v[i]; bidx = red_i[i]; }
    if (bidx == 0x7fffffff) { best = 0.f; bidx = 0; }  // all-NaN powers (non-finite input, flagged by K1)
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    float* pm = a.pmap ? a.pmap + ((int64_t)pi * a.B + b) * a.P : nullptr;
    float fl = -1.f;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int t = threadIdx.x + i * kGenThreads;
        if (t < a.P) {
            int d = abs(t - bidx);
            d = min(d, a.P - d);
            if (d > a.radius) fl = fmaxf(fl, A(i));  // acquisition.py:155-159
            if (pm) pm[t] = A(i);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
    if (lane == 0) red_f[w] = fl;
    __syncthreads();
    if (threadIdx.x == 0) {
        float f = red_f[0];
        for (int i = 1; i < nw; ++i) f = fmaxf(f, red_f[i]);
        gacq_row out;
        out.bin = b;
        out.lag = bidx;
        out.peak = best;
        out.floor = f < 0.f ? 0.f : f;
        a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
    }
}

}  // namespace gacq
