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
// the reference's circular correlation directly (j < M = N never reaches the extension).
//
//   K1 gacq_gen_fwd_kernel : per (snapshot, bin, round): bit-exact wipe-off (kernels.py:78-86),
//                            periodic extension, zero padding, forward M-point FFT -> Z.
//   K2 gacq_gen_corr_kernel: per (snapshot, bin, PRN): for every round Z . Cg on load, inverse
//                            FFT, |.|^2 of the first P lags accumulated in registers; first
//                            argmax and exclusion floor (acquisition.py:151-159).
// Both transforms are Stockham passes in shared memory (below). A CTA transforms at most
// kGenMaxMs = 8192 points (16 values per thread across a pass's barrier: no spills); larger M is
// split by one radix-L step over a cluster of L = M / 8192 CTAs (L <= 8, M <= 65536):
//   forward, CTA l < L:  X[L k' + l] = DFT_Ms( sum_m x[n + m Ms] W_L^(-l m) W_M^(-l n) ),  Ms = M / L
//   inverse, CTA l:      E_l = IDFT_Ms(Y[L k' + l]), then each CTA takes a contiguous share of the
//                        lags and combines r[tau] = sum_l W_M^(l tau) E_l[tau mod Ms], reading the
//                        other CTAs' E_l straight from their shared memory (distributed shared
//                        memory of the thread-block cluster)
// and spectra / code tables are stored residue-major: slot l Ms + k' holds frequency L k' + l.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "gacq_kernels.cuh"

namespace gacq {

constexpr int kGenMaxLogMs = 13;
constexpr int kGenMaxMs = 1 << kGenMaxLogMs;        // points per CTA transform
constexpr int kGenMaxL = 8;                         // CTAs per cluster (portable cluster size)
constexpr int kGenMaxLogMTotal = kGenMaxLogMs + 3;  // M <= 65536
constexpr int kGenThreads = 512;
constexpr int kGenVPT = kGenMaxMs / kGenThreads;    // values per thread per pass (16)
constexpr int kGenLags = kGenMaxMs / kGenThreads;   // lags per thread: a CTA's share of P is <= Ms
__host__ __device__ constexpr int gen_split(int logM) { return logM > kGenMaxLogMs ? 1 << (logM - kGenMaxLogMs) : 1; }
// the CTA transform's twiddles W_Ms^e, e < Ms/2, copied into shared memory once per CTA: the
// Stockham passes read them there instead of from global memory (long-scoreboard stalls)
__host__ __device__ constexpr int gen_tws_bytes(int logM) { return (int)sizeof(float2) * ((1 << logM) / gen_split(logM) / 2); }
// dynamic smem of both generic kernels: one padded CTA transform (gpad), then (correlation
// kernel) the power accumulators of the CTA's lags, <= Ms floats: in shared memory rather than
// registers, where they would stay live across the transform and spill; then the twiddles
__host__ __device__ constexpr int gen_smem(int logM) {
    return (int)sizeof(float2) * ((1 << logM) / gen_split(logM) + (1 << logM) / gen_split(logM) / 16) +
           (int)sizeof(float) * ((1 << logM) / gen_split(logM)) + gen_tws_bytes(logM);
}

// (cos, S sin)(2 pi e / M) for any e in [0, M) from the half table (W^(e + M/2) = -W^e)
template <int S>
__device__ __forceinline__ cx gen_tw(const float2* __restrict__ tw, int e, int M) {
    const bool hi = e >= (M >> 1);
    const float2 t = tw[hi ? e - (M >> 1) : e];  // shared-memory table in the passes, global otherwise
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


// grid: pairs_in_chunk * R * L CTAs of kGenThreads (part l = blockIdx.x % L); dynamic smem gen_smem
template <int L>
__global__ void __launch_bounds__(kGenThreads, 1) gacq_gen_fwd_kernel(GenArgs a) {
    extern __shared__ __align__(16) cx sm[];
    const int M = 1 << a.logM, logMs = a.logM - (L == 8 ? 3 : L == 4 ? 2 : L == 2 ? 1 : 0), Ms = 1 << logMs;
    const int N = a.n_coh;
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
    auto input = [&](int j) {  // transform input j: the radix-L split step folded in
        cx y = wext(j);
        if constexpr (L > 1) {
#pragma unroll
            for (int m = 1; m < L; ++m) y = add2(y, cmul(wext(j + m * Ms), gen_tw<-1>(a.tw, ((part * m) % L) * Ms, M)));
            if (part) y = cmul(y, gen_tw<-1>(a.tw, part * j, M));
        }
        return y;
    };
    float2* tws = reinterpret_cast<float2*>(reinterpret_cast<float*>(sm + Ms + Ms / 16) + Ms);
    for (int e = threadIdx.x; e < Ms / 2; e += blockDim.x) tws[e] = __ldg(&a.tw[e * L]);  // W_Ms^e = W_M^(e L)
    __syncthreads();
    gen_fft_stockham_ld<-1, kGenVPT>(sm, logMs, tws, 1, input);  // read straight into the first pass
    if (__syncthreads_or(fin == 0u) && threadIdx.x == 0) atomicMin(a.bad, (int)s);
    cx* dst = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
    for (int k = threadIdx.x; k < Ms; k += blockDim.x) dst[k] = sm[gpad(k)];
}

// grid: pairs_in_chunk * n_prn * L CTAs of kGenThreads, clusters of L along x (item =
// blockIdx.x / L = lp * n_prn + pi, part = cluster rank); dynamic smem gen_smem. CTA `part`
// owns lags [part Pc, (part + 1) Pc), Pc = ceil(P / L), and their power accumulators.
template <int L>
__global__ void __launch_bounds__(kGenThreads, 1) gacq_gen_corr_kernel(GenArgs a) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) cx sm[];
    __shared__ float red_v[kGenThreads / 32], red_f[kGenThreads / 32];
    __shared__ int red_i[kGenThreads / 32];
    __shared__ float s_best, s_floor;
    __shared__ int s_bidx;
    const int M = 1 << a.logM, logMs = a.logM - (L == 8 ? 3 : L == 4 ? 2 : L == 2 ? 1 : 0), Ms = 1 << logMs;
    const int item = blockIdx.x / L, part = blockIdx.x % L;
    const int lp = item / a.n_prn, pi = item % a.n_prn;
    const cx* cgt = a.Cg + (int64_t)pi * M + (int64_t)part * Ms;
    const int Pc = (a.P + L - 1) / L, t0 = part * Pc, t1 = min(a.P, t0 + Pc);
    cg::cluster_group cl = cg::this_cluster();
    float* acc = reinterpret_cast<float*>(sm + Ms + Ms / 16) + threadIdx.x;  // lag t0 + tid + i*512 at acc[i*512]
    float2* tws = reinterpret_cast<float2*>(reinterpret_cast<float*>(sm + Ms + Ms / 16) + Ms);
    for (int e = threadIdx.x; e < Ms / 2; e += blockDim.x) tws[e] = __ldg(&a.tw[e * L]);  // W_Ms^e = W_M^(e L)
#pragma unroll
    for (int i = 0; i < kGenLags; ++i)
        if ((int)threadIdx.x + i * kGenThreads < Ms) acc[i * kGenThreads] = 0.f;  // the region holds Ms floats
    for (int rd = 0; rd < a.R; ++rd) {
        // an opaque copy of logMs per round: the passes' thread-invariant addresses are then
        // recomputed each round instead of hoisted out of the loop and held live (spills)
        int lgs = logMs;
        asm volatile("" : "+r"(lgs));
        cx* const X = sm;
        const cx* z = a.Z + ((int64_t)lp * a.R + rd) * M + (int64_t)part * Ms;
        // Z . Cg read straight into the first pass (logMs >= 4 on this path)
        gen_fft_stockham_ld<1, kGenVPT>(X, lgs, tws, 1, [&](int k) { return cmul(__ldg(&z[k]), __ldg(&cgt[k])); });
        if constexpr (L > 1) cl.sync();  // every E_l complete
#pragma unroll 2
        for (int i = 0; i < kGenLags; ++i) {
            const int t = t0 + threadIdx.x + i * kGenThreads;
            if (t < t1) {
                const int e = gpad(t & (Ms - 1));
                cx v;
                if constexpr (L == 1) {
                    v = X[e];
                } else {  // E_l of every CTA of the cluster (distributed shared memory)
                    v = *cl.map_shared_rank(X + e, 0);
#pragma unroll
                    for (int l = 1; l < L; ++l)
                        v = add2(v, cmul(*cl.map_shared_rank(X + e, l), gen_tw<1>(a.tw, (l * t) & (M - 1), M)));
                }
                float& A = acc[i * kGenThreads];
                A = fmaf(im(v), im(v), fmaf(re(v), re(v), A));  // acquisition.py:149
            }
        }
        if constexpr (L > 1) cl.sync();  // every CTA has read E_l before the next round overwrites it
        else __syncthreads();
        // (measured: alternating two buffers to drop this barrier was no faster, at 2x the smem)
    }
    // first argmax (value desc, lag asc) over the cluster, then the exclusion floor (acquisition.py:151-159)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    auto better = [](float v, int l, float bv, int bl) { return v > bv || (v == bv && l < bl); };
    float best = -1.f;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kGenLags; ++i) {
        const int t = t0 + threadIdx.x + i * kGenThreads;
        if (t < t1 && better(acc[i * kGenThreads], t, best, bidx)) { best = acc[i * kGenThreads]; bidx = t; }
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
    for (int i = 0; i < kGenLags; ++i) {
        const int t = t0 + threadIdx.x + i * kGenThreads;
        if (t < t1) {
            int d = abs(t - bidx);
            d = min(d, a.P - d);
            if (d > a.radius) fl = fmaxf(fl, acc[i * kGenThreads]);  // acquisition.py:155-159
            if (pm) pm[t] = acc[i * kGenThreads];
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

}  // namespace gacq
