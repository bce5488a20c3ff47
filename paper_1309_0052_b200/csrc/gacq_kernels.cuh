// gacq_kernels.cuh -- sm_100a kernels of the acquisition hot path.
//
// Reference path: gnssperf/acquisition.py:128-159 (hot loop 138-149).
//
// Algorithm (see DESIGN.md section 3 for the derivation):
//   fs = D * 1.023 MHz with an exactly chip-aligned code NCO, P = 1023*D samples/period,
//   n_coh = K*P. For bin b and round r the wiped block w = x_r * carrier_b (bit-exact
//   complex64 product, kernels.py:78-86) is folded over the K code periods to wbar[P].
//   Lag tau = D*q + rho (q in [0,1023), rho in [0,D)) of the reference's circular
//   correlation ifft(fft(w) * conj(fft(code)))  equals the 1023-chip circular
//   correlation of  z_rho[m] = sum_{i<D} wbar[(D*m + rho + i) mod P]  with the chips.
//   That correlation is computed exactly as a 2048-point linear correlation:
//   g = IFFT_2048( FFT_2048(z_rho zero-padded) * Cc ),  Cc = conj(FFT_2048(d))/2048,
//   d[j] = chip[j mod 1023] (j < 2046), and lag q sits at g[1025 + q].
//
//   K1 gacq_fwd_kernel   : per (snapshot, bin, round): wipe-off + fold + D forward FFTs.
//                          Spectra are PRN-independent and written once (Z scratch).
//   K2 gacq_corr_kernel  : per (snapshot, bin, prn): for rho, round: Z*Cc on load,
//                          inverse FFT, |.|^2 accumulated in registers; the phase-major
//                          power row lives in shared memory (D <= 4) or L2 scratch;
//                          argmax + exclusion floor.
//   K3 gacq_reduce_kernel: per (snapshot, prn): merge the bin rows (peak desc, bin asc).
#pragma once
#include <cstdint>

#include "codelets.cuh"
#include "../../include/gacq.h"

namespace gacq {

constexpr int kM = 2048;        // transform length
constexpr int kT = 128;         // threads per transform (16 points each)
constexpr int kChips = 1023;
constexpr int kRow = 1024;      // phase-major power row stride (floats)
constexpr int kXchg = 2176;     // padded exchange buffer (float2): pad(2047)+1, pad(i) = i + i/16
#ifndef GACQ_CORR_MIN_BLOCKS
#define GACQ_CORR_MIN_BLOCKS 3
#endif
#ifndef GACQ_K2_TW1_SMEM
#define GACQ_K2_TW1_SMEM 0
#endif

__device__ __forceinline__ void group_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kT) : "memory");
}

// 16-byte global->shared async copy, issued only after `dep` (a value computed from the
// slot's previous contents) is available, so the slot is never overwritten early.
__device__ __forceinline__ void cp_async16_after(void* smem, const void* gmem, cx dep) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b64 p, %2, 0x7fc000017fc00001;\n"
        " @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(s),
        "l"(gmem), "l"(dep)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Exchange-buffer addresses of thread t (float2 index), all base + compile-time offset:
//   pass-0 store pad(16t + r)                  = 17t + r
//   pass-1 load  pad(t + 128r)                 = t + t/16 + 136r
//   pass-1 store pad(256(t/16) + t%16 + 16r)   = 272(t/16) + t%16 + 17r
//   pass-2 load  pad(j + 256r), j = t + 128h   = j + j/16 + 272r
struct XAddr {
    int s0, l1, s1, l2;
};
__device__ __forceinline__ XAddr xaddr(int t) {
    return XAddr{17 * t, t + (t >> 4), 272 * (t >> 4) + (t & 15), t + (t >> 4)};
}

// Stockham radix (16, 16, 8) transform of 2048 points held 16 per thread.
// Pass 0 input v[r] = x[t + 128 r]; on return u[h][r] = X[t + 128 h + 256 r].
// xs0 / xs1 are two distinct exchange buffers, so two barriers per transform suffice:
// a thread writing xs0 for transform i+1 has passed transform i's second barrier (all
// xs0 reads of i done) and one writing xs1 has passed i+1's first barrier.
// W16^r = exp(S 2 pi i r/16) as packed constants for the h = 1 pass-2 twiddles:
// W2048^((t+128) r) = W2048^(t r) * W16^r
template <int S>
__device__ __forceinline__ cx w16_mul(cx a, int r) {
    switch (r & 15) {
        case 0: return a;
        case 1: return mul_cs<S>(a, kC16, kS16);
        case 2: return mul_w8_1<S>(a);
        case 3: return mul_cs<S>(a, kS16, kC16);
        case 4: return rot<S>(a);
        case 5: return mul_cs<S>(a, -kS16, kC16);
        case 6: return mul_w8_3<S>(a);
        case 7: return mul_cs<S>(a, -kC16, kS16);
        default: return a;  // r < 8 only
    }
}

// `tw1(r)` yields the pass-1 twiddle W^(8 (t%16) r) (from registers or a shared table).
template <int S, typename Tw1, typename Sync>
__device__ __forceinline__ void fft2048(cx (&v)[16], cx (&u)[2][8], cx* __restrict__ xs0, cx* __restrict__ xs1,
                                        Tw1 tw1, const cx (&tw2)[8], const XAddr& xa, Sync sync) {
    dft16<S>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) xs0[xa.s0 + r] = v[r];
    sync();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = xs0[xa.l1 + 136 * r];
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], tw1(r));
    dft16<S>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) xs1[xa.s1 + 17 * r] = v[r];
    sync();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int r = 0; r < 8; ++r) u[h][r] = xs1[xa.l2 + 136 * h + 272 * r];
#pragma unroll
        for (int r = 1; r < 8; ++r) u[h][r] = cmul(u[h][r], h ? w16_mul<S>(tw2[r], r) : tw2[r]);
        dft8<S>(u[h]);
    }
}

// Per-thread twiddles: tw1[r] = W^(8 (t%16) r), tw2[r] = W^(t r), W = e^{S 2 pi i/2048}
template <int S>
__device__ __forceinline__ void load_twiddles(const float2* __restrict__ tw, int t, cx (&tw1)[16], cx (&tw2)[8]) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const float2 w = __ldg(&tw[((t & 15) * r * 8) & (kM - 1)]);
        tw1[r] = pk(w.x, S < 0 ? -w.y : w.y);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const float2 w = __ldg(&tw[(t * r) & (kM - 1)]);
        tw2[r] = pk(w.x, S < 0 ? -w.y : w.y);
    }
}

struct FwdArgs {
    const float2* snaps;   // batch base (device), snapshot s at snaps + s*stride
    int64_t stride;        // complex samples between snapshots
    const float2* carrier; // [B][n_coh] wipe-off replicas
    const float2* tw;      // [2048] e^{+2 pi i e/2048}
    float4* Z;             // [pairs][R][D][1024] float4 spectra (permuted layout)
    int64_t pair0;         // first (snapshot, bin) pair of this chunk, pair = s*B + b
    int B, R, n_coh, P, D, K;
};

// Row stride of the transposed wiped block wt[k][m] = wbar[D m + k]: the +16/D pad makes
// both the wipe stores (consecutive n) and the chip-sum loads (consecutive m) conflict-free.
__host__ __device__ constexpr int fwd_ws(int D) { return kRow + (D <= 16 ? 16 / D : 0); }

// Wipe-off (bit-exact, acquisition.py:141) of one coherent block x (K code periods) with the
// carrier replica c, folded over the K periods into the transposed table
// wt[k][m] = wbar[D m + k]; wt[k][1023] repeats wt[k][0] (circular chip m+1). Coalesced,
// two samples per 16-byte load. All NT threads of the CTA take part; ends with a barrier.
template <int D, int NT>
__device__ __forceinline__ void wipe_fold(const cx* __restrict__ x, const cx* __restrict__ c, int P, int K,
                                          cx* __restrict__ wt) {
    constexpr int WS = fwd_ws(D);
    auto put = [&](int n, cx w) {
        const int m = n / D, k = n - m * D;
        wt[k * WS + m] = w;
        if (m == 0) wt[k * WS + kChips] = w;
    };
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(c)) & 15) == 0 && (P & 1) == 0;
    if (vec) {
        const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(x);
        const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(c);
        const int np = P / 2;
#ifndef GACQ_WIPE_U
#define GACQ_WIPE_U 4
#endif
        constexpr int U = GACQ_WIPE_U;  // 16-byte load pairs in flight per thread
        if (K == 1) {  // one code period per block (coherent_ms = 1): no fold, twice the loads in flight
            constexpr int U1 = 2 * U;
            for (int base = threadIdx.x; base < np; base += U1 * NT) {
                ulonglong2 xv[U1], cv[U1];
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        xv[u] = __ldg(x2 + i);
                        cv[u] = __ldg(c2 + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U1; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        put(2 * i, cmul_exact(xv[u].x, cv[u].x));
                        put(2 * i + 1, cmul_exact(xv[u].y, cv[u].y));
                    }
                }
            }
            __syncthreads();
            return;
        }
        for (int base = threadIdx.x; base < np; base += U * NT) {
            cx w[U][2];
            for (int k = 0; k < K; ++k) {
                ulonglong2 xv[U], cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = base + u * NT;
                    if (i < np) {
                        xv[u] = __ldg(x2 + k * np + i);
                        cv[u] = __ldg(c2 + k * np + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const cx p0 = cmul_exact(xv[u].x, cv[u].x), p1 = cmul_exact(xv[u].y, cv[u].y);
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
            cx acc = cmul_exact(__ldg(&x[n]), __ldg(&c[n]));
            for (int k = 1; k < K; ++k) acc = add2(acc, cmul_exact(__ldg(&x[k * P + n]), __ldg(&c[k * P + n])));
            put(n, acc);
        }
    }
    __syncthreads();
}

// grid: (pairs_in_chunk * R) blocks of NG*128 threads;
// dynamic smem: (D*fwd_ws(D) + NG*2*kXchg) cx
template <int NG, int D>
__global__ void __launch_bounds__(NG * kT) gacq_fwd_kernel(FwdArgs a) {
    constexpr int WS = fwd_ws(D);
    extern __shared__ cx smem[];
    cx* wt = smem;
    const int lp = blockIdx.x / a.R, rd = blockIdx.x % a.R;
    const int64_t pair = a.pair0 + lp;
    const int64_t s = pair / a.B;
    const int b = (int)(pair % a.B);
    const cx* x = reinterpret_cast<const cx*>(a.snaps) + s * a.stride + (int64_t)rd * a.n_coh;
    const cx* c = reinterpret_cast<const cx*>(a.carrier) + (int64_t)b * a.n_coh;
    // (A) wipe-off + fold
    wipe_fold<D, NG * kT>(x, c, a.P, a.K, wt);

    // (B) group g transforms phases g, g+NG, ...; thread t owns chips m = t + 128 r (r < 8),
    //     exactly its pass-0 inputs: z_rho[m] = sum_{i<D} wbar[D m + rho + i], computed
    //     directly for the group's first phase and then slid by NG samples per phase.
    const int g = threadIdx.x / kT, t = threadIdx.x % kT;
    cx* xs0 = smem + D * WS + g * 2 * kXchg;
    cx* xs1 = xs0 + kXchg;
    cx tw1[16], tw2[8];
    load_twiddles<-1>(a.tw, t, tw1, tw2);
    const XAddr xa = xaddr(t);
    auto sync = [g]() { group_sync(1 + g); };
    cx z[8];
    for (int rho = g; rho < D; rho += NG) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int m = t + 128 * r;
            if (m >= kChips) continue;
            if (D <= 4 || rho == g) {
                cx acc = czero();
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const int k = rho + i;
                    acc = add2(acc, k < D ? wt[k * WS + m] : wt[(k - D) * WS + m + 1]);
                }
                z[r] = acc;
            } else {
#pragma unroll
                for (int j = 0; j < NG; ++j) {  // window moves from rho-NG to rho
                    const int k = rho - NG + j;
                    z[r] = add2(sub2(z[r], wt[k * WS + m]), wt[k * WS + m + 1]);
                }
            }
        }
        cx v[16], u[2][8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = (t + 128 * r < kChips) ? z[r] : czero();
#pragma unroll
        for (int r = 8; r < 16; ++r) v[r] = czero();
        fft2048<-1>(v, u, xs0, xs1, [&](int r) { return tw1[r]; }, tw2, xa, sync);
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(a.Z) + (((int64_t)lp * a.R + rd) * D + rho) * (kM / 2);
#pragma unroll
        for (int r = 0; r < 8; ++r) dst[r * 128 + t] = make_ulonglong2(u[0][r], u[1][r]);
    }
}

struct CorrArgs {
    const float4* Z;       // spectra of this chunk
    const float4* Cc;      // [n_prn][1024] conj code spectra / 2048 (permuted layout)
    const float2* tw;
    gacq_row* rows_bin;    // [n_snap][n_prn][B]
    float* pmap;           // optional [n_prn][B][P] power map (single snapshot), else null
    float* row_scratch;    // [gridDim][D*1024] when the row does not live in shared memory
    int64_t pair0;
    int64_t n_items;       // pairs_in_chunk * n_prn, item = lp * n_prn + pi
    unsigned long long* counter;  // zeroed before the launch; items >= gridDim.x are claimed here
    int B, R, D, P, n_prn, radius;
};

// Persistent: gridDim.x = resident CTA slots; CTA c starts with item c and then claims items
// in order from a global counter, so the in-flight items stay a contiguous window of the
// pair-major item list and the n_prn CTAs sharing a pair's spectra hit them in L2.
// 128 threads per CTA; dynamic smem: D*1024 floats if kRowSmem.
template <bool kRowSmem>
__global__ void __launch_bounds__(kT, GACQ_CORR_MIN_BLOCKS) gacq_corr_kernel(CorrArgs a) {
    __shared__ cx xs[2][kXchg];
    __shared__ float red_v[kT / 32];
    __shared__ int red_i[kT / 32];
    __shared__ long long s_next;
    extern __shared__ float row_smem[];  // power row [D][1024] when kRowSmem
    const int t = threadIdx.x;
    float* row = kRowSmem ? row_smem : a.row_scratch + (int64_t)blockIdx.x * a.D * kRow;
#if GACQ_K2_TW1_SMEM
    // pass-1 twiddles from a padded [16][17] table: lanes t and t+16 share a row
    // (broadcast) and the 17-stride keeps the 16 rows on distinct banks
    __shared__ cx tw1s[16 * 17];
    for (int i = t; i < 256; i += kT) {
        const float2 w = __ldg(&a.tw[((i >> 4) * (i & 15) * 8) & (kM - 1)]);
        tw1s[(i >> 4) * 17 + (i & 15)] = pk(w.x, w.y);
    }
    cx tw2[8];
    {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float2 w = __ldg(&a.tw[(t * r) & (kM - 1)]);
            tw2[r] = pk(w.x, w.y);
        }
    }
    const cx* tw1row = tw1s + (t & 15) * 17;
    auto tw1 = [tw1row](int r) { return tw1row[r]; };
    __syncthreads();
#else
    cx tw1r[16], tw2[8];
    load_twiddles<1>(a.tw, t, tw1r, tw2);
    auto tw1 = [&](int r) { return tw1r[r]; };
#endif
    const XAddr xa = xaddr(t);
    auto sync = []() { __syncthreads(); };
    const ulonglong2* Z = reinterpret_cast<const ulonglong2*>(a.Z);
    const ulonglong2* Cc = reinterpret_cast<const ulonglong2*>(a.Cc);
    const int64_t pair_span = (int64_t)a.R * a.D * (kM / 2);  // ulonglong2 per pair
    const int64_t zstep = (int64_t)a.D * (kM / 2);            // next round, same phase

    int64_t item = blockIdx.x;
    if (item >= a.n_items) return;
    // operands of the first transform
    ulonglong2 zq[8], cq[8];
    {
        const ulonglong2* zp = Z + (item / a.n_prn) * pair_span;
        const ulonglong2* cp = Cc + (item % a.n_prn) * (kM / 2);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            zq[i] = __ldg(zp + i * 128 + t);
            cq[i] = __ldg(cp + i * 128 + t);
        }
    }
    for (int64_t next; item < a.n_items; item = next) {
        if (t == 0) s_next = (long long)gridDim.x + (long long)atomicAdd(a.counter, 1ull);
        __syncthreads();
        next = s_next;
        const int64_t lp = item / a.n_prn;
        const int pi = (int)(item % a.n_prn);
        const bool has_next = next < a.n_items;
        const ulonglong2* zbase = Z + lp * pair_span;
        const ulonglong2* zbase_n = Z + (has_next ? next / a.n_prn : lp) * pair_span;
        const ulonglong2* cnext = Cc + (has_next ? next % a.n_prn : pi) * (kM / 2);
        const bool new_prn = has_next && (next % a.n_prn) != pi;

        float best = -1.f;  // this thread's first argmax over the cells it owns
        int bidx = 0x7fffffff;
        for (int rho = 0; rho < a.D; ++rho) {
            float acc[2][4];  // noncoherent power of the owned cells (acquisition.py:149)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[h][r] = 0.f;
            const ulonglong2* zp = zbase + rho * (kM / 2);
            for (int rd = 0; rd < a.R; ++rd) {
                cx v[16], u[2][8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    v[2 * i] = cmul(zq[i].x, cq[i].x);
                    v[2 * i + 1] = cmul(zq[i].y, cq[i].y);
                }
                // prefetch the next transform's spectrum (next round, next phase or next
                // item) and, when the next item is another PRN, its code spectrum
                const bool last = rd + 1 == a.R && rho + 1 == a.D;
                const ulonglong2* zn = rd + 1 < a.R ? zp + zstep : (rho + 1 < a.D ? zbase + (rho + 1) * (kM / 2) : zbase_n);
                if (!last || has_next) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) zq[i] = __ldg(zn + i * 128 + t);
                }
                if (last && new_prn) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) cq[i] = __ldg(cnext + i * 128 + t);
                }
                zp = zn;
                fft2048<1>(v, u, xs[0], xs[1], tw1, tw2, xa, sync);
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const float xr = re(u[h][4 + r]), xi = im(u[h][4 + r]);
                        acc[h][r] = fmaf(xi, xi, fmaf(xr, xr, acc[h][r]));
                    }
            }
            // output k = t + 128 h + 256 (4 + r) -> chip lag q = k - 1025; row[rho*1024 + q]
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int q = t + 128 * h + 256 * (4 + r) - 1025;
                    if (q >= 0) {
                        const float p = acc[h][r];
                        row[rho * kRow + q] = p;
                        const int lag = a.D * q + rho;
                        if (p > best || (p == best && lag < bidx)) { best = p; bidx = lag; }
                    }
                }
        }

        // first argmax of the row (acquisition.py:151): ties -> lowest lag D*q + rho
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
            if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
        }
        if ((t & 31) == 0) { red_v[t >> 5] = best; red_i[t >> 5] = bidx; }
        __syncthreads();
        best = red_v[0];
        bidx = red_i[0];
#pragma unroll
        for (int w = 1; w < kT / 32; ++w)
            if (red_v[w] > best || (red_v[w] == best && red_i[w] < bidx)) { best = red_v[w]; bidx = red_i[w]; }
        const int lag = bidx;
        // exclusion floor (acquisition.py:155-159): max over lags whose circular distance to
        // the peak, |((l - lag + P/2) mod P) - P/2| = min(|l - lag|, P - |l - lag|), exceeds
        // radius. Each thread revisits exactly the cells it wrote.
        float fl = -1.f;
        for (int rho = 0; rho < a.D; ++rho)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int q = t + 128 * h + 256 * (4 + r) - 1025;
                    if (q < 0) continue;
                    int d = abs(a.D * q + rho - lag);
                    d = min(d, a.P - d);
                    if (d > a.radius) fl = fmaxf(fl, row[rho * kRow + q]);
                }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) fl = fmaxf(fl, __shfl_xor_sync(0xffffffffu, fl, off));
        __syncthreads();
        if ((t & 31) == 0) red_v[t >> 5] = fl;
        __syncthreads();
        const int64_t pair = a.pair0 + lp;
        const int64_t s = pair / a.B;
        const int b = (int)(pair % a.B);
        if (t == 0) {
            float f = red_v[0];
#pragma unroll
            for (int w = 1; w < kT / 32; ++w) f = fmaxf(f, red_v[w]);
            gacq_row out;
            out.bin = b;
            out.lag = lag;
            out.peak = best;
            out.floor = f < 0.f ? 0.f : f;
            a.rows_bin[(s * a.n_prn + pi) * a.B + b] = out;
        }
        if (a.pmap) {
            float* dst = a.pmap + ((int64_t)pi * a.B + b) * a.P;
            for (int rho = 0; rho < a.D; ++rho)
                for (int h = 0; h < 2; ++h)
                    for (int r = 0; r < 4; ++r) {
                        const int q = t + 128 * h + 256 * (4 + r) - 1025;
                        if (q >= 0) dst[a.D * q + rho] = row[rho * kRow + q];
                    }
        }
    }
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
    int bb = 0x7fffffff;
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
    if (lane == 0) rows[w] = src[bb];
}

}  // namespace gacq
