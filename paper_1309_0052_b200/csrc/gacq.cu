// gacq.cu -- libgacq.so: C ABI (include/gacq.h) + plan/table construction + launch pipeline.
//
// Host-side responsibilities (the kernels are in gacq_kernels.cuh):
//   * validation mirroring acquisition.py:114-126 (lengths) and 201-204 (PRN list),
//   * bit-exact NCO tables: carrier replicas (kernels.py:61-62,106-114) and the
//     code chip-index sequence (kernels.py:65-70,116-128) used to prove the
//     chip-aligned structure the device algorithm relies on,
//   * conjugate code spectra (acquisition.py:84-105) computed in float64,
//   * a chunked K1 -> K2 launch pipeline over (snapshot, bin) pairs with the H2D of
//     the next snapshots overlapped on a copy stream, then K3 and one D2H.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gacq_kernels.cuh"
#include "gacq_pfa.cuh"
#include "gacq_tables.cuh"
#include "gacq_generic.cuh"
#include "gtrk_kernels.cuh"
#include "gtrk_close.h"

using namespace gacq;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(GACQ_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));       \
    } while (0)

constexpr int64_t kCarrierScale = int64_t(1) << 48;
constexpr int64_t kCodeScale = int64_t(1) << 42;
constexpr int64_t kCodeModulus = int64_t(1023) << 42;
constexpr double kChipRate = 1.023e6;
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

// Python's int(round(x)) on a finite double: round-half-even (nearbyint, default mode)
int64_t py_round(double x) { return (int64_t)std::nearbyint(x); }

int64_t py_mod(int64_t a, int64_t m) {
    int64_t r = a % m;
    return r < 0 ? r + m : r;
}

// cacode.py:41-58 -- G1 taps 3,10; G2 taps 2,3,6,8,9,10; output G1[10]^G2[s1]^G2[s2]
const int kG2Select[32][2] = {{2, 6},  {3, 7},  {4, 8},  {5, 9},  {1, 9},  {2, 10}, {1, 8},  {2, 9},
                              {3, 10}, {2, 3},  {3, 4},  {5, 6},  {6, 7},  {7, 8},  {8, 9},  {9, 10},
                              {1, 4},  {2, 5},  {3, 6},  {4, 7},  {5, 8},  {6, 9},  {1, 3},  {4, 6},
                              {5, 7},  {6, 8},  {7, 9},  {8, 10}, {1, 6},  {2, 7},  {3, 8},  {4, 9}};

void ca_code(int prn, int8_t* out) {
    int g1[10], g2[10];
    for (int i = 0; i < 10; ++i) g1[i] = g2[i] = 1;
    const int s1 = kG2Select[prn - 1][0] - 1, s2 = kG2Select[prn - 1][1] - 1;
    for (int i = 0; i < 1023; ++i) {
        out[i] = (g1[9] ^ g2[s1] ^ g2[s2]) ? 1 : -1;
        const int f1 = g1[2] ^ g1[9];
        const int f2 = g2[1] ^ g2[2] ^ g2[5] ^ g2[7] ^ g2[8] ^ g2[9];
        for (int k = 9; k > 0; --k) { g1[k] = g1[k - 1]; g2[k] = g2[k - 1]; }
        g1[0] = f1;
        g2[0] = f2;
    }
}

// Generic-path transform plan: M = n_coh when n_coh = 2^a 3^b 5^c (native, circular), else the
// power of two >= n_coh + P - 1 (linear); L CTAs of Ms = M / L points each (gacq_generic.cuh)
struct GenPlan {
    int M = 0, L = 1, Ms = 0, n_pass = 0;
    int T = 512;  // threads per CTA: 256 (two CTAs per SM) when two CTAs' shared memory fits
    bool native = false;
    signed char radix[gacq::kGenMaxPasses] = {};
    // warp split (gacq_gen_corr_ws_kernel): W = T / 32 transforms of Q = Ms / W points, W = 1 off
    int W = 1, Q = 0, n_wpass = 0;
    signed char wradix[gacq::kGenMaxPasses] = {};
    static unsigned long long code(const signed char* r, int n) {
        unsigned long long v = 0;
        for (int p = 0; p < n; ++p) v |= (unsigned long long)gacq::gen_radix_code(r[p]) << (4 * p);
        return v;
    }
    unsigned long long sched() const { return code(radix, n_pass); }
    unsigned long long wsched() const { return code(wradix, n_wpass); }
    unsigned qmagic() const { return W > 1 ? (unsigned)((0xffffffffull + Q) / (unsigned)Q) : 0u; }
};

bool smooth235(int64_t n) {
    for (int p : {2, 3, 5})
        while (n % p == 0) n /= p;
    return n == 1;
}

// Stockham radix schedule of an Ms-point CTA transform: radix 16 while it divides, one 8/4/2
// pass for the remaining power of two, then the fives and threes
// build with -DGACQ_GEN_WS=0 to keep the CTA-wide transform in the generic correlation (A/B)
#ifndef GACQ_GEN_WS
#define GACQ_GEN_WS 1
#endif
int radix_schedule(int n, bool r25, signed char* radix) {
    int m = n, e2 = 0, np = 0;
    while (m % 2 == 0) { m /= 2; ++e2; }
    // 2^e2 as radix-16 passes and one 8 or 4; a lone remaining factor 2 becomes (8, 4) in
    // place of (16, 2) (the radix-2 pass is the most expensive per flop)
    int n16 = e2 / 4, rem = e2 % 4;
    if (rem == 1 && n16 > 0) { --n16; rem = 5; }
    for (int i = 0; i < n16; ++i) radix[np++] = 16;
    if (rem == 5) { radix[np++] = 8; radix[np++] = 4; }
    else if (rem) radix[np++] = (signed char)(1 << rem);
    // fives in pairs as radix-25 passes (5 x 5 in registers: one pass and barrier pair less)
    // when a thread holds 32 values per pass
    for (; r25 && m % 25 == 0; m /= 25) radix[np++] = 25;
    for (; m % 5 == 0; m /= 5) radix[np++] = 5;
    for (; m % 3 == 0; m /= 3) radix[np++] = 3;
    return np;
}
void gen_passes(GenPlan& g) {
    g.n_pass = radix_schedule(g.Ms, g.T == 256, g.radix);
    // warp split when every warp pass fits a lane's kGenWarpVpt values (Q / R groups <= 32 (VPT / R))
    const int W = g.T / 32;
    g.W = 1;
    if (!GACQ_GEN_WS || g.Ms % W) return;
    const int Q = g.Ms / W;
    signed char wr[gacq::kGenMaxPasses];
    const int nw = radix_schedule(Q, true, wr);
    if (Q < 64 || Q > 32 * gacq::kGenWarpVpt) return;
    if (g.T == 256 && 2 * (gacq::gen_smem_ws(g.Ms, Q) + 2048) > 228 * 1024) return;  // keep two CTAs per SM
    for (int p = 0; p < nw; ++p)
        if (Q / wr[p] > 32 * (gacq::kGenWarpVpt / wr[p])) return;
    if (gacq::gen_ws_ptw(g.T) && gacq::gen_ptw_size(wr, nw) > Q) return;  // the warp passes' twiddle tables fit Q entries
    g.W = W;
    g.Q = Q;
    g.n_wpass = nw;
    std::copy(wr, wr + nw, g.wradix);
}

void gen_threads(GenPlan& g) { g.T = 2 * (gacq::gen_smem(g.Ms) + 2048) <= 228 * 1024 ? 256 : 512; }

// false when no transform of at most kGenMaxM points serves (n_coh, P)
bool gen_plan(int64_t n_coh, int64_t P, GenPlan& g) {
    if (smooth235(n_coh) && n_coh >= 16) {
        for (int L = 1; L <= gacq::kGenMaxL; L *= 2) {
            if (n_coh % L) break;
            const int64_t Ms = n_coh / L;
            const bool pow2 = (Ms & (Ms - 1)) == 0;
            // (splitting 8192 into a 2-CTA cluster of 4096-point, 256-thread CTAs measured 1.5x slower)
            if (Ms <= (pow2 ? gacq::kGenMaxMs : gacq::kGenMaxMsOdd)) {
                g.native = true;
                g.M = (int)n_coh;
                g.L = L;
                g.Ms = (int)Ms;
                gen_threads(g);
                gen_passes(g);
                return true;
            }
        }
    }
    int64_t M = 16;
    while (M < n_coh + P - 1) M *= 2;
    if (M > gacq::kGenMaxM) return false;
    g.native = false;
    g.M = (int)M;
    g.L = (int)std::max<int64_t>(1, M / gacq::kGenMaxMs);
    g.Ms = (int)(M / g.L);
    gen_threads(g);
    gen_passes(g);
    return true;
}

// mixed-radix complex DFT in float64, sign -1 (forward), any length (recursive decimation in
// time over its smallest prime factors; every twiddle from cos/sin of its own angle)
void dft_f64_rec(std::complex<double>* x, int64_t n) {
    if (n == 1) return;
    int64_t p = 2;
    while (n % p) ++p;
    const int64_t m = n / p;
    std::vector<std::complex<double>> sub((size_t)n);
    for (int64_t r = 0; r < p; ++r)
        for (int64_t j = 0; j < m; ++j) sub[(size_t)(r * m + j)] = x[j * p + r];
    for (int64_t r = 0; r < p; ++r) dft_f64_rec(sub.data() + r * m, m);
    std::vector<std::complex<double>> t((size_t)p);
    for (int64_t k = 0; k < m; ++k) {
        for (int64_t r = 0; r < p; ++r) {
            const double ang = -kTwoPi * (double)(r * k) / (double)n;
            t[(size_t)r] = sub[(size_t)(r * m + k)] * std::complex<double>(std::cos(ang), std::sin(ang));
        }
        for (int64_t q = 0; q < p; ++q) {
            std::complex<double> acc = 0.0;
            for (int64_t r = 0; r < p; ++r) {
                const double ang = -kTwoPi * (double)((r * q) % p) / (double)p;
                acc += t[(size_t)r] * std::complex<double>(std::cos(ang), std::sin(ang));
            }
            x[k + m * q] = acc;
        }
    }
}

// iterative radix-2 complex FFT in float64, sign -1 (forward)
void fft_f64(std::vector<std::complex<double>>& a) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const double ang = -kTwoPi * (double)k / (double)len;
                const std::complex<double> w(std::cos(ang), std::sin(ang));
                const auto u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

}  // namespace

struct gacq_ctx {
    std::mutex mu;
    int device = 0;
    double fs = 0;
    int n_coh = 0, P = 0, D = 0, K = 0, R = 0, B = 0, n_prn = 0, radius = 0;
    float2* d_ccp = nullptr;  // PFA conj code spectra [n_prn][kCcHalf]
    bool gen = false;         // generic power-of-two path (rates that are not chip-aligned)
    GenPlan gp;               // its transform (gacq_generic.cuh): M, CTAs per cluster, passes
    float2* d_gtw = nullptr;  // [M/2] (cos, sin)(2 pi e / M)
    float2* d_gcc = nullptr;  // [n_prn][M] conj(DFT_M(code replica)) / M
    std::vector<double> bins;
    std::vector<int32_t> prns;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    float2* d_carrier = nullptr;
    char* d_Z = nullptr;
    int64_t z_pairs = 0;     // pairs per chunk that fit in the scratch budget
    int64_t z_bytes = 0;     // allocated scratch (grown on demand, up to the budget)
    int64_t pair_bytes = 0;  // spectra of one (snapshot, bin) pair
    float2* d_in = nullptr;
    int64_t in_cap = 0;   // complex64 staging (samples)
    char* d_raw = nullptr;
    int64_t raw_cap = 0;  // quantized H2D staging (bytes)
    gacq_row* d_rows_bin = nullptr;
    int64_t rows_bin_cap = 0;
    gacq_row* d_rows = nullptr;
    int64_t rows_cap = 0;
    float* d_pmap = nullptr;
    float* d_prow = nullptr;         // K2 per-phase power rows [corr_slots][kCorrWarps][D][kPhaseRow]
    int64_t corr_slots = 0;          // resident K2 CTAs (persistent grid)
    unsigned long long* d_counter = nullptr;  // K2 work counter
    int* d_bad = nullptr;   // lowest snapshot index holding a non-finite sample (K1 atomicMin)
    int* h_bad = nullptr;   // pinned copy of d_bad
    std::vector<cudaEvent_t> copy_events;
    std::vector<cudaEvent_t> prof_events;
    cudaEvent_t wait_event = nullptr;  // gacq_wait_stream
    gacq_stats stats{};
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
int grow(T** ptr, int64_t* cap, int64_t need) {
    if (need <= *cap) return GACQ_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    if (cudaMalloc((void**)ptr, sizeof(T) * (size_t)need) != cudaSuccess) {
        cudaGetLastError();
        return fail(GACQ_ERR_RESOURCE, "cudaMalloc of %lld bytes failed", (long long)(sizeof(T) * need));
    }
    *cap = need;
    return GACQ_OK;
}

// PFA K1 instantiations: (D, warps per CTA) for every D <= 16 at which the reference's 42-bit
// code NCO is exactly chip-aligned (checked in gacq_create)
#define GACQ_PFA_FWD_VARIANTS(X) X(1, 1) X(2, 2) X(4, 4) X(5, 5) X(6, 6) X(8, 8) X(13, 7) X(14, 7) X(16, 8)

bool fwd_supported(int D) {
#define GACQ_HAS_FWD(DD, WW) if (D == DD) return true;
    GACQ_PFA_FWD_VARIANTS(GACQ_HAS_FWD)
#undef GACQ_HAS_FWD
    return false;
}

cudaError_t launch_fwd_pfa(const gacq_ctx* c, const FwdPfaArgs& fa, int64_t blocks) {
#define GACQ_LAUNCH_FWDP(DD, WW)                                                                        \
    if (c->D == DD) {                                                                                   \
        gacq_fwd_pfa_kernel<DD, WW><<<(unsigned)blocks, 32 * WW, fwd_pfa_smem(DD, WW), c->stream>>>(fa); \
        return cudaGetLastError();                                                                      \
    }
    GACQ_PFA_FWD_VARIANTS(GACQ_LAUNCH_FWDP)
#undef GACQ_LAUNCH_FWDP
    return cudaErrorInvalidConfiguration;
}

// K2 variant: phase summaries when every exclusion window spans <= 33 chip lags (kTop2), and the
// R = 1 instantiation (kR1, kR1PairsPerWarp pairs per warp per unit) on top of that
bool corr_pfa_top2(int radius, int D) { return 2 * (int64_t)radius < 33 * (int64_t)D; }
bool corr_pfa_r1(int radius, int D, int R) { return R == 1 && corr_pfa_top2(radius, D); }

cudaError_t launch_corr_pfa(const gacq_ctx* c, const CorrPfaArgs& ca) {
    const int64_t blocks = std::min<int64_t>(c->corr_slots, ca.n_units);
    // phase summaries when every exclusion window spans <= 33 chip lags (gacq_pfa.cuh, kTop2)
    const bool top2 = corr_pfa_top2(ca.radius, ca.D);
    if (corr_pfa_r1(ca.radius, ca.D, ca.R))
        gacq_corr_pfa_kernel<true, true><<<(unsigned)blocks, 32 * kCorrWarps, corr_pfa_smem(), c->stream>>>(ca);
    else if (top2)
        gacq_corr_pfa_kernel<true, false><<<(unsigned)blocks, 32 * kCorrWarps, corr_pfa_smem(), c->stream>>>(ca);
    else
        gacq_corr_pfa_kernel<false, false><<<(unsigned)blocks, 32 * kCorrWarps, corr_pfa_smem(), c->stream>>>(ca);
    return cudaGetLastError();
}

// generic kernels: clusters of gp.L CTAs (distributed shared memory, gacq_generic.cuh) of gp.T
// threads; every (L, power-of-two, T) instantiation through one dispatch
#define GACQ_GEN_DISPATCH(F)                                                                       \
    F(1, true, 256) F(1, false, 256) F(2, true, 256) F(2, false, 256) F(4, true, 256) F(4, false, 256) \
    F(8, true, 256) F(8, false, 256) F(1, true, 512) F(1, false, 512) F(2, true, 512) F(2, false, 512) \
    F(4, true, 512) F(4, false, 512) F(8, true, 512) F(8, false, 512)

template <int L, bool kP2, int T>
cudaError_t launch_gen_corr_l(const gacq_ctx* c, const GenArgs& ga, int64_t blocks) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(T);
    cfg.dynamicSmemBytes = c->gp.W > 1 ? gen_smem_ws(c->gp.Ms, c->gp.Q) : gen_smem(c->gp.Ms);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = L;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (c->gp.W > 1) return cudaLaunchKernelEx(&cfg, gacq_gen_corr_ws_kernel<L, T>, ga);
    return cudaLaunchKernelEx(&cfg, gacq_gen_corr_kernel<L, kP2, T>, ga);
}
cudaError_t launch_gen(const gacq_ctx* c, const GenArgs& ga, int64_t np, bool corr) {
    const bool p2 = (c->gp.Ms & (c->gp.Ms - 1)) == 0;
    const int L = c->gp.L, T = c->gp.T;
#define GACQ_GEN_LAUNCH(LL, PP, TT)                                                                          \
    if (L == LL && p2 == PP && T == TT) {                                                                    \
        if (corr) return launch_gen_corr_l<LL, PP, TT>(c, ga, np * c->n_prn * LL);                           \
        gacq_gen_fwd_kernel<LL, PP, TT><<<(unsigned)(np * c->R * LL), TT, gen_smem(c->gp.Ms), c->stream>>>(ga); \
        return cudaGetLastError();                                                                           \
    }
    GACQ_GEN_DISPATCH(GACQ_GEN_LAUNCH)
#undef GACQ_GEN_LAUNCH
    return cudaErrorInvalidConfiguration;
}

cudaEvent_t prof_event(gacq_ctx* c, size_t i) {
    while (c->prof_events.size() <= i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->prof_events.push_back(e);
    }
    return c->prof_events[i];
}

// Snapshot batch as handed to gacq_run / gacq_run_quantized.
struct Input {
    const void* ptr;
    int fmt;         // kFmtComplex64, or GACQ_FMT_INT8 / GACQ_FMT_INT16 interleaved I/Q
    double scale;    // full-scale amplitude of integer formats (iffile.py:32-43)
    bool on_device;
    int64_t stride;  // samples (I/Q pairs) between snapshot starts
};
constexpr int kFmtComplex64 = -1;

int sample_bytes(int fmt) { return fmt == GACQ_FMT_INT8 ? 2 : fmt == GACQ_FMT_INT16 ? 4 : (int)sizeof(float2); }

// integer I/Q -> complex64 exactly as read_if_file: float32(float64(q) * (scale / limit))
// (iffile.py:95-98; limit 127 / 32767, iffile.py:43)
cudaError_t launch_dequant(const gacq_ctx* c, const Input& in, int64_t s0, int64_t ns, const void* src,
                           int64_t src_stride, float2* dst, int64_t span) {
    const double s = in.scale / (in.fmt == GACQ_FMT_INT8 ? 127.0 : 32767.0);
    const int64_t n = ns * span;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    if (in.fmt == GACQ_FMT_INT8)
        gacq_dequant_kernel<int8_t><<<blocks, 256, 0, c->copy_stream>>>(
            (const int8_t*)src, src_stride, reinterpret_cast<cx*>(dst), span, n, s);
    else
        gacq_dequant_kernel<int16_t><<<blocks, 256, 0, c->copy_stream>>>(
            (const int16_t*)src, src_stride, reinterpret_cast<cx*>(dst), span, n, s);
    (void)s0;
    return cudaGetLastError();
}

// Core pipeline. `in.ptr` is a device pointer when in.on_device, else a host pointer.
#ifndef GACQ_CHUNK_GROWTH
#define GACQ_CHUNK_GROWTH 8  // staged input: each compute chunk this many times the previous (4: e2e -0.6% C3, -1.5% C1)
#endif
int run_impl(gacq_ctx* c, const Input& inp, int64_t n_snap, bool per_bin, bool profile, gacq_row* rows_out,
             bool rows_on_device, float* pmap) {
    const int64_t span = (int64_t)c->R * c->n_coh;
    const int64_t n_pairs = n_snap * c->B;
    const int64_t n_rows = n_snap * c->n_prn;
    const bool quantized = inp.fmt != kFmtComplex64;
    // the prime-factor K1 dequantizes integer I/Q in its wipe load; the generic path reads a
    // complex64 staging copy made by the dequant kernel on the copy stream
    const bool fused_q = quantized && !c->gen;
    const bool staged = !inp.on_device || (quantized && !fused_q);
    int rc;
    if ((rc = grow(&c->d_rows_bin, &c->rows_bin_cap, n_rows * c->B))) return rc;
    if (!per_bin && (rc = grow(&c->d_rows, &c->rows_cap, n_rows))) return rc;

    cudaEvent_t run_start = nullptr, run_end = nullptr;
    if (profile) {
        run_start = prof_event(c, 0);
        run_end = prof_event(c, 1);
        CUDA_TRY(cudaEventRecord(run_start, staged ? c->copy_stream : c->stream));
    }
    // K1 lowers d_bad to the index of any snapshot holding a NaN or an infinity
    CUDA_TRY(cudaMemsetAsync(c->d_bad, 0x7f, sizeof(int), c->stream));
    const void* in = inp.ptr;
    int64_t in_stride = inp.stride;
    // Staging in snapshot chunks on the copy stream (H2D and/or dequantization);
    // chunk k is covered by copy_events[k]
    int64_t copy_chunk = 0, n_copy_chunks = 0;
    if (staged) {
        if (!fused_q && (rc = grow(&c->d_in, &c->in_cap, n_snap * span))) return rc;
        const int64_t sb = sample_bytes(inp.fmt);
        if (quantized && !inp.on_device && (rc = grow(&c->d_raw, &c->raw_cap, n_snap * span * sb))) return rc;
        in = fused_q ? (const void*)c->d_raw : (const void*)c->d_in;
        in_stride = span;
        // fine-grained copies (<= 16 snapshots per event) so the first compute chunk, which is
        // kept small below, starts after a few MB of H2D rather than after a whole chunk
        copy_chunk = std::max<int64_t>(1, std::min<int64_t>({n_snap, c->z_pairs / c->B, (int64_t)16}));
        n_copy_chunks = (n_snap + copy_chunk - 1) / copy_chunk;
        while ((int64_t)c->copy_events.size() < n_copy_chunks) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->copy_events.push_back(e);
        }
        // the copies are enqueued lazily, a compute chunk ahead (enqueue_copies below), so the
        // first compute chunk reaches the GPU after a few API calls rather than after all of them
        if (!inp.on_device) c->stats.h2d_bytes += n_snap * span * sb;
    }
    const bool on_device = !staged;
    int64_t copies_enqueued = 0;
    // enqueue the copy chunks (H2D and/or dequantization on the copy stream) that cover
    // snapshots [0, snap_end), each ending in copy_events[k]
    auto enqueue_copies = [&](int64_t snap_end) -> int {
        if (!staged) return GACQ_OK;
        const int64_t sb = sample_bytes(inp.fmt);
        const char* src = (const char*)inp.ptr;
        for (; copies_enqueued < n_copy_chunks && copies_enqueued * copy_chunk < snap_end; ++copies_enqueued) {
            const int64_t k = copies_enqueued, s0 = k * copy_chunk, ns = std::min(copy_chunk, n_snap - s0);
            if (!quantized) {
                CUDA_TRY(cudaMemcpy2DAsync(c->d_in + s0 * span, span * sb, src + s0 * inp.stride * sb,
                                           inp.stride * sb, span * sb, ns, cudaMemcpyHostToDevice, c->copy_stream));
            } else if (!inp.on_device) {
                CUDA_TRY(cudaMemcpy2DAsync(c->d_raw + s0 * span * sb, span * sb, src + s0 * inp.stride * sb,
                                           inp.stride * sb, span * sb, ns, cudaMemcpyHostToDevice, c->copy_stream));
                if (!fused_q) {
                    CUDA_TRY(launch_dequant(c, inp, s0, ns, c->d_raw + s0 * span * sb, span, c->d_in + s0 * span, span));
                    c->stats.launches++;
                }
            } else {
                CUDA_TRY(launch_dequant(c, inp, s0, ns, src + s0 * inp.stride * sb, inp.stride, c->d_in + s0 * span,
                                        span));
                c->stats.launches++;
            }
            CUDA_TRY(cudaEventRecord(c->copy_events[k], c->copy_stream));
        }
        return GACQ_OK;
    };
    {   // spectrum scratch: the largest chunk this call runs (whole K2 pair groups)
        int64_t need = std::min(c->z_pairs, n_pairs);
        if (!c->gen) need = std::min(c->z_pairs, (need + kCorrWarps - 1) / kCorrWarps * kCorrWarps);
        if ((rc = grow(&c->d_Z, &c->z_bytes, need * c->pair_bytes))) return rc;
    }

    size_t ev = 2;
    int64_t waited = -1;
    std::vector<std::pair<size_t, int>> timed;  // (event index, kernel kind)
    // staged input: a short first chunk (its snapshots arrive first) hides the pipeline fill, and
    // the chunks then grow 8x up to z_pairs, so each one waits only for the snapshots it reads
    // while the copy stream stays ahead (H2D of a snapshot is ~10x faster than its search)
    int64_t want = !on_device ? std::min(c->z_pairs, std::max<int64_t>(copy_chunk * c->B, 2 * c->corr_slots / std::max(1, c->n_prn) + 1))
                              : c->z_pairs;
    for (int64_t p0 = 0, np = 0; p0 < n_pairs; p0 += np) {
        np = std::min(want, n_pairs - p0);
        want = std::min(c->z_pairs, GACQ_CHUNK_GROWTH * want);
        if (!on_device) {
            const int64_t last_snap = (p0 + np - 1) / c->B;
            // this chunk's copies and the next (GACQ_CHUNK_GROWTH x larger) chunk's, so the copy
            // stream stays ahead while the host enqueues this chunk's kernels
            const int64_t next_end = std::min(n_pairs, p0 + np + std::min(want, n_pairs - p0 - np));
            if ((rc = enqueue_copies((next_end + c->B - 1) / c->B))) return rc;
            const int64_t need = last_snap / copy_chunk;
            for (int64_t k = waited + 1; k <= need; ++k)
                CUDA_TRY(cudaStreamWaitEvent(c->stream, c->copy_events[k], 0));
            waited = std::max(waited, need);
        }
        cx* Zp = reinterpret_cast<cx*>(c->d_Z);  // (char-typed allocation, 16-byte aligned by cudaMalloc)
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); timed.push_back({ev++, 0}); }
        GenArgs ga{(const float2*)in, in_stride, c->d_carrier, c->d_gtw, reinterpret_cast<const cx*>(c->d_gcc), Zp, c->d_rows_bin,
                   pmap, c->d_bad, p0, c->B, c->R, c->n_coh, c->P, c->n_prn, c->radius, c->gp.M, c->gp.Ms,
                   c->gp.n_pass, c->gp.sched(), c->gp.W, c->gp.Q, c->gp.n_wpass, c->gp.wsched(), c->gp.qmagic()};
        if (c->gen) {
            CUDA_TRY(launch_gen(c, ga, np, false));
        } else {
            const int fmt = fused_q ? inp.fmt : kFmtComplex64;
            const double qs = inp.scale / (inp.fmt == GACQ_FMT_INT8 ? 127.0 : 32767.0);
            FwdPfaArgs fa{in, in_stride, fmt, qs, c->d_carrier, Zp, c->d_bad, p0, c->B, c->R, c->n_coh, c->P, c->K};
            CUDA_TRY(launch_fwd_pfa(c, fa, np * c->R));
        }
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); ev++; }
        if (!c->gen) CUDA_TRY(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned long long), c->stream));
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); timed.push_back({ev++, 1}); }
        if (c->gen) {
            CUDA_TRY(launch_gen(c, ga, np, true));
        } else {
            // pairs per warp per unit: kR1PairsPerWarp in the R = 1 instantiation launch_corr_pfa picks
            const int ipw = corr_pfa_r1(c->radius, c->D, c->R) ? kR1PairsPerWarp : 1;
            const int64_t n_units = (np + kCorrWarps * ipw - 1) / (kCorrWarps * ipw) * c->n_prn;
            if (n_units + c->corr_slots >= INT32_MAX) return fail(GACQ_ERR_UNSUPPORTED, "chunk too large");
            CorrPfaArgs ca{Zp, reinterpret_cast<const cx*>(c->d_ccp), c->d_rows_bin, pmap, c->d_prow, p0, (int)np,
                           (int)n_units, c->d_counter, c->B, c->R, c->D, c->P, c->n_prn, c->radius, 0,
                           (unsigned)(((1ull << 32) + c->D - 1) / c->D)};
            CUDA_TRY(launch_corr_pfa(c, ca));
        }
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); ev++; }
        c->stats.fwd_launches++;
        c->stats.corr_launches++;
        c->stats.launches += 2;
    }
    const gacq_row* result = c->d_rows_bin;
    int64_t n_out = n_rows * c->B;
    if (!per_bin) {
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); timed.push_back({ev++, 2}); }
        const int64_t threads = n_rows * 32;
        gacq_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, c->stream>>>(c->d_rows_bin, c->d_rows,
                                                                                    n_rows, c->B);
        CUDA_TRY(cudaGetLastError());
        if (profile) { CUDA_TRY(cudaEventRecord(prof_event(c, ev), c->stream)); ev++; }
        c->stats.reduce_launches++;
        c->stats.launches++;
        result = c->d_rows;
        n_out = n_rows;
    }
    if (rows_out) {
        if (rows_on_device) {
            CUDA_TRY(cudaMemcpyAsync(rows_out, result, n_out * sizeof(gacq_row), cudaMemcpyDeviceToDevice, c->stream));
        } else {
            CUDA_TRY(cudaMemcpyAsync(rows_out, result, n_out * sizeof(gacq_row), cudaMemcpyDeviceToHost, c->stream));
            c->stats.d2h_bytes += n_out * (int64_t)sizeof(gacq_row);
        }
    }
    CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (profile) CUDA_TRY(cudaEventRecord(run_end, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (!on_device) CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
    if (profile) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, run_start, run_end));
        c->stats.run_ms += ms;
    }
    for (auto& te : timed) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->prof_events[te.first], c->prof_events[te.first + 1]));
        (te.second == 0 ? c->stats.fwd_ms : te.second == 1 ? c->stats.corr_ms : c->stats.reduce_ms) += ms;
    }
    c->stats.calls++;
    c->stats.cells += n_snap * c->n_prn * c->B;
    // the reference refuses such buffers (IqBuffer, buffers.py:62-63); rows of the other
    // snapshots are valid
    if (*c->h_bad < n_snap)
        return fail(GACQ_ERR_INVALID, "IqBuffer samples must be finite (snapshot %d)", *c->h_bad);
    return GACQ_OK;
}

void destroy_ctx(gacq_ctx* c) {
    if (!c) return;
    {
        DeviceGuard g(c->device);
        if (c->stream) cudaStreamSynchronize(c->stream);
        cudaFree(c->d_carrier);
        cudaFree(c->d_Z);
        cudaFree(c->d_ccp);
        cudaFree(c->d_gtw);
        cudaFree(c->d_gcc);
        cudaFree(c->d_in);
        cudaFree(c->d_raw);
        cudaFree(c->d_rows_bin);
        cudaFree(c->d_rows);
        cudaFree(c->d_pmap);
        cudaFree(c->d_prow);
        cudaFree(c->d_counter);
        cudaFree(c->d_bad);
        if (c->h_bad) cudaFreeHost(c->h_bad);
        for (auto e : c->copy_events) cudaEventDestroy(e);
        for (auto e : c->prof_events) cudaEventDestroy(e);
        if (c->wait_event) cudaEventDestroy(c->wait_event);
        if (c->stream) cudaStreamDestroy(c->stream);
        if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    }
    delete c;
}

}  // namespace

extern "C" {

int gacq_version(void) { return GACQ_ABI_VERSION; }

const char* gacq_last_error(void) { return g_last_error.c_str(); }

int gacq_ca_code(int32_t prn, int8_t* out) {
    if (prn < 1 || prn > 32) return fail(GACQ_ERR_INVALID, "prn must be an integer in 1..32, got %d", prn);
    if (!out) return fail(GACQ_ERR_INVALID, "null output");
    ca_code(prn, out);
    return GACQ_OK;
}

int gacq_create(gacq_ctx** out, const gacq_params* p) {
    if (!out || !p) return fail(GACQ_ERR_INVALID, "null argument");
    *out = nullptr;
    if (!(p->sample_rate_hz > 0) || !std::isfinite(p->sample_rate_hz))
        return fail(GACQ_ERR_INVALID, "sample_rate_hz must be > 0");
    if (p->coherent_ms < 1 || p->noncoherent_rounds < 1)
        return fail(GACQ_ERR_INVALID, "coherent_ms and noncoherent_rounds must be >= 1");
    if (p->n_bins < 1 || !p->doppler_bins_hz) return fail(GACQ_ERR_INVALID, "need >= 1 Doppler bin");
    if (p->exclusion_radius_samples < 0) return fail(GACQ_ERR_INVALID, "exclusion_radius_samples must be >= 0");
    if (p->n_prn < 1 || p->n_prn > 32 || !p->prns) return fail(GACQ_ERR_INVALID, "prns must be non-empty (<= 32)");
    for (int i = 0; i < p->n_prn; ++i) {
        if (p->prns[i] < 1 || p->prns[i] > 32)
            return fail(GACQ_ERR_INVALID, "prn must be an integer in 1..32, got %d", p->prns[i]);
        for (int j = 0; j < i; ++j)
            if (p->prns[j] == p->prns[i]) return fail(GACQ_ERR_INVALID, "prns must be distinct");
    }
    const double fs = p->sample_rate_hz;
    const int64_t n_coh = py_round(fs * p->coherent_ms * 1e-3);        // acquisition.py:116
    const int64_t P = py_round(fs * 1023.0 / kChipRate);              // acquisition.py:108-109
    if (n_coh < P) return fail(GACQ_ERR_INVALID, "coherent window shorter than one code period");
    // Chip-aligned rates (fs = D * 1.023 MHz with the code NCO indexing chips exactly as
    // floor(n / D) mod 1023, kernels.py:116-128) take the 1023-point path; every other rate
    // takes the generic power-of-two path (gacq_generic.cuh).
    const int64_t code_step = py_round((kChipRate / fs) * (double)kCodeScale);
    bool aligned = P % 1023 == 0 && n_coh % P == 0 && fwd_supported((int)(P / 1023));
    if (aligned) {
        const int64_t Dl = P / 1023;
        int64_t ph = 0;
        for (int64_t n = 0; n < n_coh && aligned; ++n) {
            aligned = (ph >> 42) == (n / Dl) % 1023;
            ph = (ph + code_step) % kCodeModulus;
        }
    }
    const bool gen = !aligned || (p->plan_flags & GACQ_PLAN_GENERIC);
    GenPlan gp;
    if (gen && !gen_plan(n_coh, P, gp))
        return fail(GACQ_ERR_UNSUPPORTED,
                    "fs=%.17g Hz, coherent_ms=%d: the generic path's transform (n_coh = %lld is not 2^a 3^b 5^c "
                    "within %d points, and n_coh + P - 1 = %lld exceeds %d); chip-aligned rates "
                    "(fs = D*1.023 MHz, D <= 16) take the prime-factor path",
                    fs, p->coherent_ms, (long long)n_coh, kGenMaxM, (long long)(n_coh + P - 1), kGenMaxM);
    const int D = gen ? 0 : (int)(P / 1023), K = gen ? 0 : (int)(n_coh / P);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GACQ_ERR_CUDA, "no CUDA device visible");
    }
    if (p->device < 0 || p->device >= ndev) return fail(GACQ_ERR_INVALID, "device %d out of range", p->device);

    gacq_ctx* c = new gacq_ctx();
    c->device = p->device;
    c->fs = fs;
    c->n_coh = (int)n_coh;
    c->P = (int)P;
    c->D = D;
    c->K = K;
    c->R = p->noncoherent_rounds;
    c->B = p->n_bins;
    c->n_prn = p->n_prn;
    c->radius = p->exclusion_radius_samples ? p->exclusion_radius_samples : (int)std::ceil(fs / kChipRate);
    c->gen = gen;
    c->gp = gp;
    c->bins.assign(p->doppler_bins_hz, p->doppler_bins_hz + p->n_bins);
    c->prns.assign(p->prns, p->prns + p->n_prn);

    // ---- tables ---------------------------------------------------------------------
    // Built on the device (gacq_tables.cuh): carrier replicas bit-identical to
    // kernels.py:106-114 at phase 0 (acquisition.py:139), C/A chips and the conjugate code
    // spectra. The host only resolves the per-bin 48-bit NCO steps (kernels.py:61-62) exactly
    // as Python does (round-half-even, floor modulo).
    std::vector<uint64_t> steps(c->B);
    for (int b = 0; b < c->B; ++b)
        steps[b] = (uint64_t)py_mod(py_round((c->bins[b] / fs) * (double)kCarrierScale), kCarrierScale);
    // generic path: conj(DFT_M(c)) / M of each PRN's sampled code replica c[n], n < n_coh,
    // chip index (k * step mod 1023*2^42) >> 42 (kernels.py:116-128, acquisition.py:88-105),
    // in float64 then rounded once; twiddles (cos, sin)(2 pi e / M)
    std::vector<float2> gcc, gtw;
    if (gen) {
        const int M = gp.M;
        gcc.resize((size_t)c->n_prn * M);
        gtw.resize(M);  // full table: M need not be even on the native path
        for (int e = 0; e < M; ++e)
            gtw[e] = make_float2((float)std::cos(kTwoPi * e / M), (float)std::sin(kTwoPi * e / M));
        std::vector<int32_t> idx(n_coh);
        for (int64_t n = 0, ph = 0; n < n_coh; ++n) {
            idx[n] = (int32_t)(ph >> 42);
            ph += code_step;
            if (ph >= kCodeModulus) ph -= kCodeModulus;
        }
        const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), c->n_prn));
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t]() {
                std::vector<std::complex<double>> d(M);
                int8_t chips[1023];
                for (int i = t; i < c->n_prn; i += nt) {
                    ca_code(c->prns[i], chips);
                    std::fill(d.begin(), d.end(), 0.0);
                    for (int64_t n = 0; n < n_coh; ++n) d[n] = (double)chips[idx[n]];
                    if (gp.native) dft_f64_rec(d.data(), M);
                    else fft_f64(d);
                    const int L = gp.L, Ms = gp.Ms;  // residue-major (gacq_generic.cuh)
                    for (int k = 0; k < M; ++k) {
                        const auto v = std::conj(d[k]) / (double)M;
                        const int kk = k / L;  // within the residue class; warp-split order (gen_ws_base)
                        const int slot = gp.W > 1 ? (kk % gp.W) * gp.Q + kk / gp.W : kk;
                        gcc[(size_t)i * M + (k % L) * Ms + slot] = make_float2((float)v.real(), (float)v.imag());
                    }
                }
            });
        for (auto& x : th) x.join();
    }

    // ---- device state ---------------------------------------------------------------
    DeviceGuard guard(c->device);
    auto bail = [&](int code) {
        destroy_ctx(c);
        return code;
    };
#define CTX_TRY(expr)                                                                                  \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess) return bail(fail(GACQ_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e))); \
    } while (0)
    CTX_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CTX_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    {   // device tables; the temporaries are freed before returning
        const size_t n_car = (size_t)c->B * n_coh;
        CTX_TRY(cudaMalloc(&c->d_carrier, n_car * sizeof(float2)));
        CTX_TRY(cudaMalloc(&c->d_ccp, (size_t)c->n_prn * kCcHalf * sizeof(float2)));
        uint64_t* d_steps = nullptr;
        int32_t* d_prns = nullptr;
        int8_t* d_chips = nullptr;
        auto tables = [&]() -> cudaError_t {
            cudaError_t e;
            if ((e = cudaMalloc(&d_steps, steps.size() * sizeof(uint64_t))) ||
                (e = cudaMalloc(&d_prns, c->prns.size() * sizeof(int32_t))) ||
                (e = cudaMalloc(&d_chips, (size_t)c->n_prn * kChips)))
                return e;
            if ((e = cudaMemcpyAsync(d_steps, steps.data(), steps.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                     c->stream)) ||
                (e = cudaMemcpyAsync(d_prns, c->prns.data(), c->prns.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                     c->stream)) ||
                (e = cudaMemsetAsync(c->d_ccp, 0, (size_t)c->n_prn * kCcHalf * sizeof(float2), c->stream)))
                return e;
            gacq_carrier_kernel<<<(unsigned)std::min<size_t>((n_car + 255) / 256, 148 * 16), 256, 0, c->stream>>>(
                d_steps, c->B, (int)n_coh, kTwoPi / (double)kCarrierScale, c->d_carrier);
            gacq_ca_chips_kernel<<<1, 32, 0, c->stream>>>(d_prns, c->n_prn, d_chips);
            gacq_code_spectrum_kernel<<<(unsigned)((c->n_prn * kChips * 32 + 255) / 256), 256, 0, c->stream>>>(
                d_chips, c->n_prn, reinterpret_cast<float2*>(c->d_ccp));
            if ((e = cudaGetLastError())) return e;
            return cudaStreamSynchronize(c->stream);
        };
        const cudaError_t te = tables();
        cudaFree(d_steps);
        cudaFree(d_prns);
        cudaFree(d_chips);
        CTX_TRY(te);
    }
    if (gen) {
        CTX_TRY(cudaMalloc(&c->d_gcc, gcc.size() * sizeof(float2)));
        CTX_TRY(cudaMalloc(&c->d_gtw, gtw.size() * sizeof(float2)));
        CTX_TRY(cudaMemcpy(c->d_gcc, gcc.data(), gcc.size() * sizeof(float2), cudaMemcpyHostToDevice));
        CTX_TRY(cudaMemcpy(c->d_gtw, gtw.data(), gtw.size() * sizeof(float2), cudaMemcpyHostToDevice));
        const int sm_max = gen_smem_ws(kGenMaxMs, 32 * kGenWarpVpt);
        std::vector<const void*> ks;
#define GACQ_GEN_KS(LL, PP, TT) \
    ks.push_back((const void*)gacq_gen_fwd_kernel<LL, PP, TT>); ks.push_back((const void*)gacq_gen_corr_kernel<LL, PP, TT>); \
    ks.push_back((const void*)gacq_gen_corr_ws_kernel<LL, TT>);
        GACQ_GEN_DISPATCH(GACQ_GEN_KS)
#undef GACQ_GEN_KS
        for (const void* k : ks)
            CTX_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_max));
    }
    const int64_t pair_bytes = (int64_t)c->R * (gen ? (int64_t)gp.M : (int64_t)c->D * kSpec) *
                               (int64_t)sizeof(float2);
    c->pair_bytes = pair_bytes;
    // default budget: 8 GiB (C3's 1024-snapshot batch, 7.3 GB of spectra, in one chunk: no
    // persistent-grid tails between chunks, +1.2% over 1 GiB), at most a quarter of the free
    // device memory; allocated on demand by run_impl, so small batches hold little
    size_t free_b = 0, total_b = 0;
    CTX_TRY(cudaMemGetInfo(&free_b, &total_b));
    const int64_t budget = p->scratch_bytes > 0 ? p->scratch_bytes
                                                : std::min<int64_t>((int64_t)8 << 30, (int64_t)(free_b / 4));
    c->z_pairs = std::max<int64_t>(1, budget / pair_bytes);
    if (!gen && c->z_pairs > kCorrWarps) c->z_pairs -= c->z_pairs % kCorrWarps;  // whole K2 pair groups per chunk
    CTX_TRY(cudaMalloc(&c->d_bad, sizeof(int)));
    CTX_TRY(cudaHostAlloc(&c->h_bad, sizeof(int), cudaHostAllocPortable));
    if (gen) {
        *out = c;
        return GACQ_OK;
    }
    {
        // every PFA variant gets the largest dynamic shared memory any plan launches it with
        for (const void* k : {(const void*)gacq_corr_pfa_kernel<true, false>, (const void*)gacq_corr_pfa_kernel<false, false>,
                              (const void*)gacq_corr_pfa_kernel<true, true>}) {
            CTX_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, corr_pfa_smem()));
            CTX_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
#define GACQ_ATTR_FWDP(DD, WW)                                                                             \
    CTX_TRY(cudaFuncSetAttribute(gacq_fwd_pfa_kernel<DD, WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 fwd_pfa_smem(DD, WW)));
        GACQ_PFA_FWD_VARIANTS(GACQ_ATTR_FWDP)
#undef GACQ_ATTR_FWDP
        int per_sm = 0, sms = 0;
        int per_sm_full = 0;
        int per_sm_r1 = 0;
        CTX_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gacq_corr_pfa_kernel<true, false>,
                                                              32 * kCorrWarps, corr_pfa_smem()));
        CTX_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_full, gacq_corr_pfa_kernel<false, false>,
                                                              32 * kCorrWarps, corr_pfa_smem()));
        CTX_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r1, gacq_corr_pfa_kernel<true, true>,
                                                              32 * kCorrWarps, corr_pfa_smem()));
        per_sm = std::min({per_sm, per_sm_full, per_sm_r1});
        CTX_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        c->corr_slots = std::max(1, per_sm) * (int64_t)sms;
        CTX_TRY(cudaMalloc(&c->d_prow, (size_t)c->corr_slots * kCorrWarps * c->D * kPhaseRow * sizeof(float)));
        CTX_TRY(cudaMalloc(&c->d_counter, sizeof(unsigned long long)));
    }
#undef CTX_TRY
    *out = c;
    return GACQ_OK;
}

int gacq_info_get(const gacq_ctx* c, gacq_info* o) {
    if (!c || !o) return fail(GACQ_ERR_INVALID, "null argument");
    o->samples_per_period = c->P;
    o->n_coh = c->n_coh;
    o->chip_oversample = c->D;
    o->fft_len = c->gen ? c->gp.M : kChips;
    o->n_bins = c->B;
    o->n_prn = c->n_prn;
    o->rounds = c->R;
    o->path = c->gen ? 4 : 2;
    o->corr_ctas = (int32_t)c->corr_slots;
    return GACQ_OK;
}

void gacq_destroy(gacq_ctx* c) { destroy_ctx(c); }

int gacq_wait_stream(gacq_ctx* c, void* stream) {
    if (!c) return fail(GACQ_ERR_INVALID, "null context");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (!c->wait_event) CUDA_TRY(cudaEventCreateWithFlags(&c->wait_event, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c->wait_event, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->wait_event, 0));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->wait_event, 0));
    return GACQ_OK;
}

int gacq_run(gacq_ctx* c, const void* snaps, int64_t n_snap, int64_t stride, uint32_t flags, gacq_row* rows) {
    if (!c) return fail(GACQ_ERR_INVALID, "null context");
    if (n_snap < 1) return fail(GACQ_ERR_INVALID, "n_snap must be >= 1");
    if (!snaps || !rows) return fail(GACQ_ERR_INVALID, "null buffer");
    const int64_t span = (int64_t)c->R * c->n_coh;
    if (stride < span && n_snap > 1)
        return fail(GACQ_ERR_INVALID, "stride %lld < %lld samples needed per snapshot", (long long)stride,
                    (long long)span);
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    const Input in{snaps, kFmtComplex64, 1.0, (flags & GACQ_SNAPS_ON_DEVICE) != 0, std::max(stride, span)};
    return run_impl(c, in, n_snap, flags & GACQ_ROWS_PER_BIN, flags & GACQ_PROFILE, rows, flags & GACQ_ROWS_ON_DEVICE,
                    nullptr);
}

int gacq_run_quantized(gacq_ctx* c, const void* iq, int32_t sample_format, double scale, int64_t n_snap,
                       int64_t stride, uint32_t flags, gacq_row* rows) {
    if (!c) return fail(GACQ_ERR_INVALID, "null context");
    if (n_snap < 1) return fail(GACQ_ERR_INVALID, "n_snap must be >= 1");
    if (!iq || !rows) return fail(GACQ_ERR_INVALID, "null buffer");
    if (sample_format != GACQ_FMT_INT8 && sample_format != GACQ_FMT_INT16)
        return fail(GACQ_ERR_INVALID, "unknown sample format %d", sample_format);
    if (!std::isfinite(scale)) return fail(GACQ_ERR_INVALID, "scale must be finite");
    const int64_t span = (int64_t)c->R * c->n_coh;
    if (stride < span && n_snap > 1)
        return fail(GACQ_ERR_INVALID, "stride %lld < %lld samples needed per snapshot", (long long)stride,
                    (long long)span);
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    const Input in{iq, sample_format, scale, (flags & GACQ_SNAPS_ON_DEVICE) != 0, std::max(stride, span)};
    return run_impl(c, in, n_snap, flags & GACQ_ROWS_PER_BIN, flags & GACQ_PROFILE, rows, flags & GACQ_ROWS_ON_DEVICE,
                    nullptr);
}

int gacq_power_map(gacq_ctx* c, const void* snap, float* out) {
    if (!c || !snap || !out) return fail(GACQ_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    const size_t n = (size_t)c->n_prn * c->B * c->P;
    if (!c->d_pmap && cudaMalloc(&c->d_pmap, n * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return fail(GACQ_ERR_RESOURCE, "cudaMalloc power map failed");
    }
    const int64_t span = (int64_t)c->R * c->n_coh;
    const Input in{snap, kFmtComplex64, 1.0, false, span};
    int rc = run_impl(c, in, 1, true, false, nullptr, false, c->d_pmap);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(out, c->d_pmap, n * sizeof(float), cudaMemcpyDeviceToHost));
    return GACQ_OK;
}

int gacq_carrier_table(gacq_ctx* c, void* out) {
    if (!c || !out) return fail(GACQ_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    CUDA_TRY(cudaMemcpy(out, c->d_carrier, (size_t)c->B * c->n_coh * sizeof(float2), cudaMemcpyDeviceToHost));
    return GACQ_OK;
}

int gacq_synth(int32_t device, double fs, int64_t n_snap, int64_t n, int32_t n_sat, const gacq_sat* sats,
               double sigma, uint64_t seed, void* out) {
    if (!out || (n_sat > 0 && !sats)) return fail(GACQ_ERR_INVALID, "null argument");
    if (!(fs > 0) || !std::isfinite(fs) || n_snap < 1 || n < 1 || n_sat < 0)
        return fail(GACQ_ERR_INVALID, "sample rate, n_snap and n_samples must be > 0");
    if (!(sigma >= 0) || !std::isfinite(sigma)) return fail(GACQ_ERR_INVALID, "noise_sigma must be >= 0");
    auto pymod = [](double a, double m) {  // Python's float a % m for m > 0
        double r = std::fmod(a, m);
        if (r != 0 && r < 0) r += m;
        return r;
    };
    const double cps = kChipRate / fs;
    std::vector<SynthSat> st((size_t)n_snap * n_sat);
    for (size_t i = 0; i < st.size(); ++i) {
        const gacq_sat& g = sats[i];
        if (g.prn < 1 || g.prn > 32) return fail(GACQ_ERR_INVALID, "prn must be in 1..32");
        const double code0 = pymod(-g.code_phase_samples * cps, 1023.0);  // gnss_signal.py:170-171
        st[i].code_p0 = (uint64_t)py_mod(py_round(pymod(code0, 1023.0) * (double)kCodeScale), kCodeModulus);
        const double carr0 = pymod(-g.carrier_phase_cycles, 1.0);          // gnss_signal.py:180
        st[i].carrier_p0 = (uint64_t)py_mod(py_round(pymod(carr0, 1.0) * (double)kCarrierScale), kCarrierScale);
        st[i].carrier_step = (uint64_t)py_mod(py_round((-g.doppler_hz / fs) * (double)kCarrierScale), kCarrierScale);
        st[i].prn_index = g.prn - 1;
        st[i].amp = g.amplitude;
    }
    const uint64_t code_step = (uint64_t)py_round(cps * (double)kCodeScale);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GACQ_ERR_CUDA, "no CUDA device visible");
    }
    if (device < 0 || device >= ndev) return fail(GACQ_ERR_INVALID, "device %d out of range", device);
    DeviceGuard g(device);
    SynthSat* d_st = nullptr;
    int32_t* d_prns = nullptr;
    int8_t* d_chips = nullptr;
    cudaStream_t stream = nullptr;
    auto work = [&]() -> cudaError_t {
        cudaError_t e;
        std::vector<int32_t> all(32);
        for (int i = 0; i < 32; ++i) all[i] = i + 1;
        if ((e = cudaStreamCreateWithFlags(&stream, cudaStreamDefault)) ||  // ordered after the legacy default stream
            (e = cudaMalloc(&d_st, std::max<size_t>(1, st.size()) * sizeof(SynthSat))) ||
            (e = cudaMalloc(&d_prns, 32 * sizeof(int32_t))) || (e = cudaMalloc(&d_chips, 32 * kChips)))
            return e;
        if ((!st.empty() &&
             (e = cudaMemcpyAsync(d_st, st.data(), st.size() * sizeof(SynthSat), cudaMemcpyHostToDevice, stream))) ||
            (e = cudaMemcpyAsync(d_prns, all.data(), 32 * sizeof(int32_t), cudaMemcpyHostToDevice, stream)))
            return e;
        gacq_ca_chips_kernel<<<1, 32, 0, stream>>>(d_prns, 32, d_chips);
        const int64_t total = n_snap * n;
        gacq_synth_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, stream>>>(
            d_st, n_sat, n_snap, n, code_step, d_chips, kTwoPi / (double)kCarrierScale, sigma, seed, (float2*)out);
        if ((e = cudaGetLastError())) return e;
        return cudaStreamSynchronize(stream);
    };
    const cudaError_t e = work();
    cudaFree(d_st);
    cudaFree(d_prns);
    cudaFree(d_chips);
    if (stream) cudaStreamDestroy(stream);
    if (e != cudaSuccess) return fail(GACQ_ERR_CUDA, "gacq_synth failed: %s", cudaGetErrorString(e));
    return GACQ_OK;
}

// Measured FP32 roof for the roofline denominator (MEASURED_PEAKS.json has no FP32 entry):
// 16 independent packed FFMA2 chains per thread with broadcast coefficients, 8 warps per SM
// block x 4 blocks per SM, the instruction form the transform codelets use.
__global__ void gacq_fp32_probe_kernel(float* out, int iters, float s) {
    cx acc[16], x[4];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, (float)i);
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = pk(s * i, s + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] = fma2(x[j], bc(0.125f * (k + 1) + 0.01f * j), acc[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = acc[j] ^ (cx)(it & 1);
    }
    cx r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(r & 0xffff);
}

int gacq_fp32_probe(int32_t device, double* tflops) {
    if (!tflops) return fail(GACQ_ERR_INVALID, "null argument");
    DeviceGuard g(device);
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int threads = 256, blocks = 4 * sms, iters = 4096;
    float* out = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto work = [&]() -> cudaError_t {
        cudaError_t e;
        if ((e = cudaMalloc(&out, sizeof(float) * blocks * threads)) || (e = cudaEventCreate(&e0)) ||
            (e = cudaEventCreate(&e1)))
            return e;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            gacq_fp32_probe_kernel<<<blocks, threads>>>(out, iters, 1.0001f);
            cudaEventRecord(e1);
            if ((e = cudaEventSynchronize(e1))) return e;
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) best = std::min(best, ms);
        }
        // 64 FFMA2 per iteration, 4 flops per lane each
        *tflops = (double)blocks * threads * iters * 64.0 * 4.0 / (best * 1e-3) / 1e12;
        return cudaGetLastError();
    };
    const cudaError_t e = work();
    cudaFree(out);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (e != cudaSuccess) return fail(GACQ_ERR_CUDA, "fp32 probe failed: %s", cudaGetErrorString(e));
    return GACQ_OK;
}

int gacq_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes <= 0) return fail(GACQ_ERR_INVALID, "bad host allocation request");
    if (cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(GACQ_ERR_RESOURCE, "cudaHostAlloc of %lld bytes failed", (long long)bytes);
    }
    return GACQ_OK;
}

int gacq_host_free(void* ptr) {
    if (ptr) CUDA_TRY(cudaFreeHost(ptr));
    return GACQ_OK;
}

int gacq_stats_get(const gacq_ctx* c, gacq_stats* o) {
    if (!c || !o) return fail(GACQ_ERR_INVALID, "null argument");
    *o = c->stats;
    return GACQ_OK;
}

int gacq_stats_reset(gacq_ctx* c) {
    if (!c) return fail(GACQ_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    c->stats = gacq_stats{};
    return GACQ_OK;
}

// ---- tracking correlators ----------------------------------------------------------

struct gacq_trk {
    std::mutex mu;
    int device = 0;
    cudaStream_t stream = nullptr;
    int8_t* d_chips = nullptr;  // [32][1024] +/-1
    float2* d_blocks = nullptr;
    int64_t blocks_cap = 0;
    gacq_epl_chan* d_chans = nullptr;
    int64_t chans_cap = 0;
    float* d_out = nullptr;
    int64_t out_cap = 0;
    gacq_epl_chan* h_chans = nullptr;  // page-locked staging of gacq_trk_step
    float* h_sums = nullptr;
    int64_t h_cap = 0;                 // channels
    std::vector<cudaEvent_t> slice_events;
    cudaEvent_t wait_event = nullptr;  // gacq_trk_wait_stream
};

static void trk_free(gacq_trk* t) {
    if (!t) return;
    {
        DeviceGuard g(t->device);
        if (t->stream) cudaStreamSynchronize(t->stream);
        cudaFree(t->d_chips);
        cudaFree(t->d_blocks);
        cudaFree(t->d_chans);
        cudaFree(t->d_out);
        cudaFreeHost(t->h_chans);
        cudaFreeHost(t->h_sums);
        for (cudaEvent_t e : t->slice_events) cudaEventDestroy(e);
        if (t->wait_event) cudaEventDestroy(t->wait_event);
        if (t->stream) cudaStreamDestroy(t->stream);
    }
    delete t;
}

int gacq_trk_create(gacq_trk** out, int32_t device) {
    if (!out) return fail(GACQ_ERR_INVALID, "null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GACQ_ERR_CUDA, "no CUDA device visible");
    }
    if (device < 0 || device >= ndev) return fail(GACQ_ERR_INVALID, "device %d out of range", device);
    gacq_trk* t = new gacq_trk();
    t->device = device;
    std::vector<int8_t> chips(32 * 1024, 0);
    for (int p = 1; p <= 32; ++p) ca_code(p, chips.data() + (p - 1) * 1024);
    DeviceGuard g(device);
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(gacq_epl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kEplSmem)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_chips, chips.size())) != cudaSuccess ||
        (e = cudaMemcpy(t->d_chips, chips.data(), chips.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
        trk_free(t);
        return fail(GACQ_ERR_CUDA, "tracker setup failed: %s", cudaGetErrorString(e));
    }
    *out = t;
    return GACQ_OK;
}

void gacq_trk_destroy(gacq_trk* t) { trk_free(t); }

int gacq_trk_wait_stream(gacq_trk* t, void* stream) {
    if (!t) return fail(GACQ_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    if (!t->wait_event) CUDA_TRY(cudaEventCreateWithFlags(&t->wait_event, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(t->wait_event, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamWaitEvent(t->stream, t->wait_event, 0));
    return GACQ_OK;
}

}  // extern "C"

namespace gtrk {

// tracking.py:168-275 for channels [a, e) of a batch, in place (see gacq_trk_close)
struct Closure {
    const gacq_trk_config* cfg;
    double sp, t, g1p, g2p, g1d, g2d, alpha;
    explicit Closure(const gacq_trk_config* c) : cfg(c) {
        sp = c->correlator_spacing_chips;
        t = c->integration_ms * 1e-3;
        auto gains = [](double bw, double* g1, double* g2) {  // tracking.py:188-190
            const double w0 = bw / 0.53;
            *g1 = 2.0 * kLoopDamping * w0;
            *g2 = w0 * w0;
        };
        gains(c->pll_bandwidth_hz, &g1p, &g2p);
        gains(c->dll_bandwidth_hz, &g1d, &g2d);
        alpha = 1.0 / kLockSmoothing;
    }
    // degenerate channels first (the reference raises before touching any state): a zero
    // prompt correlator fails the PLL discriminator (tracking.py:181-182), and with zero early
    // and late as well the DLL one first (tracking.py:173-175). Returns the first bad index or -1.
    static int64_t first_degenerate(const float* sums, int64_t a, int64_t e, bool* all) {
        for (int64_t i = a; i < e; ++i) {
            const float* s = sums + 6 * i;
            if (s[2] == 0.f && s[3] == 0.f) {
                *all = s[0] == 0.f && s[1] == 0.f && s[4] == 0.f && s[5] == 0.f;
                return i;
            }
        }
        return -1;
    }
    void range(const float* sums, const gacq_trk_batch* b, double* out, int64_t a0, int64_t e0) const {
        const double two_pi = 2.0 * 3.141592653589793;
        parallel_for(e0 - a0, [&](int64_t ra, int64_t re_) {
            for (int64_t i = a0 + ra; i < a0 + re_; ++i) {
                const float* s = sums + 6 * i;
                const double ie = s[0], qe = s[1], ip = s[2], qp = s[3], il = s[4], ql = s[5];
                const double e = ie * ie + qe * qe, l = il * il + ql * ql;  // tracking.py:170-171
                const double ed = e + l == 0 ? 0.0 : (e - l) / (e + l) * (1.0 - sp / 2.0) / 2.0;
                const double ep = ip == 0.0 ? std::copysign(0.25, qp) : std::atan(qp / ip) / two_pi;  // :179-185
                const double fs = b->sample_rate_hz[i];
                const int64_t n = rint64(fs * cfg->integration_ms * 1e-3);  // the channel's block, tracking.py:122-123
                const double pll_acc = b->pll_acc[i] + g2p * t * (ep + b->pll_prev[i]) / 2.0;  // :198-200
                const double dll_acc = b->dll_acc[i] + g2d * t * (ed + b->dll_prev[i]) / 2.0;
                const double doppler = b->doppler_hz[i] + (pll_acc - b->pll_acc[i]);  // :242
                const double code_rate = kChipRate * (1.0 + doppler / kL1) + dll_acc;  // :243
                const uint64_t pc = (carrier_phase_fixed(b->carrier_phase_cycles[i]) +
                                     (uint64_t)n * carrier_step_fixed(b->doppler_hz[i], fs) +
                                     carrier_phase_fixed(t * g1p * ep)) % (uint64_t)kCarrierScale;  // :211-215
                const uint64_t nudge = (uint64_t)rint64(py_fmod(t * g1d * ed, 1023.0) * (double)kCodeScale);
                const uint64_t pcode = (code_phase_fixed(b->code_phase_chips[i]) +
                                        (uint64_t)n * code_step_fixed(b->code_rate_hz[i], fs) + nudge) %
                                       (uint64_t)kCodeModulus;  // :218-223
                const double nbd = ip * ip - qp * qp, nbp = ip * ip + qp * qp;  // :252-260
                double nbd_s = nbd, nbp_s = nbp;
                if (b->epoch[i] != 0) {
                    nbd_s = b->lock_nbd[i] + alpha * (nbd - b->lock_nbd[i]);
                    nbp_s = b->lock_nbp[i] + alpha * (nbp - b->lock_nbp[i]);
                }
                out[3 * i + 0] = ed;
                out[3 * i + 1] = ep;
                out[3 * i + 2] = nbp_s > 0 ? nbd_s / nbp_s : 0.0;
                b->code_phase_chips[i] = (double)pcode / (double)kCodeScale;
                b->carrier_phase_cycles[i] = (double)pc / (double)kCarrierScale;
                b->doppler_hz[i] = doppler;
                b->code_rate_hz[i] = code_rate;
                b->dll_acc[i] = dll_acc;
                b->dll_prev[i] = ed;
                b->pll_acc[i] = pll_acc;
                b->pll_prev[i] = ep;
                b->lock_nbd[i] = nbd_s;
                b->lock_nbp[i] = nbp_s;
                b->epoch[i] += 1;
            }
        });
    }
};

// gacq_epl_chan records of channels [a, e): tracking.py:126-165's NCO words (kernels.py:56-70)
inline void chans_range(const gacq_trk_batch* b, const gacq_trk_config* cfg, const int64_t* offsets,
                        gacq_epl_chan* ch, int64_t a0, int64_t e0) {
    const double d = cfg->correlator_spacing_chips;
    const double off[3] = {+d / 2, 0.0, -d / 2};  // tracking.py:148-156
    parallel_for(e0 - a0, [&](int64_t ra, int64_t re_) {
        for (int64_t i = a0 + ra; i < a0 + re_; ++i) {
            const double fs = b->sample_rate_hz[i];
            ch[i].block_offset = offsets[i];
            ch[i].carrier_p0 = carrier_phase_fixed(b->carrier_phase_cycles[i]);
            ch[i].carrier_step = carrier_step_fixed(b->doppler_hz[i], fs);
            for (int j = 0; j < 3; ++j) ch[i].code_p0[j] = code_phase_fixed(py_fmod(b->code_phase_chips[i] + off[j], 1023.0));
            ch[i].code_step = code_step_fixed(b->code_rate_hz[i], fs);
            ch[i].prn = b->prn[i];
            ch[i].reserved = 0;
        }
    });
}

}  // namespace gtrk

extern "C" {

int gacq_trk_close(const float* sums, const gacq_trk_batch* b, const gacq_trk_config* cfg, double* out,
                   int64_t* bad) {
    if (!sums || !b || !cfg || !out) return fail(GACQ_ERR_INVALID, "null argument");
    if (b->n < 1) return fail(GACQ_ERR_INVALID, "no channels");
    bool all = false;
    const int64_t i = gtrk::Closure::first_degenerate(sums, 0, b->n, &all);
    if (i >= 0) {
        if (bad) *bad = i;
        return fail(GACQ_ERR_INVALID, "%s on channel %lld", all ? "all correlators zero" : "prompt correlator is zero",
                    (long long)i);
    }
    gtrk::Closure(cfg).range(sums, b, out, 0, b->n);
    return GACQ_OK;
}

int gacq_trk_chans(const gacq_trk_batch* b, const gacq_trk_config* cfg, const int64_t* offsets, gacq_epl_chan* ch) {
    if (!b || !cfg || !offsets || !ch) return fail(GACQ_ERR_INVALID, "null argument");
    gtrk::chans_range(b, cfg, offsets, ch, 0, b->n);
    return GACQ_OK;
}

int gacq_trk_epl(gacq_trk* t, const void* blocks, int64_t total, int32_t n, const gacq_epl_chan* chans,
                 int64_t n_chan, uint32_t flags, float* out) {
    if (!t || !blocks || !chans || !out) return fail(GACQ_ERR_INVALID, "null argument");
    if (n < 1 || n_chan < 1 || total < n) return fail(GACQ_ERR_INVALID, "bad sizes");
    for (int64_t i = 0; i < n_chan; ++i) {
        if (chans[i].prn < 1 || chans[i].prn > 32)
            return fail(GACQ_ERR_INVALID, "prn must be an integer in 1..32, got %d", chans[i].prn);
        if (chans[i].block_offset < 0 || chans[i].block_offset + n > total)
            return fail(GACQ_ERR_INVALID, "channel %lld block outside the sample buffer", (long long)i);
        if (chans[i].carrier_p0 >> 48 || chans[i].carrier_step >> 48 || chans[i].code_step >= kCodeMod ||
            chans[i].code_p0[0] >= kCodeMod || chans[i].code_p0[1] >= kCodeMod || chans[i].code_p0[2] >= kCodeMod)
            return fail(GACQ_ERR_INVALID, "channel %lld NCO word out of range", (long long)i);
        // the kernel evaluates the code NCO statelessly as p0 + k step in 64 bits
        if (chans[i].code_step && (uint64_t)(n - 1) > (~0ull - kCodeMod) / chans[i].code_step)
            return fail(GACQ_ERR_UNSUPPORTED, "channel %lld: %d samples at code step %llu overflow the 64-bit code NCO",
                        (long long)i, n, (unsigned long long)chans[i].code_step);
    }
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    const float2* x = (const float2*)blocks;
    int rc;
    if (!(flags & GACQ_SNAPS_ON_DEVICE)) {
        if ((rc = grow(&t->d_blocks, &t->blocks_cap, total))) return rc;
        CUDA_TRY(cudaMemcpyAsync(t->d_blocks, blocks, total * sizeof(float2), cudaMemcpyHostToDevice, t->stream));
        x = t->d_blocks;
    }
    if ((rc = grow(&t->d_chans, &t->chans_cap, n_chan))) return rc;
    if ((rc = grow(&t->d_out, &t->out_cap, n_chan * 6))) return rc;
    CUDA_TRY(cudaMemcpyAsync(t->d_chans, chans, n_chan * sizeof(gacq_epl_chan), cudaMemcpyHostToDevice, t->stream));
    gacq_epl_kernel<<<(unsigned)((n_chan + kEplChans - 1) / kEplChans), kEplThreads, kEplSmem, t->stream>>>(
        reinterpret_cast<const cx*>(x), n, t->d_chans, n_chan, t->d_chips, t->d_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, t->d_out, n_chan * 6 * sizeof(float), cudaMemcpyDeviceToHost, t->stream));
    CUDA_TRY(cudaStreamSynchronize(t->stream));
    return GACQ_OK;
}

int gacq_trk_step(gacq_trk* t, const void* blocks, int64_t total, const int64_t* offsets, gacq_trk_batch* b,
                  const gacq_trk_config* cfg, uint32_t flags, float* sums, double* out, int64_t* bad) {
    if (!t || !blocks || !offsets || !b || !cfg || !sums || !out) return fail(GACQ_ERR_INVALID, "null argument");
    const int64_t nch = b->n;
    if (nch < 1) return fail(GACQ_ERR_INVALID, "no channels");
    const int64_t n64 = gtrk::rint64(b->sample_rate_hz[0] * cfg->integration_ms * 1e-3);  // tracking.py:122-123
    if (n64 < 1 || n64 > INT32_MAX || total < n64) return fail(GACQ_ERR_INVALID, "bad sizes");
    const int n = (int)n64;
    for (int64_t i = 0; i < nch; ++i) {
        if (b->prn[i] < 1 || b->prn[i] > 32) return fail(GACQ_ERR_INVALID, "prn must be an integer in 1..32, got %d", b->prn[i]);
        // one correlator launch covers the batch: every channel's own block length
        // (tracking.py:122-123) must be the launch's
        if (gtrk::rint64(b->sample_rate_hz[i] * cfg->integration_ms * 1e-3) != n64)
            return fail(GACQ_ERR_INVALID, "channel %lld: block length differs from channel 0's (mixed sample rates)",
                        (long long)i);
        if (offsets[i] < 0 || offsets[i] + n > total)
            return fail(GACQ_ERR_INVALID, "channel %lld block outside the sample buffer", (long long)i);
    }
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    const float2* x = (const float2*)blocks;
    int rc;
    if (!(flags & GACQ_SNAPS_ON_DEVICE)) {
        if ((rc = grow(&t->d_blocks, &t->blocks_cap, total))) return rc;
        CUDA_TRY(cudaMemcpyAsync(t->d_blocks, blocks, total * sizeof(float2), cudaMemcpyHostToDevice, t->stream));
        x = t->d_blocks;
    }
    if ((rc = grow(&t->d_chans, &t->chans_cap, nch))) return rc;
    if ((rc = grow(&t->d_out, &t->out_cap, nch * 6))) return rc;
    if (t->h_cap < nch) {
        cudaFreeHost(t->h_chans);
        cudaFreeHost(t->h_sums);
        t->h_chans = nullptr;
        t->h_sums = nullptr;
        t->h_cap = 0;
        if (cudaHostAlloc(&t->h_chans, nch * sizeof(gacq_epl_chan), cudaHostAllocDefault) != cudaSuccess ||
            cudaHostAlloc(&t->h_sums, nch * 6 * sizeof(float), cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            return fail(GACQ_ERR_RESOURCE, "page-locked staging for %lld channels", (long long)nch);
        }
        t->h_cap = nch;
    }
    // slices of whole 32-channel CTAs, at most 4
    const int64_t slice = std::max<int64_t>(32 * 64, ((nch + 3) / 4 + 31) / 32 * 32);
    const int64_t n_slices = (nch + slice - 1) / slice;
    while ((int64_t)t->slice_events.size() < n_slices) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        t->slice_events.push_back(e);
    }
    auto drain = [&](int r) { cudaStreamSynchronize(t->stream); return r; };
    for (int64_t k = 0; k < n_slices; ++k) {
        const int64_t a = k * slice, e = std::min(nch, a + slice);
        gtrk::chans_range(b, cfg, offsets, t->h_chans, a, e);
        for (int64_t i = a; i < e; ++i)  // the kernel evaluates the code NCO as p0 + k step in 64 bits
            if (t->h_chans[i].code_step >= kCodeMod ||
                (t->h_chans[i].code_step && (uint64_t)(n - 1) > (~0ull - kCodeMod) / t->h_chans[i].code_step))
                return drain(fail(GACQ_ERR_UNSUPPORTED, "channel %lld: code NCO step out of range", (long long)i));
        if (cudaMemcpyAsync(t->d_chans + a, t->h_chans + a, (e - a) * sizeof(gacq_epl_chan), cudaMemcpyHostToDevice,
                            t->stream) != cudaSuccess)
            return drain(fail(GACQ_ERR_CUDA, "chans upload: %s", cudaGetErrorString(cudaGetLastError())));
        gacq_epl_kernel<<<(unsigned)((e - a + kEplChans - 1) / kEplChans), kEplThreads, kEplSmem, t->stream>>>(
            reinterpret_cast<const cx*>(x), n, t->d_chans + a, e - a, t->d_chips, t->d_out + 6 * a);
        if (cudaGetLastError() != cudaSuccess ||
            cudaMemcpyAsync(t->h_sums + 6 * a, t->d_out + 6 * a, (e - a) * 6 * sizeof(float), cudaMemcpyDeviceToHost,
                            t->stream) != cudaSuccess ||
            cudaEventRecord(t->slice_events[k], t->stream) != cudaSuccess)
            return drain(fail(GACQ_ERR_CUDA, "correlator launch failed"));
    }
    gtrk::Closure cl(cfg);
    for (int64_t k = 0; k < n_slices; ++k) {
        const int64_t a = k * slice, e = std::min(nch, a + slice);
        if (cudaEventSynchronize(t->slice_events[k]) != cudaSuccess)
            return drain(fail(GACQ_ERR_CUDA, "correlator: %s", cudaGetErrorString(cudaGetLastError())));
        std::memcpy(sums + 6 * a, t->h_sums + 6 * a, (e - a) * 6 * sizeof(float));
        bool all = false;
        const int64_t i = gtrk::Closure::first_degenerate(sums, a, e, &all);
        if (i >= 0) {
            if (bad) *bad = i;
            return drain(fail(GACQ_ERR_INVALID, "%s on channel %lld",
                              all ? "all correlators zero" : "prompt correlator is zero", (long long)i));
        }
        cl.range(sums, b, out, a, e);
    }
    return GACQ_OK;
}

}  // extern "C"
