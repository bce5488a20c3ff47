// pfa.cuh -- odd-length DFT codelets for the 1023 = 31 x 33 prime-factor transform.
//
// The chip-domain correlation of the acquisition path is circular over 1023 chips. It is
// evaluated as  IDFT_1023( DFT_1023(z) * conj(DFT_1023(chip)) ), with no zero padding.
// 1023 = 31 * 33 is coprime, so Good-Thomas gives a two-stage transform with no twiddles:
//   input  index n = (33 n1 + 31 n2) mod 1023
//   output index k = (528 k1 + 496 k2) mod 1023   (k = k1 mod 31, k = k2 mod 33)
//   X[k1][k2] = sum_n2 W33^(n2 k2) sum_n1 W31^(n1 k1) x[n1][n2].
// The 33-point stage is itself 3 x 11 Good-Thomas, in registers. All odd-length DFTs use the
// real-symmetric split, which maps every twiddle product onto one packed FFMA2:
//   a_j = x_j + x_(p-j), b_j = x_j - x_(p-j), j = 1..h, h = (p-1)/2
//   X_0 = x_0 + sum a_j
//   A_k = x_0 + sum_j a_j cos(2 pi jk/p),  B_k = sum_j b_j sin(2 pi jk/p)
//   X_k = A_k + S i B_k,  X_(p-k) = A_k - S i B_k.
// S = -1 forward, +1 inverse (unnormalised), as in codelets.cuh.
#pragma once
#include "codelets.cuh"
#include "pfa_tables.cuh"

namespace gacq {

template <int P>
__device__ __forceinline__ float tcos(int m) {
    static_assert(P == 3 || P == 11 || P == 31, "no table");
    return P == 3 ? kCos3[m] : P == 11 ? kCos11[m] : kCos31[m];
}
template <int P>
__device__ __forceinline__ float tsin(int m) {
    static_assert(P == 3 || P == 11 || P == 31, "no table");
    return P == 3 ? kSin3[m] : P == 11 ? kSin11[m] : kSin31[m];
}

// P-point DFT of x (destroyed); emit(k, X_k) once for every k < P. KB output pairs are
// accumulated together (2 KB independent FFMA2 chains).
template <int S, int P, int KB, typename Emit>
__device__ __forceinline__ void dft_odd(cx (&x)[P], Emit&& emit) {
    constexpr int H = (P - 1) / 2;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
        const cx a = add2(x[j], x[P - j]), b = sub2(x[j], x[P - j]);
        x[j] = a;
        x[P - j] = b;
    }
    {
        cx s0 = x[0], s1 = czero();
#pragma unroll
        for (int j = 1; j <= H; ++j) (j & 1 ? s1 : s0) = add2(j & 1 ? s1 : s0, x[j]);
        emit(0, add2(s0, s1));
    }
#pragma unroll
    for (int k0 = 1; k0 <= H; k0 += KB) {
        cx A[KB], B[KB];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
            const int k = k0 + kk;
            if (k > H) continue;
            A[kk] = fma2(x[1], bc(tcos<P>(k % P)), x[0]);
            B[kk] = x[P - 1];  // B_k / sin(2 pi k/P): b_1's coefficient is 1
        }
#pragma unroll
        for (int j = 2; j <= H; ++j)
#pragma unroll
            for (int kk = 0; kk < KB; ++kk) {
                const int k = k0 + kk;
                if (k > H) continue;
                A[kk] = fma2(x[j], bc(tcos<P>((j * k) % P)), A[kk]);
                B[kk] = fma2(x[P - j], bc(tsin<P>((j * k) % P) / tsin<P>(k % P)), B[kk]);
            }
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
            const int k = k0 + kk;
            if (k > H) continue;
            // X_k, X_(P-k) = A_k +- S i sin(2 pi k/P) B'_k: the sine folds into the output FFMA2s
            const cx r = rot<S>(B[kk]);
            emit(k, fma2(r, bc(tsin<P>(k % P)), A[kk]));
            emit(P - k, fma2(r, bc(-tsin<P>(k % P)), A[kk]));
        }
    }
}

// Same transform for P = 31 with the inputs streamed: each input pair (j, 31-j) is folded into
// all 15 (A_k, B_k) accumulators as it arrives, so only two pairs are live beside the 60
// accumulator registers (the unstreamed form keeps all 31 inputs and all 30 accumulators live
// at once). load(j, dep) must return input j and make its address depend on `dep`, which is
// always 0 but carries the accumulators of step j-2: the scheduler then cannot hoist all loads
// to the top, and each pair's load still overlaps one step of FFMA2s. `zero` must be a runtime
// 0 the compiler cannot see through (a kernel argument).
template <int S, typename Load, typename Emit>
__device__ __forceinline__ void dft31_stream(Load&& load, int zero, Emit&& emit) {
    constexpr int P = 31, H = 15;
    const cx x0 = load(0, 0);
    cx A[H], B[H], s0 = x0, s1 = czero();
    cx nj = load(1, 0), nm = load(P - 1, 0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
        const cx xj = nj, xm = nm;
        if (j < H) {
            const int dep = j == 1 ? 0 : (int)(B[H - 1] >> 32) & zero;
            nj = load(j + 1, dep);
            nm = load(P - j - 1, dep);
        }
        const cx a = add2(xj, xm), b = sub2(xj, xm);
        (j & 1 ? s1 : s0) = add2(j & 1 ? s1 : s0, a);
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            A[k - 1] = fma2(a, bc(tcos<P>((j * k) % P)), j == 1 ? x0 : A[k - 1]);
            B[k - 1] = j == 1 ? mul2(b, bc(tsin<P>(k % P))) : fma2(b, bc(tsin<P>((j * k) % P)), B[k - 1]);
        }
    }
    emit(0, add2(s0, s1));
#pragma unroll
    for (int k = 1; k <= H; ++k) {
        const cx r = rot<S>(B[k - 1]);
        emit(k, add2(A[k - 1], r));
        emit(P - k, sub2(A[k - 1], r));
    }
}

// 3-point DFT in place, X1/X2 = A +- S i (sqrt3/2) d as two FFMA2 (ptxas folds the swap/negate
// of rot<S> into the FFMA2 operand): 6 packed instructions instead of dft_odd<S, 3>'s 7
template <int S>
__device__ __forceinline__ void dft3_fma(cx (&t)[3]) {
    const cx s = add2(t[1], t[2]), d = sub2(t[1], t[2]);
    const cx A = fma2(s, bc(-0.5f), t[0]), r = rot<S>(d);
    t[0] = add2(t[0], s);
    t[1] = fma2(r, bc(0.8660254037844386f), A);
    t[2] = fma2(r, bc(-0.8660254037844386f), A);
}

// 33-point DFT, 3 x 11 Good-Thomas: n = (11 a + 3 b) mod 33, k = (22 c + 12 e) mod 33.
template <int S, typename Emit>
__device__ __forceinline__ void dft33(cx (&x)[33], Emit&& emit) {
    cx y[3][11];
#pragma unroll
    for (int b = 0; b < 11; ++b) {
        cx t[3] = {x[(3 * b) % 33], x[(11 + 3 * b) % 33], x[(22 + 3 * b) % 33]};
        dft3_fma<S>(t);
#pragma unroll
        for (int c = 0; c < 3; ++c) y[c][b] = t[c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) dft_odd<S, 11, 5>(y[c], [&](int e, cx v) { emit((22 * c + 12 * e) % 33, v); });
}

// dft33 with its inputs loaded through load(k, dep): GACQ_DFT33_AHEAD triples are requested before
// the 3-point layer starts (11 = all 33 at once, measured fastest: the shared-memory latency is
// paid once per transform), later triples' addresses depend on the previous layer output (`dep`,
// a runtime 0) so the compiler keeps the requested window. consumed() runs once every input has
// been used (after the 3-point layer), then the 11-point layers emit the outputs.
template <int S, typename Load, typename Consumed, typename Emit>
__device__ __forceinline__ void dft33_stream(Load&& load, int zero, Consumed&& consumed, Emit&& emit) {
#ifndef GACQ_DFT33_AHEAD
#define GACQ_DFT33_AHEAD 11
#endif
    constexpr int AH = GACQ_DFT33_AHEAD;
    cx y[3][11];
    cx n[AH][3];
#pragma unroll
    for (int a = 0; a < AH; ++a) {
        n[a][0] = load((3 * a) % 33, 0);
        n[a][1] = load((11 + 3 * a) % 33, 0);
        n[a][2] = load((22 + 3 * a) % 33, 0);
    }
#pragma unroll
    for (int b = 0; b < 11; ++b) {
        cx t[3] = {n[b % AH][0], n[b % AH][1], n[b % AH][2]};
        if (b + AH < 11) {
            const int bn = b + AH;
            const int dep = b == 0 ? 0 : (int)(y[2][b - 1] >> 32) & zero;
            n[b % AH][0] = load((3 * bn) % 33, dep);
            n[b % AH][1] = load((11 + 3 * bn) % 33, dep);
            n[b % AH][2] = load((22 + 3 * bn) % 33, dep);
        }
        dft3_fma<S>(t);
#pragma unroll
        for (int c = 0; c < 3; ++c) y[c][b] = t[c];
    }
    consumed();
#pragma unroll
    for (int c = 0; c < 3; ++c) dft_odd<S, 11, 5>(y[c], [&](int e, cx v) { emit((22 * c + 12 * e) % 33, v); });
}

// One 31-point DFT spread over a warp: lane L < 31 holds x_L. Used for the 33rd row of the
// 31-point stage so that the 33 rows run on 32 lanes without a second pass.
//   lanes 1..15 accumulate A_k (k = L), lane 16 X_0, lanes 17..31 B_k (k = L - 16);
//   lane k then owns X_k and X_(31-k), lane 16 owns X_0.
// `coef(j)` (j = 1..15) is the lane's column, coop31_coef(lane, j); `scr` is 33 cx of warp
// scratch.
__device__ __forceinline__ float coop31_coef(int lane, int j) {
    if (lane >= 1 && lane <= 15) return kCos31[(j * lane) % 31];
    if (lane == 16) return 1.f;
    if (lane >= 17) return kSin31[(j * (lane - 16)) % 31];
    return 0.f;
}

template <int S, typename Coef, typename Emit>
__device__ __forceinline__ void coop31(cx x, int lane, Coef&& coef, cx* scr, Emit&& emit) {
    const cx o = __shfl_sync(0xffffffffu, x, (31 - lane) & 31);
    __syncwarp();  // the previous call's readers are done with scr
    if (lane == 0) scr[0] = x;
    if (lane >= 1 && lane <= 15) {
        scr[lane] = add2(x, o);       // a_j at j
        scr[17 + lane] = sub2(x, o);  // b_j at 17 + j (distinct bank from a_j)
    }
    __syncwarp();
    const int off = lane >= 17 ? 17 : 0;
#ifndef GACQ_COOP_CHAINS
#define GACQ_COOP_CHAINS 1
#endif
    // GACQ_COOP_CHAINS independent accumulation chains (shorter dependent FFMA2 chains)
    constexpr int NC = GACQ_COOP_CHAINS;
    cx part[NC];
    part[0] = lane >= 17 ? czero() : scr[0];
#pragma unroll
    for (int c = 1; c < NC; ++c) part[c] = czero();
#pragma unroll
    for (int j = 1; j <= 15; ++j) part[(j - 1) % NC] = fma2(scr[off + j], bc(coef(j)), part[(j - 1) % NC]);
#pragma unroll
    for (int c = 1; c < NC; ++c) part[0] = add2(part[0], part[c]);
    const cx acc = part[0];
    const cx bk = __shfl_sync(0xffffffffu, acc, (lane + 16) & 31);
    if (lane >= 1 && lane <= 15) {
        const cx r = rot<S>(bk);
        emit(0, lane, add2(acc, r));
        emit(1, 31 - lane, sub2(acc, r));
    } else if (lane == 16) {
        emit(0, 0, acc);
    }
}

}  // namespace gacq
