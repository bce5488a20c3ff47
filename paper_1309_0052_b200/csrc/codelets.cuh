// codelets.cuh -- in-register complex DFT codelets (radix 4/8/16) for sm_100a on packed
// FP32x2 arithmetic (PTX add/sub/mul/fma .f32x2 -> SASS FADD2/FMUL2/FFMA2).
//
// A complex value lives in one 64-bit register pair (cx = re | im << 32). On B200 the
// packed instructions run at the same FP32 rate as scalar FFMA (measured: 67.7 vs 67.9
// TFLOP/s, tools/fp32x2_probe.cu) but take half the issue slots, so the butterflies no
// longer compete with the shared-memory exchanges for issue. ptxas folds the operand
// forms used here into single instructions:
//   a +- i*b   -> FADD2 a, (-)b.LO_HI.NP        (swap + partial negate)
//   a * w      -> FMUL2 a, w.re(bcast) ; FFMA2 -a.LO_HI.NP, w.im(bcast), t
//   a * const  -> FMUL2 a, imm
//
// S = -1: forward transform, kernel exp(-2 pi i nk/N)  (scipy.fft.fft, dsp.py:108-112)
// S = +1: inverse direction, kernel exp(+2 pi i nk/N), unnormalised (the 1/M of
//         dsp.py:115-119 is folded into the conjugate code spectrum table).
// Natural order in, natural order out.
#pragma once
#include <cuda_runtime.h>

namespace gacq {

typedef unsigned long long cx;  // packed complex64: low word = re, high word = im

__device__ __forceinline__ cx pk(float re, float im) {
    cx r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(re), "f"(im));
    return r;
}
__device__ __forceinline__ float re(cx v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float im(cx v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ cx bc(float x) { return pk(x, x); }
__device__ __forceinline__ cx czero() { return 0ull; }

__device__ __forceinline__ cx add2(cx a, cx b) {
    cx r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx sub2(cx a, cx b) {
    cx r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx mul2(cx a, cx b) {
    cx r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx fma2(cx a, cx b, cx c) {
    cx r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// a * (S i)
template <int S>
__device__ __forceinline__ cx rot(cx a) {
    return S < 0 ? pk(im(a), -re(a)) : pk(-im(a), re(a));
}
// a * w (general complex product: 2 instructions)
__device__ __forceinline__ cx cmul(cx a, cx w) { return fma2(rot<1>(a), bc(im(w)), mul2(a, bc(re(w)))); }
// a * conj(w)
__device__ __forceinline__ cx cmul_conj(cx a, cx w) { return fma2(rot<1>(a), bc(-im(w)), mul2(a, bc(re(w)))); }
__device__ __forceinline__ float cmag2(cx a) { return re(a) * re(a) + im(a) * im(a); }

// exact complex64 product of kernels.py:78-86: round(round(ar*br) - round(ai*bi)),
// round(round(ar*bi) + round(ai*br)). Scalar __fmul_rn/__fadd_rn are never contracted;
// ptxas DOES fuse mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (observed in SASS), so the
// packed forms must not be used here.
__device__ __forceinline__ cx cmul_exact(cx a, cx b) {
    const float ar = re(a), ai = im(a), br = re(b), bi = im(b);
    return pk(__fsub_rn(__fmul_rn(ar, br), __fmul_rn(ai, bi)), __fadd_rn(__fmul_rn(ar, bi), __fmul_rn(ai, br)));
}

constexpr float kC8 = 0.70710678118654752440f;  // cos(pi/4)
constexpr float kC16 = 0.92387953251128675613f; // cos(pi/8)
constexpr float kS16 = 0.38268343236508977173f; // sin(pi/8)

// a * W8^1, W8 = exp(S i pi/4) = (1 + S i)/sqrt2
template <int S>
__device__ __forceinline__ cx mul_w8_1(cx a) { return mul2(add2(a, rot<S>(a)), bc(kC8)); }
// a * W8^3 = (-1 + S i)/sqrt2
template <int S>
__device__ __forceinline__ cx mul_w8_3(cx a) { return mul2(sub2(rot<S>(a), a), bc(kC8)); }
// a * (c + S i s)
template <int S>
__device__ __forceinline__ cx mul_cs(cx a, float c, float s) {
    return fma2(rot<S>(a), bc(s), mul2(a, bc(c)));
}

template <int S>
__device__ __forceinline__ void dft4(cx& a0, cx& a1, cx& a2, cx& a3) {
    const cx t0 = add2(a0, a2), t1 = sub2(a0, a2);
    const cx t2 = add2(a1, a3), t3 = sub2(a1, a3);
    a0 = add2(t0, t2);
    a2 = sub2(t0, t2);
    a1 = add2(t1, rot<S>(t3));
    a3 = sub2(t1, rot<S>(t3));
}

template <int S>
__device__ __forceinline__ void dft8(cx (&v)[8]) {
    cx e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    cx o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<S>(e0, e1, e2, e3);
    dft4<S>(o0, o1, o2, o3);
    o1 = mul_w8_1<S>(o1);
    o3 = mul_w8_3<S>(o3);
    v[0] = add2(e0, o0); v[4] = sub2(e0, o0);
    v[1] = add2(e1, o1); v[5] = sub2(e1, o1);
    v[2] = add2(e2, rot<S>(o2)); v[6] = sub2(e2, rot<S>(o2));
    v[3] = add2(e3, o3); v[7] = sub2(e3, o3);
}

// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
template <int S>
__device__ __forceinline__ void dft16(cx (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<S>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
    // after the first stage v[4*k1 + n2] holds Y[n2][k1]; apply W16^(n2*k1)
    v[5] = mul_cs<S>(v[5], kC16, kS16);     // n2=1,k1=1: W^1
    v[9] = mul_w8_1<S>(v[9]);               // n2=1,k1=2: W^2
    v[13] = mul_cs<S>(v[13], kS16, kC16);   // n2=1,k1=3: W^3
    v[6] = mul_w8_1<S>(v[6]);               // n2=2,k1=1: W^2
    v[10] = rot<S>(v[10]);                  // n2=2,k1=2: W^4 (folded into the adds below)
    v[14] = mul_w8_3<S>(v[14]);             // n2=2,k1=3: W^6
    v[7] = mul_cs<S>(v[7], kS16, kC16);     // n2=3,k1=1: W^3
    v[11] = mul_w8_3<S>(v[11]);             // n2=3,k1=2: W^6
    v[15] = mul_cs<S>(v[15], -kC16, -kS16); // n2=3,k1=3: W^9 = -W^1
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1 + 0], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // v[4*k1 + k2] holds X[k1 + 4*k2]: transpose 4x4 to natural order (register renaming)
    cx t;
    t = v[1]; v[1] = v[4]; v[4] = t;
    t = v[2]; v[2] = v[8]; v[8] = t;
    t = v[3]; v[3] = v[12]; v[12] = t;
    t = v[6]; v[6] = v[9]; v[9] = t;
    t = v[7]; v[7] = v[13]; v[13] = t;
    t = v[11]; v[11] = v[14]; v[14] = t;
}

}  // namespace gacq
