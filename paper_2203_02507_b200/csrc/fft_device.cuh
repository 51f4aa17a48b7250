// Register-resident FFT building blocks for sm_100a (FP32 complex).
//
// Complex arithmetic runs on Blackwell's packed FP32x2 pipe: a complex add /
// sub is one FADD2, a scaled accumulate one FFMA2, and the operand swaps and
// partial negations of "multiply by -i / +i" fold into FADD2's HI_LO / LO_HI.NP
// modifiers, so an 8-point DFT is 26 instructions instead of 52. Each FADD2 /
// FFMA2 lane is an ordinary IEEE FP32 add / fused multiply-add.
//
// Centered transforms use the checkerboard identity for even n:
//   fftshift(FFT(ifftshift(x))) = C . FFT(C . x),  C_ij = (-1)^(i+j)
// (the (-1)^(n/2) factors of the two axes cancel), which replaces the
// reference's four shift copies per fft2 (field.cpp:48-56, :69-87) by sign
// flips folded into loads and stores.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fpmk {

typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk(float2 a) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk(f32x2 r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
// s * a + b, s broadcast to both lanes
__device__ __forceinline__ float2 cfma(float s, float2 a, float2 b) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(make_float2(s, s))), "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
// s * a + b with a per-half multiplier s = (s.x, s.y): for the lane rotations
// (x + k y, y - k x) = (k, -k) swap(x) + x, one FFMA2 (the (k, -k) pair is the
// broadcast k with a half negation, the swap an operand modifier)
__device__ __forceinline__ float2 cfma_v(float2 s, float2 a, float2 b) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(s)), "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(make_float2(s, s))));
    return upk(r);
}
__device__ __forceinline__ float2 cneg(float2 a) { return make_float2(-a.x, -a.y); }
// v * w with wsw = (-w.y, w.x) precomputed: FMUL2 + FFMA2
__device__ __forceinline__ float2 cmul_sw(float2 v, float2 w, float2 wsw) {
    f32x2 t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(make_float2(v.x, v.x))), "l"(pk(w)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(make_float2(v.y, v.y))), "l"(pk(wsw)), "l"(t));
    return upk(r);
}
// v * w in two packed instructions from w alone: FMUL2 t = v w.y, then FFMA2 v w.x +
// (-t.y, t.x) (the half swap and the partial negation are operand modifiers)
__device__ __forceinline__ float2 cmul2(float2 v, float2 w) {
    const float2 t = cscale(v, w.y);
    return cfma(w.x, v, make_float2(-t.y, t.x));
}
// conj(v p) in two packed instructions: s = p.x v, then (s.x, -s.y) - p.y swap(v)
// (FFMA2 with a negated broadcast, a swapped multiplicand and a half-negated addend)
__device__ __forceinline__ float2 cmul_conj(float2 v, float2 p) {
    const float2 s = cscale(v, p.x);
    return cfma(-p.y, make_float2(v.y, v.x), make_float2(s.x, -s.y));
}
#ifndef FPM_CMUL_PACKED
#define FPM_CMUL_PACKED 1  // complex products as FMUL2 + FFMA2 (0: four scalar FMUL / FFMA)
#endif
#if FPM_CMUL_PACKED
__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return cmul2(a, b); }
// a * conj(b) = b.x a + (t.y, -t.x), t = b.y a: FMUL2 + FFMA2
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    const float2 t = cscale(a, b.y);
    return cfma(b.x, a, make_float2(t.y, -t.x));
}
#else
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
#endif
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// Single-MUFU approximations without the denormal pre/post scaling of the
// non-ftz forms; callers clamp their arguments to >= kTiny (or 0 for sqrt).
constexpr float kTiny = 1.17549435e-38f;  // FLT_MIN
__device__ __forceinline__ float sqrt_ftz(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// multiply by W8^2 = -i (fwd) / +i (inv): a swap and a sign, folded into the consumer
template <bool INV>
__device__ __forceinline__ float2 w8_2(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// In-place 8-point DFT, natural order in and out (radix-2 decimation in
// frequency, 3 stages). The W8 / W8^3 twiddles of the odd half share the
// factor 1/sqrt(2), folded into the last stage's FFMA2s. MID4: inputs 0, 1, 6, 7
// are known zero, so the first butterfly stage degenerates to copies. OMID:
// only outputs 2..5 are formed (the others are left undefined).
template <bool INV, bool MID4, bool OMID = false>
__device__ __forceinline__ void dft8(float2& x0, float2& x1, float2& x2, float2& x3, float2& x4,
                                     float2& x5, float2& x6, float2& x7) {
    float2 a0, a1, a2, a3, a4, a5, a6, a7;
    if (MID4) {
        a0 = x4; a4 = cneg(x4);
        a1 = x5; a5 = cneg(x5);
        a2 = x2; a6 = x2;
        a3 = x3; a7 = x3;
    } else {
        a0 = cadd(x0, x4); a4 = csub(x0, x4);
        a1 = cadd(x1, x5); a5 = csub(x1, x5);
        a2 = cadd(x2, x6); a6 = csub(x2, x6);
        a3 = cadd(x3, x7); a7 = csub(x3, x7);
    }
    a6 = w8_2<INV>(a6);
    const float2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
    const float2 b1 = cadd(a1, a3), b3 = w8_2<INV>(csub(a1, a3));
    const float2 b4 = cadd(a4, a6), b6 = csub(a4, a6);
    // W8 a5 = s A, W8^3 a7 = s B (fwd: A = a5 + (-i) a5, B = (-i) a7 - a7; inv: +i)
    const float2 A = cadd(a5, w8_2<INV>(a5));
    const float2 Bv = csub(w8_2<INV>(a7), a7);
    const float2 b5u = cadd(A, Bv), b7u = w8_2<INV>(csub(A, Bv));
    const float s = 0.70710678118654752440f;
    x4 = csub(b0, b1);
    x2 = cadd(b2, b3);
    x5 = cfma(-s, b5u, b4);
    x3 = cfma(s, b7u, b6);
    if (!OMID) {
        x0 = cadd(b0, b1);
        x6 = csub(b2, b3);
        x1 = cfma(s, b5u, b4);
        x7 = cfma(-s, b7u, b6);
    }
}

// 2-D 8x8 DFT over the register block v[a][b]: first along a (for each b),
// then along b. PRUNE: only a, b in [2, 6) are nonzero on entry.
template <bool INV, bool PRUNE>
__device__ __forceinline__ void dft8x8(float2 (&v)[8][8]) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (PRUNE && (b < 2 || b > 5)) continue;
        dft8<INV, PRUNE>(v[0][b], v[1][b], v[2][b], v[3][b], v[4][b], v[5][b], v[6][b], v[7][b]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
        dft8<INV, PRUNE>(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4], v[a][5], v[a][6], v[a][7]);
}

// radix-4 butterfly with a0 = a3 = 0 on entry (the pruned IFFT's zero columns):
// s02 = a2, d02 = -a2, s13 = a1, d13 = w a1 -> four FADD2 instead of eight
template <bool INV>
__device__ __forceinline__ void dft4_z03(float2& a0, float2& a1, float2& a2, float2& a3) {
    const float2 x1 = a1, x2 = a2, d13 = w8_2<INV>(x1);
    a0 = cadd(x2, x1);
    a2 = csub(x2, x1);
    a1 = csub(d13, x2);
    a3 = csub(cneg(x2), d13);
}

// radix-4 butterfly producing only outputs 1 and 2 (the pruned FFT's scatter columns)
template <bool INV>
__device__ __forceinline__ void dft4_o12(float2& a0, float2& a1, float2& a2, float2& a3) {
    const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const float2 s13 = cadd(a1, a3), d13 = w8_2<INV>(csub(a1, a3));
    a1 = cadd(d02, d13);
    a2 = csub(s02, s13);
}

// radix-4 butterfly on natural-order inputs (fwd: W4 = -i)
template <bool INV>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
    const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const float2 s13 = cadd(a1, a3), d13 = w8_2<INV>(csub(a1, a3));
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, d13);
    a3 = csub(d02, d13);
}

}  // namespace fpmk
