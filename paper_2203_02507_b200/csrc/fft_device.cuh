// Register-resident FFT building blocks for sm_100a (FP32 complex).
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

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float cabs2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// multiply by W8^k, forward sign exp(-2 pi i k/8); INV uses the conjugate
template <bool INV>
__device__ __forceinline__ float2 w8_1(float2 a) {
    const float s = 0.70710678118654752440f;
    return INV ? make_float2((a.x - a.y) * s, (a.x + a.y) * s) : make_float2((a.x + a.y) * s, (a.y - a.x) * s);
}
template <bool INV>
__device__ __forceinline__ float2 w8_2(float2 a) {  // -i (fwd) / +i (inv)
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
template <bool INV>
__device__ __forceinline__ float2 w8_3(float2 a) {
    const float s = 0.70710678118654752440f;
    return INV ? make_float2(-(a.x + a.y) * s, (a.x - a.y) * s) : make_float2((a.y - a.x) * s, -(a.x + a.y) * s);
}

// In-place 8-point DFT, natural order in and out (radix-2 decimation in
// frequency, 3 stages). MID4: inputs 0, 1, 6, 7 are known zero, so the first
// butterfly stage degenerates to copies (pruned IFFT input of a small pupil).
template <bool INV, bool MID4>
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
    // odd half: b5 = W8 a5 + W8^3 a7 and b7 = W8^2 (W8 a5 - W8^3 a7) share the
    // factor 1/sqrt(2); keep them unscaled and fold the scale into the last
    // stage's FFMAs (4 fewer instructions than multiplying by W8, W8^3)
    const float s = 0.70710678118654752440f;
    float2 b5u, b7u;
    if (!INV) {
        const float u1 = a5.x + a5.y, u2 = a5.y - a5.x, u3 = a7.y - a7.x, u4 = a7.x + a7.y;
        b5u = make_float2(u1 + u3, u2 - u4);
        b7u = make_float2(u2 + u4, u3 - u1);
    } else {
        const float v1 = a5.x - a5.y, v2 = a5.x + a5.y, v3 = a7.x + a7.y, v4 = a7.x - a7.y;
        b5u = make_float2(v1 - v3, v2 + v4);
        b7u = make_float2(v4 - v2, v1 + v3);
    }
    x0 = cadd(b0, b1); x4 = csub(b0, b1);
    x2 = cadd(b2, b3); x6 = csub(b2, b3);
    x1 = make_float2(fmaf(s, b5u.x, b4.x), fmaf(s, b5u.y, b4.y));
    x5 = make_float2(fmaf(-s, b5u.x, b4.x), fmaf(-s, b5u.y, b4.y));
    x3 = make_float2(fmaf(s, b7u.x, b6.x), fmaf(s, b7u.y, b6.y));
    x7 = make_float2(fmaf(-s, b7u.x, b6.x), fmaf(-s, b7u.y, b6.y));
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
