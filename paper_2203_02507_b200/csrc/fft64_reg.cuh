// Register-resident 64-point FFTs for the one-warp-per-tile n = 64 kernel
// (kernels_w64.cu). A lane holds a whole 64-point line in x[8][8]; the
// transform is radix-8 x 8 (n = 8 n1 + n0, k = k0 + 8 k1) with every index
// known at compile time, so the twiddles W64^(n0 k0) are __constant__ operands
// (LDCU into uniform registers, consumed directly by FMUL2 / FFMA2) and the
// output digit order is a register renaming:
//   fft64_nt: x[n1][n0] (natural)  -> x[k0][k1]
//   fft64_tn: x[n0][n1]            -> x[k1][k0] (natural)
// IN_MID: only n1 in [2, 6) is nonzero on entry (a line whose support lies in
// [16, 48)); OUT_MID: only k1 in [2, 6) is produced (outputs [16, 48)).
#pragma once

#include "fft_device.cuh"

namespace fpmk {

// W64^m = (cos, sin)(-2 pi m / 64) rounded to float, as (w, (-w.y, w.x))
__constant__ float4 cW64[64] = {
    {0x1.0000000000000p+0f, -0x0.0p+0f, 0x0.0p+0f, 0x1.0000000000000p+0f},  // m = 0
    {0x1.fd88da0000000p-1f, -0x1.917a6c0000000p-4f, 0x1.917a6c0000000p-4f, 0x1.fd88da0000000p-1f},  // m = 1
    {0x1.f6297c0000000p-1f, -0x1.8f8b840000000p-3f, 0x1.8f8b840000000p-3f, 0x1.f6297c0000000p-1f},  // m = 2
    {0x1.e9f4160000000p-1f, -0x1.2940620000000p-2f, 0x1.2940620000000p-2f, 0x1.e9f4160000000p-1f},  // m = 3
    {0x1.d906bc0000000p-1f, -0x1.87de2a0000000p-2f, 0x1.87de2a0000000p-2f, 0x1.d906bc0000000p-1f},  // m = 4
    {0x1.c38b300000000p-1f, -0x1.e2b5d40000000p-2f, 0x1.e2b5d40000000p-2f, 0x1.c38b300000000p-1f},  // m = 5
    {0x1.a9b6620000000p-1f, -0x1.1c73b40000000p-1f, 0x1.1c73b40000000p-1f, 0x1.a9b6620000000p-1f},  // m = 6
    {0x1.8bc8060000000p-1f, -0x1.44cf320000000p-1f, 0x1.44cf320000000p-1f, 0x1.8bc8060000000p-1f},  // m = 7
    {0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f},  // m = 8
    {0x1.44cf320000000p-1f, -0x1.8bc8060000000p-1f, 0x1.8bc8060000000p-1f, 0x1.44cf320000000p-1f},  // m = 9
    {0x1.1c73b40000000p-1f, -0x1.a9b6620000000p-1f, 0x1.a9b6620000000p-1f, 0x1.1c73b40000000p-1f},  // m = 10
    {0x1.e2b5d40000000p-2f, -0x1.c38b300000000p-1f, 0x1.c38b300000000p-1f, 0x1.e2b5d40000000p-2f},  // m = 11
    {0x1.87de2a0000000p-2f, -0x1.d906bc0000000p-1f, 0x1.d906bc0000000p-1f, 0x1.87de2a0000000p-2f},  // m = 12
    {0x1.2940620000000p-2f, -0x1.e9f4160000000p-1f, 0x1.e9f4160000000p-1f, 0x1.2940620000000p-2f},  // m = 13
    {0x1.8f8b840000000p-3f, -0x1.f6297c0000000p-1f, 0x1.f6297c0000000p-1f, 0x1.8f8b840000000p-3f},  // m = 14
    {0x1.917a6c0000000p-4f, -0x1.fd88da0000000p-1f, 0x1.fd88da0000000p-1f, 0x1.917a6c0000000p-4f},  // m = 15
    {0x1.1a62640000000p-54f, -0x1.0000000000000p+0f, 0x1.0000000000000p+0f, 0x1.1a62640000000p-54f},  // m = 16
    {-0x1.917a6c0000000p-4f, -0x1.fd88da0000000p-1f, 0x1.fd88da0000000p-1f, -0x1.917a6c0000000p-4f},  // m = 17
    {-0x1.8f8b840000000p-3f, -0x1.f6297c0000000p-1f, 0x1.f6297c0000000p-1f, -0x1.8f8b840000000p-3f},  // m = 18
    {-0x1.2940620000000p-2f, -0x1.e9f4160000000p-1f, 0x1.e9f4160000000p-1f, -0x1.2940620000000p-2f},  // m = 19
    {-0x1.87de2a0000000p-2f, -0x1.d906bc0000000p-1f, 0x1.d906bc0000000p-1f, -0x1.87de2a0000000p-2f},  // m = 20
    {-0x1.e2b5d40000000p-2f, -0x1.c38b300000000p-1f, 0x1.c38b300000000p-1f, -0x1.e2b5d40000000p-2f},  // m = 21
    {-0x1.1c73b40000000p-1f, -0x1.a9b6620000000p-1f, 0x1.a9b6620000000p-1f, -0x1.1c73b40000000p-1f},  // m = 22
    {-0x1.44cf320000000p-1f, -0x1.8bc8060000000p-1f, 0x1.8bc8060000000p-1f, -0x1.44cf320000000p-1f},  // m = 23
    {-0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f},  // m = 24
    {-0x1.8bc8060000000p-1f, -0x1.44cf320000000p-1f, 0x1.44cf320000000p-1f, -0x1.8bc8060000000p-1f},  // m = 25
    {-0x1.a9b6620000000p-1f, -0x1.1c73b40000000p-1f, 0x1.1c73b40000000p-1f, -0x1.a9b6620000000p-1f},  // m = 26
    {-0x1.c38b300000000p-1f, -0x1.e2b5d40000000p-2f, 0x1.e2b5d40000000p-2f, -0x1.c38b300000000p-1f},  // m = 27
    {-0x1.d906bc0000000p-1f, -0x1.87de2a0000000p-2f, 0x1.87de2a0000000p-2f, -0x1.d906bc0000000p-1f},  // m = 28
    {-0x1.e9f4160000000p-1f, -0x1.2940620000000p-2f, 0x1.2940620000000p-2f, -0x1.e9f4160000000p-1f},  // m = 29
    {-0x1.f6297c0000000p-1f, -0x1.8f8b840000000p-3f, 0x1.8f8b840000000p-3f, -0x1.f6297c0000000p-1f},  // m = 30
    {-0x1.fd88da0000000p-1f, -0x1.917a6c0000000p-4f, 0x1.917a6c0000000p-4f, -0x1.fd88da0000000p-1f},  // m = 31
    {-0x1.0000000000000p+0f, -0x1.1a62640000000p-53f, 0x1.1a62640000000p-53f, -0x1.0000000000000p+0f},  // m = 32
    {-0x1.fd88da0000000p-1f, 0x1.917a6c0000000p-4f, -0x1.917a6c0000000p-4f, -0x1.fd88da0000000p-1f},  // m = 33
    {-0x1.f6297c0000000p-1f, 0x1.8f8b840000000p-3f, -0x1.8f8b840000000p-3f, -0x1.f6297c0000000p-1f},  // m = 34
    {-0x1.e9f4160000000p-1f, 0x1.2940620000000p-2f, -0x1.2940620000000p-2f, -0x1.e9f4160000000p-1f},  // m = 35
    {-0x1.d906bc0000000p-1f, 0x1.87de2a0000000p-2f, -0x1.87de2a0000000p-2f, -0x1.d906bc0000000p-1f},  // m = 36
    {-0x1.c38b300000000p-1f, 0x1.e2b5d40000000p-2f, -0x1.e2b5d40000000p-2f, -0x1.c38b300000000p-1f},  // m = 37
    {-0x1.a9b6620000000p-1f, 0x1.1c73b40000000p-1f, -0x1.1c73b40000000p-1f, -0x1.a9b6620000000p-1f},  // m = 38
    {-0x1.8bc8060000000p-1f, 0x1.44cf320000000p-1f, -0x1.44cf320000000p-1f, -0x1.8bc8060000000p-1f},  // m = 39
    {-0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f},  // m = 40
    {-0x1.44cf320000000p-1f, 0x1.8bc8060000000p-1f, -0x1.8bc8060000000p-1f, -0x1.44cf320000000p-1f},  // m = 41
    {-0x1.1c73b40000000p-1f, 0x1.a9b6620000000p-1f, -0x1.a9b6620000000p-1f, -0x1.1c73b40000000p-1f},  // m = 42
    {-0x1.e2b5d40000000p-2f, 0x1.c38b300000000p-1f, -0x1.c38b300000000p-1f, -0x1.e2b5d40000000p-2f},  // m = 43
    {-0x1.87de2a0000000p-2f, 0x1.d906bc0000000p-1f, -0x1.d906bc0000000p-1f, -0x1.87de2a0000000p-2f},  // m = 44
    {-0x1.2940620000000p-2f, 0x1.e9f4160000000p-1f, -0x1.e9f4160000000p-1f, -0x1.2940620000000p-2f},  // m = 45
    {-0x1.8f8b840000000p-3f, 0x1.f6297c0000000p-1f, -0x1.f6297c0000000p-1f, -0x1.8f8b840000000p-3f},  // m = 46
    {-0x1.917a6c0000000p-4f, 0x1.fd88da0000000p-1f, -0x1.fd88da0000000p-1f, -0x1.917a6c0000000p-4f},  // m = 47
    {-0x1.a793940000000p-53f, 0x1.0000000000000p+0f, -0x1.0000000000000p+0f, -0x1.a793940000000p-53f},  // m = 48
    {0x1.917a6c0000000p-4f, 0x1.fd88da0000000p-1f, -0x1.fd88da0000000p-1f, 0x1.917a6c0000000p-4f},  // m = 49
    {0x1.8f8b840000000p-3f, 0x1.f6297c0000000p-1f, -0x1.f6297c0000000p-1f, 0x1.8f8b840000000p-3f},  // m = 50
    {0x1.2940620000000p-2f, 0x1.e9f4160000000p-1f, -0x1.e9f4160000000p-1f, 0x1.2940620000000p-2f},  // m = 51
    {0x1.87de2a0000000p-2f, 0x1.d906bc0000000p-1f, -0x1.d906bc0000000p-1f, 0x1.87de2a0000000p-2f},  // m = 52
    {0x1.e2b5d40000000p-2f, 0x1.c38b300000000p-1f, -0x1.c38b300000000p-1f, 0x1.e2b5d40000000p-2f},  // m = 53
    {0x1.1c73b40000000p-1f, 0x1.a9b6620000000p-1f, -0x1.a9b6620000000p-1f, 0x1.1c73b40000000p-1f},  // m = 54
    {0x1.44cf320000000p-1f, 0x1.8bc8060000000p-1f, -0x1.8bc8060000000p-1f, 0x1.44cf320000000p-1f},  // m = 55
    {0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f, -0x1.6a09e60000000p-1f, 0x1.6a09e60000000p-1f},  // m = 56
    {0x1.8bc8060000000p-1f, 0x1.44cf320000000p-1f, -0x1.44cf320000000p-1f, 0x1.8bc8060000000p-1f},  // m = 57
    {0x1.a9b6620000000p-1f, 0x1.1c73b40000000p-1f, -0x1.1c73b40000000p-1f, 0x1.a9b6620000000p-1f},  // m = 58
    {0x1.c38b300000000p-1f, 0x1.e2b5d40000000p-2f, -0x1.e2b5d40000000p-2f, 0x1.c38b300000000p-1f},  // m = 59
    {0x1.d906bc0000000p-1f, 0x1.87de2a0000000p-2f, -0x1.87de2a0000000p-2f, 0x1.d906bc0000000p-1f},  // m = 60
    {0x1.e9f4160000000p-1f, 0x1.2940620000000p-2f, -0x1.2940620000000p-2f, 0x1.e9f4160000000p-1f},  // m = 61
    {0x1.f6297c0000000p-1f, 0x1.8f8b840000000p-3f, -0x1.8f8b840000000p-3f, 0x1.f6297c0000000p-1f},  // m = 62
    {0x1.fd88da0000000p-1f, 0x1.917a6c0000000p-4f, -0x1.917a6c0000000p-4f, 0x1.fd88da0000000p-1f},  // m = 63
};

// v * W64^E (E compile-time after unrolling): multiples of 16 are a swap and a sign
__device__ __forceinline__ float2 tw64(float2 v, int E, int z) {
    E &= 63;
    if (E == 0) return v;
    if (E == 16) return make_float2(v.y, -v.x);
    if (E == 32) return make_float2(-v.x, -v.y);
    if (E == 48) return make_float2(-v.y, v.x);
    // z: a zero the compiler cannot prove (the caller derives it from a loop
    // variable), so the constant loads stay at their use instead of being hoisted
    // out of the caller's loops into (and spilled from) general registers
    const float4 w = cW64[E + z];
    return cmul_sw(v, make_float2(w.x, w.y), make_float2(w.z, w.w));
}

template <bool IN_MID, bool OUT_MID>
__device__ __forceinline__ void fft64_nt(float2 (&x)[8][8], int z) {
#pragma unroll
    for (int n0 = 0; n0 < 8; ++n0)
        dft8<false, IN_MID, false>(x[0][n0], x[1][n0], x[2][n0], x[3][n0], x[4][n0], x[5][n0], x[6][n0], x[7][n0]);
#pragma unroll
    for (int k0 = 1; k0 < 8; ++k0)
#pragma unroll
        for (int n0 = 1; n0 < 8; ++n0) x[k0][n0] = tw64(x[k0][n0], n0 * k0, z);
#pragma unroll
    for (int k0 = 0; k0 < 8; ++k0)
        dft8<false, false, OUT_MID>(x[k0][0], x[k0][1], x[k0][2], x[k0][3], x[k0][4], x[k0][5], x[k0][6], x[k0][7]);
}

template <bool OUT_MID>
__device__ __forceinline__ void fft64_tn(float2 (&x)[8][8], int z) {
#pragma unroll
    for (int n0 = 0; n0 < 8; ++n0)
        dft8<false, false, false>(x[n0][0], x[n0][1], x[n0][2], x[n0][3], x[n0][4], x[n0][5], x[n0][6], x[n0][7]);
#pragma unroll
    for (int n0 = 1; n0 < 8; ++n0)
#pragma unroll
        for (int k0 = 1; k0 < 8; ++k0) x[n0][k0] = tw64(x[n0][k0], n0 * k0, z);
#pragma unroll
    for (int k0 = 0; k0 < 8; ++k0)
        dft8<false, false, OUT_MID>(x[0][k0], x[1][k0], x[2][k0], x[3][k0], x[4][k0], x[5][k0], x[6][k0], x[7][k0]);
}

}  // namespace fpmk
