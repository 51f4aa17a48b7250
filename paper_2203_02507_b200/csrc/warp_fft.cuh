// Warp-wide n-point FFTs (n = 32 M) shared by the general-n kernels
// (kernels_box.cu, kernels_cluster.cu): a register DFT_M and a 32-point DFT
// across the lanes (5 radix-2 stages over shuffles), in two flavours that
// chain without reordering:
//   F1: x[l + 32 m] (lane l, register m)      -> X[k0 + M br5(l)] (register k0)
//   F2: x[k0 + M br5(l)]                      -> X[q + 32 r] (lane q, register r)
#pragma once

#include "fft_device.cuh"

namespace fpmk {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int brev5(int l) { return int(__brev(unsigned(l)) >> 27); }

__device__ __forceinline__ float2 shfl_x(float2 v, int m) {
    return make_float2(__shfl_xor_sync(kFull, v.x, m), __shfl_xor_sync(kFull, v.y, m));
}

template <bool INV>
__device__ __forceinline__ float2 tmul(float2 v, float2 w) {
    return INV ? cmulc(v, w) : cmul(v, w);
}

template <bool INV, int M>
__device__ __forceinline__ void dftM(float2 (&x)[M]) {
    if constexpr (M == 2) {
        const float2 a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    } else if constexpr (M == 4) {
        dft4<INV>(x[0], x[1], x[2], x[3]);
    } else {
        dft8<INV, false>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
    }
}

// Per-lane constants of the warp FFTs: cw[k] = W_(2h)^(l mod h) on the upper
// lane of the stage h = 2^k (1 on the lower lane), sgk[k] = -1 on the upper
// lane; tw[k0] = W_n^(l k0).
template <int M>
struct WarpFFT {
    float2 cw[5];
    float sgk[5];
    float2 tw[M];
    __device__ void init(int l, int n) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            double s, c;
            sincospi(-double(l & (h - 1)) / double(h), &s, &c);
            cw[k] = up ? make_float2(float(c), float(s)) : make_float2(1.f, 0.f);
            sgk[k] = up ? -1.f : 1.f;
        }
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            double s, c;
            sincospi(-2.0 * double(l * k0) / double(n), &s, &c);
            tw[k0] = make_float2(float(c), float(s));
        }
    }
    template <bool INV>
    __device__ __forceinline__ void f1(float2 (&x)[M]) const {
        dftM<INV, M>(x);
#pragma unroll
        for (int k0 = 1; k0 < M; ++k0) x[k0] = tmul<INV>(x[k0], tw[k0]);
#pragma unroll
        for (int k = 4; k >= 0; --k) {  // DIF: h = 16 .. 1
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const float2 r = shfl_x(x[k0], 1 << k);
                const float2 y = make_float2(fmaf(sgk[k], x[k0].x, r.x), fmaf(sgk[k], x[k0].y, r.y));
                x[k0] = tmul<INV>(y, cw[k]);
            }
        }
    }
    template <bool INV>
    __device__ __forceinline__ void f2(float2 (&x)[M]) const {
#pragma unroll
        for (int k = 0; k < 5; ++k) {  // DIT: h = 1 .. 16
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const float2 b = tmul<INV>(x[k0], cw[k]);
                const float2 r = shfl_x(b, 1 << k);
                x[k0] = make_float2(fmaf(sgk[k], b.x, r.x), fmaf(sgk[k], b.y, r.y));
            }
        }
#pragma unroll
        for (int k0 = 1; k0 < M; ++k0) x[k0] = tmul<INV>(x[k0], tw[k0]);
        dftM<INV, M>(x);
    }
};

}  // namespace
}  // namespace fpmk
