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

// Per-lane constants of the warp FFTs, as (w, (-w.y, w.x)) pairs for the packed
// two-instruction complex multiply: cw[k] = W_(2h)^(l mod h) on the upper lane
// of the stage h = 2^k (1 on the lower lane), sgk[k] = -1 on the upper lane;
// tw[k0] = W_n^(l k0). Forward transforms only: an inverse is run as
// conj(FFT(conj x)), the conjugations folded into the callers' loads and stores.
template <int M>
struct WarpFFT {
    float4 cw[5];  // cw[0] = 1 and cw[1] in {1, -i} are applied without multiplies (stage())
    float sgk[5];
    float4 tw[M];
    bool mi = false;  // lane of stage h = 2 whose twiddle is -i ((l & 3) == 3)
    __device__ void init(int l, int n) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            double s, c;
            sincospi(-double(l & (h - 1)) / double(h), &s, &c);
            const float wc = up ? float(c) : 1.f, ws = up ? float(s) : 0.f;
            cw[k] = make_float4(wc, ws, -ws, wc);
            sgk[k] = up ? -1.f : 1.f;
        }
        mi = (l & 3) == 3;
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            double s, c;
            sincospi(-2.0 * double(l * k0) / double(n), &s, &c);
            tw[k0] = make_float4(float(c), float(s), -float(s), float(c));
        }
    }
    // the same constants from a table tab[m] = W_n^m (m in [0, n)) in global memory
    __device__ void init_table(int l, int n, const float2* __restrict__ tab) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            const float2 w = up ? __ldg(tab + (l & (h - 1)) * (n / (2 * h))) : make_float2(1.f, 0.f);
            cw[k] = make_float4(w.x, w.y, -w.y, w.x);
            sgk[k] = up ? -1.f : 1.f;
        }
        mi = (l & 3) == 3;
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            const float2 w = __ldg(tab + (l * k0) % n);
            tw[k0] = make_float4(w.x, w.y, -w.y, w.x);
        }
    }
    static __device__ __forceinline__ float2 mul(float2 v, const float4& w) {
        return cmul_sw(v, make_float2(w.x, w.y), make_float2(w.z, w.w));
    }
    // lane twiddle of stage k: W_2^0 = 1 (none), W_4^(l mod 2) in {1, -i} (a lane-selected
    // swap and sign on the ALU pipe), a packed complex multiply from stage 2 on
    template <int K>
    __device__ __forceinline__ float2 stage(float2 v) const {
        if constexpr (K == 0) {
            return v;
        } else if constexpr (K == 1) {
            const float nx = __int_as_float(__float_as_int(v.x) ^ int(0x80000000u));
            return mi ? make_float2(v.y, nx) : v;
        } else {
            return mul(v, cw[K]);
        }
    }
    // F1: x[l + 32 m] -> X[k0 + M br5(l)]: register DFT, twiddle, lane DIF
    __device__ __forceinline__ void f1(float2 (&x)[M]) const {
        dftM<false, M>(x);
#pragma unroll
        for (int k0 = 1; k0 < M; ++k0) x[k0] = mul(x[k0], tw[k0]);
        dif_stage<4>(x);
        dif_stage<3>(x);
        dif_stage<2>(x);
        dif_stage<1>(x);
        dif_stage<0>(x);
    }
    template <int K>
    __device__ __forceinline__ void dif_stage(float2 (&x)[M]) const {  // h = 2^K
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) x[k0] = stage<K>(cfma(sgk[K], x[k0], shfl_x(x[k0], 1 << K)));
    }
    template <int K>
    __device__ __forceinline__ void dit_stage(float2 (&x)[M]) const {  // h = 2^K
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            const float2 b = stage<K>(x[k0]);
            x[k0] = cfma(sgk[K], b, shfl_x(b, 1 << K));
        }
    }
    // F2: x[k0 + M br5(l)] -> X[q + 32 r]: lane DIT, twiddle, register DFT
    __device__ __forceinline__ void f2(float2 (&x)[M]) const {
        dit_stage<0>(x);
        dit_stage<1>(x);
        dit_stage<2>(x);
        dit_stage<3>(x);
        dit_stage<4>(x);
#pragma unroll
        for (int k0 = 1; k0 < M; ++k0) x[k0] = mul(x[k0], tw[k0]);
        dftM<false, M>(x);
    }
};

}  // namespace
}  // namespace fpmk
