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

// Per-lane constants of the warp FFTs (float2; cmul2 multiplies in two packed
// instructions without a pre-swapped copy): cw[k] = W_(2h)^(l mod h) on the upper lane
// of the stage h = 2^k (1 on the lower lane), sgk[k] = -1 on the upper lane;
// tw[k0] = W_n^(l k0). Forward transforms only: an inverse is run as
// conj(FFT(conj x)), the conjugations folded into the callers' loads and stores.
template <int M>
struct WarpFFT {
    static constexpr int kBufFloat2 = 0;  // no shared-memory transpose
    float2 cw[5];  // cw[0] = 1 and cw[1] in {1, -i} are applied without multiplies (stage())
    float sgk[5];
    float2 tw[M];
    bool mi = false;  // lane of stage h = 2 whose twiddle is -i ((l & 3) == 3)
    int lb = 0;       // M br5(l)
    int ln = 0;       // l
    // index held in register k of the F1 output / F2 input ("scrambled" layout)
    __device__ __forceinline__ int scr(int k) const { return k + lb; }
    // index held in register k of the F1 input / F2 output ("natural" layout)
    __device__ __forceinline__ int nat(int k) const { return ln + 32 * k; }
    // phase roles of the box / cluster kernels: A = IFFT of a gathered box row (scrambled
    // in, natural out), C = FFT of a row before its scatter (natural in, scrambled out);
    // every register can hold box data
    __device__ __forceinline__ int a_in(int k) const { return scr(k); }
    __device__ __forceinline__ int a_out(int k) const { return nat(k); }
    __device__ __forceinline__ void fA(float2 (&x)[M]) const { f2(x); }
    __device__ __forceinline__ int c_in(int k) const { return nat(k); }
    __device__ __forceinline__ int c_out(int k) const { return scr(k); }
    __device__ __forceinline__ void fC(float2 (&x)[M]) const { f1(x); }
    __host__ __device__ static constexpr bool live(int) { return true; }
    // column XOR of a staged measurement row r that spreads the scrambled-layout
    // rows of one register over distinct banks (r = k + M br5(l): 2 br5(l))
    static __device__ __forceinline__ int isw(int r) { return 2 * (r / M); }
    __device__ __forceinline__ int isw_lane() const { return 2 * (lb / M); }
    __device__ void init(int l, int n, float2* = nullptr) {
        lb = M * brev5(l);
        ln = l;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            double s, c;
            sincospi(-double(l & (h - 1)) / double(h), &s, &c);
            const float wc = up ? float(c) : 1.f, ws = up ? float(s) : 0.f;
            cw[k] = make_float2(wc, ws);
            sgk[k] = up ? -1.f : 1.f;
        }
        mi = (l & 3) == 3;
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            double s, c;
            sincospi(-2.0 * double(l * k0) / double(n), &s, &c);
            tw[k0] = make_float2(float(c), float(s));
        }
    }
    // the same constants from a table tab[m] = W_n^m (m in [0, n)) in global memory
    __device__ void init_table(int l, int n, const float2* __restrict__ tab) {
        lb = M * brev5(l);
        ln = l;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            const float2 w = up ? __ldg(tab + (l & (h - 1)) * (n / (2 * h))) : make_float2(1.f, 0.f);
            cw[k] = w;
            sgk[k] = up ? -1.f : 1.f;
        }
        mi = (l & 3) == 3;
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            const float2 w = __ldg(tab + (l * k0) % n);
            tw[k0] = w;
        }
    }
    // the same from a copy of the table in shared memory (plain loads)
    __device__ void init_smem(int l, int n, const float2* tab) {
        lb = M * brev5(l);
        ln = l;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int h = 1 << k;
            const bool up = (l & h) != 0;
            const float2 w = up ? tab[(l & (h - 1)) * (n / (2 * h))] : make_float2(1.f, 0.f);
            cw[k] = w;
            sgk[k] = up ? -1.f : 1.f;
        }
        mi = (l & 3) == 3;
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) {
            const float2 w = tab[(l * k0) % n];
            tw[k0] = w;
        }
    }
    static __device__ __forceinline__ float2 mul(float2 v, float2 w) { return cmul2(v, w); }
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

// lane-gated rotation a x + (b x.y, -b x.x): W x for (a, b) = (cos t, sin t), W = e^{-i t};
// x itself for (1, 0). bb = (b, -b), so the FFMA2 takes x half-swapped (a free
// operand modifier) instead of a negated copy
__device__ __forceinline__ float2 rot_g(float2 x, float a, float2 bb) {
    f32x2 t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(x)), "l"(pk(make_float2(a, a))));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(make_float2(x.y, x.x))), "l"(pk(bb)), "l"(t));
    return upk(r);
}

// n = 256 as 16 x 16 with each 16-point DFT on a lane pair (l, l ^ 16): lane
// l = p + 16 h holds 8 values; a register DFT8 plus one radix-2 exchange forms
// a DFT16, and one 16 x 17 shared-memory transpose per transform replaces four
// of the five shuffle stages of WarpFFT<8> (32 instead of 80 SHFL per lane,
// and no per-stage lane twiddles: the shuffle pipe, 1 SHFL / clk / SM, was
// the binding unit). Same layouts as WarpFFT<8>'s F1 / F2 contract except the
// scrambled order:
//   F1 (DIT): x[l + 32 a] -> X[p + 16 k + 128 h]   (n = 16 n1 + n2: n2 = p, n1 = 2a + h)
//   F2 (DIF): x[p + 16 k + 128 h] -> X[l + 32 c]
// Both share one twiddle table W256^(p (2b + h)) (F1 applies it after the
// transpose, F2 before). Forward only, unnormalised.
// MID: the support box lies in [64, 192) (BASELINE config 5: [70, 187)), so of
// the natural layout only registers 2..5 hold box data: F1 prunes its first
// DFT8 to those inputs, F2 its last DFT8 to those outputs, and the kernels skip
// the other registers' loads and stores. The phase roles put the natural layout
// on the box side of every transform: A = F1 (gather natural, send scrambled),
// C = F2 (fetch scrambled, scatter natural).
template <bool MID>
struct WarpFFT256 {
    static constexpr int kBufFloat2 = 16 * 17;  // per-warp transpose buffer (row stride 17: conflict-free)
    float2 tw[8];  // two registers each: cmul2 needs no pre-swapped copy
    float ga[8];         // cos(2 pi k / 16) on the upper half (h = 1), 1 on the lower
    float2 gb[8];        // (sin, -sin)(2 pi k / 16) on the upper half, 0 on the lower
    float sg;            // +1 lower half, -1 upper
    int p, h, ln;
    float2* buf;
    __device__ __forceinline__ int scr(int k) const { return p + 16 * k + 128 * h; }
    __device__ __forceinline__ int nat(int k) const { return ln + 32 * k; }
    __host__ __device__ static constexpr bool live(int k) { return !MID || (k >= 2 && k < 6); }
    __device__ __forceinline__ int a_in(int k) const { return nat(k); }
    __device__ __forceinline__ int a_out(int k) const { return scr(k); }
    __device__ __forceinline__ void fA(float2 (&x)[8]) const { f1(x); }
    __device__ __forceinline__ int c_in(int k) const { return scr(k); }
    __device__ __forceinline__ int c_out(int k) const { return nat(k); }
    __device__ __forceinline__ void fC(float2 (&x)[8]) const { f2(x); }
    // rows p + 16 k + 128 h of one register: (p, h) -> 32 distinct banks of u16 pairs
    static __device__ __forceinline__ int isw(int r) { return 2 * ((r & 15) | ((r >> 3) & 16)); }
    // isw of every row this lane holds in the scrambled layout (independent of k)
    __device__ __forceinline__ int isw_lane() const { return 2 * (p | (16 * h)); }
    __device__ void init(int l, int n, float2* tbuf) {
        (void)n;  // 256
        p = l & 15;
        h = l >> 4;
        ln = l;
        sg = h ? -1.f : 1.f;
        buf = tbuf;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double s, c;
            sincospi(double(k) / 8.0, &s, &c);
            ga[k] = h ? float(c) : 1.f;
            gb[k] = h ? make_float2(float(s), -float(s)) : make_float2(0.f, 0.f);
            sincospi(-2.0 * double((p * (2 * k + h)) & 255) / 256.0, &s, &c);
            tw[k] = make_float2(float(c), float(s));
        }
    }
    static __device__ __forceinline__ float2 mul(float2 v, float2 w) { return cmul2(v, w); }
    // DFT16 over the pair, decimation in time: lower lane holds the even inputs,
    // upper the odd ones (register a = input 2a + h); out: register k = X[k + 8 h]
    template <bool PIN>
    __device__ __forceinline__ void dit16(float2 (&x)[8]) const {
        dft8<false, PIN>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);  // PIN: inputs 0, 1, 6, 7 zero
#pragma unroll
        for (int k = 1; k < 8; ++k) x[k] = rot_g(x[k], ga[k], gb[k]);  // upper: W16^k O[k]
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = cfma(sg, x[k], shfl_x(x[k], 16));
    }
    // DFT16 over the pair, decimation in frequency: register k = input k + 8 h;
    // out: register c = X[2c + h]
    template <bool POUT>
    __device__ __forceinline__ void dif16(float2 (&x)[8]) const {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = cfma(sg, x[k], shfl_x(x[k], 16));
#pragma unroll
        for (int k = 1; k < 8; ++k) x[k] = rot_g(x[k], ga[k], gb[k]);  // upper: (x[k] - x[k + 8]) W16^k
        dft8<false, false, POUT>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);  // POUT: outputs 2..5 only
    }
    __device__ __forceinline__ void f1(float2 (&x)[8]) const {
        dit16<MID>(x);  // register k = Y[n2 = p][k1 = k + 8h]
        float2* wr = buf + 136 * h + p;
#pragma unroll
        for (int k = 0; k < 8; ++k) wr[17 * k] = x[k];  // [k1][n2]
        __syncwarp();
        const float2* rd = buf + 17 * p + h;
#pragma unroll
        for (int b = 0; b < 8; ++b) x[b] = mul(rd[2 * b], tw[b]);  // Y[n2 = 2b + h][k1 = p] W256^(n2 k1)
        __syncwarp();
        dit16<false>(x);  // register k = X[p + 16 (k + 8h)]
    }
    __device__ __forceinline__ void f2(float2 (&x)[8]) const {
        dif16<false>(x);  // register c = Y[p][k2 = 2c + h]
        float2* wr = buf + 17 * h + p;
#pragma unroll
        for (int c = 0; c < 8; ++c) wr[34 * c] = mul(x[c], tw[c]);  // [k2][p]
        __syncwarp();
        const float2* rd = buf + 17 * p + 8 * h;
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = rd[q];  // Z[p = q + 8h][k2 = p_lane]
        __syncwarp();
        dif16<MID>(x);  // register c = X[p + 16 (2c + h)] = X[l + 32 c]
    }
};

template <int M, bool MID>
struct WarpFFTSel {
    using type = WarpFFT<M>;
};
template <bool MID>
struct WarpFFTSel<8, MID> {
    using type = WarpFFT256<MID>;
};

}  // namespace
}  // namespace fpmk
