// K2/K3 line FFTs (init_canvas, canvas_to_field) and build_pupils.
#include <cstdlib>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "warp_fft.cuh"

namespace fpmk {

namespace {

// Radix-4 (+ one radix-2) Stockham passes over `lines` rows of NL points held
// in shared memory; returns the buffer holding the result.
template <int NL, bool INV>
__device__ float2* stockham(float2* s0, float2* s1, int lines, const float2* __restrict__ tw) {
    float2* src = s0;
    float2* dst = s1;
    int Ns = 1;
#pragma unroll 1
    for (; Ns * 4 <= NL; Ns *= 4) {
        const int quarter = NL / 4;
        const int twstep = NL / (4 * Ns);
        for (int q = threadIdx.x; q < lines * quarter; q += blockDim.x) {
            const int line = q / quarter, j = q - line * quarter;
            const int k = j % Ns;
            const float2* in = src + line * NL + j;
            float2 a0 = in[0], a1 = in[quarter], a2 = in[2 * quarter], a3 = in[3 * quarter];
            if (Ns > 1) {
                const float2 w1 = __ldg(tw + k * twstep), w2 = __ldg(tw + 2 * k * twstep), w3 = __ldg(tw + 3 * k * twstep);
                a1 = INV ? cmulc(a1, w1) : cmul(a1, w1);
                a2 = INV ? cmulc(a2, w2) : cmul(a2, w2);
                a3 = INV ? cmulc(a3, w3) : cmul(a3, w3);
            }
            dft4<INV>(a0, a1, a2, a3);
            float2* out = dst + line * NL + (j / Ns) * Ns * 4 + k;
            out[0] = a0;
            out[Ns] = a1;
            out[2 * Ns] = a2;
            out[3 * Ns] = a3;
        }
        __syncthreads();
        float2* tmp = src;
        src = dst;
        dst = tmp;
    }
    if (Ns < NL) {  // one radix-2 pass (NL = 2 * 4^k)
        const int half = NL / 2;
        for (int q = threadIdx.x; q < lines * half; q += blockDim.x) {
            const int line = q / half, j = q - line * half;
            const float2 w = __ldg(tw + j);
            const float2 a0 = src[line * NL + j];
            const float2 a1 = INV ? cmulc(src[line * NL + j + half], w) : cmul(src[line * NL + j + half], w);
            dst[line * NL + j] = cadd(a0, a1);
            dst[line * NL + j + half] = csub(a0, a1);
        }
        __syncthreads();
        src = dst;
    }
    return src;
}

// WHICH 0: init rows    bilinear(sqrt(seed crop)) * C -> FFT rows -> dst
//       1: init cols    FFT cols of src -> * C * scale -> dst
//       2: final rows   src * C -> IFFT rows -> dst
//       3: final cols   IFFT cols of src -> * C * scale -> dst
template <int NL, int LPB, int WHICH>
__global__ void __launch_bounds__(256) lines_fft(const LinesArgs a) {
    constexpr bool INV = WHICH >= 2;
    constexpr bool COLS = (WHICH & 1) == 1;
    extern __shared__ float2 lbuf[];
    float2* s0 = lbuf;
    float2* s1 = lbuf + LPB * NL;
    const int tile = blockIdx.y;
    const int l0 = blockIdx.x * LPB;
    const size_t base = size_t(tile) * NL * NL;

    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        int line, e;
        if (COLS) {
            e = idx / LPB;
            line = idx - e * LPB;
        } else {
            line = idx / NL;
            e = idx - line * NL;
        }
        float2 x;
        if (WHICH == 0) {
            // upsample_bilinear (field.cpp:89-112) of the seed crop's sqrt, pixel-centre mapped
            const int i = l0 + line, j = e, n = a.n;
            const float fy = (i + 0.5f) / a.up - 0.5f, fx = (j + 0.5f) / a.up - 0.5f;
            int ya = int(floorf(fy)), xa = int(floorf(fx));
            const float wy = fy - ya, wx = fx - xa;
            const int yb = min(ya + 1, n - 1), xb = min(xa + 1, n - 1);
            ya = max(ya, 0);
            xa = max(xa, 0);
            const int2 txy = a.tile_xy[tile];
            const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
            const float v00 = sqrtf(float(f[size_t(ya) * a.pitch + xa]));
            const float v01 = sqrtf(float(f[size_t(ya) * a.pitch + xb]));
            const float v10 = sqrtf(float(f[size_t(yb) * a.pitch + xa]));
            const float v11 = sqrtf(float(f[size_t(yb) * a.pitch + xb]));
            const float val = (1.f - wy) * ((1.f - wx) * v00 + wx * v01) + wy * ((1.f - wx) * v10 + wx * v11);
            x = make_float2(((i + j) & 1) ? -val : val, 0.f);
        } else if (COLS) {
            x = a.src[base + size_t(e) * NL + l0 + line];
        } else {
            const int i = l0 + line;
            x = a.src[base + size_t(i) * NL + e];
            if (WHICH == 2 && ((i + e) & 1)) x = cneg(x);
        }
        s0[line * NL + e] = x;
    }
    __syncthreads();
    const float2* res = stockham<NL, INV>(s0, s1, LPB, a.tw);
    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        if (COLS) {
            const int e = idx / LPB, line = idx - e * LPB;
            const int i = e, j = l0 + line;
            float2 x = res[line * NL + e];
            const float sc = ((i + j) & 1) ? -a.scale : a.scale;
            const size_t o = (WHICH == 3 && a.out_off) ? size_t(a.out_off[tile]) + size_t(i) * a.out_pitch + j
                                                       : base + size_t(i) * NL + j;
            a.dst[o] = cscale(x, sc);
        } else {
            const int line = idx / NL, e = idx - line * NL;
            a.dst[base + size_t(l0 + line) * NL + e] = res[line * NL + e];
        }
    }
}

// N = 256 lines with one warp per line: the block stages LPB lines in shared
// memory exactly as lines_fft does (coalesced global traffic), then each warp
// runs a register/shuffle 256-point FFT (WarpFFT<8>, F1: natural order in,
// natural order out through the padded layout) instead of four Stockham
// passes through shared memory. Inverse transforms run as conj(FFT(conj x)).
// Padded line layout: element i at i + i / 32 (conflict-free for both the
// lane-strided reads and the digit-reversed writes of F1).
template <int WHICH>
__global__ void __launch_bounds__(512) lines_fft_w256(const LinesArgs a) {
    constexpr int NL = 256, LPB = 16, M = 8, LS = NL + NL / 32 + 1;  // odd in float2 pairs: column phases conflict-free
    constexpr bool INV = WHICH >= 2;
    constexpr bool COLS = (WHICH & 1) == 1;
    __shared__ float2 s[LPB * LS];
    __shared__ float2 tw_s[NL];  // the twiddle table, staged once per block (the warp FFTs' per-lane constants)
    for (int k = threadIdx.x; k < NL; k += blockDim.x) tw_s[k] = a.tw[k];
    const int tile = blockIdx.y;
    const int l0 = blockIdx.x * LPB;
    const size_t base = size_t(tile) * NL * NL;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    auto pad = [](int i) { return i + (i >> 5); };
    // init rows: sqrt of the seed-crop rows this block's 16 output rows interpolate
    // from, once per crop pixel instead of four times per output pixel
    constexpr int kSq = 1280;
    __shared__ float sq[WHICH == 0 ? kSq : 1];
    int sq_r0 = 0;
    bool sq_on = false;
    if (WHICH == 0) {
        const int n = a.n;
        const int ya0 = max(int(floorf((l0 + 0.5f) / a.up - 0.5f)), 0);
        const int yb1 = min(int(floorf((l0 + LPB - 1 + 0.5f) / a.up - 0.5f)) + 1, n - 1);
        sq_r0 = ya0;
        sq_on = (yb1 - ya0 + 1) * n <= kSq;
        if (sq_on) {
            const int2 txy = a.tile_xy[tile];
            const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
            for (int k = threadIdx.x; k < (yb1 - ya0 + 1) * n; k += blockDim.x) {
                const int r = k / n, c = k - r * n;
                sq[k] = sqrtf(float(f[size_t(ya0 + r) * a.pitch + c]));
            }
        }
        __syncthreads();
    }

    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        int line, e;
        if (COLS) {
            e = idx / LPB;
            line = idx - e * LPB;
        } else {
            line = idx / NL;
            e = idx - line * NL;
        }
        float2 x;
        if (WHICH == 0) {
            // upsample_bilinear (field.cpp:89-112) of the seed crop's sqrt, pixel-centre mapped
            const int i = l0 + line, j = e, n = a.n;
            const float fy = (i + 0.5f) / a.up - 0.5f, fx = (j + 0.5f) / a.up - 0.5f;
            int ya = int(floorf(fy)), xa = int(floorf(fx));
            const float wy = fy - ya, wx = fx - xa;
            const int yb = min(ya + 1, n - 1), xb = min(xa + 1, n - 1);
            ya = max(ya, 0);
            xa = max(xa, 0);
            float v00, v01, v10, v11;
            if (sq_on) {
                const float* q0 = sq + (ya - sq_r0) * n;
                const float* q1 = sq + (yb - sq_r0) * n;
                v00 = q0[xa];
                v01 = q0[xb];
                v10 = q1[xa];
                v11 = q1[xb];
            } else {
                const int2 txy = a.tile_xy[tile];
                const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
                v00 = sqrtf(float(f[size_t(ya) * a.pitch + xa]));
                v01 = sqrtf(float(f[size_t(ya) * a.pitch + xb]));
                v10 = sqrtf(float(f[size_t(yb) * a.pitch + xa]));
                v11 = sqrtf(float(f[size_t(yb) * a.pitch + xb]));
            }
            const float val = (1.f - wy) * ((1.f - wx) * v00 + wx * v01) + wy * ((1.f - wx) * v10 + wx * v11);
            x = make_float2(((i + j) & 1) ? -val : val, 0.f);
        } else if (COLS) {
            x = a.src[base + size_t(e) * NL + l0 + line];
        } else {
            const int i = l0 + line;
            x = a.src[base + size_t(i) * NL + e];
            if (WHICH == 2 && ((i + e) & 1)) x = cneg(x);
        }
        if (INV) x.y = -x.y;
        s[line * LS + pad(e)] = x;
    }
    __syncthreads();
    {
        WarpFFT<M> F;
        F.init_smem(l, NL, tw_s);
        float2* ln = s + w * LS;
        float2 x[M];
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = ln[pad(l + 32 * m)];
        F.f1(x);  // all lanes have read before the shuffles of f1 complete
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) ln[pad(k0 + M * brev5(l))] = x[k0];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        if (COLS) {
            const int e = idx / LPB, line = idx - e * LPB;
            const int i = e, j = l0 + line;
            float2 x = s[line * LS + pad(e)];
            if (INV) x.y = -x.y;
            const float sc = ((i + j) & 1) ? -a.scale : a.scale;
            const size_t o = (WHICH == 3 && a.out_off) ? size_t(a.out_off[tile]) + size_t(i) * a.out_pitch + j
                                                       : base + size_t(i) * NL + j;
            a.dst[o] = cscale(x, sc);
        } else {
            const int line = idx / NL, e = idx - line * NL;
            float2 x = s[line * LS + pad(e)];
            if (INV) x.y = -x.y;
            a.dst[base + size_t(l0 + line) * NL + e] = x;
        }
    }
}

// Box-pruned N = 256 passes (see LinesArgs): the same warp FFT and staging as
// lines_fft_w256, over fewer lines and with zero / skipped ranges:
//   0 init rows:  all 256 rows of bilinear(sqrt(seed)) * C -> FFT -> box columns only
//   1 init cols:  box columns, all rows -> FFT -> box rows * C / up^2 -> canvas and canvas0
//   2 final rows: box rows, input (canvas - canvas0) * C on box columns, 0 elsewhere -> IFFT
//                 -> the whole row back into the canvas
//   3 final cols: all columns, input the box rows (0 elsewhere) -> IFFT -> * C up^2 / N^2
//                 + bilinear(sqrt(seed)) -> dst (or the mosaic via out_off)
__device__ __forceinline__ float seed_bilinear(const LinesArgs& a, int tile, int i, int j) {
    const int n = a.n;
    const float fy = (i + 0.5f) / a.up - 0.5f, fx = (j + 0.5f) / a.up - 0.5f;
    int ya = int(floorf(fy)), xa = int(floorf(fx));
    const float wy = fy - ya, wx = fx - xa;
    const int yb = min(ya + 1, n - 1), xb = min(xa + 1, n - 1);
    ya = max(ya, 0);
    xa = max(xa, 0);
    const int2 txy = a.tile_xy[tile];
    const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
    const float v00 = sqrtf(float(f[size_t(ya) * a.pitch + xa]));
    const float v01 = sqrtf(float(f[size_t(ya) * a.pitch + xb]));
    const float v10 = sqrtf(float(f[size_t(yb) * a.pitch + xa]));
    const float v11 = sqrtf(float(f[size_t(yb) * a.pitch + xb]));
    return (1.f - wy) * ((1.f - wx) * v00 + wx * v01) + wy * ((1.f - wx) * v10 + wx * v11);
}

#ifndef FPM_LINES_BOX_MINB
#define FPM_LINES_BOX_MINB 3  // resident 512-thread blocks per SM the register budget targets
#endif
template <int WHICH>
__global__ void __launch_bounds__(512, FPM_LINES_BOX_MINB) lines_box_w256(const LinesArgs a) {
    constexpr int NL = 256, LPB = 16, M = 8, LS = NL + NL / 32 + 1;  // odd in float2 pairs: column phases conflict-free
    constexpr bool INV = WHICH >= 2;
    constexpr bool COLS = (WHICH & 1) == 1;
    __shared__ float2 s[LPB * LS];
    __shared__ float2 tw_s[NL];  // the twiddle table, staged once per block (the warp FFTs' per-lane constants)
    for (int k = threadIdx.x; k < NL; k += blockDim.x) tw_s[k] = a.tw[k];
    const int tile = blockIdx.y;
    const int b0 = a.box0, bn = a.boxn;
    const int l0 = (WHICH == 1 || WHICH == 2 ? b0 : 0) + blockIdx.x * LPB;  // first line of the block
    const size_t base = size_t(tile) * NL * NL;
    float2* c0 = a.canvas0 + size_t(tile) * bn * bn;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    auto pad = [](int i) { return i + (i >> 5); };
    auto in_box = [&](int x) { return x >= b0 && x < b0 + bn; };
    // sqrt of the seed-crop window the block's bilinear samples read (init rows: <= 6 LR rows
    // x n columns; final cols: n rows x <= 6 LR columns), staged once
    constexpr int kSq = 1536;
    __shared__ float sq[(WHICH == 0 || WHICH == 3) ? kSq : 1];
    __shared__ int2 rowab[WHICH == 3 ? NL : 1];
    __shared__ float rowwy[WHICH == 3 ? NL : 1];
    int wy0 = 0, wx0 = 0, wsw = 0;
    bool sq_on = false;
    auto lr_lo = [&](int hr0) { return max(int(floorf((hr0 + 0.5f) / a.up - 0.5f)), 0); };
    auto lr_hi = [&](int hr1) { return min(int(floorf((hr1 + 0.5f) / a.up - 0.5f)) + 1, a.n - 1); };
    if (WHICH == 0 || WHICH == 3) {
        const int n = a.n;
        int wy1, wx1;
        if (WHICH == 0) {
            wy0 = lr_lo(l0);
            wy1 = lr_hi(l0 + LPB - 1);
            wx0 = 0;
            wx1 = n - 1;
        } else {
            wy0 = 0;
            wy1 = n - 1;
            wx0 = lr_lo(l0);
            wx1 = lr_hi(l0 + LPB - 1);
        }
        wsw = wx1 - wx0 + 1;
        sq_on = (wy1 - wy0 + 1) * wsw <= kSq;
        if (WHICH == 3) {  // per output row: sq offsets of its two LR taps and the y weight
            for (int k = threadIdx.x; k < NL; k += blockDim.x) {
                const float fy = (k + 0.5f) / a.up - 0.5f;
                int ya = int(floorf(fy));
                rowwy[k] = fy - ya;
                const int yb = min(ya + 1, n - 1) - wy0;
                ya = max(ya, 0) - wy0;
                rowab[k] = make_int2(ya * wsw, yb * wsw);
            }
        }
        if (sq_on) {
            const int2 txy = a.tile_xy[tile];
            const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
            for (int k = threadIdx.x; k < (wy1 - wy0 + 1) * wsw; k += blockDim.x) {
                const int r = k / wsw, c = k - r * wsw;
                sq[k] = sqrtf(float(f[size_t(wy0 + r) * a.pitch + wx0 + c]));
            }
        }
        __syncthreads();
    }
    auto bilinear = [&](int i, int j) -> float {  // upsample_bilinear (field.cpp:89-112)
        if (!sq_on) return seed_bilinear(a, tile, i, j);
        const int n = a.n;
        const float fy = (i + 0.5f) / a.up - 0.5f, fx = (j + 0.5f) / a.up - 0.5f;
        int ya = int(floorf(fy)), xa = int(floorf(fx));
        const float wy = fy - ya, wx = fx - xa;
        const int yb = min(ya + 1, n - 1), xb = min(xa + 1, n - 1);
        ya = max(ya, 0);
        xa = max(xa, 0);
        const float* q0 = sq + (ya - wy0) * wsw - wx0;
        const float* q1 = sq + (yb - wy0) * wsw - wx0;
        return (1.f - wy) * ((1.f - wx) * q0[xa] + wx * q0[xb]) + wy * ((1.f - wx) * q1[xa] + wx * q1[xb]);
    };
    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        int line, e;
        if (COLS) {
            e = idx / LPB;
            line = idx - e * LPB;
        } else {
            line = idx / NL;
            e = idx - line * NL;
        }
        float2 x = make_float2(0.f, 0.f);
        if (WHICH == 0) {
            const int i = l0 + line, j = e;
            const float val = bilinear(i, j);
            x = make_float2(((i + j) & 1) ? -val : val, 0.f);
        } else if (WHICH == 1) {
            x = a.src[base + size_t(e) * NL + l0 + line];
        } else if (WHICH == 2) {
            const int i = l0 + line;
            if (in_box(e)) {
                x = csub(a.src[base + size_t(i) * NL + e], c0[size_t(i - b0) * bn + (e - b0)]);
                if ((i + e) & 1) x = cneg(x);
            }
        } else {
            if (in_box(e)) x = a.src[base + size_t(e) * NL + l0 + line];
        }
        if (INV) x.y = -x.y;
        s[line * LS + pad(e)] = x;
    }
    __syncthreads();
    {
        WarpFFT<M> F;
        F.init_smem(l, NL, tw_s);
        float2* ln = s + w * LS;
        float2 x[M];
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = ln[pad(l + 32 * m)];
        F.f1(x);
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) ln[pad(k0 + M * brev5(l))] = x[k0];
    }
    __syncthreads();
    if (WHICH == 3 && sq_on) {
        // final cols: a thread keeps one column (its bilinear x weights) over every 32nd row
        const int line = threadIdx.x & (LPB - 1), j = l0 + line, n = a.n;
        const float fx = (j + 0.5f) / a.up - 0.5f;
        int xa = int(floorf(fx));
        const float wx = fx - xa;
        const int xb = min(xa + 1, n - 1) - wx0;
        xa = max(xa, 0) - wx0;
        const size_t obase = a.out_off ? size_t(a.out_off[tile]) + j : base + j;
        const size_t opitch = a.out_off ? size_t(a.out_pitch) : size_t(NL);
        for (int i = threadIdx.x / LPB; i < NL; i += blockDim.x / LPB) {
            float2 x = s[line * LS + pad(i)];
            const float sc = ((i + j) & 1) ? -a.scale : a.scale;
            x = cscale(make_float2(x.x, -x.y), sc);  // conj folded into one FMUL2
            const int2 yab = rowab[i];  // the row's bilinear taps and weight (staged once per block)
            const float wy = rowwy[i];
            const float* q0 = sq + yab.x;
            const float* q1 = sq + yab.y;
            x.x += (1.f - wy) * ((1.f - wx) * q0[xa] + wx * q0[xb]) + wy * ((1.f - wx) * q1[xa] + wx * q1[xb]);
            a.dst[obase + size_t(i) * opitch] = x;
        }
        return;
    }
    for (int idx = threadIdx.x; idx < LPB * NL; idx += blockDim.x) {
        if (COLS) {
            const int e = idx / LPB, line = idx - e * LPB;
            const int i = e, j = l0 + line;
            if (WHICH == 1 && !in_box(i)) continue;
            float2 x = s[line * LS + pad(e)];
            if (INV) x.y = -x.y;
            const float sc = ((i + j) & 1) ? -a.scale : a.scale;
            x = cscale(x, sc);
            if (WHICH == 1) {
                a.dst[base + size_t(i) * NL + j] = x;
                c0[size_t(i - b0) * bn + (j - b0)] = x;
            } else {
                x.x += bilinear(i, j);
                const size_t o = a.out_off ? size_t(a.out_off[tile]) + size_t(i) * a.out_pitch + j
                                           : base + size_t(i) * NL + j;
                a.dst[o] = x;
            }
        } else {
            const int line = idx / NL, e = idx - line * NL;
            if (WHICH == 0 && !in_box(e)) continue;
            float2 x = s[line * LS + pad(e)];
            if (INV) x.y = -x.y;
            a.dst[base + size_t(l0 + line) * NL + e] = x;
        }
    }
}

// Box init rows, separably: U(i, j) = (1 - wy_i) h_ya(j) + wy_i h_yb(j), h_y the
// horizontal bilinear interpolation of sqrt(seed) LR row y, so the row spectrum
// FFT_j(C U(i, .)) = (-1)^i [(1 - wy_i) G_ya + wy_i G_yb] with G_y = FFT_j((-1)^j h_y):
// a block of 32 HR rows transforms the <= 10 LR rows they interpolate from (one warp
// each) instead of 32 HR rows, and writes the box columns of its 32 rows.
__global__ void __launch_bounds__(512) lines_box_init_rows(const LinesArgs a) {
    constexpr int NL = 256, RB = 32, MAXLR = 16, M = 8, LS = NL + NL / 32;
    __shared__ float2 s[MAXLR * LS];
    __shared__ float2 tw_s[NL];
    for (int k = threadIdx.x; k < NL; k += blockDim.x) tw_s[k] = a.tw[k];
    const int tile = blockIdx.y, i0 = blockIdx.x * RB;
    const int b0 = a.box0, bn = a.boxn, n = a.n, up = a.up;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    auto pad = [](int i) { return i + (i >> 5); };
    auto lr_of = [&](int i) { return max(int(floorf((i + 0.5f) / up - 0.5f)), 0); };
    const int y0 = lr_of(i0), y1 = min(lr_of(i0 + RB - 1) + 1, n - 1);
    const int ny = y1 - y0 + 1;  // <= 10 for up = 4 (checked by the launcher's shape)
    const int2 txy = a.tile_xy[tile];
    const uint16_t* f = a.frame + size_t(txy.y) * a.pitch + txy.x;
    // h_y(j) (-1)^j for the block's LR rows
    for (int idx = threadIdx.x; idx < ny * NL; idx += blockDim.x) {
        const int r = idx / NL, j = idx - r * NL, y = y0 + r;
        const float fx = (j + 0.5f) / up - 0.5f;
        int xa = int(floorf(fx));
        const float wx = fx - xa;
        const int xb = min(xa + 1, n - 1);
        xa = max(xa, 0);
        const float v = (1.f - wx) * sqrtf(float(f[size_t(y) * a.pitch + xa])) + wx * sqrtf(float(f[size_t(y) * a.pitch + xb]));
        s[r * LS + pad(j)] = make_float2((j & 1) ? -v : v, 0.f);
    }
    __syncthreads();
    if (w < ny) {
        WarpFFT<M> F;
        F.init_smem(l, NL, tw_s);
        float2* ln = s + w * LS;
        float2 x[M];
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = ln[pad(l + 32 * m)];
        F.f1(x);
#pragma unroll
        for (int k0 = 0; k0 < M; ++k0) ln[pad(k0 + M * brev5(l))] = x[k0];
    }
    __syncthreads();
    const size_t base = size_t(tile) * NL * NL;
    for (int idx = threadIdx.x; idx < RB * bn; idx += blockDim.x) {
        const int r = idx / bn, k = b0 + (idx - r * bn), i = i0 + r;
        const float fy = (i + 0.5f) / up - 0.5f;
        int ya = int(floorf(fy));
        const float wy = fy - ya;
        const int yb = min(ya + 1, n - 1);
        ya = max(ya, 0);
        const float2 ga = s[(ya - y0) * LS + pad(k)], gb = s[(yb - y0) * LS + pad(k)];
        const float sg = (i & 1) ? -1.f : 1.f;
        a.dst[base + size_t(i) * NL + k] = make_float2(sg * ((1.f - wy) * ga.x + wy * gb.x), sg * ((1.f - wy) * ga.y + wy * gb.y));
    }
}

template <int NL, int LPB, int WHICH>
cudaError_t launch_lines_t(const LinesArgs& a, int T, cudaStream_t s) {
    const size_t smem = size_t(2) * LPB * NL * sizeof(float2);
    auto k = lines_fft<NL, LPB, WHICH>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<dim3(NL / LPB, T), 256, smem, s>>>(a);
    return cudaGetLastError();
}

template <int NL, int LPB>
cudaError_t launch_lines_n(int which, const LinesArgs& a, int T, cudaStream_t s) {
    switch (which) {
        case 0: return launch_lines_t<NL, LPB, 0>(a, T, s);
        case 1: return launch_lines_t<NL, LPB, 1>(a, T, s);
        case 2: return launch_lines_t<NL, LPB, 2>(a, T, s);
        case 3: return launch_lines_t<NL, LPB, 3>(a, T, s);
    }
    return cudaErrorInvalidValue;
}

__global__ void build_pupils_kernel(float2* pupils, const uint8_t* support, const double* defocus, int n,
                                    int T, double dk, double inv_l2) {
    const size_t total = size_t(T) * n * n;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total; idx += size_t(gridDim.x) * blockDim.x) {
        const int t = int(idx / (size_t(n) * n));
        const int p = int(idx % (size_t(n) * n));
        const int i = p / n, j = p % n;
        float2 v = make_float2(0.f, 0.f);
        if (support[p]) {
            const double z = defocus ? defocus[t] : 0.0;
            if (z == 0.0) {
                v = make_float2(1.f, 0.f);
            } else {  // angular-spectrum defocus phase (optics.cpp:63-67)
                const double rho = hypot(double(i - n / 2), double(j - n / 2));
                const double kz = sqrt(fmax(0.0, inv_l2 - rho * dk * rho * dk));
                double sn, cs;
                sincos(2.0 * 3.14159265358979323846 * z * kz, &sn, &cs);
                v = make_float2(float(cs), float(sn));
            }
        }
        pupils[idx] = v;
    }
}

// FPM_B200_LINES_STOCKHAM=1 keeps N = 256 on the shared-memory Stockham kernel (cross-checks)
bool lines_stockham_forced() {
    const char* e = std::getenv("FPM_B200_LINES_STOCKHAM");
    return e && e[0] == '1';
}

}  // namespace

cudaError_t launch_lines(int which, int N, const LinesArgs& a, int T, cudaStream_t s) {
    if (N == 256 && !lines_stockham_forced()) {
        const dim3 grid(256 / 16, T);
        switch (which) {
            case 0: lines_fft_w256<0><<<grid, 512, 0, s>>>(a); break;
            case 1: lines_fft_w256<1><<<grid, 512, 0, s>>>(a); break;
            case 2: lines_fft_w256<2><<<grid, 512, 0, s>>>(a); break;
            case 3: lines_fft_w256<3><<<grid, 512, 0, s>>>(a); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    switch (N) {
        case 256: return launch_lines_n<256, 16>(which, a, T, s);
        case 512: return launch_lines_n<512, 8>(which, a, T, s);
        case 1024: return launch_lines_n<1024, 4>(which, a, T, s);
    }
    return cudaErrorNotSupported;  // no line-FFT instantiation for this side
}

cudaError_t launch_lines_box(int which, const LinesArgs& a, int T, cudaStream_t s) {
    if (a.boxn <= 0 || a.boxn % 16 || a.box0 % 16 || a.box0 < 0 || a.box0 + a.boxn > 256) return cudaErrorInvalidValue;
    const int blocks = (which == 1 || which == 2) ? a.boxn / 16 : 256 / 16;
    const dim3 grid(blocks, T);
    // the separable init rows need <= 16 LR rows per 32 HR rows (upsample >= 3)
    const bool sep = a.up >= 3 && std::getenv("FPM_B200_INIT_SEP") == nullptr;
    switch (which) {
        case 0:
            if (sep)
                lines_box_init_rows<<<dim3(256 / 32, T), 512, 0, s>>>(a);
            else
                lines_box_w256<0><<<grid, 512, 0, s>>>(a);
            break;
        case 1: lines_box_w256<1><<<grid, 512, 0, s>>>(a); break;
        case 2: lines_box_w256<2><<<grid, 512, 0, s>>>(a); break;
        case 3: lines_box_w256<3><<<grid, 512, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_build_pupils(float2* pupils, const uint8_t* support, const double* defocus, int n, int T,
                                double dk, double inv_l2, cudaStream_t s) {
    const size_t total = size_t(T) * n * n;
    const int blocks = int(std::min<size_t>((total + 255) / 256, 148 * 16));
    build_pupils_kernel<<<blocks, 256, 0, s>>>(pupils, support, defocus, n, T, dk, inv_l2);
    return cudaGetLastError();
}

}  // namespace fpmk
