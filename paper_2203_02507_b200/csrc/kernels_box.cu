// fpm_loop_box: the fused per-LED update for LR tile sides n = 32 M (128, 256),
// persistent over the LED loop like fpm_loop64, one CTA of 16 warps per tile.
//
// Every 1-D n-point FFT is done by one warp: a register DFT_M (M = n / 32) and
// a 32-point DFT across the lanes (5 radix-2 stages over shuffles). Two warp
// FFT flavours chain without any reordering:
//   F1: x[l + 32 m] (lane l, register m)      -> X[k0 + M br5(l)] (register k0)
//       (register DFT, twiddle W_n^(l k0), lane DFT by decimation in frequency)
//   F2: x[k0 + M br5(l)]                      -> X[q + 32 r] (lane q, register r)
//       (lane DFT by decimation in time, twiddle W_n^(k0 q), register DFT)
// The 2-D centred transforms only visit the pupil's bounding box (rows/cols
// [b0, b0 + B)), which holds every nonzero IFFT input and every FFT output the
// scatter needs (update_step touches the disk only, recon.cpp:107-130):
//   A  IFFT of the B box rows (F2, gathered from the canvas disk x P')
//   B  per column: IFFT (F1) over the B nonzero rows -> modulus with sqrt(I)
//      -> FFT (F2) -> keep the B box rows
//   C  FFT of the B box rows (F1) -> scatter into the disk (GS / EPRY)
// The B x n intermediate lives in shared memory (n = 128: 60 KB) or in a
// per-tile global scratch (n = 256: 240 KB, L2-resident). Row stride n + 1
// keeps every column access conflict-free; the staged measurement is
// XOR-swizzled so the modulus reads (rows k0 + M t) hit 32 distinct banks.
#include "kernels.cuh"
#include "warp_fft.cuh"

namespace fpmk {

namespace {

constexpr int kBoxThreads = 512;
constexpr int kBoxWarps = kBoxThreads / 32;

}  // namespace

size_t box_smem_bytes(int n, int box, int L, int iters, bool scratch_in_smem) {
    size_t b = size_t(n) * n * sizeof(uint16_t);                     // swizzled measurement
    if (scratch_in_smem) b += size_t(box) * (n + 1) * sizeof(float2);  // box-row intermediate
    b += size_t(iters) * sizeof(double) + 16;
    b += size_t(kBoxWarps) * 4 * sizeof(float);
    b += size_t(L) * (sizeof(short2) + sizeof(int) + 1) + 16;
    b = (b + 15) & ~size_t(15);
    if (n == 256) b += size_t(kBoxWarps) * WarpFFT256<false>::kBufFloat2 * sizeof(float2);  // FFT transposes
    return b;
}

template <int NLR, int MODE, int NC, bool SMEM_S, bool JIT, bool MID>
__global__ void __launch_bounds__(kBoxThreads, 1) fpm_loop_box(const LoopArgs args, BoxArgs bx) {
    constexpr int M = NLR / 32;
    constexpr int RS = NLR + 1;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int tile = blockIdx.x;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int L = args.L, B = bx.box, b0 = bx.b0;
    uint8_t* sp = smem_raw;
    uint16_t* I_s = reinterpret_cast<uint16_t*>(sp);
    sp += size_t(NLR) * NLR * sizeof(uint16_t);
    float2* S = nullptr;
    if constexpr (SMEM_S) {
        S = reinterpret_cast<float2*>(sp);
        sp += size_t(B) * RS * sizeof(float2);
    } else {
        S = bx.scratch + size_t(tile) * B * RS;
    }
    double* stage_sum = reinterpret_cast<double*>(sp);
    sp += size_t(args.iters) * sizeof(double) + 16;
    float* red = reinterpret_cast<float*>(sp);  // [warp][4]: num, den, omax, pmax
    sp += size_t(kBoxWarps) * 4 * sizeof(float);
    short2* O_s = reinterpret_cast<short2*>(sp);
    sp += size_t(L) * sizeof(short2);
    int* F_s = reinterpret_cast<int*>(sp);
    sp += size_t(L) * sizeof(int);
    uint8_t* B_s = sp;
    sp += size_t(L);
    sp = smem_raw + ((sp - smem_raw + 15) & ~15);
    using FFT = typename WarpFFTSel<M, MID>::type;
    float2* TB = reinterpret_cast<float2*>(sp) + size_t(w) * FFT::kBufFloat2;  // n = 256: this warp's transpose buffer

    float2* canvas = args.canvas + size_t(tile) * NC * NC;
    float2* pupil = args.pupils + size_t(tile) * NLR * NLR;
    const uint8_t* sup = args.support;
    const int2 txy = args.tile_xy[tile];
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        O_s[k] = args.origins[size_t(tile) * L + k];
        F_s[k] = args.seq_frame[k];
        B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
    }
    for (int k = threadIdx.x; k < args.iters; k += blockDim.x) stage_sum[k] = 0.0;
    FFT F;
    F.init(l, NLR, TB);
    const float inv_n2 = 1.0f / float(NLR * NLR);
    __syncthreads();

    // sequential: slot s = (s / L, s % L); pipelined: the slot's entries run back to back on
    // the whole CTA — they touch disjoint disks, so any order equals the concurrent one
    const int G = args.slots ? 2 : 1;
    for (int e = args.slot_begin * G; e < args.num_slots * G; ++e) {
        jitter_sleep<JIT>(args, e);
        int it, pos;
        if (G == 1) {
            it = e / L;
            pos = e % L;
        } else {
            const int2 en = args.slots[e];
            if (en.x < 0) continue;
            it = en.x;
            pos = en.y;
        }
        const short2 o = O_s[pos];
        FPM_ASSERT(tile < args.T && pos >= 0 && pos < L && it >= 0 && it < args.iters && o.x >= 0 && o.y >= 0 &&
                   o.x + NLR <= NC && o.y + NLR <= NC && F_s[pos] >= 0 && (args.F == 0 || F_s[pos] < args.F));
        const float2* cvc = canvas + size_t(o.x) * NC + o.y;
        float2* cv = canvas + size_t(o.x) * NC + o.y;

        // ---- stage the measurement crop, column index XOR 2 (row / M): the modulus
        // reads rows k0 + M t across the lanes, which then fall in 32 distinct banks
        if (args.meas_f32 == nullptr) {
            const uint16_t* fr = bx.frames + size_t(F_s[pos]) * bx.frame_stride + size_t(txy.y) * bx.pitch + txy.x;
            for (int idx = threadIdx.x; idx < NLR * NLR; idx += kBoxThreads) {
                const int r = idx / NLR, c = idx % NLR;
                I_s[r * NLR + (c ^ FFT::isw(r))] = fr[size_t(r) * bx.pitch + c];
            }
        }

        // ---- A: IFFT of the box rows of the disk block (gather x P x checkerboard)
        float omax = 0.f, pmax = 0.f;
        for (int i = b0 + w; i < b0 + B; i += kBoxWarps) {
            float2 x[M];
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int c = F.a_in(k0);
                float2 v = make_float2(0.f, 0.f);
                if (FFT::live(k0) && sup[i * NLR + c]) {
                    const float2 O = cvc[size_t(i) * NC + c];
                    const float2 P = pupil[i * NLR + c];
                    const float2 g = cmul(O, P);  // conj, signed: the row IFFT runs as conj(FFT(conj g))
                    v = ((i + c) & 1) ? make_float2(-g.x, g.y) : make_float2(g.x, -g.y);
                    if (MODE == kModeEPRY) {
                        omax = fmaxf(omax, cabs2(O));
                        pmax = fmaxf(pmax, cabs2(P));
                    }
                }
                x[k0] = v;
            }
            F.fA(x);  // S keeps conj(IFFT_rows(g)): phase B's forward column FFT undoes it
#pragma unroll
            for (int r = 0; r < M; ++r) S[size_t(i - b0) * RS + F.a_out(r)] = x[r];
        }
        if (MODE == kModeEPRY) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                omax = fmaxf(omax, __shfl_xor_sync(kFull, omax, sh));
                pmax = fmaxf(pmax, __shfl_xor_sync(kFull, pmax, sh));
            }
            if (l == 0) {
                red[w * 4 + 2] = omax;
                red[w * 4 + 3] = pmax;
            }
        }
        __syncthreads();

        // ---- B: per column, IFFT over the box rows -> modulus -> FFT -> keep the box rows
        float num = 0.f, den = 0.f;
        for (int j = w; j < NLR; j += kBoxWarps) {
            float2 x[M];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const int r = F.nat(m);
                x[m] = (FFT::live(m) && r >= b0 && r < b0 + B) ? S[size_t(r - b0) * RS + j] : make_float2(0.f, 0.f);
            }
            F.f1(x);  // = conj(e), e the unscaled 2-D IFFT
            const uint16_t* Ic = I_s + (j ^ F.isw_lane());  // one column swizzle per lane
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int row = F.scr(k0);
                float Iv;
                if (args.meas_f32 == nullptr) {
                    Iv = float(Ic[row * NLR]);
                } else {
                    Iv = args.meas_f32[row * NLR + j];
                }
                den += Iv;
                // |e| = 0 rule (recon.cpp:122) as in fpm_loop64: Re nudged by sgn 2^-60 maps
                // e = 0 to e' = sgn sqrt(I) (checkerboard sign), leaves |Re| >= 2^-35 exact
                const float meas = sqrt_ftz(Iv);
                const float2 u = x[k0];
                const float ux = u.x + (((row + j) & 1) ? -0x1p-60f : 0x1p-60f);
                const float m2 = fmaf(ux, ux, u.y * u.y);
                const float rr = rsqrt_ftz(fmaxf(m2, kTiny));
                const float dm = fmaf(m2 * rr, inv_n2, -meas);
                num = fmaf(dm, dm, num);
                const float sc = meas * rr;
                x[k0] = make_float2(ux * sc, -u.y * sc);  // e' from u = conj(e)
            }
            F.f2(x);
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const int row = F.nat(r);
                if (FFT::live(r) && row >= b0 && row < b0 + B) S[size_t(row - b0) * RS + j] = x[r];
            }
        }
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) {
            num += __shfl_xor_sync(kFull, num, sh);
            den += __shfl_xor_sync(kFull, den, sh);
        }
        if (l == 0) {
            red[w * 4] = num;
            red[w * 4 + 1] = den;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float nsum = 0.f, dsum = 0.f;
            for (int k = 0; k < kBoxWarps; ++k) {
                nsum += red[k * 4];
                dsum += red[k * 4 + 1];
            }
            stage_sum[it] += dsum > 0.f ? double(__fdividef(nsum, dsum)) : 0.0;  // as fpm_loop64
        }
        float inv_omax = 0.f, inv_pmax = 0.f;
        if (MODE == kModeEPRY) {
            float om = 0.f, pm = 0.f;
            for (int k = 0; k < kBoxWarps; ++k) {
                om = fmaxf(om, red[k * 4 + 2]);
                pm = fmaxf(pm, red[k * 4 + 3]);
            }
            inv_omax = (om > 0.f && B_s[pos]) ? args.beta / om : 0.f;  // bright-field pupil steps only
            inv_pmax = pm > 0.f ? args.alpha / pm : 0.f;
        }

        // ---- C: FFT of the box rows, scatter into the disk (recon.cpp:127-130) / EPRY
        for (int i = b0 + w; i < b0 + B; i += kBoxWarps) {
            float2 x[M];
#pragma unroll
            for (int m = 0; m < M; ++m) x[m] = S[size_t(i - b0) * RS + F.c_in(m)];
            F.fC(x);
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int c = F.c_out(k0);
                if (!FFT::live(k0) || !sup[i * NLR + c]) continue;
                const float2 psi2 = cscale(x[k0], ((i + c) & 1) ? -1.f : 1.f);
                float2* dst = cv + size_t(i) * NC + c;
                float2* pp = pupil + i * NLR + c;
                const float2 P = *pp;
                if (MODE == kModeGS) {
                    *dst = cmulc(psi2, P);
                } else {
                    const float2 O = *dst;
                    const float2 d = csub(psi2, cmul(O, P));
                    if (inv_pmax > 0.f) *dst = cadd(O, cscale(cmulc(d, P), inv_pmax));
                    if (inv_omax > 0.f) *pp = cadd(P, cscale(cmulc(d, O), inv_omax));
                }
            }
        }
        __syncthreads();  // canvas, pupil and reductions settled before the next update
    }
    store_residuals(args, tile, stage_sum, G == 1);
}

template <int NLR, int MODE, int NC, bool SMEM_S>
static cudaError_t launch_box_t(const LoopArgs& a, const BoxArgs& b, int T, cudaStream_t s) {
    const size_t smem = box_smem_bytes(NLR, b.box, a.L, a.iters, SMEM_S);
    auto k = a.jitter > 0 ? fpm_loop_box<NLR, MODE, NC, SMEM_S, true, false> : fpm_loop_box<NLR, MODE, NC, SMEM_S, false, false>;
    if constexpr (NLR == 256) {  // the support box inside [64, 192): WarpFFT256 pruned to registers 2..5
        if (b.b0 >= 64 && b.b0 + b.box <= 192 && !mid_disabled())
            k = a.jitter > 0 ? fpm_loop_box<NLR, MODE, NC, SMEM_S, true, true> : fpm_loop_box<NLR, MODE, NC, SMEM_S, false, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<T, kBoxThreads, smem, s>>>(a, b);
    return cudaGetLastError();
}

cudaError_t launch_loop_box(int n, int mode, const LoopArgs& a, const BoxArgs& b, int T, cudaStream_t s) {
#define FPM_BOX_CASE(NN, MM, NCC, SM)                       \
    if (n == NN && mode == MM && a.N == NCC)               \
        return launch_box_t<NN, MM, NCC, SM>(a, b, T, s);
    FPM_BOX_CASE(128, kModeGS, 512, true)
    FPM_BOX_CASE(128, kModeEPRY, 512, true)
    FPM_BOX_CASE(128, kModeGS, 1024, true)
    FPM_BOX_CASE(128, kModeEPRY, 1024, true)
    FPM_BOX_CASE(256, kModeGS, 1024, false)
    FPM_BOX_CASE(256, kModeEPRY, 1024, false)
    FPM_BOX_CASE(64, kModeGS, 256, true)
    FPM_BOX_CASE(64, kModeEPRY, 256, true)
#undef FPM_BOX_CASE
    return cudaErrorNotSupported;  // no instantiation for this geometry
}

}  // namespace fpmk
