// sm_100a kernels of the FPM engine.
//
// K1+K4  fpm_loop64    one CTA per tile runs every (iteration, LED) update of
//                      reconstruct_tile (recon.cpp:161-166) back to back; the
//                      fused update replaces update_step (recon.cpp:93-134):
//                      gather disk * P -> centered IFFT 64x64 -> modulus :=
//                      sqrt(I) (+ residual) -> centered FFT -> scatter (GS
//                      write-back or EPRY object + pupil update).
// K2/K3  lines_fft     N-point row/column FFT passes for init_canvas
//                      (recon.cpp:61-86) and canvas_to_field (:88-91).
//        build_pupils  build_pupil (optics.cpp:41-72) for every tile.
//
// 64x64 FFT data layout (one tile = 64 threads, 64 complex per thread):
// thread t = (tr, tc) = (t/8, t%8) owns the lattice pixels (tr + 8a, tc + 8b),
// a, b in [0, 8), in registers v[a][b]. With n = 8*n1 + n0 and
// k = k0 + 8*k1, a 64-point DFT is an 8-point DFT over n1 (in registers),
// a twiddle W64^(n0 k0), a transpose, and an 8-point DFT over n0. Doing both
// axes at once gives one 32 KB shared-memory transpose per 2-D transform, and
// the output of one transform lands in exactly the lattice layout the next
// one (and the gather/scatter) needs, so thread t touches the same 64 pixels
// in every phase of every update.
#include "fft_device.cuh"
#include "kernels.cuh"

namespace fpmk {

namespace {

constexpr int kIBytes = 64 * 64 * 2;        // staged u16 measurement, TMA 128B-swizzled
constexpr int kTStride = 65;               // transpose row stride (float2): conflict-free both ways
constexpr int kTBytes = ((64 * kTStride * 8 + 1023) / 1024) * 1024;  // transpose buffer
constexpr int kGroupBytes = kIBytes + kTBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 3-D tiled TMA load of one 64x64 u16 LR crop: coordinates (x, y, frame).
__device__ __forceinline__ void tma_load_crop(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                              int y, int f) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(f)
        : "memory");
}

// Barrier over one 64-thread group (named barrier 1 + g).
__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, 64;" ::"r"(g + 1) : "memory");
}

// Cooley-Tukey twiddle W64^(n0r k0r + n0c k0c) of the lattice block, from the
// shared W64 table (forward sign; INV uses the conjugate).
template <bool INV>
__device__ __forceinline__ void twiddle64(float2 (&v)[8][8], const float2* W_s, int tr, int tc) {
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) {
        const float2 w = W_s[(tr * k1) & 63];
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) v[k1][k2] = INV ? cmulc(v[k1][k2], w) : cmul(v[k1][k2], w);
    }
#pragma unroll
    for (int k2 = 1; k2 < 8; ++k2) {
        const float2 w = W_s[(tc * k2) & 63];
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) v[k1][k2] = INV ? cmulc(v[k1][k2], w) : cmul(v[k1][k2], w);
    }
}

// Step 2 of a 64x64 transform: 2-D 8x8 DFT over the transposed block.
// PRUNE_OUT: only output rows a in [2, 6) are consumed (scatter on a small
// pupil), so the second-axis DFTs of the other rows are skipped.
template <bool INV, bool PRUNE_OUT>
__device__ __forceinline__ void dft8x8_out(float2 (&v)[8][8]) {
#pragma unroll
    for (int b = 0; b < 8; ++b)
        dft8<INV, false>(v[0][b], v[1][b], v[2][b], v[3][b], v[4][b], v[5][b], v[6][b], v[7][b]);
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        if (PRUNE_OUT && (a < 2 || a > 5)) continue;
        dft8<INV, false>(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4], v[a][5], v[a][6], v[a][7]);
    }
}

// Full 64x64 centered-core transform on the lattice block (without the
// checkerboard signs, which the caller folds into gather/scatter).
template <bool INV, bool PRUNE_IN, bool PRUNE_OUT>
__device__ __forceinline__ void fft64x64(float2 (&v)[8][8], float2* T_s, const float2* W_s, int t, int g) {
    dft8x8<INV, PRUNE_IN>(v);
    twiddle64<INV>(v, W_s, t >> 3, t & 7);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) {
            const int d = k1 * 8 + k2;
            T_s[d * kTStride + t] = v[k1][k2];
        }
    group_sync(g);
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int s = a * 8 + b;
            v[a][b] = T_s[t * kTStride + s];
        }
    dft8x8_out<INV, PRUNE_OUT>(v);
}

template <int G>
__device__ __forceinline__ int2 slot_entry(const LoopArgs& a, int s, int g) {
    if (G == 1) return make_int2(s / a.L, s % a.L);
    return a.slots[s * G + g];
}

}  // namespace

size_t loop_smem_bytes(int G, int nslots, int L, int iters) {
    size_t b = 1024;                                  // alignment slack for the 128B-swizzled TMA box
    b += size_t(G) * kGroupBytes;                     // per-group staging + transpose
    b += size_t(nslots) * 64 * sizeof(float2);        // lattice pupil [NP][64]
    b += 64 * sizeof(float2);                         // W64 table
    b += size_t(iters) * sizeof(double);              // stage sums
    b += size_t(G) * (sizeof(uint64_t) + 8 * sizeof(float));  // mbarriers + reductions
    b += size_t(L) * (sizeof(short2) + sizeof(int) + 1);      // origins + frame map + bright-field flags
    return b;
}

// Lattice positions a thread may own inside the pupil support: with PRUNE the
// disk lies in rows/cols [16, 48), i.e. a, b in [2, 6) (16 positions);
// otherwise all 64.
template <bool PRUNE>
struct Lattice {
    static constexpr int NP = PRUNE ? 16 : 64;
    __device__ static constexpr int a(int q) { return PRUNE ? 2 + (q >> 2) : (q >> 3); }
    __device__ static constexpr int b(int q) { return PRUNE ? 2 + (q & 3) : (q & 7); }
};

template <int MODE, bool PRUNE, int MEAS, int G, int N>
__global__ void __launch_bounds__(64 * G) fpm_loop64(const __grid_constant__ CUtensorMap tmap, const LoopArgs args) {
    using Lat = Lattice<PRUNE>;
    constexpr int NP = Lat::NP;
    extern __shared__ uint8_t smem_raw[];
    // align inside the shared window by offset so every pointer keeps the shared state space
    const uint32_t base = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((base + 1023u) & ~1023u) - base);
    const int g = threadIdx.x >> 6;
    const int t = threadIdx.x & 63;
    const int tr = t >> 3, tc = t & 7;
    const int tile = blockIdx.x;
    const int L = args.L;

    uint16_t* I_s = reinterpret_cast<uint16_t*>(smem + g * kGroupBytes);
    float2* T_s = reinterpret_cast<float2*>(smem + g * kGroupBytes + kIBytes);
    size_t off = size_t(G) * kGroupBytes;
    float2* P_s = reinterpret_cast<float2*>(smem + off);  // [NP][64], zero off the support
    off += size_t(NP) * 64 * sizeof(float2);
    float2* W_s = reinterpret_cast<float2*>(smem + off);  // W64^m, m in [0, 64)
    off += 64 * sizeof(float2);
    double* stage_sum = reinterpret_cast<double*>(smem + off);
    off += size_t(args.iters) * sizeof(double);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off);
    off += size_t(G) * sizeof(uint64_t);
    float* red = reinterpret_cast<float*>(smem + off);
    off += size_t(G) * 8 * sizeof(float);
    short2* O_s = reinterpret_cast<short2*>(smem + off);
    off += size_t(L) * sizeof(short2);
    int* F_s = reinterpret_cast<int*>(smem + off);
    off += size_t(L) * sizeof(int);
    uint8_t* B_s = smem + off;
    uint64_t* bar = bars + g;

    float2* canvas = args.canvas + size_t(tile) * N * N;
    float2* pupil_g = args.pupils + size_t(tile) * 64 * 64;
    const int2 txy = args.tile_xy[tile];

    // ---- one-time setup: support mask, lattice pupil, tables, twiddle table
    uint64_t mask = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const int i = tr + 8 * Lat::a(q), j = tc + 8 * Lat::b(q);
        const bool on = args.support[i * 64 + j] != 0;
        mask |= uint64_t(on) << q;
        // the shared pupil carries the thread's checkerboard sign: P' = (-1)^(i+j) P
        if (g == 0) P_s[q * 64 + t] = on ? cscale(pupil_g[i * 64 + j], ((tr + tc) & 1) ? -1.f : 1.f) : make_float2(0.f, 0.f);
    }
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        O_s[k] = args.origins[size_t(tile) * L + k];
        F_s[k] = args.seq_frame[k];
        B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
    }
    for (int k = threadIdx.x; k < args.iters; k += blockDim.x) stage_sum[k] = 0.0;
    if (threadIdx.x < 64) {
        double s, c;
        sincospi(-double(threadIdx.x) / 32.0, &s, &c);
        W_s[threadIdx.x] = make_float2(float(c), float(s));
    }
    if (MEAS == kMeasTMA && t == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const float sgn = ((tr + tc) & 1) ? -1.f : 1.f;  // checkerboard (-1)^(i+j) is constant per thread
    const float inv_n2 = 1.0f / 4096.0f;             // ifft2's 1/(rows*cols) (field.cpp:64-66)
    uint32_t phase = 0;
    bool issued = false;

    auto issue = [&](int2 e) {
        if (MEAS == kMeasTMA && t == 0) {
            mbar_expect_tx(bar, kIBytes);
            tma_load_crop(I_s, &tmap, bar, txy.x, txy.y, F_s[e.y]);
        }
    };

    for (int s = 0; s < args.num_slots; ++s) {
        const int2 e = slot_entry<G>(args, s, g);
        if (e.x >= 0) {
            if (!issued) issue(e);
            issued = false;
            const short2 o = O_s[e.y];
            float2* cv = canvas + size_t(o.x) * N + o.y;

            // ---- gather: all disk loads in flight at once (every lattice address lies in
            // the n x n block, so the loads need no predicate), then times P and the sign
            float2 v[8][8];
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) v[a][b] = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < NP; ++q) v[Lat::a(q)][Lat::b(q)] = cv[(tr + 8 * Lat::a(q)) * N + tc + 8 * Lat::b(q)];
            float omax = 0.f, pmax = 0.f;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const float2 O = v[Lat::a(q)][Lat::b(q)];
                const float2 P = P_s[q * 64 + t];
                if (MODE == kModeEPRY) {
                    omax = fmaxf(omax, ((mask >> q) & 1ull) ? cabs2(O) : 0.f);
                    pmax = fmaxf(pmax, cabs2(P));
                }
                v[Lat::a(q)][Lat::b(q)] = cmul(O, P);  // sign folded into P'
            }
            if (MODE == kModeEPRY) {
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) {
                    omax = fmaxf(omax, __shfl_xor_sync(0xffffffffu, omax, sh));
                    pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, sh));
                }
                if ((t & 31) == 0) {
                    red[g * 8 + 4 + (t >> 5)] = omax;
                    red[g * 8 + 6 + (t >> 5)] = pmax;
                }
            }

            // ---- centered inverse transform (unscaled; 1/n^2 enters only the residual)
            fft64x64<true, PRUNE, false>(v, T_s, W_s, t, g);

            // ---- modulus replacement with sqrt(I) and residual sums (recon.cpp:115-124)
            if (MEAS == kMeasTMA) {
                mbar_wait(bar, phase);
                phase ^= 1u;
            }
            // e' = e sqrt(I)/|e| (or sqrt(I) + 0i at |e| = 0, recon.cpp:122); the residual is
            // formed from the difference |e| - sqrt(I) itself so small residuals stay exact
            // (a one-rsqrt expansion |e|^2 - 2|e|sqrt(I) + I cancels catastrophically).
            float num = 0.f, den_f = 0.f;
            uint32_t den_u = 0;
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    float Iv;
                    if (MEAS == kMeasTMA) {
                        // 128B swizzle: 16-byte chunk b of row i sits at chunk b ^ (i & 7), i & 7 == tr
                        const uint32_t Iu = I_s[(tr + 8 * a) * 64 + ((b ^ tr) << 3) + tc];
                        den_u += Iu;
                        Iv = float(Iu);
                    } else {
                        Iv = args.meas_f32[(tr + 8 * a) * 64 + tc + 8 * b];
                        den_f += Iv;
                    }
                    const float meas = Iv > 0.f ? Iv * rsqrtf(Iv) : 0.f;
                    const float2 u = v[a][b];
                    const float m2 = cabs2(u);
                    if (__builtin_expect(m2 > 0.f, 1)) {
                        const float r = rsqrtf(m2);
                        const float dm = fmaf(m2 * r, inv_n2, -meas);
                        num = fmaf(dm, dm, num);
                        v[a][b] = cscale(u, meas * r);
                    } else {
                        num = fmaf(meas, meas, num);
                        v[a][b] = make_float2(sgn * meas, 0.f);
                    }
                }
            float den = MEAS == kMeasTMA ? float(den_u) : den_f;
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                num += __shfl_xor_sync(0xffffffffu, num, sh);
                den += __shfl_xor_sync(0xffffffffu, den, sh);
            }
            if ((t & 31) == 0) {
                red[g * 8 + (t >> 5)] = num;
                red[g * 8 + 2 + (t >> 5)] = den;
            }
            group_sync(g);  // staging buffer and transpose buffer free; reductions visible

            // prefetch the measurement of this group's next update
            if (s + 1 < args.num_slots) {
                const int2 nx = slot_entry<G>(args, s + 1, g);
                if (nx.x >= 0) {
                    issue(nx);
                    issued = true;
                }
            }
            if (t == 0) {
                const float nsum = red[g * 8] + red[g * 8 + 1];
                const float dsum = red[g * 8 + 2] + red[g * 8 + 3];
                stage_sum[e.x] += dsum > 0.f ? double(nsum) / double(dsum) : 0.0;
            }
            float inv_omax = 0.f, inv_pmax = 0.f;
            if (MODE == kModeEPRY) {
                const float om = fmaxf(red[g * 8 + 4], red[g * 8 + 5]);
                const float pm = fmaxf(red[g * 8 + 6], red[g * 8 + 7]);
                inv_omax = (om > 0.f && B_s[e.y]) ? args.beta / om : 0.f;  // bright-field pupil steps only
                inv_pmax = pm > 0.f ? args.alpha / pm : 0.f;
            }

            // ---- centered forward transform of the corrected field
            fft64x64<false, false, PRUNE>(v, T_s, W_s, t, g);

            // ---- scatter into the canvas disk (recon.cpp:127-130) / EPRY update
            if (MODE == kModeGS) {
#pragma unroll
                for (int q = 0; q < NP; ++q)
                    if ((mask >> q) & 1ull)
                        cv[(tr + 8 * Lat::a(q)) * N + tc + 8 * Lat::b(q)] = cmulc(v[Lat::a(q)][Lat::b(q)], P_s[q * 64 + t]);
            } else {
                const bool upd_o = inv_pmax > 0.f, upd_p = inv_omax > 0.f;
#pragma unroll
                for (int c0 = 0; c0 < NP; c0 += 16) {
                    float2 Ov[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        Ov[q] = cv[(tr + 8 * Lat::a(c0 + q)) * N + tc + 8 * Lat::b(c0 + q)];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int qq = c0 + q;
                        const bool on = (mask >> qq) & 1ull;
                        const float2 O = Ov[q];
                        const float2 P = P_s[qq * 64 + t];
                        // with P' = sP and Psi' = s v: d' = s d, conj(P') d' = conj(P) d,
                        // P'_new = P' + beta conj(O) d' / max|O|^2 (s = checkerboard sign)
                        const float2 d = csub(v[Lat::a(qq)][Lat::b(qq)], cmul(O, P));
                        if (on && upd_o)
                            cv[(tr + 8 * Lat::a(qq)) * N + tc + 8 * Lat::b(qq)] = cadd(O, cscale(cmulc(d, P), inv_pmax));
                        if (on && upd_p) P_s[qq * 64 + t] = cadd(P, cscale(cmulc(d, O), inv_omax));
                    }
                }
            }
        }
        __syncthreads();  // round barrier: canvas writes visible to the next update's gather
    }

    // ---- per-pass mean residual; EPRY pupil back to global
    for (int k = threadIdx.x; k < args.iters; k += blockDim.x)
        args.residuals[size_t(tile) * args.iters + k] = stage_sum[k] / double(L);
    if (MODE == kModeEPRY && g == 0) {
#pragma unroll
        for (int q = 0; q < NP; ++q)
            if ((mask >> q) & 1ull) pupil_g[(tr + 8 * Lat::a(q)) * 64 + tc + 8 * Lat::b(q)] = cscale(P_s[q * 64 + t], sgn);
    }
}

template <int MODE, bool PRUNE, int MEAS, int G, int N>
static cudaError_t launch_loop_t(const CUtensorMap* tmap, const LoopArgs& a, int T, cudaStream_t s) {
    const size_t smem = loop_smem_bytes(G, a.nslots, a.L, a.iters);
    auto k = fpm_loop64<MODE, PRUNE, MEAS, G, N>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<T, 64 * G, smem, s>>>(*tmap, a);
    return cudaGetLastError();
}

cudaError_t launch_loop64(int mode, bool prune, int meas, int G, const CUtensorMap* tmap,
                          const LoopArgs& a, int T, cudaStream_t s) {
#define FPM_LOOP_CASE(M, P, ME, GG, NN)                                               \
    if (mode == M && prune == P && meas == ME && G == GG && a.N == NN)                \
        return launch_loop_t<M, P, ME, GG, NN>(tmap, a, T, s);
#define FPM_LOOP_N(M, P, ME, GG) \
    FPM_LOOP_CASE(M, P, ME, GG, 256) FPM_LOOP_CASE(M, P, ME, GG, 512) FPM_LOOP_CASE(M, P, ME, GG, 1024)
    FPM_LOOP_N(kModeGS, true, kMeasTMA, 1)
    FPM_LOOP_N(kModeEPRY, true, kMeasTMA, 1)
    FPM_LOOP_N(kModeGS, true, kMeasTMA, 2)
    FPM_LOOP_CASE(kModeGS, false, kMeasTMA, 1, 256)
    FPM_LOOP_CASE(kModeEPRY, false, kMeasTMA, 1, 256)
    FPM_LOOP_CASE(kModeGS, false, kMeasTMA, 2, 256)
    FPM_LOOP_N(kModeGS, true, kMeasF32, 1)
    FPM_LOOP_N(kModeEPRY, true, kMeasF32, 1)
    FPM_LOOP_CASE(kModeGS, false, kMeasF32, 1, 256)
    FPM_LOOP_CASE(kModeEPRY, false, kMeasF32, 1, 256)
#undef FPM_LOOP_N
#undef FPM_LOOP_CASE
    return cudaErrorInvalidConfiguration;
}

// ============================================================== line FFTs
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
            a.dst[base + size_t(i) * NL + j] = cscale(x, sc);
        } else {
            const int line = idx / NL, e = idx - line * NL;
            a.dst[base + size_t(l0 + line) * NL + e] = res[line * NL + e];
        }
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

}  // namespace

cudaError_t launch_lines(int which, int N, const LinesArgs& a, int T, cudaStream_t s) {
    switch (N) {
        case 256: return launch_lines_n<256, 16>(which, a, T, s);
        case 512: return launch_lines_n<512, 8>(which, a, T, s);
        case 1024: return launch_lines_n<1024, 4>(which, a, T, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_build_pupils(float2* pupils, const uint8_t* support, const double* defocus, int n, int T,
                                double dk, double inv_l2, cudaStream_t s) {
    const size_t total = size_t(T) * n * n;
    const int blocks = int(std::min<size_t>((total + 255) / 256, 148 * 16));
    build_pupils_kernel<<<blocks, 256, 0, s>>>(pupils, support, defocus, n, T, dk, inv_l2);
    return cudaGetLastError();
}

}  // namespace fpmk
