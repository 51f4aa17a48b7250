// K1+K4 fpm_loop64: the fused per-LED update, persistent over the LED loop.
//
// One CTA group of 128 threads per tile runs every (iteration, LED) update of
// reconstruct_tile (recon.cpp:161-166) back to back; the fused update replaces
// update_step (recon.cpp:93-134): gather disk * P -> centered IFFT 64x64 ->
// modulus := sqrt(I) (+ residual) -> centered FFT -> scatter (GS write-back or
// EPRY object + pupil update).
//
// 64x64 transform layout ("pair lattice"). Thread (p, h), p = (tr, tc) in
// [0,64), h in {0,1}, owns the 32 pixels (tr + 8a, tc + 8b), a in [0,8),
// b = 2j + h, j in [0,4), in registers v[a][j]. A 64-point DFT factors as
// 8 x 8 (n = 8 n1 + n0, k = k0 + 8 k1):
//   step 1: 8-point DFTs over n1 of both axes for residue (n0r, n0c) = (tr, tc):
//           rows in registers; columns split over the lane pair by parity of
//           n1c (decimation in time: DFT4 per lane, W8 twiddle, one shuffle
//           exchange, butterfly);
//   twiddle W64^(n0 k0), one 32 KB shared-memory transpose (row-XOR swizzle:
//           conflict-free 64-bit writes and 128-bit reads);
//   step 2: 8-point DFTs over n0; columns split over the pair by contiguous
//           halves (decimation in frequency), which returns the output in the
//           parity-split layout step 1 consumes.
// So thread (p, h) touches the same 32 pixels in gather, modulus and scatter
// of every update, and 2 x 64 = 128 threads x ~128 registers give 16 warps per
// SM at 4 tiles per SM.
//
// The centred transforms use fft2(x) = C . FFT(C . x), C = (-1)^(i+j)
// (field.cpp:48-87); C is constant per thread and folded into the shared pupil.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "ptx_util.cuh"

namespace fpmk {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kIBytes = 64 * 64 * 2;            // staged u16 measurement, TMA 128B-swizzled
constexpr int kTBytes = 64 * 64 * 8;            // transpose buffer (swizzled, unpadded)
constexpr int kGroupBytes = kIBytes + kTBytes;  // 40 KB, a multiple of 1 KB
constexpr int kGroupThreads = 128;

#if FPM_TW2
using TwEntry = float2;
__device__ __forceinline__ float2 tw_mul(float2 v, float2 w) { return cmul2(v, w); }
__device__ __forceinline__ float2 tw_entry(double c, double s) { return make_float2(float(c), float(s)); }
#else
using TwEntry = float4;
__device__ __forceinline__ float2 tw_mul(float2 v, float4 w) {
    return cmul_sw(v, make_float2(w.x, w.y), make_float2(w.z, w.w));
}
__device__ __forceinline__ float4 tw_entry(double c, double s) {
    return make_float4(float(c), float(s), -float(s), float(c));
}
#endif
#ifndef FPM_PAIR_ROT
#define FPM_PAIR_ROT 1  // step-1 pair twiddles W8^1, W8^3 as rotations (scale folded into the column twiddles)
#endif
#ifndef FPM_O_STAGE
// EPRY scatter: 1 = old canvas values staged by cp.async into the measurement buffer after
// pass 1's transpose barrier (the next crop's TMA then waits for the next update); 0 = read
// at the scatter, the next crop's TMA issued at that barrier (measured 31.74 vs 31.17 ms)
#define FPM_O_STAGE 0
#endif
#ifndef FPM_TMA_LANE
#define FPM_TMA_LANE 32  // thread (of the group) that issues the measurement TMA (0: 30.28, 32: 30.18 ms)
#endif
#ifndef FPM_SUM_LANE
#define FPM_SUM_LANE 0  // thread (of the group) that adds the update's residual ratio
#endif
#ifndef FPM_DEN_SEP
#define FPM_DEN_SEP 1  // sum(I) of a crop by a separate loop on first visits (not a predicated add per pixel)
#endif
#ifndef FPM_TW2
#define FPM_TW2 1  // twiddle tables as float2 with the two-instruction cmul2 (0: float4 (w, iw) pairs, cmul_sw)
#endif
#ifndef FPM_O_EARLY
#define FPM_O_EARLY 1  // 1: the scatter's old canvas values loaded before pass 1's step 2 (loop 30.455 vs 30.57 ms; before the alternating transposes 31.24 vs 31.16)
#endif
#ifndef FPM_MOD_SEL
#define FPM_MOD_SEL 0  // |e| = 0 rule by selects (1; measured +1.5%) or by a 2^-60 nudge of Re (0)
#endif
#ifndef FPM_P0_INPUT_SWAP
#define FPM_P0_INPUT_SWAP 1  // pass 0 step 1: swap the disk's inputs within the pair, not the outputs
#endif
#ifndef FPM_O_SMEM
#define FPM_O_SMEM 0  // EPRY: the gathered canvas values kept in shared memory for the scatter (+8 KB per CTA)
#endif
#ifndef FPM_LOOP_MINB
#define FPM_LOOP_MINB 4  // resident tiles per SM the register budget is sized for
#endif

// Barrier over one 128-thread group (named barrier 1 + g).
__device__ __forceinline__ void group_sync(int g) {
    asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory");
}

__device__ __forceinline__ float2 shfl_pair(float2 x) {
    return make_float2(__shfl_xor_sync(kFull, x.x, 1), __shfl_xor_sync(kFull, x.y, 1));
}

// v * (-i) on the odd lane of a pair, v on the even one (the pair twiddle W8^2):
// selects and a sign-bit flip on the ALU pipe instead of a two-instruction
// packed multiply on the FMA pipe
__device__ __forceinline__ float2 mul_mi_odd(float2 v, int h) {
    const float nx = __int_as_float(__float_as_int(v.x) ^ int(0x80000000u));
    return h ? make_float2(v.y, nx) : v;
}

// transpose swizzle of destination row p': XOR on slot bits 1 and 3
__device__ __forceinline__ int tswz(int pp) {
    return ((pp & 1) << 1) | ((((pp >> 1) ^ (pp >> 2)) & 1) << 3);
}

// One forward transform serves both directions (IFFT(x) = conj(FFT(conj x)), the
// conjugations folded into gather and modulus), split at the transpose: fft_first
// (step 1, twiddle, transpose write) and fft_second (transpose read, step 2), the
// group barrier between them issued by the caller. The update runs each half once
// per pass with the prunings resolved at compile time: skip_cols drops the zero
// columns of the disk-limited input (IFFT), skip_rows the rows the scatter never
// reads (FFT).
//
// Transpose layouts (one swizzle tswz for both): pass 0 uses layout A — element
// k0 = (a, 4h + m) of residue p at physical row p' = 8a + 4h + m, column p; pass 1
// uses layout B — the same element at physical row p, column p'. A thread's layout-B
// writes land in its own physical row, in the half (bit 2 of the column) that only
// it read in layout A, and its layout-A writes of the next update land in the
// column half only it read in layout B: no write can overtake another thread's
// pending read, so the transposes need only their write-to-read barriers (the
// barrier after the modulus is gone; the modulus's reductions and the measurement
// buffer are released by pass 1's transpose barrier).
__device__ __forceinline__ void fft_first(float2 (&v)[8][4], float2* T_s, const TwEntry* W4_s, int p, int h,
                                          float sg, const float2 (&tw)[4], const float2 (&twsw)[4], float kh,
                                          float c1, float c3, bool skip_cols, bool layout_b) {
    const int tr = p >> 3, tc = p & 7;
    // step 1: DFT8 over n1r (registers), then the pair DFT over n1c (DIT). Pruned IFFT
    // (skip_cols): only rows a in [2, 6) of columns j in {1, 2} hold data, and the
    // zero entries are never read (they need no initialisation)
#if FPM_P0_INPUT_SWAP
    if (skip_cols) {
        // Columns first, over the disk's four non-zero column digits b in [2, 6) (rows a in
        // [2, 6)): the pair swaps its two values per row (16 shuffles instead of the 64 of
        // the output exchange), then each lane forms its four DFT8 outputs k = 4h + m
        // directly: X = E + (-1)^h O, E from x2, x4 and O from x3, x5
        //   E = (x2 + x4, -i x2 - x4, x4 - x2, i x2 - x4),
        //   O = (s, (q - s) / sqrt2, -q, (q + s) / sqrt2), s = x3 + x5, q = -i (x3 - x5).
        // Exact outputs: pass 0 uses the unscaled column-twiddle table.
        const float sgr = sg * 0.70710678118654752440f;
#pragma unroll
        for (int a = 2; a < 6; ++a) {
            const float2 o1 = v[a][1], o2 = v[a][2];  // own: x[2 + h], x[4 + h]
            const float2 r1 = shfl_pair(o1), r2 = shfl_pair(o2);
            const float2 x2 = h ? r1 : o1, x4 = h ? r2 : o2, x3 = h ? o1 : r1, x5 = h ? o2 : r2;
            const float2 s24 = cadd(x2, x4), s35 = cadd(x3, x5), q = w8_2<false>(csub(x3, x5));
            const float2 m2 = w8_2<false>(x2);
            v[a][0] = cfma(sg, s35, s24);
            v[a][2] = cfma(-sg, q, csub(x4, x2));
            v[a][1] = cfma(sgr, csub(q, s35), csub(m2, x4));
            v[a][3] = cfma(sgr, cadd(q, s35), cneg(cadd(m2, x4)));
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
            dft8<false, true>(v[0][m], v[1][m], v[2][m], v[3][m], v[4][m], v[5][m], v[6][m], v[7][m]);
    }
#else
    if (skip_cols) {
#pragma unroll
        for (int j = 1; j < 3; ++j)
            dft8<false, true>(v[0][j], v[1][j], v[2][j], v[3][j], v[4][j], v[5][j], v[6][j], v[7][j]);
#pragma unroll
        for (int a = 0; a < 8; ++a) dft4_z03<false>(v[a][0], v[a][1], v[a][2], v[a][3]);
    }
#endif
    if (!skip_cols) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            dft8<false, false>(v[0][j], v[1][j], v[2][j], v[3][j], v[4][j], v[5][j], v[6][j], v[7][j]);
#pragma unroll
        for (int a = 0; a < 8; ++a) dft4<false>(v[a][0], v[a][1], v[a][2], v[a][3]);  // E (h = 0) or O (h = 1)
    }
    // pair DIT: X[m] = E + W8^m O (even lane), X[m + 4] = E - W8^m O (odd lane). m = 2: W8^2 = -i,
    // a swap and a sign off the FMA pipe. m = 1, 3: W8^m O = s R with s = 1/sqrt(2) and R a
    // rotation (one FFMA2 on the odd lane instead of a complex multiply): the odd lane forms
    // E - s R exactly, the even lane +-(sqrt(2) E + R), whose factor +-s rides on its column
    // twiddle (table entries pre-scaled)
    if (!(FPM_P0_INPUT_SWAP && skip_cols)) {
#if FPM_PAIR_ROT
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        v[a][1] = cfma_v(make_float2(kh, -kh), make_float2(v[a][1].y, v[a][1].x), v[a][1]);  // odd: R1 = (x + y, y - x)
        v[a][2] = mul_mi_odd(v[a][2], h);
        v[a][3] = cfma_v(make_float2(-kh, kh), make_float2(v[a][3].y, v[a][3].x), v[a][3]);  // odd: -R3 = (x - y, x + y)
        v[a][0] = cfma(sg, v[a][0], shfl_pair(v[a][0]));  // E + O | E - O
        v[a][1] = cfma(c1, v[a][1], shfl_pair(v[a][1]));  // sqrt(2) E + R1 | E - s R1
        v[a][2] = cfma(sg, v[a][2], shfl_pair(v[a][2]));
        v[a][3] = cfma(c3, v[a][3], shfl_pair(v[a][3]));  // -(sqrt(2) E + R3) | E - s R3
    }
#else
#pragma unroll
    for (int a = 0; a < 8; ++a) {
#pragma unroll
        for (int m = 1; m < 4; ++m)  // O' = W8^m O (m = 2: -i, a swap and a sign off the FMA pipe)
            v[a][m] = m == 2 ? mul_mi_odd(v[a][m], h) : cmul_sw(v[a][m], tw[m], twsw[m]);
#pragma unroll
        for (int m = 0; m < 4; ++m) v[a][m] = cfma(sg, v[a][m], shfl_pair(v[a][m]));  // E + O' | E - O'
    }
#endif
    }
    // twiddle W64^(n0r k0r + n0c k0c), k0 = (a, 4h + m); table entries (w, (-w.y, w.x))
#pragma unroll
    for (int a = 1; a < 8; ++a) {
        const TwEntry w = W4_s[(tr * a) & 63];
#pragma unroll
        for (int m = 0; m < 4; ++m) v[a][m] = tw_mul(v[a][m], w);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        // = W64^(tc (4h + m)), in lane order; [128, 192): the same without the pair trick's scale
        const TwEntry w = W4_s[((FPM_P0_INPUT_SWAP && skip_cols) ? 128 : 64) + m * 16 + 2 * tc + h];
#pragma unroll
        for (int a = 0; a < 8; ++a) v[a][m] = tw_mul(v[a][m], w);
    }
    if (!layout_b) {
        // layout A: element k0 = (a, 4h + m) of residue p goes to row p' = 8a + 4h + m, slot p
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int gm = ((m & 1) << 1) | (((((m >> 1) & 1) ^ h)) << 3);  // tswz(8a + 4h + m)
            float2* wrow = T_s + (4 * h + m) * 64 + (p ^ gm);
#pragma unroll
            for (int a = 0; a < 8; ++a) wrow[a * 512] = v[a][m];
        }
    } else {
        // layout B: own row p, columns (8a + 4h + m) ^ tswz(p) (128-bit stores of the pairs m,
        // m + 1). tswz flips column bit 3 (a's parity) by g3 and bit 1 (m) by g1: four bases,
        // the rest immediate offsets
        const int gp = tswz(p), g3 = (gp >> 3) & 1, g1 = (gp >> 1) & 1;
        float2* e0 = T_s + p * 64 + 8 * g3 + 4 * h + 2 * g1;  // even a, m = 0
        float2* e2 = e0 + 2 - 4 * g1;                          // even a, m = 2
        float2* o0 = e0 + 8 - 16 * g3;                         // odd a, m = 0
        float2* o2 = e2 + 8 - 16 * g3;                         // odd a, m = 2
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            *reinterpret_cast<float4*>(e0 + 16 * k) = make_float4(v[2 * k][0].x, v[2 * k][0].y, v[2 * k][1].x, v[2 * k][1].y);
            *reinterpret_cast<float4*>(e2 + 16 * k) = make_float4(v[2 * k][2].x, v[2 * k][2].y, v[2 * k][3].x, v[2 * k][3].y);
            *reinterpret_cast<float4*>(o0 + 16 * k) =
                make_float4(v[2 * k + 1][0].x, v[2 * k + 1][0].y, v[2 * k + 1][1].x, v[2 * k + 1][1].y);
            *reinterpret_cast<float4*>(o2 + 16 * k) =
                make_float4(v[2 * k + 1][2].x, v[2 * k + 1][2].y, v[2 * k + 1][3].x, v[2 * k + 1][3].y);
        }
    }
}

__device__ __forceinline__ void fft_second(float2 (&v)[8][4], const float2* T_s, int p, int h, float sg,
                                           const float2 (&tw)[4], const float2 (&twsw)[4], bool skip_rows,
                                           bool layout_b) {
    if (!layout_b) {
        // layout A, read row p: slots n0r * 8 + 4h + i, XOR-swizzled (bit 3 flips the row parity,
        // bit 1 the pair)
        const int gp = tswz(p);
        const float2* rrow = T_s + p * 64;
        const int ofs = (4 * h) ^ (gp & 2);
        const int rflip = gp & 8;
#pragma unroll
        for (int n0r = 0; n0r < 8; ++n0r) {
            const float2* r = rrow + ((n0r * 8) ^ rflip) + ofs;
            const float4 q0 = *reinterpret_cast<const float4*>(r);
            const float4 q1 = *reinterpret_cast<const float4*>(r + (2 ^ (gp & 2)) - (gp & 2));
            v[n0r][0] = make_float2(q0.x, q0.y);
            v[n0r][1] = make_float2(q0.z, q0.w);
            v[n0r][2] = make_float2(q1.x, q1.y);
            v[n0r][3] = make_float2(q1.z, q1.w);
        }
    } else {
        // layout B, read column p of rows 8 n0r + 4h + i (tswz of those rows: bit 1 = i & 1,
        // bit 3 = (i >> 1) ^ h, independent of n0r)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2* col = T_s + (4 * h + i) * 64 + (p ^ (((i & 1) << 1) | ((((i >> 1) & 1) ^ h) << 3)));
#pragma unroll
            for (int n0r = 0; n0r < 8; ++n0r) v[n0r][i] = col[n0r * 512];
        }
    }
    // step 2: DFT8 over n0r, then the pair DFT over n0c (DIF); pruned FFT (skip_rows):
    // only outputs a in [2, 6) of the DFT8 are formed
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (skip_rows)
            dft8<false, false, true>(v[0][i], v[1][i], v[2][i], v[3][i], v[4][i], v[5][i], v[6][i], v[7][i]);
        else
            dft8<false, false>(v[0][i], v[1][i], v[2][i], v[3][i], v[4][i], v[5][i], v[6][i], v[7][i]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        if ((a < 2 || a > 5) && skip_rows) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) v[a][i] = cfma(sg, v[a][i], shfl_pair(v[a][i]));  // y_i + y_(i+4) | y_i - y_(i+4)
#pragma unroll
        for (int i = 1; i < 4; ++i)
            v[a][i] = i == 2 ? mul_mi_odd(v[a][i], h) : (FPM_TW2 ? cmul2(v[a][i], tw[i]) : cmul_sw(v[a][i], tw[i], twsw[i]));
        if (skip_rows)  // the scatter reads columns j in {1, 2} of these rows only
            dft4_o12<false>(v[a][0], v[a][1], v[a][2], v[a][3]);
        else
            dft4<false>(v[a][0], v[a][1], v[a][2], v[a][3]);
    }
}

template <int G>
__device__ __forceinline__ int2 slot_entry(const LoopArgs& a, int s, int g) {
    if (G == 1) return make_int2(s / a.L, s % a.L);
    return a.slots[s * G + g];
}

// Lattice positions a thread may own inside the pupil support: with PRUNE the
// disk lies in rows/cols [16, 48), i.e. a in [2, 6) and b = 2j + h in [2, 6),
// j in {1, 2} (8 positions); otherwise all 32.
template <bool PRUNE>
struct Lattice {
    static constexpr int NP = PRUNE ? 8 : 32;
    __device__ static constexpr int a(int q) { return PRUNE ? 2 + (q >> 1) : (q >> 2); }
    __device__ static constexpr int j(int q) { return PRUNE ? 1 + (q & 1) : (q & 3); }
};

}  // namespace

size_t loop_smem_bytes(int G, int nslots, int L, int iters) {
    size_t b = 1024;                                              // alignment slack (128B-swizzled TMA box)
    b += size_t(G) * kGroupBytes;                                 // per-group staging + transpose
    b += size_t(nslots) * kGroupThreads * sizeof(float2);         // lattice pupil [NP][128]
    b += 192 * sizeof(float4);                                    // W64 table + column-twiddle tables
    b += size_t(iters) * sizeof(double);                          // stage sums
    b += size_t(G) * (sizeof(uint64_t) + 16 * sizeof(float));     // mbarriers + reductions
    b += size_t(L) * (sizeof(short2) + sizeof(int) + sizeof(float) + 1);  // origins, frame map, sum(I), bright flags
    b += 8;                                                       // work-queue item (4-byte aligned)
    if (FPM_O_SMEM) b = ((b + 15) & ~size_t(15)) + size_t(nslots) * kGroupThreads * sizeof(float2);
    return b;
}

// MINB: resident tiles per SM the register budget is sized for (4: 128 registers,
// the throughput build; 2: 255 registers, lower latency per update for batches
// that leave SMs with at most a few tiles)
template <int MODE, bool PRUNE, int MEAS, int G, int N, int MINB, bool JIT>
__global__ void __launch_bounds__(kGroupThreads * G, G == 1 ? MINB : 2)
    fpm_loop64(const __grid_constant__ CUtensorMap tmap, const LoopArgs args) {
    using Lat = Lattice<PRUNE>;
    constexpr int NP = Lat::NP;
    extern __shared__ uint8_t smem_raw[];
    // align inside the shared window by offset so every pointer keeps the shared state space
    const uint32_t base = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((base + 1023u) & ~1023u) - base);
    const int g = threadIdx.x / kGroupThreads;
    const int tl = threadIdx.x % kGroupThreads;
    const int p = tl >> 1, h = tl & 1;
    const int tr = p >> 3, tc = p & 7;
    const int warp = tl >> 5;
    const int L = args.L;

    uint16_t* I_s = reinterpret_cast<uint16_t*>(smem + g * kGroupBytes);
    float2* T_s = reinterpret_cast<float2*>(smem + g * kGroupBytes + kIBytes);
    size_t off = size_t(G) * kGroupBytes;
    float2* P_s = reinterpret_cast<float2*>(smem + off);  // [NP][128], P' = (-1)^(i+j) P, zero off the support
    off += size_t(NP) * kGroupThreads * sizeof(float2);
    // [0, 64): (W64^m, swizzled), m in [0, 64); [64, 128): the column twiddle W64^(tc (4h + m))
    // at 64 + 16 m + 2 tc + h, i.e. in lane order (lane = 2 (8 tr + tc) + h): conflict-free
    TwEntry* W4_s = reinterpret_cast<TwEntry*>(smem + off);
    off += 192 * sizeof(float4);  // (sized for the float4 entries of FPM_TW2 = 0)
    double* stage_sum = reinterpret_cast<double*>(smem + off);
    off += size_t(args.iters) * sizeof(double);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off);
    off += size_t(G) * sizeof(uint64_t);
    float* red = reinterpret_cast<float*>(smem + off);  // [G][16]: num[4], den[4], omax[4], pmax[4]
    off += size_t(G) * 16 * sizeof(float);
    short2* O_s = reinterpret_cast<short2*>(smem + off);
    off += size_t(L) * sizeof(short2);
    int* F_s = reinterpret_cast<int*>(smem + off);
    off += size_t(L) * sizeof(int);
    float* D_s = reinterpret_cast<float*>(smem + off);  // sum(I) per LED, formed on its first visit
    off += size_t(L) * sizeof(float);
    uint8_t* B_s = smem + off;
    off += size_t(L);
    off = (off + 3) & ~size_t(3);
    int* item_s = reinterpret_cast<int*>(smem + off);  // work queue: the CTA's current item
    off += 8;
    constexpr bool kOSm = FPM_O_SMEM && MODE == kModeEPRY && PRUNE && G == 1;
    float2* O_sm = reinterpret_cast<float2*>(smem + ((off + 15) & ~size_t(15)));  // [NP][128] (kOSm)
    uint64_t* bar = bars + g;
    float* rg = red + g * 16;

    // ---- one-time setup: W64 tables, pair twiddles, mbarrier
    for (int t = threadIdx.x; t < 192; t += blockDim.x) {
        const int e = (t - 64) & 63;  // column tables: [64, 128) pre-scaled, [128, 192) exact
        const int m = t < 64 ? t : ((((e & 15) >> 1) * (4 * (e & 1) + (e >> 4))) & 63);
        double s, c;
        sincospi(-double(m) / 32.0, &s, &c);
        // column twiddles of the even lane for m = 1, 3 carry the pair combine's +-1/sqrt(2)
        const double f = (FPM_PAIR_ROT && t >= 64 && t < 128 && (e & 1) == 0 && ((e >> 4) & 1))
                             ? ((e >> 4) == 1 ? 1.0 : -1.0) * 0.70710678118654752440 : 1.0;
        W4_s[t] = tw_entry(c * f, s * f);
    }
    // pair-combine twiddles W8^m, m = 1..3, on the odd lane (1 on the even lane)
    float2 tw[4];
    {
        const float s = 0.70710678118654752440f;
        tw[0] = make_float2(1.f, 0.f);
        tw[1] = h ? make_float2(s, -s) : make_float2(1.f, 0.f);
        tw[2] = h ? make_float2(0.f, -1.f) : make_float2(1.f, 0.f);
        tw[3] = h ? make_float2(-s, -s) : make_float2(1.f, 0.f);
    }
    float2 twsw[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) twsw[m] = make_float2(-tw[m].y, tw[m].x);
    const float sg = h ? -1.f : 1.f;
    const float kh = h ? 1.f : 0.f;  // step-1 rotations on the odd lane only
    const float c1 = h ? -0.70710678118654752440f : 1.41421356237309504880f;
    const float c3 = h ? 0.70710678118654752440f : -1.41421356237309504880f;
    if (MEAS == kMeasTMA && tl == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const float sgn = ((tr + tc) & 1) ? -1.f : 1.f;  // checkerboard (-1)^(i+j), constant per thread
    const float inv_n2 = 1.0f / 4096.0f;  // ifft2's 1/(rows*cols) (field.cpp:64-66)
    uint32_t phase = 0;
    // canvas offset of lattice position (a, j) relative to the sub-aperture origin
    const int cbase = tr * N + tc + 8 * h;
    // work queue (G == 1): items j = (it * H + part) * T + tile, H = parts per pass
    // (LED positions [part L / H, (part + 1) L / H) of pass it); item j depends on
    // item j - T (the tile's previous part), claimed 1.7 waves earlier at BASELINE
    // config 3, so the dependency wait is almost never taken. Every update runs the
    // same instructions as in the one-CTA-per-tile launch, and a part continues the
    // pass's residual sum where the previous part left it (stored unscaled in the
    // residual slot): bit-identical
    const bool queue = G == 1 && args.work != nullptr;
    const int H = queue ? args.parts : 1;
    const int n_items = args.T * args.iters * H;

    for (int round = 0;; ++round) {
    int tile, it_q = 0, part = 0, s_begin, s_end;
    if (queue) {
        __syncthreads();  // the previous item's stores (canvas, pupil, residual, sum(I)) are done
        if (threadIdx.x == 0) {
            if (round > 0) {  // release: publish the finished item (item_s still holds it)
                const int jp = *item_s;
                __threadfence();
                st_release_gpu(args.work + 1 + jp % args.T, jp / args.T + 1);
            }
            jitter_sleep<JIT>(args, -1 - round);
            const int j = atomicAdd(args.work, 1);
            *item_s = j;
            if (j < n_items && j >= args.T) {  // acquire: the tile's previous pass is complete
                const int* flag = args.work + 1 + (j % args.T);
                while (ld_acquire_gpu(flag) < j / args.T) __nanosleep(256);  // items of the tile done
                __threadfence();
            }
        }
        __syncthreads();
        const int j = *item_s;
        if (j >= n_items) break;
        tile = j % args.T;
        const int ip = j / args.T;  // it * H + part
        it_q = ip / H;
        part = ip % H;
        s_begin = it_q * L + part * L / H;
        s_end = it_q * L + (part + 1) * L / H;
    } else {
        if (round > 0) break;
        tile = blockIdx.x;
        s_begin = args.slot_begin;
        s_end = args.num_slots;
    }
    FPM_ASSERT(tile >= 0 && tile < args.T && s_begin >= 0 && s_end <= args.num_slots);

    // ---- per-tile setup: support mask, lattice pupil, origins, frame map, flags
    float2* canvas = args.canvas + size_t(tile) * N * N;
    float2* pupil_g = args.pupils + size_t(tile) * 64 * 64;
    const int2 txy = args.tile_xy[tile];
    uint32_t mask = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const int i = tr + 8 * Lat::a(q), jj = tc + 8 * (2 * Lat::j(q) + h);
        const bool on = args.support[i * 64 + jj] != 0;
        mask |= uint32_t(on) << q;
        if (g == 0) P_s[q * kGroupThreads + tl] = on ? cscale(pupil_g[i * 64 + jj], sgn) : make_float2(0.f, 0.f);
    }
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        O_s[k] = args.origins[size_t(tile) * L + k];
        F_s[k] = args.seq_frame[k];
        B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
        if (queue && it_q > 0) D_s[k] = args.isum[size_t(tile) * L + k];
    }
    for (int k = threadIdx.x; k < args.iters; k += blockDim.x)
        stage_sum[k] = queue && part > 0 && k == it_q ? args.residuals[size_t(tile) * args.iters + k] : 0.0;
    __syncthreads();

    bool issued = false;
    bool pupil_dirty = true;  // EPRY: max|P|^2 changes only after a pupil step
    auto issue = [&](int2 e) {
        if (MEAS == kMeasTMA && tl == FPM_TMA_LANE) {
            // the staging buffer's earlier generic-proxy accesses (modulus reads, the EPRY
            // canvas staging) are ordered before the TMA's async-proxy write
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, kIBytes);
            FPM_ASSERT(e.y >= 0 && e.y < L && F_s[e.y] >= 0 && (args.F == 0 || F_s[e.y] < args.F));
            tma_load_crop(I_s, &tmap, bar, txy.x, txy.y, F_s[e.y]);
        }
    };
    // sequential slots (G == 1): (iteration, position) by counters, not a division per slot
    int c_it = G == 1 ? s_begin / L : 0, c_pos = G == 1 ? s_begin - c_it * L : 0;
    for (int s = s_begin; s < s_end; ++s) {
        jitter_sleep<JIT>(args, s);
        const int2 e = G == 1 ? make_int2(c_it, c_pos) : slot_entry<G>(args, s, g);
        if (e.x >= 0) {
            if (!issued) issue(e);
            issued = false;
            const short2 o = O_s[e.y];
            // the 64 x 64 disk block lies inside the tile's N x N canvas (every lattice
            // gather and scatter below is an offset inside that block)
            FPM_ASSERT(e.x >= 0 && e.x < args.iters && e.y >= 0 && e.y < L && o.x >= 0 && o.y >= 0 &&
                       o.x + 64 <= N && o.y + 64 <= N);
            float2* cv = canvas + size_t(o.x) * N + o.y + cbase;

            // ---- gather: every disk load in flight at once (all lattice addresses lie in
            // the n x n block, so the loads need no predicate), then times P'
            float2 v[8][4];  // lattice positions outside the disk block are never read (pruned IFFT)
#pragma unroll
            for (int q = 0; q < NP; ++q) v[Lat::a(q)][Lat::j(q)] = cv[Lat::a(q) * 8 * N + 16 * Lat::j(q)];
            if constexpr (kOSm) {
#pragma unroll
                for (int q = 0; q < NP; ++q) O_sm[q * kGroupThreads + tl] = v[Lat::a(q)][Lat::j(q)];
            }
            // EPRY maxima (block-uniform branches): max|O_D|^2 only for bright-field updates (the
            // only ones that take a pupil step), max|P|^2 only after the pupil changed — otherwise
            // the reduction slots keep their last values
            const bool bright = MODE == kModeEPRY && B_s[e.y];
            if (bright) {
                float omax = 0.f;
#pragma unroll
                for (int q = 0; q < NP; ++q)
                    omax = fmaxf(omax, ((mask >> q) & 1u) ? cabs2(v[Lat::a(q)][Lat::j(q)]) : 0.f);
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) omax = fmaxf(omax, __shfl_xor_sync(kFull, omax, sh));
                if ((tl & 31) == 0) rg[8 + warp] = omax;
            }
            if (MODE == kModeEPRY && pupil_dirty) {
                float pmax = 0.f;
#pragma unroll
                for (int q = 0; q < NP; ++q) pmax = fmaxf(pmax, cabs2(P_s[q * kGroupThreads + tl]));
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(kFull, pmax, sh));
                if ((tl & 31) == 0) rg[12 + warp] = pmax;
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                // conj: the IFFT runs as conj(FFT(conj x))
                v[Lat::a(q)][Lat::j(q)] = cmul_conj(v[Lat::a(q)][Lat::j(q)], P_s[q * kGroupThreads + tl]);
            }

            // ---- pass 0: centered inverse transform (unscaled; 1/n^2 enters only the residual),
            //      run as conj(FFT(conj x)); modulus replacement
            // ---- pass 1: centered forward transform of the corrected field
            float inv_omax = 0.f, inv_pmax = 0.f;
            fft_first(v, T_s, W4_s, p, h, sg, tw, twsw, kh, c1, c3, PRUNE, false);
            group_sync(g);
            fft_second(v, T_s, p, h, sg, tw, twsw, false, false);

            // ---- modulus replacement with sqrt(I) and residual sums (recon.cpp:115-124):
            // e' = e sqrt(I)/|e| (sqrt(I) + 0i at |e| = 0, recon.cpp:122); the residual is formed
            // from |e| - sqrt(I) itself so small residuals stay exact
            if (MEAS == kMeasTMA) {
                mbar_wait(bar, phase);
                phase ^= 1u;
            }
            // sum(I) of an LED's crop is formed once, on its first visit in this launch
            const bool first = queue ? it_q == 0 : G == 1 ? s - args.slot_begin < L : e.x == 0;
            float num = 0.f, den_f = 0.f;
            uint32_t den_u = 0;
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int b = 2 * u + h;
                    float Iv;
                    if (MEAS == kMeasTMA) {
                        // FPM_MEAS_SWIZZLE: 16-byte chunk b of row i sits at chunk b ^ (i & 7), i & 7 == tr
                        const uint32_t Iu = I_s[(tr + 8 * a) * 64 + ((FPM_MEAS_SWIZZLE ? b ^ tr : b) << 3) + tc];
                        if (!FPM_DEN_SEP && first) den_u += Iu;
                        Iv = float(Iu);
                    } else {
                        Iv = args.meas_f32[(tr + 8 * a) * 64 + tc + 8 * b];
                        if (first) den_f += Iv;
                    }
                    // |e| = 0 rule (recon.cpp:122): e' = sqrt(I) + 0i, checkerboarded (sgn), by two
                    // selects on the ALU pipe
                    const float meas = sqrt_ftz(Iv);
#if FPM_MOD_SEL
                    const float2 uu = v[a][u];
                    const float m2 = fmaf(uu.x, uu.x, uu.y * uu.y);
                    const bool zero = m2 == 0.f;
                    const float r = rsqrt_ftz(fmaxf(m2, kTiny));
                    const float dm = fmaf(m2 * r, inv_n2, -meas);  // |e| - sqrt(I)
                    num = fmaf(dm, dm, num);
                    const float sc = zero ? meas : meas * r;
                    const float ux = zero ? sgn : uu.x;
#else
                    // nudging Re by sgn 2^-60 leaves every value with |Re| >= 2^-35 bit-identical
                    // and maps e = 0 to (sgn 2^-60, 0), whose replacement is sqrt(I) + 0i, signed
                    const float2 uu = v[a][u];
                    const float ux = uu.x + sgn * 0x1p-60f;
                    const float m2 = fmaf(ux, ux, uu.y * uu.y);
                    const float r = rsqrt_ftz(fmaxf(m2, kTiny));
                    const float dm = fmaf(m2 * r, inv_n2, -meas);  // |e| - sqrt(I)
                    num = fmaf(dm, dm, num);
                    const float sc = meas * r;
#endif
                    // uu = conj(e n^2): undo the conjugation
                    v[a][u] = cscale(make_float2(ux, -uu.y), sc);  // one FMUL2 (.NP negates the high half)
                }
            if (FPM_DEN_SEP && MEAS == kMeasTMA && first) {  // sum(I): a separate pass on first visits only
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        den_u += I_s[(tr + 8 * a) * 64 + (((FPM_MEAS_SWIZZLE ? (2 * u + h) ^ tr : 2 * u + h)) << 3) + tc];
            }
            float den = MEAS == kMeasTMA ? float(den_u) : den_f;
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) num += __shfl_xor_sync(kFull, num, sh);
            if (first) {
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) den += __shfl_xor_sync(kFull, den, sh);
            }
            if ((tl & 31) == 0) {
                rg[warp] = num;
                rg[4 + warp] = den;
            }
            // ---- pass 1: centred forward transform of the corrected field (layout-B transpose)
            fft_first(v, T_s, W4_s, p, h, sg, tw, twsw, kh, c1, c3, false, true);
            group_sync(g);  // pass 1's transpose written; every warp past its modulus: staging buffer free,
                            // reductions visible

            // EPRY (pruned, sequential): the scatter's old canvas values go into the now-free
            // measurement staging buffer by cp.async, their latency under pass 1's step 2; the next
            // crop's TMA is then issued at the top of the next update
            constexpr bool kOStage = FPM_O_STAGE && MODE == kModeEPRY && PRUNE && G == 1 && MEAS == kMeasTMA;
            if constexpr (kOStage) {
                float2* Ostg = reinterpret_cast<float2*>(I_s);
#pragma unroll
                for (int q = 0; q < NP; ++q)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Ostg + q * kGroupThreads + tl)),
                                 "l"(cv + Lat::a(q) * 8 * N + 16 * Lat::j(q))
                                 : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            // prefetch the measurement of this group's next update
            if (!kOStage && s + 1 < s_end) {
                const int2 nx = G == 1 ? (c_pos + 1 == L ? make_int2(c_it + 1, 0) : make_int2(c_it, c_pos + 1))
                                       : slot_entry<G>(args, s + 1, g);
                if (nx.x >= 0) {
                    issue(nx);
                    issued = true;
                }
            }
            if (tl == FPM_SUM_LANE) {
                const float nsum = (rg[0] + rg[1]) + (rg[2] + rg[3]);
                float dsum;
                if (first) {
                    dsum = (rg[4] + rg[5]) + (rg[6] + rg[7]);
                    D_s[e.y] = dsum;
                } else {
                    dsum = D_s[e.y];
                }
                // the update's ratio in FP32 (an FP64 division here cost 0.6% of the loop,
                // profiles/r2/variants_r2.txt), the pass sum in FP64
                stage_sum[e.x] += dsum > 0.f ? double(__fdividef(nsum, dsum)) : 0.0;
            }
            if (MODE == kModeEPRY) {
                const float om = fmaxf(fmaxf(rg[8], rg[9]), fmaxf(rg[10], rg[11]));
                const float pm = fmaxf(fmaxf(rg[12], rg[13]), fmaxf(rg[14], rg[15]));
                inv_omax = (om > 0.f && bright) ? __fdividef(args.beta, om) : 0.f;  // bright-field pupil steps only
                inv_pmax = pm > 0.f ? __fdividef(args.alpha, pm) : 0.f;
            }
            // EPRY: the scatter's old canvas values, loaded under pass 1's step 2
            constexpr bool kOEarly = !FPM_O_STAGE && FPM_O_EARLY && MODE == kModeEPRY && PRUNE;
            float2 Oe[kOEarly ? NP : 1];
            if constexpr (kOEarly) {
#pragma unroll
                for (int q = 0; q < NP; ++q) Oe[q] = cv[Lat::a(q) * 8 * N + 16 * Lat::j(q)];
            }
            fft_second(v, T_s, p, h, sg, tw, twsw, PRUNE, true);

            // ---- scatter into the canvas disk (recon.cpp:127-130) / EPRY update
            if (MODE == kModeGS) {
#pragma unroll
                for (int q = 0; q < NP; ++q)
                    if ((mask >> q) & 1u)
                        cv[Lat::a(q) * 8 * N + 16 * Lat::j(q)] = cmulc(v[Lat::a(q)][Lat::j(q)], P_s[q * kGroupThreads + tl]);
            } else {
                const bool upd_o = inv_pmax > 0.f, upd_p = inv_omax > 0.f;
                pupil_dirty = upd_p;
                if constexpr (FPM_O_STAGE && MODE == kModeEPRY && PRUNE && G == 1 && MEAS == kMeasTMA)
                    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own slots
                // dark-field updates (the large majority) take no pupil step: a block-uniform
                // branch into a scatter without the pupil arithmetic
                auto epry_scatter = [&](auto upd_p_tag) {
                constexpr bool kUpdP = decltype(upd_p_tag)::value;
#pragma unroll
                for (int c0 = 0; c0 < NP; c0 += 8) {
                    float2 Ov[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if constexpr (FPM_O_STAGE && MODE == kModeEPRY && PRUNE && G == 1 && MEAS == kMeasTMA)
                            Ov[q] = reinterpret_cast<const float2*>(I_s)[(c0 + q) * kGroupThreads + tl];
                        else if constexpr (kOSm)
                            Ov[q] = O_sm[(c0 + q) * kGroupThreads + tl];
                        else if constexpr (kOEarly)
                            Ov[q] = Oe[c0 + q];
                        else
                            Ov[q] = cv[Lat::a(c0 + q) * 8 * N + 16 * Lat::j(c0 + q)];
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int qq = c0 + q;
                        const bool on = (mask >> qq) & 1u;
                        const float2 O = Ov[q];
                        const float2 P = P_s[qq * kGroupThreads + tl];
                        // with P' = sP and Psi' = s v: d' = s d, conj(P') d' = conj(P) d,
                        // P'_new = P' + beta conj(O) d' / max|O|^2 (s = checkerboard sign)
                        const float2 d = csub(v[Lat::a(qq)][Lat::j(qq)], cmul(O, P));
                        if (on && upd_o)
                            cv[Lat::a(qq) * 8 * N + 16 * Lat::j(qq)] = cfma(inv_pmax, cmulc(d, P), O);
                        if constexpr (kUpdP)
                            if (on) P_s[qq * kGroupThreads + tl] = cfma(inv_omax, cmulc(d, O), P);
                    }
                }
                };
                if (upd_p)
                    epry_scatter(std::true_type{});
                else
                    epry_scatter(std::false_type{});
            }
        }
        __syncthreads();  // slot barrier: canvas writes visible to the next update's gather
        if (G == 1 && ++c_pos == L) {
            c_pos = 0;
            ++c_it;
        }
    }

    // ---- per-pass mean residual; EPRY pupil back to global
    if (queue) {
        if (threadIdx.x == 0)  // a pass's last part stores the mean, earlier parts the running sum
            args.residuals[size_t(tile) * args.iters + it_q] = part == H - 1 ? stage_sum[it_q] / double(L) : stage_sum[it_q];
        if (it_q == 0)
            for (int k = s_begin + int(threadIdx.x); k < s_end; k += blockDim.x) args.isum[size_t(tile) * L + k] = D_s[k];
    } else {
        store_residuals(args, tile, stage_sum, G == 1);
    }
    if (MODE == kModeEPRY && g == 0) {
#pragma unroll
        for (int q = 0; q < NP; ++q)
            if ((mask >> q) & 1u)
                pupil_g[(tr + 8 * Lat::a(q)) * 64 + tc + 8 * (2 * Lat::j(q) + h)] = cscale(P_s[q * kGroupThreads + tl], sgn);
    }
    }  // items
}

// FPM_B200_QUEUE: unset = work queue when the tiles exceed the resident CTAs;
// 0 = never; 1 = always (tests: a grid wider than the tile count exercises the
// dependency waits)
static int queue_override() {
    const char* e = std::getenv("FPM_B200_QUEUE");
    return e && e[0] ? (e[0] == '1' ? 1 : 0) : -1;
}

template <int MODE, bool PRUNE, int MEAS, int G, int N, int MINB>
static cudaError_t launch_loop_t(const CUtensorMap* tmap, const LoopArgs& a0, int T, cudaStream_t s) {
    const size_t smem = loop_smem_bytes(G, a0.nslots, a0.L, a0.iters);
    auto k = a0.jitter > 0 ? fpm_loop64<MODE, PRUNE, MEAS, G, N, MINB, true> : fpm_loop64<MODE, PRUNE, MEAS, G, N, MINB, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    LoopArgs a = a0;
    int grid = T;
    const int q = queue_override();
    if (G == 1 && a.work && a.isum && q != 0) {
        int dev = 0, sms = 0, per_sm = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kGroupThreads * G, smem)) != cudaSuccess)
            return e;
        const int resident = std::max(1, per_sm * sms);
        if (T > resident || q == 1) {
            // parts per pass: the fewest (<= 4) that fill the last round of items best
            const double items = double(T) * a.iters;
            double best = 0.0;
            a.parts = 1;
            for (int h = 1; h <= 4 && h <= a.L; ++h) {
                const double rounds = items * h / resident;
                const double fill = rounds / std::ceil(rounds);
                if (fill > best + 0.005) {
                    best = fill;
                    a.parts = h;
                }
            }
            if (const char* pe = std::getenv("FPM_B200_PARTS"); pe && pe[0]) a.parts = std::max(1, std::min(a.L, std::atoi(pe)));
            grid = q == 1 ? std::min(resident, T * a.iters * a.parts) : resident;
            if ((e = cudaMemsetAsync(a.work, 0, sizeof(int) * size_t(T + 1), s)) != cudaSuccess) return e;
        } else {
            a.work = nullptr;
        }
    } else {
        a.work = nullptr;
    }
    k<<<grid, kGroupThreads * G, smem, s>>>(*tmap, a);
    return cudaGetLastError();
}

// Register budget by batch: with at most 4 tiles per SM to share (T <= 4 x SMs),
// the 255-register build's shorter update latency wins (config 3 sharded over 8
// GPUs, 128 tiles: 10.6 -> 9.0 ms; 512 tiles: 20.8 -> 19.1 ms); a full FOV needs
// the 4-tiles-per-SM build (1,024 tiles: 33.2 vs 38.0 ms). FPM_B200_MINB=2|4 forces.
static int loop_minb(int G, int T) {
    if (G != 1) return 4;
    if (const char* e = std::getenv("FPM_B200_MINB"); e && e[0]) return e[0] == '2' ? 2 : 4;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return T <= 4 * sms ? 2 : 4;
}

cudaError_t launch_loop64(int mode, bool prune, int meas, int G, const CUtensorMap* tmap, const LoopArgs& a, int T,
                          cudaStream_t s) {
    const int minb = meas == kMeasTMA ? loop_minb(G, a.batch_T > 0 ? a.batch_T : T) : 4;
#define FPM_LOOP_CASE(M, P, ME, GG, NN)                                                        \
    if (mode == M && prune == P && meas == ME && G == GG && a.N == NN) {                       \
        if (GG == 1 && ME == kMeasTMA && P && minb == 2)                                       \
            return launch_loop_t<M, P, ME, GG, NN, (GG == 1 && ME == kMeasTMA && P) ? 2 : 4>(tmap, a, T, s); \
        return launch_loop_t<M, P, ME, GG, NN, FPM_LOOP_MINB>(tmap, a, T, s);                    \
    }
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
    return cudaErrorNotSupported;  // no instantiation for this geometry
}

}  // namespace fpmk
