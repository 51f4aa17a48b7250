// Kernel launch interface shared by capi.cu and kernels.cu.
#pragma once

#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fpmk {

// FPM_B200_MID=0: the n = 256 box / cluster kernels without the [64, 192) box
// pruning of WarpFFT256 (tests compare the two)
inline bool mid_disabled() {
    const char* e = std::getenv("FPM_B200_MID");
    return e && e[0] == '0';
}

enum { kModeGS = 0, kModeEPRY = 1 };

// Checked build (make check -> lib/libfpm_b200_check.so, -DFPM_CHECK=1): every
// kernel asserts the indices of its global and shared accesses (tile, origin,
// frame, work item, slab row / owner, measurement slot) and traps on a
// violation — the bounds half of compute-sanitizer's memcheck, which this GPU
// pool does not allow (profiles/r2/compute_sanitizer_refused.txt). The
// production build compiles the checks out.
#ifndef FPM_CHECK
#define FPM_CHECK 0
#endif
#if FPM_CHECK
#define FPM_ASSERT(c)                                                                                     \
    do {                                                                                                  \
        if (!(c)) {                                                                                       \
            printf("FPM_ASSERT %s:%d (%s) block %d thread %d\n", __FILE__, __LINE__, #c, int(blockIdx.x), \
                   int(threadIdx.x));                                                                     \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define FPM_ASSERT(c) \
    do {              \
    } while (0)
#endif

// Layout of the TMA-staged 64 x 64 u16 measurement crop (n = 64 loop kernels):
// 1 = 128B swizzle (16-byte chunk c of row r at chunk c ^ (r & 7)), 0 = row-major.
// Row-major: every read of a thread's 32 pixels is an immediate offset from one
// per-thread base, with the same 2-way bank pattern as the swizzled reads.
#ifndef FPM_MEAS_SWIZZLE
#define FPM_MEAS_SWIZZLE 0
#endif
enum { kMeasTMA = 0, kMeasF32 = 1 };

// Per-tile LED loop (K1 fused update + K4 persistent loop). One CTA per tile,
// G groups of 64 threads; group g runs entry g of each schedule slot.
struct LoopArgs {
    float2* canvas;           // [T][N][N] spectrum canvases (in/out)
    float2* pupils;           // [T][n][n] pupils (in; out for EPRY)
    const uint8_t* support;   // [n][n] pupil support disk (optics.cpp:59-60)
    const short2* origins;    // [T][L] sub-aperture origin (r0, c0) = N/2 + (oy, ox) - n/2
    const uint8_t* bright;    // [T][L] EPRY: 1 iff the disk holds the zero frequency (pupil step)
    const int* seq_frame;     // [L] frame index of sequence position
    const int2* tile_xy;      // [T] (x0, y0) of the LR crop
    double* residuals;        // [T][iters] pass mean residual (recon.cpp:165)
    const float* meas_f32;    // kMeasF32: [n][n] intensities (update_step API)
    const int2* slots;        // G > 1: [num_slots][G] (stage, position), stage < 0 = idle
    int num_slots;            // G == 1: iters * L (implicit slots)
    int slot_begin;           // run slots [slot_begin, num_slots) (G == 1; 0 for a whole run)
    int resid_accumulate;     // residuals of the stages touched are added to (online passes)
    int T, L, iters, N, nslots;
    float alpha, beta;        // EPRY step sizes
    // Work queue (G == 1, whole runs, more tiles than resident CTAs): a persistent
    // grid pulls (pass, part, tile) items in that order; work[0] is the item
    // counter, work[1 + t] the items of tile t completed (zeroed per launch)
    int* work;                // nullptr: one CTA per tile, the whole slot range
    float* isum;              // [T][L] sum(I) of each LED's crop, formed by the pass-0 items
    int parts;                // work queue: items per pass (a pass's LED range cut into parts)
    int batch_T;              // tiles sharing the GPU with this launch (concurrent bands); 0 = T
    int jitter;               // > 0: race hunting, every warp sleeps 0..jitter ns per update / item
    unsigned jitter_seed;
    int F;                    // frames in the LR stack (checked build: seq_frame bounds)
};

// Line FFTs for init_canvas / canvas_to_field (K2 / K3).
struct LinesArgs {
    const float2* src;        // [T][N][N]
    float2* dst;              // [T][N][N]
    const float2* tw;         // [N] forward twiddles W_N^m
    const uint16_t* frame;    // init rows: LR frame base (seed frame), row pitch below
    long long pitch;          // elements
    const int2* tile_xy;      // [T]
    int n, up;
    float scale;
    // finalize cols only: tile t's HR field written at dst + out_off[t] with row
    // pitch out_pitch (elements) — straight into a mosaic (or a peer GPU's
    // mosaic) when the tiles abut without overlap; nullptr = dst[t][N][N]
    const long long* out_off;
    long long out_pitch;
    // N = 256 canvas box (launch_lines_box): the LED loop only ever touches rows and
    // columns [box0, box0 + boxn) of a canvas, so init_canvas forms the spectrum there
    // only and canvas_to_field transforms only the change there:
    // field = U + up^2 ifft2(canvas - canvas0), U = bilinear(sqrt(seed crop))
    int box0, boxn;
    float2* canvas0;          // [T][boxn][boxn] init spectrum over the box
};

// General tile sides (n = 64, 128, 256): warp-FFT row/column passes over the
// pupil's bounding box (kernels_box.cu).
struct BoxArgs {
    float2* scratch;            // [T][box][n + 1] intermediate when it does not fit shared memory
    const uint16_t* frames;     // LR stack base, [F][H][pitch]
    long long pitch;            // elements
    long long frame_stride;     // elements per frame
    int box, b0;                // pupil bounding box: rows/cols [b0, b0 + box)
    const short2* sup_rows;     // [n] support columns [x, y) of each row (a disk: one run per row)
};
size_t box_smem_bytes(int n, int box, int L, int iters, bool scratch_in_smem);
cudaError_t launch_loop_box(int n, int mode, const LoopArgs& a, const BoxArgs& b, int T, cudaStream_t s);

// One tile split over a cluster of cl CTAs (kernels_cluster.cu).
size_t cluster_smem_bytes(int n, int box, int cl, int nw, int L, int iters);
int cluster_warps(int n, int cl);
bool cluster_supported(int n, int N, int cl);
cudaError_t launch_loop_cluster(int n, int mode, int cl, const LoopArgs& a, const BoxArgs& b, int T,
                                cudaStream_t s);

size_t loop_smem_bytes(int G, int nslots, int L, int iters);

// n = 64 with 256 threads per tile (kernels_quad.cu): sequential schedules whose
// pupil disk lies in rows/cols [16, 48) of the block, TMA-staged measurements.
size_t loop64q_smem_bytes(int L, int iters, bool osep);
cudaError_t launch_loop64q(int mode, const CUtensorMap* tmap, const LoopArgs& a, int T, cudaStream_t s);


#ifdef __CUDACC__
// Schedule perturbation for race hunting (FPM_B200_JITTER=<ns>[:<seed>]): each warp
// sleeps a pseudo-random 0..jitter ns before every update and work-queue claim, so a
// missing barrier, fence or dependency wait shows up as run-to-run bit differences
// (tests/test_race_jitter.py; compute-sanitizer is closed on the GPU pool).
// JIT is a template flag of every loop kernel: the production instantiations
// compile the hook out (the runtime test alone cost 1.2% of the config-3 loop,
// profiles/r2/jitter_cost.txt); the launchers pick the JIT ones only when
// FPM_B200_JITTER is set.
template <bool JIT>
__device__ __forceinline__ void jitter_sleep(const LoopArgs& a, int step) {
    if constexpr (!JIT) return;
    if (a.jitter > 0) {
        unsigned h = a.jitter_seed ^ (blockIdx.x * 0x9E3779B1u) ^ (unsigned(step) * 0x85EBCA77u) ^
                     ((threadIdx.x >> 5) * 0xC2B2AE3Du);
        h ^= h >> 15;
        h *= 0x2C1B3C6Du;
        h ^= h >> 12;
        __nanosleep(h % unsigned(a.jitter));
    }
}

// Per-pass mean residuals of the stages a launch touched (all of them for a
// whole run; a stage range for the online passes, accumulated).
__device__ __forceinline__ void store_residuals(const LoopArgs& a, int tile, const double* stage_sum, bool ranged) {
    const int k0 = ranged ? a.slot_begin / a.L : 0;
    const int k1 = ranged ? (a.num_slots - 1) / a.L : a.iters - 1;
    for (int k = k0 + int(threadIdx.x); k <= k1; k += blockDim.x) {
        double* r = a.residuals + size_t(tile) * a.iters + k;
        *r = (a.resid_accumulate ? *r : 0.0) + stage_sum[k] / double(a.L);
    }
}
#endif
cudaError_t launch_loop64(int mode, bool prune, int meas, int G, const CUtensorMap* tmap,
                          const LoopArgs& a, int T, cudaStream_t s);
// which: 0 init rows (frame -> canvas), 1 init cols, 2 finalize rows, 3 finalize cols
cudaError_t launch_lines(int which, int N, const LinesArgs& a, int T, cudaStream_t s);
// the box-pruned passes for N = 256 (a.box0, a.boxn multiples of 16; which as above)
cudaError_t launch_lines_box(int which, const LinesArgs& a, int T, cudaStream_t s);
// batched 2-D complex128 FFT, sides with factors 2, 3, 5 up to 4096 (fft_c128.cu)
bool fft_c128_supported(int n);
cudaError_t fft2_c128(double2* data, double2* tmp, long long batch, int rows, int cols, bool inv, cudaStream_t s);
cudaError_t launch_build_pupils(float2* pupils, const uint8_t* support, const double* defocus,
                                int n, int T, double dk, double inv_l2, cudaStream_t s);

}  // namespace fpmk
