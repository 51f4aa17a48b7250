// fpm_loop64w: the fused per-LED update for n = 64 with ONE WARP PER TILE,
// persistent over the LED loop (reconstruct_tile, recon.cpp:161-166); each
// update replaces update_step (recon.cpp:93-134).
//
// Every lane holds a whole 64-point line in registers (fft64_reg.cuh: radix
// 8 x 8, compile-time twiddles from __constant__ memory), so a transform has
// no shuffles and the tile needs no CTA barrier: the lanes hand lines to each
// other through one shared-memory buffer X (32 x 64, row stride 66) under
// __syncwarp. The pupil disk (radius 14.6 px) lies in rows/cols [16, 48) of
// the 64 x 64 block, and the 2-D transforms visit only what the update needs:
//   1  gather: lane l loads block row 16 + l (its support run) x P', the
//      centring checkerboard (-1)^(i+j) folded into P' (fft2 = C FFT(C x),
//      field.cpp:48-87), conjugated (IFFT(x) = conj(FFT(conj x)));
//      row IFFT (input rows pruned: n1 in [2, 6)) -> X[l][0..64)
//   2  per column c in {l, l + 32}: column IFFT over X's 32 rows (pruned) ->
//      modulus with sqrt(I) + residual sums (recon.cpp:115-124) -> column FFT
//      keeping output rows [16, 48) -> back into X[.][c]
//   3  row FFT of X[l] keeping columns [16, 48) -> scatter into the disk:
//      GS write-back (recon.cpp:127-130) or EPRY
// So per update the warp runs 1 + 2 + 2 + 1 line FFTs of 64 points, every one
// pruned on its input or output side (32 of the 64 rows of each 2-D transform
// are never transformed at all). The LR crop is read straight into registers
// (coalesced u16 loads, L2 evict-first), one column ahead. 27 KB of shared
// memory per tile: 8 tiles (8 warps, 2 per scheduler) per SM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fft64_reg.cuh"
#include "kernels.cuh"

namespace fpmk {

namespace {

constexpr unsigned kFullW = 0xffffffffu;
constexpr int kXS = 66;  // X row stride (float2): 16-byte rows, conflict-free row and column access
constexpr int kPS = 33;  // pupil row stride (float2)

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ldg_u16_ef(const uint16_t* a, uint64_t pol) {
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ long long opaque(long long v) {
    asm volatile("mov.b64 %0, %0;" : "+l"(v));
    return v;
}
// shared-memory load the compiler may not reuse across the update: keeps the 32
// pupil values of the gather from being held in registers until the scatter
__device__ __forceinline__ float2 lds_f2(const float2* p) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                 : "=f"(v.x), "=f"(v.y)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* a) {
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
}
__device__ __forceinline__ void st_release_gpu_w(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu_w(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

size_t loop_w64_smem_bytes(int L, int iters) {
    size_t b = size_t(32) * kXS * sizeof(float2);  // X: line hand-off buffer
    b += size_t(32) * kPS * sizeof(float2);         // P' over the 32 x 32 disk box
    b += size_t(iters) * sizeof(double);            // stage sums
    b += size_t(L) * (sizeof(short2) + sizeof(float) + 1);  // origins, sum(I), bright flags
    b += 16;                                        // work-queue item, alignment
    return b;
}

template <int MODE, int N>
__global__ void __launch_bounds__(32, 8) fpm_loop64w(const LoopArgs args, const BoxArgs bx) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int l = threadIdx.x;
    const int L = args.L;
    float2* X_s = reinterpret_cast<float2*>(smem_raw);
    float2* P_s = X_s + 32 * kXS;  // [32][kPS]: P' = (-1)^(i+j) P at block (16 + r, 16 + c), 0 off the support
    double* stage_sum = reinterpret_cast<double*>(P_s + 32 * kPS);
    short2* O_s = reinterpret_cast<short2*>(stage_sum + args.iters);
    float* D_s = reinterpret_cast<float*>(O_s + L);  // sum(I) per LED, formed on its first visit
    uint8_t* B_s = reinterpret_cast<uint8_t*>(D_s + L);
    int* item_s = reinterpret_cast<int*>(smem_raw + ((size_t(B_s + L - smem_raw) + 3) & ~size_t(3)));

    const uint64_t pol = evict_first_policy();
    const float inv_n2 = 1.0f / 4096.0f;  // ifft2's 1/(rows*cols) (field.cpp:64-66)
    const bool queue = args.work != nullptr;
    const int H = queue ? args.parts : 1;
    const int n_items = args.T * args.iters * H;

    for (int round = 0;; ++round) {
        int tile, it_q = 0, part = 0, s_begin, s_end;
        if (queue) {
            // items j = (it * H + part) * T + tile; item j depends on item j - T (see fpm_loop64)
            __syncwarp();
            if (l == 0) {
                if (round > 0) {
                    const int jp = *item_s;
                    __threadfence();
                    st_release_gpu_w(args.work + 1 + jp % args.T, jp / args.T + 1);
                }
                const int j = atomicAdd(args.work, 1);
                *item_s = j;
                if (j < n_items && j >= args.T) {
                    const int* flag = args.work + 1 + (j % args.T);
                    while (ld_acquire_gpu_w(flag) < j / args.T) __nanosleep(256);
                    __threadfence();
                }
            }
            __syncwarp();
            const int j = *item_s;
            if (j >= n_items) break;
            tile = j % args.T;
            const int ip = j / args.T;
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

        // ---- per-tile setup: P' of this lane's box row, support run, origins, flags
        float2* canvas = args.canvas + size_t(tile) * N * N;
        float2* pupil_g = args.pupils + size_t(tile) * 64 * 64;
        const int2 txy = args.tile_xy[tile];
        const int bi = 16 + l;  // this lane's block row in the row phases
        uint32_t mask = 0;
#pragma unroll 4
        for (int c = 0; c < 32; ++c) {
            const int bj = 16 + c;
            const bool on = args.support[bi * 64 + bj] != 0;
            mask |= uint32_t(on) << c;
            const float sg = ((bi + bj) & 1) ? -1.f : 1.f;
            P_s[l * kPS + c] = on ? cscale(pupil_g[bi * 64 + bj], sg) : make_float2(0.f, 0.f);
        }
        for (int k = l; k < L; k += 32) {
            O_s[k] = args.origins[size_t(tile) * L + k];
            B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
            if (queue && it_q > 0) D_s[k] = args.isum[size_t(tile) * L + k];
        }
        for (int k = l; k < args.iters; k += 32)
            stage_sum[k] = queue && part > 0 && k == it_q ? args.residuals[size_t(tile) * args.iters + k] : 0.0;
        __syncwarp();

        bool pupil_dirty = true;  // EPRY: max|P|^2 changes only after a pupil step
        float pmax = 0.f, omax = 0.f;
        const uint16_t* frames0 = bx.frames + size_t(txy.y) * bx.pitch + txy.x;

        for (int s = s_begin; s < s_end; ++s) {
            const int it = s / L, pos = s - it * L;
            const short2 o = O_s[pos];
            const uint16_t* Ib = frames0 + size_t(args.seq_frame[pos]) * bx.frame_stride;
            // the crop's 64 rows into L2 now; each column pass loads its column just before its IFFT
            prefetch_l2(Ib + size_t(l) * bx.pitch);
            prefetch_l2(Ib + size_t(l) * bx.pitch + 63);
            prefetch_l2(Ib + size_t(l + 32) * bx.pitch);
            prefetch_l2(Ib + size_t(l + 32) * bx.pitch + 63);

            // ---- 1: gather row 16 + l of the disk block x P', conjugated; row IFFT
            float2 x[8][8];
            float2* cv = canvas + size_t(o.x + bi) * N + o.y + 16;
            const bool bright = MODE == kModeEPRY && B_s[pos];
            float om = 0.f;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float2 O = ((mask >> c) & 1u) ? cv[c] : make_float2(0.f, 0.f);
                if (bright) om = fmaxf(om, cabs2(O));
                const float2 g = cmul(O, lds_f2(P_s + l * kPS + c));
                x[(16 + c) >> 3][(16 + c) & 7] = make_float2(g.x, -g.y);
            }
            if (MODE == kModeEPRY) {
                if (bright) {
#pragma unroll
                    for (int sh = 16; sh; sh >>= 1) om = fmaxf(om, __shfl_xor_sync(kFullW, om, sh));
                    omax = om;
                }
                if (pupil_dirty) {
                    float pm = 0.f;
#pragma unroll 8
                    for (int c = 0; c < 32; ++c) pm = fmaxf(pm, cabs2(lds_f2(P_s + l * kPS + c)));
#pragma unroll
                    for (int sh = 16; sh; sh >>= 1) pm = fmaxf(pm, __shfl_xor_sync(kFullW, pm, sh));
                    pmax = pm;
                }
            }
            fft64_nt<true, false>(x, s >> 30);  // x[k0][k1] = column k0 + 8 k1
#pragma unroll
            for (int k = 0; k < 64; k += 2)
                *reinterpret_cast<float4*>(X_s + l * kXS + k) =
                    make_float4(x[k & 7][k >> 3].x, x[k & 7][k >> 3].y, x[(k + 1) & 7][k >> 3].x, x[(k + 1) & 7][k >> 3].y);
            __syncwarp();

            // ---- 2: columns l and l + 32: IFFT -> modulus -> FFT (rows [16, 48) kept)
            const bool first = queue ? it_q == 0 : s - args.slot_begin < L;
            float num = 0.f;
            uint32_t den_u = 0;
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                const int c = l + 32 * half;
#pragma unroll
                for (int r = 0; r < 32; ++r) x[(16 + r) >> 3][(16 + r) & 7] = X_s[r * kXS + c];
                fft64_nt<true, false>(x, (s + half) >> 30);  // x[k0][k1] = conj(u), u = FFT2(C conj g) at row k0 + 8 k1
                // the column's measurement (L2-resident since the update's prefetch), loaded after
                // the IFFT: the FFT's temporaries and the 64 values are never live together
                uint32_t Iv[64];
                {
                    // addresses by a running pointer whose stride is opaque to the compiler,
                    // so it cannot hoist 64 precomputed row offsets into registers
                    const uint16_t* pr = Ib + c;
                    const long long st = opaque(bx.pitch);
#pragma unroll
                    for (int r = 0; r < 64; ++r) {
                        Iv[r] = ldg_u16_ef(pr, pol);
                        pr += st;
                    }
                }
                const float sgc = (c & 1) ? -1.f : 1.f;
#pragma unroll
                for (int k0 = 0; k0 < 8; ++k0) {
                    // branch-free |e| = 0 rule (recon.cpp:122), as in fpm_loop64: a nudge of
                    // sgn 2^-60 (sgn = (-1)^(row + c)) maps e = 0 to the checkerboarded sqrt(I) + 0i
                    const float eps = ((k0 & 1) ? -sgc : sgc) * 0x1p-60f;
#pragma unroll
                    for (int k1 = 0; k1 < 8; ++k1) {
                        const int row = k0 + 8 * k1;
                        const uint32_t Iu = Iv[row];
                        if (first) den_u += Iu;
                        const float meas = sqrt_ftz(float(Iu));
                        const float2 uu = x[k0][k1];
                        const float ux = uu.x + eps;
                        const float m2 = fmaf(ux, ux, uu.y * uu.y);
                        const float rr = rsqrt_ftz(fmaxf(m2, kTiny));
                        const float dm = fmaf(m2 * rr, inv_n2, -meas);  // |e| - sqrt(I)
                        num = fmaf(dm, dm, num);
                        const float sc = meas * rr;
                        x[k0][k1] = make_float2(ux * sc, -uu.y * sc);
                    }
                }
                fft64_tn<true>(x, (s + half) >> 30);  // x[k1][k0] = row k0 + 8 k1, k1 in [2, 6)
#pragma unroll
                for (int k1 = 2; k1 < 6; ++k1)
#pragma unroll
                    for (int k0 = 0; k0 < 8; ++k0) X_s[(k0 + 8 * k1 - 16) * kXS + c] = x[k1][k0];
            }
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) num += __shfl_xor_sync(kFullW, num, sh);
            float den = float(den_u);
            if (first) {
#pragma unroll
                for (int sh = 16; sh; sh >>= 1) den += __shfl_xor_sync(kFullW, den, sh);
            }
            __syncwarp();
            if (l == 0) {
                float dsum;
                if (first) {
                    D_s[pos] = den;
                    dsum = den;
                } else {
                    dsum = D_s[pos];
                }
                // the ratio in float (an inline reciprocal, not the double-division subroutine),
                // accumulated in double like the reference's pass mean
                stage_sum[it] += dsum > 0.f ? double(num * __frcp_rn(dsum)) : 0.0;
            }

            // ---- 3: row FFT of X[l] (columns [16, 48) kept) -> scatter
#pragma unroll
            for (int k = 0; k < 64; k += 2) {
                const float4 q = *reinterpret_cast<const float4*>(X_s + l * kXS + k);
                x[k >> 3][k & 7] = make_float2(q.x, q.y);
                x[(k + 1) >> 3][(k + 1) & 7] = make_float2(q.z, q.w);
            }
            fft64_nt<false, true>(x, s >> 30);  // x[k0][k1] = column k0 + 8 k1, k1 in [2, 6)
            if (MODE == kModeGS) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if ((mask >> c) & 1u) cv[c] = cmulc(x[(16 + c) & 7][(16 + c) >> 3], lds_f2(P_s + l * kPS + c));
            } else {
                // bright-field pupil steps only; __fdividef: no division subroutine (and its
                // register saves) inside the update loop
                const float inv_omax = (omax > 0.f && bright) ? __fdividef(args.beta, omax) : 0.f;
                const float inv_pmax = pmax > 0.f ? __fdividef(args.alpha, pmax) : 0.f;
                const bool upd_o = inv_pmax > 0.f, upd_p = inv_omax > 0.f;
                pupil_dirty = upd_p;
#pragma unroll
                for (int c0 = 0; c0 < 32; c0 += 8) {
                    float2 Ov[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        Ov[q] = ((mask >> (c0 + q)) & 1u) ? cv[c0 + q] : make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int c = c0 + q;
                        const bool on = (mask >> c) & 1u;
                        const float2 O = Ov[q];
                        const float2 P = lds_f2(P_s + l * kPS + c);
                        // with P' = sP and Psi' = s v: d' = s d, conj(P') d' = conj(P) d (see fpm_loop64)
                        const float2 d = csub(x[(16 + c) & 7][(16 + c) >> 3], cmul(O, P));
                        if (on && upd_o) cv[c] = cadd(O, cscale(cmulc(d, P), inv_pmax));
                        if (on && upd_p) P_s[l * kPS + c] = cadd(P, cscale(cmulc(d, O), inv_omax));
                    }
                }
            }
            __syncwarp();  // canvas rows visible to the lanes of the next update's gather
        }

        // ---- per-pass mean residual; EPRY pupil back to global
        if (queue) {
            if (l == 0)
                args.residuals[size_t(tile) * args.iters + it_q] =
                    part == H - 1 ? stage_sum[it_q] / double(L) : stage_sum[it_q];
            if (it_q == 0)
                for (int k = s_begin - it_q * L + l; k < s_end - it_q * L; k += 32) args.isum[size_t(tile) * L + k] = D_s[k];
        } else {
            store_residuals(args, tile, stage_sum, true);
        }
        if (MODE == kModeEPRY) {
#pragma unroll 4
            for (int c = 0; c < 32; ++c)
                if ((mask >> c) & 1u) {
                    const float sg = ((bi + 16 + c) & 1) ? -1.f : 1.f;
                    pupil_g[bi * 64 + 16 + c] = cscale(lds_f2(P_s + l * kPS + c), sg);
                }
        }
    }  // items
}

namespace {

template <int MODE, int N>
cudaError_t launch_w64_t(const LoopArgs& a0, const BoxArgs& b, int T, cudaStream_t s) {
    const size_t smem = loop_w64_smem_bytes(a0.L, a0.iters);
    auto k = fpm_loop64w<MODE, N>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    LoopArgs a = a0;
    int grid = T;
    const char* qe = std::getenv("FPM_B200_QUEUE");
    const int q = qe && qe[0] ? (qe[0] == '1' ? 1 : 0) : -1;
    if (a.work && a.isum && q != 0) {
        int dev = 0, sms = 0, per_sm = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem)) != cudaSuccess) return e;
        const int resident = std::max(1, per_sm * sms);
        // static launch: T CTAs in ceil(T / resident) waves; queue: T * iters * parts items
        const double waves = std::ceil(double(T) / resident);
        const double fill_static = double(T) / (waves * resident);
        double best = 0.0;
        int parts = 1;
        for (int h = 1; h <= 4 && h <= a.L; ++h) {
            const double rounds = double(T) * a.iters * h / resident;
            const double fill = rounds / std::ceil(rounds);
            if (fill > best + 0.005) {
                best = fill;
                parts = h;
            }
        }
        if (const char* pe = std::getenv("FPM_B200_PARTS"); pe && pe[0]) parts = std::max(1, std::min(a.L, std::atoi(pe)));
        (void)fill_static;
        if (q == 1 || T > resident) {  // T <= resident: at most T chains, the static launch is as full
            a.parts = parts;
            grid = q == 1 ? std::min(resident, T * a.iters * parts) : resident;
            if ((e = cudaMemsetAsync(a.work, 0, sizeof(int) * size_t(T + 1), s)) != cudaSuccess) return e;
        } else {
            a.work = nullptr;
        }
    } else {
        a.work = nullptr;
    }
    k<<<grid, 32, smem, s>>>(a, b);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_loop_w64(int mode, const LoopArgs& a, const BoxArgs& b, int T, cudaStream_t s) {
#define FPM_W64_CASE(M, NN) \
    if (mode == M && a.N == NN) return launch_w64_t<M, NN>(a, b, T, s);
    FPM_W64_CASE(kModeGS, 256)
    FPM_W64_CASE(kModeEPRY, 256)
    FPM_W64_CASE(kModeGS, 512)
    FPM_W64_CASE(kModeEPRY, 512)
    FPM_W64_CASE(kModeGS, 1024)
    FPM_W64_CASE(kModeEPRY, 1024)
#undef FPM_W64_CASE
    return cudaErrorNotSupported;
}

}  // namespace fpmk
