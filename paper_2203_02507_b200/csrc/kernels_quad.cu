// fpm_loop64q: the fused per-LED update for n = 64 with 256 threads per tile
// ("quad lattice"), persistent over the LED loop (reconstruct_tile,
// recon.cpp:161-166); each update replaces update_step (recon.cpp:93-134).
//
// Same algorithm and arithmetic as fpm_loop64 (kernels.cu), with each tile's
// 4096 pixels spread over twice the threads: thread t = 4p + 2hr + hc,
// p = 8tr + tc, owns the 16 pixels (tr + 8(2i + hr), tc + 8(2j + hc)),
// i, j in [0, 4), in registers v[i][j]. A 64-point DFT factors as 8 x 8
// (n = 8 n1 + n0, k = k0 + 8 k1):
//   step 1: 8-point DFTs over n1 of both axes for residue (n0r, n0c) = (tr, tc);
//           each axis split over a lane pair by the parity of n1 (decimation in
//           time: DFT4 per lane, W8 twiddle, one shuffle exchange — partner
//           lane ^ 2 for rows, ^ 1 for columns);
//   twiddle W64^(n0r k0r + n0c k0c), one 32 KB shared-memory transpose (rows of
//           the 64 frequency pairs (k0r, k0c), slots of the 64 residues,
//           XOR-swizzled: conflict-free writes and 4-wavefront 128-bit reads);
//   step 2: 8-point DFTs over n0 of both axes, each split over the pair by
//           contiguous halves (decimation in frequency), which returns the
//           output in the parity-split layout step 1 consumes.
// Twice the warps per tile halve each thread's share of an update, so a lone
// tile on an SM (strong-scaled ranks: 128 tiles on 148 SMs) runs its update at
// up to twice the pair lattice's speed, and a full FOV keeps more warps per
// scheduler to hide shuffle, shared-memory and barrier latency.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "ptx_util.cuh"

namespace fpmk {

namespace {

constexpr unsigned kFullQ = 0xffffffffu;
constexpr int kQThreads = 256;
constexpr int kQIBytes = 64 * 64 * 2;  // staged u16 measurement, TMA 128B-swizzled
constexpr int kQTBytes = 64 * 64 * 8;  // transpose buffer
constexpr int kQNP = 4;                // pupil-disk lattice positions per thread (i, j in {1, 2})

__device__ __forceinline__ float2 shfl_x(float2 x, int m) {
    return make_float2(__shfl_xor_sync(kFullQ, x.x, m), __shfl_xor_sync(kFullQ, x.y, m));
}

// v * (-i) on the odd lane of a pair, v on the even one (W8^2 of the pair combine)
__device__ __forceinline__ float2 mul_mi_h(float2 v, int h) {
    const float nx = __int_as_float(__float_as_int(v.x) ^ int(0x80000000u));
    return h ? make_float2(v.y, nx) : v;
}

// Per-lane constants of one pair direction (rows: partner ^ 2, columns: ^ 1).
struct PairK {
    int h;        // this lane's half
    float sg;     // +1 even lane, -1 odd lane
    float kh;     // rotation gate: 1 on the odd lane
    float c1, c3; // step-1 combine factors (the even lane's +-sqrt(2) rides on the step-1 twiddle)
    float s1, s3; // step-2 W8^1 / W8^3 scales of the rotations (1 on the even lane)
};

__device__ __forceinline__ PairK pair_k(int h) {
    const float r = 0.70710678118654752440f;
    PairK k;
    k.h = h;
    k.sg = h ? -1.f : 1.f;
    k.kh = h ? 1.f : 0.f;
    k.c1 = h ? -r : 1.41421356237309504880f;
    k.c3 = h ? r : -1.41421356237309504880f;
    k.s1 = h ? r : 1.f;
    k.s3 = h ? -r : 1.f;
    return k;
}

// Step 1 pair combine (DIT) of the four DFT4 outputs F[m] of this lane:
// X[m] = F0[m] + W8^m F1[m] (even lane), X[m + 4] = F0[m] - W8^m F1[m] (odd lane).
// W8^1, W8^3 are rotations R (one FFMA2 on the odd lane) whose 1/sqrt(2) the odd
// lane applies in the combine and the even lane defers to the step-1 twiddle.
__device__ __forceinline__ void dit_pair(float2& w0, float2& w1, float2& w2, float2& w3, int xm, const PairK& k) {
    w1 = cfma_v(make_float2(k.kh, -k.kh), make_float2(w1.y, w1.x), w1);  // odd: R1 = (x + y, y - x) = sqrt(2) W8 x
    w2 = mul_mi_h(w2, k.h);
    w3 = cfma_v(make_float2(-k.kh, k.kh), make_float2(w3.y, w3.x), w3);  // odd: (x - y, x + y) = -sqrt(2) W8^3 x
    w0 = cfma(k.sg, w0, shfl_x(w0, xm));
    w1 = cfma(k.c1, w1, shfl_x(w1, xm));
    w2 = cfma(k.sg, w2, shfl_x(w2, xm));
    w3 = cfma(k.c3, w3, shfl_x(w3, xm));
}

// Step 2 pair split (DIF) over this lane's half x[i] (even: i, odd: i + 4):
// even lane x[i] + x[i + 4], odd lane (x[i] - x[i + 4]) W8^i.
__device__ __forceinline__ void dif_pair(float2& x0, float2& x1, float2& x2, float2& x3, int xm, const PairK& k) {
    x0 = cfma(k.sg, x0, shfl_x(x0, xm));
    x1 = cfma(k.sg, x1, shfl_x(x1, xm));
    x2 = cfma(k.sg, x2, shfl_x(x2, xm));
    x3 = cfma(k.sg, x3, shfl_x(x3, xm));
    x1 = cscale(cfma_v(make_float2(k.kh, -k.kh), make_float2(x1.y, x1.x), x1), k.s1);  // W8 x = R1 / sqrt(2)
    x2 = mul_mi_h(x2, k.h);
    x3 = cscale(cfma_v(make_float2(-k.kh, k.kh), make_float2(x3.y, x3.x), x3), k.s3);  // W8^3 x = -(x - y, x + y) / sqrt(2)
}

// One forward 64 x 64 transform in the quad layout (the inverse runs as
// conj(FFT(conj x)), the conjugations folded into gather and modulus).
// PIN: only i, j in {1, 2} hold data on entry (the disk block of the IFFT);
// POUT: only outputs i, j in {1, 2} are formed (the disk the scatter reads).
template <bool PIN, bool POUT>
__device__ __forceinline__ void fft64x64_quad(float2 (&v)[4][4], float2* T_s, const float2* Wr_s, const float2* Wc_s,
                                              int t, int tr, int tc, const PairK& kr, const PairK& kc) {
    // ---- step 1 rows: DFT4 over i (n1r = 2i + hr) per column, pair over hr
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (PIN && (j == 0 || j == 3)) continue;  // columns without data stay zero until the column DFT
        if (PIN)
            dft4_z03<false>(v[0][j], v[1][j], v[2][j], v[3][j]);
        else
            dft4<false>(v[0][j], v[1][j], v[2][j], v[3][j]);
        dit_pair(v[0][j], v[1][j], v[2][j], v[3][j], 2, kr);
    }
    // ---- step 1 columns: DFT4 over j (n1c = 2j + hc) per row, pair over hc
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        if (PIN)
            dft4_z03<false>(v[m][0], v[m][1], v[m][2], v[m][3]);
        else
            dft4<false>(v[m][0], v[m][1], v[m][2], v[m][3]);
        dit_pair(v[m][0], v[m][1], v[m][2], v[m][3], 1, kc);
    }
    // ---- twiddle W64^(tr k0r + tc k0c), k0r = 4hr + m, k0c = 4hc + n; tables pre-scaled by the
    // even lanes' deferred +-1/sqrt(2); entries (w, (-w.y, w.x))
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const float2 w = Wr_s[(m * 2 + kr.h) * 8 + tr];
#pragma unroll
        for (int n = 0; n < 4; ++n) v[m][n] = cmul2(v[m][n], w);
    }
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        const float2 w = Wc_s[n * 16 + tc * 2 + kc.h];
#pragma unroll
        for (int m = 0; m < 4; ++m) v[m][n] = cmul2(v[m][n], w);
    }
    // ---- transpose: element (k0r, k0c) of residue p = 8tr + tc -> row 8k0r + k0c, slot
    // tswz_q(k0r, k0c, p) = p ^ 2k0c ^ 4(k0r >> 2) ^ 8(p >> 5): every half-warp of a 64-bit
    // store and every quarter-warp of a 128-bit load hits distinct bank groups
    const int p = 8 * tr + tc;
    const int wx = 8 * (tr >> 2);
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            const int k0c = 4 * kc.h + n;
            T_s[(8 * (4 * kr.h + m) + k0c) * 64 + (p ^ (2 * k0c) ^ (4 * kr.h) ^ wx)] = v[m][n];
        }
    __syncthreads();
    // ---- read row t >> 2 = (k0r, k0c) = (tr, tc): slots (n0r, n0c) = (4hr + i, 4hc + j)
    {
        const float2* row = T_s + (t >> 2) * 64;
        const int x = (2 * tc) ^ (4 * (tr >> 2)) ^ (8 * kr.h);  // slot bit 5 = hr here
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int s = 32 * kr.h + 8 * i + 4 * kc.h;
            const float4 q0 = *reinterpret_cast<const float4*>(row + (s ^ x));
            const float4 q1 = *reinterpret_cast<const float4*>(row + ((s + 2) ^ x));
            v[i][0] = make_float2(q0.x, q0.y);
            v[i][1] = make_float2(q0.z, q0.w);
            v[i][2] = make_float2(q1.x, q1.y);
            v[i][3] = make_float2(q1.z, q1.w);
        }
    }
    // ---- step 2 rows: pair split over hr (DIF), DFT4 over i -> k1r = 2i + hr
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        dif_pair(v[0][j], v[1][j], v[2][j], v[3][j], 2, kr);
        if (POUT)
            dft4_o12<false>(v[0][j], v[1][j], v[2][j], v[3][j]);
        else
            dft4<false>(v[0][j], v[1][j], v[2][j], v[3][j]);
    }
    // ---- step 2 columns: pair split over hc, DFT4 over j -> k1c = 2j + hc
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (POUT && (i == 0 || i == 3)) continue;
        dif_pair(v[i][0], v[i][1], v[i][2], v[i][3], 1, kc);
        if (POUT)
            dft4_o12<false>(v[i][0], v[i][1], v[i][2], v[i][3]);
        else
            dft4<false>(v[i][0], v[i][1], v[i][2], v[i][3]);
    }
}

}  // namespace

size_t loop64q_smem_bytes(int L, int iters, bool osep) {
    size_t b = 1024;                                           // alignment slack (128B-swizzled TMA box)
    if (osep) b += size_t(kQNP) * kQThreads * sizeof(float2);  // EPRY scatter operands, own buffer
    b += kQIBytes + kQTBytes;                                  // staging + transpose
    b += size_t(kQNP) * kQThreads * sizeof(float2);            // lattice pupil [NP][256]
    b += 128 * sizeof(float4);                                 // row + column twiddle tables
    b += size_t(iters) * sizeof(double);                       // stage sums
    b += sizeof(uint64_t) + 32 * sizeof(float);                // mbarrier + reductions
    b += size_t(L) * (sizeof(short2) + sizeof(int) + sizeof(float) + 1);
    b += 8;                                                    // work-queue item
    return b;
}

template <int MODE, int N, int MINB, bool JIT>
__global__ void __launch_bounds__(kQThreads, MINB)
    fpm_loop64q(const __grid_constant__ CUtensorMap tmap, const LoopArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((base + 1023u) & ~1023u) - base);
    const int t = threadIdx.x;
    const int p = t >> 2, tr = p >> 3, tc = p & 7;
    const int hr = (t >> 1) & 1, hc = t & 1;
    const int warp = t >> 5;
    const int L = args.L;

    uint16_t* I_s = reinterpret_cast<uint16_t*>(smem);
    float2* T_s = reinterpret_cast<float2*>(smem + kQIBytes);
    size_t off = kQIBytes + kQTBytes;
    float2* P_s = reinterpret_cast<float2*>(smem + off);  // [NP][256], P' = (-1)^(i+j) P, 0 off the support
    off += size_t(kQNP) * kQThreads * sizeof(float2);
    float2* Wr_s = reinterpret_cast<float2*>(smem + off);  // [m][hr][tr]: W64^(tr (4hr + m)), pre-scaled
    float2* Wc_s = Wr_s + 64;                              // [n][tc][hc]: W64^(tc (4hc + n)), pre-scaled
    off += 128 * sizeof(float4);
    double* stage_sum = reinterpret_cast<double*>(smem + off);
    off += size_t(args.iters) * sizeof(double);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + off);
    off += sizeof(uint64_t);
    float* rg = reinterpret_cast<float*>(smem + off);  // num[8], den[8], omax[8], pmax[8]
    off += 32 * sizeof(float);
    short2* O_s = reinterpret_cast<short2*>(smem + off);
    off += size_t(L) * sizeof(short2);
    int* F_s = reinterpret_cast<int*>(smem + off);
    off += size_t(L) * sizeof(int);
    float* D_s = reinterpret_cast<float*>(smem + off);
    off += size_t(L) * sizeof(float);
    uint8_t* B_s = smem + off;
    off += size_t(L);
    off = (off + 3) & ~size_t(3);
    int* item_s = reinterpret_cast<int*>(smem + off);
    off += 8;
    // low-occupancy build (MINB = 2, the strong-scaled batches): the EPRY scatter's old
    // canvas values get their own buffer, so the next crop's TMA can still be issued a
    // whole FFT ahead (otherwise they reuse the measurement staging buffer)
    constexpr bool kOSep = MINB == 2;
    float2* Ostg = kOSep ? reinterpret_cast<float2*>(smem + ((off + 15) & ~size_t(15))) : reinterpret_cast<float2*>(I_s);

    // ---- one-time setup: twiddle tables (the even lanes' m = 1, 3 entries carry +-1/sqrt(2)), mbarrier
    if (t < 128) {
        const int half = t >> 6, e = t & 63;
        int m, h, r;  // row table: e = (m * 2 + h) * 8 + tr; column table: e = m * 16 + tc * 2 + h
        if (half == 0) {
            m = e >> 4;
            h = (e >> 3) & 1;
            r = e & 7;
        } else {
            m = e >> 4;
            r = (e >> 1) & 7;
            h = e & 1;
        }
        const int ex = (r * (4 * h + m)) & 63;
        double s, c;
        sincospi(-double(ex) / 32.0, &s, &c);
        const double f = (h == 0 && (m & 1)) ? (m == 1 ? 0.70710678118654752440 : -0.70710678118654752440) : 1.0;
        Wr_s[t] = make_float2(float(c * f), float(s * f));  // float2 entries: cmul2
    }
    const PairK kr = pair_k(hr), kc = pair_k(hc);
    if (t == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const float sgn = ((tr + tc) & 1) ? -1.f : 1.f;  // checkerboard (-1)^(i+j), constant per thread
    const float inv_n2 = 1.0f / 4096.0f;
    uint32_t phase = 0;
    const int cbase = (tr + 8 * hr) * N + tc + 8 * hc;  // canvas offset of (i, j) = (0, 0)
    const bool queue = args.work != nullptr;
    const int H = queue ? args.parts : 1;
    const int n_items = args.T * args.iters * H;

    for (int round = 0;; ++round) {
    int tile, it_q = 0, part = 0, s_begin, s_end;
    if (queue) {  // work queue over (pass, part, tile) items: the fpm_loop64 protocol (kernels.cu)
        __syncthreads();
        if (t == 0) {
            if (round > 0) {
                const int jp = *item_s;
                __threadfence();
                st_release_gpu(args.work + 1 + jp % args.T, jp / args.T + 1);
            }
            jitter_sleep<JIT>(args, -1 - round);
            const int j = atomicAdd(args.work, 1);
            *item_s = j;
            if (j < n_items && j >= args.T) {
                const int* flag = args.work + 1 + (j % args.T);
                while (ld_acquire_gpu(flag) < j / args.T) __nanosleep(256);
                __threadfence();
            }
        }
        __syncthreads();
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
    FPM_ASSERT(tile >= 0 && tile < args.T && s_begin >= 0 && s_end <= args.num_slots);

    // ---- per-tile setup: support mask, lattice pupil, origins, frame map, flags
    float2* canvas = args.canvas + size_t(tile) * N * N;
    float2* pupil_g = args.pupils + size_t(tile) * 64 * 64;
    const int2 txy = args.tile_xy[tile];
    uint32_t mask = 0;
#pragma unroll
    for (int q = 0; q < kQNP; ++q) {
        const int i = 1 + (q >> 1), j = 1 + (q & 1);
        const int r = tr + 8 * (2 * i + hr), c = tc + 8 * (2 * j + hc);
        const bool on = args.support[r * 64 + c] != 0;
        mask |= uint32_t(on) << q;
        P_s[q * kQThreads + t] = on ? cscale(pupil_g[r * 64 + c], sgn) : make_float2(0.f, 0.f);
    }
    for (int k = t; k < L; k += kQThreads) {
        O_s[k] = args.origins[size_t(tile) * L + k];
        F_s[k] = args.seq_frame[k];
        B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
        if (queue && it_q > 0) D_s[k] = args.isum[size_t(tile) * L + k];
    }
    for (int k = t; k < args.iters; k += kQThreads)
        stage_sum[k] = queue && part > 0 && k == it_q ? args.residuals[size_t(tile) * args.iters + k] : 0.0;
    __syncthreads();

    bool issued = false;
    bool pupil_dirty = true;
    auto issue = [&](int led) {
        if (t == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, kQIBytes);
            FPM_ASSERT(led >= 0 && led < L && F_s[led] >= 0 && (args.F == 0 || F_s[led] < args.F));
            tma_load_crop(I_s, &tmap, bar, txy.x, txy.y, F_s[led]);
        }
    };
    int c_it = s_begin / L, c_pos = s_begin - c_it * L;
    for (int s = s_begin; s < s_end; ++s) {
        jitter_sleep<JIT>(args, s);
        if (!issued) issue(c_pos);
        issued = false;
        const short2 o = O_s[c_pos];
        FPM_ASSERT(c_pos >= 0 && c_pos < L && c_it >= 0 && c_it < args.iters && o.x >= 0 && o.y >= 0 &&
                   o.x + 64 <= N && o.y + 64 <= N);
        float2* cv = canvas + size_t(o.x) * N + o.y + cbase;

        // ---- gather the disk x P' (conjugated: the IFFT runs as conj(FFT(conj x)))
        float2 v[4][4];
#pragma unroll
        for (int q = 0; q < kQNP; ++q) v[1 + (q >> 1)][1 + (q & 1)] = cv[(q >> 1) * 16 * N + 16 * (q & 1) + 16 * N + 16];
        const bool bright = MODE == kModeEPRY && B_s[c_pos];
        if (bright) {
            float omax = 0.f;
#pragma unroll
            for (int q = 0; q < kQNP; ++q)
                omax = fmaxf(omax, ((mask >> q) & 1u) ? cabs2(v[1 + (q >> 1)][1 + (q & 1)]) : 0.f);
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) omax = fmaxf(omax, __shfl_xor_sync(kFullQ, omax, sh));
            if ((t & 31) == 0) rg[16 + warp] = omax;
        }
        if (MODE == kModeEPRY && pupil_dirty) {
            float pmax = 0.f;
#pragma unroll
            for (int q = 0; q < kQNP; ++q) pmax = fmaxf(pmax, cabs2(P_s[q * kQThreads + t]));
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(kFullQ, pmax, sh));
            if ((t & 31) == 0) rg[24 + warp] = pmax;
        }
#pragma unroll
        for (int q = 0; q < kQNP; ++q) {
            float2& x = v[1 + (q >> 1)][1 + (q & 1)];
            x = cmul_conj(x, P_s[q * kQThreads + t]);
        }

        // ---- centred inverse transform (unscaled), modulus replacement
        fft64x64_quad<true, false>(v, T_s, Wr_s, Wc_s, t, tr, tc, kr, kc);
        mbar_wait(bar, phase);
        phase ^= 1u;
        const bool first = queue ? it_q == 0 : s - args.slot_begin < L;
        float num = 0.f;
        uint32_t den_u = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = tr + 8 * (2 * i + hr), cb = 2 * j + hc;
                const uint32_t Iu = I_s[r * 64 + ((FPM_MEAS_SWIZZLE ? cb ^ tr : cb) << 3) + tc];  // kernels.cuh
                if (first) den_u += Iu;
                const float Iv = float(Iu);
                const float meas = sqrt_ftz(Iv);
                const float2 uu = v[i][j];
                const float ux = uu.x + sgn * 0x1p-60f;  // |e| = 0 -> sqrt(I) + 0i (recon.cpp:122), signed
                const float m2 = fmaf(ux, ux, uu.y * uu.y);
                const float rr = rsqrt_ftz(fmaxf(m2, kTiny));
                const float dm = fmaf(m2 * rr, inv_n2, -meas);  // |e| - sqrt(I)
                num = fmaf(dm, dm, num);
                const float sc = meas * rr;
                v[i][j] = cscale(make_float2(ux, -uu.y), sc);  // one FMUL2
            }
        float den = float(den_u);
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) num += __shfl_xor_sync(kFullQ, num, sh);
        if (first) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) den += __shfl_xor_sync(kFullQ, den, sh);
        }
        if ((t & 31) == 0) {
            rg[warp] = num;
            rg[8 + warp] = den;
        }
        __syncthreads();  // staging and transpose buffers free; reductions visible

        // EPRY: the scatter's old canvas values into the free staging buffer (cp.async, under the FFT)
        constexpr bool kOStage = MODE == kModeEPRY;
        if constexpr (kOStage) {
#pragma unroll
            for (int q = 0; q < kQNP; ++q)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Ostg + q * kQThreads + t)),
                             "l"(cv + (q >> 1) * 16 * N + 16 * (q & 1) + 16 * N + 16)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if ((!kOStage || kOSep) && s + 1 < s_end) {
            issue(c_pos + 1 == L ? 0 : c_pos + 1);
            issued = true;
        }
        if (t == 0) {
            const float nsum = ((rg[0] + rg[1]) + (rg[2] + rg[3])) + ((rg[4] + rg[5]) + (rg[6] + rg[7]));
            float dsum;
            if (first) {
                dsum = ((rg[8] + rg[9]) + (rg[10] + rg[11])) + ((rg[12] + rg[13]) + (rg[14] + rg[15]));
                D_s[c_pos] = dsum;
            } else {
                dsum = D_s[c_pos];
            }
            stage_sum[c_it] += dsum > 0.f ? double(__fdividef(nsum, dsum)) : 0.0;  // as fpm_loop64
        }
        float inv_omax = 0.f, inv_pmax = 0.f;
        if (MODE == kModeEPRY) {
            const float om = fmaxf(fmaxf(fmaxf(rg[16], rg[17]), fmaxf(rg[18], rg[19])),
                                   fmaxf(fmaxf(rg[20], rg[21]), fmaxf(rg[22], rg[23])));
            const float pm = fmaxf(fmaxf(fmaxf(rg[24], rg[25]), fmaxf(rg[26], rg[27])),
                                   fmaxf(fmaxf(rg[28], rg[29]), fmaxf(rg[30], rg[31])));
            inv_omax = (om > 0.f && bright) ? args.beta / om : 0.f;  // bright-field pupil steps only
            inv_pmax = pm > 0.f ? args.alpha / pm : 0.f;
        }

        // ---- centred forward transform of the corrected field (outputs in the disk block only)
        fft64x64_quad<false, true>(v, T_s, Wr_s, Wc_s, t, tr, tc, kr, kc);

        // ---- scatter into the canvas disk (recon.cpp:127-130) / EPRY update
        if (MODE == kModeGS) {
#pragma unroll
            for (int q = 0; q < kQNP; ++q)
                if ((mask >> q) & 1u)
                    cv[(q >> 1) * 16 * N + 16 * (q & 1) + 16 * N + 16] =
                        cmulc(v[1 + (q >> 1)][1 + (q & 1)], P_s[q * kQThreads + t]);
        } else {
            const bool upd_o = inv_pmax > 0.f, upd_p = inv_omax > 0.f;
            pupil_dirty = upd_p;
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int q = 0; q < kQNP; ++q) {
                const bool on = (mask >> q) & 1u;
                const float2 O = Ostg[q * kQThreads + t];
                const float2 P = P_s[q * kQThreads + t];
                const float2 d = csub(v[1 + (q >> 1)][1 + (q & 1)], cmul(O, P));
                if (on && upd_o) cv[(q >> 1) * 16 * N + 16 * (q & 1) + 16 * N + 16] = cfma(inv_pmax, cmulc(d, P), O);
                if (on && upd_p) P_s[q * kQThreads + t] = cfma(inv_omax, cmulc(d, O), P);
            }
        }
        __syncthreads();  // canvas writes visible to the next update's gather; buffers free
        if (++c_pos == L) {
            c_pos = 0;
            ++c_it;
        }
    }

    // ---- per-pass mean residual; EPRY pupil back to global
    if (queue) {
        if (t == 0)
            args.residuals[size_t(tile) * args.iters + it_q] = part == H - 1 ? stage_sum[it_q] / double(L) : stage_sum[it_q];
        if (it_q == 0)
            for (int k = s_begin + t; k < s_end; k += kQThreads) args.isum[size_t(tile) * L + k] = D_s[k];
    } else {
        store_residuals(args, tile, stage_sum, true);
    }
    if (MODE == kModeEPRY) {
#pragma unroll
        for (int q = 0; q < kQNP; ++q)
            if ((mask >> q) & 1u) {
                const int i = 1 + (q >> 1), j = 1 + (q & 1);
                pupil_g[(tr + 8 * (2 * i + hr)) * 64 + tc + 8 * (2 * j + hc)] = cscale(P_s[q * kQThreads + t], sgn);
            }
    }
    }  // items
}

static int queue_override_q() {
    const char* e = std::getenv("FPM_B200_QUEUE");
    return e && e[0] ? (e[0] == '1' ? 1 : 0) : -1;
}

template <int MODE, int N, int MINB>
static cudaError_t launch_q_t(const CUtensorMap* tmap, const LoopArgs& a0, int T, cudaStream_t s) {
    const size_t smem = loop64q_smem_bytes(a0.L, a0.iters, MINB == 2);
    auto k = a0.jitter > 0 ? fpm_loop64q<MODE, N, MINB, true> : fpm_loop64q<MODE, N, MINB, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    LoopArgs a = a0;
    int grid = T;
    const int q = queue_override_q();
    if (a.work && a.isum && q != 0) {
        int dev = 0, sms = 0, per_sm = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kQThreads, smem)) != cudaSuccess) return e;
        const int resident = std::max(1, per_sm * sms);
        if (T > resident || q == 1) {
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
    k<<<grid, kQThreads, smem, s>>>(*tmap, a);
    return cudaGetLastError();
}

cudaError_t launch_loop64q(int mode, const CUtensorMap* tmap, const LoopArgs& a, int T, cudaStream_t s) {
    // the low-occupancy build only (128 registers, up to 2 tiles per SM): the quad lattice
    // pays off for batches of at most one tile per SM (strong-scaled ranks)
#define FPMQ_CASE(M, NN) \
    if (mode == M && a.N == NN) return launch_q_t<M, NN, 2>(tmap, a, T, s);
    FPMQ_CASE(kModeGS, 256) FPMQ_CASE(kModeGS, 512) FPMQ_CASE(kModeGS, 1024)
    FPMQ_CASE(kModeEPRY, 256) FPMQ_CASE(kModeEPRY, 512) FPMQ_CASE(kModeEPRY, 1024)
#undef FPMQ_CASE
    return cudaErrorNotSupported;
}

}  // namespace fpmk
