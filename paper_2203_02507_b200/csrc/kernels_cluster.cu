// fpm_loop_cluster: the fused per-LED update with one tile split over a
// thread-block cluster of CL CTAs (distributed shared memory), persistent over
// the LED loop. Same arithmetic as fpm_loop_box (kernels_box.cu), so the two
// produce the same canvas bit for bit; what changes is where the work runs:
//
//   A  the CTA's box rows (row i belongs to CTA (o.x + i) mod CL: ownership by
//      absolute canvas row): gather the disk x P', IFFT (warp F2), send each
//      row's n outputs to the CTAs owning those columns — column slab c holds
//      columns [c n/CL, (c+1) n/CL) of all B box rows. n <= 128: st.async into
//      the owner's shared memory, counted in bytes on its mbarrier; n = 256:
//      DSMEM stores + cluster barrier
//   B  the CTA's own columns: IFFT over the box rows (F1) -> modulus with
//      sqrt(I) -> FFT (F2) -> keep the box rows; the measurement slab (staged
//      one update ahead by cp.async, pair-XOR swizzled) gives conflict-free
//      modulus reads
//   -- cluster barrier -- (residual and EPRY maxima reduced over the cluster)
//   C  the same rows as A: fetch the row from the column slabs (DSMEM loads),
//      FFT (F1), scatter into the canvas disk (GS / EPRY)
//   -- CTA barrier (a canvas row's next reader may be another warp of the
//      CTA); a cluster barrier only after a pupil step (pupil rows move with the
//      box rows) or, with a single slab buffer (n = 256), to free the slabs
//
// Slabs and partial sums are double-buffered for n <= 128. Use: n = 256
// tiles, whose B x n intermediate (240 KB) does not fit one SM, and
// single-tile runs, where one CTA would leave 147 SMs idle (BASELINE config 2).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "warp_fft.cuh"

namespace cg = cooperative_groups;

#ifndef FPM_CL_DENSEP
#define FPM_CL_DENSEP 1  // whole runs: sum(I) formed on pass 0 only (a separate loop), cached per (tile, LED)
#endif
#ifndef FPM_CL_ST8
#define FPM_CL_ST8 1  // n = 256: measurement slab staged by 8-byte cp.async (column XOR on groups of four)
#endif
#ifndef FPM_CL_ASY256
#define FPM_CL_ASY256 0  // n = 256, one slab buffer: phase-A rows by st.async counted on an mbarrier
#endif
#ifndef FPM_CL_SPLIT
#define FPM_CL_SPLIT 0  // n = 256: first-row loads between barrier.cluster.arrive and wait
#endif
#ifndef FPM_CL_GATE
#define FPM_CL_GATE 0  // EPRY maxima only when needed (bright update / pupil changed)
#endif
#ifndef FPM_CL_DB256
#define FPM_CL_DB256 0  // n = 256 on 8-CTA clusters: double-buffered slabs (st.async + mbarrier, no end-of-update barrier)
#endif
#ifndef FPM_CL_PF8
#define FPM_CL_PF8 1  // n = 256: the next row's disk loads in flight in registers (phase A; with the MID pruning only 4 registers: 484 vs 516 ms)
#endif

namespace fpmk {

#ifndef FPM_CL_STAGE_C
#define FPM_CL_STAGE_C 1  // n = 256: phase-C scatter operands staged the same way, under the row's FFT
#endif
#ifndef FPM_CL_STAGE
#define FPM_CL_STAGE 0  // 1: n = 256 on the shuffle FFT with canvas/pupil box rows staged one row ahead by cp.async
#endif

// n = 256: per warp the 16 x 17 transpose buffer of WarpFFT256 (FPM_CL_STAGE=1, the
// round-2 shuffle FFT: one box row of canvas and pupil staged per warp instead, box
// columns rounded up to 16 so the XOR swizzle below stays inside each group of 16)
__host__ __device__ static size_t row_stage_bytes(int n, int box, int nw) {
    if (n != 256) return 0;
    return FPM_CL_STAGE ? size_t(nw) * 2 * size_t((box + 15) & ~15) * sizeof(float2)
                        : size_t(nw) * WarpFFT256<false>::kBufFloat2 * sizeof(float2);
}

size_t cluster_smem_bytes(int n, int box, int cl, int nw, int L, int iters) {
    const size_t sw = size_t(n / cl);
    const size_t nbuf = (n <= 128 || (FPM_CL_DB256 && n == 256 && cl >= 8)) ? 2 : 1;  // double-buffered slabs
    size_t b = nbuf * size_t(box) * (sw + 1) * sizeof(float2);  // column slab(s) of the box rows
    b += sw * size_t(n) * sizeof(uint16_t);               // measurement slab
    b += size_t(n) * sizeof(short2);                      // support run per row
    b = (b + 15) & ~size_t(15);
    b += row_stage_bytes(n, box, nw);                     // phase-A row staging (n = 256)
    b += size_t(iters) * sizeof(double) + 2 * sizeof(uint64_t);
    b += nbuf * size_t(nw) * 4 * sizeof(float) + 4 * sizeof(float);
    b += size_t(L) * (sizeof(short2) + sizeof(uint16_t) + 1) + 16;
    b += 8;  // work-queue item
    return b;
}

namespace {

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t map_rank(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// asynchronous store of 8 bytes into another CTA's shared memory; completion is
// counted in bytes on that CTA's mbarrier (no release fence on this side)
__device__ __forceinline__ void st_async_f2(uint32_t raddr, float2 v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "f"(v.x), "f"(v.y), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NLR, int MODE, int NC, int CL, int NW, bool JIT, bool MID>
__global__ void __launch_bounds__(NW * 32, NLR <= 128 ? 16 / NW : 512 / (NW * 32)) fpm_loop_cluster(const LoopArgs args, const BoxArgs bx) {
    constexpr int M = NLR / 32;
    constexpr int SW = NLR / CL;  // columns per CTA
    constexpr int RS = SW + 1;    // slab row stride (float2): column reads conflict-free
    constexpr int NT = NW * 32;
    constexpr bool PF = M <= 4 || (FPM_CL_PF8 && !(FPM_CL_STAGE && NLR == 256));  // next row's disk loads in flight
#ifndef FPM_CL_PFC8
#define FPM_CL_PFC8 1
#endif
    constexpr bool PFC = M <= 4 || (FPM_CL_PFC8 && !(FPM_CL_STAGE && NLR == 256));  // phase C: scatter operands loaded before the FFT
    // DB: two slab / reduction buffers used alternately, so an update's phase A never
    // overwrites what the previous update's phase C still reads: no end-of-update barrier
    constexpr bool DB = NLR <= 128 || (FPM_CL_DB256 && NLR == 256 && CL >= 8);
    constexpr bool ASY = DB || (FPM_CL_ASY256 && NLR == 256);  // phase-A sends by st.async + mbarrier
    constexpr bool SPLIT = FPM_CL_SPLIT && NLR == 256 && !DB;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = int(cluster.block_rank());
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int L = args.L, B = bx.box, b0 = bx.b0;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* sp = smem_raw;
    float2* S0 = reinterpret_cast<float2*>(sp);
    sp += size_t(B) * RS * sizeof(float2);
    float2* S1 = S0;
    if (DB) {
        S1 = reinterpret_cast<float2*>(sp);
        sp += size_t(B) * RS * sizeof(float2);
    }
    uint16_t* I_s = reinterpret_cast<uint16_t*>(sp);  // [row][column ^ isw(row)]
    sp += size_t(SW) * NLR * sizeof(uint16_t);
    short2* SR = reinterpret_cast<short2*>(sp);  // support run [x, y) of each row
    sp += size_t(NLR) * sizeof(short2);
    sp = smem_raw + ((sp - smem_raw + 15) & ~15);
    constexpr bool STG = FPM_CL_STAGE && NLR == 256;
    using FFT = std::conditional_t<STG, WarpFFT<M>, typename WarpFFTSel<M, MID>::type>;
    const int RBW = (B + 15) & ~15;  // staged row width (box columns, XOR-swizzled in groups of 16)
    float2* RB = reinterpret_cast<float2*>(sp) + size_t(w) * 2 * RBW;  // STG: this warp's [canvas | pupil] row
    float2* TB = reinterpret_cast<float2*>(sp) + size_t(w) * FFT::kBufFloat2;  // else: its FFT transpose buffer
    sp += row_stage_bytes(NLR, B, NW);
    double* stage_sum = reinterpret_cast<double*>(sp);
    sp += size_t(args.iters) * sizeof(double);
    uint64_t* mbA = reinterpret_cast<uint64_t*>(sp);  // DB: phase-A slab arrivals, one per parity
    sp += 2 * sizeof(uint64_t);
    float* wred0 = reinterpret_cast<float*>(sp);  // [warp][4]: num, den, omax, pmax
    sp += NW * 4 * sizeof(float);
    float* wred1 = wred0;
    if (DB) {
        wred1 = reinterpret_cast<float*>(sp);
        sp += NW * 4 * sizeof(float);
    }
    float* upd = reinterpret_cast<float*>(sp);  // inv_omax, inv_pmax of the current update
    sp += 4 * sizeof(float);
    short2* O_s = reinterpret_cast<short2*>(sp);
    sp += size_t(L) * sizeof(short2);
    uint16_t* F_s = reinterpret_cast<uint16_t*>(sp);  // frame of each position (< 65536, capi.cu)
    sp += size_t(L) * sizeof(uint16_t);
    uint8_t* B_s = sp;
    sp += size_t(L);
    sp = smem_raw + ((sp - smem_raw + 3) & ~3);
    int* item_s = reinterpret_cast<int*>(sp);  // work queue: the cluster's current item (rank 0's copy)

    for (int k = threadIdx.x; k < NLR; k += NT) SR[k] = bx.sup_rows[k];
    for (int k = threadIdx.x; k < L; k += NT) F_s[k] = uint16_t(args.seq_frame[k]);
    FFT F;
    F.init(l, NLR, TB);
    const float inv_n2 = 1.0f / float(NLR * NLR);
    if (ASY && threadIdx.x == 0) {
        mbar_init1(mbA);
        mbar_init1(mbA + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();  // every CTA of the cluster is resident before any DSMEM access

    // work queue (sequential whole runs, more tiles than resident clusters): items
    // j = it * T + tile, claimed by rank 0 and read by every CTA through DSMEM; item j
    // depends on item j - T (the tile's previous pass), claimed 3.5 rounds earlier at
    // BASELINE config 5. Every update runs the same instructions as in the
    // one-cluster-per-tile launch: bit-identical
    const bool queue = args.work != nullptr;
    const int n_items = args.T * args.iters;
    int par = 0;
    uint32_t nupd = 0;  // updates run by this CTA (mbarrier phase of buffer `par` = (nupd >> 1) & 1)
    for (int round = 0;; ++round) {
    int tile, it_q = 0;
    if (queue) {
        if (rank == 0 && threadIdx.x == 0) {
            if (round > 0) {  // release: the previous item's canvas/pupil writes (cluster barrier below)
                const int jp = *item_s;
                __threadfence();
                asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(args.work + 1 + jp % args.T), "r"(jp / args.T + 1)
                             : "memory");
            }
            jitter_sleep<JIT>(args, -1 - round);
            const int j = atomicAdd(args.work, 1);
            if (j < n_items && j >= args.T) {  // acquire: the tile's previous pass is complete
                const int* flag = args.work + 1 + (j % args.T);
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                    if (v < j / args.T) __nanosleep(256);
                } while (v < j / args.T);
            }
            *item_s = j;
        }
        cluster.sync();
        const int j = *cluster.map_shared_rank(item_s, 0);
        if (threadIdx.x == 0) __threadfence();
        cluster.sync();  // every CTA has read the item before rank 0 claims the next
        if (j >= n_items) break;
        tile = j % args.T;
        it_q = j / args.T;
    } else {
        if (round > 0) break;
        tile = blockIdx.x / CL;
    }
    FPM_ASSERT(tile >= 0 && tile < args.T && rank >= 0 && rank < CL);
    float2* canvas = args.canvas + size_t(tile) * NC * NC;
    float2* pupil = args.pupils + size_t(tile) * NLR * NLR;
    const int2 txy = args.tile_xy[tile];
    for (int k = threadIdx.x; k < L; k += NT) {
        O_s[k] = args.origins[size_t(tile) * L + k];
        B_s[k] = MODE == kModeEPRY ? args.bright[size_t(tile) * L + k] : 0;
    }
    for (int k = threadIdx.x; k < args.iters; k += NT) stage_sum[k] = 0.0;
    __syncthreads();

    // schedule entries: sequential slot e = (e / L, e % L); pipelined slots hold two
    // entries each (stage < 0 = idle), run back to back
    const int G = args.slots ? 2 : 1;
    const int e_end = queue ? (it_q + 1) * L : args.num_slots * G;
    auto entry_at = [&](int e, int& it, int& pos) -> bool {
        if (G == 1) {
            it = e / L;
            pos = e % L;
            return true;
        }
        const int2 en = args.slots[e];
        it = en.x;
        pos = en.y;
        return en.x >= 0;
    };
    auto next_entry = [&](int e) -> int {
        int a, b;
        for (int f = e + 1; f < e_end; ++f)
            if (entry_at(f, a, b)) return f;
        return -1;
    };
    // measurement slab of one update: rows r, columns rank SW + jj at [r][jj ^ isw(r)]
    // (XOR on pairs: the modulus reads of rows k0 + M t land in distinct banks); staged
    // asynchronously one update ahead by 4-byte cp.async, consumed only by phase B
    const bool even_x = ((txy.x + rank * SW) & 1) == 0;
    // ST8 (WarpFFT256): 8-byte copies, the column XOR on groups of four (4 p): the modulus
    // reads of one register then cover 16 bank pairs (2-way), half the copy instructions
    constexpr bool ST8 = FPM_CL_ST8 && NLR == 256 && !STG;
    auto isw_k = [&](int r) -> int { return (ST8 ? 4 * (r & 15) : FFT::isw(r)) & (SW - 1); };
    const bool quad_x = ((txy.x + rank * SW) & 3) == 0 && (bx.pitch & 3) == 0 && (bx.frame_stride & 3) == 0 &&
                        (reinterpret_cast<uintptr_t>(bx.frames) & 7) == 0;  // every copy source 8-byte aligned
    auto stage = [&](int pos) {
        const uint16_t* fr =
            bx.frames + size_t(F_s[pos]) * bx.frame_stride + size_t(txy.y) * bx.pitch + txy.x + rank * SW;
        if (ST8 && quad_x) {
            static_assert(!ST8 || NT % (SW / 4) == 0, "stage: whole rows per pass");
            const int jq = 4 * (int(threadIdx.x) % (SW / 4));
            const uint16_t* src = fr + jq;
            for (int r = int(threadIdx.x) / (SW / 4); r < NLR; r += NT / (SW / 4))
                cp_async8(I_s + r * SW + (jq ^ isw_k(r)), src + size_t(r) * bx.pitch);
            cp_async_commit();
        } else if (even_x) {
            // thread t: column pair t mod SW/2 of rows t / (SW/2) + k NT / (SW/2) (no division per copy)
            static_assert(NT % (SW / 2) == 0, "stage: whole rows per pass");
            const int jp = 2 * (int(threadIdx.x) % (SW / 2));
            const uint16_t* src = fr + jp;
            for (int r = int(threadIdx.x) / (SW / 2); r < NLR; r += NT / (SW / 2))
                cp_async4(I_s + r * SW + (jp ^ isw_k(r)), src + size_t(r) * bx.pitch);
            cp_async_commit();
        } else {
            for (int idx = threadIdx.x; idx < NLR * SW; idx += NT) {
                const int r = idx / SW, jj = idx % SW;
                I_s[r * SW + (jj ^ isw_k(r))] = fr[size_t(r) * bx.pitch + jj];
            }
        }
    };
    int e = next_entry((queue ? it_q * L : args.slot_begin * G) - 1);
    bool pdirty = true;  // GATE: max|P|^2 changes only after a pupil step
    if (e >= 0) {
        int it0, pos0;
        entry_at(e, it0, pos0);
        stage(pos0);
    }
    float2 Oa[M], Pa[M];  // phase-A prefetch (SPLIT: loaded under the previous update's end barrier)
    bool a_loaded = false;
    for (; e >= 0;) {
        jitter_sleep<JIT>(args, e);
        int it, pos;
        entry_at(e, it, pos);
        float2* const S = par ? S1 : S0;
        float* const wred = par ? wred1 : wred0;
        // DB: this update's slab arrives by st.async, counted on mbA[par] (B rows x SW columns)
        if (ASY && threadIdx.x == 0) mbar_arm(mbA + par, uint32_t(B) * SW * sizeof(float2));
        const int e_next = next_entry(e);
        const short2 o = O_s[pos];
        FPM_ASSERT(pos >= 0 && pos < L && it >= 0 && it < args.iters && o.x >= 0 && o.y >= 0 && o.x + NLR <= NC &&
                   o.y + NLR <= NC && (args.F == 0 || F_s[pos] < args.F));
        float2* cv = canvas + size_t(o.x) * NC + o.y;
        // box rows are owned by canvas row (o.x + i) mod CL: a CTA reads in phase A only
        // canvas rows it wrote itself in earlier phases C, so consecutive updates need no
        // cross-CTA ordering of canvas memory (the disk moves with the LED)
        const int rfirst = b0 + ((rank - (int(o.x) + b0) % CL) % CL + CL) % CL;
        const bool bright = MODE == kModeEPRY && B_s[pos] != 0;
        const bool want_o = MODE == kModeEPRY && (bright || !FPM_CL_GATE);
        const bool want_p = MODE == kModeEPRY && (pdirty || !FPM_CL_GATE);

        // ---- A: IFFT of this CTA's box rows, outputs to the column owners
        // the disk loads of a warp's next row are issued before the current row's FFT
        // (n <= 128; the n = 256 kernel has no register room for a second row)
        float omax = 0.f, pmax = 0.f;
        auto load_row_at = [&](const float2* cvp, int ii) {
            const short2 run = SR[ii];
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int c = F.a_in(k0);
                const bool on = FFT::live(k0) && c >= run.x && c < run.y;
                Oa[k0] = on ? cvp[size_t(ii) * NC + c] : make_float2(0.f, 0.f);
                Pa[k0] = on ? pupil[ii * NLR + c] : make_float2(0.f, 0.f);
            }
        };
        auto load_row = [&](int ii) { load_row_at(cv, ii); };
        // n = 256: the warp's next box row (canvas and pupil over the box columns) is staged
        // into its row buffer by cp.async while the current row transforms; slot x ^ ((x >> 4) & 15)
        // makes the gather's stride-8 reads conflict-free (a half-warp's stride-16 columns land
        // in 16 distinct bank pairs)
        auto rb_slot = [](int x) { return x ^ ((x >> 4) & 15); };
        auto stage_row = [&](int ii) {
            for (int xx = l; xx < B; xx += 32) {
                cp_async8(RB + rb_slot(xx), cv + size_t(ii) * NC + b0 + xx);
                cp_async8(RB + RBW + rb_slot(xx), pupil + ii * NLR + b0 + xx);
            }
            cp_async_commit();
        };
        const int i0 = rfirst + CL * w;
        if (PF && i0 < b0 + B && !a_loaded) load_row(i0);
        a_loaded = false;
        if (STG && i0 < b0 + B) stage_row(i0);
        for (int i = i0; i < b0 + B; i += CL * NW) {
            float2 x[M];
            if constexpr (PF) {
#pragma unroll
                for (int k0 = 0; k0 < M; ++k0) {
                    const int c = F.a_in(k0);
                    const float2 g = cmul(Oa[k0], Pa[k0]);  // conj, signed: the row IFFT runs as conj(FFT(conj g))
                    x[k0] = ((i + c) & 1) ? make_float2(-g.x, g.y) : make_float2(g.x, -g.y);
                    if (want_o) omax = fmaxf(omax, cabs2(Oa[k0]));
                    if (want_p) pmax = fmaxf(pmax, cabs2(Pa[k0]));
                }
                if (i + CL * NW < b0 + B) load_row(i + CL * NW);
            } else if constexpr (STG) {
                cp_async_wait_all();
                __syncwarp();
                const short2 run = SR[i];
#pragma unroll
                for (int k0 = 0; k0 < M; ++k0) {
                    const int c = F.a_in(k0);
                    float2 v = make_float2(0.f, 0.f);
                    if (FFT::live(k0) && c >= run.x && c < run.y) {
                        const float2 O = RB[rb_slot(c - b0)];
                        const float2 P = RB[RBW + rb_slot(c - b0)];
                        const float2 g = cmul(O, P);
                        v = ((i + c) & 1) ? make_float2(-g.x, g.y) : make_float2(g.x, -g.y);
                        if (want_o) omax = fmaxf(omax, cabs2(O));
                        if (want_p) pmax = fmaxf(pmax, cabs2(P));
                    }
                    x[k0] = v;
                }
                __syncwarp();  // every lane has read the buffer
                if (i + CL * NW < b0 + B) stage_row(i + CL * NW);
            } else {
                const short2 run = SR[i];
#pragma unroll
                for (int k0 = 0; k0 < M; ++k0) {
                    const int c = F.a_in(k0);
                    float2 v = make_float2(0.f, 0.f);
                    if (FFT::live(k0) && c >= run.x && c < run.y) {
                        const float2 O = cv[size_t(i) * NC + c];
                        const float2 P = pupil[i * NLR + c];
                        const float2 g = cmul(O, P);
                        v = ((i + c) & 1) ? make_float2(-g.x, g.y) : make_float2(g.x, -g.y);
                        if (want_o) omax = fmaxf(omax, cabs2(O));
                        if (want_p) pmax = fmaxf(pmax, cabs2(P));
                    }
                    x[k0] = v;
                }
            }
            F.fA(x);  // S keeps conj(IFFT_rows(g)): phase B's forward column FFT undoes it
            FPM_ASSERT(i >= b0 && i < b0 + B);
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const int col = F.a_out(r), owner = col / SW;
                FPM_ASSERT(col >= 0 && col < NLR && owner >= 0 && owner < CL);
                if constexpr (ASY) {
                    const uint32_t off = uint32_t((size_t(i - b0) * RS + (col - owner * SW)) * sizeof(float2));
                    st_async_f2(map_rank(smem_addr(S) + off, owner), x[r], map_rank(smem_addr(mbA + par), owner));
                } else {
                    cluster.map_shared_rank(S, owner)[size_t(i - b0) * RS + (col - owner * SW)] = x[r];
                }
            }
        }
        if (MODE == kModeEPRY) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                omax = fmaxf(omax, __shfl_xor_sync(kFull, omax, sh));
                pmax = fmaxf(pmax, __shfl_xor_sync(kFull, pmax, sh));
            }
            if (l == 0) {
                wred[w * 4 + 2] = omax;
                wred[w * 4 + 3] = pmax;
            }
        }
        cp_async_wait_all();  // this thread's part of the measurement slab has landed
        if constexpr (ASY) {
            __syncthreads();  // measurement slab and the EPRY partials visible CTA-wide
            // every column of every box row landed (mbA[par]'s phase; DB alternates two barriers)
            mbar_wait_parity(mbA + par, DB ? (nupd >> 1) & 1u : nupd & 1u);
        } else {
            cluster.sync();
        }

        // ---- B: this CTA's columns: IFFT over the box rows -> modulus -> FFT -> box rows
        // (sum(I): on pass 0 of a whole run, or every update without the per-(tile, LED) cache)
        const bool den_now = !FPM_CL_DENSEP || args.isum == nullptr || it == 0;
        float num = 0.f, den = 0.f;
        for (int jj = w; jj < SW; jj += NW) {
            const int j = rank * SW + jj;
            float2 x[M];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const int r = F.nat(m);
                x[m] = (FFT::live(m) && r >= b0 && r < b0 + B) ? S[size_t(r - b0) * RS + jj] : make_float2(0.f, 0.f);
            }
            F.f1(x);  // = conj(e), e the unscaled 2-D IFFT
            // every row this lane holds shares one column swizzle (FFT::isw_lane)
            const uint16_t* Ic = I_s + (jj ^ ((ST8 ? 4 * (l & 15) : F.isw_lane()) & (SW - 1)));
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int row = F.scr(k0);
                FPM_ASSERT(row >= 0 && row < NLR && (Ic - I_s) + row * SW < SW * NLR);
                const float Iv = float(Ic[row * SW]);
                if (!FPM_CL_DENSEP) den += Iv;
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
            if (FPM_CL_DENSEP && den_now) {  // the same additions in the same order, pass 0 only
#pragma unroll
                for (int k0 = 0; k0 < M; ++k0) den += float(Ic[F.scr(k0) * SW]);
            }
            F.f2(x);
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const int row = F.nat(r);
                if (FFT::live(r) && row >= b0 && row < b0 + B) S[size_t(row - b0) * RS + jj] = x[r];
            }
        }
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) num += __shfl_xor_sync(kFull, num, sh);
        if (den_now) {
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) den += __shfl_xor_sync(kFull, den, sh);
        }
        if (l == 0) {
            wred[w * 4] = num;
            wred[w * 4 + 1] = den;
        }
        float2 Pc[PFC ? M : 1], Oc[PFC ? M : 1];
        auto load_c = [&](int ii) {
            const short2 run = SR[ii];
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int c = F.c_out(k0);
                const bool on = FFT::live(k0) && c >= run.x && c < run.y;
                Pc[k0] = on ? pupil[ii * NLR + c] : make_float2(0.f, 0.f);
                Oc[k0] = (MODE == kModeEPRY && on) ? cv[size_t(ii) * NC + c] : make_float2(0.f, 0.f);
            }
        };
        const int ic0 = rfirst + CL * w;
        if constexpr (SPLIT) {  // the first phase-C row's operands load while other CTAs finish B
            cluster_arrive_release();
            if (PFC && ic0 < b0 + B) load_c(ic0);
            cluster_wait();
        } else {
            cluster.sync();
        }
        if (e_next >= 0) {  // the slab is free: stage the next update's measurement under phase C
            int itn, posn;
            entry_at(e_next, itn, posn);
            stage(posn);
        }

        // ---- cluster-wide residual terms and EPRY maxima (fixed order: deterministic)
        if (w == 0) {
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            for (int k = l; k < CL * NW; k += 32) {
                const float* src = cluster.map_shared_rank(wred, k / NW) + (k % NW) * 4;
                a0 += src[0];
                a1 += src[1];
                if (MODE == kModeEPRY) {
                    a2 = fmaxf(a2, src[2]);
                    a3 = fmaxf(a3, src[3]);
                }
            }
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) {
                a0 += __shfl_xor_sync(kFull, a0, sh);
                a1 += __shfl_xor_sync(kFull, a1, sh);
                a2 = fmaxf(a2, __shfl_xor_sync(kFull, a2, sh));
                a3 = fmaxf(a3, __shfl_xor_sync(kFull, a3, sh));
            }
            if (l == 0) {
                if (rank == 0) {
                    if (FPM_CL_DENSEP && args.isum) {  // pass 0 stores the crop's sum(I), later passes read it
                        float* is = args.isum + size_t(tile) * L + pos;
                        if (den_now)
                            *is = a1;
                        else
                            a1 = *is;
                    }
                    stage_sum[it] += a1 > 0.f ? double(__fdividef(a0, a1)) : 0.0;  // as fpm_loop64
                }
                upd[0] = (a2 > 0.f && bright) ? args.beta / a2 : 0.f;  // bright-field pupil steps only
                if (want_p) upd[1] = a3 > 0.f ? args.alpha / a3 : 0.f;  // else the pupil's value stands
            }
        }
        __syncthreads();
        const float inv_omax = upd[0], inv_pmax = upd[1];

        // ---- C: FFT of this CTA's box rows (fetched from the column slabs), scatter
        for (int i = ic0; i < b0 + B; i += CL * NW) {
            // the scatter's disk operands are loaded first, their latency under the FFT
            const short2 run = SR[i];
            if (PFC && !(SPLIT && i == ic0)) load_c(i);
            if constexpr (STG && FPM_CL_STAGE_C) stage_row(i);  // the row's canvas and pupil, under its FFT
            float2 x[M];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const int col = F.c_in(m), owner = col / SW;
                FPM_ASSERT(col >= 0 && col < NLR && owner >= 0 && owner < CL && i >= b0 && i < b0 + B);
                x[m] = cluster.map_shared_rank(S, owner)[size_t(i - b0) * RS + (col - owner * SW)];
            }
            F.fC(x);
            if constexpr (STG && FPM_CL_STAGE_C) {
                cp_async_wait_all();
                __syncwarp();
            }
#pragma unroll
            for (int k0 = 0; k0 < M; ++k0) {
                const int c = F.c_out(k0);
                if (!FFT::live(k0) || c < run.x || c >= run.y) continue;
                const float2 psi2 = cscale(x[k0], ((i + c) & 1) ? -1.f : 1.f);
                float2* dst = cv + size_t(i) * NC + c;
                float2* pp = pupil + i * NLR + c;
                float2 P;
                if constexpr (PFC) P = Pc[k0];
                else if constexpr (STG && FPM_CL_STAGE_C) P = RB[RBW + rb_slot(c - b0)];
                else P = *pp;
                if (MODE == kModeGS) {
                    *dst = cmulc(psi2, P);
                } else {
                    float2 O;
                    if constexpr (PFC) O = Oc[k0];
                    else if constexpr (STG && FPM_CL_STAGE_C) O = RB[rb_slot(c - b0)];
                    else O = *dst;
                    const float2 d = csub(psi2, cmul(O, P));
                    if (inv_pmax > 0.f) *dst = cadd(O, cscale(cmulc(d, P), inv_pmax));
                    if (inv_omax > 0.f) *pp = cadd(P, cscale(cmulc(d, O), inv_omax));
                }
            }
            if constexpr (STG && FPM_CL_STAGE_C) __syncwarp();  // the buffer is read before the next row's staging
        }
        // slabs reusable. Only a pupil step (bright-field EPRY) leaves writes another CTA
        // reads next (pupil rows follow the moving box rows): then release; else a relaxed
        // arrive skips the fence that would wait for this phase's canvas stores
        if (MODE == kModeEPRY && inv_omax > 0.f) {
            cluster.sync();
        } else {
            __syncthreads();  // a canvas row's next reader may be another warp of this CTA
            if constexpr (SPLIT) {  // the next update's first phase-A row loads under the barrier
                cluster_arrive_relaxed();
                if (PF && e_next >= 0) {
                    int itn, posn;
                    entry_at(e_next, itn, posn);
                    const short2 on_ = O_s[posn];
                    const int rf = b0 + ((rank - (int(on_.x) + b0) % CL) % CL + CL) % CL;
                    if (rf + CL * w < b0 + B) {
                        load_row_at(canvas + size_t(on_.x) * NC + on_.y, rf + CL * w);
                        a_loaded = true;
                    }
                }
                cluster_wait();
            } else if (!DB) {
                cluster_sync_relaxed();  // single slab buffer: phase C reads done
            }
        }
        pdirty = MODE == kModeEPRY && inv_omax > 0.f;
        par ^= DB ? 1 : 0;
        ++nupd;
        e = e_next;
    }
    if (DB) cluster.sync();  // no CTA leaves (or moves to the next item) while another still reads its slab
    if (rank == 0) {
        if (queue) {
            if (threadIdx.x == 0) args.residuals[size_t(tile) * args.iters + it_q] = stage_sum[it_q] / double(L);
        } else {
            store_residuals(args, tile, stage_sum, G == 1);
        }
    }
    if (queue) cluster.sync();  // the item's canvas and pupil writes precede rank 0's release
    }  // items
}

template <int NLR, int MODE, int NC, int CL, int NW>
cudaError_t launch_cluster_t(const LoopArgs& a, const BoxArgs& b, int T, cudaStream_t s) {
    const size_t smem = cluster_smem_bytes(NLR, b.box, CL, NW, a.L, a.iters);
    // MID (n = 256): the support box inside [64, 192) lets WarpFFT256 prune to registers 2..5
    auto k = a.jitter > 0 ? fpm_loop_cluster<NLR, MODE, NC, CL, NW, true, false>
                          : fpm_loop_cluster<NLR, MODE, NC, CL, NW, false, false>;
    if constexpr (NLR == 256 && !FPM_CL_STAGE) {
        if (b.b0 >= 64 && b.b0 + b.box <= 192 && !mid_disabled())
            k = a.jitter > 0 ? fpm_loop_cluster<NLR, MODE, NC, CL, NW, true, true>
                             : fpm_loop_cluster<NLR, MODE, NC, CL, NW, false, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    if (CL > 8) {  // 16-CTA clusters are a non-portable size on sm_100
        e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    LoopArgs a2 = a;
    int clusters = T;
    {
        const char* qe = std::getenv("FPM_B200_QUEUE");
        const int q = qe && qe[0] ? (qe[0] == '1' ? 1 : 0) : -1;
        a2.work = nullptr;
        if (a.work && !a.slots && a.slot_begin == 0 && a.num_slots == a.iters * a.L && q != 0) {
            // resident clusters: the occupancy calculator for this cluster shape
            cudaLaunchConfig_t oc{};
            oc.gridDim = dim3(unsigned(T * CL));
            oc.blockDim = dim3(NW * 32);
            oc.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CL;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            oc.attrs = at;
            oc.numAttrs = 1;
            int resident = 0;
            if ((e = cudaOccupancyMaxActiveClusters(&resident, k, &oc)) != cudaSuccess) return e;
            resident = std::max(resident, 1);
            if (T > resident || q == 1) {
                a2.work = a.work;
                clusters = q == 1 ? std::min(resident, T * a.iters) : resident;
                if ((e = cudaMemsetAsync(a.work, 0, sizeof(int) * size_t(T + 1), s)) != cudaSuccess) return e;
            }
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(clusters * CL));
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a2, b);
}

}  // namespace

int cluster_warps(int n, int cl) { return (n == 64 || cl == 16) ? 4 : (n == 256 && cl == 2) ? 16 : 8; }

bool cluster_supported(int n, int N, int cl) {
    if (n == 64) return N == 256 && (cl == 4 || cl == 8 || cl == 16);
    if (n == 128) return N == 512 && (cl == 2 || cl == 4 || cl == 8 || cl == 16);
    if (n == 256) return N == 1024 && (cl == 2 || cl == 4 || cl == 8);
    return false;
}

cudaError_t launch_loop_cluster(int n, int mode, int cl, const LoopArgs& a, const BoxArgs& b, int T,
                                cudaStream_t s) {
#define FPM_CL_CASE(NN, NCC, CLL, NWW)                                                          \
    if (n == NN && a.N == NCC && cl == CLL)                                                     \
        return mode == kModeGS ? launch_cluster_t<NN, kModeGS, NCC, CLL, NWW>(a, b, T, s)       \
                               : launch_cluster_t<NN, kModeEPRY, NCC, CLL, NWW>(a, b, T, s);
    FPM_CL_CASE(64, 256, 4, 4)
    FPM_CL_CASE(64, 256, 8, 4)
    FPM_CL_CASE(64, 256, 16, 4)
    FPM_CL_CASE(128, 512, 2, 8)
    FPM_CL_CASE(128, 512, 4, 8)
    FPM_CL_CASE(128, 512, 8, 8)
    FPM_CL_CASE(128, 512, 16, 4)
    FPM_CL_CASE(256, 1024, 2, 16)
    FPM_CL_CASE(256, 1024, 4, 8)
    FPM_CL_CASE(256, 1024, 8, 8)
#undef FPM_CL_CASE
    return cudaErrorNotSupported;  // no instantiation for this geometry
}

}  // namespace fpmk
