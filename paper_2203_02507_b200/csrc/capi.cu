// C-ABI of the B200 FPM engine (include/fpm_b200.h): host geometry, plans,
// launches. No exception crosses the boundary; see guarded().
#include <cudaTypedefs.h>

#include <algorithm>
#include <complex>
#include <map>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fpm_b200.h"
#include "geometry.hpp"
#include "kernels.cuh"
#include "stitch.cuh"

using namespace fpmb;

namespace {

thread_local std::string g_err;
thread_local int g_min_lag = 0;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return FPMGPU_OK;
    } catch (const UnsafeLag& e) {
        g_err = e.what();
        g_min_lag = e.minimum;
        return FPMGPU_ERR_UNSAFE_LAG;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return FPMGPU_ERR_CONFIG;
    } catch (const DataError& e) {
        g_err = e.what();
        return FPMGPU_ERR_DATA;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return FPMGPU_ERR_DOMAIN;
    } catch (const Unsupported& e) {
        g_err = e.what();
        return FPMGPU_ERR_UNSUPPORTED;
    } catch (const CudaError& e) {
        g_err = e.what();
        return FPMGPU_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FPMGPU_ERR_INTERNAL;
    }
}

void ck(cudaError_t e, const char* what) {
    if (e == cudaErrorNotSupported)  // the launchers' "no kernel instantiated for this geometry"
        throw Unsupported(std::string(what) + ": no kernel for this tile / canvas geometry in this build");
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    T* ensure(size_t count) {
        if (count > n) {
            reset();
            ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
            n = count;
        }
        return p;
    }
    void upload(const T* h, size_t count, cudaStream_t s) {
        ensure(count);
        ck(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    }
};

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 3-D map over the LR stack [F][H][pitch] u16 with a 64x64x1 box (layout: FPM_MEAS_SWIZZLE).
CUtensorMap encode_frames_map(const uint16_t* frames, int F, int H, int W, int64_t pitch) {
    if ((pitch * 2) % 16 != 0) throw DataError("frame row pitch must be a multiple of 8 elements");
    if (reinterpret_cast<uintptr_t>(frames) % 16 != 0) throw DataError("frame base must be 16-byte aligned");
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(W), cuuint64_t(H), cuuint64_t(F)};
    cuuint64_t strides[2] = {cuuint64_t(pitch) * 2, cuuint64_t(pitch) * 2 * cuuint64_t(H)};
    cuuint32_t box[3] = {64, 64, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<uint16_t*>(frames), dims,
                                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      FPM_MEAS_SWIZZLE ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// Support-dependent kernel shape: compact pupil slots per thread and whether
// the disk lies inside the pruned lattice rows/cols [16, 48).
void lattice_shape(const std::vector<uint8_t>& support, int* nslots, bool* prune) {
    int mx = 0;
    bool inside = true;
    for (int t = 0; t < 64; ++t) {
        int c = 0;
        for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b) {
                const int i = (t >> 3) + 8 * a, j = (t & 7) + 8 * b;
                if (support[size_t(i) * 64 + j]) {
                    ++c;
                    if (a < 2 || a > 5 || b < 2 || b > 5) inside = false;
                }
            }
        mx = std::max(mx, c);
    }
    (void)mx;
    *prune = inside;
    *nslots = inside ? 8 : 32;  // pair-lattice positions per thread held in the shared pupil
}

// Bounding box [b0, b0 + box) of the support disk (same for rows and columns).
void box_of(const std::vector<uint8_t>& support, int n, int* b0, int* box) {
    int lo = n, hi = -1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (support[size_t(i) * n + j]) {
                lo = std::min(lo, std::min(i, j));
                hi = std::max(hi, std::max(i, j));
            }
    if (hi < 0) throw ConfigError("empty pupil support");
    *b0 = lo;
    *box = hi - lo + 1;
}

// FPM_B200_FORCE_BOX=1 runs n = 64 on the general warp-FFT kernel (cross-checks).
bool box_forced() {
    const char* e = std::getenv("FPM_B200_FORCE_BOX");
    return e && e[0] == '1';
}

// Cluster split of a tile (kernels_cluster.cu): n = 256, whose box-row
// intermediate (240 KB) needs two SMs' shared memory, and n = 128 batches too
// small to occupy the GPU with one CTA per tile. FPM_B200_CLUSTER=<cl> forces a
// size (1 = off).
int cluster_choice(int n, int N, int T) {
    if (const char* e = std::getenv("FPM_B200_CLUSTER")) {
        const int c = std::atoi(e);
        if (c <= 1) return 0;
        if (!fpmk::cluster_supported(n, N, c))
            throw Unsupported("no cluster kernel for n = " + std::to_string(n) + ", N = " + std::to_string(N) +
                              ", cluster " + std::to_string(c));
        return c;
    }
    // n = 256: 4-CTA clusters (2 per SM); batches small enough for 8-CTA clusters
    // to be resident at once (a strong-scaled rank of config 5: 32 tiles) take 8
    // (tools/strong_probe.py: 106 vs 131 ms for 32 tiles)
    if (n == 256 && N == 1024) return T <= 48 ? 8 : 4;
    if (n == 128 && N == 512 && T * 16 <= 148) return 16;  // single-tile latency (config 2)
    if (n == 128 && N == 512 && T * 8 <= 148) return 8;
    return 0;
}

// n = 64 on 256 threads per tile (kernels_quad.cu) for strong-scaled batches of at
// most one tile per SM: a lone tile's update is latency-bound and twice the warps
// shorten it (config 3 over 8 GPUs, 128 tiles per rank: 9.00 -> 7.93 ms); with more
// tiles per SM the 128-thread pair lattice wins (fewer shuffles: 1,024 tiles 33.2 vs
// 44.2 ms, tools/quad_probe.sh). Batches below 64 tiles (single tiles, small FOVs) stay
// on the pair lattice, whose sequential runs are bit-identical to the pipelined
// schedule (test_parallel.cpp:97-108). FPM_B200_QUAD=1|0 forces.
// The quad-lattice kernel is opt-in (FPM_B200_QUAD=1): since the packed-operand
// rewrites, the 255-register pair build is faster at one tile per SM too
// (profiles/r2/strong_probe.txt: 128 tiles 6.97 vs 7.55 ms, 64 tiles 6.84 vs 7.45 ms).
bool quad_choice(int T) {
    (void)T;
    if (const char* e = std::getenv("FPM_B200_QUAD"); e && e[0]) return e[0] == '1';
    return false;
}

std::vector<float2> twiddles(int N) {
    std::vector<float2> w(static_cast<size_t>(N));
    for (int m = 0; m < N; ++m) {
        const double a = -2.0 * 3.14159265358979323846 * double(m) / double(N);
        w[size_t(m)] = make_float2(float(std::cos(a)), float(std::sin(a)));
    }
    return w;
}

}  // namespace

// One in-flight host-buffer request: device staging, one cached plan per tile
// band (band b = tiles [band_t0[b], band_t0[b+1])), a stream per band.
struct HostSlot {
    DevBuf<uint16_t> frames;
    DevBuf<float2> hr;
    DevBuf<double> resid;
    DevBuf<float2> pup;
    std::vector<fpmgpu_plan*> plans;
    std::vector<int> band_t0;
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> arrived;  // band's LR rows on the device (recorded on the copy stream)
    std::vector<cudaEvent_t> done;     // band's outputs back on the host
    std::vector<int> key_i;
    std::vector<double> key_d;
    std::vector<float> key_f;
    long long ticket = -1;  // request in flight, -1 = idle
    int lag = 0;
};

struct fpmgpu_context {
    int device = 0;
    cudaStream_t stream = nullptr;  // copy stream of the host path; plan uploads
    DevBuf<float2> tw256, tw512, tw1024;
    // host path: two slots, so request k + 1's upload overlaps request k's reconstruction
    HostSlot slots[2];
    long long next_ticket = 0;
    int lag_of[2] = {0, 0};  // lag of the request last submitted on each slot

    const float2* twiddle_table(int N) {
        DevBuf<float2>* b = N == 256 ? &tw256 : N == 512 ? &tw512 : N == 1024 ? &tw1024 : nullptr;
        if (!b) throw Unsupported("canvas side " + std::to_string(N) + " has no line-FFT kernel (256/512/1024)");
        if (!b->p) {
            auto w = twiddles(N);
            b->upload(w.data(), w.size(), stream);
        }
        return b->p;
    }
};

struct fpmgpu_plan {
    fpmgpu_context* ctx = nullptr;
    fpmgpu_recon_request req{};
    int n = 0, N = 0, T = 0, L = 0, F = 0, G = 1, lag = 0, nslots = 1, num_slots = 0;
    bool prune = false;
    bool use_box = false;  // n != 64: warp-FFT box kernel (kernels_box.cu)
    bool quad = false;     // n = 64, sequential, disk inside [16, 48): 256 threads per tile (kernels_quad.cu)
    int cl = 0;            // > 0: each tile split over a cluster of cl CTAs (kernels_cluster.cu)
    int box = 0, b0 = 0;
    int support_px = 0;
    int batch_tiles = 0;  // tiles sharing the GPU with this plan's launch (banded host path); 0 = T
    double radius = 0.0;
    DevBuf<float2> canvas, pupils, pupils_init, scratch;
    DevBuf<uint8_t> support;
    DevBuf<short2> sup_rows;
    DevBuf<short2> origins;
    DevBuf<uint8_t> bright;
    DevBuf<int> seq_frame;
    DevBuf<int2> tile_xy, slots;
    DevBuf<double> defocus, resid;
    DevBuf<int> work;     // LED-loop work queue: item counter + per-tile passes done
    DevBuf<float> isum;   // [T][L] sum(I) per crop (work-queue items of later passes)
    bool has_defocus = false, has_pupils = false;
    // tiles abut without overlap on a full regular grid (stride n): the mosaic is a
    // plain placement of the HR tiles, so canvas_to_field can write it directly
    bool abut = false;
    std::vector<int2> xy_host;
    int x_min = 0, y_min = 0;
    DevBuf<long long> out_off;
    long long out_off_pitch = -1;
    // N = 256 canvas box: every update touches only rows / columns [cbox0, cbox0 + cboxn)
    // (origins + support box), so init_canvas and canvas_to_field prune to it
    int cbox0 = 0, cboxn = 0;
    DevBuf<float2> canvas0;          // [T][cboxn][cboxn] init spectrum over the box
    const uint16_t* seed_frame = nullptr;  // the last prologue's seed frame (the epilogue re-reads it)
    int64_t seed_pitch = 0;
    // phase events of recent executes: [slot][4] = start, after init, after loop, after finalize
    static constexpr int kEventSlots = 256;
    std::vector<cudaEvent_t> events;
    int recorded = 0;
    ~fpmgpu_plan() {
        for (auto e : events) cudaEventDestroy(e);
    }
    cudaEvent_t* slot_events() {
        if (events.empty()) {
            events.resize(size_t(kEventSlots) * 4);
            for (auto& e : events) ck(cudaEventCreate(&e), "cudaEventCreate");
        }
        if (recorded >= kEventSlots) return nullptr;
        return events.data() + size_t(recorded++) * 4;
    }
};

namespace {

void build_plan(fpmgpu_plan& p, const fpmgpu_recon_request& r) {
    const Cfg& c = r.cfg;
    validate(c);
    if (r.iters < 1) throw ConfigError("iters must be >= 1");
    if (r.mode != FPMGPU_MODE_GS && r.mode != FPMGPU_MODE_EPRY) throw ConfigError("unknown reconstruction mode");
    p.req = r;
    p.n = c.tile_size;
    p.N = c.tile_size * c.upsample;
    p.T = r.num_tiles;
    p.L = r.num_leds;
    p.F = r.num_frames;
    if (p.T < 1) throw ConfigError("no tiles to reconstruct");
    if (p.L < 1) throw DataError("min_safe_lag: empty sequence");
    p.radius = pupil_radius_px(c, p.n);  // ConfigError on Nyquist / grid checks
    if (p.n != 64 && p.n != 128 && p.n != 256)
        throw Unsupported("tile side " + std::to_string(p.n) + " has no device kernel in this build (64/128/256)");
    p.use_box = p.n != 64 || box_forced();
    if (p.N != 256 && p.N != 512 && p.N != 1024)
        throw Unsupported("canvas side " + std::to_string(p.N) + " has no line-FFT kernel (256/512/1024)");
    for (int t = 0; t < p.T; ++t) {
        const int x0 = r.tile_xy[2 * t], y0 = r.tile_xy[2 * t + 1];
        if (x0 < 0 || y0 < 0 || y0 + p.n > r.height || x0 + p.n > r.width)
            throw DataError("tile extends past frame bounds");
    }
    if (r.init_frame < 0 || r.init_frame >= p.F) throw DataError("empty frame set");
    for (int k = 0; k < p.L; ++k)
        if (r.seq_frame[k] < 0 || r.seq_frame[k] >= p.F)
            throw DataError("missing frame for sequence position " + std::to_string(k));

    std::vector<short2> org(size_t(p.T) * p.L);
    std::vector<uint8_t> bright(size_t(p.T) * p.L);
    for (int t = 0; t < p.T; ++t)
        for (int k = 0; k < p.L; ++k) {
            const int oy = r.offsets[(size_t(t) * p.L + k) * 2], ox = r.offsets[(size_t(t) * p.L + k) * 2 + 1];
            const int r0 = p.N / 2 + oy - p.n / 2, c0 = p.N / 2 + ox - p.n / 2;
            if (r0 < 0 || c0 < 0 || r0 + p.n > p.N || c0 + p.n > p.N)
                throw DataError("spectrum offset out of canvas bounds");
            org[size_t(t) * p.L + k] = make_short2(short(r0), short(c0));
            bright[size_t(t) * p.L + k] = bright_field(oy, ox, p.radius);
        }

    std::vector<uint8_t> sup = support_disk(p.n, p.radius);
    p.bright.upload(bright.data(), bright.size(), p.ctx->stream);
    p.support_px = 0;
    for (auto s : sup) p.support_px += s;
    p.cl = box_forced() ? 0 : cluster_choice(p.n, p.N, std::max(p.T, p.batch_tiles));
    if (p.cl) {
        box_of(sup, p.n, &p.b0, &p.box);
        std::vector<short2> runs(size_t(p.n), make_short2(0, 0));
        for (int i = 0; i < p.n; ++i) {
            int lo = p.n, hi = 0;
            for (int j = 0; j < p.n; ++j)
                if (sup[size_t(i) * p.n + j]) {
                    lo = std::min(lo, j);
                    hi = j + 1;
                }
            for (int j = lo; j < hi; ++j)
                if (!sup[size_t(i) * p.n + j]) throw ConfigError("pupil support row is not one run");
            if (hi > lo) runs[size_t(i)] = make_short2(short(lo), short(hi));
        }
        p.sup_rows.upload(runs.data(), runs.size(), p.ctx->stream);
        if (fpmk::cluster_smem_bytes(p.n, p.box, p.cl, fpmk::cluster_warps(p.n, p.cl), p.L, r.iters) > 232448)
            throw Unsupported("cluster slab exceeds shared memory");
        if (p.F > 65536) throw Unsupported("the cluster kernel indexes at most 65,536 frames");
    } else if (p.use_box) {
        box_of(sup, p.n, &p.b0, &p.box);
        const bool smem_s = p.n != 256;
        if (p.n == 256 && p.N != 1024) throw Unsupported("n = 256 runs with canvas side 1024 (upsample 4) in this build");
        if (p.n == 128 && p.N != 512 && p.N != 1024) throw Unsupported("n = 128 needs canvas side 512 or 1024");
        if (p.n == 64 && p.N != 256) throw Unsupported("the box kernel runs n = 64 with canvas side 256 only");
        if (!smem_s) p.scratch.ensure(size_t(p.T) * p.box * (p.n + 1));
    } else {
        lattice_shape(sup, &p.nslots, &p.prune);
        if (!p.prune && p.N != 256)
            throw Unsupported("pupil disk wider than the pruned lattice needs canvas side 256 in this build");
    }

    {
        // canvas rows / columns any update reads or writes: origin + the block rows / columns
        // the loop kernel touches — the support's range for the box and cluster kernels (they
        // mask by support run), the lattice's [16, 48) or [0, 64) for the n = 64 lattice kernels
        // (their gathers read every lattice position of the pruned block)
        int s0 = p.n, s1 = 0;
        if (!p.use_box && !p.cl) {
            s0 = p.prune ? 16 : 0;
            s1 = p.prune ? 48 : 64;
        } else {
            for (int i = 0; i < p.n; ++i)
                for (int j = 0; j < p.n; ++j)
                    if (sup[size_t(i) * p.n + j]) {
                        s0 = std::min(s0, std::min(i, j));
                        s1 = std::max(s1, std::max(i, j) + 1);
                    }
        }
        int lo = p.N, hi = 0;
        for (const short2& o : org) {
            lo = std::min(lo, std::min(int(o.x), int(o.y)) + s0);
            hi = std::max(hi, std::max(int(o.x), int(o.y)) + s1);
        }
        lo = lo / 16 * 16;
        hi = std::min(p.N, (hi + 15) / 16 * 16);
        const char* e = std::getenv("FPM_B200_CANVAS_BOX");
        const bool on = !(e && e[0] == '0');
        p.cbox0 = 0;
        p.cboxn = 0;
        if (on && p.N == 256 && hi > lo && (hi - lo) * 4 <= p.N * 3) {  // worth it below 3/4 of the side
            p.cbox0 = lo;
            p.cboxn = hi - lo;
        }
    }

    // pipelined schedule (parallel.cpp:52-111): one lag for the whole batch,
    // the largest per-tile minimum, so every tile stays sequential-equivalent
    std::vector<int2> slots;
    p.G = 1;
    p.lag = 0;
    if (r.lag != 0) {
        if (r.mode != FPMGPU_MODE_GS) throw ConfigError("pipelined schedule requires Gerchberg-Saxton mode");
        int min_lag = 1;
        for (int t = 0; t < p.T; ++t) {
            std::vector<std::pair<int, int>> offs;
            for (int k = 0; k < p.L; ++k)
                offs.emplace_back(r.offsets[(size_t(t) * p.L + k) * 2], r.offsets[(size_t(t) * p.L + k) * 2 + 1]);
            min_lag = std::max(min_lag, min_safe_lag(offs, p.radius));
        }
        const int use = r.lag < 0 ? min_lag : r.lag;
        if (use < min_lag && !r.force_unsafe_lag) throw UnsafeLag(min_lag);
        p.lag = use;
        const int R = (p.L - 1) + (r.iters - 1) * use + 1;
        std::vector<std::vector<int2>> rounds(static_cast<size_t>(R));
        for (int s = 0; s < r.iters; ++s)
            for (int q = 0; q < p.L; ++q) rounds[size_t(q + s * use)].push_back(make_int2(s, q));
        size_t widest = 1;
        for (auto& rd : rounds) widest = std::max(widest, rd.size());
        p.G = widest > 1 ? 2 : 1;
        if (p.G > 1) {
            for (auto& rd : rounds)
                for (size_t c0 = 0; c0 < rd.size(); c0 += 2)
                    for (int g = 0; g < 2; ++g)
                        slots.push_back(c0 + g < rd.size() ? rd[c0 + g] : make_int2(-1, -1));
        }
    }
    p.num_slots = p.G == 1 ? r.iters * p.L : int(slots.size() / 2);
    p.quad = !p.use_box && !p.cl && p.prune && p.G == 1 &&
             quad_choice(std::max(p.T, p.batch_tiles)) && fpmk::loop64q_smem_bytes(p.L, r.iters, true) <= 227 * 1024;

    cudaStream_t s = p.ctx->stream;
    p.support.upload(sup.data(), sup.size(), s);
    p.origins.upload(org.data(), org.size(), s);
    p.seq_frame.upload(r.seq_frame, size_t(p.L), s);
    std::vector<int2> xy(static_cast<size_t>(p.T));
    for (int t = 0; t < p.T; ++t) xy[size_t(t)] = make_int2(r.tile_xy[2 * t], r.tile_xy[2 * t + 1]);
    p.tile_xy.upload(xy.data(), xy.size(), s);
    {
        std::vector<int> xs, ys;
        for (auto& v : xy) {
            xs.push_back(v.x);
            ys.push_back(v.y);
        }
        std::sort(xs.begin(), xs.end());
        xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
        std::sort(ys.begin(), ys.end());
        ys.erase(std::unique(ys.begin(), ys.end()), ys.end());
        bool ok = size_t(p.T) == xs.size() * ys.size();
        for (size_t k = 1; k < xs.size(); ++k) ok &= xs[k] - xs[k - 1] == p.n;
        for (size_t k = 1; k < ys.size(); ++k) ok &= ys[k] - ys[k - 1] == p.n;
        std::vector<std::pair<int, int>> cells;
        for (auto& v : xy) cells.emplace_back(v.y, v.x);
        std::sort(cells.begin(), cells.end());
        ok &= std::adjacent_find(cells.begin(), cells.end()) == cells.end();
        p.abut = ok;
        p.x_min = xs.front();
        p.y_min = ys.front();
        p.xy_host = xy;
    }
    if (p.G > 1) p.slots.upload(slots.data(), slots.size(), s);
    p.has_defocus = r.tile_defocus_um != nullptr;
    if (p.has_defocus) p.defocus.upload(r.tile_defocus_um, size_t(p.T), s);
    p.has_pupils = r.pupils != nullptr;
    if (p.has_pupils)
        p.pupils_init.upload(reinterpret_cast<const float2*>(r.pupils), size_t(p.T) * p.n * p.n, s);
    p.canvas.ensure(size_t(p.T) * p.N * p.N);
    if (p.cboxn) p.canvas0.ensure(size_t(p.T) * p.cboxn * p.cboxn);
    p.pupils.ensure(size_t(p.T) * p.n * p.n);
    p.resid.ensure(size_t(p.T) * r.iters);
    p.ctx->twiddle_table(p.N);
    // the request's host arrays belong to the caller; keep only scalars
    p.req.tile_xy = nullptr;
    p.req.offsets = nullptr;
    p.req.seq_frame = nullptr;
    p.req.tile_defocus_um = nullptr;
    p.req.pupils = nullptr;
}

// pupils (build_pupil per tile, or the caller's) + init_canvas: bilinear(sqrt(seed crop)) ->
// centered FFT N x N -> / up^2 (recon.cpp:61-86)
void plan_prologue(fpmgpu_plan& p, const uint16_t* frames, int64_t pitch, cudaStream_t s) {
    const fpmgpu_recon_request& r = p.req;
    const double dk = 1.0 / (p.n * dx_obj(r.cfg));
    const double inv_l2 = 1.0 / (r.cfg.wavelength * r.cfg.wavelength);
    if (p.has_pupils)
        ck(cudaMemcpyAsync(p.pupils.p, p.pupils_init.p, sizeof(float2) * size_t(p.T) * p.n * p.n,
                           cudaMemcpyDeviceToDevice, s), "pupil copy");
    else
        ck(fpmk::launch_build_pupils(p.pupils.p, p.support.p, p.has_defocus ? p.defocus.p : nullptr, p.n, p.T, dk,
                                     inv_l2, s), "build_pupils");
    fpmk::LinesArgs la{};
    la.tw = p.ctx->twiddle_table(p.N);
    la.frame = frames + size_t(r.init_frame) * size_t(r.height) * size_t(pitch);
    la.pitch = pitch;
    la.tile_xy = p.tile_xy.p;
    la.n = p.n;
    la.up = r.cfg.upsample;
    la.src = p.canvas.p;
    la.dst = p.canvas.p;
    la.scale = 1.0f;
    p.seed_frame = la.frame;
    p.seed_pitch = pitch;
    if (p.cboxn) {  // the spectrum over the canvas box only (kernels.cuh, LinesArgs)
        la.box0 = p.cbox0;
        la.boxn = p.cboxn;
        la.canvas0 = p.canvas0.p;
        ck(fpmk::launch_lines_box(0, la, p.T, s), "init rows (box)");
        la.scale = float(1.0 / (double(r.cfg.upsample) * r.cfg.upsample));
        ck(fpmk::launch_lines_box(1, la, p.T, s), "init cols (box)");
        return;
    }
    ck(fpmk::launch_lines(0, p.N, la, p.T, s), "init rows");
    la.scale = float(1.0 / (double(r.cfg.upsample) * r.cfg.upsample));
    ck(fpmk::launch_lines(1, p.N, la, p.T, s), "init cols");
}

// the LED loop over schedule slots [s0, s1); residuals of the touched stages are
// stored (acc = false) or added (acc = true)
void plan_loop(fpmgpu_plan& p, const uint16_t* frames, int64_t pitch, double* resid, int s0, int s1, bool acc,
               cudaStream_t s) {
    const fpmgpu_recon_request& r = p.req;
    fpmk::LoopArgs a{};
    a.canvas = p.canvas.p;
    a.pupils = p.pupils.p;
    a.support = p.support.p;
    a.origins = p.origins.p;
    a.bright = p.bright.p;
    a.seq_frame = p.seq_frame.p;
    a.tile_xy = p.tile_xy.p;
    a.F = p.F;
    a.residuals = resid ? resid : p.resid.p;
    a.slots = p.G > 1 ? p.slots.p : nullptr;
    a.slot_begin = s0;
    a.num_slots = s1;
    a.resid_accumulate = acc ? 1 : 0;
    a.T = p.T;
    a.L = p.L;
    a.iters = r.iters;
    a.N = p.N;
    a.nslots = p.nslots;
#if FPM_CHECK
    // checked build self-test: a tile count of 0 makes every loop kernel's tile assert fire
    if (const char* st = std::getenv("FPM_B200_CHECK_SELFTEST"); st && st[0] == '1') a.T = 0;
#endif
    a.alpha = float(r.alpha);
    a.beta = float(r.beta);
    a.batch_T = p.batch_tiles > 0 ? p.batch_tiles : p.T;
    if (const char* j = std::getenv("FPM_B200_JITTER"); j && j[0]) {  // race hunting (kernels.cuh)
        a.jitter = std::max(0, std::atoi(j));
        const char* c = std::strchr(j, ':');
        a.jitter_seed = c ? unsigned(std::strtoul(c + 1, nullptr, 10)) : 1u;
    }
    if (p.use_box || p.cl) {
        fpmk::BoxArgs bx{};
        bx.scratch = p.scratch.p;
        bx.frames = frames;
        bx.pitch = pitch;
        bx.frame_stride = pitch * r.height;
        bx.box = p.box;
        bx.b0 = p.b0;
        bx.sup_rows = p.sup_rows.p;
        if (p.cl && p.G == 1 && s0 == 0 && s1 == p.num_slots && !acc) {  // whole run: the work queue may serve it
            a.work = p.work.ensure(size_t(p.T) + 1);
            a.isum = p.isum.ensure(size_t(p.T) * p.L);  // sum(I) per (tile, LED), formed on pass 0
        }
        if (p.cl)
            ck(fpmk::launch_loop_cluster(p.n, r.mode, p.cl, a, bx, p.T, s), "LED loop (cluster)");
        else
            ck(fpmk::launch_loop_box(p.n, r.mode, a, bx, p.T, s), "LED loop (box)");
    } else {
        const CUtensorMap map = encode_frames_map(frames, p.F, r.height, r.width, pitch);
        if (p.G == 1 && s0 == 0 && s1 == p.num_slots && !acc) {  // whole run: the work queue may serve it
            a.work = p.work.ensure(size_t(p.T) + 1);
            a.isum = p.isum.ensure(size_t(p.T) * p.L);
        }
        if (p.quad)
            ck(fpmk::launch_loop64q(r.mode, &map, a, p.T, s), "LED loop (quad)");
        else
            ck(fpmk::launch_loop64(r.mode, p.prune, fpmk::kMeasTMA, p.G, &map, a, p.T, s), "LED loop");
    }
}

// canvas_to_field: centered IFFT N x N * up^2 (the 1/N^2 of ifft2 folded in), recon.cpp:88-91
// mosaic_pitch > 0: hr is a mosaic (row 0 = the plan's top tile row, column 0 =
// its leftmost tile), tile t written at ((y0 - y_min) * up, (x0 - x_min) * up)
void plan_epilogue(fpmgpu_plan& p, float* hr, float* pupils_out, cudaStream_t s, long long mosaic_pitch = 0) {
    const fpmgpu_recon_request& r = p.req;
    fpmk::LinesArgs la{};
    if (mosaic_pitch > 0) {
        if (!p.abut) throw Unsupported("the tiles overlap or leave gaps: stitch the HR tiles instead");
        if (!hr) throw DataError("mosaic output missing");
        if (mosaic_pitch < (long long)(p.N) * (long long)(p.xy_host.size())) {
            long long w = 0;
            for (auto& v : p.xy_host) w = std::max<long long>(w, (long long)(v.x - p.x_min) * r.cfg.upsample + p.N);
            if (mosaic_pitch < w) throw DataError("mosaic pitch narrower than the band");
        }
        if (p.out_off_pitch != mosaic_pitch) {
            std::vector<long long> off(p.xy_host.size());
            for (size_t t = 0; t < off.size(); ++t)
                off[t] = (long long)(p.xy_host[t].y - p.y_min) * r.cfg.upsample * mosaic_pitch +
                         (long long)(p.xy_host[t].x - p.x_min) * r.cfg.upsample;
            p.out_off.upload(off.data(), off.size(), s);
            p.out_off_pitch = mosaic_pitch;
        }
        la.out_off = p.out_off.p;
        la.out_pitch = mosaic_pitch;
    }
    la.tw = p.ctx->twiddle_table(p.N);
    la.tile_xy = p.tile_xy.p;
    la.n = p.n;
    la.up = r.cfg.upsample;
    la.src = p.canvas.p;
    la.dst = p.canvas.p;
    la.scale = 1.0f;
    const long long* off = la.out_off;
    la.out_off = nullptr;
    if (p.cboxn) {  // field = U + up^2 ifft2(canvas - canvas0), the difference confined to the box
        la.box0 = p.cbox0;
        la.boxn = p.cboxn;
        la.canvas0 = p.canvas0.p;
        la.frame = p.seed_frame;
        la.pitch = p.seed_pitch;
        ck(fpmk::launch_lines_box(2, la, p.T, s), "final rows (box)");
    } else {
        ck(fpmk::launch_lines(2, p.N, la, p.T, s), "final rows");
    }
    la.out_off = off;
    la.dst = hr ? reinterpret_cast<float2*>(hr) : p.canvas.p;
    la.scale = float(double(r.cfg.upsample) * r.cfg.upsample / (double(p.N) * p.N));
    if (p.cboxn)
        ck(fpmk::launch_lines_box(3, la, p.T, s), "final cols (box)");
    else
        ck(fpmk::launch_lines(3, p.N, la, p.T, s), "final cols");
    if (pupils_out)
        ck(cudaMemcpyAsync(pupils_out, p.pupils.p, sizeof(float2) * size_t(p.T) * p.n * p.n,
                           cudaMemcpyDeviceToDevice, s), "pupil out");
}

void execute_plan(fpmgpu_plan& p, const uint16_t* frames, int64_t pitch, float* hr, double* resid,
                  float* pupils_out, cudaStream_t s, long long mosaic_pitch = 0) {
    cudaEvent_t* ev = p.slot_events();
    if (ev) ck(cudaEventRecord(ev[0], s), "event");
    plan_prologue(p, frames, pitch, s);
    if (ev) ck(cudaEventRecord(ev[1], s), "event");
    plan_loop(p, frames, pitch, resid, 0, p.num_slots, false, s);
    if (ev) ck(cudaEventRecord(ev[2], s), "event");
    // the pupil copy-out stays outside the finalize phase event
    plan_epilogue(p, hr, nullptr, s, mosaic_pitch);
    if (ev) ck(cudaEventRecord(ev[3], s), "event");
    if (pupils_out)
        ck(cudaMemcpyAsync(pupils_out, p.pupils.p, sizeof(float2) * size_t(p.T) * p.n * p.n,
                           cudaMemcpyDeviceToDevice, s), "pupil out");
}

bool same_request(const HostSlot& c, const fpmgpu_recon_request& r, std::vector<int>& ki,
                  std::vector<double>& kd, std::vector<float>& kf) {
    ki.clear();
    kd.clear();
    kf.clear();
    const int* cfg_i = reinterpret_cast<const int*>(&r.cfg);
    ki.insert(ki.end(), cfg_i, cfg_i + sizeof(r.cfg) / sizeof(int));
    ki.insert(ki.end(), {r.iters, r.mode, r.lag, r.force_unsafe_lag, r.num_tiles, r.num_leds, r.init_frame,
                         r.num_frames, r.height, r.width});
    ki.insert(ki.end(), r.tile_xy, r.tile_xy + 2 * size_t(r.num_tiles));
    ki.insert(ki.end(), r.offsets, r.offsets + 2 * size_t(r.num_tiles) * r.num_leds);
    ki.insert(ki.end(), r.seq_frame, r.seq_frame + r.num_leds);
    // kernel-selection overrides change the plans too
    const char* cl_env = std::getenv("FPM_B200_CLUSTER");
    const char* q_env = std::getenv("FPM_B200_QUAD");
    const char* b_env = std::getenv("FPM_B200_CANVAS_BOX");
    ki.insert(ki.end(), {box_forced() ? 1 : 0, cl_env ? std::atoi(cl_env) : -1, q_env && q_env[0] ? q_env[0] : -1,
                         b_env && b_env[0] ? b_env[0] : -1});
    kd.push_back(r.alpha);
    kd.push_back(r.beta);
    if (r.tile_defocus_um) kd.insert(kd.end(), r.tile_defocus_um, r.tile_defocus_um + r.num_tiles);
    if (r.pupils) kf.insert(kf.end(), r.pupils, r.pupils + 2 * size_t(r.num_tiles) * r.cfg.tile_size * r.cfg.tile_size);
    return !c.plans.empty() && ki == c.key_i && kd == c.key_d && kf == c.key_f;
}

}  // namespace

namespace {

// Geometry of stitch_mosaic (stitch.cpp:48-86) for a regular tile grid: tiles
// bucketed into rows by y0 (sorted by x0), cut at the overlap midlines.
struct StitchLayout {
    int rows = 0, cols = 0, n_cols = 0, n_strips = 0;
    std::vector<fpmk::StitchTile> st;
    std::vector<int> grid;            // [strip][slot] -> tile
    std::vector<int> X, Y;            // per slot / per strip HR origin
    std::vector<int> ovh, ovv;        // overlap (HR px) with the previous slot / strip
    std::vector<int> col_cut, row_cut;
    std::vector<int> row_of, col_of;  // mosaic row -> strip, column -> slot
};

StitchLayout stitch_layout(const Cfg& c, const int* xy, int T) {
    if (T < 1) throw DataError("stitch_mosaic: tile/spec count mismatch");
    const int up = c.upsample, n = c.tile_size, N = n * up;
    std::map<int, std::vector<int>> by_row;
    for (int t = 0; t < T; ++t) by_row[xy[2 * t + 1]].push_back(t);
    StitchLayout L;
    std::vector<int> xs;
    for (auto& kv : by_row) {
        std::sort(kv.second.begin(), kv.second.end(), [&](int a, int b) { return xy[2 * a] < xy[2 * b]; });
        std::vector<int> rx;
        for (int t : kv.second) rx.push_back(xy[2 * t]);
        if (xs.empty()) xs = rx;
        else if (rx != xs)
            throw Unsupported("stitch_mosaic on the device needs every tile row to share its x origins");
    }
    std::vector<int> ys;
    for (auto& kv : by_row) ys.push_back(kv.first);
    L.n_cols = int(xs.size());
    L.n_strips = int(ys.size());
    L.X.resize(size_t(L.n_cols));
    L.Y.resize(size_t(L.n_strips));
    L.ovh.assign(size_t(L.n_cols), 0);
    L.ovv.assign(size_t(L.n_strips), 0);
    L.col_cut.assign(size_t(L.n_cols) + 1, 0);
    L.row_cut.assign(size_t(L.n_strips) + 1, 0);
    for (int k = 0; k < L.n_cols; ++k) {
        L.X[size_t(k)] = (xs[size_t(k)] - xs[0]) * up;
        if (k == 0) continue;
        const int ov = xs[size_t(k) - 1] + n - xs[size_t(k)];
        if (ov < 0) throw DataError("stitch_mosaic: gap between adjacent tiles");
        const int width = L.X[size_t(k) - 1] + N;  // strip width before tile k
        const int o = ov * up;
        if (o >= width || o >= N) throw DataError("stitch_pair: overlap out of range");
        L.ovh[size_t(k)] = o;
        L.col_cut[size_t(k)] = width - o / 2;
    }
    L.cols = L.X.back() + N;
    L.col_cut[size_t(L.n_cols)] = L.cols;
    for (int k = 0; k < L.n_strips; ++k) {
        L.Y[size_t(k)] = (ys[size_t(k)] - ys[0]) * up;
        if (k == 0) continue;
        const int ov = ys[size_t(k) - 1] + n - ys[size_t(k)];
        if (ov < 0) throw DataError("stitch_mosaic: gap between tile rows");
        const int height = L.Y[size_t(k) - 1] + N;
        const int o = ov * up;
        if (o >= height || o >= N) throw DataError("stitch_pair: overlap out of range");
        L.ovv[size_t(k)] = o;
        L.row_cut[size_t(k)] = height - o / 2;
    }
    L.rows = L.Y.back() + N;
    L.row_cut[size_t(L.n_strips)] = L.rows;
    L.grid.resize(size_t(L.n_strips) * L.n_cols);
    L.st.resize(size_t(T));
    int sidx = 0;
    for (auto& kv : by_row) {
        for (int k = 0; k < L.n_cols; ++k) {
            const int t = kv.second[size_t(k)];
            L.grid[size_t(sidx) * L.n_cols + k] = t;
            fpmk::StitchTile& s = L.st[size_t(t)];
            s.X = L.X[size_t(k)];
            s.Y = L.Y[size_t(sidx)];
            s.own_c0 = L.col_cut[size_t(k)] - s.X;
            s.own_c1 = L.col_cut[size_t(k) + 1] - s.X;
            s.fre = 1.f;
            s.fim = 0.f;
        }
        ++sidx;
    }
    L.row_of.resize(size_t(L.rows));
    L.col_of.resize(size_t(L.cols));
    for (int k = 0; k < L.n_strips; ++k)
        for (int r = L.row_cut[size_t(k)]; r < L.row_cut[size_t(k) + 1]; ++r) L.row_of[size_t(r)] = k;
    for (int k = 0; k < L.n_cols; ++k)
        for (int q = L.col_cut[size_t(k)]; q < L.col_cut[size_t(k) + 1]; ++q) L.col_of[size_t(q)] = k;
    return L;
}

using C128 = std::complex<double>;

// A band of the mosaic: tiles [tile_lo, tile_hi) of the layout's tile list,
// which must be whole strips (tile rows) [strip_lo, strip_hi). The band owns
// mosaic rows [row_cut[strip_lo], row_cut[strip_hi]). The single-GPU stitch
// is the band over every tile; a multi-GPU run gives each rank its band.
struct MosaicBand {
    StitchLayout lay;
    int N = 0, tile_lo = 0, tile_hi = 0, strip_lo = 0, strip_hi = 0, row_lo = 0, row_hi = 0;
    bool exchange = false;  // some overlap > 0: the ratios need the tiles' sums
};

MosaicBand mosaic_band(const Cfg& c, const int* xy, int T, int tile_lo, int tile_hi) {
    MosaicBand b;
    b.lay = stitch_layout(c, xy, T);
    b.N = c.tile_size * c.upsample;
    if (tile_lo < 0 || tile_hi > T || tile_lo >= tile_hi) throw DataError("mosaic band: empty or out-of-range tiles");
    b.tile_lo = tile_lo;
    b.tile_hi = tile_hi;
    const StitchLayout& L = b.lay;
    b.strip_lo = L.n_strips;
    b.strip_hi = 0;
    for (int s = 0; s < L.n_strips; ++s)
        for (int k = 0; k < L.n_cols; ++k) {
            const int t = L.grid[size_t(s) * L.n_cols + k];
            if (t >= tile_lo && t < tile_hi) {
                b.strip_lo = std::min(b.strip_lo, s);
                b.strip_hi = std::max(b.strip_hi, s + 1);
            }
        }
    int cnt = 0;
    for (int s = b.strip_lo; s < b.strip_hi; ++s)
        for (int k = 0; k < L.n_cols; ++k) {
            const int t = L.grid[size_t(s) * L.n_cols + k];
            if (t < tile_lo || t >= tile_hi) throw DataError("mosaic band: the tiles must be whole tile rows");
            ++cnt;
        }
    if (cnt != tile_hi - tile_lo) throw DataError("mosaic band: the tiles must be whole tile rows");
    b.row_lo = L.row_cut[size_t(b.strip_lo)];
    b.row_hi = L.row_cut[size_t(b.strip_hi)];
    for (int o : L.ovh) b.exchange |= o > 0;
    for (int o : L.ovv) b.exchange |= o > 0;
    return b;
}

// The band's tile table: the layout's entries of tiles [tile_lo, tile_hi), band-local.
std::vector<fpmk::StitchTile> band_tiles(const MosaicBand& b) {
    return std::vector<fpmk::StitchTile>(b.lay.st.begin() + b.tile_lo, b.lay.st.begin() + b.tile_hi);
}

// Phase 1 (per band): the horizontal mean_ratio chain of each of the band's strips
// (stitch.cpp:60-70) -> ratio[t - tile_lo], and each strip's row sums
// strip_sums[s][r] = sum_k ratio_k * rowsum_k[r] over its slots (the rows of the
// assembled strip the vertical chain averages). Tiles' column / row sums come
// from the device (complex128), the ratios are formed in double on the host.
void band_sums(const MosaicBand& b, const float2* tiles, C128* strip_sums, C128* ratio, cudaStream_t s) {
    const StitchLayout& lay = b.lay;
    const int N = b.N, Tb = b.tile_hi - b.tile_lo;
    for (int t = 0; t < Tb; ++t) ratio[t] = C128(1.0, 0.0);
    if (!b.exchange) return;  // every overlap is 0: tiles concatenate unscaled (stitch.cpp:38)
    const std::vector<fpmk::StitchTile> st = band_tiles(b);
    DevBuf<fpmk::StitchTile> st_d;
    DevBuf<double> colsum_d, rowsum_d;
    st_d.upload(st.data(), st.size(), s);
    colsum_d.ensure(size_t(Tb) * N * 2);
    rowsum_d.ensure(size_t(Tb) * N * 2);
    ck(fpmk::launch_stitch_sums(tiles, st_d.p, Tb, N, colsum_d.p, rowsum_d.p, s), "stitch sums");
    std::vector<C128> colsum(size_t(Tb) * N), rowsum(size_t(Tb) * N);
    ck(cudaMemcpyAsync(colsum.data(), colsum_d.p, sizeof(C128) * colsum.size(), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(rowsum.data(), rowsum_d.p, sizeof(C128) * rowsum.size(), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "stitch sums");
    const int t0 = b.tile_lo;
    // horizontal: ratio of the strip's trailing overlap mean to the tile's leading mean
    for (int sidx = b.strip_lo; sidx < b.strip_hi; ++sidx)
        for (int k = 1; k < lay.n_cols; ++k) {
            const int o = lay.ovh[size_t(k)];
            if (o == 0) continue;  // zero overlap concatenates unscaled (stitch.cpp:38)
            const int t = lay.grid[size_t(sidx) * lay.n_cols + k] - t0;
            C128 m1 = 0.0, m2 = 0.0;
            for (int C = lay.X[size_t(k)]; C < lay.X[size_t(k)] + o; ++C) {
                // owner at the time tile k is joined: slot k-1 still reaches the strip's end
                const int j = lay.grid[size_t(sidx) * lay.n_cols + std::min(lay.col_of[size_t(C)], k - 1)] - t0;
                m1 += ratio[j] * colsum[size_t(j) * N + (C - st[size_t(j)].X)];
            }
            for (int q = 0; q < o; ++q) m2 += colsum[size_t(t) * N + q];
            const double cnt = double(N) * o;
            if (std::abs(m2 / cnt) < 1e-12) throw DataError("degenerate overlap: |mu2| vanishes");
            ratio[t] = m1 / m2;
        }
    for (int sidx = b.strip_lo; sidx < b.strip_hi; ++sidx)
        for (int r = 0; r < N; ++r) {
            C128 acc = 0.0;
            for (int k = 0; k < lay.n_cols; ++k) {
                const int j = lay.grid[size_t(sidx) * lay.n_cols + k] - t0;
                acc += ratio[j] * rowsum[size_t(j) * N + r];
            }
            strip_sums[size_t(sidx) * N + r] = acc;
        }
}

// Phase 2 (per band, after every band's strip sums are in strip_sums): the
// vertical mean_ratio chain over strips [0, strip_hi) (stitch.cpp:72-84), then
// the band's mosaic rows written at out (row 0 of the whole mosaic, `pitch`
// elements per row; a peer GPU's buffer for a multi-GPU mosaic).
void band_assemble(const MosaicBand& b, const float2* tiles, const C128* strip_sums, const C128* ratio,
                   float2* out, long long pitch, cudaStream_t s) {
    const StitchLayout& lay = b.lay;
    std::vector<C128> S(size_t(lay.n_strips), C128(1.0, 0.0));
    if (b.exchange) {
        const int N = b.N;
        for (int k = 1; k < b.strip_hi; ++k) {
            const int o = lay.ovv[size_t(k)];
            if (o == 0) continue;
            C128 m1 = 0.0, m2 = 0.0;
            for (int Rr = lay.Y[size_t(k)]; Rr < lay.Y[size_t(k)] + o; ++Rr) {
                const int so = std::min(lay.row_of[size_t(Rr)], k - 1);
                m1 += S[size_t(so)] * strip_sums[size_t(so) * N + (Rr - lay.Y[size_t(so)])];
            }
            for (int r = 0; r < o; ++r) m2 += strip_sums[size_t(k) * N + r];
            const double cnt = double(lay.cols) * o;
            if (std::abs(m2 / cnt) < 1e-12) throw DataError("degenerate overlap: |mu2| vanishes");
            S[size_t(k)] = m1 / m2;
        }
    }
    std::vector<fpmk::StitchTile> st = band_tiles(b);
    std::vector<int> grid;
    for (int sidx = b.strip_lo; sidx < b.strip_hi; ++sidx)
        for (int k = 0; k < lay.n_cols; ++k) {
            const int t = lay.grid[size_t(sidx) * lay.n_cols + k] - b.tile_lo;
            grid.push_back(t);
            const C128 f = S[size_t(sidx)] * ratio[t];
            st[size_t(t)].fre = float(f.real());
            st[size_t(t)].fim = float(f.imag());
        }
    DevBuf<fpmk::StitchTile> st_d;
    DevBuf<int> row_d, col_d, grid_d;
    st_d.upload(st.data(), st.size(), s);
    row_d.upload(lay.row_of.data(), lay.row_of.size(), s);
    col_d.upload(lay.col_of.data(), lay.col_of.size(), s);
    grid_d.upload(grid.data(), grid.size(), s);
    ck(fpmk::launch_stitch_assemble(tiles, st_d.p, row_d.p, col_d.p, grid_d.p, b.strip_lo, lay.n_cols, b.N, b.row_lo,
                                    b.row_hi - b.row_lo, lay.cols, pitch, out, s), "stitch assemble");
    ck(cudaStreamSynchronize(s), "stitch assemble");  // the temporaries above are freed on return
}

// stitch_mosaic (stitch.cpp:48-86) on one GPU: the band of every tile.
void stitch_device(const Cfg& c, const int* xy, int T, const float2* tiles, float2* out, cudaStream_t s) {
    const MosaicBand b = mosaic_band(c, xy, T, 0, T);
    std::vector<C128> sums(size_t(b.lay.n_strips) * b.N);
    std::vector<C128> ratio(static_cast<size_t>(T));
    band_sums(b, tiles, sums.data(), ratio.data(), s);
    band_assemble(b, tiles, sums.data(), ratio.data(), out, b.lay.cols, s);
}

}  // namespace

extern "C" {

int fpmgpu_version(void) { return 1; }
const char* fpmgpu_last_error(void) { return g_err.c_str(); }
int fpmgpu_last_min_lag(void) { return g_min_lag; }
void fpmgpu_default_config(fpmgpu_optical_config* cfg) { default_config(*cfg); }

int fpmgpu_validate_config(const fpmgpu_optical_config* cfg) { return guarded([&] { validate(*cfg); }); }

int fpmgpu_illumination_wavevector(const fpmgpu_optical_config* cfg, int led_row, int led_col, double cx,
                                   double cy, double* fx, double* fy) {
    return guarded([&] {
        auto k = wavevector(*cfg, led_row, led_col, cx, cy);
        *fx = k.first;
        *fy = k.second;
    });
}

int fpmgpu_build_pupil(const fpmgpu_optical_config* cfg, int grid, double defocus_um, double* values,
                       double* radius_px) {
    return guarded([&] {
        auto v = build_pupil(*cfg, grid, defocus_um, radius_px);
        if (values) std::memcpy(values, v.data(), v.size() * sizeof(double));
    });
}

int fpmgpu_synthesized_na(const fpmgpu_optical_config* cfg, double* out) {
    return guarded([&] { *out = synthesized_na(*cfg); });
}

int fpmgpu_tile_origins(int fov, int tile_size, int tile_overlap, int* out, int cap, int* count) {
    return guarded([&] {
        auto v = tile_origins(fov, tile_size, tile_overlap);
        *count = int(v.size());
        for (int i = 0; i < int(v.size()) && i < cap; ++i) out[i] = v[size_t(i)];
    });
}

int fpmgpu_partition_tiles(const fpmgpu_optical_config* cfg, int fov_w, int fov_h, const int* seq, int num_leds,
                           int cap, int* count, int* xy, double* centers, double* kvecs, int* offsets) {
    return guarded([&] {
        const auto xs = tile_origins(fov_w, cfg->tile_size, cfg->tile_overlap);
        const auto ys = tile_origins(fov_h, cfg->tile_size, cfg->tile_overlap);
        *count = int(xs.size() * ys.size());
        int t = 0;
        for (int y0 : ys)
            for (int x0 : xs) {
                if (t >= cap) return;
                auto [cx, cy] = tile_center_um(*cfg, x0, y0, fov_w, fov_h);
                if (xy) {
                    xy[2 * t] = x0;
                    xy[2 * t + 1] = y0;
                }
                if (centers) {
                    centers[2 * t] = cx;
                    centers[2 * t + 1] = cy;
                }
                for (int k = 0; k < num_leds; ++k) {
                    auto [fx, fy] = wavevector(*cfg, seq[2 * k], seq[2 * k + 1], cx, cy);
                    const size_t q = (size_t(t) * num_leds + k) * 2;
                    if (kvecs) {
                        kvecs[q] = fx;
                        kvecs[q + 1] = fy;
                    }
                    if (offsets) {
                        auto [oy, ox] = spectrum_offset_px(*cfg, fx, fy);
                        offsets[q] = oy;
                        offsets[q + 1] = ox;
                    }
                }
                ++t;
            }
    });
}

int fpmgpu_sequence_offsets(int order, int rows, int cols, int* out) {
    return guarded([&] {
        auto v = sequence_offsets(order, rows, cols);
        for (size_t i = 0; i < v.size(); ++i) {
            out[2 * i] = v[i].first;
            out[2 * i + 1] = v[i].second;
        }
    });
}

int fpmgpu_spectrum_offset_px(const fpmgpu_optical_config* cfg, double fx, double fy, int* oy, int* ox) {
    return guarded([&] {
        auto o = spectrum_offset_px(*cfg, fx, fy);
        *oy = o.first;
        *ox = o.second;
    });
}

int fpmgpu_min_safe_lag(const int* offsets, int count, double radius_px, int* out) {
    return guarded([&] {
        std::vector<std::pair<int, int>> v;
        for (int i = 0; i < count; ++i) v.emplace_back(offsets[2 * i], offsets[2 * i + 1]);
        *out = min_safe_lag(v, radius_px);
    });
}

int fpmgpu_build_schedule(int positions, int iters, int lag, int* entries, int* rounds) {
    return guarded([&] {
        if (positions < 1 || iters < 1 || lag < 1) throw ConfigError("invalid schedule parameters");
        const int R = (positions - 1) + (iters - 1) * lag + 1;
        *rounds = R;
        size_t q = 0;
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < iters; ++s) {
                const int p = r - s * lag;
                if (p < 0 || p >= positions) continue;
                entries[3 * q] = r;
                entries[3 * q + 1] = s;
                entries[3 * q + 2] = p;
                ++q;
            }
    });
}

int fpmgpu_create(int device, fpmgpu_context** out) {
    return guarded([&] {
        auto c = std::make_unique<fpmgpu_context>();
        c->device = device;
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        *out = c.release();
    });
}

int fpmgpu_destroy(fpmgpu_context* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        for (auto& sl : ctx->slots) {
            for (auto st : sl.streams) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
            for (auto* p : sl.plans) delete p;
            for (auto e : sl.arrived) cudaEventDestroy(e);
            for (auto e : sl.done) cudaEventDestroy(e);
        }
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int fpmgpu_plan_create(fpmgpu_context* ctx, const fpmgpu_recon_request* req, fpmgpu_plan** out) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        auto p = std::make_unique<fpmgpu_plan>();
        p->ctx = ctx;
        build_plan(*p, *req);
        ck(cudaStreamSynchronize(ctx->stream), "plan upload");
        *out = p.release();
    });
}

int fpmgpu_plan_execute(fpmgpu_plan* plan, const uint16_t* frames_dev, int64_t row_pitch, float* hr_dev,
                        double* residuals_dev, float* pupils_out_dev, void* stream) {
    return guarded([&] {
        execute_plan(*plan, frames_dev, row_pitch, hr_dev, residuals_dev, pupils_out_dev,
                     static_cast<cudaStream_t>(stream));
    });
}

int fpmgpu_plan_execute_mosaic(fpmgpu_plan* plan, const uint16_t* frames_dev, int64_t row_pitch, float* mosaic_dev,
                               int64_t mosaic_pitch, double* residuals_dev, float* pupils_out_dev, void* stream) {
    return guarded([&] {
        if (mosaic_pitch < 1) throw DataError("mosaic pitch must be positive");
        if (!plan->abut) throw Unsupported("the tiles overlap or leave gaps: stitch the HR tiles instead");
        execute_plan(*plan, frames_dev, row_pitch, mosaic_dev, residuals_dev, pupils_out_dev,
                     static_cast<cudaStream_t>(stream), mosaic_pitch);
    });
}

int fpmgpu_plan_destroy(fpmgpu_plan* plan) {
    return guarded([&] { delete plan; });
}

int fpmgpu_plan_get_info(const fpmgpu_plan* p, fpmgpu_plan_info* info) {
    return guarded([&] {
        std::memset(info, 0, sizeof(*info));
        info->tile_side = p->n;
        info->canvas_side = p->N;
        info->num_tiles = p->T;
        info->num_leds = p->L;
        info->iters = p->req.iters;
        info->mode = p->req.mode;
        info->lag = p->lag;
        info->groups = p->G;
        info->launches_per_execute = (p->has_pupils ? 0 : 1) + 2 + 1 + 2;
        info->loop_ctas = p->T * (p->cl ? p->cl : 1);
        info->loop_threads = p->cl ? 32 * fpmk::cluster_warps(p->n, p->cl) : p->use_box ? 512 : p->quad ? 256 : 128 * p->G;
        info->loop_smem_bytes =
            int(p->cl ? fpmk::cluster_smem_bytes(p->n, p->box, p->cl, fpmk::cluster_warps(p->n, p->cl), p->L,
                                                 p->req.iters)
                : p->use_box ? fpmk::box_smem_bytes(p->n, p->box, p->L, p->req.iters, p->n != 256)
                : p->quad    ? fpmk::loop64q_smem_bytes(p->L, p->req.iters, true)
                             : fpmk::loop_smem_bytes(p->G, p->nslots, p->L, p->req.iters));
        info->updates = double(p->T) * p->L * p->req.iters;
        info->fft_flops_per_update = 20.0 * p->n * p->n * std::log2(double(p->n));
        info->hbm_bytes_per_update = 2.0 * p->n * p->n + 16.0 * p->support_px;
        info->support_pixels = p->support_px;
        info->tiles_abut = p->abut ? 1 : 0;
    });
}

int fpmgpu_plan_phase_times(fpmgpu_plan* plan, double* ms, int* executes, int reset) {
    return guarded([&] {
        ms[0] = ms[1] = ms[2] = 0.0;
        for (int k = 0; k < plan->recorded; ++k) {
            cudaEvent_t* e = plan->events.data() + size_t(k) * 4;
            for (int ph = 0; ph < 3; ++ph) {
                float t = 0.f;
                ck(cudaEventElapsedTime(&t, e[ph], e[ph + 1]), "cudaEventElapsedTime");
                ms[ph] += t;
            }
        }
        *executes = plan->recorded;
        if (reset) plan->recorded = 0;
    });
}

namespace {

// Host-path banding: the tiles are cut into contiguous index chunks at tile-row
// changes (row-major partitions make each chunk a horizontal band of the FOV),
// so band b's LR rows can cross PCIe while band b-1 already reconstructs and
// band b-2's HR tiles travel back. FPM_B200_BANDS overrides the count (1 = off).
// The pipelined schedule picks ONE lag for the whole batch, so it stays unbanded.
std::vector<int> host_bands(const fpmgpu_recon_request& r, int want) {
    const int T = r.num_tiles;
    if (const char* e = std::getenv("FPM_B200_BANDS")) want = std::max(1, std::atoi(e));
    std::vector<int> row_start;  // tile indices where a new tile row begins
    for (int t = 0; t < T; ++t)
        if (t == 0 || r.tile_xy[2 * t + 1] != r.tile_xy[2 * t - 1]) row_start.push_back(t);
    const int rows = int(row_start.size());
    if (r.lag != 0 || want <= 1 || rows < 2) return {0, T};
    const int B = std::min(want, rows);
    std::vector<int> t0{0};
    for (int b = 1; b < B; ++b) {
        const int cut = row_start[size_t(b) * rows / B];
        if (cut > t0.back()) t0.push_back(cut);
    }
    t0.push_back(T);
    return t0;
}

}  // namespace

namespace {

void wait_slot(HostSlot& sl) {
    if (sl.ticket < 0) return;
    for (auto e : sl.done) ck(cudaEventSynchronize(e), "reconstruct");
    sl.ticket = -1;
}

// Enqueue one host-buffer reconstruction on slot `sl` (returns before it completes).
void submit(fpmgpu_context* ctx, HostSlot& sl, const fpmgpu_recon_request* req, const uint16_t* frames,
            int64_t row_pitch, float* hr, double* residuals, float* pupils_out, int bands) {
    cudaStream_t s = ctx->stream;
    std::vector<int> ki;
    std::vector<double> kd;
    std::vector<float> kf;
    const std::vector<int> t0 = host_bands(*req, bands);
    const int B = int(t0.size()) - 1;
    const bool hit = same_request(sl, *req, ki, kd, kf) && sl.band_t0 == t0;
    if (!hit) {
        for (auto* q : sl.plans) delete q;
        sl.plans.clear();
        sl.band_t0.clear();
        for (int b = 0; b < B; ++b) {
            // band b: the same request over tiles [t0[b], t0[b+1])
            fpmgpu_recon_request rb = *req;
            const int a = t0[b], cnt = t0[b + 1] - t0[b];
            rb.num_tiles = cnt;
            rb.tile_xy = req->tile_xy + 2 * size_t(a);
            rb.offsets = req->offsets + 2 * size_t(a) * req->num_leds;
            if (req->tile_defocus_um) rb.tile_defocus_um = req->tile_defocus_um + a;
            if (req->pupils) rb.pupils = req->pupils + 2 * size_t(a) * req->cfg.tile_size * req->cfg.tile_size;
            auto p = std::make_unique<fpmgpu_plan>();
            p->ctx = ctx;
            p->batch_tiles = req->num_tiles;  // the bands run concurrently: size kernels for the whole request
            build_plan(*p, rb);
            sl.plans.push_back(p.release());
        }
        sl.band_t0 = t0;
        sl.key_i.swap(ki);
        sl.key_d.swap(kd);
        sl.key_f.swap(kf);
    }
    while (int(sl.streams.size()) < B) {
        cudaStream_t bs;
        cudaEvent_t e0, e1;
        ck(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "event");
        sl.streams.push_back(bs);
        sl.arrived.push_back(e0);
        sl.done.push_back(e1);
    }
    const fpmgpu_plan& p0 = *sl.plans[0];
    const int W = req->width, H = req->height, F = req->num_frames, T = req->num_tiles;
    const int n = p0.n, N = p0.N, iters = req->iters;
    const int64_t pitch = (int64_t(W) + 63) / 64 * 64;
    uint16_t* fd = sl.frames.ensure(size_t(F) * H * pitch);
    const size_t hr_n = size_t(T) * N * N, pup_n = size_t(T) * n * n;
    float2* hr_d = hr ? sl.hr.ensure(hr_n) : nullptr;
    double* res_d = sl.resid.ensure(size_t(T) * iters);
    float2* pup_d = pupils_out ? sl.pup.ensure(pup_n) : nullptr;
    ctx->twiddle_table(N);  // its one-time upload must precede the band events on s
    // frame rows [lo, hi) of every frame: one pitched 3-D copy (x bytes, rows, frames)
    auto copy_rows = [&](int lo, int hi) {
        if (hi <= lo) return;
        cudaMemcpy3DParms m{};
        m.srcPtr = make_cudaPitchedPtr(const_cast<uint16_t*>(frames), size_t(row_pitch) * 2, size_t(W) * 2, H);
        m.dstPtr = make_cudaPitchedPtr(fd, size_t(pitch) * 2, size_t(W) * 2, H);
        m.srcPos = make_cudaPos(0, size_t(lo), 0);
        m.dstPos = make_cudaPos(0, size_t(lo), 0);
        m.extent = make_cudaExtent(size_t(W) * 2, size_t(hi - lo), size_t(F));
        m.kind = cudaMemcpyHostToDevice;
        ck(cudaMemcpy3DAsync(&m, s), "frames H2D");
    };
    int clo = 0, chi = 0;  // rows already on the device: [clo, chi)
    for (int b = 0; b < B; ++b) {
        int y0 = H, y1 = 0;
        for (int t = t0[b]; t < t0[b + 1]; ++t) {
            y0 = std::min(y0, req->tile_xy[2 * t + 1]);
            y1 = std::max(y1, req->tile_xy[2 * t + 1] + n);
        }
        if (chi <= clo) {
            copy_rows(y0, y1);
            clo = y0;
            chi = y1;
        } else {
            copy_rows(std::min(y0, clo), clo);
            copy_rows(chi, std::max(y1, chi));
            clo = std::min(y0, clo);
            chi = std::max(y1, chi);
        }
        cudaStream_t bs = sl.streams[b];
        ck(cudaEventRecord(sl.arrived[b], s), "event");
        ck(cudaStreamWaitEvent(bs, sl.arrived[b], 0), "wait");
        fpmgpu_plan& pb = *sl.plans[b];
        const size_t a = size_t(t0[b]);
        execute_plan(pb, fd, pitch, hr_d ? reinterpret_cast<float*>(hr_d + a * N * N) : nullptr, res_d + a * iters,
                     pup_d ? reinterpret_cast<float*>(pup_d + a * n * n) : nullptr, bs);
    }
    // Copies back only after every band's upload and kernels are enqueued: to
    // pageable host memory a D2H cudaMemcpyAsync returns only when it is done,
    // which would otherwise hold back the next band's upload until this band's
    // reconstruction finished (pinned outputs overlap either way).
    for (int b = 0; b < B; ++b) {
        cudaStream_t bs = sl.streams[b];
        const size_t a = size_t(t0[b]), cnt = size_t(t0[b + 1] - t0[b]);
        if (hr)
            ck(cudaMemcpyAsync(hr + 2 * a * N * N, hr_d + a * N * N, cnt * N * N * sizeof(float2),
                               cudaMemcpyDeviceToHost, bs), "hr D2H");
        if (residuals)
            ck(cudaMemcpyAsync(residuals + a * iters, res_d + a * iters, sizeof(double) * cnt * iters,
                               cudaMemcpyDeviceToHost, bs), "residual D2H");
        if (pupils_out)
            ck(cudaMemcpyAsync(pupils_out + 2 * a * n * n, pup_d + a * n * n, cnt * n * n * sizeof(float2),
                               cudaMemcpyDeviceToHost, bs), "pupil D2H");
        ck(cudaEventRecord(sl.done[b], bs), "event");
    }
    sl.lag = p0.lag;
}

// the slot a new request goes to: request k uses slot k mod 2 (waiting for k - 2)
HostSlot& slot_for(fpmgpu_context* ctx, long long ticket) { return ctx->slots[ticket & 1]; }

}  // namespace

namespace {

// Bands per request (measured on config 3): a lone call hides its upload best
// with 8 bands (54 ms vs 56 with 4); back-to-back calls already overlap one
// request's upload with the previous reconstruction, and 4 bands keep the
// launches larger (38.7 ms per request vs 41.8 with 8).
int submit_async(fpmgpu_context* ctx, const fpmgpu_recon_request* req, const uint16_t* frames, int64_t row_pitch,
                 float* hr, double* residuals, float* pupils_out, long long* ticket, int bands) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const long long t = ctx->next_ticket;
        HostSlot& sl = slot_for(ctx, t);
        wait_slot(sl);  // its buffers and plans are free once request t - 2 is done
        submit(ctx, sl, req, frames, row_pitch, hr, residuals, pupils_out, bands);
        sl.ticket = t;
        ctx->lag_of[t & 1] = sl.lag;
        ctx->next_ticket = t + 1;
        if (ticket) *ticket = t;
    });
}

}  // namespace

int fpmgpu_reconstruct_tiles_async(fpmgpu_context* ctx, const fpmgpu_recon_request* req, const uint16_t* frames,
                                   int64_t row_pitch, float* hr, double* residuals, float* pupils_out,
                                   long long* ticket) {
    return submit_async(ctx, req, frames, row_pitch, hr, residuals, pupils_out, ticket, 4);
}

int fpmgpu_wait(fpmgpu_context* ctx, long long ticket, int* lag_used) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (ticket < 0 || ticket >= ctx->next_ticket) throw DataError("unknown reconstruction ticket");
        // a ticket older than the two slots completed when its slot was reused
        HostSlot& sl = slot_for(ctx, ticket);
        if (sl.ticket == ticket) wait_slot(sl);
        if (lag_used) *lag_used = ctx->lag_of[ticket & 1];
    });
}

int fpmgpu_reconstruct_tiles(fpmgpu_context* ctx, const fpmgpu_recon_request* req, const uint16_t* frames,
                             int64_t row_pitch, float* hr, double* residuals, float* pupils_out, int* lag_used) {
    long long t = -1;
    const int rc = submit_async(ctx, req, frames, row_pitch, hr, residuals, pupils_out, &t, 8);
    if (rc != FPMGPU_OK) return rc;
    return fpmgpu_wait(ctx, t, lag_used);
}

struct fpmgpu_online {
    fpmgpu_context* ctx = nullptr;
    std::unique_ptr<fpmgpu_plan> plan;
    DevBuf<uint16_t> frames;
    DevBuf<double> resid;
    DevBuf<float2> hr;
    int64_t pitch = 0;
    cudaStream_t copy = nullptr, comp = nullptr;
    std::vector<cudaEvent_t> arrived;  // per frame: its H2D copy is complete
    std::vector<uint8_t> present;
    std::vector<int> seq_frame;  // host copy (the plan keeps no caller pointers)
    bool seeded = false;
    int next = 0;  // first sequence position not yet launched
    ~fpmgpu_online() {
        if (comp) cudaStreamSynchronize(comp);
        if (copy) cudaStreamSynchronize(copy);
        for (auto e : arrived) cudaEventDestroy(e);
        if (comp) cudaStreamDestroy(comp);
        if (copy) cudaStreamDestroy(copy);
    }
};

int fpmgpu_online_begin(fpmgpu_context* ctx, const fpmgpu_recon_request* req, fpmgpu_online** out) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (req->lag != 0) throw ConfigError("online mode runs the sequential schedule (lag 0)");
        auto on = std::make_unique<fpmgpu_online>();
        on->ctx = ctx;
        on->plan = std::make_unique<fpmgpu_plan>();
        on->plan->ctx = ctx;
        build_plan(*on->plan, *req);
        const fpmgpu_plan& p = *on->plan;
        on->pitch = (int64_t(req->width) + 63) / 64 * 64;
        on->frames.ensure(size_t(p.F) * req->height * on->pitch);
        on->resid.ensure(size_t(p.T) * req->iters);
        ck(cudaStreamCreateWithFlags(&on->copy, cudaStreamNonBlocking), "stream");
        ck(cudaStreamCreateWithFlags(&on->comp, cudaStreamNonBlocking), "stream");
        on->arrived.resize(size_t(p.F));
        for (auto& e : on->arrived) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        on->present.assign(size_t(p.F), 0);
        on->seq_frame.assign(req->seq_frame, req->seq_frame + p.L);
        ctx->twiddle_table(p.N);
        // the plan's table uploads and the twiddles went out on the context stream
        ck(cudaStreamSynchronize(ctx->stream), "online begin");
        ck(cudaMemsetAsync(on->resid.p, 0, sizeof(double) * size_t(p.T) * req->iters, on->comp), "residual clear");
        *out = on.release();
    });
}

int fpmgpu_online_push(fpmgpu_online* on, int frame_index, const uint16_t* frame, int64_t row_pitch,
                       int* positions_applied) {
    return guarded([&] {
        ck(cudaSetDevice(on->ctx->device), "cudaSetDevice");
        fpmgpu_plan& p = *on->plan;
        const fpmgpu_recon_request& r = p.req;
        if (frame_index < 0 || frame_index >= p.F) throw DataError("frame index outside the frame set");
        if (on->present[size_t(frame_index)]) throw DataError("frame pushed twice");
        uint16_t* dst = on->frames.p + size_t(frame_index) * r.height * on->pitch;
        ck(cudaMemcpy2DAsync(dst, size_t(on->pitch) * 2, frame, size_t(row_pitch) * 2, size_t(r.width) * 2,
                             size_t(r.height), cudaMemcpyHostToDevice, on->copy), "frame H2D");
        ck(cudaEventRecord(on->arrived[size_t(frame_index)], on->copy), "event");
        on->present[size_t(frame_index)] = 1;
        if (!on->seeded && on->present[size_t(r.init_frame)]) {
            ck(cudaStreamWaitEvent(on->comp, on->arrived[size_t(r.init_frame)], 0), "wait");
            plan_prologue(p, on->frames.p, on->pitch, on->comp);
            on->seeded = true;
        }
        if (on->seeded) {
            int k = on->next;
            while (k < p.L && on->present[size_t(on->seq_frame[size_t(k)])]) {
                ck(cudaStreamWaitEvent(on->comp, on->arrived[size_t(on->seq_frame[size_t(k)])], 0), "wait");
                ++k;
            }
            if (k > on->next) {  // first-pass slots [next, k): stage 0, positions next .. k-1
                plan_loop(p, on->frames.p, on->pitch, on->resid.p, on->next, k, true, on->comp);
                on->next = k;
            }
        }
        if (positions_applied) *positions_applied = on->next;
    });
}

int fpmgpu_online_finish(fpmgpu_online* on, float* hr, double* residuals, float* pupils_out) {
    return guarded([&] {
        ck(cudaSetDevice(on->ctx->device), "cudaSetDevice");
        fpmgpu_plan& p = *on->plan;
        const fpmgpu_recon_request& r = p.req;
        if (!on->seeded) throw DataError("missing frame for the canvas seed");
        if (on->next < p.L) throw DataError("missing frame for a sequence LED");
        if (r.iters > 1) plan_loop(p, on->frames.p, on->pitch, on->resid.p, p.L, r.iters * p.L, true, on->comp);
        const size_t hr_n = size_t(p.T) * p.N * p.N, pup_n = size_t(p.T) * p.n * p.n;
        float2* hr_d = hr ? on->hr.ensure(hr_n) : nullptr;
        plan_epilogue(p, reinterpret_cast<float*>(hr_d), nullptr, on->comp);
        if (hr) ck(cudaMemcpyAsync(hr, hr_d, hr_n * sizeof(float2), cudaMemcpyDeviceToHost, on->comp), "hr D2H");
        if (residuals)
            ck(cudaMemcpyAsync(residuals, on->resid.p, sizeof(double) * size_t(p.T) * r.iters,
                               cudaMemcpyDeviceToHost, on->comp), "residual D2H");
        if (pupils_out)
            ck(cudaMemcpyAsync(pupils_out, p.pupils.p, pup_n * sizeof(float2), cudaMemcpyDeviceToHost, on->comp),
               "pupil D2H");
        ck(cudaStreamSynchronize(on->comp), "online finish");
    });
}

int fpmgpu_online_destroy(fpmgpu_online* on) {
    return guarded([&] {
        if (!on) return;
        cudaSetDevice(on->ctx->device);
        delete on;
    });
}

int fpmgpu_update_step(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, float* canvas, const float* intensity,
                       double fx, double fy, float* pupil, int mode, double alpha, double beta, double* residual) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int n = cfg->tile_size, N = cfg->tile_size * cfg->upsample;
        if (n != 64 && n != 128 && n != 256)
            throw Unsupported("tile side " + std::to_string(n) + " has no device kernel in this build (64/128/256)");
        const bool use_box = n != 64 || box_forced();
        auto [oy, ox] = spectrum_offset_px(*cfg, fx, fy);
        const int r0 = N / 2 + oy - n / 2, c0 = N / 2 + ox - n / 2;
        if (r0 < 0 || c0 < 0 || r0 + n > N || c0 + n > N) throw DataError("spectrum offset out of canvas bounds");
        std::vector<uint8_t> sup(size_t(n) * n);
        for (size_t i = 0; i < sup.size(); ++i) sup[i] = pupil[2 * i] != 0.f || pupil[2 * i + 1] != 0.f;
        int nslots = 1, b0 = 0, box = 0;
        bool prune = false;
        if (N != 256 && N != 512 && N != 1024) throw Unsupported("canvas side " + std::to_string(N) + " unsupported");
        if (use_box) {
            box_of(sup, n, &b0, &box);
        } else {
            lattice_shape(sup, &nslots, &prune);
            if (!prune && N != 256)
                throw Unsupported("pupil disk wider than the pruned lattice needs canvas side 256 in this build");
        }
        cudaStream_t s = ctx->stream;
        DevBuf<float2> cv, pp;
        DevBuf<float> meas;
        DevBuf<uint8_t> sp;
        DevBuf<short2> org;
        DevBuf<uint8_t> bf;
        DevBuf<int> sf;
        DevBuf<int2> xy;
        DevBuf<double> res;
        cv.upload(reinterpret_cast<const float2*>(canvas), size_t(N) * N, s);
        pp.upload(reinterpret_cast<const float2*>(pupil), size_t(n) * n, s);
        meas.upload(intensity, size_t(n) * n, s);
        sp.upload(sup.data(), sup.size(), s);
        const short2 o = make_short2(short(r0), short(c0));
        org.upload(&o, 1, s);
        const uint8_t is_bf = bright_field(oy, ox, pupil_radius_px(*cfg, n));
        bf.upload(&is_bf, 1, s);
        const int zero = 0;
        sf.upload(&zero, 1, s);
        const int2 z2 = make_int2(0, 0);
        xy.upload(&z2, 1, s);
        res.ensure(1);
        fpmk::LoopArgs a{};
        a.canvas = cv.p;
        a.pupils = pp.p;
        a.support = sp.p;
        a.origins = org.p;
        a.bright = bf.p;
        a.seq_frame = sf.p;
        a.tile_xy = xy.p;
        a.F = 1;
        a.residuals = res.p;
        a.meas_f32 = meas.p;
        a.num_slots = 1;
        a.T = 1;
        a.L = 1;
        a.iters = 1;
        a.N = N;
        a.nslots = nslots;
        a.alpha = float(alpha);
        a.beta = float(beta);
        DevBuf<float2> scratch;
        if (use_box) {
            fpmk::BoxArgs bx{};
            if (n == 256) bx.scratch = scratch.ensure(size_t(box) * (n + 1));
            bx.box = box;
            bx.b0 = b0;
            ck(fpmk::launch_loop_box(n, mode, a, bx, 1, s), "update_step (box)");
        } else {
            CUtensorMap dummy;
            std::memset(&dummy, 0, sizeof(dummy));
            ck(fpmk::launch_loop64(mode, prune, fpmk::kMeasF32, 1, &dummy, a, 1, s), "update_step");
        }
        ck(cudaMemcpyAsync(canvas, cv.p, sizeof(float2) * size_t(N) * N, cudaMemcpyDeviceToHost, s), "canvas D2H");
        if (mode == FPMGPU_MODE_EPRY)
            ck(cudaMemcpyAsync(pupil, pp.p, sizeof(float2) * size_t(n) * n, cudaMemcpyDeviceToHost, s), "pupil D2H");
        ck(cudaMemcpyAsync(residual, res.p, sizeof(double), cudaMemcpyDeviceToHost, s), "residual D2H");
        ck(cudaStreamSynchronize(s), "update_step");
    });
}

int fpmgpu_init_canvas(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const uint16_t* frame, int height,
                       int width, int64_t row_pitch, int x0, int y0, float* canvas) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        validate(*cfg);
        const int n = cfg->tile_size, N = n * cfg->upsample;
        if (x0 < 0 || y0 < 0 || y0 + n > height || x0 + n > width) throw DataError("tile extends past frame bounds");
        cudaStream_t s = ctx->stream;
        DevBuf<uint16_t> fr;
        DevBuf<float2> cv;
        DevBuf<int2> xy;
        fr.ensure(size_t(height) * width);
        ck(cudaMemcpy2DAsync(fr.p, size_t(width) * 2, frame, size_t(row_pitch) * 2, size_t(width) * 2, size_t(height),
                             cudaMemcpyHostToDevice, s), "frame H2D");
        const int2 o = make_int2(x0, y0);
        xy.upload(&o, 1, s);
        cv.ensure(size_t(N) * N);
        fpmk::LinesArgs la{};
        la.tw = ctx->twiddle_table(N);
        la.frame = fr.p;
        la.pitch = width;
        la.tile_xy = xy.p;
        la.n = n;
        la.up = cfg->upsample;
        la.src = cv.p;
        la.dst = cv.p;
        la.scale = 1.0f;
        ck(fpmk::launch_lines(0, N, la, 1, s), "init rows");
        la.scale = float(1.0 / (double(cfg->upsample) * cfg->upsample));
        ck(fpmk::launch_lines(1, N, la, 1, s), "init cols");
        ck(cudaMemcpyAsync(canvas, cv.p, sizeof(float2) * size_t(N) * N, cudaMemcpyDeviceToHost, s), "canvas D2H");
        ck(cudaStreamSynchronize(s), "init_canvas");
    });
}

int fpmgpu_canvas_to_field(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const float* canvas, float* field) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int N = cfg->tile_size * cfg->upsample;
        cudaStream_t s = ctx->stream;
        DevBuf<float2> cv;
        cv.upload(reinterpret_cast<const float2*>(canvas), size_t(N) * N, s);
        fpmk::LinesArgs la{};
        la.tw = ctx->twiddle_table(N);
        la.src = cv.p;
        la.dst = cv.p;
        la.scale = 1.0f;
        ck(fpmk::launch_lines(2, N, la, 1, s), "final rows");
        la.scale = float(double(cfg->upsample) * cfg->upsample / (double(N) * N));
        ck(fpmk::launch_lines(3, N, la, 1, s), "final cols");
        ck(cudaMemcpyAsync(field, cv.p, sizeof(float2) * size_t(N) * N, cudaMemcpyDeviceToHost, s), "field D2H");
        ck(cudaStreamSynchronize(s), "canvas_to_field");
    });
}

int fpmgpu_stitch_mosaic(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const float* tiles, const int* xy,
                         int num_tiles, float* out, int* rows, int* cols) {
    return guarded([&] {
        const StitchLayout lay = stitch_layout(*cfg, xy, num_tiles);
        *rows = lay.rows;
        *cols = lay.cols;
        if (!out) return;
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int N = cfg->tile_size * cfg->upsample;
        DevBuf<float2> t_d, o_d;
        t_d.upload(reinterpret_cast<const float2*>(tiles), size_t(num_tiles) * N * N, ctx->stream);
        o_d.ensure(size_t(lay.rows) * lay.cols);
        stitch_device(*cfg, xy, num_tiles, t_d.p, o_d.p, ctx->stream);
        ck(cudaMemcpyAsync(out, o_d.p, sizeof(float2) * size_t(lay.rows) * lay.cols, cudaMemcpyDeviceToHost,
                           ctx->stream), "mosaic D2H");
        ck(cudaStreamSynchronize(ctx->stream), "stitch_mosaic");
    });
}

int fpmgpu_stitch_mosaic_device(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const float* tiles_dev,
                                const int* xy, int num_tiles, float* out_dev, int* rows, int* cols, void* stream) {
    return guarded([&] {
        const StitchLayout lay = stitch_layout(*cfg, xy, num_tiles);
        *rows = lay.rows;
        *cols = lay.cols;
        if (!out_dev) return;
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        stitch_device(*cfg, xy, num_tiles, reinterpret_cast<const float2*>(tiles_dev),
                      reinterpret_cast<float2*>(out_dev), static_cast<cudaStream_t>(stream));
    });
}

int fpmgpu_mosaic_band_layout(const fpmgpu_optical_config* cfg, const int* xy, int num_tiles, int tile_lo,
                              int tile_hi, fpmgpu_mosaic_band_info* info) {
    return guarded([&] {
        const MosaicBand b = mosaic_band(*cfg, xy, num_tiles, tile_lo, tile_hi);
        info->rows = b.lay.rows;
        info->cols = b.lay.cols;
        info->strips = b.lay.n_strips;
        info->strip_lo = b.strip_lo;
        info->strip_hi = b.strip_hi;
        info->row_lo = b.row_lo;
        info->row_hi = b.row_hi;
        info->canvas_side = b.N;
        info->needs_exchange = b.exchange ? 1 : 0;
    });
}

int fpmgpu_mosaic_band_sums(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const int* xy, int num_tiles,
                            int tile_lo, int tile_hi, const float* tiles_dev, double* strip_sums, double* ratios,
                            void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const MosaicBand b = mosaic_band(*cfg, xy, num_tiles, tile_lo, tile_hi);
        band_sums(b, reinterpret_cast<const float2*>(tiles_dev), reinterpret_cast<C128*>(strip_sums),
                  reinterpret_cast<C128*>(ratios), static_cast<cudaStream_t>(stream));
    });
}

int fpmgpu_mosaic_band_assemble(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const int* xy, int num_tiles,
                                int tile_lo, int tile_hi, const float* tiles_dev, const double* strip_sums,
                                const double* ratios, float* mosaic_dev, int64_t mosaic_pitch, void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        const MosaicBand b = mosaic_band(*cfg, xy, num_tiles, tile_lo, tile_hi);
        if (mosaic_pitch < b.lay.cols) throw DataError("mosaic pitch narrower than the mosaic");
        band_assemble(b, reinterpret_cast<const float2*>(tiles_dev), reinterpret_cast<const C128*>(strip_sums),
                      reinterpret_cast<const C128*>(ratios), reinterpret_cast<float2*>(mosaic_dev), mosaic_pitch,
                      static_cast<cudaStream_t>(stream));
    });
}

int fpmgpu_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset) {
    return guarded([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == FPMGPU_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof(h));
        // the handle names the whole allocation: report where dev_ptr sits in it
        static PFN_cuMemGetAddressRange_v3020 range = nullptr;
        static std::once_flag once;
        std::call_once(once, [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
        });
        if (!range) throw CudaError("cuMemGetAddressRange unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, CUdeviceptr(dev_ptr)) != CUDA_SUCCESS) throw CudaError("cuMemGetAddressRange failed");
        *offset = int64_t(CUdeviceptr(dev_ptr) - base);
    });
}

int fpmgpu_ipc_open(fpmgpu_context* ctx, const void* handle, void** dev_ptr) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        ck(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int fpmgpu_ipc_close(fpmgpu_context* ctx, void* dev_ptr) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    });
}

int fpmgpu_fft2_c128(fpmgpu_context* ctx, double* data_dev, int64_t batch, int rows, int cols, int inverse,
                     void* stream) {
    return guarded([&] {
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (batch < 0 || rows < 1 || cols < 1) throw DataError("fft2: empty or negative shape");
        if (!fpmk::fft_c128_supported(rows) || !fpmk::fft_c128_supported(cols))
            throw Unsupported("fft2: sides must factor into 2, 3 and 5 and be at most 4096");
        if (batch == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        double2* tmp = nullptr;
        const size_t bytes = size_t(batch) * rows * cols * sizeof(double2);
        ck(cudaMallocAsync(reinterpret_cast<void**>(&tmp), bytes, s), "cudaMallocAsync");
        const cudaError_t e = fpmk::fft2_c128(reinterpret_cast<double2*>(data_dev), tmp, batch, rows, cols,
                                               inverse != 0, s);
        cudaFreeAsync(tmp, s);
        ck(e, "fft2_c128");
    });
}

int fpmgpu_host_alloc(int64_t bytes, void** ptr) {
    return guarded([&] { ck(cudaHostAlloc(ptr, size_t(std::max<int64_t>(bytes, 1)), cudaHostAllocPortable), "cudaHostAlloc"); });
}

int fpmgpu_host_free(void* ptr) {
    return guarded([&] { ck(cudaFreeHost(ptr), "cudaFreeHost"); });
}

}  // extern "C"
