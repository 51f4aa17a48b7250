// fpm_b200.hpp — drop-in C++ mirror of the reference's reconstruct API
// (/root/reference/proj/include/fpm/{optics,tiles,forward,recon,parallel,stitch}.hpp)
// over the B200 C-ABI (fpm_b200.h). Same namespace, type and function names,
// argument meaning and exceptions; every transform and update runs on the GPU.
//
// Array types: with Eigen available (as in the reference build) the Eigen
// typedefs of field.hpp:11-13 are used verbatim, so reference call sites
// compile unchanged. Without Eigen a minimal column-major Array2D stands in.
//
// Header-only: link against libfpm_b200.so. The GPU context is process-wide
// (device from $FPM_B200_DEVICE, default 0), created on first use.
#pragma once

#include <chrono>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "fpm_b200.h"

#if defined(FPM_B200_USE_EIGEN) || (!defined(FPM_B200_NO_EIGEN) && __has_include(<Eigen/Dense>))
#include <Eigen/Dense>
#define FPM_B200_HAVE_EIGEN 1
#endif

namespace fpm {

using Complex = std::complex<double>;

#ifdef FPM_B200_HAVE_EIGEN
using ComplexField = Eigen::Array<Complex, Eigen::Dynamic, Eigen::Dynamic>;
using RealField = Eigen::ArrayXXd;
using IntensityImage = Eigen::Array<uint16_t, Eigen::Dynamic, Eigen::Dynamic>;
#else
// Column-major 2-D array with the Eigen calls this header and its tests use.
template <typename T>
class Array2D {
public:
    Array2D() = default;
    Array2D(long rows, long cols) : r_(rows), c_(cols), v_(size_t(rows) * size_t(cols)) {}
    static Array2D Zero(long rows, long cols) { return Array2D(rows, cols); }
    static Array2D Constant(long rows, long cols, T x) {
        Array2D a(rows, cols);
        for (auto& e : a.v_) e = x;
        return a;
    }
    long rows() const { return r_; }
    long cols() const { return c_; }
    long size() const { return long(v_.size()); }
    T& operator()(long i, long j) { return v_[size_t(i) + size_t(j) * size_t(r_)]; }
    const T& operator()(long i, long j) const { return v_[size_t(i) + size_t(j) * size_t(r_)]; }
    T* data() { return v_.data(); }
    const T* data() const { return v_.data(); }

private:
    long r_ = 0, c_ = 0;
    std::vector<T> v_;
};
using ComplexField = Array2D<Complex>;
using RealField = Array2D<double>;
using IntensityImage = Array2D<uint16_t>;
#endif

// ------------------------------------------------------------------ errors (optics.hpp:11-16, parallel.hpp:12-17)
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnsafeLagError : std::runtime_error {
    int minimum;
    explicit UnsafeLagError(int min_lag)
        : std::runtime_error("pipeline lag below the safe minimum of " + std::to_string(min_lag)), minimum(min_lag) {}
};

namespace detail {
inline void check(int rc) {
    if (rc == FPMGPU_OK) return;
    const std::string msg = fpmgpu_last_error();
    switch (rc) {
        case FPMGPU_ERR_CONFIG: throw ConfigError(msg);
        case FPMGPU_ERR_DATA: throw DataError(msg);
        case FPMGPU_ERR_UNSAFE_LAG: throw UnsafeLagError(fpmgpu_last_min_lag());
        case FPMGPU_ERR_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error("fpm_b200: " + msg);
    }
}
struct Context {
    fpmgpu_context* h = nullptr;
    Context() {
        const char* d = std::getenv("FPM_B200_DEVICE");
        check(fpmgpu_create(d ? std::atoi(d) : 0, &h));
    }
    ~Context() { fpmgpu_destroy(h); }
};
inline fpmgpu_context* ctx() {
    static Context c;
    return c.h;
}
// column-major complex<double> <-> row-major complex64 (the C-ABI layout)
template <typename F>
inline std::vector<float> to_c64(const F& f) {
    std::vector<float> out(size_t(f.rows()) * size_t(f.cols()) * 2);
    for (long i = 0; i < f.rows(); ++i)
        for (long j = 0; j < f.cols(); ++j) {
            const Complex z = f(i, j);
            out[(size_t(i) * size_t(f.cols()) + size_t(j)) * 2] = float(z.real());
            out[(size_t(i) * size_t(f.cols()) + size_t(j)) * 2 + 1] = float(z.imag());
        }
    return out;
}
inline ComplexField from_c64(const float* p, long rows, long cols) {
    ComplexField f = ComplexField::Zero(rows, cols);
    for (long i = 0; i < rows; ++i)
        for (long j = 0; j < cols; ++j)
            f(i, j) = Complex(p[(size_t(i) * size_t(cols) + size_t(j)) * 2], p[(size_t(i) * size_t(cols) + size_t(j)) * 2 + 1]);
    return f;
}
}  // namespace detail

// ------------------------------------------------------------------ optics (optics.hpp:18-78)
struct LedIndex {
    int row = 0;
    int col = 0;
    bool operator==(const LedIndex& o) const { return row == o.row && col == o.col; }
    bool operator<(const LedIndex& o) const { return row != o.row ? row < o.row : col < o.col; }
};

struct OpticalConfig {
    double wavelength = 0.525;
    double objective_na = 0.1;
    double magnification = 2.0;
    double camera_pixel = 2.4;
    double led_pitch = 2.5;
    int led_grid_rows = 64;
    int led_grid_cols = 64;
    double led_height = 83.0;
    LedIndex center_led{32, 32};
    int led_scan_rows = 13;
    int led_scan_cols = 13;
    int upsample = 4;
    int tile_size = 256;
    int tile_overlap = 26;
    double acq_pattern_delay = 0.3;
    double acq_exposure = 0.03;

    double dx_obj() const { return camera_pixel / magnification; }
    double dx_hr() const { return dx_obj() / upsample; }
    int hr_size() const { return tile_size * upsample; }
    fpmgpu_optical_config c() const {
        return {wavelength, objective_na, magnification, camera_pixel, led_pitch, led_grid_rows, led_grid_cols,
                led_height, center_led.row, center_led.col, led_scan_rows, led_scan_cols, upsample, tile_size,
                tile_overlap, acq_pattern_delay, acq_exposure};
    }
    void validate() const {
        const auto cc = c();
        detail::check(fpmgpu_validate_config(&cc));
    }
};

struct WaveVector {
    double fx = 0.0;
    double fy = 0.0;
};

struct Pupil {
    int grid = 0;
    double radius_px = 0.0;
    double defocus = 0.0;
    ComplexField values;
};

inline WaveVector illumination_wavevector(LedIndex led, std::pair<double, double> tile_center_um,
                                          const OpticalConfig& cfg) {
    const auto cc = cfg.c();
    WaveVector w;
    detail::check(fpmgpu_illumination_wavevector(&cc, led.row, led.col, tile_center_um.first, tile_center_um.second,
                                                 &w.fx, &w.fy));
    return w;
}

inline Pupil build_pupil(const OpticalConfig& cfg, int grid, double defocus_um) {
    const auto cc = cfg.c();
    Pupil p;
    p.grid = grid;
    p.defocus = defocus_um;
    std::vector<double> v(size_t(grid > 0 ? grid : 1) * size_t(grid > 0 ? grid : 1) * 2);
    detail::check(fpmgpu_build_pupil(&cc, grid, defocus_um, v.data(), &p.radius_px));
    p.values = ComplexField::Zero(grid, grid);
    for (int i = 0; i < grid; ++i)
        for (int j = 0; j < grid; ++j)
            p.values(i, j) = Complex(v[(size_t(i) * grid + j) * 2], v[(size_t(i) * grid + j) * 2 + 1]);
    return p;
}

inline double synthesized_na(const OpticalConfig& cfg) {
    const auto cc = cfg.c();
    double out = 0.0;
    detail::check(fpmgpu_synthesized_na(&cc, &out));
    return out;
}

// ------------------------------------------------------------------ tiles (tiles.hpp:13-28)
struct TileSpec {
    int x0 = 0;
    int y0 = 0;
    int size = 0;
    double center_x_um = 0.0;
    double center_y_um = 0.0;
    double defocus_um = 0.0;
    std::map<LedIndex, WaveVector> wavevectors;
};

inline std::vector<int> tile_origins(int fov, int tile_size, int tile_overlap) {
    int count = 0;
    std::vector<int> out(size_t(fov > 0 ? fov : 1) + 2);
    detail::check(fpmgpu_tile_origins(fov, tile_size, tile_overlap, out.data(), int(out.size()), &count));
    out.resize(size_t(count));
    return out;
}

inline std::vector<TileSpec> partition_tiles(int fov_w, int fov_h, const OpticalConfig& cfg, double defocus_um = 0.0) {
    std::vector<int> leds;
    for (int dr = -cfg.led_scan_rows / 2; dr <= cfg.led_scan_rows / 2; ++dr)
        for (int dc = -cfg.led_scan_cols / 2; dc <= cfg.led_scan_cols / 2; ++dc) {
            leds.push_back(cfg.center_led.row + dr);
            leds.push_back(cfg.center_led.col + dc);
        }
    const int L = int(leds.size() / 2);
    const size_t T = tile_origins(fov_w, cfg.tile_size, cfg.tile_overlap).size() *
                     tile_origins(fov_h, cfg.tile_size, cfg.tile_overlap).size();
    std::vector<int> xy(T * 2);
    std::vector<double> ce(T * 2), kv(T * size_t(L) * 2);
    int count = 0;
    const auto cc = cfg.c();
    detail::check(fpmgpu_partition_tiles(&cc, fov_w, fov_h, leds.data(), L, int(T), &count, xy.data(), ce.data(),
                                         kv.data(), nullptr));
    std::vector<TileSpec> out(T);
    for (size_t t = 0; t < T; ++t) {
        TileSpec& s = out[t];
        s.x0 = xy[2 * t];
        s.y0 = xy[2 * t + 1];
        s.size = cfg.tile_size;
        s.center_x_um = ce[2 * t];
        s.center_y_um = ce[2 * t + 1];
        s.defocus_um = defocus_um;
        for (int k = 0; k < L; ++k)
            s.wavevectors[LedIndex{leds[2 * k], leds[2 * k + 1]}] =
                WaveVector{kv[(t * L + k) * 2], kv[(t * L + k) * 2 + 1]};
    }
    return out;
}

// ------------------------------------------------------------------ frames (forward.hpp:12-26)
struct Frame {
    LedIndex led;
    IntensityImage image;
    double timestamp_s = 0.0;
};

struct FrameSet {
    std::vector<Frame> frames;
    OpticalConfig cfg;
    const Frame* find(LedIndex led) const {
        for (const auto& f : frames)
            if (f.led == led) return &f;
        return nullptr;
    }
    int width() const { return frames.empty() ? 0 : int(frames.front().image.cols()); }
    int height() const { return frames.empty() ? 0 : int(frames.front().image.rows()); }
};

// ------------------------------------------------------------------ recon (recon.hpp:8-71)
using LedSequence = std::vector<LedIndex>;
enum class UpdateOrder { Spiral, Raster };

inline UpdateOrder update_order_from_string(const std::string& s) {
    if (s == "spiral") return UpdateOrder::Spiral;
    if (s == "raster") return UpdateOrder::Raster;
    throw ConfigError("unknown update order: " + s);
}

inline std::vector<std::pair<int, int>> sequence_offsets(UpdateOrder order, int rows, int cols) {
    std::vector<int> v(size_t(rows > 0 ? rows : 1) * size_t(cols > 0 ? cols : 1) * 2);
    detail::check(fpmgpu_sequence_offsets(order == UpdateOrder::Raster ? FPMGPU_ORDER_RASTER : FPMGPU_ORDER_SPIRAL,
                                          rows, cols, v.data()));
    std::vector<std::pair<int, int>> out;
    for (int i = 0; i < rows * cols; ++i) out.emplace_back(v[2 * size_t(i)], v[2 * size_t(i) + 1]);
    return out;
}

inline LedSequence led_sequence(UpdateOrder order, const OpticalConfig& cfg) {
    LedSequence s;
    for (auto [dr, dc] : sequence_offsets(order, cfg.led_scan_rows, cfg.led_scan_cols))
        s.push_back({cfg.center_led.row + dr, cfg.center_led.col + dc});
    return s;
}

struct SpectrumCanvas {
    ComplexField spectrum;
    OpticalConfig cfg;
    std::vector<std::pair<int, int>> updated_offsets;
    int size() const { return int(spectrum.rows()); }
};

inline std::pair<int, int> spectrum_offset_px(const WaveVector& wv, const OpticalConfig& cfg) {
    const auto cc = cfg.c();
    int oy = 0, ox = 0;
    detail::check(fpmgpu_spectrum_offset_px(&cc, wv.fx, wv.fy, &oy, &ox));
    return {oy, ox};
}

inline IntensityImage crop_frame(const IntensityImage& frame, const TileSpec& tile) {
    if (tile.y0 + tile.size > frame.rows() || tile.x0 + tile.size > frame.cols())
        throw DataError("tile extends past frame bounds");
    IntensityImage out = IntensityImage::Zero(tile.size, tile.size);
    for (int i = 0; i < tile.size; ++i)
        for (int j = 0; j < tile.size; ++j) out(i, j) = frame(tile.y0 + i, tile.x0 + j);
    return out;
}

struct ReconMetrics {
    std::vector<double> pass_mean_residual;
    double wall_s = 0.0;
};
struct ReconResult {
    ComplexField hr;
    ReconMetrics metrics;
};

namespace detail {
// [F][H][W] row-major u16 copy of a FrameSet (the reference stores Eigen column-major frames)
inline std::vector<uint16_t> pack_frames(const FrameSet& fs) {
    const size_t H = size_t(fs.height()), W = size_t(fs.width());
    std::vector<uint16_t> out(fs.frames.size() * H * W);
    for (size_t f = 0; f < fs.frames.size(); ++f)
        for (size_t i = 0; i < H; ++i)
            for (size_t j = 0; j < W; ++j) out[(f * H + i) * W + j] = fs.frames[f].image(long(i), long(j));
    return out;
}
inline int seed_frame(const FrameSet& fs, const OpticalConfig& cfg) {
    for (size_t f = 0; f < fs.frames.size(); ++f)
        if (fs.frames[f].led == cfg.center_led) return int(f);
    if (fs.frames.empty()) throw DataError("empty frame set");
    std::fprintf(stderr, "fpm: warning: on-axis frame missing, initializing from brightest frame\n");
    int best = 0;
    double bm = -1.0;
    for (size_t f = 0; f < fs.frames.size(); ++f) {
        double s = 0.0;
        const auto& im = fs.frames[f].image;
        for (long i = 0; i < im.rows(); ++i)
            for (long j = 0; j < im.cols(); ++j) s += double(im(i, j));
        if (s / double(im.rows() * im.cols()) > bm) {
            bm = s / double(im.rows() * im.cols());
            best = int(f);
        }
    }
    return best;
}
struct Batch {
    std::vector<int> xy, offsets, seq_frame;
    std::vector<double> defocus;
};
inline Batch make_batch(const FrameSet& fs, const std::vector<TileSpec>& tiles, const OpticalConfig& cfg,
                        const LedSequence& seq) {
    Batch b;
    for (const auto& led : seq) {
        int idx = -1;
        for (size_t f = 0; f < fs.frames.size() && idx < 0; ++f)
            if (fs.frames[f].led == led) idx = int(f);
        if (idx < 0)
            throw DataError("missing frame for LED (" + std::to_string(led.row) + "," + std::to_string(led.col) + ")");
        b.seq_frame.push_back(idx);
    }
    for (const auto& t : tiles) {
        b.xy.push_back(t.x0);
        b.xy.push_back(t.y0);
        b.defocus.push_back(t.defocus_um);
        for (const auto& led : seq) {
            auto [oy, ox] = spectrum_offset_px(t.wavevectors.at(led), cfg);
            b.offsets.push_back(oy);
            b.offsets.push_back(ox);
        }
    }
    return b;
}
struct BatchOut {
    std::vector<float> hr;
    std::vector<double> residuals;
    int lag = 0;
};
inline BatchOut run_batch(const FrameSet& fs, const std::vector<TileSpec>& tiles, const OpticalConfig& cfg,
                          int iters, const LedSequence& seq, int lag, bool force_unsafe, int mode = FPMGPU_MODE_GS,
                          double alpha = 1.0, double beta = 1.0) {
    if (iters < 1) throw ConfigError("iters must be >= 1");
    Batch b = make_batch(fs, tiles, cfg, seq);
    const std::vector<uint16_t> px = pack_frames(fs);
    fpmgpu_recon_request r{};
    r.cfg = cfg.c();
    r.iters = iters;
    r.mode = mode;
    r.alpha = alpha;
    r.beta = beta;
    r.lag = lag;
    r.force_unsafe_lag = force_unsafe;
    r.num_tiles = int(tiles.size());
    r.tile_xy = b.xy.data();
    r.num_leds = int(seq.size());
    r.offsets = b.offsets.data();
    r.seq_frame = b.seq_frame.data();
    r.init_frame = seed_frame(fs, cfg);
    bool any_defocus = false;
    for (double z : b.defocus) any_defocus |= z != 0.0;
    r.tile_defocus_um = any_defocus ? b.defocus.data() : nullptr;
    r.num_frames = int(fs.frames.size());
    r.height = fs.height();
    r.width = fs.width();
    BatchOut o;
    const size_t N = size_t(cfg.hr_size());
    o.hr.resize(tiles.size() * N * N * 2);
    o.residuals.resize(tiles.size() * size_t(iters));
    check(fpmgpu_reconstruct_tiles(ctx(), &r, px.data(), fs.width(), o.hr.data(), o.residuals.data(), nullptr, &o.lag));
    return o;
}
}  // namespace detail

inline SpectrumCanvas init_canvas(const FrameSet& frames, const TileSpec& tile, const OpticalConfig& cfg) {
    const int f = detail::seed_frame(frames, cfg);
    const auto& im = frames.frames[size_t(f)].image;
    std::vector<uint16_t> px(size_t(im.rows()) * size_t(im.cols()));
    for (long i = 0; i < im.rows(); ++i)
        for (long j = 0; j < im.cols(); ++j) px[size_t(i) * size_t(im.cols()) + size_t(j)] = im(i, j);
    const int N = cfg.hr_size();
    std::vector<float> out(size_t(N) * N * 2);
    const auto cc = cfg.c();
    detail::check(fpmgpu_init_canvas(detail::ctx(), &cc, px.data(), int(im.rows()), int(im.cols()), im.cols(), tile.x0,
                                     tile.y0, out.data()));
    SpectrumCanvas c;
    c.cfg = cfg;
    c.spectrum = detail::from_c64(out.data(), N, N);
    return c;
}

inline ComplexField canvas_to_field(const SpectrumCanvas& canvas, int fft_threads = 1) {
    (void)fft_threads;
    const auto in = detail::to_c64(canvas.spectrum);
    std::vector<float> out(in.size());
    const auto cc = canvas.cfg.c();
    detail::check(fpmgpu_canvas_to_field(detail::ctx(), &cc, in.data(), out.data()));
    return detail::from_c64(out.data(), canvas.spectrum.rows(), canvas.spectrum.cols());
}

inline double update_step(SpectrumCanvas& canvas, const RealField& intensity, const WaveVector& wv, const Pupil& pupil,
                          int fft_threads = 1) {
    (void)fft_threads;
    const int n = pupil.grid;
    if (intensity.rows() != n || intensity.cols() != n) throw DataError("frame side must equal pupil grid");
    std::vector<float> cv = detail::to_c64(canvas.spectrum), P = detail::to_c64(pupil.values), I(size_t(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) I[size_t(i) * n + j] = float(intensity(i, j));
    double res = 0.0;
    const auto cc = canvas.cfg.c();
    detail::check(fpmgpu_update_step(detail::ctx(), &cc, cv.data(), I.data(), wv.fx, wv.fy, P.data(), FPMGPU_MODE_GS,
                                     1.0, 0.0, &res));
    canvas.spectrum = detail::from_c64(cv.data(), canvas.spectrum.rows(), canvas.spectrum.cols());
    canvas.updated_offsets.push_back(spectrum_offset_px(wv, canvas.cfg));
    return res;
}

inline double update_step(SpectrumCanvas& canvas, const IntensityImage& frame, const WaveVector& wv, const Pupil& pupil,
                          int fft_threads = 1) {
    RealField r = RealField::Zero(frame.rows(), frame.cols());
    for (long i = 0; i < frame.rows(); ++i)
        for (long j = 0; j < frame.cols(); ++j) r(i, j) = double(frame(i, j));
    return update_step(canvas, r, wv, pupil, fft_threads);
}

inline ReconResult reconstruct_tile(const FrameSet& frames, const TileSpec& tile, const OpticalConfig& cfg, int iters,
                                    const LedSequence& seq, int fft_threads = 1) {
    (void)fft_threads;
    auto o = detail::run_batch(frames, {tile}, cfg, iters, seq, 0, false);
    ReconResult r;
    r.hr = detail::from_c64(o.hr.data(), cfg.hr_size(), cfg.hr_size());
    r.metrics.pass_mean_residual = o.residuals;
    return r;
}

// ------------------------------------------------------------------ parallel (parallel.hpp:19-91)
struct PipelineSchedule {
    int lag = 1;
    int stages = 1;
    struct Entry {
        int stage;
        int position;
    };
    std::vector<std::vector<Entry>> rounds;
};

inline int min_safe_lag(const std::vector<std::pair<int, int>>& offsets_px, double radius_px) {
    std::vector<int> o;
    for (auto [a, b] : offsets_px) {
        o.push_back(a);
        o.push_back(b);
    }
    int out = 0;
    detail::check(fpmgpu_min_safe_lag(o.data(), int(offsets_px.size()), radius_px, &out));
    return out;
}

inline int min_safe_lag(const LedSequence& seq, const TileSpec& tile, const OpticalConfig& cfg) {
    std::vector<std::pair<int, int>> o;
    for (const auto& led : seq) o.push_back(spectrum_offset_px(tile.wavevectors.at(led), cfg));
    return min_safe_lag(o, build_pupil(cfg, cfg.tile_size, tile.defocus_um).radius_px);
}

inline PipelineSchedule build_schedule(int positions, int iters, int lag) {
    std::vector<int> e(size_t(positions > 0 ? positions : 1) * size_t(iters > 0 ? iters : 1) * 3);
    int rounds = 0;
    detail::check(fpmgpu_build_schedule(positions, iters, lag, e.data(), &rounds));
    PipelineSchedule s;
    s.lag = lag;
    s.stages = iters;
    s.rounds.resize(size_t(rounds));
    for (size_t q = 0; q < size_t(positions) * size_t(iters); ++q)
        s.rounds[size_t(e[3 * q])].push_back({e[3 * q + 1], e[3 * q + 2]});
    return s;
}

struct PipelineResult {
    ComplexField hr;
    ReconMetrics metrics;
    int lag = 1;
    bool nondeterministic = false;
};

inline PipelineResult pipelined_reconstruct_tile(const FrameSet& frames, const TileSpec& tile, const OpticalConfig& cfg,
                                                 int iters, const LedSequence& seq, std::optional<int> lag = std::nullopt,
                                                 bool force_unsafe = false) {
    if (iters < 1) throw ConfigError("iters must be >= 1");
    const int min_lag = min_safe_lag(seq, tile, cfg);
    const int use = lag.value_or(min_lag);
    if (use < min_lag && !force_unsafe) throw UnsafeLagError(min_lag);
    auto o = detail::run_batch(frames, {tile}, cfg, iters, seq, use, force_unsafe);
    PipelineResult r;
    r.hr = detail::from_c64(o.hr.data(), cfg.hr_size(), cfg.hr_size());
    r.metrics.pass_mean_residual = o.residuals;
    r.lag = use;
    r.nondeterministic = use < min_lag;
    return r;
}

struct TimingRow {
    std::string run_id;
    std::string mode;
    int workers = 1;
    int lag = 1;
    int tiles = 1;
    int iters = 1;
    double wall_s = 0.0;
    double per_tile_mean_s = 0.0;
};

inline std::string timing_csv_header() { return "run_id,mode,workers,lag,tiles,iters,wall_s,per_tile_mean_s"; }
inline std::string timing_csv_row(const TimingRow& r) {
    std::ostringstream os;
    os << r.run_id << ',' << r.mode << ',' << r.workers << ',' << r.lag << ',' << r.tiles << ',' << r.iters << ','
       << r.wall_s << ',' << r.per_tile_mean_s;
    return os.str();
}

struct RunResult {
    std::vector<TileSpec> specs;
    std::vector<ComplexField> tiles;
    ComplexField stitched;
    TimingRow timing;
    std::vector<ReconMetrics> tile_metrics;
    double acquisition_s = 0.0;
};

struct RunOptions {
    int iters = 5;
    int workers = 1;
    std::optional<int> lag;
    bool force_unsafe_lag = false;
    bool force_pipeline = false;
    double defocus_um = 0.0;
    std::optional<int> max_tiles;
    // B200 extensions (BASELINE configs 3-5): reconstruction mode and per-tile defocus
    int mode = FPMGPU_MODE_GS;
    double alpha = 1.0, beta = 1.0;
    std::vector<double> tile_defocus_um;
};

inline ComplexField stitch_mosaic(const std::vector<ComplexField>& tiles, const std::vector<TileSpec>& specs,
                                  const OpticalConfig& cfg) {
    if (tiles.size() != specs.size() || tiles.empty()) throw DataError("stitch_mosaic: tile/spec count mismatch");
    std::vector<int> xy;
    std::vector<float> px;
    for (size_t t = 0; t < tiles.size(); ++t) {
        xy.push_back(specs[t].x0);
        xy.push_back(specs[t].y0);
        const auto v = detail::to_c64(tiles[t]);
        px.insert(px.end(), v.begin(), v.end());
    }
    int rows = 0, cols = 0;
    const auto cc = cfg.c();
    detail::check(fpmgpu_stitch_mosaic(detail::ctx(), &cc, px.data(), xy.data(), int(tiles.size()), nullptr, &rows, &cols));
    std::vector<float> out(size_t(rows) * size_t(cols) * 2);
    detail::check(fpmgpu_stitch_mosaic(detail::ctx(), &cc, px.data(), xy.data(), int(tiles.size()), out.data(), &rows,
                                       &cols));
    return detail::from_c64(out.data(), rows, cols);
}

// All tiles of the FOV in one batched launch (one CTA per tile), then the mosaic.
inline RunResult run_offline(const FrameSet& frames, const OpticalConfig& cfg, const LedSequence& seq,
                             const RunOptions& opt) {
    if (opt.workers < 1) throw ConfigError("workers must be >= 1");
    RunResult res;
    res.specs = partition_tiles(frames.width(), frames.height(), cfg, opt.defocus_um);
    if (opt.max_tiles) {
        if (*opt.max_tiles > int(res.specs.size())) throw ConfigError("requested tile count exceeds partition");
        res.specs.resize(size_t(*opt.max_tiles));
    }
    if (!opt.tile_defocus_um.empty()) {
        if (opt.tile_defocus_um.size() != res.specs.size())
            throw ConfigError("tile_defocus_um must list one value per tile");
        for (size_t i = 0; i < res.specs.size(); ++i) res.specs[i].defocus_um = opt.tile_defocus_um[i];
    }
    const bool pipeline = opt.force_pipeline || opt.workers > int(res.specs.size());
    if (pipeline && opt.mode != FPMGPU_MODE_GS) throw ConfigError("pipelined schedule requires Gerchberg-Saxton mode");
    auto o = detail::run_batch(frames, res.specs, cfg, opt.iters, seq, pipeline ? opt.lag.value_or(-1) : 0,
                               opt.force_unsafe_lag, opt.mode, opt.alpha, opt.beta);
    const size_t N = size_t(cfg.hr_size());
    for (size_t t = 0; t < res.specs.size(); ++t) {
        res.tiles.push_back(detail::from_c64(o.hr.data() + t * N * N * 2, long(N), long(N)));
        ReconMetrics m;
        m.pass_mean_residual.assign(o.residuals.begin() + long(t) * opt.iters,
                                    o.residuals.begin() + long(t + 1) * opt.iters);
        res.tile_metrics.push_back(m);
    }
    if (!opt.max_tiles) res.stitched = stitch_mosaic(res.tiles, res.specs, cfg);
    res.timing.mode = "offline";
    res.timing.workers = opt.workers;
    res.timing.lag = opt.lag.value_or(1);
    res.timing.tiles = int(res.specs.size());
    res.timing.iters = opt.iters;
    return res;
}

// run_online (parallel.cpp:198-317): frames replayed against their timestamps
// (x delay_scale); each arrival goes to the device and the first-pass update
// of every newly complete sequence position runs on all tiles
// (fpmgpu_online_push); the remaining passes, HR fields and mosaic follow.
inline RunResult run_online(const FrameSet& frames, const OpticalConfig& cfg, const LedSequence& seq,
                            const RunOptions& opt, double delay_scale = 1.0) {
    if (opt.workers < 1) throw ConfigError("workers must be >= 1");
    if (delay_scale < 0) throw ConfigError("delay scale must be >= 0");
    const auto t0 = std::chrono::steady_clock::now();
    RunResult res;
    res.specs = partition_tiles(frames.width(), frames.height(), cfg, opt.defocus_um);
    if (opt.max_tiles) {
        if (*opt.max_tiles > int(res.specs.size())) throw ConfigError("requested tile count exceeds partition");
        res.specs.resize(size_t(*opt.max_tiles));
    }
    if (!opt.tile_defocus_um.empty()) {
        if (opt.tile_defocus_um.size() != res.specs.size())
            throw ConfigError("tile_defocus_um must list one value per tile");
        for (size_t i = 0; i < res.specs.size(); ++i) res.specs[i].defocus_um = opt.tile_defocus_um[i];
    }
    std::vector<int> stream;
    for (const auto& led : seq) {
        int idx = -1;
        for (size_t f = 0; f < frames.frames.size() && idx < 0; ++f)
            if (frames.frames[f].led == led) idx = int(f);
        if (idx < 0) throw DataError("missing frame for a sequence LED");
        stream.push_back(idx);
    }
    detail::Batch b = detail::make_batch(frames, res.specs, cfg, seq);
    const std::vector<uint16_t> px = detail::pack_frames(frames);
    fpmgpu_recon_request r{};
    r.cfg = cfg.c();
    r.iters = opt.iters;
    r.mode = opt.mode;
    r.alpha = opt.alpha;
    r.beta = opt.beta;
    r.num_tiles = int(res.specs.size());
    r.tile_xy = b.xy.data();
    r.num_leds = int(seq.size());
    r.offsets = b.offsets.data();
    r.seq_frame = b.seq_frame.data();
    r.init_frame = detail::seed_frame(frames, cfg);
    bool any_defocus = false;
    for (double z : b.defocus) any_defocus |= z != 0.0;
    r.tile_defocus_um = any_defocus ? b.defocus.data() : nullptr;
    r.num_frames = int(frames.frames.size());
    r.height = frames.height();
    r.width = frames.width();
    const size_t N = size_t(cfg.hr_size()), T = res.specs.size();
    const size_t frame_px = size_t(r.height) * size_t(r.width);
    std::vector<float> hr(T * N * N * 2);
    std::vector<double> resid(T * size_t(opt.iters));
    fpmgpu_online* on = nullptr;
    detail::check(fpmgpu_online_begin(detail::ctx(), &r, &on));
    try {
        std::vector<char> pushed(frames.frames.size(), 0);
        for (int f : stream) {  // the ordered frame source (parallel.cpp:220-233)
            std::this_thread::sleep_until(t0 + std::chrono::duration<double>(frames.frames[size_t(f)].timestamp_s *
                                                                             delay_scale));
            if (pushed[size_t(f)]) continue;
            pushed[size_t(f)] = 1;
            detail::check(fpmgpu_online_push(on, f, px.data() + size_t(f) * frame_px, r.width, nullptr));
        }
        if (!pushed[size_t(r.init_frame)])
            detail::check(fpmgpu_online_push(on, r.init_frame, px.data() + size_t(r.init_frame) * frame_px, r.width,
                                             nullptr));
        detail::check(fpmgpu_online_finish(on, hr.data(), resid.data(), nullptr));
    } catch (...) {
        fpmgpu_online_destroy(on);
        throw;
    }
    fpmgpu_online_destroy(on);
    res.acquisition_s = stream.empty() ? 0.0 : frames.frames[size_t(stream.back())].timestamp_s * delay_scale;
    for (size_t t = 0; t < T; ++t) {
        res.tiles.push_back(detail::from_c64(hr.data() + t * N * N * 2, long(N), long(N)));
        ReconMetrics m;
        m.pass_mean_residual.assign(resid.begin() + long(t) * opt.iters, resid.begin() + long(t + 1) * opt.iters);
        res.tile_metrics.push_back(m);
    }
    if (!opt.max_tiles) res.stitched = stitch_mosaic(res.tiles, res.specs, cfg);
    res.timing.mode = "online";
    res.timing.workers = opt.workers;
    res.timing.lag = 1;
    res.timing.tiles = int(T);
    res.timing.iters = opt.iters;
    res.timing.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    res.timing.per_tile_mean_s = T ? res.timing.wall_s / double(T) : 0.0;
    return res;
}

}  // namespace fpm
