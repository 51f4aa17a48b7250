// extern "C" surface of the oracle for ctypes (tests/, smoke(), bench.py's CPU
// legs only). Complex arrays are interleaved (re, im) double, row-major.
// Status codes: 0 ok, 1 ConfigError, 2 DataError, 3 UnsafeLagError, 4 domain
// error, 6 other. Message via orc_last_error().
#include <cstring>
#include <string>

#include "fpm_oracle.hpp"

using namespace orc;

namespace {

thread_local std::string g_err;
thread_local int g_min_lag = 0;

extern "C" struct orc_config {
    double wavelength, objective_na, magnification, camera_pixel, led_pitch;
    int led_grid_rows, led_grid_cols;
    double led_height;
    int center_row, center_col, led_scan_rows, led_scan_cols, upsample, tile_size, tile_overlap;
    double acq_pattern_delay, acq_exposure;
};

Optics to_optics(const orc_config* c) {
    Optics o;
    o.wavelength = c->wavelength;
    o.objective_na = c->objective_na;
    o.magnification = c->magnification;
    o.camera_pixel = c->camera_pixel;
    o.led_pitch = c->led_pitch;
    o.led_grid_rows = c->led_grid_rows;
    o.led_grid_cols = c->led_grid_cols;
    o.led_height = c->led_height;
    o.center_led = {c->center_row, c->center_col};
    o.led_scan_rows = c->led_scan_rows;
    o.led_scan_cols = c->led_scan_cols;
    o.upsample = c->upsample;
    o.tile_size = c->tile_size;
    o.tile_overlap = c->tile_overlap;
    o.acq_pattern_delay = c->acq_pattern_delay;
    o.acq_exposure = c->acq_exposure;
    return o;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const UnsafeLagError& e) {
        g_err = e.what();
        g_min_lag = e.minimum;
        return 3;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

CGrid load_c(const double* p, int rows, int cols) {
    CGrid g(rows, cols);
    std::memcpy(static_cast<void*>(g.v.data()), p, sizeof(cplx) * g.size());
    return g;
}
void store_c(const CGrid& g, double* p) { std::memcpy(p, g.v.data(), sizeof(cplx) * g.size()); }
RGrid load_r(const double* p, int rows, int cols) {
    RGrid g(rows, cols);
    std::memcpy(g.v.data(), p, sizeof(double) * g.size());
    return g;
}

Sequence load_seq(const int* rc, int n) {
    Sequence s;
    for (int i = 0; i < n; ++i) s.push_back({rc[2 * i], rc[2 * i + 1]});
    return s;
}

FrameStack load_frames(const orc_config* cfg, const uint16_t* px, const int* leds, const double* ts,
                       int F, int H, int W) {
    FrameStack fs;
    fs.cfg = to_optics(cfg);
    for (int f = 0; f < F; ++f) {
        LrFrame fr;
        fr.led = {leds[2 * f], leds[2 * f + 1]};
        fr.image = U16Grid(H, W);
        std::memcpy(fr.image.v.data(), px + size_t(f) * H * W, sizeof(uint16_t) * size_t(H) * W);
        fr.timestamp_s = ts ? ts[f] : 0.0;
        fs.frames.push_back(std::move(fr));
    }
    return fs;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_last_min_lag() { return g_min_lag; }

int orc_validate(const orc_config* c) { return guarded([&] { to_optics(c).validate(); }); }

int orc_fft2(const double* in, int rows, int cols, int inverse, int threads, double* out) {
    return guarded([&] {
        CGrid x = load_c(in, rows, cols);
        store_c(inverse ? ifft2(x, threads) : fft2(x, threads), out);
    });
}
int orc_fftshift(const double* in, int rows, int cols, int inverse, double* out) {
    return guarded([&] {
        CGrid x = load_c(in, rows, cols);
        store_c(inverse ? ifftshift(x) : fftshift(x), out);
    });
}
int orc_upsample_bilinear(const double* in, int rows, int cols, int factor, double* out) {
    return guarded([&] {
        RGrid r = upsample_bilinear(load_r(in, rows, cols), factor);
        std::memcpy(out, r.v.data(), sizeof(double) * r.size());
    });
}

int orc_illumination_wavevector(const orc_config* c, int row, int col, double cx, double cy,
                                double* fx, double* fy) {
    return guarded([&] {
        KVec k = illumination_wavevector({row, col}, {cx, cy}, to_optics(c));
        *fx = k.fx;
        *fy = k.fy;
    });
}
int orc_build_pupil(const orc_config* c, int grid, double defocus, double* values, double* radius) {
    return guarded([&] {
        PupilFn p = build_pupil(to_optics(c), grid, defocus);
        if (values) store_c(p.values, values);
        if (radius) *radius = p.radius_px;
    });
}
int orc_synthesized_na(const orc_config* c, double* out) {
    return guarded([&] { *out = synthesized_na(to_optics(c)); });
}
int orc_tile_origins(int fov, int tile, int overlap, int* out, int cap, int* count) {
    return guarded([&] {
        auto v = tile_origins(fov, tile, overlap);
        *count = int(v.size());
        for (int i = 0; i < int(v.size()) && i < cap; ++i) out[i] = v[size_t(i)];
    });
}
// Tiles: out_xy [T][2] (x0, y0); out_center [T][2] (cx, cy um); kvecs [T][L][2] (fx, fy) in
// led_sequence(seq) order; offsets [T][L][2] (oy, ox).
int orc_partition_tiles(const orc_config* c, int fov_w, int fov_h, const int* seq, int L, int cap,
                        int* count, int* out_xy, double* out_center, double* kvecs, int* offsets) {
    return guarded([&] {
        Optics o = to_optics(c);
        auto tiles = partition_tiles(fov_w, fov_h, o);
        Sequence s = load_seq(seq, L);
        *count = int(tiles.size());
        for (int t = 0; t < int(tiles.size()) && t < cap; ++t) {
            const Tile& tl = tiles[size_t(t)];
            if (out_xy) {
                out_xy[2 * t] = tl.x0;
                out_xy[2 * t + 1] = tl.y0;
            }
            if (out_center) {
                out_center[2 * t] = tl.center_x_um;
                out_center[2 * t + 1] = tl.center_y_um;
            }
            for (int k = 0; k < L; ++k) {
                KVec kv = tl.kvecs.at(s[size_t(k)]);
                if (kvecs) {
                    kvecs[(size_t(t) * L + k) * 2] = kv.fx;
                    kvecs[(size_t(t) * L + k) * 2 + 1] = kv.fy;
                }
                if (offsets) {
                    auto [oy, ox] = spectrum_offset_px(kv, o);
                    offsets[(size_t(t) * L + k) * 2] = oy;
                    offsets[(size_t(t) * L + k) * 2 + 1] = ox;
                }
            }
        }
    });
}
int orc_sequence_offsets(int order, int rows, int cols, int* out) {
    return guarded([&] {
        auto v = sequence_offsets(order ? Order::Raster : Order::Spiral, rows, cols);
        for (size_t i = 0; i < v.size(); ++i) {
            out[2 * i] = v[i].first;
            out[2 * i + 1] = v[i].second;
        }
    });
}
int orc_spectrum_offset_px(const orc_config* c, double fx, double fy, int* oy, int* ox) {
    return guarded([&] {
        auto p = spectrum_offset_px({fx, fy}, to_optics(c));
        *oy = p.first;
        *ox = p.second;
    });
}
int orc_min_safe_lag(const int* offs, int count, double radius, int* out) {
    return guarded([&] {
        std::vector<std::pair<int, int>> v;
        for (int i = 0; i < count; ++i) v.emplace_back(offs[2 * i], offs[2 * i + 1]);
        *out = min_safe_lag(v, radius);
    });
}
int orc_min_safe_lag_tile(const orc_config* c, int fov_w, int fov_h, int tile_index, const int* seq,
                          int L, int* out) {
    return guarded([&] {
        Optics o = to_optics(c);
        auto tiles = partition_tiles(fov_w, fov_h, o);
        *out = min_safe_lag(load_seq(seq, L), tiles.at(size_t(tile_index)), o);
    });
}
// entries [positions*iters][3] = (round, stage, position); *rounds = round count
int orc_build_schedule(int positions, int iters, int lag, int* entries, int* rounds) {
    return guarded([&] {
        Schedule s = build_schedule(positions, iters, lag);
        *rounds = int(s.rounds.size());
        size_t q = 0;
        for (size_t r = 0; r < s.rounds.size(); ++r)
            for (const auto& e : s.rounds[r]) {
                entries[3 * q] = int(r);
                entries[3 * q + 1] = e.stage;
                entries[3 * q + 2] = e.position;
                ++q;
            }
    });
}

int orc_synth_object(int kind, int size, unsigned long long seed, double* out) {
    return guarded([&] { store_c(synth_object(ObjectKind(kind), size, seed), out); });
}
int orc_simulate_intensity(const double* obj, const orc_config* c, double fx, double fy,
                           double defocus, double* out) {
    return guarded([&] {
        Optics o = to_optics(c);
        CGrid ob = load_c(obj, o.hr_size(), o.hr_size());
        RGrid r = simulate_intensity(ob, {fx, fy}, build_pupil(o, o.tile_size, defocus), o);
        std::memcpy(out, r.v.data(), sizeof(double) * r.size());
    });
}
// frames out: [L][H][W] u16 with H = rows/upsample, W = cols/upsample; ts out [L]
int orc_simulate_dataset(const double* obj, int rows, int cols, const orc_config* c, const int* seq,
                         int L, int noise_enabled, double photons, unsigned long long noise_seed,
                         double defocus, uint16_t* frames, double* ts) {
    return guarded([&] {
        Optics o = to_optics(c);
        CGrid ob = load_c(obj, rows, cols);
        Noise nz{noise_enabled != 0, photons, noise_seed};
        FrameStack fs = simulate_dataset(ob, load_seq(seq, L), o, nz, defocus);
        const size_t plane = size_t(fs.height()) * fs.width();
        for (int f = 0; f < L; ++f) {
            std::memcpy(frames + plane * f, fs.frames[size_t(f)].image.v.data(), plane * sizeof(uint16_t));
            if (ts) ts[f] = fs.frames[size_t(f)].timestamp_s;
        }
    });
}

int orc_init_canvas(const orc_config* c, const uint16_t* px, const int* leds, int F, int H, int W,
                    int tile_index, double* canvas) {
    return guarded([&] {
        FrameStack fs = load_frames(c, px, leds, nullptr, F, H, W);
        auto tiles = partition_tiles(W, H, fs.cfg);
        store_c(init_canvas(fs, tiles.at(size_t(tile_index)), fs.cfg).spectrum, canvas);
    });
}
int orc_canvas_to_field(const orc_config* c, const double* canvas, double* out) {
    return guarded([&] {
        Canvas cv;
        cv.cfg = to_optics(c);
        cv.spectrum = load_c(canvas, cv.cfg.hr_size(), cv.cfg.hr_size());
        store_c(canvas_to_field(cv), out);
    });
}

// One GS step on a caller-owned canvas (N x N). pupil n x n complex.
int orc_update_step(const orc_config* c, double* canvas, const double* intensity, double fx,
                    double fy, const double* pupil, double* residual) {
    return guarded([&] {
        Canvas cv;
        cv.cfg = to_optics(c);
        const int N = cv.cfg.hr_size(), n = cv.cfg.tile_size;
        cv.spectrum = load_c(canvas, N, N);
        PupilFn p;
        p.grid = n;
        p.values = load_c(pupil, n, n);
        *residual = update_step(cv, load_r(intensity, n, n), {fx, fy}, p);
        store_c(cv.spectrum, canvas);
    });
}
// One EPRY step: canvas and pupil updated in place; support = pupil != 0 on entry
// unless `support` (n x n u8) is given.
int orc_update_step_epry(const orc_config* c, double* canvas, const double* intensity, double fx,
                         double fy, double* pupil, const uint8_t* support, double alpha,
                         double beta, double* residual) {
    return guarded([&] {
        Canvas cv;
        cv.cfg = to_optics(c);
        const int N = cv.cfg.hr_size(), n = cv.cfg.tile_size;
        cv.spectrum = load_c(canvas, N, N);
        CGrid P = load_c(pupil, n, n);
        Grid<uint8_t> S(n, n, 0);
        for (size_t i = 0; i < S.size(); ++i) S.v[i] = support ? support[i] : (P.v[i] != cplx(0, 0));
        const double radius = build_pupil(cv.cfg, n, 0.0).radius_px;
        *residual = update_step_epry(cv, load_r(intensity, n, n), {fx, fy}, P, S, alpha, beta, radius);
        store_c(cv.spectrum, canvas);
        store_c(P, pupil);
    });
}

// reconstruct_tile / pipelined_reconstruct_tile on partition_tiles(W, H)[tile_index].
// lag < 0 with pipelined = auto. hr [N][N] complex, resid [iters], pupil_out [n][n] complex.
int orc_reconstruct_tile(const orc_config* c, const uint16_t* px, const int* leds, int F, int H,
                         int W, int tile_index, double tile_defocus, int iters, const int* seq,
                         int L, int mode, double alpha, double beta, int fft_threads,
                         int pipelined, int lag, int force_unsafe, double* hr, double* resid,
                         double* pupil_out, int* lag_out, int* nondet_out, double* wall_s) {
    return guarded([&] {
        FrameStack fs = load_frames(c, px, leds, nullptr, F, H, W);
        auto tiles = partition_tiles(W, H, fs.cfg, tile_defocus);
        const Tile& t = tiles.at(size_t(tile_index));
        Sequence s = load_seq(seq, L);
        TileResult r;
        if (pipelined) {
            if (mode != 0) throw ConfigError("pipelined schedule requires Gerchberg-Saxton mode");
            r = pipelined_reconstruct_tile(fs, t, fs.cfg, iters, s,
                                           lag < 0 ? std::nullopt : std::optional<int>(lag),
                                           force_unsafe != 0);
        } else {
            r = reconstruct_tile(fs, t, fs.cfg, iters, s, fft_threads, Mode(mode), {alpha, beta});
        }
        if (hr) store_c(r.hr, hr);
        if (resid)
            for (size_t i = 0; i < r.pass_mean_residual.size(); ++i) resid[i] = r.pass_mean_residual[i];
        if (pupil_out) store_c(r.pupil, pupil_out);
        if (lag_out) *lag_out = r.lag;
        if (nondet_out) *nondet_out = r.nondeterministic;
        if (wall_s) *wall_s = r.wall_s;
    });
}

// run_offline. tiles_out [T][N][N] complex or NULL; stitched [H*up][W*up] or NULL;
// resid [T][iters] or NULL; tile_defocus [T] or NULL; max_tiles < 0 = all; lag < 0 = auto.
int orc_run_offline(const orc_config* c, const uint16_t* px, const int* leds, int F, int H, int W,
                    const int* seq, int L, int iters, int workers, int lag, int force_unsafe,
                    int force_pipeline, double defocus, int max_tiles, const double* tile_defocus,
                    int n_tile_defocus, int mode, double alpha, double beta, double* tiles_out,
                    double* stitched, double* resid, int* tile_count, double* wall_s) {
    return guarded([&] {
        FrameStack fs = load_frames(c, px, leds, nullptr, F, H, W);
        OfflineOptions opt;
        opt.iters = iters;
        opt.workers = workers;
        if (lag >= 0) opt.lag = lag;
        opt.force_unsafe_lag = force_unsafe != 0;
        opt.force_pipeline = force_pipeline != 0;
        opt.defocus_um = defocus;
        if (max_tiles >= 0) opt.max_tiles = max_tiles;
        if (tile_defocus) opt.tile_defocus_um.assign(tile_defocus, tile_defocus + n_tile_defocus);
        opt.mode = Mode(mode);
        opt.epry = {alpha, beta};
        OfflineResult r = run_offline(fs, fs.cfg, load_seq(seq, L), opt);
        if (tile_count) *tile_count = int(r.tiles.size());
        const size_t plane = r.tiles.empty() ? 0 : r.tiles[0].size();
        for (size_t t = 0; t < r.tiles.size(); ++t) {
            if (tiles_out) std::memcpy(tiles_out + 2 * plane * t, r.tiles[t].v.data(), sizeof(cplx) * plane);
            if (resid)
                for (int i = 0; i < iters; ++i) resid[t * size_t(iters) + size_t(i)] = r.residuals[t][size_t(i)];
        }
        if (stitched && r.stitched.size()) store_c(r.stitched, stitched);
        if (wall_s) *wall_s = r.wall_s;
    });
}

int orc_mean_ratio(const double* f1, int r1, int c1, const double* f2, int r2, int c2, int overlap,
                   int vertical, double* out) {
    return guarded([&] {
        cplx m = mean_ratio(load_c(f1, r1, c1), load_c(f2, r2, c2), overlap,
                            vertical ? Axis::Vertical : Axis::Horizontal);
        out[0] = m.real();
        out[1] = m.imag();
    });
}
int orc_stitch_pair(const double* f1, int r1, int c1, const double* f2, int r2, int c2, int overlap,
                    int vertical, double* out, int* rows, int* cols) {
    return guarded([&] {
        CGrid s = stitch_pair(load_c(f1, r1, c1), load_c(f2, r2, c2), overlap,
                              vertical ? Axis::Vertical : Axis::Horizontal);
        *rows = s.rows;
        *cols = s.cols;
        if (out) store_c(s, out);
    });
}
// tiles [T][N][N] complex (N = tile_size*upsample), xy [T][2] origins (x0, y0)
int orc_stitch_mosaic(const orc_config* c, const double* tiles, const int* xy, int T, double* out,
                      int* rows, int* cols) {
    return guarded([&] {
        Optics o = to_optics(c);
        const int N = o.hr_size();
        std::vector<CGrid> tl;
        std::vector<Tile> specs;
        for (int t = 0; t < T; ++t) {
            tl.push_back(load_c(tiles + 2 * size_t(N) * N * t, N, N));
            Tile s;
            s.x0 = xy[2 * t];
            s.y0 = xy[2 * t + 1];
            s.size = o.tile_size;
            specs.push_back(s);
        }
        CGrid m = stitch_mosaic(tl, specs, o);
        *rows = m.rows;
        *cols = m.cols;
        if (out) store_c(m, out);
    });
}

int orc_band_limit(const double* field, int n, double na, const orc_config* c, double* out) {
    return guarded([&] { store_c(band_limit(load_c(field, n, n), na, to_optics(c)), out); });
}
int orc_global_alignment(const double* recon, const double* truth, int rows, int cols, double* out) {
    return guarded([&] {
        cplx g = global_alignment(load_c(recon, rows, cols), load_c(truth, rows, cols));
        out[0] = g.real();
        out[1] = g.imag();
    });
}
int orc_rmse(const double* a, const double* b, int rows, int cols, double* amp, double* phase) {
    return guarded([&] {
        CGrid A = load_c(a, rows, cols), B = load_c(b, rows, cols);
        *amp = amplitude_rmse(A, B);
        *phase = phase_rmse(A, B);
    });
}

}  // extern "C"
