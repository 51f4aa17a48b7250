// fpm_oracle — CPU double restatement of the reference FPM path. TEST
// INFRASTRUCTURE ONLY (see fpm_oracle.hpp). Each function cites the reference
// file:line (under /root/reference/proj) whose behaviour it restates.
#include "fpm_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <functional>
#include <mutex>
#include <random>
#include <thread>
#include <unordered_map>

namespace orc {

namespace {
constexpr double kPi = 3.14159265358979323846;
double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

// =============================================================== 1-D DFT
// Mixed-radix decimation-in-time DFT with a per-(n, direction) plan. The
// reference delegates to Eigen's kissfft backend (field.cpp:7, :22-31), whose
// bits are not pinned by any reference test (test_field.cpp pins only DC,
// round trip <= 1e-12, Parseval, linearity); any accurate DFT with the same
// sign/scale conventions is a valid restatement. Radices 4, 2, 3, 5 first,
// remaining prime factors by direct summation.
namespace {

struct DftPlan {
    int n = 0;
    std::vector<int> radix;
    std::vector<cplx> w;  // w[k] = exp(-+2 pi i k / n)
};

DftPlan make_plan(int n, bool inverse) {
    DftPlan p;
    p.n = n;
    int m = n;
    for (int r : {4, 2, 3, 5}) {
        while (m % r == 0 && m > 1) {
            p.radix.push_back(r);
            m /= r;
        }
    }
    for (int r = 7; m > 1; r += 2) {
        while (m % r == 0) {
            p.radix.push_back(r);
            m /= r;
        }
    }
    if (p.radix.empty()) p.radix.push_back(1);
    p.w.resize(size_t(n));
    const double sgn = inverse ? 1.0 : -1.0;
    for (int k = 0; k < n; ++k) {
        const double a = sgn * 2.0 * kPi * double(k) / double(n);
        p.w[size_t(k)] = cplx(std::cos(a), std::sin(a));
    }
    return p;
}

const DftPlan& plan_for(int n, bool inverse) {
    thread_local std::unordered_map<long long, DftPlan> cache;
    const long long key = (long long)n * 2 + (inverse ? 1 : 0);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, make_plan(n, inverse)).first;
    return it->second;
}

// out[0..len) = DFT_len of in[0], in[s], ..., in[(len-1) s]; `level` indexes
// the plan's radix list, `wstep` = plan.n / len.
void dft_rec(const DftPlan& P, cplx* out, const cplx* in, int len, long s, int wstep,
             size_t level) {
    const int r = P.radix[level];
    const int m = len / r;
    if (m == 1) {
        for (int q = 0; q < r; ++q) out[q] = in[q * s];
    } else {
        for (int q = 0; q < r; ++q) dft_rec(P, out + q * m, in + q * s, m, s * r, wstep * r, level + 1);
    }
    if (r == 1) return;
    const int N = P.n;
    // combine r sub-transforms Y_q (length m): X[k + m u] = sum_q W_len^{qk} Y_q[k] W_r^{qu}
    if (r == 2) {
        for (int k = 0; k < m; ++k) {
            const cplx a = out[k];
            const cplx b = out[k + m] * P.w[size_t(k) * wstep];
            out[k] = a + b;
            out[k + m] = a - b;
        }
        return;
    }
    if (r == 4) {
        // W_4 = -i (forward) or +i (inverse); read from the table to keep the sign rule in one place
        const cplx j4 = P.w[size_t(N / 4)];
        for (int k = 0; k < m; ++k) {
            const cplx y0 = out[k];
            const cplx y1 = out[k + m] * P.w[size_t(k) * wstep];
            const cplx y2 = out[k + 2 * m] * P.w[size_t(2 * k) * wstep];
            const cplx y3 = out[k + 3 * m] * P.w[size_t(3 * k) * wstep];
            const cplx s02 = y0 + y2, d02 = y0 - y2;
            const cplx s13 = y1 + y3, d13 = (y1 - y3) * j4;
            out[k] = s02 + s13;
            out[k + m] = d02 + d13;
            out[k + 2 * m] = s02 - s13;
            out[k + 3 * m] = d02 - d13;
        }
        return;
    }
    thread_local std::vector<cplx> t;
    t.resize(size_t(r));
    const long rstep = N / r;  // W_r = w[N/r]
    for (int k = 0; k < m; ++k) {
        for (int q = 0; q < r; ++q)
            t[size_t(q)] = out[k + q * m] * P.w[(size_t(q) * size_t(k) * size_t(wstep)) % size_t(N)];
        for (int u = 0; u < r; ++u) {
            cplx acc = 0.0;
            for (int q = 0; q < r; ++q) acc += t[size_t(q)] * P.w[size_t((long(q) * u % r) * rstep)];
            out[k + u * m] = acc;
        }
    }
}

}  // namespace

void dft1d(cplx* data, int n, int stride, bool inverse) {
    if (n <= 1) return;
    const DftPlan& P = plan_for(n, inverse);
    thread_local std::vector<cplx> buf;
    buf.resize(size_t(n));
    dft_rec(P, buf.data(), data, n, stride, 1, 0);
    for (int k = 0; k < n; ++k) data[long(k) * stride] = buf[size_t(k)];
}

// =============================================================== field.cpp
namespace {

// Runs 1-D transforms over every column (axis 0) or row (axis 1), optionally
// split over `threads` workers (field.cpp:18-46 splits columns the same way).
void transform_axis(CGrid& m, int axis, bool inverse, int threads) {
    const int lines = axis == 0 ? m.cols : m.rows;
    const int len = axis == 0 ? m.rows : m.cols;
    const long stride = axis == 0 ? m.cols : 1;
    const long step = axis == 0 ? 1 : m.cols;
    const double scale = inverse ? 1.0 / double(len) : 1.0;  // Eigen FFT inv divides by N
    auto work = [&](int a, int b) {
        for (int l = a; l < b; ++l) {
            cplx* base = m.v.data() + l * step;
            dft1d(base, len, int(stride), inverse);
            if (inverse)
                for (int k = 0; k < len; ++k) base[k * stride] *= scale;
        }
    };
    if (threads <= 1 || lines < 2 * threads) {
        work(0, lines);
        return;
    }
    std::vector<std::thread> pool;
    const int chunk = (lines + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int a = t * chunk, b = std::min(lines, a + chunk);
        if (a >= b) break;
        pool.emplace_back(work, a, b);
    }
    for (auto& th : pool) th.join();
}

CGrid centered_transform(const CGrid& x, bool inverse, int threads) {
    CGrid m = ifftshift(x);  // pixel (rows/2, cols/2) becomes the origin (field.cpp:50)
    transform_axis(m, 0, inverse, threads);
    transform_axis(m, 1, inverse, threads);
    return fftshift(m);
}

CGrid rotate(const CGrid& x, int dr, int dc) {
    CGrid out(x.rows, x.cols);
    for (int i = 0; i < x.rows; ++i)
        for (int j = 0; j < x.cols; ++j) out((i + dr) % x.rows, (j + dc) % x.cols) = x(i, j);
    return out;
}

}  // namespace

CGrid fft2(const CGrid& x, int threads) { return centered_transform(x, false, threads); }
CGrid ifft2(const CGrid& x, int threads) { return centered_transform(x, true, threads); }
CGrid fftshift(const CGrid& x) { return rotate(x, x.rows / 2, x.cols / 2); }
CGrid ifftshift(const CGrid& x) { return rotate(x, (x.rows + 1) / 2, (x.cols + 1) / 2); }

RGrid upsample_bilinear(const RGrid& in, int factor) {
    if (factor < 1) throw std::invalid_argument("upsample factor must be >= 1");
    const int r = in.rows, c = in.cols;
    RGrid out(r * factor, c * factor);
    // pixel-centre mapping back into the input grid, edge-clamped (field.cpp:96-108)
    for (int i = 0; i < out.rows; ++i) {
        const double y = (i + 0.5) / factor - 0.5;
        int ya = int(std::floor(y));
        const double fy = y - ya;
        const int yb = std::min(ya + 1, r - 1);
        ya = std::max(ya, 0);
        for (int j = 0; j < out.cols; ++j) {
            const double x = (j + 0.5) / factor - 0.5;
            int xa = int(std::floor(x));
            const double fx = x - xa;
            const int xb = std::min(xa + 1, c - 1);
            xa = std::max(xa, 0);
            out(i, j) = (1 - fy) * ((1 - fx) * in(ya, xa) + fx * in(ya, xb)) +
                        fy * ((1 - fx) * in(yb, xa) + fx * in(yb, xb));
        }
    }
    return out;
}

// =============================================================== optics.cpp
void Optics::validate() const {
    auto bad = [](const char* what) {
        throw ConfigError(std::string("config invariant violated: ") + what);
    };
    if (!(wavelength > 0)) bad("wavelength > 0");
    if (!(objective_na > 0 && objective_na < 1)) bad("0 < objective_na < 1");
    if (!(magnification > 0)) bad("magnification > 0");
    if (!(camera_pixel > 0)) bad("camera_pixel > 0");
    if (!(led_pitch > 0)) bad("led_pitch > 0");
    if (!(led_height > 0)) bad("led_height > 0");
    if (led_grid_rows < 1 || led_grid_cols < 1) bad("led_grid positive");
    if (led_scan_rows % 2 == 0 || led_scan_cols % 2 == 0) bad("led_scan dimensions odd");
    if (center_led.row - led_scan_rows / 2 < 0 || center_led.row + led_scan_rows / 2 >= led_grid_rows ||
        center_led.col - led_scan_cols / 2 < 0 || center_led.col + led_scan_cols / 2 >= led_grid_cols)
        bad("led_scan fits inside led_grid");
    if (upsample < 2) bad("upsample >= 2");
    if (tile_size < 1) bad("tile_size positive");
    if (!(tile_overlap >= 0 && tile_overlap < tile_size)) bad("tile_overlap < tile_size");
    if (!(acq_pattern_delay >= 0 && acq_exposure >= 0)) bad("acquisition times >= 0");
}

KVec illumination_wavevector(Led led, std::pair<double, double> center_um, const Optics& o) {
    if (led.row < 0 || led.row >= o.led_grid_rows || led.col < 0 || led.col >= o.led_grid_cols)
        throw std::domain_error("LED index (" + std::to_string(led.row) + "," +
                                std::to_string(led.col) + ") outside LED grid");
    // LED position relative to the board centre in micron (optics.cpp:31-33)
    const double pitch = o.led_pitch * 1000.0;
    const double lx = (led.col - o.center_led.col) * pitch;
    const double ly = (led.row - o.center_led.row) * pitch;
    const double h = o.led_height * 1000.0;
    const double ddx = lx - center_um.first;
    const double ddy = ly - center_um.second;
    const double dist = std::sqrt(ddx * ddx + ddy * ddy + h * h);
    return {-ddx / (o.wavelength * dist), -ddy / (o.wavelength * dist)};
}

PupilFn build_pupil(const Optics& o, int grid, double defocus_um) {
    if (grid < 32 || grid % 2 != 0) throw ConfigError("pupil grid must be even and >= 32");
    const double dk = 1.0 / (grid * o.dx_obj());
    const double radius = (o.objective_na / o.wavelength) / dk;
    if (radius >= grid / 2.0)
        throw ConfigError("pupil exceeds Nyquist of LR grid (radius " + std::to_string(radius) +
                          " px, grid " + std::to_string(grid) + ")");
    PupilFn p;
    p.grid = grid;
    p.radius_px = radius;
    p.defocus = defocus_um;
    p.values = CGrid(grid, grid, cplx(0, 0));
    const int c = grid / 2;
    const double inv_l2 = 1.0 / (o.wavelength * o.wavelength);
    for (int i = 0; i < grid; ++i)
        for (int j = 0; j < grid; ++j) {
            const double rho = std::hypot(double(i - c), double(j - c));
            if (rho > radius) continue;  // support rule optics.cpp:59-60
            if (defocus_um == 0.0) {
                p.values(i, j) = cplx(1.0, 0.0);
            } else {  // angular-spectrum defocus phase (optics.cpp:63-67)
                const double f2 = rho * dk * rho * dk;
                const double kz = std::sqrt(std::max(0.0, inv_l2 - f2));
                const double ph = 2.0 * kPi * defocus_um * kz;
                p.values(i, j) = cplx(std::cos(ph), std::sin(ph));
            }
        }
    return p;
}

double synthesized_na(const Optics& o) {
    double best = 0.0;
    const int hr = o.led_scan_rows / 2, hc = o.led_scan_cols / 2;
    for (int dr = -hr; dr <= hr; ++dr)
        for (int dc = -hc; dc <= hc; ++dc) {
            KVec k = illumination_wavevector({o.center_led.row + dr, o.center_led.col + dc}, {0.0, 0.0}, o);
            best = std::max(best, o.wavelength * std::hypot(k.fx, k.fy));
        }
    return o.objective_na + best;
}

// =============================================================== tiles.cpp
std::vector<int> tile_origins(int fov, int tile, int overlap) {
    if (fov < tile) throw ConfigError("FOV smaller than one tile");
    std::vector<int> out;
    for (int o = 0;; o += tile - overlap) {
        if (o + tile >= fov) {  // clamped final tile (tiles.cpp:11-13)
            out.push_back(fov - tile);
            break;
        }
        out.push_back(o);
    }
    return out;
}

std::vector<Tile> partition_tiles(int fov_w, int fov_h, const Optics& o, double defocus) {
    const auto xs = tile_origins(fov_w, o.tile_size, o.tile_overlap);
    const auto ys = tile_origins(fov_h, o.tile_size, o.tile_overlap);
    std::vector<Tile> out;
    out.reserve(xs.size() * ys.size());
    const int hr = o.led_scan_rows / 2, hc = o.led_scan_cols / 2;
    for (int y0 : ys)
        for (int x0 : xs) {
            Tile t;
            t.x0 = x0;
            t.y0 = y0;
            t.size = o.tile_size;
            t.defocus_um = defocus;
            // centre in object-plane micron relative to the FOV centre (tiles.cpp:35-36)
            t.center_x_um = (x0 + o.tile_size / 2.0 - fov_w / 2.0) * o.dx_obj();
            t.center_y_um = (y0 + o.tile_size / 2.0 - fov_h / 2.0) * o.dx_obj();
            for (int dr = -hr; dr <= hr; ++dr)
                for (int dc = -hc; dc <= hc; ++dc) {
                    const Led led{o.center_led.row + dr, o.center_led.col + dc};
                    t.kvecs[led] = illumination_wavevector(led, {t.center_x_um, t.center_y_um}, o);
                }
            out.push_back(std::move(t));
        }
    return out;
}

// =============================================================== recon.cpp
const LrFrame* FrameStack::find(Led led) const {
    for (const auto& f : frames)
        if (f.led == led) return &f;
    return nullptr;
}

std::vector<std::pair<int, int>> sequence_offsets(Order order, int rows, int cols) {
    if (rows % 2 == 0 || cols % 2 == 0) throw ConfigError("scan dimensions must be odd");
    const int hr = rows / 2, hc = cols / 2;
    const size_t total = size_t(rows) * size_t(cols);
    std::vector<std::pair<int, int>> out;
    out.reserve(total);
    if (order == Order::Raster) {
        for (int r = -hr; r <= hr; ++r)
            for (int c = -hc; c <= hc; ++c) out.emplace_back(r, c);
        return out;
    }
    // centre first, then legs of length 1,1,2,2,3,3,... turning +col, -row,
    // -col, +row; cells outside the scan rectangle are skipped (recon.cpp:25-39)
    static const int step[4][2] = {{0, 1}, {-1, 0}, {0, -1}, {1, 0}};
    int r = 0, c = 0, dir = 0;
    out.emplace_back(0, 0);
    for (int leg = 1; out.size() < total; ++leg) {
        for (int turn = 0; turn < 2 && out.size() < total; ++turn, dir = (dir + 1) % 4)
            for (int s = 0; s < leg && out.size() < total; ++s) {
                r += step[dir][0];
                c += step[dir][1];
                if (std::abs(r) <= hr && std::abs(c) <= hc) out.emplace_back(r, c);
            }
    }
    return out;
}

Sequence led_sequence(Order order, const Optics& o) {
    Sequence s;
    for (auto [dr, dc] : sequence_offsets(order, o.led_scan_rows, o.led_scan_cols))
        s.push_back({o.center_led.row + dr, o.center_led.col + dc});
    return s;
}

std::pair<int, int> spectrum_offset_px(const KVec& k, const Optics& o) {
    const double dk = 1.0 / (o.tile_size * o.dx_obj());
    return {int(std::lround(k.fy / dk)), int(std::lround(k.fx / dk))};
}

U16Grid crop_frame(const U16Grid& frame, const Tile& t) {
    if (t.y0 + t.size > frame.rows || t.x0 + t.size > frame.cols)
        throw DataError("tile extends past frame bounds");
    U16Grid out(t.size, t.size);
    for (int i = 0; i < t.size; ++i)
        for (int j = 0; j < t.size; ++j) out(i, j) = frame(t.y0 + i, t.x0 + j);
    return out;
}

namespace {
RGrid to_real(const U16Grid& g) {
    RGrid r(g.rows, g.cols);
    for (size_t i = 0; i < g.size(); ++i) r.v[i] = double(g.v[i]);
    return r;
}
double mean_of(const U16Grid& g) {
    double s = 0.0;
    for (auto x : g.v) s += double(x);
    return g.size() ? s / double(g.size()) : 0.0;
}
}  // namespace

Canvas init_canvas(const FrameStack& fs, const Tile& t, const Optics& o) {
    const LrFrame* seed = fs.find(o.center_led);
    if (!seed) {  // brightest-frame fallback (recon.cpp:64-75)
        double best = -1.0;
        for (const auto& f : fs.frames) {
            const double m = mean_of(f.image);
            if (m > best) {
                best = m;
                seed = &f;
            }
        }
        if (!seed) throw DataError("empty frame set");
    }
    RGrid amp = to_real(crop_frame(seed->image, t));
    for (auto& a : amp.v) a = std::sqrt(a);
    RGrid hr = upsample_bilinear(amp, o.upsample);
    CGrid field(hr.rows, hr.cols);
    for (size_t i = 0; i < hr.size(); ++i) field.v[i] = cplx(hr.v[i], 0.0);
    Canvas c;
    c.cfg = o;
    c.spectrum = fft2(field);
    const double inv = 1.0 / (double(o.upsample) * o.upsample);  // recon.cpp:81-84
    for (auto& z : c.spectrum.v) z *= inv;
    return c;
}

CGrid canvas_to_field(const Canvas& c, int threads) {
    CGrid f = ifft2(c.spectrum, threads);
    const double up2 = double(c.cfg.upsample) * c.cfg.upsample;  // recon.cpp:89-90
    for (auto& z : f.v) z *= up2;
    return f;
}

namespace {

// Sub-aperture origin and the bounds check shared by both update rules
// (recon.cpp:98-103).
std::pair<int, int> block_origin(const Canvas& c, const KVec& k, int n) {
    const int N = c.size();
    auto [oy, ox] = spectrum_offset_px(k, c.cfg);
    const int r0 = N / 2 + oy - n / 2;
    const int c0 = N / 2 + ox - n / 2;
    if (r0 < 0 || c0 < 0 || r0 + n > N || c0 + n > N)
        throw DataError("spectrum offset out of canvas bounds");
    return {r0, c0};
}

// Modulus replacement with the measured amplitude plus the residual sums
// (recon.cpp:115-124). Returns num/den.
double replace_modulus(CGrid& e, const RGrid& intensity) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < e.size(); ++i) {
        const double meas = std::sqrt(intensity.v[i]);
        const double mag = std::abs(e.v[i]);
        num += (mag - meas) * (mag - meas);
        den += intensity.v[i];
        e.v[i] = mag > 0 ? e.v[i] * (meas / mag) : cplx(meas, 0.0);
    }
    return den > 0 ? num / den : 0.0;
}

}  // namespace

// Gerchberg–Saxton projection on the disk, without the offset bookkeeping
// (recon.cpp:93-131).
double gs_project(Canvas& c, const RGrid& intensity, const KVec& k, const PupilFn& p,
                  int threads) {
    const int n = p.grid;
    if (intensity.rows != n || intensity.cols != n)
        throw DataError("frame side must equal pupil grid");
    auto [r0, c0] = block_origin(c, k, n);
    CGrid block(n, n, cplx(0, 0));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (p.values(i, j) != cplx(0, 0)) block(i, j) = c.spectrum(r0 + i, c0 + j) * p.values(i, j);
    CGrid e = ifft2(block, threads);
    const double res = replace_modulus(e, intensity);
    CGrid corr = fft2(e, threads);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (p.values(i, j) != cplx(0, 0))
                c.spectrum(r0 + i, c0 + j) = corr(i, j) * std::conj(p.values(i, j));
    return res;
}

double update_step(Canvas& c, const RGrid& intensity, const KVec& k, const PupilFn& p,
                   int threads) {
    const double res = gs_project(c, intensity, k, p, threads);
    c.touched.emplace_back(spectrum_offset_px(k, c.cfg));  // recon.cpp:132
    return res;
}

bool bright_field(std::pair<int, int> offset, double radius_px) {
    return std::hypot(double(offset.first), double(offset.second)) <= radius_px;
}

double update_step_epry(Canvas& c, const RGrid& intensity, const KVec& k, CGrid& pupil,
                        const Grid<uint8_t>& support, double alpha, double beta, double radius_px) {
    const int n = pupil.rows;
    const bool pupil_step = bright_field(spectrum_offset_px(k, c.cfg), radius_px);
    if (intensity.rows != n || intensity.cols != n)
        throw DataError("frame side must equal pupil grid");
    auto [r0, c0] = block_origin(c, k, n);
    CGrid psi(n, n, cplx(0, 0));
    double omax = 0.0, pmax = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (support(i, j)) {
                const cplx O = c.spectrum(r0 + i, c0 + j);
                psi(i, j) = O * pupil(i, j);
                omax = std::max(omax, std::norm(O));
                pmax = std::max(pmax, std::norm(pupil(i, j)));
            }
    CGrid e = ifft2(psi);
    const double res = replace_modulus(e, intensity);
    CGrid psi2 = fft2(e);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (support(i, j)) {
                const cplx O = c.spectrum(r0 + i, c0 + j);
                const cplx P = pupil(i, j);
                const cplx d = psi2(i, j) - psi(i, j);
                if (pmax > 0) c.spectrum(r0 + i, c0 + j) = O + alpha * std::conj(P) * d / pmax;
                if (omax > 0 && pupil_step) pupil(i, j) = P + beta * std::conj(O) * d / omax;
            }
    c.touched.emplace_back(spectrum_offset_px(k, c.cfg));
    return res;
}

namespace {

struct TileInputs {
    std::vector<RGrid> crops;
    std::vector<KVec> kvecs;
};

TileInputs gather_inputs(const FrameStack& fs, const Tile& t, const Sequence& seq) {
    TileInputs in;
    in.crops.reserve(seq.size());
    for (const auto& led : seq) {
        const LrFrame* f = fs.find(led);
        if (!f)
            throw DataError("missing frame for LED (" + std::to_string(led.row) + "," +
                            std::to_string(led.col) + ")");
        in.crops.push_back(to_real(crop_frame(f->image, t)));
        in.kvecs.push_back(t.kvecs.at(led));
    }
    return in;
}

Grid<uint8_t> support_of(const PupilFn& p) {
    Grid<uint8_t> s(p.grid, p.grid, 0);
    for (size_t i = 0; i < s.size(); ++i) s.v[i] = p.values.v[i] != cplx(0, 0);
    return s;
}

}  // namespace

TileResult reconstruct_tile(const FrameStack& fs, const Tile& t, const Optics& o, int iters,
                            const Sequence& seq, int threads, Mode mode, EpryParams ep) {
    if (iters < 1) throw ConfigError("iters must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    TileInputs in = gather_inputs(fs, t, seq);  // recon.cpp:146-156
    PupilFn pupil = build_pupil(o, o.tile_size, t.defocus_um);
    Canvas canvas = init_canvas(fs, t, o);
    TileResult res;
    const Grid<uint8_t> support = support_of(pupil);
    CGrid P = pupil.values;
    for (int pass = 0; pass < iters; ++pass) {  // recon.cpp:161-166
        double sum = 0.0;
        for (size_t k = 0; k < seq.size(); ++k)
            sum += mode == Mode::GS
                       ? update_step(canvas, in.crops[k], in.kvecs[k], pupil, threads)
                       : update_step_epry(canvas, in.crops[k], in.kvecs[k], P, support, ep.alpha, ep.beta,
                                          pupil.radius_px);
        res.pass_mean_residual.push_back(sum / double(seq.size()));
    }
    res.hr = canvas_to_field(canvas, threads);
    res.pupil = mode == Mode::GS ? pupil.values : P;
    res.wall_s = seconds_since(t0);
    return res;
}

// =============================================================== parallel.cpp
int min_safe_lag(const std::vector<std::pair<int, int>>& offs, double radius_px) {
    if (offs.empty()) throw DataError("min_safe_lag: empty sequence");
    // two disks conflict iff their centres are closer than 2 radius (parallel.cpp:19-25)
    const double limit = 2.0 * radius_px;
    int gap = 0;
    for (size_t i = 0; i < offs.size(); ++i)
        for (size_t j = i; j < offs.size(); ++j) {
            const double dy = offs[i].first - offs[j].first;
            const double dx = offs[i].second - offs[j].second;
            if (std::hypot(dx, dy) < limit) gap = std::max(gap, int(j - i));
        }
    return 1 + gap;
}

int min_safe_lag(const Sequence& seq, const Tile& t, const Optics& o) {
    std::vector<std::pair<int, int>> offs;
    for (const auto& led : seq) offs.push_back(spectrum_offset_px(t.kvecs.at(led), o));
    return min_safe_lag(offs, build_pupil(o, o.tile_size, t.defocus_um).radius_px);
}

Schedule build_schedule(int positions, int iters, int lag) {
    if (positions < 1 || iters < 1 || lag < 1) throw ConfigError("invalid schedule parameters");
    Schedule s;
    s.lag = lag;
    s.stages = iters;
    s.rounds.resize(size_t(positions - 1 + (iters - 1) * lag + 1));
    for (int st = 0; st < iters; ++st)  // stage s runs position p at round p + s*lag (:46-48)
        for (int p = 0; p < positions; ++p) s.rounds[size_t(p + st * lag)].push_back({st, p});
    return s;
}

TileResult pipelined_reconstruct_tile(const FrameStack& fs, const Tile& t, const Optics& o,
                                      int iters, const Sequence& seq, std::optional<int> lag,
                                      bool force_unsafe) {
    if (iters < 1) throw ConfigError("iters must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    const int min_lag = min_safe_lag(seq, t, o);
    const int use = lag.value_or(min_lag);
    bool nondet = false;
    if (use < min_lag) {  // parallel.cpp:58-64
        if (!force_unsafe) throw UnsafeLagError(min_lag);
        nondet = true;
    }
    TileInputs in = gather_inputs(fs, t, seq);
    const PupilFn pupil = build_pupil(o, o.tile_size, t.defocus_um);
    Canvas canvas = init_canvas(fs, t, o);
    const Schedule sch = build_schedule(int(seq.size()), iters, use);
    std::vector<std::vector<double>> resid(size_t(iters), std::vector<double>(seq.size(), 0.0));
    for (const auto& round : sch.rounds) {  // parallel.cpp:81-97
        if (round.size() == 1) {
            const auto& e = round.front();
            resid[size_t(e.stage)][size_t(e.position)] = update_step(
                canvas, in.crops[size_t(e.position)], in.kvecs[size_t(e.position)], pupil);
            continue;
        }
        // entries of one round touch disjoint disks and write the shared
        // spectrum concurrently; only the offset log is gathered after the join
        // (the reference pushes updated_offsets unsynchronised, recon.cpp:132)
        std::vector<std::thread> pool;
        for (const auto& e : round)
            pool.emplace_back([&, e] {
                resid[size_t(e.stage)][size_t(e.position)] = gs_project(
                    canvas, in.crops[size_t(e.position)], in.kvecs[size_t(e.position)], pupil, 1);
            });
        for (auto& th : pool) th.join();  // round barrier
        for (const auto& e : round)
            canvas.touched.push_back(spectrum_offset_px(in.kvecs[size_t(e.position)], o));
    }
    TileResult res;
    res.lag = use;
    res.nondeterministic = nondet;
    for (const auto& stage : resid) {
        double s = 0.0;
        for (double r : stage) s += r;
        res.pass_mean_residual.push_back(s / double(stage.size()));
    }
    res.hr = canvas_to_field(canvas);
    res.pupil = pupil.values;
    res.wall_s = seconds_since(t0);
    return res;
}

namespace {

void parallel_for(int workers, size_t count, const std::function<void(size_t)>& fn) {
    if (workers <= 1 || count <= 1) {
        for (size_t i = 0; i < count; ++i) fn(i);
        return;
    }
    // dynamic pool over an atomic work index (parallel.cpp:126-140)
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    const size_t nt = std::min<size_t>(size_t(workers), count);
    for (size_t t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (size_t i = next.fetch_add(1); i < count; i = next.fetch_add(1)) fn(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace

OfflineResult run_offline(const FrameStack& fs, const Optics& o, const Sequence& seq,
                          const OfflineOptions& opt) {
    if (opt.workers < 1) throw ConfigError("workers must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    OfflineResult res;
    res.specs = partition_tiles(fs.width(), fs.height(), o, opt.defocus_um);  // select_tiles :142-151
    if (opt.max_tiles) {
        if (*opt.max_tiles > int(res.specs.size())) throw ConfigError("requested tile count exceeds partition");
        res.specs.resize(size_t(*opt.max_tiles));
    }
    if (!opt.tile_defocus_um.empty()) {
        if (opt.tile_defocus_um.size() != res.specs.size())
            throw ConfigError("tile_defocus_um must list one value per tile");
        for (size_t i = 0; i < res.specs.size(); ++i) res.specs[i].defocus_um = opt.tile_defocus_um[i];
    }
    const size_t T = res.specs.size();
    res.tiles.resize(T);
    res.residuals.resize(T);
    const bool pipeline = opt.force_pipeline || opt.workers > int(T);  // parallel.cpp:166
    if (pipeline && opt.mode != Mode::GS)
        throw ConfigError("pipelined schedule requires Gerchberg-Saxton mode");
    parallel_for(opt.workers, T, [&](size_t i) {
        TileResult r = pipeline ? pipelined_reconstruct_tile(fs, res.specs[i], o, opt.iters, seq,
                                                              opt.lag, opt.force_unsafe_lag)
                                : reconstruct_tile(fs, res.specs[i], o, opt.iters, seq, 1,
                                                   opt.mode, opt.epry);
        res.tiles[i] = std::move(r.hr);
        res.residuals[i] = std::move(r.pass_mean_residual);
    });
    if (!opt.max_tiles) res.stitched = stitch_mosaic(res.tiles, res.specs, o);  // :183
    res.wall_s = seconds_since(t0);
    return res;
}

// =============================================================== stitch.cpp
namespace {
CGrid transposed(const CGrid& f) {
    CGrid t(f.cols, f.rows);
    for (int i = 0; i < f.rows; ++i)
        for (int j = 0; j < f.cols; ++j) t(j, i) = f(i, j);
    return t;
}
CGrid along(const CGrid& f, Axis a) { return a == Axis::Horizontal ? f : transposed(f); }
}  // namespace

cplx mean_ratio(const CGrid& f1, const CGrid& f2, int overlap, Axis axis) {
    if (overlap <= 0) throw DataError("mean_ratio requires a positive overlap");
    const CGrid a = along(f1, axis), b = along(f2, axis);
    if (a.rows != b.rows) throw DataError("overlap strips differ in cross-axis extent");
    if (overlap > a.cols || overlap > b.cols) throw DataError("overlap exceeds field extent");
    // complex means of f1's trailing strip and f2's leading strip (stitch.cpp:25-26)
    cplx m1 = 0.0, m2 = 0.0;
    for (int i = 0; i < a.rows; ++i)
        for (int j = 0; j < overlap; ++j) {
            m1 += a(i, a.cols - overlap + j);
            m2 += b(i, j);
        }
    const double cnt = double(a.rows) * overlap;
    m1 /= cnt;
    m2 /= cnt;
    if (std::abs(m2) < 1e-12) throw DataError("degenerate overlap: |mu2| vanishes");
    return m1 / m2;
}

CGrid stitch_pair(const CGrid& f1, const CGrid& f2, int overlap, Axis axis) {
    const CGrid a = along(f1, axis), b = along(f2, axis);
    if (a.rows != b.rows) throw DataError("stitch_pair: cross-axis dimensions differ");
    if (overlap < 0 || overlap >= a.cols || overlap >= b.cols)
        throw DataError("stitch_pair: overlap out of range");
    const cplx ratio = overlap > 0 ? mean_ratio(f1, f2, overlap, axis) : cplx(1.0, 0.0);
    const int width = a.cols + b.cols - overlap;
    const int cut = a.cols - overlap / 2;  // overlap midline, floor (stitch.cpp:40)
    const int b_from = cut - (a.cols - overlap);
    CGrid out(a.rows, width);
    for (int i = 0; i < a.rows; ++i) {
        for (int j = 0; j < cut; ++j) out(i, j) = a(i, j);
        for (int j = cut; j < width; ++j) out(i, j) = ratio * b(i, b_from + (j - cut));
    }
    return along(out, axis);
}

CGrid stitch_mosaic(const std::vector<CGrid>& tiles, const std::vector<Tile>& specs, const Optics& o) {
    if (tiles.size() != specs.size() || tiles.empty())
        throw DataError("stitch_mosaic: tile/spec count mismatch");
    const int up = o.upsample;
    std::map<int, std::vector<size_t>> rows;  // bucket by y origin (stitch.cpp:54-58)
    for (size_t i = 0; i < specs.size(); ++i) rows[specs[i].y0].push_back(i);
    for (auto& kv : rows)
        std::sort(kv.second.begin(), kv.second.end(),
                  [&](size_t a, size_t b) { return specs[a].x0 < specs[b].x0; });
    std::vector<CGrid> strips;
    std::vector<int> strip_y;
    for (auto& kv : rows) {
        const auto& idx = kv.second;
        CGrid strip = tiles[idx[0]];
        int end = specs[idx[0]].x0 + specs[idx[0]].size;
        for (size_t k = 1; k < idx.size(); ++k) {
            const Tile& s = specs[idx[k]];
            const int ov = end - s.x0;
            if (ov < 0) throw DataError("stitch_mosaic: gap between adjacent tiles");
            strip = stitch_pair(strip, tiles[idx[k]], ov * up, Axis::Horizontal);
            end = s.x0 + s.size;
        }
        strips.push_back(std::move(strip));
        strip_y.push_back(kv.first);
    }
    CGrid out = strips[0];
    int end = strip_y[0] + o.tile_size;
    for (size_t k = 1; k < strips.size(); ++k) {
        const int ov = end - strip_y[k];
        if (ov < 0) throw DataError("stitch_mosaic: gap between tile rows");
        out = stitch_pair(out, strips[k], ov * up, Axis::Vertical);
        end = strip_y[k] + o.tile_size;
    }
    return out;
}

// =============================================================== forward.cpp
namespace {

// Seeded sum of low-frequency sinusoids normalised into [-1, 1]. The draw order
// (u, v, phase, amplitude per term) follows forward.cpp:45-71 so that the same
// libstdc++ engine/distributions reproduce the reference objects bit for bit.
RGrid smooth_texture(int size, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> phase_d(0.0, 2.0 * kPi);
    std::uniform_int_distribution<int> freq_d(1, 5);
    std::uniform_real_distribution<double> amp_d(0.3, 1.0);
    constexpr int terms = 6;
    double u[terms], v[terms], ph[terms], a[terms], norm = 0.0;
    for (int k = 0; k < terms; ++k) {
        u[k] = freq_d(rng);
        v[k] = freq_d(rng);
        ph[k] = phase_d(rng);
        a[k] = amp_d(rng);
        norm += a[k];
    }
    RGrid out(size, size);
    for (int i = 0; i < size; ++i)
        for (int j = 0; j < size; ++j) {
            double s = 0.0;
            for (int k = 0; k < terms; ++k) s += a[k] * std::sin(2.0 * kPi * (u[k] * j + v[k] * i) / size + ph[k]);
            out(i, j) = s / norm;
        }
    return out;
}

struct BarLayout { int period, row_begin, row_end; };

std::vector<BarLayout> bar_layout(int size) {  // forward.cpp:22-41
    const int periods[5] = {64, 32, 16, 8, 4};
    const int band = size / 5;
    std::vector<BarLayout> g;
    for (int k = 0; k < 5; ++k) g.push_back({periods[k], k * band + band / 4, k * band + 3 * band / 4});
    return g;
}

}  // namespace

CGrid synth_object(ObjectKind kind, int size, uint64_t seed) {
    if (size < 256) throw ConfigError("object size must be >= 256");
    CGrid obj(size, size);
    if (kind == ObjectKind::PhaseDisk) {
        const double r = size / 8.0, c = size / 2.0;
        for (int i = 0; i < size; ++i)
            for (int j = 0; j < size; ++j)
                obj(i, j) = std::polar(1.0, std::hypot(i - c, j - c) <= r ? kPi / 2.0 : 0.0);
    } else if (kind == ObjectKind::Bars) {
        std::fill(obj.v.begin(), obj.v.end(), cplx(1.0, 0.0));
        for (const auto& g : bar_layout(size)) {
            const int p = g.period;
            const int start = size / 2 - (5 * p) / 4;
            for (int b = 0; b < 3; ++b)
                for (int i = g.row_begin; i < g.row_end; ++i)
                    for (int j = start + b * p; j < start + b * p + p / 2 && j < size; ++j)
                        obj(i, j) = cplx(0.1, 0.0);
        }
    } else {
        std::mt19937_64 rng(seed);
        const RGrid ta = smooth_texture(size, rng);
        const RGrid tp = smooth_texture(size, rng);
        for (size_t i = 0; i < obj.size(); ++i) obj.v[i] = std::polar(0.55 + 0.35 * ta.v[i], 1.2 * tp.v[i]);
    }
    return obj;
}

RGrid simulate_intensity(const CGrid& obj, const KVec& k, const PupilFn& p, const Optics& o) {
    const int hr = o.hr_size();
    if (obj.rows != hr || obj.cols != hr) throw DataError("object tile must be square with side tile_size*upsample");
    if (p.grid != o.tile_size) throw DataError("pupil grid must equal tile_size");
    const int n = o.tile_size;
    auto [oy, ox] = spectrum_offset_px(k, o);
    const int r0 = hr / 2 + oy - n / 2, c0 = hr / 2 + ox - n / 2;
    if (r0 < 0 || c0 < 0 || r0 + n > hr || c0 + n > hr)
        throw DataError("illumination NA too high for upsample factor");
    const CGrid spec = fft2(obj);
    CGrid block(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) block(i, j) = spec(r0 + i, c0 + j) * p.values(i, j);
    const CGrid f = ifft2(block);
    RGrid out(n, n);
    for (size_t i = 0; i < f.size(); ++i) out.v[i] = std::norm(f.v[i]);
    return out;
}

U16Grid quantize_frame(const RGrid& intensity, double scale, const Noise& noise, uint64_t idx) {
    U16Grid out(intensity.rows, intensity.cols);
    std::mt19937_64 rng(noise.seed ^ (idx * 0x9E3779B97F4A7C15ULL + 1));  // forward.cpp:151
    // traversal order fixes the noise draw sequence: rows outer, columns inner
    // (forward.cpp:152-153)
    for (int i = 0; i < intensity.rows; ++i)
        for (int j = 0; j < intensity.cols; ++j) {
            double counts = intensity(i, j) * scale;
            if (noise.enabled) {
                const double mean = counts / 65535.0 * noise.photons;
                std::poisson_distribution<long long> pd(std::max(mean, 0.0));
                counts = double(pd(rng)) / noise.photons * 65535.0;
            }
            out(i, j) = uint16_t(std::clamp(std::lround(counts), 0L, 65535L));
        }
    return out;
}

FrameStack simulate_dataset(const CGrid& obj, const Sequence& seq, const Optics& o,
                            const Noise& noise, double defocus_um) {
    o.validate();
    const int up = o.upsample;
    if (obj.rows % up != 0 || obj.cols % up != 0)
        throw DataError("object dimensions must be a multiple of upsample");
    const int fov_h = obj.rows / up, fov_w = obj.cols / up;
    const auto tiles = partition_tiles(fov_w, fov_h, o, defocus_um);
    const auto xs = tile_origins(fov_w, o.tile_size, o.tile_overlap);
    const auto ys = tile_origins(fov_h, o.tile_size, o.tile_overlap);
    const int n = o.tile_size;

    // linear feather across each shared overlap (forward.cpp:187-205)
    auto feather = [&](const std::vector<int>& org) {
        std::vector<std::vector<double>> w(org.size(), std::vector<double>(size_t(n), 1.0));
        for (size_t k = 0; k < org.size(); ++k) {
            const int a = org[k];
            if (k > 0) {
                const int prev_end = org[k - 1] + n;
                for (int x = a; x < std::min(prev_end, a + n); ++x)
                    w[k][size_t(x - a)] *= double(x - a + 1) / double(prev_end - a + 1);
            }
            if (k + 1 < org.size()) {
                const int nxt = org[k + 1];
                for (int x = std::max(nxt, a); x < a + n; ++x)
                    w[k][size_t(x - a)] *= double(a + n - x) / double(a + n - nxt + 1);
            }
        }
        return w;
    };
    const auto wx = feather(xs), wy = feather(ys);
    std::vector<RGrid> acc(seq.size(), RGrid(fov_h, fov_w, 0.0));
    RGrid wsum(fov_h, fov_w, 0.0);
    const double cutoff = o.objective_na / o.wavelength;
    const double inv_l2 = 1.0 / (o.wavelength * o.wavelength);

    for (size_t ti = 0; ti < tiles.size(); ++ti) {
        const Tile& t = tiles[ti];
        const size_t cx = ti % xs.size(), cy = ti / xs.size();
        // even guard bands up to n/2 per side (forward.cpp:214-217)
        const int gl = std::min(n / 2, t.x0) & ~1, gr = std::min(n / 2, fov_w - t.x0 - n) & ~1;
        const int gt = std::min(n / 2, t.y0) & ~1, gb = std::min(n / 2, fov_h - t.y0 - n) & ~1;
        const int pw = n + gl + gr, ph = n + gt + gb;
        const int PW = pw * up, PH = ph * up;
        CGrid crop(PH, PW);
        for (int i = 0; i < PH; ++i)
            for (int j = 0; j < PW; ++j) crop(i, j) = obj((t.y0 - gt) * up + i, (t.x0 - gl) * up + j);
        const CGrid spec = fft2(crop);
        const double dky = 1.0 / (ph * o.dx_obj()), dkx = 1.0 / (pw * o.dx_obj());
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) wsum(t.y0 + y, t.x0 + x) += wy[cy][size_t(y)] * wx[cx][size_t(x)];
        for (size_t li = 0; li < seq.size(); ++li) {
            const KVec k = t.kvecs.at(seq[li]);
            const int oy = int(std::lround(k.fy / dky)), ox = int(std::lround(k.fx / dkx));
            const int r0 = PH / 2 + oy - ph / 2, c0 = PW / 2 + ox - pw / 2;
            if (r0 < 0 || c0 < 0 || r0 + ph > PH || c0 + pw > PW)
                throw DataError("illumination NA too high for upsample factor");
            CGrid block(ph, pw, cplx(0, 0));
            for (int i = 0; i < ph; ++i)
                for (int j = 0; j < pw; ++j) {
                    const double fy = (i - ph / 2) * dky, fx = (j - pw / 2) * dkx;
                    const double fr = std::hypot(fy, fx);
                    if (fr > cutoff) continue;
                    cplx ctf(1.0, 0.0);
                    if (defocus_um != 0.0) {
                        const double kz = std::sqrt(std::max(0.0, inv_l2 - fr * fr));
                        ctf = std::polar(1.0, 2.0 * kPi * defocus_um * kz);
                    }
                    block(i, j) = spec(r0 + i, c0 + j) * ctf;
                }
            const CGrid f = ifft2(block);
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x)
                    acc[li](t.y0 + y, t.x0 + x) +=
                        wy[cy][size_t(y)] * wx[cx][size_t(x)] * std::norm(f(gt + y, gl + x));
        }
    }
    for (auto& b : acc)
        for (size_t i = 0; i < b.size(); ++i) b.v[i] /= wsum.v[i];

    // grey-scale anchor: on-axis frame when present, else the brightest (:259-268)
    double peak = 0.0;
    for (size_t li = 0; li < seq.size(); ++li) {
        const double m = *std::max_element(acc[li].v.begin(), acc[li].v.end());
        if (seq[li] == o.center_led) {
            peak = m;
            break;
        }
        peak = std::max(peak, m);
    }
    if (peak <= 0) throw DataError("dataset is identically zero");
    const double scale = 0.8 * 65535.0 / peak;
    FrameStack fs;
    fs.cfg = o;
    const double step = o.acq_pattern_delay + o.acq_exposure;
    for (size_t li = 0; li < seq.size(); ++li) {
        LrFrame f;
        f.led = seq[li];
        f.image = quantize_frame(acc[li], scale, noise, li);
        f.timestamp_s = double(li + 1) * step;
        fs.frames.push_back(std::move(f));
    }
    return fs;
}

// =============================================================== metrics.cpp
CGrid band_limit(const CGrid& field, double na, const Optics& o) {
    const int n = field.rows;
    if (field.cols != n) throw DataError("band_limit expects a square field");
    const double dk = 1.0 / (o.tile_size * o.dx_obj());
    const double radius = (na / o.wavelength) / dk;
    CGrid spec = fft2(field);
    const int c = n / 2;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (std::hypot(double(i - c), double(j - c)) > radius) spec(i, j) = cplx(0, 0);
    return ifft2(spec);
}

cplx global_alignment(const CGrid& recon, const CGrid& truth) {
    cplx num = 0.0;
    double den = 0.0;
    for (size_t i = 0; i < recon.size(); ++i) {
        num += truth.v[i] * std::conj(recon.v[i]);
        den += std::norm(recon.v[i]);
    }
    if (den <= 0) throw DataError("global_alignment: zero reconstruction");
    return num / den;
}

double amplitude_rmse(const CGrid& a, const CGrid& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw DataError("dimension mismatch");
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double d = std::abs(a.v[i]) - std::abs(b.v[i]);
        s += d * d;
    }
    return std::sqrt(s / double(a.size()));
}

double phase_rmse(const CGrid& a, const CGrid& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw DataError("dimension mismatch");
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        double d = std::arg(a.v[i]) - std::arg(b.v[i]);
        while (d > kPi) d -= 2 * kPi;
        while (d < -kPi) d += 2 * kPi;
        s += d * d;
    }
    return std::sqrt(s / double(a.size()));
}

}  // namespace orc
