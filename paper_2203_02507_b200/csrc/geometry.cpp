#include "geometry.hpp"

#include <algorithm>
#include <cmath>

namespace fpmb {

namespace {
constexpr double kPi = 3.14159265358979323846;
}

void default_config(Cfg& c) {
    c.wavelength = 0.525;
    c.objective_na = 0.1;
    c.magnification = 2.0;
    c.camera_pixel = 2.4;
    c.led_pitch = 2.5;
    c.led_grid_rows = 64;
    c.led_grid_cols = 64;
    c.led_height = 83.0;
    c.center_row = 32;
    c.center_col = 32;
    c.led_scan_rows = 13;
    c.led_scan_cols = 13;
    c.upsample = 4;
    c.tile_size = 256;
    c.tile_overlap = 26;
    c.acq_pattern_delay = 0.3;
    c.acq_exposure = 0.03;
}

void validate(const Cfg& c) {
    auto bad = [](const char* w) { throw ConfigError(std::string("config invariant violated: ") + w); };
    if (!(c.wavelength > 0)) bad("wavelength > 0");
    if (!(c.objective_na > 0 && c.objective_na < 1)) bad("0 < objective_na < 1");
    if (!(c.magnification > 0)) bad("magnification > 0");
    if (!(c.camera_pixel > 0)) bad("camera_pixel > 0");
    if (!(c.led_pitch > 0)) bad("led_pitch > 0");
    if (!(c.led_height > 0)) bad("led_height > 0");
    if (c.led_grid_rows < 1 || c.led_grid_cols < 1) bad("led_grid positive");
    if (c.led_scan_rows % 2 == 0 || c.led_scan_cols % 2 == 0) bad("led_scan dimensions odd");
    if (c.center_row - c.led_scan_rows / 2 < 0 || c.center_row + c.led_scan_rows / 2 >= c.led_grid_rows ||
        c.center_col - c.led_scan_cols / 2 < 0 || c.center_col + c.led_scan_cols / 2 >= c.led_grid_cols)
        bad("led_scan fits inside led_grid");
    if (c.upsample < 2) bad("upsample >= 2");
    if (c.tile_size < 1) bad("tile_size positive");
    if (!(c.tile_overlap >= 0 && c.tile_overlap < c.tile_size)) bad("tile_overlap < tile_size");
    if (!(c.acq_pattern_delay >= 0 && c.acq_exposure >= 0)) bad("acquisition times >= 0");
}

std::pair<double, double> wavevector(const Cfg& c, int row, int col, double cx, double cy) {
    if (row < 0 || row >= c.led_grid_rows || col < 0 || col >= c.led_grid_cols)
        throw std::domain_error("LED index (" + std::to_string(row) + "," + std::to_string(col) +
                                ") outside LED grid");
    const double pitch_um = c.led_pitch * 1000.0;
    const double dx = (col - c.center_col) * pitch_um - cx;
    const double dy = (row - c.center_row) * pitch_um - cy;
    const double h = c.led_height * 1000.0;
    const double d = std::sqrt(dx * dx + dy * dy + h * h);
    // an LED toward +x samples the -x side of the spectrum (optics.hpp:69-71)
    return {-dx / (c.wavelength * d), -dy / (c.wavelength * d)};
}

double pupil_radius_px(const Cfg& c, int grid) {
    if (grid < 32 || grid % 2 != 0) throw ConfigError("pupil grid must be even and >= 32");
    const double dk = 1.0 / (grid * dx_obj(c));
    const double r = (c.objective_na / c.wavelength) / dk;
    if (r >= grid / 2.0)
        throw ConfigError("pupil exceeds Nyquist of LR grid (radius " + std::to_string(r) +
                          " px, grid " + std::to_string(grid) + ")");
    return r;
}

std::vector<uint8_t> support_disk(int grid, double radius_px) {
    std::vector<uint8_t> s(size_t(grid) * grid, 0);
    const int c = grid / 2;
    for (int i = 0; i < grid; ++i)
        for (int j = 0; j < grid; ++j)
            s[size_t(i) * grid + j] = std::hypot(double(i - c), double(j - c)) <= radius_px;
    return s;
}

std::vector<double> build_pupil(const Cfg& c, int grid, double defocus_um, double* radius) {
    const double r = pupil_radius_px(c, grid);
    if (radius) *radius = r;
    const double dk = 1.0 / (grid * dx_obj(c));
    const double inv_l2 = 1.0 / (c.wavelength * c.wavelength);
    std::vector<double> v(size_t(grid) * grid * 2, 0.0);
    const int ctr = grid / 2;
    for (int i = 0; i < grid; ++i)
        for (int j = 0; j < grid; ++j) {
            const double rho = std::hypot(double(i - ctr), double(j - ctr));
            if (rho > r) continue;
            double re = 1.0, im = 0.0;
            if (defocus_um != 0.0) {
                const double kz = std::sqrt(std::max(0.0, inv_l2 - rho * dk * rho * dk));
                const double ph = 2.0 * kPi * defocus_um * kz;
                re = std::cos(ph);
                im = std::sin(ph);
            }
            v[(size_t(i) * grid + j) * 2] = re;
            v[(size_t(i) * grid + j) * 2 + 1] = im;
        }
    return v;
}

double synthesized_na(const Cfg& c) {
    double m = 0.0;
    for (int dr = -c.led_scan_rows / 2; dr <= c.led_scan_rows / 2; ++dr)
        for (int dc = -c.led_scan_cols / 2; dc <= c.led_scan_cols / 2; ++dc) {
            auto [fx, fy] = wavevector(c, c.center_row + dr, c.center_col + dc, 0.0, 0.0);
            m = std::max(m, c.wavelength * std::hypot(fx, fy));
        }
    return c.objective_na + m;
}

std::vector<int> tile_origins(int fov, int tile, int overlap) {
    if (fov < tile) throw ConfigError("FOV smaller than one tile");
    std::vector<int> v;
    int o = 0;
    while (o + tile < fov) {
        v.push_back(o);
        o += tile - overlap;
    }
    v.push_back(fov - tile);  // clamped final tile
    return v;
}

std::pair<double, double> tile_center_um(const Cfg& c, int x0, int y0, int fov_w, int fov_h) {
    return {(x0 + c.tile_size / 2.0 - fov_w / 2.0) * dx_obj(c),
            (y0 + c.tile_size / 2.0 - fov_h / 2.0) * dx_obj(c)};
}

std::vector<std::pair<int, int>> sequence_offsets(int order, int rows, int cols) {
    if (rows % 2 == 0 || cols % 2 == 0) throw ConfigError("scan dimensions must be odd");
    const int hr = rows / 2, hc = cols / 2;
    const size_t total = size_t(rows) * cols;
    std::vector<std::pair<int, int>> out;
    if (order == FPMGPU_ORDER_RASTER) {
        for (int r = -hr; r <= hr; ++r)
            for (int c = -hc; c <= hc; ++c) out.emplace_back(r, c);
        return out;
    }
    if (order != FPMGPU_ORDER_SPIRAL) throw ConfigError("unknown update order");
    // centre, then legs 1,1,2,2,... turning +col, -row, -col, +row
    const int dr[4] = {0, -1, 0, 1}, dc[4] = {1, 0, -1, 0};
    int r = 0, c = 0, d = 0;
    out.emplace_back(0, 0);
    for (int leg = 1; out.size() < total; ++leg)
        for (int half = 0; half < 2 && out.size() < total; ++half, d = (d + 1) & 3)
            for (int s = 0; s < leg && out.size() < total; ++s) {
                r += dr[d];
                c += dc[d];
                if (std::abs(r) <= hr && std::abs(c) <= hc) out.emplace_back(r, c);
            }
    return out;
}

std::pair<int, int> spectrum_offset_px(const Cfg& c, double fx, double fy) {
    const double dk = 1.0 / (c.tile_size * dx_obj(c));
    return {int(std::lround(fy / dk)), int(std::lround(fx / dk))};
}

int min_safe_lag(const std::vector<std::pair<int, int>>& offs, double radius_px) {
    if (offs.empty()) throw DataError("min_safe_lag: empty sequence");
    const double lim = 2.0 * radius_px;
    int gap = 0;
    for (size_t i = 0; i < offs.size(); ++i)
        for (size_t j = i + size_t(gap) + 1; j < offs.size(); ++j)  // only larger gaps can matter
            if (std::hypot(double(offs[i].second - offs[j].second),
                           double(offs[i].first - offs[j].first)) < lim)
                gap = int(j - i);
    return 1 + gap;
}

}  // namespace fpmb
