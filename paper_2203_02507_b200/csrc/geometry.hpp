// Host-side geometry of the B200 engine: the reference's double-precision
// formulas for LED wavevectors, tiles, sequences, spectrum offsets, pupils
// and the pipeline lag. Only their integer products (offsets, origins,
// support disk) reach the device, so those are bit-exact against the
// reference by construction (north-star check 1).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fpm_b200.h"

namespace fpmb {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnsafeLag : std::runtime_error {
    int minimum;
    explicit UnsafeLag(int m)
        : std::runtime_error("pipeline lag below the safe minimum of " + std::to_string(m)),
          minimum(m) {}
};
struct Unsupported : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

using Cfg = fpmgpu_optical_config;

inline double dx_obj(const Cfg& c) { return c.camera_pixel / c.magnification; }

void default_config(Cfg& c);                                          // optics.hpp:30-45
void validate(const Cfg& c);                                          // optics.cpp:7-24
std::pair<double, double> wavevector(const Cfg& c, int row, int col, double cx, double cy);  // optics.cpp:26-39
double pupil_radius_px(const Cfg& c, int grid);                       // optics.cpp:43-49 (throws)
// build_pupil (optics.cpp:41-72): complex128 interleaved [grid][grid]
std::vector<double> build_pupil(const Cfg& c, int grid, double defocus_um, double* radius);
std::vector<uint8_t> support_disk(int grid, double radius_px);        // optics.cpp:59-60
double synthesized_na(const Cfg& c);                                  // optics.cpp:74-85
std::vector<int> tile_origins(int fov, int tile, int overlap);        // tiles.cpp:5-19
std::pair<double, double> tile_center_um(const Cfg& c, int x0, int y0, int fov_w, int fov_h);  // tiles.cpp:35-36
std::vector<std::pair<int, int>> sequence_offsets(int order, int rows, int cols);  // recon.cpp:15-41
std::pair<int, int> spectrum_offset_px(const Cfg& c, double fx, double fy);        // recon.cpp:50-53
int min_safe_lag(const std::vector<std::pair<int, int>>& offs, double radius_px);  // parallel.cpp:17-29
// EPRY pupil-step rule: the sub-aperture at (oy, ox) contains the zero frequency
inline bool bright_field(int oy, int ox, double radius_px) {
    return std::hypot(double(oy), double(ox)) <= radius_px;
}

}  // namespace fpmb
