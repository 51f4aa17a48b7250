// fpm_oracle — CPU double-precision restatement of the reference FPM path.
//
// TEST INFRASTRUCTURE ONLY. This library is the parity checker and the CPU
// baseline ("port" kind) for the B200 engine. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it. The product
// (paper_2203_02507_b200) never links or calls it.
//
// The reference (/root/reference/proj) cannot be compiled here: it needs Eigen 3
// (absent from the image) and its vendored headers (proj/vendor, gitignored and
// absent). Every function below restates the reference algorithm and cites the
// file:line it follows. Storage is row-major (r, c) -> data[r*cols + c]; the
// reference's Eigen arrays are column-major, which changes no arithmetic.
//
// Parity pins (see tests/test_oracle_pins.py): the reference's own known-answer
// tests (test_optics/test_forward/test_recon/test_parallel/test_stitch/test_field)
// are re-expressed against this library and must all pass.
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace orc {

using cplx = std::complex<double>;

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnsafeLagError : std::runtime_error {
    int minimum;
    explicit UnsafeLagError(int m)
        : std::runtime_error("pipeline lag below the safe minimum of " + std::to_string(m)),
          minimum(m) {}
};

// Dense 2-D array, row-major.
template <typename T>
struct Grid {
    int rows = 0, cols = 0;
    std::vector<T> v;
    Grid() = default;
    Grid(int r, int c, T fill = T{}) : rows(r), cols(c), v(size_t(r) * size_t(c), fill) {}
    T& operator()(int r, int c) { return v[size_t(r) * cols + c]; }
    const T& operator()(int r, int c) const { return v[size_t(r) * cols + c]; }
    size_t size() const { return v.size(); }
};
using CGrid = Grid<cplx>;
using RGrid = Grid<double>;
using U16Grid = Grid<uint16_t>;

// ---------------------------------------------------------------- field (field.cpp)
// Centered 2-D transforms: fft2 = fftshift(FFT(ifftshift(x))), forward unscaled,
// inverse 1/(rows*cols) (proj/src/field.cpp:48-67).
CGrid fft2(const CGrid& x, int threads = 1);
CGrid ifft2(const CGrid& x, int threads = 1);
CGrid fftshift(const CGrid& x);   // field.cpp:69-77
CGrid ifftshift(const CGrid& x);  // field.cpp:79-87
RGrid upsample_bilinear(const RGrid& in, int factor);  // field.cpp:89-112
// 1-D in-place DFT of length n over data[k*stride], any n >= 1.
void dft1d(cplx* data, int n, int stride, bool inverse);

// ---------------------------------------------------------------- optics (optics.hpp/.cpp)
struct Led {
    int row = 0, col = 0;
    bool operator==(const Led& o) const { return row == o.row && col == o.col; }
    bool operator<(const Led& o) const { return row != o.row ? row < o.row : col < o.col; }
};

// Defaults follow proj/include/fpm/optics.hpp:29-52.
struct Optics {
    double wavelength = 0.525;
    double objective_na = 0.1;
    double magnification = 2.0;
    double camera_pixel = 2.4;
    double led_pitch = 2.5;
    int led_grid_rows = 64;
    int led_grid_cols = 64;
    double led_height = 83.0;
    Led center_led{32, 32};
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
    void validate() const;  // optics.cpp:7-24
};

struct KVec { double fx = 0.0, fy = 0.0; };

struct PupilFn {
    int grid = 0;
    double radius_px = 0.0;
    double defocus = 0.0;
    CGrid values;
};

KVec illumination_wavevector(Led led, std::pair<double, double> center_um, const Optics& o);  // optics.cpp:26-39
PupilFn build_pupil(const Optics& o, int grid, double defocus_um);                          // optics.cpp:41-72
double synthesized_na(const Optics& o);                                                     // optics.cpp:74-85

// ---------------------------------------------------------------- tiles (tiles.cpp)
struct Tile {
    int x0 = 0, y0 = 0, size = 0;
    double center_x_um = 0.0, center_y_um = 0.0, defocus_um = 0.0;
    std::map<Led, KVec> kvecs;
};
std::vector<int> tile_origins(int fov, int tile, int overlap);                            // tiles.cpp:5-19
std::vector<Tile> partition_tiles(int fov_w, int fov_h, const Optics& o, double defocus = 0.0);  // tiles.cpp:21-48

// ---------------------------------------------------------------- frames (forward.hpp)
struct LrFrame {
    Led led;
    U16Grid image;
    double timestamp_s = 0.0;
};
struct FrameStack {
    std::vector<LrFrame> frames;
    Optics cfg;
    const LrFrame* find(Led led) const;  // forward.cpp:9-13
    int width() const { return frames.empty() ? 0 : frames.front().image.cols; }
    int height() const { return frames.empty() ? 0 : frames.front().image.rows; }
};

// ---------------------------------------------------------------- recon (recon.cpp)
enum class Order { Spiral, Raster };
using Sequence = std::vector<Led>;
std::vector<std::pair<int, int>> sequence_offsets(Order order, int rows, int cols);  // recon.cpp:15-41
Sequence led_sequence(Order order, const Optics& o);                                 // recon.cpp:43-48

struct Canvas {
    CGrid spectrum;
    Optics cfg;
    std::vector<std::pair<int, int>> touched;  // recon.hpp:30 updated_offsets
    int size() const { return spectrum.rows; }
};

std::pair<int, int> spectrum_offset_px(const KVec& k, const Optics& o);  // recon.cpp:50-53
U16Grid crop_frame(const U16Grid& frame, const Tile& t);                  // recon.cpp:55-59
Canvas init_canvas(const FrameStack& fs, const Tile& t, const Optics& o); // recon.cpp:61-86
CGrid canvas_to_field(const Canvas& c, int threads = 1);                  // recon.cpp:88-91

// Gerchberg–Saxton alternating projection (recon.cpp:93-134).
double update_step(Canvas& c, const RGrid& intensity, const KVec& k, const PupilFn& p,
                   int threads = 1);

// EPRY extension (not in the reference). Ou, Zheng & Yang,
// "Embedded pupil function recovery for Fourier ptychographic microscopy",
// Opt. Express 22, 4960 (2014):
//   Psi = O_D P;  Psi' = fft2(sqrt(I) psi/|psi|),  psi = ifft2(Psi)
//   O_D <- O_D + alpha conj(P)   (Psi' - Psi) / max_D |P|^2
//   P   <- P   + beta  conj(O_D) (Psi' - Psi) / max_D |O_D|^2   (old O_D, old P)
// D = `support` (fixed binary disk of the initial pupil). With alpha = 1, beta = 0
// and |P| = 1 on D the object update equals update_step's write-back.
// The pupil is updated only from bright-field LEDs, i.e. when the disk of this
// update contains the zero frequency: hypot(oy, ox) <= radius_px. Dark-field
// pupil updates (sub-apertures without DC) make alpha = beta = 1 diverge on
// wide scans (15x15 on a 64 px tile: residual 0.15 -> 39 -> 65 over three
// passes); the bright-field rule is stable and keeps EPRY's phase gain.
double update_step_epry(Canvas& c, const RGrid& intensity, const KVec& k, CGrid& pupil,
                        const Grid<uint8_t>& support, double alpha, double beta, double radius_px);
// True iff the sub-aperture at (oy, ox) contains the zero frequency (bright field).
bool bright_field(std::pair<int, int> offset, double radius_px);

enum class Mode { GS = 0, EPRY = 1 };
struct EpryParams { double alpha = 1.0, beta = 1.0; };

struct TileResult {
    CGrid hr;
    std::vector<double> pass_mean_residual;
    CGrid pupil;  // final pupil (EPRY) or the fixed pupil (GS)
    double wall_s = 0.0;
    int lag = 1;
    bool nondeterministic = false;
};

TileResult reconstruct_tile(const FrameStack& fs, const Tile& t, const Optics& o, int iters,
                            const Sequence& seq, int threads = 1, Mode mode = Mode::GS,
                            EpryParams ep = {});

// ---------------------------------------------------------------- parallel (parallel.cpp)
int min_safe_lag(const std::vector<std::pair<int, int>>& offs, double radius_px);  // parallel.cpp:17-29
int min_safe_lag(const Sequence& seq, const Tile& t, const Optics& o);            // parallel.cpp:31-37
struct Schedule {
    int lag = 1, stages = 1;
    struct Entry { int stage, position; };
    std::vector<std::vector<Entry>> rounds;
};
Schedule build_schedule(int positions, int iters, int lag);  // parallel.cpp:39-50
TileResult pipelined_reconstruct_tile(const FrameStack& fs, const Tile& t, const Optics& o,
                                      int iters, const Sequence& seq,
                                      std::optional<int> lag = std::nullopt,
                                      bool force_unsafe = false);  // parallel.cpp:52-111

struct OfflineOptions {
    int iters = 5;
    int workers = 1;
    std::optional<int> lag;
    bool force_unsafe_lag = false;
    bool force_pipeline = false;
    double defocus_um = 0.0;
    std::optional<int> max_tiles;
    // extensions (per-tile defocus pupils, EPRY) used by BASELINE configs 3-5
    std::vector<double> tile_defocus_um;
    Mode mode = Mode::GS;
    EpryParams epry;
};
struct OfflineResult {
    std::vector<Tile> specs;
    std::vector<CGrid> tiles;
    std::vector<std::vector<double>> residuals;
    CGrid stitched;
    double wall_s = 0.0;
};
OfflineResult run_offline(const FrameStack& fs, const Optics& o, const Sequence& seq,
                          const OfflineOptions& opt);  // parallel.cpp:155-196

// ---------------------------------------------------------------- stitch (stitch.cpp)
enum class Axis { Horizontal, Vertical };
cplx mean_ratio(const CGrid& f1, const CGrid& f2, int overlap, Axis axis);   // stitch.cpp:18-29
CGrid stitch_pair(const CGrid& f1, const CGrid& f2, int overlap, Axis axis); // stitch.cpp:31-46
CGrid stitch_mosaic(const std::vector<CGrid>& tiles, const std::vector<Tile>& specs,
                    const Optics& o);                                        // stitch.cpp:48-86

// ---------------------------------------------------------------- forward (forward.cpp)
enum class ObjectKind { Bars = 0, PhaseDisk = 1, Composite = 2 };
CGrid synth_object(ObjectKind kind, int size, uint64_t seed);  // forward.cpp:73-112
struct Noise { bool enabled = false; double photons = 1e4; uint64_t seed = 0; };
RGrid simulate_intensity(const CGrid& obj, const KVec& k, const PupilFn& p, const Optics& o);  // :123-139
U16Grid quantize_frame(const RGrid& intensity, double scale, const Noise& noise, uint64_t idx);  // :148-164
FrameStack simulate_dataset(const CGrid& obj, const Sequence& seq, const Optics& o,
                            const Noise& noise = {}, double defocus_um = 0.0);  // :172-282

// ---------------------------------------------------------------- metrics (metrics.cpp)
CGrid band_limit(const CGrid& field, double na, const Optics& o);  // metrics.cpp:7-19
cplx global_alignment(const CGrid& recon, const CGrid& truth);    // metrics.cpp:21-33
double amplitude_rmse(const CGrid& a, const CGrid& b);            // metrics.cpp:35-44
double phase_rmse(const CGrid& a, const CGrid& b);                // metrics.cpp:46-57

}  // namespace orc
