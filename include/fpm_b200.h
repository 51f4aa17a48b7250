/*
 * fpm_b200.h — C-ABI of the B200-native FPM reconstruction engine.
 *
 * Drop-in boundary for the reference's per-tile reconstruction path
 * (/root/reference/proj): run_offline -> reconstruct_tile -> update_step ->
 * fft2/ifft2. The reference exposes that path as a C++ library API (no FFI
 * layer exists); every entry point below names the reference function it
 * replaces. Plain pointers and sizes only; no exceptions cross this boundary:
 * every call returns an FPMGPU_* status and fpmgpu_last_error() holds the
 * reference's message text (e.g. "missing frame", "spectrum offset out of
 * canvas bounds", "pupil exceeds Nyquist").
 *
 * Arrays are row-major. Complex values are interleaved (re, im): complex64 as
 * float[2], complex128 as double[2]. The reference's Eigen arrays are
 * column-major; the C++ mirror (fpm_b200.hpp) converts.
 */
#ifndef FPM_B200_H
#define FPM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPMGPU_OK 0
#define FPMGPU_ERR_CONFIG 1      /* fpm::ConfigError          (optics.hpp:11-13)  */
#define FPMGPU_ERR_DATA 2        /* fpm::DataError            (optics.hpp:14-16)  */
#define FPMGPU_ERR_UNSAFE_LAG 3  /* fpm::UnsafeLagError       (parallel.hpp:12-17)*/
#define FPMGPU_ERR_DOMAIN 4      /* std::domain_error         (optics.cpp:28-30)  */
#define FPMGPU_ERR_CUDA 5        /* device / driver failure                        */
#define FPMGPU_ERR_INTERNAL 6
#define FPMGPU_ERR_UNSUPPORTED 7 /* geometry without a device kernel (tile side) */

#define FPMGPU_MODE_GS 0   /* Gerchberg–Saxton replacement (recon.cpp:93-134) */
#define FPMGPU_MODE_EPRY 1 /* + embedded pupil recovery (extension) */

#define FPMGPU_ORDER_SPIRAL 0 /* UpdateOrder::Spiral (recon.hpp:12) */
#define FPMGPU_ORDER_RASTER 1

/* OpticalConfig (optics.hpp:29-52), same fields and units. */
typedef struct fpmgpu_optical_config {
    double wavelength, objective_na, magnification, camera_pixel, led_pitch;
    int led_grid_rows, led_grid_cols;
    double led_height;
    int center_row, center_col, led_scan_rows, led_scan_cols, upsample, tile_size, tile_overlap;
    double acq_pattern_delay, acq_exposure;
} fpmgpu_optical_config;

int fpmgpu_version(void);
const char* fpmgpu_last_error(void);
/* minimum lag carried by the last FPMGPU_ERR_UNSAFE_LAG (UnsafeLagError::minimum) */
int fpmgpu_last_min_lag(void);
/* fills the reference defaults (optics.hpp:30-45) */
void fpmgpu_default_config(fpmgpu_optical_config* cfg);

/* ---------------------------------------------------------------------------
 * Host geometry: exact reference arithmetic in double. The device consumes
 * only their integer outputs, so offsets, sub-aperture origins and the
 * support disk are bit-exact against the reference by construction.
 * ------------------------------------------------------------------------- */
/* OpticalConfig::validate (optics.cpp:7-24) */
int fpmgpu_validate_config(const fpmgpu_optical_config* cfg);
/* illumination_wavevector (optics.cpp:26-39) */
int fpmgpu_illumination_wavevector(const fpmgpu_optical_config* cfg, int led_row, int led_col,
                                   double center_x_um, double center_y_um, double* fx, double* fy);
/* build_pupil (optics.cpp:41-72); values: [grid][grid] complex128 or NULL */
int fpmgpu_build_pupil(const fpmgpu_optical_config* cfg, int grid, double defocus_um,
                       double* values, double* radius_px);
/* synthesized_na (optics.cpp:74-85) */
int fpmgpu_synthesized_na(const fpmgpu_optical_config* cfg, double* out);
/* tile_origins (tiles.cpp:5-19); writes min(count, cap) origins */
int fpmgpu_tile_origins(int fov, int tile_size, int tile_overlap, int* out, int cap, int* count);
/* partition_tiles (tiles.cpp:21-48) restricted to the LEDs of `seq` ([L][2] (row, col)):
 * xy [T][2] (x0, y0), centers [T][2] um, kvecs [T][L][2] (fx, fy), offsets [T][L][2]
 * (oy, ox) = spectrum_offset_px (recon.cpp:50-53). Any output may be NULL. */
int fpmgpu_partition_tiles(const fpmgpu_optical_config* cfg, int fov_w, int fov_h,
                           const int* seq, int num_leds, int cap, int* count, int* xy,
                           double* centers, double* kvecs, int* offsets);
/* sequence_offsets (recon.cpp:15-41): out [rows*cols][2] (dr, dc) */
int fpmgpu_sequence_offsets(int order, int rows, int cols, int* out);
/* spectrum_offset_px (recon.cpp:50-53) */
int fpmgpu_spectrum_offset_px(const fpmgpu_optical_config* cfg, double fx, double fy, int* oy,
                              int* ox);
/* min_safe_lag (parallel.cpp:17-29) */
int fpmgpu_min_safe_lag(const int* offsets, int count, double radius_px, int* out);
/* build_schedule (parallel.cpp:39-50): entries [positions*iters][3] (round, stage, position) */
int fpmgpu_build_schedule(int positions, int iters, int lag, int* entries, int* rounds);

/* ---------------------------------------------------------------------------
 * Device engine.
 * ------------------------------------------------------------------------- */
typedef struct fpmgpu_context fpmgpu_context;
typedef struct fpmgpu_plan fpmgpu_plan;

int fpmgpu_create(int device, fpmgpu_context** out);
int fpmgpu_destroy(fpmgpu_context* ctx);

/* One batched reconstruction: T tiles of one FOV, each the reference's
 * reconstruct_tile (recon.cpp:141-170) — or pipelined_reconstruct_tile
 * (parallel.cpp:52-111) when lag != 0 — followed by canvas_to_field. */
typedef struct fpmgpu_recon_request {
    fpmgpu_optical_config cfg; /* tile_size = n (LR side), upsample: N = n*upsample */
    int iters;                 /* passes over the sequence (>= 1) */
    int mode;                  /* FPMGPU_MODE_GS | FPMGPU_MODE_EPRY */
    double alpha, beta;        /* EPRY step sizes (ignored for GS) */
    int lag;                   /* 0 sequential; > 0 pipelined at this lag; -1 pipelined, auto lag */
    int force_unsafe_lag;      /* run a lag below min_safe_lag (result nondeterministic) */
    int num_tiles;             /* T */
    const int* tile_xy;        /* [T][2] (x0, y0) LR origin of each tile in the frames */
    int num_leds;              /* L (sequence length) */
    const int* offsets;        /* [T][L][2] (oy, ox) spectrum offsets in sequence order */
    const int* seq_frame;      /* [L] frame index of sequence position k */
    int init_frame;            /* frame seeding init_canvas (on-axis, else brightest) */
    const double* tile_defocus_um; /* [T] per-tile defocus for build_pupil, or NULL (0) */
    const float* pupils;       /* [T][n][n] complex64 initial pupils or NULL (built) */
    int num_frames, height, width; /* LR stack geometry: frames [F][H][W] u16 */
} fpmgpu_recon_request;

/* Host-buffer call (the reference-facing path): frames [F][H][row_pitch] u16 in
 * host memory; outputs to host memory (any may be NULL): hr [T][N][N]
 * complex64 (canvas_to_field units), residuals [T][iters]
 * (pass_mean_residual), pupils_out [T][n][n] complex64. Copies in/out are
 * part of the call. */
int fpmgpu_reconstruct_tiles(fpmgpu_context* ctx, const fpmgpu_recon_request* req,
                             const uint16_t* frames, int64_t row_pitch, float* hr,
                             double* residuals, float* pupils_out, int* lag_used);

/* The same call split in two, so consecutive requests overlap: request k + 1's
 * LR upload runs under request k's reconstruction (two staging slots per
 * context; a third submit first waits for the oldest). The host buffers of a
 * request must stay valid and untouched until fpmgpu_wait(ticket) returns;
 * use pinned memory for the copies to be asynchronous. A request older than the
 * two slots completed when its slot was reused; waiting on it returns at once. */
int fpmgpu_reconstruct_tiles_async(fpmgpu_context* ctx, const fpmgpu_recon_request* req,
                                   const uint16_t* frames, int64_t row_pitch, float* hr,
                                   double* residuals, float* pupils_out, long long* ticket);
int fpmgpu_wait(fpmgpu_context* ctx, long long ticket, int* lag_used);

/* Online session — replaces run_online (parallel.cpp:198-317): frames arrive one
 * at a time; each is copied to the device on arrival, and the first-pass
 * update of sequence position k is launched for every tile as soon as frames
 * seq_frame[0..k] and the seed frame (init_frame) are resident (updates wait for
 * the seed, parallel.cpp:266-273). finish() runs the remaining iters-1 passes
 * (parallel.cpp:289-303) and canvas_to_field. The update order per tile is the
 * sequential one, so results equal fpmgpu_reconstruct_tiles with lag = 0.
 * `frame` is a host pointer to one u16 frame [H][row_pitch]; it must stay valid
 * (and unchanged) until finish returns. Requires lag = 0. */
typedef struct fpmgpu_online fpmgpu_online;
int fpmgpu_online_begin(fpmgpu_context* ctx, const fpmgpu_recon_request* req, fpmgpu_online** out);
int fpmgpu_online_push(fpmgpu_online* on, int frame_index, const uint16_t* frame, int64_t row_pitch,
                       int* positions_applied);
int fpmgpu_online_finish(fpmgpu_online* on, float* hr, double* residuals, float* pupils_out);
int fpmgpu_online_destroy(fpmgpu_online* on);

/* Plans: validate + upload the geometry tables once, then execute on device
 * buffers (frames/hr/residuals/pupils_out are DEVICE pointers; row_pitch in
 * elements, row_pitch*2 must be a multiple of 16 bytes). `stream` is a
 * cudaStream_t (NULL = legacy default). */
int fpmgpu_plan_create(fpmgpu_context* ctx, const fpmgpu_recon_request* req, fpmgpu_plan** out);
int fpmgpu_plan_execute(fpmgpu_plan* plan, const uint16_t* frames_dev, int64_t row_pitch,
                        float* hr_dev, double* residuals_dev, float* pupils_out_dev, void* stream);
int fpmgpu_plan_destroy(fpmgpu_plan* plan);

/* run_offline's tiles + stitch_mosaic (parallel.cpp:170-183) in one pass when the
 * plan's tiles abut without overlap on a full grid (stitch.cpp:38: zero overlap
 * concatenates unscaled): canvas_to_field writes every HR field straight into
 * the mosaic, tile t at row (y0 - y_min)*up, column (x0 - x_min)*up of mosaic_dev
 * (mosaic_pitch elements per row). mosaic_dev may be a peer GPU's buffer
 * (fpmgpu_ipc_open): each rank of a multi-GPU run then writes its band of the
 * mosaic over NVLink. FPMGPU_ERR_UNSUPPORTED when the tiles overlap. */
int fpmgpu_plan_execute_mosaic(fpmgpu_plan* plan, const uint16_t* frames_dev, int64_t row_pitch,
                               float* mosaic_dev, int64_t mosaic_pitch, double* residuals_dev,
                               float* pupils_out_dev, void* stream);

typedef struct fpmgpu_plan_info {
    int tile_side, canvas_side, num_tiles, num_leds, iters, mode, lag, groups;
    int launches_per_execute;   /* kernels launched by one fpmgpu_plan_execute */
    int loop_ctas, loop_threads, loop_smem_bytes;
    double updates;             /* T * L * iters */
    double fft_flops_per_update;  /* 20 n^2 log2 n (nominal) */
    double hbm_bytes_per_update;  /* 2 n^2 + 16 |D| */
    int support_pixels;         /* |D| */
    int tiles_abut;             /* 1: tiles on a full grid at stride n, no overlap (execute_mosaic) */
} fpmgpu_plan_info;
int fpmgpu_plan_get_info(const fpmgpu_plan* plan, fpmgpu_plan_info* info);

/* Device time of each phase, summed over the executes recorded since the last
 * reset (CUDA events on the execute stream around every phase): ms[0] pupils +
 * init_canvas, ms[1] LED loop kernel, ms[2] canvas_to_field. Call after the
 * stream has been synchronised; reset != 0 clears the record afterwards. */
int fpmgpu_plan_phase_times(fpmgpu_plan* plan, double* ms, int* executes, int reset);

/* Single alternating-projection step on a host canvas (update_step,
 * recon.cpp:93-134; EPRY step when mode = EPRY, pupil updated in place).
 * canvas [N][N] complex64 in/out, intensity [n][n] float, pupil [n][n]
 * complex64 (in/out for EPRY). Support = pupil != 0 on entry. */
int fpmgpu_update_step(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, float* canvas,
                       const float* intensity, double fx, double fy, float* pupil, int mode,
                       double alpha, double beta, double* residual);

/* init_canvas (recon.cpp:61-86) for one tile from frame [H][row_pitch] u16 at
 * (x0, y0); canvas_to_field (recon.cpp:88-91). Host buffers, complex64. */
int fpmgpu_init_canvas(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg,
                       const uint16_t* frame, int height, int width, int64_t row_pitch, int x0,
                       int y0, float* canvas);
int fpmgpu_canvas_to_field(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg,
                           const float* canvas, float* field);

/* stitch_mosaic (stitch.cpp:48-86) of T HR tiles [T][N][N] complex64 (host) at LR
 * origins xy [T][2]; out [rows][cols] complex64 (host) or NULL to query the size. */
int fpmgpu_stitch_mosaic(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const float* tiles,
                         const int* xy, int num_tiles, float* out, int* rows, int* cols);
/* Same on device buffers (tiles_dev [T][N][N], out_dev [rows][cols] complex64;
 * out_dev NULL = size query), enqueued on `stream` (cudaStream_t). */
int fpmgpu_stitch_mosaic_device(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg,
                                const float* tiles_dev, const int* xy, int num_tiles, float* out_dev,
                                int* rows, int* cols, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU mosaic: stitch_mosaic (stitch.cpp:48-86) over tile-row bands, one
 * band per rank. xy [T][2] lists the WHOLE FOV's tile origins (the same on every
 * rank); a band is tiles [tile_lo, tile_hi) of that list and must be whole tile
 * rows. Eq. (1)'s ratios form a chain across the FOV: each band computes its
 * strips' row sums (sums), the ranks combine them (every rank needs every strip's
 * sums: an all-reduce of zero-filled [strips][N] complex128 arrays is exact),
 * and each band writes its own mosaic rows (assemble), straight into rank 0's
 * mosaic over NVLink when mosaic_dev is a peer pointer. The single-GPU
 * fpmgpu_stitch_mosaic is the one band of every tile: same arithmetic, same bits.
 * ------------------------------------------------------------------------- */
typedef struct fpmgpu_mosaic_band_info {
    int rows, cols;              /* the whole mosaic */
    int strips, strip_lo, strip_hi; /* tile rows; the band's [strip_lo, strip_hi) */
    int row_lo, row_hi;          /* mosaic rows the band writes */
    int canvas_side;             /* N */
    int needs_exchange;          /* 0: every overlap is 0, ratios are 1, no sums needed */
} fpmgpu_mosaic_band_info;
/* host-only geometry query */
int fpmgpu_mosaic_band_layout(const fpmgpu_optical_config* cfg, const int* xy, int num_tiles,
                              int tile_lo, int tile_hi, fpmgpu_mosaic_band_info* info);
/* tiles_dev: the band's HR tiles [tile_hi - tile_lo][N][N] complex64 (device).
 * strip_sums [strips][N] complex128 (host): the band's strips are written, the
 * others untouched; ratios [tile_hi - tile_lo] complex128 (host) out. Synchronous. */
int fpmgpu_mosaic_band_sums(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const int* xy,
                            int num_tiles, int tile_lo, int tile_hi, const float* tiles_dev,
                            double* strip_sums, double* ratios, void* stream);
/* strip_sums: every strip's sums (combined over the bands); ratios: this band's.
 * mosaic_dev = row 0 of the whole mosaic (device, possibly a peer's), pitch in
 * elements. Returns after the band's rows are written. */
int fpmgpu_mosaic_band_assemble(fpmgpu_context* ctx, const fpmgpu_optical_config* cfg, const int* xy,
                                int num_tiles, int tile_lo, int tile_hi, const float* tiles_dev,
                                const double* strip_sums, const double* ratios, float* mosaic_dev,
                                int64_t mosaic_pitch, void* stream);

/* CUDA IPC of a device buffer (rank 0's mosaic) to the other ranks' processes:
 * handle = FPMGPU_IPC_HANDLE_BYTES opaque bytes naming dev_ptr's allocation,
 * offset = dev_ptr's byte offset inside it (add it to the opened pointer). */
#define FPMGPU_IPC_HANDLE_BYTES 64
int fpmgpu_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset);
int fpmgpu_ipc_open(fpmgpu_context* ctx, const void* handle, void** dev_ptr);
int fpmgpu_ipc_close(fpmgpu_context* ctx, void* dev_ptr);

/* Batched 2-D complex128 FFT, in place on data_dev [batch][rows][cols] (device,
 * interleaved re/im doubles), sides with factors 2, 3, 5 up to 4096; forward
 * unnormalised, inverse scaled by 1/(rows*cols) (field.cpp:18-67 before the
 * shifts). The transforms of the GPU forward model (simulate_dataset,
 * forward.cpp:172-282), whose tile grids are 96 / 120 / 384 / 480 ... points. */
int fpmgpu_fft2_c128(fpmgpu_context* ctx, double* data_dev, int64_t batch, int rows, int cols,
                     int inverse, void* stream);

/* Page-locked host buffers (outputs of the async host path must be page-locked
 * for the copies to overlap; pageable outputs make the call synchronous). */
int fpmgpu_host_alloc(int64_t bytes, void** ptr);
int fpmgpu_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* FPM_B200_H */
