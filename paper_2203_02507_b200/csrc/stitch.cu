// Eq. (1) mosaic on the device (stitch_mosaic, stitch.cpp:48-86).
//
// The reference stitches each tile row left to right (stitch_pair with
// mean_ratio, stitch.cpp:18-46), then the strips top to bottom. Unrolled, the
// result is a grid of rectangles: mosaic pixel (R, C) belongs to the tile whose
// row/column cut intervals (cuts at the overlap midlines, stitch.cpp:40) contain
// it and equals F_t * tile_t[R - Y_t][C - X_t], F_t = S_strip * R_t. Every mean
// the reference takes is a range sum of per-tile column sums (horizontal
// strips) or of per-tile row sums over the tile's owned columns (vertical
// strips), so the device produces those sums (stitch_sums), the host forms the
// ratios in double, and one pass writes the mosaic (stitch_assemble).
#include <cuda_runtime.h>

#include "fft_device.cuh"
#include "stitch.cuh"

namespace fpmk {

namespace {

// colsum[t][c] = sum_r tile_t[r][c]  (complex128), row bands of 32 rows.
__global__ void stitch_colsum_kernel(const float2* __restrict__ tiles, int N, double* __restrict__ colsum) {
    const int t = blockIdx.y;
    const int r0 = blockIdx.x * 32;
    const float2* base = tiles + size_t(t) * N * N;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        double re = 0.0, im = 0.0;
        for (int r = r0; r < r0 + 32 && r < N; ++r) {
            const float2 v = base[size_t(r) * N + c];
            re += v.x;
            im += v.y;
        }
        atomicAdd(colsum + (size_t(t) * N + c) * 2, re);
        atomicAdd(colsum + (size_t(t) * N + c) * 2 + 1, im);
    }
}

// rowsum[t][r] = sum_{c in [own_c0, own_c1)} tile_t[r][c]; one warp per row.
__global__ void stitch_rowsum_kernel(const float2* __restrict__ tiles, const StitchTile* __restrict__ st, int N,
                                     double* __restrict__ rowsum) {
    const int t = blockIdx.y;
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= N) return;
    const StitchTile s = st[t];
    const float2* row = tiles + size_t(t) * N * N + size_t(r) * N;
    double re = 0.0, im = 0.0;
    for (int c = s.own_c0 + lane; c < s.own_c1; c += 32) {
        re += row[c].x;
        im += row[c].y;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) {
        rowsum[(size_t(t) * N + r) * 2] = re;
        rowsum[(size_t(t) * N + r) * 2 + 1] = im;
    }
}

// Mosaic pixel (R, C), R in [row0, row0 + nrows): owner tile via the strip/slot
// interval tables; grid holds the band's strips [strip0, ...) with band-local
// tile indices. out is the mosaic's row 0 (pitch in elements; a peer GPU's
// mosaic when the band is written over NVLink).
__global__ void stitch_assemble_kernel(const float2* __restrict__ tiles, const StitchTile* __restrict__ st,
                                       const int* __restrict__ row_of, const int* __restrict__ col_of,
                                       const int* __restrict__ grid, int strip0, int n_cols, int N, int row0,
                                       int nrows, int cols, long long pitch, float2* __restrict__ out) {
    const size_t total = size_t(nrows) * cols;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int R = row0 + int(idx / cols), Cc = int(idx % cols);
        const int t = grid[(row_of[R] - strip0) * n_cols + col_of[Cc]];
        const StitchTile s = st[t];
        const float2 v = tiles[size_t(t) * N * N + size_t(R - s.Y) * N + (Cc - s.X)];
        out[size_t(R) * pitch + Cc] = cmul(v, make_float2(s.fre, s.fim));
    }
}

}  // namespace

cudaError_t launch_stitch_sums(const float2* tiles, const StitchTile* st, int T, int N, double* colsum,
                               double* rowsum, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(colsum, 0, sizeof(double) * 2 * size_t(T) * N, s);
    if (e != cudaSuccess) return e;
    stitch_colsum_kernel<<<dim3((N + 31) / 32, T), 256, 0, s>>>(tiles, N, colsum);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    stitch_rowsum_kernel<<<dim3((N + 7) / 8, T), 256, 0, s>>>(tiles, st, N, rowsum);
    return cudaGetLastError();
}

cudaError_t launch_stitch_assemble(const float2* tiles, const StitchTile* st, const int* row_of, const int* col_of,
                                   const int* grid, int strip0, int n_cols, int N, int row0, int nrows, int cols,
                                   long long pitch, float2* out, cudaStream_t s) {
    const size_t total = size_t(nrows) * cols;
    if (total == 0) return cudaSuccess;
    const int blocks = int(std::min<size_t>((total + 255) / 256, size_t(148) * 32));
    stitch_assemble_kernel<<<blocks, 256, 0, s>>>(tiles, st, row_of, col_of, grid, strip0, n_cols, N, row0, nrows,
                                                  cols, pitch, out);
    return cudaGetLastError();
}

}  // namespace fpmk
