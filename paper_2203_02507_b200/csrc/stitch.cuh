// Device side of the Eq. (1) mosaic (stitch.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

namespace fpmk {

struct StitchTile {
    int X, Y;            // HR origin of the tile in the mosaic
    int own_c0, own_c1;  // tile columns this tile owns in its strip, [c0, c1)
    float fre, fim;      // final complex factor S_strip * R_t
};

// colsum [T][N] and rowsum [T][N] complex128 (rowsum over the owned columns).
cudaError_t launch_stitch_sums(const float2* tiles, const StitchTile* st, int T, int N, double* colsum,
                               double* rowsum, cudaStream_t s);
// rows [row0, row0 + nrows) of the mosaic; grid = the band's strips from strip0
cudaError_t launch_stitch_assemble(const float2* tiles, const StitchTile* st, const int* row_of, const int* col_of,
                                   const int* grid, int strip0, int n_cols, int N, int row0, int nrows, int cols,
                                   long long pitch, float2* out, cudaStream_t s);

}  // namespace fpmk
