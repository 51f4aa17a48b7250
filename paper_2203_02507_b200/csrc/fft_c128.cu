// Batched 2-D complex128 FFTs of any size whose factors are 2, 3 and 5 — the
// transforms of the GPU forward model (simulate_dataset, forward.cpp:172-282),
// whose guard-banded tile grids are 96 / 120 / 384 / 480 / 512 ... points per
// side. Not on the reconstruction path (that runs the FP32
// kernels of kernels*.cu); FP64 here because the forward model quantises to
// u16 and must reproduce the double-precision oracle's frames.
//
// One CTA per line: a Stockham autosort over shared memory (radix 4, 2, 3, 5
// passes, twiddles from sincospi in double), lines contiguous; the columns run
// as rows of a tiled transpose. Forward unnormalised; inverse scaled by
// 1 / (rows cols) (the conventions of numpy / torch.fft and of the reference's
// Eigen FFT, field.cpp:64-66).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

namespace fpmk {

namespace {

__device__ __forceinline__ double2 z_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 z_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 z_mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 z_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) / +i (inverse)
__device__ __forceinline__ double2 z_mi(double2 a, bool inv) { return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x); }

// small DFTs of radix R on x[0..R), sign by inv
template <int R>
__device__ __forceinline__ void dft_small(double2 (&x)[5], bool inv) {
    if constexpr (R == 2) {
        const double2 a = x[0], b = x[1];
        x[0] = z_add(a, b);
        x[1] = z_sub(a, b);
    } else if constexpr (R == 4) {
        const double2 s02 = z_add(x[0], x[2]), d02 = z_sub(x[0], x[2]);
        const double2 s13 = z_add(x[1], x[3]), d13 = z_mi(z_sub(x[1], x[3]), inv);
        x[0] = z_add(s02, s13);
        x[2] = z_sub(s02, s13);
        x[1] = z_add(d02, d13);
        x[3] = z_sub(d02, d13);
    } else if constexpr (R == 3) {
        const double c = -0.5, s = inv ? 0.86602540378443864676 : -0.86602540378443864676;
        const double2 t = z_add(x[1], x[2]), u = z_sub(x[1], x[2]);
        const double2 m = make_double2(x[0].x + c * t.x, x[0].y + c * t.y);
        const double2 r = make_double2(-s * u.y, s * u.x);  // i s u
        x[0] = z_add(x[0], t);
        x[1] = z_add(m, r);
        x[2] = z_sub(m, r);
    } else {  // R == 5: direct with exact-enough constants
        const double sg = inv ? 1.0 : -1.0;
        double2 y[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            double2 acc = x[0];
#pragma unroll
            for (int t = 1; t < 5; ++t) {
                double sn, cs;
                sincospi(sg * 2.0 * double((k * t) % 5) / 5.0, &sn, &cs);
                acc = z_add(acc, z_mul(x[t], make_double2(cs, sn)));
            }
            y[k] = acc;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) x[k] = y[k];
    }
}

template <int R>
__device__ __forceinline__ void stockham_pass(const double2* src, double2* dst, int L, int Ns, bool inv) {
    const int m = L / R;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const int k = j % Ns;
        double2 x[5];
#pragma unroll
        for (int t = 0; t < R; ++t) x[t] = src[j + t * m];
        if (Ns > 1) {
#pragma unroll
            for (int t = 1; t < R; ++t) {
                double sn, cs;
                sincospi((inv ? 2.0 : -2.0) * double(t * k) / double(Ns * R), &sn, &cs);
                x[t] = z_mul(x[t], make_double2(cs, sn));
            }
        }
        dft_small<R>(x, inv);
        double2* out = dst + (j / Ns) * Ns * R + k;
#pragma unroll
        for (int t = 0; t < R; ++t) out[t * Ns] = x[t];
    }
}

// radices: up to 16 passes packed 4 bits each (values 2, 3, 4, 5)
__global__ void fft_lines_c128(double2* data, int L, unsigned long long radices, int npass, int inv, double scale) {
    extern __shared__ double2 zbuf[];
    double2* a = zbuf;
    double2* b = zbuf + L;
    double2* line = data + size_t(blockIdx.x) * L;
    for (int i = threadIdx.x; i < L; i += blockDim.x) a[i] = line[i];
    __syncthreads();
    int Ns = 1;
    for (int p = 0; p < npass; ++p) {
        const int r = int((radices >> (4 * p)) & 15ull);
        switch (r) {
            case 2: stockham_pass<2>(a, b, L, Ns, inv != 0); break;
            case 3: stockham_pass<3>(a, b, L, Ns, inv != 0); break;
            case 4: stockham_pass<4>(a, b, L, Ns, inv != 0); break;
            default: stockham_pass<5>(a, b, L, Ns, inv != 0); break;
        }
        __syncthreads();
        Ns *= r;
        double2* t = a;
        a = b;
        b = t;
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) line[i] = scale == 1.0 ? a[i] : z_scale(a[i], scale);
}

// [batch][rows][cols] -> [batch][cols][rows], 32 x 32 tiles through shared memory
__global__ void transpose_c128(const double2* __restrict__ src, double2* __restrict__ dst, int rows, int cols) {
    __shared__ double2 tile[32][33];
    const size_t off = size_t(blockIdx.z) * rows * cols;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int r = r0 + dy, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[dy][threadIdx.x] = src[off + size_t(r) * cols + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int c = c0 + dy, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[off + size_t(c) * rows + r] = tile[threadIdx.x][dy];
    }
}

bool plan_radices(int L, unsigned long long* packed, int* npass) {
    if (L < 1 || L > 4096) return false;  // two lines of shared memory: <= 128 KB
    std::vector<int> rs;
    int m = L;
    while (m % 4 == 0) {
        rs.push_back(4);
        m /= 4;
    }
    while (m % 2 == 0) {
        rs.push_back(2);
        m /= 2;
    }
    while (m % 3 == 0) {
        rs.push_back(3);
        m /= 3;
    }
    while (m % 5 == 0) {
        rs.push_back(5);
        m /= 5;
    }
    if (m != 1 || rs.size() > 16) return false;
    unsigned long long p = 0;
    for (size_t i = 0; i < rs.size(); ++i) p |= (unsigned long long)(rs[i]) << (4 * i);
    *packed = p;
    *npass = int(rs.size());
    return true;
}

cudaError_t lines(double2* data, int L, long long nlines, bool inv, double scale, cudaStream_t s) {
    unsigned long long rad = 0;
    int np = 0;
    if (!plan_radices(L, &rad, &np)) return cudaErrorNotSupported;
    if (L == 1) return cudaSuccess;
    const size_t smem = size_t(2) * L * sizeof(double2);
    cudaError_t e = cudaFuncSetAttribute(fft_lines_c128, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    for (long long b0 = 0; b0 < nlines; b0 += 65535) {  // grid.x limit
        const int cnt = int(std::min<long long>(65535, nlines - b0));
        fft_lines_c128<<<cnt, 256, smem, s>>>(data + size_t(b0) * L, L, rad, np, inv ? 1 : 0, scale);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t transpose(const double2* src, double2* dst, int rows, int cols, long long batch, cudaStream_t s) {
    for (long long b0 = 0; b0 < batch; b0 += 65535) {
        const int cnt = int(std::min<long long>(65535, batch - b0));
        const dim3 grid((cols + 31) / 32, (rows + 31) / 32, cnt);
        transpose_c128<<<grid, dim3(32, 8), 0, s>>>(src + size_t(b0) * rows * cols, dst + size_t(b0) * rows * cols,
                                                     rows, cols);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

bool fft_c128_supported(int n) {
    unsigned long long r;
    int np;
    return plan_radices(n, &r, &np);
}

// in place on data [batch][rows][cols]; tmp: batch * rows * cols elements of scratch
cudaError_t fft2_c128(double2* data, double2* tmp, long long batch, int rows, int cols, bool inv, cudaStream_t s) {
    cudaError_t e = lines(data, cols, batch * rows, inv, 1.0, s);
    if (e != cudaSuccess) return e;
    if ((e = transpose(data, tmp, rows, cols, batch, s)) != cudaSuccess) return e;
    if ((e = lines(tmp, rows, batch * cols, inv, inv ? 1.0 / (double(rows) * cols) : 1.0, s)) != cudaSuccess) return e;
    return transpose(tmp, data, cols, rows, batch, s);
}

}  // namespace fpmk
