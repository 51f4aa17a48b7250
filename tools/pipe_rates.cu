// Issue rates of the instruction classes fpm_loop64 is built from, measured on
// the B200 (full occupancy, independent chains so only throughput limits):
// FFMA (three register operands), FFMA2 (fma.rn.f32x2), FMUL, FMUL2, FADD2,
// SHFL (32-bit butterfly), LDS.128 (conflict-free). Prints warp-instructions
// per clock per SM for each. Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o pipe_rates pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
constexpr int kIters = 4096;
constexpr int kChains = 8;

__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__global__ void k_ffma(float* out, float b, float c) {
    float a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float bb = b + threadIdx.x * 1e-9f, cc = c - threadIdx.x * 1e-9f;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) a[i] = fmaf(a[i], bb, cc);
    float s = 0;
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_fmul(float* out, float b) {
    float a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
    float bb = b + threadIdx.x * 1e-9f;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) a[i] = a[i] * bb;
    float s = 0;
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float b, float c) {
    u64 a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i);
    const u64 bb = pk(b + threadIdx.x * 1e-9f, b), cc = pk(c, c - threadIdx.x * 1e-9f);
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(bb), "l"(cc));
    u64 s = 0;
    for (int i = 0; i < kChains; ++i) s ^= a[i];
    if (s == 12345ull) out[threadIdx.x] = float(s);
}

__global__ void k_fmul2(float* out, float b) {
    u64 a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i);
    const u64 bb = pk(b + threadIdx.x * 1e-9f, b);
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
    u64 s = 0;
    for (int i = 0; i < kChains; ++i) s ^= a[i];
    if (s == 12345ull) out[threadIdx.x] = float(s);
}

__global__ void k_fadd2(float* out, float b) {
    u64 a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i);
    const u64 bb = pk(b + threadIdx.x * 1e-9f, b);
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
    u64 s = 0;
    for (int i = 0; i < kChains; ++i) s ^= a[i];
    if (s == 12345ull) out[threadIdx.x] = float(s);
}

__global__ void k_shfl(float* out) {
    float a[kChains];
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < kChains; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1);
    float s = 0;
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_lds128(float* out) {
    __shared__ float4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x & 1023;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(unsigned(__cvta_generic_to_shared(buf + ((idx + 32 * i) & 1023)))));
            acc.x += v.x;
        }
        idx = (idx + 1) & 1023;
    }
    if (acc.x == 12345.f) out[threadIdx.x] = acc.x;
}

template <typename F>
void run(const char* name, F launch, int insts_per_thread_iter) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const double warps = double(sms) * 8 * 256 / 32;  // 8 blocks of 256 threads per SM
    const double winst = warps * kIters * insts_per_thread_iter;
    const double cycles = ms * 1e-3 * clk_khz * 1e3;
    printf("%-8s %8.3f ms  %6.3f warp-inst/clk/SM  (%.3f per SMSP; clock %d MHz)\n", name, ms, winst / cycles / sms,
           winst / cycles / sms / 4, clk_khz / 1000);
}

int main() {
    float* out;
    cudaMalloc(&out, 4096 * sizeof(float));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const dim3 grid(sms * 8), block(256);  // 8 resident 256-thread blocks per SM = 64 warps
    run("FFMA", [&] { k_ffma<<<grid, block>>>(out, 0.999f, 1e-3f); }, kChains);
    run("FMUL", [&] { k_fmul<<<grid, block>>>(out, 0.999f); }, kChains);
    run("FFMA2", [&] { k_ffma2<<<grid, block>>>(out, 0.999f, 1e-3f); }, kChains);
    run("FMUL2", [&] { k_fmul2<<<grid, block>>>(out, 0.999f); }, kChains);
    run("FADD2", [&] { k_fadd2<<<grid, block>>>(out, 1e-3f); }, kChains);
    run("SHFL", [&] { k_shfl<<<grid, block>>>(out); }, kChains);
    run("LDS.128", [&] { k_lds128<<<grid, block>>>(out); }, kChains);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
