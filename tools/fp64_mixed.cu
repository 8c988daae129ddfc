// Do DMMA (tensor pipe) and DFMA (FP64 pipe) issue concurrently on sm_100a?
// Kernels: DMMA only, DFMA only, both interleaved in each warp, and warps
// specialised (even warps DMMA, odd warps DFMA).  Reports TFLOP/s per engine and
// combined; if the combined rate exceeds either alone, a contraction could split
// its k range between the two pipes.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// MODE 0: DMMA only, 1: DFMA only, 2: both in every warp, 3: warp-specialised
template <int MODE, int NM, int NF>
__global__ void mixed(double* out, int iters, double x, double y) {
    const int warp = threadIdx.x >> 5;
    const bool do_m = MODE == 0 || MODE == 2 || (MODE == 3 && (warp & 1) == 0);
    const bool do_f = MODE == 1 || MODE == 2 || (MODE == 3 && (warp & 1) == 1);
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[NM][2], f[NF];
#pragma unroll
    for (int q = 0; q < NM; ++q) { c[q][0] = q; c[q][1] = -q; }
#pragma unroll
    for (int q = 0; q < NF; ++q) f[q] = q * 0.5 + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        if (do_m) {
#pragma unroll
            for (int q = 0; q < NM; ++q) dmma(c[q], a, b);
        }
        if (do_f) {
#pragma unroll
            for (int q = 0; q < NF; ++q) f[q] = fma(f[q], x, y);
        }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < NM; ++q) s += c[q][0] + c[q][1];
#pragma unroll
    for (int q = 0; q < NF; ++q) s += f[q];
    if (s == 12345.678) out[0] = s;
}

template <class F>
float timeit(F f, int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; CK(cudaMalloc(&out, 8));
    const int iters = 4096, threads = 256, blocks = sms * 4;
    const double warps = (double)blocks * threads / 32;
    constexpr int NM = 8, NF = 16;
    const double fm = warps * iters * NM * 512.0, ff = warps * 32 * iters * NF * 2.0;  // flops per full-grid pass
    float t0 = timeit([&] { mixed<0, NM, NF><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    float t1 = timeit([&] { mixed<1, NM, NF><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    float t2 = timeit([&] { mixed<2, NM, NF><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    float t3 = timeit([&] { mixed<3, NM, NF><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    CK(cudaGetLastError());
    printf("DMMA only           : %.2f TFLOP/s\n", fm / t0 / 1e9);
    printf("DFMA only           : %.2f TFLOP/s\n", ff / t1 / 1e9);
    printf("both per warp       : %.2f TFLOP/s (DMMA %.2f + DFMA %.2f)\n", (fm + ff) / t2 / 1e9, fm / t2 / 1e9, ff / t2 / 1e9);
    printf("warp-specialised    : %.2f TFLOP/s (DMMA %.2f + DFMA %.2f)\n", (fm + ff) / 2 / t3 / 1e9,
           fm / 2 / t3 / 1e9, ff / 2 / t3 / 1e9);
    return 0;
}
