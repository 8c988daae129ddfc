// FP64 peak microbenchmarks on sm_100a: DFMA (CUDA cores) vs DMMA (mma.sync .f64).
// Each kernel runs ITER iterations of independent accumulator chains; reports TFLOP/s
// from cudaEvent timing.  Used once to pick the contraction engine.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 12345.678) out[0] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C/D 2 regs
template <int CH>
__global__ void dmma884_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[CH][2];
#pragma unroll
    for (int q = 0; q < CH; ++q) { c[q][0] = q; c[q][1] = -q; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.678) out[0] = s;
}

// m16n8k4: A 2 regs, B 1 reg, C/D 4 regs
template <int CH>
__global__ void dmma1684_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
    double c[CH][4];
#pragma unroll
    for (int q = 0; q < CH; ++q) { c[q][0] = q; c[q][1] = -q; c[q][2] = q; c[q][3] = 1; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 12345.678) out[0] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C/D 4 regs
template <int CH>
__global__ void dmma16816_kernel(double* out, int iters) {
    double a[8], b[4];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = 1.0 - threadIdx.x * 1e-4 * q;
    double c[CH][4];
#pragma unroll
    for (int q = 0; q < CH; ++q) { c[q][0] = q; c[q][1] = -q; c[q][2] = q; c[q][3] = 1; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                         : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
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
    const int iters = 4096;
    for (int blocksPerSM : {2, 4, 8}) {
        const int threads = 256, blocks = sms * blocksPerSM;
        const double tot = (double)blocks * threads * iters;
        float ms = timeit([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
        printf("DFMA  bps=%d: %.2f TFLOP/s\n", blocksPerSM, tot * 8 * 2 / ms / 1e9);
        ms = timeit([&] { dmma884_kernel<8><<<blocks, threads>>>(out, iters); });
        printf("DMMA m8n8k4   bps=%d: %.2f TFLOP/s\n", blocksPerSM, tot / 32 * 8 * 512 / ms / 1e9);
        ms = timeit([&] { dmma1684_kernel<4><<<blocks, threads>>>(out, iters); });
        printf("DMMA m16n8k4  bps=%d: %.2f TFLOP/s\n", blocksPerSM, tot / 32 * 4 * 1024 / ms / 1e9);
        ms = timeit([&] { dmma16816_kernel<4><<<blocks, threads>>>(out, iters / 4); });
        printf("DMMA m16n8k16 bps=%d: %.2f TFLOP/s\n", blocksPerSM, tot / 4 / 32 * 4 * 4096 / ms / 1e9);
    }
    CK(cudaGetLastError());
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer of double2
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    float ms = timeit([&] { copy_kernel<<<sms * 8, 512>>>(a, b, n); });
    printf("copy double2: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
    return 0;
}
