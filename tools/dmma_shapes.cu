// Distinct-operand DMMA throughput for warp tiles built from m8n8k4 vs m16n8k16
// (per warp 32 x 32 and 64 x 32 output tiles).  Informs the GEMM inner loop.
#include <cstdio>
#include <cuda_runtime.h>

#define MMA884(c, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b))
#define MMA16816(c, a, b) asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n" \
    : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]))
#define MMA1684(c, a, b) asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n" \
    : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b))

// mode 0: 32x32 warp tile, m8n8k4, one k4 step per iteration (16 MMA)
// mode 1: 32x32 warp tile, m16n8k16 (2x4 MMAs = 64 DMMA-equivalents per k16)
// mode 2: 32x32 warp tile, m16n8k4 (2x4 MMAs per k4 = 16 equivalents)
// mode 3: 64x32 warp tile, m8n8k4 (8x4 = 32 MMA per k4)
template <int MODE>
__global__ void kern(double* out, int iters) {
    double acc[32][2];
#pragma unroll
    for (int q = 0; q < 32; ++q) { acc[q][0] = q; acc[q][1] = -q; }
    double a[16], b[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) { a[q] = threadIdx.x * 1e-3 + q; b[q] = 1.0 - threadIdx.x * 1e-4 * q; }
    long long mmas = 0;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int fm = 0; fm < 4; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) MMA884(acc[fm * 4 + fn], a[fm], b[fn]);
        } else if (MODE == 1) {
#pragma unroll
            for (int fm = 0; fm < 2; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) MMA16816((&acc[(fm * 4 + fn) * 2][0]), (&a[fm * 8]), (&b[fn * 4]));
        } else if (MODE == 2) {
#pragma unroll
            for (int fm = 0; fm < 2; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) MMA1684((&acc[(fm * 4 + fn) * 2][0]), (&a[fm * 2]), b[fn]);
        } else {
#pragma unroll
            for (int fm = 0; fm < 8; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) MMA884(acc[fm * 4 + fn], a[fm], b[fn]);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) { a[q] += 1e-9; b[q] -= 1e-9; }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) s += acc[q][0] + acc[q][1];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(int sms, double* out, int warps) {
    const int iters = 512;
    const double per_iter = MODE == 0 ? 16 : MODE == 1 ? 64 : MODE == 2 ? 16 : 32;  // DMMA.8x8x4 equivalents
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<MODE><<<sms * (warps / 4), 128>>>(out, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<MODE><<<sms * (warps / 4), 128>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flops = (double)sms * warps * iters * per_iter * 512.0;
    printf("mode %d warps/SM %2d : %6.2f TFLOP/s  (%s)\n", MODE, warps, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    for (int w : {4, 8, 16}) { run<0>(sms, out, w); run<1>(sms, out, w); run<2>(sms, out, w); run<3>(sms, out, w); }
    return 0;
}
