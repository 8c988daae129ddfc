// DMMA m8n8k4 throughput vs operand register reuse: 16 accumulators per warp,
// A/B fragments either shared (register-reuse friendly) or distinct per MMA,
// in the loop orders a GEMM warp tile uses.  Informs DESIGN.md section 4.
#include <cstdio>
#include <cuda_runtime.h>

#define MMA(c, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b))

// MODE 0: same a,b for all; 1: a per row (4), b per col (4), fm-outer; 2: 8x2 tile (a 8, b 2);
// 3: 2x8 tile; 4: fm-outer with snake order on fn
template <int MODE>
__global__ void kern(double* out, int iters) {
    double a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { a[q] = threadIdx.x * 1e-3 + q; b[q] = 1.0 - threadIdx.x * 1e-4 * q; }
    double c[16][2];
#pragma unroll
    for (int q = 0; q < 16; ++q) { c[q][0] = q; c[q][1] = -q; }
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int q = 0; q < 16; ++q) MMA(c[q], a[0], b[0]);
        } else if (MODE == 1) {
#pragma unroll
            for (int fm = 0; fm < 4; ++fm)
#pragma unroll
                for (int fn = 0; fn < 4; ++fn) MMA(c[fm * 4 + fn], a[fm], b[fn]);
        } else if (MODE == 2) {
#pragma unroll
            for (int fm = 0; fm < 8; ++fm)
#pragma unroll
                for (int fn = 0; fn < 2; ++fn) MMA(c[fm * 2 + fn], a[fm], b[fn]);
        } else if (MODE == 3) {
#pragma unroll
            for (int fn = 0; fn < 2; ++fn)
#pragma unroll
                for (int fm = 0; fm < 8; ++fm) MMA(c[fn * 8 + fm], a[fm], b[fn]);
        } else {
#pragma unroll
            for (int fm = 0; fm < 4; ++fm)
#pragma unroll
                for (int f = 0; f < 4; ++f) { const int fn = (fm & 1) ? 3 - f : f; MMA(c[fm * 4 + fn], a[fm], b[fn]); }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) { a[q] += 1e-9; b[q] -= 1e-9; }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(int sms, double* out, int warps) {
    const int iters = 1024;
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
    const double flops = (double)sms * warps * iters * 16 * 512.0;
    printf("mode %d warps/SM %2d : %6.2f TFLOP/s\n", MODE, warps, flops / best / 1e9);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    for (int w : {4, 8, 12, 16}) { run<0>(sms, out, w); run<1>(sms, out, w); run<2>(sms, out, w); run<3>(sms, out, w); run<4>(sms, out, w); }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
