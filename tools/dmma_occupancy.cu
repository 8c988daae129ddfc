// DMMA (m8n8k4 .f64) throughput vs resident warps per SM and independent
// accumulator chains per warp.  Informs the GEMM tiling.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
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

template <int CH>
void run(int warps_per_sm, int sms, double* out) {
    const int iters = 2048;
    const int threads = 32 * warps_per_sm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dmma_kernel<CH><<<sms, threads>>>(out, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dmma_kernel<CH><<<sms, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flops = (double)sms * warps_per_sm * iters * CH * 512.0;
    printf("warps/SM %2d chains %2d : %6.2f TFLOP/s\n", warps_per_sm, CH, flops / best / 1e9);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    for (int w : {4, 8, 12, 16, 32}) {
        run<1>(w, sms, out); run<2>(w, sms, out); run<4>(w, sms, out); run<8>(w, sms, out); run<16>(w, sms, out);
    }
    return 0;
}
