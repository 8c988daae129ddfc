// Memory-system ceiling for the azimuthal kernels' access pattern (B = 128): each CTA
// reads 2*IG rings (contiguous 4 KB each) and writes them as rows of G, IG consecutive
// shells per row chunk (16*IG-byte runs), through a shared-memory transpose; no FFT.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256, B = 128;

// layout 0: G[p][bin][jp][s]   (rows of all shells; chunk = IG*16 B)
// layout 1: G[p][bin][sgroup][jp][s_local] (chunk = IG*16 B, consecutive jp CTAs adjacent)
template <int IG, int LAYOUT, bool JP_FAST>
__global__ void pattern_t(const double2* __restrict__ X, double2* __restrict__ G, int nshell) {
    extern __shared__ double2 buf[];  // [2*IG][N+1]
    const int ngx = nshell / IG;
    const int gx = JP_FAST ? blockIdx.x / B : blockIdx.x % ngx;
    const int jp = JP_FAST ? blockIdx.x % B : blockIdx.x / ngx;
    const int s0 = gx * IG;
    for (int idx = threadIdx.x; idx < 2 * IG * N; idx += blockDim.x) {
        const int q = idx / N, e = idx % N;
        const int s = s0 + (q >> 1);
        const int j = (q & 1) ? (N - 1 - jp) : jp;
        buf[q * (N + 1) + e] = __ldcs(X + ((size_t)s * N + j) * N + e);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * IG * N; idx += blockDim.x) {
        const int sl = idx % IG, rowi = idx / IG;
        const int p = rowi / N, bin = rowi % N;
        long long off;
        if (LAYOUT == 0) off = (((long long)p * N + bin) * B + jp) * nshell + s0 + sl;
        else off = ((((long long)p * N + bin) * ngx + gx) * B + jp) * IG + sl;
        G[off] = buf[(2 * sl + p) * (N + 1) + bin];
    }
}

__global__ void copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

template <class F>
float timeit(F f) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    return best;
}

template <int IG, int LAYOUT, bool JPF>
void run(const double2* X, double2* G, int nshell, double bytes) {
    const size_t smem = sizeof(double2) * 2 * IG * (N + 1);
    cudaFuncSetAttribute(pattern_t<IG, LAYOUT, JPF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = IG * 32 > 512 ? 512 : IG * 32;
    float ms = timeit([&] { pattern_t<IG, LAYOUT, JPF><<<(nshell / IG) * B, threads, smem>>>(X, G, nshell); });
    printf("IG=%2d layout=%d jp_fast=%d threads=%3d : %6.1f us  %6.0f GB/s  (%s)\n", IG, LAYOUT, (int)JPF, threads,
           ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int nshell = 256;
    const size_t n = (size_t)nshell * N * N;
    double2 *X, *G;
    cudaMalloc(&X, n * 16); cudaMalloc(&G, n * 16);
    cudaMemset(X, 0, n * 16);
    const double bytes = 2.0 * n * 16;
    float ms = timeit([&] { copy<<<148 * 8, 512>>>(X, G, n); });
    printf("plain copy : %6.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
    run<4, 0, false>(X, G, nshell, bytes);
    run<8, 0, false>(X, G, nshell, bytes);
    run<16, 0, false>(X, G, nshell, bytes);
    run<4, 0, true>(X, G, nshell, bytes);
    run<4, 1, false>(X, G, nshell, bytes);
    run<4, 1, true>(X, G, nshell, bytes);
    run<8, 1, true>(X, G, nshell, bytes);
    run<16, 1, true>(X, G, nshell, bytes);
    return 0;
}
