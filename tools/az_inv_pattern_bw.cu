// Memory-system ceiling for the inverse azimuthal access pattern (B = 128): each CTA
// gathers IG-shell chunks of the G rows (p, bin, jp) and writes 2*IG contiguous rings.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256, B = 128;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}

template <int IG, bool ASYNC>
__global__ void pattern_inv(const double2* __restrict__ G, double2* __restrict__ X, int nshell) {
    extern __shared__ double2 buf[];  // [2*IG][N+1]
    const int ngx = nshell / IG;
    const int gx = blockIdx.x % ngx, jp = blockIdx.x / ngx;
    const int s0 = gx * IG;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < 2 * IG * N; idx += blockDim.x) {
        const int sl = idx % IG, rowi = idx / IG;
        const int p = rowi / N, bin = rowi % N;
        const double2* src = G + (((long long)p * N + bin) * B + jp) * nshell + s0 + sl;
        if (ASYNC) cp_async16(&buf[(2 * sl + p) * (N + 1) + bin], src);
        else buf[(2 * sl + p) * (N + 1) + bin] = __ldcs(src);
    }
    if (ASYNC) asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * IG * N; idx += blockDim.x) {
        const int q = idx / N, e = idx % N;
        const int s = s0 + (q >> 1);
        const int j = (q & 1) ? (N - 1 - jp) : jp;
        __stcs(X + ((size_t)s * N + j) * N + e, buf[q * (N + 1) + e]);
    }
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

template <int IG, bool ASYNC>
void run(const double2* G, double2* X, int nshell, double bytes) {
    const size_t smem = sizeof(double2) * 2 * IG * (N + 1);
    cudaFuncSetAttribute(pattern_inv<IG, ASYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = IG * 32 > 512 ? 512 : IG * 32;
    float ms = timeit([&] { pattern_inv<IG, ASYNC><<<(nshell / IG) * B, threads, smem>>>(G, X, nshell); });
    printf("inverse IG=%2d async=%d : %6.1f us  %6.0f GB/s (%s)\n", IG, (int)ASYNC, ms * 1e3, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int nshell = 256;
    const size_t n = (size_t)nshell * N * N;
    double2 *X, *G;
    cudaMalloc(&X, n * 16); cudaMalloc(&G, n * 16);
    cudaMemset(G, 0, n * 16);
    const double bytes = 2.0 * n * 16;
    run<4, true>(G, X, nshell, bytes);
    run<8, true>(G, X, nshell, bytes);
    run<16, true>(G, X, nshell, bytes);
    run<4, false>(G, X, nshell, bytes);
    run<8, false>(G, X, nshell, bytes);
    return 0;
}
