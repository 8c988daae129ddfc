// Which SM does each CTA of a one-wave launch land on?  (radial forward: 568 CTAs,
// 4 resident per SM.)  Prints, per SM, the block indices it received, and the
// imbalance of a heaviest-first tile order under that mapping.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cta_map tools/cta_map.cu && tools/cta_map 568
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 4) probe(int* smid, long long* t0, long long spin) {
    extern __shared__ double sm[];
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) {
        smid[blockIdx.x] = (int)id;
        t0[blockIdx.x] = t;
    }
    sm[threadIdx.x] = (double)id;
    const long long c0 = clock64();
    while (clock64() - c0 < spin) {}
    if (sm[(threadIdx.x + 1) & 127] < -1.0) smid[0] = 0;
}
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 568;
    const long long spin = argc > 2 ? atoll(argv[2]) : 40000;
    int* d_smid; long long* d_t0;
    cudaMalloc(&d_smid, n * sizeof(int)); cudaMalloc(&d_t0, n * sizeof(long long));
    const size_t smem = 46 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 3; ++rep) probe<<<n, 128, smem>>>(d_smid, d_t0, spin);
    cudaDeviceSynchronize();
    std::vector<int> smid(n); std::vector<long long> t0(n);
    cudaMemcpy(smid.data(), d_smid, n * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(t0.data(), d_t0, n * sizeof(long long), cudaMemcpyDeviceToHost);
    int maxsm = 0; for (int s : smid) maxsm = std::max(maxsm, s);
    std::vector<std::vector<int>> per(maxsm + 1);
    for (int b = 0; b < n; ++b) per[smid[b]].push_back(b);
    long long tmin = *std::min_element(t0.begin(), t0.end());
    printf("blocks %d, SM ids up to %d\n", n, maxsm);
    for (int s = 0; s <= maxsm; ++s) {
        printf("sm %3d:", s);
        for (int b : per[s]) printf(" %4d(+%lld)", b, (t0[b] - tmin) / 1000);
        printf("\n");
    }
    printf("first 300 blocks -> sm:");
    for (int b = 0; b < std::min(n, 300); ++b) printf(" %d", smid[b]);
    printf("\n");
    return 0;
}
