// tcgen05 kind::i8 probe (sm_100a): one 128 x N x K int8 GEMM per CTA from
// shared-memory operands in the K-major no-swizzle canonical layout, int32
// accumulators in TMEM read back with tcgen05.ld; checked against a CPU
// product, then timed as a throughput loop (MMAs on resident operands) to get the
// B200 INT8 tensor rate that an FP64-by-integer-slices contraction would run at.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_umma tools/i8_umma.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrices of 8 rows x 16 bytes; element (r, k) of an
// R-row operand at [k / 16][r][k % 16] -> LBO (next 16-byte k chunk) = R * 16,
// SBO (next 8-row group) = 128.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // sm_100 descriptor version
    return d;                // base offset 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
    return (2u << 4)                      // D: s32
           | ((a_signed ? 1u : 0u) << 7)  // A: s8 / u8
           | ((b_signed ? 1u : 0u) << 10) // B
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_i8_warp(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// mode 0: single-thread issue, SS; 1: warp issue (elect), SS; 2: warp issue, A from TMEM (TS)
template <int N, int K>
__global__ void __launch_bounds__(128, 1) umma_i8_kernel(const int8_t* A, const int8_t* Bm, int* D, int reps, int asg, int bsg, int mode) {
    constexpr int M = 128;
    constexpr int kCols = (N + K / 4) <= 32 ? 32 : (N + K / 4) <= 64 ? 64 : (N + K / 4) <= 128 ? 128 : (N + K / 4) <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sa = sm;                 // M * K bytes
    uint8_t* sb = sm + M * K;         // N * K bytes
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int8_t* Ab = A + (size_t)blockIdx.x * M * K;
    for (int e = tid; e < M * K; e += 128) {
        const int r = e / K, k = e % K;
        sa[(k >> 4) * (M * 16) + r * 16 + (k & 15)] = (uint8_t)Ab[e];
    }
    for (int e = tid; e < N * K; e += 128) {
        const int r = e / K, k = e % K;
        sb[(k >> 4) * (N * 16) + r * 16 + (k & 15)] = (uint8_t)Bm[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem stores -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t td = tmem_base;
    if (mode == 2) {  // A -> TMEM columns [N, N + K/4): lane = row, 4 int8 per column
        const int row = warp * 32 + (tid & 31);
        const int8_t* ar = Ab + (size_t)row * K;
#pragma unroll
        for (int c0 = 0; c0 < K / 4; c0 += 8) {
            uint32_t w[8];
            for (int j = 0; j < 8; ++j) w[j] = *reinterpret_cast<const uint32_t*>(ar + 4 * (c0 + j));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                         ::"r"(td + ((uint32_t)(warp * 32) << 16) + N + c0), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]),
                           "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (mode == 0 && tid == 0) {
        const uint32_t id = idesc_i8(M, N, asg, bsg);
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int ks = 0; ks < K / 32; ++ks) {
                const uint64_t da = sdesc(a0 + ks * 2 * (M * 16), M * 16, 128);
                const uint64_t db = sdesc(b0 + ks * 2 * (N * 16), N * 16, 128);
                mma_i8(td, da, db, id, (r | ks) ? 1u : 0u);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    }
    if (mode != 0 && warp == 0) {
        const uint32_t id = idesc_i8(M, N, asg, bsg);
        const uint64_t da0 = sdesc(smem_u32(sa), M * 16, 128), db0 = sdesc(smem_u32(sb), N * 16, 128);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int ks = 0; ks < K / 32; ++ks) {
                if (mode == 1) mma_i8_warp(td, da0 + ks * 2 * M, db0 + ks * 2 * N, id, (r | ks) ? 1u : 0u);
                else mma_i8_ts(td, td + N + ks * 8, db0 + ks * 2 * N, id, (r | ks) ? 1u : 0u);
            }
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMAs
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(done) : "r"(smem_u32(&bar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    int* Db = D + (size_t)blockIdx.x * M * N;
    const int row = warp * 32 + (tid & 31);
#pragma unroll
    for (int c = 0; c < N; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(td + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        for (int j = 0; j < 16; ++j) Db[(size_t)row * N + c + j] = (int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(td), "r"(kCols));
}

template <int N, int K>
static int run(int asg, int bsg, int ctas, int reps_time, int mode = 0) {
    constexpr int M = 128;
    std::vector<int8_t> A((size_t)ctas * M * K), Bm((size_t)N * K);
    srand(1);
    for (auto& x : A) x = (int8_t)(asg ? (rand() % 255) - 127 : (rand() % 256));
    for (auto& x : Bm) x = (int8_t)(bsg ? (rand() % 255) - 127 : (rand() % 256));
    int8_t *dA, *dB;
    int* dD;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, Bm.size()));
    CK(cudaMalloc(&dD, (size_t)ctas * M * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bm.data(), Bm.size(), cudaMemcpyHostToDevice));
    const size_t smem = (size_t)(M + N) * K;
    CK(cudaFuncSetAttribute(umma_i8_kernel<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    umma_i8_kernel<N, K><<<ctas, 128, smem>>>(dA, dB, dD, 1, asg, bsg, mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int> D((size_t)ctas * M * N);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int c = 0; c < ctas; c += (ctas > 4 ? ctas / 4 : 1))
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long s = 0;
                for (int k = 0; k < K; ++k) {
                    const int a = asg ? (int)A[(size_t)c * M * K + i * K + k] : (int)(uint8_t)A[(size_t)c * M * K + i * K + k];
                    const int b = bsg ? (int)Bm[j * K + k] : (int)(uint8_t)Bm[j * K + k];
                    s += (long)a * b;
                }
                if (s != D[(size_t)c * M * N + i * N + j]) {
                    if (bad < 5) printf("  mismatch c%d (%d,%d): %ld vs %d\n", c, i, j, s, D[(size_t)c * M * N + i * N + j]);
                    ++bad;
                }
            }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    umma_i8_kernel<N, K><<<ctas, 128, smem>>>(dA, dB, dD, reps_time, asg, bsg, mode);
    CK(cudaEventRecord(e0));
    umma_i8_kernel<N, K><<<ctas, 128, smem>>>(dA, dB, dD, reps_time, asg, bsg, mode);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ops = 2.0 * M * N * K * (double)reps_time * ctas;
    printf("mode %d M=128 N=%d K=%d a%s b%s: %s (%ld bad); %d CTAs x %d reps: %.3f ms, %.1f TOPS\n", mode, N, K, asg ? "s8" : "u8",
           bsg ? "s8" : "u8", bad ? "WRONG" : "exact", bad, ctas, reps_time, ms, ops / ms / 1e9);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return bad ? 1 : 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int fails = 0;
    for (int mode = 0; mode < 3; ++mode) {
        fails += run<64, 128>(1, 0, 4, 1, mode);
        fails += run<32, 64>(0, 1, 4, 1, mode);
        fails += run<16, 128>(0, 0, sms, 8000, mode);
        fails += run<32, 128>(0, 1, sms, 8000, mode);
        fails += run<64, 128>(0, 1, sms, 4000, mode);
        fails += run<128, 128>(1, 1, sms, 2000, mode);
        fails += run<256, 128>(1, 1, sms, 1000, mode);
    }
    printf("%s\n", fails ? "FAILED" : "all exact");
    return fails;
}
