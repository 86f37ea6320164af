// Can a 1-D TMA bulk copy (cp.async.bulk global -> shared) read pinned, mapped
// host memory, and how fast do 142 CTAs pull a 2.3 MB table over PCIe that way
// (vs. plain 16-B loads)?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_host_probe scripts/tma_host_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_tma(const uint8_t* src, size_t per_block, uint8_t* dst, unsigned long long* t) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint8_t* s = src + blockIdx.x * per_block;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"((uint32_t)per_block) : "memory");
        const uint32_t chunk = 16384;
        for (size_t o = 0; o < per_block; o += chunk) {
            const uint32_t n = (uint32_t)((per_block - o) < chunk ? (per_block - o) : chunk);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + o)),
                         "l"(s + o), "r"(n), "r"(smem_u32(&bar)) : "memory");
        }
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t x = 0;
    for (size_t i = threadIdx.x; i < per_block; i += blockDim.x) x += sm[i];
    if (threadIdx.x == 0) { uint64_t g; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g)); t[blockIdx.x] = g; }
    atomicAdd((unsigned*)dst, x);
}
__global__ void k_ld(const uint4* src, size_t per_block16, uint8_t* dst) {
    const uint4* s = src + blockIdx.x * per_block16;
    uint32_t x = 0;
    for (size_t i = threadIdx.x; i < per_block16; i += blockDim.x) { uint4 v = s[i]; x += v.x + v.y + v.z + v.w; }
    atomicAdd((unsigned*)dst, x);
}
int main() {
    const int B = 142;
    const size_t per = 16384;  // 142 x 16 KB = 2.3 MB
    uint8_t* h; cudaHostAlloc(&h, B * per, cudaHostAllocMapped);
    for (size_t i = 0; i < B * per; ++i) h[i] = (uint8_t)(i * 7 + 3);
    uint64_t ref = 0; for (size_t i = 0; i < B * per; ++i) ref += h[i];
    uint8_t* hd; cudaHostGetDevicePointer((void**)&hd, h, 0);
    uint8_t* d; cudaMalloc(&d, 64); unsigned long long* t; cudaMalloc(&t, B * 8);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(d, 0, 64);
        cudaEventRecord(e0); k_tma<<<B, 256, per>>>(hd, per, d, t); cudaEventRecord(e1);
        cudaError_t er = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned sum; cudaMemcpy(&sum, d, 4, cudaMemcpyDeviceToHost);
        printf("tma from host: %s  sum %s  %.1f us  %.1f GB/s\n", cudaGetErrorString(er), sum == (unsigned)ref ? "ok" : "BAD", ms * 1e3, B * per / (ms * 1e-3) / 1e9);
        if (er != cudaSuccess) return 1;
    }
    for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(d, 0, 64);
        cudaEventRecord(e0); k_ld<<<B, 256>>>((const uint4*)hd, per / 16, d); cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("ld.128 from host: %.1f us  %.1f GB/s\n", ms * 1e3, B * per / (ms * 1e-3) / 1e9);
    }
    uint8_t* dd; cudaMalloc(&dd, B * per);
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0); cudaMemcpyAsync(dd, h, B * per, cudaMemcpyHostToDevice); cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("cudaMemcpyAsync H2D: %.1f us  %.1f GB/s\n", ms * 1e3, B * per / (ms * 1e-3) / 1e9);
    }
    return 0;
}
