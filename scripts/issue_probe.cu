// Per-warp issue cost of the ops on K1's dependent chains (one warp alone on
// the SM, SM cycles per iteration): how many shuffles / shared loads / votes a
// step can afford.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/issue_probe scripts/issue_probe.cu
#include <cstdio>
#include <cstdint>
#define N 1024
__global__ void probe(unsigned long long* out, int seed) {
    __shared__ uint32_t sm[2048];
    __shared__ uint16_t flag[64];
    const uint32_t lane = threadIdx.x;
    for (int i = lane; i < 2048; i += 32) sm[i] = (i * 7 + 1) & 2047;
    if (lane < 64) flag[lane] = 0x4000;
    __syncwarp();
    uint32_t x = lane + seed;
    long long t0, t1;
    int o = 0;
#define T0 t0 = clock64();
#define T1(n) t1 = clock64(); if (lane == 0) out[o] = (t1 - t0); ++o;
    // 8 independent shuffles then combine (per-warp shuffle throughput)
    T0 for (int i = 0; i < N; ++i) {
        uint32_t a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __shfl_sync(0xFFFFFFFFu, x + j, (lane + j * 5) & 31);
        x = (a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7]) & 0xFFFF;
    } T1(0)
    // 8 independent LDS, per-lane random addresses
    T0 for (int i = 0; i < N; ++i) {
        uint32_t a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = sm[(x + lane * 33 + j * 97) & 2047];
        x = (a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7]) & 0xFFFF;
    } T1(1)
    // 8 independent broadcast LDS (same address in every lane)
    T0 for (int i = 0; i < N; ++i) {
        uint32_t a[8];
        const uint32_t u = __shfl_sync(0xFFFFFFFFu, x, 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = sm[(u + j * 97) & 2047];
        x = (a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7]) & 0xFFFF;
    } T1(2)
    // 8 independent ballots
    T0 for (int i = 0; i < N; ++i) {
        uint32_t a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __ballot_sync(0xFFFFFFFFu, ((x >> j) ^ lane) & 1);
        x = (a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7]) & 0xFFFF;
    } T1(3)
    // STS + syncwarp + LDS round trip (one value through shared memory)
    T0 for (int i = 0; i < N; ++i) {
        sm[lane] = x;
        __syncwarp();
        x = sm[(x + 1) & 31] + 1;
        __syncwarp();
    } T1(4)
    // ld.acquire.cta.b16 (generic address) chain on shared memory
    T0 for (int i = 0; i < N; ++i) {
        uint16_t v;
        asm volatile("ld.acquire.cta.b16 %0, [%1];" : "=h"(v) : "l"(flag + (x & 31)) : "memory");
        x += v & 1;
    } T1(5)
    // plain LDS.U16 chain on the same words
    T0 for (int i = 0; i < N; ++i) { x += flag[x & 31] & 1; } T1(6)
    // __syncwarp alone
    T0 for (int i = 0; i < N; ++i) { x += lane; __syncwarp(); } T1(7)
    // 32 shuffles + 32-step closure (doom_closure's body)
    T0 for (int i = 0; i < N / 8; ++i) {
        uint32_t D = __ballot_sync(0xFFFFFFFFu, (x ^ lane) & 1) | 1u;
        uint32_t nj[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) nj[j] = __shfl_sync(0xFFFFFFFFu, x * lane, j);
#pragma unroll
        for (int j = 0; j < 32; ++j) D |= (nj[j] & D) ? 1u << j : 0u;
        x += (D >> lane) & 1;
    } T1(8)
    // the 32-step closure with masks from shared memory (32 broadcast LDS)
    T0 for (int i = 0; i < N / 8; ++i) {
        uint32_t D = __ballot_sync(0xFFFFFFFFu, (x ^ lane) & 1) | 1u;
        sm[lane] = x * lane;
        __syncwarp();
        uint32_t nj[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) nj[j] = sm[j];
#pragma unroll
        for (int j = 0; j < 32; ++j) D |= (nj[j] & D) ? 1u << j : 0u;
        x += (D >> lane) & 1;
        __syncwarp();
    } T1(9)
    // 4 x LDS.128 broadcast (32 words) + closure
    T0 for (int i = 0; i < N / 8; ++i) {
        uint32_t D = __ballot_sync(0xFFFFFFFFu, (x ^ lane) & 1) | 1u;
        sm[lane] = x * lane;
        __syncwarp();
        uint4 q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = reinterpret_cast<const uint4*>(sm)[j];
        const uint32_t* nj = reinterpret_cast<const uint32_t*>(q);
#pragma unroll
        for (int j = 0; j < 32; ++j) D |= (nj[j] & D) ? 1u << j : 0u;
        x += (D >> lane) & 1;
        __syncwarp();
    } T1(10)
    if (lane == 0) out[31] = x;
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 32 * 8);
    probe<<<1, 32>>>(d, 1); cudaDeviceSynchronize();
    probe<<<1, 32>>>(d, 2); cudaDeviceSynchronize();
    unsigned long long h[32]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const char* nm[] = {"8 indep shfl + xor", "8 indep lds (random)", "8 indep lds (broadcast) + 1 shfl",
                        "8 indep ballots", "sts+syncwarp+lds+syncwarp", "ld.acquire.cta.b16 chain",
                        "lds.u16 chain", "syncwarp", "doom closure (32 shfl + 32-step walk)",
                        "doom closure (sts + 32 lds + walk)", "doom closure (sts + 8 lds.128 + walk)"};
    for (int i = 0; i < 11; ++i) printf("%-42s %7.1f cycles/iter\n", nm[i], h[i] / (double)(i >= 8 ? 1024 / 8 : 1024));
    return 0;
}
