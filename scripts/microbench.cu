// Latency of the warp-collective / shared-memory ops the sweep's critical path
// uses, measured on one warp with dependent chains (SM cycles per op).
#include <cstdio>
#include <cstdint>
#define N 2048
__global__ void bench(unsigned long long* out, int seed) {
    __shared__ uint32_t sm[1024];
    const uint32_t lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    uint32_t x = lane + seed;
    long long t0, t1;
    // SHFL.IDX dependent chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xFFFFFFFFu, x, (x + lane) & 31) + 1;
    t1 = clock64(); if (lane == 0) out[0] = (t1 - t0);
    // VOTE.ANY chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x += __any_sync(0xFFFFFFFFu, (x & 3) == lane);
    t1 = clock64(); if (lane == 0) out[1] = (t1 - t0);
    // BALLOT chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x += __ballot_sync(0xFFFFFFFFu, (x & 1)) & 1;
    t1 = clock64(); if (lane == 0) out[2] = (t1 - t0);
    // MATCH.ANY chain, 8 distinct keys
    t0 = clock64();
    for (int i = 0; i < N; ++i) x += __match_any_sync(0xFFFFFFFFu, (x + lane) & 7) & 1;
    t1 = clock64(); if (lane == 0) out[3] = (t1 - t0);
    // MATCH.ANY chain, 32 distinct keys
    t0 = clock64();
    for (int i = 0; i < N; ++i) x += __match_any_sync(0xFFFFFFFFu, (x & 0xFFFF0000u) + lane) & 1;
    t1 = clock64(); if (lane == 0) out[4] = (t1 - t0);
    // REDUX max chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __reduce_max_sync(0xFFFFFFFFu, x ^ lane) + 1;
    t1 = clock64(); if (lane == 0) out[5] = (t1 - t0);
    // LDS chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = sm[(x + lane) & 1023];
    t1 = clock64(); if (lane == 0) out[6] = (t1 - t0);
    // IMNMX chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = max(x + 1u, (uint32_t)lane);
    t1 = clock64(); if (lane == 0) out[7] = (t1 - t0);
    // smem atomicMin, 32 lanes same address
    t0 = clock64();
    for (int i = 0; i < N / 8; ++i) x += atomicMin(&sm[x & 1], lane + x) & 1;
    t1 = clock64(); if (lane == 0) out[8] = (t1 - t0) * 8;
    // a settling round: K independent shuffles of the same value, max chain
    {
        uint32_t d = lane, s0 = (lane + 1) & 31, s1 = (lane + 5) & 31, s2 = (lane + 9) & 31, s3 = (lane + 17) & 31;
        t0 = clock64();
        for (int i = 0; i < N; ++i) {
            uint32_t a, b, c, e;
            asm volatile("shfl.sync.idx.b32 %0, %4, %5, 31, -1;\n\tshfl.sync.idx.b32 %1, %4, %6, 31, -1;\n\t"
                         "shfl.sync.idx.b32 %2, %4, %7, 31, -1;\n\tshfl.sync.idx.b32 %3, %4, %8, 31, -1;"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(e) : "r"(d), "r"(s0), "r"(s1), "r"(s2), "r"(s3));
            d = max(d, max(max(a, b), max(c, e)) + 1u) & 0xFFFFF;
        }
        t1 = clock64(); if (lane == 0) out[10] = (t1 - t0);
        t0 = clock64();
        for (int i = 0; i < N; ++i) {
            uint32_t a;
            asm volatile("shfl.sync.idx.b32 %0, %1, %2, 31, -1;" : "=r"(a) : "r"(d), "r"(s0));
            d = max(d, a + 1u) & 0xFFFFF;
        }
        t1 = clock64(); if (lane == 0) out[11] = (t1 - t0);
        x += d;
    }
    if (lane == 0) out[9] = x;
}
// the 4-shuffle settling round with W warps on one SM (all busy): cycles per round per warp
__global__ void contention(unsigned long long* out, int nshfl) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t d = lane, s0 = (lane + 1) & 31, s1 = (lane + 5) & 31, s2 = (lane + 9) & 31, s3 = (lane + 17) & 31;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        uint32_t a, b, c, e;
        asm volatile("shfl.sync.idx.b32 %0, %4, %5, 31, -1;\n\tshfl.sync.idx.b32 %1, %4, %6, 31, -1;\n\t"
                     "shfl.sync.idx.b32 %2, %4, %7, 31, -1;\n\tshfl.sync.idx.b32 %3, %4, %8, 31, -1;"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(e) : "r"(d), "r"(s0), "r"(s1), "r"(s2), "r"(s3));
        d = max(d, max(max(a, b), max(c, e)) + 1u) & 0xFFFFF;
        if (nshfl == 8) {
            asm volatile("shfl.sync.idx.b32 %0, %4, %5, 31, -1;\n\tshfl.sync.idx.b32 %1, %4, %6, 31, -1;\n\t"
                         "shfl.sync.idx.b32 %2, %4, %7, 31, -1;\n\tshfl.sync.idx.b32 %3, %4, %8, 31, -1;"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(e) : "r"(d ^ 1u), "r"(s0), "r"(s1), "r"(s2), "r"(s3));
            d = max(d, max(max(a, b), max(c, e))) & 0xFFFFF;
        }
    }
    const long long t1 = clock64();
    if (lane == 0) out[warp] = (t1 - t0) + (d == 12345u);
}
int main() {
    unsigned long long* d; unsigned long long h[12];
    cudaMalloc(&d, 96);
    bench<<<1, 32>>>(d, 1); cudaDeviceSynchronize();
    bench<<<1, 32>>>(d, 2); cudaMemcpy(h, d, 96, cudaMemcpyDeviceToHost);
    const char* nm[] = {"shfl.idx", "vote.any", "ballot", "match.any(8 keys)", "match.any(32 keys)", "redux.max", "lds", "imnmx", "atom.shared.min(32-way)"};
    for (int i = 0; i < 9; ++i) printf("%-26s %7.1f cycles/op\n", nm[i], (double)h[i] / N);
    printf("%-26s %7.1f cycles/round\n", "round: 4 shfl + max chain", (double)h[10] / N);
    printf("%-26s %7.1f cycles/round\n", "round: 1 shfl + max", (double)h[11] / N);
    unsigned long long* c; cudaMalloc(&c, 32 * 8);
    for (int ns = 4; ns <= 8; ns += 4)
        for (int W = 1; W <= 32; W *= 2) {
            contention<<<1, 32 * W>>>(c, ns); cudaDeviceSynchronize();
            contention<<<1, 32 * W>>>(c, ns);
            unsigned long long hc[32]; cudaMemcpy(hc, c, 8 * W, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0; for (int w = 0; w < W; ++w) mx = hc[w] > mx ? hc[w] : mx;
            printf("contention: %d shfl/round, %2d warps: %7.1f cycles/round (slowest warp)\n", ns, W, (double)mx / N);
        }
    return 0;
}
