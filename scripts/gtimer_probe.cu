// Is %globaltimer consistent with clock64 inside one thread?  Spin N cycles
// between two reads of each, in every SM at once.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory"); return t; }
__global__ void k(unsigned long long* out, long long spin) {
    if (threadIdx.x) return;
    uint64_t g0 = gt(); long long c0 = clock64();
    while (clock64() - c0 < spin) {}
    uint64_t g1 = gt(); long long c1 = clock64();
    out[blockIdx.x * 2] = g1 - g0; out[blockIdx.x * 2 + 1] = c1 - c0;
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 16);
    unsigned long long h[296];
    for (long long spin : {100LL, 2000LL, 20000LL, 200000LL}) {
        for (int rep = 0; rep < 3; ++rep) {
            k<<<148, 32>>>(d, spin); cudaMemcpy(h, d, 148 * 16, cudaMemcpyDeviceToHost);
            unsigned long long gmin = ~0ull, gmax = 0, cmax = 0;
            for (int b = 0; b < 148; ++b) { gmin = h[2*b] < gmin ? h[2*b] : gmin; gmax = h[2*b] > gmax ? h[2*b] : gmax; cmax = h[2*b+1] > cmax ? h[2*b+1] : cmax; }
            printf("spin %lld cycles: globaltimer delta ns min %llu max %llu, clock max %llu\n", spin, gmin, gmax, cmax);
        }
    }
    return 0;
}
