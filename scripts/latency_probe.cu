// Latency floor of the pieces an epoch is built from, on the B200, as seen by
// CUDA events around a graph launch (the bench's view), L2 flushed before each
// run: an empty graph, k kernels chained (plain / PDL), dependent cold global
// loads, a grid-wide barrier, a cold 1-D bulk copy per block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/latency_probe scripts/latency_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k_empty() {}

__global__ void k_pdl_empty() {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// `hops` dependent loads of a pointer chain in global memory (one thread per block)
__global__ void k_chain(const uint32_t* __restrict__ chain, int hops, uint32_t* out) {
    if (threadIdx.x) return;
    uint32_t i = blockIdx.x * 4096u;
    for (int h = 0; h < hops; ++h) i = __ldcg(chain + i);
    out[blockIdx.x] = i;
}

// grid barrier: every block arrives at a counter, then spins until all arrived
__global__ void k_gridbar(uint32_t* ctr, uint32_t* out, int rounds) {
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t target = (uint32_t)(r + 1) * gridDim.x;
            uint32_t v;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            } while (v < target);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const uint8_t* src, uint32_t bytes, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm)), "l"(src + (size_t)blockIdx.x * bytes), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}"
                 ::"r"(smem_u32(&bar)) : "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = sm[threadIdx.x + 5];
}

static uint8_t* g_flush;
static const size_t kFlush = 256ull << 20;

template <class F>
double time_graph(cudaStream_t st, F enqueue, int reps = 200, bool flush = true) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    enqueue();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    std::vector<cudaEvent_t> ev(2 * reps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int i = 0; i < 10; ++i) CK(cudaGraphLaunch(ge, st));
    for (int i = 0; i < reps; ++i) {
        if (flush) CK(cudaMemsetAsync(g_flush, i & 0xFF, kFlush, st));
        CK(cudaEventRecord(ev[2 * i], st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(ev[2 * i + 1], st));
    }
    CK(cudaStreamSynchronize(st));
    std::vector<float> t(reps);
    for (int i = 0; i < reps; ++i) CK(cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]));
    std::sort(t.begin(), t.end());
    for (auto& e : ev) cudaEventDestroy(e);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return t[reps / 2] * 1e3;
}

template <class F>
double time_plain(cudaStream_t st, F enqueue, int reps = 200) {
    std::vector<cudaEvent_t> ev(2 * reps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int i = 0; i < 10; ++i) enqueue();
    for (int i = 0; i < reps; ++i) {
        CK(cudaMemsetAsync(g_flush, i & 0xFF, kFlush, st));
        CK(cudaEventRecord(ev[2 * i], st));
        enqueue();
        CK(cudaEventRecord(ev[2 * i + 1], st));
    }
    CK(cudaStreamSynchronize(st));
    std::vector<float> t(reps);
    double sum = 0;
    for (int i = 0; i < reps; ++i) { CK(cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1])); sum += t[i]; }
    for (auto& e : ev) cudaEventDestroy(e);
    return sum / reps * 1e3;
}

static void launch_pdl(void (*k)(), cudaStream_t st, int blocks, int threads) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k));
}

int main() {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaMalloc(&g_flush, kFlush));
    uint32_t *chain, *out, *ctr;
    const size_t chain_words = 148ull * 4096 * 2;
    CK(cudaMalloc(&chain, chain_words * 4));
    {   // chain: i -> i + 64 (distinct cache lines, same block region)
        std::vector<uint32_t> h(chain_words);
        for (size_t i = 0; i < chain_words; ++i) h[i] = (uint32_t)((i + 64) % chain_words);
        CK(cudaMemcpy(chain, h.data(), chain_words * 4, cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&out, 4096 * 4));
    CK(cudaMalloc(&ctr, 4));
    uint8_t* src;
    CK(cudaMalloc(&src, 148ull << 16));
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));

    printf("plain stream launches, event to event, MEAN of 200, L2 flushed before each (us):\n");
    printf("  1 empty kernel, 148x512             %7.2f\n", time_plain(st, [&] { k_empty<<<148, 512, 0, st>>>(); }));
    printf("  3 empty kernels, 148x512            %7.2f\n", time_plain(st, [&] { for (int j = 0; j < 3; ++j) k_empty<<<148, 512, 0, st>>>(); }));
    printf("  3 PDL kernels, 148x512              %7.2f\n", time_plain(st, [&] {
               k_empty<<<148, 512, 0, st>>>();
               for (int j = 1; j < 3; ++j) launch_pdl(k_pdl_empty, st, 148, 512); }));
    printf("graph, event to event, median of 200, L2 flushed before each (us):\n");
    printf("  1 empty kernel, 1 block             %7.2f\n", time_graph(st, [&] { k_empty<<<1, 32, 0, st>>>(); }));
    printf("  1 empty kernel, 148x512             %7.2f\n", time_graph(st, [&] { k_empty<<<148, 512, 0, st>>>(); }));
    for (int k : {2, 3, 4})
        printf("  %d empty kernels chained, 148x512   %7.2f\n", k,
               time_graph(st, [&] { for (int j = 0; j < k; ++j) k_empty<<<148, 512, 0, st>>>(); }));
    for (int k : {2, 3, 4})
        printf("  %d PDL kernels chained, 148x512     %7.2f\n", k, time_graph(st, [&] {
                   k_empty<<<148, 512, 0, st>>>();
                   for (int j = 1; j < k; ++j) launch_pdl(k_pdl_empty, st, 148, 512);
               }));
    printf("  no flush: 1 empty kernel 148x512    %7.2f\n",
           time_graph(st, [&] { k_empty<<<148, 512, 0, st>>>(); }, 200, false));
    for (int h : {1, 2, 4, 8, 16})
        printf("  %2d dependent cold loads (148 blk)  %7.2f\n", h,
               time_graph(st, [&] { k_chain<<<148, 32, 0, st>>>(chain, h, out); }));
    for (int h : {4, 16})
        printf("  %2d dependent warm loads (no flush) %7.2f\n", h,
               time_graph(st, [&] { k_chain<<<148, 32, 0, st>>>(chain, h, out); }, 200, false));
    for (int r : {1, 2, 4, 8}) {
        CK(cudaMemset(ctr, 0, 4));
        printf("  grid barrier x%d (148x512)          %7.2f\n", r, time_graph(st, [&] {
                   cudaMemsetAsync(ctr, 0, 4, st);
                   k_gridbar<<<148, 512, 0, st>>>(ctr, out, r);
               }));
    }
    for (uint32_t kb : {4u, 16u, 64u})
        printf("  cold bulk copy %2u KB per block       %7.2f\n", kb,
               time_graph(st, [&] { k_bulk<<<148, 256, kb << 10, st>>>(src, kb << 10, out); }));
    return 0;
}
