// k_sweep.cu -- K1: the per-workflow sweep of the policy epoch.
//
// One CTA owns a contiguous range of whole workflows (balanced by rows on the
// host at upload).  Its slice of the SoA future table is staged into shared
// memory with 1-D TMA bulk copies (cp.async.bulk + mbarrier); each warp then
// takes whole workflows and sweeps their rows in creation order, 32 rows per
// step, computing:
//   depth  -- longest DEP u CALL path from a root (SRTF stage, PAPER.md:691;
//             SPEC S:460), saturating u16
//   doomed -- PENDING with a FAILED / doomed DEP predecessor (failures are
//             delivered like values)
//   ready  -- PENDING, not doomed, all DEP predecessors RESOLVED (push-based
//             readiness)
//   eligibility -- stateful in-order fence and first
//             placement of managed-state sessions
//   per-workflow aggregates ("aggregating metrics and metadata")
//   level  -- clamp(prio + score, 0, Lv-1) (set_priority PAPER.md:389; SRTF
//             PAPER.md:691; LPT PAPER.md:696)
//   per-instance in-flight counts (queue lengths)
// Predecessors in earlier 32-row steps are final (shared memory); those inside
// the current step are settled in rounds: a lane settles once all its in-step
// predecessors have, taking their depths by warp shuffles and their doom by
// ballots (edges point to earlier rows, so rounds = longest in-step chain).
// Finally the CTA buckets its eligible futures by resource (pin, or I + type)
// in row order -- a stable counting sort whose positions come from scans, never
// from atomics -- and adds them to the (resource, level) histogram that the
// assignment pass (and, for G > 1, the allreduce) consumes.
#include <algorithm>

#include "internal.h"

namespace nalar {

size_t k1_fixed_smem(uint32_t T, uint32_t I, uint32_t R) {
    size_t b = 64;                                  // mbarrier, ticket, counters
    b += 4 * (size_t)I;                             // in-flight counts
    b += 8 * (size_t)R;                             // per-resource count / offset
    b += 4 * (size_t)kK1Threads + 4 * kK1Warps;     // compaction list + warp counts
    b += 4 * (size_t)kP5Chunks * kK1Warps;          // per-(chunk, warp) eligible counts (P5)
    b += (size_t)T;                                 // affinity
    return (b + 127) & ~(size_t)127;
}

// The nine K1 builds live in k1_kernels.cu, compiled once per build
// (-DNALAR_K1_PART=0..8) so the objects compile in parallel.
#define NALAR_K1_DECL(NAME) __global__ void NAME(SweepParams p);
NALAR_K1_DECL(k1_sweep)
NALAR_K1_DECL(k1_sweep_x2)
NALAR_K1_DECL(k1_sweep_step)
NALAR_K1_DECL(k1_sweep_step_x2)
NALAR_K1_DECL(k1_sweep_next)
NALAR_K1_DECL(k1_sweep_next_x2)
NALAR_K1_DECL(k1_sweep_prof)
NALAR_K1_DECL(k1_sweep_x2_prof)
NALAR_K1_DECL(k1_sweep_prof_all)
#undef NALAR_K1_DECL

// clears the per-epoch exchange buffer and counters; lets the sweep launch at once
__global__ void k_zero(uint32_t* __restrict__ x, size_t n, unsigned long long* verdict) {
    asm volatile("griddepcontrol.launch_dependents;");
    // a streamed step: the sweep sets the verdict (after waiting for this grid)
    if (verdict && blockIdx.x == 0 && threadIdx.x == 0) *verdict = 0ull;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        x[i] = 0u;
}

cudaError_t launch_zero(uint32_t* x, size_t n_words, cudaStream_t s, unsigned long long* verdict) {
    const uint32_t grid = (uint32_t)std::min<size_t>(148, (n_words + 255) / 256 + 1);
    k_zero<<<grid, 256, 0, s>>>(x, n_words, verdict);
    return cudaGetLastError();
}

cudaError_t launch_sweep(const SweepParams& p_in, size_t smem, cudaStream_t s) {
    if (p_in.B == 0) return cudaSuccess;
    SweepParams p = p_in;
    // the dynamic shared-memory ceiling is a per-device function attribute
    static size_t configured_dev[64] = {};
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    size_t& configured = configured_dev[dev & 63];
    static void* const kernels[9] = {(void*)k1_sweep, (void*)k1_sweep_x2, (void*)k1_sweep_step,
                                     (void*)k1_sweep_step_x2, (void*)k1_sweep_next, (void*)k1_sweep_next_x2,
                                     (void*)k1_sweep_prof, (void*)k1_sweep_x2_prof, (void*)k1_sweep_prof_all};
    if (smem > 48 * 1024 && smem > configured) {
        for (void* k : kernels)
            if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
                return e;
        configured = smem;
    }
    // more blocks than one wave and two fit an SM: the 2-per-SM build
    static const int x2_env = [] { const char* e = getenv("NALAR_K1_X2"); return e ? atoi(e) : -1; }();
    const bool x2 = x2_env >= 0 ? x2_env != 0 : (p.B > 148u && 2 * (smem + 1024) <= 228 * 1024);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.B);
    cfg.blockDim = dim3(kK1Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool pdl = [] { const char* e = getenv("NALAR_K1_PDL"); return !e || atoi(e) != 0; }();
    cfg.numAttrs = pdl ? 1 : 0;
    p.pdl = pdl ? 1u : 0u;
    // K4's early launch is released before P5 (measured: at K1's entry the
    // early K4 blocks cost as much as they save; before P5 -0.6 us / epoch;
    // NALAR_K1_TRIGGER=0 / 1 / 2 = entry / after P2 / before P5)
    static const uint32_t trig = [] { const char* e = getenv("NALAR_K1_TRIGGER"); return e ? (uint32_t)atoi(e) : 2u; }();
    p.trig = trig;
    // the build for this epoch's modes (streamed outputs: one-wave tables only, the host checks)
    const bool out = p.o_status || p.o_level || p.o_depth || p.o_instance || p.o_new_pin;
    const bool next = p.mig_on || p.batch_head;
    int k = 0;
    if (p.prof) k = (p.stream_in || out || next) ? 8 : 6;
    else if (p.stream_in || out) k = 2;
    else if (next) k = 4;
    if (x2 && k != 8 && !(k == 2 && out)) ++k;
    void* args[] = {&p};
    return cudaLaunchKernelExC(&cfg, kernels[k], args);
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_sweep() {
    cudaFuncAttributes a;
    for (const void* k : {(const void*)k1_sweep, (const void*)k1_sweep_x2, (const void*)k1_sweep_step,
                          (const void*)k1_sweep_step_x2, (const void*)k1_sweep_next, (const void*)k1_sweep_next_x2,
                          (const void*)k1_sweep_prof, (const void*)k1_sweep_x2_prof, (const void*)k1_sweep_prof_all})
        if (cudaError_t e = cudaFuncGetAttributes(&a, k)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_zero)) return e;
    return cudaSuccess;
}

}  // namespace nalar

