// k_assign.cu -- K4: capacity-constrained assignment, one CTA per resource.
//
// Resource r < I is instance r (phase A: futures pinned to it, route(session,
// agent-type, agent-instance) PAPER.md:387); resource I + t is type t (phase B:
// unpinned futures, route(agent-type, instances, weights) PAPER.md:388, with
// weights proportional to spare in exact integer water-fill form, "actively
// balances load ... through routing" PAPER.md:663).
//
// The sequential definition (admit futures in (level desc, row
// asc) order while spare remains; phase B to the most-spare instance, ties to
// the lowest id) is reproduced data-parallel from each future's GLOBAL rank in
// its resource:
//   g(f) = #{level > lv(f)} over all ranks + #{level == lv(f)} on lower ranks
//          + stable rank of f among this rank's (resource, level) bucket,
// all read from the (allreduced) histogram H[G][R][Lv].  f is admitted iff
// g(f) < bound(r) (bound = spare for phase A, sum of phase-A-residual spare over
// the type for phase B); a phase-B future takes slot g(f) of the list
// [(s, i): 1 <= s <= spare2_i] sorted by (s desc, i asc), which equals the
// sequential greedy (tests/test_oracle_pins.py::test_water_fill_*).
// Stable ranks come from scans over the row-ordered bucket lists K1 wrote;
// atomics only ever produce counts.  Admitted rows go to the resource's region
// of the assignment list (regions sized by this rank's eligible count per
// resource, offsets = prefix of K1's per-resource totals; fetch compacts).
#include "internal.h"

#include "k4_body.cuh"

namespace nalar {

// the plain epoch's build, and one with the profile stamps, resource
// reassignment (NEXT-2) and the streamed-step paths (see k4_body)
__global__ void __launch_bounds__(kK4Threads, 1) k4_assign(AssignParams p) { k4_body<false, false>(p, blockIdx.x); }
__global__ void __launch_bounds__(kK4Threads, 1) k4_assign_all(AssignParams p) { k4_body<false, true>(p, blockIdx.x); }
// the plain build plus the profile stamps (what bench.py's spans time)
__global__ void __launch_bounds__(kK4Threads, 1) k4_assign_prof(AssignParams p) { k4_body<false, false, true>(p, blockIdx.x); }


cudaError_t launch_assign(const AssignParams& p, cudaStream_t s) {
    if (p.R == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.R);
    cfg.blockDim = dim3(kK4Threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // A programmatic (PDL) launch lets K4's blocks load their static tables
    // while K1 finishes.  Released at K1's entry it measured 0.85 us slower
    // per epoch than a plain launch; released before K1's P5 (SweepParams::trig)
    // 0.6 us faster (scripts/trig_sweep.sh).  NALAR_K4_PDL=0: plain launch.
    static const bool pdl = [] { const char* e = getenv("NALAR_K4_PDL"); return !e || atoi(e) != 0; }();
    cfg.numAttrs = pdl ? 1 : 0;
    const bool all = p.ra_on || p.stream_in || p.o_status || p.o_instance || p.o_new_pin;
    if (all) return cudaLaunchKernelEx(&cfg, k4_assign_all, p);
    // diagnostics (scripts/k4_repeat.py): NALAR_K4_REPEAT=n launches the
    // (idempotent but for the stats counters) pass n times -- the later ones
    // run with K4's code already in the SMs' instruction caches
    static const int rep = [] { const char* e = getenv("NALAR_K4_REPEAT"); return e ? atoi(e) : 1; }();
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < (rep > 1 ? rep : 1) && e == cudaSuccess; ++k)
        e = p.prof ? cudaLaunchKernelEx(&cfg, k4_assign_prof, p) : cudaLaunchKernelEx(&cfg, k4_assign, p);
    return e;
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_assign() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k4_assign)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k4_assign_all)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k4_assign_prof)) return e;
    return cudaSuccess;
}

}  // namespace nalar
