// k_batch.cu -- K6: batch coalescing of this epoch's assignments (SURVEY §8(f)
// NEXT-4; DESIGN.md Q-batch, oracle step O12).
//
// "if an agent supports batching ... Nalar can coalesce compatible futures and
// execute them together" (`batchable` PAPER.md:250); SPEC
// schedule_next S:281 coalesces up to max_batch futures with identical
// (agent type, method), highest priority first.
//
// One block per instance of a batchable type.  The futures assigned to it
// this epoch are the admitted prefix of its own phase-A region of the
// assignment list plus the phase-B entries of its type's region that name it;
// both are already in the O4 order (K4 places an admitted future at its rank),
// so a two-way merge on (level desc, row asc) yields the instance's sequence,
// which is then cut per method into batches of max_batch.  The sequences are
// short (at most the instance's spare capacity), so the merge runs on one
// thread while the others stage the per-method counters.
#include "internal.h"

namespace nalar {

__global__ void __launch_bounds__(64) k6_batch(BatchParams p) {
    __shared__ uint32_t s_cnt[256];
    __shared__ int32_t s_head[256];
    __shared__ uint32_t s_offA, s_offB;
    const uint32_t i = blockIdx.x, tid = threadIdx.x;
    const uint32_t t = p.i_type[i];
    const uint32_t mb = p.t_max_batch[t];
    if (mb <= 1u) return;
    for (uint32_t m = tid; m < 256; m += blockDim.x) { s_cnt[m] = 0; s_head[m] = -1; }
    if (tid == 0) { s_offA = 0; s_offB = 0; }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    // region starts: prefix of the per-resource region sizes
    const uint32_t rB = p.n_inst + t;
    uint32_t a = 0, b = 0;
    for (uint32_t q = tid; q < rB; q += blockDim.x) {
        const uint32_t x = p.tot_loc[q];
        if (q < i) a += x;
        b += x;
    }
    if (a) atomicAdd(&s_offA, a);
    if (b) atomicAdd(&s_offB, b);
    __syncthreads();
    if (tid != 0) return;
    const uint32_t nA = p.n_adm[i], nB = p.n_adm[rB];
    const uint32_t* A = p.arow + s_offA;
    const uint32_t* Brow = p.arow + s_offB;
    const int16_t* Binst = p.ainst + s_offB;
    uint32_t ia = 0, ib = 0, nb = 0;
    // next phase-B entry at this instance
    auto nextB = [&](uint32_t k) {
        while (k < nB && Binst[k] != (int16_t)i) ++k;
        return k;
    };
    ib = nextB(0);
    while (ia < nA || ib < nB) {
        uint32_t f;
        if (ib >= nB) f = A[ia++];
        else if (ia >= nA) { f = Brow[ib]; ib = nextB(ib + 1); }
        else {
            const uint32_t fa = A[ia], fb = Brow[ib];
            const uint32_t la = p.level[fa], lb = p.level[fb];
            if (la > lb || (la == lb && fa < fb)) { f = fa; ++ia; }
            else { f = fb; ib = nextB(ib + 1); }
        }
        const uint32_t m = p.f_method ? p.f_method[f] : 0u;
        const uint32_t k = s_cnt[m]++;
        if (k % mb == 0u) { s_head[m] = (int32_t)f; ++nb; }
        p.batch_head[f] = s_head[m];
    }
    if (nb) atomicAdd(&p.counters[C_BATCHES], nb);
}

cudaError_t launch_batch(const BatchParams& p, cudaStream_t s) {
    if (p.n_inst == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.n_inst);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k6_batch, p);
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_batch() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k6_batch)) return e;
    return cudaSuccess;
}

}  // namespace nalar
