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
// short (at most the instance's spare capacity): both are staged in shared
// memory by the block (the phase-B entries naming the instance compacted in
// order), then merged on one thread.
#include "internal.h"

namespace nalar {

constexpr uint32_t kK6Stage = 1024;     // staged entries per sequence
constexpr uint32_t kK6Scan = 1u << 16;  // phase-B region scanned by one warp at most

__global__ void __launch_bounds__(64) k6_batch(BatchParams p) {
    __shared__ uint32_t s_cnt[256];
    __shared__ int32_t s_head[256];
    __shared__ uint32_t s_offA, s_offB, s_nbi;
    __shared__ uint32_t s_a[kK6Stage], s_b[kK6Stage];
    __shared__ uint8_t s_la[kK6Stage], s_lb[kK6Stage], s_ma[kK6Stage], s_mb[kK6Stage];
    if (*p.verdict) return;              // an invalid table (K0)
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
    const uint32_t nA = p.n_adm[i], nB = p.n_adm[rB];
    const uint32_t* A = p.arow + s_offA;
    const uint32_t* Brow = p.arow + s_offB;
    const int16_t* Binst = p.ainst + s_offB;
    uint32_t nb = 0;
    if (nA <= kK6Stage && nB <= kK6Scan) {
        // stage both sequences in shared memory with their levels and methods
        // (warp 0: the phase-B entries naming this instance, compacted in
        // order; warp 1: the phase-A rows) -- the merge then runs on shared
        // memory instead of one dependent global load per entry
        const uint32_t lane = tid & 31u, warp = tid >> 5;
        if (warp == 0) {
            uint32_t n = 0;
            for (uint32_t k0 = 0; k0 < nB; k0 += 32) {
                const uint32_t k = k0 + lane;
                const bool hit = k < nB && Binst[k] == (int16_t)i;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
                if (hit) {
                    const uint32_t o = n + __popc(bal & ((1u << lane) - 1u));
                    if (o < kK6Stage) {
                        const uint32_t f = Brow[k];
                        s_b[o] = f;
                        s_lb[o] = p.level[f];
                        s_mb[o] = p.f_method ? p.f_method[f] : 0u;
                    }
                }
                n += __popc(bal);
            }
            if (lane == 0) s_nbi = n;
        } else {
            for (uint32_t k = lane; k < nA; k += 32) {
                const uint32_t f = A[k];
                s_a[k] = f;
                s_la[k] = p.level[f];
                s_ma[k] = p.f_method ? p.f_method[f] : 0u;
            }
        }
        __syncthreads();
        if (tid != 0) return;
        const uint32_t nBi = s_nbi;
        if (nBi <= kK6Stage) {
            uint32_t ia = 0, ib = 0;
            while (ia < nA || ib < nBi) {
                bool take_a;
                if (ib >= nBi) take_a = true;
                else if (ia >= nA) take_a = false;
                else take_a = s_la[ia] > s_lb[ib] || (s_la[ia] == s_lb[ib] && s_a[ia] < s_b[ib]);
                const uint32_t f = take_a ? s_a[ia] : s_b[ib];
                const uint32_t m = take_a ? s_ma[ia] : s_mb[ib];
                if (take_a) ++ia; else ++ib;
                const uint32_t k = s_cnt[m]++;
                if (k % mb == 0u) { s_head[m] = (int32_t)f; ++nb; }
                p.batch_head[f] = s_head[m];
            }
            if (nb) atomicAdd(&p.counters[C_BATCHES], nb);
            return;
        }
    } else if (tid != 0) {
        return;
    }
    // large sequences: merge straight from global memory on one thread
    uint32_t ia = 0, ib = 0;
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
