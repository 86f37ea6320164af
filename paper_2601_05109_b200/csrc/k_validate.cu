// k_validate.cu -- K0: the input contract of the live future table, checked on
// the device after upload.  Every dependency is write-once
// and exists when its consumer is created, so an edge must point
// to an EARLIER row of the SAME workflow (Q1); QUEUED/RUNNING
// futures carry an executor of their type (PAPER.md:479 executor metadata);
// pins name an instance of the future's type (state placement).
//
// Row-parallel: one thread per row (the workflow of a row from the block's
// window of workflow offsets in shared memory, which the host has checked to
// be monotone), so a deep workflow costs no more than any other -- the check
// is a few dependent loads deep, not one round trip per 32 rows of the
// longest workflow.  The
// smallest offending row wins (atomicMin), so the reported row is
// deterministic.
#include "internal.h"

namespace nalar {

// a = first row of f's workflow (found by the caller)
__device__ __forceinline__ void validate_row(const ValidateParams& p, uint32_t f, uint32_t a) {
    const uint32_t st = p.f_state[f], ty = p.f_type[f];
    const int pin = p.f_pin[f], ex = p.f_exec[f];
    const uint32_t e0 = p.f_edge_off[f], e1 = p.f_edge_off[f + 1];
    if (e1 < e0 || e1 > p.n_edges) {       // structural: CSR offsets not monotone
        atomicOr(&p.err[1], 1ull);
        return;
    }
    bool ok = st <= 4u && ty < p.n_types;
    if (ok && pin != -1 && (pin < 0 || (uint32_t)pin >= p.n_inst || p.i_type[pin] != ty)) ok = false;
    if (ok && (st == 1u || st == 2u) && (ex < 0 || (uint32_t)ex >= p.n_inst || p.i_type[ex] != ty)) ok = false;
    for (uint32_t e = e0; ok && e < e1; ++e) {
        const uint32_t s = p.edges[e] & 0x7FFFFFFFu;
        if (s < a || s >= f) ok = false;
    }
    if (!ok) atomicMin(&p.err[0], (unsigned long long)f);
}

// The last block to finish publishes the verdict straight into mapped host
// memory and re-arms the device words, so an upload needs no memset before
// and no copy after the kernel (three fewer stream operations per call).
__global__ void __launch_bounds__(kK0Threads) k0_validate(ValidateParams p) {
    // a programmatic dependent of the upload's copy kernel: launched while the
    // copy runs, it reads the table only after the copy has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // The workflows of this block's rows: one warp finds the workflow of the
    // block's first row by a 32-ary search over the offsets (3 rounds of 32
    // parallel loads instead of an 11-deep binary search per thread), then
    // the offsets covering the block (at most one per row, plus one) go to
    // shared memory, where each row finds its workflow.
    __shared__ uint32_t s_off[kK0Threads + 2];
    __shared__ uint32_t s_w0;
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t f0 = blockIdx.x * blockDim.x;
    const uint32_t f = f0 + tid;
    if (tid < 32) {
        uint32_t lo = 0, hi = p.n_wf - 1;          // last w with wf_fut_off[w] <= f0, in [lo, hi]
        while (hi > lo) {
            const uint32_t step = (hi - lo + 32u) / 32u;   // 32 segments cover [lo, hi]
            const uint32_t w = lo + lane * step;
            const bool le = w <= hi && p.wf_fut_off[w] <= f0;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, le);   // lane 0 (w = lo) always set
            const uint32_t k = 31u - __clz(bal);
            lo = lo + k * step;
            hi = min(hi, lo + step - 1u);
        }
        if (lane == 0) s_w0 = lo;
    }
    __syncthreads();
    const uint32_t w0 = s_w0;
    // offsets wf_fut_off[w0 .. w0 + L - 1]; L - 1 workflows (empty ones
    // included) -- enough unless many empty workflows sit inside the block
    const uint32_t L = min(p.n_wf - w0, (uint32_t)kK0Threads + 1u) + 1u;
    for (uint32_t k = tid; k < L; k += blockDim.x) s_off[k] = p.wf_fut_off[w0 + k];
    __syncthreads();
    if (f < p.n_fut) {
        uint32_t a;
        if (w0 + L - 1u == p.n_wf || f < s_off[L - 1u]) {
            uint32_t lo = 0, hi = L - 2u;          // last local w with s_off[w] <= f
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (s_off[mid] <= f) lo = mid;
                else hi = mid - 1;
            }
            a = s_off[lo];
        } else {                                   // beyond the window: search globally
            uint32_t lo = w0 + L - 1u, hi = p.n_wf - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (p.wf_fut_off[mid] <= f) lo = mid;
                else hi = mid - 1;
            }
            a = p.wf_fut_off[lo];
        }
        validate_row(p, f, a);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.done, 1u) == gridDim.x - 1) {
            __threadfence();
            const unsigned long long bad = atomicExch(&p.err[0], ~0ull), structural = atomicExch(&p.err[1], 0ull);
            volatile unsigned long long* h = p.host_err;
            h[0] = bad;
            h[1] = structural;
            if (p.delta_err) {                   // a delta's update errors (KD2 / KD4), then re-armed
                h[2] = atomicExch(&p.delta_err[0], ~0ull);
                h[3] = atomicExch(&p.delta_err[1], ~0ull);
            }
            // the epoch kernels of a combined step (nalar_step) may already be
            // queued behind this one: they read this word and skip an invalid table
            *p.verdict = (bad != ~0ull || structural) ? 1ull : 0ull;
            *p.done = 0;
        }
    }
}

cudaError_t launch_validate(const ValidateParams& p, cudaStream_t s) {
    // nothing to check: the table is valid; clear the verdict word the epoch
    // kernels read (a previous invalid upload may have set it)
    if (p.n_fut == 0 || p.n_wf == 0) return cudaMemsetAsync(p.verdict, 0, sizeof(unsigned long long), s);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((uint32_t)((p.n_fut + kK0Threads - 1) / kK0Threads));
    cfg.blockDim = dim3(kK0Threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k0_validate, p);
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_validate() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k0_validate)) return e;
    return cudaSuccess;
}

}  // namespace nalar
