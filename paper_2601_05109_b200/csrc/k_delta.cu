// k_delta.cu -- S0 delta ingestion: turn the resident table of epoch k into the
// table of epoch k+1 on the device (nalar_delta_apply, include/nalar.h).
//
//   KD1 apply-assigned: futures ASSIGNED by the last epoch -> QUEUED at their
//       instance (they sit in the per-resource regions of the assignment list)
//   KD2 updates: (workflow id, seq) -> row by binary search over the sorted
//       workflow ids; state / executor / pin overwritten in place
//   KD3 rebuild: one warp per workflow of the NEW table copies the kept rows
//       (edges and offsets re-based), then appends the new futures (edges given
//       as workflow-local seq), into the other buffer set
//   KD4 set_priority and instance updates
// The new table then goes through K0 validation exactly like an upload.
#include "internal.h"

namespace nalar {

__global__ void kd1_apply_assigned(DeltaParams p) {
    const uint32_t r = blockIdx.x;
    __shared__ uint32_t s_base;
    if (threadIdx.x == 0) {
        uint32_t b = 0;
        for (uint32_t q = 0; q < r; ++q) b += p.tot_loc[q];
        s_base = b;
    }
    __syncthreads();
    const uint32_t n = p.n_adm[r];
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
        const uint32_t row = p.arow[s_base + k];
        p.state[row] = 1;                       // QUEUED
        p.exec[row] = p.ainst[s_base + k];
    }
}

__global__ void kd2_updates(DeltaParams p) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.n_upd) return;
    const uint64_t id = p.upd_wf_id[k];
    uint32_t lo = 0, hi = p.n_wf;                // first index with wf_id >= id
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (p.wf_id[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    if (lo >= p.n_wf || p.wf_id[lo] != id) { atomicMin(&p.err[0], (unsigned long long)k); return; }
    const uint32_t a = p.wf_off[lo], b = p.wf_off[lo + 1];
    const uint32_t seq = p.upd_seq[k];
    if (seq >= b - a) { atomicMin(&p.err[0], (unsigned long long)k); return; }
    const uint32_t row = a + seq;
    if (p.upd_state[k] != 0xFFu) p.state[row] = p.upd_state[k];
    if (p.upd_exec[k] != -2) p.exec[row] = p.upd_exec[k];
    if (p.upd_pin[k] != -2) p.pin[row] = p.upd_pin[k];
}

// plan per new workflow (host-built): src old index (or ~0), rows kept from the
// old table, appended range, and where everything lands
__global__ void kd3_rebuild(DeltaParams p) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= p.n_wf_new) return;
    if (w == 0 && lane == 0) {               // tails of the new offset arrays
        p.n_wf_off[p.n_wf_new] = p.n_fut_new;
        p.n_eoff[p.n_fut_new] = p.n_edges_new;
    }
    const RebuildPlan pl = p.plan[w];
    // workflow arrays
    if (lane == 0) {
        p.n_wf_off[w] = pl.new_row0;
        p.n_wf_id[w] = pl.wf_id;
        p.n_wf_prio[w] = pl.src != 0xFFFFFFFFu ? p.wf_prio[pl.src] : pl.prio;
    }
    // kept rows
    const uint32_t old_r0 = pl.src != 0xFFFFFFFFu ? p.wf_off[pl.src] : 0u;
    const uint32_t old_e0 = pl.src != 0xFFFFFFFFu ? p.eoff[old_r0] : 0u;
    for (uint32_t j = lane; j < pl.n_old; j += 32) {
        const uint32_t o = old_r0 + j, n = pl.new_row0 + j;
        p.n_state[n] = p.state[o];
        p.n_type[n] = p.type[o];
        p.n_round[n] = p.round[o];
        p.n_exec[n] = p.exec[o];
        p.n_pin[n] = p.pin[o];
        p.n_eoff[n] = pl.new_edge0 + (p.eoff[o] - old_e0);
    }
    for (uint32_t j = lane; j < pl.n_old_edges; j += 32) {
        const uint32_t v = p.edges[old_e0 + j];
        const uint32_t s = (v & 0x7FFFFFFFu) - old_r0 + pl.new_row0;
        p.n_edges[pl.new_edge0 + j] = (v & 0x80000000u) | s;
    }
    // appended rows
    const uint32_t ae0 = p.app_eoff[pl.app_lo];
    for (uint32_t j = lane; j < pl.app_n; j += 32) {
        const uint32_t a = pl.app_lo + j, n = pl.new_row0 + pl.n_old + j;
        p.n_state[n] = p.app_state[a];
        p.n_type[n] = p.app_type[a];
        p.n_round[n] = p.app_round[a];
        p.n_exec[n] = p.app_exec[a];
        p.n_pin[n] = p.app_pin[a];
        p.n_eoff[n] = pl.new_edge0 + pl.n_old_edges + (p.app_eoff[a] - ae0);
    }
    const uint32_t n_app_edges = p.app_eoff[pl.app_lo + pl.app_n] - ae0;
    for (uint32_t j = lane; j < n_app_edges; j += 32) {
        const uint32_t v = p.app_edges[ae0 + j];
        p.n_edges[pl.new_edge0 + pl.n_old_edges + j] = (v & 0x80000000u) | ((v & 0x7FFFFFFFu) + pl.new_row0);
    }
}

__global__ void kd4_prio_inst(DeltaParams p) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < p.n_prio) {
        const uint64_t id = p.prio_wf_id[k];
        uint32_t lo = 0, hi = p.n_wf_new;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (p.n_wf_id[mid] < id) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= p.n_wf_new || p.n_wf_id[lo] != id) atomicMin(&p.err[1], (unsigned long long)k);
        else p.n_wf_prio[lo] = p.prio_value[k];
    }
    if (k < p.n_inst_upd) {
        const uint32_t i = p.inst_id[k];
        if (i >= p.n_inst) atomicMin(&p.err[1], (unsigned long long)(p.n_prio + k));
        else { p.i_cap[i] = p.inst_cap[k]; p.i_base[i] = p.inst_base[k]; }
    }
}

cudaError_t launch_delta(const DeltaParams& p, bool apply_assigned, uint32_t R, cudaStream_t s) {
    if (apply_assigned && R) kd1_apply_assigned<<<R, 128, 0, s>>>(p);
    if (p.n_upd) kd2_updates<<<(p.n_upd + 255) / 256, 256, 0, s>>>(p);
    if (p.n_wf_new) kd3_rebuild<<<(uint32_t)(((uint64_t)p.n_wf_new * 32 + 255) / 256), 256, 0, s>>>(p);
    const uint32_t m = p.n_prio > p.n_inst_upd ? p.n_prio : p.n_inst_upd;
    if (m) kd4_prio_inst<<<(m + 255) / 256, 256, 0, s>>>(p);
    return cudaGetLastError();
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_delta() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, kd1_apply_assigned)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, kd2_updates)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, kd3_rebuild)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, kd4_prio_inst)) return e;
    return cudaSuccess;
}

}  // namespace nalar
