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
                if (k % mb == 0u) { s_head[m] = (int32_t)(p.row_base + f); ++nb; }
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
        if (k % mb == 0u) { s_head[m] = (int32_t)(p.row_base + f); ++nb; }
        p.batch_head[f] = s_head[m];
    }
    if (nb) atomicAdd(&p.counters[C_BATCHES], nb);
}

// ---- world > 1: K6 over every rank's lists (DESIGN.md Q-batch) ------------
// The futures assigned to an instance come from every rank, so each rank's
// eligible futures of the batchable resources travel in the epoch's one
// exchange (k_lists), and every rank re-derives their admission exactly as K4
// does -- global (resource, level) counts from the exchanged histogram, stable
// in-level ranks over the ranks' lists in rank order (= the global row order),
// admitted iff rank g < bound (spare for phase A, the sum of phase-A-residual
// spare over the type for phase B, whose slot g -> instance map is K4's water
// fill) -- then merges the instance's two sequences on (level desc, global row
// asc) and cuts them per method.  Every rank computes every batch (the same
// count everywhere) and writes batch_head (a global row) for its own rows.
constexpr uint32_t kK6mThreads = 256;
constexpr uint32_t kK6mWarps = kK6mThreads / 32;

__device__ __forceinline__ uint64_t k6m_slots_above(const uint32_t* sp2, uint32_t n, uint64_t s) {
    uint64_t a = 0;
    for (uint32_t k = 0; k < n; ++k) a += sp2[k] > s ? sp2[k] - s : 0ull;
    return a;
}

__global__ void __launch_bounds__(kK6mThreads, 1) k6_batch_ranks(BatchParams p) {
    __shared__ uint32_t s_sp2[NALAR_MAX_INSTANCES_DEV], s_inst[NALAR_MAX_INSTANCES_DEV];
    __shared__ uint32_t s_A[256], s_run[256], s_wc[kK6mWarps][256], s_red[kK6mWarps];
    __shared__ uint32_t s_off[2][kPeerMaxRanks], s_cnt[2][kPeerMaxRanks + 1];
    __shared__ uint64_t s_gA[kK6Stage], s_gB[kK6Stage];   // admitted: (level, method, global row) by rank g
    __shared__ uint16_t s_iB[kK6Stage];                    // phase-B admitted: instance index
    __shared__ uint32_t s_bad, s_maxs;
    __shared__ unsigned long long s_boundB;
    if (*p.verdict) return;
    const uint32_t i = blockIdx.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t t = p.i_type[i];
    const uint32_t mb = p.t_max_batch[t];
    if (mb <= 1u) return;
    const uint32_t G = p.G, I = p.n_inst, Lv = p.levels, rA = i, rB = I + t;
    const uint32_t k0 = p.type_off[t], ni = p.type_off[t + 1] - k0;
    if (tid == 0) { s_bad = 0; s_maxs = 0; s_boundB = 0; }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    // each rank's segment of rA / rB in its batch section
    {
        uint32_t pa[kPeerMaxRanks], pb[kPeerMaxRanks];
        for (uint32_t s = 0; s < G; ++s) {
            const uint32_t* L = p.lists + (size_t)s * kListWords + kMigWords;
            uint32_t a = 0, b = 0;
            for (uint32_t q = tid; q < rB; q += kK6mThreads) {
                const uint32_t c = L[1 + q];
                a += q < rA ? c : 0u;
                b += c;
            }
            pa[s] = a; pb[s] = b;
            if (tid == 0 && L[0] == kListOverflow) s_bad = 1u;
        }
        for (uint32_t s = 0; s < G; ++s) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                pa[s] += __shfl_xor_sync(0xFFFFFFFFu, pa[s], o);
                pb[s] += __shfl_xor_sync(0xFFFFFFFFu, pb[s], o);
            }
        }
        __shared__ uint32_t s_pa[kK6mWarps][kPeerMaxRanks], s_pb[kK6mWarps][kPeerMaxRanks];
        if (lane == 0)
            for (uint32_t s = 0; s < G; ++s) { s_pa[warp][s] = pa[s]; s_pb[warp][s] = pb[s]; }
        __syncthreads();
        if (tid < G) {
            uint32_t a = 0, b = 0;
            for (int w = 0; w < kK6mWarps; ++w) { a += s_pa[w][tid]; b += s_pb[w][tid]; }
            const uint32_t* L = p.lists + (size_t)tid * kListWords + kMigWords;
            const uint32_t hdr = 1 + p.R;
            s_off[0][tid] = hdr + 2 * a;
            s_off[1][tid] = hdr + 2 * b;
            s_cnt[0][tid] = L[1 + rA];
            s_cnt[1][tid] = L[1 + rB];
        }
        __syncthreads();
        if (tid < 2) {                       // prefix over ranks
            uint32_t c = 0;
            for (uint32_t s = 0; s < G; ++s) { const uint32_t x = s_cnt[tid][s]; s_cnt[tid][s] = c; c += x; }
            s_cnt[tid][G] = c;
        }
    }
    // the type's instances: phase-A-residual spare (global inputs, as K4)
    for (uint32_t k = tid; k < ni; k += kK6mThreads) {
        const uint32_t q = p.type_inst[k0 + k];
        const uint32_t sp = p.i_spare[q], tt = p.tot[q];
        const uint32_t s2 = sp - (tt < sp ? tt : sp);
        s_inst[k] = q;
        s_sp2[k] = s2;
        atomicMax(&s_maxs, s2);
        atomicAdd(&s_boundB, (unsigned long long)s2);
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0 && p.list_err) *(volatile unsigned long long*)p.list_err = 1ull;
        return;
    }
    const uint64_t boundA = p.i_spare[i], boundB = s_boundB;
    const uint32_t maxs = s_maxs;
    uint32_t nadm[2] = {0, 0};
    // phase A (ph 0: resource i) and phase B (ph 1: resource I + t)
    for (uint32_t ph = 0; ph < 2; ++ph) {
        const uint32_t r = ph ? rB : rA;
        const uint64_t bound = ph ? boundB : boundA;
        uint32_t hl = 0;
        if (tid < Lv)
            for (uint32_t s = 0; s < G; ++s) hl += p.H[((size_t)s * p.Rh + r) * Lv + tid];
        uint32_t x = hl;                      // count strictly above each level
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, x, o);
            if (lane + o < 32) x += y;
        }
        if (lane == 0) s_red[warp] = x;
        __syncthreads();
        uint32_t a = x - hl;
        for (uint32_t w = warp + 1; w < (uint32_t)kK6mWarps; ++w) a += s_red[w];
        s_A[tid] = a;
        s_run[tid] = 0;
#pragma unroll
        for (int w = 0; w < kK6mWarps; ++w) s_wc[w][tid] = 0;
        __syncthreads();
        const uint32_t total = s_cnt[ph][G];
        const uint64_t n_adm = (uint64_t)total < bound ? total : bound;
        if (n_adm > kK6Stage) {
            if (tid == 0 && p.list_err) *(volatile unsigned long long*)p.list_err = 1ull;
            return;
        }
        nadm[ph] = (uint32_t)n_adm;
        for (uint32_t q0 = 0; q0 < total; q0 += kK6mThreads) {
            const uint32_t q = q0 + tid;
            const bool ok = q < total;
            uint32_t lv = 0x100u + tid, w0 = 0, w1 = 0;
            if (ok) {
                uint32_t s = 0;
                while (s + 1 < G && s_cnt[ph][s + 1] <= q) ++s;
                const uint32_t* L = p.lists + (size_t)s * kListWords + kMigWords + s_off[ph][s];
                const uint32_t k = q - s_cnt[ph][s];
                w0 = L[2 * k];
                w1 = L[2 * k + 1];
                lv = w0 & 0xFFu;
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, lv);
            if (ok && (__ffs(peers) - 1) == (int)lane) s_wc[warp][lv] = __popc(peers);
            __syncthreads();
            if (ok) {
                uint32_t rank = s_run[lv] + __popc(peers & ((1u << lane) - 1u));
                for (uint32_t k = 0; k < warp; ++k) rank += s_wc[k][lv];
                const uint64_t g = (uint64_t)s_A[lv] + rank;
                if (g < n_adm) {
                    const uint64_t e = ((uint64_t)w0 << 32) | w1;   // level | method << 8, global row
                    if (ph == 0) {
                        s_gA[g] = e;
                    } else {
                        // K4's water fill: slot g -> (level L, j-th instance with spare2 >= L)
                        uint64_t lo = 1, hi = maxs;
                        while (lo < hi) {
                            const uint64_t mid = lo + ((hi - lo) >> 1);
                            if (k6m_slots_above(s_sp2, ni, mid) <= g) hi = mid;
                            else lo = mid + 1;
                        }
                        uint64_t j = g - k6m_slots_above(s_sp2, ni, lo);
                        uint32_t pick = 0;
                        for (uint32_t k = 0; k < ni; ++k)
                            if (s_sp2[k] >= lo) {
                                if (j == 0) { pick = k; break; }
                                --j;
                            }
                        s_gB[g] = e;
                        s_iB[g] = (uint16_t)pick;
                    }
                }
            }
            __syncthreads();
            {
                uint32_t add = 0;
#pragma unroll
                for (int k = 0; k < kK6mWarps; ++k) { add += s_wc[k][tid]; s_wc[k][tid] = 0; }
                s_run[tid] += add;
            }
            __syncthreads();
        }
    }
    if (tid != 0) return;
    // the instance's sequence: merge (level desc, global row asc), cut per method
    uint32_t kl = 0;
    for (uint32_t k = 0; k < ni; ++k) if (s_inst[k] == i) kl = k;
    uint32_t ia = 0, ib = 0, nb = 0;
    auto nextB = [&](uint32_t k) {
        while (k < nadm[1] && s_iB[k] != kl) ++k;
        return k;
    };
    ib = nextB(0);
    uint32_t cnt[256];
    int32_t head[256];
    for (int m = 0; m < 256; ++m) { cnt[m] = 0; head[m] = -1; }
    while (ia < nadm[0] || ib < nadm[1]) {
        uint64_t e;
        if (ib >= nadm[1]) e = s_gA[ia++];
        else if (ia >= nadm[0]) { e = s_gB[ib]; ib = nextB(ib + 1); }
        else {
            const uint64_t ea = s_gA[ia], eb = s_gB[ib];
            const uint32_t la = (uint32_t)(ea >> 32) & 0xFFu, lb = (uint32_t)(eb >> 32) & 0xFFu;
            if (la > lb || (la == lb && (uint32_t)ea < (uint32_t)eb)) { e = ea; ++ia; }
            else { e = eb; ib = nextB(ib + 1); }
        }
        const uint32_t m = (uint32_t)(e >> 40) & 0xFFu, row = (uint32_t)e;
        const uint32_t k = cnt[m]++;
        if (k % mb == 0u) { head[m] = (int32_t)row; ++nb; }
        if (row >= p.row_base && row - p.row_base < p.n_rows) p.batch_head[row - p.row_base] = head[m];
    }
    if (nb) atomicAdd(&p.counters[C_BATCHES], nb);
}

cudaError_t launch_batch(const BatchParams& p, cudaStream_t s) {
    if (p.n_inst == 0) return cudaSuccess;
    if (p.G > 1) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(p.n_inst);
        cfg.blockDim = dim3(kK6mThreads);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, k6_batch_ranks, p);
    }
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
    if (cudaError_t e = cudaFuncGetAttributes(&a, k6_batch_ranks)) return e;
    return cudaSuccess;
}

}  // namespace nalar
