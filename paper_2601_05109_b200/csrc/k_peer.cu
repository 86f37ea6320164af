// k_peer.cu -- the rank exchange of the policy epoch over peer memory
// (NALAR_COLL_PEER).
//
// Between the sweep (K1) and admission (K4) every rank needs every rank's
// (resource, level) histogram slot H[s] and the sums over ranks of the
// per-instance in-flight load and per-resource totals (PAPER.md:387-388 route
// over all instances; the global rank is the row order across shards).  In
// NCCL mode that is one allreduce of the whole, mostly-zero, slot-disjoint
// buffer.  Here each rank instead STORES its own slot and partial sums
// straight into every peer's receive buffer (NVLink / NVSwitch peer memory,
// opened by CUDA IPC, or plain device memory for ranks driven by one
// process), then raises one epoch-numbered flag per peer; each rank's gather
// kernel waits for all G flags in its own buffer, copies the G slots into the
// exchange buffer K4 reads and sums the G partials.  Only the data moves (no
// reduction of G-1 zero slots), and the flags need no barrier with the host.
//
// Receive buffer (u32 words, identical layout on every rank):
//   [0, 64)                          flag[parity][src] = epoch number (parity = epoch & 1)
//   [64 + par * par_words, ...)      H[G][Rh*Lv] | loadS[G][I] | totS[G][Rh]
//   [64 + 2 * par_words, +8)         local words: epoch counter, push / gather block counters, wait ok,
//                                    sticky failure
// A failed exchange is sticky: the rank that timed out (or saw a peer's
// poison) writes kPeerPoison into its flag slots in every peer's buffer, so
// each peer's next wait fails at once instead of pairing its epoch with this
// rank's stale data, and its own later waits fail without polling.  Only a
// reconnect (nalar_peer_buffer + nalar_peer_connect on every rank, which
// clears the buffers) resumes the exchange.
// Two parities: a rank can run one epoch ahead of a peer still reading the
// previous epoch's data (it cannot run two ahead -- it waits for that peer's
// flag of the epoch in between, which the peer raises only after finishing
// the epoch before it, stream order).
#include "internal.h"

namespace nalar {

namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace

// push: this rank's slot + partial sums -> every rank's receive buffer; the
// last block to finish raises the flags
__global__ void __launch_bounds__(256) k_peer_push(PeerParams p) {
    uint32_t* loc = p.peers[p.rank] + kPeerFlagWords + 2 * p.par_words;   // local words
    const uint32_t e = loc[0] + 1u, par = e & 1u;
    const uint32_t nh = p.rh_lv, n = nh + p.I + p.Rh + 2 + p.lw;  // words sent to each peer
    const uint64_t total = (uint64_t)n * p.G;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = (uint32_t)(j / n), w = (uint32_t)(j % n);
        uint32_t* dst = p.peers[q] + kPeerFlagWords + par * p.par_words;
        uint32_t v;
        size_t o;
        if (w < nh) {
            v = p.slot[w];
            o = (size_t)p.rank * nh + w;
        } else if (w < nh + p.I) {
            v = p.load[w - nh];
            o = (size_t)p.G * nh + (size_t)p.rank * p.I + (w - nh);
        } else if (w < nh + p.I + p.Rh) {
            v = p.tot[w - nh - p.I];
            o = (size_t)p.G * (nh + p.I) + (size_t)p.rank * p.Rh + (w - nh - p.I);
        } else if (w < nh + p.I + p.Rh + 2) {
            v = p.rb_mine[w - nh - p.I - p.Rh];
            o = (size_t)p.G * (nh + p.I + p.Rh) + 2ull * p.rank + (w - nh - p.I - p.Rh);
        } else {                                  // this rank's list region (NEXT-1 candidates)
            const uint32_t k = w - nh - p.I - p.Rh - 2;
            v = p.list_mine[k];
            o = (size_t)p.G * (nh + p.I + p.Rh + 2) + (size_t)p.rank * p.lw + k;
        }
        dst[o] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t prev = atomicAdd(&loc[1], 1u);
        if (prev == gridDim.x - 1) {
            loc[1] = 0;
            __threadfence_system();
            for (uint32_t q = 0; q < p.G; ++q) st_release_sys(p.peers[q] + par * kPeerMaxRanks + p.rank, e);
        }
    }
}

// wait: one warp polls every rank's flag of this epoch (a single small block,
// so that ranks sharing a device -- one process driving several ranks --
// leave the SMs to the other ranks' sweeps while they wait)
__global__ void __launch_bounds__(32) k_peer_wait(PeerParams p) {
    uint32_t* own = p.peers[p.rank];
    uint32_t* loc = own + kPeerFlagWords + 2 * p.par_words;
    const uint32_t e = loc[0] + 1u, par = e & 1u;
    const uint32_t s = threadIdx.x;
    bool ok = loc[4] == 0u;                       // sticky: an earlier exchange failed
    if (ok && s < p.G) {
        const uint64_t t0 = gtimer_ns();
        const uint32_t* f = own + par * kPeerMaxRanks + s;
        uint32_t v;
        while ((v = ld_acquire_sys(f)) != e) {
            if (v == kPeerPoison || gtimer_ns() - t0 > kPeerTimeoutNs) { ok = false; break; }
            __nanosleep(64);
        }
    }
    ok = __all_sync(0xFFFFFFFFu, ok);
    if (!ok && s < p.G)                           // poison my flag slots (both parities) at every rank
        for (uint32_t q = 0; q < 2; ++q) st_release_sys(p.peers[s] + q * kPeerMaxRanks + p.rank, kPeerPoison);
    if (threadIdx.x == 0) {
        if (!ok && p.err) *(volatile unsigned long long*)p.err = 1ull;
        loc[3] = ok ? 1u : 0u;
        if (!ok) loc[4] = 1u;
    }
}

// gather: lay the slots and the summed partials out as K4's exchange buffer;
// the last block advances the epoch counter
__global__ void __launch_bounds__(256) k_peer_gather(PeerParams p) {
    uint32_t* own = p.peers[p.rank];
    uint32_t* loc = own + kPeerFlagWords + 2 * p.par_words;
    const uint32_t e = loc[0] + 1u, par = e & 1u;
    const bool s_ok = loc[3] != 0u;
    const uint32_t* src = own + kPeerFlagWords + par * p.par_words;
    const uint32_t nh = p.rh_lv;
    const uint64_t nH = (uint64_t)p.G * nh, n = nH + p.I + p.Rh + 2ull * p.G + (uint64_t)p.G * p.lw;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        if (j < nH) {
            v = src[j];
        } else if (j < nH + p.I) {
            const uint32_t i = (uint32_t)(j - nH);
            for (uint32_t s = 0; s < p.G; ++s) v += src[nH + (size_t)s * p.I + i];
        } else if (j < nH + p.I + p.Rh) {
            const uint32_t r = (uint32_t)(j - nH - p.I);
            for (uint32_t s = 0; s < p.G; ++s) v += src[nH + (size_t)p.G * p.I + (size_t)s * p.Rh + r];
        } else {                                  // (row base, rows) pairs, then the list regions, by rank
            v = src[nH + (size_t)p.G * (p.I + p.Rh) + (j - nH - p.I - p.Rh)];
        }
        p.x[j] = s_ok ? v : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t prev = atomicAdd(&loc[2], 1u);
        if (prev == gridDim.x - 1) {
            loc[2] = 0;
            loc[0] = e;
        }
    }
}

static uint32_t peer_grid(uint64_t words) {
    const uint64_t b = (words + 4 * 256 - 1) / (4 * 256);
    return (uint32_t)(b < 1 ? 1 : (b > 148 ? 148 : b));
}

cudaError_t launch_peer_exchange(const PeerParams& p, cudaStream_t s) {
    const uint64_t n = (uint64_t)p.rh_lv + p.I + p.Rh + 2 + p.lw;
    k_peer_push<<<peer_grid(n * p.G), 256, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_peer_wait<<<1, 32, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_peer_gather<<<peer_grid((uint64_t)p.G * p.rh_lv + p.I + p.Rh + 2ull * p.G + (uint64_t)p.G * p.lw), 256, 0, s>>>(p);
    return cudaGetLastError();
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_peer() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_peer_push)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_peer_gather)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_peer_wait)) return e;
    // same shared-memory carveout as the sweep, so a waiting block never
    // keeps an SM from taking a sweep block (the carveout changes only on an
    // idle SM)
    for (const void* k : {(const void*)k_peer_push, (const void*)k_peer_wait, (const void*)k_peer_gather})
        if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 (int)cudaSharedmemCarveoutMaxShared))
            return e;
    return cudaSuccess;
}

}  // namespace nalar
