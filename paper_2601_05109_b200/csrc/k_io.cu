// k_io.cu -- host <-> device traffic of the public API as kernels.
//
// nalar_snapshot_upload copies ~14 SoA arrays (plus the host-built type and
// block tables) to the device; nalar_fetch_decisions copies up to 11 back and
// compacts the assignment list.  Issued as one cudaMemcpyAsync each, the
// per-call driver overhead (several us each) dominates the 2-3 MB that
// actually move (SURVEY §7 "H2D upload ... costs more than the epoch itself").
// When the caller's host arrays are pinned (device-mapped under UVA), one
// kernel moves every segment instead, reading / writing host memory directly
// over the bus with 16-byte accesses and several in flight per thread; the
// fetch kernel also compacts the per-resource assignment regions on the way
// out, so a fetch is one launch and one synchronisation.
#include <algorithm>

#include "internal.h"

namespace nalar {

namespace {

__device__ __forceinline__ uint32_t seg_of(const CopyParams& p, uint64_t q) {
    uint32_t s = 0;
#pragma unroll 1
    while (s + 1 < p.n && p.chunk_off[s + 1] <= q) ++s;
    return s;
}

// one 16-byte chunk q of the concatenated segments (partial at a segment's
// end; bytewise when either side is not 16-byte aligned)
__device__ __forceinline__ void copy_chunk(const CopyParams& p, uint64_t q) {
    const uint32_t s = seg_of(p, q);
    const CopySeg& g = p.seg[s];
    const uint64_t off = (q - p.chunk_off[s]) * 16ull;
    const uint64_t n = g.bytes - off < 16ull ? g.bytes - off : 16ull;
    const uint8_t* src = (const uint8_t*)g.src + off;
    uint8_t* dst = (uint8_t*)g.dst + off;
    if (n == 16ull && (((uintptr_t)src | (uintptr_t)dst) & 15u) == 0u) {
        *(uint4*)dst = *(const uint4*)src;
    } else {
        for (uint64_t k = 0; k < n; ++k) dst[k] = src[k];
    }
}

}  // namespace

// grid-stride over the chunks, four chunks per thread per trip so several
// bus reads are in flight per thread
__global__ void __launch_bounds__(256) k_copy_segs(CopyParams p) {
    asm volatile("griddepcontrol.launch_dependents;");   // K0 may launch (it waits for completion)
    const uint64_t total = p.chunk_off[p.n];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += 4 * stride) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t q = q0 + j * stride;
            if (q < total) copy_chunk(p, q);
        }
    }
}

// fetch: blocks [0, R) compact resource r's admitted futures (region r of the
// device assignment list holds this rank's n_adm[r] admitted rows first) into
// position sum_{r' < r} n_adm[r'] of the caller's list; the remaining blocks
// copy the plain output segments.  Block 0 also publishes the counters.
__global__ void __launch_bounds__(256) k_fetch(FetchParams f, CopyParams p) {
    const uint32_t b = blockIdx.x;
    const uint32_t nlist = f.R ? f.R : 1u;      // block 0 always exists (counters)
    if (b < nlist) {
        __shared__ uint32_t s_out, s_in;
        if (threadIdx.x == 0) { s_out = 0; s_in = 0; }
        __syncthreads();
        uint32_t po = 0, pi = 0;
        for (uint32_t r = threadIdx.x; r < b; r += blockDim.x) { po += f.n_adm[r]; pi += f.tot_loc[r]; }
        if (po) atomicAdd(&s_out, po);
        if (pi) atomicAdd(&s_in, pi);
        __syncthreads();
        const uint32_t n = b < f.R ? f.n_adm[b] : 0u, o = s_out, i0 = s_in;
        const uint32_t na = f.counters[C_ASSIGNED];
        if (na <= f.a_cap) {
            for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
                if (f.out_row) f.out_row[o + k] = f.arow[i0 + k];
                if (f.out_inst) f.out_inst[o + k] = f.ainst[i0 + k];
            }
        }
        if (b == 0 && threadIdx.x < C_NUM) f.out_counters[threadIdx.x] = f.counters[threadIdx.x];
        return;
    }
    const uint64_t total = p.chunk_off[p.n];
    const uint64_t stride = (uint64_t)(gridDim.x - nlist) * blockDim.x;
    for (uint64_t q0 = (uint64_t)(b - nlist) * blockDim.x + threadIdx.x; q0 < total; q0 += 4 * stride) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t q = q0 + j * stride;
            if (q < total) copy_chunk(p, q);
        }
    }
}

static uint32_t copy_grid(uint64_t chunks) {
    const uint64_t want = (chunks + 4 * 256 - 1) / (4 * 256);
    return (uint32_t)std::min<uint64_t>(std::max<uint64_t>(want, 1), 2 * 148);
}

cudaError_t launch_copy_segs(const CopyParams& p, cudaStream_t s) {
    if (p.n == 0 || p.chunk_off[p.n] == 0) return cudaSuccess;
    k_copy_segs<<<copy_grid(p.chunk_off[p.n]), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_fetch(const FetchParams& f, const CopyParams& p, cudaStream_t s) {
    const uint64_t chunks = p.n ? p.chunk_off[p.n] : 0;
    const uint32_t nb = chunks ? copy_grid(chunks) : 0u;
    k_fetch<<<(f.R ? f.R : 1u) + nb, 256, 0, s>>>(f, p);
    return cudaGetLastError();
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_io() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_copy_segs)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_fetch)) return e;
    return cudaSuccess;
}

}  // namespace nalar
