// k_migrate.cu -- K5: head-of-line-blocking migration.
//
// "migrates a job if it's waiting in the queue and observing head-of-line
// blocking" (PAPER.md:663 [§6.1]); the migrate primitive PAPER.md:391; SPEC
// hol_migration S:441.  DESIGN.md reading Q-mig, oracle step O11.
//
// K1 marked the candidates -- QUEUED futures waiting past theta_wait at a
// blocked instance (head job past theta_head), not STATEFUL, a SESSION one
// only as its session's sole queued work -- and bucketed them like eligible
// futures under resource R + type, in row order, with their level histogram.
// One block per type t then:
//   1. ranks every candidate of t in the O4 order (level desc, row asc) from
//      the histogram suffix sums + a stable within-level rank (the same
//      counting sort the admission pass uses) and places it at that rank;
//   2. replays the sequential greedy of O11 exactly, 32 candidates at a time on
//      one warp.  The j-th move of the type lands on slot j of the destination
//      list [(level b, instance i): b >= backlog_i, i unblocked] sorted by
//      (b asc, i asc) -- "the least backlogged, ties to the lowest id", each
//      move raising that instance by one -- and a candidate from source s with
//      m earlier moves out of s moves iff level_j + delta <= backlog_s - m.
//      Speculating that all 32 move, the first lane whose test fails is the
//      only decision that changes the picture: its source can never move again
//      (level_j only grows, backlog_s - m no longer shrinks), so it is retired
//      and the batch is re-evaluated from the next lane.  Each pass decides at
//      least one lane; a batch takes at most (1 + retired sources) passes.
//
// World > 1: the candidates of every rank arrive in the epoch's one exchange
// (k_lists below writes this rank's into its list region before the
// collective).  The global O4 order is (level desc, rank asc, row asc) -- the
// shards are consecutive in the row order -- so every rank walks all ranks'
// lists in rank order with the same counting sort, runs the same greedy on the
// same (global) backlogs and reaches the same moves; it writes migrate_to for
// its own rows only.
#include "internal.h"

namespace nalar {

namespace {

constexpr int kK5Threads = 256;
constexpr int kK5Warps = kK5Threads / 32;
constexpr uint32_t kMigWin = 2048;     // candidates placed per window (ranks [w0, w0 + kMigWin))

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace

__global__ void __launch_bounds__(kK5Threads, 1) k5_migrate(MigrateParams p) {
    __shared__ uint32_t s_inst[kK5MaxInst];
    __shared__ uint32_t s_b[kK5MaxInst];                    // backlog = load + assigned
    __shared__ uint32_t s_in[kK5MaxInst], s_out[kK5MaxInst];
    __shared__ uint32_t s_moved[kK5MaxInst];
    __shared__ uint8_t s_blk[kK5MaxInst], s_alive[kK5MaxInst];
    __shared__ uint16_t s_lk[NALAR_MAX_INSTANCES_DEV];      // instance id -> index in the type
    __shared__ uint32_t s_A[256], s_run[256];
    __shared__ uint32_t s_wc[kK5Warps][256];
    __shared__ uint32_t s_pref[kK5Threads + 1], s_base[kK5Threads], s_red[kK5Warps];
    __shared__ uint2 s_c[kMigWin];                          // (row, local source) by rank - w0
    __shared__ uint32_t s_nt, s_lmin;

    __shared__ uint32_t s_loff[kPeerMaxRanks], s_lcnt[kPeerMaxRanks + 1], s_lerr;
    if (*p.verdict) return;              // an invalid table (K0)
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t t = blockIdx.x, r = p.R + t, Lv = p.levels, B = p.B;
    const uint32_t G = p.G > 1 ? p.G : 1u;
    // ---- static: the type's instances, blocked flags (before the PDL wait) --
    const uint32_t k0 = p.type_off[t], ni = p.type_off[t + 1] - k0;
    for (uint32_t k = tid; k < ni; k += kK5Threads) {
        const uint32_t i = p.type_inst[k0 + k];
        s_inst[k] = i;
        s_lk[i] = (uint16_t)k;
        s_blk[k] = p.i_head_rem[i] > p.theta_head ? 1 : 0;
        s_in[k] = 0; s_out[k] = 0; s_moved[k] = 0; s_alive[k] = 1;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");

    const uint32_t n = p.tot[r];                              // candidates of type t (all ranks)
    uint32_t hl = 0;
    if (tid < Lv)
        for (uint32_t s = 0; s < G; ++s) hl += p.H[((size_t)s * p.Rh + r) * Lv + tid];
    if (G > 1) {
        // each rank's list segment of type t: offset and count
        if (tid == 0) s_lerr = 0;
        if (tid < G) {
            const uint32_t* L = p.lists + (size_t)tid * kListWords;
            uint32_t off = 0;
            for (uint32_t u = 0; u < t; ++u) off += L[1 + u];
            s_loff[tid] = kListHdr + off;
            s_lcnt[tid] = L[1 + t];
            if (L[0] == kListOverflow) s_lerr = 1u;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t c = 0;
            for (uint32_t s = 0; s < G; ++s) { const uint32_t x = s_lcnt[s]; s_lcnt[s] = c; c += x; }
            s_lcnt[G] = c;
        }
        __syncthreads();
        if (s_lerr) {                          // some rank's candidates did not fit its list
            if (tid == 0 && t == 0 && p.list_err) *(volatile unsigned long long*)p.list_err = 1ull;
            return;
        }
    }
    for (uint32_t k = tid; k < ni; k += kK5Threads) {
        const uint32_t i = s_inst[k];
        const uint64_t b = (uint64_t)p.i_load[i] + p.i_assigned[i];
        s_b[k] = b > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)b;
    }
    if (tid == 0) { s_nt = 0; s_lmin = 0xFFFFFFFFu; }
    __syncthreads();
    for (uint32_t k = tid; k < ni; k += kK5Threads)
        if (!s_blk[k]) { atomicAdd(&s_nt, 1u); atomicMin(&s_lmin, s_b[k]); }
    // count strictly above each level (suffix sums over 256 levels)
    {
        uint32_t x = hl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, x, o);
            if (lane + o < 32) x += y;
        }
        if (lane == 0) s_red[warp] = x;
        __syncthreads();
        uint32_t a = x - hl;
        for (uint32_t w = warp + 1; w < (uint32_t)kK5Warps; ++w) a += s_red[w];
        if (tid < 256) { s_A[tid] = a; s_run[tid] = 0; }
#pragma unroll
        for (int w = 0; w < kK5Warps; ++w) s_wc[w][tid] = 0;
    }
    __syncthreads();
    const uint32_t nt = s_nt, lmin = s_lmin;
    uint32_t j = 0, n_moves = 0;                             // moves so far (warp 0)

    // slot j of the destination list: its level and instance (local index)
    auto slot = [&](uint32_t jj, uint32_t* lvl, uint32_t* kk) {
        auto below = [&](uint32_t L) {                       // slots with level < L
            uint32_t c = 0;
            for (uint32_t k = 0; k < ni; ++k)
                if (!s_blk[k] && L > s_b[k]) c += L - s_b[k];
            return c;
        };
        uint32_t lo = lmin, hi = lmin + jj;                   // max L with below(L) <= jj
        while (lo < hi) {
            const uint32_t mid = lo + ((hi - lo + 1) >> 1);
            if (below(mid) <= jj) lo = mid;
            else hi = mid - 1;
        }
        uint32_t c = jj - below(lo), pick = 0;
        for (uint32_t k = 0; k < ni; ++k)
            if (!s_blk[k] && s_b[k] <= lo) {
                if (c == 0) { pick = k; break; }
                --c;
            }
        *lvl = lo;
        *kk = pick;
    };

    for (uint32_t w0 = 0; w0 < n; w0 += kMigWin) {
        // ---- 1. place the candidates of ranks [w0, w0 + kMigWin) ------------
        if (G > 1) {
            // every rank's list, in rank order: one global sequence in row order
            const uint32_t total = s_lcnt[G];
            for (uint32_t q0 = 0; q0 < total; q0 += kK5Threads) {
                const uint32_t q = q0 + tid;
                const bool ok = q < total;
                uint32_t lv = 0x100u + tid, row = 0xFFFFFFFFu, src = 0;
                if (ok) {
                    uint32_t s = 0;
                    while (s + 1 < G && s_lcnt[s + 1] <= q) ++s;
                    const uint32_t k = q - s_lcnt[s];
                    const uint32_t e = p.lists[(size_t)s * kListWords + s_loff[s] + k];
                    lv = e & 0xFFu;
                    src = s_lk[(e >> 16) - 1u];
                    if (s == p.rank) row = p.mrow[s_loff[s] - kListHdr + k];
                }
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, lv);
                if (ok && (__ffs(peers) - 1) == (int)lane) s_wc[warp][lv] = __popc(peers);
                __syncthreads();
                if (ok) {
                    uint32_t rank = s_run[lv] + __popc(peers & lanemask_lt());
                    for (uint32_t k = 0; k < warp; ++k) rank += s_wc[k][lv];
                    const uint32_t g = s_A[lv] + rank;
                    if (g >= w0 && g < w0 + kMigWin) s_c[g - w0] = make_uint2(row, src);
                }
                __syncthreads();
                {
                    uint32_t add = 0;
#pragma unroll
                    for (int k = 0; k < kK5Warps; ++k) { add += s_wc[k][tid]; s_wc[k][tid] = 0; }
                    s_run[tid] += add;
                }
                __syncthreads();
            }
        }
        for (uint32_t b0 = 0; G == 1 && b0 < B; b0 += kK5Threads) {
            const uint32_t bb = b0 + tid;
            const uint32_t c = bb < B ? p.cnt_rb[(size_t)r * B + bb] : 0u;
            if (bb < B) s_base[tid] = p.blk_row0[bb] + p.off_rb[(size_t)r * B + bb];
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            __syncthreads();
            if (lane == 31) s_red[warp] = incl;
            __syncthreads();
            uint32_t wb = 0;
            for (uint32_t k = 0; k < warp; ++k) wb += s_red[k];
            s_pref[tid] = wb + incl - c;
            if (tid == kK5Threads - 1) s_pref[kK5Threads] = wb + incl;
            __syncthreads();
            const uint32_t total = s_pref[kK5Threads];
            const uint32_t nb = min((uint32_t)kK5Threads, B - b0);
            for (uint32_t q0 = 0; q0 < total; q0 += kK5Threads) {
                const uint32_t q = q0 + tid;
                const bool ok = q < total;
                uint32_t lv = 0x100u + tid, row = 0, src = 0;
                if (ok) {
                    uint32_t lo = 0, hi = nb - 1;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi + 1) >> 1;
                        if (s_pref[mid] <= q) lo = mid;
                        else hi = mid - 1;
                    }
                    const uint2 x = p.items[s_base[lo] + (q - s_pref[lo])];
                    row = x.x;
                    lv = x.y & 0xFFu;
                    src = s_lk[(x.y >> 16) - 1u];
                }
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, lv);
                if (ok && (__ffs(peers) - 1) == (int)lane) s_wc[warp][lv] = __popc(peers);
                __syncthreads();
                if (ok) {
                    uint32_t rank = s_run[lv] + __popc(peers & lanemask_lt());
                    for (uint32_t k = 0; k < warp; ++k) rank += s_wc[k][lv];
                    const uint32_t g = s_A[lv] + rank;
                    if (g >= w0 && g < w0 + kMigWin) s_c[g - w0] = make_uint2(row, src);
                }
                __syncthreads();
                {
                    uint32_t add = 0;
#pragma unroll
                    for (int k = 0; k < kK5Warps; ++k) { add += s_wc[k][tid]; s_wc[k][tid] = 0; }
                    s_run[tid] += add;
                }
                __syncthreads();
            }
        }
        // ---- 2. the greedy, in rank order, on warp 0 -------------------------
        const uint32_t m = min(kMigWin, n - w0);
        if (warp == 0 && nt > 0) {
            for (uint32_t pos0 = 0; pos0 < m; pos0 += 32) {
                const uint32_t pos = pos0 + lane;
                const bool valid = pos < m;
                const uint2 cx = valid ? s_c[pos] : make_uint2(0u, 0u);
                const uint32_t ks = cx.y;
                bool done = !valid;
                for (;;) {
                    const bool act = !done && s_alive[ks];
                    const uint32_t A = __ballot_sync(0xFFFFFFFFu, act);
                    if (A == 0u) break;
                    const uint32_t jj = j + __popc(A & lanemask_lt());
                    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, act ? ks : 0x10000u + lane);
                    const uint32_t mm = act ? s_moved[ks] + __popc(peers & A & lanemask_lt()) : 0u;
                    uint32_t lvl = 0, kt = 0;
                    bool okm = false;
                    if (act) {
                        slot(jj, &lvl, &kt);
                        okm = (uint64_t)lvl + p.delta + mm <= (uint64_t)s_b[ks];
                    }
                    const uint32_t F = __ballot_sync(0xFFFFFFFFu, act && !okm);
                    const uint32_t first = F ? (uint32_t)(__ffs(F) - 1) : 32u;
                    const uint32_t commit = A & (first == 32u ? 0xFFFFFFFFu : ((1u << first) - 1u));
                    const bool me = (commit >> lane) & 1u;
                    if (me) {
                        if (cx.x != 0xFFFFFFFFu) p.migrate_to[cx.x] = (int16_t)s_inst[kt];   // own rows only
                        atomicAdd(&s_in[kt], 1u);
                    }
                    // per source: its moves in this pass, added once by its lowest lane
                    const uint32_t grp = peers & commit;
                    if (me && (__ffs(grp) - 1) == (int)lane) {
                        s_moved[ks] += __popc(grp);
                        s_out[ks] += __popc(grp);
                    }
                    __syncwarp();
                    j += __popc(commit);
                    n_moves += __popc(commit);
                    if (F && lane == first) s_alive[ks] = 0;     // this source never moves again
                    done = done || lane <= first;
                    __syncwarp();
                    if (!F) break;
                }
            }
        }
        __syncthreads();
    }
    // ---- outputs: per-instance counts of the type, the move counter ------------
    for (uint32_t k = tid; k < ni; k += kK5Threads) {
        p.i_mig_in[s_inst[k]] = s_in[k];
        p.i_mig_out[s_inst[k]] = s_out[k];
    }
    if (tid == 0 && n_moves) atomicAdd(&p.counters[C_MIGRATED], n_moves);
}

// this rank's lists for the exchange (world > 1), written after the sweep:
// blocks [0, T) the migration candidates of type t (NEXT-1), blocks [T, T + R)
// (or [0, R) without migration) the eligible futures of batchable resource r
// (NEXT-4); each walks its resource's bucket items over the K1 blocks in row
// order.  See internal.h (kListWords) for the layout.
__global__ void __launch_bounds__(256) k_lists(ListParams p) {
    __shared__ uint32_t s_pref[257], s_base[256], s_red[8];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t B = p.B;
    const uint32_t nm = p.mig ? p.n_types : 0u;
    const bool is_mig = blockIdx.x < nm;
    uint32_t r, off, total, n_loc;
    uint32_t* L;
    if (is_mig) {
        const uint32_t t = blockIdx.x;
        r = p.R + t;
        off = 0; total = 0;
        for (uint32_t u = 0; u < p.n_types; ++u) {
            const uint32_t c = p.tot_loc[p.R + u];
            off += u < t ? c : 0u;
            total += c;
        }
        L = p.list;
        if (kListHdr + total > kMigWords) {
            if (t == 0 && tid == 0) L[0] = kListOverflow;
            return;
        }
        if (t == 0)
            for (uint32_t u = tid; u < kListHdr; u += blockDim.x)
                L[u] = u == 0 ? total : (u - 1 < p.n_types ? p.tot_loc[p.R + u - 1] : 0u);
        n_loc = p.tot_loc[r];
    } else {
        r = blockIdx.x - nm;
        auto batchable = [&](uint32_t q) {
            const uint32_t t = q < p.n_inst ? p.i_type[q] : q - p.n_inst;
            return p.t_max_batch[t] > 1u;
        };
        // offset of r's entries and the total, over the batchable resources
        uint32_t o = 0, tt = 0;
        for (uint32_t q = tid; q < p.R; q += blockDim.x) {
            const uint32_t c = batchable(q) ? p.tot_loc[q] : 0u;
            o += q < r ? c : 0u;
            tt += c;
        }
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) {
            o += __shfl_xor_sync(0xFFFFFFFFu, o, k);
            tt += __shfl_xor_sync(0xFFFFFFFFu, tt, k);
        }
        if (lane == 0) { s_red[warp] = o; s_pref[warp] = tt; }
        __syncthreads();
        off = 0; total = 0;
        for (uint32_t k = 0; k < 8; ++k) { off += s_red[k]; total += s_pref[k]; }
        __syncthreads();
        L = p.list + kMigWords;
        const uint32_t hdr = 1 + p.R;
        if (hdr + 2 * total > kListWords - kMigWords) {
            if (r == 0 && tid == 0) L[0] = kListOverflow;
            return;
        }
        if (r == 0)
            for (uint32_t q = tid; q < hdr; q += blockDim.x)
                L[q] = q == 0 ? total : (batchable(q - 1) ? p.tot_loc[q - 1] : 0u);
        n_loc = batchable(r) ? p.tot_loc[r] : 0u;
        off = hdr + 2 * off;
    }
    if (n_loc == 0) return;
    uint32_t done = 0;
    for (uint32_t b0 = 0; b0 < B; b0 += 256) {
        const uint32_t bb = b0 + tid;
        const uint32_t c = bb < B ? p.cnt_rb[(size_t)r * B + bb] : 0u;
        if (bb < B) s_base[tid] = p.blk_row0[bb] + p.off_rb[(size_t)r * B + bb];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        __syncthreads();
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t wb = 0;
        for (uint32_t k = 0; k < warp; ++k) wb += s_red[k];
        s_pref[tid] = wb + incl - c;
        if (tid == 255) s_pref[256] = wb + incl;
        __syncthreads();
        const uint32_t n = s_pref[256], nb = min(256u, B - b0);
        for (uint32_t q = tid; q < n; q += 256) {
            uint32_t lo = 0, hi = nb - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (s_pref[mid] <= q) lo = mid;
                else hi = mid - 1;
            }
            const uint2 x = p.items[s_base[lo] + (q - s_pref[lo])];
            if (is_mig) {
                L[kListHdr + off + done + q] = x.y;
                p.mrow[off + done + q] = x.x;
            } else {
                const uint32_t m = p.f_method ? p.f_method[x.x] : 0u;
                L[off + 2 * (done + q)] = (x.y & 0xFFu) | (m << 8);
                L[off + 2 * (done + q) + 1] = p.row_base + x.x;
            }
        }
        done += n;
        __syncthreads();
    }
}

cudaError_t launch_lists(const ListParams& p, cudaStream_t s) {
    const uint32_t nb = (p.mig ? p.n_types : 0u) + (p.batch ? p.R : 0u);
    if (nb == 0) return cudaSuccess;
    k_lists<<<nb, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_migrate(const MigrateParams& p, cudaStream_t s) {
    if (p.n_types == 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.n_types);
    cfg.blockDim = dim3(kK5Threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k5_migrate, p);
}


// load this file's kernels now (CUDA lazy loading would load them at first
// launch, which waits for the device: see nalar_create, NALAR_COLL_PEER)
cudaError_t preload_k_migrate() {
    cudaFuncAttributes a;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k5_migrate)) return e;
    if (cudaError_t e = cudaFuncGetAttributes(&a, k_lists)) return e;
    return cudaSuccess;
}

}  // namespace nalar
