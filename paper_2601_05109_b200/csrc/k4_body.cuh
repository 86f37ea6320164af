// k4_body.cuh -- the body of K4 (capacity-constrained assignment, one block
// of kK4Threads threads per resource), shared by the stand-alone kernel
// (k_assign.cu) and the fused single-rank epoch kernel (k_epoch.cu).  See
// k_assign.cu for the design.
#pragma once
#include "internal.h"

namespace nalar {

namespace {

// K4's block barrier: the whole block for the stand-alone kernel; in the fused
// epoch kernel only the first kK4Threads threads run the assignment, so a
// named barrier (1) over them
template <bool kFused>
__device__ __forceinline__ void k4_sync() {
    if (kFused) asm volatile("bar.sync 1, %0;" ::"n"(kK4Threads) : "memory");
    else __syncthreads();
}
template <bool kFused>
__device__ __forceinline__ int k4_sync_count(bool pred) {
    if (kFused) {
        int r;
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.popc.u32 %0, 1, %2, q;\n\t}"
                     : "=r"(r) : "r"((uint32_t)pred), "n"(kK4Threads) : "memory");
        return r;
    }
    return __syncthreads_count(pred);
}

constexpr uint32_t kSlotCap = 4096;   // phase-B slot table kept in smem up to this size


template <bool kFused, typename Tv>
__device__ __forceinline__ Tv block_sum(Tv v, Tv* red) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    k4_sync<kFused>();
    if (lane == 0) red[warp] = v;
    k4_sync<kFused>();
    Tv s = 0;
#pragma unroll
    for (int k = 0; k < kK4Warps; ++k) s += red[k];
    return s;
}

// number of slots with spare-level > s among the type's instances
__device__ __forceinline__ uint64_t slots_above(const uint32_t* sp2, uint32_t n, uint64_t s) {
    uint64_t a = 0;
    for (uint32_t k = 0; k < n; ++k) a += sp2[k] > s ? sp2[k] - s : 0ull;
    return a;
}

// slot g -> (level s, index j among instances with spare2 >= s)
__device__ __forceinline__ void locate_slot(const uint32_t* sp2, uint32_t n, uint64_t maxs, uint64_t g,
                                            uint64_t* s_out, uint64_t* j_out) {
    uint64_t lo = 1, hi = maxs;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (slots_above(sp2, n, mid) <= g) hi = mid;
        else lo = mid + 1;
    }
    *s_out = lo;
    *j_out = g - slots_above(sp2, n, lo);
}

// the same on a register copy of spare2 (ni <= 16): pure ALU, no LDS chain
__device__ __forceinline__ uint64_t slots_above_r(const uint32_t (&sp)[16], uint64_t s) {
    uint64_t a = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) a += sp[k] > s ? sp[k] - s : 0ull;
    return a;
}
__device__ __forceinline__ void locate_slot_r(const uint32_t (&sp)[16], uint64_t maxs, uint64_t g,
                                              uint64_t* s_out, uint64_t* j_out) {
    uint64_t lo = 1, hi = maxs;
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (slots_above_r(sp, mid) <= g) hi = mid;
        else lo = mid + 1;
    }
    *s_out = lo;
    *j_out = g - slots_above_r(sp, lo);
}

__device__ __forceinline__ uint32_t slot_instance(const uint32_t* sp2, const uint32_t* inst, uint32_t n,
                                                  uint64_t maxs, uint64_t g) {
    uint64_t s, j;
    locate_slot(sp2, n, maxs, g, &s, &j);
    for (uint32_t k = 0; k < n; ++k)
        if (sp2[k] >= s) {
            if (j == 0) return inst[k];
            --j;
        }
    return 0xFFFFFFFFu;
}

// ---- resource reassignment (DESIGN.md Q-ra) -----------
// Type block t: busy_t = sum(load) + eligible futures of t (= load + assigned +
// deferred: every eligible future is assigned or deferred), cap_t, and the kill
// candidate (least load + assigned, ties the highest id).  Global inputs only
// (allreduced loads / totals), so every rank computes the same commands.
template <bool kFused>
__device__ void reassign_stats(const AssignParams& p, bool is_type, uint32_t t, uint32_t ni, uint32_t ha_unp,
                               unsigned long long busy, unsigned long long cap, uint64_t best,
                               unsigned long long* s_rb, unsigned long long* s_rc, uint64_t* s_rbest) {
    // per-thread partials (busy = load + eligible, cap, the kill key) come from
    // the instance loops this block already ran -- no loads here
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        busy += __shfl_xor_sync(0xFFFFFFFFu, busy, o);
        cap += __shfl_xor_sync(0xFFFFFFFFu, cap, o);
        const uint64_t b2 = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        best = b2 < best ? b2 : best;
    }
    if (lane == 0) { s_rb[warp] = busy; s_rc[warp] = cap; s_rbest[warp] = best; }
    k4_sync<kFused>();
    if (!is_type || tid != 0) return;
    unsigned long long B = ha_unp, Cc = 0;          // + unpinned eligible futures of t
    uint64_t bk = ~0ull;
    for (int w = 0; w < kK4Warps; ++w) {
        B += s_rb[w];
        Cc += s_rc[w];
        bk = s_rbest[w] < bk ? s_rbest[w] : bk;
    }
    TypeStat ts;
    ts.busy = B;
    ts.cap = Cc;
    ts.n_inst = ni;
    ts.kill = bk == ~0ull ? -1 : (int32_t)(0xFFFFu - (uint32_t)(bk & 0xFFFFull));
    p.tstat[t] = ts;
    p.t_busy[t] = B > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)B;
    p.t_capsum[t] = Cc > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)Cc;
}

// another block's TypeStat, read past L1 (written before its ticket)
__device__ __forceinline__ TypeStat load_ts(const TypeStat* a, uint32_t t) {
    TypeStat x;
    x.busy = __ldcg(&a[t].busy);
    x.cap = __ldcg(&a[t].cap);
    x.n_inst = __ldcg(&a[t].n_inst);
    x.kill = __ldcg(&a[t].kill);
    return x;
}

// util(a) > util(b) as exact fractions (cap 0 with busy > 0 is infinite)
__device__ __forceinline__ bool util_gt(const TypeStat& a, const TypeStat& b) {
    const bool ia = a.cap == 0 && a.busy > 0, ib = b.cap == 0 && b.busy > 0;
    if (ia || ib) return ia && !ib;
    if (a.cap == 0) return false;
    if (b.cap == 0) return a.busy > 0;
    const unsigned long long xh = __umul64hi(a.busy, b.cap), xl = a.busy * b.cap;
    const unsigned long long yh = __umul64hi(b.busy, a.cap), yl = b.busy * a.cap;
    return xh > yh || (xh == yh && xl > yl);
}

// the last K4 block (ticket) pairs the k-th hottest with the k-th coldest type
__device__ __forceinline__ uint64_t gtimer2() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");   // memory: not hoisted across the code it times
    return t;
}
template <bool kFused>
__device__ void reassign_finish(const AssignParams& p, uint32_t blk, uint32_t* s_last, TypeStat* s_ts, const uint16_t* s_tmin,
                                const uint16_t* s_tmax) {
    unsigned long long* prof = p.prof ? p.prof + (size_t)blk * 8 : nullptr;
    k4_sync<kFused>();
    if (threadIdx.x == 0) {
        // acq_rel ticket: releases this block's TypeStat (written by this same
        // thread) and, for the last block, acquires every other block's -- a
        // full fence.sc would stall each block for microseconds
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(&p.counters[C_RA_TICKET])
                     : "memory");
        *s_last = old == p.R - 1u;
    }
    k4_sync<kFused>();
    if (prof && threadIdx.x == 0) prof[7] = gtimer2();
    if (!*s_last) return;
    const uint32_t T = p.n_types < 64u ? p.n_types : 64u;
    // every input of the pairing staged in parallel (a serial thread-0 walk over
    // global memory would pay one L2 round trip per type)
    __shared__ uint8_t s_cls[64];         // 1 hot, 2 cold
    __shared__ uint8_t s_hot[64], s_cold[64];
    __shared__ uint32_t s_nh, s_nc;
    if (threadIdx.x == 0) { s_nh = 0; s_nc = 0; }
    for (uint32_t t = threadIdx.x; t < T; t += kK4Threads) {
        const TypeStat tt = load_ts(p.tstat, t);
        s_ts[t] = tt;
        const uint32_t mn = s_tmin[t], mx = s_tmax[t];
        uint8_t cl = 0;
        if (tt.n_inst < mx && 100ull * tt.busy > (unsigned long long)p.u_hi_pct * tt.cap) cl = 1;
        else if (tt.n_inst > mn && 100ull * tt.busy < (unsigned long long)p.u_lo_pct * tt.cap) cl = 2;
        s_cls[t] = cl;
    }
    k4_sync<kFused>();
    // rank every hot type by utilisation desc and every cold one by
    // utilisation asc (ties: lower id): all T x T exact comparisons in
    // parallel into bitmasks, then one popcount per type
    __shared__ uint32_t s_gt[64][2], s_eq[64][2];   // bit u of row t: util(u) > util(t) / ==
    for (uint32_t k = threadIdx.x; k < 2 * T; k += kK4Threads) { s_gt[k >> 1][k & 1] = 0; s_eq[k >> 1][k & 1] = 0; }
    k4_sync<kFused>();
    for (uint32_t k = threadIdx.x; k < T * T; k += kK4Threads) {
        const uint32_t t = k / T, u = k - t * T;
        if (s_cls[t] == 0 || s_cls[u] != s_cls[t] || u == t) continue;
        if (util_gt(s_ts[u], s_ts[t])) atomicOr(&s_gt[t][u >> 5], 1u << (u & 31u));
        else if (!util_gt(s_ts[t], s_ts[u])) atomicOr(&s_eq[t][u >> 5], 1u << (u & 31u));
    }
    k4_sync<kFused>();
    for (uint32_t t = threadIdx.x; t < T; t += kK4Threads) {
        const uint8_t cl = s_cls[t];
        if (!cl) continue;
        const unsigned long long gt = s_gt[t][0] | ((unsigned long long)s_gt[t][1] << 32);
        const unsigned long long eq = s_eq[t][0] | ((unsigned long long)s_eq[t][1] << 32);
        unsigned long long same = 0;     // the other types of t's class
        for (uint32_t u = 0; u < T; ++u) same |= (s_cls[u] == cl && u != t) ? 1ull << u : 0ull;
        const unsigned long long lower = t ? (~0ull >> (64 - t)) : 0ull;
        const unsigned long long lt = same & ~gt & ~eq;
        const uint32_t rank = cl == 1 ? __popcll(gt) + __popcll(eq & lower)      // hot: util desc
                                      : __popcll(lt) + __popcll(eq & lower);     // cold: util asc
        if (cl == 1) { s_hot[rank] = (uint8_t)t; atomicAdd(&s_nh, 1u); }
        else { s_cold[rank] = (uint8_t)t; atomicAdd(&s_nc, 1u); }
    }
    k4_sync<kFused>();
    const uint32_t np = s_nh < s_nc ? s_nh : s_nc;
    for (uint32_t k = threadIdx.x; k < np; k += kK4Threads) {
        p.ra_kill[k] = (int16_t)s_ts[s_cold[k]].kill;
        p.ra_prov[k] = (int16_t)s_hot[k];
    }
    if (threadIdx.x != 0) return;
    p.counters[C_RA_PAIRS] = np;
    if (prof) prof[7] = gtimer2() | (1ull << 63);
}


}  // namespace

// kAll: the NALAR_F_PROFILE stamps, resource reassignment (NEXT-2) and the
// streamed-step paths compiled in; the plain epoch's build has none of them
// (code in the body costs the epoch even when a runtime flag skips it)
template <bool kFused, bool kAll = true, bool kProf = kAll>
__device__ __forceinline__ void k4_body(const AssignParams& p, uint32_t blk) {
    __shared__ uint32_t s_inst[NALAR_MAX_INSTANCES_DEV];
    __shared__ uint32_t s_spare[NALAR_MAX_INSTANCES_DEV];   // spare before phase A
    __shared__ uint32_t s_sp2[NALAR_MAX_INSTANCES_DEV];     // spare after phase A
    __shared__ uint32_t s_A[256];                           // global count above level
    __shared__ uint32_t s_before[256];                      // same level, lower ranks
    __shared__ uint32_t s_LA[256];                          // local count above level
    __shared__ uint32_t s_Hg[256];
    __shared__ uint32_t s_Hl[256];
    __shared__ uint32_t s_run[256];
    __shared__ uint32_t s_wc[kK4Warps][256];
    __shared__ uint64_t s_red64[2 * kK4Warps];
    __shared__ uint32_t s_red32[kK4Warps];
    __shared__ uint32_t s_pref[kK4Threads + 1];
    __shared__ uint32_t s_base[kK4Threads];
    __shared__ uint2 s_live[4 * kK4Threads];
    __shared__ uint16_t s_slot[kSlotCap];
    __shared__ uint64_t s_bound;
    __shared__ unsigned long long s_rb[kK4Warps], s_rc[kK4Warps];
    __shared__ uint64_t s_rbest[kK4Warps];
    __shared__ uint32_t s_last;
    __shared__ TypeStat s_ts[64];
    __shared__ uint16_t s_tmin[64], s_tmax[64];
    unsigned long long ra_busy = 0, ra_cap = 0;      // NEXT-2 partials of this thread's instances
    uint64_t ra_best = ~0ull;

    // the verdict is loaded with the first static loads below (one round trip)
    const unsigned long long verdict = (kAll && p.stream_in) ? 0ull : *p.verdict;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t I = p.n_inst, R = p.R, Lv = p.levels, G = p.G, B = p.B;
    // type resources (the longest walks: phase B of a whole type) take the
    // lowest block indices, so they are the first to find a free SM while K1
    // is still running (PDL early launch)
    const uint32_t r = blk < p.n_types ? p.n_inst + blk : blk - p.n_types;
    unsigned long long* prof = (kProf && p.prof) ? p.prof + (size_t)r * 8 : nullptr;
    if (prof && tid == 0) prof[0] = gtimer2();
    const bool is_type = r >= I;
    // ---- static data first: this kernel is a programmatic dependent of the
    // sweep (PDL) and runs this part while the sweep is still working --------
    // (this prologue runs beside K1's last ~2 us: its dependent loads are
    // kept to verdict || type list bounds -> list -> caps, base loads)
    const uint32_t t = is_type ? r - I : p.i_type[r];
    const uint32_t k0 = is_type ? p.type_off[t] : 0u;
    const uint32_t kend = is_type ? p.type_off[t + 1] : 0u;
    const uint32_t cap_r = is_type ? 0u : p.i_cap[r], base_r = is_type ? 0u : p.i_base[r];
    if (verdict) return;   // an invalid table (K0): nothing to assign
    const uint32_t ni = kend - k0;
    if (is_type) {
        for (uint32_t k = tid; k < ni; k += kK4Threads) {
            const uint32_t i = p.type_inst[k0 + k];
            s_inst[k] = i;
            s_spare[k] = p.i_cap[i];          // capacity for now
            s_sp2[k] = p.i_base[i];           // base load for now
        }
    }
    const uint8_t aff = is_type ? p.t_aff[t] : 0;
    const uint32_t blk0 = tid < B ? p.blk_row0[tid] : 0u;
    if (kAll && p.ra_on && tid < 64u && tid < p.n_types) {       // NEXT-2 directives (static)
        s_tmin[tid] = p.t_min_inst ? p.t_min_inst[tid] : 0u;
        s_tmax[tid] = p.t_max_inst ? p.t_max_inst[tid] : 0xFFFFu;
    }
    // everything below reads the sweep's results
    if (!kFused) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (kAll && p.stream_in && *p.verdict) {
        // a streamed step's sweep found an invalid row: publish K0's words to
        // the host (read after the step's one synchronisation) and re-arm them
        if (blk == 0 && threadIdx.x == 0) {
            volatile unsigned long long* h = p.host_err;
            h[0] = atomicExch(&p.err[0], ~0ull);
            h[1] = atomicExch(&p.err[1], 0ull);
        }
        return;
    }
    if (p.rb && blk == 0 && tid == 0) {
        // world > 1: the ranks' shards must be consecutive in the global row
        // order (global rank = the row order across shards); ranks without
        // rows or with an unknown base (after a delta) are not checked
        uint32_t prev_end = 0xFFFFFFFFu;
        bool bad = false;
        for (uint32_t s = 0; s < G; ++s) {
            const uint32_t base = p.rb[2 * s], n = p.rb[2 * s + 1];
            if (n == 0u) continue;
            if (base == 0xFFFFFFFFu) { prev_end = 0xFFFFFFFFu; continue; }
            if (prev_end != 0xFFFFFFFFu && base != prev_end) bad = true;
            prev_end = base + n;
        }
        if (bad) *(volatile unsigned long long*)p.order_err = 1ull;
    }
    if (prof && tid == 0) prof[4] = gtimer2();

    // ---- every load of the sweep's results this block needs first, issued
    // together (one L2 round trip instead of a chain of dependent ones) -----
    const uint32_t lv = tid;
    uint32_t hg = 0, hb = 0, hl = 0;
    if (lv < Lv) {
        for (uint32_t s = 0; s < G; ++s) {
            const uint32_t h = p.H[((size_t)s * p.Rh + r) * Lv + lv];
            hg += h;
            if (s < p.slot) hb += h;
            if (s == p.slot) hl = h;
        }
    }
    uint32_t base_part = 0;                  // offset of r's region of the assignment list
    for (uint32_t q = tid; q < r; q += kK4Threads) base_part += p.tot_loc[q];
    const uint32_t cnt0 = tid < B ? p.cnt_rb[(size_t)r * B + tid] : 0u;   // first 256 K1 blocks
    const uint32_t off0 = tid < B ? p.off_rb[(size_t)r * B + tid] : 0u;
    uint32_t ls0 = 0, ha0 = 0;
    uint64_t my_load = 0;                     // load of instance k == tid of the type (kept for NEXT-2)
    const uint32_t ha_unp = (kAll && is_type && p.ra_on && tid == 0) ? p.tot[r] : 0u;   // unpinned eligible of t
    if (is_type) {
        if (tid < ni) { ls0 = p.load_sum[s_inst[tid]]; ha0 = p.tot[s_inst[tid]]; }
    } else if (tid == 0) {
        ls0 = p.load_sum[r];
    }

    // ---- instances of type t: load, spare, phase-A admissions (all ranks) ----
    if (is_type) {
        for (uint32_t k = tid; k < ni; k += kK4Threads) {
            const uint32_t i = s_inst[k];
            const uint64_t load = (uint64_t)s_sp2[k] + (k < kK4Threads ? ls0 : p.load_sum[i]);
            const uint64_t cap = s_spare[k];
            const uint32_t spare = (uint32_t)(cap > load ? cap - load : 0ull);
            const uint32_t ha = k < kK4Threads ? ha0 : p.tot[i];
            s_spare[k] = spare;
            s_sp2[k] = spare - (ha < spare ? ha : spare);
            p.i_load[i] = load > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)load;
            if (k == tid) my_load = load;
            ra_busy += load + ha;
            ra_cap += cap;
            p.i_spare[i] = spare;
        }
    } else if (tid == 0) {
        const uint64_t load = (uint64_t)base_r + ls0;
        s_bound = cap_r > load ? cap_r - load : 0ull;
    }
    // ---- level histogram of r: global, lower-ranks, local ------------------
    {
        s_Hg[lv] = hg;
        s_Hl[lv] = hl;
        s_before[lv] = hb;
        s_run[lv] = 0;
#pragma unroll
        for (int k = 0; k < kK4Warps; ++k) s_wc[k][lv] = 0;
    }
    k4_sync<kFused>();
    if (prof && tid == 0 && !p.ra_on) prof[7] = gtimer2();    // loads of the sweep's results landed

    // ---- bound of this resource; suffix sums over levels ------------------
    uint64_t bound, maxs = 0;
    {
        uint64_t sum = 0, mx = 0;
        for (uint32_t k = tid; k < ni; k += kK4Threads) { sum += s_sp2[k]; mx = max(mx, (uint64_t)s_sp2[k]); }
        // count strictly above each level: warp suffix scans + per-warp totals
        static_assert(kK4Threads == 256, "one thread per level");
        const uint32_t hg = s_Hg[tid], hl = s_Hl[tid];
        uint32_t xg = hg, xl = hl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yg = __shfl_down_sync(0xFFFFFFFFu, xg, o);
            const uint32_t yl = __shfl_down_sync(0xFFFFFFFFu, xl, o);
            if (lane + o < 32) { xg += yg; xl += yl; }
        }
        uint32_t bp = base_part;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
            mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            bp += __shfl_xor_sync(0xFFFFFFFFu, bp, o);
        }
        if (lane == 0) {
            s_wc[0][warp] = xg;
            s_wc[1][warp] = xl;
            s_wc[2][warp] = bp;
            s_red64[warp] = sum;
            s_red64[kK4Warps + warp] = mx;
        }
        k4_sync<kFused>();
        uint32_t ag = xg - hg, al = xl - hl;
        for (uint32_t k = warp + 1; k < (uint32_t)kK4Warps; ++k) { ag += s_wc[0][k]; al += s_wc[1][k]; }
        s_A[tid] = ag;
        s_LA[tid] = al;
        uint64_t bs = 0;
        base_part = 0;
#pragma unroll
        for (int k = 0; k < kK4Warps; ++k) {
            bs += s_red64[k];
            maxs = max(maxs, s_red64[kK4Warps + k]);
            base_part += s_wc[2][k];
        }
        bound = is_type ? bs : s_bound;
        // number of this rank's futures admitted on r (closed form per level:
        // every input is this thread's own), reduced across the barrier below
        uint32_t adm_lv = 0;
        if (tid < Lv) {
            const uint64_t pre = (uint64_t)ag + s_before[tid];
            if (pre < bound) {
                const uint64_t room = bound - pre;
                adm_lv = (uint32_t)(room < hl ? room : hl);
            }
        }
        adm_lv = __reduce_add_sync(0xFFFFFFFFu, adm_lv);
        if (lane == 0) s_red32[warp] = adm_lv;
        k4_sync<kFused>();
        if (tid < 3 * kK4Warps) s_wc[tid >> 3][tid & 7] = 0;
    }
    const uint32_t list_base = base_part;
    uint32_t n_adm = 0;
#pragma unroll
    for (int k = 0; k < kK4Warps; ++k) n_adm += s_red32[k];
    if (prof && tid == 0) prof[1] = gtimer2();
    if (tid == 0) {
        p.n_adm[r] = n_adm;
        if (n_adm) atomicAdd(&p.counters[C_ASSIGNED], n_adm);
    }

    // ---- per-instance assigned counts + phase-B slot table (type blocks) ----
    const bool table = is_type && bound <= kSlotCap;
    if (is_type) {
        const uint64_t n_t = (uint64_t)s_A[0] + s_Hg[0];
        const uint64_t used = n_t < bound ? n_t : bound;
        // small types (ni <= 16, the common case): spare2 in registers, so the
        // slot arithmetic below is ALU only instead of chains of shared loads
        const bool small = ni <= 16u;
        uint32_t spr[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) spr[k] = (small && (uint32_t)k < ni) ? s_sp2[k] : 0u;
        uint64_t s0 = 0, j0 = 0;
        if (used) {
            if (small && maxs <= 32u) {
                // every candidate level at once, one per lane: the level of
                // slot g is the smallest s with slots_above(s) <= g
                const uint32_t sv = lane + 1u;
                uint32_t above = 0;
#pragma unroll
                for (int k = 0; k < 16; ++k) above += spr[k] > sv ? spr[k] - sv : 0u;
                const uint32_t okm = __ballot_sync(0xFFFFFFFFu, sv <= maxs && above <= used - 1);
                const uint32_t lvl = __ffs(okm);                 // = s0 (1-based lane index)
                s0 = lvl;
                j0 = (used - 1) - __shfl_sync(0xFFFFFFFFu, above, lvl - 1u);
            } else if (small) {
                locate_slot_r(spr, maxs, used - 1, &s0, &j0);
            } else {
                locate_slot(s_sp2, ni, maxs, used - 1, &s0, &j0);
            }
        }
        for (uint32_t k = tid; k < ni; k += kK4Threads) {
            uint64_t asg = s_spare[k] - s_sp2[k];     // phase A
            if (used) {
                const uint64_t sp = s_sp2[k];
                asg += sp > s0 ? sp - s0 : 0ull;
                if (sp >= s0) {
                    uint64_t idx = 0;
                    if (small) {
#pragma unroll
                        for (int q = 0; q < 16; ++q) idx += ((uint32_t)q < k && spr[q] >= s0) ? 1u : 0u;
                    } else {
                        for (uint32_t q = 0; q < k; ++q) idx += s_sp2[q] >= s0;
                    }
                    asg += idx <= j0;
                }
            }
            p.i_assigned[s_inst[k]] = (uint32_t)asg;
            {   // NEXT-2 kill key: least load + assigned, ties the highest id
                const uint64_t la = asg + (k == tid ? my_load : (uint64_t)p.i_load[s_inst[k]]);
                const uint64_t key = ((la > 0xFFFFFFFFull ? 0xFFFFFFFFull : la) << 32) | (0xFFFFu - s_inst[k]);
                ra_best = key < ra_best ? key : ra_best;
            }
        }
        if (table && n_adm && ni <= 16u) {
            // slots in (level desc, instance asc) order, all at once: slot
            // (s, k) sits after every slot of a higher level and after the
            // level-s slots of lower instances
            // one (instance k, level sv) pair per thread
            const uint32_t npair = ni * (uint32_t)maxs;
            for (uint32_t idx = tid; idx < npair; idx += kK4Threads) {
                const uint32_t k = idx / (uint32_t)maxs, sv = idx - k * (uint32_t)maxs + 1u;
                if (sv > s_sp2[k]) continue;
                uint32_t pos = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t x = spr[j];
                    pos += (x > sv ? x - sv : 0u) + ((uint32_t)j < k && x >= sv ? 1u : 0u);
                }
                s_slot[pos] = (uint16_t)s_inst[k];
            }
        } else if (table && n_adm && warp == 0) {
            // slots in (level desc, instance asc) order, one level per step
            uint32_t pos = 0;
            for (uint64_t sv = maxs; sv >= 1; --sv) {
                for (uint32_t k0 = 0; k0 < ni; k0 += 32) {
                    const uint32_t k = k0 + lane;
                    const bool in = k < ni && s_sp2[k] >= sv;
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, in);
                    if (in) s_slot[pos + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)s_inst[k];
                    pos += __popc(bal);
                }
            }
        }
    }
    if (prof && tid == 0) prof[2] = gtimer2();
    if (kAll && p.ra_on) reassign_stats<kFused>(p, is_type, t, ni, ha_unp, ra_busy, ra_cap, ra_best, s_rb, s_rc, s_rbest);
    if (n_adm == 0) {
        if (prof && tid == 0) prof[3] = gtimer2();
        if (kAll && p.ra_on) reassign_finish<kFused>(p, blk, &s_last, s_ts, s_tmin, s_tmax);
        return;
    }
    k4_sync<kFused>();

    // ---- walk this rank's futures of r in row order --------------------------
    // pass 1 compacts the live ones (level not yet full), pass 2 ranks them
    uint32_t found = 0;
    for (uint32_t b0 = 0; b0 < B && found < n_adm; b0 += kK4Threads) {
        // prefix of per-K1-block counts and item bases for blocks [b0, b0 + 256)
        const uint32_t bb = b0 + tid;
        uint32_t c = 0;
        if (bb < B) {
            c = b0 == 0 ? cnt0 : p.cnt_rb[(size_t)r * B + bb];
            s_base[tid] = b0 == 0 ? blk0 + off0 : p.blk_row0[bb] + p.off_rb[(size_t)r * B + bb];
        }
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        k4_sync<kFused>();
        if (lane == 31) s_red32[warp] = incl;
        k4_sync<kFused>();
        uint32_t wb = 0;
        for (uint32_t k = 0; k < warp; ++k) wb += s_red32[k];
        s_pref[tid] = wb + incl - c;
        if (tid == kK4Threads - 1) s_pref[kK4Threads] = wb + incl;
        k4_sync<kFused>();
        const uint32_t total = s_pref[kK4Threads];
        const uint32_t nb = min((uint32_t)kK4Threads, B - b0);
        if (prof && tid == 0 && b0 == 0) prof[5] = gtimer2();
        for (uint32_t q0 = 0; q0 < total && found < n_adm; q0 += 4 * kK4Threads) {
            // pass 1: four consecutive items per thread
            uint2 it[4];
            uint32_t live = 0;                // bit j: item j is live (register-resident, no local memory)
            const uint32_t qa = q0 + 4 * tid;
            if (qa < total) {
                uint32_t lo = 0, hi = nb - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (s_pref[mid] <= qa) lo = mid;
                    else hi = mid - 1;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t q = qa + j;
                    it[j] = make_uint2(0u, 0u);
                    if (q < total) {
                        if (lo + 1 < nb && s_pref[lo + 1] <= q) {
                            // item q is in a later block: binary search (a sparse
                            // resource has long runs of empty blocks -- walking
                            // them one LDS at a time cost microseconds)
                            uint32_t l2 = lo + 1, h2 = nb - 1;
                            while (l2 < h2) {
                                const uint32_t mid = (l2 + h2 + 1) >> 1;
                                if (s_pref[mid] <= q) l2 = mid;
                                else h2 = mid - 1;
                            }
                            lo = l2;
                        }
                        it[j] = p.items[s_base[lo] + (q - s_pref[lo])];
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (qa + j < total && (uint64_t)s_A[it[j].y] + s_before[it[j].y] < bound) live |= 1u << j;
            }
            const uint32_t nl = __popc(live);
            uint32_t li = nl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, li, o);
                if (lane >= (uint32_t)o) li += y;
            }
            if (lane == 31) s_red32[warp] = li;
            k4_sync<kFused>();
            uint32_t lb = 0, n_live = 0;
            for (uint32_t k = 0; k < (uint32_t)kK4Warps; ++k) {
                lb += k < warp ? s_red32[k] : 0u;
                n_live += s_red32[k];
            }
            lb += li - nl;
            {
                uint32_t o = lb;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if ((live >> j) & 1u) s_live[o++] = it[j];
            }
            k4_sync<kFused>();
            if (prof && tid == 0 && q0 == 0 && b0 == 0) prof[6] = gtimer2() + 0 * n_live;
            // pass 2: stable rank of each live item inside its level
            for (uint32_t j0 = 0; j0 < n_live; j0 += kK4Threads) {
                const uint32_t j = j0 + tid;
                const bool live = j < n_live;
                uint32_t row = 0, lv = 0xFFFFu;
                if (live) { row = s_live[j].x; lv = s_live[j].y; }
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, lv);
                const uint32_t wrank = __popc(peers & ((1u << lane) - 1u));
                if (live && (__ffs(peers) - 1) == (int)lane) s_wc[warp][lv] = __popc(peers);
                k4_sync<kFused>();
                bool adm = false;
                uint32_t rank = 0;
                if (live) {
                    rank = s_run[lv] + wrank;
                    for (uint32_t k = 0; k < warp; ++k) rank += s_wc[k][lv];
                    adm = (uint64_t)s_A[lv] + s_before[lv] + rank < bound;
                }
                k4_sync<kFused>();
                {
                    uint32_t add = 0;
#pragma unroll
                    for (int k = 0; k < kK4Warps; ++k) { add += s_wc[k][tid]; s_wc[k][tid] = 0; }
                    s_run[tid] += add;
                }
                if (adm) {
                    const uint64_t g = (uint64_t)s_A[lv] + s_before[lv] + rank;
                    int16_t inst = (int16_t)r;
                    if (is_type)
                        inst = (int16_t)(table ? s_slot[g] : slot_instance(s_sp2, s_inst, ni, maxs, g));
                    p.status[row] = 7;
                    p.instance[row] = inst;
                    p.new_pin[row] = (uint8_t)(is_type && aff != 0);
                    if (kAll) {
                        if (p.o_status) p.o_status[row] = 7;
                        if (p.o_instance) p.o_instance[row] = inst;
                        if (p.o_new_pin) p.o_new_pin[row] = (uint8_t)(is_type && aff != 0);
                    }
                    const uint32_t pos = list_base + s_LA[lv] + rank;
                    p.assign_row[pos] = row;
                    p.assign_inst[pos] = inst;
                }
                found += k4_sync_count<kFused>(adm);
            }
        }
    }
    if (prof && tid == 0) prof[3] = gtimer2();
    if (kAll && p.ra_on) reassign_finish<kFused>(p, blk, &s_last, s_ts, s_tmin, s_tmax);
}

}  // namespace nalar
