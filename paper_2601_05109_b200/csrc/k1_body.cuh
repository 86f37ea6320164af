// k1_body.cuh -- the body of K1 (the per-workflow sweep), shared by the
// stand-alone sweep kernel (k_sweep.cu) and the fused single-rank epoch
// kernel (k_epoch.cu).  See k_sweep.cu for the design.
#pragma once
#include <algorithm>

#include "internal.h"

namespace nalar {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (TMA engine).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// step-done flag of a long workflow's transfer (P2a -> P2b hand-off inside the
// block): the producer warp publishes with release, the composing warp acquires
__device__ __forceinline__ void st_release_u16(uint16_t* p, uint16_t v) {
    asm volatile("st.release.cta.b16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u16(const uint16_t* p) {
    uint16_t v;
    asm volatile("ld.acquire.cta.b16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return v;
}
constexpr uint32_t kStepDone = 0x4000u;   // aux[c0] bit: the step's transfer is written

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");   // memory: not hoisted across the code it times
    return t;
}

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// plan of one staged array: aligned global window copied into smem
struct Win {
    const uint8_t* src;
    uint32_t pre, bytes;
};
__device__ __forceinline__ Win window(const void* base, size_t elem, size_t lo, size_t hi) {
    const uint8_t* s = (const uint8_t*)base + lo * elem;
    const uint8_t* a = (const uint8_t*)((uintptr_t)s & ~(uintptr_t)15);
    Win w;
    w.src = a;
    w.pre = (uint32_t)(s - a);
    w.bytes = (uint32_t)align16(w.pre + (hi - lo) * elem);
    return w;
}

// Settling of a step transfer (see transfer_step): slots are biased u16
// halves of NP packed words; a round is K shuffles per word (K = the widest
// row's in-step predecessors) and a native u16x2 max tree.  Issue slots, not
// the shuffle pipe, bound P2a (all 16 warps settle at once), so the round is
// kept to K + (K - 1) + 3 instructions per word.
template <int K, int NP, bool kAnc>
__device__ __forceinline__ uint32_t settle_pairs(uint32_t& h0, uint32_t& h1, uint32_t& h2, uint32_t& h3, bool has,
                                                 uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3,
                                                 uint32_t& anc, uint32_t am) {
    auto vmax2 = [](uint32_t x, uint32_t y) {
        uint32_t r;
        asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
        return r;
    };
    auto round = [&](uint32_t& x) {
        uint32_t m = __shfl_sync(0xFFFFFFFFu, x, s0);
        if (K > 1) m = vmax2(m, __shfl_sync(0xFFFFFFFFu, x, s1));
        if (K > 2) m = vmax2(m, __shfl_sync(0xFFFFFFFFu, x, s2));
        if (K > 3) m = vmax2(m, __shfl_sync(0xFFFFFFFFu, x, s3));
        x = has ? vmax2(x, m + 0x00010001u) : x;
    };
    // (kAnc) the in-step doom ancestors ride along: a pending row collects
    // its pending DEP predecessors' ancestor masks (am bit i: slot i is one)
    auto round_anc = [&]() {
        uint32_t m = __shfl_sync(0xFFFFFFFFu, anc, s0) & (0u - (am & 1u));
        if (K > 1) m |= __shfl_sync(0xFFFFFFFFu, anc, s1) & (0u - ((am >> 1) & 1u));
        if (K > 2) m |= __shfl_sync(0xFFFFFFFFu, anc, s2) & (0u - ((am >> 2) & 1u));
        if (K > 3) m |= __shfl_sync(0xFFFFFFFFu, anc, s3) & (0u - ((am >> 3) & 1u));
        anc |= m;
    };
    auto all = [&]() {
        round(h0);
        if (NP > 1) round(h1);
        if (NP > 2) { round(h2); round(h3); }
        if (kAnc) round_anc();
    };
    uint32_t it = 0;
    for (;;) {
        all();
        all();
        all();
        const uint32_t b0 = h0, b1 = h1, b2 = h2, b3 = h3, ba = anc;
        all();
        ++it;
        if (!__any_sync(0xFFFFFFFFu, h0 != b0 || h1 != b1 || h2 != b2 || h3 != b3 || (kAnc && anc != ba))) break;
    }
    return it;
}

// In-step doom closure (doom reaches a PENDING row through a DEP edge from a
// doomed / FAILED row; Q3).  Rows of a step are in topological order, so one
// ascending walk over the lanes settles it: every lane's DEP-predecessor mask
// is fetched by 32 independent shuffles issued back to back, then the walk is
// a chain of three ALU ops per lane (instead of one ballot per link of the
// longest in-step chain).
__device__ __forceinline__ bool doom_closure(bool doom, bool pend, uint32_t need_dep) {
    uint32_t D = __ballot_sync(0xFFFFFFFFu, doom);
    if (D == 0u) return false;
    const uint32_t mine = pend ? need_dep : 0u;       // only PENDING rows become doomed
    uint32_t nj[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) nj[j] = __shfl_sync(0xFFFFFFFFu, mine, j);
#pragma unroll
    for (int j = 0; j < 32; ++j) D |= (nj[j] & D) ? 1u << j : 0u;
    return (D >> (threadIdx.x & 31u)) & 1u;
}


}  // namespace

// The body is instantiated twice: for a staged block every table pointer
// derives from the shared-memory window, so the compiler emits LDS/STS; for an
// unstaged (oversized) block they point into global memory.
// kIn: streamed-step staging / validation; kNext: HoL-migration candidates and
// batch-head presets (the NEXT-1 / NEXT-4 modes) -- compiled in only where used
template <bool kStaged, bool kOut = false, bool kProf = false, bool kIn = false, bool kNext = false>
__device__ __forceinline__ void k1_body(const SweepParams& p, uint8_t* smem, const uint4 ca, const uint4 cb) {
    const uint32_t b = ca.x;
    // NALAR_F_PROFILE stamps only in the profiling build: a null pointer known
    // at compile time removes every stamp and its branch from the production
    // sweep (code in P3 costs the plain epoch even when it never runs)
    unsigned long long* const prof = kProf ? p.prof : nullptr;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t T = p.n_types, I = p.n_inst, R = p.R, Rh = p.Rh, Lv = p.levels;

    const uint32_t w0 = ca.y, w1 = ca.z;
    const uint32_t r0 = ca.w, r1 = cb.x;
    const uint32_t e0 = cb.y, e1 = cb.z;
    const uint32_t nr = r1 - r0, ne = e1 - e0, nw = w1 - w0;
    constexpr bool staged = kStaged;
    unsigned long long* bprof = prof ? prof + (size_t)p.n_wf * 2 + b * 8 : nullptr;
    if (bprof && tid == 0) bprof[3] = gtimer();
    // the point where the assignment kernel may launch (PDL) is p.trig; it
    // waits for this grid's completion before reading anything the sweep writes
    if (p.trig == 0) asm volatile("griddepcontrol.launch_dependents;");

    // ---- carve the fixed part --------------------------------------------
    uint8_t* sp = smem;
    uint64_t* mbar = (uint64_t*)sp;
    uint32_t* s_ticket = (uint32_t*)(sp + 8);
    uint32_t* s_cnt = (uint32_t*)(sp + 16);      // [0] ready [1] elig [2] doomed [3] long workflows
    sp += 64;
    uint32_t* s_load = (uint32_t*)sp;
    sp += 4 * (size_t)I;
    uint32_t* s_rcnt = (uint32_t*)sp;
    sp += 4 * (size_t)Rh;
    uint32_t* s_roff = (uint32_t*)sp;
    sp += 4 * (size_t)Rh;
    uint32_t* s_list = (uint32_t*)sp;
    sp += 4 * kK1Threads;
    uint32_t* s_wc = (uint32_t*)sp;
    sp += 4 * kK1Warps;
    uint32_t* s_wcc = (uint32_t*)sp;                 // [kP5Chunks][kK1Warps] eligible counts (P5)
    sp += 4 * kP5Chunks * kK1Warps;
    uint8_t* s_aff = sp;

    // ---- per-workflow tables (always in smem) -------------------------------
    uint8_t* q = smem + p.fixed_smem;
    uint32_t* s_winfl = (uint32_t*)q;                        // [nw][2] types with futures in flight (bitset)
    uint32_t* s_wfp = (uint32_t*)(q + 8 * (size_t)nw);       // [nw][T] first PENDING non-doomed row
    uint32_t* s_wfru = s_wfp + (size_t)nw * T;               // [nw][T] first ready unpinned row
    q += align16((size_t)nw * (8 * (size_t)T + 8));
    uint32_t* s_wrnd = (uint32_t*)q;                         // [nw] max retry round
    q += align16(4 * (size_t)nw);
    uint32_t* s_lpref = (uint32_t*)q;                        // [nw+1] long-workflow step tasks
    q += align16(4 * ((size_t)nw + 1));
    uint32_t* s_perm = (uint32_t*)q;                         // [nw] task order, largest first
    q += align16(4 * (size_t)nw);
    uint32_t* s_agg = (uint32_t*)q;                          // [nw][8] counts (P3), max depth (sweep)
    q += align16(32 * (size_t)nw);
    uint32_t* s_khome = (uint32_t*)q;                        // [nw][T] session home (min pin) -- NEXT-3
    uint32_t* s_klev = s_khome + (size_t)nw * T;             // [nw][T] 1 + max level of live futures
    q += align16(8 * (size_t)nw * T);
    uint32_t* s_mq = (uint32_t*)q;                           // [nw][T] QUEUED futures (NEXT-1)
    uint32_t* s_mqrow = s_mq + (size_t)nw * T;               // [nw][T] a QUEUED row | candidate bit
    q += align16(8 * (size_t)nw * T);
    uint32_t* s_mrun = (uint32_t*)q;                         // [nw][2] types with a RUNNING future
    q += align16(8 * (size_t)nw);

    // ---- the block's slice of the table: staged in smem by TMA, or in place --
    const uint8_t* st;    // state, type, round, pin, executor: indexed by local row
    const uint8_t* ty;
    const uint8_t* rd;
    const int16_t* pn;
    const int16_t* ex;
    const uint32_t* eo;   // absolute edge offsets, indexed by local row
    const uint32_t* ed;   // edges, indexed by (edge - e0)
    const uint32_t* wfo;  // absolute workflow row offsets, indexed by local workflow
    const int32_t* wpr;   // workflow priorities, indexed by local workflow
    uint16_t* dep;        // depth (work / output)
    uint8_t* flg;         // FL_* (work)
    uint8_t* lev;         // level (work / output)
    uint32_t* tlo;        // step transfer bytes (long workflows): inputs 0..3
    uint32_t* thi;        //   inputs 4..6, root path in byte 7
    uint32_t* ifc;        //   interface rows of the step starting at this row
    uint32_t* ndp;        //   in-step doom ancestors (lane mask)
    uint16_t* aux;        //   DEP-from-interface mask, FAILED pred, all-resolved, k, ok
    if (staged) {
        // a streamed step stages the rows from the caller's pinned host arrays
        const bool si = kIn && p.stream_in != 0u;
        const Win ws = window(si ? p.src.state : p.f_state, 1, r0, r1);
        const Win wt = window(si ? p.src.type : p.f_type, 1, r0, r1);
        const Win wr = window(si ? p.src.round : p.f_round, 1, r0, r1);
        const Win wp = window(si ? p.src.pin : p.f_pin, 2, r0, r1);
        const Win wx = window(si ? p.src.exec : p.f_exec, 2, r0, r1);
        const Win we = window(si ? p.src.eoff : p.f_edge_off, 4, r0, r1 + 1);
        const Win wg = window(si ? p.src.edges : p.edges, 4, e0, e1);
        const Win wo = window(p.wf_fut_off, 4, w0, w1 + 1), wq = window(p.wf_prio, 4, w0, w1);
        uint8_t* d_s = q;   q += align16(nr + 32);
        uint8_t* d_t = q;   q += align16(nr + 32);
        uint8_t* d_r = q;   q += align16(nr + 32);
        uint8_t* d_p = q;   q += align16(2 * (size_t)nr + 32);
        uint8_t* d_x = q;   q += align16(2 * (size_t)nr + 32);
        uint8_t* d_e = q;   q += align16(4 * ((size_t)nr + 1) + 32);
        uint8_t* d_g = q;   q += align16(4 * (size_t)ne + 32);
        uint8_t* d_o = q;   q += align16(4 * ((size_t)nw + 1) + 32);
        uint8_t* d_q = q;   q += align16(4 * (size_t)nw + 32);
        dep = (uint16_t*)q; q += align16(2 * (size_t)nr);
        flg = q;            q += align16(nr);
        lev = q;            q += align16(nr);
        tlo = (uint32_t*)q; q += align16(4 * (size_t)nr);
        thi = (uint32_t*)q; q += align16(4 * (size_t)nr);
        ifc = (uint32_t*)q; q += align16(4 * (size_t)nr);
        ndp = (uint32_t*)q; q += align16(4 * (size_t)nr);
        aux = (uint16_t*)q;
        if (tid == 0) {
            mbar_init(mbar, 1);
            if (kIn && p.stream_in && blockIdx.x >= p.stage_window) {
                // pacing of a streamed step's host reads (see SweepParams)
                asm volatile("griddepcontrol.wait;" ::: "memory");   // the counter is the zero kernel's
                const uint32_t need = blockIdx.x - p.stage_window;
                const uint64_t t0 = gtimer();
                for (;;) {
                    uint32_t v;
                    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p.stage_ctr) : "memory");
                    if (v >= need || gtimer() - t0 > 200000ull) break;   // a hint, never a hang
                    __nanosleep(256);
                }
            }
            const uint32_t total = ws.bytes + wt.bytes + wr.bytes + wp.bytes + wx.bytes + we.bytes +
                                   (ne ? wg.bytes : 0u) + wo.bytes + (nw ? wq.bytes : 0u);
            mbar_arrive_expect_tx(mbar, total);
            bulk_g2s(d_s, ws.src, ws.bytes, mbar);
            bulk_g2s(d_t, wt.src, wt.bytes, mbar);
            bulk_g2s(d_r, wr.src, wr.bytes, mbar);
            bulk_g2s(d_p, wp.src, wp.bytes, mbar);
            bulk_g2s(d_x, wx.src, wx.bytes, mbar);
            bulk_g2s(d_e, we.src, we.bytes, mbar);
            if (ne) bulk_g2s(d_g, wg.src, wg.bytes, mbar);
            bulk_g2s(d_o, wo.src, wo.bytes, mbar);
            if (nw) bulk_g2s(d_q, wq.src, wq.bytes, mbar);
        }
        st = d_s + ws.pre;
        ty = d_t + wt.pre;
        rd = d_r + wr.pre;
        pn = (const int16_t*)(d_p + wp.pre);
        ex = (const int16_t*)(d_x + wx.pre);
        eo = (const uint32_t*)(d_e + we.pre);
        ed = (const uint32_t*)(d_g + wg.pre);
        wfo = (const uint32_t*)(d_o + wo.pre);
        wpr = (const int32_t*)(d_q + wq.pre);
    } else {
        st = p.f_state + r0;
        ty = p.f_type + r0;
        rd = p.f_round + r0;
        pn = p.f_pin + r0;
        ex = p.f_exec + r0;
        eo = p.f_edge_off + r0;
        ed = p.edges + e0;
        wfo = p.wf_fut_off + w0;
        wpr = p.wf_prio + w0;
        dep = p.depth + r0;
        flg = p.g_flags + r0;
        lev = p.level + r0;
        tlo = p.g_tlo + r0;
        thi = p.g_thi + r0;
        ifc = p.g_ifc + r0;
        ndp = p.g_ndp + r0;
        aux = p.g_aux + r0;
    }

    // ---- zero block state while the copies are in flight ------------------
    for (uint32_t i = tid; i < I; i += kK1Threads) s_load[i] = 0;
    for (uint32_t r = tid; r < Rh; r += kK1Threads) s_rcnt[r] = 0;
    for (uint32_t t = tid; t < T; t += kK1Threads) s_aff[t] = p.t_aff[t];
    for (uint32_t k = tid; k < nw * T; k += kK1Threads) {
        s_wfp[k] = 0xFFFFFFFFu; s_wfru[k] = 0xFFFFFFFFu; s_khome[k] = 0xFFFFFFFFu; s_klev[k] = 0u;
        s_mq[k] = 0u; s_mqrow[k] = 0u;
    }
    for (uint32_t k = tid; k < nw; k += kK1Threads) {
        s_winfl[2 * k] = 0u; s_winfl[2 * k + 1] = 0u; s_mrun[2 * k] = 0u; s_mrun[2 * k + 1] = 0u;
        s_perm[k] = p.wf_perm[w0 + k];
    }
    for (uint32_t k = tid; k < 8 * nw; k += kK1Threads) s_agg[k] = 0;
    for (uint32_t k = tid; k < nr; k += kK1Threads) aux[k] = 0;   // step-done flags
    uint32_t* s_bad = (uint32_t*)(smem + 32);      // streamed step: an invalid row in this block
    if (tid == 0) {
        *s_ticket = 0;
        s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
        *s_bad = 0;
    }
    __syncthreads();
    if (staged) mbar_wait(mbar, 0);
    if (kIn && staged && p.stream_in && tid == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        atomicAdd(p.stage_ctr, 1u);
    }
    if (kIn && staged && p.stream_in) {
        // K0's input contract (k_validate.cu validate_row, Q1) on the
        // staged rows: an edge points to an earlier row of the same workflow,
        // states / types in range, pins and executors name an instance of the
        // row's type; the smallest bad row over all blocks wins (atomicMin).
        // Offsets outside the block's edge window mean non-monotone offsets.
        const StreamIn& q = p.src;
        bool structural = false;
        for (uint32_t f = tid; f < nr; f += kK1Threads) {
            uint32_t lo = 0, hi = nw - 1;
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (wfo[mid] - r0 <= f) lo = mid;
                else hi = mid - 1;
            }
            const uint32_t a = wfo[lo];
            const uint32_t eb = eo[f], ee = eo[f + 1];
            if (ee < eb || ee > q.n_edges || eb < e0 || ee > e1) { structural = true; continue; }
            const uint32_t stv = st[f], tyv = ty[f];
            const int pinv = pn[f], exv = ex[f];
            bool ok = stv <= 4u && tyv < q.n_types;
            if (ok && pinv != -1 && (pinv < 0 || (uint32_t)pinv >= q.n_inst || q.i_type[pinv] != tyv)) ok = false;
            if (ok && (stv == 1u || stv == 2u) && (exv < 0 || (uint32_t)exv >= q.n_inst || q.i_type[exv] != tyv))
                ok = false;
            for (uint32_t e = eb; ok && e < ee; ++e) {
                const uint32_t x = ed[e - e0] & 0x7FFFFFFFu;
                if (x < a || x >= r0 + f) ok = false;
            }
            if (!ok) {
                atomicMin(&q.err[0], (unsigned long long)(r0 + f));
                *s_bad = 1u;
            }
        }
        if (structural) {
            atomicOr(&q.err[1], 1ull);
            *s_bad = 1u;
        }
        __syncthreads();
        if (*s_bad) {
            // the zero kernel clears the verdict: set it only after that grid
            if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
            if (tid == 0) *q.verdict = 1ull;
            return;
        }
        // the device copy of the table (later epochs / deltas read it)
        for (uint32_t i = tid; i < nr; i += kK1Threads) {
            const_cast<uint8_t*>(p.f_state)[r0 + i] = st[i];
            const_cast<uint8_t*>(p.f_type)[r0 + i] = ty[i];
            const_cast<uint8_t*>(p.f_round)[r0 + i] = rd[i];
            const_cast<int16_t*>(p.f_pin)[r0 + i] = pn[i];
            const_cast<int16_t*>(p.f_exec)[r0 + i] = ex[i];
        }
        for (uint32_t i = tid; i <= nr; i += kK1Threads) const_cast<uint32_t*>(p.f_edge_off)[r0 + i] = eo[i];
        for (uint32_t i = tid; i < ne; i += kK1Threads) const_cast<uint32_t*>(p.edges)[e0 + i] = ed[i];
    }
    if (bprof && tid == 0) bprof[0] = gtimer();

    if (bprof && tid == 0) bprof[6] = gtimer();

    // ---- P2: depth + doom in creation order ------------------------------------
    // Short workflows: one warp sweeps all steps (32 rows each) in order.
    // Long workflows (>= kLongSteps steps): depth is linear in the (max,+)
    // semiring, so each step has a transfer function from its interface (the
    // <= 7 distinct predecessors outside the step) to its rows:
    //   d[f] = max(c_f, max_i D[x_i] + t_f(i)),
    // doom likewise over (or, and).  P2a computes every step's transfer in
    // parallel across warps (no step waits for another); P2b then composes the
    // steps in order on one warp with a cheap evaluation per step.  Steps that
    // do not fit (wide interface / fan-in) fall back to the ordinary sweep step
    // in P2b.
    auto is_long = [&](uint32_t wi) { return wfo[wi + 1] - wfo[wi] >= p.long_rows; };
    // long-step task prefix over the workflows in task order (s_perm: largest
    // first, so the early composers' transfers lead the tickets; warp 0),
    // s_lpref[nw] = total
    if (warp == 0) {
        uint32_t carry = 0, nlong = 0;
        for (uint32_t b0 = 0; b0 < nw; b0 += 32) {
            const uint32_t j = b0 + lane;
            const uint32_t wi = j < nw ? s_perm[j] : 0u;
            const uint32_t n = (j < nw && is_long(wi)) ? (wfo[wi + 1] - wfo[wi] + 31u) / 32u : 0u;
            nlong += __popc(__ballot_sync(0xFFFFFFFFu, n != 0u));
            uint32_t incl = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (j < nw) s_lpref[j] = carry + incl - n;
            carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        if (lane == 0) { s_lpref[nw] = carry; s_cnt[3] = nlong; }
    }
    __syncthreads();
    const uint32_t n_long_tasks = s_lpref[nw];
    // The largest long workflows (at most two) are composed from the start by
    // warps 0 / 1: the compose chain is the block's critical path, so it
    // follows the transfers step by step instead of starting behind them.
    const uint32_t n_early = min(s_cnt[3], 2u);

    uint32_t m_dep = 0, m_rnd = 0;
    long long cyc_edge = 0, cyc_round = 0, cyc_rest = 0, cyc_t = 0, cyc_wait = 0;
    uint32_t n_rounds = 0;
    unsigned long long n_kp = 0;   // profile: steps by widest in-step fan-in K (12-bit fields)
    auto wf_begin = [&](uint32_t wi) {
        m_dep = m_rnd = 0;
        cyc_edge = cyc_round = cyc_rest = cyc_wait = 0;
        cyc_t = prof ? clock64() : 0;
        n_rounds = 0;
        n_kp = 0;
        if (prof && lane == 0) prof[(size_t)(w0 + wi) * 2] = gtimer();
    };
    auto wf_end = [&](uint32_t wi) {
        const uint32_t w = w0 + wi;
        m_dep = __reduce_max_sync(0xFFFFFFFFu, m_dep);
        m_rnd = __reduce_max_sync(0xFFFFFFFFu, m_rnd);
        if (lane == 0) { s_wrnd[wi] = m_rnd; s_agg[wi * 8 + 7] = m_dep; }
        if (prof && lane == 0) {
            prof[(size_t)w * 2 + 1] = gtimer();
            cyc_rest += clock64() - cyc_t;
            unsigned long long* c = prof + (size_t)p.n_wf * 2 + (size_t)p.B * 8 + (size_t)p.R * 8 + (size_t)w * 4;
            c[0] = cyc_edge; c[1] = cyc_round; c[2] = cyc_rest;
            c[3] = cyc_wait ? (unsigned long long)cyc_wait << 32 : (n_rounds | n_kp);
        }
        __syncwarp();
    };
    // final depth / doom of a step's rows -> smem (the per-workflow counts are
    // taken row-parallel in P3; the maxima ride along here)
    auto finish_step = [&](uint32_t f, bool valid, uint32_t d, bool doom, bool allres, uint32_t rdf) {
        if (valid) {
            dep[f] = (uint16_t)d;
            flg[f] = (uint8_t)((allres ? FL_ALLRES : 0) | (doom ? FL_DOOMED : 0));
            m_dep = max(m_dep, d);
            m_rnd = max(m_rnd, rdf);
        }
        __syncwarp();
    };
    // the ordinary sweep step: predecessors before the step are final in smem;
    // those inside it settle by Bellman-Ford rounds
    auto regular_step = [&](uint32_t c0, bool valid, uint32_t stf, uint32_t eb, uint32_t ee, uint32_t pva,
                            uint32_t pvb, uint32_t& d_out, bool& doom_out, bool& allres_out) {
        // predecessors before this step are final in smem; those inside the
        // step are kept as up to 4 lane slots (+ a mask for any extra ones)
        uint32_t d = 0, need_dep = 0, extra = 0, np = 0;
        uint32_t s0 = lane, s1 = lane, s2 = lane, s3 = lane;
        bool dm = false, allres = true;
        // one predecessor edge, branch-free (lanes differ in edge kinds)
        auto take = [&](uint32_t v, uint32_t ds, uint32_t fs, uint32_t ss) {
            const uint32_t s = (v & 0x7FFFFFFFu) - r0;
            const bool dep_edge = (v >> 31) == 0u;
            const bool in = s >= c0;
            allres &= !dep_edge || ss == 3u;                 // CALL edges never gate (Q2)
            dm |= dep_edge && ss == 4u;
            const uint32_t k = (s - c0) & 31u;
            s0 = (in && np == 0) ? k : s0;
            s1 = (in && np == 1) ? k : s1;
            s2 = (in && np == 2) ? k : s2;
            s3 = (in && np == 3) ? k : s3;
            extra |= (in && np >= 4) ? (1u << k) : 0u;
            need_dep |= (in && dep_edge) ? (1u << k) : 0u;
            np += in ? 1u : 0u;
            d = in ? d : max(d, ds + 1u);
            dm |= !in && dep_edge && (fs & FL_DOOMED);
        };
        uint32_t e = eb;
        for (; e + 1 < ee; e += 2) {            // two edges per step: loads overlap
            const uint32_t va = e == eb ? pva : ed[e], vb = e == eb ? pvb : ed[e + 1];
            const uint32_t sa = (va & 0x7FFFFFFFu) - r0, sb = (vb & 0x7FFFFFFFu) - r0;
            // an in-step predecessor's depth / flags are not final (settled
            // below): not read here
            const uint32_t dsa = sa < c0 ? dep[sa] : 0u, dsb = sb < c0 ? dep[sb] : 0u;
            const uint32_t fsa = sa < c0 ? flg[sa] : 0u, fsb = sb < c0 ? flg[sb] : 0u;
            const uint32_t ssa = st[sa], ssb = st[sb];
            take(va, dsa, fsa, ssa);
            take(vb, dsb, fsb, ssb);
        }
        if (e < ee) {
            const uint32_t va = e == eb ? pva : ed[e];
            const uint32_t sa = (va & 0x7FFFFFFFu) - r0;
            take(va, sa < c0 ? dep[sa] : 0u, sa < c0 ? flg[sa] : 0u, st[sa]);
        }
        if (ee > eb) d = max(d, 1u);
        // unused in-step slots repeat slot 0 (a harmless duplicate)
        s1 = np > 1 ? s1 : s0;
        s2 = np > 2 ? s2 : s0;
        s3 = np > 3 ? s3 : s0;
        const bool pend = stf == 0u;
        bool doom = pend && dm;
        if (prof) { const long long t = clock64(); cyc_edge += t - cyc_t; cyc_t = t; }
        // in-step settling: Bellman-Ford rounds on registers, depths moving
        // by shuffles (four rounds per convergence vote); then doom, a
        // boolean closure over in-step DEP edges, by ballots
        if (__any_sync(0xFFFFFFFFu, np != 0u)) {
            const bool wide = __any_sync(0xFFFFFFFFu, extra != 0u);
            const bool has = np != 0u;
            // saturation is applied once after convergence: with D the
            // unsaturated depth, min(M, 1 + max min(M, D_p)) = min(M, D_f)
            if (!wide) {
                // the common case: at most 4 slots (unused ones repeat slot
                // 0).  One settle loop for every fan-in: K-specialised copies
                // spread the step loop over more code than the SMSP's L0
                // instruction cache holds
#ifndef NALAR_K_VARIANTS
                if (prof) n_kp += 1ull << (16 + 12 * 3);
                for (;;) {
                    uint32_t before = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k == 3) before = d;    // converged once a round changes nothing
                        uint32_t x0, x1, x2, x3;
                        asm volatile(
                            "shfl.sync.idx.b32 %0, %4, %5, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %1, %4, %6, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %2, %4, %7, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %3, %4, %8, 31, -1;"
                            : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                            : "r"(d), "r"(s0), "r"(s1), "r"(s2), "r"(s3));
                        d = has ? max(d, max(max(x0, x1), max(x2, x3)) + 1u) : d;
                    }
                    n_rounds += 4;
                    if (!__any_sync(0xFFFFFFFFu, d != before)) break;
                }
#else
                const uint32_t K = __reduce_max_sync(0xFFFFFFFFu, np);
                if (prof) n_kp += 1ull << (16 + 12 * ((K < 4 ? K : 4) - 1));
                auto settle = [&](auto round) {
                    for (;;) {
                        round();
                        round();
                        round();
                        const uint32_t before = d;
                        round();
                        n_rounds += 4;
                        if (!__any_sync(0xFFFFFFFFu, d != before)) break;
                    }
                };
                if (K <= 1) {
                    settle([&]() {
                        uint32_t x0;
                        asm volatile("shfl.sync.idx.b32 %0, %1, %2, 31, -1;" : "=r"(x0) : "r"(d), "r"(s0));
                        d = has ? max(d, x0 + 1u) : d;
                    });
                } else if (K == 2) {
                    settle([&]() {
                        uint32_t x0, x1;
                        asm volatile(
                            "shfl.sync.idx.b32 %0, %2, %3, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %1, %2, %4, 31, -1;"
                            : "=r"(x0), "=r"(x1) : "r"(d), "r"(s0), "r"(s1));
                        d = has ? max(d, max(x0, x1) + 1u) : d;
                    });
                } else if (K == 3) {
                    settle([&]() {
                        uint32_t x0, x1, x2;
                        asm volatile(
                            "shfl.sync.idx.b32 %0, %3, %4, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %1, %3, %5, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %2, %3, %6, 31, -1;"
                            : "=r"(x0), "=r"(x1), "=r"(x2) : "r"(d), "r"(s0), "r"(s1), "r"(s2));
                        d = has ? max(d, max(max(x0, x1), x2) + 1u) : d;
                    });
                } else {
                    settle([&]() {
                        uint32_t x0, x1, x2, x3;
                        asm volatile(
                            "shfl.sync.idx.b32 %0, %4, %5, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %1, %4, %6, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %2, %4, %7, 31, -1;\n\t"
                            "shfl.sync.idx.b32 %3, %4, %8, 31, -1;"
                            : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                            : "r"(d), "r"(s0), "r"(s1), "r"(s2), "r"(s3));
                        d = has ? max(d, max(max(x0, x1), max(x2, x3)) + 1u) : d;
                    });
                }
#endif
            } else {
                // a row with more than four in-step predecessors (a fan-in,
                // e.g. the aggregate of many subtasks) reads the extra ones
                // from shared memory: every round the lanes publish their
                // current depth in their own row's slot (clamped -- exact,
                // the final saturation absorbs it) and only the wide lanes
                // loop over their extra bits
                auto round = [&]() {
                    const uint32_t x0 = __shfl_sync(0xFFFFFFFFu, d, s0);
                    const uint32_t x1 = __shfl_sync(0xFFFFFFFFu, d, s1);
                    const uint32_t x2 = __shfl_sync(0xFFFFFFFFu, d, s2);
                    const uint32_t x3 = __shfl_sync(0xFFFFFFFFu, d, s3);
                    uint32_t nd = max(max(x0, x1), max(x2, x3)) + 1u;
                    if (valid) dep[c0 + lane] = (uint16_t)min(d, 65535u);
                    __syncwarp();
                    for (uint32_t e = extra; e; e &= e - 1u) nd = max(nd, (uint32_t)dep[c0 + __ffs(e) - 1u] + 1u);
                    __syncwarp();
                    d = has ? max(d, nd) : d;
                };
                for (;;) {
                    const uint32_t before = d;
                    round();
                    if (!__any_sync(0xFFFFFFFFu, d != before)) break;
                }
            }
        }
        doom = doom_closure(doom, pend, need_dep);
        d_out = min(d, 65535u);
        doom_out = doom;
        allres_out = allres;
        if (prof) { const long long t = clock64(); cyc_round += t - cyc_t; cyc_t = t; }
    };
    // a whole short workflow, step by step
    auto sweep_workflow = [&](uint32_t wi) {
        const uint32_t fa = wfo[wi] - r0, fb = wfo[wi + 1] - r0;
        wf_begin(wi);
        // the next step's row inputs and first two edge words are loaded one
        // step ahead, so their shared-memory latency hides behind this step
        uint32_t q_st = 3u, q_eb = 0u, q_ee = 0u, q_va = 0u, q_vb = 0u, q_rd = 0u;
        auto prefetch = [&](uint32_t c) {
            const uint32_t g = c + lane;
            const bool ok = g < fb;
            q_st = ok ? st[g] : 3u;
            q_eb = ok ? eo[g] - e0 : 0u;
            q_ee = ok ? eo[g + 1] - e0 : 0u;
            q_rd = ok ? rd[g] : 0u;
            q_va = q_eb < q_ee ? ed[q_eb] : 0u;
            q_vb = q_eb + 1 < q_ee ? ed[q_eb + 1] : 0u;
        };
        prefetch(fa);
        for (uint32_t c0 = fa; c0 < fb; c0 += 32) {
            if (prof) { const long long t = clock64(); cyc_rest += t - cyc_t; cyc_t = t; }
            const uint32_t f = c0 + lane;
            const bool valid = f < fb;
            const uint32_t stf = q_st, eb = q_eb, ee = q_ee, rdf = q_rd;
            const uint32_t pva = q_va, pvb = q_vb;
            if (c0 + 32 < fb) prefetch(c0 + 32);
            uint32_t d;
            bool doom, allres;
            regular_step(c0, valid, stf, eb, ee, pva, pvb, d, doom, allres);
            finish_step(f, valid, d, doom, allres, rdf);
        }
        wf_end(wi);
    };
    // P2a: the transfer function of one step of a long workflow
    // NALAR_F_PROFILE: per-block cycle sums of the transfer phases
    unsigned long long* tprof =
        prof ? prof + (size_t)p.n_wf * 2 + (size_t)p.B * 8 + (size_t)p.R * 8 + (size_t)p.n_wf * 4 + b * 8 : nullptr;
    long long tt = 0;
    auto tstamp = [&](int j) {
        if (tprof) {
            const long long t = clock64();
            if (lane == 0 && j > 0) atomicAdd(&tprof[j - 1], (unsigned long long)(t - tt));
            tt = t;
        }
    };
    auto transfer_step = [&](uint32_t c0, uint32_t fb) {
        tstamp(0);
        const uint32_t f = c0 + lane;
        const bool valid = f < fb;
        const uint32_t eb = valid ? eo[f] - e0 : 0u, ee = valid ? eo[f + 1] - e0 : 0u;
        uint32_t o0 = ~0u, o1 = ~0u, o2 = ~0u, o3 = ~0u, no = 0, odep = 0;     // out-of-step preds
        uint32_t s0 = lane, s1 = lane, s2 = lane, s3 = lane, np = 0, need_dep = 0;
        bool ovf = false, failp = false, allres = true;
        for (uint32_t e = eb; e < ee; ++e) {
            const uint32_t v = ed[e];
            const uint32_t s = (v & 0x7FFFFFFFu) - r0;
            const bool dep_edge = (v >> 31) == 0u;
            const uint32_t ss = st[s];
            allres &= !dep_edge || ss == 3u;
            failp |= dep_edge && ss == 4u;
            if (s >= c0) {
                const uint32_t k = s - c0;
                s0 = np == 0 ? k : s0;
                s1 = np == 1 ? k : s1;
                s2 = np == 2 ? k : s2;
                s3 = np == 3 ? k : s3;
                ovf |= np >= 4;
                ++np;
                need_dep |= dep_edge ? (1u << k) : 0u;
            } else {
                const int q = s == o0 ? 0 : s == o1 ? 1 : s == o2 ? 2 : s == o3 ? 3 : -1;
                if (q >= 0) {
                    odep |= dep_edge ? (1u << q) : 0u;
                } else {
                    o0 = no == 0 ? s : o0;
                    o1 = no == 1 ? s : o1;
                    o2 = no == 2 ? s : o2;
                    o3 = no == 3 ? s : o3;
                    ovf |= no >= 4;
                    odep |= (dep_edge && no < 4) ? (1u << no) : 0u;
                    ++no;
                }
            }
        }
        s1 = np > 1 ? s1 : s0;
        s2 = np > 2 ? s2 : s0;
        s3 = np > 3 ? s3 : s0;
        tstamp(1);
        // the step's interface: distinct out-of-step rows, ascending, <= 7
        uint32_t k = 0, myx = 0, i0 = 0, i1 = 0, i2 = 0, i3 = 0, taken = 0;
        for (;;) {
            uint32_t cand = ~0u;
            cand = (!(taken & 1u) && no > 0) ? min(cand, o0) : cand;
            cand = (!(taken & 2u) && no > 1) ? min(cand, o1) : cand;
            cand = (!(taken & 4u) && no > 2) ? min(cand, o2) : cand;
            cand = (!(taken & 8u) && no > 3) ? min(cand, o3) : cand;
            const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, cand);
            if (m == ~0u) break;
            if (k == kMaxIface) { ovf = true; break; }
            if (lane == k) myx = m;
            if (no > 0 && o0 == m) { i0 = k; taken |= 1u; }
            if (no > 1 && o1 == m) { i1 = k; taken |= 2u; }
            if (no > 2 && o2 == m) { i2 = k; taken |= 4u; }
            if (no > 3 && o3 == m) { i3 = k; taken |= 8u; }
            ++k;
        }
        const bool ok = !__any_sync(0xFFFFFFFFu, ovf);
        // transfer bytes: byte i < k = 1 + longest path from x_i into this row,
        // byte 7 = 1 + longest path from a root of the step (0 = none).
        // While settling, slot i lives in 16-bit half (i & 1) of h[i >> 1]
        // (slot 7 = the root path; with k <= 1 it rides in the free half of
        // h[0], with k <= 3 in that of h[1]) with a bias: a valid value b is
        // 0x8000 + b, "no path" is anything below 0x8000.  A settling round is
        // then a native u16x2 max tree plus a plain add of 1 per half (invalid
        // halves stay far below the bias); +1 is monotone, so it is applied
        // once after the max.
        const uint32_t K = __reduce_max_sync(0xFFFFFFFFu, np);
        const uint32_t NPw = k <= 1 ? 1u : (k <= 3 ? 2u : 4u);
        const uint32_t root_slot = k <= 1 ? 1u : (k <= 3 ? 3u : 7u);
        uint32_t h0 = 0, h1 = 0, h2 = 0, h3 = 0, edm = 0;
        auto seth = [&](uint32_t i, uint32_t v) {
            const uint32_t sl = i == 7u ? root_slot : i;
            const uint32_t x = (0x8000u + v) << (16 * (sl & 1u));
            h0 = (sl >> 1) == 0 ? (h0 | x) : h0;
            h1 = (sl >> 1) == 1 ? (h1 | x) : h1;
            h2 = (sl >> 1) == 2 ? (h2 | x) : h2;
            h3 = (sl >> 1) == 3 ? (h3 | x) : h3;
        };
        if (ok && valid) {
            if (no > 0) { seth(i0, 2u); edm |= (odep & 1u) ? (1u << i0) : 0u; }
            if (no > 1) { seth(i1, 2u); edm |= (odep & 2u) ? (1u << i1) : 0u; }
            if (no > 2) { seth(i2, 2u); edm |= (odep & 4u) ? (1u << i2) : 0u; }
            if (no > 3) { seth(i3, 2u); edm |= (odep & 8u) ? (1u << i3) : 0u; }
            if (ee == eb) seth(7u, 1u);              // a root: c = 0
        }
        tstamp(2);
        uint32_t nit = 0;
        // In-step doom ancestors of every pending row (the pending rows that
        // reach it over DEP edges through pending rows), so the composition
        // decides a step's doom with one vote instead of a closure walk
        // (measured: doom closures on the chain cost ~430 cycles a step).
        const bool pendf = valid && st[f] == 0u;
        const uint32_t pendm = __ballot_sync(0xFFFFFFFFu, pendf);
        uint32_t anc = pendf ? (need_dep & pendm) : 0u;
        const bool doomable = __any_sync(0xFFFFFFFFu, anc != 0u);
        if (!doomable) anc = 0u;
        if (ok && K != 0u) {
            const bool has = np != 0u;
            const uint32_t am = pendf ? (((need_dep >> s0) & 1u) | (((need_dep >> s1) & 1u) << 1) |
                                         (((need_dep >> s2) & 1u) << 2) | (((need_dep >> s3) & 1u) << 3))
                                      : 0u;
#ifndef NALAR_K_VARIANTS
            // one settle per (NP, doomable): unused slots repeat slot 0, so
            // K = 4 serves every fan-in (K-specialised copies cost more in
            // instruction fetch than their spared shuffles, measured)
#define NALAR_SETTLE2(NP_, A_) nit = settle_pairs<4, NP_, A_>(h0, h1, h2, h3, has, s0, s1, s2, s3, anc, am);
#else
#define NALAR_SETTLE2(NP_, A_)                                                                          \
            switch (K) {                                                                                \
                case 1: nit = settle_pairs<1, NP_, A_>(h0, h1, h2, h3, has, s0, s1, s2, s3, anc, am); break;   \
                case 2: nit = settle_pairs<2, NP_, A_>(h0, h1, h2, h3, has, s0, s1, s2, s3, anc, am); break;   \
                case 3: nit = settle_pairs<3, NP_, A_>(h0, h1, h2, h3, has, s0, s1, s2, s3, anc, am); break;   \
                default: nit = settle_pairs<4, NP_, A_>(h0, h1, h2, h3, has, s0, s1, s2, s3, anc, am); break;  \
            }
#endif
#define NALAR_SETTLE(NP_) if (doomable) { NALAR_SETTLE2(NP_, true) } else { NALAR_SETTLE2(NP_, false) }
            if (NPw == 1u) { NALAR_SETTLE(1) }
            else if (NPw == 2u) { NALAR_SETTLE(2) }
            else { NALAR_SETTLE(4) }
#undef NALAR_SETTLE
#undef NALAR_SETTLE2
        }
        tstamp(3);
        if (tprof && lane == 0) { atomicAdd(&tprof[5], 1ull); atomicAdd(&tprof[6], (unsigned long long)K); atomicAdd(&tprof[7], (unsigned long long)k); atomicAdd(&tprof[4], (unsigned long long)nit); }
        // move the root path to slot 7 (half 1 of h[3]) and unbias to bytes:
        // a valid half 0x8000 + b gives b (<= 34), else 0
        if (root_slot == 1u) {
            h3 = h0 & 0xFFFF0000u;
            h0 &= 0xFFFFu;
        } else if (root_slot == 3u) {
            h3 = h1 & 0xFFFF0000u;
            h1 &= 0xFFFFu;
        }
        auto unbias = [](uint32_t x) {
            const uint32_t lo = (x & 0x8000u) ? (x & 0xFFu) : 0u;
            const uint32_t hi = (x & 0x80000000u) ? ((x >> 16) & 0xFFu) : 0u;
            return lo | (hi << 8);
        };
        const uint32_t tlo_v = unbias(h0) | (unbias(h1) << 16);
        const uint32_t thi_v = unbias(h2) | (unbias(h3) << 16);
        const uint32_t av = edm | (failp ? 0x80u : 0u) | (allres ? 0x100u : 0u);

        if (valid) {
            tlo[f] = tlo_v;
            thi[f] = thi_v;
            ndp[f] = anc;
            if (lane != 0) aux[f] = (uint16_t)av;
        }
        if (lane < k && ok) ifc[c0 + lane] = myx;
        // publish: lane 0's aux word (k, ok) doubles as the step-done flag
        __syncwarp();
        if (lane == 0) st_release_u16(&aux[c0], (uint16_t)(av | (k << 9) | (ok ? 0x2000u : 0u) | kStepDone));
        tstamp(4);
    };
    // P2b: compose the steps of a long workflow in order: a step needs the
    // depths / doom flags of its <= 7 interface rows, all in earlier steps.
    // Everything a step reads that does not depend on the previous step (its
    // transfer words, interface rows, state, round) is loaded while the
    // previous step runs, so the chain per step is: the interface rows'
    // depths / flags from shared memory (written by the step before), the
    // (max,+) evaluation, the doom vote, the stores.
    auto compose_workflow = [&](uint32_t wi) {
        const uint32_t fa = wfo[wi] - r0, fb = wfo[wi + 1] - r0;
        wf_begin(wi);
        auto wait_flag = [&](uint32_t c0) {
            uint32_t v = ld_acquire_u16(&aux[c0]);
            if (!(v & kStepDone)) {
                const long long tw = prof ? clock64() : 0;
                do {
                    __nanosleep(20);
                    v = ld_acquire_u16(&aux[c0]);
                } while (!(v & kStepDone));
                if (prof) cyc_wait += clock64() - tw;
            }
            return v;
        };
        // inputs of the next step
        uint32_t a0, rdf, stf, tl = 0, th = 0, av = 0x100u, nd = 0;
        uint32_t xs[kMaxIface];
        auto load_step = [&](uint32_t c0) {
            const uint32_t f = c0 + lane;
            const bool valid = f < fb;
            rdf = valid ? rd[f] : 0u;
            stf = valid ? st[f] : 3u;
            if (a0 & 0x2000u) {
                tl = valid ? tlo[f] : 0u;
                th = valid ? thi[f] : 0u;
                av = valid ? aux[f] : 0x100u;
                nd = valid ? ndp[f] : 0u;
                const uint32_t k = (a0 >> 9) & 15u;
#pragma unroll
                for (uint32_t i = 0; i < kMaxIface; ++i) xs[i] = i < k ? ifc[c0 + i] : c0;
            }
        };
        a0 = wait_flag(fa);
        load_step(fa);
        for (uint32_t c0 = fa; c0 < fb; c0 += 32) {
            if (prof) { const long long t = clock64(); cyc_rest += t - cyc_t; cyc_t = t; }
            const uint32_t f = c0 + lane;
            const bool valid = f < fb;
            const uint32_t c_rdf = rdf, c_stf = stf;
            uint32_t d;
            bool doom, allres;
            if (a0 & 0x2000u) {
                const uint32_t k = (a0 >> 9) & 15u;
                const uint32_t c_tl = tl, c_th = th, c_av = av, c_nd = nd;
                uint32_t dx[kMaxIface], fx[kMaxIface];
#pragma unroll
                for (uint32_t i = 0; i < kMaxIface; ++i) { dx[i] = dep[xs[i]]; fx[i] = flg[xs[i]]; }
                // the next step's inputs, while these loads are in flight
                if (c0 + 32 < fb) {
                    a0 = wait_flag(c0 + 32);
                    load_step(c0 + 32);
                }
                // (max,+) evaluation as a tree (the terms are independent; a
                // slot >= k has byte 0): the step chain's longest ALU run
                uint32_t a[kMaxIface + 1];
                uint32_t dmk = 0;
#pragma unroll
                for (uint32_t i = 0; i < kMaxIface; ++i) {
                    const uint32_t by = i < 4 ? (c_tl >> (8 * i)) & 0xFFu : (c_th >> (8 * (i - 4))) & 0xFFu;
                    a[i] = by ? dx[i] + by - 1u : 0u;
                    dmk |= (fx[i] & FL_DOOMED) ? 1u << i : 0u;
                }
                const uint32_t c7 = c_th >> 24;
                a[kMaxIface] = c7 ? c7 - 1u : 0u;
                static_assert(kMaxIface == 7, "the tree below takes 8 terms");
                const uint32_t best = max(max(max(a[0], a[1]), max(a[2], a[3])), max(max(a[4], a[5]), max(a[6], a[7])));
                const bool dm = (c_av & 0x80u) != 0 || (dmk & c_av & ((1u << k) - 1u) & 0x7Fu) != 0;
                d = min(best, 65535u);
                allres = (c_av & 0x100u) != 0;
                if (prof) { const long long t = clock64() + (long long)d; cyc_edge += t - cyc_t; cyc_t = t; }
                {   // in-step closure from the transfer's ancestor masks
                    const bool seed = c_stf == 0u && dm;
                    const uint32_t D = __ballot_sync(0xFFFFFFFFu, seed);
                    doom = seed || (c_stf == 0u && (c_nd & D) != 0u);
                }
                if (prof) { const long long t = clock64(); cyc_round += t - cyc_t; cyc_t = t; }
            } else {
                const uint32_t eb = valid ? eo[f] - e0 : 0u, ee = valid ? eo[f + 1] - e0 : 0u;
                const uint32_t pva = eb < ee ? ed[eb] : 0u, pvb = eb + 1 < ee ? ed[eb + 1] : 0u;
                regular_step(c0, valid, c_stf, eb, ee, pva, pvb, d, doom, allres);
                if (c0 + 32 < fb) {
                    a0 = wait_flag(c0 + 32);
                    load_step(c0 + 32);
                }
            }
            finish_step(f, valid, d, doom, allres, c_rdf);
        }
        wf_end(wi);
    };

    // Tasks by ticket (after the early composes above): every step transfer of
    // the block's long workflows (P2a; the two early composers' steps
    // alternating, then the other long workflows largest first), then the
    // remaining workflows largest first -- a long one is composed, a short
    // one swept.  A composing warp
    // follows its transfers step by step, waiting on the producer's release
    // flag.  Deadlock-free: a compose only ever waits on transfers, and every
    // transfer is claimed by one of the >= 14 warps not composing early, none
    // of which waits before finishing it.
    if (warp < n_early) compose_workflow(s_perm[warp]);
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(s_ticket, 1u);
        t = __shfl_sync(0xFFFFFFFFu, t, 0);
        if (t < n_long_tasks) {
            // the two early composers' steps alternate (each composer gets its
            // next step every other ticket), then the rest in task order
            const uint32_t nA = s_lpref[1], nB = nw > 1 ? s_lpref[2] - s_lpref[1] : 0u;
            const uint32_t m = min(nA, nB);
            uint32_t wi, k;
            if (t < 2u * m) {
                wi = s_perm[t & 1u];
                k = t >> 1;
            } else if (t < nA + nB) {
                wi = s_perm[nA > nB ? 0 : 1];
                k = m + (t - 2u * m);
            } else {
                uint32_t lo = 2, hi = nw - 1;        // last position with s_lpref <= t
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (s_lpref[mid] <= t) lo = mid;
                    else hi = mid - 1;
                }
                wi = s_perm[lo];
                k = t - s_lpref[lo];
            }
            transfer_step(wfo[wi] - r0 + 32u * k, wfo[wi + 1] - r0);
            continue;
        }
        if (t - n_long_tasks + n_early >= nw) break;
        const uint32_t wi = s_perm[t - n_long_tasks + n_early];
        if (is_long(wi)) compose_workflow(wi);
        else sweep_workflow(wi);
    }
    __syncthreads();
    if (bprof && tid == 0) bprof[1] = gtimer();

    // the exchange buffer / counters this kernel accumulates into are cleared by
    // the zero kernel this one depends on programmatically (PDL): everything
    // above only staged inputs and wrote shared memory and plain outputs
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.trig == 1) asm volatile("griddepcontrol.launch_dependents;");
    if (p.rb_mine && b == 0 && tid == 0) {        // world > 1: this rank's place in the row order
        p.rb_mine[0] = p.row_base;
        p.rb_mine[1] = p.n_rows;
    }
    if (bprof && tid == 0) bprof[7] = gtimer();

    // ---- P3 (row-parallel): level, status, outputs, histogram, minima --------
    const uint32_t pol = p.policy;
    const int64_t lmax = (int64_t)Lv - 1;
    for (uint32_t f0 = 0; f0 < nr; f0 += kK1Threads) {
        const uint32_t f = f0 + tid;
        const bool valid = f < nr;
        uint32_t kp = 0xFFFFFFFFu, kr = 0xFFFFFFFFu, wl = 0xFFFFFFFFu, tyf = 0;
        bool pend = false, ready = false, doom = false, infl_row = false, pinp = false;
        uint32_t stf = 3u;
        if (valid) {
            {   // workflow of row f (binary search over the staged offsets)
                uint32_t lo = 0, hi = nw - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (wfo[mid] - r0 <= f) lo = mid;
                    else hi = mid - 1;
                }
                wl = lo;
            }
            stf = st[f];
            const uint32_t fl = flg[f], d = dep[f];
            tyf = ty[f];
            infl_row = stf == 1u || stf == 2u;
            if (infl_row) {                     // in-flight: instance load, (w, t) fence
                atomicAdd(&s_load[ex[f]], 1u);
                atomicOr(&s_winfl[2 * wl + (tyf >> 5)], 1u << (tyf & 31u));   // native 32-bit ATOMS.OR
            }
            const int pinf = pn[f];
            pend = stf == 0u;
            doom = fl & FL_DOOMED;
            ready = pend && !doom && (fl & FL_ALLRES);      // PAPER.md:463, Q2
            pinp = pend && pinf >= 0;
            const uint32_t aff = s_aff[tyf];
            // eligibility known now unless decided per (workflow, type) in P4
            const bool elig = ready && (aff == 0u || (aff == 1u && pinf >= 0));
            uint32_t lv = 0;
            if (stf < 3u) {
                const int64_t score = pol == 1u ? (int64_t)d : (pol == 2u ? (int64_t)s_wrnd[wl] : 0);
                const int64_t x = (int64_t)wpr[wl] + score;
                lv = (uint32_t)(x < 0 ? 0 : (x > lmax ? lmax : x));
            }
            uint32_t status;
            int16_t inst = -1;
            if (stf == 3u) status = 0;
            else if (stf == 4u) status = 1;
            else if (infl_row) { status = 2; inst = ex[f]; }
            else if (doom) status = 4;
            else if (!ready) status = 3;
            else status = elig ? 6u : 5u;
            // HoL-migration candidates (NEXT-1): a QUEUED
            // future waiting past theta_wait at an instance whose head job runs
            // past theta_head; STATEFUL never moves; a SESSION future only as
            // its session's sole queued work with nothing running (decided in P4)
            bool mig = false;
            if (kNext && p.mig_on) {
                if (stf == 1u && aff != 2u) {
                    const bool c = p.f_age[r0 + f] > p.theta_wait && p.i_head_rem[ex[f]] > p.theta_head;
                    if (aff == 0u) {
                        mig = c;
                    } else {
                        atomicAdd(&s_mq[wl * T + tyf], 1u);
                        atomicMax(&s_mqrow[wl * T + tyf], f | (c ? 0x80000000u : 0u));
                    }
                }
                if (stf == 2u && aff == 1u) atomicOr(&s_mrun[2 * wl + (tyf >> 5)], 1u << (tyf & 31u));
                p.migrate_to[r0 + f] = -1;
            }
            if (kNext && p.batch_head) p.batch_head[r0 + f] = -1;
            if (kNext && p.mig_on) {
                if (mig) {
                    atomicAdd(&p.H[(size_t)(R + tyf) * Lv + lv], 1u);
                    atomicAdd(&s_rcnt[R + tyf], 1u);
                }
            }
            const uint32_t g = r0 + f;
            lev[f] = (uint8_t)lv;
            flg[f] = (uint8_t)(fl | (ready ? FL_READY : 0) | (elig ? FL_ELIG : 0) | (mig ? FL_MIG : 0));
            p.status[g] = (uint8_t)status;
            if (staged) { p.level[g] = (uint8_t)lv; p.depth[g] = (uint16_t)d; }
            p.instance[g] = inst;
            p.new_pin[g] = 0;
            // streamed outputs: straight to the caller's pinned arrays (the
            // PCIe writes overlap the rest of the epoch; K4 patches the
            // admitted rows, P4 the fence winners)
            if (kOut) {
                if (p.o_status) p.o_status[g] = (uint8_t)status;
                if (p.o_level) p.o_level[g] = (uint8_t)lv;
                if (p.o_depth) p.o_depth[g] = (uint16_t)d;
                if (p.o_instance) p.o_instance[g] = inst;
                if (p.o_new_pin) p.o_new_pin[g] = 0;
            }
            if (elig) {
                const uint32_t r = pinf >= 0 ? (uint32_t)pinf : I + tyf;
                atomicAdd(&p.H[(size_t)r * Lv + lv], 1u);
                atomicAdd(&s_rcnt[r], 1u);
            }
            if (pend && !doom) kp = wl << 6 | tyf;
            if (ready && pinf < 0) kr = wl << 6 | tyf;
            if (aff == 1u) {                // K,V retention hints (NEXT-3): home, urgency
                if (pinf >= 0) atomicMin(&s_khome[wl * T + tyf], (uint32_t)pinf);
                if (infl_row || (pend && !doom)) atomicMax(&s_klev[wl * T + tyf], lv + 1u);
            }
        }
        // per-workflow counts ("aggregating metrics and metadata"):
        // rows are in workflow order, so a warp's lanes form contiguous
        // workflow segments; the segment head adds its segment's popcounts
        {
            const uint32_t wup = __shfl_up_sync(0xFFFFFFFFu, wl, 1);
            const bool head = valid && (lane == 0 || wup != wl);
            const uint32_t hm = __ballot_sync(0xFFFFFFFFu, head | !valid);
            const uint32_t above = lane == 31 ? 0u : hm & (0xFFFFFFFEu << lane);
            const uint32_t seg = (above ? (above & (0u - above)) - 1u : 0xFFFFFFFFu) & (0xFFFFFFFFu << lane);
            const uint32_t b_pend = __ballot_sync(0xFFFFFFFFu, pend);
            const uint32_t b_ready = __ballot_sync(0xFFFFFFFFu, ready);
            const uint32_t b_infl = __ballot_sync(0xFFFFFFFFu, infl_row);
            const uint32_t b_res = __ballot_sync(0xFFFFFFFFu, stf == 3u && valid);
            const uint32_t b_fail = __ballot_sync(0xFFFFFFFFu, stf == 4u);
            const uint32_t b_doom = __ballot_sync(0xFFFFFFFFu, doom);
            const uint32_t b_pinp = __ballot_sync(0xFFFFFFFFu, pinp);
            if (head) {
                uint32_t* a = s_agg + (size_t)wl * 8;
                const uint32_t v0 = __popc(b_pend & seg), v1 = __popc(b_ready & seg), v2 = __popc(b_infl & seg);
                const uint32_t v3 = __popc(b_res & seg), v4 = __popc(b_fail & seg), v5 = __popc(b_doom & seg);
                const uint32_t v6 = __popc(b_pinp & seg);
                if (v0) atomicAdd(a + 0, v0);
                if (v1) atomicAdd(a + 1, v1);
                if (v2) atomicAdd(a + 2, v2);
                if (v3) atomicAdd(a + 3, v3);
                if (v4) atomicAdd(a + 4, v4);
                if (v5) atomicAdd(a + 5, v5);
                if (v6) atomicAdd(a + 6, v6);
            }
            if (lane == 0) {
                if (b_ready) atomicAdd(&s_cnt[0], __popc(b_ready));
                if (b_doom) atomicAdd(&s_cnt[2], __popc(b_doom));
            }
        }
        // first PENDING non-doomed / first ready unpinned row of each (w, t)
        // (a minimum: order-independent, so plain shared-memory atomics)
        if (kp != 0xFFFFFFFFu) atomicMin(&s_wfp[wl * T + tyf], f);
        if (kr != 0xFFFFFFFFu) atomicMin(&s_wfru[wl * T + tyf], f);
    }
    __syncthreads();
    if (bprof && tid == 0) bprof[4] = gtimer();

    // ---- P4: the stateful fence and first placement
    // make the per-(workflow, type) winner eligible; the per-workflow and
    // per-(workflow, type) outputs ride in the same pass over (w, t)
    // (T == 0 only for a table without futures: one pseudo-type per workflow)
    const uint32_t Tp = T ? T : 1u;
    for (uint32_t k = tid; k < nw * Tp; k += kK1Threads) {
        const uint32_t wl = k / Tp, t = k - wl * Tp;
        const uint32_t aff = s_aff[t];
        const uint32_t* a = s_agg + (size_t)wl * 8;
        if (t == 0) {
            // per-workflow aggregates: total, pending, ready, inflight, resolved,
            // failed, doomed, pinned_pending, max_depth, max_round
            uint32_t* o = p.wf_agg + (size_t)(w0 + wl) * 10;
            o[0] = wfo[wl + 1] - wfo[wl];
#pragma unroll
            for (int j = 0; j < 8; ++j) o[1 + j] = a[j];
            o[9] = s_wrnd[wl];
        }
        if (T == 0) continue;
        {
            // K,V-cache retention hints per (workflow, SESSION type) (PAPER.md:524-529,
            // SPEC kv_hint S:542; DESIGN.md Q-kv): retain while the session has a
            // live future, offload when only its workflow does, drop when neither
            const bool sess = aff == 1u;
            const uint32_t home = s_khome[k], kl = s_klev[k];
            const uint32_t wf_live = a[0] - a[5] + a[2];      // pending - doomed + in flight
            const bool has = sess && home != 0xFFFFFFFFu;
            p.kv_hint[(size_t)w0 * T + k] = (uint8_t)(has ? (kl ? 1u : (wf_live ? 2u : 3u)) : 0u);
            p.kv_level[(size_t)w0 * T + k] = (uint8_t)(sess && kl ? kl - 1u : 0u);
            p.kv_home[(size_t)w0 * T + k] = (int16_t)(has ? (int)home : -1);
        }
        uint32_t f = 0xFFFFFFFFu;
        if (aff == 2u) {
            const uint32_t c = s_wfp[k];
            if (c != 0xFFFFFFFFu && !((s_winfl[2 * wl + (t >> 5)] >> (t & 31u)) & 1u) && (flg[c] & FL_READY)) f = c;
        } else if (aff == 1u) {
            f = s_wfru[k];
        }
        if (kNext && p.mig_on && aff == 1u && s_mq[k] == 1u && !((s_mrun[2 * wl + (t >> 5)] >> (t & 31u)) & 1u) &&
            (s_mqrow[k] & 0x80000000u)) {
            const uint32_t fm = s_mqrow[k] & 0x7FFFFFFFu;   // the session's sole queued future moves
            flg[fm] |= FL_MIG;
            atomicAdd(&p.H[(size_t)(R + t) * Lv + lev[fm]], 1u);
            atomicAdd(&s_rcnt[R + t], 1u);
        }
        if (f != 0xFFFFFFFFu) {
            flg[f] |= FL_ELIG;
            p.status[r0 + f] = 6;
            if (kOut && p.o_status) p.o_status[r0 + f] = 6;
            const int pinf = pn[f];
            const uint32_t r = pinf >= 0 ? (uint32_t)pinf : I + t;
            atomicAdd(&p.H[(size_t)r * Lv + lev[f]], 1u);
            atomicAdd(&s_rcnt[r], 1u);
        }
    }
    __syncthreads();
    if (bprof && tid == 0) bprof[5] = gtimer();

    if (p.trig == 2) asm volatile("griddepcontrol.launch_dependents;");
    // ---- P5 (epilogue): loads, per-resource offsets, stable bucketing ---------
    for (uint32_t i = tid; i < I; i += kK1Threads)
        if (s_load[i]) atomicAdd(&p.load_part[i], s_load[i]);
    // exclusive scan of s_rcnt over R (serial per thread chunk + warp scan)
    {
        const uint32_t per = (Rh + kK1Threads - 1) / kK1Threads;
        const uint32_t lo = min(Rh, tid * per), hi = min(Rh, lo + per);
        uint32_t sum = 0;
        for (uint32_t r = lo; r < hi; ++r) sum += s_rcnt[r];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) s_wc[warp] = incl;
        __syncthreads();
        // the warps before this one, one lane each, summed by one reduction
        const uint32_t wbase = __reduce_add_sync(0xFFFFFFFFu, lane < warp ? s_wc[lane] : 0u);
        uint32_t run = wbase + incl - sum;
        for (uint32_t r = lo; r < hi; ++r) {
            const uint32_t c = s_rcnt[r];
            s_roff[r] = run;
            p.cnt_rb[(size_t)r * p.B + b] = c;
            p.off_rb[(size_t)r * p.B + b] = run;
            if (c) { atomicAdd(&p.tot[r], c); atomicAdd(&p.tot_loc[r], c); }
            run += c;
            s_rcnt[r] = 0;   // reused as the running rank counter below
        }
        __syncthreads();
    }
    // Every 512-row chunk at once when the block has <= kP5Chunks of them and
    // <= 512 eligible rows (one compaction, two barriers; chunk by chunk it
    // took three barriers per chunk): per-(chunk, warp) counts, their
    // exclusive prefix in (chunk, warp) = row order, the row-ordered list,
    // then warp 0 buckets it by resource as below.
    // (one-wave tables only: several waves are throughput-bound, where the
    // extra reductions cost -- C5 +2.5 us)
    const uint32_t nch = (nr + kK1Threads - 1) / kK1Threads;
    bool p5_done = false;
    if (p.B <= 148u && nch <= (uint32_t)kP5Chunks) {
        uint32_t balc[kP5Chunks];
        uint32_t ecnt = 0;
#pragma unroll
        for (int c = 0; c < kP5Chunks; ++c) {
            balc[c] = 0u;
            if ((uint32_t)c < nch) {
                const uint32_t f = (uint32_t)c * kK1Threads + tid;
                const uint32_t fl = f < nr ? flg[f] : 0u;
                ecnt += __popc(__ballot_sync(0xFFFFFFFFu, (fl & FL_ELIG) != 0u));
                balc[c] = __ballot_sync(0xFFFFFFFFu, (fl & (FL_ELIG | FL_MIG)) != 0u);
                if (lane == 0) s_wcc[c * kK1Warps + warp] = __popc(balc[c]);
            }
        }
        if (lane == 0 && ecnt) atomicAdd(&s_cnt[1], ecnt);
        __syncthreads();
        // the (chunk, warp) counts, four per lane, in row order
        const uint32_t ncw = nch * kK1Warps;
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = lane * 4u + q < ncw ? s_wcc[lane * 4u + q] : 0u;
        const uint32_t tot = __reduce_add_sync(0xFFFFFFFFu, v[0] + v[1] + v[2] + v[3]);
        if (tot <= (uint32_t)kK1Threads) {
#pragma unroll
            for (int c = 0; c < kP5Chunks; ++c) {
                if ((uint32_t)c >= nch) break;
                const uint32_t e = (uint32_t)c * kK1Warps + warp;      // this warp's entry
                // exclusive prefix of entry e: whole lanes before e / 4, then part of lane e / 4
                uint32_t part = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) part += lane * 4u + q < e ? v[q] : 0u;
                const uint32_t base = __reduce_add_sync(0xFFFFFFFFu, part);
                const uint32_t f = (uint32_t)c * kK1Threads + tid;
                if ((balc[c] >> lane) & 1u) s_list[base + __popc(balc[c] & ((1u << lane) - 1u))] = f;
            }
            __syncthreads();
            if (warp == 0) {
                for (uint32_t j0 = 0; j0 < tot; j0 += 32) {
                    const uint32_t j = j0 + lane;
                    const bool ok = j < tot;
                    uint32_t r = 0xFFFFFFFFu, ff = 0;
                    bool mg = false;
                    if (ok) {
                        ff = s_list[j];
                        mg = !(flg[ff] & FL_ELIG);                  // a HoL candidate (NEXT-1)
                        const int pinf = pn[ff];
                        r = mg ? R + ty[ff] : (pinf >= 0 ? (uint32_t)pinf : I + ty[ff]);
                    }
                    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, r);
                    const uint32_t rank = ok ? s_rcnt[r] + __popc(peers & ((1u << lane) - 1u)) : 0u;
                    __syncwarp();
                    if (ok) {
                        p.items[r0 + s_roff[r] + rank] =
                            make_uint2(r0 + ff, lev[ff] | (mg ? (uint32_t)(ex[ff] + 1) << 16 : 0u));
                        if ((__ffs(peers) - 1) == (int)lane) s_rcnt[r] += __popc(peers);
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            p5_done = true;
        }
    }
    for (uint32_t t0 = 0; !p5_done && t0 < nr; t0 += kK1Threads) {
        const uint32_t f = t0 + tid;
        const bool el = f < nr && (flg[f] & (FL_ELIG | FL_MIG));
        if (p.B > 148u || nch > (uint32_t)kP5Chunks) {   // (counted above otherwise)
            const uint32_t be = __ballot_sync(0xFFFFFFFFu, f < nr && (flg[f] & FL_ELIG));
            if (lane == 0 && be) atomicAdd(&s_cnt[1], __popc(be));
        }
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, el);
        if (lane == 0) s_wc[warp] = __popc(bal);
        __syncthreads();
        uint32_t base = 0, tot = 0;
        for (uint32_t k = 0; k < (uint32_t)kK1Warps; ++k) {
            const uint32_t c = s_wc[k];
            base += k < warp ? c : 0u;
            tot += c;
        }
        if (el) s_list[base + __popc(bal & ((1u << lane) - 1u))] = f;
        __syncthreads();
        if (warp == 0) {
            for (uint32_t j0 = 0; j0 < tot; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool ok = j < tot;
                uint32_t r = 0xFFFFFFFFu, ff = 0;
                bool mg = false;
                if (ok) {
                    ff = s_list[j];
                    mg = !(flg[ff] & FL_ELIG);                  // a HoL candidate (NEXT-1)
                    const int pinf = pn[ff];
                    r = mg ? R + ty[ff] : (pinf >= 0 ? (uint32_t)pinf : I + ty[ff]);
                }
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, r);
                const uint32_t rank = ok ? s_rcnt[r] + __popc(peers & ((1u << lane) - 1u)) : 0u;
                __syncwarp();
                if (ok) {
                    p.items[r0 + s_roff[r] + rank] =
                        make_uint2(r0 + ff, lev[ff] | (mg ? (uint32_t)(ex[ff] + 1) << 16 : 0u));
                    if ((__ffs(peers) - 1) == (int)lane) s_rcnt[r] += __popc(peers);
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
    if (bprof && tid == 0) bprof[2] = gtimer();
    if (tid == 0) {
        atomicAdd(&p.counters[C_READY], s_cnt[0]);
        atomicAdd(&p.counters[C_ELIG], s_cnt[1]);
        atomicAdd(&p.counters[C_DOOMED], s_cnt[2]);
    }
}

}  // namespace nalar
