/* nalar_oracle.c -- TEST INFRASTRUCTURE ONLY (see nalar_oracle.h).
 *
 * Plain, slow, single-threaded CPU oracle of the Nalar global controller's
 * policy epoch (arXiv 2601.05109).  Written step by step in the order of the
 * epoch definition (plus O9 for the NEXT-3 K,V
 * retention hints; readings Q1-Q22 and Q-kv listed in
 * DESIGN.md "Readings of the paper").  No blocking, fusion or reordering; the
 * only library routine used is qsort (O6/O7 sort by the total order of O4).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets).
 *
 * Pins (tests/test_oracle_pins.py), each reaching the answer another way:
 * brute-force path enumeration (depth), forward reachability (doom), closed
 * forms (chains, fan-out/fan-in, the hand-derived C1 golden file
 * tests/golden/c1_srtf.txt), brute-force subset enumeration of feasible
 * admissions (lexicographically greatest admitted set), the closed-form slot
 * list for phase B, SPEC worked examples, and invariants I1-I10.
 */
#define _POSIX_C_SOURCE 199309L   /* clock_gettime (the timing harness only) */
#include "nalar_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { S_PENDING = 0, S_QUEUED = 1, S_RUNNING = 2, S_RESOLVED = 3, S_FAILED = 4 };
enum { A_NONE = 0, A_SESSION = 1, A_STATEFUL = 2 };
enum { O_RESOLVED = 0, O_FAILED = 1, O_INFLIGHT = 2, O_WAITING = 3, O_DOOMED = 4,
       O_INELIGIBLE = 5, O_DEFERRED = 6, O_ASSIGNED = 7 };
#define CALL_BIT 0x80000000u

/* ------------------------------------------------------------------------ */
/* Validation: the input contract of the "live future table" (Q1).           */
/* Every dependency is write-once and must exist when its consumer is created */
/* (SPEC S:50-52), so every edge points to an EARLIER row of the SAME workflow */
/* (creation order is a topological order).                                   */
/* ------------------------------------------------------------------------ */
int oracle_validate(const oracle_table* t, int64_t* err_row) {
    int64_t bad = -1;
    uint32_t N = t->n_futures, W = t->n_workflows, I = t->n_instances, T = t->n_types;
    if (err_row) *err_row = -1;
    if (t->levels < 1 || t->levels > 256) return -1;
    if (t->wf_fut_off[0] != 0 || t->wf_fut_off[W] != N) return -1;
    for (uint32_t w = 0; w < W; ++w) {
        if (t->wf_fut_off[w + 1] < t->wf_fut_off[w]) return -1;
        if (w > 0 && t->wf_id[w] <= t->wf_id[w - 1]) return -1;
    }
    if (t->f_edge_off[0] != 0 || t->f_edge_off[N] != t->n_edges) return -1;
    for (uint32_t f = 0; f < N; ++f)
        if (t->f_edge_off[f + 1] < t->f_edge_off[f]) return -1;
    for (uint32_t i = 0; i < I; ++i)
        if (t->i_type[i] >= T) return -1;
    for (uint32_t k = 0; k < T; ++k)
        if (t->t_affinity[k] > A_STATEFUL) return -1;
    for (uint32_t w = 0; w < W && bad < 0; ++w) {
        for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) {
            int ok = 1;
            uint8_t st = t->f_state[f], ty = t->f_type[f];
            int pin = t->f_pin[f], ex = t->f_executor[f];
            if (st > S_FAILED) ok = 0;
            if (ty >= T) ok = 0;
            if (ok && pin != -1 && (pin < 0 || (uint32_t)pin >= I || t->i_type[pin] != ty)) ok = 0;
            if (ok && (st == S_QUEUED || st == S_RUNNING) &&
                (ex < 0 || (uint32_t)ex >= I || t->i_type[ex] != ty)) ok = 0;
            for (uint32_t e = t->f_edge_off[f]; ok && e < t->f_edge_off[f + 1]; ++e) {
                uint32_t s = t->edges[e] & ~CALL_BIT;
                if (s < t->wf_fut_off[w] || s >= f) ok = 0;
            }
            if (!ok) { bad = f; break; }
        }
    }
    if (bad >= 0) { if (err_row) *err_row = bad; return -1; }
    return 0;
}

/* total order of O4: f before g iff level[f] > level[g], or equal levels and
 * f < g (tie-break by future id / row = (workflow_id, seq), Q8). */
static const uint8_t* g_level;
static int cmp_order(const void* a, const void* b) {
    uint32_t f = *(const uint32_t*)a, g = *(const uint32_t*)b;
    if (g_level[f] != g_level[g]) return g_level[f] > g_level[g] ? -1 : 1;
    return f < g ? -1 : (f > g ? 1 : 0);
}

int oracle_epoch(const oracle_table* t, int policy, oracle_out* o) {
    uint32_t N = t->n_futures, W = t->n_workflows, I = t->n_instances, T = t->n_types;
    int64_t dummy;
    if (oracle_validate(t, &dummy) != 0) return -1;

    uint8_t* doomed = (uint8_t*)calloc(N ? N : 1, 1);
    uint8_t* ready = (uint8_t*)calloc(N ? N : 1, 1);
    uint8_t* eligible = (uint8_t*)calloc(N ? N : 1, 1);
    uint32_t* wf_of = (uint32_t*)calloc(N ? N : 1, sizeof(uint32_t));
    for (uint32_t w = 0; w < W; ++w)
        for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) wf_of[f] = w;

    /* O1 topological sweep in row order (rows are topologically ordered, Q1).
     * depth: longest path from a root over DEP u CALL edges; SRTF "later
     *   stages of the graph" P:691 [§6.2], SPEC S:460 creation-chain depth (Q4);
     *   u16 saturating (Q22).
     * doomed: PENDING with a DEP predecessor FAILED or doomed, transitively
     *   (failures are delivered like values; P:580-581 [§5]) (Q3).
     * ready: PENDING, not doomed, every DEP predecessor RESOLVED -- push-based
     *   readiness P:462-465 [§4.3.1], SPEC S:268-276 (Q2; CALL edges do not gate). */
    for (uint32_t f = 0; f < N; ++f) {
        uint32_t e0 = t->f_edge_off[f], e1 = t->f_edge_off[f + 1];
        uint32_t d = 0;
        int dm = 0, allres = 1;
        for (uint32_t e = e0; e < e1; ++e) {
            uint32_t s = t->edges[e] & ~CALL_BIT;
            int is_call = (t->edges[e] & CALL_BIT) != 0;
            uint32_t cand = (uint32_t)o->depth[s] + 1u;
            if (cand > d) d = cand;
            if (!is_call) {
                if (t->f_state[s] == S_FAILED || doomed[s]) dm = 1;
                if (t->f_state[s] != S_RESOLVED) allres = 0;
            }
        }
        o->depth[f] = (uint16_t)(d > 65535u ? 65535u : d);
        doomed[f] = (uint8_t)(t->f_state[f] == S_PENDING && dm);
        ready[f] = (uint8_t)(t->f_state[f] == S_PENDING && !doomed[f] && allres);
    }

    /* O2 per-workflow aggregates ("aggregating metrics and metadata", P:338
     * [§4.1]; per-session summaries SPEC S:365) and per-(w,t) facts used by
     * eligibility. */
    uint8_t* inflight_wt = (uint8_t*)calloc((size_t)(W ? W : 1) * (T ? T : 1), 1);
    int64_t* first_pending = (int64_t*)malloc(sizeof(int64_t) * (size_t)(W ? W : 1) * (T ? T : 1));
    int64_t* first_ready_unp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(W ? W : 1) * (T ? T : 1));
    for (size_t k = 0; k < (size_t)W * T; ++k) { first_pending[k] = -1; first_ready_unp[k] = -1; }
    for (uint32_t w = 0; w < W; ++w) {
        uint32_t* a = o->wf_agg + (size_t)w * 10;
        memset(a, 0, 10 * sizeof(uint32_t));
        for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) {
            uint8_t st = t->f_state[f];
            size_t wt = (size_t)w * T + t->f_type[f];
            a[0] += 1;                                             /* total          */
            if (st == S_PENDING) a[1] += 1;                        /* pending        */
            if (ready[f]) a[2] += 1;                               /* ready          */
            if (st == S_QUEUED || st == S_RUNNING) a[3] += 1;      /* in flight      */
            if (st == S_RESOLVED) a[4] += 1;                       /* resolved       */
            if (st == S_FAILED) a[5] += 1;                         /* failed         */
            if (doomed[f]) a[6] += 1;                              /* doomed         */
            if (st == S_PENDING && t->f_pin[f] != -1) a[7] += 1;   /* pinned pending */
            if (o->depth[f] > a[8]) a[8] = o->depth[f];            /* max depth      */
            if (t->f_round[f] > a[9]) a[9] = t->f_round[f];        /* max round      */
            if (st == S_QUEUED || st == S_RUNNING) inflight_wt[wt] = 1;
            if (st == S_PENDING && !doomed[f] && first_pending[wt] < 0) first_pending[wt] = f;
            if (ready[f] && t->f_pin[f] == -1 && first_ready_unp[wt] < 0) first_ready_unp[wt] = f;
        }
    }

    /* O3 eligibility of ready futures.
     * stateful: "a single user request and a single session are scheduled in
     *   order and routed to the same agent instance" P:267-268 [§3.4]; scope
     *   (workflow, type), fence SPEC S:222 (Q12).
     * managed state (SESSION): all requests of a session go to the same
     *   instance P:575 [§5]; an unpinned session places only its first ready
     *   future, the assignment creates the pin (Q13). */
    uint32_t n_ready = 0, n_elig = 0, n_doomed = 0;
    for (uint32_t f = 0; f < N; ++f) {
        if (doomed[f]) n_doomed++;
        if (!ready[f]) continue;
        n_ready++;
        size_t wt = (size_t)wf_of[f] * T + t->f_type[f];
        uint8_t aff = t->t_affinity[t->f_type[f]];
        int el;
        if (aff == A_STATEFUL) el = !inflight_wt[wt] && first_pending[wt] == (int64_t)f;
        else if (aff == A_SESSION && t->f_pin[f] == -1) el = first_ready_unp[wt] == (int64_t)f;
        else el = 1;
        eligible[f] = (uint8_t)el;
        n_elig += (uint32_t)el;
    }

    /* O4 priority level of every non-terminal future (Q15):
     *   level = clamp(prio[w] + score, 0, Lv-1) in 64-bit (Q7);
     *   set_priority(session, value) P:389 [§4.2 tab:scheduling-API];
     *   score: FCFS 0; SRTF depth (P:691 [§6.2]); LPT max round of the
     *   workflow ("jobs that re-enter the graph", P:696 [§6.2]) (Q6). */
    for (uint32_t f = 0; f < N; ++f) {
        uint8_t st = t->f_state[f];
        if (st == S_RESOLVED || st == S_FAILED) { o->level[f] = 0; continue; }
        int64_t score = 0;
        if (policy == 1) score = o->depth[f];
        else if (policy == 2) score = o->wf_agg[(size_t)wf_of[f] * 10 + 9];
        int64_t lv = (int64_t)t->wf_prio[wf_of[f]] + score;
        if (lv < 0) lv = 0;
        if (lv > (int64_t)t->levels - 1) lv = (int64_t)t->levels - 1;
        o->level[f] = (uint8_t)lv;
    }

    /* O5 load and spare per instance: queue lengths + running (P:332-334
     * [§4.1]); spare = max(0, cap - load), capacity hard (Q9). */
    int64_t* spare = (int64_t*)calloc(I ? I : 1, sizeof(int64_t));
    for (uint32_t i = 0; i < I; ++i) {
        uint64_t load = t->i_base_load[i];
        for (uint32_t f = 0; f < N; ++f)
            if ((t->f_state[f] == S_QUEUED || t->f_state[f] == S_RUNNING) && t->f_executor[f] == (int)i)
                load += 1;
        o->i_load[i] = (uint32_t)(load > 0xFFFFFFFFull ? 0xFFFFFFFFull : load);
        spare[i] = (int64_t)t->i_cap[i] - (int64_t)load;
        if (spare[i] < 0) spare[i] = 0;
        o->i_spare[i] = (uint32_t)spare[i];
        o->i_assigned[i] = 0;
    }

    /* statuses before admission */
    for (uint32_t f = 0; f < N; ++f) {
        uint8_t st = t->f_state[f];
        o->instance[f] = -1;
        o->new_pin[f] = 0;
        if (st == S_RESOLVED) o->status[f] = O_RESOLVED;
        else if (st == S_FAILED) o->status[f] = O_FAILED;
        else if (st == S_QUEUED || st == S_RUNNING) { o->status[f] = O_INFLIGHT; o->instance[f] = t->f_executor[f]; }
        else if (doomed[f]) o->status[f] = O_DOOMED;
        else if (!ready[f]) o->status[f] = O_WAITING;
        else if (!eligible[f]) o->status[f] = O_INELIGIBLE;
        else o->status[f] = O_DEFERRED;
    }

    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    uint32_t na = 0;
    g_level = o->level;

    /* O6 phase A: pinned futures, route(session, agent-type, agent-instance)
     * P:387 [§4.2]; a pin overrides weighted rules (Q10).
     * Each instance independently admits its first min(|A|, spare) futures in
     * the O4 order. */
    for (uint32_t p = 0; p < I; ++p) {
        uint32_t n = 0;
        for (uint32_t f = 0; f < N; ++f)
            if (eligible[f] && t->f_pin[f] == (int)p) buf[n++] = f;
        qsort(buf, n, sizeof(uint32_t), cmp_order);
        uint32_t adm = 0;
        for (uint32_t k = 0; k < n; ++k) {
            if ((int64_t)adm < spare[p]) {
                uint32_t f = buf[k];
                o->status[f] = O_ASSIGNED;
                o->instance[f] = (int16_t)p;
                o->assign_row[na] = f;
                o->assign_inst[na] = (int16_t)p;
                na++;
                adm++;
            }
        }
        spare[p] -= adm;
        o->i_assigned[p] += adm;
    }

    /* O7 phase B: unpinned futures, weighted route(agent-type, instances,
     * weights) P:388 with weights proportional to spare in its
     * exact-integer form: literal sequential greedy, each future in O4 order
     * goes to the instance of its type with the most spare, ties to the lowest
     * instance id ("actively balances load ... through routing") (Q11). */
    for (uint32_t ty = 0; ty < T; ++ty) {
        uint32_t n = 0;
        for (uint32_t f = 0; f < N; ++f)
            if (eligible[f] && t->f_pin[f] == -1 && t->f_type[f] == ty) buf[n++] = f;
        qsort(buf, n, sizeof(uint32_t), cmp_order);
        for (uint32_t k = 0; k < n; ++k) {
            uint32_t f = buf[k];
            int64_t best = -1, best_sp = 0;
            for (uint32_t i = 0; i < I; ++i)
                if (t->i_type[i] == ty && spare[i] > best_sp) { best = i; best_sp = spare[i]; }
            if (best < 0) continue;                       /* no spare: DEFERRED */
            spare[best] -= 1;
            o->i_assigned[best] += 1;
            o->status[f] = O_ASSIGNED;
            o->instance[f] = (int16_t)best;
            o->new_pin[f] = (uint8_t)(t->t_affinity[ty] != A_NONE);
            o->assign_row[na] = f;
            o->assign_inst[na] = (int16_t)best;
            na++;
        }
    }

    /* O9 K,V-cache retention hints (DESIGN.md Q-kv).
     * "Because Nalar tracks futures and knows which requests are pending or
     * likely to arrive next, it can supply the LLM serving layer with explicit
     * hints about which K,V caches should be retained" P:527 [§4.3]; whether a
     * cache "remains on the GPU, is offloaded to far memory" P:528, "that a
     * session has ended" P:525; SPEC kv_hint retain | offload | drop S:542.
     * A session is (workflow w, SESSION-affinity type t) (Q13); its cache is at
     * its home = the lowest instance any of its futures is pinned to in the
     * input table (no pin: no cache, no hint).  A future is live if QUEUED,
     * RUNNING, or PENDING and not doomed.
     *   retain  (1): the session has a live future;
     *   offload (2): it has none, but its workflow still has one (it may recur);
     *   drop    (3): its workflow has no live future (the session has ended).
     * kv_level = the highest O4 level among the session's live futures (the
     * retention urgency), 0 when none. */
    for (uint32_t w = 0; w < W; ++w) {
        uint32_t wf_live = 0;
        for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) {
            uint8_t st = t->f_state[f];
            if (st == S_QUEUED || st == S_RUNNING || (st == S_PENDING && !doomed[f])) wf_live++;
        }
        for (uint32_t ty = 0; ty < T; ++ty) {
            size_t k = (size_t)w * T + ty;
            int home = -1;
            uint32_t live = 0, lv = 0;
            if (t->t_affinity[ty] == A_SESSION) {
                for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) {
                    if (t->f_type[f] != ty) continue;
                    int pin = t->f_pin[f];
                    if (pin >= 0 && (home < 0 || pin < home)) home = pin;
                    uint8_t st = t->f_state[f];
                    if (st == S_QUEUED || st == S_RUNNING || (st == S_PENDING && !doomed[f])) {
                        live++;
                        if (o->level[f] > lv) lv = o->level[f];
                    }
                }
            }
            uint8_t hint = 0;
            if (home >= 0) hint = live > 0 ? 1 : (wf_live > 0 ? 2 : 3);
            if (o->kv_hint) o->kv_hint[k] = hint;
            if (o->kv_level) o->kv_level[k] = (uint8_t)lv;
            if (o->kv_home) o->kv_home[k] = (int16_t)home;
        }
    }

    o->n_assigned = na;
    o->n_ready = n_ready;
    o->n_eligible = n_elig;
    o->n_doomed = n_doomed;
    free(buf); free(spare); free(inflight_wt); free(first_pending); free(first_ready_unp);
    free(doomed); free(ready); free(eligible); free(wf_of);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O10 resource reassignment (DESIGN.md Q-ra).           */
/* "resource reassignment from low-load agents to high-load agents" P:663,   */
/* P:672, P:676 [§6.1]; kill / provision primitives P:393-394 [§4.2];        */
/* max_instances / min_instances directives P:252-253 (Table 1); SPEC        */
/* resource_reassign S:448-456: if type A's utilisation > u_hi and B's <     */
/* u_lo, B above min_instances and A below max_instances, emit Kill(one B     */
/* instance) + Provision(A).                                                  */
/*   busy_t = sum over t's instances of (load + assigned this epoch)          */
/*            + t's DEFERRED futures (unmet demand);  cap_t = sum of caps;    */
/*   util_t = busy_t / cap_t, compared exactly: 100 busy vs pct * cap;        */
/*   hot:  n_t < max_t and 100 busy_t > u_hi cap_t;                           */
/*   cold: n_t > min_t and 100 busy_t < u_lo cap_t;                            */
/*   hot types by util desc, cold by util asc (ties: lower type id); the k-th */
/*   hot is paired with the k-th cold: kill the cold type's instance with the */
/*   least (load + assigned) (ties: the highest id), provision the hot type.  */
/* ------------------------------------------------------------------------ */
static const uint64_t* g_busy;
static const uint64_t* g_cap;
/* util(a) > util(b) as exact fractions; cap 0 with busy > 0 is infinite */
static int util_gt(uint32_t a, uint32_t b) {
    uint64_t ba = g_busy[a], ca = g_cap[a], bb = g_busy[b], cb = g_cap[b];
    int ia = ca == 0 && ba > 0, ib = cb == 0 && bb > 0;
    if (ia || ib) return ia && !ib;
    if (ca == 0 && cb == 0) return 0;                        /* both 0/0: equal */
    if (ca == 0) return 0;                                   /* 0/0 = 0 */
    if (cb == 0) return ba > 0;
    return (unsigned __int128)ba * cb > (unsigned __int128)bb * ca;
}
static int cmp_hot(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    if (util_gt(a, b)) return -1;
    if (util_gt(b, a)) return 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static int cmp_cold(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    if (util_gt(b, a)) return -1;
    if (util_gt(a, b)) return 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

int oracle_reassign(const oracle_table* t, const oracle_out* o, const oracle_ra_params* p, oracle_ra_out* r) {
    uint32_t N = t->n_futures, I = t->n_instances, T = t->n_types;
    uint64_t* busy = (uint64_t*)calloc(T ? T : 1, sizeof(uint64_t));
    uint64_t* cap = (uint64_t*)calloc(T ? T : 1, sizeof(uint64_t));
    uint32_t* cnt = (uint32_t*)calloc(T ? T : 1, sizeof(uint32_t));
    uint32_t* hot = (uint32_t*)malloc(sizeof(uint32_t) * (T ? T : 1));
    uint32_t* cold = (uint32_t*)malloc(sizeof(uint32_t) * (T ? T : 1));
    for (uint32_t i = 0; i < I; ++i) {
        uint32_t ty = t->i_type[i];
        busy[ty] += (uint64_t)o->i_load[i] + o->i_assigned[i];
        cap[ty] += t->i_cap[i];
        cnt[ty] += 1;
    }
    for (uint32_t f = 0; f < N; ++f)
        if (o->status[f] == O_DEFERRED) busy[t->f_type[f]] += 1;
    uint32_t nh = 0, nc = 0;
    for (uint32_t ty = 0; ty < T; ++ty) {
        r->t_busy[ty] = (uint32_t)(busy[ty] > 0xFFFFFFFFull ? 0xFFFFFFFFull : busy[ty]);
        r->t_cap[ty] = (uint32_t)(cap[ty] > 0xFFFFFFFFull ? 0xFFFFFFFFull : cap[ty]);
        uint32_t mn = p->t_min_inst ? p->t_min_inst[ty] : 0u;
        uint32_t mx = p->t_max_inst ? p->t_max_inst[ty] : 0xFFFFu;
        if (cnt[ty] < mx && 100ull * busy[ty] > (uint64_t)p->u_hi_pct * cap[ty]) hot[nh++] = ty;
        else if (cnt[ty] > mn && 100ull * busy[ty] < (uint64_t)p->u_lo_pct * cap[ty]) cold[nc++] = ty;
    }
    g_busy = busy;
    g_cap = cap;
    qsort(hot, nh, sizeof(uint32_t), cmp_hot);
    qsort(cold, nc, sizeof(uint32_t), cmp_cold);
    uint32_t np = nh < nc ? nh : nc;
    for (uint32_t k = 0; k < np; ++k) {
        int64_t best = -1;
        uint64_t best_b = 0;
        for (uint32_t i = 0; i < I; ++i) {
            if (t->i_type[i] != cold[k]) continue;
            uint64_t b = (uint64_t)o->i_load[i] + o->i_assigned[i];
            if (best < 0 || b <= best_b) { best = i; best_b = b; }     /* ties: the highest id */
        }
        r->kill_inst[k] = (int16_t)best;
        r->prov_type[k] = (int16_t)hot[k];
    }
    r->n_pairs = np;
    free(busy); free(cap); free(cnt); free(hot); free(cold);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O11 head-of-line-blocking migration (DESIGN.md Q-mig). */
/* "migrates a job if it's waiting in the queue and observing head-of-line   */
/* blocking" P:663 [§6.1]; the migrate primitive P:391 and its protocol      */
/* (Fig 5); SPEC hol_migration S:441: for each Queued future whose */
/* wait age > theta_wait and whose instance's head job has predicted          */
/* remaining time > theta_head, Migrate to the instance with the smallest     */
/* (queue_len + running), provided its backlog is below the source's by      */
/* margin delta; managed-state agents move whole sessions.    */
/*   blocked(i) = head_rem[i] > theta_head; sources are blocked instances,    */
/*   destinations unblocked ones of the same type (no capacity test: a moved  */
/*   future queues there, SPEC compares backlogs only; the margin guards);    */
/*   backlog = load + assigned this epoch (O5-O7).                            */
/*   A QUEUED future f at a blocked executor s with age > theta_wait is a     */
/*   candidate unless its type is STATEFUL (in-order per session:     */
/*   never moves); a SESSION future only if it is its session's only QUEUED   */
/*   future and the session has nothing RUNNING (moving it moves the whole    */
/*   session; a running session defers).                          */
/*   Per type, candidates in the O4 order, literal sequential greedy:         */
/*   d = argmin backlog over unblocked instances of the type (ties: lowest    */
/*   id); migrate iff d exists and backlog[d] + delta <=                      */
/*   backlog[s]; then backlog[s] -= 1, backlog[d] += 1.                       */
/* ------------------------------------------------------------------------ */
int oracle_migrate(const oracle_table* t, const oracle_out* o, const oracle_mig_params* p, oracle_mig_out* r) {
    uint32_t N = t->n_futures, W = t->n_workflows, I = t->n_instances, T = t->n_types;
    int64_t* backlog = (int64_t*)calloc(I ? I : 1, sizeof(int64_t));
    uint8_t* blocked = (uint8_t*)calloc(I ? I : 1, 1);
    uint8_t* cand = (uint8_t*)calloc(N ? N : 1, 1);
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    for (uint32_t i = 0; i < I; ++i) {
        backlog[i] = (int64_t)o->i_load[i] + o->i_assigned[i];
        blocked[i] = (uint8_t)(p->i_head_rem[i] > p->theta_head);
        r->i_mig_in[i] = 0;
        r->i_mig_out[i] = 0;
    }
    for (uint32_t f = 0; f < N; ++f) r->migrate_to[f] = -1;
    /* candidates */
    for (uint32_t w = 0; w < W; ++w) {
        for (uint32_t f = t->wf_fut_off[w]; f < t->wf_fut_off[w + 1]; ++f) {
            if (t->f_state[f] != S_QUEUED) continue;
            int s = t->f_executor[f];
            uint8_t ty = t->f_type[f], aff = t->t_affinity[ty];
            if (!blocked[s] || p->f_age[f] <= p->theta_wait || aff == A_STATEFUL) continue;
            if (aff == A_SESSION) {
                uint32_t nq = 0, nr = 0;
                for (uint32_t g = t->wf_fut_off[w]; g < t->wf_fut_off[w + 1]; ++g) {
                    if (t->f_type[g] != ty) continue;
                    if (t->f_state[g] == S_QUEUED) nq++;
                    if (t->f_state[g] == S_RUNNING) nr++;
                }
                if (nq != 1 || nr != 0) continue;
            }
            cand[f] = 1;
        }
    }
    g_level = o->level;
    uint32_t nm = 0;
    for (uint32_t ty = 0; ty < T; ++ty) {
        uint32_t n = 0;
        for (uint32_t f = 0; f < N; ++f)
            if (cand[f] && t->f_type[f] == ty) buf[n++] = f;
        qsort(buf, n, sizeof(uint32_t), cmp_order);
        for (uint32_t k = 0; k < n; ++k) {
            uint32_t f = buf[k];
            int s = t->f_executor[f];
            int64_t d = -1;
            for (uint32_t i = 0; i < I; ++i)
                if (t->i_type[i] == ty && !blocked[i] && (d < 0 || backlog[i] < backlog[d])) d = i;
            if (d < 0 || backlog[d] + (int64_t)p->delta > backlog[s]) continue;
            backlog[s] -= 1;
            backlog[d] += 1;
            r->migrate_to[f] = (int16_t)d;
            r->i_mig_out[s] += 1;
            r->i_mig_in[d] += 1;
            nm++;
        }
    }
    r->n_migrated = nm;
    free(backlog); free(blocked); free(cand); free(buf);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O12 batch coalescing (DESIGN.md Q-batch).             */
/* "if an agent supports batching ... Nalar can coalesce compatible futures  */
/* and execute them together" P:261 [§3.4]; `batchable` directive P:250      */
/* (Table 1); managed state cannot be combined with batchable agents P:576;  */
/* SPEC schedule_next S:281: greedily coalesces up to max_batch queued       */
/* futures with identical (agent_type, method) into one Batch, in priority   */
/* order; compatibility key (agent_type, method) S:341.                       */
/*   For each instance i of a batchable type (max_batch > 1) and method m:   */
/*   the futures ASSIGNED to i this epoch with method m, in the O4 order, are */
/*   cut into consecutive batches of max_batch; batch_head[f] = the row of    */
/*   its batch's first future; -1 for every other future.                    */
/* ------------------------------------------------------------------------ */
int oracle_batch(const oracle_table* t, const oracle_out* o, const oracle_batch_params* p, oracle_batch_out* r) {
    uint32_t N = t->n_futures, I = t->n_instances, T = t->n_types;
    for (uint32_t ty = 0; ty < T; ++ty)
        if (p->t_max_batch[ty] > 1 && t->t_affinity[ty] != A_NONE) return -1;
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (N ? N : 1));
    for (uint32_t f = 0; f < N; ++f) r->batch_head[f] = -1;
    g_level = o->level;
    uint32_t nb = 0;
    for (uint32_t i = 0; i < I; ++i) {
        uint32_t mb = p->t_max_batch[t->i_type[i]];
        if (mb <= 1) continue;
        for (uint32_t m = 0; m < 256; ++m) {
            uint32_t n = 0;
            for (uint32_t f = 0; f < N; ++f)
                if (o->status[f] == O_ASSIGNED && o->instance[f] == (int)i &&
                    (p->f_method ? p->f_method[f] : 0u) == m)
                    buf[n++] = f;
            if (!n) continue;
            qsort(buf, n, sizeof(uint32_t), cmp_order);
            for (uint32_t k = 0; k < n; ++k) {
                r->batch_head[buf[k]] = (int32_t)buf[k - k % mb];
                if (k % mb == 0) nb++;
            }
        }
    }
    r->n_batches = nb;
    free(buf);
    return 0;
}

/* Timing harness for bench.py's cpu_baseline (not part of the method): runs
 * oracle_epoch `reps` times on the same table and writes each run's
 * wall-clock nanoseconds (CLOCK_MONOTONIC around O1-O9 only; the caller's
 * output buffers are allocated once, outside the timed region). */
int oracle_epoch_timed(const oracle_table* t, int policy, oracle_out* o, int reps, uint64_t* ns) {
    for (int r = 0; r < reps; ++r) {
        struct timespec a, b;
        clock_gettime(CLOCK_MONOTONIC, &a);
        const int rc = oracle_epoch(t, policy, o);
        clock_gettime(CLOCK_MONOTONIC, &b);
        if (rc) return rc;
        ns[r] = (uint64_t)(b.tv_sec - a.tv_sec) * 1000000000ull + (uint64_t)(b.tv_nsec - a.tv_nsec);
    }
    return 0;
}
