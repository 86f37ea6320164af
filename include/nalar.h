/* nalar.h -- C ABI of the B200 policy-epoch library (libnalar.so).
 *
 * The data-parallel hot path of Nalar's global controller (arXiv 2601.05109):
 * one POLICY EPOCH over the live future table.  "Running periodically, the
 * global controller tracks the global state ... by aggregating metrics and
 * metadata from component-level controllers ..., computing decisions related
 * (for request routing, prioritization, and resource allocation) and pushing
 * the computed decisions" (PAPER.md:338 [§4.1]); the single-threaded policy loop
 * (PAPER.md:364 [§4.2]) is re-expressed as sm_100a kernels that reproduce its
 * sequential definition bit for bit (readings Q1-Q22).
 *
 * Three calls carry the path:
 *   nalar_snapshot_upload  -- the "collect" hand-off: host SoA table -> HBM,
 *                             validated
 *   nalar_policy_epoch     -- readiness, depth, doom, per-workflow aggregates,
 *                             priority key, load, capacity-limited assignment
 *   nalar_fetch_decisions  -- the "push" hand-off: decisions -> host
 *                             (route / set_priority)
 *
 * Conventions
 *  - Every function returns NALAR_OK (0) or a negative nalar_err.  Nothing
 *    throws or aborts; nalar_last_error(ctx) describes the last failure.
 *  - Ownership: the library owns all device memory it allocates (sized once at
 *    nalar_create from the reservations in nalar_config), or carves it out of
 *    caller memory given in nalar_config.workspace.  Input host pointers are
 *    borrowed only for the duration of a call.  Outputs go to caller buffers.
 *  - Call order: upload -> epoch -> fetch; fetch/epoch before any successful
 *    upload return NALAR_E_STATE.  A ctx is not thread-safe.  Every call
 *    runs on the ctx's device and leaves the caller's current device as it was.
 *  - Multi-GPU: one ctx per GPU/rank; every rank uploads its contiguous
 *    workflow range (plus the replicated instance and type tables) and calls
 *    every function; nalar_policy_epoch is then a collective.
 *  - No CPU fallback: without a usable sm_100 device nalar_create fails.
 */
#ifndef NALAR_H
#define NALAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NALAR_ABI_VERSION 2

/* limits (DESIGN.md §3 "Data layout") */
#define NALAR_MAX_LEVELS     256      /* level is u8                          */
#define NALAR_MAX_TYPES      64
#define NALAR_MAX_INSTANCES  1024     /* instance ids are i16; R = I + T       */
#define NALAR_MAX_ROWS       0x7FFFFFFFu /* edge rows use 31 bits              */
#define NALAR_CALL_EDGE      0x80000000u /* edges[] bit 31: CALL (creator) edge */
#define NALAR_WF_AGG_FIELDS  10

typedef struct nalar_ctx nalar_ctx; /* opaque; one per GPU / rank */

enum nalar_err {
    NALAR_OK = 0,
    NALAR_E_INVAL = -1,   /* malformed snapshot or argument (see upload)     */
    NALAR_E_STATE = -2,   /* call out of order                               */
    NALAR_E_NOMEM = -3,   /* snapshot exceeds the reservation / alloc failed */
    NALAR_E_SIZE = -4,    /* caller output buffer too small (sizes written)  */
    NALAR_E_CUDA = -5,    /* CUDA runtime error / no sm_100 device           */
    NALAR_E_COMM = -6,    /* NCCL error                                      */
    NALAR_E_NOTIMPL = -7
};

/* per-future lifecycle, collapsed from SPEC S:46-53 (DESIGN.md Q-state) */
enum nalar_state { NALAR_PENDING = 0, NALAR_QUEUED = 1, NALAR_RUNNING = 2,
                   NALAR_RESOLVED = 3, NALAR_FAILED = 4 };
/* per-type state-placement directive: managed state = SESSION,
 * `stateful` directive = STATEFUL */
enum nalar_aff { NALAR_AFF_NONE = 0, NALAR_AFF_SESSION = 1, NALAR_AFF_STATEFUL = 2 };
/* priority score: FCFS, SRTF "later stages of the graph",
 * LPT "jobs that re-enter the graph" */
enum nalar_policy { NALAR_FCFS = 0, NALAR_SRTF = 1, NALAR_LPT = 2 };
/* per-future decision */
enum nalar_status { NALAR_S_RESOLVED = 0, NALAR_S_FAILED = 1, NALAR_S_INFLIGHT = 2,
                    NALAR_S_WAITING = 3, NALAR_S_DOOMED = 4, NALAR_S_INELIGIBLE = 5,
                    NALAR_S_DEFERRED = 6, NALAR_S_ASSIGNED = 7 };
/* how ranks exchange the per-epoch histogram / load buffer (world > 1) */
enum nalar_collective { NALAR_COLL_NONE = 0,     /* world == 1                       */
                        NALAR_COLL_NCCL = 1,     /* library-owned ncclComm, in-graph */
                        NALAR_COLL_EXTERNAL = 2, /* caller sums the exchange buffer
                                                    between epoch_begin / finish      */
                        NALAR_COLL_PEER = 3      /* kernels store each rank's slot into
                                                    every peer's buffer (NVLink peer
                                                    memory), world <= 8; connect with
                                                    nalar_peer_connect before the
                                                    first epoch                       */ };
/* nalar_config.flags */
#define NALAR_F_TIMING          1u  /* record per-kernel CUDA events (stats)      */
#define NALAR_F_NO_GRAPH        2u  /* launch kernels directly, no CUDA graph     */
#define NALAR_F_FORCE_UNSTAGED  4u  /* test knob: K1 reads HBM, no smem staging   */
#define NALAR_F_PROFILE         8u  /* K1 records %globaltimer stamps (diagnostics) */

typedef struct {
    int      device;          /* CUDA ordinal                                      */
    int      rank, world;     /* world == 1: single GPU                            */
    int      collective;      /* nalar_collective                                  */
    unsigned char nccl_id[128]; /* ncclUniqueId from nalar_nccl_unique_id() on rank 0,
                                 broadcast by the caller (NALAR_COLL_NCCL only)    */
    void*    stream;          /* cudaStream_t to run on (e.g. torch's), NULL = own */
    void*    workspace;       /* optional caller device memory, >= nalar_workspace_bytes() */
    size_t   workspace_bytes;
    uint32_t levels;          /* Lv, 1..256 (default 256 when 0)                   */
    uint32_t max_futures, max_edges, max_workflows, max_instances, max_types;
    uint32_t flags;           /* NALAR_F_*                                         */
} nalar_config;

/* The live future table, structure-of-arrays, rows in (workflow_id, seq) order
 * (creation order within a workflow).  HOST pointers (pageable or pinned),
 * borrowed for the call.  Field meanings: future metadata PAPER.md:469-485
 * (dependencies, creator, executor), session ids PAPER.md:519, instance metrics
 * PAPER.md:332-334, directives PAPER.md:242-258.
 *   wf_fut_off[W+1]: rows of workflow w are [wf_fut_off[w], wf_fut_off[w+1])
 *   f_edge_off[N+1], edges[E]: CSR predecessor lists; edges[e] bits 0..30 =
 *     predecessor row (an EARLIER row of the SAME workflow), bit 31 =
 *     NALAR_CALL_EDGE for the creator (CALL) edge, 0 for a DEP (argument) edge
 *   f_executor: instance a QUEUED/RUNNING future sits at (-1 otherwise)
 *   f_pin: session home instance of the future (state placement), -1 none
 *   global_row_base: index of row 0 in the all-rank row order (multi-GPU)   */
typedef struct {
    uint32_t n_futures, n_edges, n_workflows, n_instances, n_types;
    uint64_t global_row_base;
    const uint64_t* wf_id;       /* [W] strictly increasing                  */
    const uint32_t* wf_fut_off;  /* [W+1]                                    */
    const int32_t*  wf_prio;     /* [W] set_priority value     */
    const uint8_t*  f_state;     /* [N] nalar_state                          */
    const uint8_t*  f_type;      /* [N] < n_types                            */
    const uint8_t*  f_round;     /* [N] retry round (LPT input)              */
    const int16_t*  f_executor;  /* [N]                                      */
    const int16_t*  f_pin;       /* [N]                                      */
    const uint32_t* f_edge_off;  /* [N+1]                                    */
    const uint32_t* edges;       /* [E]                                      */
    const uint8_t*  i_type;      /* [I] < n_types                            */
    const uint32_t* i_cap;       /* [I] capacity (queue + running)           */
    const uint32_t* i_base_load; /* [I] load outside the table               */
    const uint8_t*  t_affinity;  /* [T] nalar_aff                            */
    /* HoL-migration inputs (NEXT-1), may be NULL (then nothing migrates):
     * wait age of each QUEUED future and the predicted remaining time of
     * each instance's head job, in one caller-chosen time unit */
    const uint32_t* f_age;       /* [N]                                      */
    const uint32_t* i_head_rem;  /* [I]                                      */
    /* batch-coalescing key with the agent type (NEXT-4), may be
     * NULL (all methods 0)                                                  */
    const uint8_t*  f_method;    /* [N]                                      */
} nalar_snapshot;

/* Delta between two epochs of a dynamic workload (SURVEY §8(c) "Delta
 * semantics"; the dynamic control flow of PAPER.md:45, 458-460: futures are
 * created as the program runs, resolve, and whole workflows retire).  Applied
 * by nalar_delta_apply in this order:
 *  1. flags & NALAR_DELTA_APPLY_ASSIGNED: every future ASSIGNED by the last
 *     epoch becomes QUEUED at its assigned instance;
 *  2. per-future updates addressed by (workflow id, seq), seq = the future's
 *     index inside its workflow in creation order; a field equal to
 *     NALAR_KEEP_STATE / NALAR_KEEP_I16 is left unchanged;
 *  3. retired workflows (by id) are removed whole;
 *  4. appended futures are added at the END of their workflow in array order
 *     (grouped by workflow id, ids ascending); an id not in the table opens a
 *     new workflow with priority app_wf_prio[first row] and must exceed every
 *     live id; an appended future's edges name EARLIER futures of the same
 *     workflow by seq (bit 31 = NALAR_CALL_EDGE);
 *  5. set_priority updates by workflow id, then instance cap / base-load
 *     updates.
 * The per-upload optional inputs (f_age / i_head_rem, f_method) describe rows
 * of the uploaded table; a delta moves rows, so it clears them (nothing
 * migrates, every method is 0) until the next nalar_snapshot_upload.
 * All pointers are HOST pointers borrowed for the call. */
#define NALAR_DELTA_APPLY_ASSIGNED 1u
#define NALAR_KEEP_STATE 0xFFu
#define NALAR_KEEP_I16   (-2)
typedef struct {
    uint32_t flags;
    uint32_t n_updates;
    const uint64_t* upd_wf_id;     /* [n_updates] */
    const uint32_t* upd_seq;
    const uint8_t*  upd_state;     /* nalar_state or NALAR_KEEP_STATE */
    const int16_t*  upd_executor;  /* instance, -1, or NALAR_KEEP_I16 */
    const int16_t*  upd_pin;       /* instance, -1, or NALAR_KEEP_I16 */
    uint32_t n_retired;
    const uint64_t* retired_wf_id; /* [n_retired] */
    uint32_t n_append, n_append_edges;
    const uint64_t* app_wf_id;     /* [n_append] */
    const int32_t*  app_wf_prio;   /* [n_append] used when the row opens a workflow */
    const uint8_t*  app_state;
    const uint8_t*  app_type;
    const uint8_t*  app_round;
    const int16_t*  app_executor;
    const int16_t*  app_pin;
    const uint32_t* app_edge_off;  /* [n_append+1] */
    const uint32_t* app_edges;     /* [n_append_edges] predecessor seq | CALL bit */
    uint32_t n_prio;
    const uint64_t* prio_wf_id;    /* [n_prio] */
    const int32_t*  prio_value;
    uint32_t n_inst;
    const uint32_t* inst_id;       /* [n_inst] */
    const uint32_t* inst_cap;
    const uint32_t* inst_base_load;
} nalar_delta;

/* Caller-allocated HOST output buffers; any pointer may be NULL (skipped).
 * *_cap = capacity in elements.  On NALAR_E_SIZE the n_* fields hold the
 * required sizes and nothing is copied. */
typedef struct {
    uint8_t*  status;     /* [N] nalar_status                                  */
    uint8_t*  level;      /* [N] priority level, 0 for terminal futures        */
    uint16_t* depth;      /* [N] longest DEP u CALL path from a root (sat. u16) */
    int16_t*  instance;   /* [N] executor (INFLIGHT) / assigned (ASSIGNED) / -1 */
    uint8_t*  new_pin;    /* [N] 1 = assignment creates the session's pin       */
    uint32_t  f_cap;
    uint32_t* wf_agg;     /* [W][10] total, pending, ready, inflight, resolved,
                             failed, doomed, pinned_pending, max_depth, max_round */
    uint32_t  wf_cap;
    uint32_t* i_load;     /* [I] base_load + in-flight futures of ALL ranks      */
    uint32_t* i_spare;    /* [I] max(0, cap - load) before this epoch's admission */
    uint32_t* i_assigned; /* [I] futures of ALL ranks assigned this epoch        */
    uint32_t  i_cap;
    uint32_t* assign_row; /* [n_assigned] this rank's assigned rows, ordered by
                             (resource, global rank); resource = pin for pinned
                             futures, I + type for unpinned ones               */
    int16_t*  assign_inst;/* [n_assigned] their instances                      */
    uint32_t  a_cap;
    uint32_t  n_f, n_w, n_i, n_assigned;  /* out */
    /* K,V-cache retention hints ("explicit
     * hints about which K,V caches should be retained", SPEC kv_hint S:542),
     * one entry per (workflow w, type t), row-major [W][T].  A session is a
     * workflow's SESSION-affinity type; its home is the lowest instance any of
     * its futures is pinned to in the uploaded table.  With a home:
     * 1 retain (a live -- QUEUED, RUNNING or non-doomed PENDING -- future of the
     * session exists), 2 offload (none, but the workflow has a live future),
     * 3 drop (the workflow has none: the session ended); 0 otherwise.        */
    uint8_t*  kv_hint;    /* [W][T]                                            */
    uint8_t*  kv_level;   /* [W][T] max level of the session's live futures    */
    int16_t*  kv_home;    /* [W][T] home instance or -1                        */
    uint32_t  kv_cap;     /* elements (>= W * T)                               */
    /* Resource reassignment (only with
     * nalar_policy_params.reassign): per type t, busy_t = sum over t's
     * instances of (load + assigned this epoch) + t's deferred futures, and
     * cap_t = sum of capacities; and the commands, pair k = Kill(ra_kill[k])
     * + Provision(type ra_prov[k]), hottest type with the
     * coldest.  Identical on every rank.                                     */
    uint32_t* t_busy;     /* [T]                                               */
    uint32_t* t_capsum;   /* [T]                                               */
    int16_t*  ra_kill;    /* [T] (n_reassign used)                             */
    int16_t*  ra_prov;    /* [T]                                               */
    uint32_t  t_cap;      /* elements of the four arrays above (>= T)          */
    uint32_t  n_reassign; /* out                                               */
    /* HoL migration (only with nalar_policy_params.migrate):
     * migrate_to[f] = destination instance of a QUEUED future (a SESSION
     * future carries its session: re-home its pin), -1 none.  world > 1: the
     * rank's own rows; i_mig_in / i_mig_out / n_migrated are global (the same
     * on every rank).                                                         */
    int16_t*  migrate_to; /* [N] (capacity f_cap)                              */
    uint32_t* i_mig_in;   /* [I] (capacity i_cap)                              */
    uint32_t* i_mig_out;  /* [I]                                               */
    uint32_t  n_migrated; /* out                                               */
    /* Batch coalescing (only with a max_batch > 1):
     * batch_head[f] = GLOBAL row (snapshot global_row_base + row) of the
     * first future of f's batch -- the futures assigned to one instance this
     * epoch with one method, in priority order, cut into batches of max_batch
     * -- or -1.  world > 1: the rank's own
     * rows (a head may be another rank's row); n_batches is global.          */
    int32_t*  batch_head; /* [N] (capacity f_cap)                              */
    uint32_t  n_batches;  /* out                                               */
} nalar_decisions;

/* Policy parameters beyond the per-epoch policy (persist on the context;
 * take effect from the next epoch). */
typedef struct {
    /* resource reassignment (NEXT-2; "resource reassignment from
     * low-load agents to high-load agents"): type A with
     * 100 busy_A > u_hi_pct cap_A and fewer than max_instances[A] instances is
     * hot, type B with 100 busy_B < u_lo_pct cap_B and more than
     * min_instances[B] is cold (max/min_instances: the Table 1 directives,
     * PAPER.md:252-253).  Hot types by utilisation desc are paired with cold
     * ones by utilisation asc (ties: lower type id); the killed instance is
     * the cold type's least-loaded (load + assigned; ties: highest id). */
    uint32_t reassign;             /* 0 off, 1 on                                  */
    uint32_t u_hi_pct, u_lo_pct;   /* percent, u_lo_pct <= u_hi_pct (SPEC: 80 / 30) */
    const uint16_t* t_min_inst;    /* [n_types] or NULL (all 0)                    */
    const uint16_t* t_max_inst;    /* [n_types] or NULL (all 65535)                */
    uint32_t n_types;              /* <= max_types                                 */
    /* HoL migration (NEXT-1; "migrates a job if it's waiting in
     * the queue and observing head-of-line blocking"): a QUEUED
     * future with age > theta_wait at an instance whose head job has
     * head_rem > theta_head (blocked) moves, in priority order, to the
     * least-backlogged (load + assigned) unblocked instance of its type while
     * that backlog + delta <= the source's; STATEFUL futures never move, a
     * SESSION future only as its session's sole queued work with nothing of
     * the session running.  world > 1: every rank's candidates travel in the
     * epoch's one exchange (a list region per rank after the (row base, rows)
     * pairs; nalar_exchange_buffer's n_words covers it) and every rank runs
     * the same greedy; more than 8127 candidates on one rank: the fetch /
     * stats return E_NOTIMPL. */
    uint32_t migrate;              /* 0 off, 1 on                                  */
    uint32_t theta_wait, theta_head, delta;
    /* batch coalescing (NEXT-4): the `batchable` directive as a per-type
     * max_batch (<= 1: not batchable; Table 1).  A batchable type
     * must have affinity NONE ("cannot be combined with batchable agents",
     * PAPER.md:576): the epoch returns E_INVAL otherwise.  world > 1: every
     * rank's eligible futures of the batchable resources travel in the
     * epoch's one exchange (the list region, as for migration) and every rank
     * re-derives their admission; E_STATE after a delta (global row base
     * unknown), E_NOTIMPL at the fetch when a rank's list overflows. */
    const uint16_t* t_max_batch;   /* [n_types] or NULL (no batching)              */
} nalar_policy_params;

/* Copies p (host arrays borrowed for the call).  E_INVAL on u_lo > u_hi or
 * n_types > max_types. */
int nalar_set_policy_params(nalar_ctx* ctx, const nalar_policy_params* p);

/* TickReport analog. */
typedef struct {
    float    epoch_us;        /* device time of the last epoch (NALAR_F_TIMING)  */
    float    k1_us, coll_us, k4_us;
    uint32_t n_futures, n_ready, n_eligible, n_assigned, n_deferred, n_doomed, n_instances;
} nalar_epoch_stats;

/* Bytes of device workspace nalar_create needs for cfg's reservations. */
size_t nalar_workspace_bytes(const nalar_config* cfg);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0 only; loads NCCL). */
int nalar_nccl_unique_id(unsigned char out[128]);

/* Create a context on cfg->device: allocate/carve device memory, create the
 * stream (if none given) and, for NALAR_COLL_NCCL, the communicator
 * (collective over all ranks).  E_INVAL on bad limits, E_CUDA without an
 * sm_100 device, E_COMM on NCCL failure. */
int nalar_create(nalar_ctx** out, const nalar_config* cfg);
int nalar_destroy(nalar_ctx* ctx);

/* Copy a snapshot to HBM and validate it (stream-ordered, then synchronises).
 * E_NOMEM if a size exceeds the reservation; E_INVAL if: offsets are not
 * monotone / do not start at 0 / end at N or E; wf_id not strictly
 * increasing; a state > 4, type >= T, affinity > 2 or instance type >= T; a
 * pin not naming an instance of the future's type; a QUEUED/RUNNING future
 * without an executor of its type; an edge not pointing to an earlier row of
 * the same workflow.  *err_row (may be NULL) = smallest offending row, or -1
 * when the error is not attributable to a row. */
int nalar_snapshot_upload(nalar_ctx* ctx, const nalar_snapshot* snap, int64_t* err_row);

/* Apply a delta to the resident table (see nalar_delta), on the device, then
 * validate it like an upload (stream-ordered, synchronises).  E_STATE before
 * any upload (or APPLY_ASSIGNED before any epoch); E_NOMEM if the table
 * outgrows the reservation; E_INVAL on an unknown (workflow id, seq) or
 * retired id, a new id not above the live ids, an appended edge not naming an
 * earlier future of its workflow, or any row the upload contract rejects.
 * *err_index (may be NULL): the offending update / retired / appended index
 * (by the stage that failed), or the smallest offending row, or -1. */
int nalar_delta_apply(nalar_ctx* ctx, const nalar_delta* delta, int64_t* err_index);

/* One policy epoch over the uploaded table (nalar_policy).  Asynchronous on
 * the ctx stream; a collective over all ranks when world > 1 (NCCL mode).
 * Repeated epochs on the same upload are idempotent. */
int nalar_policy_epoch(nalar_ctx* ctx, int policy);

/* NALAR_COLL_EXTERNAL: the epoch in two halves around a caller-side sum of
 * the exchange buffer (u32 words, slot-disjoint histogram + per-instance load,
 * DESIGN.md §5) over all ranks.  *dev_ptr is device memory owned by ctx. */
int nalar_epoch_begin(nalar_ctx* ctx, int policy);
int nalar_exchange_buffer(nalar_ctx* ctx, void** dev_ptr, size_t* n_words);
int nalar_epoch_finish(nalar_ctx* ctx);

/* NALAR_COLL_PEER.  Every rank owns a receive buffer (library cudaMalloc);
 * peers write their histogram slot and partial sums into it and raise an
 * epoch-numbered flag.  nalar_peer_buffer returns this rank's
 * buffer as a device pointer and as a CUDA IPC handle (64 bytes) for
 * ranks in other processes.  nalar_peer_connect takes, per rank q < world,
 * either ptrs[q] (a device pointer valid in this process: ranks driven by one
 * process, on one device or on peer-enabled devices) or handles[64 q] (an IPC
 * handle, opened here); ptrs / handles may be NULL, ptrs[rank] is ignored.
 * Call on every rank before its first epoch; all ranks must run the same
 * sequence of epochs.  A peer that never arrives makes the epoch's waiting
 * kernel give up after 5 s: the next fetch / stats call returns NALAR_E_COMM.
 * The failure is sticky and spreads: the failing rank poisons its flags in
 * every peer's buffer, so each peer's next exchange fails at once (never
 * pairing its epoch with stale data); later epochs on a failed context
 * return NALAR_E_COMM.  Recover by calling nalar_peer_buffer (which clears
 * this rank's buffer and epoch counter; the context's stream must be idle and
 * no peer may be mid-epoch) and then nalar_peer_connect on every rank. */
int nalar_peer_buffer(nalar_ctx* ctx, void** dev_ptr, unsigned char ipc_handle[64]);
int nalar_peer_connect(nalar_ctx* ctx, void* const* ptrs, const unsigned char* handles);

/* One controller step in one call: upload `snap` (as nalar_snapshot_upload),
 * run the policy epoch and fetch the decisions into `out` (as
 * nalar_fetch_decisions), with ONE synchronisation instead of three: the
 * table's validation (K0) is queued ahead of the epoch and its verdict is read
 * after the fetch; the epoch kernels read it on the device and skip an invalid
 * table.  Errors: those of the three calls; on NALAR_E_INVAL (invalid table,
 * *err_row = the smallest offending row as for upload) the contents of `out`
 * are unspecified and the context is left not uploaded.  Not with
 * NALAR_COLL_EXTERNAL (use the split calls).
 * Streamed step: when the per-row arrays (f_state, f_type, f_round, f_pin,
 * f_executor, f_edge_off, edges) are all in pinned (device-mapped) host memory,
 * every K1 block fits shared memory and neither HoL migration inputs nor batch
 * coalescing are in use, the sweep stages its rows straight from the caller's
 * memory (TMA over PCIe), checks K0's contract on them in shared memory and
 * writes the context's device copy of the table (so later split calls see the
 * same table); there is no separate copy of those arrays and no K0 launch.
 * Results and errors are identical to the plain path (NALAR_STREAM_STEP=0
 * disables it).  The caller must not modify those arrays until the call returns. */
int nalar_step(nalar_ctx* ctx, const nalar_snapshot* snap, int policy, nalar_decisions* out, int64_t* err_row);

/* Diagnostics: 1 if the last nalar_step on ctx was streamed (see above), else 0. */
int nalar_debug_last_step_streamed(const nalar_ctx* ctx);

/* Copy decisions to caller host buffers; synchronises the ctx stream. */
int nalar_fetch_decisions(nalar_ctx* ctx, nalar_decisions* out);

/* Counters (and kernel times with NALAR_F_TIMING) of the last epoch; syncs. */
int nalar_epoch_stats_get(nalar_ctx* ctx, nalar_epoch_stats* stats);

/* Diagnostics (NALAR_F_PROFILE): copy the last epoch's K1 timeline to host:
 * words [0, 2W): start/end ns of each workflow's sweep; then per K1 block b
 * 8 words: staged, swept, bucketed, entered, finished, fenced, prepped, dependency-waited; then per resource r 8 words of
 * K4: start, admitted count known, slot tables built, done, sweep complete, walk prefix, first
 * live compaction, 0; then per workflow 4 words:
 * SM cycles in the sweep's edge loop / settling rounds / the rest, and the
 * settling-round count (bits 0-15) with steps by slot width (12 bits each)
 * (for a long workflow: its cycles spent waiting on transfers, bits 32-63);
 * then per K1 block 8 words of summed transfer-step cycles (edges, interface,
 * settling, stores), settling iterations, steps, sum K, sum k.
 * *n_words = 2W + 8B + 8R + 4W + 8B. */
int nalar_debug_profile(nalar_ctx* ctx, uint64_t* host, size_t cap_words, size_t* n_words);

/* Diagnostics: the K1 block table of the uploaded table -- block b sweeps
 * workflows [blk_wf[b], blk_wf[b + 1]); *n_words = B + 1.  NALAR_E_SIZE if
 * cap_words is smaller (then *n_words says how many). */
int nalar_debug_blocks(nalar_ctx* ctx, uint32_t* blk_wf, size_t cap_words, size_t* n_words);

/* Device stream the ctx runs on (cudaStream_t). */
void* nalar_stream(nalar_ctx* ctx);

/* ctx == NULL: why the calling thread's last nalar_create failed. */
const char* nalar_last_error(const nalar_ctx* ctx);
int nalar_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NALAR_H */
