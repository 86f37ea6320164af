/* nalar_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, single-threaded CPU oracle of the Nalar policy epoch
 * (arXiv 2601.05109).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant with the CUDA library (include/nalar.h); the two
 * meet only at the input data format defined in nalar_gen/snapshot.py.
 */
#ifndef NALAR_ORACLE_H
#define NALAR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t n_futures, n_edges, n_workflows, n_instances, n_types, levels;
    const uint64_t* wf_id;      /* [W]   */
    const uint32_t* wf_fut_off; /* [W+1] */
    const int32_t*  wf_prio;    /* [W]   */
    const uint8_t*  f_state;    /* [N]   */
    const uint8_t*  f_type;
    const uint8_t*  f_round;
    const int16_t*  f_executor;
    const int16_t*  f_pin;
    const uint32_t* f_edge_off; /* [N+1] */
    const uint32_t* edges;      /* [E]   */
    const uint8_t*  i_type;     /* [I]   */
    const uint32_t* i_cap;
    const uint32_t* i_base_load;
    const uint8_t*  t_affinity; /* [T]   */
} oracle_table;

typedef struct {
    uint8_t*  status;     /* [N] */
    uint8_t*  level;      /* [N] */
    uint16_t* depth;      /* [N] */
    int16_t*  instance;   /* [N] */
    uint8_t*  new_pin;    /* [N] */
    uint32_t* wf_agg;     /* [W*10] */
    uint32_t* i_load;     /* [I] */
    uint32_t* i_spare;    /* [I] spare before admission */
    uint32_t* i_assigned; /* [I] */
    uint32_t* assign_row; /* [N] capacity; (resource, global rank) order */
    int16_t*  assign_inst;/* [N] */
    uint8_t*  kv_hint;    /* [W*T] O9: 0 none, 1 retain, 2 offload, 3 drop (SESSION types) */
    uint8_t*  kv_level;   /* [W*T] O9: max level of the session's live futures */
    int16_t*  kv_home;    /* [W*T] O9: the session's home instance, or -1 */
    uint32_t  n_assigned; /* out */
    uint32_t  n_ready, n_eligible, n_doomed; /* out */
} oracle_out;

/* O10 resource reassignment parameters (NEXT-2): per-type directives
 * min_instances / max_instances (Table 1) and the
 * utilisation thresholds in percent (SPEC S:452 defaults u_hi 80, u_lo 30). */
typedef struct {
    const uint16_t* t_min_inst; /* [T] */
    const uint16_t* t_max_inst; /* [T] */
    uint32_t u_hi_pct, u_lo_pct;
} oracle_ra_params;

typedef struct {
    uint32_t* t_busy;     /* [T] sum(load + assigned) over the type's instances + its DEFERRED futures */
    uint32_t* t_cap;      /* [T] sum of the type's capacities */
    int16_t*  kill_inst;  /* [T] pair k: the instance to kill */
    int16_t*  prov_type;  /* [T] pair k: the type to provision */
    uint32_t  n_pairs;    /* out */
} oracle_ra_out;

/* O11 head-of-line-blocking migration (NEXT-1): per QUEUED future its wait
 * age, per instance the predicted remaining time of its head job (same unit),
 * thresholds theta_wait / theta_head and the anti-thrash margin delta (SPEC
 * S:441 and its defaults). */
typedef struct {
    const uint32_t* f_age;       /* [N] */
    const uint32_t* i_head_rem;  /* [I] */
    uint32_t theta_wait, theta_head, delta;
} oracle_mig_params;

typedef struct {
    int16_t*  migrate_to;  /* [N] destination instance, -1 none */
    uint32_t* i_mig_in;    /* [I] */
    uint32_t* i_mig_out;   /* [I] */
    uint32_t  n_migrated;  /* out */
} oracle_mig_out;

int oracle_migrate(const oracle_table* t, const oracle_out* o, const oracle_mig_params* p, oracle_mig_out* r);

/* O12 batch coalescing (NEXT-4): per type max_batch (the `batchable`
 * directive; <= 1 = not batchable), per future its method (the
 * batch compatibility key with the agent type; NULL = 0). */
typedef struct {
    const uint16_t* t_max_batch; /* [T] */
    const uint8_t*  f_method;    /* [N] or NULL */
} oracle_batch_params;

typedef struct {
    int32_t*  batch_head;  /* [N] row of the first future of f's batch, -1 none */
    uint32_t  n_batches;   /* out */
} oracle_batch_out;

/* -1 when a batchable type is not of affinity NONE. */
int oracle_batch(const oracle_table* t, const oracle_out* o, const oracle_batch_params* p, oracle_batch_out* r);

/* O10 from a finished epoch (o from oracle_epoch on the same table). */
int oracle_reassign(const oracle_table* t, const oracle_out* o, const oracle_ra_params* p, oracle_ra_out* r);

/* 0 = valid, -1 = invalid; *err_row = smallest offending future row, or -1
 * when the violation is not attributable to a row. */
int oracle_validate(const oracle_table* t, int64_t* err_row);

/* policy: 0 FCFS, 1 SRTF, 2 LPT.  Returns 0, or -1 on an invalid table. */
int oracle_epoch(const oracle_table* t, int policy, oracle_out* o);

/* bench.py's cpu_baseline: `reps` timed runs of oracle_epoch, ns per run. */
int oracle_epoch_timed(const oracle_table* t, int policy, oracle_out* o, int reps, uint64_t* ns);

#ifdef __cplusplus
}
#endif
#endif
