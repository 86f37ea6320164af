// internal.h -- device-side parameter blocks and launch declarations shared by
// the host context (nalar_ctx.cu) and the kernels (k_*.cu) of libnalar.so.
// Nothing here is part of the C ABI (see include/nalar.h).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define NALAR_MAX_INSTANCES_DEV 1024

namespace nalar {

constexpr int kK0Threads = 256;          // validate: warp per workflow
constexpr int kK1Threads = 512;          // sweep: warp per workflow inside a block
constexpr int kK1Warps = kK1Threads / 32;
constexpr int kP5Chunks = 4;             // K1 P5 buckets up to this many 512-row chunks in one pass
constexpr uint32_t kLongSteps = 6;      // workflows of >= 6 steps use the transfer decomposition
// the threshold in rows (kLongSteps steps; NALAR_LONG_STEPS to experiment)
// rows from which a workflow is composed from step transfers.  A one-wave
// table (latency-bound: C4) uses kLongSteps; a table of several waves
// (throughput-bound: a transfer costs ~2.3x an ordinary step) kLongStepsWaves
// -- measured at C5: 6 / 10 / 16 / 24 steps -> 145 / 140 / 141 / 146 us.
// NALAR_LONG_STEPS overrides both.
constexpr uint32_t kLongStepsWaves = 10;
inline uint32_t long_rows(bool waves = false) {
    static const int env = [] {
        const char* e = getenv("NALAR_LONG_STEPS");
        return e ? atoi(e) : 0;
    }();
    const int s = env > 0 ? env : (int)(waves ? kLongStepsWaves : kLongSteps);
    return 32u * (uint32_t)(s > 1 ? s : 1);
}
constexpr uint32_t kMaxIface = 7;       // interface rows per step in a transfer
constexpr int kK4Threads = 256;          // assign: one block per resource
constexpr int kK4Warps = kK4Threads / 32;

// per-row flags produced by the sweep
enum : uint8_t { FL_DOOMED = 1, FL_READY = 2, FL_ELIG = 4, FL_ALLRES = 8, FL_MIG = 16 };

// indices into the per-epoch counters array (scratch)
enum { C_READY = 0, C_ELIG = 1, C_DOOMED = 2, C_ASSIGNED = 3, C_RA_TICKET = 4, C_RA_PAIRS = 5, C_MIGRATED = 6,
       C_BATCHES = 7, C_STAGED = 8, C_NUM = 9 };

// per-type statistics of resource reassignment (NEXT-2), written by K4's type
// blocks; the last K4 block pairs hot with cold types
struct TypeStat {
    unsigned long long busy;    // sum(load) + eligible futures of the type (= load + assigned + deferred)
    unsigned long long cap;     // sum of capacities
    uint32_t n_inst;
    int32_t kill;               // least (load + assigned) instance, ties the highest id; -1 none
};

// bytes of K1 shared memory that do not scale with the block's rows
size_t k1_fixed_smem(uint32_t n_types, uint32_t n_inst, uint32_t R);
// bytes of K1 shared memory that scale with a block's workflows (and, when
// staged, with its rows / edges)
// (inline: the host partition evaluates it once per workflow per cut)
__host__ __device__ inline size_t k1_align16(size_t x) { return (x + 15) & ~(size_t)15; }
// an upper bound of k1_block_smem(.., staged = true) without the per-array
// 16-B rounding (each of its 26 terms rounds up by < 16 B): the partition's
// cheap first test
inline size_t k1_block_smem_upper(uint32_t rows, uint32_t edges, uint32_t wfs, uint32_t T) {
    const size_t w = wfs, r = rows;
    return w * (8 * (size_t)T + 8) + 4 * w + 4 * (w + 1) + 4 * w + 32 * w + 8 * w * T + 8 * w * T + 8 * w +
           3 * (r + 32) + 2 * (2 * r + 32) + (4 * (r + 1) + 32) + (4 * (size_t)edges + 32) + (4 * (w + 1) + 32) +
           (4 * w + 32) + 2 * r + 2 * r + 4 * 4 * r + 2 * r + 26 * 16;
}
inline size_t k1_block_smem(uint32_t rows, uint32_t edges, uint32_t wfs, uint32_t T, bool staged) {
    auto align16 = k1_align16;

    size_t b = align16((size_t)wfs * (8 * (size_t)T + 8)) + align16(4 * (size_t)wfs) +
               align16(4 * ((size_t)wfs + 1)) + align16(4 * (size_t)wfs) +
               align16(32 * (size_t)wfs) + align16(8 * (size_t)wfs * T) +
               align16(8 * (size_t)wfs * T) + align16(8 * (size_t)wfs);                 // per-workflow tables
    if (staged)
        b += 3 * align16(rows + 32) + 2 * align16(2 * (size_t)rows + 32) + align16(4 * ((size_t)rows + 1) + 32) +
             align16(4 * (size_t)edges + 32) + align16(4 * ((size_t)wfs + 1) + 32) + align16(4 * (size_t)wfs + 32) +
             align16(2 * (size_t)rows) + 2 * align16(rows) +
             4 * align16(4 * (size_t)rows) + align16(2 * (size_t)rows);                // step transfers
    return b;
}



struct ValidateParams {
    const uint32_t* wf_fut_off;
    const uint8_t* f_state;
    const uint8_t* f_type;
    const int16_t* f_exec;
    const int16_t* f_pin;
    const uint32_t* f_edge_off;
    const uint32_t* edges;
    const uint8_t* i_type;
    uint32_t n_wf, n_fut, n_edges, n_types, n_inst;
    unsigned long long* err;   // [0] = min bad row (init ~0), [1] = structural flag (device)
    uint32_t* done;            // block-completion counter (0 between launches)
    unsigned long long* host_err;   // mapped host words: the last block publishes err here and re-arms it
    // after a delta: the delta's update errors (device words, ~0 = none) are
    // published to host_err[2], [3] and re-armed by the same last block
    unsigned long long* delta_err;
    unsigned long long* verdict;    // device word: 1 if the table is invalid (the epoch kernels skip)
};

// Streamed step (nalar_step with pinned snapshot arrays): K1 stages its rows
// by TMA straight from the caller's mapped host memory, checks K0's contract
// on them in shared memory, and writes them back to the device table.
struct StreamIn {
    const uint8_t* state;       // device views of the caller's pinned arrays
    const uint8_t* type;
    const uint8_t* round;
    const int16_t* pin;
    const int16_t* exec;
    const uint32_t* eoff;
    const uint32_t* edges;
    unsigned long long* err;    // [0] min bad row (~0 armed), [1] structural flag (0 armed)
    unsigned long long* verdict;   // set to 1 by a block holding an invalid row
    const uint8_t* i_type;
    uint32_t n_edges, n_types, n_inst;
};

struct SweepParams {
    const unsigned long long* verdict;   // K0's verdict: nonzero = invalid table, do nothing
    uint32_t stream_in;          // 1: rows come from `src` (host), validated here (verdict unused at entry)
    StreamIn src;
    // CTA i sweeps block blk_order[8 i] (costliest first); words 8 i + 1..7
    // are that block's first / end workflow, row and edge and its staged
    // flag, so a CTA starts with one round trip of independent loads (not a
    // chain through the block tables).  A streamed step paces
    // its host reads: CTA i >= stage_window issues its copies once
    // stage_ctr >= i - stage_window CTAs have staged (bounded wait), so the
    // costly blocks' rows cross PCIe first and their sweeps overlap the rest.
    const uint32_t* blk_order;
    uint32_t* stage_ctr;
    uint32_t stage_window;
    // nalar_step with pinned outputs: the per-row outputs also go straight to
    // the caller's mapped host arrays as they are produced (null: not wanted)
    uint8_t* o_status;
    uint8_t* o_level;
    uint16_t* o_depth;
    int16_t* o_instance;
    uint8_t* o_new_pin;
    uint32_t* rb_mine;           // world > 1: this rank's (global_row_base, rows) words of the exchange
    uint32_t row_base, n_rows;
    uint32_t long_rows;          // workflows of >= long_rows rows are composed from step transfers
    uint32_t pdl;                // launched as a programmatic dependent of the zero kernel
    uint32_t trig;               // where K1 lets its dependent launch: 0 entry, 1 after P2, 2 before P5
    const uint32_t* wf_fut_off;
    const int32_t* wf_prio;
    const uint8_t* f_state;
    const uint8_t* f_type;
    const uint8_t* f_round;
    const int16_t* f_exec;
    const int16_t* f_pin;
    const uint32_t* f_edge_off;
    const uint32_t* edges;
    const uint8_t* t_aff;
    const uint32_t* blk_wf;     // [B+1] workflow range of each block
    const uint32_t* blk_row0;   // [B+1] first row of each block
    const uint32_t* blk_edge0;  // [B+1] first edge of each block
    const uint8_t* blk_staged;  // [B]   1 = rows staged in shared memory by TMA
    const uint32_t* wf_perm;    // [W]   per block: local workflow indices, largest first (task order)
    uint32_t B, n_types, n_inst, R, levels, policy;
    uint32_t Rh;                // R + T: bucket / histogram resources (the last T: HoL candidates, NEXT-1)
    // HoL migration candidates (NEXT-1), active when mig_on
    uint32_t mig_on, theta_wait, theta_head;
    const uint32_t* f_age;      // [N]
    const uint32_t* i_head_rem; // [I]
    int16_t* migrate_to;        // [N] out (-1 here; K5 writes the moves)
    int32_t* batch_head;        // [N] out when batching is on (-1 here; K6 writes the batches)
    uint32_t fixed_smem;        // bytes of fixed smem (carve offset of staged area)
    uint8_t* g_flags;           // [N] flags scratch for unstaged blocks
    uint32_t *g_tlo, *g_thi, *g_ifc, *g_ndp;   // [N] step-transfer scratch for unstaged blocks
    uint16_t* g_aux;
    unsigned long long* prof;   // NALAR_F_PROFILE: [W][2] workflow start/end, [B][4] block phases
    uint32_t n_wf;
    // outputs
    uint8_t* status;
    uint8_t* level;
    uint16_t* depth;
    int16_t* instance;
    uint8_t* new_pin;
    uint32_t* wf_agg;           // [W][10]
    uint8_t* kv_hint;           // [W][T] K,V retention hint (NEXT-3): 0 none, 1 retain, 2 offload, 3 drop
    uint8_t* kv_level;          // [W][T] retention urgency: max level of the session's live futures
    int16_t* kv_home;           // [W][T] the session's home instance, or -1
    uint32_t* H;                // this rank's histogram slot [R][Lv]
    uint32_t* load_part;        // [I] in-flight counts of this rank's rows
    uint32_t* tot;              // [R] eligible futures per resource (this rank; summed by the allreduce)
    uint32_t* tot_loc;          // [R] the same, never reduced (assignment-list regions)
    uint2* items;               // [N] eligible (row, level), per-block regions
    uint32_t* cnt_rb;           // [R][B]
    uint32_t* off_rb;           // [R][B]
    uint32_t* counters;         // C_*
};

struct AssignParams {
    const unsigned long long* verdict;   // K0's verdict (see SweepParams)
    // streamed step: the verdict is K1's, read after the grid dependency;
    // block 0 then publishes the error words to mapped host memory and re-arms them
    uint32_t stream_in;
    unsigned long long* err;             // [0] min bad row, [1] structural (device)
    unsigned long long* host_err;        // mapped host words [0], [1]
    uint8_t* o_status;                   // streamed outputs (see SweepParams), admitted rows
    int16_t* o_instance;
    uint8_t* o_new_pin;
    const uint32_t* rb;                  // world > 1: every rank's (global_row_base, rows)
    unsigned long long* order_err;       // mapped host word: set when the ranks' row ranges are out of order
    const uint32_t* H;          // [G][R][Lv] summed over ranks
    const uint32_t* load_sum;   // [I] summed over ranks
    const uint32_t* tot;        // [R] eligible futures per resource, summed over ranks
    const uint32_t* type_off;   // [T+1] instances of type t: type_inst[type_off[t] ..]
    const uint32_t* type_inst;  // [I]   instance ids grouped by type, ascending
    uint32_t G, slot, R, n_inst, n_types, levels, B;
    uint32_t Rh;                // histogram row stride (R + T)
    const uint8_t* i_type;
    const uint32_t* i_cap;
    const uint32_t* i_base;
    const uint8_t* t_aff;
    const uint32_t* cnt_rb;
    const uint32_t* off_rb;
    const uint32_t* blk_row0;
    const uint2* items;
    // outputs
    uint8_t* status;
    int16_t* instance;
    uint8_t* new_pin;
    uint32_t* i_load;
    uint32_t* i_spare;
    uint32_t* i_assigned;
    uint32_t* assign_row;
    int16_t* assign_inst;
    const uint32_t* tot_loc;    // [R] this rank's eligible futures per resource
    uint32_t* n_adm;            // [R] this rank's admitted futures per resource
    uint32_t* counters;
    unsigned long long* prof;   // NALAR_F_PROFILE: [R][4] start, bounded, based, done
    // resource reassignment (NEXT-2), active when ra_on
    uint32_t ra_on, u_hi_pct, u_lo_pct;
    const uint16_t* t_min_inst; // [T]
    const uint16_t* t_max_inst; // [T]
    TypeStat* tstat;            // [T] scratch
    uint32_t* t_busy;           // [T] out (saturated u32)
    uint32_t* t_capsum;         // [T] out
    int16_t* ra_kill;           // [T] out: pair k's instance to kill
    int16_t* ra_prov;           // [T] out: pair k's type to provision
};

struct RebuildPlan {             // one workflow of the table after a delta
    uint64_t wf_id;
    uint32_t src;                // its index in the old table, or ~0 (new workflow)
    uint32_t n_old, n_old_edges; // rows / edges kept from the old table
    uint32_t app_lo, app_n;      // appended futures [app_lo, app_lo + app_n)
    uint32_t new_row0, new_edge0;
    int32_t prio;                // for new workflows
    uint32_t pad;
};

struct DeltaParams {
    // old (current) table, updated in place by KD1 / KD2
    uint32_t* wf_off; int32_t* wf_prio; uint64_t* wf_id;
    uint8_t* state; uint8_t* type; uint8_t* round; int16_t* exec; int16_t* pin;
    uint32_t* eoff; uint32_t* edges;
    uint32_t n_wf;
    // last epoch's assignment regions (KD1)
    const uint32_t* tot_loc; const uint32_t* n_adm; const uint32_t* arow; const int16_t* ainst;
    // updates (KD2)
    uint32_t n_upd;
    const uint64_t* upd_wf_id; const uint32_t* upd_seq; const uint8_t* upd_state;
    const int16_t* upd_exec; const int16_t* upd_pin;
    // rebuild (KD3) into the other buffer set
    uint32_t n_wf_new;
    const RebuildPlan* plan;
    uint32_t* n_wf_off; int32_t* n_wf_prio; uint64_t* n_wf_id;
    uint8_t* n_state; uint8_t* n_type; uint8_t* n_round; int16_t* n_exec; int16_t* n_pin;
    uint32_t* n_eoff; uint32_t* n_edges;
    const uint8_t* app_state; const uint8_t* app_type; const uint8_t* app_round;
    const int16_t* app_exec; const int16_t* app_pin; const uint32_t* app_eoff; const uint32_t* app_edges;
    // KD4
    uint32_t n_prio; const uint64_t* prio_wf_id; const int32_t* prio_value;
    uint32_t n_inst_upd, n_inst; const uint32_t* inst_id; const uint32_t* inst_cap; const uint32_t* inst_base;
    uint32_t* i_cap; uint32_t* i_base;
    unsigned long long* err;     // [0] bad update index, [1] bad prio / instance update index
    uint32_t n_fut_new, n_edges_new;   // tails of the new offset arrays (written by KD3)
};

// host <-> device segment copies (k_io.cu): src / dst are device-accessible
// pointers (device memory or mapped pinned host memory)
constexpr int kMaxSegs = 24;
struct CopySeg {
    const void* src;
    void* dst;
    uint64_t bytes;
};
struct CopyParams {
    CopySeg seg[kMaxSegs];
    uint64_t chunk_off[kMaxSegs + 1];   // prefix of 16-byte chunk counts
    uint32_t n;
};
struct FetchParams {
    const uint32_t* n_adm;      // [R] this rank's admitted futures per resource
    const uint32_t* tot_loc;    // [R] region sizes of the device assignment list
    const uint32_t* arow;
    const int16_t* ainst;
    const uint32_t* counters;   // C_*
    uint32_t* out_row;          // mapped host (or null)
    int16_t* out_inst;
    uint32_t* out_counters;     // mapped host [C_NUM]
    uint32_t R, a_cap;
};

// K5 HoL migration (NEXT-1, k_migrate.cu); G == 1
constexpr uint32_t kK5MaxInst = 256;    // instances per type the migration pass supports
// World > 1 with HoL migration (NEXT-1) or batch coalescing (NEXT-4) on: the
// lists these passes need from every rank travel in the ONE exchange of the
// epoch, as a region of kListWords per rank after the (row base, rows) pairs.
// Regions of other ranks are zero in a rank's own buffer, so the allreduce
// (sum) is an allgather.
//  [0, kMigWords) migration: word 0 = entries (kListOverflow: too many), words
//    [1, 1 + kMaxTypesDev) = entries per type, then per type in order the
//    rank's candidates in row order, each its bucket item's second word
//    (level | (executor + 1) << 16);
//  [kMigWords, kListWords) batching: word 0 = entries (or kListOverflow),
//    words [1, 1 + R) = entries per resource (batchable ones only), then per
//    resource in order the rank's eligible futures in row order, two words
//    each: level | method << 8, global row.
constexpr uint32_t kListWords = 16384;
constexpr uint32_t kMigWords = 8192;
constexpr uint32_t kMaxTypesDev = 64;
constexpr uint32_t kListHdr = 1 + kMaxTypesDev;
constexpr uint32_t kListOverflow = 0xFFFFFFFFu;

struct ListParams {
    uint32_t mig, batch;        // which sections to write
    const uint8_t* i_type;      // batching: which resources are batchable
    const uint16_t* t_max_batch;
    const uint8_t* f_method;    // [N] or null (method 0)
    const uint8_t* level;       // [N] (K1's levels)
    uint32_t row_base;          // this rank's global row base
    const uint32_t* tot_loc;    // [Rh] this rank's bucket totals
    const uint32_t* cnt_rb;     // [Rh][B]
    const uint32_t* off_rb;
    const uint32_t* blk_row0;
    const uint2* items;
    uint32_t* list;             // this rank's list region (kListWords)
    uint32_t* mrow;             // [kListWords] this rank's row of each list entry
    uint32_t R, B, n_types, n_inst;
};
cudaError_t launch_lists(const ListParams& p, cudaStream_t s);

struct MigrateParams {
    const unsigned long long* verdict;
    // world > 1: every rank's list region ([G][kListWords]) and this rank's rows
    const uint32_t* lists;
    const uint32_t* mrow;
    uint32_t G, rank;
    unsigned long long* list_err;      // mapped host word: a rank's list overflowed
    const uint32_t* H;          // [Rh][Lv] (this rank's slot == the sum when G == 1)
    const uint32_t* tot;        // [Rh]
    const uint32_t* cnt_rb;     // [Rh][B]
    const uint32_t* off_rb;
    const uint32_t* blk_row0;
    const uint2* items;
    const uint32_t* type_off;
    const uint32_t* type_inst;
    const uint32_t* i_load;     // after K4
    const uint32_t* i_assigned;
    const uint32_t* i_head_rem;
    uint32_t R, Rh, B, n_inst, n_types, levels, theta_head, delta;
    int16_t* migrate_to;
    uint32_t* i_mig_in;
    uint32_t* i_mig_out;
    uint32_t* counters;
};
cudaError_t launch_migrate(const MigrateParams& p, cudaStream_t s);

// K6 batch coalescing (NEXT-4, k_batch.cu); G == 1
struct BatchParams {
    const unsigned long long* verdict;
    uint32_t row_base;             // batch_head holds global rows (row_base + row)
    // world > 1 (K6 over every rank's lists, k_batch.cu k6_batch_ranks)
    uint32_t G, n_rows, R, levels, Rh;
    const uint32_t* lists;         // [G][kListWords]
    const uint32_t* H;             // [G][Rh][Lv] exchange
    const uint32_t* tot;           // [Rh] global eligible per resource
    const uint32_t* i_spare;       // [I] global (K4)
    const uint32_t* type_off;
    const uint32_t* type_inst;
    unsigned long long* list_err;  // mapped host word
    const uint8_t* i_type;
    const uint16_t* t_max_batch;   // [T]
    const uint8_t* f_method;       // [N] or null
    const uint8_t* level;          // [N]
    const uint32_t* n_adm;         // [R] admitted per resource
    const uint32_t* tot_loc;       // [R] region sizes
    const uint32_t* arow;
    const int16_t* ainst;
    uint32_t n_inst;
    int32_t* batch_head;           // [N] out (-1 preset by K1)
    uint32_t* counters;
};
cudaError_t launch_batch(const BatchParams& p, cudaStream_t s);

// rank exchange over peer memory (k_peer.cu)
constexpr uint32_t kPeerMaxRanks = 8;
constexpr uint32_t kPeerFlagWords = 64;                       // flag[2][kPeerMaxRanks], padded
constexpr unsigned long long kPeerTimeoutNs = 5000000000ull;  // a missing peer: error, not a hang
constexpr uint32_t kPeerPoison = 0xFFFFFFFFu;   // flag value of a rank whose exchange failed
constexpr uint32_t kPeerLocalWords = 8;         // epoch, push ctr, gather ctr, wait ok, sticky failed
struct PeerParams {
    uint32_t* peers[kPeerMaxRanks];   // every rank's receive buffer (own included)
    uint32_t lw;                      // list words per rank (kListWords when lists travel, else 0)
    const uint32_t* list_mine;        // this rank's list region
    const uint32_t* slot;             // this rank's H slot [Rh*Lv]
    const uint32_t* load;             // this rank's partial load [I]
    const uint32_t* tot;              // this rank's partial totals [Rh]
    const uint32_t* rb_mine;          // this rank's (global_row_base, rows)
    uint32_t* x;                      // K4's exchange buffer: H[G][Rh*Lv] | load[I] | tot[Rh]
    unsigned long long* err;          // mapped host word: set on a timed-out wait
    size_t par_words;                 // words per parity region (reservation sized)
    uint32_t G, rank, rh_lv, I, Rh;
};
inline size_t peer_par_words(uint32_t G, size_t Rhmax, uint32_t Lv, size_t Imax) {
    return (size_t)G * (Rhmax * Lv + Imax + Rhmax + 2 + kListWords);
}
inline size_t peer_buffer_bytes(uint32_t G, size_t Rhmax, uint32_t Lv, size_t Imax) {
    return 4 * (kPeerFlagWords + 2 * peer_par_words(G, Rhmax, Lv, Imax) + kPeerLocalWords);
}
cudaError_t launch_peer_exchange(const PeerParams& p, cudaStream_t s);

cudaError_t launch_copy_segs(const CopyParams& p, cudaStream_t s);
cudaError_t launch_fetch(const FetchParams& f, const CopyParams& p, cudaStream_t s);
cudaError_t launch_validate(const ValidateParams& p, cudaStream_t s);
cudaError_t launch_delta(const DeltaParams& p, bool apply_assigned, uint32_t R, cudaStream_t s);
cudaError_t launch_zero(uint32_t* x, size_t n_words, cudaStream_t s, unsigned long long* verdict = nullptr);
cudaError_t launch_sweep(const SweepParams& p, size_t smem, cudaStream_t s);
cudaError_t launch_assign(const AssignParams& p, cudaStream_t s);

// eager loading of every kernel (one per source file)
cudaError_t preload_k_assign();
cudaError_t preload_k_batch();
cudaError_t preload_k_delta();
cudaError_t preload_k_io();
cudaError_t preload_k_migrate();
cudaError_t preload_k_peer();
cudaError_t preload_k_sweep();

cudaError_t preload_k_validate();

}  // namespace nalar
