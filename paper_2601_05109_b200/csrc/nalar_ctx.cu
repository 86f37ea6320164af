// nalar_ctx.cu -- host side of libnalar.so: the C ABI of include/nalar.h.
//
// Owns device memory (one arena), the stream, the per-policy CUDA graph of the
// epoch (memset -> K1 sweep -> [NCCL allreduce] -> K4 assign) and, in
// NALAR_COLL_NCCL mode, a library-owned NCCL communicator (NCCL is dlopen'ed,
// so the library loads on machines without it).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/nalar.h"
#include "internal.h"

using namespace nalar;

namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    bool load(std::string* err) {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) { *err = std::string("dlopen libnccl failed: ") + dlerror(); return false; }
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        commInitAll = (decltype(commInitAll))dlsym(h, "ncclCommInitAll");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
        if (!getUniqueId || !commInitRank || !commInitAll || !allReduce || !commDestroy || !getErrorString) {
            *err = "libnccl: missing symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
thread_local std::string g_create_err;   // nalar_last_error(NULL) after a failed nalar_create

constexpr uint32_t kSmSplit = 148;              // B200 SMs: K1 grid target
constexpr double kLongWeight = 1.75;            // cost per row of a long workflow (partition)
// K1 blocks of one wave (NALAR_K1_BLOCKS): a few SMs stay free for the
// early-launched (PDL) K4 blocks; measured at C4 (round 1): 148 blocks 48.5 us
// / epoch, 145 46.1, 142 45.8, 138 48.8; re-measured after the round-2 K1
// changes over four C4 seeds (scripts/part_sweep.py): 142 37.6-37.9 us, 143
// 37.4, 144 36.9-37.4, 145 37.1, 147 37.6, 148 37.4
constexpr uint32_t kK1Wave = 144;
constexpr uint32_t kDeepAlone = 20;      // steps: a workflow this deep gets its own K1 block
constexpr uint32_t kDeepAloneMax = 16;   // ... while there are at most this many
constexpr size_t kStageBudget = 96 * 1024;      // max staged smem per K1 block
constexpr uint32_t kMaxBlocks = 16384;
constexpr uint32_t kMaxWfPerBlock = 4096;    // bounds the per-workflow smem tables

// Everything enqueue_epoch bakes into a captured graph or checks on the host:
// the shape, policy and parameters, the buffer set, and the per-upload inputs
// that change which kernels run or what they read (HoL inputs present, methods
// present, the type affinities the batch / migration checks depend on).
struct Key {
    uint32_t N, E, W, I, T, B, R, policy, params_gen;
    size_t smem;
    const void* table;   // current buffer set (deltas swap sets)
    uint32_t upload_flags;   // bit 0 have_mig, bit 1 have_method
    uint64_t taff_hash;      // FNV-1a of the uploaded type affinities
    uint32_t max_inst_per_type;
    uint64_t stream_key = 0;  // streamed step: hash of the caller's array addresses (0 otherwise)
    bool operator==(const Key& o) const {
        return N == o.N && E == o.E && W == o.W && I == o.I && T == o.T && B == o.B && R == o.R &&
               policy == o.policy && params_gen == o.params_gen && smem == o.smem && table == o.table &&
               upload_flags == o.upload_flags && taff_hash == o.taff_hash &&
               max_inst_per_type == o.max_inst_per_type && stream_key == o.stream_key;
    }
};

}  // namespace

struct nalar_ctx {
    nalar_config cfg{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint8_t* arena = nullptr;
    bool own_arena = false;
    size_t arena_bytes = 0;
    uint32_t Lv = 256, Rmax = 0, Rhmax = 0, Bmax = 0, Rh = 0;
    // inputs
    uint32_t *d_wf_off = nullptr, *d_eoff = nullptr, *d_edges = nullptr, *d_icap = nullptr, *d_ibase = nullptr;
    int32_t* d_wf_prio = nullptr;
    uint8_t *d_state = nullptr, *d_type = nullptr, *d_round = nullptr, *d_itype = nullptr, *d_taff = nullptr;
    int16_t *d_exec = nullptr, *d_pin = nullptr;
    uint32_t *d_blk_wf = nullptr, *d_blk_row0 = nullptr, *d_blk_edge0 = nullptr;
    uint8_t* d_blk_staged = nullptr;
    uint32_t* d_blk_order = nullptr;
    uint32_t* d_wf_perm = nullptr;
    uint32_t *d_type_off = nullptr, *d_type_inst = nullptr;
    // outputs
    uint8_t *d_status = nullptr, *d_level = nullptr, *d_newpin = nullptr, *d_gflags = nullptr;
    uint16_t* d_gwlm = nullptr;
    uint32_t *d_gtlo = nullptr, *d_gthi = nullptr, *d_gifc = nullptr, *d_gndp = nullptr;
    uint16_t* d_gaux = nullptr;
    uint16_t* d_depth = nullptr;
    int16_t *d_inst = nullptr, *d_ainst = nullptr;
    // resource reassignment (NEXT-2)
    uint16_t *d_tmin = nullptr, *d_tmax = nullptr;
    TypeStat* d_tstat = nullptr;
    uint32_t *d_tbusy = nullptr, *d_tcap = nullptr;
    int16_t *d_rakill = nullptr, *d_raprov = nullptr;
    uint32_t ra_on = 0, u_hi = 80, u_lo = 30, params_gen = 0;
    // HoL migration (NEXT-1)
    uint32_t* d_age = nullptr;
    uint32_t* d_head = nullptr;
    int16_t* d_migto = nullptr;
    uint32_t *d_migin = nullptr, *d_migout = nullptr;
    uint32_t mig_on = 0, theta_wait = 0, theta_head = 0, mig_delta = 2, max_inst_per_type = 0;
    bool have_mig = false;
    // batch coalescing (NEXT-4)
    uint16_t* d_tmaxb = nullptr;
    uint8_t* d_method = nullptr;
    int32_t* d_bhead = nullptr;
    bool batch_on = false, have_method = false;
    std::vector<uint16_t> h_tmaxb;
    std::vector<uint8_t> h_taff;      // affinities of the uploaded table
    bool mig_active() const { return mig_on && have_mig; }
    bool mig_active_for(const nalar_snapshot* s) const { return mig_on && s->f_age && s->i_head_rem; }
    uint8_t *d_kvh = nullptr, *d_kvl = nullptr;
    int16_t* d_kvhome = nullptr;
    uint32_t *d_wfagg = nullptr, *d_iload = nullptr, *d_ispare = nullptr, *d_iasg = nullptr, *d_arow = nullptr;
    // intermediates
    uint2* d_items = nullptr;
    uint32_t *d_cnt_rb = nullptr, *d_off_rb = nullptr;
    uint32_t* d_x = nullptr;          // exchange: H[G][R][Lv] then load[I]
    uint32_t* d_mrow = nullptr;       // world > 1: this rank's row of each entry of its list region
    size_t x_words = 0;
    uint32_t* d_scr = nullptr;        // counters[C_NUM], n_adm[Rmax], tot_loc[Rmax]; contiguous with d_x
    size_t zero_bytes = 0;            // bytes to clear per epoch from d_x
    unsigned long long* d_err = nullptr;
    // host pinned
    uint32_t* h_cnt = nullptr;
    uint32_t* h_reg = nullptr;         // n_adm[Rmax], tot_loc[Rmax]
    void* h_list = nullptr;
    size_t h_list_cap = 0;
    unsigned long long* h_err = nullptr;
    uint32_t* h_cnt_dev = nullptr;     // device view of h_cnt (mapped)
    // pinned staging of the host-built tables (type lists, K1 block tables,
    // task order) so they travel in the upload's single copy kernel
    uint8_t* h_tab = nullptr;
    uint8_t* h_tab_dev = nullptr;
    size_t tab_off[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // type_off, type_inst, blk_wf, blk_row0, blk_edge0, blk_staged, perm, blk_order
    // current table
    uint32_t N = 0, E = 0, W = 0, I = 0, T = 0, B = 0, R = 0;
    size_t smem = 0, fixed_smem = 0;
    bool uploaded = false, epoch_done = false, in_epoch = false;
    int last_policy = -1;
    // graphs / timing
    cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};
    Key gkey[3]{};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    ncclComm_t comm = nullptr;
    // NALAR_COLL_PEER: this rank's receive buffer and every rank's (k_peer.cu)
    uint32_t* peer_buf = nullptr;
    size_t peer_par_words = 0;
    uint32_t* peers[kPeerMaxRanks] = {};
    void* peer_ipc[kPeerMaxRanks] = {};      // opened IPC mappings (closed on destroy)
    bool peers_ready = false;
    bool peer_failed = false;                     // sticky until the next reconnect
    unsigned long long* peer_err_dev = nullptr;   // device view of h_err[4]
    unsigned long long* h_err_dev = nullptr;      // device view of h_err
    uint64_t row_base = 0;                        // the snapshot's global_row_base
    bool row_base_known = false;
    // delta mode: device workflow ids, the second table buffer set, host mirror
    uint64_t* d_wf_id = nullptr;
    struct Alt {
        uint32_t *wf_off = nullptr, *eoff = nullptr, *edges = nullptr;
        int32_t* wf_prio = nullptr;
        uint64_t* wf_id = nullptr;
        uint8_t *state = nullptr, *type = nullptr, *round = nullptr;
        int16_t *exec = nullptr, *pin = nullptr;
        void* mem = nullptr;
    } alt;
    void* d_stage = nullptr;          // delta staging (device)
    size_t stage_bytes = 0;
    uint8_t* h_dstage = nullptr;      // delta staging (pinned host): one H2D per delta
    size_t h_dstage_bytes = 0;
    std::vector<uint64_t> m_wf_id;
    std::vector<uint32_t> m_wf_off, m_wf_eoff;
    std::vector<uint32_t> m_perm;          // per-block task order (set_blocks)
    std::vector<uint32_t> m_tmp;           // set_blocks scratch
    std::vector<uint64_t> m_spare_id;      // delta: the previous mirror, reused
    std::vector<uint32_t> m_spare_off, m_spare_eoff;
    std::vector<uint8_t> m_retired;
    std::vector<uint32_t> m_cta_rec;       // per-CTA K1 block records (set_blocks)
    std::vector<RebuildPlan> m_plan;       // delta scratch (nalar_delta_apply)
    bool blocks_valid = false;              // device block tables match m_wf_off / m_wf_eoff
    uint32_t blocks_T = 0;
    bool assign_valid = false;        // last epoch's assignment regions match the table
    bool all_staged = false;          // every K1 block stages its rows in shared memory
    uint32_t long_rows = 0;           // compose threshold of the current partition (long_rows())
    // streamed step (nalar_step, pinned snapshot): K1 reads the per-row arrays
    // from the caller's host memory, validates them and writes the device copy
    bool streaming = false;
    bool last_streamed = false;
    StreamIn sin{};
    // nalar_step with pinned per-row outputs: K1 / K4 write them straight to
    // the caller's memory; the step's fetch then skips them
    struct StreamOut {
        uint8_t* status = nullptr; uint8_t* level = nullptr; uint16_t* depth = nullptr;
        int16_t* instance = nullptr; uint8_t* new_pin = nullptr;
    } sout;
    bool sout_on = false;
    Key last_key{};
    bool last_key_set = false;
    unsigned long long* d_prof = nullptr;
    size_t prof_words = 0;
    std::string err;
};

namespace {

int fail(nalar_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) return fail(c, NALAR_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

struct Layout {
    size_t off = 0;
    template <typename T>
    size_t take(size_t n) {
        const size_t o = off;
        off += ((n * sizeof(T) + 64) + 255) & ~(size_t)255;   // +64 B pad: TMA windows may over-read
        return o;
    }
};

struct Plan {
    size_t wf_off, wf_prio, wf_id, state, type, round, exec, pin, eoff, edges, itype, icap, ibase, taff;
    size_t blk_wf, blk_row0, blk_edge0, blk_staged, blk_order, wf_perm, type_off, type_inst;
    size_t status, level, newpin, gflags, gwlm, gtlo, gthi, gifc, gndp, gaux, depth, inst, ainst, wfagg, iload, ispare, iasg, arow;
    size_t kvh, kvl, kvhome, tmin, tmax, tstat, tbusy, tcap, rakill, raprov, age, head, migto, migin, migout;
    size_t tmaxb, method, bhead;
    size_t items, cnt_rb, off_rb, x, scr, err;
    size_t x_words, total, mrow;
    uint32_t Rmax, Rhmax, Bmax;
};

bool plan_layout(const nalar_config* cfg, Plan* p) {
    const uint32_t Lv = cfg->levels ? cfg->levels : 256;
    const size_t N = cfg->max_futures, E = cfg->max_edges, W = cfg->max_workflows;
    const size_t I = cfg->max_instances, T = cfg->max_types;
    const uint32_t G = cfg->world > 0 ? (uint32_t)cfg->world : 1u;
    p->Rmax = (uint32_t)(I + T);
    p->Rhmax = (uint32_t)(I + 2 * T);       // + T HoL-candidate buckets (NEXT-1)
    p->Bmax = (uint32_t)std::min<size_t>(std::max<size_t>(W, 1), kMaxBlocks);
    Layout L;
    p->wf_off = L.take<uint32_t>(W + 1);
    p->wf_prio = L.take<int32_t>(W);
    p->wf_id = L.take<uint64_t>(W);
    p->state = L.take<uint8_t>(N);
    p->type = L.take<uint8_t>(N);
    p->round = L.take<uint8_t>(N);
    p->exec = L.take<int16_t>(N);
    p->pin = L.take<int16_t>(N);
    p->eoff = L.take<uint32_t>(N + 1);
    p->edges = L.take<uint32_t>(E);
    p->itype = L.take<uint8_t>(I);
    p->icap = L.take<uint32_t>(I);
    p->ibase = L.take<uint32_t>(I);
    p->taff = L.take<uint8_t>(T);
    p->blk_wf = L.take<uint32_t>(p->Bmax + 1);
    p->blk_row0 = L.take<uint32_t>(p->Bmax + 1);
    p->blk_edge0 = L.take<uint32_t>(p->Bmax + 1);
    p->blk_staged = L.take<uint8_t>(p->Bmax);
    p->blk_order = L.take<uint32_t>(8 * (size_t)p->Bmax);   // per-CTA block records (SweepParams)
    p->wf_perm = L.take<uint32_t>(W);
    p->type_off = L.take<uint32_t>(T + 1);
    p->type_inst = L.take<uint32_t>(I);
    p->status = L.take<uint8_t>(N);
    p->level = L.take<uint8_t>(N);
    p->newpin = L.take<uint8_t>(N);
    p->gflags = L.take<uint8_t>(N);
    p->gwlm = L.take<uint16_t>(N);
    p->gtlo = L.take<uint32_t>(N);
    p->gthi = L.take<uint32_t>(N);
    p->gifc = L.take<uint32_t>(N);
    p->gndp = L.take<uint32_t>(N);
    p->gaux = L.take<uint16_t>(N);
    p->depth = L.take<uint16_t>(N);
    p->inst = L.take<int16_t>(N);
    p->ainst = L.take<int16_t>(N);
    p->wfagg = L.take<uint32_t>(W * NALAR_WF_AGG_FIELDS);
    p->kvh = L.take<uint8_t>(W * T);
    p->kvl = L.take<uint8_t>(W * T);
    p->kvhome = L.take<int16_t>(W * T);
    p->tmin = L.take<uint16_t>(T);
    p->tmax = L.take<uint16_t>(T);
    p->tstat = L.take<TypeStat>(T);
    p->tbusy = L.take<uint32_t>(T);
    p->tcap = L.take<uint32_t>(T);
    p->rakill = L.take<int16_t>(T);
    p->raprov = L.take<int16_t>(T);
    p->age = L.take<uint32_t>(N);
    p->head = L.take<uint32_t>(I);
    p->migto = L.take<int16_t>(N);
    p->migin = L.take<uint32_t>(I);
    p->migout = L.take<uint32_t>(I);
    p->tmaxb = L.take<uint16_t>(T);
    p->method = L.take<uint8_t>(N);
    p->bhead = L.take<int32_t>(N);
    p->iload = L.take<uint32_t>(I);
    p->ispare = L.take<uint32_t>(I);
    p->iasg = L.take<uint32_t>(I);
    p->arow = L.take<uint32_t>(N);
    p->items = L.take<uint2>(N);
    p->cnt_rb = L.take<uint32_t>((size_t)p->Rhmax * p->Bmax);
    p->off_rb = L.take<uint32_t>((size_t)p->Rhmax * p->Bmax);
    p->x_words = (size_t)G * p->Rhmax * Lv + I + p->Rhmax + 2ull * G    // + (row base, rows) per rank
                 + (G > 1 ? (size_t)G * kListWords : 0);                  // + list regions (NEXT-1)
    p->mrow = L.take<uint32_t>(G > 1 ? kListWords : 1);
    // exchange buffer and scratch are contiguous so one memset clears both
    p->x = L.off;
    L.off += p->x_words * 4;
    p->scr = L.off;
    L.off += (C_NUM + (size_t)p->Rmax + p->Rhmax) * 4;   // counters, n_adm[R], tot_loc[Rh]
    L.off = (L.off + 255) & ~(size_t)255;
    p->err = L.take<unsigned long long>(6);   // [0,1] delta, [2,3] K0, [4] K0 block counter, [5] verdict
    p->total = L.off + 256;
    return true;
}

template <typename T>
T* at(uint8_t* base, size_t off) { return reinterpret_cast<T*>(base + off); }

// Device-accessible address of a host pointer (pinned memory is mapped under
// UVA), or nullptr for pageable memory.
void* mapped_view(const void* h) {
    if (!h) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type == cudaMemoryTypeHost && a.devicePointer) return a.devicePointer;
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return const_cast<void*>(h);
    return nullptr;
}

// A batch of copies issued as one kernel (k_io.cu) when both sides are
// device-accessible; a pageable host side falls back to cudaMemcpyAsync.
struct CopyBatch {
    cudaStream_t st;
    CopyParams p{};
    explicit CopyBatch(cudaStream_t s) : st(s) {}
    cudaError_t add_dev(const void* src, void* dst, size_t bytes) {
        if (!bytes) return cudaSuccess;
        p.seg[p.n++] = CopySeg{src, dst, (uint64_t)bytes};
        return p.n == (uint32_t)kMaxSegs ? flush() : cudaSuccess;
    }
    cudaError_t h2d(void* d, const void* h, size_t bytes) {
        if (!bytes) return cudaSuccess;
        const void* v = mapped_view(h);
        return v ? add_dev(v, d, bytes) : cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    }
    void chunk_offsets() {
        p.chunk_off[0] = 0;
        for (uint32_t i = 0; i < p.n; ++i) p.chunk_off[i + 1] = p.chunk_off[i] + (p.seg[i].bytes + 15) / 16;
    }
    cudaError_t flush() {
        if (!p.n) return cudaSuccess;
        chunk_offsets();
        const cudaError_t e = launch_copy_segs(p, st);
        p.n = 0;
        return e;
    }
};

void destroy_graphs(nalar_ctx* c) {
    for (auto& g : c->gexec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

// The compose threshold of a one-wave table.  A table whose long workflows
// would give its blocks more than one round of step transfers (> 16 per
// block of a full wave on average: the composers then wait for a second
// ~3.5 us round) composes from one more step: C4 by SURVEY 8(d)'s recipe (80 %
// of rows in workflows of >= 6 steps, 24.7 transfers per block) 42.7 -> 40.5 us
// over four seeds at 7 steps (8: 41.0, 10: 43.4); the benched C4 generator
// (9.8 per block) keeps 6 steps (7: +0.4 us).  Used by the partition's cost
// model and the kernel alike.  NALAR_LONG_STEPS fixes the threshold;
// NALAR_LONG_ADAPT=0 disables the rule.
uint32_t one_wave_long_rows(const nalar_ctx* c, const uint32_t* wf_off) {
    static const bool fixed = getenv("NALAR_LONG_STEPS") != nullptr;
    static const bool adapt = [] { const char* e = getenv("NALAR_LONG_ADAPT"); return !e || atoi(e) != 0; }();
    const uint32_t lr = long_rows();
    if (!adapt || fixed) return lr;
    uint64_t steps = 0;
    for (uint32_t w = 0; w < c->W; ++w) {
        const uint32_t r = wf_off[w + 1] - wf_off[w];
        if (r >= lr) steps += (r + 31) / 32;
    }
    return steps > 16ull * kK1Wave ? lr + 32 : lr;
}

// Greedy partition of whole workflows into K1 blocks, balanced by rows.
// wf_off[W+1]: first row of each workflow; wf_eoff[W+1]: first edge of each workflow
void partition(nalar_ctx* c, const uint32_t* wf_off, const uint32_t* wf_eoff, std::vector<uint32_t>& bw,
               std::vector<uint32_t>& br, std::vector<uint32_t>& be, std::vector<uint8_t>& bs, size_t* max_smem,
               bool fill_sms) {
    const uint32_t W = c->W;
    // balance by estimated cost, not rows: a long workflow's rows cost more
    // (a step transfer is ~3x a sweep step, and its compose chain is serial).
    // Weight 1.75 (NALAR_LONG_WEIGHT): C4 epoch over four seeds 41.0 -> 39.9
    // us mean (1.25: 40.4, 1.5: 40.0, 2: 39.9, 2.5: 40.3, 3: 39.9;
    // scripts/part_sweep.py); C5 unchanged (120.5 us).  Without it a block
    // could take two deep workflows and five short ones (1,418 rows), whose
    // short sweeps then wait ~9 us behind the transfers for a warp
    static const double long_w = [] {
        const char* e = getenv("NALAR_LONG_WEIGHT");
        return e ? atof(e) : kLongWeight;
    }();
    const bool unit_w = long_w == 1.0;          // the default: cost = rows
    const uint32_t lr = fill_sms ? one_wave_long_rows(c, wf_off) : long_rows();
    auto cost = [&](uint32_t w) {
        const uint32_t wr = wf_off[w + 1] - wf_off[w];
        return (unit_w || wr < lr) ? (uint64_t)wr : (uint64_t)(wr * long_w);
    };
    uint64_t total = 0;
    for (uint32_t w = 0; w < W; ++w) total += cost(w);
    const uint64_t even = std::max<uint64_t>(64u, (total + kSmSplit - 1) / kSmSplit);
    // A workflow of at least kDeepAlone 32-row steps (NALAR_DEEP_ALONE, 0 =
    // off) gets a K1 block of its own, so its composition chain -- the
    // longest in the epoch -- runs without sweeps co-scheduled on its SM.
    // Measured on C4 tables of four seeds: -0.4 / 0 / -0.7 / -1.3 us per epoch
    // at 20 steps, never slower; at 12-16 steps too many blocks go to single
    // workflows and the rest overflow one wave (+8-12 us), so it applies only
    // while such workflows are few (<= kDeepAloneMax; C4 tables have 10-13).
    static const uint32_t deep_alone = [] {
        const char* e = getenv("NALAR_DEEP_ALONE");
        return e ? (uint32_t)atoi(e) : kDeepAlone;
    }();
    uint32_t n_deep = 0;
    for (uint32_t w = 0; deep_alone && w < W; ++w) n_deep += wf_off[w + 1] - wf_off[w] >= 32u * deep_alone;
    const bool alone = deep_alone && n_deep <= kDeepAloneMax;
    auto is_deep = [&](uint32_t w) { return alone && wf_off[w + 1] - wf_off[w] >= 32u * deep_alone; };
    // a workflow that would take a block further past the target than the
    // block falls short without it starts the next block (NALAR_CUT_NEAREST)
    static const bool nearest = [] { const char* e = getenv("NALAR_CUT_NEAREST"); return e && atoi(e) != 0; }();
    // one greedy cut at a given per-block target; returns the block count
    auto cut = [&](uint64_t target) -> size_t {
        bw.clear(); br.clear(); be.clear(); bs.clear();
        const size_t guess = (size_t)(total / std::max<uint64_t>(target, 1)) + 8;
        bw.reserve(guess); br.reserve(guess); be.reserve(guess); bs.reserve(guess);
        size_t mx = 0;
        uint32_t w = 0;
        while (w < W) {
            const uint32_t ws = w;
            uint32_t rows = 0;
            uint64_t cst = 0;
            while (w < W) {
                const uint32_t wr = wf_off[w + 1] - wf_off[w];
                const uint32_t e_if = wf_eoff[w + 1] - wf_eoff[ws];
                if (w > ws && ((k1_block_smem_upper(rows + wr, e_if, w - ws + 1, c->T) > kStageBudget &&
                                k1_block_smem(rows + wr, e_if, w - ws + 1, c->T, true) > kStageBudget) ||
                               w - ws + 1 > kMaxWfPerBlock || is_deep(w) ||
                               (nearest && cst + cost(w) > target && cst + cost(w) - target > target - cst)))
                    break;
                rows += wr;
                cst += cost(w);
                ++w;
                if (cst >= target || is_deep(w - 1)) break;
            }
            const uint32_t ra = wf_off[ws], rb = wf_off[w];
            const size_t need_st = k1_block_smem(rb - ra, wf_eoff[w] - wf_eoff[ws], w - ws, c->T, true);
            const bool staged = need_st <= kStageBudget && !(c->cfg.flags & NALAR_F_FORCE_UNSTAGED);
            mx = std::max(mx, staged ? need_st : k1_block_smem(rb - ra, 0, w - ws, c->T, false));
            bw.push_back(ws); br.push_back(ra); be.push_back(wf_eoff[ws]); bs.push_back(staged ? 1 : 0);
        }
        bw.push_back(W); br.push_back(wf_off[W]); be.push_back(wf_eoff[W]);
        *max_smem = mx;
        return bw.size() - 1;
    };
    // Fill the SMs (uploads): the greedy cut overshoots each block by part of a
    // workflow, so a target of total / SMs leaves SMs idle; binary-search the
    // smallest target in [0.8, 1] x even whose cut still fits one wave.  Deltas
    // (a new layout every epoch) take the single cut.
    static const bool fill_env = [] { const char* e = getenv("NALAR_FILL_SMS"); return !e || atoi(e) != 0; }();
    // blocks of one wave; a few SMs may be left to the early-launched K4 blocks
    static const uint32_t wave = [] {
        const char* e = getenv("NALAR_K1_BLOCKS");
        return e ? (uint32_t)atoi(e) : kK1Wave;
    }();
    uint64_t target = even;
    if (fill_sms && fill_env) {
        uint64_t lo = std::max<uint64_t>(64u, even * 4 / 5), hi = even;
        if (cut(lo) <= wave) {
            hi = lo;
        } else {
            for (int it = 0; it < 5 && hi > lo + 1; ++it) {
                const uint64_t mid = lo + (hi - lo) / 2;
                if (cut(mid) <= wave) hi = mid;
                else lo = mid;
            }
        }
        target = hi;
    }
    for (;;) {
        const size_t nb = cut(target);
        if (nb <= c->Bmax) return;
        target *= 2;
    }
}

// the (global_row_base, rows) words of rank s in the exchange buffer
uint32_t* x_rb(nalar_ctx* c) {
    const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
    return c->d_x + (size_t)G * c->Rh * c->Lv + c->I + c->Rh;
}

SweepParams sweep_params(nalar_ctx* c, int policy) {
    SweepParams p{};
    p.verdict = c->d_err + 5;
    p.stream_in = c->streaming ? 1u : 0u;
    p.src = c->sin;
    if (c->sout_on) {
        p.o_status = c->sout.status; p.o_level = c->sout.level; p.o_depth = c->sout.depth;
        p.o_instance = c->sout.instance; p.o_new_pin = c->sout.new_pin;
    }
    p.long_rows = c->long_rows;
    p.wf_fut_off = c->d_wf_off; p.wf_prio = c->d_wf_prio;
    p.f_state = c->d_state; p.f_type = c->d_type; p.f_round = c->d_round;
    p.f_exec = c->d_exec; p.f_pin = c->d_pin; p.f_edge_off = c->d_eoff; p.edges = c->d_edges;
    p.t_aff = c->d_taff;
    p.blk_wf = c->d_blk_wf; p.blk_row0 = c->d_blk_row0; p.blk_edge0 = c->d_blk_edge0;
    p.blk_staged = c->d_blk_staged;
    p.blk_order = c->d_blk_order;
    p.stage_ctr = c->d_scr + C_STAGED;
    static const uint32_t window = [] { const char* e = getenv("NALAR_STAGE_WINDOW"); return e ? (uint32_t)atoi(e) : 24u; }();
    p.stage_window = window ? window : 0xFFFFFFFFu;
    p.wf_perm = c->d_wf_perm;
    p.B = c->B; p.n_types = c->T; p.n_inst = c->I; p.R = c->R; p.levels = c->Lv; p.policy = (uint32_t)policy;
    p.Rh = c->Rh;
    p.mig_on = c->mig_active() ? 1u : 0u; p.theta_wait = c->theta_wait; p.theta_head = c->theta_head;
    p.f_age = c->d_age; p.i_head_rem = c->d_head; p.migrate_to = c->d_migto;
    p.batch_head = c->batch_on ? c->d_bhead : nullptr;
    p.fixed_smem = (uint32_t)c->fixed_smem;
    p.g_flags = c->d_gflags;
    p.g_tlo = c->d_gtlo; p.g_thi = c->d_gthi; p.g_ifc = c->d_gifc; p.g_ndp = c->d_gndp; p.g_aux = c->d_gaux;
    p.prof = c->d_prof;
    p.n_wf = c->W;
    p.status = c->d_status; p.level = c->d_level; p.depth = c->d_depth; p.instance = c->d_inst;
    p.new_pin = c->d_newpin; p.wf_agg = c->d_wfagg;
    p.kv_hint = c->d_kvh; p.kv_level = c->d_kvl; p.kv_home = c->d_kvhome;
    const uint32_t slot = c->cfg.world > 1 ? (uint32_t)c->cfg.rank : 0u;
    p.H = c->d_x + (size_t)slot * c->Rh * c->Lv;
    p.rb_mine = c->cfg.world > 1 ? x_rb(c) + 2 * slot : nullptr;
    // unknown after a delta (nalar_delta carries no row base): not checked
    p.row_base = c->row_base_known ? (uint32_t)c->row_base : 0xFFFFFFFFu;
    p.n_rows = c->N;
    const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
    p.load_part = c->d_x + (size_t)G * c->Rh * c->Lv;
    p.tot = p.load_part + c->I;
    p.items = c->d_items; p.cnt_rb = c->d_cnt_rb; p.off_rb = c->d_off_rb;
    p.tot_loc = c->d_scr + C_NUM + c->Rmax;
    p.counters = c->d_scr;
    return p;
}

int run_k1(nalar_ctx* c, int policy) {
    CK(launch_sweep(sweep_params(c, policy), c->smem, c->stream));
    return NALAR_OK;
}

AssignParams assign_params(nalar_ctx* c) {
    AssignParams p{};
    p.verdict = c->d_err + 5;
    p.stream_in = c->streaming ? 1u : 0u;
    p.err = c->d_err + 2;
    p.host_err = c->h_err_dev;
    if (c->sout_on) { p.o_status = c->sout.status; p.o_instance = c->sout.instance; p.o_new_pin = c->sout.new_pin; }
    const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
    p.H = c->d_x;
    p.rb = c->cfg.world > 1 ? x_rb(c) : nullptr;
    p.order_err = c->h_err_dev + 6;
    p.load_sum = c->d_x + (size_t)G * c->Rh * c->Lv;
    p.tot = p.load_sum + c->I;
    p.type_off = c->d_type_off;
    p.type_inst = c->d_type_inst;
    p.G = G; p.slot = c->cfg.world > 1 ? (uint32_t)c->cfg.rank : 0u;
    p.R = c->R; p.n_inst = c->I; p.n_types = c->T; p.levels = c->Lv; p.B = c->B;
    p.Rh = c->Rh;
    p.i_type = c->d_itype; p.i_cap = c->d_icap; p.i_base = c->d_ibase; p.t_aff = c->d_taff;
    p.cnt_rb = c->d_cnt_rb; p.off_rb = c->d_off_rb; p.blk_row0 = c->d_blk_row0; p.items = c->d_items;
    p.status = c->d_status; p.instance = c->d_inst; p.new_pin = c->d_newpin;
    p.i_load = c->d_iload; p.i_spare = c->d_ispare; p.i_assigned = c->d_iasg;
    p.assign_row = c->d_arow; p.assign_inst = c->d_ainst;
    p.n_adm = c->d_scr + C_NUM;
    p.tot_loc = c->d_scr + C_NUM + c->Rmax;
    p.prof = c->d_prof ? c->d_prof + 2ull * c->W + 8ull * c->B : nullptr;
    p.counters = c->d_scr;
    p.ra_on = c->ra_on; p.u_hi_pct = c->u_hi; p.u_lo_pct = c->u_lo;
    p.t_min_inst = c->d_tmin; p.t_max_inst = c->d_tmax; p.tstat = c->d_tstat;
    p.t_busy = c->d_tbusy; p.t_capsum = c->d_tcap; p.ra_kill = c->d_rakill; p.ra_prov = c->d_raprov;
    return p;
}

int run_k4(nalar_ctx* c) {
    CK(launch_assign(assign_params(c), c->stream));
    return NALAR_OK;
}



// world > 1 with HoL migration: every rank's candidates travel in the exchange
bool lists_on(nalar_ctx* c) { return c->cfg.world > 1 && (c->mig_active() || c->batch_on); }
// the list regions [G][kListWords], right after the (row base, rows) pairs
uint32_t* x_lists(nalar_ctx* c) {
    const uint32_t G = (uint32_t)c->cfg.world;
    return c->d_x + (size_t)G * c->Rh * c->Lv + c->I + c->Rh + 2ull * G;
}

size_t x_used_words(nalar_ctx* c) {
    const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
    return (size_t)G * c->Rh * c->Lv + c->I + c->Rh + 2ull * G + (lists_on(c) ? (size_t)G * kListWords : 0);
}


// an event inside a captured graph must be an external event-record node
cudaError_t record_ev(nalar_ctx* c, int k) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(c->stream, &cs);
    if (e != cudaSuccess) return e;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(c->ev[k], c->stream, cudaEventRecordExternal)
                                               : cudaEventRecord(c->ev[k], c->stream);
}

int enqueue_second_tail(nalar_ctx* c);

int enqueue_first_half(nalar_ctx* c, int policy) {
    const bool timing = c->cfg.flags & NALAR_F_TIMING;
    // clear exchange buffer (used part) + counters + adm_pub; contiguous region
    CK(launch_zero(c->d_x, c->x_words + C_NUM + (size_t)c->Rmax + c->Rhmax, c->stream,
                   c->streaming ? c->d_err + 5 : nullptr));
    if (timing) CK(record_ev(c, 0));
    int rc = run_k1(c, policy);
    if (rc) return rc;
    if (lists_on(c)) {               // this rank's migration candidates -> its list region
        ListParams l{};
        l.mig = c->mig_active() ? 1u : 0u;
        l.batch = c->batch_on ? 1u : 0u;
        l.i_type = c->d_itype; l.t_max_batch = c->d_tmaxb;
        l.f_method = c->have_method ? c->d_method : nullptr;
        l.level = c->d_level;
        l.row_base = (uint32_t)c->row_base;
        l.n_inst = c->I;
        l.tot_loc = c->d_scr + C_NUM + c->Rmax;
        l.cnt_rb = c->d_cnt_rb; l.off_rb = c->d_off_rb; l.blk_row0 = c->d_blk_row0; l.items = c->d_items;
        l.list = x_lists(c) + (size_t)c->cfg.rank * kListWords;
        l.mrow = c->d_mrow;
        l.R = c->R; l.B = c->B; l.n_types = c->T;
        CK(launch_lists(l, c->stream));
    }
    if (timing) CK(record_ev(c, 1));
    return NALAR_OK;
}

int enqueue_collective(nalar_ctx* c) {
    if (c->cfg.collective == NALAR_COLL_PEER) {
        if (!c->peers_ready) return fail(c, NALAR_E_STATE, "peer collective: nalar_peer_connect first");

        PeerParams p{};
        const uint32_t G = (uint32_t)c->cfg.world;
        for (uint32_t q = 0; q < G; ++q) p.peers[q] = c->peers[q];
        p.G = G; p.rank = (uint32_t)c->cfg.rank;
        p.rh_lv = c->Rh * c->Lv; p.I = c->I; p.Rh = c->Rh;
        p.slot = c->d_x + (size_t)p.rank * p.rh_lv;
        p.load = c->d_x + (size_t)G * p.rh_lv;
        p.tot = p.load + c->I;
        p.x = c->d_x;
        p.rb_mine = x_rb(c) + 2 * p.rank;
        p.err = c->peer_err_dev;
        p.par_words = c->peer_par_words;
        p.lw = lists_on(c) ? kListWords : 0u;
        p.list_mine = x_lists(c) + (size_t)p.rank * kListWords;
        CK(launch_peer_exchange(p, c->stream));
        return NALAR_OK;
    }
    if (c->cfg.collective == NALAR_COLL_NCCL) {
        // NOTE: the full reservation-sized layout keeps slot offsets identical on all ranks
        const ncclResult_t r = g_nccl.allReduce(c->d_x, c->d_x, x_used_words(c), ncclUint32, ncclSum, c->comm,
                                                c->stream);
        if (r != ncclSuccess) return fail(c, NALAR_E_COMM, "ncclAllReduce: %s", g_nccl.getErrorString(r));
    }
    return NALAR_OK;
}

int enqueue_second_half(nalar_ctx* c) {
    const bool timing = c->cfg.flags & NALAR_F_TIMING;
    if (timing) CK(record_ev(c, 2));
    int rc = run_k4(c);
    if (rc) return rc;
    return enqueue_second_tail(c);
}

// the optional passes after admission (K5 migration, K6 batches) + timing
int enqueue_second_tail(nalar_ctx* c) {
    const bool timing = c->cfg.flags & NALAR_F_TIMING;
    if (c->mig_active()) {          // K5 HoL migration (NEXT-1), after admission
        MigrateParams m{};
        m.verdict = c->d_err + 5;
        const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
        m.H = c->d_x; m.tot = c->d_x + (size_t)G * c->Rh * c->Lv + c->I;
        m.G = G; m.rank = c->cfg.world > 1 ? (uint32_t)c->cfg.rank : 0u;
        m.lists = G > 1 ? x_lists(c) : nullptr;
        m.mrow = c->d_mrow;
        m.list_err = c->h_err_dev + 7;
        m.cnt_rb = c->d_cnt_rb; m.off_rb = c->d_off_rb; m.blk_row0 = c->d_blk_row0; m.items = c->d_items;
        m.type_off = c->d_type_off; m.type_inst = c->d_type_inst;
        m.i_load = c->d_iload; m.i_assigned = c->d_iasg; m.i_head_rem = c->d_head;
        m.R = c->R; m.Rh = c->Rh; m.B = c->B; m.n_inst = c->I; m.n_types = c->T; m.levels = c->Lv;
        m.theta_head = c->theta_head; m.delta = c->mig_delta;
        m.migrate_to = c->d_migto; m.i_mig_in = c->d_migin; m.i_mig_out = c->d_migout; m.counters = c->d_scr;
        CK(launch_migrate(m, c->stream));
    }
    if (c->batch_on) {              // K6 batch coalescing (NEXT-4), after admission
        BatchParams bp{};
        bp.verdict = c->d_err + 5;
        bp.i_type = c->d_itype; bp.t_max_batch = c->d_tmaxb; bp.f_method = c->have_method ? c->d_method : nullptr;
        bp.level = c->d_level; bp.n_adm = c->d_scr + C_NUM; bp.tot_loc = c->d_scr + C_NUM + c->Rmax;
        bp.arow = c->d_arow; bp.ainst = c->d_ainst; bp.n_inst = c->I;
        bp.batch_head = c->d_bhead; bp.counters = c->d_scr;
        const uint32_t G = c->cfg.world > 1 ? (uint32_t)c->cfg.world : 1u;
        bp.row_base = (uint32_t)c->row_base;
        bp.G = G; bp.n_rows = c->N; bp.R = c->R; bp.levels = c->Lv; bp.Rh = c->Rh;
        bp.lists = G > 1 ? x_lists(c) : nullptr;
        bp.H = c->d_x; bp.tot = c->d_x + (size_t)G * c->Rh * c->Lv + c->I;
        bp.i_spare = c->d_ispare; bp.type_off = c->d_type_off; bp.type_inst = c->d_type_inst;
        bp.list_err = c->h_err_dev + 7;
        CK(launch_batch(bp, c->stream));
    }
    if (timing) CK(record_ev(c, 3));
    return NALAR_OK;
}

// host-side checks of the epoch configuration; run before every epoch, graph
// replays included (a replay must not skip them)
int epoch_checks(nalar_ctx* c) {
    if (c->cfg.collective == NALAR_COLL_PEER && c->cfg.world > 1 && c->peer_failed)
        return fail(c, NALAR_E_COMM, "peer exchange failed earlier: reconnect every rank "
                    "(nalar_peer_buffer + nalar_peer_connect)");
    if (c->batch_on)
        for (uint32_t t = 0; t < c->T && t < c->h_tmaxb.size(); ++t)
            if (c->h_tmaxb[t] > 1 && c->h_taff[t] != NALAR_AFF_NONE)
                return fail(c, NALAR_E_INVAL, "type %u: batchable with managed state (PAPER.md:576)", t);
    if (c->batch_on && c->cfg.world > 1 && !c->row_base_known)
        return fail(c, NALAR_E_STATE, "batch coalescing across ranks needs the snapshot's global_row_base "
                    "(upload a snapshot after a delta)");
    if (c->mig_active() && c->max_inst_per_type > kK5MaxInst)
        return fail(c, NALAR_E_NOTIMPL, "HoL migration supports <= %u instances per type", kK5MaxInst);
    return NALAR_OK;
}

int enqueue_epoch(nalar_ctx* c, int policy) {
    int rc = epoch_checks(c);
    if (rc) return rc;
    rc = enqueue_first_half(c, policy);
    if (!rc) rc = enqueue_collective(c);
    if (!rc) rc = enqueue_second_half(c);
    return rc;
}

// K1 block table from the host mirror of the workflow layout; profile buffer
int set_blocks(nalar_ctx* c, CopyBatch* batch, bool fill_sms = true) {
    std::vector<uint32_t> bw, br, be;
    std::vector<uint8_t> bs;
    size_t mx = 0;
    static const bool trace = getenv("NALAR_TRACE_DELTA") != nullptr || getenv("NALAR_TRACE_UPLOAD") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t0 = trace ? now() : 0;
    partition(c, c->m_wf_off.data(), c->m_wf_eoff.data(), bw, br, be, bs, &mx, fill_sms);
    const double t1 = trace ? now() : 0;
    c->B = (uint32_t)bs.size();
    c->long_rows = long_rows(c->B > kSmSplit);      // several waves: throughput-bound
    if (c->B <= kSmSplit) c->long_rows = one_wave_long_rows(c, c->m_wf_off.data());
    const uint32_t lr = c->long_rows;
    c->all_staged = std::all_of(bs.begin(), bs.end(), [](uint8_t x) { return x != 0; });
    c->fixed_smem = k1_fixed_smem(c->T, c->I, c->Rh);
    c->smem = c->fixed_smem + mx;
    cudaStream_t st = c->stream;
    // task order inside each block: largest workflow first (longest-processing-
    // time-first list scheduling of workflows onto the block's warps)
    c->m_perm.resize(c->W);
    if (c->m_tmp.size() < c->W) c->m_tmp.resize(c->W);
    for (size_t b = 0; b + 1 < bw.size(); ++b) {
        const uint32_t ws = bw[b], we = bw[b + 1];
        uint32_t* o = c->m_perm.data() + ws;
        for (uint32_t k = 0; k < we - ws; ++k) o[k] = k;
        const uint32_t* off = c->m_wf_off.data() + ws;
        if (we - ws <= 16) {
            // (size desc, index asc): a strict total order, so std::sort is
            // deterministic and allocation-free (stable_sort allocates per call)
            std::sort(o, o + (we - ws), [off](uint32_t x, uint32_t y) {
                const uint32_t sx = off[x + 1] - off[x], sy = off[y + 1] - off[y];
                return sx != sy ? sx > sy : x < y;
            });
        } else {
            // many small workflows (a delta-mode table): only the long ones
            // need to start first -- a stable O(n) partition keeps the host
            // cost flat (a full sort per block is ~25 ns per workflow here)
            // (by hand: std::stable_partition allocates a buffer per call,
            // ~50 ns x 145 blocks per delta)
            uint32_t n_long = 0;
            for (uint32_t k = 0; k < we - ws; ++k) n_long += off[k + 1] - off[k] >= lr;
            if (n_long && n_long < we - ws) {
                uint32_t* tmp = c->m_tmp.data();
                uint32_t a = 0, z = n_long;
                for (uint32_t k = 0; k < we - ws; ++k) {
                    if (off[k + 1] - off[k] >= lr) o[a++] = k;
                    else tmp[z++ - n_long] = k;
                }
                std::copy(tmp, tmp + (we - ws - n_long), o + n_long);
            }
        }
    }
    const double t2 = trace ? now() : 0;
    // into the pinned staging, then one copy kernel with the caller's batch
    CopyBatch own(st);
    CopyBatch& cb = batch ? *batch : own;
    struct Part { int slot; const void* src; size_t bytes; void* dst; };
    // CTA order: blocks by estimated sweep cost, costliest first (the
    // longest workflow's 32-row steps, then rows); CTAs are dispatched in
    // index order and a streamed step stages them in this order
    std::vector<uint32_t> order(c->B);
    if (!fill_sms) {                 // a delta's layout (no streamed step): row order
        for (uint32_t b = 0; b < c->B; ++b) order[b] = b;
    } else {
        std::vector<uint64_t> cost(c->B);
        for (uint32_t b = 0; b < c->B; ++b) {
            uint32_t mx = 0;
            for (uint32_t w = bw[b]; w < bw[b + 1]; ++w) mx = std::max(mx, c->m_wf_off[w + 1] - c->m_wf_off[w]);
            cost[b] = ((uint64_t)((mx + 31) / 32) << 32) | (br[b + 1] - br[b]);
        }
        for (uint32_t b = 0; b < c->B; ++b) order[b] = b;
        std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
            return cost[x] != cost[y] ? cost[x] > cost[y] : x < y;
        });
    }
    // per-CTA block records: {block, w0, w1, r0, r1, e0, e1, staged}
    std::vector<uint32_t>& rec = c->m_cta_rec;
    rec.resize(8ull * c->B);
    for (uint32_t i = 0; i < c->B; ++i) {
        const uint32_t b = order[i];
        uint32_t* o = rec.data() + 8ull * i;
        o[0] = b; o[1] = bw[b]; o[2] = bw[b + 1]; o[3] = br[b];
        o[4] = br[b + 1]; o[5] = be[b]; o[6] = be[b + 1]; o[7] = bs[b];
    }
    const Part parts[6] = {
        {2, bw.data(), 4ull * bw.size(), c->d_blk_wf}, {3, br.data(), 4ull * br.size(), c->d_blk_row0},
        {4, be.data(), 4ull * be.size(), c->d_blk_edge0}, {5, bs.data(), bs.size(), c->d_blk_staged},
        {6, c->m_perm.data(), 4ull * c->W, c->d_wf_perm}, {7, rec.data(), 4ull * rec.size(), c->d_blk_order}};
    for (const Part& q : parts) {
        if (!q.bytes) continue;
        memcpy(c->h_tab + c->tab_off[q.slot], q.src, q.bytes);
        CK(cb.add_dev(c->h_tab_dev + c->tab_off[q.slot], q.dst, q.bytes));
    }
    if (c->cfg.flags & NALAR_F_PROFILE) {
        const size_t need = 2ull * c->W + 8ull * c->B + 8ull * c->R + 4ull * c->W + 8ull * c->B;
        if (need > c->prof_words) {
            if (c->d_prof) cudaFree(c->d_prof);
            c->d_prof = nullptr;
            CK(cudaMalloc(&c->d_prof, 8 * std::max<size_t>(need, 1)));
        }
        c->prof_words = need;
        CK(cudaMemsetAsync(c->d_prof, 0, 8 * std::max<size_t>(need, 1), st));
    }
    const double t3 = trace ? now() : 0;
    if (!batch) CK(own.flush());
    if (trace) fprintf(stderr, "[nalar set_blocks] partition %.1f us (%u blocks), order %.1f us, staging %.1f, flush %.1f\n",
                       t1 - t0, c->B, t2 - t1, t3 - t2, now() - t3);
    return NALAR_OK;
}

// K0 over the current table; synchronises
// K0's verdict as published into mapped host memory (valid after a sync)
int validate_verdict(nalar_ctx* c, int64_t* err_row) {
    if (c->h_err[1]) return fail(c, NALAR_E_INVAL, "edge offsets not monotone");
    if (c->h_err[0] != ~0ull) {
        if (err_row) *err_row = (int64_t)c->h_err[0];
        return fail(c, NALAR_E_INVAL, "invalid future row %llu", (unsigned long long)c->h_err[0]);
    }
    return NALAR_OK;
}

int validate_table(nalar_ctx* c, int64_t* err_row, const char*, bool sync = true,
                   unsigned long long* delta_err = nullptr) {
    cudaStream_t st = c->stream;
    c->h_err[0] = ~0ull;                  // the verdict when there is nothing to check
    c->h_err[1] = 0ull;
    ValidateParams v{};
    v.wf_fut_off = c->d_wf_off; v.f_state = c->d_state; v.f_type = c->d_type; v.f_exec = c->d_exec;
    v.f_pin = c->d_pin; v.f_edge_off = c->d_eoff; v.edges = c->d_edges; v.i_type = c->d_itype;
    v.n_wf = c->W; v.n_fut = c->N; v.n_edges = c->E; v.n_types = c->T; v.n_inst = c->I;
    v.err = c->d_err + 2;                 // K0's own words (re-armed by its last block)
    v.done = (uint32_t*)(c->d_err + 4);
    v.host_err = c->h_err_dev;            // K0 publishes [0] / [1] here
    v.verdict = c->d_err + 5;
    v.delta_err = delta_err;
    CK(launch_validate(v, st));
    if (!sync) return NALAR_OK;           // nalar_step: the verdict is read after its one sync
    CK(cudaStreamSynchronize(st));
    return validate_verdict(c, err_row);
}

}  // namespace

// Every entry point runs on its context's device and restores the caller's
// (several contexts on several devices may share a host thread).
struct DevGuard {
    int prev = -1, dev;
    explicit DevGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
        else prev = -1;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ============================================================== C ABI
extern "C" {

int nalar_abi_version(void) { return NALAR_ABI_VERSION; }

size_t nalar_workspace_bytes(const nalar_config* cfg) {
    if (!cfg) return 0;
    Plan p;
    plan_layout(cfg, &p);
    return p.total;
}

int nalar_nccl_unique_id(unsigned char out[128]) {
    std::string e;
    if (!out) return NALAR_E_INVAL;
    if (!g_nccl.load(&e)) return NALAR_E_COMM;
    ncclUniqueId id;
    if (g_nccl.getUniqueId(&id) != ncclSuccess) return NALAR_E_COMM;
    memcpy(out, id.internal, 128);
    return NALAR_OK;
}

int nalar_create(nalar_ctx** out, const nalar_config* cfg) {
    if (!out || !cfg) return NALAR_E_INVAL;
    *out = nullptr;
    g_create_err.clear();
    nalar_ctx* c = new (std::nothrow) nalar_ctx();
    if (!c) return NALAR_E_NOMEM;
    c->cfg = *cfg;
    c->Lv = cfg->levels ? cfg->levels : 256;
    auto bail = [&](int code) { nalar_destroy(c); return code; };
    if (c->Lv > NALAR_MAX_LEVELS || cfg->max_types > NALAR_MAX_TYPES || cfg->max_instances > NALAR_MAX_INSTANCES ||
        cfg->max_futures > NALAR_MAX_ROWS || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world ||
        (cfg->world > 1 && cfg->collective == NALAR_COLL_NONE) ||
        (cfg->collective == NALAR_COLL_PEER && cfg->world > (int)kPeerMaxRanks))
        return bail(NALAR_E_INVAL);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return bail(NALAR_E_CUDA);
    if (cfg->device < 0 || cfg->device >= ndev) return bail(NALAR_E_INVAL);
    cudaDeviceProp prop;
    DevGuard dg(cfg->device);             // the caller's current device is restored on return
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess)
        return bail(NALAR_E_CUDA);
    if (prop.major != 10) return bail(NALAR_E_CUDA);   // built for sm_100a only
    Plan p;
    plan_layout(cfg, &p);
    c->Rmax = p.Rmax;
    c->Rhmax = p.Rhmax;
    c->Bmax = p.Bmax;
    c->x_words = p.x_words;
    if (cfg->workspace) {
        if (cfg->workspace_bytes < p.total) return bail(NALAR_E_NOMEM);
        c->arena = (uint8_t*)(((uintptr_t)cfg->workspace + 255) & ~(uintptr_t)255);
        if ((size_t)(c->arena - (uint8_t*)cfg->workspace) + p.total - 256 > cfg->workspace_bytes)
            return bail(NALAR_E_NOMEM);
    } else {
        if (cudaMalloc(&c->arena, p.total) != cudaSuccess) return bail(NALAR_E_NOMEM);
        c->own_arena = true;
    }
    c->arena_bytes = p.total;
    uint8_t* a = c->arena;
    c->d_wf_off = at<uint32_t>(a, p.wf_off); c->d_wf_prio = at<int32_t>(a, p.wf_prio);
    c->d_wf_id = at<uint64_t>(a, p.wf_id);
    c->d_state = at<uint8_t>(a, p.state); c->d_type = at<uint8_t>(a, p.type); c->d_round = at<uint8_t>(a, p.round);
    c->d_exec = at<int16_t>(a, p.exec); c->d_pin = at<int16_t>(a, p.pin);
    c->d_eoff = at<uint32_t>(a, p.eoff); c->d_edges = at<uint32_t>(a, p.edges);
    c->d_itype = at<uint8_t>(a, p.itype); c->d_icap = at<uint32_t>(a, p.icap); c->d_ibase = at<uint32_t>(a, p.ibase);
    c->d_taff = at<uint8_t>(a, p.taff);
    c->d_blk_wf = at<uint32_t>(a, p.blk_wf); c->d_blk_row0 = at<uint32_t>(a, p.blk_row0);
    c->d_blk_edge0 = at<uint32_t>(a, p.blk_edge0); c->d_blk_staged = at<uint8_t>(a, p.blk_staged);
    c->d_blk_order = at<uint32_t>(a, p.blk_order);
    c->d_wf_perm = at<uint32_t>(a, p.wf_perm);
    c->d_type_off = at<uint32_t>(a, p.type_off); c->d_type_inst = at<uint32_t>(a, p.type_inst);
    c->d_status = at<uint8_t>(a, p.status); c->d_level = at<uint8_t>(a, p.level);
    c->d_newpin = at<uint8_t>(a, p.newpin); c->d_gflags = at<uint8_t>(a, p.gflags);
    c->d_gwlm = at<uint16_t>(a, p.gwlm);
    c->d_gtlo = at<uint32_t>(a, p.gtlo); c->d_gthi = at<uint32_t>(a, p.gthi);
    c->d_gifc = at<uint32_t>(a, p.gifc); c->d_gndp = at<uint32_t>(a, p.gndp); c->d_gaux = at<uint16_t>(a, p.gaux);
    c->d_depth = at<uint16_t>(a, p.depth); c->d_inst = at<int16_t>(a, p.inst); c->d_ainst = at<int16_t>(a, p.ainst);
    c->d_wfagg = at<uint32_t>(a, p.wfagg); c->d_iload = at<uint32_t>(a, p.iload);
    c->d_kvh = at<uint8_t>(a, p.kvh); c->d_kvl = at<uint8_t>(a, p.kvl); c->d_kvhome = at<int16_t>(a, p.kvhome);
    c->d_tmin = at<uint16_t>(a, p.tmin); c->d_tmax = at<uint16_t>(a, p.tmax); c->d_tstat = at<TypeStat>(a, p.tstat);
    c->d_tbusy = at<uint32_t>(a, p.tbusy); c->d_tcap = at<uint32_t>(a, p.tcap);
    c->d_rakill = at<int16_t>(a, p.rakill); c->d_raprov = at<int16_t>(a, p.raprov);
    c->d_age = at<uint32_t>(a, p.age); c->d_head = at<uint32_t>(a, p.head); c->d_migto = at<int16_t>(a, p.migto);
    c->d_migin = at<uint32_t>(a, p.migin); c->d_migout = at<uint32_t>(a, p.migout);
    c->d_tmaxb = at<uint16_t>(a, p.tmaxb); c->d_method = at<uint8_t>(a, p.method); c->d_bhead = at<int32_t>(a, p.bhead);
    c->d_ispare = at<uint32_t>(a, p.ispare); c->d_iasg = at<uint32_t>(a, p.iasg); c->d_arow = at<uint32_t>(a, p.arow);
    c->d_items = at<uint2>(a, p.items); c->d_cnt_rb = at<uint32_t>(a, p.cnt_rb); c->d_off_rb = at<uint32_t>(a, p.off_rb);
    c->d_x = at<uint32_t>(a, p.x); c->d_scr = at<uint32_t>(a, p.scr);
    c->d_mrow = at<uint32_t>(a, p.mrow);
    c->d_err = at<unsigned long long>(a, p.err);
    if (cfg->stream) {
        c->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(NALAR_E_CUDA);
        c->own_stream = true;
    }
    if (cudaMallocHost(&c->h_cnt, 64) != cudaSuccess || cudaMallocHost(&c->h_err, 64) != cudaSuccess ||
        cudaMallocHost(&c->h_reg, 8ull * std::max<uint32_t>(c->Rmax, 1)) != cudaSuccess)
        return bail(NALAR_E_NOMEM);
    {
        const size_t Tm = cfg->max_types, Im = cfg->max_instances, Wm = cfg->max_workflows, Bm = c->Bmax;
        const size_t sz[8] = {4 * (Tm + 1), 4 * Im, 4 * (Bm + 1), 4 * (Bm + 1), 4 * (Bm + 1), Bm, 4 * Wm, 32 * Bm};
        size_t o = 0;
        for (int k = 0; k < 8; ++k) { c->tab_off[k] = o; o += (sz[k] + 15) & ~(size_t)15; }
        if (cudaMallocHost(&c->h_tab, std::max<size_t>(o, 16)) != cudaSuccess) return bail(NALAR_E_NOMEM);
        c->h_tab_dev = (uint8_t*)mapped_view(c->h_tab);
        c->h_cnt_dev = (uint32_t*)mapped_view(c->h_cnt);
        if (!c->h_tab_dev || !c->h_cnt_dev) return bail(NALAR_E_CUDA);
    }
    for (auto& e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return bail(NALAR_E_CUDA);
    c->h_err[4] = 0;
    c->h_err[6] = 0;
    c->h_err[7] = 0;
    c->h_err_dev = (unsigned long long*)mapped_view(c->h_err);
    if (!c->h_err_dev) return bail(NALAR_E_CUDA);
    {   // K0's device words: min bad row ~0, structural 0, block counter 0
        const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
        if (cudaMemcpyAsync(c->d_err, init, sizeof init, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess)
            return bail(NALAR_E_CUDA);
    }
    // Every kernel is loaded now (once per process): under CUDA lazy loading
    // the first launch of a kernel waits for the device to go idle -- a
    // latency spike in the first epoch / delta, and in NALAR_COLL_PEER, where
    // a rank's wait kernel spins until the other ranks push, ranks driven by
    // one host thread would stall until the exchange times out.
    {
        static uint64_t loaded = 0;            // per device (modules load per context)
        const uint64_t bit = 1ull << (cfg->device & 63);
        if (!(loaded & bit)) {
            for (auto f : {preload_k_assign, preload_k_batch, preload_k_delta, preload_k_io,
                           preload_k_migrate, preload_k_peer, preload_k_sweep, preload_k_validate})
                if (f() != cudaSuccess) return bail(NALAR_E_CUDA);
            loaded |= bit;
        }
    }
    if (cfg->collective == NALAR_COLL_PEER) {
        c->peer_par_words = peer_par_words((uint32_t)cfg->world, c->Rhmax, c->Lv, cfg->max_instances);
        const size_t bytes = peer_buffer_bytes((uint32_t)cfg->world, c->Rhmax, c->Lv, cfg->max_instances);
        if (cudaMalloc(&c->peer_buf, bytes) != cudaSuccess) return bail(NALAR_E_NOMEM);
        if (cudaMemset(c->peer_buf, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
            return bail(NALAR_E_CUDA);
        c->peers[cfg->rank] = c->peer_buf;
        c->peer_err_dev = (unsigned long long*)mapped_view(c->h_err + 4);
        if (!c->peer_err_dev) return bail(NALAR_E_CUDA);
    }
    if (cfg->collective == NALAR_COLL_NCCL) {   // (world == 1 allowed: a 1-rank comm, for testing)
        if (!g_nccl.load(&c->err)) { g_create_err = c->err; return bail(NALAR_E_COMM); }
        ncclUniqueId id;
        memcpy(id.internal, cfg->nccl_id, 128);
        // one rank needs no bootstrap: a single-device communicator
        const ncclResult_t r = cfg->world == 1 ? g_nccl.commInitAll(&c->comm, 1, &cfg->device)
                                               : g_nccl.commInitRank(&c->comm, cfg->world, id, cfg->rank);
        if (r != ncclSuccess) {
            g_create_err = std::string("ncclCommInitRank: ") + g_nccl.getErrorString(r);
            c->comm = nullptr;
            return bail(NALAR_E_COMM);
        }
    }
    *out = c;
    return NALAR_OK;
}

int nalar_destroy(nalar_ctx* c) {
    if (!c) return NALAR_OK;
    DevGuard dg(c->cfg.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    destroy_graphs(c);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->comm) g_nccl.commDestroy(c->comm);
    for (void* m : c->peer_ipc)
        if (m) cudaIpcCloseMemHandle(m);
    if (c->peer_buf) cudaFree(c->peer_buf);
    if (c->own_arena && c->arena) cudaFree(c->arena);
    if (c->d_prof) cudaFree(c->d_prof);
    if (c->alt.mem) cudaFree(c->alt.mem);
    if (c->d_stage) cudaFree(c->d_stage);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->h_cnt) cudaFreeHost(c->h_cnt);
    if (c->h_err) cudaFreeHost(c->h_err);
    if (c->h_reg) cudaFreeHost(c->h_reg);
    if (c->h_list) cudaFreeHost(c->h_list);
    if (c->h_tab) cudaFreeHost(c->h_tab);
    if (c->h_dstage) cudaFreeHost(c->h_dstage);
    delete c;
    return NALAR_OK;
}

int nalar_debug_profile(nalar_ctx* c, uint64_t* host, size_t cap, size_t* n_words) {
    if (!c || !n_words) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->d_prof) return fail(c, NALAR_E_STATE, "profiling not enabled (NALAR_F_PROFILE)");
    *n_words = c->prof_words;
    if (!host || cap < c->prof_words) return NALAR_E_SIZE;
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(host, c->d_prof, 8 * c->prof_words, cudaMemcpyDeviceToHost));
    return NALAR_OK;
}

int nalar_debug_blocks(nalar_ctx* c, uint32_t* host, size_t cap, size_t* n_words) {
    if (!c || !n_words) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->uploaded) return fail(c, NALAR_E_STATE, "no table uploaded");
    *n_words = (size_t)c->B + 1;
    if (!host || cap < *n_words) return NALAR_E_SIZE;
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(host, c->d_blk_wf, 4 * *n_words, cudaMemcpyDeviceToHost));
    return NALAR_OK;
}

void* nalar_stream(nalar_ctx* c) { return c ? (void*)c->stream : nullptr; }

int nalar_debug_last_step_streamed(const nalar_ctx* c) { return c && c->last_streamed ? 1 : 0; }

const char* nalar_last_error(const nalar_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

static int upload_impl(nalar_ctx* c, const nalar_snapshot* s, int64_t* err_row, bool sync, bool stream = false);

int nalar_snapshot_upload(nalar_ctx* c, const nalar_snapshot* s, int64_t* err_row) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    return upload_impl(c, s, err_row, true);
}

static int fetch_impl(nalar_ctx* c, nalar_decisions* o);
static int peer_check(nalar_ctx* c, int rc);

int nalar_step(nalar_ctx* c, const nalar_snapshot* s, int policy, nalar_decisions* out, int64_t* err_row) {
    if (!c || !s || !out) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (c->cfg.world > 1 && c->cfg.collective == NALAR_COLL_EXTERNAL)
        return fail(c, NALAR_E_STATE, "external collective: use the split calls");
    if (policy < NALAR_FCFS || policy > NALAR_LPT) return fail(c, NALAR_E_INVAL, "bad policy");
    const double t0 = getenv("NALAR_TRACE_STEP") ? std::chrono::duration<double, std::micro>(
                          std::chrono::steady_clock::now().time_since_epoch()).count() : 0;
    // Streamed step: with the per-row arrays in pinned memory, K1 stages its
    // rows straight from them (TMA over PCIe), validates them in shared memory
    // and writes the device copy -- no separate copy of the table, no K0.
    bool stream = false;
    static const bool stream_env = [] { const char* e = getenv("NALAR_STREAM_STEP"); return !e || atoi(e) != 0; }();
    if (stream_env && s->n_futures && s->n_workflows && !c->batch_on && !c->mig_active_for(s)) {
        StreamIn& q = c->sin;
        q.state = (const uint8_t*)mapped_view(s->f_state);
        q.type = (const uint8_t*)mapped_view(s->f_type);
        q.round = (const uint8_t*)mapped_view(s->f_round);
        q.pin = (const int16_t*)mapped_view(s->f_pin);
        q.exec = (const int16_t*)mapped_view(s->f_executor);
        q.eoff = (const uint32_t*)mapped_view(s->f_edge_off);
        q.edges = s->n_edges ? (const uint32_t*)mapped_view(s->edges) : (const uint32_t*)c->d_edges;
        stream = q.state && q.type && q.round && q.pin && q.exec && q.eoff && q.edges;
    }
    int rc = upload_impl(c, s, err_row, false, stream);   // copies (+ K0 unless streamed) queued, no sync
    if (rc) return rc;
    if (stream && !c->all_staged) {                    // a block too large to stage: the plain path
        c->h_err[0] = ~0ull;
        c->h_err[1] = 0ull;
        CopyBatch cb(c->stream);
        CK(cb.h2d(c->d_state, s->f_state, c->N));
        CK(cb.h2d(c->d_type, s->f_type, c->N));
        CK(cb.h2d(c->d_round, s->f_round, c->N));
        CK(cb.h2d(c->d_exec, s->f_executor, 2ull * c->N));
        CK(cb.h2d(c->d_pin, s->f_pin, 2ull * c->N));
        CK(cb.h2d(c->d_eoff, s->f_edge_off, 4ull * (c->N + 1)));
        CK(cb.h2d(c->d_edges, s->edges, 4ull * c->E));
        CK(cb.flush());
        stream = false;
        rc = validate_table(c, err_row, nullptr, false);
        if (rc) return rc;
    }
    if (stream) {
        c->sin.err = c->d_err + 2;
        c->sin.verdict = c->d_err + 5;
        c->sin.i_type = c->d_itype;
        c->sin.n_edges = c->E; c->sin.n_types = c->T; c->sin.n_inst = c->I;
    }
    c->streaming = stream;
    c->last_streamed = stream;
    // streamed outputs: every requested per-row output pinned and large enough
    {
        static const bool sout_env = [] { const char* e = getenv("NALAR_STREAM_OUT"); return !e || atoi(e) != 0; }();
        nalar_ctx::StreamOut& q = c->sout;
        q = nalar_ctx::StreamOut{};
        bool ok = sout_env && c->N && out->f_cap >= c->N && c->B <= kSmSplit &&   // one-wave tables (K1 build)
                  (out->status || out->level || out->depth || out->instance || out->new_pin);
        auto view = [&](void* h) -> void* {
            if (!h) return nullptr;
            void* v = mapped_view(h);
            if (!v) ok = false;
            return v;
        };
        q.status = (uint8_t*)view(out->status); q.level = (uint8_t*)view(out->level);
        q.depth = (uint16_t*)view(out->depth); q.instance = (int16_t*)view(out->instance);
        q.new_pin = (uint8_t*)view(out->new_pin);
        if (!ok) q = nalar_ctx::StreamOut{};
        c->sout_on = ok;
    }
    static const bool trace = getenv("NALAR_TRACE_STEP") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t1 = trace ? now() : 0;
    rc = nalar_policy_epoch(c, policy);                // kernels skip an invalid table on the device
    c->streaming = false;
    if (rc) { c->uploaded = false; c->sout_on = false; return rc; }
    const double t2 = trace ? now() : 0;
    rc = fetch_impl(c, out);                           // the one synchronisation (skips streamed outputs)
    c->sout_on = false;
    if (trace) fprintf(stderr, "[nalar step] upload queued %.1f us, epoch queued %.1f, fetch+sync %.1f (streamed %d)\n",
                       t1 - t0, t2 - t1, now() - t2, (int)stream);
    const int vr = validate_verdict(c, err_row);       // K0 ran before everything above
    if (vr) {
        c->uploaded = false;
        c->epoch_done = false;
        c->assign_valid = false;
        return vr;
    }
    return peer_check(c, rc);
}

static int upload_impl(nalar_ctx* c, const nalar_snapshot* s, int64_t* err_row, bool sync, bool stream) {
    // NALAR_TRACE_UPLOAD=1: host-side phase times of this call on stderr
    static const bool trace = getenv("NALAR_TRACE_UPLOAD") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double tt[6] = {trace ? now() : 0, 0, 0, 0, 0, 0};
    if (err_row) *err_row = -1;
    if (!c || !s) return NALAR_E_INVAL;
    c->uploaded = false;
    c->epoch_done = false;
    const nalar_config& k = c->cfg;
    if (s->n_futures > k.max_futures || s->n_edges > k.max_edges || s->n_workflows > k.max_workflows ||
        s->n_instances > k.max_instances || s->n_types > k.max_types)
        return fail(c, NALAR_E_NOMEM, "snapshot exceeds reservation");
    const uint32_t N = s->n_futures, E = s->n_edges, W = s->n_workflows, I = s->n_instances, T = s->n_types;
    if (!s->wf_fut_off || !s->f_edge_off || (W && (!s->wf_id || !s->wf_prio)) ||
        (N && (!s->f_state || !s->f_type || !s->f_round || !s->f_executor || !s->f_pin)) || (E && !s->edges) ||
        (I && (!s->i_type || !s->i_cap || !s->i_base_load)) || (T && !s->t_affinity))
        return fail(c, NALAR_E_INVAL, "null array");
    // structural checks that need no per-row work (host, O(W + I + T))
    if (s->wf_fut_off[0] != 0 || s->wf_fut_off[W] != N) return fail(c, NALAR_E_INVAL, "wf_fut_off bounds");
    for (uint32_t w = 0; w < W; ++w) {
        if (s->wf_fut_off[w + 1] < s->wf_fut_off[w]) return fail(c, NALAR_E_INVAL, "wf_fut_off not monotone");
        if (w && s->wf_id[w] <= s->wf_id[w - 1]) return fail(c, NALAR_E_INVAL, "wf_id not increasing");
    }
    if (s->f_edge_off[0] != 0 || s->f_edge_off[N] != E) return fail(c, NALAR_E_INVAL, "f_edge_off bounds");
    for (uint32_t i = 0; i < I; ++i)
        if (s->i_type[i] >= T) return fail(c, NALAR_E_INVAL, "instance type out of range");
    for (uint32_t t = 0; t < T; ++t)
        if (s->t_affinity[t] > NALAR_AFF_STATEFUL) return fail(c, NALAR_E_INVAL, "affinity out of range");
    if (N && T == 0) return fail(c, NALAR_E_INVAL, "futures without types");

    c->N = N; c->E = E; c->W = W; c->I = I; c->T = T; c->R = I + T; c->Rh = I + 2 * T;
    c->row_base = s->global_row_base;
    c->row_base_known = true;
    c->assign_valid = false;
    // host mirror of the workflow layout (delta mode re-partitions from it)
    // the K1 block partition depends only on the workflow layout (row and edge
    // offsets) and T: a steady-state controller re-uploading tables of the same
    // shape keeps its block tables on the device
    bool same_layout = c->blocks_valid && c->blocks_T == T && c->m_wf_off.size() == (size_t)W + 1 &&
                       std::equal(s->wf_fut_off, s->wf_fut_off + W + 1, c->m_wf_off.begin());
    for (uint32_t w = 0; same_layout && w <= W; ++w)
        same_layout = c->m_wf_eoff[w] == s->f_edge_off[s->wf_fut_off[w]];
    c->blocks_valid = false;                 // until the tables below are in place
    c->m_wf_id.assign(s->wf_id, s->wf_id + W);
    if (!same_layout) {
        c->m_wf_off.assign(s->wf_fut_off, s->wf_fut_off + W + 1);
        c->m_wf_eoff.resize(W + 1);
        for (uint32_t w = 0; w <= W; ++w) c->m_wf_eoff[w] = s->f_edge_off[s->wf_fut_off[w]];
    }

    if (trace) tt[1] = now();
    cudaStream_t st = c->stream;
    // every array in one copy kernel when the caller's buffers are pinned
    CopyBatch cb(st);
    auto h2d = [&](void* d, const void* h, size_t bytes) -> cudaError_t { return cb.h2d(d, h, bytes); };
    CK(h2d(c->d_wf_off, s->wf_fut_off, 4ull * (W + 1)));
    CK(h2d(c->d_wf_prio, s->wf_prio, 4ull * W));
    CK(h2d(c->d_wf_id, s->wf_id, 8ull * W));
    if (!stream) {          // (a streamed step's sweep reads these from the caller's memory)
        CK(h2d(c->d_state, s->f_state, N));
        CK(h2d(c->d_type, s->f_type, N));
        CK(h2d(c->d_round, s->f_round, N));
        CK(h2d(c->d_exec, s->f_executor, 2ull * N));
        CK(h2d(c->d_pin, s->f_pin, 2ull * N));
        CK(h2d(c->d_eoff, s->f_edge_off, 4ull * (N + 1)));
        CK(h2d(c->d_edges, s->edges, 4ull * E));
    }
    CK(h2d(c->d_itype, s->i_type, I));
    CK(h2d(c->d_icap, s->i_cap, 4ull * I));
    CK(h2d(c->d_ibase, s->i_base_load, 4ull * I));
    CK(h2d(c->d_taff, s->t_affinity, T));
    c->have_mig = s->f_age && s->i_head_rem;
    c->have_method = s->f_method != nullptr;
    c->h_taff.assign(s->t_affinity, s->t_affinity + T);
    if (c->have_method) CK(h2d(c->d_method, s->f_method, N));
    if (c->have_mig) {
        CK(h2d(c->d_age, s->f_age, 4ull * N));
        CK(h2d(c->d_head, s->i_head_rem, 4ull * I));
    }
    // instances grouped by type (ascending id), for the assignment pass
    if (trace) tt[2] = now();
    uint32_t* toff = (uint32_t*)(c->h_tab + c->tab_off[0]);
    uint32_t* tinst = (uint32_t*)(c->h_tab + c->tab_off[1]);
    std::fill(toff, toff + T + 1, 0u);
    for (uint32_t i = 0; i < I; ++i) toff[s->i_type[i] + 1]++;
    c->max_inst_per_type = 0;
    for (uint32_t t = 0; t < T; ++t) c->max_inst_per_type = std::max(c->max_inst_per_type, toff[t + 1]);
    for (uint32_t t = 0; t < T; ++t) toff[t + 1] += toff[t];
    {
        std::vector<uint32_t> cur(toff, toff + T);
        for (uint32_t i = 0; i < I; ++i) tinst[cur[s->i_type[i]]++] = i;
    }
    CK(cb.add_dev(c->h_tab_dev + c->tab_off[0], c->d_type_off, 4ull * (T + 1)));
    CK(cb.add_dev(c->h_tab_dev + c->tab_off[1], c->d_type_inst, 4ull * I));
    int rc = same_layout ? NALAR_OK : set_blocks(c, &cb);
    if (rc) return rc;
    CK(cb.flush());
    c->blocks_valid = true;
    c->blocks_T = T;
    if (trace) tt[3] = now();
    if (stream) {
        // K1 checks the rows (K0's contract) as it stages them; K4 publishes
        // a failure into h_err, read after the step's synchronisation
        c->h_err[0] = ~0ull;
        c->h_err[1] = 0ull;
        c->uploaded = true;
        return NALAR_OK;
    }
    rc = validate_table(c, err_row, nullptr, sync);
    if (trace) {
        tt[4] = now();
        fprintf(stderr, "[nalar upload] checks+mirror %.1f us, array copies issued %.1f, tables+partition+kernel %.1f, "
                "validate+sync %.1f, total %.1f\n", tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3],
                tt[4] - tt[0]);
    }
    if (rc) return rc;
    c->uploaded = true;
    return NALAR_OK;
}

int nalar_delta_apply(nalar_ctx* c, const nalar_delta* d, int64_t* err_index) {
    // NALAR_TRACE_DELTA=1: host-side phase times of this call on stderr
    static const bool trace = getenv("NALAR_TRACE_DELTA") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double tt[6] = {trace ? now() : 0, 0, 0, 0, 0, 0};
    if (err_index) *err_index = -1;
    if (!c || !d) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->uploaded) return fail(c, NALAR_E_STATE, "delta before upload");
    c->row_base_known = false;
    const bool apply_asg = d->flags & NALAR_DELTA_APPLY_ASSIGNED;
    if (apply_asg && !c->assign_valid) return fail(c, NALAR_E_STATE, "APPLY_ASSIGNED without a preceding epoch");
    if ((d->n_updates && (!d->upd_wf_id || !d->upd_seq || !d->upd_state || !d->upd_executor || !d->upd_pin)) ||
        (d->n_retired && !d->retired_wf_id) ||
        (d->n_append && (!d->app_wf_id || !d->app_wf_prio || !d->app_state || !d->app_type || !d->app_round ||
                         !d->app_executor || !d->app_pin || !d->app_edge_off)) ||
        (d->n_append_edges && !d->app_edges) || (d->n_prio && (!d->prio_wf_id || !d->prio_value)) ||
        (d->n_inst && (!d->inst_id || !d->inst_cap || !d->inst_base_load)))
        return fail(c, NALAR_E_INVAL, "null delta array");
    const uint32_t W = c->W;
    // ---- host: the new workflow list (old minus retired, plus appended) ----
    std::vector<uint8_t>& retired = c->m_retired;
    retired.assign(W, 0);
    for (uint32_t k = 0; k < d->n_retired; ++k) {
        const auto it = std::lower_bound(c->m_wf_id.begin(), c->m_wf_id.end(), d->retired_wf_id[k]);
        if (it == c->m_wf_id.end() || *it != d->retired_wf_id[k]) {
            if (err_index) *err_index = k;
            return fail(c, NALAR_E_INVAL, "retired workflow id %llu not live", (unsigned long long)d->retired_wf_id[k]);
        }
        retired[it - c->m_wf_id.begin()] = 1;
    }
    if (d->n_append && (d->app_edge_off[0] != 0 || d->app_edge_off[d->n_append] != d->n_append_edges))
        return fail(c, NALAR_E_INVAL, "app_edge_off bounds");
    for (uint32_t j = 0; j < d->n_append; ++j)
        if (d->app_edge_off[j + 1] < d->app_edge_off[j]) {
            if (err_index) *err_index = j;
            return fail(c, NALAR_E_INVAL, "app_edge_off not monotone");
        }
    // appended groups: (wf id, first index, count), ids ascending
    struct Grp { uint64_t id; uint32_t lo, n; };
    std::vector<Grp> groups;
    for (uint32_t j = 0; j < d->n_append; ++j) {
        if (!groups.empty() && groups.back().id == d->app_wf_id[j]) { groups.back().n++; continue; }
        if (!groups.empty() && d->app_wf_id[j] < groups.back().id) {
            if (err_index) *err_index = j;
            return fail(c, NALAR_E_INVAL, "appended futures not grouped by ascending workflow id");
        }
        groups.push_back({d->app_wf_id[j], j, 1});
    }
    std::vector<RebuildPlan>& plan = c->m_plan;      // reused across deltas (no allocation)
    plan.clear();
    plan.reserve(W + groups.size());
    const uint64_t max_live = W ? c->m_wf_id.back() : 0;
    size_t g = 0;
    uint32_t row = 0, edge = 0;
    auto app_edges = [&](const Grp& gr) { return d->app_edge_off[gr.lo + gr.n] - d->app_edge_off[gr.lo]; };
    for (uint32_t w = 0; w < W; ++w) {
        const uint64_t id = c->m_wf_id[w];
        while (g < groups.size() && groups[g].id < id) {   // an id between live ids is not new
            if (err_index) *err_index = groups[g].lo;
            return fail(c, NALAR_E_INVAL, "appended workflow id %llu is neither live nor new",
                        (unsigned long long)groups[g].id);
        }
        const bool has_app = g < groups.size() && groups[g].id == id;
        if (retired[w]) {
            if (has_app) {
                if (err_index) *err_index = groups[g].lo;
                return fail(c, NALAR_E_INVAL, "append to a retired workflow");
            }
            continue;
        }
        RebuildPlan pl{};
        pl.wf_id = id; pl.src = w;
        pl.n_old = c->m_wf_off[w + 1] - c->m_wf_off[w];
        pl.n_old_edges = c->m_wf_eoff[w + 1] - c->m_wf_eoff[w];
        pl.app_lo = has_app ? groups[g].lo : 0; pl.app_n = has_app ? groups[g].n : 0;
        pl.new_row0 = row; pl.new_edge0 = edge;
        row += pl.n_old + pl.app_n;
        edge += pl.n_old_edges + (has_app ? app_edges(groups[g]) : 0);
        if (has_app) ++g;
        plan.push_back(pl);
    }
    for (; g < groups.size(); ++g) {
        if (groups[g].id <= max_live && W) {
            if (err_index) *err_index = groups[g].lo;
            return fail(c, NALAR_E_INVAL, "new workflow id %llu not above the live ids", (unsigned long long)groups[g].id);
        }
        RebuildPlan pl{};
        pl.wf_id = groups[g].id; pl.src = 0xFFFFFFFFu;
        pl.app_lo = groups[g].lo; pl.app_n = groups[g].n;
        pl.prio = d->app_wf_prio[groups[g].lo];
        pl.new_row0 = row; pl.new_edge0 = edge;
        row += pl.app_n;
        edge += app_edges(groups[g]);
        plan.push_back(pl);
    }
    const uint32_t W2 = (uint32_t)plan.size(), N2 = row, E2 = edge;
    if (trace) tt[1] = now();
    if (N2 > c->cfg.max_futures || E2 > c->cfg.max_edges || W2 > c->cfg.max_workflows)
        return fail(c, NALAR_E_NOMEM, "delta outgrows the reservation");
    // ---- device: second buffer set, staging ----------------------------------
    if (!c->alt.mem) {
        Layout L;
        const size_t N = c->cfg.max_futures, E = c->cfg.max_edges, Wm = c->cfg.max_workflows;
        const size_t o_wo = L.take<uint32_t>(Wm + 1), o_wp = L.take<int32_t>(Wm), o_wi = L.take<uint64_t>(Wm);
        const size_t o_st = L.take<uint8_t>(N), o_ty = L.take<uint8_t>(N), o_rd = L.take<uint8_t>(N);
        const size_t o_ex = L.take<int16_t>(N), o_pn = L.take<int16_t>(N), o_eo = L.take<uint32_t>(N + 1);
        const size_t o_ed = L.take<uint32_t>(E);
        if (cudaMalloc(&c->alt.mem, L.off + 256) != cudaSuccess) { c->alt.mem = nullptr; return fail(c, NALAR_E_NOMEM, "delta buffers"); }
        uint8_t* m = (uint8_t*)c->alt.mem;
        c->alt.wf_off = at<uint32_t>(m, o_wo); c->alt.wf_prio = at<int32_t>(m, o_wp); c->alt.wf_id = at<uint64_t>(m, o_wi);
        c->alt.state = at<uint8_t>(m, o_st); c->alt.type = at<uint8_t>(m, o_ty); c->alt.round = at<uint8_t>(m, o_rd);
        c->alt.exec = at<int16_t>(m, o_ex); c->alt.pin = at<int16_t>(m, o_pn); c->alt.eoff = at<uint32_t>(m, o_eo);
        c->alt.edges = at<uint32_t>(m, o_ed);
    }
    Layout S;
    const uint32_t nu = d->n_updates, na = d->n_append, nae = d->n_append_edges, np = d->n_prio, ni = d->n_inst;
    const size_t s_uid = S.take<uint64_t>(nu), s_useq = S.take<uint32_t>(nu), s_ust = S.take<uint8_t>(nu);
    const size_t s_uex = S.take<int16_t>(nu), s_upn = S.take<int16_t>(nu);
    const size_t s_plan = S.take<RebuildPlan>(W2);
    const size_t s_ast = S.take<uint8_t>(na), s_aty = S.take<uint8_t>(na), s_ard = S.take<uint8_t>(na);
    const size_t s_aex = S.take<int16_t>(na), s_apn = S.take<int16_t>(na), s_aeo = S.take<uint32_t>(na + 1);
    const size_t s_aed = S.take<uint32_t>(nae);
    const size_t s_pid = S.take<uint64_t>(np), s_pvl = S.take<int32_t>(np);
    const size_t s_iid = S.take<uint32_t>(ni), s_icp = S.take<uint32_t>(ni), s_ibl = S.take<uint32_t>(ni);
    if (S.off > c->h_dstage_bytes) {
        if (c->h_dstage) cudaFreeHost(c->h_dstage);
        c->h_dstage = nullptr;
        c->h_dstage_bytes = 0;
        if (cudaMallocHost(&c->h_dstage, 2 * S.off + 4096) != cudaSuccess)
            return fail(c, NALAR_E_NOMEM, "pinned delta staging");
        c->h_dstage_bytes = 2 * S.off + 4096;
    }
    if (S.off > c->stage_bytes) {
        if (c->d_stage) cudaFree(c->d_stage);
        c->d_stage = nullptr;
        c->stage_bytes = 0;
        if (cudaMalloc(&c->d_stage, 2 * S.off + 4096) != cudaSuccess) return fail(c, NALAR_E_NOMEM, "delta staging");
        c->stage_bytes = 2 * S.off + 4096;
    }
    uint8_t* sb = (uint8_t*)c->d_stage;
    cudaStream_t st = c->stream;
    // every delta array into the pinned staging area (host memcpy), then one
    // async H2D -- instead of ~20 pageable cudaMemcpyAsync calls
    auto h2d = [&](size_t off, const void* h, size_t bytes) -> cudaError_t {
        if (bytes) memcpy(c->h_dstage + off, h, bytes);
        return cudaSuccess;
    };
    CK(h2d(s_uid, d->upd_wf_id, 8ull * nu)); CK(h2d(s_useq, d->upd_seq, 4ull * nu));
    CK(h2d(s_ust, d->upd_state, nu)); CK(h2d(s_uex, d->upd_executor, 2ull * nu)); CK(h2d(s_upn, d->upd_pin, 2ull * nu));
    CK(h2d(s_plan, plan.data(), sizeof(RebuildPlan) * W2));
    CK(h2d(s_ast, d->app_state, na)); CK(h2d(s_aty, d->app_type, na)); CK(h2d(s_ard, d->app_round, na));
    CK(h2d(s_aex, d->app_executor, 2ull * na)); CK(h2d(s_apn, d->app_pin, 2ull * na));
    if (na) { CK(h2d(s_aeo, d->app_edge_off, 4ull * (na + 1))); } else { static const uint32_t z = 0; CK(h2d(s_aeo, &z, 4)); }
    CK(h2d(s_aed, d->app_edges, 4ull * nae));
    CK(h2d(s_pid, d->prio_wf_id, 8ull * np)); CK(h2d(s_pvl, d->prio_value, 4ull * np));
    CK(h2d(s_iid, d->inst_id, 4ull * ni)); CK(h2d(s_icp, d->inst_cap, 4ull * ni)); CK(h2d(s_ibl, d->inst_base_load, 4ull * ni));
    CK(cudaMemcpyAsync(sb, c->h_dstage, S.off, cudaMemcpyHostToDevice, st));
    // (the update-error words d_err[0], [1] are armed (~0); K0's last block
    // publishes them to h_err[2], [3] after this delta and re-arms them)
    DeltaParams p{};
    p.wf_off = c->d_wf_off; p.wf_prio = c->d_wf_prio; p.wf_id = c->d_wf_id;
    p.state = c->d_state; p.type = c->d_type; p.round = c->d_round; p.exec = c->d_exec; p.pin = c->d_pin;
    p.eoff = c->d_eoff; p.edges = c->d_edges; p.n_wf = W;
    p.tot_loc = c->d_scr + C_NUM + c->Rmax; p.n_adm = c->d_scr + C_NUM; p.arow = c->d_arow; p.ainst = c->d_ainst;
    p.n_upd = nu; p.upd_wf_id = at<uint64_t>(sb, s_uid); p.upd_seq = at<uint32_t>(sb, s_useq);
    p.upd_state = at<uint8_t>(sb, s_ust); p.upd_exec = at<int16_t>(sb, s_uex); p.upd_pin = at<int16_t>(sb, s_upn);
    p.n_wf_new = W2; p.plan = at<RebuildPlan>(sb, s_plan);
    p.n_wf_off = c->alt.wf_off; p.n_wf_prio = c->alt.wf_prio; p.n_wf_id = c->alt.wf_id;
    p.n_state = c->alt.state; p.n_type = c->alt.type; p.n_round = c->alt.round; p.n_exec = c->alt.exec;
    p.n_pin = c->alt.pin; p.n_eoff = c->alt.eoff; p.n_edges = c->alt.edges;
    p.app_state = at<uint8_t>(sb, s_ast); p.app_type = at<uint8_t>(sb, s_aty); p.app_round = at<uint8_t>(sb, s_ard);
    p.app_exec = at<int16_t>(sb, s_aex); p.app_pin = at<int16_t>(sb, s_apn); p.app_eoff = at<uint32_t>(sb, s_aeo);
    p.app_edges = at<uint32_t>(sb, s_aed);
    p.n_prio = np; p.prio_wf_id = at<uint64_t>(sb, s_pid); p.prio_value = at<int32_t>(sb, s_pvl);
    p.n_inst_upd = ni; p.n_inst = c->I; p.inst_id = at<uint32_t>(sb, s_iid); p.inst_cap = at<uint32_t>(sb, s_icp);
    p.inst_base = at<uint32_t>(sb, s_ibl); p.i_cap = c->d_icap; p.i_base = c->d_ibase;
    p.err = c->d_err;
    p.n_fut_new = N2; p.n_edges_new = E2;               // KD3 writes the offset tails
    CK(launch_delta(p, apply_asg, c->R, st));
    if (W2 == 0) {                                       // (no KD3 block: write them here)
        CK(cudaMemsetAsync(c->alt.wf_off, 0, 4, st));
        CK(cudaMemsetAsync(c->alt.eoff, 0, 4, st));
    }
    c->assign_valid = false;
    if (trace) tt[2] = now();
    // ---- swap in the new table, re-partition, validate ------------------------
    std::swap(c->d_wf_off, c->alt.wf_off); std::swap(c->d_wf_prio, c->alt.wf_prio); std::swap(c->d_wf_id, c->alt.wf_id);
    std::swap(c->d_state, c->alt.state); std::swap(c->d_type, c->alt.type); std::swap(c->d_round, c->alt.round);
    std::swap(c->d_exec, c->alt.exec); std::swap(c->d_pin, c->alt.pin); std::swap(c->d_eoff, c->alt.eoff);
    std::swap(c->d_edges, c->alt.edges);
    // the new host mirror (into the spare vectors of the last delta: no allocation)
    std::vector<uint64_t>& nid = c->m_spare_id;
    std::vector<uint32_t>& noff = c->m_spare_off;
    std::vector<uint32_t>& neoff = c->m_spare_eoff;
    nid.resize(W2);
    noff.resize(W2 + 1);
    neoff.resize(W2 + 1);
    for (uint32_t w = 0; w < W2; ++w) { nid[w] = plan[w].wf_id; noff[w] = plan[w].new_row0; neoff[w] = plan[w].new_edge0; }
    noff[W2] = N2; neoff[W2] = E2;
    c->m_wf_id.swap(nid); c->m_wf_off.swap(noff); c->m_wf_eoff.swap(neoff);
    c->N = N2; c->E = E2; c->W = W2;
    c->have_mig = false;             // HoL inputs are per upload (row indices moved)
    c->have_method = false;          // so are the batch methods (d_method is in pre-delta row order)
    int rc = set_blocks(c, nullptr, /*fill_sms=*/false);
    if (trace) tt[3] = now();
    c->h_err[2] = ~0ull;
    c->h_err[3] = ~0ull;
    if (!rc && N2 && W2) {
        rc = validate_table(c, err_index, nullptr, true, c->d_err);   // synchronises; publishes the update errors
    } else {
        if (!rc) rc = validate_table(c, err_index, nullptr, false);   // (nothing to check: clears the verdict)
        cudaMemcpyAsync(c->h_err + 2, c->d_err, 16, cudaMemcpyDeviceToHost, st);
        cudaMemsetAsync(c->d_err, 0xFF, 16, st);
        cudaStreamSynchronize(st);
    }
    if (trace) {
        tt[4] = now();
        fprintf(stderr, "[nalar delta] plan %.1f us, stage+launch %.1f, swap+partition %.1f, validate+sync %.1f, "
                "total %.1f (W %u -> %u, N %u)\n", tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3],
                tt[4] - tt[0], W, W2, N2);
    }
    if (c->h_err[2] != ~0ull || c->h_err[3] != ~0ull) {
        c->uploaded = false;          // the table was partly updated in place
        const unsigned long long bad = c->h_err[2] != ~0ull ? c->h_err[2] : c->h_err[3];
        if (err_index) *err_index = (int64_t)bad;
        return fail(c, NALAR_E_INVAL, "delta update %llu names no live future / workflow / instance", bad);
    }
    if (rc) { c->uploaded = false; return rc; }
    c->epoch_done = false;
    return NALAR_OK;
}

int nalar_policy_epoch(nalar_ctx* c, int policy) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->uploaded) return fail(c, NALAR_E_STATE, "epoch before upload");
    if (policy < NALAR_FCFS || policy > NALAR_LPT) return fail(c, NALAR_E_INVAL, "bad policy");
    if (c->cfg.world > 1 && c->cfg.collective == NALAR_COLL_EXTERNAL)
        return fail(c, NALAR_E_STATE, "external collective: use nalar_epoch_begin/finish");
    int rc = epoch_checks(c);
    if (rc) return rc;
    uint64_t th = 1469598103934665603ull;
    for (uint8_t a : c->h_taff) th = (th ^ a) * 1099511628211ull;
    Key key{c->N, c->E, c->W, c->I, c->T, c->B, c->R, (uint32_t)policy, c->params_gen, c->smem, c->d_state,
            (c->have_mig ? 1u : 0u) | (c->have_method ? 2u : 0u), th, c->max_inst_per_type};
    if (c->streaming || c->sout_on) {
        const void* a[12] = {c->sin.state, c->sin.type, c->sin.round, c->sin.pin, c->sin.exec, c->sin.eoff,
                             c->sin.edges, c->sout.status, c->sout.level, c->sout.depth, c->sout.instance,
                             c->sout.new_pin};
        uint64_t h = 1469598103934665603ull ^ (c->streaming ? 7ull : 0ull);
        for (const void* x : a) h = (h ^ (uint64_t)(uintptr_t)x) * 1099511628211ull;
        key.stream_key = h | 1ull;
    }
    // a graph pays off only for a shape that repeats (not after every delta)
    const bool repeat = c->last_key_set && c->last_key == key;
    const bool cached = c->gexec[policy] && c->gkey[policy] == key;
    c->last_key = key;
    c->last_key_set = true;
    if ((c->cfg.flags & NALAR_F_NO_GRAPH) || (!repeat && !cached)) {
        rc = enqueue_epoch(c, policy);
    } else {
        cudaGraphExec_t& ge = c->gexec[policy];
        if (!ge || !(c->gkey[policy] == key)) {
            if (ge) { cudaGraphExecDestroy(ge); ge = nullptr; }
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            rc = enqueue_epoch(c, policy);
            cudaError_t e = cudaStreamEndCapture(c->stream, &g);
            if (rc) { if (e == cudaSuccess) cudaGraphDestroy(g); return rc; }
            CK(e);
            e = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            CK(e);
            c->gkey[policy] = key;
        }
        CK(cudaGraphLaunch(ge, c->stream));
        rc = NALAR_OK;
    }
    if (!rc) { c->epoch_done = true; c->last_policy = policy; c->assign_valid = true; }
    return rc;
}

int nalar_epoch_begin(nalar_ctx* c, int policy) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->uploaded) return fail(c, NALAR_E_STATE, "epoch before upload");
    if (policy < NALAR_FCFS || policy > NALAR_LPT) return fail(c, NALAR_E_INVAL, "bad policy");
    int rc = epoch_checks(c);
    if (!rc) rc = enqueue_first_half(c, policy);
    if (!rc) { c->in_epoch = true; c->last_policy = policy; }
    return rc;
}

int nalar_exchange_buffer(nalar_ctx* c, void** dev_ptr, size_t* n_words) {
    if (!c || !dev_ptr || !n_words) return NALAR_E_INVAL;
    *dev_ptr = c->d_x;
    *n_words = c->uploaded ? x_used_words(c) : c->x_words;
    return NALAR_OK;
}

int nalar_epoch_finish(nalar_ctx* c) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->in_epoch) return fail(c, NALAR_E_STATE, "finish without begin");
    c->in_epoch = false;
    int rc = enqueue_second_half(c);
    if (!rc) { c->epoch_done = true; c->assign_valid = true; }
    return rc;
}

static int fetch_impl(nalar_ctx* c, nalar_decisions* o);

// a peer exchange that timed out (k_peer_gather) fails the next synchronising call
static int peer_check(nalar_ctx* c, int rc) {
    if (rc == NALAR_OK && c->peer_buf && c->h_err[4]) {
        c->h_err[4] = 0;
        c->peer_failed = true;
        return fail(c, NALAR_E_COMM, "peer exchange: a rank's flag never arrived (timed out)");
    }
    if (rc == NALAR_OK && c->h_err[6]) {        // K4: the ranks' row ranges (world > 1)
        c->h_err[6] = 0;
        return fail(c, NALAR_E_INVAL, "ranks' workflow ranges out of order (global_row_base)");
    }
    if (rc == NALAR_OK && c->h_err[7]) {        // K5: a rank's candidate list overflowed (world > 1)
        c->h_err[7] = 0;
        return fail(c, NALAR_E_NOTIMPL, "HoL migration / batching: more candidates on a rank than its exchange "
                    "list holds (world > 1)");
    }
    return rc;
}

int nalar_fetch_decisions(nalar_ctx* c, nalar_decisions* o) {
    if (!c || !o) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    return peer_check(c, fetch_impl(c, o));
}

int nalar_peer_buffer(nalar_ctx* c, void** dev_ptr, unsigned char ipc_handle[64]) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->peer_buf) return fail(c, NALAR_E_STATE, "not a NALAR_COLL_PEER context");
    // (re)connection starts from clean flags and epoch counters on every rank
    const size_t bytes = peer_buffer_bytes((uint32_t)c->cfg.world, c->Rhmax, c->Lv, c->cfg.max_instances);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemset(c->peer_buf, 0, bytes));
    CK(cudaDeviceSynchronize());
    c->h_err[4] = 0;
    c->peers_ready = false;
    if (dev_ptr) *dev_ptr = c->peer_buf;
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, c->peer_buf));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        memcpy(ipc_handle, &h, 64);
    }
    return NALAR_OK;
}

int nalar_peer_connect(nalar_ctx* c, void* const* ptrs, const unsigned char* handles) {
    if (!c) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->peer_buf) return fail(c, NALAR_E_STATE, "not a NALAR_COLL_PEER context");
    const int G = c->cfg.world, me = c->cfg.rank;
    for (int q = 0; q < G; ++q) {
        if (q == me) continue;
        if (c->peer_ipc[q]) { cudaIpcCloseMemHandle(c->peer_ipc[q]); c->peer_ipc[q] = nullptr; }
        if (ptrs && ptrs[q]) {
            c->peers[q] = (uint32_t*)ptrs[q];
        } else if (handles) {
            cudaIpcMemHandle_t h;
            memcpy(&h, handles + 64 * (size_t)q, 64);
            void* m = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&m, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                c->peers_ready = false;
                return fail(c, NALAR_E_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
            }
            c->peer_ipc[q] = m;
            c->peers[q] = (uint32_t*)m;
        } else {
            c->peers_ready = false;
            return fail(c, NALAR_E_INVAL, "peer_connect: no pointer or handle for rank %d", q);
        }
    }
    c->peers_ready = true;
    c->peer_failed = false;
    return NALAR_OK;
}

static int fetch_impl(nalar_ctx* c, nalar_decisions* o) {
    if (!c->epoch_done) return fail(c, NALAR_E_STATE, "fetch before epoch");
    cudaStream_t st = c->stream;
    // without an active migration pass nothing moves: answer on the host
    const bool mig = c->mig_active();
    if (!mig) {
        if (o->migrate_to && o->f_cap >= c->N) std::fill_n(o->migrate_to, c->N, (int16_t)-1);
        if (o->i_mig_in && o->i_cap >= c->I) memset(o->i_mig_in, 0, 4ull * c->I);
        if (o->i_mig_out && o->i_cap >= c->I) memset(o->i_mig_out, 0, 4ull * c->I);
    }
    if (!c->batch_on && o->batch_head && o->f_cap >= c->N) std::fill_n(o->batch_head, c->N, (int32_t)-1);
    // Fast path: every requested output buffer is pinned (device-mapped) host
    // memory -> one kernel writes them all, compacting the assignment list on
    // the way, and one synchronisation.
    {
        struct Out { void* h; const void* d; size_t bytes; };
        const Out outs[20] = {{o->status, c->d_status, c->N}, {o->level, c->d_level, c->N},
                             {o->depth, c->d_depth, 2ull * c->N}, {o->instance, c->d_inst, 2ull * c->N},
                             {o->new_pin, c->d_newpin, c->N},
                             {o->wf_agg, c->d_wfagg, 4ull * NALAR_WF_AGG_FIELDS * c->W},
                             {o->i_load, c->d_iload, 4ull * c->I}, {o->i_spare, c->d_ispare, 4ull * c->I},
                             {o->i_assigned, c->d_iasg, 4ull * c->I},
                             {o->kv_hint, c->d_kvh, (size_t)c->W * c->T},
                             {o->kv_level, c->d_kvl, (size_t)c->W * c->T},
                             {o->kv_home, c->d_kvhome, 2ull * c->W * c->T},
                             {o->t_busy, c->d_tbusy, 4ull * c->T}, {o->t_capsum, c->d_tcap, 4ull * c->T},
                             {o->ra_kill, c->d_rakill, 2ull * c->T}, {o->ra_prov, c->d_raprov, 2ull * c->T},
                             {mig ? o->migrate_to : nullptr, c->d_migto, 2ull * c->N},
                             {mig ? o->i_mig_in : nullptr, c->d_migin, 4ull * c->I},
                             {mig ? o->i_mig_out : nullptr, c->d_migout, 4ull * c->I},
                             {c->batch_on ? o->batch_head : nullptr, c->d_bhead, 4ull * c->N}};
        const bool fbad = (o->status || o->level || o->depth || o->instance || o->new_pin ||
                           (mig && o->migrate_to) || (c->batch_on && o->batch_head)) && o->f_cap < c->N;
        const bool wbad = o->wf_agg && o->wf_cap < c->W;
        const bool ibad = (o->i_load || o->i_spare || o->i_assigned ||
                           (mig && (o->i_mig_in || o->i_mig_out))) && o->i_cap < c->I;
        const bool kbad = (o->kv_hint || o->kv_level || o->kv_home) && o->kv_cap < (size_t)c->W * c->T;
        const bool tbad = (o->t_busy || o->t_capsum || o->ra_kill || o->ra_prov) && o->t_cap < c->T;
        bool mapped = !(fbad || wbad || ibad || kbad || tbad);
        CopyBatch cb(st);
        const bool so = c->sout_on;      // nalar_step: K1 / K4 wrote these already
        for (const Out& q : outs) {
            if (!mapped || !q.h || !q.bytes) continue;
            if (so && (q.h == (void*)o->status || q.h == (void*)o->level || q.h == (void*)o->depth ||
                       q.h == (void*)o->instance || q.h == (void*)o->new_pin))
                continue;
            void* v = mapped_view(q.h);
            if (!v) mapped = false;
            else cb.p.seg[cb.p.n++] = CopySeg{q.d, v, (uint64_t)q.bytes};
        }
        void* v_row = o->assign_row ? mapped_view(o->assign_row) : nullptr;
        void* v_inst = o->assign_inst ? mapped_view(o->assign_inst) : nullptr;
        if ((o->assign_row && !v_row) || (o->assign_inst && !v_inst)) mapped = false;
        if (mapped) {
            cb.chunk_offsets();
            FetchParams f{};
            f.n_adm = c->d_scr + C_NUM;
            f.tot_loc = c->d_scr + C_NUM + c->Rmax;
            f.arow = c->d_arow;
            f.ainst = c->d_ainst;
            f.counters = c->d_scr;
            f.out_row = (uint32_t*)v_row;
            f.out_inst = (int16_t*)v_inst;
            f.out_counters = c->h_cnt_dev;
            f.R = c->assign_valid ? c->R : 0u;
            f.a_cap = o->a_cap;
            CK(launch_fetch(f, cb.p, st));
            CK(cudaStreamSynchronize(st));
            const uint32_t na = c->h_cnt[C_ASSIGNED];
            o->n_f = c->N; o->n_w = c->W; o->n_i = c->I; o->n_assigned = na;
            o->n_reassign = c->ra_on ? c->h_cnt[C_RA_PAIRS] : 0u;
            o->n_migrated = mig ? c->h_cnt[C_MIGRATED] : 0u;
            o->n_batches = c->batch_on ? c->h_cnt[C_BATCHES] : 0u;
            if ((o->assign_row || o->assign_inst) && o->a_cap < na)
                return fail(c, NALAR_E_SIZE, "output buffer too small");
            return NALAR_OK;
        }
    }
    CK(cudaMemcpyAsync(c->h_cnt, c->d_scr, C_NUM * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint32_t na = c->h_cnt[C_ASSIGNED];
    o->n_f = c->N; o->n_w = c->W; o->n_i = c->I; o->n_assigned = na;
    const bool fbad = (o->status || o->level || o->depth || o->instance || o->new_pin ||
                       (mig && o->migrate_to) || (c->batch_on && o->batch_head)) && o->f_cap < c->N;
    const bool wbad = o->wf_agg && o->wf_cap < c->W;
    const bool ibad = (o->i_load || o->i_spare || o->i_assigned ||
                       (mig && (o->i_mig_in || o->i_mig_out))) && o->i_cap < c->I;
    const bool abad = (o->assign_row || o->assign_inst) && o->a_cap < na;
    const bool kbad = (o->kv_hint || o->kv_level || o->kv_home) && o->kv_cap < (size_t)c->W * c->T;
    const bool tbad = (o->t_busy || o->t_capsum || o->ra_kill || o->ra_prov) && o->t_cap < c->T;
    if (fbad || wbad || ibad || abad || kbad || tbad) return fail(c, NALAR_E_SIZE, "output buffer too small");
    o->n_reassign = c->ra_on ? c->h_cnt[C_RA_PAIRS] : 0u;
    o->n_migrated = mig ? c->h_cnt[C_MIGRATED] : 0u;
    o->n_batches = c->batch_on ? c->h_cnt[C_BATCHES] : 0u;
    auto d2h = [&](void* h, const void* d, size_t bytes) -> cudaError_t {
        return (h && bytes) ? cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
    };
    CK(d2h(o->status, c->d_status, c->N));
    CK(d2h(o->level, c->d_level, c->N));
    CK(d2h(o->depth, c->d_depth, 2ull * c->N));
    CK(d2h(o->instance, c->d_inst, 2ull * c->N));
    CK(d2h(o->new_pin, c->d_newpin, c->N));
    CK(d2h(o->wf_agg, c->d_wfagg, 4ull * NALAR_WF_AGG_FIELDS * c->W));
    CK(d2h(o->kv_hint, c->d_kvh, (size_t)c->W * c->T));
    CK(d2h(o->kv_level, c->d_kvl, (size_t)c->W * c->T));
    CK(d2h(o->kv_home, c->d_kvhome, 2ull * c->W * c->T));
    CK(d2h(o->t_busy, c->d_tbusy, 4ull * c->T));
    CK(d2h(o->t_capsum, c->d_tcap, 4ull * c->T));
    CK(d2h(o->ra_kill, c->d_rakill, 2ull * c->T));
    CK(d2h(o->ra_prov, c->d_raprov, 2ull * c->T));
    if (mig) {
        CK(d2h(o->migrate_to, c->d_migto, 2ull * c->N));
        CK(d2h(o->i_mig_in, c->d_migin, 4ull * c->I));
        CK(d2h(o->i_mig_out, c->d_migout, 4ull * c->I));
    }
    if (c->batch_on) CK(d2h(o->batch_head, c->d_bhead, 4ull * c->N));
    CK(d2h(o->i_load, c->d_iload, 4ull * c->I));
    CK(d2h(o->i_spare, c->d_ispare, 4ull * c->I));
    CK(d2h(o->i_assigned, c->d_iasg, 4ull * c->I));
    // the assignment list lives in per-resource regions on the device
    // (region r = this rank's eligible futures of r); compact while copying
    const bool want_list = (o->assign_row || o->assign_inst) && na;
    if (want_list) {
        CK(cudaMemcpyAsync(c->h_reg, c->d_scr + C_NUM, 8ull * c->Rmax, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    if (want_list) {
        const uint32_t* n_adm = c->h_reg;
        const uint32_t* tot_loc = c->h_reg + c->Rmax;
        size_t n_el = 0;
        for (uint32_t r = 0; r < c->R; ++r) n_el += tot_loc[r];
        if (c->h_list_cap < n_el) {
            if (c->h_list) cudaFreeHost(c->h_list);
            c->h_list = nullptr;
            c->h_list_cap = 0;
            if (cudaMallocHost(&c->h_list, 6 * std::max<size_t>(n_el, 1)) != cudaSuccess)
                return fail(c, NALAR_E_NOMEM, "pinned staging for the assignment list");
            c->h_list_cap = n_el;
        }
        uint32_t* hr = (uint32_t*)c->h_list;
        int16_t* hi = (int16_t*)(hr + n_el);
        CK(cudaMemcpyAsync(hr, c->d_arow, 4 * n_el, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hi, c->d_ainst, 2 * n_el, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        size_t at = 0, out = 0;
        for (uint32_t r = 0; r < c->R; ++r) {
            if (o->assign_row) memcpy(o->assign_row + out, hr + at, 4ull * n_adm[r]);
            if (o->assign_inst) memcpy(o->assign_inst + out, hi + at, 2ull * n_adm[r]);
            out += n_adm[r];
            at += tot_loc[r];
        }
    }
    return NALAR_OK;
}

int nalar_set_policy_params(nalar_ctx* c, const nalar_policy_params* p) {
    if (!c || !p) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (p->u_lo_pct > p->u_hi_pct) return fail(c, NALAR_E_INVAL, "u_lo_pct > u_hi_pct");
    if (p->n_types > c->cfg.max_types) return fail(c, NALAR_E_INVAL, "n_types > max_types");
    std::vector<uint16_t> mn(c->cfg.max_types, 0), mx(c->cfg.max_types, 0xFFFF);
    for (uint32_t t = 0; t < p->n_types; ++t) {
        if (p->t_min_inst) mn[t] = p->t_min_inst[t];
        if (p->t_max_inst) mx[t] = p->t_max_inst[t];
    }
    CK(cudaMemcpyAsync(c->d_tmin, mn.data(), 2ull * mn.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_tmax, mx.data(), 2ull * mx.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    bool batch = false;
    std::vector<uint16_t> mbt(c->cfg.max_types, 0);
    for (uint32_t t = 0; p->t_max_batch && t < p->n_types; ++t) {
        mbt[t] = p->t_max_batch[t];
        batch |= mbt[t] > 1;
    }
    CK(cudaMemcpyAsync(c->d_tmaxb, mbt.data(), 2ull * mbt.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->batch_on = batch;
    c->h_tmaxb = mbt;
    c->ra_on = p->reassign ? 1u : 0u;
    c->u_hi = p->u_hi_pct;
    c->u_lo = p->u_lo_pct;
    c->mig_on = p->migrate ? 1u : 0u;
    c->theta_wait = p->theta_wait;
    c->theta_head = p->theta_head;
    c->mig_delta = p->delta;
    c->params_gen++;                      // epoch graphs bake the parameters in
    return NALAR_OK;
}

int nalar_epoch_stats_get(nalar_ctx* c, nalar_epoch_stats* s) {
    if (!c || !s) return NALAR_E_INVAL;
    DevGuard dg(c->cfg.device);
    if (!c->epoch_done) return fail(c, NALAR_E_STATE, "stats before epoch");
    memset(s, 0, sizeof *s);
    CK(cudaMemcpyAsync(c->h_cnt, c->d_scr, C_NUM * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (int rc = peer_check(c, NALAR_OK)) return rc;
    s->n_futures = c->N;
    s->n_ready = c->h_cnt[C_READY];
    s->n_eligible = c->h_cnt[C_ELIG];
    s->n_doomed = c->h_cnt[C_DOOMED];
    s->n_assigned = c->h_cnt[C_ASSIGNED];
    s->n_deferred = s->n_eligible - s->n_assigned;
    s->n_instances = c->I;
    if (c->cfg.flags & NALAR_F_TIMING) {
        CK(cudaEventElapsedTime(&s->epoch_us, c->ev[0], c->ev[3]));
        CK(cudaEventElapsedTime(&s->k1_us, c->ev[0], c->ev[1]));
        CK(cudaEventElapsedTime(&s->coll_us, c->ev[1], c->ev[2]));
        CK(cudaEventElapsedTime(&s->k4_us, c->ev[2], c->ev[3]));
        s->epoch_us *= 1000.f; s->k1_us *= 1000.f; s->coll_us *= 1000.f; s->k4_us *= 1000.f;
    }
    return NALAR_OK;
}

}  // extern "C"
