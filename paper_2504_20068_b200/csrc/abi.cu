// abi.cu -- libjitsched.so: the C ABI declared in include/jit_sched.h.
// Host side: validation, workspace carving, CUDA-graph capture of the step, result readback.
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <new>
#include <string>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include "jit_sched.h"
#include "common.cuh"
#include "select.cuh"
#include "match.cuh"
#include "stream.cuh"
#include "replay.cuh"
#include "shard.cuh"
#include "multi.cuh"

constexpr uint32_t kSpecFastCap = 256;   // k_spec's fast-path set size (spec.cuh kSpecFast)

#ifndef JIT_CMP_COST
#define JIT_CMP_COST 3
#endif
#include "exact_api.h"

using namespace jit;

static_assert(sizeof(jit_slo_group) == sizeof(Group), "group layout");

struct jit_sched {
    jit_config cfg{};
    Cfg c{};
    Table T{};
    Group* d_groups = nullptr;
    uint32_t n_groups = 0;
    Pool P{};
    Scratch S{};
    Item* d_items = nullptr;          // k_score work items (S.items), capacity item_cap
    uint32_t* d_n_items = nullptr;    // their count (S.n_items)
    uint32_t item_cap = 0;
    unsigned char* d_load = nullptr;  // load / per-step delta staging (48 B per row + 72 B per task of capacity)
    Ctrl* d_ctrl = nullptr;
    Ctrl* h_ctrl = nullptr;           // pinned
    uint32_t* h_batch = nullptr;      // pinned: the fast path writes the batch here (ids | tokens | rows)
    unsigned char* h_pin = nullptr;   // pinned staging of the per-step deltas (one H2D copy)
    uint64_t pin_cap = 0, load_bytes = 0, delta_h2d_bytes = 0;
    std::vector<unsigned char> h_delta;
    uint32_t n_items_host = 0;
    cudaStream_t stream = nullptr;    // caller's stream
    cudaStream_t cap = nullptr;       // private capture stream
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t score_node = nullptr;   // k_score: its (now, v) arguments change every step
    cudaKernelNodeParams score_params{};
    void* score_args[10];
    int arg_mode = 0;
    int64_t arg_now = 0, arg_v = 0;
    bool loaded = false, graph_dirty = true, timing = false, debug = false, pdl = true;
    float match_ms = 0.f;             // device time of the last k_match (jit_sched_last_match_ms)
    bool keys_ready = false;          // k_score already ran this step (fast sharded attempt)
    bool unfinished = false;          // a step was launched and not finished (step_async)
    uint64_t launched = 0;            // steps launched (the stamp rebase runs every 2^30)
    unsigned long long multi_epoch = 0;   // power-of-K reconciles so far (tags S.mwin words)
    uint32_t bal_w_graph = 0;             // S.bal_w captured in the step graph
    bool big_mode = false;                // the step graph chains k_spec_big_chain (large speculative sets)
    uint32_t small_streak = 0;            // consecutive finished steps whose set fit k_spec (leave big mode)
    cudaEvent_t ev[6] = {};
    cudaGraphNode_t ev_node[5] = {};      // event-record nodes of the timed graph
    std::vector<cudaEvent_t> slots;       // 5 events per recorded step
    uint32_t n_slots = 0, slot_used = 0;
    int n_sm = 148;
    uint32_t nb_score = 1, grid_pass = 1;
    std::vector<uint32_t> h_off;          // host copy of call_off (device-resident pools)
    std::vector<Item> h_items;
    std::string err;
};

// k_score instantiations: kMat (every key materialized: debug handles and the exact path's
// re-score) x kDebug (per-row debug outputs) x App. B feasibility filter
static const void* score_fn(bool mat, bool debug, bool appb) {
    if (debug) return appb ? (const void*)k_score<true, true, true> : (const void*)k_score<true, true, false>;
    if (mat) return appb ? (const void*)k_score<true, false, true> : (const void*)k_score<true, false, false>;
    return appb ? (const void*)k_score<false, false, true> : (const void*)k_score<false, false, false>;
}

static int set_err(jit_sched* h, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) h->err = buf;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return set_err(h, JIT_ECUDA, "%s: %s (%s:%d)", #call,          \
                                              cudaGetErrorString(e_), __FILE__, __LINE__);    \
    } while (0)

// ------------------------------------------------------------------------------------------
// workspace layout
// ------------------------------------------------------------------------------------------
struct Carve {
    uint64_t off = 0;
    unsigned char* base = nullptr;
    template <typename T>
    T* take(uint64_t count) {
        off = (off + 255) & ~255ull;
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += sizeof(T) * count;
        return p;
    }
};

// items of k_score for `cap` rows / `tcap` tasks: standalone chunks + one per task at most + slack
static uint32_t item_capacity(uint64_t cap, uint64_t tcap) { return (uint32_t)(cap / kItemRows + tcap + 64); }

static void carve(Carve& cv, const jit_config* cfg, const jit_len_table* tab, Pool& P, Scratch& S, Table& T,
                  Group*& groups, Ctrl*& ctrl, Item*& items, uint32_t*& n_items, unsigned char*& load) {
    const uint64_t N = ((uint64_t)cfg->capacity + 63) & ~63ull;
    const uint64_t NT = (uint64_t)cfg->task_capacity + 1;
    const bool dbg = (cfg->flags & JIT_CFG_DEBUG_ROWS) != 0;
    // what every step touches first, packed together ahead of the pool (few pages: the step's
    // first loads and the resolve stay on a handful of TLB entries): control state, SLO groups, the
    // speculative set, the batch, the work items; then the hot rows and the compound pass's task
    // arrays; the exact path's and the loaders' scratch last
    S.persist = cv.take<Persist>(1);
    S.spec_cnt = cv.take<unsigned int>(1);
    S.gpart = cv.take<BlockPart>(1);
    ctrl = cv.take<Ctrl>(1);
    n_items = cv.take<uint32_t>(1);
    groups = cv.take<Group>(256);
    S.out_ids = cv.take<uint32_t>(cfg->max_batch + 1); S.out_tokens = cv.take<uint32_t>(cfg->max_batch + 1);
    S.out_rows = cv.take<uint32_t>(cfg->max_batch + 1);
    S.spec_img = cv.take<uint64_t>(kSpecCap);
    S.spec_id = cv.take<uint32_t>(kSpecCap); S.spec_row = cv.take<uint32_t>(kSpecCap);
    S.spec_cost = cv.take<uint32_t>(kSpecCap); S.spec_len = cv.take<uint32_t>(kSpecCap);
    S.spec_meta = cv.take<uint32_t>(kSpecCap); S.spec_aux = cv.take<uint32_t>(kSpecCap);
    items = cv.take<Item>(item_capacity(N, NT));
    S.items = items; S.n_items = n_items;
    P.rows = cv.take<HotRow>(N);
    P.task = cv.take<uint32_t>(N);
    P.call_off = cv.take<uint32_t>(NT + 8);
    P.tinfo = cv.take<TaskInfo>(NT); P.tever = cv.take<uint32_t>(NT + 4);   // + bulk-copy padding
    P.crng = cv.take<uint2>(NT + 2);
    P.id = cv.take<uint32_t>(N); P.ovr = cv.take<uint32_t>(N);
    P.fair = cv.take<uint32_t>(N);
    P.img = cv.take<uint64_t>(N); P.cost = cv.take<uint32_t>(N);
    P.dbg_rate = dbg ? cv.take<double>(N) : nullptr;
    P.dbg_trem = dbg ? cv.take<int64_t>(N) : nullptr;
    P.dbg_lhat = dbg ? cv.take<uint32_t>(N) : nullptr;
    P.t_arr = cv.take<int64_t>(NT); P.t_dl = cv.take<int64_t>(NT);
    P.cur_stage = cv.take<uint32_t>(NT); P.n_stages = cv.take<uint32_t>(NT);
    P.pattern = cv.take<uint32_t>(NT * kMaxStages); P.gdone = cv.take<uint64_t>(NT);
    uint64_t mc = 1024;
    while (mc < 2 * N) mc <<= 1;
    P.idmap = cv.take<unsigned long long>(mc);
    P.map_mask = (uint32_t)(mc - 1);
    T.edges = cv.take<uint32_t>(tab->n_bins);
    T.cum = cv.take<uint32_t>((uint64_t)tab->n_rows * tab->n_bins);
    T.lhat0 = cv.take<uint32_t>(tab->n_rows);
    S.hcnt = cv.take<uint32_t>(4096); S.hcost = cv.take<unsigned long long>(4096);
    S.bucket_ck = cv.take<u128>(kBucketCap); S.bucket_cost = cv.take<uint32_t>(kBucketCap);
    uint64_t P2 = 1;                       // bitonic sorts pad |Cd| to a power of two
    while (P2 < N) P2 <<= 1;
    S.cand = cv.take<uint32_t>(N); S.sk = cv.take<uint64_t>(P2); S.sv = cv.take<uint32_t>(P2);
    S.pc = cv.take<unsigned long long>(N + 1);
    S.pf = cv.take<u128>(P2 + 1);          // also the u128 sort keys of the shard merge (pow2 slots)
    S.cand_cap = (uint32_t)N;
    S.mwin = cv.take<unsigned long long>(N);
    // load / per-step delta staging: 48 B per row (the SoA fields of jit_pool) + 72 B per task
    load = cv.take<unsigned char>(48 * N + 72 * NT + 256);
}
// staging layout of a jit_pool's arrays (rows of capacity N, tasks of capacity NT)
struct Stage {
    int64_t* arr; uint32_t *len_in, *gen, *pre, *meta, *aux, *id, *task, *ovr;
    uint32_t* call_off; int64_t *t_arr, *t_dl; uint32_t *cur_stage, *n_stages, *pattern; uint64_t* gdone;
};
static Stage stage_layout(unsigned char* base, uint64_t N, uint64_t NT) {
    Stage st;
    st.arr = reinterpret_cast<int64_t*>(base);
    uint32_t* u = reinterpret_cast<uint32_t*>(base + 8 * N);
    st.len_in = u; st.gen = u + N; st.pre = u + 2 * N; st.meta = u + 3 * N; st.aux = u + 4 * N; st.id = u + 5 * N;
    st.task = u + 6 * N; st.ovr = u + 7 * N;
    unsigned char* t = base + 40 * N;
    st.t_arr = reinterpret_cast<int64_t*>(t); st.t_dl = st.t_arr + NT; st.gdone = reinterpret_cast<uint64_t*>(st.t_dl + NT);
    uint32_t* tu = reinterpret_cast<uint32_t*>(st.gdone + NT);
    st.cur_stage = tu; st.n_stages = tu + NT; st.call_off = tu + 2 * NT; st.pattern = tu + 3 * NT + 8;
    return st;
}

static int check_config(jit_sched* h, const jit_config* c, const jit_len_table* t) {
    if (!c || !t) return set_err(h, JIT_EINVAL, "null config/table");
    if (c->capacity == 0 || c->capacity > (1u << 30)) return set_err(h, JIT_EINVAL, "capacity out of range");
    if (c->refine_interval == 0 || c->frame_steps == 0 || c->q_den == 0 || c->q_num == 0 || c->q_num > c->q_den ||
        c->p_den == 0 || c->p_num == 0 || c->p_num > c->p_den || c->prefill_chunk == 0 ||
        c->prefill_chunk > c->token_budget || c->max_batch == 0 || c->eps_ns <= 0 || c->eps_ns >= (1ll << 36) ||
        c->waiting_ns < 0 || (c->preempt && (c->pmtn_den == 0 || c->io_bw_tps == 0)) ||
        (c->fair_num && c->fair_num > c->fair_den))
        return set_err(h, JIT_EINVAL, "invalid scheduler constants (ConfigError, S:417)");
    if (t->n_rows == 0 || t->n_rows > 65536 || t->n_bins == 0 || t->l_max == 0 || t->l_max >= 65536)
        return set_err(h, JIT_EINVAL, "invalid length table shape");
    return JIT_OK;
}

extern "C" int jit_sched_workspace_bytes(const jit_config* cfg, const jit_len_table* table, uint64_t* bytes) {
    int rc = check_config(nullptr, cfg, table);
    if (rc) return rc;
    Carve cv;
    Pool P; Scratch S; Table T; Group* g; Ctrl* c; Item* it; uint32_t* ni; unsigned char* ld;
    carve(cv, cfg, table, P, S, T, g, c, it, ni, ld);
    *bytes = cv.off + 256;
    return JIT_OK;
}

extern "C" int jit_sched_init(const jit_config* cfg, const jit_slo_group* groups, uint32_t n_groups,
                              const jit_len_table* table, void* dev_workspace, uint64_t ws_bytes, jit_sched** out) {
    if (!out) return JIT_EINVAL;
    *out = nullptr;
    jit_sched* h = new (std::nothrow) jit_sched();
    if (!h) return JIT_ECAPACITY;
    int rc = check_config(h, cfg, table);
    if (rc) { *out = h; return rc; }
    if (!groups || n_groups == 0 || n_groups > 256) { *out = h; return set_err(h, JIT_EINVAL, "n_groups must be 1..256"); }
    // table sanity (host): edges strictly increasing, last = l_max; rows nondecreasing
    for (uint32_t k = 0; k < table->n_bins; ++k) {
        if ((k == 0 && table->edges[0] == 0) || (k > 0 && table->edges[k] <= table->edges[k - 1])) {
            *out = h; return set_err(h, JIT_EINVAL, "table edges not strictly increasing");
        }
    }
    if (table->edges[table->n_bins - 1] != table->l_max) { *out = h; return set_err(h, JIT_EINVAL, "edges[last] != l_max"); }
    for (uint32_t r = 0; r < table->n_rows; ++r)
        for (uint32_t k = 1; k < table->n_bins; ++k)
            if (table->cum[(size_t)r * table->n_bins + k] < table->cum[(size_t)r * table->n_bins + k - 1]) {
                *out = h; return set_err(h, JIT_EINVAL, "table row %u not monotone", r);
            }
    for (uint32_t g = 0; g < n_groups; ++g) {
        if (groups[g].type > JIT_BE || groups[g].ttft_ns < 0 || groups[g].tbt_ns < 0 || groups[g].e2el_ns < 0 ||
            groups[g].be_deadline_ns < 0) { *out = h; return set_err(h, JIT_EINVAL, "bad SLO group %u", g); }
        // the pass forms (Lhat - 1) * TBT as one 32 x 32-bit product: TBT < 2^32 ns (4.29 s)
        if (groups[g].type == JIT_LAT && groups[g].tbt_ns >= (1ll << 32)) {
            *out = h; return set_err(h, JIT_EINVAL, "SLO group %u: TBT must be < 2^32 ns", g);
        }
    }
    uint64_t need = 0;
    jit_sched_workspace_bytes(cfg, table, &need);
    if (!dev_workspace || ws_bytes < need) { *out = h; return set_err(h, JIT_ECAPACITY, "workspace too small (%llu < %llu)",
                                                                       (unsigned long long)ws_bytes, (unsigned long long)need); }
    h->cfg = *cfg;
    h->debug = (cfg->flags & JIT_CFG_DEBUG_ROWS) != 0;
    *out = h;
    CK(cudaSetDevice(cfg->device));
    CK(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, cfg->device));
    h->stream = (cudaStream_t)cfg->stream;
    CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    // zero the workspace once: SoA padding rows (read by whole-quad tile loads, then masked) and
    // every scratch array start defined
    CK(cudaMemsetAsync(dev_workspace, 0, ws_bytes, h->stream));
    Carve cv;
    cv.base = reinterpret_cast<unsigned char*>(((uintptr_t)dev_workspace + 255) & ~(uintptr_t)255);
    carve(cv, cfg, table, h->P, h->S, h->T, h->d_groups, h->d_ctrl, h->d_items, h->d_n_items, h->d_load);
    h->item_cap = item_capacity(((uint64_t)cfg->capacity + 63) & ~63ull, (uint64_t)cfg->task_capacity + 1);
    h->load_bytes = 48 * (((uint64_t)cfg->capacity + 63) & ~63ull) + 72 * ((uint64_t)cfg->task_capacity + 1);
    h->S.item_cap = h->item_cap;
    h->T.n_rows = table->n_rows; h->T.n_bins = table->n_bins; h->T.l_max = table->l_max;
    h->T.unit = 1;
    for (uint32_t k = 0; k < table->n_bins && h->T.unit; ++k) h->T.unit = table->edges[k] == k + 1;
    h->n_groups = n_groups;
    Cfg& c = h->c;
    c.token_budget = cfg->token_budget; c.max_batch = cfg->max_batch; c.chunk = cfg->prefill_chunk;
    c.R = cfg->refine_interval; c.frame = cfg->frame_steps; c.qn = cfg->q_num; c.qd = cfg->q_den;
    c.pn = cfg->p_num; c.pd = cfg->p_den; c.delta = cfg->delta_starve; c.len_key = cfg->len_key;
    c.appb = cfg->appb_filter; c.eps = cfg->eps_ns; c.waiting = cfg->waiting_ns;
    c.p = (double)c.pn / (double)c.pd;      // IEEE division, correctly rounded like __ddiv_rn
    fastdiv_magic(c.R, &c.R_m, &c.R_l);
    fastdiv_magic(c.frame, &c.F_m, &c.F_l);
    c.preempt = cfg->preempt ? 1u : 0u; c.pmtn_num = cfg->pmtn_num; c.pmtn_den = cfg->pmtn_den ? cfg->pmtn_den : 1u;
    c.io_bw = cfg->io_bw_tps ? cfg->io_bw_tps : 1ull;
    c.onepd = (double)((uint64_t)c.pmtn_den + c.pmtn_num) / (double)c.pmtn_den;   // one IEEE division
    c.fair_num = cfg->fair_num; c.fair_den = cfg->fair_num ? cfg->fair_den : 1u;
    CK(cudaMemcpyAsync((void*)h->T.edges, table->edges, 4ull * table->n_bins, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync((void*)h->T.cum, table->cum, 4ull * table->n_rows * table->n_bins, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_groups, groups, sizeof(Group) * n_groups, cudaMemcpyHostToDevice, h->stream));
    // every table row's bound at anchor 0 (the rows with g < R: seeded at load / arrival)
    k_lhat0<<<(table->n_rows + 127) / 128, 128, 0, h->stream>>>(h->T, c.qn, c.qd);
    CK(cudaGetLastError());
    CK(cudaMallocHost(&h->h_ctrl, sizeof(Ctrl)));
    CK(cudaMallocHost(&h->h_batch, 3ull * 4 * (cfg->max_batch + 1)));
    h->S.h_batch = h->h_batch;
    memset(h->h_ctrl, 0, sizeof(Ctrl));
    h->S.h_ctrl = h->h_ctrl;              // pinned + mapped (UVA): the step's last kernel writes it
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
    CK(exact::init_attributes());
    CK(cudaFuncSetAttribute(k_group_rec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(12 * kGroupSmemSort)));
    // one shared-memory carveout for every kernel of the step: switching the L1/shared split
    // between consecutive kernels costs a drain + reconfiguration of the SMs (several µs each)
    for (int m = 0; m < 8; ++m) {
        const void* k = score_fn(m & 1, m & 2, m & 4);
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)score_smem_bytes(256)));
        CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    }
    CK(cudaFuncSetAttribute(k_begin, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    {
        Persist ps{};
        ps.t_guess = kNone;                 // no speculation before the first resolved step
        CK(cudaMemcpyAsync(h->S.persist, &ps, sizeof ps, cudaMemcpyHostToDevice, h->stream));
        BlockPart g{};                      // the empty step record (k_spec resets it after reading)
        CK(cudaMemcpyAsync(h->S.gpart, &g, sizeof g, cudaMemcpyHostToDevice, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    return JIT_OK;
}

// ------------------------------------------------------------------------------------------
// load
// ------------------------------------------------------------------------------------------
// compound work items: whole tasks [t0, t0 + nt) (call rows [r0 + off[t], r0 + off[t + 1]) with
// off relative) packed greedily into items of at most kItemRows rows and kItemTasks tasks; a task
// of more calls gets an item of its own (read in chunks)
static void add_task_items(std::vector<Item>& items, const uint32_t* off, uint32_t r0, uint32_t t0, uint32_t nt) {
    Item cur{r0 + off[0], r0 + off[0], t0, t0};
    for (uint32_t t = 0; t < nt; ++t) {
        if (t0 + t > cur.t0 && (r0 + off[t + 1] - cur.r0 > kItemRows || t0 + t - cur.t0 >= kItemTasks)) {
            cur.r1 = r0 + off[t]; cur.t1 = t0 + t;
            items.push_back(cur);
            cur.r0 = r0 + off[t]; cur.t0 = t0 + t;
        }
    }
    cur.r1 = r0 + off[nt]; cur.t1 = t0 + nt;
    items.push_back(cur);
}

extern "C" int jit_sched_load(jit_sched* h, const jit_pool* p) {
    if (!h || !p) return JIT_EINVAL;
    if (p->n > h->cfg.capacity || p->n_tasks > h->cfg.task_capacity)
        return set_err(h, JIT_ECAPACITY, "pool of %u rows / %u tasks exceeds capacity", p->n, p->n_tasks);
    if (p->n_single > p->n) return set_err(h, JIT_EINVAL, "n_single > n");
    if (p->n_tasks && (!p->call_off || !p->task_arrival_ns || !p->task_deadline_ns || !p->cur_stage ||
                       !p->n_stages || !p->pattern_ms || !p->goodput_done))
        return set_err(h, JIT_EINVAL, "missing task arrays");
    if (h->unfinished) return set_err(h, JIT_ESTATE, "load while a step is unfinished (fetch its batch first)");
    const cudaMemcpyKind kind = p->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    Pool& P = h->P;
    const uint64_t n = p->n, nt = p->n_tasks;
    const uint64_t N = ((uint64_t)h->cfg.capacity + 63) & ~63ull;
    if (n) {
        // the hot fields go through the staging area (or are read in place from a device pool)
        // and are packed into 32-byte rows; the cold per-row arrays are copied as they are
        const int64_t* arr = p->arrival_ns;
        const uint32_t *li = p->input_len, *ge = p->generated, *pr = p->prefilled, *me = p->meta, *ax = p->aux;
        if (!p->on_device) {
            int64_t* s_arr = reinterpret_cast<int64_t*>(h->d_load);
            uint32_t* s_u = reinterpret_cast<uint32_t*>(h->d_load + 8 * N);
            CK(cudaMemcpyAsync(s_arr, p->arrival_ns, 8 * n, kind, h->stream));
            CK(cudaMemcpyAsync(s_u, p->input_len, 4 * n, kind, h->stream));
            CK(cudaMemcpyAsync(s_u + N, p->generated, 4 * n, kind, h->stream));
            CK(cudaMemcpyAsync(s_u + 2 * N, p->prefilled, 4 * n, kind, h->stream));
            CK(cudaMemcpyAsync(s_u + 3 * N, p->meta, 4 * n, kind, h->stream));
            CK(cudaMemcpyAsync(s_u + 4 * N, p->aux, 4 * n, kind, h->stream));
            arr = s_arr; li = s_u; ge = s_u + N; pr = s_u + 2 * N; me = s_u + 3 * N; ax = s_u + 4 * N;
        }
        k_pack<<<(uint32_t)std::min<uint64_t>((n + 255) / 256, (uint64_t)h->n_sm * 16), 256, 0, h->stream>>>(
            P.rows, (uint32_t)n, arr, li, ge, pr, me, ax);
        CK(cudaMemcpyAsync(P.id, p->id, 4 * n, kind, h->stream));
        CK(cudaMemcpyAsync(P.task, p->task, 4 * n, kind, h->stream));
        CK(cudaMemcpyAsync(P.ovr, p->override_R, 4 * n, kind, h->stream));
        if (p->fair) CK(cudaMemcpyAsync(P.fair, p->fair, 4 * n, kind, h->stream));
        else CK(cudaMemsetAsync(P.fair, 0, 4 * n, h->stream));
    }
    if (nt) {
        CK(cudaMemcpyAsync(P.call_off, p->call_off, 4 * (nt + 1), kind, h->stream));
        CK(cudaMemcpyAsync(P.t_arr, p->task_arrival_ns, 8 * nt, kind, h->stream));
        CK(cudaMemcpyAsync(P.t_dl, p->task_deadline_ns, 8 * nt, kind, h->stream));
        CK(cudaMemcpyAsync(P.cur_stage, p->cur_stage, 4 * nt, kind, h->stream));
        CK(cudaMemcpyAsync(P.n_stages, p->n_stages, 4 * nt, kind, h->stream));
        CK(cudaMemcpyAsync(P.pattern, p->pattern_ms, 4 * nt * kMaxStages, kind, h->stream));
        CK(cudaMemcpyAsync(P.gdone, p->goodput_done, 8 * nt, kind, h->stream));
    }
    P.n = p->n; P.n_single = p->n_single; P.n_tasks = p->n_tasks;
    // full reset: control block, histograms, the speculative-set counter; validate on the device
    // (also covers device-resident pools)
    k_begin<<<4, 1024, 0, h->stream>>>(h->d_ctrl, h->S.hcnt, h->S.hcost, 0, 1, h->S.spec_cnt);
    CK(cudaMemsetAsync(h->S.gpart, 0, sizeof(BlockPart), h->stream));
    const uint32_t vb = (uint32_t)std::min<uint64_t>((n + 255) / 256 + 1, (uint64_t)h->n_sm * 8);
    if (nt) k_crng_from_off<<<(uint32_t)std::min<uint64_t>((nt + 255) / 256, (uint64_t)h->n_sm * 8), 256, 0, h->stream>>>(P);
    k_validate<<<vb, 256, 0, h->stream>>>(P, h->d_groups, h->n_groups, h->T.n_rows, h->T.l_max, &h->d_ctrl->error, 0u,
                                          P.n_single, 0u, h->T.forest ? nullptr : h->T.lhat0, h->c.R);
    if (nt) k_task_prep<<<(uint32_t)std::min<uint64_t>((nt + 255) / 256, (uint64_t)h->n_sm * 8), 256, 0, h->stream>>>(P, 0u);
    // request id -> row map (the progress of a step is keyed by id)
    CK(cudaMemsetAsync(P.idmap, 0xFF, 8ull * (P.map_mask + 1ull), h->stream));
    if (n) k_map_insert<<<vb, 256, 0, h->stream>>>(P, 0u, (uint32_t)n, &h->d_ctrl->error);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctrl, h->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->h_ctrl->error) { h->loaded = false; return set_err(h, JIT_EINVAL, "invalid pool (layout / ranges / groups)"); }
    // work items of k_score: the standalone rows in chunks of kItemRows (their descriptors are
    // arithmetic in the kernel), then the compound tasks
    h->h_items.clear();
    for (uint32_t r0 = 0; r0 < P.n_single; r0 += kItemRows)
        h->h_items.push_back(Item{r0, std::min<uint32_t>(r0 + kItemRows, P.n_single), 0u, 0u});
    h->S.n_std_items = (uint32_t)h->h_items.size();
    if (nt) {
        const uint32_t* off = p->call_off;
        if (p->on_device) {
            h->h_off.resize(nt + 1);
            CK(cudaMemcpy(h->h_off.data(), p->call_off, 4 * (nt + 1), cudaMemcpyDeviceToHost));
            off = h->h_off.data();
        }
        add_task_items(h->h_items, off, 0u, 0u, (uint32_t)nt);
    }
    if (h->h_items.size() > h->item_cap) return set_err(h, JIT_ECAPACITY, "too many work items");
    const uint32_t n_items = (uint32_t)h->h_items.size();
    h->n_items_host = n_items;
    h->S.n_ring_h = n_items - h->S.n_std_items;
    // a compound call costs k_score about JIT_CMP_COST standalone rows (profiles: per-row
    // instruction counts); the standalone slabs are spread against the ring items accordingly
    {
        const uint64_t n_ring = n_items - h->S.n_std_items, n_cmp = (uint64_t)P.n - P.n_single;
        h->S.bal_w = n_ring ? (uint32_t)std::min<uint64_t>(1u << 24, 256ull * JIT_CMP_COST * n_cmp / (32ull * n_ring)) : 0u;
        if (h->S.bal_w != h->bal_w_graph) h->graph_dirty = true;
        h->bal_w_graph = h->S.bal_w;
    }
    if (n_items)
        CK(cudaMemcpyAsync(h->d_items, h->h_items.data(), sizeof(Item) * n_items, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_n_items, &h->n_items_host, 4, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    // persistent grid: every CTA that fits on the GPU (warps stride over the items), at most one
    // warp per item
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score_fn(h->debug, h->debug, h->c.appb != 0), kScoreThreads,
                                                     score_smem_bytes(h->n_groups)));
    const uint32_t nb = std::max<uint32_t>(1, std::min<uint32_t>((n_items + kScoreWarps - 1) / kScoreWarps,
                                                                 (uint32_t)h->n_sm * (uint32_t)std::max(occ, 1)));
    if (nb != h->nb_score) h->graph_dirty = true;
    h->nb_score = nb;
    h->grid_pass = std::max<uint32_t>(1, std::min<uint32_t>((P.n + kPassThreads - 1) / kPassThreads, (uint32_t)h->n_sm * 4));
    h->loaded = true;
    return JIT_OK;
}

// ------------------------------------------------------------------------------------------
// step
// ------------------------------------------------------------------------------------------
// mode 0: the step's pass (debug handles materialize every key); mode 1: the exact path's re-score
// (every key materialized, nothing counted again)
static void enqueue_score(jit_sched* h, cudaStream_t s, int64_t now, int64_t v, cudaEvent_t mid = nullptr,
                          bool capturing = false, int mode = 0) {
    Pool& P = h->P;
    Scratch& S = h->S;
    void* args[] = {&P, &h->T, &h->d_groups, &h->n_groups, &h->c, &h->d_ctrl, &S, &now, &v, &mode};
    cudaLaunchKernel(score_fn(h->debug || mode == 1, h->debug, h->c.appb != 0), dim3(h->nb_score), dim3(kScoreThreads),
                     args, score_smem_bytes(h->n_groups), s);
    if (mid) cudaEventRecordWithFlags(mid, s, capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

// host-side continuation of the radix select (only for heavy key ties, see finish_step)
static void enqueue_radix(jit_sched* h, cudaStream_t s, uint32_t first_pass, uint32_t n_passes) {
    Pool& P = h->P;
    Scratch& S = h->S;
    for (uint32_t i = 0; i < n_passes; ++i) exact::pass(P, h->c, h->d_ctrl, S, h->grid_pass, first_pass + i, s);
    exact::compact(P, h->c, h->d_ctrl, S, h->grid_pass, s);
    exact::resolve(P, h->c, h->d_ctrl, S, s);
    exact::cand(P, h->c, h->d_ctrl, S, h->grid_pass, 0, s);
    exact::group(P, h->c, h->d_ctrl, S, s);
}

// Step graph: k_score -> k_spec, two kernel nodes and nothing else.  k_score resets the control
// block; k_spec (programmatic dependent launch: its launch overlaps k_score) resolves the batch
// and copies the control block to pinned host memory.  When the speculative resolve cannot be
// exact (or the set is large), the status says so and finish_step runs the exact path from the
// host -- no device-side launches, no conditional or copy nodes (their fixed costs measured
// ~26 us and ~6 us per step on B200, profiles/host_overhead.py).  With kernel timing on,
// event-record nodes separate the kernels (full dependencies, no PDL).
// (Resolving inside k_score's last CTA instead was measured slower on B200: the resolve is
// latency-bound, ran ~40% slower in a 256-thread k_score CTA, and its code slowed k_score.)
static int build_graph(jit_sched* h) {
    if (h->exec) { cudaGraphExecDestroy(h->exec); h->exec = nullptr; }
    if (h->graph) { cudaGraphDestroy(h->graph); h->graph = nullptr; }
    cudaGraph_t g;
    cudaStream_t s = h->cap;
    Scratch& S = h->S;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    if (h->timing) cudaEventRecordWithFlags(h->ev[0], s, cudaEventRecordExternal);
    enqueue_score(h, s, 0, 1, h->timing ? h->ev[1] : nullptr, true);
    if (h->timing) cudaEventRecordWithFlags(h->ev[2], s, cudaEventRecordExternal);
    const cudaError_t le = exact::spec(h->P, h->c, h->d_ctrl, S, 0, s, !h->timing && h->pdl, h->big_mode);
    if (h->timing) {
        cudaEventRecordWithFlags(h->ev[3], s, cudaEventRecordExternal);
        cudaEventRecordWithFlags(h->ev[4], s, cudaEventRecordExternal);
    }
    if (le != cudaSuccess) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        (void)cudaGetLastError();
        if (h->pdl) { h->pdl = false; return build_graph(h); }   // no PDL in graphs here: plain edge
        return set_err(h, JIT_ECUDA, "graph capture of k_spec: %s", cudaGetErrorString(le));
    }
    CK(cudaStreamEndCapture(s, &g));
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    // locate the k_score kernel node (its (now, v) arguments are updated per launch) and the
    // timing event nodes
    const void* score_kernel = score_fn(h->debug, h->debug, h->c.appb != 0);
    h->score_node = nullptr;
    for (auto& e : h->ev_node) e = nullptr;
    for (auto nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess) { (void)cudaGetLastError(); continue; }
        if (ty == cudaGraphNodeTypeKernel && !h->score_node) {
            cudaKernelNodeParams kp;
            if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) { (void)cudaGetLastError(); continue; }
            if (kp.func == score_kernel) { h->score_node = nd; h->score_params = kp; }
        } else if (ty == cudaGraphNodeTypeEventRecord) {
            cudaEvent_t e;
            if (cudaGraphEventRecordNodeGetEvent(nd, &e) != cudaSuccess) { (void)cudaGetLastError(); continue; }
            for (int i = 0; i < 5; ++i) if (e == h->ev[i]) h->ev_node[i] = nd;
        }
    }
    (void)cudaGetLastError();
    if (!h->score_node) { cudaGraphDestroy(g); return set_err(h, JIT_ECUDA, "graph: k_score node not found"); }
    h->graph = g;                      // kept alive: score_node belongs to it
    CK(cudaGraphInstantiate(&h->exec, g, 0));
    h->graph_dirty = false;
    return JIT_OK;
}

// JIT_CFG_NO_GRAPH: the same kernels as direct launches (for profilers)
static int launch_direct(jit_sched* h, int64_t now, int64_t v) {
    cudaStream_t s = h->stream;
    const bool ev = h->timing && h->n_slots;
    cudaEvent_t* e = ev ? &h->slots[5 * (h->slot_used % h->n_slots)] : nullptr;
    if (ev) h->slot_used++;
    if (ev) cudaEventRecord(e[0], s);
    enqueue_score(h, s, now, v, ev ? e[1] : nullptr, false);
    if (ev) cudaEventRecord(e[2], s);
    CK(exact::spec(h->P, h->c, h->d_ctrl, h->S, 0, s, !ev && h->pdl, h->big_mode));
    if (ev) { cudaEventRecord(e[3], s); cudaEventRecord(e[4], s); }
    CK(cudaGetLastError());
    return JIT_OK;
}

static int launch_step(jit_sched* h, int64_t now, int64_t v, bool chain = false) {
    if (h->unfinished && !chain)
        return set_err(h, JIT_ESTATE, "a step_async step is unfinished: fetch its batch before a synchronous step");
    // every 2^30 steps: keep the steps_waited stamps of long-waiting rows within reach (pool.cuh)
    if (((++h->launched) & ((1ull << 30) - 1)) == 0 && h->P.n)
        k_rebase<<<h->grid_pass, 256, 0, h->stream>>>(h->P, h->S);
    h->unfinished = true;
    h->arg_now = now; h->arg_v = v; h->arg_mode = 0;
    if (h->cfg.flags & JIT_CFG_NO_GRAPH) return launch_direct(h, now, v);
    if (h->graph_dirty) {
        CK(cudaGetLastError());
        int rc = build_graph(h);
        if (rc) return rc;
        CK(cudaGetLastError());
    }
    h->arg_now = now; h->arg_v = v; h->arg_mode = 0;
    void** a = h->score_args;     // k_score(Pool, Table, const Group*, uint32_t, Cfg, Ctrl*, Scratch, now, v, mode)
    a[0] = &h->P; a[1] = &h->T; a[2] = &h->d_groups; a[3] = &h->n_groups; a[4] = &h->c; a[5] = &h->d_ctrl;
    a[6] = &h->S; a[7] = &h->arg_now; a[8] = &h->arg_v; a[9] = &h->arg_mode;
    cudaKernelNodeParams kp = h->score_params;
    kp.kernelParams = a;
    kp.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(h->exec, h->score_node, &kp));
    if (h->timing && h->n_slots) {
        // point the graph's event nodes at this step's slot so every timed step keeps its times
        const uint32_t slot = h->slot_used % h->n_slots;
        for (int i = 0; i < 5; ++i)
            if (h->ev_node[i]) CK(cudaGraphExecEventRecordNodeSetEvent(h->exec, h->ev_node[i], h->slots[5 * slot + i]));
        h->slot_used++;
    }
    CK(cudaGetLastError());
    CK(cudaGraphLaunch(h->exec, h->stream));
    CK(cudaGetLastError());
    return JIT_OK;
}

// the exact path from the host (rare): re-score the pool with every key and cost materialized
// (same step counter and pool state: the pass is idempotent), then the cost-weighted radix select
static void enqueue_exact(jit_sched* h, cudaStream_t s) {
    enqueue_score(h, s, h->arg_now, h->arg_v, nullptr, false, 1);
    cudaMemsetAsync(h->S.hcnt, 0, 4 * 4096, s);
    cudaMemsetAsync(h->S.hcost, 0, 8 * 4096, s);
    exact::hist0(h->P, h->c, h->d_ctrl, h->S, h->grid_pass, 0, s);
    enqueue_radix(h, s, 0, kLevels - 1);
}

static int finish_step_body(jit_sched* h, jit_batch* out) {
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaGetLastError());
    if (getenv("JITSCHED_DEBUG_CTRL")) {
        Ctrl dc;
        CK(cudaMemcpy(&dc, h->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
        fprintf(stderr, "[ctrl] device status %u err %u fb %u spec %u trace %x | host status %u err %u fb %u spec %u\n",
                dc.status, dc.error, dc.fallback, dc.spec_n, dc.trace, h->h_ctrl->status, h->h_ctrl->error,
                h->h_ctrl->fallback, h->h_ctrl->spec_n);
    }
    if (h->h_ctrl->status == ST_SPEC_BIG) {
        // a speculative set too large for k_spec's fast path (e.g. after a shift of the keys): resolve
        // it now, and chain the big-set resolve in the step graph from here on (big mode) so that
        // such steps stay on the device
        exact::spec_big(h->P, h->c, h->d_ctrl, h->S, h->stream);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
        if (!h->big_mode) { h->big_mode = true; h->graph_dirty = true; }
        h->small_streak = 0;
    } else if (h->big_mode) {                             // back to the lean graph after 8 small sets
        if (h->h_ctrl->spec_n <= kSpecFastCap) {
            if (++h->small_streak >= 8) { h->big_mode = false; h->graph_dirty = true; h->small_streak = 0; }
        } else {
            h->small_streak = 0;
        }
    }
    const uint32_t st0 = h->h_ctrl->status;
    const bool host_work = st0 == ST_FALLBACK || (st0 == ST_RESOLVED && !h->h_ctrl->window_done && !h->h_ctrl->error);
    if (host_work) {
        // the speculative resolve could not be exact (first step after a load, a threshold far
        // off, heavy key ties) or Cd was too large for k_spec's window: the exact path --
        // cost-weighted radix select over every key, candidates, window -- from the host
        if (st0 == ST_FALLBACK) enqueue_exact(h, h->stream);
        else exact::group(h->P, h->c, h->d_ctrl, h->S, h->stream);
        k_publish<<<1, 64, 0, h->stream>>>(h->d_ctrl, h->h_ctrl);
        CK(cudaGetLastError());
    }
    // the host's part of the step is done: chained steps may run again (stream-ordered before the
    // next step; only the host's own work needs waiting for -- the fast path's control block and
    // batch were complete at the first synchronize)
    CK(cudaMemsetAsync(&h->S.persist->host_pending, 0, 4, h->stream));
    if (host_work) CK(cudaStreamSynchronize(h->stream));
    const Ctrl& c = *h->h_ctrl;
    if (c.status == ST_ERROR || c.error) return set_err(h, JIT_EINVAL, "step: invalid input (error code %u)", c.error);
    if (out) {
        out->n_pending = c.n_pending; out->n_dropped = c.n_dropped; out->status = c.status;
        out->n_refresh = c.n_refresh; out->fallback = c.fallback; out->n_spec = c.spec_n;
        out->n_selected = 0; out->total_tokens = 0; out->n_candidates = 0; out->b_star = 0; out->bp = 0; out->thr = 0;
    }
    if (c.status == ST_EMPTY) return JIT_EMPTY;
    if (c.status != ST_RESOLVED) return set_err(h, JIT_ECUDA, "step: unexpected status %u", c.status);
    if (out) {
        out->n_selected = c.n_selected; out->total_tokens = c.total_tokens; out->n_candidates = c.n_cand;
        out->b_star = c.b_star; out->bp = c.bp; out->thr = c.thr;
        if (c.n_selected > out->capacity && (out->ids || out->tokens || out->rows))
            return set_err(h, JIT_ECAPACITY, "batch capacity %u < %u", out->capacity, c.n_selected);
        if (c.batch_on_host) {
            // the fast path already wrote the batch into pinned host memory
            const uint32_t* hb = h->h_batch;
            const uint64_t B = h->cfg.max_batch + 1;
            if (out->ids) memcpy(out->ids, hb, 4ull * c.n_selected);
            if (out->tokens) memcpy(out->tokens, hb + B, 4ull * c.n_selected);
            if (out->rows) memcpy(out->rows, hb + 2 * B, 4ull * c.n_selected);
        } else {
            if (out->ids) CK(cudaMemcpyAsync(out->ids, h->S.out_ids, 4ull * c.n_selected, cudaMemcpyDeviceToHost, h->stream));
            if (out->tokens) CK(cudaMemcpyAsync(out->tokens, h->S.out_tokens, 4ull * c.n_selected, cudaMemcpyDeviceToHost, h->stream));
            if (out->rows) CK(cudaMemcpyAsync(out->rows, h->S.out_rows, 4ull * c.n_selected, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
        }
    }
    return JIT_OK;
}

static int finish_step(jit_sched* h, jit_batch* out) {
    const int rc = finish_step_body(h, out);
    h->unfinished = false;
    return rc;
}

// ------------------------------------------------------------------------------------------
// per-step deltas (arrivals, task updates, progress): packed into one pinned buffer, one H2D copy
// into the device staging area, then applied by kernels on the library stream before the step
// ------------------------------------------------------------------------------------------
struct HostPack {
    std::vector<unsigned char>* buf;
    uint64_t off = 0;
    template <typename T>
    uint64_t put(const T* src, uint64_t count) {          // returns the 16-B aligned offset
        off = (off + 15) & ~15ull;
        const uint64_t at = off;
        if (buf->size() < off + sizeof(T) * count) buf->resize(off + sizeof(T) * count);
        if (count) memcpy(buf->data() + at, src, sizeof(T) * count);
        off += sizeof(T) * count;
        return at;
    }
};

static int apply_deltas(jit_sched* h, const jit_step_in* in) {
    const jit_pool* a = in->arrivals;
    const uint32_t na = a ? a->n : 0u, nat = a ? a->n_tasks : 0u, ntu = in->n_task_updates, m = in->n_progress;
    if (!na && !nat && !ntu && !m) return JIT_OK;
    Pool& P = h->P;
    if (a) {
        if (a->on_device) return set_err(h, JIT_EINVAL, "arrivals must be host arrays");
        if (a->n_single > a->n) return set_err(h, JIT_EINVAL, "arrivals: n_single > n");
        if ((uint64_t)P.n + na > h->cfg.capacity || (uint64_t)P.n_tasks + nat > h->cfg.task_capacity)
            return set_err(h, JIT_ECAPACITY, "arrivals exceed the pool capacity (reload to compact)");
        if (nat) {
            if (!a->call_off || !a->task_arrival_ns || !a->task_deadline_ns || !a->cur_stage || !a->n_stages ||
                !a->pattern_ms || !a->goodput_done) return set_err(h, JIT_EINVAL, "arrivals: missing task arrays");
            if (a->call_off[0] != a->n_single || a->call_off[nat] != na)
                return set_err(h, JIT_EINVAL, "arrivals: call_off must span the compound rows");
            for (uint32_t t = 0; t < nat; ++t)
                if (a->call_off[t] > a->call_off[t + 1]) return set_err(h, JIT_EINVAL, "arrivals: call_off not monotone");
        } else if (a->n_single != na) {
            return set_err(h, JIT_EINVAL, "arrivals: compound rows without tasks");
        }
    }
    if (m > h->cfg.capacity) return set_err(h, JIT_ECAPACITY, "too many progress rows");
    std::vector<unsigned char>& hb = h->h_delta;
    HostPack pk{&hb};
    uint64_t o_arr = 0, o_u[8] = {}, o_t[8] = {}, o_tu[4] = {}, o_pg[4] = {}, o_fair = 0;
    if (na) {
        o_arr = pk.put(a->arrival_ns, na);
        const uint32_t* f[8] = {a->input_len, a->generated, a->prefilled, a->meta, a->aux, a->id, a->task, a->override_R};
        for (int i = 0; i < 8; ++i) o_u[i] = pk.put(f[i], na);
        if (a->fair) o_fair = pk.put(a->fair, na);
    }
    if (nat) {
        o_t[0] = pk.put(a->call_off, nat + 1); o_t[1] = pk.put(a->task_arrival_ns, nat); o_t[2] = pk.put(a->task_deadline_ns, nat);
        o_t[3] = pk.put(a->cur_stage, nat); o_t[4] = pk.put(a->n_stages, nat); o_t[5] = pk.put(a->pattern_ms, (uint64_t)nat * kMaxStages);
        o_t[6] = pk.put(a->goodput_done, nat);
    }
    if (ntu) {
        if (!in->tu_task || !in->tu_cur_stage || !in->tu_goodput_done) return set_err(h, JIT_EINVAL, "task updates: missing arrays");
        o_tu[0] = pk.put(in->tu_task, ntu); o_tu[1] = pk.put(in->tu_cur_stage, ntu); o_tu[2] = pk.put(in->tu_goodput_done, ntu);
        if (in->tu_stage_deadline_ns) o_tu[3] = pk.put(in->tu_stage_deadline_ns, ntu);
    }
    // the arrivals' work items (standalone chunks, then the new tasks), staged with the deltas
    const size_t i0 = h->h_items.size();
    uint64_t o_items = 0;
    if (na) {
        const uint32_t n0 = P.n, t0 = P.n_tasks;
        for (uint32_t r0 = n0; r0 < n0 + a->n_single; r0 += kItemRows)
            h->h_items.push_back(Item{r0, std::min<uint32_t>(r0 + kItemRows, n0 + a->n_single), 0u, 0u});
        if (nat) add_task_items(h->h_items, a->call_off, n0, t0, nat);
        if (h->h_items.size() > h->item_cap) {
            h->h_items.resize(i0);
            return set_err(h, JIT_ECAPACITY, "too many work items (reload to compact)");
        }
        o_items = pk.put(h->h_items.data() + i0, h->h_items.size() - i0);
    }
    if (m) {
        o_pg[0] = pk.put(in->prog_key, m); o_pg[1] = pk.put(in->prog_generated, m);
        o_pg[2] = pk.put(in->prog_prefilled, m); o_pg[3] = pk.put(in->prog_state, m);
    }
    const uint64_t bytes = (pk.off + 15) & ~15ull;
    if (bytes > h->load_bytes) {
        h->h_items.resize(i0);
        return set_err(h, JIT_ECAPACITY, "step deltas exceed the staging area");
    }
    if (bytes > h->pin_cap) {                              // pinned mirror, grown on demand
        if (h->h_pin) cudaFreeHost(h->h_pin);
        h->h_pin = nullptr; h->pin_cap = 0;
        CK(cudaMallocHost(&h->h_pin, std::max<uint64_t>(bytes, 1 << 16)));
        h->pin_cap = std::max<uint64_t>(bytes, 1 << 16);
    }
    memcpy(h->h_pin, hb.data(), pk.off);
    unsigned char* d = h->d_load;
    CK(cudaMemcpyAsync(d, h->h_pin, bytes, cudaMemcpyHostToDevice, h->stream));
    h->delta_h2d_bytes = bytes;
    cudaStream_t s = h->stream;
    if (na) {
        Arrivals A{};
        A.arr = reinterpret_cast<const int64_t*>(d + o_arr);
        const uint32_t** fu[8] = {&A.len_in, &A.gen, &A.pre, &A.meta, &A.aux, &A.id, &A.task, &A.ovr};
        for (int i = 0; i < 8; ++i) *fu[i] = reinterpret_cast<const uint32_t*>(d + o_u[i]);
        A.fair = a->fair ? reinterpret_cast<const uint32_t*>(d + o_fair) : nullptr;
        if (nat) {
            A.call_off = reinterpret_cast<const uint32_t*>(d + o_t[0]);
            A.t_arr = reinterpret_cast<const int64_t*>(d + o_t[1]); A.t_dl = reinterpret_cast<const int64_t*>(d + o_t[2]);
            A.cur_stage = reinterpret_cast<const uint32_t*>(d + o_t[3]); A.n_stages = reinterpret_cast<const uint32_t*>(d + o_t[4]);
            A.pattern = reinterpret_cast<const uint32_t*>(d + o_t[5]); A.gdone = reinterpret_cast<const uint64_t*>(d + o_t[6]);
        }
        A.n = na; A.n_single = a->n_single; A.n_tasks = nat; A.n0 = P.n; A.t0 = P.n_tasks;
        const uint32_t n_items = (uint32_t)h->h_items.size();
        A.items_src = reinterpret_cast<const Item*>(d + o_items); A.items_dst = h->d_items + i0;
        A.n_items_dst = h->d_n_items; A.n_new_items = n_items - (uint32_t)i0; A.n_items = n_items;
        const uint32_t n0 = P.n, t0 = P.n_tasks;
        const uint32_t g = (uint32_t)std::min<uint64_t>((std::max(std::max(na, nat), A.n_new_items) + 255) / 256 + 1,
                                                        (uint64_t)h->n_sm * 8);
        uint32_t* err = &h->S.gpart->err;
        const uint32_t* lh0 = h->T.forest ? nullptr : h->T.lhat0;
        if (!nat) {                                       // standalone requests only: one launch
            P.n = n0 + na;
            k_arrive_std<<<g, 256, 0, s>>>(P, A, h->d_groups, h->n_groups, h->T.n_rows, h->T.l_max, err, lh0, h->c.R);
        } else {
            k_append<<<g, 256, 0, s>>>(P, A);
            P.n = n0 + na; P.n_tasks = t0 + nat;
            k_validate<<<g, 256, 0, s>>>(P, h->d_groups, h->n_groups, h->T.n_rows, h->T.l_max, err, n0, n0 + a->n_single,
                                         t0, lh0, h->c.R);
            k_task_prep<<<g, 256, 0, s>>>(P, t0);
            k_map_insert<<<g, 256, 0, s>>>(P, n0, P.n, err);
        }
        CK(cudaGetLastError());
        h->n_items_host = n_items;
        h->S.n_ring_h = n_items - h->S.n_std_items;
        h->grid_pass = std::max<uint32_t>(1, std::min<uint32_t>((P.n + kPassThreads - 1) / kPassThreads, (uint32_t)h->n_sm * 4));
    }
    if (ntu) {
        k_task_update<<<(ntu + 255) / 256, 256, 0, s>>>(P, reinterpret_cast<const uint32_t*>(d + o_tu[0]),
                                                       reinterpret_cast<const uint32_t*>(d + o_tu[1]),
                                                       reinterpret_cast<const uint64_t*>(d + o_tu[2]),
                                                       in->tu_stage_deadline_ns ? reinterpret_cast<const int64_t*>(d + o_tu[3]) : nullptr,
                                                       ntu, h->S);
        CK(cudaGetLastError());
    }
    if (m) {
        k_progress<<<(m + 255) / 256, 256, 0, s>>>(P, h->S, reinterpret_cast<const uint32_t*>(d + o_pg[0]),
                                                   reinterpret_cast<const uint32_t*>(d + o_pg[1]),
                                                   reinterpret_cast<const uint32_t*>(d + o_pg[2]),
                                                   reinterpret_cast<const uint32_t*>(d + o_pg[3]), m, in->progress_by_id ? 1 : 0);
        CK(cudaGetLastError());
    }
    return JIT_OK;
}

extern "C" int jit_sched_step(jit_sched* h, const jit_step_in* in, jit_batch* out) {
    if (!h || !in) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "step before load");
    if (in->v_token_ns <= 0 || in->v_token_ns >= (1ll << 36)) return set_err(h, JIT_EINVAL, "v_token must be in (0, 2^36) ns");
    if (h->unfinished) return set_err(h, JIT_ESTATE, "a step_async step is unfinished: fetch its batch first");
    int rc = apply_deltas(h, in);
    if (rc) return rc;
    rc = launch_step(h, in->now_ns, in->v_token_ns);
    if (rc) return rc;
    return finish_step(h, out);
}

extern "C" int jit_sched_step_async(jit_sched* h, int64_t now_ns, int64_t v_token_ns) {
    if (!h) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "step before load");
    if (v_token_ns <= 0 || v_token_ns >= (1ll << 36)) return set_err(h, JIT_EINVAL, "v_token must be in (0, 2^36) ns");
    return launch_step(h, now_ns, v_token_ns, true);
}

extern "C" int jit_sched_fetch_batch(jit_sched* h, jit_batch* out) {
    if (!h) return JIT_EINVAL;
    return finish_step(h, out);
}

extern "C" int jit_sched_read_rows(jit_sched* h, double* key, double* rate, int64_t* t_rem, uint32_t* lhat,
                                   uint32_t* cost, uint32_t* pending, uint32_t* meta, uint32_t* aux) {
    if (!h) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "read_rows before load");
    const uint64_t n = h->P.n;
    // per-row keys, costs and debug outputs exist only on debug handles (every step materializes
    // them there); a production step writes no per-row output
    if ((key || pending || cost || rate || t_rem || lhat) && !h->debug)
        return set_err(h, JIT_ESTATE, "key/cost/pending/rate/t_rem/lhat need JIT_CFG_DEBUG_ROWS");
    if (h->unfinished) return set_err(h, JIT_ESTATE, "read_rows while a step is unfinished");
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    std::vector<uint64_t> img;
    if (key || pending) {
        img.resize(n);
        CK(cudaMemcpy(img.data(), h->P.img, 8 * n, cudaMemcpyDeviceToHost));
        for (uint64_t r = 0; r < n; ++r) {
            if (key) { double d; uint64_t b = img[r]; memcpy(&d, &b, 8); key[r] = b == kNone ? -1.0 : d; }
            if (pending) pending[r] = img[r] != kNone;
        }
    }
    if (rate) CK(cudaMemcpy(rate, h->P.dbg_rate, 8 * n, cudaMemcpyDeviceToHost));
    if (t_rem) CK(cudaMemcpy(t_rem, h->P.dbg_trem, 8 * n, cudaMemcpyDeviceToHost));
    if (lhat) CK(cudaMemcpy(lhat, h->P.dbg_lhat, 4 * n, cudaMemcpyDeviceToHost));
    if (cost) CK(cudaMemcpy(cost, h->P.cost, 4 * n, cudaMemcpyDeviceToHost));
    if (meta || aux) {
        // the caller's view of the hot rows: meta without the internal epoch / stamp bits, aux =
        // dist_row | steps_waited (the stamp resolved against the step counter)
        std::vector<HotRow> rows(n);
        Persist ps;
        CK(cudaMemcpy(rows.data(), h->P.rows, sizeof(HotRow) * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&ps, h->S.persist, sizeof ps, cudaMemcpyDeviceToHost));
        for (uint64_t r = 0; r < n; ++r) {
            if (meta) meta[r] = rows[r].meta & 0x7FFFu;
            if (aux) aux[r] = l_row(rows[r].lrow) | (waited_of(rows[r].meta, rows[r].since, ps.steps) << 16);
        }
    }
    return JIT_OK;
}

extern "C" int jit_sched_kernel_times(jit_sched* h, int enable, float* ms_out, uint32_t n_out) {
    // enable > 0: record per-kernel events for up to `enable` steps (ring of event slots);
    // enable = 0: off; enable < 0: leave as is.  ms_out gets the AVERAGE over the recorded
    // steps of [k_score, 0, k_spec, 0, whole step].
    if (!h) return JIT_EINVAL;
    if (enable >= 0) {
        CK(cudaStreamSynchronize(h->stream));
        for (auto e : h->slots) cudaEventDestroy(e);
        h->slots.clear(); h->n_slots = 0; h->slot_used = 0;
        if (enable > 0) {
            h->slots.resize(5ull * (uint32_t)enable);
            for (auto& e : h->slots) CK(cudaEventCreate(&e));
            h->n_slots = (uint32_t)enable;
        }
        if ((enable > 0) != h->timing) { h->timing = enable > 0; h->graph_dirty = true; }
    }
    if (ms_out && n_out) {
        if (!h->timing || !h->slot_used) return set_err(h, JIT_ESTATE, "kernel timing not enabled / no step recorded");
        CK(cudaStreamSynchronize(h->stream));
        double acc[5] = {0, 0, 0, 0, 0};
        const uint32_t ns = std::min(h->slot_used, h->n_slots);
        for (uint32_t k = 0; k < ns; ++k) {
            cudaEvent_t* e = &h->slots[5 * k];
            float t;
            CK(cudaEventElapsedTime(&t, e[0], e[1])); acc[0] += t;   // k_score
            CK(cudaEventElapsedTime(&t, e[1], e[2])); acc[1] += t;   // (empty: k_score has no successor pass)
            CK(cudaEventElapsedTime(&t, e[2], e[3])); acc[2] += t;   // k_spec (+ the exact path it launched)
            CK(cudaEventElapsedTime(&t, e[3], e[4])); acc[3] += t;   // (empty: k_spec publishes)
            CK(cudaEventElapsedTime(&t, e[0], e[4])); acc[4] += t;   // total
        }
        for (uint32_t i = 0; i < n_out && i < 5; ++i) ms_out[i] = (float)(acc[i] / ns);
    }
    return JIT_OK;
}

// Back-to-back k_score launches rotating over handles (that share one stream), timed with CUDA
// events around the whole sequence: the kernel's average duration with its launch overlapped by
// the previous kernel (a single launch bracketed by event nodes also counts the node's launch
// latency).  Each handle's per-step accumulators are reset afterwards (outside the timing).
// Back-to-back k_score launches rotating over handles (that share one stream), timed with CUDA
// events around the whole sequence: the kernel's average duration with its launch overlapped by
// the previous kernel (a single launch bracketed by event nodes also counts the node's launch
// latency).  flags & JIT_TIME_FORCE_REFRESH: every cached length bound is invalidated before each
// launch (untimed) and each launch is timed alone (events around it): the pass with a stale bound
// on every row.  Each handle's per-step accumulators are reset afterwards (outside the timing).
extern "C" int jit_sched_time_scoring(jit_sched** hs, uint32_t n_handles, int64_t now_ns, int64_t v_token_ns,
                                      uint32_t launches, uint32_t flags, float* ms_per_launch) {
    if (!hs || !n_handles || !launches || !ms_per_launch) return JIT_EINVAL;
    jit_sched* h = hs[0];
    for (uint32_t i = 0; i < n_handles; ++i) {
        if (!hs[i] || !hs[i]->loaded) return set_err(h, JIT_ESTATE, "time_scoring: handle %u not loaded", i);
        if (hs[i]->stream != h->stream) return set_err(h, JIT_EINVAL, "time_scoring: handles must share one stream");
        if (hs[i]->unfinished) return set_err(h, JIT_ESTATE, "time_scoring: handle %u has an unfinished step", i);
    }
    cudaStream_t s = h->stream;
    cudaEvent_t e0 = h->ev[0], e1 = h->ev[1];
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    if (flags & JIT_TIME_READ_FLOOR) {
        // the hot rows of each handle read with k_score's load pattern and nothing else
        CK(cudaEventRecord(e0, s));
        for (uint32_t k = 0; k < launches; ++k) {
            jit_sched* hk = hs[k % n_handles];
            k_read_floor<<<4 * hk->n_sm, 256, 0, s>>>(hk->P.rows, hk->P.n, reinterpret_cast<unsigned long long*>(hk->S.sk));
        }
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *ms_per_launch = ms / (float)launches;
        return JIT_OK;
    }
    if (flags & (JIT_TIME_FORCE_REFRESH | JIT_TIME_REFRESH_2PCT)) {
        for (uint32_t k = 0; k < launches; ++k) {
            jit_sched* hk = hs[k % n_handles];
            if (flags & JIT_TIME_FORCE_REFRESH) k_invalidate_bounds<<<hk->grid_pass, 256, 0, s>>>(hk->P);
            else k_invalidate_bounds<<<hk->grid_pass, 256, 0, s>>>(hk->P, 50u, k % 50u);
            CK(cudaEventRecord(e0, s));
            enqueue_score(hk, s, now_ns, v_token_ns);
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, e0, e1));
            ms += t;
        }
    } else {
        CK(cudaEventRecord(e0, s));
        for (uint32_t k = 0; k < launches; ++k) enqueue_score(hs[k % n_handles], s, now_ns, v_token_ns);
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
    }
    *ms_per_launch = ms / (float)launches;
    for (uint32_t i = 0; i < n_handles; ++i)       // consume the accumulated partials / sets
        CK(exact::spec(hs[i]->P, hs[i]->c, hs[i]->d_ctrl, hs[i]->S, 1, s, false));
    CK(cudaStreamSynchronize(s));
    return JIT_OK;
}

extern "C" int jit_sched_counters(jit_sched* h, uint32_t* steps, uint32_t* fallbacks, uint32_t* skipped) {
    if (!h) return JIT_EINVAL;
    CK(cudaStreamSynchronize(h->stream));
    Persist ps;
    CK(cudaMemcpy(&ps, h->S.persist, sizeof ps, cudaMemcpyDeviceToHost));
    if (steps) *steps = ps.steps;
    if (fallbacks) *fallbacks = ps.fallbacks;
    if (skipped) *skipped = ps.skipped;
    return JIT_OK;
}

// tests: move the device step counter (the steps_waited stamps count against it) and the host's
// launch count (the stamp rebase runs when it reaches a multiple of 2^30), so that the counter
// wrap and the rebase are exercised in a few steps
extern "C" int jit_sched_debug_set_counter(jit_sched* h, uint32_t steps, uint64_t launched) {
    if (!h) return JIT_EINVAL;
    if (h->unfinished) return set_err(h, JIT_ESTATE, "fetch the unfinished step first");
    CK(cudaStreamSynchronize(h->stream));
    Persist ps;
    CK(cudaMemcpy(&ps, h->S.persist, sizeof ps, cudaMemcpyDeviceToHost));
    const uint32_t d = steps - ps.steps;         // keep every stamped row's count: shift its stamp too
    if (h->P.n) k_shift_stamps<<<h->grid_pass, 256, 0, h->stream>>>(h->P, d);
    ps.steps = steps;
    CK(cudaMemcpyAsync(h->S.persist, &ps, sizeof ps, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->launched = launched;
    return JIT_OK;
}

// diagnostics: the first n u64 of the exact path's sort scratch (where JIT_TIMELINE builds of
// k_score leave their per-warp %globaltimer stamps)
extern "C" int jit_sched_debug_scratch(jit_sched* h, uint64_t* out, uint32_t n) {
    if (!h || !out) return JIT_EINVAL;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaMemcpy(out, h->S.sk, 8ull * n, cudaMemcpyDeviceToHost));
    return JIT_OK;
}

extern "C" int jit_sched_phase_times(jit_sched* h, uint64_t* ns_out, uint32_t n_out) {
    if (!h || !ns_out) return JIT_EINVAL;
    CK(cudaStreamSynchronize(h->stream));
    for (uint32_t i = 0; i < n_out && i < 11; ++i) ns_out[i] = h->h_ctrl->ts[i];
    return JIT_OK;
}

extern "C" void jit_sched_destroy(jit_sched* h) {
    if (!h) return;
    if (h->exec) cudaGraphExecDestroy(h->exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    if (h->cap) cudaStreamDestroy(h->cap);
    if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
    if (h->h_batch) cudaFreeHost(h->h_batch);
    if (h->h_pin) cudaFreeHost(h->h_pin);
    for (auto e : h->ev) if (e) cudaEventDestroy(e);
    for (auto e : h->slots) cudaEventDestroy(e);
    delete h;
}

extern "C" const char* jit_sched_last_error(const jit_sched* h) { return h ? h->err.c_str() : "null handle"; }
extern "C" const char* jit_sched_version(void) { return "jitsched 0.1 sm_100a"; }

// ------------------------------------------------------------------------------------------
// replay
// ------------------------------------------------------------------------------------------
#include "replay_host.inc"

// ------------------------------------------------------------------------------------------
// sharded step (shard.cuh): the caller runs the two allgathers between these calls
// ------------------------------------------------------------------------------------------
static_assert(sizeof(Rec1) == sizeof(jit_rec1) && sizeof(Rec2) == sizeof(jit_rec2), "record layout");
constexpr uint32_t kMergeSmem = 8192;

extern "C" int jit_shard_prefix(jit_sched* h, int64_t now_ns, int64_t v_token_ns, void* d_rec1, uint32_t cap,
                                uint32_t* n_out) {
    if (!h || !d_rec1 || !n_out) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "shard_prefix before load");
    if (v_token_ns <= 0 || v_token_ns >= (1ll << 36)) return set_err(h, JIT_EINVAL, "v_token must be in (0, 2^36) ns");
    if (cap < h->cfg.max_batch + 1) return set_err(h, JIT_ECAPACITY, "round-1 buffer needs max_batch+1 records");
    cudaStream_t s = h->stream;
    Pool& P = h->P;
    Scratch& S = h->S;
    if (!h->keys_ready) {
        h->arg_now = now_ns; h->arg_v = v_token_ns;
        enqueue_score(h, s, now_ns, v_token_ns);
        // k_spec only reduces the scoring partials (n_pending, errors, ...): the round-1 export
        // needs the full radix resolve below
        CK(exact::spec(P, h->c, h->d_ctrl, S, 1, s, false));
    }
    h->keys_ready = false;                 // (after a failed fast attempt the pool state is this step's)
    // every key and cost materialized for the radix select (idempotent re-score)
    enqueue_score(h, s, h->arg_now, h->arg_v, nullptr, false, 1);
    CK(cudaMemsetAsync(S.hcnt, 0, 4 * 4096, s));
    CK(cudaMemsetAsync(S.hcost, 0, 8 * 4096, s));
    exact::hist0(P, h->c, h->d_ctrl, S, h->grid_pass, 1, s);
    for (uint32_t i = 0; i < kLevels - 1; ++i) exact::pass(P, h->c, h->d_ctrl, S, h->grid_pass, i, s);
    exact::compact(P, h->c, h->d_ctrl, S, h->grid_pass, s);
    exact::resolve(P, h->c, h->d_ctrl, S, s);
    k_export1<<<h->grid_pass, kPassThreads, 0, s>>>(P, h->d_ctrl, S, (Rec1*)d_rec1, cap);
    k_export1_tail<<<1, 1024, 0, s>>>(h->d_ctrl, S, (Rec1*)d_rec1, cap);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctrl, h->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const Ctrl& c = *h->h_ctrl;
    if (c.status == ST_ERROR || c.error || c.cand_overflow) return set_err(h, JIT_EINVAL, "shard_prefix failed (%u)", c.error);
    *n_out = c.status == ST_RESOLVED ? c.n_cand : 0;
    return c.status == ST_EMPTY ? JIT_EMPTY : JIT_OK;
}

// fast sharded step (speculative sets; see k_spec_export / k_spec_merge)
extern "C" uint32_t jit_shard_spec_bytes(void) { return exact::spec_export_bytes(); }

extern "C" int jit_shard_spec_export(jit_sched* h, int64_t now_ns, int64_t v_token_ns, void* d_out, uint32_t cap_bytes,
                                     uint32_t rank) {
    if (!h || !d_out) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "shard_spec_export before load");
    if (v_token_ns <= 0 || v_token_ns >= (1ll << 36)) return set_err(h, JIT_EINVAL, "v_token must be in (0, 2^36) ns");
    if (cap_bytes < exact::spec_export_bytes()) return set_err(h, JIT_ECAPACITY, "export buffer needs %u bytes",
                                                                exact::spec_export_bytes());
    h->arg_now = now_ns; h->arg_v = v_token_ns;
    enqueue_score(h, h->stream, now_ns, v_token_ns);
    CK(exact::spec_export(h->S, h->d_ctrl, d_out, rank, h->stream));
    h->keys_ready = true;
    return JIT_OK;
}

extern "C" int jit_shard_spec_resolve(jit_sched* h, const void* d_all, uint32_t world, uint32_t rank, jit_batch* out) {
    if (!h || !d_all || world == 0 || world > 64 || rank >= world) return JIT_EINVAL;
    if (!h->keys_ready) return set_err(h, JIT_ESTATE, "shard_spec_resolve without shard_spec_export");
    CK(exact::spec_merge(h->P, h->c, h->d_ctrl, h->S, d_all, world, rank, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const Ctrl& c = *h->h_ctrl;
    if (c.status == ST_FALLBACK) return JIT_RETRY;          // keys stay: jit_shard_prefix continues
    h->keys_ready = false;
    if (out) { out->fallback = 0; }
    return finish_step(h, out);
}

extern "C" int jit_shard_merge(jit_sched* h, const void* d_all_rec1, uint32_t n_all) {
    if (!h || (!d_all_rec1 && n_all)) return JIT_EINVAL;
    uint64_t n2 = 1;
    while (n2 < n_all) n2 <<= 1;
    const uint64_t N = ((uint64_t)h->cfg.capacity + 63) & ~63ull;
    uint64_t P2 = 1;
    while (P2 < N) P2 <<= 1;
    if (n2 > kMergeSmem && n2 > P2) return set_err(h, JIT_ECAPACITY, "merge of %u records exceeds the workspace", n_all);
    const uint32_t smem = (uint32_t)((sizeof(u128) + 4) * kMergeSmem);
    CK(cudaFuncSetAttribute(k_merge1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_merge1<<<1, 1024, smem, h->stream>>>(h->c, h->d_ctrl, (const Rec1*)d_all_rec1, n_all, h->S.pf, h->S.sv, kMergeSmem);
    CK(cudaGetLastError());
    return JIT_OK;
}

extern "C" int jit_shard_candidates(jit_sched* h, void* d_rec2, uint32_t cap, uint32_t rank, uint32_t* n_out) {
    if (!h || !n_out) return JIT_EINVAL;
    cudaStream_t s = h->stream;
    exact::cand(h->P, h->c, h->d_ctrl, h->S, h->grid_pass, 0, s);
    k_export2<<<h->grid_pass, 256, 0, s>>>(h->P, h->c, h->d_ctrl, h->S, (Rec2*)d_rec2, cap, rank);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctrl, h->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const Ctrl& c = *h->h_ctrl;
    if (c.status == ST_EMPTY) { *n_out = 0; return JIT_EMPTY; }
    if (c.status != ST_RESOLVED || c.error) return set_err(h, JIT_EINVAL, "shard_candidates: bad state %u", c.status);
    if (c.cand_overflow || c.n_cand > cap) return set_err(h, JIT_ECAPACITY, "round-2 buffer too small (%u > %u)", c.n_cand, cap);
    *n_out = c.n_cand;
    return JIT_OK;
}

extern "C" int jit_shard_finish(jit_sched* h, const void* d_all_rec2, uint32_t n_all, uint32_t rank, jit_batch* out) {
    if (!h) return JIT_EINVAL;
    cudaStream_t s = h->stream;
    uint64_t n2 = 1;
    while (n2 < n_all) n2 <<= 1;
    const uint64_t N = ((uint64_t)h->cfg.capacity + 63) & ~63ull;
    if (n_all > N) return set_err(h, JIT_ECAPACITY, "window over %u records exceeds the workspace", n_all);
    if (h->h_ctrl->status == ST_EMPTY) { if (out) { out->n_selected = 0; out->status = ST_EMPTY; } return JIT_EMPTY; }
    k_group_rec<<<1, 1024, 12 * kGroupSmemSort, s>>>(h->P, h->c, h->d_ctrl, h->S, (const Rec2*)d_all_rec2, n_all, rank);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h->h_ctrl, h->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    return finish_step(h, out);
}

// ------------------------------------------------------------------------------------------
// NEXT-2: power-of-K over M replicas (multi.cuh): export after a step, reconcile against the union
// ------------------------------------------------------------------------------------------
extern "C" uint64_t jit_multi_record_bytes(const jit_sched* h) {
    return h ? multi_rec_bytes(h->cfg.max_batch) : 0;
}

extern "C" int jit_multi_export(jit_sched* h, uint32_t replica, void* d_out) {
    if (!h || !d_out) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "multi_export before load");
    if (h->unfinished) return set_err(h, JIT_ESTATE, "multi_export while a step is unfinished");
    if (replica >= kMaxReplicas) return set_err(h, JIT_EINVAL, "replica index %u >= %u", replica, kMaxReplicas);
    k_multi_export<<<(h->cfg.max_batch + 255) / 256 + 1, 256, 0, h->stream>>>(h->d_ctrl, h->S, replica, h->cfg.max_batch,
                                                                               (unsigned char*)d_out);
    CK(cudaGetLastError());
    return JIT_OK;
}

extern "C" int jit_multi_reconcile(jit_sched* h, const void* d_all, uint32_t n_replicas, uint32_t replica, jit_batch* out) {
    if (!h || !d_all) return JIT_EINVAL;
    if (!h->loaded) return set_err(h, JIT_ESTATE, "multi_reconcile before load");
    if (h->unfinished) return set_err(h, JIT_ESTATE, "multi_reconcile while a step is unfinished");
    if (n_replicas == 0 || n_replicas > kMaxReplicas || replica >= n_replicas)
        return set_err(h, JIT_EINVAL, "replica %u of %u (at most %u replicas)", replica, n_replicas, kMaxReplicas);
    if (h->P.n_tasks) return set_err(h, JIT_EINVAL, "power-of-K replicas hold standalone requests only");
    const uint32_t cap = h->cfg.max_batch;
    const uint64_t rb = multi_rec_bytes(cap);
    const unsigned long long ep = ++h->multi_epoch;
    const unsigned char* all = (const unsigned char*)d_all;
    const uint32_t grid = (uint32_t)std::min<uint64_t>(((uint64_t)n_replicas * cap + 255) / 256, 8ull * h->n_sm);
    k_multi_mark<<<grid, 256, 0, h->stream>>>(h->P, h->S, h->d_ctrl, all, rb, n_replicas, replica, cap, h->S.mwin, ep);
    k_multi_moved<<<grid, 256, 0, h->stream>>>(h->P, h->S, h->d_ctrl, all, rb, n_replicas, replica, cap, h->S.mwin, ep);
    k_multi_finish<<<1, kMultiThreads, 0, h->stream>>>(h->S, h->d_ctrl, all, rb, n_replicas, replica, cap, h->S.mwin, ep);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    const Ctrl& c = *h->h_ctrl;
    if (c.error) return set_err(h, JIT_EINVAL, "multi_reconcile: invalid records or pool (error code %u)", c.error);
    if (out) {
        out->n_pending = c.n_pending; out->n_dropped = c.n_dropped; out->status = c.status;
        out->n_refresh = c.n_refresh; out->fallback = c.fallback; out->n_spec = c.spec_n;
        out->n_selected = c.status == ST_RESOLVED ? c.n_selected : 0;
        out->total_tokens = c.status == ST_RESOLVED ? c.total_tokens : 0;
        out->n_candidates = c.n_cand; out->b_star = c.b_star; out->bp = c.bp; out->thr = c.thr;
        if (out->n_selected > out->capacity && (out->ids || out->tokens || out->rows))
            return set_err(h, JIT_ECAPACITY, "batch capacity %u < %u", out->capacity, out->n_selected);
        const uint32_t* hb = h->h_batch;
        const uint64_t B = cap + 1;
        if (out->ids) memcpy(out->ids, hb, 4ull * out->n_selected);
        if (out->tokens) memcpy(out->tokens, hb + B, 4ull * out->n_selected);
        if (out->rows) memcpy(out->rows, hb + 2 * B, 4ull * out->n_selected);
    }
    return c.status == ST_RESOLVED ? JIT_OK : JIT_EMPTY;
}

// ------------------------------------------------------------------------------------------
// NEXT-3: batch pattern-graph matching (match.cuh)
// ------------------------------------------------------------------------------------------
static uint64_t match_layout(uint32_t np, uint32_t nq, uint64_t* off) {
    uint64_t o = 0;
    auto take = [&](uint64_t b) { o = (o + 255) & ~255ull; const uint64_t r = o; o += b; return r; };
    off[0] = take(4ull * np * (4 * kMaxStages + 2));            // patterns: ident, in, out, t_ms, n_stages, reuse
    off[1] = take(4ull * nq * (3 * kMaxStages + 2));            // queries: ident, in, out, stage, task
    off[2] = take(4ull * nq);                                   // best
    off[3] = take(8ull * nq);                                   // score
    return o + 256;
}

extern "C" int jit_match_workspace_bytes(uint32_t n_patterns, uint32_t n_queries, uint64_t* bytes) {
    if (!bytes) return JIT_EINVAL;
    uint64_t off[4];
    *bytes = match_layout(n_patterns, n_queries, off);
    return JIT_OK;
}

extern "C" int jit_sched_match(jit_sched* h, const jit_pattern_store* st, const jit_match_query* q, void* dev_workspace,
                               uint64_t ws_bytes, int32_t* best, double* score, uint32_t apply) {
    if (!h) return JIT_EINVAL;
    if (!st || !q || !best || !score || !st->n_stages || !st->ident || !st->in_len || !st->out || !st->t_ms ||
        !st->reuse || (q->n && (!q->stage || !q->ident || !q->in_len || !q->out)))
        return set_err(h, JIT_EINVAL, "match: null arrays");
    if (apply && !q->task) return set_err(h, JIT_EINVAL, "match: apply needs query task indices");
    const uint32_t np = st->n_patterns, nq = q->n;
    for (uint32_t p = 0; p < np; ++p) {                          // a pattern must define phi
        const uint32_t S = st->n_stages[p];
        uint64_t tot = 0;
        for (uint32_t u = 0; u < S && u < kMaxStages; ++u) tot += st->t_ms[(uint64_t)p * kMaxStages + u];
        if (S == 0 || S > kMaxStages || tot == 0) return set_err(h, JIT_EINVAL, "match: pattern %u malformed", p);
    }
    if (nq == 0) return JIT_OK;
    uint64_t off[4];
    const uint64_t need = match_layout(np, nq, off);
    if (!dev_workspace || ws_bytes < need) return set_err(h, JIT_ECAPACITY, "match workspace too small");
    unsigned char* base = reinterpret_cast<unsigned char*>(((uintptr_t)dev_workspace + 255) & ~(uintptr_t)255);
    cudaStream_t s = h->stream;
    uint32_t* pw = reinterpret_cast<uint32_t*>(base + off[0]);
    uint32_t* qw = reinterpret_cast<uint32_t*>(base + off[1]);
    const uint64_t P8 = (uint64_t)np * kMaxStages, Q8 = (uint64_t)nq * kMaxStages;
    if (np) {
        CK(cudaMemcpyAsync(pw, st->ident, 4 * P8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(pw + P8, st->in_len, 4 * P8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(pw + 2 * P8, st->out, 4 * P8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(pw + 3 * P8, st->t_ms, 4 * P8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(pw + 4 * P8, st->n_stages, 4ull * np, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(pw + 4 * P8 + np, st->reuse, 4ull * np, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemcpyAsync(qw, q->ident, 4 * Q8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(qw + Q8, q->in_len, 4 * Q8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(qw + 2 * Q8, q->out, 4 * Q8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(qw + 3 * Q8, q->stage, 4ull * nq, cudaMemcpyHostToDevice, s));
    if (q->task) CK(cudaMemcpyAsync(qw + 3 * Q8 + nq, q->task, 4ull * nq, cudaMemcpyHostToDevice, s));
    PatternsDev G{pw + 4 * P8, pw, pw + P8, pw + 2 * P8, pw + 3 * P8, pw + 4 * P8 + np, np};
    QueriesDev Q{qw + 3 * Q8, qw, qw + Q8, qw + 2 * Q8, q->task ? qw + 3 * Q8 + nq : nullptr, nq};
    int32_t* d_best = reinterpret_cast<int32_t*>(base + off[2]);
    double* d_score = reinterpret_cast<double*>(base + off[3]);
    const uint32_t staged = np <= kMatchSmemPatterns ? 1u : 0u;
    const uint32_t smem = staged ? 4u * np * kMatchWords : 0u;
    CK(cudaFuncSetAttribute(k_match, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4u * kMatchSmemPatterns * kMatchWords)));
    const uint32_t warps_per_cta = kMatchThreads / 32;
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((nq + warps_per_cta - 1) / warps_per_cta,
                                                                   (uint32_t)h->n_sm * 2));
    cudaEvent_t ev[2];
    CK(cudaEventCreate(&ev[0])); CK(cudaEventCreate(&ev[1]));
    CK(cudaEventRecord(ev[0], s));
    k_match<<<grid, kMatchThreads, smem, s>>>(G, Q, d_best, d_score, staged);
    CK(cudaEventRecord(ev[1], s));
    CK(cudaGetLastError());
    if (apply) {
        uint32_t* err = &h->S.gpart->err;
        k_apply_match<<<(nq + 255) / 256, 256, 0, s>>>(h->P, G, Q, d_best, err);
        if (h->P.n_tasks) k_task_prep<<<std::max<uint32_t>(1, std::min<uint32_t>((h->P.n_tasks + 255) / 256, (uint32_t)h->n_sm * 8)), 256, 0, s>>>(h->P, 0u);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(best, d_best, 4ull * nq, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(score, d_score, 8ull * nq, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventElapsedTime(&h->match_ms, ev[0], ev[1]));
    cudaEventDestroy(ev[0]); cudaEventDestroy(ev[1]);
    if (apply) {
        uint32_t e = 0;
        CK(cudaMemcpy(&e, &h->S.gpart->err, 4, cudaMemcpyDeviceToHost));
        if (e & 16u) {
            CK(cudaMemset(&h->S.gpart->err, 0, 4));
            return set_err(h, JIT_EINVAL, "match: a query's stage is not its task's current stage");
        }
    }
    return JIT_OK;
}

extern "C" int jit_sched_last_match_ms(jit_sched* h, float* ms) {
    if (!h || !ms) return JIT_EINVAL;
    *ms = h->match_ms;
    return JIT_OK;
}

// ------------------------------------------------------------------------------------------
// NEXT-4: the quantile regression forest in (a2)
// ------------------------------------------------------------------------------------------
static uint64_t forest_layout(const jit_forest* f, uint64_t* off) {
    uint64_t o = 0;
    auto take = [&](uint64_t b) { o = (o + 255) & ~255ull; const uint64_t r = o; o += b; return r; };
    off[0] = take(sizeof(ForestDev));
    off[1] = take(4ull * f->n_trees);
    for (int i = 0; i < 4; ++i) off[2 + i] = take(4ull * f->n_nodes);
    off[6] = take(4ull * std::max<uint32_t>(f->n_samples, 1));
    return o + 256;
}

static int forest_check(jit_sched* h, const jit_forest* f, uint32_t l_max) {
    if (!f->root || !f->feature || !f->threshold || !f->left || !f->right || !f->samples)
        return set_err(h, JIT_EINVAL, "forest: null arrays");
    if (f->n_trees == 0 || f->n_trees > kMaxTrees) return set_err(h, JIT_EINVAL, "forest: 1..%u trees", kMaxTrees);
    for (uint32_t v = 0; v < f->n_nodes; ++v) {
        if (f->feature[v] == kLeaf) {
            const uint64_t e = (uint64_t)f->threshold[v] + f->left[v];
            if (e > f->n_samples) return set_err(h, JIT_EINVAL, "forest: leaf %u beyond the samples", v);
            for (uint64_t i = f->threshold[v]; i < e; ++i) {
                if (f->samples[i] == 0 || f->samples[i] > l_max) return set_err(h, JIT_EINVAL, "forest: sample out of [1, l_max]");
                if (i > f->threshold[v] && f->samples[i] < f->samples[i - 1]) return set_err(h, JIT_EINVAL, "forest: leaf %u not sorted", v);
            }
        } else if (f->feature[v] >= 4 || f->left[v] >= f->n_nodes || f->right[v] >= f->n_nodes) {
            return set_err(h, JIT_EINVAL, "forest: node %u malformed", v);
        }
    }
    for (uint32_t t = 0; t < f->n_trees; ++t) {                 // every path ends in a leaf within 64 levels
        if (f->root[t] >= f->n_nodes) return set_err(h, JIT_EINVAL, "forest: bad root");
        std::vector<std::pair<uint32_t, uint32_t>> st{{f->root[t], 0u}};
        while (!st.empty()) {
            const auto [v, d] = st.back();
            st.pop_back();
            if (d > 64) return set_err(h, JIT_EINVAL, "forest: tree %u deeper than 64 (or cyclic)", t);
            if (f->feature[v] != kLeaf) { st.push_back({f->left[v], d + 1}); st.push_back({f->right[v], d + 1}); }
        }
    }
    return JIT_OK;
}

extern "C" int jit_forest_bytes(const jit_forest* f, uint64_t* bytes) {
    if (!f || !bytes) return JIT_EINVAL;
    uint64_t off[7];
    *bytes = forest_layout(f, off);
    return JIT_OK;
}

extern "C" int jit_sched_attach_forest(jit_sched* h, const jit_forest* f, void* dev_buf, uint64_t bytes) {
    if (!h) return JIT_EINVAL;
    if (h->unfinished) return set_err(h, JIT_ESTATE, "fetch the unfinished step first");
    if (!f) {
        h->T.forest = nullptr;
    } else {
        int rc = forest_check(h, f, h->T.l_max);
        if (rc) return rc;
        uint64_t off[7];
        const uint64_t need = forest_layout(f, off);
        if (!dev_buf || bytes < need) return set_err(h, JIT_ECAPACITY, "forest buffer too small");
        unsigned char* base = reinterpret_cast<unsigned char*>(((uintptr_t)dev_buf + 255) & ~(uintptr_t)255);
        cudaStream_t s = h->stream;
        ForestDev F{};
        uint32_t* d[6];
        const uint32_t* src[6] = {f->root, f->feature, f->threshold, f->left, f->right, f->samples};
        const uint64_t cnt[6] = {f->n_trees, f->n_nodes, f->n_nodes, f->n_nodes, f->n_nodes, f->n_samples};
        for (int i = 0; i < 6; ++i) {
            d[i] = reinterpret_cast<uint32_t*>(base + off[1 + i]);
            if (cnt[i]) CK(cudaMemcpyAsync(d[i], src[i], 4 * cnt[i], cudaMemcpyHostToDevice, s));
        }
        F.root = d[0]; F.feature = d[1]; F.threshold = d[2]; F.left = d[3]; F.right = d[4]; F.samples = d[5];
        F.n_trees = f->n_trees; F.n_nodes = f->n_nodes; F.n_samples = f->n_samples;
        CK(cudaMemcpyAsync(base + off[0], &F, sizeof F, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        h->T.forest = reinterpret_cast<const ForestDev*>(base + off[0]);
    }
    // every cached bound came from the other estimator: refresh them all; the step graph holds T
    if (h->P.n) k_invalidate_bounds<<<h->grid_pass, 256, 0, h->stream>>>(h->P);
    CK(cudaGetLastError());
    h->graph_dirty = true;
    CK(cudaStreamSynchronize(h->stream));
    return JIT_OK;
}

__global__ void k_qrf_batch(Table T, Cfg c, const uint32_t* x, const uint32_t* g, uint32_t n, uint32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t gi = g[i], anchor = c.R * (gi / c.R);
        const uint32_t q = qrf_bound(T.forest, x[4 * i], x[4 * i + 1], anchor, x[4 * i + 3], anchor, c.qn, c.qd, T.l_max);
        out[i] = q > gi + 1 ? q : gi + 1;                        // A5 clamp
    }
}

extern "C" int jit_qrf_workspace_bytes(uint32_t n, uint64_t* bytes) {
    if (!bytes) return JIT_EINVAL;
    *bytes = 24ull * n + 1024;
    return JIT_OK;
}

extern "C" int jit_sched_qrf_bound(jit_sched* h, const uint32_t* x, const uint32_t* g, uint32_t n, void* dev_workspace,
                                   uint64_t ws_bytes, uint32_t* out, float* kernel_ms) {
    if (!h) return JIT_EINVAL;
    if (!h->T.forest) return set_err(h, JIT_ESTATE, "no forest attached");
    if (!x || !g || !out) return set_err(h, JIT_EINVAL, "qrf: null arrays");
    if (n == 0) return JIT_OK;
    if (!dev_workspace || ws_bytes < 24ull * n + 1024) return set_err(h, JIT_ECAPACITY, "qrf workspace too small");
    for (uint32_t i = 0; i < n; ++i)
        if (g[i] >= (1u << 24)) return set_err(h, JIT_EINVAL, "qrf: generated >= 2^24");
    unsigned char* base = reinterpret_cast<unsigned char*>(((uintptr_t)dev_workspace + 255) & ~(uintptr_t)255);
    uint32_t* dx = reinterpret_cast<uint32_t*>(base);
    uint32_t* dg = dx + 4ull * n;
    uint32_t* dout = dg + n;
    cudaStream_t s = h->stream;
    CK(cudaMemcpyAsync(dx, x, 16ull * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dg, g, 4ull * n, cudaMemcpyHostToDevice, s));
    cudaEvent_t ev[2];
    CK(cudaEventCreate(&ev[0])); CK(cudaEventCreate(&ev[1]));
    CK(cudaEventRecord(ev[0], s));
    k_qrf_batch<<<std::min<uint32_t>((n + 127) / 128, (uint32_t)h->n_sm * 16), 128, 0, s>>>(h->T, h->c, dx, dg, n, dout);
    CK(cudaEventRecord(ev[1], s));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout, 4ull * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    cudaEventDestroy(ev[0]); cudaEventDestroy(ev[1]);
    if (kernel_ms) *kernel_ms = ms;
    return JIT_OK;
}
