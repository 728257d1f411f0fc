/*
 * oracle/gmax_oracle.c -- plain, slow, single-threaded CPU ORACLE of the JITServe
 * GMAX scheduling step (arXiv 2504.20068) and of the trace replay used to count goodput.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2504_20068_b200/,
 * include/) may include, link or call this file.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg load it (through oracle/__init__.py).
 * It shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / algorithm named beside it),
 * "S:n" = SPEC.md line n, "A<k>" = the reading number in DESIGN.md §3 (ambiguity register,
 * taken from SURVEY.md §8(c).2).  The order of operations follows Alg. 1:
 * AnalyzeRequest for every queued request, BatchPriority, Filter by cutoff, sort by length,
 * sliding window, return BestGroup.
 *
 * Exactness contract: every time is int64 ns; lengths/costs are integers;
 * the only floating point is (i) key = fl(A / B) with integers A, B < 2^53 (one IEEE
 * division, correctly rounded), (ii) the reported rate, same form, and (iii)
 * thr = fl(fl(p_num / p_den) * bp).  Window sums are exact u128 sums of floor(key * 2^32).
 * Compile with -O2 -ffp-contract=off (no FMA contraction).
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py
 * except the items DESIGN.md lists as "parity unpinned" (synthetic table contents, the cost
 * model constants of S:438, the phi inputs, absolute goodput levels of C2-C5).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------ */
/* Types (the oracle's own; the CUDA library declares its own in include/jit_sched.h)   */
/* ------------------------------------------------------------------------------------ */

enum { OG_LAT = 0, OG_DDL = 1, OG_CMP = 2, OG_BE = 3 };           /* §3 P:209-216 + BE P:216 */
enum { ST_QUEUED = 0, ST_RUNNING = 1, ST_PREEMPTED = 2, ST_DONE = 3, ST_DROPPED = 4,
       ST_WAITING = 5 /* compound call of a stage not yet released */,
       ST_MOVED = 6   /* NEXT-2 power-of-K: the request was assigned to another replica */ };
enum { FL_EVER = 1u, FL_COMPOUND = 2u, FL_OVERRIDE = 4u };
#define NO_TASK 0xFFFFFFFFu
#define MAX_STAGES 8u

typedef struct {
    uint32_t type, w_in, w_out, _pad;
    int64_t ttft_ns, tbt_ns, e2el_ns, be_deadline_ns;
} og_group;

typedef struct {
    uint32_t token_budget, max_batch, prefill_chunk, refine_interval, frame_steps;
    uint32_t q_num, q_den, p_num, p_den, delta_starve;
    uint32_t len_key, appb_filter;
    int64_t eps_ns, waiting_ns;
    /* NEXT-1 preemption gate (reading A46): 0 = off (the step re-selects every iteration, A30) */
    uint32_t preempt, pmtn_num, pmtn_den, _pad2;   /* delta_pmtn = pmtn_num / pmtn_den (App. D.2) */
    uint64_t io_bw_tps;                            /* KV swap bandwidth, tokens per second */
    /* NEXT-2 fairness blend (§4.3, reading A47): f = fair_num / fair_den, 0 = off */
    uint32_t fair_num, fair_den;
} og_config;

/* NEXT-4: a quantile regression forest (§4.1; SPEC estimator S:92-158; reading A50).
 * Nodes of all trees in one array: an inner node sends x to `left` iff x[feature] <= threshold,
 * else to `right`; a leaf (feature = OG_LEAF) holds samples[threshold .. threshold + left), its
 * training targets.  Features: x = (L_i, dist_row, anchor R*floor(g/R), SLO group). */
#define OG_LEAF 0xFFFFFFFFu
typedef struct {
    uint32_t n_trees, n_nodes, n_samples, n_features;
    const uint32_t* root;
    const uint32_t* feature;
    const uint32_t* threshold;
    const uint32_t* left;
    const uint32_t* right;
    const uint32_t* samples;
} og_forest;

typedef struct {
    uint32_t n_rows, n_bins, l_max, _pad;
    const uint32_t* edges;
    const uint32_t* cum;
    const og_forest* forest;   /* NULL: the table; else (a2) queries the forest (NEXT-4, A50) */
} og_table;

typedef struct {
    uint32_t n, _pad;
    const uint32_t* id;
    const int64_t* arrival_ns;
    const uint32_t* input_len;
    const uint32_t* generated;
    const uint32_t* prefilled;
    uint32_t* meta;       /* in/out: group bits 0-7, state 8-11, flags 12-15 */
    uint32_t* aux;        /* in/out: dist_row bits 0-15, steps_waited 16-31 */
    const uint32_t* task; /* NO_TASK for standalone requests */
    const uint32_t* override_R;
    const uint32_t* fair; /* NULL or Fair(r) per request (NEXT-2 blend, A47); NULL reads as 0 */
} og_pool;

typedef struct {
    uint32_t n, _pad;
    const uint32_t* call_off;     /* n+1: rows of task t are [call_off[t], call_off[t+1]) */
    const int64_t* arrival_ns;    /* a_c */
    const int64_t* deadline_ns;   /* D, relative to a_c */
    const uint32_t* cur_stage;
    const uint32_t* n_stages;
    const uint32_t* pattern_ms;   /* n * MAX_STAGES matched-pattern stage times */
    const uint64_t* goodput_done;
    const int64_t* stage_deadline_ns;   /* NULL, or per task: the stage sub-deadline a_c + D_s given by the
                                           caller (SURVEY 8(b) task updates); < 0: from the pattern */
} og_tasks;

typedef struct {
    uint32_t n_pending, n_selected, total_tokens, n_candidates, b_star, n_dropped_now;
    uint32_t error, n_preempted;   /* n_preempted: running requests evicted by the gate (A46) */
    double bp, thr;
    int64_t stall_ns;              /* KV swap stall of the evicted requests (A46) */
} og_result;

typedef struct {          /* optional per-row outputs (each pointer may be NULL) */
    double* key;
    double* rate;
    int64_t* t_rem;
    uint32_t* lhat;
    uint32_t* cost;
    uint32_t* pending;
} og_rows_out;

enum { OG_OK = 0, OG_EMPTY = 1, OG_EINVAL = -1 };

/* ------------------------------------------------------------------------------------ */
/* (a2) Conditional upper-quantile length bound.                                        */
/* §4.1: a high-quantile upper bound of the response length, re-derived      */
/* "every 50 tokens" as generation progresses; north_star: the upper quantile of */
/* the length distribution conditioned on the tokens generated so far.                  */
/* Reading A4: type-1 (inverse CDF, no interpolation) quantile on the histogram row.    */
/* Reading A5: condition on L > anchor, then clamp Lhat >= g + 1.  A6: anchor = R*floor(g/R). */
/* Reading A7: no mass above the anchor -> L_max.                                        */
/* ------------------------------------------------------------------------------------ */

static uint32_t* g_qmemo = NULL;        /* memo of Q(row, anchor), 0 = not computed */
static uint32_t g_qmemo_rows = 0, g_qmemo_anchors = 0;
static const og_table* g_qmemo_tab = NULL;
static uint32_t g_qmemo_qn = 0, g_qmemo_qd = 0, g_qmemo_R = 0;

/* Q_q(L | L > anchor): the smallest edge e_k with q_den*(C[k]-C_below) >= q_num*(N-C_below),
 * C_below = cumulative count of the bins whose upper edge is <= anchor.  Plain linear scans. */
static uint32_t cond_quantile_scan(const og_table* T, uint32_t row, uint32_t anchor,
                                   uint32_t q_num, uint32_t q_den) {
    const uint32_t* C = T->cum + (size_t)row * T->n_bins;
    uint32_t N = C[T->n_bins - 1];
    uint32_t below = 0;
    for (uint32_t k = 0; k < T->n_bins; ++k) {
        if (T->edges[k] <= anchor) below = C[k];
        else break;
    }
    if (N == below) return T->l_max;                        /* A7 */
    for (uint32_t k = 0; k < T->n_bins; ++k) {
        if (T->edges[k] <= anchor) continue;               /* only L > anchor */
        uint64_t lhs = (uint64_t)q_den * (uint64_t)(C[k] - below);
        uint64_t rhs = (uint64_t)q_num * (uint64_t)(N - below);
        if (lhs >= rhs) return T->edges[k];
    }
    return T->l_max;  /* unreachable for q <= 1 */
}

static uint32_t cond_quantile(const og_table* T, uint32_t row, uint32_t anchor,
                              uint32_t q_num, uint32_t q_den, uint32_t R) {
    /* memo keyed by (row, anchor / R); the value is a pure function of its inputs */
    if (g_qmemo_tab != T || g_qmemo_qn != q_num || g_qmemo_qd != q_den || g_qmemo_R != R ||
        g_qmemo_rows != T->n_rows) {
        free(g_qmemo);
        g_qmemo_anchors = T->l_max / R + 2;
        g_qmemo_rows = T->n_rows;
        g_qmemo = (uint32_t*)calloc((size_t)g_qmemo_rows * g_qmemo_anchors, sizeof(uint32_t));
        g_qmemo_tab = T; g_qmemo_qn = q_num; g_qmemo_qd = q_den; g_qmemo_R = R;
    }
    uint32_t a = anchor / R;
    if (g_qmemo && a < g_qmemo_anchors) {
        uint32_t* m = &g_qmemo[(size_t)row * g_qmemo_anchors + a];
        if (*m == 0) *m = cond_quantile_scan(T, row, anchor, q_num, q_den);
        return *m;
    }
    return cond_quantile_scan(T, row, anchor, q_num, q_den);
}

/* NEXT-4 (A50): Q_q over the pooled leaf samples of the trees' leaves for x, conditioned on
 * L > anchor like (a2): the ceil(q m)-th smallest of the m pooled samples above the anchor
 * (type-1 quantile, A4; every tree's leaf contributes its samples once); none -> L_max (A7). */
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}
uint32_t og_qrf_quantile(const og_forest* F, const uint32_t* x, uint32_t anchor, uint32_t q_num, uint32_t q_den,
                         uint32_t l_max) {
    uint32_t cap = 0;
    uint32_t* leaf_off = (uint32_t*)malloc(sizeof(uint32_t) * (F->n_trees ? F->n_trees : 1));
    uint32_t* leaf_cnt = (uint32_t*)malloc(sizeof(uint32_t) * (F->n_trees ? F->n_trees : 1));
    for (uint32_t t = 0; t < F->n_trees; ++t) {
        uint32_t v = F->root[t];
        while (F->feature[v] != OG_LEAF)
            v = x[F->feature[v]] <= F->threshold[v] ? F->left[v] : F->right[v];
        leaf_off[t] = F->threshold[v]; leaf_cnt[t] = F->left[v];
        cap += F->left[v];
    }
    uint32_t* pool = (uint32_t*)malloc(sizeof(uint32_t) * (cap ? cap : 1));
    uint32_t m = 0;
    for (uint32_t t = 0; t < F->n_trees; ++t)
        for (uint32_t i = 0; i < leaf_cnt[t]; ++i) {
            uint32_t y = F->samples[leaf_off[t] + i];
            if (y > anchor) pool[m++] = y;
        }
    uint32_t q = l_max;
    if (m) {
        qsort(pool, m, sizeof(uint32_t), cmp_u32);
        uint64_t k = ((uint64_t)q_num * m + q_den - 1) / q_den;   /* ceil(q m) >= 1 */
        q = pool[k - 1];
    }
    free(pool); free(leaf_off); free(leaf_cnt);
    return q;
}

/* exported for the pins: Lhat = max(Q_q(L | L > R*floor(g/R)), g + 1) */
uint32_t og_length_bound(const og_table* T, uint32_t row, uint32_t g, uint32_t R,
                         uint32_t q_num, uint32_t q_den) {
    uint32_t anchor = R * (g / R);
    uint32_t q = cond_quantile_scan(T, row, anchor, q_num, q_den);
    return q > g + 1 ? q : g + 1;
}

void og_reset_memo(void) {
    free(g_qmemo); g_qmemo = NULL; g_qmemo_tab = NULL; g_qmemo_rows = 0;
}

/* ------------------------------------------------------------------------------------ */
/* Per-request analysis (Alg. 1 AnalyzeRequest; §4.2; App. B) */
/* ------------------------------------------------------------------------------------ */

static inline uint32_t m_group(uint32_t m) { return m & 0xFFu; }
static inline uint32_t m_state(uint32_t m) { return (m >> 8) & 0xFu; }
static inline uint32_t m_flags(uint32_t m) { return (m >> 12) & 0xFu; }
static inline uint32_t m_set_state(uint32_t m, uint32_t s) { return (m & ~0xF00u) | (s << 8); }
static inline uint32_t m_set_flags(uint32_t m, uint32_t f) { return (m & ~0xF000u) | (f << 12); }
static inline uint32_t a_row(uint32_t a) { return a & 0xFFFFu; }
static inline uint32_t a_waited(uint32_t a) { return a >> 16; }

/* key = fl((G' * 10^9) / (t_gen + eps)); §4.2 P:462-467 Priority = goodput / t_gen, with the
 * App. B indicator's eps (reading A1/A2); G' = G + delta * floor(waited / Delta)
 * (starvation inflation P:467, reading A12).  Returns -1 when an operand leaves 2^53. */
static int make_key(uint64_t Gp, uint64_t t_gen, int64_t eps, double* out) {
    const uint64_t LIM = (uint64_t)1 << 53;
    if (Gp >= LIM / 1000000000ull) return -1;
    uint64_t A = Gp * 1000000000ull;
    uint64_t B = t_gen + (uint64_t)eps;
    if (B >= LIM || B < t_gen) return -1;
    *out = (double)A / (double)B;
    return 0;
}

/* reported JIT rate (tokens/s): len_rem * 10^9 / t_rem; +inf when t_rem <= 0 (A38) */
/* NEXT-2 (§4.3): priority'(r) = (1 - f) * priority(r) + f * Fair(r), f = num / den,
 * Fair(r) a developer-supplied non-negative integer score in key units (reading A47).  Written
 * over the common denominator: fl( fl( fl(key * (den - num)) + num * Fair ) / den ), three IEEE
 * operations in this order (num * Fair is an exact integer < 2^53).  f = 0 leaves the key. */
static double blend_fair(double key, uint32_t fair, uint32_t num, uint32_t den) {
    if (num == 0) return key;
    double a = key * (double)(den - num);
    double b = (double)((uint64_t)num * fair);
    return (a + b) / (double)den;
}

static double make_rate(uint64_t len_rem, int64_t t_rem) {
    if (t_rem <= 0) return __builtin_inf();
    return (double)(len_rem * 1000000000ull) / (double)t_rem;
}

/* (a6) per-step token cost: 1 for a decode step, else the next prefill chunk (A25) */
static uint32_t token_cost(uint32_t input_len, uint32_t prefilled, uint32_t chunk) {
    if (prefilled >= input_len) return 1;
    uint32_t rem = input_len - prefilled;
    return rem < chunk ? rem : chunk;
}

/* A19: exact fixed-point image floor(min(key, 2^31-1) * 2^32) used for window sums */
static uint64_t fixed_point(double key) {
    double k = key < 2147483647.0 ? key : 2147483647.0;
    return (uint64_t)(k * 4294967296.0);
}

/* ------------------------------------------------------------------------------------ */
/* One GMAX step over a request pool (Alg. 1 Schedule)                        */
/* ------------------------------------------------------------------------------------ */

typedef struct { double key; uint32_t id; uint32_t row; } by_key_t;
typedef struct { uint64_t len; uint32_t id; uint32_t row; } by_len_t;

static int cmp_key_desc_id_asc(const void* a, const void* b) {
    const by_key_t* x = (const by_key_t*)a; const by_key_t* y = (const by_key_t*)b;
    if (x->key > y->key) return -1;
    if (x->key < y->key) return 1;
    return (x->id > y->id) - (x->id < y->id);
}
static int cmp_len_asc_id_asc(const void* a, const void* b) {
    const by_len_t* x = (const by_len_t*)a; const by_len_t* y = (const by_len_t*)b;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* task view for the compound pass (a4) and the task-level admission drop (a1, reading A40) */
typedef struct {
    uint32_t n;
    const uint32_t* call_begin; const uint32_t* call_end;   /* current-stage rows */
    const int64_t* arrival_ns; const int64_t* deadline_ns;  /* a_c, D */
    const uint64_t* t_le_s; const uint64_t* t_total;        /* phi(s) = t_le_s / t_total */
    const int64_t* stage_deadline_ns;                        /* NULL or per task (< 0: from phi) */
    const uint64_t* goodput_done;
    const uint8_t* ever;                                     /* 1: some call of the task was scheduled */
    uint8_t* dropped;                                        /* out (may be NULL): 1 if dropped now */
} task_view;

/* ------------------------------------------------------------------------------------ */
/* NEXT-1: the preemption gate over GMAX's proposal (reading A46).                       */
/* §4.2: "performs preemption only when the projected gain from admitting a    */
/* higher-priority request exceeds [goodput_loss = stall_duration x token_generation_    */
/* speed]" and "scheduling updates are restricted to discrete time frames (Delta = 50    */
/* decoding steps)"; App. D.2: A may preempt the running B only if           */
/* R(A)/R(B) > 1 + delta (delta_pmtn = 0.1); S:313-321 preemption_check.          */
/*                                                                                        */
/* Running set P = the pending requests in state Running (with the gate on, Running means */
/* "in the batch the engine executes": the gate's bookkeeping keeps it so).  Q = GMAX's    */
/* window (a9).  Walk, in this order:                                                      */
/*  1. P in (key desc, id asc): a running request keeps its slot while |F| < B_max and its */
/*     cost fits the budget; one that does not fit is evicted (no gate: it cannot run).    */
/*  2. I = Q \ P in (key desc, id asc).  A newcomer takes a free slot when one is left and */
/*     its cost fits.  Otherwise, only at a frame boundary, it is paired with the weakest   */
/*     running request still kept and not in Q (P walked from its end: key asc, later id   */
/*     first); the swap happens iff                                                        */
/*        cost(in) <= budget_left + cost(out),                                             */
/*        key(in) > key(out) * fl((den + num) / den)                 (App. D.2 ratio),     */
/*        (key(in) - key(out)) * fl(Delta * v / 1e9) > fl(stall(out) / v),   */
/*     with stall(out) = floor(kv(out) * 1e9 / io_bw) ns, kv = prefilled + generated tokens */
/*     (KV size = context length), gen speed 1/v tokens per ns, the gain counted     */
/*     over one frame of Delta steps.  A failed pair skips the newcomer (the candidate stays).*/
/* Every floating-point operation is one IEEE round-to-nearest operation in this order.   */
/* ------------------------------------------------------------------------------------ */
static void gate(const og_config* cfg, uint32_t n, const uint32_t* id, const uint32_t* input_len,
                 const uint32_t* generated, const uint32_t* prefilled, const uint32_t* meta,
                 const double* key, const uint32_t* cost, const uint8_t* pend,
                 const by_len_t* Q, uint32_t nq, int64_t v_token, uint32_t frame_open,
                 uint8_t* inF, uint8_t* evict, og_result* res) {
    (void)input_len;
    uint8_t* inQ = (uint8_t*)calloc(n ? n : 1, 1);
    for (uint32_t i = 0; i < nq; ++i) inQ[Q[i].row] = 1;
    by_key_t* P = (by_key_t*)malloc(sizeof(by_key_t) * (n ? n : 1));
    by_key_t* I = (by_key_t*)malloc(sizeof(by_key_t) * (nq ? nq : 1));
    uint32_t np = 0, ni = 0;
    for (uint32_t r = 0; r < n; ++r)
        if (pend[r] && m_state(meta[r]) == ST_RUNNING) { P[np].key = key[r]; P[np].id = id[r]; P[np].row = r; ++np; }
    for (uint32_t i = 0; i < nq; ++i) {
        uint32_t r = Q[i].row;
        if (m_state(meta[r]) != ST_RUNNING) { I[ni].key = key[r]; I[ni].id = id[r]; I[ni].row = r; ++ni; }
    }
    qsort(P, np, sizeof(by_key_t), cmp_key_desc_id_asc);
    qsort(I, ni, sizeof(by_key_t), cmp_key_desc_id_asc);
    uint64_t budget = cfg->token_budget;
    uint32_t slots = cfg->max_batch;
    /* 1. running requests continue while they fit */
    for (uint32_t k = 0; k < np; ++k) {
        uint32_t r = P[k].row;
        if (slots >= 1 && cost[r] <= budget) { inF[r] = 1; --slots; budget -= cost[r]; }
        else evict[r] = 1;
    }
    /* 2. newcomers: a free slot, else a gated swap at a frame boundary */
    double onepd = (double)((uint64_t)cfg->pmtn_den + cfg->pmtn_num) / (double)cfg->pmtn_den;
    double fs = (double)((uint64_t)cfg->frame_steps * (uint64_t)v_token) / 1e9;
    uint32_t o = np;                                   /* candidates: P[o-1], P[o-2], ... */
    for (uint32_t k = 0; k < ni; ++k) {
        uint32_t r = I[k].row;
        if (slots >= 1 && cost[r] <= budget) { inF[r] = 1; --slots; budget -= cost[r]; continue; }
        if (!frame_open) continue;
        while (o > 0 && !(inF[P[o - 1].row] && !inQ[P[o - 1].row])) --o;
        if (o == 0) continue;
        uint32_t q = P[o - 1].row;
        uint64_t kv = (uint64_t)prefilled[q] + generated[q];
        int64_t stall = (int64_t)((u128)kv * 1000000000u / cfg->io_bw_tps);
        double loss = (double)stall / (double)v_token;
        double gain = (key[r] - key[q]) * fs;
        if (cost[r] <= budget + cost[q] && key[r] > key[q] * onepd && gain > loss) {
            inF[q] = 0; evict[q] = 1; inF[r] = 1;
            budget = budget + cost[q] - cost[r];
            --o;
        }
    }
    uint32_t ns = 0, tot = 0, ne = 0; int64_t stall_sum = 0;
    for (uint32_t r = 0; r < n; ++r) {
        if (inF[r]) { ++ns; tot += cost[r]; }
        if (evict[r]) {
            ++ne;
            stall_sum += (int64_t)((u128)((uint64_t)prefilled[r] + generated[r]) * 1000000000u / cfg->io_bw_tps);
        }
    }
    res->n_selected = ns; res->total_tokens = tot; res->n_preempted = ne; res->stall_ns = stall_sum;
    free(inQ); free(P); free(I);
}

/* The step.  On return, selected[0..n_selected) holds ROW indices in batch order. */
static int gmax_step(const og_config* cfg, const og_group* G, uint32_t n_groups,
                     const og_table* T, int64_t now, int64_t v_token,
                     uint32_t n, const uint32_t* id, const int64_t* arrival,
                     const uint32_t* input_len, const uint32_t* generated,
                     const uint32_t* prefilled, uint32_t* meta, uint32_t* aux,
                     const uint32_t* task, const uint32_t* override_R, const uint32_t* fair,
                     const task_view* TV,
                     og_result* res, uint32_t* selected, uint32_t* sel_cost,
                     const og_rows_out* ro, uint32_t frame_open) {
    memset(res, 0, sizeof(*res));
    if (cfg->refine_interval == 0 || cfg->frame_steps == 0 || cfg->q_den == 0 ||
        cfg->p_den == 0 || cfg->q_num == 0 || cfg->q_num > cfg->q_den || cfg->p_num == 0 ||
        cfg->p_num > cfg->p_den || cfg->prefill_chunk == 0 ||
        cfg->prefill_chunk > cfg->token_budget || cfg->max_batch == 0 || v_token <= 0 ||
        cfg->eps_ns <= 0 || (cfg->preempt && (cfg->pmtn_den == 0 || cfg->io_bw_tps == 0)) ||
        (cfg->fair_num && cfg->fair_num > cfg->fair_den)) {
        res->error = 1; return OG_EINVAL;
    }

    double* key = (double*)calloc(n ? n : 1, sizeof(double));
    uint32_t* lhat = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    uint32_t* cost = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    uint8_t* pend = (uint8_t*)calloc(n ? n : 1, 1);
    int64_t* trem = (int64_t*)calloc(n ? n : 1, sizeof(int64_t));
    double* rate = (double*)calloc(n ? n : 1, sizeof(double));
    int rc = OG_OK;

    /* (a1) admission control, P:545 ("requests unscheduled beyond [waiting_time] are dropped",
     * A29 strict) + pending set (Alg. 1 GetRequestQueue).  Reading A40: a compound task is
     * ONE API request (the API of P:544 creates it); it is dropped when none of its calls has ever
     * been scheduled and now - a_c > waiting_time, and dropping it drops every call of it that is
     * still Queued or Waiting.  A standalone request is dropped by its own arrival and flag. */
    uint32_t n_pend = 0;
    if (TV) {
        for (uint32_t t = 0; t < TV->n; ++t) {
            if (TV->dropped) TV->dropped[t] = 0;
            if (TV->ever[t] || now - TV->arrival_ns[t] <= cfg->waiting_ns) continue;
            uint32_t hit = 0;
            for (uint32_t r = TV->call_begin[t]; r < TV->call_end[t]; ++r) {
                uint32_t st = m_state(meta[r]);
                if (st == ST_QUEUED || st == ST_WAITING) {
                    meta[r] = m_set_state(meta[r], ST_DROPPED);
                    res->n_dropped_now++;
                    hit = 1;
                }
            }
            if (TV->dropped) TV->dropped[t] = (uint8_t)hit;
        }
    }
    for (uint32_t r = 0; r < n; ++r) {
        uint32_t m = meta[r], st = m_state(m), fl = m_flags(m);
        if (arrival[r] > now) continue;
        if (st == ST_QUEUED && !(fl & FL_EVER) && !(fl & FL_COMPOUND) &&
            now - arrival[r] > cfg->waiting_ns) {
            meta[r] = m_set_state(m, ST_DROPPED);
            res->n_dropped_now++;
            continue;
        }
        if (st == ST_QUEUED || st == ST_RUNNING || st == ST_PREEMPTED) { pend[r] = 1; ++n_pend; }
    }

    /* AnalyzeRequest for every pending standalone request */
    for (uint32_t r = 0; r < n && rc == OG_OK; ++r) {
        if (!pend[r]) continue;
        uint32_t m = meta[r], gi = m_group(m);
        if (gi >= n_groups || a_row(aux[r]) >= T->n_rows || input_len[r] == 0) { rc = OG_EINVAL; break; }
        uint32_t g = generated[r];
        /* (a2) PredictLength: conditional upper quantile, refined every R tokens */
        uint32_t anchor = cfg->refine_interval * (g / cfg->refine_interval);
        uint32_t q;
        if (T->forest) {                                        /* NEXT-4: the QRF (A50) */
            uint32_t x[4] = { input_len[r], a_row(aux[r]), anchor, gi };
            q = og_qrf_quantile(T->forest, x, anchor, cfg->q_num, cfg->q_den, T->l_max);
        } else {
            q = cond_quantile(T, a_row(aux[r]), anchor, cfg->q_num, cfg->q_den, cfg->refine_interval);
        }
        lhat[r] = q > g + 1 ? q : g + 1;
        cost[r] = token_cost(input_len[r], prefilled[r], cfg->prefill_chunk);
        if (m_flags(m) & FL_COMPOUND) continue;                 /* handled by (a4) below */
        const og_group* gr = &G[gi];
        uint64_t len_rem = (uint64_t)(lhat[r] - g);
        uint64_t t_gen = len_rem * (uint64_t)v_token;          /* P:447 t_gen = len_rem * v_token */
        /* (a3) EstimateRemainingTime per SLO type (reading A9 for LAT) */
        int64_t t_rem;
        switch (gr->type) {
            case OG_LAT: t_rem = arrival[r] + gr->ttft_ns + (int64_t)(lhat[r] - 1) * gr->tbt_ns - now; break;
            case OG_DDL: t_rem = arrival[r] + gr->e2el_ns - now; break;
            case OG_BE:  t_rem = arrival[r] + gr->be_deadline_ns - now; break;
            default: rc = OG_EINVAL; continue;  /* CMP group on a non-compound row */
        }
        /* (a5) EstimateGoodput (reading A10/A11; App. B R(k) P:905-908) */
        uint64_t Gk;
        if (gr->type == OG_DDL) Gk = (uint64_t)gr->w_in * input_len[r] + (uint64_t)gr->w_out * lhat[r];
        else if (gr->type == OG_LAT) Gk = (uint64_t)gr->w_out * lhat[r];
        else Gk = 0;                                             /* best effort: starvation only */
        if (m_flags(m) & FL_OVERRIDE) Gk = override_R[r];       /* App. D sets R(k) directly */
        if (t_rem <= 0) Gk = 0;                                  /* expired (A22) */
        if (cfg->appb_filter && t_gen > (uint64_t)(t_rem > 0 ? t_rem : 0)) Gk = 0; /* App. B filter */
        uint64_t Gp = Gk + (uint64_t)cfg->delta_starve * (a_waited(aux[r]) / cfg->frame_steps);
        if (make_key(Gp, t_gen, cfg->eps_ns, &key[r]) != 0) { rc = OG_EINVAL; break; }
        trem[r] = t_rem;
        rate[r] = make_rate(len_rem, t_rem);
    }

    /* (a4) compound requests: len_rem and bandwidth aggregated over all subrequests of the
     * current stage; stage sub-deadline D_s = phi(s) * D. */
    if (rc == OG_OK && TV) {
        for (uint32_t t = 0; t < TV->n && rc == OG_OK; ++t) {
            uint64_t Tsum = 0, Gcur = 0; uint32_t cnt = 0;
            for (uint32_t r = TV->call_begin[t]; r < TV->call_end[t]; ++r) {
                if (!pend[r]) continue;
                const og_group* gr = &G[m_group(meta[r])];
                Tsum += (uint64_t)(lhat[r] - generated[r]);
                Gcur += (uint64_t)gr->w_in * input_len[r] + (uint64_t)gr->w_out * lhat[r];
                ++cnt;
            }
            if (!cnt) continue;
            uint64_t Gtask = TV->goodput_done[t] + Gcur;
            if (TV->arrival_ns[t] + TV->deadline_ns[t] <= now) Gtask = 0;   /* final deadline passed */
            if (TV->t_total[t] == 0) { rc = OG_EINVAL; break; }
            int64_t Ds = (int64_t)((u128)(uint64_t)TV->deadline_ns[t] * TV->t_le_s[t] / TV->t_total[t]);
            int64_t t_rem = TV->arrival_ns[t] + Ds - now;                  /* advisory */
            if (TV->stage_deadline_ns && TV->stage_deadline_ns[t] >= 0) t_rem = TV->stage_deadline_ns[t] - now;
            uint64_t t_gen = Tsum * (uint64_t)v_token;
            if (cfg->appb_filter && t_gen > (uint64_t)(t_rem > 0 ? t_rem : 0)) Gtask = 0;
            for (uint32_t r = TV->call_begin[t]; r < TV->call_end[t]; ++r) {
                if (!pend[r]) continue;
                uint64_t Gp = Gtask + (uint64_t)cfg->delta_starve * (a_waited(aux[r]) / cfg->frame_steps);
                if (make_key(Gp, t_gen, cfg->eps_ns, &key[r]) != 0) { rc = OG_EINVAL; break; }
                trem[r] = t_rem;
                rate[r] = make_rate(Tsum, t_rem);
            }
        }
    }
    /* NEXT-2 fairness blend of every pending request's priority (A47), before (a7)-(a9) */
    if (rc == OG_OK && cfg->fair_num)
        for (uint32_t r = 0; r < n; ++r)
            if (pend[r]) key[r] = blend_fair(key[r], fair ? fair[r] : 0u, cfg->fair_num, cfg->fair_den);
    /* every row of a task range must be a compound call of that task with a CMP group */
    if (rc == OG_OK && TV)
        for (uint32_t t = 0; t < TV->n && rc == OG_OK; ++t)
            for (uint32_t r = TV->call_begin[t]; r < TV->call_end[t]; ++r)
                if (!(m_flags(meta[r]) & FL_COMPOUND) || task[r] != t || m_group(meta[r]) >= n_groups ||
                    G[m_group(meta[r])].type != OG_CMP) { rc = OG_EINVAL; break; }
    /* every pending compound row must have been covered by a task */
    for (uint32_t r = 0; r < n && rc == OG_OK; ++r)
        if (pend[r] && (m_flags(meta[r]) & FL_COMPOUND) && (!TV || task[r] == NO_TASK ||
            task[r] >= TV->n || r < TV->call_begin[task[r]] || r >= TV->call_end[task[r]]))
            rc = OG_EINVAL;

    if (ro) {
        for (uint32_t r = 0; r < n; ++r) {
            if (ro->key) ro->key[r] = pend[r] ? key[r] : -1.0;
            if (ro->rate) ro->rate[r] = pend[r] ? rate[r] : 0.0;
            if (ro->t_rem) ro->t_rem[r] = pend[r] ? trem[r] : 0;
            if (ro->lhat) ro->lhat[r] = pend[r] ? lhat[r] : 0;
            if (ro->cost) ro->cost[r] = pend[r] ? cost[r] : 0;
            if (ro->pending) ro->pending[r] = pend[r];
        }
    }
    res->n_pending = n_pend;
    if (rc != OG_OK) { res->error = 1; goto out; }
    if (n_pend == 0) { rc = OG_EMPTY; goto out; }

    {
        /* (a7) BatchPriority (Alg. 1; §4.2): order by (key desc, id asc); B* is
         * the largest prefix within the token budget and max_batch (A14); bp its last key. */
        by_key_t* P = (by_key_t*)malloc(sizeof(by_key_t) * n_pend);
        uint32_t k = 0;
        for (uint32_t r = 0; r < n; ++r) if (pend[r]) { P[k].key = key[r]; P[k].id = id[r]; P[k].row = r; ++k; }
        qsort(P, n_pend, sizeof(by_key_t), cmp_key_desc_id_asc);
        uint64_t csum = 0; uint32_t bstar = 0;
        while (bstar < n_pend && bstar + 1 <= cfg->max_batch &&
               csum + cost[P[bstar].row] <= cfg->token_budget) {
            csum += cost[P[bstar].row]; ++bstar;
        }
        double bp = P[bstar - 1].key;   /* bstar >= 1 because every cost <= chunk <= budget */
        /* (a8) Filter (Alg. 1): key >= fl(fl(p_num/p_den) * bp) (A16) */
        double p = (double)cfg->p_num / (double)cfg->p_den;
        double thr = p * bp;
        uint32_t ncd = 0;
        for (uint32_t i = 0; i < n_pend; ++i) if (P[i].key >= thr) ++ncd;
        by_len_t* Cd = (by_len_t*)malloc(sizeof(by_len_t) * ncd);
        uint32_t c = 0;
        for (uint32_t i = 0; i < n_pend; ++i) {
            if (P[i].key < thr) continue;
            uint32_t r = P[i].row;
            Cd[c].len = cfg->len_key ? (uint64_t)input_len[r] + generated[r] : (uint64_t)input_len[r];
            Cd[c].id = id[r]; Cd[c].row = r; ++c;
        }
        /* (a9) sort candidates by input length (Alg. 1; A17 tie by id), then slide a
         * window and keep the first maximum of sum(priority) (strict '>'). */
        qsort(Cd, ncd, sizeof(by_len_t), cmp_len_asc_id_asc);
        u128* pf = (u128*)malloc(sizeof(u128) * (ncd + 1));
        uint64_t* pc = (uint64_t*)malloc(sizeof(uint64_t) * (ncd + 1));
        pf[0] = 0; pc[0] = 0;
        for (uint32_t i = 0; i < ncd; ++i) {
            pf[i + 1] = pf[i] + fixed_point(key[Cd[i].row]);
            pc[i + 1] = pc[i] + cost[Cd[i].row];
        }
        u128 best = 0; int have = 0; uint32_t bi = 0, bj = 0, j = 0;
        for (uint32_t i = 0; i < ncd; ++i) {
            /* j(i): the largest j with sum_{i..j} c <= budget and j-i+1 <= max_batch; j(i) is
             * nondecreasing in i, so it is extended from j(i-1). */
            if (j < i) j = i;
            while (j + 1 < ncd && pc[j + 2] - pc[i] <= cfg->token_budget &&
                   (j + 1) - i + 1 <= cfg->max_batch) ++j;
            u128 score = pf[j + 1] - pf[i];
            if (!have || score > best) { best = score; bi = i; bj = j; have = 1; }
        }
        res->n_candidates = ncd; res->b_star = bstar; res->bp = bp; res->thr = thr;
        uint8_t* insel = (uint8_t*)calloc(n, 1);
        uint8_t* evict = (uint8_t*)calloc(n, 1);
        if (!cfg->preempt) {
            /* BestGroup is the batch */
            uint32_t tot = 0;
            for (uint32_t i = bi; i <= bj; ++i) {
                selected[i - bi] = Cd[i].row;
                if (sel_cost) sel_cost[i - bi] = cost[Cd[i].row];
                tot += cost[Cd[i].row];
                insel[Cd[i].row] = 1;
            }
            res->n_selected = bj - bi + 1; res->total_tokens = tot;
        } else {
            gate(cfg, n, id, input_len, generated, prefilled, meta, key, cost, pend, Cd + bi, bj - bi + 1,
                 v_token, frame_open, insel, evict, res);
            /* the batch in window order (len asc, id asc; A20) */
            by_len_t* F = (by_len_t*)malloc(sizeof(by_len_t) * (res->n_selected ? res->n_selected : 1));
            uint32_t f = 0;
            for (uint32_t r = 0; r < n; ++r) {
                if (!insel[r]) continue;
                F[f].len = cfg->len_key ? (uint64_t)input_len[r] + generated[r] : (uint64_t)input_len[r];
                F[f].id = id[r]; F[f].row = r; ++f;
            }
            qsort(F, f, sizeof(by_len_t), cmp_len_asc_id_asc);
            for (uint32_t i = 0; i < f; ++i) {
                selected[i] = F[i].row;
                if (sel_cost) sel_cost[i] = cost[F[i].row];
            }
            free(F);
        }

        /* bookkeeping after selection: ever_scheduled / Running for the batch, Preempted for the
         * requests the gate evicted, and steps_waited += 1 (saturating at 0xFFFF) for every
         * pending request left out; a selected request keeps its counter ("per frame"
         * waited; reading A12) */
        for (uint32_t r = 0; r < n; ++r) {
            if (!pend[r]) continue;
            if (insel[r]) {
                uint32_t m = meta[r];
                m = m_set_flags(m, m_flags(m) | FL_EVER);
                if (m_state(m) == ST_QUEUED || m_state(m) == ST_PREEMPTED) m = m_set_state(m, ST_RUNNING);
                meta[r] = m;
            } else {
                if (evict[r]) meta[r] = m_set_state(meta[r], ST_PREEMPTED);
                uint32_t w = a_waited(aux[r]);
                if (w < 0xFFFFu) ++w;
                aux[r] = (aux[r] & 0xFFFFu) | (w << 16);
            }
        }
        free(evict);
        free(insel); free(pf); free(pc); free(Cd); free(P);
    }
out:
    free(key); free(lhat); free(cost); free(pend); free(trem); free(rate);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* Public: one step over a pool snapshot                                                */
/* ------------------------------------------------------------------------------------ */

int og_step(const og_config* cfg, const og_group* groups, uint32_t n_groups,
            const og_table* T, int64_t now_ns, int64_t v_token_ns,
            const og_pool* pool, const og_tasks* tasks,
            og_result* res, uint32_t* batch_ids, uint32_t* batch_tokens, uint32_t* batch_rows,
            const og_rows_out* ro, uint32_t frame_open) {
    uint32_t n = pool->n;
    og_reset_memo();                 /* the memo lives for one call only */
    task_view tv; task_view* tvp = NULL;
    uint32_t *cb = NULL, *ce = NULL; uint64_t *tle = NULL, *tt = NULL; uint8_t* tever = NULL;
    if (tasks && tasks->n) {
        uint32_t nt = tasks->n;
        cb = (uint32_t*)malloc(4 * nt); ce = (uint32_t*)malloc(4 * nt);
        tle = (uint64_t*)malloc(8 * nt); tt = (uint64_t*)malloc(8 * nt);
        tever = (uint8_t*)calloc(nt, 1);
        for (uint32_t t = 0; t < nt; ++t) {
            cb[t] = tasks->call_off[t]; ce[t] = tasks->call_off[t + 1];
            uint32_t S = tasks->n_stages[t], s = tasks->cur_stage[t];
            if (S == 0 || S > MAX_STAGES || s >= S || ce[t] < cb[t] || ce[t] > n) {
                res->error = 1; free(cb); free(ce); free(tle); free(tt); free(tever); return OG_EINVAL;
            }
            /* A40: the task has been scheduled iff one of its calls in the pool carries ever_scheduled */
            for (uint32_t r = cb[t]; r < ce[t]; ++r)
                if (m_flags(pool->meta[r]) & FL_EVER) tever[t] = 1;
            /* phi(s) = t_{<=s} / t_total over the matched pattern */
            uint64_t le = 0, tot = 0;
            for (uint32_t u = 0; u < S; ++u) {
                uint64_t ns = (uint64_t)tasks->pattern_ms[(size_t)t * MAX_STAGES + u] * 1000000ull;
                tot += ns; if (u <= s) le += ns;
            }
            tle[t] = le; tt[t] = tot;
        }
        tv.n = nt; tv.call_begin = cb; tv.call_end = ce; tv.arrival_ns = tasks->arrival_ns;
        tv.deadline_ns = tasks->deadline_ns; tv.t_le_s = tle; tv.t_total = tt;
        tv.goodput_done = tasks->goodput_done;
        tv.ever = tever; tv.dropped = NULL; tv.stage_deadline_ns = tasks->stage_deadline_ns;
        tvp = &tv;
    }
    uint32_t* sel = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint32_t* sc = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    int rc = gmax_step(cfg, groups, n_groups, T, now_ns, v_token_ns, n, pool->id, pool->arrival_ns,
                       pool->input_len, pool->generated, pool->prefilled, pool->meta, pool->aux,
                       pool->task, pool->override_R, pool->fair, tvp, res, sel, sc, ro, frame_open);
    if (rc == OG_OK) {
        for (uint32_t i = 0; i < res->n_selected; ++i) {
            if (batch_ids) batch_ids[i] = pool->id[sel[i]];
            if (batch_tokens) batch_tokens[i] = sc[i];
            if (batch_rows) batch_rows[i] = sel[i];
        }
    }
    free(sel); free(sc); free(cb); free(ce); free(tle); free(tt); free(tever);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* (a10) Trace replay: iteration cost model, token timestamps,  */
/* goodput accounting (§3), stage barriers, v_token as the */
/* floor of the trailing mean of the last Delta iteration latencies (A24).          */
/* ------------------------------------------------------------------------------------ */

typedef struct {
    uint32_t n_rows, n_tasks;
    const int64_t* arrival_ns;      /* standalone rows; ignored for compound calls */
    const uint32_t* input_len;
    const uint32_t* true_out;       /* L_o >= 1 (hidden from the scheduler) */
    const uint32_t* group;
    const uint32_t* dist_row;
    const uint32_t* override_R;
    const uint32_t* task;           /* NO_TASK or the owning task */
    const int64_t* task_arrival_ns;
    const int64_t* task_deadline_ns;       /* D relative to a_c (before SLO scaling) */
    const uint32_t* task_n_stages;
    const uint32_t* stage_kind;            /* n_tasks*8: 0 LLM, 1 tool */
    const int64_t* stage_exec_ns;          /* n_tasks*8: tool time */
    const uint32_t* stage_pattern_ms;      /* n_tasks*8: matched-pattern stage time */
    const uint32_t* stage_call_begin;      /* n_tasks*8: rows of an LLM stage */
    const uint32_t* stage_call_end;
    const uint32_t* fair;                  /* NULL or Fair(r) per row (NEXT-2 blend, A47) */
} og_trace;

typedef struct {
    uint32_t n_steps, log_ids;
    int64_t v_token0_ns, c0_ns, c_att_ns, c_lin_ns;
    uint64_t load_num, load_den, slo_num, slo_den;   /* arrival' = a*load_den/load_num; SLO' = t*slo_num/slo_den */
    /* NEXT-2 online adaptation of p (reading A48): epsilon-greedy over P_GRID, one arm per
     * window of window_frames frames (window_frames * frame_steps steps); 0 = off */
    uint32_t p_adapt, eps_num, eps_den, window_frames;
    uint64_t seed;
} og_replay_cfg;

typedef struct {
    uint64_t token_goodput, tokens_processed;
    int64_t sim_end_ns;
    uint32_t request_goodput, n_done, n_dropped, steps, n_tasks_done, n_tasks_dropped, error, n_preempted;
} og_replay_result;

typedef struct {
    int64_t now_ns;
    uint32_t n_selected, total_tokens, n_candidates, b_star;
    double bp;
    uint64_t ids_hash;
    int64_t v_token_ns;   /* the v_token the step's keys used */
    uint32_t n_preempted, p_num;  /* requests the gate evicted this step (A46); the cutoff p_num used (A48) */
    int64_t stall_ns;             /* their KV swap stall, part of this iteration's latency */
} og_step_log;

static uint64_t fnv1a_ids(const uint32_t* ids, uint32_t n) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t i = 0; i < n; ++i)
        for (int b = 0; b < 4; ++b) { h ^= (ids[i] >> (8 * b)) & 0xFFu; h *= 1099511628211ull; }
    return h;
}

/* NEXT-2 online p ("automates and continuously adapts p online by exploring different
 * thresholds and converging to those that maximize end-to-end goodput"; reading A48, after SPEC
 * S:361): arms P_GRID / 100; each window of W = window_frames * frame_steps steps runs one arm and
 * scores it by the token goodput earned in that window.  Untried arms go first, in grid order;
 * then with probability eps_num / eps_den a uniformly drawn arm, else the arm of the highest
 * mean window goodput (sum / count compared exactly by cross products; the lowest index on a
 * tie).  The draws come from the counter-based splitmix64 of (seed + window index). */
static const uint32_t P_GRID[4] = { 80, 90, 95, 100 };
static uint64_t splitmix64_at(uint64_t x) {
    uint64_t z = x * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint32_t next_arm(const og_replay_cfg* rc, const uint64_t* gsum, const uint32_t* gcnt, uint64_t window) {
    for (uint32_t a = 0; a < 4; ++a) if (gcnt[a] == 0) return a;
    uint64_t u = splitmix64_at(rc->seed + window);
    if (u % rc->eps_den < rc->eps_num) return (uint32_t)((u >> 32) % 4u);
    uint32_t best = 0;
    for (uint32_t a = 1; a < 4; ++a)        /* mean_a > mean_best <=> sum_a * cnt_best > sum_best * cnt_a */
        if ((u128)gsum[a] * gcnt[best] > (u128)gsum[best] * gcnt[a]) best = a;
    return best;
}

int og_replay(const og_config* cfg, const og_group* groups_in, uint32_t n_groups,
              const og_table* T, const og_trace* tr, const og_replay_cfg* rc,
              og_replay_result* out, og_step_log* log, uint32_t* log_ids) {
    memset(out, 0, sizeof(*out));
    og_reset_memo();
    uint32_t n = tr->n_rows, nt = tr->n_tasks;
    if (!rc->load_num || !rc->load_den || !rc->slo_num || !rc->slo_den || n_groups > 256 ||
        (rc->p_adapt && (!rc->eps_den || rc->eps_num > rc->eps_den || !rc->window_frames))) { out->error = 1; return OG_EINVAL; }
    og_config cf = *cfg;                        /* p_num changes per window when p adapts (A48) */
    uint64_t gsum[4] = {0, 0, 0, 0}, g_start = 0, window = 0;
    uint32_t gcnt[4] = {0, 0, 0, 0}, arm = 0;
    if (rc->p_adapt) { cf.p_num = P_GRID[0]; cf.p_den = 100; }
    /* SLO scaling of the group table (§6.4 P:784-786 sweep shape) */
    og_group G[256];
    for (uint32_t g = 0; g < n_groups; ++g) {
        G[g] = groups_in[g];
        G[g].ttft_ns = (int64_t)((u128)(uint64_t)G[g].ttft_ns * rc->slo_num / rc->slo_den);
        G[g].tbt_ns = (int64_t)((u128)(uint64_t)G[g].tbt_ns * rc->slo_num / rc->slo_den);
        G[g].e2el_ns = (int64_t)((u128)(uint64_t)G[g].e2el_ns * rc->slo_num / rc->slo_den);
        G[g].be_deadline_ns = (int64_t)((u128)(uint64_t)G[g].be_deadline_ns * rc->slo_num / rc->slo_den);
    }
    uint32_t* id = (uint32_t*)malloc(4 * (n + 1));
    int64_t* arr = (int64_t*)malloc(8 * (n + 1));
    uint32_t* gen = (uint32_t*)calloc(n + 1, 4);
    uint32_t* pre = (uint32_t*)calloc(n + 1, 4);
    uint32_t* meta = (uint32_t*)malloc(4 * (n + 1));
    uint32_t* aux = (uint32_t*)malloc(4 * (n + 1));
    uint8_t* late = (uint8_t*)calloc(n + 1, 1);
    uint32_t* sel = (uint32_t*)malloc(4 * (n + 1));
    uint32_t* selc = (uint32_t*)malloc(4 * (n + 1));
    uint32_t* selid = (uint32_t*)malloc(4 * (n + 1));
    /* task state */
    uint32_t* cur = (uint32_t*)calloc(nt + 1, 4);
    uint32_t* left = (uint32_t*)calloc(nt + 1, 4);
    uint8_t* tdone = (uint8_t*)calloc(nt + 1, 1);
    int64_t* timer = (int64_t*)malloc(8 * (nt + 1));
    int64_t* ta = (int64_t*)malloc(8 * (nt + 1));
    int64_t* tD = (int64_t*)malloc(8 * (nt + 1));
    uint64_t* gdone = (uint64_t*)calloc(nt + 1, 8);
    uint32_t* cb = (uint32_t*)calloc(nt + 1, 4);
    uint32_t* ce = (uint32_t*)calloc(nt + 1, 4);
    uint64_t* tle = (uint64_t*)calloc(nt + 1, 8);
    uint64_t* ttot = (uint64_t*)calloc(nt + 1, 8);
    uint8_t* tever = (uint8_t*)calloc(nt + 1, 1);      /* A40: some call of the task was scheduled */
    uint8_t* tdrop = (uint8_t*)calloc(nt + 1, 1);
    int64_t lat_ring[1024]; uint32_t ring_n = 0, ring_pos = 0; int64_t ring_sum = 0;
    int ret = OG_OK;
    if (cfg->frame_steps > 1024) { ret = OG_EINVAL; goto done; }

    for (uint32_t r = 0; r < n; ++r) {
        id[r] = r;
        uint32_t fl = 0;
        if (tr->task[r] != NO_TASK) fl |= FL_COMPOUND;
        if (tr->override_R[r]) fl |= FL_OVERRIDE;
        if (tr->input_len[r] == 0 || tr->true_out[r] == 0 || tr->group[r] >= n_groups) { ret = OG_EINVAL; goto done; }
        if (tr->override_R[r] && groups_in[tr->group[r]].type != OG_DDL) { ret = OG_EINVAL; goto done; }
        if ((tr->task[r] != NO_TASK) != (groups_in[tr->group[r]].type == OG_CMP)) { ret = OG_EINVAL; goto done; }
        uint32_t st = (fl & FL_COMPOUND) ? ST_WAITING : ST_QUEUED;
        meta[r] = tr->group[r] | (st << 8) | (fl << 12);
        aux[r] = tr->dist_row[r] & 0xFFFFu;
        arr[r] = (fl & FL_COMPOUND) ? INT64_MAX
                                    : (int64_t)((u128)(uint64_t)tr->arrival_ns[r] * rc->load_den / rc->load_num);
    }
    for (uint32_t t = 0; t < nt; ++t) {
        ta[t] = (int64_t)((u128)(uint64_t)tr->task_arrival_ns[t] * rc->load_den / rc->load_num);
        tD[t] = (int64_t)((u128)(uint64_t)tr->task_deadline_ns[t] * rc->slo_num / rc->slo_den);
        uint32_t S = tr->task_n_stages[t];
        if (S == 0 || S > MAX_STAGES) { ret = OG_EINVAL; goto done; }
        uint64_t tot = 0;
        for (uint32_t u = 0; u < S; ++u) tot += (uint64_t)tr->stage_pattern_ms[t * MAX_STAGES + u] * 1000000ull;
        ttot[t] = tot;
        timer[t] = ta[t];      /* stage 0 "starts" when the task arrives */
        cur[t] = 0;
        cb[t] = ce[t] = 0;
    }

    int64_t now = 0;
    uint32_t steps = 0;
    for (;;) {
        /* stage starts whose time has come: timer[t] is the start time of stage cur[t]
         * (task arrival for stage 0, the end of the previous stage otherwise) */
        for (uint32_t t = 0; t < nt; ++t) {
            while (!tdone[t] && timer[t] <= now) {
                int64_t at = timer[t];
                uint32_t s = cur[t], S = tr->task_n_stages[t];
                if (s == S) {                                   /* last stage ended at `at` */
                    tdone[t] = 1; out->n_tasks_done++; timer[t] = INT64_MAX;
                    if (at <= ta[t] + tD[t]) {                  /* §3 P:213 compound goodput */
                        uint64_t tot = 0;
                        for (uint32_t u = 0; u < S; ++u) {
                            uint32_t kk = t * MAX_STAGES + u;
                            if (tr->stage_kind[kk] == 0)
                                for (uint32_t q = tr->stage_call_begin[kk]; q < tr->stage_call_end[kk]; ++q)
                                    tot += (uint64_t)G[tr->group[q]].w_in * tr->input_len[q] +
                                           (uint64_t)G[tr->group[q]].w_out * tr->true_out[q];
                        }
                        out->token_goodput += tot; out->request_goodput++;
                    }
                    break;
                }
                uint32_t k = t * MAX_STAGES + s;
                if (tr->stage_kind[k] == 1) {                   /* tool node: fixed exec time */
                    cur[t] = s + 1; timer[t] = at + tr->stage_exec_ns[k];
                    continue;
                }
                /* LLM stage: release its calls with arrival = stage start */
                cb[t] = tr->stage_call_begin[k]; ce[t] = tr->stage_call_end[k];
                left[t] = ce[t] - cb[t];
                if (left[t] == 0) { ret = OG_EINVAL; goto done; }
                for (uint32_t r = cb[t]; r < ce[t]; ++r) { arr[r] = at; meta[r] = m_set_state(meta[r], ST_QUEUED); }
                uint64_t le = 0;
                for (uint32_t u = 0; u <= s; ++u) le += (uint64_t)tr->stage_pattern_ms[t * MAX_STAGES + u] * 1000000ull;
                tle[t] = le;
                timer[t] = INT64_MAX;
            }
        }
        if (steps >= rc->n_steps) break;

        int64_t v = ring_n ? ring_sum / (int64_t)ring_n : rc->v_token0_ns;
        task_view tv = { nt, cb, ce, ta, tD, tle, ttot, NULL, gdone, tever, tdrop };
        og_result res;
        int st = gmax_step(&cf, G, n_groups, T, now, v, n, id, arr, tr->input_len, gen, pre, meta, aux,
                           tr->task, tr->override_R, tr->fair, &tv, &res, sel, selc, NULL,
                           cfg->frame_steps && steps % cfg->frame_steps == 0);
        out->n_dropped += res.n_dropped_now;
        if (st == OG_EINVAL) { ret = OG_EINVAL; goto done; }
        /* A40: a dropped task ends without goodput; the calls of its later stages are dropped too */
        for (uint32_t t = 0; t < nt; ++t) {
            if (!tdrop[t]) continue;
            tdone[t] = 1; timer[t] = INT64_MAX; cb[t] = ce[t] = 0; out->n_tasks_dropped++;
            for (uint32_t u = 0; u < tr->task_n_stages[t]; ++u) {
                uint32_t kk = t * MAX_STAGES + u;
                if (tr->stage_kind[kk] != 0) continue;
                for (uint32_t q = tr->stage_call_begin[kk]; q < tr->stage_call_end[kk]; ++q)
                    if (m_state(meta[q]) == ST_WAITING) { meta[q] = m_set_state(meta[q], ST_DROPPED); out->n_dropped++; }
            }
        }
        if (st == OG_OK)
            for (uint32_t i = 0; i < res.n_selected; ++i)
                if (tr->task[sel[i]] != NO_TASK) tever[tr->task[sel[i]]] = 1;
        if (st == OG_EMPTY) {
            /* idle: jump to the next arrival or timer; stop when nothing is left (drained) */
            int64_t nxt = INT64_MAX;
            for (uint32_t r = 0; r < n; ++r)
                if (!(m_flags(meta[r]) & FL_COMPOUND) && m_state(meta[r]) == ST_QUEUED && arr[r] > now && arr[r] < nxt) nxt = arr[r];
            for (uint32_t t = 0; t < nt; ++t)
                if (!tdone[t] && timer[t] != INT64_MAX && timer[t] > now && timer[t] < nxt) nxt = timer[t];
            if (nxt == INT64_MAX) break;
            now = nxt;
            continue;
        }
        /* iteration latency: c0 + c_att * max context + c_lin * |batch| */
        int64_t maxctx = 0;
        for (uint32_t i = 0; i < res.n_selected; ++i) {
            uint32_t r = sel[i];
            int64_t ctx = pre[r] < tr->input_len[r] ? (int64_t)pre[r] + selc[i]
                                                     : (int64_t)tr->input_len[r] + gen[r];
            if (ctx > maxctx) maxctx = ctx;
        }
        int64_t latency = rc->c0_ns + rc->c_att_ns * maxctx + rc->c_lin_ns * (int64_t)res.n_selected;
        /* NEXT-1 (A46): the KV swap-out of the requests the gate evicted stalls this iteration */
        latency += res.stall_ns;
        out->n_preempted += res.n_preempted;
        now += latency;
        ++steps;
        out->tokens_processed += res.total_tokens;
        if (log) {
            for (uint32_t i = 0; i < res.n_selected; ++i) selid[i] = sel[i];
            og_step_log* L = &log[steps - 1];
            L->now_ns = now; L->n_selected = res.n_selected; L->total_tokens = res.total_tokens;
            L->n_candidates = res.n_candidates; L->b_star = res.b_star; L->bp = res.bp;
            L->ids_hash = fnv1a_ids(selid, res.n_selected);
            L->v_token_ns = v;
            L->n_preempted = res.n_preempted; L->p_num = cf.p_num; L->stall_ns = res.stall_ns;
            if (log_ids) memcpy(log_ids + (size_t)(steps - 1) * cfg->max_batch, selid, 4 * res.n_selected);
        }
        /* progress of the executed batch (iteration end = token timestamp) */
        for (uint32_t i = 0; i < res.n_selected; ++i) {
            uint32_t r = sel[i];
            const og_group* gr = &G[tr->group[r]];
            int emit = 0;
            if (pre[r] < tr->input_len[r]) {
                pre[r] += selc[i];
                if (pre[r] == tr->input_len[r]) emit = 1;   /* A28: prefill end emits token 0 */
            } else emit = 1;
            if (!emit) continue;
            uint32_t tok = gen[r];
            if (gr->type == OG_LAT) {                       /* §3, token i on the timeline */
                if (now <= arr[r] + gr->ttft_ns + (int64_t)tok * gr->tbt_ns) out->token_goodput += gr->w_out;
                else late[r] = 1;
            }
            gen[r] = tok + 1;
            if (gen[r] < tr->true_out[r]) continue;
            /* completion */
            meta[r] = m_set_state(meta[r], ST_DONE);
            out->n_done++;
            if (gr->type == OG_DDL) {                       /* §3 P:212 all-or-nothing */
                if (now <= arr[r] + gr->e2el_ns) {
                    out->token_goodput += (m_flags(meta[r]) & FL_OVERRIDE) ? tr->override_R[r]
                        : (uint64_t)gr->w_in * tr->input_len[r] + (uint64_t)gr->w_out * tr->true_out[r];
                    out->request_goodput++;
                }
            } else if (gr->type == OG_LAT) {
                if (!late[r]) out->request_goodput++;
            } else if (gr->type == OG_CMP) {                /* §3 P:213 + stage barrier S:422-430 */
                uint32_t t = tr->task[r];
                gdone[t] += (uint64_t)gr->w_in * tr->input_len[r] + (uint64_t)gr->w_out * tr->true_out[r];
                if (--left[t] == 0) {                       /* stage barrier: next stage starts now */
                    cur[t] += 1; cb[t] = ce[t] = 0; timer[t] = now;
                }
            }
        }
        /* v_token: floor of the trailing mean of the last Delta latencies */
        if (ring_n < cfg->frame_steps) { lat_ring[ring_n++] = latency; ring_sum += latency; }
        else { ring_sum += latency - lat_ring[ring_pos]; lat_ring[ring_pos] = latency; ring_pos = (ring_pos + 1) % cfg->frame_steps; }
        /* NEXT-2 online p (A48): the window's goodput scores its arm; the next arm is chosen */
        if (rc->p_adapt && steps % ((uint64_t)rc->window_frames * cfg->frame_steps) == 0) {
            gsum[arm] += out->token_goodput - g_start; gcnt[arm] += 1;
            g_start = out->token_goodput;
            window += 1;
            arm = next_arm(rc, gsum, gcnt, window);
            cf.p_num = P_GRID[arm];
        }
    }
    out->steps = steps; out->sim_end_ns = now;
done:
    out->error = ret != OG_OK;
    free(id); free(arr); free(gen); free(pre); free(meta); free(aux); free(late); free(sel); free(selc); free(selid);
    free(cur); free(left); free(tdone); free(timer); free(ta); free(tD); free(gdone); free(cb); free(ce); free(tle); free(ttot);
    free(tever); free(tdrop);
    return ret;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-3: pattern-graph matching (§4.1; SPEC patterns S:160-263; reading A49). */
/* A pattern graph is stage-structured (<= 8 stages, the pattern store of Fig. 6): stage u */
/* has an identity (kind << 31 | model / tool id), an input-length attribute in_len (the   */
/* edges into its LLM calls), a node attribute out (LLM output length, or the tool's       */
/* execution time in ms) and its execution time t_u (ms).  A query is a task at stage s:   */
/* identities of stages 0..s are revealed, stages 0..s-1 are complete.                     */
/*  - prefix pruning ("prunes past patterns whose prefix structures diverge"): a     */
/*    pattern survives iff it has > s stages and the identities of stages 0..s match;     */
/*  - similarity: Gaussian kernels k(a,b) = exp(-(a-b)^2 / (2 sigma^2)),       */
/*    sigma = max(0.25 max(a,b), 1), over the node attributes of stages 0..s-1 and  */
/*    the input lengths of the LLM stages 1..s; the score is their arithmetic mean in      */
/*    stage order, nodes first then edges per stage; no term -> score 1;           */
/*  - the best pattern: the highest score, then the higher reuse count, then the lower    */
/*    index; -1 when every pattern is pruned (NoMatch).                            */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    uint32_t n, _pad;
    const uint32_t* n_stages;     /* [n] */
    const uint32_t* ident;        /* [n*8] kind << 31 | id */
    const uint32_t* in_len;       /* [n*8] */
    const uint32_t* out;          /* [n*8] */
    const uint32_t* t_ms;         /* [n*8] */
    const uint32_t* reuse;        /* [n] */
} og_patterns;

typedef struct {
    uint32_t n, _pad;
    const uint32_t* stage;        /* [n] revealed stage s */
    const uint32_t* ident;        /* [n*8] */
    const uint32_t* in_len;       /* [n*8] */
    const uint32_t* out;          /* [n*8] */
} og_queries;

double og_kernel_sim(uint32_t a, uint32_t b) {
    double mx = (double)(a > b ? a : b);
    double sigma = 0.25 * mx;
    if (sigma < 1.0) sigma = 1.0;
    double d = (double)a - (double)b;
    return exp(-(d * d) / (2.0 * sigma * sigma));
}

/* the score of pattern p for query q, or -1 when pruned */
double og_match_score(const og_patterns* P, uint32_t p, const og_queries* Q, uint32_t q) {
    uint32_t s = Q->stage[q];
    if (s >= MAX_STAGES || P->n_stages[p] <= s) return -1.0;
    for (uint32_t u = 0; u <= s; ++u)
        if (P->ident[p * MAX_STAGES + u] != Q->ident[q * MAX_STAGES + u]) return -1.0;
    double sum = 0.0; uint32_t cnt = 0;
    for (uint32_t u = 0; u <= s; ++u) {
        uint32_t id = Q->ident[q * MAX_STAGES + u];
        if (u < s) { sum += og_kernel_sim(Q->out[q * MAX_STAGES + u], P->out[p * MAX_STAGES + u]); ++cnt; }
        if (u >= 1 && !(id >> 31)) { sum += og_kernel_sim(Q->in_len[q * MAX_STAGES + u], P->in_len[p * MAX_STAGES + u]); ++cnt; }
    }
    return cnt ? sum / (double)cnt : 1.0;
}

int og_match(const og_patterns* P, const og_queries* Q, int32_t* best, double* score) {
    for (uint32_t q = 0; q < Q->n; ++q) {
        int32_t b = -1; double bs = -1.0;
        for (uint32_t p = 0; p < P->n; ++p) {
            double sc = og_match_score(P, p, Q, q);
            if (sc < 0.0) continue;
            if (b < 0 || sc > bs || (sc == bs && P->reuse[p] > P->reuse[b])) { b = (int32_t)p; bs = sc; }
        }
        best[q] = b; score[q] = bs;
    }
    return OG_OK;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-2 power-of-K over M model replicas (§4.3, reading A51).                 */
/* Every request has dummies on K sampled replicas (replica m's pool holds its dummies,    */
/* standalone requests only); a dummy on replica m is keyed with m's v_token, so it carries */
/* a replica-specific priority.  Each replica runs GMAX over its own pool ("scheduling     */
/* proceeds as usual over the enlarged set").  A request proposed by several replicas in   */
/* the same step is assigned to the one where its priority is highest: key_m = A /         */
/* (len_rem v_m + eps) with A and len_rem replica-independent, so the smallest v_m, ties to */
/* the lower index; it leaves the other replicas' batches (no refill).  "Once a request is */
/* assigned to a replica, its other dummies are removed": every other replica's dummy of   */
/* an assigned request becomes Moved (terminal, never pending).                             */
/* ------------------------------------------------------------------------------------ */
int og_multi_step(const og_config* cfg, const og_group* G, uint32_t n_groups, const og_table* T, int64_t now,
                  uint32_t M, const int64_t* v, og_pool* const* pools, og_result* res,
                  uint32_t* const* batch_rows, uint32_t* const* batch_tokens) {
    uint32_t** sel = (uint32_t**)calloc(M, sizeof(uint32_t*));
    uint32_t** scst = (uint32_t**)calloc(M, sizeof(uint32_t*));
    int* st = (int*)calloc(M, sizeof(int));
    uint32_t* nprop = NULL;            /* each replica's proposal size (before the assignment) */
    int ret = OG_OK;
    /* 1. every replica's GMAX step on its own dummies */
    for (uint32_t m = 0; m < M; ++m) {
        og_pool* P = pools[m];
        for (uint32_t r = 0; r < P->n; ++r)
            if (P->task[r] != NO_TASK) { ret = OG_EINVAL; goto done; }     /* standalone requests only */
        sel[m] = (uint32_t*)malloc(sizeof(uint32_t) * (P->n ? P->n : 1));
        scst[m] = (uint32_t*)malloc(sizeof(uint32_t) * (P->n ? P->n : 1));
        og_reset_memo();
        st[m] = gmax_step(cfg, G, n_groups, T, now, v[m], P->n, P->id, P->arrival_ns, P->input_len,
                          P->generated, P->prefilled, P->meta, P->aux, P->task, P->override_R, P->fair,
                          NULL, &res[m], sel[m], scst[m], NULL, 1);
        if (st[m] == OG_EINVAL) { ret = OG_EINVAL; goto done; }
    }
    /* 2. the winner of every proposed request: the smallest v, then the lower replica index */
    nprop = (uint32_t*)calloc(M, sizeof(uint32_t));
    for (uint32_t m = 0; m < M; ++m) nprop[m] = st[m] == OG_OK ? res[m].n_selected : 0u;
    for (uint32_t m = 0; m < M; ++m) {
        if (st[m] != OG_OK) continue;
        uint32_t k = 0, tot = 0;
        for (uint32_t i = 0; i < nprop[m]; ++i) {
            uint32_t id = pools[m]->id[sel[m][i]];
            uint32_t win = m;
            for (uint32_t w = 0; w < M; ++w) {
                if (w == m || st[w] != OG_OK) continue;
                for (uint32_t j = 0; j < nprop[w]; ++j)
                    if (pools[w]->id[sel[w][j]] == id && (v[w] < v[win] || (v[w] == v[win] && w < win))) win = w;
            }
            if (win != m) continue;
            batch_rows[m][k] = sel[m][i]; batch_tokens[m][k] = scst[m][i]; tot += scst[m][i]; ++k;
        }
        res[m].n_selected = k; res[m].total_tokens = tot;
    }
    /* 3. sibling removal: a request proposed anywhere is assigned to its winner; every dummy of it
     * on another replica (proposed there or not) becomes Moved */
    for (uint32_t w = 0; w < M; ++w) {
        if (st[w] != OG_OK) continue;
        for (uint32_t j = 0; j < res[w].n_selected; ++j) {
            uint32_t id = pools[w]->id[batch_rows[w][j]];
            for (uint32_t m = 0; m < M; ++m) {
                if (m == w) continue;
                for (uint32_t r = 0; r < pools[m]->n; ++r)
                    if (pools[m]->id[r] == id) pools[m]->meta[r] = m_set_state(pools[m]->meta[r], ST_MOVED);
            }
        }
    }
done:
    for (uint32_t m = 0; m < M; ++m) { free(sel[m]); free(scst[m]); res[m].error = st[m] == OG_EINVAL; }
    free(sel); free(scst); free(st); free(nprop);
    return ret;
}
