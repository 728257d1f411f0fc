/*
 * jit_sched.h -- C ABI of libjitsched.so: the JITServe GMAX scheduling step (arXiv 2504.20068)
 * as hand-written CUDA for sm_100a (B200).
 *
 * The library runs, over every pending request of a pool resident in HBM, the per-iteration
 * step of Alg. 1:
 *   (a1) admission control: drop requests unscheduled after waiting_time
 *   (a2) conservative remaining length: an upper quantile of the length distribution
 *        conditioned on the tokens generated so far, refreshed every R tokens
 *   (a3) just-in-time rate / remaining time per SLO type
 *   (a4) compound requests: len_rem and goodput aggregated over the calls of the current
 *        stage against the stage sub-deadline D_s = phi(s) D
 *   (a5) margin-goodput key = goodput / t_gen (App. B I(k) P:911-915) with
 *        starvation inflation
 *   (a6) per-step token cost (chunked prefill)
 *   (a7)-(a9) BatchPriority bp, cutoff filter p*bp and length-sorted sliding window
 *        (Alg. 1; §4.2) under a per-step token budget
 * and a trace replay (a10) that runs the step inside an iteration cost model and counts
 * token / request goodput (§3).  Readings of the paper are numbered A1..A39 in
 * DESIGN.md §3; the exact arithmetic contract is DESIGN.md §4.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Every pointer is a HOST pointer unless the field says otherwise.
 *  - The caller owns every buffer it passes.  Inputs are consumed during the call; nothing
 *    is retained.  The library owns only its handle; all device memory it uses is carved
 *    from the caller-provided workspace (allocated by PyTorch's caching allocator).
 *  - Calls are synchronous with respect to their outputs on return, and enqueue their
 *    device work on cfg.stream (a cudaStream_t; NULL = legacy default stream).
 *  - Return value: JIT_OK (0), JIT_EMPTY (1, no pending request; an empty batch), or a
 *    negative error.  jit_sched_last_error() returns a message owned by the handle.
 *  - No C++ exception crosses the ABI.  A handle is not thread-safe; handles are independent.
 */
#ifndef JIT_SCHED_H
#define JIT_SCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    JIT_OK = 0,
    JIT_EMPTY = 1,        /* no pending request (SPEC EmptyQueue); n_selected = 0 */
    JIT_RETRY = 2,        /* jit_shard_spec_resolve only: resolve this step with the exact protocol */
    JIT_EINVAL = -1,      /* bad config / table / pool (S:55-63 InvalidLength, ConfigError) */
    JIT_ETRACE = -2,      /* bad replay trace (S:417 InvalidTrace) */
    JIT_ECAPACITY = -3,   /* more rows / tasks / candidates than the workspace was sized for */
    JIT_ECUDA = -4,       /* a CUDA runtime error (message in last_error) */
    JIT_ESTATE = -6       /* call order violated (e.g. step before load) */
};

/* SLO types, §3; best effort P:216 */
enum { JIT_LAT = 0, JIT_DDL = 1, JIT_CMP = 2, JIT_BE = 3 };
/* request states + WAITING = compound call whose stage is not released yet */
enum { JIT_QUEUED = 0, JIT_RUNNING = 1, JIT_PREEMPTED = 2, JIT_DONE = 3, JIT_DROPPED = 4, JIT_WAITING = 5,
       JIT_MOVED = 6      /* power-of-K: the request was assigned to another replica (terminal) */ };
/* request flags */
enum { JIT_F_EVER = 1, JIT_F_COMPOUND = 2, JIT_F_OVERRIDE = 4 };
#define JIT_NO_TASK 0xFFFFFFFFu
#define JIT_MAX_STAGES 8
/* jit_config.flags */
#define JIT_CFG_DEBUG_ROWS 1u   /* keep per-row rate / t_rem / Lhat / cost for jit_sched_read_rows */
#define JIT_CFG_NO_GRAPH 2u     /* launch the step's kernels (k_score, k_spec) directly instead of
                                   as one CUDA graph (for tools that do not follow graphs) */

/* One SLO group (a row of the SLO table; reading A35).  Times are int64 ns.
 * LAT uses ttft/tbt, DDL e2el, CMP e2el per stage (D = e2el * stages), BE be_deadline.
 * Base goodput R(k) = w_in * L_i + w_out * L_o (App. B). */
typedef struct jit_slo_group {
    uint32_t type, w_in, w_out, reserved;
    int64_t ttft_ns, tbt_ns, e2el_ns, be_deadline_ns;
} jit_slo_group;

/* Length-distribution table (stand-in for the QRF of P:269; reading A8).
 * edges[n_bins]: strictly increasing, edges[0] >= 1, edges[n_bins-1] = l_max (< 65536).
 * cum[n_rows * n_bins]: row-major, nondecreasing per row: cum[r][k] = #samples with L <= edges[k]. */
typedef struct jit_len_table {
    uint32_t n_rows, n_bins, l_max, reserved;
    const uint32_t* edges;
    const uint32_t* cum;
} jit_len_table;

/* Scheduler configuration (defaults in DESIGN.md §2 / SURVEY Appendix A). */
typedef struct jit_config {
    uint32_t token_budget;     /* tau: per-step token budget (A14) */
    uint32_t max_batch;        /* B_max */
    uint32_t prefill_chunk;    /* chunked-prefill size (A25), 1 <= chunk <= tau */
    uint32_t refine_interval;  /* R: refresh the length bound every R tokens */
    uint32_t frame_steps;      /* Delta: steps per starvation frame */
    uint32_t q_num, q_den;     /* length quantile q = q_num/q_den in (0,1] (A3) */
    uint32_t p_num, p_den;     /* cutoff p in (0,1] */
    uint32_t delta_starve;     /* goodput added per frame waited (A12) */
    uint32_t len_key;          /* 0: group by input length; 1: by input+generated (A17) */
    uint32_t appb_filter;      /* 1: App. B filter t_gen <= t_rem, else goodput 0 (A22) */
    int64_t eps_ns;            /* epsilon of App. B I(k) (A2) */
    int64_t waiting_ns;        /* admission waiting_time, strict '>' (A29) */
    uint32_t capacity;         /* max pool rows the workspace holds */
    uint32_t task_capacity;    /* max compound tasks */
    uint32_t flags;            /* JIT_CFG_* */
    int32_t device;            /* CUDA device ordinal */
    void* stream;              /* cudaStream_t for all device work */
    /* NEXT-1 preemption gate (reading A46; §4.2, App. D.2): 0 = off, the
     * batch is GMAX's window every step (A30).  On: Running means "in the executing batch"; a
     * running request keeps its slot unless, at a frame boundary (every frame_steps steps),
     * a proposed request beats it by R(in)/R(out) > 1 + pmtn_num/pmtn_den and its gain over a
     * frame exceeds the KV swap loss (KV = prefilled + generated tokens at io_bw_tps tokens/s).
     * Implemented in the trace replay (jit_sched_replay). */
    uint32_t preempt, pmtn_num, pmtn_den, reserved2;
    uint64_t io_bw_tps;
    /* NEXT-2 fairness blend (§4.3, reading A47): priority' = (1-f) priority + f Fair(r)
     * with f = fair_num / fair_den (0 = off), Fair(r) the pool's per-request `fair` score, as
     * fl(fl(fl(key * (den - num)) + num * Fair) / den).  Step and replay. */
    uint32_t fair_num, fair_den;
} jit_config;

/* A pool snapshot (SoA, n rows).  Layout rule: standalone rows first, then compound calls
 * grouped by task: rows of task t are [call_off[t], call_off[t+1]), call_off[0] = n_single,
 * call_off[n_tasks] = n.  meta = group (bits 0-7) | state << 8 | flags << 12 (bits 16-31
 * must be 0); aux = dist_row (bits 0-15) | steps_waited << 16.  If on_device != 0 every
 * array pointer is a device pointer (read during the call only). */
typedef struct jit_pool {
    uint32_t n, n_single, n_tasks;
    int32_t on_device;
    const uint32_t* id;            /* request id, the tie-break of every order (A18) */
    const int64_t* arrival_ns;
    const uint32_t* input_len;     /* L_i >= 1 */
    const uint32_t* generated;     /* g */
    const uint32_t* prefilled;     /* prompt tokens already prefilled */
    const uint32_t* meta;
    const uint32_t* aux;
    const uint32_t* task;          /* owning task or JIT_NO_TASK */
    const uint32_t* override_R;    /* R(k) set directly (App. D constructions) when JIT_F_OVERRIDE */
    /* compound tasks (may be NULL when n_tasks == 0) */
    const uint32_t* call_off;      /* n_tasks + 1 */
    const int64_t* task_arrival_ns;   /* a_c */
    const int64_t* task_deadline_ns;  /* D relative to a_c */
    const uint32_t* cur_stage;        /* s */
    const uint32_t* n_stages;         /* S <= JIT_MAX_STAGES */
    const uint32_t* pattern_ms;       /* n_tasks * 8: matched-pattern stage times (phi) */
    const uint64_t* goodput_done;     /* goodput of the task's finished calls */
    const uint32_t* fair;             /* NULL (= 0) or Fair(r) per row, key units (NEXT-2, A47) */
} jit_pool;

/* Per-step input: the step's clock and v_token, and what changed since the previous step, applied
 * in this order before the step's pass (the API of P:544: requests arrive with their SLO
 * parameters; the engine reports generation progress; compound tasks advance stage by stage):
 *  - arrivals (optional): new requests appended to the resident pool, in the jit_pool layout of
 *    jit_sched_load -- standalone rows first, then whole new compound tasks whose call_off is
 *    relative to the arrivals' own rows (call_off[0] = n_single, call_off[n_tasks] = n) and whose
 *    task fields index the arrivals' own tasks (0 .. n_tasks-1).  The library appends them after the
 *    current rows / tasks (a new task gets the index previous n_tasks + its own).  Ids must be new.
 *    Capacity is fixed at init: JIT_ECAPACITY when rows or tasks would exceed it (reload to compact).
 *  - task updates (optional): per updated task (index into the resident tasks) its new current
 *    stage, the goodput of its finished calls, and optionally an absolute stage sub-deadline
 *    a_c + D_s (tu_stage_deadline_ns[i] < 0 or NULL: derived from the pattern).  The
 *    calls of a newly released stage become schedulable through progress (state Queued).
 *  - progress (optional): per request its tokens generated, prompt tokens prefilled and state;
 *    keyed by request id (progress_by_id = 1) or by pool row (0).  Done and Dropped are final;
 *    generated < 2^24 and prefilled <= L_i.  A violation fails the step (JIT_EINVAL).
 * Every array is a host array of the stated count. */
typedef struct jit_step_in {
    int64_t now_ns;
    int64_t v_token_ns;            /* average per-token generation time v_token, < 2^36 ns */
    uint32_t n_progress, progress_by_id;
    const uint32_t* prog_key;      /* request ids (progress_by_id = 1) or pool rows */
    const uint32_t* prog_generated;
    const uint32_t* prog_prefilled;
    const uint32_t* prog_state;
    const struct jit_pool* arrivals;   /* NULL: none */
    uint32_t n_task_updates, reserved;
    const uint32_t* tu_task;
    const uint32_t* tu_cur_stage;
    const uint64_t* tu_goodput_done;
    const int64_t* tu_stage_deadline_ns;  /* NULL, or per update: absolute a_c + D_s (< 0: from the pattern) */
} jit_step_in;

/* Selected batch (BestGroup, Alg. 1), in window order (len asc, id asc; A20).
 * ids / tokens / rows are host arrays of `capacity` entries (any may be NULL). */
typedef struct jit_batch {
    uint32_t capacity;
    uint32_t n_selected, total_tokens, n_candidates, b_star, n_pending, n_dropped, status;
    uint32_t n_refresh;            /* length bounds recomputed this step (the rest hit the cache) */
    uint32_t fallback;             /* 1: the exact radix path ran instead of the speculative set */
    uint32_t n_spec;               /* size of the speculative set {key >= t_guess} */
    double bp, thr;                /* batch priority and cutoff threshold fl(p * bp) */
    uint32_t* ids;
    uint32_t* tokens;
    uint32_t* rows;
} jit_batch;

typedef struct jit_sched jit_sched;

/* Device workspace the handle needs for cfg (capacity / task_capacity / table size). */
int jit_sched_workspace_bytes(const jit_config* cfg, const jit_len_table* table, uint64_t* bytes);

/* Create a handle.  groups: n_groups <= 256 SLO groups; table: copied to the workspace.
 * dev_workspace: device memory of ws_bytes >= jit_sched_workspace_bytes(), 256-B aligned. */
int jit_sched_init(const jit_config* cfg, const jit_slo_group* groups, uint32_t n_groups,
                   const jit_len_table* table, void* dev_workspace, uint64_t ws_bytes, jit_sched** out);

/* Replace the resident pool (H2D or D2D copy + pack).  Invalidates the cached length bounds. */
int jit_sched_load(jit_sched* h, const jit_pool* pool);

/* One GMAX step over the resident pool; writes the batch.  Mutates the pool's admission
 * state, steps_waited (+1 saturating for pending requests left out) and ever_scheduled. */
int jit_sched_step(jit_sched* h, const jit_step_in* in, jit_batch* out);

/* Enqueue one step without waiting for it (results stay on the device; read them with
 * jit_sched_fetch_batch).  Steps may be chained (several step_async before one fetch): each
 * step that resolves on the device (the steady state) leaves its bookkeeping done; if a step
 * needs the host (exact path, large speculative set), every later step of the chain does
 * nothing (counted in jit_sched_counters' `skipped`) until fetch_batch runs the host's part and
 * returns that step's batch.  jit_sched_step / load after an unfinished async step fail with
 * JIT_ESTATE (fetch first).  Progress updates are not allowed here. */
int jit_sched_step_async(jit_sched* h, int64_t now_ns, int64_t v_token_ns);
int jit_sched_fetch_batch(jit_sched* h, jit_batch* out);

/* Copy per-row state / outputs of the last step to host arrays of n entries (NULL = skip).
 * key: -1 for rows not pending.  rate / t_rem / lhat / cost need JIT_CFG_DEBUG_ROWS. */
int jit_sched_read_rows(jit_sched* h, double* key, double* rate, int64_t* t_rem, uint32_t* lhat,
                        uint32_t* cost, uint32_t* pending, uint32_t* meta, uint32_t* aux);

/* Per-kernel device time, from CUDA events recorded (as graph event nodes) on cfg.stream
 * around each kernel of the step.  enable > 0 keeps one event set per step for up to
 * `enable` steps; 0 turns timing off; < 0 leaves it unchanged.  ms_out (n_out <= 5) gets the
 * average in ms over the recorded steps of [k_score, 0, k_spec, 0, whole step] (the exact
 * path, when the host runs it after a step, is not included). */
int jit_sched_kernel_times(jit_sched* h, int enable, float* ms_out, uint32_t n_out);

/* Measurement: `launches` back-to-back launches of the scoring kernel (k_score, rows (a1)-(a6)),
 * rotating over n_handles loaded handles that share one stream, timed with CUDA events around the
 * sequence; *ms_per_launch = average.  The pass writes no per-row state in the steady state and the
 * step counter moves only with a resolved step, so the pools are left as they were (the per-step
 * accumulators and speculative sets are reset afterwards).  flags & JIT_TIME_FORCE_REFRESH: every
 * cached length bound is invalidated before each launch (untimed; each launch timed alone), i.e.
 * the pass with a stale bound on every row (SURVEY 8(d) "forced refresh"); flags & JIT_TIME_REFRESH_2PCT: the
 * same with every 50th row stale (the steady state's ~2% refresh). */
#define JIT_TIME_FORCE_REFRESH 1u
#define JIT_TIME_REFRESH_2PCT 2u   /* every 50th row's bound invalidated before each launch (SURVEY 8(d) "about 2%") */
#define JIT_TIME_READ_FLOOR 4u     /* instead of k_score: the hot rows read with its load pattern and nothing else */
int jit_sched_time_scoring(jit_sched** hs, uint32_t n_handles, int64_t now_ns, int64_t v_token_ns, uint32_t launches,
                           uint32_t flags, float* ms_per_launch);

/* Device counters of the handle (synchronizes its stream): steps resolved since init (the
 * steps_waited stamps count against this counter), steps resolved by the exact radix path, and
 * chained jit_sched_step_async steps that did nothing because an earlier step of the chain still
 * needed the host (each of those must be re-run; a timed region must see 0). */
int jit_sched_counters(jit_sched* h, uint32_t* steps, uint32_t* fallbacks, uint32_t* skipped);

/* Tests: set the device step counter that the steps_waited stamps count against (every stamped
 * row's stamp moves with it, so no count changes) and the host's count of launched steps (the
 * stamp rebase of pool.cuh runs each time it reaches a multiple of 2^30), so that the counter's
 * wrap at 2^32 and the rebase are reached in a few steps.  JIT_ESTATE with an unfinished async
 * step. */
int jit_sched_debug_set_counter(jit_sched* h, uint32_t steps, uint64_t launched);

/* Diagnostics: copy the first n u64 of the exact path's sort scratch to host memory `out`
 * (JIT_TIMELINE builds of the scoring kernel leave per-warp %globaltimer stamps there). */
int jit_sched_debug_scratch(jit_sched* h, uint64_t* out, uint32_t n);

/* Diagnostics: %globaltimer stamps (ns) of the phases of the single-CTA resolve of the last
 * synchronized step: [k_spec start, partials reduced, set loaded, set sorted, budget walk,
 * Cd gathered, window sort start, window sorted, prefix sums, argmax, batch written]. */
int jit_sched_phase_times(jit_sched* h, uint64_t* ns_out, uint32_t n_out);

/* ---------------------------------------------------------------------------------------
 * Trace replay (a10): one persistent CTA per replay runs the step, the iteration cost model
 * c0 + c_att * max context + c_lin * |batch|, token timestamps at the
 * iteration end, LAT/DDL/CMP goodput (§3), stage barriers and
 * v_token = floor(mean of the last Delta latencies).  Replays are independent.
 * ------------------------------------------------------------------------------------- */
typedef struct jit_trace {
    uint32_t n_rows, n_tasks;
    const int64_t* arrival_ns;     /* standalone rows (compound calls arrive at stage release) */
    const uint32_t* input_len;
    const uint32_t* true_out;      /* L_o >= 1, hidden from the scheduler */
    const uint32_t* group;
    const uint32_t* dist_row;
    const uint32_t* override_R;    /* 0 = none; only on DDL rows */
    const uint32_t* task;          /* JIT_NO_TASK or owning task (CMP group) */
    const int64_t* task_arrival_ns;
    const int64_t* task_deadline_ns;
    const uint32_t* task_n_stages;
    const uint32_t* stage_kind;        /* n_tasks * 8: 0 LLM stage, 1 tool stage */
    const int64_t* stage_exec_ns;      /* tool execution time */
    const uint32_t* stage_pattern_ms;  /* matched-pattern stage time (phi) */
    const uint32_t* stage_call_begin;  /* rows of an LLM stage: [begin, end) */
    const uint32_t* stage_call_end;
    const uint32_t* fair;              /* NULL (= 0) or Fair(r) per row (NEXT-2 blend, A47) */
} jit_trace;

typedef struct jit_replay_spec {
    uint32_t trace;                /* index into the traces array */
    uint32_t reserved;
    uint64_t load_num, load_den;   /* arrival' = floor(arrival * load_den / load_num) */
    uint64_t slo_num, slo_den;     /* SLO time' = floor(t * slo_num / slo_den) */
} jit_replay_spec;

typedef struct jit_replay_cfg {
    uint32_t n_steps, n_replays, log_steps, reserved;   /* log_steps: rows of the step log */
    int64_t v_token0_ns, c0_ns, c_att_ns, c_lin_ns;
    const jit_replay_spec* specs;  /* n_replays */
    /* NEXT-2 online p (reading A48): 1 = epsilon-greedy over p in {0.80, 0.90, 0.95, 1.00},
     * one arm per window of window_frames * frame_steps steps, scored by the window's token
     * goodput; explore with probability eps_num / eps_den (splitmix64 of seed + window index) */
    uint32_t p_adapt, eps_num, eps_den, window_frames;
    uint64_t seed;
} jit_replay_cfg;

typedef struct jit_replay_result {
    uint64_t token_goodput, tokens_processed;
    int64_t sim_end_ns;
    uint32_t request_goodput, n_done, n_dropped, steps, n_tasks_done;
    uint32_t n_tasks_dropped;      /* compound tasks dropped by admission (never scheduled, A40) */
    uint32_t error;
    uint32_t n_preempted;          /* running requests the preemption gate evicted (A46) */
} jit_replay_result;

typedef struct jit_step_log {
    int64_t now_ns;
    uint32_t n_selected, total_tokens, n_candidates, b_star;
    double bp;
    uint64_t ids_hash;             /* FNV-1a 64 over the batch ids (u32 LE) in batch order */
    int64_t v_token_ns;            /* the v_token the step's keys used */
    uint32_t n_preempted;          /* requests the gate evicted this step (A46) */
    uint32_t p_num;                /* the cutoff p (in 1/100 when adapting, A48) this step used */
    int64_t stall_ns;              /* their KV swap stall, included in this step's latency */
} jit_step_log;

/* Device workspace for a replay call. */
int jit_replay_workspace_bytes(const jit_config* cfg, const jit_trace* traces, uint32_t n_traces,
                               const jit_replay_cfg* rc, uint64_t* bytes);

/* Run rc->n_replays replays on h's device / stream.  out: n_replays results.  log (optional):
 * n_replays * rc->log_steps entries (replay-major).  Uses h's groups, table and config
 * (token_budget, max_batch, ... ); the pool state of h is untouched. */
int jit_sched_replay(jit_sched* h, const jit_trace* traces, uint32_t n_traces, const jit_replay_cfg* rc,
                     void* dev_workspace, uint64_t ws_bytes, jit_replay_result* out, jit_step_log* log);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: pattern-graph matching (§4.1; reading A49).  A stored pattern graph is
 * stage-structured (<= JIT_MAX_STAGES stages): per stage an identity (kind << 31 | model or
 * tool id, kind 1 = tool), an input-length attribute (edges into its LLM calls), a node
 * attribute (LLM output length, or tool execution time in ms) and the stage time t_u in ms.
 * A query is a compound task revealed up to stage s: identities and input lengths of stages
 * 0..s, node attributes of stages 0..s-1.  Patterns whose identities differ on stages 0..s (or
 * with <= s stages) are pruned; the rest score the mean of Gaussian-kernel similarities
 * exp(-(a-b)^2 / (2 sigma^2)), sigma = max(0.25 max(a,b), 1), over those attributes;
 * the best is (score desc, reuse desc, index asc); -1 / -1.0 when everything is pruned.
 * All arrays are host arrays, row-major [n][8] for per-stage fields.
 * --------------------------------------------------------------------------------------- */
typedef struct jit_pattern_store {
    uint32_t n_patterns, reserved;
    const uint32_t* n_stages;      /* [n] 1..8 */
    const uint32_t* ident;         /* [n*8] */
    const uint32_t* in_len;        /* [n*8] */
    const uint32_t* out;           /* [n*8] */
    const uint32_t* t_ms;          /* [n*8] stage times (phi); sum > 0 */
    const uint32_t* reuse;         /* [n] reuse count (tie-break) */
} jit_pattern_store;

typedef struct jit_match_query {
    uint32_t n, reserved;
    const uint32_t* stage;         /* [n] revealed stage s */
    const uint32_t* ident;         /* [n*8] */
    const uint32_t* in_len;        /* [n*8] */
    const uint32_t* out;           /* [n*8] (stages < s) */
    const uint32_t* task;          /* [n] resident task index (apply), or NULL */
} jit_match_query;

/* Device workspace for one jit_sched_match call. */
int jit_match_workspace_bytes(uint32_t n_patterns, uint32_t n_queries, uint64_t* bytes);

/* Match every query against the store on h's device (one warp per query).  best / score: host
 * arrays of q->n.  apply = 1: each matched query's task in the resident pool takes the pattern's
 * stage count and stage times (phi(s) = t_<=s / t_total, D_s = phi(s) D) -- the query's
 * stage must be the task's current stage (JIT_EINVAL otherwise).  JIT_EINVAL on a malformed
 * pattern (0 or > 8 stages, zero total time). */
int jit_sched_match(jit_sched* h, const jit_pattern_store* store, const jit_match_query* q, void* dev_workspace,
                    uint64_t ws_bytes, int32_t* best, double* score, uint32_t apply);

/* Device time (CUDA events on h's stream) of the matching kernel of the last jit_sched_match. */
int jit_sched_last_match_ms(jit_sched* h, float* ms);

/* ---------------------------------------------------------------------------------------
 * NEXT-4: a quantile regression forest in (a2) (§4.1; reading A50).
 * All trees' nodes in one array; an inner node sends x to `left` iff x[feature] <= threshold,
 * else to `right`; a leaf (feature = 0xFFFFFFFF) holds samples[threshold .. threshold + left),
 * its training targets sorted ascending (1 <= sample <= l_max).  Features x = (L_i, dist_row,
 * anchor R*floor(g/R), SLO group).  The bound: the ceil(q m)-th smallest of the m pooled leaf
 * samples above the anchor (every tree's leaf contributes its samples once), L_max when m = 0,
 * then max(., g + 1) -- the table's conditional quantile with the forest's leaves as the sample.
 * --------------------------------------------------------------------------------------- */
typedef struct jit_forest {
    uint32_t n_trees, n_nodes, n_samples, reserved;   /* n_trees <= 64, depth <= 64 */
    const uint32_t* root;          /* [n_trees] */
    const uint32_t* feature;       /* [n_nodes] 0..3, or 0xFFFFFFFF for a leaf */
    const uint32_t* threshold;     /* [n_nodes] split value; leaf: first sample */
    const uint32_t* left;          /* [n_nodes] left child; leaf: sample count */
    const uint32_t* right;         /* [n_nodes] */
    const uint32_t* samples;       /* [n_samples] */
} jit_forest;

/* Device bytes a forest needs (jit_sched_attach_forest's buffer). */
int jit_forest_bytes(const jit_forest* f, uint64_t* bytes);

/* Copy forest f (host arrays, validated) into dev_buf, which the caller keeps alive while it is
 * attached, and make it h's length estimator for steps and replays (f = NULL: back to the
 * table).  Invalidates every cached bound. */
int jit_sched_attach_forest(jit_sched* h, const jit_forest* f, void* dev_buf, uint64_t bytes);

/* Workspace for jit_sched_qrf_bound over n queries. */
int jit_qrf_workspace_bytes(uint32_t n, uint64_t* bytes);

/* Batch length bounds from the attached forest (one thread per query): x [n*4] = (L_i, dist_row,
 * -, group) host array (the anchor is derived from g with h's R), g [n] tokens generated; out [n]
 * = max(Q, g + 1).  kernel_ms (optional): device time of the kernel. */
int jit_sched_qrf_bound(jit_sched* h, const uint32_t* x, const uint32_t* g, uint32_t n, void* dev_workspace,
                        uint64_t ws_bytes, uint32_t* out, float* kernel_ms);

/* ---------------------------------------------------------------------------------------
 * Exact sharded step over W ranks (north_star "pool sharded by request id ... NCCL allgather
 * of candidates followed by a global merge").  Each rank loads its shard (ids
 * unique across ranks) and calls, in order, with the caller allgathering in between:
 *   jit_shard_prefix      (a1)-(a7) on the shard; writes the shard's first min(B*_r+1, |P_r|)
 *                         requests in (key desc, id asc) order as jit_rec1 to d_rec1 (device,
 *                         cap >= max_batch+1 records); *n_out = count.
 *   -- allgather the round-1 records of all ranks (unused slots: img = ~0) --
 *   jit_shard_merge       exact global B*, bp, thr from the union (every rank, identical).
 *   jit_shard_candidates  the shard's candidates key >= thr as jit_rec2 to d_rec2 (device).
 *   -- allgather the round-2 records (pad with img = ~0) --
 *   jit_shard_finish      the window (a9) over the union: the identical batch on every rank;
 *                         the bookkeeping is applied to this rank's own selected rows;
 *                         out->rows[i] = local row, or 0xFFFFFFFF for another rank's request.
 * Correctness: the global prefix restricted to a shard is a shard-local prefix within the
 * budget, and the global boundary request is in a shard's prefix or is its first misfit. */
typedef struct jit_rec1 { uint64_t img; uint32_t id, cost; } jit_rec1;
typedef struct jit_rec2 { uint64_t img; uint32_t id, cost, len, row, rank, reserved; } jit_rec2;

int jit_shard_prefix(jit_sched* h, int64_t now_ns, int64_t v_token_ns, void* d_rec1, uint32_t cap, uint32_t* n_out);

/* Fast sharded step (the speculative resolve of DESIGN.md §7 across ranks), tried first:
 *   jit_shard_spec_export   (a1)-(a6) on the shard, then writes jit_shard_spec_bytes() bytes to
 *                           d_out (device): a 64-byte header (the shard's pending count, cost sum,
 *                           min key, errors, set size) and the shard's speculative set
 *                           {key >= t} as 32-byte records (at most 1024; asynchronous).
 *   -- allgather the W exports in rank order (W * jit_shard_spec_bytes() bytes) --
 *   jit_shard_spec_resolve  every rank resolves the union: all ranks share the threshold t (they
 *                           resolved the same previous step), so the union of the local sets is
 *                           the global speculative set, a prefix of the global priority order,
 *                           and the exactness checks of the single-GPU resolve apply with the
 *                           global pending count.  Returns JIT_OK / JIT_EMPTY with the batch
 *                           (identical on every rank; bookkeeping on the owner's rows;
 *                           out->rows[i] = 0xFFFFFFFF for another rank's request), or JIT_RETRY:
 *                           the set is too large or a check failed -- continue this step with
 *                           jit_shard_prefix ... jit_shard_finish (the keys are not recomputed). */
uint32_t jit_shard_spec_bytes(void);
int jit_shard_spec_export(jit_sched* h, int64_t now_ns, int64_t v_token_ns, void* d_out, uint32_t cap_bytes,
                          uint32_t rank);
int jit_shard_spec_resolve(jit_sched* h, const void* d_all, uint32_t world, uint32_t rank, jit_batch* out);
int jit_shard_merge(jit_sched* h, const void* d_all_rec1, uint32_t n_all);
int jit_shard_candidates(jit_sched* h, void* d_rec2, uint32_t cap, uint32_t rank, uint32_t* n_out);
int jit_shard_finish(jit_sched* h, const void* d_all_rec2, uint32_t n_all, uint32_t rank, jit_batch* out);

/* ---------------------------------------------------------------------------------------
 * NEXT-2 power-of-K over M model replicas (§4.3: "each request has dummies on K
 * replicas ... once a request is assigned to a replica, its other dummies are removed";
 * DESIGN.md reading A51).  One handle per replica holds that replica's dummies (a standalone
 * pool: JIT_EINVAL with compound tasks; request ids shared across replicas) and runs the
 * ordinary step with the replica's own v_token (jit_sched_step).  Then:
 *   jit_multi_export     writes the replica's proposal -- a 32-byte header (the step's v_token,
 *                        replica index, count, capacity, resolved flag) and the batch ids in
 *                        window order -- to d_out (device, jit_multi_record_bytes() bytes;
 *                        asynchronous on cfg.stream).
 *   -- concatenate the M records in replica order (an allgather across ranks, one replica per
 *      GPU; or device copies on one GPU) --
 *   jit_multi_reconcile  every replica, against the union d_all (device, M records): a request
 *                        proposed by several replicas is assigned to the one with the smallest
 *                        v_token (priority G / (len_rem v + eps) is highest there), ties to the
 *                        lower index; the replica's batch keeps the requests it won in window
 *                        order (no refill) and `out` gets that batch (other fields as the step
 *                        left them); every dummy in this pool of a request assigned to another
 *                        replica becomes JIT_MOVED (terminal, never pending).
 * All replicas must share max_batch (capacity of the records).  Records whose header does not
 * match its slot fail with JIT_EINVAL.  Returns JIT_OK, or JIT_EMPTY if this replica's step had
 * no pending request. */
uint64_t jit_multi_record_bytes(const jit_sched* h);
int jit_multi_export(jit_sched* h, uint32_t replica, void* d_out);
int jit_multi_reconcile(jit_sched* h, const void* d_all, uint32_t n_replicas, uint32_t replica, jit_batch* out);

void jit_sched_destroy(jit_sched* h);
const char* jit_sched_last_error(const jit_sched* h);
const char* jit_sched_version(void);

#ifdef __cplusplus
}
#endif
#endif /* JIT_SCHED_H */
