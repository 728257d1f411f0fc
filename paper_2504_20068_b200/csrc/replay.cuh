// replay.cuh -- (a10) persistent trace replay: one CTA per replay (grid-stride over replays).
//
// Each CTA owns one replay at a time; the request state lives in shared memory for a few small
// traces, else in a per-CTA global slice (L2-resident), the selection working set in shared
// memory when it fits.  Per simulated iteration: stage releases / tool timers ->
// GMAX step over the replay's live rows (a1-a9, block-level: speculative sort of the pending
// composite keys {key >= t} -- bitonic, or rank sort for 129-384 keys, or one warp's registers
// for <= 32 pending rows --, block scan of costs for B*/bp, cutoff, sort of Cd by (len, id),
// one fused u64/u128 prefix scan for the windows) ->
// iteration latency c0 + c_att*max ctx + c_lin*|batch| -> token emission and goodput
// accounting (§3) -> stage barriers -> v_token = floor(trailing mean of Delta
// latencies).  Integer sums are order independent, so results are deterministic.
#pragma once
#include "common.cuh"
#include "select.cuh"

namespace jit {
// --------------------------------------------------------------------------------------
// per-row scoring of a standalone request: (a1) admission, (a2) length bound, (a3) t_rem,
// (a5) key, (a6) cost.  Pure function of the row + config; returns what to write back.
// --------------------------------------------------------------------------------------
struct RowRes {
    uint64_t img;
    uint32_t cost, meta, lhat, aux;
    bool pending, dropped, w_meta, w_lhat, err;
    double rate; int64_t trem; uint32_t lhatc;
};

// Per-group constants in the form the scoring loop uses (staged to shared memory per CTA):
//   t_rem = arrival + base + (Lhat-1)*tok - now      (LAT: base=TTFT, tok=TBT  [A9];
//                                                     DDL: base=E2EL; BE: base=default deadline)
//   G     = w_in_eff * L_i + w_out_eff * Lhat        (DDL: w_in, w_out; LAT: 0, w_out; BE: 0, 0)
struct GroupFast {
    int64_t base, tok;
    uint32_t w_in_eff, w_out_eff, type, pad;
};
__host__ __device__ inline GroupFast make_fast(const Group& g) {
    GroupFast f;
    f.type = g.type; f.pad = 0;
    f.base = g.type == kLAT ? g.ttft_ns : g.type == kDDL ? g.e2el_ns : g.type == kBE ? g.be_deadline_ns : 0;
    f.tok = g.type == kLAT ? g.tbt_ns : 0;
    f.w_in_eff = (g.type == kDDL || g.type == kCMP) ? g.w_in : 0;   // CMP: used by the compound pass
    f.w_out_eff = g.type != kBE ? g.w_out : 0;
    return f;
}

template <bool kDebug>
__device__ __forceinline__ void score_standalone(const Cfg& c, const Table& T, const GroupFast* sg, uint32_t n_groups,
                                                 const uint32_t* ovr, uint32_t row, int64_t now, int64_t v,
                                                 int64_t arr, uint32_t L_i, uint32_t g, uint32_t pre,
                                                 uint32_t lhat, uint32_t meta, uint32_t aux, uint32_t fair, RowRes& o) {
    o.img = kNone; o.cost = 0; o.meta = meta; o.lhat = lhat; o.aux = aux;
    o.pending = o.dropped = o.w_meta = o.w_lhat = o.err = false;
    if (kDebug) { o.rate = 0.0; o.trem = 0; o.lhatc = 0; }
    if (arr > now) return;
    const uint32_t st = m_state(meta), fl = m_flags(meta);
    if (st == kQueued && !(fl & kEver) && !(fl & kCompound) && now - arr > c.waiting) {   // (a1) P:545
        o.meta = m_with_state(meta, kDropped); o.w_meta = true; o.dropped = true;
        return;
    }
    if (st > kPreempted) return;
    o.pending = true;
    const uint32_t gi = m_group(meta);
    const uint32_t drow = aux & 0xFFFFu;
    if (gi >= n_groups || drow >= T.n_rows || (fl & kCompound)) { o.err = true; return; }
    const GroupFast G = sg[gi];
    if (G.type == kCMP) { o.err = true; return; }
    // (a2) conservative remaining length, refreshed every R tokens; cached per epoch
    const uint32_t ep = fastdiv(g, c.R, c.R_m, c.R_l);
    if (lhat == 0 || ep >= 65536u || m_epoch(meta) != ep) {
        lhat = T.forest ? qrf_bound(T.forest, L_i, drow, ep * c.R, gi, ep * c.R, c.qn, c.qd, T.l_max)
                        : ep == 0 ? __ldg(T.lhat0 + drow)    // anchor 0: the per-row table (k_lhat0)
                        : cond_quantile(T, drow, ep * c.R, c.qn, c.qd);
        o.lhat = lhat; o.w_lhat = true;
        if (ep < 65536u) { o.meta = (meta & 0xFFFFu) | (ep << 16); o.w_meta = true; }
    }
    const uint32_t Lh = lhat > g + 1 ? lhat : g + 1;
    const uint32_t len_rem = Lh - g;
    o.cost = token_cost(L_i, pre, c.chunk);
    const uint64_t t_gen = (uint64_t)len_rem * (uint64_t)v;
    const int64_t trem = arr + G.base + (int64_t)(Lh - 1) * G.tok - now;  // (a3)
    uint64_t Gk = (uint64_t)G.w_in_eff * L_i + (uint64_t)G.w_out_eff * Lh;  // (a5) A10/A11
    if (fl & kOverride) Gk = __ldg(ovr + row);
    if (trem <= 0) Gk = 0;                                      // A22
    if (c.appb && t_gen > (uint64_t)(trem > 0 ? trem : 0)) Gk = 0;
    const uint64_t Gp = Gk + (uint64_t)c.delta * fastdiv(aux >> 16, c.frame, c.F_m, c.F_l);
    double key;
    if (!make_key(Gp, t_gen, c.eps, &key)) { o.err = true; return; }
    if (c.fair_num) key = blend_fair(key, fair, c.fair_num, c.fair_den);   // NEXT-2 (A47)
    o.img = (uint64_t)__double_as_longlong(key);
    if (kDebug) { o.rate = make_rate(len_rem, trem); o.trem = trem; o.lhatc = Lh; }
}

}  // namespace jit

namespace jit {

// one replay = one CTA: 512 threads when a few replays run (one long trace: the per-step passes
// spread wide), 128 threads x 8 CTAs per SM for sweeps (more replays in flight per SM: the step is
// barrier- and latency-bound).  C5(i) sweep on B200 (profiles/sweep_variants.py): 256 threads x 3
// CTAs (2048 sort rows in shared memory) 9.8 M steps/s; 128 x 6 (1024 rows) 11.0; 128 x 6 (512)
// 12.5; 128 x 8 (512 rows, 64 registers) 13.0; 128 x 8 (256) 12.2; 96 x 8 11.4; 64 x 12 8.9; then
// the warp path for <= 32 pending rows in sweeps too (+5%) and rank sorts for sets of 129-384 keys.
// A step whose live rows exceed the shared sort buffers sorts in the CTA's global slice.
constexpr uint32_t kReplayThreads = 512;
constexpr uint32_t kReplayThreadsSweep = 128;
constexpr uint32_t kReplayThreadsMid = 256;
#ifndef JIT_REPLAY_MARGIN
#define JIT_REPLAY_MARGIN 0.97
#endif
// next step's speculative threshold: this cutoff x margin.  C5(i) sweep on B200 (steps/s; full
// re-sorts after a failed check per 4096 steps of the highest-load replay): 0.85 16.0 M; 0.90
// 17.2 M; 0.95 18.4 M (102); 0.97 18.75 M (121); 0.99 18.8 M (153)
constexpr double kReplayMargin = JIT_REPLAY_MARGIN;    // sweeps of fewer than 6 replays per SM: 3 CTAs per SM
constexpr uint32_t kReplaySweepRows = 512;     // sweep CTAs: rows sorted in shared memory
constexpr uint32_t kReplaySweepCtas = 8;       // sweep CTAs per SM (launch bounds: <= 64 registers)
constexpr uint32_t kReplayThreadsTiny = 64;     // traces of <= 64 rows (e.g. C1): two warps, cheap barriers
constexpr uint32_t kReplayTinyRows = 64;
constexpr uint32_t kReplaySmemRows = 2048;    // rows sorted in shared memory up to this size

struct TraceMeta { uint32_t row_off, task_off, n_rows, n_tasks, n_std, pad; };   // n_std: standalone rows

struct Spec { uint32_t trace, reserved; uint64_t load_num, load_den, slo_num, slo_den; };

struct RLog { int64_t now_ns; uint32_t n_selected, total_tokens, n_candidates, b_star; double bp; uint64_t ids_hash;
              int64_t v_token_ns; uint32_t n_preempted, p_num; int64_t stall_ns; };

struct RResult {
    unsigned long long token_goodput, tokens_processed;
    int64_t sim_end_ns;
    uint32_t request_goodput, n_done, n_dropped, steps, n_tasks_done, n_tasks_dropped, error, n_preempted;
};

struct ReplayArgs {
    const TraceMeta* traces;
    const int64_t* arrival; const uint32_t *len_in, *true_out, *group, *dist_row, *ovr, *task, *fair;
    const uint32_t* order;      // per trace: its standalone rows by (arrival, row) (admission order)
    const int64_t *t_arr, *t_dl; const uint32_t* t_nst;
    const uint32_t* st_kind; const int64_t* st_exec; const uint32_t *st_pat, *st_cb, *st_ce;
    const Spec* specs;
    uint32_t n_replays, n_steps, log_steps, max_rows, max_tasks, n_groups, state_smem, pad1;
    int64_t v0, c0, c_att, c_lin;
    Table T; const Group* groups; Cfg c;
    unsigned char* state; uint64_t state_stride;
    RResult* out; RLog* log;
    uint32_t p_adapt, eps_num, eps_den, window_frames;   // NEXT-2 online p (A48)
    uint64_t seed;
};

// NEXT-2 online p (A48): the arms p = kPGrid[a] / 100 and the counter-based draw
__constant__ uint32_t kPGrid[4] = {80, 90, 95, 100};
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t x) {
    uint64_t z = x * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// per-CTA state slice layout
struct RState {
    int64_t* arr; uint32_t *gen, *pre, *lhat, *meta, *aux, *late, *cost; uint64_t* img;
    uint32_t *cur, *left, *tdone, *cb, *ce, *tever; int64_t *timer, *ta, *tD; unsigned long long* gdone;
    uint64_t *tle, *ttot;
    unsigned long long *tT, *tG; int64_t* tDs;   // per-step stage sums (len_rem, goodput); D_s
    u128* gA; uint32_t* gAv; uint64_t* gB; uint32_t* gBv; unsigned long long* gpc; u128* gpf;  // global sort scratch
    uint32_t* batch; int64_t* ring;
    uint32_t* live;             // the rows that can be pending: arrived / released, not Done or Dropped
};

__host__ __device__ inline uint64_t replay_state_bytes(uint32_t M, uint32_t MT, uint32_t max_batch) {
    const uint64_t m = M + 64, mt = MT + 1;
    uint64_t b = 0;
    b += 8 * m + 4 * m * 7 + 8 * m + 4 * m;    // arr, gen..cost, img, live
    b += 4 * mt * 6 + 8 * mt * 3 + 8 * mt + 16 * mt + 24 * mt;   // task u32 x6, i64 x3, gdone, tle+ttot, tT+tG+tDs
    uint64_t p2 = 1;                            // bitonic sorts pad to a power of two
    while (p2 < m) p2 <<= 1;
    b += 16 * p2 + 4 * p2 + 8 * p2 + 4 * p2 + 8 * (m + 1) + 16 * (m + 1);
    b += 4 * (uint64_t)(max_batch + 1) + 8 * 1024;
    return b + 64 * 32;                         // alignment slack
}

// the per-replay state without the global sort scratch (rows, tasks, batch, v_token ring): kept
// in shared memory when it fits beside the sort buffers (traces of <= kReplaySmemRows rows)
__host__ __device__ inline uint64_t replay_core_bytes(uint32_t M, uint32_t MT, uint32_t max_batch) {
    const uint64_t m = M + 64, mt = MT + 1;
    auto r = [](uint64_t b) { return (b + 63) & ~63ull; };
    return r(8 * m) + 7 * r(4 * m) + r(8 * m) + 6 * r(4 * mt) + 9 * r(8 * mt) + r(4 * (uint64_t)(max_batch + 1)) +
           r(8 * 1024) + r(4 * m);
}
__device__ inline RState carve_core(unsigned char* p, uint32_t M, uint32_t MT, uint32_t max_batch) {
    const uint64_t m = M + 64, mt = MT + 1;
    RState s{};
    auto take = [&](uint64_t bytes) { unsigned char* q = p; p += (bytes + 63) & ~63ull; return q; };
    s.arr = (int64_t*)take(8 * m);
    s.gen = (uint32_t*)take(4 * m); s.pre = (uint32_t*)take(4 * m); s.lhat = (uint32_t*)take(4 * m);
    s.meta = (uint32_t*)take(4 * m); s.aux = (uint32_t*)take(4 * m); s.late = (uint32_t*)take(4 * m);
    s.cost = (uint32_t*)take(4 * m); s.img = (uint64_t*)take(8 * m);
    s.cur = (uint32_t*)take(4 * mt); s.left = (uint32_t*)take(4 * mt); s.tdone = (uint32_t*)take(4 * mt);
    s.cb = (uint32_t*)take(4 * mt); s.ce = (uint32_t*)take(4 * mt); s.tever = (uint32_t*)take(4 * mt);
    s.timer = (int64_t*)take(8 * mt); s.ta = (int64_t*)take(8 * mt); s.tD = (int64_t*)take(8 * mt);
    s.gdone = (unsigned long long*)take(8 * mt); s.tle = (uint64_t*)take(8 * mt); s.ttot = (uint64_t*)take(8 * mt);
    s.tT = (unsigned long long*)take(8 * mt); s.tG = (unsigned long long*)take(8 * mt); s.tDs = (int64_t*)take(8 * mt);
    s.batch = (uint32_t*)take(4 * (uint64_t)(max_batch + 1)); s.ring = (int64_t*)take(8 * 1024);
    s.live = (uint32_t*)take(4 * m);
    return s;
}

__device__ inline RState carve_state(unsigned char* p, uint32_t M, uint32_t MT, uint32_t max_batch) {
    const uint64_t m = M + 64, mt = MT + 1;
    RState s;
    auto take = [&](uint64_t bytes) { unsigned char* q = p; p += (bytes + 63) & ~63ull; return q; };
    s.arr = (int64_t*)take(8 * m);
    s.gen = (uint32_t*)take(4 * m); s.pre = (uint32_t*)take(4 * m); s.lhat = (uint32_t*)take(4 * m);
    s.meta = (uint32_t*)take(4 * m); s.aux = (uint32_t*)take(4 * m); s.late = (uint32_t*)take(4 * m);
    s.cost = (uint32_t*)take(4 * m); s.img = (uint64_t*)take(8 * m);
    s.cur = (uint32_t*)take(4 * mt); s.left = (uint32_t*)take(4 * mt); s.tdone = (uint32_t*)take(4 * mt);
    s.cb = (uint32_t*)take(4 * mt); s.ce = (uint32_t*)take(4 * mt); s.tever = (uint32_t*)take(4 * mt);
    s.timer = (int64_t*)take(8 * mt); s.ta = (int64_t*)take(8 * mt); s.tD = (int64_t*)take(8 * mt);
    s.gdone = (unsigned long long*)take(8 * mt); s.tle = (uint64_t*)take(8 * mt); s.ttot = (uint64_t*)take(8 * mt);
    s.tT = (unsigned long long*)take(8 * mt); s.tG = (unsigned long long*)take(8 * mt); s.tDs = (int64_t*)take(8 * mt);
    uint64_t p2 = 1;
    while (p2 < m) p2 <<= 1;
    s.gA = (u128*)take(16 * p2); s.gAv = (uint32_t*)take(4 * p2); s.gB = (uint64_t*)take(8 * p2);
    s.gBv = (uint32_t*)take(4 * p2); s.gpc = (unsigned long long*)take(8 * (m + 1)); s.gpf = (u128*)take(16 * (m + 1));
    s.batch = (uint32_t*)take(4 * (uint64_t)(max_batch + 1)); s.ring = (int64_t*)take(8 * 1024);
    s.live = (uint32_t*)take(4 * m);
    return s;
}

__device__ __forceinline__ int64_t scale_t(int64_t t, uint64_t num, uint64_t den) {
    return (int64_t)((u128)(uint64_t)t * num / den);
}

__device__ __forceinline__ uint64_t call_R(const Group& g, uint32_t L_i, uint32_t L_o) {
    return (uint64_t)g.w_in * L_i + (uint64_t)g.w_out * L_o;
}

__host__ __device__ inline uint32_t replay_groups_bytes(uint32_t n_groups) {
    return (uint32_t)(((sizeof(Group) + sizeof(GroupFast)) * n_groups + 63) & ~63ull);
}

// diagnostics (-DJIT_REPLAY_STAMPS=k): %globaltimer per step phase of replay k - 1, printed at its end
#ifdef JIT_REPLAY_STAMPS
constexpr uint32_t kStampRep = JIT_REPLAY_STAMPS - 1;
#define RSTAMP(i) do { if (threadIdx.x == 0 && rep == kStampRep) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); if ((i) > 0) s_ph[(i)] += t_ - s_ph_last; s_ph_last = t_; } } while (0)
#else
#define RSTAMP(i) do {} while (0)
#endif
template <uint32_t NT, uint32_t SR, uint32_t MINB>
__global__ void __launch_bounds__(NT, MINB) k_replay(ReplayArgs A) {
#ifdef JIT_REPLAY_STAMPS
    __shared__ unsigned long long s_ph[20], s_ph_last;
    if (threadIdx.x < 20) s_ph[threadIdx.x] = 0;
#endif
    extern __shared__ __align__(16) unsigned char smem[];
    Group* sg = reinterpret_cast<Group*>(smem);                                   // the SLO groups
    GroupFast* sgf = reinterpret_cast<GroupFast*>(smem + sizeof(Group) * A.n_groups);   // their scoring form
    unsigned char* sbuf = smem + replay_groups_bytes(A.n_groups);
    // region A (24 cap + 64 B): pending sort (u128 key + u32 row), later reused for the
    // window prefix sums (u64 cost + u128 fixed-point key); region B: Cd sort (u64 + u32)
    u128* sA = reinterpret_cast<u128*>(sbuf);
    uint32_t* sAv = reinterpret_cast<uint32_t*>(sbuf + 16 * SR);
    uint64_t* sB = reinterpret_cast<uint64_t*>(sbuf + 24 * SR + 64);
    uint32_t* sBv = reinterpret_cast<uint32_t*>(sbuf + 32 * SR + 64);
    __shared__ uint64_t s_scan[32];
    __shared__ u128 s_scan128[32];
    __shared__ u128 s_best[32];
    __shared__ uint32_t s_bi[32], s_bj[32];
    __shared__ unsigned long long s_good, s_tok, s_min;
    __shared__ uint32_t s_reqg, s_done, s_drop, s_tdone, s_tdrop, s_err, s_npend, s_cnt;
    __shared__ int64_t s_now, s_maxctx, s_nxt;
    __shared__ long long s_tmin;                  // <= every task timer: no stage starts before it
    __shared__ uint32_t s_steps, s_ring_n, s_ring_pos;
    __shared__ uint32_t s_nlive, s_aptr;          // live rows; next standalone row to admit (arrival order)
    __shared__ int64_t s_ring_sum;
    __shared__ uint32_t s_bstar, s_ncd, s_nsel, s_tot;
    __shared__ double s_bp, s_thr;
    __shared__ uint64_t s_thr_img, s_tguess;
    __shared__ uint32_t s_m, s_spec_ok;
    __shared__ bool s_stop;
    __shared__ uint32_t s_npre, s_gate_n;           // NEXT-1 gate: evictions this step / total; P+I count
    __shared__ unsigned long long s_stall;
    __shared__ double s_p;                            // the cutoff p of this step (A48 adapts it)
    __shared__ uint32_t s_pnum, s_arm, s_gcnt[4];
    __shared__ unsigned long long s_gsum[4], s_gstart, s_window;

    const Cfg c = A.c;
    const Table T = A.T;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // the replay state in shared memory (behind the sort buffers) when it fits, else in this CTA's
    // global slice
    RState S = A.state_smem ? carve_core(sbuf + 36 * SR + 64, A.max_rows, A.max_tasks, c.max_batch)
                            : carve_state(A.state + (uint64_t)blockIdx.x * A.state_stride, A.max_rows, A.max_tasks,
                                          c.max_batch);

    for (uint32_t rep = blockIdx.x; rep < A.n_replays; rep += gridDim.x) {
        const Spec sp = A.specs[rep];
        const TraceMeta tm = A.traces[sp.trace];
        const uint32_t n = tm.n_rows, nt = tm.n_tasks, n_std = tm.n_std;
        const uint32_t* order = A.order + tm.row_off;
        const int64_t* tr_arr = A.arrival + tm.row_off;
        const uint32_t* L_in = A.len_in + tm.row_off;
        const uint32_t* L_out = A.true_out + tm.row_off;
        const uint32_t* grp = A.group + tm.row_off;
        const uint32_t* drow = A.dist_row + tm.row_off;
        const uint32_t* ovr = A.ovr + tm.row_off;
        const uint32_t* tsk = A.task + tm.row_off;
        const uint32_t* st_kind = A.st_kind + (uint64_t)tm.task_off * kMaxStages;
        const int64_t* st_exec = A.st_exec + (uint64_t)tm.task_off * kMaxStages;
        const uint32_t* st_pat = A.st_pat + (uint64_t)tm.task_off * kMaxStages;
        const uint32_t* st_cb = A.st_cb + (uint64_t)tm.task_off * kMaxStages;
        const uint32_t* st_ce = A.st_ce + (uint64_t)tm.task_off * kMaxStages;

        // ---- setup: SLO-scaled groups, initial row and task state
        for (uint32_t g = threadIdx.x; g < A.n_groups; g += blockDim.x) {
            Group G = A.groups[g];
            G.ttft_ns = scale_t(G.ttft_ns, sp.slo_num, sp.slo_den);
            G.tbt_ns = scale_t(G.tbt_ns, sp.slo_num, sp.slo_den);
            G.e2el_ns = scale_t(G.e2el_ns, sp.slo_num, sp.slo_den);
            G.be_deadline_ns = scale_t(G.be_deadline_ns, sp.slo_num, sp.slo_den);
            sg[g] = G;
            sgf[g] = make_fast(G);
        }
        if (threadIdx.x == 0) {
            s_good = 0; s_tok = 0; s_reqg = 0; s_done = 0; s_drop = 0; s_tdone = 0; s_tdrop = 0; s_err = 0;
            s_now = 0; s_steps = 0; s_ring_n = 0; s_ring_pos = 0; s_ring_sum = 0; s_stop = false;
            s_nlive = 0; s_aptr = 0; s_tmin = LLONG_MAX;
            s_tguess = kNone;                              // no speculative threshold before the first step
            s_npre = 0; s_stall = 0;
            s_arm = 0; s_gstart = 0; s_window = 0;
            for (int a = 0; a < 4; ++a) { s_gcnt[a] = 0; s_gsum[a] = 0; }
            s_pnum = A.p_adapt ? kPGrid[0] : c.pn;
            s_p = A.p_adapt ? __ddiv_rn((double)kPGrid[0], 100.0) : c.p;
        }
        uint32_t n_preempted_total = 0;                    // (thread 0)
        __syncthreads();
        for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
            const bool comp = tsk[r] != kNoTask;
            uint32_t fl = (comp ? kCompound : 0u) | (ovr[r] ? kOverride : 0u);
            const uint32_t g = grp[r];
            bool bad = L_in[r] == 0 || L_out[r] == 0 || g >= A.n_groups || drow[r] >= T.n_rows ||
                       (ovr[r] && sg[g].type != kDDL) || (comp != (sg[g].type == kCMP)) || (comp && tsk[r] >= nt);
            if (bad) atomicOr(&s_err, 1u);
            S.meta[r] = g | ((comp ? kWaiting : kQueued) << 8) | (fl << 12);
            S.aux[r] = drow[r] & 0xFFFFu;
            S.gen[r] = 0; S.pre[r] = 0; S.lhat[r] = 0; S.late[r] = 0;
            S.arr[r] = comp ? INT64_MAX : scale_t(tr_arr[r], sp.load_den, sp.load_num);
        }
        for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
            const uint32_t tg = tm.task_off + t;
            S.ta[t] = scale_t(A.t_arr[tg], sp.load_den, sp.load_num);
            S.tD[t] = scale_t(A.t_dl[tg], sp.slo_num, sp.slo_den);
            const uint32_t Sn = A.t_nst[tg];
            if (Sn == 0 || Sn > kMaxStages) atomicOr(&s_err, 1u);
            uint64_t tot = 0;
            for (uint32_t u = 0; u < Sn && u < kMaxStages; ++u) tot += (uint64_t)st_pat[t * kMaxStages + u] * 1000000ull;
            S.ttot[t] = tot; S.tle[t] = 0; S.tDs[t] = 0;
            atomicMin(&s_tmin, (long long)S.ta[t]);
            S.timer[t] = S.ta[t]; S.cur[t] = 0; S.cb[t] = 0; S.ce[t] = 0; S.left[t] = 0; S.tdone[t] = 0; S.gdone[t] = 0;
            S.tever[t] = 0;
        }
        __syncthreads();

        while (!s_err) {
            const int64_t now = s_now;
            RSTAMP(0);
            // ---- stage starts whose time has come (task arrival or the end of the previous stage);
            // none before s_tmin (a lower bound of every timer), so most steps skip the task walk
            if (now >= s_tmin) {
            long long my_min = LLONG_MAX;
            for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
                const uint32_t Sn = A.t_nst[tm.task_off + t];
                while (!S.tdone[t] && S.timer[t] <= now) {
                    const int64_t at = S.timer[t];
                    const uint32_t s = S.cur[t];
                    if (s == Sn) {
                        S.tdone[t] = 1; atomicAdd(&s_tdone, 1u); S.timer[t] = INT64_MAX;
                        if (at <= S.ta[t] + S.tD[t]) {                       // §3
                            unsigned long long tot = 0;
                            for (uint32_t u = 0; u < Sn; ++u) {
                                const uint32_t kk = t * kMaxStages + u;
                                if (st_kind[kk] == 0)
                                    for (uint32_t q = st_cb[kk]; q < st_ce[kk]; ++q) tot += call_R(sg[grp[q]], L_in[q], L_out[q]);
                            }
                            atomicAdd(&s_good, tot); atomicAdd(&s_reqg, 1u);
                        }
                        break;
                    }
                    const uint32_t k = t * kMaxStages + s;
                    if (st_kind[k] == 1) { S.cur[t] = s + 1; S.timer[t] = at + st_exec[k]; continue; }
                    const uint32_t b = st_cb[k], e = st_ce[k];
                    if (b >= e || e > n) { atomicOr(&s_err, 1u); break; }
                    S.cb[t] = b; S.ce[t] = e; S.left[t] = e - b;
                    const uint32_t lp = atomicAdd(&s_nlive, e - b);        // the stage's calls become live
                    for (uint32_t r = b; r < e; ++r) {
                        S.arr[r] = at; S.meta[r] = m_with_state(S.meta[r], kQueued); S.live[lp + r - b] = r;
                    }
                    uint64_t le = 0;
                    for (uint32_t u = 0; u <= s; ++u) le += (uint64_t)st_pat[t * kMaxStages + u] * 1000000ull;
                    S.tle[t] = le;
                    // D_s = floor(D t_<=s / t_total) (A43): fixed until the next stage release
                    S.tDs[t] = S.ttot[t] ? (int64_t)((u128)(uint64_t)S.tD[t] * le / S.ttot[t]) : 0;
                    S.timer[t] = INT64_MAX;
                }
                if (!S.tdone[t] && S.timer[t] < my_min) my_min = S.timer[t];
            }
            __syncthreads();
            if (threadIdx.x == 0) s_tmin = LLONG_MAX;
            __syncthreads();
            if (my_min != LLONG_MAX) atomicMin(&s_tmin, my_min);
            }
            __syncthreads();
            RSTAMP(1);
            if (s_steps >= A.n_steps || s_err) break;
            const int64_t v = s_ring_n ? s_ring_sum / (int64_t)s_ring_n : A.v0;
            // ---- the live rows: drop the finished ones (stable compaction), admit the standalone
            // arrivals up to now (rows in arrival order: the admitted ones are a prefix).  Every
            // per-row pass below runs over the live rows only -- rows not yet arrived and rows that
            // are Done or Dropped can never be pending, and no pass writes them.
            {
                const uint32_t nl = s_nlive;
                uint32_t carry = 0;
                for (uint32_t base = 0; base < nl; base += blockDim.x) {
                    const uint32_t i = base + threadIdx.x;
                    uint32_t r = 0, keep = 0;
                    if (i < nl) {
                        r = S.live[i];
                        const uint32_t st = m_state(S.meta[r]);
                        keep = st != kDone && st != kDropped;
                    }
                    uint64_t tot;
                    const uint32_t pos = (uint32_t)block_exclusive_scan_u64(keep, s_scan, &tot);
                    if (keep) S.live[carry + pos] = r;
                    carry += (uint32_t)tot;
                    __syncthreads();
                }
                uint32_t ap = s_aptr;
                while (true) {
                    const uint32_t i = ap + threadIdx.x;
                    uint32_t r = 0;
                    bool adm = false;
                    if (i < n_std) { r = order[i]; adm = S.arr[r] <= now; }
                    const uint32_t k = (uint32_t)__syncthreads_count(adm);
                    if (adm) S.live[carry + threadIdx.x] = r;
                    carry += k; ap += k;
                    if (k < blockDim.x) break;
                }
                __syncthreads();
                if (threadIdx.x == 0) { s_nlive = carry; s_aptr = ap; }
                __syncthreads();
                RSTAMP(2);
            }
            const uint32_t nl = s_nlive;
            // every sort / prefix array of the step holds at most the live rows: shared memory when
            // they fit (whatever the trace length), else this CTA's global scratch
            const bool in_smem = nl <= SR;
            u128* bA = in_smem ? sA : S.gA;
            uint32_t* bAv = in_smem ? sAv : S.gAv;
            uint64_t* bB = in_smem ? sB : S.gB;
            uint32_t* bBv = in_smem ? sBv : S.gBv;

            // ---- (a1)-(a6) scoring of every row; steps_waited+1 for pending rows
            uint32_t my_pend = 0, my_drop = 0, my_err = 0;
            for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                const uint32_t r = S.live[i];
                const uint32_t meta = S.meta[r];
                if (m_flags(meta) & kCompound) continue;
                RowRes o;
                score_standalone<false>(c, T, sgf, A.n_groups, ovr, r, now, v, S.arr[r], L_in[r], S.gen[r], S.pre[r],
                                        S.lhat[r], meta, S.aux[r], A.fair ? A.fair[tm.row_off + r] : 0u, o);
                S.img[r] = o.img; S.cost[r] = o.cost; S.aux[r] = o.aux;
                if (o.w_meta) S.meta[r] = o.meta;
                if (o.w_lhat) S.lhat[r] = o.lhat;
                my_pend += o.img != kNone; my_drop += o.dropped; my_err |= o.err;
            }
            RSTAMP(16);
            // (a4) compound tasks, in three passes: per task the admission drop (A40) and the reset
            // of its stage sums; per live call (in parallel) the refreshed bound and its share of the
            // stage sums (integer atomics: order independent); per live call its key from its task's
            // sums.  The same rows, sums and keys as one thread walking each task's stage.
            for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
                if (S.tdone[t]) continue;
                S.tT[t] = 0; S.tG[t] = 0;
                if (!S.tever[t] && now - S.ta[t] > c.waiting) {
                    // (a1) P:545, A40: a task none of whose calls was ever scheduled is dropped once it
                    // waited longer than waiting_time: its Queued / Waiting calls of every stage
                    const uint32_t b = S.cb[t], e = S.ce[t];
                    bool hit = false;
                    for (uint32_t r = b; r < e; ++r) {
                        const uint32_t st = m_state(S.meta[r]);
                        hit |= st == kQueued || st == kWaiting;
                    }
                    if (hit) {
                        const uint32_t Sn = A.t_nst[tm.task_off + t];
                        for (uint32_t u = 0; u < Sn; ++u) {
                            const uint32_t kk = t * kMaxStages + u;
                            if (st_kind[kk] != 0) continue;
                            for (uint32_t r = st_cb[kk]; r < st_ce[kk]; ++r) {
                                const uint32_t st = m_state(S.meta[r]);
                                if (st == kQueued || st == kWaiting) { S.meta[r] = m_with_state(S.meta[r], kDropped); ++my_drop; }
                            }
                        }
                        S.tdone[t] = 1; S.timer[t] = INT64_MAX; S.cb[t] = 0; S.ce[t] = 0;
                        atomicAdd(&s_tdrop, 1u);
                    }
                }
            }
            __syncthreads();
            RSTAMP(18);
            // the live compound rows are exactly the calls of the tasks' current stages that are
            // not Done / Dropped; the pending ones (arrived, state <= Preempted) contribute
            for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                const uint32_t r = S.live[i];
                const uint32_t meta = S.meta[r];
                if (!(m_flags(meta) & kCompound)) continue;
                if (S.arr[r] > now || m_state(meta) > kPreempted) { S.img[r] = kNone; S.cost[r] = 0; continue; }
                const uint32_t g = S.gen[r];
                uint32_t lhat = S.lhat[r];
                const uint32_t ep = g / c.R;
                if (lhat == 0 || ep >= 65536u || m_epoch(meta) != ep) {
                    lhat = T.forest ? qrf_bound(T.forest, L_in[r], S.aux[r] & 0xFFFFu, ep * c.R, m_group(meta),
                                                ep * c.R, c.qn, c.qd, T.l_max)
                                    : ep == 0 ? __ldg(T.lhat0 + (S.aux[r] & 0xFFFFu))
                                    : cond_quantile(T, S.aux[r] & 0xFFFFu, ep * c.R, c.qn, c.qd);
                    S.lhat[r] = lhat;
                    if (ep < 65536u) S.meta[r] = (meta & 0xFFFFu) | (ep << 16);
                }
                const uint32_t Lh = lhat > g + 1 ? lhat : g + 1;
                const Group& G = sg[m_group(meta)];
                const uint32_t t = tsk[r];
                atomicAdd(&S.tT[t], (unsigned long long)(Lh - g));
                atomicAdd(&S.tG[t], (unsigned long long)((uint64_t)G.w_in * L_in[r] + (uint64_t)G.w_out * Lh));
            }
            __syncthreads();
            RSTAMP(19);
            for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                const uint32_t r = S.live[i];
                const uint32_t meta = S.meta[r];
                if (!(m_flags(meta) & kCompound) || S.arr[r] > now || m_state(meta) > kPreempted) continue;
                const uint32_t t = tsk[r];
                uint64_t Gt = S.gdone[t] + S.tG[t];
                if (S.ta[t] + S.tD[t] <= now) Gt = 0;
                const int64_t trem = S.ta[t] + S.tDs[t] - now;
                const uint64_t t_gen = S.tT[t] * (uint64_t)v;
                if (c.appb && t_gen > (uint64_t)(trem > 0 ? trem : 0)) Gt = 0;
                const uint64_t Gp = Gt + (uint64_t)c.delta * ((S.aux[r] >> 16) / c.frame);
                double key;
                if (!make_key(Gp, t_gen, c.eps, &key)) my_err = 1;
                if (c.fair_num) key = blend_fair(key, A.fair ? A.fair[tm.row_off + r] : 0u, c.fair_num, c.fair_den);
                S.img[r] = (uint64_t)__double_as_longlong(key);
                S.cost[r] = token_cost(L_in[r], S.pre[r], c.chunk);
                ++my_pend;
            }
            RSTAMP(17);
            my_pend = warp_sum(my_pend); my_drop = warp_sum(my_drop);
            my_err = __reduce_or_sync(0xffffffffu, my_err);
            if (threadIdx.x == 0) { s_npend = 0; }
            __syncthreads();
            if (lane == 0) { atomicAdd(&s_npend, my_pend); atomicAdd(&s_drop, my_drop); if (my_err) atomicOr(&s_err, 1u); }
            __syncthreads();
            RSTAMP(3);
            if (s_err) break;
            const uint32_t np = s_npend;
            if (np == 0) {
                // idle: jump to the next arrival / stage start; stop when drained
                if (threadIdx.x == 0) s_nxt = INT64_MAX;
                __syncthreads();
                // the next standalone arrival is the first row not admitted yet (arrival order)
                int64_t my = (threadIdx.x == 0 && s_aptr < n_std) ? S.arr[order[s_aptr]] : INT64_MAX;
                for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x)
                    if (!S.tdone[t] && S.timer[t] != INT64_MAX && S.timer[t] > now && S.timer[t] < my) my = S.timer[t];
                atomicMin((unsigned long long*)&s_nxt, (unsigned long long)my);
                __syncthreads();
                if (s_nxt == INT64_MAX) break;
                if (threadIdx.x == 0) s_now = s_nxt;
                __syncthreads();
                continue;
            }

            // ---- (a7)-(a9) for at most 32 pending rows: warp 0 alone, everything in registers and
            // shuffles (the block's many short barrier-separated phases dominate a small step);
            // the same orders, sums and tie-breaks as the general path below, so the same batch.
            if (np <= 32u) {
                if (wid == 0) {
                    // the pending rows (img != kNone) of the live list, compacted to lanes 0..np-1
                    uint32_t cnt = 0;
                    for (uint32_t base = 0; base < nl; base += 32) {
                        const uint32_t i = base + lane;
                        const uint32_t r = i < nl ? S.live[i] : 0u;
                        const bool p = i < nl && S.img[r] != kNone;
                        const unsigned pm = __ballot_sync(0xffffffffu, p);
                        if (p) bAv[cnt + __popc(pm & ((1u << lane) - 1u))] = r;
                        cnt += __popc(pm);
                    }
                    __syncwarp();
                    const bool own = lane < np;
                    uint32_t row = own ? bAv[lane] : 0u;
                    u128 ck = own ? make_ck(S.img[row], row) : ~(u128)0;
                    // (a7) ascending composite key (key desc, id asc): 32-lane bitonic network
                    for (uint32_t size = 2; size <= 32; size <<= 1)
                        for (uint32_t j = size >> 1; j > 0; j >>= 1) {
                            const u128 ok = shfl_xor_u128(ck, (int)j);
                            const uint32_t orow = __shfl_xor_sync(0xffffffffu, row, (int)j);
                            const bool up = (lane & size) == 0, lower = (lane & j) == 0;
                            if (lower == up ? (ok < ck) : (ok > ck)) { ck = ok; row = orow; }
                        }
                    const uint64_t img = own ? ck_img(ck) : kNone;
                    uint64_t pre = own ? (uint64_t)S.cost[row] : 0ull;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint64_t y = __shfl_up_sync(0xffffffffu, pre, o);
                        if (lane >= (uint32_t)o) pre += y;
                    }
                    const bool fits = own && lane + 1 <= c.max_batch && pre <= c.token_budget;
                    const uint32_t bstar = __popc(__ballot_sync(0xffffffffu, fits));
                    const uint64_t bp_img = __shfl_sync(0xffffffffu, img, bstar ? bstar - 1 : 0);
                    const double bp = __longlong_as_double((long long)bp_img);
                    const double thr = __dmul_rn(s_p, bp);
                    const uint64_t thr_img = (uint64_t)__double_as_longlong(thr);
                    // (a8) Cd = the prefix with key >= thr; (a9) its (len, id) order
                    const bool cd = own && img >= thr_img;
                    const uint32_t ncd_w = __popc(__ballot_sync(0xffffffffu, cd));
                    uint64_t wk = cd ? (((uint64_t)(c.len_key ? L_in[row] + S.gen[row] : L_in[row]) << 32) | row) : ~0ull;
                    for (uint32_t size = 2; size <= 32; size <<= 1)
                        for (uint32_t j = size >> 1; j > 0; j >>= 1) {
                            const uint64_t ok = __shfl_xor_sync(0xffffffffu, wk, (int)j);
                            const uint32_t orow = __shfl_xor_sync(0xffffffffu, row, (int)j);
                            const bool up = (lane & size) == 0, lower = (lane & j) == 0;
                            if (lower == up ? (ok < wk) : (ok > wk)) { wk = ok; row = orow; }
                        }
                    const bool inw = lane < ncd_w;
                    const uint64_t cv = inw ? (uint64_t)S.cost[row] : 0ull;
                    const u128 fv = inw ? (u128)fixed_point(__longlong_as_double((long long)S.img[row])) : (u128)0;
                    uint64_t pci = cv;                                  // inclusive prefix sums in window order
                    u128 pfi = fv;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint64_t yc = __shfl_up_sync(0xffffffffu, pci, o);
                        const u128 yf = shfl_up_u128(pfi, o);
                        if (lane >= (uint32_t)o) { pci += yc; pfi += yf; }
                    }
                    const uint64_t pce = pci - cv;                      // exclusive (pc[i])
                    const u128 pfe = pfi - fv;
                    // the window of start i: the largest j <= min(ncd - 1, i + B_max - 1) with
                    // pc[j + 1] <= pc[i] + tau (a uniform 5-step binary search over the lanes)
                    const uint64_t lim = pce + c.token_budget;
                    uint32_t lo = lane, hi = inw ? (uint32_t)min((uint64_t)ncd_w - 1, (uint64_t)lane + c.max_batch - 1) : lane;
                    for (int it = 0; it < 5; ++it) {
                        const uint32_t mid = lo < hi ? (lo + hi + 1) >> 1 : lo;
                        const uint64_t v = __shfl_sync(0xffffffffu, pci, mid);
                        if (lo < hi) { if (v <= lim) lo = mid; else hi = mid - 1; }
                    }
                    const uint64_t hi64 = __shfl_sync(0xffffffffu, (uint64_t)(pfi >> 64), lo);
                    const uint64_t lo64 = __shfl_sync(0xffffffffu, (uint64_t)pfi, lo);
                    u128 best = (((u128)hi64 << 64) | lo64) - pfe;
                    uint32_t bi = inw ? lane : 0xFFFFFFFFu, bj = lo;
                    for (int o = 16; o > 0; o >>= 1) {                  // first maximum (strict >)
                        const u128 ob = shfl_xor_u128(best, o);
                        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
                        if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
                    }
                    if (inw) bBv[lane] = row;                           // window order, the batch = [bi, bj]
                    const uint64_t tot = __shfl_sync(0xffffffffu, pci, bj) - __shfl_sync(0xffffffffu, pce, bi);
                    if (lane == 0) {
                        s_bstar = bstar; s_bp = bp; s_thr = thr; s_thr_img = thr_img;
                        s_tguess = (uint64_t)__double_as_longlong(__dmul_rn(thr, kReplayMargin));
                        s_m = np; s_ncd = ncd_w; s_nsel = bj - bi + 1; s_tot = (uint32_t)tot; s_bi[0] = bi;
                    }
                }
                __syncthreads();
                RSTAMP(7);
            } else {
            // ---- (a7) order pending by (key desc, id asc).  Attempt 0 sorts only the speculative
            // set S = {key >= t} (t = kReplayMargin x the previous step's cutoff): S is a prefix of the
            // priority order, so its budget walk is exact when it stops inside S (or S holds every
            // pending row), and Cd lies in S when thr >= t.  Otherwise attempt 1
            // sorts every pending row.  Both give the same B*, bp, thr and Cd.
            for (uint32_t attempt = 0; attempt < 2; ++attempt) {
                const uint64_t t = attempt == 0 ? s_tguess : 0ull;
                {
                    uint32_t cntl = 0;
                    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                        const uint32_t r = S.live[i];
                        cntl += S.img[r] != kNone && S.img[r] >= t;
                    }
                    uint64_t tot;
                    uint32_t pos = (uint32_t)block_exclusive_scan_u64(cntl, s_scan, &tot);
                    const uint32_t m = (uint32_t)tot;
                    if (attempt == 0 && (m == 0 || m > 512u)) {     // not worth it / too big: full sort
                        if (threadIdx.x == 0) s_m = 0;
                        __syncthreads();
                        continue;
                    }
                    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                        const uint32_t r = S.live[i];
                        if (S.img[r] != kNone && S.img[r] >= t) { bA[pos] = make_ck(S.img[r], r); bAv[pos] = r; ++pos; }
                    }
                    uint32_t m2 = 1;
                    while (m2 < m) m2 <<= 1;
                    for (uint32_t i = m + threadIdx.x; i < m2; i += blockDim.x) { bA[i] = ~(u128)0; bAv[i] = 0; }
                    if (threadIdx.x == 0) s_m = m;
                    __syncthreads();
                    RSTAMP(4);
                    block_sort_small<u128>(bA, bAv, m, m2);
                    RSTAMP(14);
                }
                const uint32_t m = s_m;
                // B* = longest prefix within tau and B_max (monotone predicate -> count)
                uint64_t carry = 0;
                uint32_t fits = 0;
                for (uint32_t base = 0; base < m; base += blockDim.x) {
                    const uint32_t i = base + threadIdx.x;
                    const uint64_t cv = i < m ? S.cost[bAv[i]] : 0;
                    uint64_t tot;
                    const uint64_t ex = block_exclusive_scan_u64(cv, s_scan, &tot);
                    const bool f = i < m && (uint64_t)i + 1 <= c.max_batch && carry + ex + cv <= c.token_budget;
                    fits += __syncthreads_count(f);
                    carry += tot;
                }
                if (threadIdx.x == 0) {
                    s_bstar = fits;
                    const double bp = __longlong_as_double((long long)ck_img(bA[fits - 1]));
                    s_bp = bp;
                    s_thr = __dmul_rn(s_p, bp);
                    s_thr_img = (uint64_t)__double_as_longlong(s_thr);
                    // speculative attempt: exact iff the walk stopped inside S (or S = all pending)
                    // and Cd = {key >= thr} lies in S
                    s_spec_ok = attempt == 1 || m == np || (fits < m && s_thr_img >= t);
#ifdef JIT_REPLAY_STAMPS
                    if (rep == kStampRep) { s_ph[10] += attempt; s_ph[11] += np; s_ph[12] += m; s_ph[13] += (attempt == 0 && s_m == 0); }
#endif
                }
                __syncthreads();
                RSTAMP(15);
                if (s_spec_ok) break;
            }
#ifdef JIT_REPLAY_DUMP_STEP
            if (threadIdx.x == 0 && s_steps == JIT_REPLAY_DUMP_STEP) {
                printf("dump step %u m %u np %u bstar %u spec_ok %u\n", s_steps, s_m, np, s_bstar, s_spec_ok);
                for (uint32_t r = 0; r < n; ++r)
                    if (S.img[r] != kNone)
                        printf("row %u key %.10f cost %u st %u w %u pre %u gen %u L %u\n", r,
                               __longlong_as_double((long long)S.img[r]), S.cost[r], m_state(S.meta[r]), S.aux[r] >> 16,
                               S.pre[r], S.gen[r], L_in[r]);
            }
            __syncthreads();
            RSTAMP(4);
#endif
            if (threadIdx.x == 0) s_tguess = (uint64_t)__double_as_longlong(__dmul_rn(s_thr, kReplayMargin));
            const uint32_t np_sorted = s_m;   // rows in the sorted prefix array bA (Cd is a prefix of it)
            // ---- (a8) Cd = prefix of the key-ordered list with key >= thr
            {
                uint32_t ncd = 0;
                for (uint32_t base = 0; base < np_sorted; base += blockDim.x) {
                    const uint32_t i = base + threadIdx.x;
                    ncd += __syncthreads_count(i < np_sorted && ck_img(bA[i]) >= s_thr_img);
                }
                if (threadIdx.x == 0) s_ncd = ncd;
                __syncthreads();
            }
            const uint32_t ncd = s_ncd;
            uint32_t m2 = 1;
            while (m2 < ncd) m2 <<= 1;
            for (uint32_t i = threadIdx.x; i < m2; i += blockDim.x) {
                if (i < ncd) {
                    const uint32_t r = bAv[i];
                    const uint64_t len = c.len_key ? (uint64_t)L_in[r] + S.gen[r] : (uint64_t)L_in[r];
                    bB[i] = (len << 32) | r; bBv[i] = r;
                } else { bB[i] = ~0ull; bBv[i] = 0; }
            }
            __syncthreads();
            // ---- (a9) sort Cd by (len, id); windows within tau / B_max; first argmax
            block_sort_small<uint64_t>(bB, bBv, ncd, m2);
            unsigned long long* pc = in_smem ? reinterpret_cast<unsigned long long*>(sA) : S.gpc;   // reuse region A
            u128* pf = in_smem ? reinterpret_cast<u128*>(sbuf + ((8 * (SR + 1) + 15) & ~15u)) : S.gpf;
            {
                uint64_t carry_c = 0; u128 carry_f = 0;
                for (uint32_t base = 0; base < ncd; base += blockDim.x) {
                    const uint32_t i = base + threadIdx.x;
                    uint64_t cv = 0; u128 fv = 0;
                    if (i < ncd) {
                        const uint32_t r = bBv[i];
                        cv = S.cost[r];
                        fv = (u128)fixed_point(__longlong_as_double((long long)S.img[r]));
                    }
                    uint64_t tc, ec; u128 tf, ef;
                    block_exclusive_scan_pair(cv, fv, s_scan, s_scan128, ec, ef, tc, tf);
                    if (i < ncd) { pc[i] = carry_c + ec; pf[i] = carry_f + ef; }
                    carry_c += tc; carry_f += tf;
                }
                if (threadIdx.x == 0) { pc[ncd] = carry_c; pf[ncd] = carry_f; }
                __syncthreads();
                RSTAMP(5);
            }
            {
                u128 best = 0; uint32_t bi = 0xFFFFFFFFu, bj = 0;
                for (uint32_t i = threadIdx.x; i < ncd; i += blockDim.x) {
                    const uint64_t lim = (uint64_t)pc[i] + c.token_budget;
                    uint32_t lo = i, hi = (uint32_t)min((uint64_t)ncd - 1, (uint64_t)i + c.max_batch - 1);
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi + 1) >> 1;
                        if (pc[mid + 1] <= lim) lo = mid; else hi = mid - 1;
                    }
                    const u128 sc = pf[lo + 1] - pf[i];
                    if (bi == 0xFFFFFFFFu || sc > best) { best = sc; bi = i; bj = lo; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const u128 ob = shfl_xor_u128(best, o);
                    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
                }
                if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; s_bj[wid] = bj; }
                __syncthreads();
                RSTAMP(6);
                if (wid == 0) {
                    const uint32_t nw = blockDim.x >> 5;
                    best = lane < nw ? s_best[lane] : (u128)0; bi = lane < nw ? s_bi[lane] : 0xFFFFFFFFu; bj = lane < nw ? s_bj[lane] : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const u128 ob = shfl_xor_u128(best, o);
                        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
                        if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
                    }
                    if (lane == 0) {
                        s_nsel = bj - bi + 1;
                        s_tot = (uint32_t)(pc[bj + 1] - pc[bi]);
                        s_bi[0] = bi;
                    }
                }
                __syncthreads();
                RSTAMP(7);
            }
            }
            uint32_t nsel = s_nsel;
            const uint32_t* selv = bBv + s_bi[0];          // the batch rows: GMAX's window ...
            if (c.preempt) {
                // ---- NEXT-1 preemption gate (reading A46; App. D.2):
                // P = pending & Running, I = window \ P, both in (key desc, id asc); a single thread
                // walks them (|P| + |I| <= 2 B_max), marks in S.late bits 1 (in window), 2 (in the
                // batch), 3 (evicted); then the batch is put in window order (len asc, id asc).
                const bool frame_open = s_steps % c.frame == 0;
                for (uint32_t k = threadIdx.x; k < nsel; k += blockDim.x) S.late[selv[k]] |= 2u;
                __syncthreads();
                uint32_t cnt = 0;
                for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                    const uint32_t r = S.live[i];
                    const bool run = S.img[r] != kNone && m_state(S.meta[r]) == kRunning;
                    cnt += run || ((S.late[r] & 2u) && !run);
                }
                uint64_t tot;
                uint32_t pos = (uint32_t)block_exclusive_scan_u64(cnt, s_scan, &tot);
                const uint32_t ng = (uint32_t)tot;
                for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                    const uint32_t r = S.live[i];
                    const bool run = S.img[r] != kNone && m_state(S.meta[r]) == kRunning;
                    if (run || (S.late[r] & 2u)) {
                        bA[pos] = ((u128)(run ? 0u : 1u) << 96) | make_ck(S.img[r], r);
                        bAv[pos] = r; ++pos;
                    }
                }
                uint32_t g2 = 1;
                while (g2 < ng) g2 <<= 1;
                for (uint32_t i = ng + threadIdx.x; i < g2; i += blockDim.x) { bA[i] = ~(u128)0; bAv[i] = 0; }
                __syncthreads();
                block_sort<u128>(bA, bAv, g2);
                if (threadIdx.x == 0) {
                    uint64_t budget = c.token_budget;
                    uint32_t slots = c.max_batch, np_run = 0;
                    while (np_run < ng && (uint32_t)(bA[np_run] >> 96) == 0u) ++np_run;
                    for (uint32_t k = 0; k < np_run; ++k) {          // 1. running requests keep their slot
                        const uint32_t r = bAv[k], cs = S.cost[r];
                        if (slots >= 1 && cs <= budget) { S.late[r] |= 4u; --slots; budget -= cs; }
                        else S.late[r] |= 8u;                        // does not fit: evicted
                    }
                    const double fs = __ddiv_rn(__ull2double_rn((uint64_t)c.frame * (uint64_t)v), 1e9);
                    uint32_t o = np_run;
                    for (uint32_t k = np_run; k < ng; ++k) {         // 2. newcomers
                        const uint32_t r = bAv[k], cs = S.cost[r];
                        if (slots >= 1 && cs <= budget) { S.late[r] |= 4u; --slots; budget -= cs; continue; }
                        if (!frame_open) continue;
                        while (o > 0 && !((S.late[bAv[o - 1]] & 4u) && !(S.late[bAv[o - 1]] & 2u))) --o;
                        if (o == 0) continue;
                        const uint32_t q = bAv[o - 1];
                        const uint64_t kv = (uint64_t)S.pre[q] + S.gen[q];
                        const int64_t st = (int64_t)((u128)kv * 1000000000u / c.io_bw);
                        const double loss = __ddiv_rn(__ll2double_rn(st), __ll2double_rn(v));
                        const double ki = __longlong_as_double((long long)S.img[r]);
                        const double kq = __longlong_as_double((long long)S.img[q]);
                        const double gain = __dmul_rn(__dsub_rn(ki, kq), fs);
                        if (cs <= budget + S.cost[q] && ki > __dmul_rn(kq, c.onepd) && gain > loss) {
                            S.late[q] = (S.late[q] & ~4u) | 8u;
                            S.late[r] |= 4u;
                            budget = budget + S.cost[q] - cs;
                            --o;
                        }
                    }
                    s_npre = 0; s_stall = 0;
                }
                __syncthreads();
                // the batch in window order; evicted rows become Preempted (their KV is swapped out)
                uint32_t cf = 0, myev = 0, mytok = 0;
                unsigned long long mystall = 0;
                for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                    const uint32_t r = S.live[i];
                    const uint32_t lt = S.late[r];
                    cf += (lt >> 2) & 1u;
                    if (lt & 4u) mytok += S.cost[r];
                    if (lt & 8u) {
                        ++myev;
                        mystall += (unsigned long long)((u128)((uint64_t)S.pre[r] + S.gen[r]) * 1000000000u / c.io_bw);
                        S.meta[r] = m_with_state(S.meta[r], kPreempted);
                    }
                }
                pos = (uint32_t)block_exclusive_scan_u64(cf, s_scan, &tot);
                const uint32_t nf = (uint32_t)tot;
                for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                    const uint32_t r = S.live[i];
                    if (S.late[r] & 4u) {
                        const uint64_t len = c.len_key ? (uint64_t)L_in[r] + S.gen[r] : (uint64_t)L_in[r];
                        bB[pos] = (len << 32) | r; bBv[pos] = r; ++pos;
                    }
                }
                uint32_t f2 = 1;
                while (f2 < nf) f2 <<= 1;
                for (uint32_t i = nf + threadIdx.x; i < f2; i += blockDim.x) { bB[i] = ~0ull; bBv[i] = 0; }
                myev = warp_sum(myev); mytok = warp_sum(mytok);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) mystall += __shfl_xor_sync(0xffffffffu, mystall, off);
                if (lane == 0) { atomicAdd(&s_npre, myev); atomicAdd(&s_stall, mystall); }
                __syncthreads();
                block_sort<uint64_t>(bB, bBv, f2);
                for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) S.late[S.live[i]] &= 1u;   // marks off
                if (threadIdx.x == 0) { s_nsel = nf; s_tot = 0; }
                __syncthreads();
                if (lane == 0) atomicAdd(&s_tot, mytok);
                nsel = nf;
                selv = bBv;                                  // ... or the gated batch
                __syncthreads();
            }
            // batch rows, bookkeeping (ever_scheduled, Running), max context; a selected row keeps
            // its steps_waited and is unmarked as pending (img) for the +1 of the others below
            int64_t myctx = 0;
            for (uint32_t k = threadIdx.x; k < nsel; k += blockDim.x) {
                const uint32_t r = selv[k];
                S.batch[k] = r;
                uint32_t m = S.meta[r] | (kEver << 12);
                if (m_state(m) == kQueued || m_state(m) == kPreempted) m = m_with_state(m, kRunning);
                S.meta[r] = m;
                if (tsk[r] != kNoTask) S.tever[tsk[r]] = 1;
                const int64_t ctx = S.pre[r] < L_in[r] ? (int64_t)S.pre[r] + S.cost[r] : (int64_t)L_in[r] + S.gen[r];
                myctx = ctx > myctx ? ctx : myctx;
            }
            if (threadIdx.x == 0) s_maxctx = 0;
            __syncthreads();
            atomicMax((unsigned long long*)&s_maxctx, (unsigned long long)myctx);
            for (uint32_t k = threadIdx.x; k < nsel; k += blockDim.x) S.img[S.batch[k]] = kNone;
            __syncthreads();
            RSTAMP(8);
            // steps_waited + 1 (saturating) for every pending request left out (A12)
            for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
                const uint32_t r = S.live[i];
                if (S.img[r] != kNone && (S.aux[r] >> 16) < 0xFFFFu) S.aux[r] += 1u << 16;
            }
            // ---- (a10) iteration latency and time advance
            // + the KV swap stall of the requests the gate evicted (NEXT-1, A46)
            const int64_t stall = c.preempt ? (int64_t)s_stall : 0;
            const int64_t latency = A.c0 + A.c_att * s_maxctx + A.c_lin * (int64_t)nsel + stall;
            const int64_t tnow = now + latency;
            if (threadIdx.x == 0) {
                s_now = tnow;
                s_steps += 1;
                s_tok += s_tot;
                if (c.preempt) n_preempted_total += s_npre;
                if (A.log && s_steps <= A.log_steps) {
                    uint64_t h = 1469598103934665603ull;
                    for (uint32_t k = 0; k < nsel; ++k) h = fnv1a_u32(h, S.batch[k]);
                    RLog L;
                    L.now_ns = tnow; L.n_selected = nsel; L.total_tokens = s_tot; L.n_candidates = s_ncd;
                    L.b_star = s_bstar; L.bp = s_bp; L.ids_hash = h; L.v_token_ns = v;
                    L.n_preempted = c.preempt ? s_npre : 0u; L.p_num = s_pnum; L.stall_ns = stall;
                    A.log[(uint64_t)rep * A.log_steps + s_steps - 1] = L;
                }
                // v_token ring (Delta = frame_steps latencies)
                if (s_ring_n < c.frame) { S.ring[s_ring_n] = latency; s_ring_n += 1; s_ring_sum += latency; }
                else { s_ring_sum += latency - S.ring[s_ring_pos]; S.ring[s_ring_pos] = latency; s_ring_pos = (s_ring_pos + 1) % c.frame; }
            }
            __syncthreads();
            // progress of the executed batch, token timestamps = iteration end
            for (uint32_t k = threadIdx.x; k < nsel; k += blockDim.x) {
                const uint32_t r = S.batch[k];
                const Group& G = sg[grp[r]];
                bool emit = false;
                if (S.pre[r] < L_in[r]) {
                    S.pre[r] += S.cost[r];
                    if (S.pre[r] == L_in[r]) emit = true;            // prefill end emits token 0
                } else emit = true;
                if (!emit) continue;
                const uint32_t tok = S.gen[r];
                if (G.type == kLAT) {                                  // §3
                    if (tnow <= S.arr[r] + G.ttft_ns + (int64_t)tok * G.tbt_ns) atomicAdd(&s_good, (unsigned long long)G.w_out);
                    else S.late[r] = 1;
                }
                S.gen[r] = tok + 1;
                if (tok + 1 < L_out[r]) continue;
                S.meta[r] = m_with_state(S.meta[r], kDone);
                atomicAdd(&s_done, 1u);
                if (G.type == kDDL) {                                  // §3
                    if (tnow <= S.arr[r] + G.e2el_ns) {
                        atomicAdd(&s_good, (unsigned long long)(ovr[r] ? (uint64_t)ovr[r] : call_R(G, L_in[r], L_out[r])));
                        atomicAdd(&s_reqg, 1u);
                    }
                } else if (G.type == kLAT) {
                    if (!S.late[r]) atomicAdd(&s_reqg, 1u);
                } else if (G.type == kCMP) {                           // stage barrier
                    const uint32_t t = tsk[r];
                    atomicAdd(&S.gdone[t], (unsigned long long)call_R(G, L_in[r], L_out[r]));
                    if (atomicSub(&S.left[t], 1u) == 1u) {
                        S.cur[t] += 1; S.cb[t] = 0; S.ce[t] = 0; S.timer[t] = tnow;
                        atomicMin(&s_tmin, (long long)tnow);
                    }
                }
            }
            __syncthreads();
            RSTAMP(9);
            // NEXT-2 online p (A48): at the end of a window its token goodput scores its arm; the
            // next arm: an untried one in grid order, else explore (prob eps) or the best mean
            if (A.p_adapt && threadIdx.x == 0 && s_steps % (A.window_frames * c.frame) == 0) {
                const uint32_t a0 = s_arm;
                s_gsum[a0] += s_good - s_gstart; s_gcnt[a0] += 1;
                s_gstart = s_good;
                s_window += 1;
                uint32_t nxt = 4;
                for (uint32_t a = 0; a < 4 && nxt == 4; ++a) if (s_gcnt[a] == 0) nxt = a;
                if (nxt == 4) {
                    const uint64_t u = splitmix64_at(A.seed + s_window);
                    if (u % A.eps_den < A.eps_num) nxt = (uint32_t)((u >> 32) % 4u);
                    else {
                        nxt = 0;
                        for (uint32_t a = 1; a < 4; ++a)
                            if ((u128)s_gsum[a] * s_gcnt[nxt] > (u128)s_gsum[nxt] * s_gcnt[a]) nxt = a;
                    }
                }
                s_arm = nxt; s_pnum = kPGrid[nxt];
                s_p = __ddiv_rn((double)kPGrid[nxt], 100.0);
            }
            __syncthreads();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            RResult R;
            R.token_goodput = s_good; R.tokens_processed = s_tok; R.sim_end_ns = s_now;
            R.request_goodput = s_reqg; R.n_done = s_done; R.n_dropped = s_drop; R.steps = s_steps;
            R.n_tasks_done = s_tdone; R.n_tasks_dropped = s_tdrop; R.error = s_err; R.n_preempted = n_preempted_total;
            A.out[rep] = R;
#ifdef JIT_REPLAY_STAMPS
            if (rep == kStampRep) {
                printf("replay %u: %u steps, ns/step:", kStampRep, s_steps);
                for (int i = 1; i < 20; ++i) printf(" p%d=%llu", i, s_ph[i] / (s_steps ? s_steps : 1));
                printf(" full_sorts=%llu", s_ph[10]);
                printf("\n");
            }
#endif
        }
        __syncthreads();
    }
}

// dynamic shared memory of k_replay: groups, sort buffers, (the replay state)
inline uint32_t replay_smem_bytes(uint32_t n_groups, uint64_t core, uint32_t sort_rows = kReplaySmemRows) {
    return (uint32_t)(replay_groups_bytes(n_groups) + 36 * sort_rows + 64 + core);
}

}  // namespace jit
