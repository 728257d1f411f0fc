// stream.cuh -- k_score: the streaming pass of the GMAX step over every request of the pool,
// rows (a1)-(a6) of SURVEY §8(a).
//
//   * persistent CTAs; each warp walks work items (i, i + W, ...) of at most kItemRows hot rows
//     through its own ring of shared-memory slots: one elected lane streams an item's 32-byte
//     rows (and a compound item's task ids) in with ONE bulk asynchronous copy (the 1-D TMA path,
//     mbarrier completion) kStagesW items ahead, so HBM reads overlap the scoring of earlier items
//     without holding registers;
//   * standalone rows: (a1) admission / pending, (a2) length bound (cached per R-token epoch),
//     (a3) t_rem, (a5) goodput G' = G + delta * floor(waited / Delta);
//   * compound items hold whole tasks: the warp sums (len_rem, call goodput) per task in shared
//     memory (a4), forms each task's goodput and t_gen + eps once, then keys every call;
//   * everything that is rare in the steady state -- a stale cached bound (two binary searches
//     on the L2-resident table row), a drop, a row entering or leaving the pending set
//     (steps_waited stamp, pool.cuh), an overridden goodput -- runs behind one warp vote per row;
//   * the key fl(G' 1e9 / (t_gen + eps)) is divided out only for rows that can reach the
//     speculative threshold t (a conservative fp64 pre-test, exact: DESIGN.md §7); rows with
//     key >= t join the speculative set, which k_spec resolves;
//   * nothing is written per row in the steady state.  kMat (debug handles, the exact path's
//     re-score) also stores every row's key image and token cost.
#pragma once
#include "pool.cuh"
#include "select.cuh"

namespace jit {

#ifndef JIT_SCORE_THREADS
#define JIT_SCORE_THREADS 128
#endif
#ifndef JIT_SCORE_MINB
#define JIT_SCORE_MINB 4
#endif
#ifndef JIT_STAGES_W
#define JIT_STAGES_W 2
#endif
constexpr uint32_t kStagesW = JIT_STAGES_W;     // shared-memory item slots per warp
constexpr uint32_t kScoreThreads = JIT_SCORE_THREADS;
constexpr uint32_t kScoreWarps = kScoreThreads / 32;
#ifndef JIT_ROWS_PER_LANE
#define JIT_ROWS_PER_LANE 4
#endif
constexpr uint32_t kR = JIT_ROWS_PER_LANE;      // hot rows per lane per item chunk
constexpr uint32_t kItemRows = 32 * kR;         // rows per item (chunk)
constexpr uint32_t kItemTasks = 32;             // tasks per compound item (one per lane; <= 32)
#ifndef JIT_STD_ROWS_PER_LANE
#define JIT_STD_ROWS_PER_LANE 2
#endif
constexpr uint32_t kRs = JIT_STD_ROWS_PER_LANE;  // standalone rows per lane per chunk (direct loads)
static_assert(kItemTasks <= 32, "a compound item's task sums live in one lane each");

// per-group constants of the pass, with `now` folded in (per launch):
//   t_rem = arr + bn + (Lhat - 1) * tok       bn = base - now (LAT: TTFT, DDL: E2EL, BE: default)
//   G     = w_in * L_i + w_out * Lhat         (DDL: w_in, w_out; LAT: 0, w_out; BE: 0, 0)
struct GroupNow {
    int64_t bn;
    uint32_t tok, w_in, w_out, pad;
};

struct Part {
    uint32_t pend, drop, ref, err;
    uint64_t mn;           // kMat: smallest key image
};

// Rows whose key image reaches the speculative threshold t join the speculative set (warp ballot,
// one atomic per warp).  The entry carries everything the resolve needs, as this pass left it.
__device__ __forceinline__ void spec_add(const Scratch& S, const Pool& P, const Cfg& c, bool take, uint64_t img,
                                         uint32_t row, const HotRow& q) {
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(S.spec_cnt, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) {
        const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
        if (slot < kSpecCap) {
            S.spec_img[slot] = img; S.spec_id[slot] = __ldg(P.id + row); S.spec_row[slot] = row;
            S.spec_cost[slot] = token_cost(q.len_in, q.pre, c.chunk);
            S.spec_len[slot] = c.len_key ? q.len_in + q.gen : q.len_in;
            S.spec_meta[slot] = q.meta; S.spec_aux[slot] = q.since;
        }
    }
}

// the rare work of one row (only lanes whose row needs it): regime of the steps_waited stamp --
// pending rows carry a stamp, the others a frozen count (pool.cuh) -- written with the meta only
// when it changes or the row is dropped; a stale cached bound re-derived from the table (a2).
// Scalar arguments and a returned triple: a reference would push the caller's rows to the stack.
struct Rare {
    uint32_t meta, since, lrow;
};
__device__ __noinline__ Rare row_rare(const uint32_t* edges, const uint32_t* cum, uint32_t n_bins, uint32_t l_max,
                                      uint32_t unit, uint32_t R, uint32_t qn, uint32_t qd, HotRow* rp, uint32_t meta,
                                      uint32_t since, uint32_t lrow, bool pend, bool drop, bool stale, uint32_t ep,
                                      uint32_t sc, const ForestDev* forest, uint32_t len_in) {
    const bool stamped = (meta >> 12) & kStamped;
    if (drop || pend != stamped) {
        if (pend) {                                     // became pending: count from here on
            since = sc - since;
            meta |= kStamped << 12;
        } else if (stamped) {                           // left the pending set: freeze the count
            since = waited_of(meta, since, sc);
            meta &= ~(kStamped << 12);
        }
        if (drop) meta = m_with_state(meta, kDropped);
    }
    if (stale) {                                        // refreshed every R tokens
        const uint32_t lh = forest ? qrf_bound(forest, len_in, l_row(lrow), ep * R, m_group(meta), ep * R, qn, qd, l_max)
                                   : cond_quantile_v(edges, cum, n_bins, l_max, unit, l_row(lrow), ep * R, qn, qd);
        lrow = l_row(lrow) | (lh << 16);
        rp->lrow = lrow;
        meta = (meta & 0xFFFFu) | (ep < 65535u ? (ep + 1u) << 16 : 0u);   // epoch field = floor(g/R) + 1
    }
    *reinterpret_cast<uint2*>(&rp->meta) = make_uint2(meta, since);
    return Rare{meta, since, lrow};
}
__device__ __forceinline__ void rare_row(const Table& T, const Cfg& c, HotRow* rp, HotRow& q, bool pend, bool drop,
                                         bool stale, uint32_t ep, uint32_t sc, uint32_t& ref) {
    const Rare o = row_rare(T.edges, T.cum, T.n_bins, T.l_max, T.unit, c.R, c.qn, c.qd, rp, q.meta, q.since, q.lrow,
                            pend, drop, stale, ep, sc, T.forest, q.len_in);
    q.meta = o.meta; q.since = o.since; q.lrow = o.lrow;
    ref += stale;
}

// The pre-test in fp32: A_f = fl(G' 1e9) (G' < 2^24 and 1e9 are exact fp32 integers, one rounding),
// B_f = fl(len_rem v_f + eps_f) (v_f, eps_f rounded), t_lo_f = t (1 - 2^-16) rounded toward zero.
// If A_f < fl(t_lo_f B_f) then A/B < t (1 - 2^-16)(1 + 2^-22) / (1 - 2^-24) < t (1 - 2^-17), so
// fl(A/B) < t: the row cannot reach the speculative set.
__device__ __forceinline__ bool below_t(uint32_t Gp, uint32_t len_rem, float v_f, float eps_f, float t_lo_f) {
    const float Af = __fmul_rn(__uint2float_rn(Gp), 1e9f);
    const float Bf = __fmaf_rn(__uint2float_rn(len_rem), v_f, eps_f);
    return Af < __fmul_rn(t_lo_f, Bf);
}

// ---- per-warp ring of item slots fed by bulk asynchronous copies (PTX, sm_90+)
struct WarpSlot {
    HotRow rows[kItemRows];
    uint32_t task[kItemRows + 4];       // task ids from the 16-byte aligned row r0 & ~3
    TaskInfo tinfo[kItemTasks];         // compound items: the tasks' constants
    uint32_t tever[kItemTasks + 4];     // ... their ever-scheduled flags, from task t0 & ~3
    uint32_t off[kItemTasks + 8];       // ... and their CSR row offsets, from task t0 & ~3
};
static_assert(sizeof(WarpSlot) % 16 == 0, "slot alignment");
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// The pool streams through L2 once per step: its bulk reads carry an evict-first policy so that
// what is reused every step (code, tables, partials, the speculative set) keeps its L2 lines
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol) : "memory");
}
// Bounded wait: a phase that never completes (a bulk copy that faulted, a protocol bug) traps
// after ~2^26 probes instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0, tries = 0;
    while (true) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
        if (ok) return;
        if (++tries == (1u << 26)) __trap();
    }
}
// lane 0: start streaming item `it` into slot `sl` (completes on bar).  A big compound item
// (more rows than a slot) is read from global memory instead: its phase completes at once.
__device__ __forceinline__ void issue_item(const Pool& P, const Item& it, WarpSlot* sl, uint64_t* bar, uint64_t pol) {
    const uint32_t nr = it.r1 - it.r0;
    if (nr > kItemRows || nr == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
        return;
    }
    const bool cmp = it.t1 != it.t0;
    const uint32_t tb = it.r0 & ~3u, eb = it.t0 & ~3u, nt = it.t1 - it.t0;
    const uint32_t tbytes = cmp ? ((it.r1 - tb) * 4u + 15u) & ~15u : 0u;   // the per-row / per-task
    const uint32_t ebytes = cmp ? ((it.t1 - eb) * 4u + 15u) & ~15u : 0u;   // arrays are padded
    const uint32_t obytes = cmp ? ((it.t1 + 1 - eb) * 4u + 15u) & ~15u : 0u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(nr * 32u + tbytes + (cmp ? nt * (uint32_t)sizeof(TaskInfo) + ebytes + obytes : 0u)) : "memory");
    bulk_g2s(sl->rows, P.rows + it.r0, nr * 32u, bar, pol);
    if (cmp) {
        bulk_g2s(sl->task, P.task + tb, tbytes, bar, pol);
        bulk_g2s(sl->tinfo, P.tinfo + it.t0, nt * (uint32_t)sizeof(TaskInfo), bar, pol);
        bulk_g2s(sl->tever, P.tever + eb, ebytes, bar, pol);
        bulk_g2s(sl->off, P.call_off + eb, obytes, bar, pol);
    }
}

__device__ __forceinline__ HotRow ld_row_s(const HotRow* p) {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0];
    const uint4 b = reinterpret_cast<const uint4*>(p)[1];
    HotRow r;
    r.arr = (int64_t)(((uint64_t)a.y << 32) | a.x);
    r.len_in = a.z; r.gen = a.w; r.pre = b.x; r.lrow = b.y; r.meta = b.z; r.since = b.w;
    return r;
}

// the rows with key >= t join the speculative set (one ballot per row slab; rare)
template <uint32_t KR, typename RowAt>
__device__ __forceinline__ void spec_rows(const Scratch& S, const Pool& P, const Cfg& c, uint32_t mem_m,
                                          const uint64_t* img, uint32_t base, RowAt row_at) {
    const uint32_t lane = threadIdx.x & 31;
    if (!__any_sync(0xffffffffu, mem_m)) return;
#pragma unroll
    for (uint32_t k = 0; k < KR; ++k) {
        const bool take = (mem_m >> k) & 1u;
        const uint32_t r = base + 32 * k + lane;
        spec_add(S, P, c, take, img[k], r, take ? row_at(k, r) : HotRow{0, 0, 0, 0, 0, 0, 0});
    }
}

// 256-bit load of a hot row straight from global memory (sm_100: LDG.E.256), read once per
// pass (no L1 allocation, evict-first in L2: the pool streams through L2 once per step)
__device__ __forceinline__ HotRow ld_row_g(const HotRow* p) {
    uint32_t a0, a1, a2, a3, a4, a5, a6, a7;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6), "=r"(a7) : "l"(p));
    HotRow r;
    r.arr = (int64_t)(((uint64_t)a1 << 32) | a0);
    r.len_in = a2; r.gen = a3; r.pre = a4; r.lrow = a5; r.meta = a6; r.since = a7;
    return r;
}

// ---- standalone rows r0 + 32 k + lane (k < KR, valid while 32 k + lane < nr), already loaded in
// q; KR rows per lane whose arithmetic chains interleave (warp votes only per chunk: rare work,
// divisions, set members)
template <bool kMat, bool kDebug, bool kAppB, uint32_t KR>
__device__ __forceinline__ void std_core(const Pool& P, const Table& T, const GroupNow* sg, const Cfg& c,
                                         const Scratch& S, int64_t now, double v_d, int64_t v, uint32_t sc,
                                         uint64_t t_img, float t_lo_f, uint32_t r0, uint32_t nr, HotRow (&q)[KR],
                                         Part& A) {
    const uint32_t lane = threadIdx.x & 31;
    const double eps_d = (double)c.eps;
    const float v_f = (float)v, eps_f = (float)c.eps;
    const int64_t drop_before = now - c.waiting;           // now - arr > waiting <=> arr < now - waiting
    const bool blend = c.fair_num != 0;                    // NEXT-2: no pre-test, exact keys blended
    uint32_t pend_m = 0, rare_m = 0, drop_m = 0;
#pragma unroll
    for (uint32_t k = 0; k < KR; ++k) {                    // (a1) admission / pending; what is rare
        const uint32_t o = 32 * k + lane;
        const bool valid = o < nr;
        const HotRow& x = q[k];
        const uint32_t st = m_state(x.meta), fl = m_flags(x.meta);
        const bool arrived = valid && x.arr <= now;
        const bool drop = arrived && st == kQueued && !(fl & (kEver | kCompound)) && x.arr < drop_before;
        const bool pend = arrived && !drop && st <= kPreempted;
        const uint32_t ep = fastdiv(x.gen, c.R, c.R_m, c.R_l);
        const bool stale = pend && m_epoch(x.meta) != ep + 1u;
        const bool regime = drop || (valid && pend != (bool)(fl & kStamped));
        pend_m |= (uint32_t)pend << k;
        drop_m |= (uint32_t)drop << k;
        rare_m |= (uint32_t)(regime || stale) << k;
    }
    A.drop += __popc(drop_m);
    if (__any_sync(0xffffffffu, rare_m)) {                 // stamp regime, stale bound (rare)
#pragma unroll
        for (uint32_t k = 0; k < KR; ++k) {
            if (!((rare_m >> k) & 1u)) continue;
            const bool pend = (pend_m >> k) & 1u;
            const uint32_t ep = fastdiv(q[k].gen, c.R, c.R_m, c.R_l);
            rare_row(T, c, P.rows + r0 + 32 * k + lane, q[k], pend, (drop_m >> k) & 1u,
                     pend && m_epoch(q[k].meta) != ep + 1u, ep, sc, A.ref);
        }
    }
    // (a3) t_rem, (a5) goodput (A9-A11, A22), starvation inflation (A12), the pre-test
    uint32_t Gk32[KR], Lr[KR];
    uint32_t div_m = 0;
#pragma unroll
    for (uint32_t k = 0; k < KR; ++k) {
        const HotRow& x = q[k];
        const bool pend = (pend_m >> k) & 1u;
        const uint32_t Lh = max(l_hat(x.lrow), x.gen + 1);
        const uint32_t len_rem = Lh - x.gen;
        const GroupNow G = sg[m_group(x.meta)];
        const int64_t trem = x.arr + G.bn + (int64_t)((uint64_t)(Lh - 1) * G.tok);
        uint64_t Gk = (uint64_t)G.w_in * x.len_in + (uint64_t)G.w_out * Lh;
        if (m_flags(x.meta) & kOverride) Gk = __ldg(P.ovr + r0 + 32 * k + lane);   // App. D sets R(k)
        if (trem <= 0) Gk = 0;
        if (kAppB && (uint64_t)len_rem * (uint64_t)v > (uint64_t)(trem > 0 ? trem : 0)) Gk = 0;
        const uint32_t waited = min(sc - x.since, 0xFFFFu);
        const uint64_t Gp = Gk + (uint64_t)c.delta * fastdiv(waited, c.frame, c.F_m, c.F_l);
        if (pend && Gp >= kTwo53 / 1000000000ull) A.err = 1;   // G' * 1e9 must stay an exact integer
        Gk32[k] = (uint32_t)Gp; Lr[k] = len_rem;
        div_m |= (uint32_t)(pend && (kMat || blend || !below_t((uint32_t)Gp, len_rem, v_f, eps_f, t_lo_f))) << k;
        if (kDebug && 32 * k + lane < nr) {
            const uint32_t r = r0 + 32 * k + lane;
            P.dbg_rate[r] = pend ? make_rate(len_rem, trem) : 0.0;
            P.dbg_trem[r] = pend ? trem : 0;
            P.dbg_lhat[r] = pend ? Lh : 0u;
        }
    }
    uint64_t img[KR];
#pragma unroll
    for (uint32_t k = 0; k < KR; ++k) img[k] = ((pend_m >> k) & 1u) ? 0ull : kNone;   // 0: below t
    if (__any_sync(0xffffffffu, div_m)) {
#pragma unroll
        for (uint32_t k = 0; k < KR; ++k)
            if ((div_m >> k) & 1u)
                img[k] = (uint64_t)__double_as_longlong(div_rn_int(__dmul_rn(__uint2double_rn(Gk32[k]), 1e9),
                                                                   __fma_rn(__uint2double_rn(Lr[k]), v_d, eps_d)));
        if (blend) {                                       // NEXT-2 fairness blend (A47), every pending row
#pragma unroll
            for (uint32_t k = 0; k < KR; ++k)
                if ((div_m >> k) & 1u)
                    img[k] = (uint64_t)__double_as_longlong(blend_fair(__longlong_as_double((long long)img[k]),
                                                                       __ldg(P.fair + r0 + 32 * k + lane),
                                                                       c.fair_num, c.fair_den));
        }
    }
    A.pend += __popc(pend_m);
    uint32_t mem_m = 0;
#pragma unroll
    for (uint32_t k = 0; k < KR; ++k) {
        const uint32_t o = 32 * k + lane;
        mem_m |= (uint32_t)(((pend_m >> k) & 1u) && img[k] >= t_img) << k;
        if (kMat && o < nr) {
            const bool pend = (pend_m >> k) & 1u;
            P.img[r0 + o] = img[k];
            P.cost[r0 + o] = pend ? token_cost(q[k].len_in, q[k].pre, c.chunk) : 0u;
            if (pend && img[k] < A.mn) A.mn = img[k];
        }
    }
    spec_rows<KR>(S, P, c, mem_m, img, r0, [&](uint32_t k, uint32_t) { return q[k]; });
}

// one standalone item staged in the ring slot `sl` (rows appended after a load)
template <bool kMat, bool kDebug, bool kAppB>
__device__ __forceinline__ void std_item(const Pool& P, const Table& T, const GroupNow* sg, const Cfg& c,
                                         const Scratch& S, int64_t now, double v_d, int64_t v, uint32_t sc,
                                         uint64_t t_img, float t_lo_f, const Item& it, WarpSlot* sl, Part& A) {
    const uint32_t lane = threadIdx.x & 31, nr = it.r1 - it.r0;
    HotRow q[kR];
#pragma unroll
    for (uint32_t k = 0; k < kR; ++k) q[k] = 32 * k + lane < nr ? ld_row_s(sl->rows + 32 * k + lane) : HotRow{0, 0, 0, 0, 0, 0, 0};
    std_core<kMat, kDebug, kAppB, kR>(P, T, sg, c, S, now, v_d, v, sc, t_img, t_lo_f, it.r0, nr, q, A);
}

// ---- one compound item: whole tasks [it.t0, it.t1) on rows [it.r0, it.r1), staged in slot
// `sl` -- or, for one task of more calls than a slot holds, read from global memory in chunks.
// Per-warp shared-memory task slots.
struct TaskSlots {
    uint32_t T[kItemTasks];       // sum of len_rem over the task's pending calls
    uint32_t F[kItemTasks];       // 4: task dropped (A40)
    unsigned long long G[kItemTasks];   // sum of the calls' goodput, then the task goodput G_task
    double B[kItemTasks];         // fl(t_gen + eps) of the task, -1 when out of the exact range
    float Bf[kItemTasks];         // fl32 of it (the pre-test)
};

// phase A of a chunk of calls (rows base + 32 k + lane): pending / drop / regime / bound (a1, a2),
// the call's len_rem and goodput summed per task (a4) -- the rows are ordered by task, so the
// tasks of a 32-row slab are a contiguous range of lane groups: one whole-warp reduction per
// (slab, task), no atomics.  Leaves per row: the item-local task (lt), frames waited, pending.
template <typename RowAt, typename TaskAt, typename WriteBack>
__device__ __forceinline__ void cmp_phase_a(const Pool& P, const Table& T, const GroupNow* sg, const Cfg& c,
                                            int64_t now, uint32_t sc, const Item& it, uint32_t base, TaskSlots& ts,
                                            RowAt row_at, TaskAt task_at, WriteBack write_back, uint32_t* lt,
                                            uint32_t* fr, uint32_t& pend_m, uint32_t& accT,
                                            unsigned long long& accG, Part& A) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ntl = it.t1 - it.t0;
    HotRow q[kR];
    uint32_t rare_m = 0, drop_m = 0;
    pend_m = 0;
#pragma unroll
    for (uint32_t k = 0; k < kR; ++k) {
        const uint32_t r = base + 32 * k + lane;
        const bool in = r < it.r1;
        q[k] = in ? row_at(r) : HotRow{0, 0, 0, 0, 0, 0, 0};
        lt[k] = in ? task_at(r) - it.t0 : 0xFFFFFFFFu;
        const bool valid = lt[k] < ntl;
        if (in && !valid) A.err = 1;                          // a call outside its item (validated at load)
        const HotRow& x = q[k];
        const uint32_t F = valid ? ts.F[lt[k]] : 0u, st = m_state(x.meta);
        const bool drop = (F & 4u) && (st == kQueued || st == kWaiting);
        const bool pend = valid && x.arr <= now && st <= kPreempted && !drop;
        const uint32_t ep = fastdiv(x.gen, c.R, c.R_m, c.R_l);
        const bool stale = pend && m_epoch(x.meta) != ep + 1u;
        pend_m |= (uint32_t)pend << k;
        drop_m |= (uint32_t)drop << k;
        rare_m |= (uint32_t)(drop || (valid && pend != (bool)(m_flags(x.meta) & kStamped)) || stale) << k;
    }
    A.drop += __popc(drop_m);
    if (__any_sync(0xffffffffu, rare_m)) {
#pragma unroll
        for (uint32_t k = 0; k < kR; ++k) {
            if (!((rare_m >> k) & 1u)) continue;
            const bool pend = (pend_m >> k) & 1u;
            const uint32_t ep = fastdiv(q[k].gen, c.R, c.R_m, c.R_l);
            rare_row(T, c, P.rows + base + 32 * k + lane, q[k], pend, (drop_m >> k) & 1u,
                     pend && m_epoch(q[k].meta) != ep + 1u, ep, sc, A.ref);
            write_back(base + 32 * k + lane, q[k]);        // phase B reads the row again
        }
    }
#pragma unroll
    for (uint32_t k = 0; k < kR; ++k) {
        const HotRow& x = q[k];
        const bool pend = (pend_m >> k) & 1u;
        fr[k] = fastdiv(min(sc - x.since, 0xFFFFu), c.frame, c.F_m, c.F_l);
        uint32_t Tl = 0, Gc = 0;
        if (pend) {
            const uint32_t Lh = max(l_hat(x.lrow), x.gen + 1);
            const GroupNow G = sg[m_group(x.meta)];
            const uint64_t g64 = (uint64_t)G.w_in * x.len_in + (uint64_t)G.w_out * Lh;   // call goodput
            if (g64 >> 27) A.err = 1;            // a slab's sum (32 calls) must fit 32 bits (validated at load)
            Tl = Lh - x.gen; Gc = (uint32_t)g64;
        }
        if (base + 32 * k >= it.r1) continue;                 // warp-uniform: the slab is empty
        // the slab's tasks: from lane 0's to the last row's (rows ordered by task)
        const uint32_t last = base + 32 * k + 31 < it.r1 ? 31u : it.r1 - 1 - (base + 32 * k);
        const uint32_t tf = __shfl_sync(0xffffffffu, lt[k], 0), tl = __shfl_sync(0xffffffffu, lt[k], last);
        if (tf >= ntl || tl >= ntl) continue;                 // malformed (A.err already set)
        for (uint32_t t = tf; t <= tl; ++t) {                  // warp-uniform (usually 1-3 tasks)
            const bool mine = lt[k] == t;
            const uint32_t sT = __reduce_add_sync(0xffffffffu, mine ? Tl : 0u);
            const uint32_t sG = __reduce_add_sync(0xffffffffu, mine ? Gc : 0u);
            if (lane == (t & 31u)) { accT += sT; accG += sG; }  // task t's sums live in lane t % 32
        }
    }
}

template <bool kMat, bool kDebug, bool kAppB>
__device__ __forceinline__ void cmp_item(const Pool& P, const Table& T, const GroupNow* sg, const Cfg& c,
                                         const Scratch& S, int64_t now, int64_t v, uint32_t sc, uint64_t t_img,
                                         float t_lo_f, const Item& it, WarpSlot* sl, TaskSlots& ts, Part& A) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ntl = it.t1 - it.t0;
    const bool big = it.r1 - it.r0 > kItemRows;             // read from global memory, in chunks
    const uint32_t tb = it.r0 & ~3u;
    const uint32_t eb = it.t0 & ~3u;
    auto row_at = [&](uint32_t r) -> HotRow { return big ? ld_row(P.rows + r) : ld_row_s(sl->rows + (r - it.r0)); };
    auto task_at = [&](uint32_t r) -> uint32_t { return big ? __ldg(P.task + r) : sl->task[r - tb]; };
    auto tinfo_at = [&](uint32_t i) -> TaskInfo { return big ? P.tinfo[it.t0 + i] : sl->tinfo[i]; };
    // (a1) P:545, A40: a task none of whose calls was ever scheduled is dropped once it waited
    // longer than waiting_time; of a dropped task only its Running / Preempted calls stay pending
    for (uint32_t i = lane; i < ntl; i += 32) {
        ts.T[i] = 0; ts.G[i] = 0;
        const uint32_t ever = big ? P.tever[it.t0 + i] : sl->tever[it.t0 + i - eb];
        ts.F[i] = (!ever && now - tinfo_at(i).ac > c.waiting) ? 4u : 0u;
    }
    __syncwarp();
#ifdef JIT_TIMELINE
    auto gtc = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    unsigned long long* tlc = reinterpret_cast<unsigned long long*>(S.sk) + 16ull * (blockIdx.x * kScoreWarps + (threadIdx.x >> 5)) + 8;
    const unsigned long long c0 = gtc();
#endif
    uint32_t lt[kR], fr[kR], pend_m = 0, accT = 0;
    unsigned long long accG = 0;                            // task `lane`'s sums (kItemTasks <= 32)
    for (uint32_t base = it.r0; base < it.r1; base += kItemRows)   // warp-uniform trip count
        cmp_phase_a(P, T, sg, c, now, sc, it, base, ts, row_at, task_at,
                    [&](uint32_t r, const HotRow& x) { if (!big) sl->rows[r - it.r0] = x; }, lt, fr, pend_m,
                    accT, accG, A);
    if (lane < ntl) { ts.T[lane] = accT; ts.G[lane] = accG; }
    __syncwarp();
#ifdef JIT_TIMELINE
    const unsigned long long c1 = gtc();
#endif
    // ---- per task: G_task and fl(t_gen + eps) (a4)
    for (uint32_t i = lane; i < ntl; i += 32) {
        uint64_t Gt = 0;
        double Bd = -1.0;
        if (ts.T[i]) {                                    // some call pending (len_rem >= 1 each)
            const TaskInfo ti = tinfo_at(i);
            const uint64_t Tsum = ts.T[i];
            const int64_t trem = ti.dls - now;                // stage sub-deadline (advisory)
            Gt = ti.dlf <= now ? 0 : ti.gdone + ts.G[i];      // final deadline passed (A43)
            const uint64_t t_gen = Tsum * (uint64_t)v;
            if (kAppB && t_gen > (uint64_t)(trem > 0 ? trem : 0)) Gt = 0;
            const uint64_t Bi = t_gen + (uint64_t)c.eps;
            // exact range: Tsum v without overflow (high word 0), + eps below 2^53
            if (Bi < kTwo53 && Bi >= t_gen && __umul64hi(Tsum, (uint64_t)v) == 0) Bd = __ull2double_rn(Bi);
        }
        ts.G[i] = Gt; ts.B[i] = Bd; ts.Bf[i] = Bd < 0.0 ? 1.0f : __double2float_rn(Bd);
    }
    __syncwarp();
#ifdef JIT_TIMELINE
    const unsigned long long c2 = gtc();
#endif
    // ---- phase B: the key of every pending call (a5 over the task aggregate); a one-chunk item
    // keeps phase A's per-call values in registers, a big one recomputes them chunk by chunk
    for (uint32_t base = it.r0; base < it.r1; base += kItemRows) {   // warp-uniform trip count
        if (big) {
#pragma unroll
            for (uint32_t k = 0; k < kR; ++k) {
                const uint32_t r = base + 32 * k + lane;
                const bool in = r < it.r1;
                const HotRow x = in ? row_at(r) : HotRow{0, 0, 0, 0, 0, 0, 0};
                lt[k] = in ? task_at(r) - it.t0 : 0xFFFFFFFFu;
                const bool pend = lt[k] < ntl && x.arr <= now && m_state(x.meta) <= kPreempted;  // drops are written
                pend_m = (pend_m & ~(1u << k)) | ((uint32_t)pend << k);
                fr[k] = fastdiv(min(sc - x.since, 0xFFFFu), c.frame, c.F_m, c.F_l);
            }
        }
        uint32_t Gk32[kR];
        double Bk[kR];
        uint32_t div_m = 0;
#pragma unroll
        for (uint32_t k = 0; k < kR; ++k) {
            const bool pend = (pend_m >> k) & 1u;
            const uint32_t j = pend ? lt[k] : 0u;
            const double Bd = ts.B[j];
            if (pend && Bd < 0.0) A.err = 1;
            const uint64_t Gp = ts.G[j] + (uint64_t)c.delta * fr[k];
            if (pend && Gp >= kTwo53 / 1000000000ull) A.err = 1;
            Gk32[k] = (uint32_t)Gp;
            Bk[k] = Bd < 0.0 ? 1.0 : Bd;
            // the fp32 pre-test with B_f = fl(B) (relative error 2^-24, within below_t's margin)
            const bool below = __fmul_rn(__uint2float_rn((uint32_t)Gp), 1e9f) < __fmul_rn(t_lo_f, ts.Bf[j]);
            div_m |= (uint32_t)(pend && (kMat || c.fair_num || !below)) << k;
            if (kDebug && base + 32 * k + lane < it.r1) {
                const uint32_t r = base + 32 * k + lane;
                const HotRow x = row_at(r);
                int64_t trem = 0;
                double rate = 0.0;
                if (pend) {
                    trem = tinfo_at(j).dls - now;
                    rate = make_rate(ts.T[j], trem);
                }
                P.dbg_rate[r] = rate; P.dbg_trem[r] = trem;
                P.dbg_lhat[r] = pend ? max(l_hat(x.lrow), x.gen + 1) : 0u;
            }
        }
        uint64_t img[kR];
#pragma unroll
        for (uint32_t k = 0; k < kR; ++k) img[k] = ((pend_m >> k) & 1u) ? 0ull : kNone;
        if (__any_sync(0xffffffffu, div_m)) {
#pragma unroll
            for (uint32_t k = 0; k < kR; ++k)
                if ((div_m >> k) & 1u)
                    img[k] = (uint64_t)__double_as_longlong(div_rn_int(__dmul_rn(__uint2double_rn(Gk32[k]), 1e9), Bk[k]));
            if (c.fair_num) {                              // NEXT-2 fairness blend (A47)
#pragma unroll
                for (uint32_t k = 0; k < kR; ++k)
                    if ((div_m >> k) & 1u)
                        img[k] = (uint64_t)__double_as_longlong(blend_fair(__longlong_as_double((long long)img[k]),
                                                                           __ldg(P.fair + base + 32 * k + lane),
                                                                           c.fair_num, c.fair_den));
            }
        }
        A.pend += __popc(pend_m);
        uint32_t mem_m = 0;
#pragma unroll
        for (uint32_t k = 0; k < kR; ++k) {
            const uint32_t r = base + 32 * k + lane;
            mem_m |= (uint32_t)(((pend_m >> k) & 1u) && img[k] >= t_img) << k;
            if (kMat && r < it.r1) {
                const bool pend = (pend_m >> k) & 1u;
                const HotRow x = row_at(r);
                P.img[r] = img[k];
                P.cost[r] = pend ? token_cost(x.len_in, x.pre, c.chunk) : 0u;
                if (pend && img[k] < A.mn) A.mn = img[k];
            }
        }
        spec_rows<kR>(S, P, c, mem_m, img, base, [&](uint32_t, uint32_t r) { return row_at(r); });
    }
    __syncwarp();
#ifdef JIT_TIMELINE
    if (lane == 0) { tlc[0] += c1 - c0; tlc[1] += c2 - c1; tlc[2] += gtc() - c2; tlc[3] += 1; }
#endif
}

// per-CTA reduction of the warps' partials, one set of global atomics per CTA
__device__ __forceinline__ void store_part(BlockPart* gpart, Ctrl* ctrl, Part A, bool count, bool mat) {
    __shared__ uint32_t s_pend, s_drop, s_ref, s_err;
    __shared__ unsigned long long s_mn;
    if (threadIdx.x == 0) { s_pend = 0; s_drop = 0; s_ref = 0; s_err = 0; s_mn = kNone; }
    __syncthreads();
    const uint32_t pend = warp_sum(A.pend), drop = warp_sum(A.drop), ref = warp_sum(A.ref);
    const uint32_t err = __reduce_or_sync(0xffffffffu, A.err);
    const uint64_t mn = mat ? warp_min_u64(A.mn) : kNone;
    if ((threadIdx.x & 31) == 0) {
        if (pend) atomicAdd(&s_pend, pend);
        if (drop) atomicAdd(&s_drop, drop);
        if (ref) atomicAdd(&s_ref, ref);
        if (err) atomicOr(&s_err, err);
        if (mn != kNone) atomicMin(&s_mn, (unsigned long long)mn);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (count) {
            if (s_pend || s_drop)
                atomicAdd(&gpart->cnt, (unsigned long long)s_pend | ((unsigned long long)s_drop << 32));
            if (s_ref) atomicAdd(&gpart->refresh, s_ref);
        }
        if (s_err) atomicOr(&gpart->err, s_err);
        if (mat && s_mn != kNone) atomicMin(&ctrl->min_img, s_mn);
    }
}

// dynamic shared memory: SLO groups (256 max), per warp its task slots and its ring of item slots
struct WarpSmem {
    WarpSlot slot[kStagesW];
    TaskSlots ts;
    uint64_t bar[kStagesW];
};
__host__ __device__ constexpr uint32_t score_smem_bytes(uint32_t n_groups) {
    return (uint32_t)(((sizeof(GroupNow) * n_groups + 127) & ~127ull) + sizeof(WarpSmem) * kScoreWarps);
}

// The standalone slabs of warp w (of W): a warp that owns more ring items (compound tasks, cost
// bal_w / 256 slabs each) gets fewer slabs, so that every warp's share of the pass is about the
// same.  Closed form: quota q = max(0, t - bal_w * ring items) in 1/256 slab, t = the mean share;
// warp w starts at f(w) = floor(n32 * (sum of the quotas before it) / (sum of all quotas)).  f is
// evaluated in fp64 with one reciprocal (no 64-bit division at kernel entry): the same monotone expression
// on every warp, so consecutive ranges meet exactly; the last warp ends at n32.
__device__ __forceinline__ void std_slabs(uint32_t w, uint32_t W, uint32_t n32, uint32_t n_ring, uint32_t bal_w,
                                          uint32_t& s0, uint32_t& s1) {
    const uint64_t B = bal_w, T = (uint64_t)n32 * 256u + B * n_ring;
    const uint64_t t = (uint64_t)__double2ull_rd(__dmul_rn(__ull2double_rn(T), __drcp_rn((double)W)));
    const uint32_t base = n_ring / W, ex = n_ring - base * W;
    const uint64_t qhi = t > B * (base + 1) ? t - B * (base + 1) : 0, qlo = t > B * base ? t - B * base : 0;
    auto pre = [&](uint64_t x) { return (x < ex ? x : ex) * qhi + (x > ex ? x - ex : 0) * qlo; };
    const double tot = __ull2double_rn(pre(W)), n = (double)n32, rt = __drcp_rn(tot);
    auto f = [&](uint32_t x) -> uint32_t {
        if (x >= W) return n32;
        return min(n32, (uint32_t)__double2uint_rd(__dmul_rn(__dmul_rn(n, __ull2double_rn(pre(x))), rt)));
    };
    s0 = tot > 0.0 ? f(w) : 0u;
    s1 = tot > 0.0 ? f(w + 1) : 0u;
}

// mode 0: a step (partials counted, speculative set collected); mode 1: re-score for the exact
// path (kMat; keys and costs only, nothing counted again -- the pool state is already this
// step's, so the pass is idempotent)
template <bool kMat, bool kDebug, bool kAppB>
__global__ void __launch_bounds__(kScoreThreads, JIT_SCORE_MINB) k_score(Pool P, Table T, const Group* groups,
                                                                         uint32_t n_groups, Cfg c, Ctrl* ctrl,
                                                                         Scratch S, int64_t now, int64_t v, int mode) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef JIT_TIMELINE
    // diagnostic builds: %globaltimer per warp (start, prologue done, items done, end) -> S.sk
    auto gt = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    const unsigned long long tl0 = gt();
    unsigned long long* tl = reinterpret_cast<unsigned long long*>(S.sk) + 16ull * (blockIdx.x * kScoreWarps + warp);
    if (lane == 0) for (int z = 8; z < 16; ++z) tl[z] = 0;
#endif
    const uint32_t W = gridDim.x * kScoreWarps;
    const uint32_t i0 = blockIdx.x * kScoreWarps + warp;
    uint32_t s0 = 0, s1 = 0;
    HotRow cur[kRs], nxt[kRs];
    auto load = [&](HotRow* q, uint32_t sb) {
#pragma unroll
        for (uint32_t k = 0; k < kRs; ++k) {
            const uint32_t r = 32 * (sb + k) + lane;
            q[k] = (sb + k < s1 && r < P.n_single) ? ld_row_g(P.rows + r) : HotRow{0, 0, 0, 0, 0, 0, 0};
        }
    };
    // every independent global load of the prologue at once (one round trip): the handle's
    // counters and the item count (one thread per CTA: every warp reading the same line would queue
    // 4x the requests on one L2 slice), the SLO groups, this warp's ring-item descriptors (ring item
    // j in lane j; beyond 32 read when needed; the items array is readable up to its capacity).
    // The ring items are items [n_std_items, n_items): compound tasks and standalone rows appended
    // since the load.
    __shared__ Persist s_ps;
    __shared__ uint32_t s_n_items;
    if (threadIdx.x == 0) { s_ps = *S.persist; s_n_items = *S.n_items; }
    const uint32_t nstd = S.n_std_items;
    Item dsc{0, 0, 0, 0};
    if (nstd + i0 + lane * W < S.item_cap) dsc = S.items[nstd + i0 + lane * W];
    Group g0{};
    if (threadIdx.x < n_groups) g0 = groups[threadIdx.x];
    // while those are in flight: this warp's standalone slabs (balanced against the ring items it
    // owns, std_slabs; the host's ring count at launch) and the first chunk's row loads
#ifndef JIT_SKIP_STD
    std_slabs(i0, W, (P.n_single + 31) >> 5, S.n_ring_h, S.bal_w, s0, s1);
    if (s0 < s1) load(cur, s0);
#endif
    __syncthreads();
    const Persist ps = s_ps;
    const uint32_t n_items = s_n_items;
    if (mode == 0 && ps.host_pending) {                    // chained after a step that needs the host
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&S.persist->skipped, 1u);
        return;
    }
#ifdef JIT_TIMELINE
    const unsigned long long tpa = gt();
#endif
    GroupNow* sg = reinterpret_cast<GroupNow*>(smem);
    WarpSmem* ws = reinterpret_cast<WarpSmem*>(smem + ((sizeof(GroupNow) * n_groups + 127) & ~127ull)) + warp;
    const uint32_t n_ring = n_items > nstd ? n_items - nstd : 0u;
    const uint32_t n_mine = i0 < n_ring ? (n_ring - i0 + W - 1) / W : 0u;   // ring items i0 + j W of this warp
    const uint64_t pol = evict_first_policy();
    auto item_j = [&](uint32_t j) -> Item {                // warp-uniform j
        if (j >= 32) return S.items[nstd + i0 + j * W];
        return Item{__shfl_sync(0xffffffffu, dsc.r0, j), __shfl_sync(0xffffffffu, dsc.r1, j),
                    __shfl_sync(0xffffffffu, dsc.t0, j), __shfl_sync(0xffffffffu, dsc.t1, j)};
    };
    if (lane == 0) {
        for (uint32_t s = 0; s < kStagesW; ++s) mbar_init(&ws->bar[s], 1);
        mbar_init_fence();
    }
    // fill the ring: the ring items' bytes stream in while the warp scores its standalone slabs.
    // Issued after the first standalone chunk, so that the prologue does not wait for the item
    // descriptors
    bool ring_filled = false;
    auto fill_ring = [&]() {
        for (uint32_t s = 0; s < kStagesW && s < n_mine; ++s) {
            const Item it = item_j(s);
            if (lane == 0) issue_item(P, it, &ws->slot[s], &ws->bar[s], pol);
        }
        ring_filled = true;
    };
#ifdef JIT_TIMELINE
    const unsigned long long tpb = gt();
#endif
    for (uint32_t g = threadIdx.x; g < n_groups; g += kScoreThreads) {
        const Group G = g < kScoreThreads ? g0 : groups[g];
        GroupNow x;
        const int64_t base = G.type == kLAT ? G.ttft_ns : G.type == kDDL ? G.e2el_ns : G.type == kBE ? G.be_deadline_ns : 0;
        x.bn = base - now;
        x.tok = G.type == kLAT ? (uint32_t)G.tbt_ns : 0u;          // tbt < 2^32 (validated at init)
        x.w_in = (G.type == kDDL || G.type == kCMP) ? G.w_in : 0u;
        x.w_out = G.type != kBE ? G.w_out : 0u;
        x.pad = 0;
        sg[g] = x;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && mode == 0) { ctrl->now = now; ctrl->v = v; }
    const uint64_t t_img = mode == 0 ? ps.t_guess : kNone;
    const uint32_t sc = ps.steps;
    // t_lo_f = t (1 - 2^-16) rounded toward zero (below_t); no threshold (kNone): nothing can
    // join, no key is needed
    const float t_lo_f = t_img == kNone ? __int_as_float(0x7F800000)
                                        : __double2float_rz(__dmul_rn(__longlong_as_double((long long)t_img),
                                                                      1.0 - 1.52587890625e-05));
#ifdef JIT_TIMELINE
    const unsigned long long tpc = gt();
#endif
    __syncthreads();
    pdl_launch_dependents();                               // k_spec may launch now (it waits for us)
#ifdef JIT_TIMELINE
    const unsigned long long tl1 = gt();
    unsigned long long tlw = 0, tls = 0, tlc = 0;          // waiting for slots; in std / cmp items
    uint32_t nls = 0, nlc = 0;
#endif
    Part A{0u, 0u, 0u, 0u, kNone};
    const double v_d = (double)v;
#ifndef JIT_SKIP_STD
    // ---- the standalone rows [0, n_single): kRs rows per lane read with 256-bit loads straight
    // into registers, the next chunk's loads issued before the current chunk is scored
    for (uint32_t sb = s0; sb < s1; sb += kRs) {           // warp-uniform
        if (sb + kRs < s1) load(nxt, sb + kRs);
        const uint32_t nr = min(32u * min(s1 - sb, kRs), P.n_single - 32u * sb);
#ifdef JIT_STD_FLOOR
        if (cur[0].gen == 0xFFFFFFFFu || cur[kRs - 1].gen == 0xFFFFFFFFu) A.err = 1;
#else
        std_core<kMat, kDebug, kAppB, kRs>(P, T, sg, c, S, now, v_d, v, sc, t_img, t_lo_f, 32u * sb, nr, cur, A);
#endif
#pragma unroll
        for (uint32_t k = 0; k < kRs; ++k) cur[k] = nxt[k];
        if (!ring_filled) fill_ring();
    }
#endif
    if (!ring_filled) fill_ring();
#ifdef JIT_TIMELINE
    tls = gt() - tl1; nls = (s1 - s0 + kRs - 1) / kRs;     // the standalone phase and its chunks
#endif
    uint32_t s = 0, par = 0;                               // ring position and its phase parity
    for (uint32_t j = 0; j < n_mine; ++j) {
        const Item it = item_j(j);
#ifdef JIT_TIMELINE
        const unsigned long long tw0 = gt();
        mbar_wait(&ws->bar[s], par);
        const unsigned long long tw1 = gt();
        tlw += tw1 - tw0;
#else
        mbar_wait(&ws->bar[s], par);
#endif
#ifdef JIT_SCORE_FLOOR
        // timing experiment only (profiles/tune_*.sh): the item stream without the row math
        if (lane == 0 && ws->slot[s].rows[0].gen == 0xFFFFFFFFu) A.err = 1;
        if (false)
#endif
        if (it.t1 == it.t0) std_item<kMat, kDebug, kAppB>(P, T, sg, c, S, now, v_d, v, sc, t_img, t_lo_f, it, &ws->slot[s], A);
        else
#ifdef JIT_SKIP_CMP
        { if (lane == 0 && ws->slot[s].rows[0].gen == 0xFFFFFFFFu) A.err = 1; }
#else
        cmp_item<kMat, kDebug, kAppB>(P, T, sg, c, S, now, v, sc, t_img, t_lo_f, it, &ws->slot[s], ws->ts, A);
#endif
        __syncwarp();                                      // every lane is done with the slot
#ifdef JIT_TIMELINE
        tlc += gt() - tw1; ++nlc;
#endif
        if (j + kStagesW < n_mine) {
            const Item nx = item_j(j + kStagesW);
            if (lane == 0) issue_item(P, nx, &ws->slot[s], &ws->bar[s], pol);
        }
        if (++s == kStagesW) { s = 0; par ^= 1u; }
    }
#ifdef JIT_TIMELINE
    const unsigned long long tl2 = gt();
#endif
    store_part(S.gpart, ctrl, A, mode == 0, kMat);
#ifdef JIT_TIMELINE
    if (lane == 0) { tl[0] = tl0; tl[1] = tl1; tl[2] = tl2; tl[3] = gt(); tl[4] = tlw; tl[5] = n_mine;
                     tl[6] = tls | ((unsigned long long)nls << 48); tl[7] = tlc | ((unsigned long long)nlc << 48);
                     tl[12] = tpa - tl0; tl[13] = tpb - tl0; tl[14] = tpc - tl0; }
#endif
}

// Measurement only (jit_sched_time_scoring, JIT_TIME_READ_FLOOR): the pool's hot rows read the
// way k_score reads its standalone slabs (256-bit loads, 2 rows per lane, the next chunk in flight)
// and nothing else -- the achievable time of this footprint, the denominator k_score is compared
// with beside the copy peak.
__global__ void __launch_bounds__(256) k_read_floor(const HotRow* rows, uint32_t n, unsigned long long* sink) {
    const uint32_t lane = threadIdx.x & 31, W = gridDim.x * 8, w = blockIdx.x * 8 + (threadIdx.x >> 5);
    const uint32_t n32 = (n + 31) >> 5, s0 = (uint32_t)((uint64_t)n32 * w / W), s1 = (uint32_t)((uint64_t)n32 * (w + 1) / W);
    uint64_t acc = 0;
    HotRow cur[2], nxt[2];
    auto load = [&](HotRow* q, uint32_t sb) {
#pragma unroll
        for (uint32_t k = 0; k < 2; ++k) {
            const uint32_t r = 32 * (sb + k) + lane;
            q[k] = (sb + k < s1 && r < n) ? ld_row_g(rows + r) : HotRow{0, 0, 0, 0, 0, 0, 0};
        }
    };
    if (s0 < s1) load(cur, s0);
    for (uint32_t sb = s0; sb < s1; sb += 2) {
        if (sb + 2 < s1) load(nxt, sb + 2);
#pragma unroll
        for (uint32_t k = 0; k < 2; ++k)
            acc ^= (uint64_t)cur[k].arr ^ cur[k].len_in ^ cur[k].gen ^ cur[k].pre ^ cur[k].lrow ^ cur[k].meta ^ cur[k].since;
#pragma unroll
        for (uint32_t k = 0; k < 2; ++k) cur[k] = nxt[k];
    }
    if (acc == 0x0123456789ABCDEFull) sink[blockIdx.x & 63] = acc;       // keeps the loads alive
}

}  // namespace jit
