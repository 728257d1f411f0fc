// spec.cuh -- the speculative resolve of the step (a7)-(a9) and its sharded variant.
//
//   k_spec        one CTA, launched as a programmatic dependent of k_score: exact B*, bp, thr, Cd
//                 and the window from the speculative set S = {key >= t}
//   k_spec_big    the same for a set larger than k_spec's one-element-per-thread path
//   k_spec_export / k_spec_merge   the sharded step's union of the ranks' sets
#pragma once
#include "select.cuh"

namespace jit {

// --------------------------------------------------------------------------------------
// The small-set resolve, shared by k_score's last CTA (the step's fast path) and k_spec
// --------------------------------------------------------------------------------------
// thread 0: give up on the speculative resolve -> the host runs the exact radix path after the
// step (finish_step in abi.cu); rare: first step after a load, a threshold far off, huge ties
__device__ __forceinline__ void spec_fallback(Ctrl* ctrl, int* fb) {
    ctrl->status = ST_FALLBACK; ctrl->fallback = 1;
    *fb = 1;
}

// Small speculative set (n <= kSpecFast, the steady state): one element per thread and no sort.
// Element i's rank in the priority order (key desc, id asc) and its inclusive cost prefix come
// from one pass over the set (shared-memory broadcast reads), so B* = #{i : rank_i < B_max and
// prefix_i <= tau} (monotone in the rank) is one barrier count; the same for Cd's (len, id) order.
#ifndef JIT_SPEC_UNROLL
#define JIT_SPEC_UNROLL 5              // the window argmax's shuffle levels (1: a loop, smaller code)
#endif
constexpr int kSpecUnroll = JIT_SPEC_UNROLL;
constexpr uint32_t kSpecFast = 256;
constexpr uint32_t kSpecFastChunk = (1u << 24) - 1;   // costs <= chunk: kSpecFast costs sum below 2^32
// priority-order rank record: (key image, id) as one 96-bit word V = img_hi : img_lo : ~id, so
// "q before me" (key desc, id asc) is V_q > V_me -- the borrow of V_me - V_q (three subtractions);
// w = -cost, so borrow_mask * w adds cost
__device__ __forceinline__ uint4 rank_rec(uint64_t img, uint32_t id, uint32_t cost) {
    return make_uint4(~id, (uint32_t)img, (uint32_t)(img >> 32), 0u - cost);
}
__device__ __forceinline__ uint32_t before_mask(const uint4& q, const uint4& me) {
    uint32_t t, b;
    asm("sub.cc.u32 %0, %2, %5;\n\t"
        "subc.cc.u32 %0, %3, %6;\n\t"
        "subc.cc.u32 %0, %4, %7;\n\t"
        "subc.u32 %1, 0, 0;"
        : "=&r"(t), "=r"(b) : "r"(me.x), "r"(me.y), "r"(me.z), "r"(q.x), "r"(q.y), "r"(q.z));
    (void)t;
    return b;                                   // 0xFFFFFFFF when q precedes me, else 0
}
// dynamic shared memory of the small-set resolve (f_rec, f_img, f_id, f_cost, f_wk, pc, pf, o_elem):
// k_spec launches with only this much, so its CTA fits beside k_score's draining CTAs early
constexpr uint32_t kSpecFastSmem = 16 * kSpecFast + 8 * kSpecFast + 4 * kSpecFast + 4 * kSpecFast + 8 * kSpecFast +
                                   8 * (kSpecFast + 2) + 16 * (kSpecFast + 1) + 4 * kSpecFast;
struct SpecEl {                 // one element of the speculative set, preloaded by k_spec
    uint64_t img;
    uint32_t id, cost, len, row, meta, since;
    uint32_t own;               // 1: the row belongs to this handle (a sharded step merges all ranks' sets)
};
template <uint32_t NT>
static __device__ __forceinline__ void spec_fast(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t n,
                                              bool whole, uint64_t t_img, const SpecEl& el, unsigned char* smem) {
    uint4* f_rec = reinterpret_cast<uint4*>(smem);                           // [kSpecFast] rank_rec
    uint64_t* f_img = reinterpret_cast<uint64_t*>(f_rec + kSpecFast);        // [kSpecFast]
    uint32_t* f_id = reinterpret_cast<uint32_t*>(f_img + kSpecFast);         // [kSpecFast]
    uint32_t* f_cost = f_id + kSpecFast;                                     // [kSpecFast]
    uint64_t* f_wk = reinterpret_cast<uint64_t*>(f_cost + kSpecFast);        // window key (len << 32 | id), ~0 if not in Cd
    unsigned long long* pc = reinterpret_cast<unsigned long long*>(f_wk + kSpecFast);   // [kSpecFast + 1]
    u128* pf = reinterpret_cast<u128*>(pc + kSpecFast + 2);                               // [kSpecFast + 1]
    uint32_t* o_elem = reinterpret_cast<uint32_t*>(pf + kSpecFast + 1);                  // window position -> element
    __shared__ uint64_t f_scan[32];
    __shared__ u128 f_scan128[32];
    __shared__ u128 f_best[32];
    __shared__ uint32_t f_bi[32], f_bj[32];
    const uint32_t tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const bool own = tid < n;
    const uint32_t sc = S.persist->steps;            // read before any barrier (thread 0 bumps it last)
    const uint64_t img = own ? el.img : kNone;
    const uint32_t id = el.id, cost = own ? el.cost : 0u, len = el.len;
    __shared__ uint32_t f_rank2[kSpecFast];
    __shared__ uint32_t f_pre2[kSpecFast];
    if (own) {
        f_rec[tid] = rank_rec(img, id, cost);
        f_img[tid] = img; f_id[tid] = id; f_cost[tid] = cost;
        f_rank2[tid] = 0; f_pre2[tid] = 0;
    }
    __syncthreads();
    stamp(ctrl, 2);
    // (a7) rank in the priority order and inclusive cost prefix.  The n^2 comparisons are spread
    // over the whole CTA: element e is counted by F = NT / n threads (tid = e + n * part), each
    // over a 1/F share of the set (16-B broadcast reads, 2 accumulators), summed in shared memory.
    {
        const uint32_t F = n ? min(NT / n, 8u) : 1u;
        const uint32_t e = n ? tid % n : 0u, part = n ? tid / n : 1u;
        if (part < F) {
            const uint32_t j0 = (uint32_t)((uint64_t)n * part / F), j1 = (uint32_t)((uint64_t)n * (part + 1) / F);
            const uint4 me = f_rec[e];
            uint32_t ra = 0, rb = 0, pa = 0, pb = 0;   // cost prefixes < 2^32 (costs <= kSpecFastChunk)
            uint32_t j = j0;
            for (; j + 1 < j1; j += 2) {
                const uint4 q0 = f_rec[j], q1 = f_rec[j + 1];
                const uint32_t b0 = before_mask(q0, me), b1 = before_mask(q1, me);
                ra -= b0; pa += b0 * q0.w;
                rb -= b1; pb += b1 * q1.w;
            }
            if (j < j1) {
                const uint4 q0 = f_rec[j];
                const uint32_t b0 = before_mask(q0, me);
                ra -= b0; pa += b0 * q0.w;
            }
            if (F == 1) { f_rank2[e] = ra + rb; f_pre2[e] = pa + pb; }
            else { atomicAdd(&f_rank2[e], ra + rb); atomicAdd(&f_pre2[e], pa + pb); }
        }
        __syncthreads();
    }
    uint32_t rank = own ? f_rank2[tid] : 0u;          // own => tid < kSpecFast: written by itself
    const uint64_t pre = own ? (uint64_t)f_pre2[tid] + cost : 0ull;
    const bool fits = own && rank + 1 <= c.max_batch && pre <= c.token_budget;
    __shared__ uint64_t f_byrank[kSpecFast];                // key image by priority rank
    if (own) f_byrank[rank] = img;
    const uint32_t bstar = (uint32_t)__syncthreads_count(fits);
    const uint64_t bp_img = bstar ? f_byrank[bstar - 1] : kNone;   // the B*-th request (A15)
    stamp(ctrl, 3);
    // every thread derives bp, thr and the exactness verdict from the same block-uniform values
    // (no serial thread-0 section and no broadcast barrier); thread 0 records them
    uint64_t thr_img = 0;
    {
        int fb = 0;
        double bp = 0.0, thr = 0.0;
        if (bstar == 0) fb = 2;
        else if (bstar == n && !whole) fb = 1;          // every entry of S fits: exact only when S
        else {                                          // is the whole pending set (bp = its min key)
            bp = __longlong_as_double((long long)bp_img);
            thr = __dmul_rn(c.p, bp);                   // A16
            thr_img = (uint64_t)__double_as_longlong(thr);
            if (!whole && thr_img < t_img) fb = 1;      // Cd may leave S
        }
        if (tid == 0) {
            if (fb == 2) { ctrl->error |= 1u; ctrl->status = ST_ERROR; }
            else if (fb == 1) { ctrl->status = ST_FALLBACK; ctrl->fallback = 1; }
            else { ctrl->b_star = bstar; ctrl->bp = bp; ctrl->thr = thr; ctrl->thr_img = thr_img; }
        }
        if (fb) return;
    }
    // (a8) Cd = {key >= thr}; (a9) its (len, id) order (A17/A18)
    const bool cd = own && img >= thr_img;
    const uint64_t wk = ((uint64_t)len << 32) | id;
    // Cd is a prefix of the priority order: its elements hold the ranks 0..|Cd|-1, which serve as
    // compact indices (f_pre2 is free again: reused for the window positions)
    if (cd) f_wk[rank] = wk;
    if (tid < kSpecFast) f_pre2[tid] = 0;
    const uint32_t ncd = (uint32_t)__syncthreads_count(cd);
    {   // window position of each Cd element: #{Cd elements before it in (len, id) order}, the
        // comparisons spread over the CTA as above
        const uint32_t F = ncd ? min(NT / ncd, 8u) : 1u;
        const uint32_t e = ncd ? tid % ncd : 0u, part = ncd ? tid / ncd : 1u;
        if (part < F && e < ncd) {
            const uint64_t mk = f_wk[e];
            const uint32_t j0 = (uint32_t)((uint64_t)ncd * part / F), j1 = (uint32_t)((uint64_t)ncd * (part + 1) / F);
            uint32_t pa = 0, pb = 0, j = j0;
            for (; j + 1 < j1; j += 2) { pa += f_wk[j] < mk; pb += f_wk[j + 1] < mk; }
            if (j < j1) pa += f_wk[j] < mk;
            if (F == 1) f_pre2[e] = pa + pb; else atomicAdd(&f_pre2[e], pa + pb);
        }
        __syncthreads();
        if (cd) o_elem[f_pre2[rank]] = tid;
    }
    __shared__ uint32_t f_row[kSpecFast], f_meta[kSpecFast], f_since[kSpecFast];
    if (own) { f_row[tid] = el.own ? el.row : 0xFFFFFFFFu; f_meta[tid] = el.meta; f_since[tid] = el.since; }
    if (tid == 0) { ctrl->n_cand = ncd; ctrl->status = ST_RESOLVED; }
    __syncthreads();
    stamp(ctrl, 4);
    // prefix sums in window order: position p = tid
    {
        uint64_t cv = 0;
        u128 fv = 0;
        if (tid < ncd) {
            const uint32_t e = o_elem[tid];
            cv = f_cost[e];
            fv = (u128)fixed_point(__longlong_as_double((long long)f_img[e]));    // A19
        }
        // one exclusive block scan of the pair (two barriers, not two scans of three)
        uint64_t xc = cv;
        u128 xf = fv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t yc = __shfl_up_sync(0xffffffffu, xc, o);
            const u128 yf = shfl_up_u128(xf, o);
            if (lane >= o) { xc += yc; xf += yf; }
        }
        if (lane == 31) { f_scan[wid] = xc; f_scan128[wid] = xf; }
        __syncthreads();
        constexpr int nw = NT / 32;
        if (wid == 0) {
            uint64_t sc = lane < nw ? f_scan[lane] : 0ull;
            u128 sf = lane < nw ? f_scan128[lane] : (u128)0;
#pragma unroll
            for (int o = 1; o < nw; o <<= 1) {
                const uint64_t yc = __shfl_up_sync(0xffffffffu, sc, o);
                const u128 yf = shfl_up_u128(sf, o);
                if (lane >= o) { sc += yc; sf += yf; }
            }
            if (lane < nw) { f_scan[lane] = sc; f_scan128[lane] = sf; }
        }
        __syncthreads();
        if (tid < ncd) {
            pc[tid] = (wid ? f_scan[wid - 1] : 0ull) + xc - cv;
            pf[tid] = (wid ? f_scan128[wid - 1] : (u128)0) + xf - fv;
        }
        if (tid == 0) { pc[ncd] = f_scan[nw - 1]; pf[ncd] = f_scan128[nw - 1]; }
    }
    __syncthreads();
    stamp(ctrl, 5);
    // first argmax over i of the window [i, j(i)] (j(i): largest end within tau and B_max; P:424 strict >)
    u128 best = 0;
    uint32_t bi = 0xFFFFFFFFu, bj = 0;
    if (tid < ncd) {
        const uint64_t lim = (uint64_t)pc[tid] + c.token_budget;
        uint32_t lo = tid, hi = (uint32_t)min((uint64_t)ncd - 1, (uint64_t)tid + c.max_batch - 1);
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (pc[mid + 1] <= lim) lo = mid; else hi = mid - 1;
        }
        best = pf[lo + 1] - pf[tid]; bi = tid; bj = lo;
    }
    const uint32_t nwc = (ncd + 31) >> 5;                  // warps holding window starts (ncd >= 1: bp is in Cd)
    if ((uint32_t)wid < nwc) {
#pragma unroll kSpecUnroll
        for (int o = 16; o > 0; o >>= 1) {
            const u128 ob = shfl_xor_u128(best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
        }
        if (lane == 0) { f_best[wid] = best; f_bi[wid] = bi; f_bj[wid] = bj; }
    }
    __syncthreads();
    // every thread reduces the per-warp winners in warp (= start position) order; strict > keeps
    // the first maximum -- no second barrier
    best = f_best[0]; bi = f_bi[0]; bj = f_bj[0];
    for (uint32_t w = 1; w < nwc; ++w) {
        const u128 ob = f_best[w];
        if (ob > best) { best = ob; bi = f_bi[w]; bj = f_bj[w]; }
    }
    stamp(ctrl, 6);
    // the batch in window order and its bookkeeping: ever_scheduled, Running, the steps_waited stamp
    const uint32_t ns = bj - bi + 1;
    if (tid < ns) {
        const uint32_t e = o_elem[bi + tid];
        const uint32_t r = f_row[e];
        S.out_ids[tid] = f_id[e];
        S.out_tokens[tid] = f_cost[e];
        S.out_rows[tid] = r;
        const uint32_t B = c.max_batch + 1;                 // and the pinned host mirror (no D2H copy)
        S.h_batch[tid] = f_id[e]; S.h_batch[B + tid] = f_cost[e]; S.h_batch[2 * B + tid] = r;
        if (r != 0xFFFFFFFFu) book_selected(P, r, f_meta[e], f_since[e], sc);   // meta / since as k_score left them
    }
    if (tid == 0) {
        ctrl->n_selected = ns;
        ctrl->total_tokens = (uint32_t)(pc[bj + 1] - pc[bi]);
        ctrl->i_best = bi; ctrl->j_best = bj;
        ctrl->window_done = 1; ctrl->batch_on_host = 1;
        finish_counters(S.persist, ctrl);               // next step's threshold: this cutoff with a 3% margin
    }
    stamp(ctrl, 7);
}

#ifdef JIT_EXACT_TU
// --------------------------------------------------------------------------------------
// k_spec: one CTA of 512 threads.  Reduces the scoring partials, then resolves (a7)/(a8)
// exactly from the speculative set S = {key >= t} and runs the window (a9) on Cd, all in
// shared memory.  S is upward closed in the (key desc, id asc) order, i.e. a PREFIX of the
// priority order, so the budget walk restricted to S is the exact walk as long as it stops
// inside S (or S holds every pending row); Cd = {key >= thr} lies in S when thr >= t.
// Otherwise the host runs the exact radix path after the step (finish_step in abi.cu).
//   1. one pass over S: key images / costs to smem + a cost-weighted histogram of the key
//      image (2048 bins of 2^-9 relative width above t, the top bin open-ended);
//   2. one block scan over the bins (count and cost packed in one u64) finds the boundary bin,
//      the first (from the top) whose inclusive (count, cost) exceeds (B_max, tau);
//   3. only the boundary bin is ordered (rank sort by (key desc, id asc)) and walked: every
//      bin above it fits whole, so B*, bp and thr = fl(p * bp) follow;
//   4. Cd = {key >= thr} is compacted with its (len, id) keys, cost and fixed-point key, rank-
//      sorted by (len, id), scanned, and the first argmax window is taken.
// No full sort of S, and no pool gathers until the batch is written.
// --------------------------------------------------------------------------------------
#ifndef JIT_SPEC_THREADS
#define JIT_SPEC_THREADS 512
#endif
constexpr uint32_t kSpecThreads = JIT_SPEC_THREADS;
constexpr uint32_t kSpecWindow = 2048;        // |Cd| windowed in this CTA (larger: k_group)
constexpr uint32_t kSelCap = 2048;            // boundary-bin entries ordered in this CTA
constexpr uint32_t kSpecBins = 2048;
constexpr uint32_t kSpecBinShift = 43;        // 2^43 image units = 2^-9 relative (4 octaves over t)
static_assert(kSpecThreads * 4 == kSpecBins, "the boundary-bin scan gives every thread 4 bins");
// dynamic shared memory layout (bytes)
constexpr uint32_t kSpImgOff = 0;                                   // u64[kSpecCap]; later pc / pf
constexpr uint32_t kSpCostOff = kSpImgOff + 8 * kSpecCap;           // u32[kSpecCap]
constexpr uint32_t kSpHistOff = kSpCostOff + 4 * kSpecCap;          // u64[kSpecBins]
constexpr uint32_t kSpSelOff = kSpHistOff + 8 * kSpecBins;          // u32[kSelCap]
constexpr uint32_t kSpOrdOff = kSpSelOff + 4 * kSelCap;             // u32[max(kSelCap, kSpecWindow)]
constexpr uint32_t kSpWKeyOff = kSpOrdOff + 4 * kSpecWindow;        // u64[kSpecWindow] (len << 32 | id)
constexpr uint32_t kSpWFxOff = kSpWKeyOff + 8 * kSpecWindow;        // u64[kSpecWindow] fixed-point keys
constexpr uint32_t kSpWCostOff = kSpWFxOff + 8 * kSpecWindow;       // u32[kSpecWindow]
constexpr uint32_t kSpWIdxOff = kSpWCostOff + 4 * kSpecWindow;      // u32[kSpecWindow] entry of S
constexpr uint32_t kSpecSmem = kSpWIdxOff + 4 * kSpecWindow;
constexpr uint32_t kSpPcOff = 0;                                    // u64[kSpecWindow + 1] (over img)
constexpr uint32_t kSpPfOff = 8 * (kSpecWindow + 2);                // u128[kSpecWindow + 1]
static_assert(kSpPfOff + 16 * (kSpecWindow + 1) <= kSpCostOff, "prefix arrays must fit the image region");
static_assert(kSelCap <= kSpecWindow, "s_ord doubles as the boundary-bin order");
static_assert(kSpecSmem <= 227 * 1024, "k_spec shared memory");
// the boundary-bin ordering borrows the window arrays: (img, id) of the selected entries
static_assert(8 * kSelCap <= 8 * kSpecWindow && 4 * kSelCap <= 4 * kSpecWindow, "boundary scratch");

__device__ __forceinline__ uint32_t spec_bin(uint64_t img, uint64_t t_img) {
    const uint64_t d = (img - t_img) >> kSpecBinShift;          // img >= t_img for every entry
    return d >= kSpecBins - 1 ? kSpecBins - 1 : (uint32_t)d;
}
constexpr uint64_t kPackCount = 1ull << 48;   // histogram word: count << 48 | cost (cost sum < 2^48)

template <bool kBig>
static __device__ void spec_body(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, int reduce_only,
                                 unsigned char* smem, bool merged = false);
// the step's last kernel: resolve a small speculative set (the steady state), then publish the
// control block to pinned host memory.  Its code is kept small on purpose: it runs on one SM
// once per step, so every instruction-cache line it touches is a miss to L2 / HBM; a larger set
// is resolved by k_spec_big, which the host launches (status ST_SPEC_BIG).
// The control block lives in shared memory while k_spec runs: it starts as the reset block k_score
// wrote (built here before the dependency wait, so no global read-back) and is stored once at the
// end to the device copy and the pinned host mirror -- no load round trip on the tail.
// (now / v, word 1, are left as k_score wrote them: nothing reads them back.)
static_assert(offsetof(Ctrl, now) == 16 && offsetof(Ctrl, v) == 24, "ctrl word 1 = (now, v)");
__global__ void __launch_bounds__(kSpecThreads) k_spec(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int reduce_only,
                                                      int big_chain) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Ctrl s_ctrl;
    __shared__ uint32_t s_skip;
    reset_ctrl_block(&s_ctrl, 0, 0);
    pdl_wait();
    // a chained step after one that still needs the host (step_async): k_score did nothing, and
    // the control block of that step must survive for the host's path
    if (threadIdx.x == 0) s_skip = reduce_only ? 0u : S.persist->host_pending;
    __syncthreads();
    if (s_skip) return;
    spec_body<false>(P, c, &s_ctrl, S, reduce_only, smem);
    __syncthreads();
    if (threadIdx.x == 0 && !reduce_only) {
        const uint32_t st = s_ctrl.status;
        S.persist->host_pending = (st == ST_FALLBACK || (st == ST_SPEC_BIG && !big_chain) ||
                                   (st == ST_RESOLVED && !s_ctrl.window_done && !s_ctrl.error)) ? 1u : 0u;
    }
    for (uint32_t i = threadIdx.x; i < sizeof(Ctrl) / 16; i += blockDim.x) {
        if (i == 1) continue;
        const uint4 w = reinterpret_cast<const uint4*>(&s_ctrl)[i];
        reinterpret_cast<uint4*>(ctrl)[i] = w;
        reinterpret_cast<uint4*>(S.h_ctrl)[i] = w;
    }
}
__global__ void __launch_bounds__(kSpecThreads) k_spec_big(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    extern __shared__ __align__(16) unsigned char smem[];
    spec_body<true>(P, c, ctrl, S, 0, smem);
    publish_ctrl(ctrl, S.h_ctrl);
}
// the tail of a big-mode step graph (after k_spec_big_chain and k_group): whether the host still
// has work (exact path), then the control block to pinned host memory
__global__ void k_chain_publish(Ctrl* ctrl, Persist* ps, Ctrl* host) {
    if (threadIdx.x == 0) {
        const uint32_t st = ctrl->status;
        ps->host_pending = (st == ST_FALLBACK || st == ST_SPEC_BIG ||
                            (st == ST_RESOLVED && !ctrl->window_done && !ctrl->error)) ? 1u : 0u;
    }
    publish_ctrl(ctrl, host);
}
// The big-set resolve chained in the step graph (the handle's "big mode", chosen by the host when
// the speculative sets outgrow k_spec's fast path, e.g. C4): runs only when k_spec left
// ST_SPEC_BIG, so a step resolves on the device without a host round trip; else it returns.
// Followed by k_group (a large Cd's window) and k_chain_publish.
__global__ void __launch_bounds__(kSpecThreads) k_spec_big_chain(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_go;
    if (threadIdx.x == 0) s_go = ctrl->status == ST_SPEC_BIG;
    __syncthreads();
    if (!s_go) return;
    spec_body<true>(P, c, ctrl, S, 0, smem);             // host flag and publish: k_chain_publish
}

// ---- fast sharded step (the speculative variant): every rank scores its shard and
// exports its speculative set; after an allgather every rank resolves the union exactly like
// k_spec.  All ranks share the threshold t (they resolved the same previous step), so the union
// of the local sets {key >= t} IS the global speculative set and the exactness checks carry over
// with the global pending count.  Anything else (a set too large, a failed check) falls back to
// the exact two-round protocol (shard.cuh) without rescoring.
struct SpecHdr {                 // first 64 B of a rank's export
    uint32_t n_pending, n_dropped, err, refresh, n_set, rank, pad[10];
};
struct SpecRec {                 // 32 B per element
    unsigned long long img;
    uint32_t id, cost, len, row, meta, since;
};
constexpr uint32_t kSpecExportCap = 1024;        // records per rank
constexpr uint32_t kSpecExportBytes = 64 + 32 * kSpecExportCap;
static_assert(sizeof(SpecHdr) == 64 && sizeof(SpecRec) == 32, "export layout");

__global__ void __launch_bounds__(kSpecThreads) k_spec_export(Ctrl* ctrl, Scratch S, unsigned char* out, uint32_t rank) {
    const uint32_t tid = threadIdx.x;
    const uint32_t n_set = *reinterpret_cast<volatile unsigned int*>(S.spec_cnt);
    SpecRec* rec = reinterpret_cast<SpecRec*>(out + 64);
    for (uint32_t i = tid; i < kSpecExportCap; i += blockDim.x) {
        SpecRec q;
        if (i < n_set && n_set <= kSpecExportCap) {
            q.img = S.spec_img[i]; q.id = S.spec_id[i]; q.cost = S.spec_cost[i]; q.len = S.spec_len[i];
            q.row = S.spec_row[i]; q.meta = S.spec_meta[i]; q.since = S.spec_aux[i];
        } else {
            q.img = kNone; q.id = q.cost = q.len = q.row = q.meta = q.since = 0;
        }
        rec[i] = q;
    }
    __syncthreads();
    if (tid == 0) {
        BlockPart* g = S.gpart;
        SpecHdr hd{};
        const unsigned long long cnt = __ldcg(&g->cnt);
        hd.n_pending = (uint32_t)cnt; hd.n_dropped = (uint32_t)(cnt >> 32);
        hd.err = __ldcg(&g->err); hd.refresh = __ldcg(&g->refresh);
        hd.n_set = n_set; hd.rank = rank;
        *reinterpret_cast<SpecHdr*>(out) = hd;
        // this rank's own totals, as k_spec(reduce_only) would leave them for the exact protocol
        reset_ctrl(ctrl, ctrl->now, ctrl->v);
        ctrl->n_pending = hd.n_pending; ctrl->n_dropped = hd.n_dropped;
        ctrl->n_refresh = hd.refresh; ctrl->spec_n = n_set;
        if (hd.err) ctrl->error |= 1u;
        g->cnt = 0; g->err = 0; g->refresh = 0;
        *S.spec_cnt = 0;
    }
}

__global__ void __launch_bounds__(kSpecThreads) k_spec_merge(Pool P, Cfg c, Ctrl* ctrl, Scratch S, const unsigned char* all,
                                                             uint32_t world, uint32_t rank) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t m_off[65], m_pend, m_err, m_fb;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        uint32_t off = 0, pend = 0, err = 0, big = 0;
        for (uint32_t w = 0; w < world; ++w) {
            const SpecHdr* hd = reinterpret_cast<const SpecHdr*>(all + (size_t)w * kSpecExportBytes);
            m_off[w] = off;
            off += hd->n_set; pend += hd->n_pending; err |= hd->err; big |= hd->n_set > kSpecExportCap;
        }
        m_off[world] = off; m_pend = pend; m_err = err;
        // a rank whose own set overflowed its export, or nothing to resolve: the exact protocol
        m_fb = (err || pend == 0 || off == 0 || off > kSpecCap || big) ? 1u : 0u;
        ctrl->spec_n = off;
        if (m_fb) { ctrl->status = (err ? ST_ERROR : pend == 0 ? ST_EMPTY : ST_FALLBACK); if (err) ctrl->error |= 1u; }
    }
    __syncthreads();
    if (m_fb) { publish_ctrl(ctrl, S.h_ctrl); return; }
    if (m_off[world] > kSpecFast || c.chunk > kSpecFastChunk) {
        // a larger union: copy it into this handle's speculative-set arrays (another rank's rows
        // get row = ~0) and resolve it with k_spec_big's histogram path
        const uint32_t n = m_off[world];
        for (uint32_t i = tid; i < n; i += kSpecThreads) {
            uint32_t w = 0;
            while (m_off[w + 1] <= i) ++w;
            const SpecRec q = reinterpret_cast<const SpecRec*>(all + (size_t)w * kSpecExportBytes + 64)[i - m_off[w]];
            S.spec_img[i] = q.img; S.spec_id[i] = q.id; S.spec_cost[i] = q.cost; S.spec_len[i] = q.len;
            S.spec_row[i] = (w == rank) ? q.row : 0xFFFFFFFFu;
            S.spec_meta[i] = q.meta; S.spec_aux[i] = q.since;
        }
        if (tid == 0) { ctrl->n_pending = m_pend; ctrl->spec_n = n; }
        __syncthreads();
        spec_body<true>(P, c, ctrl, S, 0, smem, true);
        publish_ctrl(ctrl, S.h_ctrl);
        return;
    }
    // element tid of the union: rank w = the one whose range holds tid (ranks in order)
    SpecEl el{kNone, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    const uint32_t n = m_off[world];
    if (tid < n) {
        uint32_t w = 0;
        while (m_off[w + 1] <= tid) ++w;
        const SpecRec q = reinterpret_cast<const SpecRec*>(all + (size_t)w * kSpecExportBytes + 64)[tid - m_off[w]];
        el.img = q.img; el.id = q.id; el.cost = q.cost; el.len = q.len; el.row = q.row; el.meta = q.meta; el.since = q.since;
        el.own = (w == rank) ? 1u : 0u;
    }
    if (tid == 0) ctrl->n_pending = m_pend;
    spec_fast<kSpecThreads>(P, c, ctrl, S, n, n == m_pend, S.persist->t_guess, el, smem);
    publish_ctrl(ctrl, S.h_ctrl);
}

template <bool kBig>
static __device__ void spec_body(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, int reduce_only,
                                 unsigned char* smem, bool merged) {
    uint64_t* s_img = reinterpret_cast<uint64_t*>(smem + kSpImgOff);
    uint32_t* s_cost = reinterpret_cast<uint32_t*>(smem + kSpCostOff);
    unsigned long long* s_hist = reinterpret_cast<unsigned long long*>(smem + kSpHistOff);
    uint32_t* s_sel = reinterpret_cast<uint32_t*>(smem + kSpSelOff);
    uint32_t* s_ord = reinterpret_cast<uint32_t*>(smem + kSpOrdOff);
    uint64_t* w_key = reinterpret_cast<uint64_t*>(smem + kSpWKeyOff);
    uint64_t* w_fx = reinterpret_cast<uint64_t*>(smem + kSpWFxOff);
    uint32_t* w_cost = reinterpret_cast<uint32_t*>(smem + kSpWCostOff);
    uint32_t* w_idx = reinterpret_cast<uint32_t*>(smem + kSpWIdxOff);
    __shared__ uint64_t s_scan[32];
    __shared__ u128 s_scan128[32];
    __shared__ unsigned long long s_min, s_min_above, s_above;
    __shared__ uint32_t s_pend, s_drop, s_err, s_ref, s_n, s_first, s_nsel, s_ncd, s_fits;
    __shared__ uint64_t s_thr_img;
    __shared__ int s_fb;
    const uint32_t tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    stamp(ctrl, 0);
    const uint64_t t_img = S.persist->t_guess;
    // every load of this prologue is issued at once (one L2 round trip): the set size, each
    // thread's element of a small set -- loaded before the size is known, entries past it are
    // ignored (the workspace is zeroed at init) -- and, by thread 0, k_score's partials record
    const uint32_t n_set = kBig ? ctrl->spec_n : *reinterpret_cast<volatile unsigned int*>(S.spec_cnt);
    SpecEl el{kNone, 0u, 0u, 0u, 0u, 0u, 0u, 1u};
    if (!kBig && !reduce_only && tid < kSpecFast) {
        el.img = S.spec_img[tid]; el.id = S.spec_id[tid]; el.cost = S.spec_cost[tid]; el.len = S.spec_len[tid];
        el.row = S.spec_row[tid]; el.meta = S.spec_meta[tid]; el.since = S.spec_aux[tid];
    }
    if (tid == 0) {
        uint32_t pend, drop, err = 0, ref;
        if (kBig) {                                        // k_spec already reduced them into ctrl
            pend = ctrl->n_pending; drop = ctrl->n_dropped; ref = ctrl->n_refresh;
        } else {                                           // k_score's global record; reset for the next step
            BlockPart* g = S.gpart;
            const unsigned long long cnt = __ldcg(&g->cnt);
            pend = (uint32_t)cnt; drop = (uint32_t)(cnt >> 32);
            err = __ldcg(&g->err); ref = __ldcg(&g->refresh);
            g->cnt = 0; g->err = 0; g->refresh = 0;
        }
        s_pend = pend; s_drop = drop; s_err = err; s_ref = ref; s_min = kNone;
        s_n = n_set;
        s_first = kSpecBins; s_nsel = 0; s_ncd = 0; s_min_above = kNone; s_above = 0; s_fb = 0;
        ctrl->spec_n = n_set;
        ctrl->n_pending = pend; ctrl->n_dropped = drop; ctrl->n_refresh = ref;
        if (err) ctrl->error |= 1u;
    }
    if (kBig) for (uint32_t b = tid; b < kSpecBins; b += kSpecThreads) s_hist[b] = 0;
    __syncthreads();
    if (!kBig && tid == 0) *S.spec_cnt = 0;                // next step's set starts empty (all read it)
    const uint32_t n = s_n < kSpecCap ? s_n : kSpecCap;
    if (kBig) {                                            // (1) the set -> smem + histogram (+ its min key)
        uint64_t mn = kNone;
        for (uint32_t i = tid; i < n; i += kSpecThreads) {
            const uint64_t img = S.spec_img[i];
            const uint32_t cs = S.spec_cost[i];
            s_img[i] = img; s_cost[i] = cs;
            mn = img < mn ? img : mn;
            atomicAdd(&s_hist[spec_bin(img, t_img)], kPackCount | cs);
        }
        mn = warp_min_u64(mn);
        if (lane == 0 && mn != kNone) atomicMin(&s_min, (unsigned long long)mn);
        __syncthreads();
    }
    if (reduce_only) return;                               // sharded step: the radix path follows
    stamp(ctrl, 1);
    const uint32_t np = s_pend;
    const bool whole = (s_n == np);                        // S holds every pending row
    if (tid == 0) {
        if (s_err) { ctrl->status = ST_ERROR; s_fb = 2; }
        else if (np == 0) { ctrl->status = ST_EMPTY; s_fb = 2; }
        else if (s_n > kSpecCap || s_n == 0) spec_fallback(ctrl, &s_fb);
    }
    __syncthreads();
    if (s_fb) return;                                      // published as is (k_spec)
    if constexpr (!kBig) {
        if (n <= kSpecFast && c.chunk <= kSpecFastChunk)
            spec_fast<kSpecThreads>(P, c, ctrl, S, n, whole, t_img, el, smem);
        else if (tid == 0) ctrl->status = ST_SPEC_BIG;     // the host launches k_spec_big
        return;
    }
    // (2) boundary bin: thread t owns bins [2047 - 4t - 3, 2047 - 4t], scanned from the top
    {
        uint64_t h[4], loc = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) { h[k] = s_hist[kSpecBins - 1 - 4 * tid - k]; loc += h[k]; }
        uint64_t tot;
        uint64_t run = block_exclusive_scan_u64(loc, s_scan, &tot);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t inc = run + h[k];
            if ((inc >> 48) > c.max_batch || (inc & (kPackCount - 1)) > c.token_budget) {
                atomicMin(&s_first, 4 * tid + k);
                break;
            }
            run = inc;
        }
        __syncthreads();
        // the owner of the boundary bin publishes what lies above it (its loop stopped there,
        // so run is the exclusive (count, cost) of that bin)
        const uint32_t f = s_first;
        if (f < kSpecBins && f / 4 == tid) s_above = run;
    }
    __syncthreads();
    stamp(ctrl, 2);
    const uint32_t first = s_first;
    if (first == kSpecBins) {
        // every entry of S fits the budget: exact only if S is the whole pending set
        if (tid == 0) {
            if (!whole) spec_fallback(ctrl, &s_fb);
            else {
                s_fits = n;
                const double bp = __longlong_as_double((long long)s_min);
                const double thr = __dmul_rn(c.p, bp);
                ctrl->b_star = n; ctrl->bp = bp; ctrl->thr = thr;
                ctrl->thr_img = s_thr_img = (uint64_t)__double_as_longlong(thr);
            }
        }
        __syncthreads();
        if (s_fb) return;
    } else {
        // (3) gather the boundary bin; min key image of the bins above it
        const uint32_t bbin = kSpecBins - 1 - first;
        uint64_t mn_above = kNone;
        for (uint32_t i = tid; i < n; i += kSpecThreads) {
            const uint64_t img = s_img[i];
            const uint32_t b = spec_bin(img, t_img);
            if (b == bbin) {
                const uint32_t slot = atomicAdd(&s_nsel, 1u);
                if (slot < kSelCap) s_sel[slot] = i;
            } else if (b > bbin && img < mn_above) {
                mn_above = img;
            }
        }
        mn_above = warp_min_u64(mn_above);
        if (lane == 0 && mn_above != kNone) atomicMin(&s_min_above, (unsigned long long)mn_above);
        __syncthreads();
        const uint32_t m = s_nsel;
        if (m > kSelCap) {                                 // a huge tie bin: exact path
            if (tid == 0) spec_fallback(ctrl, &s_fb);
            __syncthreads();
            return;
        }
        // order the boundary bin by (key desc, id asc) = composite key ascending (unique):
        // s_ord[rank] = j (index into s_sel).  Rank sort when small, bitonic otherwise.
        u128* b_ck = reinterpret_cast<u128*>(w_key);       // w_key + w_fx: 16 * kSelCap bytes, free until (4)
        static_assert(16 * kSelCap <= kSpWCostOff - kSpWKeyOff, "boundary keys fit w_key + w_fx");
        uint32_t m2 = 1;
        while (m2 < m) m2 <<= 1;
        for (uint32_t j = tid; j < m2; j += kSpecThreads) {
            if (j < m) { const uint32_t e = s_sel[j]; b_ck[j] = make_ck(s_img[e], S.spec_id[e]); }
            else b_ck[j] = ~(u128)0;
            s_ord[j] = j;
        }
        __syncthreads();
        if (m <= kSpecThreads) {
            uint32_t rank = 0, j = tid;
            u128 kj = 0;
            if (j < m) { kj = b_ck[j]; for (uint32_t q = 0; q < m; ++q) rank += b_ck[q] < kj; }
            __syncthreads();
            if (j < m) s_ord[rank] = j;
        } else {
            block_sort<u128>(b_ck, s_ord, m2);
        }
        __syncthreads();
        // walk the boundary bin (warp 0): the prefix through rank k fits while
        // above_count + k + 1 <= B_max and above_cost + cost(rank <= k) <= tau
        if (wid == 0) {
            const uint64_t above = s_above;
            const uint64_t a_cnt = above >> 48, a_cost = above & (kPackCount - 1);
            const uint32_t per = (m + 31) / 32, r0 = lane * per;
            uint64_t loc = 0;
            for (uint32_t k = 0; k < per; ++k) if (r0 + k < m) loc += s_cost[s_sel[s_ord[r0 + k]]];
            uint64_t inc = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint64_t run = inc - loc;
            uint32_t fit = 0;
            for (uint32_t k = 0; k < per; ++k) {
                const uint32_t r = r0 + k;
                if (r >= m) break;
                run += s_cost[s_sel[s_ord[r]]];
                if (a_cnt + r + 1 <= c.max_batch && a_cost + run <= c.token_budget) ++fit;   // monotone
            }
            fit = warp_sum(fit);
            if (lane == 0) {
                const uint32_t fits = (uint32_t)a_cnt + fit;
                const uint64_t bimg = fit ? s_img[s_sel[s_ord[fit - 1]]] : (uint64_t)s_min_above;
                if (fits == 0 || bimg == kNone) {
                    ctrl->error |= 1u; ctrl->status = ST_ERROR; s_fb = 2;
                } else {
                    const double bp = __longlong_as_double((long long)bimg);
                    const double thr = __dmul_rn(c.p, bp);
                    const uint64_t ti = (uint64_t)__double_as_longlong(thr);
                    if (!whole && ti < t_img) spec_fallback(ctrl, &s_fb);
                    else { ctrl->b_star = fits; ctrl->bp = bp; ctrl->thr = thr; ctrl->thr_img = s_thr_img = ti; }
                }
            }
        }
        __syncthreads();
        if (s_fb) return;
    }
    stamp(ctrl, 3);
    // (4) Cd = {key >= thr}: compact with its window key (len, id), cost, fixed-point key
    const uint64_t thr_img = s_thr_img;
    for (uint32_t i = tid; i < n; i += kSpecThreads) {
        const uint64_t img = s_img[i];
        if (img >= thr_img) {
            const uint32_t slot = atomicAdd(&s_ncd, 1u);
            if (slot < kSpecWindow) {
                w_key[slot] = ((uint64_t)S.spec_len[i] << 32) | S.spec_id[i];   // (len asc, id asc) A17/A18
                w_fx[slot] = fixed_point(__longlong_as_double((long long)img));
                w_cost[slot] = s_cost[i];
                w_idx[slot] = i;
            }
        }
    }
    __syncthreads();
    const uint32_t ncd = s_ncd;
    if (tid == 0) { ctrl->n_cand = ncd; ctrl->status = ST_RESOLVED; }
    if (ncd > kSpecWindow && merged) {                     // a sharded union: the exact protocol takes over
        if (tid == 0) { ctrl->status = ST_FALLBACK; ctrl->fallback = 1; }
        return;
    }
    if (ncd > kSpecWindow) {
        // a large Cd: hand it to k_group (launched from here)
        if (tid == 0) s_nsel = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kSpecThreads)
            if (s_img[i] >= thr_img) {                     // k_group reads the Cd rows' key and cost
                const uint32_t r = S.spec_row[i];
                S.cand[atomicAdd(&s_nsel, 1u)] = r;
                P.img[r] = s_img[i]; P.cost[r] = s_cost[i];
            }
        __syncthreads();
        return;                                            // window_done = 0: the host runs k_group
    }
    stamp(ctrl, 4);
    // (a9) sort Cd by (len, id) (keys unique): s_ord[rank] = slot.  Rank sort when small,
    // bitonic on a copy in the (now free) image region otherwise.
    if (ncd <= kSpecThreads) {
        uint32_t rank = 0;
        if (tid < ncd) { const uint64_t kj = w_key[tid]; for (uint32_t q = 0; q < ncd; ++q) rank += w_key[q] < kj; }
        if (tid < ncd) s_ord[rank] = tid;
    } else {
        uint64_t* sk = reinterpret_cast<uint64_t*>(smem + kSpImgOff);
        uint32_t n2 = 1;
        while (n2 < ncd) n2 <<= 1;
        for (uint32_t j = tid; j < n2; j += kSpecThreads) { sk[j] = j < ncd ? w_key[j] : ~0ull; s_ord[j] = j; }
        __syncthreads();
        block_sort<uint64_t>(sk, s_ord, n2);
    }
    __syncthreads();
    stamp(ctrl, 5);
    // prefix sums in window order (the image region is free now): pc u64, pf u128, n+1 each
    unsigned long long* pc = reinterpret_cast<unsigned long long*>(smem + kSpPcOff);
    u128* pf = reinterpret_cast<u128*>(smem + kSpPfOff);
    {
        const uint32_t per = (ncd + kSpecThreads - 1) / kSpecThreads, r0 = tid * per;
        uint64_t lc = 0;
        u128 lf = 0;
        for (uint32_t k = 0; k < per; ++k)
            if (r0 + k < ncd) { const uint32_t j = s_ord[r0 + k]; lc += w_cost[j]; lf += (u128)w_fx[j]; }
        uint64_t tc;
        u128 tf;
        uint64_t ec = block_exclusive_scan_u64(lc, s_scan, &tc);
        u128 ef = block_exclusive_scan_u128(lf, s_scan128, &tf);
        for (uint32_t k = 0; k < per; ++k) {
            const uint32_t r = r0 + k;
            if (r >= ncd) break;
            const uint32_t j = s_ord[r];
            pc[r] = ec; pf[r] = ef;
            ec += w_cost[j]; ef += (u128)w_fx[j];
        }
        if (tid == 0) { pc[ncd] = tc; pf[ncd] = tf; }
    }
    __syncthreads();
    stamp(ctrl, 6);
    // first argmax over i of the window [i, j(i)] (j(i): largest end within tau and B_max)
    __shared__ u128 s_best[32];
    __shared__ uint32_t s_bi[32], s_bj[32];
    {
        u128 best = 0;
        uint32_t bi = 0xFFFFFFFFu, bj = 0;
        for (uint32_t i = tid; i < ncd; i += kSpecThreads) {
            const uint64_t lim = (uint64_t)pc[i] + c.token_budget;
            uint32_t lo = i, hi = (uint32_t)min((uint64_t)ncd - 1, (uint64_t)i + c.max_batch - 1);
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (pc[mid + 1] <= lim) lo = mid; else hi = mid - 1;
            }
            const u128 sc = pf[lo + 1] - pf[i];
            if (bi == 0xFFFFFFFFu || sc > best) { best = sc; bi = i; bj = lo; }   // i increasing per thread
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u128 ob = shfl_xor_u128(best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
        }
        if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; s_bj[wid] = bj; }
        __syncthreads();
        if (wid == 0) {
            constexpr int nw = kSpecThreads / 32;
            best = lane < nw ? s_best[lane] : (u128)0; bi = lane < nw ? s_bi[lane] : 0xFFFFFFFFu; bj = lane < nw ? s_bj[lane] : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const u128 ob = shfl_xor_u128(best, o);
                const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
            }
            if (lane == 0) { s_bi[0] = bi; s_bj[0] = bj; }
        }
        __syncthreads();
    }
    const uint32_t bi = s_bi[0], bj = s_bj[0];
    stamp(ctrl, 7);
    // the batch and its bookkeeping: ever_scheduled, Running, the steps_waited stamp
    const uint32_t ns = bj - bi + 1;
    const uint32_t sc = S.persist->steps;
    __syncthreads();
    for (uint32_t k = tid; k < ns; k += kSpecThreads) {
        const uint32_t j = s_ord[bi + k];
        const uint32_t e = w_idx[j];
        const uint32_t r = S.spec_row[e];
        S.out_ids[k] = (uint32_t)w_key[j];
        S.out_tokens[k] = w_cost[j];
        S.out_rows[k] = r;
        if (r == 0xFFFFFFFFu) continue;                     // another rank's request (sharded union)
        book_selected(P, r, S.spec_meta[e], S.spec_aux[e], sc);
    }
    if (tid == 0) {
        ctrl->n_selected = ns;
        ctrl->total_tokens = (uint32_t)(pc[bj + 1] - pc[bi]);
        ctrl->i_best = bi; ctrl->j_best = bj;
        ctrl->window_done = 1;
        finish_counters(S.persist, ctrl);               // next step's threshold: this cutoff with a 3% margin
    }
    stamp(ctrl, 8);
}
#endif  // JIT_EXACT_TU

}  // namespace jit
