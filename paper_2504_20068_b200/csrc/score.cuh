// score.cuh -- the streaming pass over the pool (a1)-(a6) and the speculative resolve.
//
//   k_score  every row: persistent 128-thread CTAs (6 per SM) walk 256-row work items whose
//            SoA slices are staged into a shared-memory ring by bulk (TMA 1-D) copies, kRPT = 2
//            consecutive rows per thread; standalone rows get their key image (a5) and cost
//            (a6); compound calls are scored by CTAs that own whole tasks, so the task aggregate
//            (a4) and the calls' keys come out of the same pass (shared-memory sums, no global
//            atomics).  Per-CTA partial counts are reduced in the CTA and added once into a
//            global record.
//   k_spec   one CTA: exact B*, bp, thr, Cd and the window from the speculative set.
#pragma once
#include "select.cuh"

namespace jit {

// Rows whose key image is >= the speculative threshold t (the previous step's cutoff with a
// margin) join the speculative set; warp ballot + one atomic per warp (all lanes convergent).
// The entry carries everything the resolve needs (key image, id, row, cost, window length, and
// the row's meta / aux as this pass left them), so k_spec needs no dependent loads.
__device__ __forceinline__ void spec_add(const Scratch& S, const uint32_t* ids, bool valid, uint64_t img,
                                         uint32_t row, uint32_t cost, uint32_t len, uint32_t meta, uint32_t aux,
                                         uint64_t t) {
    const bool take = valid && img >= t;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(S.spec_cnt, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) {
        const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
        if (slot < kSpecCap) {
            S.spec_img[slot] = img; S.spec_id[slot] = __ldg(ids + row); S.spec_row[slot] = row;
            S.spec_cost[slot] = cost; S.spec_len[slot] = len; S.spec_meta[slot] = meta; S.spec_aux[slot] = aux;
        }
    }
}

// block reduction of the per-thread partials, then one set of atomics per CTA into the step's
// global accumulator (read and reset by k_spec: a single record instead of one per CTA)
__device__ __forceinline__ void store_part(BlockPart* gpart, uint32_t pend, uint32_t drop, uint32_t err,
                                           uint64_t mn, uint64_t cost, uint32_t refresh) {
    __shared__ unsigned long long s_min, s_cost;
    __shared__ uint32_t s_pend, s_drop, s_err, s_ref;
    if (threadIdx.x == 0) { s_min = kNone; s_cost = 0; s_pend = 0; s_drop = 0; s_err = 0; s_ref = 0; }
    __syncthreads();
    pend = warp_sum(pend); drop = warp_sum(drop); err = __reduce_or_sync(0xffffffffu, err);
    mn = warp_min_u64(mn); cost = warp_sum(cost); refresh = warp_sum(refresh);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_pend, pend); atomicAdd(&s_drop, drop); atomicOr(&s_err, err); atomicAdd(&s_ref, refresh);
        atomicMin(&s_min, (unsigned long long)mn); atomicAdd(&s_cost, (unsigned long long)cost);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_min != kNone) atomicMin(&gpart->min_img, s_min);
        if (s_cost) atomicAdd(&gpart->tot_cost, s_cost);
        if (s_pend) atomicAdd(&gpart->n_pending, s_pend);
        if (s_drop) atomicAdd(&gpart->n_dropped, s_drop);
        if (s_err) atomicOr(&gpart->err, s_err);
        if (s_ref) atomicAdd(&gpart->refresh, s_ref);
    }
}

// Per-row scoring of the pool pass, written branch-light (the length-bound refresh is the only
// real branch; rows that are not pending compute and discard).  Group / table / flag ranges were
// validated at load (k_validate) and the device never changes them.
struct RowOut {
    uint64_t img;
    uint32_t cost, aux, Lh, len_rem;
    bool err;
};

// standalone request, after (a1) admission and (a2) the bound refresh: (a3) t_rem, (a5) key,
// (a6) cost, steps_waited+1.  Rows that are not pending compute and discard.
template <bool kDebug, bool kAppB>
__device__ __forceinline__ void row_std(const Cfg& c, const GroupFast* sg, const uint32_t* ovr, uint32_t row,
                                        bool pend, int64_t now, int64_t v, double v_d, double eps_d, int64_t arr,
                                        uint32_t L_i, uint32_t g, uint32_t pre, uint32_t lhat, uint32_t meta,
                                        uint32_t aux, RowOut& o, double& d_rate, int64_t& d_trem) {
    const uint32_t Lh = max(lhat, g + 1);
    const uint32_t len_rem = Lh - g;
    const GroupFast G = sg[pend ? m_group(meta) : 0u];      // rows outside the item: any valid group
    const int64_t trem = arr + G.base + (int64_t)(Lh - 1) * G.tok - now;             // (a3), A9
    uint64_t Gk = (uint64_t)G.w_in_eff * L_i + (uint64_t)G.w_out_eff * Lh;          // (a5) A10/A11
    if (m_flags(meta) & kOverride) Gk = __ldg(ovr + row);
    if (trem <= 0) Gk = 0;                                                          // A22
    if (kAppB && (uint64_t)len_rem * (uint64_t)v > (uint64_t)(trem > 0 ? trem : 0)) Gk = 0;   // App. B filter
    const uint64_t Gp = Gk + (uint64_t)c.delta * fastdiv(aux >> 16, c.frame, c.F_m, c.F_l);
    double key;
    const bool ok = make_key_lv(Gp, len_rem, v_d, eps_d, &key);
    o.err = pend && !ok;
    o.img = (pend && ok) ? (uint64_t)__double_as_longlong(key) : kNone;
    o.cost = pend ? token_cost(L_i, pre, c.chunk) : 0u;
    o.aux = (pend && (aux >> 16) < 0xFFFFu) ? aux + (1u << 16) : aux;   // steps_waited+1; undone if selected
    o.Lh = Lh; o.len_rem = len_rem;
    if (kDebug) { d_rate = pend ? make_rate(len_rem, trem) : 0.0; d_trem = pend ? trem : 0; }
}

// 64-bit shared-memory sum of a value < 2^32 with 32-bit atomics (a 64-bit shared atomicAdd is a
// CAS loop on sm_100): add to the low word, carry into the high word on wrap-around
__device__ __forceinline__ void smem_add64(unsigned long long* p, uint32_t x) {
    uint32_t* w = reinterpret_cast<uint32_t*>(p);
    const uint32_t old = atomicAdd(w, x);
    if (old + x < old) atomicAdd(w + 1, 1u);
}

__device__ __forceinline__ bool is_frames_tag(uint64_t img) {
    return (img & 0xFFF8000000000000ull) == kFramesTag;
}

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
#ifndef JIT_SPEC_BUCKET
#define JIT_SPEC_BUCKET 0              // 1: small-set ranks by a counting sort on the key image
#endif
constexpr uint32_t kFB = 1024;         // JIT_SPEC_BUCKET bins: 128 per octave of the key above t
constexpr uint32_t kFBShift = 45;
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
    uint32_t id, cost, len, row, meta, aux;
    uint32_t own;               // 1: the row belongs to this handle (a sharded step merges all ranks' sets)
};
template <uint32_t NT>
static __device__ __forceinline__ void spec_fast(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t n,
                                              bool whole, uint64_t t_img, uint64_t min_img, const SpecEl& el,
                                              unsigned char* smem) {
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
    const uint64_t img = own ? el.img : kNone;
    const uint32_t id = el.id, cost = own ? el.cost : 0u, len = el.len;
    __shared__ uint32_t f_rank2[kSpecFast];
    __shared__ uint32_t f_pre2[kSpecFast];
    if (own) {
        f_rec[tid] = rank_rec(img, id, cost);
        f_img[tid] = img; f_id[tid] = id; f_cost[tid] = cost;
        f_rank2[tid] = 0; f_pre2[tid] = 0;
    }
#if JIT_SPEC_BUCKET
    __shared__ unsigned long long f_h[kFB + 1];           // per bin: count << 32 | cost; then the prefix
    __shared__ uint4 f_srt[kSpecFast];                     // rank records grouped by bin
    __shared__ uint64_t f_bscan[32];
    for (uint32_t i = tid; i <= kFB; i += NT) f_h[i] = 0ull;
#endif
    __syncthreads();
    stamp(ctrl, 2);
#if JIT_SPEC_BUCKET
    // (a7) rank and cost prefix via a counting sort on the key image: bins of 2^-7 relative width
    // above t (the top bin open-ended) in priority order (rb = 0: the highest keys); an element's
    // rank / prefix = the bins before its own (one block scan) + the elements of its own bin
    // that precede it (one 96-bit comparison each)
    {
        uint32_t rb = 0, slot = 0;
        if (own) {
            const uint64_t d = img > t_img ? (img - t_img) >> kFBShift : 0ull;
            rb = kFB - 1u - (uint32_t)(d >= kFB - 1u ? kFB - 1u : d);
            slot = (uint32_t)(atomicAdd(&f_h[rb], (1ull << 32) | cost) >> 32);
        }
        __syncthreads();
        static_assert(kFB % NT == 0, "bins per thread");
        constexpr uint32_t kPer = kFB / NT;                // bins per thread
        unsigned long long loc[kPer], v = 0;
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) { loc[k] = f_h[tid * kPer + k]; v += loc[k]; }
        unsigned long long tot;
        unsigned long long base = block_exclusive_scan_u64(v, f_bscan, reinterpret_cast<uint64_t*>(&tot));
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) { f_h[tid * kPer + k] = base; base += loc[k]; }
        if (tid == 0) f_h[kFB] = tot;
        __syncthreads();
        const uint4 me = own ? f_rec[tid] : make_uint4(0u, 0u, 0u, 0u);
        const unsigned long long b0 = own ? f_h[rb] : 0ull;
        const uint32_t lo = (uint32_t)(b0 >> 32), hi = own ? (uint32_t)(f_h[rb + 1] >> 32) : 0u;
        if (own) f_srt[lo + slot] = me;
        __syncthreads();
        uint32_t ra = lo, pa = (uint32_t)b0;
        for (uint32_t j = lo; j < hi; ++j) {
            const uint4 q = f_srt[j];
            const uint32_t bm = before_mask(q, me);
            ra -= bm; pa += bm * q.w;
        }
        if (own) { f_rank2[tid] = ra; f_pre2[tid] = pa; }
    }
#else
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
#endif
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
        else {                                          // is the whole pending set (bp = min key)
            bp = __longlong_as_double((long long)(bstar == n ? min_img : bp_img));
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
    __shared__ uint32_t f_row[kSpecFast], f_meta[kSpecFast], f_aux[kSpecFast];
    if (own) { f_row[tid] = el.own ? el.row : 0xFFFFFFFFu; f_meta[tid] = el.meta; f_aux[tid] = el.aux; }
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
    // the batch in window order and its bookkeeping: ever_scheduled, Running, undo steps_waited+1
    const uint32_t ns = bj - bi + 1;
    if (tid < ns) {
        const uint32_t e = o_elem[bi + tid];
        const uint32_t r = f_row[e];
        S.out_ids[tid] = f_id[e];
        S.out_tokens[tid] = f_cost[e];
        S.out_rows[tid] = r;
        const uint32_t B = c.max_batch + 1;                 // and the pinned host mirror (no D2H copy)
        S.h_batch[tid] = f_id[e]; S.h_batch[B + tid] = f_cost[e]; S.h_batch[2 * B + tid] = r;
        if (r != 0xFFFFFFFFu) {                             // bookkeeping of this handle's rows
            uint32_t mt = f_meta[e] | (kEver << 12);        // meta / aux as k_score left them (preloaded)
            if (m_state(mt) == kQueued || m_state(mt) == kPreempted) mt = m_with_state(mt, kRunning);
            P.meta[r] = mt;
            const uint32_t aux = f_aux[e];
            if ((aux >> 16) < 0xFFFFu) P.aux[r] = aux - (1u << 16);
        }
    }
    if (tid == 0) {
        ctrl->n_selected = ns;
        ctrl->total_tokens = (uint32_t)(pc[bj + 1] - pc[bi]);
        ctrl->i_best = bi; ctrl->j_best = bj;
        ctrl->window_done = 1; ctrl->batch_on_host = 1;
        // next step's speculative threshold: this step's cutoff with a 15% margin
        Persist* ps = S.persist;
        ps->t_guess = (unsigned long long)__double_as_longlong(__dmul_rn(ctrl->thr, 0.85));
        ps->steps += 1;
    }
    stamp(ctrl, 7);
}

// k_score: the hot pass, compiled into abi.cu (whole-program mode: -rdc costs the scoring loop
// registers).  Persistent CTAs walk work items of at most kTile rows; the next item's hot state
// streams into shared memory through bulk asynchronous copies (TMA 1D, mbarrier completion)
// while the current one is scored, kRPT consecutive rows per thread (vector shared loads and
// vector global stores of key image, cost and steps_waited).
//   * standalone items: tile i = rows [kTile i, kTile i + kTile) of [0, n_single) -- (a1)-(a3),
//     (a5), (a6) per row;
//   * compound items: one CRange of whole tasks each (a4): phase A scores the calls and sums
//     (len_rem, call goodput) per task in shared memory, phase B turns the sums into the task's
//     goodput and t_gen (one thread per task), phase C keys every pending call
//     (G_task + delta * frames) * 1e9 / (t_gen + eps) from registers -- no global atomics, no
//     second kernel.  A range wider than one tile (a single task > kTile calls) is read from
//     global memory and parks the frame count in the key slot between A and C.
// Every row whose key image reaches the speculative threshold joins the speculative set; per-CTA
// partial counts are reduced per CTA, then added atomically into one global record.
// --------------------------------------------------------------------------------------
#ifndef JIT_EXACT_TU
#ifndef JIT_ITEM_SNAKE
#define JIT_ITEM_SNAKE 1
#endif
#ifndef JIT_SCORE_MINB
#define JIT_SCORE_MINB 6
#endif
struct Acc {
    uint32_t pend, drop, err, ref;
    uint64_t mn;                   // smallest key image (compound path)
    uint32_t cost;                 // per thread: <= (rows per thread) x chunk, far below 2^32
    double mn_d;                   // smallest key (standalone path; keys >= 0 order like their images)
};

// kRPT consecutive rows per thread: vector loads / stores of kRPT fields (64- or 128-bit)
__device__ __forceinline__ void ld_rows(const uint32_t* p, uint32_t* v) {
    if constexpr (kRPT == 4) { const uint4 t = *reinterpret_cast<const uint4*>(p); v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
    else if constexpr (kRPT == 2) { const uint2 t = *reinterpret_cast<const uint2*>(p); v[0] = t.x; v[1] = t.y; }
    else v[0] = *p;
}
__device__ __forceinline__ void ld_rows64(const int64_t* p, int64_t* v) {
    if constexpr (kRPT >= 2) {
        const longlong2 a = *reinterpret_cast<const longlong2*>(p);
        v[0] = a.x; v[1] = a.y;
    } else {
        v[0] = *p;
    }
    if constexpr (kRPT == 4) { const longlong2 b = *reinterpret_cast<const longlong2*>(p + 2); v[2] = b.x; v[3] = b.y; }
}
// per-row outputs: streaming stores (cache-streaming: evict-first in L2)
__device__ __forceinline__ void st_rows(uint32_t* p, const uint32_t* v) {
    if constexpr (kRPT == 4) __stcs(reinterpret_cast<uint4*>(p), make_uint4(v[0], v[1], v[2], v[3]));
    else if constexpr (kRPT == 2) __stcs(reinterpret_cast<uint2*>(p), make_uint2(v[0], v[1]));
    else __stcs(p, v[0]);
}
__device__ __forceinline__ void st_rows64(uint64_t* p, const uint64_t* v) {
    if constexpr (kRPT >= 2) __stcs(reinterpret_cast<ulonglong2*>(p), make_ulonglong2(v[0], v[1]));
    else __stcs(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v[0]);
    if constexpr (kRPT == 4) __stcs(reinterpret_cast<ulonglong2*>(p) + 1, make_ulonglong2(v[2], v[3]));
}

// the 32-B hot state of rows q0..q0+kRPT-1 (q0 % kRPT == 0; the SoA capacity is padded to 64 rows)
struct Quad {
    int64_t ar[kRPT];
    uint32_t li[kRPT], ge[kRPT], pr[kRPT], lh[kRPT], me[kRPT], ax[kRPT];
};
__device__ __forceinline__ void load_quad(const Pool& P, uint32_t q0, Quad& Q) {
    ld_rows64(P.arr + q0, Q.ar);
    ld_rows(P.len_in + q0, Q.li); ld_rows(P.gen + q0, Q.ge); ld_rows(P.pre + q0, Q.pr);
    ld_rows(P.lhat + q0, Q.lh); ld_rows(P.meta + q0, Q.me); ld_rows(P.aux + q0, Q.ax);
}
__device__ __forceinline__ void zero_quad(Quad& Q) {
#pragma unroll
    for (int k = 0; k < (int)kRPT; ++k) { Q.ar[k] = 0; Q.li[k] = Q.ge[k] = Q.pr[k] = Q.lh[k] = Q.me[k] = Q.ax[k] = 0; }
}

// One staged tile: kTile rows starting at a 16-byte aligned row (r0 & ~3), one array per SoA
// field, filled by bulk asynchronous copies (cp.async.bulk, the 1D TMA path) that complete on an
// mbarrier; compound items also stage the constants of their first kTaskStage tasks.  A ring
// of kStages such buffers per CTA keeps kStages - 1 items in flight while one is scored.
#ifndef JIT_STAGES
#define JIT_STAGES 2
#endif
constexpr uint32_t kStages = JIT_STAGES;
#ifndef JIT_TASK_STAGE
#define JIT_TASK_STAGE 64
#endif
constexpr uint32_t kTaskStage = JIT_TASK_STAGE;
struct TileBuf {
    int64_t ar[kTile];
    uint32_t li[kTile], ge[kTile], pr[kTile], lh[kTile], me[kTile], ax[kTile], tk[kTile];
    TaskInfo ti[kTaskStage];
};
__device__ __forceinline__ void load_quad_smem(const TileBuf* B, uint32_t o, Quad& Q, uint32_t* tk) {
    ld_rows64(B->ar + o, Q.ar);
    ld_rows(B->li + o, Q.li); ld_rows(B->ge + o, Q.ge); ld_rows(B->pr + o, Q.pr);
    ld_rows(B->lh + o, Q.lh); ld_rows(B->me + o, Q.me); ld_rows(B->ax + o, Q.ax);
    if (tk) ld_rows(B->tk + o, tk);
}

// --- mbarrier + bulk copy (PTX; sm_90+) ---
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// The pool streams through L2 once per step: its bulk reads carry an evict-first policy so that
// what is reused every step (code, tables, partials, the speculative set) keeps its L2 lines
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(evict_first_policy()) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Bounded wait: a phase that never completes (a bulk copy that faulted, a protocol bug) traps
// after ~2^26 hardware-suspended probes instead of hanging the GPU.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
#ifdef JIT_MBAR_HINT
    // suspend (not spin) until the phase completes or the hint (ns) expires
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity), "n"(JIT_MBAR_HINT) : "memory");
#else
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
#endif
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t tries = 0;
    while (!mbar_try(bar, parity))
        if (++tries == (1u << 26)) __trap();
}

// standalone rows q0..q0+kRPT-1 (those < n_single)
template <bool kDebug, bool kAppB>
__device__ __forceinline__ void std_quad(const Pool& P, const Table& T, const GroupFast* s_g, const Cfg& c,
                                         const Scratch& S, int64_t now, int64_t v, uint64_t t_guess, uint32_t q0,
                                         uint32_t ns, const TileBuf* B, uint32_t o, uint64_t* empty, Acc& A) {
    const bool any = q0 < ns, full = q0 + kRPT - 1 < ns;
    const double v_d = (double)v, eps_d = (double)c.eps;
    Quad Q;
    if (any) load_quad_smem(B, o, Q, nullptr);
    else zero_quad(Q);
    mbar_arrive(empty);                                    // this thread is done with the tile buffer
#ifdef JIT_SCORE_FLOOR
    {   // timing experiment only (profiles/variants.sh): the memory pipeline without the row math
        uint64_t img[kRPT];
        uint32_t cost[kRPT], aux[kRPT];
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) {
            img[k] = (uint64_t)Q.ar[k] ^ Q.li[k] ^ Q.ge[k]; cost[k] = Q.pr[k] ^ Q.lh[k]; aux[k] = Q.me[k] ^ Q.ax[k];
        }
        if (full) { st_rows64(P.img + q0, img); st_rows(P.cost + q0, cost); st_rows(P.aux + q0, aux); }
        return;
    }
#endif
    // (a1) admission and pending, (a2) which cached bounds are stale
    const int64_t drop_before = now - c.waiting;           // now - arrival > waiting <=> arrival < now - waiting
    bool pend[kRPT], drop[kRPT], need[kRPT];
    uint32_t ep[kRPT];
    bool any_need = false, any_drop = false;
#pragma unroll
    for (int k = 0; k < (int)kRPT; ++k) {
        const uint32_t st = m_state(Q.me[k]), fl = m_flags(Q.me[k]);
        const bool arrived = q0 + k < ns && Q.ar[k] <= now;
        drop[k] = arrived && st == kQueued && !(fl & (kEver | kCompound)) && Q.ar[k] < drop_before;
        pend[k] = arrived && !drop[k] && st <= kPreempted;
        ep[k] = fastdiv(Q.ge[k], c.R, c.R_m, c.R_l);
        need[k] = pend[k] && (Q.lh[k] == 0 || ep[k] >= 65536u || m_epoch(Q.me[k]) != ep[k]);
        any_need |= need[k]; any_drop |= drop[k];
    }
    if (__any_sync(0xffffffffu, any_need)) {              // rare in steady state: refresh off the main path
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) {
            if (need[k]) {
                Q.lh[k] = cond_quantile(T, Q.ax[k] & 0xFFFFu, ep[k] * c.R, c.qn, c.qd);
                P.lhat[q0 + k] = Q.lh[k];
                if (ep[k] < 65536u) { Q.me[k] = (Q.me[k] & 0xFFFFu) | (ep[k] << 16); P.meta[q0 + k] = Q.me[k]; }
                A.ref += 1;
            }
        }
    }
    if (any_drop) {
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k)
            if (drop[k]) { P.meta[q0 + k] = m_with_state(Q.me[k], kDropped); A.drop += 1; }
    }
    uint64_t img[kRPT];
    uint32_t cost[kRPT], aux[kRPT];
#pragma unroll
    for (int k = 0; k < (int)kRPT; ++k) {
        const uint32_t r = q0 + k;
        RowOut ro;
        double d_rate = 0.0;
        int64_t d_trem = 0;
        row_std<kDebug, kAppB>(c, s_g, P.ovr, r, pend[k], now, v, v_d, eps_d, Q.ar[k], Q.li[k], Q.ge[k], Q.pr[k],
                               Q.lh[k], Q.me[k], Q.ax[k], ro, d_rate, d_trem);
        img[k] = ro.img; cost[k] = ro.cost; aux[k] = ro.aux;
        A.err |= ro.err;
        A.pend += pend[k]; A.cost += ro.cost;                 // (an error fails the whole step)
        A.mn_d = fmin(A.mn_d, __longlong_as_double((long long)ro.img));   // kNone is a NaN: ignored
        if (kDebug && r < ns) { P.dbg_rate[r] = d_rate; P.dbg_trem[r] = d_trem; P.dbg_lhat[r] = pend[k] ? ro.Lh : 0; }
    }
    if (full) {
        st_rows64(P.img + q0, img);
        st_rows(P.cost + q0, cost);
        st_rows(P.aux + q0, aux);
    } else if (any) {
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k)
            if (q0 + k < ns) { P.img[q0 + k] = img[k]; P.cost[q0 + k] = cost[k]; P.aux[q0 + k] = aux[k]; }
    }
#pragma unroll
    for (int k = 0; k < (int)kRPT; ++k)
        spec_add(S, P.id, img[k] != kNone, img[k], q0 + k, cost[k], c.len_key ? Q.li[k] + Q.ge[k] : Q.li[k], Q.me[k],
                 aux[k], t_guess);
}

// phase B of a compound range: the task's goodput and t_gen (a4) from its load-time constants
template <bool kAppB>
__device__ __forceinline__ void task_totals(const Cfg& c, int64_t now, int64_t v, const TaskInfo& ti, uint64_t Tsum,
                                            uint64_t Gsum, uint64_t& Gt, uint64_t& t_gen, int64_t& trem,
                                            uint32_t& err) {
    trem = ti.dls - now;                                    // stage sub-deadline (advisory)
    Gt = ti.dlf <= now ? 0 : ti.gdone + Gsum;               // final deadline passed (A43)
    t_gen = Tsum * (uint64_t)v;
    if (kAppB && t_gen > (uint64_t)(trem > 0 ? trem : 0)) Gt = 0;
    err |= ti.err;
}

// phase C key of one call: (G_task + delta * frames) * 1e9 / (t_gen + eps); B_d < 0 marks a task
// whose t_gen + eps left the exact range
__device__ __forceinline__ uint64_t call_key(uint64_t Gt, uint32_t fr, const Cfg& c, double B_d, uint32_t& err) {
    const uint64_t Gp = Gt + (uint64_t)c.delta * fr;
    if (Gp >= kTwo53 / 1000000000ull || B_d < 0.0) { err = 1; return kNone; }
    return (uint64_t)__double_as_longlong(div_rn_int(__dmul_rn(__uint2double_rn((uint32_t)Gp), 1e9), B_d));
}

// one compound range (see above); every thread of the CTA calls it.  kStaged: the range is one
// tile already staged in B (rows from rg.r0 & ~3); else it is read from global memory.
template <bool kDebug, bool kAppB, bool kStaged>
__device__ __forceinline__ void cmp_range(const Pool& P, const Table& T, const GroupFast* s_g, const Cfg& c,
                                          const Scratch& S, int64_t now, int64_t v, uint64_t t_guess,
                                          const CRange rg, unsigned long long* s_TG, uint32_t tbz,
                                          long long* s_R, double* s_rate, const TileBuf* B, uint64_t* empty, Acc& A) {
    const uint32_t tid = threadIdx.x;
    const uint32_t ntl = rg.t1 - rg.t0;
#ifdef JIT_TG_DOUBLE
    // s_T / s_G arrive zeroed: the task sums are double-buffered (tbz bit 0 = this range's buffer),
    // and phase B of a range clears the other buffer's first tbz >> 1 entries (the previous range's
    // tasks; every thread is past that range's phase C once this range's A -> B barrier is passed)
    unsigned long long* s_T = s_TG + 2 * (tbz & 1u) * kTile;
    unsigned long long* s_G = s_T + kTile;
#else
    unsigned long long* s_T = s_TG;
    unsigned long long* s_G = s_T + kTile;
    __syncthreads();                                       // the previous range's phase C is done with s_T / s_G
    for (uint32_t i = tid; i < ntl; i += kScoreThreads) { s_T[i] = 0; s_G[i] = 0; }
    __syncthreads();
#endif
    const uint32_t qbase = rg.r0 & ~3u;
    const bool single = kStaged || rg.r1 - qbase <= kTile;
    uint32_t kf[kRPT] = {}, kt[kRPT] = {}, kc[kRPT] = {}, kl[kRPT] = {};   // kf: 0x80000000 | frames if pending
    uint32_t km[kRPT] = {}, ka[kRPT] = {};                                 // meta / aux after this pass
    // ---- phase A: per call (a2, a6) + the task sums
    for (uint32_t base = qbase; base < rg.r1; base += kTile) {     // one iteration when staged
        const uint32_t q0 = base + kRPT * tid;
        const bool any = q0 < rg.r1, full = q0 >= rg.r0 && q0 + kRPT - 1 < rg.r1;
        Quad Q;
        uint32_t tk[kRPT];
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) tk[k] = kNoTask;
        if (any && kStaged) {
            load_quad_smem(B, q0 - qbase, Q, tk);
        } else if (any) {
            load_quad(P, q0, Q);
            ld_rows(P.task + q0, tk);
        } else {
            zero_quad(Q);
        }
        // pending calls (no admission drop, A40) and stale cached bounds
        uint32_t inm = 0, pendm = 0, needm = 0, ep[kRPT];
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) {
            const uint32_t r = q0 + k;
            const bool in = any && r >= rg.r0 && r < rg.r1;
            const bool pend = in && Q.ar[k] <= now && m_state(Q.me[k]) <= kPreempted && tk[k] - rg.t0 < ntl;
            ep[k] = fastdiv(Q.ge[k], c.R, c.R_m, c.R_l);
            const bool need = pend && (Q.lh[k] == 0 || ep[k] >= 65536u || m_epoch(Q.me[k]) != ep[k]);
            inm |= (uint32_t)in << k; pendm |= (uint32_t)pend << k; needm |= (uint32_t)need << k;
            if (in && tk[k] - rg.t0 >= ntl) A.err = 1;          // a call outside its range (validated at load)
        }
        if (__any_sync(0xffffffffu, needm != 0)) {
#pragma unroll
            for (int k = 0; k < (int)kRPT; ++k) {
                if (needm & (1u << k)) {
                    Q.lh[k] = cond_quantile(T, Q.ax[k] & 0xFFFFu, ep[k] * c.R, c.qn, c.qd);
                    P.lhat[q0 + k] = Q.lh[k];
                    if (ep[k] < 65536u) { Q.me[k] = (Q.me[k] & 0xFFFFu) | (ep[k] << 16); P.meta[q0 + k] = Q.me[k]; }
                }
            }
            A.ref += __popc(needm);
        }
        uint32_t cost[kRPT], aux[kRPT];
        uint64_t img[kRPT];
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) {
            const bool pend = (pendm >> k) & 1u;
            const uint32_t Lh = max(Q.lh[k], Q.ge[k] + 1);
            const GroupFast G = s_g[pend ? m_group(Q.me[k]) : 0u];
            const uint64_t Gc = (uint64_t)G.w_in_eff * Q.li[k] + (uint64_t)G.w_out_eff * Lh;   // call goodput
            const uint32_t lt = tk[k] - rg.t0;
            cost[k] = pend ? token_cost(Q.li[k], Q.pr[k], c.chunk) : 0u;
            aux[k] = (pend && (Q.ax[k] >> 16) < 0xFFFFu) ? Q.ax[k] + (1u << 16) : Q.ax[k];
            img[k] = kNone; kf[k] = 0;
            if (kDebug && ((inm >> k) & 1u)) P.dbg_lhat[q0 + k] = pend ? Lh : 0;
            if (pend) {
                if (Gc >> 32) A.err = 1;                          // goodput out of the exact range
                const uint32_t fr = fastdiv(Q.ax[k] >> 16, c.frame, c.F_m, c.F_l);   // pre-increment value
                smem_add64(&s_T[lt], Lh - Q.ge[k]);
                smem_add64(&s_G[lt], (uint32_t)Gc);
                kf[k] = 0x80000000u | fr; kt[k] = lt; kc[k] = cost[k];
                kl[k] = c.len_key ? Q.li[k] + Q.ge[k] : Q.li[k];
                km[k] = Q.me[k]; ka[k] = aux[k];
                img[k] = kFramesTag | fr;
                A.pend += 1; A.cost += cost[k];
            }
        }
        if (full) {
            st_rows(P.cost + q0, cost);
            st_rows(P.aux + q0, aux);
            if (!single) st_rows64(P.img + q0, img);
        } else if (any) {
#pragma unroll
            for (int k = 0; k < (int)kRPT; ++k) {
                const uint32_t r = q0 + k;
                if (r >= rg.r0 && r < rg.r1) { P.cost[r] = cost[k]; P.aux[r] = aux[k]; if (!single) P.img[r] = img[k]; }
            }
        }
    }
    if (kStaged) mbar_arrive(empty);                       // this thread is done with the tile buffer
    __syncthreads();
    // ---- phase B: per task of the range (a4); s_G <- G_task, s_T <- fp64 (t_gen + eps)
    for (uint32_t i = tid; i < ntl; i += kScoreThreads) {
        const uint64_t Tsum = s_T[i];
        if (!Tsum) continue;
        uint64_t Gt, t_gen;
        int64_t trem;
        const TaskInfo ti = (kStaged && i < kTaskStage) ? B->ti[i] : P.tinfo[rg.t0 + i];
        task_totals<kAppB>(c, now, v, ti, Tsum, s_G[i], Gt, t_gen, trem, A.err);
        const uint64_t B = t_gen + (uint64_t)c.eps;
        const bool okB = B < kTwo53 && B >= t_gen && t_gen / (uint64_t)v == Tsum;
        s_G[i] = Gt;
        s_T[i] = (unsigned long long)__double_as_longlong(okB ? __ull2double_rn(B) : -1.0);
        if (kDebug) { s_R[i] = trem; s_rate[i] = make_rate(Tsum, trem); }
    }
#ifdef JIT_TG_DOUBLE
    {
        unsigned long long* z = s_TG + 2 * ((tbz & 1u) ^ 1u) * kTile;
        for (uint32_t i = tid; i < (tbz >> 1); i += kScoreThreads) { z[i] = 0; z[kTile + i] = 0; }
    }
#endif
    __syncthreads();
    // ---- phase C: the key of every pending call (a5 over the task aggregate)
    if (single) {
        const uint32_t q0 = qbase + kRPT * tid;
        const bool any = q0 < rg.r1, full = q0 >= rg.r0 && q0 + kRPT - 1 < rg.r1;
        uint64_t img[kRPT];
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k) {
            img[k] = kNone;
            if (kf[k]) {
                img[k] = call_key(s_G[kt[k]], kf[k] & 0xFFFFu, c, __longlong_as_double((long long)s_T[kt[k]]), A.err);
                A.mn = img[k] < A.mn ? img[k] : A.mn;
            }
        }
        if (full) st_rows64(P.img + q0, img);
        else if (any) {
#pragma unroll
            for (int k = 0; k < (int)kRPT; ++k) if (q0 + k >= rg.r0 && q0 + k < rg.r1) P.img[q0 + k] = img[k];
        }
        if (kDebug) {
#pragma unroll
            for (int k = 0; k < (int)kRPT; ++k) {
                const uint32_t r = q0 + k;
                if (any && r >= rg.r0 && r < rg.r1) {
                    P.dbg_rate[r] = kf[k] ? s_rate[kt[k]] : 0.0;
                    P.dbg_trem[r] = kf[k] ? s_R[kt[k]] : 0;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < (int)kRPT; ++k)
            spec_add(S, P.id, img[k] != kNone, img[k], q0 + k, kc[k], kl[k], km[k], ka[k], t_guess);
    } else if (!kStaged) {
        for (uint32_t base = qbase; base < rg.r1; base += kTile) {
#pragma unroll
            for (int k = 0; k < (int)kRPT; ++k) {
                const uint32_t r = base + kRPT * tid + k;
                uint64_t img = kNone;
                uint32_t cst = 0, len = 0;
                if (r >= rg.r0 && r < rg.r1) {
                    img = P.img[r];
                    const uint32_t t = P.task[r] - rg.t0;
                    if (is_frames_tag(img) && t < ntl) {
                        img = call_key(s_G[t], (uint32_t)(img & 0xFFFFu), c, __longlong_as_double((long long)s_T[t]), A.err);
                        A.mn = img < A.mn ? img : A.mn;
                        cst = P.cost[r];
                        len = c.len_key ? P.len_in[r] + P.gen[r] : P.len_in[r];
                    }
                    P.img[r] = img;
                    if (kDebug && t < ntl) {
                        const bool pd = img != kNone;
                        P.dbg_rate[r] = pd ? s_rate[t] : 0.0;
                        P.dbg_trem[r] = pd ? s_R[t] : 0;
                    }
                }
                spec_add(S, P.id, img != kNone, img, r, cst, len, img != kNone ? P.meta[r] : 0u,
                         img != kNone ? P.aux[r] : 0u, t_guess);
            }
        }
    }
}

// the rows of work item `it`: standalone tile it (< n_std) or compound range it - n_std
__device__ __forceinline__ CRange item_rows(const Pool& P, const Scratch& S, uint32_t it) {
    if (it < S.n_std) {
        const uint32_t r0 = it * kTile;
        return CRange{r0, min(r0 + kTile, P.n_single), 0u, 0u};
    }
    return S.crange[it - S.n_std];
}
__device__ __forceinline__ bool stageable(const CRange& rg) { return rg.r1 - (rg.r0 & ~3u) <= kTile; }

// thread 0: bulk-copy the hot state of an item into a tile buffer (completes on bar)
__device__ __forceinline__ void stage_item(const Pool& P, const CRange& rg, bool compound, TileBuf* B, uint64_t* bar) {
    const uint32_t q0 = rg.r0 & ~3u;
    const uint32_t nr = (rg.r1 - q0 + 3) & ~3u;          // whole quads; <= kTile; the SoA is padded
    const uint32_t bytes = nr * (8u + 24u + (compound ? 4u : 0u)) +
                           (compound ? (uint32_t)sizeof(TaskInfo) * min(rg.t1 - rg.t0, kTaskStage) : 0u);
    mbar_expect_tx(bar, bytes);
    if (nr) {                                            // a range of empty tasks has no rows
        bulk_g2s(B->ar, P.arr + q0, 8 * nr, bar);
        bulk_g2s(B->li, P.len_in + q0, 4 * nr, bar);
        bulk_g2s(B->ge, P.gen + q0, 4 * nr, bar);
        bulk_g2s(B->pr, P.pre + q0, 4 * nr, bar);
        bulk_g2s(B->lh, P.lhat + q0, 4 * nr, bar);
        bulk_g2s(B->me, P.meta + q0, 4 * nr, bar);
        bulk_g2s(B->ax, P.aux + q0, 4 * nr, bar);
    }
    if (compound) {
        if (nr) bulk_g2s(B->tk, P.task + q0, 4 * nr, bar);
        const uint32_t nt = min(rg.t1 - rg.t0, kTaskStage);
        if (nt) bulk_g2s(B->ti, P.tinfo + rg.t0, (uint32_t)sizeof(TaskInfo) * nt, bar);
    }
}

#ifdef JIT_TG_DOUBLE
constexpr uint32_t kTGBuffers = 2;
#else
constexpr uint32_t kTGBuffers = 1;
#endif
// dynamic shared memory of k_score: the tile ring + the task sums (+ debug per-task outputs)
// (the SLO-group table sits at the end, sized by the handle's group count)
__host__ __device__ constexpr uint32_t score_smem_bytes(bool debug, uint32_t n_groups = 256) {
    return kStages * (uint32_t)sizeof(TileBuf) + kTGBuffers * 16u * kTile + (debug ? 16u * kTile : 0u) +
           (uint32_t)sizeof(GroupFast) * n_groups;
}

// Persistent: CTA b walks the work items b, b + grid, ...; item j of the CTA lives in ring slot
// j % kStages, and thread 0 keeps the next kStages - 1 items streaming in (HBM reads of several
// items overlap the scoring of one).  Per slot: `full` completes when the bulk copies land,
// `empty` when every thread has read its rows out of the slot.
template <bool kDebug, bool kAppB>
__global__ void __launch_bounds__(kScoreThreads, JIT_SCORE_MINB) k_score(Pool P, Table T, const Group* groups,
                                                                         uint32_t n_groups, Cfg c, Ctrl* ctrl,
                                                                         Scratch S, int64_t now, int64_t v) {
    extern __shared__ __align__(128) unsigned char smem[];
    TileBuf* buf = reinterpret_cast<TileBuf*>(smem);
    unsigned long long* s_TG = reinterpret_cast<unsigned long long*>(smem + kStages * sizeof(TileBuf));  // task sums
    long long* s_R = reinterpret_cast<long long*>(s_TG + kTGBuffers * 2 * kTile);   // kDebug only
    double* s_rate = reinterpret_cast<double*>(s_R + kTile);              // kDebug only
    GroupFast* s_g = reinterpret_cast<GroupFast*>(smem + score_smem_bytes(kDebug, 0));
    __shared__ __align__(8) uint64_t s_full[kStages], s_empty[kStages];
    const uint32_t tid = threadIdx.x;
    const uint32_t n_items = S.n_std + S.n_crange;
    const uint32_t G = gridDim.x;
    // the CTA's item of round r (r-th pass over the grid).  JIT_ITEM_SNAKE: compound ranges (the
    // heavier items) first, and odd rounds walk the grid backwards, so the CTAs that draw a
    // compound range in the partial rounds are not the ones that draw an item in the last round
    const uint32_t bx = blockIdx.x;
    auto item_at = [&](uint32_t r) -> uint32_t {
#if JIT_ITEM_SNAKE
        const uint32_t lg = r * G + ((r & 1u) ? G - 1u - bx : bx);
        if (lg >= n_items) return 0xFFFFFFFFu;
        return lg < S.n_crange ? S.n_std + lg : lg - S.n_crange;
#else
        const uint32_t lg = r * G + bx;
        return lg < n_items ? lg : 0xFFFFFFFFu;
#endif
    };
    uint32_t fpar = 0, fused = 0;                          // thread 0, per slot: fill-count parity, ever filled
    // thread 0: fill slot s with item it (after every thread released the slot's previous fill)
    auto produce = [&](uint32_t it, uint32_t s) {
        if (it >= n_items) return;
        const CRange rn = item_rows(P, S, it);
        if (!stageable(rn)) return;
        if (fused & (1u << s)) mbar_wait(&s_empty[s], ((fpar >> s) & 1u) ^ 1u);
        stage_item(P, rn, it >= S.n_std, &buf[s], &s_full[s]);
        fpar ^= 1u << s; fused |= 1u << s;
    };
    if (tid == 0) {
        for (uint32_t s = 0; s < kStages; ++s) { mbar_init(&s_full[s], 1); mbar_init(&s_empty[s], kScoreThreads); }
        mbar_init_fence();
        for (uint32_t j = 0; j + 1 < kStages; ++j) produce(item_at(j), j);
    }
    for (uint32_t gi = tid; gi < n_groups; gi += kScoreThreads) s_g[gi] = make_fast(groups[gi]);
#ifdef JIT_TG_DOUBLE
    for (uint32_t i = tid; i < 4 * kTile; i += kScoreThreads) s_TG[i] = 0;
#endif
    // first kernel of the step: a fresh control block (nothing else touches ctrl during this
    // kernel) and cleared fallback histograms, spread over the CTAs
    if (blockIdx.x == 0) reset_ctrl_block(ctrl, now, v);
    for (uint32_t b = blockIdx.x * kScoreThreads + tid; b < 4096; b += G * kScoreThreads) {
        S.hcnt[b] = 0; S.hcost[b] = 0;
    }
    __syncthreads();
    const uint64_t t_guess = S.persist->t_guess;
    pdl_launch_dependents();                               // k_spec may launch now (it waits for us)
    Acc A{0u, 0u, 0u, 0u, kNone, 0u, __longlong_as_double((long long)kNone)};
    uint32_t cpar = 0;                                     // consumer: per-slot parity of the fills consumed
    uint32_t tbz = 0;                                      // JIT_TG_DOUBLE: task-sum buffer | entries to clear << 1
    uint32_t s = 0;
    for (uint32_t r = 0;; ++r, s = (s + 1 == kStages) ? 0u : s + 1) {
        const uint32_t it = item_at(r);
        if (it == 0xFFFFFFFFu) break;
        if (tid == 0) produce(item_at(r + kStages - 1), s == 0 ? kStages - 1 : s - 1);
        const CRange rg = item_rows(P, S, it);
        if (it < S.n_std) {
            mbar_wait(&s_full[s], (cpar >> s) & 1u); cpar ^= 1u << s;
            std_quad<kDebug, kAppB>(P, T, s_g, c, S, now, v, t_guess, rg.r0 + kRPT * tid, rg.r1, &buf[s], kRPT * tid, &s_empty[s], A);
        } else if (stageable(rg)) {
            mbar_wait(&s_full[s], (cpar >> s) & 1u); cpar ^= 1u << s;
            cmp_range<kDebug, kAppB, true>(P, T, s_g, c, S, now, v, t_guess, rg, s_TG, tbz, s_R, s_rate, &buf[s], &s_empty[s], A);
            tbz = ((rg.t1 - rg.t0) << 1) | ((tbz & 1u) ^ 1u);
        } else {
            cmp_range<kDebug, kAppB, false>(P, T, s_g, c, S, now, v, t_guess, rg, s_TG, tbz, s_R, s_rate, nullptr, nullptr, A);
            tbz = ((rg.t1 - rg.t0) << 1) | ((tbz & 1u) ^ 1u);
        }
    }
    {
        const uint64_t md = (uint64_t)__double_as_longlong(A.mn_d);
        const uint64_t m_std = A.mn_d == A.mn_d ? md : kNone;    // NaN: no pending standalone row
        store_part(S.gpart, A.pend, A.drop, A.err, m_std < A.mn ? m_std : A.mn, A.cost, A.ref);
    }
}
#endif  // !JIT_EXACT_TU


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
__global__ void __launch_bounds__(kSpecThreads) k_spec(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int reduce_only) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Ctrl s_ctrl;
    reset_ctrl_block(&s_ctrl, 0, 0);
    pdl_wait();
    spec_body<false>(P, c, &s_ctrl, S, reduce_only, smem);
    __syncthreads();
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

// ---- fast sharded step (the speculative variant): every rank scores its shard and
// exports its speculative set; after an allgather every rank resolves the union exactly like
// k_spec.  All ranks share the threshold t (they resolved the same previous step), so the union
// of the local sets {key >= t} IS the global speculative set and the exactness checks carry over
// with the global pending count.  Anything else (a set too large, a failed check) falls back to
// the exact two-round protocol (shard.cuh) without rescoring.
struct SpecHdr {                 // first 64 B of a rank's export
    unsigned long long min_img, tot_cost;
    uint32_t n_pending, n_dropped, err, refresh, n_set, rank, pad[6];
};
struct SpecRec {                 // 32 B per element
    unsigned long long img;
    uint32_t id, cost, len, row, meta, aux;
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
            q.row = S.spec_row[i]; q.meta = S.spec_meta[i]; q.aux = S.spec_aux[i];
        } else {
            q.img = kNone; q.id = q.cost = q.len = q.row = q.meta = q.aux = 0;
        }
        rec[i] = q;
    }
    __syncthreads();
    if (tid == 0) {
        BlockPart* g = S.gpart;
        SpecHdr hd{};
        hd.min_img = __ldcg(&g->min_img); hd.tot_cost = __ldcg(&g->tot_cost); hd.n_pending = __ldcg(&g->n_pending);
        hd.n_dropped = __ldcg(&g->n_dropped); hd.err = __ldcg(&g->err); hd.refresh = __ldcg(&g->refresh);
        hd.n_set = n_set; hd.rank = rank;
        *reinterpret_cast<SpecHdr*>(out) = hd;
        // this rank's own totals, as k_spec(reduce_only) would leave them for the exact protocol
        ctrl->n_pending = hd.n_pending; ctrl->n_dropped = hd.n_dropped; ctrl->min_img = hd.min_img;
        ctrl->tot_cost = hd.tot_cost; ctrl->n_refresh = hd.refresh; ctrl->spec_n = n_set;
        if (hd.err) ctrl->error |= 1u;
        g->n_pending = 0; g->n_dropped = 0; g->err = 0; g->tot_cost = 0; g->refresh = 0; g->min_img = kNone;
        *S.spec_cnt = 0;
    }
}

__global__ void __launch_bounds__(kSpecThreads) k_spec_merge(Pool P, Cfg c, Ctrl* ctrl, Scratch S, const unsigned char* all,
                                                             uint32_t world, uint32_t rank) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t m_off[65], m_pend, m_err, m_fb;
    __shared__ unsigned long long m_min;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        uint32_t off = 0, pend = 0, err = 0, big = 0;
        unsigned long long mn = kNone;
        for (uint32_t w = 0; w < world; ++w) {
            const SpecHdr* hd = reinterpret_cast<const SpecHdr*>(all + (size_t)w * kSpecExportBytes);
            m_off[w] = off;
            off += hd->n_set; pend += hd->n_pending; err |= hd->err; big |= hd->n_set > kSpecExportCap;
            if (hd->min_img < mn) mn = hd->min_img;
        }
        m_off[world] = off; m_pend = pend; m_err = err; m_min = mn;
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
        }
        if (tid == 0) { ctrl->n_pending = m_pend; ctrl->min_img = m_min; ctrl->spec_n = n; }
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
        el.img = q.img; el.id = q.id; el.cost = q.cost; el.len = q.len; el.row = q.row; el.meta = q.meta; el.aux = q.aux;
        el.own = (w == rank) ? 1u : 0u;
    }
    if (tid == 0) { ctrl->n_pending = m_pend; ctrl->min_img = m_min; }
    spec_fast<kSpecThreads>(P, c, ctrl, S, n, n == m_pend, S.persist->t_guess, m_min, el, smem);
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
    __shared__ unsigned long long s_min, s_cost_tot, s_min_above, s_above;
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
        el.row = S.spec_row[tid]; el.meta = S.spec_meta[tid]; el.aux = S.spec_aux[tid];
    }
    if (tid == 0) {
        uint32_t pend, drop, err = 0, ref;
        uint64_t mn, cost;
        if (kBig) {                                        // k_spec already reduced them into ctrl
            pend = ctrl->n_pending; drop = ctrl->n_dropped; mn = ctrl->min_img; cost = ctrl->tot_cost;
            ref = ctrl->n_refresh;
        } else {                                           // k_score's global record; reset for the next step
            BlockPart* g = S.gpart;
            pend = __ldcg(&g->n_pending); drop = __ldcg(&g->n_dropped); err = __ldcg(&g->err);
            cost = __ldcg(&g->tot_cost); ref = __ldcg(&g->refresh); mn = __ldcg(&g->min_img);
            g->n_pending = 0; g->n_dropped = 0; g->err = 0; g->tot_cost = 0; g->refresh = 0; g->min_img = kNone;
        }
        s_pend = pend; s_drop = drop; s_err = err; s_ref = ref; s_min = mn; s_cost_tot = cost;
        s_n = n_set;
        s_first = kSpecBins; s_nsel = 0; s_ncd = 0; s_min_above = kNone; s_above = 0; s_fb = 0;
        ctrl->spec_n = n_set;
        ctrl->n_pending = pend; ctrl->n_dropped = drop; ctrl->min_img = mn; ctrl->tot_cost = cost;
        ctrl->n_refresh = ref;
        if (err) ctrl->error |= 1u;
    }
    if (kBig) for (uint32_t b = tid; b < kSpecBins; b += kSpecThreads) s_hist[b] = 0;
    __syncthreads();
    if (!kBig && tid == 0) *S.spec_cnt = 0;                // next step's set starts empty (all read it)
    const uint32_t n = s_n < kSpecCap ? s_n : kSpecCap;
    if (kBig) {                                            // (1) the set -> smem + histogram
        for (uint32_t i = tid; i < n; i += kSpecThreads) {
            const uint64_t img = S.spec_img[i];
            const uint32_t cs = S.spec_cost[i];
            s_img[i] = img; s_cost[i] = cs;
            atomicAdd(&s_hist[spec_bin(img, t_img)], kPackCount | cs);
        }
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
            spec_fast<kSpecThreads>(P, c, ctrl, S, n, whole, t_img, (uint64_t)s_min, el, smem);
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
            if (s_img[i] >= thr_img) S.cand[atomicAdd(&s_nsel, 1u)] = S.spec_row[i];
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
    // the batch and its bookkeeping: ever_scheduled, Running, undo this step's steps_waited+1
    const uint32_t ns = bj - bi + 1;
    for (uint32_t k = tid; k < ns; k += kSpecThreads) {
        const uint32_t j = s_ord[bi + k];
        const uint32_t e = w_idx[j];
        const uint32_t r = S.spec_row[e];
        S.out_ids[k] = (uint32_t)w_key[j];
        S.out_tokens[k] = w_cost[j];
        S.out_rows[k] = r;
        if (r == 0xFFFFFFFFu) continue;                     // another rank's request (sharded union)
        uint32_t mt = P.meta[r] | (kEver << 12);
        if (m_state(mt) == kQueued || m_state(mt) == kPreempted) mt = m_with_state(mt, kRunning);
        P.meta[r] = mt;
        const uint32_t aux = P.aux[r];
        if ((aux >> 16) < 0xFFFFu) P.aux[r] = aux - (1u << 16);
    }
    if (tid == 0) {
        ctrl->n_selected = ns;
        ctrl->total_tokens = (uint32_t)(pc[bj + 1] - pc[bi]);
        ctrl->i_best = bi; ctrl->j_best = bj;
        ctrl->window_done = 1;
        // next step's speculative threshold: this step's cutoff with a 15% margin
        Persist* ps = S.persist;
        ps->t_guess = (unsigned long long)__double_as_longlong(__dmul_rn(ctrl->thr, 0.85));
        ps->steps += 1;
    }
    stamp(ctrl, 8);
}
#endif  // JIT_EXACT_TU

}  // namespace jit
