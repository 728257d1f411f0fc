// score.cuh -- the streaming pass over the pool (a1)-(a6) and the speculative resolve.
//
//   k_score  every row, one row per thread per iteration over a persistent-style grid: the
//            32-B hot state is read with warp-coalesced loads (the next iteration's row is
//            loaded before the current one is scored), standalone rows get their key image
//            (a5) and cost (a6); compound calls get their bound and cost and add (len_rem,
//            call goodput) to their task's accumulators through a segmented warp reduction
//            (tasks are contiguous row ranges), i.e. (a4) is row-parallel whatever the fan-out.
//            Per-CTA partial counts go to an array (no global atomics on a shared line).
//   k_ctask  every task: its aggregate goodput / t_gen (a4/a5), min / max call key; keys the
//            calls of tasks that can reach the speculative set.
//   k_ckey_full  keys the remaining compound calls (fallback body, debug, shard path).
//   k_spec   one CTA: exact B*, bp, thr, Cd from the speculative set.
#pragma once
#include "select.cuh"

namespace jit {

// Rows whose key image is >= the speculative threshold t (the previous step's cutoff with a
// margin) join the speculative set; warp ballot + one atomic per warp (all lanes convergent).
__device__ __forceinline__ void spec_add(const Scratch& S, const uint32_t* ids, bool valid, uint64_t img,
                                         uint32_t row, uint32_t cost, uint32_t len, uint64_t t) {
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
            S.spec_cost[slot] = cost; S.spec_len[slot] = len;
        }
    }
}

// block reduction of the per-thread partials into part[blockIdx.x]
__device__ __forceinline__ void store_part(BlockPart* part, uint32_t pend, uint32_t drop, uint32_t err,
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
        BlockPart b;
        b.min_img = s_min; b.tot_cost = s_cost; b.n_pending = s_pend; b.n_dropped = s_drop; b.err = s_err;
        b.refresh = s_ref;
        part[blockIdx.x] = b;
    }
}

// compound call (a4, per row): bound, cost; returns pending
template <bool kDebug>
__device__ __forceinline__ bool score_call(const Cfg& c, const Table& T, const GroupFast* sg, uint32_t n_groups,
                                           int64_t now, int64_t arr, uint32_t L_i, uint32_t g, uint32_t pre,
                                           uint32_t lhat, uint32_t meta, uint32_t aux, uint32_t& o_lhat,
                                           uint32_t& o_meta, bool& w_lh, uint64_t& len_rem, uint64_t& Gc,
                                           uint32_t& cost, uint32_t& Lh_out, bool& err) {
    w_lh = false; o_meta = meta; o_lhat = lhat; len_rem = 0; Gc = 0; cost = 0; Lh_out = 0;
    if (arr > now || m_state(meta) > kPreempted) return false;      // no admission drop (A40)
    const uint32_t gi = m_group(meta), drow = aux & 0xFFFFu;
    if (gi >= n_groups || sg[gi].type != kCMP || !(m_flags(meta) & kCompound) || drow >= T.n_rows) {
        err = true; return false;
    }
    const uint32_t ep = fastdiv(g, c.R, c.R_m, c.R_l);
    if (lhat == 0 || ep >= 65536u || m_epoch(meta) != ep) {
        lhat = cond_quantile(T, drow, ep * c.R, c.qn, c.qd);
        o_lhat = lhat; w_lh = true;
        if (ep < 65536u) o_meta = (meta & 0xFFFFu) | (ep << 16);
    }
    const uint32_t Lh = lhat > g + 1 ? lhat : g + 1;
    len_rem = (uint64_t)(Lh - g);
    Gc = (uint64_t)sg[gi].w_in_eff * L_i + (uint64_t)sg[gi].w_out_eff * Lh;
    cost = token_cost(L_i, pre, c.chunk);
    Lh_out = Lh;
    return true;
}

__device__ __forceinline__ bool is_frames_tag(uint64_t img) {
    return (img & 0xFFF8000000000000ull) == kFramesTag;
}

// k_score / k_ctask: the hot pass, compiled into abi.cu (whole-program mode: -rdc costs the
// scoring loop ~50 registers); k_ckey_full / k_spec: the separately linked exact.cu
#ifndef JIT_EXACT_TU
// 4 CTAs of 256 per SM: caps k_score at 64 registers without spills (uncapped it takes ~104,
// i.e. 2 CTAs per SM -- too few warps for a latency-bound streaming pass)
#ifndef JIT_SCORE_MINB
#define JIT_SCORE_MINB 4
#endif
template <bool kDebug>
__global__ void __launch_bounds__(kScoreThreads, JIT_SCORE_MINB) k_score(Pool P, Table T, const Group* groups, uint32_t n_groups,
                                                         Cfg c, Ctrl* ctrl, Scratch S, int64_t now, int64_t v) {
    __shared__ GroupFast s_g[256];
    for (uint32_t gi = threadIdx.x; gi < n_groups; gi += blockDim.x) s_g[gi] = make_fast(groups[gi]);
    // first kernel of the step: a fresh control block (nothing else touches ctrl during this
    // kernel) and cleared fallback histograms, spread over the CTAs
    if (blockIdx.x == 0) reset_ctrl_block(ctrl, now, v);
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < 4096; b += gridDim.x * blockDim.x) {
        S.hcnt[b] = 0; S.hcost[b] = 0;
    }
    __syncthreads();
    const uint64_t t_guess = S.persist->t_guess;
    const int lane = threadIdx.x & 31;
    const bool any_compound = P.n_single < P.n;
    uint32_t my_pend = 0, my_drop = 0, my_err = 0, my_ref = 0;
    uint64_t my_min = kNone, my_cost = 0;
    const uint32_t n = P.n, ns = P.n_single;
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    int64_t a_arr = 0;
    uint32_t a_li = 0, a_g = 0, a_pr = 0, a_lh = 0, a_me = 0, a_ax = 0, a_tk = kNoTask;
    if (r < n) {
        a_arr = __ldcs(P.arr + r); a_li = __ldcs(P.len_in + r); a_g = __ldcs(P.gen + r); a_pr = __ldcs(P.pre + r);
        a_lh = __ldcs(P.lhat + r); a_me = __ldcs(P.meta + r); a_ax = __ldcs(P.aux + r);
        if (r >= ns) a_tk = __ldg(P.task + r);
    }
#pragma unroll 1
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < n; wr += stride, r += stride) {
        const bool act = r < n;
        const uint32_t rn = r + stride;
        int64_t b_arr = 0;
        uint32_t b_li = 0, b_g = 0, b_pr = 0, b_lh = 0, b_me = 0, b_ax = 0, b_tk = kNoTask;
        if (rn < n) {                                    // prefetch the next iteration's row
            b_arr = __ldcs(P.arr + rn); b_li = __ldcs(P.len_in + rn); b_g = __ldcs(P.gen + rn);
            b_pr = __ldcs(P.pre + rn); b_lh = __ldcs(P.lhat + rn); b_me = __ldcs(P.meta + rn);
            b_ax = __ldcs(P.aux + rn);
            if (rn >= ns) b_tk = __ldg(P.task + rn);
        }
        uint64_t img = kNone;
        bool valid = false;
        uint64_t vT = 0, vG = 0;                       // compound contributions
        uint32_t fr = 0, sp_cost = 0;
        uint32_t key_task = kNoTask;
        if (act && r < ns) {
            RowRes o;
            score_standalone<kDebug>(c, T, s_g, n_groups, P.ovr, r, now, v, a_arr, a_li, a_g, a_pr, a_lh, a_me, a_ax, o);
            P.img[r] = o.img; P.cost[r] = o.cost;
            sp_cost = o.cost;
            if (o.aux != a_ax) P.aux[r] = o.aux;
            if (o.w_meta) P.meta[r] = o.meta;
            if (o.w_lhat) P.lhat[r] = o.lhat;
            if (kDebug) {
                P.dbg_rate[r] = o.pending ? o.rate : 0.0;
                P.dbg_trem[r] = o.pending ? o.trem : 0;
                P.dbg_lhat[r] = o.pending ? o.lhatc : 0;
            }
            img = o.img;
            valid = img != kNone;
            my_drop += o.dropped; my_err |= o.err; my_ref += o.w_lhat;
            if (valid) { my_pend += 1; my_cost += o.cost; if (img < my_min) my_min = img; }
        } else if (act) {
            uint32_t o_lhat, o_meta, cost, Lh;
            bool w_lh, err = false;
            uint64_t len_rem, Gc;
            const bool pend = score_call<kDebug>(c, T, s_g, n_groups, now, a_arr, a_li, a_g, a_pr, a_lh, a_me, a_ax,
                                                 o_lhat, o_meta, w_lh, len_rem, Gc, cost, Lh, err);
            P.cost[r] = cost;                          // > 0 marks a pending call
            if (w_lh) { P.lhat[r] = o_lhat; if (o_meta != a_me) P.meta[r] = o_meta; }
            if (kDebug) P.dbg_lhat[r] = pend ? Lh : 0;
            my_err |= err; my_ref += w_lh;
            if (pend) {
                // the key needs the task's sums: park floor(waited/Delta) (pre-increment value)
                // in the key slot and do steps_waited+1 here (the task pass never touches aux)
                fr = fastdiv(a_ax >> 16, c.frame, c.F_m, c.F_l);
                P.img[r] = kFramesTag | fr;
                if ((a_ax >> 16) < 0xFFFFu) P.aux[r] = a_ax + (1u << 16);
                my_pend += 1; my_cost += cost; vT = len_rem; vG = Gc;
            } else {
                P.img[r] = kNone;
            }
            key_task = (a_tk < P.n_tasks) ? a_tk : kNoTask;
            if (a_tk >= P.n_tasks) my_err = 1;
        }
        // segmented warp reduction per task (rows of a task are contiguous) of the sums of
        // (len_rem, goodput) and the min / max starvation frames; warps that hold no compound
        // call skip it (warp-uniform)
        if (any_compound && __any_sync(0xffffffffu, key_task != kNoTask)) {
            uint64_t sT = vT, sG = vG;
            uint32_t fx = vT ? fr : 0u, fn = vT ? fr : 0xFFFFFFFFu;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t uT = __shfl_up_sync(0xffffffffu, sT, d);
                const uint64_t uG = __shfl_up_sync(0xffffffffu, sG, d);
                const uint32_t ux = __shfl_up_sync(0xffffffffu, fx, d);
                const uint32_t un = __shfl_up_sync(0xffffffffu, fn, d);
                const uint32_t uk = __shfl_up_sync(0xffffffffu, key_task, d);
                if (lane >= d && uk == key_task) { sT += uT; sG += uG; fx = max(fx, ux); fn = min(fn, un); }
            }
            const uint32_t nk = __shfl_down_sync(0xffffffffu, key_task, 1);
            if (key_task != kNoTask && (lane == 31 || nk != key_task) && sT) {
                atomicAdd(&S.tacc[key_task].T, (unsigned long long)sT);
                atomicAdd(&S.tacc[key_task].G, (unsigned long long)sG);
                atomicMax(&S.tacc[key_task].fmax, fx);
                atomicMin(&S.tacc[key_task].fmin, fn);
            }
        }
        spec_add(S, P.id, valid, img, r, sp_cost, c.len_key ? a_li + a_g : a_li, t_guess);
        a_arr = b_arr; a_li = b_li; a_g = b_g; a_pr = b_pr; a_lh = b_lh; a_me = b_me; a_ax = b_ax; a_tk = b_tk;
    }
    store_part(S.part, my_pend, my_drop, my_err, my_min, my_cost, my_ref);
}

// --------------------------------------------------------------------------------------
// k_ctask: one thread per task (a4/a5).  G_task = goodput_done + sum of the current stage's
// pending call goodput (zero once a_c + D has passed, A43), t_gen = (sum len_rem) * v_token;
// the key of call i is (G_task + delta*floor(waited_i/Delta)) * 1e9 / (t_gen + eps).  The key
// is non-decreasing in the frame count, so the task's extreme keys come from its min / max
// frames (k_score): kmin feeds the pool minimum exactly, and only a task whose kmax reaches
// the speculative threshold ("hot") has its calls keyed here -- by one warp, lanes over the
// calls, so the speculative-set ballot stays convergent.  Every other call keeps its tagged
// frame count until k_ckey_full (fallback body / debug / shard path) keys it.
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kScoreThreads) k_ctask(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    const int64_t now = ctrl->now, v = ctrl->v;
    const uint64_t t_guess = S.persist->t_guess;
    const int lane = threadIdx.x & 31;
    uint32_t my_err = 0;
    uint64_t my_min = kNone;
    const uint32_t nt = P.n_tasks;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t wt = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wt < nt; wt += stride) {
        const uint32_t t = wt + lane;
        bool hot = false;
        uint64_t Gt = 0, t_gen = 0;
        if (t < nt) {
            const TaskAcc acc = S.tacc[t];
            if (acc.T) {
                const int64_t a_c = __ldg(P.t_arr + t), D = __ldg(P.t_dl + t);
                const uint32_t s = __ldg(P.cur_stage + t), Sn = __ldg(P.n_stages + t);
                const uint4 p0 = __ldg(reinterpret_cast<const uint4*>(P.pattern) + 2 * t);
                const uint4 p1 = __ldg(reinterpret_cast<const uint4*>(P.pattern) + 2 * t + 1);
                const uint32_t pt[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
                // phi(s) = t_<=s / t_total, D_s = floor(D * phi); in ms the ratio is
                // identical and D*le fits u64 when D < 2^40 ns and t_total < 2^24 ms
                uint64_t le = 0, tot = 0;
#pragma unroll
                for (uint32_t u = 0; u < kMaxStages; ++u) {
                    const uint64_t ms = u < Sn ? pt[u] : 0u;
                    tot += ms; if (u <= s) le += ms;
                }
                if (tot == 0 || Sn == 0 || Sn > kMaxStages || s >= Sn) my_err = 1;
                const int64_t Ds = !tot ? 0
                    : ((uint64_t)D < (1ull << 40) && tot < (1ull << 24)) ? (int64_t)((uint64_t)D * le / tot)
                                                                         : (int64_t)((u128)(uint64_t)D * le / tot);
                const int64_t trem = a_c + Ds - now;               // advisory stage deadline
                Gt = __ldg(P.gdone + t) + acc.G;
                if (a_c + D <= now) Gt = 0;                         // final deadline passed
                t_gen = acc.T * (uint64_t)v;
                if (c.appb && t_gen > (uint64_t)(trem > 0 ? trem : 0)) Gt = 0;
                double kmin, kmax;
                const bool ok_min = make_key(Gt + (uint64_t)c.delta * acc.fmin, t_gen, c.eps, &kmin);
                const bool ok_max = make_key(Gt + (uint64_t)c.delta * acc.fmax, t_gen, c.eps, &kmax);
                if (!ok_min || !ok_max) my_err = 1;
                const uint64_t imin = (uint64_t)__double_as_longlong(kmin);
                const uint64_t imax = (uint64_t)__double_as_longlong(kmax);
                if (imin < my_min) my_min = imin;
                hot = ok_max && imax >= t_guess;
                TaskAcc o;                                          // consumed: re-zero the sums
                o.T = 0; o.G = 0; o.Gt = Gt; o.tgen = t_gen; o.trem = trem; o.Tr = acc.T;
                o.fmax = 0; o.fmin = 0xFFFFFFFFu;
                S.tacc[t] = o;
            }
        }
        // hot tasks: the warp keys their calls together (speculative-set ballot convergent)
        unsigned hm = __ballot_sync(0xffffffffu, hot);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            const uint32_t ht = __shfl_sync(0xffffffffu, t, src);
            const uint64_t hG = __shfl_sync(0xffffffffu, Gt, src);
            const uint64_t hB = __shfl_sync(0xffffffffu, t_gen, src);
            const uint32_t r0 = __ldg(P.call_off + ht), r1 = __ldg(P.call_off + ht + 1);
            for (uint32_t wr = r0; wr < r1; wr += 32) {
                const uint32_t r = wr + lane;
                uint64_t img = kNone;
                bool valid = false;
                uint32_t cost = 0, len = 0;
                if (r < r1) {
                    img = P.img[r];
                    if (is_frames_tag(img)) {
                        const uint32_t fr = (uint32_t)(img & 0xFFFFFFFFu);
                        double key;
                        make_key(hG + (uint64_t)c.delta * fr, hB, c.eps, &key);
                        img = (uint64_t)__double_as_longlong(key);
                        P.img[r] = img;
                        valid = true;
                        cost = P.cost[r];
                        len = c.len_key ? P.len_in[r] + P.gen[r] : P.len_in[r];
                    }
                }
                spec_add(S, P.id, valid, img, r, cost, len, t_guess);
            }
        }
    }
    store_part(S.part2, 0, 0, my_err, my_min, 0, 0);
}
#endif  // !JIT_EXACT_TU

#ifdef JIT_EXACT_TU
// k_ckey_full: row-parallel keying of every call still carrying its frame tag (after
// k_ctask); in debug mode also the per-call rate / t_rem outputs of every compound row.
template <bool kDebug>
__global__ void __launch_bounds__(kScoreThreads) k_ckey_full(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int force) {
    if (!kDebug && blockIdx.x == 0 && threadIdx.x == 0 && ctrl->chain) {   // exact path: next k_hist0
        atomicOr(&ctrl->trace, 2u);
        k_hist0<<<S.grid_pass, kPassThreads, 0, cudaStreamTailLaunch>>>(P, c, ctrl, S, 0);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { ctrl->error |= 2u; ctrl->status = ST_ERROR; ctrl->launch_err = e; }
    }
    if (!force && ctrl->status != ST_FALLBACK) return;
    const uint32_t n = P.n;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t r = P.n_single + blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
        const uint64_t img = P.img[r];
        const bool tagged = is_frames_tag(img);
        if (!tagged && !kDebug) continue;
        const uint32_t t = __ldg(P.task + r);
        if (t >= P.n_tasks) continue;
        if (tagged) {
            double key;
            make_key(S.tacc[t].Gt + (uint64_t)c.delta * (uint32_t)(img & 0xFFFFFFFFu), S.tacc[t].tgen, c.eps, &key);
            P.img[r] = (uint64_t)__double_as_longlong(key);
        }
        if (kDebug) {
            if (P.cost[r]) { P.dbg_rate[r] = make_rate(S.tacc[t].Tr, S.tacc[t].trem); P.dbg_trem[r] = S.tacc[t].trem; }
            else { P.dbg_rate[r] = 0.0; P.dbg_trem[r] = 0; }
        }
    }
}

// --------------------------------------------------------------------------------------
// k_spec: one CTA of 512 threads.  Reduces the scoring partials, then resolves (a7)/(a8)
// exactly from the speculative set S = {key >= t} and runs the window (a9) on Cd, all in
// shared memory.  S is upward closed in the (key desc, id asc) order, i.e. a PREFIX of the
// priority order, so the budget walk restricted to S is the exact walk as long as it stops
// inside S (or S holds every pending row); Cd = {key >= thr} lies in S when thr >= t.
// Otherwise the exact radix path runs (launch_exact_path).
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
constexpr uint32_t kSpecThreads = 512;
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

// The exact path, launched from the device only when needed (CUDA dynamic parallelism): a
// chain of tail launches, each kernel launching its successor (select.cuh) -- a tail launch
// runs once its launching grid has finished, and the step (graph node or stream work)
// completes only after the whole chain.  radix = false: just the window over a large Cd.
// Called by one thread; false if the launch failed.
__device__ __noinline__ bool launch_exact_path(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, bool radix) {
    ctrl->chain = 1;
    if (!radix)
        k_group<<<1, 1024, 12 * kGroupSmemSort, cudaStreamTailLaunch>>>(P, c, ctrl, S);
    else if (P.n_single < P.n)                 // key the compound calls still tagged, then k_hist0
        k_ckey_full<false><<<S.nb_full, kScoreThreads, 0, cudaStreamTailLaunch>>>(P, c, ctrl, S, 1);
    else
        k_hist0<<<S.grid_pass, kPassThreads, 0, cudaStreamTailLaunch>>>(P, c, ctrl, S, 0);
    const cudaError_t e = cudaGetLastError();
    ctrl->trace |= 1u;
    ctrl->launch_err = e;
    return e == cudaSuccess;
}

// thread 0: give up on the speculative resolve -> exact path (sets *fb: 1 launched, 3 failed)
__device__ __forceinline__ void spec_fallback(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, int* fb) {
    ctrl->status = ST_FALLBACK; ctrl->fallback = 1;
    *fb = launch_exact_path(P, c, ctrl, S, true) ? 1 : 3;
    if (*fb == 3) { ctrl->status = ST_ERROR; ctrl->error |= 2u; }
}

__global__ void __launch_bounds__(kSpecThreads) k_spec(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int reduce_only) {
    extern __shared__ __align__(16) unsigned char smem[];
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
    if (tid == 0) {
        s_min = kNone; s_cost_tot = 0; s_pend = 0; s_drop = 0; s_err = 0; s_ref = 0;
        s_n = *S.spec_cnt;
        *S.spec_cnt = 0;                                   // next step's set starts empty
        ctrl->spec_n = s_n;
        s_first = kSpecBins; s_nsel = 0; s_ncd = 0; s_min_above = kNone; s_above = 0; s_fb = 0;
    }
    for (uint32_t b = tid; b < kSpecBins; b += kSpecThreads) s_hist[b] = 0;
    __syncthreads();
    const uint32_t n = s_n < kSpecCap ? s_n : kSpecCap;
    {   // partials of k_score and k_ctask, and (1) the set -> smem + histogram, in one pass
        uint32_t pend = 0, drop = 0, err = 0, ref = 0;
        uint64_t mn = kNone, cost = 0;
        for (uint32_t i = tid; i < S.n_part + S.n_part2; i += kSpecThreads) {
            const BlockPart b = i < S.n_part ? S.part[i] : S.part2[i - S.n_part];
            pend += b.n_pending; drop += b.n_dropped; err |= b.err; cost += b.tot_cost; ref += b.refresh;
            if (b.min_img < mn) mn = b.min_img;
        }
        if (!reduce_only) {
            for (uint32_t i = tid; i < n; i += kSpecThreads) {
                const uint64_t img = S.spec_img[i];
                const uint32_t cs = S.spec_cost[i];
                s_img[i] = img; s_cost[i] = cs;
                atomicAdd(&s_hist[spec_bin(img, t_img)], kPackCount | cs);
            }
        }
        pend = warp_sum(pend); drop = warp_sum(drop); err = __reduce_or_sync(0xffffffffu, err);
        mn = warp_min_u64(mn); cost = warp_sum(cost); ref = warp_sum(ref);
        if (lane == 0) {
            atomicAdd(&s_pend, pend); atomicAdd(&s_drop, drop); atomicOr(&s_err, err); atomicAdd(&s_ref, ref);
            atomicMin(&s_min, (unsigned long long)mn); atomicAdd(&s_cost_tot, (unsigned long long)cost);
        }
        __syncthreads();
        if (tid == 0) {
            ctrl->n_pending = s_pend; ctrl->n_dropped = s_drop; ctrl->min_img = s_min; ctrl->tot_cost = s_cost_tot;
            ctrl->n_refresh = s_ref;
            if (s_err) ctrl->error |= 1u;
        }
    }
    if (reduce_only) return;                               // sharded step: the radix path follows
    stamp(ctrl, 1);
    const uint32_t np = s_pend;
    const bool whole = (s_n == np);                        // S holds every pending row
    if (tid == 0) {
        if (s_err) { ctrl->status = ST_ERROR; s_fb = 2; }
        else if (np == 0) { ctrl->status = ST_EMPTY; s_fb = 2; }
        else if (s_n > kSpecCap || s_n == 0) spec_fallback(P, c, ctrl, S, &s_fb);
    }
    __syncthreads();
    if (s_fb) return;                                      // k_publish (next node) reports it
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
            if (!whole) spec_fallback(P, c, ctrl, S, &s_fb);
            else {
                s_fits = n;
                const double bp = __longlong_as_double((long long)s_min);
                const double thr = __dmul_rn(__ddiv_rn((double)c.pn, (double)c.pd), bp);
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
            if (tid == 0) spec_fallback(P, c, ctrl, S, &s_fb);
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
                    const double thr = __dmul_rn(__ddiv_rn((double)c.pn, (double)c.pd), bp);
                    const uint64_t ti = (uint64_t)__double_as_longlong(thr);
                    if (!whole && ti < t_img) spec_fallback(P, c, ctrl, S, &s_fb);
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
    if (ncd > kSpecWindow) {
        // a large Cd: hand it to k_group (launched from here)
        if (tid == 0) s_nsel = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kSpecThreads)
            if (s_img[i] >= thr_img) S.cand[atomicAdd(&s_nsel, 1u)] = S.spec_row[i];
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            s_fb = launch_exact_path(P, c, ctrl, S, false) ? 1 : 3;
            if (s_fb == 3) { ctrl->status = ST_ERROR; ctrl->error |= 2u; }
        }
        return;
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
