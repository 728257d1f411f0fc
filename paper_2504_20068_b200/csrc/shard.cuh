// shard.cuh -- exact sharded GMAX step across ranks.
//
// Rank r holds a shard P_r of the pool (request ids unique across ranks).
//  round 1: every rank exports its first min(B*_r + 1, |P_r|) requests in (key desc, id asc)
//           order (the local budget prefix T_r plus the first request that does not fit).  The
//           global prefix restricted to P_r is a local prefix within the budget, so it lies in
//           T_r, and the global boundary request lies in T_r or is the exported b_r; hence the
//           walk over the sorted union of the exports yields the exact global B* and bp.
//  round 2: every rank exports its candidates {key >= thr}; the union is the global Cd and
//           every rank runs the same window (a9) on it -> identical batch everywhere.
// The exchanges themselves are NCCL allgathers issued by the caller (torch.distributed).
#pragma once
#include "select.cuh"

namespace jit {

struct Rec1 { uint64_t img; uint32_t id, cost; };                               // 16 B
struct Rec2 { uint64_t img; uint32_t id, cost, len, row, rank, pad; };         // 32 B

// rows above the final bucket (or every pending row when all fit) -> Rec1, plus the first
// nf+1 elements of the sorted bucket (written by k_resolve into S.bucket_ck / bucket_cost)
__global__ void __launch_bounds__(kPassThreads) k_export1(Pool P, Ctrl* ctrl, Scratch S, Rec1* out, uint32_t cap) {
    const uint32_t st = ctrl->status;
    if (st != ST_RESOLVED) return;
    const bool all = ctrl->level == 0;                 // resolved at level 0: every pending row fits
    const uint32_t L = ctrl->level;
    const u128 prefix = ctrl->prefix;
    const uint32_t sh_prev = all ? 0 : digit_shift(L - 1);
    const bool need_id = !all && sh_prev < 32;
    const uint32_t stride = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < P.n; wr += stride) {
        const uint32_t r = wr + lane;
        bool take = false;
        uint64_t img = kNone;
        if (r < P.n) {
            img = P.img[r];
            if (img != kNone) take = all || ((make_ck(img, need_id ? P.id[r] : 0u) >> sh_prev) < prefix);
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&ctrl->exp_fill, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (take) {
                const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < cap) { Rec1 q; q.img = img; q.id = P.id[r]; q.cost = P.cost[r]; out[slot] = q; }
                else ctrl->cand_overflow = 1;
            }
        }
    }
}

// after k_export1: append the sorted bucket's first min(nf+1, bucket) elements
__global__ void k_export1_tail(Ctrl* ctrl, Scratch S, Rec1* out, uint32_t cap) {
    if (ctrl->status != ST_RESOLVED) return;
    if (ctrl->level == 0) { if (threadIdx.x == 0) ctrl->n_cand = ctrl->exp_fill; return; }
    const uint32_t nf = ctrl->b_star - ctrl->before_count;
    const uint32_t take = min(nf + 1, ctrl->bucket_count);
    const uint32_t base = ctrl->exp_fill;              // rows above the bucket already written
    for (uint32_t i = threadIdx.x; i < take; i += blockDim.x) {
        if (base + i >= cap) { ctrl->cand_overflow = 1; continue; }
        const u128 ck = S.bucket_ck[i];
        Rec1 q; q.img = ck_img(ck); q.id = (uint32_t)ck; q.cost = S.bucket_cost[i];
        out[base + i] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) ctrl->n_cand = base + take;   // export count
}

// one CTA: exact global B*, bp, thr from the union of the round-1 exports
__global__ void __launch_bounds__(1024) k_merge1(Cfg c, Ctrl* ctrl, const Rec1* all, uint32_t n_all, u128* gk, uint32_t* gv,
                                                 uint32_t smem_cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t s_scan[32];
    __shared__ uint32_t s_nv, s_fit;
    if (threadIdx.x == 0) { s_nv = 0; s_fit = 0; }
    __syncthreads();
    uint32_t mine = 0;
    for (uint32_t i = threadIdx.x; i < n_all; i += blockDim.x) mine += all[i].img != kNone;
    atomicAdd(&s_nv, mine);
    __syncthreads();
    const uint32_t nv = s_nv;
    if (nv == 0) { if (threadIdx.x == 0) { ctrl->status = ST_EMPTY; ctrl->n_pending = 0; } return; }
    uint32_t n2 = 1;
    while (n2 < nv) n2 <<= 1;
    u128* k = n2 <= smem_cap ? reinterpret_cast<u128*>(smem) : gk;
    uint32_t* v = n2 <= smem_cap ? reinterpret_cast<uint32_t*>(smem + 16 * (uint64_t)smem_cap) : gv;
    // deterministic compaction of valid records (block scan over fixed chunks)
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n_all; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool ok = i < n_all && all[i].img != kNone;
        uint64_t tot;
        const uint32_t pos = carry + (uint32_t)block_exclusive_scan_u64(ok ? 1 : 0, s_scan, &tot);
        if (ok) { k[pos] = make_ck(all[i].img, all[i].id); v[pos] = all[i].cost; }
        carry += (uint32_t)tot;
    }
    for (uint32_t i = nv + threadIdx.x; i < n2; i += blockDim.x) { k[i] = ~(u128)0; v[i] = 0; }
    __syncthreads();
    block_sort<u128>(k, v, n2);
    uint64_t cc = 0;
    uint32_t fits = 0;
    for (uint32_t base = 0; base < nv; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const uint64_t cv = i < nv ? v[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_exclusive_scan_u64(cv, s_scan, &tot);
        fits += __syncthreads_count(i < nv && (uint64_t)i + 1 <= c.max_batch && cc + ex + cv <= c.token_budget);
        cc += tot;
    }
    if (threadIdx.x == 0) {
        ctrl->b_star = fits;
        const double bp = __longlong_as_double((long long)ck_img(k[fits - 1]));
        ctrl->bp = bp;
        ctrl->thr = __dmul_rn(c.p, bp);
        ctrl->thr_img = (unsigned long long)__double_as_longlong(ctrl->thr);
        ctrl->status = ST_RESOLVED;
        ctrl->n_cand = 0;
        ctrl->cand_overflow = 0;
    }
}

// round 2 export: local candidates as Rec2 (after k_cand)
__global__ void k_export2(Pool P, Cfg c, Ctrl* ctrl, Scratch S, Rec2* out, uint32_t cap, uint32_t rank) {
    if (ctrl->status != ST_RESOLVED) return;
    const uint32_t n = ctrl->n_cand;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i >= cap) { ctrl->cand_overflow = 1; continue; }
        const uint32_t r = S.cand[i];
        Rec2 q;
        q.img = P.img[r]; q.id = P.id[r]; q.cost = P.cost[r];
        q.len = c.len_key ? P.rows[r].len_in + P.rows[r].gen : P.rows[r].len_in;
        q.row = r; q.rank = rank; q.pad = 0;
        out[i] = q;
    }
}

// one CTA: the window (a9) over the union of the round-2 exports; bookkeeping for own rows
__global__ void __launch_bounds__(1024) k_group_rec(Pool P, Cfg c, Ctrl* ctrl, Scratch S, const Rec2* all, uint32_t n_all,
                                                    uint32_t rank) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ u128 s_scan128[32];
    __shared__ uint64_t s_scan[32];
    __shared__ u128 s_best[32];
    __shared__ uint32_t s_bi[32], s_bj[32], s_nv;
    if (threadIdx.x == 0) s_nv = 0;
    __syncthreads();
    uint32_t mine = 0;
    for (uint32_t i = threadIdx.x; i < n_all; i += blockDim.x) mine += all[i].img != kNone;
    atomicAdd(&s_nv, mine);
    __syncthreads();
    const uint32_t n = s_nv;
    if (n == 0) { if (threadIdx.x == 0) { ctrl->error = 8; ctrl->status = ST_ERROR; } return; }
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    uint64_t* sk = n2 <= kGroupSmemSort ? reinterpret_cast<uint64_t*>(smem) : S.sk;
    uint32_t* sv = n2 <= kGroupSmemSort ? reinterpret_cast<uint32_t*>(smem + 8 * kGroupSmemSort) : S.sv;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n_all; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool ok = i < n_all && all[i].img != kNone;
        uint64_t tot;
        const uint32_t pos = carry + (uint32_t)block_exclusive_scan_u64(ok ? 1 : 0, s_scan, &tot);
        if (ok) { sk[pos] = ((uint64_t)all[i].len << 32) | all[i].id; sv[pos] = i; }
        carry += (uint32_t)tot;
    }
    for (uint32_t i = n + threadIdx.x; i < n2; i += blockDim.x) { sk[i] = ~0ull; sv[i] = 0; }
    __syncthreads();
    block_sort<uint64_t>(sk, sv, n2);
    uint64_t carry_c = 0;
    u128 carry_f = 0;
    for (uint32_t base = 0; base < n; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint64_t cv = 0; u128 fv = 0;
        if (i < n) { const Rec2& q = all[sv[i]]; cv = q.cost; fv = (u128)fixed_point(__longlong_as_double((long long)q.img)); }
        uint64_t tc; u128 tf;
        const uint64_t ec = block_exclusive_scan_u64(cv, s_scan, &tc);
        const u128 ef = block_exclusive_scan_u128(fv, s_scan128, &tf);
        if (i < n) { S.pc[i] = carry_c + ec; S.pf[i] = carry_f + ef; }
        carry_c += tc; carry_f += tf;
    }
    if (threadIdx.x == 0) { S.pc[n] = carry_c; S.pf[n] = carry_f; }
    __syncthreads();
    u128 best = 0; uint32_t bi = 0xFFFFFFFFu, bj = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t lim = (uint64_t)S.pc[i] + c.token_budget;
        uint32_t lo = i, hi = (uint32_t)min((uint64_t)n - 1, (uint64_t)i + c.max_batch - 1);
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (S.pc[mid + 1] <= lim) lo = mid; else hi = mid - 1;
        }
        const u128 sc = S.pf[lo + 1] - S.pf[i];
        if (bi == 0xFFFFFFFFu || sc > best) { best = sc; bi = i; bj = lo; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const u128 ob = shfl_xor_u128(best, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
    }
    if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; s_bj[wid] = bj; }
    __syncthreads();
    if (wid == 0) {
        best = s_best[lane]; bi = s_bi[lane]; bj = s_bj[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u128 ob = shfl_xor_u128(best, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
        }
        if (lane == 0) { s_bi[0] = bi; s_bj[0] = bj; }
    }
    __syncthreads();
    bi = s_bi[0]; bj = s_bj[0];
    const uint32_t ns = bj - bi + 1;
    const uint32_t sc = S.persist->steps;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < ns; k += blockDim.x) {
        const Rec2& q = all[sv[bi + k]];
        S.out_ids[k] = q.id;
        S.out_tokens[k] = q.cost;
        S.out_rows[k] = q.rank == rank ? q.row : 0xFFFFFFFFu;
        if (q.rank == rank)                            // bookkeeping for this shard's rows
            book_selected(P, q.row, P.rows[q.row].meta, P.rows[q.row].since, sc);
    }
    if (threadIdx.x == 0) {
        ctrl->n_selected = ns;
        ctrl->n_cand = n;
        ctrl->total_tokens = (uint32_t)(S.pc[bj + 1] - S.pc[bi]);
        ctrl->window_done = 1;
        // next step's speculative threshold (identical on every rank: thr is global) and counters
        finish_counters(S.persist, ctrl);
    }
}

}  // namespace jit
