// multi.cuh -- NEXT-2 power-of-K over M model replicas (§4.3; SPEC S:322-330;
// reading A51).
//
// Every request has dummies on K sampled replicas; replica m's handle holds its dummies (a
// standalone pool) and runs the ordinary GMAX step keyed with its own v_token ("scheduling
// proceeds as usual over the enlarged set").  A request proposed by several replicas in the same
// step is assigned to the replica where its priority is highest -- key_m = A / (len_rem v_m + eps)
// with A and len_rem replica-independent, so the smallest v_m, ties to the lower replica index --
// and leaves the other batches (no refill).  Once assigned, its other dummies are removed: every
// other replica's dummy of the request becomes Moved (terminal, never pending).
//
// Exchange: after its step every replica exports a record {header, proposed ids}; the M records
// are concatenated (one allgather across ranks, or a device copy on one GPU); every replica then
// reconciles against the union with three kernels on its stream:
//   k_multi_mark    grid: for every proposal (w, id) found in this replica's pool (the own batch
//                   by row, the others through the id map) atomicMax the row's winner word with
//                   (epoch << 8) | (255 - rank(w)), rank(w) = position of (v_w, w) in ascending
//                   order -- the row's winner is the lowest rank that proposed its request
//   k_multi_moved   grid: every such row whose winner is another replica becomes Moved
//   k_multi_finish  one CTA: the own batch keeps the entries this replica won (window order kept),
//                   total tokens, pinned host mirror + control block
// The epoch in the winner word makes a reset pass unnecessary (stale words compare lower).
#pragma once
#include "select.cuh"

namespace jit {

constexpr uint32_t kMaxReplicas = 256;

struct MultiHdr {          // 32 bytes, then cap proposal ids
    int64_t v;             // the step's v_token (ns)
    uint32_t replica, n, cap, status;   // status: 1 = a resolved step (n proposals), 0 = none
    uint32_t pad[2];
};
static_assert(sizeof(MultiHdr) == 32, "multi header");
__host__ __device__ __forceinline__ uint64_t multi_rec_bytes(uint32_t cap) {
    return sizeof(MultiHdr) + ((4ull * cap + 31) & ~31ull);
}
__device__ __forceinline__ const MultiHdr* multi_hdr(const unsigned char* all, uint64_t rb, uint32_t w) {
    return reinterpret_cast<const MultiHdr*>(all + rb * w);
}
__device__ __forceinline__ const uint32_t* multi_ids(const unsigned char* all, uint64_t rb, uint32_t w) {
    return reinterpret_cast<const uint32_t*>(all + rb * w + sizeof(MultiHdr));
}

// the replica's proposal after its step (ids in window order)
__global__ void k_multi_export(const Ctrl* ctrl, Scratch S, uint32_t replica, uint32_t cap, unsigned char* out) {
    const bool ok = ctrl->status == ST_RESOLVED && ctrl->error == 0;
    const uint32_t n = ok ? ctrl->n_selected : 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        MultiHdr h{};
        h.v = ctrl->v; h.replica = replica; h.n = n; h.cap = cap; h.status = ok ? 1u : 0u;
        *reinterpret_cast<MultiHdr*>(out) = h;
    }
    uint32_t* ids = reinterpret_cast<uint32_t*>(out + sizeof(MultiHdr));
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) ids[i] = S.out_ids[i];
}

// ranks of the M replicas in (v, replica) ascending order (shared memory, every CTA); a header
// whose replica field or capacity disagrees with its slot is an error
__device__ __forceinline__ void multi_ranks(const unsigned char* all, uint64_t rb, uint32_t M, uint32_t cap,
                                            uint32_t* s_rank, Ctrl* ctrl) {
    for (uint32_t w = threadIdx.x; w < M; w += blockDim.x) {
        const MultiHdr* hw = multi_hdr(all, rb, w);
        uint32_t r = 0;
        for (uint32_t u = 0; u < M; ++u) {
            const int64_t vu = multi_hdr(all, rb, u)->v;
            r += vu < hw->v || (vu == hw->v && u < w);
        }
        s_rank[w] = r;
        if (hw->replica != w || hw->cap != cap || hw->n > cap) atomicOr(&ctrl->error, 64u);
    }
    __syncthreads();
}

// the row of proposal i of replica w in this pool (0xFFFFFFFF: not here)
__device__ __forceinline__ uint32_t multi_row(const Pool& P, const Scratch& S, const unsigned char* all, uint64_t rb,
                                              uint32_t w, uint32_t i, uint32_t me) {
    const uint32_t id = multi_ids(all, rb, w)[i];
    if (w == me) return S.out_rows[i];
    return map_find(P, id);
}

__global__ void __launch_bounds__(256) k_multi_mark(Pool P, Scratch S, Ctrl* ctrl, const unsigned char* all, uint64_t rb,
                                                    uint32_t M, uint32_t me, uint32_t cap, unsigned long long* win,
                                                    unsigned long long epoch) {
    __shared__ uint32_t s_rank[kMaxReplicas];
    multi_ranks(all, rb, M, cap, s_rank, ctrl);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < (uint64_t)M * cap;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = (uint32_t)(e / cap), i = (uint32_t)(e % cap);
        const MultiHdr* hw = multi_hdr(all, rb, w);
        if (i >= min(hw->n, cap)) continue;
        const uint32_t r = multi_row(P, S, all, rb, w, i, me);
        if (r >= P.n) continue;
        if (m_flags(P.rows[r].meta) & kCompound) { atomicOr(&ctrl->error, 128u); continue; }   // standalone only
        atomicMax(win + r, (epoch << 8) | (255u - s_rank[w]));
    }
}

__global__ void __launch_bounds__(256) k_multi_moved(Pool P, Scratch S, Ctrl* ctrl, const unsigned char* all, uint64_t rb,
                                                     uint32_t M, uint32_t me, uint32_t cap,
                                                     const unsigned long long* win, unsigned long long epoch) {
    __shared__ uint32_t s_rank[kMaxReplicas];
    multi_ranks(all, rb, M, cap, s_rank, ctrl);
    const unsigned long long mine = (epoch << 8) | (255u - s_rank[me]);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < (uint64_t)M * cap;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = (uint32_t)(e / cap), i = (uint32_t)(e % cap);
        const MultiHdr* hw = multi_hdr(all, rb, w);
        if (i >= min(hw->n, cap)) continue;
        const uint32_t r = multi_row(P, S, all, rb, w, i, me);
        if (r >= P.n || win[r] == mine) continue;
        // assigned to another replica: this dummy is removed; the stamp regime is left as it
        // is (the next pass freezes the steps_waited count of a row that is no longer pending)
        uint32_t* mp = &P.rows[r].meta;
        *mp = m_with_state(*mp, kMoved);
    }
}

// one CTA of kMultiThreads: the own batch keeps the proposals this replica won, in window order
constexpr uint32_t kMultiThreads = 1024;
__global__ void __launch_bounds__(kMultiThreads) k_multi_finish(Scratch S, Ctrl* ctrl, const unsigned char* all, uint64_t rb,
                                                                uint32_t M, uint32_t me, uint32_t cap,
                                                                const unsigned long long* win, unsigned long long epoch) {
    __shared__ uint32_t s_rank[kMaxReplicas];
    __shared__ uint32_t s_cnt[kMultiThreads / 32];
    __shared__ unsigned long long s_tok[kMultiThreads / 32];
    multi_ranks(all, rb, M, cap, s_rank, ctrl);
    const unsigned long long mine = (epoch << 8) | (255u - s_rank[me]);
    const uint32_t n = min(multi_hdr(all, rb, me)->n, cap);
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // contiguous runs of ceil(n / threads) entries per thread (order kept by an exclusive scan)
    const uint32_t per = (n + kMultiThreads - 1) / kMultiThreads;
    const uint32_t b = min(tid * per, n), e = min(b + per, n);
    uint32_t cnt = 0;
    unsigned long long tok = 0;
    for (uint32_t i = b; i < e; ++i)
        if (win[S.out_rows[i]] == mine) { ++cnt; tok += S.out_tokens[i]; }
    // block exclusive scan of cnt
    uint32_t inc = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += x;
    }
    const unsigned long long wt = warp_sum(tok);
    if (lane == 31) s_cnt[wid] = inc;
    if (lane == 0) s_tok[wid] = wt;
    __syncthreads();
    uint32_t before = 0, kept = 0;
    unsigned long long total = 0;
    for (uint32_t w = 0; w < kMultiThreads / 32; ++w) {
        if (w < wid) before += s_cnt[w];
        kept += s_cnt[w];
        total += s_tok[w];
    }
    uint32_t pos = before + inc - cnt;
    // gather this thread's kept entries first (in-place compaction only moves entries left, but a
    // thread's target range may overlap another thread's source range)
    uint32_t kid[8], ktk[8], krw[8];
    uint32_t nk = 0;
    bool spill = per > 8;
    if (!spill)
        for (uint32_t i = b; i < e; ++i)
            if (win[S.out_rows[i]] == mine) { kid[nk] = S.out_ids[i]; ktk[nk] = S.out_tokens[i]; krw[nk] = S.out_rows[i]; ++nk; }
    __syncthreads();
    if (spill) {                       // n > 8 * threads: serial compaction by thread 0 (not reached for cap <= 8192)
        if (tid == 0) {
            uint32_t k = 0;
            for (uint32_t i = 0; i < n; ++i)
                if (win[S.out_rows[i]] == mine) {
                    S.out_ids[k] = S.out_ids[i]; S.out_tokens[k] = S.out_tokens[i]; S.out_rows[k] = S.out_rows[i]; ++k;
                }
        }
    } else {
        for (uint32_t j = 0; j < nk; ++j, ++pos) { S.out_ids[pos] = kid[j]; S.out_tokens[pos] = ktk[j]; S.out_rows[pos] = krw[j]; }
    }
    __syncthreads();
    const uint32_t B = cap + 1;
    for (uint32_t i = tid; i < kept; i += kMultiThreads) {
        S.h_batch[i] = S.out_ids[i]; S.h_batch[B + i] = S.out_tokens[i]; S.h_batch[2 * B + i] = S.out_rows[i];
    }
    if (tid == 0 && multi_hdr(all, rb, me)->status) {
        ctrl->n_selected = kept;
        ctrl->total_tokens = (uint32_t)total;
        ctrl->batch_on_host = 1;
    }
    publish_ctrl(ctrl, S.h_ctrl);
}

}  // namespace jit
