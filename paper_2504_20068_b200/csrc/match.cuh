// match.cuh -- NEXT-3: batch pattern-graph matching on the GPU (§4.1, reading A49).
//
// One warp per query (a compound task revealed up to stage s), its lanes over the stored pattern
// graphs (staged once per CTA in shared memory when they fit, else read through L2): prefix
// pruning on the stage identities 0..s, then the mean of Gaussian-kernel similarities over the
// node attributes of stages 0..s-1 and the input lengths of the LLM stages 1..s, in stage order
// (nodes first, then the edge, per stage); the best pattern by (score desc, reuse desc, index
// asc) from a warp reduction.  The matched pattern's stage times give phi(s) = t_<=s / t_total
// (P:310-313), applied to the resident pool's task (k_apply_match + k_task_prep).
#pragma once
#include <cstdint>
#include "common.cuh"
#include "pool.cuh"

namespace jit {

constexpr uint32_t kMatchThreads = 256;
constexpr uint32_t kMatchWords = 3 * kMaxStages + 2;        // ident[8] in[8] out[8] n_stages reuse
constexpr uint32_t kMatchSmemPatterns = 1024;               // 104 KB of shared memory

struct PatternsDev {
    const uint32_t *n_stages, *ident, *in_len, *out, *t_ms, *reuse;
    uint32_t n;
};
struct QueriesDev {
    const uint32_t *stage, *ident, *in_len, *out, *task;
    uint32_t n;
};

// Gaussian kernel exp(-(a-b)^2 / (2 sigma^2)), sigma = max(0.25 max(a, b), 1); the
// operation order of the oracle's og_kernel_sim (no FMA contraction: --fmad=false)
__device__ __forceinline__ double kernel_sim(uint32_t a, uint32_t b) {
    const double mx = (double)(a > b ? a : b);
    double sigma = 0.25 * mx;
    if (sigma < 1.0) sigma = 1.0;
    const double d = (double)a - (double)b;
    return exp(-(d * d) / (2.0 * sigma * sigma));
}

// pattern word w of pattern p: layout [p][kMatchWords] in shared memory, SoA in global memory
struct PatView {
    const uint32_t* sm;     // shared copy or nullptr
    PatternsDev G;
    __device__ __forceinline__ uint32_t ident(uint32_t p, uint32_t u) const {
        return sm ? sm[p * kMatchWords + u] : __ldg(G.ident + p * kMaxStages + u);
    }
    __device__ __forceinline__ uint32_t in(uint32_t p, uint32_t u) const {
        return sm ? sm[p * kMatchWords + kMaxStages + u] : __ldg(G.in_len + p * kMaxStages + u);
    }
    __device__ __forceinline__ uint32_t out(uint32_t p, uint32_t u) const {
        return sm ? sm[p * kMatchWords + 2 * kMaxStages + u] : __ldg(G.out + p * kMaxStages + u);
    }
    __device__ __forceinline__ uint32_t ns(uint32_t p) const {
        return sm ? sm[p * kMatchWords + 3 * kMaxStages] : __ldg(G.n_stages + p);
    }
    __device__ __forceinline__ uint32_t reuse(uint32_t p) const {
        return sm ? sm[p * kMatchWords + 3 * kMaxStages + 1] : __ldg(G.reuse + p);
    }
};

__global__ void __launch_bounds__(kMatchThreads) k_match(PatternsDev G, QueriesDev Q, int32_t* best, double* score,
                                                         uint32_t staged) {
    extern __shared__ __align__(16) uint32_t s_pat[];
    if (staged) {
        for (uint32_t i = threadIdx.x; i < G.n * kMatchWords; i += blockDim.x) {
            const uint32_t p = i / kMatchWords, w = i % kMatchWords;
            uint32_t v;
            if (w < kMaxStages) v = G.ident[p * kMaxStages + w];
            else if (w < 2 * kMaxStages) v = G.in_len[p * kMaxStages + w - kMaxStages];
            else if (w < 3 * kMaxStages) v = G.out[p * kMaxStages + w - 2 * kMaxStages];
            else if (w == 3 * kMaxStages) v = G.n_stages[p];
            else v = G.reuse[p];
            s_pat[i] = v;
        }
        __syncthreads();
    }
    const PatView V{staged ? s_pat : nullptr, G};
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < Q.n; q += warps) {
        const uint32_t s = min(Q.stage[q], kMaxStages);
        uint32_t qi[kMaxStages], qin[kMaxStages], qout[kMaxStages];
#pragma unroll
        for (uint32_t u = 0; u < kMaxStages; ++u) {
            qi[u] = Q.ident[q * kMaxStages + u];
            qin[u] = Q.in_len[q * kMaxStages + u];
            qout[u] = Q.out[q * kMaxStages + u];
        }
        double bs = -1.0;
        uint32_t br = 0, bp = 0xFFFFFFFFu;
        if (s < kMaxStages) {
            for (uint32_t p = lane; p < G.n; p += 32) {
                if (V.ns(p) <= s) continue;
                bool keep = true;
#pragma unroll
                for (uint32_t u = 0; u < kMaxStages; ++u)
                    if (u <= s && V.ident(p, u) != qi[u]) keep = false;
                if (!keep) continue;
                double sum = 0.0;
                uint32_t cnt = 0;
#pragma unroll
                for (uint32_t u = 0; u < kMaxStages; ++u) {
                    if (u > s) break;
                    if (u < s) { sum += kernel_sim(qout[u], V.out(p, u)); ++cnt; }
                    if (u >= 1 && !(qi[u] >> 31)) { sum += kernel_sim(qin[u], V.in(p, u)); ++cnt; }
                }
                const double sc = cnt ? sum / (double)cnt : 1.0;
                const uint32_t ru = V.reuse(p);
                if (bp == 0xFFFFFFFFu || sc > bs || (sc == bs && ru > br)) { bs = sc; br = ru; bp = p; }
            }
        }
        // warp reduction: (score desc, reuse desc, index asc); lanes visit ascending indices
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, bs, o);
            const uint32_t orr = __shfl_xor_sync(0xffffffffu, br, o), op = __shfl_xor_sync(0xffffffffu, bp, o);
            const bool take = op != 0xFFFFFFFFu &&
                              (bp == 0xFFFFFFFFu || os > bs || (os == bs && (orr > br || (orr == br && op < bp))));
            if (take) { bs = os; br = orr; bp = op; }
        }
        if (lane == 0) {
            best[q] = bp == 0xFFFFFFFFu ? -1 : (int32_t)bp;
            score[q] = bp == 0xFFFFFFFFu ? -1.0 : bs;
        }
    }
}

// the matched patterns' stage structure becomes the tasks' (n_stages, stage times): the
// dependency estimate of a4; a query's stage must be its task's current stage
__global__ void k_apply_match(Pool P, PatternsDev G, QueriesDev Q, const int32_t* best, uint32_t* err) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < Q.n; q += gridDim.x * blockDim.x) {
        const int32_t b = best[q];
        const uint32_t t = Q.task[q];
        if (b < 0) continue;
        if (t >= P.n_tasks || P.cur_stage[t] != Q.stage[q]) { atomicOr(err, 16u); continue; }
        P.n_stages[t] = G.n_stages[b];
        for (uint32_t u = 0; u < kMaxStages; ++u)
            P.pattern[(size_t)t * kMaxStages + u] = u < G.n_stages[b] ? G.t_ms[(size_t)b * kMaxStages + u] : 0u;
    }
}

}  // namespace jit
