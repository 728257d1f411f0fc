// select.cuh -- shared types of the pool step (Pool, Ctrl, Scratch, TaskInfo, ...), the row
// scoring helpers used by the replay, and the EXACT path of the step (sm_100a).
//
// The step itself is k_score (stream.cuh) -> k_spec (spec.cuh, the speculative
// resolve).  When the speculation cannot be exact, finish_step (abi.cu) re-scores the pool with
// every key materialized (k_score, kMat) and runs the exact path from the host:
//   k_hist0    level-0 cost-weighted histogram of the composite key (key desc, id asc); the last
//              CTA resolves the boundary bin
//   k_pass     one more 12-bit digit while the boundary bucket is larger than kBucketCap
//   k_compact  gathers the boundary bucket (composite key, cost) + the smallest key above it
//   k_resolve  one CTA: sorts the bucket, block-scans costs -> exact B*, bp, thr (a7, a8)
//   k_cand     compacts Cd = {key >= thr} (warp ballots)
//   k_group    one CTA: sorts Cd by (len, id), u64/u128 prefix sums, sliding windows within
//              the token budget, first argmax (a9); writes the batch and the bookkeeping
//   k_publish  copies the control block to pinned host memory
#pragma once
#include "common.cuh"
#include "pool.cuh"

namespace jit {

constexpr uint32_t kBucketCap = 4096;
constexpr uint32_t kSpecCap = 8192;            // speculative set resolved in shared memory up to this size
constexpr uint32_t kGroupSmemSort = 8192;     // |Cd| sorted in shared memory up to this size
constexpr uint32_t kGroupSmemWin = 4096;      // |Cd| whose window prefix sums live in shared memory
constexpr uint32_t kGroupPfOff = (12 * kGroupSmemSort + 8 * (kGroupSmemWin + 1) + 15) & ~15u;
constexpr uint32_t kGroupSmemBytes = kGroupPfOff + 16 * (kGroupSmemWin + 1);   // k_group's dynamic smem
static_assert(kGroupSmemBytes <= 227 * 1024, "k_group shared memory");
constexpr uint32_t kPassThreads = 512;

enum : uint32_t { ST_RUN = 0, ST_HIST = 1, ST_COMPACT = 2, ST_RESOLVED = 3, ST_EMPTY = 4, ST_ERROR = 5, ST_FALLBACK = 6,
                  ST_SPEC_BIG = 7 };

struct alignas(16) Ctrl {
    u128 prefix;                     // digits resolved so far (top bits of the composite key)
    int64_t now, v;
    unsigned long long min_img;      // smallest key image over pending rows
    unsigned long long pred_min_img; // smallest key image above the final bucket
    unsigned long long before_cost;  // cost of the rows strictly above the current bucket
    unsigned long long thr_img;
    double bp, thr;
    uint32_t n_pending, n_dropped, error, status;
    uint32_t level, bucket_count, bucket_fill, before_count;
    uint32_t b_star, n_cand, n_selected, total_tokens;
    uint32_t done[16];
    uint32_t i_best, j_best, cand_overflow, exp_fill;
    unsigned long long tot_cost;     // sum of the token costs of all pending rows
    uint32_t spec_n, spec_ovf, fallback, window_done;
    uint32_t n_refresh;                         // length-bound refreshes this step (a2)
    uint32_t batch_on_host;                     // 1: the batch is in the pinned host mirror (fast path)
    uint32_t steps, fallbacks;                  // the handle's counters after this step (Persist)
    uint32_t trace, pad_t;                      // exact-path kernels that ran (bit mask)
    unsigned long long ts[12];                  // %globaltimer stamps of the single-CTA phases (JIT_PHASE_STAMPS)
};

// state that survives across steps of one handle (not cleared by a step)
struct Persist {
    unsigned long long t_guess;      // speculative key-image threshold for the next step
    uint32_t steps;                  // step counter: the steps_waited stamps count against it
    uint32_t fallbacks;              // steps resolved by the exact path (device count)
    uint32_t host_pending;           // 1: the last step needs the host (exact path / big set / k_group)
    uint32_t skipped;                // chained steps that did nothing because of host_pending
};

// the step's k_score partials, reduced by atomics (one set per CTA), read and reset by k_spec
struct BlockPart {
    unsigned long long cnt;          // pending (bits 0-31) | dropped this step (bits 32-63)
    uint32_t refresh, err;
};

// %globaltimer (ns) stamp of a phase boundary, taken by thread 0 of a single-CTA kernel
// (diagnostics only: compiled in with -DJIT_PHASE_STAMPS)
__device__ __forceinline__ void stamp(Ctrl* ctrl, int i) {
#ifdef JIT_PHASE_STAMPS
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ctrl->ts[i] = t;
    }
#else
    (void)ctrl; (void)i;
#endif
}

// bookkeeping of one selected row (the batch of Alg. 1): ever_scheduled, Queued / Preempted ->
// Running, and its steps_waited stamp moves with the counter (a selected request keeps its count)
__device__ __forceinline__ void book_selected(const Pool& P, uint32_t r, uint32_t meta, uint32_t since, uint32_t sc) {
    uint32_t mt = meta | (kEver << 12);
    if (m_state(mt) == kQueued || m_state(mt) == kPreempted) mt = m_with_state(mt, kRunning);
    *reinterpret_cast<uint2*>(&P.rows[r].meta) = make_uint2(mt, since_after_select(since, sc));
    if (m_flags(meta) & kCompound) P.tever[P.task[r]] = 1u;      // the task has been scheduled (A40)
}
// thread 0 of the resolving kernel, after the batch: next step's speculative threshold and the counters
// the next step's speculative threshold t = fl(margin x this step's cutoff thr).  C3 on B200: 0.85
// 24.9 us per step, 0.93 24.7, 0.97 23.8 (the set shrinks toward Cd; k_spec's O(|S|^2) ranks),
// 0 fallbacks over the timed chains and the serving loop with arrivals either way
#ifndef JIT_STEP_MARGIN
#define JIT_STEP_MARGIN 0.97
#endif
__device__ __forceinline__ void finish_counters(Persist* ps, Ctrl* ctrl) {
    ps->t_guess = (unsigned long long)__double_as_longlong(__dmul_rn(ctrl->thr, JIT_STEP_MARGIN));
    ps->steps += 1;
    ps->fallbacks += ctrl->fallback;
    ctrl->steps = ps->steps; ctrl->fallbacks = ps->fallbacks;
}

struct Scratch {
    uint32_t* hcnt;          // 4096
    unsigned long long* hcost;  // 4096
    u128* bucket_ck;         // kBucketCap
    uint32_t* bucket_cost;   // kBucketCap
    uint32_t* cand;          // candidate rows (capacity)
    uint64_t* sk;            // global sort keys (capacity)   -- large-|Cd| path
    uint32_t* sv;            // global sort values
    unsigned long long* pc;  // prefix costs (capacity+1)
    u128* pf;                // prefix fixed-point keys (capacity+1)
    uint32_t* out_ids;       // max_batch
    uint32_t* out_tokens;
    uint32_t* out_rows;
    uint32_t cand_cap, pad;
    // the speculative set (kSpecCap entries): rows with key image >= t_guess, with what k_spec
    // needs of them (key image, id, row, token cost, window length key, meta and since stamp)
    uint64_t* spec_img;
    uint32_t *spec_id, *spec_row, *spec_cost, *spec_len, *spec_meta, *spec_aux;
    Persist* persist;
    BlockPart* gpart;        // the step's k_score partials, reduced atomically (reset by k_spec)
    const Item* items;       // work items of k_score (standalone row ranges, compound task ranges)
    const uint32_t* n_items; // device count of items (appends grow it without a graph update)
    uint32_t item_cap;         // capacity of items[] (every slot readable)
    uint32_t n_std_items;      // items [0, n_std_items) are the standalone chunks of [0, n_single)
    uint32_t bal_w;            // k_score balance: cost of one ring item in 1/256 standalone slabs (std_slabs)
    uint32_t n_ring_h;         // ring items at launch (host count; only balances the standalone slabs)
    unsigned int* spec_cnt;  // size of the speculative set (k_score atomics; reset by k_spec)
    Ctrl* h_ctrl;            // pinned host copy of the control block, written by the step's last kernel
    uint32_t* h_batch;       // pinned host mirror of the batch: ids | tokens | rows, (max_batch + 1) each
    unsigned long long* mwin;   // NEXT-2 power-of-K: per row (epoch << 8) | (255 - winner rank) (multi.cuh)
};

// The last kernel of a step writes the control block straight into pinned host memory (no
// memcpy node in the graph); whole block, after its last write to ctrl.
__device__ __forceinline__ void publish_ctrl(const Ctrl* ctrl, Ctrl* host) {
    __syncthreads();
    constexpr uint32_t kWords = sizeof(Ctrl) / 16;
    static_assert(sizeof(Ctrl) % 16 == 0, "ctrl is copied in 16-byte words");
    for (uint32_t i = threadIdx.x; i < kWords; i += blockDim.x)
        reinterpret_cast<uint4*>(host)[i] = __ldcg(reinterpret_cast<const uint4*>(ctrl) + i);
    // no system fence: the host reads the block only after synchronizing with the stream, and
    // kernel completion makes these writes visible
}

__device__ __forceinline__ bool is_last_block(uint32_t* counter) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t prev = atomicAdd(counter, 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// warp-aggregated shared-memory histogram update (all 32 lanes must call convergently)
__device__ __forceinline__ void warp_hist_add(uint32_t* s_cnt, uint32_t* s_cost, bool valid, uint32_t bin,
                                              uint32_t cost) {
    const int lane = threadIdx.x & 31;
    unsigned todo = __ballot_sync(0xffffffffu, valid);
    while (todo) {
        const int leader = __ffs(todo) - 1;
        const uint32_t b = __shfl_sync(0xffffffffu, bin, leader);
        const bool mine = valid && bin == b;
        const unsigned m = __ballot_sync(0xffffffffu, mine);
        const uint32_t c = __reduce_add_sync(0xffffffffu, mine ? cost : 0u);
        if (lane == leader) {
            atomicAdd(&s_cnt[b], (uint32_t)__popc(m));
            atomicAdd(&s_cost[b], c);
        }
        todo &= ~m;
    }
}

// --------------------------------------------------------------------------------------
// Resolve one radix level from the global histogram (executed by the last CTA of a pass).
// Bins are in ascending composite-key order = descending key.  The boundary bin is the
// first whose inclusive cumulative (count, cost), plus what lies above the bucket, exceeds
// (max_batch, token_budget) -- the (B*+1)-th request of Alg. 1's priority order lies in it.
// --------------------------------------------------------------------------------------
static __device__ void resolve_level(const Cfg& c, Ctrl* ctrl, uint32_t* hcnt, unsigned long long* hcost, uint32_t L) {
    __shared__ uint64_t s_scan[32];
    __shared__ uint32_t s_first;
    const uint32_t nb = digit_bins(L);
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint64_t lc = 0, lk = 0;
    for (uint32_t k = 0; k < per; ++k) {
        uint32_t b = b0 + k;
        if (b < nb) { lc += __ldcg(hcnt + b); lk += __ldcg(hcost + b); }
    }
    uint64_t tc, tk;
    uint64_t ec = block_exclusive_scan_u64(lc, s_scan, &tc);
    uint64_t ek = block_exclusive_scan_u64(lk, s_scan, &tk);
    if (threadIdx.x == 0) s_first = nb;
    __syncthreads();
    const uint64_t bc = ctrl->before_count, bk = ctrl->before_cost;
    uint64_t cc = ec, ck = ek;
    uint32_t my_first = nb;
    uint64_t my_exc = 0, my_exk = 0;
    for (uint32_t k = 0; k < per; ++k) {
        uint32_t b = b0 + k;
        if (b >= nb) break;
        const uint64_t hc = __ldcg(hcnt + b), hk = __ldcg(hcost + b);
        if (bc + cc + hc > c.max_batch || bk + ck + hk > c.token_budget) {
            my_first = b; my_exc = cc; my_exk = ck;
            atomicMin(&s_first, b);
            break;
        }
        cc += hc; ck += hk;
    }
    __syncthreads();
    const uint32_t first = s_first;
    if (my_first == first && first < nb) {     // the owner of the boundary bin publishes it
        if (ctrl->error) {
            ctrl->status = ST_ERROR;
        } else if (L == 0 && ctrl->n_pending == 0) {
            ctrl->status = ST_EMPTY;
        } else {
            ctrl->before_count += (uint32_t)my_exc;
            ctrl->before_cost += my_exk;
            ctrl->prefix = (L == 0) ? (u128)first : ((ctrl->prefix << 12) | (u128)first);
            ctrl->bucket_count = __ldcg(hcnt + first);
            ctrl->level = L + 1;
            ctrl->status = (ctrl->bucket_count <= kBucketCap) ? ST_COMPACT : ST_HIST;
        }
    }
    if (threadIdx.x == 0 && first == nb) {
        if (ctrl->error) {
            ctrl->status = ST_ERROR;
        } else if (ctrl->n_pending == 0) {
            ctrl->status = ST_EMPTY;
        } else if (L == 0) {
            // every pending request fits: B* = |P| and bp = the minimum key (A15)
            ctrl->b_star = ctrl->n_pending;
            const double bp = __longlong_as_double((long long)ctrl->min_img);
            ctrl->bp = bp;
            ctrl->thr = __dmul_rn(c.p, bp);
            ctrl->thr_img = (unsigned long long)__double_as_longlong(ctrl->thr);
            ctrl->status = ST_RESOLVED;
        } else {
            ctrl->error = 4; ctrl->status = ST_ERROR;     // a boundary bucket must contain the boundary
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < 4096; b += blockDim.x) { hcnt[b] = 0; hcost[b] = 0; }
}

// --------------------------------------------------------------------------------------
// k_begin
// --------------------------------------------------------------------------------------
// fresh control block of a step (written by one thread before any other use in the step)
__device__ __forceinline__ void reset_ctrl(Ctrl* ctrl, int64_t now, int64_t v) {
    Ctrl z;
    memset(&z, 0, sizeof(z));
    z.now = now; z.v = v;
    z.min_img = kNone; z.pred_min_img = kNone;
    *ctrl = z;
}

// the same by a whole CTA in 16-byte words (no Ctrl temporary in registers / on the stack)
__device__ __forceinline__ void reset_ctrl_block(Ctrl* ctrl, int64_t now, int64_t v) {
    for (uint32_t i = threadIdx.x; i < sizeof(Ctrl) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(ctrl)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (threadIdx.x == 0) { ctrl->now = now; ctrl->v = v; ctrl->min_img = kNone; ctrl->pred_min_img = kNone; }
}

#ifndef JIT_EXACT_TU
// full reset (load / sharded step); the graph step needs none: k_score resets ctrl and the
// histograms, k_spec the set counter
__global__ void k_begin(Ctrl* ctrl, uint32_t* hcnt, unsigned long long* hcost, int64_t now, int64_t v,
                        unsigned int* spec_cnt) {
    const uint32_t tid = threadIdx.x + blockIdx.x * blockDim.x, nt = blockDim.x * gridDim.x;
    for (uint32_t b = tid; b < 4096; b += nt) { hcnt[b] = 0; hcost[b] = 0; }
    if (tid == 0) { reset_ctrl(ctrl, now, v); *spec_cnt = 0; }
}
#endif  // !JIT_EXACT_TU

// ======================================================================================
// The exact path (radix select .. window): compiled into the separately linked unit
// exact.cu only, because k_spec launches these kernels from the device (-rdc).
// ======================================================================================
// block exclusive scan of u128 (blockDim 1024)
__device__ __forceinline__ u128 block_exclusive_scan_u128(u128 v, u128* scratch, u128* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u128 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u128 y = shfl_up_u128(x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[wid] = x;
    __syncthreads();
    if (wid == 0) {
        u128 s = lane < nw ? scratch[lane] : (u128)0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u128 y = shfl_up_u128(s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) scratch[lane] = s;
    }
    __syncthreads();
    u128 base = wid ? scratch[wid - 1] : (u128)0;
    u128 t = scratch[nw - 1];
    __syncthreads();
    if (total) *total = t;
    return base + x - v;
}

// the window's two prefix sums (token cost u64, fixed-point key u128) in ONE exclusive block scan:
// three barriers for the pair instead of three each
__device__ __forceinline__ void block_exclusive_scan_pair(uint64_t vc, u128 vf, uint64_t* scr_c, u128* scr_f,
                                                          uint64_t& ec, u128& ef, uint64_t& tc, u128& tf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t xc = vc;
    u128 xf = vf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t yc = __shfl_up_sync(0xffffffffu, xc, o);
        const u128 yf = shfl_up_u128(xf, o);
        if (lane >= o) { xc += yc; xf += yf; }
    }
    if (lane == 31) { scr_c[wid] = xc; scr_f[wid] = xf; }
    __syncthreads();
    if (wid == 0) {
        uint64_t sc = lane < nw ? scr_c[lane] : 0ull;
        u128 sf = lane < nw ? scr_f[lane] : (u128)0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t yc = __shfl_up_sync(0xffffffffu, sc, o);
            const u128 yf = shfl_up_u128(sf, o);
            if (lane >= o) { sc += yc; sf += yf; }
        }
        if (lane < nw) { scr_c[lane] = sc; scr_f[lane] = sf; }
    }
    __syncthreads();
    const uint64_t bc = wid ? scr_c[wid - 1] : 0ull;
    const u128 bf = wid ? scr_f[wid - 1] : (u128)0;
    tc = scr_c[nw - 1]; tf = scr_f[nw - 1];
    __syncthreads();
    ec = bc + xc - vc; ef = bf + xf - vf;
}

#ifdef JIT_EXACT_TU
// The exact path (host-launched by finish_step when the speculative resolve cannot be exact):
// k_hist0 -> k_pass x <= 7 -> k_compact -> k_resolve -> k_cand -> k_group; each kernel returns at
// once unless the control block's status says it has work.
__global__ void k_pass(Pool P, Cfg c, Ctrl* ctrl, Scratch S, uint32_t pass_idx);
__global__ void k_compact(Pool P, Cfg c, Ctrl* ctrl, Scratch S);
__global__ void k_resolve(Pool P, Cfg c, Ctrl* ctrl, Scratch S);
__global__ void k_cand(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int only_after_fallback);
__global__ void k_group(Pool P, Cfg c, Ctrl* ctrl, Scratch S);

// level-0 histogram of the key images (fallback path only), last CTA resolves level 0
__global__ void __launch_bounds__(kPassThreads) k_hist0(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int force) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctrl->trace, 4u);
    if (!force && ctrl->status != ST_FALLBACK) return;
    uint32_t* hcnt = S.hcnt;
    unsigned long long* hcost = S.hcost;
    __shared__ uint32_t s_cnt[2048], s_cost[2048];
    for (uint32_t b = threadIdx.x; b < 2048; b += blockDim.x) { s_cnt[b] = 0; s_cost[b] = 0; }
    __syncthreads();
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < P.n; wr += stride) {
        const uint32_t r = wr + (threadIdx.x & 31);
        uint64_t img = kNone;
        uint32_t cost = 0;
        if (r < P.n) { img = P.img[r]; cost = P.cost[r]; }
        const bool valid = img != kNone;
        const uint32_t bin = (uint32_t)(make_ck(img, 0) >> digit_shift(0)) & 2047u;
        warp_hist_add(s_cnt, s_cost, valid, bin, cost);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < 2048; b += blockDim.x)
        if (s_cnt[b]) { atomicAdd(hcnt + b, s_cnt[b]); atomicAdd(hcost + b, (unsigned long long)s_cost[b]); }
    if (is_last_block(&ctrl->done[0])) {
        resolve_level(c, ctrl, hcnt, hcost, 0);
    }
}

// --------------------------------------------------------------------------------------
// k_pass: one further digit of the cost-weighted radix select (only while status == HIST)
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kPassThreads) k_pass(Pool P, Cfg c, Ctrl* ctrl, Scratch S, uint32_t pass_idx) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctrl->trace, 16u);
    if (ctrl->status != ST_HIST) return;
    uint32_t* hcnt = S.hcnt;
    unsigned long long* hcost = S.hcost;
    __shared__ uint32_t s_cnt[4096], s_cost[4096];
    for (uint32_t b = threadIdx.x; b < 4096; b += blockDim.x) { s_cnt[b] = 0; s_cost[b] = 0; }
    __syncthreads();
    const uint32_t L = ctrl->level;
    const u128 prefix = ctrl->prefix;
    const uint32_t sh_prev = digit_shift(L - 1), sh = digit_shift(L);
    const bool need_id = sh < 32;
    const uint32_t stride = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < P.n; wr += stride) {
        const uint32_t r = wr + lane;
        bool valid = false;
        uint32_t bin = 0, cost = 0;
        if (r < P.n) {
            const uint64_t img = P.img[r];
            if (img != kNone) {
                const u128 ck = make_ck(img, need_id ? P.id[r] : 0u);
                if ((ck >> sh_prev) == prefix) {
                    valid = true;
                    bin = (uint32_t)(ck >> sh) & 4095u;
                    cost = P.cost[r];
                }
            }
        }
        warp_hist_add(s_cnt, s_cost, valid, bin, cost);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < 4096; b += blockDim.x)
        if (s_cnt[b]) { atomicAdd(hcnt + b, s_cnt[b]); atomicAdd(hcost + b, (unsigned long long)s_cost[b]); }
    if (is_last_block(&ctrl->done[1 + (pass_idx & 7)])) {
        resolve_level(c, ctrl, hcnt, hcost, L);
    }
}

// --------------------------------------------------------------------------------------
// k_compact: gather the final bucket and the smallest key image above it
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kPassThreads) k_compact(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctrl->trace, 32u);
    if (ctrl->status != ST_COMPACT) return;
    const uint32_t L = ctrl->level;
    const u128 prefix = ctrl->prefix;
    const uint32_t sh_prev = digit_shift(L - 1);
    const bool need_id_prefix = sh_prev < 32;
    const uint32_t stride = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    uint64_t my_min = kNone;
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < P.n; wr += stride) {
        const uint32_t r = wr + lane;
        bool take = false;
        u128 ck = 0;
        if (r < P.n) {
            const uint64_t img = P.img[r];
            if (img != kNone) {
                ck = make_ck(img, need_id_prefix ? P.id[r] : 0u);
                const u128 top = ck >> sh_prev;
                if (top == prefix) { take = true; if (!need_id_prefix) ck |= (u128)P.id[r]; }
                else if (top < prefix && img < my_min) my_min = img;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&ctrl->bucket_fill, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (take) {
                const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < kBucketCap) { S.bucket_ck[slot] = ck; S.bucket_cost[slot] = P.cost[r]; }
            }
        }
    }
    my_min = warp_min_u64(my_min);
    if (lane == 0 && my_min != kNone) atomicMin(&ctrl->pred_min_img, (unsigned long long)my_min);
}

// --------------------------------------------------------------------------------------
// k_resolve: one CTA (1024 threads) -- exact B*, bp, thr from the sorted bucket (a7, a8)
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_resolve(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    if (threadIdx.x == 0) atomicOr(&ctrl->trace, 64u);
    if (ctrl->status != ST_COMPACT) return;
    extern __shared__ __align__(16) unsigned char smem[];
    u128* sk = reinterpret_cast<u128*>(smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(smem + sizeof(u128) * kBucketCap);
    __shared__ uint64_t s_scan[32];
    __shared__ uint32_t s_fit;
    const uint32_t n = ctrl->bucket_fill;
    if (n > kBucketCap || n != ctrl->bucket_count) {       // cannot happen: counts are exact
        if (threadIdx.x == 0) { ctrl->error = 1; ctrl->status = ST_ERROR; }
        return;
    }
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < n) { sk[i] = S.bucket_ck[i]; sv[i] = S.bucket_cost[i]; }
        else { sk[i] = ~(u128)0; sv[i] = 0; }
    }
    __syncthreads();
    block_sort<u128>(sk, sv, n2);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) { S.bucket_ck[i] = sk[i]; S.bucket_cost[i] = sv[i]; }
    // block scan of costs over the sorted bucket (4 consecutive per thread)
    const uint32_t i0 = threadIdx.x * 4;
    uint64_t loc = 0;
    for (uint32_t k = 0; k < 4; ++k) if (i0 + k < n) loc += sv[i0 + k];
    uint64_t tot;
    uint64_t ex = block_exclusive_scan_u64(loc, s_scan, &tot);
    if (threadIdx.x == 0) s_fit = 0;
    __syncthreads();
    const uint64_t bc = ctrl->before_count, bk = ctrl->before_cost;
    uint32_t fits = 0;
    uint64_t run = ex;
    for (uint32_t k = 0; k < 4; ++k) {
        const uint32_t i = i0 + k;
        if (i >= n) break;
        run += sv[i];
        if (bc + i + 1 <= c.max_batch && bk + run <= c.token_budget) ++fits;   // monotone predicate
    }
    if (fits) atomicAdd(&s_fit, fits);
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nf = s_fit;
        ctrl->b_star = (uint32_t)bc + nf;
        const uint64_t bimg = nf ? ck_img(sk[nf - 1]) : (uint64_t)ctrl->pred_min_img;
        const double bp = __longlong_as_double((long long)bimg);
        ctrl->bp = bp;
        ctrl->thr = __dmul_rn(c.p, bp);   // A16
        ctrl->thr_img = (unsigned long long)__double_as_longlong(ctrl->thr);
        if (nf == 0 && ctrl->pred_min_img == kNone) { ctrl->error = 1; ctrl->status = ST_ERROR; }
        else ctrl->status = ST_RESOLVED;
    }
}

// --------------------------------------------------------------------------------------
// k_cand: Cd = {pending : key >= thr} (Alg. 1 Filter)
// --------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kPassThreads) k_cand(Pool P, Cfg c, Ctrl* ctrl, Scratch S, int only_after_fallback) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctrl->trace, 128u);
    if (ctrl->status != ST_RESOLVED) return;
    if (only_after_fallback && !ctrl->fallback) return;      // k_spec already produced Cd
    const uint64_t thr_img = ctrl->thr_img;
    const uint32_t stride = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (uint32_t wr = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wr < P.n; wr += stride) {
        const uint32_t r = wr + lane;
        bool take = false;
        if (r < P.n) {
            const uint64_t img = P.img[r];
            take = img != kNone && img >= thr_img;
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (m) {
            uint32_t base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&ctrl->n_cand, (uint32_t)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (take) {
                const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < S.cand_cap) S.cand[slot] = r; else ctrl->cand_overflow = 1;
            }
        }
    }
}


#endif  // JIT_EXACT_TU

// --------------------------------------------------------------------------------------
// (a9) Alg. 1 step 2 under the token budget, executed by ONE CTA of 1024 threads:
// sort Cd by (len asc, id asc), u64 prefix of costs and u128 prefix of fixed-point keys,
// j(i) = largest window end within tau and B_max (binary search), first argmax of the window
// score (strict '>').  sk/sv: n2 (power of two) sort slots; pc/pf: n+1 prefix slots
// (shared memory when they fit, else global scratch).  Writes the batch and the bookkeeping
// (ever_scheduled, Running, undo steps_waited+1) and the next step's speculative threshold.
// --------------------------------------------------------------------------------------
static __device__ void window_select(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint64_t* sk, uint32_t* sv,
                              uint32_t n, unsigned long long* pc, u128* pf) {
    __shared__ u128 s_scan128[32];
    __shared__ uint64_t s_scan[32];
    __shared__ u128 s_best[32];
    __shared__ uint32_t s_bi[32], s_bj[32];
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (uint32_t i = n + threadIdx.x; i < n2; i += blockDim.x) { sk[i] = ~0ull; sv[i] = 0; }
    __syncthreads();
    stamp(ctrl, 6);
    block_sort_wide(sk, sv, n2);
    stamp(ctrl, 7);
    uint64_t carry_c = 0;
    u128 carry_f = 0;
    for (uint32_t base = 0; base < n; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint64_t cv = 0; u128 fv = 0;
        if (i < n) {
            const uint32_t r = sv[i];
            cv = P.cost[r];
            fv = (u128)fixed_point(__longlong_as_double((long long)P.img[r]));
        }
        uint64_t tc, ec; u128 tf, ef;
        block_exclusive_scan_pair(cv, fv, s_scan, s_scan128, ec, ef, tc, tf);
        if (i < n) { pc[i] = carry_c + ec; pf[i] = carry_f + ef; }
        carry_c += tc; carry_f += tf;
    }
    if (threadIdx.x == 0) { pc[n] = carry_c; pf[n] = carry_f; }
    __syncthreads();
    stamp(ctrl, 8);
    u128 best = 0; uint32_t bi = 0xFFFFFFFFu, bj = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t lim = (uint64_t)pc[i] + c.token_budget;
        uint32_t lo = i, hi = (uint32_t)min((uint64_t)n - 1, (uint64_t)i + c.max_batch - 1);
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (pc[mid + 1] <= lim) lo = mid; else hi = mid - 1;
        }
        const u128 sc = pf[lo + 1] - pf[i];
        if (bi == 0xFFFFFFFFu || sc > best) { best = sc; bi = i; bj = lo; }   // i increasing per thread
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const u128 ob = shfl_xor_u128(best, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o), oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if ((oi != 0xFFFFFFFFu) && (bi == 0xFFFFFFFFu || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; bj = oj; }
    }
    if (lane == 0) { s_best[wid] = best; s_bi[wid] = bi; s_bj[wid] = bj; }
    __syncthreads();
    if (wid == 0) {
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
    bi = s_bi[0]; bj = s_bj[0];
    stamp(ctrl, 9);
    const uint32_t ns = bj - bi + 1;
    const uint32_t sc = S.persist->steps;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < ns; k += blockDim.x) {
        const uint32_t r = sv[bi + k];
        S.out_ids[k] = P.id[r];
        S.out_tokens[k] = P.cost[r];
        S.out_rows[k] = r;
        book_selected(P, r, P.rows[r].meta, P.rows[r].since, sc);
    }
    if (threadIdx.x == 0) {
        ctrl->n_selected = ns;
        ctrl->total_tokens = (uint32_t)(pc[bj + 1] - pc[bi]);
        ctrl->i_best = bi; ctrl->j_best = bj;
        ctrl->window_done = 1;
        finish_counters(S.persist, ctrl);      // next step's threshold: this cutoff with a 3% margin
    }
    stamp(ctrl, 10);
}

#ifdef JIT_EXACT_TU
// k_group: the window over Cd = S.cand (after the radix path or a too-large speculative Cd)
static __device__ void group_body(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, unsigned char* smem);
__global__ void __launch_bounds__(1024) k_group(Pool P, Cfg c, Ctrl* ctrl, Scratch S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_run;
    if (threadIdx.x == 0) { s_run = ctrl->status == ST_RESOLVED && !ctrl->window_done; atomicOr(&ctrl->trace, 256u); }
    __syncthreads();
    if (s_run) group_body(P, c, ctrl, S, smem);
}

static __device__ void group_body(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, unsigned char* smem) {
    const uint32_t n = ctrl->n_cand;
    if (ctrl->cand_overflow || n == 0) {
        if (threadIdx.x == 0) { ctrl->error = 1; ctrl->status = ST_ERROR; }
        return;
    }
    uint32_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    uint64_t* sk;
    uint32_t* sv;
    if (n2 <= kGroupSmemSort) { sk = reinterpret_cast<uint64_t*>(smem); sv = reinterpret_cast<uint32_t*>(smem + 8 * kGroupSmemSort); }
    else { sk = S.sk; sv = S.sv; }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t r = S.cand[i];
        const uint64_t len = c.len_key ? (uint64_t)P.rows[r].len_in + P.rows[r].gen : (uint64_t)P.rows[r].len_in;
        sk[i] = (len << 32) | P.id[r];                      // (len asc, id asc), A17/A18
        sv[i] = r;
    }
    // the window's prefix sums (read by every start's binary search) in shared memory when they fit
    const bool win_smem = n <= kGroupSmemWin;
    window_select(P, c, ctrl, S, sk, sv, n,
                  win_smem ? reinterpret_cast<unsigned long long*>(smem + 12 * kGroupSmemSort) : S.pc,
                  win_smem ? reinterpret_cast<u128*>(smem + kGroupPfOff) : S.pf);
}

#endif  // JIT_EXACT_TU

#ifndef JIT_EXACT_TU
// k_publish: copies the control block to pinned host memory (end of the host-run exact path)
__global__ void k_publish(const Ctrl* ctrl, Ctrl* host) { publish_ctrl(ctrl, host); }


// load: pack the caller's SoA pool into hot rows.  lrow = dist_row | L-hat unset; the count in
// aux's high half becomes the frozen steps_waited (the first step stamps the pending rows).
// A row with g < R has the anchor 0, so its cached bound is the table row's unconditioned
// quantile Q_q(L | L > 0): set from the per-row table (lhat0, nullptr with a forest) when a row
// enters the pool (k_validate after a load / an arrival), epoch field 1 -- the bound the pass's
// refresh would compute, without a search on the step's path.
__device__ __forceinline__ void seed_bound(HotRow& q, const uint32_t* lhat0, uint32_t n_rows, uint32_t R) {
    const uint32_t drow = q.lrow & 0xFFFFu;
    if (lhat0 && q.gen < R && drow < n_rows) {
        q.lrow = drow | (__ldg(lhat0 + drow) << 16);
        q.meta = (q.meta & 0xFFFFu) | (1u << 16);
    }
}
__global__ void k_lhat0(Table T, uint32_t qn, uint32_t qd) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < T.n_rows; r += gridDim.x * blockDim.x)
        T.lhat0[r] = cond_quantile(T, r, 0u, qn, qd);
}
__global__ void k_pack(HotRow* rows, uint32_t n, const int64_t* arr, const uint32_t* len_in, const uint32_t* gen,
                       const uint32_t* pre, const uint32_t* meta, const uint32_t* aux) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        HotRow q;
        q.arr = arr[r]; q.len_in = len_in[r]; q.gen = gen[r]; q.pre = pre[r];
        q.lrow = aux[r] & 0xFFFFu;
        q.meta = meta[r] & ~(kStamped << 12);     // caller meta: bits 16-31 zero (validated)
        q.since = aux[r] >> 16;
        rows[r] = q;
    }
}

// progress updates from the engine (keyed by request id or by row), applied before the step's
// pass.  A row leaving the pending set freezes its steps_waited (the handle's counter); the ranges
// the pass relies on are checked (generated < 2^24, prefilled <= L_i, state <= Moved, no way out
// of Done / Dropped / Moved, known id); a violation fails the step (gpart->err).
__global__ void k_progress(Pool P, Scratch S, const uint32_t* key, const uint32_t* gen, const uint32_t* pre,
                           const uint32_t* state, uint32_t n, int by_id) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = by_id ? map_find(P, key[i]) : key[i];
    if (r >= P.n) { atomicOr(&S.gpart->err, 8u); return; }
    HotRow* rp = P.rows + r;
    const uint32_t st = state[i], old_st = m_state(rp->meta);
    if (gen[i] >= (1u << 24) || pre[i] > rp->len_in || st > kMoved ||
        ((old_st == kDone || old_st == kDropped || old_st == kMoved) && st != old_st)) {
        atomicOr(&S.gpart->err, 8u);
        return;
    }
    uint32_t meta = m_with_state(rp->meta, st), since = rp->since;
    if ((meta >> 12) & kStamped && st > kPreempted) {          // left the pending set: freeze
        since = waited_of(meta, since, S.persist->steps);
        meta &= ~(kStamped << 12);
    }
    rp->gen = gen[i];
    rp->pre = pre[i];
    *reinterpret_cast<uint2*>(&rp->meta) = make_uint2(meta, since);
}

// request id -> row map: insert rows [r0, r1) (a duplicate id fails the load / step)
__device__ __forceinline__ void map_insert_row(const Pool& P, uint32_t id, uint32_t r, uint32_t* err) {
    const unsigned long long e = ((unsigned long long)id << 32) | r;
    for (uint32_t h = map_hash(id, P.map_mask), k = 0; k <= P.map_mask; h = (h + 1) & P.map_mask, ++k) {
        const unsigned long long old = atomicCAS(&P.idmap[h], kMapEmpty, e);
        if (old == kMapEmpty) break;
        if ((uint32_t)(old >> 32) == id) { atomicOr(err, 16u); break; }
    }
}
__global__ void k_map_insert(Pool P, uint32_t r0, uint32_t r1, uint32_t* err) {
    for (uint32_t r = r0 + blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += gridDim.x * blockDim.x)
        map_insert_row(P, P.id[r], r, err);
}

// the range / layout checks of one loaded or appended row (k_validate, k_arrive_std)
__device__ __forceinline__ bool row_invalid(const Pool& P, const Group* groups, uint32_t n_groups, uint32_t n_rows_tab,
                                            uint32_t l_max, uint32_t r, const HotRow& q, uint32_t std_end,
                                            uint32_t t_begin) {
    const uint32_t meta = q.meta;
    const uint32_t gi = m_group(meta);
    const bool comp = (m_flags(meta) & kCompound) != 0;
    bool rb = false;
    if (gi >= n_groups || l_row(q.lrow) >= n_rows_tab || q.len_in == 0 || q.len_in >= (1u << 24) ||
        q.gen >= (1u << 24) || q.pre > q.len_in || (meta >> 16) != 0 || m_state(meta) > kMoved ||
        q.since > 0xFFFFu || comp != (r >= std_end)) rb = true;
    else if (!comp) {
        if (P.task[r] != kNoTask || groups[gi].type == kCMP) rb = true;
    } else {
        const uint32_t t = P.task[r];
        if (t >= P.n_tasks || t < t_begin || groups[gi].type != kCMP || (m_flags(meta) & kOverride)) rb = true;
        else if (r < P.crng[t].x || r >= P.crng[t].y) rb = true;
        // a call's goodput w_in L_i + w_out L-hat stays below 2^27 (the pass sums 32 calls in u32)
        else if ((uint64_t)groups[gi].w_in * q.len_in + (uint64_t)groups[gi].w_out * (l_max + 1ull) >= (1ull << 27))
            rb = true;
    }
    if (!rb && (m_flags(meta) & kOverride) && groups[gi].type == kCMP) rb = true;
    return rb;
}

// arrivals: the new rows / tasks (staged SoA, arrival-local task indices and call offsets) appended
// after rows n0 and tasks t0 of the resident pool
struct Arrivals {
    const int64_t* arr; const uint32_t *len_in, *gen, *pre, *meta, *aux, *id, *task, *ovr;
    const uint32_t* fair;       // NULL: 0
    const uint32_t* call_off; const int64_t *t_arr, *t_dl; const uint32_t *cur_stage, *n_stages, *pattern;
    const uint64_t* gdone;
    uint32_t n, n_single, n_tasks, n0, t0, pad;
    const Item* items_src;      // the arrivals' new work items (staged with the deltas) ...
    Item* items_dst;            // ... copied to the item array here, with its new count
    uint32_t* n_items_dst;
    uint32_t n_new_items, n_items;
};
__global__ void k_append(Pool P, Arrivals A) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_new_items; i += stride) A.items_dst[i] = A.items_src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.n_items_dst = A.n_items;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += stride) {
        const uint32_t r = A.n0 + i;
        HotRow q;
        q.arr = A.arr[i]; q.len_in = A.len_in[i]; q.gen = A.gen[i]; q.pre = A.pre[i];
        q.lrow = A.aux[i] & 0xFFFFu;
        q.meta = A.meta[i] & ~(kStamped << 12);
        q.since = A.aux[i] >> 16;
        P.rows[r] = q;
        P.id[r] = A.id[i];
        P.task[r] = A.task[i] == kNoTask ? kNoTask : A.t0 + A.task[i];
        P.ovr[r] = A.ovr[i];
        P.fair[r] = A.fair ? A.fair[i] : 0u;
    }
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < A.n_tasks; t += stride) {
        const uint32_t g = A.t0 + t;
        P.t_arr[g] = A.t_arr[t]; P.t_dl[g] = A.t_dl[t]; P.cur_stage[g] = A.cur_stage[t]; P.n_stages[g] = A.n_stages[t];
        for (uint32_t u = 0; u < kMaxStages; ++u) P.pattern[(size_t)g * kMaxStages + u] = A.pattern[(size_t)t * kMaxStages + u];
        P.gdone[g] = A.gdone[t];
        P.crng[g] = make_uint2(A.n0 + A.call_off[t], A.n0 + A.call_off[t + 1]);
    }
}

// standalone-only arrivals in one launch: each new row appended, validated (row_invalid), its
// bound seeded (seed_bound) and its id inserted in the map; the new work items copied
__global__ void k_arrive_std(Pool P, Arrivals A, const Group* groups, uint32_t n_groups, uint32_t n_rows_tab,
                             uint32_t l_max, uint32_t* err, const uint32_t* lhat0, uint32_t R) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_new_items; i += stride) A.items_dst[i] = A.items_src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.n_items_dst = A.n_items;
    bool bad = false;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += stride) {
        const uint32_t r = A.n0 + i;
        HotRow q;
        q.arr = A.arr[i]; q.len_in = A.len_in[i]; q.gen = A.gen[i]; q.pre = A.pre[i];
        q.lrow = A.aux[i] & 0xFFFFu;
        q.meta = A.meta[i] & ~(kStamped << 12);
        q.since = A.aux[i] >> 16;
        const uint32_t id = A.id[i];
        P.id[r] = id;
        P.task[r] = A.task[i];                           // standalone: kNoTask (checked)
        P.ovr[r] = A.ovr[i];
        P.fair[r] = A.fair ? A.fair[i] : 0u;
        const bool rb = row_invalid(P, groups, n_groups, n_rows_tab, l_max, r, q, A.n0 + A.n, 0u);
        bad |= rb;
        if (!rb && lhat0 && q.gen < R) seed_bound(q, lhat0, n_rows_tab, R);
        P.rows[r] = q;
        map_insert_row(P, id, r, err);
    }
    if (bad) atomicOr(err, 2u);
}

// task updates: a new current stage (its sub-deadline from the pattern, or given), the goodput of
// the finished calls
__global__ void k_task_update(Pool P, const uint32_t* task, const uint32_t* stage, const uint64_t* gdone,
                              const int64_t* dls, uint32_t n, Scratch S) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = task[i];
    if (t >= P.n_tasks || stage[i] >= P.n_stages[t]) { atomicOr(&S.gpart->err, 8u); return; }
    P.cur_stage[t] = stage[i];
    P.gdone[t] = gdone[i];
    TaskInfo ti = P.tinfo[t];
    ti.gdone = gdone[i];
    if (dls && dls[i] >= 0) {
        ti.dls = dls[i];
    } else {
        uint64_t le = 0, tot = 0;
        for (uint32_t u = 0; u < kMaxStages; ++u) {
            const uint64_t ms = u < P.n_stages[t] ? P.pattern[(size_t)t * kMaxStages + u] : 0u;
            tot += ms; if (u <= stage[i]) le += ms;
        }
        const int64_t D = P.t_dl[t];
        ti.dls = P.t_arr[t] + (tot ? (int64_t)((u128)(uint64_t)D * le / tot) : 0);
    }
    P.tinfo[t] = ti;
}

// measurement only (jit_sched_time_scoring, JIT_TIME_FORCE_REFRESH): every cached bound stale
// every `stride`-th row from `phase` (stride 1: all) gets its cached length bound invalidated
__global__ void k_invalidate_bounds(Pool P, uint32_t stride = 1, uint32_t phase = 0) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < P.n; r += gridDim.x * blockDim.x)
        if (stride == 1 || r % stride == phase) P.rows[r].meta &= 0xFFFFu;   // epoch field 0: unset
}

// load: every task's call rows from the CSR
__global__ void k_crng_from_off(Pool P) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < P.n_tasks; t += gridDim.x * blockDim.x)
        P.crng[t] = make_uint2(P.call_off[t], P.call_off[t + 1]);
}

// every 2^30 steps: keep the stamps of rows that wait for ever within 0xFFFF of the counter, so
// that step - since never wraps (the count saturates at 0xFFFF anyway)
__global__ void k_rebase(Pool P, Scratch S) {
    const uint32_t sc = S.persist->steps;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < P.n; r += gridDim.x * blockDim.x) {
        HotRow* rp = P.rows + r;
        if (((rp->meta >> 12) & kStamped) && sc - rp->since > 0xFFFFu) rp->since = sc - 0xFFFFu;
    }
}

// tests (jit_sched_debug_set_counter): the counter moves by d, every stamp with it
__global__ void k_shift_stamps(Pool P, uint32_t d) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < P.n; r += gridDim.x * blockDim.x) {
        HotRow* rp = P.rows + r;
        if ((rp->meta >> 12) & kStamped) rp->since += d;
    }
}

// load-time per-task constants (TaskInfo); D * le fits u64 when D < 2^40 ns and t_total < 2^24 ms
__global__ void k_task_prep(Pool P, uint32_t t_begin) {
    for (uint32_t t = t_begin + blockIdx.x * blockDim.x + threadIdx.x; t < P.n_tasks; t += gridDim.x * blockDim.x) {
        const int64_t a_c = P.t_arr[t], D = P.t_dl[t];
        const uint32_t s = P.cur_stage[t], Sn = P.n_stages[t];
        uint64_t le = 0, tot = 0;
        for (uint32_t u = 0; u < kMaxStages; ++u) {
            const uint64_t ms = u < Sn ? P.pattern[(size_t)t * kMaxStages + u] : 0u;
            tot += ms; if (u <= s) le += ms;
        }
        const int64_t Ds = !tot ? 0
            : ((uint64_t)D < (1ull << 40) && tot < (1ull << 24)) ? (int64_t)((uint64_t)D * le / tot)
                                                                 : (int64_t)((u128)(uint64_t)D * le / tot);
        TaskInfo ti;
        ti.dls = a_c + Ds;                // advisory stage deadline: missing it only sets rate = inf
        ti.dlf = a_c + D;                 // final deadline: missing it zeroes the task goodput (A43)
        ti.ac = a_c;                      // admission of the task (A40)
        ti.gdone = P.gdone[t];
        P.tinfo[t] = ti;
        uint32_t ever = 0;                // A40: some call of the task in the pool was scheduled
        for (uint32_t r = P.crng[t].x; r < P.crng[t].y && r < P.n; ++r)
            ever |= (m_flags(P.rows[r].meta) & kEver) ? 1u : 0u;
        P.tever[t] = ever;
    }
}

// validation of loaded / appended rows [r_begin, n) and tasks [t_begin, n_tasks): rows
// [r_begin, std_end) are standalone, the rest compound calls inside their task's rows (crng);
// group types, ranges.  A load (t_begin == 0) also checks the CSR layout of jit_pool.
__global__ void k_validate(Pool P, const Group* groups, uint32_t n_groups, uint32_t n_rows_tab, uint32_t l_max,
                           uint32_t* err, uint32_t r_begin, uint32_t std_end, uint32_t t_begin,
                           const uint32_t* lhat0, uint32_t R) {
    const uint32_t stride = gridDim.x * blockDim.x;
    bool bad = false;
    for (uint32_t r = r_begin + blockIdx.x * blockDim.x + threadIdx.x; r < P.n; r += stride) {
        HotRow q = P.rows[r];
        const bool rb = row_invalid(P, groups, n_groups, n_rows_tab, l_max, r, q, std_end, t_begin);
        bad |= rb;
        if (!rb && lhat0 && q.gen < R) {                   // seed the bound of a row with g < R
            seed_bound(q, lhat0, n_rows_tab, R);
            P.rows[r].lrow = q.lrow;
            P.rows[r].meta = q.meta;
        }
    }
    for (uint32_t t = t_begin + blockIdx.x * blockDim.x + threadIdx.x; t < P.n_tasks; t += stride) {
        const uint32_t S = P.n_stages[t], s = P.cur_stage[t];
        if (P.crng[t].x > P.crng[t].y || P.crng[t].y > P.n || S == 0 || S > kMaxStages || s >= S) bad = true;
        else {
            uint64_t tot = 0;
            for (uint32_t u = 0; u < S; ++u) tot += P.pattern[t * kMaxStages + u];
            if (tot == 0) bad = true;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && t_begin == 0 && r_begin == 0) {   // a load: the CSR of jit_pool
        if (P.n_tasks && (P.call_off[0] != P.n_single || P.call_off[P.n_tasks] != P.n)) bad = true;
        if (!P.n_tasks && P.n_single != P.n) bad = true;
    }
    if (bad) atomicOr(err, 2u);
}

#endif  // !JIT_EXACT_TU

}  // namespace jit
