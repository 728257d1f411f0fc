// pool.cuh -- the request pool as it lives in HBM: one 32-byte hot row per
// request, read by every step with two 128-bit loads, plus cold per-row arrays read only for
// the rows a step selects (id, task, override R(k)) and the per-task constants of (a4).
//
// Hot row (32 B, 32-B aligned):
//   arr    i64  arrival (ns)
//   len_in u32  L_i
//   gen    u32  tokens generated g
//   pre    u32  prompt tokens prefilled
//   lrow   u32  dist_row (bits 0-15) | cached length bound L-hat (bits 16-31, 0 = unset)
//   meta   u32  group:8 | state:4 | flags:4 | epoch:16 (epoch = floor(g/R) of the cached bound)
//   since  u32  steps_waited as a stamp (flag kStamped): waited = min(step - since, 0xFFFF) with
//               `step` the handle's step counter; else the frozen count itself
//
// steps_waited as a stamp (reading A12/A41): a pending request left out of the batch waits one
// more step, a selected one keeps its count, a request that is not pending keeps its count.
// With the stamp the step counter does the +1 of every unselected pending row at once; the
// streaming pass writes a row only when it changes regime (it became pending: stamp it; it left
// the pending set: freeze the count), the batch bookkeeping moves a selected row's stamp by one.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace jit {

constexpr uint32_t kStamped = 8;               // meta flag: `since` holds a stamp (row is pending)

struct __align__(32) HotRow {
    int64_t arr;
    uint32_t len_in, gen, pre, lrow, meta, since;
};
static_assert(sizeof(HotRow) == 32, "hot row is 32 bytes");

__host__ __device__ __forceinline__ uint32_t l_row(uint32_t lrow) { return lrow & 0xFFFFu; }
__host__ __device__ __forceinline__ uint32_t l_hat(uint32_t lrow) { return lrow >> 16; }
__host__ __device__ __forceinline__ uint32_t m_flags_all(uint32_t m) { return (m >> 12) & 0xFu; }

// effective steps_waited of a row at step counter sc
__host__ __device__ __forceinline__ uint32_t waited_of(uint32_t meta, uint32_t since, uint32_t sc) {
    if (!((meta >> 12) & kStamped)) return since;
    const uint32_t d = sc - since;
    return d < 0xFFFFu ? d : 0xFFFFu;
}
// the stamp a selected row carries into the next step (its count unchanged; the distance to the
// counter stays <= 0xFFFF once saturated, so it never wraps)
__device__ __forceinline__ uint32_t since_after_select(uint32_t since, uint32_t sc) {
    return (sc - since) >= 0xFFFFu ? sc + 1u - 0xFFFFu : since + 1u;
}

__device__ __forceinline__ HotRow ld_row(const HotRow* p) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
    HotRow r;
    r.arr = (int64_t)(((uint64_t)a.y << 32) | a.x);
    r.len_in = a.z; r.gen = a.w; r.pre = b.x; r.lrow = b.y; r.meta = b.z; r.since = b.w;
    return r;
}

// per-task constants of the compound pass (a4), derived by k_task_prep from the task arrays:
// absolute stage sub-deadline a_c + D_s (D_s = floor(D * t_<=s / t_total)), absolute
// final deadline a_c + D, the task's arrival a_c (admission, A40), goodput of finished calls
struct TaskInfo {
    int64_t dls, dlf, ac;
    uint64_t gdone;
};

// a work item of the streaming pass: rows [r0, r1); standalone when t1 == t0, else whole compound
// tasks [t0, t1) (big: one task of more rows than an item holds, read in several chunks)
struct Item {
    uint32_t r0, r1, t0, t1;
};

struct Pool {
    HotRow* rows;
    uint32_t *id, *task, *ovr;
    uint32_t* fair;         // Fair(r) of the NEXT-2 blend (read only when it is on)
    uint64_t* img;          // materialized key images (exact path / debug): kNone when not pending
    uint32_t* cost;         // materialized token costs (0 when not pending)
    double* dbg_rate;       // optional debug outputs
    int64_t* dbg_trem;
    uint32_t* dbg_lhat;
    uint32_t n, n_single, n_tasks, pad;
    uint32_t* call_off;
    int64_t *t_arr, *t_dl;
    uint32_t *cur_stage, *n_stages, *pattern;
    uint64_t* gdone;
    TaskInfo* tinfo;
    uint32_t* tever;        // per task: 1 once any of its calls was scheduled (admission, A40)
    uint2* crng;            // per task: its call rows [begin, end) (load: the CSR; arrivals: appended blocks)
    unsigned long long* idmap;   // request id -> row: open addressing, (id << 32) | row, empty = ~0
    uint32_t map_mask, pad2;     // capacity - 1 (a power of two >= 2 x rows)
};

constexpr unsigned long long kMapEmpty = ~0ull;
__host__ __device__ __forceinline__ uint32_t map_hash(uint32_t id, uint32_t mask) {
    return (id * 0x9E3779B1u) & mask;
}
// the row of request `id`, or 0xFFFFFFFF
__device__ __forceinline__ uint32_t map_find(const Pool& P, uint32_t id) {
    for (uint32_t h = map_hash(id, P.map_mask), n = 0; n <= P.map_mask; h = (h + 1) & P.map_mask, ++n) {
        const unsigned long long e = P.idmap[h];
        if (e == kMapEmpty) return 0xFFFFFFFFu;
        if ((uint32_t)(e >> 32) == id) return (uint32_t)e;
    }
    return 0xFFFFFFFFu;
}

}  // namespace jit
