// exact_api.h -- host-side launchers of the kernels compiled into exact.cu: the speculative
// resolve (k_spec, k_spec_big) and the exact radix path the host runs when the speculation
// cannot be exact.
#pragma once
#include <cuda_runtime.h>
#include "select.cuh"

namespace jit {
namespace exact {

// function attributes (dynamic shared memory, carveout) of every exact.cu kernel
cudaError_t init_attributes();

// k_spec: reduce the scoring partials; reduce_only = 0: resolve from the speculative set and run
// the window, or mark the step for the host-driven exact path (status FALLBACK / window_done 0);
// publishes the control block to pinned host memory.  pdl: programmatic dependent launch after
// k_score (its launch overlaps k_score; it waits with griddepcontrol.wait)
cudaError_t spec(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, int reduce_only, cudaStream_t s, bool pdl,
                 bool big_chain = false);
// fast sharded step: export this rank's speculative set + totals (after k_score), and resolve the
// allgathered union on every rank (status FALLBACK: run the exact two-round protocol)
cudaError_t spec_export(const Scratch& S, Ctrl* ctrl, void* out, uint32_t rank, cudaStream_t s);
cudaError_t spec_merge(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, const void* all, uint32_t world,
                       uint32_t rank, cudaStream_t s);
uint32_t spec_export_bytes();
// k_spec_big: the resolve of a speculative set larger than k_spec's fast path (status ST_SPEC_BIG)
void spec_big(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s);
void hist0(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, int force, cudaStream_t s);
void pass(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, uint32_t pass_idx, cudaStream_t s);
void compact(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, cudaStream_t s);
void resolve(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s);
void cand(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, int only_after_fallback,
          cudaStream_t s);
void group(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s);

}  // namespace exact
}  // namespace jit
