// exact.cu -- the speculative resolve (k_spec, k_spec_big) and the exact radix path the host
// launches when the speculation cannot be exact (k_hist0, k_pass, k_compact, k_resolve, k_cand,
// k_group).  A separate translation unit from abi.cu (the hot scoring kernel), so each compiles
// with its own register allocation.
#define JIT_EXACT_TU 1
#include "common.cuh"
#include "select.cuh"
#include "spec.cuh"
#include "exact_api.h"

namespace jit {
namespace exact {

cudaError_t init_attributes() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((sizeof(u128) + 4) * kBucketCap))) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_group, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kGroupSmemBytes))) !=
        cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpecSmem)) !=
        cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_spec_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpecSmem)) !=
        cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_spec_big_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpecSmem)) !=
        cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_spec_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpecSmem)) !=
        cudaSuccess) return e;
    // one shared-memory carveout for every kernel of the step (see abi.cu)
    const void* ks[] = {(const void*)k_spec, (const void*)k_spec_big, (const void*)k_spec_big_chain,
                        (const void*)k_hist0, (const void*)k_pass, (const void*)k_compact, (const void*)k_resolve,
                        (const void*)k_cand, (const void*)k_group};
    for (const void* k : ks)
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared)) != cudaSuccess) return e;
    return cudaSuccess;
}

cudaError_t spec(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, int reduce_only, cudaStream_t s, bool pdl,
                 bool big_chain) {
    cudaLaunchConfig_t cfg = {};
    // k_spec only runs the small-set resolve (a larger set goes to k_spec_big): its smem is small
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(kSpecThreads); cfg.dynamicSmemBytes = kSpecFastSmem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_spec, P, c, ctrl, S, reduce_only, (int)big_chain);
    if (e != cudaSuccess || !big_chain) return e;
    // big mode: the big-set resolve, then the window over a large Cd (k_group runs only when the
    // resolve left it undone), then the host flag and the published control block
    k_spec_big_chain<<<1, kSpecThreads, kSpecSmem, s>>>(P, c, ctrl, S);
    k_group<<<1, 1024, kGroupSmemBytes, s>>>(P, c, ctrl, S);
    k_chain_publish<<<1, 64, 0, s>>>(ctrl, S.persist, S.h_ctrl);
    return cudaGetLastError();
}
cudaError_t spec_export(const Scratch& S, Ctrl* ctrl, void* out, uint32_t rank, cudaStream_t s) {
    k_spec_export<<<1, kSpecThreads, 0, s>>>(ctrl, S, reinterpret_cast<unsigned char*>(out), rank);
    return cudaGetLastError();
}
cudaError_t spec_merge(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, const void* all, uint32_t world,
                       uint32_t rank, cudaStream_t s) {
    k_spec_merge<<<1, kSpecThreads, kSpecSmem, s>>>(P, c, ctrl, S, reinterpret_cast<const unsigned char*>(all), world, rank);
    return cudaGetLastError();
}
uint32_t spec_export_bytes() { return kSpecExportBytes; }
void spec_big(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s) {
    k_spec_big<<<1, kSpecThreads, kSpecSmem, s>>>(P, c, ctrl, S);
}
void hist0(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, int force, cudaStream_t s) {
    k_hist0<<<grid, kPassThreads, 0, s>>>(P, c, ctrl, S, force);
}
void pass(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, uint32_t pass_idx, cudaStream_t s) {
    k_pass<<<grid, kPassThreads, 0, s>>>(P, c, ctrl, S, pass_idx);
}
void compact(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, cudaStream_t s) {
    k_compact<<<grid, kPassThreads, 0, s>>>(P, c, ctrl, S);
}
void resolve(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s) {
    k_resolve<<<1, 1024, (sizeof(u128) + 4) * kBucketCap, s>>>(P, c, ctrl, S);
}
void cand(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, uint32_t grid, int only_after_fallback,
          cudaStream_t s) {
    k_cand<<<grid, kPassThreads, 0, s>>>(P, c, ctrl, S, only_after_fallback);
}
void group(const Pool& P, const Cfg& c, Ctrl* ctrl, const Scratch& S, cudaStream_t s) {
    k_group<<<1, 1024, kGroupSmemBytes, s>>>(P, c, ctrl, S);
}

}  // namespace exact
}  // namespace jit
