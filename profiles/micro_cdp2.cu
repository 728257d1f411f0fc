// micro_cdp2.cu -- ordering of CDP tail launches made by a kernel node of a CUDA graph.
// Every graph launch bumps an iteration counter; the child (and, nested, the grandchild) write
// the current iteration; a later node of the same graph and the host (after a stream sync,
// through pinned memory) check they see it.  Counts violations per mode.
// Build: nvcc -O3 -rdc=true -gencode arch=compute_100a,code=sm_100a micro_cdp2.cu -lcudadevrt -o micro_cdp2
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_inc(int* it) { if (threadIdx.x == 0 && blockIdx.x == 0) it[0] += 1; }
__global__ void k_grand(const int* it, int* flag, int* hflag) {
    if (threadIdx.x == 0 && blockIdx.x == 0) { flag[1] = it[0]; *(volatile int*)hflag = it[0]; __threadfence_system(); }
}
__global__ void k_child(const int* it, int* flag, int* hflag, int nested) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        flag[0] = it[0];
        if (nested) k_grand<<<1, 32, 0, cudaStreamTailLaunch>>>(it, flag, hflag);
        else { *(volatile int*)hflag = it[0]; __threadfence_system(); }
    }
}
__global__ void k_parent(const int* it, int* flag, int* hflag, int nested) {
    if (threadIdx.x == 0) k_child<<<148, 256, 0, cudaStreamTailLaunch>>>(it, flag, hflag, nested);
}
// closer to the library's chain: 512-thread parent with 160 KB of dynamic smem, an 888-CTA
// child launching a 592x512 grandchild (16 KB static smem) whose LAST CTA launches the end
__global__ void k_end(const int* it, int* flag, int* hflag) {
    if (threadIdx.x == 0) { flag[1] = it[0]; *(volatile int*)hflag = it[0]; __threadfence_system(); }
}
__global__ void __launch_bounds__(512) k_g2(const int* it, int* flag, int* hflag, unsigned* done) {
    __shared__ unsigned sm[4096];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) { __threadfence(); last = atomicAdd(done, 1u) == gridDim.x - 1; }
    __syncthreads();
    if (last && threadIdx.x == 0) { *done = 0; k_end<<<1, 1024, 0, cudaStreamTailLaunch>>>(it, flag, hflag); }
    if (sm[threadIdx.x] == 12345) flag[3] = 1;
}
__global__ void k_c2(const int* it, int* flag, int* hflag, unsigned* done) {
    if (threadIdx.x == 0 && blockIdx.x == 0) { flag[0] = it[0]; k_g2<<<592, 512, 0, cudaStreamTailLaunch>>>(it, flag, hflag, done); }
}
__global__ void __launch_bounds__(512) k_p2(const int* it, int* flag, int* hflag, unsigned* done) {
    extern __shared__ unsigned dsm[];
    dsm[threadIdx.x] = 1;
    __syncthreads();
    if (threadIdx.x == 0) k_c2<<<888, 256, 0, cudaStreamTailLaunch>>>(it, flag, hflag, done);
}
__global__ void k_check(const int* it, const int* flag, int nested, int* bad) {
    if (threadIdx.x == 0 && (flag[0] != it[0] || (nested && flag[1] != it[0]))) atomicAdd(bad, 1);
}

int main() {
    int *it, *flag, *bad, *hflag;
    cudaMalloc(&it, 4); cudaMalloc(&flag, 64); cudaMalloc(&bad, 4);
    cudaMallocHost(&hflag, 64);
    cudaStream_t s; cudaStreamCreate(&s);
    unsigned* done; cudaMalloc(&done, 4); cudaMemset(done, 0, 4);
    cudaFuncSetAttribute(k_p2, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (int mode = 0; mode < 6; ++mode) {
        // 0: first level + check node; 1: nested + check node; 2: first level, host check only;
        // 3: nested, host check only
        // 4: library-like chain + check node; 5: library-like chain, host check only
        const int nested = mode >= 4 ? 1 : (mode & 1), node_check = mode < 2 || mode == 4;
        cudaMemset(it, 0, 4); cudaMemset(flag, 0, 64); cudaMemset(bad, 0, 4); *hflag = 0;
        cudaDeviceSynchronize();
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_inc<<<1, 32, 0, s>>>(it);
        if (mode >= 4) k_p2<<<1, 512, 160 * 1024, s>>>(it, flag, hflag, done);
        else k_parent<<<1, 32, 0, s>>>(it, flag, hflag, nested);
        if (node_check) k_check<<<1, 32, 0, s>>>(it, flag, nested, bad);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        int host_bad = 0;
        const int K = 500;
        for (int i = 1; i <= K; ++i) {
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            if (*(volatile int*)hflag != i) ++host_bad;
        }
        int hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("mode %d (nested %d, check node %d): node violations %d, host violations %d / %d, err %s\n",
               mode, nested, node_check, hb, host_bad, K, cudaGetErrorString(cudaGetLastError()));
        // the same without a graph (plain stream launches)
        cudaMemset(it, 0, 4); cudaDeviceSynchronize(); *hflag = 0; host_bad = 0;
        for (int i = 1; i <= K; ++i) {
            k_inc<<<1, 32, 0, s>>>(it);
            if (mode >= 4) k_p2<<<1, 512, 160 * 1024, s>>>(it, flag, hflag, done);
            else k_parent<<<1, 32, 0, s>>>(it, flag, hflag, nested);
            cudaStreamSynchronize(s);
            if (*(volatile int*)hflag != i) ++host_bad;
        }
        printf("        stream launches: host violations %d / %d\n", host_bad, K);
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return 0;
}
