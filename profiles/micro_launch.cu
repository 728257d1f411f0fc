// micro_launch.cu -- why do the single-CTA kernels of the step take ~15-20 µs?
// Times chains "stream kernel (grid of 888x256, 12 KB smem) -> single CTA kernel" with the
// single CTA using {0, 96, 160} KB of dynamic smem and {256, 1024} threads, with and without
// a common carveout, as CUDA graphs and as plain launches.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro_launch profiles/micro_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_stream(float* a, int n) {
    __shared__ float s[3072];
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    s[threadIdx.x] = i;
    __syncthreads();
    for (; i < n; i += gridDim.x * blockDim.x) a[i] = a[i] * 1.0001f + s[threadIdx.x];
}

__global__ void k_single(float* a) {
    extern __shared__ float d[];
    d[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) a[0] += d[blockDim.x - 1];
}

int main() {
    const int n = 1 << 20;
    float* a;
    cudaMalloc(&a, n * sizeof(float));
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(k_single, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int smems[] = {4 * 1024, 48 * 1024, 96 * 1024, 160 * 1024};
    const int threads[] = {256, 1024};
    for (int carve = 0; carve < 2; ++carve) {
        int pref = carve ? cudaSharedmemCarveoutMaxShared : cudaSharedmemCarveoutDefault;
        cudaFuncSetAttribute(k_stream, cudaFuncAttributePreferredSharedMemoryCarveout, pref);
        cudaFuncSetAttribute(k_single, cudaFuncAttributePreferredSharedMemoryCarveout, pref);
        for (int th : threads)
            for (int sm : smems) {
                for (int graph = 0; graph < 2; ++graph) {
                    cudaGraphExec_t ex = nullptr;
                    if (graph) {
                        cudaGraph_t g;
                        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                        k_stream<<<888, 256, 0, s>>>(a, n);
                        k_single<<<1, th, sm, s>>>(a);
                        cudaStreamEndCapture(s, &g);
                        cudaGraphInstantiate(&ex, g, 0);
                    }
                    float best_chain = 1e9, best_stream = 1e9;
                    for (int rep = 0; rep < 5; ++rep) {
                        cudaEventRecord(e0, s);
                        for (int k = 0; k < 50; ++k) {
                            if (graph) cudaGraphLaunch(ex, s);
                            else { k_stream<<<888, 256, 0, s>>>(a, n); k_single<<<1, th, sm, s>>>(a); }
                        }
                        cudaEventRecord(e1, s);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        best_chain = ms < best_chain ? ms : best_chain;
                        cudaEventRecord(e0, s);
                        for (int k = 0; k < 50; ++k) k_stream<<<888, 256, 0, s>>>(a, n);
                        cudaEventRecord(e1, s);
                        cudaEventSynchronize(e1);
                        cudaEventElapsedTime(&ms, e0, e1);
                        best_stream = ms < best_stream ? ms : best_stream;
                    }
                    printf("carveout=%s threads=%4d smem=%3dKB %s: chain %.2f us, stream-only %.2f us, single-CTA cost %.2f us\n",
                           carve ? "maxshared" : "default  ", th, sm / 1024, graph ? "graph " : "launch",
                           best_chain * 1000 / 50, best_stream * 1000 / 50, (best_chain - best_stream) * 1000 / 50);
                    if (ex) cudaGraphExecDestroy(ex);
                }
            }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
