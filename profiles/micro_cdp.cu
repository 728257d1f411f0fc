// micro_cdp.cu -- does a device-side tail launch (CDP2) from a kernel inside a CUDA graph
// (a) complete before the graph's next node runs, (b) cost anything when NOT taken?
// Build: nvcc -O3 -rdc=true -gencode arch=compute_100a,code=sm_100a micro_cdp.cu -lcudadevrt -o micro_cdp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_big(int* buf) {                 // stand-in for the scoring pass: 592 CTAs
    if (threadIdx.x == 0) atomicAdd(buf + 8, 1);
}
__global__ void k_child2(int* flag, int v) { if (threadIdx.x == 0) flag[1] = v; }
__global__ void k_child(int* flag, int v) {
    if (threadIdx.x == 0) flag[0] = v;
    if (threadIdx.x == 0 && blockIdx.x == 0) k_child2<<<1, 32, 0, cudaStreamTailLaunch>>>(flag, v);
}
__global__ void k_parent(int* flag, int take, int v) {
    if (threadIdx.x == 0 && take) {
        k_child<<<148, 256, 0, cudaStreamTailLaunch>>>(flag, v);
    }
}
__global__ void k_parent_graph(cudaGraphExec_t ge, int take) {
    if (threadIdx.x == 0 && take) cudaGraphLaunch(ge, cudaStreamGraphTailLaunch);
}
__global__ void k_check(int* flag, int v, int* bad) {
    if (threadIdx.x == 0 && (flag[0] != v || flag[1] != v)) atomicAdd(bad, 1);
}
__global__ void k_parent_plain(int* flag, int take, int v) {
    if (threadIdx.x == 0 && take) flag[0] = v, flag[1] = v;
}

int main() {
    int *flag, *bad, *buf;
    cudaMalloc(&flag, 64); cudaMalloc(&bad, 4); cudaMalloc(&buf, 64);
    cudaMemset(flag, 0, 64); cudaMemset(bad, 0, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    void* hbuf; cudaMallocHost(&hbuf, 1024);
    // device graph for modes 5/6: k_child (148 CTAs, nested tail k_child2) + k_child2
    cudaGraphExec_t dge;
    {
        cudaGraph_t dg;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_child2<<<148, 256, 0, s>>>(flag, 11);
        k_child2<<<1, 32, 0, s>>>(flag, 11);
        cudaStreamEndCapture(s, &dg);
        cudaError_t e = cudaGraphInstantiate(&dge, dg, cudaGraphInstantiateFlagDeviceLaunch);
        printf("device graph instantiate: %s\n", cudaGetErrorString(e));
        e = cudaGraphUpload(dge, s);
        printf("device graph upload: %s\n", cudaGetErrorString(e));
        cudaMemcpy(flag, flag, 0, cudaMemcpyDeviceToDevice);
    }
    for (int mode = 0; mode < 7; ++mode) {          // 0: plain parent, 1: CDP parent not taken, 2: taken,
                                                    // 3: plain parent + IF node (not taken), 4: + D2H memcpy node
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        k_big<<<592, 256, 0, s>>>(buf);
        if (mode == 0 || mode == 3 || mode == 4) k_parent_plain<<<1, 32, 0, s>>>(flag, 1, 7);
        else if (mode >= 5) { k_parent_plain<<<1, 32, 0, s>>>(flag, 1, 7); k_parent_graph<<<1, 32, 0, s>>>(dge, mode == 6); }
        else k_parent<<<1, 32, 0, s>>>(flag, mode == 2, 7 + mode);
        if (mode == 3) {
            cudaStreamCaptureStatus cs; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
            cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd);
            cudaGraphConditionalHandle hc;
            cudaGraphConditionalHandleCreate(&hc, cg, 0, cudaGraphCondAssignDefault);
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hc;
            cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
            cudaGraphNode_t cnode;
            cudaGraphAddNode(&cnode, cg, deps, nd, &cp);
            cudaStream_t s2; cudaStreamCreate(&s2);
            cudaStreamBeginCaptureToGraph(s2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
            k_big<<<592, 256, 0, s2>>>(buf);
            cudaStreamEndCapture(s2, nullptr);
            cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies);
        }
        if (mode == 4) cudaMemcpyAsync(hbuf, flag, 512, cudaMemcpyDeviceToHost, s);
        k_check<<<1, 32, 0, s>>>(flag, mode == 6 ? 11 : ((mode == 0 || mode >= 3) ? 7 : (mode == 2 ? 9 : 7)), bad);
        k_big<<<592, 256, 0, s>>>(buf);
        cudaError_t ec = cudaStreamEndCapture(s, &g);
        if (ec != cudaSuccess) { printf("capture mode %d: %s\n", mode, cudaGetErrorString(ec)); return 1; }
        ec = cudaGraphInstantiate(&ge, g, 0);
        if (ec != cudaSuccess) { printf("instantiate mode %d: %s\n", mode, cudaGetErrorString(ec)); return 1; }
        for (int i = 0; i < 50; ++i) cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaMemset(bad, 0, 4);
        cudaEventRecord(e0, s);
        const int K = 2000;
        for (int i = 0; i < K; ++i) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaError_t e = cudaStreamSynchronize(s);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("mode %d: %.2f us/graph, ordering violations %d, err %s\n", mode, 1e3 * ms / K, hb, cudaGetErrorString(e));
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
    return 0;
}
