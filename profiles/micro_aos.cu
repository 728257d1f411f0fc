// micro_aos.cu -- read-only streaming floor of the pool pass on B200 for the round-2 layout:
// 32-B AoS hot rows (one stream) vs the round-1 7-field SoA, no per-row writes (a per-block
// reduction keeps the loads alive).  N = 2^20 rows, 16 rotated pool copies (537 MB > 4x L2).
//   aos1   : one row per thread, grid = N / 256 (two LDG.128 per row)
//   aosW   : R rows per lane, lane-strided inside a warp's 32R-row item (coalesced per k),
//            loads of all R rows issued before any math; grid = N / (256 R)
//   soa1   : one row per thread over the 7 SoA fields
// +math=M adds M rounds of a dependent integer / fp64 chain per row (issue pressure).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro_aos micro_aos.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(16) Row { int64_t arr; uint32_t li, ge, pr, lr, me, si; };
struct Soa { int64_t* arr; uint32_t *li, *ge, *pr, *lh, *me, *ax; };

template <int M>
__device__ __forceinline__ uint64_t fake_math(uint64_t a, uint32_t b, uint32_t c) {
    uint64_t x = a;
    double d = (double)b + 1.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        x = x * 0x9E3779B97F4A7C15ull + (b ^ (uint32_t)i);
        const uint32_t q = __umulhi((uint32_t)x, 0x51EB851Fu) >> 4;
        x ^= (uint64_t)q << 17;
        d = __fma_rn(d, 1.0000001, (double)(c & 0xFF));
    }
    return x ^ (uint64_t)__double_as_longlong(d);
}

__device__ __forceinline__ void sink(uint64_t v, unsigned long long* out) {
    __shared__ unsigned long long s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicXor(&s, (unsigned long long)v);
    __syncthreads();
    if (threadIdx.x == 0 && s == 0x123456789ull) out[blockIdx.x & 1023] = s;   // never true in practice
}

__device__ __forceinline__ Row ldrow(const Row* p) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
    Row r;
    r.arr = (int64_t)(((uint64_t)a.y << 32) | a.x); r.li = a.z; r.ge = a.w; r.pr = b.x; r.lr = b.y; r.me = b.z; r.si = b.w;
    return r;
}

__device__ __forceinline__ Row ldrow8(const Row* p) {
    uint32_t a0, a1, a2, a3, a4, a5, a6, a7;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6), "=r"(a7) : "l"(p));
    Row r;
    r.arr = (int64_t)(((uint64_t)a1 << 32) | a0); r.li = a2; r.ge = a3; r.pr = a4; r.lr = a5; r.me = a6; r.si = a7;
    return r;
}

// one 256-bit load per row (sm_100: LDG.E.256), R rows per lane, lane-strided in a warp's 32R-row item
template <int R, int M, int T>
__global__ void __launch_bounds__(T) k_v8(const Row* rows, uint32_t n, unsigned long long* out) {
    const uint32_t w = (blockIdx.x * T + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t base = w * 32 * R + lane;
    Row q[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const uint32_t r = base + 32 * k;
        if (r < n) q[k] = ldrow8(rows + r); else q[k] = Row{};
    }
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        uint64_t x = (uint64_t)q[k].arr ^ q[k].li ^ q[k].ge ^ q[k].pr ^ q[k].lr ^ q[k].me ^ q[k].si;
        if (M) x = fake_math<M>(x, q[k].li, q[k].ge);
        v ^= x;
    }
    sink(v, out);
}

// persistent: grid-stride over 32R-row warp items with the next item's rows loaded before the
// current item's math (register double buffer)
template <int R, int M, int T>
__global__ void __launch_bounds__(T) k_v8p(const Row* rows, uint32_t n, unsigned long long* out) {
    const uint32_t W = gridDim.x * (T / 32), lane = threadIdx.x & 31;
    uint32_t w = (blockIdx.x * T + threadIdx.x) >> 5;
    const uint32_t nit = (n + 32 * R - 1) / (32 * R);
    Row q[R], nx[R];
    auto load = [&](Row* d, uint32_t it) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const uint32_t r = it * 32 * R + lane + 32 * k;
            if (it < nit && r < n) d[k] = ldrow8(rows + r); else d[k] = Row{};
        }
    };
    load(q, w);
    uint64_t v = 0;
    for (; w < nit; w += W) {
        load(nx, w + W);
#pragma unroll
        for (int k = 0; k < R; ++k) {
            uint64_t x = (uint64_t)q[k].arr ^ q[k].li ^ q[k].ge ^ q[k].pr ^ q[k].lr ^ q[k].me ^ q[k].si;
            if (M) x = fake_math<M>(x, q[k].li, q[k].ge);
            v ^= x;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) q[k] = nx[k];
    }
    sink(v, out);
}

template <int M>
__global__ void __launch_bounds__(256) k_aos1(const Row* rows, uint32_t n, unsigned long long* out) {
    const uint32_t r = blockIdx.x * 256 + threadIdx.x;
    uint64_t v = 0;
    if (r < n) {
        const Row q = ldrow(rows + r);
        v = (uint64_t)q.arr ^ q.li ^ q.ge ^ q.pr ^ q.lr ^ q.me ^ q.si;
        if (M) v = fake_math<M>(v, q.li, q.ge);
    }
    sink(v, out);
}

template <int R, int M>
__global__ void __launch_bounds__(256) k_aosW(const Row* rows, uint32_t n, unsigned long long* out) {
    const uint32_t w = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t base = w * 32 * R + lane;
    Row q[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const uint32_t r = base + 32 * k;
        if (r < n) q[k] = ldrow(rows + r); else q[k] = Row{};
    }
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        uint64_t x = (uint64_t)q[k].arr ^ q[k].li ^ q[k].ge ^ q[k].pr ^ q[k].lr ^ q[k].me ^ q[k].si;
        if (M) x = fake_math<M>(x, q[k].li, q[k].ge);
        v ^= x;
    }
    sink(v, out);
}

template <int M>
__global__ void __launch_bounds__(256) k_soa1(Soa P, uint32_t n, unsigned long long* out) {
    const uint32_t r = blockIdx.x * 256 + threadIdx.x;
    uint64_t v = 0;
    if (r < n) {
        v = (uint64_t)__ldcs(P.arr + r) ^ __ldcs(P.li + r) ^ __ldcs(P.ge + r) ^ __ldcs(P.pr + r) ^ __ldcs(P.lh + r) ^
            __ldcs(P.me + r) ^ __ldcs(P.ax + r);
        if (M) v = fake_math<M>(v, (uint32_t)v, (uint32_t)(v >> 32));
    }
    sink(v, out);
}

constexpr int kCopies = 16;
constexpr uint32_t N = 1u << 20;

template <typename F>
static void timeit(const char* name, F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 2 * kCopies; ++i) launch(i % kCopies);
    cudaDeviceSynchronize();
    const int L = 8 * kCopies;
    cudaEventRecord(a);
    for (int i = 0; i < L; ++i) launch(i % kCopies);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1000.0 * ms / L;
    printf("%-28s %8.2f us  %7.0f GB/s (32 B/row)\n", name, us, 32.0 * N / (us * 1e3));
}

int main() {
    Row* rows[kCopies];
    Soa soa[kCopies];
    for (int c = 0; c < kCopies; ++c) {
        cudaMalloc(&rows[c], sizeof(Row) * N);
        cudaMemset(rows[c], c, sizeof(Row) * N);
        cudaMalloc(&soa[c].arr, 8ull * N);
        cudaMalloc(&soa[c].li, 4ull * N); cudaMalloc(&soa[c].ge, 4ull * N); cudaMalloc(&soa[c].pr, 4ull * N);
        cudaMalloc(&soa[c].lh, 4ull * N); cudaMalloc(&soa[c].me, 4ull * N); cudaMalloc(&soa[c].ax, 4ull * N);
    }
    unsigned long long* out;
    cudaMalloc(&out, 8 * 1024);
    timeit("aos1", [&](int c) { k_aos1<0><<<N / 256, 256>>>(rows[c], N, out); });
    timeit("aos1 math=8", [&](int c) { k_aos1<8><<<N / 256, 256>>>(rows[c], N, out); });
    timeit("aos1 math=16", [&](int c) { k_aos1<16><<<N / 256, 256>>>(rows[c], N, out); });
    timeit("aosW R=2", [&](int c) { k_aosW<2, 0><<<N / 512, 256>>>(rows[c], N, out); });
    timeit("aosW R=4", [&](int c) { k_aosW<4, 0><<<N / 1024, 256>>>(rows[c], N, out); });
    timeit("aosW R=4 math=8", [&](int c) { k_aosW<4, 8><<<N / 1024, 256>>>(rows[c], N, out); });
    timeit("aosW R=4 math=16", [&](int c) { k_aosW<4, 16><<<N / 1024, 256>>>(rows[c], N, out); });
    timeit("aosW R=8", [&](int c) { k_aosW<8, 0><<<N / 2048, 256>>>(rows[c], N, out); });
    timeit("v8 R=1 T=256", [&](int c) { k_v8<1, 0, 256><<<N / 256, 256>>>(rows[c], N, out); });
    timeit("v8 R=2 T=256", [&](int c) { k_v8<2, 0, 256><<<N / 512, 256>>>(rows[c], N, out); });
    timeit("v8 R=4 T=256", [&](int c) { k_v8<4, 0, 256><<<N / 1024, 256>>>(rows[c], N, out); });
    timeit("v8 R=4 T=128", [&](int c) { k_v8<4, 0, 128><<<N / 512, 128>>>(rows[c], N, out); });
    timeit("v8 R=2 T=256 math=8", [&](int c) { k_v8<2, 8, 256><<<N / 512, 256>>>(rows[c], N, out); });
    timeit("v8 R=2 T=256 math=16", [&](int c) { k_v8<2, 16, 256><<<N / 512, 256>>>(rows[c], N, out); });
    timeit("v8 R=4 T=256 math=8", [&](int c) { k_v8<4, 8, 256><<<N / 1024, 256>>>(rows[c], N, out); });
    timeit("v8 R=4 T=256 math=16", [&](int c) { k_v8<4, 16, 256><<<N / 1024, 256>>>(rows[c], N, out); });
    for (int cps : {4, 6, 8}) {
        char nm[64];
        snprintf(nm, 64, "v8p R=2 T=256 cps=%d", cps);
        timeit(nm, [&](int c) { k_v8p<2, 0, 256><<<148 * cps, 256>>>(rows[c], N, out); });
        snprintf(nm, 64, "v8p R=2 T=256 cps=%d math=8", cps);
        timeit(nm, [&](int c) { k_v8p<2, 8, 256><<<148 * cps, 256>>>(rows[c], N, out); });
        snprintf(nm, 64, "v8p R=2 T=256 cps=%d math=16", cps);
        timeit(nm, [&](int c) { k_v8p<2, 16, 256><<<148 * cps, 256>>>(rows[c], N, out); });
    }
    timeit("soa1", [&](int c) { k_soa1<0><<<N / 256, 256>>>(soa[c], N, out); });
    timeit("soa1 math=8", [&](int c) { k_soa1<8><<<N / 256, 256>>>(soa[c], N, out); });
    // a plain device-to-device copy of the same 32 MiB (read + write) for reference
    timeit("memcpy D2D 32MiB (r+w/2)", [&](int c) { cudaMemcpyAsync(rows[(c + 1) % kCopies], rows[c], sizeof(Row) * N / 2, cudaMemcpyDeviceToDevice); });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
