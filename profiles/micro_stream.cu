// micro_stream.cu -- how fast can one SM-resident pipeline stream the pool's 7 hot SoA fields
// (32 B/row) into a CTA on B200?  Three readers over N = 2^20 rows (x4 rotated copies, > L2):
//   tma   : persistent CTAs, ring of S stages of T rows, one thread issues 7 cp.async.bulk per
//           stage (mbarrier completion), consumers read the stage from shared memory
//   ldg   : persistent CTAs, each thread loads R consecutive rows of every field with vector
//           loads (plain LDG), grid-stride over tiles
//   ldg1  : one row per thread, grid = rows / threads (non-persistent)
// Every reader writes 16 B/row back (key image 8, cost 4, aux 4) as the pool pass does.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro_stream micro_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Pool {
    int64_t* arr;
    uint32_t *li, *ge, *pr, *lh, *me, *ax;
    uint64_t* img;
    uint32_t *cost, *aux2;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t b, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(d)), "l"(s), "r"(b), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t* bar, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                 ::"r"(sa(bar)), "r"(par) : "memory");
}

// synthetic per-row math of roughly the pool pass's size: M rounds of mixed 64-bit integer and
// fp64 work (a dependent chain per row, 2 rows per thread are independent)
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
        if ((x & 7) == 3) x += c;
    }
    return x ^ (uint64_t)__double_as_longlong(d);
}

template <int T, int S, int M = 0>
__global__ void __launch_bounds__(256) k_tma(Pool P, uint32_t n_items) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr uint32_t kB = T * 32;                     // bytes per stage
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const uint32_t tid = threadIdx.x, G = gridDim.x;
    uint32_t fpar = 0, fused = 0;
    auto produce = [&](uint32_t it, uint32_t s) {
        if (it >= n_items) return;
        if (fused & (1u << s)) wait_par(&empty[s], ((fpar >> s) & 1u) ^ 1u);
        unsigned char* b = smem + s * kB;
        const uint32_t r0 = it * T;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(kB) : "memory");
        bulk(b, P.arr + r0, 8 * T, &full[s]);
        bulk(b + 8 * T, P.li + r0, 4 * T, &full[s]);
        bulk(b + 12 * T, P.ge + r0, 4 * T, &full[s]);
        bulk(b + 16 * T, P.pr + r0, 4 * T, &full[s]);
        bulk(b + 20 * T, P.lh + r0, 4 * T, &full[s]);
        bulk(b + 24 * T, P.me + r0, 4 * T, &full[s]);
        bulk(b + 28 * T, P.ax + r0, 4 * T, &full[s]);
        fpar ^= 1u << s; fused |= 1u << s;
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(256));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j + 1 < S; ++j) produce(blockIdx.x + j * G, j);
    }
    __syncthreads();
    uint32_t cpar = 0, s = 0;
    for (uint32_t it = blockIdx.x; it < n_items; it += G, s = (s + 1 == S) ? 0 : s + 1) {
        if (tid == 0) produce(it + (S - 1) * G, s == 0 ? S - 1 : s - 1);
        wait_par(&full[s], (cpar >> s) & 1u); cpar ^= 1u << s;
        const unsigned char* b = smem + s * kB;
        constexpr int R = T / 256;
        uint64_t im[R]; uint32_t co[R], ax[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const uint32_t o = tid + 256 * k;
            const int64_t a = reinterpret_cast<const int64_t*>(b)[o];
            const uint32_t* u = reinterpret_cast<const uint32_t*>(b + 8 * T);
            im[k] = (uint64_t)a ^ u[o] ^ u[T + o]; co[k] = u[2 * T + o] ^ u[3 * T + o]; ax[k] = u[4 * T + o] ^ u[5 * T + o];
            if constexpr (M > 0) im[k] = fake_math<M>(im[k], co[k], ax[k]);
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const uint32_t r = it * T + tid + 256 * k;
            P.img[r] = im[k]; P.cost[r] = co[k]; P.aux2[r] = ax[k];
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_ldg(Pool P, uint32_t n) {
    const uint32_t stride = gridDim.x * 256 * R;
    for (uint32_t r0 = (blockIdx.x * 256 + threadIdx.x) * R; r0 < n; r0 += stride) {
        int64_t a[R]; uint32_t l[R], g[R], p[R], h[R], m[R], x[R];
        if constexpr (R == 4) {
            const longlong2 a0 = *reinterpret_cast<const longlong2*>(P.arr + r0), a1 = *reinterpret_cast<const longlong2*>(P.arr + r0 + 2);
            a[0] = a0.x; a[1] = a0.y; a[2] = a1.x; a[3] = a1.y;
#define L4(f, v) { const uint4 t = *reinterpret_cast<const uint4*>(P.f + r0); v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w; }
            L4(li, l) L4(ge, g) L4(pr, p) L4(lh, h) L4(me, m) L4(ax, x)
        } else {
            a[0] = P.arr[r0]; l[0] = P.li[r0]; g[0] = P.ge[r0]; p[0] = P.pr[r0]; h[0] = P.lh[r0]; m[0] = P.me[r0]; x[0] = P.ax[r0];
        }
        uint64_t im[R]; uint32_t co[R], ax[R];
#pragma unroll
        for (int k = 0; k < R; ++k) { im[k] = (uint64_t)a[k] ^ l[k] ^ g[k]; co[k] = p[k] ^ h[k]; ax[k] = m[k] ^ x[k]; }
        if constexpr (R == 4) {
            reinterpret_cast<ulonglong2*>(P.img + r0)[0] = make_ulonglong2(im[0], im[1]);
            reinterpret_cast<ulonglong2*>(P.img + r0)[1] = make_ulonglong2(im[2], im[3]);
            *reinterpret_cast<uint4*>(P.cost + r0) = make_uint4(co[0], co[1], co[2], co[3]);
            *reinterpret_cast<uint4*>(P.aux2 + r0) = make_uint4(ax[0], ax[1], ax[2], ax[3]);
        } else {
            P.img[r0] = im[0]; P.cost[r0] = co[0]; P.aux2[r0] = ax[0];
        }
    }
}

int main() {
    const uint32_t N = 1u << 20;
    const int ROT = 4;
    Pool pools[ROT];
    for (int i = 0; i < ROT; ++i) {
        Pool& P = pools[i];
        cudaMalloc(&P.arr, 8ull * N);
        cudaMalloc(&P.li, 4ull * N); cudaMalloc(&P.ge, 4ull * N); cudaMalloc(&P.pr, 4ull * N);
        cudaMalloc(&P.lh, 4ull * N); cudaMalloc(&P.me, 4ull * N); cudaMalloc(&P.ax, 4ull * N);
        cudaMalloc(&P.img, 8ull * N); cudaMalloc(&P.cost, 4ull * N); cudaMalloc(&P.aux2, 4ull * N);
        cudaMemset(P.arr, 1, 8ull * N);
        for (uint32_t* q : {P.li, P.ge, P.pr, P.lh, P.me, P.ax}) cudaMemset(q, 2, 4ull * N);
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytes = 48.0 * N;
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch(pools[w % ROT]);
        cudaDeviceSynchronize();
        const int K = 40;
        cudaEventRecord(e0);
        for (int k = 0; k < K; ++k) launch(pools[k % ROT]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / K;
        printf("%-34s %7.2f us  %7.0f GB/s  (%s)\n", name, us, bytes / (us * 1e3), cudaGetErrorString(cudaGetLastError()));
    };
#define TMA(T, S, CPS)                                                                                     \
    {                                                                                                      \
        const uint32_t smem = (T) * 32 * (S);                                                              \
        cudaFuncSetAttribute(k_tma<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);          \
        char nm[64];                                                                                       \
        snprintf(nm, sizeof nm, "tma T=%d S=%d ctas/sm=%d", T, S, CPS);                                    \
        run(nm, [&](Pool P) { k_tma<T, S><<<nsm * (CPS), 256, smem>>>(P, N / (T)); });                     \
    }
    TMA(512, 4, 2) TMA(512, 4, 3) TMA(1024, 3, 2) TMA(1024, 4, 1) TMA(2048, 3, 1) TMA(2048, 2, 2) TMA(256, 8, 4)
    TMA(512, 8, 2) TMA(1024, 6, 1)
#define TMAM(T, S, CPS, M)                                                                                  \
    {                                                                                                      \
        const uint32_t smem = (T) * 32 * (S);                                                              \
        cudaFuncSetAttribute(k_tma<T, S, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
        char nm[64];                                                                                       \
        snprintf(nm, sizeof nm, "tma T=%d S=%d ctas/sm=%d math=%d", T, S, CPS, M);                         \
        run(nm, [&](Pool P) { k_tma<T, S, M><<<nsm * (CPS), 256, smem>>>(P, N / (T)); });                  \
    }
    TMAM(512, 4, 3, 4) TMAM(512, 4, 3, 8) TMAM(512, 4, 3, 16) TMAM(512, 4, 3, 24) TMAM(512, 2, 3, 16)
    for (int cps : {2, 4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "ldg R=4 persistent ctas/sm=%d", cps);
        run(nm, [&](Pool P) { k_ldg<4><<<nsm * cps, 256>>>(P, N); });
    }
    run("ldg R=4 grid=N/1024", [&](Pool P) { k_ldg<4><<<N / 1024, 256>>>(P, N); });
    run("ldg R=1 grid=N/256", [&](Pool P) { k_ldg<1><<<N / 256, 256>>>(P, N); });
    run("ldg R=1 persistent 8/sm", [&](Pool P) { k_ldg<1><<<nsm * 8, 256>>>(P, N); });
    return 0;
}
