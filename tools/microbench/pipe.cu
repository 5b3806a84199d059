// Memory-pipeline microbenchmark shaped like the azimuth sweep: persistent
// CTAs stream 32-KB items (global -> smem via cp.async, STAGES deep) and
// write them back; an optional busy loop of `work` dependent DFMAs per item
// stands in for the solve.  Reports effective GB/s (read + write).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int STAGES>
__global__ void kpipe(const double2* __restrict__ src, double2* __restrict__ dst, long items, int per, int item_elems,
                      int work, double a) {
    extern __shared__ double2 sm[];
    const long i0 = (long)blockIdx.x * per;
    long i1 = i0 + per; if (i1 > items) i1 = items;
    if (i0 >= i1) return;
    const int per_thread = item_elems / blockDim.x;
    auto fetch = [&](long it, int st) {
        for (int k = 0; k < per_thread; ++k) {
            int e = k * blockDim.x + threadIdx.x;
            cp16(sm + st * item_elems + e, src + it * item_elems + e);
        }
    };
    for (int p = 0; p < STAGES - 1; ++p) { if (i0 + p < i1) fetch(i0 + p, p); commit(); }
    int slot = 0;
    double acc = a;
    for (long it = i0; it < i1; ++it) {
        if (it + STAGES - 1 < i1) fetch(it + STAGES - 1, (slot + STAGES - 1) % STAGES);
        commit();
        waitg<STAGES - 1>();
        for (int w = 0; w < work; ++w) acc = fma(acc, 0.999999, 1e-9);
        for (int k = 0; k < per_thread; ++k) {
            int e = k * blockDim.x + threadIdx.x;
            double2 v = sm[slot * item_elems + e];
            v.x += acc * 1e-300;
            __stcs(dst + it * item_elems + e, v);
        }
        slot = (slot + 1) % STAGES;
    }
}

__global__ void kcopy(const double2* __restrict__ src, double2* __restrict__ dst, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const long n = 16L * 1024 * 1024;           // 256 MiB of complex128
    double2 *a, *b;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); kcopy<<<sms * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("grid-stride copy: %.0f GB/s\n", 2.0 * n * 16 / ms / 1e6);
    const int item_elems = 2048;                  // 32 KB
    const long items = n / item_elems;
    for (int threads : {128, 256}) {
        for (int stages : {2, 3, 4}) {
            for (int ctas_per_sm : {2, 3, 4, 6}) {
                size_t smem = (size_t)stages * item_elems * 16;
                if (smem * ctas_per_sm > 220 * 1024) continue;
                for (int work : {0, 200, 800}) {
                    long ctas = (long)sms * ctas_per_sm;
                    int per = (int)((items + ctas - 1) / ctas);
                    int grid = (int)((items + per - 1) / per);
                    auto run = [&]() {
                        if (stages == 2) { cudaFuncSetAttribute(kpipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); kpipe<2><<<grid, threads, smem>>>(a, b, items, per, item_elems, work, 1.0); }
                        if (stages == 3) { cudaFuncSetAttribute(kpipe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); kpipe<3><<<grid, threads, smem>>>(a, b, items, per, item_elems, work, 1.0); }
                        if (stages == 4) { cudaFuncSetAttribute(kpipe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); kpipe<4><<<grid, threads, smem>>>(a, b, items, per, item_elems, work, 1.0); }
                    };
                    run();
                    cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms, e0, e1);
                    printf("thr %3d stages %d ctas/sm %d work %4d: %6.0f GB/s  (%.1f us)\n", threads, stages, ctas_per_sm, work,
                           2.0 * n * 16 / ms / 1e6, ms * 1e3);
                }
            }
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
