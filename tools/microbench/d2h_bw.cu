// Pinned device-to-host copy bandwidth of one 268 MB slab (the cfg4 final
// slab) split into 1, 2, 4 or 8 concurrent copies on separate streams.
// nvcc -gencode arch=compute_100a,code=sm_100a -o d2h_bw d2h_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t bytes = size_t(64) * 256 * 1024 * 16;
    void *d, *h;
    cudaMalloc(&d, bytes);
    cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    cudaMemset(d, 1, bytes);
    cudaStream_t st[8];
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int n : {1, 2, 4, 8, 1, 2, 4, 8}) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, st[0]);
        for (int k = 1; k < n; ++k) cudaStreamWaitEvent(st[k], a, 0);
        const size_t chunk = bytes / n;
        for (int k = 0; k < n; ++k)
            cudaMemcpyAsync(static_cast<char*>(h) + k * chunk, static_cast<char*>(d) + k * chunk, chunk,
                            cudaMemcpyDeviceToHost, st[k]);
        for (int k = 1; k < n; ++k) {
            cudaEvent_t e;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            cudaEventRecord(e, st[k]);
            cudaStreamWaitEvent(st[0], e, 0);
        }
        cudaEventRecord(b, st[0]);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%d copies: %.3f ms, %.1f GB/s\n", n, ms, bytes / (ms * 1e6));
    }
    // host-to-device for comparison
    cudaDeviceSynchronize();
    cudaEventRecord(a, st[0]);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st[0]);
    cudaEventRecord(b, st[0]);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("H2D 1 copy: %.3f ms, %.1f GB/s\n", ms, bytes / (ms * 1e6));
    return 0;
}
