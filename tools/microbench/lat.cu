// Latency microbenchmark (one warp): dependent chains of fp64 ops, shuffles,
// shared-memory round trips and barriers, timed with clock64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[1024];
    double x = a + threadIdx.x, y = b;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, a);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * y;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // double shuffle chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_down_sync(0xffffffffu, x, 1) + 1.0;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // smem store/load round trip chain
    int idx = threadIdx.x;
    sm[idx] = x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = (int(v) & 511) + threadIdx.x; sm[idx] = v + 1.0; }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // barrier chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    t1 = clock64();
    cyc[5] = t1 - t0;
    // FFMA chain for reference
    float xf = a, yf = b;
    t0 = clock64();
    for (int i = 0; i < n; ++i) xf = fmaf(xf, yf, 1.0f);
    t1 = clock64();
    cyc[6] = t1 - t0;
    // DFMA throughput: 8 independent chains
    double z[8];
    for (int j = 0; j < 8; ++j) z[j] = a + j;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) z[j] = fma(z[j], y, a);
    t1 = clock64();
    cyc[7] = t1 - t0;
    double s = 0;
    for (int j = 0; j < 8; ++j) s += z[j];
    out[threadIdx.x] = x + y + xf + s + idx;
}

// fp64 throughput: all SMs, many warps, independent chains
__global__ void kthr(double* out, double a, double b, int n) {
    double z[8];
    for (int j = 0; j < 8; ++j) z[j] = a + j + threadIdx.x;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) z[j] = fma(z[j], b, a);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += z[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 64 * sizeof(long long));
    const int n = 1000;
    for (int threads : {32, 256}) {
        k<<<1, threads>>>(out, cyc, 1.0000001, 0.9999999, n);
        long long h[8];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        const char* names[8] = {"DFMA chain", "DADD chain", "DMUL chain", "SHFL(f64)+DADD chain", "STS/LDS chain",
                                "BAR.SYNC", "FFMA chain", "8 indep DFMA chains"};
        printf("threads=%d (cycles per op)\n", threads);
        for (int i = 0; i < 8; ++i) printf("  %-22s %.1f\n", names[i], double(h[i]) / n / (i == 7 ? 8 : 1));
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int nthr = 20000;
    for (int bs : {256, 512, 1024}) {
        kthr<<<sms * 4, bs>>>(out, 1.0000001, 0.9999999, 10);
        cudaEventRecord(e0);
        kthr<<<sms * (2048 / bs), bs>>>(out, 1.0000001, 0.9999999, nthr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * nthr * double(sms) * 2048;
        printf("DFMA throughput (block %d): %.2f TFLOP/s\n", bs, flops / ms / 1e9);
    }
    return 0;
}
