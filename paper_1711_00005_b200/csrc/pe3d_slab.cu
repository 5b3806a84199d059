// pe3d_slab.cu -- cross-rank ordering for the slab march's fused transposes
// (SURVEY.md §8(e)).
//
// With peer-direct transposes the depth sweep of rank p stores its tiles
// straight into the azimuth-sweep inputs of the other ranks and vice versa
// (NVLink peer memory, CUDA IPC mappings across processes, plain device
// memory for virtual ranks).  The only remaining exchange is ordering: a
// rank may start a sweep once every rank has finished writing its input.
// Each rank owns two monotonic counters (K1 done, K2 done) in IPC-exported
// device memory; after a sweep completes (stream order: its writes, local and
// remote, are performed), one thread raises the counter of every rank with a
// system-scope release, and a rank waits for N * (phase + 1) with a
// system-scope acquire before launching the next sweep.

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

namespace pe3d {

struct SlabFlags {
    unsigned long long* f[MAX_PEERS];
};

__global__ void k_slab_signal(SlabFlags flags, int n) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int q = 0; q < n; ++q)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;\n" ::"l"(flags.f[q]) : "memory");
}

__global__ void k_slab_wait(const unsigned long long* flag, unsigned long long target) {
    if (threadIdx.x != 0) return;
    unsigned long long v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flag) : "memory");
        if (v >= target) break;
        __nanosleep(256);
    }
    __threadfence_system();
}

cudaError_t launch_slab_signal(unsigned long long* const* flags, int n, cudaStream_t s) {
    SlabFlags f{};
    for (int q = 0; q < n && q < MAX_PEERS; ++q) f.f[q] = flags[q];
    k_slab_signal<<<1, 32, 0, s>>>(f, n);
    return cudaGetLastError();
}

cudaError_t launch_slab_wait(const unsigned long long* flag, unsigned long long target, cudaStream_t s) {
    k_slab_wait<<<1, 32, 0, s>>>(flag, target);
    return cudaGetLastError();
}

}  // namespace pe3d
