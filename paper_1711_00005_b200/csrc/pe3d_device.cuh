// pe3d_device.cuh -- complex fp64 arithmetic and shared types for the
// sm_100a range-marching kernels.
//
// Complex multiply follows the FMA pattern numpy's complex128 loops use on
// the reference host: re = fma(ar, br, -(ai*bi)),
// im = fma(ar, bi, ai*br); complex division uses Smith's algorithm as
// numpy does.  Matching them is not required by the 1e-9 parity contract
// but keeps the drift against the oracle at the 1e-15 level per step.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pe3d {

struct __align__(16) cplx {
    double re, im;
};

__host__ __device__ __forceinline__ cplx mk(double re, double im) { cplx c; c.re = re; c.im = im; return c; }
__host__ __device__ __forceinline__ cplx czero() { return mk(0.0, 0.0); }
__host__ __device__ __forceinline__ cplx cone() { return mk(1.0, 0.0); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(a.re + b.re, a.im + b.im); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return mk(a.re - b.re, a.im - b.im); }
__host__ __device__ __forceinline__ cplx cneg(cplx a) { return mk(-a.re, -a.im); }
// real scalar times complex, as numpy's float64 * complex128 (imaginary part of the scalar is 0)
__host__ __device__ __forceinline__ cplx crmul(double s, cplx a) { return mk(s * a.re, s * a.im); }

__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
    return mk(fma(a.re, b.re, -(a.im * b.im)), fma(a.re, b.im, a.im * b.re));
}
// a*b + c with fused accumulation (used on the scan paths, not reference-ordered)
__host__ __device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
    return mk(fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im)));
}

// Smith's complex division a / b (numpy's algorithm for complex128).
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
    const double abr = fabs(b.re), abi = fabs(b.im);
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0) return mk(a.re / abr, a.im / abi);
        const double rat = b.im / b.re;
        const double scl = 1.0 / (b.re + b.im * rat);
        return mk((a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl);
    }
    const double rat = b.re / b.im;
    const double scl = 1.0 / (b.im + b.re * rat);
    return mk((a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl);
}
__host__ __device__ __forceinline__ cplx crecip(cplx b) { return cdiv(cone(), b); }
__host__ __device__ __forceinline__ double cabs(cplx a) { return hypot(a.re, a.im); }

// principal square root
__host__ __device__ __forceinline__ cplx csqrt(cplx z) {
    if (z.re == 0.0 && z.im == 0.0) return czero();
    const double r = hypot(z.re, z.im);
    if (z.re >= 0.0) {
        const double a = sqrt(0.5 * (r + z.re));
        return mk(a, z.im / (2.0 * a));
    }
    const double b = copysign(sqrt(0.5 * (r - z.re)), z.im);
    return mk(z.im / (2.0 * b), b);
}

__device__ __forceinline__ cplx ldc(const cplx* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return mk(v.x, v.y);
}
__device__ __forceinline__ cplx ldc_stream(const cplx* p) {
    const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
    return mk(v.x, v.y);
}
__device__ __forceinline__ void stc(cplx* p, cplx v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im);
}
__device__ __forceinline__ void stc_stream(cplx* p, cplx v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
}

__device__ __forceinline__ cplx shfl_up(cplx v, int d) {
    return mk(__shfl_up_sync(0xffffffffu, v.re, d), __shfl_up_sync(0xffffffffu, v.im, d));
}
__device__ __forceinline__ cplx shfl_down(cplx v, int d) {
    return mk(__shfl_down_sync(0xffffffffu, v.re, d), __shfl_down_sync(0xffffffffu, v.im, d));
}
__device__ __forceinline__ cplx shfl_xor(cplx v, int m) {
    return mk(__shfl_xor_sync(0xffffffffu, v.re, m), __shfl_xor_sync(0xffffffffu, v.im, m));
}
__device__ __forceinline__ cplx shfl_idx(cplx v, int src) {
    return mk(__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src));
}

constexpr double PIVOT_FLOOR = 1e-300;   // ref tridiag.py:31
constexpr double TL_FLOOR_DB = 300.0;    // ref environment.py:29
constexpr int TILE_ROWS = 8;             // depth rows per 128-B device tile

// Per-frequency constants, built on the host from pe3d_coeffs.
struct FreqDev {
    double k0;
    double s_z;          // 1/(k0 dz)^2                  (ref operators.py:94)
    cplx cx_lhs, cx_rhs, cy_lhs, cy_rhs;
    cplx off_z;          // cx_lhs * s_z: depth off-diagonal (ref operators.py:231)
};

// Device layout of the field ("depth tiles"): element (f, m, l) lives at
//   ((f * n_tiles + l / 8) * n_theta + m) * 8 + l % 8
// so the 8 depths of one azimuth form one 128-byte line.  A depth column
// is n_tiles lines of 128 B; an azimuth ring of 8 depths is contiguous.
__host__ __device__ __forceinline__ int64_t tidx(int f, int m, int l, int n_tiles, int n_theta) {
    return ((int64_t(f) * n_tiles + (l >> 3)) * n_theta + m) * 8 + (l & 7);
}

// Error flag shared by all kernels of a march: the first failure (lowest
// packed key) wins.  key = (step << 40) | (sweep << 39) | (freq << 24) | member
struct __align__(16) DevError {
    unsigned long long key;   // ~0ull = none
    int32_t pivot;            // (key, pivot, rank1) change together: one 128-bit CAS
    int32_t rank1;
    int32_t aborted;          // slab march: a peer rank's signal never came (k_slab_wait timeout)
    int32_t pad;
};

// ------------------------------------------------------------- shared helpers

// Record a failure if its key is lower than the recorded one.  The key and
// its payload (pivot, rank1) are replaced together by a 128-bit compare-and-
// swap, so the surviving record is always one failure's own (the lowest key
// with its pivot), whatever the interleaving of concurrent reports.
__device__ __forceinline__ void report_failure(DevError* err, unsigned long long key, int pivot, int rank1) {
    const unsigned long long payload =
        static_cast<unsigned long long>(static_cast<unsigned>(pivot)) | (static_cast<unsigned long long>(rank1) << 32);
    unsigned long long* p = &err->key;
    unsigned long long cur_k = *reinterpret_cast<volatile unsigned long long*>(p);
    unsigned long long cur_p = *reinterpret_cast<volatile unsigned long long*>(p + 1);
    while (key < cur_k) {
        unsigned long long got_k, got_p;
        asm volatile(
            "{\n"
            ".reg .b128 cmp, val, old;\n"
            "mov.b128 cmp, {%2, %3};\n"
            "mov.b128 val, {%4, %5};\n"
            "atom.global.cas.b128 old, [%6], cmp, val;\n"
            "mov.b128 {%0, %1}, old;\n"
            "}\n"
            : "=l"(got_k), "=l"(got_p)
            : "l"(cur_k), "l"(cur_p), "l"(key), "l"(payload), "l"(p)
            : "memory");
        if (got_k == cur_k && got_p == cur_p) break;      // swapped
        cur_k = got_k;
        cur_p = got_p;
    }
}

__host__ __device__ __forceinline__ unsigned long long fail_key(int step, int sweep, int f, int member) {
    return (static_cast<unsigned long long>(step) << 40) | (static_cast<unsigned long long>(sweep) << 39) |
           (static_cast<unsigned long long>(f) << 24) | static_cast<unsigned long long>(member);
}

// s_theta = 1/(k0 r dtheta)^2, evaluated in the reference's order (operators.py:102)
__host__ __device__ __forceinline__ double azimuth_scale(double k0, double r, double dth) {
    const double x = (k0 * r) * dth;
    return 1.0 / (x * x);
}

// cp.async (LDGSTS): 16-byte global -> shared copies, grouped and awaited per thread.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- TMA / mbarrier
// (sm_90+ async proxy; used by the depth sweep to move whole column tiles)

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// Shared-memory complex load/store at a 32-bit shared address (the swizzled
// stage addresses are formed as line_base ^ (i << 4): one LOP3 per element).
__device__ __forceinline__ cplx lds_at(unsigned a) {
    cplx v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.re), "=d"(v.im) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_at(unsigned a, cplx v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v.re), "d"(v.im) : "memory");
}

// Wait for a phase completed by st.async writes of other CTAs of the cluster
// (distributed shared memory).  The writes land in this CTA's shared memory
// and are counted on this CTA's mbarrier as transaction bytes, exactly like a
// TMA load, so the CTA-scope acquire of the default try_wait suffices.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// Address of the same shared-memory object in CTA `rank` of the cluster.
__device__ __forceinline__ unsigned mapa_shared(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16-byte asynchronous store into a cluster peer's shared memory; completion
// (and visibility) is signalled on the peer's mbarrier as transaction bytes.
__device__ __forceinline__ void st_async_cplx(unsigned raddr, cplx v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
                 "d"(v.re), "d"(v.im), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// 4-D tiled TMA load global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const void* tmap, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];\n" ::"r"(smem_addr(smem_dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
        : "memory");
}
// 4-D tiled TMA store shared -> global (bulk group).
__device__ __forceinline__ void tma_store_4d(const void* tmap, int c0, int c1, int c2, int c3, const void* smem_src) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(tmap),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(smem_src))
        : "memory");
}
// 3-D tiled TMA load (the halo granules of a ring segment, k_azimuth_tma HALO).
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_addr(smem_dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
        : "memory");
}
// 5-D tiled TMA load / store (the azimuth sweep's ring segments, see k_azimuth_tma).
__device__ __forceinline__ void tma_load_5d(void* smem_dst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];\n" ::"r"(smem_addr(smem_dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                             const void* smem_src) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(tmap),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(smem_src))
        : "memory");
}
// Plain arrive (release, CTA scope) on a shared-memory mbarrier.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
// Plain bulk copy global -> shared (16-B aligned, size % 16 == 0), completion counted on `bar`.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
// Programmatic dependent launch: wait for the preceding grid (its memory
// visible), and allow the next grid to launch.  Both are no-ops when the
// kernel was not launched with programmatic stream serialization.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace pe3d
