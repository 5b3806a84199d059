// pe3d_host.h -- host-side internals shared by the C ABI translation units
// (pe3d_abi.cu: handles and marches; pe3d_slab.cu: the slab-decomposed
// march): device workspace buffers, the handle, error records and the small
// helpers every entry point uses.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/pe3d_b200.h"
#include "pe3d_internal.h"

namespace pe3d_host {

using pe3d::cplx;

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    uint64_t gen = 0;           // bumped on every (re)allocation: part of the cached graph's key
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        ++gen;
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// Page-locked host staging (the march's parameter uploads are memcpy nodes of
// its graph, so their source must stay valid and in place).
struct PinBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
        cudaError_t e = cudaHostAlloc(&ptr, want, cudaHostAllocDefault);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

struct Handle {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    // march workspace
    DevBuf field_a, field_b, field_c;     // device tiles [F][n_tiles][n_theta][8]
    DevBuf loc_tab, mul_tab, fdev, w_abs, err, k1_tab;
    DevBuf az_cp, az_inv, az_q, az_ring, fail_row, fail_mag, ring_tab;
    // staging for the host entry points
    DevBuf h_local, h_local2, h_u0, h_final, h_tl, h_snap, h_clamped;
    // solve_batch
    DevBuf sb_in, sb_x, sb_cp, sb_inv, sb_y, sb_q;
    // extended medium (profile, lattice, two local-term grids)
    DevBuf med_prof, med_lat, med_local;
    // slab march: ordering counters of the peer-direct transposes
    DevBuf slab_flags;
    // split long columns (LaunchCtx::split): totals, carry responses, carries
    DevBuf sp_tot, sp_aq, sp_pa, sp_cd;
    // column starter: the first temp as one column per frequency (MarchPlan::temp_col)
    DevBuf col_tab;
    // every workspace buffer (release, allocation generation)
    std::vector<DevBuf*> buffers() {
        return {&field_a, &field_b, &field_c, &loc_tab, &mul_tab, &fdev, &w_abs, &err, &k1_tab, &az_cp, &az_inv,
                &az_q, &az_ring, &fail_row, &fail_mag, &ring_tab, &h_local, &h_local2, &h_u0, &h_final, &h_tl,
                &h_snap, &h_clamped, &sb_in, &sb_x, &sb_cp, &sb_inv, &sb_y, &sb_q, &med_prof, &med_lat, &med_local,
                &slab_flags, &sp_tot, &sp_aq, &sp_pa, &sp_cd, &col_tab};
    }
    // changes whenever any workspace buffer was reallocated since the last call
    uint64_t alloc_generation() {
        uint64_t g = 0;
        for (DevBuf* b : buffers()) g += b->gen;
        return g;
    }
    // one cached step-loop graph (reused when a march repeats with identical arguments)
    std::vector<unsigned char> graph_key;
    cudaGraphExec_t graph_exec = nullptr;
    // PE3D_FLAG_PROFILE accounting
    // classes: 0 depth sweep, 1 azimuth sweep, 2 other (3: unused since the split rings
    // became one kernel)
    double prof_ms[4] = {0, 0, 0, 0};
    int32_t prof_n[4] = {0, 0, 0, 0};
    std::vector<double> prof_list[4];     // per launch, in launch order
    // kernels launched by the last march (graph replays included)
    int64_t graph_launches = 0, last_launches = 0;
    int64_t last_h2d_bytes = 0, last_d2h_bytes = 0;     // pe3d_march_host: bytes moved each way
    // concurrent step-loop chains over disjoint frequency groups
    static constexpr int MAX_CHAINS = 8;
    cudaStream_t chain_stream[MAX_CHAINS] = {};
    cudaEvent_t chain_fork = nullptr, chain_join[MAX_CHAINS] = {};
    // TL streaming to the host (pe3d_march_host): one copy stream per chain
    // plus one for the starting sample, and their events
    cudaStream_t tl_side[MAX_CHAINS + 1] = {};
    std::vector<cudaEvent_t> tl_ev;
    // whole-march graph (pe3d_march_device): parameter staging, and the side
    // branch that builds the factorisation and ring tables during the prologue
    PinBuf params_pin;
    PinBuf err_pin;             // the march's error record lands here (page-locked: the readback is asynchronous)
    cudaStream_t pro_side = nullptr;
    cudaEvent_t pro_fork = nullptr, pro_join = nullptr;
    // cached march graphs of pe3d_march_device, most recently used last (a grouped
    // pe3d_march_host marches several frequency groups per call, one graph pair each)
    struct MarchGraph {
        std::vector<unsigned char> key;
        cudaGraphExec_t pre = nullptr, steps = nullptr;
        int64_t launches = 0;
    };
    static constexpr int MAX_MARCH_GRAPHS = 16;    // LRU; a grouped host march uses one entry per frequency group
    std::vector<MarchGraph> march_graphs;
    // pe3d_march_host: copy stream for the per-group results and its event
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_ev = nullptr;
    // a device-to-host copy the next march enqueues on copy_stream right behind its last kernel,
    // before the host waits for the march (pe3d_march_host: a group's final slab)
    struct PostCopy { void* dst = nullptr; const void* src = nullptr; size_t bytes = 0; } post_copy;
};

// Launch wrapper: in profile mode, bracket each launch with events.
struct Prof {
    Handle* h;
    bool on;
    cudaStream_t s;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    int64_t launches = 0;                               // kernels enqueued through run()
    template <class F> cudaError_t run(int cls, F&& f) {
        ++launches;
        if (!on) return f();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        cudaError_t e = f();
        cudaEventRecord(b, s);
        ev.push_back({cls, {a, b}});
        return e;
    }
    void collect() {
        if (!on) return;
        for (int k = 0; k < 4; ++k) { h->prof_ms[k] = 0; h->prof_n[k] = 0; h->prof_list[k].clear(); }
        for (auto& p : ev) {
            float ms = 0;
            cudaEventSynchronize(p.second.second);
            cudaEventElapsedTime(&ms, p.second.first, p.second.second);
            h->prof_ms[p.first] += ms;
            h->prof_n[p.first] += 1;
            h->prof_list[p.first].push_back(ms);
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        ev.clear();
    }
};

constexpr unsigned long long NO_ERROR = ~0ull;

inline void set_error(pe3d_error* err, int32_t range_index, int32_t sweep, const char* fmt, const char* what) {
    if (!err) return;
    std::memset(err, 0, sizeof(*err));
    err->range_index = range_index;
    err->sweep = sweep;
    std::snprintf(err->message, sizeof(err->message), fmt, what);
}

inline int cuda_fail(pe3d_error* err, cudaError_t e, const char* where) {
    if (err) {
        std::memset(err, 0, sizeof(*err));
        err->range_index = -1;
        std::snprintf(err->message, sizeof(err->message), "%s: %s", where, cudaGetErrorString(e));
    }
    return PE3D_CUDA_ERROR;
}

inline int bad_arg(pe3d_error* err, const char* what) {
    set_error(err, -1, 0, "%s", what);
    return PE3D_BAD_ARGUMENT;
}

#define CK(call, where)                                   \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(err, e_, where); \
    } while (0)

inline int check_grid(const pe3d_grid* g, const pe3d_coeffs* c, pe3d_error* err) {
    if (!g || !c) return bad_arg(err, "null grid or coefficients");
    if (g->n_freq < 1) return bad_arg(err, "n_freq >= 1");
    if (g->n_theta < 3 || g->n_depth < 3) return bad_arg(err, "n_theta >= 3 and n_depth >= 3");
    if (g->n_theta > 4096) return bad_arg(err, "n_theta <= 4096 (ring kernels)");
    if (g->n_depth > 4096) return bad_arg(err, "n_depth <= 4096 (depth kernels)");
    if (g->n_steps < 0) return bad_arg(err, "n_steps >= 0");
    if (g->output_stride < 1) return bad_arg(err, "output_stride >= 1");
    if (g->topology != PE3D_PERIODIC && g->topology != PE3D_SECTOR) return bad_arg(err, "topology");
    if (!(g->delta_r > 0) || !(g->delta_theta > 0) || !(g->delta_z > 0)) return bad_arg(err, "spacings > 0");
    if (!(g->r_input > 0)) return bad_arg(err, "r_input > 0");
    for (int f = 0; f < g->n_freq; ++f)
        if (!(c[f].k0 > 0)) return bad_arg(err, "k0 > 0");
    return PE3D_OK;
}

inline std::vector<pe3d::FreqDev> freq_table(const pe3d_grid* g, const pe3d_coeffs* c) {
    std::vector<pe3d::FreqDev> t(g->n_freq);
    for (int f = 0; f < g->n_freq; ++f) {
        pe3d::FreqDev& d = t[f];
        d.k0 = c[f].k0;
        const double kz = c[f].k0 * g->delta_z;
        d.s_z = 1.0 / (kz * kz);                                    // ref operators.py:94
        d.cx_lhs = pe3d::mk(c[f].cx_lhs.re, c[f].cx_lhs.im);
        d.cx_rhs = pe3d::mk(c[f].cx_rhs.re, c[f].cx_rhs.im);
        d.cy_lhs = pe3d::mk(c[f].cy_lhs.re, c[f].cy_lhs.im);
        d.cy_rhs = pe3d::mk(c[f].cy_rhs.re, c[f].cy_rhs.im);
        d.off_z = pe3d::mk(d.cx_lhs.re * d.s_z, d.cx_lhs.im * d.s_z);  // complex(coeff * s)
    }
    return t;
}

// |w(r)| exactly as the reference computes it (environment.py:287-294):
// abs(complex(cos(k0 r), sin(k0 r)) / sqrt(r))
inline double hankel_abs_host(double k0, double r) {
    const double s = std::sqrt(r);
    return std::hypot(std::cos(k0 * r) / s, std::sin(k0 * r) / s);
}

inline bool needs_serial(const pe3d_grid* g, const std::vector<pe3d::FreqDev>& fd) {
    if (g->flags & PE3D_FLAG_SERIAL) return true;
    for (const auto& d : fd)
        if (d.off_z.re == 0.0 && d.off_z.im == 0.0) return true;
    return false;
}

// ------------------------------------------------------------ azimuth failures
// The periodic azimuth sweep solves B = diag I + off (S + S^-1) by its
// circulant factorisation, which has no pivots.  Which steps the REFERENCE
// would abort on is decided here, on the host, by the reference's own
// algorithm: the Sherman-Morrison cyclic solve of the constant matrix
// (ref tridiag.py:186-212 with operators.py:256-262: sub = sup = off,
// main = diag), its pivot checks (tridiag.py:145-167) and its rank-1
// denominator check (:205-210), in numpy's arithmetic (pe3d_device.cuh).
// All Nz members share the matrix, so the failing member is 0 (argmin of
// equal magnitudes, ref tridiag.py:146-148, lowest tile :274-280).  A strictly
// diagonally dominant matrix with margin cannot fail those checks, so the
// O(n) recurrence runs only for the others.
struct HostFail {
    unsigned long long key = ~0ull;
    int32_t pivot = 0, rank1 = 0;
};

// true when the reference's cyclic solve of (diag, off) of size n raises
inline bool reference_cyclic_fails(pe3d::cplx diag, pe3d::cplx off, int n, int32_t* pivot, int32_t* rank1) {
    using namespace pe3d;
    const double ad = cabs(diag), ao = cabs(off);
    if (ad - 2.0 * ao > 1e-200 * ad && ad - 2.0 * ao > 1e-280) return false;
    const cplx alpha = off, beta = off;
    const cplx gamma = ad > 0.0 ? cneg(diag) : cone();
    const cplx main0 = csub(diag, gamma);
    const cplx mainl = csub(diag, cdiv(cmul(alpha, beta), gamma));
    auto main_at = [&](int k) { return k == 0 ? main0 : (k == n - 1 ? mainl : diag); };
    std::vector<cplx> cp(n > 1 ? n - 1 : 1), inv(n), x(n);
    for (int k = 0; k < n; ++k) {
        const cplx denom = k == 0 ? main_at(0) : csub(main_at(k), cmul(off, cp[k - 1]));
        if (cabs(denom) < PIVOT_FLOOR) { *pivot = k; *rank1 = 0; return true; }
        inv[k] = crecip(denom);
        if (k < n - 1) cp[k] = cmul(off, inv[k]);
    }
    // q = A'^-1 (gamma e_0 + beta e_(n-1))
    for (int k = 0; k < n; ++k) {
        const cplx spike = k == 0 ? gamma : (k == n - 1 ? beta : czero());
        x[k] = k == 0 ? cmul(spike, inv[0]) : cmul(csub(spike, cmul(off, x[k - 1])), inv[k]);
    }
    for (int k = n - 2; k >= 0; --k) x[k] = csub(x[k], cmul(cp[k], x[k + 1]));
    const cplx weight = cdiv(alpha, gamma);
    const cplx denom = cadd(cadd(cone(), x[0]), cmul(weight, x[n - 1]));
    if (cabs(denom) < PIVOT_FLOOR) { *pivot = n; *rank1 = 1; return true; }
    return false;
}

// lowest (step, frequency) at which the reference's periodic azimuth solve
// would raise, over the steps of a march
inline HostFail azimuth_failures(const pe3d_grid* g, const pe3d_coeffs* c) {
    HostFail hf;
    if (g->topology != PE3D_PERIODIC) return hf;
    for (int s = 0; s < g->n_steps; ++s) {
        const int j_new = g->first_index + s + 1;
        const double r_new = g->r_start + j_new * g->delta_r;          // Grid3D.range_at
        for (int f = 0; f < g->n_freq; ++f) {
            const pe3d::cplx cy = pe3d::mk(c[f].cy_lhs.re, c[f].cy_lhs.im);
            const double sc = pe3d::azimuth_scale(c[f].k0, r_new, g->delta_theta);
            const pe3d::cplx diag = pe3d::csub(pe3d::cone(), pe3d::crmul(sc, pe3d::crmul(2.0, cy)));
            const pe3d::cplx off = pe3d::crmul(sc, cy);
            int32_t pivot, rank1;
            if (reference_cyclic_fails(diag, off, g->n_theta, &pivot, &rank1)) {
                const unsigned long long key = pe3d::fail_key(j_new, 1, f, 0);
                if (key < hf.key) hf = HostFail{key, pivot, rank1};
            }
        }
        if (hf.key != ~0ull) break;                                     // later steps have larger keys
    }
    return hf;
}

inline int decode_error(Handle* h, cudaStream_t stream, pe3d_error* err, const HostFail* hf = nullptr) {
    CK(h->err_pin.ensure(sizeof(pe3d::DevError)), "alloc pinned error record");
    CK(cudaMemcpyAsync(h->err_pin.ptr, h->err.ptr, sizeof(pe3d::DevError), cudaMemcpyDeviceToHost, stream),
       "error readback");
    if (h->post_copy.bytes) {
        // the caller's copy of this march's result (pe3d_march_host: a group's final slab) leaves
        // right behind the last kernel -- queued after the error record, which the host waits for,
        // and before the host has seen the march complete (~0.2 ms later)
        const Handle::PostCopy pc = h->post_copy;
        h->post_copy = Handle::PostCopy{};
        CK(cudaEventRecord(h->copy_ev, stream), "event");
        CK(cudaStreamWaitEvent(h->copy_stream, h->copy_ev, 0), "event");
        CK(cudaMemcpyAsync(pc.dst, pc.src, pc.bytes, cudaMemcpyDeviceToHost, h->copy_stream), "D2H");
    }
    CK(cudaStreamSynchronize(stream), "march");
    pe3d::DevError de;
    std::memcpy(&de, h->err_pin.ptr, sizeof(de));
    if (hf && hf->key < de.key) {
        de.key = hf->key;
        de.pivot = hf->pivot;
        de.rank1 = hf->rank1;
    }
    if (de.aborted) {
        if (err) {
            std::memset(err, 0, sizeof(*err));
            err->range_index = -1;
            std::snprintf(err->message, sizeof(err->message),
                          "slab march aborted: a peer rank did not signal within PE3D_SLAB_TIMEOUT_MS");
        }
        return PE3D_CUDA_ERROR;
    }
    if (de.key == NO_ERROR) return PE3D_OK;
    if (err) {
        std::memset(err, 0, sizeof(*err));
        err->range_index = int32_t(de.key >> 40);
        err->sweep = int32_t((de.key >> 39) & 1);
        err->frequency = int32_t((de.key >> 24) & 0x7fff);
        err->member = int32_t(de.key & 0xffffff);
        err->pivot = de.pivot;
        err->rank1 = de.rank1;
        std::snprintf(err->message, sizeof(err->message), "singular system: pivot %d, batch member %d", de.pivot,
                      err->member);
    }
    return PE3D_SINGULAR;
}

}  // namespace pe3d_host
