// pe3d_abi.cu -- the C ABI of libpe3d_b200.so (include/pe3d_b200.h): handle
// and workspace management, the device-resident march (one CUDA graph per
// call), the general single step, the batched tridiagonal solve and the
// device-medium march.  The slab-decomposed march is in pe3d_slab.cu.
//
// Reference entry points replaced (pkg/src/pe3d): run_frequency
// (marching.py:144-193) and the frequency batch of frequency_farm
// (parallel.py:143-185) -> pe3d_march_*; range_step (marching.py:93-136)
// -> pe3d_step_general_host; solve_batch (tridiag.py:248-281) ->
// pe3d_solve_batch_host.

#include <complex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <tuple>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include "../../include/pe3d_b200.h"
#include "pe3d_host.h"
#include "pe3d_internal.h"

using pe3d::cplx;

namespace {

using namespace pe3d_host;

struct MarchPlan {
    pe3d::LaunchCtx ctx;
    bool serial;
    int64_t field_elems;
    int n_samples;
    // column starter: the prologue leaves the first temp as one column per frequency
    // ([F][n_tiles][8]) and the first depth sweep reads it (null: the full field)
    pe3d::cplx* temp_col;
    // split rings (k_azimuth_tma SEG/HALO): per step the number of neighbouring points per side
    // a ring segment takes its carries from (0: that step runs the cluster kernel)
    const int* sr_span;
};

// Split-ring plan of a march: per step, the number of neighbouring points per side
// whose weights |rho|^t still matter to a ring segment's carries, from the largest
// |rho| of the step's frequencies: the dropped terms are below 1e-22 of the carries.
// 0 (the exact cluster kernel) where that span exceeds max_span, the halo a segment
// can load (cfg5: the first 168 steps, rho -> 1 at short range).
static std::vector<int> sring_spans(const pe3d_grid* g, const std::vector<pe3d::FreqDev>& fd, int max_span) {
    std::vector<int> span(g->n_steps, 0);
    for (int s = 0; s < g->n_steps; ++s) {
        const double r_new = g->r_start + double(g->first_index + s + 1) * g->delta_r;
        double rmax = 0.0;
        for (const auto& d : fd) {
            const double sc = pe3d::azimuth_scale(d.k0, r_new, g->delta_theta);
            const cplx diag = pe3d::csub(pe3d::cone(), pe3d::crmul(sc, pe3d::crmul(2.0, d.cy_lhs)));
            const cplx off = pe3d::crmul(sc, d.cy_lhs);
            if (off.re == 0.0 && off.im == 0.0) continue;          // rho = 0
            const cplx tq = pe3d::crmul(0.5, pe3d::cneg(pe3d::cdiv(diag, off)));
            cplx sq = pe3d::csqrt(pe3d::csub(pe3d::cmul(tq, tq), pe3d::cone()));
            if (tq.re * sq.re + tq.im * sq.im < 0.0) sq = pe3d::cneg(sq);
            rmax = std::max(rmax, pe3d::cabs(pe3d::crecip(pe3d::cadd(tq, sq))));
        }
        if (rmax == 0.0) { span[s] = 1; continue; }
        if (!(rmax < 1.0 - 1e-9)) continue;
        const double need = (std::log(1e-22) + std::log(1.0 - rmax * rmax)) / std::log(rmax) + 2.0;
        if (need <= double(max_span)) span[s] = std::max(1, int(std::ceil(need)));
    }
    return span;
}

// Number of concurrent step-loop chains.  Frequencies are independent, so a
// march runs disjoint frequency groups as parallel graph branches: each
// chain's launch ramp, pipeline fill and tail are filled by the other chains'
// CTAs.  Measured on cfg4 (per-GPU step, 1 -> 2 chains): 64 frequencies
// 216 -> 208 us, 32: 119 -> 105, 16: 66 -> 57, 8: 39 -> 34.5.  Three chains
// pay off only with few columns per resident CTA (8 frequencies: 33.2 ->
// 31.9 us; 16: 56.9 -> 61.5).  PE3D_CHAINS overrides.
int step_chains(const pe3d::LaunchCtx& c, bool profiling) {
    if (profiling || c.n_freq < 2) return 1;
    const char* env = getenv("PE3D_CHAINS");
    const int64_t cols = int64_t(c.n_freq) * c.n_theta;
    // few columns per SM (8 frequencies per GPU): one chain per frequency, up to
    // MAX_CHAINS (8 frequencies: 3 chains 31.2 us, 4 chains 29.6-30.0, 8 chains
    // 28.3 us per step); otherwise two (16 frequencies: 2 chains 54.2 us, 4 chains 55.4)
    int n = env ? atoi(env) : (cols <= int64_t(6) * 3 * c.num_sms ? Handle::MAX_CHAINS : 2);
    if (n > Handle::MAX_CHAINS) n = Handle::MAX_CHAINS;
    if (n > c.n_freq) n = c.n_freq;
    return n < 1 ? 1 : n;
}

// TL streaming (pe3d_march_host): the device keeps a ring of R samples per
// frequency; after the kernel that writes sample k of a chain's frequencies,
// the chain's copy stream moves it to the page-locked host stack, and the
// kernel that writes sample k + R into the same slot waits for that copy.
// The copies are graph nodes next to the sweeps, so they overlap the march.
struct TlSink {
    double* host;       // [F][S][n_theta][n_depth], page-locked
    int S;              // samples of the host stack
    int R;              // device ring slots per frequency
    int col0;           // sample 0 is the same for every azimuth (column starter on a periodic ring):
                        // only its first azimuth row leaves the device, the caller replicates it
    int pad_;           // (the struct's bytes are part of the graph key: no padding)
};

// events: per copy stream c (0..MAX_CHAINS): R "copied" slots + 1 "written"
static cudaEvent_t& tl_event(Handle* h, int c, int slot, const TlSink& sk) {
    return h->tl_ev[size_t(c) * (sk.R + 1) + slot];
}

static cudaError_t tl_prepare(Handle* h, const TlSink& sk) {
    const size_t need = size_t(Handle::MAX_CHAINS + 1) * (sk.R + 1);
    while (h->tl_ev.size() < need) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r != cudaSuccess) return r;
        h->tl_ev.push_back(e);
    }
    for (int c = 0; c <= Handle::MAX_CHAINS; ++c)
        if (!h->tl_side[c]) {
            cudaError_t r = cudaStreamCreateWithFlags(&h->tl_side[c], cudaStreamNonBlocking);
            if (r != cudaSuccess) return r;
        }
    return cudaSuccess;
}

// before the kernel writing sample k (k >= 1) of copy stream c: the slot's
// previous sample (k - R) must have left for the host
static cudaError_t tl_before(Handle* h, const TlSink& sk, int c, int k, cudaStream_t st) {
    const int prev = k - sk.R;
    if (prev < 0) return cudaSuccess;
    const int cs = prev == 0 ? Handle::MAX_CHAINS : c;      // sample 0 is copied by the starter stream
    return cudaStreamWaitEvent(st, tl_event(h, cs, prev % sk.R, sk), 0);
}

// after the kernel writing sample k of frequencies [f0, f0 + nf) on st
static cudaError_t tl_after(Handle* h, const TlSink& sk, int c, int k, int f0, int nf, int64_t oe,
                            const double* ring, cudaStream_t st, int64_t width = 0) {
    cudaStream_t side = h->tl_side[c];
    cudaError_t e = cudaEventRecord(tl_event(h, c, sk.R, sk), st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, tl_event(h, c, sk.R, sk), 0);
    const size_t w = size_t(oe) * sizeof(double);
    const size_t wcopy = width ? size_t(width) * sizeof(double) : w;     // the sample's leading doubles only
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(sk.host + (int64_t(f0) * sk.S + k) * oe, sk.S * w, ring + (int64_t(f0) * sk.R + k % sk.R) * oe,
                              sk.R * w, wcopy, nf, cudaMemcpyDeviceToHost, side);
    if (e == cudaSuccess) e = cudaEventRecord(tl_event(h, c, k % sk.R, sk), side);
    return e;
}

// join every copy stream back into st (end of the step loop)
static cudaError_t tl_join(Handle* h, const TlSink& sk, int n_copy_streams, cudaStream_t st) {
    cudaError_t first = cudaSuccess;
    for (int c = 0; c <= Handle::MAX_CHAINS; ++c) {
        if (c >= n_copy_streams && c != Handle::MAX_CHAINS) continue;
        // a chain's copy stream joined the step loop (and a graph capture) only if
        // the loop records a sample (k >= 1); joining an idle one would wait on
        // work outside the capture
        if (c != Handle::MAX_CHAINS && sk.S <= 1) continue;
        cudaError_t e = cudaEventRecord(tl_event(h, c, sk.R, sk), h->tl_side[c]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, tl_event(h, c, sk.R, sk), 0);
        if (e != cudaSuccess && first == cudaSuccess) first = e;
    }
    return first;
}

// Step loop of the parallel (scan) path for frequencies [f0, f0 + nf) on
// stream `st`; all pointers are offset to the group.
cudaError_t enqueue_group(Handle* h, const pe3d_grid* g, const MarchPlan& p, int f0, int nf, cudaStream_t st,
                          double* d_tl, cplx* d_snap, cplx* d_final, int64_t* d_clamped, const double* d_wabs,
                          Prof& prof, const TlSink* sink, int chain) {
    const pe3d::LaunchCtx& c = p.ctx;
    const int E = pe3d::ring_table_elems(c.n_theta);
    const int64_t fe = int64_t(c.n_tiles) * c.n_theta * 8;     // field elements per frequency
    const int64_t oe = int64_t(c.n_theta) * g->n_depth;         // output elements per frequency and sample
    pe3d::LaunchCtx cg = c;
    cg.n_freq = nf;
    cg.fdev = c.fdev + f0;
    cg.loc_tab = c.loc_tab + int64_t(f0) * c.n_tiles * 8;
    cg.mul_tab = c.mul_tab + int64_t(f0) * c.n_tiles * 8;
    if (c.k1_tab)
        cg.k1_tab = c.k1_tab + (c.split ? int64_t(f0) * c.split * pe3d::k1_stride(128) : pe3d::k1_tab_elems(f0, c.n_tiles));
    if (c.split) {
        cg.sp_tot = c.sp_tot + int64_t(f0) * c.split * c.n_theta * 2;
        cg.sp_aq = c.sp_aq + int64_t(f0) * c.n_tiles * 16;
        cg.sp_pa = c.sp_pa + int64_t(f0) * c.split * 3;
        cg.sp_cd = c.sp_cd + int64_t(f0) * c.split * 2 * c.n_theta;
    }
    cg.stream = st;
    // programmatic dependent launch of the step sweeps: each sweep's table
    // loads and CTA launch overlap the previous sweep's tail (8 frequencies
    // per GPU 27.9 -> 26.9 us/step; neutral at 64)
    cg.pdl = getenv("PE3D_NO_PDL") == nullptr;
    cplx* A = h->field_a.as<cplx>() + f0 * fe;
    cplx* B = h->field_b.as<cplx>() + f0 * fe;
    // With few columns per CTA (few frequencies per GPU) each chain's persistent
    // depth-sweep grid is sized for its share of the SMs, so both chains' CTAs
    // are resident together instead of one chain queueing behind the other
    // (8 frequencies per GPU: 33.7 -> 33.2 us; with 16 it costs 3%, hence the bound)
    pe3d::LaunchCtx ck1 = cg;
    if (nf < c.n_freq && int64_t(nf) * c.n_theta <= int64_t(3) * 3 * c.num_sms)
        ck1.num_sms = std::max(1, int(int64_t(c.num_sms) * nf / c.n_freq));
    for (int s = 0; s < g->n_steps; ++s) {
        const int j_new = g->first_index + s + 1;
        const double r_new = g->r_start + j_new * g->delta_r;      // Grid3D.range_at
        pe3d::LaunchCtx ck = ck1;
        if (s == 0 && p.temp_col) ck.src_col = p.temp_col + int64_t(f0) * c.n_tiles * 8;
        cudaError_t e = prof.run(0, [&] { return pe3d::launch_depth_scan(ck, A, B); });
        if (e != cudaSuccess) return e;
        if (c.split) {                                      // exact sub-column carries for the azimuth sweep
            e = prof.run(2, [&] { return pe3d::launch_split_carry(cg); });
            if (e != cudaSuccess) return e;
        }
        pe3d::EpilogueArgs ea{};
        const bool record = ((s + 1) % g->output_stride) == 0;
        const int k = (s + 1) / g->output_stride;          // sample index
        const bool stream_tl = record && d_tl && sink;
        const int tl_slots = sink ? sink->R : p.n_samples;
        if (stream_tl) {
            e = tl_before(h, *sink, chain, k, st);
            if (e != cudaSuccess) return e;
        }
        ea.n_samples = p.n_samples;
        ea.tl = record && d_tl ? d_tl + int64_t(f0) * tl_slots * oe : nullptr;
        ea.snap = record && d_snap ? d_snap + int64_t(f0) * p.n_samples * oe : nullptr;
        ea.final_out = (s == g->n_steps - 1) && d_final ? d_final + f0 * oe : nullptr;
        ea.clamped = d_clamped ? d_clamped + f0 : nullptr;
        ea.sample = k;
        ea.w_abs = d_wabs + int64_t(k) * g->n_freq + f0;
        ea.periodic = true;
        ea.write_temp = (s < g->n_steps - 1);
        if (sink && !d_snap) {                              // TL in the device ring
            ea.n_samples = sink->R;
            ea.sample = k % sink->R;
        }
        const cplx* tab = h->ring_tab.as<cplx>() + (int64_t(s) * c.n_freq + f0) * E;
        if (p.sr_span && p.sr_span[s] > 0 && !ea.final_out) {
            // segments on all SMs, carries from the neighbours' halo points, TL in the same kernel
            e = prof.run(1, [&] { return pe3d::launch_azimuth_halo(cg, B, A, tab, ea, p.sr_span[s]); });
        } else {
            e = prof.run(1, [&] { return pe3d::launch_azimuth_scan(cg, B, A, tab, r_new, ea); });
        }
        if (e != cudaSuccess) return e;
        if (stream_tl) {
            e = tl_after(h, *sink, chain, k, f0, nf, oe, d_tl, st);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t enqueue_steps_body(Handle* h, const pe3d_grid* g, const MarchPlan& p, const cplx* d_local,
                               double* d_tl, cplx* d_snap, cplx* d_final, int64_t* d_clamped,
                               const double* d_wabs, Prof& prof, const TlSink* sink, int* n_copy_streams);

// Enqueue the step loop (the body graphed by pe3d_march_device).  With a TL
// sink the starting sample (written by the prologue) leaves first, and every
// copy stream is joined back at the end.
cudaError_t enqueue_steps(Handle* h, const pe3d_grid* g, const MarchPlan& p, const cplx* d_local,
                          double* d_tl, cplx* d_snap, cplx* d_final, int64_t* d_clamped,
                          const double* d_wabs, Prof& prof, const TlSink* sink) {
    const pe3d::LaunchCtx& c = p.ctx;
    if (sink && d_tl) {
        const int64_t oe = int64_t(c.n_theta) * g->n_depth;
        cudaError_t e = tl_after(h, *sink, Handle::MAX_CHAINS, 0, 0, c.n_freq, oe, d_tl, c.stream,
                                 sink->col0 ? g->n_depth : oe);
        if (e != cudaSuccess) return e;
    }
    int n_copy = 0;
    cudaError_t e = enqueue_steps_body(h, g, p, d_local, d_tl, d_snap, d_final, d_clamped, d_wabs, prof,
                                       sink && d_tl ? sink : nullptr, &n_copy);
    if (sink && d_tl) {
        cudaError_t e2 = tl_join(h, *sink, n_copy, c.stream);
        if (e == cudaSuccess) e = e2;
    }
    return e;
}

cudaError_t enqueue_steps_body(Handle* h, const pe3d_grid* g, const MarchPlan& p, const cplx* d_local,
                               double* d_tl, cplx* d_snap, cplx* d_final, int64_t* d_clamped,
                               const double* d_wabs, Prof& prof, const TlSink* sink, int* n_copy_streams) {
    const pe3d::LaunchCtx& c = p.ctx;
    cplx* A = h->field_a.as<cplx>();
    cplx* B = h->field_b.as<cplx>();
    cplx* C = h->field_c.as<cplx>();
    const bool periodic = g->topology == PE3D_PERIODIC;
    *n_copy_streams = 1;
    if (periodic && !p.serial) {
        const int chains = step_chains(c, prof.on);
        *n_copy_streams = chains;
        if (chains == 1)
            return enqueue_group(h, g, p, 0, c.n_freq, c.stream, d_tl, d_snap, d_final, d_clamped, d_wabs, prof, sink,
                                 0);
        cudaError_t e = cudaSuccess;
        if (!h->chain_fork) e = cudaEventCreateWithFlags(&h->chain_fork, cudaEventDisableTiming);
        for (int k = 0; k < chains && e == cudaSuccess; ++k) {
            if (!h->chain_stream[k]) e = cudaStreamCreateWithFlags(&h->chain_stream[k], cudaStreamNonBlocking);
            if (e == cudaSuccess && !h->chain_join[k])
                e = cudaEventCreateWithFlags(&h->chain_join[k], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) return e;
        e = cudaEventRecord(h->chain_fork, c.stream);
        if (e != cudaSuccess) return e;
        // every forked chain is joined back, also after a failed launch, so a
        // stream capture in progress can always be ended cleanly
        cudaError_t first = cudaSuccess;
        for (int k = 0; k < chains; ++k) {
            const int f0 = int(int64_t(c.n_freq) * k / chains), f1 = int(int64_t(c.n_freq) * (k + 1) / chains);
            e = cudaStreamWaitEvent(h->chain_stream[k], h->chain_fork, 0);
            if (e != cudaSuccess) { if (first == cudaSuccess) first = e; break; }
            if (first == cudaSuccess) {
                e = enqueue_group(h, g, p, f0, f1 - f0, h->chain_stream[k], d_tl, d_snap, d_final, d_clamped, d_wabs,
                                  prof, sink, k);
                if (e != cudaSuccess) first = e;
            }
            cudaError_t e2 = cudaEventRecord(h->chain_join[k], h->chain_stream[k]);
            if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(c.stream, h->chain_join[k], 0);
            if (e2 != cudaSuccess && first == cudaSuccess) first = e2;
        }
        return first;
    }
    for (int s = 0; s < g->n_steps; ++s) {
        const int j_new = g->first_index + s + 1;
        const double r_new = g->r_start + j_new * g->delta_r;          // Grid3D.range_at
        cudaError_t e;
        if (p.serial) {
            e = prof.run(0, [&] { return pe3d::launch_depth_serial(c, A, B, C, d_local, d_local, g->n_depth, 0, 1,
                                                                   h->fail_row.as<int>(), h->fail_mag.as<double>()); });
            if (e == cudaSuccess)
                e = prof.run(2, [&] { return pe3d::launch_reduce_failures(h->fail_row.as<int>(), h->fail_mag.as<double>(),
                                                                          c.n_freq, c.n_theta, j_new, 0, -1, c.err,
                                                                          c.stream); });
        } else {
            e = prof.run(0, [&] { return pe3d::launch_depth_scan(c, A, B); });
        }
        if (e != cudaSuccess) return e;
        pe3d::EpilogueArgs ea{};
        const bool record = ((s + 1) % g->output_stride) == 0;
        const int k = (s + 1) / g->output_stride;
        const bool stream_tl = record && d_tl && sink;
        if (stream_tl) {
            e = tl_before(h, *sink, 0, k, c.stream);
            if (e != cudaSuccess) return e;
        }
        ea.tl = record ? d_tl : nullptr;
        ea.snap = record ? d_snap : nullptr;
        ea.final_out = (s == g->n_steps - 1) ? d_final : nullptr;
        ea.clamped = d_clamped;
        ea.n_samples = p.n_samples;
        ea.sample = k;
        ea.w_abs = d_wabs + int64_t(k) * g->n_freq;
        ea.periodic = periodic;
        ea.write_temp = (s < g->n_steps - 1);
        if (sink && !d_snap) {
            ea.n_samples = sink->R;
            ea.sample = k % sink->R;
        }
        e = prof.run(1, [&] { return pe3d::launch_azimuth_serial(c, B, C, h->az_cp.as<cplx>(), h->az_inv.as<cplx>(),
                                                                 h->az_q.as<cplx>(), h->az_ring.as<cplx>(), r_new,
                                                                 j_new); });
        if (e == cudaSuccess) e = prof.run(2, [&] { return pe3d::launch_finish(c, C, 1, A, r_new, ea); });
        if (e != cudaSuccess) return e;
        if (stream_tl) {
            e = tl_after(h, *sink, 0, k, 0, c.n_freq, int64_t(c.n_theta) * g->n_depth, d_tl, c.stream);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

}  // namespace

extern "C" {

int pe3d_abi_version(void) { return PE3D_ABI_VERSION; }

int pe3d_device_count(int32_t* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = (e == cudaSuccess) ? n : 0;
    return e == cudaSuccess ? PE3D_OK : PE3D_CUDA_ERROR;
}

int32_t pe3d_sample_count(int32_t n_steps, int32_t output_stride) {
    if (n_steps < 0 || output_stride < 1) return -1;
    return 1 + n_steps / output_stride;
}

int pe3d_handle_create(int32_t device, void** handle, pe3d_error* err) {
    if (!handle) return bad_arg(err, "null handle pointer");
    *handle = nullptr;
    int n = 0;
    CK(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) return bad_arg(err, "device index out of range");
    CK(cudaSetDevice(device), "cudaSetDevice");
    Handle* h = new (std::nothrow) Handle();
    if (!h) return bad_arg(err, "out of host memory");
    h->device = device;
    CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device), "attribute");
    CK(cudaStreamCreate(&h->stream), "cudaStreamCreate");
    *handle = h;
    return PE3D_OK;
}

int pe3d_handle_destroy(void* handle) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return PE3D_OK;
    cudaSetDevice(h->device);
    for (DevBuf* b : h->buffers()) b->release();
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    for (auto& mg : h->march_graphs) {
        if (mg.pre) cudaGraphExecDestroy(mg.pre);
        if (mg.steps) cudaGraphExecDestroy(mg.steps);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->copy_ev) cudaEventDestroy(h->copy_ev);
    for (int k = 0; k <= Handle::MAX_CHAINS; ++k)
        if (h->tl_side[k]) cudaStreamDestroy(h->tl_side[k]);
    for (cudaEvent_t e : h->tl_ev) cudaEventDestroy(e);
    for (int k = 0; k < Handle::MAX_CHAINS; ++k) {
        if (h->chain_stream[k]) cudaStreamDestroy(h->chain_stream[k]);
        if (h->chain_join[k]) cudaEventDestroy(h->chain_join[k]);
    }
    if (h->chain_fork) cudaEventDestroy(h->chain_fork);
    if (h->pro_side) cudaStreamDestroy(h->pro_side);
    if (h->pro_fork) cudaEventDestroy(h->pro_fork);
    if (h->pro_join) cudaEventDestroy(h->pro_join);
    h->params_pin.release();
    h->err_pin.release();
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return PE3D_OK;
}

static int march_device_impl(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_c128* d_local,
                             const pe3d_c128* d_u0, pe3d_c128* d_u_final, double* d_tl, pe3d_c128* d_snapshots,
                             int64_t* d_clamped, void* stream_v, pe3d_error* err, const TlSink* sink);

int pe3d_march_device(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_c128* d_local,
                      const pe3d_c128* d_u0, pe3d_c128* d_u_final, double* d_tl, pe3d_c128* d_snapshots,
                      int64_t* d_clamped, void* stream_v, pe3d_error* err) {
    return march_device_impl(handle, g, coeffs, d_local, d_u0, d_u_final, d_tl, d_snapshots, d_clamped, stream_v, err,
                             nullptr);
}

// sink != null (pe3d_march_host with a page-locked TL stack): d_tl is the
// device ring [F][R][n_theta][n_depth] and the samples stream to sink->host.
static int march_device_impl(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_c128* d_local,
                             const pe3d_c128* d_u0, pe3d_c128* d_u_final, double* d_tl, pe3d_c128* d_snapshots,
                             int64_t* d_clamped, void* stream_v, pe3d_error* err, const TlSink* sink) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return bad_arg(err, "null handle");
    int st = check_grid(g, coeffs, err);
    if (st != PE3D_OK) return st;
    if (!d_local || !d_u0) return bad_arg(err, "null local or u0");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    cudaStream_t stream = stream_v ? static_cast<cudaStream_t>(stream_v) : h->stream;

    const int F = g->n_freq, NT = g->n_theta, NZ = g->n_depth;
    const int n_tiles = (NZ + 7) / 8;
    const int64_t field = int64_t(F) * n_tiles * NT * 8;
    const int S = pe3d_sample_count(g->n_steps, g->output_stride);
    std::vector<pe3d::FreqDev> fd = freq_table(g, coeffs);
    MarchPlan p{};
    p.serial = needs_serial(g, fd);
    p.field_elems = field;
    p.n_samples = S;

    CK(h->field_a.ensure(field * sizeof(cplx)), "alloc field");
    CK(h->field_b.ensure(field * sizeof(cplx)), "alloc field");
    CK(h->loc_tab.ensure(int64_t(F) * n_tiles * 8 * sizeof(cplx)), "alloc tables");
    CK(h->mul_tab.ensure(int64_t(F) * n_tiles * 8 * sizeof(cplx)), "alloc tables");
    const int64_t k1_elems = pe3d::k1_tab_elems(F, n_tiles);
    const bool k1_table = k1_elems > 0 && !getenv("PE3D_NO_K1_TABLE");    // A/B: in-kernel frequency setup
    if (k1_table) CK(h->k1_tab.ensure(k1_elems * sizeof(cplx)), "alloc tables");
    CK(h->fdev.ensure(F * sizeof(pe3d::FreqDev)), "alloc coeffs");
    CK(h->w_abs.ensure(int64_t(S) * F * sizeof(double)), "alloc w");
    CK(h->err.ensure(sizeof(pe3d::DevError)), "alloc err");
    const bool need_c = p.serial || g->topology != PE3D_PERIODIC;
    if (need_c) {
        CK(h->field_c.ensure(field * sizeof(cplx)), "alloc field");
        CK(h->az_cp.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc az");
        CK(h->az_inv.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc az");
        CK(h->az_q.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc az");
        CK(h->az_ring.ensure(int64_t(F) * 2 * sizeof(cplx)), "alloc az");
        CK(h->fail_row.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(int)), "alloc fail");
        CK(h->fail_mag.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(double)), "alloc fail");
    }

    // per-sample |w(r)| table [S][F]
    std::vector<double> wabs(int64_t(S) * F);
    for (int s = 0; s < S; ++s) {
        const double r = (s == 0) ? g->r_input : g->r_start + (g->first_index + int64_t(s) * g->output_stride) * g->delta_r;
        for (int f = 0; f < F; ++f) wabs[int64_t(s) * F + f] = hankel_abs_host(coeffs[f].k0, r);
    }
    pe3d::DevError de0{NO_ERROR, 0, 0};
    const bool use_graph = !(g->flags & (PE3D_FLAG_NO_GRAPH | PE3D_FLAG_PROFILE)) && g->n_steps >= 2;

    pe3d::LaunchCtx& c = p.ctx;
    c.n_freq = F; c.n_theta = NT; c.n_depth = NZ; c.n_tiles = n_tiles;
    c.sector = g->topology == PE3D_SECTOR;
    c.num_sms = h->num_sms;
    c.delta_theta = g->delta_theta;
    c.fdev = h->fdev.as<pe3d::FreqDev>();
    c.loc_tab = h->loc_tab.as<cplx>();
    c.mul_tab = h->mul_tab.as<cplx>();
    c.k1_tab = k1_table ? h->k1_tab.as<cplx>() : nullptr;
    c.err = h->err.as<pe3d::DevError>();
    c.stream = stream;
    if (!p.serial && g->n_steps > 0) c.split = pe3d::depth_split_plan(c, g->topology == PE3D_PERIODIC);
    if (c.split) {
        CK(h->sp_tot.ensure(int64_t(F) * c.split * NT * 2 * sizeof(cplx)), "alloc split");
        CK(h->sp_aq.ensure(int64_t(F) * n_tiles * 16 * sizeof(cplx)), "alloc split");
        CK(h->sp_pa.ensure(int64_t(F) * c.split * 3 * sizeof(cplx)), "alloc split");
        CK(h->sp_cd.ensure(int64_t(F) * c.split * 2 * NT * sizeof(cplx)), "alloc split");
        c.sp_tot = h->sp_tot.as<cplx>();
        c.sp_aq = h->sp_aq.as<cplx>();
        c.sp_pa = h->sp_pa.as<cplx>();
        c.sp_cd = h->sp_cd.as<cplx>();
    }
    const bool ring_tables = !p.serial && g->topology == PE3D_PERIODIC && g->n_steps > 0;
    if (ring_tables) CK(h->ring_tab.ensure(int64_t(g->n_steps) * F * pe3d::ring_table_elems(NT) * sizeof(cplx)),
                        "alloc ring table");
    // split rings for cluster-sized rings (cfg5): steps whose carries only reach the
    // neighbouring segments' edges run the segmented halo sweep instead of the cluster kernel
    std::vector<int> sr_span;
    if (ring_tables && !getenv("PE3D_NO_SPLIT_RING") && pe3d::sring_segment(NT)) {
        sr_span = sring_spans(g, fd, pe3d::sring_halo_max_span());
        p.sr_span = sr_span.data();
    }

    const cplx* local = reinterpret_cast<const cplx*>(d_local);
    Prof prof{h, (g->flags & PE3D_FLAG_PROFILE) != 0, stream, {}};
    // setup: the depth factorisation (+ per-march sweep tables) and the ring tables
    auto enqueue_depth_setup = [&](pe3d::LaunchCtx& cs) -> cudaError_t {
        return p.serial ? cudaSuccess
                        : prof.run(2, [&] { return pe3d::launch_factor_depth(cs, local, NZ, g->first_index + 1); });
    };
    auto enqueue_ring_setup = [&](pe3d::LaunchCtx& cs) -> cudaError_t {
        if (!ring_tables) return cudaSuccess;
        return prof.run(2, [&] { return pe3d::launch_ring_setup(cs, h->ring_tab.as<cplx>(), g->n_steps,
                                                                g->first_index, g->r_start, g->delta_r); });
    };
    auto enqueue_setup = [&](pe3d::LaunchCtx& cs) -> cudaError_t {
        cudaError_t e = enqueue_depth_setup(cs);
        return e == cudaSuccess ? enqueue_ring_setup(cs) : e;
    };
    // starter: boundary, TL sample 0, first temp (ref marching.py:159-172)
    pe3d::EpilogueArgs ea0{};
    ea0.tl = d_tl;
    ea0.snap = reinterpret_cast<cplx*>(d_snapshots);
    ea0.final_out = g->n_steps == 0 ? reinterpret_cast<cplx*>(d_u_final) : nullptr;
    ea0.clamped = d_clamped;
    ea0.w_abs = h->w_abs.as<double>();
    ea0.n_samples = sink ? sink->R : S;
    ea0.sample = 0;
    ea0.periodic = g->topology == PE3D_PERIODIC;
    ea0.write_temp = g->n_steps > 0;
    ea0.src_column = (g->flags & PE3D_FLAG_STARTER_COLUMN) != 0;
    // a column starter on a periodic ring stays one column through the prologue: the first
    // depth sweep reads it directly (the azimuth-uniform first temp is never written)
    if (ea0.src_column && ea0.periodic && !p.serial && g->n_steps > 0 && pe3d::depth_sweep_takes_column(c)) {
        CK(h->col_tab.ensure(int64_t(F) * n_tiles * 8 * sizeof(cplx)), "alloc column");
        p.temp_col = h->col_tab.as<cplx>();
        ea0.temp_col = p.temp_col;
    }
    if (sink) CK(tl_prepare(h, *sink), "tl streams");
    auto enqueue_prologue = [&]() -> cudaError_t {
        return prof.run(2, [&] { return pe3d::launch_finish(c, reinterpret_cast<const cplx*>(d_u0), 0,
                                                            h->field_a.as<cplx>(), g->r_input, ea0); });
    };

    if (use_graph) {
        // The whole march as two cached graphs (prologue graph, step graph; see the
        // capture below).  Issued from the host, the uploads and the serial setup
        // kernels before the prologue used to cost ~85 us of the march (cfg4,
        // tools/timeline.py).  The page-locked staging feeds the copy fallback for
        // parameter sets too large for one kernel node.
        const size_t fd_b = F * sizeof(pe3d::FreqDev), w_b = wabs.size() * sizeof(double);
        const size_t w_o = (fd_b + 15) & ~size_t(15), e_o = (w_o + w_b + 15) & ~size_t(15);
        CK(h->params_pin.ensure(e_o + sizeof(de0)), "alloc pinned params");
        unsigned char* pin = static_cast<unsigned char*>(h->params_pin.ptr);
        // the previous march on this handle has completed (decode_error synchronises), so
        // nothing reads the staging while it is rewritten
        std::memcpy(pin, fd.data(), fd_b);
        std::memcpy(pin + w_o, wabs.data(), w_b);
        std::memcpy(pin + e_o, &de0, sizeof(de0));
        if (!h->pro_side) CK(cudaStreamCreateWithFlags(&h->pro_side, cudaStreamNonBlocking), "stream");
        if (!h->pro_fork) CK(cudaEventCreateWithFlags(&h->pro_fork, cudaEventDisableTiming), "event");
        if (!h->pro_join) CK(cudaEventCreateWithFlags(&h->pro_join, cudaEventDisableTiming), "event");

        // The graph bakes pointers and scalars into its nodes: reuse the
        // instantiated graph only when every one of them is unchanged.
        std::vector<unsigned char> key;
        auto add = [&](const void* q, size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(q);
            key.insert(key.end(), b, b + n);
        };
        const void* ptrs[10] = {d_local, d_tl, d_snapshots, d_u_final, d_clamped, h->field_a.ptr, h->field_b.ptr,
                                h->field_c.ptr, d_u0, h->params_pin.ptr};
        add(g, sizeof(*g));
        add(coeffs, sizeof(pe3d_coeffs) * F);
        add(ptrs, sizeof(ptrs));
        add(&stream, sizeof(stream));
        const void* tabs[7] = {h->w_abs.ptr, h->fdev.ptr, h->loc_tab.ptr, h->err.ptr, h->ring_tab.ptr, p.ctx.k1_tab,
                               p.temp_col};
        add(tabs, sizeof(tabs));
        if (!sr_span.empty()) add(sr_span.data(), sr_span.size() * sizeof(int));
        const int chains = step_chains(p.ctx, false);
        add(&chains, sizeof(chains));
        // any workspace reallocation (also by other entry points on this handle)
        // may have moved a buffer the graph's kernels address
        const uint64_t gen = h->alloc_generation();
        add(&gen, sizeof(gen));
        add(&p.ctx.split, sizeof(p.ctx.split));
        // the A/B switches pick kernels and launch attributes baked into the graph
        for (const char* name : {"PE3D_NO_PDL", "PE3D_CLUSTER_L", "PE3D_DEPTH_NO_CLUSTER", "PE3D_RING_BLOCK",
                                 "PE3D_RING_CPASYNC", "PE3D_DEPTH_NO_SPLIT", "PE3D_FACTOR_SERIAL",
                                 "PE3D_PREPARE_STAGED", "PE3D_PARAMS_MEMCPY", "PE3D_FINAL_STORES",
                                 "PE3D_FIRST_STEP_FIELD", "PE3D_NO_SPLIT_RING", "PE3D_DEPTH_SMALL_CTA_OFF"}) {
            const char* v = getenv(name);
            const std::string val = v ? std::string("=") + v : std::string("-");
            add(val.data(), val.size() + 1);
        }
        const TlSink none{nullptr, 0, 0, 0, 0};
        add(sink ? sink : &none, sizeof(TlSink));
        int hit = -1;
        for (int i = 0; i < int(h->march_graphs.size()); ++i)
            if (h->march_graphs[i].key == key) hit = i;
        if (hit >= 0) {                                     // most recently used goes last
            Handle::MarchGraph mg = h->march_graphs[hit];
            h->march_graphs.erase(h->march_graphs.begin() + hit);
            h->march_graphs.push_back(mg);
        } else {
            if (int(h->march_graphs.size()) >= Handle::MAX_MARCH_GRAPHS) {
                Handle::MarchGraph& old = h->march_graphs.front();
                if (old.pre) cudaGraphExecDestroy(old.pre);
                if (old.steps) cudaGraphExecDestroy(old.steps);
                h->march_graphs.erase(h->march_graphs.begin());
            }
            Handle::MarchGraph mg;
            auto capture = [&](cudaGraphExec_t* out, auto&& body) -> cudaError_t {
                cudaGraph_t graph = nullptr;
                cudaError_t e = cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal);
                if (e != cudaSuccess) return e;
                e = body();
                const cudaError_t e2 = cudaStreamEndCapture(stream, &graph);
                if (e == cudaSuccess) e = e2;
                if (e == cudaSuccess) e = cudaGraphInstantiate(out, graph, 0);
                if (graph) cudaGraphDestroy(graph);
                if (e == cudaSuccess) e = cudaGraphUpload(*out, stream);    // device-side setup off the first launch
                return e;
            };
            const int64_t before = prof.launches;
            // Two graphs.  The prologue graph: the parameter uploads, then the prologue on
            // the main branch and the setup kernels on a side branch.  A graph submits a
            // second branch only after the main branch's nodes, so with the step loop in the
            // same graph the setup branch started after the whole loop had been submitted
            // (+110 us at 64 frequencies x 20 steps, +390 us at 100 steps, +350 us at 8
            // frequencies x 20 steps on 8 chains; tools/timeline.py).
            cudaError_t e = capture(&mg.pre, [&]() -> cudaError_t {
                // the parameters travel by value in one small kernel node (they are part of the
                // graph key); larger ones as copies from the page-locked staging
                const void* srcs[3] = {fd.data(), wabs.data(), &de0};
                const int sizes[3] = {int(fd_b), int(w_b), int(sizeof(de0))};
                void* dsts[3] = {h->fdev.ptr, h->w_abs.ptr, h->err.ptr};
                cudaError_t e = getenv("PE3D_PARAMS_MEMCPY")
                                    ? cudaErrorNotSupported
                                    : pe3d::launch_params(3, srcs, sizes, dsts, d_clamped, d_clamped ? F : 0, stream);
                if (e == cudaErrorNotSupported) {
                    e = cudaMemcpyAsync(h->fdev.ptr, pin, fd_b, cudaMemcpyHostToDevice, stream);
                    if (e == cudaSuccess) e = cudaMemcpyAsync(h->w_abs.ptr, pin + w_o, w_b, cudaMemcpyHostToDevice, stream);
                    if (e == cudaSuccess) e = cudaMemcpyAsync(h->err.ptr, pin + e_o, sizeof(de0), cudaMemcpyHostToDevice, stream);
                    if (e == cudaSuccess && d_clamped) e = cudaMemsetAsync(d_clamped, 0, F * sizeof(int64_t), stream);
                }
                if (e == cudaSuccess) e = cudaEventRecord(h->pro_fork, stream);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(h->pro_side, h->pro_fork, 0);
                if (e != cudaSuccess) return e;
                // main: prologue, then the ring tables; side: the depth factorisation and the
                // sweep tables (8 frequencies: setup branch 35 -> 22 us)
                cudaError_t ep = enqueue_prologue();
                if (ep == cudaSuccess) ep = enqueue_ring_setup(c);
                pe3d::LaunchCtx cs = c;
                cs.stream = h->pro_side;
                const cudaError_t es = ep == cudaSuccess ? enqueue_depth_setup(cs) : cudaSuccess;
                cudaError_t ej = cudaEventRecord(h->pro_join, h->pro_side);     // always joined: capture ends cleanly
                if (ej == cudaSuccess) ej = cudaStreamWaitEvent(stream, h->pro_join, 0);
                return ep != cudaSuccess ? ep : (es != cudaSuccess ? es : ej);
            });
            if (e == cudaSuccess)
                e = capture(&mg.steps, [&]() -> cudaError_t {
                    return enqueue_steps(h, g, p, local, d_tl, reinterpret_cast<cplx*>(d_snapshots),
                                         reinterpret_cast<cplx*>(d_u_final), d_clamped, h->w_abs.as<double>(), prof,
                                         sink);
                });
            mg.launches = prof.launches - before;
            prof.launches = before;
            if (e != cudaSuccess) {
                if (mg.pre) cudaGraphExecDestroy(mg.pre);
                if (mg.steps) cudaGraphExecDestroy(mg.steps);
                return cuda_fail(err, e, "march graph");
            }
            mg.key = std::move(key);
            h->march_graphs.push_back(mg);
        }
        const Handle::MarchGraph& mg = h->march_graphs.back();
        CK(cudaGraphLaunch(mg.pre, stream), "graph launch");
        CK(cudaGraphLaunch(mg.steps, stream), "graph launch");
        prof.launches += mg.launches;
    } else {
        CK(cudaMemcpyAsync(h->fdev.ptr, fd.data(), F * sizeof(pe3d::FreqDev), cudaMemcpyHostToDevice, stream), "H2D");
        CK(cudaMemcpyAsync(h->w_abs.ptr, wabs.data(), wabs.size() * sizeof(double), cudaMemcpyHostToDevice, stream),
           "H2D");
        CK(cudaMemcpyAsync(h->err.ptr, &de0, sizeof(de0), cudaMemcpyHostToDevice, stream), "H2D");
        if (d_clamped) CK(cudaMemsetAsync(d_clamped, 0, F * sizeof(int64_t), stream), "memset");
        CK(enqueue_setup(c), "setup");
        CK(enqueue_prologue(), "prepare");
        CK(enqueue_steps(h, g, p, local, d_tl, reinterpret_cast<cplx*>(d_snapshots),
                         reinterpret_cast<cplx*>(d_u_final), d_clamped, h->w_abs.as<double>(), prof, sink),
           "enqueue");
    }
    CK(cudaGetLastError(), "launch");
    prof.collect();
    h->last_launches = prof.launches;
    HostFail hf;
    if (!p.serial && g->topology == PE3D_PERIODIC) hf = azimuth_failures(g, coeffs);   // the ring sweep has no pivots
    return decode_error(h, stream, err, &hf);
}

}  // extern "C"

// Host threads that replicate the first azimuth row of TL sample 0 over the other
// azimuths of frequencies [f0, f1) of a [F][S][n_theta][n_depth] stack (streaming
// stores: the rows are written once and read by the caller much later).  Joined by
// join() or the destructor, so every return path of the caller leaves no thread behind.
struct RowReplicator {
    std::vector<std::thread> threads;
    static void fill(double* tl, int f0, int f1, int64_t S, int n_theta, int n_depth, int part, int parts) {
        const int64_t rows = int64_t(f1 - f0) * (n_theta - 1);
        const int64_t r0 = rows * part / parts, r1 = rows * (part + 1) / parts;
        for (int64_t r = r0; r < r1; ++r) {
            const int f = f0 + int(r / (n_theta - 1)), m = 1 + int(r % (n_theta - 1));
            const double* src = tl + int64_t(f) * S * n_theta * n_depth;
            double* dst = tl + (int64_t(f) * S * n_theta + m) * n_depth;
#if defined(__x86_64__)
            int l = 0;
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)
                for (; l + 2 <= n_depth; l += 2) _mm_stream_pd(dst + l, _mm_loadu_pd(src + l));
            for (; l < n_depth; ++l) dst[l] = src[l];
#else
            std::memcpy(dst, src, size_t(n_depth) * sizeof(double));
#endif
        }
#if defined(__x86_64__)
        _mm_sfence();
#endif
    }
    void start(double* tl, int f0, int f1, int64_t S, int n_theta, int n_depth) {
        // two threads per group: measured best at cfg4's 20-step march (1-2 threads 6.6-6.9 ms,
        // 4 threads 6.8-7.6 ms, full copy 7.9-8.1 ms; profiles/r02_ab_tl0_row.txt)
        int parts = std::thread::hardware_concurrency() >= 4 ? 2 : 1;
        if (const char* env = getenv("PE3D_TL0_THREADS")) parts = std::max(1, atoi(env));
        for (int k = 0; k < parts; ++k) {
            try {
                threads.emplace_back(fill, tl, f0, f1, S, n_theta, n_depth, k, parts);
            } catch (...) {                         // no thread to be had: this part on the calling thread
                fill(tl, f0, f1, S, n_theta, n_depth, k, parts);
            }
        }
    }
    void join() {
        for (std::thread& t : threads)
            if (t.joinable()) t.join();
        threads.clear();
    }
    ~RowReplicator() { join(); }
};

// Frequency groups of a pe3d_march_host call (see there): >1 only when the final
// slab's copy to the host (PCIe, modelled at 57 GB/s) would take longer than half
// the march (modelled at 5.5 TB/s of HBM for the 64 B per grid point and step);
// PE3D_HOST_GROUPS=n forces n.
static int host_groups(const pe3d_grid* g, bool has_final, bool has_snapshots) {
    const int F = g->n_freq;
    int G = 1;
    if (const char* env = getenv("PE3D_HOST_GROUPS")) {
        G = atoi(env);
    } else if (has_final && !has_snapshots && g->topology == PE3D_PERIODIC && g->n_steps >= 2) {
        const double points = double(F) * g->n_theta * g->n_depth;
        const double t_copy = points * 16 / 57e9, t_march = points * 64 * g->n_steps / 5.5e12;
        if (t_copy > 0.5 * t_march) G = 4;
    }
    if (has_snapshots) G = 1;                   // snapshots leave after the march
    G = std::min(G, F / 2);                     // at least two frequencies per group
    return G < 1 ? 1 : G;
}

// Propagate a non-singular failure of one group unchanged.
static int cuda_or(pe3d_error* err, int st, const pe3d_error& e) {
    if (err) *err = e;
    return st;
}

extern "C" {

int pe3d_march_host(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_c128* local,
                    const pe3d_c128* u0, pe3d_c128* u_final, double* tl, pe3d_c128* snapshots, int64_t* clamped,
                    pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return bad_arg(err, "null handle");
    int st = check_grid(g, coeffs, err);
    if (st != PE3D_OK) return st;
    if (!local || !u0) return bad_arg(err, "null local or u0");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    const int64_t F = g->n_freq, slab = int64_t(g->n_theta) * g->n_depth;
    const int64_t S = pe3d_sample_count(g->n_steps, g->output_stride);
    const int64_t u0_elems = F * ((g->flags & PE3D_FLAG_STARTER_COLUMN) ? g->n_depth : slab);
    cudaStream_t s = h->stream;
    CK(h->h_local.ensure(F * g->n_depth * sizeof(cplx)), "alloc");
    CK(h->h_u0.ensure(u0_elems * sizeof(cplx)), "alloc");
    CK(h->h_clamped.ensure(F * sizeof(int64_t)), "alloc");
    if (u_final) CK(h->h_final.ensure(F * slab * sizeof(cplx)), "alloc");
    // A page-locked TL stack (and no snapshots): stream the samples out while
    // the march runs, through a device ring of a few samples per frequency.
    TlSink sink{nullptr, 0, 0, 0, 0};
    if (tl && !snapshots && !getenv("PE3D_NO_TL_STREAM")) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, tl) == cudaSuccess && pa.type == cudaMemoryTypeHost)
            sink = TlSink{tl, int(S), int(S < 4 ? S : 4), 0, 0};
        cudaGetLastError();                                  // pageable memory: not an error
    }
    if (tl) CK(h->h_tl.ensure(F * (sink.host ? sink.R : S) * slab * sizeof(double)), "alloc");
    if (snapshots) CK(h->h_snap.ensure(F * S * slab * sizeof(cplx)), "alloc");
    CK(cudaMemcpyAsync(h->h_local.ptr, local, F * g->n_depth * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_u0.ptr, u0, u0_elems * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    // Short marches with a final slab are bound by its device-to-host copy (PCIe,
    // ~57 GB/s: 4.7 ms for cfg4's 268 MB against a 3.8 ms 20-step march).  Then the
    // frequencies are marched in groups, one after another, and each group's final
    // slab leaves on a copy stream while the next group marches.
    const int G = host_groups(g, u_final != nullptr, snapshots != nullptr);
    if (u_final) {                                          // every march's final slab leaves on the copy stream
        if (!h->copy_stream) CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking), "stream");
        if (!h->copy_ev) CK(cudaEventCreateWithFlags(&h->copy_ev, cudaEventDisableTiming), "event");
    }
    const int64_t u0_per = (g->flags & PE3D_FLAG_STARTER_COLUMN) ? g->n_depth : slab;
    const int64_t tl_per = (sink.host ? sink.R : S) * slab;
    // A copy-bound march (G > 1) of column starters on a periodic ring: the starting TL sample is
    // the same for every azimuth, so only its first azimuth row crosses PCIe (cfg4: 0.5 MB instead
    // of 134 MB of the 402 MB a 20-step march sends) and host threads replicate it while the later
    // groups march and the final slabs leave.
    if (sink.host && G > 1 && (g->flags & PE3D_FLAG_STARTER_COLUMN) && g->topology == PE3D_PERIODIC &&
        g->n_theta > 1 && !getenv("PE3D_TL0_FULL"))
        sink.col0 = 1;
    h->last_h2d_bytes = (F * g->n_depth + u0_elems) * int64_t(sizeof(cplx));
    h->last_d2h_bytes = (u_final ? F * slab * int64_t(sizeof(cplx)) : 0) + (clamped ? F * int64_t(sizeof(int64_t)) : 0) +
                        (snapshots ? F * S * slab * int64_t(sizeof(cplx)) : 0) +
                        (tl ? F * ((S - (sink.col0 ? 1 : 0)) * slab + (sink.col0 ? g->n_depth : 0)) * int64_t(sizeof(double)) : 0);
    RowReplicator rep;
    pe3d_error best{};
    int best_st = PE3D_OK;
    // (equal groups: a shorter first group, to start the copies earlier, was measured slower --
    // an 8-frequency march costs 92 us per frequency against 66 us in a group of 16-19)
    for (int gi = 0; gi < G; ++gi) {
        const int f0 = int(F * gi / G), f1 = int(F * (gi + 1) / G);
        pe3d_grid gg = *g;
        gg.n_freq = f1 - f0;
        TlSink sk = sink;
        if (sk.host) sk.host = tl + int64_t(f0) * S * slab;
        pe3d_error e_g{};
        if (u_final)                                        // this group's slab leaves while the next marches
            h->post_copy = Handle::PostCopy{u_final + f0 * slab, h->h_final.as<cplx>() + f0 * slab,
                                            size_t(f1 - f0) * slab * sizeof(cplx)};
        const int st_g =
            march_device_impl(handle, &gg, coeffs + f0, h->h_local.as<pe3d_c128>() + int64_t(f0) * g->n_depth,
                              h->h_u0.as<pe3d_c128>() + f0 * u0_per,
                              u_final ? h->h_final.as<pe3d_c128>() + f0 * slab : nullptr,
                              tl ? h->h_tl.as<double>() + f0 * tl_per : nullptr,
                              snapshots ? h->h_snap.as<pe3d_c128>() : nullptr, h->h_clamped.as<int64_t>() + f0, s,
                              &e_g, sk.host ? &sk : nullptr);
        h->post_copy = Handle::PostCopy{};                  // (a march that failed before its launch left it set)
        if (st_g != PE3D_OK) {
            // the batch reports the lowest (step, sweep, frequency, member), as one march would
            if (st_g != PE3D_SINGULAR) {
                if (u_final) cudaStreamSynchronize(h->copy_stream);    // no copy in flight into the caller's buffers
                return cuda_or(err, st_g, e_g);
            }
            e_g.frequency += f0;
            const bool lower = best_st == PE3D_OK ||
                               std::make_tuple(e_g.range_index, e_g.sweep, e_g.frequency, e_g.member) <
                                   std::make_tuple(best.range_index, best.sweep, best.frequency, best.member);
            if (lower) { best = e_g; best_st = st_g; }
            continue;
        }
        if (sink.col0) rep.start(tl, f0, f1, S, g->n_theta, g->n_depth);   // the march synchronised: row 0 is there
    }
    if (u_final) CK(cudaStreamSynchronize(h->copy_stream), "sync");
    rep.join();
    if (best_st != PE3D_OK) {
        if (err) *err = best;
        return best_st;
    }
    if (tl && !sink.host)
        CK(cudaMemcpyAsync(tl, h->h_tl.ptr, F * S * slab * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    if (snapshots)
        CK(cudaMemcpyAsync(snapshots, h->h_snap.ptr, F * S * slab * sizeof(cplx), cudaMemcpyDeviceToHost, s), "D2H");
    if (clamped) CK(cudaMemcpyAsync(clamped, h->h_clamped.ptr, F * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "sync");
    return PE3D_OK;
}

int pe3d_step_general_host(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_c128* local_now,
                           const pe3d_c128* local_new, const pe3d_c128* u_in, pe3d_c128* u_out, double* tl_out,
                           int64_t* clamped, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return bad_arg(err, "null handle");
    int st = check_grid(g, coeffs, err);
    if (st != PE3D_OK) return st;
    if (g->n_steps != 1) return bad_arg(err, "n_steps == 1 for a single step");
    if (!local_now || !local_new || !u_in || !u_out) return bad_arg(err, "null buffer");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    cudaStream_t s = h->stream;
    const int F = g->n_freq, NT = g->n_theta, NZ = g->n_depth, n_tiles = (NZ + 7) / 8;
    const int64_t slab = int64_t(NT) * NZ, field = int64_t(F) * n_tiles * NT * 8;
    std::vector<pe3d::FreqDev> fd = freq_table(g, coeffs);
    CK(h->field_a.ensure(field * sizeof(cplx)), "alloc");
    CK(h->field_b.ensure(field * sizeof(cplx)), "alloc");
    CK(h->field_c.ensure(field * sizeof(cplx)), "alloc");
    CK(h->fdev.ensure(F * sizeof(pe3d::FreqDev)), "alloc");
    CK(h->err.ensure(sizeof(pe3d::DevError)), "alloc");
    CK(h->w_abs.ensure(F * sizeof(double)), "alloc");
    CK(h->az_cp.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_inv.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_q.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_ring.ensure(int64_t(F) * 2 * sizeof(cplx)), "alloc");
    CK(h->fail_row.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(int)), "alloc");
    CK(h->fail_mag.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(double)), "alloc");
    CK(h->h_local.ensure(F * slab * sizeof(cplx)), "alloc");
    CK(h->h_local2.ensure(F * slab * sizeof(cplx)), "alloc");
    CK(h->h_u0.ensure(F * slab * sizeof(cplx)), "alloc");
    CK(h->h_final.ensure(F * slab * sizeof(cplx)), "alloc");
    CK(h->h_tl.ensure(F * slab * sizeof(double)), "alloc");
    CK(h->h_clamped.ensure(F * sizeof(int64_t)), "alloc");
    pe3d::DevError de0{NO_ERROR, 0, 0};
    const int j_new = g->first_index + 1;
    const double r_new = g->r_start + j_new * g->delta_r;
    std::vector<double> wabs(F);
    for (int f = 0; f < F; ++f) wabs[f] = hankel_abs_host(coeffs[f].k0, r_new);
    CK(cudaMemcpyAsync(h->w_abs.ptr, wabs.data(), F * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemsetAsync(h->h_clamped.ptr, 0, F * sizeof(int64_t), s), "memset");
    CK(cudaMemcpyAsync(h->fdev.ptr, fd.data(), F * sizeof(pe3d::FreqDev), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->err.ptr, &de0, sizeof(de0), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_local.ptr, local_now, F * slab * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_local2.ptr, local_new, F * slab * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_u0.ptr, u_in, F * slab * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");

    pe3d::LaunchCtx c{};
    c.n_freq = F; c.n_theta = NT; c.n_depth = NZ; c.n_tiles = n_tiles;
    c.sector = g->topology == PE3D_SECTOR;
    c.num_sms = h->num_sms;
    c.delta_theta = g->delta_theta;
    c.fdev = h->fdev.as<pe3d::FreqDev>();
    c.err = h->err.as<pe3d::DevError>();
    c.stream = s;
    pe3d::EpilogueArgs ea{};
    ea.periodic = g->topology == PE3D_PERIODIC;
    ea.write_temp = 1;
    ea.w_abs = h->w_abs.as<double>();
    CK(pe3d::launch_finish(c, h->h_u0.as<cplx>(), 0, h->field_a.as<cplx>(), g->r_input, ea), "prepare");
    CK(pe3d::launch_depth_serial(c, h->field_a.as<cplx>(), h->field_b.as<cplx>(), h->field_c.as<cplx>(),
                                 h->h_local.as<cplx>(), h->h_local2.as<cplx>(), slab, NZ, 1, h->fail_row.as<int>(),
                                 h->fail_mag.as<double>()),
       "depth");
    CK(pe3d::launch_reduce_failures(h->fail_row.as<int>(), h->fail_mag.as<double>(), F, NT, j_new, 0, -1, c.err, s),
       "reduce");
    pe3d::EpilogueArgs ef{};
    ef.periodic = ea.periodic;
    ef.final_out = h->h_final.as<cplx>();
    ef.w_abs = h->w_abs.as<double>();
    ef.tl = tl_out ? h->h_tl.as<double>() : nullptr;
    ef.clamped = h->h_clamped.as<int64_t>();
    ef.n_samples = 1;
    ef.write_temp = 0;
    CK(pe3d::launch_azimuth_serial(c, h->field_b.as<cplx>(), h->field_c.as<cplx>(), h->az_cp.as<cplx>(),
                                   h->az_inv.as<cplx>(), h->az_q.as<cplx>(), h->az_ring.as<cplx>(), r_new, j_new),
       "azimuth");
    CK(pe3d::launch_finish(c, h->field_c.as<cplx>(), 1, h->field_a.as<cplx>(), r_new, ef), "finish");
    st = decode_error(h, s, err);
    if (st != PE3D_OK) return st;
    CK(cudaMemcpyAsync(u_out, h->h_final.ptr, F * slab * sizeof(cplx), cudaMemcpyDeviceToHost, s), "D2H");
    if (tl_out) CK(cudaMemcpyAsync(tl_out, h->h_tl.ptr, F * slab * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    if (clamped) CK(cudaMemcpyAsync(clamped, h->h_clamped.ptr, F * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "sync");
    return PE3D_OK;
}

int pe3d_solve_batch_host(void* handle, int32_t n, int32_t members, int32_t cyclic, pe3d_strided sub,
                          pe3d_strided main_diag, pe3d_strided sup, pe3d_strided rhs, pe3d_c128* x, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return bad_arg(err, "null handle");
    if (members < 1) return bad_arg(err, "batch nonempty");
    if (n < 1 || (cyclic && n < 3)) return bad_arg(err, cyclic ? "n >= 3 for cyclic systems" : "n >= 1");
    if (!sub.ptr || !main_diag.ptr || !sup.ptr || !rhs.ptr || !x) return bad_arg(err, "null buffer");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    cudaStream_t s = h->stream;
    const int n_off = cyclic ? n : n - 1;
    // Copy the four operands into one device buffer; each keeps its strides.
    auto extent = [&](const pe3d_strided& a, int rows) -> int64_t {
        if (rows <= 0) return 1;
        return (rows - 1) * a.row_stride + int64_t(members - 1) * a.member_stride + 1;
    };
    const int64_t e_sub = extent(sub, n_off), e_main = extent(main_diag, n), e_sup = extent(sup, n_off),
                  e_rhs = extent(rhs, n);
    const int64_t total = e_sub + e_main + e_sup + e_rhs;
    CK(h->sb_in.ensure(total * sizeof(cplx)), "alloc");
    CK(h->sb_x.ensure(int64_t(members) * n * sizeof(cplx)), "alloc");
    for (DevBuf* b : {&h->sb_cp, &h->sb_inv, &h->sb_y, &h->sb_q}) CK(b->ensure(int64_t(members) * n * sizeof(cplx)), "alloc");
    CK(h->fail_row.ensure(int64_t(members) * sizeof(int)), "alloc");
    CK(h->fail_mag.ensure(int64_t(members) * sizeof(double)), "alloc");
    CK(h->err.ensure(sizeof(pe3d::DevError)), "alloc");
    cplx* base = h->sb_in.as<cplx>();
    int64_t off = 0;
    pe3d::StridedC dsub, dmain, dsup, drhs;
    auto put = [&](const pe3d_strided& a, int64_t ext, pe3d::StridedC& d) -> cudaError_t {
        d.ptr = base + off;
        d.row_stride = a.row_stride;
        d.member_stride = a.member_stride;
        cudaError_t e = cudaMemcpyAsync(base + off, a.ptr, ext * sizeof(cplx), cudaMemcpyHostToDevice, s);
        off += ext;
        return e;
    };
    CK(put(sub, e_sub, dsub), "H2D");
    CK(put(main_diag, e_main, dmain), "H2D");
    CK(put(sup, e_sup, dsup), "H2D");
    CK(put(rhs, e_rhs, drhs), "H2D");
    pe3d::DevError de0{NO_ERROR, 0, 0};
    CK(cudaMemcpyAsync(h->err.ptr, &de0, sizeof(de0), cudaMemcpyHostToDevice, s), "H2D");
    CK(pe3d::launch_solve_batch(n, members, cyclic, dsub, dmain, dsup, drhs, h->sb_x.as<cplx>(), h->sb_cp.as<cplx>(),
                                h->sb_inv.as<cplx>(), h->sb_y.as<cplx>(), h->sb_q.as<cplx>(), h->fail_row.as<int>(),
                                h->fail_mag.as<double>(), s),
       "solve");
    CK(pe3d::launch_reduce_failures(h->fail_row.as<int>(), h->fail_mag.as<double>(), 1, members, 0, 0, n,
                                    h->err.as<pe3d::DevError>(), s),
       "reduce");

    int st = decode_error(h, s, err);
    if (st != PE3D_OK) {
        if (err) err->range_index = -1;
        if (err && err->rank1) std::snprintf(err->message, sizeof(err->message),
                                             "singular system: pivot %d, batch member %d (singular rank-1 correction)",
                                             err->pivot, err->member);
        return st;
    }
    CK(cudaMemcpyAsync(x, h->sb_x.ptr, int64_t(members) * n * sizeof(cplx), cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "sync");
    return PE3D_OK;
}

int pe3d_march_medium_host(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, const pe3d_medium* md,
                           const pe3d_c128* u0, pe3d_c128* u_final, double* tl, pe3d_c128* snapshots,
                           int64_t* clamped, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return bad_arg(err, "null handle");
    int st = check_grid(g, coeffs, err);
    if (st != PE3D_OK) return st;
    if (!md || !u0 || md->n_profile < 1 || !md->profile_z || !md->profile_c) return bad_arg(err, "medium / u0");
    if (!(md->interface_width > 0)) return bad_arg(err, "interface_width > 0");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    cudaStream_t s = h->stream;
    const int F = g->n_freq, NT = g->n_theta, NZ = g->n_depth, n_tiles = (NZ + 7) / 8;
    const int64_t slab = int64_t(NT) * NZ, field = int64_t(F) * n_tiles * NT * 8;
    const int S = pe3d_sample_count(g->n_steps, g->output_stride);
    std::vector<pe3d::FreqDev> fd = freq_table(g, coeffs);
    for (DevBuf* b : {&h->field_a, &h->field_b, &h->field_c}) CK(b->ensure(field * sizeof(cplx)), "alloc");
    CK(h->fdev.ensure(F * sizeof(pe3d::FreqDev)), "alloc");
    CK(h->err.ensure(sizeof(pe3d::DevError)), "alloc");
    CK(h->w_abs.ensure(int64_t(S) * F * sizeof(double)), "alloc");
    CK(h->az_cp.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_inv.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_q.ensure(int64_t(F) * NT * sizeof(cplx)), "alloc");
    CK(h->az_ring.ensure(int64_t(F) * 2 * sizeof(cplx)), "alloc");
    CK(h->fail_row.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(int)), "alloc");
    CK(h->fail_mag.ensure(int64_t(F) * (NT > NZ ? NT : NZ) * sizeof(double)), "alloc");
    CK(h->med_local.ensure(2 * field * sizeof(cplx)), "alloc");      // >= 2 slabs; tile layout for the scan path
    CK(h->med_prof.ensure(2 * md->n_profile * sizeof(double)), "alloc");
    const int64_t n_lat = md->lattice ? int64_t(md->lat_nx) * md->lat_ny * md->lat_nz : 0;
    if (n_lat) CK(h->med_lat.ensure(n_lat * sizeof(double)), "alloc");
    const int64_t u0_elems = F * ((g->flags & PE3D_FLAG_STARTER_COLUMN) ? NZ : slab);
    CK(h->h_u0.ensure(u0_elems * sizeof(cplx)), "alloc");
    CK(h->h_clamped.ensure(F * sizeof(int64_t)), "alloc");
    if (u_final) CK(h->h_final.ensure(F * slab * sizeof(cplx)), "alloc");
    if (tl) CK(h->h_tl.ensure(int64_t(F) * S * slab * sizeof(double)), "alloc");
    if (snapshots) CK(h->h_snap.ensure(int64_t(F) * S * slab * sizeof(cplx)), "alloc");

    std::vector<double> wabs(int64_t(S) * F);
    for (int k = 0; k < S; ++k) {
        const double r = (k == 0) ? g->r_input : g->r_start + (g->first_index + int64_t(k) * g->output_stride) * g->delta_r;
        for (int f = 0; f < F; ++f) wabs[int64_t(k) * F + f] = hankel_abs_host(coeffs[f].k0, r);
    }
    pe3d::DevError de0{NO_ERROR, 0, 0};
    CK(cudaMemcpyAsync(h->fdev.ptr, fd.data(), F * sizeof(pe3d::FreqDev), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->w_abs.ptr, wabs.data(), wabs.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->err.ptr, &de0, sizeof(de0), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->med_prof.ptr, md->profile_z, md->n_profile * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->med_prof.as<double>() + md->n_profile, md->profile_c, md->n_profile * sizeof(double),
                       cudaMemcpyHostToDevice, s), "H2D");
    if (n_lat) CK(cudaMemcpyAsync(h->med_lat.ptr, md->lattice, n_lat * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_u0.ptr, u0, u0_elems * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemsetAsync(h->h_clamped.ptr, 0, F * sizeof(int64_t), s), "memset");
    cudaStreamSynchronize(s);   // host staging (vectors) must outlive the copies

    pe3d::MediumDev M{};
    M.c0 = md->c0;
    M.n_prof = md->n_profile;
    M.pz = h->med_prof.as<double>();
    M.pc = h->med_prof.as<double>() + md->n_profile;
    M.rho_w = md->water_density;
    M.alpha_w = md->water_alpha;
    M.c_b = md->bottom_speed;
    M.rho_b = md->bottom_density;
    M.alpha_b = md->bottom_alpha;
    M.h0 = md->bathy_depth0;
    M.tan_slope = std::tan(md->bathy_slope_deg * 3.141592653589793 / 180.0);
    M.hmin = md->bathy_min_depth;
    M.sponge_n = md->sponge_points;
    M.sponge_max = md->sponge_max_alpha;
    M.w = md->interface_width;
    M.lat = n_lat ? h->med_lat.as<double>() : nullptr;
    M.nx = md->lat_nx; M.ny = md->lat_ny; M.nz = md->lat_nz;
    M.ext_h = md->lat_extent_h; M.dh = md->lat_spacing_h; M.dv = md->lat_spacing_v;
    M.eta = 1.0 / (40.0 * 3.141592653589793 * std::log10(std::exp(1.0)));

    pe3d::LaunchCtx c{};
    c.n_freq = F; c.n_theta = NT; c.n_depth = NZ; c.n_tiles = n_tiles;
    c.sector = g->topology == PE3D_SECTOR;
    c.num_sms = h->num_sms;
    c.delta_theta = g->delta_theta;
    c.fdev = h->fdev.as<pe3d::FreqDev>();
    c.err = h->err.as<pe3d::DevError>();
    c.stream = s;
    cplx* L[2] = {h->med_local.as<cplx>(), h->med_local.as<cplx>() + field};
    cplx* A = h->field_a.as<cplx>();
    cplx* B = h->field_b.as<cplx>();
    cplx* Cc = h->field_c.as<cplx>();
    const bool periodic = g->topology == PE3D_PERIODIC;
    cplx* d_final = u_final ? h->h_final.as<cplx>() : nullptr;
    double* d_tl = tl ? h->h_tl.as<double>() : nullptr;
    cplx* d_snap = snapshots ? h->h_snap.as<cplx>() : nullptr;
    int64_t* d_cl = h->h_clamped.as<int64_t>();
    if (periodic && g->n_steps > 0) {
        const int64_t E = pe3d::ring_table_elems(NT);
        CK(h->ring_tab.ensure(int64_t(g->n_steps) * F * E * sizeof(cplx)), "alloc ring table");
        CK(pe3d::launch_ring_setup(c, h->ring_tab.as<cplx>(), g->n_steps, g->first_index, g->r_start, g->delta_r),
           "ring setup");
    }
    // starter: local term at the input range, boundary, TL sample 0, first temp
    const bool scan_path = !(g->flags & PE3D_FLAG_SERIAL) && n_tiles <= 512;
    if (scan_path) CK(pe3d::launch_medium_local_tiles(c, M, L[0], g->delta_z, g->r_input), "medium");
    else CK(pe3d::launch_medium_local(c, M, L[0], g->delta_z, g->r_input), "medium");
    pe3d::EpilogueArgs ea0{};
    ea0.tl = d_tl;
    ea0.snap = d_snap;
    ea0.final_out = g->n_steps == 0 ? d_final : nullptr;
    ea0.clamped = d_cl;
    ea0.w_abs = h->w_abs.as<double>();
    ea0.n_samples = S;
    ea0.sample = 0;
    ea0.periodic = periodic;
    ea0.write_temp = g->n_steps > 0;
    ea0.src_column = (g->flags & PE3D_FLAG_STARTER_COLUMN) != 0;
    CK(pe3d::launch_finish(c, h->h_u0.as<cplx>(), 0, A, g->r_input, ea0), "prepare");
    const int64_t E = periodic ? pe3d::ring_table_elems(NT) : 0;
    // The step loop.  Scan path: the medium at r_(j+1) is evaluated on the
    // whole grid by a wide kernel on a side stream, one step ahead, so it
    // overlaps the previous step's azimuth sweep; the per-column scan reads
    // it (that kernel has one small CTA per column and is latency bound).
    const bool pre = scan_path;
    if (pre) {
        if (!h->chain_stream[0]) CK(cudaStreamCreateWithFlags(&h->chain_stream[0], cudaStreamNonBlocking), "stream");
        for (int k = 0; k < 2; ++k)
            if (!h->chain_join[k]) CK(cudaEventCreateWithFlags(&h->chain_join[k], cudaEventDisableTiming), "event");
        if (!h->chain_fork) CK(cudaEventCreateWithFlags(&h->chain_fork, cudaEventDisableTiming), "event");
    }
    cudaStream_t sd = h->chain_stream[0];
    cudaEvent_t ev_med = h->chain_join[0], ev_scan = h->chain_join[1];
    auto step_loop = [&]() -> cudaError_t {
        cudaError_t e = cudaSuccess;
        if (pre && g->n_steps > 0) {                    // medium of step 0, on the side stream
            e = cudaEventRecord(h->chain_fork, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, h->chain_fork, 0);
            if (e == cudaSuccess) {
                pe3d::LaunchCtx cs = c;
                cs.stream = sd;
                e = pe3d::launch_medium_local_tiles(cs, M, L[1], g->delta_z,
                                                    g->r_start + (g->first_index + 1) * g->delta_r);
            }
            if (e == cudaSuccess) e = cudaEventRecord(ev_med, sd);
        }
        for (int k = 0; k < g->n_steps && e == cudaSuccess; ++k) {
            const int j_new = g->first_index + k + 1;
            const double r_new = g->r_start + j_new * g->delta_r;
            cplx* now = L[k & 1];
            cplx* nxt = L[(k + 1) & 1];
            if (scan_path) {
                if (pre) e = cudaStreamWaitEvent(s, ev_med, 0);
                if (e == cudaSuccess)
                    e = pe3d::launch_depth_medium_scan(c, M, A, B, now, nxt, g->delta_z, r_new, h->fail_row.as<int>(),
                                                       h->fail_mag.as<double>(), pre ? 1 : 0);
                if (pre && e == cudaSuccess) {          // medium of step k+1 into `now`, once the scan read it
                    e = cudaEventRecord(ev_scan, s);
                    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev_scan, 0);
                    if (e == cudaSuccess && k + 1 < g->n_steps) {
                        pe3d::LaunchCtx cs = c;
                        cs.stream = sd;
                        e = pe3d::launch_medium_local_tiles(cs, M, now, g->delta_z, r_new + g->delta_r);
                    }
                    if (e == cudaSuccess) e = cudaEventRecord(ev_med, sd);
                }
            } else {
                e = pe3d::launch_medium_local(c, M, nxt, g->delta_z, r_new);
                if (e == cudaSuccess)
                    e = pe3d::launch_depth_serial(c, A, B, Cc, now, nxt, int64_t(NZ) * NT, 1, NT, h->fail_row.as<int>(),
                                                  h->fail_mag.as<double>());
            }
            if (e == cudaSuccess)
                e = pe3d::launch_reduce_failures(h->fail_row.as<int>(), h->fail_mag.as<double>(), F, NT, j_new, 0, -1,
                                                 c.err, s);
            if (e != cudaSuccess) break;
            pe3d::EpilogueArgs ea{};
            const bool record = ((k + 1) % g->output_stride) == 0;
            ea.tl = record ? d_tl : nullptr;
            ea.snap = record ? d_snap : nullptr;
            ea.final_out = (k == g->n_steps - 1) ? d_final : nullptr;
            ea.clamped = d_cl;
            ea.n_samples = S;
            ea.sample = (k + 1) / g->output_stride;
            ea.w_abs = h->w_abs.as<double>() + int64_t(ea.sample) * F;
            ea.periodic = periodic;
            ea.write_temp = (k < g->n_steps - 1);
            if (periodic) {
                e = pe3d::launch_azimuth_scan(c, B, A, h->ring_tab.as<cplx>() + int64_t(k) * F * E, r_new, ea);
            } else {
                e = pe3d::launch_azimuth_serial(c, B, Cc, h->az_cp.as<cplx>(), h->az_inv.as<cplx>(),
                                                h->az_q.as<cplx>(), h->az_ring.as<cplx>(), r_new, j_new);
                if (e == cudaSuccess) e = pe3d::launch_finish(c, Cc, 1, A, r_new, ea);
            }
        }
        if (pre && g->n_steps > 0) {                    // join the side stream (always, for a clean capture)
            cudaError_t e2 = cudaStreamWaitEvent(s, ev_med, 0);
            if (e == cudaSuccess) e = e2;
        }
        return e;
    };
    if (!(g->flags & PE3D_FLAG_NO_GRAPH) && g->n_steps >= 2) {
        // one CUDA graph for the step loop (the side stream included), reused
        // while every baked-in argument repeats (the handle's graph cache)
        std::vector<unsigned char> key;
        auto add = [&](const void* q, size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(q);
            key.insert(key.end(), b, b + n);
        };
        const char tag[] = "medium";
        add(tag, sizeof(tag));
        add(g, sizeof(*g));
        add(coeffs, sizeof(pe3d_coeffs) * F);
        add(&M, sizeof(M));
        const void* ptrs[12] = {A, B, Cc, L[0], L[1], d_tl, d_snap, d_final, d_cl, h->ring_tab.ptr, h->w_abs.ptr,
                                h->fail_row.ptr};
        add(ptrs, sizeof(ptrs));
        add(&s, sizeof(s));
        const int flags2[2] = {pre ? 1 : 0, scan_path ? 1 : 0};
        add(flags2, sizeof(flags2));
        const uint64_t gen = h->alloc_generation();        // fdev, err, az_*, fail_mag ... not moved since capture
        add(&gen, sizeof(gen));
        if (!(h->graph_exec && key == h->graph_key)) {
            if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
            h->graph_exec = nullptr;
            h->graph_key.clear();
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
            cudaError_t e = step_loop();
            cudaError_t e2 = cudaStreamEndCapture(s, &graph);
            if (e != cudaSuccess) { if (graph) cudaGraphDestroy(graph); return cuda_fail(err, e, "enqueue"); }
            if (e2 != cudaSuccess) return cuda_fail(err, e2, "end capture");
            e = cudaGraphInstantiate(&h->graph_exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) { h->graph_exec = nullptr; return cuda_fail(err, e, "instantiate"); }
            h->graph_key = key;
        }
        CK(cudaGraphLaunch(h->graph_exec, s), "graph launch");
    } else {
        CK(step_loop(), "enqueue");
    }
    HostFail hf;
    if (periodic) hf = azimuth_failures(g, coeffs);          // the ring sweep has no pivots
    st = decode_error(h, s, err, &hf);
    if (st != PE3D_OK) return st;
    if (u_final) CK(cudaMemcpyAsync(u_final, h->h_final.ptr, F * slab * sizeof(cplx), cudaMemcpyDeviceToHost, s), "D2H");
    if (tl) CK(cudaMemcpyAsync(tl, h->h_tl.ptr, int64_t(F) * S * slab * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    if (snapshots)
        CK(cudaMemcpyAsync(snapshots, h->h_snap.ptr, int64_t(F) * S * slab * sizeof(cplx), cudaMemcpyDeviceToHost, s),
           "D2H");
    if (clamped) CK(cudaMemcpyAsync(clamped, h->h_clamped.ptr, F * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "sync");
    return PE3D_OK;
}

// NCCL is loaded lazily (only the slab march needs it), so the library has
// no link-time dependency on a particular libnccl.
int pe3d_last_copy_bytes(void* handle, int64_t* h2d, int64_t* d2h) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return PE3D_BAD_ARGUMENT;
    if (h2d) *h2d = h->last_h2d_bytes;
    if (d2h) *d2h = h->last_d2h_bytes;
    return PE3D_OK;
}

int pe3d_last_launches(void* handle, int64_t* launches) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h || !launches) return PE3D_BAD_ARGUMENT;
    *launches = h->last_launches;
    return PE3D_OK;
}

int pe3d_profile_launches(void* handle, int32_t cls, double* ms, int32_t capacity, int32_t* count) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h || cls < 0 || cls > 3 || capacity < 0) return PE3D_BAD_ARGUMENT;
    const std::vector<double>& v = h->prof_list[cls];
    if (count) *count = int32_t(v.size());
    for (int32_t i = 0; ms && i < capacity && i < int32_t(v.size()); ++i) ms[i] = v[i];
    return PE3D_OK;
}

int pe3d_host_alloc(uint64_t bytes, void** ptr) {
    if (!ptr) return PE3D_BAD_ARGUMENT;
    *ptr = nullptr;
    if (bytes == 0) return PE3D_OK;
    return cudaHostAlloc(ptr, size_t(bytes), cudaHostAllocDefault) == cudaSuccess ? PE3D_OK : PE3D_CUDA_ERROR;
}

int pe3d_host_free(void* ptr) {
    if (!ptr) return PE3D_OK;
    return cudaFreeHost(ptr) == cudaSuccess ? PE3D_OK : PE3D_CUDA_ERROR;
}

int pe3d_profile_last(void* handle, double* ms, int32_t* launches) {
    Handle* h = static_cast<Handle*>(handle);
    if (!h) return PE3D_BAD_ARGUMENT;
    for (int k = 0; k < 3; ++k) {
        if (ms) ms[k] = h->prof_ms[k];
        if (launches) launches[k] = h->prof_n[k];
    }
    return PE3D_OK;
}

}  // extern "C"
