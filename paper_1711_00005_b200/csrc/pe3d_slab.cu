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

#include <dlfcn.h>
#include <nccl.h>

#include "pe3d_device.cuh"
#include "pe3d_host.h"
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

// Bounded: after timeout_ns without the peers' signals (a failed rank) the
// wait gives up, marks the march aborted in the error record (decoded as
// PE3D_CUDA_ERROR) and every later wait of the march returns at once, so no
// rank's stream can hang on a peer that will never signal.
__global__ void k_slab_wait(const unsigned long long* flag, unsigned long long target, DevError* err,
                            unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    if (*reinterpret_cast<volatile int32_t*>(&err->aborted)) return;
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flag) : "memory");
        if (v >= target) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
            atomicExch(&err->aborted, 1);
            return;
        }
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

// PE3D_SLAB_TIMEOUT_MS bounds every cross-rank wait (default 20 s)
cudaError_t launch_slab_wait(const unsigned long long* flag, unsigned long long target, DevError* err,
                             cudaStream_t s) {
    const char* env = getenv("PE3D_SLAB_TIMEOUT_MS");
    const unsigned long long ms = env ? strtoull(env, nullptr, 10) : 20000ull;
    k_slab_wait<<<1, 32, 0, s>>>(flag, target, err, ms * 1000000ull);
    return cudaGetLastError();
}

}  // namespace pe3d

// ------------------------------------------------------------------ host side
// The slab-decomposed march (pe3d_march_slab, pe3d_slab_p2p_export,
// pe3d_march_slab_p2p): buffers, transports and the step loop.

using pe3d::cplx;
using namespace pe3d_host;

namespace {

struct Nccl {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

static Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (lib) {
            n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
            n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(lib, "ncclCommInitRank"));
            n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(lib, "ncclCommDestroy"));
            n.send = reinterpret_cast<decltype(n.send)>(dlsym(lib, "ncclSend"));
            n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(lib, "ncclRecv"));
            n.groupStart = reinterpret_cast<decltype(n.groupStart)>(dlsym(lib, "ncclGroupStart"));
            n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(dlsym(lib, "ncclGroupEnd"));
            n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(lib, "ncclGetErrorString"));
            n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.send && n.recv && n.groupStart &&
                   n.groupEnd;
        }
    }
    return n;
}


// Slab buffers of one rank in the peer-direct transport: A (depth-sweep
// input, azimuth slab), R (azimuth-sweep input, depth slab, rank-chunked) and
// the two ordering counters (K1 done, K2 done).
struct SlabPeer {
    cplx* A;
    cplx* R;
    unsigned long long* flags;
};

enum SlabMode { SLAB_VIRT_COPY, SLAB_VIRT_PEER, SLAB_NCCL, SLAB_IPC_PEER };

static bool slab_peer_ok(const pe3d_grid* g, int N) {
    const int NZT = g->n_depth / 8, NZT_s = NZT / N;
    return NZT_s % 32 == 0 && (NZT <= 512 || (NZT % 128 == 0 && NZT / 128 <= 8));
}

static int slab_impl(Handle* h, const pe3d_grid* g, const pe3d_coeffs* coeffs, int32_t N, int32_t rank,
                     SlabMode mode, const void* nccl_id, const SlabPeer* peers, const pe3d_c128* local,
                     const pe3d_c128* u0, pe3d_c128* u_final, double* tl, int64_t* clamped, double* ms_steps,
                     pe3d_error* err) {
    cudaStream_t s = h->stream;
    const bool virt = mode == SLAB_VIRT_COPY || mode == SLAB_VIRT_PEER;
    const bool peer = mode == SLAB_VIRT_PEER || mode == SLAB_IPC_PEER;
    const int NT = g->n_theta, NZ = g->n_depth, NZT = NZ / 8;
    const int C = NT / N, NZT_s = NZT / N, NZ_s = NZ / N;
    const int64_t part = int64_t(NZT) * C * 8;             // elements per rank buffer
    const int64_t chunk = int64_t(NZT_s) * C * 8;          // elements per all-to-all chunk
    const int S = pe3d_sample_count(g->n_steps, g->output_stride);
    const int R = virt ? N : 1;                            // ranks driven by this process
    const int r0 = virt ? 0 : rank;

    ncclComm_t comm = nullptr;
    if (mode == SLAB_NCCL && N > 1) {
        Nccl& n = nccl();
        if (!n.ok) return cuda_fail(err, cudaErrorNotSupported, "libnccl.so.2 not loadable");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t nr = n.commInitRank(&comm, N, id, rank);
        if (nr != ncclSuccess) {
            set_error(err, -1, 0, "ncclCommInitRank: %s", n.errorString ? n.errorString(nr) : "?");
            return PE3D_CUDA_ERROR;
        }
    }
    struct CommGuard {
        ncclComm_t c;
        ~CommGuard() { if (c) nccl().commDestroy(c); }
    } guard{comm};

    std::vector<pe3d::FreqDev> fd = freq_table(g, coeffs);
    // buffers.  Copy / NCCL transports: per driven rank A (K1 in), B (K1 out),
    // Rb (K2 in), W (K2 out).  Peer transports: A and Rb only -- the sweeps
    // store straight into the owners' inputs.
    if (mode != SLAB_IPC_PEER) {
        CK(h->field_a.ensure(size_t(R) * part * (peer ? 1 : 2) * sizeof(cplx)), "alloc");
        CK(h->field_b.ensure(size_t(R) * part * (peer ? 1 : 2) * sizeof(cplx)), "alloc");
    }
    cplx* Abuf = h->field_a.as<cplx>();
    cplx* Bbuf = Abuf + int64_t(R) * part;
    cplx* Rbuf = h->field_b.as<cplx>();
    cplx* Wbuf = Rbuf + int64_t(R) * part;
    std::vector<SlabPeer> P(N);                             // every rank's A / R / counters
    if (mode == SLAB_VIRT_PEER) {
        CK(h->slab_flags.ensure(size_t(N) * 2 * sizeof(unsigned long long)), "alloc");
        CK(cudaMemsetAsync(h->slab_flags.ptr, 0, size_t(N) * 2 * sizeof(unsigned long long), s), "memset");
        for (int q = 0; q < N; ++q)
            P[q] = {Abuf + q * part, Rbuf + q * part, h->slab_flags.as<unsigned long long>() + 2 * q};
    } else if (mode == SLAB_IPC_PEER) {
        for (int q = 0; q < N; ++q) P[q] = peers[q];
    }
    auto own = [&](int q) -> const SlabPeer& { return P[virt ? q : rank]; };
    CK(h->loc_tab.ensure(int64_t(NZ) * sizeof(cplx)), "alloc");
    CK(h->mul_tab.ensure(int64_t(NZ) * sizeof(cplx)), "alloc");
    CK(h->fdev.ensure(sizeof(pe3d::FreqDev)), "alloc");
    CK(h->err.ensure(sizeof(pe3d::DevError)), "alloc");
    CK(h->w_abs.ensure(int64_t(S) * sizeof(double)), "alloc");
    CK(h->h_local.ensure(int64_t(NZ) * sizeof(cplx)), "alloc");
    const int64_t slab_s = int64_t(NT) * NZ_s;             // one depth slab, reference layout
    CK(h->h_u0.ensure(R * slab_s * sizeof(cplx)), "alloc");
    CK(h->h_final.ensure(R * slab_s * sizeof(cplx)), "alloc");
    CK(h->h_tl.ensure(int64_t(R) * S * slab_s * sizeof(double)), "alloc");
    CK(h->h_clamped.ensure(R * sizeof(int64_t)), "alloc");
    const int64_t E = pe3d::ring_table_elems(NT);
    if (g->n_steps > 0) CK(h->ring_tab.ensure(int64_t(g->n_steps) * E * sizeof(cplx)), "alloc");

    std::vector<double> wabs(S);
    for (int k = 0; k < S; ++k) {
        const double r = (k == 0) ? g->r_input : g->r_start + (g->first_index + int64_t(k) * g->output_stride) * g->delta_r;
        wabs[k] = hankel_abs_host(coeffs[0].k0, r);
    }
    pe3d::DevError de0{NO_ERROR, 0, 0};
    CK(cudaMemcpyAsync(h->fdev.ptr, fd.data(), sizeof(pe3d::FreqDev), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->w_abs.ptr, wabs.data(), S * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->err.ptr, &de0, sizeof(de0), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemcpyAsync(h->h_local.ptr, local, NZ * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    CK(cudaMemsetAsync(h->h_clamped.ptr, 0, R * sizeof(int64_t), s), "memset");
    // u0: host [NT][NZ] (virtual: split into depth slabs) or this rank's slab [NT][NZ_s]
    for (int q = 0; q < R; ++q) {
        if (virt)
            CK(cudaMemcpy2DAsync(h->h_u0.as<cplx>() + q * slab_s, NZ_s * sizeof(cplx), u0 + int64_t(q) * NZ_s,
                                 NZ * sizeof(cplx), NZ_s * sizeof(cplx), NT, cudaMemcpyHostToDevice, s), "H2D");
        else
            CK(cudaMemcpyAsync(h->h_u0.ptr, u0, slab_s * sizeof(cplx), cudaMemcpyHostToDevice, s), "H2D");
    }

    // launch contexts: K1 on azimuth slabs, K2 on depth slabs
    pe3d::LaunchCtx c1{};
    c1.n_freq = 1; c1.n_theta = C; c1.n_depth = NZ; c1.n_tiles = NZT;
    c1.sector = 0; c1.num_sms = h->num_sms; c1.delta_theta = g->delta_theta;
    c1.fdev = h->fdev.as<pe3d::FreqDev>(); c1.loc_tab = h->loc_tab.as<cplx>(); c1.mul_tab = h->mul_tab.as<cplx>();
    c1.err = h->err.as<pe3d::DevError>(); c1.stream = s;
    pe3d::LaunchCtx c2 = c1;
    c2.n_theta = NT; c2.n_depth = NZ_s; c2.n_tiles = NZT_s;
    CK(pe3d::launch_factor_depth(c1, h->h_local.as<cplx>(), NZ, g->first_index + 1), "factor");
    if (g->n_steps > 0)
        CK(pe3d::launch_ring_setup(c2, h->ring_tab.as<cplx>(), g->n_steps, g->first_index, g->r_start, g->delta_r),
           "ring setup");

    auto ring_ea = [&](int q) {
        pe3d::EpilogueArgs ea{};
        ea.periodic = 1;
        ea.row_offset = (r0 + q) * NZ_s;
        ea.chunk_cols = C;
        ea.chunk_gap = int64_t(NZT_s - 1) * C * 8;
        ea.clamped = h->h_clamped.as<int64_t>() + q;
        ea.n_samples = S;
        return ea;
    };
    // peer-direct transposes: K2 of depth slab q writes azimuth chunk p of its
    // next temp into A_p at chunk q; K1 of azimuth slab p writes depth slab q
    // of its output into R_q at chunk p
    auto set_peers_k2 = [&](pe3d::EpilogueArgs& ea, int q) {
        for (int p = 0; p < N; ++p) ea.peer[p] = P[p].A + int64_t(r0 + q) * chunk;
    };
    auto k1_ctx = [&](int p) {
        pe3d::LaunchCtx c = c1;
        if (peer) {
            c.n_peers = N;
            c.peer_tiles = NZT_s;
            for (int q = 0; q < N; ++q) c.peer_dst[q] = P[q].R + int64_t(r0 + p) * chunk;
        }
        return c;
    };
    std::vector<unsigned long long*> f0(N), f1(N);          // every rank's K1-done / K2-done counters
    if (peer)
        for (int q = 0; q < N; ++q) { f0[q] = P[q].flags; f1[q] = P[q].flags + 1; }
    // transport W -> A (after K2) and B -> R (after K1), copy / NCCL modes
    auto transpose = [&](cplx* send_base, cplx* recv_base) -> cudaError_t {
        if (virt) {
            for (int a = 0; a < N; ++a)          // sender
                for (int b = 0; b < N; ++b) {    // receiver
                    cudaError_t e = cudaMemcpyAsync(recv_base + int64_t(b) * part + int64_t(a) * chunk,
                                                    send_base + int64_t(a) * part + int64_t(b) * chunk,
                                                    chunk * sizeof(cplx), cudaMemcpyDeviceToDevice, s);
                    if (e != cudaSuccess) return e;
                }
            return cudaSuccess;
        }
        if (N == 1)
            return cudaMemcpyAsync(recv_base, send_base, chunk * sizeof(cplx), cudaMemcpyDeviceToDevice, s);
        Nccl& n = nccl();
        n.groupStart();
        for (int p = 0; p < N; ++p) {
            n.send(send_base + int64_t(p) * chunk, chunk * 2, ncclFloat64, p, comm, s);
            n.recv(recv_base + int64_t(p) * chunk, chunk * 2, ncclFloat64, p, comm, s);
        }
        return n.groupEnd() == ncclSuccess ? cudaSuccess : cudaErrorUnknown;
    };

    // starter on depth slabs -> first temp (into W, or straight into every A)
    for (int q = 0; q < R; ++q) {
        pe3d::EpilogueArgs ea0 = ring_ea(q);
        ea0.tl = tl ? h->h_tl.as<double>() + int64_t(q) * S * slab_s : nullptr;
        ea0.final_out = g->n_steps == 0 ? h->h_final.as<cplx>() + q * slab_s : nullptr;
        ea0.w_abs = h->w_abs.as<double>();
        ea0.sample = 0;
        ea0.write_temp = g->n_steps > 0;
        if (peer && g->n_steps > 0) set_peers_k2(ea0, q);
        CK(pe3d::launch_finish(c2, h->h_u0.as<cplx>() + q * slab_s, 0, peer ? own(q).R : Wbuf + q * part,
                               g->r_input, ea0), "prepare");
        if (peer) CK(pe3d::launch_slab_signal(f1.data(), N, s), "signal");
    }
    const bool stall_test = getenv("PE3D_SLAB_TEST_STALL") != nullptr;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0), "event");
    CK(cudaEventCreate(&e1), "event");
    CK(cudaEventRecord(e0, s), "event");
    if (!peer && g->n_steps > 0) CK(transpose(Wbuf, Abuf), "transpose");
    for (int k = 0; k < g->n_steps; ++k) {
        const int j_new = g->first_index + k + 1;
        const double r_new = g->r_start + j_new * g->delta_r;
        const unsigned long long target = (unsigned long long)N * (k + 1);
        for (int q = 0; q < R; ++q) {
            if (peer) {
                CK(pe3d::launch_slab_wait(own(q).flags + 1, target, c1.err, s), "wait");
                const pe3d::LaunchCtx c = k1_ctx(q);
                CK(pe3d::launch_depth_scan(c, own(q).A, own(q).R), "depth");
                if (!(stall_test && k == 1 && q == R - 1))      // PE3D_SLAB_TEST_STALL: a rank that never signals
                    CK(pe3d::launch_slab_signal(f0.data(), N, s), "signal");
            } else {
                CK(pe3d::launch_depth_scan(c1, Abuf + q * part, Bbuf + q * part), "depth");
            }
        }
        if (!peer) CK(transpose(Bbuf, Rbuf), "transpose");
        const bool record = ((k + 1) % g->output_stride) == 0;
        for (int q = 0; q < R; ++q) {
            pe3d::EpilogueArgs ea = ring_ea(q);
            ea.sample = (k + 1) / g->output_stride;
            ea.tl = (record && tl) ? h->h_tl.as<double>() + int64_t(q) * S * slab_s : nullptr;
            ea.final_out = (k == g->n_steps - 1) ? h->h_final.as<cplx>() + q * slab_s : nullptr;
            ea.w_abs = h->w_abs.as<double>() + ea.sample;
            ea.write_temp = (k < g->n_steps - 1);
            if (peer) {
                if (ea.write_temp) set_peers_k2(ea, q);
                CK(pe3d::launch_slab_wait(own(q).flags, target, c1.err, s), "wait");
                CK(pe3d::launch_azimuth_scan(c2, own(q).R, own(q).R, h->ring_tab.as<cplx>() + int64_t(k) * E, r_new,
                                             ea),
                   "azimuth");
                CK(pe3d::launch_slab_signal(f1.data(), N, s), "signal");
            } else {
                CK(pe3d::launch_azimuth_scan(c2, Rbuf + q * part, Wbuf + q * part,
                                             h->ring_tab.as<cplx>() + int64_t(k) * E, r_new, ea),
                   "azimuth");
            }
        }
        if (!peer && k < g->n_steps - 1) CK(transpose(Wbuf, Abuf), "transpose");
    }
    CK(cudaEventRecord(e1, s), "event");
    const HostFail hf = azimuth_failures(g, coeffs);          // the ring sweep has no pivots
    int st = decode_error(h, s, err, &hf);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms_steps) *ms_steps = ms;
    if (st != PE3D_OK) return st;
    // results: virtual -> reassemble full slabs; one rank -> this rank's slab
    for (int q = 0; q < R; ++q) {
        if (u_final) {
            if (virt)
                CK(cudaMemcpy2DAsync(u_final + int64_t(q) * NZ_s, NZ * sizeof(cplx), h->h_final.as<cplx>() + q * slab_s,
                                     NZ_s * sizeof(cplx), NZ_s * sizeof(cplx), NT, cudaMemcpyDeviceToHost, s), "D2H");
            else
                CK(cudaMemcpyAsync(u_final, h->h_final.ptr, slab_s * sizeof(cplx), cudaMemcpyDeviceToHost, s), "D2H");
        }
        if (tl) {
            if (virt)
                CK(cudaMemcpy2DAsync(tl + int64_t(q) * NZ_s, NZ * sizeof(double),
                                     h->h_tl.as<double>() + int64_t(q) * S * slab_s, NZ_s * sizeof(double),
                                     NZ_s * sizeof(double), int64_t(S) * NT, cudaMemcpyDeviceToHost, s), "D2H");
            else
                CK(cudaMemcpyAsync(tl, h->h_tl.ptr, int64_t(S) * slab_s * sizeof(double), cudaMemcpyDeviceToHost, s),
                   "D2H");
        }
    }
    if (clamped) {
        std::vector<int64_t> cl(R);
        CK(cudaMemcpyAsync(cl.data(), h->h_clamped.ptr, R * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
        CK(cudaStreamSynchronize(s), "sync");
        int64_t tot = 0;
        for (auto v : cl) tot += v;
        *clamped = tot;
    }
    CK(cudaStreamSynchronize(s), "sync");
    return PE3D_OK;
}

static int slab_check(Handle* h, const pe3d_grid* g, const pe3d_coeffs* coeffs, int32_t N, pe3d_error* err) {
    if (!h) return bad_arg(err, "null handle");
    int st = coeffs ? check_grid(g, coeffs, err) : PE3D_OK;
    if (st != PE3D_OK) return st;
    if (!g) return bad_arg(err, "null grid");
    if (g->n_freq != 1) return bad_arg(err, "slab march: n_freq == 1");
    if (g->topology != PE3D_PERIODIC) return bad_arg(err, "slab march: periodic azimuth");
    if (N < 1 || N > pe3d::MAX_PEERS || g->n_theta % N || g->n_depth % (8 * N))
        return bad_arg(err, "slab march: 1 <= N <= 16, n_theta % N, n_depth % 8N");
    return PE3D_OK;
}

}  // namespace

extern "C" {

int pe3d_slab_unique_id(void* out, int32_t bytes) {
    if (!out || bytes < int32_t(sizeof(ncclUniqueId))) return PE3D_BAD_ARGUMENT;
    Nccl& n = nccl();
    if (!n.ok) return PE3D_CUDA_ERROR;
    ncclUniqueId id;
    if (n.getUniqueId(&id) != ncclSuccess) return PE3D_CUDA_ERROR;
    std::memcpy(out, &id, sizeof(id));
    return PE3D_OK;
}

int pe3d_march_slab(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, int32_t N, int32_t rank,
                    const void* nccl_id, const pe3d_c128* local, const pe3d_c128* u0, pe3d_c128* u_final, double* tl,
                    int64_t* clamped, double* ms_steps, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    int st = slab_check(h, g, coeffs, N, err);
    if (st != PE3D_OK) return st;
    if (!local || !u0) return bad_arg(err, "null local or u0");
    const bool virt = nccl_id == nullptr;
    if (!virt && (rank < 0 || rank >= N)) return bad_arg(err, "rank out of range");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    SlabMode mode = SLAB_NCCL;
    if (virt) mode = (slab_peer_ok(g, N) && !getenv("PE3D_SLAB_COPY")) ? SLAB_VIRT_PEER : SLAB_VIRT_COPY;
    return slab_impl(h, g, coeffs, N, rank, mode, nccl_id, nullptr, local, u0, u_final, tl, clamped, ms_steps, err);
}

int pe3d_slab_p2p_export(void* handle, const pe3d_grid* g, int32_t N, int32_t rank, void* out, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    int st = slab_check(h, g, nullptr, N, err);
    if (st != PE3D_OK) return st;
    if (rank < 0 || rank >= N || !out) return bad_arg(err, "rank out of range or null output");
    if (!slab_peer_ok(g, N)) return bad_arg(err, "peer transposes need n_depth / (8 N) % 32 == 0 and a TMA depth sweep");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    const int64_t part = int64_t(g->n_depth / 8) * (g->n_theta / N) * 8;
    CK(h->field_a.ensure(size_t(part) * sizeof(cplx)), "alloc");
    CK(h->field_b.ensure(size_t(part) * sizeof(cplx)), "alloc");
    CK(h->slab_flags.ensure(2 * sizeof(unsigned long long)), "alloc");
    CK(cudaMemset(h->slab_flags.ptr, 0, 2 * sizeof(unsigned long long)), "memset");
    // the counters must be zero before any peer can signal (the caller's barrier
    // follows this call): cudaMemset may return before the device ran it
    CK(cudaDeviceSynchronize(), "sync");
    cudaIpcMemHandle_t hd[3];
    CK(cudaIpcGetMemHandle(&hd[0], h->field_a.ptr), "ipc handle");
    CK(cudaIpcGetMemHandle(&hd[1], h->field_b.ptr), "ipc handle");
    CK(cudaIpcGetMemHandle(&hd[2], h->slab_flags.ptr), "ipc handle");
    std::memcpy(out, hd, sizeof(hd));
    return PE3D_OK;
}

int pe3d_march_slab_p2p(void* handle, const pe3d_grid* g, const pe3d_coeffs* coeffs, int32_t N, int32_t rank,
                        const void* blobs, const pe3d_c128* local, const pe3d_c128* u0, pe3d_c128* u_final,
                        double* tl, int64_t* clamped, double* ms_steps, pe3d_error* err) {
    Handle* h = static_cast<Handle*>(handle);
    int st = slab_check(h, g, coeffs, N, err);
    if (st != PE3D_OK) return st;
    if (rank < 0 || rank >= N || !blobs) return bad_arg(err, "rank out of range or null handles");
    if (!local || !u0) return bad_arg(err, "null local or u0");
    if (!slab_peer_ok(g, N)) return bad_arg(err, "peer transposes need n_depth / (8 N) % 32 == 0 and a TMA depth sweep");
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    // map every other rank's A / R / counters into this process (NVLink peer memory)
    std::vector<SlabPeer> P(N);
    std::vector<void*> opened;
    struct Closer {
        std::vector<void*>& v;
        ~Closer() { for (void* p : v) cudaIpcCloseMemHandle(p); }
    } closer{opened};
    const cudaIpcMemHandle_t* hd = static_cast<const cudaIpcMemHandle_t*>(blobs);
    for (int q = 0; q < N; ++q) {
        if (q == rank) {
            P[q] = {h->field_a.as<cplx>(), h->field_b.as<cplx>(), h->slab_flags.as<unsigned long long>()};
            continue;
        }
        void* ptr[3];
        for (int k = 0; k < 3; ++k) {
            CK(cudaIpcOpenMemHandle(&ptr[k], hd[3 * q + k], cudaIpcMemLazyEnablePeerAccess), "ipc open");
            opened.push_back(ptr[k]);
        }
        P[q] = {static_cast<cplx*>(ptr[0]), static_cast<cplx*>(ptr[1]), static_cast<unsigned long long*>(ptr[2])};
    }
    return slab_impl(h, g, coeffs, N, rank, SLAB_IPC_PEER, nullptr, P.data(), local, u0, u_final, tl, clamped,
                     ms_steps, err);
}

}  // extern "C"
