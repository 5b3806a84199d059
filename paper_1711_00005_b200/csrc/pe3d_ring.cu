// pe3d_ring.cu -- K2, the azimuth sweep of one range step of Eq. (4)
// (arXiv 1711.00005; reference pe3d marching.py:124-136, 167-172).
//
// For every (frequency, depth) row: solve the periodic system
// [1 + cy_lhs Y(r_{j+1})] u = v (ref operators.py:244-262, solved there by
// Sherman-Morrison + Thomas, tridiag.py:186-212), impose the boundary
// (marching.py:133-134), record TL / snapshots / the final slab when asked
// (marching.py:167-172), and apply the NEXT step's explicit azimuth factor
// temp' = [1 + cy_rhs Y(r_{j+1})] u (operators.py:207-208), so that the depth
// sweep needs no azimuth halo.
//
// B is a symmetric circulant with |diag| > 2|off|: B = (-off/rho)(I - rho S)
// (I - rho S^-1), |rho| < 1, so B^-1 v is two cyclic first-order recurrences
// with the uniform multiplier rho.  Each thread runs its chunk of L points
// in registers; chunks are chained by scans whose multipliers are powers of
// rho.  Those powers depend only on (frequency, step) and are tabulated for
// the whole march by k_ring_setup.

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

namespace pe3d {

// Circulant factorisation of B = diag*I + off*(S + S^-1):
// rho + 1/rho = -diag/off, |rho| < 1;  B^-1 = (-rho/off) (I - rho S^-1)^-1 (I - rho S)^-1.
struct RingFactor {
    cplx rho, scale, diag;
    bool diagonal;     // off == 0: B = diag * I
};

__device__ __forceinline__ RingFactor ring_factor(const FreqDev& fd, double s) {
    RingFactor rf;
    // ref operators.py:256-257: diag = 1 - 2*coeff*s, off = coeff*s
    const cplx two_c = crmul(2.0, fd.cy_lhs);
    rf.diag = csub(cone(), crmul(s, two_c));
    const cplx off = crmul(s, fd.cy_lhs);
    rf.diagonal = (off.re == 0.0 && off.im == 0.0);
    if (rf.diagonal) { rf.rho = czero(); rf.scale = crecip(rf.diag); return rf; }
    const cplx tq = crmul(0.5, cneg(cdiv(rf.diag, off)));       // (rho + 1/rho)/2
    cplx sq = csqrt(csub(cmul(tq, tq), cone()));
    if (tq.re * sq.re + tq.im * sq.im < 0.0) sq = cneg(sq);     // larger-magnitude root first (no cancellation)
    rf.rho = crecip(cadd(tq, sq));
    rf.scale = cneg(cdiv(rf.rho, off));
    return rf;
}

__device__ __forceinline__ cplx cpow_int(cplx z, int n) {
    cplx r = cone();
    while (n) {
        if (n & 1) r = cmul(r, z);
        z = cmul(z, z);
        n >>= 1;
    }
    return r;
}

// Ring table of one (step, frequency): [0] rho, [1] scale = -rho/off,
// [2] 1/(1 - rho^N), [3] (diagonal flag, 0), then pw[k] = rho^k (k = 0..L),
// then qp[j] = rho^(jL) (j = 0..n_qp-1).
struct RingLayout {
    int L, G, n_chunks, n_qp, E;
};

__host__ __device__ inline RingLayout ring_layout(int n_theta, int L, int RW) {
    RingLayout r;
    r.L = L;
    r.G = 32 / RW;
    r.n_chunks = (n_theta + L - 1) / L;
    r.n_qp = (r.n_chunks > r.G ? r.n_chunks : r.G) + 1;
    r.E = 4 + (L + 1) + r.n_qp;
    return r;
}

// One thread per (step, frequency), once per march.
__global__ void k_ring_setup(cplx* __restrict__ table, const FreqDev* __restrict__ fdev, int n_freq, int n_steps,
                             int first_index, double r_start, double delta_r, double delta_theta, int n_theta,
                             RingLayout lay, DevError* err) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n_freq * n_steps) return;
    const int s = gid / n_freq, f = gid % n_freq;
    const int j_new = first_index + s + 1;
    const double r_new = r_start + j_new * delta_r;             // Grid3D.range_at
    const FreqDev fd = fdev[f];
    const RingFactor rf = ring_factor(fd, azimuth_scale(fd.k0, r_new, delta_theta));
    cplx* T = table + int64_t(gid) * lay.E;
    cplx* pw = T + 4;
    cplx* qp = pw + lay.L + 1;
    cplx p = cone();
    for (int k = 0; k <= lay.L; ++k) { pw[k] = p; p = cmul(p, rf.rho); }
    const cplx R = pw[lay.L];
    qp[0] = cone();
    for (int j = 1; j < lay.n_qp; ++j) qp[j] = (j & 1) ? cmul(qp[j - 1], R) : cmul(qp[j >> 1], qp[j >> 1]);
    const int q_last = lay.n_chunks - 1;
    const cplx rhoN = cmul(qp[q_last], pw[n_theta - q_last * lay.L]);
    const cplx wrap = csub(cone(), rhoN);
    if (!rf.diagonal && cabs(wrap) < PIVOT_FLOOR) report_failure(err, fail_key(j_new, 1, f, 0), n_theta, 1);
    T[0] = rf.rho;
    T[1] = rf.scale;
    T[2] = crecip(wrap);
    T[3] = mk(rf.diagonal ? 1.0 : 0.0, 0.0);
}

// Given u on this thread's azimuth chunk of one depth row, write the TL
// sample / snapshot / final slab if requested and the next step's
// temp = u + cy_rhs * s_theta * d2_theta(u)  (ref operators.py:105-122,
// 142-153, 207-208; periodic roll order or sector zero-exterior order).
template <int L>
__device__ __forceinline__ void ring_epilogue(cplx (&u)[L], int q, int n_chunks, int nvalid, int i, int rw,
                                              int m0, int l, const EpilogueArgs& ea, int f, int n_theta,
                                              int n_depth, cplx cy_rhs, double s_theta, cplx* sFirst,
                                              cplx* sLast, cplx* dst_row /* blocked, element (m) at m*8 */,
                                              bool in_range) {
    const bool periodic = ea.periodic;
    if (in_range) {
        sFirst[q * rw + i] = u[0];
        if (nvalid == L) {
            sLast[q * rw + i] = u[L - 1];
        } else {
            // partial (last) chunk: predicated stores, the last one wins (a
            // select on u[nvalid-1] would demote u[] to local memory)
#pragma unroll
            for (int k = 0; k < L - 1; ++k)
                if (k < nvalid) sLast[q * rw + i] = u[k];
        }
    }
    __syncthreads();
    if (!in_range) return;
    cplx prev, next;
    if (q > 0) prev = sLast[(q - 1) * rw + i];
    else prev = periodic ? sLast[(n_chunks - 1) * rw + i] : czero();
    if (q < n_chunks - 1) next = sFirst[(q + 1) * rw + i];
    else next = periodic ? sFirst[i] : czero();

    const bool real_row = l < n_depth;
    // TL / snapshots / final slab in the reference layout [..][m][l]
    if (real_row && (ea.tl || ea.snap || ea.final_out)) {
        long long zeros = 0;
#pragma unroll
        for (int k = 0; k < L; ++k) {
            if (k >= nvalid) break;
            const int m = m0 + k;
            const int64_t o = (int64_t(f) * n_theta + m) * n_depth + l;
            if (ea.tl) {
                const double mag = cabs(u[k]) * ea.w_abs[f];
                const double tl = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
                if (mag == 0.0) ++zeros;
                ea.tl[(int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth + (int64_t(m) * n_depth + l)] = tl;
            }
            if (ea.snap) stc(ea.snap + (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth + (int64_t(m) * n_depth + l), u[k]);
            if (ea.final_out) stc(ea.final_out + o, u[k]);
        }
        if (ea.tl && zeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), (unsigned long long)zeros);
    }
    if (!ea.write_temp) return;
    // next step's azimuth factor
#pragma unroll
    for (int k = 0; k < L; ++k) {
        if (k >= nvalid) break;
        const cplx um = k ? u[k - 1] : prev;
        const cplx up = (k + 1 < L && k < nvalid - 1) ? u[(k + 1) % L] : next;
        cplx d2;
        if (periodic) {
            d2 = csub(cadd(up, um), crmul(2.0, u[k]));
        } else {
            const int m = m0 + k;
            if (m == 0) d2 = csub(up, crmul(2.0, u[k]));
            else if (m == n_theta - 1) d2 = csub(um, crmul(2.0, u[k]));
            else d2 = cadd(csub(up, crmul(2.0, u[k])), um);
        }
        const cplx yu = crmul(s_theta, d2);
        stc_stream(dst_row + int64_t(m0 + k) * 8, cadd(u[k], cmul(cy_rhs, yu)));
    }
}

// Solve B u = v for this thread's chunk (registers), given the ring table
// in shared memory.  Thread t = i + RW*q: row i of the CTA's row group,
// chunk q.  Only the last chunk may be partial; the scans never apply a
// multiplier across it to a non-zero value.  Contains
// three __syncthreads (uniform).
template <int L, int RW>
__device__ __forceinline__ void ring_solve(cplx (&v)[L], const cplx* __restrict__ T, int q, int i, int lane, int warp,
                                           int nwarps, int n_theta, int nvalid, cplx* sW, cplx* sV, cplx* sTot) {
    constexpr int G = 32 / RW;
    const int qw = lane / RW;
    const int n_chunks = (n_theta + L - 1) / L;
    const int q_last = n_chunks - 1;
    const int nv_last = n_theta - q_last * L;
    const int n_qp = (n_chunks > G ? n_chunks : G) + 1;
    const cplx* pw = T + 4;
    const cplx* qp = pw + L + 1;
    const cplx rho = T[0], scale = T[1], inv_wrap = T[2];
    if (T[3].re != 0.0) {             // off == 0: B = diag * I (uniform branch)
#pragma unroll
        for (int k = 0; k < L; ++k) v[k] = cmul(v[k], scale);
        __syncthreads();
        __syncthreads();
        __syncthreads();
        return;
    }
    // ---- forward cyclic recurrence w_m = v_m + rho w_{m-1}
    cplx Y = czero();
#pragma unroll
    for (int k = 0; k < L; ++k) if (k < nvalid) { Y = cfma(rho, Y, v[k]); v[k] = Y; }
    const cplx Yloc = Y;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx Yp = shfl_up(Y, d * RW);
        if (qw >= d) Y = cfma(qp[d], Yp, Y);
    }
    cplx ex = shfl_up(Y, RW);
    if (qw == 0) ex = czero();
    if (qw == G - 1) sW[warp * RW + i] = Y;
    __syncthreads();
    cplx C = czero();
    for (int w = 0; w < warp; ++w) C = cfma(qp[G], C, sW[w * RW + i]);
    const cplx Yex = cfma(qp[qw], C, ex);                       // w entering chunk q (non-cyclic)
    if (q == q_last) sTot[i] = cfma(pw[nv_last], Yex, Yloc);    // w at m = N-1 (non-cyclic)
    __syncthreads();
    const cplx w_last = cmul(sTot[i], inv_wrap);
    const cplx c_in = cfma(qp[q < n_qp ? q : 0], w_last, Yex);
#pragma unroll
    for (int k = 0; k < L; ++k) if (k < nvalid) v[k] = cfma(pw[k + 1], c_in, v[k]);

    // ---- backward cyclic recurrence x_m = w_m + rho x_{m+1}
    cplx X = czero();
#pragma unroll
    for (int k = L - 1; k >= 0; --k) if (k < nvalid) { X = cfma(rho, X, v[k]); v[k] = X; }
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx Xn = shfl_down(X, d * RW);
        if (qw + d < G) X = cfma(qp[d], Xn, X);
    }
    const cplx nx = shfl_down(X, RW);
    if (qw == 0) sV[warp * RW + i] = X;
    __syncthreads();
    cplx D = czero();
    for (int w = nwarps - 1; w > warp; --w) D = cfma(qp[G], D, sV[w * RW + i]);
    if (q == 0) sTot[RW + i] = cfma(qp[G], D, X);                 // S_0
    const cplx S_next = (qw == G - 1) ? D : cfma(qp[G - qw - 1], D, nx);
    __syncthreads();
    const cplx x0 = cmul(sTot[RW + i], inv_wrap);
    cplx c_up;
    if (q >= q_last) c_up = x0;
    else c_up = cfma(cmul(qp[q_last - q - 1], pw[nv_last]), x0, S_next);
    const cplx cs = cmul(scale, c_up);
#pragma unroll
    for (int k = 0; k < L; ++k) if (k < nvalid) v[k] = cfma(pw[nvalid - k], cs, cmul(scale, v[k]));
}

template <int L, int RW>
struct RingSmem {
    // element offsets inside the dynamic shared memory of the ring kernels
    int table, sW, sV, sTot, sFirst, sLast, stage, total;
    __host__ __device__ RingSmem(int n_theta, int nthreads, int E, int stages) {
        const int n_chunks = (n_theta + L - 1) / L;
        const int nwarps = nthreads / 32;
        stage = 0;
        table = stages * RW * n_theta;
        sW = table + E;
        sV = sW + nwarps * RW;
        sTot = sV + nwarps * RW;
        sFirst = sTot + 2 * RW;
        sLast = sFirst + n_chunks * RW;
        total = sLast + n_chunks * RW;
    }
};

// Persistent, pipelined azimuth sweep for rings whose 8-row tile fits a
// shared-memory stage (RW = 8).  Work items are (frequency, depth tile);
// each thread cp.asyncs its own chunk of item n+STAGES-1 while item n is
// solved, so no CTA barrier is needed for the staged data.
template <int L, int STAGES>
__global__ void __launch_bounds__(512, 1)
k_azimuth_pipe(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ table, int E,
               const FreqDev* __restrict__ fdev, int n_theta, int n_tiles, int n_depth, int64_t total_items,
               int items_per_cta, double r_new, double delta_theta, EpilogueArgs ea) {
    constexpr int RW = 8;
    extern __shared__ cplx smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
    const int i = t % RW, q = t / RW;
    const int n_chunks = (n_theta + L - 1) / L;
    const bool in_range = q < n_chunks;
    const RingSmem<L, RW> lay(n_theta, blockDim.x, E, STAGES);
    cplx* T = smem + lay.table;
    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t ring = int64_t(n_theta) * 8;      // elements per (f, tile) item

    const int64_t it0 = int64_t(blockIdx.x) * items_per_cta;
    const int64_t it1 = it0 + items_per_cta < total_items ? it0 + items_per_cta : total_items;
    if (it0 >= it1) return;
    auto fetch = [&](int64_t item, int st) {
        const cplx* g = src + item * ring + i;
        cplx* d = smem + st * RW * n_theta + i;
#pragma unroll
        for (int k = 0; k < L; ++k)
            if (k < nvalid) cp_async16(d + (m0 + k) * RW, g + int64_t(m0 + k) * 8);
    };
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (it0 + p < it1) fetch(it0 + p, p);
        cp_async_commit();
    }
    int cur_f = -1;
    int slot = 0;
    for (int64_t item = it0; item < it1; ++item, slot = (slot + 1 == STAGES) ? 0 : slot + 1) {
        const int f = int(item / n_tiles);
        const int tile = int(item - int64_t(f) * n_tiles);
        if (f != cur_f) {
            __syncthreads();
            for (int e = t; e < E; e += blockDim.x) T[e] = table[int64_t(f) * E + e];
            __syncthreads();
            cur_f = f;
        }
        {
            const int64_t ip = item + STAGES - 1;
            if (ip < it1) fetch(ip, (slot + STAGES - 1) % STAGES);
            cp_async_commit();
            cp_async_wait<STAGES - 1>();
        }
        cplx v[L];
        const cplx* stg = smem + slot * RW * n_theta + i;
#pragma unroll
        for (int k = 0; k < L; ++k) v[k] = (k < nvalid) ? stg[(m0 + k) * RW] : czero();
        ring_solve<L, RW>(v, T, q, i, lane, warp, nwarps, n_theta, nvalid, smem + lay.sW, smem + lay.sV,
                          smem + lay.sTot);
        const int l = tile * 8 + i;
        if (l == 0 || l >= n_depth) {
#pragma unroll
            for (int k = 0; k < L; ++k) v[k] = czero();
        }
        const FreqDev fd = fdev[f];
        ring_epilogue<L>(v, q, n_chunks, nvalid, i, RW, m0, l, ea, f, n_theta, n_depth, fd.cy_rhs,
                         azimuth_scale(fd.k0, r_new, delta_theta), smem + lay.sFirst, smem + lay.sLast,
                         dst + item * ring + i, in_range);
    }
    cp_async_wait<0>();
}

// Direct variant (one CTA per (frequency, row group), registers only) for
// rings too wide for a shared-memory stage (RW < 8).
template <int L, int RW>
__global__ void __launch_bounds__(512)
k_azimuth_direct(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ table, int E,
                 const FreqDev* __restrict__ fdev, int n_theta, int n_tiles, int n_depth, double r_new,
                 double delta_theta, EpilogueArgs ea) {
    extern __shared__ cplx smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
    const int i = t % RW, q = t / RW;
    const int n_chunks = (n_theta + L - 1) / L;
    const bool in_range = q < n_chunks;
    const RingSmem<L, RW> lay(n_theta, blockDim.x, E, 0);
    const int groups = 8 / RW;
    const int tile = blockIdx.x / groups;
    const int l = tile * 8 + (blockIdx.x % groups) * RW + i;
    const int f = blockIdx.y;
    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t row_base = (int64_t(f) * n_tiles + tile) * n_theta * 8 + (l & 7);
    cplx v[L];
#pragma unroll
    for (int k = 0; k < L; ++k) v[k] = (k < nvalid) ? ldc_stream(src + row_base + int64_t(m0 + k) * 8) : czero();
    cplx* T = smem + lay.table;
    for (int e = t; e < E; e += blockDim.x) T[e] = table[int64_t(f) * E + e];
    __syncthreads();
    ring_solve<L, RW>(v, T, q, i, lane, warp, nwarps, n_theta, nvalid, smem + lay.sW, smem + lay.sV,
                      smem + lay.sTot);
    if (l == 0 || l >= n_depth) {
#pragma unroll
        for (int k = 0; k < L; ++k) v[k] = czero();
    }
    const FreqDev fd = fdev[f];
    ring_epilogue<L>(v, q, n_chunks, nvalid, i, RW, m0, l, ea, f, n_theta, n_depth, fd.cy_rhs,
                     azimuth_scale(fd.k0, r_new, delta_theta), smem + lay.sFirst, smem + lay.sLast,
                     dst + row_base, in_range);
}

// Load u (reference layout [f][m][l] or device tiles), apply the boundary
// (ref marching.py:80-90) and run the ring epilogue at range r.
template <int L, int RW>
__global__ void __launch_bounds__(512)
k_finish(const cplx* __restrict__ src, int src_tiled, cplx* __restrict__ dst, const FreqDev* __restrict__ fdev,
         int n_theta, int n_tiles, int n_depth, double r, double delta_theta, EpilogueArgs ea) {
    extern __shared__ cplx smem[];
    const int t = threadIdx.x;
    const int i = t % RW, q = t / RW;
    const int n_chunks = (n_theta + L - 1) / L;
    const bool in_range = q < n_chunks;
    cplx* sFirst = smem;
    cplx* sLast = sFirst + n_chunks * RW;
    const int groups = 8 / RW;
    const int tile = blockIdx.x / groups;
    const int l = tile * 8 + (blockIdx.x % groups) * RW + i;
    const int f = blockIdx.y;
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r, delta_theta);
    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t row_base = (int64_t(f) * n_tiles + tile) * n_theta * 8 + (l & 7);
    cplx u[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
        cplx v = czero();
        const int m = m0 + k;
        if (k < nvalid && l < n_depth) {
            v = src_tiled ? ldc(src + row_base + int64_t(m) * 8) : ldc(src + (int64_t(f) * n_theta + m) * n_depth + l);
            if (l == 0 || (!ea.periodic && (m == 0 || m == n_theta - 1))) v = czero();
        }
        u[k] = v;
    }
    ring_epilogue<L>(u, q, n_chunks, nvalid, i, RW, m0, l, ea, f, n_theta, n_depth, fd.cy_rhs, s, sFirst, sLast,
                     dst + row_base, in_range);
}

// ------------------------------------------------------------ launchers

static int round32(int x) { return (x + 31) / 32 * 32; }

// Chunk length L and rows per CTA RW for a ring of n_theta points: the widest
// row group (full 128-B lines) with short chunks that fits 512 threads.
void ring_shape(int n_theta, int* L, int* RW) {
    const int cand_L[2] = {8, 16};
    for (int li = 0; li < 2; ++li)
        for (int rw = 8; rw >= 2; rw /= 2)
            if (round32(rw * ((n_theta + cand_L[li] - 1) / cand_L[li])) <= 512) { *L = cand_L[li]; *RW = rw; return; }
    *L = 0; *RW = 0;   // n_theta > 4096: not supported by the ring kernels
}

int ring_table_elems(int n_theta) {
    int L, RW;
    ring_shape(n_theta, &L, &RW);
    return ring_layout(n_theta, L, RW).E;
}

cudaError_t launch_ring_setup(const LaunchCtx& c, cplx* table, int n_steps, int first_index, double r_start,
                              double delta_r) {
    int L, RW;
    ring_shape(c.n_theta, &L, &RW);
    const RingLayout lay = ring_layout(c.n_theta, L, RW);
    const int total = c.n_freq * n_steps;
    if (total == 0) return cudaSuccess;
    k_ring_setup<<<(total + 63) / 64, 64, 0, c.stream>>>(table, c.fdev, c.n_freq, n_steps, first_index, r_start,
                                                         delta_r, c.delta_theta, c.n_theta, lay, c.err);
    return cudaGetLastError();
}

template <class K>
static cudaError_t set_smem(K kern, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

cudaError_t launch_azimuth_scan(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, double r_new,
                                const EpilogueArgs& ea) {
    int L, RW;
    ring_shape(c.n_theta, &L, &RW);
    const RingLayout rl = ring_layout(c.n_theta, L, RW);
    const int nthreads = round32(RW * rl.n_chunks);
    const size_t stage_bytes = sizeof(cplx) * size_t(RW) * c.n_theta;
    if (RW == 8 && 2 * stage_bytes <= 160 * 1024) {
        const int stages = (3 * stage_bytes <= 100 * 1024) ? 3 : 2;
        const int64_t items = int64_t(c.n_freq) * c.n_tiles;
        auto go = [&](auto kern, int Lv) -> cudaError_t {
            RingSmem<8, 8> dummy(0, 0, 0, 0);
            (void)dummy;
            const int n_chunks = (c.n_theta + Lv - 1) / Lv;
            const size_t elems = size_t(stages) * RW * c.n_theta + rl.E + 2 * (nthreads / 32) * RW + 2 * RW +
                                 2 * size_t(n_chunks) * RW;
            const size_t bytes = sizeof(cplx) * elems;
            cudaError_t e = set_smem(kern, bytes);
            if (e != cudaSuccess) return e;
            int per_sm = int((228 * 1024) / (bytes + 1024));
            if (per_sm < 1) per_sm = 1;
            const int64_t ctas = int64_t(c.num_sms) * per_sm;
            const int per = int((items + ctas - 1) / ctas);
            const int grid = int((items + per - 1) / per);
            kern<<<grid, nthreads, bytes, c.stream>>>(src, dst, table_step, rl.E, c.fdev, c.n_theta, c.n_tiles,
                                                      c.n_depth, items, per, r_new, c.delta_theta, ea);
            return cudaGetLastError();
        };
        if (L == 8 && stages == 3) return go(k_azimuth_pipe<8, 3>, 8);
        if (L == 8 && stages == 2) return go(k_azimuth_pipe<8, 2>, 8);
        if (L == 16 && stages == 3) return go(k_azimuth_pipe<16, 3>, 16);
        if (L == 16 && stages == 2) return go(k_azimuth_pipe<16, 2>, 16);
    }
    dim3 grid(c.n_tiles * (8 / RW), c.n_freq);
    auto direct = [&](auto kern, int Lv, int RWv) -> cudaError_t {
        const int n_chunks = (c.n_theta + Lv - 1) / Lv;
        const size_t bytes = sizeof(cplx) * (rl.E + 2 * (nthreads / 32) * RWv + 2 * RWv + 2 * size_t(n_chunks) * RWv);
        cudaError_t e = set_smem(kern, bytes);
        if (e != cudaSuccess) return e;
        kern<<<grid, nthreads, bytes, c.stream>>>(src, dst, table_step, rl.E, c.fdev, c.n_theta, c.n_tiles, c.n_depth,
                                                  r_new, c.delta_theta, ea);
        return cudaGetLastError();
    };
    if (L == 8 && RW == 8) return direct(k_azimuth_direct<8, 8>, 8, 8);
    if (L == 8 && RW == 4) return direct(k_azimuth_direct<8, 4>, 8, 4);
    if (L == 8 && RW == 2) return direct(k_azimuth_direct<8, 2>, 8, 2);
    if (L == 16 && RW == 8) return direct(k_azimuth_direct<16, 8>, 16, 8);
    if (L == 16 && RW == 4) return direct(k_azimuth_direct<16, 4>, 16, 4);
    if (L == 16 && RW == 2) return direct(k_azimuth_direct<16, 2>, 16, 2);
    return cudaErrorInvalidConfiguration;
}

cudaError_t launch_finish(const LaunchCtx& c, const cplx* src, int src_tiled, cplx* dst, double r,
                          const EpilogueArgs& ea) {
    int L, RW;
    ring_shape(c.n_theta, &L, &RW);
    const int n_chunks = (c.n_theta + L - 1) / L;
    const int nthreads = round32(RW * n_chunks);
    dim3 grid(c.n_tiles * (8 / RW), c.n_freq);
    const size_t sm = sizeof(cplx) * 2 * n_chunks * RW;
#define CALL(Lv, RWv)                                                                                           \
    if (L == Lv && RW == RWv) {                                                                                 \
        k_finish<Lv, RWv><<<grid, nthreads, sm, c.stream>>>(src, src_tiled, dst, c.fdev, c.n_theta, c.n_tiles, \
                                                            c.n_depth, r, c.delta_theta, ea);                   \
        return cudaGetLastError();                                                                              \
    }
    CALL(8, 8) CALL(8, 4) CALL(8, 2) CALL(16, 8) CALL(16, 4) CALL(16, 2)
#undef CALL
    return cudaErrorInvalidConfiguration;
}

}  // namespace pe3d
