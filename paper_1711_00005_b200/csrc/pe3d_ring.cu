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

#include <algorithm>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>

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
// [2] 1/(1 - rho^N), [3] (diagonal flag, 0), [4] b1, [5] b2 (the epilogue's
// next-temp weights, see ring_epilogue), [6] 1/(1 - rho^2), [7] rho/(1 - rho^2)
// (the halo closure of k_azimuth_tma HALO), then pw[k] = rho^k (k = 0..L), then
// qp[j] = rho^(jL) (j = 0..n_qp-1).
constexpr int RING_HDR = 8;
struct RingLayout {
    int L, G, n_chunks, n_qp, E;
};

__host__ __device__ inline RingLayout ring_layout(int n_theta, int L, int RW) {
    RingLayout r;
    r.L = L;
    r.G = 32 / RW;
    r.n_chunks = (n_theta + L - 1) / L;
    r.n_qp = (r.n_chunks > r.G ? r.n_chunks : r.G) + 1;
    r.E = RING_HDR + (L + 1) + r.n_qp;
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
    const double r_new = __dadd_rn(r_start, __dmul_rn(double(j_new), delta_r));   // Grid3D.range_at (no FMA, as the host)
    const FreqDev fd = fdev[f];
    const RingFactor rf = ring_factor(fd, azimuth_scale(fd.k0, r_new, delta_theta));
    cplx* T = table + int64_t(gid) * lay.E;
    cplx* pw = T + RING_HDR;
    cplx* qp = pw + lay.L + 1;
    cplx p = cone();
    for (int k = 0; k <= lay.L; ++k) { pw[k] = p; p = cmul(p, rf.rho); }
    const cplx R = pw[lay.L];
    qp[0] = cone();
    for (int j = 1; j < lay.n_qp; ++j) qp[j] = (j & 1) ? cmul(qp[j - 1], R) : cmul(qp[j >> 1], qp[j >> 1]);
    const int q_last = lay.n_chunks - 1;
    const cplx rhoN = cmul(qp[q_last], pw[n_theta - q_last * lay.L]);
    const cplx wrap = csub(cone(), rhoN);
    // failures: the reference's own pivot checks of this matrix decide, on the
    // host (pe3d_host.h azimuth_failures); the circulant factorisation has none
    T[0] = rf.rho;
    T[1] = rf.scale;
    T[2] = crecip(wrap);
    T[3] = mk(rf.diagonal ? 1.0 : 0.0, 0.0);
    // next temp = b1 x + b2 (x+ + x-) (same arithmetic as the sweeps' own)
    const cplx alpha = crmul(azimuth_scale(fd.k0, r_new, delta_theta), fd.cy_rhs);
    const cplx b2 = cmul(rf.scale, alpha);
    T[4] = csub(rf.scale, cadd(b2, b2));
    T[5] = b2;
    const cplx s_inf = crecip(csub(cone(), cmul(rf.rho, rf.rho)));
    T[6] = s_inf;
    T[7] = cmul(rf.rho, s_inf);
}

// Given u on this thread's azimuth chunk of RT depth rows, write the TL
// sample / snapshot / final slab if requested and the next step's
// temp = u + cy_rhs * s_theta * d2_theta(u)  (ref operators.py:105-122,
// 142-153, 207-208; periodic roll order or sector zero-exterior order).
// Row h of this thread is row-in-group r_h = i + h*RWT of the CTA's RW rows;
// its device-tile element (m) is at dst_tile[m*8 + r_h + row0].
template <int L, int RT>
__device__ __forceinline__ void ring_epilogue(cplx (&u)[RT][L], int q, int n_chunks, int nvalid, int i, int RWT,
                                              int RW, int m0, int row0, int l0, const EpilogueArgs& ea, int f,
                                              int n_theta, int n_depth, cplx scale, cplx cy_rhs, double s_theta,
                                              cplx* sFirst, cplx* sLast, cplx* dst_tile, bool in_range) {
    // u holds x with the field = scale * x.  temp = field + cy_rhs s (x+ + x- - 2x) scale
    //   = b1 x + b2 (x+ + x-),  b1 = scale (1 - 2 alpha),  b2 = scale alpha,  alpha = cy_rhs s
    const cplx alpha = crmul(s_theta, cy_rhs);
    const cplx b2 = cmul(scale, alpha);
    const cplx b1 = csub(scale, cadd(b2, b2));
    const bool periodic = ea.periodic;
    if (in_range) {
#pragma unroll
        for (int h = 0; h < RT; ++h) {
            const int r = i + h * RWT;
            sFirst[q * RW + r] = u[h][0];
            if (nvalid == L) {
                sLast[q * RW + r] = u[h][L - 1];
            } else {
                // partial (last) chunk: predicated stores, the last one wins (a
                // select on u[nvalid-1] would demote u[] to local memory)
#pragma unroll
                for (int k = 0; k < L - 1; ++k)
                    if (k < nvalid) sLast[q * RW + r] = u[h][k];
            }
        }
    }
    __syncthreads();
    if (!in_range) return;
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        const int r = i + h * RWT;
        const int l = l0 + r;
        cplx prev, next;
        if (q > 0) prev = sLast[(q - 1) * RW + r];
        else prev = periodic ? sLast[(n_chunks - 1) * RW + r] : czero();
        if (q < n_chunks - 1) next = sFirst[(q + 1) * RW + r];
        else next = periodic ? sFirst[r] : czero();

        // TL / snapshots / final slab in the reference layout [..][m][l]
        if (l < n_depth && (ea.tl || ea.snap || ea.final_out)) {
            long long zeros = 0;
#pragma unroll
            for (int k = 0; k < L; ++k) {
                if (k >= nvalid) break;
                const int m = m0 + k;
                const int64_t o = (int64_t(f) * n_theta + m) * n_depth + l;
                const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth + (int64_t(m) * n_depth + l);
                const cplx uf = cmul(scale, u[h][k]);
                if (ea.tl) {
                    const double mag = cabs(uf) * ea.w_abs[f];
                    const double tl = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
                    if (mag == 0.0) ++zeros;
                    ea.tl[so] = tl;
                }
                if (ea.snap) stc(ea.snap + so, uf);
                if (ea.final_out) stc(ea.final_out + o, uf);
            }
            if (ea.tl && zeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), (unsigned long long)zeros);
        }
        if (!ea.write_temp) continue;
        // next step's azimuth factor (zero exterior on a sector ring: prev/next = 0)
        cplx* dst_row = dst_tile + row0 + r;
#pragma unroll
        for (int k = 0; k < L; ++k) {
            if (k >= nvalid) break;
            const cplx um = k ? u[h][k - 1] : prev;
            const cplx up = (k + 1 < L && k < nvalid - 1) ? u[h][(k + 1) % L] : next;
            const cplx tv = cfma(b1, u[h][k], cmul(b2, cadd(up, um)));
            if (ea.peer[0]) stc_stream(peer_elem(ea, m0 + k, l0 >> 3, row0 + r), tv);   // fused transpose
            else stc_stream(dst_row + ring_off(m0 + k, ea.chunk_cols, ea.chunk_gap), tv);
        }
    }
}

// Solve B u = v for this thread's chunk of RT rows (registers), given the
// ring table T in shared memory.  Thread t = i + RWT*q (RWT = RW/RT lane
// slots per chunk) holds rows i + h*RWT of the CTA's RW rows, chunk q.  The
// RT rows are independent systems interleaved for instruction-level
// parallelism.  Only the last chunk may be partial; the scans never apply a
// multiplier across it to a non-zero value.  Contains
// three __syncthreads (uniform).
template <int L, int RW, int RT, bool FULL>
__device__ __forceinline__ void ring_solve(cplx (&v)[RT][L], const cplx* __restrict__ T, int q, int i, int lane,
                                           int warp, int nwarps, int n_theta, int nvalid_, cplx* sW, cplx* sV,
                                           cplx* sTot) {
    const int nvalid = FULL ? L : nvalid_;
    constexpr int RWT = RW / RT;
    constexpr int G = 32 / RWT;                      // chunks per warp
    const int qw = lane / RWT;
    const int n_chunks = (n_theta + L - 1) / L;
    const int q_last = n_chunks - 1;
    const int nv_last = n_theta - q_last * L;
    const int n_qp = (n_chunks > G ? n_chunks : G) + 1;
    const cplx* pw = T + RING_HDR;
    const cplx* qp = pw + L + 1;
    const cplx rho = T[0], inv_wrap = T[2];
    if (T[3].re != 0.0) {             // off == 0: B = diag * I, x = v (the scale is applied by the epilogue)
        __syncthreads();
        __syncthreads();
        __syncthreads();
        return;
    }
    // ---- forward cyclic recurrence w_m = v_m + rho w_{m-1}
    cplx Y[RT], Yloc[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) Y[h] = czero();
    if (FULL || nvalid == L) {
#pragma unroll
        for (int k = 0; k < L; ++k)
#pragma unroll
            for (int h = 0; h < RT; ++h) { Y[h] = cfma(rho, Y[h], v[h][k]); v[h][k] = Y[h]; }
    } else {
#pragma unroll
        for (int k = 0; k < L; ++k)
            if (k < nvalid)
#pragma unroll
                for (int h = 0; h < RT; ++h) { Y[h] = cfma(rho, Y[h], v[h][k]); v[h][k] = Y[h]; }
    }
#pragma unroll
    for (int h = 0; h < RT; ++h) Yloc[h] = Y[h];
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx m = (qw >= d) ? qp[d] : czero();
#pragma unroll
        for (int h = 0; h < RT; ++h) Y[h] = cfma(m, shfl_up(Y[h], d * RWT), Y[h]);
    }
    cplx ex[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        ex[h] = shfl_up(Y[h], RWT);
        if (qw == 0) ex[h] = czero();
        if (qw == G - 1) sW[warp * RW + i + h * RWT] = Y[h];
    }
    __syncthreads();
    cplx C[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) C[h] = czero();
    for (int w = 0; w < warp; ++w)
#pragma unroll
        for (int h = 0; h < RT; ++h) C[h] = cfma(qp[G], C[h], sW[w * RW + i + h * RWT]);
    cplx Yex[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        Yex[h] = cfma(qp[qw], C[h], ex[h]);                                       // w entering chunk q
        if (q == q_last) sTot[i + h * RWT] = cfma(pw[nv_last], Yex[h], Yloc[h]);  // w at m = N-1 (non-cyclic)
    }
    __syncthreads();
    const cplx qpq = qp[q < n_qp ? q : 0];
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        const cplx c_in = cfma(qpq, cmul(sTot[i + h * RWT], inv_wrap), Yex[h]);
#pragma unroll
        for (int k = 0; k < L; ++k) if (k < nvalid) v[h][k] = cfma(pw[k + 1], c_in, v[h][k]);
    }

    // ---- backward cyclic recurrence x_m = w_m + rho x_{m+1}
    cplx X[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) X[h] = czero();
    if (FULL || nvalid == L) {
#pragma unroll
        for (int k = L - 1; k >= 0; --k)
#pragma unroll
            for (int h = 0; h < RT; ++h) { X[h] = cfma(rho, X[h], v[h][k]); v[h][k] = X[h]; }
    } else {
#pragma unroll
        for (int k = L - 1; k >= 0; --k)
            if (k < nvalid)
#pragma unroll
                for (int h = 0; h < RT; ++h) { X[h] = cfma(rho, X[h], v[h][k]); v[h][k] = X[h]; }
    }
    if (q >= n_chunks) {              // idle lanes (FULL mode runs them unpredicated) contribute nothing
#pragma unroll
        for (int h = 0; h < RT; ++h) X[h] = czero();
    }
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx m = (qw + d < G) ? qp[d] : czero();
#pragma unroll
        for (int h = 0; h < RT; ++h) X[h] = cfma(m, shfl_down(X[h], d * RWT), X[h]);
    }
    cplx nx[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        nx[h] = shfl_down(X[h], RWT);
        if (qw == 0) sV[warp * RW + i + h * RWT] = X[h];
    }
    __syncthreads();
    cplx D[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) D[h] = czero();
    for (int w = nwarps - 1; w > warp; --w)
#pragma unroll
        for (int h = 0; h < RT; ++h) D[h] = cfma(qp[G], D[h], sV[w * RW + i + h * RWT]);
    cplx S_next[RT];
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        if (q == 0) sTot[RW + i + h * RWT] = cfma(qp[G], D[h], X[h]);           // S_0
        S_next[h] = (qw == G - 1) ? D[h] : cfma(qp[G - qw - 1], D[h], nx[h]);
    }
    __syncthreads();
    const cplx up_mult = (q >= q_last) ? czero() : cmul(qp[q_last - q - 1], pw[nv_last]);
#pragma unroll
    for (int h = 0; h < RT; ++h) {
        const cplx x0 = cmul(sTot[RW + i + h * RWT], inv_wrap);
        const cplx c_up = (q >= q_last) ? x0 : cfma(up_mult, x0, S_next[h]);
#pragma unroll
        for (int k = 0; k < L; ++k) if (k < nvalid) v[h][k] = cfma(pw[nvalid - k], c_up, v[h][k]);
    }
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
// shared-memory stage.  Work items are (frequency, depth tile); each thread
// cp.asyncs its own RT x L points of item n+STAGES-1 while item n is solved,
// so no CTA barrier is needed for the staged data.  Stage slot of (m, r):
// m*8 + (r ^ 4*((m/L)&1)), conflict free for the thread-own reads.
template <int L, int STAGES, int RT, bool FULL>
__global__ void __launch_bounds__(256, 2)
k_azimuth_pipe(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ table, int E,
               const FreqDev* __restrict__ fdev, int n_theta, int n_tiles, int n_depth, int64_t total_items,
               int items_per_cta, double r_new, double delta_theta, EpilogueArgs ea) {
    constexpr int RW = 8, RWT = RW / RT;
    extern __shared__ cplx smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
    const int i = t % RWT, q = t / RWT;
    const int n_chunks = (n_theta + L - 1) / L;
    const bool in_range = q < n_chunks;
    const RingSmem<L, RW> lay(n_theta, blockDim.x, E, STAGES);
    cplx* T = smem + lay.table;
    const int m0 = q * L;
    const int nvalid = FULL ? (in_range ? L : 0) : (in_range ? min(L, n_theta - m0) : 0);
    const int swz = 4 * (q & 1);
    const int64_t ring = int64_t(n_theta) * 8;      // elements per (f, tile) item

    const int64_t it0 = int64_t(blockIdx.x) * items_per_cta;
    const int64_t it1 = it0 + items_per_cta < total_items ? it0 + items_per_cta : total_items;
    if (it0 >= it1) return;
    auto fetch = [&](int64_t item, int st) {
        const cplx* g = src + item * ring;
        cplx* d = smem + st * RW * n_theta;
#pragma unroll
        for (int h = 0; h < RT; ++h) {
            const int r = i + h * RWT;
#pragma unroll
            for (int k = 0; k < L; ++k)
                if (k < nvalid) cp_async16(d + (m0 + k) * 8 + (r ^ swz), g + int64_t(m0 + k) * 8 + r);
        }
    };
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (it0 + p < it1) fetch(it0 + p, p);
        cp_async_commit();
    }
    int f = int(it0 / n_tiles), tile = int(it0 - int64_t(f) * n_tiles);
    int cur_f = -1;
    int slot = 0;
    for (int64_t item = it0; item < it1; ++item) {
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
        cplx v[RT][L];
        const cplx* stg = smem + slot * RW * n_theta;
#pragma unroll
        for (int h = 0; h < RT; ++h)
#pragma unroll
            for (int k = 0; k < L; ++k)
                v[h][k] = (k < nvalid) ? stg[(m0 + k) * 8 + ((i + h * RWT) ^ swz)] : czero();
        // FULL: every chunk has L points; idle threads (q >= n_chunks) carry zeros
        ring_solve<L, RW, RT, FULL>(v, T, q, i, lane, warp, nwarps, n_theta, nvalid, smem + lay.sW,
                                    smem + lay.sV, smem + lay.sTot);
        const int l0 = tile * 8;
#pragma unroll
        for (int h = 0; h < RT; ++h) {
            const int l = l0 + i + h * RWT;
            if (l + ea.row_offset == 0 || l >= n_depth) {
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = czero();
            }
        }
        const FreqDev fd = fdev[f];
        ring_epilogue<L, RT>(v, q, n_chunks, nvalid, i, RWT, RW, m0, 0, l0, ea, f, n_theta, n_depth, T[1],
                             fd.cy_rhs, azimuth_scale(fd.k0, r_new, delta_theta), smem + lay.sFirst,
                             smem + lay.sLast, dst + item * ring, in_range);
        if (++tile == n_tiles) { tile = 0; ++f; }
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}


// ------------------------------------------- ring-per-warp azimuth sweep
// For rings of 32*L points (L = 2..16): one warp solves whole rings, lane q
// holding chunk q (L points) of RT rows.  All chaining is done with warp
// shuffles -- the forward/backward scans (5 levels, multipliers R^d with
// R = rho^L), the cyclic wrap (lane 31 / lane 0 broadcasts) and the
// epilogue's azimuth neighbours -- so the solve itself needs no shared
// memory and no barrier.  The CTA's 8/RT warps cover the 8 rows of a depth
// tile; the tile (one contiguous 32*L*128-B block) is moved with full-line
// coalesced cp.async / stores through a stage whose slot for (m, r) is
// m*8 + (r ^ ((m/L) & 7)): conflict free both for the line-wise copies and
// for the lane-per-chunk reads.
template <int L>
__device__ __forceinline__ int ring_slot(int m, int r) { return m * 8 + (r ^ ((m / L) & 7)); }

// CHUNKED: rank-chunked ring layout of the slab march (ea.chunk_cols /
// chunk_gap); the standard march compiles the plain contiguous addressing.
template <int L, int RT, int STAGES, bool CHUNKED, bool PEER = false>
__global__ void __launch_bounds__(32 * 8 / RT)
k_azimuth_warp(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ table, int E,
               const FreqDev* __restrict__ fdev, int n_tiles, int n_depth, int64_t total_items, int items_per_cta,
               double r_new, double delta_theta, EpilogueArgs ea) {
    constexpr int NT = 32 * L;                      // ring length
    constexpr int ITEM = NT * 8;                    // elements per (f, tile) item
    constexpr int NTHR = 32 * 8 / RT;
    constexpr int PER = ITEM / NTHR;                // 16-B chunks per thread per item
    extern __shared__ cplx smem[];
    cplx* T = smem + STAGES * ITEM;                 // ring table of the current frequency
    const cplx* pw = T + RING_HDR;                         // rho^k, k = 0..L
    const cplx* qp = pw + L + 1;                    // R^j, j = 0..32
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane, swz = q & 7;
    const int m0 = q * L;

    const int64_t it0 = int64_t(blockIdx.x) * items_per_cta;
    const int64_t it1 = it0 + items_per_cta < total_items ? it0 + items_per_cta : total_items;
    if (it0 >= it1) return;
    const int C = CHUNKED ? ea.chunk_cols : NT;
    const int64_t gap = CHUNKED ? ea.chunk_gap : 0;
    auto item_base = [&](int64_t item) {
        const int fi = int(item / n_tiles);
        return ring_base(fi, int(item - int64_t(fi) * n_tiles), n_tiles, NT, C);
    };
    auto fetch = [&](int64_t item, int st) {
        const cplx* g = src + item_base(item);
        cplx* d = smem + st * ITEM;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int e = j * NTHR + tid;
            cp_async16(d + ring_slot<L>(e >> 3, e & 7), g + e + (CHUNKED ? int64_t((e >> 3) / C) * gap : 0));
        }
    };
    int f = int(it0 / n_tiles), tile = int(it0 - int64_t(f) * n_tiles);
    // The first item's ring table and frequency constants are requested
    // before the item prefetches (as the oldest cp.async group and register
    // loads), so they do not queue behind the field traffic of every CTA;
    // later frequencies load them at the switch.
    for (int e = tid; e < E; e += NTHR) cp_async16(T + e, table + int64_t(f) * E + e);
    cp_async_commit();
    double fk0 = fdev[f].k0;
    cplx fcy = fdev[f].cy_rhs;
    griddep_wait();                                 // the field belongs to the previous sweep until here
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (it0 + p < it1) fetch(it0 + p, p);
        cp_async_commit();
    }
    int cur_f = -1;
    int slot = 0;
    cplx rho = czero(), inv_wrap = czero(), scale = czero(), b1 = czero(), b2 = czero();
    bool diagonal = false;
    for (int64_t item = it0; item < it1; ++item) {
        __syncthreads();                            // previous item's stage fully stored
        if (item == it1 - 1) griddep_launch();      // last item: the next sweep may start launching
        const bool new_f = f != cur_f;
        if (new_f && cur_f >= 0) {
            for (int e = tid; e < E; e += NTHR) T[e] = table[int64_t(f) * E + e];
            fk0 = fdev[f].k0;
            fcy = fdev[f].cy_rhs;
        }
        {
            const int64_t ip = item + STAGES - 1;
            if (ip < it1) fetch(ip, (slot + STAGES - 1) % STAGES);
            cp_async_commit();
            cp_async_wait<STAGES - 1>();            // also the first frequency's table (the oldest group)
        }
        __syncthreads();                            // item's lines (and a new table) visible to every warp
        if (new_f) {
            cur_f = f;
            rho = T[0];
            scale = T[1];
            inv_wrap = T[2];
            diagonal = T[3].re != 0.0;
            const cplx alpha = crmul(azimuth_scale(fk0, r_new, delta_theta), fcy);
            b2 = cmul(scale, alpha);
            b1 = csub(scale, cadd(b2, b2));
        }
        cplx* stg = smem + slot * ITEM;
        cplx v[RT][L];
#pragma unroll
        for (int h = 0; h < RT; ++h)
#pragma unroll
            for (int k = 0; k < L; ++k) v[h][k] = stg[(m0 + k) * 8 + ((warp * RT + h) ^ swz)];

        if (!diagonal) {
            // ---- forward cyclic recurrence w_m = v_m + rho w_{m-1}
            cplx Y[RT];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                Y[h] = czero();
#pragma unroll
                for (int k = 0; k < L; ++k) { Y[h] = cfma(rho, Y[h], v[h][k]); v[h][k] = Y[h]; }
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const cplx m = lane >= d ? qp[d] : czero();
#pragma unroll
                for (int h = 0; h < RT; ++h) Y[h] = cfma(m, shfl_up(Y[h], d), Y[h]);
            }
            const cplx qpq = qp[q];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                cplx ex = shfl_up(Y[h], 1);
                if (lane == 0) ex = czero();
                const cplx w_last = cmul(shfl_idx(Y[h], 31), inv_wrap);   // cyclic closure
                const cplx c_in = cfma(qpq, w_last, ex);
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[k + 1], c_in, v[h][k]);
            }
            // ---- backward cyclic recurrence x_m = w_m + rho x_{m+1}
            cplx X[RT];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                X[h] = czero();
#pragma unroll
                for (int k = L - 1; k >= 0; --k) { X[h] = cfma(rho, X[h], v[h][k]); v[h][k] = X[h]; }
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const cplx m = lane + d < 32 ? qp[d] : czero();
#pragma unroll
                for (int h = 0; h < RT; ++h) X[h] = cfma(m, shfl_down(X[h], d), X[h]);
            }
            const cplx qup = qp[31 - q];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                cplx nx = shfl_down(X[h], 1);
                if (lane == 31) nx = czero();
                const cplx x0 = cmul(shfl_idx(X[h], 0), inv_wrap);       // cyclic closure
                const cplx c_up = cfma(qup, x0, nx);
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[L - k], c_up, v[h][k]);
            }
        }
        // ---- boundary (surface and pad rows), TL / snapshot / final, next temp
        const int l0 = tile * 8 + warp * RT;
#pragma unroll
        for (int h = 0; h < RT; ++h) {
            const int l = l0 + h;
            if (l + ea.row_offset == 0 || l >= n_depth) {
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = czero();
            }
            if (l < n_depth && (ea.tl || ea.snap || ea.final_out)) {
                long long zeros = 0;
#pragma unroll
                for (int k = 0; k < L; ++k) {
                    const int m = m0 + k;
                    const cplx uf = cmul(scale, v[h][k]);
                    const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * NT * n_depth + (int64_t(m) * n_depth + l);
                    if (ea.tl) {
                        const double mag = cabs(uf) * ea.w_abs[f];
                        if (mag == 0.0) ++zeros;
                        ea.tl[so] = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
                    }
                    if (ea.snap) stc(ea.snap + so, uf);
                    if (ea.final_out) stc(ea.final_out + (int64_t(f) * NT + m) * n_depth + l, uf);
                }
                if (ea.tl && zeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), (unsigned long long)zeros);
            }
            if (ea.write_temp) {
                cplx prev = shfl_up(v[h][L - 1], 1), next = shfl_down(v[h][0], 1);
                const cplx wrap_prev = shfl_idx(v[h][L - 1], 31), wrap_next = shfl_idx(v[h][0], 0);
                if (lane == 0) prev = wrap_prev;
                if (lane == 31) next = wrap_next;
                const int r = (warp * RT + h) ^ swz;
#pragma unroll
                for (int k = 0; k < L; ++k) {
                    const cplx um = k ? v[h][k - 1] : prev;
                    const cplx up = (k + 1 < L) ? v[h][(k + 1) % L] : next;
                    stg[(m0 + k) * 8 + r] = cfma(b1, v[h][k], cmul(b2, cadd(up, um)));   // own slots only
                }
            }
        }
        if (ea.write_temp) {
            __syncthreads();                        // every warp's rows written
            cplx* g = dst + item_base(item);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int e = j * NTHR + tid;
                if (PEER) stc_stream(peer_elem(ea, e >> 3, tile, e & 7), stg[ring_slot<L>(e >> 3, e & 7)]);
                else stc_stream(g + e + (CHUNKED ? int64_t((e >> 3) / C) * gap : 0), stg[ring_slot<L>(e >> 3, e & 7)]);
            }
        }
        if (++tile == n_tiles) { tile = 0; ++f; }
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

// Wide rings (n_theta = CL * 32L, CL = 2..16): one thread-block cluster per
// (frequency, depth tile) item.  CTA s of the cluster stages the contiguous
// segment of azimuths [s*32L, (s+1)*32L) of the item's 8 rows (coalesced
// cp.async into the swizzled stage of k_azimuth_warp) and runs the same
// ring-per-warp solve on it with zero carry-in.  The segments are joined by
// two DSMEM exchanges of per-row segment totals, combined with Horner in
// R = rho^(32L):
//   forward  w entering segment s = sum_{s'<s} R^(s-1-s') W_s'
//                                  + R^s * (sum_s' R^(CL-1-s') W_s') / (1 - rho^N)
//   backward x entering from the right = sum_{s'>s} R^(s'-s-1) X_s'
//                                  + R^(CL-1-s) * (sum_s' R^s' X_s') / (1 - rho^N)
// and the epilogue's neighbours across segment edges follow from the
// recurrences themselves: x_(m-1) = w_(m-1) + rho x_m, x_(m+32L) = the right
// carry.  The totals are pushed with st.async into every peer's table and
// counted on the peer's mbarrier (no cluster-wide barrier, hence no GPU-scope
// fence behind the streaming stores, inside the item loop); the tables are
// double-buffered by item parity, which is race free because a CTA can only
// start item i+2 after every peer has sent its item i+1 totals, i.e. after
// every peer has finished reading item i.  Persistent: every CTA of a
// cluster walks the same item range.
template <int L, int RT, int STAGES>
__global__ void __launch_bounds__(32 * 8 / RT, (L == 8 ? 3 : 2))
k_azimuth_cluster(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ table, int E,
                  const FreqDev* __restrict__ fdev, int n_theta, int n_tiles, int n_depth, int64_t total_items,
                  int items_per_cluster, double r_new, double delta_theta, EpilogueArgs ea) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = int(cluster.num_blocks());
    const int s = int(cluster.block_rank());
    constexpr int NS = 32 * L;                      // segment length
    constexpr int ITEM = NS * 8;                    // elements per segment of an item
    constexpr int NTHR = 32 * 8 / RT;
    constexpr int PER = ITEM / NTHR;
    constexpr int TE = RING_HDR + (L + 1) + 33;     // table entries used: header, rho^0..L, R^0..32
    extern __shared__ cplx smem[];
    cplx* T = smem + STAGES * ITEM;
    cplx* segW = T + TE;                            // [2][16][8] forward totals of every segment
    cplx* segX = segW + 2 * 16 * 8;                 // [2][16][8] backward totals
    cplx* Rp = segX + 2 * 16 * 8;                   // [17] R^k, k = 0..16
    uint64_t* bars = reinterpret_cast<uint64_t*>(Rp + 17);   // [0..1] forward, [2..3] backward
    const cplx* pw = T + RING_HDR;
    const cplx* qp = pw + L + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane, swz = q & 7;
    const int m0 = q * L;
    const int mseg = s * NS;

    const int64_t it0 = int64_t(blockIdx.x / CL) * items_per_cluster;
    const int64_t it1 = it0 + items_per_cluster < total_items ? it0 + items_per_cluster : total_items;
    if (it0 >= it1) return;                         // uniform over the cluster
    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) mbar_init(&bars[b], 1);
        mbar_fence_init();
    }
    cluster_barrier();                              // peers' barriers initialised before any st.async
    const unsigned exch_bytes = unsigned(CL) * 8 * sizeof(cplx);
    // push this segment's per-row value to table[buf][s][row] of every peer (lane j -> rank j)
    auto push = [&](cplx* table_, uint64_t* bar, int row, cplx val) {
        if (lane < CL) st_async_cplx(mapa_shared(smem_addr(table_ + s * 8 + row), lane), val,
                                     mapa_shared(smem_addr(bar), lane));
    };
    const int C = ea.chunk_cols ? ea.chunk_cols : n_theta;
    const int64_t gap = ea.chunk_gap;
    auto item_base = [&](int64_t item) {
        const int fi = int(item / n_tiles);
        return ring_base(fi, int(item - int64_t(fi) * n_tiles), n_tiles, n_theta, C);
    };
    auto goff = [&](int e) -> int64_t {
        const int ge = s * ITEM + e;
        return ge + (gap ? int64_t((ge >> 3) / C) * gap : 0);
    };
    auto fetch = [&](int64_t item, int st) {
        cplx* d = smem + st * ITEM;
        if (gap == 0) {                             // standard layout: the segment is contiguous
            const cplx* g = src + item_base(item) + s * ITEM + tid;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int e = j * NTHR + tid;
                cp_async16(d + ring_slot<L>(e >> 3, e & 7), g + j * NTHR);
            }
        } else {
            const cplx* g = src + item_base(item);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int e = j * NTHR + tid;
                cp_async16(d + ring_slot<L>(e >> 3, e & 7), g + goff(e));
            }
        }
    };
    griddep_wait();                                 // the field belongs to the previous sweep until here
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (it0 + p < it1) fetch(it0 + p, p);
        cp_async_commit();
    }
    int f = int(it0 / n_tiles), tile = int(it0 - int64_t(f) * n_tiles);
    int cur_f = -1;
    int slot = 0;
    cplx rho = czero(), R = czero(), inv_wrap = czero(), scale = czero(), b1 = czero(), b2 = czero();
    cplx Rs = cone(), Rr = cone();                  // R^s, R^(CL-1-s)
    bool diagonal = false;
    for (int64_t item = it0; item < it1; ++item) {
        if (item == it1 - 1) griddep_launch();      // last item: the next sweep may start launching
        const int kk = int(item - it0);
        const int buf = kk & 1;
        const unsigned par = unsigned(kk >> 1) & 1u;
        cplx* tW = segW + buf * 128;
        cplx* tX = segX + buf * 128;
        __syncthreads();                            // previous item's stage fully stored
        if (tid == 0) {
            mbar_expect_tx(&bars[buf], exch_bytes);
            mbar_expect_tx(&bars[2 + buf], exch_bytes);
        }
        if (f != cur_f) {
            for (int e = tid; e < TE; e += NTHR) T[e] = table[int64_t(f) * E + e];
            __syncthreads();
            cur_f = f;
            rho = T[0];
            scale = T[1];
            inv_wrap = T[2];
            diagonal = T[3].re != 0.0;
            R = qp[32];
            if (tid == 0) {
                cplx p = cone();
                for (int k = 0; k <= 16; ++k) { Rp[k] = p; p = cmul(p, R); }
            }
            __syncthreads();
            Rs = Rp[s];
            Rr = Rp[CL - 1 - s];
            const FreqDev fd = fdev[f];
            const cplx alpha = crmul(azimuth_scale(fd.k0, r_new, delta_theta), fd.cy_rhs);
            b2 = cmul(scale, alpha);
            b1 = csub(scale, cadd(b2, b2));
        }
        {
            const int64_t ip = item + STAGES - 1;
            if (ip < it1) fetch(ip, (slot + STAGES - 1) % STAGES);
            cp_async_commit();
            cp_async_wait<STAGES - 1>();
        }
        __syncthreads();                            // item's lines visible to every warp
        cplx* stg = smem + slot * ITEM;
        cplx v[RT][L];
#pragma unroll
        for (int h = 0; h < RT; ++h)
#pragma unroll
            for (int k = 0; k < L; ++k) v[h][k] = stg[(m0 + k) * 8 + ((warp * RT + h) ^ swz)];

        cplx prev_edge[RT], next_edge[RT];         // x at mseg-1 and mseg+NS (cyclic)
        if (!diagonal) {
            // ---- forward recurrence w_m = v_m + rho w_{m-1} on the segment, zero carry-in
            cplx Y[RT];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                Y[h] = czero();
#pragma unroll
                for (int k = 0; k < L; ++k) { Y[h] = cfma(rho, Y[h], v[h][k]); v[h][k] = Y[h]; }
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const cplx m = lane >= d ? qp[d] : czero();
#pragma unroll
                for (int h = 0; h < RT; ++h) Y[h] = cfma(m, shfl_up(Y[h], d), Y[h]);
            }
#pragma unroll
            for (int h = 0; h < RT; ++h) push(tW, &bars[buf], warp * RT + h, shfl_idx(Y[h], 31));
            mbar_wait_cluster(&bars[buf], par);     // every segment's forward totals
            // half-warp hh = lane/16 serves row warp*RT+hh; its lane j < CL weighs
            // segment j's total by its power of R; a 4-level butterfly sums
            cplx carry_w[RT];
            {
                const int hh = lane >> 4, j = lane & 15;
                const bool use = j < CL && hh < RT;
                const cplx w = use ? tW[j * 8 + warp * RT + (hh < RT ? hh : 0)] : czero();
                cplx cin = (use && j < s) ? cmul(Rp[j < s ? s - 1 - j : 0], w) : czero();
                cplx wend = use ? cmul(Rp[j < CL ? CL - 1 - j : 0], w) : czero();
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    cin = cadd(cin, shfl_xor(cin, o));
                    wend = cadd(wend, shfl_xor(wend, o));
                }
                const cplx cw = cfma(Rs, cmul(wend, inv_wrap), cin);      // w_(mseg-1), cyclic
#pragma unroll
                for (int h = 0; h < RT; ++h) carry_w[h] = shfl_idx(cw, 16 * h);
            }
            const cplx qpq = qp[q];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                cplx ex = shfl_up(Y[h], 1);
                if (lane == 0) ex = czero();
                const cplx c_in = cfma(qpq, carry_w[h], ex);
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[k + 1], c_in, v[h][k]);
            }
            // ---- backward recurrence x_m = w_m + rho x_{m+1}, zero carry-in
            cplx X[RT];
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                X[h] = czero();
#pragma unroll
                for (int k = L - 1; k >= 0; --k) { X[h] = cfma(rho, X[h], v[h][k]); v[h][k] = X[h]; }
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const cplx m = lane + d < 32 ? qp[d] : czero();
#pragma unroll
                for (int h = 0; h < RT; ++h) X[h] = cfma(m, shfl_down(X[h], d), X[h]);
            }
#pragma unroll
            for (int h = 0; h < RT; ++h) push(tX, &bars[2 + buf], warp * RT + h, shfl_idx(X[h], 0));
            mbar_wait_cluster(&bars[2 + buf], par);
            const cplx qup = qp[31 - q];
            cplx carry_xr[RT];
            {
                const int hh = lane >> 4, j = lane & 15;
                const bool use = j < CL && hh < RT;
                const cplx xs = use ? tX[j * 8 + warp * RT + (hh < RT ? hh : 0)] : czero();
                cplx dn = (use && j > s) ? cmul(Rp[(j > s && j < CL) ? j - s - 1 : 0], xs) : czero();
                cplx x0 = use ? cmul(Rp[j < CL ? j : 0], xs) : czero();
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    dn = cadd(dn, shfl_xor(dn, o));
                    x0 = cadd(x0, shfl_xor(x0, o));
                }
                const cplx cx = cfma(Rr, cmul(x0, inv_wrap), dn);         // x_(mseg+NS), cyclic
#pragma unroll
                for (int h = 0; h < RT; ++h) carry_xr[h] = shfl_idx(cx, 16 * h);
            }
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                const cplx carry_x = carry_xr[h];
                cplx nx = shfl_down(X[h], 1);
                if (lane == 31) nx = czero();
                const cplx c_up = cfma(qup, carry_x, nx);
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[L - k], c_up, v[h][k]);
                next_edge[h] = carry_x;
                prev_edge[h] = cfma(rho, shfl_idx(v[h][0], 0), carry_w[h]);   // x_(mseg-1) = w + rho x_mseg
            }
        } else {
            // off == 0 (B = diag I): x = v; the edges are the neighbours' raw values
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                push(tW, &bars[buf], warp * RT + h, shfl_idx(v[h][L - 1], 31));
                push(tX, &bars[2 + buf], warp * RT + h, shfl_idx(v[h][0], 0));
            }
            mbar_wait_cluster(&bars[buf], par);
            mbar_wait_cluster(&bars[2 + buf], par);
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                prev_edge[h] = tW[((s + CL - 1) % CL) * 8 + warp * RT + h];
                next_edge[h] = tX[((s + 1) % CL) * 8 + warp * RT + h];
            }
        }
        // ---- boundary (surface and pad rows), TL / snapshot / final, next temp
        const int l0 = tile * 8 + warp * RT;
#pragma unroll
        for (int h = 0; h < RT; ++h) {
            const int l = l0 + h;
            if (l + ea.row_offset == 0 || l >= n_depth) {
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = czero();
                prev_edge[h] = czero();
                next_edge[h] = czero();
            }
            if (l < n_depth && (ea.tl || ea.snap || ea.final_out)) {
                long long zeros = 0;
#pragma unroll
                for (int k = 0; k < L; ++k) {
                    const int m = mseg + m0 + k;
                    const cplx uf = cmul(scale, v[h][k]);
                    const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth +
                                       (int64_t(m) * n_depth + l);
                    if (ea.tl) {
                        const double mag = cabs(uf) * ea.w_abs[f];
                        if (mag == 0.0) ++zeros;
                        ea.tl[so] = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
                    }
                    if (ea.snap) stc(ea.snap + so, uf);
                    if (ea.final_out) stc(ea.final_out + (int64_t(f) * n_theta + m) * n_depth + l, uf);
                }
                if (ea.tl && zeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), (unsigned long long)zeros);
            }
            if (ea.write_temp) {
                cplx prev = shfl_up(v[h][L - 1], 1), next = shfl_down(v[h][0], 1);
                if (lane == 0) prev = prev_edge[h];
                if (lane == 31) next = next_edge[h];
                const int r = (warp * RT + h) ^ swz;
#pragma unroll
                for (int k = 0; k < L; ++k) {
                    const cplx um = k ? v[h][k - 1] : prev;
                    const cplx up = (k + 1 < L) ? v[h][(k + 1) % L] : next;
                    stg[(m0 + k) * 8 + r] = cfma(b1, v[h][k], cmul(b2, cadd(up, um)));   // own slots only
                }
            }
        }
        if (ea.write_temp) {
            __syncthreads();                        // every warp's rows written
            if (ea.peer[0]) {                       // fused transpose: straight into the owners' inputs
#pragma unroll
                for (int jj = 0; jj < PER; ++jj) {
                    const int e = jj * NTHR + tid;
                    stc_stream(peer_elem(ea, mseg + (e >> 3), tile, e & 7), stg[ring_slot<L>(e >> 3, e & 7)]);
                }
            } else if (gap == 0) {
                cplx* g = dst + item_base(item) + s * ITEM + tid;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const int e = j * NTHR + tid;
                    stc_stream(g + j * NTHR, stg[ring_slot<L>(e >> 3, e & 7)]);
                }
            } else {
                cplx* g = dst + item_base(item);
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const int e = j * NTHR + tid;
                    stc_stream(g + goff(e), stg[ring_slot<L>(e >> 3, e & 7)]);
                }
            }
        }
        if (++tile == n_tiles) { tile = 0; ++f; }
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
    cluster_barrier();                              // no CTA leaves while peers may still address it
}

// ------------------------------------- TMA azimuth sweep (warp-specialised)
// The Blackwell form of k_azimuth_warp / k_azimuth_cluster for the standard
// field layout: one producer warp moves whole ring segments with the tensor
// engine (TMA load of segment n+S while the consumer warps solve segment n,
// TMA store of the solved temp straight from the stage), the 8/RT consumer
// warps run the ring-per-warp solve of k_azimuth_warp on their RT rows, and
// stage slots are handed over by full/empty mbarriers -- no CTA-wide barrier
// and no per-thread copies in the item loop.
//
// Stage layout of one segment (NS = 32L azimuths x 8 rows): the 128-B line
// k*32 + q holds azimuth m = q*L + k (lane q's k-th point) with its row r at
// 16-B chunk r ^ (q & 7).  The 5-D tensor map {16 doubles, q: 32 (stride
// L*128 B), k: L (stride 128 B), segment (stride NS*128 B), item (stride
// n_theta*128 B)} with box {16, 32, L, 1, 1} and the 128-B swizzle writes
// exactly this transposed layout, so the lane-per-chunk reads (fixed k,
// q = 0..31) hit 8 distinct chunks per 8-lane phase: conflict free.  The
// ring table of the item's (step, frequency) rides along into a per-slot
// table on the same mbarrier (tab_elems entries: header, rho^0..L, and the
// R^j run the solve reads).
//
// CLUSTER (rings of CL*NS points): CTA s of a cluster stages segment s and
// the segments are joined exactly as in k_azimuth_cluster, with one pair of
// exchange mbarriers per consumer warp (a warp's RT rows are exchanged only
// with the same warp of the peer CTAs), double-buffered by item parity.
__device__ __forceinline__ int tma_slot(int q, int k, int r) { return ((k * 32 + q) << 3) + (r ^ (q & 7)); }

//
// CORR (split long columns, LaunchCtx::split): the depth sweep left the
// zero-carry sub-column solutions x0; with every segment the producer also
// copies the exact carries cin/din of the item's (f, sub-column, segment)
// (k_split_carry, already in lane order) and the rows' unit-carry responses
// (a_l, q_l), and the consumers load x = x0 + a_l cin + q_l din.  (Measured
// and not kept: three extra "fixer" warps applying the correction to the
// staged segment in place, releasing it on a second mbarrier -- cfg5 azimuth
// sweep 149 -> 181 us; the fixers' pass lands on the item pipeline's path.)
//
// (Measured and not kept: half-tile items -- 4 rows, 64-B swizzle, two
// cluster CTAs per SM instead of one: cfg5 azimuth sweep 136 us either way,
// 147 -> 237 us with the split-column correction.)
template <int RT>
__host__ __device__ constexpr int ring_tma_threads() { return 32 * (8 / RT + 1); }

//
// HALO (with SEG): a segment of a longer ring whose carries only reach `span`
// points across its edges (|rho|^span below 1e-22 of them; the host picks the
// steps).  With the segment the producer loads halo_g 32-line granules of the
// neighbouring segments on either side (3-D map {16 doubles, azimuth, tile},
// box {16, 32, 1}, the same 128-B swizzle), and each consumer warp sums its row of
// them into the carries that the cluster kernel gets from its peers:
//   w at the point before the segment   = sum_(t>=0) rho^t v_(a-1-t),
//   x at the point after the segment    = [sum_(s>=0) rho^s v_(b+s) + rho w_(b-1)] / (1 - rho^2),
// so the segment is solved, its TL recorded and its next temp written in this one
// kernel on all SMs: no cluster, no carry kernel and no edge fix.
constexpr int RING_HALO_G = 3;                      // granules per side a slot can hold (span <= 96)

template <int L, int RT, int S, bool CLUSTER, int MINB, bool CORR = false, bool SEG = false, bool HALO = false>
__global__ void __launch_bounds__(ring_tma_threads<RT>(), MINB)
k_azimuth_tma(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_dst,
              const cplx* __restrict__ table, int E, int tab_elems, int n_theta, int n_tiles, int n_depth,
              int64_t total_items, int n_units, EpilogueArgs ea, const cplx* __restrict__ sp_cd,
              const cplx* __restrict__ sp_aq, const cplx* __restrict__ sp_pa, int split, int tile_perm,
              const __grid_constant__ CUtensorMap tm_fin, int fin_tma,
              const __grid_constant__ CUtensorMap tm_halo, int halo_g) {
    static_assert(!SEG || (!CLUSTER && RT == 1), "segmented rings: plain kernel, one row per warp");
    static_assert(HALO == SEG, "segmented rings take their carries from the halo");
    constexpr int HALO_SLOT = HALO ? 2 * RING_HALO_G * 256 : 0;   // cplx per slot: [side][granule][32 lines x 8 rows]
    namespace cg = cooperative_groups;
    constexpr int NW = 8 / RT;                      // consumer warps; warp NW is the TMA producer
    constexpr int NS = 32 * L;                      // segment length
    constexpr int ITEM = NS * 8;                    // elements per segment
    constexpr unsigned ITEM_BYTES = ITEM * sizeof(cplx);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    cplx* stage = reinterpret_cast<cplx*>(smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));
    const int tab_pad = (tab_elems + 7) & ~7;
    cplx* halo = stage + S * ITEM;                  // HALO: [S][2][RING_HALO_G][256], 1024-B aligned granules
    cplx* tabs = halo + S * HALO_SLOT;              // [S][tab_pad]
    // CORR: per slot the carries cin[NS], din[NS] of the item's (f, sub-column,
    // segment) and the (a_l, q_l) of its 8 rows, copied with every item (measured
    // faster than keeping one copy per run of items of a sub-column: 149 vs 158 us
    // at cfg5)
    constexpr int CORRE = CORR ? 2 * NS + 16 : 0;
    cplx* corr = tabs + S * tab_pad;                // [S][CORRE]
    cplx* segW = corr + S * CORRE;                  // cluster: [2][16][8] forward totals
    cplx* segX = segW + (CLUSTER ? 2 * 16 * 8 : 0); // cluster: [2][16][8] backward totals
    uint64_t* full = reinterpret_cast<uint64_t*>(segX + (CLUSTER ? 2 * 16 * 8 : 0));
    uint64_t* empty = full + S;
    uint64_t* xbar = empty + S;                     // cluster: [NW][4]: fwd buf 0/1, bwd buf 0/1
    int* need = reinterpret_cast<int*>(xbar + (CLUSTER ? 4 * NW : 0));   // CORR: [S] the slot's item is corrected
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int CL = 1, s = 0;
    if constexpr (CLUSTER) {
        cg::cluster_group cluster = cg::this_cluster();
        CL = int(cluster.num_blocks());
        s = int(cluster.block_rank());
    }
    // item indices fit an int (checked by the launcher): no 64-bit division in the loop.
    // CTA u of the plain kernel takes items u, u + G, u + 2G, ... (strided: at any time
    // the grid streams through one contiguous stretch of the field; cfg4 azimuth sweep
    // 100.8 -> 96.3 us against contiguous ranges; the ring table rides with every
    // item, so frequency switches cost nothing).  Cluster u takes the contiguous range
    // [u * per, (u + 1) * per) (strided measured 137 -> 148 us at cfg5).
    const int unit = CLUSTER ? int(blockIdx.x) / CL : int(blockIdx.x);
    const int G = CLUSTER ? 1 : n_units;
    const int first = CLUSTER ? unit * n_units : unit;
    if (first >= int(total_items)) return;          // uniform over a cluster
    const int N = CLUSTER ? min(n_units, int(total_items) - first) : (int(total_items) - unit + G - 1) / G;
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < S; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], NW);
        }
        if (CLUSTER)
            for (int b = 0; b < 4 * NW; ++b) mbar_init(&xbar[b], 1);
        mbar_fence_init();
    }
    if (CLUSTER) cluster_barrier();                 // peers' barriers initialised before any st.async
    else __syncthreads();

    if (warp == NW) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            griddep_wait();                         // the field belongs to the previous sweep until here
            const unsigned tab_bytes = unsigned(tab_elems) * unsigned(sizeof(cplx));
            int span_fs = -1, a_span = 0, q_span = 0;
            const int nseg = SEG ? n_theta / NS : 1;
            auto load = [&](int n, int slot) {
                const int item = (first + n * G) / nseg, seg = SEG ? (first + n * G) % nseg : s;
                const int f = item / n_tiles;
                const int titem = f * n_tiles + (item - f * n_tiles) * tile_perm % n_tiles;   // permuted tile
                bool corr_item = false;
                if constexpr (CORR) {
                    // rows [r0, r0 + 8) of the sub-column: inside a carry-response span?
                    const int tile = titem - f * n_tiles, tps = n_tiles / split;
                    const int sub = tile / tps, r0 = (tile - sub * tps) * 8;
                    const int fs = f * split + sub;
                    if (fs != span_fs) {
                        const cplx sp = ldc(sp_pa + 3 * fs + 2);
                        span_fs = fs;
                        a_span = int(sp.re);
                        q_span = int(sp.im);
                    }
                    corr_item = (sub > 0 && r0 < a_span) || (sub < split - 1 && r0 + 8 > tps * 8 - q_span);
                    need[slot] = corr_item ? 1 : 0;    // published by the arrive below (release)
                }
                const unsigned corr_bytes = corr_item ? CORRE * unsigned(sizeof(cplx)) : 0u;
                const unsigned halo_bytes = HALO ? 2u * unsigned(halo_g) * 4096u : 0u;
                mbar_expect_tx(&full[slot], ITEM_BYTES + tab_bytes + corr_bytes + halo_bytes);
                tma_load_5d(stage + slot * ITEM, &tm_src, 0, 0, 0, seg, titem, &full[slot]);
                if constexpr (HALO) {
                    cplx* hs = halo + slot * HALO_SLOT;
                    for (int g = 0; g < halo_g; ++g) {
                        int lo = seg * NS - 32 * (g + 1), hi = (seg + 1) * NS + 32 * g;   // cyclic
                        if (lo < 0) lo += n_theta;
                        if (hi >= n_theta) hi -= n_theta;
                        tma_load_3d(hs + g * 256, &tm_halo, 0, lo, titem, &full[slot]);
                        tma_load_3d(hs + (RING_HALO_G + g) * 256, &tm_halo, 0, hi, titem, &full[slot]);
                    }
                }
                bulk_load(tabs + slot * tab_pad, table + int64_t(f) * E, tab_bytes, &full[slot]);
                if (CORR && corr_item) {
                    const int tile = titem - f * n_tiles;
                    const int sub = tile / (n_tiles / split);
                    const cplx* cd = sp_cd + (int64_t(f) * split + sub) * 2 * n_theta + seg * NS;
                    cplx* dstc = corr + slot * CORRE;
                    bulk_load(dstc, cd, NS * unsigned(sizeof(cplx)), &full[slot]);
                    bulk_load(dstc + NS, cd + n_theta, NS * unsigned(sizeof(cplx)), &full[slot]);
                    bulk_load(dstc + 2 * NS, sp_aq + (int64_t(f) * n_tiles + tile) * 16, 16 * unsigned(sizeof(cplx)),
                              &full[slot]);
                }
            };
            for (int p = 0; p < S && p < N; ++p) load(p, p);
            for (int n = 0; n < N; ++n) {
                const int slot = n % S;
                mbar_wait(&empty[slot], unsigned(n / S) & 1u);      // consumers wrote the temp (or are done)
                if (!CLUSTER && fin_tma) {
                    // last step: the slot holds the final slab's tile (reference layout via tm_fin)
                    const int item = first + n * G, f = item / n_tiles;
                    tma_store_5d(&tm_fin, 0, 0, 0, (item - f * n_tiles) * tile_perm % n_tiles, f, stage + slot * ITEM);
                    bulk_commit();
                } else if (ea.write_temp) {
                    const int item = (first + n * G) / nseg, seg = SEG ? (first + n * G) % nseg : s;
                    const int f = item / n_tiles;
                    tma_store_5d(&tm_dst, 0, 0, 0, seg, f * n_tiles + (item - f * n_tiles) * tile_perm % n_tiles,
                                 stage + slot * ITEM);
                    bulk_commit();
                }
                if (n + S < N) {
                    bulk_wait_read<0>();            // the store has left the slot
                    load(n + S, slot);
                }
            }
            bulk_wait_read<0>();
        }
        __syncwarp();
        griddep_launch();
    } else {
        // ------------------------------------------------ consumer warps
        const int q = lane;
        const int m0 = q * L, mseg = s * NS;
        const unsigned exch_bytes = unsigned(CL) * RT * unsigned(sizeof(cplx));
        auto push = [&](cplx* table_, uint64_t* bar, int row, cplx val) {
            if (lane < CL) st_async_cplx(mapa_shared(smem_addr(table_ + s * 8 + row), lane), val,
                                         mapa_shared(smem_addr(bar), lane));
        };
        const int nseg = SEG ? n_theta / NS : 1;
        for (int n = 0; n < N; ++n) {
            const int item = (first + n * G) / nseg, seg = SEG ? (first + n * G) % nseg : 0;
            const int f = item / n_tiles, tile = (item - f * n_tiles) * tile_perm % n_tiles;
            const int slot = n % S;
            const int buf = n & 1;
            const unsigned xpar = unsigned(n >> 1) & 1u;
            if (n == N - 1) griddep_launch();       // last item: the next sweep may start launching
            if (CLUSTER && lane == 0) {
                mbar_expect_tx(&xbar[warp * 4 + buf], exch_bytes);
                mbar_expect_tx(&xbar[warp * 4 + 2 + buf], exch_bytes);
            }
            mbar_wait(&full[slot], unsigned(n / S) & 1u);
            const cplx* T = tabs + slot * tab_pad;
            const cplx* pw = T + RING_HDR;          // rho^k, k = 0..L
            const cplx* qp = pw + L + 1;            // R^j, j = 0..32 (cluster: R^(32k) = qp[32k])
            const cplx rho = T[0], scale = T[1], inv_wrap = T[2], b1 = T[4], b2 = T[5];
            const bool diagonal = !SEG && T[3].re != 0.0;   // SEG: rho = 0 runs the general recurrences
            cplx* stg = stage + slot * ITEM;
            cplx v[RT][L];
#pragma unroll
            for (int h = 0; h < RT; ++h)
#pragma unroll
                for (int k = 0; k < L; ++k) v[h][k] = stg[tma_slot(q, k, warp * RT + h)];
            if (CORR && need[slot]) {               // x = x0 + a_l cin + q_l din (split long columns)
                const cplx* cs = corr + slot * CORRE;
                const cplx* aq = cs + 2 * NS;
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    const cplx a = aq[2 * (warp * RT + h)], qr = aq[2 * (warp * RT + h) + 1];
#pragma unroll
                    for (int k = 0; k < L; ++k) v[h][k] = cfma(a, cs[k * 32 + q], cfma(qr, cs[NS + k * 32 + q], v[h][k]));
                }
            }

            cplx prev_edge[RT], next_edge[RT];     // cluster: x at mseg-1 and mseg+NS (cyclic)
            cplx halo_w = czero(), halo_x = czero();
            if constexpr (HALO) {
                // lane q reads line q of every granule (row `warp`): point t = 32 g + 31 - q before the
                // segment, s = 32 g + q after it; Horner over the granules, the lane's own power, lane sum
                const cplx* hs = halo + slot * HALO_SLOT;
                const int pos = (q << 3) + (warp ^ (q & 7));
                const cplx R32 = cmul(qp[32 / L], pw[32 % L]);
                const bool fix = CORR && need[slot];
                cplx a_l = czero(), q_l = czero();
                const cplx* cdb = sp_cd;
                if (fix) {
                    const cplx* aq = corr + slot * CORRE + 2 * NS;
                    a_l = aq[2 * warp];
                    q_l = aq[2 * warp + 1];
                    cdb = sp_cd + (int64_t(f) * split + tile / (n_tiles / split)) * 2 * n_theta;
                }
                for (int g = halo_g - 1; g >= 0; --g) {
                    cplx a = hs[g * 256 + pos], b = hs[(RING_HALO_G + g) * 256 + pos];
                    if (fix) {                      // the neighbours' raw points need the split-column carries too
                        int ma = seg * NS - 32 * (g + 1) + q, mb = (seg + 1) * NS + 32 * g + q;
                        if (ma < 0) ma += n_theta;
                        if (mb >= n_theta) mb -= n_theta;
                        const int ia = ma / NS * NS + (ma % L) * 32 + (ma % NS) / L;   // lane order within its segment
                        const int ib = mb / NS * NS + (mb % L) * 32 + (mb % NS) / L;
                        a = cfma(a_l, ldc(cdb + ia), cfma(q_l, ldc(cdb + n_theta + ia), a));
                        b = cfma(a_l, ldc(cdb + ib), cfma(q_l, ldc(cdb + n_theta + ib), b));
                    }
                    halo_w = cfma(R32, halo_w, a);
                    halo_x = cfma(R32, halo_x, b);
                }
                const int tl = 31 - q;
                halo_w = cmul(cmul(qp[tl / L], pw[tl % L]), halo_w);
                halo_x = cmul(cmul(qp[q / L], pw[q % L]), halo_x);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    halo_w = cadd(halo_w, shfl_xor(halo_w, o));
                    halo_x = cadd(halo_x, shfl_xor(halo_x, o));
                }
            }
            if (!diagonal) {
                // ---- forward cyclic recurrence w_m = v_m + rho w_{m-1}
                cplx Y[RT];
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    Y[h] = czero();
#pragma unroll
                    for (int k = 0; k < L; ++k) { Y[h] = cfma(rho, Y[h], v[h][k]); v[h][k] = Y[h]; }
                }
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const cplx m = lane >= d ? qp[d] : czero();
#pragma unroll
                    for (int h = 0; h < RT; ++h) Y[h] = cfma(m, shfl_up(Y[h], d), Y[h]);
                }
                cplx carry_w[RT];
                if constexpr (CLUSTER) {
                    cplx* tW = segW + buf * 128;
#pragma unroll
                    for (int h = 0; h < RT; ++h) push(tW, &xbar[warp * 4 + buf], warp * RT + h, shfl_idx(Y[h], 31));
                    mbar_wait_cluster(&xbar[warp * 4 + buf], xpar);
                    // half-warp hh serves row warp*RT+hh; lane j < CL weighs segment j's total
                    const int hh = lane >> 4, j = lane & 15;
                    const bool use = j < CL && hh < RT;
                    const cplx w = use ? tW[j * 8 + warp * RT + (hh < RT ? hh : 0)] : czero();
                    cplx cin = (use && j < s) ? cmul(qp[32 * (j < s ? s - 1 - j : 0)], w) : czero();
                    cplx wend = use ? cmul(qp[32 * (j < CL ? CL - 1 - j : 0)], w) : czero();
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        cin = cadd(cin, shfl_xor(cin, o));
                        wend = cadd(wend, shfl_xor(wend, o));
                    }
                    const cplx cw = cfma(qp[32 * s], cmul(wend, inv_wrap), cin);   // w_(mseg-1), cyclic
#pragma unroll
                    for (int h = 0; h < RT; ++h) carry_w[h] = shfl_idx(cw, 16 * h);
                } else if constexpr (HALO) {
                    carry_w[0] = halo_w;                    // w at the point before the segment
                } else {
#pragma unroll
                    for (int h = 0; h < RT; ++h) carry_w[h] = cmul(shfl_idx(Y[h], 31), inv_wrap);   // cyclic closure
                }
                const cplx qpq = qp[q];
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    cplx ex = shfl_up(Y[h], 1);
                    if (lane == 0) ex = czero();
                    const cplx c_in = cfma(qpq, carry_w[h], ex);
#pragma unroll
                    for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[k + 1], c_in, v[h][k]);
                }
                // ---- backward cyclic recurrence x_m = w_m + rho x_{m+1}
                cplx X[RT];
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    X[h] = czero();
#pragma unroll
                    for (int k = L - 1; k >= 0; --k) { X[h] = cfma(rho, X[h], v[h][k]); v[h][k] = X[h]; }
                }
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const cplx m = lane + d < 32 ? qp[d] : czero();
#pragma unroll
                    for (int h = 0; h < RT; ++h) X[h] = cfma(m, shfl_down(X[h], d), X[h]);
                }
                cplx carry_x[RT];
                if constexpr (CLUSTER) {
                    cplx* tX = segX + buf * 128;
#pragma unroll
                    for (int h = 0; h < RT; ++h) push(tX, &xbar[warp * 4 + 2 + buf], warp * RT + h, shfl_idx(X[h], 0));
                    mbar_wait_cluster(&xbar[warp * 4 + 2 + buf], xpar);
                    const int hh = lane >> 4, j = lane & 15;
                    const bool use = j < CL && hh < RT;
                    const cplx xs = use ? tX[j * 8 + warp * RT + (hh < RT ? hh : 0)] : czero();
                    cplx dn = (use && j > s) ? cmul(qp[32 * ((j > s && j < CL) ? j - s - 1 : 0)], xs) : czero();
                    cplx x0 = use ? cmul(qp[32 * (j < CL ? j : 0)], xs) : czero();
#pragma unroll
                    for (int o = 1; o < 16; o <<= 1) {
                        dn = cadd(dn, shfl_xor(dn, o));
                        x0 = cadd(x0, shfl_xor(x0, o));
                    }
                    const cplx cx = cfma(qp[32 * (CL - 1 - s)], cmul(x0, inv_wrap), dn);   // x_(mseg+NS), cyclic
#pragma unroll
                    for (int h = 0; h < RT; ++h) carry_x[h] = shfl_idx(cx, 16 * h);
                } else if constexpr (HALO) {
                    // x at the point after the segment: the halo's own forward sums closed by
                    // 1/(1 - rho^2), plus the segment's last w (carry applied above) carried through
                    carry_x[0] = cfma(T[7], shfl_idx(v[0][L - 1], 31), cmul(T[6], halo_x));
                } else {
#pragma unroll
                    for (int h = 0; h < RT; ++h) carry_x[h] = cmul(shfl_idx(X[h], 0), inv_wrap);    // cyclic closure
                }
                const cplx qup = qp[31 - q];
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    cplx nx = shfl_down(X[h], 1);
                    if (lane == 31) nx = czero();
                    const cplx c_up = cfma(qup, carry_x[h], nx);
#pragma unroll
                    for (int k = 0; k < L; ++k) v[h][k] = cfma(pw[L - k], c_up, v[h][k]);
                    if constexpr (CLUSTER || HALO) {
                        next_edge[h] = carry_x[h];
                        prev_edge[h] = cfma(rho, shfl_idx(v[h][0], 0), carry_w[h]);   // x_(mseg-1) = w + rho x_mseg
                    }
                }
            } else if constexpr (CLUSTER) {
                // off == 0 (B = diag I): x = v; the edges are the neighbours' raw values
                cplx* tW = segW + buf * 128;
                cplx* tX = segX + buf * 128;
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    push(tW, &xbar[warp * 4 + buf], warp * RT + h, shfl_idx(v[h][L - 1], 31));
                    push(tX, &xbar[warp * 4 + 2 + buf], warp * RT + h, shfl_idx(v[h][0], 0));
                }
                mbar_wait_cluster(&xbar[warp * 4 + buf], xpar);
                mbar_wait_cluster(&xbar[warp * 4 + 2 + buf], xpar);
#pragma unroll
                for (int h = 0; h < RT; ++h) {
                    prev_edge[h] = tW[((s + CL - 1) % CL) * 8 + warp * RT + h];
                    next_edge[h] = tX[((s + 1) % CL) * 8 + warp * RT + h];
                }
            }
            // ---- boundary (surface and pad rows), TL / snapshot / final, next temp
            const int l0 = tile * 8 + warp * RT;
#pragma unroll
            for (int h = 0; h < RT; ++h) {
                const int l = l0 + h;
                if (l + ea.row_offset == 0 || l >= n_depth) {
#pragma unroll
                    for (int k = 0; k < L; ++k) v[h][k] = czero();
                    if constexpr (CLUSTER || HALO) {
                        prev_edge[h] = czero();
                        next_edge[h] = czero();
                    }
                }
                if (l < n_depth && (ea.tl || ea.snap || ea.final_out)) {
                    long long zeros = 0;
#pragma unroll
                    for (int k = 0; k < L; ++k) {
                        const int m = (SEG ? seg * NS : mseg) + m0 + k;
                        const cplx uf = cmul(scale, v[h][k]);
                        if (!CLUSTER && fin_tma) stg[tma_slot(q, k, warp * RT + h)] = uf;   // stored by the producer's TMA
                        const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth +
                                           (int64_t(m) * n_depth + l);
                        if (ea.tl) {
                            const double mag = cabs(uf) * ea.w_abs[f];
                            if (mag == 0.0) ++zeros;
                            ea.tl[so] = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
                        }
                        if (ea.snap) stc(ea.snap + so, uf);
                        if (ea.final_out && (CLUSTER || !fin_tma)) stc(ea.final_out + (int64_t(f) * n_theta + m) * n_depth + l, uf);
                    }
                    if (ea.tl && zeros)
                        atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), (unsigned long long)zeros);
                }
                if (ea.write_temp) {
                    cplx prev = shfl_up(v[h][L - 1], 1), next = shfl_down(v[h][0], 1);
                    if constexpr (CLUSTER || HALO) {
                        if (lane == 0) prev = prev_edge[h];
                        if (lane == 31) next = next_edge[h];
                    } else {
                        const cplx wrap_prev = shfl_idx(v[h][L - 1], 31), wrap_next = shfl_idx(v[h][0], 0);
                        if (lane == 0) prev = wrap_prev;
                        if (lane == 31) next = wrap_next;
                    }
#pragma unroll
                    for (int k = 0; k < L; ++k) {
                        const cplx um = k ? v[h][k - 1] : prev;
                        const cplx up = (k + 1 < L) ? v[h][(k + 1) % L] : next;
                        stg[tma_slot(q, k, warp * RT + h)] = cfma(b1, v[h][k], cmul(b2, cadd(up, um)));   // own slots
                    }
                }
            }
            fence_proxy_async_smem();               // the temp is read by the TMA store (async proxy)
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    }
    if (CLUSTER) cluster_barrier();                 // no CTA leaves while peers may still address it
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
    const int row0 = (blockIdx.x % groups) * RW;
    const int f = blockIdx.y;
    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t rb = ring_base(f, tile, n_tiles, n_theta, ea.chunk_cols ? ea.chunk_cols : n_theta);
    cplx* tile_base = dst + rb;
    const cplx* src_tile = src + rb + row0 + i;
    cplx v[1][L];
#pragma unroll
    for (int k = 0; k < L; ++k)
        v[0][k] = (k < nvalid) ? ldc_stream(src_tile + ring_off(m0 + k, ea.chunk_cols, ea.chunk_gap)) : czero();
    cplx* T = smem + lay.table;
    for (int e = t; e < E; e += blockDim.x) T[e] = table[int64_t(f) * E + e];
    __syncthreads();
    ring_solve<L, RW, 1, false>(v, T, q, i, lane, warp, nwarps, n_theta, nvalid, smem + lay.sW, smem + lay.sV,
                                smem + lay.sTot);
    const int l = tile * 8 + row0 + i;
    if (l + ea.row_offset == 0 || l >= n_depth) {
#pragma unroll
        for (int k = 0; k < L; ++k) v[0][k] = czero();
    }
    const FreqDev fd = fdev[f];
    ring_epilogue<L, 1>(v, q, n_chunks, nvalid, i, RW, RW, m0, row0, tile * 8 + row0, ea, f, n_theta, n_depth,
                        T[1], fd.cy_rhs, azimuth_scale(fd.k0, r_new, delta_theta), smem + lay.sFirst,
                        smem + lay.sLast, tile_base, in_range);
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
    const int row0 = (blockIdx.x % groups) * RW;
    const int l = tile * 8 + row0 + i;
    const int f = blockIdx.y;
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r, delta_theta);
    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t tile_off = ring_base(f, tile, n_tiles, n_theta, ea.chunk_cols ? ea.chunk_cols : n_theta);
    cplx u[1][L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
        cplx v = czero();
        const int m = m0 + k;
        if (k < nvalid && l < n_depth) {
            v = src_tiled ? ldc(src + tile_off + ring_off(m, ea.chunk_cols, ea.chunk_gap) + row0 + i)
                          : ldc(src + (int64_t(f) * (ea.src_column ? 1 : n_theta) + (ea.src_column ? 0 : m)) * n_depth + l);
            if (l + ea.row_offset == 0 || (!ea.periodic && (m == 0 || m == n_theta - 1))) v = czero();
        }
        u[0][k] = v;
    }
    ring_epilogue<L, 1>(u, q, n_chunks, nvalid, i, RW, RW, m0, row0, tile * 8 + row0, ea, f, n_theta, n_depth,
                        cone(), fd.cy_rhs, s, sFirst, sLast, dst + tile_off, in_range);
}

// March prologue from the reference layout u0 [f][m][l] (depth fastest):
// boundary, the starting TL sample / snapshot, and the first temp = [1 +
// cy_rhs Y] u in the device tiles.  A CTA owns 32 azimuths x 64 depths of
// one frequency and stages them (plus one azimuth of halo either side) in
// shared memory, so u0 is read as 1 KB runs, TL is written as depth runs and
// the tiles as 4 KB runs.  Same arithmetic as ring_epilogue with scale 1.
constexpr int PREP_MB = 32, PREP_DB = 64;
__global__ void __launch_bounds__(256)
k_prepare(const cplx* __restrict__ u0, cplx* __restrict__ dst, const FreqDev* __restrict__ fdev, int n_theta,
          int n_tiles, int n_depth, double r, double delta_theta, EpilogueArgs ea) {
    __shared__ cplx sx[PREP_MB + 2][PREP_DB];
    __shared__ unsigned long long szeros;
    const int f = blockIdx.z;
    const int m0 = blockIdx.x * PREP_MB, l0 = blockIdx.y * PREP_DB;
    const int tid = threadIdx.x;
    const bool periodic = ea.periodic;
    if (tid == 0) szeros = 0;
    // stage azimuths m0-1 .. m0+MB (periodic wrap, zero exterior for a sector)
    for (int e = tid; e < (PREP_MB + 2) * PREP_DB; e += blockDim.x) {
        const int a = e / PREP_DB, dl = e % PREP_DB;
        int m = m0 - 1 + a;
        const int l = l0 + dl;
        bool ok = l < n_depth && l + ea.row_offset != 0;
        if (m < 0 || m >= n_theta) {
            if (periodic) m = (m + n_theta) % n_theta;
            else ok = false;
        }
        if (!periodic && (m == 0 || m == n_theta - 1)) ok = false;    // sector edges (marching.py:87-89)
        sx[a][dl] = ok ? ldc(u0 + (ea.src_column ? int64_t(f) * n_depth + l : (int64_t(f) * n_theta + m) * n_depth + l))
                       : czero();
    }
    __syncthreads();
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r, delta_theta);
    const cplx b2 = crmul(s, fd.cy_rhs);                     // scale 1: b2 = alpha, b1 = 1 - 2 alpha
    const cplx b1 = csub(cone(), cadd(b2, b2));
    // TL / snapshot / final in the reference layout: depth-fastest runs
    if (ea.tl || ea.snap || ea.final_out) {
        unsigned long long zeros = 0;
        for (int e = tid; e < PREP_MB * PREP_DB; e += blockDim.x) {
            const int a = e / PREP_DB, dl = e % PREP_DB;
            const int m = m0 + a, l = l0 + dl;
            if (l >= n_depth) continue;
            const cplx uf = sx[a + 1][dl];
            const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth + (int64_t(m) * n_depth + l);
            if (ea.tl) {
                const double mag = cabs(uf) * ea.w_abs[f];
                if (mag == 0.0) ++zeros;
                ea.tl[so] = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
            }
            if (ea.snap) stc(ea.snap + so, uf);
            if (ea.final_out) stc(ea.final_out + (int64_t(f) * n_theta + m) * n_depth + l, uf);
        }
        if (ea.tl && zeros) atomicAdd(&szeros, zeros);
    }
    // next temp into the device tiles: tile-major, 32 azimuths x 8 rows = 4 KB runs
    if (ea.write_temp) {
        cplx* base = dst + ring_base(f, 0, n_tiles, n_theta, n_theta);
        for (int e = tid; e < PREP_MB * PREP_DB; e += blockDim.x) {
            const int tl = e / (PREP_MB * 8), rem = e % (PREP_MB * 8);
            const int a = rem / 8, rr = rem % 8;
            const int dl = tl * 8 + rr;
            const int tile = (l0 + dl) >> 3;
            if (tile >= n_tiles) continue;
            const cplx um = sx[a][dl], uc = sx[a + 1][dl], up = sx[a + 2][dl];
            stc_stream(base + (int64_t(tile) * n_theta + m0 + a) * 8 + rr, cfma(b1, uc, cmul(b2, cadd(up, um))));
        }
    }
    __syncthreads();
    if (tid == 0 && szeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), szeros);
}

// March prologue for an azimuth-independent starter on a periodic ring
// (PE3D_FLAG_STARTER_COLUMN, the Gaussian starter of every drop-in march):
// u0 is one depth column per frequency, so the boundary, the TL sample and
// the first temp = [1 + cy_rhs Y] u are the same for every azimuth.  A CTA
// computes PREPC_ROWS rows of one frequency once (k_prepare's arithmetic with
// u_(m-1) = u_m = u_(m+1)) and streams them out: the temp as whole tiles
// (n_theta contiguous 128-B lines per tile), TL / snapshot / final as
// depth runs of every azimuth.  The prologue is pure write bandwidth
// (cfg4: 134 MB TL + 268 MB temp); k_prepare staged 34 x 64 input points
// per 32 x 64 outputs and ran at ~2 TB/s (199 us of the march at cfg4).
constexpr int PREPC_ROWS = 64;
__global__ void __launch_bounds__(256)
k_prepare_column(const cplx* __restrict__ u0, cplx* __restrict__ dst, const FreqDev* __restrict__ fdev, int n_theta,
                 int n_tiles, int n_depth, double r, double delta_theta, EpilogueArgs ea) {
    __shared__ cplx su[PREPC_ROWS], st[PREPC_ROWS];
    __shared__ double stl[PREPC_ROWS];
    __shared__ unsigned long long szeros;
    const int f = blockIdx.y, l0 = blockIdx.x * PREPC_ROWS, tid = threadIdx.x;
    const int rows = min(PREPC_ROWS, n_tiles * 8 - l0);            // rows of this block inside the tiles
    if (tid == 0) szeros = 0;
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r, delta_theta);
    const cplx b2 = crmul(s, fd.cy_rhs);                           // scale 1: b2 = alpha, b1 = 1 - 2 alpha
    const cplx b1 = csub(cone(), cadd(b2, b2));
    if (tid < PREPC_ROWS) {
        const int l = l0 + tid;
        const bool ok = tid < rows && l < n_depth && l + ea.row_offset != 0;
        const cplx u = ok ? ldc(u0 + int64_t(f) * n_depth + l) : czero();
        su[tid] = u;
        st[tid] = cfma(b1, u, cmul(b2, cadd(u, u)));               // periodic: both neighbours are u
        if (ea.tl && l < n_depth) {
            const double mag = cabs(u) * ea.w_abs[f];
            if (mag == 0.0) atomicAdd(&szeros, (unsigned long long)n_theta);
            stl[tid] = (mag == 0.0) ? TL_FLOOR_DB : -20.0 * log10(mag);
        }
    }
    __syncthreads();
    // first temp: one column per frequency for the first depth sweep (LaunchCtx::src_col) ...
    if (ea.write_temp && ea.temp_col) {
        if (tid < rows) ea.temp_col[(int64_t(f) * n_tiles * 8) + l0 + tid] = st[tid];
    } else if (ea.write_temp) {
        // ... or tiles [l0/8, l0/8 + rows/8), each n_theta lines of 8 rows
        cplx* base = dst + ring_base(f, 0, n_tiles, n_theta, n_theta) + int64_t(l0 / 8) * n_theta * 8;
        const int line_elems = n_theta * 8, n = (rows / 8) * line_elems;   // <= 2^18: 32-bit indices
        for (int e = tid; e < n; e += blockDim.x) stc_stream(base + e, st[(e / line_elems) * 8 + (e & 7)]);
    }
    // TL / snapshot / final in the reference layout [.][m][l]: depth runs of every azimuth
    const int dr = min(rows, n_depth - l0);
    if (dr > 0 && (ea.tl || ea.snap || ea.final_out)) {
        const int n = n_theta * dr;
        const int64_t so = (int64_t(f) * ea.n_samples + ea.sample) * n_theta * n_depth + l0;
        for (int e = tid; e < n; e += blockDim.x) {
            const int m = e / dr, dl = e - m * dr;
            const int64_t off = int64_t(m) * n_depth + dl;
            if (ea.tl) ea.tl[so + off] = stl[dl];
            if (ea.snap) stc(ea.snap + so + off, su[dl]);
            if (ea.final_out) stc(ea.final_out + int64_t(f) * n_theta * n_depth + l0 + off, su[dl]);
        }
    }
    __syncthreads();
    if (tid == 0 && szeros) atomicAdd(reinterpret_cast<unsigned long long*>(ea.clamped + f), szeros);
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

// Which azimuth kernel serves a ring of n_theta points, and its table layout.
struct RingPlan {
    int kind;          // 0: ring-per-warp, 1: block pipeline / direct
    int L, RW;
    RingLayout lay;
};

// Segment chunk of the cluster ring kernel: 16 (segments of 512 azimuths,
// one 8-warp CTA per SM, measured faster at cfg5) when n_theta allows it,
// else 8 (segments of 256, three 4-warp CTAs per SM).  PE3D_CLUSTER_L forces.
static int cluster_chunk(int n_theta) {
    const char* env = getenv("PE3D_CLUSTER_L");
    if (env) return atoi(env) == 16 ? 16 : 8;
    return (n_theta % 512 == 0 && n_theta / 512 >= 2) ? 16 : 8;
}

static RingPlan ring_plan(int n_theta) {
    RingPlan p;
    const bool block = getenv("PE3D_RING_BLOCK") != nullptr;
    // ring-per-warp kernels are instantiated for L = 2, 4, 8, 16 (see launch_azimuth_scan)
    const int Lw = n_theta / 32;
    if (n_theta % 32 == 0 && (Lw == 2 || Lw == 4 || Lw == 8 || Lw == 16) && !block) {
        p.kind = 0;
        p.L = n_theta / 32;
        p.RW = 1;
        p.lay = ring_layout(n_theta, p.L, 1);     // 32 chunks, qp[0..32]
        return p;
    }
    const int cl_L = cluster_chunk(n_theta);
    if (n_theta % (32 * cl_L) == 0 && n_theta / (32 * cl_L) >= 2 && n_theta / (32 * cl_L) <= 16 && !block) {
        p.kind = 2;                               // cluster of n_theta/(32L) segments
        p.L = cl_L;
        p.RW = 1;
        p.lay = ring_layout(n_theta, p.L, 1);     // qp[0..32] leads the R^j run
        return p;
    }
    p.kind = 1;
    ring_shape(n_theta, &p.L, &p.RW);
    p.lay = ring_layout(n_theta, p.L, p.RW);
    return p;
}

int ring_table_elems(int n_theta) { return ring_plan(n_theta).lay.E; }

int ring_segment(int n_theta) {
    const RingPlan p = ring_plan(n_theta);
    return (p.kind == 0 || p.kind == 2) ? 32 * p.L : 0;
}

cudaError_t launch_ring_setup(const LaunchCtx& c, cplx* table, int n_steps, int first_index, double r_start,
                              double delta_r) {
    const RingLayout lay = ring_plan(c.n_theta).lay;
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

// TMA ring maps over the standard field layout: {16 doubles, q: 32, k: L,
// segment: n_theta / (32L), item: F * n_tiles} (see k_azimuth_tma).
static bool ring_tensor_map(CUtensorMap* tm, const void* base, int n_theta, int L, int64_t tiles) {
    const int NS = 32 * L;
    const uint64_t dims[5] = {16, 32, uint64_t(L), uint64_t(n_theta / NS), uint64_t(tiles)};
    const uint64_t strides[4] = {uint64_t(L) * 128, 128, uint64_t(NS) * 128, uint64_t(n_theta) * 128};
    const uint32_t box[5] = {16, 32, uint32_t(L), 1, 1};
    return encode_swizzled_map(tm, base, 5, dims, strides, box, 128);
}

// Occupancy of a kernel configuration, cached per (kernel, device, smem bytes)
// in a small thread-safe table (the launchers run from several handles).
struct OccKey { const void* kern; int dev; size_t bytes; int cluster; };
int cached_occupancy(const void* kern, size_t bytes, int cluster, int nthr, cudaLaunchConfig_t* cfg) {
    static std::mutex mu;
    static OccKey keys[64];
    static int vals[64];
    static int n = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; ++i)
        if (keys[i].kern == kern && keys[i].dev == dev && keys[i].bytes == bytes && keys[i].cluster == cluster)
            return vals[i];
    int v = 0;
    cudaError_t e;
    if (cluster > 1) e = cudaOccupancyMaxActiveClusters(&v, kern, cfg);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, nthr, bytes);
    if (e != cudaSuccess || v < 1) return 0;
    if (n < 64) { keys[n] = OccKey{kern, dev, bytes, cluster}; vals[n] = v; ++n; }
    return v;
}

template <int L, int RT, int S, bool CLUSTER, int MINB = 1, bool CORR = false, bool SEG = false, bool HALO = false>
static cudaError_t launch_tma_ring(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, int E,
                                   const EpilogueArgs& ea, int span = 0) {
    constexpr int NS = 32 * L, NW = 8 / RT;
    const int CL = c.n_theta / NS;
    if (c.n_theta % NS != 0 || (CLUSTER ? (CL < 2 || CL > 16) : (SEG ? (CL < 2 || CL > 16) : CL != 1)))
        return cudaErrorNotSupported;
    const int halo_g = HALO ? (span + 31) / 32 : 0;
    if (HALO && (ea.final_out || halo_g < 1 || halo_g > RING_HALO_G)) return cudaErrorNotSupported;
    const int64_t tiles = int64_t(c.n_freq) * c.n_tiles;
    const int64_t items = SEG ? tiles * CL : tiles;
    if (items > 0x7fffffff) return cudaErrorNotSupported;
    CUtensorMap tm_src, tm_dst;
    if (!ring_tensor_map(&tm_src, src, c.n_theta, L, tiles) || !ring_tensor_map(&tm_dst, dst, c.n_theta, L, tiles))
        return cudaErrorNotSupported;
    CUtensorMap tm_halo = tm_dst;
    if (HALO) {                                     // 32-line granules of a tile's ring, same swizzle as the segments
        const uint64_t dims[3] = {16, uint64_t(c.n_theta), uint64_t(tiles)};
        const uint64_t strides[2] = {128, uint64_t(c.n_theta) * 128};
        const uint32_t box[3] = {16, 32, 1};
        if (!encode_swizzled_map(&tm_halo, src, 3, dims, strides, box, 128)) return cudaErrorNotSupported;
    }
    const int tab_elems = RING_HDR + L + 1 + (CLUSTER ? std::max(32, 32 * (CL - 1) + 1) : 32);
    if (tab_elems > E) return cudaErrorNotSupported;
    const int tab_pad = (tab_elems + 7) & ~7;
    const size_t corre = CORR ? 2 * NS + 16 : 0;    // per slot: the carries and the rows' (a_l, q_l)
    const size_t bytes = 1024 +
                         sizeof(cplx) * (size_t(S) * NS * 8 + size_t(S) * tab_pad + S * corre + (CLUSTER ? 512 : 0) +
                                         (HALO ? size_t(S) * 2 * RING_HALO_G * 256 : 0)) +
                         sizeof(uint64_t) * (2 * S + (CLUSTER ? 4 * NW : 0)) + sizeof(int) * S;
    if (bytes > 227 * 1024) return cudaErrorNotSupported;
    if (CORR && (c.split < 2 || c.n_tiles % c.split != 0 || !c.sp_cd || !c.sp_aq)) return cudaErrorNotSupported;
    auto kern = k_azimuth_tma<L, RT, S, CLUSTER, MINB, CORR, SEG, HALO>;
    cudaError_t e = set_smem(kern, bytes);
    if (e != cudaSuccess) return e;
    const int nthr = ring_tma_threads<RT>();
    if constexpr (!CLUSTER) {
        const int per_sm = cached_occupancy(reinterpret_cast<const void*>(kern), bytes, 1, nthr, nullptr);
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        const int64_t ctas = int64_t(c.num_sms) * per_sm;
        // few items (a chain of an 8-frequency shard): one item per CTA, where the
        // round-1 cp.async kernel's lighter CTAs share the SMs with the other chains'
        // sweeps better (8 frequencies, 8 chains: 30.9 -> 27.0 us per step; with more
        // items per CTA the TMA pipeline wins: 64 frequencies 101 -> 96 us per sweep)
        if (!CORR && !SEG && items <= 2 * ctas) return cudaErrorNotSupported;
        int per = int((items + ctas - 1) / ctas);
        if (items <= 2 * ctas) per = 1;               // few items: let the block scheduler balance the tail
        const int grid = int((items + per - 1) / per);
        // last step: the final slab leaves through the stage with one TMA store per item
        // (reference layout [f][m][l]: an item's 8 rows of azimuth m are one 128-B run)
        // instead of 16-B stores strided by n_depth (cfg4 last azimuth sweep 166-189 -> 97-99 us,
        // 20-step march 3945 -> 3841 us; bitwise the same slab)
        CUtensorMap tm_fin = tm_dst;
        int fin_tma = 0;
        if (ea.final_out && !ea.write_temp && c.n_depth % 8 == 0 && !getenv("PE3D_FINAL_STORES")) {
            const uint64_t NZb = uint64_t(c.n_depth) * 16;
            const uint64_t dims[5] = {16, 32, uint64_t(L), uint64_t(c.n_tiles), uint64_t(c.n_freq)};
            const uint64_t strides[4] = {uint64_t(L) * NZb, NZb, 128, uint64_t(c.n_theta) * NZb};
            const uint32_t box[5] = {16, 32, uint32_t(L), 1, 1};
            fin_tma = encode_swizzled_map(&tm_fin, ea.final_out, 5, dims, strides, box, 128) ? 1 : 0;
        }
        return launch_pdl(c.pdl != 0, kern, dim3(grid), dim3(nthr), bytes, c.stream, tm_src, tm_dst, table_step, E,
                          tab_elems, c.n_theta, c.n_tiles, c.n_depth, items, grid, ea, (const cplx*)c.sp_cd,
                          (const cplx*)c.sp_aq, (const cplx*)c.sp_pa, c.split, 1, tm_fin, fin_tma, tm_halo, halo_g);
    } else {
        if (CL > 8) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(nthr);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = c.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(CL * c.num_sms);
        const int resident = cached_occupancy(reinterpret_cast<const void*>(kern), bytes, CL, nthr, &cfg);
        if (resident < 1) return cudaErrorInvalidConfiguration;
        const int per = int((items + resident - 1) / resident);
        const int clusters = int((items + per - 1) / per);
        cfg.gridDim = dim3(clusters * CL);
        // split columns: the corrected tiles (near sub-column edges) are contiguous; a
        // coprime stride P through each frequency's tiles spreads them over the clusters'
        // contiguous item ranges (P ~ 0.618 n_tiles, gcd(P, n_tiles) = 1)
        int perm = 1;
        if (CORR) {
            auto gcd = [](int a, int b) { while (b) { const int t = a % b; a = b; b = t; } return a; };
            perm = int(0.618 * c.n_tiles) | 1;
            while (gcd(perm, c.n_tiles) != 1) perm += 2;
        }
        return cudaLaunchKernelEx(&cfg, kern, tm_src, tm_dst, table_step, E, tab_elems, c.n_theta, c.n_tiles,
                                  c.n_depth, items, per, ea, (const cplx*)c.sp_cd, (const cplx*)c.sp_aq,
                                  (const cplx*)c.sp_pa, c.split, perm, tm_dst, 0, tm_dst, 0);
    }
}

template <int L, int RT, int STAGES>
static cudaError_t launch_warp_ring(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, int E,
                                   double r_new, const EpilogueArgs& ea) {
    const bool chunked = ea.chunk_gap != 0 || (ea.chunk_cols != 0 && ea.chunk_cols != c.n_theta);
    auto kern = ea.peer[0] ? k_azimuth_warp<L, RT, STAGES, true, true>
                           : (chunked ? k_azimuth_warp<L, RT, STAGES, true> : k_azimuth_warp<L, RT, STAGES, false>);
    const int nthr = 32 * 8 / RT;
    const size_t bytes = sizeof(cplx) * (size_t(STAGES) * 32 * L * 8 + E);
    cudaError_t e = set_smem(kern, bytes);
    if (e != cudaSuccess) return e;
    int per_sm = int((227 * 1024) / (bytes + 1024));
    if (per_sm > 2048 / nthr) per_sm = 2048 / nthr;
    if (per_sm < 1) per_sm = 1;
    const int64_t items = int64_t(c.n_freq) * c.n_tiles;
    const int64_t ctas = int64_t(c.num_sms) * per_sm;
    // persistent CTAs walk several items with the next one prefetched; with at
    // most two items per resident CTA (few frequencies per GPU) one item per
    // CTA lets the block scheduler balance the tail instead
    // (cfg4, 8 frequencies per GPU: step 34.3 -> 33.9 us)
    int per = int((items + ctas - 1) / ctas);
    if (items <= 2 * ctas) per = 1;
    const int grid = int((items + per - 1) / per);
    return launch_pdl(c.pdl != 0, kern, dim3(grid), dim3(nthr), bytes, c.stream, src, dst, table_step, E, c.fdev,
                      c.n_tiles, c.n_depth, items, per, r_new, c.delta_theta, ea);
}

template <int L, int RT, int STAGES>
static cudaError_t launch_cluster_ring(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, int E,
                                       double r_new, const EpilogueArgs& ea) {
    auto kern = k_azimuth_cluster<L, RT, STAGES>;
    constexpr int NS = 32 * L;
    const int CL = c.n_theta / NS;
    const int nthr = 32 * 8 / RT;
    const size_t bytes = sizeof(cplx) * (size_t(STAGES) * NS * 8 + RING_HDR + (L + 1) + 33 + 4 * 128 + 17) + 4 * sizeof(uint64_t);
    cudaError_t e = set_smem(kern, bytes);
    if (e != cudaSuccess) return e;
    if (CL > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(nthr);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // persistent: as many clusters as can be co-resident (cached per kernel, device and smem size)
    cfg.gridDim = dim3(CL * c.num_sms);
    const int resident = cached_occupancy((const void*)kern, bytes, CL, nthr, &cfg);
    if (resident < 1) return cudaErrorInvalidConfiguration;
    const int64_t items = int64_t(c.n_freq) * c.n_tiles;
    const int per = int((items + resident - 1) / resident);
    const int clusters = int((items + per - 1) / per);
    cfg.gridDim = dim3(clusters * CL);
    // no PDL here: this persistent grid launched early is placed around the
    // depth sweep's retiring CTAs and loses co-residency (cfg5, 32 of 33
    // cluster slots: 309 -> 390 us per step)
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, src, dst, table_step, E, c.fdev, c.n_theta, c.n_tiles, c.n_depth, items, per,
                              r_new, c.delta_theta, ea);
}

// Halo form of the split-ring sweep: the carries come from `span` (<= 32 RING_HALO_G)
// points of the neighbouring segments loaded with every segment; TL and snapshots
// are recorded in the same kernel (not the final slab).
int sring_halo_max_span() { return 32 * RING_HALO_G; }
cudaError_t launch_azimuth_halo(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step,
                                const EpilogueArgs& ea, int span) {
    const RingPlan plan = ring_plan(c.n_theta);
    if (plan.kind != 2 || plan.L != 16 || !ea.periodic || ea.chunk_gap != 0 || ea.peer[0] || ea.row_offset != 0 ||
        (ea.chunk_cols != 0 && ea.chunk_cols != c.n_theta))
        return cudaErrorNotSupported;
    const int E = plan.lay.E;
    if (c.split >= 2) return launch_tma_ring<16, 1, 2, false, 1, true, true, true>(c, src, dst, table_step, E, ea, span);
    return launch_tma_ring<16, 1, 2, false, 1, false, true, true>(c, src, dst, table_step, E, ea, span);
}

cudaError_t launch_azimuth_scan(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, double r_new,
                                const EpilogueArgs& ea) {
    const RingPlan plan = ring_plan(c.n_theta);
    const bool standard = ea.chunk_gap == 0 && (ea.chunk_cols == 0 || ea.chunk_cols == c.n_theta) && !ea.peer[0] &&
                          ea.row_offset == 0;
    if (c.split >= 2) {
        // split long columns: only the TMA kernels apply the sub-column carries
        if (!standard || !ea.periodic) return cudaErrorNotSupported;
        const int E = plan.lay.E;
        if (plan.kind == 0 && plan.L == 8) return launch_tma_ring<8, 2, 2, false, 2, true>(c, src, dst, table_step, E, ea);
        if (plan.kind == 0 && plan.L == 16) return launch_tma_ring<16, 1, 2, false, 1, true>(c, src, dst, table_step, E, ea);
        if (plan.kind == 0 && plan.L == 4) return launch_tma_ring<4, 2, 3, false, 1, true>(c, src, dst, table_step, E, ea);
        if (plan.kind == 0 && plan.L == 2) return launch_tma_ring<2, 2, 3, false, 1, true>(c, src, dst, table_step, E, ea);
        if (plan.kind == 2 && plan.L == 16) return launch_tma_ring<16, 1, 2, true, 1, true>(c, src, dst, table_step, E, ea);
        if (plan.kind == 2 && plan.L == 8) return launch_tma_ring<8, 2, 2, true, 1, true>(c, src, dst, table_step, E, ea);
        return cudaErrorNotSupported;
    }
    if (standard && ea.periodic && (plan.kind == 0 || plan.kind == 2) && !getenv("PE3D_RING_CPASYNC")) {
        // TMA + warp-specialised sweep; falls through to the cp.async kernels
        // only when the tensor map cannot describe the ring
        cudaError_t e = cudaErrorNotSupported;
        const int E = plan.lay.E;
        if (plan.kind == 0) {
            switch (plan.L) {
                case 2: e = launch_tma_ring<2, 2, 3, false>(c, src, dst, table_step, E, ea); break;
                case 4: e = launch_tma_ring<4, 2, 3, false>(c, src, dst, table_step, E, ea); break;
                case 8: e = launch_tma_ring<8, 2, 3, false, 2>(c, src, dst, table_step, E, ea); break;   // 2 CTAs/SM
                case 16: e = launch_tma_ring<16, 1, 2, false>(c, src, dst, table_step, E, ea); break;
                default: break;
            }
        } else if (plan.L == 16) {
            e = launch_tma_ring<16, 1, 2, true>(c, src, dst, table_step, E, ea);
        } else {
            e = launch_tma_ring<8, 2, 2, true>(c, src, dst, table_step, E, ea);
        }
        if (e != cudaErrorNotSupported) return e;
    }
    if (plan.kind == 2 && ea.periodic) {
        // 512-azimuth segments: single-stage CTAs (64 KB, 128 registers), two per
        // SM, so the second CTA hides the first one's loads (measured faster at
        // cfg5 than one double-buffered CTA per SM)
        if (plan.L == 16) return launch_cluster_ring<16, 1, 1>(c, src, dst, table_step, plan.lay.E, r_new, ea);
        return launch_cluster_ring<8, 2, 2>(c, src, dst, table_step, plan.lay.E, r_new, ea);
    }
    if (plan.kind == 0 && ea.periodic) {
        const int E = plan.lay.E;
        switch (plan.L) {
            case 2: return launch_warp_ring<2, 2, 3>(c, src, dst, table_step, E, r_new, ea);
            case 4: return launch_warp_ring<4, 2, 3>(c, src, dst, table_step, E, r_new, ea);
            case 8: return launch_warp_ring<8, 2, 2>(c, src, dst, table_step, E, r_new, ea);
            case 16: return launch_warp_ring<16, 1, 2>(c, src, dst, table_step, E, r_new, ea);
            default: break;
        }
    }
    const int L = plan.L, RW = plan.RW;
    const RingLayout rl = plan.lay;
    const int nthreads = round32(RW * rl.n_chunks);
    const size_t stage_bytes = sizeof(cplx) * size_t(RW) * c.n_theta;
    if (RW == 8 && 2 * stage_bytes <= 110 * 1024 && ea.chunk_gap == 0 && !ea.peer[0]) {
        const int stages = (3 * stage_bytes <= 72 * 1024) ? 3 : 2;
        const int64_t items = int64_t(c.n_freq) * c.n_tiles;
        constexpr int RT = 2;
        const int nthr = round32((8 / RT) * rl.n_chunks);
        auto go = [&](auto kern, int Lv) -> cudaError_t {
            const int n_chunks = (c.n_theta + Lv - 1) / Lv;
            const size_t elems = size_t(stages) * RW * c.n_theta + rl.E + 2 * (nthr / 32) * RW + 2 * RW +
                                 2 * size_t(n_chunks) * RW;
            const size_t bytes = sizeof(cplx) * elems;
            cudaError_t e = set_smem(kern, bytes);
            if (e != cudaSuccess) return e;
            int per_sm = int((228 * 1024) / (bytes + 1024));
            if (per_sm > 2048 / nthr) per_sm = 2048 / nthr;
            if (per_sm < 1) per_sm = 1;
            const int64_t ctas = int64_t(c.num_sms) * per_sm;
            const int per = int((items + ctas - 1) / ctas);
            const int grid = int((items + per - 1) / per);
            kern<<<grid, nthr, bytes, c.stream>>>(src, dst, table_step, rl.E, c.fdev, c.n_theta, c.n_tiles,
                                                  c.n_depth, items, per, r_new, c.delta_theta, ea);
            return cudaGetLastError();
        };
        const bool full = c.n_theta % L == 0;
        if (nthr <= 256 && L == 8) {
            if (full && stages == 3) return go(k_azimuth_pipe<8, 3, RT, true>, 8);
            if (full && stages == 2) return go(k_azimuth_pipe<8, 2, RT, true>, 8);
            if (stages == 3) return go(k_azimuth_pipe<8, 3, RT, false>, 8);
            if (stages == 2) return go(k_azimuth_pipe<8, 2, RT, false>, 8);
        }
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

int sring_segment(int n_theta) {
    const RingPlan p = ring_plan(n_theta);
    return (p.kind == 2 && p.L == 16) ? 32 * p.L : 0;
}

cudaError_t launch_finish(const LaunchCtx& c, const cplx* src, int src_tiled, cplx* dst, double r,
                          const EpilogueArgs& ea) {
    const bool standard = ea.chunk_gap == 0 && (ea.chunk_cols == 0 || ea.chunk_cols == c.n_theta) && !ea.peer[0];
    if (!src_tiled && standard && ea.src_column && ea.periodic && (ea.temp_col || !getenv("PE3D_PREPARE_STAGED"))) {
        dim3 grid((c.n_tiles * 8 + PREPC_ROWS - 1) / PREPC_ROWS, c.n_freq);
        k_prepare_column<<<grid, 256, 0, c.stream>>>(src, dst, c.fdev, c.n_theta, c.n_tiles, c.n_depth, r,
                                                     c.delta_theta, ea);
        return cudaGetLastError();
    }
    if (ea.temp_col) return cudaErrorInvalidValue;         // only the column prologue writes a temp column
    if (!src_tiled && standard && c.n_theta % PREP_MB == 0) {
        dim3 grid(c.n_theta / PREP_MB, (c.n_tiles * 8 + PREP_DB - 1) / PREP_DB, c.n_freq);
        k_prepare<<<grid, 256, 0, c.stream>>>(src, dst, c.fdev, c.n_theta, c.n_tiles, c.n_depth, r, c.delta_theta, ea);
        return cudaGetLastError();
    }
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
