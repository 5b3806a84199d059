// pe3d_depth.cu -- K1, the depth sweep of one range step of Eq. (4)
// (arXiv 1711.00005; reference pe3d marching.py:109-123).
//
// For every (frequency, azimuth) column: the explicit depth factor
// rhs = [1 + cx_rhs X(n_j)] temp, with temp = [1 + cy_rhs Y(r_j)] u already
// applied by the previous azimuth sweep (ref operators.py:197-210), the
// surface row rhs_0 = 0 (marching.py:114), and the solve of
// [1 + cx_lhs X(n_{j+1})] v = rhs with the surface row imposed as v_0 = 0
// (operators.py:213-241, tridiag.py:151-178).
//
// The depth matrix of a range-independent medium is the same for every
// azimuth and every step.  k_factor_depth factors it once per frequency with
// the reference's Thomas recurrence; the sweep then only runs the two
// linear recurrences of the substitution,
//     y_l = b_l + m_l y_{l-1},     x_l = y_l + m_l x_{l+1},
// with b_l = inv_l rhs_l and m_l = -cp_l = -off inv_l (m_0 = 0), split over
// threads (8 rows each), chained by affine scans and re-run with the exact
// carries.  Memory: one 128-B line per (tile, column) in, one out
// (32 B per grid point); columns stream through a cp.async ring.

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

namespace pe3d {

// One thread per frequency: Thomas pivots of the depth matrix with the
// surface row imposed (ref operators.py:227-238, tridiag.py:151-167) using
// the reference's recurrence and Smith reciprocals; writes the local term
// and the recurrence multipliers m_l = -(off * inv_l) (m_0 = 0, pads 0).
__global__ void k_factor_depth(const cplx* __restrict__ local, int64_t local_fstride,
                               cplx* __restrict__ loc_tab, cplx* __restrict__ mul_tab,
                               const FreqDev* __restrict__ fdev, int n_depth, int nz8,
                               int step_for_error, DevError* err) {
    const int f = blockIdx.x;
    if (threadIdx.x != 0) return;
    const FreqDev fd = fdev[f];
    const cplx* lc = local + f * local_fstride;
    cplx* lt = loc_tab + int64_t(f) * nz8;
    cplx* mt = mul_tab + int64_t(f) * nz8;
    const double two_s = 2.0 * fd.s_z;
    cplx cp = czero();      // cp_{k-1}
    bool failed = false;
    for (int l = 0; l < nz8; ++l) {
        if (l >= n_depth) { lt[l] = czero(); mt[l] = czero(); continue; }
        const cplx loc = lc[l];
        lt[l] = loc;
        const cplx main_l = (l == 0) ? cone() : cadd(cone(), cmul(fd.cx_lhs, mk(loc.re - two_s, loc.im)));
        // denom_k = main_k - sub_{k-1} * cp_{k-1}   (sub = off everywhere, sub[0] kept)
        const cplx denom = (l == 0) ? main_l : csub(main_l, cmul(fd.off_z, cp));
        if (!failed && cabs(denom) < PIVOT_FLOOR) {
            failed = true;
            report_failure(err, fail_key(step_for_error, 0, f, 0), l, 0);
        }
        const cplx inv = crecip(denom);
        const cplx sup = (l == 0) ? czero() : fd.off_z;    // sup[0] = 0 (surface row)
        cp = cmul(sup, inv);
        mt[l] = (l == 0) ? czero() : cneg(cmul(fd.off_z, inv));
    }
}

// Per-lane addressing of one column's 32 depth tiles of this warp (32 lines
// of 128 B): lane -> (line 4k + lane/8, element lane%8), k = 0..7, so one
// warp instruction moves 4 full lines.  In shared memory the element is
// XOR-swizzled by the line index so that the per-thread tile reads
// (lane = line) are bank-conflict free.
struct LaneLines {
    int64_t goff;          // global element offset of k = 0 relative to the column base
    int64_t gstep;         // 4 lines
    int soff_even, soff_odd;
    unsigned valid;        // bit k: line 4k + lane/8 exists
};

__device__ __forceinline__ LaneLines lane_lines(int warp, int lane, int n_tiles, int64_t line_stride) {
    LaneLines ll;
    const int ln = lane >> 3, e = lane & 7;
    ll.goff = int64_t(warp * 32 + ln) * line_stride + e;
    ll.gstep = 4 * line_stride;
    ll.soff_even = ln * 8 + (e ^ ln);
    ll.soff_odd = ln * 8 + (e ^ (ln | 4));
    ll.valid = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (warp * 32 + 4 * k + ln < n_tiles) ll.valid |= 1u << k;
    return ll;
}

__device__ __forceinline__ void stage_column(cplx* stage, const cplx* col_base, const LaneLines& ll) {
    const cplx* gp = col_base + ll.goff;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        cplx* d = stage + 32 * k + ((k & 1) ? ll.soff_odd : ll.soff_even);
        if (ll.valid & (1u << k)) cp_async16(d, gp);
        else *d = czero();
        gp += ll.gstep;
    }
}

__device__ __forceinline__ void unstage_column(cplx* col_base, const cplx* stage, const LaneLines& ll) {
    cplx* gp = col_base + ll.goff;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (ll.valid & (1u << k)) stc(gp, stage[32 * k + ((k & 1) ? ll.soff_odd : ll.soff_even)]);
        gp += ll.gstep;
    }
}

template <int MAXT> struct DepthCfg;
template <> struct DepthCfg<128> { static constexpr int STAGES = 3, MINB = 3; static constexpr bool PRECOMP = true; };
template <> struct DepthCfg<256> { static constexpr int STAGES = 2, MINB = 2; static constexpr bool PRECOMP = true; };
template <> struct DepthCfg<512> { static constexpr int STAGES = 2, MINB = 1; static constexpr bool PRECOMP = false; };

template <int MAXT>
__host__ __device__ constexpr size_t depth_smem_elems(int nthreads) {
    return size_t(nthreads / 32) * DepthCfg<MAXT>::STAGES * 256 +
           (DepthCfg<MAXT>::PRECOMP ? 12 * size_t(nthreads) : 0) + 5 * size_t(nthreads / 32);
}

// Persistent CTA over a contiguous run of global columns g = f*n_theta + m.
// Thread t owns depth tile t (rows 8t..8t+7).  Registers hold the tile's
// column-independent coefficients
//   A_l = kappa (1 + cx_rhs local_l),  m_l,   (kappa = -1/off)
// so that b_l = m_l (A_l x_l + beta d2_l) = inv_l rhs_l with
// beta = kappa cx_rhs s_z.  The Kogge-Stone multipliers of the tile scans
// (products of m_l over windows of tiles) are column independent too and,
// for up to 256 threads, are computed once per frequency into shared memory
// -- with zeros where a lane has no partner, so the scans are branch free.
template <int MAXT>
__global__ void __launch_bounds__(MAXT, DepthCfg<MAXT>::MINB)
k_depth_scan(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ loc_tab,
             const cplx* __restrict__ mul_tab, const FreqDev* __restrict__ fdev, int n_theta, int n_tiles,
             int64_t total_cols, int cols_per_cta, int sector) {
    constexpr int STAGES = DepthCfg<MAXT>::STAGES;
    constexpr bool PRECOMP = DepthCfg<MAXT>::PRECOMP;
    extern __shared__ cplx smem[];
    const int nthreads = blockDim.x;
    const int nwarps = nthreads >> 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    cplx* stage = smem + warp * (STAGES * 256);
    cplx* mf = smem + nwarps * (STAGES * 256);      // [5][nthreads]   (PRECOMP)
    cplx* mb = mf + (PRECOMP ? 5 * nthreads : 0);   // [5][nthreads]
    cplx* pincf = mb + (PRECOMP ? 5 * nthreads : 0);
    cplx* pincb = pincf + (PRECOMP ? nthreads : 0);
    cplx* spw = pincb + (PRECOMP ? nthreads : 0);   // [nwarps] warp products
    cplx* sY = spw + nwarps;
    cplx* sX = sY + nwarps;
    cplx* sUp = sX + nwarps;
    cplx* sDn = sUp + nwarps;

    const int64_t g0 = int64_t(blockIdx.x) * cols_per_cta;
    const int64_t g1 = g0 + cols_per_cta < total_cols ? g0 + cols_per_cta : total_cols;
    if (g0 >= g1) return;
    const int n_cols = int(g1 - g0);
    const bool active = t < n_tiles;
    const int64_t nz8 = int64_t(n_tiles) * 8;
    const int64_t line_stride = int64_t(n_theta) * 8;
    const int64_t freq_stride = int64_t(n_tiles) * line_stride;
    const LaneLines ll = lane_lines(warp, lane, n_tiles, line_stride);

    // (frequency, column) of the next column to prefetch
    int pf = int(g0 / n_theta), pc = int(g0 - int64_t(pf) * n_theta);
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (p < n_cols) {
            stage_column(stage + p * 256, src + pf * freq_stride + int64_t(pc) * 8, ll);
            if (++pc == n_theta) { pc = 0; ++pf; }
        }
        cp_async_commit();
    }

    int f = int(g0 / n_theta), col = int(g0 - int64_t(f) * n_theta);
    int cur_f = -1;
    cplx A[8], M[8], beta = czero();
    int slot = 0;
    for (int it = 0; it < n_cols; ++it) {
        if (f != cur_f) {
            // ---- per-frequency coefficients and scan multipliers
            const FreqDev fd = fdev[f];
            const cplx kappa = crecip(cneg(fd.off_z));
            beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
            cplx P = cone();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const cplx lc = active ? ldc(loc_tab + f * nz8 + 8 * t + i) : czero();
                M[i] = active ? ldc(mul_tab + f * nz8 + 8 * t + i) : czero();
                // A'_l = kappa (1 + cx_rhs local_l) - 2 beta  (the -2x of d2 folded in)
                A[i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc))), cadd(beta, beta));
                P = cmul(M[i], P);
            }
            if (!active) P = cone();
            __syncthreads();                       // previous column done with the tables
            cplx Pf = P, Pb = P;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const int o = 1 << d;
                if (PRECOMP) {
                    mf[d * nthreads + t] = lane >= o ? Pf : czero();
                    mb[d * nthreads + t] = lane + o < 32 ? Pb : czero();
                }
                const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
                if (lane >= o) Pf = cmul(Pf, pu);
                if (lane + o < 32) Pb = cmul(Pb, pd);
            }
            if (PRECOMP) { pincf[t] = Pf; pincb[t] = Pb; }
            if (lane == 31) spw[warp] = Pf;
            __syncthreads();
            cur_f = f;
        }
        // ---- prefetch column it + STAGES - 1, then wait for column it
        {
            const int ps = (slot + STAGES - 1) % STAGES;
            if (it + STAGES - 1 < n_cols) {
                stage_column(stage + ps * 256, src + pf * freq_stride + int64_t(pc) * 8, ll);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
            cp_async_commit();
            cp_async_wait<STAGES - 1>();
            __syncwarp();
        }
        cplx* cur = stage + slot * 256;
        const int sw = lane & 7;
        cplx x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = cur[lane * 8 + (i ^ sw)];

        // ---- halos: last row of the tile above, first row of the tile below
        cplx up = shfl_up(x[7], 1), dn = shfl_down(x[0], 1);
        if (lane == 31) sUp[warp] = x[7];
        if (lane == 0) sDn[warp] = x[0];
        __syncthreads();
        if (lane == 0) up = warp > 0 ? sUp[warp - 1] : czero();
        if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : czero();
        if (t == 0) up = czero();
        if (t >= n_tiles - 1) dn = czero();

        // ---- r'_l = kappa rhs_l = A'_l x_l + beta (x_{l+1} + x_{l-1})
        //      (ref operators.py:115-121,139,210; marching.py:114: row 0 has m_0 = 0)
        cplx b[8];
        if (sector && (col == 0 || col == n_theta - 1)) {       // uniform per CTA
#pragma unroll
            for (int i = 0; i < 8; ++i) b[i] = czero();
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const cplx um = i ? x[i - 1] : up;
                const cplx upp = i < 7 ? x[i + 1] : dn;
                b[i] = cfma(A[i], x[i], cmul(beta, cadd(upp, um)));
            }
        }

        // ---- forward elimination y_l = m_l (r'_l + y_{l-1}): local chunk, scan, exact re-run
        // (inactive threads have m = 0 and x = 0, hence Y = 0)
        cplx Y = czero();
#pragma unroll
        for (int i = 0; i < 8; ++i) Y = cmul(M[i], cadd(b[i], Y));
        cplx Pacc = cone();
        if (!PRECOMP) {
#pragma unroll
            for (int i = 0; i < 8; ++i) Pacc = cmul(M[i], Pacc);
            if (!active) Pacc = cone();
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int o = 1 << d;
            const cplx Yp = shfl_up(Y, o);
            if (PRECOMP) {
                Y = cfma(mf[d * nthreads + t], Yp, Y);
            } else {
                const cplx Pp = shfl_up(Pacc, o);
                if (lane >= o) { Y = cfma(Pacc, Yp, Y); Pacc = cmul(Pacc, Pp); }
            }
        }
        if (lane == 31) sY[warp] = Y;
        __syncthreads();
        cplx C = czero();
        for (int w = 0; w < warp; ++w) C = cfma(spw[w], C, sY[w]);
        cplx y = shfl_up(cfma(PRECOMP ? pincf[t] : Pacc, C, Y), 1);
        if (lane == 0) y = C;
#pragma unroll
        for (int i = 0; i < 8; ++i) { y = cmul(M[i], cadd(b[i], y)); b[i] = y; }

        // ---- back substitution
        cplx X = czero();
#pragma unroll
        for (int i = 7; i >= 0; --i) X = cfma(M[i], X, b[i]);
        cplx Qacc = cone();
        if (!PRECOMP) {
#pragma unroll
            for (int i = 0; i < 8; ++i) Qacc = cmul(M[i], Qacc);
            if (!active) Qacc = cone();
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int o = 1 << d;
            const cplx Xn = shfl_down(X, o);
            if (PRECOMP) {
                X = cfma(mb[d * nthreads + t], Xn, X);
            } else {
                const cplx Qn = shfl_down(Qacc, o);
                if (lane + o < 32) { X = cfma(Qacc, Xn, X); Qacc = cmul(Qacc, Qn); }
            }
        }
        if (lane == 0) sX[warp] = X;
        __syncthreads();
        cplx D = czero();
        for (int w = nwarps - 1; w > warp; --w) D = cfma(spw[w], D, sX[w]);
        cplx xv = shfl_down(cfma(PRECOMP ? pincb[t] : Qacc, D, X), 1);
        if (lane == 31) xv = D;
#pragma unroll
        for (int i = 7; i >= 0; --i) { xv = cfma(M[i], xv, b[i]); b[i] = xv; }

        // ---- stage out through the same buffer, full-line stores
#pragma unroll
        for (int i = 0; i < 8; ++i) cur[lane * 8 + (i ^ sw)] = b[i];
        __syncwarp();
        unstage_column(dst + f * freq_stride + int64_t(col) * 8, cur, ll);
        __syncwarp();
        if (++col == n_theta) { col = 0; ++f; }
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

static int round32(int x) { return (x + 31) / 32 * 32; }

cudaError_t launch_depth_scan(const LaunchCtx& c, const cplx* src, cplx* dst) {
    const int nthreads = round32(c.n_tiles);
    const int64_t total = int64_t(c.n_freq) * c.n_theta;
    auto go = [&](auto kern, size_t elems, int per_sm) -> cudaError_t {
        const size_t sm = sizeof(cplx) * elems;
        if (sm > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            if (e != cudaSuccess) return e;
        }
        const int64_t ctas = int64_t(c.num_sms) * per_sm;
        const int per = int((total + ctas - 1) / ctas);
        const int grid = int((total + per - 1) / per);
        kern<<<grid, nthreads, sm, c.stream>>>(src, dst, c.loc_tab, c.mul_tab, c.fdev, c.n_theta, c.n_tiles, total,
                                               per, c.sector);
        return cudaGetLastError();
    };
    if (nthreads <= 128) return go(k_depth_scan<128>, depth_smem_elems<128>(nthreads), DepthCfg<128>::MINB);
    if (nthreads <= 256) return go(k_depth_scan<256>, depth_smem_elems<256>(nthreads), DepthCfg<256>::MINB);
    return go(k_depth_scan<512>, depth_smem_elems<512>(nthreads), DepthCfg<512>::MINB);
}

cudaError_t launch_factor_depth(const LaunchCtx& c, const cplx* local, int64_t local_fstride, int step_for_error) {
    k_factor_depth<<<c.n_freq, 1, 0, c.stream>>>(local, local_fstride, c.loc_tab, c.mul_tab, c.fdev, c.n_depth,
                                                 c.n_tiles * 8, step_for_error, c.err);
    return cudaGetLastError();
}

}  // namespace pe3d
