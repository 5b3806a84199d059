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
// (32 B per grid point); columns stream through a TMA stage ring
// (k_depth_tma, k_depth_tma_cluster; k_depth_scan is the cp.async fallback).
// Each frequency's per-CTA setup (folded coefficients, scan multipliers) is
// built once per march by k_depth_setup / k_depth_setup_cluster; the sweeps
// run with programmatic dependent launch, so their table loads overlap the
// previous sweep's tail (griddep_wait before the first field access).

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

#include <cooperative_groups.h>

#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

namespace pe3d {

#ifdef PE3D_PHASE_TIMING
// Phase timing of the depth sweeps (profiling builds only): per CTA, thread 0
// accumulates clock64 deltas of each phase in shared memory (no global
// round trip inside the timed phases) and adds them to g_phase[blockIdx][phase]
// at the end.
__device__ unsigned long long g_phase[4096][16];
#define PHASE_BEGIN                                                         \
    __shared__ unsigned long long _ph_acc[16];                              \
    if (threadIdx.x == 0)                                                   \
        for (int _k = 0; _k < 16; ++_k) _ph_acc[_k] = 0;                    \
    long long _ph_t = clock64();
#define PHASE(k) do { if (threadIdx.x == 0) { long long _n = clock64(); _ph_acc[k] += _n - _ph_t; _ph_t = _n; } } while (0)
#define PHASE_END do { if (threadIdx.x == 0) for (int _k = 0; _k < 16; ++_k) g_phase[blockIdx.x][_k] += _ph_acc[_k]; } while (0)
#else
#define PHASE_BEGIN
#define PHASE(k) do {} while (0)
#define PHASE_END do {} while (0)
#endif

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

// Column staging.  A thread owns RPT consecutive rows (RPT = 8: a whole
// 128-B tile line; RPT = 4: half a line); a warp owns LPW = 4*RPT lines of
// a column.  Global <-> shared copies are line-wise (lane -> line 4k + lane/8,
// element lane%8: one warp instruction moves 4 full lines); in shared memory
// element e of line ln sits at ln*8 + (e ^ swz(ln)), swz = ln&7 (RPT 8) or
// ln&3 (RPT 4), which makes both the line-wise copies and the per-thread
// row reads bank-conflict free.
template <int RPT>
struct Lines {
    static constexpr int LPW = 4 * RPT;            // lines per warp
    static constexpr int KIN = LPW / 4;            // copy instructions per lane
    __device__ static int swz(int ln) { return RPT == 8 ? (ln & 7) : (ln & 3); }
};

template <int RPT>
struct LaneLines {
    int64_t goff, gstep;
    int soff[Lines<RPT>::KIN];
    unsigned valid;
    __device__ LaneLines(int warp, int lane, int n_tiles, int64_t line_stride) {
        const int ln0 = lane >> 3, e = lane & 7;
        goff = int64_t(warp * Lines<RPT>::LPW + ln0) * line_stride + e;
        gstep = 4 * line_stride;
        valid = 0;
#pragma unroll
        for (int k = 0; k < Lines<RPT>::KIN; ++k) {
            const int ln = 4 * k + ln0;
            soff[k] = ln * 8 + (e ^ Lines<RPT>::swz(ln));
            if (warp * Lines<RPT>::LPW + ln < n_tiles) valid |= 1u << k;
        }
    }
};

template <int RPT>
__device__ __forceinline__ void stage_column(cplx* stage, const cplx* col_base, const LaneLines<RPT>& ll) {
    const cplx* gp = col_base + ll.goff;
#pragma unroll
    for (int k = 0; k < Lines<RPT>::KIN; ++k) {
        if (ll.valid & (1u << k)) cp_async16(stage + ll.soff[k], gp);
        else stage[ll.soff[k]] = czero();
        gp += ll.gstep;
    }
}

template <int RPT>
__device__ __forceinline__ void unstage_column(cplx* col_base, const cplx* stage, const LaneLines<RPT>& ll) {
    cplx* gp = col_base + ll.goff;
#pragma unroll
    for (int k = 0; k < Lines<RPT>::KIN; ++k) {
        if (ll.valid & (1u << k)) stc(gp, stage[ll.soff[k]]);
        gp += ll.gstep;
    }
}

// Launch configurations: rows per thread, max threads, pipeline depth,
// min CTAs per SM, and whether the scan multipliers live in shared memory.
template <int RPT, int MAXT> struct DepthCfg;
template <> struct DepthCfg<4, 256> { static constexpr int STAGES = 2, MINB = 3; static constexpr bool PRECOMP = true; };
template <> struct DepthCfg<8, 128> { static constexpr int STAGES = 3, MINB = 3; static constexpr bool PRECOMP = true; };
template <> struct DepthCfg<8, 256> { static constexpr int STAGES = 2, MINB = 2; static constexpr bool PRECOMP = true; };
template <> struct DepthCfg<8, 512> { static constexpr int STAGES = 2, MINB = 1; static constexpr bool PRECOMP = false; };

template <int RPT, int MAXT>
__host__ __device__ constexpr size_t depth_smem_elems(int nthreads) {
    return size_t(nthreads / 32) * DepthCfg<RPT, MAXT>::STAGES * (Lines<RPT>::LPW * 8) +
           (DepthCfg<RPT, MAXT>::PRECOMP ? 10 * size_t(nthreads) : 0) + 5 * size_t(nthreads / 32);
}

// Persistent CTA over a contiguous run of global columns g = f*n_theta + m.
// Thread t owns rows RPT*t .. RPT*t + RPT-1.  Registers hold the rows'
// column-independent coefficients
//   A'_l = kappa (1 + cx_rhs local_l) - 2 beta,  m_l,   (kappa = -1/off,
//   beta = kappa cx_rhs s_z)
// so that r'_l = A'_l x_l + beta (x_{l+1} + x_{l-1}) = kappa rhs_l and the
// forward elimination is y_l = m_l (r'_l + y_{l-1}).  The Kogge-Stone
// multipliers of the row-chunk scans (products of m_l over windows of
// threads) are column independent and, except for the largest CTAs, are
// computed once per frequency into shared memory -- zero where a lane has
// no partner, so the scans are branch free.
template <int RPT, int MAXT>
__global__ void __launch_bounds__(MAXT, (DepthCfg<RPT, MAXT>::MINB))
k_depth_scan(const cplx* __restrict__ src, cplx* __restrict__ dst, const cplx* __restrict__ loc_tab,
             const cplx* __restrict__ mul_tab, const FreqDev* __restrict__ fdev, int n_theta, int n_tiles,
             int64_t total_cols, int cols_per_cta, int sector) {
    constexpr int STAGES = DepthCfg<RPT, MAXT>::STAGES;
    constexpr bool PRECOMP = DepthCfg<RPT, MAXT>::PRECOMP;
    constexpr int SW = Lines<RPT>::LPW * 8;         // stage elements per warp per column
    extern __shared__ cplx smem[];
    const int nthreads = blockDim.x;
    const int nwarps = nthreads >> 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    cplx* stage = smem + warp * (STAGES * SW);
    cplx* mf = smem + nwarps * (STAGES * SW);       // [4][nthreads] forward multipliers, levels 1..4
    cplx* mb = mf + (PRECOMP ? 4 * nthreads : 0);   // [4][nthreads] backward
    cplx* pincf = mb + (PRECOMP ? 4 * nthreads : 0);
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
    const int nz8 = n_tiles * 8;
    const bool active = t * RPT < nz8;
    const int64_t line_stride = int64_t(n_theta) * 8;
    const int64_t freq_stride = int64_t(n_tiles) * line_stride;
    const LaneLines<RPT> ll(warp, lane, n_tiles, line_stride);
    // this thread's rows inside its warp's stage: line, first element
    const int my_line = lane * RPT / 8, my_e0 = (lane * RPT) & 7;
    const int my_swz = Lines<RPT>::swz(my_line);

    // (frequency, column) of the next column to prefetch
    int pf = int(g0 / n_theta), pc = int(g0 - int64_t(pf) * n_theta);
#pragma unroll
    for (int p = 0; p < STAGES - 1; ++p) {
        if (p < n_cols) {
            stage_column<RPT>(stage + p * SW, src + pf * freq_stride + int64_t(pc) * 8, ll);
            if (++pc == n_theta) { pc = 0; ++pf; }
        }
        cp_async_commit();
    }

    int f = int(g0 / n_theta), col = int(g0 - int64_t(f) * n_theta);
    int cur_f = -1;
    cplx A[RPT], M[RPT], beta = czero(), P0f = czero(), P0b = czero();
    int slot = 0;
    PHASE_BEGIN
    for (int it = 0; it < n_cols; ++it) {
        if (f != cur_f) {
            // ---- per-frequency coefficients and scan multipliers
            const FreqDev fd = fdev[f];
            const cplx kappa = crecip(cneg(fd.off_z));
            beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
            cplx P = cone();
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const cplx lc = active ? ldc(loc_tab + int64_t(f) * nz8 + RPT * t + i) : czero();
                M[i] = active ? ldc(mul_tab + int64_t(f) * nz8 + RPT * t + i) : czero();
                A[i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc))), cadd(beta, beta));
                P = cmul(M[i], P);
            }
            if (!active) P = cone();
            __syncthreads();                       // previous column done with the tables
            P0f = lane >= 1 ? P : czero();         // level-0 multipliers (own tile product)
            P0b = lane + 1 < 32 ? P : czero();
            cplx Pf = P, Pb = P;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const int o = 1 << d;
                if (PRECOMP && d > 0) {
                    mf[(d - 1) * nthreads + t] = lane >= o ? Pf : czero();
                    mb[(d - 1) * nthreads + t] = lane + o < 32 ? Pb : czero();
                }
                const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
                if (lane >= o) Pf = cmul(Pf, pu);
                if (lane + o < 32) Pb = cmul(Pb, pd);
            }
            if (PRECOMP) { pincf[t] = Pf; pincb[t] = Pb; }
            if (lane == 31) spw[warp] = Pf;
            __syncthreads();
            cur_f = f;
            PHASE(0);
        }
        // ---- prefetch column it + STAGES - 1, then wait for column it
        {
            const int ps = (slot + STAGES - 1) % STAGES;
            if (it + STAGES - 1 < n_cols) {
                stage_column<RPT>(stage + ps * SW, src + pf * freq_stride + int64_t(pc) * 8, ll);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
            cp_async_commit();
            PHASE(1);
            cp_async_wait<STAGES - 1>();
            __syncwarp();
            PHASE(2);
        }
        cplx* cur = stage + slot * SW;
        cplx x[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) x[i] = cur[my_line * 8 + ((my_e0 + i) ^ my_swz)];

        // ---- halos: last row of the chunk above, first row of the chunk below
        cplx up = shfl_up(x[RPT - 1], 1), dn = shfl_down(x[0], 1);
        if (lane == 31) sUp[warp] = x[RPT - 1];
        if (lane == 0) sDn[warp] = x[0];
        PHASE(3);
        __syncthreads();
        PHASE(4);
        if (lane == 0) up = warp > 0 ? sUp[warp - 1] : czero();
        if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : czero();
        if (t == 0) up = czero();

        // ---- r'_l = kappa rhs_l = A'_l x_l + beta (x_{l+1} + x_{l-1})
        //      (ref operators.py:115-121,139,210; marching.py:114: row 0 has m_0 = 0)
        cplx b[RPT];
        if (sector && (col == 0 || col == n_theta - 1)) {       // uniform per CTA
#pragma unroll
            for (int i = 0; i < RPT; ++i) b[i] = czero();
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const cplx um = i ? x[i - 1] : up;
                const cplx upp = i < RPT - 1 ? x[i + 1] : dn;
                b[i] = cfma(A[i], x[i], cmul(beta, cadd(upp, um)));
            }
        }

        // ---- forward elimination y_l = m_l (r'_l + y_{l-1}): local chunk, scan, exact re-run
        // (inactive threads have m = 0, hence Y = 0; pad rows have m = 0)
        cplx Y = czero();
#pragma unroll
        for (int i = 0; i < RPT; ++i) Y = cmul(M[i], cadd(b[i], Y));
        cplx Pacc = cone();
        if (!PRECOMP) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) Pacc = cmul(M[i], Pacc);
            if (!active) Pacc = cone();
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int o = 1 << d;
            const cplx Yp = shfl_up(Y, o);
            if (PRECOMP) {
                Y = cfma(d == 0 ? P0f : mf[(d - 1) * nthreads + t], Yp, Y);
            } else {
                const cplx Pp = shfl_up(Pacc, o);
                if (lane >= o) { Y = cfma(Pacc, Yp, Y); Pacc = cmul(Pacc, Pp); }
            }
        }
        if (lane == 31) sY[warp] = Y;
        PHASE(5);
        __syncthreads();
        PHASE(6);
        cplx C = czero();
        for (int w = 0; w < warp; ++w) C = cfma(spw[w], C, sY[w]);
        cplx y = shfl_up(cfma(PRECOMP ? pincf[t] : Pacc, C, Y), 1);
        if (lane == 0) y = C;
#pragma unroll
        for (int i = 0; i < RPT; ++i) { y = cmul(M[i], cadd(b[i], y)); b[i] = y; }

        // ---- back substitution x_l = y_l + m_l x_{l+1}
        cplx X = czero();
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) X = cfma(M[i], X, b[i]);
        cplx Qacc = cone();
        if (!PRECOMP) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) Qacc = cmul(M[i], Qacc);
            if (!active) Qacc = cone();
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int o = 1 << d;
            const cplx Xn = shfl_down(X, o);
            if (PRECOMP) {
                X = cfma(d == 0 ? P0b : mb[(d - 1) * nthreads + t], Xn, X);
            } else {
                const cplx Qn = shfl_down(Qacc, o);
                if (lane + o < 32) { X = cfma(Qacc, Xn, X); Qacc = cmul(Qacc, Qn); }
            }
        }
        if (lane == 0) sX[warp] = X;
        PHASE(7);
        __syncthreads();
        PHASE(8);
        cplx D = czero();
        for (int w = nwarps - 1; w > warp; --w) D = cfma(spw[w], D, sX[w]);
        cplx xv = shfl_down(cfma(PRECOMP ? pincb[t] : Qacc, D, X), 1);
        if (lane == 31) xv = D;
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) { xv = cfma(M[i], xv, b[i]); b[i] = xv; }
        PHASE(9);

        // ---- stage out through the same buffer, full-line stores
#pragma unroll
        for (int i = 0; i < RPT; ++i) cur[my_line * 8 + ((my_e0 + i) ^ my_swz)] = b[i];
        __syncwarp();
        unstage_column<RPT>(dst + f * freq_stride + int64_t(col) * 8, cur, ll);
        __syncwarp();
        PHASE(10);
        if (++col == n_theta) { col = 0; ++f; }
        slot = (slot + 1 == STAGES) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
    PHASE_END;
}

// Output tensor maps of the TMA depth sweeps: tiles [q*nzt, (q+1)*nzt) of
// every column go through map m[q].  The plain march uses one map over all
// tiles; the slab march's fused transpose uses one map per destination rank
// (the rank's depth-sweep output chunk in its azimuth-sweep input).
struct DepthDst {
    CUtensorMap m[MAX_PEERS];
    int nzt;
};

// ------------------------------------------------------------- TMA variant
// Same math as k_depth_scan<8, *>, but each warp's 32 column tiles move
// through the Tensor Memory Accelerator: one 4-D tiled TMA load per warp and
// column (box {16 doubles, 1 azimuth, 32 tiles, 1 frequency}, hardware
// 128-B swizzle = the line swizzle the threads read with, zero fill past the
// last tile), completion on a per-warp mbarrier, and one TMA bulk store of
// the solved column from the same stage.  The warps issue no per-line
// copies at all; a 3-deep per-warp stage ring keeps two columns in flight.
//
// SPLIT (long columns, LaunchCtx::split): the launch sees every 1024-row
// sub-column s of frequency f as a column of virtual frequency f*split + s;
// rows across sub-column edges enter the depth stencil as halo values read
// from the input one column ahead (edge threads), the sub-column is solved
// with zero carries, and its bottom y and top x go to sp_tot for
// k_split_carry.
template <int STAGES, int MINB, int MAXT, int NTH = 0, bool TAB = false, bool SPLIT = false>
__global__ void __launch_bounds__(MAXT, MINB)
k_depth_tma(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ DepthDst tm_dst,
            const cplx* __restrict__ loc_tab, const cplx* __restrict__ mul_tab, const FreqDev* __restrict__ fdev,
            const cplx* __restrict__ k1_tab, int n_theta, int n_tiles, int64_t total_cols, int cols_per_cta,
            int sector, const cplx* __restrict__ src_raw, int split, cplx* __restrict__ sp_tot, int src_col) {
    constexpr int RPT = 8;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int nthreads = NTH ? NTH : int(blockDim.x);   // compile-time when NTH: constant table offsets
    const int nwarps = nthreads >> 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    // 1024-B aligned stage ring (128-B swizzle atoms), then barriers and tables
    // offset arithmetic on the shared array keeps the shared address space (LDS/STS, not generic LD/ST)
    cplx* base = reinterpret_cast<cplx*>(smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));
    cplx* stage = base + warp * (STAGES * 256);
    cplx* mf = base + nwarps * (STAGES * 256);      // [4][nthreads]
    cplx* mb = mf + 4 * nthreads;
    cplx* pincf = mb + 4 * nthreads;
    cplx* pincb = pincf + nthreads;
    cplx* spw = pincb + nthreads;
    cplx* sY = spw + nwarps;
    cplx* sX = sY + nwarps;
    cplx* sUp = sX + nwarps;
    cplx* sDn = sUp + nwarps;
    cplx* shalo = sDn + nwarps;                     // SPLIT: [2 edge threads][2 buffers] halo rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(shalo + 4) + warp * STAGES;
    uint64_t* tbar = reinterpret_cast<uint64_t*>(shalo + 4) + nwarps * STAGES;   // frequency-table copy

    const int64_t g0 = int64_t(blockIdx.x) * cols_per_cta;
    const int64_t g1 = g0 + cols_per_cta < total_cols ? g0 + cols_per_cta : total_cols;
    if (g0 >= g1) return;
    const int n_cols = int(g1 - g0);
    const int nz8 = n_tiles * 8;
    const bool active = t * RPT < nz8;
    const int tile0 = warp * 32;
    const int qdst = tile0 / tm_dst.nzt;            // output map of this warp's tiles

    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < STAGES; ++k) mbar_init(&bars[k], 1);
        if (t == 0) mbar_init(tbar, 1);
        mbar_fence_init();
    }
    __syncthreads();

    int f = int(g0 / n_theta), col = int(g0 - int64_t(f) * n_theta);
    int cur_f = -1;
    cplx A[RPT], M[RPT], beta = czero(), P0f = czero(), P0b = czero();
    // A frequency's tables and constants are loaded in ONE round of
    // independent loads ahead of any arithmetic on them (under full HBM load
    // each dependent round costs microseconds); the first frequency's round
    // is issued before the column prefetches so it does not queue behind them.
    cplx lc[RPT];
    FreqDev fd;
    // With the per-march table (k_depth_setup) a frequency is one bulk copy of
    // its shared-memory image plus register loads, no arithmetic.
    const int img = k1_img(nthreads), kstride = k1_stride(nthreads);
    unsigned tpar = 0;
    auto load_freq = [&](int ff) {
        if constexpr (TAB) {
            const cplx* kt = k1_tab + int64_t(ff) * kstride;
            if (t == 0) {
                const unsigned bytes = unsigned(10 * nthreads + nwarps) * unsigned(sizeof(cplx));
                mbar_expect_tx(tbar, bytes);
                bulk_load(mf, kt, bytes, tbar);
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                A[i] = ldc(kt + img + RPT * t + i);
                M[i] = active ? ldc(mul_tab + int64_t(ff) * nz8 + RPT * t + i) : czero();
            }
            P0f = ldc(kt + img + 8 * nthreads + t);
            P0b = ldc(kt + img + 9 * nthreads + t);
            beta = ldc(kt + img + 10 * nthreads);
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                lc[i] = active ? ldc(loc_tab + int64_t(ff) * nz8 + RPT * t + i) : czero();
                M[i] = active ? ldc(mul_tab + int64_t(ff) * nz8 + RPT * t + i) : czero();
            }
            fd = fdev[ff];
        }
    };
    PHASE_BEGIN
    load_freq(f);
    griddep_wait();                                 // the field (input and output) belongs to the previous sweep until here

    int pf = int(g0 / n_theta), pc = int(g0 - int64_t(pf) * n_theta);
    if (lane == 0) {
#pragma unroll
        for (int p = 0; p < STAGES - 1; ++p) {
            if (p < n_cols) {
                mbar_expect_tx(&bars[p], 32 * 128);
                tma_load_4d(stage + p * 256, &tm_src, 0, src_col ? 0 : pc, tile0, pf, &bars[p]);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
        }
    }
    // SPLIT: the stencil rows across the sub-column edges (thread 0: the row
    // above the sub-column, the last thread: the row below), copied one column
    // ahead into a double buffer in shared memory (cp.async: the wait happens a
    // column later, off this column's path); a sub-column edge that is the
    // real column's surface or bottom gets zero
    const bool edge_thread = SPLIT && (t == 0 || t == nthreads - 1);
    cplx* my_halo = shalo + (t == 0 ? 0 : 2);
    auto halo_fetch = [&](int hf, int hc, int buf) {
        const int hs = hf % split;
        const bool inner = t == 0 ? hs > 0 : hs < split - 1;
        if (inner)
            cp_async16(&my_halo[buf], t == 0 ? src_raw + ((int64_t(hf) * n_tiles - 1) * n_theta + hc) * 8 + 7
                                             : src_raw + ((int64_t(hf) * n_tiles + n_tiles) * n_theta + hc) * 8);
        else
            my_halo[buf] = czero();
        cp_async_commit();
    };
    if (edge_thread) halo_fetch(f, col, 0);

    auto setup_freq = [&]() {
        if constexpr (TAB) {
            mbar_wait(tbar, tpar);
            tpar ^= 1u;
            cur_f = f;
        } else {
            const cplx kappa = crecip(cneg(fd.off_z));
            beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
            cplx P = cone();
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                A[i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc[i]))), cadd(beta, beta));
                P = cmul(M[i], P);
            }
            if (!active) P = cone();
            __syncthreads();
            P0f = lane >= 1 ? P : czero();
            P0b = lane + 1 < 32 ? P : czero();
            cplx Pf = P, Pb = P;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const int o = 1 << d;
                if (d > 0) {
                    mf[(d - 1) * nthreads + t] = lane >= o ? Pf : czero();
                    mb[(d - 1) * nthreads + t] = lane + o < 32 ? Pb : czero();
                }
                const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
                if (lane >= o) Pf = cmul(Pf, pu);
                if (lane + o < 32) Pb = cmul(Pb, pd);
            }
            pincf[t] = Pf;
            pincb[t] = Pb;
            if (lane == 31) spw[warp] = Pf;
            __syncthreads();
            cur_f = f;
        }
    };
    setup_freq();           // first frequency outside the loop: lc and fd are not loop-carried
    PHASE(11);

    int slot = 0;
    unsigned parity = 0;
    for (int it = 0; it < n_cols; ++it) {
        if (f != cur_f) {
            if constexpr (TAB) __syncthreads();     // every warp is done with the old shared tables
            load_freq(f);
            setup_freq();
            PHASE(0);
        }
        cplx* cur = stage + slot * 256;
        if (it == n_cols - 1) griddep_launch();     // last column: the next sweep may start launching
        cplx hal = czero();
        if (edge_thread) {
            cp_async_wait<0>();                     // this column's halo (issued a column ago)
            hal = my_halo[it & 1];
            if (it + 1 < n_cols) {
                if (col + 1 == n_theta) halo_fetch(f + 1, 0, (it + 1) & 1);
                else halo_fetch(f, col + 1, (it + 1) & 1);
            }
        }
        PHASE(1);
        mbar_wait(&bars[slot], parity);
        PHASE(2);
        // this lane's 128-B line of the swizzled stage: chunk i at line ^ (i << 4)
        const unsigned line = smem_addr(cur + lane * 8) + ((lane & 7) << 4);
        cplx x[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) x[i] = lds_at(line ^ unsigned(i << 4));

        cplx up = shfl_up(x[RPT - 1], 1), dn = shfl_down(x[0], 1);
        if (lane == 31) sUp[warp] = x[RPT - 1];
        if (lane == 0) sDn[warp] = x[0];
        PHASE(3);
        __syncthreads();
        PHASE(4);
        if (lane == 0) up = warp > 0 ? sUp[warp - 1] : czero();
        if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : czero();
        if (t == 0) up = czero();
        if (SPLIT) {
            if (t == 0) up = hal;
            if (t == nthreads - 1) dn = hal;
        }

        cplx b[RPT];
        if (sector && (col == 0 || col == n_theta - 1)) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) b[i] = czero();
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const cplx um = i ? x[i - 1] : up;
                const cplx upp = i < RPT - 1 ? x[i + 1] : dn;
                b[i] = cmul(M[i], cfma(A[i], x[i], cmul(beta, cadd(upp, um))));   // m_l r'_l, off the chain
            }
        }
        cplx Y = czero();
#pragma unroll
        for (int i = 0; i < RPT; ++i) Y = cfma(M[i], Y, b[i]);
#pragma unroll
        for (int d = 0; d < 5; ++d) Y = cfma(d == 0 ? P0f : mf[(d - 1) * nthreads + t], shfl_up(Y, 1 << d), Y);
        if (lane == 31) sY[warp] = Y;
        PHASE(5);
        __syncthreads();
        PHASE(6);
        cplx C = czero();
        if (NTH) {                                  // compile-time warp count: predicated, unrolled
#pragma unroll
            for (int w = 0; w < (NTH ? NTH : 32) / 32; ++w)
                if (w < warp) C = cfma(spw[w], C, sY[w]);
        } else {
            for (int w = 0; w < warp; ++w) C = cfma(spw[w], C, sY[w]);
        }
        cplx y = shfl_up(cfma(pincf[t], C, Y), 1);
        if (lane == 0) y = C;
#pragma unroll
        for (int i = 0; i < RPT; ++i) { y = cfma(M[i], y, b[i]); b[i] = y; }
        if (SPLIT && t == nthreads - 1) stc(sp_tot + (int64_t(f) * n_theta + col) * 2, y);   // zero-carry bottom y

        cplx X = czero();
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) X = cfma(M[i], X, b[i]);
#pragma unroll
        for (int d = 0; d < 5; ++d) X = cfma(d == 0 ? P0b : mb[(d - 1) * nthreads + t], shfl_down(X, 1 << d), X);
        if (lane == 0) sX[warp] = X;
        PHASE(7);
        __syncthreads();
        PHASE(8);
        cplx D = czero();
        if (NTH) {
#pragma unroll
            for (int w = (NTH ? NTH : 32) / 32 - 1; w >= 0; --w)
                if (w > warp) D = cfma(spw[w], D, sX[w]);
        } else {
            for (int w = nwarps - 1; w > warp; --w) D = cfma(spw[w], D, sX[w]);
        }
        cplx xv = shfl_down(cfma(pincb[t], D, X), 1);
        if (lane == 31) xv = D;
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) { xv = cfma(M[i], xv, b[i]); b[i] = xv; }
        if (SPLIT && t == 0) stc(sp_tot + (int64_t(f) * n_theta + col) * 2 + 1, xv);          // zero-carry top x

        PHASE(9);
        // ---- solved column back through the stage, one TMA store per warp
#pragma unroll
        for (int i = 0; i < RPT; ++i) sts_at(line ^ unsigned(i << 4), b[i]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_4d(&tm_dst.m[qdst], 0, col, tile0 - qdst * tm_dst.nzt, f, cur);
            bulk_commit();
            bulk_wait_read<1>();            // the previous column's store has left its stage slot
            if (it + STAGES - 1 < n_cols) {
                const int ps = (slot + STAGES - 1) % STAGES;
                mbar_expect_tx(&bars[ps], 32 * 128);
                tma_load_4d(stage + ps * 256, &tm_src, 0, src_col ? 0 : pc, tile0, pf, &bars[ps]);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
        }
        __syncwarp();
        PHASE(10);
        if (++col == n_theta) { col = 0; ++f; }
        if (++slot == STAGES) { slot = 0; parity ^= 1u; }
    }
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    PHASE(12);
    PHASE_END;
}

// Per-frequency setup of k_depth_tma, once per march (one CTA of nt threads
// per frequency): exactly the arithmetic k_depth_tma otherwise performs at
// every frequency it meets -- folded RHS coefficients, the column-independent
// Kogge-Stone multipliers and warp products -- written as the k1_tab record
// (pe3d_internal.h), so the sweep's frequency setup is loads only.
// fdiv > 1: records of the virtual frequencies of split columns (fdev[f / fdiv]).
__global__ void k_depth_setup(const cplx* __restrict__ loc_tab, const cplx* __restrict__ mul_tab,
                              const FreqDev* __restrict__ fdev, int n_tiles, cplx* __restrict__ k1_tab, int fdiv) {
    constexpr int RPT = 8;
    const int f = blockIdx.x;
    const int nthreads = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nz8 = n_tiles * 8;
    const bool active = t * RPT < nz8;
    cplx* kt = k1_tab + int64_t(f) * k1_stride(nthreads);
    const int img = k1_img(nthreads);
    cplx* mf = kt;
    cplx* mb = mf + 4 * nthreads;
    cplx* pincf = mb + 4 * nthreads;
    cplx* pincb = pincf + nthreads;
    cplx* spw = pincb + nthreads;
    const FreqDev fd = fdev[f / fdiv];
    const cplx kappa = crecip(cneg(fd.off_z));
    const cplx beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
    cplx P = cone();
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const cplx lc = active ? ldc(loc_tab + int64_t(f) * nz8 + RPT * t + i) : czero();
        const cplx m = active ? ldc(mul_tab + int64_t(f) * nz8 + RPT * t + i) : czero();
        kt[img + RPT * t + i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc))), cadd(beta, beta));
        P = cmul(m, P);
    }
    if (!active) P = cone();
    kt[img + 8 * nthreads + t] = lane >= 1 ? P : czero();
    kt[img + 9 * nthreads + t] = lane + 1 < 32 ? P : czero();
    cplx Pf = P, Pb = P;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int o = 1 << d;
        if (d > 0) {
            mf[(d - 1) * nthreads + t] = lane >= o ? Pf : czero();
            mb[(d - 1) * nthreads + t] = lane + o < 32 ? Pb : czero();
        }
        const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
        if (lane >= o) Pf = cmul(Pf, pu);
        if (lane + o < 32) Pb = cmul(Pb, pd);
    }
    pincf[t] = Pf;
    pincb[t] = Pb;
    if (lane == 31) spw[warp] = Pf;
    if (t == 0) kt[img + 10 * nthreads] = beta;
}

// The same for the long-column cluster sweep: one 128-thread CTA per
// (frequency, sub-column s), rows [1024 s, 1024 (s + 1)), exactly the
// arithmetic of k_depth_tma_cluster's in-kernel setup, written as the
// K1C record (pe3d_internal.h).
__global__ void __launch_bounds__(128) k_depth_setup_cluster(const cplx* __restrict__ loc_tab,
                                                             const cplx* __restrict__ mul_tab,
                                                             const FreqDev* __restrict__ fdev, int n_tiles,
                                                             cplx* __restrict__ k1_tab) {
    constexpr int RPT = 8, nthreads = 128, nwarps = 4;
    const int n_sub = n_tiles / 128;
    const int f = blockIdx.x / n_sub, s = blockIdx.x - f * n_sub;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nz8 = n_tiles * 8, row0 = s * 1024;
    cplx* kt = k1_tab + int64_t(blockIdx.x) * K1C_STRIDE;
    cplx* mf = kt;
    cplx* mb = mf + 4 * nthreads;
    cplx* pincf_g = mb + 4 * nthreads;
    cplx* pincb_g = pincf_g + nthreads;
    cplx* pexc = pincb_g + nthreads;
    cplx* psuf = pexc + nthreads;
    cplx* spw_g = psuf + nthreads;
    __shared__ cplx pincf[nthreads], pincb[nthreads], spw[nwarps];
    const FreqDev fd = fdev[f];
    const cplx kappa = crecip(cneg(fd.off_z));
    const cplx beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
    cplx P = cone();
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int64_t o = int64_t(f) * nz8 + row0 + RPT * t + i;
        const cplx lc = ldc(loc_tab + o);
        const cplx m = ldc(mul_tab + o);
        kt[K1C_IMG + RPT * t + i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc))), cadd(beta, beta));
        P = cmul(m, P);
    }
    kt[K1C_IMG + 8 * nthreads + t] = lane >= 1 ? P : czero();
    kt[K1C_IMG + 9 * nthreads + t] = lane + 1 < 32 ? P : czero();
    cplx Pf = P, Pb = P;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int o = 1 << d;
        if (d > 0) {
            mf[(d - 1) * nthreads + t] = lane >= o ? Pf : czero();
            mb[(d - 1) * nthreads + t] = lane + o < 32 ? Pb : czero();
        }
        const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
        if (lane >= o) Pf = cmul(Pf, pu);
        if (lane + o < 32) Pb = cmul(Pb, pd);
    }
    pincf[t] = pincf_g[t] = Pf;
    pincb[t] = pincb_g[t] = Pb;
    if (lane == 31) spw[warp] = spw_g[warp] = Pf;
    __syncthreads();
    cplx before = cone(), after = cone(), Pcta = cone();
    for (int w = 0; w < nwarps; ++w) {
        if (w < warp) before = cmul(before, spw[w]);
        if (w > warp) after = cmul(after, spw[w]);
        Pcta = cmul(Pcta, spw[w]);
    }
    pexc[t] = lane > 0 ? cmul(before, pincf[t - 1]) : before;
    psuf[t] = lane < 31 ? cmul(after, pincb[t + 1]) : after;
    if (t == 0) {
        kt[K1C_IMG + 10 * nthreads] = beta;
        kt[K1C_IMG + 10 * nthreads + 1] = Pcta;
    }
}

// Long columns (cfg5: 4096 rows): a thread-block cluster of CL CTAs per
// column, CTA s solving rows [s*R, (s+1)*R) (R = 8*tiles_per_cta <= 1024)
// with exactly the 128-thread k_depth_tma scheme above, so the SM runs three
// such CTAs like the cfg4 column kernel instead of one 16-warp CTA.  The
// sub-columns are chained by the scan structure of the substitutions:
//   forward  y entering CTA s = sum_{s'<s} (prod_{s'<u<s} P_u) Ytot_s'
//   backward x entering from below = sum_{s'>s} (prod_{s<u<s'} P_u) Xtot_s'
// with Ytot/Xtot the CTA's zero-carry totals and P_u the product of its
// multipliers; each thread adds (prefix product before it) x carry.  The
// totals travel by st.async into every peer's double-buffered table
// (mbarrier transaction counts, no cluster barrier in the loop).  The depth
// stencil's halo rows across sub-column edges are plain global loads of the
// (read-only) input.
template <int STAGES, int MINB, int NTH, bool TAB = false>
__global__ void __launch_bounds__(NTH, MINB)
k_depth_tma_cluster(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ DepthDst tm_dst,
                    const cplx* __restrict__ src_raw, const cplx* __restrict__ loc_tab,
                    const cplx* __restrict__ mul_tab, const FreqDev* __restrict__ fdev,
                    const cplx* __restrict__ k1_tab, int n_theta, int n_tiles, int64_t total_cols,
                    int cols_per_cluster, int sector) {
    constexpr int RPT = 8;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = int(cluster.num_blocks());
    const int s = int(cluster.block_rank());
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    constexpr int nthreads = NTH;                   // one tile per thread (= tiles per CTA)
    constexpr int nwarps = NTH / 32;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    cplx* base = reinterpret_cast<cplx*>(smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));
    cplx* stage = base + warp * (STAGES * 256);
    cplx* mf = base + nwarps * (STAGES * 256);      // [4][nthreads]
    cplx* mb = mf + 4 * nthreads;
    cplx* pincf = mb + 4 * nthreads;
    cplx* pincb = pincf + nthreads;
    cplx* pexc = pincb + nthreads;                  // product of the CTA's multipliers before thread t
    cplx* psuf = pexc + nthreads;                   // ... after thread t
    cplx* spw = psuf + nthreads;
    cplx* sY = spw + nwarps;
    cplx* sX = sY + nwarps;
    cplx* sUp = sX + nwarps;
    cplx* sDn = sUp + nwarps;
    constexpr int MAXCL = 8;                        // cluster sizes the launcher uses (n_tiles / 128 <= 8)
    cplx* xF = sDn + nwarps;                        // [2][MAXCL][2]: (Ytot, P) of every CTA
    cplx* xB = xF + 2 * MAXCL * 2;                  // [2][MAXCL]: Xtot, then [2][2] halo rows
    uint64_t* xbar = reinterpret_cast<uint64_t*>(xB + 2 * MAXCL + 4);   // [0..1] forward, [2..3] backward
    uint64_t* tbar = xbar + 4;                      // frequency-table copy
    uint64_t* bars = xbar + 5 + warp * STAGES;

    const int tpc = n_tiles / CL;                   // tiles per CTA (= nthreads)
    const int row0 = s * tpc * 8;
    const int64_t g0 = int64_t(blockIdx.x / CL) * cols_per_cluster;
    const int64_t g1 = g0 + cols_per_cluster < total_cols ? g0 + cols_per_cluster : total_cols;
    if (g0 >= g1) return;                           // uniform over the cluster
    const int n_cols = int(g1 - g0);
    const int nz8 = n_tiles * 8;
    const int tile0 = s * tpc + warp * 32;
    const int qdst = tile0 / tm_dst.nzt;            // output map of this warp's tiles

    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < STAGES; ++k) mbar_init(&bars[k], 1);
    }
    if (t == 0) {
#pragma unroll
        for (int k = 0; k < 5; ++k) mbar_init(&xbar[k], 1);
    }
    if (lane == 0) mbar_fence_init();
    cluster_barrier();                              // every peer's barriers initialised

    int f = int(g0 / n_theta), col = int(g0 - int64_t(f) * n_theta);
    int cur_f = -1;
    cplx A[RPT], M[RPT], beta = czero(), P0f = czero(), P0b = czero(), Pcta = czero();
    // With the per-march table (k_depth_setup_cluster) a frequency is one bulk
    // copy of this CTA's shared-memory image plus register loads, issued for
    // the first frequency before the column prefetches.
    const int n_sub = n_tiles / 128;
    unsigned tpar = 0;
    auto load_freq = [&](int ff) {
        if constexpr (TAB) {
            const cplx* kt = k1_tab + (int64_t(ff) * n_sub + s) * K1C_STRIDE;
            if (t == 0) {
                constexpr unsigned bytes = unsigned(12 * nthreads + nwarps) * unsigned(sizeof(cplx));
                mbar_expect_tx(tbar, bytes);
                bulk_load(mf, kt, bytes, tbar);
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                A[i] = ldc(kt + K1C_IMG + RPT * t + i);
                M[i] = ldc(mul_tab + int64_t(ff) * nz8 + row0 + RPT * t + i);
            }
            P0f = ldc(kt + K1C_IMG + 8 * nthreads + t);
            P0b = ldc(kt + K1C_IMG + 9 * nthreads + t);
            beta = ldc(kt + K1C_IMG + 10 * nthreads);
            Pcta = ldc(kt + K1C_IMG + 10 * nthreads + 1);
        }
    };
    if constexpr (TAB) load_freq(f);
    griddep_wait();                                 // the field belongs to the previous sweep until here

    int pf = int(g0 / n_theta), pc = int(g0 - int64_t(pf) * n_theta);
    if (lane == 0) {
#pragma unroll
        for (int p = 0; p < STAGES - 1; ++p) {
            if (p < n_cols) {
                mbar_expect_tx(&bars[p], 32 * 128);
                tma_load_4d(stage + p * 256, &tm_src, 0, pc, tile0, pf, &bars[p]);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
        }
    }

    // thread 0 keeps the row above the sub-column, the last thread the row below
    const bool halo_thread = (t == 0 && s > 0) || (t == nthreads - 1 && s < CL - 1);
    cplx* halo = xB + 2 * MAXCL + (t == 0 ? 0 : 2); // [2] per edge thread
    auto halo_src = [&](int hf, int hc) -> const cplx* {
        return t == 0 ? src_raw + ((int64_t(hf) * n_tiles + (row0 >> 3) - 1) * n_theta + hc) * 8 + 7
                      : src_raw + ((int64_t(hf) * n_tiles + (row0 >> 3) + tpc) * n_theta + hc) * 8;
    };
    if (halo_thread) {
        cp_async16(&halo[0], halo_src(f, col));
        cp_async_commit();
    }
    int slot = 0;
    unsigned parity = 0;
    PHASE_BEGIN
    for (int it = 0; it < n_cols; ++it) {
        const int buf = it & 1;
        const unsigned xpar = unsigned(it >> 1) & 1u;
        cplx* tF = xF + buf * (2 * MAXCL);
        cplx* tB = xB + buf * MAXCL;
        if (t == 0) {
            mbar_expect_tx(&xbar[buf], unsigned(CL) * 2 * sizeof(cplx));
            mbar_expect_tx(&xbar[2 + buf], unsigned(CL) * sizeof(cplx));
        }
        // halo rows across the sub-column edges (input is read-only here),
        // copied one column ahead by the two edge threads (cp.async into shared)
        cplx up_g = czero(), dn_g = czero();
        if (halo_thread) {
            cp_async_wait<0>();
            const cplx h = halo[buf];
            if (t == 0) up_g = h; else dn_g = h;
            if (it + 1 < n_cols) {
                const int nf = col + 1 == n_theta ? f + 1 : f, nc = col + 1 == n_theta ? 0 : col + 1;
                cp_async16(&halo[buf ^ 1], halo_src(nf, nc));
                cp_async_commit();
            }
        }
        if (TAB && f != cur_f) {
            if (cur_f >= 0) {
                __syncthreads();                    // every warp is done with the old shared tables
                load_freq(f);
            }
            mbar_wait(tbar, tpar);
            tpar ^= 1u;
            cur_f = f;
            PHASE(0);
        }
        if (!TAB && f != cur_f) {
            const FreqDev fd = fdev[f];
            const cplx kappa = crecip(cneg(fd.off_z));
            beta = cmul(kappa, crmul(fd.s_z, fd.cx_rhs));
            cplx P = cone();
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int64_t o = int64_t(f) * nz8 + row0 + RPT * t + i;
                const cplx lc = ldc(loc_tab + o);
                M[i] = ldc(mul_tab + o);
                A[i] = csub(cmul(kappa, cadd(cone(), cmul(fd.cx_rhs, lc))), cadd(beta, beta));
                P = cmul(M[i], P);
            }
            __syncthreads();
            P0f = lane >= 1 ? P : czero();
            P0b = lane + 1 < 32 ? P : czero();
            cplx Pf = P, Pb = P;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const int o = 1 << d;
                if (d > 0) {
                    mf[(d - 1) * nthreads + t] = lane >= o ? Pf : czero();
                    mb[(d - 1) * nthreads + t] = lane + o < 32 ? Pb : czero();
                }
                const cplx pu = shfl_up(Pf, o), pd = shfl_down(Pb, o);
                if (lane >= o) Pf = cmul(Pf, pu);
                if (lane + o < 32) Pb = cmul(Pb, pd);
            }
            pincf[t] = Pf;
            pincb[t] = Pb;
            if (lane == 31) spw[warp] = Pf;
            __syncthreads();
            {
                cplx before = cone(), after = cone();
                Pcta = cone();
                for (int w = 0; w < nwarps; ++w) {
                    if (w < warp) before = cmul(before, spw[w]);
                    if (w > warp) after = cmul(after, spw[w]);
                    Pcta = cmul(Pcta, spw[w]);
                }
                pexc[t] = lane > 0 ? cmul(before, pincf[t - 1]) : before;
                psuf[t] = lane < 31 ? cmul(after, pincb[t + 1]) : after;
            }
            cur_f = f;
            PHASE(0);
        }
        cplx* cur = stage + slot * 256;
        if (it == n_cols - 1) griddep_launch();     // last column: the next sweep may start launching
        PHASE(1);
        mbar_wait(&bars[slot], parity);
        PHASE(2);
        const int sw = lane & 7;
        cplx x[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) x[i] = cur[lane * 8 + (i ^ sw)];

        cplx up = shfl_up(x[RPT - 1], 1), dn = shfl_down(x[0], 1);
        if (lane == 31) sUp[warp] = x[RPT - 1];
        if (lane == 0) sDn[warp] = x[0];
        PHASE(3);
        __syncthreads();
        PHASE(4);
        if (lane == 0) up = warp > 0 ? sUp[warp - 1] : up_g;
        if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : dn_g;

        cplx b[RPT];
        if (sector && (col == 0 || col == n_theta - 1)) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) b[i] = czero();
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const cplx um = i ? x[i - 1] : up;
                const cplx upp = i < RPT - 1 ? x[i + 1] : dn;
                b[i] = cmul(M[i], cfma(A[i], x[i], cmul(beta, cadd(upp, um))));   // m_l r'_l, off the chain
            }
        }
        cplx Y = czero();
#pragma unroll
        for (int i = 0; i < RPT; ++i) Y = cfma(M[i], Y, b[i]);
#pragma unroll
        for (int d = 0; d < 5; ++d) Y = cfma(d == 0 ? P0f : mf[(d - 1) * nthreads + t], shfl_up(Y, 1 << d), Y);
        if (lane == 31) sY[warp] = Y;
        PHASE(5);
        __syncthreads();
        PHASE(6);
        cplx C = czero();
        for (int w = 0; w < warp; ++w) C = cfma(spw[w], C, sY[w]);
        const cplx yinc = cfma(pincf[t], C, Y);         // y at this thread's last row, zero CTA carry
        // forward totals to every peer: (Ytot, P) from the CTA's last thread
        if (warp == nwarps - 1) {
            const cplx ytot = shfl_idx(yinc, 31);
            if (lane < CL) {
                const unsigned rb = mapa_shared(smem_addr(&xbar[buf]), lane);
                st_async_cplx(mapa_shared(smem_addr(tF + 2 * s), lane), ytot, rb);
                st_async_cplx(mapa_shared(smem_addr(tF + 2 * s + 1), lane), Pcta, rb);
            }
        }
        cplx y = shfl_up(yinc, 1);
        if (lane == 0) y = C;
        PHASE(15);
        mbar_wait(&xbar[buf], xpar);
        PHASE(13);
        {
            cplx cin = czero();
            for (int u = 0; u < s; ++u) cin = cfma(tF[2 * u + 1], cin, tF[2 * u]);
            y = cfma(pexc[t], cin, y);                  // + carry entering the CTA, propagated
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) { y = cfma(M[i], y, b[i]); b[i] = y; }

        cplx X = czero();
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) X = cfma(M[i], X, b[i]);
#pragma unroll
        for (int d = 0; d < 5; ++d) X = cfma(d == 0 ? P0b : mb[(d - 1) * nthreads + t], shfl_down(X, 1 << d), X);
        if (lane == 0) sX[warp] = X;
        PHASE(7);
        __syncthreads();
        PHASE(8);
        cplx D = czero();
        for (int w = nwarps - 1; w > warp; --w) D = cfma(spw[w], D, sX[w]);
        const cplx xinc = cfma(pincb[t], D, X);         // x at this thread's first row, zero carry from below
        if (warp == 0) {
            const cplx xtot = shfl_idx(xinc, 0);
            if (lane < CL)
                st_async_cplx(mapa_shared(smem_addr(tB + s), lane), xtot, mapa_shared(smem_addr(&xbar[2 + buf]), lane));
        }
        cplx xv = shfl_down(xinc, 1);
        if (lane == 31) xv = D;
        PHASE(9);
        mbar_wait(&xbar[2 + buf], xpar);
        PHASE(14);
        {
            cplx din = czero();
            for (int u = CL - 1; u > s; --u) din = cfma(tF[2 * u + 1], din, tB[u]);
            xv = cfma(psuf[t], din, xv);
        }
#pragma unroll
        for (int i = RPT - 1; i >= 0; --i) { xv = cfma(M[i], xv, b[i]); b[i] = xv; }

        PHASE(11);
#pragma unroll
        for (int i = 0; i < RPT; ++i) cur[lane * 8 + (i ^ sw)] = b[i];
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_4d(&tm_dst.m[qdst], 0, col, tile0 - qdst * tm_dst.nzt, f, cur);
            bulk_commit();
            bulk_wait_read<1>();
            if (it + STAGES - 1 < n_cols) {
                const int ps = (slot + STAGES - 1) % STAGES;
                mbar_expect_tx(&bars[ps], 32 * 128);
                tma_load_4d(stage + ps * 256, &tm_src, 0, pc, tile0, pf, &bars[ps]);
                if (++pc == n_theta) { pc = 0; ++pf; }
            }
        }
        __syncwarp();
        PHASE(10);
        if (++col == n_theta) { col = 0; ++f; }
        if (++slot == STAGES) { slot = 0; parity ^= 1u; }
    }
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    PHASE(12);
    PHASE_END;
    cluster_barrier();                              // no CTA leaves while peers may still address it
}

static int round32(int x) { return (x + 31) / 32 * 32; }

// Host side of the TMA path: 4-D tiled tensor maps over the device field
// (dims {16 doubles, n_theta, n_tiles, n_freq}).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Generic tiled FLOAT64 map with the 128-B swizzle (used by the azimuth sweep's
// ring maps, pe3d_ring.cu); false when the driver entry point or the encoder refuses.
bool encode_swizzled_map(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                         const uint32_t* box, int swizzle_bytes) {
    auto enc = tensor_map_encoder();
    if (!enc || rank < 1 || rank > 5) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], e[5];
    for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; e[i] = 1; }
    for (int i = 0; i + 1 < rank; ++i) st[i] = strides[i];
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank), const_cast<void*>(base), d, st, b, e,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool field_tensor_map(CUtensorMap* tm, const void* base, const LaunchCtx& c) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[4] = {16, cuuint64_t(c.n_theta), cuuint64_t(c.n_tiles), cuuint64_t(c.n_freq)};
    const cuuint64_t strides[3] = {128, cuuint64_t(c.n_theta) * 128, cuuint64_t(c.n_theta) * 128 * c.n_tiles};
    const cuuint32_t box[4] = {16, 1, 32, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The first step's input when it is one column per frequency (LaunchCtx::src_col):
// [F][n_tiles][8] complex, one azimuth.
static bool column_tensor_map(CUtensorMap* tm, const void* base, const LaunchCtx& c) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[4] = {16, 1, cuuint64_t(c.n_tiles), cuuint64_t(c.n_freq)};
    const cuuint64_t strides[3] = {128, 128, cuuint64_t(c.n_tiles) * 128};
    const cuuint32_t box[4] = {16, 1, 32, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output maps: the plain field, or one map per peer chunk (slab march).
static bool depth_dst_maps(DepthDst* d, const void* dst, const LaunchCtx& c) {
    if (c.n_peers == 0) {
        d->nzt = c.n_tiles;
        return field_tensor_map(&d->m[0], dst, c);
    }
    if (c.n_freq != 1 || c.peer_tiles % 32 != 0 || c.n_peers * c.peer_tiles != c.n_tiles) return false;
    LaunchCtx cp = c;
    cp.n_tiles = c.peer_tiles;
    for (int q = 0; q < c.n_peers; ++q)
        if (!field_tensor_map(&d->m[q], c.peer_dst[q], cp)) return false;
    d->nzt = c.peer_tiles;
    return true;
}

template <int STAGES, int MINB, int MAXT, bool SPLIT = false>
static cudaError_t launch_depth_tma_cfg(const LaunchCtx& c, const cplx* src, cplx* dst) {
    CUtensorMap tm_src;
    DepthDst tm_dst;
    // c.src_col: the input is one column per frequency ([F][n_tiles][8]), the same for every
    // azimuth (the first step after a column starter's prologue): a map with one azimuth,
    // every column loads azimuth 0
    if (c.src_col && (SPLIT || c.sector)) return cudaErrorNotSupported;
    const bool ok = c.src_col ? column_tensor_map(&tm_src, c.src_col, c) : field_tensor_map(&tm_src, src, c);
    if (!ok || !depth_dst_maps(&tm_dst, dst, c)) return cudaErrorNotSupported;
    const int nthreads = (c.n_tiles + 31) / 32 * 32;
    const int nwarps = nthreads / 32;
    const size_t bytes = 1024 + sizeof(cplx) * (size_t(nwarps) * STAGES * 256 + 10 * size_t(nthreads) + 5 * nwarps + 4) +
                         sizeof(uint64_t) * (nwarps * STAGES + 1);
    if (bytes > 227 * 1024) return cudaErrorNotSupported;
    const cplx* k1 = (c.k1_tab && c.n_tiles <= K1_TAB_MAX_TILES && nthreads == round32(c.n_tiles)) ? c.k1_tab : nullptr;
    if (SPLIT && !(k1 && MAXT == 128 && nthreads == 128)) return cudaErrorNotSupported;
    auto kern = SPLIT ? k_depth_tma<STAGES, MINB, MAXT, 128, true, true>
                      : (MAXT == 128 && nthreads == 128)
                            ? (k1 ? k_depth_tma<STAGES, MINB, MAXT, 128, true> : k_depth_tma<STAGES, MINB, MAXT, 128>)
                      : (MAXT == 64 && nthreads == 64)
                            ? (k1 ? k_depth_tma<STAGES, MINB, MAXT, 64, true> : k_depth_tma<STAGES, MINB, MAXT, 64>)
                      : (MAXT == 32 && nthreads == 32)
                            ? (k1 ? k_depth_tma<STAGES, MINB, MAXT, 32, true> : k_depth_tma<STAGES, MINB, MAXT, 32>)
                            : (k1 ? k_depth_tma<STAGES, MINB, MAXT, 0, true> : k_depth_tma<STAGES, MINB, MAXT>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e != cudaSuccess) return e;
    const int64_t total = int64_t(c.n_freq) * c.n_theta;
    int per_sm = int((227 * 1024) / (bytes + 1024));
    if (per_sm > MINB) per_sm = MINB;
    if (per_sm < 1) per_sm = 1;
    int64_t ctas = int64_t(c.num_sms) * per_sm;
#ifdef PE3D_PHASE_CTAS
    ctas = PE3D_PHASE_CTAS;         // phase-timing builds: uncontended critical path with few CTAs
#endif
    const int per = int((total + ctas - 1) / ctas);
    const int grid = int((total + per - 1) / per);
    return launch_pdl(c.pdl != 0, kern, dim3(grid), dim3(nthreads), bytes, c.stream, tm_src, tm_dst, c.loc_tab,
                      c.mul_tab, c.fdev, k1, c.n_theta, c.n_tiles, total, per, c.sector, src, c.split, c.sp_tot,
                      c.src_col ? 1 : 0);
}

static cudaError_t launch_depth_tma_cluster(const LaunchCtx& c, const cplx* src, cplx* dst, int CL) {
    CUtensorMap tm_src;
    DepthDst tm_dst;
    if (!field_tensor_map(&tm_src, src, c) || !depth_dst_maps(&tm_dst, dst, c)) return cudaErrorNotSupported;
    constexpr int STAGES = 3, MINB = 3;
    const int nthreads = c.n_tiles / CL;
    const int nwarps = nthreads / 32;
    const size_t bytes = 1024 + sizeof(cplx) * (size_t(nwarps) * STAGES * 256 + 12 * size_t(nthreads) + 5 * nwarps +
                                                2 * 8 * 2 + 2 * 8 + 4) +
                         sizeof(uint64_t) * (5 + nwarps * STAGES);
    if (nthreads != 128 || CL > K1C_MAX_SUB) return cudaErrorNotSupported;
    const cplx* k1 = c.k1_tab;                      // the march builds the K1C records for this column length
    auto kern = k1 ? k_depth_tma_cluster<STAGES, MINB, 128, true> : k_depth_tma_cluster<STAGES, MINB, 128>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(nthreads);
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
    // co-resident clusters, cached per kernel (table / no table), device and smem size
    cfg.gridDim = dim3(CL * c.num_sms);
    const int resident = cached_occupancy((const void*)kern, bytes, CL, nthreads, &cfg);
    if (resident < 1) return cudaErrorInvalidConfiguration;
    const int64_t total = int64_t(c.n_freq) * c.n_theta;
    const int per = int((total + resident - 1) / resident);
    const int clusters = int((total + per - 1) / per);
    cfg.gridDim = dim3(clusters * CL);
    // PDL only when the grid leaves most co-resident cluster slots free (cfg2:
    // 128 of 222); a full persistent grid launched early loses co-residency
    // (see launch_cluster_ring, pe3d_ring.cu)
    cfg.numAttrs = (c.pdl && 4 * clusters <= 3 * resident) ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, tm_src, tm_dst, src, c.loc_tab, c.mul_tab, c.fdev, k1, c.n_theta,
                              c.n_tiles, total, per, c.sector);
}

// Columns of up to 128 tiles: 128-thread CTAs, 3 stages, 3 CTAs per SM.
// Longer columns split into CL = n_tiles/128 sub-columns of 128 tiles, one
// per CTA of a cluster (cfg5: 4096 rows, CL = 4); otherwise one 512-thread
// CTA per SM.
static cudaError_t launch_depth_tma(const LaunchCtx& c, const cplx* src, cplx* dst) {
    // the SM runs 12 column warps whatever the column length (168 registers, ~70 KB of
    // shared memory per 4-warp CTA): shorter columns get more, smaller CTAs (512-row
    // columns: 3 x 2 warps 152 us -> 6 x 2 warps 109.5 us per 16.8 M points, tools/ring_probe.py)
    if (!getenv("PE3D_DEPTH_SMALL_CTA_OFF")) {
        if (c.n_tiles <= 32) return launch_depth_tma_cfg<3, 12, 32>(c, src, dst);
        if (c.n_tiles <= 64) return launch_depth_tma_cfg<3, 6, 64>(c, src, dst);
    }
    if (c.n_tiles <= 128) return launch_depth_tma_cfg<3, 3, 128>(c, src, dst);
    if (c.n_tiles % 128 == 0 && c.n_tiles / 128 <= 8 && !getenv("PE3D_DEPTH_NO_CLUSTER"))
        return launch_depth_tma_cluster(c, src, dst, c.n_tiles / 128);
    return launch_depth_tma_cfg<2, 1, 512>(c, src, dst);
}

// ------------------------------------------------------ split long columns
// Responses of one 1024-row sub-column to unit carries, once per march (one
// thread per (f, s), rows [1024 s, 1024 (s + 1))): with y_l = m_l y_(l-1) + b_l
// and x_l = m_l x_(l+1) + y_l, a carry c entering at the top adds
// a_l c to x_l (p_l = m_l p_(l-1), p_(top-1) = 1; a_l = m_l a_(l+1) + p_l,
// a_(bottom+1) = 0) and a carry d entering from below adds q_l d
// (q_l = m_l q_(l+1), q_(bottom+1) = 1).  sp_pa[fs] = (P_s = prod m_l over the
// sub-column = p_bottom = q_top, A_s = a_top, (a_span, q_span)).
//
// The responses decay geometrically away from the sub-column edges (|m_l| <
// 1): rows where both |a_l| and |q_l| are below SPLIT_TAU take no correction
// (a dropped term is below 1e-30 of the carry, i.e. of the field's scale;
// the contract is 1e-9).  a_span = rows from the top with |a_l| >= tau,
// q_span = rows from the bottom with |q_l| >= tau; a and q are zeroed
// outside, so the azimuth sweep can skip whole tiles.
constexpr double SPLIT_TAU = 1e-30;
__global__ void k_split_setup(const cplx* __restrict__ mul_tab, int n_virtual, cplx* __restrict__ sp_aq,
                              cplx* __restrict__ sp_pa) {
    const int fs = blockIdx.x * blockDim.x + threadIdx.x;
    if (fs >= n_virtual) return;
    const cplx* m = mul_tab + int64_t(fs) * 1024;
    cplx* aq = sp_aq + int64_t(fs) * 2048;          // (a_l, q_l) pairs of the sub-column's rows
    cplx p = cone();
    for (int l = 0; l < 1024; ++l) {
        p = cmul(ldc(m + l), p);
        stc(aq + 2 * l, p);                         // p_l, overwritten by a_l below
    }
    cplx a = czero(), q = cone();
    int a_span = 0, q_span = 0;
    for (int l = 1023; l >= 0; --l) {
        const cplx ml = ldc(m + l);
        a = cfma(ml, a, ldc(aq + 2 * l));
        q = cmul(ml, q);
        if (a_span == 0 && cabs(a) >= SPLIT_TAU) a_span = l + 1;
        if (cabs(q) >= SPLIT_TAU) q_span = 1024 - l;
        stc(aq + 2 * l, a);
        stc(aq + 2 * l + 1, q);
    }
    const cplx A = a;
    for (int l = 0; l < 1024; ++l) {                // exact zeros outside the spans
        if (l >= a_span) stc(aq + 2 * l, czero());
        if (l < 1024 - q_span) stc(aq + 2 * l + 1, czero());
    }
    stc(sp_pa + 3 * fs, p);
    stc(sp_pa + 3 * fs + 1, A);
    stc(sp_pa + 3 * fs + 2, mk(double(a_span), double(q_span)));
}

// Exact carries of every sub-column from the zero-carry totals, one thread
// per (f, column):  cin_0 = 0, cin_(s+1) = T_s + P_s cin_s;  din_(CL-1) = 0,
// din_(s-1) = X_s + A_s cin_s + P_s din_s.  Written lane-ordered for the
// azimuth sweep's stage (azimuth m = seg*NS + q*L + k at seg*NS + k*32 + q).
constexpr int SPLIT_MAX = 8;
__global__ void __launch_bounds__(64) k_split_carry(const cplx* __restrict__ sp_tot, const cplx* __restrict__ sp_pa,
                                                     cplx* __restrict__ sp_cd, int n_freq, int n_theta, int split,
                                                     int L) {
    griddep_wait();                                 // the depth sweep's totals
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= int64_t(n_freq) * n_theta) return;
    const int f = int(gid / n_theta), m = int(gid - int64_t(f) * n_theta);
    const int NS = 32 * L;
    const int seg = m / NS, w = m - seg * NS;
    const int mp = seg * NS + (w % L) * 32 + w / L;
    cplx cin[SPLIT_MAX], T[SPLIT_MAX], X[SPLIT_MAX], P[SPLIT_MAX], A[SPLIT_MAX];
#pragma unroll
    for (int s = 0; s < SPLIT_MAX; ++s) {
        if (s < split) {
            const int64_t fs = int64_t(f) * split + s;
            T[s] = ldc(sp_tot + (fs * n_theta + m) * 2);
            X[s] = ldc(sp_tot + (fs * n_theta + m) * 2 + 1);
            P[s] = ldc(sp_pa + 3 * fs);
            A[s] = ldc(sp_pa + 3 * fs + 1);
        }
    }
    cplx c = czero();
#pragma unroll
    for (int s = 0; s < SPLIT_MAX; ++s) {
        if (s < split) {
            cin[s] = c;
            c = cfma(P[s], c, T[s]);
        }
    }
    cplx d = czero();
#pragma unroll
    for (int s = SPLIT_MAX - 1; s >= 0; --s) {
        if (s < split) {
            cplx* o = sp_cd + (int64_t(f) * split + s) * 2 * n_theta;
            stc(o + mp, cin[s]);
            stc(o + n_theta + mp, d);
            d = cfma(A[s], cin[s], cfma(P[s], d, X[s]));
        }
    }
}

int depth_split_plan(const LaunchCtx& c, int periodic) {
    const int CL = c.n_tiles / 128;
    if (!periodic || c.sector || c.n_peers > 0 || !c.k1_tab || c.n_tiles % 128 != 0 || CL < 2 || CL > SPLIT_MAX)
        return 0;
    if (ring_segment(c.n_theta) == 0 || !tensor_map_encoder()) return 0;
    for (const char* name : {"PE3D_DEPTH_NO_SPLIT", "PE3D_RING_CPASYNC"})
        if (getenv(name)) return 0;
    return CL;
}

cudaError_t launch_split_carry(const LaunchCtx& c) {
    const int64_t n = int64_t(c.n_freq) * c.n_theta;
    // small CTAs: one thread per column is little work, so spread it over many SMs (latency bound)
    return launch_pdl(c.pdl != 0, k_split_carry, dim3(unsigned((n + 63) / 64)), dim3(64), 0, c.stream, c.sp_tot,
                      c.sp_pa, c.sp_cd, c.n_freq, c.n_theta, c.split, ring_segment(c.n_theta) / 32);
}

bool depth_sweep_takes_column(const LaunchCtx& c) {
    return c.split < 2 && !c.sector && c.n_peers == 0 && c.n_tiles <= 128 && !getenv("PE3D_FIRST_STEP_FIELD");
}

cudaError_t launch_depth_scan(const LaunchCtx& c, const cplx* src, cplx* dst) {
    if (c.src_col) return c.n_tiles <= 128 ? launch_depth_tma(c, src, dst) : cudaErrorNotSupported;
    if (c.split >= 2) {
        // every 1024-row sub-column as a column of its own virtual frequency
        LaunchCtx v = c;
        v.n_freq = c.n_freq * c.split;
        v.n_tiles = 128;
        v.n_depth = 1024;
        return launch_depth_tma_cfg<3, 3, 128, true>(v, src, dst);
    }
    const int64_t total = int64_t(c.n_freq) * c.n_theta;
    auto go = [&](auto kern, int nthreads, size_t elems, int per_sm) -> cudaError_t {
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
    if (c.n_peers > 0 || c.n_tiles <= 512) {
        cudaError_t e = launch_depth_tma(c, src, dst);
        if (e != cudaErrorNotSupported || c.n_peers > 0) return e;    // peer output needs the TMA kernels
    }
    const int nt = round32(c.n_tiles);
    if (nt <= 128) return go(k_depth_scan<8, 128>, nt, depth_smem_elems<8, 128>(nt), DepthCfg<8, 128>::MINB);
    if (nt <= 256) return go(k_depth_scan<8, 256>, nt, depth_smem_elems<8, 256>(nt), DepthCfg<8, 256>::MINB);
    return go(k_depth_scan<8, 512>, nt, depth_smem_elems<8, 512>(nt), DepthCfg<8, 512>::MINB);
}

// Factor tables once per march: the parallel continuant scan (pe3d_medium.cu)
// for columns of up to 4096 rows; the reference-order single-thread
// recurrence when PE3D_FACTOR_SERIAL is set (it was 0.46 ms per cfg4 march).
static cudaError_t launch_depth_setup(const LaunchCtx& c) {
    if (!c.k1_tab) return cudaSuccess;
    if (c.split >= 2) {
        // 1024-row sub-columns as virtual frequencies, plus the carry responses
        k_depth_setup<<<c.n_freq * c.split, 128, 0, c.stream>>>(c.loc_tab, c.mul_tab, c.fdev, 128, c.k1_tab, c.split);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        k_split_setup<<<(c.n_freq * c.split + 31) / 32, 32, 0, c.stream>>>(c.mul_tab, c.n_freq * c.split, c.sp_aq,
                                                                             c.sp_pa);
        return cudaGetLastError();
    }
    if (c.n_tiles <= K1_TAB_MAX_TILES)
        k_depth_setup<<<c.n_freq, round32(c.n_tiles), 0, c.stream>>>(c.loc_tab, c.mul_tab, c.fdev, c.n_tiles, c.k1_tab, 1);
    else if (k1_tab_elems(c.n_freq, c.n_tiles) > 0)
        k_depth_setup_cluster<<<c.n_freq * (c.n_tiles / 128), 128, 0, c.stream>>>(c.loc_tab, c.mul_tab, c.fdev,
                                                                                 c.n_tiles, c.k1_tab);
    return cudaGetLastError();
}

cudaError_t launch_factor_depth(const LaunchCtx& c, const cplx* local, int64_t local_fstride, int step_for_error) {
    if (!getenv("PE3D_FACTOR_SERIAL")) {
        const cudaError_t e = launch_factor_depth_scan(c, local, local_fstride, step_for_error);
        if (e != cudaErrorNotSupported) return e != cudaSuccess ? e : launch_depth_setup(c);
    }
    k_factor_depth<<<c.n_freq, 1, 0, c.stream>>>(local, local_fstride, c.loc_tab, c.mul_tab, c.fdev, c.n_depth,
                                                 c.n_tiles * 8, step_for_error, c.err);
    const cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? e : launch_depth_setup(c);
}

}  // namespace pe3d
