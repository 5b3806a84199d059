// pe3d_kernels.cu -- sm_100a kernels of one range step of Eq. (4)
// (arXiv 1711.00005; reference pe3d marching.py:93-136).
//
// Per step, two fused sweeps over the complex128 field, each one HBM read
// + one HBM write of 16 B per grid point (64 B/point/step):
//
//   k_depth_scan   (K1)  temp -> v : RHS [1 + cx_rhs X(n_j)] applied to
//                        temp = [1 + cy_rhs Y(r_j)] u, then the depth system
//                        [1 + cx_lhs X(n_{j+1})] v = rhs with the surface row
//                        v = 0 (ref operators.py:197-241, tridiag.py:151-178).
//   k_azimuth_scan (K2)  v -> temp': the periodic azimuth system
//                        [1 + cy_lhs Y(r_{j+1})] u = v per depth (ref
//                        operators.py:244-262, tridiag.py:186-212), then the
//                        boundary (marching.py:133-134), the TL record
//                        (marching.py:167-172) and the NEXT step's azimuth
//                        factor temp' = [1 + cy_rhs Y(r_{j+1})] u, so that K1
//                        needs no azimuth halo.
//
// Both sweeps are first-order linear recurrences once the matrices are
// factored: the depth matrix A is the same for every azimuth and every
// step of a range-independent medium (factored once per frequency by
// k_factor_depth with the reference's recurrence), and the azimuth matrix B
// is a symmetric circulant, B = (-c/rho)(I - rho S)(I - rho S^-1) with
// |rho| < 1, whose inverse is two cyclic first-order recurrences.  Each
// recurrence is split into per-thread chunks held in registers, chained by
// a warp-shuffle + shared-memory affine scan, and re-run with the exact
// carry.  The thread-per-system kernels at the end of the file follow the
// reference's operation order literally; they serve sector grids,
// range/azimuth-dependent media and solve_batch.

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

namespace pe3d {

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ void report_failure(DevError* err, unsigned long long key, int pivot, int rank1) {
    const unsigned long long old = atomicMin(&err->key, key);
    if (key < old) {            // benign race on the payload: the lowest key's writer wins last
        err->pivot = pivot;
        err->rank1 = rank1;
    }
}

__host__ __device__ __forceinline__ unsigned long long fail_key(int step, int sweep, int f, int member) {
    return (static_cast<unsigned long long>(step) << 40) | (static_cast<unsigned long long>(sweep) << 39) |
           (static_cast<unsigned long long>(f) << 24) | static_cast<unsigned long long>(member);
}

// s = 1/(k0 r dtheta)^2, evaluated in the reference's order (operators.py:102)
__device__ __forceinline__ double azimuth_scale(double k0, double r, double dth) {
    const double x = (k0 * r) * dth;
    return 1.0 / (x * x);
}

// |w(r)| for w = (cos k0 r + i sin k0 r)/sqrt(r)  (environment.py:287-294)
__device__ __forceinline__ double hankel_abs(double k0, double r) {
    const double sr = sqrt(r);
    const double kr = k0 * r;
    return hypot(cos(kr) / sr, sin(kr) / sr);
}

// ------------------------------------------------------ depth factorization

// One thread per frequency: Thomas pivots of the depth matrix with the
// surface row imposed (ref operators.py:227-238, tridiag.py:151-167) using
// the reference's recurrence and Smith reciprocals; writes the local term
// and the recurrence multipliers m_l = -cp_l = -(off * inv_l) (m_0 = 0).
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
        cplx main_l = (l == 0) ? cone() : cadd(cone(), cmul(fd.cx_lhs, mk(loc.re - two_s, loc.im)));
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

// ------------------------------------------------------------ block scans

// Forward affine scan: thread t holds the map y_out = Y + P * y_in of its
// chunk; returns the true y entering thread t's chunk (carry-in 0 at t=0).
__device__ __forceinline__ cplx scan_forward(cplx P, cplx Y, cplx* sP, cplx* sY, int lane, int warp) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const cplx Pp = shfl_up(P, d), Yp = shfl_up(Y, d);
        if (lane >= d) { Y = cfma(P, Yp, Y); P = cmul(P, Pp); }
    }
    if (lane == 31) { sP[warp] = P; sY[warp] = Y; }
    __syncthreads();
    cplx C = czero();
    for (int w = 0; w < warp; ++w) C = cfma(sP[w], C, sY[w]);
    const cplx inc = cfma(P, C, Y);
    cplx ex = shfl_up(inc, 1);
    if (lane == 0) ex = C;
    return ex;
}

// Backward affine scan: x_out (top of chunk t) = X + Q * x_in (from chunk
// t+1); returns the true x entering from below (0 below the last chunk).
__device__ __forceinline__ cplx scan_backward(cplx Q, cplx X, cplx* sQ, cplx* sX, int lane, int warp,
                                              int nwarps) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const cplx Qn = shfl_down(Q, d), Xn = shfl_down(X, d);
        if (lane + d < 32) { X = cfma(Q, Xn, X); Q = cmul(Q, Qn); }
    }
    if (lane == 0) { sQ[warp] = Q; sX[warp] = X; }
    __syncthreads();
    cplx C = czero();
    for (int w = nwarps - 1; w > warp; --w) C = cfma(sQ[w], C, sX[w]);
    const cplx inc = cfma(Q, C, X);
    cplx ex = shfl_down(inc, 1);
    if (lane == 31) ex = C;
    return ex;
}

// ------------------------------------------------------ K1: depth sweep

// One CTA = one frequency x a run of azimuth columns; thread t owns depth
// tile t (rows 8t..8t+7) and keeps that tile's local term and recurrence
// multipliers in registers for all its columns.  A column's tiles are
// staged through shared memory (128-B XOR swizzle) so that global loads
// and stores are full 128-B lines, 512 B per warp instruction.
__global__ void __launch_bounds__(512)
k_depth_scan(const cplx* __restrict__ src, cplx* __restrict__ dst,
             const cplx* __restrict__ loc_tab, const cplx* __restrict__ mul_tab,
             const FreqDev* __restrict__ fdev, int n_theta, int n_tiles, int cols_per_block,
             int sector) {
    extern __shared__ cplx smem[];
    const int nwarps = blockDim.x >> 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    cplx* stage = smem + warp * 256;
    cplx* sP = smem + nwarps * 256;
    cplx* sY = sP + nwarps;
    cplx* sQ = sY + nwarps;
    cplx* sX = sQ + nwarps;
    cplx* sUp = sX + nwarps;
    cplx* sDn = sUp + nwarps;

    const int f = blockIdx.y;
    const bool active = t < n_tiles;
    const FreqDev fd = fdev[f];
    const int64_t nz8 = int64_t(n_tiles) * 8;
    cplx LC[8], M[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        LC[i] = active ? ldc(loc_tab + f * nz8 + 8 * t + i) : czero();
        M[i] = active ? ldc(mul_tab + f * nz8 + 8 * t + i) : czero();
    }
    const cplx kappa = crecip(cneg(fd.off_z));   // b_l = inv_l * r_l = m_l * (r_l * kappa)
    const int c_begin = blockIdx.x * cols_per_block;
    const int c_end = min(n_theta, c_begin + cols_per_block);
    const int64_t line_stride = int64_t(n_theta) * 8;                // elements between depth tiles
    const cplx* src_f = src + int64_t(f) * n_tiles * line_stride;
    cplx* dst_f = dst + int64_t(f) * n_tiles * line_stride;

    for (int col = c_begin; col < c_end; ++col) {
        // ---- stage in: lane -> (line 4k + lane/8, element lane%8)
        cplx x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int line = 4 * k + (lane >> 3), e = lane & 7, tile = warp * 32 + line;
            const cplx v = (tile < n_tiles) ? ldc_stream(src_f + tile * line_stride + int64_t(col) * 8 + e) : czero();
            stage[line * 8 + (e ^ (line & 7))] = v;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = stage[lane * 8 + (i ^ (lane & 7))];

        // ---- halos: last row of the tile above, first row of the tile below
        cplx up = shfl_up(x[7], 1), dn = shfl_down(x[0], 1);
        if (lane == 31) sUp[warp] = x[7];
        if (lane == 0) sDn[warp] = x[0];
        __syncthreads();
        if (lane == 0) up = warp > 0 ? sUp[warp - 1] : czero();
        if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : czero();
        if (t == 0) up = czero();
        if (t >= n_tiles - 1) dn = czero();

        // ---- right-hand side (ref operators.py:115-121,139,210; marching.py:114)
        const bool zero_col = sector && (col == 0 || col == n_theta - 1);
        cplx b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const cplx um = i ? x[i - 1] : up;
            const cplx upp = i < 7 ? x[i + 1] : dn;
            const cplx d2 = cadd(csub(upp, crmul(2.0, x[i])), um);
            const cplx xt = cadd(cmul(LC[i], x[i]), crmul(fd.s_z, d2));
            cplx r = cadd(x[i], cmul(fd.cx_rhs, xt));
            if (zero_col) r = czero();
            b[i] = cmul(M[i], cmul(r, kappa));       // row 0 and pad rows: M = 0 -> b = 0
        }

        // ---- forward elimination y_l = b_l + m_l y_{l-1}: local chunk, scan, exact re-run
        cplx P = cone(), Y = czero();
#pragma unroll
        for (int i = 0; i < 8; ++i) { Y = cfma(M[i], Y, b[i]); P = cmul(M[i], P); }
        if (!active) { P = cone(); Y = czero(); }
        cplx y = scan_forward(P, Y, sP, sY, lane, warp);
#pragma unroll
        for (int i = 0; i < 8; ++i) { y = cfma(M[i], y, b[i]); b[i] = y; }

        // ---- back substitution x_l = y_l + m_l x_{l+1}
        cplx Q = cone(), X = czero();
#pragma unroll
        for (int i = 7; i >= 0; --i) { X = cfma(M[i], X, b[i]); Q = cmul(M[i], Q); }
        if (!active) { Q = cone(); X = czero(); }
        cplx xv = scan_backward(Q, X, sQ, sX, lane, warp, nwarps);
#pragma unroll
        for (int i = 7; i >= 0; --i) { xv = cfma(M[i], xv, b[i]); b[i] = xv; }

        // ---- stage out (same swizzle), full-line stores
#pragma unroll
        for (int i = 0; i < 8; ++i) stage[lane * 8 + (i ^ (lane & 7))] = b[i];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int line = 4 * k + (lane >> 3), e = lane & 7, tile = warp * 32 + line;
            if (tile < n_tiles) stc(dst_f + tile * line_stride + int64_t(col) * 8 + e, stage[line * 8 + (e ^ (line & 7))]);
        }
        __syncthreads();   // stage / scan scratch reuse by the next column
    }
}

// ------------------------------------------ ring epilogue (K2 and finish)

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
        sLast[q * rw + i] = u[nvalid - 1];
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
        const cplx up = (k < nvalid - 1) ? u[k + 1] : next;
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

// ------------------------------------------------ K2: azimuth sweep

// Group-interleaved scans: scan groups are the RW depth rows of the CTA;
// thread t = i + RW*q holds row i, azimuth chunk q.
template <int RW>
__device__ __forceinline__ void group_scan_fwd(cplx P, cplx Y, cplx& Pex, cplx& Yex, cplx& Ptot, cplx& Ytot,
                                               cplx* sP, cplx* sY, int lane, int warp, int nwarps, int i) {
    constexpr int G = 32 / RW;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx Pp = shfl_up(P, d * RW), Yp = shfl_up(Y, d * RW);
        if (lane >= d * RW) { Y = cfma(P, Yp, Y); P = cmul(P, Pp); }
    }
    if (lane >= 32 - RW) { sP[warp * RW + i] = P; sY[warp * RW + i] = Y; }
    __syncthreads();
    cplx CP = cone(), CY = czero(), TP, TY;
    for (int w = 0; w < warp; ++w) {
        CY = cfma(sP[w * RW + i], CY, sY[w * RW + i]);
        CP = cmul(sP[w * RW + i], CP);
    }
    TP = CP; TY = CY;
    for (int w = warp; w < nwarps; ++w) {
        TY = cfma(sP[w * RW + i], TY, sY[w * RW + i]);
        TP = cmul(sP[w * RW + i], TP);
    }
    const cplx Pinc = cmul(P, CP), Yinc = cfma(P, CY, Y);
    Pex = shfl_up(Pinc, RW);
    Yex = shfl_up(Yinc, RW);
    if (lane < RW) { Pex = CP; Yex = CY; }
    Ptot = TP; Ytot = TY;
}

template <int RW>
__device__ __forceinline__ void group_scan_bwd(cplx Q, cplx X, cplx& Qex, cplx& Xex, cplx& Qtot, cplx& Xtot,
                                               cplx* sQ, cplx* sX, int lane, int warp, int nwarps, int i) {
    constexpr int G = 32 / RW;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const cplx Qn = shfl_down(Q, d * RW), Xn = shfl_down(X, d * RW);
        if (lane + d * RW < 32) { X = cfma(Q, Xn, X); Q = cmul(Q, Qn); }
    }
    if (lane < RW) { sQ[warp * RW + i] = Q; sX[warp * RW + i] = X; }
    __syncthreads();
    cplx CQ = cone(), CX = czero(), TQ, TX;
    for (int w = nwarps - 1; w > warp; --w) {
        CX = cfma(sQ[w * RW + i], CX, sX[w * RW + i]);
        CQ = cmul(sQ[w * RW + i], CQ);
    }
    TQ = CQ; TX = CX;
    for (int w = warp; w >= 0; --w) {
        TX = cfma(sQ[w * RW + i], TX, sX[w * RW + i]);
        TQ = cmul(sQ[w * RW + i], TQ);
    }
    const cplx Qinc = cmul(Q, CQ), Xinc = cfma(Q, CX, X);
    Qex = shfl_down(Qinc, RW);
    Xex = shfl_down(Xinc, RW);
    if (lane >= 32 - RW) { Qex = CQ; Xex = CX; }
    Qtot = TQ; Xtot = TX;
}

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

// One CTA = one frequency x RW depth rows x the whole azimuth ring.
template <int L, int RW>
__global__ void __launch_bounds__(512)
k_azimuth_scan(const cplx* __restrict__ src, cplx* __restrict__ dst, const FreqDev* __restrict__ fdev,
               int n_theta, int n_tiles, int n_depth, double r_new, double delta_theta,
               EpilogueArgs ea, int step_for_error, DevError* err) {
    extern __shared__ cplx smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
    const int i = t % RW, q = t / RW;
    const int n_chunks = (n_theta + L - 1) / L;
    const bool in_range = q < n_chunks;
    cplx* sP = smem;                 // [nwarps*RW] x 4 scan arrays
    cplx* sY = sP + nwarps * RW;
    cplx* sQ = sY + nwarps * RW;
    cplx* sX = sQ + nwarps * RW;
    cplx* sFirst = sX + nwarps * RW; // [n_chunks*RW] x 2
    cplx* sLast = sFirst + n_chunks * RW;

    const int groups = 8 / RW;
    const int tile = blockIdx.x / groups;
    const int l = tile * 8 + (blockIdx.x % groups) * RW + i;
    const int f = blockIdx.y;
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r_new, delta_theta);
    const RingFactor rf = ring_factor(fd, s);

    const int m0 = q * L;
    const int nvalid = in_range ? min(L, n_theta - m0) : 0;
    const int64_t row_base = (int64_t(f) * n_tiles + tile) * n_theta * 8 + (l & 7);
    cplx v[L];
#pragma unroll
    for (int k = 0; k < L; ++k) v[k] = (k < nvalid) ? ldc_stream(src + row_base + int64_t(m0 + k) * 8) : czero();

    if (rf.diagonal) {
#pragma unroll
        for (int k = 0; k < L; ++k) v[k] = cmul(v[k], rf.scale);
    } else {
        const cplx rho = rf.rho;
        // forward cyclic recurrence w_m = v_m + rho w_{m-1}
        cplx P = cone(), Y = czero();
#pragma unroll
        for (int k = 0; k < L; ++k) if (k < nvalid) { Y = cfma(rho, Y, v[k]); P = cmul(rho, P); }
        cplx Pex, Yex, Ptot, Ytot;
        group_scan_fwd<RW>(P, Y, Pex, Yex, Ptot, Ytot, sP, sY, lane, warp, nwarps, i);
        const cplx wrap = csub(cone(), Ptot);                    // 1 - rho^N
        if (cabs(wrap) < PIVOT_FLOOR && q == 0)
            report_failure(err, fail_key(step_for_error, 1, f, l), n_theta, 1);
        const cplx w_last = cdiv(Ytot, wrap);
        cplx w = cfma(Pex, w_last, Yex);
#pragma unroll
        for (int k = 0; k < L; ++k) if (k < nvalid) { w = cfma(rho, w, v[k]); v[k] = w; }
        // backward cyclic recurrence x_m = w_m + rho x_{m+1}
        cplx Q = cone(), X = czero();
#pragma unroll
        for (int k = L - 1; k >= 0; --k) if (k < nvalid) { X = cfma(rho, X, v[k]); Q = cmul(rho, Q); }
        cplx Qex, Xex, Qtot, Xtot;
        group_scan_bwd<RW>(Q, X, Qex, Xex, Qtot, Xtot, sQ, sX, lane, warp, nwarps, i);
        const cplx x_first = cdiv(Xtot, csub(cone(), Qtot));
        cplx xx = cfma(Qex, x_first, Xex);
#pragma unroll
        for (int k = L - 1; k >= 0; --k) if (k < nvalid) { xx = cfma(rho, xx, v[k]); v[k] = cmul(rf.scale, xx); }
    }
    // boundary: surface row and pad rows are zero (ref marching.py:86)
    if (l == 0 || l >= n_depth) {
#pragma unroll
        for (int k = 0; k < L; ++k) v[k] = czero();
    }
    cplx* dst_row = dst + row_base;
    ring_epilogue<L>(v, q, n_chunks, nvalid, i, RW, m0, l, ea, f, n_theta, n_depth, fd.cy_rhs, s, sFirst, sLast,
                     dst_row, in_range);
}

// ------------------------------------------------ finish / prepare

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

// ----------------------------------- thread-per-system kernels (reference order)

// Depth sweep for media given per (azimuth, depth) at both ranges (ref
// marching.py:109-123 with operators.py:197-241 and tridiag.py:151-178, in
// the reference's operation order).  One thread per (frequency, azimuth);
// x is written to dst (device tiles), cp to `scratch` (device tiles).
__global__ void k_depth_serial(const cplx* __restrict__ src, cplx* __restrict__ dst, cplx* __restrict__ scratch,
                               const cplx* __restrict__ local_now, const cplx* __restrict__ local_new,
                               int64_t local_fstride, int64_t local_mstride, const FreqDev* __restrict__ fdev,
                               int n_freq, int n_theta, int n_tiles, int n_depth, int sector,
                               int* __restrict__ fail_row, double* __restrict__ fail_mag) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n_freq * n_theta) return;
    const int f = gid / n_theta, m = gid % n_theta;
    const FreqDev fd = fdev[f];
    const cplx* ln = local_now + f * local_fstride + m * local_mstride;
    const cplx* lw = local_new + f * local_fstride + m * local_mstride;
    const bool zero_col = sector && (m == 0 || m == n_theta - 1);
    const double two_s = 2.0 * fd.s_z;
    auto at = [&](int l) { return tidx(f, m, l, n_tiles, n_theta); };
    cplx t_prev = czero(), t_cur = ldc(src + at(0));
    cplx cp_prev = czero(), x_prev = czero();
    int failed_row = 0x7fffffff;
    double failed_mag = 0.0;
    for (int l = 0; l < n_depth; ++l) {
        const cplx t_next = (l + 1 < n_depth) ? ldc(src + at(l + 1)) : czero();
        cplx d2;
        if (l == 0) d2 = csub(t_next, crmul(2.0, t_cur));
        else if (l == n_depth - 1) d2 = csub(t_prev, crmul(2.0, t_cur));
        else d2 = cadd(csub(t_next, crmul(2.0, t_cur)), t_prev);
        const cplx xt = cadd(cmul(ln[l], t_cur), crmul(fd.s_z, d2));
        cplx rhs = cadd(t_cur, cmul(fd.cx_rhs, xt));
        if (l == 0 || zero_col) rhs = czero();
        const cplx loc = lw[l];
        const cplx main_l = (l == 0) ? cone() : cadd(cone(), cmul(fd.cx_lhs, mk(loc.re - two_s, loc.im)));
        const cplx denom = (l == 0) ? main_l : csub(main_l, cmul(fd.off_z, cp_prev));
        if (failed_row == 0x7fffffff && cabs(denom) < PIVOT_FLOOR) { failed_row = l; failed_mag = cabs(denom); }
        const cplx inv = crecip(denom);
        const cplx cp = (l == 0 || l == n_depth - 1) ? czero() : cmul(fd.off_z, inv);
        const cplx x = (l == 0) ? cmul(rhs, inv) : cmul(csub(rhs, cmul(fd.off_z, x_prev)), inv);
        stc(dst + at(l), x);
        stc(scratch + at(l), cp);
        cp_prev = cp;
        x_prev = x;
        t_prev = t_cur;
        t_cur = t_next;
    }
    cplx xn = x_prev;
    for (int l = n_depth - 2; l >= 0; --l) {
        const cplx x = csub(ldc(dst + at(l)), cmul(ldc(scratch + at(l)), xn));
        stc(dst + at(l), x);
        xn = x;
    }
    fail_row[gid] = failed_row;
    fail_mag[gid] = failed_mag;
}

// The azimuth matrix of a step is shared by every depth row: factor it
// once per frequency (one thread each), reference order: open with
// identity edge rows (sector, operators.py:263-272) or Sherman-Morrison
// cyclic (tridiag.py:186-212).  Table per frequency: cp[n], inv[n], q[n],
// plus weight alpha/gamma and 1/denom in `ring_tab`.
__global__ void k_factor_azimuth(cplx* __restrict__ cp_tab, cplx* __restrict__ inv_tab, cplx* __restrict__ q_tab,
                                 cplx* __restrict__ ring_tab, const FreqDev* __restrict__ fdev, int n_freq,
                                 int n_theta, double r_new, double delta_theta, int periodic, int step_for_error,
                                 DevError* err) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n_freq) return;
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r_new, delta_theta);
    const cplx diag = csub(cone(), crmul(s, crmul(2.0, fd.cy_lhs)));
    const cplx off = crmul(s, fd.cy_lhs);
    const int n = n_theta;
    cplx* cp = cp_tab + int64_t(f) * n;
    cplx* inv = inv_tab + int64_t(f) * n;
    cplx* qv = q_tab + int64_t(f) * n;
    bool failed = false;
    auto check = [&](cplx d, int row, int rank1) {
        if (!failed && cabs(d) < PIVOT_FLOOR) {
            failed = true;
            report_failure(err, fail_key(step_for_error, 1, f, 0), row, rank1);
        }
    };
    if (!periodic) {
        // main[0] = main[n-1] = 1, sup[0] = 0, sub[n-2] = 0
        for (int k = 0; k < n; ++k) {
            const cplx main_k = (k == 0 || k == n - 1) ? cone() : diag;
            const cplx sub_km1 = (k == n - 1) ? czero() : off;
            const cplx denom = (k == 0) ? main_k : csub(main_k, cmul(sub_km1, cp[k - 1]));
            check(denom, k, 0);
            inv[k] = crecip(denom);
            const cplx sup_k = (k == 0) ? czero() : off;
            cp[k] = (k < n - 1) ? cmul(sup_k, inv[k]) : czero();
        }
        return;
    }
    // Sherman-Morrison: alpha = sub[0], beta = sup[n-1], gamma = -main[0] (or 1)
    const cplx alpha = off, beta = off;
    const cplx gamma = (cabs(diag) > 0.0) ? cneg(diag) : cone();
    for (int k = 0; k < n; ++k) {
        cplx main_k = diag;
        if (k == 0) main_k = csub(diag, gamma);
        if (k == n - 1) main_k = csub(diag, cdiv(cmul(alpha, beta), gamma));
        const cplx denom = (k == 0) ? main_k : csub(main_k, cmul(off, cp[k - 1]));
        check(denom, k, 0);
        inv[k] = crecip(denom);
        cp[k] = (k < n - 1) ? cmul(off, inv[k]) : czero();
    }
    // q = A'^-1 (gamma e_0 + beta e_{n-1})
    cplx x = cmul(gamma, inv[0]);
    qv[0] = x;
    for (int k = 1; k < n; ++k) {
        const cplx rhs = (k == n - 1) ? beta : czero();
        x = cmul(csub(rhs, cmul(off, x)), inv[k]);
        qv[k] = x;
    }
    for (int k = n - 2; k >= 0; --k) qv[k] = csub(qv[k], cmul(cp[k], qv[k + 1]));
    const cplx weight = cdiv(alpha, gamma);
    const cplx denom = cadd(cadd(cone(), qv[0]), cmul(weight, qv[n - 1]));
    check(denom, n, 1);
    ring_tab[2 * f] = weight;
    ring_tab[2 * f + 1] = denom;
}

// One thread per (frequency, depth row): substitutions with the shared
// factorization; writes u into dst (device tiles).
__global__ void k_azimuth_serial(const cplx* __restrict__ src, cplx* __restrict__ dst,
                                 const cplx* __restrict__ cp_tab, const cplx* __restrict__ inv_tab,
                                 const cplx* __restrict__ q_tab, const cplx* __restrict__ ring_tab,
                                 const FreqDev* __restrict__ fdev, int n_freq, int n_theta, int n_tiles,
                                 int n_depth, double r_new, double delta_theta, int periodic) {
    const int nz8 = n_tiles * 8;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n_freq * nz8) return;
    const int f = gid / nz8, l = gid % nz8;
    const int n = n_theta;
    auto at = [&](int m) { return tidx(f, m, l, n_tiles, n_theta); };
    if (l >= n_depth) {
        for (int m = 0; m < n; ++m) stc(dst + at(m), czero());
        return;
    }
    const FreqDev fd = fdev[f];
    const double s = azimuth_scale(fd.k0, r_new, delta_theta);
    const cplx off = crmul(s, fd.cy_lhs);
    const cplx* cp = cp_tab + int64_t(f) * n;
    const cplx* inv = inv_tab + int64_t(f) * n;
    // forward: x_0 = rhs_0 inv_0; x_k = (rhs_k - sub_{k-1} x_{k-1}) inv_k
    cplx x = czero();
    for (int k = 0; k < n; ++k) {
        cplx rhs = ldc(src + at(k));
        if (!periodic && (k == 0 || k == n - 1)) rhs = czero();
        const cplx sub_km1 = (!periodic && k == n - 1) ? czero() : off;
        x = (k == 0) ? cmul(rhs, inv[0]) : cmul(csub(rhs, cmul(sub_km1, x)), inv[k]);
        stc(dst + at(k), x);
    }
    for (int k = n - 2; k >= 0; --k) {
        x = csub(ldc(dst + at(k)), cmul(cp[k], x));
        stc(dst + at(k), x);
    }
    if (periodic) {
        const cplx* qv = q_tab + int64_t(f) * n;
        const cplx weight = ring_tab[2 * f], denom = ring_tab[2 * f + 1];
        const cplx y0 = ldc(dst + at(0)), yl = ldc(dst + at(n - 1));
        const cplx factor = cdiv(cadd(y0, cmul(weight, yl)), denom);
        for (int k = 0; k < n; ++k) stc(dst + at(k), csub(ldc(dst + at(k)), cmul(qv[k], factor)));
    }
}

// solve_batch (ref tridiag.py:248-281): one thread per member, reference
// order; per-member first failing pivot recorded for the host to apply the
// reference's lowest-member rule.
__global__ void k_solve_batch(int n, int members, int cyclic, StridedC sub, StridedC mainv, StridedC sup,
                              StridedC rhs, cplx* __restrict__ x_out, cplx* __restrict__ cp_s,
                              cplx* __restrict__ inv_s, cplx* __restrict__ y_s, cplx* __restrict__ q_s,
                              int* __restrict__ fail_row, double* __restrict__ fail_mag) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= members) return;
    auto A = [&](const StridedC& s, int k) { return ldc(s.ptr + k * s.row_stride + w * s.member_stride); };
    auto S = [&](cplx* base, int k) -> cplx* { return base + int64_t(k) * members + w; };
    int frow = 0x7fffffff;
    double fmag = 0.0;
    auto check = [&](cplx d, int row) {
        if (frow == 0x7fffffff && cabs(d) < PIVOT_FLOOR) { frow = row; fmag = cabs(d); }
    };
    // open system view: sub_o[k] (k < n-1), main_o[k], sup_o[k]
    cplx alpha = czero(), beta = czero(), gamma = cone();
    const int off_shift = cyclic ? 1 : 0;       // cyclic: sub_open = sub[1:]
    if (cyclic) {
        alpha = A(sub, 0);
        beta = A(sup, n - 1);
        const cplx m0 = A(mainv, 0);
        gamma = (cabs(m0) > 0.0) ? cneg(m0) : cone();
    }
    auto main_o = [&](int k) {
        cplx mk_ = A(mainv, k);
        if (cyclic) {
            if (k == 0) mk_ = csub(mk_, gamma);
            if (k == n - 1) mk_ = csub(mk_, cdiv(cmul(alpha, beta), gamma));
        }
        return mk_;
    };
    // factor
    cplx cp_prev = czero();
    for (int k = 0; k < n; ++k) {
        const cplx denom = (k == 0) ? main_o(0) : csub(main_o(k), cmul(A(sub, k - 1 + off_shift), cp_prev));
        check(denom, k);
        if (frow != 0x7fffffff) break;
        const cplx inv = crecip(denom);
        *S(inv_s, k) = inv;
        if (k < n - 1) { cp_prev = cmul(A(sup, k), inv); *S(cp_s, k) = cp_prev; }
    }
    if (frow == 0x7fffffff) {
        // y = A'^-1 rhs (and q = A'^-1 spike when cyclic)
        cplx y = cmul(A(rhs, 0), *S(inv_s, 0));
        cplx qq = cyclic ? cmul(gamma, *S(inv_s, 0)) : czero();
        *S(y_s, 0) = y;
        if (cyclic) *S(q_s, 0) = qq;
        for (int k = 1; k < n; ++k) {
            const cplx sb = A(sub, k - 1 + off_shift);
            y = cmul(csub(A(rhs, k), cmul(sb, y)), *S(inv_s, k));
            *S(y_s, k) = y;
            if (cyclic) {
                const cplx sp = (k == n - 1) ? beta : czero();
                qq = cmul(csub(sp, cmul(sb, qq)), *S(inv_s, k));
                *S(q_s, k) = qq;
            }
        }
        for (int k = n - 2; k >= 0; --k) {
            y = csub(*S(y_s, k), cmul(*S(cp_s, k), y));
            *S(y_s, k) = y;
            if (cyclic) { qq = csub(*S(q_s, k), cmul(*S(cp_s, k), qq)); *S(q_s, k) = qq; }
        }
        if (cyclic) {
            const cplx weight = cdiv(alpha, gamma);
            const cplx denom = cadd(cadd(cone(), *S(q_s, 0)), cmul(weight, *S(q_s, n - 1)));
            check(denom, n);
            if (frow == 0x7fffffff) {
                const cplx factor = cdiv(cadd(*S(y_s, 0), cmul(weight, *S(y_s, n - 1))), denom);
                for (int k = 0; k < n; ++k) stc(x_out + int64_t(w) * n + k, csub(*S(y_s, k), cmul(*S(q_s, k), factor)));
            }
        } else {
            for (int k = 0; k < n; ++k) stc(x_out + int64_t(w) * n + k, *S(y_s, k));
        }
    }
    fail_row[w] = frow;
    fail_mag[w] = fmag;
}

// The reference solves members in fixed 64-wide tiles (tridiag.py:32) and,
// within a tile, stops at the first row where any pivot falls below the
// floor, naming argmin |pivot| over the tile (tridiag.py:145-148); across
// tiles the lowest such member wins (tridiag.py:274-280).  Reproduce that
// rule from per-member (first failing row, |pivot|) records.
__global__ void k_reduce_failures(const int* __restrict__ fail_row, const double* __restrict__ fail_mag, int n_freq,
                                  int members, int step, int sweep, int rank1_row, DevError* err) {
    const int tiles = (members + 63) / 64;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= n_freq * tiles) return;
    const int f = gid / tiles, tile = gid % tiles;
    const int lo = tile * 64, hi = min(members, lo + 64);
    int best_row = 0x7fffffff, best = -1;
    double best_mag = 0.0;
    for (int w = lo; w < hi; ++w) {
        const int r = fail_row[int64_t(f) * members + w];
        const double mg = fail_mag[int64_t(f) * members + w];
        if (r < best_row || (r == best_row && r != 0x7fffffff && mg < best_mag)) { best_row = r; best_mag = mg; best = w; }
    }
    if (best_row != 0x7fffffff) report_failure(err, fail_key(step, sweep, f, best), best_row, best_row == rank1_row);
}

cudaError_t launch_reduce_failures(const int* fail_row, const double* fail_mag, int n_freq, int members, int step,
                                   int sweep, int rank1_row, DevError* err, cudaStream_t stream) {
    const int total = n_freq * ((members + 63) / 64);
    k_reduce_failures<<<(total + 127) / 128, 128, 0, stream>>>(fail_row, fail_mag, n_freq, members, step, sweep,
                                                               rank1_row, err);
    return cudaGetLastError();
}

// Pad the host-given local term [F][n_depth] (any stride) into nothing: the
// factorization kernel reads it directly.  Zero-fill helper for buffers.
__global__ void k_zero(cplx* p, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        stc(p + i, czero());
}

// ------------------------------------------------------------ launchers

template <int L, int RW>
static size_t az_smem(int n_theta, int nthreads) {
    const int n_chunks = (n_theta + L - 1) / L;
    return sizeof(cplx) * (4 * (nthreads / 32) * RW + 2 * n_chunks * RW);
}

static int round32(int x) { return (x + 31) / 32 * 32; }

// choose chunk length L and rows per CTA RW for an azimuth ring of n_theta:
// the widest row group (full 128-B lines) with short chunks that fits 1024 threads
void ring_shape(int n_theta, int* L, int* RW) {
    const int cand_L[2] = {8, 16};
    for (int li = 0; li < 2; ++li)
        for (int rw = 8; rw >= 2; rw /= 2)
            if (round32(rw * ((n_theta + cand_L[li] - 1) / cand_L[li])) <= 512) { *L = cand_L[li]; *RW = rw; return; }
    *L = 0; *RW = 0;   // n_theta > 4096: not supported by the ring kernels
}

#define PE3D_RING_DISPATCH(Lv, RWv, CALL)                       \
    if (L == Lv && RW == RWv) { CALL(Lv, RWv); return cudaGetLastError(); }

cudaError_t launch_azimuth_scan(const LaunchCtx& c, const cplx* src, cplx* dst, double r_new,
                                const EpilogueArgs& ea, int step_for_error) {
    int L, RW;
    ring_shape(c.n_theta, &L, &RW);
    const int n_chunks = (c.n_theta + L - 1) / L;
    const int nthreads = round32(RW * n_chunks);
    dim3 grid(c.n_tiles * (8 / RW), c.n_freq);
#define CALL(Lv, RWv)                                                                              \
    k_azimuth_scan<Lv, RWv><<<grid, nthreads, az_smem<Lv, RWv>(c.n_theta, nthreads), c.stream>>>( \
        src, dst, c.fdev, c.n_theta, c.n_tiles, c.n_depth, r_new, c.delta_theta, ea, step_for_error, c.err)
    PE3D_RING_DISPATCH(8, 8, CALL)
    PE3D_RING_DISPATCH(8, 4, CALL)
    PE3D_RING_DISPATCH(8, 2, CALL)
    PE3D_RING_DISPATCH(16, 8, CALL)
    PE3D_RING_DISPATCH(16, 4, CALL)
    PE3D_RING_DISPATCH(16, 2, CALL)
#undef CALL
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
#define CALL(Lv, RWv)                                                                                 \
    k_finish<Lv, RWv><<<grid, nthreads, sm, c.stream>>>(src, src_tiled, dst, c.fdev, c.n_theta, c.n_tiles, \
                                                        c.n_depth, r, c.delta_theta, ea)
    PE3D_RING_DISPATCH(8, 8, CALL)
    PE3D_RING_DISPATCH(8, 4, CALL)
    PE3D_RING_DISPATCH(8, 2, CALL)
    PE3D_RING_DISPATCH(16, 8, CALL)
    PE3D_RING_DISPATCH(16, 4, CALL)
    PE3D_RING_DISPATCH(16, 2, CALL)
#undef CALL
    return cudaErrorInvalidConfiguration;
}

int depth_cols_per_block(const LaunchCtx& c) {
    // aim for ~8 resident CTAs' worth of columns per SM across the grid
    const int64_t columns = int64_t(c.n_freq) * c.n_theta;
    const int64_t target_ctas = int64_t(c.num_sms) * 4;
    int per = int((columns + target_ctas - 1) / target_ctas);
    if (per < 1) per = 1;
    if (per > 16) per = 16;
    return per;
}

cudaError_t launch_depth_scan(const LaunchCtx& c, const cplx* src, cplx* dst, int cols_per_block) {
    const int nthreads = round32(c.n_tiles);
    const int nwarps = nthreads / 32;
    const size_t sm = sizeof(cplx) * (nwarps * 256 + 6 * nwarps);
    dim3 grid((c.n_theta + cols_per_block - 1) / cols_per_block, c.n_freq);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_depth_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
    }
    k_depth_scan<<<grid, nthreads, sm, c.stream>>>(src, dst, c.loc_tab, c.mul_tab, c.fdev, c.n_theta, c.n_tiles,
                                                   cols_per_block, c.sector);
    return cudaGetLastError();
}

cudaError_t launch_factor_depth(const LaunchCtx& c, const cplx* local, int64_t local_fstride, int step_for_error) {
    k_factor_depth<<<c.n_freq, 1, 0, c.stream>>>(local, local_fstride, c.loc_tab, c.mul_tab, c.fdev, c.n_depth,
                                                 c.n_tiles * 8, step_for_error, c.err);
    return cudaGetLastError();
}

cudaError_t launch_depth_serial(const LaunchCtx& c, const cplx* src, cplx* dst, cplx* scratch, const cplx* local_now,
                                const cplx* local_new, int64_t fstride, int64_t mstride, int* fail_row,
                                double* fail_mag) {
    const int total = c.n_freq * c.n_theta;
    k_depth_serial<<<(total + 127) / 128, 128, 0, c.stream>>>(src, dst, scratch, local_now, local_new, fstride, mstride,
                                                              c.fdev, c.n_freq, c.n_theta, c.n_tiles, c.n_depth,
                                                              c.sector, fail_row, fail_mag);
    return cudaGetLastError();
}

cudaError_t launch_azimuth_serial(const LaunchCtx& c, const cplx* src, cplx* dst, cplx* cp, cplx* inv, cplx* qv,
                                  cplx* ring, double r_new, int step_for_error) {
    k_factor_azimuth<<<(c.n_freq + 31) / 32, 32, 0, c.stream>>>(cp, inv, qv, ring, c.fdev, c.n_freq, c.n_theta, r_new,
                                                                c.delta_theta, !c.sector, step_for_error, c.err);
    const int total = c.n_freq * c.n_tiles * 8;
    k_azimuth_serial<<<(total + 127) / 128, 128, 0, c.stream>>>(src, dst, cp, inv, qv, ring, c.fdev, c.n_freq,
                                                                c.n_theta, c.n_tiles, c.n_depth, r_new,
                                                                c.delta_theta, !c.sector);
    return cudaGetLastError();
}

cudaError_t launch_solve_batch(int n, int members, int cyclic, StridedC sub, StridedC mainv, StridedC sup,
                               StridedC rhs, cplx* x, cplx* cp, cplx* inv, cplx* y, cplx* q, int* fail_row,
                               double* fail_mag, cudaStream_t stream) {
    k_solve_batch<<<(members + 127) / 128, 128, 0, stream>>>(n, members, cyclic, sub, mainv, sup, rhs, x, cp, inv, y, q,
                                                             fail_row, fail_mag);
    return cudaGetLastError();
}

cudaError_t launch_zero(cplx* p, int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    k_zero<<<1184, 256, 0, stream>>>(p, n);
    return cudaGetLastError();
}

}  // namespace pe3d
