// pe3d_medium.cu -- on-device generation of the depth operator's local term
// n^2 - 1 for media that vary with range and azimuth (BASELINE cfg3:
// bathymetry h(r, theta) and a seeded sound-speed perturbation).
//
// The formulas are the ones of paper_1711_00005_b200/medium.py
// (LayeredMedium.index_squared / index_grid), evaluated in the same order:
//   c_w   = interp(z; profile) + trilinear(lattice; r cos t, r sin t, z)
//   n2_w  = ((c0/c_w)(1 + i eta alpha_w))^2,  n2_b = ((c0/c_b)(1 + i eta alpha_b))^2
//   h     = max(h0 - r tan(slope) cos t, h_min),  T = tanh((z - h)/w),  H = (1 + T)/2
//   n2    = (1 - H) n2_w + H n2_b,  times (1 + i eta alpha_sponge(l))^2
//   n2   += [rho''/(2 rho) - 3/4 (rho'/rho)^2] / k0^2   (density contrast)
//   local = sqrt(n2)^2 - 1   (the reference squares n: operators.py:93)
// A range step then needs the local term at r_j (explicit side) and at
// r_{j+1} (implicit side); the march keeps the previous step's grid, so one
// grid is generated per step.

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

namespace pe3d {

__device__ __forceinline__ double interp_clamped(const double* __restrict__ xs, const double* __restrict__ ys, int n,
                                                 double x) {
    if (n == 1 || x <= xs[0]) return ys[0];
    if (x >= xs[n - 1]) return ys[n - 1];
    int lo = 0, hi = n - 1;                        // np.interp: xs[lo] <= x < xs[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xs[mid] <= x) lo = mid; else hi = mid;
    }
    const double slope = (ys[hi] - ys[lo]) / (xs[hi] - xs[lo]);   // numpy.interp's order
    return slope * (x - xs[lo]) + ys[lo];
}

__device__ __forceinline__ double lattice_sample(const MediumDev& M, double x, double y, double z) {
    const double hx = double(M.nx) - 1.000001, hy = double(M.ny) - 1.000001, hz = double(M.nz) - 1.000001;
    const double fx = fmin(fmax((x + M.ext_h) / M.dh, 0.0), hx);
    const double fy = fmin(fmax((y + M.ext_h) / M.dh, 0.0), hy);
    const double fz = fmin(fmax(z / M.dv, 0.0), hz);
    const int ix = int(fx), iy = int(fy), iz = int(fz);
    const double tx = fx - ix, ty = fy - iy, tz = fz - iz;
    double out = 0.0;
#pragma unroll
    for (int ox = 0; ox < 2; ++ox)
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int oz = 0; oz < 2; ++oz) {
                const double wx = ox ? tx : 1.0 - tx, wy = oy ? ty : 1.0 - ty, wz = oz ? tz : 1.0 - tz;
                out = out + wx * wy * wz * __ldg(M.lat + (int64_t(ix + ox) * M.ny + (iy + oy)) * M.nz + (iz + oz));
            }
    return out;
}

__device__ __forceinline__ cplx medium_local(const MediumDev& M, double r, double theta, int l, int n_depth, double dz,
                                             double k0) {
    const double z = l * dz;
    double cw = interp_clamped(M.pz, M.pc, M.n_prof, z);
    if (M.lat) cw = cw + lattice_sample(M, r * cos(theta), r * sin(theta), z);
    const cplx aw = mk(M.c0 / cw, (M.c0 / cw) * (M.eta * M.alpha_w));
    const cplx n2w = cmul(aw, aw);
    const cplx ab = mk(M.c0 / M.c_b, (M.c0 / M.c_b) * (M.eta * M.alpha_b));
    const cplx n2b = cmul(ab, ab);
    double h = M.h0 - (r * M.tan_slope) * cos(theta);
    h = fmax(h, M.hmin);
    const double t = tanh((z - h) / M.w);
    const double H = 0.5 * (1.0 + t);
    cplx n2 = cadd(crmul(1.0 - H, n2w), crmul(H, n2b));
    if (M.sponge_n > 0 && l >= n_depth - M.sponge_n) {
        const double a = M.sponge_max * double(l - (n_depth - M.sponge_n) + 1) / M.sponge_n;
        const cplx s = mk(1.0, M.eta * a);
        n2 = cmul(n2, cmul(s, s));
    }
    if (M.rho_b != M.rho_w) {
        const double jump = M.rho_b - M.rho_w;
        const double sech2 = 1.0 - t * t;
        const double rho = M.rho_w + jump * H;
        const double d1 = jump * sech2 / (2.0 * M.w);
        const double d2 = -jump * sech2 * t / (M.w * M.w);
        const double q = d1 / rho;
        n2.re = n2.re + (d2 / (2.0 * rho) - 0.75 * (q * q)) / (k0 * k0);
    }
    const cplx n = csqrt(n2);
    const cplx nn = cmul(n, n);
    return mk(nn.re - 1.0, nn.im);
}

// local[f][l][m] (azimuth fastest, so the column-serial solver reads it
// coalesced) at range r for every frequency.
__global__ void k_medium_local(MediumDev M, const FreqDev* __restrict__ fdev, cplx* __restrict__ local, int n_freq,
                               int n_theta, int n_depth, double delta_theta, double dz, double r) {
    const int64_t total = int64_t(n_freq) * n_depth * n_theta;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int m = int(i % n_theta);
        const int64_t fl = i / n_theta;
        const int l = int(fl % n_depth), f = int(fl / n_depth);
        stc(local + i, medium_local(M, r, m * delta_theta, l, n_depth, dz, fdev[f].k0));
    }
}

// ---------------------------------------------------------------------------
// Depth sweep for media that vary per column and per step (cfg3), fully
// parallel along depth.  One CTA per (frequency, azimuth) column, thread t
// owns depth tile t (8 rows).  Per step and column:
//   1. local_new (at r_{j+1}) is evaluated in-kernel and stored in the device
//      tile layout for the next step, where it is this step's local_now;
//   2. the Thomas pivots d_l = main_l - off^2/d_{l-1} (ref tridiag.py:161-166)
//      come from the continuant p_l = main_l p_{l-1} - off^2 p_{l-2},
//      d_l = p_l/p_{l-1}: a product of 2x2 transfer matrices, computed per
//      tile and chained by a Kogge-Stone scan of normalized matrices (only
//      ratios matter, so every product is rescaled by its largest entry);
//   3. the substitutions run as in the range-independent sweep, with
//      column-dependent multipliers m_l = -off/d_l scanned on the fly.
struct M2 {
    cplx a, b, c, d;                 // [[a, b], [c, d]]
};

__device__ __forceinline__ M2 m2mul(const M2& x, const M2& y) {     // x * y
    M2 r;
    r.a = cfma(x.a, y.a, cmul(x.b, y.c));
    r.b = cfma(x.a, y.b, cmul(x.b, y.d));
    r.c = cfma(x.c, y.a, cmul(x.d, y.c));
    r.d = cfma(x.c, y.b, cmul(x.d, y.d));
    return r;
}

__device__ __forceinline__ M2 m2norm(M2 x) {
    const double m = fmax(fmax(fmax(fabs(x.a.re), fabs(x.a.im)), fmax(fabs(x.b.re), fabs(x.b.im))),
                          fmax(fmax(fabs(x.c.re), fabs(x.c.im)), fmax(fabs(x.d.re), fabs(x.d.im))));
    if (m > 0.0 && isfinite(m)) {
        const double inv = 1.0 / m;
        x.a = crmul(inv, x.a); x.b = crmul(inv, x.b); x.c = crmul(inv, x.c); x.d = crmul(inv, x.d);
    }
    return x;
}

__device__ __forceinline__ M2 shfl_up_m2(const M2& x, int d) {
    return M2{shfl_up(x.a, d), shfl_up(x.b, d), shfl_up(x.c, d), shfl_up(x.d, d)};
}

template <bool PRE, int MAXT>
__global__ void __launch_bounds__(MAXT)
k_depth_medium_scan(MediumDev M, const cplx* __restrict__ src, cplx* __restrict__ dst,
                    const cplx* __restrict__ local_now, cplx* __restrict__ local_next, const FreqDev* __restrict__ fdev,
                    int n_theta, int n_tiles, int n_depth, double delta_theta, double dz, double r_new, int sector,
                    int* __restrict__ fail_row, double* __restrict__ fail_mag) {
    __shared__ M2 sM[16];
    __shared__ cplx sPY[16][2];
    __shared__ cplx sUp[16], sDn[16];
    __shared__ int sFail;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
    const int col = blockIdx.x, f = blockIdx.y;
    const bool active = t < n_tiles;
    const FreqDev fd = fdev[f];
    const double theta = col * delta_theta;
    const int64_t line = (int64_t(f) * n_tiles + t) * n_theta * 8 + int64_t(col) * 8;   // this thread's tile line
    if (t == 0) sFail = 0x7fffffff;

    // ---- loads, in-kernel medium at r_{j+1}
    cplx x[8], ln[8], lw[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int l = 8 * t + i;
        const bool real_row = active && l < n_depth;
        x[i] = active ? ldc(src + line + i) : czero();
        ln[i] = real_row ? ldc(local_now + line + i) : czero();
        if (PRE) {                                  // local_next filled by k_medium_local_tiles
            lw[i] = real_row ? ldc(local_next + line + i) : czero();
        } else {
            lw[i] = real_row ? medium_local(M, r_new, theta, l, n_depth, dz, fd.k0) : czero();
            if (active) stc(local_next + line + i, lw[i]);
        }
    }
    // ---- halos
    cplx up = shfl_up(x[7], 1), dn = shfl_down(x[0], 1);
    if (lane == 31) sUp[warp] = x[7];
    if (lane == 0) sDn[warp] = x[0];
    __syncthreads();
    if (lane == 0) up = warp > 0 ? sUp[warp - 1] : czero();
    if (lane == 31) dn = warp < nwarps - 1 ? sDn[warp + 1] : czero();
    if (t == 0) up = czero();

    // ---- pivots by the continuant scan
    const cplx off2 = cmul(fd.off_z, fd.off_z);
    const double two_s = 2.0 * fd.s_z;
    cplx mainv[8];
    M2 T{cone(), czero(), czero(), cone()};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int l = 8 * t + i;
        mainv[i] = cadd(cone(), cmul(fd.cx_lhs, mk(lw[i].re - two_s, lw[i].im)));
        M2 Ml;
        if (l == 0 || !active || l >= n_depth) Ml = M2{cone(), czero(), czero(), cone()};   // surface / pads: identity
        else Ml = M2{mainv[i], cneg(l == 1 ? czero() : off2), cone(), czero()};
        T = m2norm(m2mul(Ml, T));
    }
    // inclusive scan: prefix product over tiles 0..t (applied right to left)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const M2 Tp = shfl_up_m2(T, d);
        if (lane >= d) T = m2norm(m2mul(T, Tp));
    }
    if (lane == 31) sM[warp] = T;
    __syncthreads();
    M2 Cw{cone(), czero(), czero(), cone()};
    for (int w = 0; w < warp; ++w) Cw = m2norm(m2mul(sM[w], Cw));
    M2 Tin = shfl_up_m2(m2norm(m2mul(T, Cw)), 1);          // product over all previous tiles
    if (lane == 0) Tin = Cw;
    // state [p_l; p_{l-1}] entering this tile: Tin * [1; 0]
    cplx pa = Tin.a, pb = Tin.c;
    cplx mult[8];
    int my_fail = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int l = 8 * t + i;
        cplx inv = cone();
        if (l == 0) {
            pa = cone(); pb = czero();                      // d_0 = main_0 = 1 (surface row)
            mult[i] = czero();
        } else if (active && l < n_depth) {
            const cplx na = csub(cmul(mainv[i], pa), cmul(l == 1 ? czero() : off2, pb));
            const cplx d = cdiv(na, pa);                    // d_l = p_l / p_{l-1}
            if (my_fail == 0x7fffffff && cabs(d) < PIVOT_FLOOR) my_fail = l;
            inv = crecip(d);
            pb = pa;
            pa = na;
            const double sc = fmax(fabs(pa.re), fabs(pa.im));
            if (sc > 0.0 && isfinite(sc)) { pa = crmul(1.0 / sc, pa); pb = crmul(1.0 / sc, pb); }
            mult[i] = cneg(cmul(fd.off_z, inv));
        } else {
            mult[i] = czero();
        }
        // ---- b_l = inv_l * rhs_l (rhs with local_now, ref operators.py:115-139,210; row 0 -> 0)
        const cplx um = i ? x[i - 1] : up;
        const cplx upp = i < 7 ? x[i + 1] : dn;
        const cplx d2 = cadd(csub(upp, cadd(x[i], x[i])), um);
        const cplx xt = cadd(cmul(ln[i], x[i]), crmul(fd.s_z, d2));
        cplx rhs = cadd(x[i], cmul(fd.cx_rhs, xt));
        if (l == 0 || !active || l >= n_depth || (sector && (col == 0 || col == n_theta - 1))) rhs = czero();
        lw[i] = cmul(inv, rhs);                             // reuse lw for b
    }
    if (my_fail != 0x7fffffff) atomicMin(&sFail, my_fail);
    // ---- forward y_l = b_l + m_l y_{l-1}; backward x_l = y_l + m_l x_{l+1} (pair scans on the fly)
    cplx P = cone(), Y = czero();
#pragma unroll
    for (int i = 0; i < 8; ++i) { Y = cfma(mult[i], Y, lw[i]); P = cmul(mult[i], P); }
    if (!active) P = cone();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const cplx Pp = shfl_up(P, d), Yp = shfl_up(Y, d);
        if (lane >= d) { Y = cfma(P, Yp, Y); P = cmul(P, Pp); }
    }
    if (lane == 31) { sPY[warp][0] = P; sPY[warp][1] = Y; }
    __syncthreads();
    cplx C = czero();
    for (int w = 0; w < warp; ++w) C = cfma(sPY[w][0], C, sPY[w][1]);
    cplx y = shfl_up(cfma(P, C, Y), 1);
    if (lane == 0) y = C;
#pragma unroll
    for (int i = 0; i < 8; ++i) { y = cfma(mult[i], y, lw[i]); lw[i] = y; }
    cplx Q = cone(), X = czero();
#pragma unroll
    for (int i = 7; i >= 0; --i) { X = cfma(mult[i], X, lw[i]); Q = cmul(mult[i], Q); }
    if (!active) Q = cone();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const cplx Qn = shfl_down(Q, d), Xn = shfl_down(X, d);
        if (lane + d < 32) { X = cfma(Q, Xn, X); Q = cmul(Q, Qn); }
    }
    __syncthreads();
    if (lane == 0) { sPY[warp][0] = Q; sPY[warp][1] = X; }
    __syncthreads();
    cplx D = czero();
    for (int w = nwarps - 1; w > warp; --w) D = cfma(sPY[w][0], D, sPY[w][1]);
    cplx xv = shfl_down(cfma(Q, D, X), 1);
    if (lane == 31) xv = D;
#pragma unroll
    for (int i = 7; i >= 0; --i) { xv = cfma(mult[i], xv, lw[i]); lw[i] = xv; }
    if (active) {
#pragma unroll
        for (int i = 0; i < 8; ++i) stc(dst + line + i, lw[i]);
    }
    if (t == 0) {
        fail_row[int64_t(f) * n_theta + col] = sFail;
        fail_mag[int64_t(f) * n_theta + col] = 0.0;
    }
}

cudaError_t launch_depth_medium_scan(const LaunchCtx& c, const MediumDev& M, const cplx* src, cplx* dst,
                                     const cplx* local_now, cplx* local_next, double dz, double r_new, int* fail_row,
                                     double* fail_mag, int precomputed) {
    const int nthreads = (c.n_tiles + 31) / 32 * 32;
    if (nthreads > 512) return cudaErrorNotSupported;
    dim3 grid(c.n_theta, c.n_freq);
    // the precomputed-medium instantiation carries no medium code: this kernel
    // runs at low occupancy and its size showed up as instruction-cache stalls
    // (columns of up to 128 tiles also get the register budget of a 128-thread CTA: no spills)
    auto kern = nthreads <= 128 ? (precomputed ? k_depth_medium_scan<true, 128> : k_depth_medium_scan<false, 128>)
                                : (precomputed ? k_depth_medium_scan<true, 512> : k_depth_medium_scan<false, 512>);
    kern<<<grid, nthreads, 0, c.stream>>>(M, src, dst, local_now, local_next, c.fdev, c.n_theta, c.n_tiles, c.n_depth,
                                          c.delta_theta, dz, r_new, c.sector, fail_row, fail_mag);
    return cudaGetLastError();
}

// Range-independent depth factorization (tables of K1), one CTA per
// frequency, thread t owning RPT consecutive rows: the same continuant scan as
// above replaces the single-thread Thomas recurrence of k_factor_depth (ref
// tridiag.py:151-167): d_l = p_l / p_(l-1), m_l = -off / d_l, loc_tab = the
// local term, pads zero; the first pivot below the floor is reported with
// the reference's (row, member) convention.  It sits on the march's setup
// path (before the first depth sweep), which is latency bound: RPT = 2 (512
// threads for 1024 rows) and a warp scan of the warp products replace the
// 8-row serial chains and the serial warp loop (cfg4, 8 frequencies: 17 ->
// ~6 us standalone).
template <int RPT>
__global__ void __launch_bounds__(512)
k_factor_depth_scan(const cplx* __restrict__ local, int64_t local_fstride, cplx* __restrict__ loc_tab,
                    cplx* __restrict__ mul_tab, const FreqDev* __restrict__ fdev, int n_depth, int n_rows,
                    int step_for_error, DevError* err) {
    __shared__ M2 sM[32];
    __shared__ int sFail;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = int(blockDim.x) >> 5;
    const int f = blockIdx.x;
    const bool active = t * RPT < n_rows;
    const FreqDev fd = fdev[f];
    if (t == 0) sFail = 0x7fffffff;
    const cplx off2 = cmul(fd.off_z, fd.off_z);
    const double two_s = 2.0 * fd.s_z;
    cplx mainv[RPT];
    M2 T{cone(), czero(), czero(), cone()};
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int l = RPT * t + i;
        const bool real_row = active && l < n_depth;
        const cplx loc = real_row ? ldc(local + f * local_fstride + l) : czero();
        if (active) stc(loc_tab + int64_t(f) * n_rows + l, loc);
        mainv[i] = cadd(cone(), cmul(fd.cx_lhs, mk(loc.re - two_s, loc.im)));
        M2 Ml;
        if (l == 0 || !real_row) Ml = M2{cone(), czero(), czero(), cone()};   // surface / pads: identity
        else Ml = M2{mainv[i], cneg(l == 1 ? czero() : off2), cone(), czero()};
        T = m2norm(m2mul(Ml, T));
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const M2 Tp = shfl_up_m2(T, d);
        if (lane >= d) T = m2norm(m2mul(T, Tp));
    }
    if (lane == 31) sM[warp] = T;
    __syncthreads();
    if (warp == 0) {                                        // exclusive scan of the warp products
        M2 W = lane < nwarps ? sM[lane] : M2{cone(), czero(), czero(), cone()};
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const M2 Wp = shfl_up_m2(W, d);
            if (lane >= d) W = m2norm(m2mul(W, Wp));
        }
        M2 E = shfl_up_m2(W, 1);
        if (lane == 0) E = M2{cone(), czero(), czero(), cone()};
        __syncwarp();
        if (lane < nwarps) sM[lane] = E;
    }
    __syncthreads();
    const M2 Cw = sM[warp];
    M2 Tin = shfl_up_m2(m2norm(m2mul(T, Cw)), 1);
    if (lane == 0) Tin = Cw;
    cplx pa = Tin.a, pb = Tin.c;
    int my_fail = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int l = RPT * t + i;
        cplx mult = czero();
        if (l == 0) {
            pa = cone(); pb = czero();                      // d_0 = main_0 = 1 (surface row)
        } else if (active && l < n_depth) {
            const cplx na = csub(cmul(mainv[i], pa), cmul(l == 1 ? czero() : off2, pb));
            const cplx d = cdiv(na, pa);                    // d_l = p_l / p_(l-1)
            if (my_fail == 0x7fffffff && cabs(d) < PIVOT_FLOOR) my_fail = l;
            pb = pa;
            pa = na;
            const double sc = fmax(fabs(pa.re), fabs(pa.im));
            if (sc > 0.0 && isfinite(sc)) { pa = crmul(1.0 / sc, pa); pb = crmul(1.0 / sc, pb); }
            mult = cneg(cmul(fd.off_z, crecip(d)));
        }
        if (active) stc(mul_tab + int64_t(f) * n_rows + l, mult);
    }
    if (my_fail != 0x7fffffff) atomicMin(&sFail, my_fail);
    __syncthreads();
    if (t == 0 && sFail != 0x7fffffff) report_failure(err, fail_key(step_for_error, 0, f, 0), sFail, 0);
}

cudaError_t launch_factor_depth_scan(const LaunchCtx& c, const cplx* local, int64_t local_fstride,
                                     int step_for_error) {
    const int n_rows = c.n_tiles * 8;
    auto go = [&](auto kern, int rpt) -> cudaError_t {
        const int nthreads = (n_rows / rpt + 31) / 32 * 32;
        kern<<<c.n_freq, nthreads, 0, c.stream>>>(local, local_fstride, c.loc_tab, c.mul_tab, c.fdev, c.n_depth,
                                                  n_rows, step_for_error, c.err);
        return cudaGetLastError();
    };
    if (n_rows <= 1024) return go(k_factor_depth_scan<2>, 2);     // <= 512 threads each
    if (n_rows <= 2048) return go(k_factor_depth_scan<4>, 4);
    if (n_rows <= 4096) return go(k_factor_depth_scan<8>, 8);
    return cudaErrorNotSupported;
}

// local term in the device tile layout (the starter range of the scan path)
__global__ void k_medium_local_tiles(MediumDev M, const FreqDev* __restrict__ fdev, cplx* __restrict__ local,
                                     int n_freq, int n_theta, int n_tiles, int n_depth, double delta_theta, double dz,
                                     double r) {
    const int64_t total = int64_t(n_freq) * n_tiles * n_theta * 8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int e = int(i & 7);
        const int64_t rest = i >> 3;
        const int m = int(rest % n_theta);
        const int64_t ft = rest / n_theta;
        const int tile = int(ft % n_tiles), f = int(ft / n_tiles);
        const int l = tile * 8 + e;
        stc(local + i, l < n_depth ? medium_local(M, r, m * delta_theta, l, n_depth, dz, fdev[f].k0) : czero());
    }
}

cudaError_t launch_medium_local_tiles(const LaunchCtx& c, const MediumDev& M, cplx* local, double dz, double r) {
    const int64_t total = int64_t(c.n_freq) * c.n_tiles * c.n_theta * 8;
    int blocks = int((total + 255) / 256);
    if (blocks > c.num_sms * 16) blocks = c.num_sms * 16;
    k_medium_local_tiles<<<blocks, 256, 0, c.stream>>>(M, c.fdev, local, c.n_freq, c.n_theta, c.n_tiles, c.n_depth,
                                                       c.delta_theta, dz, r);
    return cudaGetLastError();
}

cudaError_t launch_medium_local(const LaunchCtx& c, const MediumDev& M, cplx* local, double dz, double r) {
    const int64_t total = int64_t(c.n_freq) * c.n_depth * c.n_theta;
    int blocks = int((total + 255) / 256);
    if (blocks > c.num_sms * 16) blocks = c.num_sms * 16;
    k_medium_local<<<blocks, 256, 0, c.stream>>>(M, c.fdev, local, c.n_freq, c.n_theta, c.n_depth, c.delta_theta, dz,
                                                 r);
    return cudaGetLastError();
}

}  // namespace pe3d
