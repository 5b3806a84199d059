// pe3d_serial.cu -- thread-per-system kernels in the reference's operation
// order: depth sweep for media that vary with range/azimuth, the azimuth
// sweep for sector grids, the batched solve_batch, and the reduction that
// applies the reference's lowest-failing-member rule.
//
// Reference: pkg/src/pe3d/tridiag.py:145-281 (Thomas, Sherman-Morrison,
// batch tiles and error rule), operators.py:197-272 (RHS and assembly),
// marching.py:93-136 (step order).

#include "pe3d_device.cuh"
#include "pe3d_internal.h"

#include <cstring>

namespace pe3d {

// ----------------------------------- thread-per-system kernels (reference order)

// Depth sweep for media given per (azimuth, depth) at both ranges (ref
// marching.py:109-123 with operators.py:197-241 and tridiag.py:151-178, in
// the reference's operation order).  One thread per (frequency, azimuth);
// x is written to dst (device tiles), cp to `scratch` (device tiles).
__global__ void k_depth_serial(const cplx* __restrict__ src, cplx* __restrict__ dst, cplx* __restrict__ scratch,
                               const cplx* __restrict__ local_now, const cplx* __restrict__ local_new,
                               int64_t local_fstride, int64_t local_mstride, int64_t local_lstride,
                               const FreqDev* __restrict__ fdev,
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
        const cplx xt = cadd(cmul(ln[l * local_lstride], t_cur), crmul(fd.s_z, d2));
        cplx rhs = cadd(t_cur, cmul(fd.cx_rhs, xt));
        if (l == 0 || zero_col) rhs = czero();
        const cplx loc = lw[l * local_lstride];
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
    // one warp per (frequency, 64-member tile): the tile's failure is its
    // lowest failing row, then the smallest pivot magnitude, then the lowest
    // member -- the order of the reference's sequential scan of the tile
    const int tiles = (members + 63) / 64;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= n_freq * tiles) return;
    const int f = gw / tiles, tile = gw % tiles;
    const int lo = tile * 64, hi = min(members, lo + 64);
    int best_row = 0x7fffffff, best = 0x7fffffff;
    double best_mag = 0.0;
    for (int w = lo + lane; w < hi; w += 32) {
        const int r = fail_row[int64_t(f) * members + w];
        const double mg = fail_mag[int64_t(f) * members + w];
        if (r < best_row || (r == best_row && r != 0x7fffffff && mg < best_mag)) { best_row = r; best_mag = mg; best = w; }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const int r = __shfl_xor_sync(0xffffffffu, best_row, d);
        const double mg = __shfl_xor_sync(0xffffffffu, best_mag, d);
        const int w = __shfl_xor_sync(0xffffffffu, best, d);
        if (r < best_row || (r == best_row && r != 0x7fffffff && (mg < best_mag || (!(best_mag < mg) && w < best)))) {
            best_row = r;
            best_mag = mg;
            best = w;
        }
    }
    if (lane == 0 && best_row != 0x7fffffff)
        report_failure(err, fail_key(step, sweep, f, best), best_row, best_row == rank1_row);
}

cudaError_t launch_reduce_failures(const int* fail_row, const double* fail_mag, int n_freq, int members, int step,
                                   int sweep, int rank1_row, DevError* err, cudaStream_t stream) {
    const int total = n_freq * ((members + 63) / 64) * 32;       // one warp per (frequency, tile)
    k_reduce_failures<<<(total + 127) / 128, 128, 0, stream>>>(fail_row, fail_mag, n_freq, members, step, sweep,
                                                               rank1_row, err);
    return cudaGetLastError();
}

// Pad the host-given local term [F][n_depth] (any stride) into nothing: the
// factorization kernel reads it directly.  Zero-fill helper for buffers.
// March parameters carried by value in the kernel's parameter space (baked into
// the march graph, which is rebuilt whenever they change): copies `bytes` of the
// blob to `dst` and zeroes n_zero int64 (the clamped counters).  One kernel node
// instead of H2D copies from page-locked staging plus a memset, whose copy-engine
// to SM hand-off delayed the first kernel of the march by ~25 us.
template <int CAP>
struct ParamBlob {
    unsigned char b[CAP];
};
struct ParamSegs {
    unsigned char* dst[4];
    int end[4];                 // prefix byte offsets of the segments in the blob (multiples of 4)
    int n;
};
template <int CAP>
__global__ void __launch_bounds__(256) k_params(const __grid_constant__ ParamBlob<CAP> blob, ParamSegs segs,
                                               int64_t* __restrict__ zero, int n_zero) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(blob.b);
    int begin = 0;
    for (int k = 0; k < segs.n; ++k) {
        uint32_t* d = reinterpret_cast<uint32_t*>(segs.dst[k]);
        for (int i = begin / 4 + int(threadIdx.x); i < segs.end[k] / 4; i += blockDim.x) d[i - begin / 4] = s[i];
        begin = segs.end[k];
    }
    if (zero)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
}

cudaError_t launch_params(int n_seg, const void* const* src, const int* bytes, void* const* dst, int64_t* zero,
                          int n_zero, cudaStream_t stream) {
    if (n_seg < 0 || n_seg > 4) return cudaErrorInvalidValue;
    ParamSegs segs{};
    segs.n = n_seg;
    int total = 0;
    for (int k = 0; k < n_seg; ++k) {
        if (bytes[k] % 4 != 0) return cudaErrorInvalidValue;
        total += bytes[k];
        segs.dst[k] = static_cast<unsigned char*>(dst[k]);
        segs.end[k] = total;
    }
    auto go = [&](auto tag) -> cudaError_t {
        using Blob = decltype(tag);
        Blob blob;
        int off = 0;
        for (int k = 0; k < n_seg; ++k) {
            std::memcpy(blob.b + off, src[k], size_t(bytes[k]));
            off += bytes[k];
        }
        k_params<<<1, 256, 0, stream>>>(blob, segs, zero, n_zero);
        return cudaGetLastError();
    };
    if (total <= 2048) return go(ParamBlob<2048>{});
    if (total <= 8192) return go(ParamBlob<8192>{});
    if (total <= 30720) return go(ParamBlob<30720>{});
    return cudaErrorNotSupported;
}

__global__ void k_zero(cplx* p, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        stc(p + i, czero());
}

// ------------------------------------------------------------ launchers

cudaError_t launch_depth_serial(const LaunchCtx& c, const cplx* src, cplx* dst, cplx* scratch, const cplx* local_now,
                                const cplx* local_new, int64_t fstride, int64_t mstride, int64_t lstride, int* fail_row,
                                double* fail_mag) {
    const int total = c.n_freq * c.n_theta;
    k_depth_serial<<<(total + 127) / 128, 128, 0, c.stream>>>(src, dst, scratch, local_now, local_new, fstride, mstride, lstride,
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
