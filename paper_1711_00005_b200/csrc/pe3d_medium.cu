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

cudaError_t launch_medium_local(const LaunchCtx& c, const MediumDev& M, cplx* local, double dz, double r) {
    const int64_t total = int64_t(c.n_freq) * c.n_depth * c.n_theta;
    int blocks = int((total + 255) / 256);
    if (blocks > c.num_sms * 16) blocks = c.num_sms * 16;
    k_medium_local<<<blocks, 256, 0, c.stream>>>(M, c.fdev, local, c.n_freq, c.n_theta, c.n_depth, c.delta_theta, dz,
                                                 r);
    return cudaGetLastError();
}

}  // namespace pe3d
