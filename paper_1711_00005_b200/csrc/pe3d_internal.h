// pe3d_internal.h -- launch interface between the C ABI (pe3d_abi.cu) and
// the kernels (pe3d_depth.cu, pe3d_ring.cu, pe3d_serial.cu, pe3d_medium.cu,
// pe3d_slab.cu).  Not part of the public ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "pe3d_device.cuh"

namespace pe3d {

struct StridedC {
    const cplx* ptr;
    int64_t row_stride;
    int64_t member_stride;
};

// What the ring epilogue writes besides nothing: TL sample, snapshot,
// final slab (reference layout), and the next step's temp (device tiles).
// Peer-direct transposes of the slab march: at most this many ranks.
constexpr int MAX_PEERS = 16;

struct EpilogueArgs {
    double* tl;             // [F][n_samples][n_theta][n_depth] or null
    cplx* snap;             // [F][n_samples][n_theta][n_depth] or null
    cplx* final_out;        // [F][n_theta][n_depth] or null
    int64_t* clamped;       // [F]
    const double* w_abs;    // [F] |w(r)| of this sample
    int n_samples;
    int sample;
    int periodic;
    int write_temp;
    // Slab march: the ring tiles of this rank hold global
    // rows row_offset + l, and rings may be stored rank-chunked: element m of
    // the ring of (f, tile) is at ring_base + m*8 + (m / chunk_cols)*chunk_gap.
    // Standard layout: row_offset 0, chunk_cols = n_theta, chunk_gap = 0.
    int row_offset;
    int chunk_cols;
    int64_t chunk_gap;
    // Peer-direct output (fused K2 -> K1 transpose): when peer[0] is set, the
    // next temp of azimuth m, local tile t, row r goes to
    // peer[m / chunk_cols] + (t * chunk_cols + m % chunk_cols) * 8 + r, i.e.
    // straight into the depth-sweep input of the rank owning azimuth chunk
    // m / chunk_cols (this rank's chunk of it).
    cplx* peer[MAX_PEERS];
    // march prologue only: the starter u0 is one column per frequency ([F][n_depth],
    // PE3D_FLAG_STARTER_COLUMN) instead of a [F][n_theta][n_depth] slab
    int src_column;
    // march prologue only, with src_column: write the first temp as one column per
    // frequency ([F][n_tiles][8]) here instead of the azimuth-uniform field
    cplx* temp_col;
};

// Destination of the next temp of ring element (m, row r) of local tile t.
__host__ __device__ __forceinline__ cplx* peer_elem(const EpilogueArgs& ea, int m, int tile, int r) {
    const int p = m / ea.chunk_cols;
    return ea.peer[p] + (int64_t(tile) * ea.chunk_cols + (m - p * ea.chunk_cols)) * 8 + r;
}

__host__ __device__ __forceinline__ int64_t ring_base(int f, int tile, int n_tiles, int n_theta, int chunk_cols) {
    return (int64_t(f) * n_tiles * n_theta + int64_t(tile) * chunk_cols) * 8;
}
__host__ __device__ __forceinline__ int64_t ring_off(int m, int chunk_cols, int64_t chunk_gap) {
    return int64_t(m) * 8 + (chunk_gap ? int64_t(m / chunk_cols) * chunk_gap : 0);
}

// Device view of an extended medium (pe3d_medium in the public header).
struct MediumDev {
    double c0;
    int n_prof;
    const double* pz;
    const double* pc;
    double rho_w, alpha_w, c_b, rho_b, alpha_b;
    double h0, tan_slope, hmin;
    int sponge_n;
    double sponge_max;
    double w;
    const double* lat;
    int nx, ny, nz;
    double ext_h, dh, dv;
    double eta;
};

struct LaunchCtx {
    int n_freq, n_theta, n_depth, n_tiles;
    int sector;
    int num_sms;
    double delta_theta;
    const FreqDev* fdev;
    cplx* loc_tab;          // [F][n_tiles*8]
    cplx* mul_tab;          // [F][n_tiles*8]
    // Per-frequency setup of the column depth sweep (k_depth_tma), built once
    // per march by launch_factor_depth when set (null: computed in-kernel):
    // [F][k1_stride(nt)], nt = threads per column, layout in k1_img / k1_stride.
    cplx* k1_tab;
    DevError* err;
    cudaStream_t stream;
    // Peer-direct output of the depth sweep (fused K1 -> K2 transpose): when
    // n_peers > 0, tiles [q*peer_tiles, (q+1)*peer_tiles) of every column go to
    // peer_dst[q], laid out [tile][column][8] (n_theta columns).
    // Launch the step-loop sweeps with programmatic stream serialization
    // (PDL): a sweep's independent prologue overlaps the previous sweep's tail.
    int pdl;
    // Split long columns (SURVEY §8(a) a11-a12 for n_depth = 128*8*split rows,
    // cfg5): when split >= 2 the depth sweep solves every 1024-row sub-column on
    // its own with zero carries (virtual frequency fs = f*split + s, the
    // k_depth_tma kernel of 1024-row columns), records per (fs, column) its
    // zero-carry bottom y and top x in sp_tot, k_split_carry turns those into
    // the exact carries entering every sub-column (sp_cd, lane-ordered for the
    // azimuth sweep), and the azimuth sweep applies x = x0 + a_l cin + q_l din
    // to every element it loads (sp_aq: per (f, row) responses to unit carries;
    // sp_pa: per (f, s) product of the multipliers and the top response).
    int split;
    cplx* sp_tot;           // [F*split][n_theta][2]
    cplx* sp_aq;            // [F][n_tiles*8][2]
    cplx* sp_pa;            // [F*split][3]: P_s, A_s, (a_span, q_span) rows needing the correction
    cplx* sp_cd;            // [F][split][2][n_theta]
    // First step after a column starter's prologue (depth_sweep_takes_column): the depth
    // sweep reads its input from one column per frequency, [F][n_tiles][8], instead of the
    // azimuth-uniform field the prologue would otherwise have to write
    const cplx* src_col;
    int n_peers;
    int peer_tiles;
    cplx* peer_dst[MAX_PEERS];
};

// k1_tab record of one frequency for nt threads per column (nt % 32 == 0):
//   [0, 10 nt + nt/32)     shared-memory image: scan multipliers mf[4][nt],
//                          mb[4][nt], pincf[nt], pincb[nt], warp products spw
//   [img, img + 8 nt)      folded RHS coefficients A'_l, thread-contiguous
//   [img + 8 nt, +2 nt)    first-level scan multipliers P0f[nt], P0b[nt]
//   img + 10 nt            beta
__host__ __device__ __forceinline__ int k1_img(int nt) { return (10 * nt + nt / 32 + 7) / 8 * 8; }
__host__ __device__ __forceinline__ int k1_stride(int nt) { return (k1_img(nt) + 10 * nt + 1 + 7) / 8 * 8; }
constexpr int K1_TAB_MAX_TILES = 128;   // columns the table path covers (one 128-thread CTA)
// Long columns (k_depth_tma_cluster, n_tiles = 128 * n_sub, n_sub <= 8): one
// record per (frequency, sub-column CTA) of 128 threads:
//   [0, 12*128 + 4)        shared-memory image: mf[4][128], mb[4][128], pincf,
//                          pincb, pexc, psuf [128] each, warp products spw[4]
//   [K1C_IMG, +8*128)      folded RHS coefficients A'_l, thread-contiguous
//   [K1C_IMG + 1024, +256) P0f[128], P0b[128];  K1C_IMG + 1280: beta, + 1281: Pcta
constexpr int K1C_IMG = (12 * 128 + 4 + 7) / 8 * 8;
constexpr int K1C_STRIDE = (K1C_IMG + 10 * 128 + 2 + 7) / 8 * 8;
constexpr int K1C_MAX_SUB = 8;
// k1_tab elements a march of F frequencies needs (0: no table path for this column length)
__host__ __device__ __forceinline__ int64_t k1_tab_elems(int n_freq, int n_tiles) {
    if (n_tiles <= K1_TAB_MAX_TILES) return int64_t(n_freq) * k1_stride((n_tiles + 31) / 32 * 32);
    if (n_tiles % 128 == 0 && n_tiles / 128 <= K1C_MAX_SUB) return int64_t(n_freq) * (n_tiles / 128) * K1C_STRIDE;
    return 0;
}

// cudaLaunchKernelEx with the programmatic-serialization attribute when pdl is set.
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Occupancy of a launch configuration (clusters when cluster > 1, else CTAs
// per SM), cached per (kernel, device, dynamic smem, cluster size); 0 on error.
int cached_occupancy(const void* kern, size_t bytes, int cluster, int nthr, cudaLaunchConfig_t* cfg);
bool encode_swizzled_map(CUtensorMap* tm, const void* base, int rank, const uint64_t* dims,
                         const uint64_t* strides, const uint32_t* box, int swizzle_bytes);
cudaError_t launch_slab_signal(unsigned long long* const* flags, int n, cudaStream_t s);
cudaError_t launch_slab_wait(const unsigned long long* flag, unsigned long long target, DevError* err,
                             cudaStream_t s);
void ring_shape(int n_theta, int* L, int* RW);
int ring_table_elems(int n_theta);   // complex entries per (step, frequency) ring table
cudaError_t launch_factor_depth(const LaunchCtx& c, const cplx* local, int64_t local_fstride, int step_for_error);
cudaError_t launch_factor_depth_scan(const LaunchCtx& c, const cplx* local, int64_t local_fstride, int step_for_error);
cudaError_t launch_depth_scan(const LaunchCtx& c, const cplx* src, cplx* dst);
bool depth_sweep_takes_column(const LaunchCtx& c);
// Split-column plan for a march (0: no split) and the per-step carry kernel.
int depth_split_plan(const LaunchCtx& c, int periodic);
cudaError_t launch_split_carry(const LaunchCtx& c);
// segment length of the TMA ring kernel serving n_theta (the lane order of sp_cd)
int ring_segment(int n_theta);
cudaError_t launch_ring_setup(const LaunchCtx& c, cplx* table, int n_steps, int first_index, double r_start,
                              double delta_r);
cudaError_t launch_azimuth_scan(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step, double r_new,
                                const EpilogueArgs& ea);
cudaError_t launch_finish(const LaunchCtx& c, const cplx* src, int src_tiled, cplx* dst, double r,
                          const EpilogueArgs& ea);
// Split rings (pe3d_ring.cu, k_azimuth_tma SEG/HALO): a cluster-sized ring swept segment by
// segment on all SMs, each segment taking its carries from `span` neighbouring points per side
// loaded with it.  sring_segment: segment length (0: the ring is not split).
int sring_segment(int n_theta);
int sring_halo_max_span();
cudaError_t launch_azimuth_halo(const LaunchCtx& c, const cplx* src, cplx* dst, const cplx* table_step,
                                const EpilogueArgs& ea, int span);
cudaError_t launch_depth_serial(const LaunchCtx& c, const cplx* src, cplx* dst, cplx* scratch, const cplx* local_now,
                                const cplx* local_new, int64_t fstride, int64_t mstride, int64_t lstride, int* fail_row,
                                double* fail_mag);
cudaError_t launch_medium_local(const LaunchCtx& c, const MediumDev& M, cplx* local, double dz, double r);
cudaError_t launch_medium_local_tiles(const LaunchCtx& c, const MediumDev& M, cplx* local, double dz, double r);
cudaError_t launch_depth_medium_scan(const LaunchCtx& c, const MediumDev& M, const cplx* src, cplx* dst,
                                     const cplx* local_now, cplx* local_next, double dz, double r_new, int* fail_row,
                                     double* fail_mag, int precomputed);
cudaError_t launch_azimuth_serial(const LaunchCtx& c, const cplx* src, cplx* dst, cplx* cp, cplx* inv, cplx* qv,
                                  cplx* ring, double r_new, int step_for_error);
cudaError_t launch_solve_batch(int n, int members, int cyclic, StridedC sub, StridedC mainv, StridedC sup,
                               StridedC rhs, cplx* x, cplx* cp, cplx* inv, cplx* y, cplx* q, int* fail_row,
                               double* fail_mag, cudaStream_t stream);
cudaError_t launch_zero(cplx* p, int64_t n, cudaStream_t stream);
// copy up to 4 small host segments (<= 30 KB in total, carried in the kernel's
// parameters) to their device destinations and zero n_zero int64 at `zero`;
// cudaErrorNotSupported when they are too large
cudaError_t launch_params(int n_seg, const void* const* src, const int* bytes, void* const* dst, int64_t* zero,
                          int n_zero, cudaStream_t stream);
cudaError_t launch_reduce_failures(const int* fail_row, const double* fail_mag, int n_freq, int members, int step,
                                   int sweep, int rank1_row, DevError* err, cudaStream_t stream);

}  // namespace pe3d
