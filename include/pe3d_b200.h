/*
 * pe3d_b200.h -- C ABI of the B200 (sm_100a) range-marching library
 * libpe3d_b200.so.  Plain C types only: pointers, sizes, doubles; no torch
 * or CUDA types in the signatures (streams are passed as void*).
 *
 * The reference package (pe3d, pure Python + numpy) has no FFI; its
 * "operator API" is a handful of Python functions.  Each entry point below
 * names the reference interface it replaces; the Python host
 * (paper_1711_00005_b200/) binds them with ctypes and keeps the reference's
 * names, argument meaning and exceptions.
 *
 * Layouts at the boundary are the reference's: a slab is [n_theta][n_depth]
 * complex128, depth fastest (ref environment.py:199-222); TL stacks are
 * [S][n_theta][n_depth] float64 (ref marching.py:185-193); tridiagonal
 * batches are (row, member) structure-of-arrays (ref tridiag.py:82-142).
 * Frequencies are an outer batch dimension.  The device-side field layout
 * is private.
 *
 * Conventions: every function returns a pe3d_status; on failure the
 * optional pe3d_error record is filled.  Nothing aborts or exits.  A handle
 * owns device scratch and must be used from one host thread at a time.
 */
#ifndef PE3D_B200_H
#define PE3D_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PE3D_ABI_VERSION 1

#if defined(__GNUC__)
#define PE3D_API __attribute__((visibility("default")))
#else
#define PE3D_API
#endif

typedef struct { double re, im; } pe3d_c128;

typedef enum {
    PE3D_OK = 0,
    PE3D_SINGULAR = 1,      /* SingularSystemError / StepError (ref errors.py:33-60) */
    PE3D_BAD_ARGUMENT = 2,  /* shape / invariant violation detected by the library */
    PE3D_CUDA_ERROR = 3     /* no device, launch or copy failure */
} pe3d_status;

typedef enum { PE3D_PERIODIC = 0, PE3D_SECTOR = 1 } pe3d_topology;  /* ref environment.py:24-26 */
typedef enum { PE3D_SWEEP_DEPTH = 0, PE3D_SWEEP_AZIMUTH = 1 } pe3d_sweep;

/* Failure record.  For a failed step it carries StepError(range_index,
 * sweep, member_index) with the SingularSystemError(pivot, member) cause
 * (ref marching.py:122-131, tridiag.py:274-280: lowest failing member). */
typedef struct {
    int32_t range_index;   /* step number j+1, or -1 outside a step (solve_batch) */
    int32_t sweep;         /* pe3d_sweep */
    int32_t member;        /* lowest failing batch member */
    int32_t pivot;         /* elimination row of the failing pivot */
    int32_t rank1;         /* 1: the cyclic rank-1 correction was singular */
    int32_t frequency;     /* index of the failing frequency inside the batch */
    char message[208];
} pe3d_error;

/* Grid and march controls (ref Grid3D environment.py:34-90, RunOptions
 * config.py:71-95, run_frequency marching.py:144-193). */
typedef struct {
    int32_t n_freq;         /* frequencies in this batch (>= 1) */
    int32_t n_theta;        /* azimuth points (>= 3) */
    int32_t n_depth;        /* depth points (>= 3) */
    int32_t topology;       /* pe3d_topology */
    int32_t n_steps;        /* range steps to take (>= 0), after max_range */
    int32_t output_stride;  /* TL sample every stride steps; sample 0 = input slab */
    int32_t first_index;    /* range index j of the input slab (StepError numbering) */
    int32_t flags;          /* PE3D_FLAG_* */
    double delta_r, delta_theta, delta_z;
    double r_start;         /* grid r_start: the slab after step s is at r_start + (first_index+s+1)*delta_r
                               (ref Grid3D.range_at, environment.py:89-90) */
    double r_input;         /* range_m of the input slab (ref FieldSlab.range_m) */
} pe3d_grid;

#define PE3D_FLAG_NO_GRAPH   1   /* launch the step loop directly instead of a CUDA graph */
#define PE3D_FLAG_SERIAL     2   /* use the thread-per-system kernels (reference op order) */
#define PE3D_FLAG_PROFILE    4   /* no graph; CUDA events around every launch (see pe3d_profile_last) */
#define PE3D_FLAG_STARTER_COLUMN 8  /* pe3d_march_*: u0 is [F][n_depth], the same column at every azimuth
                                       (the reference's Gaussian starter, ref environment.py:270-284) */

/* Per-frequency step coefficients (ref operators.py:31-62, StepCoefficients). */
typedef struct {
    double k0;
    pe3d_c128 cx_lhs, cx_rhs, cy_lhs, cy_rhs;
} pe3d_coeffs;

PE3D_API int pe3d_abi_version(void);
PE3D_API int pe3d_device_count(int32_t* count);

PE3D_API int pe3d_handle_create(int32_t device, void** handle, pe3d_error* err);
PE3D_API int pe3d_handle_destroy(void* handle);

/* Number of TL samples a march of n_steps with this stride records:
 * 1 + floor(n_steps / stride)  (ref marching.py:167-183). */
PE3D_API int32_t pe3d_sample_count(int32_t n_steps, int32_t output_stride);

/*
 * pe3d_march_host -- replaces run_frequency (ref marching.py:144-193) for
 * range-independent media, for a batch of frequencies (the body of
 * frequency_farm, ref parallel.py:126-185).  HOST buffers; the copies are
 * part of the call.
 *   local      [F][n_depth]            n^2 - 1 (ref operators.py:93)
 *   u0         [F][n_theta][n_depth]   input slab at range r_start + first_index*delta_r
 *   u_final    [F][n_theta][n_depth]   slab after n_steps (NULL: not returned)
 *   tl         [F][S][n_theta][n_depth] transmission loss (NULL: not recorded)
 *   snapshots  [F][S][n_theta][n_depth] field at each TL sample (NULL: off)
 *   clamped    [F]                     exactly-zero TL samples (ref environment.py:308-315)
 */
PE3D_API int pe3d_march_host(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs,
                    const pe3d_c128* local, const pe3d_c128* u0,
                    pe3d_c128* u_final, double* tl, pe3d_c128* snapshots,
                    int64_t* clamped, pe3d_error* err);

/* Same with DEVICE pointers, enqueued on `stream` (a cudaStream_t, NULL =
 * legacy default stream).  Synchronises the stream before returning so
 * that failures can be reported. */
PE3D_API int pe3d_march_device(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs,
                      const pe3d_c128* d_local, const pe3d_c128* d_u0,
                      pe3d_c128* d_u_final, double* d_tl, pe3d_c128* d_snapshots,
                      int64_t* d_clamped, void* stream, pe3d_error* err);

/*
 * Extended medium for on-device generation of the local term n^2 - 1
 * (paper_1711_00005_b200/medium.py LayeredMedium; BASELINE cfg3): water
 * profile (piecewise linear, clamped), fluid bottom below the bathymetry
 * h(r, theta) = max(depth0 - r tan(slope) cos(theta), min_depth) blended by a
 * tanh step of width interface_width, attenuation in dB per wavelength,
 * absorbing layer over the last sponge_points rows, density through the
 * effective-index term, and an optional perturbation lattice
 * [lat_nx][lat_ny][lat_nz] (trilinear in x = r cos t, y = r sin t, z).
 * All pointers are HOST pointers; the library uploads them.
 */
typedef struct {
    double c0;
    int32_t n_profile;
    const double* profile_z;
    const double* profile_c;
    double water_density, water_alpha;
    double bottom_speed, bottom_density, bottom_alpha;
    double bathy_depth0, bathy_slope_deg, bathy_min_depth;
    int32_t sponge_points;
    double sponge_max_alpha;
    double interface_width;
    const double* lattice;          /* NULL: no perturbation */
    int32_t lat_nx, lat_ny, lat_nz;
    double lat_extent_h, lat_spacing_h, lat_spacing_v;
} pe3d_medium;

/*
 * pe3d_march_medium_host -- run_frequency (ref marching.py:144-193) for
 * media that vary with range and azimuth: the local term is generated on
 * the device every step (at r_j for the explicit side, r_{j+1} for the
 * implicit side, ref marching.py:110,116), and each depth column is
 * factored per step.  Buffers as in pe3d_march_host (host pointers).
 */
PE3D_API int pe3d_march_medium_host(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs,
                                    const pe3d_medium* medium, const pe3d_c128* u0, pe3d_c128* u_final,
                                    double* tl, pe3d_c128* snapshots, int64_t* clamped, pe3d_error* err);

/*
 * pe3d_step_general_host -- replaces range_step (ref marching.py:93-136)
 * for media that vary with range and azimuth: one step with explicit
 * per-point local terms at the old and the new range, host buffers.
 *   local_now, local_new [F][n_theta][n_depth]; u_in, u_out [F][n_theta][n_depth]
 * grid->n_steps must be 1; grid->first_index is j of u_in.  tl_out
 * [F][n_theta][n_depth] and clamped [F] (NULL: skipped) receive the TL of
 * u_out at the new range.
 */
PE3D_API int pe3d_step_general_host(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs,
                           const pe3d_c128* local_now, const pe3d_c128* local_new,
                           const pe3d_c128* u_in, pe3d_c128* u_out,
                           double* tl_out, int64_t* clamped, pe3d_error* err);

/*
 * pe3d_solve_batch_host -- replaces solve_batch (ref tridiag.py:248-281):
 * `members` systems of size n, one topology.  Diagonals and rhs are
 * (row, member) SoA with element (k, i) at [k*row_stride + i*member_stride];
 * a stride of 0 broadcasts (the reference's broadcast views).  Off-diagonals
 * have n rows (cyclic, corners at sub[0] / sup[n-1]) or n-1 rows (open).
 * Output x is [members][n].
 */
typedef struct {
    const pe3d_c128* ptr;
    int64_t row_stride;
    int64_t member_stride;
} pe3d_strided;

PE3D_API int pe3d_solve_batch_host(void* handle, int32_t n, int32_t members, int32_t cyclic,
                          pe3d_strided sub, pe3d_strided main_diag, pe3d_strided sup,
                          pe3d_strided rhs, pe3d_c128* x, pe3d_error* err);

/*
 * Slab-decomposed march of ONE large grid over nranks GPUs (SURVEY.md §8(e),
 * BASELINE cfg5): the depth sweep runs on azimuth slabs (nranks column
 * ranges), the azimuth sweep on depth slabs (nranks tile ranges), joined
 * twice per step by an equal-split all-to-all (NCCL send/recv pairs, or the
 * peer-direct stores of pe3d_march_slab_p2p below), with
 * the ring sweep reading/writing the rank-chunked layout the all-to-all
 * delivers (no pack/unpack kernels).  No reference counterpart: the
 * reference never splits one frequency's grid.
 *
 * nccl_id == NULL: nranks VIRTUAL ranks driven by this process on its one
 *   device (peer-direct stores into the other virtual ranks' buffers, or
 *   device-to-device copies when PE3D_SLAB_COPY is set or the shape does not
 *   allow peer output); u0 / u_final are full
 *   [n_theta][n_depth] slabs and tl is [S][n_theta][n_depth].
 * nccl_id != NULL: this process is rank `rank` of nranks (one GPU each; id
 *   from pe3d_slab_unique_id on rank 0, broadcast by the caller); u0 /
 *   u_final are this rank's depth slab [n_theta][n_depth/nranks] and tl is
 *   [S][n_theta][n_depth/nranks].
 * Requirements: n_freq == 1, periodic, n_theta % nranks == 0,
 * n_depth % (8*nranks) == 0.  *ms_steps receives the device time of the
 * step loop (CUDA events), for measurement.
 */
PE3D_API int pe3d_slab_unique_id(void* out, int32_t bytes);
PE3D_API int pe3d_march_slab(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs, int32_t nranks,
                             int32_t rank, const void* nccl_id, const pe3d_c128* local, const pe3d_c128* u0,
                             pe3d_c128* u_final, double* tl, int64_t* clamped, double* ms_steps, pe3d_error* err);

/*
 * Peer-direct (fused) transposes of the slab march: the depth sweep of rank
 * p stores its output tiles straight into the azimuth-sweep input of every
 * rank (NVLink peer memory mapped with CUDA IPC), and the azimuth sweep
 * stores its next temp straight into the depth-sweep inputs; device-side
 * counters order the sweeps across ranks.  No all-to-all and no send/receive
 * buffers.  (The virtual-rank mode of pe3d_march_slab uses the same kernels
 * with all ranks' buffers on one device, unless PE3D_SLAB_COPY is set.)
 *
 * pe3d_slab_p2p_export: allocate this rank's slab buffers for `grid` on the
 *   handle's device, reset its counters, and write PE3D_SLAB_IPC_BYTES bytes
 *   of CUDA IPC handles to `out`.
 * pe3d_march_slab_p2p: `blobs` holds the nranks exported blobs in rank
 *   order.  Every rank must have exported (its counters reset) before any
 *   rank starts marching -- the caller barriers in between.  u0 / u_final /
 *   tl are this rank's depth slab as in pe3d_march_slab.
 * Requirements as pe3d_march_slab, plus n_depth / (8 nranks) % 32 == 0 and
 * nranks <= 16.
 */
#define PE3D_SLAB_IPC_BYTES 192
PE3D_API int pe3d_slab_p2p_export(void* handle, const pe3d_grid* grid, int32_t nranks, int32_t rank, void* out,
                                  pe3d_error* err);
PE3D_API int pe3d_march_slab_p2p(void* handle, const pe3d_grid* grid, const pe3d_coeffs* coeffs, int32_t nranks,
                                 int32_t rank, const void* blobs, const pe3d_c128* local, const pe3d_c128* u0,
                                 pe3d_c128* u_final, double* tl, int64_t* clamped, double* ms_steps, pe3d_error* err);

/*
 * pe3d_profile_last -- kernel timings of the last march run with
 * PE3D_FLAG_PROFILE on this handle: ms[k] is the summed CUDA-event time and
 * launches[k] the launch count of kernel class k (0 depth sweep, 1 azimuth
 * sweep, 2 everything else).  No reference counterpart (measurement only).
 */
PE3D_API int pe3d_profile_last(void* handle, double* ms, int32_t* launches);

/*
 * pe3d_last_launches -- number of kernels the last pe3d_march_device /
 * pe3d_march_host call on this handle launched, graph replays included
 * (measurement only).
 */
PE3D_API int pe3d_last_launches(void* handle, int64_t* launches);

/*
 * pe3d_last_copy_bytes -- bytes the last pe3d_march_host call on this handle
 * moved host-to-device and device-to-host (a grouped march of column
 * starters sends one azimuth row of the starting TL sample and replicates it
 * on the host, so d2h can be less than the size of the result buffers).
 * Measurement only.
 */
PE3D_API int pe3d_last_copy_bytes(void* handle, int64_t* h2d, int64_t* d2h);

/*
 * pe3d_profile_launches -- the individual CUDA-event times (ms, launch order)
 * of kernel class `cls` (0 depth sweep, 1 azimuth sweep, 2 other, 3 unused
 * since the split rings became one kernel) in the last PE3D_FLAG_PROFILE
 * march on this handle; writes min(count, capacity) entries and the full count
 * to *count (measurement only: steady-state launches for the bench's roofline).
 */
PE3D_API int pe3d_profile_launches(void* handle, int32_t cls, double* ms, int32_t capacity, int32_t* count);

/*
 * pe3d_host_alloc / pe3d_host_free -- page-locked host memory for the
 * caller's TL and slab stacks (cudaHostAlloc).  A page-locked TL stack lets
 * pe3d_march_host stream the samples to the host while the march runs; the
 * Python drop-in (run_frequency / frequency_farm, ref marching.py:144-193,
 * parallel.py:143-185) returns its results in such memory.
 */
PE3D_API int pe3d_host_alloc(uint64_t bytes, void** ptr);
PE3D_API int pe3d_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* PE3D_B200_H */
