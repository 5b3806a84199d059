// Phase-timing driver for the cfg4 depth sweep (k_depth_tma) (built with -DPE3D_PHASE_TIMING):
// marches cfg4-shaped data (F frequencies, argv[1], default 64) for a few steps through the C ABI and prints the
// mean cycles per column of each phase for CTA-thread 0.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/pe3d_b200.h"
namespace pe3d { extern __device__ unsigned long long g_phase[4096][16]; }
int main(int argc, char** argv) {
    const int F = argc > 1 ? atoi(argv[1]) : 64, NT = argc > 2 ? atoi(argv[2]) : 256, NZ = argc > 3 ? atoi(argv[3]) : 1024,
              steps = 4;
    pe3d_grid g{F, NT, NZ, PE3D_PERIODIC, steps, steps, 0, PE3D_FLAG_NO_GRAPH, 1.0, 6.283185307179586 / NT, 0.25, 1.0, 1.0};
    std::vector<pe3d_coeffs> co(F);
    for (int f = 0; f < F; ++f) {
        double k0 = 2 * 3.141592653589793 * (50.0 * (1 + f * 0.1)) / 1500.0;
        double q = k0 * 1.0 / 4.0;
        co[f] = {k0, {0.25, -q}, {0.25, q}, {0, -q}, {0, q}};
    }
    std::vector<pe3d_c128> local(size_t(F) * NZ, {-0.01, 0.0}), u0(size_t(F) * NT * NZ, {1e-3, 0.0});
    void* h; pe3d_error err;
    pe3d_handle_create(0, &h, &err);
    pe3d_c128 *dl, *du, *df; double* dtl; long long* dc;
    cudaMalloc(&dl, local.size() * 16); cudaMalloc(&du, u0.size() * 16); cudaMalloc(&df, u0.size() * 16);
    cudaMalloc(&dtl, size_t(F) * 2 * NT * NZ * 8); cudaMalloc(&dc, F * 8);
    cudaMemcpy(dl, local.data(), local.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(du, u0.data(), u0.size() * 16, cudaMemcpyHostToDevice);
    int rc = pe3d_march_device(h, &g, co.data(), dl, du, df, dtl, nullptr, (int64_t*)dc, nullptr, &err);
    std::vector<unsigned long long> ph(4096 * 16);
    cudaMemcpyFromSymbol(ph.data(), pe3d::g_phase, ph.size() * 8);
    // phase k = time from the previous PHASE mark to PHASE(k), thread 0 of each CTA
    const bool cluster = NZ > 1024;     // k_depth_tma_cluster (long columns) instead of k_depth_tma
    const char* names_tma[16] = {"freq switch", "loop/freq check", "wait stage (mbarrier)", "load+halo publish",
                                 "BAR halo", "rhs+fwd local+scan", "BAR fwd", "carry+rerun+bwd local+scan", "BAR bwd",
                                 "carry+rerun", "stage out+TMA store+next load", "", "", "", "", ""};
    const char* names_cl[16] = {"freq setup", "loop top (halo cp.async)", "wait stage (mbarrier)", "load+halo publish",
                                "BAR halo", "rhs+fwd local+scan", "BAR fwd", "cin+rerun+bwd local+scan", "BAR bwd",
                                "carry+push bwd totals", "stage out+TMA store+next load", "din+rerun", "",
                                "WAIT fwd cluster totals", "WAIT bwd cluster totals", "carry+push fwd totals"};
    const char** names = cluster ? names_cl : names_tma;
    double cols = double(F) * NT * steps;
    int ctas = 0;
    for (int b = 0; b < 4096; ++b) if (ph[b * 16 + 2]) ++ctas;   // CTAs that waited on a stage
    // a cluster CTA handles sub-columns: columns per CTA = cluster size x columns / CTAs
    const double cl_size = cluster ? NZ / 1024.0 : 1.0;
    const double per_cta_cols = cols * cl_size / ctas;
    printf("rc=%d ctas=%d cols/cta/launch=%.1f%s\n", rc, ctas, per_cta_cols / steps, cluster ? " (1024-row sub-columns)" : "");
    double total = 0;
    for (int k = 0; k < 16; ++k) {
        if (!names[k][0]) continue;
        double s = 0; for (int b = 0; b < 4096; ++b) s += ph[b * 16 + k];
        const double per_col = s / (cols * cl_size);
        if (k > 0) total += per_col;
        printf("  %-32s %8.0f cycles/column\n", names[k], per_col);
    }
    printf("  %-32s %8.0f cycles/column\n", "TOTAL (excl. phase 0)", total);
    if (!cluster) {
        const char* once[2] = {"first setup (per CTA)", "store drain (per CTA)"};
        for (int k = 11; k < 13; ++k) {
            double s = 0; for (int b = 0; b < 4096; ++b) s += ph[b * 16 + k];
            printf("  %-32s %8.0f cycles per CTA per launch\n", once[k - 11], s / ctas / steps);
        }
    }
    return 0;
}
