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
    const int F = argc > 1 ? atoi(argv[1]) : 64, NT = 256, NZ = 1024, steps = 4;
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
    // phase k = time from PHASE(k-1) (or the previous column's PHASE(10)) to PHASE(k)
    const char* names[11] = {"freq prologue", "loop/freq check", "wait stage (mbarrier)", "load+halo publish",
                             "BAR halo", "rhs+fwd local+scan", "BAR fwd", "carry+rerun+bwd local+scan", "BAR bwd",
                             "carry+rerun", "stage out+TMA store+next load"};
    double cols = double(F) * NT * steps;
    int ctas = 0;
    for (int b = 0; b < 4096; ++b) if (ph[b * 16 + 2]) ++ctas;
    double per_cta_cols = cols / ctas;
    printf("rc=%d ctas=%d cols/cta/launch=%.1f\n", rc, ctas, per_cta_cols / steps);
    double total = 0;
    for (int k = 0; k < 11; ++k) {
        double s = 0; for (int b = 0; b < 4096; ++b) s += ph[b * 16 + k];
        double per_col = s / cols;
        if (k > 0) total += per_col;
        printf("  %-30s %8.0f cycles/column\n", names[k], per_col);
    }
    printf("  %-30s %8.0f cycles/column\n", "TOTAL (excl. prologue)", total);
    const char* once[2] = {"first setup (per CTA)", "store drain (per CTA)"};
    for (int k = 11; k < 13; ++k) {
        double s = 0; for (int b = 0; b < 4096; ++b) s += ph[b * 16 + k];
        printf("  %-30s %8.0f cycles per CTA per launch\n", once[k - 11], s / ctas / steps);
    }
    return 0;
}
