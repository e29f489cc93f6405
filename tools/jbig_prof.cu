// Phase profile of the reference-order Jacobi grid (sgp_jbig.cuh) at d = 2083 on a seeded
// diagonally dominant matrix.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -DSGP_JBIG_PROF -o tools/jbig_prof tools/jbig_prof.cu
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2511_06407_b200/csrc/sgp_core.cuh"
#include "../paper_2511_06407_b200/csrc/sgp_jbig.cuh"

int main(int argc, char **argv) {
    const int d = argc > 1 ? atoi(argv[1]) : 2083;
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> A((size_t)d * d), V((size_t)d * d, 0.0);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j <= i; ++j) {
            const double v = (i == j) ? 10.0 * nd(g) : 0.02 * nd(g);
            A[(size_t)i * d + j] = A[(size_t)j * d + i] = v;
        }
    for (int i = 0; i < d; ++i) V[(size_t)i * d + i] = 1.0;
    double *dA, *dV;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dV, V.size() * 8);
    cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
    JbWS w;
    const int caps[2] = {1, 30};
    for (int c : caps) {
        cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(jb_prof, z, sizeof(z));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        const int sw = jb_jacobi(w, dA, dV, d, 1e-13 * 1e3, 1e-13 * 1e3 / d, c, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long p[16];
        cudaMemcpyFromSymbol(p, jb_prof, sizeof(p));
        const double nwin = (double)p[8];
        printf("cap %d: sweeps %d, %.1f ms, windows %.0f\n", c, sw, ms, nwin);
        const char *names[] = {"chain window", "chain start barrier", "lookahead", "lookahead owner wait",
                               "io publish", "io deferred load", "io prefetch", "end barrier (warp 0)",
                               "windows", "lookahead wait for chain", "lookahead fold+stores"};
        for (int i = 0; i < 11; ++i)
            if (i != 8) printf("  %-24s %10.0f cycles/window\n", names[i], p[i] / nwin);
    }
    return 0;
}
