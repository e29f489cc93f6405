// Phase cycles of the tridiagonalisation panel kernel (CTA 0), per column.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSGP_DC_PROF_CYC -o tools/dc_prof tools/dc_prof.cu
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../paper_2511_06407_b200/csrc/sgp_dc.cuh"

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 2083;
    std::vector<double> h((size_t)n * n);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) h[(size_t)i * n + j] = h[(size_t)j * n + i] = nd(g);
    double *dh, *lam, *psi;
    cudaMalloc(&dh, sizeof(double) * n * n);
    cudaMalloc(&lam, sizeof(double) * n);
    cudaMalloc(&psi, sizeof(double) * n * n);
    cudaMemcpy(dh, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    DcWS w;
    dc_eigh(w, dh, n, n, lam, psi, n, 0);
    cudaDeviceSynchronize();
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(dc_prof, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dc_eigh(w, dh, n, n, lam, psi, n, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long p[8];
    cudaMemcpyFromSymbol(p, dc_prof, sizeof(p));
    const char *names[] = {"prologue (column k0)", "grid barriers (2)", "P (reflector, v staging)",
                           "S (symv + dots)", "W (reductions, w, next column)", "-"};
    printf("n=%d total %.2f ms (%s)\n", n, ms, cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 5; ++i) printf("  %-32s %8.0f cycles/column\n", names[i], (double)p[i] / (n - 1));
    return 0;
}
