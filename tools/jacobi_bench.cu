// Cycle cost per rotation of the bit-exact cyclic Jacobi (sgp_core.cuh) on a
// near-diagonal d x d matrix, with A / V in shared or global memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/jacobi_bench tools/jacobi_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../paper_2511_06407_b200/csrc/sgp_core.cuh"

__global__ void bench(const double *A0, double *Ag, double *Vg, int d, int mode, long long *cyc, int *sw) {
    extern __shared__ double sm[];
    double *red = sm;
    double *As = sm + 64;
    double *Vs = (mode & 1) ? As : As + d * d;
    double *A = (mode & 1) ? Ag + blockIdx.x * d * d : As;
    double *V = (mode & 2) ? Vg + blockIdx.x * d * d : Vs;
    for (int i = threadIdx.x; i < d * d; i += blockDim.x) {
        A[i] = A0[i];
        V[i] = (i / d == i % d) ? 1.0 : 0.0;
    }
    __syncthreads();
    long long t0 = clock64();
    int s = jacobi_cyclic(A, V, d, 1e-13 * 100.0, 1e-13 * 100.0 / d, 30, red, Vg + 1024 * d * d + blockIdx.x * sgp_jacobi_log_doubles(d));
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *cyc = t1 - t0;
        *sw = s;
    }
}

int main(int argc, char **argv) {
    int d = argc > 1 ? atoi(argv[1]) : 34;
    std::vector<double> a(d * d);
    srand(1);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j <= i; ++j) {
            double v = (i == j) ? 1.0 + i : 1e-3 * ((rand() % 2000) / 1000.0 - 1.0);
            a[i * d + j] = a[j * d + i] = v;
        }
    double *A0, *Ag, *Vg;
    long long *cyc, hc;
    int *sw, hs;
    cudaMalloc(&A0, d * d * 8);
    cudaMalloc(&Ag, 2048 * d * d * 8);
    cudaMalloc(&Vg, 2048 * (d * d + sgp_jacobi_log_doubles(d)) * 8);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sw, 4);
    cudaMemcpy(A0, a.data(), d * d * 8, cudaMemcpyHostToDevice);
    size_t smem_full = (64 + 2 * d * d) * 8;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::min<size_t>(smem_full, 227 * 1024));
    const char *names[] = {"A smem, V smem", "A glob, V smem", "A smem, V glob", "A glob, V glob"};
    // optional argv[2]: one block size only, A and V in shared memory, one CTA (for ncu)
    const int only = argc > 2 ? atoi(argv[2]) : 0;
    const int only_mode = argc > 3 ? atoi(argv[3]) : 0;
    std::vector<int> nts = only ? std::vector<int>{only} : std::vector<int>{32, 64, 256};
    for (int nt : nts) {
        for (int mode = only ? only_mode : 0; mode < (only ? only_mode + 1 : 4); ++mode) {
            const size_t smem = (64 + ((mode & 1) ? 0 : d * d) + ((mode & 2) ? 0 : d * d)) * 8;
            if (smem > 227 * 1024) continue;
            for (int blocks : {1, 148}) {
                bench<<<blocks, nt, smem>>>(A0, Ag, Vg, d, mode, cyc, sw);
                cudaDeviceSynchronize();
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                bench<<<blocks, nt, smem>>>(A0, Ag, Vg, d, mode, cyc, sw);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(&hs, sw, 4, cudaMemcpyDeviceToHost);
                double rot = (double)hs * d * (d - 1) / 2;
                printf("d=%d nt=%3d %-16s blocks=%4d sweeps=%d  %.0f cyc/rotation  (%.3f ms)\n", d, nt, names[mode],
                       blocks, hs, hc / rot, ms);
#ifdef SGP_JPROF
                long long jp[8];
                cudaMemcpyFromSymbol(jp, sgp_jprof, sizeof(jp));
                if (jp[3]) printf("   warp0 per iteration: barrier %.0f, chain %.0f, tail %.0f cycles; %lld it, %lld rotated; sweep total %.0f per it\n",
                                  (double)jp[0] / jp[3], (double)jp[1] / jp[3], (double)jp[2] / jp[3], jp[3], jp[4], (double)jp[5] / jp[3]);
                if (jp[3]) printf("   row start barrier %.0f, row end barrier %.0f cycles per iteration\n", (double)jp[6] / jp[3], (double)jp[7] / jp[3]);
                long long z8[8] = {0};
                cudaMemcpyToSymbol(sgp_jprof, z8, sizeof(z8));
#endif
            }
        }
    }
    return 0;
}
