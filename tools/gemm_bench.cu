// Correctness and throughput of the DMMA GEMM (sgp_gemm.cuh).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_bench tools/gemm_bench.cu -lcublas
// Throughput cases use random operands (zero operands draw less power and run at higher clocks)
// and time cuBLAS DGEMM on the same shapes (row-major C = A B as column-major C^T = B^T A^T).
#include <cublas_v2.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2511_06407_b200/csrc/sgp_gemm.cuh"

static void ref(const GemmArgs &g, const std::vector<double> &A, const std::vector<double> &B,
                const std::vector<double> &s, std::vector<double> &C) {
    for (int m = 0; m < g.M; ++m)
        for (int n = 0; n < g.N; ++n) {
            double acc = 0;
            for (int k = 0; k < g.K; ++k) {
                double a = g.TA ? A[(size_t)k * g.lda + m] : A[(size_t)m * g.lda + k];
                double b = g.TB ? B[(size_t)n * g.ldb + k] : B[(size_t)k * g.ldb + n];
                acc += a * (s.empty() ? 1.0 : s[k]) * b;
            }
            C[(size_t)m * g.ldc + n] = acc;
        }
}

__global__ void k_fill(double *p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)i * 2654435761u ^ seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
    }
}

int main() {
    int fails = 0;
    cublasHandle_t hb;
    cublasCreate(&hb);
    for (int ta = 0; ta < 2; ++ta)
        for (int tb = 0; tb < 2; ++tb)
            for (int sc = 0; sc < 2; ++sc) {
                int M = 67, N = 45, K = 83;
                GemmArgs g{};
                g.M = M; g.N = N; g.K = K; g.TA = ta; g.TB = tb;
                g.lda = ((ta ? M : K) + 1) & ~1; g.ldb = ((tb ? K : N) + 1) & ~1; g.ldc = (N + 1) & ~1;
                g.alpha = 1; g.beta = 0;
                std::vector<double> A((size_t)(ta ? K : M) * g.lda), B((size_t)(tb ? N : K) * g.ldb),
                    S(sc ? K : 0), C((size_t)M * g.ldc), R((size_t)M * g.ldc);
                for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
                for (auto &v : B) v = rand() / (double)RAND_MAX - 0.5;
                for (auto &v : S) v = rand() / (double)RAND_MAX;
                double *dA, *dB, *dC, *dS = nullptr;
                cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
                cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
                cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
                if (sc) { cudaMalloc(&dS, K * 8); cudaMemcpy(dS, S.data(), K * 8, cudaMemcpyHostToDevice); }
                g.A = dA; g.B = dB; g.C = dC; g.scale = dS;
                gemm_launch(g, 0);
                cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
                ref(g, A, B, S, R);
                double err = 0;
                for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n)
                    err = fmax(err, fabs(C[(size_t)m * g.ldc + n] - R[(size_t)m * g.ldc + n]));
                printf("TA=%d TB=%d scale=%d max err %.3e\n", ta, tb, sc, err);
                fails += err > 1e-12;
                cudaFree(dA); cudaFree(dB); cudaFree(dC); if (dS) cudaFree(dS);
            }
    for (int up = 0; up < 2; ++up)  // shapes large enough for the 128 x 64 tiles (gemm_big_tiles)
        for (int ta = 0; ta < 2; ++ta) {
            const int M = up ? 2400 : 3000, N = up ? 2400 : 1200, K = 40;
            GemmArgs g{};
            g.M = M; g.N = N; g.K = K; g.TA = ta; g.TB = 0; g.upper_only = up;
            g.lda = ta ? M : K; g.ldb = N; g.ldc = N; g.alpha = 1;
            std::vector<double> A((size_t)(ta ? K : M) * g.lda), B((size_t)K * N), C((size_t)M * N, 0.0),
                R((size_t)M * N), S;
            for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
            for (auto &v : B) v = rand() / (double)RAND_MAX - 0.5;
            double *dA, *dB, *dC;
            cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
            cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
            cudaMemset(dC, 0, C.size() * 8);
            g.A = dA; g.B = dB; g.C = dC;
            const bool big = gemm_big_tiles(g);
            gemm_launch(g, 0);
            cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
            ref(g, A, B, S, R);
            double err = 0;
            for (int m = 0; m < M; ++m)
                for (int n = up ? m : 0; n < N; ++n) err = fmax(err, fabs(C[(size_t)m * N + n] - R[(size_t)m * N + n]));
            printf("big-tile case TA=%d upper=%d (big=%d) max err %.3e\n", ta, up, (int)big, err);
            fails += err > 1e-12 || !big;
            cudaFree(dA); cudaFree(dB); cudaFree(dC);
        }
    {   // odd leading dimensions (d = 2083-style buffers) use 8-byte copies
        int M = 37, N = 29, K = 41;
        GemmArgs g{};
        g.M = M; g.N = N; g.K = K; g.TA = 1; g.TB = 0; g.lda = M; g.ldb = N; g.ldc = N; g.alpha = 1;
        std::vector<double> A((size_t)K * M), B((size_t)K * N), C((size_t)M * N), R((size_t)M * N), S;
        for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
        for (auto &v : B) v = rand() / (double)RAND_MAX - 0.5;
        double *dA, *dB, *dC;
        cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
        cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
        g.A = dA; g.B = dB; g.C = dC;
        gemm_launch(g, 0);
        cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
        ref(g, A, B, S, R);
        double err = 0;
        for (size_t i = 0; i < C.size(); ++i) err = fmax(err, fabs(C[i] - R[i]));
        printf("odd ld max err %.3e\n", err);
        fails += err > 1e-12;
    }
    // stream-K path (full big-tile GEMM with a partial last wave: 11 x 32 = 352 tiles), all
    // transposes, per-k scale and beta = 1
    for (int ta = 0; ta < 2; ++ta)
        for (int tb = 0; tb < 2; ++tb) {
            int M = 1300, N = 2000, K = 200;
            GemmArgs g{};
            g.M = M; g.N = N; g.K = K; g.TA = ta; g.TB = tb;
            g.lda = ((ta ? M : K) + 3) & ~3; g.ldb = ((tb ? K : N) + 3) & ~3; g.ldc = (N + 3) & ~3;
            g.alpha = 0.7; g.beta = 1.0;
            std::vector<double> A((size_t)(ta ? K : M) * g.lda), B((size_t)(tb ? N : K) * g.ldb), S(K),
                C0((size_t)M * g.ldc), R((size_t)M * g.ldc), C((size_t)M * g.ldc);
            for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
            for (auto &v : B) v = rand() / (double)RAND_MAX - 0.5;
            for (auto &v : S) v = rand() / (double)RAND_MAX;
            for (auto &v : C0) v = rand() / (double)RAND_MAX - 0.5;
            double *dA, *dB, *dC, *dS;
            cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
            cudaMalloc(&dS, K * 8);
            cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dS, S.data(), K * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dC, C0.data(), C0.size() * 8, cudaMemcpyHostToDevice);
            g.A = dA; g.B = dB; g.C = dC; g.scale = dS;
            cudaError_t e = gemm_launch(g, 0);
            cudaDeviceSynchronize();
            cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
            GemmArgs gr = g; gr.alpha = 1.0; gr.beta = 0.0;
            ref(gr, A, B, S, R);
            double err = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    const size_t i = (size_t)m * g.ldc + n;
                    err = std::max(err, std::fabs(C[i] - (0.7 * R[i] + C0[i])));
                }
            printf("stream-K TA=%d TB=%d (launch %s) max err %.3e\n", ta, tb, cudaGetErrorString(e), err);
            fails += err > 1e-12 || e != cudaSuccess;
            cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dS);
        }
    // throughput
    struct Case { const char *name; int M, N, K, ta, tb, sc; } cases[] = {
        {"d^3 NN 2083", 2083, 2083, 2083, 0, 0, 0},
        {"d^3 NN 2083 odd-ld", 2083, 2083, 2083, 0, 0, -1},
        {"d^3 TN 2083", 2083, 2083, 2083, 1, 0, 0},
        {"d^3 NT 2083", 2083, 2083, 2083, 0, 1, 0},
        {"Hessian blk 1040x1040x8192 TN+scale", 1040, 1040, 8192, 1, 0, 1},
        {"trace Y 8192x2080x2080 NN", 8192, 2080, 2080, 0, 0, 0},
        {"square 4096", 4096, 4096, 4096, 0, 0, 0},
    };
    for (auto &c : cases) {
        GemmArgs g{};
        g.M = c.M; g.N = c.N; g.K = c.K; g.TA = c.ta; g.TB = c.tb;
        g.lda = ((c.ta ? c.M : c.K) + 3) & ~3; g.ldb = ((c.tb ? c.K : c.N) + 3) & ~3; g.ldc = (c.N + 3) & ~3;
        if (c.sc < 0) { g.lda = c.ta ? c.M : c.K; g.ldb = c.tb ? c.K : c.N; g.ldc = c.N; c.sc = 0; }
        g.alpha = 1; g.beta = 0;
        double *dA, *dB, *dC, *dS = nullptr;
        size_t na = (size_t)(c.ta ? c.K : c.M) * g.lda, nb = (size_t)(c.tb ? c.N : c.K) * g.ldb;
        cudaMalloc(&dA, na * 8); cudaMalloc(&dB, nb * 8); cudaMalloc(&dC, (size_t)c.M * g.ldc * 8);
        k_fill<<<592, 256>>>(dA, na, 1u); k_fill<<<592, 256>>>(dB, nb, 2u);
        if (c.sc) { cudaMalloc(&dS, c.K * 8); k_fill<<<16, 256>>>(dS, c.K, 3u); }
        g.A = dA; g.B = dB; g.C = dC; g.scale = dS;
        g.a16 = (g.lda % 2 == 0); g.b16 = (g.ldb % 2 == 0);
        gemm_launch(g, 0);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) gemm_launch(g, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        // cuBLAS: C^T (N x M, ld ldc) = op(B)^T op(A)^T in column-major terms
        const double one = 1.0, zero = 0.0;
        auto cub = [&]() {
            cublasDgemm(hb, c.tb ? CUBLAS_OP_T : CUBLAS_OP_N, c.ta ? CUBLAS_OP_T : CUBLAS_OP_N, c.N, c.M, c.K, &one, dB,
                        g.ldb, dA, g.lda, &zero, dC, g.ldc);
        };
        cub();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) cub();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float mc; cudaEventElapsedTime(&mc, e0, e1); mc /= 5;
        const double fl = 2.0 * c.M * c.N * (double)c.K;
        printf("%-40s ours %8.3f ms %6.2f TF/s | cuBLAS %8.3f ms %6.2f TF/s\n", c.name, ms, fl / (ms * 1e-3) / 1e12, mc,
               fl / (mc * 1e-3) / 1e12);
        cudaFree(dA); cudaFree(dB); cudaFree(dC); if (dS) cudaFree(dS);
    }
    printf(fails ? "FAIL\n" : "OK\n");
    return fails;
}
