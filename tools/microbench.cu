// Microbenchmarks for the design of the small-d chain kernel on B200:
// latency of dependent FP64 ops (DFMA, div, sqrt, rcp), of one Jacobi
// rotation-parameter chain, of L1 store->load round trips, and DMMA vs DFMA
// throughput.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <mma.h>

__device__ double sink;

__global__ void lat_dfma(double a, double b, int n, long long *cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
__global__ void lat_div(double a, double b, int n, long long *cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(b, x + 1.0);
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
__global__ void lat_rcp(double a, double b, int n, long long *cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __drcp_rn(x + b);
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
__global__ void lat_sqrt(double a, double b, int n, long long *cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dsqrt_rn(x + b);
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
__device__ __forceinline__ void rot(double app, double aqq, double apq, double &c, double &s, double &t) {
    const double theta = __ddiv_rn(__dsub_rn(aqq, app), __dmul_rn(2.0, apq));
    const double r = __drcp_rn(__dadd_rn(fabs(theta), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(theta, theta)))));
    t = theta >= 0.0 ? r : -r;
    c = __drcp_rn(__dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
    s = __dmul_rn(t, c);
}
__global__ void lat_rot(double a, double b, int n, long long *cyc) {
    double app = a, aqq = b, apq = 0.3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double c, s, t;
        rot(app, aqq, apq, c, s, t);
        app = __dsub_rn(app, __dmul_rn(t, apq));
        apq = __dsub_rn(__dmul_rn(c, 0.2), __dmul_rn(s, 0.1)) + 0.25;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = app + apq; *cyc = t1 - t0; }
}
// global store then load by the same thread (L1 write policy)
__global__ void lat_st_ld(double *buf, int n, long long *cyc) {
    double x = 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        buf[threadIdx.x] = x;
        x = buf[threadIdx.x] + 1.0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
__global__ void lat_smem(int n, long long *cyc) {
    __shared__ double buf[64];
    double x = 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        buf[threadIdx.x] = x;
        __syncwarp();
        x = buf[(threadIdx.x + 1) & 31] + 1.0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { sink = x; *cyc = t1 - t0; }
}
// throughput: many independent DFMA chains per thread, full occupancy
__global__ void thr_dfma(double a, int n, double *out) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, 0.999, 0.001); x1 = fma(x1, 0.999, 0.001); x2 = fma(x2, 0.999, 0.001);
        x3 = fma(x3, 0.999, 0.001); x4 = fma(x4, 0.999, 0.001); x5 = fma(x5, 0.999, 0.001);
        x6 = fma(x6, 0.999, 0.001); x7 = fma(x7, 0.999, 0.001);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// throughput: DMMA m8n8k4 (mma.sync f64)
__global__ void thr_dmma(int n, double *out) {
    double a = 1.0001, b = 0.9999;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    double d0 = 0, d1 = 0, e0 = 0, e1 = 0;
    for (int i = 0; i < n; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c2), "+d"(c3) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + d0 + d1 + e0 + e1;
}

int main() {
    long long *dc, hc;
    double *buf, *out;
    cudaMalloc(&dc, 8);
    cudaMalloc(&buf, 1 << 20);
    cudaMalloc(&out, 148 * 1024 * 8 * 8);
    const int n = 10000;
    auto rep = [&](const char *name, int per) {
        cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %8.1f cycles\n", name, (double)hc / n / per);
    };
    lat_dfma<<<1, 32>>>(1.0, 0.999, n, dc); cudaDeviceSynchronize(); lat_dfma<<<1, 32>>>(1.0, 0.999, n, dc); rep("DFMA dependent", 1);
    lat_div<<<1, 32>>>(1.0, 0.7, n, dc); cudaDeviceSynchronize(); lat_div<<<1, 32>>>(1.0, 0.7, n, dc); rep("ddiv_rn (+add)", 1);
    lat_rcp<<<1, 32>>>(1.0, 0.7, n, dc); cudaDeviceSynchronize(); lat_rcp<<<1, 32>>>(1.0, 0.7, n, dc); rep("drcp_rn (+add)", 1);
    lat_sqrt<<<1, 32>>>(1.0, 0.7, n, dc); cudaDeviceSynchronize(); lat_sqrt<<<1, 32>>>(1.0, 0.7, n, dc); rep("dsqrt_rn (+add)", 1);
    lat_rot<<<1, 32>>>(1.0, 2.0, n, dc); cudaDeviceSynchronize(); lat_rot<<<1, 32>>>(1.0, 2.0, n, dc); rep("jacobi rotation chain", 1);
    lat_st_ld<<<1, 32>>>(buf, n, dc); cudaDeviceSynchronize(); lat_st_ld<<<1, 32>>>(buf, n, dc); rep("global st->ld (same thr)", 1);
    lat_smem<<<1, 32>>>(n, dc); cudaDeviceSynchronize(); lat_smem<<<1, 32>>>(n, dc); rep("smem st->syncwarp->ld", 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int m = 20000;
    thr_dfma<<<148 * 8, 256>>>(1.0, 100, out);
    cudaEventRecord(e0);
    thr_dfma<<<148 * 8, 256>>>(1.0, m, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput   %8.2f TFLOP/s\n", 2.0 * 8 * m * 148.0 * 8 * 256 / (ms * 1e-3) / 1e12);
    thr_dmma<<<148 * 8, 256>>>(100, out);
    cudaEventRecord(e0);
    thr_dmma<<<148 * 8, 256>>>(m, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA throughput   %8.2f TFLOP/s\n", 2.0 * 256 * 4 * m * 148.0 * 8 * 8 / (ms * 1e-3) / 1e12);
    return 0;
}
