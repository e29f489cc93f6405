// sgp_dc.cuh — symmetric eigensolver for latent-function-sized d: blocked Householder
// tridiagonalisation + divide and conquer (north star (3)).
//
// Role: the fast cold decomposition of the large-d path (cold_order="dc": chain start, every
// rejection, rung starts -- metric.py:112-127 semantics: eigenvalues + orthonormal eigenvectors
// of the symmetrised Hessian) and the public sgp_eigh_dc entry.  It is not order-exact with the
// reference's cyclic Jacobi (eigenvalues come out ascending, eigenvector signs are its own); the
// SoftAbs metric G = Psi f(Lambda) Psi^T is invariant to both, so chains that use it are checked
// statistically, like warm_order="refine".
//
// Stage 1 -- tridiagonalisation T = Q^T A Q (LAPACK dsytrd/dlatrd semantics, lower):
//   32-column panels.  One cooperative persistent kernel per panel runs the panel's columns;
//   per column: (1) the column minus the panel's rank-2j correction, (2) the reflector (dlarfg),
//   (3) y = A22 v (the symmetric mat-vec against the panel-start trailing matrix) with the panel
//   dot products W^T v, V^T v, (4) w = tau (y - V W^T v - W V^T v), (5) w -= tau/2 (w^T v) v.
//   Three grid barriers per column; rows are owned by warps (row r -> warp r mod warps).  The
//   trailing matrix then takes A22 -= V W^T + W V^T as two DMMA GEMMs (sgp_gemm.cuh).
// Stage 2 -- tridiagonal divide and conquer (Cuppen; Gu-Eisenstat eigenvectors):
//   leaves of <= 48 rows (2^k leaves) solved by parallel-order Jacobi in shared memory; each
//   merge D + rho z z^T: deflation of small z and close poles (Givens, dlaed2 rules), the
//   secular roots (one warp per root, two-pole rational model inside a bisection bracket,
//   origin at the nearer pole as in dlaed4), z-hat recomputed from the roots (Loewner) so the
//   eigenvectors are orthogonal to working accuracy, then Q_new = Q V as one batched DMMA GEMM
//   per tree level.
// Stage 3 -- back-transformation Psi = Q Z by blocks of reflectors in compact-WY form
//   (I - V T V^T, T from dlarft's recurrence), three DMMA GEMMs per panel.
//
// Layout: every matrix row-major with leading dimension ld (even); Psi[i*ld + k] is component i
// of eigenvector k.  Single-stream, no host synchronisation inside.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>
#include "sgp_gemm.cuh"

#define DC_NB 32     // reflectors per panel
#define DC_PT 512    // threads of the panel kernel
#define DC_PS 72     // per-CTA partial stride (doubles): [0] |x|^2, [1..32] W^T v, [33..64] V^T v, [65] v^T y, [66] y(c+1)
#define DC_LEAF 48   // max leaf size
#define DC_MT 1024   // threads of the deflation kernel
#define DC_NMAX 4096 // largest d (one merge is sorted in shared memory)
#define DC_BT 128    // reflectors per back-transformation block

__device__ __forceinline__ unsigned dc_ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double dc_warp_sum(double v) {
    // xor butterfly: a + b == b + a, so every lane holds the bit-identical total
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double dc_warp_prod(double v) {
    for (int o = 16; o; o >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// grid barrier of the cooperative panel kernel (counter zeroed before the launch)
__device__ __forceinline__ void dc_grid_sync(unsigned *bar, unsigned &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (dc_ld_acquire(bar) < target) {
        }
    }
    __syncthreads();
}
// sum over the CTAs' partials part[b * DC_PS + t] by one warp, in the same order in every CTA
__device__ __forceinline__ double dc_warp_parts(const double *part, int t, int nb) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(part + (size_t)b * DC_PS + t);
    return dc_warp_sum(s);
}

#ifdef SGP_DC_PROF_CYC
#ifndef DC_PROF_BLK
#define DC_PROF_BLK 0
#endif
// cycles of CTA 0 per panel-kernel phase, summed over columns (tools/dc_prof.cu)
__device__ unsigned long long dc_prof[8];
#define DC_T0(v) long long v = clock64()
#define DC_ACC(i, v)                                                                \
    do {                                                                            \
        if (blockIdx.x == DC_PROF_BLK && threadIdx.x == 0) dc_prof[i] += clock64() - (v); \
        v = clock64();                                                              \
    } while (0)
#else
#define DC_T0(v)
#define DC_ACC(i, v)
#endif

// ---------------------------------------------------------------------------
// stage 1: one panel of the tridiagonalisation

struct DcPanel {
    double *A;  // n x ld, full symmetric; row c receives the updated column c
    int ld, n, k0, nbp;
    double *V;  // n x ld: V[r*ld + c] = v_c(r) (zero for r <= c, 1 at r = c+1)
    double *W;  // n x ld (first DC_NB columns): the panel's W
    double *y, *wt;            // [n] scratch
    double *dv, *ev, *tau;     // tridiagonal diagonal, off-diagonal, reflector scalars
    double *part;              // [grid][DC_PS]
    unsigned *bar;
};

// rows a warp owns (row r -> warp r mod warps): n <= DC_RPW * warps
#define DC_RPW 2
// most CTAs of the cooperative panel kernel (partials reduced with all loads in flight)
#define DC_MAXG 160

// symmetric mat-vec of one row segment against v (smem), 16 loads in flight per lane.  Plain
// (L1-allocating) loads: a warp re-reads its own rows every column, and a row is never written
// while it is inside the mat-vec range (row c+1 is rewritten only after its last mat-vec).
__device__ __forceinline__ double dc_ld_l1(const double *p) {
    double v;
    asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double dc_row_dot(const double *row, const double *v, int m) {
    const int lane = threadIdx.x & 31;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    double buf[8], nxt[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int i = lane + 32 * u;
        buf[u] = i < m ? dc_ld_l1(row + i) : 0.0;
    }
    for (int base = 0; base < m; base += 256) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + 256 + lane + 32 * u;
            nxt[u] = i < m ? dc_ld_l1(row + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + lane + 32 * u;
            const double vi = i < m ? v[i] : 0.0;
            if (u & 1) {
                if (u & 2) acc3 = __fma_rn(buf[u], vi, acc3);
                else acc1 = __fma_rn(buf[u], vi, acc1);
            } else {
                if (u & 2) acc2 = __fma_rn(buf[u], vi, acc2);
                else acc0 = __fma_rn(buf[u], vi, acc0);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) buf[u] = nxt[u];
    }
    return dc_warp_sum((acc0 + acc1) + (acc2 + acc3));
}

// Per column c (panel index j) with two grid barriers:
//   P  reflector of column c (its update is already in row c): ||x||^2 from the partials,
//      v staged in shared memory
//   S  y = A22 v on the owned rows, partials of W^T v, V^T v and v^T y          -> barrier A
//   W  s = w^T v = tau (v^T y - 2 (W^T v).(V^T v)) (no third reduction), w = tau (y - V W^T v
//      - W V^T v) - tau/2 s v stored as W(:, j), then column c+1 minus the rank-2(j+1)
//      correction into row c+1 with its ||x||^2 partial                          -> barrier B
__global__ void __launch_bounds__(DC_PT, 1) k_dc_panel(DcPanel a) {
    extern __shared__ double vs[];  // v of the current column, rows c+1..n-1
    constexpr int NW = DC_PT / 32;
    __shared__ double red[NW][2 * DC_NB + 2];
    __shared__ double u[2 * DC_NB + 2];  // u1 = W^T v [0, j), u2 = V^T v [j, 2j), v^T y [2j], y(c+1) [2j+1]
    __shared__ double rowv[DC_NB + 1], roww[DC_NB + 1];  // V(c+1, :), W(c+1, :)
    __shared__ double sc[4];
    const int n = a.n, ld = a.ld, k0 = a.k0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * NW + warp, NWG = gridDim.x * NW;
    unsigned target = 0;
    auto first_row = [&](int lo) { return lo + (gw - lo % NWG + NWG) % NWG; };
    auto put_sq = [&](double sq) {  // ||x||^2 partial of this CTA -> part[b][0]
        sq = dc_warp_sum(sq);
        if (lane == 0) red[warp][0] = sq;
        __syncthreads();
        if (warp == 0) {
            double v = lane < NW ? red[lane][0] : 0.0;
            v = dc_warp_sum(v);
            if (lane == 0) a.part[(size_t)blockIdx.x * DC_PS] = v;
        }
    };
    {  // prologue: column k0 needs no panel correction
        DC_T0(tp);
        double sq = 0.0;
        for (int r = first_row(k0); r < n; r += NWG) {
            if (lane == 0) {
                const double arc = __ldcg(a.A + (size_t)r * ld + k0);
                a.A[(size_t)k0 * ld + r] = arc;
                if (r == k0) a.dv[k0] = arc;
                if (r >= k0 + 2) sq = __fma_rn(arc, arc, sq);
            }
        }
        put_sq(sq);
        DC_ACC(0, tp);
        dc_grid_sync(a.bar, target);
        DC_ACC(1, tp);
    }
    for (int j = 0; j < a.nbp; ++j) {
        const int c = k0 + j, m = n - c - 1;
        DC_T0(tp);
        // ---- P: the reflector H = I - tau v v^T with H x = beta e1 (dlarfg), in every CTA
        double raw[(DC_NMAX + DC_PT - 1) / DC_PT];
#pragma unroll
        for (int q = 0; q < (DC_NMAX + DC_PT - 1) / DC_PT; ++q) {
            const int i = threadIdx.x + q * DC_PT;
            raw[q] = i < m ? __ldcg(a.A + (size_t)c * ld + c + 1 + i) : 0.0;
        }
        if (warp == 0) {
            const double xn2 = dc_warp_parts(a.part, 0, gridDim.x);
            if (lane == 0) {
                const double alpha = raw[0];
                double tau = 0.0, scal = 0.0, beta = alpha;
                if (xn2 > 0.0) {
                    beta = -copysign(sqrt(__fma_rn(alpha, alpha, xn2)), alpha);
                    tau = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
                sc[0] = tau;
                sc[1] = scal;
                if (blockIdx.x == 0 && m > 0) {
                    a.ev[c] = beta;
                    a.tau[c] = tau;
                }
            }
        }
        __syncthreads();
        const double tau = sc[0], scal = sc[1];
#pragma unroll
        for (int q = 0; q < (DC_NMAX + DC_PT - 1) / DC_PT; ++q) {
            const int i = threadIdx.x + q * DC_PT;
            if (i < m) vs[i] = i == 0 ? 1.0 : raw[q] * scal;
        }
        __syncthreads();
        DC_ACC(2, tp);
        // ---- S: y = A22 v on the owned rows; partial dot products; prefetch for W
        double yq[DC_RPW], vq[DC_RPW], vr[DC_RPW], wr[DC_RPW], an[DC_RPW];
        double acc1 = 0.0, acc2 = 0.0, yv = 0.0;
        {
            const int r0 = first_row(c + 1);
#pragma unroll
            for (int q = 0; q < DC_RPW; ++q) {
                const int r = r0 + q * NWG;
                if (r >= n) break;
                vr[q] = lane < j ? __ldcg(a.V + (size_t)r * ld + k0 + lane) : 0.0;
                wr[q] = lane < j ? __ldcg(a.W + (size_t)r * ld + lane) : 0.0;
                an[q] = (j + 1 < a.nbp && lane == 0) ? __ldcg(a.A + (size_t)r * ld + c + 1) : 0.0;
                const double yr = dc_row_dot(a.A + (size_t)r * ld + c + 1, vs, m);
                const double vv = vs[r - c - 1];
                yq[q] = yr;
                vq[q] = vv;
                if (lane == 0) {
                    a.y[r] = yr;
                    yv = __fma_rn(yr, vv, yv);
                }
                acc1 = __fma_rn(wr[q], vv, acc1);
                acc2 = __fma_rn(vr[q], vv, acc2);
            }
        }
        red[warp][lane] = acc1;
        red[warp][DC_NB + lane] = acc2;
        if (lane == 0) {
            red[warp][2 * DC_NB] = yv;
            red[warp][2 * DC_NB + 1] = (first_row(c + 1) == c + 1 && m > 0) ? yq[0] : 0.0;  // y(c+1) owner
        }
        __syncthreads();
        if (threadIdx.x < 2 * DC_NB + 2) {
            double v = 0.0;
            for (int w = 0; w < NW; ++w) v += red[w][threadIdx.x];
            a.part[(size_t)blockIdx.x * DC_PS + 1 + threadIdx.x] = v;
        }
        DC_ACC(3, tp);
        dc_grid_sync(a.bar, target);
        DC_ACC(1, tp);
        // ---- W: the reductions, 4 lanes per value (same order in every CTA)
        {
            // value g: u1 [0, j), u2 [j, 2j), v^T y (2j), y(c+1) (2j+1); 8 lanes per value
            const int g = threadIdx.x >> 3, sub = threadIdx.x & 7;
            const int idx = g < j ? 1 + g : (g < 2 * j ? 1 + DC_NB + (g - j) : 1 + 2 * DC_NB + (g - 2 * j));
            constexpr int MAXB = (DC_MAXG + 7) / 8;
            double pv[MAXB];
#pragma unroll
            for (int t = 0; t < MAXB; ++t) {
                const int b = sub + 8 * t;
                pv[t] = (g <= 2 * j + 1 && b < (int)gridDim.x) ? __ldcg(a.part + (size_t)b * DC_PS + idx) : 0.0;
            }
            double sm = 0.0;
#pragma unroll
            for (int t = 0; t < MAXB; ++t) sm += pv[t];
            sm += __shfl_xor_sync(0xffffffffu, sm, 1);
            sm += __shfl_xor_sync(0xffffffffu, sm, 2);
            sm += __shfl_xor_sync(0xffffffffu, sm, 4);
            if (sub == 0 && g <= 2 * j + 1) u[g] = sm;
            if (warp == 1 && lane < j) {
                rowv[lane] = __ldcg(a.V + (size_t)(c + 1) * ld + k0 + lane);
                roww[lane] = __ldcg(a.W + (size_t)(c + 1) * ld + lane);
            }
        }
        __syncthreads();
        if (warp == 0) {
            // alpha2 = -tau/2 w^T v with w^T v = tau (v^T y - 2 u1.u2)
            double t = lane < j ? u[lane] * u[j + lane] : 0.0;
            t = dc_warp_sum(t);
            const double s = tau * (u[2 * j] - 2.0 * t);
            const double alpha2 = -0.5 * tau * s;
            // W(c+1, j): row c+1 recomputed identically in every CTA
            double t2 = 0.0;
            if (m > 0 && lane < j) t2 = __fma_rn(rowv[lane], u[lane], __dmul_rn(roww[lane], u[j + lane]));
            t2 = dc_warp_sum(t2);
            if (lane == 0) {
                sc[2] = alpha2;
                const double w1 = m > 0 ? alpha2 + tau * (u[2 * j + 1] - t2) : 0.0;
                sc[3] = w1;
                if (blockIdx.x == 0 && m > 0) {
                    a.W[(size_t)(c + 1) * ld + j] = w1;
                    a.V[(size_t)(c + 1) * ld + c] = 1.0;
                }
            }
        }
        __syncthreads();
        const double alpha2 = sc[2], wrow = sc[3];
        const bool next = j + 1 < a.nbp;
        // V(c+1, i) and W(c+1, i) for i <= j, as the next column's update needs them
        const double v1 = lane < j ? rowv[lane] : (lane == j ? 1.0 : 0.0);
        const double w1 = lane < j ? roww[lane] : (lane == j ? wrow : 0.0);
        double sq = 0.0;
        {
            const int r0 = first_row(c + 1);
#pragma unroll
            for (int q = 0; q < DC_RPW; ++q) {
                const int r = r0 + q * NWG;
                if (r >= n) break;
                double t = 0.0;
                if (lane < j) t = __fma_rn(vr[q], u[lane], __dmul_rn(wr[q], u[j + lane]));
                t = dc_warp_sum(t);
                const double w = r == c + 1 ? wrow : __fma_rn(alpha2, vq[q], tau * (yq[q] - t));
                if (lane == 0 && r >= c + 2) {
                    a.W[(size_t)r * ld + j] = w;
                    a.V[(size_t)r * ld + c] = vq[q];
                }
                if (next) {  // column c+1 of row r minus sum_{i<=j} V(r,i) W(c+1,i) + W(r,i) V(c+1,i)
                    const double vri = lane == j ? vq[q] : vr[q], wri = lane == j ? w : wr[q];
                    double cr = lane <= j ? __fma_rn(vri, w1, __dmul_rn(wri, v1)) : 0.0;
                    cr = dc_warp_sum(cr);
                    if (lane == 0) {
                        const double arc = an[q] - cr;
                        a.A[(size_t)(c + 1) * ld + r] = arc;
                        if (r == c + 1) a.dv[c + 1] = arc;
                        if (r >= c + 3) sq = __fma_rn(arc, arc, sq);
                    }
                }
            }
        }
        if (next) {
            put_sq(sq);
            DC_ACC(4, tp);
            dc_grid_sync(a.bar, target);
            DC_ACC(1, tp);
        } else {
            DC_ACC(4, tp);
        }
    }
}

__global__ void k_dc_copy_in(const double *H, int ldh, double *A, int ld, int n) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)n * n;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (size_t)i * n);
        // symmetrised input (metric.py:117: 0.5 (H + H^T))
        A[(size_t)i * ld + j] = 0.5 * (H[(size_t)i * ldh + j] + H[(size_t)j * ldh + i]);
    }
}
__global__ void k_dc_last_diag(const double *A, int ld, int n, double *dv) {
    if (threadIdx.x == 0 && blockIdx.x == 0) dv[n - 1] = A[(size_t)(n - 1) * ld + n - 1];
}

// ---------------------------------------------------------------------------
// stage 2: divide and conquer on (dv, ev)

// leaf: the tridiagonal block [s, e) with the rank-one tears at its ends removed
// (d_{s} -= |e_{s-1}|, d_{e-1} -= |e_{e-1}|), by parallel-order (round-robin) Jacobi
__global__ void __launch_bounds__(256) k_dc_leaf(const double *dv, const double *ev, const int *bnd, int n, int ld,
                                                 double *D, double *Q) {
    __shared__ double A[DC_LEAF][DC_LEAF + 1], V[DC_LEAF][DC_LEAF + 1];
    __shared__ double rc[DC_LEAF / 2], rs[DC_LEAF / 2];
    __shared__ int rp[DC_LEAF / 2], rq[DC_LEAF / 2];
    __shared__ int rotated;
    __shared__ double fro;
    const int s = bnd[blockIdx.x], e = bnd[blockIdx.x + 1], m = e - s;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
        const int i = idx / m, k = idx - i * m;
        double v = 0.0;
        if (i == k) {
            v = dv[s + i];
            if (i == 0 && s > 0) v -= fabs(ev[s - 1]);
            if (i == m - 1 && e < n) v -= fabs(ev[e - 1]);
        } else if (k == i + 1 || i == k + 1) {
            v = ev[s + min(i, k)];
        }
        A[i][k] = v;
        V[i][k] = i == k ? 1.0 : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double f = 0.0;
        for (int i = 0; i < m; ++i)
            for (int k = 0; k < m; ++k) f += A[i][k] * A[i][k];
        fro = sqrt(f);
    }
    __syncthreads();
    const int mp = m + (m & 1), np = mp / 2;
    for (int sweep = 0; sweep < 60 && m > 1; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int r = 0; r < mp - 1; ++r) {
            if (threadIdx.x < np) {
                const int i = threadIdx.x;
                int p, q;
                if (i == 0) {
                    p = r;
                    q = mp - 1;
                } else {
                    p = (r + i) % (mp - 1);
                    q = (r - i + mp - 1) % (mp - 1);
                }
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, sn = 0.0;
                if (q < m) {
                    const double apq = A[p][q], app = A[p][p], aqq = A[q][q];
                    if (fabs(apq) > 2.2e-16 * sqrt(fabs(app)) * sqrt(fabs(aqq)) && fabs(apq) > 1e-18 * fro) {
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = copysign(1.0, th) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        sn = t * c;
                        rotated = 1;
                    }
                }
                rp[i] = p;
                rq[i] = q < m ? q : p;
                rc[i] = c;
                rs[i] = sn;
            }
            __syncthreads();
            for (int idx = threadIdx.x; idx < np * m; idx += blockDim.x) {  // A <- J^T A
                const int i = idx / m, k = idx - i * m, p = rp[i], q = rq[i];
                if (p == q) continue;
                const double c = rc[i], sn = rs[i], ap = A[p][k], aq = A[q][k];
                A[p][k] = c * ap - sn * aq;
                A[q][k] = sn * ap + c * aq;
            }
            __syncthreads();
            for (int idx = threadIdx.x; idx < np * m; idx += blockDim.x) {  // A <- A J, V <- V J
                const int i = idx / m, k = idx - i * m, p = rp[i], q = rq[i];
                if (p == q) continue;
                const double c = rc[i], sn = rs[i];
                const double ap = A[k][p], aq = A[k][q];
                A[k][p] = c * ap - sn * aq;
                A[k][q] = sn * ap + c * aq;
                const double vp = V[k][p], vq = V[k][q];
                V[k][p] = c * vp - sn * vq;
                V[k][q] = sn * vp + c * vq;
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    for (int k = threadIdx.x; k < m; k += blockDim.x) D[s + k] = A[k][k];
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
        const int i = idx / m, k = idx - i * m;
        Q[(size_t)(s + i) * ld + s + k] = V[i][k];
    }
}

// one merge: rows [s, s + n) torn at s + n1 (rho = ev[s + n1 - 1])
struct DcMerge {
    int s, n1, n;
};

// Deflation (dlaed2 rules) of D + rho z z^T, z = [last row of Q1; sign(rho) first row of Q2]/sqrt 2,
// rho' = 2|rho|.  Outputs at offset s: kept poles (ascending) pole/zk/col[0..K), deflated
// eigenvalues D[s+K+m] with their Q columns col[K+m]; the Givens rotations of close poles are
// applied to Q's columns here.
__global__ void __launch_bounds__(DC_MT) k_dc_deflate(const DcMerge *mg, const double *ev, int ld, double *D,
                                                      double *Q, double *pole, double *zk, int *col, int *kc,
                                                      double *rhov, double *rot) {
    extern __shared__ double sm[];
    const DcMerge g = mg[blockIdx.x];
    const int s = g.s, n1 = g.n1, n = g.n;
    int P = 1;
    while (P < n) P <<= 1;
    double *key = sm;                  // [P]
    double *z = key + P;               // [n]
    double *dl = z + n;                // [n] local eigenvalues (rotations change them)
    int *idx = reinterpret_cast<int *>(dl + n);  // [P]
    int *kept = idx + P;               // [n]
    int *defl = kept + n;              // [n]
    int *rpair = defl + n;             // [2n]
    __shared__ int nk, nd, nr;
    __shared__ double zmax_s;
    const double rho = ev[s + n1 - 1];
    const double sig = rho >= 0.0 ? 1.0 : -1.0, rh = 2.0 * fabs(rho);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < n) {
            const double zi = i < n1 ? Q[(size_t)(s + n1 - 1) * ld + s + i] : sig * Q[(size_t)(s + n1) * ld + s + i];
            z[i] = zi * 0.70710678118654752440;
            dl[i] = D[s + i];
            key[i] = dl[i];
        } else {
            key[i] = INFINITY;
        }
        idx[i] = i;
    }
    __syncthreads();
    // bitonic sort of (key, idx) ascending; ties by index
    for (int k = 2; k <= P; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int l = i ^ jj;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const double ki = key[i], kl = key[l];
                    const int ii = idx[i], il = idx[l];
                    const bool gt = ki > kl || (ki == kl && ii > il);
                    if (gt == up) {
                        key[i] = kl;
                        key[l] = ki;
                        idx[i] = il;
                        idx[l] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x < 32) {
        double zm = 0.0;
        for (int i = threadIdx.x; i < n; i += 32) zm = fmax(zm, fabs(z[i]));
        for (int o = 16; o; o >>= 1) zm = fmax(zm, __shfl_xor_sync(0xffffffffu, zm, o));
        if (threadIdx.x == 0) zmax_s = zm;
    }
    __syncthreads();
    const double eps = 1.1102230246251565e-16;
    const double tol = 8.0 * eps * fmax(fmax(fabs(key[0]), fabs(key[n - 1])), zmax_s);
    // Fast path (the common case): when no two neighbouring non-small poles are close, the
    // sequential scan below keeps exactly the non-small entries and deflates the small ones,
    // both in sorted order -- a block-wide compaction; the closeness test is the scan's own
    // expression, so both paths decide identically.  Any close pair -> the sequential scan.
    __shared__ int wsum[32], close_any;
    {
        const int per = (n + (int)blockDim.x - 1) / (int)blockDim.x;
        const int t0 = min(n, (int)threadIdx.x * per), t1 = min(n, t0 + per);
        int cnt = 0;
        for (int t = t0; t < t1; ++t) cnt += !(rh * fabs(z[idx[t]]) <= tol);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        if (threadIdx.x == 0) close_any = 0;
        __syncthreads();
        if (warp == 0) {
            int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        int big_before = (warp ? wsum[warp - 1] : 0) + incl - cnt;
        for (int t = t0; t < t1; ++t) {
            const int jx = idx[t];
            if (!(rh * fabs(z[jx]) <= tol))
                kept[big_before++] = jx;
            else
                defl[t - big_before] = jx;
        }
        __syncthreads();
        const int Kf = wsum[((blockDim.x >> 5) - 1)];
        for (int i = 1 + threadIdx.x; i < Kf; i += blockDim.x) {
            const int pj = kept[i - 1], jx = kept[i];
            double sn = z[pj], c = z[jx];
            const double tau = hypot(c, sn);
            const double tt = dl[jx] - dl[pj];
            c /= tau;
            sn = -sn / tau;
            if (fabs(tt * c * sn) <= tol) close_any = 1;
        }
        __syncthreads();
        if (!close_any && threadIdx.x == 0) {
            nk = Kf;
            nd = n - Kf;
            nr = 0;
            kc[blockIdx.x] = Kf;
            rhov[blockIdx.x] = rh;
        }
    }
    if (close_any && threadIdx.x == 0) {
        int K = 0, M = 0, R = 0, pj = -1;
        for (int t = 0; t < n; ++t) {
            const int jx = idx[t];
            if (rh * fabs(z[jx]) <= tol) {
                defl[M++] = jx;
                continue;
            }
            if (pj < 0) {
                pj = jx;
                continue;
            }
            double sn = z[pj], c = z[jx];
            const double tau = hypot(c, sn);
            const double tt = dl[jx] - dl[pj];
            c /= tau;
            sn = -sn / tau;
            if (fabs(tt * c * sn) <= tol) {
                z[jx] = tau;
                z[pj] = 0.0;
                rpair[2 * R] = pj;
                rpair[2 * R + 1] = jx;
                rot[2 * (s + R)] = c;
                rot[2 * (s + R) + 1] = sn;
                ++R;
                const double t2 = dl[pj] * c * c + dl[jx] * sn * sn;
                dl[jx] = dl[pj] * sn * sn + dl[jx] * c * c;
                dl[pj] = t2;
                defl[M++] = pj;
            } else {
                kept[K++] = pj;
            }
            pj = jx;
        }
        if (pj >= 0) kept[K++] = pj;
        nk = K;
        nd = M;
        nr = R;
        kc[blockIdx.x] = K;
        rhov[blockIdx.x] = rh;
    }
    __syncthreads();
    const int K = nk, M = nd, R = nr;
    // Givens rotations of close poles on Q's columns (each thread owns rows: no barriers)
    if (R > 0) {
        __threadfence_block();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double *row = Q + (size_t)(s + i) * ld + s;
            for (int r = 0; r < R; ++r) {
                const int p = rpair[2 * r], q = rpair[2 * r + 1];
                const double c = rot[2 * (s + r)], sn = rot[2 * (s + r) + 1];
                const double x = row[p], y = row[q];
                row[p] = c * x + sn * y;
                row[q] = c * y - sn * x;
            }
        }
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const int jx = kept[k];
        pole[s + k] = dl[jx];
        zk[s + k] = z[jx];
        col[s + k] = jx;
    }
    for (int mm = threadIdx.x; mm < M; mm += blockDim.x) {
        const int jx = defl[mm];
        D[s + K + mm] = dl[jx];
        col[s + K + mm] = jx;
    }
}

// Secular roots: one warp per root k of 1/rho + sum_j z_j^2 / (p_j - lambda) = 0 (poles p
// ascending).  lambda_k = p_org + tau with org the nearer pole; DELTA[(s+k)*ld + s+j] =
// (p_j - p_org) - tau (= p_j - lambda_k, accurately).
__global__ void __launch_bounds__(256) k_dc_secular(const DcMerge *mg, const int *kc, const double *rhov,
                                                    const double *pole, const double *zk, int ld, double *D,
                                                    double *DELTA) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const DcMerge g = mg[blockIdx.y];
    const int K = kc[blockIdx.y], s = g.s;
    if (k >= K) return;
    const double *p = pole + s, *z = zk + s;
    const double rinv = 1.0 / rhov[blockIdx.y];
    const double eps = 1.1102230246251565e-16;
    int org;
    double lo, hi;
    if (k < K - 1) {
        const double gap = p[k + 1] - p[k], mid = 0.5 * gap;
        // f at the midpoint decides which pole is nearer the root
        double f = 0.0;
        for (int jj = lane; jj < K; jj += 32) {
            const double zj = z[jj];
            f += zj * zj / ((p[jj] - p[k]) - mid);
        }
        f = rinv + dc_warp_sum(f);
        if (f >= 0.0) {  // root in (p_k, p_k + gap/2]
            org = k;
            lo = 0.0;
            hi = mid;
        } else {  // root in (p_{k+1} - gap/2, p_{k+1})
            org = k + 1;
            lo = -mid;
            hi = 0.0;
        }
    } else {
        double zz = 0.0;
        for (int jj = lane; jj < K; jj += 32) zz += z[jj] * z[jj];
        zz = dc_warp_sum(zz);
        org = k;
        lo = 0.0;
        hi = zz / rinv;  // lambda_max <= p_max + rho |z|^2
    }
    const double po = p[org];
    double tau = 0.5 * (lo + hi);
    for (int it = 0; it < 100; ++it) {
        // psi: poles at or below the root's interval, phi: above; values and tau-derivatives
        double ps = 0.0, dps = 0.0, ph = 0.0, dph = 0.0, fa = 0.0;
        for (int jj = lane; jj < K; jj += 32) {
            const double zj = z[jj], dl = (p[jj] - po) - tau;
            const double t = zj * zj / dl, t2 = t / dl;
            if (jj <= k) {
                ps += t;
                dps += t2;
            } else {
                ph += t;
                dph += t2;
            }
            fa += fabs(t);
        }
        ps = dc_warp_sum(ps);
        dps = dc_warp_sum(dps);
        ph = dc_warp_sum(ph);
        dph = dc_warp_sum(dph);
        fa = rinv + dc_warp_sum(fa);
        const double f = rinv + ps + ph;
        if (f == 0.0 || fabs(f) <= 4.0 * eps * fa) break;
        if (f < 0.0)
            lo = tau;
        else
            hi = tau;
        // rational model matching psi, phi and their derivatives (the middle way of dlaed4):
        // psi(tau + e) ~ (psi - x psi') + x^2 psi' / (x - e), phi likewise at the upper pole y
        const double x = (p[k] - po) - tau, S1 = x * x * dps;
        double nt;
        if (k + 1 < K) {
            const double y = (p[k + 1] - po) - tau, S2 = y * y * dph;
            const double cc = rinv + (ps - x * dps) + (ph - y * dph);
            // cc (x-e)(y-e) + S1 (y-e) + S2 (x-e) = 0, root e in (x, y)
            const double A2 = cc, A1 = -(cc * (x + y) + S1 + S2), A0 = x * y * f;
            double e = NAN;
            if (fabs(A2) <= 1e-300 * (fabs(A1) + fabs(A0))) {
                e = -A0 / A1;
            } else {
                const double disc = A1 * A1 - 4.0 * A2 * A0;
                if (disc >= 0.0) {
                    const double q = -0.5 * (A1 + copysign(sqrt(disc), A1));
                    const double e1 = q / A2, e2 = A0 / q;
                    e = (e1 > x && e1 < y) ? e1 : e2;
                }
            }
            nt = tau + e;
        } else {
            const double cc = rinv + (ps - x * dps);
            nt = tau + x + S1 / cc;
        }
        if (!(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
        if (nt == tau || hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi))) {
            tau = nt;
            break;
        }
        tau = nt;
    }
    if (lane == 0) D[s + k] = po + tau;
    double *drow = DELTA + (size_t)(s + k) * ld + s;
    for (int jj = lane; jj < K; jj += 32) drow[jj] = (p[jj] - po) - tau;
}

// z-hat_j^2 rho = prod_k (lambda_k - p_j) / prod_{k != j} (p_k - p_j)  (Gu-Eisenstat), warp per j
__global__ void __launch_bounds__(256) k_dc_zhat(const DcMerge *mg, const int *kc, const double *rhov,
                                                 const double *pole, const double *zk, int ld, const double *DELTA,
                                                 double *zhat) {
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const DcMerge g = mg[blockIdx.y];
    const int K = kc[blockIdx.y], s = g.s;
    if (j >= K) return;
    const double *p = pole + s;
    double pr = 1.0;
    for (int k = lane; k < K; k += 32) {
        const double dlt = -DELTA[(size_t)(s + k) * ld + s + j];  // lambda_k - p_j
        pr *= k == j ? dlt : dlt / (p[k] - p[j]);
    }
    pr = dc_warp_prod(pr);
    if (lane == 0) zhat[s + j] = copysign(sqrt(fmax(pr, 0.0) / rhov[blockIdx.y]), zk[s + j]);
}

// eigenvectors of the merge in the children's basis, transposed: VT[(s+k)*ld + s + col_j] = v_k(j)
// (kept roots: zhat_j / (p_j - lambda_k), normalised; deflated: unit vectors)
__global__ void __launch_bounds__(256) k_dc_vec(const DcMerge *mg, const int *kc, const int *col, const double *zhat,
                                                int ld, const double *DELTA, double *VT) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const DcMerge g = mg[blockIdx.y];
    const int K = kc[blockIdx.y], s = g.s;
    if (k >= g.n) return;
    double *vrow = VT + (size_t)(s + k) * ld + s;
    if (k >= K) {
        if (lane == 0) vrow[col[s + k]] = 1.0;
        return;
    }
    const double *drow = DELTA + (size_t)(s + k) * ld + s;
    double nn = 0.0;
    for (int jj = lane; jj < K; jj += 32) {
        const double v = zhat[s + jj] / drow[jj];
        nn += v * v;
    }
    const double inv = 1.0 / sqrt(dc_warp_sum(nn));
    for (int jj = lane; jj < K; jj += 32) vrow[col[s + jj]] = zhat[s + jj] / drow[jj] * inv;
}

// ---------------------------------------------------------------------------
// stage 3: back-transformation

// compact-WY T of a back-transformation block from its Gram G = V^T V (dlarft recurrence):
// T(j,j) = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j)
__global__ void __launch_bounds__(DC_BT) k_dc_tblock(const double *Gm, const double *tau, int n, double *Tb) {
    extern __shared__ double T[];  // DC_BT x (DC_BT + 1)
    constexpr int LT = DC_BT + 1;
    const int b = blockIdx.x, k0 = b * DC_BT, nbb = min(DC_BT, n - 1 - k0);
    const double *G = Gm + (size_t)b * DC_BT * DC_BT;
    const int i = threadIdx.x;
    for (int l = 0; l < DC_BT; ++l) T[i * LT + l] = 0.0;
    __syncthreads();
    for (int j = 0; j < nbb; ++j) {
        const double tj = tau[k0 + j];
        double v = 0.0;
        if (i < j)
            for (int l = i; l < j; ++l) v = __fma_rn(T[i * LT + l], G[(size_t)l * DC_BT + j], v);
        __syncthreads();
        if (i < j) T[i * LT + j] = -tj * v;
        if (i == j) T[j * LT + j] = tj;
        __syncthreads();
    }
    for (int l = 0; l < DC_BT; ++l) Tb[(size_t)b * DC_BT * DC_BT + (size_t)i * DC_BT + l] = T[i * LT + l];
}

// ascending eigenvalues (bitonic, one CTA) and the permutation
__global__ void __launch_bounds__(1024) k_dc_sort(const double *D, int n, double *lam, int *perm) {
    extern __shared__ double sm[];
    int P = 1;
    while (P < n) P <<= 1;
    double *key = sm;
    int *idx = reinterpret_cast<int *>(key + P);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        key[i] = i < n ? D[i] : INFINITY;
        idx[i] = i;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int l = i ^ jj;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const double ki = key[i], kl = key[l];
                    const int ii = idx[i], il = idx[l];
                    const bool gt = ki > kl || (ki == kl && ii > il);
                    if (gt == up) {
                        key[i] = kl;
                        key[l] = ki;
                        idx[i] = il;
                        idx[l] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        lam[i] = key[i];
        perm[i] = idx[i];
    }
}
__global__ void k_dc_gather(const double *Z, int ld, const int *perm, int n, double *psi, int ldp) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)n * n;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), k = (int)(idx - (size_t)i * n);
        psi[(size_t)i * ldp + k] = Z[(size_t)i * ld + perm[k]];
    }
}

// ---------------------------------------------------------------------------
// host side

struct DcWS {
    int n = 0, ld = 0, nctas = 0, L = 0, levels = 0;
    double *base = nullptr;
    double *A, *V, *W, *y, *wt, *dv, *ev, *tau, *part, *Q[2], *VT, *D, *pole, *zk, *zh, *rhov, *rot, *X, *Y;
    double *G, *Tb;     // back-transform blocks: Gram V_b^T V_b and the compact-WY T_b
    GemmArgs *gdesc;    // the blocks' Gram GEMMs (one batched launch)
    int nbt;
    int *col, *kc, *bnd, *perm;
    unsigned *bar;
    DcMerge *mg;
    GemmArgs *desc;
    std::vector<int> loff, lcnt, lmax;  // per level: first merge, merges, largest merge
};

static inline void dc_ws_free(DcWS &w) {
    if (w.base) cudaFree(w.base);
    w.base = nullptr;
    w.n = 0;
}

static inline int dc_ws_alloc(DcWS &w, int n) {
    if (w.base && w.n == n) return 0;
    dc_ws_free(w);
    if (n < 1 || n > DC_NMAX) return -1;
    const int ld = (n + 3) & ~3;
    const size_t nl = (size_t)n * ld;
    int L = 1;
    while ((n + L - 1) / L > DC_LEAF) L <<= 1;
    int levels = 0;
    while ((1 << levels) < L) ++levels;
    std::vector<int> bnd(L + 1);
    for (int i = 0; i <= L; ++i) bnd[i] = (int)((long)i * n / L);
    std::vector<DcMerge> mg;
    w.loff.assign(levels + 1, 0);
    w.lcnt.assign(levels + 1, 0);
    w.lmax.assign(levels + 1, 0);
    for (int l = 1; l <= levels; ++l) {
        w.loff[l] = (int)mg.size();
        const int cnt = L >> l;
        for (int i = 0; i < cnt; ++i) {
            DcMerge g;
            g.s = bnd[i << l];
            g.n1 = bnd[(i << l) + (1 << (l - 1))] - g.s;
            g.n = bnd[(i + 1) << l] - g.s;
            mg.push_back(g);
            w.lmax[l] = std::max(w.lmax[l], g.n);
        }
        w.lcnt[l] = cnt;
    }
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t psmem = sizeof(double) * (size_t)n;
    cudaFuncSetAttribute(k_dc_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem + 1024);
    // the owned rows' mat-vec reads are re-used from L1 column after column: smallest carveout
    cudaFuncSetAttribute(k_dc_panel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dc_panel, DC_PT, psmem) != cudaSuccess || occ < 1)
        return -1;
    const int G = std::min(sms, DC_MAXG);  // one CTA per SM (co-resident: cooperative launch)
    if (n > DC_RPW * G * (DC_PT / 32)) return -1;  // rows per warp held in registers
    const int nbt = std::max(1, (n - 1 + DC_BT - 1) / DC_BT);  // back-transform blocks
    size_t off = 0;
    auto take = [&](size_t cnt) {
        size_t o = off;
        off += (cnt + 3) & ~size_t(3);
        return o;
    };
    const size_t oA = take(nl), oV = take(nl), oW = take(nl), oy = take(n), owt = take(n),
                 odv = take(n), oev = take(n), otau = take(n), opart = take((size_t)G * DC_PS), oQ0 = take(nl),
                 oQ1 = take(nl), oVT = take(nl), oD = take(n), opole = take(n), ozk = take(n), ozh = take(n),
                 orho = take(mg.size() + 1), orot = take(2 * (size_t)n),
                 oX = take((size_t)2 * DC_BT * ld), oY = take((size_t)DC_BT * ld),
                 oG = take((size_t)nbt * DC_BT * DC_BT), oTb = take((size_t)nbt * DC_BT * DC_BT),
                 ogd = take(nbt * ((sizeof(GemmArgs) + 7) / 8) + 2), ocol = take(n), okc = take(mg.size() + 1),
                 obnd = take(L + 1), operm = take(n), obar = take(1), omg = take(3 * mg.size() + 2),
                 odesc = take(mg.size() * ((sizeof(GemmArgs) + 7) / 8) + 2);
    double *base = nullptr;
    if (cudaMalloc(&base, off * sizeof(double)) != cudaSuccess) return -1;
    w.base = base;
    w.n = n;
    w.ld = ld;
    w.nctas = G;
    w.L = L;
    w.levels = levels;
    w.A = base + oA;
    w.V = base + oV;
    w.W = base + oW;
    w.y = base + oy;
    w.wt = base + owt;
    w.dv = base + odv;
    w.ev = base + oev;
    w.tau = base + otau;
    w.part = base + opart;
    w.Q[0] = base + oQ0;
    w.Q[1] = base + oQ1;
    w.VT = base + oVT;
    w.D = base + oD;
    w.pole = base + opole;
    w.zk = base + ozk;
    w.zh = base + ozh;
    w.rhov = base + orho;
    w.rot = base + orot;
    w.X = base + oX;
    w.Y = base + oY;
    w.G = base + oG;
    w.Tb = base + oTb;
    w.gdesc = reinterpret_cast<GemmArgs *>(base + ((ogd + 1) & ~size_t(1)));
    w.nbt = nbt;
    w.col = reinterpret_cast<int *>(base + ocol);
    w.kc = reinterpret_cast<int *>(base + okc);
    w.bnd = reinterpret_cast<int *>(base + obnd);
    w.perm = reinterpret_cast<int *>(base + operm);
    w.bar = reinterpret_cast<unsigned *>(base + obar);
    w.mg = reinterpret_cast<DcMerge *>(base + omg);
    w.desc = reinterpret_cast<GemmArgs *>(base + ((odesc + 1) & ~size_t(1)));
    // merge GEMM descriptors: Q_out[s.., s..] = Q_in[s.., s..] VT[s.., s..]^T (ping-pong by level parity)
    std::vector<GemmArgs> desc(mg.size());
    for (int l = 1; l <= levels; ++l) {
        const int in = (l - 1) & 1, out = l & 1;
        for (int i = 0; i < w.lcnt[l]; ++i) {
            const DcMerge &g = mg[w.loff[l] + i];
            GemmArgs a{};
            a.M = a.N = a.K = g.n;
            a.A = w.Q[in] + (size_t)g.s * ld + g.s;
            a.lda = ld;
            a.TA = 0;
            a.B = w.VT + (size_t)g.s * ld + g.s;
            a.ldb = ld;
            a.TB = 1;
            a.C = w.Q[out] + (size_t)g.s * ld + g.s;
            a.ldc = ld;
            a.alpha = 1.0;
            a.beta = 0.0;
            a.a16 = (reinterpret_cast<uintptr_t>(a.A) & 15) == 0;
            a.b16 = (reinterpret_cast<uintptr_t>(a.B) & 15) == 0;
            desc[w.loff[l] + i] = a;
        }
    }
    std::vector<GemmArgs> gd(nbt);
    for (int b = 0; b < nbt; ++b) {  // G_b = V_b^T V_b over rows k0+1..n-1
        const int k0 = b * DC_BT, nbb = std::max(0, std::min(DC_BT, n - 1 - k0)), r0 = k0 + 1;
        GemmArgs a{};
        a.M = a.N = nbb;
        a.K = std::max(0, n - r0);
        a.A = w.V + (size_t)r0 * ld + k0;
        a.lda = ld;
        a.TA = 1;
        a.B = a.A;
        a.ldb = ld;
        a.TB = 0;
        a.C = w.G + (size_t)b * DC_BT * DC_BT;
        a.ldc = DC_BT;
        a.alpha = 1.0;
        a.beta = 0.0;
        a.a16 = a.b16 = (reinterpret_cast<uintptr_t>(a.A) & 15) == 0;
        gd[b] = a;
    }
    bool ok = cudaMemset(base, 0, off * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMemcpy(w.gdesc, gd.data(), sizeof(GemmArgs) * nbt, cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && cudaMemcpy(w.bnd, bnd.data(), sizeof(int) * (L + 1), cudaMemcpyHostToDevice) == cudaSuccess;
    if (!mg.empty()) {
        ok = ok && cudaMemcpy(w.mg, mg.data(), sizeof(DcMerge) * mg.size(), cudaMemcpyHostToDevice) == cudaSuccess;
        ok = ok && cudaMemcpy(w.desc, desc.data(), sizeof(GemmArgs) * desc.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    const size_t dsm = (size_t)DC_NMAX * 12 + (size_t)DC_NMAX * 16 + (size_t)DC_NMAX * 16 + 64;
    ok = ok && cudaFuncSetAttribute(k_dc_deflate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm) == cudaSuccess;
    ok = ok && cudaFuncSetAttribute(k_dc_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, DC_NMAX * 12) == cudaSuccess;
    ok = ok && cudaFuncSetAttribute(k_dc_tblock, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(double) * DC_BT * (DC_BT + 1))) == cudaSuccess;
    if (!ok) {
        dc_ws_free(w);
        return -1;
    }
    return 0;
}

static inline cudaError_t dc_gemm(int M, int N, int K, const double *A, int lda, int TA, const double *B, int ldb,
                                  int TB, double *C, int ldc, double alpha, double beta, cudaStream_t s) {
    GemmArgs g{};
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.TA = TA;
    g.B = B;
    g.ldb = ldb;
    g.TB = TB;
    g.C = C;
    g.ldc = ldc;
    g.alpha = alpha;
    g.beta = beta;
    return gemm_launch(g, s);
}

// diagnostics: SGP_DC_DUMP=<prefix> writes the stage outputs of each call (host copies)
static inline void dc_dump(const char *tag, const double *dptr, size_t cnt, cudaStream_t s) {
    const char *pre = getenv("SGP_DC_DUMP");
    if (!pre) return;
    std::vector<double> h(cnt);
    cudaMemcpyAsync(h.data(), dptr, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    char path[512];
    snprintf(path, sizeof(path), "%s_%s.bin", pre, tag);
    FILE *f = fopen(path, "wb");
    if (f) {
        fwrite(h.data(), sizeof(double), cnt, f);
        fclose(f);
    }
}

// Eigen-decomposition of the symmetric part of H (n x n, leading dimension ldh): lam ascending,
// psi[i*ldp + k] = component i of eigenvector k.  Returns 0 or -1 (CUDA error / unsupported n).
static inline int dc_eigh(DcWS &w, const double *H, int ldh, int n, double *lam, double *psi, int ldp,
                          cudaStream_t s) {
    if (dc_ws_alloc(w, n)) return -1;
    const int ld = w.ld;
    // SGP_DC_PROF=1: per-stage device times on stderr (events on the stream)
    const bool prof = getenv("SGP_DC_PROF") != nullptr;
    cudaEvent_t ev[4] = {};
    if (prof)
        for (auto &e : ev) cudaEventCreate(&e);
    if (prof) cudaEventRecord(ev[0], s);
    const size_t nl = (size_t)n * ld;
    k_dc_copy_in<<<148 * 4, 256, 0, s>>>(H, ldh, w.A, ld, n);
    if (n == 1) {
        cudaMemcpyAsync(lam, w.A, sizeof(double), cudaMemcpyDeviceToDevice, s);
        const double one = 1.0;
        cudaMemcpyAsync(psi, &one, sizeof(double), cudaMemcpyHostToDevice, s);
        return cudaStreamSynchronize(s) == cudaSuccess ? 0 : -1;
    }
    cudaMemsetAsync(w.V, 0, sizeof(double) * nl, s);
    // ---- stage 1
    for (int k0 = 0; k0 < n - 1; k0 += DC_NB) {
        const int nbp = std::min(DC_NB, n - 1 - k0);
        DcPanel a;
        a.A = w.A;
        a.ld = ld;
        a.n = n;
        a.k0 = k0;
        a.nbp = nbp;
        a.V = w.V;
        a.W = w.W;
        a.y = w.y;
        a.wt = w.wt;
        a.dv = w.dv;
        a.ev = w.ev;
        a.tau = w.tau;
        a.part = w.part;
        a.bar = w.bar;
        cudaMemsetAsync(w.bar, 0, sizeof(unsigned), s);
        void *args[] = {&a};
        if (cudaLaunchCooperativeKernel((void *)k_dc_panel, w.nctas, DC_PT, args, sizeof(double) * n, s) != cudaSuccess)
            return -1;
        const int r0 = k0 + nbp, m = n - r0;
        if (m > 0) {  // A22 -= V W^T + W V^T: one K = 2 nbp GEMM, [V W] [W V]^T by the K-split gather
            double *A22 = w.A + (size_t)r0 * ld + r0;
            const double *Vp = w.V + (size_t)r0 * ld + k0, *Wp = w.W + (size_t)r0 * ld;
            if (nbp % GM_BK == 0) {
                GemmArgs g{};
                g.M = g.N = m;
                g.K = 2 * nbp;
                g.A = Vp;
                g.A2 = Wp;
                g.lda = ld;
                g.B = Wp;
                g.B2 = Vp;
                g.ldb = ld;
                g.TB = 1;
                g.ksplit = nbp;
                g.C = A22;
                g.ldc = ld;
                g.alpha = -1.0;
                g.beta = 1.0;
                gemm_launch(g, s);
            } else {
                dc_gemm(m, m, nbp, Vp, ld, 0, Wp, ld, 1, A22, ld, -1.0, 1.0, s);
                dc_gemm(m, m, nbp, Wp, ld, 0, Vp, ld, 1, A22, ld, -1.0, 1.0, s);
            }
        }
    }
    k_dc_last_diag<<<1, 32, 0, s>>>(w.A, ld, n, w.dv);
    if (prof) cudaEventRecord(ev[1], s);
    dc_dump("dv", w.dv, n, s);
    dc_dump("ev", w.ev, n, s);
    dc_dump("tau", w.tau, n, s);
    dc_dump("V", w.V, nl, s);
    // ---- stage 2
    cudaMemsetAsync(w.Q[0], 0, sizeof(double) * nl, s);
    cudaMemsetAsync(w.Q[1], 0, sizeof(double) * nl, s);
    k_dc_leaf<<<w.L, 256, 0, s>>>(w.dv, w.ev, w.bnd, n, ld, w.D, w.Q[0]);
    const size_t dsm_base = 64;
    for (int l = 1; l <= w.levels; ++l) {
        const int in = (l - 1) & 1, cnt = w.lcnt[l], mx = w.lmax[l];
        int P = 1;
        while (P < mx) P <<= 1;
        const size_t dsm = (size_t)P * 12 + (size_t)mx * 16 + (size_t)mx * 16 + dsm_base;
        const DcMerge *mg = w.mg + w.loff[l];
        double *rh = w.rhov + w.loff[l];
        int *kc = w.kc + w.loff[l];
        k_dc_deflate<<<cnt, DC_MT, dsm, s>>>(mg, w.ev, ld, w.D, w.Q[in], w.pole, w.zk, w.col, kc, rh, w.rot);
        const dim3 g2((mx + 7) / 8, cnt);
        k_dc_secular<<<g2, 256, 0, s>>>(mg, kc, rh, w.pole, w.zk, ld, w.D, w.A);  // DELTA in A (free now)
        k_dc_zhat<<<g2, 256, 0, s>>>(mg, kc, rh, w.pole, w.zk, ld, w.A, w.zh);
        cudaMemsetAsync(w.VT, 0, sizeof(double) * nl, s);
        k_dc_vec<<<g2, 256, 0, s>>>(mg, kc, w.col, w.zh, ld, w.A, w.VT);
        if (gemm_launch_batched<0, 1>(w.desc + w.loff[l], cnt, mx, mx, s) != cudaSuccess) return -1;
    }
    double *Z = w.Q[w.levels & 1];
    if (prof) cudaEventRecord(ev[2], s);
    dc_dump("D", w.D, n, s);
    dc_dump("Z", Z, nl, s);
    // ---- stage 3: Z <- Q_H Z, blocks of DC_BT reflectors last to first
    if (gemm_launch_batched<1, 0>(w.gdesc, w.nbt, DC_BT, DC_BT, s) != cudaSuccess) return -1;
    k_dc_tblock<<<w.nbt, DC_BT, sizeof(double) * DC_BT * (DC_BT + 1), s>>>(w.G, w.tau, n, w.Tb);
    for (int b = w.nbt - 1; b >= 0; --b) {
        const int k0 = b * DC_BT, nbb = std::min(DC_BT, n - 1 - k0), r0 = k0 + 1, m = n - r0;
        if (nbb <= 0) continue;
        const double *Vb = w.V + (size_t)r0 * ld + k0, *Tb = w.Tb + (size_t)b * DC_BT * DC_BT;
        double *X0 = w.X, *X1 = w.X + (size_t)DC_BT * ld;
        const int mh = (m / 2) & ~31;
        if (nbb % GM_BK == 0 && mh >= 64) {
            // split-K: X0 = V_b^T Z over the first mh rows, X1 over the rest; Y = [T T][X0; X1]
            dc_gemm(nbb, n, mh, Vb, ld, 1, Z + (size_t)r0 * ld, ld, 0, X0, ld, 1.0, 0.0, s);
            dc_gemm(nbb, n, m - mh, Vb + (size_t)mh * ld, ld, 1, Z + (size_t)(r0 + mh) * ld, ld, 0, X1, ld, 1.0, 0.0,
                    s);
            GemmArgs g{};
            g.M = nbb;
            g.N = n;
            g.K = 2 * nbb;
            g.A = Tb;
            g.A2 = Tb;
            g.lda = DC_BT;
            g.B = X0;
            g.B2 = X1;
            g.ldb = ld;
            g.ksplit = nbb;
            g.C = w.Y;
            g.ldc = ld;
            g.alpha = 1.0;
            g.beta = 0.0;
            gemm_launch(g, s);
        } else {
            dc_gemm(nbb, n, m, Vb, ld, 1, Z + (size_t)r0 * ld, ld, 0, X0, ld, 1.0, 0.0, s);   // X = V^T Z
            dc_gemm(nbb, n, nbb, Tb, DC_BT, 0, X0, ld, 0, w.Y, ld, 1.0, 0.0, s);             // Y = T X
        }
        dc_gemm(m, n, nbb, Vb, ld, 0, w.Y, ld, 0, Z + (size_t)r0 * ld, ld, -1.0, 1.0, s);   // Z -= V Y
    }
    k_dc_sort<<<1, 1024, (size_t)12 * DC_NMAX, s>>>(w.D, n, lam, w.perm);
    k_dc_gather<<<148 * 4, 256, 0, s>>>(Z, ld, w.perm, n, psi, ldp);
    if (prof) {
        cudaEventRecord(ev[3], s);
        cudaEventSynchronize(ev[3]);
        float t1 = 0, t2 = 0, t3 = 0;
        cudaEventElapsedTime(&t1, ev[0], ev[1]);
        cudaEventElapsedTime(&t2, ev[1], ev[2]);
        cudaEventElapsedTime(&t3, ev[2], ev[3]);
        fprintf(stderr, "dc n=%d: tridiagonalisation %.3f ms, divide and conquer %.3f ms, back-transform %.3f ms\n", n,
                t1, t2, t3);
        for (auto &e : ev) cudaEventDestroy(e);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
