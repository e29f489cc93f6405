// sgp_grid.cuh — Laplace-grid evidence oracle on device (
// reference evidence.py:330-426 and lbfgs.py:27-150).
//
// One CTA per (c_g, sigma_g) grid node.  Each CTA runs the reference's
// L-BFGS (memory 10, strong Wolfe search with bisection zoom, the same
// acceptance tests and restart rules) on the coefficient block in
// prior-whitened coordinates, with the posterior potential and gradient from
// the same CTA-level evaluator the sampler uses; then the Hessian's
// coefficient block is Cholesky-factorised in the CTA (right-looking, fails
// exactly where LAPACK dpotrf reports a non-positive pivot) for the log
// determinant.  Nodes are independent: every node first starts at a = 0
// instead of the reference's serpentine warm start (same optimum within the
// optimiser tolerance, tests/test_gpu_laplace.py); nodes that fail from there
// are retried warm-started from the last converged node before them in
// serpentine order, which is the reference's own a_warm rule.
#pragma once
#include "sgp_chain.cuh"

__host__ __device__ inline size_t sgp_grid_scratch_extra(int d, int m) { return (size_t)2 * m * d + 2 * (size_t)m + 8; }

struct GridDev {
    int nc, ns;                // centers per axis
    double c_mesh, s_mesh;
    int n_pinned;
    int pin_pos[3];
    double pin_q[3];           // sampled-coordinate value of each pinned hyper
    double gtol;
    int max_iters, memory;
    double log_area;
};

// in whitened coordinates x (n coefficients): f = U(q), g = grad_U[coef] * scale
struct GridCtx {
    ChainWS *w;
    EvalCtx *E;
    const int *cidx;   // coefficient coordinates (n)
    const double *sc;  // scales (n)
    double *q;         // full point (d)
    double tau;
    int n, d;
};

__device__ __noinline__ double grid_fg(GridCtx &G, const double *x, double *g) {
    for (int i = threadIdx.x; i < G.n; i += SGP_NT) G.q[G.cidx[i]] = x[i] * G.sc[i];
    __syncthreads();
    EvalOut o;
    eval_state(*G.E, G.q, G.tau, SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT, G.w->grad, nullptr, o);
    const bool bad = *G.E->status != 0;
    __syncthreads();
    for (int i = threadIdx.x; i < G.n; i += SGP_NT) g[i] = bad ? 0.0 : G.w->grad[G.cidx[i]] * G.sc[i];
    if (threadIdx.x == 0) *G.E->status = 0;  // DomainError / DivergenceError -> +inf (evidence.py:397-398)
    __syncthreads();
    return bad ? INFINITY : o.pot;
}

__device__ __forceinline__ double vdot(const double *a, const double *b, int n, double *red) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += SGP_NT) s += a[i] * b[i];
    return block_sum(s, red);
}
__device__ __forceinline__ double vmaxabs(const double *a, int n, double *red) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += SGP_NT) s = fmax(s, fabs(a[i]));
    return block_max_nan(s, red);
}
// out = x + a d
__device__ __forceinline__ void vaxpy(double *out, const double *x, double a, const double *d, int n) {
    for (int i = threadIdx.x; i < n; i += SGP_NT) out[i] = __dadd_rn(x[i], __dmul_rn(a, d[i]));  // numpy rounding
    __syncthreads();
}

// strong Wolfe line search (lbfgs.py:43-86); on success returns alpha with f, g at
// x + alpha d in (*fo, go); alpha < 0 = failure
struct LsBuf {
    double *xt, *gt, *glo;  // trial point, trial gradient, scratch
};
__device__ double grid_zoom(GridCtx &G, LsBuf &B, const double *x, const double *d, double f0, double dphi0,
                            double lo, double f_lo, double hi, double c1, double c2, double *fo, double *go,
                            int *evals) {
    double *red = G.E->red;
    for (int it = 0; it < 30; ++it) {
        const double a = 0.5 * (lo + hi);
        vaxpy(B.xt, x, a, d, G.n);
        const double f = grid_fg(G, B.xt, B.gt);
        ++*evals;
        const double dphi = isfinite(f) ? vdot(B.gt, d, G.n, red) : INFINITY;
        if (!isfinite(f) || f > f0 + c1 * a * dphi0 || f >= f_lo) {
            hi = a;
        } else {
            if (fabs(dphi) <= -c2 * dphi0) {
                *fo = f;
                for (int i = threadIdx.x; i < G.n; i += SGP_NT) go[i] = B.gt[i];
                __syncthreads();
                return a;
            }
            if (dphi * (hi - lo) >= 0.0) hi = lo;
            lo = a;
            f_lo = f;
        }
        if (fabs(hi - lo) <= 1e-14 * fmax(1.0, fabs(lo))) break;
    }
    vaxpy(B.xt, x, lo, d, G.n);
    const double f = grid_fg(G, B.xt, B.gt);
    ++*evals;
    if (isfinite(f) && f <= f0 + c1 * lo * dphi0 && lo > 0.0) {
        *fo = f;
        for (int i = threadIdx.x; i < G.n; i += SGP_NT) go[i] = B.gt[i];
        __syncthreads();
        return lo;
    }
    return -1.0;
}

__device__ double grid_wolfe(GridCtx &G, LsBuf &B, const double *x, double f0, const double *g0, const double *d,
                             double c1, double c2, double *fo, double *go, int *evals) {
    double *red = G.E->red;
    const double dphi0 = vdot(g0, d, G.n, red);
    double a_prev = 0.0, f_prev = f0, a = 1.0;
    for (int i = 0; i < 25; ++i) {
        vaxpy(B.xt, x, a, d, G.n);
        const double f = grid_fg(G, B.xt, B.gt);
        ++*evals;
        if (!isfinite(f) || f > f0 + c1 * a * dphi0 || (i > 0 && f >= f_prev))
            return grid_zoom(G, B, x, d, f0, dphi0, a_prev, f_prev, a, c1, c2, fo, go, evals);
        const double dphi = vdot(B.gt, d, G.n, red);
        if (fabs(dphi) <= -c2 * dphi0) {
            *fo = f;
            for (int k = threadIdx.x; k < G.n; k += SGP_NT) go[k] = B.gt[k];
            __syncthreads();
            return a;
        }
        if (dphi >= 0.0) return grid_zoom(G, B, x, d, f0, dphi0, a, f, a_prev, c1, c2, fo, go, evals);
        a_prev = a;
        f_prev = f;
        a *= 2.0;
    }
    return -1.0;
}

// two-loop recursion (lbfgs.py:27-40); hist rows are ring-ordered oldest..newest
__device__ void grid_two_loop(const double *g, double *q, const double *S, const double *Y, const double *rho,
                              int m, int head, int cnt, int n, int ld, double *alpha, double *red) {
    for (int i = threadIdx.x; i < n; i += SGP_NT) q[i] = g[i];
    __syncthreads();
    for (int k = cnt - 1; k >= 0; --k) {
        const int r = (head + k) % m;
        const double a = rho[r] * vdot(S + (size_t)r * ld, q, n, red);
        if (threadIdx.x == 0) alpha[k] = a;
        for (int i = threadIdx.x; i < n; i += SGP_NT) q[i] = __dsub_rn(q[i], __dmul_rn(a, Y[(size_t)r * ld + i]));
        __syncthreads();
    }
    if (cnt > 0) {
        const int r = (head + cnt - 1) % m;
        const double sy = vdot(S + (size_t)r * ld, Y + (size_t)r * ld, n, red);
        const double yy = vdot(Y + (size_t)r * ld, Y + (size_t)r * ld, n, red);
        const double f = sy / yy;
        for (int i = threadIdx.x; i < n; i += SGP_NT) q[i] = __dmul_rn(q[i], f);
        __syncthreads();
    }
    for (int k = 0; k < cnt; ++k) {
        const int r = (head + k) % m;
        const double b = rho[r] * vdot(Y + (size_t)r * ld, q, n, red);
        const double a = alpha[k];
        for (int i = threadIdx.x; i < n; i += SGP_NT) q[i] = __dadd_rn(q[i], __dmul_rn(__dsub_rn(a, b), S[(size_t)r * ld + i]));
        __syncthreads();
    }
}

// In-place Cholesky of the n x n matrix A (row-major), lower factor; returns
// log det A, or NaN when a pivot is not positive (numpy LinAlgError).
__device__ double chol_logdet(double *A, int n, double *red) {
    __shared__ int fail;
    if (threadIdx.x == 0) fail = 0;
    __syncthreads();
    double ld = 0.0;
    for (int k = 0; k < n; ++k) {
        const double akk = A[(size_t)k * n + k];
        if (!(akk > 0.0)) {
            if (threadIdx.x == 0) fail = 1;
            __syncthreads();
            break;
        }
        const double lkk = sqrt(akk);
        ld += log(lkk);
        __syncthreads();
        for (int i = k + 1 + threadIdx.x; i < n; i += SGP_NT) A[(size_t)i * n + k] /= lkk;
        __syncthreads();
        const int m = n - k - 1;
        for (int idx = threadIdx.x; idx < m * m; idx += SGP_NT) {
            const int i = k + 1 + idx / m, j = k + 1 + idx % m;
            if (j <= i) A[(size_t)i * n + j] -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
        }
        __syncthreads();
    }
    return fail ? NAN : 2.0 * ld;
}

// The reference's L-BFGS (lbfgs.py:89-150) on the CTA; x holds the start and
// returns the iterate, g its gradient, *fout its value.  History rows of
// stride d in Sh/Yh, ring-ordered.  Returns 0 converged, 1 not converged,
// 3 objective not finite at the start (lbfgs.py:110 raises ValueError).
__device__ __noinline__ int grid_lbfgs(GridCtx &G, LsBuf &B, double *x, double *g, double *dir, double *xn,
                                       double *gn, double *sv, double *yv, double *Sh, double *Yh, double *rho,
                                       double *alph, int m, double gtol, int max_iters, int *iters, double *fout) {
    const int n = G.n, d = G.d;
    int evals = 1, head = 0, cnt = 0, st = 1, it = 0;
    double f = grid_fg(G, x, g);
    if (!isfinite(f)) {
        st = 3;
    } else {
        for (it = 0; it < max_iters; ++it) {
            if (vmaxabs(g, n, G.E->red) <= gtol) {
                st = 0;
                break;
            }
            grid_two_loop(g, dir, Sh, Yh, rho, m, head, cnt, n, d, alph, G.E->red);
            for (int i = threadIdx.x; i < n; i += SGP_NT) dir[i] = -dir[i];
            __syncthreads();
            if (vdot(g, dir, n, G.E->red) >= 0.0) {
                cnt = 0;
                head = 0;
                for (int i = threadIdx.x; i < n; i += SGP_NT) dir[i] = -g[i];
                __syncthreads();
            }
            double fnew = f;
            double alpha = grid_wolfe(G, B, x, f, g, dir, 1e-4, 0.9, &fnew, gn, &evals);
            if (alpha < 0.0 && cnt > 0) {
                // stale curvature pairs near the optimum: retry once from steepest descent
                cnt = 0;
                head = 0;
                for (int i = threadIdx.x; i < n; i += SGP_NT) dir[i] = -g[i];
                __syncthreads();
                alpha = grid_wolfe(G, B, x, f, g, dir, 1e-4, 0.9, &fnew, gn, &evals);
            }
            if (alpha < 0.0) {
                st = vmaxabs(g, n, G.E->red) <= gtol ? 0 : 1;
                break;
            }
            // s = x_new - x, y = g_new - g
            vaxpy(xn, x, alpha, dir, n);
            for (int i = threadIdx.x; i < n; i += SGP_NT) {
                sv[i] = xn[i] - x[i];
                yv[i] = gn[i] - g[i];
            }
            __syncthreads();
            const double sy = vdot(sv, yv, n, G.E->red);
            const double ss = vdot(sv, sv, n, G.E->red), yy = vdot(yv, yv, n, G.E->red);
            if (sy > 1e-12 * sqrt(ss) * sqrt(yy)) {
                // ring: append at the end, drop the oldest when full (lbfgs.py:140-146)
                const int slot = (head + cnt) % m;
                for (int i = threadIdx.x; i < n; i += SGP_NT) {
                    Sh[(size_t)slot * d + i] = sv[i];
                    Yh[(size_t)slot * d + i] = yv[i];
                }
                if (threadIdx.x == 0) rho[slot] = 1.0 / sy;
                if (cnt < m)
                    ++cnt;
                else
                    head = (head + 1) % m;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += SGP_NT) {
                x[i] = xn[i];
                g[i] = gn[i];
            }
            f = fnew;
            __syncthreads();
        }
        if (it == max_iters) st = vmaxabs(g, n, G.E->red) <= gtol ? 0 : 1;
    }
    *iters = it;
    *fout = f;
    return st;
}

__device__ __forceinline__ double inv_gamma_logpdf(double th, double a, double b) {
    return a * log(b) - lgamma(a) - (a + 1.0) * log(th) - b / th;
}

// status: 0 ok, 1 optimiser did not converge, 2 Cholesky failed, 3 objective not
// finite at the start (the reference raises ValueError there)
// list == nullptr: nodes node0 + blockIdx.x (first pass, a = 0 starts);
// else node = list[node0 + blockIdx.x] warm-started from the optimum asrc of node
// src[...] (the reference's serpentine a_warm, evidence.py:393-399; src < 0: a = 0).
// The optimum of every node whose L-BFGS converged is kept in aopt[node * d + i]
// (raw coefficients), before the Cholesky test, as the reference updates a_warm.
__global__ void __launch_bounds__(SGP_MAX_NT) k_laplace_grid(ModelDev M, SmemPlan pl, GridDev gd, int node0,
                                                            int nodes, double *scratch, size_t spc, size_t stride,
                                                            double *val, int *status, int *iters, const int *list,
                                                            const int *src, const double *asrc, double *aopt) {
    const int slot_id = node0 + blockIdx.x;
    if (slot_id >= nodes) return;
    const int node = list ? list[slot_id] : slot_id;
    const int from = list ? src[slot_id] : -1;
    const ModelParams &mp = M.mp;
    const int d = mp.d;
    ChainWS w;
    EvalCtx E;
    double *my = scratch + (size_t)blockIdx.x * stride;
    setup_ws(w, E, sgp_smem, pl, M, my);
    // node -> (c, sigma), serpentine order (evidence.py:370-372)
    const int si = node / gd.nc, j = node - si * gd.nc;
    const int ci = (si % 2 == 0) ? j : gd.nc - 1 - j;
    const double c = (ci + 0.5) * gd.c_mesh, sg = (si + 0.5) * gd.s_mesh;
    const bool logt = mp.transform == SGP_TRANSFORM_LOG;
    // point: pinned hypers, node hypers, coefficients 0 (vectors: q0 = q, qc/qn/qs/p/ph/pn/v0 = work)
    double *q = w.q0;
    for (int a = threadIdx.x; a < d; a += SGP_NT) q[a] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 0; k < gd.n_pinned; ++k) q[gd.pin_pos[k]] = gd.pin_q[k];
        q[mp.hpos[0]] = logt ? log(c) : c;
        q[mp.hpos[1]] = logt ? log(sg) : sg;
    }
    __syncthreads();
    // coefficient list and prior scales (posterior.py:289-307)
    // T slot (never aliased): coefficient list + scales; history after the chain scratch
    int *cidx = reinterpret_cast<int *>(w.T);
    double *scl = w.T + d;
    int *ncoef = reinterpret_cast<int *>(E.red + 100);
    if (threadIdx.x == 0) {
        int n = 0;
        for (int a = 0; a < d; ++a)
            if (M.ckind[a] != CK_HYPER) cidx[n++] = a;
        *ncoef = n;
    }
    __syncthreads();
    const int n = *ncoef;
    for (int i = threadIdx.x; i < n; i += SGP_NT) {
        const int a = cidx[i];
        const int k = M.ckind[a];
        if (k == CK_INTERCEPT) {
            scl[i] = sqrt(mp.sigma);
        } else {
            CoefD cd;
            coef_derivs(mp, k, M.cw[a], q, cd);
            scl[i] = exp(-0.5 * cd.rho);
        }
    }
    __syncthreads();
    GridCtx G{&w, &E, cidx, scl, q, 1.0, n, d};
    // L-BFGS state (lbfgs.py:89-150): vectors in the chain vectors, history in W
    double *x = w.qc, *g = w.qn, *dir = w.qs, *xn = w.p, *gn = w.ph;
    LsBuf B{w.pn, w.v0, w.tv};
    const int m = gd.memory;
    double *hist = my + spc;  // sgp_grid_scratch_extra(d, m) doubles
    double *Sh = hist, *Yh = hist + (size_t)m * d, *rho = hist + (size_t)2 * m * d, *alph = rho + m;
    double *sv = w.bv, *yv = w.tmp;  // candidate pair before acceptance
    for (int i = threadIdx.x; i < n; i += SGP_NT) x[i] = from >= 0 ? asrc[(size_t)from * d + i] / scl[i] : 0.0;
    __syncthreads();
    int it = 0;
    double f = 0.0;
    int st = grid_lbfgs(G, B, x, g, dir, xn, gn, sv, yv, Sh, Yh, rho, alph, m, gd.gtol, gd.max_iters, &it, &f);
    double value = NAN;
    if (st == 0)
        for (int i = threadIdx.x; i < n; i += SGP_NT) aopt[(size_t)node * d + i] = x[i] * scl[i];
    if (st == 0) {
        // node value at the optimum (evidence.py:400-410)
        for (int i = threadIdx.x; i < n; i += SGP_NT) q[cidx[i]] = x[i] * scl[i];
        __syncthreads();
        EvalOut o;
        eval_state(E, q, 1.0, SGP_EVAL_POTENTIAL | SGP_EVAL_HESSIAN, w.grad, w.H, o);
        double hp = 0.0;
        if (threadIdx.x == 0) {
            for (int s = 0; s < 3; ++s) {
                if (mp.hpos[s] < 0) continue;
                double u[4];
                hyperprior(mp, s, q[mp.hpos[s]], u);
                hp += u[0];
            }
            E.red[90] = hp;
        }
        __syncthreads();
        hp = E.red[90];
        const double conditional = o.pot - hp;
        // coefficient block of H into P0 (n x n), Cholesky
        double *Hc = w.P[0];
        for (int idx = threadIdx.x; idx < n * n; idx += SGP_NT) {
            const int i = idx / n, jj = idx - i * n;
            Hc[idx] = w.H[(size_t)cidx[i] * d + cidx[jj]];
        }
        __syncthreads();
        const double logdet = chol_logdet(Hc, n, E.red);
        if (isnan(logdet) || *E.status) {
            st = 2;
        } else {
            value = -conditional + 0.5 * n * SGP_LN_2PI - 0.5 * logdet +
                    inv_gamma_logpdf(c, mp.alpha[0], mp.beta[0]) + inv_gamma_logpdf(sg, mp.alpha[1], mp.beta[1]) +
                    gd.log_area;
        }
    }
    if (threadIdx.x == 0) {
        val[node] = value;
        status[node] = st;
        iters[node] = it;
    }
}

// laplace_full (evidence.py:277-304) for one posterior: L-BFGS over all d
// coordinates from q0, Hessian at the mode, cold cyclic Jacobi (bit-exact
// with the reference's Numba sweeps) for the eigenvalues.  out[0] value,
// out[1] U(q*), out[2] log det, out[3] min eigenvalue; *status 0 ok,
// 1 mode search did not reach gtol, 2 not positive definite, 3 objective not
// finite at the start, 4 Jacobi sweep cap (JacobiError); *iters L-BFGS iterations.
__global__ void __launch_bounds__(SGP_MAX_NT) k_laplace_full(ModelDev M, SmemPlan pl, const double *q0, double tau,
                                                            double gtol, int max_iters, int memory, double zeta,
                                                            int sweep_cap, double *scratch, size_t spc, double *out,
                                                            int *status, int *iters) {
    const ModelParams &mp = M.mp;
    const int d = mp.d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, scratch);
    int *cidx = reinterpret_cast<int *>(w.T);
    double *scl = w.T + d;
    for (int i = threadIdx.x; i < d; i += SGP_NT) {
        cidx[i] = i;
        scl[i] = 1.0;
    }
    double *q = w.q0, *x = w.qc, *g = w.qn, *dir = w.qs, *xn = w.p, *gn = w.ph;
    for (int i = threadIdx.x; i < d; i += SGP_NT) x[i] = q0[i];
    __syncthreads();
    GridCtx G{&w, &E, cidx, scl, q, tau, d, d};
    LsBuf B{w.pn, w.v0, w.tv};
    double *hist = scratch + spc;
    double *Sh = hist, *Yh = hist + (size_t)memory * d, *rho = hist + (size_t)2 * memory * d, *alph = rho + memory;
    int it = 0;
    double f = 0.0;
    int st = grid_lbfgs(G, B, x, g, dir, xn, gn, w.bv, w.tmp, Sh, Yh, rho, alph, memory, gtol, max_iters, &it, &f);
    double ld = 0.0, lmin = NAN, value = NAN;
    if (st == 0) {
        for (int i = threadIdx.x; i < d; i += SGP_NT) q[i] = x[i];
        __syncthreads();
        EvalOut o;
        eval_state(E, q, tau, SGP_EVAL_HESSIAN, w.grad, w.H, o);
        if (*E.status) {
            st = 2;
        } else {
            sgp_chain_config cfg{};
            cfg.zeta = zeta;
            cfg.sweep_cap = sweep_cap;
            cfg.kappa = 1.0;
            int sw = 0;
            if (eig_cold(w, E, d, cfg, 0, &sw)) {
                st = 4;
            } else {
                double s = 0.0, mn = INFINITY;
                for (int j = threadIdx.x; j < d; j += SGP_NT) {
                    mn = fmin(mn, w.lam[0][j]);
                    s += log(w.lam[0][j]);
                }
                mn = -block_max_nan(-mn, E.red);
                s = block_sum(s, E.red);
                lmin = mn;
                if (!(mn > 0.0)) {
                    st = 2;
                } else {
                    ld = s;
                    value = -f + 0.5 * d * SGP_LN_2PI - 0.5 * ld;
                }
            }
        }
    }
    if (threadIdx.x == 0) {
        out[0] = value;
        out[1] = f;
        out[2] = ld;
        out[3] = lmin;
        *status = st;
        *iters = it;
    }
}
