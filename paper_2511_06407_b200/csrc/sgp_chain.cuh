// sgp_chain.cuh — generalized leapfrog and the MH move loop, one chain per
// CTA, entirely on the device (sampler.py:163-418 in the reference).
#pragma once
#include "sgp_eval.cuh"

struct ChainWS {
    double *P[2];  // eigenvector ping-pong (frame / next q-iterate)
    double *T;     // divided differences of the frame metric
    double *W;     // contraction matrix W2 - W1
    double *X;     // GEMM temporary
    double *H;     // Hessian, then Psi^T H Psi
    double *q0, *qc, *qn, *qs, *p, *ph, *pn, *v0, *grad, *tv, *bv, *tmp;
    double *lam[2], *g[2];
    double *prm;   // parallel-Jacobi parameters
    double *jlog;  // rotation log of the cyclic Jacobi (scratch)
    double *sc;    // shared scalars: [0..1] logdet[2], [2] pot, [3] su, [4] pot_start
    int *si;       // shared ints: [0..1] since[2]
};

// Shared-memory layout (host and device compute it identically).
// Matrices, in placement priority: H (the serial Jacobi works in it every
// rotation), Wp (padded contraction matrix read by every trace tile; aliases
// H when H is placed), W, P0, P1, X (aliases the tile stage when it fits), T.  Those that do not fit the per-CTA budget live in the chain's
// L2-resident scratch slice, so several chains can share an SM.
#define SGP_NMAT 7
struct SmemPlan {
    int CH;
    size_t off_vec, off_prm, off_stage, bytes;
    size_t stage_cap;  // doubles in the stage region (>= sgp_stage_doubles)
    size_t off_mat[SGP_NMAT];  // byte offset in smem, or (size_t)-1 if in scratch
};

__host__ __device__ inline size_t sgp_round2(size_t x) { return (x + 1) & ~size_t(1); }

// double-buffered Phi / weight stage + the trace's per-tile partial sums
__host__ __device__ inline size_t sgp_stage_doubles(int Dp, int CH, int nt) {
    return sgp_round2(2 * ((size_t)CH * (Dp + 2) + 3 * (size_t)CH) +
                      (size_t)sgp_trace_ks(Dp, CH, nt) * (Dp / 4) * CH * 3 + 2);
}

__host__ __device__ inline size_t sgp_mat_doubles(int i, int d, int Dp) {
    return i == 1 ? (size_t)Dp * Dp : (size_t)d * d;
}

__host__ __device__ inline SmemPlan sgp_smem_plan(int d, int Dp, int nt, size_t budget, int ch = 0) {
    SmemPlan s;
    s.CH = ch > 0 ? ch : (nt <= 64 ? 16 : ((Dp <= 48 && nt >= 128) ? 64 : 32));
    // smaller sample chunks when the fixed part alone would exceed the per-CTA budget
    // (keeps two 256-thread CTAs per SM at d ~ 160)
    auto fixed_bytes = [&](int CH) {
        return (128 + sgp_round2(16 * (size_t)d + 8) + sgp_round2(6 * (size_t)((d + 2) / 2) + 8) +
                sgp_stage_doubles(Dp, CH, nt)) * sizeof(double);
    };
    while (ch <= 0 && s.CH > 16 && fixed_bytes(s.CH) > budget) s.CH >>= 1;
    size_t off = 0;
    off += 128 * sizeof(double);  // red + status + scalars + ints
    s.off_vec = off;
    off += sgp_round2(16 * (size_t)d + 8) * sizeof(double);
    s.off_prm = off;
    off += sgp_round2(6 * (size_t)((d + 2) / 2) + 8) * sizeof(double);
    s.off_stage = off;
    s.stage_cap = sgp_stage_doubles(Dp, s.CH, nt);
    {
        // CTAs without V-update overlap keep the eigenvector working copy and one
        // rotation-log slot in the stage during a Jacobi: grow the stage to hold
        // both when that still leaves room for H (the Jacobi matrix)
        const size_t need = sgp_round2((size_t)d * d) + sgp_jlog_slot(d);
        const size_t hdd = sgp_round2((size_t)d * d) * sizeof(double);
        if (nt <= 64 && d <= 256 && need > s.stage_cap && off + need * sizeof(double) + hdd <= budget)
            s.stage_cap = sgp_round2(need);
    }
    off += s.stage_cap * sizeof(double);
    for (int i = 0; i < SGP_NMAT; ++i) {
        const size_t m = sgp_round2(sgp_mat_doubles(i, d, Dp)) * sizeof(double);
        // Wp (padded trace operand) shares H's slot: H is consumed by the
        // eigendecomposition right after every Hessian evaluation and Wp
        // lives only inside one trace contraction
        if (i == 1 && s.off_mat[0] != (size_t)-1 && (size_t)Dp * Dp <= (size_t)d * d) {
            s.off_mat[1] = s.off_mat[0];
            continue;
        }
        // X (product scratch of the W formation and Psi^T H Psi) shares the
        // tile stage, which is idle in both
        if (i == 5 && (size_t)d * d <= s.stage_cap) {
            s.off_mat[5] = s.off_stage;
            continue;
        }
        if (off + m <= budget) {
            s.off_mat[i] = off;
            off += m;
        } else {
            s.off_mat[i] = (size_t)-1;
        }
    }
    s.bytes = off;
    return s;
}

// per-chain scratch (doubles): per-sample fields (nf of them: sgp_fields), the 7 matrices, Jacobi log
__host__ __device__ inline size_t sgp_scratch_mat_offset(int ld, int d, int Dp, int i, int nf) {
    size_t off = (size_t)nf * ld;
    for (int k = 0; k < i; ++k) off += sgp_round2(sgp_mat_doubles(k, d, Dp));
    return off;
}
__host__ __device__ inline size_t sgp_scratch_per_chain(int ld, int d, int Dp, int nf) {
    return sgp_scratch_mat_offset(ld, d, Dp, SGP_NMAT, nf) + sgp_jacobi_log_doubles(d) + 2 * (size_t)d + 64;
}

__device__ inline void setup_ws(ChainWS &w, EvalCtx &E, char *smem, const SmemPlan &pl, const ModelDev &M,
                                double *scratch) {
    const int d = M.mp.d, Dp = M.mp.Dp, ld = M.mp.ld;
    E.M = M;
    E.red = reinterpret_cast<double *>(smem);
    E.status = reinterpret_cast<int *>(smem + 64 * sizeof(double));
    w.sc = reinterpret_cast<double *>(smem + 80 * sizeof(double));
    w.si = reinterpret_cast<int *>(smem + 120 * sizeof(double));
    double *v = reinterpret_cast<double *>(smem + pl.off_vec);
    double **vecs[] = {&w.q0, &w.qc, &w.qn, &w.qs, &w.p, &w.ph, &w.pn, &w.v0, &w.grad, &w.tv, &w.bv, &w.tmp,
                       &w.lam[0], &w.lam[1], &w.g[0], &w.g[1]};
    for (int k = 0; k < 16; ++k) *vecs[k] = v + (size_t)k * d;
    w.prm = reinterpret_cast<double *>(smem + pl.off_prm);
    E.stage = reinterpret_cast<double *>(smem + pl.off_stage);
    E.CH = pl.CH;
    E.stage_cap = (int)pl.stage_cap;
    E.S = scratch;
    E.ext_trace = 0;
    double **mats[SGP_NMAT] = {&w.H, &E.wp, &w.W, &w.P[0], &w.P[1], &w.X, &w.T};
    for (int i = 0; i < SGP_NMAT; ++i)
        *mats[i] = pl.off_mat[i] != (size_t)-1 ? reinterpret_cast<double *>(smem + pl.off_mat[i])
                                               : scratch + sgp_scratch_mat_offset(ld, d, Dp, i, sgp_fields(M.mp));
    w.jlog = scratch + sgp_scratch_mat_offset(ld, d, Dp, SGP_NMAT, sgp_fields(M.mp));
    if (threadIdx.x == 0) *E.status = 0;
    __syncthreads();
}

// Working copy of the eigenvector matrix during a cyclic Jacobi, stored
// column-major so the row-parallel log application is coalesced (global) /
// conflict-free (shared): the tile stage when it fits (idle during the
// Jacobi), else the X scratch matrix (free between Psi^T H Psi and the next W).
__device__ __forceinline__ double *jac_vwork(const ChainWS &w, const EvalCtx &E, int d) {
    if (E.stage && (size_t)d * d <= (size_t)E.stage_cap) return E.stage;
    return w.X;
}
// one rotation-log slot after the V working copy in the stage, when both fit
__device__ __forceinline__ double *jac_log_smem(const EvalCtx &E, const double *Vt, int d) {
    if (Vt != E.stage) return nullptr;
    const size_t off = sgp_round2((size_t)d * d);
    return off + sgp_jlog_slot(d) <= (size_t)E.stage_cap ? E.stage + off : nullptr;
}
// Vt (column-major) -> P (row-major)
__device__ __forceinline__ void jac_vwork_out(double *P, const double *Vt, int d) {
    for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) {
        const int j = idx / d, k = idx - j * d;
        P[k * d + j] = Vt[idx];
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// eigendecompositions into ping-pong slot `dst`

// Cold: H is consumed (becomes A); V = P[dst] from identity (metric.py:112-142).
__device__ __noinline__ int eig_cold(ChainWS &w, EvalCtx &E, int d, const sgp_chain_config &cfg, int dst, int *sweeps_out) {
    mat_symmetrize(w.H, d);
    const double hnorm = sqrt(frob2(w.H, d * d, E.red));
    const double tol = cfg.zeta * hnorm;
    const double skip = d ? tol / d : 0.0;
    double *Vt = jac_vwork(w, E, d);
    for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) {
        const int j = idx / d, k = idx - j * d;
        Vt[idx] = k == j ? 1.0 : 0.0;
    }
    __syncthreads();
    int sw;
    {
        SGP_PROF(8);
        sw = jacobi_cyclic(w.H, Vt, d, tol, skip, cfg.sweep_cap, E.red, w.jlog, 1, d, jac_log_smem(E, Vt, d));
    }
    jac_vwork_out(w.P[dst], Vt, d);
    if (sweeps_out) *sweeps_out = sw;
    if (sw < 0) return SGP_STATUS_JACOBI;
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.lam[dst][j] = w.H[j * d + j];
    __syncthreads();
    double ld = metric_g(w.lam[dst], w.g[dst], d, cfg.kappa, E.red);
    if (threadIdx.x == 0) {
        w.sc[dst] = ld;
        w.si[dst] = 0;
    }
    __syncthreads();
    return 0;
}

// Warm: previous basis in P[src] (may be re-orthonormalised in place), result
// in P[dst] (metric.py:145-185).  H is consumed.
__device__ __noinline__ int eig_warm(ChainWS &w, EvalCtx &E, int d, const sgp_chain_config &cfg, int src, int dst,
                        int *sweeps_out) {
    int since = w.si[src] + 1;
    if (cfg.gs_interval && since >= cfg.gs_interval) {
        SGP_PROF(3);
        mgs(w.P[src], d, E.red);
        since = 0;
    }
    const double hnorm = sqrt(frob2(w.H, d * d, E.red));
    {
        SGP_PROF(4);
        mat_mul<2>(w.X, w.P[src], w.H, d);  // X = Psi^T H
        mat_mul<0>(w.H, w.X, w.P[src], d);  // A = X Psi
        mat_symmetrize(w.H, d);
    }
    const double tol = cfg.zeta * hnorm;
    const double skip = d ? tol / d : 0.0;
    int sw;
    SGP_PROF(5);
    if (cfg.warm_order == SGP_ORDER_CYCLIC) {
        // rotations applied to Psi directly (== Psi Q), in shared memory when it fits
        double *Vt = jac_vwork(w, E, d);
        for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) {
            const int j = idx / d, k = idx - j * d;
            Vt[idx] = w.P[src][k * d + j];
        }
        __syncthreads();
        sw = jacobi_cyclic(w.H, Vt, d, tol, skip, cfg.sweep_cap, E.red, w.jlog, 1, d, jac_log_smem(E, Vt, d));
        jac_vwork_out(w.P[dst], Vt, d);
    } else {
        mat_copy(w.P[dst], w.P[src], d * d);
        sw = jacobi_parallel(w.H, w.P[dst], d, tol, skip, cfg.sweep_cap, E.red, w.prm);
    }
    if (sweeps_out) *sweeps_out = sw;
    if (sw < 0) return SGP_STATUS_JACOBI;
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.lam[dst][j] = w.H[j * d + j];
    __syncthreads();
    double ld = metric_g(w.lam[dst], w.g[dst], d, cfg.kappa, E.red);
    if (threadIdx.x == 0) {
        w.sc[dst] = ld;
        w.si[dst] = since;
    }
    __syncthreads();
    return 0;
}

// ---------------------------------------------------------------------------

struct LFDiag {
    int fp_p, fp_q, nsweep;
    int *sweeps;  // optional per-decomposition log (smem, >= fp_max_iters ints) or null
    double sweep_sum;
    int sweep_cnt;
};

__device__ __forceinline__ void vec_axpy3(double *out, const double *a, double s, const double *b,
                                          const double *c, double cs, int d) {
    // out = a + s * (b + cs * c)
    for (int j = threadIdx.x; j < d; j += SGP_NT) out[j] = a[j] - s * (b[j] + cs * c[j]);
    __syncthreads();
}

// Evaluates the state at w.qc with the requested parts; Hessian into w.H.
__device__ int eval_at(ChainWS &w, EvalCtx &E, const double *q, double tau, int what) {
    EvalOut o;
    eval_state(E, q, tau, what, w.grad, w.H, o);
    if (threadIdx.x == 0) {
        w.sc[2] = o.pot;
        w.sc[3] = o.sumpot;
    }
    __syncthreads();
    return *E.status;
}

// One generalized leapfrog.  Frame = (w.q0, w.grad, per-sample S, metric slot f,
// w.T valid for slot f); momentum in w.p.  On success the frame and w.p are
// advanced and f may change.  Returns a status (sampler.py:209-258).
__device__ __noinline__ int leapfrog_riemann(ChainWS &w, EvalCtx &E, const sgp_chain_config &cfg, double tau, int &f,
                                LFDiag &dg) {
    SGP_PROF(9);
    const int d = E.M.mp.d;
    const double eps = cfg.epsilon;
    // ---- implicit momentum half step, W2 fixed (sampler.py:216-232)
    metric_w(w.W, w.X, w.bv, w.P[f], w.lam[f], w.g[f], w.T, w.p, d, true, true);
    eval_trace(E, w.q0, tau, w.W, w.tv);
    if (*E.status) return *E.status;
    vec_axpy3(w.ph, w.p, 0.5 * eps, w.grad, w.tv, 0.5, d);
    bool conv = false;
    for (int it = 0; it < cfg.fp_max_iters; ++it) {
        { SGP_PROF(0); metric_w(w.W, w.X, w.bv, w.P[f], w.lam[f], w.g[f], w.T, w.ph, d, true, true);
        }
        { SGP_PROF(1); eval_trace(E, w.q0, tau, w.W, w.tv); }
        if (*E.status) return *E.status;
        vec_axpy3(w.pn, w.p, 0.5 * eps, w.grad, w.tv, 0.5, d);
        double dl = 0.0;
        for (int j = threadIdx.x; j < d; j += SGP_NT) dl = fmax(dl, fabs(w.pn[j] - w.ph[j]));
        // NaN deltas fail the <= test, as in numpy
        bool nan_here = false;
        for (int j = threadIdx.x; j < d; j += SGP_NT) nan_here |= isnan(w.pn[j] - w.ph[j]);
        double delta = block_max_nan(nan_here ? NAN : dl, E.red);
        for (int j = threadIdx.x; j < d; j += SGP_NT) w.ph[j] = w.pn[j];
        __syncthreads();
        if (delta <= cfg.fp_tol) {
            conv = true;
            dg.fp_p = it + 1;
            break;
        }
    }
    if (!conv) return SGP_STATUS_STALL_P;
    // ---- implicit position step (sampler.py:234-252)
    metric_apply(w.v0, w.tmp, w.P[f], w.g[f], w.ph, d, 0);
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.qc[j] = w.q0[j] + eps * w.v0[j];
    __syncthreads();
    int prev = f, cur = f;
    conv = false;
    for (int it = 0; it < cfg.fp_max_iters; ++it) {
        int st;
        {
            SGP_PROF(2);
            st = eval_at(w, E, w.qc, tau, SGP_EVAL_HESSIAN);
        }
        if (st) return st;
        const int nxt = 1 - prev;
        int sw = 0;
        if (cfg.metric == SGP_METRIC_STATIC)
            st = eig_cold(w, E, d, cfg, nxt, &sw);
        else
            st = eig_warm(w, E, d, cfg, prev, nxt, &sw);
        if (threadIdx.x == 0 && dg.sweeps && dg.nsweep < 32) dg.sweeps[dg.nsweep] = sw;
        dg.nsweep++;
        if (st) return st;
        dg.sweep_sum += sw;
        dg.sweep_cnt++;
        cur = nxt;
        metric_apply(w.tmp, w.bv, w.P[cur], w.g[cur], w.ph, d, 0);
        double dl = 0.0;
        bool nan_here = false;
        for (int j = threadIdx.x; j < d; j += SGP_NT) {
            double qn = w.q0[j] + 0.5 * eps * (w.v0[j] + w.tmp[j]);
            w.qn[j] = qn;
            dl = fmax(dl, fabs(qn - w.qc[j]));
            nan_here |= isnan(qn - w.qc[j]);
        }
        double delta = block_max_nan(nan_here ? NAN : dl, E.red);
        if (delta <= cfg.fp_tol) {
            conv = true;
            dg.fp_q = it + 1;
            break;
        }
        for (int j = threadIdx.x; j < d; j += SGP_NT) w.qc[j] = w.qn[j];
        __syncthreads();
        prev = cur;
    }
    if (!conv) return SGP_STATUS_STALL_Q;
    // ---- explicit final half step at the new state (sampler.py:254-257)
    f = cur;
    t_matrix(w.T, w.lam[f], w.g[f], d, cfg.kappa);
    metric_w(w.W, w.X, w.bv, w.P[f], w.lam[f], w.g[f], w.T, w.ph, d, true, true);
    {
        EvalOut o;
        eval_state(E, w.qc, tau, SGP_EVAL_GRADIENT | SGP_EVAL_REUSE, w.grad, w.H, o);
        if (*E.status) return *E.status;
    }
    eval_trace(E, w.qc, tau, w.W, w.tv);
    if (*E.status) return *E.status;
    for (int j = threadIdx.x; j < d; j += SGP_NT) {
        w.p[j] = w.ph[j] - 0.5 * eps * (w.grad[j] + 0.5 * w.tv[j]);
        w.q0[j] = w.qc[j];
    }
    __syncthreads();
    return 0;
}

// Euclidean leapfrog (sampler.py:261-267).
__device__ int leapfrog_euclid(ChainWS &w, EvalCtx &E, const sgp_chain_config &cfg, double tau) {
    const int d = E.M.mp.d;
    const double eps = cfg.epsilon;
    for (int j = threadIdx.x; j < d; j += SGP_NT) {
        w.ph[j] = w.p[j] - 0.5 * eps * w.grad[j];
        w.qc[j] = w.q0[j] + eps * w.ph[j];
    }
    __syncthreads();
    int st = eval_at(w, E, w.qc, tau, SGP_EVAL_GRADIENT);
    if (st) return st;
    for (int j = threadIdx.x; j < d; j += SGP_NT) {
        w.p[j] = w.ph[j] - 0.5 * eps * w.grad[j];
        w.q0[j] = w.qc[j];
    }
    __syncthreads();
    return 0;
}

// kinetic + volume terms of the Hamiltonian of the frame (sampler.py:163-169)
__device__ double frame_kinetic(ChainWS &w, EvalCtx &E, const sgp_chain_config &cfg, int f) {
    const int d = E.M.mp.d;
    if (cfg.metric == SGP_METRIC_EUCLIDEAN) {
        double s = 0.0;
        for (int j = threadIdx.x; j < d; j += SGP_NT) s += w.p[j] * w.p[j];
        s = block_sum(s, E.red);
        return 0.5 * s + 0.5 * d * SGP_LN_2PI;
    }
    double qd = metric_quad(w.tmp, w.P[f], w.g[f], w.p, d, E.red);
    return 0.5 * qd + 0.5 * (d * SGP_LN_2PI + w.sc[f]);
}

// Builds the frame at w.q0: potential, gradient, per-sample S and (unless
// Euclidean) the cold metric in slot 0 plus its T matrix (sampler.py:322-328).
__device__ __noinline__ int frame_build(ChainWS &w, EvalCtx &E, const sgp_chain_config &cfg, double tau, int &f) {
    const int d = E.M.mp.d;
    const bool euclid = cfg.metric == SGP_METRIC_EUCLIDEAN;
    int st = eval_at(w, E, w.q0, tau,
                     SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT | (euclid ? 0 : SGP_EVAL_HESSIAN));
    if (st) return st;
    f = 0;
    if (euclid) return 0;
    st = eig_cold(w, E, d, cfg, 0, nullptr);
    if (st) return st;
    t_matrix(w.T, w.lam[0], w.g[0], d, cfg.kappa);
    return 0;
}

// Re-derives the frame from a stored (q, psi, lam, since) without a new
// decomposition: potential, gradient, S, g, logdet, T.
__device__ __noinline__ int frame_resume(ChainWS &w, EvalCtx &E, const sgp_chain_config &cfg, double tau, const double *psi,
                            const double *lam, int since, int &f) {
    const int d = E.M.mp.d;
    int st = eval_at(w, E, w.q0, tau, SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT);
    if (st) return st;
    f = 0;
    if (cfg.metric == SGP_METRIC_EUCLIDEAN) return 0;
    mat_copy(w.P[0], psi, d * d);
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.lam[0][j] = lam[j];
    __syncthreads();
    double ld = metric_g(w.lam[0], w.g[0], d, cfg.kappa, E.red);
    if (threadIdx.x == 0) {
        w.sc[0] = ld;
        w.si[0] = since;
    }
    __syncthreads();
    t_matrix(w.T, w.lam[0], w.g[0], d, cfg.kappa);
    return 0;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
