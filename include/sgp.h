/*
 * sgp.h — C ABI of libsgp.so, the B200 (sm_100a) implementation of the
 * SoftAbs-metric RMHMC inner loop of arxiv 2511.06407 (reference package
 * softabs-gp, /root/reference/pkg/src/softabs_gp).
 *
 * Conventions
 *   - All array arguments named d_* are DEVICE pointers, fp64 row-major,
 *     owned by the caller (the Python host wraps torch tensors).  The library
 *     never frees caller memory.  Host pointers are named h_*.
 *   - Every compute entry point takes a cudaStream_t (passed as void*) and is
 *     asynchronous on it; per-chain status words are written to device memory.
 *   - Batched calls operate on Z independent chains; chain z's data lives at
 *     offset z*stride of each array (stride = d, d*d or N as documented).
 *   - Return value: SGP_OK, or a negative usage/CUDA error.  Numerical
 *     outcomes are per chain in d_status (SGP_STATUS_*), mapping onto the
 *     reference's exception classes:
 *        SGP_STATUS_DIVERGENCE  -> posterior.DivergenceError   (posterior.py:49)
 *        SGP_STATUS_DOMAIN      -> posterior.DomainError       (posterior.py:45)
 *        SGP_STATUS_JACOBI      -> metric.JacobiError          (metric.py:28)
 *        SGP_STATUS_STALL_P/Q   -> DivergenceError "fixed point stalled"
 *                                  (sampler.py:232, 252)
 *        SGP_STATUS_CHAIN_START / _FIRST_MOVE -> sampler.ChainError (sampler.py:349, 389)
 */
#ifndef SGP_H
#define SGP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define SGP_OK 0
#define SGP_EINVAL (-1)
#define SGP_ECUDA (-2)
#define SGP_ENOMEM (-3)

/* per-chain status words */
#define SGP_STATUS_OK 0
#define SGP_STATUS_DIVERGENCE 1
#define SGP_STATUS_DOMAIN 2
#define SGP_STATUS_JACOBI 3
#define SGP_STATUS_STALL_P 4
#define SGP_STATUS_STALL_Q 5
#define SGP_STATUS_CHAIN_START 6
#define SGP_STATUS_FIRST_MOVE 7

/* model vocabulary (rrgp.py:40-47) */
#define SGP_LIK_LOGISTIC 0          /* "logistic"          */
#define SGP_LIK_GAUSSIAN_MEANVAR 1  /* "gaussian_meanvar"  */
#define SGP_LIK_QUADRATIC 2         /* constant-Hessian Gaussian target (tests/conftest.py:14-61) */
#define SGP_KERNEL_GAUSSIAN 0       /* "gaussian_1d" */
#define SGP_KERNEL_LINEAR 1         /* "linear"      */
#define SGP_TRANSFORM_LOG 0
#define SGP_TRANSFORM_IDENTITY 1
#define SGP_HYPER_CG 0              /* HYPER_ORDER = (c_g, sigma_g, c_l), rrgp.py:47 */
#define SGP_HYPER_SG 1
#define SGP_HYPER_CL 2

/* metric modes (sampler.py:40) */
#define SGP_METRIC_DYNAMIC 0        /* "softabs-dynamic" */
#define SGP_METRIC_STATIC 1         /* "softabs-static"  */
#define SGP_METRIC_EUCLIDEAN 2      /* "euclidean"       */

/* warm eigensolver pivot order */
#define SGP_ORDER_CYCLIC 0          /* reference order, _jacobi.py:54-55 */
#define SGP_ORDER_PARALLEL 1        /* round-robin (Brent-Luk) order: d/2 rotations per round */
#define SGP_ORDER_REFINE 2          /* warm only, d > 256: GEMM eigenvector refinement (Ogita-Aishima),
                                       block-Jacobi fallback; elsewhere treated as PARALLEL */
#define SGP_ORDER_DC 3              /* cold only, large-d path: Householder tridiagonalisation +
                                       divide and conquer (sgp_eigh_dc); eigenvalues ascending */

/* what sgp_eval computes */
#define SGP_EVAL_POTENTIAL 1
#define SGP_EVAL_GRADIENT 2
#define SGP_EVAL_HESSIAN 4
#define SGP_EVAL_SUMPOT 8

typedef struct sgp_kernel_desc {
    int kind;           /* SGP_KERNEL_* */
    int covariate;      /* column of x */
    int features;       /* M (1 for linear) */
    double half_width;  /* L */
} sgp_kernel_desc;

/* Mirrors ModelSpec + Dataset (rrgp.py:87-265).  x/y are HOST arrays; the
 * library uploads them and assembles the design matrices on the device. */
typedef struct sgp_model_desc {
    int likelihood;                 /* SGP_LIK_* */
    int n_rows;                     /* N */
    int n_cols;                     /* P */
    const double *h_x;              /* N*P row-major */
    const double *h_y;              /* N */
    int n_functions;                /* J (1 or 2) */
    int n_kernels[2];
    const sgp_kernel_desc *kernels[2];
    int transform;                  /* SGP_TRANSFORM_* */
    double intercept_variance;      /* Sigma */
    double variance_floor;          /* delta */
    int hyper_sampled[3];           /* 1 if sampled (ModelSpec.hyperparameters) */
    double hyper_fixed[3];          /* theta when fixed (ModelSpec.fixed_hypers) */
    double prior_alpha[3];
    double prior_beta[3];
    /* SGP_LIK_QUADRATIC only: U = 0.5 (q-m)^T P (q-m) - tau*c */
    int quad_dim;
    const double *h_precision;      /* quad_dim^2 */
    const double *h_mean;           /* quad_dim */
    double loglik_const;
} sgp_model_desc;

typedef struct sgp_model sgp_model;  /* opaque: device design matrices + tables */

/* Per-chain state for the fused sampler, all device arrays of n_chains rows. */
typedef struct sgp_chain_state {
    int n_chains;
    double *q;          /* Z*d   current position (frame)                      */
    double *psi;        /* Z*d*d frame metric eigenvectors (columns)            */
    double *lam;        /* Z*d   eigenvalues (natural Jacobi order, unsorted)   */
    double *tau;        /* Z     temperature of each chain's target             */
    int *since;         /* Z     MetricState.steps_since_refresh                */
    int *status;        /* Z     SGP_STATUS_*                                   */
    double *scratch;    /* Z*sgp_scratch_doubles(model)                         */
} sgp_chain_state;

/* Chain settings (ChainConfig, sampler.py:49-83). */
typedef struct sgp_chain_config {
    double epsilon;
    int leapfrogs;
    double kappa;
    double zeta;
    int fp_max_iters;
    double fp_tol;
    int gs_interval;
    int sweep_cap;
    int metric;         /* SGP_METRIC_* */
    int warm_order;     /* SGP_ORDER_* of warm decompositions (dynamic_eigendecompose) */
    int cold_order;     /* SGP_ORDER_* of cold decompositions (static_eigendecompose); the
                           fused small-d kernel always uses the reference order */
    int path;           /* SGP_PATH_AUTO: one CTA per chain for d <= 256, the large path above;
                           SGP_PATH_LATENCY: every chain on the whole GPU (large path) */
} sgp_chain_config;
#define SGP_PATH_AUTO 0
#define SGP_PATH_LATENCY 1

/* Per-move records (ChainRecord, sampler.py:86-99), arrays of moves*Z
 * (index move*Z + z); d_rec_q is moves*Z*d or NULL. */
typedef struct sgp_move_records {
    double *logpost;
    double *h_before;
    double *h_after;    /* NaN when divergent */
    double *sweeps_mean;
    double *wall_ms;
    uint8_t *accept;
    uint8_t *divergent;
    double *q;
} sgp_move_records;

/* Diagnostics of one leapfrog (sampler.py:270-271), per chain. */
typedef struct sgp_leapfrog_diag {
    int *fp_p_iters;    /* Z */
    int *fp_q_iters;    /* Z */
    int *sweeps;        /* Z*fp_max_iters, -1 padded */
} sgp_leapfrog_diag;

/* ---- model ------------------------------------------------------------ */
/* Builds Phi_j on the device (FeatureCache, rrgp.py:310-344). */
int sgp_model_create(const sgp_model_desc *desc, sgp_model **out);
int sgp_model_destroy(sgp_model *model);
int sgp_model_dim(const sgp_model *model);              /* d (BlockLayout.dim) */
int sgp_model_rows(const sgp_model *model);             /* N */
int sgp_model_features(const sgp_model *model, int j);  /* D_j incl. intercept */
/* Copies the design matrix of function j (N x D_j row-major) into d_out. */
int sgp_model_phi(const sgp_model *model, int j, double *d_out, void *stream);
size_t sgp_scratch_doubles(const sgp_model *model);     /* per chain */

/* ---- posterior evaluation (PosteriorState, posterior.py:310-542) ------- */
/* Potential (posterior.py:392), gradient (416), Hessian (442), sum_i U_i (383). */
int sgp_eval(const sgp_model *model, int Z, const double *d_tau, const double *d_q,
             int what, double *d_pot, double *d_grad, double *d_hess, double *d_sumpot,
             int *d_status, double *d_scratch, void *stream);
/* Structured third-order contraction t_i = tr(W dH/dq_i) (posterior.py:486-542). */
int sgp_trace(const sgp_model *model, int Z, const double *d_tau, const double *d_q,
              const double *d_w, double *d_t, int *d_status, double *d_scratch,
              void *stream);
/* Per-sample U, dU/df, d2U, d3U (rrgp.py:351-423): f is n*J, outputs n, n*J,
 * n*J*J, n*J*J*J. */
int sgp_potential_derivatives(int likelihood, int n, int J, const double *d_f,
                              const double *d_y, double variance_floor, double *d_u,
                              double *d_d1, double *d_d2, double *d_d3, void *stream);

/* ---- eigensolvers (metric.py:101-185, _jacobi.py) --------------------- */
/* Cold decomposition from the identity, reference pivot order, no FMA:
 * bit-compatible with _jacobi.jacobi_sweeps.  d_sweeps = -1 on cap. */
int sgp_eigh_cold(int Z, int d, const double *d_h, double zeta, int sweep_cap,
                  double *d_lam, double *d_psi, int *d_sweeps, void *stream);
/* Symmetric eigendecomposition of 0.5 (H + H^T) by blocked Householder tridiagonalisation +
 * divide and conquer (north star (3)): lam ascending, psi[i*d + k] = component i of
 * eigenvector k.  Not order-exact with the reference's Jacobi (static_eigendecompose,
 * metric.py:112-127, up to eigenpair order and signs).  1 <= d <= 4096. */
int sgp_eigh_dc(int Z, int d, const double *d_h, double *d_lam, double *d_psi, void *stream);
/* Warm decomposition in the previous basis (dynamic_eigendecompose). */
int sgp_eigh_warm(int Z, int d, const double *d_h, const double *d_psi_prev,
                  const int *d_since_prev, int gs_interval, double zeta, int sweep_cap,
                  int order, double *d_lam, double *d_psi, int *d_since, int *d_sweeps,
                  void *stream);
/* In-place column modified Gram-Schmidt (_jacobi.py:89-107). */
int sgp_mgs(int Z, int d, double *d_psi, void *stream);

/* ---- metric algebra (metric.py:32-241) ----------------------------------- */
#define SGP_W_W1 1
#define SGP_W_W2 2
#define SGP_W_W2_MINUS_W1 3
int sgp_t_matrix(int Z, int d, const double *d_lam, double kappa, double *d_t, void *stream);
/* W1 = Psi((b b^T) o T)Psi^T, b = Psi^T p / g ; W2 = Psi diag(g'/g) Psi^T. */
int sgp_metric_w(int Z, int d, const double *d_psi, const double *d_lam, double kappa,
                 const double *d_p, int which, double *d_w, void *stream);
/* out = G^-1 v (mode 0), G v (mode 1), Psi diag(sqrt g) z (mode 2). */
int sgp_metric_apply(int Z, int d, const double *d_psi, const double *d_lam, double kappa,
                     const double *d_v, int mode, double *d_out, void *stream);
/* p^T G^-1 p and logdet = sum ln g, per chain. */
int sgp_metric_scalars(int Z, int d, const double *d_psi, const double *d_lam, double kappa,
                       const double *d_p, double *d_quad, double *d_logdet, void *stream);

/* ---- integrator and chain ---------------------------------------------- */
/* One generalized leapfrog from (q, p, metric) (leapfrog_step, sampler.py:280-292).
 * Updates d_q, d_p and the metric (psi, lam, since) in place. */
int sgp_leapfrog(const sgp_model *model, const sgp_chain_config *cfg,
                 const sgp_chain_state *st, double *d_p, sgp_leapfrog_diag *diag,
                 void *stream);
/* Builds the initial frame (cold metric at q), _initial_frame sampler.py:322-328. */
int sgp_chain_init(const sgp_model *model, const sgp_chain_config *cfg,
                   const sgp_chain_state *st, void *stream);
/* Runs `moves` MH moves of `cfg->leapfrogs` generalized leapfrogs for every
 * chain, entirely on the device (run_chain's move loop, sampler.py:355-411).
 * d_z: moves*Z*d standard normals, d_logu: moves*Z log-uniforms, both drawn
 * on the host in the reference's RNG order.  move_offset is the index of the
 * first move (move 0 divergence -> SGP_STATUS_FIRST_MOVE). */
int sgp_run_moves(const sgp_model *model, const sgp_chain_config *cfg,
                  const sgp_chain_state *st, int moves, int move_offset,
                  const double *d_z, const double *d_logu, sgp_move_records *rec,
                  void *stream);

/* The thermodynamic-integration ladder walk of every chain in ONE launch (replaces
 * evidence.py:142-163 _ladder_walk): for rung s = 0..n_rungs-1 each chain's
 * target moves to d_taus[s], its frame is rebuilt cold at its current position (a rung is a new
 * run_chain, sampler.py:322-328), moves_per_rung moves run with the rung's draws, and
 * d_values[z * n_rungs + s] = log_likelihood at the rung's end (posterior.py:277-279), or the
 * average over the rung's moves when rung_average.  d_z: n_rungs*moves*Z*d normals,
 * d_logu: n_rungs*moves*Z log-uniforms, in the reference's per-rung RNG order.  A chain that
 * fails (status != 0) stops; its remaining values are untouched.  One CTA per chain: models on
 * the large path (d > 256 or path = latency) return SGP_EINVAL and are walked rung by rung. */
int sgp_ladder_walk(const sgp_model *model, const sgp_chain_config *cfg, const sgp_chain_state *st,
                    int n_rungs, const double *d_taus, int moves_per_rung, int rung_average,
                    const double *d_z, const double *d_logu, double *d_values, void *stream);

/* Laplace-grid evidence oracle (replaces evidence.py:330-426
 * laplace_grid_oracle's node loop).  The grid of
 * (c_g, sigma_g) midpoints is round(c_max/c_mesh) x round(sigma_max/sigma_mesh)
 * nodes in the reference's serpentine order; every node optimises the
 * coefficient block in prior-whitened coordinates with the reference's
 * L-BFGS (memory, strong Wolfe search, gtol, max_iters) from a = 0 (all nodes
 * concurrently; nodes that fail are retried warm-started from the optimum of
 * the last converged node before them in serpentine order, the reference's
 * a_warm) and Cholesky-factorises the coefficient Hessian block.  Outputs per node, on the
 * host: the node log-evidence term (evidence.py:403-410), a status (0 ok,
 * 1 optimiser did not converge, 2 Cholesky failed, 3 objective not finite at
 * the start) and the L-BFGS iteration count.  The caller validates the model
 * (both Gaussian-kernel hypers sampled, others pinned) and combines the nodes
 * (skip tolerance, log-sum-exp).  Models on the large-d path are rejected. */
typedef struct {
    double c_max, c_mesh, sigma_max, sigma_mesh;
    int n_pinned;
    int pinned_pos[3];       /* sampled coordinates of pinned hypers */
    double pinned_value[3];  /* their sampled-coordinate values (ln value for the log transform) */
    double gtol;
    int max_iters, memory;
    int mode;                /* SGP_GRID_REFERENCE (default) or SGP_GRID_ROBUST */
} sgp_grid_spec;
/* SGP_GRID_REFERENCE: node k is (re)started from the optimum of the last node before it in
 * serpentine order whose L-BFGS converged -- the reference's a_warm rule -- so the failure
 * count (and the skip-tolerance RuntimeError) follows the reference.  SGP_GRID_ROBUST: nodes
 * start from a = 0 and failures are retried warm-started; fewer failures than the reference
 * (opt-in, documented as a deviation). */
#define SGP_GRID_REFERENCE 0
#define SGP_GRID_ROBUST 1
int sgp_laplace_grid(const sgp_model *model, const sgp_grid_spec *spec, int n_nodes, double *h_values,
                     int *h_status, int *h_iters, void *stream);

/* laplace_full (replaces evidence.py:277-304): L-BFGS mode search over all d
 * coordinates from h_q0 (tempered posterior, tau), Hessian at the mode and its
 * eigenvalues by the cold cyclic Jacobi (zeta, sweep_cap as
 * static_eigendecompose).  h_out4 = {ln evidence, U(q*), ln det H, min
 * eigenvalue}; *h_status 0 ok, 1 mode search did not reach gtol, 2 not positive
 * definite, 3 objective not finite at the start, 4 Jacobi sweep cap. */
int sgp_laplace_full(const sgp_model *model, double tau, const double *h_q0, double gtol, int max_iters,
                     double zeta, int sweep_cap, double *h_out4, int *h_status, int *h_iters, void *stream);

/* Diagnostics: cycles spent by chain 0 in each leapfrog phase (clock64), 16
 * slots: 0 W formation, 1 trace contraction, 2 state + Hessian, 3 MGS,
 * 4 Psi^T H Psi, 5 warm Jacobi, 8 cold Jacobi, 9 whole leapfrog. */
int sgp_debug_phase_cycles(unsigned long long *h_out16, int reset);

/* Self-check of the branch-free fp64 div/sqrt/rcp fast paths the cyclic
 * Jacobi uses (sgp_core.cuh) against the CUDA library calls on n random
 * samples: h_counts4 = {rotation (c,s,t) bitwise mismatches on the fast path,
 * rotations sent to the library path, primitive mismatches on random bit
 * patterns, n}.  Both mismatch counts must be 0. */
int sgp_debug_rotation_check(long long n, unsigned long long seed, long long *h_counts4);

/* Device properties the host reports (SM count, name) and library version. */
int sgp_device_info(int *sm_count, int *cc_major, int *cc_minor);
const char *sgp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SGP_H */
