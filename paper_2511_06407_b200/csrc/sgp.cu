// sgp.cu — kernels and the C ABI of libsgp.so (see include/sgp.h).
//
// Every batched entry point launches one CTA of SGP_NT threads per chain;
// the CTA runs the collective building blocks of sgp_core/sgp_eval/sgp_chain.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "sgp_chain.cuh"
#include "sgp_large.cuh"

extern __shared__ __align__(16) char sgp_smem[];

#include "sgp_grid.cuh"

struct sgp_model {
    ModelDev dev;
    double *d_phi, *d_phis, *d_y, *d_cw, *d_prec, *d_mean;
    int8_t *d_ckind;
    // large-d path workspace (allocated on first use)
    void *lg_owner;
    LgPtrs lg;
};

static const LgPtrs *large_ws(const sgp_model *mc) {
    sgp_model *m = const_cast<sgp_model *>(mc);
    if (!m->lg_owner && lg_alloc(m->dev, m->lg, &m->lg_owner) != SGP_OK) return nullptr;
    return &m->lg;
}

#define CUDA_TRY(x)                                                                  \
    do {                                                                             \
        cudaError_t err__ = (x);                                                     \
        if (err__ != cudaSuccess) {                                                  \
            fprintf(stderr, "libsgp: %s failed: %s\n", #x, cudaGetErrorString(err__)); \
            return SGP_ECUDA;                                                        \
        }                                                                            \
    } while (0)

static inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename K>
static int launch_prep(K kernel, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            fprintf(stderr, "libsgp: smem attribute (%zu B): %s\n", smem, cudaGetErrorString(e));
            return SGP_ECUDA;
        }
    }
    return SGP_OK;
}

static int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "libsgp: launch failed: %s\n", cudaGetErrorString(e));
        return SGP_ECUDA;
    }
    return SGP_OK;
}

// ===========================================================================
// model: design matrix assembly (FeatureCache, rrgp.py:310-344)

struct FeatRow {
    int kind;  // 0 sin basis, 1 linear, 2 ones
    int cov;
    double m, L;
};

__global__ void k_assemble_phi(const double *__restrict__ x, int N, int P, int ld, const FeatRow *__restrict__ rows,
                               int Dtot, double *__restrict__ phi) {
    const int a = blockIdx.y;
    const FeatRow r = rows[a];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (i < N) {
            if (r.kind == 0) {
                const double xv = x[(size_t)i * P + r.cov];
                v = sin(SGP_PI * r.m * (xv + r.L) / (2.0 * r.L));
            } else if (r.kind == 1) {
                v = x[(size_t)i * P + r.cov];
            } else {
                v = 1.0;
            }
        }
        phi[(size_t)a * ld + i] = v;
    }
}

// sample-major, function-padded copy used by the tiled contractions
__global__ void k_pad_phi(const double *__restrict__ phi, ModelParams mp, double *__restrict__ phis) {
    const int total = mp.ld * mp.Dp;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int i = idx / mp.Dp, a = idx - i * mp.Dp;
        int c;
        if (a < mp.Dp0)
            c = a < mp.D[0] ? a : -1;
        else
            c = a - mp.Dp0 < mp.D[1] ? mp.D[0] + a - mp.Dp0 : -1;
        phis[idx] = (c >= 0 && i < mp.N) ? phi[(size_t)c * mp.ld + i] : 0.0;
    }
}

extern "C" int sgp_model_create(const sgp_model_desc *desc, sgp_model **out) {
    if (!desc || !out) return SGP_EINVAL;
    *out = nullptr;
    sgp_model *m = (sgp_model *)calloc(1, sizeof(sgp_model));
    if (!m) return SGP_ENOMEM;
    ModelParams &mp = m->dev.mp;
    mp.lik = desc->likelihood;
    mp.transform = desc->transform;
    mp.sigma = desc->intercept_variance;
    mp.vfloor = desc->variance_floor;
    mp.loglik_const = desc->loglik_const;
    for (int s = 0; s < 3; ++s) {
        mp.hpos[s] = -1;
        mp.hfixed[s] = desc->hyper_fixed[s];
        mp.alpha[s] = desc->prior_alpha[s];
        mp.beta[s] = desc->prior_beta[s];
        mp.norm[s] = desc->hyper_sampled[s] ? lgamma(mp.alpha[s]) - mp.alpha[s] * log(mp.beta[s]) : 0.0;
    }
    if (mp.lik == SGP_LIK_QUADRATIC) {
        const int d = desc->quad_dim;
        if (d < 1 || !desc->h_precision || !desc->h_mean) {
            free(m);
            return SGP_EINVAL;
        }
        mp.d = d;
        mp.J = 0;
        mp.N = 0;
        mp.ld = 0;
        mp.Dtot = 0;
        CUDA_TRY(cudaMalloc(&m->d_prec, sizeof(double) * d * d));
        CUDA_TRY(cudaMalloc(&m->d_mean, sizeof(double) * d));
        CUDA_TRY(cudaMemcpy(m->d_prec, desc->h_precision, sizeof(double) * d * d, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(m->d_mean, desc->h_mean, sizeof(double) * d, cudaMemcpyHostToDevice));
        std::vector<int8_t> ck(d, CK_HYPER);
        CUDA_TRY(cudaMalloc(&m->d_ckind, d));
        CUDA_TRY(cudaMemcpy(m->d_ckind, ck.data(), d, cudaMemcpyHostToDevice));
        m->dev.prec = m->d_prec;
        m->dev.mean = m->d_mean;
        m->dev.ckind = m->d_ckind;
        *out = m;
        return SGP_OK;
    }
    const int J = desc->n_functions;
    if (J < 1 || J > 2 || desc->n_rows < 1 || desc->n_cols < 1) {
        free(m);
        return SGP_EINVAL;
    }
    mp.J = J;
    mp.N = desc->n_rows;
    mp.ld = (mp.N + 31) & ~31;
    std::vector<FeatRow> rows;
    std::vector<int8_t> ck;
    std::vector<double> cw;
    int pos = 0;
    for (int j = 0; j < J; ++j) {
        mp.fstart[j] = pos;
        for (int k = 0; k < desc->n_kernels[j]; ++k) {
            const sgp_kernel_desc &kd = desc->kernels[j][k];
            if (kd.covariate < 0 || kd.covariate >= desc->n_cols) {
                free(m);
                return SGP_EINVAL;
            }
            if (kd.kind == SGP_KERNEL_GAUSSIAN) {
                for (int mm = 1; mm <= kd.features; ++mm) {
                    rows.push_back({0, kd.covariate, (double)mm, kd.half_width});
                    ck.push_back(CK_GAUSS);
                    const double t = SGP_PI * (double)mm / (2.0 * kd.half_width);
                    cw.push_back(t * t / 4.0);
                    mp.n_gauss++;
                }
            } else {
                rows.push_back({1, kd.covariate, 0.0, 0.0});
                ck.push_back(CK_LIN);
                cw.push_back(0.0);
                mp.n_lin++;
            }
            pos += (kd.kind == SGP_KERNEL_GAUSSIAN) ? kd.features : 1;
        }
        rows.push_back({2, 0, 0.0, 0.0});
        ck.push_back(CK_INTERCEPT);
        cw.push_back(0.0);
        ++pos;
        mp.D[j] = pos - mp.fstart[j];
    }
    if (J == 1) {
        mp.D[1] = 0;
        mp.fstart[1] = pos;
    }
    mp.Dtot = pos;
    mp.Dp0 = (mp.D[0] + 3) & ~3;
    mp.Dp1 = (mp.D[1] + 3) & ~3;
    mp.Dp = mp.Dp0 + mp.Dp1;
    for (int s = 0; s < 3; ++s) {
        if (desc->hyper_sampled[s]) {
            mp.hpos[s] = pos++;
            ck.push_back(CK_HYPER);
            cw.push_back(0.0);
        }
    }
    mp.d = pos;
    const int Dt = mp.Dtot, N = mp.N, P = desc->n_cols, ld = mp.ld;
    double *d_x = nullptr;
    FeatRow *d_rows = nullptr;
    CUDA_TRY(cudaMalloc(&d_x, sizeof(double) * (size_t)N * P));
    CUDA_TRY(cudaMalloc(&d_rows, sizeof(FeatRow) * Dt));
    CUDA_TRY(cudaMalloc(&m->d_phi, sizeof(double) * (size_t)Dt * ld));
    CUDA_TRY(cudaMalloc(&m->d_y, sizeof(double) * ld));
    CUDA_TRY(cudaMalloc(&m->d_ckind, mp.d));
    CUDA_TRY(cudaMalloc(&m->d_cw, sizeof(double) * mp.d));
    CUDA_TRY(cudaMemcpy(d_x, desc->h_x, sizeof(double) * (size_t)N * P, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(d_rows, rows.data(), sizeof(FeatRow) * Dt, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(m->d_y, 0, sizeof(double) * ld));
    CUDA_TRY(cudaMemcpy(m->d_y, desc->h_y, sizeof(double) * N, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(m->d_ckind, ck.data(), mp.d, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(m->d_cw, cw.data(), sizeof(double) * mp.d, cudaMemcpyHostToDevice));
    dim3 grid((ld + 255) / 256, Dt);
    k_assemble_phi<<<grid, 256>>>(d_x, N, P, ld, d_rows, Dt, m->d_phi);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMalloc(&m->d_phis, sizeof(double) * (size_t)ld * mp.Dp));
    k_pad_phi<<<(ld * mp.Dp + 255) / 256, 256>>>(m->d_phi, mp, m->d_phis);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(d_x);
    cudaFree(d_rows);
    m->dev.phi = m->d_phi;
    m->dev.phis = m->d_phis;
    m->dev.y = m->d_y;
    m->dev.ckind = m->d_ckind;
    m->dev.cw = m->d_cw;
    *out = m;
    return SGP_OK;
}

extern "C" int sgp_model_destroy(sgp_model *m) {
    if (!m) return SGP_OK;
    cudaFree(m->d_phi);
    cudaFree(m->d_phis);
    if (m->lg_owner) {
        lg_free_handles(m->lg);
        cudaFree(m->lg_owner);
    }
    cudaFree(m->d_y);
    cudaFree(m->d_cw);
    cudaFree(m->d_ckind);
    cudaFree(m->d_prec);
    cudaFree(m->d_mean);
    free(m);
    return SGP_OK;
}

extern "C" int sgp_model_dim(const sgp_model *m) { return m ? m->dev.mp.d : SGP_EINVAL; }
extern "C" int sgp_model_rows(const sgp_model *m) { return m ? m->dev.mp.N : SGP_EINVAL; }
extern "C" int sgp_model_features(const sgp_model *m, int j) {
    if (!m || j < 0 || j >= m->dev.mp.J) return SGP_EINVAL;
    return m->dev.mp.D[j];
}
extern "C" size_t sgp_scratch_doubles(const sgp_model *m) {
    if (!m) return 0;
    if (lg_is_large(m->dev)) return 64;  // the large path keeps its state in the model workspace
    return sgp_scratch_per_chain(m->dev.mp.ld, m->dev.mp.d, m->dev.mp.Dp, sgp_fields(m->dev.mp));
}

__global__ void k_phi_out(const double *phi, int ld, int N, int a0, int Dj, double *out) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < N * Dj; idx += gridDim.x * blockDim.x) {
        const int i = idx / Dj, a = idx - i * Dj;
        out[idx] = phi[(size_t)(a0 + a) * ld + i];
    }
}

extern "C" int sgp_model_phi(const sgp_model *m, int j, double *d_out, void *stream) {
    if (!m || j < 0 || j >= m->dev.mp.J || !d_out) return SGP_EINVAL;
    const ModelParams &mp = m->dev.mp;
    const int a0 = j == 0 ? 0 : mp.D[0];
    const int n = mp.N * mp.D[j];
    k_phi_out<<<(n + 255) / 256, 256, 0, S(stream)>>>(m->dev.phi, mp.ld, mp.N, a0, mp.D[j], d_out);
    return check_launch();
}

// ===========================================================================
// posterior evaluation

__global__ void __launch_bounds__(SGP_MAX_NT) k_eval(ModelDev M, SmemPlan pl, const double *tau, const double *q, int what,
                                                 double *pot, double *grad, double *hess, double *sumpot, int *status,
                                                 double *scratch, size_t spc) {
    const int z = blockIdx.x;
    const int d = M.mp.d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, scratch + (size_t)z * spc);
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.q0[j] = q[(size_t)z * d + j];
    __syncthreads();
    double *H = hess ? hess + (size_t)z * d * d : w.H;
    EvalOut o;
    eval_state(E, w.q0, tau[z], what, w.grad, H, o);
    if (grad)
        for (int j = threadIdx.x; j < d; j += SGP_NT) grad[(size_t)z * d + j] = w.grad[j];
    if (threadIdx.x == 0) {
        if (pot) pot[z] = o.pot;
        if (sumpot) sumpot[z] = o.sumpot;
        status[z] = *E.status;
    }
}

static SmemPlan plan_for(const sgp_model *m, int allow_mats) {
    return sgp_smem_plan(m->dev.mp.d, m->dev.mp.Dp, SGP_MAX_NT, allow_mats ? 200 * 1024 : 16 * 1024);
}

// Launch shape of the fused chain kernel: threads per CTA and the number of
// CTAs (chains) meant to share an SM.  Small models run 64-thread CTAs, eight
// per SM, with their d x d matrices in L2-resident scratch: the reference-order
// Jacobi is a serial ~500-cycle-per-rotation chain, so throughput comes from
// overlapping many chains per SM.  SGP_CHAIN_THREADS=64|128|256 overrides.
struct ChainLaunch {
    int nt, per_sm;
    SmemPlan pl;
};
static ChainLaunch chain_launch(const sgp_model *m, const sgp_chain_config *cfg = nullptr) {
    int nt = m->dev.mp.d <= 64 ? 64 : 256;
    // path="latency" at small d: one wide CTA per chain (few chains, each alone on an SM)
    if (cfg && cfg->path == SGP_PATH_LATENCY) nt = 256;
    const char *env = getenv("SGP_CHAIN_THREADS");
    if (env) {
        int v = atoi(env);
        if (v == 32 || v == 64 || v == 128 || v == 256) nt = v;
    }
    ChainLaunch L;
    L.nt = nt;
    // 64-thread CTAs: four per SM.  Six fit the registers, but at four the larger shared-memory
    // budget keeps more of each chain's matrices on chip: same C2 throughput, DRAM traffic
    // 42 -> 9.8 GB per bench launch (profiles/r2_traffic_k_run_moves.json)
    L.per_sm = nt == 32 ? 12 : (nt == 64 ? 4 : (nt == 128 ? 4 : 2));
    const char *eps = getenv("SGP_CHAINS_PER_SM");
    if (eps && atoi(eps) > 0) L.per_sm = atoi(eps);
    const char *ech = getenv("SGP_STAGE_CH");
    const int ch = ech ? atoi(ech) : 0;
    const size_t budget = (227 * 1024) / L.per_sm - 1024;
    L.pl = sgp_smem_plan(m->dev.mp.d, m->dev.mp.Dp, nt, budget, (ch == 8 || ch == 16 || ch == 32 || ch == 64) ? ch : 0);
    return L;
}

extern "C" int sgp_eval(const sgp_model *m, int Z, const double *d_tau, const double *d_q, int what, double *d_pot,
                        double *d_grad, double *d_hess, double *d_sumpot, int *d_status, double *d_scratch,
                        void *stream) {
    if (!m || Z < 1 || !d_tau || !d_q || !d_status || !d_scratch) return SGP_EINVAL;
    if ((what & SGP_EVAL_GRADIENT) && !d_grad) return SGP_EINVAL;
    if ((what & SGP_EVAL_HESSIAN) && !d_hess) return SGP_EINVAL;
    if (lg_is_large(m->dev)) {
        const LgPtrs *L = large_ws(m);
        if (!L) return SGP_ENOMEM;
        return lg_eval_api(*L, Z, d_tau, d_q, what & 15, d_pot, d_grad, d_hess, d_sumpot, d_status, S(stream));
    }
    SmemPlan pl = plan_for(m, 0);
    int rc = launch_prep(k_eval, pl.bytes);
    if (rc) return rc;
    k_eval<<<Z, SGP_MAX_NT, pl.bytes, S(stream)>>>(m->dev, pl, d_tau, d_q, what & 15, d_pot, d_grad, d_hess, d_sumpot,
                                                 d_status, d_scratch, sgp_scratch_doubles(m));
    return check_launch();
}

__global__ void __launch_bounds__(SGP_MAX_NT) k_trace(ModelDev M, SmemPlan pl, const double *tau, const double *q,
                                                  const double *Win, double *tout, int *status, double *scratch,
                                                  size_t spc) {
    const int z = blockIdx.x;
    const int d = M.mp.d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, scratch + (size_t)z * spc);
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.q0[j] = q[(size_t)z * d + j];
    const double *Wz = Win + (size_t)z * d * d;
    for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) {
        const int i = idx / d, k = idx - i * d;
        w.W[idx] = 0.5 * (Wz[idx] + Wz[k * d + i]);
    }
    __syncthreads();
    EvalOut o;
    eval_state(E, w.q0, tau[z], 0, w.grad, w.H, o);
    if (*E.status == 0) eval_trace(E, w.q0, tau[z], w.W, w.tv);
    for (int j = threadIdx.x; j < d; j += SGP_NT) tout[(size_t)z * d + j] = w.tv[j];
    if (threadIdx.x == 0) status[z] = *E.status;
}

extern "C" int sgp_trace(const sgp_model *m, int Z, const double *d_tau, const double *d_q, const double *d_w,
                         double *d_t, int *d_status, double *d_scratch, void *stream) {
    if (!m || Z < 1 || !d_tau || !d_q || !d_w || !d_t || !d_status || !d_scratch) return SGP_EINVAL;
    if (lg_is_large(m->dev)) {
        const LgPtrs *L = large_ws(m);
        if (!L) return SGP_ENOMEM;
        return lg_trace_api(*L, Z, d_tau, d_q, d_w, d_t, d_status, S(stream));
    }
    SmemPlan pl = plan_for(m, 0);
    int rc = launch_prep(k_trace, pl.bytes);
    if (rc) return rc;
    k_trace<<<Z, SGP_MAX_NT, pl.bytes, S(stream)>>>(m->dev, pl, d_tau, d_q, d_w, d_t, d_status, d_scratch,
                                                  sgp_scratch_doubles(m));
    return check_launch();
}

__global__ void k_potential_derivatives(int lik, int n, int J, const double *f, const double *y, double vfloor,
                                        double *u, double *d1, double *d2, double *d3) {
    double S[F_COUNT];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double f0 = f[(size_t)i * J], f1 = J == 2 ? f[(size_t)i * J + 1] : 0.0;
        lik_sample(lik, vfloor, y[i], f0, f1, S, 1, 0);
        u[i] = S[F_U];
        if (J == 1) {
            d1[i] = S[F_D1_0];
            d2[i] = S[F_D2_00];
            d3[i] = S[F_D3_000];
        } else {
            d1[2 * i] = S[F_D1_0];
            d1[2 * i + 1] = S[F_D1_1];
            double *h = d2 + 4 * (size_t)i;
            h[0] = S[F_D2_00];
            h[1] = h[2] = S[F_D2_01];
            h[3] = S[F_D2_11];
            double *t = d3 + 8 * (size_t)i;
            t[0] = S[F_D3_000];
            t[1] = t[2] = t[4] = S[F_D3_001];
            t[3] = t[5] = t[6] = S[F_D3_011];
            t[7] = S[F_D3_111];
        }
    }
}

extern "C" int sgp_potential_derivatives(int lik, int n, int J, const double *d_f, const double *d_y,
                                         double variance_floor, double *d_u, double *d_d1, double *d_d2,
                                         double *d_d3, void *stream) {
    if (n < 1 || !d_f || !d_y || !d_u || !d_d1 || !d_d2 || !d_d3) return SGP_EINVAL;
    if (!((lik == SGP_LIK_LOGISTIC && J == 1) || (lik == SGP_LIK_GAUSSIAN_MEANVAR && J == 2))) return SGP_EINVAL;
    k_potential_derivatives<<<(n + 255) / 256, 256, 0, S(stream)>>>(lik, n, J, d_f, d_y, variance_floor, d_u, d_d1,
                                                                    d_d2, d_d3);
    return check_launch();
}

// ===========================================================================
// eigensolvers

__global__ void __launch_bounds__(SGP_MAX_NT) k_eigh_cold(int d, const double *Hin, double zeta, int cap, double *lam,
                                                      double *psi, int *sweeps, double *tmp) {
    __shared__ double red[64];
    const int z = blockIdx.x;
    const size_t dd = (size_t)d * d;
    double *A = tmp + z * dd;
    double *V = psi + z * dd;
    const double *H = Hin + z * dd;
    for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) {
        const int i = idx / d, k = idx - i * d;
        A[idx] = (i == k) ? H[idx] : 0.5 * (H[idx] + H[k * d + i]);
        V[idx] = (i == k) ? 1.0 : 0.0;
    }
    __syncthreads();
    const double hnorm = sqrt(frob2(A, d * d, red));
    const double tol = zeta * hnorm;
    const double skip = d ? tol / d : 0.0;
    int sw = jacobi_cyclic(A, V, d, tol, skip, cap, red, tmp + gridDim.x * dd + z * sgp_jacobi_log_doubles(d));
    for (int j = threadIdx.x; j < d; j += SGP_NT) lam[(size_t)z * d + j] = A[j * d + j];
    if (threadIdx.x == 0) sweeps[z] = sw;
}

// d at and above which cold decompositions use the grid-wide reference-order Jacobi
// (sgp_jbig.cuh) instead of one CTA per matrix; SGP_JBIG_MIN_D overrides (tests)
static int jbig_min_d() {
    const char *e = getenv("SGP_JBIG_MIN_D");
    return e ? atoi(e) : 257;
}

__global__ void k_sym_eye(const double *H, double *A, double *V, int d) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / d), k = (int)(idx - (size_t)i * d);
        A[idx] = (i == k) ? H[idx] : 0.5 * (H[idx] + H[(size_t)k * d + i]);
        V[idx] = (i == k) ? 1.0 : 0.0;
    }
}
__global__ void k_frob_part(const double *A, size_t n, double *part) {
    __shared__ double red[32];
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += A[i] * A[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
__global__ void k_copy_diag(const double *A, int d, double *lam) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) lam[i] = A[(size_t)i * d + i];
}

// Cold decomposition of one large matrix through sgp_jbig.cuh (metric.py:112-127)
static int eigh_cold_big(int Z, int d, const double *d_h, double zeta, int cap, double *d_lam, double *d_psi,
                         int *d_sweeps, cudaStream_t s) {
    const size_t dd = (size_t)d * d;
    double *A = nullptr, *part = nullptr;
    CUDA_TRY(cudaMalloc(&A, sizeof(double) * dd));
    CUDA_TRY(cudaMalloc(&part, sizeof(double) * 148));
    JbWS w;
    int rc = SGP_OK;
    std::vector<int> sw(Z);
    for (int z = 0; z < Z && rc == SGP_OK; ++z) {
        k_sym_eye<<<148 * 4, 256, 0, s>>>(d_h + z * dd, A, d_psi + z * dd, d);
        k_frob_part<<<148, 256, 0, s>>>(A, dd, part);
        std::vector<double> hp(148);
        cudaMemcpyAsync(hp.data(), part, sizeof(double) * 148, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) {
            rc = SGP_ECUDA;
            break;
        }
        double t = 0.0;
        for (double v : hp) t += v;
        const double tol = zeta * sqrt(t), skip = tol / d;
        const int r = jb_jacobi(w, A, d_psi + z * dd, d, tol, skip, cap, s);
        if (r == -2) rc = SGP_ECUDA;
        sw[z] = r < 0 ? -1 : r;
        k_copy_diag<<<8, 256, 0, s>>>(A, d, d_lam + (size_t)z * d);
    }
    if (rc == SGP_OK) cudaMemcpyAsync(d_sweeps, sw.data(), sizeof(int) * Z, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    jb_ws_free(w);
    cudaFree(A);
    cudaFree(part);
    return rc;
}

extern "C" int sgp_eigh_dc(int Z, int d, const double *d_h, double *d_lam, double *d_psi, void *stream) {
    if (Z < 1 || d < 1 || d > DC_NMAX || !d_h || !d_lam || !d_psi) return SGP_EINVAL;
    // one workspace per host thread and device, kept between calls (re-allocated when d changes)
    struct Cache {
        DcWS w[16];
        ~Cache() {
            for (DcWS &x : w) dc_ws_free(x);
        }
    };
    static thread_local Cache cache;
    int dev = 0;
    cudaGetDevice(&dev);
    DcWS &w = cache.w[dev & 15];
    int rc = SGP_OK;
    const size_t dd = (size_t)d * d;
    for (int z = 0; z < Z && rc == SGP_OK; ++z)
        if (dc_eigh(w, d_h + z * dd, d, d, d_lam + (size_t)z * d, d_psi + z * dd, d, S(stream))) rc = SGP_ECUDA;
    if (cudaStreamSynchronize(S(stream)) != cudaSuccess) rc = SGP_ECUDA;
    return rc;
}

extern "C" int sgp_eigh_cold(int Z, int d, const double *d_h, double zeta, int cap, double *d_lam, double *d_psi,
                             int *d_sweeps, void *stream) {
    if (Z < 1 || d < 1 || !d_h || !d_lam || !d_psi || !d_sweeps) return SGP_EINVAL;
    if (d >= jbig_min_d() && d >= 2) return eigh_cold_big(Z, d, d_h, zeta, cap, d_lam, d_psi, d_sweeps, S(stream));
    double *tmp = nullptr;
    CUDA_TRY(cudaMallocAsync(&tmp, sizeof(double) * Z * ((size_t)d * d + sgp_jacobi_log_doubles(d)), S(stream)));
    k_eigh_cold<<<Z, SGP_MAX_NT, 0, S(stream)>>>(d, d_h, zeta, cap, d_lam, d_psi, d_sweeps, tmp);
    int rc = check_launch();
    cudaFreeAsync(tmp, S(stream));
    return rc;
}

__global__ void __launch_bounds__(SGP_MAX_NT) k_eigh_warm(int d, const double *Hin, const double *psi_prev,
                                                      const int *since_prev, int gs, double zeta, int cap, int order,
                                                      double *lam, double *psi, int *since_out, int *sweeps,
                                                      double *tmp) {
    __shared__ double red[64];
    extern __shared__ __align__(16) char dyn[];
    double *prm = reinterpret_cast<double *>(dyn);
    const int z = blockIdx.x;
    const size_t dd = (size_t)d * d;
    double *A = tmp + 2 * z * dd, *X = A + dd;
    double *V = psi + z * dd;
    const double *H = Hin + z * dd;
    for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) V[idx] = psi_prev[z * dd + idx];
    __syncthreads();
    int since = since_prev[z] + 1;
    if (gs && since >= gs) {
        mgs(V, d, red);
        since = 0;
    }
    const double hnorm = sqrt(frob2(H, d * d, red));
    mat_mul<2>(X, V, H, d);
    mat_mul<0>(A, X, V, d);
    mat_symmetrize(A, d);
    const double tol = zeta * hnorm;
    const double skip = d ? tol / d : 0.0;
    int sw = order == SGP_ORDER_CYCLIC
                 ? jacobi_cyclic(A, V, d, tol, skip, cap, red, tmp + 2 * gridDim.x * dd + z * sgp_jacobi_log_doubles(d))
                                       : jacobi_parallel(A, V, d, tol, skip, cap, red, prm);
    for (int j = threadIdx.x; j < d; j += SGP_NT) lam[(size_t)z * d + j] = A[j * d + j];
    if (threadIdx.x == 0) {
        sweeps[z] = sw;
        since_out[z] = since;
    }
}

extern "C" int sgp_eigh_warm(int Z, int d, const double *d_h, const double *d_psi_prev, const int *d_since_prev,
                             int gs_interval, double zeta, int cap, int order, double *d_lam, double *d_psi,
                             int *d_since, int *d_sweeps, void *stream) {
    if (Z < 1 || d < 1 || !d_h || !d_psi_prev || !d_since_prev || !d_lam || !d_psi || !d_since || !d_sweeps)
        return SGP_EINVAL;
    double *tmp = nullptr;
    CUDA_TRY(cudaMallocAsync(&tmp, sizeof(double) * Z * (2 * (size_t)d * d + sgp_jacobi_log_doubles(d)), S(stream)));
    size_t smem = (6 * (size_t)((d + 2) / 2) + 8) * sizeof(double);
    int rc = launch_prep(k_eigh_warm, smem);
    if (rc) return rc;
    k_eigh_warm<<<Z, SGP_MAX_NT, smem, S(stream)>>>(d, d_h, d_psi_prev, d_since_prev, gs_interval, zeta, cap, order,
                                                 d_lam, d_psi, d_since, d_sweeps, tmp);
    rc = check_launch();
    cudaFreeAsync(tmp, S(stream));
    return rc;
}

__global__ void __launch_bounds__(SGP_MAX_NT) k_mgs(int d, double *psi) {
    __shared__ double red[64];
    mgs(psi + (size_t)blockIdx.x * d * d, d, red);
}

extern "C" int sgp_mgs(int Z, int d, double *d_psi, void *stream) {
    if (Z < 1 || d < 1 || !d_psi) return SGP_EINVAL;
    k_mgs<<<Z, SGP_MAX_NT, 0, S(stream)>>>(d, d_psi);
    return check_launch();
}

// ===========================================================================
// metric algebra

__global__ void __launch_bounds__(SGP_MAX_NT) k_metric(int d, const double *psi, const double *lamv, double kappa,
                                                   const double *pin, int op, int which, double *out, double *out2,
                                                   double *tmp) {
    __shared__ double red[64];
    const int z = blockIdx.x;
    const size_t dd = (size_t)d * d;
    const double *P = psi + z * dd;
    const double *lam = lamv + (size_t)z * d;
    double *T = tmp + 3 * z * dd, *X = T + dd;
    double *g = X + dd, *b = g + d, *t2 = b + d;
    metric_g(lam, g, d, kappa, red);
    __syncthreads();
    const double *p = pin ? pin + (size_t)z * d : nullptr;
    if (op == 0) {  // T matrix
        t_matrix(out + z * dd, lam, g, d, kappa);
    } else if (op == 1) {  // W1 / W2 / W2 - W1
        const bool w1 = which & SGP_W_W1, w2 = which & SGP_W_W2;
        if (w1) t_matrix(T, lam, g, d, kappa);
        metric_w(out + z * dd, X, b, P, lam, g, T, p, d, w1, w2, w2 ? -1.0 : 1.0);
    } else if (op == 2) {  // apply
        metric_apply(out + (size_t)z * d, t2, P, g, p, d, which);
    } else {  // scalars: quad, logdet
        double ldv = 0.0;
        for (int j = threadIdx.x; j < d; j += SGP_NT) ldv += log(g[j]);
        ldv = block_sum(ldv, red);
        double qv = p ? metric_quad(t2, P, g, p, d, red) : 0.0;
        if (threadIdx.x == 0) {
            if (out) out[z] = qv;
            if (out2) out2[z] = ldv;
        }
    }
}

static int metric_launch(int Z, int d, const double *psi, const double *lam, double kappa, const double *p, int op,
                         int which, double *out, double *out2, void *stream) {
    double *tmp = nullptr;
    CUDA_TRY(cudaMallocAsync(&tmp, sizeof(double) * Z * (3 * (size_t)d * d), S(stream)));
    k_metric<<<Z, SGP_MAX_NT, 0, S(stream)>>>(d, psi, lam, kappa, p, op, which, out, out2, tmp);
    int rc = check_launch();
    cudaFreeAsync(tmp, S(stream));
    return rc;
}

extern "C" int sgp_t_matrix(int Z, int d, const double *d_lam, double kappa, double *d_t, void *stream) {
    if (Z < 1 || d < 1 || !d_lam || !d_t || !(kappa > 0.0)) return SGP_EINVAL;
    return metric_launch(Z, d, d_lam /*unused psi*/, d_lam, kappa, nullptr, 0, 0, d_t, nullptr, stream);
}

extern "C" int sgp_metric_w(int Z, int d, const double *d_psi, const double *d_lam, double kappa, const double *d_p,
                            int which, double *d_w, void *stream) {
    if (Z < 1 || d < 1 || !d_psi || !d_lam || !d_w || which < 1 || which > 3) return SGP_EINVAL;
    if ((which & SGP_W_W1) && !d_p) return SGP_EINVAL;
    return metric_launch(Z, d, d_psi, d_lam, kappa, d_p, 1, which, d_w, nullptr, stream);
}

extern "C" int sgp_metric_apply(int Z, int d, const double *d_psi, const double *d_lam, double kappa,
                                const double *d_v, int mode, double *d_out, void *stream) {
    if (Z < 1 || d < 1 || !d_psi || !d_lam || !d_v || !d_out || mode < 0 || mode > 2) return SGP_EINVAL;
    return metric_launch(Z, d, d_psi, d_lam, kappa, d_v, 2, mode, d_out, nullptr, stream);
}

extern "C" int sgp_metric_scalars(int Z, int d, const double *d_psi, const double *d_lam, double kappa,
                                  const double *d_p, double *d_quad, double *d_logdet, void *stream) {
    if (Z < 1 || d < 1 || !d_psi || !d_lam) return SGP_EINVAL;
    return metric_launch(Z, d, d_psi, d_lam, kappa, d_p, 3, 0, d_quad, d_logdet, stream);
}

// ===========================================================================
// integrator and chains

__global__ void __launch_bounds__(SGP_MAX_NT) k_leapfrog(ModelDev M, SmemPlan pl, sgp_chain_config cfg,
                                                     sgp_chain_state st, double *pio, sgp_leapfrog_diag dgo,
                                                     size_t spc) {
    const int z = blockIdx.x;
    const int d = M.mp.d;
    const size_t dd = (size_t)d * d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, st.scratch + (size_t)z * spc);
    const double tau = st.tau[z];
    for (int j = threadIdx.x; j < d; j += SGP_NT) {
        w.q0[j] = st.q[(size_t)z * d + j];
        w.p[j] = pio[(size_t)z * d + j];
    }
    __syncthreads();
    int f = 0;
    int s = frame_resume(w, E, cfg, tau, st.psi + z * dd, st.lam + (size_t)z * d, st.since[z], f);
    LFDiag dg;
    dg.fp_p = dg.fp_q = dg.nsweep = dg.sweep_cnt = 0;
    dg.sweep_sum = 0.0;
    __shared__ int sweep_log[32];
    dg.sweeps = sweep_log;
    if (!s) {
        if (cfg.metric == SGP_METRIC_EUCLIDEAN)
            s = leapfrog_euclid(w, E, cfg, tau);
        else
            s = leapfrog_riemann(w, E, cfg, tau, f, dg);
    }
    if (!s) {
        for (int j = threadIdx.x; j < d; j += SGP_NT) {
            st.q[(size_t)z * d + j] = w.q0[j];
            pio[(size_t)z * d + j] = w.p[j];
        }
        if (cfg.metric != SGP_METRIC_EUCLIDEAN) {
            for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) st.psi[z * dd + idx] = w.P[f][idx];
            for (int j = threadIdx.x; j < d; j += SGP_NT) st.lam[(size_t)z * d + j] = w.lam[f][j];
        }
    }
    if (threadIdx.x == 0) {
        st.status[z] = s;
        if (!s && cfg.metric != SGP_METRIC_EUCLIDEAN) st.since[z] = w.si[f];
        if (dgo.fp_p_iters) dgo.fp_p_iters[z] = dg.fp_p;
        if (dgo.fp_q_iters) dgo.fp_q_iters[z] = dg.fp_q;
        if (dgo.sweeps)
            for (int k = 0; k < cfg.fp_max_iters; ++k)
                dgo.sweeps[(size_t)z * cfg.fp_max_iters + k] = k < dg.nsweep && k < 32 ? dg.sweeps[k] : -1;
    }
}

static int chain_plan(const sgp_model *m, SmemPlan &pl) {
    pl = plan_for(m, 1);
    return SGP_OK;
}

extern "C" int sgp_leapfrog(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st, double *d_p,
                            sgp_leapfrog_diag *diag, void *stream) {
    if (!m || !cfg || !st || !d_p || st->n_chains < 1) return SGP_EINVAL;
    if (cfg->fp_max_iters < 1 || cfg->fp_max_iters > 32) return SGP_EINVAL;
    if (lg_is_large(m->dev) || lg_route_latency(m->dev, *cfg)) {
        const LgPtrs *L = large_ws(m);
        if (!L) return SGP_ENOMEM;
        return lg_leapfrog_api(*L, cfg, st, d_p, diag, S(stream));
    }
    SmemPlan pl;
    chain_plan(m, pl);
    int rc = launch_prep(k_leapfrog, pl.bytes);
    if (rc) return rc;
    sgp_leapfrog_diag dg = diag ? *diag : sgp_leapfrog_diag{nullptr, nullptr, nullptr};
    k_leapfrog<<<st->n_chains, SGP_MAX_NT, pl.bytes, S(stream)>>>(m->dev, pl, *cfg, *st, d_p, dg,
                                                                sgp_scratch_doubles(m));
    return check_launch();
}

__global__ void __launch_bounds__(SGP_MAX_NT) k_chain_init(ModelDev M, SmemPlan pl, sgp_chain_config cfg,
                                                       sgp_chain_state st, size_t spc) {
    const int z = blockIdx.x;
    const int d = M.mp.d;
    const size_t dd = (size_t)d * d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, st.scratch + (size_t)z * spc);
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.q0[j] = st.q[(size_t)z * d + j];
    __syncthreads();
    int f = 0;
    int s = frame_build(w, E, cfg, st.tau[z], f);
    if (!s && cfg.metric != SGP_METRIC_EUCLIDEAN) {
        for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) st.psi[z * dd + idx] = w.P[0][idx];
        for (int j = threadIdx.x; j < d; j += SGP_NT) st.lam[(size_t)z * d + j] = w.lam[0][j];
    }
    if (threadIdx.x == 0) {
        st.status[z] = s ? SGP_STATUS_CHAIN_START : 0;
        st.since[z] = 0;
    }
}

extern "C" int sgp_chain_init(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st,
                              void *stream) {
    if (!m || !cfg || !st || st->n_chains < 1) return SGP_EINVAL;
    if (lg_is_large(m->dev) || lg_route_latency(m->dev, *cfg)) {
        const LgPtrs *L = large_ws(m);
        if (!L) return SGP_ENOMEM;
        return lg_chain_init(*L, cfg, st, S(stream));
    }
    SmemPlan pl;
    chain_plan(m, pl);
    int rc = launch_prep(k_chain_init, pl.bytes);
    if (rc) return rc;
    k_chain_init<<<st->n_chains, SGP_MAX_NT, pl.bytes, S(stream)>>>(m->dev, pl, *cfg, *st, sgp_scratch_doubles(m));
    return check_launch();
}

// The MH move loop (sampler.py:355-411), C leapfrogs per move, all on device.
// n_rungs > 0: the whole thermodynamic-integration ladder walk of a chain in the same launch
// (evidence.py:142-163): for every rung s the chain's target moves to taus[s], the frame is
// rebuilt cold at the current position (each rung is a new run_chain: _initial_frame,
// sampler.py:322-328), `moves` moves run with the rung's draws (dz/dlogu indexed by rung), and
// values[z * n_rungs + s] = log_likelihood at the rung's end (posterior.py:277-279), or its
// average over the rung's moves when rung_average.  Per-move records are optional then.
// LADDER = false compiles the plain move loop without the rung machinery (its code shape
// otherwise costs the register-capped 256-thread instance ~11 %: C5 2437 vs 2708/s).
template <int NT, int MINB, bool LADDER>
__global__ void __launch_bounds__(NT, MINB) k_run_moves(ModelDev M, SmemPlan pl, sgp_chain_config cfg,
                                                      sgp_chain_state st, int moves, int move_offset,
                                                      const double *dz, const double *dlogu, sgp_move_records rec,
                                                      size_t spc, int n_rungs_arg, const double *taus,
                                                      int rung_average, double *values) {
    const int n_rungs = LADDER ? n_rungs_arg : 0;
    const int z = blockIdx.x;
    const int Z = st.n_chains;
    const int d = M.mp.d;
    const size_t dd = (size_t)d * d;
    ChainWS w;
    EvalCtx E;
    setup_ws(w, E, sgp_smem, pl, M, st.scratch + (size_t)z * spc);
    if (st.status[z] != 0) return;
    const bool euclid = cfg.metric == SGP_METRIC_EUCLIDEAN;
    for (int j = threadIdx.x; j < d; j += SGP_NT) w.q0[j] = st.q[(size_t)z * d + j];
    __syncthreads();
    int f = 0;
    if (n_rungs == 0) {
        int s = frame_resume(w, E, cfg, st.tau[z], st.psi + z * dd, st.lam + (size_t)z * d, st.since[z], f);
        if (s) {
            if (threadIdx.x == 0) st.status[z] = SGP_STATUS_CHAIN_START;
            return;
        }
    }
    int final_status = 0;
    const int rungs = n_rungs > 0 ? n_rungs : 1;
    for (int rg = 0; rg < rungs && !final_status; ++rg) {
        const double tau = n_rungs > 0 ? taus[rg] : st.tau[z];
        if (n_rungs > 0) {
            if (frame_build(w, E, cfg, tau, f)) {  // rung start: a cold frame (sampler.py:322-328)
                final_status = SGP_STATUS_CHAIN_START;
                break;
            }
        }
        double ll_sum = 0.0;
        const size_t moff = (size_t)rg * moves;
        // log_likelihood(q) = -sum_i U_i (posterior.py:277-279); the frame carries it except at
        // tau = 0, where the tempered state skips the likelihood: evaluate it separately then
        // (sum only; the trace ignores the per-sample fields at tau = 0) and keep the frame's U
        auto loglik = [&]() -> double {
            if (tau != 0.0) return -w.sc[3];
            const double pot = w.sc[2];
            eval_at(w, E, w.q0, tau, SGP_EVAL_SUMPOT);
            const double ll = -w.sc[3];
            __syncthreads();
            if (threadIdx.x == 0) {
                w.sc[2] = pot;
                *E.status = 0;
            }
            __syncthreads();
            return ll;
        };
        for (int mv = 0; mv < moves; ++mv) {
            const unsigned long long t0 = globaltimer_ns();
            const double *zz = dz + ((moff + mv) * Z + z) * d;
            if (euclid) {
                for (int j = threadIdx.x; j < d; j += SGP_NT) w.p[j] = zz[j];
                __syncthreads();
            } else {
                for (int j = threadIdx.x; j < d; j += SGP_NT) w.pn[j] = zz[j];
                __syncthreads();
                metric_apply(w.p, w.tmp, w.P[f], w.g[f], w.pn, d, 2);
            }
            const double pot_before = w.sc[2];
            const double h_before = pot_before + frame_kinetic(w, E, cfg, f);
            for (int j = threadIdx.x; j < d; j += SGP_NT) w.qs[j] = w.q0[j];
            __syncthreads();
            LFDiag dg;
            dg.fp_p = dg.fp_q = dg.nsweep = dg.sweep_cnt = 0;
            dg.sweep_sum = 0.0;
            dg.sweeps = nullptr;
            int fr = f;
            int ls = 0;
            for (int l = 0; l < cfg.leapfrogs; ++l) {
                ls = euclid ? leapfrog_euclid(w, E, cfg, tau) : leapfrog_riemann(w, E, cfg, tau, fr, dg);
                if (ls) break;
            }
            bool div = ls != 0;
            double h_after = NAN;
            if (!div) {
                h_after = w.sc[2] + frame_kinetic(w, E, cfg, fr);
                if (!isfinite(h_after)) div = true;
            }
            if (div) h_after = NAN;
            const bool accept = !div && (h_before - h_after) > dlogu[(moff + mv) * Z + z];
            __syncthreads();
            if (threadIdx.x == 0) *E.status = 0;
            __syncthreads();
            if (accept) {
                f = fr;
            } else {
                // a divergence on a run_chain's first move raises ChainError (sampler.py:388-391);
                // every rung of a ladder walk is its own run_chain
                if (div && (n_rungs > 0 ? mv : mv + move_offset) == 0) {
                    final_status = SGP_STATUS_FIRST_MOVE;
                } else {
                    for (int j = threadIdx.x; j < d; j += SGP_NT) w.q0[j] = w.qs[j];
                    __syncthreads();
                    int rs = frame_build(w, E, cfg, tau, f);  // cold resync (sampler.py:392-397)
                    if (rs) final_status = rs;
                }
            }
            if (n_rungs > 0 && rung_average && !final_status) ll_sum += loglik();  // at the recorded q
            const size_t ri = (moff + mv) * Z + z;
            if (threadIdx.x == 0 && rec.logpost) {
                rec.logpost[ri] = -w.sc[2];
                rec.h_before[ri] = h_before;
                rec.h_after[ri] = h_after;
                rec.accept[ri] = accept;
                rec.divergent[ri] = div;
                rec.sweeps_mean[ri] = dg.sweep_cnt ? dg.sweep_sum / dg.sweep_cnt : 0.0;
                rec.wall_ms[ri] = (double)(globaltimer_ns() - t0) * 1e-6;
            }
            if (rec.q)
                for (int j = threadIdx.x; j < d; j += SGP_NT) rec.q[ri * d + j] = (final_status ? w.qs[j] : w.q0[j]);
            if (final_status) break;
        }
        if (n_rungs > 0 && !final_status) {
            const double v = rung_average ? ll_sum / moves : loglik();
            if (threadIdx.x == 0) values[(size_t)z * n_rungs + rg] = v;
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += SGP_NT) st.q[(size_t)z * d + j] = w.q0[j];
    if (!euclid && !final_status) {
        for (int idx = threadIdx.x; idx < d * d; idx += SGP_NT) st.psi[z * dd + idx] = w.P[f][idx];
        for (int j = threadIdx.x; j < d; j += SGP_NT) st.lam[(size_t)z * d + j] = w.lam[f][j];
    }
    if (threadIdx.x == 0) {
        st.status[z] = final_status;
        if (!euclid && !final_status) st.since[z] = w.si[f];
    }
}

static int launch_moves(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st, int moves,
                        int move_offset, const double *d_z, const double *d_logu, const sgp_move_records *rec,
                        int n_rungs, const double *d_taus, int rung_average, double *d_values, void *stream);

extern "C" int sgp_run_moves(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st, int moves,
                             int move_offset, const double *d_z, const double *d_logu, sgp_move_records *rec,
                             void *stream) {
    if (!m || !cfg || !st || !rec || st->n_chains < 1 || moves < 0 || !d_z || !d_logu) return SGP_EINVAL;
    if (!rec->logpost || !rec->h_before || !rec->h_after || !rec->accept || !rec->divergent || !rec->sweeps_mean ||
        !rec->wall_ms)
        return SGP_EINVAL;
    return launch_moves(m, cfg, st, moves, move_offset, d_z, d_logu, rec, 0, nullptr, 0, nullptr, stream);
}

extern "C" int sgp_ladder_walk(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st,
                               int n_rungs, const double *d_taus, int moves_per_rung, int rung_average,
                               const double *d_z, const double *d_logu, double *d_values, void *stream) {
    if (!m || !cfg || !st || st->n_chains < 1 || n_rungs < 1 || moves_per_rung < 1 || !d_taus || !d_z || !d_logu ||
        !d_values)
        return SGP_EINVAL;
    if (lg_is_large(m->dev) || lg_route_latency(m->dev, *cfg)) return SGP_EINVAL;  // the caller walks rung by rung
    sgp_move_records none{};
    return launch_moves(m, cfg, st, moves_per_rung, 0, d_z, d_logu, &none, n_rungs, d_taus, rung_average, d_values,
                        stream);
}

static int launch_moves(const sgp_model *m, const sgp_chain_config *cfg, const sgp_chain_state *st, int moves,
                        int move_offset, const double *d_z, const double *d_logu, const sgp_move_records *rec,
                        int n_rungs, const double *d_taus, int rung_average, double *d_values, void *stream) {
    if (cfg->fp_max_iters < 1 || cfg->leapfrogs < 1) return SGP_EINVAL;
    if (moves == 0) return SGP_OK;
    if (lg_is_large(m->dev) || lg_route_latency(m->dev, *cfg)) {
        const LgPtrs *LW = large_ws(m);
        if (!LW) return SGP_ENOMEM;
        return lg_run_moves(*LW, cfg, st, moves, move_offset, d_z, d_logu, const_cast<sgp_move_records *>(rec),
                            S(stream));
    }
    const ChainLaunch L = chain_launch(m, cfg);
    const size_t spc = sgp_scratch_doubles(m);
    int rc;
#define SGP_LAUNCH_MOVES_L(NT_, MB_, LD_)                                                                   \
    rc = launch_prep(k_run_moves<NT_, MB_, LD_>, L.pl.bytes);                                              \
    if (rc) return rc;                                                                                      \
    k_run_moves<NT_, MB_, LD_><<<st->n_chains, NT_, L.pl.bytes, S(stream)>>>(                                \
        m->dev, L.pl, *cfg, *st, moves, move_offset, d_z, d_logu, *rec, spc, n_rungs, d_taus, rung_average, d_values)
#define SGP_LAUNCH_MOVES(NT_, MB_)              \
    if (n_rungs > 0) {                          \
        SGP_LAUNCH_MOVES_L(NT_, MB_, true);     \
    } else {                                    \
        SGP_LAUNCH_MOVES_L(NT_, MB_, false);    \
    }
    if (L.nt == 32) {
        SGP_LAUNCH_MOVES(32, 12);
    } else if (L.nt == 64) {
        if (L.per_sm >= 10) {
            SGP_LAUNCH_MOVES(64, 10);
        } else if (L.per_sm >= 8) {
            SGP_LAUNCH_MOVES(64, 8);
        } else {
            SGP_LAUNCH_MOVES(64, 6);
        }
    } else if (L.nt == 128) {
        SGP_LAUNCH_MOVES(128, 4);
    } else {
        SGP_LAUNCH_MOVES(256, 2);
    }
#undef SGP_LAUNCH_MOVES
#undef SGP_LAUNCH_MOVES_L
    return check_launch();
}

extern "C" int sgp_device_info(int *sm_count, int *cc_major, int *cc_minor) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    return SGP_OK;
}

extern "C" const char *sgp_version(void) { return "sgp 0.1.0 sm_100a"; }

extern "C" int sgp_debug_phase_cycles(unsigned long long *h_out16, int reset) {
    if (h_out16) CUDA_TRY(cudaMemcpyFromSymbol(h_out16, sgp_prof_cycles, sizeof(unsigned long long) * 16));
    if (reset) {
        unsigned long long z[16] = {0};
        CUDA_TRY(cudaMemcpyToSymbol(sgp_prof_cycles, z, sizeof(z)));
    }
    return SGP_OK;
}

// ---------------------------------------------------------------------------
// Self-check of the branch-free fast paths (sgp_core.cuh) against the library
// calls: counts[0] rotations whose (c, s, t) differ bitwise although the fast
// path reported success, counts[1] rotations routed to the library path,
// counts[2] div/sqrt/rcp results that differ on random bit patterns although
// the fast path reported success, counts[3] total samples.
__device__ __forceinline__ unsigned long long sgp_mix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double sgp_u01(unsigned long long x) { return (double)(x >> 11) * 0x1.0p-53; }

__global__ void k_rotation_check(long long n, unsigned long long seed, unsigned long long *cnt) {
    unsigned long long bad = 0, slow = 0, badop = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h0 = sgp_mix64(seed ^ (unsigned long long)i), h1 = sgp_mix64(h0), h2 = sgp_mix64(h1),
                                 h3 = sgp_mix64(h2), h4 = sgp_mix64(h3);
        // Jacobi-like operands: diagonal entries over 8 decades, pivots over 20
        double app = (sgp_u01(h0) < 0.5 ? -1.0 : 1.0) * exp10(8.0 * sgp_u01(h1) - 3.0);
        double aqq = (h2 & 1) ? app * (1.0 + 1e-9 * (sgp_u01(h2) - 0.5)) : (sgp_u01(h2) - 0.5) * exp10(8.0 * sgp_u01(h3) - 3.0);
        const double apq = ((h4 & 2) ? -1.0 : 1.0) * exp10(20.0 * sgp_u01(h4) - 16.0);
        if ((h0 & 0xff) == 7) aqq = app;  // theta = 0
        double c0, s0, t0, c1, s1, t1;
        jacobi_rot(app, aqq, apq, c0, s0, t0);
        if (jacobi_rot_fast(app, aqq, apq, c1, s1, t1)) {
            if (__double_as_longlong(c0) != __double_as_longlong(c1) || __double_as_longlong(s0) != __double_as_longlong(s1) ||
                __double_as_longlong(t0) != __double_as_longlong(t1))
                ++bad;
        } else {
            ++slow;
        }
        // raw bit patterns (any sign / exponent) for the three primitives
        const double a = __longlong_as_double((long long)h1), b = __longlong_as_double((long long)h3);
        bool ok = true;
        double v = ddiv_fast(a, b, ok);
        if (ok && __double_as_longlong(v) != __double_as_longlong(__ddiv_rn(a, b))) ++badop;
        const double x = fabs(a);
        ok = true;
        v = dsqrt_fast(x, ok);
        if (ok && __double_as_longlong(v) != __double_as_longlong(__dsqrt_rn(x))) ++badop;
        ok = true;
        v = drcp_fast(b, ok);
        if (ok && __double_as_longlong(v) != __double_as_longlong(__drcp_rn(b))) ++badop;
    }
    atomicAdd(&cnt[0], bad);
    atomicAdd(&cnt[1], slow);
    atomicAdd(&cnt[2], badop);
}

extern "C" int sgp_debug_rotation_check(long long n, unsigned long long seed, long long *h_counts4) {
    if (!h_counts4 || n < 0) return SGP_EINVAL;
    unsigned long long *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, 3 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(d, 0, 3 * sizeof(unsigned long long)));
    k_rotation_check<<<148 * 8, 256>>>(n, seed, d);
    unsigned long long h[3];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return SGP_ECUDA;
    h_counts4[0] = (long long)h[0];
    h_counts4[1] = (long long)h[1];
    h_counts4[2] = (long long)h[2];
    h_counts4[3] = n;
    return SGP_OK;
}

// ---------------------------------------------------------------------------
// Laplace-grid evidence oracle (evidence.py:330-426): per-node values on device.
extern "C" int sgp_laplace_grid(const sgp_model *m, const sgp_grid_spec *spec, int n_nodes, double *h_values,
                                int *h_status, int *h_iters, void *stream) {
    if (!m || !spec || !h_values || !h_status || n_nodes < 1) return SGP_EINVAL;
    const ModelParams &mp = m->dev.mp;
    if (lg_is_large(m->dev) || mp.hpos[0] < 0 || mp.hpos[1] < 0) return SGP_EINVAL;
    if (!(spec->c_mesh > 0.0) || !(spec->sigma_mesh > 0.0) || spec->memory < 1 || spec->max_iters < 0) return SGP_EINVAL;
    GridDev gd{};
    gd.nc = (int)std::lround(spec->c_max / spec->c_mesh);
    gd.ns = (int)std::lround(spec->sigma_max / spec->sigma_mesh);
    if (gd.nc * gd.ns != n_nodes || spec->n_pinned < 0 || spec->n_pinned > 3) return SGP_EINVAL;
    gd.c_mesh = spec->c_mesh;
    gd.s_mesh = spec->sigma_mesh;
    gd.n_pinned = spec->n_pinned;
    for (int k = 0; k < spec->n_pinned; ++k) {
        if (spec->pinned_pos[k] < 0 || spec->pinned_pos[k] >= mp.d) return SGP_EINVAL;
        gd.pin_pos[k] = spec->pinned_pos[k];
        gd.pin_q[k] = spec->pinned_value[k];
    }
    gd.gtol = spec->gtol;
    gd.max_iters = spec->max_iters;
    gd.memory = spec->memory;
    gd.log_area = std::log(spec->c_mesh) + std::log(spec->sigma_mesh);
    const ChainLaunch L = chain_launch(m);
    const size_t spc = sgp_scratch_doubles(m);
    const size_t stride = spc + sgp_grid_scratch_extra(mp.d, spec->memory);
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int batch = std::max(1, std::min(n_nodes, sms * L.per_sm * 2));
    double *d_scr = nullptr, *d_val = nullptr, *d_aopt = nullptr;
    int *d_st = nullptr, *d_it = nullptr, *d_list = nullptr;
    const size_t d = mp.d;
    if (cudaMalloc(&d_scr, stride * batch * sizeof(double)) != cudaSuccess) return SGP_ENOMEM;
    if (cudaMalloc(&d_val, n_nodes * sizeof(double)) != cudaSuccess || cudaMalloc(&d_st, n_nodes * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&d_it, n_nodes * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&d_aopt, (size_t)n_nodes * d * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&d_list, 2 * (size_t)n_nodes * sizeof(int)) != cudaSuccess) {
        cudaFree(d_scr);
        cudaFree(d_val);
        cudaFree(d_st);
        cudaFree(d_it);
        cudaFree(d_aopt);
        return SGP_ENOMEM;
    }
    int rc = launch_prep(k_laplace_grid, L.pl.bytes);
    // pass 1: every node from a = 0, concurrently
    for (int node0 = 0; !rc && node0 < n_nodes; node0 += batch) {
        const int nb = std::min(batch, n_nodes - node0);
        k_laplace_grid<<<nb, L.nt, L.pl.bytes, S(stream)>>>(m->dev, L.pl, gd, node0, n_nodes, d_scr, spc, stride,
                                                             d_val, d_st, d_it, nullptr, nullptr, nullptr, d_aopt);
        rc = check_launch();
    }
    std::vector<int> st(n_nodes), list, src;
    if (spec->mode == SGP_GRID_REFERENCE) {
        // The reference's rule (evidence.py:374-403): node k starts from a_warm, the optimum of
        // the last node before it in serpentine order whose L-BFGS converged (updated before the
        // Cholesky test), 0 until the first one.  Its chain is sequential; here every node is
        // re-run concurrently from the pass-1 optimum of that predecessor (the optimum a
        // converged L-BFGS reaches does not depend on its start beyond gtol), so failures are
        // counted for the reference's starting points and the skip tolerance keeps its meaning.
        double *d_a1 = nullptr;
        if (!rc && (cudaMemcpyAsync(st.data(), d_st, n_nodes * sizeof(int), cudaMemcpyDeviceToHost, S(stream)) !=
                        cudaSuccess ||
                    cudaStreamSynchronize(S(stream)) != cudaSuccess))
            rc = SGP_ECUDA;
        if (!rc && cudaMalloc(&d_a1, (size_t)n_nodes * d * sizeof(double)) != cudaSuccess) rc = SGP_ENOMEM;
        if (!rc) {
            cudaMemcpyAsync(d_a1, d_aopt, (size_t)n_nodes * d * sizeof(double), cudaMemcpyDeviceToDevice, S(stream));
            int last = -1;
            for (int k = 0; k < n_nodes; ++k) {
                if (last >= 0) {  // nodes with no converged predecessor start at 0: pass 1 already is theirs
                    list.push_back(k);
                    src.push_back(last);
                }
                if (st[k] == 0 || st[k] == 2) last = k;
            }
            const int nl = (int)list.size();
            if (nl) {
                cudaMemcpyAsync(d_list, list.data(), nl * sizeof(int), cudaMemcpyHostToDevice, S(stream));
                cudaMemcpyAsync(d_list + n_nodes, src.data(), nl * sizeof(int), cudaMemcpyHostToDevice, S(stream));
            }
            for (int node0 = 0; !rc && node0 < nl; node0 += batch) {
                const int nb = std::min(batch, nl - node0);
                k_laplace_grid<<<nb, L.nt, L.pl.bytes, S(stream)>>>(m->dev, L.pl, gd, node0, nl, d_scr, spc, stride,
                                                                     d_val, d_st, d_it, d_list, d_list + n_nodes, d_a1,
                                                                     d_aopt);
                rc = check_launch();
            }
            cudaStreamSynchronize(S(stream));
        }
        cudaFree(d_a1);
    }
    // SGP_GRID_ROBUST passes 2..: failed nodes again, warm-started from the optimum of the
    // last converged node before them in serpentine order (fewer failures than the reference)
    for (int pass = 0; !rc && spec->mode != SGP_GRID_REFERENCE && pass < 4; ++pass) {
        if (cudaMemcpyAsync(st.data(), d_st, n_nodes * sizeof(int), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
            cudaStreamSynchronize(S(stream)) != cudaSuccess) {
            rc = SGP_ECUDA;
            break;
        }
        list.clear();
        src.clear();
        int last = -1;
        for (int k = 0; k < n_nodes; ++k) {
            if (st[k] == 0) {
                last = k;
            } else if ((st[k] == 1 || st[k] == 2) && last >= 0) {
                list.push_back(k);
                src.push_back(last);
            }
        }
        if (list.empty()) break;
        const int nl = (int)list.size();
        cudaMemcpyAsync(d_list, list.data(), nl * sizeof(int), cudaMemcpyHostToDevice, S(stream));
        cudaMemcpyAsync(d_list + n_nodes, src.data(), nl * sizeof(int), cudaMemcpyHostToDevice, S(stream));
        for (int node0 = 0; !rc && node0 < nl; node0 += batch) {
            const int nb = std::min(batch, nl - node0);
            k_laplace_grid<<<nb, L.nt, L.pl.bytes, S(stream)>>>(m->dev, L.pl, gd, node0, nl, d_scr, spc, stride, d_val,
                                                                 d_st, d_it, d_list, d_list + n_nodes, d_aopt, d_aopt);
            rc = check_launch();
        }
    }
    if (!rc) {
        if (cudaMemcpyAsync(h_values, d_val, n_nodes * sizeof(double), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
            cudaMemcpyAsync(h_status, d_st, n_nodes * sizeof(int), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
            (h_iters && cudaMemcpyAsync(h_iters, d_it, n_nodes * sizeof(int), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) ||
            cudaStreamSynchronize(S(stream)) != cudaSuccess)
            rc = SGP_ECUDA;
    }
    cudaFree(d_scr);
    cudaFree(d_val);
    cudaFree(d_st);
    cudaFree(d_it);
    cudaFree(d_aopt);
    cudaFree(d_list);
    return rc;
}

// laplace_full (evidence.py:277-304) on one posterior: host q0 (d) in,
// host out[4] = {value, U(q*), log det H, min eigenvalue}, status, iterations.
extern "C" int sgp_laplace_full(const sgp_model *m, double tau, const double *h_q0, double gtol, int max_iters,
                                double zeta, int sweep_cap, double *h_out4, int *h_status, int *h_iters, void *stream) {
    if (!m || !h_q0 || !h_out4 || !h_status || max_iters < 0) return SGP_EINVAL;
    if (lg_is_large(m->dev)) return SGP_EINVAL;
    const int d = m->dev.mp.d, memory = 10;
    SmemPlan pl;
    chain_plan(m, pl);
    const size_t spc = sgp_scratch_doubles(m) + sgp_grid_scratch_extra(d, memory);
    double *buf = nullptr;
    int *ib = nullptr;
    if (cudaMalloc(&buf, (spc + d + 4) * sizeof(double)) != cudaSuccess) return SGP_ENOMEM;
    if (cudaMalloc(&ib, 2 * sizeof(int)) != cudaSuccess) {
        cudaFree(buf);
        return SGP_ENOMEM;
    }
    double *d_q0 = buf + spc, *d_out = d_q0 + d;
    int rc = launch_prep(k_laplace_full, pl.bytes);
    if (!rc && cudaMemcpyAsync(d_q0, h_q0, d * sizeof(double), cudaMemcpyHostToDevice, S(stream)) != cudaSuccess)
        rc = SGP_ECUDA;
    if (!rc) {
        k_laplace_full<<<1, SGP_MAX_NT, pl.bytes, S(stream)>>>(m->dev, pl, d_q0, tau, gtol, max_iters, memory, zeta,
                                                               sweep_cap, buf, sgp_scratch_doubles(m), d_out, ib,
                                                               ib + 1);
        rc = check_launch();
    }
    int hb[2] = {0, 0};
    if (!rc && (cudaMemcpyAsync(h_out4, d_out, 4 * sizeof(double), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
                cudaMemcpyAsync(hb, ib, 2 * sizeof(int), cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
                cudaStreamSynchronize(S(stream)) != cudaSuccess))
        rc = SGP_ECUDA;
    *h_status = hb[0];
    if (h_iters) *h_iters = hb[1];
    cudaFree(buf);
    cudaFree(ib);
    return rc;
}
