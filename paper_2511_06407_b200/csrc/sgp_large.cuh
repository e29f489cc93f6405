// sgp_large.cuh — large-d path (nl-meanvar, N = 8192,
// d = 2083), one chain at a time occupying the whole GPU.
//
// The O(N d^2) and O(d^3) contractions run as DMMA GEMMs (sgp_gemm.cuh):
//   Hessian   H_lik[j1,j2] = Phi_j1^T diag(tau d2_{j1 j2}) Phi_j2      (posterior.py:449-460)
//   trace     Y_j1 = Phi_j1 W[blk j1, :], s^(j1 j2)_i = <Y_j1[i, blk j2], phi_j2(x_i)>   (:495-509)
//   metric    W = Psi M Psi^T, M = diag((lam/g)/g) - (b b^T) o T       (metric.py:188-204)
//   warm eigh A = Psi^T H Psi                                           (metric.py:170)
// Warm decompositions use the block Jacobi (round-robin order of 64 x 64 pair
// problems, warm_order="parallel") or the reference's cyclic order (sgp_jbig.cuh,
// bit-exact); cold decompositions keep the reference order unless
// cold_order="parallel" (chain start, rejections, rung starts).  The O(d) and
// O(N d) glue (per-sample derivatives, prior terms, mat-vecs, fixed-point
// updates) reuses the CTA-level functions on one CTA.  The leapfrog control
// flow runs on the host thread, reading back one status/delta word per
// fixed-point iteration.
#pragma once
#include "sgp_chain.cuh"
#include "sgp_gemm.cuh"
#include "sgp_jbig.cuh"
#include "sgp_dc.cuh"

#define LG_NT 256
#define LG_NCORR 4  // warm calls per leapfrog with a stored refinement correction

struct LgPtrs {
    ModelDev M;
    double *S, *H, *X, *W, *P[2], *Y, *sacc, *vec, *sc, *jlog, *jprm, *red;
    int *si, *status, *jpairs;
    // block Jacobi (round-robin order, warm and cold decompositions at large d)
    int bj_dp, bj_nbk;           // padded dimension (multiple of 2*BJ_B), number of blocks (even)
    double *bjA, *bjT, *bjV[2];  // bj_dp x bj_dp working matrices
    double *bjU, *bjLam, *bjPart;
    int *bjCnt;
    GemmArgs *bjDesc;            // [round][col A | row A | col V even | col V odd][2 * pairs]
    GemmArgs *hdesc;             // the likelihood-Hessian blocks' batched GEMM descriptors (4)
    double *hpart;               // second K half of the off-diagonal likelihood block (J = 2)
    double *Dcorr[LG_NCORR][3];  // per warm-call index: the last three leapfrogs' refinement corrections
    int4 *htiles;                // grouped stream-K tile list of the likelihood blocks (built once)
    long *hprefix;
    int hntiles;
    // host handles owned by this workspace (one per model, like the buffers above): the
    // high-priority stream of the block-Jacobi A chain and the events ordering it against
    // the caller's stream (in, solved, chain, V update of even / odd rounds)
    cudaStream_t bj_hs;
    cudaEvent_t bj_ev[5];
    // reference-order Jacobi (sgp_jbig.cuh) workspace, allocated on first use
    JbWS *jb;
    // tridiagonalisation + divide and conquer workspace (cold_order="dc"), allocated on first use
    DcWS *dc;
    // pinned host staging of the scalars read back at every host decision (lg_sync)
    double *hsync;
};

static void lg_free_handles(LgPtrs &L) {
    if (L.jb) {
        jb_ws_free(*L.jb);
        delete L.jb;
        L.jb = nullptr;
    }
    if (L.dc) {
        dc_ws_free(*L.dc);
        delete L.dc;
        L.dc = nullptr;
    }
    if (L.hsync) cudaFreeHost(L.hsync);
    L.hsync = nullptr;
    if (L.bj_hs) cudaStreamDestroy(L.bj_hs);
    for (cudaEvent_t &e : L.bj_ev)
        if (e) cudaEventDestroy(e);
    L.bj_hs = nullptr;
    for (cudaEvent_t &e : L.bj_ev) e = nullptr;
}

struct LargeWS {
    LgPtrs p;
    size_t bytes;
};

__device__ inline void lg_setup(ChainWS &w, EvalCtx &E, const LgPtrs &L, char *smem) {
    const int d = L.M.mp.d;
    E.M = L.M;
    E.red = reinterpret_cast<double *>(smem);
    E.status = L.status;
    E.S = L.S;
    E.stage = nullptr;
    E.wp = nullptr;
    E.CH = 32;
    E.stage_cap = 0;
    E.ext_trace = 2;
    E.su_ext = 0.0;
    w.sc = L.sc;
    w.si = L.si;
    double **vecs[] = {&w.q0, &w.qc, &w.qn, &w.qs, &w.p, &w.ph, &w.pn, &w.v0, &w.grad, &w.tv, &w.bv, &w.tmp,
                       &w.lam[0], &w.lam[1], &w.g[0], &w.g[1]};
    for (int k = 0; k < 16; ++k) *vecs[k] = L.vec + (size_t)k * d;
    w.H = L.H;
    w.X = L.X;
    w.W = L.W;
    w.P[0] = L.P[0];
    w.P[1] = L.P[1];
    w.T = nullptr;
    w.prm = L.jprm;
    w.jlog = L.jlog;
}

// single-CTA glue operations
enum LgOp {
    LG_STATE = 0,      // eval_state(q = vec[a0], what = i0): pot -> sc[2], sumpot -> sc[3]
    LG_TRACE = 1,      // t -> tv from S (c^(j) precomputed) at q = vec[a0]
    // 2, 3: (Psi^T v, G^-1 v) now grid kernels, lg_tvec / lg_apply_g
    LG_GLAM = 4,       // lam_slot = diag(H); g_slot, logdet -> sc[slot]; since -> si[slot] = i0
    // 5, 6: (MGS, kinetic) now grid kernels, lg_mgs / k_lg_kinetic_fin
    LG_COLD = 7,       // cold cyclic Jacobi of H into P_slot (bit-exact reference order)
    LG_OFFNORM = 8,    // sc[7] = off-norm of H (full storage)
    LG_LOADFRAME = 9,  // P_0 <- psi, lam_0 <- lam (from chain state), since
    LG_QDELTA = 10,    // qn = q0 + 0.5 eps (v0 + tmp); sc[5] = max|qn - qc|
    LG_PHALF = 11,     // out = p - 0.5 eps (grad + 0.5 tv); sc[5] = max|out - ph| if i0
    LG_JCYC = 12,      // reference-order Jacobi of H (as is) into P_slot (as is), tol sc[9], skip sc[10]
};

struct LgOpArgs {
    int op, slot, a0, a1, i0;
    double eps;
    sgp_chain_config cfg;
    double tau;
};

// one instantiation per op (OP only names the kernel, so profiles attribute time per op)
template <int OP>
__global__ void __launch_bounds__(LG_NT) k_lg_op(LgPtrs L, LgOpArgs a) {
    __shared__ __align__(16) char smem[128 * sizeof(double)];
    ChainWS w;
    EvalCtx E;
    lg_setup(w, E, L, smem);
    const int d = L.M.mp.d;
    double *V = L.vec;
    switch (a.op) {
        case LG_STATE: {
            EvalOut o;
            E.su_ext = w.sc[3];
            eval_state(E, V + (size_t)a.a0 * d, a.tau, a.i0 | SGP_EVAL_EXTLIK, w.grad, w.H, o);
            // a gradient-only pass over an already evaluated point keeps the stored potential
            if (threadIdx.x == 0 && !(a.i0 & SGP_EVAL_REUSE)) w.sc[2] = o.pot;
            break;
        }
        case LG_TRACE:
            eval_trace(E, V + (size_t)a.a0 * d, a.tau, w.W, w.tv);
            break;
        case LG_GLAM: {
            for (int j = threadIdx.x; j < d; j += SGP_NT) w.lam[a.slot][j] = w.H[(size_t)j * d + j];
            __syncthreads();
            const double ld = metric_g(w.lam[a.slot], w.g[a.slot], d, a.cfg.kappa, E.red);
            if (threadIdx.x == 0) {
                w.sc[a.slot] = ld;
                w.si[a.slot] = a.i0;
            }
            break;
        }
        case LG_COLD: {
            mat_symmetrize(w.H, d);
            const double hnorm = sqrt(frob2(w.H, d * d, E.red));
            const double tol = a.cfg.zeta * hnorm;
            const double skip = d ? tol / d : 0.0;
            mat_identity(w.P[a.slot], d);
            const int sw = jacobi_cyclic(w.H, w.P[a.slot], d, tol, skip, a.cfg.sweep_cap, E.red, w.jlog);
            if (threadIdx.x == 0) {
                w.si[4] = sw;
                if (sw < 0) *E.status = SGP_STATUS_JACOBI;
            }
            break;
        }
        case LG_JCYC: {
            const int sw = jacobi_cyclic(w.H, w.P[a.slot], d, w.sc[9], w.sc[10], a.cfg.sweep_cap, E.red, w.jlog);
            if (threadIdx.x == 0) {
                w.si[4] = sw;
                if (sw < 0) *E.status = SGP_STATUS_JACOBI;
            }
            break;
        }
        case LG_OFFNORM: {
            const double off = sqrt(offdiag2(w.H, d, E.red));
            if (threadIdx.x == 0) w.sc[7] = off;
            break;
        }
        case LG_QDELTA: {
            double dl = 0.0;
            bool nan_here = false;
            for (int j = threadIdx.x; j < d; j += SGP_NT) {
                const double qn = w.q0[j] + 0.5 * a.eps * (w.v0[j] + w.tmp[j]);
                w.qn[j] = qn;
                dl = fmax(dl, fabs(qn - w.qc[j]));
                nan_here |= isnan(qn - w.qc[j]);
            }
            const double delta = block_max_nan(nan_here ? NAN : dl, E.red);
            if (threadIdx.x == 0) w.sc[5] = delta;
            break;
        }
        case LG_PHALF: {
            // out = vec[a1]; p = w.p; grad, tv
            double *out = V + (size_t)a.a1 * d;
            double dl = 0.0;
            bool nan_here = false;
            for (int j = threadIdx.x; j < d; j += SGP_NT) {
                const double v = w.p[j] - 0.5 * a.eps * (w.grad[j] + 0.5 * w.tv[j]);
                if (a.i0) {
                    dl = fmax(dl, fabs(v - w.ph[j]));
                    nan_here |= isnan(v - w.ph[j]);
                }
                out[j] = v;
            }
            if (a.i0) {
                const double delta = block_max_nan(nan_here ? NAN : dl, E.red);
                if (threadIdx.x == 0) w.sc[5] = delta;
            }
            break;
        }
        default:
            break;
    }
}

// M[j][l] = [(lam/g)/g]_j delta_jl + c1 b_j T_jl b_l, T from lam, g (metric.py:46-59)
__global__ void k_lg_mmat(LgPtrs L, int slot, double kappa, double c1, int with_w1, int with_w2) {
    const int d = L.M.mp.d;
    const double *lam = L.vec + (size_t)(12 + slot) * d, *g = L.vec + (size_t)(14 + slot) * d;
    const double *b = L.vec + (size_t)10 * d;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < d^2 < 2^32: 32-bit division
        const int j = (int)(u_ / (unsigned)d), l = (int)(u_ - (unsigned)j * (unsigned)d);
        double m = 0.0;
        if (with_w1) {
            const double diff = lam[j] - lam[l];
            const double T = (fabs(diff) <= kappa * 1e-10) ? lam[j] / g[j] : (g[j] - g[l]) / diff;
            m = c1 * ((b[j] * T) * b[l]);
        }
        if (with_w2 && j == l) m += (lam[j] / g[j]) / g[j];
        L.W[idx] = m;
    }
}

// A <- 0.5 (A + A^T): tile pairs (ti, tj), ti <= tj, through shared memory (both sides
// coalesced).  Launch: grid (nt, nt), block (32, 8).
__global__ void k_lg_symmetrize_tiled(double *A, int d) {
    __shared__ double up[32][33], lo[32][33];
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (ti > tj) return;
    const int r0 = ti * 32, c0 = tj * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = r0 + k, c = c0 + threadIdx.x;
        if (r < d && c < d) up[k][threadIdx.x] = A[(size_t)r * d + c];
        const int r2 = c0 + k, c2 = r0 + threadIdx.x;
        if (r2 < d && c2 < d) lo[k][threadIdx.x] = A[(size_t)r2 * d + c2];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        // upper element (r0+k, c0+x) pairs with lower (c0+x, r0+k) = lo[x][k]
        const int r = r0 + k, c = c0 + threadIdx.x;
        if (r < d && c < d && r < c) A[(size_t)r * d + c] = 0.5 * (up[k][threadIdx.x] + lo[threadIdx.x][k]);
        const int r2 = c0 + k, c2 = r0 + threadIdx.x;
        if (r2 < d && c2 < d && r2 > c2) A[(size_t)r2 * d + c2] = 0.5 * (up[threadIdx.x][k] + lo[k][threadIdx.x]);
    }
}
static inline void lg_symmetrize(double *A, int d, cudaStream_t s) {
    const int nt = (d + 31) / 32;
    k_lg_symmetrize_tiled<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(A, d);
}

__global__ void k_lg_copy(double *dst, const double *src, size_t n) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x)
        dst[idx] = src[idx];
}

__global__ void k_lg_zero(double *dst, size_t n) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x)
        dst[idx] = 0.0;
}

// per-sample quadratic forms from Y_j1 (ld x Dtot, coordinate columns): warp per sample
__global__ void k_lg_rowdot(LgPtrs L, int j1, int final_pass) {
    const ModelParams &mp = L.M.mp;
    const int Dt = mp.Dtot, ld = mp.ld;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = warp; i < mp.N; i += nw) {
        const double *y = L.Y + (size_t)i * Dt;
        const double *ph = L.M.phis + (size_t)i * mp.Dp;
        double s0 = 0.0, s1 = 0.0;
        // second block (J = 2): only its own columns were formed (s10 = s01, W symmetric)
        for (int b = (j1 == 1 ? mp.D[0] : 0) + lane; b < Dt; b += 32) {
            const bool blk1 = b >= mp.D[0];
            const int pb = blk1 ? mp.Dp0 + (b - mp.D[0]) : b;
            const double v = y[b] * ph[pb];
            if (blk1)
                s1 += v;
            else
                s0 += v;
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        if (lane == 0) {
            double *sa = L.sacc;
            if (j1 == 0) {
                sa[i] = s0;           // s00
                sa[ld + i] = s1;      // s01 (cross, first half)
                sa[2 * ld + i] = 0.0;
            } else {
                // s01 + s10 with s10 = s01: W is exactly symmetric (mirrored), so
                // phi_1^T W_10 phi_0 equals phi_0^T W_01 phi_1 up to rounding (posterior.py:495-509
                // forms both)
                sa[ld + i] += sa[ld + i];
                sa[2 * ld + i] = s1;  // s11
            }
            if (final_pass) {
                double *S = L.S;
                if (mp.J == 1) {
                    S[F_C0 * ld + i] = S[F_D3_000 * ld + i] * sa[i];
                } else {
                    const double a00 = sa[i], ax = sa[ld + i], a11 = sa[2 * ld + i];
                    const double t001 = S[F_D3_001 * ld + i], t011 = S[F_D3_011 * ld + i];
                    const double t111 = S[F_D3_111 * ld + i];
                    S[F_C0 * ld + i] = t001 * ax + t011 * a11;
                    S[F_C1 * ld + i] = t001 * a00 + t011 * ax + t111 * a11;
                }
            }
        }
    }
}

// ---- grid-parallel Jacobi (round-robin order) -------------------------------
// prm per pair: c, s, t*apq, app, aqq ; pairs: p, q (p = -1 inactive)
__global__ void k_lg_jrows(double *A, int d, int r, double skip, double *prm, int *pairs) {
    const int m = d + (d & 1), np = m >> 1;
    const int k = blockIdx.x;
    if (k >= np) return;
    __shared__ double cs[2];
    __shared__ int pq[2];
    if (threadIdx.x == 0) {
        int a, b;
        if (k == 0) {
            a = r;
            b = m - 1;
        } else {
            a = (r + k) % (m - 1);
            b = (r - k + m - 1) % (m - 1);
        }
        int p = min(a, b), q = max(a, b);
        int act = 0;
        if (q < d) {
            const double apq = A[(size_t)p * d + q];
            if (fabs(apq) > skip) {
                const double app = A[(size_t)p * d + p], aqq = A[(size_t)q * d + q];
                double c, s, t;
                jacobi_rot(app, aqq, apq, c, s, t);
                prm[5 * k + 0] = c;
                prm[5 * k + 1] = s;
                prm[5 * k + 2] = t * apq;
                prm[5 * k + 3] = app;
                prm[5 * k + 4] = aqq;
                cs[0] = c;
                cs[1] = s;
                act = 1;
            }
        }
        pq[0] = act ? p : -1;
        pq[1] = q;
        pairs[2 * k] = pq[0];
        pairs[2 * k + 1] = q;
    }
    __syncthreads();
    const int p = pq[0];
    if (p < 0) return;
    const int q = pq[1];
    const double c = cs[0], s = cs[1];
    double *rp = A + (size_t)p * d, *rq = A + (size_t)q * d;
    for (int l = threadIdx.x; l < d; l += blockDim.x) {
        const double ap = rp[l], aq = rq[l];
        rp[l] = c * ap - s * aq;
        rq[l] = s * ap + c * aq;
    }
}

__global__ void k_lg_jcols(double *A, double *V, int d, const double *prm, const int *pairs) {
    const int m = d + (d & 1), np = m >> 1;
    // one CTA per row l; threads over pairs
    for (int l = blockIdx.x; l < d; l += gridDim.x) {
        double *ra = A + (size_t)l * d, *rv = V + (size_t)l * d;
        for (int k = threadIdx.x; k < np; k += blockDim.x) {
            const int p = pairs[2 * k];
            if (p < 0) continue;
            const int q = pairs[2 * k + 1];
            const double c = prm[5 * k], s = prm[5 * k + 1];
            const double ap = ra[p], aq = ra[q];
            ra[p] = c * ap - s * aq;
            ra[q] = s * ap + c * aq;
            const double vp = rv[p], vq = rv[q];
            rv[p] = c * vp - s * vq;
            rv[q] = s * vp + c * vq;
            if (l == p) {
                ra[p] = prm[5 * k + 3] - prm[5 * k + 2];
                ra[q] = 0.0;
            } else if (l == q) {
                ra[q] = prm[5 * k + 4] + prm[5 * k + 2];
                ra[p] = 0.0;
            }
        }
    }
}

__global__ void k_lg_transpose_block(double *H, int d, int r0, int c0, int nr, int nc) {
    // H[c0 + j][r0 + i] = H[r0 + i][c0 + j]
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)nr * nc;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < nc^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)nc), j = (int)(u_ - (unsigned)i * (unsigned)nc);
        H[(size_t)(c0 + j) * d + r0 + i] = H[(size_t)(r0 + i) * d + c0 + j];
    }
}

// off-diagonal likelihood block computed as two K halves: H[r0+i][c0+j] += P[i][j] (P: the
// second half, nr x nc, leading dimension ldp), then mirrored into H[c0+j][r0+i]; 32 x 32 tiles
// through shared memory so both the row and the mirrored column side are coalesced
__global__ void k_lg_addt_block(double *H, int d, int r0, int c0, int nr, int nc, const double *P, int ldp) {
    __shared__ double t[32][33];
    const int ti = blockIdx.y * 32, tj = blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = ti + k, j = tj + threadIdx.x;
        if (i < nr && j < nc) {
            double *h = H + (size_t)(r0 + i) * d + c0 + j;
            const double v = *h + P[(size_t)i * ldp + j];
            *h = v;
            t[k][threadIdx.x] = v;
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = tj + k, i = ti + threadIdx.x;
        if (i < nr && j < nc) H[(size_t)(c0 + j) * d + r0 + i] = t[threadIdx.x][k];
    }
}

// dst = src^T (d x d), 32x32 tiles through shared memory (both sides coalesced)
__global__ void k_lg_transpose(double *dst, const double *src, int d) {
    __shared__ double t[32][33];
    const int nt = (d + 31) / 32;
    for (int tile = blockIdx.x; tile < nt * nt; tile += gridDim.x) {
        const int by = tile / nt, bx = tile - by * nt;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = by * 32 + r, j = bx * 32 + threadIdx.x;
            if (i < d && j < d) t[r][threadIdx.x] = src[(size_t)i * d + j];
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = bx * 32 + r, j = by * 32 + threadIdx.x;
            if (i < d && j < d) dst[(size_t)i * d + j] = t[threadIdx.x][r];
        }
        __syncthreads();
    }
}

// Step i of modified Gram-Schmidt on the ROWS of X = Psi^T, i.e. on the
// columns of Psi as _jacobi.py:90-107 does: column i /= ||column i||, then
// every column j > i loses its component along column i.  Every block
// normalises row i into shared memory from the unmodified row; block 0 writes
// the normalised row i-1 of the previous step (nobody reads it any more), so
// the steps need no grid-wide barrier.  nrm[0]: norm of row i-1 (0 = skipped).
__global__ void k_lg_mgs_step(double *X, int d, int i, double *nrm) {
    extern __shared__ double xi[];
    __shared__ double red[32];
    if (blockIdx.x == 0 && i > 0) {
        const double n0 = nrm[0];
        __syncthreads();
        if (n0 != 0.0)
            for (int k = threadIdx.x; k < d; k += blockDim.x) X[(size_t)(i - 1) * d + k] /= n0;
    }
    if (i >= d) return;
    const double *ri = X + (size_t)i * d;
    double s = 0.0;
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        const double v = ri[k];
        xi[k] = v;
        s += v * v;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const double n = sqrt(tot);
    if (blockIdx.x == 0 && threadIdx.x == 0) nrm[0] = n;
    if (n == 0.0) return;
    for (int k = threadIdx.x; k < d; k += blockDim.x) xi[k] /= n;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = (int)(gridDim.x * (blockDim.x >> 5));
    for (int j = i + 1 + (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); j < d; j += warps) {
        double *rj = X + (size_t)j * d;
        double dot = 0.0;
        for (int k = lane; k < d; k += 32) dot += xi[k] * rj[k];
        dot = warp_sum(dot);
        for (int k = lane; k < d; k += 32) rj[k] -= dot * xi[k];
    }
}

__global__ void k_lg_mirror_block(double *H, int d, int o, int n) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)n * n;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < n^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)n), j = (int)(u_ - (unsigned)i * (unsigned)n);
        if (i > j) H[(size_t)(o + i) * d + o + j] = H[(size_t)(o + j) * d + o + i];
    }
}

__global__ void k_lg_frob(const double *A, size_t n, double *out) {
    __shared__ double red[64];
    double s = 0.0;
    for (size_t idx = threadIdx.x; idx < n; idx += blockDim.x) s += A[idx] * A[idx];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

__global__ void k_lg_eye(double *P, int d) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x)
        P[idx] = (idx / d == idx % d) ? 1.0 : 0.0;
}

__global__ void k_lg_set2(double *dst, double a, double b) {
    dst[0] = a;
    dst[1] = b;
}

// ---- grid-wide O(N d) glue ------------------------------------------------
// latent values and per-sample derivatives; block partial sums of U and a
// non-finite flag into red[blockIdx.x], red[gridDim.x + blockIdx.x]
// f = Phi q and the per-sample likelihood fields.  32 samples per CTA (one per lane, coalesced
// feature-major Phi rows); the 8 warps split the features with four accumulators each, so
// 8192 samples keep 2048 warps streaming Phi (136 MB at C4) instead of 256 serial dot products.
#define LG_LIK_SPB 32
__global__ void __launch_bounds__(256) k_lg_lik(LgPtrs L, const double *q) {
    __shared__ double part[2][8][LG_LIK_SPB + 1];
    __shared__ double red[64];
    const ModelParams &mp = L.M.mp;
    const int ld = mp.ld, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * LG_LIK_SPB + lane;
    for (int j = 0; j < mp.J; ++j) {
        const int D = mp.D[j], a0 = (D * warp) / 8, a1 = (D * (warp + 1)) / 8;
        const double *ph = L.M.phi + (size_t)(j ? mp.D[0] : 0) * ld + i;
        const double *qq = q + (j ? mp.fstart[1] : 0);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (i < ld) {
            int a = a0;
            for (; a + 3 < a1; a += 4) {
                s0 = fma(ph[(size_t)a * ld], qq[a], s0);
                s1 = fma(ph[(size_t)(a + 1) * ld], qq[a + 1], s1);
                s2 = fma(ph[(size_t)(a + 2) * ld], qq[a + 2], s2);
                s3 = fma(ph[(size_t)(a + 3) * ld], qq[a + 3], s3);
            }
            for (; a < a1; ++a) s0 = fma(ph[(size_t)a * ld], qq[a], s0);
        }
        part[j][warp][lane] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    double su = 0.0, bad = 0.0;
    if (warp == 0 && i < ld) {
        double f0 = 0.0, f1 = 0.0;
        for (int w = 0; w < 8; ++w) {
            f0 += part[0][w][lane];
            if (mp.J == 2) f1 += part[1][w][lane];
        }
        if (i < mp.N) {
            if (!isfinite(f0) || !isfinite(f1)) bad = 1.0;
            L.S[F_F0 * ld + i] = f0;
            L.S[F_F1 * ld + i] = f1;
            lik_sample(mp.lik, mp.vfloor, L.M.y[i], f0, f1, L.S, ld, i);
            su = L.S[F_U * ld + i];
        } else {
            for (int k = 0; k < F_COUNT; ++k) L.S[k * ld + i] = 0.0;
        }
    }
    su = block_sum(su, red);
    __syncthreads();
    bad = block_sum(bad, red);
    if (threadIdx.x == 0) {
        L.red[blockIdx.x] = su;
        L.red[gridDim.x + blockIdx.x] = bad;
    }
}

// sc[3] = sum of the block partials (fixed order); status DIVERGENCE on a flag
__global__ void k_lg_lik_finish(LgPtrs L, int nblocks) {
    if (threadIdx.x != 0) return;
    double su = 0.0, bad = 0.0;
    for (int b = 0; b < nblocks; ++b) {
        su += L.red[b];
        bad += L.red[nblocks + b];
    }
    L.sc[3] = su;
    if (bad > 0.0 && *L.status == 0) *L.status = SGP_STATUS_DIVERGENCE;
}

// out[a] = tau sum_i phi[a, i] S[field(j(a)), i] for a < Dtot (warp per row)
__global__ void k_lg_project(LgPtrs L, double tau, int field0, int field1, double *out) {
    const ModelParams &mp = L.M.mp;
    const int ld = mp.ld;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int a = warp; a < mp.Dtot; a += nw) {
        const int f = (a < mp.D[0]) ? field0 : field1;
        const double *pr = L.M.phi + (size_t)a * ld;
        const double *sr = L.S + (size_t)f * ld;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = lane;
        for (; i + 96 < mp.N; i += 128) {
            s0 += pr[i] * sr[i];
            s1 += pr[i + 32] * sr[i + 32];
            s2 += pr[i + 64] * sr[i + 64];
            s3 += pr[i + 96] * sr[i + 96];
        }
        for (; i < mp.N; i += 32) s0 += pr[i] * sr[i];
        const double s = warp_sum((s0 + s1) + (s2 + s3));
        if (lane == 0) out[a] = tau * s;
    }
}

// ---------------------------------------------------------------------------
// Block Jacobi for large d (round-robin pair order: warm
// decompositions are order-insensitive to the Jacobi tolerance).  The padded
// matrix is split into blocks of BJ_B; each round pairs the blocks
// round-robin, every pair's 2*BJ_B x 2*BJ_B subproblem [A_II A_IJ; A_JI A_JJ]
// is diagonalised in shared memory by the same rotation formula, skip rule
// and (per inner sweep) convergence rule as the reference, and the pair
// transformations U are applied to A (columns, then rows) and to V as
// batched FP64 tensor-core GEMMs (DMMA, K gathered from the two blocks).
// Convergence: off-norm(A) <= tol before each outer sweep (_jacobi.py:50-51).
#define BJ_B 32
#define BJ_N (2 * BJ_B)
#define BJ_INNER_CAP 60
// S and U (rows padded to BJ_N + 1), then the per-sweep rotation log: c and s of
// every (step, pair) and the pivot indices (p = 0xff marks a skipped rotation)
#define BJ_LOG_N ((BJ_N - 1) * (BJ_N / 2))
#define BJ_SMEM ((size_t)2 * BJ_N * (BJ_N + 1) * sizeof(double) + (size_t)BJ_LOG_N * (2 * sizeof(double) + 2))

__host__ __device__ inline void bj_pair(int r, int k, int nbk, int &I, int &J) {
    int a, b;
    if (k == 0) {
        a = r;
        b = nbk - 1;
    } else {
        a = (r + k) % (nbk - 1);
        b = (r - k + nbk - 1) % (nbk - 1);
    }
    I = a < b ? a : b;
    J = a < b ? b : a;
}

#define BJ_SOLVE_NT 1024
__global__ void __launch_bounds__(BJ_SOLVE_NT) k_bj_solve(const double *A, int dp, int r, int nbk, double skip, double *Uall,
                                                  double *lamall, int *cnt, int inner_cap) {
    extern __shared__ double bjsm[];  // S and U, rows padded to BJ_N + 1
    double(*S)[BJ_N + 1] = reinterpret_cast<double(*)[BJ_N + 1]>(bjsm);
    double(*U)[BJ_N + 1] = reinterpret_cast<double(*)[BJ_N + 1]>(bjsm + BJ_N * (BJ_N + 1));
    double *lc = bjsm + 2 * BJ_N * (BJ_N + 1), *ls = lc + BJ_LOG_N;
    unsigned char *lp = reinterpret_cast<unsigned char *>(ls + BJ_LOG_N), *lq = lp + BJ_LOG_N;
    __shared__ double rc[BJ_N / 2], rs[BJ_N / 2], rt[BJ_N / 2], rpp[BJ_N / 2], rqq[BJ_N / 2];
    __shared__ int rp[BJ_N / 2], rq[BJ_N / 2], ract[BJ_N / 2];
    __shared__ int any, nrot;
    const int k = blockIdx.x, tid = threadIdx.x;
    int I, J;
    bj_pair(r, k, nbk, I, J);
    for (int idx = tid; idx < BJ_N * BJ_N; idx += blockDim.x) {
        const int i = idx / BJ_N, j = idx - i * BJ_N;
        const int gi = i < BJ_B ? I * BJ_B + i : J * BJ_B + i - BJ_B;
        const int gj = j < BJ_B ? I * BJ_B + j : J * BJ_B + j - BJ_B;
        S[i][j] = A[(size_t)gi * dp + gj];
        U[i][j] = i == j ? 1.0 : 0.0;
    }
    if (tid == 0) nrot = 0;
    __syncthreads();
    constexpr int m = BJ_N, np = BJ_N / 2;
    for (int sweep = 0; sweep < inner_cap; ++sweep) {
        if (tid == 0) any = 0;
        __syncthreads();
        for (int rr = 0; rr < m - 1; ++rr) {
            if (tid < np) {
                int a, b;
                if (tid == 0) {
                    a = rr;
                    b = m - 1;
                } else {
                    a = (rr + tid) % (m - 1);
                    b = (rr - tid + m - 1) % (m - 1);
                }
                const int p = min(a, b), q = max(a, b);
                const double apq = S[p][q];
                const bool act = fabs(apq) > skip;
                double c = 1.0, sn = 0.0, t = 0.0;
                const double app = S[p][p], aqq = S[q][q];
                if (act && !jacobi_rot_fast(app, aqq, apq, c, sn, t)) jacobi_rot(app, aqq, apq, c, sn, t);
                rc[tid] = c;
                rs[tid] = sn;
                rt[tid] = t * apq;
                rpp[tid] = app;
                rqq[tid] = aqq;
                rp[tid] = p;
                rq[tid] = q;
                ract[tid] = act;
                lc[rr * np + tid] = c;
                ls[rr * np + tid] = sn;
                lp[rr * np + tid] = act ? (unsigned char)p : (unsigned char)0xff;
                lq[rr * np + tid] = (unsigned char)q;
                const unsigned bal = __ballot_sync(0xffffffffu, act);
                if (tid == 0 && bal) {
                    any = 1;
                    nrot += __popc(bal);
                }
            }
            __syncthreads();
            // fused two-sided update: thread (P, Q) owns the 2x2 block rows {p_P, q_P} x
            // cols {p_Q, q_Q}; row rotation P then column rotation Q, in registers
            // (the same rounded operations as a row pass followed by a column pass)
            double nv[4];
            int bi[2], bj[2];
            bool act_blk = false;
            if (tid < np * np) {
                const int P = tid / np, Q = tid - P * np;
                const bool aP = ract[P], aQ = ract[Q];
                act_blk = aP || aQ;
                const int p1 = rp[P], q1 = rq[P], p2 = rp[Q], q2 = rq[Q];
                bi[0] = p1;
                bi[1] = q1;
                bj[0] = p2;
                bj[1] = q2;
                if (act_blk) {
                    if (P == Q) {
                        nv[0] = rpp[P] - rt[P];
                        nv[1] = 0.0;
                        nv[2] = 0.0;
                        nv[3] = rqq[P] + rt[P];
                    } else {
                        const double cP = rc[P], sP = rs[P], cQ = rc[Q], sQ = rs[Q];
                        const double a00 = S[p1][p2], a01 = S[p1][q2], a10 = S[q1][p2], a11 = S[q1][q2];
                        double r00 = a00, r01 = a01, r10 = a10, r11 = a11;
                        if (aP) {
                            r00 = cP * a00 - sP * a10;
                            r10 = sP * a00 + cP * a10;
                            r01 = cP * a01 - sP * a11;
                            r11 = sP * a01 + cP * a11;
                        }
                        if (aQ) {
                            nv[0] = cQ * r00 - sQ * r01;
                            nv[1] = sQ * r00 + cQ * r01;
                            nv[2] = cQ * r10 - sQ * r11;
                            nv[3] = sQ * r10 + cQ * r11;
                        } else {
                            nv[0] = r00;
                            nv[1] = r01;
                            nv[2] = r10;
                            nv[3] = r11;
                        }
                    }
                }
            }
            __syncthreads();
            if (act_blk) {
                S[bi[0]][bj[0]] = nv[0];
                S[bi[0]][bj[1]] = nv[1];
                S[bi[1]][bj[0]] = nv[2];
                S[bi[1]][bj[1]] = nv[3];
            }
            __syncthreads();
        }
        // U = U R_0 R_1 ... from the log, off the S chain: rows of U are independent,
        // so one warp walks its rows through all steps with only warp-level syncs
        // (each lane one pair of a step; the same rounded operations as a per-step update)
        {
            const int lane = tid & 31, nwarp = blockDim.x >> 5;
            for (int l0 = tid >> 5; l0 < m; l0 += 2 * nwarp) {
                const int l1 = l0 + nwarp;  // two rows per pass for latency overlap
                const bool two = l1 < m;
                for (int rr = 0; rr < m - 1; ++rr) {
                    for (int kk = lane; kk < np; kk += 32) {
                        const int p = lp[rr * np + kk];
                        if (p != 0xff) {
                            const int q = lq[rr * np + kk];
                            const double c = lc[rr * np + kk], sn = ls[rr * np + kk];
                            const double up0 = U[l0][p], uq0 = U[l0][q];
                            const double up1 = two ? U[l1][p] : 0.0, uq1 = two ? U[l1][q] : 0.0;
                            U[l0][p] = c * up0 - sn * uq0;
                            U[l0][q] = sn * up0 + c * uq0;
                            if (two) {
                                U[l1][p] = c * up1 - sn * uq1;
                                U[l1][q] = sn * up1 + c * uq1;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
        }
        if (!any) break;
    }
    double *Uk = Uall + (size_t)k * BJ_N * BJ_N;
    for (int idx = tid; idx < BJ_N * BJ_N; idx += blockDim.x) Uk[idx] = U[idx / BJ_N][idx % BJ_N];
    // the transformed subproblem (diagonal when the inner sweeps converged)
    for (int idx = tid; idx < BJ_N * BJ_N; idx += blockDim.x) lamall[(size_t)k * BJ_N * BJ_N + idx] = S[idx / BJ_N][idx % BJ_N];
    if (tid == 0) cnt[k] = nrot;
}

// diagonal blocks of every pair after its transformation: the inner solver's
// transformed subproblem (exact zeros where it annihilated, as the reference does)
__global__ void k_bj_fix(double *A, int dp, int r, int nbk, const double *lamall, const int *cnt) {
    const int k = blockIdx.x;
    if (!cnt[k]) return;
    int I, J;
    bj_pair(r, k, nbk, I, J);
    for (int idx = threadIdx.x; idx < BJ_N * BJ_N; idx += blockDim.x) {
        const int i = idx / BJ_N, j = idx - i * BJ_N;
        const int gi = i < BJ_B ? I * BJ_B + i : J * BJ_B + i - BJ_B;
        const int gj = j < BJ_B ? I * BJ_B + j : J * BJ_B + j - BJ_B;
        A[(size_t)gi * dp + gj] = lamall[(size_t)k * BJ_N * BJ_N + idx];
    }
}

// off-diagonal sum of squares, deterministic: per-block partials then one ordered sum
__global__ void k_bj_offnorm(const double *A, int dp, double *part) {
    __shared__ double red[32];
    double s = 0.0;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)dp * dp;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t i = idx / dp, j = idx - i * dp;
        if (i != j) s += A[idx] * A[idx];
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
// ---- grid mat-vecs of the metric algebra (metric.py:188-241) at large d ----
#define LG_TV_KS 32
// part[ks][j] = sum_{k in chunk ks} P[k][j] v[k]   (Psi^T v, coalesced over j)
__global__ void k_lg_tvec_part(const double *P, const double *v, int d, double *part) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, ks = blockIdx.y;
    const int chunk = (d + LG_TV_KS - 1) / LG_TV_KS, k0 = ks * chunk, k1 = min(d, k0 + chunk);
    if (j >= d) return;
    // four independent accumulators: the loads of four rows are in flight together
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int k = k0;
    for (; k + 3 < k1; k += 4) {
        s0 += P[(size_t)k * d + j] * v[k];
        s1 += P[(size_t)(k + 1) * d + j] * v[k + 1];
        s2 += P[(size_t)(k + 2) * d + j] * v[k + 2];
        s3 += P[(size_t)(k + 3) * d + j] * v[k + 3];
    }
    for (; k < k1; ++k) s0 += P[(size_t)k * d + j] * v[k];
    part[(size_t)ks * d + j] = (s0 + s1) + (s2 + s3);
}
// out[j] = f(sum_ks part[ks][j]): mode 0: /g, 1: *g, 3: plain; 4: kinetic terms t^2/g into out
__global__ void k_lg_tvec_fin(const double *part, const double *g, int d, int mode, double *out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    double s = 0.0;
    for (int ks = 0; ks < LG_TV_KS; ++ks) s += part[(size_t)ks * d + j];
    out[j] = mode == 0 ? s / g[j] : (mode == 1 ? g[j] * s : (mode == 4 ? s * s / g[j] : s));
}
// out[j] = sum_k P[j][k] t[k]   (Psi t, one warp per row)
__global__ void k_lg_vec(const double *P, const double *t, int d, double *out) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
    if (w >= d) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const double *row = P + (size_t)w * d;
    int k = l;
    for (; k + 96 < d; k += 128) {
        s0 += row[k] * t[k];
        s1 += row[k + 32] * t[k + 32];
        s2 += row[k + 64] * t[k + 64];
        s3 += row[k + 96] * t[k + 96];
    }
    for (; k < d; k += 32) s0 += row[k] * t[k];
    const double s = warp_sum((s0 + s1) + (s2 + s3));
    if (l == 0) out[w] = s;
}
__global__ void k_lg_sqrtg_v(const double *g, const double *v, int d, double *out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < d) out[j] = sqrt(g[j]) * v[j];
}
// sc[6] = 0.5 * sum(terms) + 0.5 (d ln 2 pi + logdet)   (one warp, ordered)
__global__ void k_lg_kinetic_fin(const double *terms, int d, const double *sc_logdet, double *out) {
    const int l = threadIdx.x;
    double s = 0.0;
    for (int k = l; k < d; k += 32) s += terms[k];
    s = warp_sum(s);
    if (l == 0) *out = 0.5 * s + 0.5 * (d * SGP_LN_2PI + *sc_logdet);
}

// non-finite Hessian entry -> DivergenceError (posterior.py:479)
__global__ void k_lg_finite(const double *H, size_t n, int *status) {
    bool bad = false;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x)
        bad |= !isfinite(H[idx]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(status, 0, SGP_STATUS_DIVERGENCE);
}

__global__ void k_bj_sumsq(const double *A, size_t n, double *part) {
    __shared__ double red[32];
    double s = 0.0;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x)
        s += A[idx] * A[idx];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
__global__ void k_bj_sum_final(const double *part, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += part[i];
        *out = t;
    }
}
__global__ void k_bj_offnorm_final(const double *part, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += part[i];
        *out = sqrt(t);
    }
}

// padded working copies in / results out
__global__ void k_bj_in(double *Ap, double *Vp, const double *H, const double *P, int d, int dp, int identity) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)dp * dp;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < dp^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)dp), j = (int)(u_ - (unsigned)i * (unsigned)dp);
        const bool in = i < d && j < d;
        Ap[idx] = in ? H[(size_t)i * d + j] : 0.0;
        Vp[idx] = in ? (identity ? (i == j ? 1.0 : 0.0) : P[(size_t)i * d + j]) : (i == j ? 1.0 : 0.0);
    }
}
__global__ void k_bj_out(double *H, double *P, const double *Ap, const double *Vp, int d, int dp) {
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < d^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)d), j = (int)(u_ - (unsigned)i * (unsigned)d);
        P[idx] = Vp[(size_t)i * dp + j];
        if (i == j) H[idx] = Ap[(size_t)i * dp + j];
    }
}

// Descriptors of the three batched update GEMMs of every round (host side):
// one 64-wide GEMM per pair and kind, K gathered from blocks I and J and the
// output split back into blocks I and J.
static void bj_build_desc(const LgPtrs &L, std::vector<GemmArgs> &out) {
    const int dp = L.bj_dp, nbk = L.bj_nbk, np = nbk / 2;
    out.clear();
    for (int r = 0; r < nbk - 1; ++r) {
        for (int kind = 0; kind < 4; ++kind) {  // 0 col A, 1 row A, 2 col V (V0->V1), 3 col V (V1->V0)
            for (int k = 0; k < np; ++k) {
                int I, J;
                bj_pair(r, k, nbk, I, J);
                // U of round r lives in buffer r & 1 (the V update of round r may still be
                // reading it while round r + 1 is being solved on the other stream)
                const double *Uk = L.bjU + ((size_t)(r & 1) * np + k) * BJ_N * BJ_N;
                GemmArgs g{};
                g.alpha = 1.0;
                g.beta = 0.0;
                g.K = BJ_N;
                g.ksplit = BJ_B;
                if (kind == 1) {
                    // A[I|J rows, :] = U^T T[I|J rows, :]
                    g.M = BJ_N;
                    g.N = dp;
                    g.A = Uk;
                    g.lda = BJ_N;
                    g.TA = 1;
                    g.B = L.bjT + (size_t)I * BJ_B * dp;
                    g.B2 = L.bjT + (size_t)J * BJ_B * dp;
                    g.ldb = dp;
                    g.C = L.bjA + (size_t)I * BJ_B * dp;
                    g.C2 = L.bjA + (size_t)J * BJ_B * dp;
                    g.msplit = BJ_B;
                } else {
                    // X[:, I|J cols] = Y[:, I|J cols] U
                    const double *Y = kind == 0 ? L.bjA : (kind == 2 ? L.bjV[0] : L.bjV[1]);
                    double *X = kind == 0 ? L.bjT : (kind == 2 ? L.bjV[1] : L.bjV[0]);
                    g.M = dp;
                    g.N = BJ_N;
                    g.A = Y + (size_t)I * BJ_B;
                    g.A2 = Y + (size_t)J * BJ_B;
                    g.lda = dp;
                    g.B = Uk;
                    g.ldb = BJ_N;
                    g.C = X + (size_t)I * BJ_B;
                    g.C2 = X + (size_t)J * BJ_B;
                    g.nsplit = BJ_B;
                }
                g.ldc = dp;
                g.a16 = 1;
                g.b16 = 1;
                out.push_back(g);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host driver

enum { V_Q0 = 0, V_QC, V_QN, V_QS, V_P, V_PH, V_PN, V_V0, V_GRAD, V_TV, V_BV, V_TMP, V_LAM0, V_LAM1, V_G0, V_G1 };

static inline int lg_blocks(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }

struct LgCtx {
    LgPtrs L;
    cudaStream_t s;
    sgp_chain_config cfg;
    double tau;
    int d;
    double sc[16];  // host mirrors of the device scalars
    int si[16];
    int status;
    int since[2];
    // refinement warm start by correction transfer: call i of a leapfrog's position fixed point
    // starts from its natural basis S plus the correction R - S that call i made in the previous
    // leapfrog (Dcorr[i], valid while the trajectory and the column order continue)
    int corr_n[LG_NCORR];       // stored corrections of call i (up to 3: D(k-1), D(k-2), D(k-3))
    int corr_cur[LG_NCORR];     // ring slot holding D(k-1); D(k-j) at (cur - j + 1) mod 3
    long corr_lf[LG_NCORR][3];  // leapfrog index each stored correction was made in
    long lf_count;              // leapfrogs made by this context
    int warm_idx;      // index of the warm call being made (-1: none / no transfer)
    bool basis_reset;
};

static void lg_op(LgCtx &c, int op, int slot = 0, int a0 = 0, int a1 = 0, int i0 = 0, double eps = 0.0) {
    LgOpArgs a;
    a.op = op;
    a.slot = slot;
    a.a0 = a0;
    a.a1 = a1;
    a.i0 = i0;
    a.eps = eps;
    a.cfg = c.cfg;
    a.tau = c.tau;
    switch (op) {
#define LG_OP_CASE(K) \
    case K:           \
        k_lg_op<K><<<1, LG_NT, 0, c.s>>>(c.L, a); \
        break;
        LG_OP_CASE(LG_STATE)
        LG_OP_CASE(LG_TRACE)
        LG_OP_CASE(LG_GLAM)
        LG_OP_CASE(LG_COLD)
        LG_OP_CASE(LG_OFFNORM)
        LG_OP_CASE(LG_LOADFRAME)
        LG_OP_CASE(LG_QDELTA)
        LG_OP_CASE(LG_PHALF)
        LG_OP_CASE(LG_JCYC)
#undef LG_OP_CASE
        default:
            k_lg_op<-1><<<1, LG_NT, 0, c.s>>>(c.L, a);
    }
}

static int lg_sync(LgCtx &c) {
    if (c.L.hsync) {
        // sc, si and status are adjacent in the workspace: one copy into pinned staging
        const size_t n = (size_t)(reinterpret_cast<const double *>(c.L.status) - c.L.sc) + 1;
        cudaMemcpyAsync(c.L.hsync, c.L.sc, sizeof(double) * n, cudaMemcpyDeviceToHost, c.s);
        if (cudaStreamSynchronize(c.s) != cudaSuccess) return -1;
        memcpy(c.sc, c.L.hsync, sizeof(c.sc));
        memcpy(c.si, c.L.hsync + (reinterpret_cast<const double *>(c.L.si) - c.L.sc), sizeof(c.si));
        memcpy(&c.status, c.L.hsync + (reinterpret_cast<const double *>(c.L.status) - c.L.sc), sizeof(int));
        return c.status;
    }
    cudaMemcpyAsync(c.sc, c.L.sc, sizeof(c.sc), cudaMemcpyDeviceToHost, c.s);
    cudaMemcpyAsync(c.si, c.L.si, sizeof(c.si), cudaMemcpyDeviceToHost, c.s);
    cudaMemcpyAsync(&c.status, c.L.status, sizeof(int), cudaMemcpyDeviceToHost, c.s);
    if (cudaStreamSynchronize(c.s) != cudaSuccess) return -1;
    return c.status;
}

static void lg_clear_status(LgCtx &c) { cudaMemsetAsync(c.L.status, 0, sizeof(int), c.s); }

// grid versions of LG_BVEC / LG_APPLY / LG_KINETIC (same formulas as metric_apply etc.)
static void lg_tvec(LgCtx &c, int slot, const double *v, int mode, double *out) {
    const int d = c.d;
    k_lg_tvec_part<<<dim3((d + 127) / 128, LG_TV_KS), 128, 0, c.s>>>(c.L.P[slot], v, d, c.L.X);
    k_lg_tvec_fin<<<(d + 127) / 128, 128, 0, c.s>>>(c.L.X, c.L.vec + (size_t)(14 + slot) * d, d, mode, out);
}
static void lg_apply_g(LgCtx &c, int slot, int vin, int vout, int mode) {
    const int d = c.d;
    double *tmp = c.L.vec + (size_t)10 * d;  // V_BV, clobbered as in metric_apply
    const double *g = c.L.vec + (size_t)(14 + slot) * d;
    if (mode == 2)
        k_lg_sqrtg_v<<<(d + 127) / 128, 128, 0, c.s>>>(g, c.L.vec + (size_t)vin * d, d, tmp);
    else
        lg_tvec(c, slot, c.L.vec + (size_t)vin * d, mode, tmp);
    k_lg_vec<<<(d * 32 + 255) / 256, 256, 0, c.s>>>(c.L.P[slot], tmp, d, c.L.vec + (size_t)vout * d);
}

static void lg_gemm(LgCtx &c, int M, int N, int K, const double *A, int lda, int TA, const double *B, int ldb, int TB,
                    const double *scale, double *C, int ldc, double alpha, int upper) {
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
    g.scale = scale;
    g.C = C;
    g.ldc = ldc;
    g.alpha = alpha;
    g.beta = 0.0;
    g.upper_only = upper;
    gemm_launch(g, c.s);
}

// State at vec[qv]: potential (sc[2]), sum U (sc[3]), gradient (vec GRAD) if
// asked, per-sample fields; Hessian into H via DMMA GEMMs + prior terms.
static int lg_state(LgCtx &c, int qv, int what) {
    const ModelParams &mp = c.L.M.mp;
    const int d = c.d;
    const bool hess = what & SGP_EVAL_HESSIAN;
    const bool lik = mp.lik != SGP_LIK_QUADRATIC && (c.tau != 0.0 || (what & SGP_EVAL_SUMPOT));
    if (lik && !(what & SGP_EVAL_REUSE)) {
        const int nb = (mp.ld + LG_LIK_SPB - 1) / LG_LIK_SPB;
        k_lg_lik<<<nb, 256, 0, c.s>>>(c.L, c.L.vec + (size_t)qv * d);
        k_lg_lik_finish<<<1, 32, 0, c.s>>>(c.L, nb);
    } else if (!(what & SGP_EVAL_REUSE)) {
        k_lg_set2<<<1, 1, 0, c.s>>>(c.L.sc + 3, 0.0, c.sc[4]);
    }
    if ((what & SGP_EVAL_GRADIENT) && c.tau != 0.0 && mp.lik != SGP_LIK_QUADRATIC)
        k_lg_project<<<lg_blocks((size_t)mp.Dtot * 32), 256, 0, c.s>>>(c.L, c.tau, F_D1_0, F_D1_1,
                                                                      c.L.vec + (size_t)V_GRAD * d);
    lg_op(c, LG_STATE, 0, qv, 0, what & ~SGP_EVAL_HESSIAN);
    if (hess) {
        if (lg_sync(c)) return c.status;
        k_lg_zero<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.H, (size_t)d * d);
        if (c.tau != 0.0 && mp.lik != SGP_LIK_QUADRATIC) {
            const int fields[3] = {F_D2_00, F_D2_01, F_D2_11};
            // the J(J+1)/2 likelihood blocks in one batched launch (each 1040 x 1040 block alone
            // fills about half a wave of the GPU at C4)
            // preferred: the J(J+1)/2 blocks as ONE grouped stream-K launch over 128 x 64 tiles
            // (tile list built once per model); else the batched 64 x 64 launch below with the
            // off-diagonal block split over K (595 tiles = 2.01 waves -> 884 tiles ~3 waves)
            GemmArgs hd[4];
            int nbk = 0, maxM = 0, maxN = 0;
            const char *skg_env = getenv("SGP_GEMM_STREAMK");
            const bool grouped = c.L.hntiles > 0 && !(skg_env && skg_env[0] == '0');
            const int kh = (c.L.hpart && !grouped) ? ((mp.N / 2) & ~(GM_BK - 1)) : 0;
            auto push = [&](int j1, int j2, int k0, int k1, double *C, int ldc) {
                GemmArgs &g = hd[nbk++];
                g = GemmArgs{};
                g.M = mp.D[j1];
                g.N = mp.D[j2];
                g.K = k1 - k0;
                g.A = c.L.M.phis + (size_t)k0 * mp.Dp + (j1 ? mp.Dp0 : 0);
                g.lda = mp.Dp;
                g.TA = 1;
                g.B = c.L.M.phis + (size_t)k0 * mp.Dp + (j2 ? mp.Dp0 : 0);
                g.ldb = mp.Dp;
                g.scale = c.L.S + (size_t)fields[j1 + j2] * mp.ld + k0;
                g.C = C;
                g.ldc = ldc;
                g.alpha = c.tau;
                g.upper_only = j1 == j2;
                g.a16 = (g.lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0);
                g.b16 = (g.ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(g.B) & 15) == 0);
                maxM = std::max(maxM, g.M);
                maxN = std::max(maxN, g.N);
            };
            bool split = false;
            if (grouped) {  // descriptor order = the tile list's (j1 <= j2)
                for (int j1 = 0; j1 < mp.J; ++j1)
                    for (int j2 = j1; j2 < mp.J; ++j2)
                        push(j1, j2, 0, mp.N, c.L.H + (size_t)mp.fstart[j1] * d + mp.fstart[j2], d);
            } else {
                for (int j = 0; j < mp.J; ++j)
                    push(j, j, 0, mp.N, c.L.H + (size_t)mp.fstart[j] * d + mp.fstart[j], d);
                split = mp.J == 2 && kh > 0;
                if (mp.J == 2) {
                    push(0, 1, 0, split ? kh : mp.N, c.L.H + (size_t)mp.fstart[0] * d + mp.fstart[1], d);
                    if (split) push(0, 1, kh, mp.N, c.L.hpart, mp.D[1]);
                }
            }
            // all blocks share TA/TB; the alignment flags agree (same Phi buffer, same ld)
            cudaMemcpyAsync(c.L.hdesc, hd, sizeof(GemmArgs) * nbk, cudaMemcpyHostToDevice, c.s);
            if (!(grouped && gemm_launch_skg<1, 0>(c.L.hdesc, c.L.htiles, c.L.hprefix, c.L.hntiles, c.s)))
                gemm_launch_batched<1, 0>(c.L.hdesc, nbk, maxM, maxN, c.s);
            for (int j1 = 0; j1 < mp.J; ++j1)
                for (int j2 = j1; j2 < mp.J; ++j2) {
                    if (j1 == j2)
                        k_lg_mirror_block<<<lg_blocks((size_t)mp.D[j1] * mp.D[j1]), 256, 0, c.s>>>(
                            c.L.H, d, mp.fstart[j1], mp.D[j1]);
                    else if (split)
                        k_lg_addt_block<<<dim3((mp.D[j2] + 31) / 32, (mp.D[j1] + 31) / 32), dim3(32, 8), 0, c.s>>>(
                            c.L.H, d, mp.fstart[j1], mp.fstart[j2], mp.D[j1], mp.D[j2], c.L.hpart, mp.D[j2]);
                    else
                        k_lg_transpose_block<<<lg_blocks((size_t)mp.D[j1] * mp.D[j2]), 256, 0, c.s>>>(
                            c.L.H, d, mp.fstart[j1], mp.fstart[j2], mp.D[j1], mp.D[j2]);
                }
        }
        lg_op(c, LG_STATE, 0, qv, 0, SGP_EVAL_HESSIAN | SGP_EVAL_HPRIOR | SGP_EVAL_REUSE);
        k_lg_finite<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.H, (size_t)d * d, c.L.status);
    }
    return lg_sync(c);
}

// W = Psi_slot (diag r - (b b^T) o T) Psi_slot^T, b from vec[pv]
static void lg_contraction(LgCtx &c, int slot, int pv) {
    const int d = c.d;
    lg_tvec(c, slot, c.L.vec + (size_t)pv * d, 0, c.L.vec + (size_t)V_BV * d);
    k_lg_mmat<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L, slot, c.cfg.kappa, -1.0, 1, 1);
    lg_gemm(c, d, d, d, c.L.P[slot], d, 0, c.L.W, d, 0, nullptr, c.L.X, d, 1.0, 0);  // X = Psi M
    lg_gemm(c, d, d, d, c.L.X, d, 0, c.L.P[slot], d, 1, nullptr, c.L.W, d, 1.0, 1);  // W = X Psi^T
    mirror_upper(c.L.W, d, d, c.s);
}

// t (vec TV) = tr(W dH/dq) at vec[qv]; per-sample derivatives already in S
static int lg_trace(LgCtx &c, int qv) {
    const ModelParams &mp = c.L.M.mp;
    const int d = c.d;
    if (c.tau != 0.0 && mp.lik != SGP_LIK_QUADRATIC) {
        for (int j1 = 0; j1 < mp.J; ++j1) {
            const double *a = c.L.M.phis + (j1 ? mp.Dp0 : 0);
            const double *b = c.L.W + (size_t)mp.fstart[j1] * d;
            if (j1 == 1)  // Y_1 over block 1's columns only: the (1,0) block repeats (0,1) (W symmetric)
                lg_gemm(c, mp.N, mp.D[1], mp.D[1], a, mp.Dp, 0, b + mp.fstart[1], d, 0, nullptr, c.L.Y + mp.D[0],
                        mp.Dtot, 1.0, 0);
            else
                lg_gemm(c, mp.N, mp.Dtot, mp.D[j1], a, mp.Dp, 0, b, d, 0, nullptr, c.L.Y, mp.Dtot, 1.0, 0);
            k_lg_rowdot<<<lg_blocks((size_t)mp.N * 32), 256, 0, c.s>>>(c.L, j1, j1 == mp.J - 1);
        }
        k_lg_project<<<lg_blocks((size_t)mp.Dtot * 32), 256, 0, c.s>>>(c.L, c.tau, F_C0, F_C1,
                                                                      c.L.vec + (size_t)V_TV * d);
    } else {
        k_lg_zero<<<lg_blocks(d), 256, 0, c.s>>>(c.L.vec + (size_t)V_TV * d, d);
    }
    lg_op(c, LG_TRACE, 0, qv);
    return lg_sync(c);
}

static double lg_hnorm(LgCtx &c) {
    // ||H||_F^2 as per-block partials and one ordered sum (deterministic)
    const int nb = 148 * 2;
    k_bj_sumsq<<<nb, 256, 0, c.s>>>(c.L.H, (size_t)c.d * c.d, c.L.bjPart);
    k_bj_sum_final<<<1, 32, 0, c.s>>>(c.L.bjPart, nb, c.L.sc + 8);
    lg_sync(c);
    return sqrt(c.sc[8]);
}

// Block Jacobi of H (symmetric) with V = P_dst on entry (identity when cold):
// on exit H's diagonal holds the eigenvalues and P_dst the eigenvectors.
static int lg_jacobi_block(LgCtx &c, int dst, double tol, double skip, int *sweeps) {
    const int d = c.d, dp = c.L.bj_dp, nbk = c.L.bj_nbk, np = nbk / 2;
    // P_dst holds the starting basis (identity when cold, the previous basis when warm)
    k_bj_in<<<lg_blocks((size_t)dp * dp), 256, 0, c.s>>>(c.L.bjA, c.L.bjV[0], c.L.H, c.L.P[dst], d, dp, 0);
    static bool configured = false;
    static int inner_cap = 1;
    if (!configured) {
        cudaFuncSetAttribute(k_bj_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BJ_SMEM);
        const char *e = getenv("SGP_BJ_INNER");  // inner sweeps per pair subproblem (tuning)
        if (e && atoi(e) > 0) inner_cap = atoi(e);
        configured = true;
    }
    // Two streams per round: the A chain (pair solve -> column update -> row update -> fix)
    // runs on a high-priority stream; the eigenvector update V' = V U, which nothing in the
    // chain reads, runs on the caller's stream and overlaps the next round's pair solve
    // (np CTAs, a fraction of the SMs).  U is double-buffered by round parity.
    static bool overlap_env = true, overlap_read = false;
    if (!overlap_read) {
        const char *e = getenv("SGP_BJ_OVERLAP");  // 0: everything on the caller's stream (A/B timing)
        overlap_env = !(e && e[0] == '0');
        overlap_read = true;
    }
    const bool overlap = overlap_env && c.L.bj_hs;
    cudaStream_t hs = c.L.bj_hs;
    const cudaEvent_t ev_in = c.L.bj_ev[0], ev_solved = c.L.bj_ev[1], ev_chain = c.L.bj_ev[2];
    const cudaEvent_t ev_v[2] = {c.L.bj_ev[3], c.L.bj_ev[4]};
    cudaStream_t as = overlap ? hs : c.s;
    int vcur = 0, sw = 0;
    const size_t per_round = (size_t)4 * np;
    const size_t ubuf = (size_t)np * BJ_N * BJ_N;
    const int nb_part = 148 * 2;
    for (;;) {
        k_bj_offnorm<<<nb_part, 256, 0, c.s>>>(c.L.bjA, dp, c.L.bjPart);
        k_bj_offnorm_final<<<1, 32, 0, c.s>>>(c.L.bjPart, nb_part, c.L.sc + 7);
        lg_sync(c);
        if (c.sc[7] <= tol) break;
        if (sw >= c.cfg.sweep_cap) {
            *sweeps = -1;
            return SGP_STATUS_JACOBI;
        }
        if (overlap) {
            cudaEventRecord(ev_in, c.s);
            cudaStreamWaitEvent(hs, ev_in, 0);
        }
        for (int r = 0; r < nbk - 1; ++r) {
            const GemmArgs *D = c.L.bjDesc + (size_t)r * per_round;
            double *Ur = c.L.bjU + (size_t)(r & 1) * ubuf;
            if (overlap) cudaStreamWaitEvent(hs, ev_v[r & 1], 0);  // V update of round r - 2 read Ur
            k_bj_solve<<<np, BJ_SOLVE_NT, BJ_SMEM, as>>>(c.L.bjA, dp, r, nbk, skip, Ur, c.L.bjLam, c.L.bjCnt,
                                                     inner_cap);
            if (overlap) {
                cudaEventRecord(ev_solved, hs);
                cudaStreamWaitEvent(c.s, ev_solved, 0);
            }
            gemm_launch_batched<0, 0>(D, np, dp, BJ_N, as);                              // T = A U (columns)
            gemm_launch_batched<1, 0>(D + np, np, BJ_N, dp, as);                         // A = U^T T (rows)
            gemm_launch_batched<0, 0>(D + (size_t)(vcur ? 3 : 2) * np, np, dp, BJ_N, c.s);  // V' = V U
            if (overlap) cudaEventRecord(ev_v[r & 1], c.s);
            k_bj_fix<<<np, 256, 0, as>>>(c.L.bjA, dp, r, nbk, c.L.bjLam, c.L.bjCnt);
            vcur ^= 1;
        }
        if (overlap) {
            cudaEventRecord(ev_chain, hs);
            cudaStreamWaitEvent(c.s, ev_chain, 0);
        }
        ++sw;
    }
    k_bj_out<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.H, c.L.P[dst], c.L.bjA, c.L.bjV[vcur], d, dp);
    *sweeps = sw;
    return 0;
}

// Jacobi on H with V = P_dst: parallel (grid, round-robin) or reference order (one warp)
static int lg_jacobi(LgCtx &c, int dst, double tol, double skip, bool parallel, int *sweeps) {
    const int d = c.d;
    if (!parallel) {
        // reference pivot order, bit-identical (sgp_jbig.cuh); H is symmetric here
        if (!c.L.jb) return SGP_STATUS_JACOBI;
        const int sw = jb_jacobi(*c.L.jb, c.L.H, c.L.P[dst], d, tol, skip, c.cfg.sweep_cap, c.s);
        if (sw == -2) return SGP_STATUS_JACOBI;
        *sweeps = sw;
        return sw < 0 ? SGP_STATUS_JACOBI : 0;
    }
    const char *sj = getenv("SGP_LG_SCALAR_JACOBI");
    if (!(sj && sj[0] == '1') && c.L.bjA) return lg_jacobi_block(c, dst, tol, skip, sweeps);
    const int m = d + (d & 1), np = m >> 1;
    int sw = 0;
    for (;;) {
        lg_op(c, LG_OFFNORM);
        lg_sync(c);
        if (c.sc[7] <= tol) break;
        if (sw >= c.cfg.sweep_cap) {
            *sweeps = -1;
            return SGP_STATUS_JACOBI;
        }
        for (int r = 0; r < m - 1; ++r) {
            k_lg_jrows<<<np, 256, 0, c.s>>>(c.L.H, d, r, skip, c.L.jprm, c.L.jpairs);
            k_lg_jcols<<<std::min(d, 148 * 8), 256, 0, c.s>>>(c.L.H, c.L.P[dst], d, c.L.jprm, c.L.jpairs);
        }
        ++sw;
    }
    *sweeps = sw;
    return 0;
}

// cold decomposition of H into slot dst (metric.py:112-142)
__global__ void k_lg_set_diag(double *H, const double *lam, int d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        H[(size_t)i * d + i] = lam[i];
}

static int lg_eig_cold(LgCtx &c, int dst, int *sweeps) {
    const int d = c.d;
    if (c.cfg.cold_order == SGP_ORDER_DC && c.L.dc && d <= DC_NMAX) {
        // tridiagonalisation + divide and conquer (sgp_dc.cuh); symmetrises H itself
        double *lam = c.L.vec + (size_t)V_TMP * d;
        if (dc_eigh(*c.L.dc, c.L.H, d, d, lam, c.L.P[dst], d, c.s)) return SGP_STATUS_JACOBI;
        k_lg_set_diag<<<lg_blocks(d), 256, 0, c.s>>>(c.L.H, lam, d);
        *sweeps = 0;
        lg_op(c, LG_GLAM, dst, 0, 0, 0);
        c.since[dst] = 0;
        return lg_sync(c);
    }
    lg_symmetrize(c.L.H, d, c.s);
    const double hnorm = lg_hnorm(c);
    const double tol = c.cfg.zeta * hnorm, skip = d ? tol / d : 0.0;
    k_lg_eye<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.P[dst], d);
    // cold decompositions keep the reference's pivot order unless cold_order says otherwise
    // (the momentum p = Psi (sqrt(g) o z) depends on Psi's column order: SURVEY.md M6)
    const int st = lg_jacobi(c, dst, tol, skip, c.cfg.cold_order == SGP_ORDER_PARALLEL, sweeps);
    if (st) return st;
    lg_op(c, LG_GLAM, dst, 0, 0, 0);
    c.since[dst] = 0;
    return lg_sync(c);
}

// MGS inside one panel of rows [r0, r1) of X = Psi^T (one CTA; rows of the
// earlier panels have already been projected out).
__global__ void __launch_bounds__(1024) k_lg_mgs_panel(double *X, int d, int r0, int r1) {
    __shared__ double red[32];
    __shared__ double nrm;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = r0; i < r1; ++i) {
        double *ri = X + (size_t)i * d;
        double s = 0.0;
        for (int k = threadIdx.x; k < d; k += blockDim.x) s += ri[k] * ri[k];
        s = warp_sum(s);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[w];
            nrm = sqrt(t);
        }
        __syncthreads();
        const double n = nrm;
        if (n == 0.0) continue;  // _jacobi.py:98-99
        for (int k = threadIdx.x; k < d; k += blockDim.x) ri[k] /= n;
        __syncthreads();
        for (int j = i + 1 + warp; j < r1; j += nw) {
            double *rj = X + (size_t)j * d;
            double dot = 0.0;
            for (int k = lane; k < d; k += 32) dot += ri[k] * rj[k];
            dot = warp_sum(dot);
            for (int k = lane; k < d; k += 32) rj[k] -= dot * ri[k];
        }
        __syncthreads();
    }
}

// Blocked Gram-Schmidt of P_slot's columns: rows of X = Psi^T in panels of
// 64; each panel is made orthogonal to all earlier rows by classical
// Gram-Schmidt applied twice (two DMMA GEMM pairs: C = X_p X_prev^T,
// X_p -= C X_prev), then orthonormalised by MGS inside the panel.  For the
// nearly orthonormal bases this re-orthonormalises (_jacobi.py:90-107: every
// 10th warm call), the result equals the column MGS to rounding (the same
// QR factor).  X and W are free at this point.
static void lg_mgs_blocked(LgCtx &c, int slot) {
    const int d = c.d, bs = 64;
    const int nt = (d + 31) / 32;
    const int tgrid = std::min(nt * nt, 148 * 8);
    k_lg_transpose<<<tgrid, dim3(32, 8), 0, c.s>>>(c.L.X, c.L.P[slot], d);
    for (int p0 = 0; p0 < d; p0 += bs) {
        const int pe = std::min(d, p0 + bs), nb = pe - p0;
        double *Xp = c.L.X + (size_t)p0 * d;
        for (int rep = 0; p0 > 0 && rep < 2; ++rep) {
            GemmArgs g{};
            g.M = nb;
            g.N = p0;
            g.K = d;
            g.A = Xp;
            g.lda = d;
            g.B = c.L.X;
            g.ldb = d;
            g.TB = 1;  // B(k, n) = X[n][k]
            g.C = c.L.W;
            g.ldc = p0;
            g.alpha = 1.0;
            gemm_launch(g, c.s);  // C = X_p X_prev^T
            GemmArgs h{};
            h.M = nb;
            h.N = d;
            h.K = p0;
            h.A = c.L.W;
            h.lda = p0;
            h.B = c.L.X;
            h.ldb = d;
            h.C = Xp;
            h.ldc = d;
            h.alpha = -1.0;
            h.beta = 1.0;
            gemm_launch(h, c.s);  // X_p -= C X_prev
        }
        k_lg_mgs_panel<<<1, 1024, 0, c.s>>>(c.L.X, d, p0, pe);
    }
    k_lg_transpose<<<tgrid, dim3(32, 8), 0, c.s>>>(c.L.P[slot], c.L.X, d);
}

// Re-orthonormalisation of P_slot's columns for the non-bit-exact warm orders.  MGS returns
// Q = Psi R^-1 with R the Cholesky factor of G = Psi^T Psi (_jacobi.py:89-107 is the column
// form of that QR).  Warm bases drift from orthonormality only by rounding (|G - I| ~ 1e-13
// after gs_interval calls), so R = I + F + O(|G-I|^2) with F = triu(G - I, 1) + diag(G - I)/2,
// and Q = Psi (I - F) to O(|G-I|^2) ~ 1e-26: two DMMA GEMMs instead of d sequential grid
// steps (48 ms per call at d = 2083).  Falls back to the MGS steps when |G - I| > 1e-6.
__global__ void k_cholqr_m(const double *G, int d, double *M, double *part) {
    __shared__ double red[32];
    double mx = 0.0;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < d^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)d), j = (int)(u_ - (unsigned)i * (unsigned)d);
        const double e = G[idx] - (i == j ? 1.0 : 0.0);
        mx = fmax(mx, fabs(e));
        M[idx] = (i == j) ? 1.0 - 0.5 * e : (i < j ? -e : 0.0);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        part[blockIdx.x] = m;
    }
}
__global__ void k_max_final(const double *part, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < n; ++i) m = fmax(m, part[i]);
        *out = m;
    }
}

static void lg_mgs(LgCtx &c, int slot);

static void lg_cholqr(LgCtx &c, int slot) {
    const int d = c.d;
    const size_t dd = (size_t)d * d;
    double *psi = c.L.P[slot], *G = c.L.bjA, *Mm = c.L.bjT, *Pn = c.L.bjV[0];
    GemmArgs g{};
    g.M = g.N = g.K = d;
    g.A = psi;
    g.lda = d;
    g.TA = 1;
    g.B = psi;
    g.ldb = d;
    g.C = G;
    g.ldc = d;
    g.alpha = 1.0;
    g.upper_only = 1;
    gemm_launch(g, c.s);  // G = Psi^T Psi (upper tiles)
    mirror_upper(G, d, d, c.s);
    k_cholqr_m<<<148, 256, 0, c.s>>>(G, d, Mm, c.L.bjPart);
    k_max_final<<<1, 32, 0, c.s>>>(c.L.bjPart, 148, c.L.sc + 15);
    lg_sync(c);
    if (!(c.sc[15] <= 1e-6)) {
        lg_mgs(c, slot);
        return;
    }
    GemmArgs h{};
    h.M = h.N = h.K = d;
    h.A = psi;
    h.lda = d;
    h.B = Mm;
    h.ldb = d;
    h.C = Pn;
    h.ldc = d;
    h.alpha = 1.0;
    gemm_launch(h, c.s);  // Psi (I - F)
    k_lg_copy<<<lg_blocks(dd), 256, 0, c.s>>>(psi, Pn, dd);
}

// Modified Gram-Schmidt of P_slot's columns (_jacobi.py:90-107) as d grid
// steps on the transposed matrix (rows contiguous); X is free at this point.
static void lg_mgs(LgCtx &c, int slot) {
    const int d = c.d;
    const int nt = (d + 31) / 32;
    const int tgrid = std::min(nt * nt, 148 * 8);
    k_lg_transpose<<<tgrid, dim3(32, 8), 0, c.s>>>(c.L.X, c.L.P[slot], d);
    const size_t smem = (size_t)d * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_lg_mgs_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i <= d; ++i) {
        const int rows = d - 1 - i;
        const int blocks = std::max(1, std::min((rows + 7) / 8, 148 * 4));
        k_lg_mgs_step<<<blocks, 256, smem, c.s>>>(c.L.X, d, i, c.L.sc + 12);
    }
    k_lg_transpose<<<tgrid, dim3(32, 8), 0, c.s>>>(c.L.P[slot], c.L.X, d);
}

// ---- warm decomposition by eigenvector refinement (warm_order = "refine") ----
//
// A warm call starts from the previous basis Psi, which already nearly diagonalises the new
// Hessian (measured at C4: off(Psi^T H Psi) ~ 1e-5 ||H||, every coupling below 4 % of its
// eigenvalue gap; profiles/r2_c4_warm_structure.md).  Instead of Jacobi rounds it applies the
// Ogita-Aishima refinement (Ogita & Aishima 2018, "Iterative refinement for symmetric
// eigenvalue decomposition"), all rotations of a sweep at once through four DMMA GEMMs:
//   S = Psi^T H Psi,  G = Psi^T Psi,  lam_i = s_ii / g_ii,
//   E_ij = (s_ij + lam_j r_ij) / (lam_j - lam_i)  (i != j),  E_ii = r_ii / 2,  r = I - G,
//   Psi <- Psi + Psi E,
// which converges quadratically and keeps Psi orthonormal to rounding (the r terms), so the
// every-gs_interval Gram-Schmidt of the Jacobi path is folded into every iteration.  The stop
// test is the reference's: off(S) <= zeta ||H||_F (metric.py:101-109, 172).  Columns keep their
// order (Psi moves by O(E)), so eigenvalues stay in the warm natural order.  Couplings below
// the reference's skip threshold tol/d are not rotated (only the orthogonality term applies),
// as the Jacobi skips them.  Pairs whose coupling exceeds their gap are still updated: the
// iteration recovers within one or two steps (measured on C4 warm problems with ratios up to
// 1.8, tools/refine_sim.py), orthogonality included.  A coupling 1e3 times its gap, an off-norm
// that stops decreasing, a non-finite value, or more than 8 iterations hand the call to the
// block Jacobi from the same starting basis.
__global__ void k_oa_lam(const double *S, const double *G, int d, double *lam) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        lam[i] = S[(size_t)i * d + i] / G[(size_t)i * d + i];
}
#define OA_NB 592  // k_oa_E blocks (4 per SM): enough loads in flight for the d x d pass
#define OA_ETA 1e3  // a coupling this far above its eigenvalue gap goes to the block Jacobi
#define OA_MAXPAIRS 1024
// off-norm^2 of sym(S) and E (when G is given); partials per CTA: [off2, max ratio of the
// pairs in the first-order regime]; pairs with |s_ij| > OA_ETA |gap| are counted in *npairs
// (the first OA_MAXPAIRS listed in pairs, for diagnostics)
__global__ void k_oa_E(const double *S, const double *G, const double *lam, int d, double *E, double *part,
                       int *pairs = nullptr, int *npairs = nullptr, double skip = 0.0) {
    __shared__ double r0[32], r1[32];
    double off2 = 0.0, mr = 0.0;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < (size_t)d * d;
         idx += (size_t)gridDim.x * blockDim.x) {
        const unsigned u_ = (unsigned)idx;  // idx < d^2 < 2^32: 32-bit division
        const int i = (int)(u_ / (unsigned)d), j = (int)(u_ - (unsigned)i * (unsigned)d);
        if (i == j) {
            if (G) E[idx] = 0.5 * (1.0 - G[idx]);
            continue;
        }
        // S and G arrive mirrored from their upper triangles (k_mirror_upper), so
        // 0.5 (s_ij + s_ji) == s_ij exactly: no strided transposed reads
        const double sij = S[idx];
        off2 += sij * sij;
        if (G) {
            const double rij = -G[idx];
            if (fabs(sij) <= skip) {
                // below the reference's skip threshold (|a_pq| <= tol/d, _jacobi.py:57-58): no
                // rotation, only the orthogonality correction (Ogita-Aishima's clustered case)
                E[idx] = 0.5 * rij;
                continue;
            }
            const double gap = lam[j] - lam[i];
            const double e = (sij + lam[j] * rij) / gap;
            E[idx] = e;
            const double ratio = fabs(sij) / fabs(gap);
            if (pairs && ratio > OA_ETA && !(ratio != ratio) && sij != 0.0) {
                if (i < j) {
                    const int k = atomicAdd(npairs, 1);
                    if (k < OA_MAXPAIRS) {
                        pairs[2 * k] = i;
                        pairs[2 * k + 1] = j;
                    }
                }
            } else {
                mr = (ratio > mr || ratio != ratio) ? ratio : mr;  // NaN propagates
            }
        }
    }
    off2 = warp_sum(off2);
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_down_sync(0xffffffffu, mr, o);
        mr = (v > mr || v != v) ? v : mr;
    }
    if ((threadIdx.x & 31) == 0) {
        r0[threadIdx.x >> 5] = off2;
        r1[threadIdx.x >> 5] = mr;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += r0[w];
            b = (r1[w] > b || r1[w] != r1[w]) ? r1[w] : b;
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}
// one warp: lanes take partials lane, lane+32, ... (fixed order), xor trees (sum; max with NaN
// propagation) give every lane the same totals
__global__ void k_oa_fin(const double *part, int n, double *out) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) {
        a += part[2 * i];
        b = (part[2 * i + 1] > b || part[2 * i + 1] != part[2 * i + 1]) ? part[2 * i + 1] : b;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        const double v = __shfl_xor_sync(0xffffffffu, b, o);
        b = (v > b || v != v) ? v : b;
    }
    if (threadIdx.x == 0) {
        out[0] = sqrt(a);
        out[1] = b;
    }
}
__global__ void k_oa_setdiag(double *H, const double *S, int d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        H[(size_t)i * d + i] = S[(size_t)i * d + i];
}

static void lg_gemm_ab(LgCtx &c, int M, int N, int K, const double *A, int lda, int TA, const double *B, int ldb,
                       int TB, double *C, int ldc, double alpha, double beta, int upper) {
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
    g.upper_only = upper;
    gemm_launch(g, c.s);
}

static int lg_eig_warm_jacobi(LgCtx &c, int src, int dst, int *sweeps);

// out = a + sb b (warm start: natural basis + transferred correction; correction = a - b); with
// older corrections c (and e) the correction is extrapolated over leapfrogs: a + (2b - c) linearly,
// a + (3b - 3c + e) quadratically
__global__ void k_lg_axpb(double *out, const double *a, const double *b, double sb, size_t n,
                          const double *c = nullptr, const double *e = nullptr) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = e ? a[i] + (3.0 * (b[i] - c[i]) + e[i]) : (c ? a[i] + (2.0 * b[i] - c[i]) : a[i] + sb * b[i]);
}

static int lg_eig_refine(LgCtx &c, int src, int dst, int *sweeps) {
    const int d = c.d;
    const size_t dd = (size_t)d * d;
    int since = c.since[src] + 1;
    if (c.cfg.gs_interval && since >= c.cfg.gs_interval) since = 0;  // orthonormality is refined every iteration
    const double hnorm = lg_hnorm(c);  // ||H||_F of the unsymmetrised Hessian (metric.py:172)
    const double tol = c.cfg.zeta * hnorm;
    lg_symmetrize(c.L.H, d, c.s);
    double *psi = c.L.P[dst], *Y = c.L.X, *Sm = c.L.W, *G = c.L.bjA, *E = c.L.bjT, *Pn = c.L.bjV[0];
    double *lam = c.L.vec + (size_t)V_TMP * d;  // scratch d-vector (free during the eigensolver)
    const int wi = c.warm_idx;
    if (wi >= 0 && wi < LG_NCORR && c.corr_n[wi] > 0 && c.corr_lf[wi][c.corr_cur[wi]] == c.lf_count - 1) {
        // start from the natural basis plus the correction this call made in the previous leapfrog,
        // extrapolated linearly when two are stored (the fixed-point iterates move smoothly along
        // the trajectory)
        // extrapolation order per call (measured at C4): the first call moves a whole step and
        // takes the quadratic fit, the second the linear one; later calls' corrections are tiny
        // and noisy, extrapolating them only amplifies the noise
        static const int max_order = getenv("SGP_REFINE_TRANSFER") ? atoi(getenv("SGP_REFINE_TRANSFER")) : 3;
        const int want = std::min(max_order, wi == 0 ? 3 : (wi == 1 ? 2 : 1));
        const int cur = c.corr_cur[wi], p1 = (cur + 2) % 3, p2 = (cur + 1) % 3;
        const bool two = want >= 2 && c.corr_n[wi] >= 2 && c.corr_lf[wi][p1] == c.lf_count - 2;
        const bool three = two && want >= 3 && c.corr_n[wi] >= 3 && c.corr_lf[wi][p2] == c.lf_count - 3;
        k_lg_axpb<<<lg_blocks(dd), 256, 0, c.s>>>(psi, c.L.P[src], c.L.Dcorr[wi][cur], 1.0, dd,
                                                   two ? c.L.Dcorr[wi][p1] : nullptr,
                                                   three ? c.L.Dcorr[wi][p2] : nullptr);
    } else {
        k_lg_copy<<<lg_blocks(dd), 256, 0, c.s>>>(psi, c.L.P[src], dd);
    }
    const int nb = OA_NB;  // two partials per CTA in bjPart
    double prev_off = INFINITY;
    for (int it = 0;; ++it) {
        lg_gemm_ab(c, d, d, d, c.L.H, d, 0, psi, d, 0, Y, d, 1.0, 0.0, 0);  // Y = H Psi
        lg_gemm_ab(c, d, d, d, psi, d, 1, Y, d, 0, Sm, d, 1.0, 0.0, 1);     // S = Psi^T Y (upper tiles)
        mirror_upper(Sm, d, d, c.s);
        k_oa_E<<<nb, 256, 0, c.s>>>(Sm, nullptr, nullptr, d, nullptr, c.L.bjPart);
        k_oa_fin<<<1, 32, 0, c.s>>>(c.L.bjPart, nb, c.L.sc + 13);
        lg_sync(c);
        const double off = c.sc[13];
        if (getenv("SGP_DEBUG_REFINE")) fprintf(stderr, "refine it %d off %.3e tol %.3e\n", it, off, tol);
        if (it == 0 && getenv("SGP_DUMP_REFINE")) {  // diagnostics: the warm problem of this call
            static int dumped = 0;
            std::vector<double> hS(dd);
            cudaMemcpyAsync(hS.data(), Sm, sizeof(double) * dd, cudaMemcpyDeviceToHost, c.s);
            cudaStreamSynchronize(c.s);
            char path[512];
            snprintf(path, sizeof(path), "%s_%d.bin", getenv("SGP_DUMP_REFINE"), dumped++);
            if (dumped <= 12) {
                FILE *f = fopen(path, "wb");
                if (f) {
                    fwrite(&tol, sizeof(double), 1, f);
                    fwrite(hS.data(), sizeof(double), dd, f);
                    fclose(f);
                }
            }
        }
        if (off <= tol) {
            k_oa_setdiag<<<lg_blocks(d), 256, 0, c.s>>>(c.L.H, Sm, d);
            *sweeps = it;
            lg_op(c, LG_GLAM, dst, 0, 0, since);
            c.since[dst] = since;
            return lg_sync(c);
        }
        // quadratic convergence or hand over: non-finite, not decreasing, or too many iterations
        // (SGP_REFINE_MAX_ITERS: test hook forcing the hand-over)
        const char *mi = getenv("SGP_REFINE_MAX_ITERS");
        const int max_it = mi ? atoi(mi) : 8;
        if (!(off < prev_off) || it >= std::min(c.cfg.sweep_cap, max_it)) break;
        prev_off = off;
        lg_gemm_ab(c, d, d, d, psi, d, 1, psi, d, 0, G, d, 1.0, 0.0, 1);  // G = Psi^T Psi (upper tiles)
        mirror_upper(G, d, d, c.s);
        k_oa_lam<<<lg_blocks(d), 256, 0, c.s>>>(Sm, G, d, lam);
        int *pairs = c.L.jpairs, *npairs = c.L.jpairs + 2 * OA_MAXPAIRS;
        cudaMemsetAsync(npairs, 0, sizeof(int), c.s);
        k_oa_E<<<nb, 256, 0, c.s>>>(Sm, G, lam, d, E, c.L.bjPart, pairs, npairs, tol / d);
        int np_h = 0;
        cudaMemcpyAsync(&np_h, npairs, sizeof(int), cudaMemcpyDeviceToHost, c.s);
        lg_sync(c);
        if (np_h > 0) break;  // a (numerically) degenerate coupled pair: the Jacobi handles it
        k_lg_copy<<<lg_blocks(dd), 256, 0, c.s>>>(Pn, psi, dd);
        lg_gemm_ab(c, d, d, d, psi, d, 0, E, d, 0, Pn, d, 1.0, 1.0, 0);  // Psi + Psi E
        k_lg_copy<<<lg_blocks(dd), 256, 0, c.s>>>(psi, Pn, dd);
    }
    // hand over: a full decomposition of the symmetric Hessian by tridiagonalisation + divide
    // and conquer (sgp_dc.cuh, ~30 ms at d = 2083), or with SGP_REFINE_FALLBACK=jacobi the block
    // Jacobi from the original basis
    const char *fb = getenv("SGP_REFINE_FALLBACK");
    if (!(fb && strcmp(fb, "jacobi") == 0) && c.L.dc && d <= DC_NMAX) {
        if (getenv("SGP_DEBUG_REFINE")) fprintf(stderr, "refine -> divide-and-conquer fallback\n");
        c.basis_reset = true;  // new column order: no correction transfer across this call
        if (dc_eigh(*c.L.dc, c.L.H, d, d, lam, c.L.P[dst], d, c.s)) return SGP_STATUS_JACOBI;
        k_lg_set_diag<<<lg_blocks(d), 256, 0, c.s>>>(c.L.H, lam, d);
        *sweeps = std::min(c.cfg.sweep_cap, 8) + 1;
        lg_op(c, LG_GLAM, dst, 0, 0, 0);
        c.since[dst] = 0;
        return lg_sync(c);
    }
    if (getenv("SGP_DEBUG_REFINE")) fprintf(stderr, "refine -> block Jacobi fallback\n");
    c.basis_reset = true;
    return lg_eig_warm_jacobi(c, src, dst, sweeps);
}

// warm decomposition of H in P_src's basis into slot dst (metric.py:145-185)
static int lg_eig_warm(LgCtx &c, int src, int dst, int *sweeps) {
    if (c.cfg.warm_order == SGP_ORDER_REFINE) return lg_eig_refine(c, src, dst, sweeps);
    return lg_eig_warm_jacobi(c, src, dst, sweeps);
}

static int lg_eig_warm_jacobi(LgCtx &c, int src, int dst, int *sweeps) {
    const int d = c.d;
    int since = c.since[src] + 1;
    if (c.cfg.gs_interval && since >= c.cfg.gs_interval) {
        if (c.cfg.warm_order == SGP_ORDER_CYCLIC) {
            // the reference's column MGS, d grid steps (bit-faithful order of operations;
            // measured faster at d = 2083 than the blocked form)
            const char *e = getenv("SGP_LG_BLOCK_MGS");
            if (e && e[0] == '1')
                lg_mgs_blocked(c, src);
            else
                lg_mgs(c, src);
        } else {
            lg_cholqr(c, src);  // same Q to rounding, two DMMA GEMMs instead of d grid steps
        }
        since = 0;
    }
    const double hnorm = lg_hnorm(c);
    lg_gemm(c, d, d, d, c.L.P[src], d, 1, c.L.H, d, 0, nullptr, c.L.X, d, 1.0, 0);  // X = Psi^T H
    lg_gemm(c, d, d, d, c.L.X, d, 0, c.L.P[src], d, 0, nullptr, c.L.H, d, 1.0, 0);  // A = X Psi
    lg_symmetrize(c.L.H, d, c.s);
    k_lg_copy<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.P[dst], c.L.P[src], (size_t)d * d);
    const double tol = c.cfg.zeta * hnorm, skip = d ? tol / d : 0.0;
    const int st = lg_jacobi(c, dst, tol, skip, c.cfg.warm_order != SGP_ORDER_CYCLIC, sweeps);
    if (st) return st;
    lg_op(c, LG_GLAM, dst, 0, 0, since);
    c.since[dst] = since;
    return lg_sync(c);
}

// one generalized leapfrog (sampler.py:209-258); frame: vec Q0, GRAD, S, slot f
static int lg_leapfrog(LgCtx &c, int &f, int *fp_p, int *fp_q, double *sweep_sum, int *sweep_cnt, int *sweep_log) {
    const int d = c.d;
    const double eps = c.cfg.epsilon;
    int st;
    lg_contraction(c, f, V_P);
    if ((st = lg_trace(c, V_Q0))) return st;
    lg_op(c, LG_PHALF, 0, 0, V_PH, 0, eps);
    bool conv = false;
    for (int it = 0; it < c.cfg.fp_max_iters; ++it) {
        lg_contraction(c, f, V_PH);
        if ((st = lg_trace(c, V_Q0))) return st;
        lg_op(c, LG_PHALF, 0, 0, V_PN, 1, eps);
        cudaMemcpyAsync(c.L.vec + (size_t)V_PH * d, c.L.vec + (size_t)V_PN * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, c.s);
        lg_sync(c);
        if (c.sc[5] <= c.cfg.fp_tol) {
            conv = true;
            if (fp_p) *fp_p = it + 1;
            break;
        }
    }
    if (!conv) return SGP_STATUS_STALL_P;
    lg_apply_g(c, f, V_PH, V_V0, 0);
    // qc = q0 + eps v0 (QDELTA with the roles shifted: use tmp = v0 -> qn = q0 + eps v0)
    cudaMemcpyAsync(c.L.vec + (size_t)V_TMP * d, c.L.vec + (size_t)V_V0 * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    lg_op(c, LG_QDELTA, 0, 0, 0, 0, 2.0 * eps / 2.0 * 1.0);  // qn = q0 + 0.5*eps*(v0 + v0)
    cudaMemcpyAsync(c.L.vec + (size_t)V_QC * d, c.L.vec + (size_t)V_QN * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    int prev = f, cur = f;
    conv = false;
    static const bool transfer_on = !(getenv("SGP_REFINE_TRANSFER") && getenv("SGP_REFINE_TRANSFER")[0] == '0');
    const bool transfer = transfer_on && c.cfg.metric == SGP_METRIC_DYNAMIC && c.cfg.warm_order == SGP_ORDER_REFINE;
    for (int it = 0; it < c.cfg.fp_max_iters; ++it) {
        if ((st = lg_state(c, V_QC, SGP_EVAL_HESSIAN))) return st;
        const int nxt = 1 - prev;
        int sw = 0;
        c.warm_idx = transfer ? it : -1;
        c.basis_reset = false;
        st = c.cfg.metric == SGP_METRIC_STATIC ? lg_eig_cold(c, nxt, &sw) : lg_eig_warm(c, prev, nxt, &sw);
        c.warm_idx = -1;
        if (transfer && it < LG_NCORR) {
            if (c.basis_reset) {  // a hand-over changed the column order: drop every stored correction
                for (int k = 0; k < LG_NCORR; ++k) c.corr_n[k] = 0;
            } else {  // this call's correction R - S for the next leapfrog (the older one is kept)
                const int slot = c.corr_n[it] > 0 ? (c.corr_cur[it] + 1) % 3 : c.corr_cur[it];
                k_lg_axpb<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.Dcorr[it][slot], c.L.P[nxt], c.L.P[prev],
                                                                    -1.0, (size_t)d * d);
                c.corr_cur[it] = slot;
                c.corr_lf[it][slot] = c.lf_count;
                c.corr_n[it] = std::min(3, c.corr_n[it] + 1);
            }
        }
        if (sweep_log && it < 32) sweep_log[it] = sw;
        if (st) return st;
        *sweep_sum += sw;
        ++*sweep_cnt;
        cur = nxt;
        lg_apply_g(c, cur, V_PH, V_TMP, 0);
        lg_op(c, LG_QDELTA, 0, 0, 0, 0, eps);
        lg_sync(c);
        if (c.sc[5] <= c.cfg.fp_tol) {
            conv = true;
            if (fp_q) *fp_q = it + 1;
            break;
        }
        cudaMemcpyAsync(c.L.vec + (size_t)V_QC * d, c.L.vec + (size_t)V_QN * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, c.s);
        prev = cur;
    }
    if (!conv) return SGP_STATUS_STALL_Q;
    f = cur;
    ++c.lf_count;
    lg_contraction(c, f, V_PH);
    if ((st = lg_state(c, V_QC, SGP_EVAL_GRADIENT | SGP_EVAL_REUSE))) return st;
    if ((st = lg_trace(c, V_QC))) return st;
    // p_new = ph - 0.5 eps (grad + 0.5 tv): PHALF computes p - ..., so stage ph into p first
    cudaMemcpyAsync(c.L.vec + (size_t)V_P * d, c.L.vec + (size_t)V_PH * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    lg_op(c, LG_PHALF, 0, 0, V_P, 0, eps);
    cudaMemcpyAsync(c.L.vec + (size_t)V_Q0 * d, c.L.vec + (size_t)V_QC * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    lg_sync(c);
    return 0;
}

// ---- workspace (one chain at a time; cached per model) ----------------------

// d > 256 (or very wide designs) take the GEMM path; SGP_FORCE_LARGE=1 routes
// any model through it (used by the parity tests on the golden chains).
// Latency path (ChainConfig.path = "latency", SGP_PATH_LATENCY): each chain's leapfrog runs on
// the whole GPU through the large path (DMMA GEMMs, the grid-wide reference-order Jacobi or the
// refinement) instead of one CTA per chain; chains of the batch run one after the other.
// Measured single-chain ms per leapfrog (tools/latency_single_chain.py, profiles/r2_latency.md),
// one CTA vs latency path: d = 83 cyclic 16.2 / 14.9, parallel 15.1 / 4.6; d = 163 cyclic
// 78 / 24, parallel 75 / 4.3; at d = 34 one CTA is faster (2.7 ms).  Opt-in, because the two
// paths agree with the reference to 1e-9 but not bit for bit with each other, and the default
// keeps a chain's bits independent of the batch it runs in.
// At d <= 64 path="latency" stays on the fused kernel with 256-thread CTAs instead
// (chain_launch): C1 1.96 ms/leapfrog cyclic, 1.07 parallel, vs 4.6 / 3.1 on this path.
#define LG_LATENCY_MIN_D 65
static bool lg_route_latency(const ModelDev &M, const sgp_chain_config &cfg) {
    return cfg.path == SGP_PATH_LATENCY && M.mp.lik != SGP_LIK_QUADRATIC && M.mp.d >= LG_LATENCY_MIN_D;
}

static bool lg_is_large(const ModelDev &M) {
    if (M.mp.lik == SGP_LIK_QUADRATIC) return false;
    const char *f = getenv("SGP_FORCE_LARGE");
    if (f && f[0] == '1') return true;
    return M.mp.d > 256 || M.mp.Dp > 512;
}

static int lg_alloc(const ModelDev &M, LgPtrs &L, void **owner) {
    const int d = M.mp.d, ld = M.mp.ld;
    const size_t dd = (size_t)d * d;
    const size_t np = (size_t)(d + 1) / 2 + 1;
    size_t off = 0;
    auto take = [&](size_t n) {
        size_t o = off;
        off += (n + 3) & ~size_t(3);
        return o;
    };
    const size_t oS = take((size_t)F_COUNT * ld), oH = take(dd), oX = take(std::max(dd, (size_t)LG_TV_KS * d))  /* also the Psi^T v partials */, oW = take(dd), oP0 = take(dd),
                 oP1 = take(dd), oY = take((size_t)std::max(M.mp.N, 1) * std::max(M.mp.Dtot, 1)),
                 osa = take(3 * (size_t)ld), ov = take(16 * (size_t)d), osc = take(16), osi = take(16),
                 ost = take(2), ojl = take(sgp_jacobi_log_doubles(d)), ojp = take(5 * np), ojq = take(std::max(2 * np, (size_t)4096)),  // + refine pair/cluster lists
                
                 ored = take(std::max<size_t>(64, 2 * (size_t)((ld + 31) / 32) + 8));  // k_lg_lik partials
    // block Jacobi
    const int nbk = ((d + 2 * BJ_B - 1) / (2 * BJ_B)) * 2, dp = nbk * BJ_B, bnp = nbk / 2;
    const size_t dpp = (size_t)dp * dp;
    const size_t obA = take(dpp), obT = take(dpp), obV0 = take(dpp), obV1 = take(dpp),
                 obU = take((size_t)2 * bnp * BJ_N * BJ_N), obL = take((size_t)bnp * BJ_N * BJ_N), obP = take(2 * OA_NB + 8),
                 obC = take((size_t)bnp);
    const size_t ndesc = (size_t)(nbk - 1) * 4 * bnp;
    const size_t obD = take((ndesc * sizeof(GemmArgs) + sizeof(double) - 1) / sizeof(double) + 2);
    const size_t ohD = take((4 * sizeof(GemmArgs) + sizeof(double) - 1) / sizeof(double) + 2);
    // grouped stream-K tile list of the likelihood Hessian blocks (j1 <= j2; diagonal blocks upper)
    std::vector<int4> htl;
    std::vector<long> hpf;
    {
        GemmArgs shp[3];
        int nb = 0;
        for (int j1 = 0; j1 < M.mp.J; ++j1)
            for (int j2 = j1; j2 < M.mp.J; ++j2) {
                shp[nb] = GemmArgs{};
                shp[nb].M = M.mp.D[j1];
                shp[nb].N = M.mp.D[j2];
                shp[nb].K = M.mp.N;
                shp[nb].upper_only = j1 == j2;
                ++nb;
            }
        if (M.mp.lik != SGP_LIK_QUADRATIC && M.mp.N > 0) gemm_group_tiles(shp, nb, htl, hpf);
    }
    const size_t oht = take(2 * htl.size() + 2), ohp = take(hpf.size() + 1), odc = take(3 * LG_NCORR * dd);
    const size_t ohp_part = take(M.mp.J == 2 ? (size_t)M.mp.D[0] * M.mp.D[1] : 0);
    double *base = nullptr;
    if (cudaMalloc(&base, off * sizeof(double)) != cudaSuccess) return SGP_ENOMEM;
    cudaMemset(base, 0, off * sizeof(double));
    L.M = M;
    L.S = base + oS;
    L.H = base + oH;
    L.X = base + oX;
    L.W = base + oW;
    L.P[0] = base + oP0;
    L.P[1] = base + oP1;
    L.Y = base + oY;
    L.sacc = base + osa;
    L.vec = base + ov;
    L.sc = base + osc;
    L.si = reinterpret_cast<int *>(base + osi);
    L.status = reinterpret_cast<int *>(base + ost);
    L.jlog = base + ojl;
    L.jprm = base + ojp;
    L.jpairs = reinterpret_cast<int *>(base + ojq);
    L.red = base + ored;
    L.bj_dp = dp;
    L.bj_nbk = nbk;
    L.bjA = base + obA;
    L.bjT = base + obT;
    L.bjV[0] = base + obV0;
    L.bjV[1] = base + obV1;
    L.bjU = base + obU;
    L.bjLam = base + obL;
    L.bjPart = base + obP;
    L.bjCnt = reinterpret_cast<int *>(base + obC);
    L.bjDesc = reinterpret_cast<GemmArgs *>(base + ((obD + 1) & ~size_t(1)));  // 16-byte aligned
    L.hdesc = reinterpret_cast<GemmArgs *>(base + ((ohD + 1) & ~size_t(1)));
    L.hpart = M.mp.J == 2 ? base + ohp_part : nullptr;
    L.htiles = reinterpret_cast<int4 *>(base + ((oht + 1) & ~size_t(1)));
    L.hprefix = reinterpret_cast<long *>(base + ohp);
    for (int k = 0; k < LG_NCORR; ++k)
        for (int h = 0; h < 3; ++h) L.Dcorr[k][h] = base + odc + (3 * k + h) * dd;
    L.hntiles = (int)htl.size();
    if (!htl.empty() && (cudaMemcpy(L.htiles, htl.data(), sizeof(int4) * htl.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
                         cudaMemcpy(L.hprefix, hpf.data(), sizeof(long) * hpf.size(), cudaMemcpyHostToDevice) != cudaSuccess))
        L.hntiles = 0;
    {
        L.bj_hs = nullptr;
        for (cudaEvent_t &e : L.bj_ev) e = nullptr;
        int lo = 0, hi = 0;
        bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess &&
                  cudaStreamCreateWithPriority(&L.bj_hs, cudaStreamNonBlocking, hi) == cudaSuccess;
        for (cudaEvent_t &e : L.bj_ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        if (!ok) lg_free_handles(L);  // no overlap: the block Jacobi then runs on the caller's stream
    }
    {
        std::vector<GemmArgs> desc;
        bj_build_desc(L, desc);
        if (cudaMemcpy(L.bjDesc, desc.data(), desc.size() * sizeof(GemmArgs), cudaMemcpyHostToDevice) != cudaSuccess) {
            lg_free_handles(L);
            cudaFree(base);
            return SGP_ENOMEM;
        }
    }
    L.jb = new JbWS();
    L.dc = new DcWS();
    if (cudaMallocHost(&L.hsync, sizeof(double) * 64) != cudaSuccess) L.hsync = nullptr;
    *owner = base;
    return SGP_OK;
}

// Builds the frame at vec Q0: potential, gradient, S; cold metric in slot 0
// (or resumes from a stored psi/lam when resume != 0).
static int lg_frame(LgCtx &c, bool resume, const double *psi, const double *lam, int since, int &f) {
    const int d = c.d;
    const bool euclid = c.cfg.metric == SGP_METRIC_EUCLIDEAN;
    f = 0;
    if (resume || euclid) {
        int st = lg_state(c, V_Q0, SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT);
        if (st || euclid) return st;
        cudaMemcpyAsync(c.L.P[0], psi, sizeof(double) * d * d, cudaMemcpyDeviceToDevice, c.s);
        // lam -> H diagonal is not needed: load lam into slot 0 directly
        cudaMemcpyAsync(c.L.vec + (size_t)V_LAM0 * d, lam, sizeof(double) * d, cudaMemcpyDeviceToDevice, c.s);
        // g, logdet from lam: reuse GLAM on a diagonal H
        k_lg_zero<<<lg_blocks((size_t)d * d), 256, 0, c.s>>>(c.L.H, (size_t)d * d);

        cudaMemcpy2DAsync(c.L.H, (d + 1) * sizeof(double), lam, sizeof(double), sizeof(double), d,
                          cudaMemcpyDeviceToDevice, c.s);
        lg_op(c, LG_GLAM, 0, 0, 0, since);
        c.since[0] = since;
        return lg_sync(c);
    }
    int st = lg_state(c, V_Q0, SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT | SGP_EVAL_HESSIAN);
    if (st) return st;
    int sw;
    return lg_eig_cold(c, 0, &sw);
}

static void lg_ctx(LgCtx &c, const LgPtrs &L, const sgp_chain_config &cfg, double tau, cudaStream_t s) {
    c.L = L;
    c.s = s;
    c.cfg = cfg;
    c.tau = tau;
    c.d = L.M.mp.d;
    c.since[0] = c.since[1] = 0;
    for (int k = 0; k < LG_NCORR; ++k) c.corr_n[k] = c.corr_cur[k] = 0;
    c.lf_count = 0;
    c.warm_idx = -1;
    c.basis_reset = false;
    memset(c.sc, 0, sizeof(c.sc));
    memset(c.si, 0, sizeof(c.si));
    c.status = 0;
}

static int lg_euclid_leapfrog(LgCtx &c) {
    // p_half = p - eps/2 grad ; q = q0 + eps p_half ; grad at q ; p = p_half - eps/2 grad
    const int d = c.d;
    const double eps = c.cfg.epsilon;
    // reuse PHALF with tv = 0: out = p - 0.5 eps (grad + 0.5*0)
    k_lg_zero<<<lg_blocks(d), 256, 0, c.s>>>(c.L.vec + (size_t)V_TV * d, d);
    lg_op(c, LG_PHALF, 0, 0, V_PH, 0, eps);
    cudaMemcpyAsync(c.L.vec + (size_t)V_V0 * d, c.L.vec + (size_t)V_PH * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    cudaMemcpyAsync(c.L.vec + (size_t)V_TMP * d, c.L.vec + (size_t)V_PH * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    lg_op(c, LG_QDELTA, 0, 0, 0, 0, eps);  // qn = q0 + eps p_half
    cudaMemcpyAsync(c.L.vec + (size_t)V_Q0 * d, c.L.vec + (size_t)V_QN * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    int st = lg_state(c, V_Q0, SGP_EVAL_POTENTIAL | SGP_EVAL_GRADIENT);
    if (st) return st;
    cudaMemcpyAsync(c.L.vec + (size_t)V_P * d, c.L.vec + (size_t)V_PH * d, sizeof(double) * d,
                    cudaMemcpyDeviceToDevice, c.s);
    lg_op(c, LG_PHALF, 0, 0, V_P, 0, eps);
    return lg_sync(c);
}

static double lg_kinetic(LgCtx &c, int f) {
    if (c.cfg.metric == SGP_METRIC_EUCLIDEAN) {
        // 0.5 p.p + 0.5 d ln 2pi via metric_quad with identity is not available: compute on host
        std::vector<double> p(c.d);
        cudaMemcpyAsync(p.data(), c.L.vec + (size_t)V_P * c.d, sizeof(double) * c.d, cudaMemcpyDeviceToHost, c.s);
        cudaStreamSynchronize(c.s);
        double s = 0.0;
        for (double v : p) s += v * v;
        return 0.5 * s + 0.5 * c.d * SGP_LN_2PI;
    }
    lg_tvec(c, f, c.L.vec + (size_t)V_P * c.d, 4, c.L.vec + (size_t)V_BV * c.d);
    k_lg_kinetic_fin<<<1, 32, 0, c.s>>>(c.L.vec + (size_t)V_BV * c.d, c.d, c.L.sc + f, c.L.sc + 6);
    lg_sync(c);
    return c.sc[6];
}

// ---- large-path implementations of the C ABI entry points -------------------

static int lg_chain_init(const LgPtrs &L, const sgp_chain_config *cfg, const sgp_chain_state *st, cudaStream_t s) {
    const int d = L.M.mp.d;
    std::vector<int> status(st->n_chains, 0);
    std::vector<double> tau(st->n_chains);
    cudaMemcpy(tau.data(), st->tau, sizeof(double) * st->n_chains, cudaMemcpyDeviceToHost);
    cudaMemcpy(status.data(), st->status, sizeof(int) * st->n_chains, cudaMemcpyDeviceToHost);
    for (int z = 0; z < st->n_chains; ++z) {
        if (status[z]) continue;
        LgCtx c;
        lg_ctx(c, L, *cfg, tau[z], s);
        lg_clear_status(c);
        cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, st->q + (size_t)z * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, s);
        int f = 0;
        const int rc = lg_frame(c, false, nullptr, nullptr, 0, f);
        status[z] = rc ? SGP_STATUS_CHAIN_START : 0;
        if (!rc && cfg->metric != SGP_METRIC_EUCLIDEAN) {
            cudaMemcpyAsync(st->psi + (size_t)z * d * d, L.P[0], sizeof(double) * d * d, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(st->lam + (size_t)z * d, L.vec + (size_t)V_LAM0 * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
        }
    }
    cudaMemcpyAsync(st->status, status.data(), sizeof(int) * st->n_chains, cudaMemcpyHostToDevice, s);
    std::vector<int> zero(st->n_chains, 0);
    cudaMemcpyAsync(st->since, zero.data(), sizeof(int) * st->n_chains, cudaMemcpyHostToDevice, s);
    return cudaStreamSynchronize(s) == cudaSuccess ? SGP_OK : SGP_ECUDA;
}

static int lg_run_moves(const LgPtrs &L, const sgp_chain_config *cfg, const sgp_chain_state *st, int moves,
                        int move_offset, const double *d_z, const double *d_logu, sgp_move_records *rec,
                        cudaStream_t s) {
    const int d = L.M.mp.d, Z = st->n_chains;
    const bool euclid = cfg->metric == SGP_METRIC_EUCLIDEAN;
    std::vector<int> status(Z), since(Z);
    std::vector<double> tau(Z), logu((size_t)moves * Z);
    cudaMemcpy(tau.data(), st->tau, sizeof(double) * Z, cudaMemcpyDeviceToHost);
    cudaMemcpy(status.data(), st->status, sizeof(int) * Z, cudaMemcpyDeviceToHost);
    cudaMemcpy(since.data(), st->since, sizeof(int) * Z, cudaMemcpyDeviceToHost);
    cudaMemcpy(logu.data(), d_logu, sizeof(double) * moves * Z, cudaMemcpyDeviceToHost);
    const size_t R = (size_t)moves * Z;
    std::vector<double> lp(R), hb(R), ha(R), sm(R), wall(R);
    std::vector<uint8_t> acc(R), dv(R);
    for (int z = 0; z < Z; ++z) {
        if (status[z]) continue;
        LgCtx c;
        lg_ctx(c, L, *cfg, tau[z], s);
        lg_clear_status(c);
        cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, st->q + (size_t)z * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, s);
        int f = 0;
        if (lg_frame(c, true, st->psi + (size_t)z * d * d, st->lam + (size_t)z * d, since[z], f)) {
            status[z] = SGP_STATUS_CHAIN_START;
            continue;
        }
        int final_status = 0;
        for (int mv = 0; mv < moves; ++mv) {
            const auto t0 = std::chrono::steady_clock::now();
            const double *zz = d_z + ((size_t)mv * Z + z) * d;
            if (euclid) {
                cudaMemcpyAsync(L.vec + (size_t)V_P * d, zz, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
            } else {
                cudaMemcpyAsync(L.vec + (size_t)V_PN * d, zz, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
                lg_apply_g(c, f, V_PN, V_P, 2);
            }
            lg_sync(c);
            const double pot_before = c.sc[2];
            const double h_before = pot_before + lg_kinetic(c, f);
            cudaMemcpyAsync(L.vec + (size_t)V_QS * d, L.vec + (size_t)V_Q0 * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
            double sweep_sum = 0.0;
            int sweep_cnt = 0;
            int fr = f, ls = 0;
            for (int k = 0; k < LG_NCORR; ++k) c.corr_n[k] = 0;  // a new momentum: nothing to transfer
            for (int l = 0; l < cfg->leapfrogs && !ls; ++l)
                ls = euclid ? lg_euclid_leapfrog(c) : lg_leapfrog(c, fr, nullptr, nullptr, &sweep_sum, &sweep_cnt,
                                                                   nullptr);
            bool div = ls != 0;
            double h_after = NAN;
            if (!div) {
                lg_sync(c);
                h_after = c.sc[2] + lg_kinetic(c, fr);
                if (!std::isfinite(h_after)) div = true;
            }
            if (div) h_after = NAN;
            const size_t ri = (size_t)mv * Z + z;
            const bool accept = !div && (h_before - h_after) > logu[ri];
            lg_clear_status(c);
            if (accept) {
                f = fr;
            } else if (div && mv + move_offset == 0) {
                final_status = SGP_STATUS_FIRST_MOVE;
            } else {
                cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, L.vec + (size_t)V_QS * d, sizeof(double) * d,
                                cudaMemcpyDeviceToDevice, s);
                const int rs = lg_frame(c, false, nullptr, nullptr, 0, f);  // cold resync
                if (rs) final_status = rs;
            }
            lg_sync(c);
            lp[ri] = -c.sc[2];
            hb[ri] = h_before;
            ha[ri] = h_after;
            acc[ri] = accept;
            dv[ri] = div;
            sm[ri] = sweep_cnt ? sweep_sum / sweep_cnt : 0.0;
            wall[ri] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (rec->q)
                cudaMemcpyAsync(rec->q + ri * d, L.vec + (size_t)(final_status ? V_QS : V_Q0) * d,
                                sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
            if (final_status) break;
        }
        cudaMemcpyAsync(st->q + (size_t)z * d, L.vec + (size_t)V_Q0 * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, s);
        if (!euclid && !final_status) {
            cudaMemcpyAsync(st->psi + (size_t)z * d * d, L.P[f], sizeof(double) * d * d, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(st->lam + (size_t)z * d, L.vec + (size_t)(V_LAM0 + f) * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
            since[z] = c.since[f];
        }
        status[z] = final_status;
    }
    cudaMemcpyAsync(rec->logpost, lp.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->h_before, hb.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->h_after, ha.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->sweeps_mean, sm.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->wall_ms, wall.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->accept, acc.data(), R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(rec->divergent, dv.data(), R, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(st->status, status.data(), sizeof(int) * Z, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(st->since, since.data(), sizeof(int) * Z, cudaMemcpyHostToDevice, s);
    return cudaStreamSynchronize(s) == cudaSuccess ? SGP_OK : SGP_ECUDA;
}

static int lg_leapfrog_api(const LgPtrs &L, const sgp_chain_config *cfg, const sgp_chain_state *st, double *d_p,
                           sgp_leapfrog_diag *diag, cudaStream_t s) {
    const int d = L.M.mp.d, Z = st->n_chains;
    std::vector<double> tau(Z);
    std::vector<int> since(Z), status(Z, 0);
    cudaMemcpy(tau.data(), st->tau, sizeof(double) * Z, cudaMemcpyDeviceToHost);
    cudaMemcpy(since.data(), st->since, sizeof(int) * Z, cudaMemcpyDeviceToHost);
    for (int z = 0; z < Z; ++z) {
        LgCtx c;
        lg_ctx(c, L, *cfg, tau[z], s);
        lg_clear_status(c);
        cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, st->q + (size_t)z * d, sizeof(double) * d,
                        cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(L.vec + (size_t)V_P * d, d_p + (size_t)z * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
        int f = 0, fp_p = 0, fp_q = 0, cnt = 0, slog[32];
        double ssum = 0.0;
        for (int k = 0; k < 32; ++k) slog[k] = -1;
        int rc = lg_frame(c, true, st->psi + (size_t)z * d * d, st->lam + (size_t)z * d, since[z], f);
        if (!rc)
            rc = cfg->metric == SGP_METRIC_EUCLIDEAN ? lg_euclid_leapfrog(c)
                                                     : lg_leapfrog(c, f, &fp_p, &fp_q, &ssum, &cnt, slog);
        status[z] = rc;
        if (!rc) {
            cudaMemcpyAsync(st->q + (size_t)z * d, L.vec + (size_t)V_Q0 * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(d_p + (size_t)z * d, L.vec + (size_t)V_P * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
            if (cfg->metric != SGP_METRIC_EUCLIDEAN) {
                cudaMemcpyAsync(st->psi + (size_t)z * d * d, L.P[f], sizeof(double) * d * d, cudaMemcpyDeviceToDevice,
                                s);
                cudaMemcpyAsync(st->lam + (size_t)z * d, L.vec + (size_t)(V_LAM0 + f) * d, sizeof(double) * d,
                                cudaMemcpyDeviceToDevice, s);
                since[z] = c.since[f];
            }
        }
        if (diag) {
            if (diag->fp_p_iters) cudaMemcpyAsync(diag->fp_p_iters + z, &fp_p, sizeof(int), cudaMemcpyHostToDevice, s);
            if (diag->fp_q_iters) cudaMemcpyAsync(diag->fp_q_iters + z, &fp_q, sizeof(int), cudaMemcpyHostToDevice, s);
            if (diag->sweeps)
                cudaMemcpyAsync(diag->sweeps + (size_t)z * cfg->fp_max_iters, slog, sizeof(int) * cfg->fp_max_iters,
                                cudaMemcpyHostToDevice, s);
            cudaStreamSynchronize(s);
        }
    }
    cudaMemcpyAsync(st->status, status.data(), sizeof(int) * Z, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(st->since, since.data(), sizeof(int) * Z, cudaMemcpyHostToDevice, s);
    return cudaStreamSynchronize(s) == cudaSuccess ? SGP_OK : SGP_ECUDA;
}

static int lg_eval_api(const LgPtrs &L, int Z, const double *d_tau, const double *d_q, int what, double *d_pot,
                       double *d_grad, double *d_hess, double *d_sumpot, int *d_status, cudaStream_t s) {
    const int d = L.M.mp.d;
    std::vector<double> tau(Z);
    cudaMemcpy(tau.data(), d_tau, sizeof(double) * Z, cudaMemcpyDeviceToHost);
    sgp_chain_config cfg{};
    for (int z = 0; z < Z; ++z) {
        LgCtx c;
        lg_ctx(c, L, cfg, tau[z], s);
        lg_clear_status(c);
        cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, d_q + (size_t)z * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
        const int rc = lg_state(c, V_Q0, what);
        if (d_pot) cudaMemcpyAsync(d_pot + z, L.sc + 2, sizeof(double), cudaMemcpyDeviceToDevice, s);
        if (d_sumpot) cudaMemcpyAsync(d_sumpot + z, L.sc + 3, sizeof(double), cudaMemcpyDeviceToDevice, s);
        if (d_grad && (what & SGP_EVAL_GRADIENT))
            cudaMemcpyAsync(d_grad + (size_t)z * d, L.vec + (size_t)V_GRAD * d, sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s);
        if (d_hess && (what & SGP_EVAL_HESSIAN))
            cudaMemcpyAsync(d_hess + (size_t)z * d * d, L.H, sizeof(double) * d * d, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(d_status + z, &rc, sizeof(int), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
    }
    return SGP_OK;
}

static int lg_trace_api(const LgPtrs &L, int Z, const double *d_tau, const double *d_q, const double *d_w,
                        double *d_t, int *d_status, cudaStream_t s) {
    const int d = L.M.mp.d;
    std::vector<double> tau(Z);
    cudaMemcpy(tau.data(), d_tau, sizeof(double) * Z, cudaMemcpyDeviceToHost);
    sgp_chain_config cfg{};
    for (int z = 0; z < Z; ++z) {
        LgCtx c;
        lg_ctx(c, L, cfg, tau[z], s);
        lg_clear_status(c);
        cudaMemcpyAsync(L.vec + (size_t)V_Q0 * d, d_q + (size_t)z * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
        int rc = lg_state(c, V_Q0, 0);
        if (!rc) {
            cudaMemcpyAsync(L.W, d_w + (size_t)z * d * d, sizeof(double) * d * d, cudaMemcpyDeviceToDevice, s);
            lg_symmetrize(L.W, d, c.s);
            rc = lg_trace(c, V_Q0);
        }
        cudaMemcpyAsync(d_t + (size_t)z * d, L.vec + (size_t)V_TV * d, sizeof(double) * d, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(d_status + z, &rc, sizeof(int), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
    }
    return SGP_OK;
}
