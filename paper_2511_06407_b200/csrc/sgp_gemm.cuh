// sgp_gemm.cuh — FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) GEMM for the
// large-d path (d = 2083, N = 8192).
//
//   C[m][n] = alpha * sum_k A(m,k) * s(k) * B(k,n) + beta * C[m][n]
//   A(m,k) = TA ? A[k*lda + m] : A[m*lda + k],  B(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n]
//   s(k) = scale ? scale[k] : 1   (diag(tau d2) of the likelihood Hessian)
//
// tcgen05 has no f64 kind; DMMA is the only FP64 tensor path on sm_100a and
// measures 37.1 TF/s vs 34.3 TF/s for DFMA on B200 (profiles/r1_microbench.md).
// CTA tile 64 x 64 x 32, 4 warps each owning a 32 x 32 sub-tile = 4 x 4 DMMA
// fragments (32 accumulator doubles per thread).  Operand tiles keep their
// global layout in shared memory so a 3-stage cp.async pipeline stages them
// with 16-byte copies; row strides are padded by 4 doubles, which makes every
// fragment load bank-conflict free.  Requires lda, ldb, ldc multiples of 2 and
// 16-byte aligned bases (the large-path buffers are allocated that way).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <vector>

#define GM_BK 32

// CTA tile configurations.  Big: 128 x 64 tile, 2 x 2 warps of 64 x 32 (8 x 4 DMMA fragments,
// 64 accumulator doubles per thread), 2 stages -- more independent DMMAs per warp and half
// the operand traffic per flop (+16 % on d^3 at d = 2083, measured with tools/gemm_bench.cu).
// Small: 64 x 64, 2 x 2 warps of 32 x 32, 3 stages, for outputs with too few big tiles to
// fill the GPU (the 1040 x 1040 Hessian blocks, the block-Jacobi 64 x 64 updates).
struct GmSmall {
    static constexpr int BM = 64, BN = 64, WARPS_M = 2, WARPS_N = 2, STAGES = 3;
};
struct GmBig {
    static constexpr int BM = 128, BN = 64, WARPS_M = 2, WARPS_N = 2, STAGES = 2;
};
template <class CFG>
struct GmGeo {
    static constexpr int THREADS = 32 * CFG::WARPS_M * CFG::WARPS_N;
    static constexpr int FI = CFG::BM / (8 * CFG::WARPS_M), FJ = CFG::BN / (8 * CFG::WARPS_N);
};
#define GM_THREADS_MAX 128

struct GemmArgs {
    int M, N, K;
    const double *A;
    int lda;
    int TA;
    const double *B;
    int ldb;
    int TB;
    const double *scale;  // per-k multipliers or null
    double *C;
    int ldc;
    double alpha, beta;
    int upper_only;  // only tiles with m-tile <= n-tile (symmetric outputs, mirrored later)
    int a16, b16;    // operand rows 16-byte aligned (set by gemm_launch); else 8-byte copies
    // K-split gather (block-Jacobi updates): for k >= ksplit the operand with a
    // non-null second base reads A2 / B2 at k - ksplit.  ksplit % GM_BK == 0.
    const double *A2, *B2;
    int ksplit;
    // output split: rows m >= msplit (or columns n >= nsplit) go to C2 at m - msplit (n - nsplit)
    double *C2;
    int msplit, nsplit;
};

__device__ __forceinline__ void dmma_m8n8k4(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void gm_cp16(void *dst, const void *src, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void gm_cp8(void *dst, const void *src, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0));
}

// shared tile geometry: "row" = the contiguous global dimension
// A: TA ? [BK][BM] : [BM][BK];  B: TB ? [BN][BK] : [BK][BN]
template <int TA, int TB, class CFG>
struct GmTile {
    static constexpr int A_ROWS = TA ? GM_BK : CFG::BM, A_COLS = TA ? CFG::BM : GM_BK;
    static constexpr int B_ROWS = TB ? CFG::BN : GM_BK, B_COLS = TB ? GM_BK : CFG::BN;
    static constexpr int A_LD = A_COLS + 4, B_LD = B_COLS + 4;
    static constexpr int A_SZ = A_ROWS * A_LD, B_SZ = B_ROWS * B_LD;
    static constexpr int STAGE = A_SZ + B_SZ + GM_BK;  // + per-k scale
    static constexpr size_t SMEM = (size_t)CFG::STAGES * STAGE * sizeof(double);
};

template <int TA, int TB, class CFG>
__device__ __forceinline__ void gm_issue(const GemmArgs &g, double *st, int m0, int n0, int k0) {
    using T = GmTile<TA, TB, CFG>;
    constexpr int GM_THREADS = GmGeo<CFG>::THREADS, GM_BM = CFG::BM, GM_BN = CFG::BN;
    const int tid = threadIdx.x;
    double *As = st, *Bs = st + T::A_SZ, *Ss = st + T::A_SZ + T::B_SZ;
    // operand bases and k offsets of this k-tile (K-split gather)
    const bool sa = g.A2 && g.ksplit && k0 >= g.ksplit, sb = g.B2 && g.ksplit && k0 >= g.ksplit;
    const double *Ab = sa ? g.A2 : g.A, *Bb = sb ? g.B2 : g.B;
    const int dka = sa ? -g.ksplit : 0, dkb = sb ? -g.ksplit : 0;
    // A: rows of A_COLS doubles, A_COLS/2 16-byte chunks per row
    constexpr int ACH = T::A_COLS / 2, BCH = T::B_COLS / 2;
    // interior tiles (no edge, no K-split switch inside the tile): one base pointer, no
    // per-copy bounds tests -- the index arithmetic of the general path dominated the
    // issue slots of the main loop
    const bool a_in = g.a16 && !sa && !(g.A2 && g.ksplit && k0 + GM_BK > g.ksplit) && m0 + GM_BM <= g.M &&
                      k0 + GM_BK <= g.K;
    const bool b_in = g.b16 && !sb && !(g.B2 && g.ksplit && k0 + GM_BK > g.ksplit) && n0 + GM_BN <= g.N &&
                      k0 + GM_BK <= g.K;
    if (a_in) {
        const double *base = Ab + (size_t)(TA ? k0 : m0) * g.lda + (TA ? m0 : k0);
#pragma unroll
        for (int e = tid; e < T::A_ROWS * ACH; e += GM_THREADS) {
            const int r = e / ACH, c = (e - r * ACH) * 2;
            gm_cp16(As + r * T::A_LD + c, base + (size_t)r * g.lda + c, true);
        }
    } else if (!g.a16) {
        for (int e = tid; e < T::A_ROWS * T::A_COLS; e += GM_THREADS) {
            const int r = e / T::A_COLS, c = e - r * T::A_COLS;
            const int gr = (TA ? k0 : m0) + r, gc = (TA ? m0 : k0) + c;
            const bool ok = gr < (TA ? g.K : g.M) && gc < (TA ? g.M : g.K);
            const int ar = gr + (TA ? dka : 0), ac = gc + (TA ? 0 : dka);
            gm_cp8(As + r * T::A_LD + c, Ab + (ok ? (size_t)ar * g.lda + ac : 0), ok);
        }
    } else {
#pragma unroll
    for (int e = tid; e < T::A_ROWS * ACH; e += GM_THREADS) {
        const int r = e / ACH, c = (e - r * ACH) * 2;
        const int gr = (TA ? k0 : m0) + r, gc = (TA ? m0 : k0) + c;
        const int rlim = TA ? g.K : g.M, clim = TA ? g.M : g.K;
        const bool ok = gr < rlim && gc < clim;
        // the pair (gc, gc+1): when gc+1 is past the edge the row tail is zero-filled by a 8-byte copy
        const int ar = gr + (TA ? dka : 0), ac = gc + (TA ? 0 : dka);
        const double *src = Ab + (size_t)(ok ? ar : 0) * g.lda + (ok ? ac : 0);
        if (ok && gc + 1 >= clim) {
            gm_cp8(As + r * T::A_LD + c, src, true);
            gm_cp8(As + r * T::A_LD + c + 1, src, false);
        } else {
            gm_cp16(As + r * T::A_LD + c, src, ok);
        }
    }
    }
    if (b_in) {
        const double *base = Bb + (size_t)(TB ? n0 : k0) * g.ldb + (TB ? k0 : n0);
#pragma unroll
        for (int e = tid; e < T::B_ROWS * BCH; e += GM_THREADS) {
            const int r = e / BCH, c = (e - r * BCH) * 2;
            gm_cp16(Bs + r * T::B_LD + c, base + (size_t)r * g.ldb + c, true);
        }
    } else if (!g.b16) {
        for (int e = tid; e < T::B_ROWS * T::B_COLS; e += GM_THREADS) {
            const int r = e / T::B_COLS, c = e - r * T::B_COLS;
            const int gr = (TB ? n0 : k0) + r, gc = (TB ? k0 : n0) + c;
            const bool ok = gr < (TB ? g.N : g.K) && gc < (TB ? g.K : g.N);
            const int br = gr + (TB ? 0 : dkb), bc = gc + (TB ? dkb : 0);
            gm_cp8(Bs + r * T::B_LD + c, Bb + (ok ? (size_t)br * g.ldb + bc : 0), ok);
        }
    } else
#pragma unroll
    for (int e = tid; e < T::B_ROWS * BCH; e += GM_THREADS) {
        const int r = e / BCH, c = (e - r * BCH) * 2;
        const int gr = (TB ? n0 : k0) + r, gc = (TB ? k0 : n0) + c;
        const int rlim = TB ? g.N : g.K, clim = TB ? g.K : g.N;
        const bool ok = gr < rlim && gc < clim;
        const int br = gr + (TB ? 0 : dkb), bc = gc + (TB ? dkb : 0);
        const double *src = Bb + (size_t)(ok ? br : 0) * g.ldb + (ok ? bc : 0);
        if (ok && gc + 1 >= clim) {
            gm_cp8(Bs + r * T::B_LD + c, src, true);
            gm_cp8(Bs + r * T::B_LD + c + 1, src, false);
        } else {
            gm_cp16(Bs + r * T::B_LD + c, src, ok);
        }
    }
    if (g.scale && tid < GM_BK / 2) {
        const int c = tid * 2;
        const bool ok = k0 + c < g.K;
        if (ok && k0 + c + 1 >= g.K) {
            gm_cp8(Ss + c, g.scale + k0 + c, true);
            gm_cp8(Ss + c + 1, g.scale, false);
        } else {
            gm_cp16(Ss + c, g.scale + (ok ? k0 + c : 0), ok);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

// The cp.async pipeline over k-tiles [kt0, kt1) of output tile (tm, tn), accumulated into acc.
template <int TA, int TB, class CFG>
__device__ __forceinline__ void gm_accum(const GemmArgs &g, int tm, int tn, int kt0, int kt1, double *gsm,
                                         double (&acc)[GmGeo<CFG>::FI][GmGeo<CFG>::FJ][2]) {
    using T = GmTile<TA, TB, CFG>;
    constexpr int GM_BM = CFG::BM, GM_BN = CFG::BN, GM_STAGES = CFG::STAGES;
    constexpr int GM_WARPS_N = CFG::WARPS_N, GM_WARPS_M = CFG::WARPS_M;
    constexpr int GM_FI = GmGeo<CFG>::FI, GM_FJ = GmGeo<CFG>::FJ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp / GM_WARPS_N) * (GM_BM / GM_WARPS_M), wn = (warp % GM_WARPS_N) * (GM_BN / GM_WARPS_N);
    const int gid = lane >> 2, tig = lane & 3;
    const int m0 = tm * GM_BM, n0 = tn * GM_BN;
    const bool has_scale = g.scale != nullptr;
    const int nk = kt1 - kt0;
#pragma unroll
    for (int s = 0; s < GM_STAGES - 1; ++s) {
        if (s < nk)
            gm_issue<TA, TB, CFG>(g, gsm + s * T::STAGE, m0, n0, (kt0 + s) * GM_BK);
        else
            asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int kt = 0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(GM_STAGES - 2));
        __syncthreads();
        const int nxt = kt + GM_STAGES - 1;
        if (nxt < nk)
            gm_issue<TA, TB, CFG>(g, gsm + (nxt % GM_STAGES) * T::STAGE, m0, n0, (kt0 + nxt) * GM_BK);
        else
            asm volatile("cp.async.commit_group;\n" ::);
        const double *As = gsm + (kt % GM_STAGES) * T::STAGE;
        const double *Bs = As + T::A_SZ, *Ss = As + T::A_SZ + T::B_SZ;
#pragma unroll
        for (int k4 = 0; k4 < GM_BK; k4 += 4) {
            const int kk = k4 + tig;
            double af[GM_FI], bf[GM_FJ];
#pragma unroll
            for (int i = 0; i < GM_FI; ++i) {
                const int mm = wm + i * 8 + gid;
                af[i] = TA ? As[kk * T::A_LD + mm] : As[mm * T::A_LD + kk];
            }
            if (has_scale) {
                const double sk = Ss[kk];
#pragma unroll
                for (int i = 0; i < GM_FI; ++i) af[i] *= sk;
            }
#pragma unroll
            for (int j = 0; j < GM_FJ; ++j) {
                const int nn = wn + j * 8 + gid;
                bf[j] = TB ? Bs[nn * T::B_LD + kk] : Bs[kk * T::B_LD + nn];
            }
#pragma unroll
            for (int i = 0; i < GM_FI; ++i)
#pragma unroll
                for (int j = 0; j < GM_FJ; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();  // the stages may be refilled by the caller's next tile
}

// C fragment (row gid, cols 2*tig, 2*tig+1) of tile (tm, tn): alpha acc + beta C
template <int TA, int TB, class CFG>
__device__ __forceinline__ void gm_epilogue(const GemmArgs &g, int tm, int tn,
                                            const double (&acc)[GmGeo<CFG>::FI][GmGeo<CFG>::FJ][2]) {
    constexpr int GM_BM = CFG::BM, GM_BN = CFG::BN;
    constexpr int GM_WARPS_N = CFG::WARPS_N, GM_WARPS_M = CFG::WARPS_M;
    constexpr int GM_FI = GmGeo<CFG>::FI, GM_FJ = GmGeo<CFG>::FJ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp / GM_WARPS_N) * (GM_BM / GM_WARPS_M), wn = (warp % GM_WARPS_N) * (GM_BN / GM_WARPS_N);
    const int gid = lane >> 2, tig = lane & 3;
    const int m0 = tm * GM_BM, n0 = tn * GM_BN;
#pragma unroll
    for (int i = 0; i < GM_FI; ++i) {
        const int m = m0 + wm + i * 8 + gid;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < GM_FJ; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = n0 + wn + j * 8 + 2 * tig + h;
                if (n >= g.N) continue;
                double v = g.alpha * acc[i][j][h];
                double *cp;
                if (g.C2 && g.nsplit && n >= g.nsplit)
                    cp = g.C2 + (size_t)m * g.ldc + (n - g.nsplit);
                else if (g.C2 && g.msplit && m >= g.msplit)
                    cp = g.C2 + (size_t)(m - g.msplit) * g.ldc + n;
                else
                    cp = g.C + (size_t)m * g.ldc + n;
                if (g.beta != 0.0) v += g.beta * *cp;
                *cp = v;
            }
        }
    }
}

template <int TA, int TB, class CFG>
__device__ __forceinline__ void gm_body(const GemmArgs &g) {
    constexpr int GM_BM = CFG::BM, GM_BN = CFG::BN;
    const int tm = blockIdx.y, tn = blockIdx.x;
    // symmetric outputs: skip tiles entirely below the diagonal (mirrored afterwards)
    if (g.upper_only && tm * GM_BM > tn * GM_BN + GM_BN - 1) return;
    if (tm * GM_BM >= g.M || tn * GM_BN >= g.N) return;  // batched launches size the grid for the largest
    extern __shared__ __align__(16) double gsm[];
    double acc[GmGeo<CFG>::FI][GmGeo<CFG>::FJ][2];
#pragma unroll
    for (int i = 0; i < GmGeo<CFG>::FI; ++i)
#pragma unroll
        for (int j = 0; j < GmGeo<CFG>::FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    gm_accum<TA, TB, CFG>(g, tm, tn, 0, (g.K + GM_BK - 1) / GM_BK, gsm, acc);
    gm_epilogue<TA, TB, CFG>(g, tm, tn, acc);
}

// Stream-K (full outputs only): a persistent grid of co-resident CTAs splits the
// tiles_m x tiles_n x nkt k-iterations evenly.  A CTA's range is the tail of a tile, whole tiles,
// then the head of a tile.  Tails and middles go to the workspace (one slot per CTA: its first
// work item is the only one that can be a non-head segment); the CTA holding a tile's head adds
// the later segments' partials in k order (deterministic) after their flags carry this launch's
// epoch, then writes the tile.  Removes the partial last wave of tile-parallel launches.
__device__ __forceinline__ unsigned gm_ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <int TA, int TB, class CFG>
__global__ void __launch_bounds__(GmGeo<CFG>::THREADS) k_gemm_dmma_sk(GemmArgs g, int tiles_n, int nkt, long total,
                                                                      double *ws, unsigned *flags, unsigned epoch) {
    constexpr int FI = GmGeo<CFG>::FI, FJ = GmGeo<CFG>::FJ, NT = GmGeo<CFG>::THREADS;
    constexpr int NACC = FI * FJ * 2;
    extern __shared__ __align__(16) double gsm[];
    const long per = (total + gridDim.x - 1) / gridDim.x;
    const long it0 = (long)blockIdx.x * per, it1 = min(total, it0 + per);
    long it = it0;
    double acc[FI][FJ][2];
    while (it < it1) {
        const long tile = it / nkt;
        const int kt0 = (int)(it - tile * nkt);
        const int kt1 = (int)min((long)nkt, (long)kt0 + (it1 - it));
        const int tm = (int)(tile / tiles_n), tn = (int)(tile - (long)tm * tiles_n);
#pragma unroll
        for (int i = 0; i < FI; ++i)
#pragma unroll
            for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gm_accum<TA, TB, CFG>(g, tm, tn, kt0, kt1, gsm, acc);
        if (kt0 != 0) {
            // tail or middle segment: publish the partial for the tile's head CTA
            double *slot = ws + (size_t)blockIdx.x * NACC * NT;
#pragma unroll
            for (int i = 0; i < FI; ++i)
#pragma unroll
                for (int j = 0; j < FJ; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) __stcg(slot + ((i * FJ + j) * 2 + h) * NT + threadIdx.x, acc[i][j][h]);
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) atomicExch(flags + blockIdx.x, epoch);
        } else {
            // head segment: add the later segments in k order, then write the tile
            long nit = it + (kt1 - kt0);
            int kt = kt1;
            while (kt < nkt) {
                const int owner = (int)(nit / per);
                if (threadIdx.x == 0)
                    while (gm_ld_acquire(flags + owner) != epoch) {
                    }
                __syncthreads();
                const double *slot = ws + (size_t)owner * NACC * NT;
#pragma unroll
                for (int i = 0; i < FI; ++i)
#pragma unroll
                    for (int j = 0; j < FJ; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            acc[i][j][h] += __ldcg(slot + ((i * FJ + j) * 2 + h) * NT + threadIdx.x);
                const long oend = min(total, (long)(owner + 1) * per);
                const int seg = (int)min((long)(nkt - kt), oend - nit);
                kt += seg;
                nit += seg;
            }
            gm_epilogue<TA, TB, CFG>(g, tm, tn, acc);
        }
        it += kt1 - kt0;
    }
}

template <int TA, int TB, class CFG>
__global__ void __launch_bounds__(GM_THREADS_MAX) k_gemm_dmma(GemmArgs g) {
    gm_body<TA, TB, CFG>(g);
}

// one GEMM per blockIdx.z (independent outputs); grid sized for the largest
template <int TA, int TB>
__global__ void __launch_bounds__(GM_THREADS_MAX) k_gemm_dmma_batched(const GemmArgs *gs) {
    const GemmArgs g = gs[blockIdx.z];
    gm_body<TA, TB, GmSmall>(g);
}

// mirror the upper triangle of an n x n matrix into the lower one: tile (ti, tj), ti >= tj, of
// the lower triangle is the transpose of upper tile (tj, ti), staged through shared memory so
// both the read and the write are coalesced.  Launch: grid (nt, nt), block (32, 8).
__global__ void k_mirror_upper_tiled(double *C, int n, int ldc) {
    __shared__ double t[32][33];
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (ti < tj) return;
    const int r0 = tj * 32, c0 = ti * 32;  // source tile (upper): rows r0.., columns c0..
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = r0 + k, c = c0 + threadIdx.x;
        if (r < n && c < n) t[k][threadIdx.x] = C[(size_t)r * ldc + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = c0 + k, c = r0 + threadIdx.x;  // destination (lower): row r > column c
        if (r < n && c < n && r > c) C[(size_t)r * ldc + c] = t[threadIdx.x][k];
    }
}
static inline void mirror_upper(double *C, int n, int ldc, cudaStream_t s) {
    const int nt = (n + 31) / 32;
    k_mirror_upper_tiled<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(C, n, ldc);
}

template <int TA, int TB, class CFG>
static inline cudaError_t gemm_launch_t(const GemmArgs &g, cudaStream_t s) {
    using T = GmTile<TA, TB, CFG>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k_gemm_dmma<TA, TB, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)T::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid((g.N + CFG::BN - 1) / CFG::BN, (g.M + CFG::BM - 1) / CFG::BM);
    k_gemm_dmma<TA, TB, CFG><<<grid, GmGeo<CFG>::THREADS, T::SMEM, s>>>(g);
    return cudaGetLastError();
}

// Tiles a launch computes (upper_only skips those entirely below the diagonal).
template <class CFG>
static inline long gemm_tiles(const GemmArgs &g) {
    const int tm = (g.M + CFG::BM - 1) / CFG::BM, tn = (g.N + CFG::BN - 1) / CFG::BN;
    if (!g.upper_only) return (long)tm * tn;
    long n = 0;
    for (int i = 0; i < tm; ++i)
        for (int j = 0; j < tn; ++j) n += (i * CFG::BM <= j * CFG::BN + CFG::BN - 1);
    return n;
}
// Big tiles when they fill at least ~0.85 of a wave of two CTAs per SM on 148 SMs (measured:
// d^3 at d = 2083 28.8 vs 25.1 TF/s; the 1040 x 1040 Hessian blocks, 153 big tiles, stay small).
static inline bool gemm_big_tiles(const GemmArgs &g) { return gemm_tiles<GmBig>(g) >= 250; }

// Grouped stream-K: several GEMMs (same TA/TB; descriptors in device memory) as one iteration
// space.  tiles[t] = (descriptor, tm, tn, k-tiles), prefix[t] = k-iterations before tile t
// (prefix[ntiles] = total); upper_only descriptors list only their computed tiles.  Same
// partial/flag protocol as k_gemm_dmma_sk.
template <int TA, int TB, class CFG>
__global__ void __launch_bounds__(GmGeo<CFG>::THREADS)
    k_gemm_dmma_skg(const GemmArgs *descs, const int4 *tiles, const long *prefix, int ntiles, double *ws,
                    unsigned *flags, unsigned epoch) {
    constexpr int FI = GmGeo<CFG>::FI, FJ = GmGeo<CFG>::FJ, NT = GmGeo<CFG>::THREADS;
    constexpr int NACC = FI * FJ * 2;
    extern __shared__ __align__(16) double gsm[];
    const long total = prefix[ntiles];
    const long per = (total + gridDim.x - 1) / gridDim.x;
    const long it0 = (long)blockIdx.x * per, it1 = min(total, it0 + per);
    if (it0 >= it1) return;
    int t = 0;
    {  // first tile with prefix[t + 1] > it0
        int lo = 0, hi = ntiles - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (prefix[mid + 1] > it0)
                hi = mid;
            else
                lo = mid + 1;
        }
        t = lo;
    }
    long it = it0;
    double acc[FI][FJ][2];
    while (it < it1) {
        const int4 tl = tiles[t];
        const GemmArgs g = descs[tl.x];
        const int nkt = tl.w;
        const int kt0 = (int)(it - prefix[t]);
        const int kt1 = (int)min((long)nkt, (long)kt0 + (it1 - it));
#pragma unroll
        for (int i = 0; i < FI; ++i)
#pragma unroll
            for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gm_accum<TA, TB, CFG>(g, tl.y, tl.z, kt0, kt1, gsm, acc);
        if (kt0 != 0) {
            double *slot = ws + (size_t)blockIdx.x * NACC * NT;
#pragma unroll
            for (int i = 0; i < FI; ++i)
#pragma unroll
                for (int j = 0; j < FJ; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) __stcg(slot + ((i * FJ + j) * 2 + h) * NT + threadIdx.x, acc[i][j][h]);
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) atomicExch(flags + blockIdx.x, epoch);
        } else {
            long nit = it + (kt1 - kt0);
            int kt = kt1;
            while (kt < nkt) {
                const int owner = (int)(nit / per);
                if (threadIdx.x == 0)
                    while (gm_ld_acquire(flags + owner) != epoch) {
                    }
                __syncthreads();
                const double *slot = ws + (size_t)owner * NACC * NT;
#pragma unroll
                for (int i = 0; i < FI; ++i)
#pragma unroll
                    for (int j = 0; j < FJ; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            acc[i][j][h] += __ldcg(slot + ((i * FJ + j) * 2 + h) * NT + threadIdx.x);
                const long oend = min(total, (long)(owner + 1) * per);
                const int seg = (int)min((long)(nkt - kt), oend - nit);
                kt += seg;
                nit += seg;
            }
            gm_epilogue<TA, TB, CFG>(g, tl.y, tl.z, acc);
        }
        it += kt1 - kt0;
        ++t;
    }
}

// Tile list of a grouped GEMM (host): descriptors' shapes only.
static inline void gemm_group_tiles(const GemmArgs *gs, int n, std::vector<int4> &tiles, std::vector<long> &prefix) {
    tiles.clear();
    prefix.assign(1, 0);
    for (int di = 0; di < n; ++di) {
        const GemmArgs &g = gs[di];
        const int tm_n = (g.M + GmBig::BM - 1) / GmBig::BM, tn_n = (g.N + GmBig::BN - 1) / GmBig::BN;
        const int nkt = (g.K + GM_BK - 1) / GM_BK;
        for (int tm = 0; tm < tm_n; ++tm)
            for (int tn = 0; tn < tn_n; ++tn) {
                if (g.upper_only && tm * GmBig::BM > tn * GmBig::BN + GmBig::BN - 1) continue;
                tiles.push_back(make_int4(di, tm, tn, nkt));
                prefix.push_back(prefix.back() + nkt);
            }
    }
}

// Stream-K launch of a full big-tile GEMM when tile-parallel waves would waste more than 3 %
// (C4: d^3 at d = 2083 561 tiles = 1.90 waves of 296 CTA slots, the trace 2112 = 7.14 waves).
// Workspace (partials + flags) per (device, stream); SGP_GEMM_STREAMK=0 disables.
struct GmSkWS {
    int dev = -1;
    cudaStream_t stream = nullptr;
    double *ws = nullptr;
    unsigned *flags = nullptr;
    unsigned epoch = 0;
    int grid = 0;
};
// partials + flags of the stream-K launches on stream s (one set per device and stream)
static inline GmSkWS *gm_sk_ws(cudaStream_t s, int slots) {
    static GmSkWS cache[8];
    int dev = 0;
    cudaGetDevice(&dev);
    for (GmSkWS &c : cache)
        if (c.ws && c.dev == dev && c.stream == s) return c.grid >= slots ? &c : nullptr;
    GmSkWS *w = nullptr;
    for (GmSkWS &c : cache)
        if (!c.ws) {
            w = &c;
            break;
        }
    if (!w) return nullptr;
    const size_t nacc = (size_t)GmGeo<GmBig>::FI * GmGeo<GmBig>::FJ * 2 * GmGeo<GmBig>::THREADS;
    if (cudaMalloc(&w->ws, sizeof(double) * nacc * slots) != cudaSuccess) {
        w->ws = nullptr;
        return nullptr;
    }
    if (cudaMalloc(&w->flags, sizeof(unsigned) * slots) != cudaSuccess ||
        cudaMemset(w->flags, 0, sizeof(unsigned) * slots) != cudaSuccess) {
        cudaFree(w->ws);
        w->ws = nullptr;
        return nullptr;
    }
    w->dev = dev;
    w->stream = s;
    w->grid = slots;
    return w;
}

// Grouped stream-K launch (descriptors and tile list in device memory); false if unavailable.
template <int TA, int TB>
static inline bool gemm_launch_skg(const GemmArgs *d_descs, const int4 *d_tiles, const long *d_prefix, int ntiles,
                                   cudaStream_t s) {
    using CFG = GmBig;
    using T = GmTile<TA, TB, CFG>;
    static bool configured = false;
    static int per_sm = 0, sms = 0;
    if (!configured) {
        if (cudaFuncSetAttribute(k_gemm_dmma_skg<TA, TB, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)T::SMEM) != cudaSuccess)
            return false;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm_dmma_skg<TA, TB, CFG>,
                                                          GmGeo<CFG>::THREADS, T::SMEM) != cudaSuccess)
            per_sm = 0;
        configured = true;
    }
    if (per_sm < 1 || ntiles < 1) return false;
    const int slots = per_sm * sms;
    GmSkWS *w = gm_sk_ws(s, slots);
    if (!w) return false;
    unsigned epoch = ++w->epoch;
    if (epoch == 0) epoch = ++w->epoch;
    double *ws = w->ws;
    unsigned *flags = w->flags;
    int nt = ntiles;
    void *args[] = {(void *)&d_descs, (void *)&d_tiles, (void *)&d_prefix, &nt, &ws, &flags, &epoch};
    const cudaError_t err = cudaLaunchCooperativeKernel((void *)k_gemm_dmma_skg<TA, TB, CFG>, slots,
                                                        GmGeo<CFG>::THREADS, args, T::SMEM, s);
    if (err != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

template <int TA, int TB>
static inline bool gemm_launch_sk(const GemmArgs &g, cudaStream_t s, cudaError_t &err) {
    using CFG = GmBig;
    using T = GmTile<TA, TB, CFG>;
    static const bool enabled = !(getenv("SGP_GEMM_STREAMK") && getenv("SGP_GEMM_STREAMK")[0] == '0');
    if (!enabled || g.upper_only || g.ksplit || g.C2 || g.K <= 0) return false;
    static bool configured = false;
    static int per_sm = 0, sms = 0;
    if (!configured) {
        if (cudaFuncSetAttribute(k_gemm_dmma_sk<TA, TB, CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)T::SMEM) != cudaSuccess)
            return false;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm_dmma_sk<TA, TB, CFG>,
                                                          GmGeo<CFG>::THREADS, T::SMEM) != cudaSuccess)
            per_sm = 0;
        configured = true;
    }
    if (per_sm < 1) return false;
    const int slots = per_sm * sms;
    const int tiles_m = (g.M + CFG::BM - 1) / CFG::BM, tiles_n = (g.N + CFG::BN - 1) / CFG::BN;
    const long tiles = (long)tiles_m * tiles_n;
    if (tiles < slots) return false;
    const long waves = (tiles + slots - 1) / slots;
    if ((double)tiles / (double)(waves * slots) >= 0.97) return false;
    GmSkWS *w = gm_sk_ws(s, slots);
    if (!w) return false;
    unsigned epoch = ++w->epoch;
    if (epoch == 0) epoch = ++w->epoch;  // 0 is the flags' initial value
    const int nkt = (g.K + GM_BK - 1) / GM_BK;
    long total = tiles * nkt;
    GemmArgs ga = g;
    int tn = tiles_n, nk = nkt;
    double *ws = w->ws;
    unsigned *flags = w->flags;
    void *args[] = {&ga, &tn, &nk, &total, &ws, &flags, &epoch};
    err = cudaLaunchCooperativeKernel((void *)k_gemm_dmma_sk<TA, TB, CFG>, w->grid, GmGeo<CFG>::THREADS, args,
                                      T::SMEM, s);
    return err == cudaSuccess;
}

static inline cudaError_t gemm_launch(GemmArgs g, cudaStream_t s) {
    g.a16 = (g.lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0);
    g.b16 = (g.ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(g.B) & 15) == 0);
    const bool big = gemm_big_tiles(g) && !g.ksplit && !g.C2;
    if (big) {
        cudaError_t err = cudaSuccess;
        bool done;
        if (g.TA)
            done = g.TB ? gemm_launch_sk<1, 1>(g, s, err) : gemm_launch_sk<1, 0>(g, s, err);
        else
            done = g.TB ? gemm_launch_sk<0, 1>(g, s, err) : gemm_launch_sk<0, 0>(g, s, err);
        if (done) return err;
        if (err != cudaSuccess) cudaGetLastError();  // a refused cooperative launch: tile-parallel instead
    }
    if (g.TA) {
        if (g.TB) return big ? gemm_launch_t<1, 1, GmBig>(g, s) : gemm_launch_t<1, 1, GmSmall>(g, s);
        return big ? gemm_launch_t<1, 0, GmBig>(g, s) : gemm_launch_t<1, 0, GmSmall>(g, s);
    }
    if (g.TB) return big ? gemm_launch_t<0, 1, GmBig>(g, s) : gemm_launch_t<0, 1, GmSmall>(g, s);
    return big ? gemm_launch_t<0, 0, GmBig>(g, s) : gemm_launch_t<0, 0, GmSmall>(g, s);
}

// Batched launch: nb descriptors in device memory (all with the same TA, TB
// and alignment flags, set by the caller); grid covers max M x max N.
template <int TA, int TB>
static inline cudaError_t gemm_launch_batched(const GemmArgs *d_gs, int nb, int maxM, int maxN, cudaStream_t s) {
    using T = GmTile<TA, TB, GmSmall>;
    constexpr int GM_BM = GmSmall::BM, GM_BN = GmSmall::BN, GM_THREADS = GmGeo<GmSmall>::THREADS;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k_gemm_dmma_batched<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)T::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid((maxN + GM_BN - 1) / GM_BN, (maxM + GM_BM - 1) / GM_BM, nb);
    k_gemm_dmma_batched<TA, TB><<<grid, GM_THREADS, T::SMEM, s>>>(d_gs);
    return cudaGetLastError();
}
