// sgp_jbig.cuh — reference-order (cyclic-by-row) Jacobi for large d, bit-identical to
// _jacobi.jacobi_sweeps (_jacobi.py:37-86), spread over a cooperative grid.
//
// Why a new kernel: the reference's cold decompositions (chain start, every rejection,
// every TI rung start: metric.py:112-142, sampler.py:322-328,392-397) must keep its pivot
// order, because the momentum p = Psi (sqrt(g) o z) depends on the order and signs of
// Psi's columns.  The single-warp generic sweep of sgp_core.cuh takes
// ~60 s per sweep at d = 2083 (27 us per rotation: every rotation walks a strided column
// of a 35 MB matrix on one warp).  Here the serial part is reduced to what really is serial.
//
// Structure of one sweep (proved from _jacobi.py:54-85).  Pass p = rotations (p, q),
// q = p+1 .. d-1, in order.  Rotation (p, q) rewrites, for every k != p, q, the pair
// (a_kp, a_kq) -> (c a_kp - s a_kq, s a_kp + c a_kq) and sets a_pq = 0, a_pp -= t a_pq,
// a_qq += t a_pq.  Rows k are independent of each other inside a rotation; what makes the
// sweep serial is only the pivot chain: rotation (p, q+1) needs a_{q+1,p} after rotation
// (p, q), i.e. c x - s y with x = a_{q+1,p} after (p, q-1) and y = a_{q+1,q}.
//
// The pivots of a pass are processed in windows W_m = [q0, q0+32), q0 = p+1+32m.
//   * chain CTA, warp 0 ("chain"): lane l owns row q0+l of W_m.  It runs the window's 32
//     rotations (the rotation-parameter chain, replicated in every lane, is the only serial
//     work), holding the running a_kp in a register and the 32 x 32 diagonal block
//     W_m x W_m in shared memory; rotation j-1 is applied to the lanes while rotation j's
//     parameters are computed (software pipelining as in jacobi_sweep_warp).
//   * chain CTA, warp 1 ("lookahead"): rows W_{m+1}.  It first applies window m-1's
//     rotations (all known) and then follows window m's rotations two or three steps behind
//     the chain, so the next window's running a_kp are ready when the chain gets there.
//   * chain CTA, warps 2-3 ("io"): load the next diagonal block, write the finished
//     window back to global memory (diagonal block, a_kp, the rotation log) and publish it.
//   * owner CTAs: every other row k (all but W_m, W_{m+1}, W_{m+2}); each owner has a fixed
//     block of rows and applies a published window's 32 rotations to them (one window
//     behind the chain).  The elements a_kq of row k for the 32 pivots q of the window are
//     one contiguous 256-byte segment L[k][q0..q0+31] when k > q, or one element of each of
//     the 32 window rows L[q][k] when k < q (coalesced across k).
// Every element receives exactly the reference's sequence of rounded operations (no FMA),
// in the reference's order, so the result is bit-identical; the dependency rules between the
// three roles are spelled out at jb_need_diag / the owner wait below.
//
// Storage: A is the d x d row-major buffer; element (i, j), i > j, lives at L[i*d + j] (the
// lower triangle, like lt_index); the diagonal lives in dg[] (a shared-memory copy in the
// chain CTA during the sweep).  The eigenvector update (_jacobi.py:81-85) is applied after
// the sweep from the rotation log by k_jb_vapply on a second stream (row k of V only ever
// sees rotations in log order), overlapping the next sweep.
#pragma once

#define JB_W 32
#define JB_NT 128
#define JB_MAX_OWN 32
#define JB_LDB 33  // padded stride of the 32 x 32 shared-memory blocks

struct JbArgs {
    double *L;       // d x d, lower triangle used
    double *dg;      // d diagonal (in at sweep start, out at sweep end)
    double *R;       // d running a_kp of owner rows between windows
    double *logcs;   // (c, s) of every rotation slot (p, q) of this sweep
    int *logf;       // 1 = rotated, 0 = skipped
    unsigned *pub;   // [0] last window published by the chain CTA (1-based window sequence)
    unsigned *prog;  // [nown] last window completed by each owner
    int d, nown;
    double skip;
};

#ifdef SGP_JBIG_PROF
// phase cycles of the chain CTA (summed over windows): 0 chain warp in its window, 1 chain warp
// at the start barrier, 2 lookahead total, 3 lookahead owner wait, 4 io publish, 5 io deferred
// load, 6 io prefetch, 7 end barrier wait (warp 0), 8 windows
__device__ unsigned long long jb_prof[16];
#define JB_T0(v) const long long v = clock64()
#define JB_ACC(i, v) atomicAdd(&jb_prof[i], (unsigned long long)(clock64() - (v)))
#else
#define JB_T0(v)
#define JB_ACC(i, v)
#endif

__device__ __forceinline__ unsigned jb_ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void jb_st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int jb_nw(int d, int p) { return (d - 1 - p + JB_W - 1) / JB_W; }
__device__ __forceinline__ size_t jb_slot(int d, int p) {  // first log slot of pass p
    return (size_t)p * (size_t)(2 * d - p - 1) / 2;
}

// Minimum owner progress before the chain CTA may read the elements of window (p, m):
// the diagonal block W_m x W_m and the lookahead tiles W_{m+1} x (W_{m-1} u W_m) carry
// indices below q0(m+2) = p+1+32(m+2); their last update of pass p-1 happened in pass p-1's
// window min(m+2, last) at the latest (pass p-1's windows are shifted by one index).
__device__ __forceinline__ unsigned jb_need_diag(int m, unsigned prev_start, int prev_nw) {
    if (prev_nw <= 0) return 0u;
    return prev_start + (unsigned)min(m + 2, prev_nw - 1);
}

// wait until every owner has completed window `need` (one warp, warp-uniform).  *cache holds
// the smallest owner progress this warp last observed with an acquire load; while it covers
// `need` nothing is polled (the earlier acquire already ordered the data behind it).
__device__ __forceinline__ void jb_wait_owners(const JbArgs &a, unsigned need, volatile unsigned *cache) {
    if (need == 0u || *cache >= need) return;
    const int lane = threadIdx.x & 31;
    for (;;) {
        const unsigned v = lane < a.nown ? jb_ld_acquire(a.prog + lane) : 0xffffffffu;
        unsigned mn = v;
        for (int o = 16; o; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if (mn >= need) {
            if (lane == 0) *cache = mn;
            __syncwarp();
            break;
        }
        __nanosleep(64);
    }
}

// ---------------------------------------------------------------------------
// chain CTA

struct JbShared {
    double *dg;                    // [d]
    double *B[2];                  // [32 x 33] diagonal blocks (window parity)
    double *rc[2], *rs[2];         // [32] rotation ring (window parity)
    int *rf[2];                    // [32]
    double *rnext, *rfin;          // [32] lookahead -> chain, chain -> io
    volatile int *cnt;             // rotations of the current window published by the chain
    volatile unsigned *own_la, *own_io;  // owner-progress caches of the lookahead and io warps
};

__device__ __forceinline__ void jb_chain_window(const JbArgs &a, const JbShared &sh, int p, int m, unsigned seq,
                                                double &app) {
    const int d = a.d, lane = threadIdx.x & 31;
    const int q0 = p + 1 + JB_W * m, n = min(JB_W, d - q0);
    const bool valid = lane < n;
    const int k = q0 + lane;
    double *B = sh.B[seq & 1];
    double *rc = sh.rc[seq & 1], *rs = sh.rs[seq & 1];
    int *rf = sh.rf[seq & 1];
    double r = 0.0, dq = 0.0;
    if (valid) {
        r = (m == 0) ? __ldcg(a.L + (size_t)k * d + p) : sh.rnext[lane];
        dq = sh.dg[k];
    }
    __syncwarp();
    double piv = __shfl_sync(0xffffffffu, r, 0);
    double aqq = __shfl_sync(0xffffffffu, dq, 0);
    const double skip = a.skip;
    double my_c = 1.0, my_s = 0.0;
    int my_f = 0;
    // pending rotation j-1, applied to the lanes while rotation j's parameters are computed
    bool has = false;
    double pc = 1.0, ps = 0.0, pdq = 0.0;
    int pj = 0;
    // branch-free (predicated) application, so it shares a basic block with the parameter chain
    auto apply_pending = [&]() {
        const bool upd = has && valid && lane != pj;
        const bool own = has && lane == pj;
        const int hi = max(lane, pj), lo = min(lane, pj);
        double *e = B + hi * JB_LDB + lo;
        const double akp = r, akq = *e;
        const double nkp = __dsub_rn(__dmul_rn(pc, akp), __dmul_rn(ps, akq));
        const double nkq = __dadd_rn(__dmul_rn(ps, akp), __dmul_rn(pc, akq));
        r = upd ? nkp : (own ? 0.0 : r);
        dq = own ? pdq : dq;
        if (upd) *e = nkq;
    };
    for (int j = 0; j < n; ++j) {
        const int jn = (j + 1) & 31;
        // a_{q_{j+1}, q_j}: touched only by rotations j and j+1, so still the pre-rotation-j value
        const double Y = (j + 1 < n) ? B[(j + 1) * JB_LDB + j] : 0.0;
        const bool rot = !(fabs(piv) <= skip);  // warp-uniform; NaN rotates as in the reference
        double c = 1.0, s = 0.0, t = 0.0, X;
        if (rot) {
            const bool fast = jacobi_rot_fast(app, aqq, piv, c, s, t);
            apply_pending();
            X = __shfl_sync(0xffffffffu, r, jn);  // a_{q_{j+1}, p} after rotation j-1
            if (!fast) jacobi_rot(app, aqq, piv, c, s, t);  // warp-uniform, rare
        } else {
            apply_pending();
            X = __shfl_sync(0xffffffffu, r, jn);
        }
        const double aqn = __shfl_sync(0xffffffffu, dq, jn);  // changed only by rotation j+1
        if (rot) {
            const double tp = __dmul_rn(t, piv);
            app = __dsub_rn(app, tp);
            pdq = __dadd_rn(aqq, tp);
            piv = __dsub_rn(__dmul_rn(c, X), __dmul_rn(s, Y));
        } else {
            piv = X;
        }
        if (lane == j) {  // rotation j's parameters stay with lane j until the window ends
            my_c = c;
            my_s = s;
            my_f = rot ? 1 : 0;
        }
        has = rot;
        pc = c;
        ps = s;
        pj = j;
        aqq = aqn;
        __syncwarp();
    }
    apply_pending();
    __syncwarp();
    if (valid) {
        sh.rfin[(seq & 1) * JB_W + lane] = r;
        sh.dg[k] = dq;
    }
    // the window's rotation ring, written once (the lookahead folds it after the window)
    rc[lane] = my_c;
    rs[lane] = my_s;
    rf[lane] = lane < n ? my_f : 0;
}

// Lookahead warp at window (p, m): rows W_{m+1}.  Their running a_kp must enter the chain's
// window m+1 current through window m.  They come from the owners current through window
// m-2 (owners skip W_{m+1} at windows m-1 and m), then window m-1's rotations (all known)
// and window m's rotations (as the chain publishes them) are applied here.
__device__ __forceinline__ void jb_lookahead(const JbArgs &a, const JbShared &sh, int p, int m, unsigned seq,
                                             unsigned start, unsigned prev_start, int prev_nw) {
    const int d = a.d, lane = threadIdx.x & 31;
    const int q0 = p + 1 + JB_W * m, n = min(JB_W, d - q0);
    if (q0 + JB_W >= d) {  // no next window in this pass
        asm volatile("bar.sync 4, 64;" ::: "memory");
        return;
    }
    const int k = q0 + JB_W + lane;
    const bool valid = k < d;
    unsigned need = jb_need_diag(m, prev_start, prev_nw);
    if (m >= 2) need = max(need, start + (unsigned)(m - 2));
    JB_T0(tw);
    jb_wait_owners(a, need, sh.own_la);
    if (lane == 0) JB_ACC(3, tw);
    double *rowk = a.L + (size_t)(valid ? k : d - 1) * d;
    double r = 0.0;
    if (valid) r = (m <= 1) ? __ldcg(rowk + p) : __ldcg(a.R + k);
    if (m >= 1) {  // catch-up: window m-1 (a full window), ring parity (seq - 1)
        const volatile double *rc = sh.rc[(seq - 1) & 1], *rs = sh.rs[(seq - 1) & 1];
        const volatile int *rf = sh.rf[(seq - 1) & 1];
        double *seg = rowk + (q0 - JB_W);
        double e[JB_W];
#pragma unroll
        for (int j = 0; j < JB_W; ++j) e[j] = valid ? __ldcg(seg + j) : 0.0;
#pragma unroll
        for (int j = 0; j < JB_W; ++j) {
            if (rf[j]) {
                const double c = rc[j], s = rs[j];
                const double akp = r, akq = e[j];
                r = __dsub_rn(__dmul_rn(c, akp), __dmul_rn(s, akq));
                e[j] = __dadd_rn(__dmul_rn(s, akp), __dmul_rn(c, akq));
            }
        }
        if (valid) {
#pragma unroll
            for (int j = 0; j < JB_W; ++j) __stcg(seg + j, e[j]);
        }
    }
    {  // window m: its tile is loaded while the chain runs, folded once the chain is done
        double *seg = rowk + q0;
        double e[JB_W];
#pragma unroll
        for (int j = 0; j < JB_W; ++j) e[j] = (valid && j < n) ? __ldcg(seg + j) : 0.0;
        JB_T0(tlb);
        asm volatile("bar.sync 4, 64;" ::: "memory");  // the chain wrote the window's ring
        if (lane == 0) JB_ACC(9, tlb);
        JB_T0(tlf);
        const double *rc = sh.rc[seq & 1], *rs = sh.rs[seq & 1];
        const int *rf = sh.rf[seq & 1];
        // ring read 8 rotations ahead of the arithmetic, flags applied by selection (the same
        // rounded operations as a per-rotation branch, without a shared-memory load on the
        // serial path of every step)
#pragma unroll
        for (int j0 = 0; j0 < JB_W; j0 += 8) {
            double cj[8], sj[8];
            int fj[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                cj[t] = rc[j0 + t];
                sj[t] = rs[j0 + t];
                fj[t] = rf[j0 + t];
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int j = j0 + t;
                const bool on = j < n && fj[t] != 0;
                const double akp = r, akq = e[j];
                const double nr = __dsub_rn(__dmul_rn(cj[t], akp), __dmul_rn(sj[t], akq));
                const double ne = __dadd_rn(__dmul_rn(sj[t], akp), __dmul_rn(cj[t], akq));
                r = on ? nr : r;
                e[j] = on ? ne : e[j];
            }
        }
        if (valid) {
            sh.rnext[lane] = r;
#pragma unroll
            for (int j = 0; j < JB_W; ++j)
                if (j < n) __stcg(seg + j, e[j]);
        }
        if (lane == 0) JB_ACC(10, tlf);
    }
    // no fence here: these stores are ordered before the io warps' fence and release of this
    // window by the CTA barrier that ends it (happens-before is transitive across the scopes)
}

// io warps (64 threads): write window (p, m) of the chain back and publish it as `seq`
__device__ __forceinline__ void jb_publish(const JbArgs &a, const JbShared &sh, int p, int m, int nw, unsigned seq,
                                           int io_t) {
    const int d = a.d;
    const int q0 = p + 1 + JB_W * m, n = min(JB_W, d - q0);
    const double *B = sh.B[seq & 1];
    for (int idx = io_t; idx < JB_W * JB_W; idx += 64) {
        const int l = idx >> 5, j = idx & 31;
        if (j < l && l < n) __stcg(a.L + (size_t)(q0 + l) * d + q0 + j, B[l * JB_LDB + j]);
    }
    if (io_t < n) {
        const double r = sh.rfin[(seq & 1) * JB_W + io_t];
        if (m == nw - 1)
            __stcg(a.L + (size_t)(q0 + io_t) * d + p, r);  // final column p entry
        else
            __stcg(a.R + q0 + io_t, r);
        const size_t slot = jb_slot(d, p) + (size_t)JB_W * m + io_t;
        __stcg(a.logcs + 2 * slot, sh.rc[seq & 1][io_t]);
        __stcg(a.logcs + 2 * slot + 1, sh.rs[seq & 1][io_t]);
        __stcg(a.logf + slot, sh.rf[seq & 1][io_t]);
    }
    __threadfence();
    asm volatile("bar.sync 3, 64;" ::: "memory");
    if (io_t == 0) jb_st_release(a.pub, seq);
}

// io warps: diagonal block W_m x W_m of window (p, m) into B[parity]
__device__ __forceinline__ void jb_load_diag(const JbArgs &a, double *B, int p, int m, int io_t) {
    const int d = a.d;
    const int q0 = p + 1 + JB_W * m, n = min(JB_W, d - q0);
    // all 16 loads of a thread in flight before the stores (one L2 round trip, not 16)
    double v[JB_W * JB_W / 64];
#pragma unroll
    for (int t = 0; t < JB_W * JB_W / 64; ++t) {
        const int idx = io_t + 64 * t, l = idx >> 5, j = idx & 31;
        v[t] = (j < l && l < n) ? __ldcg(a.L + (size_t)(q0 + l) * d + q0 + j) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < JB_W * JB_W / 64; ++t) {
        const int idx = io_t + 64 * t, l = idx >> 5, j = idx & 31;
        if (j < l && l < n) B[l * JB_LDB + j] = v[t];
    }
}

__device__ void jb_chain_cta(const JbArgs &a, double *smem) {
    const int d = a.d, warp = threadIdx.x >> 5, io_t = threadIdx.x - 64;
    JbShared sh;
    double *q = smem;
    sh.dg = q;
    q += (d + 1) & ~1;
    sh.B[0] = q;
    q += JB_W * JB_LDB + 1;
    sh.B[1] = q;
    q += JB_W * JB_LDB + 1;
    for (int b = 0; b < 2; ++b) {
        sh.rc[b] = q;
        q += JB_W;
        sh.rs[b] = q;
        q += JB_W;
    }
    sh.rnext = q;
    q += JB_W;
    sh.rfin = q;  // two parities
    q += 2 * JB_W;
    sh.rf[0] = reinterpret_cast<int *>(q);
    sh.rf[1] = sh.rf[0] + JB_W;
    sh.cnt = reinterpret_cast<volatile int *>(sh.rf[1] + JB_W);
    sh.own_la = reinterpret_cast<volatile unsigned *>(sh.rf[1] + JB_W + 1);
    sh.own_io = sh.own_la + 1;
    for (int i = threadIdx.x; i < d; i += JB_NT) sh.dg[i] = __ldcg(a.dg + i);
    if (threadIdx.x == 0) {
        *sh.cnt = 0;
        *sh.own_la = 0u;
        *sh.own_io = 0u;
    }
    __syncthreads();
    unsigned seq = 1, start = 1, prev_start = 0;
    int prev_nw = 0;
    bool deferred = true;
    int pp = -1, pm = 0, pnw = 0;
    double app = 0.0;
    for (int p = 0; p < d - 1; ++p) {
        const int nw = jb_nw(d, p);
        start = seq;
        if (warp == 0) app = sh.dg[p];
        for (int m = 0; m < nw; ++m, ++seq) {
            if (warp >= 2) {
                // release the chain first when this window's block is already loaded; the
                // previous window's buffers (other parity) are written back meanwhile
                if (!deferred) asm volatile("bar.sync 2, 96;" ::: "memory");
                JB_T0(tp);
                if (pp >= 0) jb_publish(a, sh, pp, pm, pnw, seq - 1, io_t);
                if (io_t == 0) JB_ACC(4, tp);
                if (deferred) {
                    JB_T0(td);
                    if (warp == 2) jb_wait_owners(a, jb_need_diag(m, prev_start, prev_nw), sh.own_io);
                    asm volatile("bar.sync 3, 64;" ::: "memory");
                    jb_load_diag(a, sh.B[seq & 1], p, m, io_t);
                    if (io_t == 0) JB_ACC(5, td);
                    asm volatile("bar.sync 2, 96;" ::: "memory");
                }
                JB_T0(tf);
                // prefetch the next window's diagonal block when its sources are final
                int np = p, nm = m + 1;
                unsigned need;
                if (nm < nw) {
                    need = jb_need_diag(nm, prev_start, prev_nw);
                } else {
                    np = p + 1;
                    nm = 0;
                    need = jb_need_diag(0, start, nw);
                }
                if (np < d - 1 && need <= seq - 1) {
                    if (warp == 2) jb_wait_owners(a, need, sh.own_io);
                    asm volatile("bar.sync 3, 64;" ::: "memory");
                    jb_load_diag(a, sh.B[(seq + 1) & 1], np, nm, io_t);
                    deferred = false;
                } else {
                    deferred = true;
                }
                if (io_t == 0) JB_ACC(6, tf);
            } else if (warp == 0) {
                JB_T0(tb);
                asm volatile("bar.sync 2, 96;" ::: "memory");
                if (threadIdx.x == 0) JB_ACC(1, tb);
                JB_T0(tc);
                jb_chain_window(a, sh, p, m, seq, app);
                __syncwarp();
                asm volatile("bar.sync 4, 64;" ::: "memory");  // hand the ring to the lookahead
                if (m == nw - 1 && threadIdx.x == 0) sh.dg[p] = app;
                if (threadIdx.x == 0) JB_ACC(0, tc);
            } else {
                JB_T0(tl);
                jb_lookahead(a, sh, p, m, seq, start, prev_start, prev_nw);
                if (threadIdx.x == 32) JB_ACC(2, tl);
            }
            JB_T0(te);
            __syncthreads();
            if (threadIdx.x == 0) {
                JB_ACC(7, te);
#ifdef SGP_JBIG_PROF
                atomicAdd(&jb_prof[8], 1ull);
#endif
            }
            pp = p;
            pm = m;
            pnw = nw;
        }
        prev_start = start;
        prev_nw = nw;
    }
    if (warp >= 2) {
        if (pp >= 0) jb_publish(a, sh, pp, pm, pnw, seq - 1, io_t);
        for (int i = io_t; i < d; i += 64) __stcg(a.dg + i, sh.dg[i]);
    }
}

// ---------------------------------------------------------------------------
// owner CTAs: rows [klo, khi) minus the chain CTA's rows, one published window at a time

__device__ void jb_owner_cta(const JbArgs &a, double *smem) {
    const int d = a.d, c = blockIdx.x - 1;
    const int rpo = (d + a.nown - 1) / a.nown;
    const int klo = c * rpo, khi = min(d, klo + rpo);
    double *rc = smem, *rs = smem + JB_W;
    int *rf = reinterpret_cast<int *>(smem + 2 * JB_W);
    int *anyrot = rf + JB_W;
    volatile unsigned *pub_cache = reinterpret_cast<volatile unsigned *>(anyrot + 1);
    volatile unsigned *own_cache = pub_cache + 1;
    if (threadIdx.x == 0) {
        *pub_cache = 0u;
        *own_cache = 0u;
    }
    __syncthreads();
    unsigned seq = 1;
    for (int p = 0; p < d - 1; ++p) {
        const int nw = jb_nw(d, p);
        const unsigned start = seq;
        for (int m = 0; m < nw; ++m, ++seq) {
            const int q0 = p + 1 + JB_W * m, n = min(JB_W, d - q0);
            const bool last = m == nw - 1;
            if (threadIdx.x == 0 && *pub_cache < seq) {
                unsigned v;
                while ((v = jb_ld_acquire(a.pub)) < seq) __nanosleep(32);
                *pub_cache = v;
            }
            // What this window reads was last written (a) by any owner anywhere in pass p-1,
            // or (b) in pass p by the chain CTA (covered by pub >= seq) or by an owner at the
            // window of the element's earlier index, three or more windows back.  So: every
            // owner past pass p-1 for the first three windows of a pass, else past seq - 3.
            if (threadIdx.x < 32) jb_wait_owners(a, m >= 3 ? seq - 3 : start - 1, own_cache);
            __syncthreads();
            if (threadIdx.x < 32) {
                const int j = threadIdx.x;
                const size_t slot = jb_slot(d, p) + (size_t)JB_W * m + j;
                int f = 0;
                if (j < n) {
                    f = __ldcg(a.logf + slot);
                    rc[j] = __ldcg(a.logcs + 2 * slot);
                    rs[j] = __ldcg(a.logcs + 2 * slot + 1);
                }
                rf[j] = f;
                const unsigned b = __ballot_sync(0xffffffffu, f != 0);
                if (j == 0) *anyrot = b != 0u;
            }
            __syncthreads();
            const bool any = *anyrot != 0;
            for (int k = klo + (int)threadIdx.x; k < khi; k += JB_NT) {
                if (k == p || (k >= q0 && k < q0 + 3 * JB_W)) continue;  // chain CTA rows
                double *colp = k > p ? a.L + (size_t)k * d + p : a.L + (size_t)p * d + k;
                if (!any) {
                    if (m == 0 && !last) __stcg(a.R + k, __ldcg(colp));
                    else if (m > 0 && last) __stcg(colp, __ldcg(a.R + k));
                    continue;
                }
                double r = (m == 0) ? __ldcg(colp) : __ldcg(a.R + k);
                double e[JB_W];
                if (k < q0) {  // a_kq = L[q][k]: one element of each window row
                    const double *src = a.L + (size_t)q0 * d + k;
#pragma unroll
                    for (int j = 0; j < JB_W; ++j) e[j] = j < n ? __ldcg(src + (size_t)j * d) : 0.0;
                } else {  // a_kq = L[k][q]: one contiguous segment of row k
                    const double *src = a.L + (size_t)k * d + q0;
#pragma unroll
                    for (int j = 0; j < JB_W; ++j) e[j] = j < n ? __ldcg(src + j) : 0.0;
                }
#pragma unroll
                for (int j = 0; j < JB_W; ++j) {
                    if (rf[j]) {
                        const double cj = rc[j], sj = rs[j];
                        const double akp = r, akq = e[j];
                        r = __dsub_rn(__dmul_rn(cj, akp), __dmul_rn(sj, akq));
                        e[j] = __dadd_rn(__dmul_rn(sj, akp), __dmul_rn(cj, akq));
                    }
                }
                if (k < q0) {
                    double *dst = a.L + (size_t)q0 * d + k;
#pragma unroll
                    for (int j = 0; j < JB_W; ++j)
                        if (j < n && rf[j]) __stcg(dst + (size_t)j * d, e[j]);
                } else {
                    double *dst = a.L + (size_t)k * d + q0;
#pragma unroll
                    for (int j = 0; j < JB_W; ++j)
                        if (j < n && rf[j]) __stcg(dst + j, e[j]);
                }
                if (last)
                    __stcg(colp, r);
                else
                    __stcg(a.R + k, r);
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) jb_st_release(a.prog + c, seq);
        }
    }
}

__global__ void __launch_bounds__(JB_NT) k_jb_sweep(JbArgs a) {
    extern __shared__ __align__(16) double jb_smem[];
    if (blockIdx.x == 0)
        jb_chain_cta(a, jb_smem);
    else
        jb_owner_cta(a, jb_smem);
}

static size_t jb_smem_bytes(int d) {
    return sizeof(double) * ((size_t)((d + 1) & ~1) + 2 * (JB_W * JB_LDB + 1) + 4 * JB_W + 3 * JB_W) +
           sizeof(int) * (2 * JB_W + 8);
}

// Eigenvector update (_jacobi.py:81-85) on Vt = V^T: element (k, p) of V is Vt[p][k].  Thread
// k walks the sweep's log in order; within a pass every rotation shares p, so v_kp is carried
// in a register and the 32 v_kq of a log batch are loaded ahead (distinct q: no aliasing).
__global__ void __launch_bounds__(32) k_jb_vapply(double *__restrict__ Vt, const double *__restrict__ logcs,
                                                  const int *__restrict__ logf, int d) {
    const int lane = threadIdx.x, k = blockIdx.x * 32 + lane;
    const bool valid = k < d;
    const int kk = valid ? k : d - 1;
    for (int p = 0; p < d - 1; ++p) {
        double vp = __ldcg(Vt + (size_t)p * d + kk);
        size_t slot = jb_slot(d, p);
        for (int q0 = p + 1; q0 < d; q0 += 32, slot += 32) {
            const int nb = min(32, d - q0);
            int f = 0;
            double c = 0.0, s = 0.0;
            if (lane < nb) {
                f = __ldcg(logf + slot + lane);
                c = __ldcg(logcs + 2 * (slot + lane));
                s = __ldcg(logcs + 2 * (slot + lane) + 1);
            }
            const unsigned mask = __ballot_sync(0xffffffffu, f != 0);
            if (!mask) continue;
            double *col = Vt + (size_t)q0 * d + kk;
#pragma unroll
            for (int h = 0; h < 32; h += 16) {
                if (!((mask >> h) & 0xffffu)) continue;
                double vq[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    vq[j] = ((mask >> (h + j)) & 1u) ? __ldcg(col + (size_t)(h + j) * d) : 0.0;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double cj = __shfl_sync(0xffffffffu, c, h + j), sj = __shfl_sync(0xffffffffu, s, h + j);
                    if ((mask >> (h + j)) & 1u) {
                        const double nvp = __dsub_rn(__dmul_rn(cj, vp), __dmul_rn(sj, vq[j]));
                        vq[j] = __dadd_rn(__dmul_rn(sj, vp), __dmul_rn(cj, vq[j]));
                        vp = nvp;
                    }
                }
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if ((mask >> (h + j)) & 1u) __stcg(col + (size_t)(h + j) * d, vq[j]);
                }
            }
        }
        if (valid) __stcg(Vt + (size_t)p * d + kk, vp);
    }
}

// deterministic sum of squares of the strict lower triangle (one partial per CTA)
__global__ void k_jb_offpart(const double *L, int d, double *part) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int i = blockIdx.x; i < d; i += gridDim.x) {
        const double *row = L + (size_t)i * d;
        for (int j = threadIdx.x; j < i; j += blockDim.x) acc += row[j] * row[j];
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}
__global__ void k_jb_offfin(const double *part, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += part[i];
        *out = sqrt(2.0 * t);
    }
}
__global__ void k_jb_diag(double *A, double *dg, int d, int to_dg) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
        if (to_dg)
            dg[i] = A[(size_t)i * d + i];
        else
            A[(size_t)i * d + i] = dg[i];
    }
}
__global__ void k_jb_transpose(double *dst, const double *src, int d) {
    __shared__ double t[32][33];
    const int nt = (d + 31) / 32;
    for (int tile = blockIdx.x; tile < nt * nt; tile += gridDim.x) {
        const int bi = tile / nt, bj = tile % nt;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = bi * 32 + r, j = bj * 32 + threadIdx.x;
            if (i < d && j < d) t[r][threadIdx.x] = src[(size_t)i * d + j];
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = bj * 32 + r, j = bi * 32 + threadIdx.x;
            if (i < d && j < d) dst[(size_t)i * d + j] = t[threadIdx.x][r];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host driver

struct JbWS {
    int d = 0, nown = 0;
    double *Vt = nullptr, *R = nullptr, *dg = nullptr, *logcs[2] = {nullptr, nullptr}, *part = nullptr,
           *off = nullptr, *off_h = nullptr;
    int *logf[2] = {nullptr, nullptr};
    unsigned *cnt = nullptr;
    cudaStream_t s2 = nullptr;
    cudaEvent_t evA[2] = {nullptr, nullptr}, evV[2] = {nullptr, nullptr};
    size_t smem = 0;
};

static void jb_ws_free(JbWS &w) {
    cudaFree(w.Vt);
    cudaFree(w.R);
    cudaFree(w.dg);
    cudaFree(w.part);
    cudaFree(w.off);
    cudaFree(w.cnt);
    for (int b = 0; b < 2; ++b) {
        cudaFree(w.logcs[b]);
        cudaFree(w.logf[b]);
        if (w.evA[b]) cudaEventDestroy(w.evA[b]);
        if (w.evV[b]) cudaEventDestroy(w.evV[b]);
    }
    if (w.off_h) cudaFreeHost(w.off_h);
    if (w.s2) cudaStreamDestroy(w.s2);
    w = JbWS();
}

#define JB_NPART 148
static int jb_ws_alloc(JbWS &w, int d) {
    if (w.d == d) return 0;
    jb_ws_free(w);
    const size_t E = (size_t)d * (d - 1) / 2 + 64;
    w.d = d;
    w.nown = std::min(JB_MAX_OWN, std::max(1, (d + JB_NT - 1) / JB_NT));
    bool ok = cudaMalloc(&w.Vt, sizeof(double) * (size_t)d * d) == cudaSuccess &&
              cudaMalloc(&w.R, sizeof(double) * d) == cudaSuccess &&
              cudaMalloc(&w.dg, sizeof(double) * d) == cudaSuccess &&
              cudaMalloc(&w.part, sizeof(double) * JB_NPART) == cudaSuccess &&
              cudaMalloc(&w.off, sizeof(double)) == cudaSuccess &&
              cudaMalloc(&w.cnt, sizeof(unsigned) * (1 + JB_MAX_OWN)) == cudaSuccess &&
              cudaMallocHost(&w.off_h, sizeof(double)) == cudaSuccess &&
              cudaStreamCreateWithFlags(&w.s2, cudaStreamNonBlocking) == cudaSuccess;
    for (int b = 0; ok && b < 2; ++b) {
        ok = cudaMalloc(&w.logcs[b], sizeof(double) * 2 * E) == cudaSuccess &&
             cudaMalloc(&w.logf[b], sizeof(int) * E) == cudaSuccess &&
             cudaEventCreateWithFlags(&w.evA[b], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&w.evV[b], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventRecord(w.evV[b], w.s2) == cudaSuccess;
    }
    w.smem = jb_smem_bytes(d);
    if (ok && w.smem > 48 * 1024)
        ok = cudaFuncSetAttribute(k_jb_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w.smem) == cudaSuccess;
    if (!ok) {
        jb_ws_free(w);
        return -1;
    }
    return 0;
}

// Cyclic Jacobi in the reference order on the symmetric d x d matrix A (row-major, lower
// triangle read), accumulating into V (row-major, columns = basis).  On return A's diagonal
// holds the eigenvalues (the strict lower triangle the rotated matrix, the upper triangle is
// stale) and V = V_in J.  Returns the completed sweeps, or -1 at the cap (_jacobi.py:37-86),
// or -2 on a CUDA error.  The off-norm test runs on the host between sweeps.
static int jb_jacobi(JbWS &w, double *A, double *V, int d, double tol, double skip, int cap, cudaStream_t s) {
    if (d < 2) return 0;
    if (jb_ws_alloc(w, d)) return -2;
    const int nt = (d + 31) / 32;
    const int tg = std::min(nt * nt, 148 * 8);
    k_jb_diag<<<std::min((d + 255) / 256, 148), 256, 0, s>>>(A, w.dg, d, 1);
    k_jb_transpose<<<tg, dim3(32, 8), 0, s>>>(w.Vt, V, d);
    int sw = 0;
    int rc = 0;
    for (;;) {
        k_jb_offpart<<<JB_NPART, 256, 0, s>>>(A, d, w.part);
        k_jb_offfin<<<1, 32, 0, s>>>(w.part, JB_NPART, w.off);
        cudaMemcpyAsync(w.off_h, w.off, sizeof(double), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) {
            rc = -2;
            break;
        }
        if (*w.off_h <= tol) {
            rc = sw;
            break;
        }
        if (sw >= cap) {
            rc = -1;
            break;
        }
        const int b = sw & 1;
        cudaStreamWaitEvent(s, w.evV[b], 0);  // the V update of sweep sw-2 has consumed log b
        cudaMemsetAsync(w.cnt, 0, sizeof(unsigned) * (1 + JB_MAX_OWN), s);
        JbArgs a;
        a.L = A;
        a.dg = w.dg;
        a.R = w.R;
        a.logcs = w.logcs[b];
        a.logf = w.logf[b];
        a.pub = w.cnt;
        a.prog = w.cnt + 1;
        a.d = d;
        a.nown = w.nown;
        a.skip = skip;
        void *args[] = {&a};
        static const bool dbg = getenv("SGP_DEBUG_JBIG") != nullptr;
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        if (dbg) {
            cudaEventCreate(&t0);
            cudaEventCreate(&t1);
            cudaEventRecord(t0, s);
        }
        if (cudaLaunchCooperativeKernel((const void *)k_jb_sweep, dim3(1 + w.nown), dim3(JB_NT), args, w.smem, s) !=
            cudaSuccess) {
            rc = -2;
            break;
        }
        if (dbg) {  // diagnostics: sweep time against rotations applied
            cudaEventRecord(t1, s);
            cudaEventSynchronize(t1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            const size_t E = (size_t)d * (d - 1) / 2;
            std::vector<int> f(E);
            cudaMemcpy(f.data(), w.logf[b], sizeof(int) * E, cudaMemcpyDeviceToHost);
            long nrot = 0;
            for (int v : f) nrot += v;
            fprintf(stderr, "jbig d=%d sweep %d: %.1f ms, %ld of %zu rotations (%.3f us/rotation)\n", d, sw, ms, nrot, E,
                    nrot ? 1e3 * ms / nrot : 0.0);
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
        }
        cudaEventRecord(w.evA[b], s);
        cudaStreamWaitEvent(w.s2, w.evA[b], 0);
        k_jb_vapply<<<(d + 31) / 32, 32, 0, w.s2>>>(w.Vt, w.logcs[b], w.logf[b], d);
        cudaEventRecord(w.evV[b], w.s2);
        ++sw;
    }
    for (int b = 0; b < 2; ++b) cudaStreamWaitEvent(s, w.evV[b], 0);
    k_jb_diag<<<std::min((d + 255) / 256, 148), 256, 0, s>>>(A, w.dg, d, 0);
    k_jb_transpose<<<tg, dim3(32, 8), 0, s>>>(V, w.Vt, d);
    if (cudaGetLastError() != cudaSuccess) rc = -2;
    return rc;
}
