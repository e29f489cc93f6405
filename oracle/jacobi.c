/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's compiled
 * Jacobi kernels, used as the parity checker for the CUDA eigensolvers.
 * Nothing in paper_2511_06407_b200/ links or loads this file.
 *
 * Follows /root/reference/pkg/src/softabs_gp/_jacobi.py:
 *   off_diagonal_norm      _jacobi.py:26-34
 *   jacobi_sweeps          _jacobi.py:37-86   (cyclic-by-row, threshold skip,
 *                                              convergence test before each sweep)
 *   modified_gram_schmidt  _jacobi.py:89-107
 * The reference is Numba-compiled without FMA contraction; this file must be
 * compiled with -ffp-contract=off (see oracle/Makefile) so every rotation is
 * rounded exactly as the reference rounds it.
 */
#include <math.h>
#include <stddef.h>

double oracle_off_norm(const double *a, long d)
{
    double acc = 0.0;
    for (long r = 0; r < d; ++r)
        for (long c = 0; c < d; ++c)
            if (r != c) acc += a[r * d + c] * a[r * d + c];
    return sqrt(acc);
}

/* Returns completed sweeps, or -1 when max_sweeps ran out. */
long oracle_jacobi_sweeps(double *a, double *v, long d, double tol, double skip,
                          long max_sweeps)
{
    long done = 0;
    for (;;) {
        if (oracle_off_norm(a, d) <= tol) return done;
        if (done >= max_sweeps) return -1;
        for (long p = 0; p + 1 < d; ++p) {
            for (long q = p + 1; q < d; ++q) {
                const double apq = a[p * d + q];
                if (fabs(apq) <= skip) continue;
                const double theta = (a[q * d + q] - a[p * d + p]) / (2.0 * apq);
                double t;
                if (fabs(theta) > 1e154)
                    t = 0.5 / theta;
                else if (theta >= 0.0)
                    t = 1.0 / (theta + sqrt(1.0 + theta * theta));
                else
                    t = -1.0 / (-theta + sqrt(1.0 + theta * theta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = t * c;
                a[p * d + p] -= t * apq;
                a[q * d + q] += t * apq;
                a[p * d + q] = 0.0;
                a[q * d + p] = 0.0;
                for (long k = 0; k < d; ++k) {
                    if (k == p || k == q) continue;
                    const double akp = a[k * d + p];
                    const double akq = a[k * d + q];
                    a[k * d + p] = c * akp - s * akq;
                    a[p * d + k] = a[k * d + p];
                    a[k * d + q] = s * akp + c * akq;
                    a[q * d + k] = a[k * d + q];
                }
                for (long k = 0; k < d; ++k) {
                    const double vkp = v[k * d + p];
                    const double vkq = v[k * d + q];
                    v[k * d + p] = c * vkp - s * vkq;
                    v[k * d + q] = s * vkp + c * vkq;
                }
            }
        }
        ++done;
    }
}

/* Passes p0 .. p1-1 of one cyclic sweep (the body of _jacobi.py:54-85 for those pivot rows);
 * returns the number of rotations applied.  Used only to time a bounded sample of a sweep for
 * the CPU baseline at large d (bench.py); a full sweep is passes 0 .. d-2. */
long oracle_jacobi_passes(double *a, double *v, long d, long p0, long p1, double skip)
{
    long nrot = 0;
    for (long p = p0; p < p1 && p + 1 < d; ++p) {
        for (long q = p + 1; q < d; ++q) {
            const double apq = a[p * d + q];
            if (fabs(apq) <= skip) continue;
            const double theta = (a[q * d + q] - a[p * d + p]) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e154)
                t = 0.5 / theta;
            else if (theta >= 0.0)
                t = 1.0 / (theta + sqrt(1.0 + theta * theta));
            else
                t = -1.0 / (-theta + sqrt(1.0 + theta * theta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = t * c;
            a[p * d + p] -= t * apq;
            a[q * d + q] += t * apq;
            a[p * d + q] = 0.0;
            a[q * d + p] = 0.0;
            for (long k = 0; k < d; ++k) {
                if (k == p || k == q) continue;
                const double akp = a[k * d + p];
                const double akq = a[k * d + q];
                a[k * d + p] = c * akp - s * akq;
                a[p * d + k] = a[k * d + p];
                a[k * d + q] = s * akp + c * akq;
                a[q * d + k] = a[k * d + q];
            }
            for (long k = 0; k < d; ++k) {
                const double vkp = v[k * d + p];
                const double vkq = v[k * d + q];
                v[k * d + p] = c * vkp - s * vkq;
                v[k * d + q] = s * vkp + c * vkq;
            }
            ++nrot;
        }
    }
    return nrot;
}

void oracle_mgs(double *psi, long d)
{
    for (long i = 0; i < d; ++i) {
        double nrm = 0.0;
        for (long k = 0; k < d; ++k) nrm += psi[k * d + i] * psi[k * d + i];
        nrm = sqrt(nrm);
        if (nrm == 0.0) continue;
        for (long k = 0; k < d; ++k) psi[k * d + i] /= nrm;
        for (long j = i + 1; j < d; ++j) {
            double dot = 0.0;
            for (long k = 0; k < d; ++k) dot += psi[k * d + i] * psi[k * d + j];
            for (long k = 0; k < d; ++k) psi[k * d + j] -= dot * psi[k * d + i];
        }
    }
}
