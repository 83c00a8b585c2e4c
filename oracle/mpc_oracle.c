/*
 * mpc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's complex multi-component (DD/TD/QD)
 * expansion arithmetic, complex GEMM and blocked LU, used as the parity
 * checker for the CUDA product path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library;
 * the product package never links or calls it.
 *
 * Every routine follows the reference's numba kernels statement by statement
 * (file:line cited per function, paths relative to
 * /root/reference/pkg/src/mpclu/).  The reference runs under strict IEEE
 * binary64 with no FMA contraction (numba, no fastmath, _kernels.py:8-9), so
 * this file MUST be compiled with -ffp-contract=off and without -ffast-math
 * (see oracle/Makefile).  TwoProd uses Dekker splitting exactly as the
 * reference does (_kernels.py:45-60); the GPU uses FMA-TwoProd, which is
 * bit-identical for in-range inputs -- comparing the two is part of the pin.
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by importing the reference itself
 * (oracle/gen_golden.py -> tests/golden/).
 *
 * Layout: planar (k, rows, cols) row-major float64, one array per Re / Im
 * (rmatrix.py:1-7).  Sub-matrices are addressed with (ld, plane stride).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define SPLITTER 134217729.0 /* 2^27 + 1, _kernels.py:23 */
#define MAX_K 16             /* _kernels.py:25 */
#define SCRATCH(k) ((k) * (k) + 2 * (k) + 4) /* scratch_len, _kernels.py:268-271 */
#define SCRATCH_MAX (MAX_K * MAX_K + 2 * MAX_K + 4)

/* ---------------------------------------------------------------- EFTs */

/* _kernels.py:28-34 */
static inline void two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

/* _kernels.py:37-42 */
static inline void quick_two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    *e = b - (ss - a);
    *s = ss;
}

/* _kernels.py:45-60 (Dekker) */
static inline void two_prod(double a, double b, double *p, double *e) {
    double pp = a * b;
    double ca = SPLITTER * a;
    double ahi = ca - (ca - a);
    double alo = a - ahi;
    double cb = SPLITTER * b;
    double bhi = cb - (cb - b);
    double blo = b - bhi;
    *e = ((ahi * bhi - pp) + ahi * blo + alo * bhi) + alo * blo;
    *p = pp;
}

/* ------------------------------------------------------- renormalization */

/* _kernels.py:67-78: insertion sort by (|v| desc, v desc) */
static void sort_desc(double *buf, int m) {
    for (int i = 1; i < m; i++) {
        double v = buf[i];
        double av = fabs(v);
        int j = i - 1;
        while (j >= 0 && (fabs(buf[j]) < av || (fabs(buf[j]) == av && buf[j] < v))) {
            buf[j + 1] = buf[j];
            j--;
        }
        buf[j + 1] = v;
    }
}

/* _kernels.py:81-105 */
static void vecsum_extract(double *buf, int m, double *out, int k) {
    double s = buf[m - 1], e;
    for (int i = m - 2; i >= 0; i--) {
        two_sum(buf[i], s, &s, &e);
        buf[i + 1] = e;
    }
    buf[0] = s;
    for (int i = 0; i < k; i++) out[i] = 0.0;
    int j = 0;
    double eps = buf[0];
    for (int i = 0; i < m - 1; i++) {
        double r, enew;
        two_sum(eps, buf[i + 1], &r, &enew);
        if (enew != 0.0) {
            if (j >= k - 1) {
                eps = r;
                break;
            }
            out[j] = r;
            j++;
            eps = enew;
        } else {
            eps = r;
        }
    }
    out[j] = eps;
}

/* np.spacing for a non-negative argument */
static inline double spacing_pos(double x) { return nextafter(x, INFINITY) - x; }

/* _kernels.py:108-121 */
static int is_nonoverlapping(const double *out, int k) {
    for (int i = 0; i < k - 1; i++) {
        double hi = out[i], lo = out[i + 1];
        if (hi == 0.0) {
            if (lo != 0.0) return 0;
        } else if (fabs(lo) > 0.5 * spacing_pos(fabs(hi)) || hi + lo != hi) {
            return 0;
        }
    }
    return 1;
}

/* _kernels.py:124-139 */
void orc_renorm(double *buf, int m, double *out, int k) {
    sort_desc(buf, m);
    vecsum_extract(buf, m, out, k);
    int it = 0;
    while (!is_nonoverlapping(out, k) && it < 6) {
        for (int i = 0; i < k; i++) buf[i] = out[i];
        vecsum_extract(buf, k, out, k);
        it++;
    }
}

/* --------------------------------------------------------- DD fast paths */

/* _kernels.py:146-155 */
static inline void dd_add(double x0, double x1, double y0, double y1, double *r0, double *r1) {
    double s1, s2, t1, t2;
    two_sum(x0, y0, &s1, &s2);
    two_sum(x1, y1, &t1, &t2);
    s2 += t1;
    quick_two_sum(s1, s2, &s1, &s2);
    s2 += t2;
    quick_two_sum(s1, s2, &s1, &s2);
    *r0 = s1;
    *r1 = s2;
}

/* _kernels.py:158-164 */
static inline void dd_mul(double x0, double x1, double y0, double y1, double *r0, double *r1) {
    double p, e;
    two_prod(x0, y0, &p, &e);
    double t = x0 * y1 + x1 * y0;
    e += t + x1 * y1;
    quick_two_sum(p, e, &p, &e);
    *r0 = p;
    *r1 = e;
}

/* ------------------------------------------------- generic expansion ops */
/* out may alias x or y: inputs are consumed before out is written */

/* _kernels.py:174-184 */
void orc_exp_add(const double *x, const double *y, double *buf, double *out, int k) {
    if (k == 2) {
        double a, b;
        dd_add(x[0], x[1], y[0], y[1], &a, &b);
        out[0] = a;
        out[1] = b;
        return;
    }
    for (int i = 0; i < k; i++) {
        buf[i] = x[i];
        buf[k + i] = y[i];
    }
    orc_renorm(buf, 2 * k, out, k);
}

/* _kernels.py:187-197 */
void orc_exp_sub(const double *x, const double *y, double *buf, double *out, int k) {
    if (k == 2) {
        double a, b;
        dd_add(x[0], x[1], -y[0], -y[1], &a, &b);
        out[0] = a;
        out[1] = b;
        return;
    }
    for (int i = 0; i < k; i++) {
        buf[i] = x[i];
        buf[k + i] = -y[i];
    }
    orc_renorm(buf, 2 * k, out, k);
}

/* _kernels.py:200-222 */
void orc_exp_mul(const double *x, const double *y, double *buf, double *out, int k) {
    if (k == 2) {
        double a, b;
        dd_mul(x[0], x[1], y[0], y[1], &a, &b);
        out[0] = a;
        out[1] = b;
        return;
    }
    int m = 0;
    for (int s = 0; s < k - 1; s++) {
        for (int i = 0; i < s + 1; i++) {
            double p, e;
            two_prod(x[i], y[s - i], &p, &e);
            buf[m] = p;
            buf[m + 1] = e;
            m += 2;
        }
    }
    for (int i = 0; i < k; i++) buf[m++] = x[i] * y[k - 1 - i];
    for (int i = 1; i < k; i++) buf[m++] = x[i] * y[k - i];
    orc_renorm(buf, m, out, k);
}

/* _kernels.py:225-255 */
void orc_exp_div(const double *x, const double *y, double *buf, double *out, int k) {
    double q[MAX_K + 2], r[MAX_K] = {0}, t[MAX_K];
    for (int i = 0; i < k; i++) r[i] = x[i];
    int nq = 0;
    for (int it = 0; it < k + 1; it++) {
        double qi = r[0] / y[0];
        q[nq++] = qi;
        if (qi == 0.0 || it == k) break;
        int m = 0;
        for (int i = 0; i < k; i++) buf[m++] = r[i];
        for (int i = 0; i < k; i++) {
            double p, e;
            two_prod(qi, y[i], &p, &e);
            buf[m] = -p;
            buf[m + 1] = -e;
            m += 2;
        }
        orc_renorm(buf, m, t, k);
        for (int i = 0; i < k; i++) r[i] = t[i];
    }
    for (int i = 0; i < nq; i++) buf[i] = q[i];
    orc_renorm(buf, nq, out, k);
}

/* _kernels.py:258-265 */
static inline void exp_abs(const double *x, double *out, int k) {
    if (x[0] < 0.0)
        for (int i = 0; i < k; i++) out[i] = -x[i];
    else
        for (int i = 0; i < k; i++) out[i] = x[i];
}

/* ----------------------------------------------------- complex scalars */

/* _kernels.py:527-537 */
void orc_cmul_3m(const double *ar, const double *ai, const double *br, const double *bi,
                 double *outr, double *outi, int k) {
    double s1[MAX_K], s2[MAX_K], s3[MAX_K], buf[SCRATCH_MAX];
    orc_exp_mul(ar, br, buf, s1, k);
    orc_exp_mul(ai, bi, buf, s2, k);
    orc_exp_sub(s1, s2, buf, outr, k);
    orc_exp_add(ar, ai, buf, s3, k);
    orc_exp_add(br, bi, buf, outi, k);
    orc_exp_mul(s3, outi, buf, s3, k);
    orc_exp_sub(s3, s1, buf, s3, k);
    orc_exp_sub(s3, s2, buf, outi, k);
}

/* _kernels.py:539-546 */
void orc_cmul_4m(const double *ar, const double *ai, const double *br, const double *bi,
                 double *outr, double *outi, int k) {
    double s1[MAX_K], s2[MAX_K], buf[SCRATCH_MAX];
    orc_exp_mul(ar, br, buf, s1, k);
    orc_exp_mul(ai, bi, buf, s2, k);
    orc_exp_sub(s1, s2, buf, outr, k);
    orc_exp_mul(ai, br, buf, s1, k);
    orc_exp_mul(ar, bi, buf, s2, k);
    orc_exp_add(s1, s2, buf, outi, k);
}

/* _kernels.py:549-561 */
void orc_cdiv(const double *ar, const double *ai, const double *br, const double *bi,
              double *outr, double *outi, int k) {
    double s1[MAX_K], s2[MAX_K], s3[MAX_K], buf[SCRATCH_MAX];
    orc_exp_mul(br, br, buf, s1, k);
    orc_exp_mul(bi, bi, buf, s2, k);
    orc_exp_add(s1, s2, buf, s1, k);
    orc_exp_mul(ar, br, buf, s2, k);
    orc_exp_mul(ai, bi, buf, s3, k);
    orc_exp_add(s2, s3, buf, s2, k);
    orc_exp_mul(ai, br, buf, s3, k);
    orc_exp_mul(ar, bi, buf, outi, k);
    orc_exp_sub(s3, outi, buf, s3, k);
    orc_exp_div(s2, s1, buf, outr, k);
    orc_exp_div(s3, s1, buf, outi, k);
}

static inline void cmul(int use3m, const double *ar, const double *ai, const double *br,
                        const double *bi, double *outr, double *outi, int k) {
    if (use3m)
        orc_cmul_3m(ar, ai, br, bi, outr, outi, k);
    else
        orc_cmul_4m(ar, ai, br, bi, outr, outi, k);
}

/* ------------------------------------------------------ matrix kernels */
/* element (c, i, j) of a planar view: base[c*ps + i*ld + j] */
#define AT(base, c, i, j, ld, ps) ((base)[(int64_t)(c) * (ps) + (int64_t)(i) * (ld) + (j)])

/* mat_add_k, _kernels.py:327-342.  C = A + sign*B (sign = +-1). */
void orc_mat_add(int k, int64_t m, int64_t n, const double *A, int64_t lda, int64_t psa,
                 const double *B, int64_t ldb, int64_t psb, double *C, int64_t ldc,
                 int64_t psc, double sign) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        double x[MAX_K], y[MAX_K], out[MAX_K], buf[SCRATCH_MAX];
        for (int64_t j = 0; j < n; j++) {
            for (int c = 0; c < k; c++) {
                x[c] = AT(A, c, i, j, lda, psa);
                y[c] = sign * AT(B, c, i, j, ldb, psb);
            }
            orc_exp_add(x, y, buf, out, k);
            for (int c = 0; c < k; c++) AT(C, c, i, j, ldc, psc) = out[c];
        }
    }
}

/* rgemm_naive_k + _gemm_row_run, _kernels.py:363-395.  C = A B, fresh chain
 * acc = 0; for t ascending: acc = add(acc, mul(A[i,t], B[t,j])). */
void orc_rgemm(int k, int64_t m, int64_t n, int64_t l, const double *A, int64_t lda,
               int64_t psa, const double *B, int64_t ldb, int64_t psb, double *C,
               int64_t ldc, int64_t psc) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; i++) {
        double acc[MAX_K], x[MAX_K], y[MAX_K], out[MAX_K], buf[SCRATCH_MAX];
        for (int64_t j = 0; j < l; j++) {
            for (int c = 0; c < k; c++) acc[c] = 0.0;
            for (int64_t t = 0; t < n; t++) {
                for (int c = 0; c < k; c++) {
                    x[c] = AT(A, c, i, t, lda, psa);
                    y[c] = AT(B, c, t, j, ldb, psb);
                }
                orc_exp_mul(x, y, buf, out, k);
                orc_exp_add(acc, out, buf, acc, k);
            }
            for (int c = 0; c < k; c++) AT(C, c, i, j, ldc, psc) = acc[c];
        }
    }
}

/* cgemm_3m / cgemm_4m, cmatrix.py:145-169, composed from real products and
 * plane additions exactly as the reference does (temporaries per call).
 * Output planes are contiguous (k, m, l). */
void orc_cgemm(int k, int method, int64_t m, int64_t n, int64_t l, const double *are,
               const double *aim, int64_t lda, int64_t psa, const double *bre,
               const double *bim, int64_t ldb, int64_t psb, double *cre, double *cim) {
    int64_t pc = m * l;
    double *t1 = malloc(sizeof(double) * k * pc);
    double *t2 = malloc(sizeof(double) * k * pc);
    double *t3 = malloc(sizeof(double) * k * pc);
    if (method == 3) {
        double *sa = malloc(sizeof(double) * k * m * n);
        double *sb = malloc(sizeof(double) * k * n * l);
        orc_rgemm(k, m, n, l, are, lda, psa, bre, ldb, psb, t1, l, pc);
        orc_rgemm(k, m, n, l, aim, lda, psa, bim, ldb, psb, t2, l, pc);
        orc_mat_add(k, m, n, are, lda, psa, aim, lda, psa, sa, n, m * n, 1.0);
        orc_mat_add(k, n, l, bre, ldb, psb, bim, ldb, psb, sb, l, n * l, 1.0);
        orc_rgemm(k, m, n, l, sa, n, m * n, sb, l, n * l, t3, l, pc);
        orc_mat_add(k, m, l, t1, l, pc, t2, l, pc, cre, l, pc, -1.0);
        orc_mat_add(k, m, l, t3, l, pc, t1, l, pc, t3, l, pc, -1.0);
        orc_mat_add(k, m, l, t3, l, pc, t2, l, pc, cim, l, pc, -1.0);
        free(sa);
        free(sb);
    } else {
        double *t4 = malloc(sizeof(double) * k * pc);
        orc_rgemm(k, m, n, l, are, lda, psa, bre, ldb, psb, t1, l, pc); /* rr */
        orc_rgemm(k, m, n, l, aim, lda, psa, bim, ldb, psb, t2, l, pc); /* ii */
        orc_rgemm(k, m, n, l, aim, lda, psa, bre, ldb, psb, t3, l, pc); /* ir */
        orc_rgemm(k, m, n, l, are, lda, psa, bim, ldb, psb, t4, l, pc); /* ri */
        orc_mat_add(k, m, l, t1, l, pc, t2, l, pc, cre, l, pc, -1.0);
        orc_mat_add(k, m, l, t3, l, pc, t4, l, pc, cim, l, pc, 1.0);
        free(t4);
    }
    free(t1);
    free(t2);
    free(t3);
}

/* renorm_planes, _kernels.py:485-499 (in place, contiguous (k, m, n)) */
void orc_renorm_planes(int k, int64_t m, int64_t n, double *R) {
    int64_t ps = m * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        double out[MAX_K], buf[SCRATCH_MAX];
        for (int64_t j = 0; j < n; j++) {
            for (int c = 0; c < k; c++) buf[c] = R[c * ps + i * n + j];
            orc_renorm(buf, k, out, k);
            for (int c = 0; c < k; c++) R[c * ps + i * n + j] = out[c];
        }
    }
}

/* acc_plane, _kernels.py:502-517 */
void orc_acc_plane(int k, int64_t m, int64_t n, double *C, const double *P) {
    int64_t ps = m * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        double h[MAX_K + 1];
        for (int64_t j = 0; j < n; j++) {
            double q = P[i * n + j], e;
            for (int c = k - 1; c >= 0; c--) {
                two_sum(q, C[c * ps + i * n + j], &q, &e);
                h[c + 1] = e;
            }
            h[0] = q;
            for (int c = 0; c < k; c++) C[c * ps + i * n + j] = h[c];
        }
    }
}

/* ------------------------------------------------------------------ LU */
/* square n x n planar matrices, contiguous planes (k, n, n) */

/* _pivot_row, _kernels.py:568-594 */
static int64_t pivot_row(const double *re, const double *im, int64_t j, int k, int64_t n) {
    int64_t best = -1;
    double bs[MAX_K], cand[MAX_K], t[MAX_K], u[MAX_K], buf[SCRATCH_MAX];
    int64_t ps = n * n;
    int nz = 0;
    for (int c = 0; c < k; c++) bs[c] = 0.0;
    for (int64_t i = j; i < n; i++) {
        for (int c = 0; c < k; c++) {
            t[c] = re[c * ps + i * n + j];
            u[c] = im[c * ps + i * n + j];
        }
        exp_abs(t, t, k);
        exp_abs(u, u, k);
        orc_exp_add(t, u, buf, cand, k);
        orc_exp_sub(cand, bs, buf, t, k);
        if (t[0] > 0.0) {
            best = i;
            for (int c = 0; c < k; c++) bs[c] = cand[c];
            nz = 1;
        }
    }
    if (!nz) return -1;
    return best;
}

/* _swap_rows, _kernels.py:597-608 */
static void swap_rows(double *re, double *im, int k, int64_t r1, int64_t r2, int64_t n) {
    if (r1 == r2) return;
    int64_t ps = n * n;
    for (int c = 0; c < k; c++) {
        for (int64_t j = 0; j < n; j++) {
            double tmp = re[c * ps + r1 * n + j];
            re[c * ps + r1 * n + j] = re[c * ps + r2 * n + j];
            re[c * ps + r2 * n + j] = tmp;
            tmp = im[c * ps + r1 * n + j];
            im[c * ps + r1 * n + j] = im[c * ps + r2 * n + j];
            im[c * ps + r2 * n + j] = tmp;
        }
    }
}

/* lu_panel, _kernels.py:611-665.  Returns -1 or the singular column. */
int64_t orc_lu_panel(int k, int use3m, int64_t n, double *re, double *im, int64_t *piv,
                     int64_t jb, int64_t kw) {
    int64_t ps = n * n;
    for (int64_t j = jb; j < jb + kw; j++) {
        int64_t p = pivot_row(re, im, j, k, n);
        if (p < 0) return j;
        swap_rows(re, im, k, j, p, n);
        piv[j] = p;
#pragma omp parallel for schedule(static)
        for (int64_t i = j + 1; i < n; i++) {
            double ar[MAX_K], ai[MAX_K], br[MAX_K], bi[MAX_K], lr[MAX_K], li[MAX_K];
            double pr[MAX_K], pi[MAX_K], buf[SCRATCH_MAX];
            for (int c = 0; c < k; c++) {
                ar[c] = re[c * ps + i * n + j];
                ai[c] = im[c * ps + i * n + j];
                br[c] = re[c * ps + j * n + j];
                bi[c] = im[c * ps + j * n + j];
            }
            orc_cdiv(ar, ai, br, bi, lr, li, k);
            for (int c = 0; c < k; c++) {
                re[c * ps + i * n + j] = lr[c];
                im[c * ps + i * n + j] = li[c];
            }
            for (int64_t t = j + 1; t < jb + kw; t++) {
                for (int c = 0; c < k; c++) {
                    br[c] = re[c * ps + j * n + t];
                    bi[c] = im[c * ps + j * n + t];
                }
                cmul(use3m, lr, li, br, bi, pr, pi, k);
                for (int c = 0; c < k; c++) {
                    ar[c] = re[c * ps + i * n + t];
                    ai[c] = im[c * ps + i * n + t];
                }
                orc_exp_sub(ar, pr, buf, ar, k);
                orc_exp_sub(ai, pi, buf, ai, k);
                for (int c = 0; c < k; c++) {
                    re[c * ps + i * n + t] = ar[c];
                    im[c * ps + i * n + t] = ai[c];
                }
            }
        }
    }
    return -1;
}

/* trsm_ll_unit, _kernels.py:668-705.  L is K x K (ldl, psl), A is K x M
 * (lda, psa), solved in place. */
void orc_trsm_ll_unit(int k, int use3m, int64_t K, int64_t M, const double *lre,
                      const double *lim, int64_t ldl, int64_t psl, double *are, double *aim,
                      int64_t lda, int64_t psa) {
#pragma omp parallel for schedule(static)
    for (int64_t col = 0; col < M; col++) {
        double xr[MAX_K], xi[MAX_K], yr[MAX_K], yi[MAX_K], lr[MAX_K], li[MAX_K];
        double pr[MAX_K], pi[MAX_K], buf[SCRATCH_MAX];
        for (int64_t r = 1; r < K; r++) {
            for (int c = 0; c < k; c++) {
                xr[c] = AT(are, c, r, col, lda, psa);
                xi[c] = AT(aim, c, r, col, lda, psa);
            }
            for (int64_t s = 0; s < r; s++) {
                for (int c = 0; c < k; c++) {
                    lr[c] = AT(lre, c, r, s, ldl, psl);
                    li[c] = AT(lim, c, r, s, ldl, psl);
                    yr[c] = AT(are, c, s, col, lda, psa);
                    yi[c] = AT(aim, c, s, col, lda, psa);
                }
                cmul(use3m, lr, li, yr, yi, pr, pi, k);
                orc_exp_sub(xr, pr, buf, xr, k);
                orc_exp_sub(xi, pi, buf, xi, k);
            }
            for (int c = 0; c < k; c++) {
                AT(are, c, r, col, lda, psa) = xr[c];
                AT(aim, c, r, col, lda, psa) = xi[c];
            }
        }
    }
}

/* lu._factor, lu.py:129-163 (in place on re/im; piv preset to arange by the
 * caller, as lu.py:134).  Returns -1 or the singular column. */
/* The panels jb in [jb0, jb1) of lu._factor's loop (jb0 a multiple of K): a
 * long factorization can be run in stages, the matrix and piv carried over
 * (oracle/gen_cfg4.py --stage).  orc_factor is the whole range. */
int64_t orc_factor_range(int k, int use3m, int64_t n, int64_t K, double *re, double *im,
                         int64_t *piv, int64_t jb0, int64_t jb1) {
    int64_t ps = n * n;
    for (int64_t jb = jb0; jb < n && jb < jb1; jb += K) {
        int64_t kw = (K < n - jb) ? K : n - jb;
        int64_t status = orc_lu_panel(k, use3m, n, re, im, piv, jb, kw);
        if (status >= 0) return status;
        int64_t end = jb + kw;
        if (end == n) break;
        int64_t M = n - end;
        /* TRSM in place on the A12 block (identical arithmetic to the copy
         * the reference makes at lu.py:145-151) */
        orc_trsm_ll_unit(k, use3m, kw, M, re + jb * n + jb, im + jb * n + jb, n, ps,
                         re + jb * n + end, im + jb * n + end, n, ps);
        /* P = cgemm(L21, U12), then A22 = A22 - P (lu.py:152-161) */
        double *pre = malloc(sizeof(double) * k * M * M);
        double *pim = malloc(sizeof(double) * k * M * M);
        orc_cgemm(k, use3m ? 3 : 4, M, kw, M, re + end * n + jb, im + end * n + jb, n, ps,
                  re + jb * n + end, im + jb * n + end, n, ps, pre, pim);
        orc_mat_add(k, M, M, re + end * n + end, n, ps, pre, M, M * M, re + end * n + end, n,
                    ps, -1.0);
        orc_mat_add(k, M, M, im + end * n + end, n, ps, pim, M, M * M, im + end * n + end, n,
                    ps, -1.0);
        free(pre);
        free(pim);
    }
    return -1;
}

int64_t orc_factor(int k, int use3m, int64_t n, int64_t K, double *re, double *im,
                   int64_t *piv) {
    return orc_factor_range(k, use3m, n, K, re, im, piv, 0, n);
}

/* solve_fb, _kernels.py:708-775 (b overwritten by x; vectors (k, n)) */
/* phases: 1 = interchanges + forward sweep, 2 = backward sweep, 3 = both
 * (solve_fb itself) -- the halves checked separately by the GPU tests. */
void orc_solve_phases(int k, int use3m, int64_t n, const double *re, const double *im,
                      const int64_t *piv, double *br, double *bi, int phases) {
    int64_t ps = n * n;
    for (int64_t i = 0; (phases & 1) && i < n; i++) {
        int64_t p = piv[i];
        if (p != i) {
            for (int c = 0; c < k; c++) {
                double tmp = br[c * n + i];
                br[c * n + i] = br[c * n + p];
                br[c * n + p] = tmp;
                tmp = bi[c * n + i];
                bi[c * n + i] = bi[c * n + p];
                bi[c * n + p] = tmp;
            }
        }
    }
    double xr[MAX_K], xi[MAX_K], yr[MAX_K], yi[MAX_K], lr[MAX_K], li[MAX_K];
    double pr[MAX_K], pi[MAX_K], buf[SCRATCH_MAX];
    for (int64_t i = 1; (phases & 1) && i < n; i++) {
        for (int c = 0; c < k; c++) {
            xr[c] = br[c * n + i];
            xi[c] = bi[c * n + i];
        }
        for (int64_t j = 0; j < i; j++) {
            for (int c = 0; c < k; c++) {
                lr[c] = re[c * ps + i * n + j];
                li[c] = im[c * ps + i * n + j];
                yr[c] = br[c * n + j];
                yi[c] = bi[c * n + j];
            }
            cmul(use3m, lr, li, yr, yi, pr, pi, k);
            orc_exp_sub(xr, pr, buf, xr, k);
            orc_exp_sub(xi, pi, buf, xi, k);
        }
        for (int c = 0; c < k; c++) {
            br[c * n + i] = xr[c];
            bi[c * n + i] = xi[c];
        }
    }
    for (int64_t i = n - 1; (phases & 2) && i >= 0; i--) {
        for (int c = 0; c < k; c++) {
            xr[c] = br[c * n + i];
            xi[c] = bi[c * n + i];
        }
        for (int64_t j = i + 1; j < n; j++) {
            for (int c = 0; c < k; c++) {
                lr[c] = re[c * ps + i * n + j];
                li[c] = im[c * ps + i * n + j];
                yr[c] = br[c * n + j];
                yi[c] = bi[c * n + j];
            }
            cmul(use3m, lr, li, yr, yi, pr, pi, k);
            orc_exp_sub(xr, pr, buf, xr, k);
            orc_exp_sub(xi, pi, buf, xi, k);
        }
        for (int c = 0; c < k; c++) {
            lr[c] = re[c * ps + i * n + i];
            li[c] = im[c * ps + i * n + i];
        }
        orc_cdiv(xr, xi, lr, li, yr, yi, k);
        for (int c = 0; c < k; c++) {
            br[c * n + i] = yr[c];
            bi[c * n + i] = yi[c];
        }
    }
}

void orc_solve_fb(int k, int use3m, int64_t n, const double *re, const double *im,
                  const int64_t *piv, double *br, double *bi) {
    orc_solve_phases(k, use3m, n, re, im, piv, br, bi, 3);
}

/* ------------------------------------------------------- scalar wrappers */
void orc_renorm1(const double *raw, int m, double *out, int k) {
    double buf[4 * SCRATCH_MAX];
    int cap = (int)(sizeof(buf) / sizeof(buf[0]));
    if (m > cap) m = cap;
    for (int i = 0; i < m; i++) buf[i] = raw[i];
    orc_renorm(buf, m, out, k);
}
int orc_nonoverlapping(const double *x, int k) { return is_nonoverlapping(x, k); }
void orc_two_sum(double a, double b, double *s, double *e) { two_sum(a, b, s, e); }
void orc_two_prod(double a, double b, double *p, double *e) { two_prod(a, b, p, e); }
void orc_exp_add1(const double *x, const double *y, double *out, int k) {
    double buf[SCRATCH_MAX];
    orc_exp_add(x, y, buf, out, k);
}
void orc_exp_sub1(const double *x, const double *y, double *out, int k) {
    double buf[SCRATCH_MAX];
    orc_exp_sub(x, y, buf, out, k);
}
void orc_exp_mul1(const double *x, const double *y, double *out, int k) {
    double buf[SCRATCH_MAX];
    orc_exp_mul(x, y, buf, out, k);
}
void orc_exp_div1(const double *x, const double *y, double *out, int k) {
    double buf[SCRATCH_MAX];
    orc_exp_div(x, y, buf, out, k);
}

int orc_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}
