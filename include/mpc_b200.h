/*
 * mpc_b200.h -- C ABI of libmpcb200.so, the B200 (sm_100a) implementation of
 * the reference's complex multi-component (DD/TD/QD) GEMM + blocked LU path.
 *
 * The reference (mpclu, /root/reference/pkg/src/mpclu) is Python over numba
 * kernels; its compiled cut points take raw planar float64 arrays and do no
 * validation (_kernels.py:1-10).  Each entry point below replaces one of
 * those cut points (cited per function) and is what a Python host binds with
 * ctypes (see INTEGRATION.md and paper_2403_16013_b200/_lib.py).
 *
 * Conventions
 *   k         component count: 2 (double-double), 3 (triple-double),
 *             4 (quad-double).
 *   method    3 (3M) or 4 (4M) complex multiplication (cmatrix.py:1-16).
 *   layout    planar limbs, row-major planes (rmatrix.py:1-7): limb c of
 *             element (i, j) of a view lives at base[c*ps + i*ld + j];
 *             complex matrices pass separate Re and Im bases that share
 *             (ld, ps).
 *   pointers  either ALL device pointers (work is enqueued on `stream`,
 *             asynchronous unless stated), or ALL host pointers (staged
 *             through device memory; the call returns when results are back
 *             in host memory).  Mixing is an error.
 *   stream    a cudaStream_t (NULL = legacy default stream).
 *   status    int functions return 0 on success and MPC_ERR (-2) on error
 *             (message via mpc_last_error()).  LU functions return -1 on
 *             success, the first exactly-singular column (>= 0) like
 *             lu_panel (_kernels.py:622-624), or MPC_ERR.
 *
 * Results are bit-identical to the reference for GEMM, mat_add, the panel,
 * the TRSM and the whole blocked factorization (pivots and packed factors);
 * the backward half of the solve is tolerance-parity.
 */
#ifndef MPC_B200_H
#define MPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPC_ABI_VERSION 1
#define MPC_ERR (-2)

int mpc_abi_version(void);
/* last error message of the calling thread ("" if none) */
const char* mpc_last_error(void);
/* number of visible CUDA devices (0 if none / no driver) */
int mpc_device_count(void);

/* mat_add_k (_kernels.py:327-342) as called by mat_add / mat_sub
 * (rmatrix.py:105-118): C = A + sign*B elementwise, sign = +1 or -1. */
int mpc_mat_add(int k, int64_t rows, int64_t cols,
                const double* a, int64_t lda, int64_t psa,
                const double* b, int64_t ldb, int64_t psb,
                double* c, int64_t ldc, int64_t psc, double sign, void* stream);

/* renorm_planes (_kernels.py:485-499): in-place elementwise renormalization. */
int mpc_renorm_planes(int k, int64_t rows, int64_t cols, double* r, int64_t ld, int64_t ps,
                      void* stream);

/* rgemm_naive_k / rgemm_blocked_k (_kernels.py:384-434) behind rgemm_naive /
 * rgemm_blocked (rgemm.py:53-73): C (m x l) = A (m x n) B (n x l), every
 * element one t-ascending chain from zero. */
int mpc_rgemm(int k, int64_t m, int64_t n, int64_t l,
              const double* a, int64_t lda, int64_t psa,
              const double* b, int64_t ldb, int64_t psb,
              double* c, int64_t ldc, int64_t psc, void* stream);

/* cgemm_3m / cgemm_4m (cmatrix.py:145-177) fused into one kernel.
 * epilogue 0: C = A B;  1: C = C - A B, rounded exactly like the LU trailing
 * update P = cgemm(L21, U12); A22 = mat_sub(A22, P) (lu.py:152-161). */
int mpc_cgemm(int k, int method, int64_t m, int64_t n, int64_t l,
              const double* a_re, const double* a_im, int64_t lda, int64_t psa,
              const double* b_re, const double* b_im, int64_t ldb, int64_t psb,
              double* c_re, double* c_im, int64_t ldc, int64_t psc, int epilogue,
              void* stream);

/* trsm_ll_unit (_kernels.py:668-705) behind trsm_unit_lower (lu.py:190-202):
 * solve L X = A in place on A; L is K x K unit lower (strictly lower part
 * read), A is K x M. */
int mpc_trsm_ll_unit(int k, int method, int64_t K, int64_t M,
                     const double* l_re, const double* l_im, int64_t ldl, int64_t psl,
                     double* a_re, double* a_im, int64_t lda, int64_t psa, void* stream);

/* lu_panel (_kernels.py:611-665) on a square n x n matrix (ld = n, ps = n*n):
 * eliminate columns [jb, jb+kw) with partial pivoting; rows are interchanged
 * across all n columns, piv[j] receives the pivot row of column j.
 * Synchronous (returns the status). */
int64_t mpc_lu_panel(int k, int method, int64_t n, double* re, double* im, int64_t* piv,
                     int64_t jb, int64_t kw, void* stream);

/* The same panel elimination restricted to the panel's own columns (the
 * interchanges are NOT applied outside [jb, jb+kw); apply them with
 * mpc_laswp).  re/im point at element (0, jb) of the matrix: element
 * (i, jb + t), 0 <= t < kw, is at re[i*ld + t]; rows [jb, n) are factored and
 * piv[jb .. jb+kw) (absolute row numbers) is written.  Used by the
 * column-distributed multi-GPU driver.  Synchronous. */
int64_t mpc_panel_factor(int k, int method, int64_t n, int64_t jb, int64_t kw,
                         double* re, double* im, int64_t ld, int64_t ps, int64_t* piv,
                         void* stream);

/* Asynchronous variant (device pointers only): enqueues the panel on
 * `stream` and writes the status (-1 or the singular column) to the device
 * word *status_out instead of returning it; returns 0 or MPC_ERR. */
int mpc_panel_factor_async(int k, int method, int64_t n, int64_t jb, int64_t kw,
                           double* re, double* im, int64_t ld, int64_t ps, int64_t* piv,
                           int64_t* status_out, void* stream);

/* Apply the interchanges piv[r0..r1) in order to columns [0, ncols) of a
 * (rows x ncols) view (the deferred part of _swap_rows, _kernels.py:597-608). */
int mpc_laswp(int k, int64_t ncols, double* re, double* im, int64_t ld, int64_t ps,
              const int64_t* piv, int64_t r0, int64_t r1, void* stream);

/* lu._factor (lu.py:129-163): blocked right-looking LU with panel width K
 * (K = n is lu_normal, lu.py:166-170).  In place on (re, im) (ld = n,
 * ps = n*n); piv (n entries) is initialised to 0..n-1 and receives the
 * pivots.  Synchronous (returns the status). */
int64_t mpc_getrf(int k, int method, int64_t n, int64_t K, double* re, double* im,
                  int64_t* piv, void* stream);

/* Multi-GPU lu._factor (mpc_getrf with ngpus and
 * lookahead): 1-D block-column-cyclic over `ngpus` devices of this process
 * (device ordinals current, current+1, ...), panel + pivots + status pulled
 * by every rank from the panel owner over NVLink peer copies, depth-1
 * lookahead when lookahead != 0.  real_kernel 0 = the EFT GEMM (mpc_getrf),
 * 1 = the Ozaki tensor-core GEMM (mpc_getrf_ozaki; d, split_bits as there).
 * Pointers: host (pageable or pinned) or device memory; piv receives the
 * pivots.  Bit-identical to mpc_getrf / mpc_getrf_ozaki.  ngpus = 1 is
 * mpc_getrf (or mpc_getrf_ozaki); ngpus above the device count is an error
 * unless MPC_MGPU_OVERSUBSCRIBE=1 (ranks share devices; test mode).
 * Synchronous (returns the status like mpc_getrf). */
int64_t mpc_getrf_ngpu(int k, int method, int64_t n, int64_t K, double* re, double* im,
                       int64_t* piv, int ngpus, int lookahead, int real_kernel, int d,
                       int split_bits, void* stream);

/* solve_fb (_kernels.py:708-775) behind solve (lu.py:205-218): x from
 * L U x = P b on packed factors; b (k x n planes, Re and Im) is overwritten.
 * The caller checks the U diagonal for exact zeros (lu.py:213-215). */
int mpc_getrs(int k, int method, int64_t n, const double* re, const double* im,
              const int64_t* piv, double* b_re, double* b_im, void* stream);

/* The halves of solve_fb (_kernels.py:708-775) separately (LAPACK getrs
 * style): phases 1 = the interchanges (_kernels.py:711-721) + the unit-lower
 * forward substitution (734-752; bit-identical to the reference), 2 = the
 * backward substitution with the cdiv by U_ii (753-775; b holds the forward
 * result), 3 = both (= mpc_getrs). */
int mpc_getrs_phases(int k, int method, int64_t n, const double* re, const double* im,
                     const int64_t* piv, double* b_re, double* b_im, int phases,
                     void* stream);

/* max_rel_err (lu.py:263-282): max_i |xhat_i - x_i| / |x_i| over complex
 * moduli in k-component expansion arithmetic, bit for bit the reference's
 * value (csub, exp_mul / exp_add / exp_div per entry, first strict maximum,
 * _exp_sqrt's three Newton steps, lu.py:253-260).  Vectors are planar (k, n);
 * out receives the k components; *zero_index is the first index whose true
 * component is zero (the reference raises ValueError there) or -1. */
int mpc_max_rel_err(int k, int64_t n, const double* xhat_re, const double* xhat_im,
                    const double* x_re, const double* x_im, double* out, int64_t* zero_index,
                    void* stream);

/* ---- Ozaki scheme (ozaki.py:79-159): the alternative real kernel ---- */
/* ozaki_split (ozaki.py:79-108) of a (rows x cols) planar operand into d
 * binary64 parts (contiguous (d, rows, cols)) with grid units `scales`
 * ((d, rows) for side 0 = "left", (d, cols) for side 1 = "right"). */
int mpc_ozaki_split(int k, int64_t rows, int64_t cols, const double* a, int64_t lda,
                    int64_t psa, int d, int width, int side, double* parts, double* scales,
                    void* stream);
/* acc_plane (_kernels.py:502-517): C += P by ordered two-sum insertion. */
int mpc_acc_plane(int k, int64_t rows, int64_t cols, double* c, int64_t ldc, int64_t psc,
                  const double* p, int64_t ldp, void* stream);
/* The f64_gemm seam (ozaki.py:127-142): Z = X Y in binary64 (cuBLAS DGEMM;
 * exact, hence bit-identical to np.matmul, for Ozaki parts). */
int mpc_f64_gemm(int64_t m, int64_t n, int64_t l, const double* x, int64_t ldx,
                 const double* y, int64_t ldy, double* z, int64_t ldz, void* stream);
/* rgemm_ozaki (ozaki.py:124-159); split_bits 0 = the default width. */
int mpc_rgemm_ozaki(int k, int64_t m, int64_t n, int64_t l, const double* a, int64_t lda,
                    int64_t psa, const double* b, int64_t ldb, int64_t psb, double* c,
                    int64_t ldc, int64_t psc, int d, int split_bits, void* stream);
/* cgemm_3m / cgemm_4m with real_kernel="ozaki" (cmatrix.py:128-169);
 * epilogue as mpc_cgemm. */
int mpc_cgemm_ozaki(int k, int method, int64_t m, int64_t n, int64_t l,
                    const double* a_re, const double* a_im, int64_t lda, int64_t psa,
                    const double* b_re, const double* b_im, int64_t ldb, int64_t psb,
                    double* c_re, double* c_im, int64_t ldc, int64_t psc, int d, int split_bits,
                    int epilogue, void* stream);
/* lu_blocked with kc.real_kernel == "ozaki" (lu.py:129-163); piv must hold
 * 0..n-1 on entry (lu.py:134).  Synchronous. */
int64_t mpc_getrf_ozaki(int k, int method, int64_t n, int64_t K, double* re, double* im,
                        int64_t* piv, int d, int split_bits, void* stream);

/* Page-lock (cudaHostRegister) / release an existing host range, so the LU
 * entry points overlap its copies with the factorization (the drop-in
 * lu_blocked registers its output copy of A for the call). */
int mpc_host_register(void* p, int64_t bytes);
int mpc_host_unregister(void* p);

/* ---- measurement hooks (bench.py) ---- */
/* Per-launch CUDA-event timing of the kernel classes whose bit is set in
 * `mask` (bit c = class c below; 0 disables).  Clears previous records. */
void mpc_prof_enable(int mask);
/* Sum per kernel class (0 GEMM, 1 S-update, 2 panel, 3 TRSM diagonal,
 * 4 LASWP, 5 other, 6 solve) of event-timed ms, algorithmic FP64 ops (op model v1)
 * and launch counts since the last mpc_prof_enable(1).  Returns the number of
 * classes or MPC_ERR. */
int mpc_prof_summary(double* ms, double* ops, long long* count, int nclass);
/* Kernels launched by this library since load (always counted). */
long long mpc_launch_count(void);
/* Measured FP64 (DADD) issue rate of the current device, lane-ops/s. */
double mpc_fp64_peak(int iters, void* stream);

/* Measured INT8 tensor-core rate of the current device (tcgen05.mma
 * kind::i8 M=128 N=256 K=32 back to back on every SM; ops/s, 2 per MAC):
 * the roofline denominator of the Ozaki tensor-core kernel. */
double mpc_int8_peak(int iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPC_B200_H */
