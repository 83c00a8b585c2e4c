// ozaki.cu -- the Ozaki-scheme real kernel on the B200.
//
// Reference: ozaki.py:79-159 (ozaki_split, _pair_schedule, rgemm_ozaki),
// _kernels.py:485-517 (renorm_planes, acc_plane), cmatrix.py:128-169 (the 3M /
// 4M composition over a real kernel), lu.py:129-163 (the LU trailing update).
//
// Bit-exactness: the split (row / column max, frexp/ldexp, (r + S) - S,
// renorm) and the ordered two-sum insertion (acc_plane) are elementwise
// restatements with round-to-nearest intrinsics; every scheduled part
// product is an EXACT binary64 GEMM (integer multiples of a common grid,
// |sum| <= 2^53 units by the width bound, ozaki.py:33-38), so any summation
// order gives the same bits -- it runs on cuBLAS DGEMM (the "f64_gemm seam",
// ozaki.py:124-142; B200 FP64 tensor cores).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "abi_util.h"
#include "ozaki_tc.h"
#include "prof.h"

using namespace mpcabi;

namespace mpc {
namespace {

// mu[i] = max_j |R0[i, j]| (left split, per row)
__global__ void absmax_rows_kernel(const double* r0, int64_t rows, int64_t cols, int64_t ld,
                                   double* mu) {
  __shared__ double sm[256];
  int64_t i = blockIdx.x;
  double m = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) m = fmax(m, fabs(r0[i * ld + j]));
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) mu[i] = sm[0];
}

// mu[j] = max_i |R0[i, j]| (right split, per column)
__global__ void absmax_cols_kernel(const double* r0, int64_t rows, int64_t cols, int64_t ld,
                                   double* mu) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double m = 0.0;
  for (int64_t i = 0; i < rows; i++) m = fmax(m, fabs(r0[i * ld + j]));
  mu[j] = m;
}

// one split step (ozaki.py:97-107): w = 2^ex with frexp(mu) = (f, ex);
// sigma = w * 2^(53 - width); part = (r0 + S) - S; r0 -= part; renorm the
// element's limbs (renorm_planes); scale = ldexp(w, -width).
template <int K>
__global__ void split_step_kernel(View R, int64_t rows, int64_t cols, int side, const double* mu,
                                  int width, double* part, double* scale) {
  int64_t total = rows * cols;
  const double shift = ldexp(1.0, 53 - width);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    int64_t g = side == 0 ? i : j;
    int ex = 0;
    frexp(mu[g], &ex);
    double w = ldexp(1.0, ex);
    double S = __dmul_rn(w, shift);
    double* p0 = R.re + i * R.ld + j;
    double r0 = *p0;
    double pt = __dsub_rn(__dadd_rn(r0, S), S);
    part[i * cols + j] = pt;
    double buf[K];
    buf[0] = __dsub_rn(r0, pt);
#pragma unroll
    for (int c = 1; c < K; c++) buf[c] = p0[c * R.ps];
    Exp<K> o = renorm<K, K>(buf, K);
    stexp_<K>(p0, R.ps, o);
    if ((side == 0 && j == 0) || (side == 1 && i == 0)) scale[g] = ldexp(w, -width);
  }
}

// acc_plane (_kernels.py:502-517): C += P, error-free insertion from the
// least significant component up, truncated to k
template <int K>
__global__ void acc_plane_kernel(View C, int64_t rows, int64_t cols, const double* P,
                                 int64_t ldp) {
  int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    double* c0 = C.re + i * C.ld + j;
    double q = P[i * ldp + j];
    double h[K + 1];
#pragma unroll
    for (int c = K - 1; c >= 0; c--) {
      double s, err;
      two_sum(q, c0[c * C.ps], s, err);
      q = s;
      h[c + 1] = err;
    }
    h[0] = q;
#pragma unroll
    for (int c = 0; c < K; c++) c0[c * C.ps] = h[c];
  }
}

unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

template <int K>
void split_step(View R, int64_t rows, int64_t cols, int side, double* mu, int width, double* part,
                double* scale, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  int tok = prof_begin(PC_OTHER, 0.0, st);
  if (side == 0)
    absmax_rows_kernel<<<(unsigned)rows, 256, 0, st>>>(R.re, rows, cols, R.ld, mu);
  else
    absmax_cols_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(R.re, rows, cols, R.ld, mu);
  split_step_kernel<K><<<grid_for(rows * cols), 256, 0, st>>>(R, rows, cols, side, mu, width, part,
                                                               scale);
  prof_end(tok, st);
  check_launch("ozaki split");
}

template <int K>
void acc_plane(View C, int64_t rows, int64_t cols, const double* P, int64_t ldp, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  int tok = prof_begin(PC_OTHER, 0.0, st);
  acc_plane_kernel<K><<<grid_for(rows * cols), 256, 0, st>>>(C, rows, cols, P, ldp);
  prof_end(tok, st);
  check_launch("acc_plane");
}

void split_dispatch(int k, View R, int64_t rows, int64_t cols, int side, double* mu, int width,
                    double* part, double* scale, cudaStream_t st) {
  switch (k) {
    case 2: split_step<2>(R, rows, cols, side, mu, width, part, scale, st); break;
    case 3: split_step<3>(R, rows, cols, side, mu, width, part, scale, st); break;
    default: split_step<4>(R, rows, cols, side, mu, width, part, scale, st); break;
  }
}

void acc_dispatch(int k, View C, int64_t rows, int64_t cols, const double* P, int64_t ldp,
                  cudaStream_t st) {
  switch (k) {
    case 2: acc_plane<2>(C, rows, cols, P, ldp, st); break;
    case 3: acc_plane<3>(C, rows, cols, P, ldp, st); break;
    default: acc_plane<4>(C, rows, cols, P, ldp, st); break;
  }
}

// one cuBLAS handle per device
cublasHandle_t handle_for_current_device() {
  static std::mutex mu;
  static std::vector<cublasHandle_t> hs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if ((int)hs.size() <= dev) hs.resize(dev + 1, nullptr);
  if (!hs[dev]) {
    if (cublasCreate(&hs[dev]) != CUBLAS_STATUS_SUCCESS) throw CudaError{"cublasCreate failed"};
  }
  return hs[dev];
}

// Z (m x l) = X (m x n) Y (n x l), row-major, exact inputs -> exact result
void f64_gemm(int64_t m, int64_t n, int64_t l, const double* x, int64_t ldx, const double* y,
              int64_t ldy, double* z, int64_t ldz, cudaStream_t st) {
  if (m <= 0 || l <= 0) return;
  if (n == 0) {
    ck(cudaMemset2DAsync(z, ldz * 8, 0, l * 8, m, st), "memset");
    return;
  }
  cublasHandle_t h = handle_for_current_device();
  cublasSetStream(h, st);
  const double one = 1.0, zero = 0.0;
  int tok = prof_begin(PC_GEMM, 2.0 * (double)m * (double)n * (double)l, st);
  // row-major Z = X Y  <=>  column-major Z^T = Y^T X^T
  cublasStatus_t r = cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)l, (int)m, (int)n, &one, y,
                                 (int)ldy, x, (int)ldx, &zero, z, (int)ldz);
  prof_end(tok, st);
  if (r != CUBLAS_STATUS_SUCCESS) throw CudaError{"cublasDgemm failed"};
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    retain_pool();
    if (bytes) ck(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  double* d() { return (double*)p; }
};

void copy_view(int k, View dst, View src, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  for (int c = 0; c < k; c++)
    ck(cudaMemcpy2DAsync(dst.re + c * dst.ps, dst.ld * 8, src.re + c * src.ps, src.ld * 8, cols * 8,
                         rows, cudaMemcpyDeviceToDevice, st),
       "copy");
}

}  // namespace

// _pair_schedule, ozaki.py:111-121
std::vector<std::pair<int, int>> pair_schedule(int d, int width, int k) {
  std::vector<std::pair<int, int>> pairs;
  int cutoff = 53 * k + 53;
  for (int s = 0; s < d; s++) {
    if (s * std::max(width - 1, 1) >= cutoff) break;
    for (int p = 0; p <= s; p++) pairs.emplace_back(p, s - p);
  }
  return pairs;
}

// split_exactness_bound, ozaki.py:33-38
int split_exactness_bound(int64_t inner) {
  if (inner <= 1) return 53 / 2;
  int e = 0;
  while (((int64_t)1 << e) < inner) e++;  // ceil(log2(inner))
  return (53 - e) / 2;
}

// _resolve_width, ozaki.py:41-51; returns -1 if over budget
int resolve_width(int k, int64_t inner, int split_bits) {
  int bound = split_exactness_bound(inner);
  if (bound < 1) return -1;
  if (split_bits <= 0) {
    int def = (k == 2) ? 19 : (k == 3) ? 21 : (k == 4) ? 18 : bound;
    return std::min(def, bound);
  }
  if (split_bits > bound) return -1;
  return split_bits;
}

// rgemm_ozaki (ozaki.py:124-159) on device views; C (m x l) receives the result
// (with cb: returns true iff the tensor-core path also applied the fused
// complex composition, see OzCombine; C is then untouched)
bool rgemm_ozaki_dev(int k, int64_t m, int64_t n, int64_t l, View A, View B, View C, int d,
                     int width, cudaStream_t st, const OzCombine* cb = nullptr) {
  const OpsTable* T = table_for(k);
  if (m <= 0 || l <= 0) return false;
  const auto pairs = pair_schedule(d, width, k);
  // fused split + exact part products on the INT8 tensor cores + acc_plane + renorm
  if (ozaki_tc_enabled() && ozaki_tc_rgemm(k, m, n, l, A, B, C, d, pairs, width, st, cb))
    return cb != nullptr;
  DevBuf ra(sizeof(double) * k * m * n, st), rb(sizeof(double) * k * n * l, st);
  DevBuf pa(sizeof(double) * d * m * n, st), pb(sizeof(double) * d * n * l, st);
  DevBuf mua(sizeof(double) * (m + 1), st), mub(sizeof(double) * (l + 1), st);
  DevBuf sca(sizeof(double) * d * (m + 1), st), scb(sizeof(double) * d * (l + 1), st);
  View RA{ra.d(), nullptr, n, m * n}, RB{rb.d(), nullptr, l, n * l};
  copy_view(k, RA, A, m, n, st);
  copy_view(k, RB, B, n, l, st);
  for (int s = 0; s < d; s++) {
    split_dispatch(k, RA, m, n, 0, mua.d(), width, pa.d() + (int64_t)s * m * n,
                   sca.d() + (int64_t)s * m, st);
    split_dispatch(k, RB, n, l, 1, mub.d(), width, pb.d() + (int64_t)s * n * l,
                   scb.d() + (int64_t)s * l, st);
  }
  // binary64 seam: zero C (acc_plane accumulates into a fresh RealMatrix.zeros)
  for (int c = 0; c < k; c++)
    ck(cudaMemset2DAsync(C.re + c * C.ps, C.ld * 8, 0, l * 8, m, st), "memset");
  DevBuf P(sizeof(double) * m * l, st);
  for (auto pq : pairs) {
    f64_gemm(m, n, l, pa.d() + (int64_t)pq.first * m * n, n, pb.d() + (int64_t)pq.second * n * l,
             l, P.d(), l, st);
    acc_dispatch(k, C, m, l, P.d(), l, st);
  }
  T->renorm_planes(m, l, C, st);
  return false;
}

// cgemm_3m / cgemm_4m over the Ozaki real kernel (cmatrix.py:145-169), with
// the LU epilogue C = C - P (lu.py:158-161) when epi == 1
void cgemm_ozaki_dev(int k, bool use3m, int64_t m, int64_t n, int64_t l, View A, View B, View C,
                     int epi, int d, int width, cudaStream_t st) {
  const OpsTable* T = table_for(k);
  auto mk = [&](int64_t r, int64_t c, DevBuf& b) { return View{b.d(), nullptr, c, r * c}; };
  View Ar{A.re, nullptr, A.ld, A.ps}, Ai{A.im, nullptr, A.ld, A.ps};
  View Br{B.re, nullptr, B.ld, B.ps}, Bi{B.im, nullptr, B.ld, B.ps};
  size_t ml = sizeof(double) * k * m * l;
  DevBuf t1(ml, st), t2(ml, st), t3(use3m ? 0 : ml, st);
  View T1 = mk(m, l, t1), T2 = mk(m, l, t2), T3 = mk(m, l, t3);
  View Cr{C.re, nullptr, C.ld, C.ps}, Ci{C.im, nullptr, C.ld, C.ps};
  // the last real product carries the composition + LU subtraction in its
  // epilogue on the tensor-core path (OzCombine); otherwise the reference's
  // mat_add sequence runs as separate passes
  OzCombine cb{use3m ? 3 : 4, epi, T1, T2, T3, C};
  auto finish = [&](View Tl) {  // Tl: the last product (T3 for 3M, ri for 4M)
    DevBuf pre(ml, st), pim(ml, st);
    View PR = mk(m, l, pre), PI = mk(m, l, pim);
    T->mat_add(m, l, T1, T2, PR, -1.0, st);
    if (use3m) {
      T->mat_add(m, l, Tl, T1, Tl, -1.0, st);
      T->mat_add(m, l, Tl, T2, PI, -1.0, st);
    } else {
      T->mat_add(m, l, T3, Tl, PI, 1.0, st);
    }
    if (epi == 1) {
      T->mat_add(m, l, Cr, PR, Cr, -1.0, st);
      T->mat_add(m, l, Ci, PI, Ci, -1.0, st);
    } else {
      copy_view(k, Cr, PR, m, l, st);
      copy_view(k, Ci, PI, m, l, st);
    }
  };
  if (use3m) {
    DevBuf sa(sizeof(double) * k * m * n, st), sb(sizeof(double) * k * n * l, st);
    View SA = mk(m, n, sa), SB = mk(n, l, sb);
    rgemm_ozaki_dev(k, m, n, l, Ar, Br, T1, d, width, st);
    rgemm_ozaki_dev(k, m, n, l, Ai, Bi, T2, d, width, st);
    T->mat_add(m, n, Ar, Ai, SA, 1.0, st);
    T->mat_add(n, l, Br, Bi, SB, 1.0, st);
    DevBuf tl(ml, st);
    View TL = mk(m, l, tl);
    if (!rgemm_ozaki_dev(k, m, n, l, SA, SB, TL, d, width, st, &cb)) finish(TL);
  } else {
    rgemm_ozaki_dev(k, m, n, l, Ar, Br, T1, d, width, st);  // rr
    rgemm_ozaki_dev(k, m, n, l, Ai, Bi, T2, d, width, st);  // ii
    rgemm_ozaki_dev(k, m, n, l, Ai, Br, T3, d, width, st);  // ir
    DevBuf tl(ml, st);
    View TL = mk(m, l, tl);
    if (!rgemm_ozaki_dev(k, m, n, l, Ar, Bi, TL, d, width, st, &cb)) finish(TL);  // ri
  }
}

}  // namespace mpc

extern "C" {

int mpc_ozaki_split(int k, int64_t rows, int64_t cols, const double* a, int64_t lda, int64_t psa,
                    int d, int width, int side, double* parts, double* scales, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (d < 1) return fail("d must be >= 1");
  if (side != 0 && side != 1) return fail("side must be 0 (left) or 1 (right)");
  if (width < 1 || width > 26) return fail("width outside [1, 26]");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({a, parts, scales})) return MPC_ERR;
  int64_t ng = side == 0 ? rows : cols;
  double* da = sg.map(const_cast<double*>(a), extent(k, rows, cols, lda, psa), true, false);
  double* dp = sg.map(parts, (int64_t)d * rows * cols, false, true);
  double* ds = sg.map(scales, (int64_t)d * ng, false, true);
  if (rows > 0 && cols > 0) {
    mpc::DevBuf r(sizeof(double) * k * rows * cols, st), mu(sizeof(double) * (ng + 1), st);
    mpc::View R{r.d(), nullptr, cols, rows * cols};
    mpc::copy_view(k, R, mpc::View{da, nullptr, lda, psa}, rows, cols, st);
    for (int s = 0; s < d; s++)
      mpc::split_dispatch(k, R, rows, cols, side, mu.d(), width, dp + (int64_t)s * rows * cols,
                          ds + (int64_t)s * ng, st);
  }
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_acc_plane(int k, int64_t rows, int64_t cols, double* c, int64_t ldc, int64_t psc,
                  const double* p, int64_t ldp, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({c, p})) return MPC_ERR;
  double* dc = sg.map(c, extent(k, rows, cols, ldc, psc), true, true);
  double* dp = sg.map(const_cast<double*>(p), extent(1, rows, cols, ldp, 0), true, false);
  mpc::acc_dispatch(k, mpc::View{dc, nullptr, ldc, psc}, rows, cols, dp, ldp, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_f64_gemm(int64_t m, int64_t n, int64_t l, const double* x, int64_t ldx, const double* y,
                 int64_t ldy, double* z, int64_t ldz, void* stream) {
  if (m < 0 || n < 0 || l < 0) return fail("negative dimension");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({x, y, z})) return MPC_ERR;
  double* dx = sg.map(const_cast<double*>(x), extent(1, m, n, ldx, 0), true, false);
  double* dy = sg.map(const_cast<double*>(y), extent(1, n, l, ldy, 0), true, false);
  double* dz = sg.map(z, extent(1, m, l, ldz, 0), false, true);
  mpc::f64_gemm(m, n, l, dx, ldx, dy, ldy, dz, ldz, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_rgemm_ozaki(int k, int64_t m, int64_t n, int64_t l, const double* a, int64_t lda,
                    int64_t psa, const double* b, int64_t ldb, int64_t psb, double* c, int64_t ldc,
                    int64_t psc, int d, int split_bits, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (d < 1) return fail("d must be >= 1");
  if (m < 0 || n < 0 || l < 0) return fail("negative dimension");
  int width = mpc::resolve_width(k, n, split_bits);
  if (width < 0) return fail("dimension exceeds split exactness budget");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({a, b, c})) return MPC_ERR;
  double* da = sg.map(const_cast<double*>(a), extent(k, m, n, lda, psa), true, false);
  double* db = sg.map(const_cast<double*>(b), extent(k, n, l, ldb, psb), true, false);
  double* dc = sg.map(c, extent(k, m, l, ldc, psc), false, true);
  mpc::rgemm_ozaki_dev(k, m, n, l, mpc::View{da, nullptr, lda, psa},
                       mpc::View{db, nullptr, ldb, psb}, mpc::View{dc, nullptr, ldc, psc}, d,
                       width, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_cgemm_ozaki(int k, int method, int64_t m, int64_t n, int64_t l, const double* a_re,
                    const double* a_im, int64_t lda, int64_t psa, const double* b_re,
                    const double* b_im, int64_t ldb, int64_t psb, double* c_re, double* c_im,
                    int64_t ldc, int64_t psc, int d, int split_bits, int epilogue, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (d < 1) return fail("d must be >= 1");
  if (m < 0 || n < 0 || l < 0) return fail("negative dimension");
  int width = mpc::resolve_width(k, n, split_bits);
  if (width < 0) return fail("dimension exceeds split exactness budget");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({a_re, a_im, b_re, b_im, c_re, c_im})) return MPC_ERR;
  int64_t ea = extent(k, m, n, lda, psa), eb = extent(k, n, l, ldb, psb),
          ec = extent(k, m, l, ldc, psc);
  double* dar = sg.map(const_cast<double*>(a_re), ea, true, false);
  double* dai = sg.map(const_cast<double*>(a_im), ea, true, false);
  double* dbr = sg.map(const_cast<double*>(b_re), eb, true, false);
  double* dbi = sg.map(const_cast<double*>(b_im), eb, true, false);
  double* dcr = sg.map(c_re, ec, epilogue == 1, true);
  double* dci = sg.map(c_im, ec, epilogue == 1, true);
  if (m > 0 && l > 0)
    mpc::cgemm_ozaki_dev(k, method == 3, m, n, l, mpc::View{dar, dai, lda, psa},
                         mpc::View{dbr, dbi, ldb, psb}, mpc::View{dcr, dci, ldc, psc}, epilogue, d,
                         width, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

// lu._factor with kc.real_kernel == "ozaki" (lu.py:129-163): the same panel
// and TRSM as mpc_getrf, the trailing update through the Ozaki cgemm and
// mat_sub (sequential schedule).
int64_t mpc_getrf_ozaki(int k, int method, int64_t n, int64_t K, double* re, double* im,
                        int64_t* piv, int d, int split_bits, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0) return fail("negative dimension");
  if (n > 0 && (K < 1 || K > n)) return fail("panel width K outside [1, n]");
  if (d < 1) return fail("d must be >= 1");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv})) return MPC_ERR;
  int64_t e = extent(k, n, n, n, n * n);
  // pinned host factors: copies overlapped with the LU as in mpc_getrf
  const bool overlap = HostOverlap::usable(sg, n, re, im);
  double* dr = sg.map(re, e, !overlap, !overlap);
  double* di = sg.map(im, e, !overlap, !overlap);
  int64_t* dp = sg.map(piv, n, true, true);
  int64_t status = -1;
  HostOverlap ho;
  if (overlap) ho.start(st, dr, di, re, im, k, n, K);
  auto need = [&](int64_t c1) {
    if (overlap) HostOverlap::need(&ho, std::min(c1, n), st);
  };
  auto rows_done = [&](int64_t r0, int64_t r1) {
    if (overlap) HostOverlap::rows_done(&ho, r0, r1, st);
  };
  if (n > 0) {
    const mpc::OpsTable* T = table_for(k);
    bool use3m = method == 3;
    mpc::View A{dr, di, n, n * n};
    WsHolder w(k, n, st);
    // the budget applies to the trailing update only (none when K >= n)
    if (n > K && mpc::resolve_width(k, K, split_bits) < 0)
      return fail("dimension exceeds split exactness budget");
    // Same schedule as mpc_getrf (depth-1 lookahead): the narrow update of
    // block b+1, its panel factorization on a high-priority side stream, the
    // rest of block b's update overlapping it.  Column ranges of the Ozaki
    // update are independent (right-operand grids are per column, left-
    // operand grids per row of L21), so the split schedule is bit-identical
    // to lu.py's sequential one.  A singular panel sets the device status;
    // later panels early-out and the status is read once at the end (the
    // reference raises at the first singular column, lu.py:139-141).
    auto update_cols = [&](int64_t jb, int64_t kw, int64_t c0, int64_t c1, cudaStream_t s) {
      if (c1 <= c0) return;
      int64_t end = jb + kw;
      T->laswp(A, c0, c1 - c0, dp, jb, end, s, w.ws.status);
      T->trsm(use3m, kw, c1 - c0, A.sub(jb, jb), A.sub(jb, c0), s, w.ws.status);
      mpc::cgemm_ozaki_dev(k, use3m, n - end, kw, c1 - c0, A.sub(end, jb), A.sub(jb, c0),
                           A.sub(end, c0), 1, d, mpc::resolve_width(k, kw, split_bits), s);
    };
    mpc::SideStream ss;
    ss.set_main(st);
    cudaStream_t sp = ss.sp;
    cudaEvent_t ev_narrow = ss.ev_narrow, ev_panel = ss.ev_panel;
    // MPC_TRACE=1: per-step timeline on stderr (as mpc_getrf)
    static const bool trace = getenv("MPC_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      tev.push_back(e);
    };
    mark(st);
    need(std::min(K, n));
    T->panel_rec(use3m, A, n, 0, std::min(K, n), dp, w.ws, st);
    mark(st);
    for (int64_t jb = 0; jb < n; jb += K) {
      int64_t kw = std::min(K, n - jb);
      int64_t end = jb + kw;
      T->laswp(A, 0, jb, dp, jb, end, st, w.ws.status);  // left of the panel
      if (end == n) {
        rows_done(jb, end);
        break;
      }
      int64_t kw2 = std::min(K, n - end);
      if (jb == 0) need(end + kw2);
      update_cols(jb, kw, end, end + kw2, st);
      cudaEventRecord(ev_narrow, st);
      mark(st);
      cudaStreamWaitEvent(sp, ev_narrow, 0);
      T->panel_rec(use3m, A, n, end, kw2, dp, w.ws, sp);
      cudaEventRecord(ev_panel, sp);
      mark(sp);
      if (jb == 0 && overlap) {
        // step 0 in column chunks behind their host-to-device blocks (the
        // Ozaki update is per column range, so no bits change)
        for (int64_t c0 = end + kw2; c0 < n; c0 += ho.chunk) {
          need(c0 + ho.chunk);
          update_cols(jb, kw, c0, std::min(n, c0 + ho.chunk), st);
        }
      } else {
        update_cols(jb, kw, end + kw2, n, st);
      }
      rows_done(jb, end);
      mark(st);
      cudaStreamWaitEvent(st, ev_panel, 0);
      mark(st);
    }
    if (trace) {
      cudaStreamSynchronize(st);
      float t;
      cudaEventElapsedTime(&t, tev[0], tev[1]);
      fprintf(stderr, "MPC_TRACE ozaki n=%lld K=%lld first-panel %.3f ms\n", (long long)n,
              (long long)K, t);
      for (size_t i = 1; i + 4 < tev.size(); i += 4) {
        float tn, tp, tr, tj;
        cudaEventElapsedTime(&tn, tev[i], tev[i + 1]);
        cudaEventElapsedTime(&tp, tev[i + 1], tev[i + 2]);
        cudaEventElapsedTime(&tr, tev[i + 1], tev[i + 3]);
        cudaEventElapsedTime(&tj, tev[i], tev[i + 4]);
        fprintf(stderr,
                "MPC_TRACE step %zu: narrow %.3f  panel(side) %.3f  rest %.3f  step %.3f ms\n",
                (i - 1) / 4, tn, tp, tr, tj);
      }
      for (auto e : tev) cudaEventDestroy(e);
    }
    status = w.read_status();
  }
  if (overlap) ho.join(st);
  sg.finish();
  return status;
  MPC_CATCH
}

}  // extern "C"
