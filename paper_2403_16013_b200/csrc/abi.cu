// abi.cu -- extern "C" entry points of libmpcb200.so (declared in
// include/mpc_b200.h): argument checks, host-pointer staging, dispatch on the
// component count to the per-K operation tables.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "abi_util.h"
#include "prof.h"

// ------------------------------------------------------------ profiling
namespace mpc {
namespace {
struct ProfRec {
  int cls;
  double ops;
  cudaEvent_t a, b;
};
struct ProfState {
  std::mutex mu;
  bool on = false;
  int mask = 0;
  std::atomic<long long> launches{0};
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
ProfState& P() {
  static ProfState s;
  return s;
}
}  // namespace

int prof_begin(int cls, double ops, cudaStream_t st) {
  ProfState& p = P();
  p.launches++;
  if (!p.on || !((p.mask >> cls) & 1)) return -1;
  std::lock_guard<std::mutex> g(p.mu);
  ProfRec r{cls, ops, p.get(), p.get()};
  cudaEventRecord(r.a, st);
  p.recs.push_back(r);
  return (int)p.recs.size() - 1;
}

void prof_end(int tok, cudaStream_t st) {
  if (tok < 0) return;
  ProfState& p = P();
  std::lock_guard<std::mutex> g(p.mu);
  cudaEventRecord(p.recs[tok].b, st);
}
}  // namespace mpc

namespace mpcabi {
thread_local std::string g_err;
}  // namespace mpcabi

using namespace mpcabi;

namespace {

__global__ void fp64_peak_kernel(double* out, int iters, double c) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = __dadd_rn(a[i], c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; i++) s = __dadd_rn(s, a[i]);
  if (s == 1234.5) out[0] = s;
}

__global__ void iota_kernel(int64_t* p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

}  // namespace

extern "C" {

int mpc_abi_version(void) { return MPC_ABI_VERSION; }

const char* mpc_last_error(void) { return g_err.c_str(); }

int mpc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void mpc_prof_enable(int on) {
  mpc::ProfState& p = mpc::P();
  std::lock_guard<std::mutex> g(p.mu);
  for (auto& r : p.recs) {
    p.pool.push_back(r.a);
    p.pool.push_back(r.b);
  }
  p.recs.clear();
  p.on = on != 0;
  p.mask = on;
}

long long mpc_launch_count(void) { return mpc::P().launches.load(); }

int mpc_prof_summary(double* ms, double* ops, long long* count, int nclass) {
  mpc::ProfState& p = mpc::P();
  std::lock_guard<std::mutex> g(p.mu);
  for (int c = 0; c < nclass; c++) {
    ms[c] = 0.0;
    ops[c] = 0.0;
    count[c] = 0;
  }
  for (auto& r : p.recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return fail("event sync failed");
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return fail("event time failed");
    if (r.cls >= 0 && r.cls < nclass) {
      ms[r.cls] += t;
      ops[r.cls] += r.ops;
      count[r.cls] += 1;
    }
  }
  return mpc::PC_N;
}

double mpc_fp64_peak(int iters, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* out = nullptr;
  if (cudaMallocAsync((void**)&out, 8, st) != cudaSuccess) return -1.0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned blocks = (unsigned)sms * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fp64_peak_kernel<<<blocks, 256, 0, st>>>(out, iters / 10 + 1, 1e-9);  // warm-up
  cudaEventRecord(a, st);
  fp64_peak_kernel<<<blocks, 256, 0, st>>>(out, iters, 1e-9);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(out, st);
  if (cudaGetLastError() != cudaSuccess || t <= 0.f) return -1.0;
  double ops = (double)blocks * 256.0 * 16.0 * (double)iters;
  return ops / (t * 1e-3);  // FP64 instructions (lane-ops) per second
}

int mpc_mat_add(int k, int64_t rows, int64_t cols, const double* a, int64_t lda, int64_t psa,
                const double* b, int64_t ldb, int64_t psb, double* c, int64_t ldc, int64_t psc,
                double sign, void* stream) {
  if (bad_k_gemm(k)) return fail("k must be 2, 3, 4 (or 5, 6, 8: verification kernels)");
  if (rows < 0 || cols < 0) return fail("negative dimension");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({a, b, c})) return MPC_ERR;
  double* da = sg.map(const_cast<double*>(a), extent(k, rows, cols, lda, psa), true, false);
  double* db = sg.map(const_cast<double*>(b), extent(k, rows, cols, ldb, psb), true, false);
  double* dc = sg.map(c, extent(k, rows, cols, ldc, psc), true, true);
  table_for(k)->mat_add(rows, cols, mpc::View{da, nullptr, lda, psa},
                        mpc::View{db, nullptr, ldb, psb}, mpc::View{dc, nullptr, ldc, psc},
                        sign, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_renorm_planes(int k, int64_t rows, int64_t cols, double* r, int64_t ld, int64_t ps,
                      void* stream) {
  if (bad_k_gemm(k)) return fail("k must be 2, 3, 4 (or 5, 6, 8: verification kernels)");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({r})) return MPC_ERR;
  double* dr = sg.map(r, extent(k, rows, cols, ld, ps), true, true);
  table_for(k)->renorm_planes(rows, cols, mpc::View{dr, nullptr, ld, ps}, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_rgemm(int k, int64_t m, int64_t n, int64_t l, const double* a, int64_t lda, int64_t psa,
              const double* b, int64_t ldb, int64_t psb, double* c, int64_t ldc, int64_t psc,
              void* stream) {
  if (bad_k_gemm(k)) return fail("k must be 2, 3, 4 (or 5, 6, 8: verification kernels)");
  if (m < 0 || n < 0 || l < 0) return fail("negative dimension");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({a, b, c})) return MPC_ERR;
  double* da = sg.map(const_cast<double*>(a), extent(k, m, n, lda, psa), true, false);
  double* db = sg.map(const_cast<double*>(b), extent(k, n, l, ldb, psb), true, false);
  double* dc = sg.map(c, extent(k, m, l, ldc, psc), true, true);
  table_for(k)->rgemm(m, n, l, mpc::View{da, nullptr, lda, psa}, mpc::View{db, nullptr, ldb, psb},
                      mpc::View{dc, nullptr, ldc, psc}, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_cgemm(int k, int method, int64_t m, int64_t n, int64_t l, const double* a_re,
              const double* a_im, int64_t lda, int64_t psa, const double* b_re,
              const double* b_im, int64_t ldb, int64_t psb, double* c_re, double* c_im,
              int64_t ldc, int64_t psc, int epilogue, void* stream) {
  if (bad_k_gemm(k)) return fail("k must be 2, 3, 4 (or 5, 6, 8: verification kernels)");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (m < 0 || n < 0 || l < 0) return fail("negative dimension");
  if (epilogue != 0 && epilogue != 1) return fail("epilogue must be 0 or 1");
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
  table_for(k)->cgemm(method == 3, m, n, l, mpc::View{dar, dai, lda, psa},
                      mpc::View{dbr, dbi, ldb, psb}, mpc::View{dcr, dci, ldc, psc}, epilogue, st,
                      nullptr);
  sg.finish();
  return 0;
  MPC_CATCH
}

int mpc_trsm_ll_unit(int k, int method, int64_t K, int64_t M, const double* l_re,
                     const double* l_im, int64_t ldl, int64_t psl, double* a_re, double* a_im,
                     int64_t lda, int64_t psa, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (K < 0 || M < 0) return fail("negative dimension");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({l_re, l_im, a_re, a_im})) return MPC_ERR;
  int64_t el = extent(k, K, K, ldl, psl), ea = extent(k, K, M, lda, psa);
  double* dlr = sg.map(const_cast<double*>(l_re), el, true, false);
  double* dli = sg.map(const_cast<double*>(l_im), el, true, false);
  double* dar = sg.map(a_re, ea, true, true);
  double* dai = sg.map(a_im, ea, true, true);
  table_for(k)->trsm(method == 3, K, M, mpc::View{dlr, dli, ldl, psl},
                     mpc::View{dar, dai, lda, psa}, st, nullptr);
  sg.finish();
  return 0;
  MPC_CATCH
}

int64_t mpc_panel_factor(int k, int method, int64_t n, int64_t jb, int64_t kw, double* re,
                         double* im, int64_t ld, int64_t ps, int64_t* piv, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0 || jb < 0 || kw < 0 || jb + kw > n) return fail("panel outside the matrix");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv})) return MPC_ERR;
  // re/im point at element (0, jb): column jb + t is at re[i*ld + t]
  int64_t e = extent(k, n, kw, ld, ps);
  double* dr = sg.map(re, e, true, true);
  double* di = sg.map(im, e, true, true);
  int64_t* dp = sg.map(piv, n, true, true);
  int64_t status = -1;
  if (kw > 0) {
    WsHolder w(k, n, st);
    // shift so that global column indices address the panel (never
    // dereferenced left of column jb)
    table_for(k)->panel_rec(method == 3, mpc::View{dr - jb, di - jb, ld, ps}, n, jb, kw, dp,
                            w.ws, st);
    status = w.read_status();
  }
  sg.finish();
  return status;
  MPC_CATCH
}

int mpc_panel_factor_async(int k, int method, int64_t n, int64_t jb, int64_t kw, double* re,
                           double* im, int64_t ld, int64_t ps, int64_t* piv, int64_t* status_out,
                           void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0 || jb < 0 || kw < 0 || jb + kw > n) return fail("panel outside the matrix");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  int dev = -1;
  for (const void* p : {(const void*)re, (const void*)im, (const void*)piv, (const void*)status_out})
    if (ptr_kind(p, &dev) != 2) return fail("mpc_panel_factor_async needs device pointers");
  ck(cudaSetDevice(dev), "cudaSetDevice");
  WsHolder w(k, n, st);
  if (kw > 0)
    table_for(k)->panel_rec(method == 3, mpc::View{re - jb, im - jb, ld, ps}, n, jb, kw, piv,
                            w.ws, st);
  ck(cudaMemcpyAsync(status_out, w.ws.status, sizeof(int64_t), cudaMemcpyDeviceToDevice, st),
     "status copy");
  ck(cudaGetLastError(), "kernel launch");
  return 0;
  MPC_CATCH
}

int mpc_laswp(int k, int64_t ncols, double* re, double* im, int64_t ld, int64_t ps,
              const int64_t* piv, int64_t r0, int64_t r1, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (r0 < 0 || r1 < r0 || ncols < 0) return fail("bad interchange range");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv})) return MPC_ERR;
  // rows touched: up to max(piv[r0..r1)) -- host mode stages the whole
  // leading r1.. rows range conservatively from the pivots
  int64_t rows = r1;
  if (sg.host()) {
    for (int64_t r = r0; r < r1; r++) rows = std::max(rows, piv[r] + 1);
  }
  int64_t e = sg.host() ? extent(k, rows, ncols, ld, ps) : 0;
  double* dr = sg.map(re, e, true, true);
  double* di = sg.map(im, e, true, true);
  const int64_t* dp = sg.map(const_cast<int64_t*>(piv), r1, true, false);
  table_for(k)->laswp(mpc::View{dr, di, ld, ps}, 0, ncols, dp, r0, r1, st, nullptr);
  sg.finish();
  return 0;
  MPC_CATCH
}

int64_t mpc_lu_panel(int k, int method, int64_t n, double* re, double* im, int64_t* piv,
                     int64_t jb, int64_t kw, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0 || jb < 0 || kw < 0 || jb + kw > n) return fail("panel outside the matrix");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv})) return MPC_ERR;
  int64_t e = extent(k, n, n, n, n * n);
  double* dr = sg.map(re, e, true, true);
  double* di = sg.map(im, e, true, true);
  int64_t* dp = sg.map(piv, n, true, true);
  int64_t status = -1;
  if (kw > 0) {
    WsHolder w(k, n, st);
    table_for(k)->lu_panel(method == 3, mpc::View{dr, di, n, n * n}, n, jb, kw, dp, w.ws, st);
    status = w.read_status();
  }
  sg.finish();
  return status;
  MPC_CATCH
}

namespace {
struct HookGuard {  // getrf's host hooks never outlive the call (exceptions included)
  ~HookGuard() {
    mpc::row_sink() = mpc::RowSink{nullptr, nullptr};
    mpc::col_source() = mpc::ColSource{nullptr, nullptr, 0};
  }
};
}  // namespace

int64_t mpc_getrf(int k, int method, int64_t n, int64_t K, double* re, double* im, int64_t* piv,
                  void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0) return fail("negative dimension");
  if (n > 0 && (K < 1 || K > n)) return fail("panel width K outside [1, n]");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv})) return MPC_ERR;
  int64_t e = extent(k, n, n, n, n * n);
  // host factors in pinned memory: the input arrives in column blocks and
  // finished row blocks stream back while the LU runs (HostOverlap)
  const bool overlap = HostOverlap::usable(sg, n, re, im);
  double* dr = sg.map(re, e, !overlap, !overlap);
  double* di = sg.map(im, e, !overlap, !overlap);
  int64_t* dp = sg.map(piv, n, false, true);
  int64_t status = -1;
  HostOverlap ho;
  HookGuard guard;
  if (overlap) {
    ho.start(st, dr, di, re, im, k, n, K);
    mpc::row_sink() = mpc::RowSink{HostOverlap::rows_done, &ho};
    mpc::col_source() = mpc::ColSource{HostOverlap::need, &ho, ho.chunk};
  }
  if (n > 0) {
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dp, n);
    WsHolder w(k, n, st);
    table_for(k)->getrf(method == 3, mpc::View{dr, di, n, n * n}, n, K, dp, w.ws, st);
    mpc::row_sink() = mpc::RowSink{nullptr, nullptr};
    mpc::col_source() = mpc::ColSource{nullptr, nullptr, 0};
    status = w.read_status();
  }
  if (overlap) ho.join(st);
  sg.finish();
  return status;
  MPC_CATCH
}

int mpc_host_register(void* p, int64_t bytes) {
  if (p == nullptr || bytes <= 0) return fail("bad host range");
  MPC_TRY
  ck(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault), "cudaHostRegister");
  return 0;
  MPC_CATCH
}

int mpc_host_unregister(void* p) {
  MPC_TRY
  ck(cudaHostUnregister(p), "cudaHostUnregister");
  return 0;
  MPC_CATCH
}

int mpc_getrs(int k, int method, int64_t n, const double* re, const double* im,
              const int64_t* piv, double* b_re, double* b_im, void* stream) {
  return mpc_getrs_phases(k, method, n, re, im, piv, b_re, b_im, 3, stream);
}

int mpc_getrs_phases(int k, int method, int64_t n, const double* re, const double* im,
                     const int64_t* piv, double* b_re, double* b_im, int phases, void* stream) {
  if (phases < 1 || phases > 3) return fail("phases must be 1, 2 or 3");
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0) return fail("negative dimension");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({re, im, piv, b_re, b_im})) return MPC_ERR;
  int64_t e = extent(k, n, n, n, n * n);
  double* dr = sg.map(const_cast<double*>(re), e, true, false);
  double* di = sg.map(const_cast<double*>(im), e, true, false);
  const int64_t* dp = sg.map(const_cast<int64_t*>(piv), n, true, false);
  double* dbr = sg.map(b_re, (int64_t)k * n, true, true);
  double* dbi = sg.map(b_im, (int64_t)k * n, true, true);
  if (n > 0)
    table_for(k)->getrs(method == 3, mpc::View{dr, di, n, n * n}, n, dp, dbr, dbi, phases, st);
  sg.finish();
  return 0;
  MPC_CATCH
}

}  // extern "C"
