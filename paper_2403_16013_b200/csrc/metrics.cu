// metrics.cu -- max_rel_err (lu.py:263-282 of the reference) on the GPU, in
// the reference's own expansion arithmetic, so the metric is the reference's
// value bit for bit (the reference carries it as a k-component expansion and
// prints it with exp_to_string; a binary64 restatement would differ in the
// digits beyond double precision).
//
// Per entry i (one thread each):
//   d      = csub(xhat_i, x_i)                      (cscalar.py:74-76)
//   d2     = exp_add(exp_mul(d.re, d.re), exp_mul(d.im, d.im))
//   x2     = exp_add(exp_mul(x.re, x.re), exp_mul(x.im, x.im))
//   ratio  = exp_div(d2, x2)
// then the first entry whose ratio is strictly greater than every earlier one
// (the sign of the exact expansion difference, ties to the lower index: a
// total preorder, so the block reduction returns the reference's entry),
// then sqrt by three Newton steps from the binary64 seed (_exp_sqrt,
// lu.py:253-260).  A zero true component reports its index (the reference
// raises ValueError there).
#include <cuda_runtime.h>

#include <cstdint>

#include "abi_util.h"
#include "expansion.cuh"
#include "prof.h"

namespace mpc {

template <int K>
struct Ratio {
  Exp<K> v;
  int64_t idx;  // -1: none
};

template <int K>
MPC_DI bool ratio_better(const Ratio<K>& a, const Ratio<K>& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  Exp<K> d = exp_sub(a.v, b.v);
  if (d.c[0] > 0.0) return true;
  if (d.c[0] < 0.0) return false;
  return a.idx < b.idx;
}

template <int K>
MPC_DI Ratio<K> shfl_ratio(const Ratio<K>& r, int off) {
  Ratio<K> o;
#pragma unroll
  for (int c = 0; c < K; c++) o.v.c[c] = __shfl_down_sync(0xffffffffu, r.v.c[c], off);
  o.idx = __shfl_down_sync(0xffffffffu, r.idx, off);
  return o;
}

constexpr int MNT = 256;

// out[0..K): the result; info[0]: index of the first zero true component or -1
template <int K>
__global__ void __launch_bounds__(MNT) max_rel_err_kernel(const double* __restrict__ hr,
                                                          const double* __restrict__ hi,
                                                          const double* __restrict__ xr,
                                                          const double* __restrict__ xi, int64_t n,
                                                          double* out, int64_t* info) {
  __shared__ double sv[MNT / 32][K];
  __shared__ int64_t si[MNT / 32];
  __shared__ unsigned long long zero_at;
  if (threadIdx.x == 0) zero_at = ~0ull;
  __syncthreads();
  Ratio<K> best;
  best.idx = -1;
  best.v = exp_zero<K>();
  for (int64_t i = threadIdx.x; i < n; i += MNT) {
    Exp<K> ar, ai, br, bi;
#pragma unroll
    for (int c = 0; c < K; c++) {
      ar.c[c] = hr[c * n + i];
      ai.c[c] = hi[c * n + i];
      br.c[c] = xr[c * n + i];
      bi.c[c] = xi[c * n + i];
    }
    if (br.c[0] == 0.0 && bi.c[0] == 0.0) {  // ComplexScalar.is_zero (cscalar.py:54-55)
      atomicMin(&zero_at, (unsigned long long)i);
      continue;
    }
    const Exp<K> dr = exp_sub(ar, br), di = exp_sub(ai, bi);
    const Exp<K> d2 = exp_add(exp_mul(dr, dr), exp_mul(di, di));
    const Exp<K> x2 = exp_add(exp_mul(br, br), exp_mul(bi, bi));
    Ratio<K> r;
    r.v = exp_div(d2, x2);
    r.idx = i;
    if (ratio_better(r, best)) best = r;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Ratio<K> o = shfl_ratio(best, off);
    if (ratio_better(o, best)) best = o;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < K; c++) sv[w][c] = best.v.c[c];
    si[w] = best.idx;
  }
  __syncthreads();
  if (w != 0) return;
  if (lane < MNT / 32) {
#pragma unroll
    for (int c = 0; c < K; c++) best.v.c[c] = sv[lane][c];
    best.idx = si[lane];
  } else {
    best.idx = -1;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Ratio<K> o = shfl_ratio(best, off);
    if (ratio_better(o, best)) best = o;
  }
  if (lane != 0) return;
  info[0] = zero_at == ~0ull ? -1 : (int64_t)zero_at;
  Exp<K> s = exp_zero<K>();
  if (best.idx >= 0 && best.v.c[0] != 0.0) {  // _exp_sqrt: Newton from the binary64 seed
    s.c[0] = __dsqrt_rn(best.v.c[0]);
    Exp<K> half = exp_zero<K>();
    half.c[0] = 0.5;
    for (int it = 0; it < 3; it++) s = exp_mul(exp_add(s, exp_div(best.v, s)), half);
  }
#pragma unroll
  for (int c = 0; c < K; c++) out[c] = s.c[c];
}

template <int K>
void launch_max_rel_err(const double* hr, const double* hi, const double* xr, const double* xi,
                        int64_t n, double* out, int64_t* info, cudaStream_t st) {
  int tok_ = prof_begin(PC_OTHER, 0.0, st);
  max_rel_err_kernel<K><<<1, MNT, 0, st>>>(hr, hi, xr, xi, n, out, info);
  prof_end(tok_, st);
}

}  // namespace mpc

using namespace mpcabi;

extern "C" int mpc_max_rel_err(int k, int64_t n, const double* xhat_re, const double* xhat_im,
                               const double* x_re, const double* x_im, double* out,
                               int64_t* zero_index, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (n < 1) return fail("n must be >= 1");
  MPC_TRY
  cudaStream_t st = (cudaStream_t)stream;
  Stager sg(st);
  if (!sg.classify({xhat_re, xhat_im, x_re, x_im, out, zero_index})) return MPC_ERR;
  const int64_t e = (int64_t)k * n;
  const double* hr = sg.map(const_cast<double*>(xhat_re), e, true, false);
  const double* hi = sg.map(const_cast<double*>(xhat_im), e, true, false);
  const double* xr = sg.map(const_cast<double*>(x_re), e, true, false);
  const double* xi = sg.map(const_cast<double*>(x_im), e, true, false);
  double* o = sg.map(out, k, false, true);
  int64_t* z = sg.map(zero_index, 1, false, true);
  if (k == 2) mpc::launch_max_rel_err<2>(hr, hi, xr, xi, n, o, z, st);
  else if (k == 3) mpc::launch_max_rel_err<3>(hr, hi, xr, xi, n, o, z, st);
  else mpc::launch_max_rel_err<4>(hr, hi, xr, xi, n, o, z, st);
  sg.finish();
  return 0;
  MPC_CATCH
}
