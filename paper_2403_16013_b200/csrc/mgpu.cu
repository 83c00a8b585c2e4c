// mgpu.cu -- single-process multi-GPU blocked LU (mpc_getrf_ngpu): the
// SURVEY.md §8b/§8e entry point `mpc_getrf(..., ngpus, lookahead, ...)`.
//
// lu._factor (lu.py:129-163) over P devices of this process with a 1-D
// block-column-cyclic distribution: block column b (global columns
// [b*K, min((b+1)*K, n))) lives on rank b mod P, each rank storing its blocks
// side by side in a local (k, n, ncols) array per Re / Im.  Step b:
//   1. the owner factors panel b in its local storage (recursive panel,
//      interchanges applied inside the panel only) and packs rows [jb, n)
//      of it into a contiguous panel slot (k, n-jb, kw);
//   2. every other rank PULLS the slot, piv[jb, jb+kw) and the status word
//      from the owner over NVLink (peer copies on its own copy stream, so
//      the transfer of panel b+1 overlaps step b's trailing update);
//   3. every rank applies the interchanges to its other columns (LASWP),
//      solves its U12 columns (TRSM with L11 from the slot) and applies the
//      fused trailing update A22 -= L21 U12 (EFT 3M/4M GEMM or the Ozaki
//      tensor-core GEMM) to its columns right of the panel.
// Depth-1 lookahead: the owner of block b+1 updates that block first, then
// factors and packs panel b+1 on a high-priority side stream while its main
// stream finishes step b.  Every element keeps the operation sequence of the
// 1-GPU factorization (panel, TRSM and GEMM chains are per element and
// independent of the column distribution), so the result is bit-identical
// to mpc_getrf and to the reference.
//
// Ranks map to device ordinals (current + r) mod device_count; ngpus larger
// than the device count is an error unless MPC_MGPU_OVERSUBSCRIBE=1 (then
// several ranks share a device -- a correctness mode for 1-GPU test boxes:
// only stream/event dependencies, no kernel ever waits on another).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <vector>

#include "abi_util.h"

namespace mpc {
// ozaki.cu
int resolve_width(int k, int64_t inner, int split_bits);
void cgemm_ozaki_dev(int k, bool use3m, int64_t m, int64_t n, int64_t l, View A, View B, View C,
                     int epi, int d, int width, cudaStream_t st);
}  // namespace mpc

using namespace mpcabi;

namespace {

__global__ void iota_kernel_mg(int64_t* p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

struct DevScope {  // restores the caller's current device
  int prev = 0;
  DevScope() { cudaGetDevice(&prev); }
  ~DevScope() { cudaSetDevice(prev); }
};

struct Rank {
  int dev = 0;
  cudaStream_t st = nullptr, sp = nullptr, cs = nullptr;  // main, side (panel), copy-in
  double *loc_re = nullptr, *loc_im = nullptr;
  double *pan_re[2] = {nullptr, nullptr}, *pan_im[2] = {nullptr, nullptr};
  int64_t* piv = nullptr;
  void* wsmem = nullptr;
  mpc::PanelWs ws{};
  int64_t ncols = 0;
  std::vector<int> owned;         // block indices, ascending
  std::vector<int64_t> lcol;      // local column of every block (-1: not owned)
  ~Rank() {
    cudaSetDevice(dev);
    for (void* p : {(void*)loc_re, (void*)loc_im, (void*)pan_re[0], (void*)pan_re[1],
                    (void*)pan_im[0], (void*)pan_im[1], (void*)piv, wsmem})
      if (p) cudaFree(p);
    for (cudaStream_t s : {st, sp, cs})
      if (s) cudaStreamDestroy(s);
  }
};

struct Events {  // all per-step events, destroyed together
  std::vector<cudaEvent_t> all;
  cudaEvent_t make() {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    all.push_back(e);
    return e;
  }
  ~Events() {
    for (auto e : all) cudaEventDestroy(e);
  }
};

void* dmalloc(size_t bytes) {
  void* p = nullptr;
  ck(cudaMalloc(&p, bytes ? bytes : 8), "cudaMalloc");
  return p;
}

}  // namespace

extern "C" {

int64_t mpc_getrf_ngpu(int k, int method, int64_t n, int64_t K, double* re, double* im,
                       int64_t* piv, int ngpus, int lookahead, int real_kernel, int d,
                       int split_bits, void* stream) {
  if (bad_k(k)) return fail("k must be 2, 3 or 4");
  if (bad_method(method)) return fail("method must be 3 (3M) or 4 (4M)");
  if (n < 0) return fail("negative dimension");
  if (n > 0 && (K < 1 || K > n)) return fail("panel width K outside [1, n]");
  if (ngpus < 1) return fail("ngpus must be >= 1");
  if (real_kernel != 0 && real_kernel != 1) return fail("real_kernel must be 0 (EFT) or 1 (ozaki)");
  if (real_kernel == 1 && d < 1) return fail("d must be >= 1");
  if (ngpus == 1 && real_kernel == 0 && lookahead) return mpc_getrf(k, method, n, K, re, im, piv, stream);
  if (ngpus == 1 && real_kernel == 1) return mpc_getrf_ozaki(k, method, n, K, re, im, piv, d, split_bits, stream);
  MPC_TRY
  DevScope restore;
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  const char* ov = getenv("MPC_MGPU_OVERSUBSCRIBE");
  const bool oversub = ov && ov[0] == '1';
  if (ngpus > ndev && !oversub)
    return fail("ngpus exceeds the visible CUDA devices (" + std::to_string(ndev) + ")");
  if (n == 0) return -1;
  if (real_kernel == 1 && n > K && mpc::resolve_width(k, K, split_bits) < 0)
    return fail("dimension exceeds split exactness budget");
  const int P = ngpus;
  const bool use3m = method == 3;
  const mpc::OpsTable* T = table_for(k);
  const int nb = (int)((n + K - 1) / K);
  auto width = [&](int b) { return std::min<int64_t>(K, n - (int64_t)b * K); };
  auto owner = [&](int b) { return b % P; };
  int cur = 0;
  ck(cudaGetDevice(&cur), "cudaGetDevice");
  cudaStream_t caller = (cudaStream_t)stream;
  // the caller's stream may still be producing device-pointer inputs
  cudaEvent_t ev_in;
  ck(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventRecord(ev_in, caller), "cudaEventRecord");
  std::vector<std::unique_ptr<Rank>> R;
  for (int r = 0; r < P; r++) {
    auto rk = std::make_unique<Rank>();
    rk->dev = (cur + r) % ndev;
    rk->lcol.assign(nb, -1);
    for (int b = r; b < nb; b += P) {
      rk->owned.push_back(b);
      rk->lcol[b] = rk->ncols;
      rk->ncols += width(b);
    }
    R.push_back(std::move(rk));
  }
  // peer access between every pair of distinct devices (NVLink / NVSwitch)
  for (int a = 0; a < P; a++)
    for (int b = 0; b < P; b++) {
      int da = R[a]->dev, db = R[b]->dev, can = 0;
      if (da == db) continue;
      ck(cudaSetDevice(da), "cudaSetDevice");
      if (cudaDeviceCanAccessPeer(&can, da, db) == cudaSuccess && can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          ck(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    }
  int lo = 0, hi = 0;
  ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
  const size_t pitch_h = sizeof(double) * (size_t)n;
  for (auto& rk : R) {
    ck(cudaSetDevice(rk->dev), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&rk->st, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithPriority(&rk->sp, cudaStreamNonBlocking, hi), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&rk->cs, cudaStreamNonBlocking), "cudaStreamCreate");
    const size_t loc = sizeof(double) * (size_t)k * n * rk->ncols;
    rk->loc_re = (double*)dmalloc(loc);
    rk->loc_im = (double*)dmalloc(loc);
    const size_t pan = sizeof(double) * (size_t)k * n * std::min<int64_t>(K, n);
    for (int s = 0; s < 2; s++) {
      rk->pan_re[s] = (double*)dmalloc(pan);
      rk->pan_im[s] = (double*)dmalloc(pan);
    }
    rk->piv = (int64_t*)dmalloc(sizeof(int64_t) * n);
    rk->wsmem = dmalloc(mpc::panel_ws_bytes(k, n));
    rk->ws = mpc::panel_ws_carve(rk->wsmem, k, n);
    ck(cudaStreamWaitEvent(rk->st, ev_in, 0), "cudaStreamWaitEvent");
    ck(mpc::panel_ws_init(rk->ws, rk->st), "memset ws");
    iota_kernel_mg<<<(unsigned)((n + 255) / 256), 256, 0, rk->st>>>(rk->piv, n);
    ck(cudaGetLastError(), "iota");
    // scatter: this rank's block columns, every limb plane (H2D, or peer /
    // device copies for device-pointer inputs -- UVA picks the direction)
    for (int b : rk->owned) {
      const size_t w8 = sizeof(double) * (size_t)width(b);
      for (int q = 0; q < k; q++) {
        const size_t ho = (size_t)q * n * n + (size_t)b * K;
        const size_t lo_ = (size_t)q * n * rk->ncols + (size_t)rk->lcol[b];
        ck(cudaMemcpy2DAsync(rk->loc_re + lo_, sizeof(double) * rk->ncols, re + ho, pitch_h, w8,
                             (size_t)n, cudaMemcpyDefault, rk->st), "scatter");
        ck(cudaMemcpy2DAsync(rk->loc_im + lo_, sizeof(double) * rk->ncols, im + ho, pitch_h, w8,
                             (size_t)n, cudaMemcpyDefault, rk->st), "scatter");
      }
    }
  }
  cudaEventDestroy(ev_in);

  Events E;
  // ev_packed[b]: owner's slot b%2 holds panel b (rows jb..n), its piv and status
  // ev_pulled[r][b]: rank r's slot b%2 holds panel b
  // ev_used[r][b]: rank r's main stream finished every use of slot b%2 for step b
  std::vector<cudaEvent_t> ev_packed(nb), ev_narrow(nb);
  std::vector<std::vector<cudaEvent_t>> ev_pulled(P, std::vector<cudaEvent_t>(nb)),
      ev_used(P, std::vector<cudaEvent_t>(nb));
  for (int b = 0; b < nb; b++) {
    ck(cudaSetDevice(R[owner(b)]->dev), "cudaSetDevice");
    ev_packed[b] = E.make();
    ev_narrow[b] = E.make();
    for (int r = 0; r < P; r++) {
      ck(cudaSetDevice(R[r]->dev), "cudaSetDevice");
      ev_pulled[r][b] = E.make();
      ev_used[r][b] = E.make();
    }
  }
  auto lview = [&](Rank& rk) {
    return mpc::View{rk.loc_re, rk.loc_im, rk.ncols, n * rk.ncols};
  };
  auto sview = [&](Rank& rk, int b) {
    const int64_t jb = (int64_t)b * K, kw = width(b);
    return mpc::View{rk.pan_re[b & 1], rk.pan_im[b & 1], kw, (n - jb) * kw};
  };
  // before rank r's slot (b % 2) is written for step b: its own step b-2
  // uses are done, and if r owned step b-2 every other rank has pulled it
  auto wait_slot_free = [&](int r, int b, cudaStream_t s) {
    if (b < 2) return;
    ck(cudaStreamWaitEvent(s, ev_used[r][b - 2], 0), "wait slot");
    if (owner(b - 2) == r)
      for (int o = 0; o < P; o++)
        if (o != r) ck(cudaStreamWaitEvent(s, ev_pulled[o][b - 2], 0), "wait slot");
  };
  // owner: factor panel b in place and pack it into its slot, on stream s
  auto factor_pack = [&](int b, cudaStream_t s) {
    const int o = owner(b);
    Rank& rk = *R[o];
    ck(cudaSetDevice(rk.dev), "cudaSetDevice");
    const int64_t jb = (int64_t)b * K, kw = width(b), lc = rk.lcol[b];
    mpc::View V{rk.loc_re + lc - jb, rk.loc_im + lc - jb, rk.ncols, n * rk.ncols};
    T->panel_rec(use3m, V, n, jb, kw, rk.piv, rk.ws, s);
    wait_slot_free(o, b, s);
    for (int q = 0; q < k; q++) {
      const size_t src = (size_t)q * n * rk.ncols + (size_t)jb * rk.ncols + (size_t)lc;
      const size_t dst = (size_t)q * (n - jb) * kw;
      ck(cudaMemcpy2DAsync(rk.pan_re[b & 1] + dst, sizeof(double) * kw, rk.loc_re + src,
                           sizeof(double) * rk.ncols, sizeof(double) * kw, (size_t)(n - jb),
                           cudaMemcpyDeviceToDevice, s), "pack");
      ck(cudaMemcpy2DAsync(rk.pan_im[b & 1] + dst, sizeof(double) * kw, rk.loc_im + src,
                           sizeof(double) * rk.ncols, sizeof(double) * kw, (size_t)(n - jb),
                           cudaMemcpyDeviceToDevice, s), "pack");
    }
    ck(cudaEventRecord(ev_packed[b], s), "cudaEventRecord");
    ck(cudaEventRecord(ev_pulled[o][b], s), "cudaEventRecord");
  };
  // rank r != owner: pull panel b, its pivots and the status word
  auto pull = [&](int r, int b) {
    const int o = owner(b);
    Rank& rk = *R[r];
    Rank& ok_ = *R[o];
    ck(cudaSetDevice(rk.dev), "cudaSetDevice");
    const int64_t jb = (int64_t)b * K, kw = width(b);
    ck(cudaStreamWaitEvent(rk.cs, ev_packed[b], 0), "wait packed");
    wait_slot_free(r, b, rk.cs);
    const size_t bytes = sizeof(double) * (size_t)k * (n - jb) * kw;
    ck(cudaMemcpyAsync(rk.pan_re[b & 1], ok_.pan_re[b & 1], bytes, cudaMemcpyDefault, rk.cs), "pull");
    ck(cudaMemcpyAsync(rk.pan_im[b & 1], ok_.pan_im[b & 1], bytes, cudaMemcpyDefault, rk.cs), "pull");
    ck(cudaMemcpyAsync(rk.piv + jb, ok_.piv + jb, sizeof(int64_t) * kw, cudaMemcpyDefault, rk.cs),
       "pull piv");
    ck(cudaMemcpyAsync(rk.ws.status, ok_.ws.status, sizeof(int64_t), cudaMemcpyDefault, rk.cs),
       "pull status");
    ck(cudaEventRecord(ev_pulled[r][b], rk.cs), "cudaEventRecord");
  };
  auto update = [&](Rank& rk, const mpc::View& S, int64_t jb, int64_t kw, int64_t lo_c,
                    int64_t hi_c, cudaStream_t s) {
    if (hi_c <= lo_c) return;
    const int64_t end = jb + kw, M = hi_c - lo_c;
    mpc::View L = lview(rk);
    T->trsm(use3m, kw, M, S, L.sub(jb, lo_c), s, rk.ws.status);
    if (end < n) {
      if (real_kernel == 1)
        mpc::cgemm_ozaki_dev(k, use3m, n - end, kw, M, S.sub(kw, 0), L.sub(jb, lo_c),
                             L.sub(end, lo_c), 1, d, mpc::resolve_width(k, kw, split_bits), s);
      else
        T->cgemm(use3m, n - end, kw, M, S.sub(kw, 0), L.sub(jb, lo_c), L.sub(end, lo_c), 1, s,
                 rk.ws.status);
    }
  };
  auto swaps = [&](Rank& rk, int b, int64_t lo_c, int64_t hi_c, cudaStream_t s) {
    // interchanges of panel b on local columns [lo_c, hi_c), except the panel itself
    const int64_t jb = (int64_t)b * K, end = jb + width(b);
    mpc::View L = lview(rk);
    int64_t pl = rk.lcol[b], ph = pl >= 0 ? pl + width(b) : -1;
    if (pl < 0 || hi_c <= pl || lo_c >= ph) {
      T->laswp(L, lo_c, hi_c - lo_c, rk.piv, jb, end, s, rk.ws.status);
    } else {
      T->laswp(L, lo_c, pl - lo_c, rk.piv, jb, end, s, rk.ws.status);
      T->laswp(L, ph, hi_c - ph, rk.piv, jb, end, s, rk.ws.status);
    }
  };
  auto first_owned_after = [&](Rank& rk, int b) -> int {
    for (int ob : rk.owned)
      if (ob > b) return ob;
    return -1;
  };

  factor_pack(0, R[owner(0)]->st);
  for (int r = 0; r < P; r++)
    if (r != owner(0)) pull(r, 0);
  for (int b = 0; b < nb; b++) {
    const int64_t jb = (int64_t)b * K, kw = width(b);
    const int nxt = b + 1 < nb ? b + 1 : -1;
    for (int r = 0; r < P; r++) {
      Rank& rk = *R[r];
      ck(cudaSetDevice(rk.dev), "cudaSetDevice");
      ck(cudaStreamWaitEvent(rk.st, ev_pulled[r][b], 0), "wait pulled");
      const mpc::View S = sview(rk, b);
      const int tb = first_owned_after(rk, b);
      const int64_t t0 = tb >= 0 ? rk.lcol[tb] : rk.ncols;  // trailing local columns [t0, ncols)
      if (nxt >= 0 && owner(nxt) == r && lookahead) {
        // narrow update of block nxt, then its panel on the side stream
        const int64_t c0 = rk.lcol[nxt], c1 = c0 + width(nxt);
        swaps(rk, b, c0, c1, rk.st);
        update(rk, S, jb, kw, c0, c1, rk.st);
        ck(cudaEventRecord(ev_narrow[nxt], rk.st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(rk.sp, ev_narrow[nxt], 0), "wait narrow");
        factor_pack(nxt, rk.sp);
        ck(cudaSetDevice(rk.dev), "cudaSetDevice");
        swaps(rk, b, 0, c0, rk.st);
        swaps(rk, b, c1, rk.ncols, rk.st);
        update(rk, S, jb, kw, std::max(t0, c1), rk.ncols, rk.st);
        ck(cudaEventRecord(ev_used[r][b], rk.st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(rk.st, ev_packed[nxt], 0), "wait own panel");
      } else {
        swaps(rk, b, 0, rk.ncols, rk.st);
        update(rk, S, jb, kw, t0, rk.ncols, rk.st);
        ck(cudaEventRecord(ev_used[r][b], rk.st), "cudaEventRecord");
        if (nxt >= 0 && owner(nxt) == r) {  // no lookahead: factor after the whole update
          factor_pack(nxt, rk.st);
        }
      }
    }
    if (nxt >= 0)
      for (int r = 0; r < P; r++)
        if (r != owner(nxt)) pull(r, nxt);
  }
  // gather: every rank's blocks back to the caller's buffers, pivots from rank 0
  for (auto& rk : R) {
    ck(cudaSetDevice(rk->dev), "cudaSetDevice");
    for (int b : rk->owned) {
      const size_t w8 = sizeof(double) * (size_t)width(b);
      for (int q = 0; q < k; q++) {
        const size_t ho = (size_t)q * n * n + (size_t)b * K;
        const size_t lo_ = (size_t)q * n * rk->ncols + (size_t)rk->lcol[b];
        ck(cudaMemcpy2DAsync(re + ho, pitch_h, rk->loc_re + lo_, sizeof(double) * rk->ncols, w8,
                             (size_t)n, cudaMemcpyDefault, rk->st), "gather");
        ck(cudaMemcpy2DAsync(im + ho, pitch_h, rk->loc_im + lo_, sizeof(double) * rk->ncols, w8,
                             (size_t)n, cudaMemcpyDefault, rk->st), "gather");
      }
    }
  }
  Rank& r0 = *R[0];
  ck(cudaSetDevice(r0.dev), "cudaSetDevice");
  ck(cudaMemcpyAsync(piv, r0.piv, sizeof(int64_t) * n, cudaMemcpyDefault, r0.st), "pivots");
  int64_t status = -1;
  ck(cudaMemcpyAsync(&status, r0.ws.status, sizeof(int64_t), cudaMemcpyDeviceToHost, r0.st),
     "status");
  for (auto& rk : R) {
    ck(cudaSetDevice(rk->dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(rk->st), "cudaStreamSynchronize");
    ck(cudaStreamSynchronize(rk->sp), "cudaStreamSynchronize");
    ck(cudaStreamSynchronize(rk->cs), "cudaStreamSynchronize");
  }
  ck(cudaGetLastError(), "kernel launch");
  return status;
  MPC_CATCH
}

}  // extern "C"
