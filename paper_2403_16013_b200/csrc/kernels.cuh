// kernels.cuh -- sm_100a kernels and the host-side launch logic for the
// complex multi-component GEMM and blocked LU (templated on the component
// count K; instantiated per K in inst_k*.cu).
//
// Reference path (paths relative to /root/reference/pkg/src/mpclu/):
//   cgemm_3m / cgemm_4m   cmatrix.py:145-177   -> gemm_kernel<MODE_G3/G4>
//   rgemm_naive/blocked   rgemm.py:53-73, _kernels.py:363-434 -> MODE_REAL
//   mat_add_k             _kernels.py:327-342  -> mat_add_kernel
//   renorm_planes         _kernels.py:485-499  -> renorm_planes_kernel
//   lu_panel              _kernels.py:611-665  -> panel_rec (pivot/step kernels + S)
//   trsm_ll_unit          _kernels.py:668-705  -> trsm_rec (diag kernel + S)
//   lu._factor            lu.py:129-163        -> getrf
//   solve_fb              _kernels.py:708-775  -> getrs
//
// Bit-exactness contract: every output element keeps the
// reference's exact sequence of expansion operations.  GEMM chains are
// output-stationary, t-ascending, never split along the inner dimension; the
// in-panel / TRSM updates ("S" mode) keep each element's chained subtractions
// a -= cmul(l, u) in column order; row interchanges are deferred (LASWP),
// which commutes with the row operations.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdint>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>
#include "expansion.cuh"
#include "prof.h"

namespace mpc {

// ------------------------------------------------------------------ views
struct View {  // planar complex (or real: im unused) sub-matrix
  double* re;
  double* im;
  int64_t ld;  // row stride (elements)
  int64_t ps;  // plane (limb) stride (elements)
  __host__ __device__ View sub(int64_t r, int64_t c) const {
    return View{re + r * ld + c, im ? im + r * ld + c : nullptr, ld, ps};
  }
};

template <int K>
MPC_DI Exp<K> ldexp_(const double* p, int64_t ps) {
  Exp<K> e;
#pragma unroll
  for (int c = 0; c < K; c++) e.c[c] = p[c * ps];
  return e;
}
template <int K>
MPC_DI void stexp_(double* p, int64_t ps, const Exp<K>& e) {
#pragma unroll
  for (int c = 0; c < K; c++) p[c * ps] = e.c[c];
}

// --------------------------------------------------------- GEMM family
// grouped raster: G consecutive row tiles sweep the column tiles together
#ifndef MPC_GEMM_RASTER_G
#define MPC_GEMM_RASTER_G 32
#endif
enum Mode { MODE_REAL = 0, MODE_G3 = 1, MODE_G4 = 2, MODE_S3 = 3, MODE_S4 = 4 };

template <int MODE>
struct ModeInfo;
// NLOAD operands staged from global per side (re[, im]); NS smem slots per
// side (3M adds the Re+Im sum slot, formed once per staged element);
// NACC expansions accumulated per output element.
template <> struct ModeInfo<MODE_REAL> { static constexpr int NLOAD = 1, NS = 1, NACC = 1; static constexpr bool SUMS = false, CHAINED = false; };
template <> struct ModeInfo<MODE_G3>   { static constexpr int NLOAD = 2, NS = 3, NACC = 3; static constexpr bool SUMS = true,  CHAINED = false; };
template <> struct ModeInfo<MODE_G4>   { static constexpr int NLOAD = 2, NS = 2, NACC = 4; static constexpr bool SUMS = false, CHAINED = false; };
template <> struct ModeInfo<MODE_S3>   { static constexpr int NLOAD = 2, NS = 3, NACC = 2; static constexpr bool SUMS = true,  CHAINED = true; };
template <> struct ModeInfo<MODE_S4>   { static constexpr int NLOAD = 2, NS = 2, NACC = 2; static constexpr bool SUMS = false, CHAINED = true; };

struct GemmArgs {
  int64_t m, n, l;  // C (m x l) op= A (m x n) * B (n x l)
  View a, b, c;
  int epi;  // G modes: 0 -> C = P, 1 -> C = C - P (lu.py:157-161 order)
  const int64_t* status;  // LU early-out: skip when *status >= 0
  // tile queue (nullptr: one tile per CTA, tile = blockIdx.x): persistent CTAs
  // claim tiles with atomicAdd, so a launch may use fewer CTAs than tiles and
  // several launches can share one queue (getrf's capped trailing update)
  unsigned* tile_ctr = nullptr;
};

MPC_DI void cp_async8(void* smem_ptr, const double* gptr, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gptr), "r"(sz));
}
MPC_DI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
MPC_DI void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One CTA computes a BM x BN tile of C with (BM/TM) x (BN/TN) threads; each
// thread owns a TM x TN strided micro-tile and NACC expansion chains per
// element.  The inner dimension is staged through shared memory in BK slabs
// with a two-stage cp.async pipeline.  Shared layout per stage keeps the
// limbs of one element adjacent (one LDS.128 per DD operand):
//   As[NS][BM][BK][K], Bs[NS][BK][BN][K].
// Per slab: compute(kt) | wait(kt+1), barrier | Re+Im sums of kt+1 (3M) and
// issue the loads of kt+2 | barrier -- two barriers per slab (one without
// sums).
template <int K, int MODE, int BM, int BN, int BK, int TM, int TN>
struct GemmCfg {
  using MI = ModeInfo<MODE>;
  static constexpr int SX = BN / TN, SY = BM / TM, NT = SX * SY;
  static constexpr int A_STAGE = MI::NS * K * BM * BK;
  static constexpr int B_STAGE = MI::NS * K * BK * BN;
  static constexpr size_t SMEM = sizeof(double) * 2 * (A_STAGE + B_STAGE);
};

// K consecutive doubles from shared memory (vectorised for even K)
template <int K>
MPC_DI Exp<K> lds_exp(const double* p) {
  Exp<K> e;
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 2) {
      double2 v = *reinterpret_cast<const double2*>(p + c);
      e.c[c] = v.x;
      e.c[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < K; c++) e.c[c] = p[c];
  }
  return e;
}
template <int K>
MPC_DI void sts_exp(double* p, const Exp<K>& e) {
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 2)
      *reinterpret_cast<double2*>(p + c) = make_double2(e.c[c], e.c[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < K; c++) p[c] = e.c[c];
  }
}

template <int K, int MODE, int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__(GemmCfg<K, MODE, BM, BN, BK, TM, TN>::NT, MINB)
    gemm_kernel(GemmArgs g) {
  using Cfg = GemmCfg<K, MODE, BM, BN, BK, TM, TN>;
  using MI = ModeInfo<MODE>;
  constexpr int SX = Cfg::SX, SY = Cfg::SY, NT = Cfg::NT;
  constexpr int NS = MI::NS, NL = MI::NLOAD, NACC = MI::NACC;
  constexpr int A_STAGE = Cfg::A_STAGE, B_STAGE = Cfg::B_STAGE;
  constexpr int AE = NL * K * BM * BK, BE = NL * K * BK * BN;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + 2 * A_STAGE;

  if (g.status != nullptr && *g.status >= 0) return;
  const int tid = threadIdx.x;
  const int tx = tid % SX, ty = tid / SX;
  // grouped raster: G consecutive row tiles sweep the column tiles together,
  // so one B column panel is reused from L2 by G CTAs in flight
  constexpr int64_t G = MPC_GEMM_RASTER_G;
  const int64_t tiles_m = (g.m + BM - 1) / BM, tiles_n = (g.l + BN - 1) / BN;
  __shared__ unsigned next_tile;
  for (;;) {
  int64_t bid = blockIdx.x;
  if (g.tile_ctr != nullptr) {
    __syncthreads();  // everyone is done with the previous tile's slabs / next_tile
    if (tid == 0) next_tile = atomicAdd(g.tile_ctr, 1u);
    __syncthreads();
    bid = next_tile;
    if (bid >= tiles_m * tiles_n) return;
  }
  const int64_t grp = bid / (G * tiles_n);
  const int64_t first_m = grp * G;
  const int64_t gsz = min(tiles_m - first_m, G);
  const int64_t in_grp = bid - grp * G * tiles_n;
  const int64_t row0 = (first_m + in_grp % gsz) * BM, col0 = (in_grp / gsz) * BN;

  // accumulators
  Exp<K> acc[TM][TN][NACC];
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int c = 0; c < TN; c++) {
      if constexpr (MI::CHAINED) {
        int64_t gi = row0 + ty + r * SY, gj = col0 + tx + c * SX;
        if (gi < g.m && gj < g.l) {
          acc[r][c][0] = ldexp_<K>(g.c.re + gi * g.c.ld + gj, g.c.ps);
          acc[r][c][1] = ldexp_<K>(g.c.im + gi * g.c.ld + gj, g.c.ps);
        } else {
          acc[r][c][0] = exp_zero<K>();
          acc[r][c][1] = exp_zero<K>();
        }
      } else {
#pragma unroll
        for (int q = 0; q < NACC; q++) acc[r][c][q] = exp_zero<K>();
      }
    }

  // element e of a stage: tt (A) / cc (B) fastest -> coalesced global reads
  auto load_stage = [&](int st, int64_t t0) {
    double* as = As + st * A_STAGE;
    double* bs = Bs + st * B_STAGE;
#pragma unroll
    for (int i = 0; i < (AE + NT - 1) / NT; i++) {
      const int e = tid + i * NT;
      if (AE % NT != 0 && e >= AE) break;
      const int tt = e % BK, r = (e / BK) % BM, c = (e / (BK * BM)) % K, op = e / (BK * BM * K);
      const int64_t gi = row0 + r, gt = t0 + tt;
      const bool v = gi < g.m && gt < g.n;
      const double* base = (op == 0) ? g.a.re : g.a.im;
      const double* src = v ? base + c * g.a.ps + gi * g.a.ld + gt : base;
      cp_async8(as + ((op * BM + r) * BK + tt) * K + c, src, v);
    }
#pragma unroll
    for (int i = 0; i < (BE + NT - 1) / NT; i++) {
      const int e = tid + i * NT;
      if (BE % NT != 0 && e >= BE) break;
      const int cc = e % BN, tt = (e / BN) % BK, c = (e / (BN * BK)) % K, op = e / (BN * BK * K);
      const int64_t gt = t0 + tt, gj = col0 + cc;
      const bool v = gt < g.n && gj < g.l;
      const double* base = (op == 0) ? g.b.re : g.b.im;
      const double* src = v ? base + c * g.b.ps + gt * g.b.ld + gj : base;
      cp_async8(bs + ((op * BK + tt) * BN + cc) * K + c, src, v);
    }
  };

  // slot 2 = Re + Im (mat_add_k / cmul_3m_core's exp_add), once per element
  auto sums = [&](int st) {
    if constexpr (MI::SUMS) {
      double* as = As + st * A_STAGE;
      double* bs = Bs + st * B_STAGE;
      for (int e = tid; e < BM * BK; e += NT) {
        Exp<K> x = lds_exp<K>(as + e * K);
        Exp<K> y = lds_exp<K>(as + (BM * BK + e) * K);
        sts_exp<K>(as + (2 * BM * BK + e) * K, exp_add(x, y));
      }
      for (int e = tid; e < BK * BN; e += NT) {
        Exp<K> x = lds_exp<K>(bs + e * K);
        Exp<K> y = lds_exp<K>(bs + (BK * BN + e) * K);
        sts_exp<K>(bs + (2 * BK * BN + e) * K, exp_add(x, y));
      }
    }
  };

  const int64_t nk = (g.n + BK - 1) / BK;
  if (nk > 0) {
    load_stage(0, 0);
    cp_async_commit();
    if (nk > 1) {
      load_stage(1, BK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if constexpr (MI::SUMS) {
      sums(0);
      __syncthreads();
    }
  }
  for (int64_t kt = 0; kt < nk; kt++) {
    const int st = (int)(kt & 1);
    const double* as = As + st * A_STAGE;
    const double* bs = Bs + st * B_STAGE;
    const int tlen = (int)min((int64_t)BK, g.n - kt * BK);
    // K >= 3: one copy of the slab body (the renorm networks make it ~4.7k /
    // ~10k instructions for TD / QD; unrolled over BK the kernel was 0.6 /
    // 1.3 MB of code and stalled on instruction fetch -- ncu r2:
    // no_instruction was the top stall reason)
#pragma unroll(K == 2 ? BK : 1)
    for (int t = 0; t < BK; t++) {
      if constexpr (K >= 3 && K <= 4 && TM == 1 && TN == 1 && !MI::CHAINED) {
        // TD / QD: ONE copy of exp_mul + exp_add, looped over the NACC chains
        // (operands picked from shared memory by slot, accumulators indexed
        // at run time, i.e. L1-resident local memory): a third / a quarter of
        // the code again, so the slab body stays in the instruction cache
        if (t < tlen) {
#pragma unroll 1
          for (int q = 0; q < NACC; q++) {
            // G3: (re, re) (im, im) (sum, sum); G4: rr, ii, ir, ri; REAL: slot 0
            const int sa = MODE == MODE_G4 ? ((q == 1 || q == 2) ? 1 : 0) : q;
            const int sb = MODE == MODE_G4 ? ((q == 1 || q == 3) ? 1 : 0) : q;
            const Exp<K> a = lds_exp<K>(as + ((sa * BM + ty) * BK + t) * K);
            const Exp<K> b = lds_exp<K>(bs + ((sb * BK + t) * BN + tx) * K);
            acc[0][0][q] = exp_add(acc[0][0][q], exp_mul(a, b));
          }
        }
      } else if (t < tlen) {
        Exp<K> av[NS][TM], bv[NS][TN];
#pragma unroll
        for (int s = 0; s < NS; s++) {
#pragma unroll
          for (int r = 0; r < TM; r++)
            av[s][r] = lds_exp<K>(as + ((s * BM + ty + r * SY) * BK + t) * K);
#pragma unroll
          for (int c = 0; c < TN; c++)
            bv[s][c] = lds_exp<K>(bs + ((s * BK + t) * BN + tx + c * SX) * K);
        }
#pragma unroll
        for (int r = 0; r < TM; r++)
#pragma unroll
          for (int c = 0; c < TN; c++) {
            if constexpr (MODE == MODE_REAL) {
              acc[r][c][0] = exp_add(acc[r][c][0], exp_mul(av[0][r], bv[0][c]));
            } else if constexpr (MODE == MODE_G3) {
#pragma unroll
              for (int q = 0; q < 3; q++)
                acc[r][c][q] = exp_add(acc[r][c][q], exp_mul(av[q][r], bv[q][c]));
            } else if constexpr (MODE == MODE_G4) {
              acc[r][c][0] = exp_add(acc[r][c][0], exp_mul(av[0][r], bv[0][c]));  // rr
              acc[r][c][1] = exp_add(acc[r][c][1], exp_mul(av[1][r], bv[1][c]));  // ii
              acc[r][c][2] = exp_add(acc[r][c][2], exp_mul(av[1][r], bv[0][c]));  // ir
              acc[r][c][3] = exp_add(acc[r][c][3], exp_mul(av[0][r], bv[1][c]));  // ri
            } else if constexpr (MODE == MODE_S3) {
              Cx<K> p = cmul3_pre(av[0][r], av[1][r], av[2][r], bv[0][c], bv[1][c], bv[2][c]);
              acc[r][c][0] = exp_sub(acc[r][c][0], p.re);
              acc[r][c][1] = exp_sub(acc[r][c][1], p.im);
            } else {  // MODE_S4
              Cx<K> p = cmul4(av[0][r], av[1][r], bv[0][c], bv[1][c]);
              acc[r][c][0] = exp_sub(acc[r][c][0], p.re);
              acc[r][c][1] = exp_sub(acc[r][c][1], p.im);
            }
          }
      }
    }
    if (kt + 1 < nk) {
      cp_async_wait<0>();  // this thread's copies of slab kt+1 have landed
      __syncthreads();     // ... everyone's, and everyone is done with slab kt
      sums(st ^ 1);
      if (kt + 2 < nk) {
        load_stage(st, (kt + 2) * BK);  // refill the slab just consumed
        cp_async_commit();
      }
      if constexpr (MI::SUMS) __syncthreads();
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int c = 0; c < TN; c++) {
      int64_t gi = row0 + ty + r * SY, gj = col0 + tx + c * SX;
      if (gi >= g.m || gj >= g.l) continue;
      int64_t off = gi * g.c.ld + gj;
      if constexpr (MODE == MODE_REAL) {
        stexp_<K>(g.c.re + off, g.c.ps, acc[r][c][0]);
      } else if constexpr (MI::CHAINED) {
        stexp_<K>(g.c.re + off, g.c.ps, acc[r][c][0]);
        stexp_<K>(g.c.im + off, g.c.ps, acc[r][c][1]);
      } else {
        Exp<K> re, im;
        if constexpr (MODE == MODE_G3) {  // cmatrix.py:166-168
          re = exp_sub(acc[r][c][0], acc[r][c][1]);
          im = exp_sub(exp_sub(acc[r][c][2], acc[r][c][0]), acc[r][c][1]);
        } else {  // cmatrix.py:153
          re = exp_sub(acc[r][c][0], acc[r][c][1]);
          im = exp_add(acc[r][c][2], acc[r][c][3]);
        }
        if (g.epi == 1) {  // lu.py:158-161: A22 := mat_sub(A22, P)
          re = exp_sub(ldexp_<K>(g.c.re + off, g.c.ps), re);
          im = exp_sub(ldexp_<K>(g.c.im + off, g.c.ps), im);
        }
        stexp_<K>(g.c.re + off, g.c.ps, re);
        stexp_<K>(g.c.im + off, g.c.ps, im);
      }
    }
  if (g.tile_ctr == nullptr) return;
  }  // tile loop
}

// ------------------------------------------------------- elementwise
// mat_add_k, _kernels.py:327-342: C = A + sign*B (sign = +-1)
template <int K>
__global__ void mat_add_kernel(int64_t rows, int64_t cols, View a, View b, View c, double sign) {
  int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    Exp<K> x = ldexp_<K>(a.re + i * a.ld + j, a.ps);
    Exp<K> y = ldexp_<K>(b.re + i * b.ld + j, b.ps);
#pragma unroll
    for (int q = 0; q < K; q++) y.c[q] = dmul(sign, y.c[q]);
    stexp_<K>(c.re + i * c.ld + j, c.ps, exp_add(x, y));
  }
}

// renorm_planes, _kernels.py:485-499 (in place)
template <int K>
__global__ void renorm_planes_kernel(int64_t rows, int64_t cols, View a) {
  int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / cols, j = e % cols;
    double buf[K];
#pragma unroll
    for (int q = 0; q < K; q++) buf[q] = a.re[q * a.ps + i * a.ld + j];
    Exp<K> o = renorm<K, K>(buf, K);
    stexp_<K>(a.re + i * a.ld + j, a.ps, o);
  }
}

// ------------------------------------------------------------ pivoting
// Pivot candidate: (|Re| + |Im|, row), _pivot_row (_kernels.py:568-594).
// Reduction order-independence: the reference keeps the FIRST row whose
// value is strictly greater (sign of the exact expansion difference), i.e.
// the lowest row among the maxima; `better` is that total preorder with
// ties to the lower row, so any reduction tree returns the same row.
template <int K>
struct Cand {
  Exp<K> v;
  int64_t row;  // -1: no nonzero candidate
};

template <int K>
MPC_DI bool cand_better(const Cand<K>& a, const Cand<K>& b) {
  if (a.row < 0) return false;
  if (b.row < 0) return true;
  Exp<K> d = exp_sub(a.v, b.v);
  if (d.c[0] > 0.0) return true;
  if (d.c[0] < 0.0) return false;
  return a.row < b.row;
}

template <int K>
MPC_DI Cand<K> make_cand(const View& A, int64_t i, int64_t j) {
  Exp<K> t = exp_abs(ldexp_<K>(A.re + i * A.ld + j, A.ps));
  Exp<K> u = exp_abs(ldexp_<K>(A.im + i * A.ld + j, A.ps));
  Cand<K> c;
  c.v = exp_add(t, u);
  // the reference only accepts cand when (cand - best)[0] > 0, best starting at 0
  c.row = exp_greater(c.v, exp_zero<K>()) ? i : -1;
  return c;
}

template <int K>
MPC_DI Cand<K> shfl_cand(const Cand<K>& c, int off) {
  Cand<K> o;
#pragma unroll
  for (int q = 0; q < K; q++) o.v.c[q] = __shfl_down_sync(0xffffffffu, c.v.c[q], off);
  o.row = __shfl_down_sync(0xffffffffu, c.row, off);
  return o;
}

// block-wide argmax; result valid in thread 0
template <int K, int NT>
MPC_DI Cand<K> block_reduce_cand(Cand<K> c) {
  __shared__ Exp<K> sv[NT / 32];
  __shared__ int64_t sr[NT / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Cand<K> o = shfl_cand(c, off);
    if (cand_better(o, c)) c = o;
  }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    sv[w] = c.v;
    sr[w] = c.row;
  }
  __syncthreads();
  if (w == 0) {
    if (lane < NT / 32) {
      c.v = sv[lane];
      c.row = sr[lane];
    } else {
      c.row = -1;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Cand<K> o = shfl_cand(c, off);
      if (cand_better(o, c)) c = o;
    }
  }
  return c;
}

struct PanelWs {     // device workspace for the pivot reductions
  double* pv;        // [maxblocks][K]
  int64_t* prow;     // [maxblocks]
  unsigned* counter; // last-block detection
  int64_t* status;   // -1 ok, else first singular column
  unsigned* gbar;    // panel_grid_kernel: [0] barrier arrivals, [1] exits (both 0 between launches)
  unsigned* tile_ctr;  // getrf: tile queue of the capped trailing update
  double* slots;     // panel_grid_kernel: [2][PANEL_GRID_GMAX][PANEL_GRID_SLOT] candidates + pivot rows
};

// Workspace layout (one allocation): a 64-byte header -- status at 0, counter
// at 16, gbar at 24, tile_ctr at 32 -- then prow, pv and the grid-panel slots.
constexpr int PANEL_GRID_GMAX = 256;  // CTAs of one panel_grid_kernel launch
constexpr int PANEL_GRID_SLOT = 40;   // doubles per CTA slot (>= K + 1 + 2 K W)
inline size_t panel_ws_bytes(int k, int64_t n) {
  const int64_t nb = (n + 255) / 256 + 1;
  return 64 + sizeof(int64_t) * nb + sizeof(double) * nb * k +
         sizeof(double) * 2 * PANEL_GRID_GMAX * PANEL_GRID_SLOT;
}
inline PanelWs panel_ws_carve(void* mem, int k, int64_t n) {
  const int64_t nb = (n + 255) / 256 + 1;
  char* b = (char*)mem;
  PanelWs ws;
  ws.status = (int64_t*)b;
  ws.counter = (unsigned*)(b + 16);
  ws.gbar = (unsigned*)(b + 24);
  ws.tile_ctr = (unsigned*)(b + 32);
  ws.prow = (int64_t*)(b + 64);
  ws.pv = (double*)(b + 64 + sizeof(int64_t) * nb);
  ws.slots = ws.pv + nb * k;
  return ws;
}
// status = -1, counters = 0 (stream ordered)
inline cudaError_t panel_ws_init(const PanelWs& ws, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(ws.status, 0xFF, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  return cudaMemsetAsync(ws.counter, 0, 24, st);  // counter, gbar[0..1], tile_ctr
}

constexpr int PNT = 256;  // threads per block of the panel kernels

// Host-side hook of getrf: called (on the enqueueing thread) once the work
// that finalizes rows [r0, r1) of every plane has been enqueued on st --
// row block b is final after step b's trailing-update enqueue (later steps
// only swap and update rows >= its end).  The ABI uses it to overlap the
// device-to-host copy of finished row blocks with the rest of the LU.
struct RowSink {
  void (*fn)(void* ctx, int64_t r0, int64_t r1, cudaStream_t st);
  void* ctx;
};
inline RowSink& row_sink() {
  static thread_local RowSink s{nullptr, nullptr};
  return s;
}
// The input side: getrf calls need(ctx, c1, st) before st first touches
// columns [.., c1) of any row, so the host-to-device copy of later column
// blocks can still be in flight (step 0's trailing update then runs in
// column chunks that each wait only for their own columns).
struct ColSource {
  void (*need)(void* ctx, int64_t c1, cudaStream_t st);
  void* ctx;
  int64_t chunk;  // columns per update chunk at step 0
};
inline ColSource& col_source() {
  static thread_local ColSource s{nullptr, nullptr, 0};
  return s;
}

// Final stage shared by the pivot kernels: the last block to finish reduces
// the per-block partials (in block order), records piv[j] and swaps rows j
// and p inside the active column range [c0, cend) (the other columns are
// swapped later by LASWP, which commutes with the row operations).
template <int K>
MPC_DI void pivot_finish(const View& A, int64_t j, int64_t c0, int64_t cend, int64_t* piv,
                         PanelWs ws, Cand<K> mine) {
  __shared__ bool last;
  __shared__ int64_t prow_s;
  __threadfence();  // every thread's row updates visible before the arrival count
  __syncthreads();
  if (threadIdx.x == 0) {
    stexp_<K>(ws.pv + blockIdx.x * K, 1, mine.v);
    ws.prow[blockIdx.x] = mine.row;
    __threadfence();
    unsigned done = atomicAdd(ws.counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Cand<K> c;
  c.row = -1;
  c.v = exp_zero<K>();
  for (int64_t b = threadIdx.x; b < gridDim.x; b += PNT) {
    Cand<K> o;
#pragma unroll
    for (int q = 0; q < K; q++) o.v.c[q] = __ldcg(ws.pv + b * K + q);
    o.row = __ldcg(ws.prow + b);
    if (cand_better(o, c)) c = o;
  }
  c = block_reduce_cand<K, PNT>(c);
  if (threadIdx.x == 0) {
    prow_s = c.row;
    *ws.counter = 0u;
    if (c.row < 0) {
      if (*ws.status < 0) *ws.status = j;  // lu_panel returns j (_kernels.py:622-624)
    } else {
      piv[j] = c.row;
    }
  }
  __syncthreads();
  int64_t p = prow_s;
  if (p < 0 || p == j) return;
  int64_t w = cend - c0;
  for (int64_t e = threadIdx.x; e < 2 * K * w; e += PNT) {
    int64_t t = c0 + e % w;
    int q = (int)(e / w);
    double* base = (q < K) ? A.re + q * A.ps : A.im + (q - K) * A.ps;
    double x = __ldcg(base + j * A.ld + t);
    double y = __ldcg(base + p * A.ld + t);
    base[j * A.ld + t] = y;
    base[p * A.ld + t] = x;
  }
}

// pivot search for the first column j of a base panel
template <int K>
__global__ void __launch_bounds__(PNT) pivot_first_kernel(View A, int64_t n, int64_t j,
                                                           int64_t c0, int64_t cend,
                                                           int64_t* piv, PanelWs ws) {
  if (*ws.status >= 0) return;
  int64_t i = j + (int64_t)blockIdx.x * PNT + threadIdx.x;
  Cand<K> c;
  c.row = -1;
  c.v = exp_zero<K>();
  if (i < n) c = make_cand<K>(A, i, j);
  c = block_reduce_cand<K, PNT>(c);
  pivot_finish<K>(A, j, c0, cend, piv, ws, c);
}

// Column step j of lu_panel (_kernels.py:627-664) restricted to the base
// panel's columns (j, cend), fused with the pivot search of column j+1.
// One thread per row i > j: l = cdiv(a_ij, a_jj); a_ij = l;
// a_it -= cmul(l, a_jt) for t in (j, cend).
template <int K>
__global__ void __launch_bounds__(PNT) panel_step_kernel(View A, int64_t n, int64_t j,
                                                          int64_t c0, int64_t cend, int use3m,
                                                          int64_t* piv, PanelWs ws) {
  if (*ws.status >= 0) return;
  int64_t i = j + 1 + (int64_t)blockIdx.x * PNT + threadIdx.x;
  Cand<K> c;
  c.row = -1;
  c.v = exp_zero<K>();
  if (i < n) {
    Exp<K> ar = ldexp_<K>(A.re + i * A.ld + j, A.ps);
    Exp<K> ai = ldexp_<K>(A.im + i * A.ld + j, A.ps);
    Exp<K> br = ldexp_<K>(A.re + j * A.ld + j, A.ps);
    Exp<K> bi = ldexp_<K>(A.im + j * A.ld + j, A.ps);
    Cx<K> l = cdiv(ar, ai, br, bi);
    stexp_<K>(A.re + i * A.ld + j, A.ps, l.re);
    stexp_<K>(A.im + i * A.ld + j, A.ps, l.im);
    for (int64_t t = j + 1; t < cend; t++) {
      Exp<K> ur = ldexp_<K>(A.re + j * A.ld + t, A.ps);
      Exp<K> ui = ldexp_<K>(A.im + j * A.ld + t, A.ps);
      Cx<K> p = cmul(use3m != 0, l.re, l.im, ur, ui);
      Exp<K> xr = ldexp_<K>(A.re + i * A.ld + t, A.ps);
      Exp<K> xi = ldexp_<K>(A.im + i * A.ld + t, A.ps);
      stexp_<K>(A.re + i * A.ld + t, A.ps, exp_sub(xr, p.re));
      stexp_<K>(A.im + i * A.ld + t, A.ps, exp_sub(xi, p.im));
    }
    if (j + 1 < cend) c = make_cand<K>(A, i, j + 1);
  }
  if (j + 1 >= cend) return;  // uniform across the grid
  c = block_reduce_cand<K, PNT>(c);
  pivot_finish<K>(A, j + 1, c0, cend, piv, ws, c);
}

// ------------------------------------------------- cluster base panel
// The whole base panel (columns [c0, c0+w), rows [c0, n)) in ONE launch of a
// thread-block cluster: per column, every thread updates its rows (cdiv +
// chained cmul updates, exactly panel_step_kernel's arithmetic), the pivot
// candidates of the next column are reduced warp -> CTA -> cluster (CTA 0
// reads the other CTAs' partials through distributed shared memory), CTA 0
// swaps the two rows inside the panel, and two cluster barriers (release /
// acquire, L1 invalidated) publish the result.  Replaces 1 + w kernel
// launches and their last-block atomics per base panel.
template <int K>
struct PanelCluster {
  // threads per CTA / per row: DD keeps one row per thread with all update
  // columns in registers (2 threads per row measured 15% slower); TD / QD
  // split a row's update columns over 2 threads (register footprint)
  static constexpr int NT = K == 2 ? 256 : 512;
  static constexpr int TPR = K == 2 ? 1 : 2;
  static constexpr int WMAX = K == 2 ? 8 : 4;       // base panel width (registers: k limbs x 4 arrays)
};

template <int K>
MPC_DI void cluster_pick_and_swap(const View& A, int64_t jj, int64_t c0, int64_t cend,
                                  int64_t* piv, int64_t* status, Cand<K> c) {
  namespace cg = cooperative_groups;
  constexpr int NT = PanelCluster<K>::NT;
  __shared__ Exp<K> cta_v;
  __shared__ int64_t cta_r;
  __shared__ int64_t pick;
  cg::cluster_group cluster = cg::this_cluster();
  c = block_reduce_cand<K, NT>(c);
  if (threadIdx.x == 0) {
    cta_v = c.v;
    cta_r = c.row;
  }
  cluster.sync();  // partials visible cluster-wide
  if (cluster.block_rank() == 0) {
    if (threadIdx.x < 32) {
      Cand<K> b;
      b.row = -1;
      b.v = exp_zero<K>();
      if (threadIdx.x < cluster.num_blocks()) {
        Exp<K>* rv = cluster.map_shared_rank(&cta_v, threadIdx.x);
        int64_t* rr = cluster.map_shared_rank(&cta_r, threadIdx.x);
        b.v = *rv;
        b.row = *rr;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        Cand<K> o = shfl_cand(b, off);
        if (cand_better(o, b)) b = o;
      }
      if (threadIdx.x == 0) {
        pick = b.row;
        if (b.row < 0) {
          if (*status < 0) *status = jj;  // lu_panel returns jj (_kernels.py:622-624)
        } else {
          piv[jj] = b.row;
        }
      }
    }
    __syncthreads();
    int64_t p = pick;
    if (p >= 0 && p != jj) {
      int64_t w = cend - c0;
      for (int64_t e = threadIdx.x; e < 2 * K * w; e += NT) {
        int64_t t = c0 + e % w;
        int q = (int)(e / w);
        double* base = (q < K) ? A.re + q * A.ps : A.im + (q - K) * A.ps;
        double x = base[jj * A.ld + t];
        base[jj * A.ld + t] = base[p * A.ld + t];
        base[p * A.ld + t] = x;
      }
    }
    __threadfence();
  }
  cluster.sync();  // swap and status visible
}

template <int K>
__global__ void __launch_bounds__(PanelCluster<K>::NT, 1)
    panel_cluster_kernel(View A, int64_t n, int64_t c0, int64_t w, int use3m, int64_t* piv,
                         int64_t* status) {
  namespace cg = cooperative_groups;
  constexpr int NT = PanelCluster<K>::NT, TPR = PanelCluster<K>::TPR;
  cg::cluster_group cluster = cg::this_cluster();
  // TPR threads share a row: each updates W / TPR of the base panel's
  // columns (smaller register footprint -> more warps to hide the FP64
  // latency chains); the multiplier l = cdiv(a_ij, a_jj) is computed by
  // every thread of the row (identical bits), stored by the first one
  const int64_t T = (int64_t)cluster.num_blocks() * (NT / TPR);
  const int part = (int)(threadIdx.x % TPR);
  const int64_t gt = (int64_t)cluster.block_rank() * (NT / TPR) + threadIdx.x / TPR;
  const int64_t cend = c0 + w;
  if (*(volatile int64_t*)status >= 0) return;  // uniform: written only by earlier launches
  {
    Cand<K> c;
    c.row = -1;
    c.v = exp_zero<K>();
    if (part == 0)
      for (int64_t i = c0 + gt; i < n; i += T) {
        Cand<K> o = make_cand<K>(A, i, c0);
        if (cand_better(o, c)) c = o;
      }
    cluster_pick_and_swap<K>(A, c0, c0, cend, piv, status, c);
  }
  constexpr int W = PanelCluster<K>::WMAX, WP = W / TPR;
  for (int64_t j = c0; j < cend; j++) {
    if (*(volatile int64_t*)status >= 0) return;  // uniform after the barrier
    // the pivot row (a_jj and this thread's a_jt) in registers, one round trip
    const Exp<K> br = ldexp_<K>(A.re + j * A.ld + j, A.ps);
    const Exp<K> bi = ldexp_<K>(A.im + j * A.ld + j, A.ps);
    Exp<K> ur[WP], ui[WP];
#pragma unroll
    for (int q = 0; q < WP; q++) {
      int64_t t = j + 1 + part * WP + q;
      if (t < cend) {
        ur[q] = ldexp_<K>(A.re + j * A.ld + t, A.ps);
        ui[q] = ldexp_<K>(A.im + j * A.ld + t, A.ps);
      }
    }
    Cand<K> c;
    c.row = -1;
    c.v = exp_zero<K>();
    for (int64_t i = j + 1 + gt; i < n; i += T) {
      Exp<K> ar = ldexp_<K>(A.re + i * A.ld + j, A.ps);
      Exp<K> ai = ldexp_<K>(A.im + i * A.ld + j, A.ps);
      Exp<K> xr[WP], xi[WP];
#pragma unroll
      for (int q = 0; q < WP; q++) {
        int64_t t = j + 1 + part * WP + q;
        if (t < cend) {
          xr[q] = ldexp_<K>(A.re + i * A.ld + t, A.ps);
          xi[q] = ldexp_<K>(A.im + i * A.ld + t, A.ps);
        }
      }
      Cx<K> l = cdiv(ar, ai, br, bi);
      if (part == 0) {
        stexp_<K>(A.re + i * A.ld + j, A.ps, l.re);
        stexp_<K>(A.im + i * A.ld + j, A.ps, l.im);
      }
#pragma unroll
      for (int q = 0; q < WP; q++) {
        int64_t t = j + 1 + part * WP + q;
        if (t < cend) {  // independent across q: a_it -= cmul(l, a_jt)
          Cx<K> pr = cmul(use3m != 0, l.re, l.im, ur[q], ui[q]);
          xr[q] = exp_sub(xr[q], pr.re);
          xi[q] = exp_sub(xi[q], pr.im);
          stexp_<K>(A.re + i * A.ld + t, A.ps, xr[q]);
          stexp_<K>(A.im + i * A.ld + t, A.ps, xi[q]);
        }
      }
      if (part == 0 && j + 1 < cend) {  // candidate of the next column from the fresh value
        Cand<K> o;
        o.v = exp_add(exp_abs(xr[0]), exp_abs(xi[0]));
        o.row = exp_greater(o.v, exp_zero<K>()) ? i : -1;
        if (cand_better(o, c)) c = o;
      }
    }
    if (j + 1 < cend) cluster_pick_and_swap<K>(A, j + 1, c0, cend, piv, status, c);
  }
}

// ------------------------------------------------- grid-wide base panel
// The base panel (columns [c0, c0+w), w <= W, rows [c0, n)) in ONE cooperative
// launch with one row per thread and the row's w columns resident in
// registers for the whole launch -- the cluster kernel above gives every
// thread ceil(rows / 4096) rows per column and re-reads them from memory.
//
// Row interchanges are virtual: every thread carries the current position
// `pos` of its row (_swap_rows, _kernels.py:597-608, exchanges positions jj
// and p -- here the two owning threads exchange their `pos`), the thread whose
// row becomes the pivot row retires, and the rows are written to their final
// positions at the end.  The candidate order (|Re| + |Im|, ties to the lower
// CURRENT position) is the reference's.
//
// Per column ONE grid barrier: every CTA reduces its candidates, the owning
// thread publishes (value, position, the row's values) to the CTA's slot and
// arrives; after the barrier warp 0 of every CTA reduces the slots -- the
// comparator is a total preorder, so every CTA picks the same row -- and
// stages the pivot row in shared memory.  Only l = cdiv(a, pivot) and the
// update of the NEXT column sit on the critical path: the updates of the
// remaining columns run after the next arrival, under the barrier latency.
// Element operation sequences are those of panel_step_kernel.
template <int K>
struct PanelGrid {
  static constexpr int NT = 256;
  static constexpr int W = K == 2 ? 8 : 4;
  static_assert(K + 1 + 2 * K * W <= PANEL_GRID_SLOT, "slot too small");
};

// Poll of the grid-barrier word.  Relaxed (L2) loads, NOT ld.acquire: an
// acquire load invalidates the SM's L1 on every poll (CCTL.IVALL, ~40 polls
// per barrier in the ncu capture), and the rows live in L1-resident local
// memory.  Everything read after the barrier is read with ld.cg (L2), after
// the writers' __threadfence() + arrival, so no L1 line can be stale.
MPC_DI unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// cand_better on (value, position) pairs.  DD: candidates are dd_add outputs,
// i.e. normalized (hi = fl(hi + lo)), whose representation is unique, so
// different leading limbs already order the exact values; equal leading
// limbs (and k >= 3) take the reference's exact test.
template <int K>
MPC_DI bool cand_better_f(const Exp<K>& av, int64_t ar, const Exp<K>& bv, int64_t br) {
  if (ar < 0) return false;
  if (br < 0) return true;
  if constexpr (K == 2) {
    if (av.c[0] != bv.c[0]) return av.c[0] > bv.c[0];
  }
  Exp<K> d = exp_sub(av, bv);
  if (d.c[0] > 0.0) return true;
  if (d.c[0] < 0.0) return false;
  return ar < br;
}

// TPR = 2: two adjacent lanes share a row (same values, same operations)
// and split l = cdiv(a, pivot) -- the longest dependent chain of a column
// step -- between them: lane 0 forms Re l = (ar br + ai bi) / d, lane 1
// Im l = (ai br - ar bi) / d (cdiv_core, _kernels.py:549-561; exp_sub(x, y) is
// exp_add(x, -y), so both lanes run one instruction stream), exchanged by
// shuffle.  Only lane 0 of a row competes for the pivot and stores.
template <int K, int TPR>
__global__ void __launch_bounds__(PanelGrid<K>::NT, 1)
    panel_grid_kernel(View A, int64_t n, int64_t c0, int w, int use3m, int64_t* piv,
                      int64_t* status, unsigned* gbar, double* slots) {
  using PG = PanelGrid<K>;
  constexpr int NT = PG::NT, W = PG::W, NW = NT / 32, SLOT = PANEL_GRID_SLOT;
  constexpr int ROWS = NT / TPR;
  __shared__ double ubuf[2][2 * K * W];  // pivot row: [Re limbs][W], [Im limbs][W]
  __shared__ int64_t pick_s[2];
  __shared__ double red_v[NW][K];
  __shared__ int64_t red_r[NW];
  __shared__ int red_t[NW];
  __shared__ double win_v[K];
  __shared__ int64_t win_r;
  __shared__ int win_tid;

  if (*(volatile int64_t*)status >= 0) return;  // uniform: written only by earlier launches
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned G = gridDim.x;
  const int sub = tid % TPR;  // lane within the row's group
  const int64_t home = c0 + (int64_t)blockIdx.x * ROWS + tid / TPR;
  const bool valid = home < n;
  int64_t pos = home;
  bool active = valid;
  Exp<K> xr[W], xi[W];
#pragma unroll
  for (int i = 0; i < W; i++) {
    if (valid && i < w) {
      xr[i] = ldexp_<K>(A.re + home * A.ld + c0 + i, A.ps);
      xi[i] = ldexp_<K>(A.im + home * A.ld + c0 + i, A.ps);
    } else {
      xr[i] = exp_zero<K>();
      xi[i] = exp_zero<K>();
    }
  }
  unsigned epoch = 0;
  for (int q = 0; q < w; q++) {
    const int par = q & 1;
    const int64_t jj = c0 + q;
    // 1. this row's candidate for column q
    Exp<K> cv = exp_zero<K>();
    int64_t crow = -1;
    int ctid = tid;
    if (active && sub == 0) {
      Exp<K> ar = exp_zero<K>(), ai = exp_zero<K>();
#pragma unroll
      for (int i = 0; i < W; i++)
        if (i == q) {
          ar = xr[i];
          ai = xi[i];
        }
      cv = exp_add(exp_abs(ar), exp_abs(ai));
      crow = exp_greater(cv, exp_zero<K>()) ? pos : -1;
    }
    // 2. CTA argmax, carrying the owning thread
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Exp<K> ov;
#pragma unroll
      for (int c = 0; c < K; c++) ov.c[c] = __shfl_down_sync(0xffffffffu, cv.c[c], off);
      const int64_t orow = __shfl_down_sync(0xffffffffu, crow, off);
      const int otid = __shfl_down_sync(0xffffffffu, ctid, off);
      if (cand_better_f<K>(ov, orow, cv, crow)) {
        cv = ov;
        crow = orow;
        ctid = otid;
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < K; c++) red_v[wid][c] = cv.c[c];
      red_r[wid] = crow;
      red_t[wid] = ctid;
    }
    __syncthreads();
    if (wid == 0) {
      if (lane < NW) {
#pragma unroll
        for (int c = 0; c < K; c++) cv.c[c] = red_v[lane][c];
        crow = red_r[lane];
        ctid = red_t[lane];
      } else {
        crow = -1;
      }
#pragma unroll
      for (int off = NW / 2; off > 0; off >>= 1) {
        Exp<K> ov;
#pragma unroll
        for (int c = 0; c < K; c++) ov.c[c] = __shfl_down_sync(0xffffffffu, cv.c[c], off);
        const int64_t orow = __shfl_down_sync(0xffffffffu, crow, off);
        const int otid = __shfl_down_sync(0xffffffffu, ctid, off);
        if (cand_better_f<K>(ov, orow, cv, crow)) {
          cv = ov;
          crow = orow;
          ctid = otid;
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < K; c++) win_v[c] = cv.c[c];
        win_r = crow;
        win_tid = crow >= 0 ? ctid : 0;
      }
    }
    __syncthreads();
    // the previous column's deferred updates (columns > q): l = x[q-1], u =
    // the previous pivot row.  The CTA's candidate row runs them before it is
    // published (its values become U's row), every other row under the barrier
    auto deferred = [&]() {
      Exp<K> lr = exp_zero<K>(), li = exp_zero<K>();
#pragma unroll
      for (int i = 0; i < W; i++)
        if (i == q - 1) {
          lr = xr[i];
          li = xi[i];
        }
      const double* ub = &ubuf[par ^ 1][0];
#pragma unroll
      for (int i = 2; i < W; i++)
        if (i > q && i < w) {
          Exp<K> ur, ui;
#pragma unroll
          for (int c = 0; c < K; c++) {
            ur.c[c] = ub[c * W + i];
            ui.c[c] = ub[(K + c) * W + i];
          }
          Cx<K> pr = cmul(use3m != 0, lr, li, ur, ui);
          xr[i] = exp_sub(xr[i], pr.re);
          xi[i] = exp_sub(xi[i], pr.im);
        }
    };
    const bool is_pub = tid == win_tid;
    if (is_pub) {  // publish the CTA's candidate and its row, then arrive
      if (q > 0 && active) deferred();
      double* sl = slots + ((size_t)par * PANEL_GRID_GMAX + blockIdx.x) * SLOT;
      const int64_t wr = win_r;
      if (G > 1) {
#pragma unroll
        for (int c = 0; c < K; c++) sl[c] = win_v[c];
        sl[K] = __longlong_as_double(wr);
      }
      if (wr >= 0) {
        double* dst = G > 1 ? sl + K + 1 : &ubuf[par][0];
#pragma unroll
        for (int i = 0; i < W; i++)
#pragma unroll
          for (int c = 0; c < K; c++) {
            dst[c * W + i] = xr[i].c[c];
            dst[(K + c) * W + i] = xi[i].c[c];
          }
      }
      if (G > 1) {
        __threadfence();
        atomicAdd(&gbar[0], 1u);
      } else {
        pick_s[par] = wr;
      }
    }
    // 3. the other rows' deferred updates, under the barrier
    if (q > 0 && active && !is_pub) deferred();
    // 4. every CTA's candidate is published
    if (G > 1) {
      epoch++;
      if (tid == 0)
        while (ld_relaxed_u32(&gbar[0]) < epoch * G) {
        }
      __syncthreads();
      // 5. warp 0: the global argmax (same result in every CTA), pivot row to smem
      if (wid == 0) {
        Exp<K> bv = exp_zero<K>();
        int64_t brow = -1;
        unsigned bb = 0;
        for (unsigned b = lane; b < G; b += 32) {
          const double* sl = slots + ((size_t)par * PANEL_GRID_GMAX + b) * SLOT;
          Exp<K> ov;
#pragma unroll
          for (int c = 0; c < K; c++) ov.c[c] = __ldcg(sl + c);
          const int64_t orow = __double_as_longlong(__ldcg(sl + K));
          if (cand_better_f<K>(ov, orow, bv, brow)) {
            bv = ov;
            brow = orow;
            bb = b;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          Exp<K> ov;
#pragma unroll
          for (int c = 0; c < K; c++) ov.c[c] = __shfl_down_sync(0xffffffffu, bv.c[c], off);
          const int64_t orow = __shfl_down_sync(0xffffffffu, brow, off);
          const unsigned ob = __shfl_down_sync(0xffffffffu, bb, off);
          if (cand_better_f<K>(ov, orow, bv, brow)) {
            bv = ov;
            brow = orow;
            bb = ob;
          }
        }
        brow = __shfl_sync(0xffffffffu, brow, 0);
        bb = __shfl_sync(0xffffffffu, bb, 0);
        if (brow >= 0) {
          const double* sl = slots + ((size_t)par * PANEL_GRID_GMAX + bb) * SLOT + K + 1;
          for (int e = lane; e < 2 * K * W; e += 32) ubuf[par][e] = __ldcg(sl + e);
        }
        if (lane == 0) pick_s[par] = brow;
      }
    }
    __syncthreads();
    const int64_t P = pick_s[par];
    if (P < 0) {  // lu_panel returns jj (_kernels.py:622-624); uniform across the grid
      if (blockIdx.x == 0 && tid == 0 && *status < 0) *status = jj;
      break;
    }
    if (blockIdx.x == 0 && tid == 0) piv[jj] = P;
    if (active) {
      if (pos == P) {
        pos = jj;
        active = false;  // this row is U's row jj now
      } else if (pos == jj) {
        pos = P;
      }
    }
    Cx<K> l;
    if constexpr (TPR == 2) {
      Exp<K> quo = exp_zero<K>();
      if (active) {
        Exp<K> ar = exp_zero<K>(), ai = exp_zero<K>(), br, bi;
#pragma unroll
        for (int i = 0; i < W; i++)
          if (i == q) {
            ar = xr[i];
            ai = xi[i];
          }
        const double* ub = &ubuf[par][0];
#pragma unroll
        for (int c = 0; c < K; c++) {
          br.c[c] = ub[c * W + q];
          bi.c[c] = ub[(K + c) * W + q];
        }
        const Exp<K> d = exp_add(exp_mul(br, br), exp_mul(bi, bi));
        const Exp<K> t1 = exp_mul(sub ? ai : ar, br);
        Exp<K> t2 = exp_mul(sub ? ar : ai, bi);
        if (sub) t2 = exp_neg(t2);
        quo = exp_div(exp_add(t1, t2), d);
      }
      Exp<K> oth;  // the partner lane's quotient (every lane takes part)
#pragma unroll
      for (int c = 0; c < K; c++) oth.c[c] = __shfl_xor_sync(0xffffffffu, quo.c[c], 1);
      l.re = sub ? oth : quo;
      l.im = sub ? quo : oth;
    }
    if (active) {
      const double* ub = &ubuf[par][0];
      if constexpr (TPR == 1) {
        Exp<K> ar = exp_zero<K>(), ai = exp_zero<K>(), br, bi;
#pragma unroll
        for (int i = 0; i < W; i++)
          if (i == q) {
            ar = xr[i];
            ai = xi[i];
          }
#pragma unroll
        for (int c = 0; c < K; c++) {
          br.c[c] = ub[c * W + q];
          bi.c[c] = ub[(K + c) * W + q];
        }
        l = cdiv(ar, ai, br, bi);
      }
#pragma unroll
      for (int i = 0; i < W; i++)
        if (i == q) {
          xr[i] = l.re;
          xi[i] = l.im;
        }
      if (q + 1 < w) {  // the next column first: its candidates gate the next barrier
        Exp<K> ur, ui;
#pragma unroll
        for (int c = 0; c < K; c++) {
          ur.c[c] = ub[c * W + q + 1];
          ui.c[c] = ub[(K + c) * W + q + 1];
        }
        Cx<K> pr = cmul(use3m != 0, l.re, l.im, ur, ui);
#pragma unroll
        for (int i = 1; i < W; i++)
          if (i == q + 1) {
            xr[i] = exp_sub(xr[i], pr.re);
            xi[i] = exp_sub(xi[i], pr.im);
          }
      }
    }
  }
  // rows to their final positions (every CTA loaded its rows before its first
  // arrival, so no row is overwritten before its owner has read it)
  if (valid && sub == 0) {
#pragma unroll
    for (int i = 0; i < W; i++)
      if (i < w) {
        stexp_<K>(A.re + pos * A.ld + c0 + i, A.ps, xr[i]);
        stexp_<K>(A.im + pos * A.ld + c0 + i, A.ps, xi[i]);
      }
  }
  if (G > 1 && tid == 0) {  // the last CTA out re-arms the barrier words
    __threadfence();
    if (atomicAdd(&gbar[1], 1u) == G - 1) {
      gbar[0] = 0u;
      gbar[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------- LASWP
// Apply the interchanges piv[r0..r1) in order to columns [col0, col0+ncols)
// of every limb plane (the deferred part of _swap_rows, _kernels.py:597-608).
//
// One thread per (limb plane, column).  The interchanges are applied in
// chunks of LASWP_HC: a chunk touches at most 2 HC rows -- its own rows
// [rc, rc+hc) and the pivot rows below them -- and the chunk's net row
// permutation is composed once per CTA on positions (thread 0, shared
// memory: position j < HC is row rc+j, position HC+i the pivot row of
// interchange i where it first occurs), so every thread then moves its
// column's values with independent loads followed by independent stores --
// one memory round trip per chunk instead of one per interchange (the serial
// loop was latency-bound: ~0.6 us per interchange, 150 us for a 256-row
// block; ncu r2).
constexpr int LASWP_HC = 32;
constexpr int LASWP_NT = 128;
template <int K>
__global__ void __launch_bounds__(LASWP_NT)
    laswp_kernel(View A, int64_t col0, int64_t ncols, const int64_t* piv, int64_t r0, int64_t r1,
                 const int64_t* status) {
  constexpr int HC = LASWP_HC, NT = LASWP_NT;
  __shared__ int64_t pv[HC];
  __shared__ int first[HC];
  __shared__ int src[2 * HC];
  const int tid = threadIdx.x;
  const int64_t cidx = (int64_t)blockIdx.x * NT + tid;
  const bool live = cidx < ncols;
  const int q = blockIdx.y;
  double* base = ((q < K) ? A.re + q * A.ps : A.im + (q - K) * A.ps) + col0 + cidx;
  int64_t rend = r1;
  if (status != nullptr && *status >= 0 && *status < rend) rend = *status;
  for (int64_t rc = r0; rc < rend; rc += HC) {
    const int hc = (int)min((int64_t)HC, rend - rc);
    __syncthreads();  // the previous chunk's tables are no longer read
    if (tid < hc) pv[tid] = piv[rc + tid];
    if (tid < 2 * HC) src[tid] = tid;
    __syncthreads();
    if (tid < hc) {
      int f = tid;
      for (int i = tid - 1; i >= 0; i--)
        if (pv[i] == pv[tid]) f = i;
      first[tid] = f;
    }
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < hc; j++) {
        const int64_t p = pv[j];
        if (p == rc + j) continue;
        const int b2 = p < rc + hc ? (int)(p - rc) : HC + first[j];
        const int t = src[j];
        src[j] = src[b2];
        src[b2] = t;
      }
    }
    __syncthreads();
    if (live) {
      // position -> row: i < HC: rc + i; else the pivot row of interchange i - HC
      double val[2 * HC];  // registers: both loops are fully unrolled
#pragma unroll
      for (int i = 0; i < 2 * HC; i++) {
        const int sidx = src[i];
        if (sidx != i) {
          const int64_t row = sidx < HC ? rc + sidx : pv[sidx - HC];
          val[i] = base[row * A.ld];
        }
      }
#pragma unroll
      for (int i = 0; i < 2 * HC; i++) {
        if (src[i] != i) {
          const int64_t row = i < HC ? rc + i : pv[i - HC];
          base[row * A.ld] = val[i];
        }
      }
    }
  }
}

// -------------------------------------------------------------- TRSM
// Diagonal block of trsm_ll_unit (_kernels.py:687-705), right-looking and
// lane-parallel: a group of 16 lanes owns one column, lane r holds x_r.  At
// step s lane s's value is final (all its subtractions s' < s are done); it
// is broadcast by shuffle and every lane r > s applies x_r -= cmul(L_rs, x_s).
// Each x_r therefore receives exactly the reference's chain (s ascending).
// TB = rows of the diagonal block = lanes per column (16 or 32).
template <int K, int TB>
MPC_DI Exp<K> shfl_exp(const Exp<K>& v, int src) {
  Exp<K> o;
#pragma unroll
  for (int q = 0; q < K; q++) o.c[q] = __shfl_sync(0xffffffffu, v.c[q], src, TB);
  return o;
}

template <int K, int TB>
__global__ void trsm_diag_kernel(View L, View X, int64_t kb, int64_t M, int use3m,
                                 const int64_t* status) {
  if (status != nullptr && *status >= 0) return;
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int r = (int)(gid % TB);
  int64_t col = gid / TB;
  bool live = col < M && r < kb;  // whole TB-lane groups share a column
  Exp<K> xr = exp_zero<K>(), xi = exp_zero<K>();
  if (live) {
    xr = ldexp_<K>(X.re + r * X.ld + col, X.ps);
    xi = ldexp_<K>(X.im + r * X.ld + col, X.ps);
  }
  for (int s = 0; s + 1 < (int)kb; s++) {
    Exp<K> yr = shfl_exp<K, TB>(xr, s);
    Exp<K> yi = shfl_exp<K, TB>(xi, s);
    if (live && r > s) {
      Exp<K> lr = ldexp_<K>(L.re + r * L.ld + s, L.ps);
      Exp<K> li = ldexp_<K>(L.im + r * L.ld + s, L.ps);
      Cx<K> p = cmul(use3m != 0, lr, li, yr, yi);
      xr = exp_sub(xr, p.re);
      xi = exp_sub(xi, p.im);
    }
  }
  if (live && r > 0) {
    stexp_<K>(X.re + r * X.ld + col, X.ps, xr);
    stexp_<K>(X.im + r * X.ld + col, X.ps, xi);
  }
}

// -------------------------------------------------------------- solve
// solve_fb (_kernels.py:708-775) as a blocked triangular solve with
// KB-row diagonal blocks, one launch per block and direction.
//
// Interchanges: the reference swaps b_i <-> b_{piv[i]} for i ascending
// (_kernels.py:711-721).  The same swaps applied to an index vector (one
// thread, shared memory) give idx with b_new[i] = b_old[idx[i]]; a parallel
// gather then permutes all 2k limb planes at once.
template <int K>
__global__ void perm_compose_kernel(const int64_t* __restrict__ piv, int64_t n,
                                    int64_t* __restrict__ idx, int use_smem) {
  extern __shared__ int sidx[];
  if (use_smem) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sidx[i] = (int)i;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int64_t i = 0; i < n; i++) {
        int64_t p = __ldg(piv + i);
        if (p != i) {
          int x = sidx[i];
          sidx[i] = sidx[p];
          sidx[p] = x;
        }
      }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) idx[i] = sidx[i];
  } else {  // n beyond shared memory: the same sequence on the global vector
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) idx[i] = i;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int64_t i = 0; i < n; i++) {
        int64_t p = __ldg(piv + i);
        if (p != i) {
          int64_t x = idx[i];
          idx[i] = idx[p];
          idx[p] = x;
        }
      }
  }
}

// y[q][i] = b_q[idx[i]] for the 2k limb planes (q < k: Re, else Im)
template <int K>
__global__ void perm_gather_kernel(const double* br, const double* bi, const int64_t* idx,
                                   int64_t n, double* y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 2 * K * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int q = (int)(e / n);
    int64_t i = e - (int64_t)q * n;
    int64_t s = idx[i];
    y[e] = q < K ? br[q * n + s] : bi[(q - K) * n + s];
  }
}

template <int K>
struct SolveCfg {
  static constexpr int KB = 32;                // diagonal block = one warp
  static constexpr int RT = K == 2 ? 128 : 64;  // off-diagonal rows per CTA (one per thread)
  static constexpr int LDS = KB + 1;            // padded row: conflict-free 8-byte reads
  static constexpr size_t SMEM = sizeof(double) * 2 * K * (size_t)(KB + RT) * LDS;
};

// One diagonal block [r0, r0+kb) of the forward (FWD: unit lower, reference
// order) or backward (upper, cdiv by U_ii) substitution, plus the
// off-diagonal update of RT rows per CTA (FWD: rows >= r0+kb, else rows
// < r0).  Working values live in (wr, wi) -- (2k, n)-shaped planar vectors
// (limb c of entry i at c*n + i) -- and the block's final values go to
// (fr, fi), so no CTA overwrites what another still reads.
//   * diagonal block (every CTA, redundantly, in warp 0): lane r holds x_r;
//     FWD: for s ascending, x_s is final, broadcast by shuffle, lanes r > s
//     apply x_r -= cmul(L_rs, x_s) -- exactly the reference's chain order
//     (j ascending); BWD: for s descending, lane s scales by the precomputed
//     reciprocal z_s = cdiv(1, U_ss) (the reference divides, cdiv(x_s, U_ss):
//     one cdiv per row would sit on the sequential critical path, n deep),
//     then lanes r < s apply x_r -= cmul(U_rs, x_s).
//   * off-diagonal rows: one thread per row, x_i -= cmul(F_ij, x_j) for j
//     ascending over the block, F tile staged coalesced in shared memory.
// Forward chains therefore equal the reference's (blocks ascending, j
// ascending within each): bitwise.  Backward applies blocks in descending
// order -- the reference's row chain (j ascending up to n) is inherently
// sequential (n^2/2 dependent steps) -- and multiplies by reciprocals, so it
// is tolerance-parity.
//
// diag_inv_kernel: z_i = cdiv(1, U_ii) for every row (cdiv_core,
// _kernels.py:549-561), one thread per row.
template <int K>
__global__ void diag_inv_kernel(View F, int64_t n, double* inv, int use3m) {
  (void)use3m;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Exp<K> one = exp_zero<K>(), zero = exp_zero<K>();
  one.c[0] = 1.0;
  Exp<K> ur = ldexp_<K>(F.re + i * F.ld + i, F.ps), ui = ldexp_<K>(F.im + i * F.ld + i, F.ps);
  Cx<K> z = cdiv(one, zero, ur, ui);
  stexp_<K>(inv + i, n, z.re);
  stexp_<K>(inv + K * n + i, n, z.im);
}
template <int K, bool FWD>
__global__ void __launch_bounds__(SolveCfg<K>::RT)
    trsv_block_kernel(View F, double* wr, double* wi, double* fr, double* fi, int64_t n,
                      int64_t r0, int64_t kb, int use3m, const double* __restrict__ inv) {
  using C = SolveCfg<K>;
  constexpr int KB = C::KB, RT = C::RT, LDS = C::LDS;
  extern __shared__ double sm[];
  double* Ld = sm;                      // [2k][KB][LDS] diagonal block
  double* Lt = sm + 2 * K * KB * LDS;   // [2k][RT][LDS] off-diagonal rows
  __shared__ double xs[2 * K][KB];      // the block's final x
  __shared__ double xsum[K][KB];        // Re + Im of x (3M operand sums)
  const int t = threadIdx.x;
  const int64_t row0 = FWD ? r0 + kb + (int64_t)blockIdx.x * RT : (int64_t)blockIdx.x * RT;
  const int64_t rowEnd = FWD ? n : r0;
  // staging with cp.async (no register round trip, every load in flight at
  // once), lane = column of the 32-wide block: group 0 = the diagonal block,
  // group 1 = the off-diagonal rows, which keep landing while warp 0 solves
  // the diagonal block
  {
    const int lane = t & 31, wid = t >> 5;
    constexpr int NW = RT / 32;
    const bool colok = lane < kb;
#pragma unroll
    for (int q = 0; q < 2 * K; q++) {
      const double* base = (q < K ? F.re + q * F.ps : F.im + (q - K) * F.ps) + r0 + lane;
      for (int rr = wid; rr < KB; rr += NW) {
        const bool ok = colok && rr < kb;
        cp_async8(&Ld[(q * KB + rr) * LDS + lane], ok ? base + (r0 + rr) * F.ld : base, ok);
      }
    }
    cp_async_commit();
#pragma unroll
    for (int q = 0; q < 2 * K; q++) {
      const double* base = (q < K ? F.re + q * F.ps : F.im + (q - K) * F.ps) + r0 + lane;
      for (int rr = wid; rr < RT; rr += NW) {
        const bool ok = colok && row0 + rr < rowEnd;
        cp_async8(&Lt[(q * RT + rr) * LDS + lane], ok ? base + (row0 + rr) * F.ld : base, ok);
      }
    }
    cp_async_commit();
  }
  cp_async_wait<1>();
  __syncthreads();
  if (t < 32) {
    const int r = t;
    const bool live = r < kb;
    Exp<K> xr = exp_zero<K>(), xi = exp_zero<K>();
    if (live) {
      xr = ldexp_<K>(wr + r0 + r, n);
      xi = ldexp_<K>(wi + r0 + r, n);
    }
    auto ld_d = [&](int rr, int jj, Exp<K>& lr, Exp<K>& li) {
#pragma unroll
      for (int c = 0; c < K; c++) {
        lr.c[c] = Ld[(c * KB + rr) * LDS + jj];
        li.c[c] = Ld[((K + c) * KB + rr) * LDS + jj];
      }
    };
    if constexpr (FWD) {
      for (int s = 0; s + 1 < (int)kb; s++) {
        Exp<K> yr, yi;
#pragma unroll
        for (int c = 0; c < K; c++) {
          yr.c[c] = __shfl_sync(0xffffffffu, xr.c[c], s);
          yi.c[c] = __shfl_sync(0xffffffffu, xi.c[c], s);
        }
        if (live && r > s) {
          Exp<K> lr, li;
          ld_d(r, s, lr, li);
          Cx<K> p = cmul(use3m != 0, lr, li, yr, yi);
          xr = exp_sub(xr, p.re);
          xi = exp_sub(xi, p.im);
        }
      }
    } else {
      // z_r = 1 / U_rr (cdiv, precomputed for every row by diag_inv_kernel,
      // off the critical path): x_s = cmul(x_s, z_s) at step s
      Exp<K> zr = exp_zero<K>(), zi = exp_zero<K>();
      if (live) {
        zr = ldexp_<K>(inv + r0 + r, n);
        zi = ldexp_<K>(inv + K * n + r0 + r, n);
      }
      for (int s = (int)kb - 1; s >= 0; s--) {
        if (r == s) {
          Cx<K> q = cmul(use3m != 0, xr, xi, zr, zi);
          xr = q.re;
          xi = q.im;
        }
        Exp<K> yr, yi;
#pragma unroll
        for (int c = 0; c < K; c++) {
          yr.c[c] = __shfl_sync(0xffffffffu, xr.c[c], s);
          yi.c[c] = __shfl_sync(0xffffffffu, xi.c[c], s);
        }
        if (r < s) {
          Exp<K> lr, li;
          ld_d(r, s, lr, li);
          Cx<K> p = cmul(use3m != 0, lr, li, yr, yi);
          xr = exp_sub(xr, p.re);
          xi = exp_sub(xi, p.im);
        }
      }
    }
    if (live) {
      Exp<K> sx = exp_add(xr, xi);  // cmul_3m_core's b-operand sum (_kernels.py:534)
#pragma unroll
      for (int c = 0; c < K; c++) {
        xs[c][r] = xr.c[c];
        xs[K + c][r] = xi.c[c];
        xsum[c][r] = sx.c[c];
      }
      if (blockIdx.x == 0) {
        stexp_<K>(fr + r0 + r, n, xr);
        stexp_<K>(fi + r0 + r, n, xi);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  const int64_t i = row0 + t;
  if (i >= rowEnd) return;
  Exp<K> xr = ldexp_<K>(wr + i, n), xi = ldexp_<K>(wi + i, n);
  // x_i -= cmul(F_ij, x_j), j ascending; the products do not depend on x_i,
  // so unrolling lets the next products overlap the subtraction chain
#pragma unroll 4
  for (int j = 0; j < (int)kb; j++) {
    Exp<K> lr, li, yr, yi, sy;
#pragma unroll
    for (int c = 0; c < K; c++) {
      lr.c[c] = Lt[(c * RT + t) * LDS + j];
      li.c[c] = Lt[((K + c) * RT + t) * LDS + j];
      yr.c[c] = xs[c][j];
      yi.c[c] = xs[K + c][j];
      sy.c[c] = xsum[c][j];
    }
    Cx<K> p = use3m ? cmul3_pre(lr, li, exp_add(lr, li), yr, yi, sy) : cmul4(lr, li, yr, yi);
    xr = exp_sub(xr, p.re);
    xi = exp_sub(xi, p.im);
  }
  stexp_<K>(wr + i, n, xr);
  stexp_<K>(wi + i, n, xi);
}

// ===================================================== host-side launchers
// Algorithmic FP64 operation model v1: DADD,
// DSUB, DMUL, DFMA each count 1.  The k >= 3 figures count VecSum +
// extraction of every renorm and exclude sorting / repeat passes.
template <int K>
struct OpModel {
  // (k >= 5: the verification kernels, not part of the op model)
  static constexpr double real_mac = K == 2 ? 31.0 : (K == 3 ? 195.0 : (K == 4 ? 325.0 : 0.0));
  // panel / TRSM element update a -= cmul(l, u): cmul + 2 subtractions
  static constexpr double upd3 = K == 2 ? 173.0 : (K == 3 ? 833.0 : 1323.0);
  static constexpr double upd4 = K == 2 ? 124.0 : (K == 3 ? 780.0 : 1300.0);
  static double upd(bool use3m) { return use3m ? upd3 : upd4; }
  // the chained "S" update kernel forms the two 3M operand sums once per
  // STAGED element (cmul3_pre), not once per output element: 3 products + 5
  // additions per update are what the FP64 pipe executes (charging
  // 173 overstated the S-class rate by ~30%)
  static constexpr double upd3_exec = K == 2 ? 133.0 : (K == 3 ? 709.0 : 1149.0);
};

struct LaunchError {
  const char* what;
};

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw LaunchError{what};
}

// Stream-ordered temporaries (cudaMallocAsync) come from the device's default
// pool; keep freed blocks in the pool instead of returning them to the OS at
// every synchronisation, so per-call workspaces cost no page mapping.
inline void retain_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// The grid-wide base panel needs all its CTAs resident at once (it spins on
// a grid barrier).  A cooperative launch guarantees that, but the hardware
// runs a cooperative grid only once it can place ALL its CTAs, which beside a
// trailing-update kernel means draining that kernel's CTAs first (measured:
// with persistent GEMM CTAs resident the panel did not start until the GEMM
// had finished).  A plain launch places CTAs as slots free up and cannot
// deadlock as long as the grids that spin fit the device together: a grid is
// at most PANEL_GRID_GMAX CTAs of <= 20k registers (3 per SM, 444 slots on
// 148 SMs), everything else on the device (GEMM tiles, S updates) retires on
// its own.  So ONE factorization per device at a time -- the first to claim
// the device's slot -- uses plain launches; any other concurrent caller keeps
// the cooperative launch.  The slot is released by a host callback once the
// claiming call's stream work has drained.
inline std::atomic<int>& panel_slot(int dev) {
  static std::atomic<int> slots[64];
  return slots[dev & 63];
}
inline bool& panel_plain_launch_ok() {
  static thread_local bool ok = false;
  return ok;
}
inline void CUDART_CB panel_slot_release(void* p) {
  static_cast<std::atomic<int>*>(p)->fetch_sub(1);
}

// The lookahead schedule's high-priority side stream and its two events,
// released on every exit path (a failed launch throws LaunchError mid-loop).
struct SideStream {
  cudaStream_t main = nullptr;  // set by the driver (set_main): the stream whose drain releases the slot
  bool has_main = false;        // (the legacy default stream is a null handle)
  void set_main(cudaStream_t s) {
    main = s;
    has_main = true;
  }
  std::atomic<int>* slot = nullptr;
  cudaStream_t sp = nullptr;
  cudaStream_t sh = nullptr;  // helper launches of the capped trailing update
  cudaEvent_t ev_narrow = nullptr, ev_panel = nullptr, ev_queue = nullptr, ev_helper = nullptr;
  SideStream() {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&sp, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_narrow, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_queue, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_helper, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming) != cudaSuccess) {
      release();
      throw LaunchError{"side stream / event creation"};
    }
    static const bool plain = [] {
      const char* e = getenv("MPC_PANEL_COOP");
      return !(e && e[0] == '1');
    }();
    int dev = 0;
    cudaGetDevice(&dev);
    if (plain) {
      slot = &panel_slot(dev);
      if (slot->fetch_add(1) == 0) {
        panel_plain_launch_ok() = true;
      } else {
        slot->fetch_sub(1);
        slot = nullptr;
      }
    }
  }
  ~SideStream() {
    if (slot != nullptr) {
      panel_plain_launch_ok() = false;
      // after everything this call enqueued (the last panel joins `main`)
      if (!has_main || cudaLaunchHostFunc(main, panel_slot_release, slot) != cudaSuccess) {
        cudaGetLastError();
        cudaDeviceSynchronize();
        slot->fetch_sub(1);
      }
    }
    release();
  }
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
  void release() {
    if (ev_panel) cudaEventDestroy(ev_panel);
    if (ev_narrow) cudaEventDestroy(ev_narrow);
    if (ev_queue) cudaEventDestroy(ev_queue);
    if (ev_helper) cudaEventDestroy(ev_helper);
    if (sp) cudaStreamDestroy(sp);
    if (sh) cudaStreamDestroy(sh);
    sp = sh = nullptr;
    ev_narrow = ev_panel = ev_queue = ev_helper = nullptr;
  }
};

// True the first time a call site asks for the current device (one bit per
// device in the site's mask): per-function attributes (dynamic shared memory,
// non-portable clusters) are per device, and the multi-GPU driver launches on
// several devices from one process.
inline bool first_on_device(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}

inline unsigned cdiv_u(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }
// SMs of the current device (read once)
inline int64_t sm_count() {
  static int64_t n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return (int64_t)v;
  }();
  return n;
}

template <int K>
struct Ops {
  // tile configurations (tuned per K)
  static constexpr int BM = (K == 2) ? 32 : 16;
  static constexpr int BN = (K == 2) ? 32 : 16;
  // K=2: BK=8 with the limb-interleaved layout measured best (cfg1 n=4096:
  // 93.2% of the FP64 peak; profiles/r1_gemm_variants.txt)
  static constexpr int BK = 8;
  static constexpr int TM = (K == 2) ? 2 : 1;
  static constexpr int TN = (K == 2) ? 2 : 1;

  template <int MODE, int BM_, int BN_, int BK_, int TM_, int TN_, int MINB_>
  static void launch_cfg(const GemmArgs& g, cudaStream_t st, int cls, double ops, int ctas = 0) {
    using Cfg = GemmCfg<K, MODE, BM_, BN_, BK_, TM_, TN_>;
    auto kern = gemm_kernel<K, MODE, BM_, BN_, BK_, TM_, TN_, MINB_>;
    static unsigned long long attr_set = 0;
    if (first_on_device(attr_set))
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    int64_t tiles = (int64_t)cdiv_u(g.l, BN_) * (int64_t)cdiv_u(g.m, BM_);
    if (g.tile_ctr != nullptr) tiles = std::min<int64_t>(tiles, std::max(ctas, 1));  // persistent CTAs
    dim3 grid((unsigned)tiles);
    // a helper launch on a shared queue (ops < 0) is not timed: it runs inside
    // the main launch's interval, which already carries the work
    int tok_ = ops >= 0.0 ? prof_begin(cls, ops, st) : -1;
    kern<<<grid, Cfg::NT, Cfg::SMEM, st>>>(g);
    if (ops >= 0.0) prof_end(tok_, st);
    check_launch("gemm_kernel");
  }

  // tile variant for K = 2 (MPC_GEMM_VARIANT, read once)
  static int variant() {
    static int v = [] {
      const char* e = getenv("MPC_GEMM_VARIANT");
      return e ? atoi(e) : 0;
    }();
    return v;
  }

  template <int MODE>
  static void gemm_launch(const GemmArgs& g, cudaStream_t st, int cls, double per_elem) {
    if (g.m <= 0 || g.l <= 0) return;
    double ops = (double)g.m * (double)g.l * (double)g.n * per_elem;
    // matrix-vector products (reference_rhs at k = 8, the backward-error
    // probe at k + 2): 32 x 1 tiles, no idle columns
    if (g.l == 1) {
      launch_cfg<MODE, 32, 1, BK, 1, 1, (K >= 5 ? 1 : 2)>(g, st, cls, ops);
      return;
    }
    if constexpr (K == 2) {
      // alternatives measured in round 1 (profiles/r1_gemm_variants.txt):
      // BK=16, 1 CTA/SM with 132 regs, 64x32 tile with a 4x2 micro-tile --
      // all slower than 32x32 / BK=8 / 2x2 / 2 CTAs per SM
      (void)variant;
      // grids under one wave (TRSM / panel updates on few columns): 16 x 16
      // tiles, one element per thread -- 4x the CTAs for the same chains
      // (each element's operation order does not depend on the tiling)
      if ((int64_t)cdiv_u(g.l, BN) * (int64_t)cdiv_u(g.m, BM) < 2 * sm_count()) {
        launch_cfg<MODE, 16, 16, BK, 1, 1, 2>(g, st, cls, ops);
        return;
      }
    }
    // K=3,4: 2 CTAs/SM (register cap 128) measured best for config 3
    // (TD 1.13 s / QD 2.31 s vs 1.39 / 3.14 s at 1 CTA/SM; 128-thread tiles
    // in between -- profiles/r1_cfg3_tdqd.txt)
    if constexpr (K >= 5) {  // verification kernels: registers over occupancy
      launch_cfg<MODE, BM, BN, BK, TM, TN, 1>(g, st, cls, ops);
    } else if constexpr ((K == 3 || K == 4) && !ModeInfo<MODE>::CHAINED) {
      // TD / QD: the kernel is latency-bound on the renorm dependency chains
      // (ncu r2: "wait" is the top stall at 16 warps / SM), and with the
      // accumulators in local memory it fits 62 / 76 registers without
      // spills: 4 (3) CTAs per SM instead of 2 (MPC_TDQD_MINB for the A/B)
      static const int minb = [] {
        const char* e = getenv("MPC_TDQD_MINB");
        const int v = e ? atoi(e) : 4;
        return v >= 2 && v <= 4 ? v : 4;
      }();
      if (minb == 4)
        launch_cfg<MODE, BM, BN, BK, TM, TN, 4>(g, st, cls, ops);
      else if (minb == 3)
        launch_cfg<MODE, BM, BN, BK, TM, TN, 3>(g, st, cls, ops);
      else
        launch_cfg<MODE, BM, BN, BK, TM, TN, 2>(g, st, cls, ops);
    } else {
      launch_cfg<MODE, BM, BN, BK, TM, TN, 2>(g, st, cls, ops);
    }
  }

  static void rgemm(int64_t m, int64_t n, int64_t l, View a, View b, View c, cudaStream_t st) {
    GemmArgs g{m, n, l, a, b, c, 0, nullptr};
    gemm_launch<MODE_REAL>(g, st, PC_GEMM, OpModel<K>::real_mac);
  }

  // P = A B (epi 0) or C = C - A B (epi 1), 3M or 4M
  static void cgemm(bool use3m, int64_t m, int64_t n, int64_t l, View a, View b, View c, int epi,
                    cudaStream_t st, const int64_t* status) {
    GemmArgs g{m, n, l, a, b, c, epi, status};
    if (use3m)
      gemm_launch<MODE_G3>(g, st, PC_GEMM, 3 * OpModel<K>::real_mac);
    else
      gemm_launch<MODE_G4>(g, st, PC_GEMM, 4 * OpModel<K>::real_mac);
  }

  // The same product computed by `ctas` persistent CTAs that claim tiles from
  // the queue `ctr` (zeroed by the caller, stream ordered).  Several launches
  // may share one queue: getrf caps the trailing update while the next panel
  // is being factored and adds the remaining CTAs once it is done.  Tiles are
  // the full-size configuration's, so every element's chain is unchanged.
  // helper = true: not timed / counted as work (it runs inside the main
  // launch's interval).
  static void cgemm_queued(bool use3m, int64_t m, int64_t n, int64_t l, View a, View b, View c,
                           int epi, cudaStream_t st, const int64_t* status, unsigned* ctr, int ctas,
                           bool helper) {
    if (m <= 0 || l <= 0) return;
    GemmArgs g{m, n, l, a, b, c, epi, status};
    g.tile_ctr = ctr;
    const double ops = helper ? -1.0
                              : (double)m * (double)l * (double)n * (use3m ? 3.0 : 4.0) *
                                    OpModel<K>::real_mac;
    if (use3m)
      launch_cfg<MODE_G3, BM, BN, BK, TM, TN, QMINB>(g, st, PC_GEMM, ops, ctas);
    else
      launch_cfg<MODE_G4, BM, BN, BK, TM, TN, QMINB>(g, st, PC_GEMM, ops, ctas);
  }
  // resident CTAs per SM of the queued (persistent) update
  static constexpr int QMINB = (K == 3 || K == 4) ? 4 : 2;

  // chained update C -= L (x) U, each element's subtractions in column order
  static void supdate(bool use3m, int64_t m, int64_t kb, int64_t l, View L, View U, View C,
                      cudaStream_t st, const int64_t* status) {
    if (m <= 0 || l <= 0 || kb <= 0) return;
    GemmArgs g{m, kb, l, L, U, C, 0, status};
    if (use3m)
      gemm_launch<MODE_S3>(g, st, PC_SUPD, OpModel<K>::upd3_exec);
    else
      gemm_launch<MODE_S4>(g, st, PC_SUPD, OpModel<K>::upd4);
  }

  static void mat_add(int64_t rows, int64_t cols, View a, View b, View c, double sign,
                      cudaStream_t st) {
    int64_t total = rows * cols;
    if (total <= 0) return;
    unsigned blocks = (unsigned)std::min<int64_t>(cdiv_u(total, 256), 148 * 16);
    int tok_ = prof_begin(PC_OTHER, 0.0, st);
    mat_add_kernel<K><<<blocks, 256, 0, st>>>(rows, cols, a, b, c, sign);
    prof_end(tok_, st);
    check_launch("mat_add_kernel");
  }

  static void renorm_planes(int64_t rows, int64_t cols, View a, cudaStream_t st) {
    int64_t total = rows * cols;
    if (total <= 0) return;
    unsigned blocks = (unsigned)std::min<int64_t>(cdiv_u(total, 256), 148 * 16);
    int tok_ = prof_begin(PC_OTHER, 0.0, st);
    renorm_planes_kernel<K><<<blocks, 256, 0, st>>>(rows, cols, a);
    prof_end(tok_, st);
    check_launch("renorm_planes_kernel");
  }

  static void laswp(View A, int64_t col0, int64_t ncols, const int64_t* piv, int64_t r0,
                    int64_t r1, cudaStream_t st, const int64_t* status) {
    if (ncols <= 0 || r1 <= r0) return;
    dim3 grid(cdiv_u(ncols, LASWP_NT), 2 * K);
    int tok_ = prof_begin(PC_LASWP, 0.0, st);
    laswp_kernel<K><<<grid, LASWP_NT, 0, st>>>(A, col0, ncols, piv, r0, r1, status);
    prof_end(tok_, st);
    check_launch("laswp_kernel");
  }

  // rows of a diagonal block handled by one trsm_diag_kernel launch: 16, or
  // 32 (half the launches of the recursion, twice the serial steps per
  // launch; MPC_TRSM_BASE for the A/B)
  static int trsm_base() {
    static int b = [] {
      const char* e = getenv("MPC_TRSM_BASE");
      return e && atoi(e) == 32 ? 32 : 16;
    }();
    return b;
  }
  // L (kb x kb, unit lower, strictly-lower part read) and X (kb x M) views
  static void trsm(bool use3m, int64_t kb, int64_t M, View L, View X, cudaStream_t st,
                   const int64_t* status) {
    if (kb <= 1 || M <= 0) return;
    const int TB = trsm_base();
    if (kb <= TB) {
      int tok_ = prof_begin(PC_TRSM, (double)M * (double)(kb * (kb - 1) / 2) * OpModel<K>::upd(use3m), st);
      if (TB == 32)
        trsm_diag_kernel<K, 32><<<cdiv_u(M * 32, 128), 128, 0, st>>>(L, X, kb, M, use3m ? 1 : 0,
                                                                    status);
      else
        trsm_diag_kernel<K, 16><<<cdiv_u(M * 16, 128), 128, 0, st>>>(L, X, kb, M, use3m ? 1 : 0,
                                                                    status);
      prof_end(tok_, st);
      check_launch("trsm_diag_kernel");
      return;
    }
    int64_t h = kb / 2;
    trsm(use3m, h, M, L, X, st, status);
    supdate(use3m, kb - h, h, M, L.sub(h, 0), X, X.sub(h, 0), st, status);
    trsm(use3m, kb - h, M, L.sub(h, h), X.sub(h, 0), st, status);
  }

  // base-panel width (<= WMAX); MPC_PANEL_BASE overrides for experiments
  static int panel_base_w() {
    static int b = [] {
      const char* e = getenv("MPC_PANEL_BASE");
      int v = e ? atoi(e) : PanelCluster<K>::WMAX;
      return (v >= 1 && v <= PanelCluster<K>::WMAX) ? v : PanelCluster<K>::WMAX;
    }();
    return b;
  }
  // base panel: columns [c0, c0+w) over rows [c0, n), swaps within [c0, c0+w)
  // cluster size for the base panel: the largest of 16 / 8 / 4 / 2 that can
  // be co-scheduled (0 = use the per-column launches; MPC_PANEL=launches)
  static int panel_cluster_size() {
    static int cs = [] {
      const char* e = getenv("MPC_PANEL");
      if (e && std::string(e) == "launches") return 0;
      auto kern = panel_cluster_kernel<K>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      const char* cap_s = getenv("MPC_PANEL_CLUSTER");  // cap (experiments)
      const int cap = cap_s ? atoi(cap_s) : 16;
      for (int c : {16, 8, 4, 2}) {
        if (c > cap) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c);
        cfg.blockDim = dim3(PanelCluster<K>::NT);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0)
          return c;
        cudaGetLastError();
      }
      return 0;
    }();
    return cs;
  }

  // CTAs of panel_grid_kernel that can be co-resident (0: use the cluster /
  // per-column kernels -- MPC_PANEL=cluster or =launches, or no cooperative
  // launch support)
  static int panel_grid_max() {
    static int g = [] {
      const char* e = getenv("MPC_PANEL");
      if (e && (std::string(e) == "launches" || std::string(e) == "cluster")) return 0;
      int dev = 0, coop = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
      if (!coop) return 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panel_grid_kernel<K, 2>,
                                                        PanelGrid<K>::NT, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
      }
      return (int)std::min<int64_t>(PANEL_GRID_GMAX, per_sm * sm_count());
    }();
    return g;
  }

  static void panel_base(bool use3m, View A, int64_t n, int64_t c0, int64_t w, int64_t* piv,
                         PanelWs ws, cudaStream_t st) {
    int64_t cend = c0 + w;
    // one row per thread, rows resident in registers: a cooperative grid
    if (const int gmax = panel_grid_max()) {
      // two lanes per row (split cdiv) while the grid fits, else one
      static const int tpr_max = [] {
        const char* e = getenv("MPC_PANEL_TPR");
        return e && atoi(e) == 1 ? 1 : 2;
      }();
      constexpr int NT = PanelGrid<K>::NT;
      const int tpr = (tpr_max == 2 && (n - c0 + NT / 2 - 1) / (NT / 2) <= gmax) ? 2 : 1;
      const int64_t G = (n - c0 + NT / tpr - 1) / (NT / tpr);
      if (G <= gmax && w <= PanelGrid<K>::W) {
        int wi = (int)w, u3 = use3m ? 1 : 0;
        void* args[] = {&A, &n, &c0, &wi, &u3, &piv, &ws.status, &ws.gbar, &ws.slots};
        double ops = 0.0;
        for (int64_t j = c0; j < cend; j++) ops += (double)(n - j - 1) * (double)(cend - j - 1);
        int tok_ = prof_begin(PC_PANEL, ops * OpModel<K>::upd(use3m), st);
        void* kern = tpr == 2 ? (void*)panel_grid_kernel<K, 2> : (void*)panel_grid_kernel<K, 1>;
        if (panel_plain_launch_ok())  // this call owns the device's slot (see panel_slot)
          cudaLaunchKernel(kern, dim3((unsigned)G), dim3(NT), args, 0, st);
        else
          cudaLaunchCooperativeKernel(kern, dim3((unsigned)G), dim3(NT), args, 0, st);
        prof_end(tok_, st);
        check_launch("panel_grid_kernel");
        return;
      }
    }
    if (int csmax = panel_cluster_size()) {
      static unsigned long long attr = 0;
      if (first_on_device(attr))
        cudaFuncSetAttribute(panel_cluster_kernel<K>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1);
      // smallest power-of-two cluster giving every thread at most one row
      int cs = 1;
      while (cs < csmax &&
             (int64_t)cs * (PanelCluster<K>::NT / PanelCluster<K>::TPR) < n - c0)
        cs *= 2;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(PanelCluster<K>::NT);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      double ops = 0.0;
      for (int64_t j = c0; j < cend; j++) ops += (double)(n - j - 1) * (double)(cend - j - 1);
      int tok_ = prof_begin(PC_PANEL, ops * OpModel<K>::upd(use3m), st);
      cudaLaunchKernelEx(&cfg, panel_cluster_kernel<K>, A, n, c0, w, use3m ? 1 : 0, piv,
                         ws.status);
      prof_end(tok_, st);
      check_launch("panel_cluster_kernel");
      return;
    }
    int tok_ = prof_begin(PC_PANEL, 0.0, st);
    pivot_first_kernel<K><<<cdiv_u(n - c0, PNT), PNT, 0, st>>>(A, n, c0, c0, cend, piv, ws);
    prof_end(tok_, st);
    check_launch("pivot_first_kernel");
    for (int64_t j = c0; j < cend; j++) {
      int64_t rows = n - j - 1;
      if (rows <= 0) break;
      int tok_ = prof_begin(PC_PANEL, (double)rows * (double)(cend - j - 1) * OpModel<K>::upd(use3m), st);
      panel_step_kernel<K><<<cdiv_u(rows, PNT), PNT, 0, st>>>(A, n, j, c0, cend, use3m ? 1 : 0,
                                                              piv, ws);
      prof_end(tok_, st);
      check_launch("panel_step_kernel");
    }
  }

  // recursive panel factorization of columns [c0, c0+w); on return every
  // interchange piv[c0..c0+w) has been applied to columns [c0, c0+w)
  static void panel_rec(bool use3m, View A, int64_t n, int64_t c0, int64_t w, int64_t* piv,
                        PanelWs ws, cudaStream_t st) {
    const int64_t PANEL_BASE = panel_base_w();
    if (w <= PANEL_BASE) {
      panel_base(use3m, A, n, c0, w, piv, ws, st);
      return;
    }
    int64_t h = ((w / 2 + PANEL_BASE - 1) / PANEL_BASE) * PANEL_BASE;
    if (h >= w) h = w / 2;
    panel_rec(use3m, A, n, c0, h, piv, ws, st);
    laswp(A, c0 + h, w - h, piv, c0, c0 + h, st, ws.status);
    trsm(use3m, h, w - h, A.sub(c0, c0), A.sub(c0, c0 + h), st, ws.status);
    supdate(use3m, n - c0 - h, h, w - h, A.sub(c0 + h, c0), A.sub(c0, c0 + h),
            A.sub(c0 + h, c0 + h), st, ws.status);
    panel_rec(use3m, A, n, c0 + h, w - h, piv, ws, st);
    laswp(A, c0, h, piv, c0 + h, c0 + w, st, ws.status);
  }

  // lu_panel on an n x n matrix: factor [jb, jb+kw) and apply the
  // interchanges to every other column (full-row swap semantics)
  static void lu_panel(bool use3m, View A, int64_t n, int64_t jb, int64_t kw, int64_t* piv,
                       PanelWs ws, cudaStream_t st) {
    panel_rec(use3m, A, n, jb, kw, piv, ws, st);
    laswp(A, 0, jb, piv, jb, jb + kw, st, ws.status);
    laswp(A, jb + kw, n - jb - kw, piv, jb, jb + kw, st, ws.status);
  }

  // Trailing work of panel b = [jb, jb+kw) on the column range [c0, c1)
  // (all right of the panel): interchanges, U12 TRSM, fused A22 -= L21 U12.
  static void update_cols(bool use3m, View A, int64_t n, int64_t jb, int64_t kw, int64_t c0,
                          int64_t c1, const int64_t* piv, const int64_t* status,
                          cudaStream_t st) {
    if (c1 <= c0) return;
    int64_t end = jb + kw;
    laswp(A, c0, c1 - c0, piv, jb, end, st, status);
    trsm(use3m, kw, c1 - c0, A.sub(jb, jb), A.sub(jb, c0), st, status);
    cgemm(use3m, n - end, kw, c1 - c0, A.sub(end, jb), A.sub(jb, c0), A.sub(end, c0), 1, st,
          status);
  }

  // CTAs of the trailing update's first (capped) launch while the next panel
  // is factored beside it (MPC_GEMM_CAP; 0 = one uncapped launch)
  // (unset: automatic, see gemm_cap_for; 0: never; N: always N CTAs)
  static int gemm_cap_env() {
    static int c = [] {
      const char* e = getenv("MPC_GEMM_CAP");
      return e ? atoi(e) : -1;
    }();
    return c;
  }
  // Automatic rule: cap the update at 7/8 of the CTA slots when the next
  // panel is not comfortably hidden behind it -- estimated update time under
  // five times the estimated panel time (panel: dependent latency per column
  // + its chained updates; constants measured on one B200: 16 us / column,
  // updates at 14 T op/s, GEMM at 16.5).  Config 2: 196 -> 190 ms; config 4
  // only reaches the rule in its last steps (capping every step costs it 3%:
  // profiles/r2_gemm_cap_ab.txt).
  static int gemm_cap_for(bool use3m, int64_t rows, int64_t kw, int64_t cols, int64_t kw2) {
    const int e = gemm_cap_env();
    if (e >= 0) return e;
    // TD / QD: measured no gain (config 3: 590 vs 598 ms, 1118 vs 1153 ms with
    // the cap) -- their panels are bound by the expansion arithmetic's own
    // latency, not by waiting for CTA slots -- so the rule is DD only
    if constexpr (K != 2) return 0;
    constexpr double col_us = 16.0, gemm_tops = 16.5, supd_tops = 14.0;
    const double rest_ms = (double)rows * (double)kw * (double)cols * (use3m ? 3.0 : 4.0) *
                           OpModel<K>::real_mac / (gemm_tops * 1e9);
    const double panel_ms = col_us * 1e-3 * (double)kw2 +
                            0.485 * (double)rows * (double)kw2 * (double)kw2 *
                                OpModel<K>::upd(use3m) / (supd_tops * 1e9);
    const int full = QMINB * (int)sm_count();
    return rest_ms < 5.0 * panel_ms ? full - full / 8 : 0;
  }

  // lu._factor (lu.py:129-163) with depth-1 lookahead: while `st` applies
  // panel b's trailing update to columns right of block b+1, panel b+1
  // (already updated by b) is factored on a high-priority side stream.
  // Element operation sequences are unchanged (bit-identical to the
  // sequential schedule); only independent column ranges overlap.
  static void getrf(bool use3m, View A, int64_t n, int64_t Kp, int64_t* piv, PanelWs ws,
                    cudaStream_t st) {
    SideStream ss;
    ss.set_main(st);
    cudaStream_t sp = ss.sp;
    cudaEvent_t ev_narrow = ss.ev_narrow, ev_panel = ss.ev_panel;
    // MPC_TRACE=1: per-step timeline (stderr) -- where the step time goes
    static const bool trace = getenv("MPC_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      tev.push_back(e);
    };
    bool helper_pending = false;
    const ColSource src = col_source();
    auto need = [&](int64_t c1) {
      if (src.need) src.need(src.ctx, std::min(c1, n), st);
    };
    mark(st);
    need(std::min(Kp, n));
    panel_rec(use3m, A, n, 0, std::min(Kp, n), piv, ws, st);
    mark(st);
    for (int64_t jb = 0; jb < n; jb += Kp) {
      int64_t kw = std::min(Kp, n - jb);
      int64_t end = jb + kw;
      laswp(A, 0, jb, piv, jb, end, st, ws.status);  // left of the panel
      if (end == n) {
        if (row_sink().fn) row_sink().fn(row_sink().ctx, jb, end, st);
        break;
      }
      int64_t kw2 = std::min(Kp, n - end);
      // narrow update of block b+1, then factor it on the side stream
      if (jb == 0) need(end + kw2);
      update_cols(use3m, A, n, jb, kw, end, end + kw2, piv, ws.status, st);
      cudaEventRecord(ev_narrow, st);
      mark(st);
      cudaStreamWaitEvent(sp, ev_narrow, 0);
      panel_rec(use3m, A, n, end, kw2, piv, ws, sp);
      cudaEventRecord(ev_panel, sp);
      mark(sp);
      // rest of panel b's update overlaps the panel factorization
      if (jb == 0 && src.need) {
        // step 0 in column chunks, each behind its own host-to-device copy
        // (per-column work, so the chunking does not change any bits)
        const int64_t ch = std::max<int64_t>(src.chunk, Kp);
        for (int64_t c0 = end + kw2; c0 < n; c0 += ch) {
          need(c0 + ch);
          update_cols(use3m, A, n, jb, kw, c0, std::min(n, c0 + ch), piv, ws.status, st);
        }
      } else if (const int cap_req = (end + kw2 < n) ? gemm_cap_for(use3m, n - end, kw, n - end - kw2, kw2) : 0) {
        // capped trailing update: `cap` persistent CTAs claim tiles from a
        // queue, leaving room on every SM for the panel's kernels (which
        // otherwise wait for whole 0.4 - 0.8 ms GEMM CTAs to retire before
        // each of their ~300 dependent launches); once the panel is done a
        // helper launch on the same queue restores full occupancy
        const int64_t c0 = end + kw2;
        const int full = QMINB * (int)sm_count();
        const int cap = std::min(cap_req, full);
        laswp(A, c0, n - c0, piv, jb, end, st, ws.status);
        trsm(use3m, kw, n - c0, A.sub(jb, jb), A.sub(jb, c0), st, ws.status);
        cudaMemsetAsync(ws.tile_ctr, 0, sizeof(unsigned), st);
        cudaEventRecord(ss.ev_queue, st);
        cgemm_queued(use3m, n - end, kw, n - c0, A.sub(end, jb), A.sub(jb, c0), A.sub(end, c0), 1,
                     st, ws.status, ws.tile_ctr, cap, false);
        if (cap < full) {
          cudaStreamWaitEvent(ss.sh, ss.ev_queue, 0);
          cudaStreamWaitEvent(ss.sh, ev_panel, 0);
          cgemm_queued(use3m, n - end, kw, n - c0, A.sub(end, jb), A.sub(jb, c0), A.sub(end, c0),
                       1, ss.sh, ws.status, ws.tile_ctr, full - cap, true);
          cudaEventRecord(ss.ev_helper, ss.sh);
          helper_pending = true;
        }
      } else {
        update_cols(use3m, A, n, jb, kw, end + kw2, n, piv, ws.status, st);
      }
      if (row_sink().fn) row_sink().fn(row_sink().ctx, jb, end, st);
      mark(st);
      cudaStreamWaitEvent(st, ev_panel, 0);
      if (helper_pending) {
        cudaStreamWaitEvent(st, ss.ev_helper, 0);
        helper_pending = false;
      }
      mark(st);
    }
    if (trace) {
      cudaStreamSynchronize(st);
      float t;
      cudaEventElapsedTime(&t, tev[0], tev[1]);
      fprintf(stderr, "MPC_TRACE n=%lld K=%lld first-panel %.3f ms\n", (long long)n, (long long)Kp, t);
      // per step: [start(prev end), narrow done, panel done (side), rest done, joined]
      for (size_t i = 1; i + 4 < tev.size(); i += 4) {
        float tn, tp, tr, tj;
        cudaEventElapsedTime(&tn, tev[i], tev[i + 1]);
        cudaEventElapsedTime(&tp, tev[i + 1], tev[i + 2]);
        cudaEventElapsedTime(&tr, tev[i + 1], tev[i + 3]);
        cudaEventElapsedTime(&tj, tev[i], tev[i + 4]);
        fprintf(stderr, "MPC_TRACE step %zu: narrow %.3f  panel(side) %.3f  rest %.3f  step %.3f ms\n",
                (i - 1) / 4, tn, tp, tr, tj);
      }
      for (auto e : tev) cudaEventDestroy(e);
    }
  }

  // solve_fb (_kernels.py:708-775); b overwritten by x.  phases: 1 = the
  // interchanges + forward (unit lower) substitution, 2 = the backward
  // substitution (b holds the forward result), 3 = both (solve_fb).
  static void getrs(bool use3m, View F, int64_t n, const int64_t* piv, double* br, double* bi,
                    int phases, cudaStream_t st) {
    if (n <= 0 || phases == 0) return;
    using C = SolveCfg<K>;
    const int u3 = use3m ? 1 : 0;
    const int64_t vec = 2 * (int64_t)K * n;
    double *y = nullptr, *z = nullptr, *inv = nullptr;
    int64_t* idx = nullptr;
    auto ck = [](cudaError_t e, const char* w) {
      if (e != cudaSuccess) throw LaunchError{w};
    };
    struct Free {  // stream-ordered frees on every exit path
      cudaStream_t st;
      void* p[4];
      ~Free() {
        for (void* q : p)
          if (q) cudaFreeAsync(q, st);
      }
    } fr_{st, {nullptr, nullptr, nullptr, nullptr}};
    retain_pool();
    ck(cudaMallocAsync((void**)&y, sizeof(double) * vec, st), "getrs workspace");
    fr_.p[0] = y;
    ck(cudaMallocAsync((void**)&z, sizeof(double) * vec, st), "getrs workspace");
    fr_.p[1] = z;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
      cudaFuncSetAttribute(trsv_block_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::SMEM);
      cudaFuncSetAttribute(trsv_block_kernel<K, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
      cudaFuncSetAttribute(perm_compose_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
    }
    const unsigned gblocks = (unsigned)std::min<int64_t>(cdiv_u(vec, 256), 148 * 8);
    if (phases & 1) {
      ck(cudaMallocAsync((void**)&idx, sizeof(int64_t) * n, st), "getrs workspace");
      fr_.p[2] = idx;
      const bool smem = n * (int64_t)sizeof(int) <= 200 * 1024;
      int tok_ = prof_begin(PC_SOLVE, 0.0, st);
      perm_compose_kernel<K><<<1, 256, smem ? n * sizeof(int) : 0, st>>>(piv, n, idx,
                                                                         smem ? 1 : 0);
      prof_end(tok_, st);
      check_launch("perm_compose_kernel");
      tok_ = prof_begin(PC_SOLVE, 0.0, st);
      perm_gather_kernel<K><<<gblocks, 256, 0, st>>>(br, bi, idx, n, y);
      prof_end(tok_, st);
      check_launch("perm_gather_kernel");
      for (int64_t r0 = 0; r0 < n; r0 += C::KB) {
        int64_t kb = std::min<int64_t>(C::KB, n - r0);
        int64_t rows = n - r0 - kb;
        unsigned grid = rows > 0 ? cdiv_u(rows, C::RT) : 1u;
        int tok_ = prof_begin(PC_SOLVE, ((double)rows * kb + kb * (kb - 1) / 2.0) * OpModel<K>::upd(use3m), st);
        trsv_block_kernel<K, true><<<grid, C::RT, C::SMEM, st>>>(F, y, y + K * n, z, z + K * n, n,
                                                                 r0, kb, u3, nullptr);
        prof_end(tok_, st);
        check_launch("trsv_block_kernel<fwd>");
      }
      if (!(phases & 2)) {
        ck(cudaMemcpyAsync(br, z, sizeof(double) * K * n, cudaMemcpyDeviceToDevice, st), "getrs copy");
        ck(cudaMemcpyAsync(bi, z + K * n, sizeof(double) * K * n, cudaMemcpyDeviceToDevice, st),
           "getrs copy");
        return;
      }
    } else {
      ck(cudaMemcpyAsync(z, br, sizeof(double) * K * n, cudaMemcpyDeviceToDevice, st), "getrs copy");
      ck(cudaMemcpyAsync(z + K * n, bi, sizeof(double) * K * n, cudaMemcpyDeviceToDevice, st),
         "getrs copy");
    }
    ck(cudaMallocAsync((void**)&inv, sizeof(double) * vec, st), "getrs workspace");
    fr_.p[3] = inv;
    {
      int tok_ = prof_begin(PC_SOLVE, 0.0, st);
      diag_inv_kernel<K><<<cdiv_u(n, 128), 128, 0, st>>>(F, n, inv, u3);
      prof_end(tok_, st);
      check_launch("diag_inv_kernel");
    }
    const int64_t nb = (n + C::KB - 1) / C::KB;
    for (int64_t b = nb - 1; b >= 0; b--) {
      int64_t r0 = b * C::KB;
      int64_t kb = std::min<int64_t>(C::KB, n - r0);
      unsigned grid = r0 > 0 ? cdiv_u(r0, C::RT) : 1u;
      int tok_ = prof_begin(PC_SOLVE, ((double)r0 * kb + kb * (kb - 1) / 2.0) * OpModel<K>::upd(use3m), st);
      trsv_block_kernel<K, false><<<grid, C::RT, C::SMEM, st>>>(F, z, z + K * n, br, bi, n, r0, kb,
                                                                u3, inv);
      prof_end(tok_, st);
      check_launch("trsv_block_kernel<bwd>");
    }
  }
};

}  // namespace mpc
