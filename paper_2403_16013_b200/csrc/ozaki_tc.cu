// ozaki_tc.cu -- the Ozaki scheme's exact part products on the B200 INT8
// tensor cores (BASELINE.json north_star item 3).
//
// Reference: ozaki.py:79-159 (split grids, _pair_schedule, rgemm_ozaki),
// _kernels.py:485-517 (acc_plane, renorm_planes).
//
// Why this is bit-identical to the reference's binary64 seam (np.matmul):
// every entry of split part p is an integer multiple of its row (left) or
// column (right) grid, part = I * 2^e with |I| <= 2^width (ozaki.py:54-60,
// 97-107), and width <= (53 - ceil(log2 n)) / 2 (ozaki.py:33-38) makes
// every part product  P = A_p B_q = 2^(ea_i + eb_j) * sum_t Ia_it Ib_tj  an
// exact binary64 number -- the reference's GEMM returns exactly
// J_ij * 2^(ea_i + eb_j) with the exact integer J.  Here J is formed from
// INT8 digit slices:  I = a0 2^(2b) + a1 2^b + a2  (b = 7: all digits s8,
// |a0| <= 64; b = 8: a0 s8, a1/a2 u8), so
//     J = sum_{s=0..4} 2^(b(4-s)) G_s,   G_s = sum_{i+j=s} A_i B_j^T,
// five int32 tcgen05 accumulators per pair (|G_s| < 2^31 is checked on the
// host from n and the digit bounds), recombined in int64 (exact, |J| <=
// 2^53), converted exactly to binary64 and scaled by the two powers of two.
// The acc_plane insertion (schedule order) and the final renorm_planes run
// in the same kernel on the per-thread accumulators -- one launch replaces
// the reference's npairs GEMMs + npairs acc_plane passes + renorm pass.
// (Subnormal grids, i.e. operands below ~1e-290, are outside this argument;
// the split kernels already follow the reference there.)
//
// Kernel shape (per CTA: one 128 x BN output tile, 128 threads):
//   * operands: K-major INT8 slices in global memory, padded to the tile
//     grid; staged by cp.async (16 B) into a 3-stage ring in the canonical
//     no-swizzle K-major UMMA layout (8-row x 16-byte core matrices);
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::i8
//     (M=128, N=BN, K=32) -- 9 per 32-deep k-step into 5 TMEM accumulator
//     groups -- and tcgen05.commit's to per-stage mbarriers, so the ring
//     slots are recycled as soon as the tensor core has read them;
//   * after a pair's last k-step, all 4 warps drain the groups with
//     tcgen05.ld.32x32b (thread = output row), recombine, scale and run
//     acc_plane into register-resident expansions; the next pair's loads
//     are already in flight.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "ozaki_tc.h"
#include "prof.h"

namespace mpc {
namespace otc {

constexpr int BM = 128;     // MMA M (one TMEM lane per output row)
constexpr int BKB = 64;     // K bytes per pipeline stage = 2 MMAs of K = 32
constexpr int NSL = 3;      // digit slices per part
constexpr int NGRP = 5;     // accumulator groups s = i + j
// epilogue warps: 4 per TMEM lane quadrant (16); 12 for DD (-DMPC_OZAKI_DD_NEPI=12,
// 3 column groups of 16, 128 registers) measured 1.5% slower at the LU shape
#ifndef MPC_OZAKI_DD_NEPI
#define MPC_OZAKI_DD_NEPI 16
#endif
template <int KL>
struct Epi {
  static constexpr int NEPI = KL == 2 ? MPC_OZAKI_DD_NEPI : 16;
  static constexpr int NTHR = (NEPI + 2) * 32;  // + producer warp + MMA warp
};
constexpr int MAXPAIRS = 160;
#ifndef SPLIT_SMEM_CAP
#define SPLIT_SMEM_CAP (72 * 1024)  // split CTAs: up to 3 per SM (200 KB: 2x slower, 36 KB: 20% slower)
#endif
constexpr uint32_t TCOLS = 512;        // two accumulator buffers at columns 0 / 256

template <int KL>
struct Tile {
  static constexpr int BN = KL == 2 ? 48 : 32;  // 5 * BN <= 256: double-buffered TMEM
  static constexpr int A_BYTES = NSL * BM * BKB;
  static constexpr int B_BYTES = NSL * BN * BKB;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (220 * 1024) / STAGE;
  static constexpr int SMEM = STAGES * STAGE;
};

struct Params {
  const int8_t* sa;       // [d][NSL][Mp/BM][Kp/16][BM][16]  (stage-contiguous tiles)
  const int8_t* sb;       // [d][NSL][Lp/BN][Kp/16][BN][16]
  const double* scale_a;  // [d][m]
  const double* scale_b;  // [d][l]
  int64_t m, l, Mp, Lp, Kp;
  int npairs, shift;
  View C;
  // fused complex composition (OzCombine): 0 = plain C = A B; 3 / 4 = this is
  // the last real product of a 3M / 4M cgemm, T1 / T2 / T3 hold the earlier
  // ones; epi = 1 subtracts the complex result from Cc (lu.py:158-161)
  int mode, epi;
  View T1, T2, T3, Cc;
  unsigned char pp[MAXPAIRS], pq[MAXPAIRS];
};

MPC_DI uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

MPC_DI void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

MPC_DI void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

MPC_DI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

MPC_DI void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// bulk global -> shared copy, completion counted on the mbarrier (async proxy)
MPC_DI void bulk_g2s(uint32_t sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          sdst),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// multicast variant: the same smem offset / mbarrier in every CTA of ctaMask
MPC_DI void bulk_g2s_mc(uint32_t sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                        uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1], %2, [%3], %4;\n" ::"r"(sdst),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

MPC_DI bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

MPC_DI uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

MPC_DI void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

MPC_DI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
MPC_DI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// canonical K-major, no-swizzle shared-memory matrix descriptor: 8-row x
// 16-byte core matrices, LBO = byte distance of the two 16-byte K halves of
// one MMA, SBO = byte distance of consecutive 8-row groups
MPC_DI uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, layout SWIZZLE_NONE
}

// instruction descriptor: D = s32, A/B s8 or u8, both K-major, M = 128
__host__ __device__ constexpr uint32_t make_idesc(int n, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

MPC_DI void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                   uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

MPC_DI void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

MPC_DI void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

MPC_DI void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
MPC_DI void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                   taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
MPC_DI void tmem_ld4(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
MPC_DI void tmem_st4(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
template <int W>
MPC_DI void tmem_ldw(uint32_t taddr, uint32_t (&r)[8]) {
  if constexpr (W == 8) tmem_ld8(taddr, r); else tmem_ld4(taddr, r);
}
template <int W>
MPC_DI void tmem_stw(uint32_t taddr, const uint32_t (&r)[8]) {
  if constexpr (W == 8) tmem_st8(taddr, r); else tmem_st4(taddr, r);
}
MPC_DI void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
MPC_DI void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// acc_plane insertion of one exact binary64 product (_kernels.py:502-517)
template <int KL>
MPC_DI void acc_insert(Exp<KL>& c, double q) {
  double h[KL + 1];
#pragma unroll
  for (int i = KL - 1; i >= 0; i--) {
    double s, e;
    two_sum(q, c.c[i], s, e);
    q = s;
    h[i + 1] = e;
  }
  h[0] = q;
#pragma unroll
  for (int i = 0; i < KL; i++) c.c[i] = h[i];
}

// Warp roles: warps 0..15 epilogue (warp w drains TMEM lane quadrant w % 4,
// column group w / 4), warp 16 producer (one lane issues the bulk copies),
// warp 17 MMA issuer (one lane).  Pipelines: smem ring full/empty (bulk copy
// -> MMA -> tcgen05.commit), TMEM double buffer full/empty (MMA -> epilogue).
template <int KL, int CN, int SB>
__global__ void __launch_bounds__(Epi<KL>::NTHR, 1) ozaki_tc_kernel(const __grid_constant__ Params P) {
  using T = Tile<KL>;
  constexpr int NEPI = Epi<KL>::NEPI;
  constexpr int BN = T::BN, S = T::STAGES;
  constexpr int NCG = NEPI / 4, CPT = BN / NCG;  // column groups, columns per thread
  constexpr int CW = CPT % 8 == 0 ? 8 : 4;       // TMEM load width (x8 or x4)
  static_assert(CPT % CW == 0, "columns per thread must be a multiple of the TMEM load");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[S], empty[S], accf[2], acce[2];
  __shared__ uint32_t tmem_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // column tile / row tile.  Without clusters: grouped raster -- 8 row tiles
  // sweep the column tiles together, so each B slice tile is fetched from
  // DRAM once per group instead of once per row tile (the A tiles of the
  // group stay L2-resident).  With clusters: the cluster shares a row tile.
  int64_t ct, rt;
  if constexpr (CN == 1) {
    constexpr int64_t G = 8;
    const int64_t tiles_m = P.Mp / BM, tiles_n = P.Lp / BN;
    const int64_t bid = blockIdx.x;
    const int64_t grp = bid / (G * tiles_n), first_m = grp * G;
    const int64_t gsz = tiles_m - first_m < G ? tiles_m - first_m : G;
    const int64_t in_grp = bid - grp * G * tiles_n;
    rt = first_m + in_grp % gsz;
    ct = in_grp / gsz;
  } else {
    ct = blockIdx.x;
    rt = blockIdx.y;
  }
  const int64_t col0 = ct * BN, row0 = rt * BM;

  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CN);  // every CTA of the cluster frees the slot
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], NEPI * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (CN > 1) cluster_sync();  // peers' barriers initialised before any multicast
  const uint32_t tmem = tmem_slot;
  const uint32_t crank = CN > 1 ? cluster_rank() : 0u;
  const uint32_t sbase = smem_u32(smem);
  const int nk = (int)(P.Kp / BKB);
  const int64_t kch = P.Kp / 16;

  if (warp == NEPI) {
    // ---------------- producer: one lane streams the stage-contiguous slices
    if (lane == 0) {
      const int64_t tilesA = P.Mp / BM, tilesB = P.Lp / BN;
      int slot = 0;
      uint32_t ph = 0;
      for (int t = 0; t < P.npairs; t++) {
        const int8_t* ga = P.sa + (((int64_t)P.pp[t] * NSL * tilesA + rt) * kch) * (BM * 16);
        // B: the NSL slices of a 16-deep K chunk are stacked (3*BN rows), so
        // one stage is one contiguous block
        const int8_t* gb = P.sb + (((int64_t)P.pq[t] * tilesB + ct) * kch) * (NSL * BN * 16);
        for (int kc = 0; kc < nk; kc++) {
          mbar_wait(&empty[slot], ph ^ 1u);
          const uint32_t sA = sbase + (uint32_t)(slot * T::STAGE), sB = sA + T::A_BYTES;
          mbar_expect_tx(&full[slot], (uint32_t)T::STAGE);
          // the A tile is shared by the cluster (same row tile): CTA r fetches
          // the r-th 1/CN of each slice and multicasts it to every peer
#pragma unroll
          for (int i = 0; i < NSL; i++) {
            const uint32_t off = crank * (BM * BKB / CN);
            const int8_t* src = ga + ((int64_t)i * tilesA * kch + kc * 4) * (BM * 16) + off;
            if constexpr (CN > 1)
              bulk_g2s_mc(sA + i * (BM * BKB) + off, src, BM * BKB / CN, &full[slot],
                          (uint16_t)((1u << CN) - 1u));
            else
              bulk_g2s(sA + i * (BM * BKB), src, BM * BKB, &full[slot]);
          }
          bulk_g2s(sB, gb + (int64_t)kc * 4 * (NSL * BN * 16), T::B_BYTES, &full[slot]);
          if (++slot == S) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == NEPI + 1) {
    // ---------------- MMA issuer: the whole warp walks the pipeline, one
    // elected lane issues.  Descriptors are precomputed: only the 14-bit
    // start-address field of the low word moves (smem < 256 KB, no carry).
    const uint32_t hi = (128u >> 4) | (1u << 14);  // SBO = 128 B, version 1
    const uint32_t loA = ((uint32_t)(BM * 16) >> 4) << 16,
                   loB = ((uint32_t)(NSL * BN * 16) >> 4) << 16;
    // one MMA per A slice against the stacked B slices: N = 3 BN columns,
    // landing on the consecutive groups i, i+1, i+2 (group g at column g BN)
    constexpr uint32_t ID = make_idesc(NSL * BN, true, true);
    const bool leader = elect_one();
    int slot = 0;
    uint32_t ph = 0;
    for (int t = 0; t < P.npairs; t++) {
      const int buf = t & 1;
      mbar_wait(&acce[buf], (uint32_t)((t >> 1) & 1));  // drained and zeroed
      tc_fence_after();
      const uint32_t tacc = tmem + (uint32_t)(buf * 256);
      for (int kc = 0; kc < nk; kc++) {
        mbar_wait(&full[slot], ph);
        tc_fence_after();
        const uint32_t sA = sbase + (uint32_t)(slot * T::STAGE), sB = sA + T::A_BYTES;
        // (the shared::cta window address carries the cluster rank above bit 18;
        // the descriptor takes the 14-bit CTA-local offset)
        const uint32_t a0 = loA | ((sA >> 4) & 0x3FFFu), b0 = loB | ((sB >> 4) & 0x3FFFu);
        if (leader) {
#pragma unroll
          for (int ks = 0; ks < BKB / 32; ks++) {
            const uint64_t bd =
                ((uint64_t)hi << 32) | (b0 + (uint32_t)((ks * 2 * (NSL * BN * 16)) >> 4));
#pragma unroll
            for (int i = 0; i < NSL; i++) {
              const uint64_t ad =
                  ((uint64_t)hi << 32) | (a0 + (uint32_t)((i * (BM * BKB) + ks * 2 * (BM * 16)) >> 4));
              mma_i8(tacc + (uint32_t)(i * BN), ad, bd, ID, 1u);
            }
          }
          // slot free (in every CTA of the cluster) once these MMAs have read it
          if constexpr (CN > 1)
            mma_commit_mc(&empty[slot], (uint16_t)((1u << CN) - 1u));
          else
            mma_commit(&empty[slot]);
        }
        __syncwarp();
        if (++slot == S) {
          slot = 0;
          ph ^= 1u;
        }
      }
      if (leader) mma_commit(&accf[buf]);  // accumulators of pair t complete
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: J = sum_s 2^(b(4-s)) G_s, P = J 2^ea 2^eb, acc_plane
    const int quad = warp & 3, cgrp = warp >> 2;
    const int64_t grow = row0 + quad * 32 + lane;
    const int cbase = cgrp * CPT;
    Exp<KL> acc[CPT];
#pragma unroll
    for (int j = 0; j < CPT; j++) acc[j] = exp_zero<KL>();
    // zero this thread's accumulator columns of both buffers (the MMAs always
    // accumulate), then hand the buffers to the MMA warp
    const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)cbase;
    uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (int bb = 0; bb < 2; bb++) {
#pragma unroll
      for (int g = 0; g < NGRP; g++)
#pragma unroll
        for (int cc = 0; cc < CPT / CW; cc++) tmem_stw<CW>(tq + (uint32_t)(bb * 256 + g * BN + cc * CW), z);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&acce[bb]);
    }
    for (int t = 0; t < P.npairs; t++) {
      const int buf = t & 1;
      mbar_wait(&accf[buf], (uint32_t)((t >> 1) & 1));
      tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * 256 + cbase);
      const double sav = grow < P.m ? P.scale_a[(int64_t)P.pp[t] * P.m + grow] : 0.0;
      const double* sbp = P.scale_b + (int64_t)P.pq[t] * P.l;
#pragma unroll
      for (int cc = 0; cc < CPT / CW; cc++) {
        uint32_t r[NGRP][8];
#pragma unroll
        for (int g = 0; g < NGRP; g++) tmem_ldw<CW>(trow + (uint32_t)(g * BN + cc * CW), r[g]);
        tmem_wait_ld();
#pragma unroll
        for (int g = 0; g < NGRP; g++) tmem_stw<CW>(trow + (uint32_t)(g * BN + cc * CW), z);
        if (cc == CPT / CW - 1) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&acce[buf]);  // drained and re-zeroed for pair t + 2
        }
#pragma unroll
        for (int jj = 0; jj < CW; jj++) {
          // J = sum_s 2^(SB (4 - s)) G_s as int32 x constant -> int64
          // multiply-adds (exact: |J| <= 2^53)
          long long J = (long long)(int)r[4][jj];
          J += (long long)(int)r[3][jj] * (1ll << SB);
          J += (long long)(int)r[2][jj] * (1ll << (2 * SB));
          J += (long long)(int)r[1][jj] * (1ll << (3 * SB));
          J += (long long)(int)r[0][jj] * (1ll << (4 * SB));
          const int64_t gc = col0 + cbase + cc * CW + jj;
          const double sbv = gc < P.l ? sbp[gc] : 0.0;
          // P = J 2^ea 2^eb: exact binary64 (the grids are powers of two)
          const double v = __dmul_rn(__dmul_rn(__ll2double_rn(J), sav), sbv);
          acc_insert<KL>(acc[cc * CW + jj], v);
        }
      }
    }
    // renorm_planes (_kernels.py:485-499) into a shared-memory tile (the
    // operand ring is idle now: every stage has been consumed), then a
    // coalesced pass over the tile stores C -- or applies the fused complex
    // composition / LU subtraction (OzCombine) elementwise.
    constexpr int OS = BN + 1;  // padded row stride (doubles)
    static_assert(KL * BM * OS * 8 <= T::SMEM, "output tile must fit the ring");
    double* otile = reinterpret_cast<double*>(smem);
    const int lrow = quad * 32 + lane;
#pragma unroll
    for (int j = 0; j < CPT; j++) {
      double bufv[KL];
#pragma unroll
      for (int c = 0; c < KL; c++) bufv[c] = acc[j].c[c];
      Exp<KL> o = renorm<KL, KL>(bufv, KL);
#pragma unroll
      for (int c = 0; c < KL; c++) otile[(c * BM + lrow) * OS + cbase + j] = o.c[c];
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(NEPI * 32) : "memory");
    for (int e = tid; e < BM * BN; e += NEPI * 32) {
      const int row = e / BN, col = e % BN;
      const int64_t gr = row0 + row, gc = col0 + col;
      if (gr >= P.m || gc >= P.l) continue;
      Exp<KL> o;
#pragma unroll
      for (int c = 0; c < KL; c++) o.c[c] = otile[(c * BM + row) * OS + col];
      if (P.mode == 0) {
        stexp_<KL>(P.C.re + gr * P.C.ld + gc, P.C.ps, o);
      } else {
        // cmatrix.py:153 / 166-168 and lu.py:158-161, elementwise in the
        // reference's order (mat_add_k with sign -1 == exp_sub)
        const Exp<KL> t1 = ldexp_<KL>(P.T1.re + gr * P.T1.ld + gc, P.T1.ps);
        const Exp<KL> t2 = ldexp_<KL>(P.T2.re + gr * P.T2.ld + gc, P.T2.ps);
        Exp<KL> re = exp_sub(t1, t2), im;
        if (P.mode == 3) {
          im = exp_sub(exp_sub(o, t1), t2);  // (T3 - T1) - T2, o = T3
        } else {
          im = exp_add(ldexp_<KL>(P.T3.re + gr * P.T3.ld + gc, P.T3.ps), o);  // ir + ri
        }
        const int64_t off = gr * P.Cc.ld + gc;
        if (P.epi) {
          re = exp_sub(ldexp_<KL>(P.Cc.re + off, P.Cc.ps), re);
          im = exp_sub(ldexp_<KL>(P.Cc.im + off, P.Cc.ps), im);
        }
        stexp_<KL>(P.Cc.re + off, P.Cc.ps, re);
        stexp_<KL>(P.Cc.im + off, P.Cc.ps, im);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CN > 1) cluster_sync();  // no peer still signals / writes into this CTA
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TCOLS));
  }
}

// Fused ozaki_split (ozaki.py:79-108) of one operand, straight to digit
// slices.  A CTA owns NL grid lines (rows of the left operand, columns of the
// right one); their k-limb residuals stay in shared memory for all d steps:
//   mu = max |r0| per line, (f, ex) = frexp(mu), S = 2^ex 2^(53-width),
//   part = (r0 + S) - S, r0 -= part, renorm the limbs (renorm_planes),
//   scale = 2^(ex - width), I = part / scale -> NSL balanced digits.
// Each element sees exactly the reference's operation sequence, so parts and
// grids are bit-identical to ozaki_split's.
// src element (r, t): trans == 0 -> src[r*ld + t] (left), src[t*ld + r]
// (right).  Loads are coalesced along the contiguous index; the compute phase
// gives thread (line tl = tid % NL, tt = tid / NL) the 16-deep K groups
// tt, tt + 256/NL, ... of its line (one int4 store per digit slice); lines are
// padded to an odd stride in shared memory (conflict-free).
template <int KL>
__global__ void __launch_bounds__(256) split_lines_kernel(const double* src, int64_t ld, int64_t ps,
                                                          int trans, int64_t R, int64_t n, int NL,
                                                          int d, int width, int shift,
                                                          int8_t* out, int64_t Rp, int64_t Kp,
                                                          int TR, int stackB, double* scale) {
  extern __shared__ double res[];  // [KL][NL][n | 1]
  __shared__ double red[256];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * NL;
  const int64_t ls = n | 1;  // odd line stride (doubles)
  const int64_t cs = ls * NL;
  for (int64_t idx = tid; idx < (int64_t)NL * n; idx += 256) {
    const int64_t line = trans ? idx % NL : idx / n, t = trans ? idx / NL : idx % n;
    const int64_t r = r0 + line;
#pragma unroll
    for (int c = 0; c < KL; c++)
      res[c * cs + line * ls + t] =
          r < R ? (trans ? src[c * ps + t * ld + r] : src[c * ps + r * ld + t]) : 0.0;
  }
  __syncthreads();
  const int TPL = 256 / NL;  // threads per line
  const int tl = tid % NL, tt = tid / NL;
  const int64_t r = r0 + tl;
  const int64_t kch = Kp / 16, slice = Rp * Kp;
  const int64_t sstride = stackB ? (int64_t)TR * 16 : slice;
  const int64_t gstride = stackB ? (int64_t)NSL * TR * 16 : (int64_t)TR * 16;
  const long long mask = (1ll << shift) - 1, half = 1ll << (shift - 1);
  const double shiftS = ldexp(1.0, 53 - width);
  const int64_t ng = (n + 15) / 16;
  double* line0 = res + tl * ls;
  for (int p = 0; p < d; p++) {
    double m = 0.0;
    for (int64_t g = tt; g < ng; g += TPL)
#pragma unroll
      for (int i = 0; i < 16; i++)
        if (g * 16 + i < n) m = fmax(m, fabs(line0[g * 16 + i]));
    red[tid] = m;
    __syncthreads();
    // max over the TPL threads of each line (they sit at stride NL)
    if (tt == 0) {
      for (int w = 1; w < TPL; w++) m = fmax(m, red[tl + w * NL]);
      red[tl] = m;  // (slots >= NL are only read above: no race)
    }
    __syncthreads();
    m = red[tl];
    __syncthreads();  // red reused next step
    int ex = 0;
    frexp(m, &ex);
    const double w = ldexp(1.0, ex);
    const double S = __dmul_rn(w, shiftS);
    const int es = ex - width;  // scale = ldexp(w, -width) = 2^es
    if (tt == 0 && r < R) scale[(int64_t)p * R + r] = ldexp(w, -width);
    if (r < R) {
      int8_t* o = out + (int64_t)p * NSL * slice + ((r / TR) * kch) * gstride + (r % TR) * 16;
      for (int64_t g = tt; g < ng; g += TPL) {
        union {
          int8_t b[16];
          int4 v;
        } d0, d1, d2;
#pragma unroll
        for (int i = 0; i < 16; i++) {
          const int64_t t = g * 16 + i;
          long long I = 0;
          if (t < n) {
            const double x0 = line0[t];
            const double pt = __dsub_rn(__dadd_rn(x0, S), S);
            double buf[KL];
            buf[0] = __dsub_rn(x0, pt);
#pragma unroll
            for (int c = 1; c < KL; c++) buf[c] = line0[c * cs + t];
            Exp<KL> e = renorm<KL, KL>(buf, KL);
#pragma unroll
            for (int c = 0; c < KL; c++) line0[c * cs + t] = e.c[c];
            I = __double2ll_rn(ldexp(pt, -es));  // exact: pt is a multiple of 2^es
          }
          // balanced signed digits: I = a0 2^(2b) + a1 2^b + a2, a1, a2 in
          // [-2^(b-1), 2^(b-1)), |a0| <= 2^(w-2b) + 1 -- all s8
          const long long a2 = ((I + half) & mask) - half;
          const long long I1 = (I - a2) >> shift;
          const long long a1 = ((I1 + half) & mask) - half;
          d0.b[i] = (int8_t)((I1 - a1) >> shift);
          d1.b[i] = (int8_t)a1;
          d2.b[i] = (int8_t)a2;
        }
        int8_t* og = o + g * gstride;
        *reinterpret_cast<int4*>(og) = d0.v;
        *reinterpret_cast<int4*>(og + sstride) = d1.v;
        *reinterpret_cast<int4*>(og + 2 * sstride) = d2.v;
      }
    }
    __syncthreads();
  }
}

unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

template <int KL, int CN, int SB>
void launch_cn(const Params& P, cudaStream_t st, double ops) {
  using T = Tile<KL>;
  static unsigned long long attr = 0;
  auto kern = ozaki_tc_kernel<KL, CN, SB>;
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    if (CN > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = CN == 1 ? dim3((unsigned)((P.Lp / T::BN) * (P.Mp / BM)))
                        : dim3((unsigned)(P.Lp / T::BN), (unsigned)(P.Mp / BM));
  cfg.blockDim = dim3(Epi<KL>::NTHR);
  cfg.dynamicSmemBytes = T::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int tok = prof_begin(PC_GEMM, ops, st);
  cudaLaunchKernelEx(&cfg, kern, P);
  prof_end(tok, st);
  check_launch("ozaki_tc_kernel");
}

// cluster size along the column tiles (A-tile multicast), MPC_OZAKI_CLUSTER
inline int cluster_n() {
  static int cn = [] {
    const char* e = getenv("MPC_OZAKI_CLUSTER");
    int v = e ? atoi(e) : 1;  // multicast measured no faster at LU shapes (K = 512)
    return v == 2 ? 2 : 1;
  }();
  return cn;
}

template <int KL>
void launch(const Params& P, cudaStream_t st, double ops) {
  switch (cluster_n()) {
    case 2:
      if (P.shift == 7) launch_cn<KL, 2, 7>(P, st, ops); else launch_cn<KL, 2, 8>(P, st, ops);
      break;
    default:
      if (P.shift == 7) launch_cn<KL, 1, 7>(P, st, ops); else launch_cn<KL, 1, 8>(P, st, ops);
      break;
  }
}

// INT8 tensor-core issue-rate microbenchmark (the roofline denominator of
// the Ozaki kernel): one CTA per SM, one thread issuing back-to-back
// tcgen05.mma.kind::i8 M=128 N=256 K=32 from a resident 12 KB smem tile into
// two TMEM accumulators; int8 ops = 2 * 128 * 256 * 32 per MMA.
__global__ void __launch_bounds__(128, 1) int8_peak_kernel(int iters, int* sink, int ncols = 256) {
  __shared__ __align__(128) int8_t tile[BM * 32 + 256 * 32];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < (BM * 32 + 256 * 32) / 4; i += blockDim.x)
    reinterpret_cast<int*>(tile)[i] = 0x01010101 * (i & 3);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x < 32) {
    const uint32_t s = smem_u32(tile);
    const uint32_t hi = (128u >> 4) | (1u << 14);
    const uint64_t ad = ((uint64_t)hi << 32) | (((uint32_t)(BM * 16) >> 4) << 16) | ((s >> 4) & 0x3FFFu);
    const uint64_t bd = ((uint64_t)hi << 32) | (((uint32_t)(256 * 16) >> 4) << 16) |
                        (((s + BM * 32) >> 4) & 0x3FFFu);
    const uint32_t ID = make_idesc(ncols, true, true);
    if (elect_one()) {
      for (int it = 0; it < iters; it++) mma_i8(tmem + (uint32_t)((it & 1) * 256), ad, bd, ID, 1u);
      mma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (threadIdx.x == 0 && iters < 0) sink[0] = (int)tmem;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TCOLS));
  }
}

}  // namespace otc

bool ozaki_tc_enabled() {
  const char* e = getenv("MPC_OZAKI_GEMM");
  return !(e && strcmp(e, "dgemm") == 0);
}

bool ozaki_tc_rgemm(int k, int64_t m, int64_t n, int64_t l, View A, View B, View C, int d,
                    const std::vector<std::pair<int, int>>& pairs, int width, cudaStream_t st,
                    const OzCombine* cb) {
  using namespace otc;
  if (k < 2 || k > 4 || m <= 0 || l <= 0 || n <= 0) return false;
  if ((int)pairs.size() > MAXPAIRS || d > 255) return false;
  int shift;
  double gmax;
  if (width <= 20) {
    shift = 7;
    gmax = 12416.0;  // largest |G_s| term per k: 65*64*2 + 64*64
  } else if (width <= 22) {
    shift = 8;
    gmax = 33024.0;  // 65*128*2 + 128*128
  } else {
    return false;
  }
  if (gmax * (double)n >= 2147483648.0) return false;
  if (sizeof(double) * (size_t)k * (size_t)(n | 1) > 200 * 1024) return false;
  const int BN = k == 2 ? Tile<2>::BN : Tile<3>::BN;
  const int64_t LT = (int64_t)BN * cluster_n();  // column tiles come in whole clusters
  const int64_t Mp = (m + BM - 1) / BM * BM, Lp = (l + LT - 1) / LT * LT,
                Kp = (n + BKB - 1) / BKB * BKB;
  const size_t bytes_a = (size_t)d * NSL * Mp * Kp, bytes_b = (size_t)d * NSL * Lp * Kp;
  const size_t bytes_s = sizeof(double) * (size_t)d * (size_t)(m + l);
  int8_t* buf = nullptr;
  retain_pool();
  if (cudaMallocAsync((void**)&buf, bytes_a + bytes_b + bytes_s, st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaMemsetAsync(buf, 0, bytes_a + bytes_b, st);
  int8_t* sa = buf;
  int8_t* sb = buf + bytes_a;
  double* sca = reinterpret_cast<double*>(buf + bytes_a + bytes_b);
  double* scb = sca + (int64_t)d * m;
  int tok = prof_begin(PC_OTHER, 0.0, st);
  auto split = [&](auto kl, const double* src, int64_t ld, int64_t ps, int trans, int64_t R,
                   int8_t* out, int64_t Rp, int TR, double* sc) {
    const int stackB = trans;  // right operand: slices stacked per K chunk
    constexpr int KL = decltype(kl)::value;
    static unsigned long long attr = 0;
    if (first_on_device(attr))
      cudaFuncSetAttribute(split_lines_kernel<KL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
    int NL = 16;  // lines per CTA: as many as fit 200 KB of residual
    while (NL > 1 && (size_t)NL * (size_t)(n | 1) * KL * 8 > SPLIT_SMEM_CAP) NL /= 2;
    const size_t smem = (size_t)NL * (size_t)(n | 1) * KL * 8;
    split_lines_kernel<KL><<<(unsigned)((R + NL - 1) / NL), 256, smem, st>>>(
        src, ld, ps, trans, R, n, NL, d, width, shift, out, Rp, Kp, TR, stackB, sc);
  };
  switch (k) {
    case 2:
      split(std::integral_constant<int, 2>{}, A.re, A.ld, A.ps, 0, m, sa, Mp, BM, sca);
      split(std::integral_constant<int, 2>{}, B.re, B.ld, B.ps, 1, l, sb, Lp, BN, scb);
      break;
    case 3:
      split(std::integral_constant<int, 3>{}, A.re, A.ld, A.ps, 0, m, sa, Mp, BM, sca);
      split(std::integral_constant<int, 3>{}, B.re, B.ld, B.ps, 1, l, sb, Lp, BN, scb);
      break;
    default:
      split(std::integral_constant<int, 4>{}, A.re, A.ld, A.ps, 0, m, sa, Mp, BM, sca);
      split(std::integral_constant<int, 4>{}, B.re, B.ld, B.ps, 1, l, sb, Lp, BN, scb);
      break;
  }
  prof_end(tok, st);
  check_launch("ozaki split_lines_kernel");
  Params P;
  memset(&P, 0, sizeof(P));
  P.sa = sa;
  P.sb = sb;
  P.scale_a = sca;
  P.scale_b = scb;
  P.m = m;
  P.l = l;
  P.Mp = Mp;
  P.Lp = Lp;
  P.Kp = Kp;
  P.npairs = (int)pairs.size();
  P.shift = shift;
  P.C = C;
  if (cb) {
    P.mode = cb->mode;
    P.epi = cb->epi;
    P.T1 = cb->T1;
    P.T2 = cb->T2;
    P.T3 = cb->T3;
    P.Cc = cb->Cc;
  }
  for (size_t i = 0; i < pairs.size(); i++) {
    P.pp[i] = (unsigned char)pairs[i].first;
    P.pq[i] = (unsigned char)pairs[i].second;
  }
  const double ops = 2.0 * NSL * NSL * (double)pairs.size() * (double)m * (double)n * (double)l;
  switch (k) {
    case 2: launch<2>(P, st, ops); break;
    case 3: launch<3>(P, st, ops); break;
    default: launch<4>(P, st, ops); break;
  }
  cudaFreeAsync(buf, st);
  return true;
}

}  // namespace mpc

// MMA N for the microbenchmark: 256 (the roofline denominator) unless
// MPC_INT8_PEAK_N says otherwise (diagnostics: the Ozaki kernel issues N = 144
// / 96 MMAs, tools/probe_int8_n.py)
static int int8_peak_n() {
  const char* e = getenv("MPC_INT8_PEAK_N");
  const int v = e ? atoi(e) : 256;
  return (v >= 16 && v <= 256 && v % 16 == 0) ? v : 256;
}

extern "C" double mpc_int8_peak(int iters, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int ncols = int8_peak_n();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mpc::otc::int8_peak_kernel<<<sms, 128, 0, st>>>(iters / 10 + 1, nullptr, ncols);  // warm-up
  cudaEventRecord(a, st);
  mpc::otc::int8_peak_kernel<<<sms, 128, 0, st>>>(iters, nullptr, ncols);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (cudaGetLastError() != cudaSuccess || t <= 0.f) return -1.0;
  const double ops = (double)sms * (double)iters * 2.0 * mpc::otc::BM * (double)ncols * 32.0;
  return ops / (t * 1e-3);  // INT8 tensor-core ops per second
}
