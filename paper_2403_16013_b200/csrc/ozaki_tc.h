// ozaki_tc.h -- Ozaki-scheme part products on the sm_100a INT8 tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).  See ozaki_tc.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace mpc {


// rgemm_ozaki (ozaki.py:124-159) end to end on the tensor-core path: the
// fused split (ozaki_split of A by rows, of B by columns, straight to digit
// slices) and ozaki_tc_gemm's kernel.  A: m x n, B: n x l, C: m x l views
// (k planes).  Returns false when outside the supported regime.
// cb != nullptr fuses the complex composition into the epilogue of the
// LAST real product of a 3M / 4M cgemm (C is then unused): cb->mode 3:
// Re = T1 - T2, Im = (T3' - T1) - T2 with T3' this product; mode 4:
// Re = T1 - T2, Im = T3 + this product; epi 1: Cc -= (Re, Im), else Cc = ...
struct OzCombine {
  int mode, epi;
  View T1, T2, T3, Cc;
};
bool ozaki_tc_rgemm(int k, int64_t m, int64_t n, int64_t l, View A, View B, View C, int d,
                    const std::vector<std::pair<int, int>>& pairs, int width, cudaStream_t st,
                    const OzCombine* cb = nullptr);

// MPC_OZAKI_GEMM=dgemm forces the cuBLAS binary64 seam (A/B comparisons)
bool ozaki_tc_enabled();

}  // namespace mpc
