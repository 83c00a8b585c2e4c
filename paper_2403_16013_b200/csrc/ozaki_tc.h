// ozaki_tc.h -- Ozaki-scheme part products on the sm_100a INT8 tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).  See ozaki_tc.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

namespace mpc {

struct View;

// The pair loop of rgemm_ozaki (ozaki.py:142-158) for split operands:
// every scheduled part product A_p B_q is formed EXACTLY from INT8 digit
// slices on the tensor cores (int32 TMEM accumulators, recombined in int64),
// accumulated into C in schedule order with the reference's acc_plane, then
// renormalized (renorm_planes) -- all in one kernel.  parts_a: [d][m][n],
// parts_b: [d][n][l] (row-major binary64, as ozaki_split produces them),
// scale_a: [d][m] row grids, scale_b: [d][l] column grids.  C: m x l, k
// planes, overwritten.  Returns false (nothing launched) when the width /
// inner dimension fall outside the exact int32 slicing regime; the caller
// then uses the binary64 GEMM seam.
bool ozaki_tc_gemm(int k, int64_t m, int64_t n, int64_t l, const double* parts_a,
                   const double* parts_b, const double* scale_a, const double* scale_b, int d,
                   const std::vector<std::pair<int, int>>& pairs, int width, View C,
                   cudaStream_t st);

// rgemm_ozaki (ozaki.py:124-159) end to end on the tensor-core path: the
// fused split (ozaki_split of A by rows, of B by columns, straight to digit
// slices) and ozaki_tc_gemm's kernel.  A: m x n, B: n x l, C: m x l views
// (k planes).  Returns false when outside the supported regime.
bool ozaki_tc_rgemm(int k, int64_t m, int64_t n, int64_t l, View A, View B, View C, int d,
                    const std::vector<std::pair<int, int>>& pairs, int width, cudaStream_t st);

// MPC_OZAKI_GEMM=dgemm forces the cuBLAS binary64 seam (A/B comparisons)
bool ozaki_tc_enabled();

}  // namespace mpc
