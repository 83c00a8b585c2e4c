// The verification kernels at k = 5, 6, 8: the real
// GEMM, the 3M / 4M complex GEMM, mat_add and renorm_planes -- what
// lu.reconstruction_error (k + 2, lu.py:236-250), the backward-error probe
// and the reference's k = 8 right-hand side / matmul check
// (bench.py:199-213, 336-348; REFERENCE_K = 8) call.  No LU machinery at
// these k.  One translation unit per k includes this with MPC_HIK_K set.
#include "kernels.cuh"
#include "ops.h"

#ifndef MPC_HIK_K
#error "define MPC_HIK_K before including inst_hik.cuh"
#endif

namespace mpc {

const OpsTable* MPC_HIK_FN() {
  using O = Ops<MPC_HIK_K>;
  static const OpsTable t{MPC_HIK_K, O::rgemm,  O::cgemm, nullptr, O::mat_add,
                          O::renorm_planes, nullptr, nullptr, nullptr, nullptr,
                          nullptr, nullptr};
  return &t;
}

}  // namespace mpc
