// Instantiates the k = 5 and k = 6 kernels that serve only verification at
// k + 2 components (lu.reconstruction_error at k + 2,
// the backward-error probe for TD / QD factors): the real GEMM, the 4M
// complex GEMM, mat_add and renorm_planes.  No LU machinery at these k.
#include "kernels.cuh"
#include "ops.h"

namespace mpc {
namespace {

template <int K>
void cgemm_4m_only(bool use3m, int64_t m, int64_t n, int64_t l, View a, View b, View c, int epi,
                   cudaStream_t st, const int64_t* status) {
  if (use3m) throw LaunchError{"k = 5, 6 (verification kernels): 4M only"};
  GemmArgs g{m, n, l, a, b, c, epi, status};
  Ops<K>::template gemm_launch<MODE_G4>(g, st, PC_OTHER, 0.0);
}

template <int K>
const OpsTable* table() {
  using O = Ops<K>;
  static const OpsTable t{K,       O::rgemm, cgemm_4m_only<K>, nullptr, O::mat_add,
                          O::renorm_planes, nullptr, nullptr, nullptr, nullptr,
                          nullptr, nullptr};
  return &t;
}

}  // namespace

const OpsTable* ops_k5() { return table<5>(); }
const OpsTable* ops_k6() { return table<6>(); }

}  // namespace mpc
