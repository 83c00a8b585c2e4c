// Instantiates the K=2 (2-component expansion) kernels and launchers.
#include "kernels.cuh"
#include "ops.h"

namespace mpc {
const OpsTable* ops_k2() {
  using O = Ops<2>;
  static const OpsTable t{2,          O::rgemm,   O::cgemm,  O::supdate,  O::mat_add,
                          O::renorm_planes, O::laswp, O::trsm, O::panel_rec, O::lu_panel,
                          O::getrf,    O::getrs};
  return &t;
}
}  // namespace mpc
