// Instantiates the K=3 (3-component expansion) kernels and launchers.
#include "kernels.cuh"
#include "ops.h"

namespace mpc {
const OpsTable* ops_k3() {
  using O = Ops<3>;
  static const OpsTable t{3,          O::rgemm,   O::cgemm,  O::supdate,  O::mat_add,
                          O::renorm_planes, O::laswp, O::trsm, O::panel_rec, O::lu_panel,
                          O::getrf,    O::getrs};
  return &t;
}
}  // namespace mpc
