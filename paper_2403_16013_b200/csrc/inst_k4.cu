// Instantiates the K=4 (4-component expansion) kernels and launchers.
#include "kernels.cuh"
#include "ops.h"

namespace mpc {
const OpsTable* ops_k4() {
  using O = Ops<4>;
  static const OpsTable t{4,          O::rgemm,   O::cgemm,  O::supdate,  O::mat_add,
                          O::renorm_planes, O::laswp, O::trsm, O::panel_rec, O::lu_panel,
                          O::getrf,    O::getrs};
  return &t;
}
}  // namespace mpc
