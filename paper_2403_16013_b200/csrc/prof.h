// prof.h -- launch accounting shared by all translation units: a launch
// counter (always on) and optional per-class CUDA-event timing of every
// launch (mpc_prof_enable), used by bench.py for the roofline figures.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mpc {

enum ProfClass {
  PC_GEMM = 0,   // fused complex GEMM (trailing update / cgemm), MODE_G3/G4/REAL
  PC_SUPD = 1,   // chained "S" updates inside panel and TRSM
  PC_PANEL = 2,  // pivot search + column steps
  PC_TRSM = 3,   // TRSM diagonal blocks
  PC_LASWP = 4,  // row interchanges
  PC_OTHER = 5,  // elementwise, misc
  PC_SOLVE = 6,  // triangular solves (getrs)
  PC_N = 7
};

// Called around every kernel launch.  `ops` is the algorithmic FP64 op count
// of the launch (op model v1).  Returns a token for prof_end.
int prof_begin(int cls, double ops, cudaStream_t st);
void prof_end(int token, cudaStream_t st);

}  // namespace mpc
