// k = 6 verification kernels (see inst_hik.cuh)
#define MPC_HIK_K 6
#define MPC_HIK_FN ops_k6
#include "inst_hik.cuh"
