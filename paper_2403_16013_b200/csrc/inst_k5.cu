// k = 5 verification kernels (see inst_hik.cuh)
#define MPC_HIK_K 5
#define MPC_HIK_FN ops_k5
#include "inst_hik.cuh"
