// k = 8 verification kernels (see inst_hik.cuh)
#define MPC_HIK_K 8
#define MPC_HIK_FN ops_k8
#include "inst_hik.cuh"
