// ops.h -- per-K operation table (one translation unit per K instantiates
// the templated kernels; abi.cu dispatches on k at run time).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mpc {

struct View;
struct PanelWs;

struct OpsTable {
  int k;
  void (*rgemm)(int64_t m, int64_t n, int64_t l, View a, View b, View c, cudaStream_t st);
  void (*cgemm)(bool use3m, int64_t m, int64_t n, int64_t l, View a, View b, View c, int epi,
                cudaStream_t st, const int64_t* status);
  void (*supdate)(bool use3m, int64_t m, int64_t kb, int64_t l, View L, View U, View C,
                  cudaStream_t st, const int64_t* status);
  void (*mat_add)(int64_t rows, int64_t cols, View a, View b, View c, double sign,
                  cudaStream_t st);
  void (*renorm_planes)(int64_t rows, int64_t cols, View a, cudaStream_t st);
  void (*laswp)(View A, int64_t col0, int64_t ncols, const int64_t* piv, int64_t r0, int64_t r1,
                cudaStream_t st, const int64_t* status);
  void (*trsm)(bool use3m, int64_t kb, int64_t M, View L, View X, cudaStream_t st,
               const int64_t* status);
  void (*panel_rec)(bool use3m, View A, int64_t n, int64_t c0, int64_t w, int64_t* piv,
                    PanelWs ws, cudaStream_t st);
  void (*lu_panel)(bool use3m, View A, int64_t n, int64_t jb, int64_t kw, int64_t* piv,
                   PanelWs ws, cudaStream_t st);
  void (*getrf)(bool use3m, View A, int64_t n, int64_t Kp, int64_t* piv, PanelWs ws,
                cudaStream_t st);
  void (*getrs)(bool use3m, View F, int64_t n, const int64_t* piv, double* br, double* bi,
                int phases, cudaStream_t st);
};

const OpsTable* ops_k2();
const OpsTable* ops_k3();
const OpsTable* ops_k4();
// verification only (inst_hik.cuh): rgemm, 3M / 4M cgemm, mat_add, renorm_planes
const OpsTable* ops_k5();
const OpsTable* ops_k6();
const OpsTable* ops_k8();

}  // namespace mpc
