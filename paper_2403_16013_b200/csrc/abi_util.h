// abi_util.h -- shared helpers of the C-ABI translation units (abi.cu,
// ozaki.cu): error reporting, pointer classification, host staging, the
// pivot-reduction workspace.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mpc_b200.h"
#include "kernels.cuh"
#include "ops.h"

namespace mpcabi {

extern thread_local std::string g_err;

inline int fail(const std::string& msg) {
  g_err = msg;
  return MPC_ERR;
}

struct CudaError {
  std::string what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
}

inline const mpc::OpsTable* table_for(int k) {
  switch (k) {
    case 2: return mpc::ops_k2();
    case 3: return mpc::ops_k3();
    case 4: return mpc::ops_k4();
    case 5: return mpc::ops_k5();  // verification kernels (GEMM / elementwise only)
    case 6: return mpc::ops_k6();
    case 8: return mpc::ops_k8();  // REFERENCE_K (bench.py:46)
    default: return nullptr;
  }
}

// 0: null, 1: host, 2: device
inline int ptr_kind(const void* p, int* device) {
  if (p == nullptr) return 0;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    if (device) *device = a.device;
    return 2;
  }
  return 1;
}

inline int64_t extent(int k, int64_t rows, int64_t cols, int64_t ld, int64_t ps) {
  if (rows <= 0 || cols <= 0) return 0;
  return (int64_t)(k - 1) * ps + (rows - 1) * ld + cols;
}

// Maps every pointer of one call to device memory.  All-device calls pass
// through untouched; all-host calls are staged (H2D before, D2H after, then
// the stream is synchronised).
class Stager {
 public:
  explicit Stager(cudaStream_t st) : st_(st) {}
  ~Stager() {
    for (auto& r : regs_)
      if (r.dev) cudaFreeAsync(r.dev, st_);
  }
  bool classify(std::initializer_list<const void*> ptrs) {
    int kinds = 0;
    int dev = -1;
    for (const void* p : ptrs) {
      int d = -1;
      int kd = ptr_kind(p, &d);
      if (kd == 0) continue;
      kinds |= (1 << kd);
      if (kd == 2) dev = d;
    }
    if (kinds == ((1 << 1) | (1 << 2))) {
      g_err = "mixed host and device pointers in one call";
      return false;
    }
    host_ = (kinds == (1 << 1));
    if (!host_ && dev >= 0) ck(cudaSetDevice(dev), "cudaSetDevice");
    return true;
  }
  bool host() const { return host_; }
  template <typename T>
  T* map(T* p, int64_t nelem, bool in, bool out) {
    if (!host_ || p == nullptr || nelem <= 0) return p;
    Region r{(void*)p, (size_t)nelem * sizeof(T), out, nullptr};
    mpc::retain_pool();
    ck(cudaMallocAsync(&r.dev, r.bytes, st_), "cudaMallocAsync");
    regs_.push_back(r);
    if (in) ck(cudaMemcpyAsync(r.dev, p, r.bytes, cudaMemcpyHostToDevice, st_), "H2D");
    return (T*)r.dev;
  }
  void finish() {
    if (host_) {
      for (auto& r : regs_)
        if (r.out) ck(cudaMemcpyAsync(r.host, r.dev, r.bytes, cudaMemcpyDeviceToHost, st_), "D2H");
    }
    ck(cudaGetLastError(), "kernel launch");
    if (host_) ck(cudaStreamSynchronize(st_), "cudaStreamSynchronize");
  }

 private:
  struct Region {
    void* host;
    size_t bytes;
    bool out;
    void* dev;
  };
  cudaStream_t st_;
  bool host_ = false;
  std::vector<Region> regs_;
};

// pinned (page-locked) host memory: async copies from it do not block the host
inline bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host-buffer LU (mpc_getrf / mpc_getrf_ozaki on pinned host factors): the
// input goes host-to-device in column blocks on a copy stream (boundaries
// K, 2K, then 4K wide -- the first panel, the narrow update and step 0's
// update chunks), the LU waits per block (need), and each row block is
// copied back as soon as its step has finished it (rows_done; later steps
// only touch rows below it).  MPC_HOST_OVERLAP=0 falls back to staged
// copies; MPC_H2D_WHOLE=1 copies the input as one 1-D block per plane (A/B).
class HostOverlap {
 public:
  int64_t chunk = 0;
  static bool usable(const Stager& sg, int64_t n, const void* re, const void* im) {
    static const bool on = [] {
      const char* e = getenv("MPC_HOST_OVERLAP");
      return !(e && e[0] == '0');
    }();
    return on && sg.host() && n > 0 && is_pinned(re) && is_pinned(im);
  }
  void start(cudaStream_t st, double* dr, double* di, double* hr, double* hi, int k, int64_t n,
             int64_t K) {
    dr_ = dr;
    di_ = di;
    hr_ = hr;
    hi_ = hi;
    k_ = k;
    n_ = n;
    chunk = 4 * K;
    ck(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming), "cudaEventCreate");
    // the copy stream starts after the allocations enqueued on st
    ck(cudaEventRecord(ev_, st), "cudaEventRecord");
    ck(cudaStreamWaitEvent(cs_, ev_, 0), "cudaStreamWaitEvent");
    static const bool whole = [] {
      const char* e = getenv("MPC_H2D_WHOLE");
      return e && e[0] == '1';
    }();
    const size_t pitch = sizeof(double) * (size_t)n;
    int64_t c = 0;
    while (c < n) {
      int64_t c1 = whole ? n : std::min(n, c + ((c < 2 * K) ? K : chunk));
      for (int q = 0; q < k; q++) {
        const size_t off = (size_t)q * n * n + (size_t)c;
        const size_t w = sizeof(double) * (size_t)(c1 - c);
        ck(cudaMemcpy2DAsync(dr + off, pitch, hr + off, pitch, w, (size_t)n,
                             cudaMemcpyHostToDevice, cs_), "H2D");
        ck(cudaMemcpy2DAsync(di + off, pitch, hi + off, pitch, w, (size_t)n,
                             cudaMemcpyHostToDevice, cs_), "H2D");
      }
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventRecord(e, cs_), "cudaEventRecord");
      lo_.push_back(c);
      blk_.push_back(e);
      c = c1;
    }
  }
  // st is about to touch columns [.., c1)
  static void need(void* ctx, int64_t c1, cudaStream_t st) {
    auto* s = (HostOverlap*)ctx;
    while (s->waited_ < s->blk_.size() && s->lo_[s->waited_] < c1)
      ck(cudaStreamWaitEvent(st, s->blk_[s->waited_++], 0), "cudaStreamWaitEvent");
  }
  // rows [r0, r1) are final once the work enqueued on st so far completes
  static void rows_done(void* ctx, int64_t r0, int64_t r1, cudaStream_t st) {
    auto* s = (HostOverlap*)ctx;
    ck(cudaEventRecord(s->ev_, st), "cudaEventRecord");
    ck(cudaStreamWaitEvent(s->cs_, s->ev_, 0), "cudaStreamWaitEvent");
    const size_t bytes = sizeof(double) * (size_t)(r1 - r0) * (size_t)s->n_;
    for (int q = 0; q < s->k_; q++) {
      const size_t off = (size_t)q * s->n_ * s->n_ + (size_t)r0 * s->n_;
      ck(cudaMemcpyAsync(s->hr_ + off, s->dr_ + off, bytes, cudaMemcpyDeviceToHost, s->cs_), "D2H");
      ck(cudaMemcpyAsync(s->hi_ + off, s->di_ + off, bytes, cudaMemcpyDeviceToHost, s->cs_), "D2H");
    }
  }
  // order st (the staged buffers are freed on it) after the copy stream
  void join(cudaStream_t st) {
    ck(cudaEventRecord(ev_, cs_), "cudaEventRecord");
    ck(cudaStreamWaitEvent(st, ev_, 0), "cudaStreamWaitEvent");
  }
  ~HostOverlap() {
    if (!cs_) return;
    cudaStreamSynchronize(cs_);
    for (auto e : blk_) cudaEventDestroy(e);
    cudaEventDestroy(ev_);
    cudaStreamDestroy(cs_);
  }

 private:
  cudaStream_t cs_ = nullptr;
  cudaEvent_t ev_ = nullptr;
  double *dr_ = nullptr, *di_ = nullptr, *hr_ = nullptr, *hi_ = nullptr;
  int k_ = 0;
  int64_t n_ = 0;
  std::vector<int64_t> lo_;
  std::vector<cudaEvent_t> blk_;
  size_t waited_ = 0;
};

// pivot-reduction workspace + status word, stream ordered
struct WsHolder {
  mpc::PanelWs ws{};
  cudaStream_t st;
  void* mem = nullptr;
  WsHolder(int k, int64_t n, cudaStream_t s) : st(s) {
    mpc::retain_pool();
    ck(cudaMallocAsync(&mem, mpc::panel_ws_bytes(k, n), st), "cudaMallocAsync(ws)");
    ws = mpc::panel_ws_carve(mem, k, n);
    ck(mpc::panel_ws_init(ws, st), "memset ws");
  }
  int64_t read_status() {
    int64_t h = -1;
    ck(cudaMemcpyAsync(&h, ws.status, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H status");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return h;
  }
  ~WsHolder() {
    if (mem) cudaFreeAsync(mem, st);
  }
};

// k = 2, 3, 4: every entry point; k = 5, 6 (the k + 2 verification
// kernels): mat_add, renorm_planes, rgemm and the 4M cgemm
inline bool bad_k(int k) { return k < 2 || k > 4; }
inline bool bad_k_gemm(int k) { return table_for(k) == nullptr; }
inline bool bad_method(int m) { return m != 3 && m != 4; }

#define MPC_TRY try {
#define MPC_CATCH                                                          \
  }                                                                        \
  catch (const mpcabi::CudaError& e) {                                     \
    return mpcabi::fail(e.what);                                           \
  }                                                                        \
  catch (const mpc::LaunchError& e) {                                      \
    return mpcabi::fail(std::string("launch failed: ") + e.what + ": " +   \
                        cudaGetErrorString(cudaGetLastError()));           \
  }                                                                        \
  catch (const std::exception& e) {                                        \
    return mpcabi::fail(e.what());                                         \
  }

}  // namespace mpcabi
