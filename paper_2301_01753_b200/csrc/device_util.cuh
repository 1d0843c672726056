// Device-side helpers shared by the leapfrog and Yee kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.hpp"

namespace sfeec_b200 {

#define SFEEC_CUDA(call)                                                               \
  do {                                                                                 \
    cudaError_t err_ = (call);                                                         \
    if (err_ != cudaSuccess)                                                           \
      throw ::sfeec_b200::Error(err_ == cudaErrorMemoryAllocation ? SFEEC_ENOMEM       \
                                                                  : SFEEC_ECUDA,       \
                                std::string(#call) + ": " + cudaGetErrorString(err_)); \
  } while (0)

#define SFEEC_LAUNCH_CHECK() SFEEC_CUDA(cudaGetLastError())

// Programmatic dependent launch (PDL). A kernel launched with launch_pdl may
// start while the previous kernel in the stream is still finishing: it runs
// its prologue (barrier init, index math), then pdl_wait() blocks until the
// previous grid has completed and its writes are visible. pdl_trigger() lets
// the next PDL kernel be scheduled once every CTA of this grid has issued it
// (or exited). Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  if (!pdl) {
    kern<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SFEEC_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// One CTA-resident persistent grid worth of blocks for grid-stride kernels:
// 148 SMs x 8.
constexpr int kReduceBlocks = 148 * 8;
constexpr int kReduceThreads = 256;

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    n = count;
    if (count) SFEEC_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) SFEEC_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  }
  void zero(cudaStream_t s) {
    if (n) SFEEC_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
  }
};

// an owned non-blocking stream
struct Stream {
  cudaStream_t s = nullptr;
  Stream() { SFEEC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
};

// device CSR (int64 row pointers), produced by the device assembly
struct DevCSR {
  int64_t rows = 0, cols = 0, nnz = 0;
  DevBuf<int64_t> rp;
  DevBuf<int32_t> ci;
  DevBuf<double> val;
};

// Checks there is a usable device and makes `device` current.
void select_device(int device);

// Deterministic reductions (fixed grid, fixed combine order): dot(x, y) and
// max |x| over n doubles, result to host.
double device_dot(const double* x, const double* y, int64_t n, double* partials,
                  cudaStream_t s);
double device_max_abs(const double* x, int64_t n, double* partials, cudaStream_t s);
double device_sumsq(const float* x, int64_t n, double* partials, cudaStream_t s);

}  // namespace sfeec_b200
