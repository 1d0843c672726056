// Device utilities: device selection and deterministic reductions.
#include "device_util.cuh"

namespace sfeec_b200 {

void select_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Error(SFEEC_ECUDA, "no CUDA device available (the sfeec_b200 kernels have no CPU "
                             "fallback)");
  if (device < 0 || device >= n) throw Error(SFEEC_EINVAL, "device index out of range");
  SFEEC_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SFEEC_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    throw Error(SFEEC_ECUDA, std::string("sfeec_b200 is built for sm_100a; device is ") +
                                 prop.name);
}

namespace {

template <int OP>  // 0: sum x*y, 1: max |x|, 2: sum x*x (float input)
__device__ __forceinline__ double combine(double a, double b) {
  return OP == 1 ? fmax(a, b) : a + b;
}

template <int OP, class T>
__global__ void __launch_bounds__(kReduceThreads)
    reduce_partial(const T* __restrict__ x, const T* __restrict__ y, int64_t n,
                   double* __restrict__ partials) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (OP == 0)
      v = (double)x[i] * (double)y[i];
    else if (OP == 1)
      v = fabs((double)x[i]);
    else
      v = (double)x[i] * (double)x[i];
    acc = combine<OP>(acc, v);
  }
  for (int o = 16; o > 0; o >>= 1) acc = combine<OP>(acc, __shfl_down_sync(0xffffffffu, acc, o));
  __shared__ double warp_acc[kReduceThreads / 32];
  if ((threadIdx.x & 31) == 0) warp_acc[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kReduceThreads / 32; ++w) t = combine<OP>(t, warp_acc[w]);
    partials[blockIdx.x] = t;
  }
}

template <int OP>
__global__ void reduce_final(double* partials, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t = combine<OP>(t, partials[i]);
    partials[n] = t;
  }
}

template <int OP, class T>
double run_reduce(const T* x, const T* y, int64_t n, double* partials, cudaStream_t s) {
  reduce_partial<OP, T><<<kReduceBlocks, kReduceThreads, 0, s>>>(x, y, n, partials);
  SFEEC_LAUNCH_CHECK();
  reduce_final<OP><<<1, 32, 0, s>>>(partials, kReduceBlocks);
  SFEEC_LAUNCH_CHECK();
  double out = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&out, partials + kReduceBlocks, sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  return out;
}

}  // namespace

double device_dot(const double* x, const double* y, int64_t n, double* partials,
                  cudaStream_t s) {
  return run_reduce<0, double>(x, y, n, partials, s);
}
double device_max_abs(const double* x, int64_t n, double* partials, cudaStream_t s) {
  return run_reduce<1, double>(x, x, n, partials, s);
}
double device_sumsq(const float* x, int64_t n, double* partials, cudaStream_t s) {
  return run_reduce<2, float>(x, x, n, partials, s);
}

}  // namespace sfeec_b200

extern "C" int sfeec_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
