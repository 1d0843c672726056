// Sliced SpMV with the operator stream staged by bulk async copies
// (SFEEC_SELL_TMA=1; measured slower than k_sell_pipe, see sell_tma_enabled).
//
// k_sell_pipe keeps the next chunk's columns / values in registers, which
// caps the bytes in flight per SM (ncu: 72% of DRAM peak, long-scoreboard
// stalls). Here every warp owns a private ring of shared-memory stages; its
// lane 0 issues cp.async.bulk copies of the next stages' columns and values
// (mbarrier transaction counts) while the warp computes the current stage
// from shared memory, so the DRAM stream is decoupled from the gathers and
// the in-flight bytes are bounded by shared memory, not registers. A stage
// is a k-range of one slice (column-major inside the slice, so contiguous):
// a whole slice for the first-order Q (16 entries x 32 rows), ~1/19 of one
// for config 4's 300-wide rows; rows are summed in CSR order across stages.
#include <algorithm>
#include <cstdlib>

#include "spmv_kernels.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kTWarps = 16;               // warps per CTA (one CTA per SM)
constexpr int kTStages = 2;               // ring stages per warp
constexpr int kTSE = 512;                 // entries per stage (6 KB)
constexpr int kTStageBytes = kTSE * 12;   // int32 columns + fp64 values
struct StageInfo {                        // written by lane 0 before the copy
  int64_t row0;
  int32_t nr, k0, k1, w;
};
constexpr int kTSmem = kTWarps * kTStages * (kTStageBytes + 8 + (int)sizeof(StageInfo));

__device__ __forceinline__ uint32_t t_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void t_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra TWAIT_%=;\n}" ::"r"(t_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void t_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(t_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(t_u32(bar))
      : "memory");
}

// entries per lane of one stage of a slice with nr rows (a multiple of 4, so
// every stage starts 16-byte aligned)
__device__ __forceinline__ int stage_k(int nr) { return (kTSE / nr) & ~3; }

template <bool ACC>
__global__ void __launch_bounds__(kTWarps * 32, 1)
    k_sell_tma(int64_t n_slices, const int64_t* __restrict__ srow,
               const int64_t* __restrict__ sptr, const int32_t* __restrict__ sw,
               const int32_t* __restrict__ col, const double* __restrict__ val,
               const double* __restrict__ x, double* __restrict__ y, double alpha) {
  extern __shared__ __align__(128) unsigned char tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* mine = tsm + warp * kTStages * kTStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tsm + kTWarps * kTStages * kTStageBytes) +
                   warp * kTStages;
  StageInfo* info = reinterpret_cast<StageInfo*>(
                        tsm + kTWarps * kTStages * (kTStageBytes + 8)) + warp * kTStages;
  const int64_t tw = (int64_t)gridDim.x * kTWarps;
  // producer cursor (lane 0): slice ps at entry k pk; the metadata of the
  // warp's next slice is loaded one slice ahead (its latency hides behind a
  // whole slice of stages)
  int64_t ps = (int64_t)blockIdx.x * kTWarps + warp;
  int pk = 0;
  int64_t c_r0 = 0, c_ptr = 0, n_r0 = 0, n_r1 = 0, n_ptr = 0;
  int c_nr = 0, c_w = 0, n_w = 0;
  auto meta_load = [&](int64_t sl) {
    if (sl < n_slices) {
      n_r0 = srow[sl];
      n_r1 = srow[sl + 1];
      n_w = sw[sl];
      n_ptr = sptr[sl];
    }
  };
  auto meta_take = [&]() {
    c_r0 = n_r0;
    c_nr = (int)(n_r1 - n_r0);
    c_w = n_w;
    c_ptr = n_ptr;
  };
  if (lane == 0) {
    for (int i = 0; i < kTStages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(t_u32(&bars[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    meta_load(ps);
    meta_take();
    meta_load(ps + tw);
  }
  __syncwarp();
  // lane 0: issue the next stage into ring slot `slot`; false when done
  auto produce = [&](int slot) -> bool {
    if (ps >= n_slices) return false;
    const int nr = c_nr, w = c_w;
    const int kc = stage_k(nr);
    const int k1 = min(w, pk + kc);
    const int64_t e0 = c_ptr + (int64_t)pk * nr;
    const uint32_t cnt = (uint32_t)(((k1 - pk) * nr + 3) & ~3);
    StageInfo& si = info[slot];
    si.row0 = c_r0;
    si.nr = nr;
    si.k0 = pk;
    si.k1 = k1;
    si.w = w;
    unsigned char* buf = mine + slot * kTStageBytes;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(t_u32(&bars[slot])),
                 "r"(cnt * 12u)
                 : "memory");
    t_bulk(buf, col + e0, cnt * 4u, &bars[slot]);
    t_bulk(buf + kTSE * 4, val + e0, cnt * 8u, &bars[slot]);
    pk = k1;
    if (pk >= w) {
      ps += tw;
      pk = 0;
      meta_take();
      meta_load(ps + tw);
    }
    return true;
  };
  int issued = 0;
  if (lane == 0)
    for (int i = 0; i < kTStages; ++i)
      if (produce(i)) ++issued;
  issued = __shfl_sync(0xffffffffu, issued, 0);
  double acc = 0.0, y0 = 0.0;
  for (int i = 0; i < issued; ++i) {
    const int slot = i % kTStages;
    t_mbar_wait(&bars[slot], (uint32_t)(i / kTStages) & 1u);
    const StageInfo si = info[slot];
    const int32_t* sc = reinterpret_cast<const int32_t*>(mine + slot * kTStageBytes);
    const double* sv = reinterpret_cast<const double*>(mine + slot * kTStageBytes + kTSE * 4);
    if (lane < si.nr) {
      if (ACC && si.k0 == 0) y0 = y[si.row0 + lane];
      const int n = si.k1 - si.k0, nr = si.nr;
      const int32_t* cl = sc + lane;
      const double* vl = sv + lane;
      int k = 0;
      for (; k + 16 <= n; k += 16) {  // 16 gathers in flight per lane
        int c[16];
        double v[16], xv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          c[j] = cl[(k + j) * nr];
          v[j] = vl[(k + j) * nr];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) xv[j] = __ldg(x + c[j]);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc = fma(v[j], xv[j], acc);
      }
      for (; k < n; k += 4) {  // the tail, 4 at a time
        int c[4];
        double v[4], xv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          c[j] = k + j < n ? cl[(k + j) * nr] : -1;
          v[j] = k + j < n ? vl[(k + j) * nr] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) xv[j] = c[j] >= 0 ? __ldg(x + c[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c[j] >= 0) acc = fma(v[j], xv[j], acc);
      }
      if (si.k1 == si.w) {
        y[si.row0 + lane] = ACC ? fma(alpha, acc, y0) : acc;
        acc = 0.0;
      }
    }
    __syncwarp();
    if (lane == 0 && produce(slot)) ++issued;
    issued = __shfl_sync(0xffffffffu, issued, 0);
  }
}

}  // namespace

// SFEEC_SELL_TMA=1 selects this kernel. Off by default: measured on B200 at
// tet128 (K-Q, 237M nnz) 0.74-0.87 ms against 0.57-0.58 for k_sell_pipe,
// config 4 9.18 against 7.18 ms. ncu: 16 warps per SM (1 CTA, 197 KB of
// stages) leave the gathers' L2 latency exposed (long-scoreboard on the FMA
// chain) and DRAM at 39-62% of peak.
bool sell_tma_enabled() {
  const char* e = std::getenv("SFEEC_SELL_TMA");
  return e && std::atoi(e) == 1;
}

// the kernels' shared-memory opt-in, once per process (at operator build time,
// so that no attribute call happens inside a CUDA-graph capture)
void prepare_sell_tma() {
  static bool attr = false;
  if (attr) return;
  SFEEC_CUDA(cudaFuncSetAttribute(k_sell_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kTSmem));
  SFEEC_CUDA(cudaFuncSetAttribute(k_sell_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kTSmem));
  attr = true;
}

void launch_sell_tma(const DevOperator& a, const double* x, double* y, double alpha,
                     bool accumulate, cudaStream_t s) {
  prepare_sell_tma();
  const unsigned g = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(148, (a.n_slices + kTWarps - 1) / kTWarps));
  if (accumulate)
    k_sell_tma<true><<<g, kTWarps * 32, kTSmem, s>>>(a.n_slices, a.slice_row.p, a.slice_ptr.p,
                                                     a.slice_w.p, a.sell_col.p, a.sell_val.p, x,
                                                     y, alpha);
  else
    k_sell_tma<false><<<g, kTWarps * 32, kTSmem, s>>>(a.n_slices, a.slice_row.p, a.slice_ptr.p,
                                                      a.slice_w.p, a.sell_col.p, a.sell_val.p,
                                                      x, y, alpha);
  SFEEC_LAUNCH_CHECK();
}

}  // namespace sfeec_b200
