// SpMV kernels for the leapfrog chain. All are HBM-bound sparse contractions
// (~0.17 flop/byte): no tensor cores; the design goals are contiguous
// (coalesced) streaming of the operator arrays, L1/L2 hits on the gathered
// neighbour values, and enough loads in flight per SM.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "spmv_kernels.cuh"
#include "stencil.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int32_t kPad = 0x7fffffff;  // padding slot in the signed sliced layout

// Streaming (evict-first) loads of the operator arrays with an optional L2
// prefetch-size hint: PF 0 = plain ld.global.cs, 1 = .L2::128B, 2 = .L2::256B
// (on a miss the L2 fetches the whole 128/256-byte block, so the next
// warp-wide chunk of the same stream is already on its way). Values unchanged.
template <int PF>
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  if constexpr ((PF & 3) == 0) {
    return __ldcs(p);
  } else {
    int32_t v;
    if constexpr ((PF & 3) == 1)
      asm volatile("ld.global.cs.L2::128B.s32 %0, [%1];" : "=r"(v) : "l"(p));
    else
      asm volatile("ld.global.cs.L2::256B.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
  }
}
template <int PF>
__device__ __forceinline__ double ld_stream(const double* p) {
  if constexpr ((PF & 3) == 0) {
    return __ldcs(p);
  } else {
    double v;
    if constexpr ((PF & 3) == 1)
      asm volatile("ld.global.cs.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else
      asm volatile("ld.global.cs.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
}

// Gather of the input vector: PF bit 2 adds an L2 evict_last policy, so the
// gathered x (re-read by neighbouring rows) outlives the evict-first operator
// streams in L2. PF & 3 is the stream prefetch size (ld_stream).
template <int PF>
__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
  if constexpr ((PF & 4) == 0) {
    return __ldg(p);
  } else {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
  }
}
template <int PF>
__device__ __forceinline__ uint64_t gather_policy() {
  uint64_t pol = 0;
  if constexpr ((PF & 4) != 0)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ---- strict: reference-order, no FMA ------------------------------------
// sparse.cpp:98-103: acc += val*x in stored order; then the flow's axpy
// (dynamics.cpp:50,53,66) as a separate multiply and add.
template <bool ACC>
__global__ void __launch_bounds__(kThreads)
    k_csr_strict(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                 const double* __restrict__ v, const double* __restrict__ x,
                 double* __restrict__ y, double alpha) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double acc = 0.0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], x[ci[k]]));
  if (ACC)
    y[r] = __dadd_rn(y[r], __dmul_rn(alpha, acc));
  else
    y[r] = acc;
}

// ---- production CSR-vector: TPR lanes per row, shuffle reduction ---------
template <int TPR, bool ACC>
__global__ void __launch_bounds__(kThreads)
    k_csr_vec(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
              const double* __restrict__ v, const double* __restrict__ x,
              double* __restrict__ y, double alpha) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gt / TPR;
  const int lane = threadIdx.x & (TPR - 1);
  double acc = 0.0;
  if (row < rows) {
    const int64_t b = __ldg(rp + row), e = __ldg(rp + row + 1);
#pragma unroll 4
    for (int64_t k = b + lane; k < e; k += TPR) acc = fma(__ldg(v + k), __ldg(x + __ldg(ci + k)), acc);
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, TPR);
  if (lane == 0 && row < rows) y[row] = ACC ? fma(alpha, acc, y[row]) : acc;
}

// ---- wide rows (avg >= 64 nnz, e.g. the S(M1^2) SPAI of config 4): a warp
// per row, U entries per lane per round with every column/value load issued
// before any gather and every gather before any FMA; the operator is
// streamed (ld.global.cs) so L2 keeps the gathered vector.
template <bool ACC, int U>
__global__ void __launch_bounds__(kThreads)
    k_csr_wide(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const double* __restrict__ v, const double* __restrict__ x,
               double* __restrict__ y, double alpha) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t b = __ldg(rp + row), e = __ldg(rp + row + 1);
  double acc = 0.0;
  for (int64_t k0 = b + lane; k0 < e; k0 += 32 * U) {
    int c[U];
    double w[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + 32 * u;
      c[u] = k < e ? __ldcs(ci + k) : 0;
      w[u] = k < e ? __ldcs(v + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(w[u], xv[u], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = ACC ? fma(alpha, acc, y[row]) : acc;
}

// ---- sliced layout: persistent warps, one lane per row -------------------
// Warp w processes slices w, w + W, w + 2W, ... (W = warps in the grid). The
// metadata of the next slice and the y value of the current row (for the
// accumulating form) are loaded before the current slice's entries, so the
// only serialized memory round trips per slice are the ones of the entry
// chunks: all column/value loads of a chunk of CH entries are issued before
// any gather and all gathers before any FMA -> 2 * ceil(w / CH) round trips
// per slice. Operator arrays are read once: streaming loads (ld.global.cs)
// keep L1/L2 for the gathered vector.
struct SliceMeta {
  int64_t r0, ptr;
  int nr, w;
};

__device__ __forceinline__ SliceMeta load_meta(const int64_t* __restrict__ srow,
                                               const int64_t* __restrict__ sptr,
                                               const int32_t* __restrict__ sw, int64_t s) {
  SliceMeta m;
  m.r0 = __ldg(srow + s);
  m.nr = (int)(__ldg(srow + s + 1) - m.r0);
  m.ptr = __ldg(sptr + s);
  m.w = __ldg(sw + s);
  return m;
}

template <bool ACC, bool SIGNED, int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_sell(int64_t n_slices, const int64_t* __restrict__ srow, const int64_t* __restrict__ sptr,
           const int32_t* __restrict__ sw, const int32_t* __restrict__ col,
           const double* __restrict__ val, double scale, const double* __restrict__ x,
           double* __restrict__ y, double alpha) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  SliceMeta m = load_meta(srow, sptr, sw, s);
  while (true) {
    const int64_t sn = s + nwarps;
    SliceMeta mn;
    if (sn < n_slices) mn = load_meta(srow, sptr, sw, sn);
    if (lane < m.nr) {
      const int64_t row = m.r0 + lane;
      const double y0 = ACC ? y[row] : 0.0;
      const int64_t base = m.ptr + lane;
      double acc = 0.0;
      for (int k0 = 0; k0 < m.w; k0 += CH) {
        int32_t p[CH];
        double v[CH], xv[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const bool ok = k0 + j < m.w;
          const int64_t o = base + (int64_t)(k0 + j) * m.nr;
          p[j] = ok ? __ldcs(col + o) : kPad;
          if (!SIGNED) v[j] = ok ? __ldcs(val + o) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          if (SIGNED)
            xv[j] = p[j] != kPad ? __ldg(x + (p[j] < 0 ? ~p[j] : p[j])) : 0.0;
          else
            xv[j] = p[j] != kPad ? __ldg(x + p[j]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          if (SIGNED)
            acc += p[j] < 0 ? -xv[j] : xv[j];
          else
            acc = fma(v[j], xv[j], acc);
        }
      }
      const double r = SIGNED ? scale * acc : acc;
      y[row] = ACC ? fma(alpha, r, y0) : r;
    }
    if (sn >= n_slices) break;
    s = sn;
    m = mn;
  }
}

// ---- sliced layout, software-pipelined (wide rows: config 4's Q, ~300/row)
// As k_sell (fp64 values), but the column/value loads of chunk c+1 are issued
// before the gathers of chunk c, so a chunk costs one gather round trip and
// the streaming loads overlap it.
template <bool ACC, int CH, int MINB, int PF = 0>
__global__ void __launch_bounds__(kThreads, MINB)
    k_sell_pipe(int64_t n_slices, const int64_t* __restrict__ srow, const int64_t* __restrict__ sptr,
                const int32_t* __restrict__ sw, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x,
                double* __restrict__ y, double alpha, int rev) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = gather_policy<PF>();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  // rev: slices in descending order (the previous kernel's last-written rows,
  // still in L2, come first); every row's arithmetic is unchanged
  const int64_t last = n_slices - 1;
  SliceMeta m = load_meta(srow, sptr, sw, rev ? last - s : s);
  pdl_wait();  // PDL: x and y come from the previous kernels
  pdl_trigger();
  while (true) {
    const int64_t sn = s + nwarps;
    SliceMeta mn;
    if (sn < n_slices) mn = load_meta(srow, sptr, sw, rev ? last - sn : sn);
    if (lane < m.nr) {
      const int64_t row = m.r0 + lane;
      const double y0 = ACC ? y[row] : 0.0;
      const int64_t base = m.ptr + lane;
      double acc = 0.0;
      int32_t p[CH];
      double v[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const bool ok = j < m.w;
        const int64_t o = base + (int64_t)j * m.nr;
        p[j] = ok ? ld_stream<PF>(col + o) : kPad;
        v[j] = ok ? ld_stream<PF>(val + o) : 0.0;
      }
      for (int k0 = 0; k0 < m.w; k0 += CH) {
        int32_t pn[CH];
        double vn[CH], xv[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const bool ok = k0 + CH + j < m.w;
          const int64_t o = base + (int64_t)(k0 + CH + j) * m.nr;
          pn[j] = ok ? ld_stream<PF>(col + o) : kPad;
          vn[j] = ok ? ld_stream<PF>(val + o) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) xv[j] = p[j] != kPad ? ld_gather<PF>(x + p[j], pol) : 0.0;
#pragma unroll
        for (int j = 0; j < CH; ++j) acc = fma(v[j], xv[j], acc);
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          p[j] = pn[j];
          v[j] = vn[j];
        }
      }
      y[row] = ACC ? fma(alpha, acc, y0) : acc;
    }
    if (sn >= n_slices) break;
    s = sn;
    m = mn;
  }
}

// ---- sliced layout, software-pipelined + L2 bulk prefetch -----------------
// As k_sell_pipe, and lane 0 issues cp.async.bulk.prefetch.L2 for the column
// and value arrays of the warp's NEXT slice (its first kPfCols entries per
// row) while the current one streams, plus, inside wide slices (config 4's
// ~300/row), the next kPfCols columns every kPfCols: the HBM requests run a
// slice ahead of the loads with no registers held for them, and the loads
// then hit L2.
constexpr int kPfCols = 32;

__device__ __forceinline__ void l2_prefetch_bytes(const char* base, int64_t b0, int64_t b1,
                                                  int64_t bmax) {
  b0 &= ~int64_t(15);
  b1 = min((b1 + 15) & ~int64_t(15), bmax & ~int64_t(15));
  if (b1 > b0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + b0),
                 "r"((unsigned)(b1 - b0))
                 : "memory");
}
// entries [e0, e1) of the sliced column / value arrays (n entries in all)
__device__ __forceinline__ void l2_prefetch_entries(const int32_t* col, const double* val,
                                                    int64_t e0, int64_t e1, int64_t n) {
  l2_prefetch_bytes(reinterpret_cast<const char*>(col), 4 * e0, 4 * e1, 4 * n);
  l2_prefetch_bytes(reinterpret_cast<const char*>(val), 8 * e0, 8 * e1, 8 * n);
}

template <bool ACC, int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_sell_pf(int64_t n_slices, const int64_t* __restrict__ srow, const int64_t* __restrict__ sptr,
              const int32_t* __restrict__ sw, const int32_t* __restrict__ col,
              const double* __restrict__ val, const double* __restrict__ x,
              double* __restrict__ y, double alpha, int64_t n_entries) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  SliceMeta m = load_meta(srow, sptr, sw, s);
  SliceMeta mn;
  if (s + nwarps < n_slices) mn = load_meta(srow, sptr, sw, s + nwarps);
  if (lane == 0)
    l2_prefetch_entries(col, val, m.ptr, m.ptr + (int64_t)min(m.w, kPfCols) * m.nr, n_entries);
  while (true) {
    const int64_t sn = s + nwarps;
    SliceMeta mnn;
    if (sn + nwarps < n_slices) mnn = load_meta(srow, sptr, sw, sn + nwarps);
    if (lane == 0 && sn < n_slices)
      l2_prefetch_entries(col, val, mn.ptr, mn.ptr + (int64_t)min(mn.w, kPfCols) * mn.nr,
                          n_entries);
    if (lane < m.nr) {
      const int64_t row = m.r0 + lane;
      const double y0 = ACC ? y[row] : 0.0;
      const int64_t base = m.ptr + lane;
      double acc = 0.0;
      int32_t p[CH];
      double v[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const bool ok = j < m.w;
        const int64_t o = base + (int64_t)j * m.nr;
        p[j] = ok ? __ldcs(col + o) : kPad;
        v[j] = ok ? __ldcs(val + o) : 0.0;
      }
      for (int k0 = 0; k0 < m.w; k0 += CH) {
        if (lane == 0 && (k0 % kPfCols) == 0 && k0 + kPfCols < m.w)
          l2_prefetch_entries(col, val, m.ptr + (int64_t)(k0 + kPfCols) * m.nr,
                              m.ptr + (int64_t)min(k0 + 2 * kPfCols, m.w) * m.nr, n_entries);
        int32_t pn[CH];
        double vn[CH], xv[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const bool ok = k0 + CH + j < m.w;
          const int64_t o = base + (int64_t)(k0 + CH + j) * m.nr;
          pn[j] = ok ? __ldcs(col + o) : kPad;
          vn[j] = ok ? __ldcs(val + o) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) xv[j] = p[j] != kPad ? __ldg(x + p[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < CH; ++j) acc = fma(v[j], xv[j], acc);
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          p[j] = pn[j];
          v[j] = vn[j];
        }
      }
      y[row] = ACC ? fma(alpha, acc, y0) : acc;
    }
    if (sn >= n_slices) break;
    s = sn;
    m = mn;
    mn = mnn;
  }
}

// ---- sliced layout, two lanes per row (wide rows, e.g. Q_sym ~16/row) -----
// A warp takes half a slice pair: lanes 2i, 2i+1 share row i of 16 rows and
// take alternate entries, so each lane holds <= CH entries of a <= 2*CH row
// in one chunk: 2 memory round trips per row, then one shuffle. Persistent
// warps with the next slice's metadata prefetched, as k_sell.
template <bool ACC, int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_sell_tpr2(int64_t n_slices, const int64_t* __restrict__ srow,
                const int64_t* __restrict__ sptr, const int32_t* __restrict__ sw,
                const int32_t* __restrict__ col, const double* __restrict__ val,
                const double* __restrict__ x, double* __restrict__ y, double alpha) {
  const int lane = threadIdx.x & 31;
  const int half = lane & 1, rl = lane >> 1;  // row within the 16-row group
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // work item = (slice, 16-row group g in {0,1})
  const int64_t n_items = 2 * n_slices;
  int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (it >= n_items) return;
  SliceMeta m = load_meta(srow, sptr, sw, it >> 1);
  while (true) {
    const int64_t itn = it + nwarps;
    SliceMeta mn;
    if (itn < n_items) mn = load_meta(srow, sptr, sw, itn >> 1);
    const int li = (int)(it & 1) * 16 + rl;  // row index inside the slice
    const bool active = li < m.nr;
    double acc = 0.0, y0 = 0.0;
    const int64_t row = m.r0 + li;
    if (active) {
      if (ACC && half == 0) y0 = y[row];
      const int64_t base = m.ptr + li;
      for (int k0 = 0; k0 < m.w; k0 += 2 * CH) {
        int32_t p[CH];
        double v[CH], xv[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int k = k0 + 2 * j + half;
          const bool ok = k < m.w;
          const int64_t o = base + (int64_t)k * m.nr;
          p[j] = ok ? __ldcs(col + o) : -1;
          v[j] = ok ? __ldcs(val + o) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) xv[j] = p[j] >= 0 ? __ldg(x + p[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < CH; ++j) acc = fma(v[j], xv[j], acc);
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (active && half == 0) y[row] = ACC ? fma(alpha, acc, y0) : acc;
    if (itn >= n_items) break;
    it = itn;
    m = mn;
  }
}

// ---- plain ELL for narrow operators: one thread per row ------------------
template <bool ACC, bool SIGNED, int W, int PF = 0>
__global__ void __launch_bounds__(kThreads)
    k_ell(int64_t rows, const int32_t* __restrict__ col, const double* __restrict__ val,
          double scale, const double* __restrict__ x, double* __restrict__ y, double alpha,
          int rev) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows) return;
  const int64_t r = rev ? rows - 1 - g : g;  // rev: descending rows (see k_sell_pipe)
  const uint64_t pol = gather_policy<PF>();
  int32_t p[W];
  double v[W], xv[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    p[k] = ld_stream<PF>(col + (int64_t)k * rows + r);
    if (!SIGNED) v[k] = ld_stream<PF>(val + (int64_t)k * rows + r);
  }
  // PDL: the operator stream above does not depend on the previous kernel;
  // x and y do (no-ops without a programmatic launch)
  pdl_wait();
  pdl_trigger();
  const double y0 = ACC ? y[r] : 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (SIGNED)
      xv[k] = p[k] != kPad ? ld_gather<PF>(x + (p[k] < 0 ? ~p[k] : p[k]), pol) : 0.0;
    else
      xv[k] = ld_gather<PF>(x + p[k], pol);
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (SIGNED)
      acc += p[k] < 0 ? -xv[k] : xv[k];
    else
      acc = fma(v[k], xv[k], acc);
  }
  const double res = SIGNED ? scale * acc : acc;
  y[r] = ACC ? fma(alpha, res, y0) : res;
}

// ---- column-delta layouts (DSlice in spmv_kernels.cuh) --------------------
// Entry code (uint16): sel << 15 | delta (values, delta <= 32766) or
// sel << 15 | delta << 1 | negative (incidence, delta <= 16382); the column is
// base_sel[k] + lane + delta. Two bases per entry cover a slice / group that
// straddles two entity types (k-th neighbours in two id ranges). 0xffff pads.
constexpr unsigned kDPad = 0xffffu;

__device__ __forceinline__ unsigned dcode_of(uint2 d, int j) {
  const unsigned w = j < 2 ? d.x : d.y;
  return (j & 1) ? (w >> 16) : (w & 0xffffu);
}
__device__ __forceinline__ int bse(int4 b, int j) {
  return j == 0 ? b.x : j == 1 ? b.y : j == 2 ? b.z : b.w;
}

// one chunk of 4 entries -> gathered x (0 for pads) and, for SIGNED, the sign
template <bool SIGNED>
__device__ __forceinline__ void dgather(int4 b0, int4 b1, uint2 d, int lane,
                                        const double* __restrict__ x, double (&xv)[4],
                                        bool (&neg)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const unsigned u = dcode_of(d, j);
    const int off = SIGNED ? (int)((u >> 1) & 0x3fffu) : (int)(u & 0x7fffu);
    const int base = (u >> 15) ? bse(b1, j) : bse(b0, j);
    neg[j] = SIGNED && (u & 1u);
    xv[j] = u != kDPad ? __ldg(x + (base + lane + off)) : 0.0;
  }
}

// sliced column-delta layout, persistent warps (one per slice per round),
// software-pipelined as k_sell_pipe: the base / code / value loads of chunk
// c+1 are issued before the gathers of chunk c. Rows summed in CSR order.
template <bool ACC, bool SIGNED, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_dsell(int64_t n_slices, const DSlice* __restrict__ meta, const int32_t* __restrict__ dbase,
            const uint16_t* __restrict__ dcol, const double* __restrict__ val, double scale,
            const double* __restrict__ x, double* __restrict__ y, double alpha) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  auto ld = [&](int64_t i) {
    const int4* p = reinterpret_cast<const int4*>(meta + i);
    const int4 a = __ldg(p), b = __ldg(p + 1);
    DSlice m;
    m.r0 = ((int64_t)(unsigned)a.y << 32) | (unsigned)a.x;
    m.vptr = ((int64_t)(unsigned)a.w << 32) | (unsigned)a.z;
    m.dptr = ((int64_t)(unsigned)b.y << 32) | (unsigned)b.x;
    m.bptr = b.z;
    m.nw = b.w;
    return m;
  };
  DSlice m = ld(s);
  while (true) {
    const int64_t sn = s + nwarps;
    DSlice mn;
    if (sn < n_slices) mn = ld(sn);
    const int w = m.nw & 0xfffff, nr = (m.nw >> 20) & 63;
    const bool full = (m.nw >> 26) & 1;
    if (lane < nr) {
      const int64_t row = m.r0 + lane;
      const double y0 = ACC ? y[row] : 0.0;
      const double* vp = SIGNED ? nullptr : val + m.vptr + lane;
      double acc = 0.0;
      if (!full) {
        const int4* bp = reinterpret_cast<const int4*>(dbase + m.bptr);
        const uint2* dp = reinterpret_cast<const uint2*>(dcol + m.dptr) + lane;
        int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
        if (w > 0) {
          b0 = __ldg(bp);
          b1 = __ldg(bp + 1);
        }
        uint2 d = w > 0 ? __ldcs(dp) : make_uint2(0u, 0u);
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (!SIGNED && j < w) ? __ldcs(vp + (int64_t)j * nr) : 0.0;
        for (int k0 = 0, c = 0; k0 < w; k0 += 4, ++c) {
          int4 b0n = b0, b1n = b1;
          uint2 dn = d;
          double vn[4];
          if (k0 + 4 < w) {
            b0n = __ldg(bp + 2 * c + 2);
            b1n = __ldg(bp + 2 * c + 3);
            dn = __ldcs(dp + (int64_t)(c + 1) * nr);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            vn[j] = (!SIGNED && k0 + 4 + j < w) ? __ldcs(vp + (int64_t)(k0 + 4 + j) * nr) : 0.0;
          double xv[4];
          bool neg[4];
          dgather<SIGNED>(b0, b1, d, lane, x, xv, neg);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (SIGNED)
              acc += neg[j] ? -xv[j] : xv[j];
            else
              acc = fma(v[j], xv[j], acc);
          }
          b0 = b0n;
          b1 = b1n;
          d = dn;
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = vn[j];
        }
      } else {
        // int32 columns (the codes did not fit; rare), as k_sell
        const int32_t* cp = reinterpret_cast<const int32_t*>(dcol + m.dptr) + lane;
        for (int k0 = 0; k0 < w; k0 += 4) {
          int32_t p[4];
          double v[4], xv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const bool ok = k0 + j < w;
            p[j] = ok ? __ldcs(cp + (int64_t)(k0 + j) * nr) : kPad;
            v[j] = (!SIGNED && ok) ? __ldcs(vp + (int64_t)(k0 + j) * nr) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            xv[j] = p[j] != kPad ? __ldg(x + (SIGNED && p[j] < 0 ? ~p[j] : p[j])) : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (SIGNED)
              acc += p[j] < 0 ? -xv[j] : xv[j];
            else
              acc = fma(v[j], xv[j], acc);
          }
        }
      }
      const double r = SIGNED ? scale * acc : acc;
      y[row] = ACC ? fma(alpha, r, y0) : r;
    }
    if (sn >= n_slices) break;
    s = sn;
    m = mn;
  }
}

// ELL column-delta layout (narrow operators, width W <= 8): one thread per
// row, 32-row groups; every load of a row is independent of the others (the
// group's bases are warp broadcasts, its full-column index another).
template <bool ACC, bool SIGNED, int W>
__global__ void __launch_bounds__(kThreads)
    k_dell(int64_t rows, const int32_t* __restrict__ dbase, const uint16_t* __restrict__ dcol,
           const int32_t* __restrict__ dfull, const int32_t* __restrict__ fcol,
           const double* __restrict__ val, double scale, const double* __restrict__ x,
           double* __restrict__ y, double alpha) {
  constexpr int NC = (W + 3) / 4;  // code chunks per row
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t g = r >> 5;
  const int lane = threadIdx.x & 31;
  const double y0 = ACC ? y[r] : 0.0;
  const int fi = __ldg(dfull + g);
  int4 b0[NC], b1[NC];
  uint2 d[NC];
  double v[W];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int4* bp = reinterpret_cast<const int4*>(dbase + g * 8 * NC) + 2 * c;
    b0[c] = __ldg(bp);
    b1[c] = __ldg(bp + 1);
    d[c] = __ldcs(reinterpret_cast<const uint2*>(dcol + g * 128 * NC) + c * 32 + lane);
  }
  if (!SIGNED) {
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = __ldcs(val + g * 32 * W + k * 32 + lane);
  }
  double xv[4 * NC];
  bool neg[4 * NC];
  if (fi < 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double xc[4];
      bool nc[4];
      dgather<SIGNED>(b0[c], b1[c], d[c], lane, x, xc, nc);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xv[4 * c + j] = xc[j];
        neg[4 * c + j] = nc[j];
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int32_t p = __ldcs(fcol + (int64_t)fi * 32 * W + k * 32 + lane);
      neg[k] = SIGNED && p < 0 && p != kPad;
      xv[k] = p != kPad ? __ldg(x + (SIGNED && p < 0 ? ~p : p)) : 0.0;
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (SIGNED)
      acc += neg[k] ? -xv[k] : xv[k];
    else
      acc = fma(v[k], xv[k], acc);
  }
  const double res = SIGNED ? scale * acc : acc;
  y[r] = ACC ? fma(alpha, res, y0) : res;
}

// ---- delta layout builders ----
// the two bases of entry k for the rows r0 .. r0+nr-1 (lane = row - r0):
// b0 = min(col - lane) over the rows that have an entry k, b1 = the min of
// those beyond b0 + lim; *fit = 0 if some row is beyond b1 + lim too
__device__ __forceinline__ int2 dbase_entry(const int64_t* __restrict__ rp,
                                            const int32_t* __restrict__ ci, int64_t r0, int nr,
                                            int k, int lane, int lim, bool* fit) {
  int v = INT_MAX;
  if (lane < nr) {
    const int64_t b = rp[r0 + lane], e = rp[r0 + lane + 1];
    if (b + k < e) v = ci[b + k] - lane;
  }
  const int m0 = __reduce_min_sync(0xffffffffu, v);
  if (m0 == INT_MAX) return make_int2(0, 0);  // no row has entry k
  const bool in0 = (int64_t)v - m0 <= lim;
  const int m1 = __reduce_min_sync(0xffffffffu, in0 ? INT_MAX : v);
  if (m1 == INT_MAX) return make_int2(m0, m0);
  const bool in1 = !in0 && (int64_t)v - m1 <= lim;
  if (__any_sync(0xffffffffu, v != INT_MAX && !in0 && !in1)) *fit = false;
  return make_int2(m0, m1);
}

// code of entry k of lane `lane` (kDPad for a pad slot)
__device__ __forceinline__ uint16_t dcode(const int64_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci,
                                          const double* __restrict__ cv, bool sg, int64_t row,
                                          int k, int lane, int32_t b0, int32_t b1) {
  const int64_t b = rp[row], e = rp[row + 1];
  if (b + k >= e) return (uint16_t)kDPad;
  const int lim = sg ? 16382 : 32766;
  const int v = ci[b + k] - lane;
  const unsigned sel = (int64_t)v - b0 <= lim ? 0u : 1u;
  const unsigned dl = (unsigned)(v - (sel ? b1 : b0));
  return (uint16_t)((sel << 15) | (sg ? (dl << 1) | (cv[b + k] < 0 ? 1u : 0u) : dl));
}

// pass 1 of the sliced form: bases of every slice + fit flags (warp per
// slice); slice s, chunk c: b0 of entries 4c..4c+3 at sb[s] + 8c, b1 at +4
__global__ void k_dsell_bases(int64_t n_slices, const int64_t* __restrict__ srow,
                              const int32_t* __restrict__ sw, const int32_t* __restrict__ sb,
                              const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              int lim, int32_t* __restrict__ base, uint8_t* __restrict__ fit) {
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= n_slices) return;
  const int64_t r0 = srow[sl];
  const int nr = (int)(srow[sl + 1] - r0), w = sw[sl];
  bool ok = true;
  for (int k = 0; k < ((w + 3) & ~3); ++k) {
    const int2 bk = k < w ? dbase_entry(rp, ci, r0, nr, k, lane, lim, &ok) : make_int2(0, 0);
    if (lane == 0) {
      base[sb[sl] + 8 * (k >> 2) + (k & 3)] = bk.x;
      base[sb[sl] + 8 * (k >> 2) + 4 + (k & 3)] = bk.y;
    }
  }
  if (lane == 0) fit[sl] = ok ? 1 : 0;
}

// pass 2: codes (or int32 columns) and values, warp per slice
__global__ void k_dsell_fill(int64_t n_slices, const DSlice* __restrict__ meta,
                             const int32_t* __restrict__ base, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, const double* __restrict__ cv,
                             bool sg, uint16_t* __restrict__ dcol, double* __restrict__ sv) {
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= n_slices) return;
  const DSlice m = meta[sl];
  const int w = m.nw & 0xfffff, nr = (m.nw >> 20) & 63;
  const bool full = (m.nw >> 26) & 1;
  if (lane >= nr) return;
  const int64_t row = m.r0 + lane, b = rp[row], e = rp[row + 1];
  for (int k = 0; k < w; ++k) {
    if (!sg) sv[m.vptr + (int64_t)k * nr + lane] = b + k < e ? cv[b + k] : 0.0;
    if (full) {
      int32_t* fc = reinterpret_cast<int32_t*>(dcol + m.dptr);
      int32_t c = kPad;
      if (b + k < e)
        c = sg && cv[b + k] < 0 ? ~ci[b + k] : ci[b + k];
      else if (!sg)
        c = e > b ? ci[b] : 0;  // val 0, a column the row reads anyway
      fc[(int64_t)k * nr + lane] = c;
    }
  }
  if (!full)
    for (int k = 0; k < ((w + 3) & ~3); ++k) {
      const int32_t* bk = base + m.bptr + 8 * (k >> 2) + (k & 3);
      dcol[m.dptr + (int64_t)(k >> 2) * 4 * nr + 4 * lane + (k & 3)] =
          k < w ? dcode(rp, ci, cv, sg, row, k, lane, bk[0], bk[4]) : (uint16_t)kDPad;
    }
}

// ELL form, pass 1: bases per 32-row group (warp per group), same chunk
// layout as the sliced form at g * 2 * W4
__global__ void k_dell_bases(int64_t rows, int w, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, int lim, int32_t* __restrict__ base,
                             uint8_t* __restrict__ fit) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g * 32 >= rows) return;
  const int nr = rows - g * 32 < 32 ? (int)(rows - g * 32) : 32;
  const int w4 = (w + 3) & ~3;
  bool ok = true;
  for (int k = 0; k < w4; ++k) {
    const int2 bk = k < w ? dbase_entry(rp, ci, g * 32, nr, k, lane, lim, &ok) : make_int2(0, 0);
    if (lane == 0) {
      base[g * 2 * w4 + 8 * (k >> 2) + (k & 3)] = bk.x;
      base[g * 2 * w4 + 8 * (k >> 2) + 4 + (k & 3)] = bk.y;
    }
  }
  if (lane == 0) fit[g] = ok ? 1 : 0;
}

// ELL form, pass 2: one thread per row
__global__ void k_dell_fill(int64_t rows, int w, const int32_t* __restrict__ base,
                            const int32_t* __restrict__ dfull, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ cv,
                            bool sg, uint16_t* __restrict__ dcol, int32_t* __restrict__ fcol,
                            double* __restrict__ sv) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t g = r >> 5;
  const int lane = (int)(r & 31), w4 = (w + 3) & ~3;
  const int64_t b = rp[r], e = rp[r + 1];
  const int fi = dfull[g];
  for (int k = 0; k < w4; ++k) {
    const int64_t o = g * 32 * w4 + (int64_t)(k >> 2) * 128 + 4 * lane + (k & 3);
    const int32_t* bk = base + g * 2 * w4 + 8 * (k >> 2) + (k & 3);
    dcol[o] = (fi < 0 && k < w) ? dcode(rp, ci, cv, sg, r, k, lane, bk[0], bk[4])
                                : (uint16_t)kDPad;
  }
  for (int k = 0; k < w; ++k) {
    if (!sg) sv[g * 32 * w + k * 32 + lane] = b + k < e ? cv[b + k] : 0.0;
    if (fi >= 0) {
      int32_t c = kPad;
      if (b + k < e)
        c = sg && cv[b + k] < 0 ? ~ci[b + k] : ci[b + k];
      else if (!sg)
        c = e > b ? ci[b] : 0;
      fcol[(int64_t)fi * 32 * w + k * 32 + lane] = c;
    }
  }
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double alpha,
                       int64_t n, int strict) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = strict ? __dadd_rn(y[i], __dmul_rn(alpha, x[i])) : fma(alpha, x[i], y[i]);
}

__global__ void k_div_copy(double* __restrict__ x, const double* __restrict__ y, double nrm,
                           int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = y[i] / nrm;  // dynamics.cpp:130
}

inline unsigned blocks_for(int64_t threads) {
  return (unsigned)std::max<int64_t>(1, (threads + kThreads - 1) / kThreads);
}

}  // namespace

// SFEEC_WIDE_CSR=1: rows of >= 64 entries stay plain CSR with a warp per row
// (k_csr_wide). Measured on config 4 (S(M1^2) Q, ~308 per row): faster at
// 32^3 (4.79 vs 3.81 TB/s) but slower at 64^3 (4.28 vs 4.66 TB/s), where the
// sliced layout's lane-per-row gathers coalesce better (consecutive rows'
// j-th neighbours are consecutive ids); so the sliced layout is the default.
static bool wide_rows(double avg) {
  const char* env = std::getenv("SFEEC_WIDE_CSR");
  return env && std::atoi(env) == 1 && avg >= 64.0;
}

// SFEEC_DELTA=1 selects the column-delta layouts. Off by default: measured on
// B200 (tet128 K-Q 0.564 -> 0.612 ms, config 4 K-Q 6.96 -> 7.59 ms) the
// 17% fewer bytes do not pay for the longer per-entry decode (ncu: 47% more
// instructions, issue-bound); the narrow ELL operators gain 1-2%.
static bool delta_enabled() {
  const char* e = std::getenv("SFEEC_DELTA");
  return e && std::atoi(e) == 1;
}

// the sliced delta form pays when its bytes (values + int16 deltas + int32
// bases + 32 B metadata per slice) undercut the int32 form's (values + int32
// columns + 20 B metadata per slice): not for short slices of short rows
static bool dsell_pays(const std::vector<int64_t>& hrow, const std::vector<int32_t>& hw,
                       bool sg) {
  double b_delta = 0, b_int = 0;
  const double vb = sg ? 0.0 : 8.0;
  for (size_t i = 0; i < hw.size(); ++i) {
    const double nr = (double)(hrow[i + 1] - hrow[i]), w = hw[i], w4 = (hw[i] + 3) & ~3;
    b_delta += nr * w * vb + 2.0 * nr * w4 + 8.0 * w4 + 32.0;
    b_int += nr * w * (vb + 4.0) + 20.0;
  }
  return b_delta < b_int;
}

void DevOperator::build_dsell(const int64_t* drp, const int32_t* dci, const double* dv,
                              const std::vector<int64_t>& hrow, const std::vector<int32_t>& hw,
                              cudaStream_t s) {
  const bool sg = layout == kSigned;
  n_slices = (int64_t)hw.size();
  std::vector<int32_t> hb((size_t)n_slices);
  int64_t nb = 0;
  for (int64_t i = 0; i < n_slices; ++i) {
    if (hw[(size_t)i] >= (1 << 20)) throw Error(SFEEC_EINVAL, "sliced delta layout: row too wide");
    hb[(size_t)i] = (int32_t)nb;
    nb += 2 * ((hw[(size_t)i] + 3) & ~3);
  }
  if (nb > INT32_MAX) throw Error(SFEEC_EINVAL, "sliced delta layout: too many base columns");
  DevBuf<int64_t> srow;
  DevBuf<int32_t> sw, sb;
  srow.upload(hrow.data(), hrow.size(), s);
  sw.upload(hw.data(), hw.size(), s);
  sb.upload(hb.data(), hb.size(), s);
  dbase.alloc((size_t)std::max<int64_t>(nb, 8));
  DevBuf<uint8_t> fit;
  fit.alloc((size_t)n_slices);
  k_dsell_bases<<<blocks_for(n_slices * 32), kThreads, 0, s>>>(
      n_slices, srow.p, sw.p, sb.p, drp, dci, sg ? 16382 : 32766, dbase.p, fit.p);
  SFEEC_LAUNCH_CHECK();
  std::vector<uint8_t> hf((size_t)n_slices);
  SFEEC_CUDA(cudaMemcpyAsync(hf.data(), fit.p, hf.size(), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  std::vector<DSlice> hm((size_t)n_slices);
  int64_t vp = 0, dp = 0;
  n_full = 0;
  for (int64_t i = 0; i < n_slices; ++i) {
    const int64_t nr = hrow[(size_t)i + 1] - hrow[(size_t)i], w = hw[(size_t)i];
    const bool full = hf[(size_t)i] == 0;
    n_full += full;
    hm[(size_t)i] = DSlice{hrow[(size_t)i], vp, dp, hb[(size_t)i],
                           (int32_t)(w | (nr << 20) | ((int64_t)full << 26))};
    vp += w * nr;
    dp += full ? ((2 * w * nr + 3) & ~int64_t(3)) : ((w + 3) & ~int64_t(3)) * nr;
  }
  sell_entries = vp;
  dslice.upload(hm.data(), hm.size(), s);
  dcol.alloc((size_t)std::max<int64_t>(dp, 4));
  if (!sg) sell_val.alloc((size_t)std::max<int64_t>(vp, 1));
  k_dsell_fill<<<blocks_for(n_slices * 32), kThreads, 0, s>>>(
      n_slices, dslice.p, dbase.p, drp, dci, dv, sg, dcol.p, sell_val.p);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
  ell = false;
  delta = true;
}

void DevOperator::build_dell(const int64_t* drp, const int32_t* dci, const double* dv, int w,
                             cudaStream_t s) {
  const bool sg = layout == kSigned;
  const int64_t G = (rows + 31) / 32, w4 = (w + 3) & ~3;
  dbase.alloc((size_t)(G * 2 * w4));
  DevBuf<uint8_t> fit;
  fit.alloc((size_t)G);
  k_dell_bases<<<blocks_for(G * 32), kThreads, 0, s>>>(rows, w, drp, dci, sg ? 16382 : 32766,
                                                        dbase.p, fit.p);
  SFEEC_LAUNCH_CHECK();
  std::vector<uint8_t> hf((size_t)G);
  SFEEC_CUDA(cudaMemcpyAsync(hf.data(), fit.p, hf.size(), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> hfull((size_t)G);
  n_full = 0;
  for (int64_t g = 0; g < G; ++g) hfull[(size_t)g] = hf[(size_t)g] ? -1 : (int32_t)n_full++;
  dfull.upload(hfull.data(), hfull.size(), s);
  dcol.alloc((size_t)(G * 32 * w4));
  if (!sg) sell_val.alloc((size_t)(G * 32 * w));
  sell_col.alloc((size_t)std::max<int64_t>(1, n_full * 32 * w));
  k_dell_fill<<<blocks_for(rows), kThreads, 0, s>>>(rows, w, dbase.p, dfull.p, drp, dci, dv, sg,
                                                     dcol.p, sell_col.p, sell_val.p);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
  ell = true;
  ell_w = w;
  sell_entries = G * 32 * w;
  delta = true;
}

void DevOperator::upload(const HostCSR& h, bool strict_only, cudaStream_t s) {
  rows = h.rows;
  cols = h.cols;
  nnz = h.nnz();
  rp.upload(h.row_ptr.data(), h.row_ptr.size(), s);
  ci.upload(h.col_idx.data(), h.col_idx.size(), s);
  val.upload(h.val.data(), h.val.size(), s);
  double avg = rows ? (double)nnz / (double)rows : 0.0;
  tpr = 1;
  while (tpr < 32 && tpr * 2 <= avg) tpr *= 2;
  layout = kCsr;
  if (strict_only || rows == 0 || nnz == 0 || wide_rows(avg)) {
    SFEEC_CUDA(cudaStreamSynchronize(s));
    return;
  }
  // greedy slices: <= 32 consecutive rows whose lengths stay within 1/8 of
  // the slice width
  std::vector<int64_t> hrow{0}, hptr{0};
  std::vector<int32_t> hw;
  {
    int64_t r = 0;
    while (r < rows) {
      int64_t w = h.row_ptr[(size_t)r + 1] - h.row_ptr[(size_t)r];
      int64_t e = r + 1;
      while (e < rows && e - r < 32) {
        int64_t l = h.row_ptr[(size_t)e + 1] - h.row_ptr[(size_t)e];
        int64_t tol = std::max<int64_t>(1, std::max(w, l) / 8);
        if (std::llabs(l - w) > tol) break;
        w = std::max(w, l);
        ++e;
      }
      hw.push_back((int32_t)w);
      // slice starts 4-entry aligned (16 B of columns: bulk copies, k_sell_tma)
      hptr.push_back(hptr.back() + ((w * (e - r) + 3) & ~int64_t(3)));
      hrow.push_back(e);
      r = e;
    }
  }
  n_slices = (int64_t)hw.size();
  sell_entries = hptr.back();
  const double mag = std::fabs(h.val[0]);
  bool signed_ok = mag > 0;
  for (double v : h.val)
    if (std::fabs(v) != mag) {
      signed_ok = false;
      break;
    }
  const double rows_per_slice = (double)rows / (double)n_slices;
  const double pad_ratio = (double)sell_entries / (double)nnz;
  if (rows_per_slice >= 8 && signed_ok && pad_ratio <= 2.5) {
    layout = kSigned;
    scale = mag;
  } else if (rows_per_slice >= 8 && pad_ratio <= 1.15) {
    layout = kSell;
  } else {
    SFEEC_CUDA(cudaStreamSynchronize(s));
    return;
  }
  if (win_enabled() && build_win(rp.p, ci.p, val.p, hrow, hw, s)) {
    drop_csr();
    return;
  }
  // narrow operators (C: 3, C^T: <= 6, M2: 7 per row) go to plain ELL: one
  // thread per row, entry k of row r at k*rows + r, no slice metadata and
  // no persistent loop -- the short rows are latency-bound, so every row's
  // loads must be independent and the grid as large as the row count
  int64_t wmax = 0;
  for (int64_t r = 0; r < rows; ++r) wmax = std::max(wmax, h.row_ptr[(size_t)r + 1] - h.row_ptr[(size_t)r]);
  const double ell_pad = (double)(rows * wmax) / (double)nnz;
  if (wmax >= 1 && wmax <= 8 && ell_pad <= (layout == kSigned ? 1.3 : 1.1) && delta_enabled()) {
    build_dell(rp.p, ci.p, val.p, (int)wmax, s);
    drop_csr();
    return;
  }
  if (wmax >= 1 && wmax <= 8 && ell_pad <= (layout == kSigned ? 1.3 : 1.1)) {
    ell = true;
    ell_w = (int)wmax;
    sell_entries = rows * wmax;
    std::vector<int32_t> ec((size_t)sell_entries, layout == kSigned ? kPad : 0);
    std::vector<double> evv;
    if (layout == kSell) evv.assign((size_t)sell_entries, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t b = h.row_ptr[(size_t)r], e = h.row_ptr[(size_t)r + 1];
      for (int64_t k = 0; k < wmax; ++k) {
        const size_t o = (size_t)(k * rows + r);
        if (b + k < e) {
          const int32_t c = h.col_idx[(size_t)(b + k)];
          const double v = h.val[(size_t)(b + k)];
          if (layout == kSigned) {
            ec[o] = v < 0 ? ~c : c;
          } else {
            ec[o] = c;
            evv[o] = v;
          }
        } else if (layout == kSell) {
          ec[o] = e > b ? h.col_idx[(size_t)b] : 0;  // val 0
        }
      }
    }
    sell_col.upload(ec.data(), ec.size(), s);
    if (layout == kSell) sell_val.upload(evv.data(), evv.size(), s);
    SFEEC_CUDA(cudaStreamSynchronize(s));
    drop_csr();
    return;
  }
  if (delta_enabled() && dsell_pays(hrow, hw, layout == kSigned)) {
    build_dsell(rp.p, ci.p, val.p, hrow, hw, s);
    drop_csr();
    return;
  }
  std::vector<int32_t> hc((size_t)sell_entries + 4, layout == kSigned ? kPad : 0);
  std::vector<double> hv;
  if (layout == kSell) hv.assign((size_t)sell_entries + 4, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t sl = 0; sl < n_slices; ++sl) {
    const int64_t r0 = hrow[(size_t)sl], nr = hrow[(size_t)sl + 1] - r0;
    for (int64_t lane = 0; lane < nr; ++lane) {
      const int64_t r = r0 + lane;
      const int64_t b = h.row_ptr[(size_t)r], e = h.row_ptr[(size_t)r + 1];
      for (int64_t k = 0; k < hw[(size_t)sl]; ++k) {
        const size_t o = (size_t)(hptr[(size_t)sl] + k * nr + lane);
        if (b + k < e) {
          const int32_t c = h.col_idx[(size_t)(b + k)];
          const double v = h.val[(size_t)(b + k)];
          if (layout == kSigned) {
            hc[o] = v < 0 ? ~c : c;
          } else {
            hc[o] = c;
            hv[o] = v;
          }
        } else if (layout == kSell && e > b) {
          hc[o] = h.col_idx[(size_t)b];  // val 0, a column the row reads anyway
        }
      }
    }
  }
  if (layout == kSell) prepare_sell_tma();
  slice_row.upload(hrow.data(), hrow.size(), s);
  slice_ptr.upload(hptr.data(), hptr.size(), s);
  slice_w.upload(hw.data(), hw.size(), s);
  sell_col.upload(hc.data(), hc.size(), s);
  if (layout == kSell) sell_val.upload(hv.data(), hv.size(), s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
  drop_csr();
  // the host vectors die at return: make the async copies complete first
  SFEEC_CUDA(cudaStreamSynchronize(s));
}

namespace {

__global__ void k_abs_uniform(int64_t nnz, const double* __restrict__ v, int* __restrict__ not_uniform) {
  const double m = fabs(v[0]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x)
    if (fabs(v[i]) != m) *not_uniform = 1;
}

// CSR -> ELL (column-major, width w), one thread per row
__global__ void k_to_ell(int64_t rows, int w, bool sg, const int64_t* __restrict__ rp,
                         const int32_t* __restrict__ ci, const double* __restrict__ cv,
                         int32_t* __restrict__ ec, double* __restrict__ ev) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t b = rp[r], e = rp[r + 1];
  for (int k = 0; k < w; ++k) {
    const int64_t o = (int64_t)k * rows + r;
    if (b + k < e) {
      const int32_t c = ci[b + k];
      if (sg) {
        ec[o] = cv[b + k] < 0 ? ~c : c;
      } else {
        ec[o] = c;
        ev[o] = cv[b + k];
      }
    } else if (sg) {
      ec[o] = kPad;
    } else {
      ec[o] = e > b ? ci[b] : 0;
      ev[o] = 0.0;
    }
  }
}

// CSR -> sliced layout, one warp per slice
__global__ void k_to_sell(int64_t n_slices, bool sg, const int64_t* __restrict__ srow,
                          const int64_t* __restrict__ sptr, const int32_t* __restrict__ sw,
                          const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ cv, int32_t* __restrict__ sc,
                          double* __restrict__ sv) {
  const int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= n_slices) return;
  const int64_t r0 = srow[sl], nr = srow[sl + 1] - r0;
  if (lane >= nr) return;
  const int64_t r = r0 + lane, b = rp[r], e = rp[r + 1];
  for (int k = 0; k < sw[sl]; ++k) {
    const int64_t o = sptr[sl] + (int64_t)k * nr + lane;
    if (b + k < e) {
      const int32_t c = ci[b + k];
      if (sg) {
        sc[o] = cv[b + k] < 0 ? ~c : c;
      } else {
        sc[o] = c;
        sv[o] = cv[b + k];
      }
    } else if (sg) {
      sc[o] = kPad;
    } else {
      sc[o] = e > b ? ci[b] : 0;
      sv[o] = 0.0;
    }
  }
}

}  // namespace

void DevOperator::upload_device(DevCSR&& d, cudaStream_t s) {
  rows = d.rows;
  cols = d.cols;
  nnz = d.nnz;
  layout = kCsr;
  const double avg = rows ? (double)nnz / (double)rows : 0.0;
  tpr = 1;
  while (tpr < 32 && tpr * 2 <= avg) tpr *= 2;
  if (rows == 0 || nnz == 0 || wide_rows(avg)) {
    adopt_csr(std::move(d));
    return;
  }
  std::vector<int64_t> hrp((size_t)rows + 1);
  SFEEC_CUDA(cudaMemcpyAsync(hrp.data(), d.rp.p, sizeof(int64_t) * hrp.size(),
                             cudaMemcpyDeviceToHost, s));
  DevBuf<int> flag;
  flag.alloc(1);
  flag.zero(s);
  k_abs_uniform<<<148 * 8, 256, 0, s>>>(nnz, d.val.p, flag.p);
  SFEEC_LAUNCH_CHECK();
  int not_uniform = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&not_uniform, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  // the same layout decisions as upload()
  std::vector<int64_t> hrow{0}, hptr{0};
  std::vector<int32_t> hw;
  int64_t wmax = 0;
  for (int64_t r = 0; r < rows; ++r) wmax = std::max(wmax, hrp[(size_t)r + 1] - hrp[(size_t)r]);
  {
    int64_t r = 0;
    while (r < rows) {
      int64_t w = hrp[(size_t)r + 1] - hrp[(size_t)r];
      int64_t e = r + 1;
      while (e < rows && e - r < 32) {
        int64_t l = hrp[(size_t)e + 1] - hrp[(size_t)e];
        int64_t tol = std::max<int64_t>(1, std::max(w, l) / 8);
        if (std::llabs(l - w) > tol) break;
        w = std::max(w, l);
        ++e;
      }
      hw.push_back((int32_t)w);
      // slice starts 4-entry aligned (16 B of columns: bulk copies, k_sell_tma)
      hptr.push_back(hptr.back() + ((w * (e - r) + 3) & ~int64_t(3)));
      hrow.push_back(e);
      r = e;
    }
  }
  n_slices = (int64_t)hw.size();
  const bool signed_ok = not_uniform == 0;
  const double rows_per_slice = (double)rows / (double)n_slices;
  const double pad_ratio = (double)hptr.back() / (double)nnz;
  if (rows_per_slice >= 8 && signed_ok && pad_ratio <= 2.5) {
    layout = kSigned;
    SFEEC_CUDA(cudaMemcpyAsync(&scale, d.val.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
    scale = std::fabs(scale);
  } else if (rows_per_slice >= 8 && pad_ratio <= 1.15) {
    layout = kSell;
  } else {
    adopt_csr(std::move(d));
    return;
  }
  const bool sg = layout == kSigned;
  const double ell_pad = (double)(rows * wmax) / (double)nnz;
  if (win_enabled() && build_win(d.rp.p, d.ci.p, d.val.p, hrow, hw, s)) {
    d.rp.reset();
    d.ci.reset();
    d.val.reset();
    return;
  }
  const bool ell_ok = wmax >= 1 && wmax <= 8 && ell_pad <= (sg ? 1.3 : 1.1);
  if (delta_enabled() && (ell_ok || dsell_pays(hrow, hw, sg))) {
    if (ell_ok)
      build_dell(d.rp.p, d.ci.p, d.val.p, (int)wmax, s);
    else
      build_dsell(d.rp.p, d.ci.p, d.val.p, hrow, hw, s);
    d.rp.reset();
    d.ci.reset();
    d.val.reset();
    return;
  }
  if (wmax >= 1 && wmax <= 8 && ell_pad <= (sg ? 1.3 : 1.1)) {
    ell = true;
    ell_w = (int)wmax;
    sell_entries = rows * wmax;
    sell_col.alloc((size_t)sell_entries);
    if (!sg) sell_val.alloc((size_t)sell_entries);
    k_to_ell<<<blocks_for(rows), kThreads, 0, s>>>(rows, ell_w, sg, d.rp.p, d.ci.p, d.val.p,
                                                   sell_col.p, sell_val.p);
  } else {
    sell_entries = hptr.back();
    slice_row.upload(hrow.data(), hrow.size(), s);
    slice_ptr.upload(hptr.data(), hptr.size(), s);
    slice_w.upload(hw.data(), hw.size(), s);
    if (!sg) prepare_sell_tma();
    sell_col.alloc((size_t)sell_entries + 4);  // + the alignment over-read of k_sell_tma
    if (!sg) sell_val.alloc((size_t)sell_entries + 4);
    k_to_sell<<<blocks_for(n_slices * 32), kThreads, 0, s>>>(n_slices, sg, slice_row.p,
                                                             slice_ptr.p, slice_w.p, d.rp.p,
                                                             d.ci.p, d.val.p, sell_col.p,
                                                             sell_val.p);
  }
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
  d.rp.reset();
  d.ci.reset();
  d.val.reset();
}

double DevOperator::stream_bytes() const {
  if (win && layout != kCsr)
    return (layout == kSell ? 8.0 * (double)sell_val.n : 0.0) + 2.0 * (double)dcol.n +
           (double)sizeof(DSlice) * (double)dslice.n +
           (double)sizeof(WUnit) * (double)wunit.n + 8.0 * (double)wseg.n;
  if (delta && layout != kCsr)
    return (layout == kSell ? 8.0 * (double)sell_val.n : 0.0) + 2.0 * (double)dcol.n +
           4.0 * (double)dbase.n + (ell ? 4.0 * (double)(dfull.n + sell_col.n)
                                        : (double)sizeof(DSlice) * (double)dslice.n);
  const double meta = ell ? 0.0 : 20.0 * (double)n_slices;
  switch (layout) {
    case kSigned:
      return 4.0 * (double)sell_entries + meta;
    case kSell:
      return 12.0 * (double)sell_entries + meta;
    default:
      return 12.0 * (double)nnz + 8.0 * (double)(rows + 1);
  }
}

void DevOperator::download_csr(int64_t* row_ptr, int32_t* col_idx, double* v,
                               cudaStream_t s) const {
  if (row_ptr)
    SFEEC_CUDA(cudaMemcpyAsync(row_ptr, rp.p, sizeof(int64_t) * (size_t)(rows + 1),
                               cudaMemcpyDeviceToHost, s));
  if (col_idx && nnz)
    SFEEC_CUDA(cudaMemcpyAsync(col_idx, ci.p, sizeof(int32_t) * (size_t)nnz,
                               cudaMemcpyDeviceToHost, s));
  if (v && nnz)
    SFEEC_CUDA(cudaMemcpyAsync(v, val.p, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToHost,
                               s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
}

void launch_spmv_strict(const DevOperator& a, const double* x, double* y, cudaStream_t s) {
  if (a.rows == 0) return;
  k_csr_strict<false><<<blocks_for(a.rows), kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p,
                                                              x, y, 0.0);
  SFEEC_LAUNCH_CHECK();
}

void launch_spmv_axpy_strict(const DevOperator& a, const double* x, double* y, double alpha,
                             cudaStream_t s) {
  if (a.rows == 0) return;
  k_csr_strict<true><<<blocks_for(a.rows), kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p,
                                                             x, y, alpha);
  SFEEC_LAUNCH_CHECK();
}

template <bool ACC>
static void launch_vec(const DevOperator& a, const double* x, double* y, double alpha,
                       cudaStream_t s) {
  unsigned g = blocks_for(a.rows * a.tpr);
  if (a.tpr == 32) {
    const char* env = std::getenv("SFEEC_WIDE_U");
    const int u = env ? std::atoi(env) : 4;
    if (u == 2)
      k_csr_wide<ACC, 2><<<g, kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p, x, y, alpha);
    else if (u == 8)
      k_csr_wide<ACC, 8><<<g, kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p, x, y, alpha);
    else
      k_csr_wide<ACC, 4><<<g, kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p, x, y, alpha);
    return;
  }
  switch (a.tpr) {
#define SFEEC_TPR(T)                                                                   \
  case T:                                                                              \
    k_csr_vec<T, ACC><<<g, kThreads, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p, x, y, alpha); \
    break;
    SFEEC_TPR(1)
    SFEEC_TPR(2)
    SFEEC_TPR(4)
    SFEEC_TPR(8)
    SFEEC_TPR(16)
    SFEEC_TPR(32)
#undef SFEEC_TPR
    default:
      throw Error(SFEEC_ECUDA, "bad threads-per-row");
  }
}

template <bool ACC, bool SG>
static void launch_delta_t(const DevOperator& a, const double* x, double* y, double alpha,
                           cudaStream_t s) {
  const double sc = SG ? a.scale : 1.0;
  if (a.ell) {
    const unsigned g = blocks_for(a.rows);
#define SFEEC_DELL_W(W)                                                                     \
  case W:                                                                                   \
    k_dell<ACC, SG, W><<<g, kThreads, 0, s>>>(a.rows, a.dbase.p, a.dcol.p, a.dfull.p,      \
                                              a.sell_col.p, a.sell_val.p, sc, x, y, alpha); \
    break;
    switch (a.ell_w) {
      SFEEC_DELL_W(1)
      SFEEC_DELL_W(2)
      SFEEC_DELL_W(3)
      SFEEC_DELL_W(4)
      SFEEC_DELL_W(5)
      SFEEC_DELL_W(6)
      SFEEC_DELL_W(7)
      SFEEC_DELL_W(8)
      default:
        throw Error(SFEEC_ECUDA, "bad ELL width");
    }
#undef SFEEC_DELL_W
  } else {
    // SFEEC_DSELL_MB: resident CTAs per SM (3: 85 registers, 4: 64)
    const char* env = std::getenv("SFEEC_DSELL_MB");
    const int mb = env ? std::atoi(env) : 4;
    auto grid = [&](int m) {
      return (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 32), 148 * m);
    };
    if (mb == 4)
      k_dsell<ACC, SG, 4><<<grid(4), kThreads, 0, s>>>(a.n_slices, a.dslice.p, a.dbase.p,
                                                       a.dcol.p, a.sell_val.p, sc, x, y, alpha);
    else
      k_dsell<ACC, SG, 3><<<grid(3), kThreads, 0, s>>>(a.n_slices, a.dslice.p, a.dbase.p,
                                                       a.dcol.p, a.sell_val.p, sc, x, y, alpha);
  }
  SFEEC_LAUNCH_CHECK();
}

static void launch_delta(const DevOperator& a, const double* x, double* y, double alpha,
                         bool accumulate, cudaStream_t s) {
  const bool sg = a.layout == DevOperator::kSigned;
  if (accumulate) {
    if (sg)
      launch_delta_t<true, true>(a, x, y, alpha, s);
    else
      launch_delta_t<true, false>(a, x, y, alpha, s);
  } else {
    if (sg)
      launch_delta_t<false, true>(a, x, y, alpha, s);
    else
      launch_delta_t<false, false>(a, x, y, alpha, s);
  }
}

// SFEEC_L2PF: L2 hints in k_ell and the default k_sell_pipe: bits 0-1 the
// prefetch size of the operator streams (1 = 128 B, 2 = 256 B), bit 2 an
// evict_last policy on the gathered x (valid: 0, 1, 2, 4, 6); results unchanged
// k_ell and k_sell_pipe are launched as programmatic dependents
// (device_util.cuh), so each one's launch and operator prefetch overlap the
// previous kernel's tail; results unchanged. Measured: tet16 (launch-bound)
// 0.0109 -> 0.0090 ms/step, tet128 +0.3%. SFEEC_PDL=0 turns it off.
static bool pdl_enabled() {
  const char* e = std::getenv("SFEEC_PDL");
  return !(e && std::atoi(e) == 0);
}

static int l2_prefetch_size() {
  const char* e = std::getenv("SFEEC_L2PF");
  return e ? std::atoi(e) : 0;
}

void launch_spmv(const DevOperator& a, const double* x, double* y, double alpha,
                 bool accumulate, cudaStream_t s, bool reverse) {
  const int rev = reverse ? 1 : 0;  // k_ell / k_sell_pipe only; the others ignore it
  const int l2pf = l2_prefetch_size();  // k_ell / k_sell_pipe streaming-load hint
  const bool pdl = pdl_enabled();        // k_ell / k_sell_pipe programmatic launches
  if (a.rows == 0) return;
  if (a.nnz == 0) {
    if (!accumulate) SFEEC_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)a.rows, s));
    return;
  }
  if (a.layout == DevOperator::kStencil) {
    launch_stencil(*a.st, x, y, alpha, accumulate, s);
    return;
  }
  if (a.win && a.layout != DevOperator::kCsr) {
    launch_win(a, x, y, alpha, accumulate, s);
    return;
  }
  if (a.delta && a.layout != DevOperator::kCsr) {
    launch_delta(a, x, y, alpha, accumulate, s);
    return;
  }
  if (a.ell && a.layout != DevOperator::kCsr) {
    const unsigned g = blocks_for(a.rows);
    const bool sg = a.layout == DevOperator::kSigned;
#define SFEEC_ELL_PF(W, PF)                                                                   \
  if (sg) {                                                                                  \
    if (accumulate)                                                                          \
      launch_pdl(pdl, k_ell<true, true, W, PF>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, (const double*)nullptr, a.scale, x, y, alpha, rev); \
    else                                                                                     \
      launch_pdl(pdl, k_ell<false, true, W, PF>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, (const double*)nullptr, a.scale, x, y, alpha, rev); \
  } else {                                                                                   \
    if (accumulate)                                                                          \
      launch_pdl(pdl, k_ell<true, false, W, PF>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, a.sell_val.p, 1.0, x, y, alpha, rev); \
    else                                                                                     \
      launch_pdl(pdl, k_ell<false, false, W, PF>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, a.sell_val.p, 1.0, x, y, alpha, rev); \
  }
#define SFEEC_ELL_W(W)                                                                       \
  case W:                                                                                    \
    if (l2pf == 1) {                                                                         \
      SFEEC_ELL_PF(W, 1)                                                                     \
    } else if (l2pf == 2) {                                                                  \
      SFEEC_ELL_PF(W, 2)                                                                     \
    } else if (l2pf == 4) {                                                                  \
      SFEEC_ELL_PF(W, 4)                                                                     \
    } else if (l2pf == 6) {                                                                  \
      SFEEC_ELL_PF(W, 6)                                                                     \
    } else {                                                                                 \
      SFEEC_ELL_PF(W, 0)                                                                     \
    }                                                                                        \
    break;
    switch (a.ell_w) {
      SFEEC_ELL_W(1)
      SFEEC_ELL_W(2)
      SFEEC_ELL_W(3)
      SFEEC_ELL_W(4)
      SFEEC_ELL_W(5)
      SFEEC_ELL_W(6)
      SFEEC_ELL_W(7)
      SFEEC_ELL_W(8)
      default:
        throw Error(SFEEC_ECUDA, "bad ELL width");
    }
#undef SFEEC_ELL_W
#undef SFEEC_ELL_PF
    SFEEC_LAUNCH_CHECK();
    return;
  }
  // persistent grid sized to the residency of the chosen variant (148 SMs x
  // MINB CTAs of 8 warps); one warp per slice per iteration.
  // SFEEC_SELL_VARIANT selects (CH, MINB) for tuning: 0 -> (8,3), 1 -> (4,4), 2 -> (6,4)
  // default: the software-pipelined fp64 sliced kernel (variant 9); variant 1
  // is the previous non-pipelined k_sell (CH 4, MINB 4). Measured (K-Q):
  // tet128 4.77 -> 5.27 TB/s, config 4 (64^3 P2) 4.65 -> 5.07 TB/s.
  const char* venv = std::getenv("SFEEC_SELL_VARIANT");
  const int variant = venv ? std::atoi(venv) : 9;
  const char* senv = std::getenv("SFEEC_SELL_SVARIANT");
  const int svariant = senv ? std::atoi(senv) : 0;
  auto grid_for = [&](int minb) {
    return (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 32), 148 * minb);
  };
#define SFEEC_SELL_V(ACC, SG, CH, MB)                                                     \
  k_sell<ACC, SG, CH, MB><<<grid_for(MB), kThreads, 0, s>>>(                             \
      a.n_slices, a.slice_row.p, a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p,  \
      a.scale, x, y, alpha)
#define SFEEC_SELL(ACC, SG)                 \
  do {                                      \
    if (SG) {                               \
      if (svariant == 1)                    \
        SFEEC_SELL_V(ACC, SG, 4, 6);        \
      else if (svariant == 2)               \
        SFEEC_SELL_V(ACC, SG, 2, 8);        \
      else if (svariant == 3)               \
        SFEEC_SELL_V(ACC, SG, 8, 4);        \
      else                                  \
        SFEEC_SELL_V(ACC, SG, 4, 4);        \
    } else if (variant == 1)                \
      SFEEC_SELL_V(ACC, SG, 4, 4);          \
    else if (variant == 4)                  \
      SFEEC_SELL_V(ACC, SG, 8, 4);          \
    else if (variant == 8)                  \
      SFEEC_SELL_V(ACC, SG, 16, 2);         \
    else if (variant == 2)                  \
      SFEEC_SELL_V(ACC, SG, 4, 5);          \
    else if (variant == 3)                  \
      SFEEC_SELL_V(ACC, SG, 2, 8);          \
    else                                    \
      SFEEC_SELL_V(ACC, SG, 8, 3);          \
  } while (0)
  switch (a.layout) {
    case DevOperator::kSigned:
      if (accumulate)
        SFEEC_SELL(true, true);
      else
        SFEEC_SELL(false, true);
      break;
    case DevOperator::kSell:
      if (sell_tma_enabled() && !venv) {
        launch_sell_tma(a, x, y, alpha, accumulate, s);
      } else if (variant >= 14 && variant <= 16) {
#define SFEEC_PF(CH, MB)                                                                          \
  do {                                                                                            \
    const unsigned g9 = (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 32), 148 * MB);       \
    if (accumulate)                                                                               \
      k_sell_pf<true, CH, MB><<<g9, kThreads, 0, s>>>(a.n_slices, a.slice_row.p, a.slice_ptr.p,   \
          a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha, (int64_t)std::min(a.sell_col.n, a.sell_val.n));           \
    else                                                                                          \
      k_sell_pf<false, CH, MB><<<g9, kThreads, 0, s>>>(a.n_slices, a.slice_row.p, a.slice_ptr.p,  \
          a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha, (int64_t)std::min(a.sell_col.n, a.sell_val.n));           \
  } while (0)
        if (variant == 15)
          SFEEC_PF(2, 4);
        else if (variant == 16)
          SFEEC_PF(4, 3);
        else
          SFEEC_PF(4, 4);
#undef SFEEC_PF
      } else if (variant >= 9 && variant <= 13) {
#define SFEEC_PIPE_PF(CH, MB, PF)                                                                 \
  do {                                                                                            \
    const unsigned g9 = (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 32), 148 * MB);       \
    if (accumulate)                                                                               \
      launch_pdl(pdl, k_sell_pipe<true, CH, MB, PF>, dim3(g9), dim3(kThreads), 0, s, a.n_slices,  \
          a.slice_row.p, a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha, rev); \
    else                                                                                          \
      launch_pdl(pdl, k_sell_pipe<false, CH, MB, PF>, dim3(g9), dim3(kThreads), 0, s, a.n_slices, \
          a.slice_row.p, a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha, rev); \
  } while (0)
#define SFEEC_PIPE(CH, MB) SFEEC_PIPE_PF(CH, MB, 0)
        if (variant == 10)
          SFEEC_PIPE(2, 4);
        else if (variant == 11)
          SFEEC_PIPE(4, 5);
        else if (variant == 12)
          SFEEC_PIPE(2, 8);
        else if (variant == 13)
          SFEEC_PIPE(3, 6);
        else if (l2pf == 1)
          SFEEC_PIPE_PF(4, 4, 1);
        else if (l2pf == 2)
          SFEEC_PIPE_PF(4, 4, 2);
        else if (l2pf == 4)
          SFEEC_PIPE_PF(4, 4, 4);
        else if (l2pf == 6)
          SFEEC_PIPE_PF(4, 4, 6);
        else
          SFEEC_PIPE(4, 4);
#undef SFEEC_PIPE
#undef SFEEC_PIPE_PF
      } else if (variant >= 5) {
#define SFEEC_TPR2(CH, MB)                                                                   \
  do {                                                                                       \
    const unsigned g2 = (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 64), 148 * MB);  \
    if (accumulate)                                                                          \
      k_sell_tpr2<true, CH, MB><<<g2, kThreads, 0, s>>>(a.n_slices, a.slice_row.p,           \
          a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha);              \
    else                                                                                     \
      k_sell_tpr2<false, CH, MB><<<g2, kThreads, 0, s>>>(a.n_slices, a.slice_row.p,          \
          a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y, alpha);              \
  } while (0)
        if (variant == 5)
          SFEEC_TPR2(8, 4);
        else if (variant == 6)
          SFEEC_TPR2(4, 4);
        else
          SFEEC_TPR2(8, 3);
#undef SFEEC_TPR2
      } else if (accumulate) {
        SFEEC_SELL(true, false);
      } else {
        SFEEC_SELL(false, false);
      }
      break;
    default:
      if (accumulate)
        launch_vec<true>(a, x, y, alpha, s);
      else
        launch_vec<false>(a, x, y, alpha, s);
  }
#undef SFEEC_SELL
#undef SFEEC_SELL_V
  SFEEC_LAUNCH_CHECK();
}

void launch_axpy(double* y, const double* x, double alpha, int64_t n, bool strict,
                 cudaStream_t s) {
  if (n == 0) return;
  unsigned g = (unsigned)std::min<int64_t>(blocks_for(n), 148 * 16);
  k_axpy<<<g, kThreads, 0, s>>>(y, x, alpha, n, strict ? 1 : 0);
  SFEEC_LAUNCH_CHECK();
}

void launch_scale_copy(double* x, const double* y, double /*inv*/, double nrm, int64_t n,
                       cudaStream_t s) {
  if (n == 0) return;
  unsigned g = (unsigned)std::min<int64_t>(blocks_for(n), 148 * 16);
  k_div_copy<<<g, kThreads, 0, s>>>(x, y, nrm, n);
  SFEEC_LAUNCH_CHECK();
}

}  // namespace sfeec_b200
