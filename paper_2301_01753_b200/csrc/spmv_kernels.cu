// SpMV kernels for the leapfrog chain. All are HBM-bound sparse contractions
// (~0.17 flop/byte): no tensor cores; the design goals are contiguous
// (coalesced) streaming of the operator arrays, L1/L2 hits on the gathered
// neighbour values, and enough loads in flight per SM.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "spmv_kernels.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int32_t kPad = 0x7fffffff;  // padding slot in the signed sliced layout

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
template <bool ACC, int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_sell_pipe(int64_t n_slices, const int64_t* __restrict__ srow, const int64_t* __restrict__ sptr,
                const int32_t* __restrict__ sw, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x,
                double* __restrict__ y, double alpha) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  SliceMeta m = load_meta(srow, sptr, sw, s);
  pdl_wait();  // PDL: x and y come from the previous kernels
  pdl_trigger();
  while (true) {
    const int64_t sn = s + nwarps;
    SliceMeta mn;
    if (sn < n_slices) mn = load_meta(srow, sptr, sw, sn);
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
  }
}

// ---- plain ELL for narrow operators: one thread per row ------------------
template <bool ACC, bool SIGNED, int W>
__global__ void __launch_bounds__(kThreads)
    k_ell(int64_t rows, const int32_t* __restrict__ col, const double* __restrict__ val,
          double scale, const double* __restrict__ x, double* __restrict__ y, double alpha) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int32_t p[W];
  double v[W], xv[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    p[k] = __ldcs(col + (int64_t)k * rows + r);
    if (!SIGNED) v[k] = __ldcs(val + (int64_t)k * rows + r);
  }
  // PDL: the operator stream above does not depend on the previous kernel;
  // x and y do (no-ops without a programmatic launch)
  pdl_wait();
  pdl_trigger();
  const double y0 = ACC ? y[r] : 0.0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (SIGNED)
      xv[k] = p[k] != kPad ? __ldg(x + (p[k] < 0 ? ~p[k] : p[k])) : 0.0;
    else
      xv[k] = __ldg(x + p[k]);
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
  if (strict_only || rows == 0 || nnz == 0) {
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
  // narrow operators (C: 3, C^T: <= 6, M2: 7 per row) go to plain ELL: one
  // thread per row, entry k of row r at k*rows + r, no slice metadata and
  // no persistent loop -- the short rows are latency-bound, so every row's
  // loads must be independent and the grid as large as the row count
  int64_t wmax = 0;
  for (int64_t r = 0; r < rows; ++r) wmax = std::max(wmax, h.row_ptr[(size_t)r + 1] - h.row_ptr[(size_t)r]);
  const double ell_pad = (double)(rows * wmax) / (double)nnz;
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
  if (rows == 0 || nnz == 0) {
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
  const bool ell_ok = wmax >= 1 && wmax <= 8 && ell_pad <= (sg ? 1.3 : 1.1);
  if (ell_ok) {
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
    sell_col.alloc((size_t)sell_entries + 4);
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
  if (a.tpr == 32) {  // wide rows: a warp per row, batched loads
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

// k_ell and k_sell_pipe are launched as programmatic dependents when the
// operator's pdl flag is set (device_util.cuh): each one's launch and
// operator-stream loads overlap the previous kernel's tail; results unchanged.
// Measured: tet16 (launch-bound) 0.0109 -> 0.0090 ms/step, tet128 +0.3%.
void launch_spmv(const DevOperator& a, const double* x, double* y, double alpha,
                 bool accumulate, cudaStream_t s) {
  const bool pdl = a.pdl;
  if (a.rows == 0) return;
  if (a.nnz == 0) {
    if (!accumulate) SFEEC_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)a.rows, s));
    return;
  }
  const bool sg = a.layout == DevOperator::kSigned;
  if (a.ell && a.layout != DevOperator::kCsr) {
    const unsigned g = blocks_for(a.rows);
    const double* v = sg ? nullptr : a.sell_val.p;
    const double sc = sg ? a.scale : 1.0;
#define SFEEC_ELL_W(W)                                                                       \
  case W:                                                                                    \
    if (sg && accumulate)                                                                    \
      launch_pdl(pdl, k_ell<true, true, W>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, v, sc, x, y, alpha); \
    else if (sg)                                                                             \
      launch_pdl(pdl, k_ell<false, true, W>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, v, sc, x, y, alpha); \
    else if (accumulate)                                                                     \
      launch_pdl(pdl, k_ell<true, false, W>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, v, sc, x, y, alpha); \
    else                                                                                     \
      launch_pdl(pdl, k_ell<false, false, W>, dim3(g), dim3(kThreads), 0, s, a.rows, a.sell_col.p, v, sc, x, y, alpha); \
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
    SFEEC_LAUNCH_CHECK();
    return;
  }
  // sliced layouts: a persistent grid sized to the residency (148 SMs x 4
  // CTAs of 8 warps), one warp per slice per iteration. fp64 values: the
  // software-pipelined k_sell_pipe (tuned CH 4; measured tet128 K-Q 4.77 ->
  // 5.27 TB/s against the plain k_sell). Signed incidence: k_sell.
  const unsigned grid = (unsigned)std::min<int64_t>(blocks_for(a.n_slices * 32), 148 * 4);
  switch (a.layout) {
    case DevOperator::kSigned:
      if (accumulate)
        k_sell<true, true, 4, 4><<<grid, kThreads, 0, s>>>(a.n_slices, a.slice_row.p,
            a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, a.scale, x, y, alpha);
      else
        k_sell<false, true, 4, 4><<<grid, kThreads, 0, s>>>(a.n_slices, a.slice_row.p,
            a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, a.scale, x, y, alpha);
      break;
    case DevOperator::kSell:
      if (accumulate)
        launch_pdl(pdl, k_sell_pipe<true, 4, 4>, dim3(grid), dim3(kThreads), 0, s, a.n_slices,
                   a.slice_row.p, a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y,
                   alpha);
      else
        launch_pdl(pdl, k_sell_pipe<false, 4, 4>, dim3(grid), dim3(kThreads), 0, s, a.n_slices,
                   a.slice_row.p, a.slice_ptr.p, a.slice_w.p, a.sell_col.p, a.sell_val.p, x, y,
                   alpha);
      break;
    default:
      if (accumulate)
        launch_vec<true>(a, x, y, alpha, s);
      else
        launch_vec<false>(a, x, y, alpha, s);
  }
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
