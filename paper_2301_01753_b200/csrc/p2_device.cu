// Second-order (P2^-) system on the device, BASELINE config 4: S(M1^2)
// pattern with the M1^2 values, the SPAI on that pattern, Q_sym and C^T.
//
// The S(M1^2) SPAI solves, per column l, the normal equations of
// min ||M q - e_l|| over the 2-ring pattern I_l (spai.cpp:127-286):
// Gram G = (M^2)(I_l, I_l) of order k ~ 250-470, rhs = M(l, I_l), Cholesky
// with the 1e-12 trace pivot test. 9.8M such solves at 64^3 are ~1e14 flop,
// so each column is a CTA: G in a per-CTA global workspace (L2), panels of
// 32 columns factored in shared memory, the trailing update as 4x4 register
// tiles from the panel, blocked triangular solves. Columns that fail the
// pivot test are reported (the eigenvalue-thresholded fallback is host-only).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dev_handle.hpp"
#include "device_util.cuh"
#include "p2_device.hpp"
#include "table_lattice.cuh"
#include "spmv_kernels.cuh"
#include "tet_device.hpp"

namespace sfeec_b200 {

namespace {

inline unsigned nblk2(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

constexpr int kMaxM1Row = 96;  // lists merged per S(M1^2) row (3 per lane)

// S(M1^2) row i = sorted union of the rows of M1 listed in row i; with vals,
// (M1^2)(i, c) = sum_k M1(i, k) M1(k, c) in ascending k, separate rounding
// (bitwise the host sparse_square order, host_tet.cpp sq_entry). Warp per
// row, a 3-list-per-lane merge. Pass 1 (cnt != null) counts, pass 2 fills.
__global__ void k_sq_rows(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ val, int64_t* __restrict__ cnt,
                          const int64_t* __restrict__ orp, int32_t* __restrict__ oci,
                          double* __restrict__ oval, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t b = rp[i];
  const int len = (int)(rp[i + 1] - b);
  if (len > kMaxM1Row) {
    if (lane == 0) *bad = 1;
    return;
  }
  int64_t pos[3], end[3];
  int head[3];
  double w[3];  // M1(i, k) of this lane's lists
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int t = lane + 32 * j;
    if (t < len) {
      const int32_t k = ci[b + t];
      w[j] = val[b + t];
      pos[j] = rp[k];
      end[j] = rp[k + 1];
    } else {
      w[j] = 0.0;
      pos[j] = end[j] = 0;
    }
    head[j] = pos[j] < end[j] ? ci[pos[j]] : INT_MAX;
  }
  int64_t out = cnt ? 0 : orp[i];
  for (;;) {
    int m = min(head[0], min(head[1], head[2]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (m == INT_MAX) break;
    if (!cnt) {
      // contributions of the lists whose head is m, summed in ascending list
      // index t = lane + 32 j (= ascending k)
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const bool hit = head[j] == m;
        const double pr = hit ? __dmul_rn(w[j], val[pos[j]]) : 0.0;
        unsigned bits = __ballot_sync(0xffffffffu, hit);
        while (bits) {
          const int src = __ffs(bits) - 1;
          bits &= bits - 1;
          s = __dadd_rn(s, __shfl_sync(0xffffffffu, pr, src));
        }
      }
      if (lane == 0) {
        oci[out] = m;
        oval[out] = s;
      }
    }
    ++out;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (head[j] == m) {
        ++pos[j];
        head[j] = pos[j] < end[j] ? ci[pos[j]] : INT_MAX;
      }
  }
  if (cnt && lane == 0) cnt[i] = out;
}

// ---- large-pattern SPAI ----------------------------------------------------
constexpr int kT = 512;    // threads per CTA
constexpr int kNb = 32;    // panel width
constexpr int kKmax = 512; // largest pattern column (= kT: a panel row per thread)

struct SpaiSmem {
  double panel[kKmax * kNb];
  double y[kKmax];
  double x[kKmax];
  double lbb[kNb * kNb];
  int32_t idx[kKmax];
  double red[kT / 32];
  double colj[kNb];
  double piv;
};

__device__ __forceinline__ int find_sorted(const int32_t* a, int k, int32_t v) {
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < k && a[lo] == v) ? lo : -1;
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kT / 32; ++w) s += red[w];
  return s;
}

__global__ void __launch_bounds__(kT, 1)
    k_spai_big(int64_t n, const int64_t* __restrict__ prp, const int32_t* __restrict__ pci,
               const double* __restrict__ pval, const int64_t* __restrict__ mrp,
               const int32_t* __restrict__ mci, const double* __restrict__ mval,
               double* __restrict__ ws, double* __restrict__ qcol, int32_t* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SpaiSmem& S = *reinterpret_cast<SpaiSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* G = ws + (size_t)blockIdx.x * kKmax * kKmax;
  for (int64_t l = blockIdx.x; l < n; l += gridDim.x) {
    const int64_t b0 = prp[l];
    const int k = (int)(prp[l + 1] - b0);
    const int ld = k;
    for (int a = tid; a < k; a += kT) {
      S.idx[a] = pci[b0 + a];
      S.y[a] = 0.0;
    }
    for (int bcol = warp; bcol < k; bcol += kT / 32)  // lower triangle only
      for (int a = bcol + lane; a < k; a += 32) G[a + (int64_t)bcol * ld] = 0.0;
    __syncthreads();
    // Gram: G(a, b) = (M^2)(I_a, I_b), lower triangle (I_b <= I_a)
    for (int a = warp; a < k; a += kT / 32) {
      const int32_t row = S.idx[a];
      const int64_t s = prp[row], e = prp[row + 1];
      for (int64_t t = s + lane; t < e; t += 32) {
        const int32_t c = pci[t];
        if (c > row) break;
        const int bb = find_sorted(S.idx, a + 1, c);
        if (bb >= 0) G[a + (int64_t)bb * ld] = pval[t];
      }
    }
    // rhs(a) = M(l, I_a)
    for (int64_t t = mrp[l] + tid; t < mrp[l + 1]; t += kT) {
      const int bb = find_sorted(S.idx, k, mci[t]);
      if (bb >= 0) S.y[bb] = mval[t];
    }
    __syncthreads();
    double tr = 0.0;
    for (int a = tid; a < k; a += kT) tr += G[a + (int64_t)a * ld];
    const double trace = block_sum(tr, S.red);
    // ---- blocked right-looking Cholesky, G = L L^T (lower, in place) ----
    double dmin = INFINITY;
    bool ok = true;
    for (int p0 = 0; p0 < k && ok; p0 += kNb) {
      const int w = min(kNb, k - p0), m = k - p0;
      // panel factorization with the panel rows in registers: thread i owns
      // panel row i (m <= kKmax = kT); per column: pivot, scale, rank-1 update
      // of the later panel columns from the broadcast column j
      double* P = S.panel;  // P[i + j m]: the factored panel, for the trailing update
      const int i = tid;
      double r[kNb];
#pragma unroll
      for (int j = 0; j < kNb; ++j)
        r[j] = (i < m && j < w && i >= j) ? G[(p0 + i) + (int64_t)(p0 + j) * ld] : 0.0;
#pragma unroll
      for (int j = 0; j < kNb; ++j) {
        if (j < w && ok) {  // uniform
          if (i == j) S.piv = r[j];
          __syncthreads();
          const double d = S.piv;
          if (d > 0.0) {
            dmin = fmin(dmin, d);
            const double inv = rsqrt(d);  // one rsqrt instead of sqrt + divide per step
            if (i == j)
              r[j] = d * inv;
            else if (i > j)
              r[j] = r[j] * inv;
            if (i > j && i < w) S.colj[i] = r[j];
          } else {
            ok = false;
          }
          __syncthreads();
          if (ok) {
#pragma unroll
            for (int jj = j + 1; jj < kNb; ++jj)
              if (jj < w && i >= jj) r[jj] = fma(-r[j], S.colj[jj], r[jj]);
          }
        }
      }
      if (!ok) break;
      if (i < m) {
#pragma unroll
        for (int j = 0; j < kNb; ++j)
          if (j < w) {
            P[i + j * m] = r[j];
            if (i >= j) G[(p0 + i) + (int64_t)(p0 + j) * ld] = r[j];
          }
      }
      __syncthreads();
      // trailing update of rows / cols [p0 + w, k): 64 x 64 tiles, 4 x 4 per
      // thread, two 256-thread groups on alternate tiles; the G tile is loaded
      // before the panel products so its latency overlaps them
      const int mt = m - w;
      const int ntile = (mt + 63) / 64;
      const int t256 = tid & 255, grp = tid >> 8;
      const int tx = t256 & 15, ty = t256 >> 4;
      for (int tile = grp; tile < ntile * (ntile + 1) / 2; tile += kT / 256) {
        int ti = 0;
        while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
        const int tj = tile - ti * (ti + 1) / 2;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int r = ti * 64 + tx + 16 * u, c = tj * 64 + ty + 16 * v;
            acc[u][v] = (r < mt && c < mt && r >= c)
                            ? G[(p0 + w + r) + (int64_t)(p0 + w + c) * ld] : 0.0;
          }
        for (int t = 0; t < w; ++t) {
          double a[4], bv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int r = ti * 64 + tx + 16 * u;
            a[u] = r < mt ? P[w + r + t * m] : 0.0;
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int c = tj * 64 + ty + 16 * v;
            bv[v] = c < mt ? P[w + c + t * m] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(-a[u], bv[v], acc[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int r = ti * 64 + tx + 16 * u, c = tj * 64 + ty + 16 * v;
            if (r < mt && c < mt && r >= c) G[(p0 + w + r) + (int64_t)(p0 + w + c) * ld] = acc[u][v];
          }
      }
      __syncthreads();
    }
    // uniform decision (every thread saw the same pivots)
    ok = ok && dmin > 1e-12 * trace;
    if (ok) {
      // forward: L z = rhs, right-looking by 32-row blocks
      for (int p0 = 0; p0 < k; p0 += kNb) {
        const int w = min(kNb, k - p0);
        for (int e = tid; e < kNb * kNb; e += kT) {
          const int i = e % kNb, j = e / kNb;
          S.lbb[e] = (i < w && j < w && i >= j) ? G[(p0 + i) + (int64_t)(p0 + j) * ld] : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
          double yi = lane < w ? S.y[p0 + lane] : 0.0;
          for (int j = 0; j < w; ++j) {
            const double yj = __shfl_sync(0xffffffffu, yi, j) / S.lbb[j + j * kNb];
            if (lane == j) yi = yj;
            if (lane > j) yi -= S.lbb[lane + j * kNb] * yj;
          }
          if (lane < w) S.x[p0 + lane] = yi;
        }
        __syncthreads();
        for (int i = p0 + w + tid; i < k; i += kT) {
          double s = 0.0;
          for (int t = 0; t < w; ++t) s = fma(G[i + (int64_t)(p0 + t) * ld], S.x[p0 + t], s);
          S.y[i] -= s;
        }
        __syncthreads();
      }
      // backward: L^T q = z, by 32-row blocks from the bottom; q overwrites x
      for (int p0 = ((k - 1) / kNb) * kNb; p0 >= 0; p0 -= kNb) {
        const int w = min(kNb, k - p0);
        // z_B -= L(>B, B)^T q(>B): one dot per column of the block, a warp each
        for (int j = warp; j < w; j += kT / 32) {
          double s = 0.0;
          for (int i = p0 + w + lane; i < k; i += 32) s = fma(G[i + (int64_t)(p0 + j) * ld], S.x[i], s);
#pragma unroll
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) S.y[p0 + j] = S.x[p0 + j] - s;
        }
        for (int e = tid; e < kNb * kNb; e += kT) {
          const int i = e % kNb, j = e / kNb;
          S.lbb[e] = (i < w && j < w && i >= j) ? G[(p0 + i) + (int64_t)(p0 + j) * ld] : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
          double zi = lane < w ? S.y[p0 + lane] : 0.0;
          for (int j = w - 1; j >= 0; --j) {
            const double xj = __shfl_sync(0xffffffffu, zi, j) / S.lbb[j + j * kNb];
            if (lane == j) zi = xj;
            if (lane < j) zi -= S.lbb[j + lane * kNb] * xj;
          }
          if (lane < w) S.x[p0 + lane] = zi;
        }
        __syncthreads();
      }
      bool fin = true;
      for (int a = tid; a < k; a += kT) {
        const double q = S.x[a];
        fin = fin && isfinite(q);
        qcol[b0 + a] = q;
      }
      fin = __syncthreads_and(fin);
      if (tid == 0) flags[l] = fin ? 0 : 1;
    } else {
      for (int a = tid; a < k; a += kT) qcol[b0 + a] = 0.0;
      if (tid == 0) flags[l] = 1;
    }
    __syncthreads();
  }
}

}  // namespace

void square_pattern_device(const DevCSR& m1, DevCSR& out, cudaStream_t s) {
  const int64_t n = m1.rows;
  out.rows = out.cols = n;
  out.rp.alloc((size_t)n + 1);
  DevBuf<int> bad;
  bad.alloc(1);
  bad.zero(s);
  SFEEC_CUDA(cudaMemsetAsync(out.rp.p, 0, sizeof(int64_t) * (size_t)(n + 1), s));
  k_sq_rows<<<nblk2(n * 32, 256), 256, 0, s>>>(n, m1.rp.p, m1.ci.p, m1.val.p, out.rp.p, nullptr,
                                                 nullptr, nullptr, bad.p);
  SFEEC_LAUNCH_CHECK();
  int hb = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  require(hb == 0, "S(M1^2): an M1 row exceeds 96 entries");
  exclusive_scan(out.rp.p, n, s);
  SFEEC_CUDA(cudaMemcpyAsync(&out.nnz, out.rp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  out.ci.alloc((size_t)std::max<int64_t>(1, out.nnz));
  out.val.alloc((size_t)std::max<int64_t>(1, out.nnz));
  k_sq_rows<<<nblk2(n * 32, 256), 256, 0, s>>>(n, m1.rp.p, m1.ci.p, m1.val.p, nullptr, out.rp.p,
                                                 out.ci.p, out.val.p, bad.p);
  SFEEC_LAUNCH_CHECK();
}

int64_t spai_big_device(const DevCSR& m1, const DevCSR& sq, DevBuf<double>& qcol, cudaStream_t s) {
  const int64_t n = m1.rows;
  // largest column of the pattern
  std::vector<int64_t> hrp((size_t)n + 1);
  SFEEC_CUDA(cudaMemcpyAsync(hrp.data(), sq.rp.p, sizeof(int64_t) * hrp.size(),
                             cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  int64_t kmax = 0;
  for (int64_t i = 0; i < n; ++i) kmax = std::max(kmax, hrp[(size_t)i + 1] - hrp[(size_t)i]);
  require(kmax <= kKmax, "device SPAI: a pattern column exceeds 512 entries");
  int dev = 0, sms = 148;
  SFEEC_CUDA(cudaGetDevice(&dev));
  SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)std::min<int64_t>(n, sms);
  DevBuf<double> ws;
  ws.alloc((size_t)grid * kKmax * kKmax);
  DevBuf<int32_t> flags;
  flags.alloc((size_t)std::max<int64_t>(1, n));
  qcol.alloc((size_t)std::max<int64_t>(1, sq.nnz));
  const size_t smem = sizeof(SpaiSmem);
  SFEEC_CUDA(cudaFuncSetAttribute(k_spai_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  SFEEC_CUDA(cudaEventCreate(&e0));
  SFEEC_CUDA(cudaEventCreate(&e1));
  SFEEC_CUDA(cudaEventRecord(e0, s));
  k_spai_big<<<grid, kT, smem, s>>>(n, sq.rp.p, sq.ci.p, sq.val.p, m1.rp.p, m1.ci.p, m1.val.p, ws.p,
                                    qcol.p, flags.p);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaEventRecord(e1, s));
  if (std::getenv("SFEEC_VERBOSE")) {
    float ms = 0;
    SFEEC_CUDA(cudaEventSynchronize(e1));
    SFEEC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    std::fprintf(stderr, "sfeec spai: %lld columns, k_max %lld, kernel %.1f ms (%.2f us/column/CTA)\n",
                 (long long)n, (long long)kmax, ms, 1e3 * ms * grid / (double)n);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::vector<int32_t> hf((size_t)n);
  SFEEC_CUDA(cudaMemcpyAsync(hf.data(), flags.p, sizeof(int32_t) * hf.size(), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  int64_t fb = 0;
  for (int32_t f : hf) fb += f != 0;
  return fb;
}

void build_p2_system_device(const TetMesh& mesh, const P2Dofs& dofs, bool want_div,
                            DevP2System& out, cudaStream_t s) {
  const bool verbose = std::getenv("SFEEC_VERBOSE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!verbose) return;
    SFEEC_CUDA(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "sfeec p2 setup: %-28s %8.3f s\n", what,
                 std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  auto up = [&](HostCSR&& h, DevCSR& d) {
    d.rows = h.rows;
    d.cols = h.cols;
    d.nnz = (int64_t)h.val.size();
    d.rp.upload(h.row_ptr.data(), h.row_ptr.size(), s);
    d.ci.upload(h.col_idx.data(), std::max<size_t>(1, h.col_idx.size()), s);
    d.val.upload(h.val.data(), std::max<size_t>(1, h.val.size()), s);
    SFEEC_CUDA(cudaStreamSynchronize(s));
  };
  out.n1 = dofs.n1;
  out.n2 = dofs.n2;
  out.n3 = dofs.n3;
  DevCSR m1;
  up(p2_mass(mesh, dofs, 1), m1);
  lap("host M1 + upload");
  up(p2_curl(mesh, dofs), out.c);
  up(p2_mass(mesh, dofs, 2), out.m2);
  if (want_div) up(p2_div(mesh, dofs), out.d);
  lap("host C, M2, D + upload");
  DevCSR sq;
  square_pattern_device(m1, sq, s);
  lap("S(M1^2) pattern + values");
  DevBuf<double> qcol;
  out.fallback = spai_big_device(m1, sq, qcol, s);
  lap("SPAI (device)");
  require(out.fallback == 0,
          "device SPAI: some columns need the eigenvalue-thresholded fallback; use the host builder");
  m1 = DevCSR();
  sq.val.reset();  // M1^2 values no longer needed; Q_sym reuses the pattern
  out.qsym.rows = out.qsym.cols = dofs.n1;
  out.qsym.nnz = sq.nnz;
  out.qsym.val.alloc((size_t)std::max<int64_t>(1, sq.nnz));
  qsym_device(dofs.n1, sq.rp.p, sq.ci.p, qcol.p, out.qsym.val.p, s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
  out.qsym.rp = std::move(sq.rp);
  out.qsym.ci = std::move(sq.ci);
  transpose_dev(out.c, out.ct, s);
  lap("Q_sym + C^T");
}

}  // namespace sfeec_b200

using namespace sfeec_b200;


namespace {

HostCSR download_csr(DevCSR& a, cudaStream_t s) {
  HostCSR h;
  h.rows = a.rows;
  h.cols = a.cols;
  h.row_ptr.resize((size_t)a.rows + 1);
  h.col_idx.resize((size_t)a.nnz);
  h.val.resize((size_t)a.nnz);
  SFEEC_CUDA(cudaMemcpyAsync(h.row_ptr.data(), a.rp.p, sizeof(int64_t) * h.row_ptr.size(),
                             cudaMemcpyDeviceToHost, s));
  if (a.nnz) {
    SFEEC_CUDA(cudaMemcpyAsync(h.col_idx.data(), a.ci.p, sizeof(int32_t) * (size_t)a.nnz,
                               cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaMemcpyAsync(h.val.data(), a.val.p, sizeof(double) * (size_t)a.nnz,
                               cudaMemcpyDeviceToHost, s));
  }
  SFEEC_CUDA(cudaStreamSynchronize(s));
  return h;
}

// (type, vertex) of every P2- DOF for the table lattice: 1-forms = edge type
// t, moment s -> 2 t + s, then face type f, moment s -> 14 + 2 f + s; 2-forms
// = face f, moment s -> 3 f + s, then tet permutation p, moment s -> 36 + 3 p
// + s at the cube's lowest vertex (the order of p2_mesh.hpp's numbering)
void p2_table_dofs(const TetMesh& m, const P2Dofs& d, TLDofs& d1, TLDofs& d2) {
  d1.ntypes = 38;
  d1.mb = 2;  // both moments of an edge / face couple to the same entities: 2 x 2 blocks
  d2.ntypes = 54;
  d2.mb = 3;  // the three moments of a face / tet: 3 x 3 blocks of M2
  d1.type.resize((size_t)d.n1);
  d1.vertex.resize((size_t)d.n1);
  d2.type.resize((size_t)d.n2);
  d2.vertex.resize((size_t)d.n2);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < d.n1; ++r) {
    const int64_t ent = d.ent1[(size_t)r];
    const int kind = d.ks1[(size_t)r] & 1, slot = d.ks1[(size_t)r] >> 1;
    if (kind == 0) {
      d1.type[(size_t)r] = 2 * m.edge_t[(size_t)ent] + slot;
      d1.vertex[(size_t)r] = m.edge_v[(size_t)ent];
    } else {
      d1.type[(size_t)r] = 14 + 2 * m.face_t[(size_t)ent] + slot;
      d1.vertex[(size_t)r] = m.face_v[(size_t)ent];
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < d.n2; ++r) {
    const int64_t ent = d.ent2[(size_t)r];
    const int kind = d.ks2[(size_t)r] & 1, slot = d.ks2[(size_t)r] >> 1;
    if (kind == 0) {
      d2.type[(size_t)r] = 3 * m.face_t[(size_t)ent] + slot;
      d2.vertex[(size_t)r] = m.face_v[(size_t)ent];
    } else {
      const int64_t cube = ent / 6;
      const int i = (int)(cube % m.n), j = (int)((cube / m.n) % m.n);
      const int k = (int)(cube / ((int64_t)m.n * m.n));
      d2.type[(size_t)r] = 36 + 3 * (int)(ent % 6) + slot;
      d2.vertex[(size_t)r] = m.vid(i, j, k);
    }
  }
}

struct P2Stream {
  cudaStream_t s = nullptr;
  P2Stream() { SFEEC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~P2Stream() {
    if (s) cudaStreamDestroy(s);
  }
};

}  // namespace

extern "C" {

int sfeec_p2_dev_create(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                        int split_kind, int device, int flags, int with_div, sfeec_dev** out,
                        int64_t* counts) {
  return guarded([&] {
    require(out != nullptr, "null out");
    *out = nullptr;
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    select_device(device);
    TetMesh mesh;
    mesh.build(n, jitter, seed);
    P2Dofs dofs;
    dofs.build(mesh);
    P2Stream st;
    DevP2System sys;
    build_p2_system_device(mesh, dofs, with_div != 0, sys, st.s);
    if (counts) {
      counts[0] = sys.n1;
      counts[1] = sys.n2;
      counts[2] = sys.n3;
      counts[3] = sys.qsym.nnz;
      counts[4] = sys.fallback;
    }
    // advance() runs on the table-driven Kuhn lattice (table_lattice.cuh):
    // Q_sym and M2 as per-vertex coefficient arrays with each symmetric pair
    // stored once, C / C^T as constants of the slot tables; the sliced / ELL
    // operators below serve every other entry point. Small meshes are
    // launch-bound either way and keep the sliced step.
    std::unique_ptr<LatticeOps> lat;
    const bool want_lat = !(flags & SFEEC_STRICT) && !(flags & SFEEC_TET_NO_LATTICE) &&
                          (n >= 12 || ((flags & SFEEC_TET_LATTICE) && n >= 6));
    if (want_lat) {
      TLDofs d1, d2;
      p2_table_dofs(mesh, dofs, d1, d2);
      auto tl = std::make_unique<TableLattice>();
      tl->build(n, 2, d1, d2, sys.qsym, sys.m2, sys.c, sys.ct, st.s);
      lat = std::move(tl);
    }
    mesh = TetMesh();
    dofs = P2Dofs();
    DevOperator q, c, ct, m2, div;
    q.upload_device(std::move(sys.qsym), st.s);
    m2.upload_device(std::move(sys.m2), st.s);
    c.upload_device(std::move(sys.c), st.s);
    ct.upload_device(std::move(sys.ct), st.s);
    if (with_div) div.upload_device(std::move(sys.d), st.s);
    cudaStream_t hs;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
    *out = make_dev_from_ops(std::move(q), std::move(c), std::move(ct), std::move(m2),
                             with_div ? &div : nullptr, sys.n1, sys.n2, dt, eps0, mu0, split_kind,
                             device, flags & ~(SFEEC_TET_NO_LATTICE | SFEEC_TET_LATTICE), hs,
                             std::move(lat));
  });
}

int sfeec_p2_dev_operators(int n, double jitter, uint64_t seed, int device, sfeec_csr_owned* c,
                           sfeec_csr_owned* m2, sfeec_csr_owned* d, sfeec_csr_owned* q_sym,
                           sfeec_csr_owned* ct) {
  return guarded([&] {
    select_device(device);
    TetMesh mesh;
    mesh.build(n, jitter, seed);
    P2Dofs dofs;
    dofs.build(mesh);
    P2Stream st;
    DevP2System sys;
    build_p2_system_device(mesh, dofs, d != nullptr, sys, st.s);
    if (c) csr_to_owned(download_csr(sys.c, st.s), c);
    if (m2) csr_to_owned(download_csr(sys.m2, st.s), m2);
    if (d) csr_to_owned(download_csr(sys.d, st.s), d);
    if (q_sym) csr_to_owned(download_csr(sys.qsym, st.s), q_sym);
    if (ct) csr_to_owned(download_csr(sys.ct, st.s), ct);
  });
}

// S(M1^2) pattern + M1^2 values and the SPAI columns of a caller's M1 (for
// tests of the large-pattern solver against the host SPAI)
int sfeec_p2_spai_device(const sfeec_csr* m1, int device, sfeec_csr_owned* q, int64_t* fallback) {
  return guarded([&] {
    require(m1 && q, "null argument");
    csr_validate(*m1, "M1");
    require(m1->rows == m1->cols, "spai: square operator required");
    select_device(device);
    P2Stream st;
    HostCSR hm = csr_from_view(*m1);
    DevCSR dm;
    dm.rows = hm.rows;
    dm.cols = hm.cols;
    dm.nnz = (int64_t)hm.val.size();
    dm.rp.upload(hm.row_ptr.data(), hm.row_ptr.size(), st.s);
    dm.ci.upload(hm.col_idx.data(), std::max<size_t>(1, hm.col_idx.size()), st.s);
    dm.val.upload(hm.val.data(), std::max<size_t>(1, hm.val.size()), st.s);
    DevCSR sq;
    square_pattern_device(dm, sq, st.s);
    DevBuf<double> qcol;
    const int64_t fb = spai_big_device(dm, sq, qcol, st.s);
    if (fallback) *fallback = fb;
    // Q by rows: Q(i, l) = q_l[pos of i in I_l]; with a symmetric pattern
    // that is the transpose of the column layout
    DevCSR qt;
    qt.rows = qt.cols = hm.rows;
    qt.nnz = sq.nnz;
    qt.rp = std::move(sq.rp);
    qt.ci = std::move(sq.ci);
    qt.val = std::move(qcol);
    DevCSR qr;
    transpose_dev(qt, qr, st.s);
    csr_to_owned(download_csr(qr, st.s), q);
  });
}

}  // extern "C"
