// Windowed sliced SpMV (WUnit in spmv_kernels.cuh): the gathered neighbour
// values of a unit of rows are staged in shared memory by bulk async copies
// (cp.async.bulk + mbarrier transaction counts), so the per-entry gather is a
// shared-memory load instead of an L2 round trip, and a column costs a 16-bit
// window index instead of a 32-bit id. The operator stream (values + indices)
// is the only HBM traffic of any size: the x window of a unit is a few
// contiguous id ranges that L2 already holds (the units run in row order, so
// neighbouring units re-read the same vertex planes).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "spmv_kernels.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kCB = 32;             // columns per window block (256 B of x)
constexpr int kBitWords = 8192;     // bitmap words per unit: 262144 blocks of span
constexpr int kScanThreads = 512;
constexpr unsigned kWPad = 0xffffu;  // pad slot: contributes 0
constexpr int kWConsumers = 8;       // consumer warps per CTA
constexpr int kWThreads = 32 * (kWConsumers + 1);  // + one producer warp
constexpr int kWSmem = 2 * kWinCap * 8 + 64;       // two window buffers + 4 mbarriers

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void w_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void w_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void w_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void w_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WWAIT_%=;\n}" ::"r"(s_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(s_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(s_u32(bar))
      : "memory");
}

__device__ __forceinline__ DSlice load_dslice(const DSlice* __restrict__ meta, int64_t i) {
  const int4* p = reinterpret_cast<const int4*>(meta + i);
  const int4 a = __ldg(p), b = __ldg(p + 1);
  DSlice m;
  m.r0 = ((int64_t)(unsigned)a.y << 32) | (unsigned)a.x;
  m.vptr = ((int64_t)(unsigned)a.w << 32) | (unsigned)a.z;
  m.dptr = ((int64_t)(unsigned)b.y << 32) | (unsigned)b.x;
  m.bptr = b.z;
  m.nw = b.w;
  return m;
}

__device__ __forceinline__ unsigned wcode(uint4 d, int j) {
  const unsigned w = j < 2 ? d.x : j < 4 ? d.y : j < 6 ? d.z : d.w;
  return (j & 1) ? (w >> 16) : (w & 0xffffu);
}

// one slice's streamed operands in registers (NARROW: <= 8 entries, codes
// entry-major; wide: the first 16 entries = two chunks of 8; entries beyond
// 16 are loaded when the slice is computed)
template <bool ACC, bool SIGNED, bool NARROW>
struct SliceRegs {
  static constexpr int E = NARROW ? 8 : 16;
  int64_t row, dptr, vptr;
  int w, nr, it;
  uint32_t c[E / 2];  // two codes per register
  double v[SIGNED ? 1 : E];
  double y0;
};

template <bool ACC, bool SIGNED, bool NARROW>
__device__ __forceinline__ void slice_load(SliceRegs<ACC, SIGNED, NARROW>& r, const DSlice& m,
                                           int it, int lane, const uint16_t* __restrict__ dcol,
                                           const double* __restrict__ val,
                                           const double* __restrict__ y) {
  constexpr int E = SliceRegs<ACC, SIGNED, NARROW>::E;
  r.w = m.nw & 0xfffff;
  r.nr = (m.nw >> 20) & 63;
  r.it = it;
  r.dptr = m.dptr;
  r.vptr = m.vptr;
  r.row = m.r0 + lane;
  if (lane >= r.nr) return;
  if (NARROW) {
    const uint16_t* cp = dcol + m.dptr + lane;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const unsigned lo = j < r.w ? (unsigned)__ldcs(cp + j * r.nr) : kWPad;
      const unsigned hi = j + 1 < r.w ? (unsigned)__ldcs(cp + (j + 1) * r.nr) : kWPad;
      r.c[j / 2] = lo | (hi << 16);
    }
  } else {
    const uint4* dp = reinterpret_cast<const uint4*>(dcol + m.dptr) + lane;
    const uint4 pad = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    const uint4 a = r.w > 0 ? __ldcs(dp) : pad;
    const uint4 b = r.w > 8 ? __ldcs(dp + r.nr) : pad;
    r.c[0] = a.x, r.c[1] = a.y, r.c[2] = a.z, r.c[3] = a.w;
    r.c[4] = b.x, r.c[5] = b.y, r.c[6] = b.z, r.c[7] = b.w;
  }
  if (!SIGNED) {
    const double* vp = val + m.vptr + lane;
#pragma unroll
    for (int j = 0; j < E; ++j) r.v[j] = j < r.w ? __ldcs(vp + j * r.nr) : 0.0;
  }
  r.y0 = ACC ? y[r.row] : 0.0;
}

template <bool SIGNED>
__device__ __forceinline__ void win_acc(double& acc, unsigned cd, double v,
                                        const double* win) {
  const double xv = cd != kWPad ? win[SIGNED ? (cd >> 1) : cd] : 0.0;
  if (SIGNED)
    acc += (cd & 1u) ? -xv : xv;
  else
    acc = fma(v, xv, acc);
}

template <bool ACC, bool SIGNED, bool NARROW>
__device__ __forceinline__ void slice_compute(const SliceRegs<ACC, SIGNED, NARROW>& r,
                                              const double* win, int lane,
                                              const uint16_t* __restrict__ dcol,
                                              const double* __restrict__ val, double scale,
                                              double* __restrict__ y, double alpha) {
  constexpr int E = SliceRegs<ACC, SIGNED, NARROW>::E;
  if (lane >= r.nr) return;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < E; ++j)
    win_acc<SIGNED>(acc, (r.c[j / 2] >> (16 * (j & 1))) & 0xffffu, SIGNED ? 0.0 : r.v[j], win);
  if (!NARROW && r.w > 16) {  // wider rows: the remaining chunks, one at a time
    const uint4* dp = reinterpret_cast<const uint4*>(dcol + r.dptr) + lane;
    const double* vp = SIGNED ? nullptr : val + r.vptr + lane;
    for (int k0 = 16; k0 < r.w; k0 += 8) {
      const uint4 d = __ldcs(dp + (k0 >> 3) * r.nr);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = (!SIGNED && k0 + j < r.w) ? __ldcs(vp + (k0 + j) * r.nr) : 0.0;
        win_acc<SIGNED>(acc, wcode(d, j), v, win);
      }
    }
  }
  const double res = SIGNED ? scale * acc : acc;
  y[r.row] = ACC ? fma(alpha, res, r.y0) : res;
}

// ---- the SpMV -------------------------------------------------------------
// Persistent, one CTA per SM (~225 KB of shared memory). The last warp is the
// producer: for unit i it waits until the 8 consumer warps released buffer
// i&1 (their use for unit i-2), then issues the unit's segment copies into
// it. Consumer warps take the unit's slices warp-strided, one lane per row,
// rows summed in CSR order; the next slice's codes / values / y are loaded
// before the current slice's shared-memory gathers.
template <bool ACC, bool SIGNED, bool NARROW>
__global__ void __launch_bounds__(kWThreads, 1)
    k_win(int64_t n_units, const WUnit* __restrict__ units, const int2* __restrict__ segs,
          const DSlice* __restrict__ meta, const uint16_t* __restrict__ dcol,
          const double* __restrict__ val, double scale, const double* __restrict__ x,
          int64_t xcols, double* __restrict__ y, double alpha) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* wb = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + 2 * kWinCap * 8);
  uint64_t* empty = full + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    w_mbar_init(&full[0], 1);
    w_mbar_init(&full[1], 1);
    w_mbar_init(&empty[0], kWConsumers);
    w_mbar_init(&empty[1], kWConsumers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  if (warp == kWConsumers) {
    if (lane != 0) return;
    int it = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += G, ++it) {
      const int b = it & 1;
      if (it >= 2) w_mbar_wait(&empty[b], ((it >> 1) - 1) & 1);
      const WUnit U = units[u];
      double* dst = wb + b * kWinCap;
      uint32_t bytes = 0;
      for (int j = 0; j < U.nseg; ++j) {
        const int2 sg = segs[U.seg0 + j];
        const int len = (j + 1 < U.nseg ? segs[U.seg0 + j + 1].y : U.wsize) - sg.y;
        const int64_t rem = xcols - sg.x, n = len < rem ? len : rem;
        bytes += (uint32_t)(n & ~int64_t(1)) * 8u;
        if (n & 1) dst[sg.y + n - 1] = x[sg.x + n - 1];  // an odd tail: not 16 B
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      w_mbar_expect_tx(&full[b], bytes);  // release: orders the tail stores
      for (int j = 0; j < U.nseg; ++j) {
        const int2 sg = segs[U.seg0 + j];
        const int len = (j + 1 < U.nseg ? segs[U.seg0 + j + 1].y : U.wsize) - sg.y;
        const int64_t rem = xcols - sg.x, n = (len < rem ? len : rem) & ~int64_t(1);
        if (n) bulk_g2s(dst + sg.y, x + sg.x, (uint32_t)n * 8u, &full[b]);
      }
    }
    return;
  }
  // consumers: the warp's slices of its units in order; the codes / values / y
  // of the next slice are loaded before the current one is computed (its
  // gathers need only the window), across unit boundaries too
  const int64_t wstride = kWConsumers;
  int64_t lu = blockIdx.x, ls = 0, lend = 0;
  int lit = 0;
  auto seek = [&]() {  // the first slice of this warp at or after (lu, ls)
    while (lu < n_units && ls >= lend) {
      lu += G;
      ++lit;
      if (lu < n_units) {
        const WUnit U = units[lu];
        ls = U.s0 + warp;
        lend = U.s0 + U.ns;
      }
    }
  };
  if (lu < n_units) {
    const WUnit U = units[lu];
    ls = U.s0 + warp;
    lend = U.s0 + U.ns;
    seek();
  }
  // the metadata of the slice at the cursor is loaded one slice earlier still
  SliceRegs<ACC, SIGNED, NARROW> A, B;
  DSlice mc;
  bool have_a = lu < n_units;
  if (have_a) {
    slice_load(A, load_dslice(meta, ls), lit, lane, dcol, val, y);
    ls += wstride;
    seek();
    if (lu < n_units) mc = load_dslice(meta, ls);
  }
  int it = 0;
  for (int64_t u = blockIdx.x; u < n_units; u += G, ++it) {
    const int b = it & 1;
    w_mbar_wait(&full[b], (it >> 1) & 1);  // every warp, so arrivals stay per use
    const double* win = wb + b * kWinCap;
    while (have_a && A.it == it) {
      const bool have_b = lu < n_units;
      if (have_b) {
        slice_load(B, mc, lit, lane, dcol, val, y);
        ls += wstride;
        seek();
        if (lu < n_units) mc = load_dslice(meta, ls);
      }
      slice_compute(A, win, lane, dcol, val, scale, y, alpha);
      A = B;
      have_a = have_b;
    }
    __syncwarp();
    if (lane == 0) w_mbar_arrive(&empty[b]);
  }
}

// ---- the build --------------------------------------------------------------
__device__ __forceinline__ void unit_entries(const int64_t* __restrict__ us,
                                             const int64_t* __restrict__ srow,
                                             const int64_t* __restrict__ rp, int64_t u,
                                             int64_t* e0, int64_t* e1) {
  *e0 = rp[srow[us[u]]];
  *e1 = rp[srow[us[u + 1]]];
}

template <class T, class Op>
__device__ T block_reduce(T v, Op op, T* red) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = red[0];
  for (int i = 1; i < nwarps; ++i) r = op(r, red[i]);
  return r;
}

// the unit's window-block bitmap in shared memory; returns false if the
// column span is too wide (then *cb0 is meaningless)
__device__ bool unit_bitmap(const int32_t* __restrict__ ci, int64_t e0, int64_t e1,
                            uint32_t* bm, int* red, int* cb0, int* nwords) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int c = ci[e];
    mn = min(mn, c);
    mx = max(mx, c);
  }
  mn = block_reduce(mn, [](int a, int b) { return min(a, b); }, red);
  mx = block_reduce(mx, [](int a, int b) { return max(a, b); }, red);
  *cb0 = mn / kCB;
  const int64_t span = (int64_t)(mx / kCB) - *cb0 + 1;
  if (span > (int64_t)kBitWords * 32) return false;
  *nwords = (int)((span + 31) / 32);
  for (int i = threadIdx.x; i < *nwords; i += blockDim.x) bm[i] = 0;
  __syncthreads();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int bi = ci[e] / kCB - *cb0;
    atomicOr(&bm[bi >> 5], 1u << (bi & 31));
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ uint32_t run_starts(const uint32_t* bm, int i) {
  return bm[i] & ~((bm[i] << 1) | (i > 0 ? bm[i - 1] >> 31 : 0u));
}

// pass 1: window size and segment count per unit (INT_MAX: span too wide)
__global__ void __launch_bounds__(kScanThreads)
    k_win_scan(int64_t n_units, const int64_t* __restrict__ us, const int64_t* __restrict__ srow,
               const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
               int32_t* __restrict__ wsize, int32_t* __restrict__ nseg) {
  __shared__ uint32_t bm[kBitWords];
  __shared__ int red[32];
  const int64_t u = blockIdx.x;
  int64_t e0, e1;
  unit_entries(us, srow, rp, u, &e0, &e1);
  if (e1 == e0) {
    if (threadIdx.x == 0) wsize[u] = nseg[u] = 0;
    return;
  }
  int cb0, nw;
  if (!unit_bitmap(ci, e0, e1, bm, red, &cb0, &nw)) {
    if (threadIdx.x == 0) wsize[u] = nseg[u] = INT_MAX;
    return;
  }
  int pop = 0, runs = 0;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) {
    pop += __popc(bm[i]);
    runs += __popc(run_starts(bm, i));
  }
  pop = block_reduce(pop, [](int a, int b) { return a + b; }, red);
  runs = block_reduce(runs, [](int a, int b) { return a + b; }, red);
  if (threadIdx.x == 0) {
    wsize[u] = pop * kCB;
    nseg[u] = runs;
  }
}

// pass 2: segments, codes and values (slice layout, chunks of 8 per lane)
__global__ void __launch_bounds__(kScanThreads)
    k_win_fill(int64_t n_units, const int64_t* __restrict__ us, const int64_t* __restrict__ srow,
               const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const double* __restrict__ cv, bool sg, bool narrow,
               const WUnit* __restrict__ units, const DSlice* __restrict__ meta,
               int2* __restrict__ segs,
               uint16_t* __restrict__ dcol, double* __restrict__ sv) {
  extern __shared__ uint32_t dsm[];
  uint32_t* bm = dsm;                 // kBitWords
  uint32_t* rk = dsm + kBitWords;     // exclusive rank prefix per word
  __shared__ int red[32];
  __shared__ int tsum[2][kScanThreads];
  const int64_t u = blockIdx.x;
  int64_t e0, e1;
  unit_entries(us, srow, rp, u, &e0, &e1);
  if (e1 == e0) return;  // empty rows only: no codes (their slices have w = 0)
  int cb0, nw;
  if (!unit_bitmap(ci, e0, e1, bm, red, &cb0, &nw)) return;  // cannot happen after pass 1
  // exclusive scans of popcounts and run starts: thread t owns words
  // [t*per, (t+1)*per)
  const int per = (nw + blockDim.x - 1) / blockDim.x;
  const int w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
  int p = 0, r = 0;
  for (int i = w0; i < w1; ++i) {
    p += __popc(bm[i]);
    r += __popc(run_starts(bm, i));
  }
  tsum[0][threadIdx.x] = p;
  tsum[1][threadIdx.x] = r;
  __syncthreads();
  if (threadIdx.x < 2) {  // serial scan of 512 partials (setup only)
    int run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int v = tsum[threadIdx.x][t];
      tsum[threadIdx.x][t] = run;
      run += v;
    }
  }
  __syncthreads();
  p = tsum[0][threadIdx.x];
  r = tsum[1][threadIdx.x];
  const WUnit U = units[u];
  for (int i = w0; i < w1; ++i) {
    rk[i] = p;
    uint32_t st = run_starts(bm, i);
    while (st) {
      const int bit = __ffs(st) - 1;
      st &= st - 1;
      const int rank = p + __popc(bm[i] & ((1u << bit) - 1u));
      segs[U.seg0 + r] = make_int2((cb0 + i * 32 + bit) * kCB, rank * kCB);
      ++r;
    }
    p += __popc(bm[i]);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int64_t s = U.s0 + warp; s < U.s0 + U.ns; s += nwarps) {
    const DSlice m = meta[s];
    const int w = m.nw & 0xfffff, nr = (m.nw >> 20) & 63;
    if (lane >= nr) continue;
    const int64_t row = m.r0 + lane, b = rp[row], e = rp[row + 1];
    const int w8 = narrow ? w : (w + 7) & ~7;
    for (int k = 0; k < w8; ++k) {
      unsigned code = kWPad;
      if (b + k < e) {
        const int c = ci[b + k];
        const int bi = c / kCB - cb0;
        const int idx = (int)(rk[bi >> 5] + __popc(bm[bi >> 5] & ((1u << (bi & 31)) - 1u))) * kCB +
                        c % kCB;
        code = sg ? ((unsigned)idx << 1) | (cv[b + k] < 0 ? 1u : 0u) : (unsigned)idx;
      }
      dcol[narrow ? m.dptr + (int64_t)k * nr + lane
                  : m.dptr + (int64_t)(k >> 3) * 8 * nr + 8 * lane + (k & 7)] = (uint16_t)code;
      if (!sg && k < w) sv[m.vptr + (int64_t)k * nr + lane] = b + k < e ? cv[b + k] : 0.0;
    }
  }
}

}  // namespace

// SFEEC_WIN_NARROW=1 also windows the narrow operators (C, C^T, M2: <= 8
// per row); off by default: the one-thread-per-row ELL kernels keep more
// rows in flight per SM than the consumer warps (measured at tet128:
// K-M2 0.36 -> 0.67 ms, K-Cb 0.17 -> 0.46 ms with one slice in flight per warp)
static bool win_narrow_enabled() {
  const char* e = std::getenv("SFEEC_WIN_NARROW");
  return e && std::atoi(e) == 1;
}

// SFEEC_WIN=1 selects the windowed layout for the wide operators. Off by
// default: measured at tet128 K-Q 0.570 ms (int32 sliced, k_sell_pipe) ->
// 0.637 (16 consumer warps, one slice in flight each) -> 0.777 (8 warps, next
// slice prefetched): too few bytes in flight per SM with register staging.
bool win_enabled() {
  const char* e = std::getenv("SFEEC_WIN");
  return e && std::atoi(e) == 1;
}

bool DevOperator::build_win(const int64_t* drp, const int32_t* dci, const double* dv,
                            const std::vector<int64_t>& hrow, const std::vector<int32_t>& hw,
                            cudaStream_t s) {
  const bool sg = layout == kSigned;
  const int64_t ns_all = (int64_t)hw.size();
  if (ns_all == 0 || cols >= (int64_t)INT32_MAX) return false;
  for (int32_t w : hw)
    if (w >= (1 << 20)) return false;
  static bool attr = false;
  if (!attr) {
#define SFEEC_WIN_ATTR(A, B, C)                                                  \
  SFEEC_CUDA(cudaFuncSetAttribute(k_win<A, B, C>,                                \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem))
    SFEEC_WIN_ATTR(false, false, false);
    SFEEC_WIN_ATTR(true, false, false);
    SFEEC_WIN_ATTR(false, true, false);
    SFEEC_WIN_ATTR(true, true, false);
    SFEEC_WIN_ATTR(false, false, true);
    SFEEC_WIN_ATTR(true, false, true);
    SFEEC_WIN_ATTR(false, true, true);
    SFEEC_WIN_ATTR(true, true, true);
#undef SFEEC_WIN_ATTR
    SFEEC_CUDA(cudaFuncSetAttribute(k_win_fill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    2 * kBitWords * 4));
    attr = true;
  }
  DevBuf<int64_t> srow;
  srow.upload(hrow.data(), hrow.size(), s);
  std::vector<int64_t> us;
  std::vector<int32_t> hws, hns;
  DevBuf<int64_t> dus;
  DevBuf<int32_t> dws, dns;
  int64_t target = 2048;
  bool ok = false;
  for (; target >= 64; target = target * 3 / 4) {
    us.assign(1, 0);
    int64_t r = 0;
    for (int64_t sl = 0; sl < ns_all; ++sl) {
      const int64_t nr = hrow[(size_t)sl + 1] - hrow[(size_t)sl];
      if (r > 0 && r + nr > target) {
        us.push_back(sl);
        r = 0;
      }
      r += nr;
    }
    us.push_back(ns_all);
    const int64_t nu = (int64_t)us.size() - 1;
    dus.upload(us.data(), us.size(), s);
    dws.alloc((size_t)nu);
    dns.alloc((size_t)nu);
    k_win_scan<<<(unsigned)nu, kScanThreads, 0, s>>>(nu, dus.p, srow.p, drp, dci, dws.p, dns.p);
    SFEEC_LAUNCH_CHECK();
    hws.resize((size_t)nu);
    hns.resize((size_t)nu);
    SFEEC_CUDA(cudaMemcpyAsync(hws.data(), dws.p, 4 * (size_t)nu, cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaMemcpyAsync(hns.data(), dns.p, 4 * (size_t)nu, cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
    if (*std::max_element(hws.begin(), hws.end()) <= kWinCap) {
      ok = true;
      break;
    }
  }
  if (!ok) return false;
  const int64_t nu = (int64_t)us.size() - 1;
  const bool narrow = *std::max_element(hw.begin(), hw.end()) <= 8;
  if (narrow && !win_narrow_enabled()) return false;
  std::vector<DSlice> hm((size_t)ns_all);
  int64_t vp = 0, dp = 0;
  for (int64_t i = 0; i < ns_all; ++i) {
    const int64_t nr = hrow[(size_t)i + 1] - hrow[(size_t)i], w = hw[(size_t)i];
    hm[(size_t)i] = DSlice{hrow[(size_t)i], vp, dp, 0, (int32_t)(w | (nr << 20))};
    vp += w * nr;
    dp += (narrow ? w : (w + 7) & ~int64_t(7)) * nr;
  }
  std::vector<WUnit> hu((size_t)nu);
  int64_t nseg = 0;
  for (int64_t u = 0; u < nu; ++u) {
    hu[(size_t)u] = WUnit{us[(size_t)u], (int32_t)(us[(size_t)u + 1] - us[(size_t)u]),
                          (int32_t)nseg, hns[(size_t)u], hws[(size_t)u], {0, 0}};
    nseg += hns[(size_t)u];
  }
  if (nseg >= (int64_t)INT32_MAX) return false;
  n_slices = ns_all;
  n_units = nu;
  win_rows = target;
  sell_entries = vp;
  dslice.upload(hm.data(), hm.size(), s);
  wunit.upload(hu.data(), hu.size(), s);
  wseg.alloc((size_t)std::max<int64_t>(nseg, 1));
  dcol.alloc((size_t)std::max<int64_t>(dp, 8));
  if (!sg) sell_val.alloc((size_t)std::max<int64_t>(vp, 1));
  k_win_fill<<<(unsigned)nu, kScanThreads, 2 * kBitWords * 4, s>>>(
      nu, dus.p, srow.p, drp, dci, dv, sg, narrow, wunit.p, dslice.p, wseg.p, dcol.p,
      sell_val.p);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
  win = true;
  win_narrow = narrow;
  ell = false;
  delta = false;
  return true;
}

void launch_win(const DevOperator& a, const double* x, double* y, double alpha, bool accumulate,
                cudaStream_t s) {
  if (reinterpret_cast<uintptr_t>(x) & 15)
    throw Error(SFEEC_EINVAL, "windowed SpMV: x must be 16-byte aligned");
  const unsigned g = (unsigned)std::min<int64_t>(a.n_units, 148);
  const bool sg = a.layout == DevOperator::kSigned;
  const double sc = sg ? a.scale : 1.0;
#define SFEEC_WIN_L(ACC, SG)                                                                  \
  do {                                                                                        \
    if (a.win_narrow)                                                                         \
      k_win<ACC, SG, true><<<g, kWThreads, kWSmem, s>>>(a.n_units, a.wunit.p, a.wseg.p,       \
          a.dslice.p, a.dcol.p, a.sell_val.p, sc, x, a.cols, y, alpha);                       \
    else                                                                                      \
      k_win<ACC, SG, false><<<g, kWThreads, kWSmem, s>>>(a.n_units, a.wunit.p, a.wseg.p,      \
          a.dslice.p, a.dcol.p, a.sell_val.p, sc, x, a.cols, y, alpha);                       \
  } while (0)
  if (accumulate) {
    if (sg)
      SFEEC_WIN_L(true, true);
    else
      SFEEC_WIN_L(true, false);
  } else {
    if (sg)
      SFEEC_WIN_L(false, true);
    else
      SFEEC_WIN_L(false, false);
  }
#undef SFEEC_WIN_L
  SFEEC_LAUNCH_CHECK();
}

}  // namespace sfeec_b200
