// Producer -> consumer SpMV pairs of the leapfrog step in ONE persistent
// wavefront kernel each:
//   He:  t = Q_sym e ;  b += alpha C t      (flow_he, reference dynamics.cpp:47-55)
//   Ha:  u = M2 b    ;  e += alpha C^T u    (flow_ha, reference dynamics.cpp:57-67)
// The unfused chain runs these as 4 kernels per step and the intermediates t
// (N1 doubles) and u (N2 doubles) make a round trip through HBM. The tet DOF
// numbering is k-major: a consumer row only references
// producer rows within a vertex plane or two of its own id, so the consumer
// rows can run a short distance behind the producer rows in the same kernel
// and read t / u from L2 while they are still resident.
//
// Work items (host plan, build_wave_plan): producer items are runs of whole
// slices (sliced layout, ~kProdEntries entries) or kEllItem rows (ELL);
// consumer items are kEllItem rows of the consumer ELL operator, each with the
// range [dep_lo, dep_hi] of producer items its columns fall in, placed in the
// item sequence `lag` positions after producer item dep_hi. Warp w of the W
// resident warps takes items w, w + W, w + 2W, ... in sequence order (static:
// a ticket counter serialises on one L2 address, ~3 ns per item, measured);
// an item only waits on earlier items, and with every warp resident the
// smallest unfinished item is always runnable, so the kernel cannot deadlock
// (the grid is sized by the occupancy API; a spin that exceeds ~4 s traps
// instead of hanging the GPU). Producers
// count completed items per block of 64 (warp barrier + red.release.gpu);
// consumers acquire the counters of the blocks their range covers and read t / u with ld.global.cg (L2: another SM's
// L1 may not hold them, and this SM's L1 may hold stale lines).
//
// Every row is computed with exactly the arithmetic of the unfused kernels
// (k_sell_pipe / k_ell in spmv_kernels.cu): results are bitwise identical.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "spmv_kernels.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kWThreads = 256;
constexpr int kWMinBlocks = 4;
constexpr int32_t kWPad = 0x7fffffff;   // padding slot of signed layouts
constexpr int kFlagBase = 32;           // ticket counter alone in its 128 B line
constexpr int kConsumerBit = 1 << 30;   // item.y: count | kConsumerBit
constexpr int kBlockShift = 6;          // producer items per completion counter: 64

struct WaveArgs {
  const int4* items;  // {begin, count | consumer bit, producer: own index;
                      //  consumer: first and last producer block it reads}
  int n_items;
  int n_prod;
  int batch;
  int* sync;          // [0] ticket; completion counters at kFlagBase + producer block
  // producer (sliced: srow/sptr/sw + pcol/pval; ELL: pcol/pval [k*prows + r])
  const int64_t* srow;
  const int64_t* sptr;
  const int32_t* sw;
  const int32_t* pcol;
  const double* pval;
  int64_t prows;
  const double* x;  // producer input (read-only in this kernel)
  double* t;        // intermediate
  // consumer (ELL, [k*crows + r])
  const int32_t* ccol;
  const double* cval;
  int64_t crows;
  double cscale;
  double* y;
  double alpha;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// one slice of the sliced fp64 layout, lane per row: the k_sell_pipe body
// (CH = 4, non-accumulating)
template <int CH>
__device__ __forceinline__ void slice_rows(int64_t r0, int nr, int64_t ptr, int w, int lane,
                                           const int32_t* __restrict__ col,
                                           const double* __restrict__ val,
                                           const double* __restrict__ x, double* __restrict__ y) {
  if (lane >= nr) return;
  const int64_t row = r0 + lane;
  const int64_t base = ptr + lane;
  double acc = 0.0;
  int32_t p[CH];
  double v[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const bool ok = j < w;
    const int64_t o = base + (int64_t)j * nr;
    p[j] = ok ? __ldcs(col + o) : kWPad;
    v[j] = ok ? __ldcs(val + o) : 0.0;
  }
  for (int k0 = 0; k0 < w; k0 += CH) {
    int32_t pn[CH];
    double vn[CH], xv[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const bool ok = k0 + CH + j < w;
      const int64_t o = base + (int64_t)(k0 + CH + j) * nr;
      pn[j] = ok ? __ldcs(col + o) : kWPad;
      vn[j] = ok ? __ldcs(val + o) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) xv[j] = p[j] != kWPad ? __ldg(x + p[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) acc = fma(v[j], xv[j], acc);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      p[j] = pn[j];
      v[j] = vn[j];
    }
  }
  y[row] = acc;
}

template <bool CG>
__device__ __forceinline__ double gather(const double* x, int64_t i) {
  return CG ? __ldcg(x + i) : __ldg(x + i);
}

// ELL rows [r_begin, r_end), R rows per lane per round (rows r, r + 32, ...,
// all their loads issued before any gather): the k_ell body. CG: x was
// written inside this kernel -> L2 reads.
template <bool ACC, bool SIGNED, int W, int R, bool CG>
__device__ __forceinline__ void ell_rows(int64_t rows, const int32_t* __restrict__ col,
                                         const double* __restrict__ val, double scale,
                                         const double* x, double* __restrict__ y, double alpha,
                                         int64_t r_begin, int64_t r_end, int lane) {
  for (int64_t ra = r_begin + lane; ra < r_end; ra += 32 * R) {
    bool on[R];
    int32_t p[R][W];
    double v[R][W], xv[R][W], y0[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int64_t r = ra + 32 * h;
      on[h] = r < r_end;
      y0[h] = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        p[h][k] = on[h] ? __ldcs(col + (int64_t)k * rows + r) : (SIGNED ? kWPad : 0);
        if (!SIGNED) v[h][k] = on[h] ? __ldcs(val + (int64_t)k * rows + r) : 0.0;
      }
      if (ACC && on[h]) y0[h] = y[r];
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (SIGNED)
          xv[h][k] = p[h][k] != kWPad ? gather<CG>(x, p[h][k] < 0 ? ~p[h][k] : p[h][k]) : 0.0;
        else
          xv[h][k] = on[h] ? gather<CG>(x, p[h][k]) : 0.0;
      }
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (SIGNED)
          acc += p[h][k] < 0 ? -xv[h][k] : xv[h][k];
        else
          acc = fma(v[h][k], xv[h][k], acc);
      }
      const double res = SIGNED ? scale * acc : acc;
      if (on[h]) y[ra + 32 * h] = ACC ? fma(alpha, res, y0[h]) : res;
    }
  }
}

// rows per lane per round: ~8-12 entries of each row group in flight
__host__ __device__ constexpr int rows_per_round(int w) { return w <= 2 ? 4 : w <= 4 ? 3 : 2; }

// PW = 0: sliced producer; PW > 0: ELL producer of width PW
template <int PW, bool CSG, int CW>
__global__ void __launch_bounds__(kWThreads, kWMinBlocks) k_wave(WaveArgs a) {
  const int lane = threadIdx.x & 31;
  int* flags = a.sync + kFlagBase;
  // a ticket (atomicAdd on sync[0]) buys `batch` consecutive items; the
  // next ticket is taken at the start of a batch, its latency hidden
  const int batch = a.batch;
  int tk = 0;
  if (lane == 0) tk = atomicAdd(a.sync, 1);
  tk = __shfl_sync(0xffffffffu, tk, 0) * batch;
  while (tk < a.n_items) {
    int nt = 0;
    if (lane == 0) nt = atomicAdd(a.sync, 1);
    const int tend = min(tk + batch, a.n_items);
    for (; tk < tend; ++tk) {
    const int4 it = __ldg(a.items + tk);
    const int count = it.y & (kConsumerBit - 1);
    if (!(it.y & kConsumerBit)) {
      if (PW == 0) {
        // slices [begin, begin + count); next slice's metadata prefetched
        int64_t s = it.x;
        int64_t r0 = __ldg(a.srow + s), r1 = __ldg(a.srow + s + 1), ptr = __ldg(a.sptr + s);
        int w = __ldg(a.sw + s);
        for (int i = 0; i < count; ++i) {
          int64_t r1n = 0, ptrn = 0;
          int wn = 0;
          if (i + 1 < count) {
            r1n = __ldg(a.srow + s + 2);
            ptrn = __ldg(a.sptr + s + 1);
            wn = __ldg(a.sw + s + 1);
          }
          slice_rows<4>(r0, (int)(r1 - r0), ptr, w, lane, a.pcol, a.pval, a.x, a.t);
          ++s;
          r0 = r1;
          r1 = r1n;
          ptr = ptrn;
          w = wn;
        }
      } else {
        constexpr int PWW = PW > 0 ? PW : 1;
        ell_rows<false, false, PWW, rows_per_round(PWW), false>(
            a.prows, a.pcol, a.pval, 1.0, a.x, a.t, 0.0, it.x, (int64_t)it.x + count, lane);
      }
      // warp barrier, then a gpu-scope release by lane 0 (cumulative over the
      // lanes' stores ordered before it by the barrier: the CUTLASS
      // semaphore pattern)
      __syncwarp();
      if (lane == 0) red_release_add(flags + (it.z >> kBlockShift), 1);
    } else {
      // producer blocks [dep_lo, dep_hi] (the plan rounds a consumer's range
      // out to whole blocks and places it after the last one): one counter
      // per block of 2^kBlockShift items, 32 blocks per pass, one round trip
      // when they are complete (the usual case: the plan lags consumers)
      for (int b = it.z + lane; b <= it.w; b += 32) {
        const int need = min(1 << kBlockShift, a.n_prod - (b << kBlockShift));
        if (ld_acquire(flags + b) < need) {
          const long long t0 = clock64();
          while (ld_acquire(flags + b) < need) {
            __nanosleep(32);
            // ~4 s at 2 GHz: a broken plan traps instead of hanging the GPU
            if (clock64() - t0 > (1ll << 33)) __trap();
          }
        }
      }
      __syncwarp();
      ell_rows<true, CSG, CW, rows_per_round(CW), true>(a.crows, a.ccol, a.cval, a.cscale, a.t,
                                                        a.y, a.alpha, it.x,
                                                        (int64_t)it.x + count, lane);
    }
    }
    tk = __shfl_sync(0xffffffffu, nt, 0) * batch;
  }
}

// per consumer item: [min, max] column over its rows, padding skipped
// (signed: kWPad; fp64: value 0 -- stored operators hold no zeros)
__global__ void k_item_colrange(int64_t rows, int w, int sg, const int32_t* __restrict__ col,
                                const double* __restrict__ val, int item_rows, int n_items,
                                int2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int item = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (item >= n_items) return;
  const int64_t r0 = (int64_t)item * item_rows;
  const int64_t r1 = r0 + item_rows < rows ? r0 + item_rows : rows;
  int lo = INT_MAX, hi = -1;
  for (int64_t r = r0 + lane; r < r1; r += 32)
    for (int k = 0; k < w; ++k) {
      const int64_t o = (int64_t)k * rows + r;
      int c = col[o];
      if (sg) {
        if (c == kWPad) continue;
        if (c < 0) c = ~c;
      } else if (val[o] == 0.0) {
        continue;
      }
      lo = min(lo, c);
      hi = max(hi, c);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) out[item] = make_int2(lo, hi);
}

constexpr int kEllItem = 256;          // rows per ELL item (producer or consumer)
constexpr int64_t kProdEntries = 4096;  // target entries per sliced producer item

bool plain_sliced(const DevOperator& a) {
  return a.layout == DevOperator::kSell && !a.ell && !a.delta && !a.win && a.n_slices > 0;
}
bool plain_ell(const DevOperator& a) {
  return (a.layout == DevOperator::kSell || a.layout == DevOperator::kSigned) && a.ell &&
         !a.delta && !a.win;
}

using WaveKernel = void (*)(WaveArgs);

template <int PW, bool CSG>
WaveKernel pick_cw(int cw) {
  switch (cw) {
    case 3: return k_wave<PW, CSG, 3>;
    case 4: return k_wave<PW, CSG, 4>;
    case 6: return k_wave<PW, CSG, 6>;
    case 7: return k_wave<PW, CSG, 7>;
    default: return nullptr;
  }
}
template <int PW>
WaveKernel pick_c(bool csg, int cw) {
  return csg ? pick_cw<PW, true>(cw) : pick_cw<PW, false>(cw);
}
WaveKernel pick_kernel(const DevOperator& p, const DevOperator& c) {
  const bool csg = c.layout == DevOperator::kSigned;
  if (plain_sliced(p)) return pick_c<0>(csg, c.ell_w);
  if (plain_ell(p) && p.layout == DevOperator::kSell) {
    switch (p.ell_w) {
      case 1: return pick_c<1>(csg, c.ell_w);
      case 7: return pick_c<7>(csg, c.ell_w);
      default: return nullptr;
    }
  }
  return nullptr;
}

}  // namespace

// Off by default (SFEEC_WAVE=1 turns it on): measured on B200 at 128^3
// (config 3) the fused step is 1.39-1.40 ms against 1.20 ms for the 4-kernel
// chain. Both halves lose: He 0.87-0.94 ms vs K-Q + K-Cb 0.74, Ha 0.51-0.58
// vs K-M2 + K-CTe 0.49, whatever the item size (1k-16k entries), lag or
// ticket batch. The kernel holds 32 warps per SM (64 registers) where the
// ELL kernels run 64, and a row block's dependency wait replaces the launch
// boundary it saves; the intermediates were never the bound.
bool wave_enabled() {
  const char* e = std::getenv("SFEEC_WAVE");
  return e && std::atoi(e) != 0;
}

bool build_wave_plan(const DevOperator& p, const DevOperator& c, WavePlan& plan,
                     cudaStream_t s) {
  plan = WavePlan();
  plan.built = true;
  if (p.rows == 0 || c.rows == 0 || c.cols != p.rows || !plain_ell(c)) return false;
  WaveKernel kern = pick_kernel(p, c);
  if (!kern) return false;
  if (p.rows >= INT32_MAX || c.rows >= INT32_MAX || p.n_slices >= INT32_MAX) return false;

  // producer items: first row of each (prow), and (begin, count)
  std::vector<int64_t> prow;
  std::vector<int2> pitem;
  if (plain_sliced(p)) {
    std::vector<int64_t> srow((size_t)p.n_slices + 1), sptr((size_t)p.n_slices + 1);
    SFEEC_CUDA(cudaMemcpyAsync(srow.data(), p.slice_row.p, sizeof(int64_t) * srow.size(),
                               cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaMemcpyAsync(sptr.data(), p.slice_ptr.p, sizeof(int64_t) * sptr.size(),
                               cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
    const char* env = std::getenv("SFEEC_WAVE_ENTRIES");
    const int64_t target = env ? std::max<int64_t>(1, std::atoll(env)) : kProdEntries;
    for (int64_t s0 = 0; s0 < p.n_slices;) {
      int64_t s1 = s0 + 1;
      while (s1 < p.n_slices && sptr[(size_t)s1 + 1] - sptr[(size_t)s0] <= target) ++s1;
      prow.push_back(srow[(size_t)s0]);
      pitem.push_back(make_int2((int)s0, (int)(s1 - s0)));
      s0 = s1;
    }
  } else {
    for (int64_t r = 0; r < p.rows; r += kEllItem) {
      prow.push_back(r);
      pitem.push_back(make_int2((int)r, (int)std::min<int64_t>(kEllItem, p.rows - r)));
    }
  }
  const int64_t np = (int64_t)pitem.size();

  // consumer items and their producer-item ranges
  const int nc = (int)((c.rows + kEllItem - 1) / kEllItem);
  DevBuf<int2> rng;
  rng.alloc((size_t)nc);
  k_item_colrange<<<(unsigned)((nc * 32 + 255) / 256), 256, 0, s>>>(
      c.rows, c.ell_w, c.layout == DevOperator::kSigned ? 1 : 0, c.sell_col.p,
      c.layout == DevOperator::kSigned ? nullptr : c.sell_val.p, kEllItem, nc, rng.p);
  SFEEC_LAUNCH_CHECK();
  std::vector<int2> hr((size_t)nc);
  SFEEC_CUDA(cudaMemcpyAsync(hr.data(), rng.p, sizeof(int2) * hr.size(), cudaMemcpyDeviceToHost,
                             s));
  SFEEC_CUDA(cudaStreamSynchronize(s));

  int occ = 0;
  SFEEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWThreads, 0));
  int dev = 0, sms = 0;
  SFEEC_CUDA(cudaGetDevice(&dev));
  SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  occ = std::max(1, std::min(occ, kWMinBlocks));
  const int64_t warps = (int64_t)sms * occ * (kWThreads / 32);
  const char* lenv = std::getenv("SFEEC_WAVE_LAG");
  const char* benv = std::getenv("SFEEC_WAVE_BATCH");
  plan.batch = benv ? std::max(1, std::atoi(benv)) : 2;
  const int64_t lag = lenv ? std::max<int64_t>(0, std::atoll(lenv)) : 2 * warps * plan.batch;

  // sequence: producers in order; consumer j is emitted once the sequence is
  // `lag` positions past its last producer item (a min-heap on that ready
  // position), so it is picked up roughly when that producer has finished
  std::vector<int4> citem((size_t)nc);
  std::vector<int> chi((size_t)nc);
  for (int j = 0; j < nc; ++j) {
    const int64_t r0 = (int64_t)j * kEllItem;
    const int cnt = (int)std::min<int64_t>(kEllItem, c.rows - r0);
    int lo = 0, hi = -1;
    if (hr[(size_t)j].y >= 0) {
      lo = (int)(std::upper_bound(prow.begin(), prow.end(), (int64_t)hr[(size_t)j].x) -
                 prow.begin()) - 1;
      hi = (int)(std::upper_bound(prow.begin(), prow.end(), (int64_t)hr[(size_t)j].y) -
                 prow.begin()) - 1;
    }
    // whole producer blocks: wait on block counters, placed after the block
    const int blo = hi < 0 ? 0 : lo >> kBlockShift, bhi = hi < 0 ? -1 : hi >> kBlockShift;
    citem[(size_t)j] = make_int4((int)r0, cnt | kConsumerBit, blo, bhi);
    chi[(size_t)j] = hi < 0 ? -1 : (int)std::min<int64_t>(np - 1, ((int64_t)bhi + 1 << kBlockShift) - 1);
  }
  // consumers ordered by their last producer item (stable)
  std::vector<int> corder((size_t)nc);
  for (int j = 0; j < nc; ++j) corder[(size_t)j] = j;
  std::stable_sort(corder.begin(), corder.end(),
                   [&](int x, int y) { return chi[(size_t)x] < chi[(size_t)y]; });
  std::vector<int64_t> ppos((size_t)np);
  std::vector<int4> items;
  items.reserve((size_t)(np + nc));
  size_t cj = 0;
  auto ready = [&](size_t k) {
    const int h = chi[(size_t)corder[k]];
    return h < 0 || (h < (int)np && ppos[(size_t)h] >= 0 &&
                     (int64_t)items.size() >= ppos[(size_t)h] + lag);
  };
  std::fill(ppos.begin(), ppos.end(), -1);
  for (int64_t i = 0; i < np; ++i) {
    while (cj < (size_t)nc && chi[(size_t)corder[cj]] < i && ready(cj))
      items.push_back(citem[(size_t)corder[cj++]]);
    ppos[(size_t)i] = (int64_t)items.size();
    items.push_back(make_int4(pitem[(size_t)i].x, pitem[(size_t)i].y, (int)i, -1));
  }
  while (cj < (size_t)nc) items.push_back(citem[(size_t)corder[cj++]]);
  plan.items.upload(items.data(), items.size(), s);
  plan.n_items = (int)items.size();
  plan.n_prod = np;
  plan.sync.alloc((size_t)(kFlagBase + ((np + (1 << kBlockShift) - 1) >> kBlockShift)));
  plan.grid = (unsigned)(sms * occ);  // every CTA resident: static item assignment
  plan.kernel = (void*)kern;
  SFEEC_CUDA(cudaStreamSynchronize(s));
  plan.ok = true;
  return true;
}

void launch_wave(const WavePlan& plan, const DevOperator& p, const DevOperator& c,
                 const double* x, double* t, double* y, double alpha, cudaStream_t s) {
  SFEEC_CUDA(cudaMemsetAsync(plan.sync.p, 0, sizeof(int) * plan.sync.n, s));
  WaveArgs a{};
  a.items = plan.items.p;
  a.n_items = plan.n_items;
  a.n_prod = (int)plan.n_prod;
  a.batch = plan.batch;
  a.sync = plan.sync.p;
  a.srow = p.slice_row.p;
  a.sptr = p.slice_ptr.p;
  a.sw = p.slice_w.p;
  a.pcol = p.sell_col.p;
  a.pval = p.sell_val.p;
  a.prows = p.rows;
  a.x = x;
  a.t = t;
  a.ccol = c.sell_col.p;
  a.cval = c.layout == DevOperator::kSigned ? nullptr : c.sell_val.p;
  a.crows = c.rows;
  a.cscale = c.layout == DevOperator::kSigned ? c.scale : 1.0;
  a.y = y;
  a.alpha = alpha;
  reinterpret_cast<WaveKernel>(plan.kernel)<<<plan.grid, kWThreads, 0, s>>>(a);
  SFEEC_LAUNCH_CHECK();
}

}  // namespace sfeec_b200
