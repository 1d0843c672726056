// Table-driven Kuhn-lattice step (table_lattice.cuh).
//
// Kernels: one thread per (vertex, row type). A block is kTL consecutive
// positions of one vertex plane for ONE row type, and the row type is the
// fastest block index, so the blocks in flight at any time work on the same
// few hundred vertices and share the gathered x values in L2. The block
// stages its row type's slot table in shared memory; every thread then walks
// it in the CSR column order of an interior row, several slots per trip: the
// trip's coefficient and x loads are all issued before its first FMA, and the
// FMAs chain in slot order, so a row sums like a CSR row of the k-major
// numbering does away from the 32-vertex x-block edges. (__launch_bounds__
// with a minimum block count matters: without it ptxas schedules for 32
// registers and runs one slot's loads at a time.)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>
#include <type_traits>

#include "table_lattice.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kTL = 128;   // threads per block
constexpr int kUnroll = 8;  // slots per trip

// ---- apply kernels ----------------------------------------------------------
// block -> (row type, chunk of the plane's rows 0..n, plane), row type
// fastest; false off the mesh. (Sweeping strips of a few rows through all
// planes, so that the lines a transposed slot reads at dk < 0 might still be
// in L2, was measured slower on config 4: K-Q 3.5-3.6 vs 3.3 ms. With ~900
// blocks in flight, each streaming its own 1.3 MB of coefficients, the window
// between a block's canonical read and the transposed read of the same line
// is far more than the L2 holds whatever the block order.)
struct TLMap {
  int ntypes, chunks;  // chunks per plane
};
// grid = (row types, chunks, planes): x is the fastest block index
__device__ __forceinline__ bool tl_vertex(const TLGeom& g, const TLMap&, int& r, int64_t& idx) {
  r = (int)blockIdx.x;
  const int k = (int)blockIdx.z;
  const int p = (int)blockIdx.y * kTL + (int)threadIdx.x;  // over the padded rows j = 0..n
  if (p >= (g.n + 1) * g.S) return false;
  const int i = p % g.S - g.H;
  idx = g.P0 + g.PS * (k + g.H) + (int64_t)g.S * g.H + p;
  return i >= 0 && i <= g.n;
}

// the block's row type's slot table, staged once in shared memory (read by
// every warp of the block for every trip; no thread leaves before the barrier)
__device__ __forceinline__ void tl_stage_table(const TLSlot* __restrict__ slots, int s0, int s1,
                                               longlong2* tab) {
  for (int s = s0 + threadIdx.x; s < s1; s += kTL)
    tab[s - s0] = __ldg(reinterpret_cast<const longlong2*>(slots + s));
  __syncthreads();
}

__global__ void __launch_bounds__(kTL, 6)
    k_tl_sym(TLGeom g, TLMap map, const int* __restrict__ beg,
             const TLSlot* __restrict__ slots, const double* __restrict__ coef,
             const double* __restrict__ x, double* __restrict__ y,
             const uint64_t* __restrict__ mask) {
  extern __shared__ __align__(16) longlong2 tab[];
  int r;
  int64_t idx;
  const bool on = tl_vertex(g, map, r, idx);
  const int ns = beg[r + 1] - beg[r];
  tl_stage_table(slots, beg[r], beg[r + 1], tab);
  if (!on || !((mask[idx] >> r) & 1)) return;
  const double* cb = coef + idx;
  const double* xb = x + idx;
  int s = 0;
  double acc = 0.0;
  // a trip: N table entries, then N coefficient and N x loads, then the FMAs
  auto trip = [&](auto n_) {
    constexpr int N = decltype(n_)::value;
    longlong2 sl[N];
    double c[N], v[N];
#pragma unroll
    for (int u = 0; u < N; ++u) sl[u] = tab[s + u];
#pragma unroll
    for (int u = 0; u < N; ++u) c[u] = __ldg(cb + sl[u].x);
#pragma unroll
    for (int u = 0; u < N; ++u) v[u] = __ldg(xb + sl[u].y);
#pragma unroll
    for (int u = 0; u < N; ++u) acc = fma(c[u], v[u], acc);
    s += N;
  };
#pragma unroll 1
  while (s + kUnroll <= ns) trip(std::integral_constant<int, kUnroll>{});
  if (s + 4 <= ns) trip(std::integral_constant<int, 4>{});
  if (s + 2 <= ns) trip(std::integral_constant<int, 2>{});
  if (s < ns) trip(std::integral_constant<int, 1>{});
  y[(int64_t)r * g.NP + idx] = acc;
}

// The same for a space with two moments per entity (P2- 1-forms): one thread
// per (vertex, ENTITY type) computes both moment rows. A slot is a 2 x 2
// block: the field is stored as (moment 0, moment 1) pairs per entity and
// position, the coefficients as 4 doubles per canonical block and position,
// so a slot costs one 16-byte x load, one 32-byte coefficient load and one
// table entry for four multiply-adds (the scalar kernel: eight loads and four
// table entries). A transposed slot reads the neighbour's block and applies
// its transpose. Row sums run in slot order, column moments innermost.
constexpr int kUnroll2 = 4;
__global__ void __launch_bounds__(kTL, 6)
    k_tl_sym2(TLGeom g, TLMap map, const int* __restrict__ beg,
              const TLSlot* __restrict__ slots, const double2* __restrict__ coef,
              const double2* __restrict__ x, double2* __restrict__ y,
              const uint64_t* __restrict__ mask) {
  extern __shared__ __align__(16) longlong2 tab[];
  int r;
  int64_t idx;
  const bool on = tl_vertex(g, map, r, idx);
  const int ns = beg[r + 1] - beg[r];
  tl_stage_table(slots, beg[r], beg[r + 1], tab);
  if (!on || !((mask[idx] >> (2 * r)) & 1)) return;
  const double2* cb = coef + 2 * idx;
  const double2* xb = x + idx;
  int s = 0;
  double a0 = 0.0, a1 = 0.0;
  auto term = [&](const double2& c0, const double2& c1, const double2& v, bool mirror) {
    // block = [c0.x c0.y; c1.x c1.y]; mirror: the transpose
    const double m01 = mirror ? c1.x : c0.y, m10 = mirror ? c0.y : c1.x;
    a0 = fma(c0.x, v.x, a0);
    a0 = fma(m01, v.y, a0);
    a1 = fma(m10, v.x, a1);
    a1 = fma(c1.y, v.y, a1);
  };
  auto trip = [&](auto n_) {
    constexpr int N = decltype(n_)::value;
    longlong2 sl[N];
    double2 c0[N], c1[N], v[N];
#pragma unroll
    for (int u = 0; u < N; ++u) sl[u] = tab[s + u];
#pragma unroll
    for (int u = 0; u < N; ++u) {
      c0[u] = __ldg(cb + 2 * sl[u].x);
      c1[u] = __ldg(cb + 2 * sl[u].x + 1);
    }
#pragma unroll
    for (int u = 0; u < N; ++u) v[u] = __ldg(xb + (sl[u].y >> 1));
#pragma unroll
    for (int u = 0; u < N; ++u) term(c0[u], c1[u], v[u], (sl[u].y & 1) != 0);
    s += N;
  };
#pragma unroll 1
  while (s + kUnroll2 <= ns) trip(std::integral_constant<int, kUnroll2>{});
  if (s + 2 <= ns) trip(std::integral_constant<int, 2>{});
  if (s < ns) trip(std::integral_constant<int, 1>{});
  y[(int64_t)r * g.NP + idx] = make_double2(a0, a1);
}

// Moment blocks with plain (type-major) fields: one thread per (vertex,
// entity type) computes the MB moment rows of its entity; a slot is an MB x MB
// block whose MB * MB values are MB * MB consecutive coefficient ARRAYS (so
// every load stays a coalesced run over the positions) and whose MB x values
// serve all MB rows. Used for the P2- 2-forms (MB = 3: three moments per face
// and per tet): 9 coefficient loads, 3 x loads and one table entry per nine
// multiply-adds, where scalar slots need 18 loads and 9 entries.
template <int MB>
__global__ void __launch_bounds__(kTL, 6)
    k_tl_symb(TLGeom g, TLMap map, const int* __restrict__ beg,
              const TLSlot* __restrict__ slots, const double* __restrict__ coef,
              const double* __restrict__ x, double* __restrict__ y,
              const uint64_t* __restrict__ mask) {
  extern __shared__ __align__(16) longlong2 tab[];
  int r;
  int64_t idx;
  const bool on = tl_vertex(g, map, r, idx);
  const int ns = beg[r + 1] - beg[r];
  tl_stage_table(slots, beg[r], beg[r + 1], tab);
  if (!on || !((mask[idx] >> (MB * r)) & 1)) return;
  const double* cb = coef + idx;
  const double* xb = x + idx;
  double acc[MB];
#pragma unroll
  for (int m = 0; m < MB; ++m) acc[m] = 0.0;
  int s = 0;
  auto trip = [&](auto n_) {
    constexpr int N = decltype(n_)::value;
    longlong2 sl[N];
    double c[N][MB * MB], v[N][MB];
#pragma unroll
    for (int u = 0; u < N; ++u) sl[u] = tab[s + u];
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
      for (int e = 0; e < MB * MB; ++e) c[u][e] = __ldg(cb + sl[u].x + (int64_t)e * g.NP);
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
      for (int m = 0; m < MB; ++m) v[u][m] = __ldg(xb + (sl[u].y >> 1) + (int64_t)m * g.NP);
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const bool mirror = (sl[u].y & 1) != 0;  // the neighbour's block, transposed
#pragma unroll
      for (int mr = 0; mr < MB; ++mr)
#pragma unroll
        for (int mc = 0; mc < MB; ++mc)
          acc[mr] = fma(mirror ? c[u][mc * MB + mr] : c[u][mr * MB + mc], v[u][mc], acc[mr]);
    }
    s += N;
  };
#pragma unroll 1
  while (s + 2 <= ns) trip(std::integral_constant<int, 2>{});
  if (s < ns) trip(std::integral_constant<int, 1>{});
#pragma unroll
  for (int m = 0; m < MB; ++m) y[(int64_t)(MB * r + m) * g.NP + idx] = acc[m];
}

// y_r += alpha * sum_s val_s x(s); mbx / mby = moments per entity of the x / y
// space (element (type t, position p) of a field with mb moments per entity
// lives at ((t / mb) NP + p) mb + t % mb; the slots' xoff is in elements)
__global__ void __launch_bounds__(kTL)
    k_tl_inc(TLGeom g, TLMap map, const int* __restrict__ beg,
             const TLCSlot* __restrict__ slots, double alpha, const double* __restrict__ x,
             int mbx, double* __restrict__ y, int mby, const uint64_t* __restrict__ mask) {
  int r;
  int64_t idx;
  if (!tl_vertex(g, map, r, idx)) return;
  if (!((mask[idx] >> r) & 1)) return;
  const double* xb = x + idx * mbx;
  const int s0 = beg[r], s1 = beg[r + 1];
  double* yp = y + ((int64_t)(r / mby) * g.NP + idx) * mby + r % mby;
  const double y0 = *yp;
  double acc = 0.0;
#pragma unroll 4
  for (int s = s0; s < s1; ++s) {
    const TLCSlot sl = slots[s];
    acc = fma(sl.val, __ldg(xb + sl.xoff), acc);
  }
  *yp = fma(alpha, acc, y0);
}

// ---- setup kernels ------------------------------------------------------------
constexpr int kKeyShift = 40;
__host__ __device__ inline int64_t tl_key(int ctype, int64_t off) {
  return ((int64_t)ctype << kKeyShift) | (off + ((int64_t)1 << (kKeyShift - 1)));
}

// One warp per CSR row: each entry finds its slot by (column type, offset) in
// the row type's sorted key list. Symmetric operators (kval == nullptr):
// canonical slots (karr >= 0) store the value at the row's position. Constant
// operators: the value must equal the slot's constant. bad: 1 = an entry
// without a slot, 2 = a constant mismatch.
__global__ void k_tl_fill(int64_t rows, const int64_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ val,
                          const int64_t* __restrict__ rpos, const int64_t* __restrict__ cpos,
                          int64_t NP, const int* __restrict__ kbeg,
                          const int64_t* __restrict__ keys, const int* __restrict__ karr,
                          const double* __restrict__ kval, double* __restrict__ coef, int mb,
                          int soa, int* __restrict__ bad) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  // (mb > 1: the tables are per ENTITY type, type = entity type * mb + moment,
  // and a canonical block stores its mb x mb values row-major per position)
  const int64_t p = rpos[r];
  const int tfull = (int)(p / NP);
  const int64_t idx = p - (int64_t)tfull * NP;
  const int t = tfull / mb, mr = tfull % mb;
  const int k0 = kbeg[t], k1 = kbeg[t + 1];
  for (int64_t q = rp[r] + lane; q < rp[r + 1]; q += 32) {
    const int64_t pc = cpos[ci[q]];
    const int t2full = (int)(pc / NP);
    const int t2 = t2full / mb, mc = t2full % mb;
    const int64_t key = tl_key(t2, (pc - (int64_t)t2full * NP) - idx);
    int lo = k0, hi = k1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= k1 || keys[lo] != key) {
      atomicExch(bad, 1);
      continue;
    }
    if (kval) {
      if (kval[lo] != val[q]) atomicExch(bad, 2);
    } else if (karr[lo] >= 0) {
      // a block's values: interleaved per position, or (soa) mb * mb arrays
      if (soa)
        coef[(((int64_t)karr[lo] * mb + mr) * mb + mc) * NP + idx] = val[q];
      else
        coef[(((int64_t)karr[lo] * NP + idx) * mb + mr) * mb + mc] = val[q];
    }
  }
}

__global__ void k_tl_mask(int64_t n, const int64_t* __restrict__ pos, int64_t NP,
                          unsigned long long* __restrict__ mask) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t p = pos[r];
  const int t = (int)(p / NP);
  atomicOr(mask + (p - (int64_t)t * NP), 1ull << t);
}
__global__ void k_tl_scatter(int64_t n, const int64_t* __restrict__ pos,
                             const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[pos[r]] = src[r];
}
__global__ void k_tl_gather(int64_t n, const int64_t* __restrict__ pos,
                            const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[pos[r]];
}

inline unsigned blocks256(int64_t n) { return (unsigned)((n + 255) / 256); }

// ---- host side: the interior stencils, read off the assembled operators --------
struct HostSlot {
  int ctype = 0;
  int64_t off = 0;   // linear offset in the padded box
  double val = 0;    // the entry of the reference row
  int array = -1;    // symmetric: coefficient array (own or the mirror's)
  bool mirror = false;
};

struct HostRow {
  std::vector<int32_t> ci;
  std::vector<double> val;
};
HostRow fetch_row(const DevCSR& a, int64_t r, cudaStream_t s) {
  int64_t rp[2];
  SFEEC_CUDA(cudaMemcpyAsync(rp, a.rp.p + r, sizeof(rp), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  HostRow out;
  const size_t n = (size_t)(rp[1] - rp[0]);
  out.ci.resize(n);
  out.val.resize(n);
  if (n) {
    SFEEC_CUDA(cudaMemcpyAsync(out.ci.data(), a.ci.p + rp[0], sizeof(int32_t) * n,
                               cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaMemcpyAsync(out.val.data(), a.val.p + rp[0], sizeof(double) * n,
                               cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
  }
  return out;
}

struct Builder {
  const TLGeom& g;
  int64_t vref;  // the reference vertex (id in the (n + 1)^3 numbering)
  int64_t lin(int64_t v) const {  // vertex id -> position in the padded box
    const int m = g.n + 1;
    return g.pos((int)(v % m), (int)((v / m) % m), (int)(v / ((int64_t)m * m)));
  }
  // DOF of each type at the reference vertex
  std::vector<int64_t> ref_rows(const TLDofs& d) const {
    std::vector<int64_t> out((size_t)d.ntypes, -1);
    for (size_t r = 0; r < d.type.size(); ++r)
      if (d.vertex[r] == vref) out[(size_t)d.type[r]] = (int64_t)r;
    for (int64_t r : out)
      require(r >= 0, "table lattice: the reference vertex lacks a DOF type (mesh too small)");
    return out;
  }
  // slot lists per row type, in the reference rows' CSR order
  std::vector<std::vector<HostSlot>> stencils(const DevCSR& a, const TLDofs& rows,
                                              const TLDofs& cols, cudaStream_t s) const {
    const std::vector<int64_t> rr = ref_rows(rows);
    std::vector<std::vector<HostSlot>> out((size_t)rows.ntypes);
    const int64_t p0 = lin(vref);
    for (int t = 0; t < rows.ntypes; ++t) {
      const HostRow row = fetch_row(a, rr[(size_t)t], s);
      for (size_t k = 0; k < row.ci.size(); ++k) {
        HostSlot sl;
        const size_t c = (size_t)row.ci[k];
        sl.ctype = cols.type[c];
        sl.off = lin(cols.vertex[c]) - p0;
        sl.val = row.val[k];
        out[(size_t)t].push_back(sl);
      }
    }
    return out;
  }
};

// sorted (key -> slot) lists per row type for the fill kernel
struct KeyTable {
  std::vector<int> beg;
  std::vector<int64_t> keys;
  std::vector<int> arr;
  std::vector<double> val;
};
KeyTable key_table(const std::vector<std::vector<HostSlot>>& st) {
  KeyTable kt;
  kt.beg.push_back(0);
  for (const auto& row : st) {
    std::vector<std::tuple<int64_t, int, double>> v;
    for (const HostSlot& sl : row)
      v.emplace_back(tl_key(sl.ctype, sl.off), sl.mirror ? -1 : sl.array, sl.val);
    std::sort(v.begin(), v.end());
    for (auto& [k, a, x] : v) {
      kt.keys.push_back(k);
      kt.arr.push_back(a);
      kt.val.push_back(x);
    }
    kt.beg.push_back((int)kt.keys.size());
  }
  return kt;
}

void fill(const DevCSR& a, const int64_t* rpos, const int64_t* cpos, int64_t NP,
          const KeyTable& kt, bool constant, double* coef, int mb, bool soa, const char* name,
          cudaStream_t s) {
  DevBuf<int> kbeg, karr, bad;
  DevBuf<int64_t> keys;
  DevBuf<double> kval;
  kbeg.upload(kt.beg.data(), kt.beg.size(), s);
  keys.upload(kt.keys.data(), kt.keys.size(), s);
  karr.upload(kt.arr.data(), kt.arr.size(), s);
  if (constant) kval.upload(kt.val.data(), kt.val.size(), s);
  bad.alloc(1);
  bad.zero(s);
  if (a.rows)
    k_tl_fill<<<blocks256(a.rows * 32), 256, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.val.p, rpos, cpos,
                                                     NP, kbeg.p, keys.p, karr.p,
                                                     constant ? kval.p : nullptr, coef, mb,
                                                     soa ? 1 : 0, bad.p);
  SFEEC_LAUNCH_CHECK();
  int hbad = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  require(hbad != 1, std::string("table lattice: an entry of ") + name +
                         " lies outside the interior stencil");
  require(hbad != 2, std::string("table lattice: an entry of ") + name +
                         " differs from its stencil constant");
}

// entity-level stencils of a space with mb moments per entity (type = entity
// type * mb + moment): the (column entity type, offset) blocks of each row
// entity type in order of first appearance in its moment-0 row. Every block
// must be full (mb x mb) and every moment row must show the same blocks.
std::vector<std::vector<HostSlot>> entity_stencils(
    const std::vector<std::vector<HostSlot>>& full, int mb, const char* name) {
  if (mb == 1) return full;
  const int ne = (int)full.size() / mb;
  std::vector<std::vector<HostSlot>> out((size_t)ne);
  for (int R = 0; R < ne; ++R) {
    auto blocks = [&](int m) {
      std::vector<std::pair<int, int64_t>> v;
      for (const HostSlot& sl : full[(size_t)(R * mb + m)]) {
        const std::pair<int, int64_t> key{sl.ctype / mb, sl.off};
        if (std::find(v.begin(), v.end(), key) == v.end()) v.push_back(key);
      }
      return v;
    };
    const auto b0 = blocks(0);
    for (int m = 0; m < mb; ++m)
      require(full[(size_t)(R * mb + m)].size() == (size_t)mb * b0.size() && blocks(m) == b0,
              std::string("table lattice: the stencil of ") + name +
                  " is not made of full moment blocks");
    for (const auto& [C, off] : b0) {
      HostSlot sl;
      sl.ctype = C;
      sl.off = off;
      out[(size_t)R].push_back(sl);
    }
  }
  return out;
}

// soa: an mb x mb block is mb * mb arrays and the field stays type-major
// (k_tl_symb); otherwise the block and the field are interleaved per position
// (k_tl_sym2, mb = 2)
void build_sym(const Builder& b, const DevCSR& a, const TLDofs& d, int mb, bool soa,
               const int64_t* pos, const char* name, TLSym& out, cudaStream_t s) {
  auto st = entity_stencils(b.stencils(a, d, d, s), mb, name);
  const int ne = d.ntypes / mb;
  // canonical slots get the arrays, in (row type, slot) order
  std::map<std::tuple<int, int, int64_t>, int> canon;  // (row type, column type, offset)
  int narr = 0;
  for (int t = 0; t < ne; ++t)
    for (HostSlot& sl : st[(size_t)t]) {
      sl.mirror = !(sl.off > 0 || (sl.off == 0 && sl.ctype >= t));
      if (!sl.mirror) {
        sl.array = narr++;
        canon[{t, sl.ctype, sl.off}] = sl.array;
      }
    }
  for (int t = 0; t < ne; ++t)
    for (HostSlot& sl : st[(size_t)t])
      if (sl.mirror) {
        auto it = canon.find({sl.ctype, t, -sl.off});
        require(it != canon.end(),
                std::string("table lattice: the stencil of ") + name + " is not symmetric");
        sl.array = it->second;
      }
  out.ntypes = ne;
  out.mb = mb;
  out.soa = soa;
  out.narrays = narr;
  std::vector<int> beg{0};
  std::vector<TLSlot> slots;
  for (int t = 0; t < ne; ++t) {
    for (const HostSlot& sl : st[(size_t)t]) {
      // (blocked kernels: bit 0 of the second word flags a transposed slot)
      const int64_t xoff = (int64_t)sl.ctype * (soa ? mb : 1) * b.g.NP + sl.off;
      slots.push_back({(int64_t)sl.array * (soa ? mb * mb : 1) * b.g.NP + (sl.mirror ? sl.off : 0),
                       mb == 1 ? xoff : (xoff << 1) | (sl.mirror ? 1 : 0)});
    }
    beg.push_back((int)slots.size());
    out.max_slots = std::max(out.max_slots, beg[beg.size() - 1] - beg[beg.size() - 2]);
  }
  require(out.max_slots * sizeof(TLSlot) <= 48 * 1024,
          std::string("table lattice: the stencil of ") + name + " exceeds the table staging");
  out.nslots = (int64_t)slots.size();
  out.beg.upload(beg.data(), beg.size(), s);
  out.slots.upload(slots.data(), slots.size(), s);
  out.coef.alloc((size_t)narr * (size_t)b.g.NP * (size_t)(mb * mb));
  out.coef.zero(s);
  fill(a, pos, pos, b.g.NP, key_table(st), false, out.coef.p, mb, soa, name, s);
}

// mbx: moments per entity of the column (x) space; xoff in elements
void build_inc(const Builder& b, const DevCSR& a, const TLDofs& rows, const TLDofs& cols,
               int mbx, const int64_t* rpos, const int64_t* cpos, const char* name, TLInc& out,
               cudaStream_t s) {
  auto st = b.stencils(a, rows, cols, s);
  out.ntypes = rows.ntypes;
  std::vector<int> beg{0};
  std::vector<TLCSlot> slots;
  for (int t = 0; t < rows.ntypes; ++t) {
    for (const HostSlot& sl : st[(size_t)t])
      slots.push_back({sl.val, ((int64_t)(sl.ctype / mbx) * b.g.NP + sl.off) * mbx +
                                   sl.ctype % mbx});
    beg.push_back((int)slots.size());
  }
  out.nslots = (int64_t)slots.size();
  out.beg.upload(beg.data(), beg.size(), s);
  out.slots.upload(slots.data(), slots.size(), s);
  fill(a, rpos, cpos, b.g.NP, key_table(st), true, nullptr, 1, false, name, s);
}

}  // namespace

void TableLattice::build(int n, int halo, const TLDofs& d1, const TLDofs& d2, const DevCSR& qsym,
                         const DevCSR& m2csr, const DevCSR& ccsr, const DevCSR& ctcsr,
                         cudaStream_t s) {
  require(halo >= 1 && n >= 2 * halo + 2,
          "table lattice: the mesh is too small for an interior reference vertex");
  require(d1.ntypes <= 64 && d2.ntypes <= 64, "table lattice: at most 64 DOF types per vertex");
  require((d1.mb == 1 || d1.mb == 2) && d1.ntypes % d1.mb == 0 &&
              (d2.mb == 1 || d2.mb == 3) && d2.ntypes % d2.mb == 0,
          "table lattice: moment blocks of 1 or 2 (1-forms), 1 or 3 (2-forms)");
  mb1 = d1.mb;
  g.init(n, halo);
  n1 = (int64_t)d1.type.size();
  n2 = (int64_t)d2.type.size();
  nt1 = d1.ntypes;
  nt2 = d2.ntypes;
  require(qsym.rows == n1 && m2csr.rows == n2 && ccsr.rows == n2 && ccsr.cols == n1 &&
              ctcsr.rows == n1 && ctcsr.cols == n2,
          "table lattice: operator dimensions do not match the DOF maps");
  const int c0 = n / 2;
  const int m = n + 1;
  Builder b{g, (int64_t)c0 + (int64_t)m * (c0 + (int64_t)m * c0)};
  {
    std::vector<int64_t> ep((size_t)n1), fp((size_t)n2);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n1; ++r)
      ep[(size_t)r] = (int64_t)d1.type[(size_t)r] * g.NP + b.lin(d1.vertex[(size_t)r]);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n2; ++r)
      fp[(size_t)r] = (int64_t)d2.type[(size_t)r] * g.NP + b.lin(d2.vertex[(size_t)r]);
    epos.upload(ep.data(), ep.size(), s);
    fpos.upload(fp.data(), fp.size(), s);
    if (mb1 > 1) {  // element addresses of the interleaved 1-form fields
      std::vector<int64_t> ea((size_t)n1);
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < n1; ++r) {
        const int t = d1.type[(size_t)r];
        ea[(size_t)r] = ((int64_t)(t / mb1) * g.NP + b.lin(d1.vertex[(size_t)r])) * mb1 + t % mb1;
      }
      eaddr.upload(ea.data(), ea.size(), s);
      SFEEC_CUDA(cudaStreamSynchronize(s));
    }
    SFEEC_CUDA(cudaStreamSynchronize(s));  // the host vectors die here
  }
  mask1.alloc((size_t)g.NP);
  mask2.alloc((size_t)g.NP);
  mask1.zero(s);
  mask2.zero(s);
  static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "mask word");
  if (n1)
    k_tl_mask<<<blocks256(n1), 256, 0, s>>>(n1, epos.p, g.NP,
                                            reinterpret_cast<unsigned long long*>(mask1.p));
  if (n2)
    k_tl_mask<<<blocks256(n2), 256, 0, s>>>(n2, fpos.p, g.NP,
                                            reinterpret_cast<unsigned long long*>(mask2.p));
  SFEEC_LAUNCH_CHECK();
  build_sym(b, qsym, d1, mb1, false, epos.p, "Q_sym", q, s);
  build_sym(b, m2csr, d2, d2.mb, true, fpos.p, "M2", m2, s);
  build_inc(b, ccsr, d2, d1, mb1, fpos.p, epos.p, "C", c, s);
  build_inc(b, ctcsr, d1, d2, 1, epos.p, fpos.p, "C^T", ct, s);
  for (auto* f : {&E, &T}) {
    f->alloc((size_t)nt1 * (size_t)g.NP);
    f->zero(s);
  }
  for (auto* f : {&B, &U}) {
    f->alloc((size_t)nt2 * (size_t)g.NP);
    f->zero(s);
  }
  SFEEC_CUDA(cudaStreamSynchronize(s));
  valid = newer = false;
}

void TableLattice::scatter(const double* b, const double* e, cudaStream_t s) {
  if (n2) k_tl_scatter<<<blocks256(n2), 256, 0, s>>>(n2, fpos.p, b, B.p);
  if (n1) k_tl_scatter<<<blocks256(n1), 256, 0, s>>>(n1, mb1 > 1 ? eaddr.p : epos.p, e, E.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::gather(double* b, double* e, cudaStream_t s) const {
  if (n2) k_tl_gather<<<blocks256(n2), 256, 0, s>>>(n2, fpos.p, B.p, b);
  if (n1) k_tl_gather<<<blocks256(n1), 256, 0, s>>>(n1, mb1 > 1 ? eaddr.p : epos.p, E.p, e);
  SFEEC_LAUNCH_CHECK();
}

namespace {
TLMap tl_map(const TLGeom& g, int ntypes) {
  return TLMap{ntypes, ((g.n + 1) * g.S + kTL - 1) / kTL};
}
dim3 tl_grid(const TLGeom& g, const TLMap& m) {
  return dim3((unsigned)m.ntypes, (unsigned)m.chunks, (unsigned)(g.n + 1));
}
}  // namespace

void TableLattice::apply_q(cudaStream_t s) const {
  const TLMap m = tl_map(g, q.ntypes);
  const size_t smem = sizeof(TLSlot) * (size_t)q.max_slots;
  if (q.mb == 2)
    k_tl_sym2<<<tl_grid(g, m), kTL, smem, s>>>(
        g, m, q.beg.p, q.slots.p, reinterpret_cast<const double2*>(q.coef.p),
        reinterpret_cast<const double2*>(E.p), reinterpret_cast<double2*>(T.p), mask1.p);
  else
    k_tl_sym<<<tl_grid(g, m), kTL, smem, s>>>(g, m, q.beg.p, q.slots.p, q.coef.p, E.p, T.p,
                                              mask1.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_m2(cudaStream_t s) const {
  const TLMap m = tl_map(g, m2.ntypes);
  const size_t smem = sizeof(TLSlot) * (size_t)m2.max_slots;
  if (m2.mb == 3)
    k_tl_symb<3><<<tl_grid(g, m), kTL, smem, s>>>(g, m, m2.beg.p, m2.slots.p, m2.coef.p, B.p, U.p,
                                                  mask2.p);
  else
    k_tl_sym<<<tl_grid(g, m), kTL, smem, s>>>(g, m, m2.beg.p, m2.slots.p, m2.coef.p, B.p, U.p,
                                              mask2.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_cb(double h, cudaStream_t s) const {
  const TLMap m = tl_map(g, nt2);
  k_tl_inc<<<tl_grid(g, m), kTL, 0, s>>>(g, m, c.beg.p, c.slots.p, -h, T.p, mb1, B.p, 1, mask2.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_cte(double f, cudaStream_t s) const {
  const TLMap m = tl_map(g, nt1);
  k_tl_inc<<<tl_grid(g, m), kTL, 0, s>>>(g, m, ct.beg.p, ct.slots.p, f, U.p, 1, E.p, mb1, mask1.p);
  SFEEC_LAUNCH_CHECK();
}

// bytes per launch: coefficient arrays and the gathered field read once over
// the V = (n + 1)^3 vertices, outputs written (and, for the incidence
// kernels, read) once per DOF
double TableLattice::bytes_q() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (g.n + 1);
  return 8.0 * ((double)q.narrays * q.mb * q.mb * V + (double)n1 + (double)n1);
}
double TableLattice::bytes_m2() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (g.n + 1);
  return 8.0 * ((double)m2.narrays * m2.mb * m2.mb * V + (double)n2 + (double)n2);
}
double TableLattice::bytes_cb() const { return 8.0 * ((double)n1 + 2.0 * (double)n2); }
double TableLattice::bytes_cte() const { return 8.0 * ((double)n2 + 2.0 * (double)n1); }

}  // namespace sfeec_b200
