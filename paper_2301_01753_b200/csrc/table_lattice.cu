// Table-driven Kuhn-lattice step (table_lattice.cuh).
//
// Kernels: one thread per (vertex, row type). A block is kTL consecutive
// positions of one vertex plane for ONE row type, and the row type is the
// fastest block index, so the blocks in flight at any time work on the same
// few hundred vertices: the gathered x values and the mirrored coefficient
// lines they share stay in L1 / L2. Every thread walks its row type's slot
// table (uniform across the block) in the CSR column order of an interior
// row, eight slots per trip: the eight coefficient loads and the eight x
// loads are issued before the first FMA, and the FMAs chain in slot order, so
// a row sums exactly like a CSR row of the k-major numbering does away from
// the 32-vertex x-block edges.
#include <algorithm>
#include <cstdio>
#include <map>
#include <tuple>

#include "table_lattice.cuh"

namespace sfeec_b200 {

namespace {

constexpr int kTL = 128;   // threads per block
constexpr int kUnroll = 8;  // slots per trip

// ---- apply kernels ----------------------------------------------------------
// block -> (row type, chunk of the plane's rows 0..n, plane); false off the mesh
__device__ __forceinline__ bool tl_vertex(const TLGeom& g, int ntypes, int chunks, int& r,
                                          int64_t& idx) {
  int64_t b = blockIdx.x;
  r = (int)(b % ntypes);
  b /= ntypes;
  const int chunk = (int)(b % chunks);
  const int k = (int)(b / chunks);
  const int p = chunk * kTL + threadIdx.x;  // over the padded rows j = 0..n of the plane
  if (p >= (g.n + 1) * g.S) return false;
  const int i = p % g.S - g.H;
  idx = g.PS * (k + g.H) + (int64_t)g.S * g.H + p;
  return i >= 0 && i <= g.n;
}

__global__ void __launch_bounds__(kTL)
    k_tl_sym(TLGeom g, int ntypes, int chunks, const int* __restrict__ beg,
             const TLSlot* __restrict__ slots, const double* __restrict__ coef,
             const double* __restrict__ x, double* __restrict__ y,
             const uint64_t* __restrict__ mask) {
  int r;
  int64_t idx;
  if (!tl_vertex(g, ntypes, chunks, r, idx)) return;
  if (!((mask[idx] >> r) & 1)) return;
  const double* cb = coef + idx;
  const double* xb = x + idx;
  int s = beg[r];
  const int s1 = beg[r + 1];
  double acc = 0.0;
  for (; s + kUnroll <= s1; s += kUnroll) {
    double c[kUnroll], v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const longlong2 sl = __ldg(reinterpret_cast<const longlong2*>(slots + s + u));
      c[u] = __ldg(cb + sl.x);
      v[u] = __ldg(xb + sl.y);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc = fma(c[u], v[u], acc);
  }
  for (; s < s1; ++s) {
    const longlong2 sl = __ldg(reinterpret_cast<const longlong2*>(slots + s));
    acc = fma(__ldg(cb + sl.x), __ldg(xb + sl.y), acc);
  }
  y[(int64_t)r * g.NP + idx] = acc;
}

// y_r += alpha * sum_s val_s x(s)
__global__ void __launch_bounds__(kTL)
    k_tl_inc(TLGeom g, int ntypes, int chunks, const int* __restrict__ beg,
             const TLCSlot* __restrict__ slots, double alpha, const double* __restrict__ x,
             double* __restrict__ y, const uint64_t* __restrict__ mask) {
  int r;
  int64_t idx;
  if (!tl_vertex(g, ntypes, chunks, r, idx)) return;
  if (!((mask[idx] >> r) & 1)) return;
  const double* xb = x + idx;
  const int s0 = beg[r], s1 = beg[r + 1];
  double* yp = y + (int64_t)r * g.NP + idx;
  const double y0 = *yp;
  double acc = 0.0;
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
                          const double* __restrict__ kval, double* __restrict__ coef,
                          int* __restrict__ bad) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t p = rpos[r];
  const int t = (int)(p / NP);
  const int64_t idx = p - (int64_t)t * NP;
  const int k0 = kbeg[t], k1 = kbeg[t + 1];
  for (int64_t q = rp[r] + lane; q < rp[r + 1]; q += 32) {
    const int64_t pc = cpos[ci[q]];
    const int t2 = (int)(pc / NP);
    const int64_t key = tl_key(t2, (pc - (int64_t)t2 * NP) - idx);
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
      coef[(int64_t)karr[lo] * NP + idx] = val[q];
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
          const KeyTable& kt, bool constant, double* coef, const char* name, cudaStream_t s) {
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
                                                     constant ? kval.p : nullptr, coef, bad.p);
  SFEEC_LAUNCH_CHECK();
  int hbad = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  require(hbad != 1, std::string("table lattice: an entry of ") + name +
                         " lies outside the interior stencil");
  require(hbad != 2, std::string("table lattice: an entry of ") + name +
                         " differs from its stencil constant");
}

void build_sym(const Builder& b, const DevCSR& a, const TLDofs& d, const int64_t* pos,
               const char* name, TLSym& out, cudaStream_t s) {
  auto st = b.stencils(a, d, d, s);
  // canonical slots get the arrays, in (row type, slot) order
  std::map<std::tuple<int, int, int64_t>, int> canon;  // (row type, column type, offset)
  int narr = 0;
  for (int t = 0; t < d.ntypes; ++t)
    for (HostSlot& sl : st[(size_t)t]) {
      sl.mirror = !(sl.off > 0 || (sl.off == 0 && sl.ctype >= t));
      if (!sl.mirror) {
        sl.array = narr++;
        canon[{t, sl.ctype, sl.off}] = sl.array;
      }
    }
  for (int t = 0; t < d.ntypes; ++t)
    for (HostSlot& sl : st[(size_t)t])
      if (sl.mirror) {
        auto it = canon.find({sl.ctype, t, -sl.off});
        require(it != canon.end(),
                std::string("table lattice: the stencil of ") + name + " is not symmetric");
        sl.array = it->second;
      }
  out.ntypes = d.ntypes;
  out.narrays = narr;
  std::vector<int> beg{0};
  std::vector<TLSlot> slots;
  for (int t = 0; t < d.ntypes; ++t) {
    for (const HostSlot& sl : st[(size_t)t])
      slots.push_back({(int64_t)sl.array * b.g.NP + (sl.mirror ? sl.off : 0),
                       (int64_t)sl.ctype * b.g.NP + sl.off});
    beg.push_back((int)slots.size());
  }
  out.nslots = (int64_t)slots.size();
  out.beg.upload(beg.data(), beg.size(), s);
  out.slots.upload(slots.data(), slots.size(), s);
  out.coef.alloc((size_t)narr * (size_t)b.g.NP);
  out.coef.zero(s);
  fill(a, pos, pos, b.g.NP, key_table(st), false, out.coef.p, name, s);
}

void build_inc(const Builder& b, const DevCSR& a, const TLDofs& rows, const TLDofs& cols,
               const int64_t* rpos, const int64_t* cpos, const char* name, TLInc& out,
               cudaStream_t s) {
  auto st = b.stencils(a, rows, cols, s);
  out.ntypes = rows.ntypes;
  std::vector<int> beg{0};
  std::vector<TLCSlot> slots;
  for (int t = 0; t < rows.ntypes; ++t) {
    for (const HostSlot& sl : st[(size_t)t])
      slots.push_back({sl.val, (int64_t)sl.ctype * b.g.NP + sl.off});
    beg.push_back((int)slots.size());
  }
  out.nslots = (int64_t)slots.size();
  out.beg.upload(beg.data(), beg.size(), s);
  out.slots.upload(slots.data(), slots.size(), s);
  fill(a, rpos, cpos, b.g.NP, key_table(st), true, nullptr, name, s);
}

}  // namespace

void TableLattice::build(int n, int halo, const TLDofs& d1, const TLDofs& d2, const DevCSR& qsym,
                         const DevCSR& m2csr, const DevCSR& ccsr, const DevCSR& ctcsr,
                         cudaStream_t s) {
  require(halo >= 1 && n >= 2 * halo + 2,
          "table lattice: the mesh is too small for an interior reference vertex");
  require(d1.ntypes <= 64 && d2.ntypes <= 64, "table lattice: at most 64 DOF types per vertex");
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
  build_sym(b, qsym, d1, epos.p, "Q_sym", q, s);
  build_sym(b, m2csr, d2, fpos.p, "M2", m2, s);
  build_inc(b, ccsr, d2, d1, fpos.p, epos.p, "C", c, s);
  build_inc(b, ctcsr, d1, d2, epos.p, fpos.p, "C^T", ct, s);
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
  if (n1) k_tl_scatter<<<blocks256(n1), 256, 0, s>>>(n1, epos.p, e, E.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::gather(double* b, double* e, cudaStream_t s) const {
  if (n2) k_tl_gather<<<blocks256(n2), 256, 0, s>>>(n2, fpos.p, B.p, b);
  if (n1) k_tl_gather<<<blocks256(n1), 256, 0, s>>>(n1, epos.p, E.p, e);
  SFEEC_LAUNCH_CHECK();
}

namespace {
int tl_chunks(const TLGeom& g) { return ((g.n + 1) * g.S + kTL - 1) / kTL; }
unsigned tl_grid(const TLGeom& g, int ntypes) {
  return (unsigned)((int64_t)ntypes * tl_chunks(g) * (g.n + 1));
}
}  // namespace

void TableLattice::apply_q(cudaStream_t s) const {
  k_tl_sym<<<tl_grid(g, nt1), kTL, 0, s>>>(g, nt1, tl_chunks(g), q.beg.p, q.slots.p, q.coef.p,
                                           E.p, T.p, mask1.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_m2(cudaStream_t s) const {
  k_tl_sym<<<tl_grid(g, nt2), kTL, 0, s>>>(g, nt2, tl_chunks(g), m2.beg.p, m2.slots.p, m2.coef.p,
                                           B.p, U.p, mask2.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_cb(double h, cudaStream_t s) const {
  k_tl_inc<<<tl_grid(g, nt2), kTL, 0, s>>>(g, nt2, tl_chunks(g), c.beg.p, c.slots.p, -h, T.p, B.p,
                                           mask2.p);
  SFEEC_LAUNCH_CHECK();
}
void TableLattice::apply_cte(double f, cudaStream_t s) const {
  k_tl_inc<<<tl_grid(g, nt1), kTL, 0, s>>>(g, nt1, tl_chunks(g), ct.beg.p, ct.slots.p, f, U.p,
                                           E.p, mask1.p);
  SFEEC_LAUNCH_CHECK();
}

// bytes per launch: coefficient arrays and the gathered field read once over
// the V = (n + 1)^3 vertices, outputs written (and, for the incidence
// kernels, read) once per DOF
double TableLattice::bytes_q() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (g.n + 1);
  return 8.0 * (q.narrays * V + (double)n1 + (double)n1);
}
double TableLattice::bytes_m2() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (g.n + 1);
  return 8.0 * (m2.narrays * V + (double)n2 + (double)n2);
}
double TableLattice::bytes_cb() const { return 8.0 * ((double)n1 + 2.0 * (double)n2); }
double TableLattice::bytes_cte() const { return 8.0 * ((double)n2 + 2.0 * (double)n1); }

}  // namespace sfeec_b200
