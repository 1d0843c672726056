// Stencil operator layout for the Kuhn tet mesh (see stencil.cuh).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "stencil.cuh"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

HostCSR tet_curl(const TetMesh& m);
HostCSR tet_mass(const TetMesh& m, int form);

namespace {

constexpr int kMaxQ = 24, kMaxM2 = 8, kMaxC = 4, kMaxCT = 8;
constexpr int kThreads = 256;

// slot = (di, dj, dk, entity type, sign)
struct Tables {
  int8_t q[7][kMaxQ][5];
  int nq[7];
  int8_t m2[12][kMaxM2][5];
  int nm2[12];
  int8_t c[12][kMaxC][5];
  int nc[12];
  int8_t ct[7][kMaxCT][5];
  int nct[7];
};
__constant__ Tables cT;
Tables hT;
std::once_flag tables_once;

int width_of(int kind, int type) {
  switch (kind) {
    case kStQ: return hT.nq[type];
    case kStM2: return hT.nm2[type];
    case kStC: return hT.nc[type];
    default: return hT.nct[type];
  }
}

__device__ __forceinline__ const int8_t* slot(int kind, int type, int s) {
  switch (kind) {
    case kStQ: return cT.q[type][s];
    case kStM2: return cT.m2[type][s];
    case kStC: return cT.c[type][s];
    default: return cT.ct[type][s];
  }
}
__device__ __forceinline__ int width(int kind, int type) {
  switch (kind) {
    case kStQ: return cT.nq[type];
    case kStM2: return cT.nm2[type];
    case kStC: return cT.nc[type];
    default: return cT.nct[type];
  }
}

struct Dev {
  int n;
  int64_t nv;
  const int32_t* tab;    // column-entity table, [types][nv]
  const int32_t* row_v;  // base vertex of each row entity
};

// column id of slot s of a row at vertex (i, j, k); -1 if absent
__device__ __forceinline__ int32_t col_of(const Dev& d, const int8_t* sl, int64_t v, int i, int j,
                                          int k) {
  const int ii = i + sl[0], jj = j + sl[1], kk = k + sl[2];
  if (ii < 0 || ii > d.n || jj < 0 || jj > d.n || kk < 0 || kk > d.n) return -1;
  const int64_t N = d.n + 1;
  const int64_t vn = v + sl[0] + N * (sl[1] + N * (int64_t)sl[2]);
  return __ldg(d.tab + (int64_t)sl[3] * d.nv + vn);
}

template <bool ACC, int KIND, int CH>
__global__ void __launch_bounds__(kThreads, 4)
    k_st(Dev d, int64_t n_slices, const int64_t* __restrict__ srow, const int64_t* __restrict__ sptr,
         const int8_t* __restrict__ stype, const double* __restrict__ val,
         const double* __restrict__ x, double* __restrict__ y, double alpha) {
  constexpr bool VALUED = KIND == kStQ || KIND == kStM2;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  int64_t r0 = __ldg(srow + s), nr = __ldg(srow + s + 1) - r0, ptr = __ldg(sptr + s);
  int type = __ldg(stype + s);
  int32_t vv = lane < nr ? __ldg(d.row_v + r0 + lane) : 0;
  while (true) {
    const int64_t sn = s + nwarps;
    int64_t r0n = 0, nrn = 0, ptrn = 0;
    int typen = 0;
    int32_t vvn = 0;
    if (sn < n_slices) {  // prefetch the next slice's metadata and row vertices
      r0n = __ldg(srow + sn);
      nrn = __ldg(srow + sn + 1) - r0n;
      ptrn = __ldg(sptr + sn);
      typen = __ldg(stype + sn);
      vvn = lane < nrn ? __ldg(d.row_v + r0n + lane) : 0;
    }
    if (lane < nr) {
      const int64_t row = r0 + lane;
      const double y0 = ACC ? y[row] : 0.0;
      const int64_t N = d.n + 1;
      const int i = (int)(vv % N), j = (int)((vv / N) % N), k = (int)(vv / (N * N));
      const int w = width(KIND, type);
      double acc = 0.0;
      for (int k0 = 0; k0 < w; k0 += CH) {
        int32_t c[CH];
        double v[CH], xv[CH];
        int8_t sg[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const bool ok = k0 + q < w;
          const int8_t* sl = slot(KIND, type, ok ? k0 + q : 0);
          c[q] = ok ? col_of(d, sl, vv, i, j, k) : -1;
          sg[q] = sl[4];
          if (VALUED) v[q] = ok ? __ldcs(val + ptr + (int64_t)(k0 + q) * nr + lane) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) xv[q] = c[q] >= 0 ? __ldg(x + c[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          if (VALUED)
            acc = fma(v[q], xv[q], acc);
          else
            acc += sg[q] > 0 ? xv[q] : -xv[q];
        }
      }
      y[row] = ACC ? fma(alpha, acc, y0) : acc;
    }
    if (sn >= n_slices) break;
    s = sn;
    r0 = r0n;
    nr = nrn;
    ptr = ptrn;
    type = typen;
    vv = vvn;
  }
}

// fill the values of a valued stencil operator from its CSR, and check that
// the stencil covers every CSR entry (with matching signs for C / C^T)
template <int KIND>
__global__ void k_st_fill(Dev d, int64_t rows, const int8_t* __restrict__ row_type,
                          const int64_t* __restrict__ row_slice, const int64_t* __restrict__ srow,
                          const int64_t* __restrict__ sptr, const int64_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ cv,
                          double* __restrict__ val, int* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int type = row_type[r];
  const int64_t sl = row_slice[r];
  const int64_t nr = srow[sl + 1] - srow[sl], lane = r - srow[sl];
  const int64_t vv = d.row_v[r];
  const int64_t N = d.n + 1;
  const int i = (int)(vv % N), j = (int)((vv / N) % N), k = (int)(vv / (N * N));
  const int w = width(KIND, type);
  int64_t found = 0;
  for (int s = 0; s < w; ++s) {
    const int8_t* slp = slot(KIND, type, s);
    const int32_t c = col_of(d, slp, vv, i, j, k);
    double value = 0.0;
    if (c >= 0) {
      int64_t lo = rp[r], hi = rp[r + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ci[mid] < c)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < rp[r + 1] && ci[lo] == c) {
        value = cv[lo];
        ++found;
        if ((KIND == kStC || KIND == kStCT) && value != (double)slp[4]) atomicExch(bad, 2);
      }
    }
    if (KIND == kStQ || KIND == kStM2) val[sptr[sl] + s * nr + lane] = value;
  }
  if (found != rp[r + 1] - rp[r]) atomicExch(bad, 1);
}

unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// (offset, type) of an entity relative to the reference entity at (3,3,3)
void add_slot(int8_t* out, const int base[3], const int c[3], int type, double sign) {
  for (int d = 0; d < 3; ++d) out[d] = (int8_t)(c[d] - base[d]);
  out[3] = (int8_t)type;
  out[4] = (int8_t)(sign > 0 ? 1 : -1);
}

}  // namespace

void stencil_init_tables() {
  std::call_once(tables_once, [] {
    std::memset(&hT, 0, sizeof(hT));
    TetMesh m;
    m.build(6, 0.1, 1);
    const int base[3] = {3, 3, 3};
    const int64_t v0 = m.vid(3, 3, 3);
    HostCSR m1 = tet_mass(m, 1), mm2 = tet_mass(m, 2), c = tet_curl(m);
    HostCSR ct = csr_transpose(c);
    auto ecoord = [&](int64_t e, int cc[3]) { m.coords(m.edge_v[(size_t)e], cc); };
    auto fcoord = [&](int64_t f, int cc[3]) { m.coords(m.face_v[(size_t)f], cc); };
    for (int t = 0; t < 7; ++t) {
      const int32_t e = m.eid[(size_t)(v0 * 7 + t)];
      require(e >= 0, "stencil: reference edge missing");
      int k = 0;
      for (int64_t p = m1.row_ptr[(size_t)e]; p < m1.row_ptr[(size_t)e + 1]; ++p, ++k) {
        require(k < kMaxQ, "stencil: Q row too wide");
        int cc[3];
        ecoord(m1.col_idx[(size_t)p], cc);
        add_slot(hT.q[t][k], base, cc, m.edge_t[(size_t)m1.col_idx[(size_t)p]], 1.0);
      }
      hT.nq[t] = k;
      k = 0;
      for (int64_t p = ct.row_ptr[(size_t)e]; p < ct.row_ptr[(size_t)e + 1]; ++p, ++k) {
        require(k < kMaxCT, "stencil: C^T row too wide");
        int cc[3];
        fcoord(ct.col_idx[(size_t)p], cc);
        add_slot(hT.ct[t][k], base, cc, m.face_t[(size_t)ct.col_idx[(size_t)p]], ct.val[(size_t)p]);
      }
      hT.nct[t] = k;
    }
    for (int f = 0; f < 12; ++f) {
      const int32_t id = m.fid[(size_t)(v0 * 12 + f)];
      require(id >= 0, "stencil: reference face missing");
      int k = 0;
      for (int64_t p = mm2.row_ptr[(size_t)id]; p < mm2.row_ptr[(size_t)id + 1]; ++p, ++k) {
        require(k < kMaxM2, "stencil: M2 row too wide");
        int cc[3];
        fcoord(mm2.col_idx[(size_t)p], cc);
        add_slot(hT.m2[f][k], base, cc, m.face_t[(size_t)mm2.col_idx[(size_t)p]], 1.0);
      }
      hT.nm2[f] = k;
      k = 0;
      for (int64_t p = c.row_ptr[(size_t)id]; p < c.row_ptr[(size_t)id + 1]; ++p, ++k) {
        require(k < kMaxC, "stencil: C row too wide");
        int cc[3];
        ecoord(c.col_idx[(size_t)p], cc);
        add_slot(hT.c[f][k], base, cc, m.edge_t[(size_t)c.col_idx[(size_t)p]], c.val[(size_t)p]);
      }
      hT.nc[f] = k;
    }
  });
  SFEEC_CUDA(cudaMemcpyToSymbol(cT, &hT, sizeof(hT)));
}

std::shared_ptr<StencilMesh> stencil_mesh(const TetMesh& m, cudaStream_t s) {
  auto sm = std::make_shared<StencilMesh>();
  sm->n = m.n;
  sm->nv = m.nv;
  sm->n_edges = m.n_edges;
  sm->n_faces = m.n_faces;
  std::vector<int32_t> tmp((size_t)(m.nv * 12));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < m.nv; ++v)
    for (int t = 0; t < 7; ++t) tmp[(size_t)(t * m.nv + v)] = m.eid[(size_t)(v * 7 + t)];
  sm->eidT.upload(tmp.data(), (size_t)(7 * m.nv), s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < m.nv; ++v)
    for (int f = 0; f < 12; ++f) tmp[(size_t)(f * m.nv + v)] = m.fid[(size_t)(v * 12 + f)];
  sm->fidT.upload(tmp.data(), (size_t)(12 * m.nv), s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> ev(m.edge_v.begin(), m.edge_v.end()), fv(m.face_v.begin(), m.face_v.end());
  sm->edge_v.upload(ev.data(), ev.size(), s);
  sm->face_v.upload(fv.data(), fv.size(), s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
  return sm;
}

static Dev dev_view(const StencilOp& a) {
  const StencilMesh& m = *a.mesh;
  const bool rows_are_edges = a.kind == kStQ || a.kind == kStCT;
  const bool cols_are_edges = a.kind == kStQ || a.kind == kStC;
  return Dev{m.n, m.nv, cols_are_edges ? m.eidT.p : m.fidT.p,
             rows_are_edges ? m.edge_v.p : m.face_v.p};
}

void stencil_build(const TetMesh& hm, const std::shared_ptr<StencilMesh>& sm, int kind,
                   const DevCSR* csr, StencilOp& out, cudaStream_t s) {
  stencil_init_tables();
  out.kind = kind;
  out.mesh = sm;
  const bool rows_are_edges = kind == kStQ || kind == kStCT;
  out.rows = rows_are_edges ? hm.n_edges : hm.n_faces;
  const std::vector<int8_t>& rt = rows_are_edges ? hm.edge_t : hm.face_t;
  // slices: <= 32 consecutive rows of one entity type
  std::vector<int64_t> hrow{0}, hptr{0}, rslice((size_t)out.rows);
  std::vector<int8_t> htype;
  int64_t r = 0;
  while (r < out.rows) {
    int64_t e = r + 1;
    while (e < out.rows && e - r < 32 && rt[(size_t)e] == rt[(size_t)r]) ++e;
    for (int64_t q = r; q < e; ++q) rslice[(size_t)q] = (int64_t)htype.size();
    htype.push_back(rt[(size_t)r]);
    hptr.push_back(hptr.back() + (int64_t)width_of(kind, rt[(size_t)r]) * (e - r));
    hrow.push_back(e);
    r = e;
  }
  out.n_slices = (int64_t)htype.size();
  out.slice_row.upload(hrow.data(), hrow.size(), s);
  out.slice_ptr.upload(hptr.data(), hptr.size(), s);
  out.slice_type.upload(htype.data(), htype.size(), s);
  const bool valued = kind == kStQ || kind == kStM2;
  if (valued) out.val.alloc((size_t)std::max<int64_t>(1, hptr.back()));
  if (csr) {  // values from the CSR + coverage / sign check
    DevBuf<int8_t> drt;
    DevBuf<int64_t> drs;
    DevBuf<int> bad;
    drt.upload(rt.data(), rt.size(), s);
    drs.upload(rslice.data(), rslice.size(), s);
    bad.alloc(1);
    bad.zero(s);
    Dev d = dev_view(out);
#define SFEEC_FILL(K)                                                                         \
  k_st_fill<K><<<nblk(out.rows, 256), 256, 0, s>>>(d, out.rows, drt.p, drs.p, out.slice_row.p, \
                                                   out.slice_ptr.p, csr->rp.p, csr->ci.p,     \
                                                   csr->val.p, out.val.p, bad.p)
    switch (kind) {
      case kStQ: SFEEC_FILL(kStQ); break;
      case kStM2: SFEEC_FILL(kStM2); break;
      case kStC: SFEEC_FILL(kStC); break;
      default: SFEEC_FILL(kStCT); break;
    }
#undef SFEEC_FILL
    SFEEC_LAUNCH_CHECK();
    int hb = 0;
    SFEEC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
    require(hb == 0, hb == 1 ? "stencil: operator entry outside the mesh stencil"
                             : "stencil: incidence sign differs from the stencil");
  }
  SFEEC_CUDA(cudaStreamSynchronize(s));
}

double StencilOp::stream_bytes() const {
  const bool valued = kind == kStQ || kind == kStM2;
  return (valued ? 8.0 * (double)val.n : 0.0) + 4.0 * (double)rows;
}

void launch_stencil(const StencilOp& a, const double* x, double* y, double alpha, bool accumulate,
                    cudaStream_t s) {
  if (a.rows == 0) return;
  const Dev d = dev_view(a);
  const unsigned g = (unsigned)std::min<int64_t>(nblk(a.n_slices * 32, kThreads), 148 * 4);
#define SFEEC_ST(K)                                                                            \
  if (accumulate)                                                                              \
    k_st<true, K, 4><<<g, kThreads, 0, s>>>(d, a.n_slices, a.slice_row.p, a.slice_ptr.p,       \
                                            a.slice_type.p, a.val.p, x, y, alpha);            \
  else                                                                                         \
    k_st<false, K, 4><<<g, kThreads, 0, s>>>(d, a.n_slices, a.slice_row.p, a.slice_ptr.p,      \
                                             a.slice_type.p, a.val.p, x, y, alpha);
  switch (a.kind) {
    case kStQ: SFEEC_ST(kStQ) break;
    case kStM2: SFEEC_ST(kStM2) break;
    case kStC: SFEEC_ST(kStC) break;
    default: SFEEC_ST(kStCT) break;
  }
#undef SFEEC_ST
  SFEEC_LAUNCH_CHECK();
}

}  // namespace sfeec_b200
