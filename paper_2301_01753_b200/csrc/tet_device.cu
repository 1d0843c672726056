// Device assembly of the tet SFEEC system: C, D,
// M1, M2, the S(M1) SPAI and Q_sym built on the B200 straight into HBM, so
// configs 3 and 5 (128^3, 256^3 x 6 tets) set up in seconds instead of host
// minutes (and without ~200 GB of host memory at 256^3).
//
// Every entry is computed with the same operation sequence as the host
// builders (host_tet.cpp / host_sparse.cpp), with explicit round-to-nearest
// intrinsics (no FMA contraction), so the device operators are bitwise the
// host ones -- tests/test_gpu_tetdev.py checks that against the host path,
// which is itself bitwise the numpy construction oracle.
#include <cub/cub.cuh>

#include <memory>
#include <vector>

#include "dev_handle.hpp"
#include "device_util.cuh"
#include "spmv_kernels.cuh"
#include "table_lattice.cuh"
#include "tet_device.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

namespace {

__constant__ int dET[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0},
                              {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
__constant__ int dFT[12][2] = {{0, 3}, {1, 3}, {1, 4}, {2, 4}, {0, 5}, {2, 5},
                               {0, 6}, {1, 6}, {2, 6}, {3, 6}, {4, 6}, {5, 6}};
__constant__ int dPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int dLE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
__constant__ int dLF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

// exact IEEE operations (the host builds without FMA)
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

struct DMesh {
  int n;   // cubes along x, y
  int nz;  // cubes along z (TetMesh::nz: the whole mesh or a slab of it)
  const double* xyz;
  const int32_t* eid;  // nv * 7
  const int32_t* fid;  // nv * 12
  const int64_t* edge_v;
  const int8_t* edge_t;
  const int64_t* face_v;
  const int8_t* face_t;

  __device__ int64_t vid(int i, int j, int k) const {
    return (int64_t)i + (int64_t)(n + 1) * ((int64_t)j + (int64_t)(n + 1) * k);
  }
  __device__ void coords(int64_t v, int c[3]) const {
    c[0] = (int)(v % (n + 1));
    c[1] = (int)((v / (n + 1)) % (n + 1));
    c[2] = (int)(v / ((int64_t)(n + 1) * (n + 1)));
  }
  __device__ static int type_of(int dx, int dy, int dz) {
    for (int t = 0; t < 7; ++t)
      if (dET[t][0] == dx && dET[t][1] == dy && dET[t][2] == dz) return t;
    return -1;
  }
  __device__ void tet_vertices(int64_t tet, int64_t vv[4]) const {
    int64_t cube = tet / 6;
    int p = (int)(tet % 6);
    int c[3] = {(int)(cube % n), (int)((cube / n) % n), (int)(cube / ((int64_t)n * n))};
    vv[0] = vid(c[0], c[1], c[2]);
    c[dPerm[p][0]] += 1;
    vv[1] = vid(c[0], c[1], c[2]);
    c[dPerm[p][1]] += 1;
    vv[2] = vid(c[0], c[1], c[2]);
    c[dPerm[p][2]] += 1;
    vv[3] = vid(c[0], c[1], c[2]);
  }
  __device__ int32_t edge_of(int64_t a, int64_t b) const {
    int ca[3], cb[3];
    coords(a, ca);
    coords(b, cb);
    return eid[a * 7 + type_of(cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2])];
  }
  __device__ int32_t face_of(int64_t a, int64_t b, int64_t c) const {
    int ca[3], cb[3], cc[3];
    coords(a, ca);
    coords(b, cb);
    coords(c, cc);
    int t1 = type_of(cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2]);
    int t2 = type_of(cc[0] - ca[0], cc[1] - ca[1], cc[2] - ca[2]);
    for (int f = 0; f < 12; ++f)
      if (dFT[f][0] == t1 && dFT[f][1] == t2) return fid[a * 12 + f];
    return -1;
  }
  __device__ void edge_vertices(int64_t e, int64_t out[2]) const {
    int c[3];
    coords(edge_v[e], c);
    const int t = edge_t[e];
    out[0] = edge_v[e];
    out[1] = vid(c[0] + dET[t][0], c[1] + dET[t][1], c[2] + dET[t][2]);
  }
  __device__ void face_vertices(int64_t f, int64_t out[3]) const {
    int c[3];
    coords(face_v[f], c);
    const int ft = face_t[f];
    const int t1 = dFT[ft][0], t2 = dFT[ft][1];
    out[0] = face_v[f];
    out[1] = vid(c[0] + dET[t1][0], c[1] + dET[t1][1], c[2] + dET[t1][2]);
    out[2] = vid(c[0] + dET[t2][0], c[1] + dET[t2][1], c[2] + dET[t2][2]);
  }
  __device__ int containing_tets(const int64_t* vs, int m, int64_t out[8]) const {
    int c0[3];
    coords(vs[0], c0);
    int cnt = 0;
    for (int dz = 1; dz >= 0; --dz)
      for (int dy = 1; dy >= 0; --dy)
        for (int dx = 1; dx >= 0; --dx) {
          int w[3] = {c0[0] - dx, c0[1] - dy, c0[2] - dz};
          if (w[0] < 0 || w[0] >= n || w[1] < 0 || w[1] >= n || w[2] < 0 || w[2] >= nz) continue;
          int64_t cube = (int64_t)w[0] + (int64_t)n * ((int64_t)w[1] + (int64_t)n * w[2]);
          for (int p = 0; p < 6; ++p) {
            int64_t vv[4];
            tet_vertices(cube * 6 + p, vv);
            bool all = true;
            for (int q = 0; q < m && all; ++q)
              all = vs[q] == vv[0] || vs[q] == vv[1] || vs[q] == vv[2] || vs[q] == vv[3];
            if (all) out[cnt++] = cube * 6 + p;
          }
        }
    return cnt;
  }

  // gradients of the barycentric coordinates and int lambda_a lambda_b,
  // TetMesh::element's exact operation order
  __device__ void geometry(int64_t tet, double gl[4][3], double ml[4][4]) const {
    int64_t vv[4];
    tet_vertices(tet, vv);
    double x[4][3];
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 3; ++d) x[a][d] = xyz[3 * vv[a] + d];
    double e[3][3];
    for (int a = 0; a < 3; ++a)
      for (int d = 0; d < 3; ++d) e[a][d] = sub(x[a + 1][d], x[0][d]);
    auto cross = [](const double* u, const double* v, double* w) {
      w[0] = sub(mul(u[1], v[2]), mul(u[2], v[1]));
      w[1] = sub(mul(u[2], v[0]), mul(u[0], v[2]));
      w[2] = sub(mul(u[0], v[1]), mul(u[1], v[0]));
    };
    double c12[3], c20[3], c01[3];
    cross(e[1], e[2], c12);
    cross(e[2], e[0], c20);
    cross(e[0], e[1], c01);
    const double vol6 = add(add(mul(e[0][0], c12[0]), mul(e[0][1], c12[1])), mul(e[0][2], c12[2]));
    for (int d = 0; d < 3; ++d) {
      gl[1][d] = dv(c12[d], vol6);
      gl[2][d] = dv(c20[d], vol6);
      gl[3][d] = dv(c01[d], vol6);
      gl[0][d] = -add(add(gl[1][d], gl[2][d]), gl[3][d]);
    }
    const double vol = dv(fabs(vol6), 6.0);
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) ml[a][b] = a == b ? dv(vol, 10.0) : dv(vol, 20.0);
  }
};

__device__ __forceinline__ double gdot(const double* a, const double* b) {
  return add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2]));
}

// M1 element entry (p, q), TetMesh::element
__device__ double m1_entry(const double gl[4][3], const double ml[4][4], int p, int q) {
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
  const int i = dLE[p][0], j = dLE[p][1], k = dLE[q][0], l = dLE[q][1];
  double v = mul(ml[i][k], gdot(gl[j], gl[l]));
  v = sub(v, mul(ml[i][l], gdot(gl[j], gl[k])));
  v = sub(v, mul(ml[j][k], gdot(gl[i], gl[l])));
  v = add(v, mul(ml[j][l], gdot(gl[i], gl[k])));
  return v;
}

// M2 element entry (f, h)
__device__ double m2_entry(const double gl[4][3], const double ml[4][4], int f, int h) {
  if (f > h) {
    int t = f;
    f = h;
    h = t;
  }
  auto terms = [&](int face, int t, double cv[3]) -> int {
    const int a = dLF[face][0], b = dLF[face][1], c = dLF[face][2];
    const int tri[3][3] = {{a, b, c}, {b, c, a}, {c, a, b}};
    const double* u = gl[tri[t][1]];
    const double* v = gl[tri[t][2]];
    cv[0] = sub(mul(u[1], v[2]), mul(u[2], v[1]));
    cv[1] = sub(mul(u[2], v[0]), mul(u[0], v[2]));
    cv[2] = sub(mul(u[0], v[1]), mul(u[1], v[0]));
    return tri[t][0];
  };
  double acc = 0.0;
  for (int s = 0; s < 3; ++s) {
    double cf[3];
    const int lf = terms(f, s, cf);
    for (int t = 0; t < 3; ++t) {
      double ch[3];
      const int lh = terms(h, t, ch);
      acc = add(acc, mul(ml[lf][lh], gdot(cf, ch)));
    }
  }
  return mul(4.0, acc);
}

// small per-thread accumulator: (col, value) pairs summed in arrival order
template <int CAP>
struct RowAcc {
  int32_t c[CAP];
  double v[CAP];
  int n = 0;
  __device__ void add_to(int32_t col, double val) {
    for (int i = 0; i < n; ++i)
      if (c[i] == col) {
        v[i] = add(v[i], val);
        return;
      }
    c[n] = col;
    v[n] = add(0.0, val);
    ++n;
  }
  // sort by column (stable insertion), drop exact zeros; returns count
  __device__ int finish() {
    for (int i = 1; i < n; ++i) {
      int32_t kc = c[i];
      double kv = v[i];
      int j = i - 1;
      while (j >= 0 && c[j] > kc) {
        c[j + 1] = c[j];
        v[j + 1] = v[j];
        --j;
      }
      c[j + 1] = kc;
      v[j + 1] = kv;
    }
    int w = 0;
    for (int i = 0; i < n; ++i)
      if (v[i] != 0.0) {
        c[w] = c[i];
        v[w] = v[i];
        ++w;
      }
    return w;
  }
};

// OP: 0 C (faces x edges), 1 M1 (edges), 2 M2 (faces), 3 D (tets x faces)
template <int OP, int CAP>
__device__ int build_row(const DMesh& m, int64_t r, RowAcc<CAP>& acc) {
  if (OP == 0) {
    int64_t v[3];
    m.face_vertices(r, v);
    const int64_t pr[3][2] = {{v[1], v[2]}, {v[0], v[2]}, {v[0], v[1]}};
    const double sg[3] = {1.0, -1.0, 1.0};
    for (int t = 0; t < 3; ++t) {
      int32_t e = m.edge_of(pr[t][0], pr[t][1]);
      if (e >= 0) acc.add_to(e, sg[t]);
    }
  } else if (OP == 3) {
    int64_t v[4];
    m.tet_vertices(r, v);
    for (int f = 0; f < 4; ++f)
      acc.add_to(m.face_of(v[dLF[f][0]], v[dLF[f][1]], v[dLF[f][2]]), (f % 2 == 0) ? 1.0 : -1.0);
  } else {
    const int nl = OP == 1 ? 6 : 4;
    int64_t vs[3];
    int nvs;
    if (OP == 1) {
      m.edge_vertices(r, vs);
      nvs = 2;
    } else {
      m.face_vertices(r, vs);
      nvs = 3;
    }
    int64_t tets[8];
    const int nt = m.containing_tets(vs, nvs, tets);
    for (int a = 0; a < nt; ++a) {
      const int64_t t = tets[a];
      int64_t vv[4];
      m.tet_vertices(t, vv);
      int32_t ids[6];
      int p = -1;
      for (int q = 0; q < nl; ++q) {
        ids[q] = OP == 1 ? m.edge_of(vv[dLE[q][0]], vv[dLE[q][1]])
                         : m.face_of(vv[dLF[q][0]], vv[dLF[q][1]], vv[dLF[q][2]]);
        if (ids[q] == (int32_t)r) p = q;
      }
      double gl[4][3], ml[4][4];
      m.geometry(t, gl, ml);
      for (int q = 0; q < nl; ++q) {
        if (ids[q] < 0) continue;  // boundary edge (PEC)
        acc.add_to(ids[q], OP == 1 ? m1_entry(gl, ml, p, q) : m2_entry(gl, ml, p, q));
      }
    }
  }
  return acc.finish();
}

template <int OP, int CAP>
__global__ void __launch_bounds__(128) k_rows(DMesh m, int64_t rows, int64_t* __restrict__ row_len,
                                              const int64_t* __restrict__ rp,
                                              int32_t* __restrict__ ci, double* __restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  RowAcc<CAP> acc;
  const int w = build_row<OP, CAP>(m, r, acc);
  if (row_len) {
    row_len[r] = w;
    return;
  }
  const int64_t o = rp[r];
  for (int i = 0; i < w; ++i) {
    ci[o + i] = acc.c[i];
    val[o + i] = acc.v[i];
  }
}

// ---- SPAI: one warp per column (spai.cpp:176-233 / host_tet.cpp spai) ----
constexpr int kSpaiK = 32;  // max pattern size handled on the device
constexpr int kSpaiWarps = 4;

__global__ void __launch_bounds__(32 * kSpaiWarps)
    k_spai(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ va, double* __restrict__ qcol, int32_t* __restrict__ flags,
           double* __restrict__ res2) {
  __shared__ double sG[kSpaiWarps][kSpaiK][kSpaiK + 1];
  __shared__ double sQ[kSpaiWarps][kSpaiK];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t l = (int64_t)blockIdx.x * kSpaiWarps + w;
  if (l >= n) return;
  const int64_t b = rp[l];
  const int k = (int)(rp[l + 1] - b);
  if (k > kSpaiK) {
    if (lane == 0) flags[l] = 2;  // too large for the device path
    return;
  }
  double(*G)[kSpaiK + 1] = sG[w];
  // Gram(a, c) = sum_m M(idx_a, m) M(idx_c, m), m ascending (sparse_square order)
  const int npairs = k * (k + 1) / 2;
  for (int pidx = lane; pidx < npairs; pidx += 32) {
    int a = 0, rem = pidx;
    while (rem >= k - a) {
      rem -= k - a;
      ++a;
    }
    const int c = a + rem;
    const int32_t ra = ci[b + a], rc = ci[b + c];
    int64_t x = rp[ra], xe = rp[ra + 1], y = rp[rc], ye = rp[rc + 1];
    double s = 0.0;
    while (x < xe && y < ye) {
      const int32_t cx = ci[x], cy = ci[y];
      if (cx == cy) {
        s = add(s, mul(va[x], va[y]));
        ++x;
        ++y;
      } else if (cx < cy) {
        ++x;
      } else {
        ++y;
      }
    }
    G[a][c] = s;
    G[c][a] = s;
  }
  __syncwarp();
  double trace = 0.0;
  for (int a = 0; a < k; ++a) trace = add(trace, G[a][a]);  // every lane, same order
  // Cholesky in place (lower), host_tet.cpp order: column j, then rows i > j
  bool ok = true;
  double dmin = INFINITY;
  for (int j = 0; j < k; ++j) {
    double d = G[j][j];
    for (int p = 0; p < j; ++p) d = sub(d, mul(G[j][p], G[j][p]));
    if (!(d > 0)) {
      ok = false;
      break;
    }
    dmin = fmin(dmin, d);
    const double ljj = __dsqrt_rn(d);
    __syncwarp();
    for (int i = j + 1 + lane; i < k; i += 32) {
      double s = G[i][j];
      for (int p = 0; p < j; ++p) s = sub(s, mul(G[i][p], G[j][p]));
      G[i][j] = dv(s, ljj);
    }
    __syncwarp();
    if (lane == 0) G[j][j] = ljj;
    __syncwarp();
  }
  if (ok && dmin > mul(1e-12, trace)) {
    if (lane == 0) {
      double* q = sQ[w];
      for (int i = 0; i < k; ++i) {
        double s = va[b + i];  // rhs(a) = M(l, idx_a)
        for (int p = 0; p < i; ++p) s = sub(s, mul(G[i][p], q[p]));
        q[i] = dv(s, G[i][i]);
      }
      for (int i = k - 1; i >= 0; --i) {
        double s = q[i];
        for (int p = i + 1; p < k; ++p) s = sub(s, mul(G[p][i], q[p]));
        q[i] = dv(s, G[i][i]);
      }
      bool fin = true;
      for (int i = 0; i < k; ++i) fin = fin && isfinite(q[i]);
      flags[l] = fin ? 0 : 1;
    }
  } else if (lane == 0) {
    flags[l] = 1;  // eigenvalue-thresholded fallback needed (host)
  }
  __syncwarp();
  if (flags[l] == 0)
    for (int i = lane; i < k; i += 32) qcol[b + i] = sQ[w][i];
  if (res2 && lane == 0) res2[l] = 0.0;
}

// Q_sym(r, c) = 0.5 Q(r, c) + 0.5 Q(c, r), Q(r, c) = q_c[pos of r in I_c]
// (csr_symmetric_part on the SPAI assembled by rows)
__device__ __forceinline__ int64_t find_in_row(const int64_t* rp, const int32_t* ci, int32_t row,
                                               int32_t col) {
  int64_t lo = rp[row], hi = rp[row + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ci[mid] < col)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_qsym(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ qcol, double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    const int32_t c = ci[k];
    const double q_rc = qcol[find_in_row(rp, ci, c, (int32_t)r)];  // column c at row r
    const double q_cr = qcol[k];                                    // column r at row c
    out[k] = add(add(0.0, mul(0.5, q_rc)), mul(0.5, q_cr));
  }
}

// ---- transpose via key sort ----------------------------------------------
__global__ void k_keys(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       uint64_t* __restrict__ keys, int64_t* __restrict__ idx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    keys[k] = ((uint64_t)(uint32_t)ci[k] << 32) | (uint64_t)(uint32_t)r;
    idx[k] = k;
  }
}
__global__ void k_unkeys(int64_t nnz, const uint64_t* __restrict__ keys, const int64_t* __restrict__ idx,
                         const double* __restrict__ val, int32_t* __restrict__ tci,
                         double* __restrict__ tval, unsigned long long* __restrict__ counts) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  tci[k] = (int32_t)(keys[k] & 0xffffffffu);
  tval[k] = val[idx[k]];
  atomicAdd(&counts[(keys[k] >> 32) + 1], 1ull);
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace


void exclusive_scan(int64_t* d, int64_t n, cudaStream_t s) {
  // in-place exclusive scan of n + 1 entries (last = total)
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, d, d, n + 1, s);
  DevBuf<char> t;
  t.alloc(tmp);
  cub::DeviceScan::ExclusiveSum(t.p, tmp, d, d, n + 1, s);
  SFEEC_LAUNCH_CHECK();
}

template <int OP, int CAP>
static void build_op(const DMesh& m, int64_t rows, int64_t cols, DevCSR& out, cudaStream_t s) {
  out.rows = rows;
  out.cols = cols;
  out.rp.alloc((size_t)rows + 1);
  SFEEC_CUDA(cudaMemsetAsync(out.rp.p, 0, sizeof(int64_t) * (size_t)(rows + 1), s));
  k_rows<OP, CAP><<<nblk(rows, 128), 128, 0, s>>>(m, rows, out.rp.p, nullptr, nullptr, nullptr);
  SFEEC_LAUNCH_CHECK();
  exclusive_scan(out.rp.p, rows, s);
  SFEEC_CUDA(cudaMemcpyAsync(&out.nnz, out.rp.p + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  out.ci.alloc((size_t)std::max<int64_t>(1, out.nnz));
  out.val.alloc((size_t)std::max<int64_t>(1, out.nnz));
  k_rows<OP, CAP><<<nblk(rows, 128), 128, 0, s>>>(m, rows, nullptr, out.rp.p, out.ci.p, out.val.p);
  SFEEC_LAUNCH_CHECK();
}

void transpose_dev(const DevCSR& a, DevCSR& t, cudaStream_t s) {
  t.rows = a.cols;
  t.cols = a.rows;
  t.nnz = a.nnz;
  DevBuf<uint64_t> k0, k1;
  DevBuf<int64_t> i0, i1;
  k0.alloc((size_t)a.nnz);
  k1.alloc((size_t)a.nnz);
  i0.alloc((size_t)a.nnz);
  i1.alloc((size_t)a.nnz);
  k_keys<<<nblk(a.rows, 256), 256, 0, s>>>(a.rows, a.rp.p, a.ci.p, k0.p, i0.p);
  SFEEC_LAUNCH_CHECK();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.p, k1.p, i0.p, i1.p, (int64_t)a.nnz, 0, 64, s);
  {
    DevBuf<char> tb;
    tb.alloc(tmp);
    cub::DeviceRadixSort::SortPairs(tb.p, tmp, k0.p, k1.p, i0.p, i1.p, (int64_t)a.nnz, 0, 64, s);
    SFEEC_LAUNCH_CHECK();
    SFEEC_CUDA(cudaStreamSynchronize(s));
  }
  k0.reset();
  i0.reset();
  t.ci.alloc((size_t)std::max<int64_t>(1, a.nnz));
  t.val.alloc((size_t)std::max<int64_t>(1, a.nnz));
  DevBuf<unsigned long long> cnt;
  cnt.alloc((size_t)t.rows + 1);
  SFEEC_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * (size_t)(t.rows + 1), s));
  k_unkeys<<<nblk(a.nnz, 256), 256, 0, s>>>(a.nnz, k1.p, i1.p, a.val.p, t.ci.p, t.val.p, cnt.p);
  SFEEC_LAUNCH_CHECK();
  t.rp.alloc((size_t)t.rows + 1);
  size_t tmp2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp2, (int64_t*)cnt.p, t.rp.p, t.rows + 1, s);
  DevBuf<char> tb2;
  tb2.alloc(tmp2);
  cub::DeviceScan::InclusiveSum(tb2.p, tmp2, (int64_t*)cnt.p, t.rp.p, t.rows + 1, s);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
}

void qsym_device(int64_t n, const int64_t* rp, const int32_t* ci, const double* qcol, double* out,
                 cudaStream_t s) {
  k_qsym<<<nblk(n, 256), 256, 0, s>>>(n, rp, ci, qcol, out);
  SFEEC_LAUNCH_CHECK();
}

namespace {
__global__ void k_slice_rp(int64_t n, const int64_t* __restrict__ rp, int64_t r0,
                           int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = rp[r0 + i] - rp[r0];
}
__global__ void k_slice_ci(int64_t nnz, const int32_t* __restrict__ ci, const double* __restrict__ v,
                           int64_t off, int64_t c0, int64_t ncols, int32_t* __restrict__ oci,
                           double* __restrict__ ov, int* __restrict__ bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int64_t c = (int64_t)ci[off + k] - c0;
  if (c < 0 || c >= ncols) *bad = 1;
  oci[k] = (int32_t)c;
  ov[k] = v[off + k];
}
}  // namespace

void slice_rows_device(const DevCSR& a, int64_t r0, int64_t r1, int64_t c0, int64_t ncols,
                       DevCSR& out, cudaStream_t s) {
  int64_t off = 0, end = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&off, a.rp.p + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaMemcpyAsync(&end, a.rp.p + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  out.rows = r1 - r0;
  out.cols = ncols;
  out.nnz = end - off;
  out.rp.alloc((size_t)out.rows + 1);
  out.ci.alloc((size_t)std::max<int64_t>(1, out.nnz));
  out.val.alloc((size_t)std::max<int64_t>(1, out.nnz));
  DevBuf<int> bad;
  bad.alloc(1);
  bad.zero(s);
  k_slice_rp<<<nblk(out.rows + 1, 256), 256, 0, s>>>(out.rows, a.rp.p, r0, out.rp.p);
  if (out.nnz)
    k_slice_ci<<<nblk(out.nnz, 256), 256, 0, s>>>(out.nnz, a.ci.p, a.val.p, off, c0, ncols,
                                                   out.ci.p, out.val.p, bad.p);
  SFEEC_LAUNCH_CHECK();
  int hb = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  require(hb == 0, "partition: an owned row references entities beyond the one-plane halo");
}

// Builds the first-order S(M1) system of mesh `h` on the current device.
void build_tet_system_device(const TetMesh& h, bool want_div, DevTetSystem& out, cudaStream_t s,
                             int exact_lo, int exact_hi) {
  DevBuf<double> xyz;
  DevBuf<int32_t> eid, fid;
  DevBuf<int64_t> ev, fv;
  DevBuf<int8_t> et, ft;
  xyz.upload(h.xyz.data(), h.xyz.size(), s);
  eid.upload(h.eid.data(), h.eid.size(), s);
  fid.upload(h.fid.data(), h.fid.size(), s);
  ev.upload(h.edge_v.data(), h.edge_v.size(), s);
  et.upload(h.edge_t.data(), h.edge_t.size(), s);
  fv.upload(h.face_v.data(), h.face_v.size(), s);
  ft.upload(h.face_t.data(), h.face_t.size(), s);
  DMesh m{h.n, h.nz, xyz.p, eid.p, fid.p, ev.p, et.p, fv.p, ft.p};
  out.n1 = h.n_edges;
  out.n2 = h.n_faces;
  out.nt = h.n_tets;
  build_op<0, 4>(m, h.n_faces, h.n_edges, out.c, s);
  build_op<2, 8>(m, h.n_faces, h.n_faces, out.m2, s);
  if (want_div) build_op<3, 4>(m, h.n_tets, h.n_faces, out.d, s);
  DevCSR m1;
  build_op<1, 32>(m, h.n_edges, h.n_edges, m1, s);
  // SPAI on S(M1): column l's pattern is M1's row l
  DevBuf<double> qcol;
  DevBuf<int32_t> flags;
  qcol.alloc((size_t)m1.nnz);
  flags.alloc((size_t)h.n_edges);
  k_spai<<<nblk(h.n_edges, kSpaiWarps), 32 * kSpaiWarps, 0, s>>>(h.n_edges, m1.rp.p, m1.ci.p,
                                                                  m1.val.p, qcol.p, flags.p, nullptr);
  SFEEC_LAUNCH_CHECK();
  {
    std::vector<int32_t> hf((size_t)h.n_edges);
    SFEEC_CUDA(cudaMemcpyAsync(hf.data(), flags.p, sizeof(int32_t) * hf.size(), cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
    // (on a slab, columns near the cut planes see incomplete M1 rows; only
    // the columns of edges in local planes [exact_lo, exact_hi) must solve)
    for (int64_t l = 0; l < h.n_edges; ++l) {
      if (!hf[(size_t)l]) continue;
      int c[3];
      h.coords(h.edge_v[(size_t)l], c);
      out.fallback += c[2] >= exact_lo && c[2] < exact_hi;
    }
  }
  require(out.fallback == 0,
          "device SPAI: some columns need the eigenvalue-thresholded fallback; use the host builder");
  out.qsym.rows = out.qsym.cols = h.n_edges;
  out.qsym.nnz = m1.nnz;
  out.qsym.val.alloc((size_t)m1.nnz);
  k_qsym<<<nblk(h.n_edges, 256), 256, 0, s>>>(h.n_edges, m1.rp.p, m1.ci.p, qcol.p, out.qsym.val.p);
  SFEEC_LAUNCH_CHECK();
  SFEEC_CUDA(cudaStreamSynchronize(s));
  // Q_sym shares M1's pattern (S(M1) is symmetric; no exact zeros in practice:
  // checked on download in the tests)
  out.qsym.rp = std::move(m1.rp);
  out.qsym.ci = std::move(m1.ci);
  transpose_dev(out.c, out.ct, s);
}

}  // namespace sfeec_b200

using namespace sfeec_b200;


namespace {

HostCSR download(DevCSR& a, cudaStream_t s) {
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
  a.rp.reset();
  a.ci.reset();
  a.val.reset();
  return h;
}

}  // namespace

extern "C" {

// Tet system of BASELINE configs 1/3/5 assembled on the device (mesh
// numbering on the host, C, D, M1, M2, S(M1) SPAI, Q_sym on the GPU), then
// the leapfrog handle. counts[3] = {N1, N2, T} (nullable).
int sfeec_tet_dev_create(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                         int split_kind, int device, int flags, int with_div, sfeec_dev** out,
                         int64_t* counts) {
  return guarded([&] {
    require(out != nullptr, "null out");
    *out = nullptr;
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    select_device(device);
    TetMesh mesh;
    mesh.build(n, jitter, seed);
    Stream st;
    DevTetSystem sys;
    build_tet_system_device(mesh, with_div != 0, sys, st.s);
    if (counts) {
      counts[0] = sys.n1;
      counts[1] = sys.n2;
      counts[2] = sys.nt;
    }
    if (!(flags & SFEEC_TET_HOST_LAYOUT) && !(flags & SFEEC_TET_STENCIL_LAYOUT)) {
      // default: the sliced / ELL layouts built on the device from the device
      // CSRs (only row pointers visit the host)
      // plus, by default, the Kuhn-lattice form of Q_sym and M2 that
      // advance() runs on (lattice.cuh; SFEEC_TET_NO_LATTICE keeps the
      // sliced / ELL kernels for the step as well)
      std::unique_ptr<LatticeOps> lat;
      // the lattice kernels' one-wave grids are latency-bound below ~48^3
      // cubes, where the sliced kernels (PDL, CUDA graphs) step faster:
      // tet16 0.0179 vs 0.0089 ms per step
      const bool want_lat = (flags & SFEEC_TET_LATTICE) || (!(flags & SFEEC_TET_NO_LATTICE) && n >= 48);
      if ((flags & SFEEC_TET_TABLE_LATTICE) && !(flags & SFEEC_STRICT)) {
        // the table-driven lattice (config 4's layout) on the first-order system
        TLDofs d1, d2;
        d1.ntypes = 7;
        d1.type.assign(mesh.edge_t.begin(), mesh.edge_t.end());
        d1.vertex = mesh.edge_v;
        d2.ntypes = 12;
        d2.type.assign(mesh.face_t.begin(), mesh.face_t.end());
        d2.vertex = mesh.face_v;
        auto tl = std::make_unique<TableLattice>();
        tl->build(n, 1, d1, d2, sys.qsym, sys.m2, sys.c, sys.ct, st.s);
        lat = std::move(tl);
      } else if (want_lat && !(flags & SFEEC_STRICT)) {
        auto l1 = std::make_unique<Lattice>();
        l1->build(mesh, sys.qsym, sys.m2, st.s);
        lat = std::move(l1);
      }
      DevOperator q, c, ct, m2, div;
      q.upload_device(std::move(sys.qsym), st.s);
      m2.upload_device(std::move(sys.m2), st.s);
      c.upload_device(std::move(sys.c), st.s);
      ct.upload_device(std::move(sys.ct), st.s);
      if (with_div) div.upload_device(std::move(sys.d), st.s);
      cudaStream_t hs;
      SFEEC_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
      *out = make_dev_from_ops(std::move(q), std::move(c), std::move(ct), std::move(m2),
                               with_div ? &div : nullptr, sys.n1, sys.n2, dt, eps0, mu0,
                               split_kind, device, flags & ~(SFEEC_TET_NO_LATTICE | SFEEC_TET_LATTICE | SFEEC_TET_TABLE_LATTICE), hs,
                               std::move(lat));
      return;
    }
    require(!(flags & SFEEC_TET_STENCIL_LAYOUT), "the stencil layout was removed");
    sys.ct.rp.reset();  // the handle transposes C itself
    sys.ct.ci.reset();
    sys.ct.val.reset();
    HostCSR hc = download(sys.c, st.s);
    HostCSR hm2 = download(sys.m2, st.s);
    HostCSR hq = download(sys.qsym, st.s);
    std::unique_ptr<HostCSR> hd;
    if (with_div) hd = std::make_unique<HostCSR>(download(sys.d, st.s));
    mesh = TetMesh();
    *out = make_dev_from_host(std::move(hq), std::move(hc), std::move(hm2), hd.get(), dt, eps0, mu0,
                              split_kind, SFEEC_FORM_BE, device, flags | SFEEC_Q_IS_SYMMETRIC);
  });
}

// The device-assembled operators, downloaded (nullable outputs): for parity
// tests against the host builders.
int sfeec_tet_dev_operators(int n, double jitter, uint64_t seed, int device, sfeec_csr_owned* c,
                            sfeec_csr_owned* m2, sfeec_csr_owned* d, sfeec_csr_owned* q_sym,
                            sfeec_csr_owned* ct) {
  return guarded([&] {
    select_device(device);
    TetMesh mesh;
    mesh.build(n, jitter, seed);
    Stream st;
    DevTetSystem sys;
    build_tet_system_device(mesh, d != nullptr, sys, st.s);
    if (c) csr_to_owned(download(sys.c, st.s), c);
    if (m2) csr_to_owned(download(sys.m2, st.s), m2);
    if (d) csr_to_owned(download(sys.d, st.s), d);
    if (q_sym) csr_to_owned(download(sys.qsym, st.s), q_sym);
    if (ct) csr_to_owned(download(sys.ct, st.s), ct);
  });
}

}  // extern "C"
