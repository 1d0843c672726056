// Host builders for the lumped (Yee) SFEEC operators in the sfeec_yee DOF
// numbering (yee_layout.hpp). Setup only.
//
// Entry values follow derivative_q1_p1 (reference operators.cpp:29-42):
// sign * |sub-face| / |face| with the measures taken from the unwrapped
// lattice coordinates exactly as face_volume (operators.cpp:13-27) does, so
// the periodic operator is bitwise the reference's. Boundary incidence and
// orientation follow generate_cubical_lattice (mesh_cubical.cpp:59-115):
//   face normal a, a1 = a+1, a2 = a+2:  +e_a1(p) +e_a2(p+a1) -e_a1(p+a2) -e_a2(p)
//   cell: +f_a(p+a) -f_a(p) for a = 0,1,2.
// PEC (new): boundary-edge columns are dropped.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.hpp"
#include "yee_layout.hpp"

namespace sfeec_b200 {

namespace {

struct V3 {
  double x, y, z;
};
inline double norm3(const V3& v) { return std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }

struct Lattice {
  YeeGeom g;
  double d[3];
  V3 corner(int i, int j, int k) const { return {i * d[0], j * d[1], k * d[2]}; }
  int wrap(int c, int dim) const {
    if (g.bc) return c;
    int n = g.n[dim];
    return ((c % n) + n) % n;
  }
  // measure of the axis-`ax` edge whose tail is (wrapped) c
  double edge_len(int ax, const int c[3]) const {
    int h[3] = {c[0], c[1], c[2]};
    h[ax] += 1;
    V3 a = corner(c[0], c[1], c[2]), b = corner(h[0], h[1], h[2]);
    return norm3({b.x - a.x, b.y - a.y, b.z - a.z});
  }
  // measure of the normal-`a` face at (wrapped) c: |x10 - x00| * |x01 - x00|
  double face_area(int a, const int c[3]) const {
    int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    int p10[3] = {c[0], c[1], c[2]}, p01[3] = {c[0], c[1], c[2]};
    p10[a1] += 1;
    p01[a2] += 1;
    V3 x00 = corner(c[0], c[1], c[2]), x10 = corner(p10[0], p10[1], p10[2]),
       x01 = corner(p01[0], p01[1], p01[2]);
    return norm3({x10.x - x00.x, x10.y - x00.y, x10.z - x00.z}) *
           norm3({x01.x - x00.x, x01.y - x00.y, x01.z - x00.z});
  }
};

// sparse.cpp:20-61 applied to one row's (col, val) list in input order
void finish_row(std::vector<std::pair<int32_t, double>>& in,
                std::vector<std::pair<int32_t, double>>& out) {
  std::stable_sort(in.begin(), in.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  out.clear();
  size_t i = 0;
  while (i < in.size()) {
    double s = 0;
    size_t j = i;
    while (j < in.size() && in[j].first == in[i].first) s += in[j++].second;
    if (s != 0.0) out.push_back({in[i].first, s});
    i = j;
  }
}

template <class RowFn>
HostCSR build_rows(int64_t rows, int64_t cols, RowFn&& fn, int max_row = 8) {
  HostCSR m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign((size_t)rows + 1, 0);
  std::vector<int32_t> tc((size_t)rows * max_row);
  std::vector<double> tv((size_t)rows * max_row);
  std::vector<int> cnt((size_t)rows);
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> in, out;
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      in.clear();
      fn(r, in);
      finish_row(in, out);
      if ((int)out.size() > max_row) out.resize((size_t)max_row + 1);  // flagged below
      cnt[(size_t)r] = (int)out.size();
      for (size_t k = 0; k < out.size() && (int)k < max_row; ++k) {
        tc[(size_t)r * max_row + k] = out[k].first;
        tv[(size_t)r * max_row + k] = out[k].second;
      }
    }
  }
  for (int64_t r = 0; r < rows; ++r) {
    require(cnt[(size_t)r] <= max_row, "lattice assembly: row longer than expected");
    m.row_ptr[(size_t)r + 1] = m.row_ptr[(size_t)r] + cnt[(size_t)r];
  }
  m.col_idx.resize((size_t)m.row_ptr[(size_t)rows]);
  m.val.resize((size_t)m.row_ptr[(size_t)rows]);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int k = 0; k < cnt[(size_t)r]; ++k) {
      m.col_idx[(size_t)(m.row_ptr[(size_t)r] + k)] = tc[(size_t)r * max_row + k];
      m.val[(size_t)(m.row_ptr[(size_t)r] + k)] = tv[(size_t)r * max_row + k];
    }
  return m;
}

}  // namespace

void build_yee_operators(int nx, int ny, int nz, double dx, double dy, double dz, int bc,
                         HostCSR* curl, HostCSR* div) {
  require(nx >= 1 && ny >= 1 && nz >= 1, "cubical lattice: cell counts must be >= 1");
  require(dx > 0 && dy > 0 && dz > 0, "cubical lattice: spacings must be > 0");
  require(bc == SFEEC_BC_PERIODIC || bc == SFEEC_BC_PEC, "unknown boundary condition");
  Lattice L;
  L.g = make_yee_geom(nx, ny, nz, bc);
  L.d[0] = dx;
  L.d[1] = dy;
  L.d[2] = dz;
  const YeeGeom& g = L.g;
  const int64_t n_faces = g.face_off[3], n_edges = g.edge_off[3];
  if (curl) {
    *curl = build_rows(n_faces, n_edges, [&](int64_t f, auto& in) {
      int a;
      int64_t s;
      g.dof_to_storage(true, f, a, s);
      int c[3] = {(int)(s % g.P0), (int)((s / g.P0) % g.S[1]),
                  (int)(s / ((int64_t)g.P0 * g.S[1]))};
      int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
      const double area = L.face_area(a, c);
      struct {
        int ax, d1, d2, sign;
      } terms[4] = {{a1, 0, 0, +1}, {a2, 1, 0, +1}, {a1, 0, 1, -1}, {a2, 0, 0, -1}};
      for (auto& t : terms) {
        int p[3] = {c[0], c[1], c[2]};
        p[a1] += t.d1;
        p[a2] += t.d2;
        for (int d = 0; d < 3; ++d) p[d] = L.wrap(p[d], d);
        int64_t e = g.dof_id(false, t.ax, p[0], p[1], p[2]);
        if (e < 0) continue;  // PEC: boundary edge, not a DOF
        double v = t.sign;
        v *= L.edge_len(t.ax, p) / area;
        in.push_back({(int32_t)e, v});
      }
    });
  }
  if (div) {
    const int64_t n_cells = (int64_t)nx * ny * nz;
    const double vol = dx * dy * dz;  // PeriodicMesh::cell_volume (mesh_common.cpp:11-16)
    *div = build_rows(n_cells, n_faces, [&](int64_t cell, auto& in) {
      int c[3] = {(int)(cell % nx), (int)((cell / nx) % ny), (int)(cell / ((int64_t)nx * ny))};
      for (int a = 0; a < 3; ++a) {
        for (int up = 1; up >= 0; --up) {
          int p[3] = {c[0], c[1], c[2]};
          p[a] += up;
          for (int d = 0; d < 3; ++d) p[d] = L.wrap(p[d], d);
          int64_t f = g.dof_id(true, a, p[0], p[1], p[2]);
          double v = up ? 1.0 : -1.0;
          v *= L.face_area(a, p) / vol;
          in.push_back({(int32_t)f, v});
        }
      }
    });
  }
}

// Consistent Q1- mass matrices of the lattice: reference mass_matrix
// (operators.cpp:133-179) with the Q1 element (form_space.cpp:295-321: basis
// values need no transform on cubes, jac_abs = dx dy dz) and the order-3 cube
// rule (quadrature.cpp:90-107: 2-point Gauss-Legendre per axis, weight
// 0.125 w_i w_j w_k). Element entries are summed over the rule in its point
// order with dot products over components from 0, scaled, mirrored exactly;
// rows gather their cells in ascending cell id and slot order, so duplicates
// sum in the reference's triplet order (sparse.cpp:20-61). Bitwise the
// reference on periodic lattices (its only case); PEC drops boundary edges.
HostCSR build_yee_mass(int nx, int ny, int nz, double dx, double dy, double dz, int bc, int form) {
  require(nx >= 1 && ny >= 1 && nz >= 1, "cubical lattice: cell counts must be >= 1");
  require(dx > 0 && dy > 0 && dz > 0, "cubical lattice: spacings must be > 0");
  require(bc == SFEEC_BC_PERIODIC || bc == SFEEC_BC_PEC, "unknown boundary condition");
  require(form == 1 || form == 2, "mass: form must be 1 or 2");
  Lattice L;
  L.g = make_yee_geom(nx, ny, nz, bc);
  L.d[0] = dx;
  L.d[1] = dy;
  L.d[2] = dz;
  const YeeGeom& g = L.g;
  const int nl = form == 1 ? 12 : 6;
  // reference basis values at the 8 rule points
  const double gx[2] = {-0.5773502691896257645, 0.5773502691896257645}, gw[2] = {1, 1};
  double rp[8][3], rw[8], ref[8][12][3];
  {
    int q = 0;
    for (int k = 0; k < 2; ++k)
      for (int j = 0; j < 2; ++j)
        for (int i = 0; i < 2; ++i, ++q) {
          rp[q][0] = 0.5 * (gx[i] + 1.0);
          rp[q][1] = 0.5 * (gx[j] + 1.0);
          rp[q][2] = 0.5 * (gx[k] + 1.0);
          rw[q] = 0.125 * gw[i] * gw[j] * gw[k];
        }
  }
  auto lshape = [](int b, double t) { return b ? t : 1.0 - t; };
  const int bb[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
  for (int q = 0; q < 8; ++q) {
    std::memset(ref[q], 0, sizeof(ref[q]));
    int l = 0;
    for (int a = 0; a < 3; ++a) {
      const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
      if (form == 1) {
        for (auto& b : bb) ref[q][l++][a] = lshape(b[0], rp[q][a1]) * lshape(b[1], rp[q][a2]);
      } else {
        for (int b = 0; b <= 1; ++b) ref[q][l++][a] = lshape(b, rp[q][a]);
      }
    }
  }
  const double scale = dx * dy * dz;
  double me[12][12];
  for (int i = 0; i < nl; ++i)
    for (int j = i; j < nl; ++j) {
      double acc = 0;
      for (int q = 0; q < 8; ++q) {
        double dot = 0;
        for (int k = 0; k < 3; ++k) dot += ref[q][i][k] * ref[q][j][k];
        acc += rw[q] * dot;
      }
      acc *= scale;
      me[i][j] = acc;
      me[j][i] = acc;
    }
  // local DOFs of cell c (mesh_cubical.cpp:136-165 local order), -1 = PEC boundary
  auto cell_dofs = [&](const int c[3], int64_t out[12]) {
    int l = 0;
    for (int a = 0; a < 3; ++a) {
      const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
      if (form == 1) {
        for (auto& b : bb) {
          int p[3] = {c[0], c[1], c[2]};
          p[a1] += b[0];
          p[a2] += b[1];
          for (int d = 0; d < 3; ++d) p[d] = L.wrap(p[d], d);
          out[l++] = g.dof_id(false, a, p[0], p[1], p[2]);
        }
      } else {
        for (int b = 0; b <= 1; ++b) {
          int p[3] = {c[0], c[1], c[2]};
          p[a] += b;
          for (int d = 0; d < 3; ++d) p[d] = L.wrap(p[d], d);
          out[l++] = g.dof_id(true, a, p[0], p[1], p[2]);
        }
      }
    }
  };
  const int n[3] = {nx, ny, nz};
  const int64_t rows = form == 1 ? g.edge_off[3] : g.face_off[3];
  return build_rows(rows, rows, [&](int64_t r, auto& in) {
    int a;
    int64_t s;
    g.dof_to_storage(form == 2, r, a, s);
    const int p[3] = {(int)(s % g.P0), (int)((s / g.P0) % g.S[1]),
                      (int)(s / ((int64_t)g.P0 * g.S[1]))};
    // candidate cells: a 1-form of axis a touches the 4 cells around it in the
    // (a1, a2) plane, a 2-form of normal a the 2 cells on either side
    const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    std::vector<int64_t> cells;
    for (int u = -1; u <= 0; ++u)
      for (int v = -1; v <= 0; ++v) {
        int c[3] = {p[0], p[1], p[2]};
        if (form == 1) {
          c[a1] += u;
          c[a2] += v;
        } else {
          if (v != 0) continue;
          c[a] += u;
        }
        bool ok = true;
        for (int d = 0; d < 3; ++d) {
          if (bc == SFEEC_BC_PERIODIC)
            c[d] = ((c[d] % n[d]) + n[d]) % n[d];
          else if (c[d] < 0 || c[d] >= n[d])
            ok = false;
        }
        if (ok) cells.push_back((int64_t)c[0] + (int64_t)nx * ((int64_t)c[1] + (int64_t)ny * c[2]));
      }
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    for (int64_t cid : cells) {
      const int c[3] = {(int)(cid % nx), (int)((cid / nx) % ny), (int)(cid / ((int64_t)nx * ny))};
      int64_t ld[12];
      cell_dofs(c, ld);
      for (int i = 0; i < nl; ++i) {
        if (ld[i] != r) continue;
        for (int j = 0; j < nl; ++j)
          if (ld[j] >= 0) in.push_back({(int32_t)ld[j], me[i][j]});
      }
    }
  }, form == 1 ? 16 : 8);
}

}  // namespace sfeec_b200

using namespace sfeec_b200;

extern "C" int sfeec_build_yee_mass(int nx, int ny, int nz, double dx, double dy, double dz,
                                    int bc, int form, sfeec_csr_owned* m) {
  return guarded([&] {
    require(m != nullptr, "null argument");
    csr_to_owned(build_yee_mass(nx, ny, nz, dx, dy, dz, bc, form), m);
  });
}

extern "C" int sfeec_build_yee_curl(int nx, int ny, int nz, double dx, double dy, double dz,
                                    int bc, sfeec_csr_owned* c, sfeec_csr_owned* div) {
  return guarded([&] {
    HostCSR hc, hd;
    build_yee_operators(nx, ny, nz, dx, dy, dz, bc, c ? &hc : nullptr, div ? &hd : nullptr);
    if (c) csr_to_owned(std::move(hc), c);
    if (div) csr_to_owned(std::move(hd), div);
  });
}
