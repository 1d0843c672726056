// Second-order trimmed Whitney forms P2^- Lambda^k on the Kuhn tet mesh
// (BASELINE config 4). DOF conventions and tables: tools/gen_p2_tables.py,
// DESIGN.md 3.3. Numbering is k-major like the first-order one (tet_mesh.hpp):
// block (k, j, 32-vertex x-block), then
//   1-forms: edge type t, slot s (moments 1, 2t-1), i   (interior edges)
//            face type f, slot s (int dp^u, int dq^u), i (interior faces)
//   2-forms: face type f, slot s (moments l_a, l_b, l_c), i (all faces)
//            tet perm p, slot s (int ds_k ^ w), i          (all tets)
// so a z-slab of vertex planes is a contiguous range of every DOF vector.
#pragma once
#include <cmath>
#include <cstdint>
#include <memory>
#include <vector>

#include "p2_tables.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

struct P2Dofs {
  int64_t n1 = 0, n2 = 0, n3 = 0;
  std::vector<int32_t> e1;  // 2 * n_edges: 1-form DOFs of interior edges
  std::vector<int32_t> f1;  // 2 * n_faces: 1-form DOFs of faces (-1 on the PEC boundary)
  std::vector<int32_t> f2;  // 3 * n_faces
  std::vector<int32_t> t2;  // 3 * n_tets
  // inverse maps: entity id and (kind | slot << 1); kind 0 edge / face, 1 face / tet
  std::vector<int64_t> ent1, ent2;
  std::vector<int8_t> ks1, ks2;

  static bool boundary_face(const TetMesh& m, const int c[3], int f) {
    const int* a = kET[kFT[f][0]];
    const int* b = kET[kFT[f][1]];
    for (int d = 0; d < 3; ++d)
      if (a[d] == 0 && b[d] == 0 && (c[d] == 0 || c[d] == m.n)) return true;
    return false;
  }

  void build(const TetMesh& m) {
    const int n = m.n;
    e1.assign((size_t)(2 * m.n_edges), -1);
    f1.assign((size_t)(2 * m.n_faces), -1);
    f2.assign((size_t)(3 * m.n_faces), -1);
    t2.assign((size_t)(3 * m.n_tets), -1);
    int64_t a1 = 0, a2 = 0;
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n; ++j)
        for (int ib = 0; ib <= n; ib += kBlock) {
          const int ie = std::min(ib + kBlock, n + 1);
          for (int t = 0; t < 7; ++t)
            for (int s = 0; s < 2; ++s)
              for (int i = ib; i < ie; ++i) {
                const int32_t e = m.eid[(size_t)(m.vid(i, j, k) * 7 + t)];
                if (e >= 0) e1[(size_t)(2 * e + s)] = (int32_t)a1++;
              }
          for (int f = 0; f < 12; ++f)
            for (int s = 0; s < 2; ++s)
              for (int i = ib; i < ie; ++i) {
                const int32_t id = m.fid[(size_t)(m.vid(i, j, k) * 12 + f)];
                const int c[3] = {i, j, k};
                if (id >= 0 && !boundary_face(m, c, f)) f1[(size_t)(2 * id + s)] = (int32_t)a1++;
              }
          for (int f = 0; f < 12; ++f)
            for (int s = 0; s < 3; ++s)
              for (int i = ib; i < ie; ++i) {
                const int32_t id = m.fid[(size_t)(m.vid(i, j, k) * 12 + f)];
                if (id >= 0) f2[(size_t)(3 * id + s)] = (int32_t)a2++;
              }
          if (j < n && k < n)
            for (int p = 0; p < 6; ++p)
              for (int s = 0; s < 3; ++s)
                for (int i = ib; i < std::min(ie, n); ++i) {
                  const int64_t cube = (int64_t)i + (int64_t)n * ((int64_t)j + (int64_t)n * k);
                  t2[(size_t)(3 * (6 * cube + p) + s)] = (int32_t)a2++;
                }
        }
    require(a1 < INT32_MAX && a2 < INT32_MAX, "P2 mesh: DOF count exceeds int32");
    n1 = a1;
    n2 = a2;
    n3 = 4 * m.n_tets;
    ent1.assign((size_t)n1, 0);
    ks1.assign((size_t)n1, 0);
    ent2.assign((size_t)n2, 0);
    ks2.assign((size_t)n2, 0);
    for (int64_t e = 0; e < m.n_edges; ++e)
      for (int s = 0; s < 2; ++s) {
        const int32_t d = e1[(size_t)(2 * e + s)];
        ent1[(size_t)d] = e;
        ks1[(size_t)d] = (int8_t)(0 | (s << 1));
      }
    for (int64_t f = 0; f < m.n_faces; ++f) {
      for (int s = 0; s < 2; ++s) {
        const int32_t d = f1[(size_t)(2 * f + s)];
        if (d < 0) continue;
        ent1[(size_t)d] = f;
        ks1[(size_t)d] = (int8_t)(1 | (s << 1));
      }
      for (int s = 0; s < 3; ++s) {
        const int32_t d = f2[(size_t)(3 * f + s)];
        ent2[(size_t)d] = f;
        ks2[(size_t)d] = (int8_t)(0 | (s << 1));
      }
    }
    for (int64_t t = 0; t < m.n_tets; ++t)
      for (int s = 0; s < 3; ++s) {
        const int32_t d = t2[(size_t)(3 * t + s)];
        ent2[(size_t)d] = t;
        ks2[(size_t)d] = (int8_t)(1 | (s << 1));
      }
  }

  // global DOF ids of tet t's local 1-form (20) and 2-form (15) DOFs, -1 if
  // not a DOF (PEC boundary)
  void local_dofs(const TetMesh& m, int64_t t, int32_t d1[20], int32_t d2[15]) const {
    int64_t v[4];
    m.tet_vertices(t, v);
    for (int p = 0; p < 6; ++p) {
      const int32_t e = m.edge_of(v[kLE[p][0]], v[kLE[p][1]]);
      for (int s = 0; s < 2; ++s) d1[2 * p + s] = e >= 0 ? e1[(size_t)(2 * e + s)] : -1;
    }
    for (int q = 0; q < 4; ++q) {
      const int32_t f = m.face_of(v[kLF[q][0]], v[kLF[q][1]], v[kLF[q][2]]);
      for (int s = 0; s < 2; ++s) d1[12 + 2 * q + s] = f1[(size_t)(2 * f + s)];
      for (int s = 0; s < 3; ++s) d2[3 * q + s] = f2[(size_t)(3 * f + s)];
    }
    for (int s = 0; s < 3; ++s) d2[12 + s] = t2[(size_t)(3 * t + s)];
  }
};

// Metric tensors of tet t: G1 = |det J| J^-1 J^-T, G2 = J^T J / |det J|,
// J = [x1 - x0, x2 - x0, x3 - x0] in ascending local vertex order. Returns det J.
inline double p2_metric(const TetMesh& m, int64_t t, double g1[3][3], double g2[3][3]) {
  int64_t v[4];
  m.tet_vertices(t, v);
  double J[3][3];  // J[d][c] = (x_{c+1} - x_0)_d
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d)
      J[d][c] = m.xyz[(size_t)(3 * v[c + 1] + d)] - m.xyz[(size_t)(3 * v[0] + d)];
  // cofactors: inv = adj / det
  double cof[3][3];
  cof[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  cof[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  cof[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  cof[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  cof[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  cof[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  cof[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  cof[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  cof[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = (J[0][0] * cof[0][0] + J[0][1] * cof[0][1]) + J[0][2] * cof[0][2];
  const double ad = std::fabs(det);
  // J^-1 = cof^T / det, so (J^-1 J^-T)_{kl} = sum_d cof[d][k] cof[d][l] / det^2
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) {
      const double s = (cof[0][k] * cof[0][l] + cof[1][k] * cof[1][l]) + cof[2][k] * cof[2][l];
      g1[k][l] = s / ad;
      const double u = (J[0][k] * J[0][l] + J[1][k] * J[1][l]) + J[2][k] * J[2][l];
      g2[k][l] = u / ad;
    }
  return det;
}

// element entry sum_{k,l} G[k][l] I[i][j][k][l], (i, j) taken with i <= j so
// the element matrix is exactly symmetric
inline double p2_m1_entry(const double g[3][3], int i, int j) {
  if (i > j) std::swap(i, j);
  double acc = 0.0;
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) acc = acc + g[k][l] * p2t::kI1[i][j][k][l];
  return acc;
}
inline double p2_m2_entry(const double g[3][3], int i, int j) {
  if (i > j) std::swap(i, j);
  double acc = 0.0;
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) acc = acc + g[k][l] * p2t::kI2[i][j][k][l];
  return acc;
}

HostCSR p2_curl(const TetMesh& m, const P2Dofs& d);
HostCSR p2_div(const TetMesh& m, const P2Dofs& d);
HostCSR p2_mass(const TetMesh& m, const P2Dofs& d, int form);

}  // namespace sfeec_b200

// the sfeec_tetmesh handle (host_tet.cpp, host_p2.cpp); the P2 numbering is
// built on first use
struct sfeec_tetmesh {
  sfeec_b200::TetMesh m;
  mutable std::unique_ptr<sfeec_b200::P2Dofs> p2;
  const sfeec_b200::P2Dofs& p2dofs() const {
    if (!p2) {
      p2 = std::make_unique<sfeec_b200::P2Dofs>();
      p2->build(m);
    }
    return *p2;
  }
};
