// Host builders of the second-order P2^- system on the Kuhn tet mesh
// (BASELINE config 4; new code -- the reference's P2^- is 2-D only,
// form_space.cpp:41-166). Conventions follow the first-order builders
// (host_tet.cpp): rows assembled from their containing tets in ascending tet
// id, sums from 0.0, exact zeros dropped, element matrices exactly symmetric.
#include <cstring>
#include <memory>

#include "assembly.hpp"
#include "common.hpp"
#include "p2_mesh.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

namespace {

// first (lowest-id) tet containing face f
int64_t first_tet_of_face(const TetMesh& m, int64_t f) {
  int64_t v[3], tets[8];
  m.face_vertices(f, v);
  const int nt = m.containing_tets(v, 3, tets);
  require(nt >= 1, "P2 mesh: face without a tet");
  return tets[0];
}

// local index (0..nloc) of global DOF r in tet t's list
inline int local_index(const int32_t* d, int nloc, int32_t r) {
  for (int q = 0; q < nloc; ++q)
    if (d[q] == r) return q;
  return -1;
}

}  // namespace

// C: 2-form DOFs x 1-form DOFs, C(i, j) = DOF2_i(d phi_j) (exact rationals;
// a face row from its first tet -- the trace is single-valued)
HostCSR p2_curl(const TetMesh& m, const P2Dofs& d) {
  return assemble_rows(d.n2, d.n1, 20, [&](int64_t r, auto& acc) {
    const int kind = d.ks2[(size_t)r] & 1;
    const int64_t ent = d.ent2[(size_t)r];
    const int64_t t = kind == 0 ? first_tet_of_face(m, ent) : ent;
    int32_t d1[20], d2[15];
    d.local_dofs(m, t, d1, d2);
    const int p = local_index(d2, 15, (int32_t)r);
    for (int q = 0; q < 20; ++q)
      if (d1[q] >= 0 && p2t::kC[p][q] != 0.0) add_to(acc, d1[q], p2t::kC[p][q]);
  });
}

// D: 3-form DOFs (4 per tet, moments against l_0..l_3) x 2-form DOFs
HostCSR p2_div(const TetMesh& m, const P2Dofs& d) {
  return assemble_rows(d.n3, d.n2, 15, [&](int64_t r, auto& acc) {
    const int64_t t = r / 4;
    const int p = (int)(r % 4);
    int32_t d1[20], d2[15];
    d.local_dofs(m, t, d1, d2);
    for (int q = 0; q < 15; ++q)
      if (p2t::kD[p][q] != 0.0) add_to(acc, d2[q], p2t::kD[p][q]);
  });
}

HostCSR p2_mass(const TetMesh& m, const P2Dofs& d, int form) {
  // metric tensors per tet (and the orientation check of host_tet.cpp)
  std::vector<double> g((size_t)(9 * m.n_tets));
  bool bad = false;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < m.n_tets; ++t) {
    double g1[3][3], g2[3][3];
    const double det = p2_metric(m, t, g1, g2);
    const int p = (int)(t % 6);
    const double parity = (p == 0 || p == 3 || p == 4) ? 1.0 : -1.0;
    if (!(det * parity > 0)) bad = true;
    std::memcpy(&g[(size_t)(9 * t)], form == 1 ? &g1[0][0] : &g2[0][0], sizeof(double) * 9);
  }
  require(!bad, "tet mesh: non-positive tetrahedron volume (jitter too large)");
  const int nloc = form == 1 ? 20 : 15;
  const int64_t rows = form == 1 ? d.n1 : d.n2;
  return assemble_rows(rows, rows, form == 1 ? 96 : 32, [&](int64_t r, auto& acc) {
    const int8_t ks = form == 1 ? d.ks1[(size_t)r] : d.ks2[(size_t)r];
    const int64_t ent = form == 1 ? d.ent1[(size_t)r] : d.ent2[(size_t)r];
    int64_t tets[8];
    int nt;
    if (form == 2 && (ks & 1)) {  // tet-interior 2-form DOF
      tets[0] = ent;
      nt = 1;
    } else {
      int64_t v[3];
      int nv;
      if (form == 1 && (ks & 1) == 0) {
        m.edge_vertices(ent, v);
        nv = 2;
      } else {
        m.face_vertices(ent, v);
        nv = 3;
      }
      nt = m.containing_tets(v, nv, tets);
    }
    for (int a = 0; a < nt; ++a) {
      const int64_t t = tets[a];
      int32_t d1[20], d2[15];
      d.local_dofs(m, t, d1, d2);
      const int32_t* dl = form == 1 ? d1 : d2;
      const int p = local_index(dl, nloc, (int32_t)r);
      double gt[3][3];
      std::memcpy(&gt[0][0], &g[(size_t)(9 * t)], sizeof(double) * 9);
      for (int q = 0; q < nloc; ++q) {
        if (dl[q] < 0) continue;  // PEC boundary DOF
        add_to(acc, dl[q], form == 1 ? p2_m1_entry(gt, p, q) : p2_m2_entry(gt, p, q));
      }
    }
  });
}

}  // namespace sfeec_b200

using namespace sfeec_b200;

extern "C" {

int sfeec_tetmesh_p2_counts(const sfeec_tetmesh* h, int64_t* n1, int64_t* n2, int64_t* n3) {
  return guarded([&] {
    require(h, "null handle");
    const P2Dofs& d = h->p2dofs();
    if (n1) *n1 = d.n1;
    if (n2) *n2 = d.n2;
    if (n3) *n3 = d.n3;
  });
}

int sfeec_tetmesh_p2_operator(const sfeec_tetmesh* h, int which, sfeec_csr_owned* out) {
  return guarded([&] {
    require(h && out, "null argument");
    const P2Dofs& d = h->p2dofs();
    switch (which) {
      case 0: csr_to_owned(p2_curl(h->m, d), out); break;
      case 1: csr_to_owned(p2_mass(h->m, d, 1), out); break;
      case 2: csr_to_owned(p2_mass(h->m, d, 2), out); break;
      case 3: csr_to_owned(p2_div(h->m, d), out); break;
      default: throw Error(SFEEC_EINVAL, "unknown operator (0 C, 1 M1, 2 M2, 3 D)");
    }
  });
}

int sfeec_tetmesh_p2_dofs(const sfeec_tetmesh* h, int form, int64_t* entity, int8_t* kind_slot) {
  return guarded([&] {
    require(h, "null handle");
    require(form == 1 || form == 2, "P2 DOFs: form must be 1 or 2");
    const P2Dofs& d = h->p2dofs();
    const auto& ent = form == 1 ? d.ent1 : d.ent2;
    const auto& ks = form == 1 ? d.ks1 : d.ks2;
    if (entity) std::memcpy(entity, ent.data(), sizeof(int64_t) * ent.size());
    if (kind_slot) std::memcpy(kind_slot, ks.data(), ks.size());
  });
}

}  // extern "C"
