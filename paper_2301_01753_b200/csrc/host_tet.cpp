// Host setup for first-order Whitney SFEEC on a jittered Kuhn/Freudenthal
// tetrahedral mesh of the unit cube with PEC walls (BASELINE configs 1, 3, 5).
// None of this exists in the reference (its meshes are 2-D
// triangulations and periodic cubes); it follows the reference's conventions:
//   * simplices oriented by ascending global vertex id (SPEC.md:78,
//     mesh_simplicial.cpp:16-38), boundary = sum_i (-1)^i [.., v_i omitted, ..];
//   * integral DOFs, so d is the signed incidence (+-1) as in
//     derivative_q1_p1 for P1 (operators.cpp:29-42);
//   * mass matrices assembled cell by cell with an exact symmetric mirror and
//     duplicates summed in ascending cell order, exact zeros dropped
//     (operators.cpp:133-179 + sparse.cpp:20-61 semantics);
//   * SPAI per column on the normal equations Gram = M^2(I_l, I_l),
//     rhs = M(l, I_l), accept if min pivot > 1e-12 trace else the
//     eigenvalue-thresholded minimum-norm solve (spai.cpp:127-286).
// The full numbering/geometry contract is written out in DESIGN.md and
// restated independently in oracle/tetmesh_oracle.py.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>

#include "assembly.hpp"
#include "common.hpp"
#include "p2_mesh.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {


HostCSR tet_curl(const TetMesh& m) {
  // face [v0,v1,v2]: +[v1,v2] -[v0,v2] +[v0,v1]
  return assemble_rows(m.n_faces, m.n_edges, 3, [&](int64_t f, auto& acc) {
    int64_t v[3];
    m.face_vertices(f, v);
    const int64_t pr[3][2] = {{v[1], v[2]}, {v[0], v[2]}, {v[0], v[1]}};
    const double sg[3] = {1.0, -1.0, 1.0};
    for (int t = 0; t < 3; ++t) {
      int32_t e = m.edge_of(pr[t][0], pr[t][1]);
      if (e >= 0) add_to(acc, e, sg[t]);
    }
  });
}

HostCSR tet_div(const TetMesh& m) {
  // tet [v0..v3]: +[v1v2v3] -[v0v2v3] +[v0v1v3] -[v0v1v2]
  return assemble_rows(m.n_tets, m.n_faces, 4, [&](int64_t t, auto& acc) {
    int64_t v[4];
    m.tet_vertices(t, v);
    for (int f = 0; f < 4; ++f) {
      int32_t id = m.face_of(v[kLF[f][0]], v[kLF[f][1]], v[kLF[f][2]]);
      add_to(acc, id, (f % 2 == 0) ? 1.0 : -1.0);
    }
  });
}

HostCSR tet_mass(const TetMesh& m, int form) {
  const int64_t rows = form == 1 ? m.n_edges : m.n_faces;
  // precompute element matrices (upper triangles) in parallel
  const int nl = form == 1 ? 6 : 4;
  const int nu = nl * (nl + 1) / 2;
  std::vector<double> loc((size_t)(m.n_tets * nu));
  std::vector<int32_t> ids((size_t)(m.n_tets * nl));
  bool bad = false;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < m.n_tets; ++t) {
    double m1[6][6], m2[4][4];
    double vol6 = m.element(t, m1, m2);
    // the jittered tet must keep the orientation of its Kuhn parent
    // (permutation parity: 0,3,4 even; 1,2,5 odd)
    const int p = (int)(t % 6);
    const double parity = (p == 0 || p == 3 || p == 4) ? 1.0 : -1.0;
    if (!(vol6 * parity > 0)) bad = true;
    int u = 0;
    for (int p = 0; p < nl; ++p)
      for (int q = p; q < nl; ++q) loc[(size_t)(t * nu + u++)] = form == 1 ? m1[p][q] : m2[p][q];
    int64_t v[4];
    m.tet_vertices(t, v);
    for (int p = 0; p < nl; ++p)
      ids[(size_t)(t * nl + p)] = form == 1 ? m.edge_of(v[kLE[p][0]], v[kLE[p][1]])
                                            : m.face_of(v[kLF[p][0]], v[kLF[p][1]], v[kLF[p][2]]);
  }
  require(!bad, "tet mesh: non-positive tetrahedron volume (jitter too large)");
  auto upper = [nl](int p, int q) {
    if (p > q) std::swap(p, q);
    return p * nl - p * (p - 1) / 2 + (q - p);
  };
  return assemble_rows(rows, rows, form == 1 ? 40 : 8, [&](int64_t r, auto& acc) {
    int64_t vs[3];
    int nvs;
    if (form == 1) {
      m.edge_vertices(r, vs);
      nvs = 2;
    } else {
      m.face_vertices(r, vs);
      nvs = 3;
    }
    int64_t tets[8];
    int nt = m.containing_tets(vs, nvs, tets);
    for (int a = 0; a < nt; ++a) {
      const int64_t t = tets[a];
      int p = -1;
      for (int q = 0; q < nl; ++q)
        if (ids[(size_t)(t * nl + q)] == (int32_t)r) p = q;
      for (int q = 0; q < nl; ++q) {
        int32_t c = ids[(size_t)(t * nl + q)];
        if (c < 0) continue;  // boundary edge (PEC)
        add_to(acc, c, loc[(size_t)(t * nu + upper(p, q))]);
      }
    }
  });
}

// ---- SPAI (spai.cpp:31-72, 127-286) ---------------------------------------
struct SpaiReport {
  double frobenius_residual = 0, avg_nnz_per_row = 0, max_column_residual = 0;
  int64_t fallback_columns = 0;
};

// pattern kinds: 0 diagonal, 1 S(M1), 2 S(M1^2)
std::vector<std::vector<int32_t>> make_pattern(const HostCSR& m, int kind) {
  std::vector<std::vector<int32_t>> p((size_t)m.rows);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < m.rows; ++i) {
    auto& out = p[(size_t)i];
    if (kind == 0) {
      out = {(int32_t)i};
    } else if (kind == 1) {
      out.assign(m.col_idx.begin() + m.row_ptr[(size_t)i], m.col_idx.begin() + m.row_ptr[(size_t)i + 1]);
    } else {
      for (int64_t k = m.row_ptr[(size_t)i]; k < m.row_ptr[(size_t)i + 1]; ++k) {
        int32_t j = m.col_idx[(size_t)k];
        out.insert(out.end(), m.col_idx.begin() + m.row_ptr[(size_t)j],
                   m.col_idx.begin() + m.row_ptr[(size_t)j + 1]);
      }
      std::sort(out.begin(), out.end());
      out.erase(std::unique(out.begin(), out.end()), out.end());
    }
  }
  return p;
}

namespace {

// (M^2)(i, j) = sum_k M(i,k) M(k,j), k ascending (sparse_square, spai.cpp:77-123)
inline double sq_entry(const HostCSR& m, int32_t i, int32_t j) {
  int64_t a = m.row_ptr[(size_t)i], ae = m.row_ptr[(size_t)i + 1];
  int64_t b = m.row_ptr[(size_t)j], be = m.row_ptr[(size_t)j + 1];
  double s = 0.0;
  while (a < ae && b < be) {
    int32_t ca = m.col_idx[(size_t)a], cb = m.col_idx[(size_t)b];
    if (ca == cb) {
      s = s + m.val[(size_t)a] * m.val[(size_t)b];
      ++a;
      ++b;
    } else if (ca < cb) {
      ++a;
    } else {
      ++b;
    }
  }
  return s;
}

inline double entry(const HostCSR& m, int32_t r, int32_t c) {
  auto b = m.col_idx.begin() + m.row_ptr[(size_t)r], e = m.col_idx.begin() + m.row_ptr[(size_t)r + 1];
  auto it = std::lower_bound(b, e, c);
  return (it != e && *it == c) ? m.val[(size_t)(it - m.col_idx.begin())] : 0.0;
}

// cyclic Jacobi eigen-decomposition of a symmetric k x k matrix (row-major)
void jacobi_eigen(int k, std::vector<double>& a, std::vector<double>& v) {
  v.assign((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) v[(size_t)i * k + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < k; ++i)
      for (int j = i + 1; j < k; ++j) off += a[(size_t)i * k + j] * a[(size_t)i * k + j];
    if (off < 1e-300) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        double apq = a[(size_t)p * k + q];
        if (std::fabs(apq) < 1e-300) continue;
        double app = a[(size_t)p * k + p], aqq = a[(size_t)q * k + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < k; ++r) {
          double arp = a[(size_t)r * k + p], arq = a[(size_t)r * k + q];
          a[(size_t)r * k + p] = c * arp - s * arq;
          a[(size_t)r * k + q] = s * arp + c * arq;
        }
        for (int r = 0; r < k; ++r) {
          double apr = a[(size_t)p * k + r], aqr = a[(size_t)q * k + r];
          a[(size_t)p * k + r] = c * apr - s * aqr;
          a[(size_t)q * k + r] = s * apr + c * aqr;
        }
        for (int r = 0; r < k; ++r) {
          double vrp = v[(size_t)r * k + p], vrq = v[(size_t)r * k + q];
          v[(size_t)r * k + p] = c * vrp - s * vrq;
          v[(size_t)r * k + q] = s * vrp + c * vrq;
        }
      }
  }
}

}  // namespace

HostCSR spai(const HostCSR& m, const std::vector<std::vector<int32_t>>& pat, SpaiReport* rep) {
  require(m.rows == m.cols, "spai: square operator required");
  require((int64_t)pat.size() == m.rows, "spai: pattern dimension mismatch");
  for (const auto& c : pat) require(!c.empty(), "spai: empty pattern column");
  const int64_t n = m.rows;
  std::vector<std::vector<double>> colvals((size_t)n);
  std::vector<double> res2((size_t)n, 0.0);
  std::vector<char> fb((size_t)n, 0);
  const double eig_cut = 1e-12;
#pragma omp parallel
  {
    std::vector<double> gram, L, v, resid((size_t)n, 0.0);
    std::vector<int32_t> touched;
#pragma omp for schedule(dynamic, 256)
    for (int64_t l = 0; l < n; ++l) {
      const auto& idx = pat[(size_t)l];
      const int k = (int)idx.size();
      gram.assign((size_t)k * k, 0.0);
      double trace = 0;
      for (int a = 0; a < k; ++a)
        for (int b = a; b < k; ++b) {
          double g = sq_entry(m, idx[(size_t)a], idx[(size_t)b]);
          gram[(size_t)a * k + b] = g;
          gram[(size_t)b * k + a] = g;
        }
      for (int a = 0; a < k; ++a) trace += gram[(size_t)a * k + a];
      std::vector<double> rhs((size_t)k), q((size_t)k);
      for (int a = 0; a < k; ++a) rhs[(size_t)a] = entry(m, (int32_t)l, idx[(size_t)a]);
      // Cholesky G = L L^T; pivots d_a = L_aa^2 play the role of LDLT's D
      L = gram;
      bool ok = true;
      double dmin = INFINITY;
      for (int j = 0; j < k && ok; ++j) {
        double d = L[(size_t)j * k + j];
        for (int p = 0; p < j; ++p) d -= L[(size_t)j * k + p] * L[(size_t)j * k + p];
        if (!(d > 0)) {
          ok = false;
          break;
        }
        dmin = std::min(dmin, d);
        double ljj = std::sqrt(d);
        L[(size_t)j * k + j] = ljj;
        for (int i = j + 1; i < k; ++i) {
          double s = L[(size_t)i * k + j];
          for (int p = 0; p < j; ++p) s -= L[(size_t)i * k + p] * L[(size_t)j * k + p];
          L[(size_t)i * k + j] = s / ljj;
        }
      }
      if (ok && dmin > eig_cut * trace) {
        for (int i = 0; i < k; ++i) {
          double s = rhs[(size_t)i];
          for (int p = 0; p < i; ++p) s -= L[(size_t)i * k + p] * q[(size_t)p];
          q[(size_t)i] = s / L[(size_t)i * k + i];
        }
        for (int i = k - 1; i >= 0; --i) {
          double s = q[(size_t)i];
          for (int p = i + 1; p < k; ++p) s -= L[(size_t)p * k + i] * q[(size_t)p];
          q[(size_t)i] = s / L[(size_t)i * k + i];
        }
        for (double x : q)
          if (!std::isfinite(x)) ok = false;
      } else {
        ok = false;
      }
      if (!ok) {  // minimum-norm solve with eigenvalue thresholding (spai.cpp:222-231)
        std::vector<double> a = gram;
        jacobi_eigen(k, a, v);
        const double cut = eig_cut * trace;
        std::fill(q.begin(), q.end(), 0.0);
        for (int e = 0; e < k; ++e) {
          double w = a[(size_t)e * k + e];
          if (!(w > cut)) continue;
          double y = 0;
          for (int i = 0; i < k; ++i) y += v[(size_t)i * k + e] * rhs[(size_t)i];
          y /= w;
          for (int i = 0; i < k; ++i) q[(size_t)i] += v[(size_t)i * k + e] * y;
        }
        fb[(size_t)l] = 1;
      }
      colvals[(size_t)l] = q;
      // true residual ||M q - e_l||^2 by sparse scatter (spai.cpp:237-253)
      touched.clear();
      for (int a = 0; a < k; ++a) {
        int32_t r = idx[(size_t)a];
        for (int64_t t = m.row_ptr[(size_t)r]; t < m.row_ptr[(size_t)r + 1]; ++t) {
          int32_t c = m.col_idx[(size_t)t];
          if (resid[(size_t)c] == 0.0) touched.push_back(c);
          resid[(size_t)c] += m.val[(size_t)t] * q[(size_t)a];
        }
      }
      if (resid[(size_t)l] == 0.0) touched.push_back((int32_t)l);
      resid[(size_t)l] -= 1.0;
      double r2 = 0;
      for (int32_t t : touched) {
        r2 += resid[(size_t)t] * resid[(size_t)t];
        resid[(size_t)t] = 0.0;
      }
      res2[(size_t)l] = r2;
    }
  }
  // assemble Q by rows: Q(idx[a], l) = q_l[a]  (spai.cpp:258-268)
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  for (int64_t l = 0; l < n; ++l)
    for (int32_t r : pat[(size_t)l]) cnt[(size_t)r + 1]++;
  HostCSR q;
  q.rows = q.cols = n;
  q.row_ptr.assign((size_t)n + 1, 0);
  for (int64_t r = 0; r < n; ++r) cnt[(size_t)r + 1] += cnt[(size_t)r];
  std::vector<int32_t> tc((size_t)cnt[(size_t)n]);
  std::vector<double> tv((size_t)cnt[(size_t)n]);
  {
    std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
    for (int64_t l = 0; l < n; ++l) {  // ascending l -> columns sorted within each row
      const auto& idx = pat[(size_t)l];
      for (size_t a = 0; a < idx.size(); ++a) {
        int64_t s = cur[(size_t)idx[a]]++;
        tc[(size_t)s] = (int32_t)l;
        tv[(size_t)s] = colvals[(size_t)l][a];
      }
    }
  }
  for (int64_t r = 0; r < n; ++r) {
    int64_t w = 0;
    for (int64_t s = cnt[(size_t)r]; s < cnt[(size_t)r + 1]; ++s)
      if (tv[(size_t)s] != 0.0) ++w;
    q.row_ptr[(size_t)r + 1] = q.row_ptr[(size_t)r] + w;
  }
  q.col_idx.reserve((size_t)q.row_ptr[(size_t)n]);
  q.val.reserve((size_t)q.row_ptr[(size_t)n]);
  for (int64_t s = 0; s < cnt[(size_t)n]; ++s)
    if (tv[(size_t)s] != 0.0) {
      q.col_idx.push_back(tc[(size_t)s]);
      q.val.push_back(tv[(size_t)s]);
    }
  if (rep) {
    double fro = 0, mx = 0;
    int64_t nfb = 0;
    for (int64_t l = 0; l < n; ++l) {
      fro += res2[(size_t)l];
      mx = std::max(mx, res2[(size_t)l]);
      nfb += fb[(size_t)l];
    }
    rep->frobenius_residual = std::sqrt(fro);
    rep->max_column_residual = std::sqrt(mx);
    rep->avg_nnz_per_row = (double)q.nnz() / (double)n;
    rep->fallback_columns = nfb;
  }
  return q;
}

}  // namespace sfeec_b200

using namespace sfeec_b200;


extern "C" {

int sfeec_tetmesh_create(int n, double jitter, uint64_t seed, sfeec_tetmesh** out) {
  return guarded([&] {
    require(out != nullptr, "null out");
    auto h = std::make_unique<sfeec_tetmesh>();
    h->m.build(n, jitter, seed);
    *out = h.release();
  });
}

int sfeec_tetmesh_create_slab(int n, int nzg, int k0, int k1, double jitter, uint64_t seed,
                              sfeec_tetmesh** out) {
  return guarded([&] {
    require(out != nullptr, "null out");
    auto h = std::make_unique<sfeec_tetmesh>();
    h->m.build_slab(n, nzg, k0, k1, jitter, seed);
    *out = h.release();
  });
}

void sfeec_tetmesh_destroy(sfeec_tetmesh* h) { delete h; }

int sfeec_tetmesh_counts(const sfeec_tetmesh* h, int64_t* n_vertices, int64_t* n_edges,
                         int64_t* n_faces, int64_t* n_tets) {
  return guarded([&] {
    require(h, "null handle");
    if (n_vertices) *n_vertices = h->m.nv;
    if (n_edges) *n_edges = h->m.n_edges;
    if (n_faces) *n_faces = h->m.n_faces;
    if (n_tets) *n_tets = h->m.n_tets;
  });
}

// Canonical projection of a sum of Gaussian pulses onto the DOF edges
// [e0, e1): a_e = int_e A . dx with A = sum_k exp(-|x - x0_k|^2 / (2 sigma^2))
// p_k, 3-point Gauss-Legendre along the edge (the P1 integral DOF of the
// reference form_space.cpp:410-429). The pulse parameters come from
// inputs.pulse_params; inputs.pulse_one_form is the numpy statement of the
// same sum (tests compare the two).
int sfeec_tetmesh_pulse(const sfeec_tetmesh* h, int npulses, const double* x0, const double* p,
                        double sigma, int64_t e0, int64_t e1, double* out) {
  return guarded([&] {
    require(h && out && (npulses == 0 || (x0 && p)), "null argument");
    const TetMesh& m = h->m;
    require(e0 >= 0 && e0 <= e1 && e1 <= m.n_edges, "pulse: edge range out of bounds");
    const double q = std::sqrt(0.6);
    const double gs[3] = {0.5 - 0.5 * q, 0.5, 0.5 + 0.5 * q};
    const double gw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
    const double inv = 1.0 / (2.0 * sigma * sigma);
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      int64_t v[2];
      m.edge_vertices(e, v);
      double xa[3], d[3];
      for (int c = 0; c < 3; ++c) {
        xa[c] = m.xyz[(size_t)(3 * v[0] + c)];
        d[c] = m.xyz[(size_t)(3 * v[1] + c)] - xa[c];
      }
      double a = 0.0;
      for (int k = 0; k < npulses; ++k) {
        const double* c0 = x0 + 3 * k;
        const double* pk = p + 3 * k;
        const double tang = (d[0] * pk[0] + d[1] * pk[1]) + d[2] * pk[2];
        for (int s = 0; s < 3; ++s) {
          double r2 = 0.0;
          for (int c = 0; c < 3; ++c) {
            const double x = (xa[c] + gs[s] * d[c]) - c0[c];
            r2 += x * x;
          }
          a += gw[s] * std::exp(-r2 * inv) * tang;
        }
      }
      out[e - e0] = a;
    }
  });
}

int sfeec_tetmesh_geometry(const sfeec_tetmesh* h, double* xyz, int64_t* edge_vertices,
                           int64_t* face_vertices, int64_t* tet_vertices) {
  return guarded([&] {
    require(h, "null handle");
    const TetMesh& m = h->m;
    if (xyz) std::memcpy(xyz, m.xyz.data(), sizeof(double) * m.xyz.size());
    if (edge_vertices) {
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < m.n_edges; ++e) m.edge_vertices(e, edge_vertices + 2 * e);
    }
    if (face_vertices) {
#pragma omp parallel for schedule(static)
      for (int64_t f = 0; f < m.n_faces; ++f) m.face_vertices(f, face_vertices + 3 * f);
    }
    if (tet_vertices) {
#pragma omp parallel for schedule(static)
      for (int64_t t = 0; t < m.n_tets; ++t) m.tet_vertices(t, tet_vertices + 4 * t);
    }
  });
}

int sfeec_tetmesh_operator(const sfeec_tetmesh* h, int which, sfeec_csr_owned* out) {
  return guarded([&] {
    require(h && out, "null argument");
    switch (which) {
      case 0: csr_to_owned(tet_curl(h->m), out); break;
      case 1: csr_to_owned(tet_mass(h->m, 1), out); break;
      case 2: csr_to_owned(tet_mass(h->m, 2), out); break;
      case 3: csr_to_owned(tet_div(h->m), out); break;
      default: throw Error(SFEEC_EINVAL, "unknown operator (0 C, 1 M1, 2 M2, 3 D)");
    }
  });
}

int sfeec_make_pattern(const sfeec_csr* m, int kind, sfeec_csr_owned* out) {
  return guarded([&] {
    require(m && out, "null argument");
    csr_validate(*m, "M");
    require(m->rows == m->cols, "make_pattern: square operator");
    require(kind >= 0 && kind <= 2, "make_pattern: kind must be 0 (diagonal), 1 (M1), 2 (M1^2)");
    HostCSR hm = csr_from_view(*m);
    auto p = make_pattern(hm, kind);
    HostCSR pc;
    pc.rows = pc.cols = hm.rows;
    pc.row_ptr.assign((size_t)hm.rows + 1, 0);
    for (int64_t i = 0; i < hm.rows; ++i)
      pc.row_ptr[(size_t)i + 1] = pc.row_ptr[(size_t)i] + (int64_t)p[(size_t)i].size();
    for (auto& r : p) pc.col_idx.insert(pc.col_idx.end(), r.begin(), r.end());
    pc.val.assign(pc.col_idx.size(), 1.0);
    csr_to_owned(std::move(pc), out);
  });
}

int sfeec_spai(const sfeec_csr* m, int kind, sfeec_csr_owned* q, double* report) {
  return guarded([&] {
    require(m && q, "null argument");
    csr_validate(*m, "M");
    require(m->rows == m->cols, "spai: square operator required");
    require(kind >= 0 && kind <= 2, "spai: pattern kind must be 0, 1 or 2");
    HostCSR hm = csr_from_view(*m);
    SpaiReport rep;
    HostCSR hq = spai(hm, make_pattern(hm, kind), &rep);
    if (report) {
      report[0] = rep.frobenius_residual;
      report[1] = rep.avg_nnz_per_row;
      report[2] = rep.max_column_residual;
      report[3] = (double)rep.fallback_columns;
    }
    csr_to_owned(std::move(hq), q);
  });
}

}  // extern "C"
