// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/src/{sparse,dynamics,yee,mesh_cubical}.cpp), compiled
// in place by oracle/Makefile into oracle/_ref/libsfeec_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// load it, as the checker and the reference CPU arm.
//
// Everything here is glue: it converts plain CSR buffers to the reference's
// sfeec::SparseOperator (proj/include/sfeec/sparse.hpp:14-33) and forwards to
//   SplitScheme ctor / flow_he / flow_ha / step / energy / gauss_residual /
//   cfl_number                      proj/src/dynamics.cpp:29-133
//   operator_from_triplets / transpose / spmv   proj/src/sparse.cpp:20-104
//   YeeGrid / yee_fdtd_step / yee_advance_b      proj/src/yee.cpp:9-74
//   generate_cubical_lattice                      proj/src/mesh_cubical.cpp:15-173
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sfeec/dynamics.hpp"
#include "sfeec/mesh.hpp"
#include "sfeec/sparse.hpp"
#include "sfeec/yee.hpp"

using namespace sfeec;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const InvalidParameter*>(&e)) return 1;
  return 2;
}

SparseOperator to_op(int rows, int cols, const int* rp, const int* ci, const double* v,
                     int symmetric) {
  SparseOperator m;
  m.rows = rows;
  m.cols = cols;
  m.symmetric = symmetric != 0;
  m.row_ptr.assign(rp, rp + rows + 1);
  int nnz = rp[rows];
  m.col_idx.assign(ci, ci + nnz);
  m.val.assign(v, v + nnz);
  return m;
}

struct Scheme {
  SplitScheme s;
};

void export_op(const SparseOperator& m, int* rp, int* ci, double* v) {
  if (rp) std::memcpy(rp, m.row_ptr.data(), sizeof(int) * m.row_ptr.size());
  if (ci) std::memcpy(ci, m.col_idx.data(), sizeof(int) * m.col_idx.size());
  if (v) std::memcpy(v, m.val.data(), sizeof(double) * m.val.size());
}

}  // namespace

extern "C" {

const char* sfeec_ref_last_error() { return g_err.c_str(); }

// ---- SplitScheme (dynamics.cpp:29-133) ------------------------------------
void* sfeec_ref_scheme_create(int kind, double dt, int qn, const int* qrp, const int* qci,
                              const double* qv, int cr, int cc, const int* crp,
                              const int* cci, const double* cv, const int* mrp,
                              const int* mci, const double* mv, double eps0, double mu0,
                              int dr, const int* drp, const int* dci, const double* dv,
                              int warn_cfl) {
  try {
    SparseOperator q = to_op(qn, qn, qrp, qci, qv, 0);
    SparseOperator c = to_op(cr, cc, crp, cci, cv, 0);
    SparseOperator m2 = to_op(cr, cr, mrp, mci, mv, 1);
    std::optional<SparseOperator> div;
    if (drp) div = to_op(dr, cr, drp, dci, dv, 0);
    UnitSystem u{eps0, mu0};
    auto* h = new Scheme{SplitScheme(kind ? SplitKind::Strang : SplitKind::LieTrotter, dt,
                                     q, c, m2, u, div ? &*div : nullptr, warn_cfl != 0)};
    return h;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void sfeec_ref_scheme_destroy(void* h) { delete static_cast<Scheme*>(h); }

int sfeec_ref_scheme_qsym_nnz(void* h) { return static_cast<Scheme*>(h)->s.q_sym().nnz(); }

void sfeec_ref_scheme_qsym(void* h, int* rp, int* ci, double* v) {
  export_op(static_cast<Scheme*>(h)->s.q_sym(), rp, ci, v);
}

void sfeec_ref_scheme_curl_t(void* h, int* rp, int* ci, double* v) {
  export_op(static_cast<Scheme*>(h)->s.curl_t(), rp, ci, v);
}

static FieldState make(int form, const double* first, int nf, const double* e, int ne,
                       double t) {
  return make_state(form ? Formulation::BE : Formulation::AE,
                    std::vector<double>(first, first + nf), std::vector<double>(e, e + ne),
                    t);
}

// nsteps x SplitScheme::step, in place; optional energy history after each step
int sfeec_ref_scheme_steps(void* hp, int form, double* first, int nf, double* e, int ne,
                           double* time, int nsteps, double* energy_hist,
                           double* seconds) {
  try {
    auto& s = static_cast<Scheme*>(hp)->s;
    FieldState st = make(form, first, nf, e, ne, *time);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < nsteps; ++i) {
      st = s.step(st);
      if (energy_hist) energy_hist[i] = s.energy(st);
    }
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(first, st.first.data(), sizeof(double) * (size_t)nf);
    std::memcpy(e, st.e.data(), sizeof(double) * (size_t)ne);
    *time = st.time;
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int sfeec_ref_scheme_flow(void* hp, int which, int form, double* first, int nf, double* e,
                          int ne, double dt) {
  try {
    auto& s = static_cast<Scheme*>(hp)->s;
    FieldState st = make(form, first, nf, e, ne, 0.0);
    if (which == 0)
      s.flow_he(st, dt);
    else
      s.flow_ha(st, dt);
    std::memcpy(first, st.first.data(), sizeof(double) * (size_t)nf);
    std::memcpy(e, st.e.data(), sizeof(double) * (size_t)ne);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int sfeec_ref_scheme_energy(void* hp, int form, const double* first, int nf, const double* e,
                            int ne, double* out) {
  try {
    *out = static_cast<Scheme*>(hp)->s.energy(make(form, first, nf, e, ne, 0.0));
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int sfeec_ref_scheme_gauss(void* hp, int form, const double* first, int nf, const double* e,
                           int ne, double* out) {
  try {
    *out = static_cast<Scheme*>(hp)->s.gauss_residual(make(form, first, nf, e, ne, 0.0));
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int sfeec_ref_scheme_cfl(void* hp, double* out) {
  try {
    *out = static_cast<Scheme*>(hp)->s.cfl_number();
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// ---- sparse.cpp -----------------------------------------------------------
void sfeec_ref_spmv(int rows, int cols, const int* rp, const int* ci, const double* v,
                    const double* x, double* y) {
  SparseOperator a = to_op(rows, cols, rp, ci, v, 0);
  spmv(a, x, y);
}

// operator_from_triplets; returns nnz, fills outputs when non-null (call twice)
int sfeec_ref_from_triplets(int rows, int cols, int n, const int* r, const int* c,
                            const double* v, int* rp, int* ci, double* val) {
  try {
    std::vector<Triplet> t((size_t)n);
    for (int i = 0; i < n; ++i) t[(size_t)i] = {r[i], c[i], v[i]};
    SparseOperator m = operator_from_triplets(rows, cols, std::move(t));
    export_op(m, rp, ci, val);
    return m.nnz();
  } catch (const std::exception& ex) {
    fail(ex);
    return -1;
  }
}

void sfeec_ref_transpose(int rows, int cols, const int* rp, const int* ci, const double* v,
                         int* trp, int* tci, double* tv) {
  export_op(transpose(to_op(rows, cols, rp, ci, v, 0)), trp, tci, tv);
}

// ---- cubical lattice + Q1 curl (mesh_cubical.cpp:15-173; entry rule of
// operators.cpp:37 = sign * |edge| / |face|, i.e. +-1/spacing) ---------------
int sfeec_ref_cubical_curl(int nx, int ny, int nz, double dx, double dy, double dz,
                           int* rp, int* ci, double* v) {
  try {
    PeriodicMesh m = generate_cubical_lattice(nx, ny, nz, dx, dy, dz);
    const int N = nx * ny * nz;
    // face_volume (operators.cpp:13-27) from the unwrapped face_coords
    auto fc = [&](int p, int id) -> const std::vector<Vec3>& {
      return m.face_coords[(size_t)p][(size_t)id];
    };
    std::vector<Triplet> tri;
    for (int f = 0; f < 3 * N; ++f) {
      const auto& xs = fc(2, f);
      double vol_f = (xs[1] - xs[0]).norm() * (xs[3] - xs[0]).norm();
      for (auto [edge, sign] : m.boundary[2][(size_t)f]) {
        const auto& es = fc(1, edge);
        double v = sign;
        v *= (es[1] - es[0]).norm() / vol_f;
        tri.push_back({f, edge, v});
      }
    }
    SparseOperator c = operator_from_triplets(3 * N, 3 * N, std::move(tri));
    export_op(c, rp, ci, v);
    return c.nnz();
  } catch (const std::exception& ex) {
    return -fail(ex);
  }
}

// ---- Yee FDTD oracle (yee.cpp:9-74) ---------------------------------------
void* sfeec_ref_yee_create(int nx, int ny, int nz, double dx, double dy, double dz) {
  return new YeeGrid(nx, ny, nz, dx, dy, dz);
}
void sfeec_ref_yee_destroy(void* g) { delete static_cast<YeeGrid*>(g); }
// which: 0 = e, 1 = b; component-major arrays of 3*nx*ny*nz
void sfeec_ref_yee_set(void* gp, int which, const double* x) {
  auto* g = static_cast<YeeGrid*>(gp);
  size_t nc = g->e[0].size();
  for (int a = 0; a < 3; ++a) {
    auto& dst = which ? g->b[a] : g->e[a];
    std::memcpy(dst.data(), x + a * nc, sizeof(double) * nc);
  }
}
void sfeec_ref_yee_get(void* gp, int which, double* x) {
  auto* g = static_cast<YeeGrid*>(gp);
  size_t nc = g->e[0].size();
  for (int a = 0; a < 3; ++a) {
    auto& src = which ? g->b[a] : g->e[a];
    std::memcpy(x + a * nc, src.data(), sizeof(double) * nc);
  }
}
void sfeec_ref_yee_step(void* gp, double dt, double eps0, double mu0, int nsteps) {
  for (int i = 0; i < nsteps; ++i)
    yee_fdtd_step(*static_cast<YeeGrid*>(gp), dt, UnitSystem{eps0, mu0});
}
void sfeec_ref_yee_advance_b(void* gp, double dt) {
  yee_advance_b(*static_cast<YeeGrid*>(gp), dt);
}

}  // extern "C"
