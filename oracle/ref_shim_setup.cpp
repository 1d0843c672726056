// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" glue over the UNMODIFIED reference setup code, compiled in place
// by oracle/Makefile (target refsetup) into oracle/_ref/libsfeec_ref_setup.so
// together with every reference source file (proj/src/*.cpp). The reference's
// form_space.cpp / operators.cpp / spai.cpp include Eigen, which this image
// lacks; they compile against the Eigen-subset stand-in under
// oracle/eigen_shim. The glue forwards to
//   make_pattern                 proj/src/spai.cpp:31-72
//   spai_approximate_inverse     proj/src/spai.cpp:127-286
//   build_space (Q1)             proj/src/form_space.cpp:177-192
//   derivative_matrix            proj/src/operators.cpp:111-118
//   mass_matrix                  proj/src/operators.cpp:133-179
// so the product's SPAI and cubical operators are checked against the
// reference's own code, not only against restatements of it.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sfeec/mesh.hpp"
#include "sfeec/operators.hpp"
#include "sfeec/spai.hpp"

using namespace sfeec;

namespace {

thread_local std::string g_err;

struct OpHandle {
  SparseOperator m;
  double report[4] = {0, 0, 0, 0};
};

SparseOperator to_op(int rows, int cols, const int* rp, const int* ci, const double* v,
                     int symmetric) {
  SparseOperator m;
  m.rows = rows;
  m.cols = cols;
  m.symmetric = symmetric != 0;
  m.row_ptr.assign(rp, rp + rows + 1);
  m.col_idx.assign(ci, ci + rp[rows]);
  m.val.assign(v, v + rp[rows]);
  return m;
}

PatternKind kind_of(int k) {
  switch (k) {
    case 0: return PatternKind::Diagonal;
    case 1: return PatternKind::M1;
    case 2: return PatternKind::M1Squared;
    case 3: return PatternKind::Dense;
  }
  throw InvalidParameter("unknown pattern kind");
}

}  // namespace

extern "C" {

const char* sfeec_refs_last_error() { return g_err.c_str(); }

int sfeec_refs_op_rows(void* h) { return static_cast<OpHandle*>(h)->m.rows; }
int sfeec_refs_op_cols(void* h) { return static_cast<OpHandle*>(h)->m.cols; }
int sfeec_refs_op_nnz(void* h) { return static_cast<OpHandle*>(h)->m.nnz(); }
void sfeec_refs_op_export(void* h, int* rp, int* ci, double* v, double* report) {
  const OpHandle& o = *static_cast<OpHandle*>(h);
  std::memcpy(rp, o.m.row_ptr.data(), sizeof(int) * o.m.row_ptr.size());
  std::memcpy(ci, o.m.col_idx.data(), sizeof(int) * o.m.col_idx.size());
  std::memcpy(v, o.m.val.data(), sizeof(double) * o.m.val.size());
  if (report) std::memcpy(report, o.report, sizeof(o.report));
}
void sfeec_refs_op_destroy(void* h) { delete static_cast<OpHandle*>(h); }

// make_pattern: row l of the result = the index set I_l (unit values)
void* sfeec_refs_pattern(int n, const int* rp, const int* ci, const double* v, int kind) {
  try {
    SparsityPattern p = make_pattern(to_op(n, n, rp, ci, v, 1), kind_of(kind));
    auto h = new OpHandle;
    h->m.rows = h->m.cols = n;
    h->m.row_ptr.assign((size_t)n + 1, 0);
    for (int l = 0; l < n; ++l) {
      h->m.row_ptr[(size_t)l + 1] = h->m.row_ptr[(size_t)l] + (int)p.cols[(size_t)l].size();
      h->m.col_idx.insert(h->m.col_idx.end(), p.cols[(size_t)l].begin(), p.cols[(size_t)l].end());
    }
    h->m.val.assign(h->m.col_idx.size(), 1.0);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// spai_approximate_inverse on make_pattern(m, kind); report = {Frobenius
// residual, average nnz per row, max column residual, fallback columns}
void* sfeec_refs_spai(int n, const int* rp, const int* ci, const double* v, int kind,
                      int use_cg) {
  try {
    SparseOperator m = to_op(n, n, rp, ci, v, 1);
    SpaiOptions opts;
    opts.use_cg = use_cg != 0;
    auto [q, rep] = spai_approximate_inverse(m, make_pattern(m, kind_of(kind)), opts);
    auto h = new OpHandle;
    h->m = std::move(q);
    h->report[0] = rep.frobenius_residual;
    h->report[1] = rep.avg_nnz_per_row;
    h->report[2] = rep.max_column_residual;
    h->report[3] = (double)rep.fallback_columns;
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Q1 operators of the reference's periodic cubical lattice: which = 0 the
// curl (derivative_matrix of 1-forms to 2-forms), 1 M1, 2 M2, 3 the
// divergence (2-forms to 3-forms)
void* sfeec_refs_cubical(int nx, int ny, int nz, double dx, double dy, double dz, int which) {
  try {
    PeriodicMesh mesh = generate_cubical_lattice(nx, ny, nz, dx, dy, dz);
    auto space = [&](int p) {
      FormSpace s = build_space(mesh, Family::Q1, p);
      s.mesh = &mesh;
      return s;
    };
    auto h = new OpHandle;
    switch (which) {
      case 0: h->m = derivative_matrix(space(1), space(2)); break;
      case 1: h->m = mass_matrix(space(1)); break;
      case 2: h->m = mass_matrix(space(2)); break;
      case 3: h->m = derivative_matrix(space(2), space(3)); break;
      default: delete h; throw InvalidParameter("unknown operator");
    }
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // extern "C"
