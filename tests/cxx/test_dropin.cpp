// C++ drop-in test: code written against the reference API
// (/root/reference/proj/include/sfeec/{sparse,dynamics}.hpp) compiled against
// include/sfeec/ and linked to libsfeec_b200.so. Restates reference tests
// (test_dynamics.cpp:67-148, 252-311) and checks the device step against the
// plain-C oracle (oracle/sfeec_oracle.c, the test-only checker).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "sfeec/dynamics.hpp"
#include "sfeec_b200.h"

extern "C" {
#include "../../oracle/sfeec_oracle.h"
}

using namespace sfeec;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static SparseOperator from_owned(sfeec_csr_owned& m) {
  SparseOperator s;
  s.rows = (int)m.rows;
  s.cols = (int)m.cols;
  s.row_ptr.assign(m.row_ptr, m.row_ptr + m.rows + 1);
  s.col_idx.assign(m.col_idx, m.col_idx + m.nnz);
  s.val.assign(m.val, m.val + m.nnz);
  sfeec_csr_free(&m);
  return s;
}

static std::vector<double> uniform(uint64_t seed, int n) {
  std::vector<double> v((size_t)n);
  or_rng_fill_uniform(seed, -1, 1, v.data(), n);
  return v;
}

static double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

struct Lattice {
  SparseOperator c, d;
};

static Lattice pec_lattice(int nx, int ny, int nz, double dx, double dy, double dz) {
  sfeec_csr_owned c, d;
  if (sfeec_build_yee_curl(nx, ny, nz, dx, dy, dz, SFEEC_BC_PEC, &c, &d)) std::abort();
  return {from_owned(c), from_owned(d)};
}

// host-side API: core.hpp's Rng is the reference splitmix64 stream, and the
// coordinate-list export / import round-trips (test_operators.cpp:294-320)
static void host_checks() {
  {
    Rng r(42);
    std::vector<double> want = uniform(42, 5), got;
    for (int k = 0; k < 5; ++k) got.push_back(r.uniform(-1, 1));
    CHECK(got == want);
  }
  std::vector<Triplet> tri;
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 7; ++c)
      if ((r + c) % 3 != 1) tri.push_back({r, c, 1.0 / (1.0 + r + c) + (r == c)});
  SparseOperator m = operator_from_triplets(7, 7, tri);
  const std::string text = to_coordinate_list(m);
  std::istringstream is(text);
  int pr = -1, pc = -1, r, c;
  double v;
  while (is >> r >> c >> v) {  // sorted by (row, col)
    CHECK(r > pr || (r == pr && c > pc));
    pr = r;
    pc = c;
  }
  std::istringstream is2(text);
  SparseOperator m2 = read_coordinate_list(is2);
  CHECK(m2.rows == 7 && m2.cols == 7 && m2.nnz() == m.nnz() && m2.symmetric);
  CHECK(m2.val == m.val && m2.col_idx == m.col_idx && m2.row_ptr == m.row_ptr);
  std::ostringstream os;
  write_coordinate_list(os, m2);
  CHECK(os.str() == text);
  std::istringstream is3("0 1 2.5\n2 0 -1\n");  // explicit shape, not symmetric
  SparseOperator m3 = read_coordinate_list(is3, 4, 3);
  CHECK(m3.rows == 4 && m3.cols == 3 && m3.nnz() == 2 && !m3.symmetric);
}

int main() {
  host_checks();
  if (sfeec_device_count() == 0) {
    std::puts(failures ? "host checks FAILED; no GPU: device checks skipped"
                       : "no GPU: skipped");
    return failures ? 1 : 0;
  }
  // ---- sub-flow closed forms (test_dynamics.cpp:67-94) --------------------
  {
    Lattice L = pec_lattice(3, 3, 3, 1, 1, 1);
    const int n1 = L.c.cols;
    SparseOperator q = scaled_identity(n1, 1.0), m2 = scaled_identity(L.c.rows, 1.0);
    SplitScheme scheme(SplitKind::Strang, 0.1, q, L.c, m2);
    FieldState s = make_state(Formulation::AE, uniform(1, n1), std::vector<double>(n1, 0.0));
    FieldState t = s;
    scheme.flow_he(t, 0.34);
    CHECK(max_abs_diff(s.first, t.first) == 0.0);
    s = make_state(Formulation::AE, uniform(2, n1), uniform(3, n1));
    t = s;
    scheme.flow_he(t, 0.0);
    scheme.flow_ha(t, 0.0);
    CHECK(max_abs_diff(s.first, t.first) == 0.0 && max_abs_diff(s.e, t.e) == 0.0);
  }
  // ---- scalar toy (test_dynamics.cpp:96-111) -------------------------------
  {
    SparseOperator q = scaled_identity(1, 0.5), c;
    c.rows = c.cols = 1;
    c.row_ptr = {0, 0};
    SparseOperator m2 = scaled_identity(1, 1.0);
    SplitScheme scheme(SplitKind::Strang, 0.25, q, c, m2, UnitSystem{}, nullptr, false);
    FieldState s = make_state(Formulation::AE, {1.0}, {0.5});
    scheme.flow_he(s, 0.25);
    CHECK(std::abs(s.first[0] - (1.0 - 0.25 * 0.5 / 2.0)) <= 1e-15);
    CHECK(s.e[0] == 0.5 && s.time == 0.0);
  }
  // ---- errors as the reference (dynamics.cpp:11-12, 41-43) -----------------
  {
    Lattice L = pec_lattice(2, 2, 2, 1, 1, 1);
    SparseOperator q = scaled_identity(L.c.cols, 1.0), m2 = scaled_identity(L.c.rows, 1.0);
    bool threw = false;
    try {
      SplitScheme s(SplitKind::Strang, -1.0, q, L.c, m2);
    } catch (const InvalidParameter&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      SplitScheme s(SplitKind::Strang, 0.1, scaled_identity(L.c.cols + 1, 1.0), L.c, m2);
    } catch (const InvalidParameter&) {
      threw = true;
    }
    CHECK(threw);
  }
  // ---- device step vs the C oracle, Gauss law, energy ----------------------
  {
    Lattice L = pec_lattice(6, 5, 7, 1.0, 0.8, 1.25);
    const double dv = 1.0 * 0.8 * 1.25;
    const int n1 = L.c.cols, n2 = L.c.rows;
    SparseOperator q = scaled_identity(n1, 1.0 / dv), m2 = scaled_identity(n2, dv);
    SplitScheme scheme(SplitKind::Strang, 0.2, q, L.c, m2, UnitSystem{}, &L.d, false);
    std::vector<double> a0 = uniform(3, n1), b0 = matvec(L.c, a0), e0 = uniform(4, n1);
    FieldState s = make_state(Formulation::BE, b0, e0);
    CHECK(scheme.gauss_residual(s) <= 1e-14);
    FieldState out = scheme.advance(s, 100);
    CHECK(std::abs(out.time - 100 * 0.2) <= 1e-12);
    CHECK(scheme.gauss_residual(out) <= 1e-13);
    // oracle
    std::vector<int64_t> rp[4];
    const SparseOperator* ops[4] = {&scheme.q_sym(), &L.c, &scheme.curl_t(), &m2};
    or_csr oc[4];
    for (int k = 0; k < 4; ++k) {
      rp[k].assign(ops[k]->row_ptr.begin(), ops[k]->row_ptr.end());
      oc[k] = {ops[k]->rows, ops[k]->cols, rp[k].data(), ops[k]->col_idx.data(),
               ops[k]->val.data()};
    }
    or_scheme os{1, 1, 0.2, 1.0, 1.0, oc[0], oc[1], oc[2], oc[3], nullptr};
    std::vector<double> pb = b0, pe = e0;
    or_steps(&os, pb.data(), pe.data(), 100, nullptr);
    double nb = 0, db = 0, ne = 0, de = 0;
    for (int i = 0; i < n2; ++i) {
      nb += pb[i] * pb[i];
      db += (pb[i] - out.first[i]) * (pb[i] - out.first[i]);
    }
    for (int i = 0; i < n1; ++i) {
      ne += pe[i] * pe[i];
      de += (pe[i] - out.e[i]) * (pe[i] - out.e[i]);
    }
    CHECK(std::sqrt(db / nb) <= 1e-12 && std::sqrt(de / ne) <= 1e-12);
    CHECK(std::abs(scheme.energy(out) - or_energy(&os, pb.data(), pe.data())) <=
          1e-12 * or_energy(&os, pb.data(), pe.data()));
    // spmv on the device is bitwise the reference's (sparse.cpp:96-104)
    std::vector<double> y1 = matvec(L.c, a0), y2((size_t)n2);
    or_spmv(&oc[1], a0.data(), y2.data());
    CHECK(max_abs_diff(y1, y2) == 0.0);
  }
  // ---- symplectic (test_dynamics.cpp:252-276) ------------------------------
  {
    Lattice L = pec_lattice(2, 2, 3, 1.0, 0.7, 1.3);
    const int n1 = L.c.cols;
    SparseOperator m2 = scaled_identity(L.c.rows, 0.91);
    for (double dt : {0.0, 0.05, 0.4})
      for (SplitKind sk : {SplitKind::Strang, SplitKind::LieTrotter}) {
        SplitScheme scheme(sk, dt, scaled_identity(n1, 1.0 / 0.91), L.c, m2, UnitSystem{},
                           nullptr, false);
        CHECK(symplectic_check(scheme, n1) <= 1e-12);
      }
  }
  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::puts("drop-in C++ API: all checks passed");
  return 0;
}
