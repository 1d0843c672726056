// The C++ drop-in (include/sfeec/{sparse,dynamics}.hpp) over the C ABI.
// Mirrors the reference's classes (sparse.hpp:14-66, dynamics.hpp:9-76) and
// error contract (InvalidParameter for bad parameters, std::runtime_error for
// device failures). Setup helpers run on the host; every SpMV and every
// step runs on the B200.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <ostream>
#include <sstream>

#include "common.hpp"
#include "sfeec/dynamics.hpp"

namespace sfeec {

namespace {

void check(int code) {
  if (code == SFEEC_OK) return;
  if (code == SFEEC_EINVAL) throw InvalidParameter(sfeec_last_error());
  throw std::runtime_error(std::string("sfeec_b200: ") + sfeec_last_error());
}

// int32 reference CSR <-> int64 C-ABI view
struct View {
  std::vector<int64_t> rp;
  sfeec_csr v;
  explicit View(const SparseOperator& a) : rp(a.row_ptr.begin(), a.row_ptr.end()) {
    if (rp.empty()) rp.assign((size_t)a.rows + 1, 0);
    v.rows = a.rows;
    v.cols = a.cols;
    v.row_ptr = rp.data();
    v.col_idx = a.col_idx.data();
    v.val = a.val.data();
  }
};

SparseOperator from_host(const sfeec_b200::HostCSR& h, bool symmetric) {
  if (h.nnz() > INT32_MAX || h.rows > INT32_MAX)
    throw InvalidParameter("operator exceeds the int32 SparseOperator (use the C ABI)");
  SparseOperator m;
  m.rows = (int)h.rows;
  m.cols = (int)h.cols;
  m.symmetric = symmetric;
  m.row_ptr.assign(h.row_ptr.begin(), h.row_ptr.end());
  m.col_idx.assign(h.col_idx.begin(), h.col_idx.end());
  m.val = h.val;
  return m;
}

sfeec_b200::HostCSR to_host(const SparseOperator& a) {
  sfeec_b200::HostCSR h;
  h.rows = a.rows;
  h.cols = a.cols;
  h.row_ptr.assign(a.row_ptr.begin(), a.row_ptr.end());
  if (h.row_ptr.empty()) h.row_ptr.assign((size_t)a.rows + 1, 0);
  h.col_idx.assign(a.col_idx.begin(), a.col_idx.end());
  h.val = a.val;
  return h;
}

}  // namespace

double SparseOperator::at(int r, int c) const {
  auto cs = row_cols(r);
  auto it = std::lower_bound(cs.begin(), cs.end(), c);
  if (it == cs.end() || *it != c) return 0.0;
  return row_vals(r)[(size_t)(it - cs.begin())];
}

SparseOperator operator_from_triplets(int rows, int cols, std::vector<Triplet> triplets,
                                      bool symmetric) {
  std::vector<int32_t> r(triplets.size()), c(triplets.size());
  std::vector<double> v(triplets.size());
  for (size_t i = 0; i < triplets.size(); ++i) {
    r[i] = triplets[i].r;
    c[i] = triplets[i].c;
    v[i] = triplets[i].v;
  }
  try {
    return from_host(sfeec_b200::csr_from_triplets(rows, cols, (int64_t)triplets.size(),
                                                    r.data(), c.data(), v.data()),
                     symmetric);
  } catch (const sfeec_b200::Error& e) {
    throw InvalidParameter(e.what());
  }
}

SparseOperator scaled_identity(int n, double s) {
  SparseOperator m;
  m.rows = m.cols = n;
  m.symmetric = true;
  m.row_ptr.resize((size_t)n + 1);
  m.col_idx.resize((size_t)n);
  m.val.assign((size_t)n, s);
  for (int i = 0; i <= n; ++i) m.row_ptr[(size_t)i] = i;
  for (int i = 0; i < n; ++i) m.col_idx[(size_t)i] = i;
  return m;
}

SparseOperator transpose(const SparseOperator& a) {
  return from_host(sfeec_b200::csr_transpose(to_host(a)), a.symmetric);
}

void spmv(const SparseOperator& a, const double* x, double* y) {
  View v(a);
  check(sfeec_spmv(&v.v, x, y, 0));
}

void spmv_serial(const SparseOperator& a, const double* x, double* y) { spmv(a, x, y); }

std::vector<double> matvec(const SparseOperator& a, const std::vector<double>& x) {
  if ((int)x.size() != a.cols) throw InvalidParameter("spmv: dimension mismatch");
  std::vector<double> y((size_t)a.rows);
  spmv(a, x.data(), y.data());
  return y;
}

double max_abs(const SparseOperator& a) {
  double m = 0;
  for (double v : a.val) m = std::max(m, std::abs(v));
  return m;
}

double max_asymmetry(const SparseOperator& a) {
  if (a.rows != a.cols) throw InvalidParameter("max_asymmetry: square only");
  double m = 0;
  for (int r = 0; r < a.rows; ++r) {
    auto cs = a.row_cols(r);
    auto vs = a.row_vals(r);
    for (size_t k = 0; k < cs.size(); ++k) m = std::max(m, std::abs(vs[k] - a.at(cs[k], r)));
  }
  return m;
}

void write_coordinate_list(std::ostream& os, const SparseOperator& a) {
  // rows ascending, stored (ascending) column order within a row
  char line[80];
  for (int r = 0; r < a.rows; ++r)
    for (int k = a.row_ptr[(size_t)r]; k < a.row_ptr[(size_t)r + 1]; ++k) {
      const int n = std::snprintf(line, sizeof(line), "%d %d %.17g\n", r,
                                  a.col_idx[(size_t)k], a.val[(size_t)k]);
      os.write(line, n);
    }
}

std::string to_coordinate_list(const SparseOperator& a) {
  std::ostringstream os;
  write_coordinate_list(os, a);
  return os.str();
}

SparseOperator read_coordinate_list(std::istream& is, int rows, int cols) {
  std::vector<Triplet> entries;
  int hi_r = -1, hi_c = -1;
  for (Triplet t; is >> t.r >> t.c >> t.v;) {  // until the first unparsable token
    hi_r = std::max(hi_r, t.r);
    hi_c = std::max(hi_c, t.c);
    entries.push_back(t);
  }
  SparseOperator m = operator_from_triplets(rows < 0 ? hi_r + 1 : rows,
                                            cols < 0 ? hi_c + 1 : cols, std::move(entries));
  m.symmetric = m.rows == m.cols && max_asymmetry(m) == 0.0;
  return m;
}

std::vector<double> to_dense(const SparseOperator& a) {
  std::vector<double> d((size_t)a.rows * (size_t)a.cols, 0.0);
  for (int r = 0; r < a.rows; ++r) {
    auto cs = a.row_cols(r);
    auto vs = a.row_vals(r);
    for (size_t k = 0; k < cs.size(); ++k) d[(size_t)r * (size_t)a.cols + (size_t)cs[k]] = vs[k];
  }
  return d;
}

// ---- SplitScheme ------------------------------------------------------------
namespace {
SparseOperator symmetric_part(const SparseOperator& q) {
  if (q.rows != q.cols) throw InvalidParameter("SplitScheme: Q must be square");
  return from_host(sfeec_b200::csr_symmetric_part(to_host(q)), true);
}
}  // namespace

SplitScheme::SplitScheme(SplitKind kind, double dt, const SparseOperator& q,
                         const SparseOperator& c, const SparseOperator& m2, UnitSystem units,
                         const SparseOperator* div, bool warn_cfl)
    : kind_(kind),
      dt_(dt),
      units_(units),
      q_sym_(symmetric_part(q)),
      c_(c),
      ct_(transpose(c)),
      m2_(m2),
      warn_cfl_(warn_cfl) {
  if (!(dt >= 0)) throw InvalidParameter("SplitScheme: dt must be >= 0");
  if (m2_.rows != c_.rows || q_sym_.rows != c_.cols)
    throw InvalidParameter("SplitScheme: operator dimensions inconsistent");
  if (div) div_ = *div;
}

SplitScheme::~SplitScheme() {
  for (auto& h : dev_)
    if (h) sfeec_dev_destroy(h);
}

SplitScheme::SplitScheme(SplitScheme&& o) noexcept
    : kind_(o.kind_),
      dt_(o.dt_),
      units_(o.units_),
      q_sym_(std::move(o.q_sym_)),
      c_(std::move(o.c_)),
      ct_(std::move(o.ct_)),
      m2_(std::move(o.m2_)),
      div_(std::move(o.div_)),
      warn_cfl_(o.warn_cfl_),
      warned_(o.warned_) {
  dev_[0] = o.dev_[0];
  dev_[1] = o.dev_[1];
  o.dev_[0] = o.dev_[1] = nullptr;
}

SplitScheme& SplitScheme::operator=(SplitScheme&& o) noexcept {
  if (this != &o) {
    this->~SplitScheme();
    new (this) SplitScheme(std::move(o));
  }
  return *this;
}

sfeec_dev* SplitScheme::device(Formulation f) const {
  const int i = f == Formulation::BE ? 1 : 0;
  if (!dev_[i]) {
    View q(q_sym_), c(c_), m(m2_);
    std::optional<View> d;
    if (div_) d.emplace(*div_);
    check(sfeec_dev_create(&q.v, &c.v, &m.v, d ? &d->v : nullptr, dt_, units_.eps0, units_.mu0,
                           kind_ == SplitKind::Strang ? SFEEC_SPLIT_STRANG
                                                      : SFEEC_SPLIT_LIE_TROTTER,
                           i == 1 ? SFEEC_FORM_BE : SFEEC_FORM_AE, 0,
                           SFEEC_Q_IS_SYMMETRIC | SFEEC_NO_CFL_WARN, &dev_[i]));
  }
  return dev_[i];
}

void SplitScheme::load(sfeec_dev* h, const FieldState& s) const {
  check(sfeec_dev_set_state(h, s.first.data(), (int64_t)s.first.size(), s.e.data(),
                            (int64_t)s.e.size(), s.time));
}

void SplitScheme::fetch(sfeec_dev* h, FieldState& s) const {
  double t = 0;
  check(sfeec_dev_get_state(h, s.first.data(), s.e.data(), &t));
  s.time = t;
}

void SplitScheme::flow_he(FieldState& s, double dt) const {
  sfeec_dev* h = device(s.formulation);
  double t = s.time;
  load(h, s);
  check(sfeec_dev_flow_he(h, dt));
  fetch(h, s);
  s.time = t;
}

void SplitScheme::flow_ha(FieldState& s, double dt) const {
  sfeec_dev* h = device(s.formulation);
  double t = s.time;
  load(h, s);
  check(sfeec_dev_flow_ha(h, dt));
  fetch(h, s);
  s.time = t;
}

FieldState SplitScheme::step(const FieldState& s) const { return advance(s, 1); }

FieldState SplitScheme::advance(const FieldState& s, std::int64_t nsteps) const {
  if (warn_cfl_ && !warned_) {  // dynamics.cpp:70-78
    warned_ = true;
    double nu = cfl_number();
    if (nu > 2.0)
      std::fprintf(stderr,
                   "sfeec: warning: CFL number %.3g > 2; the splitting is likely unstable at "
                   "dt = %.3g\n",
                   nu, dt_);
  }
  sfeec_dev* h = device(s.formulation);
  FieldState out = s;
  load(h, out);
  check(sfeec_dev_advance(h, nsteps));
  fetch(h, out);
  return out;
}

double SplitScheme::energy(const FieldState& s) const {
  sfeec_dev* h = device(s.formulation);
  load(h, s);
  double e = 0;
  check(sfeec_dev_energy(h, &e));
  return e;
}

double SplitScheme::gauss_residual(const FieldState& s) const {
  if (s.formulation != Formulation::BE)
    throw InvalidParameter("gauss_residual: (b, e) formulation required");
  sfeec_dev* h = device(s.formulation);
  load(h, s);
  double g = 0;
  check(sfeec_dev_gauss_residual(h, &g));
  return g;
}

double SplitScheme::cfl_number() const {
  sfeec_dev* h = dev_[1] ? dev_[1] : device(Formulation::AE);
  double nu = 0;
  check(sfeec_dev_cfl_number(h, &nu));
  return nu;
}

FieldState make_state(Formulation f, std::vector<double> first, std::vector<double> e,
                      double time) {
  FieldState s;
  s.formulation = f;
  s.first = std::move(first);
  s.e = std::move(e);
  s.time = time;
  return s;
}

namespace {
// `copies` copies of `a` on the diagonal, as an int64 C-ABI view
struct BlockDiag {
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  sfeec_csr view;
  BlockDiag(const SparseOperator& a, int copies) {
    const int64_t nnz = (int64_t)a.val.size();
    rp.resize((size_t)a.rows * copies + 1);
    ci.resize((size_t)(nnz * copies));
    v.resize((size_t)(nnz * copies));
    rp[0] = 0;
    for (int b = 0; b < copies; ++b) {
      const int64_t off = nnz * b;
      for (int r = 0; r < a.rows; ++r) rp[(size_t)b * a.rows + r + 1] = off + a.row_ptr[r + 1];
      for (int64_t k = 0; k < nnz; ++k) {
        ci[(size_t)(off + k)] = a.col_idx[(size_t)k] + b * a.cols;
        v[(size_t)(off + k)] = a.val[(size_t)k];
      }
    }
    view.rows = (int64_t)a.rows * copies;
    view.cols = (int64_t)a.cols * copies;
    view.row_ptr = rp.data();
    view.col_idx = ci.data();
    view.val = v.data();
  }
};
}  // namespace

// Symplecticity of the one-step map Phi (the property of dynamics.cpp:145-185):
// max |Phi^T J Phi - J| with J = (1/eps0) [[0, -I], [I, 0]] on (a, e).
// Phi is taken in one device pass: the 2 n1 unit initial states are the
// diagonal blocks of one block-diagonal system, advanced together by one
// resident step; then with Phi = [A; E] (A the a-rows, E the e-rows),
// Phi^T J Phi = (1/eps0) (P - P^T) for P = E^T A.
double symplectic_check(const SplitScheme& scheme, int n1, int max_dofs) {
  if (2 * n1 > max_dofs)
    throw InvalidParameter("symplectic_check: system too large for the dense check");
  if (n1 != scheme.q_sym().rows)
    throw InvalidParameter("symplectic_check: n1 must equal the 1-form dimension");
  const int m = 2 * n1;  // columns of Phi = batch size
  BlockDiag q(scheme.q_sym(), m), c(scheme.curl(), m), m2(scheme.m2(), m);
  sfeec_dev* h = nullptr;
  check(sfeec_dev_create(&q.view, &c.view, &m2.view, nullptr, scheme.dt(), scheme.units().eps0,
                         scheme.units().mu0,
                         scheme.kind() == SplitKind::Strang ? SFEEC_SPLIT_STRANG
                                                            : SFEEC_SPLIT_LIE_TROTTER,
                         SFEEC_FORM_AE, 0, SFEEC_Q_IS_SYMMETRIC | SFEEC_NO_CFL_WARN, &h));
  std::unique_ptr<sfeec_dev, void (*)(sfeec_dev*)> guard(h, sfeec_dev_destroy);
  // batch b starts from unit vector b of (a, e): a-part for b < n1, e-part after
  const size_t nb = (size_t)n1 * (size_t)m;
  std::vector<double> a(nb, 0.0), e(nb, 0.0);
  for (int b = 0; b < m; ++b) (b < n1 ? a : e)[(size_t)b * n1 + (size_t)(b % n1)] = 1.0;
  check(sfeec_dev_set_state(h, a.data(), (int64_t)nb, e.data(), (int64_t)nb, 0.0));
  check(sfeec_dev_advance(h, 1));
  double t = 0;
  check(sfeec_dev_get_state(h, a.data(), e.data(), &t));
  // column b of A / E is block b of the advanced batch
  std::vector<double> p((size_t)m * (size_t)m);
  for (int i = 0; i < m; ++i) {
    const double* ei = &e[(size_t)i * n1];
    for (int j = 0; j < m; ++j) {
      const double* aj = &a[(size_t)j * n1];
      double s = 0;
      for (int k = 0; k < n1; ++k) s += ei[k] * aj[k];
      p[(size_t)i * m + j] = s;
    }
  }
  const double se = 1.0 / scheme.units().eps0;
  double dev = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      const double jij = (j - i == n1) ? -se : (i - j == n1) ? se : 0.0;
      dev = std::max(dev, std::abs(se * (p[(size_t)i * m + j] - p[(size_t)j * m + i]) - jij));
    }
  return dev;
}

}  // namespace sfeec
