// Host-side CSR construction (setup, not timed): deterministic COO->CSR,
// symmetric part, transpose, and the lumped Yee curl/divergence builders.
// Semantics follow the reference exactly (bitwise), but the algorithms are
// O(nnz) bucket/merge passes instead of the reference's global sort so they
// scale to the 10^9-nonzero operators of configs 3-5.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.hpp"

namespace sfeec_b200 {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

void csr_validate(const sfeec_csr& v, const char* name) {
  require(v.rows >= 0 && v.cols >= 0, std::string(name) + ": negative dimension");
  require(v.row_ptr != nullptr, std::string(name) + ": null row_ptr");
  require(v.row_ptr[0] == 0, std::string(name) + ": row_ptr[0] != 0");
  int64_t nnz = v.row_ptr[v.rows];
  require(nnz == 0 || (v.col_idx && v.val), std::string(name) + ": null col_idx/val");
  for (int64_t r = 0; r < v.rows; ++r) {
    require(v.row_ptr[r + 1] >= v.row_ptr[r], std::string(name) + ": row_ptr not monotone");
    for (int64_t k = v.row_ptr[r]; k < v.row_ptr[r + 1]; ++k)
      require(v.col_idx[k] >= 0 && v.col_idx[k] < v.cols,
              std::string(name) + ": column index out of range");
  }
}

HostCSR csr_from_view(const sfeec_csr& v) {
  HostCSR m;
  m.rows = v.rows;
  m.cols = v.cols;
  int64_t nnz = v.row_ptr[v.rows];
  m.row_ptr.assign(v.row_ptr, v.row_ptr + v.rows + 1);
  m.col_idx.assign(v.col_idx, v.col_idx + nnz);
  m.val.assign(v.val, v.val + nnz);
  return m;
}

// sparse.cpp:20-61 semantics: entries ordered by (row, col, input position);
// duplicates summed in input order starting from 0.0; exact zeros dropped.
HostCSR csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int32_t* r,
                          const int32_t* c, const double* v) {
  for (int64_t i = 0; i < n; ++i)
    require(r[i] >= 0 && r[i] < rows && c[i] >= 0 && c[i] < cols,
            "triplet index out of range");
  // stable bucket by row keeps input order inside each row
  std::vector<int64_t> start((size_t)rows + 1, 0);
  for (int64_t i = 0; i < n; ++i) start[(size_t)r[i] + 1]++;
  for (int64_t i = 0; i < rows; ++i) start[(size_t)i + 1] += start[(size_t)i];
  std::vector<int64_t> order((size_t)n);
  {
    std::vector<int64_t> cur(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < n; ++i) order[(size_t)cur[(size_t)r[i]]++] = i;
  }
  HostCSR m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign((size_t)rows + 1, 0);
  std::vector<int64_t> cnt((size_t)rows, 0);
  std::vector<int32_t> tmp_c((size_t)n);
  std::vector<double> tmp_v((size_t)n);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t row = 0; row < rows; ++row) {
    int64_t b = start[(size_t)row], e = start[(size_t)row + 1];
    // stable sort by column keeps input order among duplicates
    std::stable_sort(order.begin() + b, order.begin() + e,
                     [&](int64_t x, int64_t y) { return c[x] < c[y]; });
    int64_t w = b;
    int64_t i = b;
    while (i < e) {
      int32_t col = c[order[(size_t)i]];
      double sum = 0;
      int64_t j = i;
      while (j < e && c[order[(size_t)j]] == col) sum += v[order[(size_t)j++]];
      if (sum != 0.0) {
        tmp_c[(size_t)w] = col;
        tmp_v[(size_t)w] = sum;
        ++w;
      }
      i = j;
    }
    cnt[(size_t)row] = w - b;
  }
  for (int64_t row = 0; row < rows; ++row)
    m.row_ptr[(size_t)row + 1] = m.row_ptr[(size_t)row] + cnt[(size_t)row];
  m.col_idx.resize((size_t)m.row_ptr[(size_t)rows]);
  m.val.resize((size_t)m.row_ptr[(size_t)rows]);
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < rows; ++row) {
    int64_t b = start[(size_t)row], o = m.row_ptr[(size_t)row];
    for (int64_t k = 0; k < cnt[(size_t)row]; ++k) {
      m.col_idx[(size_t)(o + k)] = tmp_c[(size_t)(b + k)];
      m.val[(size_t)(o + k)] = tmp_v[(size_t)(b + k)];
    }
  }
  return m;
}

// sparse.cpp:75-94
HostCSR csr_transpose(const HostCSR& a) {
  HostCSR t;
  t.rows = a.cols;
  t.cols = a.rows;
  t.row_ptr.assign((size_t)a.cols + 1, 0);
  for (int32_t c : a.col_idx) t.row_ptr[(size_t)c + 1]++;
  for (int64_t i = 0; i < a.cols; ++i) t.row_ptr[(size_t)i + 1] += t.row_ptr[(size_t)i];
  t.col_idx.resize(a.col_idx.size());
  t.val.resize(a.val.size());
  std::vector<int64_t> cur(t.row_ptr.begin(), t.row_ptr.end() - 1);
  for (int64_t r = 0; r < a.rows; ++r)
    for (int64_t k = a.row_ptr[(size_t)r]; k < a.row_ptr[(size_t)r + 1]; ++k) {
      int64_t slot = cur[(size_t)a.col_idx[(size_t)k]]++;
      t.col_idx[(size_t)slot] = (int32_t)r;
      t.val[(size_t)slot] = a.val[(size_t)k];
    }
  return t;
}

// dynamics.cpp:10-25. The reference emits (r,c,q/2),(c,r,q/2) pairs and sums
// per slot from 0.0; a slot receives at most one term from Q and one from Q^T
// and two-term sums commute, so a merge of Q/2 with Q^T/2 is bitwise equal.
HostCSR csr_symmetric_part(const HostCSR& q) {
  require(q.rows == q.cols, "SplitScheme: Q must be square");
  HostCSR qt = csr_transpose(q);
  HostCSR s;
  s.rows = s.cols = q.rows;
  s.row_ptr.assign((size_t)q.rows + 1, 0);
  std::vector<int64_t> cnt((size_t)q.rows);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < q.rows; ++r) {
    int64_t a = q.row_ptr[(size_t)r], ae = q.row_ptr[(size_t)r + 1];
    int64_t b = qt.row_ptr[(size_t)r], be = qt.row_ptr[(size_t)r + 1];
    int64_t n = 0;
    while (a < ae || b < be) {
      int32_t ca = a < ae ? q.col_idx[(size_t)a] : INT32_MAX;
      int32_t cb = b < be ? qt.col_idx[(size_t)b] : INT32_MAX;
      double sum = 0;
      if (ca <= cb) sum += 0.5 * q.val[(size_t)a++];
      if (cb <= ca) sum += 0.5 * qt.val[(size_t)b++];
      if (sum != 0.0) ++n;
    }
    cnt[(size_t)r] = n;
  }
  for (int64_t r = 0; r < q.rows; ++r) s.row_ptr[(size_t)r + 1] = s.row_ptr[(size_t)r] + cnt[(size_t)r];
  s.col_idx.resize((size_t)s.row_ptr[(size_t)q.rows]);
  s.val.resize((size_t)s.row_ptr[(size_t)q.rows]);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < q.rows; ++r) {
    int64_t a = q.row_ptr[(size_t)r], ae = q.row_ptr[(size_t)r + 1];
    int64_t b = qt.row_ptr[(size_t)r], be = qt.row_ptr[(size_t)r + 1];
    int64_t w = s.row_ptr[(size_t)r];
    while (a < ae || b < be) {
      int32_t ca = a < ae ? q.col_idx[(size_t)a] : INT32_MAX;
      int32_t cb = b < be ? qt.col_idx[(size_t)b] : INT32_MAX;
      int32_t col = std::min(ca, cb);
      double sum = 0;
      if (ca <= cb) sum += 0.5 * q.val[(size_t)a++];
      if (cb <= ca) sum += 0.5 * qt.val[(size_t)b++];
      if (sum != 0.0) {
        s.col_idx[(size_t)w] = col;
        s.val[(size_t)w++] = sum;
      }
    }
  }
  return s;
}

void csr_to_owned(HostCSR&& m, sfeec_csr_owned* out) {
  out->rows = m.rows;
  out->cols = m.cols;
  out->nnz = m.nnz();
  out->row_ptr = (int64_t*)std::malloc(sizeof(int64_t) * (size_t)(m.rows + 1));
  out->col_idx = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)std::max<int64_t>(1, m.nnz()));
  out->val = (double*)std::malloc(sizeof(double) * (size_t)std::max<int64_t>(1, m.nnz()));
  if (!out->row_ptr || !out->col_idx || !out->val) throw std::bad_alloc();
  std::memcpy(out->row_ptr, m.row_ptr.data(), sizeof(int64_t) * (size_t)(m.rows + 1));
  std::memcpy(out->col_idx, m.col_idx.data(), sizeof(int32_t) * (size_t)m.nnz());
  std::memcpy(out->val, m.val.data(), sizeof(double) * (size_t)m.nnz());
}

}  // namespace sfeec_b200

using namespace sfeec_b200;

extern "C" {

const char* sfeec_last_error(void) { return g_err.c_str(); }

const char* sfeec_version(void) { return "sfeec_b200 0.1 (sm_100a)"; }

void sfeec_csr_free(sfeec_csr_owned* m) {
  if (!m) return;
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->val);
  m->row_ptr = nullptr;
  m->col_idx = nullptr;
  m->val = nullptr;
}

int sfeec_csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int32_t* r,
                            const int32_t* c, const double* v, sfeec_csr_owned* out) {
  return guarded([&] { csr_to_owned(csr_from_triplets(rows, cols, n, r, c, v), out); });
}

int sfeec_csr_symmetric_part(const sfeec_csr* q, sfeec_csr_owned* out) {
  return guarded([&] {
    csr_validate(*q, "Q");
    csr_to_owned(csr_symmetric_part(csr_from_view(*q)), out);
  });
}

int sfeec_csr_transpose(const sfeec_csr* a, sfeec_csr_owned* out) {
  return guarded([&] {
    csr_validate(*a, "A");
    csr_to_owned(csr_transpose(csr_from_view(*a)), out);
  });
}

}  // extern "C"
