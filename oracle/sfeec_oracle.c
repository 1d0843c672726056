/* TEST INFRASTRUCTURE ONLY -- see sfeec_oracle.h. Plain-C restatement of the
 * reference hot path; every function cites /root/reference/proj file:line. */
#include "sfeec_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- core.hpp:44-63 --------------------------------------------------- */
uint64_t or_rng_next_u64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double or_rng_uniform(uint64_t* state, double lo, double hi) {
  double u = (double)(or_rng_next_u64(state) >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * u;
}

void or_rng_fill_uniform(uint64_t seed, double lo, double hi, double* out, int64_t n) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) out[i] = or_rng_uniform(&s, lo, hi);
}

/* ---- sparse.cpp:96-104 ------------------------------------------------ */
void or_spmv(const or_csr* a, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < a->rows; ++r) {
    double acc = 0;
    for (int64_t k = a->row_ptr[r]; k < a->row_ptr[r + 1]; ++k)
      acc += a->val[k] * x[a->col_idx[k]];
    y[r] = acc;
  }
}

/* ---- sparse.cpp:20-61 ------------------------------------------------- */
typedef struct {
  int32_t r, c;
  int64_t i;
} trip_key;

static int trip_cmp(const void* pa, const void* pb) {
  const trip_key* a = (const trip_key*)pa;
  const trip_key* b = (const trip_key*)pb;
  if (a->r != b->r) return a->r < b->r ? -1 : 1;
  if (a->c != b->c) return a->c < b->c ? -1 : 1;
  return a->i < b->i ? -1 : (a->i > b->i); /* stable within a slot */
}

int64_t or_from_triplets(int64_t rows, int64_t n, const int32_t* r, const int32_t* c,
                         const double* v, int64_t* row_ptr, int32_t* col_idx, double* val) {
  trip_key* k = (trip_key*)malloc(sizeof(trip_key) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    k[i].r = r[i];
    k[i].c = c[i];
    k[i].i = i;
  }
  qsort(k, (size_t)n, sizeof(trip_key), trip_cmp);
  if (row_ptr)
    for (int64_t i = 0; i <= rows; ++i) row_ptr[i] = 0;
  int64_t nnz = 0, i = 0;
  while (i < n) {
    double sum = 0;
    int64_t j = i;
    while (j < n && k[j].r == k[i].r && k[j].c == k[i].c) {
      sum += v[k[j].i];
      ++j;
    }
    if (sum != 0.0) {
      if (col_idx) col_idx[nnz] = k[i].c;
      if (val) val[nnz] = sum;
      if (row_ptr) row_ptr[k[i].r + 1] += 1;
      ++nnz;
    }
    i = j;
  }
  if (row_ptr)
    for (int64_t q = 0; q < rows; ++q) row_ptr[q + 1] += row_ptr[q];
  free(k);
  return nnz;
}

/* ---- dynamics.cpp:10-25 ----------------------------------------------- */
int64_t or_symmetric_part(const or_csr* q, int64_t* row_ptr, int32_t* col_idx, double* val) {
  int64_t nnz = q->row_ptr[q->rows];
  int32_t* r = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * nnz + 1));
  int32_t* c = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * nnz + 1));
  double* v = (double*)malloc(sizeof(double) * (size_t)(2 * nnz + 1));
  int64_t t = 0;
  for (int64_t row = 0; row < q->rows; ++row)
    for (int64_t k = q->row_ptr[row]; k < q->row_ptr[row + 1]; ++k) {
      r[t] = (int32_t)row;
      c[t] = q->col_idx[k];
      v[t++] = 0.5 * q->val[k];
      r[t] = q->col_idx[k];
      c[t] = (int32_t)row;
      v[t++] = 0.5 * q->val[k];
    }
  int64_t out = or_from_triplets(q->rows, t, r, c, v, row_ptr, col_idx, val);
  free(r);
  free(c);
  free(v);
  return out;
}

/* ---- sparse.cpp:75-94 ------------------------------------------------- */
void or_transpose(const or_csr* a, int64_t* row_ptr, int32_t* col_idx, double* val) {
  int64_t nnz = a->row_ptr[a->rows];
  for (int64_t i = 0; i <= a->cols; ++i) row_ptr[i] = 0;
  for (int64_t k = 0; k < nnz; ++k) row_ptr[a->col_idx[k] + 1] += 1;
  for (int64_t i = 0; i < a->cols; ++i) row_ptr[i + 1] += row_ptr[i];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(a->cols + 1));
  memcpy(cursor, row_ptr, sizeof(int64_t) * (size_t)a->cols);
  for (int64_t r = 0; r < a->rows; ++r)
    for (int64_t k = a->row_ptr[r]; k < a->row_ptr[r + 1]; ++k) {
      int64_t slot = cursor[a->col_idx[k]]++;
      col_idx[slot] = (int32_t)r;
      val[slot] = a->val[k];
    }
  free(cursor);
}

/* ---- dynamics.cpp:47-90 ----------------------------------------------- */
static double* vec(int64_t n) { return (double*)calloc((size_t)(n ? n : 1), sizeof(double)); }

void or_flow_he(const or_scheme* s, double* first, double* e, double dt) {
  double* qe = vec(s->q_sym.rows);
  or_spmv(&s->q_sym, e, qe);
  if (!s->be) {
    for (int64_t i = 0; i < s->q_sym.rows; ++i) first[i] -= dt * qe[i];
  } else {
    double* cqe = vec(s->c.rows);
    or_spmv(&s->c, qe, cqe);
    for (int64_t i = 0; i < s->c.rows; ++i) first[i] -= dt * cqe[i];
    free(cqe);
  }
  free(qe);
}

void or_flow_ha(const or_scheme* s, double* first, double* e, double dt) {
  const double c2 = 1.0 / (s->eps0 * s->mu0);
  const double f = dt * c2;
  double* mb = vec(s->m2.rows);
  double* ctm = vec(s->ct.rows);
  if (!s->be) {
    double* ca = vec(s->c.rows);
    or_spmv(&s->c, first, ca);
    or_spmv(&s->m2, ca, mb);
    free(ca);
  } else {
    or_spmv(&s->m2, first, mb);
  }
  or_spmv(&s->ct, mb, ctm);
  for (int64_t i = 0; i < s->ct.rows; ++i) e[i] += f * ctm[i];
  free(mb);
  free(ctm);
}

void or_steps(const or_scheme* s, double* first, double* e, int64_t nsteps,
              double* energy_hist) {
  for (int64_t n = 0; n < nsteps; ++n) {
    if (s->strang) {
      or_flow_he(s, first, e, 0.5 * s->dt);
      or_flow_ha(s, first, e, s->dt);
      or_flow_he(s, first, e, 0.5 * s->dt);
    } else {
      or_flow_he(s, first, e, s->dt);
      or_flow_ha(s, first, e, s->dt);
    }
    if (energy_hist) energy_hist[n] = or_energy(s, first, e);
  }
}

/* ---- dynamics.cpp:92-102 ---------------------------------------------- */
double or_energy(const or_scheme* s, const double* first, const double* e) {
  int64_t n1 = s->q_sym.rows, n2 = s->m2.rows;
  double* qe = vec(n1);
  or_spmv(&s->q_sym, e, qe);
  double he = 0;
  for (int64_t i = 0; i < n1; ++i) he += e[i] * qe[i];
  double* b = vec(n2);
  if (!s->be)
    or_spmv(&s->c, first, b);
  else
    memcpy(b, first, sizeof(double) * (size_t)n2);
  double* mb = vec(n2);
  or_spmv(&s->m2, b, mb);
  double ha = 0;
  for (int64_t i = 0; i < n2; ++i) ha += b[i] * mb[i];
  free(qe);
  free(b);
  free(mb);
  return 0.5 * (s->eps0 * he + ha / s->mu0);
}

/* ---- dynamics.cpp:104-112 --------------------------------------------- */
double or_gauss_residual(const or_scheme* s, const double* b) {
  if (!s->div) return 0.0;
  double* db = vec(s->div->rows);
  or_spmv(s->div, b, db);
  double m = 0;
  for (int64_t i = 0; i < s->div->rows; ++i) m = fmax(m, fabs(db[i]));
  free(db);
  return m;
}

/* ---- dynamics.cpp:114-133 --------------------------------------------- */
double or_cfl_number(const or_scheme* s) {
  const int64_t n = s->q_sym.rows;
  double* x = vec(n);
  double* t2 = vec(s->c.rows);
  double* t3 = vec(s->m2.rows);
  double* t1 = vec(n);
  double* y = vec(n);
  uint64_t st = 0x5fec5fec;
  for (int64_t i = 0; i < n; ++i) x[i] = or_rng_uniform(&st, -1, 1);
  double lambda = 0;
  for (int it = 0; it < 40; ++it) {
    or_spmv(&s->c, x, t2);
    or_spmv(&s->m2, t2, t3);
    or_spmv(&s->ct, t3, t1);
    or_spmv(&s->q_sym, t1, y);
    double nrm = 0;
    for (int64_t i = 0; i < n; ++i) nrm += y[i] * y[i];
    nrm = sqrt(nrm);
    if (nrm == 0) break;
    lambda = nrm;
    for (int64_t i = 0; i < n; ++i) x[i] = y[i] / nrm;
  }
  free(x);
  free(t1);
  free(t2);
  free(t3);
  free(y);
  return s->dt * sqrt((1.0 / (s->eps0 * s->mu0)) * lambda);
}

/* ---- yee.cpp:9-74 ------------------------------------------------------ */
static inline int64_t wrapi(int64_t i, int64_t n) { return ((i % n) + n) % n; }
static inline int64_t yidx(int nx, int ny, int nz, int64_t i, int64_t j, int64_t k) {
  return wrapi(i, nx) + (int64_t)nx * (wrapi(j, ny) + (int64_t)ny * wrapi(k, nz));
}

void or_yee_advance_e(int nx, int ny, int nz, const double d[3], double* e, const double* b,
                      double dt, double c2) {
  const int64_t nc = (int64_t)nx * ny * nz;
  double* next = vec(nc);
  for (int a = 0; a < 3; ++a) {
    int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    const double* ba1 = b + a1 * nc;
    const double* ba2 = b + a2 * nc;
    double* ea = e + a * nc;
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          int64_t s1[3] = {0, 0, 0}, s2[3] = {0, 0, 0};
          s1[a1] = 1;
          s2[a2] = 1;
          int64_t here = yidx(nx, ny, nz, i, j, k);
          int64_t m1 = yidx(nx, ny, nz, i - s1[0], j - s1[1], k - s1[2]);
          int64_t m2 = yidx(nx, ny, nz, i - s2[0], j - s2[1], k - s2[2]);
          double curl = (ba2[here] - ba2[m1]) / d[a1] - (ba1[here] - ba1[m2]) / d[a2];
          next[here] = ea[here] + c2 * dt * curl;
        }
    memcpy(ea, next, sizeof(double) * (size_t)nc);
  }
  free(next);
}

void or_yee_advance_b(int nx, int ny, int nz, const double d[3], const double* e, double* b,
                      double dt) {
  const int64_t nc = (int64_t)nx * ny * nz;
  double* next = vec(nc);
  for (int a = 0; a < 3; ++a) {
    int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
    const double* ea1 = e + a1 * nc;
    const double* ea2 = e + a2 * nc;
    double* ba = b + a * nc;
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          int64_t s1[3] = {0, 0, 0}, s2[3] = {0, 0, 0};
          s1[a1] = 1;
          s2[a2] = 1;
          int64_t here = yidx(nx, ny, nz, i, j, k);
          int64_t p2 = yidx(nx, ny, nz, i + s2[0], j + s2[1], k + s2[2]);
          int64_t p1 = yidx(nx, ny, nz, i + s1[0], j + s1[1], k + s1[2]);
          double curl = (ea1[p2] - ea1[here]) / d[a2] - (ea2[p1] - ea2[here]) / d[a1];
          next[here] = ba[here] + dt * curl;
        }
    memcpy(ba, next, sizeof(double) * (size_t)nc);
  }
  free(next);
}
