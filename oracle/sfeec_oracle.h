/* TEST INFRASTRUCTURE ONLY -- the CPU checker, never linked into the product.
 *
 * Plain-C restatement of the reference's leapfrog hot path
 * (/root/reference/proj/src/{sparse,dynamics,yee}.cpp). Every function cites
 * the reference lines it follows. Arithmetic order matches the reference
 * exactly (sequential per-row accumulation in CSR order, separate multiply and
 * add: the Makefile builds with -ffp-contract=off), so on the same inputs the
 * outputs are bitwise equal to oracle/_ref/libsfeec_ref.so -- the tests check
 * that, and check both against the committed fixtures in tests/golden/.
 *
 * Index widths: row pointers are int64 so the checker can also read the
 * product's device layouts; column indices are int32 like the reference.
 */
#ifndef SFEEC_ORACLE_H
#define SFEEC_ORACLE_H
#include <stdint.h>

typedef struct {
  int64_t rows, cols;
  const int64_t* row_ptr; /* rows + 1 */
  const int32_t* col_idx;
  const double* val;
} or_csr;

/* splitmix64, core.hpp:44-63 */
uint64_t or_rng_next_u64(uint64_t* state);
double or_rng_uniform(uint64_t* state, double lo, double hi);
void or_rng_fill_uniform(uint64_t seed, double lo, double hi, double* out, int64_t n);

/* y = A x, sparse.cpp:96-104 */
void or_spmv(const or_csr* a, const double* x, double* y);

/* COO -> CSR, sparse.cpp:20-61: stable (row, col) sort, duplicates summed in
 * input order, exact zeros dropped. Returns nnz; call with NULL outputs first
 * to size them. */
int64_t or_from_triplets(int64_t rows, int64_t n, const int32_t* r, const int32_t* c,
                         const double* v, int64_t* row_ptr, int32_t* col_idx, double* val);

/* Q_sym = Q/2 + Q^T/2, dynamics.cpp:10-25 (same triplet order). Returns nnz. */
int64_t or_symmetric_part(const or_csr* q, int64_t* row_ptr, int32_t* col_idx, double* val);

/* transpose, sparse.cpp:75-94 */
void or_transpose(const or_csr* a, int64_t* row_ptr, int32_t* col_idx, double* val);

typedef struct {
  int strang;      /* SplitKind: 1 Strang, 0 LieTrotter */
  int be;          /* Formulation: 1 BE (b, e), 0 AE (a, e) */
  double dt, eps0, mu0;
  or_csr q_sym, c, ct, m2;
  const or_csr* div; /* nullable */
} or_scheme;

/* dynamics.cpp:47-55 */
void or_flow_he(const or_scheme* s, double* first, double* e, double dt);
/* dynamics.cpp:57-67 */
void or_flow_ha(const or_scheme* s, double* first, double* e, double dt);
/* dynamics.cpp:69-90 (without the CFL warning), repeated nsteps times; if
 * energy_hist != NULL it receives or_energy after every step. */
void or_steps(const or_scheme* s, double* first, double* e, int64_t nsteps,
              double* energy_hist);
/* dynamics.cpp:92-102 */
double or_energy(const or_scheme* s, const double* first, const double* e);
/* dynamics.cpp:104-112 (BE only; 0 when no div) */
double or_gauss_residual(const or_scheme* s, const double* b);
/* dynamics.cpp:114-133 */
double or_cfl_number(const or_scheme* s);

/* Yee FDTD, yee.cpp:9-74: component-major arrays of 3*nx*ny*nz, periodic. */
void or_yee_advance_e(int nx, int ny, int nz, const double d[3], double* e, const double* b,
                      double dt, double c2);
void or_yee_advance_b(int nx, int ny, int nz, const double d[3], const double* e, double* b,
                      double dt);

#endif
