/* TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Plain-C restatement of the 3-D Kuhn/Freudenthal construction of configs
 * 1, 3 and 5 (C, D, M1, M2, the S(M1) SPAI and Q_sym), written from the
 * construction contract in DESIGN.md 3.2 and independent of the product's
 * C++ (csrc/host_tet.cpp, csrc/tet_device.cu). It is the fast (OpenMP)
 * companion of the numpy restatement oracle/tetmesh_oracle.py, used
 *   * by tests/ to check the device-assembled operators at full size
 *     (128^3: structure and M1/M2/C/D values bitwise, Q_sym to a tolerance),
 *   * by bench.py's reference arm to build the operators the UNMODIFIED
 *     reference SplitScheme::step (oracle/_ref) is timed on, so that arm
 *     maps no product library.
 *
 * Parity status: the reference has no 3-D tets; this file is
 * pinned bitwise against oracle/tetmesh_oracle.py (numbering, signs, patterns,
 * masses) and, for the SPAI values, against a numpy least-squares solve.
 * The reference conventions it follows:
 *   ascending-vertex-id orientation      mesh_simplicial.cpp:16-38
 *   integral DOFs -> +-1 incidence        operators.cpp:29-42 (P1 branch)
 *   mass assembly: element contributions summed per (row, col) in ascending
 *   cell order from 0.0, exact zeros dropped   operators.cpp:133-179,
 *                                              sparse.cpp:20-61
 *   S(M1) pattern = rows of M1            spai.cpp:31-72
 *   SPAI normal equations, Gram = (M^2)(I, I) with k ascending, rhs = M(l, I),
 *   pivot threshold 1e-12 * trace         spai.cpp:141-233
 *   Q(I, l) = q_l, Q_sym = Q/2 + Q^T/2    spai.cpp:258-268, dynamics.cpp:10-25
 * The SPAI solve here is an unpivoted LDL^T (the reference uses Eigen's LDLT,
 * which is absent), so Q values agree to rounding, not bitwise. A column that
 * fails the pivot test is counted and left to the caller (the reference's
 * eigen fallback is not restated; the configs never need it).
 * Build: oracle/Makefile, -ffp-contract=off (separate multiply and add). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t rows, cols, nnz;
  int64_t* rp;
  int32_t* ci;
  double* v;
} to_csr;

/* edge types (offsets in {0,1}^3), face types (pairs of edge types t1 < t2
 * with t1's offset a subset of t2's), Kuhn permutations, local sub-simplices */
static const int ET[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0},
                             {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
static const int FT[12][2] = {{0, 3}, {1, 3}, {1, 4}, {2, 4}, {0, 5}, {2, 5},
                              {0, 6}, {1, 6}, {2, 6}, {3, 6}, {4, 6}, {5, 6}};
static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int LF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
#define BLOCK 32
#define MAXW 64

typedef struct {
  int n;
  int64_t nv, ne, nf, nt;
  double* xyz;     /* 3 nv */
  int32_t* eid;    /* 7 nv: DOF id of edge (v, type) or -1 */
  int32_t* fid;    /* 12 nv */
  int64_t* ebase;  /* per DOF edge: base vertex * 8 + type */
  int64_t* fbase;  /* per face: base vertex * 16 + type */
} tmesh;

/* k-th output (0-based) of splitmix64 seeded with `seed` (core.hpp:44-63) */
static uint64_t smix(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static int64_t vidx(int n, int i, int j, int k) {
  return (int64_t)i + (int64_t)(n + 1) * ((int64_t)j + (int64_t)(n + 1) * k);
}
static void vcoord(int n, int64_t v, int c[3]) {
  c[0] = (int)(v % (n + 1));
  c[1] = (int)((v / (n + 1)) % (n + 1));
  c[2] = (int)(v / ((int64_t)(n + 1) * (n + 1)));
}
static int etype(const int d[3]) {
  for (int t = 0; t < 7; ++t)
    if (ET[t][0] == d[0] && ET[t][1] == d[1] && ET[t][2] == d[2]) return t;
  return -1;
}

static void mesh_free(tmesh* m) {
  free(m->xyz);
  free(m->eid);
  free(m->fid);
  free(m->ebase);
  free(m->fbase);
}

static int mesh_build(tmesh* m, int n, double jitter, uint64_t seed) {
  memset(m, 0, sizeof(*m));
  m->n = n;
  const int64_t N = n + 1;
  m->nv = N * N * N;
  m->nt = 6 * (int64_t)n * n * n;
  m->xyz = (double*)malloc(sizeof(double) * 3 * m->nv);
  m->eid = (int32_t*)malloc(sizeof(int32_t) * 7 * m->nv);
  m->fid = (int32_t*)malloc(sizeof(int32_t) * 12 * m->nv);
  if (!m->xyz || !m->eid || !m->fid) return -1;
  const double h = 1.0 / n;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < m->nv; ++v) {
    int c[3];
    vcoord(n, v, c);
    const int inner = c[0] > 0 && c[0] < n && c[1] > 0 && c[1] < n && c[2] > 0 && c[2] < n;
    for (int d = 0; d < 3; ++d) {
      double x = (double)c[d] * h;
      if (inner && jitter > 0) {
        const double u = (double)(smix(seed, (uint64_t)(3 * v + d)) >> 11) * 0x1.0p-53;
        x = x + (jitter * h) * (2.0 * u - 1.0);
      }
      m->xyz[3 * v + d] = x;
    }
  }
  for (int64_t s = 0; s < 7 * m->nv; ++s) m->eid[s] = -1;
  for (int64_t s = 0; s < 12 * m->nv; ++s) m->fid[s] = -1;
  /* DOF order: vertex plane k, row j, 32-vertex block along x, entity type,
   * then i; PEC drops edges on a wall they lie in (an axis d with zero
   * offset and the base coordinate on that axis 0 or n) */
  int64_t ne = 0, nf = 0;
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n; ++j)
      for (int ib = 0; ib <= n; ib += BLOCK) {
        const int ie = ib + BLOCK < n + 1 ? ib + BLOCK : n + 1;
        for (int t = 0; t < 7; ++t)
          for (int i = ib; i < ie; ++i) {
            const int c[3] = {i, j, k};
            int ok = 1;
            for (int d = 0; d < 3; ++d) {
              if (c[d] + ET[t][d] > n) ok = 0;
              if (ET[t][d] == 0 && (c[d] == 0 || c[d] == n)) ok = 0;
            }
            if (ok) m->eid[7 * vidx(n, i, j, k) + t] = (int32_t)ne++;
          }
        for (int f = 0; f < 12; ++f)
          for (int i = ib; i < ie; ++i) {
            const int* o = ET[FT[f][1]];
            if (i + o[0] > n || j + o[1] > n || k + o[2] > n) continue;
            m->fid[12 * vidx(n, i, j, k) + f] = (int32_t)nf++;
          }
      }
  m->ne = ne;
  m->nf = nf;
  m->ebase = (int64_t*)malloc(sizeof(int64_t) * (ne ? ne : 1));
  m->fbase = (int64_t*)malloc(sizeof(int64_t) * (nf ? nf : 1));
  if (!m->ebase || !m->fbase) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < m->nv; ++v) {
    for (int t = 0; t < 7; ++t)
      if (m->eid[7 * v + t] >= 0) m->ebase[m->eid[7 * v + t]] = v * 8 + t;
    for (int f = 0; f < 12; ++f)
      if (m->fid[12 * v + f] >= 0) m->fbase[m->fid[12 * v + f]] = v * 16 + f;
  }
  return 0;
}

/* the four (ascending) vertex ids of tet 6 * cube + p */
static void tet_verts(int n, int64_t tet, int64_t vv[4]) {
  const int64_t cube = tet / 6;
  const int p = (int)(tet % 6);
  int c[3] = {(int)(cube % n), (int)((cube / n) % n), (int)(cube / ((int64_t)n * n))};
  vv[0] = vidx(n, c[0], c[1], c[2]);
  for (int s = 0; s < 3; ++s) {
    c[PERM[p][s]] += 1;
    vv[s + 1] = vidx(n, c[0], c[1], c[2]);
  }
}

/* edge DOF id of vertices a < b (-1: a PEC wall edge) */
static int32_t edge_id(const tmesh* m, int64_t a, int64_t b) {
  int ca[3], cb[3];
  vcoord(m->n, a, ca);
  vcoord(m->n, b, cb);
  const int d[3] = {cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2]};
  return m->eid[7 * a + etype(d)];
}
static int32_t face_id(const tmesh* m, int64_t a, int64_t b, int64_t c) {
  int ca[3], cb[3], cc[3];
  vcoord(m->n, a, ca);
  vcoord(m->n, b, cb);
  vcoord(m->n, c, cc);
  const int d1[3] = {cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2]};
  const int d2[3] = {cc[0] - ca[0], cc[1] - ca[1], cc[2] - ca[2]};
  const int t1 = etype(d1), t2 = etype(d2);
  for (int f = 0; f < 12; ++f)
    if (FT[f][0] == t1 && FT[f][1] == t2) return m->fid[12 * a + f];
  return -1;
}

/* tets (ascending ids) having all of the vertices vs[0..k) (vs[0] the lowest):
 * they lie in the <= 8 cubes whose corner is vs[0] - (dx, dy, dz) */
static int tets_with(const tmesh* m, const int64_t* vs, int k, int64_t out[24]) {
  const int n = m->n;
  int c0[3];
  vcoord(n, vs[0], c0);
  int cnt = 0;
  for (int dz = 1; dz >= 0; --dz)
    for (int dy = 1; dy >= 0; --dy)
      for (int dx = 1; dx >= 0; --dx) {
        const int w[3] = {c0[0] - dx, c0[1] - dy, c0[2] - dz};
        if (w[0] < 0 || w[1] < 0 || w[2] < 0 || w[0] >= n || w[1] >= n || w[2] >= n) continue;
        const int64_t cube = (int64_t)w[0] + (int64_t)n * ((int64_t)w[1] + (int64_t)n * w[2]);
        for (int p = 0; p < 6; ++p) {
          int64_t vv[4];
          tet_verts(n, cube * 6 + p, vv);
          int all = 1;
          for (int q = 0; q < k; ++q)
            all = all && (vs[q] == vv[0] || vs[q] == vv[1] || vs[q] == vv[2] || vs[q] == vv[3]);
          if (all) out[cnt++] = cube * 6 + p;
        }
      }
  return cnt;
}

static void cross3(const double* u, const double* v, double* w) {
  w[0] = u[1] * v[2] - u[2] * v[1];
  w[1] = u[2] * v[0] - u[0] * v[2];
  w[2] = u[0] * v[1] - u[1] * v[0];
}

/* Whitney P1- element matrices: with barycentric gradients
 * gl and L_ab = int lambda_a lambda_b = |T| (1 + delta_ab) / 20,
 *   M1[(i,j),(k,l)] = L_ik g_jl - L_il g_jk - L_jk g_il + L_jl g_ik,
 *   M2[f,h] = 4 sum_{s,t} L_{a_s b_t} (grad l x grad l)_s . (grad l x grad l)_t
 * with w_f = 2 sum_cyc lambda_a grad lambda_b x grad lambda_c. Each entry is
 * evaluated once for the upper triangle and mirrored (exact symmetry). */
static void element(const tmesh* m, int64_t tet, double m1[6][6], double m2[4][4]) {
  int64_t vv[4];
  tet_verts(m->n, tet, vv);
  double x[4][3], e[3][3];
  for (int a = 0; a < 4; ++a)
    for (int d = 0; d < 3; ++d) x[a][d] = m->xyz[3 * vv[a] + d];
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d) e[a][d] = x[a + 1][d] - x[0][d];
  double c12[3], c20[3], c01[3], gl[4][3];
  cross3(e[1], e[2], c12);
  cross3(e[2], e[0], c20);
  cross3(e[0], e[1], c01);
  const double vol6 = e[0][0] * c12[0] + e[0][1] * c12[1] + e[0][2] * c12[2];
  for (int d = 0; d < 3; ++d) {
    gl[1][d] = c12[d] / vol6;
    gl[2][d] = c20[d] / vol6;
    gl[3][d] = c01[d] / vol6;
    gl[0][d] = -((gl[1][d] + gl[2][d]) + gl[3][d]);
  }
  const double vol = fabs(vol6) / 6.0;
  double L[4][4], g[4][4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      L[a][b] = a == b ? vol / 10.0 : vol / 20.0;
      g[a][b] = (gl[a][0] * gl[b][0] + gl[a][1] * gl[b][1]) + gl[a][2] * gl[b][2];
    }
  if (m1)
    for (int p = 0; p < 6; ++p)
      for (int q = p; q < 6; ++q) {
        const int i = LE[p][0], j = LE[p][1], k = LE[q][0], l = LE[q][1];
        double s = L[i][k] * g[j][l];
        s = s - L[i][l] * g[j][k];
        s = s - L[j][k] * g[i][l];
        s = s + L[j][l] * g[i][k];
        m1[p][q] = m1[q][p] = s;
      }
  if (m2) {
    double cv[4][3][3];
    int ci[4][3];
    for (int f = 0; f < 4; ++f) {
      const int a = LF[f][0], b = LF[f][1], c = LF[f][2];
      const int cyc[3][3] = {{a, b, c}, {b, c, a}, {c, a, b}};
      for (int t = 0; t < 3; ++t) {
        ci[f][t] = cyc[t][0];
        cross3(gl[cyc[t][1]], gl[cyc[t][2]], cv[f][t]);
      }
    }
    for (int f = 0; f < 4; ++f)
      for (int h = f; h < 4; ++h) {
        double acc = 0.0;
        for (int s = 0; s < 3; ++s)
          for (int t = 0; t < 3; ++t) {
            const double dot = (cv[f][s][0] * cv[h][t][0] + cv[f][s][1] * cv[h][t][1]) +
                               cv[f][s][2] * cv[h][t][2];
            acc = acc + L[ci[f][s]][ci[h][t]] * dot;
          }
        acc = 4.0 * acc;
        m2[f][h] = m2[h][f] = acc;
      }
  }
}

/* sorted (column, value) accumulator of one row */
typedef struct {
  int w;
  int32_t c[MAXW];
  double v[MAXW];
} rowacc;
static void acc_add(rowacc* r, int32_t c, double v) {
  int lo = 0, hi = r->w;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (r->c[mid] < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < r->w && r->c[lo] == c) {
    r->v[lo] = r->v[lo] + v;
    return;
  }
  if (r->w >= MAXW) abort();
  memmove(r->c + lo + 1, r->c + lo, sizeof(int32_t) * (r->w - lo));
  memmove(r->v + lo + 1, r->v + lo, sizeof(double) * (r->w - lo));
  r->c[lo] = c;
  r->v[lo] = 0.0 + v;
  r->w++;
}
static void acc_drop_zeros(rowacc* r) {
  int o = 0;
  for (int s = 0; s < r->w; ++s)
    if (r->v[s] != 0.0) {
      r->c[o] = r->c[s];
      r->v[o] = r->v[s];
      ++o;
    }
  r->w = o;
}

/* one row of operator `which` (0 C, 1 D, 2 M1, 3 M2) */
static void make_row(const tmesh* m, int which, int64_t r, rowacc* out) {
  const int n = m->n;
  out->w = 0;
  if (which == 0 || which == 3) { /* faces */
    const int64_t v = m->fbase[r] >> 4;
    const int f = (int)(m->fbase[r] & 15);
    int c[3];
    vcoord(n, v, c);
    const int* o1 = ET[FT[f][0]];
    const int* o2 = ET[FT[f][1]];
    const int64_t fv[3] = {v, vidx(n, c[0] + o1[0], c[1] + o1[1], c[2] + o1[2]),
                           vidx(n, c[0] + o2[0], c[1] + o2[1], c[2] + o2[2])};
    if (which == 0) { /* boundary of [v0, v1, v2]: [v1,v2] - [v0,v2] + [v0,v1] */
      const int64_t pr[3][2] = {{fv[1], fv[2]}, {fv[0], fv[2]}, {fv[0], fv[1]}};
      const double sg[3] = {1.0, -1.0, 1.0};
      for (int s = 0; s < 3; ++s) {
        const int32_t e = edge_id(m, pr[s][0], pr[s][1]);
        if (e >= 0) acc_add(out, e, sg[s]);
      }
      acc_drop_zeros(out);
      return;
    }
    int64_t tt[24];
    const int nt = tets_with(m, fv, 3, tt);
    for (int s = 0; s < nt; ++s) {
      int64_t vv[4];
      tet_verts(n, tt[s], vv);
      int me = -1;
      for (int h = 0; h < 4; ++h)
        if (vv[LF[h][0]] == fv[0] && vv[LF[h][1]] == fv[1] && vv[LF[h][2]] == fv[2]) me = h;
      double e2[4][4];
      element(m, tt[s], NULL, e2);
      for (int h = 0; h < 4; ++h)
        acc_add(out, face_id(m, vv[LF[h][0]], vv[LF[h][1]], vv[LF[h][2]]), e2[me][h]);
    }
    acc_drop_zeros(out);
    return;
  }
  if (which == 1) { /* D: tet r -> +f0 - f1 + f2 - f3 */
    int64_t vv[4];
    tet_verts(n, r, vv);
    const double sg[4] = {1.0, -1.0, 1.0, -1.0};
    for (int h = 0; h < 4; ++h)
      acc_add(out, face_id(m, vv[LF[h][0]], vv[LF[h][1]], vv[LF[h][2]]), sg[h]);
    acc_drop_zeros(out);
    return;
  }
  /* M1 row of edge r */
  const int64_t v = m->ebase[r] >> 3;
  const int t = (int)(m->ebase[r] & 7);
  int c[3];
  vcoord(n, v, c);
  const int64_t ev[2] = {v, vidx(n, c[0] + ET[t][0], c[1] + ET[t][1], c[2] + ET[t][2])};
  int64_t tt[24];
  const int nt = tets_with(m, ev, 2, tt);
  for (int s = 0; s < nt; ++s) {
    int64_t vv[4];
    tet_verts(n, tt[s], vv);
    int me = -1;
    for (int q = 0; q < 6; ++q)
      if (vv[LE[q][0]] == ev[0] && vv[LE[q][1]] == ev[1]) me = q;
    double e1[6][6];
    element(m, tt[s], e1, NULL);
    for (int q = 0; q < 6; ++q) {
      const int32_t col = edge_id(m, vv[LE[q][0]], vv[LE[q][1]]);
      if (col >= 0) acc_add(out, col, e1[me][q]);
    }
  }
  acc_drop_zeros(out);
}

static int assemble(const tmesh* m, int which, to_csr* out) {
  const int64_t rows = which == 1 ? m->nt : (which == 2 ? m->ne : m->nf);
  out->rows = rows;
  out->cols = which == 0 || which == 2 ? m->ne : m->nf;
  out->rp = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  if (!out->rp) return -1;
#pragma omp parallel
  {
    rowacc r;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t i = 0; i < rows; ++i) {
      make_row(m, which, i, &r);
      out->rp[i + 1] = r.w;
    }
  }
  for (int64_t i = 0; i < rows; ++i) out->rp[i + 1] += out->rp[i];
  out->nnz = out->rp[rows];
  out->ci = (int32_t*)malloc(sizeof(int32_t) * (size_t)(out->nnz ? out->nnz : 1));
  out->v = (double*)malloc(sizeof(double) * (size_t)(out->nnz ? out->nnz : 1));
  if (!out->ci || !out->v) return -1;
#pragma omp parallel
  {
    rowacc r;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t i = 0; i < rows; ++i) {
      make_row(m, which, i, &r);
      memcpy(out->ci + out->rp[i], r.c, sizeof(int32_t) * r.w);
      memcpy(out->v + out->rp[i], r.v, sizeof(double) * r.w);
    }
  }
  return 0;
}

/* value of a(r, c) (0 if absent) */
static double entry_of(const to_csr* a, int64_t r, int32_t c, int64_t* pos) {
  int64_t lo = a->rp[r], hi = a->rp[r + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (a->ci[mid] < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (pos) *pos = lo;
  return lo < a->rp[r + 1] && a->ci[lo] == c ? a->v[lo] : 0.0;
}

/* S(M1) SPAI columns (values aligned with M1's CSR: q_l over pattern row l),
 * normal equations solved by LDL^T; returns the count of columns that failed
 * the pivot test (left zero) */
static int64_t spai_columns(const to_csr* m1, double* qcol) {
  int64_t failed = 0;
#pragma omp parallel reduction(+ : failed)
  {
    double G[MAXW * MAXW], Lm[MAXW * MAXW], d[MAXW], rhs[MAXW], y[MAXW], w[MAXW];
#pragma omp for schedule(dynamic, 256)
    for (int64_t l = 0; l < m1->rows; ++l) {
      const int64_t b = m1->rp[l];
      const int k = (int)(m1->rp[l + 1] - b);
      const int32_t* I = m1->ci + b;
      double trace = 0.0;
      for (int a = 0; a < k; ++a)
        for (int c = a; c < k; ++c) {
          /* (M^2)(I_a, I_c) = sum over the common columns, ascending */
          int64_t p = m1->rp[I[a]], pe = m1->rp[I[a] + 1];
          int64_t q = m1->rp[I[c]], qe = m1->rp[I[c] + 1];
          double s = 0.0;
          while (p < pe && q < qe) {
            if (m1->ci[p] == m1->ci[q]) {
              s = s + m1->v[p] * m1->v[q];
              ++p;
              ++q;
            } else if (m1->ci[p] < m1->ci[q]) {
              ++p;
            } else {
              ++q;
            }
          }
          G[a * k + c] = G[c * k + a] = s;
        }
      for (int a = 0; a < k; ++a) {
        trace += G[a * k + a];
        rhs[a] = entry_of(m1, l, I[a], NULL);
      }
      /* G = L D L^T, unit lower L */
      double dmin = INFINITY;
      for (int j = 0; j < k; ++j) {
        for (int p = 0; p < j; ++p) w[p] = Lm[j * k + p] * d[p];
        double dj = G[j * k + j];
        for (int p = 0; p < j; ++p) dj -= Lm[j * k + p] * w[p];
        d[j] = dj;
        if (dj < dmin) dmin = dj;
        for (int i = j + 1; i < k; ++i) {
          double s = G[i * k + j];
          for (int p = 0; p < j; ++p) s -= Lm[i * k + p] * w[p];
          Lm[i * k + j] = s / dj;
        }
      }
      double* q = qcol + b;
      if (!(dmin > 1e-12 * trace)) {
        for (int a = 0; a < k; ++a) q[a] = 0.0;
        failed += 1;
        continue;
      }
      for (int i = 0; i < k; ++i) { /* L y = rhs */
        double s = rhs[i];
        for (int p = 0; p < i; ++p) s -= Lm[i * k + p] * y[p];
        y[i] = s;
      }
      for (int i = 0; i < k; ++i) y[i] = y[i] / d[i];
      for (int i = k - 1; i >= 0; --i) { /* L^T q = y */
        double s = y[i];
        for (int p = i + 1; p < k; ++p) s -= Lm[p * k + i] * q[p];
        q[i] = s;
      }
    }
  }
  return failed;
}

/* Q_sym(r, c) = Q(r, c)/2 + Q(c, r)/2 on the (symmetric) S(M1) pattern, with
 * Q(r, c) = q_c[r]: the two halves of the reference's triplet sum (a + b is
 * exact-commutative, so the order does not matter); exact zeros dropped */
static int qsym_from_columns(const to_csr* m1, const double* qcol, to_csr* out) {
  const int64_t n = m1->rows;
  out->rows = out->cols = n;
  out->rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(m1->nnz ? m1->nnz : 1));
  if (!out->rp || !tmp) return -1;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    int64_t cnt = 0;
    for (int64_t s = m1->rp[r]; s < m1->rp[r + 1]; ++s) {
      const int32_t c = m1->ci[s];
      int64_t pos = 0;
      entry_of(m1, c, (int32_t)r, &pos); /* r sits in pattern column c at pos */
      const double v = 0.0 + 0.5 * qcol[s] + 0.5 * qcol[pos];
      tmp[s] = v;
      cnt += v != 0.0;
    }
    out->rp[r + 1] = cnt;
  }
  for (int64_t r = 0; r < n; ++r) out->rp[r + 1] += out->rp[r];
  out->nnz = out->rp[n];
  out->ci = (int32_t*)malloc(sizeof(int32_t) * (size_t)(out->nnz ? out->nnz : 1));
  out->v = (double*)malloc(sizeof(double) * (size_t)(out->nnz ? out->nnz : 1));
  if (!out->ci || !out->v) {
    free(tmp);
    return -1;
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    int64_t o = out->rp[r];
    for (int64_t s = m1->rp[r]; s < m1->rp[r + 1]; ++s)
      if (tmp[s] != 0.0) {
        out->ci[o] = m1->ci[s];
        out->v[o] = tmp[s];
        ++o;
      }
  }
  free(tmp);
  return 0;
}

void to_free(to_csr* a) {
  if (!a) return;
  free(a->rp);
  free(a->ci);
  free(a->v);
  a->rp = NULL;
  a->ci = NULL;
  a->v = NULL;
}

/* want: bit 0 C, 1 D, 2 M1, 3 M2, 4 Q_sym (S(M1) SPAI). counts = {N1, N2, T,
 * SPAI columns that failed the pivot test}. Returns 0, or -1 on allocation
 * failure / bad arguments. */
int to_build(int n, double jitter, uint64_t seed, int want, to_csr* c, to_csr* d, to_csr* m1,
             to_csr* m2, to_csr* qsym, int64_t* counts) {
  if (n < 1 || !(jitter >= 0 && jitter < 0.25)) return -1;
  tmesh m;
  if (mesh_build(&m, n, jitter, seed)) {
    mesh_free(&m);
    return -1;
  }
  int rc = 0;
  to_csr mm1 = {0};
  if (counts) {
    counts[0] = m.ne;
    counts[1] = m.nf;
    counts[2] = m.nt;
    counts[3] = 0;
  }
  if (!rc && (want & 1)) rc = assemble(&m, 0, c);
  if (!rc && (want & 2)) rc = assemble(&m, 1, d);
  if (!rc && (want & 8)) rc = assemble(&m, 3, m2);
  if (!rc && (want & (4 | 16))) rc = assemble(&m, 2, &mm1);
  if (!rc && (want & 16)) {
    double* qcol = (double*)malloc(sizeof(double) * (size_t)(mm1.nnz ? mm1.nnz : 1));
    if (!qcol) rc = -1;
    if (!rc) {
      const int64_t failed = spai_columns(&mm1, qcol);
      if (counts) counts[3] = failed;
      rc = qsym_from_columns(&mm1, qcol, qsym);
    }
    free(qcol);
  }
  if (!rc && (want & 4))
    *m1 = mm1;
  else
    to_free(&mm1);
  mesh_free(&m);
  return rc;
}
