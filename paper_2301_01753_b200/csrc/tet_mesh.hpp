// Host-side Kuhn/Freudenthal tet mesh (numbering, geometry, element
// matrices) shared by the host builders (host_tet.cpp) and the device
// assembly (tet_device.cu). Contract: DESIGN.md 3.2.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace sfeec_b200 {

namespace tetc {

// edge types: offsets in {0,1}^3 \ {0}
inline constexpr int kET[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0},
                           {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
// face types: chains 0 < t1 < t2 (bit-subset), as edge-type indices
inline constexpr int kFT[12][2] = {{0, 3}, {1, 3}, {1, 4}, {2, 4}, {0, 5}, {2, 5},
                            {0, 6}, {1, 6}, {2, 6}, {3, 6}, {4, 6}, {5, 6}};
// Kuhn tets of a cube: axis permutations (first, second) step
inline constexpr int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
// local edges / faces of a tet (local vertex indices, ascending)
inline constexpr int kLE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
inline constexpr int kLF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
inline constexpr int kBlock = 32;  // vertex block along x used by the DOF numbering

inline uint64_t splitmix(uint64_t seed, uint64_t k) {  // k-th output (0-based), core.hpp:48-53
  uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline double u01(uint64_t seed, uint64_t k) { return (double)(splitmix(seed, k) >> 11) * 0x1.0p-53; }

inline int type_of(int dx, int dy, int dz) {
  for (int t = 0; t < 7; ++t)
    if (kET[t][0] == dx && kET[t][1] == dy && kET[t][2] == dz) return t;
  return -1;
}

}  // namespace tetc

using namespace tetc;

// The Kuhn mesh of an n x n x nzg box of cubes (spacing 1/n; the unit cube
// when nzg = n), or a z-slab of it: local vertex planes 0..nz are the whole
// mesh's planes kz0..kz0+nz. Vertex ids, jitter streams and PEC walls follow
// the whole mesh (a slab's cut planes are not walls), so every entity of a
// slab has the entity ids' relative order, geometry and DOF status of the
// whole mesh -- a slab's complete rows are bitwise the whole mesh's.
struct TetMesh {
  int n = 0;                  // cubes along x and y
  int nz = 0;                 // cubes along z in this (slab of the) mesh
  int nzg = 0;                // cubes along z of the whole mesh
  int kz0 = 0;                // whole-mesh index of local vertex plane 0
  bool wall_lo = true, wall_hi = true;  // local planes 0 / nz are PEC walls
  double amp = 0;
  uint64_t seed = 0;
  int64_t nv = 0, n_edges = 0, n_faces = 0, n_tets = 0;
  std::vector<double> xyz;       // 3 * nv
  std::vector<int32_t> eid;      // nv * 7: interior-edge DOF id or -1
  std::vector<int32_t> fid;      // nv * 12: face id or -1
  std::vector<int64_t> edge_v;   // base vertex of each DOF edge
  std::vector<int8_t> edge_t;    // type of each DOF edge
  std::vector<int64_t> face_v;
  std::vector<int8_t> face_t;

  int64_t vid(int i, int j, int k) const {
    return (int64_t)i + (int64_t)(n + 1) * ((int64_t)j + (int64_t)(n + 1) * k);
  }
  void coords(int64_t v, int c[3]) const {
    c[0] = (int)(v % (n + 1));
    c[1] = (int)((v / (n + 1)) % (n + 1));
    c[2] = (int)(v / ((int64_t)(n + 1) * (n + 1)));
  }
  bool inside(const int c[3]) const {
    return c[0] >= 0 && c[0] <= n && c[1] >= 0 && c[1] <= n && c[2] >= 0 && c[2] <= nz;
  }
  // coordinate c on axis d lies on a PEC wall
  bool on_wall(int d, int c) const {
    if (d < 2) return c == 0 || c == n;
    return (c == 0 && wall_lo) || (c == nz && wall_hi);
  }
  // tet id -> ascending vertex ids
  void tet_vertices(int64_t tet, int64_t vv[4]) const {
    int64_t cube = tet / 6;
    int p = (int)(tet % 6);
    int c[3] = {(int)(cube % n), (int)((cube / n) % n), (int)(cube / ((int64_t)n * n))};
    vv[0] = vid(c[0], c[1], c[2]);  // cubes: n x n x nz, x fastest
    c[kPerm[p][0]] += 1;
    vv[1] = vid(c[0], c[1], c[2]);
    c[kPerm[p][1]] += 1;
    vv[2] = vid(c[0], c[1], c[2]);
    c[kPerm[p][2]] += 1;
    vv[3] = vid(c[0], c[1], c[2]);
  }
  // edge DOF id of the ascending vertex pair (a, b), -1 if boundary
  int32_t edge_of(int64_t a, int64_t b) const {
    int ca[3], cb[3];
    coords(a, ca);
    coords(b, cb);
    int t = type_of(cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2]);
    return eid[(size_t)(a * 7 + t)];
  }
  int32_t face_of(int64_t a, int64_t b, int64_t c) const {
    int ca[3], cb[3], cc[3];
    coords(a, ca);
    coords(b, cb);
    coords(c, cc);
    int t1 = type_of(cb[0] - ca[0], cb[1] - ca[1], cb[2] - ca[2]);
    int t2 = type_of(cc[0] - ca[0], cc[1] - ca[1], cc[2] - ca[2]);
    for (int f = 0; f < 12; ++f)
      if (kFT[f][0] == t1 && kFT[f][1] == t2) return fid[(size_t)(a * 12 + f)];
    return -1;
  }
  // tets containing all of the (ascending) vertices vs[0..m), ascending ids
  int containing_tets(const int64_t* vs, int m, int64_t out[8]) const {
    int c0[3];
    coords(vs[0], c0);
    int cnt = 0;
    for (int dz = 1; dz >= 0; --dz)
      for (int dy = 1; dy >= 0; --dy)
        for (int dx = 1; dx >= 0; --dx) {
          int w[3] = {c0[0] - dx, c0[1] - dy, c0[2] - dz};
          bool ok = true;
          for (int d = 0; d < 3; ++d)
            if (w[d] < 0 || w[d] >= (d < 2 ? n : nz)) ok = false;
          if (!ok) continue;
          int64_t cube = (int64_t)w[0] + (int64_t)n * ((int64_t)w[1] + (int64_t)n * w[2]);
          for (int p = 0; p < 6; ++p) {
            int64_t vv[4];
            tet_vertices(cube * 6 + p, vv);
            bool all = true;
            for (int q = 0; q < m && all; ++q)
              all = vs[q] == vv[0] || vs[q] == vv[1] || vs[q] == vv[2] || vs[q] == vv[3];
            if (all) out[cnt++] = cube * 6 + p;
          }
        }
    return cnt;
  }

  // the unit cube, n^3 cubes
  void build(int n_, double amp_, uint64_t seed_) { build_slab(n_, n_, 0, n_, amp_, seed_); }

  // vertex planes [k0, k1] of the n x n x nzg_ mesh
  void build_slab(int n_, int nzg_, int k0, int k1, double amp_, uint64_t seed_) {
    n = n_;
    nzg = nzg_;
    kz0 = k0;
    nz = k1 - k0;
    wall_lo = k0 == 0;
    wall_hi = k1 == nzg_;
    amp = amp_;
    seed = seed_;
    require(n >= 1 && nzg >= 1, "tet mesh: n must be >= 1");
    require(k0 >= 0 && k1 <= nzg && nz >= 1, "tet mesh: bad slab plane range");
    require(amp >= 0 && amp < 0.25, "tet mesh: jitter amplitude must be in [0, 0.25)");
    nv = (int64_t)(n + 1) * (n + 1) * (nz + 1);
    n_tets = 6 * (int64_t)n * n * nz;
    require(n_tets < ((int64_t)1 << 40), "tet mesh: too large");
    const double h = 1.0 / n;
    xyz.resize((size_t)(3 * nv));
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nv; ++v) {
      int c[3];
      coords(v, c);
      const int kg = c[2] + kz0;  // whole-mesh plane
      const bool interior = c[0] > 0 && c[0] < n && c[1] > 0 && c[1] < n && kg > 0 && kg < nzg;
      // the whole mesh's vertex id keys the jitter stream
      const uint64_t vg = (uint64_t)c[0] + (uint64_t)(n + 1) * ((uint64_t)c[1] + (uint64_t)(n + 1) * kg);
      const int cg[3] = {c[0], c[1], kg};
      for (int d = 0; d < 3; ++d) {
        double x = (double)cg[d] * h;
        if (interior && amp > 0) x = x + (amp * h) * (2.0 * u01(seed, 3 * vg + d) - 1.0);
        xyz[(size_t)(3 * v + d)] = x;
      }
    }
    eid.assign((size_t)(nv * 7), -1);
    fid.assign((size_t)(nv * 12), -1);
    // numbering: (k, j, x-block of 32 vertices, type, i)
    int64_t ne = 0, nf = 0;
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= n; ++j)
        for (int ib = 0; ib <= n; ib += kBlock) {
          const int ie = std::min(ib + kBlock, n + 1);
          for (int t = 0; t < 7; ++t)
            for (int i = ib; i < ie; ++i) {
              int c[3] = {i, j, k}, e[3] = {i + kET[t][0], j + kET[t][1], k + kET[t][2]};
              if (!inside(e)) continue;
              bool bnd = false;
              for (int d = 0; d < 3; ++d)
                if (kET[t][d] == 0 && on_wall(d, c[d])) bnd = true;
              if (bnd) continue;  // PEC: boundary edges are not DOFs
              eid[(size_t)(vid(i, j, k) * 7 + t)] = (int32_t)ne++;
            }
          for (int f = 0; f < 12; ++f)
            for (int i = ib; i < ie; ++i) {
              const int* t2 = kET[kFT[f][1]];
              int e[3] = {i + t2[0], j + t2[1], k + t2[2]};
              if (!inside(e)) continue;
              fid[(size_t)(vid(i, j, k) * 12 + f)] = (int32_t)nf++;
            }
        }
    require(ne < INT32_MAX && nf < INT32_MAX, "tet mesh: DOF count exceeds int32");
    n_edges = ne;
    n_faces = nf;
    edge_v.resize((size_t)ne);
    edge_t.resize((size_t)ne);
    face_v.resize((size_t)nf);
    face_t.resize((size_t)nf);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nv; ++v) {
      for (int t = 0; t < 7; ++t) {
        int32_t e = eid[(size_t)(v * 7 + t)];
        if (e >= 0) {
          edge_v[(size_t)e] = v;
          edge_t[(size_t)e] = (int8_t)t;
        }
      }
      for (int f = 0; f < 12; ++f) {
        int32_t id = fid[(size_t)(v * 12 + f)];
        if (id >= 0) {
          face_v[(size_t)id] = v;
          face_t[(size_t)id] = (int8_t)f;
        }
      }
    }
  }

  void edge_vertices(int64_t e, int64_t out[2]) const {
    int c[3];
    coords(edge_v[(size_t)e], c);
    const int* t = kET[edge_t[(size_t)e]];
    out[0] = edge_v[(size_t)e];
    out[1] = vid(c[0] + t[0], c[1] + t[1], c[2] + t[2]);
  }
  void face_vertices(int64_t f, int64_t out[3]) const {
    int c[3];
    coords(face_v[(size_t)f], c);
    const int* t1 = kET[kFT[face_t[(size_t)f]][0]];
    const int* t2 = kET[kFT[face_t[(size_t)f]][1]];
    out[0] = face_v[(size_t)f];
    out[1] = vid(c[0] + t1[0], c[1] + t1[1], c[2] + t1[2]);
    out[2] = vid(c[0] + t2[0], c[1] + t2[1], c[2] + t2[2]);
  }

  // Whitney P1- element matrices.
  // m1: 6x6 over kLE, m2: 4x4 over kLF; returns 6|T|.
  double element(int64_t tet, double m1[6][6], double m2[4][4]) const {
    int64_t vv[4];
    tet_vertices(tet, vv);
    double x[4][3];
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 3; ++d) x[a][d] = xyz[(size_t)(3 * vv[a] + d)];
    double e[3][3];
    for (int a = 0; a < 3; ++a)
      for (int d = 0; d < 3; ++d) e[a][d] = x[a + 1][d] - x[0][d];
    auto cross = [](const double* u, const double* v, double* w) {
      w[0] = u[1] * v[2] - u[2] * v[1];
      w[1] = u[2] * v[0] - u[0] * v[2];
      w[2] = u[0] * v[1] - u[1] * v[0];
    };
    double c12[3], c20[3], c01[3];
    cross(e[1], e[2], c12);
    cross(e[2], e[0], c20);
    cross(e[0], e[1], c01);
    const double vol6 = e[0][0] * c12[0] + e[0][1] * c12[1] + e[0][2] * c12[2];
    double gl[4][3];
    for (int d = 0; d < 3; ++d) {
      gl[1][d] = c12[d] / vol6;
      gl[2][d] = c20[d] / vol6;
      gl[3][d] = c01[d] / vol6;
      gl[0][d] = -((gl[1][d] + gl[2][d]) + gl[3][d]);
    }
    // ascending-id order is a combinatorial orientation: the odd axis
    // permutations give a negative determinant. |T| enters the integrals.
    const double vol = std::fabs(vol6) / 6.0;
    double ml[4][4], g[4][4];
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        ml[a][b] = a == b ? vol / 10.0 : vol / 20.0;  // int lambda_a lambda_b
        g[a][b] = (gl[a][0] * gl[b][0] + gl[a][1] * gl[b][1]) + gl[a][2] * gl[b][2];
      }
    for (int p = 0; p < 6; ++p)
      for (int q = p; q < 6; ++q) {
        const int i = kLE[p][0], j = kLE[p][1], k = kLE[q][0], l = kLE[q][1];
        double v = ml[i][k] * g[j][l];
        v = v - ml[i][l] * g[j][k];
        v = v - ml[j][k] * g[i][l];
        v = v + ml[j][l] * g[i][k];
        m1[p][q] = v;
        m1[q][p] = v;  // exact symmetric mirror
      }
    // 2-forms: w_f = 2 sum_cyc lambda_i (grad l_j x grad l_k)
    double cv[4][3][3];  // face, term, component
    int ci[4][3];        // face, term -> lambda index
    for (int f = 0; f < 4; ++f) {
      const int a = kLF[f][0], b = kLF[f][1], c = kLF[f][2];
      const int tri[3][3] = {{a, b, c}, {b, c, a}, {c, a, b}};
      for (int t = 0; t < 3; ++t) {
        ci[f][t] = tri[t][0];
        cross(gl[tri[t][1]], gl[tri[t][2]], cv[f][t]);
      }
    }
    for (int f = 0; f < 4; ++f)
      for (int h = f; h < 4; ++h) {
        double acc = 0.0;
        for (int s = 0; s < 3; ++s)
          for (int t = 0; t < 3; ++t) {
            const double dot =
                (cv[f][s][0] * cv[h][t][0] + cv[f][s][1] * cv[h][t][1]) + cv[f][s][2] * cv[h][t][2];
            acc = acc + ml[ci[f][s]][ci[h][t]] * dot;
          }
        acc = 4.0 * acc;
        m2[f][h] = acc;
        m2[h][f] = acc;
      }
    return vol6;
  }
};

}  // namespace sfeec_b200
