// DOF numbering and HBM storage of the structured (Yee / lumped-mass SFEEC)
// path. Shared by the host builders (host_yee.cpp) and the kernels (yee.cu).
//
// Storage: six component arrays (Ex, Ey, Ez, Bx, By, Bz), each of np_alloc
// elements with index s(i,j,k) = i + P0*(j + Y*k), i fastest (P0 = row pitch).
//   periodic: X,Y,Z = nx,ny,nz; the SFEEC numbering is a*N + s(i,j,k), i.e.
//             exactly the reference's axis-major ids (mesh_cubical.cpp:11-14,
//             52-53) and YeeGrid's component-major arrays (yee.hpp:15-17).
//   PEC:      X,Y,Z = nx+1,ny+1,nz+1 (vertex-aligned); boundary edges are not
//             DOFs and stay 0 in storage; every face is a DOF.
// PEC SFEEC numbering (documented in DESIGN.md): axis-major blocks; inside
// an axis block, lexicographic (i fastest) over the DOF ranges
//   edge a: coord a in [0, n_a), other coords in [1, n_d - 1]
//   face a: coord a in [0, n_a], other coords in [0, n_d - 1]
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define SFEEC_HD __host__ __device__ __forceinline__
#else
#define SFEEC_HD inline
#endif

namespace sfeec_b200 {

struct YeeGeom {
  int n[3];
  int bc;   // SFEEC_BC_PERIODIC / SFEEC_BC_PEC
  int S[3]; // storage extents X, Y, Z
  int P0;   // row pitch (elements) >= S[0]; PEC rows padded to 16-byte multiples for TMA
  int64_t np_alloc;  // elements per component array (padded to a multiple of 32)
  // z-slab decomposition (multi-GPU): global k = local storage plane + kofs;
  // local planes [kown_lo, kown_hi) hold this slab's DOFs, the others are
  // ghost planes refreshed by the halo exchange. Single domain: kofs = 0,
  // owned = [0, S[2]).
  int kofs, kown_lo, kown_hi;
  int64_t edge_off[4], face_off[4];

  SFEEC_HD int64_t npts() const { return np_alloc; }
  SFEEC_HD int64_t sidx(int i, int j, int k) const {
    return (int64_t)i + (int64_t)P0 * ((int64_t)j + (int64_t)S[1] * k);
  }
  // DOF range of component a: lo[d], ext[d]
  SFEEC_HD void range(bool face, int a, int lo[3], int ext[3]) const {
    for (int d = 0; d < 3; ++d) {
      if (bc == 0) {
        lo[d] = 0;
        ext[d] = n[d];
      } else if (face) {
        lo[d] = 0;
        ext[d] = d == a ? n[d] + 1 : n[d];
      } else {
        lo[d] = d == a ? 0 : 1;
        ext[d] = d == a ? n[d] : n[d] - 1;
      }
      if (ext[d] < 0) ext[d] = 0;
    }
    // restrict z to the owned planes, in local storage coordinates
    int zlo = lo[2] > kown_lo + kofs ? lo[2] : kown_lo + kofs;
    int zhi = lo[2] + ext[2] < kown_hi + kofs ? lo[2] + ext[2] : kown_hi + kofs;
    lo[2] = zlo - kofs;
    ext[2] = zhi > zlo ? zhi - zlo : 0;
  }
  SFEEC_HD void init_offsets() {
    for (int f = 0; f < 2; ++f) {
      int64_t* off = f ? face_off : edge_off;
      off[0] = 0;
      for (int a = 0; a < 3; ++a) {
        int lo[3], ext[3];
        range(f == 1, a, lo, ext);
        off[a + 1] = off[a] + (int64_t)ext[0] * ext[1] * ext[2];
      }
    }
  }
  // DOF id -> (component axis, storage index)
  SFEEC_HD void dof_to_storage(bool face, int64_t id, int& a, int64_t& s) const {
    const int64_t* off = face ? face_off : edge_off;
    a = id < off[1] ? 0 : (id < off[2] ? 1 : 2);
    int lo[3], ext[3];
    range(face, a, lo, ext);
    int64_t l = id - off[a];
    int i = (int)(l % ext[0]);
    int64_t r = l / ext[0];
    int j = (int)(r % ext[1]);
    int k = (int)(r / ext[1]);
    s = sidx(i + lo[0], j + lo[1], k + lo[2]);
  }
  // storage coords -> DOF id or -1
  SFEEC_HD int64_t dof_id(bool face, int a, int i, int j, int k) const {
    int lo[3], ext[3];
    range(face, a, lo, ext);
    int c[3] = {i - lo[0], j - lo[1], k - lo[2]};
    for (int d = 0; d < 3; ++d)
      if (c[d] < 0 || c[d] >= ext[d]) return -1;
    const int64_t* off = face ? face_off : edge_off;
    return off[a] + c[0] + (int64_t)ext[0] * (c[1] + (int64_t)ext[1] * c[2]);
  }
};

inline YeeGeom make_yee_geom(int nx, int ny, int nz, int bc) {
  YeeGeom g;
  g.n[0] = nx;
  g.n[1] = ny;
  g.n[2] = nz;
  g.bc = bc;
  for (int d = 0; d < 3; ++d) g.S[d] = bc ? g.n[d] + 1 : g.n[d];
  g.P0 = bc ? (g.S[0] + 7) / 8 * 8 : g.S[0];
  g.np_alloc = ((int64_t)g.P0 * g.S[1] * g.S[2] + 31) / 32 * 32;
  g.kofs = 0;
  g.kown_lo = 0;
  g.kown_hi = g.S[2];
  g.init_offsets();
  return g;
}

// Slab r of R of a PEC lattice with nz global cells (nz divisible by R):
// local storage planes 0 (ghost below), 1..nzl (owned), nzl+1 (ghost above;
// on the last slab this is the global top wall plane, owned and constant).
// ghost planes per side of a slab: 2, so the two-step sweep (two leapfrog
// steps per pass, yee.cu k_fused2_tma) has its halo; the one-step kernels
// read only the inner ghost plane
inline constexpr int kYeeGhost = 2;

inline YeeGeom make_yee_slab(int nx, int ny, int nz, int r, int R, int G = kYeeGhost) {
  YeeGeom g = make_yee_geom(nx, ny, nz, 1);
  const int nzl = nz / R;
  g.S[2] = nzl + 2 * G;
  g.np_alloc = ((int64_t)g.P0 * g.S[1] * g.S[2] + 31) / 32 * 32;
  g.kofs = r * nzl - G;
  g.kown_lo = G;
  g.kown_hi = (r == R - 1) ? G + nzl + 1 : G + nzl;  // the last slab owns the top wall
  g.init_offsets();
  return g;
}

}  // namespace sfeec_b200
