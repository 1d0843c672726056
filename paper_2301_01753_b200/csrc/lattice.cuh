// Kuhn-lattice layout of the first-order tet leapfrog (configs 1, 3, 5;
// DESIGN.md 3.4). The DOFs of the k-major numbering live in vertex-lattice
// component arrays instead: e and t as 7 arrays (edge types), b and u as 12
// (face types), each over the (n+3)^3 padded vertex box (one zero halo layer,
// so every stencil read stays in bounds). Non-DOF slots (PEC wall edges,
// faces outside the cube) hold 0 and are never written.
//
// Q_sym and M2 are stored as per-vertex coefficient arrays, one per
// "canonical" stencil slot (lattice_tables.hpp): both operators are exactly
// symmetric, so each off-diagonal pair is stored once and the transposed slot
// reads it at the neighbour's position. C and C^T are structural (+-1 by the
// ascending-vertex orientation) and stream nothing. Column indices are not
// stored at all: the lattice position of a neighbour is its row's position
// plus a constant offset. Per vertex and step: 61 Q and 48 M2 coefficients
// (8 B each) instead of 115 + 84 entries at 12 B in the CSR/sliced layouts.
#pragma once
#include <memory>

#include "device_util.cuh"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

// The padded box of a mesh (TetMesh): x, y vertices 0..n, local z planes
// 0..nz (whole-mesh planes kz0..kz0+nz of an n x n x nzg mesh; a slab of it
// on a multi-rank run). Masks (DOF edges, existing faces) use whole-mesh
// planes, so a slab's cut planes are not walls.
struct LatGeom {
  int n = 0;        // cubes along x, y (vertices 0..n)
  int nz = 0;       // local cubes along z
  int kz0 = 0;      // whole-mesh plane of local plane 0
  int nzg = 0;      // whole-mesh cubes along z
  static constexpr int64_t kPlaneAlign = 256;  // doubles
  int S = 0;        // row pitch: padded vertices along x (n + 3)
  int64_t PS = 0;   // plane pitch: S * (n + 3) rows, rounded up to kPlaneAlign
  int64_t NP = 0;   // the component stride: PS * (nz + 3) planes
  int64_t org = 0;  // position of vertex (0, 0, 0)
  void init(int n_, int nz_, int kz0_, int nzg_) {
    n = n_;
    nz = nz_;
    kz0 = kz0_;
    nzg = nzg_;
    S = n + 3;
    // The plane pitch is rounded up to 2 KB: a block's 256 positions start at a
    // multiple of 256 in the plane, so with an aligned plane every own-position
    // request of a warp (the coefficient streams, the field's own rows) is
    // exactly 8 sectors of 2 lines instead of 9 of 3. Measured on tet256: step
    // 4.88 -> 4.72 ms (32 / 64 / 256 / 1024 doubles: 4.76 / 4.75 / 4.72 / 4.72),
    // bitwise the same state. The row pitch stays n + 3: rounding it to 4 / 8 /
    // 16 doubles measured slower (4.76 / 4.81 / 4.94), and skewing the component
    // stride changes nothing.
    PS = ((int64_t)S * (n + 3) + kPlaneAlign - 1) / kPlaneAlign * kPlaneAlign;
    NP = PS * (nz + 3);
    org = PS + S + 1;
  }
#ifdef __CUDACC__
  __host__ __device__
#endif
  int64_t pos(int i, int j, int k) const { return org + i + (int64_t)S * j + PS * k; }
  // first element of local plane k in a component array
#ifdef __CUDACC__
  __host__ __device__
#endif
  int64_t plane(int k) const { return PS * (k + 1); }
};

// What LeapfrogDev::advance() needs of a lattice form of the step: the state
// maps and the four kernels, over the whole mesh. Two implementations: the
// first-order Kuhn lattice below (stencils unrolled at compile time) and the
// table-driven lattice of table_lattice.cuh (any order; config 4).
struct LatticeOps {
  // state bookkeeping of the owning handle: `valid` = the lattice fields hold
  // the handle's state (or a newer one), `newer` = the DOF vectors are stale
  bool valid = false, newer = false;
  virtual ~LatticeOps() = default;
  virtual void scatter(const double* b, const double* e, cudaStream_t s) = 0;
  virtual void gather(double* b, double* e, cudaStream_t s) const = 0;
  virtual void apply_q(cudaStream_t s) const = 0;              // T = Q_sym E
  virtual void apply_cb(double h, cudaStream_t s) const = 0;   // B -= h C T
  virtual void apply_m2(cudaStream_t s) const = 0;             // U = M2 B
  virtual void apply_cte(double f, cudaStream_t s) const = 0;  // E += f C^T U
  // bytes each kernel moves (arrays read once, outputs written once)
  virtual double bytes_q() const = 0;
  virtual double bytes_cb() const = 0;
  virtual double bytes_m2() const = 0;
  virtual double bytes_cte() const = 0;
};

struct Lattice : LatticeOps {
  LatGeom g;
  int64_t n1 = 0, n2 = 0;
  DevBuf<double> qc;         // kQArrays * NP: canonical Q_sym coefficients
  DevBuf<double> mc;         // kMArrays * NP: canonical M2 coefficients
  DevBuf<double> E, T, B, U;  // 7, 7, 12, 12 components * NP
  DevBuf<int64_t> epos, fpos;  // DOF id -> component * NP + position
  bool pdl = true;

  // coefficient arrays from the device CSRs of the k-major numbering (the
  // CSRs are read, not consumed); throws if an entry falls outside the
  // interior stencil (it cannot for the Kuhn mesh)
  void build(const TetMesh& mesh, const DevCSR& qsym, const DevCSR& m2, cudaStream_t s);
  // DOF vectors <-> lattice state
  void scatter(const double* b, const double* e, cudaStream_t s) override;
  void gather(double* b, double* e, cudaStream_t s) const override;
  // the four step kernels over local vertex planes [k0, k1) (default: all)
  int k0 = 0, k1 = -1;  // compute range; k1 < 0: every local plane
  // (an explicit [kb, ke) overrides the range: the multi-rank overlap runs the
  // boundary planes first)
  void apply_q(cudaStream_t s, int kb, int ke) const;              // T = Q_sym E
  void apply_cb(double h, cudaStream_t s, int kb, int ke) const;   // B -= h C T
  void apply_m2(cudaStream_t s, int kb, int ke) const;             // U = M2 B
  void apply_cte(double f, cudaStream_t s, int kb, int ke) const;  // E += f C^T U
  void apply_q(cudaStream_t s) const override { apply_q(s, -1, -1); }
  void apply_cb(double h, cudaStream_t s) const override { apply_cb(h, s, -1, -1); }
  void apply_m2(cudaStream_t s) const override { apply_m2(s, -1, -1); }
  void apply_cte(double f, cudaStream_t s) const override { apply_cte(f, s, -1, -1); }
  int kbeg() const { return k0; }
  int kend() const { return k1 < 0 ? g.nz + 1 : k1; }
  // bytes each kernel moves (arrays read once, outputs written once)
  double bytes_q() const override;
  double bytes_cb() const override;
  double bytes_m2() const override;
  double bytes_cte() const override;
  double step_bytes() const { return bytes_q() + bytes_cb() + bytes_m2() + bytes_cte(); }
};

}  // namespace sfeec_b200
