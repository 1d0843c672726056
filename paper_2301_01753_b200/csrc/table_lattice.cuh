// Table-driven Kuhn-lattice form of the leapfrog step: the
// layout of lattice.cuh for any Whitney order on the Kuhn mesh, used for the
// second-order system of config 4 (P2-, S(M1^2) SPAI: 38 1-form and 54
// 2-form DOF types per vertex, ~12,000 Q_sym stencil slots per vertex).
//
// Every DOF is (vertex, type); a field is one array per type over the padded
// vertex box (halo = the stencil reach, 2 for S(M1^2)), zero where the slot
// is not a DOF. The interior stencil of each row type -- (column type, vertex
// offset) per slot, in the CSR column order of an interior row -- is read off
// the assembled operators at build time, not generated ahead of time:
//   * Q_sym and M2 (exactly symmetric): one coefficient array per canonical
//     slot (offset lexicographically positive, or zero with column type >=
//     row type); the transposed slot reads the same array at the neighbour's
//     position. 8 B per stored pair, no column indices.
//   * C and C^T: the entries are the same constants (+-1, +-1/2) for every
//     vertex -- the exterior derivative is metric-free -- so they live in the
//     slot table and stream nothing.
// The build checks every entry of the assembled CSRs against the tables (an
// entry without a slot, or an incidence value that differs from its slot's
// constant, fails the build), so a lattice that builds applies the same
// operators as the CSR layouts.
#pragma once
#include <vector>

#include "lattice.cuh"

namespace sfeec_b200 {

struct TLGeom {
  int n = 0;        // cubes per axis (vertices 0..n)
  int H = 0;        // halo layers
  int S = 0;        // padded vertices per axis (n + 1 + 2 H)
  int64_t PS = 0;   // padded plane
  int64_t NP = 0;   // padded box: the type stride
  static constexpr int64_t kAlign = 32;  // positions
  int64_t P0 = 0;   // leading pad: puts the first swept position of a plane on an aligned address
  void init(int n_, int h_) {
    n = n_;
    H = h_;
    S = n + 1 + 2 * H;
    // The plane pitch and the first swept position of a plane (row j = 0) are
    // multiples of kAlign positions, so a block's 128 positions start on a
    // sector boundary in every array (measured on config 4: step 4.05 -> 3.95
    // ms with 32 or 128, bitwise the same state).
    PS = ((int64_t)S * S + kAlign - 1) / kAlign * kAlign;
    P0 = (kAlign - ((int64_t)S * H) % kAlign) % kAlign;
    NP = (PS * S + P0 + kAlign - 1) / kAlign * kAlign;
  }
#ifdef __CUDACC__
  __host__ __device__
#endif
  int64_t pos(int i, int j, int k) const {
    return P0 + (i + H) + (int64_t)S * (j + H) + PS * (k + H);
  }
};

struct TLSlot {   // symmetric operator: y_r(v) += coef[coff + v] * x[xoff + v]
  int64_t coff;   // array * NP (+ the neighbour offset for a transposed slot)
  int64_t xoff;   // column type * NP + neighbour offset
};
struct TLCSlot {  // constant operator: y_r(v) += val * x[xoff + v]
  double val;
  int64_t xoff;
};

struct TLSym {
  int mb = 1;  // moments per entity: the tables are per entity type, a slot is an mb x mb block
  bool soa = false;  // blocks as mb * mb arrays (type-major fields) instead of interleaved
  int ntypes = 0, narrays = 0;
  int64_t nslots = 0;
  int max_slots = 0;       // longest row type's table (staged in shared memory)
  DevBuf<int> beg;         // ntypes + 1: slot range of each row type
  DevBuf<TLSlot> slots;
  DevBuf<double> coef;     // narrays * NP * mb * mb (a block's values row-major per position)
};
struct TLInc {
  int ntypes = 0;
  int64_t nslots = 0;
  DevBuf<int> beg;
  DevBuf<TLCSlot> slots;
};

// DOF -> (type, vertex id of the (n + 1)^3 vertex numbering)
struct TLDofs {
  int ntypes = 0;
  int mb = 1;  // moments per entity: type = entity type * mb + moment
  std::vector<int32_t> type;
  std::vector<int64_t> vertex;
};

struct TableLattice : LatticeOps {
  TLGeom g;
  int64_t n1 = 0, n2 = 0;
  int nt1 = 0, nt2 = 0;      // 1-form / 2-form DOF types per vertex
  TLSym q, m2;
  TLInc c, ct;
  DevBuf<double> E, T, B, U;       // nt1, nt1, nt2, nt2 arrays of NP
  DevBuf<int64_t> epos, fpos;      // DOF id -> type * NP + position
  DevBuf<int64_t> eaddr;           // mb1 > 1: DOF id -> element of the interleaved E / T
  int mb1 = 1;  // moments per 1-form entity: E / T hold (moment 0, moment 1, ..) per entity
  DevBuf<uint64_t> mask1, mask2;   // per position: bit t = (vertex, type t) is a DOF

  // tables and coefficient arrays from the device CSRs (read, not consumed).
  // Throws if the mesh is too small for an interior reference vertex
  // (n < 2 halo + 2), or if an operator entry does not fit the tables.
  void build(int n, int halo, const TLDofs& d1, const TLDofs& d2, const DevCSR& qsym,
             const DevCSR& m2csr, const DevCSR& ccsr, const DevCSR& ctcsr, cudaStream_t s);

  void scatter(const double* b, const double* e, cudaStream_t s) override;
  void gather(double* b, double* e, cudaStream_t s) const override;
  void apply_q(cudaStream_t s) const override;
  void apply_cb(double h, cudaStream_t s) const override;
  void apply_m2(cudaStream_t s) const override;
  void apply_cte(double f, cudaStream_t s) const override;
  double bytes_q() const override;
  double bytes_cb() const override;
  double bytes_m2() const override;
  double bytes_cte() const override;
};

}  // namespace sfeec_b200
