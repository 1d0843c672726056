// Device-assembled tet system (tet_device.cu), shared with the partitioned
// path (partition.cu).
#pragma once
#include "device_util.cuh"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

struct DevTetSystem {
  DevCSR c, ct, m2, d, qsym;
  int64_t n1 = 0, n2 = 0, nt = 0;
  int64_t fallback = 0;
};

// C, D (optional), M1 -> S(M1) SPAI -> Q_sym, M2 and C^T of mesh `h`, built on
// the current device, bitwise the host builders' operators
// (exact_lo/hi: on a slab, the local vertex planes whose edges' SPAI columns
// must solve; the others, near the cut planes, are not used)
void build_tet_system_device(const TetMesh& h, bool want_div, DevTetSystem& out, cudaStream_t s,
                             int exact_lo = 0, int exact_hi = 1 << 30);

// in-place exclusive scan of d[0..n] (d[n] = total)
void exclusive_scan(int64_t* d, int64_t n, cudaStream_t s);
// t = a^T (cub radix sort on (col, row) keys)
void transpose_dev(const DevCSR& a, DevCSR& t, cudaStream_t s);
// out[k] = 0.5 Q(r, c) + 0.5 Q(c, r) on a symmetric pattern (rp, ci), where
// qcol holds the SPAI columns in pattern layout (qcol[rp[c] + a] = q_c[a])
void qsym_device(int64_t n, const int64_t* rp, const int32_t* ci, const double* qcol, double* out,
                 cudaStream_t s);

// rows [r0, r1) of `a` with columns shifted by -c0 into [0, ncols)
void slice_rows_device(const DevCSR& a, int64_t r0, int64_t r1, int64_t c0, int64_t ncols,
                       DevCSR& out, cudaStream_t s);

}  // namespace sfeec_b200
