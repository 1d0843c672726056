// Device side of the second-order P2^- system (p2_device.cu).
#pragma once
#include "device_util.cuh"
#include "p2_mesh.hpp"

namespace sfeec_b200 {

struct DevP2System {
  DevCSR c, ct, m2, d, qsym;
  int64_t n1 = 0, n2 = 0, n3 = 0;
  int64_t fallback = 0;
};

// S(M1^2) pattern of M1 with the values of M1^2 (ascending-k sums,
// separate rounding: bitwise the host sparse_square entries)
void square_pattern_device(const DevCSR& m1, DevCSR& out, cudaStream_t s);
// SPAI of M1 on the pattern of `sq` (whose values are M1^2); qcol[rp[l] + a]
// = q_l[a]; returns the number of columns that failed the pivot test
int64_t spai_big_device(const DevCSR& m1, const DevCSR& sq, DevBuf<double>& qcol, cudaStream_t s);
// C, M1, M2 (and D) from the host builders, then S(M1^2), SPAI, Q_sym and
// C^T on the device
void build_p2_system_device(const TetMesh& mesh, const P2Dofs& dofs, bool want_div,
                            DevP2System& out, cudaStream_t s);

}  // namespace sfeec_b200
