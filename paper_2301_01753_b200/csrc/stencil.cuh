// Mesh-aware ("stencil") operator layout for the structured Kuhn tet mesh.
//
// On the Kuhn mesh every entity type has a fixed neighbour stencil (the
// edges/faces sharing a tet with it), so an operator row of an entity at
// vertex v with type t touches entity (v + offset_s, type_s) in slot s. The
// column ids are recomputed in the kernel from a per-type vertex -> DOF table
// (eidT[t][v] / fidT[f][v], -1 for PEC boundary edges) instead of being
// streamed: Q_sym and M2 stream 8 B per entry instead of 12, and the
// incidence matrices C and C^T stream nothing but their vectors (their signs
// are part of the stencil). Stencils are derived from the assembled CSR rows
// of an interior entity of a small reference mesh (stencil.cu), so they are
// exactly the operators' topological patterns.
#pragma once
#include <memory>

#include "device_util.cuh"

namespace sfeec_b200 {

struct TetMesh;
struct DevCSR;

// tables shared by the four stencil operators of one mesh
struct StencilMesh {
  int n = 0;
  int64_t nv = 0, n_edges = 0, n_faces = 0;
  DevBuf<int32_t> eidT, fidT;  // [7][nv], [12][nv]
  DevBuf<int32_t> edge_v, face_v;  // base vertex per DOF
};

enum StencilKind { kStQ = 0, kStM2 = 1, kStC = 2, kStCT = 3 };

// device layout of one stencil operator
struct StencilOp {
  int kind = 0;
  std::shared_ptr<StencilMesh> mesh;
  int64_t rows = 0, n_slices = 0;
  DevBuf<int64_t> slice_row, slice_ptr;
  DevBuf<int8_t> slice_type;
  DevBuf<double> val;  // Q, M2 only
  double stream_bytes() const;
};

// stencil sizes / tables (host copy, also uploaded to __constant__)
void stencil_init_tables();
// builds the stencil operator `kind` from the device CSR of the same operator
// (values looked up by column; every CSR entry must be covered by the stencil)
void stencil_build(const TetMesh& host_mesh, const std::shared_ptr<StencilMesh>& sm, int kind,
                   const DevCSR* csr, StencilOp& out, cudaStream_t s);
std::shared_ptr<StencilMesh> stencil_mesh(const TetMesh& host_mesh, cudaStream_t s);
// accumulate ? y += alpha * A x : y = A x
void launch_stencil(const StencilOp& a, const double* x, double* y, double alpha, bool accumulate,
                    cudaStream_t s);

}  // namespace sfeec_b200
