// Kuhn-lattice kernels of the first-order leapfrog (lattice.cuh, DESIGN.md
// 3.4): one thread per vertex computes all edge (7) or face (12) rows of its
// vertex. Every stencil is unrolled at compile time from lattice_tables.hpp,
// so each neighbour read is a constant offset from the thread's position:
// 32 lanes = 32 consecutive positions of a padded row -> coalesced loads of
// the coefficient and field arrays, no index streams.
//
// Summation order per row = the slot order (dk, dj, type, di), which is the
// ascending column order of the k-major numbering for rows away from the
// 32-vertex x-block edges: those rows are summed exactly like the sliced /
// ELL kernels (spmv_kernels.cu) sum their CSR rows.
#include <utility>
#include <vector>

#include "lattice_kernels.cuh"

namespace sfeec_b200 {

using namespace latk;

namespace {

// ---- setup: coefficient arrays from a CSR of the k-major numbering -----------
// Entry (r, c) of row type t at offset off: the slot of t's stencil with
// (type(c), off); canonical slots store the value at the row's position.
template <class Op, int T, int... I>
__device__ __forceinline__ bool fill_match(std::integer_sequence<int, I...>, int t2,
                                           int64_t off, const LatGeom& g, double v,
                                           double* __restrict__ coef, int64_t idx) {
  bool found = false;
  (
      [&] {
        constexpr lat::Slot sl = Op::tab(Op::slot_off(T) + I);
        if (!found && sl.t == t2 && off == offset_of(g, sl.di, sl.dj, sl.dk)) {
          found = true;
          if (!sl.mirror) coef[(int64_t)(Op::canon_off(T) + sl.si) * g.NP + idx] = v;
        }
      }(),
      ...);
  return found;
}
template <class Op, int... Ts>
__device__ __forceinline__ bool fill_dispatch(std::integer_sequence<int, Ts...>, int t, int t2,
                                              int64_t off, const LatGeom& g, double v,
                                              double* __restrict__ coef, int64_t idx) {
  bool found = false;
  ((t == Ts ? (void)(found = fill_match<Op, Ts>(
                         std::make_integer_sequence<int, Op::slot_off(Ts + 1) - Op::slot_off(Ts)>{},
                         t2, off, g, v, coef, idx))
            : (void)0),
   ...);
  return found;
}
template <class Op>
__global__ void k_lat_fill(int64_t rows, const int64_t* __restrict__ rp,
                           const int32_t* __restrict__ ci, const double* __restrict__ val,
                           const int64_t* __restrict__ pos, LatGeom g, double* __restrict__ coef,
                           int* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t p = pos[r];
  const int t = (int)(p / g.NP);
  const int64_t idx = p - (int64_t)t * g.NP;
  for (int64_t q = rp[r]; q < rp[r + 1]; ++q) {
    const int64_t pc = pos[ci[q]];
    const int t2 = (int)(pc / g.NP);
    const int64_t off = (pc - (int64_t)t2 * g.NP) - idx;
    if (!fill_dispatch<Op>(std::make_integer_sequence<int, Op::kTypes>{}, t, t2, off, g, val[q],
                           coef, idx))
      atomicExch(bad, 1);
  }
}

__global__ void k_lat_scatter(int64_t n, const int64_t* __restrict__ pos,
                              const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[pos[r]] = src[r];
}
__global__ void k_lat_gather(int64_t n, const int64_t* __restrict__ pos,
                             const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[pos[r]];
}

inline unsigned blocks(int64_t n) { return (unsigned)((n + kLT - 1) / kLT); }



}  // namespace

void Lattice::build(const TetMesh& mesh, const DevCSR& qsym, const DevCSR& m2,
                    cudaStream_t s) {
  g.init(mesh.n, mesh.nz, mesh.kz0, mesh.nzg);
  n1 = mesh.n_edges;
  n2 = mesh.n_faces;
  require(qsym.rows == n1 && m2.rows == n2, "lattice: operator dimensions do not match the mesh");
  {  // DOF -> lattice position (component * NP + vertex position)
    std::vector<int64_t> ep((size_t)n1), fp((size_t)n2);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n1; ++r) {
      int c[3];
      mesh.coords(mesh.edge_v[(size_t)r], c);
      ep[(size_t)r] = (int64_t)mesh.edge_t[(size_t)r] * g.NP + g.pos(c[0], c[1], c[2]);
    }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n2; ++r) {
      int c[3];
      mesh.coords(mesh.face_v[(size_t)r], c);
      fp[(size_t)r] = (int64_t)mesh.face_t[(size_t)r] * g.NP + g.pos(c[0], c[1], c[2]);
    }
    epos.upload(ep.data(), ep.size(), s);
    fpos.upload(fp.data(), fp.size(), s);
    SFEEC_CUDA(cudaStreamSynchronize(s));  // the host vectors die here
  }
  qc.alloc((size_t)(lat::kQArrays * g.NP));
  mc.alloc((size_t)(lat::kMArrays * g.NP));
  qc.zero(s);
  mc.zero(s);
  DevBuf<int> bad;
  bad.alloc(1);
  bad.zero(s);
  if (n1)
    k_lat_fill<QOp><<<blocks(n1), kLT, 0, s>>>(n1, qsym.rp.p, qsym.ci.p, qsym.val.p, epos.p, g,
                                                qc.p, bad.p);
  if (n2)
    k_lat_fill<MOp><<<blocks(n2), kLT, 0, s>>>(n2, m2.rp.p, m2.ci.p, m2.val.p, fpos.p, g, mc.p,
                                               bad.p);
  SFEEC_LAUNCH_CHECK();
  int hbad = 0;
  SFEEC_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SFEEC_CUDA(cudaStreamSynchronize(s));
  require(hbad == 0, "lattice: an operator entry lies outside the Kuhn-lattice stencil");
  // (+ slack: the staged segments of the last plane read up to kSegLen past
  // the last component's end)
  for (auto* b : {&E, &T}) {
    b->alloc((size_t)(7 * g.NP + 2 * kSegLenMax));
    b->zero(s);
  }
  for (auto* b : {&B, &U}) {
    b->alloc((size_t)(12 * g.NP + 2 * kSegLenMax));
    b->zero(s);
  }
  SFEEC_CUDA(cudaStreamSynchronize(s));
  valid = newer = false;





}

void Lattice::scatter(const double* b, const double* e, cudaStream_t s) {
  if (n2) k_lat_scatter<<<blocks(n2), kLT, 0, s>>>(n2, fpos.p, b, B.p);
  if (n1) k_lat_scatter<<<blocks(n1), kLT, 0, s>>>(n1, epos.p, e, E.p);
  SFEEC_LAUNCH_CHECK();
}

void Lattice::gather(double* b, double* e, cudaStream_t s) const {
  if (n2) k_lat_gather<<<blocks(n2), kLT, 0, s>>>(n2, fpos.p, B.p, b);
  if (n1) k_lat_gather<<<blocks(n1), kLT, 0, s>>>(n1, epos.p, E.p, e);
  SFEEC_LAUNCH_CHECK();
}

// one thread per vertex computes all of its rows (the neighbour loads the
// rows share are loaded once); a block is 256 consecutive positions of one
// padded plane; grids cover local planes [kbeg(), kend()). Brick-shaped blocks
// (32x8x1, 32x4x2, 32x2x4, 64x4x1, 64x2x2 vertices, for L1 reuse of the dj / dk
// neighbours and mirrored coefficients), with and without a 128-byte-aligned
// row pitch, measured slower on tet256: K-Q 2.13-2.26 vs 2.02 ms, K-M2 1.55-1.63
// vs 1.48, K-CTe 0.68-0.71 vs 0.66; the aligned pitch alone 2.06 / 1.53 / 0.67.
// ncu (profiles/round2_tet256_lattice.md): L2 47%, L1 35%, DRAM 67% busy.
// Measured and rejected (tet256, ms per launch, this kernel form first): one
// warp per row type (K-Q 2.03 vs 2.77, K-M2 1.49 vs 2.14), two threads per
// vertex (2.03 vs 2.16, 1.49 vs 1.71), z-sweeps fusing K-Q + K-Cb and K-M2 +
// K-CTe with t / u in shared memory (5.1 vs 8.1 ms per step: one barrier per
// plane serialises the 125 KB-per-plane coefficient streams of a tile).
void Lattice::apply_q(cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  // (e staged by bulk copies as in K-Cb, coefficients loaded as here, was
  // measured slower: 2.26 ms with 128-position chunks, 3.39 with 256, vs 2.02)
  k_lat_q<MapSym><<<MapSym::grid(g, kb, ke), kSymThreads, 0, s>>>(g, kb, ke, qc.p, E.p, T.p);
  SFEEC_LAUNCH_CHECK();
}
template <bool TRANS, int kCH, int kAL = 2>
static void launch_inc_bulk(const LatGeom& g, int kb, int ke, double alpha, const double* x,
                            double* y, cudaStream_t s) {
  constexpr int NSEG = IncTab<TRANS>::nseg();
  const int smem = 2 * NSEG * (kCH + 2 + kAL) * (int)sizeof(double);
  static int per_sm = 0, sms = 0;  // resident CTAs (the shared memory decides)
  if (!per_sm) {
    SFEEC_CUDA(cudaFuncSetAttribute(k_lat_inc_bulk<TRANS, kCH, kAL>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SFEEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lat_inc_bulk<TRANS, kCH, kAL>, kCH,
                                                             smem));
    int dev = 0;
    SFEEC_CUDA(cudaGetDevice(&dev));
    SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    per_sm = std::max(per_sm, 1);
  }
  const int64_t nchunk = ((g.PS + kCH - 1) / kCH) * (int64_t)(ke - kb);
  const unsigned grid = (unsigned)std::min<int64_t>(nchunk, (int64_t)per_sm * sms);
  k_lat_inc_bulk<TRANS, kCH, kAL><<<grid, kCH, smem, s>>>(g, kb, ke, alpha, x, y);
  SFEEC_LAUNCH_CHECK();
}

void Lattice::apply_cb(double h, cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  // t staged by bulk copies (measured, tet256: 0.71 vs 0.95 ms for the plain
  // k_lat_cb; the same staging of u slows K-CTe, 0.75-0.83 vs 0.66 ms: its 21
  // segments leave room for two CTAs per SM; starting the copies on 32 /
  // 128 / 256-byte boundaries instead of 16 changes nothing: 0.720 ms each)
  launch_inc_bulk<false, 256>(g, kb, ke, -h, T.p, B.p, s);
}
void Lattice::apply_m2(cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  // (b staged by bulk copies: 1.83 / 2.25 ms vs 1.48, as for K-Q)
  k_lat_m2<MapSym><<<MapSym::grid(g, kb, ke), kSymThreads, 0, s>>>(g, kb, ke, mc.p, B.p, U.p);
  SFEEC_LAUNCH_CHECK();
}
void Lattice::apply_cte(double f, cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  k_lat_cte<MapLine><<<MapLine::grid(g, kb, ke), kLT, 0, s>>>(g, kb, ke, f, U.p, E.p);
  SFEEC_LAUNCH_CHECK();
}

// bytes per launch (each array read once, each output written once; the
// padded halo is not counted): V vertices, 8 B per value; the outputs are the
// DOFs on the whole mesh, all 7 / 12 slots of the computed planes on a slab
double Lattice::bytes_q() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (kend() - kbeg());
  return 8.0 * (lat::kQArrays * V + 7.0 * V + (k1 < 0 ? (double)n1 : 7.0 * V));
}
double Lattice::bytes_cb() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (kend() - kbeg());
  return 8.0 * (7.0 * V + 2.0 * (k1 < 0 ? (double)n2 : 12.0 * V));
}
double Lattice::bytes_m2() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (kend() - kbeg());
  return 8.0 * (lat::kMArrays * V + 12.0 * V + (k1 < 0 ? (double)n2 : 12.0 * V));
}
double Lattice::bytes_cte() const {
  const double V = (double)(g.n + 1) * (g.n + 1) * (kend() - kbeg());
  return 8.0 * (12.0 * V + 2.0 * (k1 < 0 ? (double)n1 : 7.0 * V));
}

}  // namespace sfeec_b200
