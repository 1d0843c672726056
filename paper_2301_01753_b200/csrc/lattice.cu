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

#include "bulk_copy.cuh"
#include "lattice.cuh"
#include "lattice_tables.hpp"

namespace sfeec_b200 {

namespace {

constexpr int kLT = 256;  // threads per block (positions of one padded plane)

SFEEC_HD constexpr int et(int t, int d) {
  constexpr int v[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0},
                           {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
  return v[t][d];
}
// second (largest) edge type of face type f (kFT[f][1])
SFEEC_HD constexpr int ft_hi(int f) {
  constexpr int v[12] = {3, 3, 4, 4, 5, 5, 6, 6, 6, 6, 6, 6};
  return v[f];
}

// operator policies over the generated tables
struct QOp {
  static constexpr int kTypes = lat::kQTypes;
  static constexpr int kArrays = lat::kQArrays;
  SFEEC_HD static constexpr lat::Slot tab(int s) { return lat::kQTab(s); }
  SFEEC_HD static constexpr int slot_off(int t) { return lat::kQSlotOff(t); }
  SFEEC_HD static constexpr int canon_off(int t) { return lat::kQCanonOff(t); }
};
struct MOp {
  static constexpr int kTypes = lat::kMTypes;
  static constexpr int kArrays = lat::kMArrays;
  SFEEC_HD static constexpr lat::Slot tab(int s) { return lat::kMTab(s); }
  SFEEC_HD static constexpr int slot_off(int t) { return lat::kMSlotOff(t); }
  SFEEC_HD static constexpr int canon_off(int t) { return lat::kMCanonOff(t); }
};

__device__ __forceinline__ int64_t offset_of(const LatGeom& g, int di, int dj, int dk) {
  return di + (int64_t)g.S * dj + g.PS * dk;
}

// this thread's vertex (i, j, local plane k) and lattice position; false off
// the mesh. Block row y covers local plane kbeg + y.
__device__ __forceinline__ bool my_vertex(const LatGeom& g, int kbeg, int& i, int& j, int& k,
                                          int64_t& idx) {
  const int p = blockIdx.x * kLT + threadIdx.x;
  if (p >= g.PS) return false;
  k = kbeg + blockIdx.y;
  j = p / g.S - 1;
  i = p - (j + 1) * g.S - 1;
  idx = g.PS * (k + 1) + p;
  return i >= 0 && i <= g.n && j >= 0 && j <= g.n;
}

// edge (v, t) is a DOF: inside the mesh and not on a wall it lies in (PEC);
// z is judged on the whole mesh (kg = whole-mesh plane, nzg)
template <int T>
__device__ __forceinline__ bool edge_dof(int i, int j, int k, const LatGeom& g) {
  const int kg = k + g.kz0;
  bool ok = i + et(T, 0) <= g.n && j + et(T, 1) <= g.n && kg + et(T, 2) <= g.nzg;
  if (et(T, 0) == 0) ok = ok && i != 0 && i != g.n;
  if (et(T, 1) == 0) ok = ok && j != 0 && j != g.n;
  if (et(T, 2) == 0) ok = ok && kg != 0 && kg != g.nzg;
  return ok;
}
// face (v, f) exists: its farthest vertex is inside the mesh
template <int F>
__device__ __forceinline__ bool face_ok(int i, int j, int k, const LatGeom& g) {
  return i + et(ft_hi(F), 0) <= g.n && j + et(ft_hi(F), 1) <= g.n &&
         k + g.kz0 + et(ft_hi(F), 2) <= g.nzg;
}

// ---- symmetric stencil rows (Q_sym, M2) ------------------------------------
template <class Op, int S>
__device__ __forceinline__ void sym_term(double& acc, const double* __restrict__ coef,
                                         const double* __restrict__ x, int64_t idx,
                                         const LatGeom& g) {
  constexpr lat::Slot sl = Op::tab(S);
  const int64_t off = offset_of(g, sl.di, sl.dj, sl.dk);
  const double c =
      __ldg(coef + (int64_t)(Op::canon_off(sl.st) + sl.si) * g.NP + idx + (sl.mirror ? off : 0));
  acc = fma(c, __ldg(x + (int64_t)sl.t * g.NP + idx + off), acc);
}
template <class Op, int T, int... I>
__device__ __forceinline__ double sym_row(std::integer_sequence<int, I...>,
                                          const double* __restrict__ coef,
                                          const double* __restrict__ x, int64_t idx,
                                          const LatGeom& g) {
  double acc = 0.0;
  (sym_term<Op, Op::slot_off(T) + I>(acc, coef, x, idx, g), ...);
  return acc;
}
template <class Op, int T>
__device__ __forceinline__ double sym_row(const double* __restrict__ coef,
                                          const double* __restrict__ x, int64_t idx,
                                          const LatGeom& g) {
  return sym_row<Op, T>(std::make_integer_sequence<int, Op::slot_off(T + 1) - Op::slot_off(T)>{},
                        coef, x, idx, g);
}

// t = Q_sym e on the DOF edges of one vertex (7 rows)
template <int... Ts>
__device__ __forceinline__ void q_vertex(std::integer_sequence<int, Ts...>, const LatGeom& g,
                                         int i, int j, int k, int64_t idx,
                                         const double* __restrict__ qc,
                                         const double* __restrict__ E, double* __restrict__ T) {
  const double r[sizeof...(Ts)] = {sym_row<QOp, Ts>(qc, E, idx, g)...};
  ((edge_dof<Ts>(i, j, k, g) ? (void)(T[(int64_t)Ts * g.NP + idx] = r[Ts]) : (void)0), ...);
}
// 2 blocks per SM: 128 registers, every load of the vertex's 7 rows in flight
// (measured: 80 / 64-register caps spill and run 1.6x / 2.4x slower; one
// block per SM at 247 registers runs 1.05x (K-Q) / 1.15x (K-M2) slower)
__global__ void __launch_bounds__(kLT, 2) k_lat_q(LatGeom g, int kbeg, const double* __restrict__ qc,
                                               const double* __restrict__ E,
                                               double* __restrict__ T) {
  int i, j, k;
  int64_t idx;
  if (!my_vertex(g, kbeg, i, j, k, idx)) return;
  q_vertex(std::make_integer_sequence<int, 7>{}, g, i, j, k, idx, qc, E, T);
}

// u = M2 b on the faces of one vertex (12 rows)
template <int... Fs>
__device__ __forceinline__ void m2_vertex(std::integer_sequence<int, Fs...>, const LatGeom& g,
                                          int i, int j, int k, int64_t idx,
                                          const double* __restrict__ mc,
                                          const double* __restrict__ B, double* __restrict__ U) {
  const double r[sizeof...(Fs)] = {sym_row<MOp, Fs>(mc, B, idx, g)...};
  ((face_ok<Fs>(i, j, k, g) ? (void)(U[(int64_t)Fs * g.NP + idx] = r[Fs]) : (void)0), ...);
}
__global__ void __launch_bounds__(kLT, 2) k_lat_m2(LatGeom g, int kbeg, const double* __restrict__ mc,
                                                const double* __restrict__ B,
                                                double* __restrict__ U) {
  int i, j, k;
  int64_t idx;
  if (!my_vertex(g, kbeg, i, j, k, idx)) return;
  m2_vertex(std::make_integer_sequence<int, 12>{}, g, i, j, k, idx, mc, B, U);
}

// ---- incidence rows (C, C^T): signed sums, then y = fma(alpha, sum, y) ----
template <bool TRANS, int S>
__device__ __forceinline__ void inc_term(double& acc, const double* __restrict__ x, int64_t idx,
                                         const LatGeom& g) {
  constexpr lat::CSlot sl = TRANS ? lat::kCTTab(S) : lat::kCTab(S);
  const double v = __ldg(x + (int64_t)sl.t * g.NP + idx + offset_of(g, sl.di, sl.dj, sl.dk));
  acc += sl.sign > 0 ? v : -v;
}
template <bool TRANS, int BASE, int... I>
__device__ __forceinline__ double inc_row(std::integer_sequence<int, I...>,
                                          const double* __restrict__ x, int64_t idx,
                                          const LatGeom& g) {
  double acc = 0.0;
  (inc_term<TRANS, BASE + I>(acc, x, idx, g), ...);
  return acc;
}
// e += f C^T u on the DOF edges of one vertex
template <int... Ts>
__device__ __forceinline__ void cte_vertex(std::integer_sequence<int, Ts...>, const LatGeom& g,
                                           int i, int j, int k, int64_t idx, double alpha,
                                           const double* __restrict__ U, double* __restrict__ E) {
  const double r[sizeof...(Ts)] = {inc_row<true, lat::kCTOff(Ts)>(
      std::make_integer_sequence<int, lat::kCTOff(Ts + 1) - lat::kCTOff(Ts)>{}, U, idx, g)...};
  ((edge_dof<Ts>(i, j, k, g)
        ? (void)(E[(int64_t)Ts * g.NP + idx] = fma(alpha, r[Ts], E[(int64_t)Ts * g.NP + idx]))
        : (void)0),
   ...);
}
__global__ void __launch_bounds__(kLT) k_lat_cte(LatGeom g, int kbeg, double alpha,
                                                 const double* __restrict__ U,
                                                 double* __restrict__ E) {
  int i, j, k;
  int64_t idx;
  if (!my_vertex(g, kbeg, i, j, k, idx)) return;
  cte_vertex(std::make_integer_sequence<int, 7>{}, g, i, j, k, idx, alpha, U, E);
}

// ---- K-Cb: the gathered vector staged by bulk copies ------------------------
// K-Cb reads 14 distinct (component, dj, dk) row segments of t (K-CTe: 21 of u)
// around a chunk of kCH consecutive positions of one plane. One thread issues
// their bulk copies (cp.async.bulk) into a two-stage shared-memory ring one
// chunk ahead; the block's threads (one per position) sum the rows from shared
// memory and update b / e in place. Persistent CTAs take chunks round-robin.
constexpr int kSegLenMax = 256 + 4;  // doubles per staged segment at most (allocation slack)

template <bool TRANS>
struct IncTab {
  static constexpr int kSlots = 36;
  SFEEC_HD static constexpr lat::CSlot slot(int s) { return TRANS ? lat::kCTTab(s) : lat::kCTab(s); }
  // first slot with the same (t, dj, dk) as slot s
  SFEEC_HD static constexpr int rep(int s) {
    for (int r = 0; r < s; ++r)
      if (slot(r).t == slot(s).t && slot(r).dj == slot(s).dj && slot(r).dk == slot(s).dk) return r;
    return s;
  }
  SFEEC_HD static constexpr int nseg() {
    int n = 0;
    for (int s = 0; s < kSlots; ++s) n += rep(s) == s;
    return n;
  }
  // segment index of slot s (segments numbered in first-occurrence order)
  SFEEC_HD static constexpr int seg(int s) {
    int n = 0;
    for (int r = 0; r < rep(s); ++r) n += rep(r) == r;
    return n;
  }
  // the representative slot of segment i
  SFEEC_HD static constexpr int seg_slot(int i) {
    int n = 0;
    for (int s = 0; s < kSlots; ++s)
      if (rep(s) == s) {
        if (n == i) return s;
        ++n;
      }
    return 0;
  }
};

template <bool TRANS, int SEGLEN, int S>
__device__ __forceinline__ void inc_term_stage(double& acc, const double* __restrict__ stage,
                                               const int* __restrict__ shift, int q) {
  using Tb = IncTab<TRANS>;
  constexpr lat::CSlot sl = Tb::slot(S);
  constexpr int sg = Tb::seg(S);
  const double v = stage[sg * SEGLEN + shift[sg] + 1 + sl.di + q];
  acc += sl.sign > 0 ? v : -v;
}
template <bool TRANS, int SEGLEN, int BASE, int... I>
__device__ __forceinline__ double inc_row_stage(std::integer_sequence<int, I...>,
                                                const double* __restrict__ stage,
                                                const int* __restrict__ shift, int q) {
  double acc = 0.0;
  (inc_term_stage<TRANS, SEGLEN, BASE + I>(acc, stage, shift, q), ...);
  return acc;
}
template <bool TRANS, int R>
__device__ __forceinline__ constexpr int inc_base() {
  return TRANS ? lat::kCTOff(R) : 3 * R;
}
template <bool TRANS, int R>
__device__ __forceinline__ constexpr int inc_len() {
  return TRANS ? lat::kCTOff(R + 1) - lat::kCTOff(R) : 3;
}
template <bool TRANS, int SEGLEN, int... Rs>
__device__ __forceinline__ void inc_vertex_stage(std::integer_sequence<int, Rs...>,
                                                 const LatGeom& g, int i, int j, int k,
                                                 int64_t idx, double alpha,
                                                 const double* __restrict__ stage,
                                                 const int* __restrict__ shift, int q,
                                                 double* __restrict__ y) {
  // the own values first (independent of the staged rows)
  const double y0[sizeof...(Rs)] = {y[(int64_t)Rs * g.NP + idx]...};
  const double r[sizeof...(Rs)] = {inc_row_stage<TRANS, SEGLEN, inc_base<TRANS, Rs>()>(
      std::make_integer_sequence<int, inc_len<TRANS, Rs>()>{}, stage, shift, q)...};
  (((TRANS ? edge_dof<Rs>(i, j, k, g) : face_ok<Rs>(i, j, k, g))
        ? (void)(y[(int64_t)Rs * g.NP + idx] = fma(alpha, r[Rs], y0[Rs]))
        : (void)0),
   ...);
}

template <bool TRANS, int kCH>
__global__ void __launch_bounds__(kCH)
    k_lat_inc_bulk(LatGeom g, int kbeg, int kend, double alpha, const double* __restrict__ x,
                   double* __restrict__ y) {
  constexpr int kSegLen = kCH + 4;  // di in -1..1 plus 16-byte alignment
  using Tb = IncTab<TRANS>;
  constexpr int NSEG = Tb::nseg();
  constexpr int NR = TRANS ? 7 : 12;
  extern __shared__ __align__(16) double sm[];  // 2 stages x NSEG x kSegLen
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int shift[2][NSEG];
  const int per_plane = (int)((g.PS + kCH - 1) / kCH);
  const int64_t nchunk = (int64_t)per_plane * (kend - kbeg);
  const int t = threadIdx.x;
  if (t == 0) {
    bc_mbar_init(&bar[0], 1);
    bc_mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage one chunk: segment (t, dj, dk) = x[t*NP + plane(k+dk) + S*dj + x0 - 1 + (0..kCH+1)],
  // copied from the 16-byte-aligned start below it
  auto issue = [&](int64_t c, int st) {
    const int k = kbeg + (int)(c / per_plane);
    const int64_t x0 = (c % per_plane) * kCH;
    bc_mbar_expect_tx(&bar[st], NSEG * kSegLen * 8);
#pragma unroll
    for (int sgi = 0; sgi < NSEG; ++sgi) {
      const lat::CSlot sl = Tb::slot(Tb::seg_slot(sgi));
      const int64_t g0 = (int64_t)sl.t * g.NP + g.PS * (k + 1 + sl.dk) + (int64_t)g.S * sl.dj + x0 - 1;
      const int64_t a0 = g0 & ~(int64_t)1;
      shift[st][sgi] = (int)(g0 - a0);
      bc_copy(sm + (st * NSEG + sgi) * kSegLen, x + a0, kSegLen * 8, &bar[st]);
    }
  };
  int64_t c = blockIdx.x;
  if (t == 0 && c < nchunk) issue(c, 0);
  for (int it = 0; c < nchunk; ++it, c += gridDim.x) {
    const int st = it & 1;
    if (t == 0 && c + gridDim.x < nchunk) issue(c + gridDim.x, st ^ 1);
    const int k = kbeg + (int)(c / per_plane);
    const int64_t p = (c % per_plane) * kCH + t;
    const int j = (int)(p / g.S) - 1;
    const int i = (int)(p - (int64_t)(j + 1) * g.S) - 1;
    const bool ok = p < g.PS && i >= 0 && i <= g.n && j >= 0 && j <= g.n;
    bc_mbar_wait(&bar[st], (it >> 1) & 1);
    if (ok)
      inc_vertex_stage<TRANS, kSegLen>(std::make_integer_sequence<int, NR>{}, g, i, j, k,
                              g.PS * (k + 1) + p, alpha, sm + st * NSEG * kSegLen, shift[st], t,
                              y);
    __syncthreads();  // the stage is free for the chunk after next
  }
}

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
// padded plane; grids cover local planes [kbeg(), kend()). (32 x 8 vertex
// tiles per block, for L1 reuse of the dj neighbours, measured slower: K-Q
// 3.50 vs 3.20 ms in the same build.)
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
  k_lat_q<<<dim3(blocks(g.PS), (unsigned)(ke - kb)), kLT, 0, s>>>(g, kb, qc.p, E.p, T.p);
  SFEEC_LAUNCH_CHECK();
}
template <bool TRANS, int kCH>
static void launch_inc_bulk(const LatGeom& g, int kb, int ke, double alpha, const double* x,
                            double* y, cudaStream_t s) {
  constexpr int NSEG = IncTab<TRANS>::nseg();
  const int smem = 2 * NSEG * (kCH + 4) * (int)sizeof(double);
  static int per_sm = 0, sms = 0;  // resident CTAs (the shared memory decides)
  if (!per_sm) {
    SFEEC_CUDA(cudaFuncSetAttribute(k_lat_inc_bulk<TRANS, kCH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SFEEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lat_inc_bulk<TRANS, kCH>, kCH,
                                                             smem));
    int dev = 0;
    SFEEC_CUDA(cudaGetDevice(&dev));
    SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    per_sm = std::max(per_sm, 1);
  }
  const int64_t nchunk = ((g.PS + kCH - 1) / kCH) * (int64_t)(ke - kb);
  const unsigned grid = (unsigned)std::min<int64_t>(nchunk, (int64_t)per_sm * sms);
  k_lat_inc_bulk<TRANS, kCH><<<grid, kCH, smem, s>>>(g, kb, ke, alpha, x, y);
  SFEEC_LAUNCH_CHECK();
}

void Lattice::apply_cb(double h, cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  // t staged by bulk copies (measured, tet256: 0.71 vs 0.95 ms for the plain
  // k_lat_cb; the same staging of u slows K-CTe, 0.75-0.83 vs 0.66 ms: its 21
  // segments leave room for two CTAs per SM)
  launch_inc_bulk<false, 256>(g, kb, ke, -h, T.p, B.p, s);
}
void Lattice::apply_m2(cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  // (b staged by bulk copies: 1.83 / 2.25 ms vs 1.48, as for K-Q)
  k_lat_m2<<<dim3(blocks(g.PS), (unsigned)(ke - kb)), kLT, 0, s>>>(g, kb, mc.p, B.p, U.p);
  SFEEC_LAUNCH_CHECK();
}
void Lattice::apply_cte(double f, cudaStream_t s, int kb, int ke) const {
  if (kb < 0) kb = kbeg(), ke = kend();
  if (ke <= kb) return;
  k_lat_cte<<<dim3(blocks(g.PS), (unsigned)(ke - kb)), kLT, 0, s>>>(g, kb, f, U.p, E.p);
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
