// Device side of the Kuhn-lattice step (lattice.cu): the
// stencil rows unrolled at compile time from lattice_tables.hpp, the
// thread -> vertex maps and the four step kernels as templates over the map.
#pragma once
#include <utility>

#include "bulk_copy.cuh"
#include "lattice.cuh"
#include "lattice_tables.hpp"

namespace sfeec_b200 {
namespace latk {

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

// ---- thread -> vertex maps ------------------------------------------------
// MapLineN<NT>: a block is NT consecutive positions of one padded plane (grid
// y = plane). vertex(): this thread's vertex (i, j, local plane k) and lattice
// position; false off the mesh. (Brick-shaped maps were measured slower,
// lattice.cu.)
template <int NT>
struct MapLineN {
  static constexpr int kThreads = NT;
  __device__ static __forceinline__ bool vertex(const LatGeom& g, int kbeg, int kend, int& i,
                                                int& j, int& k, int64_t& idx) {
    const int p = blockIdx.x * NT + threadIdx.x;
    if (p >= g.PS) return false;
    k = kbeg + blockIdx.y;
    j = p / g.S - 1;
    i = p - (j + 1) * g.S - 1;
    idx = g.PS * (k + 1) + p;
    return i >= 0 && i <= g.n && j >= 0 && j <= g.n;
  }
  static dim3 grid(const LatGeom& g, int kb, int ke) {
    return dim3((unsigned)((g.PS + NT - 1) / NT), (unsigned)(ke - kb));
  }
};
using MapLine = MapLineN<kLT>;
// K-Q and K-M2 run 128-thread blocks, four per SM (the same 128 registers and
// 16 warps per SM as two 256-thread blocks; measured on tet256 over 300 steps:
// K-Q 2.006 -> 1.958 ms, K-M2 1.468 -> 1.452, step 4.84 -> 4.79; 64 threads the
// same, 512 slower)
constexpr int kSymThreads = 128;
using MapSym = MapLineN<kSymThreads>;
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
// 512 threads per SM: 128 registers, every load of the vertex's 7 rows in flight
// (measured: 80 / 64-register caps spill and run 1.6x / 2.4x slower; one
// block per SM at 247 registers runs 1.05x (K-Q) / 1.15x (K-M2) slower)
template <class Map>
__global__ void __launch_bounds__(Map::kThreads, 512 / Map::kThreads) k_lat_q(LatGeom g, int kbeg, int kend,
                                               const double* __restrict__ qc,
                                               const double* __restrict__ E,
                                               double* __restrict__ T) {
  int i, j, k;
  int64_t idx;
  if (!Map::vertex(g, kbeg, kend, i, j, k, idx)) return;
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
template <class Map>
__global__ void __launch_bounds__(Map::kThreads, 512 / Map::kThreads) k_lat_m2(LatGeom g, int kbeg, int kend,
                                                const double* __restrict__ mc,
                                                const double* __restrict__ B,
                                                double* __restrict__ U) {
  int i, j, k;
  int64_t idx;
  if (!Map::vertex(g, kbeg, kend, i, j, k, idx)) return;
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
template <class Map>
__global__ void __launch_bounds__(kLT) k_lat_cte(LatGeom g, int kbeg, int kend, double alpha,
                                                 const double* __restrict__ U,
                                                 double* __restrict__ E) {
  int i, j, k;
  int64_t idx;
  if (!Map::vertex(g, kbeg, kend, i, j, k, idx)) return;
  cte_vertex(std::make_integer_sequence<int, 7>{}, g, i, j, k, idx, alpha, U, E);
}

// ---- K-Cb: the gathered vector staged by bulk copies ------------------------
// K-Cb reads 14 distinct (component, dj, dk) row segments of t (K-CTe: 21 of u)
// around a chunk of kCH consecutive positions of one plane. One thread issues
// their bulk copies (cp.async.bulk) into a two-stage shared-memory ring one
// chunk ahead; the block's threads (one per position) sum the rows from shared
// memory and update b / e in place. Persistent CTAs take chunks round-robin.
constexpr int kSegLenMax = 256 + 34;  // doubles per staged segment at most (allocation slack)

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

template <bool TRANS, int kCH, int kAL = 2>
__global__ void __launch_bounds__(kCH)
    k_lat_inc_bulk(LatGeom g, int kbeg, int kend, double alpha, const double* __restrict__ x,
                   double* __restrict__ y) {
  // di in -1..1 plus the alignment of the copy's start (kAL doubles: 2 = the
  // 16 bytes a bulk copy needs, 16 = whole 128-byte lines)
  constexpr int kSegLen = kCH + 2 + kAL;
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
      const int64_t a0 = g0 & ~(int64_t)(kAL - 1);
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

}  // namespace latk
}  // namespace sfeec_b200
