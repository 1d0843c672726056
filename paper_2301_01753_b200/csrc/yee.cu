// Structured lumped-mass SFEEC (the Yee special case, config 2) on one B200.
//
// With Q = I/dV and M2 = dV I (lumped_mass, reference yee.cpp:76-81) the
// SplitScheme sub-flows become the FDTD stencils (yee.cpp:31-69):
//   e-kick  e_a += f*dV * [ (b_a2 - b_a2(-a1))/d_a1 - (b_a1 - b_a1(-a2))/d_a2 ]
//   b-kick  b_a += h/dV * [ (e_a1(+a2) - e_a1)/d_a2 - (e_a2(+a1) - e_a2)/d_a1 ]
// (f = dt c^2; b is the SFEEC 2-form, B = dV b). Strang half-kicks of
// consecutive steps are merged, so advance(n) = b-kick(dt/2), then n-1 fused
// (e-kick, b-kick) sweeps, then an e-kick and a final b-kick(dt/2).
//
// Kernels:
//   k_bkick / k_ekick   in-place, one thread per storage point (3 comps)
//   k_fused_pec         one e-kick + b-kick per pass, 2.5-D sweep along z:
//                       each CTA owns a TX x TY column tile and a z-chunk,
//                       stages the B planes (with a 1-point halo) and the
//                       freshly updated E planes in shared memory, so e and b
//                       are each read once and written once per step:
//                       2*w*(N1+N2) HBM bytes. Ping-pong
//                       buffers make tiles and chunks independent (halo
//                       points are recomputed, never exchanged).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "device_util.cuh"
#include "ipc_group.hpp"
#include "nccl_loader.hpp"
#include "yee_layout.hpp"

namespace sfeec_b200 {

template <class T>
struct Fields {
  T* c[6];  // ex ey ez bx by bz
};

template <class T>
struct YeeCoef {
  T ce[3];   // e-kick: f*m2/d_x, /d_y, /d_z
  T cb[3];   // b-kick: h*q/d_x, /d_y, /d_z
  T cb2[3];  // the two-step sweep's second b-kick (the closing half-kick of
             // an advance() is folded into its last sweep)
};

namespace {

constexpr int kThreads = 256;

// One curl update x + c1*d1 - c2*d2 with the rounding pinned, so every Yee
// kernel (one-step, fused, two-step) produces bitwise the same point values
// whatever the compiler would contract.
#ifndef YEE_UPD_MUL
// two chained FMAs, x + c1 d1 - c2 d2 = fma(c1, d1, fma(-c2, d2, x)): two
// FP64 operations and two dependent latencies per update
__device__ __forceinline__ double yee_upd(double x, double c1, double d1, double c2, double d2) {
  return __fma_rn(c1, d1, __fma_rn(-c2, d2, x));
}
__device__ __forceinline__ float yee_upd(float x, float c1, float d1, float c2, float d2) {
  return __fmaf_rn(c1, d1, __fmaf_rn(-c2, d2, x));
}
#else
// previous form: x + (c1 d1 - c2 d2), one mul, one fma, one add
__device__ __forceinline__ double yee_upd(double x, double c1, double d1, double c2, double d2) {
  return __dadd_rn(x, __fma_rn(c1, d1, -__dmul_rn(c2, d2)));
}
__device__ __forceinline__ float yee_upd(float x, float c1, float d1, float c2, float d2) {
  return __fadd_rn(x, __fmaf_rn(c1, d1, -__fmul_rn(c2, d2)));
}
#endif

// DOF masks (PEC), yee_layout.hpp. k is the local storage plane; the masks
// are evaluated at the global plane k + kofs, and only owned planes count.
__device__ __forceinline__ bool owned(const YeeGeom& g, int k) {
  return k >= g.kown_lo && k < g.kown_hi;
}
__device__ __forceinline__ bool e_dof(const YeeGeom& g, int a, int i, int j, int kl) {
  if (!owned(g, kl)) return false;
  if (g.bc == 0) return true;
  const int c[3] = {i, j, kl + g.kofs};
  for (int d = 0; d < 3; ++d) {
    if (d == a) {
      if (c[d] < 0 || c[d] >= g.n[d]) return false;
    } else if (c[d] < 1 || c[d] > g.n[d] - 1) {
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ bool b_dof(const YeeGeom& g, int a, int i, int j, int kl) {
  if (!owned(g, kl)) return false;
  const int c[3] = {i, j, kl + g.kofs};
  for (int d = 0; d < 3; ++d) {
    int hi = (g.bc == 0 || d != a) ? g.n[d] - 1 : g.n[d];
    if (c[d] < 0 || c[d] > hi) return false;
  }
  return true;
}

__device__ __forceinline__ int wrapm(int c, int n) { return c < 0 ? c + n : (c >= n ? c - n : c); }

// ---- unfused, in place ----------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_bkick(YeeGeom g, Fields<T> f, YeeCoef<T> k) {
  const int64_t np = g.npts();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < np;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(s % g.P0);
    const int j = (int)((s / g.P0) % g.S[1]);
    const int kk = (int)(s / ((int64_t)g.P0 * g.S[1]));
    if (i >= g.S[0] || kk >= g.S[2]) continue;  // row / tail padding
    int ip = i + 1, jp = j + 1, kp = kk + 1;
    if (g.bc == 0) {
      ip = wrapm(ip, g.n[0]);
      jp = wrapm(jp, g.n[1]);
      kp = wrapm(kp, g.n[2]);
    }
    const T* ex = f.c[0];
    const T* ey = f.c[1];
    const T* ez = f.c[2];
    if (b_dof(g, 0, i, j, kk)) {
      const T ey0 = ey[s], ez0 = ez[s];
      f.c[3][s] = yee_upd(f.c[3][s], k.cb[2], ey[g.sidx(i, j, kp)] - ey0, k.cb[1], ez[g.sidx(i, jp, kk)] - ez0);
    }
    if (b_dof(g, 1, i, j, kk)) {
      const T ez0 = ez[s], ex0 = ex[s];
      f.c[4][s] = yee_upd(f.c[4][s], k.cb[0], ez[g.sidx(ip, j, kk)] - ez0, k.cb[2], ex[g.sidx(i, j, kp)] - ex0);
    }
    if (b_dof(g, 2, i, j, kk)) {
      const T ex0 = ex[s], ey0 = ey[s];
      f.c[5][s] = yee_upd(f.c[5][s], k.cb[1], ex[g.sidx(i, jp, kk)] - ex0, k.cb[0], ey[g.sidx(ip, j, kk)] - ey0);
    }
  }
}

template <class T>
__global__ void __launch_bounds__(kThreads) k_ekick(YeeGeom g, Fields<T> f, YeeCoef<T> k) {
  const int64_t np = g.npts();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < np;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(s % g.P0);
    const int j = (int)((s / g.P0) % g.S[1]);
    const int kk = (int)(s / ((int64_t)g.P0 * g.S[1]));
    if (i >= g.S[0] || kk >= g.S[2]) continue;  // row / tail padding
    int im = i - 1, jm = j - 1, km = kk - 1;
    if (g.bc == 0) {
      im = wrapm(im, g.n[0]);
      jm = wrapm(jm, g.n[1]);
      km = wrapm(km, g.n[2]);
    }
    const T* bx = f.c[3];
    const T* by = f.c[4];
    const T* bz = f.c[5];
    if (e_dof(g, 0, i, j, kk)) {
      const T bz0 = bz[s], by0 = by[s];
      f.c[0][s] = yee_upd(f.c[0][s], k.ce[1], bz0 - bz[g.sidx(i, jm, kk)], k.ce[2], by0 - by[g.sidx(i, j, km)]);
    }
    if (e_dof(g, 1, i, j, kk)) {
      const T bx0 = bx[s], bz0 = bz[s];
      f.c[1][s] = yee_upd(f.c[1][s], k.ce[2], bx0 - bx[g.sidx(i, j, km)], k.ce[0], bz0 - bz[g.sidx(im, j, kk)]);
    }
    if (e_dof(g, 2, i, j, kk)) {
      const T by0 = by[s], bx0 = bx[s];
      f.c[2][s] = yee_upd(f.c[2][s], k.ce[0], by0 - by[g.sidx(im, j, kk)], k.ce[1], bx0 - bx[g.sidx(i, jm, kk)]);
    }
  }
}

// ---- fused e-kick + b-kick sweep (PEC) -------------------------------------
template <class T, int TX, int TY>
__global__ void __launch_bounds__(TX* TY)
    k_fused_pec(YeeGeom g, Fields<T> in, Fields<T> out, YeeCoef<T> ck, int kchunk) {
  constexpr int BX = TX + 2, BY = TY + 2;  // B tile incl. 1-point halo on both sides
  constexpr int EX = TX + 1, EY = TY + 1;  // E tile incl. 1-point halo on + side
  __shared__ T sB[2][3][BY][BX];
  __shared__ T sE[2][3][EY][EX];
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int Z = g.S[2];
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, Z);
  if (k0 >= Z) return;

  auto load_b = [&](int buf, int kp) {
    for (int p = tid; p < BX * BY; p += TX * TY) {
      const int ei = p % BX, ej = p / BX;
      const int i = i0 - 1 + ei, j = j0 - 1 + ej;
      const bool in_range = kp >= 0 && kp < Z && i >= 0 && i < g.S[0] && j >= 0 && j < g.S[1];
      const int64_t s = in_range ? g.sidx(i, j, kp) : 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) sB[buf][c][ej][ei] = in_range ? in.c[3 + c][s] : T(0);
    }
  };

  int cur = 0;
  load_b(1, k0 - 1);  // B_old(k0-1) -> prev
  for (int kk = k0; kk <= k1; ++kk) {
    const int prev = cur ^ 1;
    load_b(cur, kk);
    __syncthreads();
    // E_new(kk) on [i0, i0+TX] x [j0, j0+TY]
    for (int p = tid; p < EX * EY; p += TX * TY) {
      const int li = p % EX, lj = p / EX;
      const int i = i0 + li, j = j0 + lj;
      const int bi = li + 1, bj = lj + 1;
      const bool in_range = kk < Z && i < g.S[0] && j < g.S[1];
      const int64_t s = in_range ? g.sidx(i, j, kk) : 0;
      T e[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) e[c] = in_range ? in.c[c][s] : T(0);
      if (in_range) {
        if (e_dof(g, 0, i, j, kk))
          e[0] = yee_upd(e[0], ck.ce[1], sB[cur][2][bj][bi] - sB[cur][2][bj - 1][bi], ck.ce[2], sB[cur][1][bj][bi] - sB[prev][1][bj][bi]);
        if (e_dof(g, 1, i, j, kk))
          e[1] = yee_upd(e[1], ck.ce[2], sB[cur][0][bj][bi] - sB[prev][0][bj][bi], ck.ce[0], sB[cur][2][bj][bi] - sB[cur][2][bj][bi - 1]);
        if (e_dof(g, 2, i, j, kk))
          e[2] = yee_upd(e[2], ck.ce[0], sB[cur][1][bj][bi] - sB[cur][1][bj][bi - 1], ck.ce[1], sB[cur][0][bj][bi] - sB[cur][0][bj - 1][bi]);
        if (li < TX && lj < TY && kk < k1) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            if (e_dof(g, c, i, j, kk)) out.c[c][s] = e[c];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) sE[cur][c][lj][li] = e[c];
    }
    __syncthreads();
    // B_new(kk-1) on the own tile
    if (kk > k0) {
      const int li = tid % TX, lj = tid / TX;
      const int i = i0 + li, j = j0 + lj, kb = kk - 1;
      if (i < g.S[0] && j < g.S[1]) {
        const int64_t s = g.sidx(i, j, kb);
        const int bi = li + 1, bj = lj + 1;
        if (b_dof(g, 0, i, j, kb))
          out.c[3][s] = yee_upd(sB[prev][0][bj][bi], ck.cb[2], sE[cur][1][lj][li] - sE[prev][1][lj][li], ck.cb[1], sE[prev][2][lj + 1][li] - sE[prev][2][lj][li]);
        if (b_dof(g, 1, i, j, kb))
          out.c[4][s] = yee_upd(sB[prev][1][bj][bi], ck.cb[0], sE[prev][2][lj][li + 1] - sE[prev][2][lj][li], ck.cb[2], sE[cur][0][lj][li] - sE[prev][0][lj][li]);
        if (b_dof(g, 2, i, j, kb))
          out.c[5][s] = yee_upd(sB[prev][2][bj][bi], ck.cb[1], sE[prev][0][lj + 1][li] - sE[prev][0][lj][li], ck.cb[0], sE[prev][1][lj][li + 1] - sE[prev][1][lj][li]);
      }
    }
    __syncthreads();
    cur ^= 1;
  }
}

// ---- fused sweep, TMA-pipelined, persistent (PEC; the default) -------------
// Same arithmetic as k_fused_pec, but every B/E plane tile (with halo) is
// fetched by one elected thread with cp.async.bulk.tensor (TMA) into an
// NS-stage shared-memory ring, D = NS-2 planes ahead of the sweep, completion
// tracked by one mbarrier per stage. Out-of-box coordinates (the -1 halo and
// the PEC walls) are zero-filled by the TMA unit. CTAs are persistent and take
// (z-chunk, tile) work units round-robin in chunk-major order, so CTAs running
// concurrently sweep neighbouring tiles over the same planes and the halo
// re-reads hit L2. Only the compute domain [0,n)^3 is swept: the faces on the
// far PEC walls have empty C rows and stay constant (present in both buffers).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// TMA requires the innermost box coordinate to be 16-byte aligned (measured:
// a -1 start faults with "illegal instruction"), so the B tile starts OFF =
// 16/sizeof(T) points left of the tile instead of 1; widths are rounded to
// 16-byte multiples.
template <class T, int TX, int TY, int NS>
struct TmaCfg {
  static constexpr int kOff = 16 / (int)sizeof(T);
  static constexpr int kBWB = (((TX + 1 + kOff) * (int)sizeof(T) + 15) / 16 * 16) / (int)sizeof(T);
  static constexpr int kBWE = (((TX + 1) * (int)sizeof(T) + 15) / 16 * 16) / (int)sizeof(T);
  static constexpr int kBBox = 3 * (TY + 2) * kBWB * (int)sizeof(T);  // bytes per B plane tile
  static constexpr int kEBox = 3 * (TY + 1) * kBWE * (int)sizeof(T);  // bytes per E plane tile
  static constexpr int kBStride = (kBBox + 127) / 128 * 128;
  static constexpr int kEStride = (kEBox + 127) / 128 * 128;
  static constexpr int kStage = kBStride + kEStride;
  static constexpr int kEnew = 3 * (TY + 1) * (TX + 1);  // elements per E_new buffer
  static constexpr int kBarOff = (NS * kStage + 3 * kEnew * (int)sizeof(T) + 15) / 16 * 16;
  static constexpr int kSmem = kBarOff + NS * 8 + 128;
  static constexpr int kD = NS - 3;  // prefetch distance in planes
};

// One CTA = TX*TY threads. Per plane kk of a unit:
//   wait(stage of plane kk) -> E_new(kk) on the (TX+1)x(TY+1) region from the
//   staged B(kk), B(kk-1), E(kk) -> sync -> B_new(kk-1) on the own tile from
//   E_new(kk-1), E_new(kk) and the staged B(kk-1).
// One __syncthreads per plane: E_new is triple-buffered and the TMA ring has
// D + 3 stages, so the producer never overwrites a stage or an E_new buffer
// that a lagging warp of the previous plane may still read.
template <class T, int TX, int TY, int NS, int NTH>
__global__ void __launch_bounds__(NTH)
    k_fused_tma(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapE,
                YeeGeom g, Fields<T> out, YeeCoef<T> ck, int kchunk, int n_tiles_x, int n_tiles,
                int n_units, int kbeg, int kend) {
  using Cfg = TmaCfg<T, TX, TY, NS>;
  constexpr int D = Cfg::kD;
  constexpr int BWB = Cfg::kBWB, BWE = Cfg::kBWE, OFF = Cfg::kOff;
  constexpr int NT = NTH, NE = (TX + 1) * (TY + 1);
  static_assert(NE <= 2 * NT && TX * TY <= NT, "E region needs at most two passes");
  extern __shared__ unsigned char smem_raw[];
  // 128-byte aligned start, as an offset into the shared array so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* sEn = reinterpret_cast<T*>(base + NS * Cfg::kStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + Cfg::kBarOff);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapE)) : "memory");
  }
  __syncthreads();
  uint32_t gplane = 0;  // planes issued by this CTA so far (stage = gp % NS, parity = gp / NS)
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int64_t kstride = (int64_t)g.P0 * g.S[1];
  // E-region points of this thread: pass 0 -> p = tid, pass 1 -> p = tid + NT
  const int pl[2] = {tid, tid + NT};
  int li_[2], lj_[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    li_[q] = pl[q] % (TX + 1);
    lj_[q] = pl[q] / (TX + 1);
  }
  const bool has1 = tid < NE, has2 = tid + NT < NE;
  const int bli = tid % TX, blj = tid / TX;  // own B point (tid < TX * TY)

  for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
    const int chunk = unit / n_tiles, tile = unit - chunk * n_tiles;
    const int i0 = (tile % n_tiles_x) * TX, j0 = (tile / n_tiles_x) * TY;
    // local planes [kbeg, kend) are swept (single domain: [0, n); slab: the
    // owned planes between the ghosts); masks use the global plane kk + kofs
    const int k0 = kbeg + chunk * kchunk, k1 = min(k0 + kchunk, kend);
    const int P = k1 - k0 + 2;  // local planes p <-> z = k0 - 1 + p
    // (i, j) parts of the PEC DOF masks (yee_layout.hpp) and write permissions
    uint32_t m[2];
    int64_t sij[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = i0 + li_[q], j = j0 + lj_[q];
      const bool ix = i < n0, iy = i >= 1 && i <= n0 - 1;
      const bool jx = j < n1, jy = j >= 1 && j <= n1 - 1;
      const bool own = li_[q] < TX && lj_[q] < TY && i < n0 && j < n1 && pl[q] < NE;
      m[q] = (ix && jy ? 1u : 0u) | (iy && jx ? 2u : 0u) | (iy && jy ? 4u : 0u) | (own ? 8u : 0u);
      sij[q] = (int64_t)i + (int64_t)g.P0 * j;
    }
    const bool bown = tid < TX * TY && i0 + bli < n0 && j0 + blj < n1;
    const int64_t bsij = (int64_t)(i0 + bli) + (int64_t)g.P0 * (j0 + blj);

    auto issue = [&](int p) {
      const uint32_t gp = gplane + p;
      const int st = gp % NS;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(&bars[st], Cfg::kBBox + Cfg::kEBox);
      tma_load_4d(base + st * Cfg::kStage, &mapB, &bars[st], i0 - OFF, j0 - 1, k0 - 1 + p, 3);
      tma_load_4d(base + st * Cfg::kStage + Cfg::kBStride, &mapE, &bars[st], i0, j0, k0 - 1 + p, 0);
    };
    if (tid == 0)
      for (int p = 0; p <= D && p < P; ++p) issue(p);
    for (int jp = 0; jp + 1 < P; ++jp) {
      const int kk = k0 + jp;
      if (tid == 0 && jp + 1 + D < P) issue(jp + 1 + D);
      const uint32_t gc = gplane + jp + 1, gv = gplane + jp;
      const int sc = gc % NS, sv = gv % NS;
      if (jp == 0) mbar_wait(&bars[sv], (gv / NS) & 1);
      mbar_wait(&bars[sc], (gc / NS) & 1);
      const T* __restrict__ Bc = reinterpret_cast<const T*>(base + sc * Cfg::kStage);
      const T* __restrict__ Bp = reinterpret_cast<const T*>(base + sv * Cfg::kStage);
      const T* __restrict__ Ec = reinterpret_cast<const T*>(base + sc * Cfg::kStage + Cfg::kBStride);
      T* Enc = sEn + ((gplane + jp) % 3) * Cfg::kEnew;
      const T* Enp = sEn + ((gplane + jp + 2) % 3) * Cfg::kEnew;
#define BC(c, y, x) Bc[((c) * (TY + 2) + (y)) * BWB + (x)]
#define BP(c, y, x) Bp[((c) * (TY + 2) + (y)) * BWB + (x)]
#define EC(c, y, x) Ec[((c) * (TY + 1) + (y)) * BWE + (x)]
#define EN(buf, c, y, x) buf[((c) * (TY + 1) + (y)) * (TX + 1) + (x)]
      const int kg = kk + g.kofs;
      const bool kin = kg >= 1 && kg <= n2 - 1, kz = kg < n2, kw = kk < k1;
      // E_new(kk) on [i0, i0+TX] x [j0, j0+TY]
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if ((q == 0 && !has1) || (q == 1 && !has2)) break;
        const int li = li_[q], lj = lj_[q];
        const int bi = li + OFF, bj = lj + 1;
        T e0 = EC(0, lj, li), e1 = EC(1, lj, li), e2 = EC(2, lj, li);
        const bool d0 = (m[q] & 1) && kin, d1 = (m[q] & 2) && kin, d2 = (m[q] & 4) && kz;
        if (d0)
          e0 = yee_upd(e0, ck.ce[1], BC(2, bj, bi) - BC(2, bj - 1, bi), ck.ce[2], BC(1, bj, bi) - BP(1, bj, bi));
        if (d1)
          e1 = yee_upd(e1, ck.ce[2], BC(0, bj, bi) - BP(0, bj, bi), ck.ce[0], BC(2, bj, bi) - BC(2, bj, bi - 1));
        if (d2)
          e2 = yee_upd(e2, ck.ce[0], BC(1, bj, bi) - BC(1, bj, bi - 1), ck.ce[1], BC(0, bj, bi) - BC(0, bj - 1, bi));
        if ((m[q] & 8) && kw) {
          const int64_t s = sij[q] + kstride * kk;
          if (d0) out.c[0][s] = e0;
          if (d1) out.c[1][s] = e1;
          if (d2) out.c[2][s] = e2;
        }
        EN(Enc, 0, lj, li) = e0;
        EN(Enc, 1, lj, li) = e1;
        EN(Enc, 2, lj, li) = e2;
      }
      __syncthreads();
      // B_new(kk-1) on the own tile (every face of [0,n)^3 is a DOF)
      if (jp > 0 && bown) {
        const int li = bli, lj = blj;
        const int64_t s = bsij + kstride * (kk - 1);
        const int bi = li + OFF, bj = lj + 1;
        out.c[3][s] = yee_upd(BP(0, bj, bi), ck.cb[2], EN(Enc, 1, lj, li) - EN(Enp, 1, lj, li), ck.cb[1], EN(Enp, 2, lj + 1, li) - EN(Enp, 2, lj, li));
        out.c[4][s] = yee_upd(BP(1, bj, bi), ck.cb[0], EN(Enp, 2, lj, li + 1) - EN(Enp, 2, lj, li), ck.cb[2], EN(Enc, 0, lj, li) - EN(Enp, 0, lj, li));
        out.c[5][s] = yee_upd(BP(2, bj, bi), ck.cb[1], EN(Enp, 0, lj + 1, li) - EN(Enp, 0, lj, li), ck.cb[0], EN(Enp, 1, lj, li + 1) - EN(Enp, 1, lj, li));
      }
#undef BC
#undef BP
#undef EC
#undef EN
    }
    gplane += P;
    __syncthreads();  // unit boundary: the next unit's prologue refills every stage
  }
}
// ---- variant 4: two leapfrog steps per z-sweep (temporal blocking) --------
// The sweep of k_fused_tma advances one (e-kick, b-kick) pair per pass; this
// one advances two: per plane z of a unit it computes
//   E1(z) -> B1(z-1) -> E2(z-1) -> B2(z-2)
// (1 = after the first pair, 2 = after the second), keeping E1, B1 and E2 in
// shared memory (triple-buffered planes) and writing only E2 and B2, so e and
// b are read and written once per TWO steps. The regions shrink by one point
// per half step on the sides the staggered differences reach (E uses B at
// -1, B uses E at +1): E1 on [i0-1, i0+TX+1] x [j0-1, j0+TY+1], B1 on
// [i0-1, i0+TX] x [j0-1, j0+TY], E2 on [i0, i0+TX] x [j0, j0+TY], B2 on the
// tile; the B0 / E0 boxes start at i0 - OFF (TMA's 16-byte alignment; OFF =
// 16/sizeof(T) >= 2). Every point update is the same expression as in
// k_fused_tma (yee_e_upd / yee_b_upd), so the result equals two single
// sweeps. Two barriers per plane; NS = D + 1 TMA stages; the E1 and E2
// planes are double-buffered, B1 single, so with NS = 3 two CTAs fit per SM
// (fp64). One thread per E1-region point keeps that point's E1, B1, E2 and
// old B of the current and previous plane in registers.
template <class T, int TX, int TY, int NS, int NB1 = 1>
struct TmaCfg2 {
  static constexpr int kOff = 16 / (int)sizeof(T);
  static constexpr int kBW = (((TX + 2 + kOff) * (int)sizeof(T) + 15) / 16 * 16) / (int)sizeof(T);
  static constexpr int kBBox = 3 * (TY + 4) * kBW * (int)sizeof(T);  // B0: y in [j0-2, j0+TY+1]
  static constexpr int kEBox = 3 * (TY + 3) * kBW * (int)sizeof(T);  // E0: y in [j0-1, j0+TY+1]
  static constexpr int kBStride = (kBBox + 127) / 128 * 128;
  static constexpr int kEStride = (kEBox + 127) / 128 * 128;
  static constexpr int kStage = kBStride + kEStride;
  static constexpr int kX1 = TX + 3, kY1 = TY + 3;  // E1 region, origin (i0-1, j0-1)
  static constexpr int kXB = TX + 2, kYB = TY + 2;  // B1 region, origin (i0-1, j0-1)
  static constexpr int kX2 = TX + 1, kY2 = TY + 1;  // E2 region, origin (i0, j0)
  static constexpr int kE1 = 3 * kX1 * kY1, kB1 = 3 * kXB * kYB, kE2 = 3 * kX2 * kY2;
  // E1 and E2 planes double-buffered, B1 single (NB1 = 1) or double (NB1 =
  // 2), all on the E1 region grid
  static constexpr int kBufBytes = (4 + NB1) * 3 * kX1 * kY1 * (int)sizeof(T);
  static constexpr int kBarOff = (NS * kStage + kBufBytes + 15) / 16 * 16;
  static constexpr int kSmem = kBarOff + NS * 8 + 128;
  // prefetch distance in planes: a stage is read only in phase 1 of its own
  // plane (the own old B is carried to the next plane in registers), so the
  // stage of plane p-1 is free once plane p starts
  static constexpr int kD = NS - 1;
};

// E DOF mask bits of (i, j) (yee_layout.hpp): 1 Ex, 2 Ey, 4 Ez (z parts apart)
__device__ __forceinline__ uint32_t e_mask_xy(int i, int j, int n0, int n1) {
  const bool ix = i >= 0 && i < n0, iy = i >= 1 && i <= n0 - 1;
  const bool jx = j >= 0 && j < n1, jy = j >= 1 && j <= n1 - 1;
  return (ix && jy ? 1u : 0u) | (iy && jx ? 2u : 0u) | (iy && jy ? 4u : 0u);
}

// The B1 plane is double-buffered: phase 2 of plane p+1 writes the other
// buffer than the one phase 3 of plane p reads, and the only other reason for
// a barrier between phases 1 and 2 (E1(z-1) neighbours) is already covered by
// the previous plane's barrier, so each plane needs one barrier, not two.
// The E1-region points are ordered so that the TX x TY own tile comes first,
// one warp per tile row (TX = 32), then the rims the E2, B1 and E1 regions
// add. Phases 2-4 run only on their region's points (the others' values are
// never read), so the idle rim warps skip them, and the own-point stores are
// whole 32-wide rows.
template <int TX, int TY>
__device__ __forceinline__ void region_point(int t, int& x, int& y) {
  constexpr int kOwn = TX * TY;
  constexpr int kE2 = kOwn + TY + (TX + 1);       // + column TX+1, row TY+1
  constexpr int kB1 = kE2 + (TY + 2) + (TX + 1);  // + column 0, row 0
  if (t < kOwn) {
    x = 1 + t % TX;
    y = 1 + t / TX;
  } else if (t < kE2) {
    const int u = t - kOwn;
    if (u < TY) {
      x = TX + 1;
      y = 1 + u;
    } else {
      x = 1 + (u - TY);
      y = TY + 1;
    }
  } else if (t < kB1) {
    const int u = t - kE2;
    if (u < TY + 2) {
      x = 0;
      y = u;
    } else {
      x = 1 + (u - (TY + 2));
      y = 0;
    }
  } else {  // E1 rim: column TX+2 (y 0..TY+2), row TY+2 (x 0..TX+1)
    const int u = t - kB1;
    if (u < TY + 3) {
      x = TX + 2;
      y = u;
    } else {
      x = u - (TY + 3);
      y = TY + 2;
    }
  }
}

template <class T, int TX, int TY, int NS, int NTH, int NPT, int MINB>
__global__ void __launch_bounds__(NTH, MINB)
    k_fused2_tma(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapE,
                 YeeGeom g, Fields<T> out, YeeCoef<T> ck, int kchunk, int n_tiles_x, int n_tiles,
                 int n_units, int kbeg, int kend, const int4* __restrict__ sched,
                 const int* __restrict__ cta_ptr) {
  constexpr int NB1 = 2;
  using Cfg = TmaCfg2<T, TX, TY, NS, NB1>;
  constexpr int D = Cfg::kD, BW = Cfg::kBW, OFF = Cfg::kOff;
  // NPT points of the E1 region (origin (i0-1, j0-1)) per thread: points
  // tid + h*NH, h < NPT. The B1, E2 and B2 regions are subsets in the same
  // coordinates, so a thread keeps its points' E1, B1, E2 and old B of the
  // current and previous plane in registers; only the x/y neighbours go
  // through shared memory. Several points per thread amortise the per-plane
  // control (barrier waits, stage and buffer addressing) and add ILP.
  constexpr int X1 = Cfg::kX1, Y1 = Cfg::kY1, NP = X1 * Y1;
  // (the stride is rounded up to whole warps, so every h keeps the
  // one-tile-row-per-warp layout)
  constexpr int NH = ((NP + NPT - 1) / NPT + 31) / 32 * 32;
  static_assert(NH <= NTH, "NPT region points per thread");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* sE1 = reinterpret_cast<T*>(base + NS * Cfg::kStage);  // 2 planes x 3 comps x NP
  T* sB1 = sE1 + 2 * 3 * NP;                                 // NB1 planes
  T* sE2 = sB1 + NB1 * 3 * NP;                               // 2 planes
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + Cfg::kBarOff);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapE)) : "memory");
  }
  __syncthreads();
  uint32_t gplane = 0;
  const int n0 = g.n[0], n1 = g.n[1], n2 = g.n[2];
  const int64_t kstride = (int64_t)g.P0 * g.S[1];
  // own points: region index me[h], box offsets (B0: row bj, col bi; E0: row
  // ej, col bi), region membership
  int me[NPT], xo[NPT], yo[NPT], ob[NPT], oe[NPT];
  bool pt[NPT], inB1[NPT], inE2[NPT];
#pragma unroll
  for (int h = 0; h < NPT; ++h) {
    const int t = tid + h * NH;
    pt[h] = tid < NH && t < NP;
    region_point<TX, TY>(t, xo[h], yo[h]);  // own tile rows, then the rims
    me[h] = yo[h] * X1 + xo[h];  // shared-memory index on the E1 region grid
    ob[h] = (yo[h] + 1) * BW + xo[h] + OFF - 1;
    oe[h] = yo[h] * BW + xo[h] + OFF - 1;
    inB1[h] = pt[h] && xo[h] <= TX + 1 && yo[h] <= TY + 1;
    inE2[h] = pt[h] && xo[h] >= 1 && xo[h] <= TX + 1 && yo[h] >= 1 && yo[h] <= TY + 1;
  }
  const bool any = pt[0];  // point 0 exists whenever any does
  // PDL: everything above is prologue; the previous sweep's output is read
  // from here on (a no-op without a programmatic launch)
  pdl_wait();
  pdl_trigger();

  // per-point state of one plane: E1, B1, E2 and the old B (B0). Two sets
  // ping-pong (cur/prev) through a 2x unrolled plane loop, so no register
  // moves rotate them.
  struct Pt {
    T e1[3], b1[3], e2[3], b0[3];
  };
  const T ce0 = ck.ce[0], ce1 = ck.ce[1], ce2 = ck.ce[2];
  const T cb0 = ck.cb[0], cb1 = ck.cb[1], cb2 = ck.cb[2];
  const T db0 = ck.cb2[0], db1 = ck.cb2[1], db2 = ck.cb2[2];  // second b-kick

  // units: (tile, z-chunk) round-robin over the CTAs, or, with a schedule,
  // the CTA's own list of (tile, k0, k1) (Yee2Sched)
  const int u_beg = sched ? cta_ptr[blockIdx.x] : (int)blockIdx.x;
  const int u_end = sched ? cta_ptr[blockIdx.x + 1] : n_units;
  const int u_step = sched ? 1 : (int)gridDim.x;
  for (int unit = u_beg; unit < u_end; unit += u_step) {
    int tile, k0, k1;
    if (sched) {
      const int4 w = sched[unit];
      tile = w.x;
      k0 = w.y;
      k1 = w.z;
    } else {
      const int chunk = unit / n_tiles;
      tile = unit - chunk * n_tiles;
      k0 = kbeg + chunk * kchunk;
      k1 = min(k0 + kchunk, kend);
    }
    const int i0 = (tile % n_tiles_x) * TX, j0 = (tile / n_tiles_x) * TY;
    const int P = k1 - k0 + 4;  // local planes p <-> z = k0 - 2 + p
    uint32_t m[NPT];
    bool b1up[NPT], own[NPT];
    int64_t sij[NPT];
#pragma unroll
    for (int h = 0; h < NPT; ++h) {
      const int i = i0 - 1 + xo[h], j = j0 - 1 + yo[h];
      m[h] = pt[h] ? e_mask_xy(i, j, n0, n1) : 0u;
      b1up[h] = inB1[h] && i >= 0 && i < n0 && j >= 0 && j < n1;
      own[h] = inE2[h] && xo[h] <= TX && yo[h] <= TY && i < n0 && j < n1;
      sij[h] = (int64_t)i + (int64_t)g.P0 * j;
    }

    auto issue = [&](int p) {
      const uint32_t gp = gplane + p;
      const int st = gp % NS;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(&bars[st], Cfg::kBBox + Cfg::kEBox);
      tma_load_4d(base + st * Cfg::kStage, &mapB, &bars[st], i0 - OFF, j0 - 2, k0 - 2 + p, 3);
      tma_load_4d(base + st * Cfg::kStage + Cfg::kBStride, &mapE, &bars[st], i0 - OFF, j0 - 1,
                  k0 - 2 + p, 0);
    };
    if (tid == 0)
      for (int p = 0; p < D && p < P; ++p) issue(p);

    // plane p of the unit (PAR = p & 1 selects the E1/E2 double buffers at
    // compile time): C receives this plane's values, V holds the previous
    // plane's
    auto plane = [&](auto par, int p, Pt* C, const Pt* V) {
      constexpr int PAR = decltype(par)::value;
      const uint32_t gc = gplane + p;
      const int st = gc % NS;
      if (tid == 0 && p + D < P) issue(p + D);
      mbar_wait(&bars[st], (gc / NS) & 1);
      const int z = k0 - 2 + p;
      const T* __restrict__ B0c = reinterpret_cast<const T*>(base + st * Cfg::kStage);
      const T* __restrict__ E0c = reinterpret_cast<const T*>(base + st * Cfg::kStage + Cfg::kBStride);
      T* E1z = sE1 + PAR * 3 * NP;            // E1(z)
      const T* E1y = sE1 + (1 - PAR) * 3 * NP;  // E1(z-1)
      T* E2y = sE2 + (1 - PAR) * 3 * NP;        // E2(z-1)
      T* B1p = sB1 + PAR * 3 * NP;              // B1(z-1)
      const T* E2x = sE2 + PAR * 3 * NP;        // E2(z-2)
      constexpr int BC = (TY + 4) * BW, EC = (TY + 3) * BW;  // component strides in the boxes
#define R(buf, c, idx) buf[(c) * NP + (idx)]
      // ---- phase 1: E1(z); the own B0(z) is kept for the next plane (it is
      // B0(z-1) there)
      if (any) {
        const int zg = z + g.kofs;
        const bool kin = zg >= 1 && zg <= n2 - 1, kz = zg >= 0 && zg < n2;
#pragma unroll
        for (int h = 0; h < NPT; ++h) {
          if (!pt[h]) continue;
          const T* b = B0c + ob[h];
          C[h].b0[0] = b[0];
          C[h].b0[1] = b[BC];
          C[h].b0[2] = b[2 * BC];
          if (p >= 1) {
            const T* e = E0c + oe[h];
            const T e0 = e[0], e1 = e[EC], e2 = e[2 * EC];
            const T u0 = yee_upd(e0, ce1, C[h].b0[2] - b[2 * BC - BW], ce2, C[h].b0[1] - V[h].b0[1]);
            const T u1 = yee_upd(e1, ce2, C[h].b0[0] - V[h].b0[0], ce0, C[h].b0[2] - b[2 * BC - 1]);
            const T u2 = yee_upd(e2, ce0, C[h].b0[1] - b[BC - 1], ce1, C[h].b0[0] - b[-BW]);
            C[h].e1[0] = (m[h] & 1) && kin ? u0 : e0;
            C[h].e1[1] = (m[h] & 2) && kin ? u1 : e1;
            C[h].e1[2] = (m[h] & 4) && kz ? u2 : e2;
            R(E1z, 0, me[h]) = C[h].e1[0];
            R(E1z, 1, me[h]) = C[h].e1[1];
            R(E1z, 2, me[h]) = C[h].e1[2];
          }
        }
      }
      // ---- phase 2: B1(z-1) (E1(z-1) neighbours from smem)
      if (p >= 2 && any) {
        const int zg = z - 1 + g.kofs;
        const bool zin = zg >= 0 && zg < n2;
#pragma unroll
        for (int h = 0; h < NPT; ++h) {
          if (!inB1[h]) continue;
          const int q = me[h];
          const bool up = b1up[h] && zin;
          const Pt& v = V[h];
          const T u0 = yee_upd(v.b0[0], cb2, C[h].e1[1] - v.e1[1], cb1, R(E1y, 2, q + X1) - v.e1[2]);
          const T u1 = yee_upd(v.b0[1], cb0, R(E1y, 2, q + 1) - v.e1[2], cb2, C[h].e1[0] - v.e1[0]);
          const T u2 = yee_upd(v.b0[2], cb1, R(E1y, 0, q + X1) - v.e1[0], cb0, R(E1y, 1, q + 1) - v.e1[1]);
          C[h].b1[0] = up ? u0 : v.b0[0];
          C[h].b1[1] = up ? u1 : v.b0[1];
          C[h].b1[2] = up ? u2 : v.b0[2];
          R(B1p, 0, q) = C[h].b1[0];
          R(B1p, 1, q) = C[h].b1[1];
          R(B1p, 2, q) = C[h].b1[2];
        }
      }
      __syncthreads();  // B1(z-1) complete
      // ---- phase 3: E2(z-1) (B1(z-1) neighbours from smem)
      if (p >= 3 && any) {
        const int ze = z - 1;
        const int zg = ze + g.kofs;
        const bool kin = zg >= 1 && zg <= n2 - 1, kz = zg >= 0 && zg < n2;
        const bool zw = ze >= k0 && ze < k1;
#pragma unroll
        for (int h = 0; h < NPT; ++h) {
          if (!inE2[h]) continue;
          const int q = me[h];
          const Pt& v = V[h];
          const bool d0 = (m[h] & 1) && kin, d1 = (m[h] & 2) && kin, d2 = (m[h] & 4) && kz;
          const T u0 = yee_upd(v.e1[0], ce1, C[h].b1[2] - R(B1p, 2, q - X1), ce2, C[h].b1[1] - v.b1[1]);
          const T u1 = yee_upd(v.e1[1], ce2, C[h].b1[0] - v.b1[0], ce0, C[h].b1[2] - R(B1p, 2, q - 1));
          const T u2 = yee_upd(v.e1[2], ce0, C[h].b1[1] - R(B1p, 1, q - 1), ce1, C[h].b1[0] - R(B1p, 0, q - X1));
          C[h].e2[0] = d0 ? u0 : v.e1[0];
          C[h].e2[1] = d1 ? u1 : v.e1[1];
          C[h].e2[2] = d2 ? u2 : v.e1[2];
          if (own[h] && zw) {
            const int64_t s = sij[h] + kstride * ze;
            if (d0) out.c[0][s] = C[h].e2[0];
            if (d1) out.c[1][s] = C[h].e2[1];
            if (d2) out.c[2][s] = C[h].e2[2];
          }
          R(E2y, 0, q) = C[h].e2[0];
          R(E2y, 1, q) = C[h].e2[1];
          R(E2y, 2, q) = C[h].e2[2];
        }
      }
      // ---- phase 4: B2(z-2) on the own tile points (E2(z-2) neighbours,
      // written in the previous plane, from smem)
      if (p >= 4) {
        const int zb = z - 2;
        if (zb >= k0 && zb < k1) {
#pragma unroll
          for (int h = 0; h < NPT; ++h) {
            if (!own[h]) continue;
            const int q = me[h];
            const Pt& v = V[h];
            const int64_t s = sij[h] + kstride * zb;
            out.c[3][s] = yee_upd(v.b1[0], db2, C[h].e2[1] - v.e2[1], db1, R(E2x, 2, q + X1) - v.e2[2]);
            out.c[4][s] = yee_upd(v.b1[1], db0, R(E2x, 2, q + 1) - v.e2[2], db2, C[h].e2[0] - v.e2[0]);
            out.c[5][s] = yee_upd(v.b1[2], db1, R(E2x, 0, q + X1) - v.e2[0], db0, R(E2x, 1, q + 1) - v.e2[1]);
          }
        }
      }
#undef R
    };
    Pt A[NPT], B[NPT];
    for (int p = 0; p < P; p += 2) {
      plane(std::integral_constant<int, 0>{}, p, A, B);
      if (p + 1 < P) plane(std::integral_constant<int, 1>{}, p + 1, B, A);
    }
    gplane += P;
    __syncthreads();
  }
}

template <class T>
__global__ void k_scatter(YeeGeom g, bool face, const double* __restrict__ src, int64_t n,
                          Fields<T> f) {
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n;
       id += (int64_t)gridDim.x * blockDim.x) {
    int a;
    int64_t s;
    g.dof_to_storage(face, id, a, s);
    f.c[(face ? 3 : 0) + a][s] = (T)src[id];
  }
}

template <class T>
__global__ void k_gather(YeeGeom g, bool face, double* __restrict__ dst, int64_t n,
                         Fields<T> f) {
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n;
       id += (int64_t)gridDim.x * blockDim.x) {
    int a;
    int64_t s;
    g.dof_to_storage(face, id, a, s);
    dst[id] = (double)f.c[(face ? 3 : 0) + a][s];
  }
}

}  // namespace

// One state-modifying kernel of the step sequence; the multi-slab paths
// exchange ghost planes after every phase.
struct Phase {
  // 0 b-kick(h1), 1 e-kick(h1), 2 fused e-kick(h1) + b-kick(h2), 3 two of
  // those: e(h1) b(h2) e(h1) b(h3)
  int kind;
  double h1, h2, h3 = 0;
};

// Unit schedule of the two-step sweep over planes [kbeg, kend) of `ntiles`
// tile columns on `ncta` persistent CTAs. A unit over planes [k0, k1) costs
// k1 - k0 + 4 plane iterations (two halo planes each side), so the
// round-robin 32-plane chunks spend 4/32 of the sweep on z halos. When there
// are fewer tile columns than CTAs, each of the first `ntiles` CTAs instead
// takes the bottom [kbeg, kbeg + Z) of one column in one unit -- all of them
// march through z together, so x/y neighbours share their halo rows in L2 --
// and the remaining CTAs take the tops [kbeg + Z, kend), m columns each, with
// Z chosen so both kinds of CTA run the same number of plane iterations.
// Otherwise (or for short ranges) it is the round-robin chunking.
struct Yee2Sched {
  DevBuf<int4> units;
  DevBuf<int> cta_ptr;
  int grid = 0;
};

inline Yee2Sched make_yee2_sched(int ntiles, int kbeg, int kend, int ncta, int kchunk = 32) {
  std::vector<int4> u;
  std::vector<int> ptr(1, 0);
  const int L = kend - kbeg, R = ncta - ntiles;
  if (R > 0 && L >= 16) {
    const int m = (ntiles + R - 1) / R;
    // Z + 4 = m (L - Z + 4)
    int Z = (int)std::lround((double)(m * (L + 4) - 4) / (double)(m + 1));
    Z = std::max(1, std::min(Z, L));
    for (int t = 0; t < ntiles; ++t) {
      u.push_back(make_int4(t, kbeg, kbeg + Z, 0));
      ptr.push_back((int)u.size());
    }
    if (Z < L)
      for (int r = 0; r < R; ++r) {
        for (int t = r; t < ntiles; t += R) u.push_back(make_int4(t, kbeg + Z, kend, 0));
        if ((int)u.size() > ptr.back()) ptr.push_back((int)u.size());
      }
  } else {
    const int nch = (L + kchunk - 1) / kchunk, n = ntiles * nch;
    const int grid = std::max(1, std::min(n, ncta));
    for (int b = 0; b < grid; ++b) {
      for (int w = b; w < n; w += grid) {
        const int c = w / ntiles, t = w - c * ntiles;
        u.push_back(make_int4(t, kbeg + c * kchunk, std::min(kbeg + (c + 1) * kchunk, kend), 0));
      }
      ptr.push_back((int)u.size());
    }
  }
  Yee2Sched s;
  s.grid = (int)ptr.size() - 1;
  s.units.alloc(std::max<size_t>(1, u.size()));
  s.cta_ptr.alloc(ptr.size());
  SFEEC_CUDA(cudaMemcpy(s.units.p, u.data(), sizeof(int4) * u.size(), cudaMemcpyHostToDevice));
  SFEEC_CUDA(cudaMemcpy(s.cta_ptr.p, ptr.data(), sizeof(int) * ptr.size(), cudaMemcpyHostToDevice));
  return s;
}

struct YeeDev {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  YeeGeom g;
  double d[3] = {1, 1, 1};
  double dt = 0, eps0 = 1, mu0 = 1, dv = 1;
  int prec = 8;
  // fused-sweep variant: SFEEC_YEE_VARIANT overrides the default (A/B runs).
  // Default 4: two leapfrog steps per z-sweep (k_fused2_tma), measured fastest
  // (256^3 fp64 0.219 vs 0.288 ms/step for the one-step sweep, variant 2)
  int variant = [] {
    const char* v = std::getenv("SFEEC_YEE_VARIANT");
    return v ? std::atoi(v) : 4;
  }();
  // TMA descriptors of the two ping-pong buffers (B box, E box), PEC only
  CUtensorMap mapB[2], mapE[2];
  bool have_maps = false;
  int tma_blocks = 0;
  // variant 4 (two steps per sweep): its own boxes
  CUtensorMap mapB2[2], mapE2[2];
  bool have_maps2 = false;
  int tma_blocks2 = 0;
  // programmatic dependent launch of the two-step sweeps (SFEEC_PDL=0: off;
  // read once per handle). Off on NCCL slabs: a programmatic launch after the
  // exchange-event wait has not been verified against a multi-process run.
  bool pdl = env_flag("SFEEC_PDL", true);
  // balanced unit schedule of the two-step sweep (make_yee2_sched)
  std::map<std::pair<int, int>, Yee2Sched> scheds2;
  const Yee2Sched& schedule2(int ntiles, int kbeg, int kend) {
    auto key = std::make_pair(kbeg, kend);
    auto it = scheds2.find(key);
    if (it == scheds2.end()) it = scheds2.emplace(key, make_yee2_sched(ntiles, kbeg, kend, tma_blocks2)).first;
    return it->second;
  }
  DevBuf<char> buf[2];
  int cur = 0;
  DevBuf<double> stage, stage_b, partials;  // host-state staging (e / b), reductions
  double time = 0;
  int64_t launches = 0;
  int64_t n_edges = 0, n_faces = 0;
  // dominant-kernel timing (CUDA events on the launch stream)
  bool timing = false;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double kernel_ms = 0;
  int64_t kernel_launches = 0;
  // z-slab decomposition (yee_layout.hpp make_yee_slab)
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  // CUDA-IPC transport (host-synchronised; the ranks may share a GPU): the
  // neighbours' two ping-pong buffers mapped into this process
  struct IpcSlot {
    cudaIpcMemHandle_t h[2];
    int64_t npts;  // that slab's component stride
    int s2;        // its z planes, ghosts included
  };
  std::unique_ptr<IpcGroup> ipc;
  char* peer_lo[2] = {nullptr, nullptr};
  char* peer_hi[2] = {nullptr, nullptr};
  cudaStream_t comm_stream = nullptr;  // overlapped halo exchange
  cudaEvent_t ev_bnd = nullptr, ev_xch = nullptr;
  // host-state copies: a copy stream, so one vector's scatter / gather runs
  // while the other crosses PCIe
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_cp[3] = {nullptr, nullptr, nullptr};

  void make_copy_stream() {
    if (copy_stream) return;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    for (auto& e : ev_cp) SFEEC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }

  ~YeeDev() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_cp)
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_xch) cudaEventDestroy(ev_xch);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (comm) Nccl::get().comm_destroy(comm);
    for (char* q : {peer_lo[0], peer_lo[1], peer_hi[0], peer_hi[1]})
      if (q) cudaIpcCloseMemHandle(q);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  bool slab() const { return nranks > 1; }
  int64_t plane() const { return (int64_t)g.P0 * g.S[1]; }

  template <class T>
  Fields<T> fields(int which) const {
    Fields<T> f;
    const int64_t np = g.npts();
    for (int c = 0; c < 6; ++c) f.c[c] = reinterpret_cast<T*>(buf[which].p) + c * np;
    return f;
  }
  template <class T>
  YeeCoef<T> coef(double e_factor, double h, double h2 = -1.0) const {
    YeeCoef<T> k;
    const double m2 = dv, q = 1.0 / dv;
    if (h2 < 0) h2 = h;
    for (int a = 0; a < 3; ++a) {
      k.ce[a] = (T)(e_factor * m2 / d[a]);
      k.cb[a] = (T)(h * q / d[a]);
      k.cb2[a] = (T)(h2 * q / d[a]);
    }
    return k;
  }
  unsigned pt_blocks() const {
    return (unsigned)std::min<int64_t>((g.npts() + kThreads - 1) / kThreads, 148 * 64);
  }

  template <class T>
  void bkick(double h) {
    k_bkick<T><<<pt_blocks(), kThreads, 0, stream>>>(g, fields<T>(cur), coef<T>(0, h));
    SFEEC_LAUNCH_CHECK();
    ++launches;
  }
  template <class T>
  void ekick(double h) {
    k_ekick<T><<<pt_blocks(), kThreads, 0, stream>>>(g, fields<T>(cur), coef<T>(h / (eps0 * mu0), 0));
    SFEEC_LAUNCH_CHECK();
    ++launches;
  }
  template <class T>
  void fused(double h_e, double h_b) {
    constexpr int TX = 32, TY = 8;
    const int kchunk = 32;
    dim3 grid((g.S[0] + TX - 1) / TX, (g.S[1] + TY - 1) / TY, (g.S[2] + kchunk - 1) / kchunk);
    k_fused_pec<T, TX, TY><<<grid, TX * TY, 0, stream>>>(
        g, fields<T>(cur), fields<T>(cur ^ 1), coef<T>(h_e / (eps0 * mu0), h_b), kchunk);
    SFEEC_LAUNCH_CHECK();
    cur ^= 1;
    ++launches;
  }

  // kNT1: threads of the one-step sweep -- (TX+1)(TY+1) = 297 E points, so 320
  // threads cover the E region in one pass instead of 256 + 41
  static constexpr int kTX = 32, kTY = 8, kNS = 5, kChunk = 32, kNT1 = 320;
  // two-step sweep, per precision: tile kTX x kTY2, kNT2 threads (one per
  // E1-region point, (kTX+3)(kTY2+3) of them), kNS2 TMA stages, kMB2 CTAs
  // per SM (the register budget). Measured on 256^3 (tools/yee2_ab.sh).
#ifndef YEE2_TY64
#define YEE2_TY64 16
#define YEE2_NT64 672
#define YEE2_MB64 1
#endif
#ifndef YEE2_TY32
#define YEE2_TY32 16
#define YEE2_NT32 672
#define YEE2_MB32 1
#endif
#ifndef YEE2_NPT
#define YEE2_NPT 1
#endif
#ifndef YEE2_NS
#define YEE2_NS 3
#endif
  static constexpr int kNS2 = YEE2_NS, kNPT2 = YEE2_NPT;
  template <class T>
  static constexpr int kTY2 = sizeof(T) == 8 ? YEE2_TY64 : YEE2_TY32;
  template <class T>
  static constexpr int kNT2 = sizeof(T) == 8 ? YEE2_NT64 : YEE2_NT32;
  template <class T>
  static constexpr int kMB2 = sizeof(T) == 8 ? YEE2_MB64 : YEE2_MB32;

  template <class T>
  void make_maps() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      SFEEC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !fn)
        throw Error(SFEEC_ECUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t w = sizeof(T);
    cuuint64_t dims[4] = {(cuuint64_t)g.S[0], (cuuint64_t)g.S[1], (cuuint64_t)g.S[2], 6};
    cuuint64_t strides[3] = {(cuuint64_t)g.P0 * w, (cuuint64_t)g.P0 * g.S[1] * w,
                             (cuuint64_t)g.npts() * w};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    using Cfg = TmaCfg<T, kTX, kTY, kNS>;
    cuuint32_t boxB[4] = {(cuuint32_t)Cfg::kBWB, kTY + 2, 1, 3};
    cuuint32_t boxE[4] = {(cuuint32_t)Cfg::kBWE, kTY + 1, 1, 3};
    const CUtensorMapDataType dt_ = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                   : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    for (int b = 0; b < 2; ++b) {
      void* ptr = buf[b].p;
      for (int which = 0; which < 2; ++which) {
        CUresult r = encode(which ? &mapE[b] : &mapB[b], dt_, 4, ptr, dims, strides,
                            which ? boxE : boxB, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(SFEEC_ECUDA, "cuTensorMapEncodeTiled failed");
      }
    }
    auto kern = k_fused_tma<T, kTX, kTY, kNS, kNT1>;
    SFEEC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
    int per_sm = 0, sms = 0;
    SFEEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT1, Cfg::kSmem));
    SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    tma_blocks = std::max(1, per_sm) * sms;
    have_maps = true;
  }

  template <class T>
  void make_maps2() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      SFEEC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !fn)
        throw Error(SFEEC_ECUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t w = sizeof(T);
    cuuint64_t dims[4] = {(cuuint64_t)g.S[0], (cuuint64_t)g.S[1], (cuuint64_t)g.S[2], 6};
    cuuint64_t strides[3] = {(cuuint64_t)g.P0 * w, (cuuint64_t)g.P0 * g.S[1] * w,
                             (cuuint64_t)g.npts() * w};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    using Cfg = TmaCfg2<T, kTX, kTY2<T>, kNS2>;
    cuuint32_t boxB[4] = {(cuuint32_t)Cfg::kBW, kTY2<T> + 4, 1, 3};
    cuuint32_t boxE[4] = {(cuuint32_t)Cfg::kBW, kTY2<T> + 3, 1, 3};
    const CUtensorMapDataType dt_ = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                   : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    for (int b = 0; b < 2; ++b) {
      void* ptr = buf[b].p;
      for (int which = 0; which < 2; ++which) {
        CUresult r = encode(which ? &mapE2[b] : &mapB2[b], dt_, 4, ptr, dims, strides,
                            which ? boxE : boxB, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(SFEEC_ECUDA, "cuTensorMapEncodeTiled failed");
      }
    }
    using Cfg2 = TmaCfg2<T, kTX, kTY2<T>, kNS2, 2>;
    auto kern = k_fused2_tma<T, kTX, kTY2<T>, kNS2, kNT2<T>, kNPT2, kMB2<T>>;
    const int smem = Cfg2::kSmem;
    SFEEC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0, sms = 0;
    SFEEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT2<T>, smem));
    SFEEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    tma_blocks2 = std::max(1, per_sm) * sms;
    have_maps2 = true;
  }

  // two fused steps over local planes [kbeg, kend): buf[cur] -> buf[cur^1]
  template <class T>
  void launch_range2(double h_e, double h_b, int kbeg, int kend, double h_b2) {
    if (!have_maps2) make_maps2<T>();
    const int ntx = (g.n[0] + kTX - 1) / kTX, nty = (g.n[1] + kTY2<T> - 1) / kTY2<T>;
    const int nchunks = (kend - kbeg + kChunk - 1) / kChunk;
    const int n_units = ntx * nty * nchunks;
    const Yee2Sched* sc = &schedule2(ntx * nty, kbeg, kend);
    const int grid = sc->grid;
    launch_pdl(pdl && !comm, k_fused2_tma<T, kTX, kTY2<T>, kNS2, kNT2<T>, kNPT2, kMB2<T>>, dim3(grid),
               dim3(kNT2<T>), TmaCfg2<T, kTX, kTY2<T>, kNS2, 2>::kSmem, stream, mapB2[cur],
               mapE2[cur], g, fields<T>(cur ^ 1), coef<T>(h_e / (eps0 * mu0), h_b, h_b2), kChunk, ntx,
               ntx * nty, n_units, kbeg, kend, sc->units.p, sc->cta_ptr.p);
    SFEEC_LAUNCH_CHECK();
    ++launches;
  }

  template <class T>
  void fused2_tma(double h_e, double h_b, double h_b2) {
    launch_range2<T>(h_e, h_b, sweep_beg(), sweep_end(), h_b2);
    cur ^= 1;
  }

  // planes swept by the fused kernel: [0, n) on one domain, [1, nzl + 1) on a slab
  int ghost() const { return slab() ? g.kown_lo : 0; }  // ghost planes per side
  int sweep_beg() const { return slab() ? ghost() : 0; }
  int sweep_end() const { return slab() ? g.S[2] - ghost() : g.n[2]; }
  int sweep_chunks() const { return (sweep_end() - sweep_beg() + kChunk - 1) / kChunk; }

  template <class T>
  void fused_tma(double h_e, double h_b) {
    launch_range<T>(h_e, h_b, sweep_beg(), sweep_end());
    cur ^= 1;
  }

  // Split sweep for overlapping the halo exchange: part 0 = the z-chunks that
  // produce the planes the neighbours need (the bottom and top `ghost()`
  // owned planes), part 1 = the rest. two: the two-step sweep. Neither flips
  // the buffers.
  template <class T>
  void fused_part(double h_e, double h_b, int part, bool two = false, double h_b2 = -1.0) {
    const int kb = sweep_beg(), ke = sweep_end(), G = ghost();
    auto range = [&](int a, int b) {
      if (b <= a) return;
      if (two)
        launch_range2<T>(h_e, h_b, a, b, h_b2 < 0 ? h_b : h_b2);
      else
        launch_range<T>(h_e, h_b, a, b);
    };
    const int lo_end = std::min(kb + kChunk, ke);
    // first chunk of the top part: the chunk holding plane ke - G (chunks are
    // aligned to kb), but never below the bottom chunk's end
    const int hi_beg = std::max(lo_end, kb + ((ke - G - kb) / kChunk) * kChunk);
    if (part == 0) {
      range(kb, lo_end);
      range(hi_beg, ke);
    } else {
      range(lo_end, hi_beg);
    }
  }

  // fused sweep over local planes [kbeg, kend): reads buf[cur], writes buf[cur^1]
  template <class T>
  void launch_range(double h_e, double h_b, int kbeg, int kend) {
    if (!have_maps) make_maps<T>();
    using Cfg = TmaCfg<T, kTX, kTY, kNS>;
    const int ntx = (g.n[0] + kTX - 1) / kTX, nty = (g.n[1] + kTY - 1) / kTY;
    const int nchunks = (kend - kbeg + kChunk - 1) / kChunk;
    const int n_units = ntx * nty * nchunks;
    const int grid = std::min(n_units, tma_blocks);
    k_fused_tma<T, kTX, kTY, kNS, kNT1><<<grid, kNT1, Cfg::kSmem, stream>>>(
        mapB[cur], mapE[cur], g, fields<T>(cur ^ 1), coef<T>(h_e / (eps0 * mu0), h_b), kChunk,
        ntx, ntx * nty, n_units, kbeg, kend);
    SFEEC_LAUNCH_CHECK();
    ++launches;
  }

  // one fused step on a slab with the NCCL exchange overlapped: boundary
  // chunks -> (comm stream) exchange of the new buffer's edge planes, while the
  // interior chunks run; the compute stream waits for the exchange before the
  // next kernel reads the ghosts. The exchange touches only ghost planes and
  // the boundary chunks' planes, the interior sweep only interior planes.
  template <class T>
  void fused_overlapped(double h_e, double h_b, bool two = false, double h_b2 = -1.0) {
    if (!comm_stream) {
      SFEEC_CUDA(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
      SFEEC_CUDA(cudaEventCreateWithFlags(&ev_bnd, cudaEventDisableTiming));
      SFEEC_CUDA(cudaEventCreateWithFlags(&ev_xch, cudaEventDisableTiming));
    }
    fused_part<T>(h_e, h_b, 0, two, h_b2);
    SFEEC_CUDA(cudaEventRecord(ev_bnd, stream));
    SFEEC_CUDA(cudaStreamWaitEvent(comm_stream, ev_bnd, 0));
    exchange_nccl(cur ^ 1, comm_stream);
    SFEEC_CUDA(cudaEventRecord(ev_xch, comm_stream));
    fused_part<T>(h_e, h_b, 1, two, h_b2);
    SFEEC_CUDA(cudaStreamWaitEvent(stream, ev_xch, 0));
    cur ^= 1;
  }

  // Strang with merged half-kicks: b(dt/2), n-1 x [e(dt) b(dt)], e(dt), b(dt/2)
  std::vector<Phase> plan(int64_t n) const {
    std::vector<Phase> p;
    if (n <= 0) return p;
    const bool use_fused = variant >= 1 && g.bc == SFEEC_BC_PEC;
    const bool two = variant == 4 && g.bc == SFEEC_BC_PEC && (!slab() || ghost() >= 2);
    // merged Strang b(h/2) [e(h) b(h)]^(n-1) e(h) b(h/2) = b(h/2), then n
    // (e, b) pairs whose last b-kick is the closing half-kick: folded into the
    // last sweep (bitwise the separate kick: every update is yee_upd)
    p.push_back({0, 0.5 * dt, 0});
    for (int64_t s = 0; s < n; ++s) {
      if (two && s + 1 < n) {  // two fused steps per sweep
        p.push_back({3, dt, dt, s + 2 == n ? 0.5 * dt : dt});
        ++s;
      } else if (use_fused) {
        p.push_back({2, dt, s + 1 == n ? 0.5 * dt : dt});
      } else {
        p.push_back({1, dt, 0});
        p.push_back({0, s + 1 == n ? 0.5 * dt : dt, 0});
      }
    }
    return p;
  }

  template <class T>
  void run_t(const Phase& p) {
    if (p.kind == 0)
      bkick<T>(p.h1);
    else if (p.kind == 1)
      ekick<T>(p.h1);
    else if (p.kind == 3)
      fused2_tma<T>(p.h1, p.h2, p.h3);
    else if (variant >= 2 || slab())
      fused_tma<T>(p.h1, p.h2);
    else
      fused<T>(p.h1, p.h2);
  }
  void run(const Phase& p) {
    if (prec == 8)
      run_t<double>(p);
    else
      run_t<float>(p);
  }

  // ghost-plane exchange over NCCL (one process per GPU): the first G owned
  // planes (E and B) go down into the lower neighbour's top ghosts; the top G
  // owned planes go up into the upper neighbour's bottom ghosts (B only when
  // G = 1: the one-step kernels never read E below). Each component's G
  // planes are contiguous, so one message per component and direction.
  // join the ranks' shared segment and map the neighbours' buffers
  void init_ipc(const void* id128) {
    ipc = std::make_unique<IpcGroup>("sfeec_yee", id128, rank, nranks, sizeof(IpcSlot));
    IpcSlot& me = *(IpcSlot*)ipc->slot(rank);
    for (int b = 0; b < 2; ++b) SFEEC_CUDA(cudaIpcGetMemHandle(&me.h[b], buf[b].p));
    me.npts = g.npts();
    me.s2 = g.S[2];
    ipc->barrier();
    for (int b = 0; b < 2; ++b) {
      void* q = nullptr;
      if (rank > 0) {
        SFEEC_CUDA(cudaIpcOpenMemHandle(&q, ((IpcSlot*)ipc->slot(rank - 1))->h[b],
                                        cudaIpcMemLazyEnablePeerAccess));
        peer_lo[b] = (char*)q;
      }
      if (rank < nranks - 1) {
        SFEEC_CUDA(cudaIpcOpenMemHandle(&q, ((IpcSlot*)ipc->slot(rank + 1))->h[b],
                                        cudaIpcMemLazyEnablePeerAccess));
        peer_hi[b] = (char*)q;
      }
    }
    ipc->barrier();
    ipc->unlink_name();
  }
  // the same planes and components as exchange_nccl, pulled from the
  // neighbours' buffers between two host barriers
  void exchange_ipc(int bufsel, cudaStream_t es) {
    const int G = ghost();
    const size_t pb = (size_t)plane() * (size_t)prec, cnt = pb * (size_t)G;
    char* base = buf[bufsel].p;
    auto at = [&](char* b0, int64_t npts, int comp, int pl) {
      return b0 + ((size_t)comp * (size_t)npts) * (size_t)prec + (size_t)pl * pb;
    };
    const int c_up = G == 1 ? 3 : 0;
    SFEEC_CUDA(cudaStreamSynchronize(es));  // our planes are written ...
    ipc->barrier();                         // ... and so are the neighbours'
    if (rank > 0) {  // bottom ghosts <- the lower neighbour's top owned planes
      const IpcSlot& lo = *(const IpcSlot*)ipc->slot(rank - 1);
      for (int c = c_up; c < 6; ++c)
        SFEEC_CUDA(cudaMemcpyAsync(at(base, g.npts(), c, 0),
                                   at(peer_lo[bufsel], lo.npts, c, lo.s2 - 2 * G), cnt,
                                   cudaMemcpyDeviceToDevice, es));
    }
    if (rank < nranks - 1) {  // top ghosts <- the upper neighbour's first owned planes
      const IpcSlot& hi = *(const IpcSlot*)ipc->slot(rank + 1);
      for (int c = 0; c < 6; ++c)
        SFEEC_CUDA(cudaMemcpyAsync(at(base, g.npts(), c, g.S[2] - G),
                                   at(peer_hi[bufsel], hi.npts, c, G), cnt,
                                   cudaMemcpyDeviceToDevice, es));
    }
    SFEEC_CUDA(cudaStreamSynchronize(es));  // our pulls are done ...
    ipc->barrier();                         // ... before anyone overwrites a source plane
  }
  void exchange_nccl() { exchange_nccl(cur, stream); }
  void exchange_nccl(int bufsel, cudaStream_t es) {
    if (slab() && ipc) return exchange_ipc(bufsel, es);
    if (!slab() || !comm) return;
    const Nccl& nc = Nccl::get();
    const ncclDataType_t ty = prec == 8 ? ncclFloat64 : ncclFloat32;
    const int G = ghost();
    const size_t cnt = (size_t)plane() * (size_t)G;
    char* base = buf[bufsel].p;
    cudaStream_t stream = es;
    auto at = [&](int comp, int pl) {
      return base + ((size_t)comp * (size_t)g.npts() + (size_t)pl * (size_t)plane()) * (size_t)prec;
    };
    const int c_up = G == 1 ? 3 : 0;
    nc.check(nc.group_start(), "ncclGroupStart");
    if (rank > 0) {
      for (int c = 0; c < 6; ++c) nc.check(nc.send(at(c, G), cnt, ty, rank - 1, comm, stream), "ncclSend");
      for (int c = c_up; c < 6; ++c) nc.check(nc.recv(at(c, 0), cnt, ty, rank - 1, comm, stream), "ncclRecv");
    }
    if (rank < nranks - 1) {
      for (int c = 0; c < 6; ++c)
        nc.check(nc.recv(at(c, g.S[2] - G), cnt, ty, rank + 1, comm, stream), "ncclRecv");
      for (int c = c_up; c < 6; ++c)
        nc.check(nc.send(at(c, g.S[2] - 2 * G), cnt, ty, rank + 1, comm, stream), "ncclSend");
    }
    nc.check(nc.group_end(), "ncclGroupEnd");
  }

  void advance(int64_t n) {
    launches = 0;
    if (n <= 0) return;
    auto p = plan(n);
    const bool t = timing && n > 1;
    const bool overlap = slab() && comm && variant >= 2;
    for (size_t i = 0; i < p.size(); ++i) {
      if (t && i == 1) SFEEC_CUDA(cudaEventRecord(ev[0], stream));  // the sweeps: phases 1..
      if (overlap && (p[i].kind == 2 || p[i].kind == 3)) {
        if (prec == 8)
          fused_overlapped<double>(p[i].h1, p[i].h2, p[i].kind == 3, p[i].h3);
        else
          fused_overlapped<float>(p[i].h1, p[i].h2, p[i].kind == 3, p[i].h3);
        continue;
      }
      run(p[i]);
      exchange_nccl();
    }
    if (t) {
      SFEEC_CUDA(cudaEventRecord(ev[1], stream));
      SFEEC_CUDA(cudaEventSynchronize(ev[1]));
      float ms = 0;
      SFEEC_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      kernel_ms += ms;
      kernel_launches += (int64_t)p.size() - 1;
    }
    for (int64_t s = 0; s < n; ++s) time = time + dt;
  }

  void flow_he(double h) {
    launches = 0;
    run({0, h, 0});
    exchange_nccl();
  }
  void flow_ha(double h) {
    launches = 0;
    run({1, h, 0});
    exchange_nccl();
  }

  // 0.5 (eps0 e^T Q e + b^T M2 b / mu0), dynamics.cpp:92-102 with lumped Q, M2;
  // a slab sums its owned planes only (the caller adds the ranks' parts)
  double energy() {
    const int64_t off = (int64_t)g.kown_lo * plane();
    const int64_t cnt = std::min<int64_t>((int64_t)(g.kown_hi - g.kown_lo) * plane(), g.npts() - off);
    double se = 0, sb = 0;
    for (int c = 0; c < 3; ++c) {
      if (prec == 8) {
        Fields<double> f = fields<double>(cur);
        se += device_dot(f.c[c] + off, f.c[c] + off, cnt, partials.p, stream);
        sb += device_dot(f.c[3 + c] + off, f.c[3 + c] + off, cnt, partials.p, stream);
      } else {
        Fields<float> f = fields<float>(cur);
        se += device_sumsq(f.c[c] + off, cnt, partials.p, stream);
        sb += device_sumsq(f.c[3 + c] + off, cnt, partials.p, stream);
      }
    }
    return 0.5 * (eps0 * (se / dv) + (sb * dv) / mu0);
  }

  // device scatter of the (b, e) DOF vectors (already in `stage` buffers)
  // (ready_b / ready_e: optional events the b / e staging copies record)
  void set_state_dev(const double* b_dev, const double* e_dev, cudaEvent_t ready_b = nullptr,
                     cudaEvent_t ready_e = nullptr) {
    buf[0].zero(stream);
    buf[1].zero(stream);
    cur = 0;
    for (int face = 1; face >= 0; --face) {
      const int64_t n = face ? n_faces : n_edges;
      const cudaEvent_t ready = face ? ready_b : ready_e;
      if (ready) SFEEC_CUDA(cudaStreamWaitEvent(stream, ready, 0));
      if (!n) continue;
      unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
      // both ping-pong buffers: the fused sweep never rewrites the constant
      // PEC boundary faces (empty C rows), so they must be present in both
      for (int bsel = 0; bsel < 2; ++bsel) {
        if (prec == 8)
          k_scatter<double><<<blocks, 256, 0, stream>>>(g, face, face ? b_dev : e_dev, n,
                                                        fields<double>(bsel));
        else
          k_scatter<float><<<blocks, 256, 0, stream>>>(g, face, face ? b_dev : e_dev, n,
                                                       fields<float>(bsel));
        SFEEC_LAUNCH_CHECK();
      }
    }
  }

  void set_state(const double* b, const double* e) {
    // persistent staging: no allocation on the host-state path
    if (stage_b.n < (size_t)std::max<int64_t>(1, n_faces))
      stage_b.alloc((size_t)std::max<int64_t>(1, n_faces));
    make_copy_stream();
    // b then e over PCIe on the copy stream; the buffer clears and b's scatter
    // run on the compute stream while e is still crossing
    SFEEC_CUDA(cudaEventRecord(ev_cp[2], stream));  // earlier work on the stage buffers
    SFEEC_CUDA(cudaStreamWaitEvent(copy_stream, ev_cp[2], 0));
    SFEEC_CUDA(cudaMemcpyAsync(stage_b.p, b, sizeof(double) * (size_t)n_faces,
                               cudaMemcpyHostToDevice, copy_stream));
    SFEEC_CUDA(cudaEventRecord(ev_cp[0], copy_stream));
    SFEEC_CUDA(cudaMemcpyAsync(stage.p, e, sizeof(double) * (size_t)n_edges,
                               cudaMemcpyHostToDevice, copy_stream));
    SFEEC_CUDA(cudaEventRecord(ev_cp[1], copy_stream));
    set_state_dev(stage_b.p, stage.p, ev_cp[0], ev_cp[1]);
    // ghosts of both buffers: exchange once per buffer
    exchange_nccl();
    cur ^= 1;
    exchange_nccl();
    cur ^= 1;
    SFEEC_CUDA(cudaStreamSynchronize(stream));
  }

  void get_state(double* b, double* e) {
    // e gathered into `stage`, b into `stage_b`: b's gather runs while e
    // crosses PCIe on the copy stream
    if (stage_b.n < (size_t)std::max<int64_t>(1, n_faces))
      stage_b.alloc((size_t)std::max<int64_t>(1, n_faces));
    make_copy_stream();
    for (int face = 0; face < 2; ++face) {
      double* dst = face ? b : e;
      const int64_t n = face ? n_faces : n_edges;
      if (!dst || !n) continue;
      double* st = face ? stage_b.p : stage.p;
      unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
      if (prec == 8)
        k_gather<double><<<blocks, 256, 0, stream>>>(g, face, st, n, fields<double>(cur));
      else
        k_gather<float><<<blocks, 256, 0, stream>>>(g, face, st, n, fields<float>(cur));
      SFEEC_LAUNCH_CHECK();
      SFEEC_CUDA(cudaEventRecord(ev_cp[face], stream));
      SFEEC_CUDA(cudaStreamWaitEvent(copy_stream, ev_cp[face], 0));
      SFEEC_CUDA(cudaMemcpyAsync(dst, st, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost,
                                 copy_stream));
    }
    SFEEC_CUDA(cudaStreamSynchronize(copy_stream));
    SFEEC_CUDA(cudaStreamSynchronize(stream));
  }

  void init(int dev, const YeeGeom& geom, double dx, double dy, double dz, double dt_,
            double eps0_, double mu0_, int precision) {
    device = dev;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    own_stream = true;
    g = geom;
    d[0] = dx;
    d[1] = dy;
    d[2] = dz;
    dv = dx * dy * dz;
    dt = dt_;
    eps0 = eps0_;
    mu0 = mu0_;
    prec = precision;
    n_edges = g.edge_off[3];
    n_faces = g.face_off[3];
    const size_t bytes = (size_t)g.npts() * 6 * (size_t)precision;
    buf[0].alloc(bytes);
    buf[1].alloc(bytes);
    buf[0].zero(stream);
    buf[1].zero(stream);
    stage.alloc((size_t)std::max<int64_t>(1, std::max(n_edges, n_faces)));
    partials.alloc(kReduceBlocks + 1);
    SFEEC_CUDA(cudaStreamSynchronize(stream));
  }
};

// R slabs of one lattice on ONE device with in-process ghost copies: the same
// kernels, ghost layout and step plan as the NCCL path, with the transport
// replaced by cudaMemcpyAsync -- how the multi-rank path is verified with a
// single GPU (ranks are advanced in lockstep, phase by phase; no kernel ever
// waits on another).
struct YeeGroup {
  std::vector<std::unique_ptr<YeeDev>> s;
  YeeGeom global;

  // flip = 1: exchange into the buffers being written (the split sweep);
  // the same planes and components as YeeDev::exchange_nccl
  void exchange(int flip = 0) {
    const int R = (int)s.size();
    for (int r = 0; r < R; ++r) {
      YeeDev& a = *s[(size_t)r];
      const int G = a.ghost();
      const size_t bytes = (size_t)a.plane() * (size_t)a.prec * (size_t)G;
      auto at = [&](YeeDev& d, int comp, int pl) {
        return d.buf[d.cur ^ flip].p +
               ((size_t)comp * (size_t)d.g.npts() + (size_t)pl * (size_t)d.plane()) * (size_t)d.prec;
      };
      if (r > 0) {
        YeeDev& lo = *s[(size_t)r - 1];
        for (int c = 0; c < 6; ++c)
          SFEEC_CUDA(cudaMemcpyAsync(at(lo, c, lo.g.S[2] - G), at(a, c, G), bytes,
                                     cudaMemcpyDeviceToDevice, a.stream));
      }
      if (r < R - 1) {
        YeeDev& hi = *s[(size_t)r + 1];
        for (int c = G == 1 ? 3 : 0; c < 6; ++c)
          SFEEC_CUDA(cudaMemcpyAsync(at(hi, c, 0), at(a, c, a.g.S[2] - 2 * G), bytes,
                                     cudaMemcpyDeviceToDevice, a.stream));
      }
    }
  }
  void run_all(const Phase& p) {
    if ((p.kind == 2 || p.kind == 3) && s[0]->variant >= 2) {
      // the NCCL path's overlapped schedule, serialised: boundary chunks,
      // exchange into the new buffers, interior chunks, flip
      const bool two = p.kind == 3;
      for (auto& d : s) {
        if (d->prec == 8)
          d->fused_part<double>(p.h1, p.h2, 0, two, p.h3);
        else
          d->fused_part<float>(p.h1, p.h2, 0, two, p.h3);
      }
      exchange(1);
      for (auto& d : s) {
        if (d->prec == 8)
          d->fused_part<double>(p.h1, p.h2, 1, two, p.h3);
        else
          d->fused_part<float>(p.h1, p.h2, 1, two, p.h3);
        d->cur ^= 1;
      }
      return;
    }
    for (auto& d : s) d->run(p);
    exchange();
  }
  void advance(int64_t n) {
    auto p = s[0]->plan(n);
    for (auto& ph : p) run_all(ph);
    for (auto& d : s)
      for (int64_t k = 0; k < n; ++k) d->time = d->time + d->dt;
  }
};

}  // namespace sfeec_b200

using namespace sfeec_b200;

struct sfeec_yee {
  YeeDev d;
};

struct sfeec_yee_group {
  YeeGroup g;
};

namespace {
void check_lattice(int nx, int ny, int nz, double dx, double dy, double dz, double dt, int bc,
                   int precision) {
  require(nx >= 1 && ny >= 1 && nz >= 1, "cubical lattice: cell counts must be >= 1");
  require(dx > 0 && dy > 0 && dz > 0, "cubical lattice: spacings must be > 0");
  require(dt >= 0, "SplitScheme: dt must be >= 0");
  require(bc == SFEEC_BC_PERIODIC || bc == SFEEC_BC_PEC, "unknown boundary condition");
  require(precision == 8 || precision == 4, "precision must be 8 (fp64) or 4 (fp32)");
  require(bc == SFEEC_BC_PEC || (nx >= 2 && ny >= 2 && nz >= 2),
          "periodic Yee kernels need >= 2 cells per axis");
}
// local -> global DOF ids of slab r (host, for set/get of distributed state)
void slab_maps(int nx, int ny, int nz, int r, int R, int64_t* emap, int64_t* fmap) {
  YeeGeom gl = make_yee_geom(nx, ny, nz, 1), sl = make_yee_slab(nx, ny, nz, r, R);
  for (int face = 0; face < 2; ++face) {
    int64_t* m = face ? fmap : emap;
    if (!m) continue;
    const int64_t n = face ? sl.face_off[3] : sl.edge_off[3];
#pragma omp parallel for schedule(static)
    for (int64_t id = 0; id < n; ++id) {
      int a;
      int64_t st;
      sl.dof_to_storage(face == 1, id, a, st);
      int i = (int)(st % sl.P0), j = (int)((st / sl.P0) % sl.S[1]);
      int k = (int)(st / ((int64_t)sl.P0 * sl.S[1])) + sl.kofs;
      m[id] = gl.dof_id(face == 1, a, i, j, k);
    }
  }
}
}  // namespace

extern "C" {

int sfeec_yee_create(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                     double eps0, double mu0, int bc, int precision, int device,
                     sfeec_yee** out) {
  return guarded([&] {
    require(out != nullptr, "sfeec_yee_create: null out");
    *out = nullptr;
    check_lattice(nx, ny, nz, dx, dy, dz, dt, bc, precision);
    select_device(device);
    auto h = std::make_unique<sfeec_yee>();
    h->d.init(device, make_yee_geom(nx, ny, nz, bc), dx, dy, dz, dt, eps0, mu0, precision);
    *out = h.release();
  });
}

int sfeec_nccl_unique_id(void* out128) {
  return guarded([&] {
    require(out128 != nullptr, "null out");
    ncclUniqueId id;
    Nccl::get().check(Nccl::get().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

// Exercises the run-time NCCL binding (nccl_loader.hpp) on one device: a
// 1-rank communicator, a grouped send/recv to self of n doubles on a stream,
// the comparison, destroy. The multi-rank calls are the same entry points.
int sfeec_nccl_selftest(int device, int64_t n, double* max_err) {
  return guarded([&] {
    require(n >= 1 && max_err, "bad argument");
    select_device(device);
    const Nccl& nc = Nccl::get();
    ncclUniqueId id;
    nc.check(nc.get_unique_id(&id), "ncclGetUniqueId");
    ncclComm_t comm = nullptr;
    nc.check(nc.comm_init_rank(&comm, 1, id, 0), "ncclCommInitRank");
    cudaStream_t st;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<double> h((size_t)n), back((size_t)n);
    for (int64_t i = 0; i < n; ++i) h[(size_t)i] = 0.5 * (double)i - 3.0;
    DevBuf<double> x, y;
    x.upload(h.data(), h.size(), st);
    y.alloc((size_t)n);
    y.zero(st);
    nc.check(nc.group_start(), "ncclGroupStart");
    nc.check(nc.send(x.p, (size_t)n, ncclFloat64, 0, comm, st), "ncclSend");
    nc.check(nc.recv(y.p, (size_t)n, ncclFloat64, 0, comm, st), "ncclRecv");
    nc.check(nc.group_end(), "ncclGroupEnd");
    SFEEC_CUDA(cudaMemcpyAsync(back.data(), y.p, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, st));
    SFEEC_CUDA(cudaStreamSynchronize(st));
    double err = 0;
    for (int64_t i = 0; i < n; ++i) err = std::max(err, std::fabs(back[(size_t)i] - h[(size_t)i]));
    *max_err = err;
    cudaStreamDestroy(st);
    nc.check(nc.comm_destroy(comm), "ncclCommDestroy");
  });
}

int sfeec_yee_create_slab(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                          double eps0, double mu0, int precision, int rank, int nranks,
                          const void* nccl_id, int device, sfeec_yee** out) {
  return sfeec_yee_create_slab_transport(nx, ny, nz, dx, dy, dz, dt, eps0, mu0, precision, rank,
                                         nranks, SFEEC_TRANSPORT_NCCL, nccl_id, device, out);
}

int sfeec_yee_create_slab_transport(int nx, int ny, int nz, double dx, double dy, double dz,
                                    double dt, double eps0, double mu0, int precision, int rank,
                                    int nranks, int transport, const void* comm_id, int device,
                                    sfeec_yee** out) {
  const void* nccl_id = comm_id;
  return guarded([&] {
    require(out != nullptr, "sfeec_yee_create_slab: null out");
    require(transport == SFEEC_TRANSPORT_NCCL || transport == SFEEC_TRANSPORT_IPC,
            "sfeec_yee_create_slab: unknown transport");
    *out = nullptr;
    check_lattice(nx, ny, nz, dx, dy, dz, dt, SFEEC_BC_PEC, precision);
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    require(nz % nranks == 0 && nz / nranks >= 2, "nz must be a multiple of nranks (>= 2 planes each)");
    select_device(device);
    auto h = std::make_unique<sfeec_yee>();
    YeeDev& d = h->d;
    if (nranks == 1) {
      d.init(device, make_yee_geom(nx, ny, nz, SFEEC_BC_PEC), dx, dy, dz, dt, eps0, mu0, precision);
    } else {
      require(nccl_id != nullptr, "multi-rank slab needs a communicator id");
      d.init(device, make_yee_slab(nx, ny, nz, rank, nranks), dx, dy, dz, dt, eps0, mu0, precision);
      d.rank = rank;
      d.nranks = nranks;
      if (transport == SFEEC_TRANSPORT_IPC) {
        d.init_ipc(comm_id);
      } else {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        Nccl::get().check(Nccl::get().comm_init_rank(&d.comm, nranks, id, rank),
                          "ncclCommInitRank");
      }
    }
    *out = h.release();
  });
}

int sfeec_yee_slab_dof_map(int nx, int ny, int nz, int rank, int nranks, int64_t* edge_map,
                           int64_t* face_map) {
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    require(nz % nranks == 0 && nz / nranks >= 2, "nz must be a multiple of nranks (>= 2 planes each)");
    slab_maps(nx, ny, nz, rank, nranks, edge_map, face_map);
  });
}

int sfeec_yee_slab_dof_counts(int nx, int ny, int nz, int rank, int nranks, int64_t* n_edges,
                              int64_t* n_faces) {
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    require(nz % nranks == 0 && nz / nranks >= 2, "nz must be a multiple of nranks (>= 2 planes each)");
    YeeGeom g = nranks == 1 ? make_yee_geom(nx, ny, nz, 1) : make_yee_slab(nx, ny, nz, rank, nranks);
    if (n_edges) *n_edges = g.edge_off[3];
    if (n_faces) *n_faces = g.face_off[3];
  });
}

int sfeec_yee_group_create(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                           double eps0, double mu0, int precision, int nranks, int device,
                           sfeec_yee_group** out) {
  return guarded([&] {
    require(out != nullptr, "null out");
    *out = nullptr;
    check_lattice(nx, ny, nz, dx, dy, dz, dt, SFEEC_BC_PEC, precision);
    require(nranks >= 2, "a group needs >= 2 slabs");
    require(nz % nranks == 0 && nz / nranks >= 2, "nz must be a multiple of nranks (>= 2 planes each)");
    select_device(device);
    auto h = std::make_unique<sfeec_yee_group>();
    h->g.global = make_yee_geom(nx, ny, nz, SFEEC_BC_PEC);
    for (int r = 0; r < nranks; ++r) {
      auto d = std::make_unique<YeeDev>();
      d->init(device, make_yee_slab(nx, ny, nz, r, nranks), dx, dy, dz, dt, eps0, mu0, precision);
      d->rank = r;
      d->nranks = nranks;
      h->g.s.push_back(std::move(d));
    }
    // one stream for the whole group keeps the lockstep order
    for (size_t r = 1; r < h->g.s.size(); ++r) {
      cudaStreamDestroy(h->g.s[r]->stream);
      h->g.s[r]->stream = h->g.s[0]->stream;
      h->g.s[r]->own_stream = false;
    }
    *out = h.release();
  });
}

void sfeec_yee_group_destroy(sfeec_yee_group* h) { delete h; }

int sfeec_yee_group_set_variant(sfeec_yee_group* h, int variant) {
  return guarded([&] {
    require(h && (variant == 0 || variant == 2 || variant == 4), "slabs support variants 0, 2 and 4");
    for (auto& d : h->g.s) d->variant = variant;
  });
}

// global (b, e) in the single-domain PEC numbering
int sfeec_yee_group_set_state(sfeec_yee_group* h, const double* b, const double* e) {
  return guarded([&] {
    require(h && b && e, "null argument");
    auto& G = h->g;
    const int R = (int)G.s.size();
    for (int r = 0; r < R; ++r) {
      YeeDev& d = *G.s[(size_t)r];
      SFEEC_CUDA(cudaSetDevice(d.device));
      std::vector<int64_t> em((size_t)d.n_edges), fm((size_t)d.n_faces);
      slab_maps(G.global.n[0], G.global.n[1], G.global.n[2], r, R, em.data(), fm.data());
      std::vector<double> lb((size_t)d.n_faces), le((size_t)d.n_edges);
      for (size_t i = 0; i < lb.size(); ++i) lb[i] = b[fm[i]];
      for (size_t i = 0; i < le.size(); ++i) le[i] = e[em[i]];
      DevBuf<double> db;
      db.upload(lb.data(), lb.size(), d.stream);
      SFEEC_CUDA(cudaMemcpyAsync(d.stage.p, le.data(), sizeof(double) * le.size(),
                                 cudaMemcpyHostToDevice, d.stream));
      d.set_state_dev(db.p, d.stage.p);
      SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    }
    for (int k = 0; k < 2; ++k) {  // ghosts of both ping-pong buffers
      G.exchange();
      for (auto& d : G.s) d->cur ^= 1;
    }
    SFEEC_CUDA(cudaStreamSynchronize(G.s[0]->stream));
  });
}

int sfeec_yee_group_get_state(sfeec_yee_group* h, double* b, double* e) {
  return guarded([&] {
    require(h && b && e, "null argument");
    auto& G = h->g;
    const int R = (int)G.s.size();
    for (int r = 0; r < R; ++r) {
      YeeDev& d = *G.s[(size_t)r];
      std::vector<int64_t> em((size_t)d.n_edges), fm((size_t)d.n_faces);
      slab_maps(G.global.n[0], G.global.n[1], G.global.n[2], r, R, em.data(), fm.data());
      std::vector<double> lb((size_t)d.n_faces), le((size_t)d.n_edges);
      d.get_state(lb.data(), le.data());
      for (size_t i = 0; i < lb.size(); ++i) b[fm[i]] = lb[i];
      for (size_t i = 0; i < le.size(); ++i) e[em[i]] = le[i];
    }
  });
}

int sfeec_yee_group_advance(sfeec_yee_group* h, int64_t nsteps) {
  return guarded([&] {
    require(h, "null handle");
    require(nsteps >= 0, "advance: nsteps must be >= 0");
    SFEEC_CUDA(cudaSetDevice(h->g.s[0]->device));
    h->g.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->g.s[0]->stream));
  });
}

int sfeec_yee_group_energy(sfeec_yee_group* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    double e = 0;
    for (auto& d : h->g.s) e += d->energy();
    *out = e;
  });
}

void sfeec_yee_destroy(sfeec_yee* h) { delete h; }

int sfeec_yee_dof_counts(const sfeec_yee* h, int64_t* n_edges, int64_t* n_faces) {
  return guarded([&] {
    require(h, "null handle");
    if (n_edges) *n_edges = h->d.n_edges;
    if (n_faces) *n_faces = h->d.n_faces;
  });
}

int sfeec_yee_set_state(sfeec_yee* h, const double* b, const double* e, double time) {
  return guarded([&] {
    require(h && b && e, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.set_state(b, e);
    h->d.time = time;
  });
}

int sfeec_yee_get_state(sfeec_yee* h, double* b, double* e, double* time) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.get_state(b, e);
    if (time) *time = h->d.time;
  });
}

int sfeec_yee_advance(sfeec_yee* h, int64_t nsteps) {
  return guarded([&] {
    require(h, "null handle");
    require(nsteps >= 0, "advance: nsteps must be >= 0");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_yee_flow_he(sfeec_yee* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.flow_he(dt);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_yee_flow_ha(sfeec_yee* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.flow_ha(dt);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_yee_energy(sfeec_yee* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.energy();
  });
}

int sfeec_yee_set_stream(sfeec_yee* h, void* s) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    if (d.own_stream) cudaStreamDestroy(d.stream);
    d.stream = (cudaStream_t)s;
    d.own_stream = false;
  });
}

int sfeec_yee_set_variant(sfeec_yee* h, int variant) {
  return guarded([&] {
    require(h, "null handle");
    require(variant >= 0 && variant <= 4 && variant != 3, "variant must be 0, 1, 2 or 4");
    h->d.variant = variant;
  });
}

int64_t sfeec_yee_last_launches(sfeec_yee* h) { return h ? h->d.launches : -1; }

int sfeec_yee_kernel_timing(sfeec_yee* h, int enable, double* ms_total, int64_t* launches) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    if (ms_total) *ms_total = d.kernel_ms;
    if (launches) *launches = d.kernel_launches;
    d.kernel_ms = 0;
    d.kernel_launches = 0;
    d.timing = enable != 0;
    SFEEC_CUDA(cudaSetDevice(d.device));
    for (auto& e : d.ev)
      if (!e) SFEEC_CUDA(cudaEventCreate(&e));
  });
}

// 2 * w * (N1 + N2)
double sfeec_yee_step_bytes(sfeec_yee* h) {
  if (!h) return 0;
  return 2.0 * h->d.prec * (double)(h->d.n_edges + h->d.n_faces);
}

}  // extern "C"
