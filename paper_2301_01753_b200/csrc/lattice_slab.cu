// Multi-rank Kuhn-lattice leapfrog: one process per GPU, the mesh split into
// z-slabs of whole vertex planes.
//
// Rank r of R owns the whole-mesh vertex planes [P_r, P_{r+1}), P_r =
// floor(r (nzg + 1) / R), and everything based on them. It assembles only
// its own slab of the mesh -- planes [P_r - 4, P_{r+1} + 4] (TetMesh
// build_slab, the device assembly of tet_device.cu) -- which makes its
// coefficients bitwise the whole mesh's on the planes it reads ([P_r - 1,
// P_{r+1}]): the S(M1) columns behind them see complete M1 rows four planes
// out. The step runs the four lattice kernels on the owned planes; between
// them one-plane ghosts move to the z-neighbours:
//   t = Q e    -> t's first owned plane down   (C reads t one plane up)
//   b -= h C t -> b's boundary planes both ways (M2 reads b at +-1)
//   u = M2 b   -> u's last owned plane up      (C^T reads u one plane down)
//   e += f C^T u -> e's boundary planes both ways (Q reads e at +-1)
// Reductions (energy, the CFL power iteration's norms) are summed per vertex
// plane in a fixed order, the plane sums exchanged (each plane has one owner,
// so the all-reduce adds exact zeros) and added in plane order: every rank
// count gives bitwise the same number.
//
// Transports (SlabComm):
//   NCCL  ncclSend/ncclRecv of the ghost planes in one group on the compute
//         stream; ncclAllReduce of the plane sums (one GPU per rank);
//   IPC   host-synchronised pulls of the neighbours' planes through CUDA IPC
//         mappings, with a process-shared barrier in POSIX shared memory.
//         No kernel ever waits on another rank, so ranks may share one GPU:
//         this is the transport the single-GPU multi-process tests use.

#include <climits>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "ipc_group.hpp"
#include "lattice.cuh"
#include "nccl_loader.hpp"
#include "tet_device.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

namespace {

constexpr int kPT = 256;  // threads of the per-plane reduction blocks

// sum over local planes [k0, k0 + gridDim.x) of sum_c X[c] . Y[c] over the
// plane's positions, one block per plane, fixed order
__global__ void __launch_bounds__(kPT) k_plane_dot(LatGeom g, int k0, int ncomp,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ y,
                                                   double* __restrict__ out) {
  __shared__ double red[kPT / 32];
  const int k = k0 + blockIdx.x;
  const int64_t base = g.plane(k);
  double acc = 0.0;
  for (int c = 0; c < ncomp; ++c)
    for (int64_t p = threadIdx.x; p < g.PS; p += kPT) {
      const int64_t o = (int64_t)c * g.NP + base + p;
      acc += x[o] * y[o];
    }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kPT / 32; ++w) s += red[w];
    out[blockIdx.x] = s;
  }
}

// x = y / nrm on local planes [k0, k1) of all ncomp components
__global__ void k_plane_div(LatGeom g, int k0, int k1, int ncomp, double* __restrict__ x,
                            const double* __restrict__ y, double nrm) {
  const int64_t n = (int64_t)(k1 - k0) * g.PS;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * ncomp;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / n);
    const int64_t o = (int64_t)c * g.NP + g.plane(k0) + (t - (int64_t)c * n);
    x[o] = y[o] / nrm;
  }
}

// the reference's power-iteration start (dynamics.cpp:117-120): U(-1, 1) of
// the splitmix64 stream at 0x5fec5fec, drawn in whole-mesh DOF order
__global__ void k_uniform_start(int64_t n, int64_t gid0, const int64_t* __restrict__ pos,
                                double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint64_t z = 0x5fec5fecull + (uint64_t)(gid0 + r + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  dst[pos[r]] = -1.0 + 2.0 * ((double)(z >> 11) * 0x1.0p-53);
}

__global__ void k_scatter_owned(int64_t n, const int64_t* __restrict__ pos,
                                const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[pos[r]] = src[r];
}
__global__ void k_gather_owned(int64_t n, const int64_t* __restrict__ pos,
                               const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) dst[r] = src[pos[r]];
}

inline unsigned nb(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

// DOF edges / faces based on one vertex plane kg of the n x n x nzg mesh
int64_t plane_dofs(int n, int nzg, int kg, bool faces) {
  int64_t cnt = 0;
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      const int c[3] = {i, j, kg};
      if (!faces) {
        for (int t = 0; t < 7; ++t) {
          bool ok = true;
          for (int d = 0; d < 3; ++d) {
            const int lim = d < 2 ? n : nzg;
            if (c[d] + kET[t][d] > lim) ok = false;
            if (kET[t][d] == 0 && (c[d] == 0 || c[d] == lim)) ok = false;
          }
          cnt += ok;
        }
      } else {
        for (int f = 0; f < 12; ++f) {
          const int* o = kET[kFT[f][1]];
          cnt += (i + o[0] <= n && j + o[1] <= n && kg + o[2] <= nzg);
        }
      }
    }
  return cnt;
}
// whole-mesh DOFs based on planes [0, P)
int64_t dofs_below(int n, int nzg, int P, bool faces) {
  if (P <= 0) return 0;
  int64_t s = plane_dofs(n, nzg, 0, faces);
  if (P > 1) s += (int64_t)std::min(P - 1, nzg - 1) * plane_dofs(n, nzg, 1, faces);
  if (P > nzg) s += plane_dofs(n, nzg, nzg, faces);
  return s;
}

}  // namespace

// ---- transports -------------------------------------------------------------
struct SlabComm {
  virtual ~SlabComm() = default;
  // ghost planes of `field` (ncomp components): down = every rank's first
  // owned plane to the rank below (its ghost above), up = every rank's last
  // owned plane to the rank above (its ghost below)
  virtual void exchange(double* field, int ncomp, bool up, bool down, cudaStream_t s) = 0;
  // element-wise sum over the ranks of host vectors whose nonzeros are disjoint
  virtual void allreduce_disjoint(double* host, int n, cudaStream_t s) = 0;
};

struct SlabPlan {  // the geometry a transport needs
  int rank = 0, nranks = 1;
  LatGeom g;
  int o0 = 0, o1 = 0;  // owned local planes [o0, o1)
};

struct NcclComm final : SlabComm {
  ncclComm_t comm = nullptr;
  SlabPlan p;
  DevBuf<double> red;
  NcclComm(const SlabPlan& plan, const void* id128) : p(plan) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    Nccl::get().check(Nccl::get().comm_init_rank(&comm, p.nranks, id, p.rank),
                      "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm) Nccl::get().comm_destroy(comm);
  }
  void exchange(double* f, int ncomp, bool up, bool down, cudaStream_t s) override {
    const Nccl& nc = Nccl::get();
    const size_t cnt = (size_t)p.g.PS;
    nc.check(nc.group_start(), "ncclGroupStart");
    for (int c = 0; c < ncomp; ++c) {
      double* base = f + (int64_t)c * p.g.NP;
      if (down) {
        if (p.rank > 0)
          nc.check(nc.send(base + p.g.plane(p.o0), cnt, ncclFloat64, p.rank - 1, comm, s), "send");
        if (p.rank < p.nranks - 1)
          nc.check(nc.recv(base + p.g.plane(p.o1), cnt, ncclFloat64, p.rank + 1, comm, s), "recv");
      }
      if (up) {
        if (p.rank < p.nranks - 1)
          nc.check(nc.send(base + p.g.plane(p.o1 - 1), cnt, ncclFloat64, p.rank + 1, comm, s),
                   "send");
        if (p.rank > 0)
          nc.check(nc.recv(base + p.g.plane(p.o0 - 1), cnt, ncclFloat64, p.rank - 1, comm, s),
                   "recv");
      }
    }
    nc.check(nc.group_end(), "ncclGroupEnd");
  }
  void allreduce_disjoint(double* host, int n, cudaStream_t s) override {
    if ((int)red.n < n) red.alloc((size_t)n);
    SFEEC_CUDA(cudaMemcpyAsync(red.p, host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    Nccl::get().check(
        Nccl::get().all_reduce(red.p, red.p, (size_t)n, ncclFloat64, ncclSum, comm, s),
        "ncclAllReduce");
    SFEEC_CUDA(cudaMemcpyAsync(host, red.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
  }
};

// ---- CUDA IPC transport (host-synchronised) ---------------------------------
constexpr int kIpcMaxRanks = 16;
struct IpcRank {
  cudaIpcMemHandle_t h[4];  // E, T, B, U
  int64_t np = 0;           // component stride of that rank's box
  int kz0 = 0, p0 = 0, p1 = 0;
  // followed by nred doubles: this rank's row of an all-reduce
};

// The shared segment, its barrier and the per-rank slots are ipc_group.hpp's;
// a slot holds IpcRank and the rank's reduction row.
struct IpcComm final : SlabComm {
  SlabPlan p;
  int nred;
  IpcGroup grp;
  double* peer[kIpcMaxRanks][4] = {};
  double* mine[4] = {};

  const IpcRank& info(int q) const { return *(const IpcRank*)grp.slot(q); }
  double* row(int q) const { return (double*)((char*)grp.slot(q) + sizeof(IpcRank)); }

  IpcComm(const SlabPlan& plan, const void* id128, double* fields[4], int p0, int p1, int nred_)
      : p(plan),
        nred(nred_),
        grp("sfeec_lslab", id128, plan.rank, plan.nranks,
            sizeof(IpcRank) + sizeof(double) * (size_t)nred_) {
    require(p.nranks <= kIpcMaxRanks, "IPC transport: at most 16 ranks");
    IpcRank& me = *(IpcRank*)grp.slot(p.rank);
    for (int f = 0; f < 4; ++f) {
      mine[f] = fields[f];
      SFEEC_CUDA(cudaIpcGetMemHandle(&me.h[f], fields[f]));
    }
    me.np = p.g.NP;
    me.kz0 = p.g.kz0;
    me.p0 = p0;
    me.p1 = p1;
    grp.barrier();
    for (int q = 0; q < p.nranks; ++q) {
      if (q == p.rank || (q != p.rank - 1 && q != p.rank + 1)) continue;
      for (int f = 0; f < 4; ++f) {
        void* ptr = nullptr;
        SFEEC_CUDA(cudaIpcOpenMemHandle(&ptr, info(q).h[f], cudaIpcMemLazyEnablePeerAccess));
        peer[q][f] = (double*)ptr;
      }
    }
    grp.barrier();
    grp.unlink_name();  // every rank has it mapped
  }
  ~IpcComm() override {
    for (int q = 0; q < kIpcMaxRanks; ++q)
      for (int f = 0; f < 4; ++f)
        if (peer[q][f]) cudaIpcCloseMemHandle(peer[q][f]);
  }
  void barrier() { grp.barrier(); }
  int field_index(const double* f) const {
    for (int i = 0; i < 4; ++i)
      if (mine[i] == f) return i;
    throw Error(SFEEC_EINVAL, "IPC transport: unknown field");
  }
  // peer q's local plane holding whole-mesh plane kg
  const double* peer_plane(int q, int fi, int c, int kg) const {
    const IpcRank& pr = info(q);
    return peer[q][fi] + (int64_t)c * pr.np + p.g.PS * (int64_t)(kg - pr.kz0 + 1);
  }
  void exchange(double* f, int ncomp, bool up, bool down, cudaStream_t s) override {
    const int fi = field_index(f);
    const size_t b = sizeof(double) * (size_t)p.g.PS;
    SFEEC_CUDA(cudaStreamSynchronize(s));  // our planes are written ...
    barrier();                             // ... and so are the neighbours'
    for (int c = 0; c < ncomp; ++c) {
      double* base = f + (int64_t)c * p.g.NP;
      if (down && p.rank < p.nranks - 1)  // ghost above <- rank+1's first owned plane
        SFEEC_CUDA(cudaMemcpyAsync(base + p.g.plane(p.o1),
                                   peer_plane(p.rank + 1, fi, c, info(p.rank + 1).p0), b,
                                   cudaMemcpyDeviceToDevice, s));
      if (up && p.rank > 0)  // ghost below <- rank-1's last owned plane
        SFEEC_CUDA(cudaMemcpyAsync(base + p.g.plane(p.o0 - 1),
                                   peer_plane(p.rank - 1, fi, c, info(p.rank - 1).p1 - 1), b,
                                   cudaMemcpyDeviceToDevice, s));
    }
    SFEEC_CUDA(cudaStreamSynchronize(s));  // our pulls are done ...
    barrier();                             // ... before anyone overwrites a source plane
  }
  void allreduce_disjoint(double* host, int n, cudaStream_t s) override {
    (void)s;
    require(n <= nred, "IPC transport: reduction longer than the segment row");
    std::memcpy(row(p.rank), host, sizeof(double) * n);
    barrier();
    for (int i = 0; i < n; ++i) {
      double v = 0.0;
      for (int q = 0; q < p.nranks; ++q) v += row(q)[i];
      host[i] = v;
    }
    barrier();
  }
};

// ---- the slab handle -----------------------------------------------------------
struct LatSlab {
  int device = 0, rank = 0, nranks = 1, n = 0, nzg = 0;
  int P0 = 0, P1 = 0, K0 = 0, K1 = 0;  // owned / assembled whole-mesh vertex planes
  cudaStream_t stream = nullptr;
  Lattice L;
  std::unique_ptr<SlabComm> comm;
  int64_t eo0 = 0, eo1 = 0, fo0 = 0, fo1 = 0;  // owned DOFs (slab-local ids)
  int64_t e_glob = 0, f_glob = 0;              // whole-mesh id of the first owned DOF
  DevBuf<int64_t> epos_own, fpos_own;           // owned DOF -> lattice position
  DevBuf<double> partials;
  double dt = 0, eps0 = 1, mu0 = 1, time = 0, cfl_cache = -1;
  int kind = SFEEC_SPLIT_STRANG;
  int64_t launches = 0;
  // per-kernel timing with CUDA events on the stream (classes: 0 K-Q, 1 K-Cb,
  // 2 K-CTe, 3 K-M2); the exchanges fall between the events
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, size_t>> ev_used;
  double class_ms[4] = {0, 0, 0, 0};
  int64_t class_n[4] = {0, 0, 0, 0};

  ~LatSlab() {
    if (comm_stream) cudaStreamSynchronize(comm_stream);
    comm.reset();
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_xch) cudaEventDestroy(ev_xch);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
  void tic(int cls) {
    if (!timing) return;
    const size_t i = ev_used.size() * 2;
    while (ev_pool.size() < i + 2) {
      cudaEvent_t e;
      SFEEC_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    ev_used.push_back({cls, i});
    SFEEC_CUDA(cudaEventRecord(ev_pool[i], stream));
  }
  void toc() {
    if (timing) SFEEC_CUDA(cudaEventRecord(ev_pool[ev_used.back().second + 1], stream));
  }
  void collect() {
    if (ev_used.empty()) return;
    SFEEC_CUDA(cudaStreamSynchronize(stream));
    for (auto [cls, i] : ev_used) {
      float ms = 0;
      SFEEC_CUDA(cudaEventElapsedTime(&ms, ev_pool[i], ev_pool[i + 1]));
      class_ms[cls] += ms;
      class_n[cls] += 1;
    }
    ev_used.clear();
  }
  double c2() const { return 1.0 / (eps0 * mu0); }
  int o0() const { return P0 - K0; }
  int o1() const { return P1 - K0; }

  void xch(double* f, int nc, bool up, bool down) {
    if (nranks > 1) comm->exchange(f, nc, up, down, stream);
  }

  // Overlap (SFEEC_PART_OVERLAP, default on with more than one rank): a
  // kernel whose output is exchanged first computes the boundary planes the
  // neighbours need, an event releases their exchange on the comm stream,
  // and the interior planes run meanwhile; the next kernel waits for the
  // exchange (it is the first to read the ghosts). The exchanged planes are
  // not written again before that wait, and the ghosts are written only by
  // the exchange. Results are bitwise the serialised schedule's.
  bool overlap = false;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_xch = nullptr;
  bool pending = false;
  void make_overlap() {
    overlap = nranks > 1 && env_flag("SFEEC_PART_OVERLAP", true);
    if (!overlap) return;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
    SFEEC_CUDA(cudaEventCreateWithFlags(&ev_bnd, cudaEventDisableTiming));
    SFEEC_CUDA(cudaEventCreateWithFlags(&ev_xch, cudaEventDisableTiming));
  }
  void wait_pending() {
    if (pending) SFEEC_CUDA(cudaStreamWaitEvent(stream, ev_xch, 0));
    pending = false;
  }
  // run kern(kb, ke) over the owned planes and exchange field f
  template <class K>
  void produce(K&& kern, double* f, int nc, bool up, bool down) {
    wait_pending();
    const int a = o0(), b = o1();
    if (!overlap) {
      kern(a, b);
      xch(f, nc, up, down);
      return;
    }
    int ib = a, ie = b;
    if (down && rank > 0 && ib < ie) {  // the first owned plane goes to the rank below
      kern(ib, ib + 1);
      ib += 1;
    }
    if (up && rank < nranks - 1 && ie > ib) {  // the last one to the rank above
      kern(ie - 1, ie);
      ie -= 1;
    }
    SFEEC_CUDA(cudaEventRecord(ev_bnd, stream));
    SFEEC_CUDA(cudaStreamWaitEvent(comm_stream, ev_bnd, 0));
    comm->exchange(f, nc, up, down, comm_stream);
    SFEEC_CUDA(cudaEventRecord(ev_xch, comm_stream));
    pending = true;
    kern(ib, ie);  // the interior planes, beside the exchange
  }

  // the four kernels + their ghost exchanges (see the file comment)
  void he(double h) {
    tic(0);
    produce([&](int kb, int ke) { L.apply_q(stream, kb, ke); }, L.T.p, 7, false, true);
    toc();
    tic(1);
    produce([&](int kb, int ke) { L.apply_cb(h, stream, kb, ke); }, L.B.p, 12, true, true);
    toc();
    launches += 2;
  }
  void ha(double h) {
    tic(3);
    produce([&](int kb, int ke) { L.apply_m2(stream, kb, ke); }, L.U.p, 12, true, false);
    toc();
    tic(2);
    const double f = h * c2();
    produce([&](int kb, int ke) { L.apply_cte(f, stream, kb, ke); }, L.E.p, 7, true, true);
    toc();
    launches += 2;
  }
  void advance(int64_t nsteps) {
    launches = 0;
    if (nsteps <= 0) return;
    if (kind == SFEEC_SPLIT_LIE_TROTTER) {
      for (int64_t s = 0; s < nsteps; ++s) {
        he(dt);
        ha(dt);
      }
      wait_pending();
    } else {  // merged Strang: He(h/2) [Ha(h) He(h)]^(n-1) Ha(h) He(h/2)
      he(0.5 * dt);
      for (int64_t s = 1; s < nsteps; ++s) {
        ha(dt);
        he(dt);
      }
      ha(dt);
      he(0.5 * dt);
    }
    wait_pending();
    for (int64_t s = 0; s < nsteps; ++s) time = time + dt;
  }

  // sum over owned planes of X . Y, plane sums combined across the ranks
  double plane_sum(int ncomp, const double* x, const double* y) {
    const int nown = o1() - o0();
    std::vector<double> all((size_t)nzg + 1, 0.0);
    if (nown > 0) {
      k_plane_dot<<<nown, kPT, 0, stream>>>(L.g, o0(), ncomp, x, y, partials.p);
      SFEEC_LAUNCH_CHECK();
      SFEEC_CUDA(cudaMemcpyAsync(all.data() + P0, partials.p, sizeof(double) * nown,
                                 cudaMemcpyDeviceToHost, stream));
      SFEEC_CUDA(cudaStreamSynchronize(stream));
    }
    if (nranks > 1) comm->allreduce_disjoint(all.data(), nzg + 1, stream);
    double s = 0.0;
    for (double v : all) s += v;
    return s;
  }

  // 1/2 (eps0 e.Q e + b.M2 b / mu0) (dynamics.cpp:92-102); uses T and U as
  // scratch (the flows recompute them before reading)
  double energy() {
    L.apply_q(stream);
    const double he_ = plane_sum(7, L.E.p, L.T.p);
    L.apply_m2(stream);
    const double ha_ = plane_sum(12, L.B.p, L.U.p);
    return 0.5 * (eps0 * he_ + ha_ / mu0);
  }

  // dt sqrt(c^2 lambda), lambda the power iteration's spectral radius of
  // Q C^T M2 C (dynamics.cpp:114-133, 40 iterations from the reference start)
  double cfl_number() {
    if (cfl_cache >= 0) return cfl_cache;
    const size_t ne = (size_t)(7 * L.g.NP), nf = (size_t)(12 * L.g.NP);
    DevBuf<double> keepE, keepB;  // the state survives the iteration
    keepE.alloc(ne);
    keepB.alloc(nf);
    SFEEC_CUDA(cudaMemcpyAsync(keepE.p, L.E.p, sizeof(double) * ne, cudaMemcpyDeviceToDevice, stream));
    SFEEC_CUDA(cudaMemcpyAsync(keepB.p, L.B.p, sizeof(double) * nf, cudaMemcpyDeviceToDevice, stream));
    L.T.zero(stream);
    if (eo1 > eo0)
      k_uniform_start<<<nb(eo1 - eo0), 256, 0, stream>>>(eo1 - eo0, e_glob, epos_own.p, L.T.p);
    SFEEC_LAUNCH_CHECK();
    double lambda = 0.0;
    for (int it = 0; it < 40; ++it) {
      // B = C x (x in T), U = M2 B, E = C^T U, T = Q E
      xch(L.T.p, 7, false, true);
      L.B.zero(stream);
      L.apply_cb(-1.0, stream);
      xch(L.B.p, 12, true, true);
      L.apply_m2(stream);
      xch(L.U.p, 12, true, false);
      L.E.zero(stream);
      L.apply_cte(1.0, stream);
      xch(L.E.p, 7, true, true);
      L.apply_q(stream);
      const double nrm = std::sqrt(plane_sum(7, L.T.p, L.T.p));
      if (nrm == 0) break;
      lambda = nrm;
      const int nown = o1() - o0();
      if (nown > 0) {
        k_plane_div<<<148 * 8, 256, 0, stream>>>(L.g, o0(), o1(), 7, L.T.p, L.T.p, nrm);
        SFEEC_LAUNCH_CHECK();
      }
    }
    SFEEC_CUDA(cudaMemcpyAsync(L.E.p, keepE.p, sizeof(double) * ne, cudaMemcpyDeviceToDevice, stream));
    SFEEC_CUDA(cudaMemcpyAsync(L.B.p, keepB.p, sizeof(double) * nf, cudaMemcpyDeviceToDevice, stream));
    SFEEC_CUDA(cudaStreamSynchronize(stream));
    cfl_cache = dt * std::sqrt(c2() * lambda);
    return cfl_cache;
  }

  void set_state(const double* b, const double* e, bool host) {
    const cudaMemcpyKind k = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    DevBuf<double> db, de;
    db.alloc((size_t)std::max<int64_t>(1, fo1 - fo0));
    de.alloc((size_t)std::max<int64_t>(1, eo1 - eo0));
    if (fo1 > fo0)
      SFEEC_CUDA(cudaMemcpyAsync(db.p, b, sizeof(double) * (size_t)(fo1 - fo0), k, stream));
    if (eo1 > eo0)
      SFEEC_CUDA(cudaMemcpyAsync(de.p, e, sizeof(double) * (size_t)(eo1 - eo0), k, stream));
    L.B.zero(stream);
    L.E.zero(stream);
    if (fo1 > fo0) k_scatter_owned<<<nb(fo1 - fo0), 256, 0, stream>>>(fo1 - fo0, fpos_own.p, db.p, L.B.p);
    if (eo1 > eo0) k_scatter_owned<<<nb(eo1 - eo0), 256, 0, stream>>>(eo1 - eo0, epos_own.p, de.p, L.E.p);
    SFEEC_LAUNCH_CHECK();
    xch(L.B.p, 12, true, true);
    xch(L.E.p, 7, true, true);
    SFEEC_CUDA(cudaStreamSynchronize(stream));
  }
  void get_state(double* b, double* e) {
    DevBuf<double> db, de;
    db.alloc((size_t)std::max<int64_t>(1, fo1 - fo0));
    de.alloc((size_t)std::max<int64_t>(1, eo1 - eo0));
    if (fo1 > fo0) k_gather_owned<<<nb(fo1 - fo0), 256, 0, stream>>>(fo1 - fo0, fpos_own.p, L.B.p, db.p);
    if (eo1 > eo0) k_gather_owned<<<nb(eo1 - eo0), 256, 0, stream>>>(eo1 - eo0, epos_own.p, L.E.p, de.p);
    SFEEC_LAUNCH_CHECK();
    if (b && fo1 > fo0)
      SFEEC_CUDA(cudaMemcpyAsync(b, db.p, sizeof(double) * (size_t)(fo1 - fo0), cudaMemcpyDeviceToHost, stream));
    if (e && eo1 > eo0)
      SFEEC_CUDA(cudaMemcpyAsync(e, de.p, sizeof(double) * (size_t)(eo1 - eo0), cudaMemcpyDeviceToHost, stream));
    SFEEC_CUDA(cudaStreamSynchronize(stream));
  }
  // b = C a on the owned faces (e.g. B0 = C A); the state is left as (b, a)
  void curl(const double* a, double* b) {
    std::vector<double> zero((size_t)std::max<int64_t>(1, fo1 - fo0), 0.0);
    set_state(zero.data(), a, true);
    SFEEC_CUDA(cudaMemcpyAsync(L.T.p, L.E.p, sizeof(double) * (size_t)(7 * L.g.NP),
                               cudaMemcpyDeviceToDevice, stream));
    L.apply_cb(-1.0, stream);  // B -= (-1) C T
    SFEEC_LAUNCH_CHECK();
    get_state(b, nullptr);
  }
};

}  // namespace sfeec_b200

using namespace sfeec_b200;

struct sfeec_lslab {
  LatSlab d;
};

extern "C" {

int sfeec_ipc_unique_id(void* out128) {
  return guarded([&] {
    require(out128 != nullptr, "null out");
    std::random_device rd;
    unsigned char* b = (unsigned char*)out128;
    std::memset(b, 0, 128);
    for (int i = 0; i < 16; ++i) b[i] = (unsigned char)(rd() & 0xff);
  });
}

// Host-only check of the IPC group (ipc_group.hpp): every rank writes
// rank + round into its slot, and after a barrier sums all slots; `rounds`
// rounds, the last sum out. No CUDA call: runs without a GPU.
int sfeec_ipc_group_selftest(const void* id128, int rank, int nranks, int rounds, double* out) {
  return guarded([&] {
    require(id128 && out && nranks >= 1 && rank >= 0 && rank < nranks && rounds >= 1,
            "sfeec_ipc_group_selftest: bad argument");
    IpcGroup g("sfeec_selftest", id128, rank, nranks, sizeof(double));
    g.barrier();
    g.unlink_name();
    double sum = 0.0;
    for (int r = 0; r < rounds; ++r) {
      *(double*)g.slot(rank) = (double)(rank + r);
      g.barrier();  // every slot of this round is written
      sum = 0.0;
      for (int q = 0; q < nranks; ++q) sum += *(const double*)g.slot(q);
      g.barrier();  // ... and read, before the next round overwrites it
    }
    *out = sum;
  });
}

int sfeec_lslab_create(int n, int nzg, double jitter, uint64_t seed, double dt, double eps0,
                       double mu0, int split_kind, int rank, int nranks, int transport,
                       const void* comm_id, int device, sfeec_lslab** out, int64_t* info) {
  return guarded([&] {
    require(out != nullptr, "null out");
    *out = nullptr;
    require(n >= 1 && nzg >= 1, "lattice slab: n, nzg must be >= 1");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "lattice slab: bad rank / nranks");
    require(nranks <= nzg + 1, "lattice slab: need nranks <= nzg + 1 vertex planes");
    require(nranks == 1 || comm_id, "lattice slab: multi-rank needs a communicator id");
    require(transport == 0 || transport == 1, "lattice slab: transport 0 (NCCL) or 1 (IPC)");
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    select_device(device);
    auto h = std::make_unique<sfeec_lslab>();
    LatSlab& d = h->d;
    d.device = device;
    d.rank = rank;
    d.nranks = nranks;
    d.n = n;
    d.nzg = nzg;
    d.dt = dt;
    d.eps0 = eps0;
    d.mu0 = mu0;
    d.kind = split_kind;
    d.P0 = (int)((int64_t)rank * (nzg + 1) / nranks);
    d.P1 = (int)((int64_t)(rank + 1) * (nzg + 1) / nranks);
    d.K0 = std::max(0, d.P0 - 4);
    d.K1 = std::min(nzg, d.P1 + 4);
    SFEEC_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    {
      TetMesh mesh;
      mesh.build_slab(n, nzg, d.K0, d.K1, jitter, seed);
      // owned DOFs: based on local planes [o0, o1) -- contiguous ids (k-major)
      auto first_at = [&](const std::vector<int64_t>& base, int k) {
        const int64_t v = (int64_t)(n + 1) * (n + 1) * k;
        return (int64_t)(std::lower_bound(base.begin(), base.end(), v) - base.begin());
      };
      d.eo0 = first_at(mesh.edge_v, d.o0());
      d.eo1 = first_at(mesh.edge_v, d.o1());
      d.fo0 = first_at(mesh.face_v, d.o0());
      d.fo1 = first_at(mesh.face_v, d.o1());
      d.e_glob = dofs_below(n, nzg, d.P0, false);
      d.f_glob = dofs_below(n, nzg, d.P0, true);
      Stream st;
      DevTetSystem sys;
      build_tet_system_device(mesh, false, sys, st.s, d.o0() - 3, d.o1() + 3);
      d.L.build(mesh, sys.qsym, sys.m2, st.s);
      d.L.k0 = d.o0();
      d.L.k1 = d.o1();
      d.epos_own.alloc((size_t)std::max<int64_t>(1, d.eo1 - d.eo0));
      d.fpos_own.alloc((size_t)std::max<int64_t>(1, d.fo1 - d.fo0));
      if (d.eo1 > d.eo0)
        SFEEC_CUDA(cudaMemcpyAsync(d.epos_own.p, d.L.epos.p + d.eo0,
                                   sizeof(int64_t) * (size_t)(d.eo1 - d.eo0),
                                   cudaMemcpyDeviceToDevice, st.s));
      if (d.fo1 > d.fo0)
        SFEEC_CUDA(cudaMemcpyAsync(d.fpos_own.p, d.L.fpos.p + d.fo0,
                                   sizeof(int64_t) * (size_t)(d.fo1 - d.fo0),
                                   cudaMemcpyDeviceToDevice, st.s));
      SFEEC_CUDA(cudaStreamSynchronize(st.s));
      d.L.epos.reset();  // the owned maps are all the slab keeps
      d.L.fpos.reset();
    }
    d.partials.alloc((size_t)std::max(1, d.o1() - d.o0()));
    if (nranks > 1) {
      SlabPlan plan{rank, nranks, d.L.g, d.o0(), d.o1()};
      if (transport == 0) {
        d.comm = std::make_unique<NcclComm>(plan, comm_id);
      } else {
        double* fields[4] = {d.L.E.p, d.L.T.p, d.L.B.p, d.L.U.p};
        d.comm = std::make_unique<IpcComm>(plan, comm_id, fields, d.P0, d.P1, nzg + 1);
      }
      d.make_overlap();
    }
    if (info) {
      info[0] = d.eo1 - d.eo0;  // owned edges
      info[1] = d.fo1 - d.fo0;  // owned faces
      info[2] = d.e_glob;       // whole-mesh id of the first owned edge
      info[3] = d.f_glob;
      info[4] = d.P0;
      info[5] = d.P1;
      info[6] = d.K0;
      info[7] = d.K1;
      info[8] = d.eo0;  // slab-local id of the first owned edge / face
      info[9] = d.fo0;
    }
    *out = h.release();
  });
}

void sfeec_lslab_destroy(sfeec_lslab* h) { delete h; }

int sfeec_lslab_set_state(sfeec_lslab* h, const double* b, const double* e, double time) {
  return guarded([&] {
    require(h && (b || h->d.fo1 == h->d.fo0) && (e || h->d.eo1 == h->d.eo0), "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.set_state(b, e, true);
    h->d.time = time;
  });
}

int sfeec_lslab_get_state(sfeec_lslab* h, double* b, double* e, double* time) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.get_state(b, e);
    if (time) *time = h->d.time;
  });
}

int sfeec_lslab_advance(sfeec_lslab* h, int64_t nsteps) {
  return guarded([&] {
    require(h && nsteps >= 0, "bad argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_lslab_energy(sfeec_lslab* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.energy();
  });
}

int sfeec_lslab_cfl_number(sfeec_lslab* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.cfl_number();
  });
}

int sfeec_lslab_set_dt(sfeec_lslab* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    auto& d = h->d;
    d.cfl_cache = (d.cfl_cache >= 0 && d.dt > 0) ? d.cfl_cache / d.dt * dt : -1;
    d.dt = dt;
  });
}

int sfeec_lslab_curl(sfeec_lslab* h, const double* a, double* b) {
  return guarded([&] {
    require(h && b && (a || h->d.eo1 == h->d.eo0), "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.curl(a, b);
  });
}

int sfeec_lslab_stream(sfeec_lslab* h, void** stream) {
  return guarded([&] {
    require(h && stream, "null argument");
    *stream = (void*)h->d.stream;
  });
}

int64_t sfeec_lslab_last_launches(sfeec_lslab* h) { return h ? h->d.launches : -1; }

// bytes one step's four lattice kernels move on this rank (lattice.cu counts)
double sfeec_lslab_step_bytes(sfeec_lslab* h) { return h ? h->d.L.step_bytes() : 0.0; }

// device time per kernel class since the last call (0 K-Q, 1 K-Cb, 2 K-CTe,
// 3 K-M2, as sfeec_dev_kernel_timing), launches and bytes per launch; then
// (dis)arms the timing
int sfeec_lslab_kernel_timing(sfeec_lslab* h, int enable, double* ms, int64_t* launches,
                              double* bytes) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    d.collect();
    for (int k = 0; k < 4; ++k) {
      if (ms) ms[k] = d.class_ms[k];
      if (launches) launches[k] = d.class_n[k];
      d.class_ms[k] = 0;
      d.class_n[k] = 0;
    }
    if (bytes) {
      bytes[0] = d.L.bytes_q();
      bytes[1] = d.L.bytes_cb();
      bytes[2] = d.L.bytes_cte();
      bytes[3] = d.L.bytes_m2();
    }
    d.timing = enable != 0;
  });
}

}  // extern "C"
