// Partitioned unstructured leapfrog: one z-slab of a tet mesh per GPU.
//
// The tet DOF numbering is k-major (host_tet.cpp), so the entities whose base
// vertex lies in a range of z-planes are a contiguous id range. Rank r owns
// planes [P_r, P_{r+1}); its local vectors cover planes [P_r - 1, P_{r+1}]
// (one halo plane each side = the one-layer halo of SURVEY.md 8(e)), and its
// local operators are the owned rows with columns shifted into that range:
//   Q_sym, C^T : rows = owned edges      C, M2 : rows = owned faces
// The merged Strang step needs four halo refreshes (b before K-M2, u before
// K-CTe, e before K-Q, t before K-Cb); each sends the first owned plane(s)
// down and the last owned plane(s) up (contiguous ranges, no packing) with
// ncclSend/ncclRecv. Each operator is split by output rows (SplitOp): the
// producing kernel computes the rows to be sent first, the exchange then runs
// on a comm stream beside the interior rows, and the next kernel waits on it.
// To verify the multi-rank path on one GPU, handles advanced in lockstep run
// the same split schedule with device copies between phases.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "dev_handle.hpp"
#include "device_util.cuh"
#include "ipc_group.hpp"
#include "nccl_loader.hpp"
#include "spmv_kernels.cuh"
#include "p2_device.hpp"
#include "tet_device.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {

struct PartRange {
  int64_t len = 0, own_lo = 0, own_hi = 0, first_len = 0, last_len = 0;
};

// An operator split by output rows: the rows whose values the lower / upper
// neighbour needs come first, the interior rows after, so the halo exchange of
// the produced vector can overlap the interior part. Each part is an ordinary
// sliced / ELL operator, so every row's arithmetic (and result) is unchanged.
struct SplitOp {
  DevOperator part[3];  // 0: rows sent down, 1: rows sent up, 2: interior
  int64_t row0[3] = {0, 0, 0};
  int64_t rows = 0, cols = 0, nnz = 0;
  bool incidence = false;  // +-1 entries (5 B per entry in the algorithmic count)

  void build(DevCSR&& a, int64_t lo_rows, int64_t hi_rows, cudaStream_t s) {
    rows = a.rows;
    cols = a.cols;
    nnz = a.nnz;
    const int64_t lo = std::min(lo_rows, rows);
    const int64_t hi = std::min(hi_rows, rows - lo);
    const int64_t r0[3] = {0, rows - hi, lo}, r1[3] = {lo, rows, rows - hi};
    for (int k = 0; k < 3; ++k) {
      row0[k] = r0[k];
      if (r1[k] <= r0[k]) continue;
      DevCSR sub;
      slice_rows_device(a, r0[k], r1[k], 0, cols, sub, s);
      part[k].upload_device(std::move(sub), s);
      incidence = incidence || part[k].layout == DevOperator::kSigned;
    }
  }
  // which: 0 / 1 / 2 a single part, -1 the boundary parts, -2 all
  void launch(int which, const double* x, double* y, double alpha, bool acc,
              cudaStream_t s) const {
    for (int k = 0; k < 3; ++k) {
      const bool sel = which == -2 || (which == -1 && k < 2) || which == k;
      if (sel && part[k].rows > 0) launch_spmv(part[k], x, y + row0[k], alpha, acc, s);
    }
  }
};

struct PartDev {
  int device = 0;
  cudaStream_t stream = nullptr;
  // overlap: the exchange of a produced vector runs on comm_stream while the
  // interior rows are computed; the next kernel waits for it (ev_xch)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_xch = nullptr;
  bool overlap = true, xch_pending = false;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  // CUDA-IPC transport (host-synchronised; the ranks may share a GPU): the
  // neighbours' e, t, b, u vectors mapped into this process
  struct IpcSlot {
    cudaIpcMemHandle_t h[4];
    PartRange r1, r2;
  };
  std::unique_ptr<IpcGroup> ipc;
  double* peer_lo[4] = {nullptr, nullptr, nullptr, nullptr};
  double* peer_hi[4] = {nullptr, nullptr, nullptr, nullptr};
  double dt = 0, eps0 = 1, mu0 = 1;
  PartRange r1, r2;  // edges, faces
  SplitOp q, c, ct, m2;
  DevBuf<double> e, t, b, u, partials;
  double time = 0;
  int64_t launches = 0;
  // per-class launch timing with CUDA events on the compute stream
  // (0 K-Q, 1 K-Cb, 2 K-CTe, 3 K-M2, 4 halo exchange)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, size_t>> ev_used;
  double class_ms[5] = {0, 0, 0, 0, 0};
  int64_t class_launches[5] = {0, 0, 0, 0, 0};

  ~PartDev() {
    for (auto ev : ev_pool) cudaEventDestroy(ev);
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_xch) cudaEventDestroy(ev_xch);
    if (comm) Nccl::get().comm_destroy(comm);
    for (int f = 0; f < 4; ++f) {
      if (peer_lo[f]) cudaIpcCloseMemHandle(peer_lo[f]);
      if (peer_hi[f]) cudaIpcCloseMemHandle(peer_hi[f]);
    }
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (stream) cudaStreamDestroy(stream);
  }

  void tic(int cls) {
    if (!timing) return;
    const size_t i = ev_used.size() * 2;
    while (ev_pool.size() < i + 2) {
      cudaEvent_t ev;
      SFEEC_CUDA(cudaEventCreate(&ev));
      ev_pool.push_back(ev);
    }
    ev_used.push_back({cls, i});
    SFEEC_CUDA(cudaEventRecord(ev_pool[i], stream));
  }
  void toc() {
    if (timing) SFEEC_CUDA(cudaEventRecord(ev_pool[ev_used.back().second + 1], stream));
  }
  void collect_timing() {
    if (ev_used.empty()) return;
    SFEEC_CUDA(cudaStreamSynchronize(stream));
    for (auto [cls, i] : ev_used) {
      float ms = 0;
      SFEEC_CUDA(cudaEventElapsedTime(&ms, ev_pool[i], ev_pool[i + 1]));
      class_ms[cls] += ms;
      class_launches[cls] += 1;
    }
    ev_used.clear();
  }

  // op codes of the step program
  enum Op { kXe, kXt, kXb, kXu, kQ, kCb, kM2, kCTe };
  struct Step {
    Op op;
    double alpha;
  };

  std::vector<Step> program(int64_t n) const {
    std::vector<Step> p;
    if (n <= 0) return p;
    const double f = dt / (eps0 * mu0);
    p.push_back({kXe, 0});
    p.push_back({kQ, 0});
    p.push_back({kXt, 0});
    p.push_back({kCb, -0.5 * dt});
    for (int64_t s = 0; s < n; ++s) {
      p.push_back({kXb, 0});
      p.push_back({kM2, 0});
      p.push_back({kXu, 0});
      p.push_back({kCTe, f});
      p.push_back({kXe, 0});
      p.push_back({kQ, 0});
      p.push_back({kXt, 0});
      p.push_back({kCb, s == n - 1 ? -0.5 * dt : -dt});
    }
    return p;
  }

  void operands(Op op, const SplitOp*& A, const double*& x, double*& y, bool& acc) {
    acc = false;
    switch (op) {
      case kQ: A = &q; x = e.p; y = t.p + r1.own_lo; break;
      case kCb: A = &c; x = t.p; y = b.p + r2.own_lo; acc = true; break;
      case kM2: A = &m2; x = b.p; y = u.p + r2.own_lo; break;
      case kCTe: A = &ct; x = u.p; y = e.p + r1.own_lo; acc = true; break;
      default: A = nullptr; x = nullptr; y = nullptr; break;
    }
  }
  // one part selection of a kernel (the lockstep driver's split schedule)
  void kernel_part(const Step& s, int which) {
    const SplitOp* A;
    const double* x;
    double* y;
    bool acc;
    operands(s.op, A, x, y, acc);
    if (A) A->launch(which, x, y, s.alpha, acc, stream);
    if (which != -1) ++launches;
  }

  // the exchange that follows each kernel in the program
  static Op produced(Op k) { return k == kQ ? kXt : k == kCb ? kXb : k == kM2 ? kXu : kXe; }

  // xchg: the program's next step exchanges this kernel's output -- with
  // NCCL and overlap on, the boundary rows go first and the exchange runs on
  // comm_stream beside the interior rows
  void kernel(const Step& s, bool xchg = false) {
    if (s.op < kQ) return;
    if (xch_pending) {  // this kernel reads the halo exchanged last
      SFEEC_CUDA(cudaStreamWaitEvent(stream, ev_xch, 0));
      xch_pending = false;
    }
    tic(s.op == kQ ? 0 : s.op == kCb ? 1 : s.op == kCTe ? 2 : 3);
    const SplitOp* A = nullptr;
    const double* x = nullptr;
    double* y = nullptr;
    bool acc = false;
    operands(s.op, A, x, y, acc);
    if (xchg && overlap && nranks > 1 && comm) {
      A->launch(-1, x, y, s.alpha, acc, stream);
      SFEEC_CUDA(cudaEventRecord(ev_bnd, stream));
      SFEEC_CUDA(cudaStreamWaitEvent(comm_stream, ev_bnd, 0));
      exchange_nccl(produced(s.op), comm_stream);
      SFEEC_CUDA(cudaEventRecord(ev_xch, comm_stream));
      xch_pending = true;
      A->launch(2, x, y, s.alpha, acc, stream);
    } else {
      A->launch(-2, x, y, s.alpha, acc, stream);
    }
    toc();
    ++launches;
  }

  double* vec(Op x) { return x == kXe ? e.p : x == kXt ? t.p : x == kXb ? b.p : u.p; }
  const PartRange& range(Op x) const { return (x == kXe || x == kXt) ? r1 : r2; }

  static int vec_index(Op x) { return x == kXe ? 0 : x == kXt ? 1 : x == kXb ? 2 : 3; }
  // join the ranks' shared segment and map the neighbours' vectors (collective)
  void attach_ipc(const void* id128) {
    require(nranks > 1 && !comm && !ipc, "attach_ipc: a multi-rank handle without a transport");
    ipc = std::make_unique<IpcGroup>("sfeec_part", id128, rank, nranks, sizeof(IpcSlot));
    IpcSlot& me = *(IpcSlot*)ipc->slot(rank);
    double* mine[4] = {e.p, t.p, b.p, u.p};
    for (int f = 0; f < 4; ++f) SFEEC_CUDA(cudaIpcGetMemHandle(&me.h[f], mine[f]));
    me.r1 = r1;
    me.r2 = r2;
    ipc->barrier();
    for (int f = 0; f < 4; ++f) {
      void* q = nullptr;
      if (rank > 0) {
        SFEEC_CUDA(cudaIpcOpenMemHandle(&q, ((IpcSlot*)ipc->slot(rank - 1))->h[f],
                                        cudaIpcMemLazyEnablePeerAccess));
        peer_lo[f] = (double*)q;
      }
      if (rank < nranks - 1) {
        SFEEC_CUDA(cudaIpcOpenMemHandle(&q, ((IpcSlot*)ipc->slot(rank + 1))->h[f],
                                        cudaIpcMemLazyEnablePeerAccess));
        peer_hi[f] = (double*)q;
      }
    }
    ipc->barrier();
    ipc->unlink_name();
  }
  // the ranges exchange_nccl sends, pulled from the neighbours' vectors
  // between two host barriers
  void exchange_ipc(Op x, cudaStream_t st) {
    const int f = vec_index(x);
    const bool edges = x == kXe || x == kXt;
    const PartRange& R = range(x);
    double* v = vec(x);
    SFEEC_CUDA(cudaStreamSynchronize(st));  // our rows are written ...
    ipc->barrier();                         // ... and so are the neighbours'
    if (rank > 0) {  // halo below <- the lower neighbour's last owned plane(s)
      const IpcSlot& lo = *(const IpcSlot*)ipc->slot(rank - 1);
      const PartRange& Lr = edges ? lo.r1 : lo.r2;
      require(Lr.last_len == R.own_lo, "partition: halo sizes disagree");
      SFEEC_CUDA(cudaMemcpyAsync(v, peer_lo[f] + Lr.own_hi - Lr.last_len,
                                 sizeof(double) * (size_t)R.own_lo, cudaMemcpyDeviceToDevice, st));
    }
    if (rank < nranks - 1) {  // halo above <- the upper neighbour's first owned plane(s)
      const IpcSlot& hi = *(const IpcSlot*)ipc->slot(rank + 1);
      const PartRange& Hr = edges ? hi.r1 : hi.r2;
      require(Hr.first_len == R.len - R.own_hi, "partition: halo sizes disagree");
      SFEEC_CUDA(cudaMemcpyAsync(v + R.own_hi, peer_hi[f] + Hr.own_lo,
                                 sizeof(double) * (size_t)(R.len - R.own_hi),
                                 cudaMemcpyDeviceToDevice, st));
    }
    SFEEC_CUDA(cudaStreamSynchronize(st));  // our pulls are done ...
    ipc->barrier();                         // ... before anyone overwrites a source row
  }
  void exchange_nccl(Op x) { exchange_nccl(x, stream); }
  void exchange_nccl(Op x, cudaStream_t stream) {
    if (nranks > 1 && ipc) return exchange_ipc(x, stream);
    if (nranks == 1 || !comm) return;
    const Nccl& nc = Nccl::get();
    const PartRange& R = range(x);
    double* v = vec(x);
    nc.check(nc.group_start(), "ncclGroupStart");
    if (rank > 0) {
      nc.check(nc.send(v + R.own_lo, (size_t)R.first_len, ncclFloat64, rank - 1, comm, stream), "ncclSend");
      nc.check(nc.recv(v, (size_t)R.own_lo, ncclFloat64, rank - 1, comm, stream), "ncclRecv");
    }
    if (rank < nranks - 1) {
      nc.check(nc.recv(v + R.own_hi, (size_t)(R.len - R.own_hi), ncclFloat64, rank + 1, comm, stream),
               "ncclRecv");
      nc.check(nc.send(v + R.own_hi - R.last_len, (size_t)R.last_len, ncclFloat64, rank + 1, comm, stream),
               "ncclSend");
    }
    nc.check(nc.group_end(), "ncclGroupEnd");
  }

  void advance(int64_t n) {
    launches = 0;
    const auto prog = program(n);
    for (size_t i = 0; i < prog.size(); ++i) {
      const Step& s = prog[i];
      if (s.op <= kXu) {
        if (nranks == 1 || (!comm && !ipc)) continue;
        if (comm && overlap && i > 0 && prog[i - 1].op >= kQ && produced(prog[i - 1].op) == s.op)
          continue;  // already in flight beside the interior rows
        tic(4);
        exchange_nccl(s.op, stream);
        toc();
      } else {
        const bool xchg = i + 1 < prog.size() && prog[i + 1].op == produced(s.op);
        kernel(s, xchg);
      }
    }
    if (xch_pending) {
      SFEEC_CUDA(cudaStreamWaitEvent(stream, ev_xch, 0));
      xch_pending = false;
    }
    for (int64_t k = 0; k < n; ++k) time = time + dt;
  }

  // SURVEY.md 8(d) accounting of this rank's rows (as sfeec_dev_step_bytes)
  double op_bytes(int cls) const {
    const double o1 = (double)(r1.own_hi - r1.own_lo), o2 = (double)(r2.own_hi - r2.own_lo);
    switch (cls) {
      case 0: return 12.0 * (double)q.nnz + 16.0 * o1;
      case 1: return (c.incidence ? 5.0 : 12.0) * (double)c.nnz + 8.0 * o1 + 16.0 * o2;
      case 2: return (ct.incidence ? 5.0 : 12.0) * (double)ct.nnz + 8.0 * o2 + 16.0 * o1;
      case 3: return 12.0 * (double)m2.nnz + 16.0 * o2;
      default: return 0.0;
    }
  }


  // this rank's part of 0.5 (eps0 e^T Q e + b^T M2 b / mu0); halos of e and b
  // must be current (the callers refresh them)
  double energy() {
    q.launch(-2, e.p, t.p + r1.own_lo, 0.0, false, stream);
    m2.launch(-2, b.p, u.p + r2.own_lo, 0.0, false, stream);
    double he = device_dot(e.p + r1.own_lo, t.p + r1.own_lo, r1.own_hi - r1.own_lo, partials.p, stream);
    double ha = device_dot(b.p + r2.own_lo, u.p + r2.own_lo, r2.own_hi - r2.own_lo, partials.p, stream);
    return 0.5 * (eps0 * he + ha / mu0);
  }
};

// lockstep driver for R handles on one device (local transport)
void local_exchange(std::vector<PartDev*>& hs, PartDev::Op x) {
  const int R = (int)hs.size();
  for (int r = 0; r < R; ++r) {
    PartDev& a = *hs[(size_t)r];
    const PartRange& A = a.range(x);
    double* va = a.vec(x);
    if (r > 0) {  // my first owned plane -> lower neighbour's halo above
      PartDev& lo = *hs[(size_t)r - 1];
      const PartRange& L = lo.range(x);
      require(L.len - L.own_hi == A.first_len, "partition: halo sizes disagree");
      SFEEC_CUDA(cudaMemcpyAsync(lo.vec(x) + L.own_hi, va + A.own_lo, sizeof(double) * (size_t)A.first_len,
                                 cudaMemcpyDeviceToDevice, a.stream));
    }
    if (r < R - 1) {  // my last owned plane -> upper neighbour's halo below
      PartDev& hi = *hs[(size_t)r + 1];
      const PartRange& H = hi.range(x);
      require(H.own_lo == A.last_len, "partition: halo sizes disagree");
      SFEEC_CUDA(cudaMemcpyAsync(hi.vec(x), va + A.own_hi - A.last_len, sizeof(double) * (size_t)A.last_len,
                                 cudaMemcpyDeviceToDevice, a.stream));
    }
  }
}

}  // namespace sfeec_b200

using namespace sfeec_b200;

struct sfeec_part {
  PartDev d;
};


namespace {

void part_ranges(PartDev& d, const int64_t* edge_range, const int64_t* face_range) {
  PartRange* rs[2] = {&d.r1, &d.r2};
  const int64_t* in[2] = {edge_range, face_range};
  for (int k = 0; k < 2; ++k) {
    rs[k]->len = in[k][0];
    rs[k]->own_lo = in[k][1];
    rs[k]->own_hi = in[k][2];
    rs[k]->first_len = in[k][3];
    rs[k]->last_len = in[k][4];
    require(0 <= rs[k]->own_lo && rs[k]->own_lo <= rs[k]->own_hi && rs[k]->own_hi <= rs[k]->len,
            "partition: bad owned range");
  }
}

DevCSR to_dev(const HostCSR& h, cudaStream_t s) {
  DevCSR d;
  d.rows = h.rows;
  d.cols = h.cols;
  d.nnz = (int64_t)h.val.size();
  d.rp.upload(h.row_ptr.data(), h.row_ptr.size(), s);
  d.ci.upload(h.col_idx.data(), std::max<size_t>(1, h.col_idx.size()), s);
  d.val.upload(h.val.data(), std::max<size_t>(1, h.val.size()), s);
  SFEEC_CUDA(cudaStreamSynchronize(s));
  return d;
}

// the local operators split by output rows (rows sent down / up first)
void part_ops(PartDev& d, DevCSR&& q, DevCSR&& c, DevCSR&& ct, DevCSR&& m2) {
  const bool lo = d.rank > 0, hi = d.rank < d.nranks - 1;
  const int64_t lo1 = lo ? d.r1.first_len : 0, hi1 = hi ? d.r1.last_len : 0;
  const int64_t lo2 = lo ? d.r2.first_len : 0, hi2 = hi ? d.r2.last_len : 0;
  d.q.build(std::move(q), lo1, hi1, d.stream);
  d.ct.build(std::move(ct), lo1, hi1, d.stream);
  d.c.build(std::move(c), lo2, hi2, d.stream);
  d.m2.build(std::move(m2), lo2, hi2, d.stream);
}

void part_setup(PartDev& d, double dt, double eps0, double mu0, int rank, int nranks, int device) {
  select_device(device);
  d.device = device;
  d.rank = rank;
  d.nranks = nranks;
  d.dt = dt;
  d.eps0 = eps0;
  d.mu0 = mu0;
  SFEEC_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  SFEEC_CUDA(cudaStreamCreateWithFlags(&d.comm_stream, cudaStreamNonBlocking));
  SFEEC_CUDA(cudaEventCreateWithFlags(&d.ev_bnd, cudaEventDisableTiming));
  SFEEC_CUDA(cudaEventCreateWithFlags(&d.ev_xch, cudaEventDisableTiming));
  const char* ov = std::getenv("SFEEC_PART_OVERLAP");
  d.overlap = !(ov && std::atoi(ov) == 0);
}

// state vectors, reduction scratch and (multi-rank with an id) the NCCL
// communicator -- collective over the ranks
void part_finish(PartDev& d, const void* nccl_id) {
  for (auto* v : {&d.e, &d.t}) {
    v->alloc((size_t)std::max<int64_t>(1, d.r1.len));
    v->zero(d.stream);
  }
  for (auto* v : {&d.b, &d.u}) {
    v->alloc((size_t)std::max<int64_t>(1, d.r2.len));
    v->zero(d.stream);
  }
  d.partials.alloc(kReduceBlocks + 1);
  SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  if (d.nranks > 1 && nccl_id) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    Nccl::get().check(Nccl::get().comm_init_rank(&d.comm, d.nranks, id, d.rank), "ncclCommInitRank");
  }
  // PDL stays off on NCCL slabs (a programmatic launch after the exchange
  // event wait is not verified against a multi-process run); SFEEC_PDL=0
  // turns it off everywhere
  const bool pdl = env_flag("SFEEC_PDL", true) && !d.comm;
  for (SplitOp* o : {&d.q, &d.c, &d.ct, &d.m2})
    for (auto& p : o->part) p.pdl = pdl;
}

// partition.py plane_splits / entity_plane_offsets / slab_system: the rank's
// {len, own_lo, own_hi, first_len, last_len} and {local start, owned lo, hi}
// with an h-plane halo (h = 1 first order, 2 for the S(M1^2) Q of config 4).
// `base` = base vertex of each DOF's entity: its plane is nondecreasing.
void slab_range(const std::vector<int64_t>& base, int n, int rank, int nranks, int h,
                int64_t rng[5], int64_t glob[3]) {
  const int64_t plane = (int64_t)(n + 1) * (n + 1);
  std::vector<int64_t> off((size_t)n + 2);
  for (int k = 0; k <= n + 1; ++k)
    off[(size_t)k] = std::lower_bound(base.begin(), base.end(), (int64_t)k * plane) - base.begin();
  const int p0 = (int)((int64_t)rank * (n + 1) / nranks);
  const int p1 = (int)((int64_t)(rank + 1) * (n + 1) / nranks);
  require(p1 - p0 >= h, "partition: every rank must own at least `halo` vertex planes");
  const int64_t g_lo = off[(size_t)std::max(p0 - h, 0)];
  const int64_t g_hi = off[(size_t)std::min(p1 + h, n + 1)];
  const int64_t o_lo = off[(size_t)p0], o_hi = off[(size_t)p1];
  rng[0] = g_hi - g_lo;
  rng[1] = o_lo - g_lo;
  rng[2] = o_hi - g_lo;
  rng[3] = off[(size_t)p0 + h] - off[(size_t)p0];  // first h owned planes (sent down)
  rng[4] = off[(size_t)p1] - off[(size_t)p1 - h];  // last h owned planes (sent up)
  glob[0] = g_lo;
  glob[1] = o_lo;
  glob[2] = o_hi;
}

}  // namespace

extern "C" {

int sfeec_part_create(const sfeec_csr* q, const sfeec_csr* c, const sfeec_csr* ct,
                      const sfeec_csr* m2, const int64_t* edge_range, const int64_t* face_range,
                      double dt, double eps0, double mu0, int rank, int nranks,
                      const void* nccl_id, int device, sfeec_part** out) {
  return guarded([&] {
    require(out && q && c && ct && m2 && edge_range && face_range, "null argument");
    *out = nullptr;
    csr_validate(*q, "Q");
    csr_validate(*c, "C");
    csr_validate(*ct, "CT");
    csr_validate(*m2, "M2");
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    auto h = std::make_unique<sfeec_part>();
    PartDev& d = h->d;
    part_ranges(d, edge_range, face_range);
    const int64_t o1 = d.r1.own_hi - d.r1.own_lo, o2 = d.r2.own_hi - d.r2.own_lo;
    require(q->rows == o1 && q->cols == d.r1.len, "partition: Q must be owned edges x local edges");
    require(ct->rows == o1 && ct->cols == d.r2.len, "partition: C^T must be owned edges x local faces");
    require(c->rows == o2 && c->cols == d.r1.len, "partition: C must be owned faces x local edges");
    require(m2->rows == o2 && m2->cols == d.r2.len, "partition: M2 must be owned faces x local faces");
    part_setup(d, dt, eps0, mu0, rank, nranks, device);
    part_ops(d, to_dev(csr_from_view(*q), d.stream), to_dev(csr_from_view(*c), d.stream),
             to_dev(csr_from_view(*ct), d.stream), to_dev(csr_from_view(*m2), d.stream));
    part_finish(d, nccl_id);
    *out = h.release();
  });
}

void sfeec_part_destroy(sfeec_part* h) { delete h; }

// owned parts of (b, e)
int sfeec_part_set_state(sfeec_part* h, const double* b, const double* e, double time) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    const int64_t o1 = d.r1.own_hi - d.r1.own_lo, o2 = d.r2.own_hi - d.r2.own_lo;
    if (o1) SFEEC_CUDA(cudaMemcpyAsync(d.e.p + d.r1.own_lo, e, sizeof(double) * (size_t)o1,
                                       cudaMemcpyHostToDevice, d.stream));
    if (o2) SFEEC_CUDA(cudaMemcpyAsync(d.b.p + d.r2.own_lo, b, sizeof(double) * (size_t)o2,
                                       cudaMemcpyHostToDevice, d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    d.time = time;
  });
}

int sfeec_part_get_state(sfeec_part* h, double* b, double* e, double* time) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    const int64_t o1 = d.r1.own_hi - d.r1.own_lo, o2 = d.r2.own_hi - d.r2.own_lo;
    if (e && o1) SFEEC_CUDA(cudaMemcpyAsync(e, d.e.p + d.r1.own_lo, sizeof(double) * (size_t)o1,
                                            cudaMemcpyDeviceToHost, d.stream));
    if (b && o2) SFEEC_CUDA(cudaMemcpyAsync(b, d.b.p + d.r2.own_lo, sizeof(double) * (size_t)o2,
                                            cudaMemcpyDeviceToHost, d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    if (time) *time = d.time;
  });
}

int sfeec_part_advance(sfeec_part* h, int64_t nsteps) {
  return guarded([&] {
    require(h, "null handle");
    require(nsteps >= 0, "advance: nsteps must be >= 0");
    require(h->d.nranks == 1 || h->d.comm || h->d.ipc,
            "multi-rank handle without a transport: use sfeec_part_advance_local");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_part_attach_ipc(sfeec_part* h, const void* ipc_id) {
  return guarded([&] {
    require(h && ipc_id, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.attach_ipc(ipc_id);
  });
}

int sfeec_part_advance_local(sfeec_part** hs, int nranks, int64_t nsteps) {
  return guarded([&] {
    require(hs && nranks >= 1, "null argument");
    std::vector<PartDev*> v;
    for (int r = 0; r < nranks; ++r) {
      require(hs[r] && hs[r]->d.rank == r && hs[r]->d.nranks == nranks, "handles out of order");
      require(hs[r]->d.device == hs[0]->d.device, "local transport needs one device");
      v.push_back(&hs[r]->d);
    }
    SFEEC_CUDA(cudaSetDevice(v[0]->device));
    // one stream for the whole lockstep group
    cudaStream_t s = v[0]->stream;
    auto prog = v[0]->program(nsteps);
    for (auto* d : v) d->launches = 0;
    auto sync_all = [&] {
      for (auto* d : v) SFEEC_CUDA(cudaStreamSynchronize(d->stream));
    };
    // the schedule of the overlapped NCCL path: boundary rows, exchange,
    // interior rows (here the exchange is device copies between phases)
    for (size_t i = 0; i < prog.size(); ++i) {
      const auto& st = prog[i];
      if (st.op <= PartDev::kXu) {
        if (i > 0 && prog[i - 1].op >= PartDev::kQ && PartDev::produced(prog[i - 1].op) == st.op)
          continue;  // exchanged inside the producing kernel's schedule
        sync_all();
        local_exchange(v, st.op);
        sync_all();
      } else if (i + 1 < prog.size() && prog[i + 1].op == PartDev::produced(st.op)) {
        for (auto* d : v) d->kernel_part(st, -1);
        sync_all();
        local_exchange(v, PartDev::produced(st.op));
        sync_all();
        for (auto* d : v) d->kernel_part(st, 2);
      } else {
        for (auto* d : v) d->kernel(st);
      }
    }
    for (auto* d : v) {
      SFEEC_CUDA(cudaStreamSynchronize(d->stream));
      for (int64_t k = 0; k < nsteps; ++k) d->time = d->time + d->dt;
    }
    (void)s;
  });
}

int sfeec_part_energy(sfeec_part* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.exchange_nccl(PartDev::kXe);
    h->d.exchange_nccl(PartDev::kXb);
    *out = h->d.energy();
  });
}

int sfeec_part_energy_local(sfeec_part** hs, int nranks, double* out) {
  return guarded([&] {
    require(hs && out && nranks >= 1, "null argument");
    std::vector<PartDev*> v;
    for (int r = 0; r < nranks; ++r) v.push_back(&hs[r]->d);
    SFEEC_CUDA(cudaSetDevice(v[0]->device));
    for (auto* d : v) SFEEC_CUDA(cudaStreamSynchronize(d->stream));
    local_exchange(v, PartDev::kXe);
    local_exchange(v, PartDev::kXb);
    for (auto* d : v) SFEEC_CUDA(cudaStreamSynchronize(d->stream));
    double e = 0;
    for (auto* d : v) e += d->energy();
    *out = e;
  });
}

int64_t sfeec_part_last_launches(sfeec_part* h) { return h ? h->d.launches : -1; }

}  // extern "C"

namespace {

// Slices a device-built system into rank d.rank's slab and finishes the handle:
// owned rows, local columns; dt <= 0 -> 0.5 x the CFL estimate of the full
// operators (the single-GPU value, bitwise); info as sfeec_part_create_tet.
void part_from_system(PartDev& d, DevCSR& qsym, DevCSR& c, DevCSR& ct, DevCSR& m2, int64_t n1,
                      int64_t n2, const int64_t er[5], const int64_t fr[5], const int64_t eg[3],
                      const int64_t fg[3], double dt, double eps0, double mu0, int device,
                      const void* nccl_id, int64_t* info) {
  part_ranges(d, er, fr);
  DevCSR lq, lct, lc, lm2;
  slice_rows_device(qsym, eg[1], eg[2], eg[0], er[0], lq, d.stream);
  slice_rows_device(ct, eg[1], eg[2], fg[0], fr[0], lct, d.stream);
  slice_rows_device(c, fg[1], fg[2], eg[0], er[0], lc, d.stream);
  slice_rows_device(m2, fg[1], fg[2], fg[0], fr[0], lm2, d.stream);
  if (dt <= 0) {
    DevOperator oq, oc, oct, om2;
    oq.upload_device(std::move(qsym), d.stream);
    om2.upload_device(std::move(m2), d.stream);
    oc.upload_device(std::move(c), d.stream);
    oct.upload_device(std::move(ct), d.stream);
    cudaStream_t hs;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
    std::unique_ptr<sfeec_dev, void (*)(sfeec_dev*)> full(
        make_dev_from_ops(std::move(oq), std::move(oc), std::move(oct), std::move(om2), nullptr,
                          n1, n2, 1.0, eps0, mu0, SFEEC_SPLIT_STRANG, device, SFEEC_NO_CFL_WARN,
                          hs),
        sfeec_dev_destroy);
    double nu = 0;
    require(sfeec_dev_cfl_number(full.get(), &nu) == 0, "partition: CFL estimate failed");
    require(nu > 0, "partition: zero CFL estimate");
    d.dt = 0.5 * 2.0 * 1.0 / nu;
  }
  qsym = DevCSR();
  c = DevCSR();
  ct = DevCSR();
  m2 = DevCSR();
  part_ops(d, std::move(lq), std::move(lc), std::move(lct), std::move(lm2));
  part_finish(d, nccl_id);
  if (info) {
    info[0] = n1;
    info[1] = n2;
    for (int k = 0; k < 5; ++k) {
      info[2 + k] = er[k];
      info[7 + k] = fr[k];
    }
    for (int k = 0; k < 3; ++k) {
      info[12 + k] = eg[k];
      info[15 + k] = fg[k];
    }
    std::memcpy(&info[18], &d.dt, sizeof(double));
  }
}

void check_part_args(int n, int rank, int nranks, sfeec_part** out) {
  require(out != nullptr, "null out");
  *out = nullptr;
  require(n >= 1, "tet mesh: n must be >= 1");
  require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
  require(nranks <= n + 1, "partition: need nranks <= n + 1 vertex planes");
}

}  // namespace

extern "C" {

int sfeec_part_create_tet(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                          int rank, int nranks, const void* nccl_id, int device,
                          sfeec_part** out, int64_t* info) {
  return guarded([&] {
    check_part_args(n, rank, nranks, out);
    auto h = std::make_unique<sfeec_part>();
    PartDev& d = h->d;
    part_setup(d, dt > 0 ? dt : 0.0, eps0, mu0, rank, nranks, device);
    int64_t er[5], fr[5], eg[3], fg[3];
    DevTetSystem sys;
    {
      TetMesh mesh;
      mesh.build(n, jitter, seed);
      slab_range(mesh.edge_v, n, rank, nranks, 1, er, eg);
      slab_range(mesh.face_v, n, rank, nranks, 1, fr, fg);
      build_tet_system_device(mesh, false, sys, d.stream);
    }
    part_from_system(d, sys.qsym, sys.c, sys.ct, sys.m2, sys.n1, sys.n2, er, fr, eg, fg, dt, eps0,
                     mu0, device, nccl_id, info);
    *out = h.release();
  });
}

int sfeec_part_create_p2(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                         int rank, int nranks, const void* nccl_id, int device,
                         sfeec_part** out, int64_t* info) {
  return guarded([&] {
    check_part_args(n, rank, nranks, out);
    auto h = std::make_unique<sfeec_part>();
    PartDev& d = h->d;
    part_setup(d, dt > 0 ? dt : 0.0, eps0, mu0, rank, nranks, device);
    int64_t er[5], fr[5], eg[3], fg[3];
    DevP2System sys;
    {
      TetMesh mesh;
      mesh.build(n, jitter, seed);
      P2Dofs dofs;
      dofs.build(mesh);
      // base vertex of each DOF's entity (k-major: planes nondecreasing)
      std::vector<int64_t> b1((size_t)dofs.n1), b2((size_t)dofs.n2);
      for (int64_t i = 0; i < dofs.n1; ++i) {
        const int64_t e = dofs.ent1[(size_t)i];
        b1[(size_t)i] = (dofs.ks1[(size_t)i] & 1) ? mesh.face_v[(size_t)e] : mesh.edge_v[(size_t)e];
      }
      for (int64_t i = 0; i < dofs.n2; ++i) {
        const int64_t e = dofs.ent2[(size_t)i];
        if (dofs.ks2[(size_t)i] & 1) {
          const int64_t cube = e / 6;
          b2[(size_t)i] = mesh.vid((int)(cube % n), (int)((cube / n) % n), (int)(cube / ((int64_t)n * n)));
        } else {
          b2[(size_t)i] = mesh.face_v[(size_t)e];
        }
      }
      // Q = S(M1^2) SPAI reaches two vertex planes: a two-plane halo
      slab_range(b1, n, rank, nranks, 2, er, eg);
      slab_range(b2, n, rank, nranks, 2, fr, fg);
      build_p2_system_device(mesh, dofs, false, sys, d.stream);
    }
    part_from_system(d, sys.qsym, sys.c, sys.ct, sys.m2, sys.n1, sys.n2, er, fr, eg, fg, dt, eps0,
                     mu0, device, nccl_id, info);
    *out = h.release();
  });
}

int sfeec_part_apply(sfeec_part* h, int which, const double* x_local, double* y_owned) {
  return guarded([&] {
    require(h && x_local && y_owned, "null argument");
    auto& d = h->d;
    SplitOp* ops[4] = {&d.q, &d.c, &d.ct, &d.m2};
    require(which >= 0 && which < 4, "unknown operator");
    SplitOp& a = *ops[which];
    SFEEC_CUDA(cudaSetDevice(d.device));
    DevBuf<double> dx, dy;
    dx.upload(x_local, (size_t)std::max<int64_t>(1, a.cols), d.stream);
    dy.alloc((size_t)std::max<int64_t>(1, a.rows));
    a.launch(-2, dx.p, dy.p, 0.0, false, d.stream);
    SFEEC_CUDA(cudaMemcpyAsync(y_owned, dy.p, sizeof(double) * (size_t)a.rows,
                               cudaMemcpyDeviceToHost, d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  });
}

int sfeec_part_device_ptrs(sfeec_part* h, double** b_local, double** e_local, void** stream) {
  return guarded([&] {
    require(h, "null handle");
    if (b_local) *b_local = h->d.b.p;
    if (e_local) *e_local = h->d.e.p;
    if (stream) *stream = (void*)h->d.stream;
  });
}

int sfeec_part_kernel_timing(sfeec_part* h, int enable, double* ms, int64_t* launches,
                             double* bytes) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    d.collect_timing();
    for (int k = 0; k < 5; ++k) {
      if (ms) ms[k] = d.class_ms[k];
      if (launches) launches[k] = d.class_launches[k];
      if (bytes) bytes[k] = d.op_bytes(k);
      d.class_ms[k] = 0;
      d.class_launches[k] = 0;
    }
    d.timing = enable != 0;
  });
}

// this rank's share of sfeec_dev_step_bytes: 12 nnz(Q) + 12 nnz(M2) +
// 5 (nnz(C) + nnz(C^T)) + 16 (owned edges + owned faces)
double sfeec_part_step_bytes(sfeec_part* h) {
  if (!h) return 0;
  const auto& d = h->d;
  return 12.0 * (double)d.q.nnz + 12.0 * (double)d.m2.nnz +
         (d.c.incidence ? 5.0 : 12.0) * (double)(d.c.nnz + d.ct.nnz) +
         16.0 * (double)(d.r1.own_hi - d.r1.own_lo + d.r2.own_hi - d.r2.own_lo);
}

}  // extern "C"
