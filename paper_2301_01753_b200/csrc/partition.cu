// Partitioned unstructured leapfrog: one z-slab of a tet mesh per GPU.
//
// The tet DOF numbering is k-major (host_tet.cpp), so the entities whose base
// vertex lies in a range of z-planes are a contiguous id range. Rank r owns
// planes [P_r, P_{r+1}); its local vectors cover planes [P_r - 1, P_{r+1}]
// (one halo plane each side = the one-layer halo of SURVEY.md 8(e)), and its
// local operators are the owned rows with columns shifted into that range:
//   Q_sym, C^T : rows = owned edges      C, M2 : rows = owned faces
// The merged Strang step needs four halo refreshes (b before K-M2, u before
// K-CTe, e before K-Q, t before K-Cb); each sends the first owned plane down
// and the last owned plane up (contiguous ranges, no packing) with
// ncclSend/ncclRecv on the compute stream, or -- to verify the multi-rank
// path on one GPU -- with device copies between handles advanced in lockstep.
#include <cstring>
#include <memory>
#include <vector>

#include "device_util.cuh"
#include "nccl_loader.hpp"
#include "spmv_kernels.cuh"

namespace sfeec_b200 {

struct PartRange {
  int64_t len = 0, own_lo = 0, own_hi = 0, first_len = 0, last_len = 0;
};

struct PartDev {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  double dt = 0, eps0 = 1, mu0 = 1;
  PartRange r1, r2;  // edges, faces
  DevOperator q, c, ct, m2;
  DevBuf<double> e, t, b, u, partials;
  double time = 0;
  int64_t launches = 0;

  ~PartDev() {
    if (comm) Nccl::get().comm_destroy(comm);
    if (stream) cudaStreamDestroy(stream);
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

  void kernel(const Step& s) {
    switch (s.op) {
      case kQ: launch_spmv(q, e.p, t.p + r1.own_lo, 0.0, false, stream); break;
      case kCb: launch_spmv(c, t.p, b.p + r2.own_lo, s.alpha, true, stream); break;
      case kM2: launch_spmv(m2, b.p, u.p + r2.own_lo, 0.0, false, stream); break;
      case kCTe: launch_spmv(ct, u.p, e.p + r1.own_lo, s.alpha, true, stream); break;
      default: return;
    }
    ++launches;
  }

  double* vec(Op x) { return x == kXe ? e.p : x == kXt ? t.p : x == kXb ? b.p : u.p; }
  const PartRange& range(Op x) const { return (x == kXe || x == kXt) ? r1 : r2; }

  void exchange_nccl(Op x) {
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

  void run(const Step& s) {
    if (s.op <= kXu)
      exchange_nccl(s.op);
    else
      kernel(s);
  }

  void advance(int64_t n) {
    launches = 0;
    for (const auto& s : program(n)) run(s);
    for (int64_t k = 0; k < n; ++k) time = time + dt;
  }

  // this rank's part of 0.5 (eps0 e^T Q e + b^T M2 b / mu0); halos of e and b
  // must be current (the callers refresh them)
  double energy() {
    launch_spmv(q, e.p, t.p + r1.own_lo, 0.0, false, stream);
    launch_spmv(m2, b.p, u.p + r2.own_lo, 0.0, false, stream);
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
    const int64_t o1 = d.r1.own_hi - d.r1.own_lo, o2 = d.r2.own_hi - d.r2.own_lo;
    require(q->rows == o1 && q->cols == d.r1.len, "partition: Q must be owned edges x local edges");
    require(ct->rows == o1 && ct->cols == d.r2.len, "partition: C^T must be owned edges x local faces");
    require(c->rows == o2 && c->cols == d.r1.len, "partition: C must be owned faces x local edges");
    require(m2->rows == o2 && m2->cols == d.r2.len, "partition: M2 must be owned faces x local faces");
    select_device(device);
    d.device = device;
    d.rank = rank;
    d.nranks = nranks;
    d.dt = dt;
    d.eps0 = eps0;
    d.mu0 = mu0;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    d.q.upload(csr_from_view(*q), false, d.stream);
    d.c.upload(csr_from_view(*c), false, d.stream);
    d.ct.upload(csr_from_view(*ct), false, d.stream);
    d.m2.upload(csr_from_view(*m2), false, d.stream);
    for (auto* v : {&d.e, &d.t}) {
      v->alloc((size_t)std::max<int64_t>(1, d.r1.len));
      v->zero(d.stream);
    }
    for (auto* v : {&d.b, &d.u}) {
      v->alloc((size_t)std::max<int64_t>(1, d.r2.len));
      v->zero(d.stream);
    }
    d.partials.alloc(kReduceBlocks + 1);
    if (nranks > 1 && nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      Nccl::get().check(Nccl::get().comm_init_rank(&d.comm, nranks, id, rank), "ncclCommInitRank");
    }
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
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
    require(h->d.nranks == 1 || h->d.comm, "multi-rank handle without NCCL: use sfeec_part_advance_local");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
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
    for (const auto& st : prog) {
      if (st.op <= PartDev::kXu) {
        for (auto* d : v) SFEEC_CUDA(cudaStreamSynchronize(d->stream));
        local_exchange(v, st.op);
        for (auto* d : v) SFEEC_CUDA(cudaStreamSynchronize(d->stream));
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
