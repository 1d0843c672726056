// The unstructured SFEEC leapfrog on one B200: device-resident Q_sym, C, C^T,
// M2 (and D), state (first, e) and the step sequence of
//   SplitScheme::flow_he / flow_ha / step   (reference dynamics.cpp:47-90)
// over CSR operators (reference sparse.hpp:14-33, spmv sparse.cpp:96-104).
//
// Two execution modes:
//   production  merged Strang half-kicks, FMA, sub-warp-per-row CSR-vector or
//               sliced-ELL kernels chosen per operator (spmv_kernels.cuh);
//   strict      the reference's three sub-flows, one thread per row in CSR
//               order, separate multiply/add -> bitwise equal to the CPU step.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>

#include "dev_handle.hpp"
#include "device_util.cuh"
#include "lattice.cuh"
#include "spmv_kernels.cuh"

namespace sfeec_b200 {

struct LeapfrogDev {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int kind = SFEEC_SPLIT_STRANG, form = SFEEC_FORM_BE, flags = 0;
  double dt = 0, eps0 = 1, mu0 = 1;
  DevOperator q, c, ct, m2, div;
  HostCSR q_host;  // Q_sym for export when the device keeps no CSR copy
  bool has_div = false;
  int64_t n1 = 0, n2 = 0, n_first = 0;
  DevBuf<double> first, e, t1, t2, t3, partials;
  double time = 0;
  bool warned = false;
  double cfl_cache = -1;
  int64_t launches = 0;
  bool graphs = env_flag("SFEEC_GRAPHS", true);
  // programmatic dependent launches of k_ell / k_sell_pipe (SFEEC_PDL, read
  // once here); the operators carry the flag to launch_spmv
  void set_pdl(bool on) {
    for (DevOperator* a : {&q, &c, &ct, &m2, &div}) a->pdl = on;
  }
  // per-operator launch timing with CUDA events on the launch stream
  // (kernel classes: 0 K-Q, 1 K-C, 2 K-CT, 3 K-M2, 4 other)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, size_t>> ev_used;  // (class, first event index)
  double class_ms[5] = {0, 0, 0, 0, 0};
  int64_t class_launches[5] = {0, 0, 0, 0, 0};
  bool strict() const { return (flags & SFEEC_STRICT) != 0; }

  // Kuhn-lattice layout (lattice.cuh) of a device-assembled first-order tet
  // system: advance() runs the step on the lattice state; every other entry
  // point works on the DOF vectors, gathered back when the lattice is newer
  std::unique_ptr<LatticeOps> lat;
  bool use_lat = false;  // inside advance(): the flows run on the lattice
  bool lat_on() const { return lat && !strict() && form == SFEEC_FORM_BE; }
  void sync_dof() {
    if (lat && lat->newer) {
      lat->gather(first.p, e.p, stream);
      lat->newer = false;
    }
  }
  void dof_changed() {
    if (lat) lat->valid = lat->newer = false;
  }
  double c2() const { return 1.0 / (eps0 * mu0); }

  ~LeapfrogDev() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  int op_class(const DevOperator& a) const {
    return &a == &q ? 0 : &a == &c ? 1 : &a == &ct ? 2 : &a == &m2 ? 3 : 4;
  }
  void tic(const DevOperator& a) { tic_class(op_class(a)); }
  void tic_class(int cls) {
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
    if (!timing) return;
    SFEEC_CUDA(cudaEventRecord(ev_pool[ev_used.back().second + 1], stream));
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

  // y = A x
  void apply(const DevOperator& a, const double* x, double* y) {
    tic(a);
    if (strict())
      launch_spmv_strict(a, x, y, stream);
    else
      launch_spmv(a, x, y, 0.0, false, stream);
    toc();
    ++launches;
  }
  // y += alpha * A x   (strict: y = y + alpha*(A x) with separate rounding)
  void apply_axpy(const DevOperator& a, const double* x, double* y, double alpha) {
    tic(a);
    if (strict())
      launch_spmv_axpy_strict(a, x, y, alpha, stream);
    else
      launch_spmv(a, x, y, alpha, true, stream);
    toc();
    ++launches;
  }

  // dynamics.cpp:47-55
  void flow_he(double h) {
    if (use_lat) {  // t = Q e, b -= h C t on the lattice
      tic_class(0);
      lat->apply_q(stream);
      toc();
      tic_class(1);
      lat->apply_cb(h, stream);
      toc();
      launches += 2;
      return;
    }
    apply(q, e.p, t1.p);
    if (form == SFEEC_FORM_AE) {
      axpy_vec(first.p, t1.p, -h, n1);
    } else {
      apply_axpy(c, t1.p, first.p, -h);
    }
  }
  void axpy_vec(double* y, const double* x, double alpha, int64_t n) {
    launch_axpy(y, x, alpha, n, strict(), stream);
    ++launches;
  }
  // dynamics.cpp:57-67
  void flow_ha(double h) {
    const double f = h * c2();
    if (use_lat) {  // u = M2 b, e += f C^T u on the lattice
      tic_class(3);
      lat->apply_m2(stream);
      toc();
      tic_class(2);
      lat->apply_cte(f, stream);
      toc();
      launches += 2;
      return;
    }
    const double* b = first.p;
    if (form == SFEEC_FORM_AE) {
      apply(c, first.p, t3.p);
      b = t3.p;
    }
    apply(m2, b, t2.p);
    apply_axpy(ct, t2.p, e.p, f);
  }

  void check_cfl_once() {
    if ((flags & SFEEC_NO_CFL_WARN) || warned) return;
    warned = true;
    double nu = cfl_number();
    if (nu > 2.0)
      std::fprintf(stderr,
                   "sfeec: warning: CFL number %.3g > 2; the splitting is likely unstable at "
                   "dt = %.3g\n",
                   nu, dt);
  }

  // CUDA graph of kGraphPairs merged [Ha(dt) He(dt)] pairs, replayed for the
  // bulk of advance(n): small, launch-bound systems (config 1: ~7 us per
  // kernel launched one by one) pay one graph launch per kGraphPairs x 4
  // kernels. Rebuilt when dt changes; off while per-kernel timing is on or
  // with SFEEC_GRAPHS=0 (read once per handle, like SFEEC_PDL: a captured
  // graph and the directly launched kernels always run in the same mode).
  static constexpr int kGraphPairs = 32;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  double graph_dt = -1;
  int64_t graph_kernels = 0;

  bool graphs_on() const { return !timing && graphs; }
  void build_graph() {
    if (graph_exec) {
      cudaGraphExecDestroy(graph_exec);
      graph_exec = nullptr;
    }
    if (!cap_stream) SFEEC_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    cudaStream_t saved = stream;
    const int64_t saved_launches = launches;
    stream = cap_stream;
    SFEEC_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < kGraphPairs; ++k) {
      flow_ha(dt);
      flow_he(dt);
    }
    cudaGraph_t gph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cap_stream, &gph);
    stream = saved;
    graph_kernels = launches - saved_launches;
    launches = saved_launches;
    SFEEC_CUDA(ec);
    const cudaError_t ei = cudaGraphInstantiate(&graph_exec, gph, 0);
    cudaGraphDestroy(gph);
    SFEEC_CUDA(ei);
    graph_dt = dt;
  }
  void pairs(int64_t m) {  // m x [Ha(dt) He(dt)]
    if (m >= kGraphPairs && graphs_on()) {
      if (!graph_exec || graph_dt != dt) build_graph();
      for (; m >= kGraphPairs; m -= kGraphPairs) {
        SFEEC_CUDA(cudaGraphLaunch(graph_exec, stream));
        launches += graph_kernels;
      }
    }
    for (; m > 0; --m) {
      flow_ha(dt);
      flow_he(dt);
    }
  }

  void advance(int64_t n) {
    launches = 0;
    if (n <= 0) return;
    check_cfl_once();
    if (lat_on()) {
      if (!lat->valid) lat->scatter(first.p, e.p, stream);
      lat->valid = true;
      use_lat = true;
      struct Off {
        bool& f;
        ~Off() { f = false; }
      } off{use_lat};
      advance_flows(n);
      lat->newer = true;
    } else {
      advance_flows(n);
    }
    for (int64_t s = 0; s < n; ++s) time = time + dt;  // dynamics.cpp:88, per step
  }

  void advance_flows(int64_t n) {
    if (strict() || kind == SFEEC_SPLIT_LIE_TROTTER || form == SFEEC_FORM_AE) {
      for (int64_t s = 0; s < n; ++s) {
        if (kind == SFEEC_SPLIT_STRANG) {
          flow_he(0.5 * dt);
          flow_ha(dt);
          flow_he(0.5 * dt);
        } else {
          flow_he(dt);
          flow_ha(dt);
        }
      }
    } else {
      // merged Strang: He(h/2) [Ha(h) He(h)]^(n-1) Ha(h) He(h/2)
      flow_he(0.5 * dt);
      pairs(n - 1);
      flow_ha(dt);
      flow_he(0.5 * dt);
    }
  }

  // dynamics.cpp:92-102
  double energy() {
    sync_dof();
    apply(q, e.p, t1.p);
    double he = device_dot(e.p, t1.p, n1, partials.p, stream);
    const double* b = first.p;
    if (form == SFEEC_FORM_AE) {
      apply(c, first.p, t3.p);
      b = t3.p;
    }
    apply(m2, b, t2.p);
    double ha = device_dot(b, t2.p, n2, partials.p, stream);
    return 0.5 * (eps0 * he + ha / mu0);
  }

  // dynamics.cpp:104-112
  double gauss_residual() {
    require(form == SFEEC_FORM_BE, "gauss_residual: (b, e) formulation required");
    if (!has_div) return 0.0;
    sync_dof();
    DevBuf<double> db;
    db.alloc((size_t)div.rows);
    apply(div, first.p, db.p);
    return device_max_abs(db.p, div.rows, partials.p, stream);
  }

  // dynamics.cpp:114-133 (power iteration on Q C^T M2 C, seed 0x5fec5fec)
  double cfl_number() {
    if (cfl_cache >= 0) return cfl_cache;
    std::vector<double> hx((size_t)n1);
    uint64_t st = 0x5fec5fec;
    for (auto& v : hx) {
      uint64_t z = (st += 0x9e3779b97f4a7c15ull);
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      z ^= z >> 31;
      v = -1.0 + 2.0 * ((double)(z >> 11) * 0x1.0p-53);
    }
    DevBuf<double> x, y, w2, w3;
    x.upload(hx.data(), hx.size(), stream);
    y.alloc((size_t)n1);
    w2.alloc((size_t)n2);
    w3.alloc((size_t)n2);
    double lambda = 0;
    for (int it = 0; it < 40; ++it) {
      apply(c, x.p, w2.p);
      apply(m2, w2.p, w3.p);
      apply(ct, w3.p, t1.p);
      apply(q, t1.p, y.p);
      double nrm = std::sqrt(device_dot(y.p, y.p, n1, partials.p, stream));
      if (nrm == 0) break;
      lambda = nrm;
      launch_scale_copy(x.p, y.p, 1.0 / nrm, nrm, n1, stream);
    }
    cfl_cache = dt * std::sqrt(c2() * lambda);
    return cfl_cache;
  }
};

}  // namespace sfeec_b200

using namespace sfeec_b200;

struct sfeec_dev {
  LeapfrogDev d;
};


// Builds a device handle from host operators (Q already symmetric). Shared by
// sfeec_dev_create and the device-assembled tet system (tet_device.cu).
sfeec_dev* make_dev_from_host(HostCSR&& hq, HostCSR&& hc, HostCSR&& hm2, HostCSR* hdiv, double dt,
                              double eps0, double mu0, int split_kind, int formulation,
                              int device, int flags) {
  select_device(device);
  auto h = std::make_unique<sfeec_dev>();
  LeapfrogDev& d = h->d;
  d.device = device;
  SFEEC_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  d.own_stream = true;
  d.kind = split_kind;
  d.form = formulation;
  d.flags = flags;
  d.dt = dt;
  d.eps0 = eps0;
  d.mu0 = mu0;
  const bool strict = (flags & SFEEC_STRICT) != 0;
  d.n1 = hc.cols;
  d.n2 = hc.rows;
  {
    HostCSR hct = csr_transpose(hc);
    d.ct.upload(hct, strict, d.stream);
  }
  d.c.upload(hc, strict, d.stream);
  hc = HostCSR();
  d.m2.upload(hm2, strict, d.stream);
  hm2 = HostCSR();
  d.q.upload(hq, strict, d.stream);
  if (!d.q.has_csr()) d.q_host = std::move(hq);
  if (hdiv) {
    d.div.upload(*hdiv, strict, d.stream);
    d.has_div = true;
  }
  d.n_first = formulation == SFEEC_FORM_BE ? d.n2 : d.n1;
  d.first.alloc((size_t)d.n_first);
  d.first.zero(d.stream);
  d.e.alloc((size_t)d.n1);
  d.e.zero(d.stream);
  d.t1.alloc((size_t)d.n1);
  d.t2.alloc((size_t)std::max<int64_t>(d.n2, 1));
  d.t3.alloc((size_t)std::max<int64_t>(d.n2, 1));
  d.partials.alloc(kReduceBlocks + 1);
  d.set_pdl(env_flag("SFEEC_PDL", true));
  SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  return h.release();
}

// Builds a handle around operators that already live on the device (the
// device-assembled tet system in stencil layout). Production mode only.
sfeec_dev* make_dev_from_ops(DevOperator&& q, DevOperator&& c, DevOperator&& ct, DevOperator&& m2,
                             DevOperator* div, int64_t n1, int64_t n2, double dt, double eps0,
                             double mu0, int split_kind, int device, int flags, cudaStream_t s,
                             std::unique_ptr<LatticeOps> lat) {  // (dev_handle.hpp)
  require(!(flags & SFEEC_STRICT), "strict mode needs CSR operators (use the host builders)");
  select_device(device);
  auto h = std::make_unique<sfeec_dev>();
  LeapfrogDev& d = h->d;
  d.device = device;
  d.stream = s;
  d.own_stream = true;
  d.kind = split_kind;
  d.form = SFEEC_FORM_BE;
  d.flags = flags | SFEEC_Q_IS_SYMMETRIC;
  d.dt = dt;
  d.eps0 = eps0;
  d.mu0 = mu0;
  d.q = std::move(q);
  d.c = std::move(c);
  d.ct = std::move(ct);
  d.m2 = std::move(m2);
  if (div) {
    d.div = std::move(*div);
    d.has_div = true;
  }
  d.n1 = n1;
  d.n2 = n2;
  d.n_first = n2;
  d.lat = std::move(lat);
  d.first.alloc((size_t)n2);
  d.first.zero(d.stream);
  d.e.alloc((size_t)n1);
  d.e.zero(d.stream);
  d.t1.alloc((size_t)n1);
  d.t2.alloc((size_t)std::max<int64_t>(n2, 1));
  d.t3.alloc((size_t)std::max<int64_t>(n2, 1));
  d.partials.alloc(kReduceBlocks + 1);
  d.set_pdl(env_flag("SFEEC_PDL", true));
  SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  return h.release();
}

extern "C" {

int sfeec_dev_create(const sfeec_csr* q, const sfeec_csr* c, const sfeec_csr* m2,
                     const sfeec_csr* div, double dt, double eps0, double mu0, int split_kind,
                     int formulation, int device, int flags, sfeec_dev** out) {
  return guarded([&] {
    require(out != nullptr, "sfeec_dev_create: null out");
    *out = nullptr;
    require(q && c && m2, "sfeec_dev_create: null operator");
    csr_validate(*q, "Q");
    csr_validate(*c, "C");
    csr_validate(*m2, "M2");
    if (div) csr_validate(*div, "div");
    // dynamics.cpp:11-12 then :41-43
    require(q->rows == q->cols, "SplitScheme: Q must be square");
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    require(m2->rows == c->rows && m2->cols == c->rows && q->rows == c->cols,
            "SplitScheme: operator dimensions inconsistent");
    require(!div || div->cols == c->rows, "SplitScheme: divergence dimensions inconsistent");
    require(split_kind == 0 || split_kind == 1, "SplitScheme: unknown split kind");
    require(formulation == 0 || formulation == 1, "SplitScheme: unknown formulation");
    HostCSR hq = csr_from_view(*q);
    if (!(flags & SFEEC_Q_IS_SYMMETRIC)) hq = csr_symmetric_part(hq);
    std::unique_ptr<HostCSR> hd;
    if (div) hd = std::make_unique<HostCSR>(csr_from_view(*div));
    *out = make_dev_from_host(std::move(hq), csr_from_view(*c), csr_from_view(*m2), hd.get(), dt,
                              eps0, mu0, split_kind, formulation, device, flags);
  });
}

void sfeec_dev_destroy(sfeec_dev* h) { delete h; }

int sfeec_dev_set_state(sfeec_dev* h, const double* first, int64_t n_first, const double* e,
                        int64_t n_e, double time) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    require(n_first == d.n_first && n_e == d.n1, "spmv: dimension mismatch");
    SFEEC_CUDA(cudaSetDevice(d.device));
    if (n_first)
      SFEEC_CUDA(cudaMemcpyAsync(d.first.p, first, sizeof(double) * (size_t)n_first,
                                 cudaMemcpyHostToDevice, d.stream));
    if (n_e)
      SFEEC_CUDA(cudaMemcpyAsync(d.e.p, e, sizeof(double) * (size_t)n_e,
                                 cudaMemcpyHostToDevice, d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    d.dof_changed();
    d.time = time;
  });
}

int sfeec_dev_get_state(sfeec_dev* h, double* first, double* e, double* time) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    d.sync_dof();
    if (first && d.n_first)
      SFEEC_CUDA(cudaMemcpyAsync(first, d.first.p, sizeof(double) * (size_t)d.n_first,
                                 cudaMemcpyDeviceToHost, d.stream));
    if (e && d.n1)
      SFEEC_CUDA(cudaMemcpyAsync(e, d.e.p, sizeof(double) * (size_t)d.n1,
                                 cudaMemcpyDeviceToHost, d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    if (time) *time = d.time;
  });
}

int sfeec_dev_advance(sfeec_dev* h, int64_t nsteps) {
  return guarded([&] {
    require(h, "null handle");
    require(nsteps >= 0, "advance: nsteps must be >= 0");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.advance(nsteps);
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_dev_advance_diag(sfeec_dev* h, int64_t nsteps, int64_t diag_every,
                           double* energy_hist, double* gauss_hist) {
  return guarded([&] {
    require(h, "null handle");
    require(nsteps >= 0 && diag_every >= 1, "advance_diag: bad step counts");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    int64_t done = 0, slot = 0;
    while (done < nsteps) {
      int64_t k = std::min(diag_every, nsteps - done);
      d.advance(k);
      done += k;
      if (k == diag_every) {
        if (energy_hist) energy_hist[slot] = d.energy();
        if (gauss_hist) gauss_hist[slot] = d.form == SFEEC_FORM_BE ? d.gauss_residual() : 0.0;
        ++slot;
      }
    }
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  });
}

int sfeec_dev_flow_he(sfeec_dev* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.sync_dof();
    h->d.flow_he(dt);
    h->d.dof_changed();
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_dev_flow_ha(sfeec_dev* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.sync_dof();
    h->d.flow_ha(dt);
    h->d.dof_changed();
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
  });
}

int sfeec_dev_energy(sfeec_dev* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.energy();
  });
}

int sfeec_dev_gauss_residual(sfeec_dev* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.gauss_residual();
  });
}

int sfeec_dev_cfl_number(sfeec_dev* h, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    *out = h->d.cfl_number();
  });
}

int sfeec_dev_q_sym(sfeec_dev* h, int64_t* nnz, int64_t* row_ptr, int32_t* col_idx,
                    double* val) {
  return guarded([&] {
    require(h, "null handle");
    auto& q = h->d.q;
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    if (nnz) *nnz = q.nnz;
    if (q.has_csr()) {
      q.download_csr(row_ptr, col_idx, val, h->d.stream);
    } else {
      const HostCSR& hq = h->d.q_host;
      if (row_ptr) std::memcpy(row_ptr, hq.row_ptr.data(), sizeof(int64_t) * hq.row_ptr.size());
      if (col_idx) std::memcpy(col_idx, hq.col_idx.data(), sizeof(int32_t) * hq.col_idx.size());
      if (val) std::memcpy(val, hq.val.data(), sizeof(double) * hq.val.size());
    }
  });
}

int sfeec_dev_set_stream(sfeec_dev* h, void* s) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
    if (d.own_stream) cudaStreamDestroy(d.stream);
    d.stream = (cudaStream_t)s;
    d.own_stream = false;
  });
}

int sfeec_dev_state_device_ptrs(sfeec_dev* h, double** first, double** e) {
  return guarded([&] {
    require(h, "null handle");
    SFEEC_CUDA(cudaSetDevice(h->d.device));
    h->d.sync_dof();  // the caller may read or write the DOF vectors
    SFEEC_CUDA(cudaStreamSynchronize(h->d.stream));
    h->d.dof_changed();
    if (first) *first = h->d.first.p;
    if (e) *e = h->d.e.p;
  });
}

int64_t sfeec_dev_last_launches(sfeec_dev* h) { return h ? h->d.launches : -1; }

// spmv (sparse.cpp:96-104) on the device: stored-order accumulation, no FMA,
// so y is bitwise the reference's. Stages the operator per call.
int sfeec_spmv(const sfeec_csr* a, const double* x, double* y, int device) {
  return guarded([&] {
    require(a && (a->cols == 0 || x) && (a->rows == 0 || y), "null argument");
    csr_validate(*a, "A");
    select_device(device);
    cudaStream_t s;
    SFEEC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Guard {
      cudaStream_t s;
      ~Guard() { cudaStreamDestroy(s); }
    } guard{s};
    DevOperator op;
    op.upload(csr_from_view(*a), true, s);
    DevBuf<double> dx, dy;
    dx.upload(x, (size_t)a->cols, s);
    dy.alloc((size_t)a->rows);
    launch_spmv_strict(op, dx.p, dy.p, s);
    if (a->rows)
      SFEEC_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * (size_t)a->rows,
                                 cudaMemcpyDeviceToHost, s));
    SFEEC_CUDA(cudaStreamSynchronize(s));
  });
}

// y = A x with one of the handle's resident operators (0 Q_sym, 1 C, 2 C^T,
// 3 M2, 4 D): e.g. B0 = C A for a device-assembled system
int sfeec_dev_apply(sfeec_dev* h, int which, const double* x, double* y) {
  return guarded([&] {
    require(h && x && y, "null argument");
    auto& d = h->d;
    DevOperator* ops[5] = {&d.q, &d.c, &d.ct, &d.m2, &d.div};
    require(which >= 0 && which < 5 && (which != 4 || d.has_div), "unknown operator");
    DevOperator& a = *ops[which];
    SFEEC_CUDA(cudaSetDevice(d.device));
    DevBuf<double> dx, dy;
    dx.upload(x, (size_t)a.cols, d.stream);
    dy.alloc((size_t)a.rows);
    d.apply(a, dx.p, dy.p);
    SFEEC_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * (size_t)a.rows, cudaMemcpyDeviceToHost,
                               d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  });
}

// apply_curl_of_curl (reference operators.cpp:268-290): y = Q C^T M2 C a,
// host buffers; the intermediates stay on the device
int sfeec_dev_curl_curl(sfeec_dev* h, const double* a, double* y) {
  return guarded([&] {
    require(h && a && y, "null argument");
    auto& d = h->d;
    require(d.c.cols == d.n1 && d.m2.rows == d.c.rows, "apply_curl_of_curl: dimension mismatch");
    SFEEC_CUDA(cudaSetDevice(d.device));
    DevBuf<double> da, dw2, dw3, dw1, dy;
    da.upload(a, (size_t)d.n1, d.stream);
    dw2.alloc((size_t)std::max<int64_t>(1, d.n2));
    dw3.alloc((size_t)std::max<int64_t>(1, d.n2));
    dw1.alloc((size_t)d.n1);
    dy.alloc((size_t)d.n1);
    d.apply(d.c, da.p, dw2.p);
    d.apply(d.m2, dw2.p, dw3.p);
    d.apply(d.ct, dw3.p, dw1.p);
    d.apply(d.q, dw1.p, dy.p);
    SFEEC_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * (size_t)d.n1, cudaMemcpyDeviceToHost,
                               d.stream));
    SFEEC_CUDA(cudaStreamSynchronize(d.stream));
  });
}

int sfeec_dev_set_dt(sfeec_dev* h, double dt) {
  return guarded([&] {
    require(h, "null handle");
    require(dt >= 0, "SplitScheme: dt must be >= 0");
    auto& d = h->d;
    if (d.cfl_cache >= 0 && d.dt > 0) d.cfl_cache = d.cfl_cache / d.dt * dt;
    else d.cfl_cache = -1;
    d.dt = dt;
  });
}

int sfeec_dev_kernel_timing(sfeec_dev* h, int enable, double* ms, int64_t* launches,
                            double* bytes) {
  return guarded([&] {
    require(h, "null handle");
    auto& d = h->d;
    SFEEC_CUDA(cudaSetDevice(d.device));
    d.collect_timing();
    const DevOperator* ops[4] = {&d.q, &d.c, &d.ct, &d.m2};
    for (int k = 0; k < 5; ++k) {
      if (ms) ms[k] = d.class_ms[k];
      if (launches) launches[k] = d.class_launches[k];
      d.class_ms[k] = 0;
      d.class_launches[k] = 0;
    }
    // algorithmic bytes per launch of each class (SURVEY.md 8(d) accounting:
    // 12 B per fp64 nonzero, 5 B per incidence entry (int8 sign + int32
    // column), 8 B per vector element read or written)
    if (bytes && d.lat_on()) {  // what the lattice kernels move (lattice.cu)
      bytes[0] = d.lat->bytes_q();
      bytes[1] = d.lat->bytes_cb();
      bytes[2] = d.lat->bytes_cte();
      bytes[3] = d.lat->bytes_m2();
      bytes[4] = 0;
    } else if (bytes) {
      // an incidence C (+-1) streams 5 B per entry, a general one (P2-) 12 B
      const double cb = d.c.layout == DevOperator::kSigned ? 5.0 : 12.0;
      const double ctb = d.ct.layout == DevOperator::kSigned ? 5.0 : 12.0;
      bytes[0] = 12.0 * d.q.nnz + 16.0 * d.n1;   // t = Q e: e gathered once, t written
      bytes[1] = cb * d.c.nnz + 8.0 * d.n1 + 16.0 * d.n2;  // b -= h C t
      bytes[2] = ctb * d.ct.nnz + 8.0 * d.n2 + 16.0 * d.n1; // e += f C^T u
      bytes[3] = 12.0 * d.m2.nnz + 16.0 * d.n2;  // u = M2 b
      bytes[4] = 0;
    }
    d.timing = enable != 0;
  });
}

int sfeec_dev_layout_info(sfeec_dev* h, int which, int64_t* info, double* bytes) {
  return guarded([&] {
    require(h, "null handle");
    require(which >= 0 && which <= 4, "layout_info: which must be 0..4");
    auto& d = h->d;
    const DevOperator* ops[5] = {&d.q, &d.c, &d.ct, &d.m2, &d.div};
    const DevOperator& a = *ops[which];
    if (info) {
      info[0] = (int64_t)a.layout;
      info[1] = 0;  // (column-delta layouts: removed)
      info[2] = a.ell ? 1 : 0;
      info[3] = a.ell ? (a.rows + 31) / 32 : a.n_slices;
      info[4] = 0;
      info[5] = a.sell_entries;
      info[6] = a.nnz;
      info[7] = 0;  // (windowed layout: removed)
      info[8] = 0;
    }
    if (bytes) *bytes = a.stream_bytes();
  });
}

// 12 nnz(Q) + 12 nnz(M2) + 2*5 nnz(C) + 16 (N1 + N2); a
// non-incidence C (P2-, config 4) streams 12 B per entry
double sfeec_dev_step_bytes(sfeec_dev* h) {
  if (!h) return 0;
  auto& d = h->d;
  const double cb = d.c.layout == DevOperator::kSigned ? 5.0 : 12.0;  // +-1 incidence or P2-
  return 12.0 * (double)d.q.nnz + 12.0 * (double)d.m2.nnz + 2.0 * cb * (double)d.c.nnz +
         16.0 * (double)(d.n1 + d.n2);
}

}  // extern "C"
