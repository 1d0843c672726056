// Constructors of the leapfrog handle (leapfrog.cu) shared by the setup paths
// (tet_device.cu, p2_device.cu, partition.cu). Global namespace, like the
// opaque sfeec_dev of the C ABI.
#pragma once
#include <memory>

#include "lattice.cuh"
#include "spmv_kernels.cuh"

struct sfeec_dev;

// a handle around operators already on the device (production mode only);
// `lat`: the Kuhn-lattice form of the same system, used by advance()
sfeec_dev* make_dev_from_ops(sfeec_b200::DevOperator&& q, sfeec_b200::DevOperator&& c,
                             sfeec_b200::DevOperator&& ct, sfeec_b200::DevOperator&& m2,
                             sfeec_b200::DevOperator* div, int64_t n1, int64_t n2, double dt,
                             double eps0, double mu0, int split_kind, int device, int flags,
                             cudaStream_t s, std::unique_ptr<sfeec_b200::LatticeOps> lat = nullptr);
// a handle from host CSR operators (Q already symmetric)
sfeec_dev* make_dev_from_host(sfeec_b200::HostCSR&& hq, sfeec_b200::HostCSR&& hc,
                              sfeec_b200::HostCSR&& hm2, sfeec_b200::HostCSR* hdiv, double dt,
                              double eps0, double mu0, int split_kind, int formulation,
                              int device, int flags);
