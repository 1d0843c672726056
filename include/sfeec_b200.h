/*
 * sfeec_b200.h -- the C ABI of the B200-native SFEEC leapfrog.
 *
 * This is the drop-in boundary for the reference's time-stepping hot path.
 * The reference has no FFI: its boundary is the C++ API in
 * /root/reference/proj/include/sfeec/{sparse,dynamics,yee}.hpp, and the
 * C++ classes in include/sfeec/ (same names and signatures) forward to the
 * functions below. Each entry point cites the reference interface it
 * replaces. Conventions:
 *
 *   - return 0 on success; SFEEC_EINVAL (1) where the reference throws
 *     sfeec::InvalidParameter, SFEEC_ECUDA (2) / SFEEC_ENCCL (3) /
 *     SFEEC_ENOMEM (4) where it would throw std::runtime_error. The message
 *     is in sfeec_last_error() (thread-local).
 *   - host buffers are caller-owned and copied; calls are blocking and not
 *     thread-safe per handle (same as the reference's mutable CFL cache).
 *   - no CPU fallback: without a usable sm_100 device every compute entry
 *     point fails with SFEEC_ECUDA.
 */
#ifndef SFEEC_B200_H
#define SFEEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SFEEC_OK = 0,
  SFEEC_EINVAL = 1,
  SFEEC_ECUDA = 2,
  SFEEC_ENCCL = 3,
  SFEEC_ENOMEM = 4
};

/* CSR view of a sfeec::SparseOperator (sparse.hpp:14-33): row_ptr[rows+1],
 * column-sorted col_idx/val, no stored zeros. int64 row pointers so operators
 * above 2^31 nonzeros fit. */
typedef struct {
  int64_t rows, cols;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
} sfeec_csr;

/* CSR owned by the library (returned by the builders); free with sfeec_csr_free. */
typedef struct {
  int64_t rows, cols, nnz;
  int64_t* row_ptr;
  int32_t* col_idx;
  double* val;
} sfeec_csr_owned;

const char* sfeec_last_error(void);
const char* sfeec_version(void);
void sfeec_csr_free(sfeec_csr_owned* m);
/* number of CUDA devices usable by the library (0 without a GPU) */
int sfeec_device_count(void);

/* ---- the unstructured leapfrog (SplitScheme, dynamics.hpp:31-67) ---------- */
typedef struct sfeec_dev sfeec_dev;

enum {
  SFEEC_SPLIT_LIE_TROTTER = 0, /* SplitKind::LieTrotter */
  SFEEC_SPLIT_STRANG = 1       /* SplitKind::Strang */
};
enum {
  SFEEC_FORM_AE = 0, /* Formulation::AE: first = a */
  SFEEC_FORM_BE = 1  /* Formulation::BE: first = b = C a */
};
/* flags */
enum {
  /* q is already symmetric (skip symmetric_part, dynamics.cpp:10-25) */
  SFEEC_Q_IS_SYMMETRIC = 1,
  /* bitwise-reference mode: the three sub-flows of dynamics.cpp:80-83,
   * one thread per CSR row in stored order, separate multiply and add
   * (no FMA) -- reproduces the reference CPU step bit for bit */
  SFEEC_STRICT = 2,
  /* do not run the CFL check on the first step (warn_cfl = false) */
  SFEEC_NO_CFL_WARN = 4
};

/* Replaces SplitScheme::SplitScheme (dynamics.hpp:33-36, dynamics.cpp:29-45):
 * copies Q (symmetrised like symmetric_part unless SFEEC_Q_IS_SYMMETRIC), C,
 * C^T, M2 and the optional divergence D to device `device`. Errors as the
 * reference: dt < 0, non-square Q, or inconsistent dimensions -> EINVAL. */
int sfeec_dev_create(const sfeec_csr* q, const sfeec_csr* c, const sfeec_csr* m2,
                     const sfeec_csr* div /* nullable */, double dt, double eps0, double mu0,
                     int split_kind, int formulation, int device, int flags,
                     sfeec_dev** out);
void sfeec_dev_destroy(sfeec_dev* h);

/* Resident state (FieldState, dynamics.hpp:20-25). n_first = rows of C for
 * BE, cols of C for AE; n_e = cols of C. */
int sfeec_dev_set_state(sfeec_dev* h, const double* first, int64_t n_first, const double* e,
                        int64_t n_e, double time);
int sfeec_dev_get_state(sfeec_dev* h, double* first, double* e, double* time);

/* nsteps x SplitScheme::step (dynamics.cpp:69-90) on the resident state.
 * Production mode merges the adjacent half-kicks of consecutive Strang steps
 * (exact in real arithmetic); SFEEC_STRICT runs the three sub-flows. */
int sfeec_dev_advance(sfeec_dev* h, int64_t nsteps);
/* as advance, recording energy (dynamics.cpp:92-102) and the Gauss residual
 * (dynamics.cpp:104-112; 0 without div) after every diag_every-th step into
 * the nullable arrays (nsteps / diag_every entries). */
int sfeec_dev_advance_diag(sfeec_dev* h, int64_t nsteps, int64_t diag_every,
                           double* energy_hist, double* gauss_hist);
/* exact sub-flows, dynamics.cpp:47-67; do not advance the clock */
int sfeec_dev_flow_he(sfeec_dev* h, double dt);
int sfeec_dev_flow_ha(sfeec_dev* h, double dt);
int sfeec_dev_energy(sfeec_dev* h, double* out);
int sfeec_dev_gauss_residual(sfeec_dev* h, double* out);
/* dynamics.cpp:114-133: 40 power iterations from U(-1,1), seed 0x5fec5fec */
int sfeec_dev_cfl_number(sfeec_dev* h, double* out);
/* Q_sym as stored on the device (nnz query with NULL outputs) */
int sfeec_dev_q_sym(sfeec_dev* h, int64_t* nnz, int64_t* row_ptr, int32_t* col_idx,
                    double* val);

/* y = A x on the device (replaces spmv, sparse.cpp:96-104): stored-order
 * accumulation without FMA, bitwise the reference's result. Stages A per
 * call; the leapfrog keeps its operators resident instead. */
int sfeec_spmv(const sfeec_csr* a, const double* x, double* y, int device);

/* device-resident access for benchmarks / multi-GPU plumbing */
int sfeec_dev_set_stream(sfeec_dev* h, void* cuda_stream);
int sfeec_dev_state_device_ptrs(sfeec_dev* h, double** first, double** e);
/* number of kernel launches issued by the last advance call */
int64_t sfeec_dev_last_launches(sfeec_dev* h);
/* algorithmic HBM bytes of one merged leapfrog step */
double sfeec_dev_step_bytes(sfeec_dev* h);
/* change dt (the scheme is otherwise unchanged; the cached CFL number is
 * rescaled) -- used to set dt = 0.5 * dt_CFL after sfeec_dev_cfl_number */
int sfeec_dev_set_dt(sfeec_dev* h, double dt);
/* Returns (and resets) per-kernel-class device time accumulated since the
 * last call, measured with CUDA events around every launch on the launch
 * stream, then enables/disables timing. Classes: 0 K-Q (Q e), 1 K-Cb
 * (C t), 2 K-CTe (C^T u), 3 K-M2 (M2 b), 4 other. ms[5], launches[5] and
 * bytes[5] (algorithmic bytes per launch) are nullable. */
int sfeec_dev_kernel_timing(sfeec_dev* h, int enable, double* ms, int64_t* launches,
                            double* bytes);

/* ---- structured Yee / lumped-mass SFEEC (yee.hpp:12-37) ------------------ */
typedef struct sfeec_yee sfeec_yee;
enum { SFEEC_BC_PERIODIC = 0, SFEEC_BC_PEC = 1 };

/* Lumped SFEEC on an nx*ny*nz cubical lattice: Q = I/dV, M2 = dV I
 * (lumped_mass, yee.cpp:76-81), C with entries +-1/spacing
 * (operators.cpp:37). bc = PERIODIC reproduces yee_equivalence_check
 * (yee.cpp:83-135); bc = PEC drops boundary edges. precision 8 = fp64,
 * 4 = fp32 fields. DOF numbering: sfeec_yee_dof_counts / DESIGN.md. */
int sfeec_yee_create(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                     double eps0, double mu0, int bc, int precision, int device,
                     sfeec_yee** out);
void sfeec_yee_destroy(sfeec_yee* h);
int sfeec_yee_dof_counts(const sfeec_yee* h, int64_t* n_edges, int64_t* n_faces);
/* (b, e) state in the SFEEC numbering, always passed as fp64 */
int sfeec_yee_set_state(sfeec_yee* h, const double* b, const double* e, double time);
int sfeec_yee_get_state(sfeec_yee* h, double* b, double* e, double* time);
/* nsteps Strang steps (b half-kicks merged across steps) */
int sfeec_yee_advance(sfeec_yee* h, int64_t nsteps);
int sfeec_yee_flow_he(sfeec_yee* h, double dt);
int sfeec_yee_flow_ha(sfeec_yee* h, double dt);
int sfeec_yee_energy(sfeec_yee* h, double* out);
int sfeec_yee_set_stream(sfeec_yee* h, void* cuda_stream);
/* 0: two kernels (e-kick, b-kick); 1: fused single-sweep step with plain
 * loads; 2 (default): fused sweep, persistent, TMA-pipelined (PEC only;
 * periodic lattices always use 0) */
int sfeec_yee_set_variant(sfeec_yee* h, int variant);
int64_t sfeec_yee_last_launches(sfeec_yee* h);
/* Returns (and resets) the accumulated device time of the steady-state step
 * kernels (the fused sweep, or the e/b-kick pair) measured with CUDA events on
 * the launch stream, then enables/disables timing for later advance calls. */
int sfeec_yee_kernel_timing(sfeec_yee* h, int enable, double* ms_total, int64_t* launches);
double sfeec_yee_step_bytes(sfeec_yee* h);

/* ---- multi-GPU: z-slab decomposition of the PEC Yee lattice -------------- */
/* Slab r of nranks owns global planes [r*nz/nranks, (r+1)*nz/nranks) (the last
 * slab also the top wall plane) plus one ghost plane below and above. After
 * every kernel of the step the ghosts are refreshed over NCCL: plane 1 (E, B)
 * goes to rank-1, the top owned B plane to rank+1. The state of
 * a slab is passed in its local numbering; sfeec_yee_slab_dof_map gives the
 * local -> global DOF ids. sfeec_yee_energy on a slab returns its own part. */
int sfeec_nccl_unique_id(void* out128);
/* Self-check of the run-time NCCL binding on one device: a 1-rank
 * communicator, grouped send/recv of n doubles to self; max |error| out. */
int sfeec_nccl_selftest(int device, int64_t n, double* max_err);
int sfeec_yee_create_slab(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                          double eps0, double mu0, int precision, int rank, int nranks,
                          const void* nccl_id /* 128 bytes from rank 0 */, int device,
                          sfeec_yee** out);
/* The same slab with the ghost transport chosen: SFEEC_TRANSPORT_NCCL (comm_id
 * = the 128-byte ncclUniqueId; one GPU per rank) or SFEEC_TRANSPORT_IPC (CUDA
 * IPC on one node, comm_id from sfeec_ipc_unique_id: the neighbours' buffers
 * are mapped and the ghost planes pulled between two host-side barriers, so
 * no kernel waits on another rank and the ranks may share one GPU). */
#define SFEEC_TRANSPORT_NCCL 0
#define SFEEC_TRANSPORT_IPC 1
int sfeec_yee_create_slab_transport(int nx, int ny, int nz, double dx, double dy, double dz,
                                    double dt, double eps0, double mu0, int precision, int rank,
                                    int nranks, int transport, const void* comm_id, int device,
                                    sfeec_yee** out);
int sfeec_yee_slab_dof_counts(int nx, int ny, int nz, int rank, int nranks, int64_t* n_edges,
                              int64_t* n_faces);
int sfeec_yee_slab_dof_map(int nx, int ny, int nz, int rank, int nranks, int64_t* edge_map,
                           int64_t* face_map);
/* All slabs of one lattice on ONE device, ghosts exchanged by device copies:
 * the multi-rank kernels and ghost logic, verifiable with a single GPU.
 * State in the single-domain PEC numbering. */
typedef struct sfeec_yee_group sfeec_yee_group;
int sfeec_yee_group_create(int nx, int ny, int nz, double dx, double dy, double dz, double dt,
                           double eps0, double mu0, int precision, int nranks, int device,
                           sfeec_yee_group** out);
void sfeec_yee_group_destroy(sfeec_yee_group* h);
int sfeec_yee_group_set_variant(sfeec_yee_group* h, int variant);
int sfeec_yee_group_set_state(sfeec_yee_group* h, const double* b, const double* e);
int sfeec_yee_group_get_state(sfeec_yee_group* h, double* b, double* e);
int sfeec_yee_group_advance(sfeec_yee_group* h, int64_t nsteps);
int sfeec_yee_group_energy(sfeec_yee_group* h, double* out);

/* ---- multi-GPU: z-slab partition of the unstructured (tet) leapfrog ------- */
/* With the k-major tet numbering a slab of vertex planes owns a contiguous id
 * range; local vectors cover one halo plane each side. Operators: Q_sym and
 * C^T with owned-edge rows, C and M2 with owned-face rows, columns in the
 * local ranges. edge_range / face_range = {local length, owned lo, owned hi,
 * first owned plane length, last owned plane length}. Built by
 * paper_2301_01753_b200.partition.slab_system. */
typedef struct sfeec_part sfeec_part;
int sfeec_part_create(const sfeec_csr* q_sym, const sfeec_csr* c, const sfeec_csr* ct,
                      const sfeec_csr* m2, const int64_t* edge_range, const int64_t* face_range,
                      double dt, double eps0, double mu0, int rank, int nranks,
                      const void* nccl_id /* NULL: local transport */, int device,
                      sfeec_part** out);
void sfeec_part_destroy(sfeec_part* h);
int sfeec_part_set_state(sfeec_part* h, const double* b_owned, const double* e_owned, double time);
int sfeec_part_get_state(sfeec_part* h, double* b_owned, double* e_owned, double* time);
/* merged-Strang steps with NCCL halo exchange (one process per GPU) */
int sfeec_part_advance(sfeec_part* h, int64_t nsteps);
/* the same program for all ranks' handles on one device, halos copied */
int sfeec_part_advance_local(sfeec_part** hs, int nranks, int64_t nsteps);
/* Gives a multi-rank handle created without an NCCL id (nccl_id = NULL) the
 * host-synchronised CUDA-IPC transport (ipc_id from sfeec_ipc_unique_id, the
 * same bytes on every rank; collective over the ranks of one node, which may
 * share a GPU): sfeec_part_advance / _set_state / _energy then pull the halo
 * rows sfeec_part's NCCL path sends from the neighbours' mapped vectors. */
int sfeec_part_attach_ipc(sfeec_part* h, const void* ipc_id);
int sfeec_part_energy(sfeec_part* h, double* out);  /* this rank's part */
int sfeec_part_energy_local(sfeec_part** hs, int nranks, double* out);
int64_t sfeec_part_last_launches(sfeec_part* h);
/* One rank's slab of the tet system of BASELINE configs 1/3/5, assembled on
 * ITS OWN device (tet_device.cu) and row-sliced there: no host CSR. dt <= 0:
 * dt = 0.5 x the CFL estimate of the FULL operators (the single-GPU
 * tet_device_scheme + configs.cfl_dt value, bitwise). info (nullable, 19):
 * {N1, N2, edge_range[5], face_range[5], edge_global[3] = {local start, owned
 * lo, owned hi}, face_global[3], dt}, dt as the bits of a double. */
int sfeec_part_create_tet(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                          int rank, int nranks, const void* nccl_id, int device,
                          sfeec_part** out, int64_t* info);
/* The same for the config-4 system (P2-, S(M1^2) SPAI, p2_device.cu): its Q
 * reaches two vertex planes, so local vectors carry a two-plane halo and the
 * exchanges move two planes; every rank must own >= 2 vertex planes. */
int sfeec_part_create_p2(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                         int rank, int nranks, const void* nccl_id, int device,
                         sfeec_part** out, int64_t* info);
/* y_owned = A x_local on the device, host buffers; which: 0 Q_sym, 1 C,
 * 2 C^T, 3 M2 (e.g. the BE initial b = C a from a local-range potential) */
int sfeec_part_apply(sfeec_part* h, int which, const double* x_local, double* y_owned);
/* device pointers of the local (halo-extended) b and e and the compute
 * stream, for zero-copy loads / timing (nullable) */
int sfeec_part_device_ptrs(sfeec_part* h, double** b_local, double** e_local, void** stream);
/* per-class launch timing (as sfeec_dev_kernel_timing; classes 0 K-Q, 1 K-Cb,
 * 2 K-CTe, 3 K-M2, 4 halo exchange), arrays of 5, nullable */
int sfeec_part_kernel_timing(sfeec_part* h, int enable, double* ms, int64_t* launches,
                             double* bytes);
/* this rank's algorithmic bytes per step (SURVEY.md 8(d) over its rows) */
double sfeec_part_step_bytes(sfeec_part* h);

/* ---- host operator builders (setup, not timed) ---------------------------- */
/* Lumped Yee operators in the sfeec_yee DOF numbering: C (faces x edges,
 * +-1/spacing), and the divergence D (cells x faces). Replaces
 * generate_cubical_lattice + derivative_matrix for Q1 (mesh_cubical.cpp:15-173,
 * operators.cpp:29-42), extended with PEC. */
/* The consistent Q1- mass matrices of the same lattice (form 1: M1 over the
 * edge DOFs, form 2: M2 over the faces): reference mass_matrix
 * (operators.cpp:133-179) with the Q1 element (form_space.cpp:295-321) and the
 * order-3 cube rule (quadrature.cpp:90-107), duplicates summed in the
 * reference's triplet order -- bitwise the reference on periodic lattices.
 * The cubical SFEEC (non-lumped) system is C, M2 and the SPAI of M1. */
int sfeec_build_yee_mass(int nx, int ny, int nz, double dx, double dy, double dz, int bc,
                         int form, sfeec_csr_owned* m);
int sfeec_build_yee_curl(int nx, int ny, int nz, double dx, double dy, double dz, int bc,
                         sfeec_csr_owned* c, sfeec_csr_owned* div);
/* Jittered Kuhn/Freudenthal tetrahedral mesh of the unit cube (n^3 cubes x 6
 * tets), PEC walls, first-order Whitney forms (BASELINE configs 1, 3, 5). New:
 * the reference meshes are 2-D or periodic cubes; conventions
 * follow mesh_simplicial.cpp:16-38 (ascending-id orientation) and
 * operators.cpp:29-42,133-179. Numbering contract: DESIGN.md. */
typedef struct sfeec_tetmesh sfeec_tetmesh;
int sfeec_tetmesh_create(int n, double jitter, uint64_t seed, sfeec_tetmesh** out);
/* vertex planes [k0, k1] of the n x n x nzg mesh (spacing 1/n): a z-slab
 * with the whole mesh's vertex jitter, entity order and PEC walls (the cut
 * planes are not walls), so its complete rows equal the whole mesh's */
int sfeec_tetmesh_create_slab(int n, int nzg, int k0, int k1, double jitter, uint64_t seed,
                              sfeec_tetmesh** out);
void sfeec_tetmesh_destroy(sfeec_tetmesh* h);
int sfeec_tetmesh_counts(const sfeec_tetmesh* h, int64_t* n_vertices, int64_t* n_edges,
                         int64_t* n_faces, int64_t* n_tets);
/* nullable outputs: xyz[3*nv], edge_vertices[2*N1], face_vertices[3*N2],
 * tet_vertices[4*T] (ascending vertex ids) */
int sfeec_tetmesh_geometry(const sfeec_tetmesh* h, double* xyz, int64_t* edge_vertices,
                           int64_t* face_vertices, int64_t* tet_vertices);
/* which: 0 C (faces x interior edges, +-1), 1 M1 (interior edges), 2 M2
 * (faces), 3 D (tets x faces, +-1) */
/* Gaussian-pulse initial potential on the DOF edges [e0, e1) (configs 3 and 5;
 * DESIGN.md 6.4): a_e = int_e sum_k exp(-|x - x0_k|^2 / (2 sigma^2)) p_k . dx by
 * 3-point Gauss-Legendre; x0, p: 3 * npulses each. Host (OpenMP). */
int sfeec_tetmesh_pulse(const sfeec_tetmesh* h, int npulses, const double* x0, const double* p,
                        double sigma, int64_t e0, int64_t e1, double* out);
/* The Fig. 3 accuracy pipeline (reference operators.cpp:181-257 l2_error,
 * convergence.cpp:107-116) for the PEC cube's TE cavity family: kind 0 =
 * A_m = sin(m pi y) sin(m pi z) dx, kind 1 = curl curl A_m = 2 (m pi)^2 A_m.
 * project_cavity: canonical projection of A_m onto the DOF edges (integral
 * DOFs, 4-point Gauss-Legendre; host). l2_error: abs_rel = {||w_h - f||,
 * ||w_h - f|| / ||f||} over the mesh, w on the DOF edges (host buffer),
 * computed on the device (64-point collapsed Gauss rule per tet). */
int sfeec_tetmesh_project_cavity(const sfeec_tetmesh* h, int mode, double* out);
int sfeec_tet_l2_error(const sfeec_tetmesh* h, const double* w, int kind, int mode, int device,
                       double* abs_rel);
int sfeec_tetmesh_operator(const sfeec_tetmesh* h, int which, sfeec_csr_owned* out);
/* Second-order trimmed forms P2^- on the same mesh (BASELINE config 4; the
 * reference's P2^- is 2-D only, form_space.cpp:41-166 -- the 3-D element
 * follows its DOF conventions). 1-forms: 2 moments per
 * interior edge + 2 per interior face; 2-forms: 3 per face + 3 per tet;
 * 3-forms: 4 per tet. k-major numbering (z-slabs are contiguous ranges). */
int sfeec_tetmesh_p2_counts(const sfeec_tetmesh* h, int64_t* n1, int64_t* n2, int64_t* n3);
/* which: 0 C (N2 x N1), 1 M1, 2 M2, 3 D (N3 x N2) */
int sfeec_tetmesh_p2_operator(const sfeec_tetmesh* h, int which, sfeec_csr_owned* out);
/* per DOF of form 1 or 2: entity id (edge / face for 1-forms, face / tet for
 * 2-forms) and kind | slot << 1 (kind 0 = the lower-dimensional entity) */
int sfeec_tetmesh_p2_dofs(const sfeec_tetmesh* h, int form, int64_t* entity, int8_t* kind_slot);
/* The config-4 system on the device: C, M1, M2 (D) from the host builders,
 * then S(M1^2) with the M1^2 values, the SPAI on S(M1^2) (one CTA per
 * column: blocked Cholesky of the ~300x300 Gram, the 1e-12 trace pivot test
 * of spai.cpp:213-216), Q_sym and C^T on the GPU, wrapped in a leapfrog
 * handle (BE). counts (nullable, 5) = {N1, N2, N3, nnz(Q_sym), fallback
 * columns}. Columns failing the pivot test -> EINVAL (host builder). */
int sfeec_p2_dev_create(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                        int split_kind, int device, int flags, int with_div, sfeec_dev** out,
                        int64_t* counts);
/* the device-built config-4 operators, downloaded (nullable outputs) */
int sfeec_p2_dev_operators(int n, double jitter, uint64_t seed, int device, sfeec_csr_owned* c,
                           sfeec_csr_owned* m2, sfeec_csr_owned* d, sfeec_csr_owned* q_sym,
                           sfeec_csr_owned* ct);
/* the device S(M1^2) SPAI of a caller's symmetric M1 (Q by rows, not
 * symmetrised; spai_approximate_inverse with PatternKind::M1Squared) */
int sfeec_p2_spai_device(const sfeec_csr* m1, int device, sfeec_csr_owned* q, int64_t* fallback);
/* The same first-order S(M1) system assembled ON THE DEVICE (C, D, M1, M2,
 * SPAI, Q_sym; bitwise the host builders' operators) and wrapped in a
 * leapfrog handle (BE formulation). counts = {N1, N2, T} (nullable). The
 * setup path for 128^3 / 256^3 (configs 3, 5). */
/* layout flags for sfeec_tet_dev_create. Default: the sliced / ELL layouts
 * built on the device. HOST_LAYOUT: the same layouts built through the host
 * (the sfeec_dev_create path). STENCIL_LAYOUT (16) is rejected (the
 * table-driven stencil layout was measured slower and removed). By default
 * advance() runs on the Kuhn-lattice form of the system (per-vertex
 * coefficient arrays, no index streams) for n >= 48 and on the
 * sliced / ELL kernels below (faster for the small, launch-bound meshes);
 * NO_LATTICE / LATTICE force either. TABLE_LATTICE runs the step on the
 * table-driven lattice instead (table_lattice.cuh: stencils read off the
 * assembled operators at build time, n >= 4) -- the layout of the
 * second-order system (sfeec_p2_dev_create: on by default for n >= 12,
 * LATTICE forces it from n >= 6, NO_LATTICE keeps the sliced kernels),
 * available here as a cross-check of the compile-time-unrolled kernels. */
enum {
  SFEEC_TET_HOST_LAYOUT = 8,
  SFEEC_TET_STENCIL_LAYOUT = 16,
  SFEEC_TET_NO_LATTICE = 32,
  SFEEC_TET_LATTICE = 64,
  SFEEC_TET_TABLE_LATTICE = 128
};
int sfeec_tet_dev_create(int n, double jitter, uint64_t seed, double dt, double eps0, double mu0,
                         int split_kind, int device, int flags, int with_div, sfeec_dev** out,
                         int64_t* counts);
/* device-assembled operators, downloaded (parity tests); nullable outputs */
int sfeec_tet_dev_operators(int n, double jitter, uint64_t seed, int device, sfeec_csr_owned* c,
                            sfeec_csr_owned* m2, sfeec_csr_owned* d, sfeec_csr_owned* q_sym,
                            sfeec_csr_owned* ct);
/* device layout of a resident operator (0 Q_sym, 1 C, 2 C^T, 3 M2, 4 D):
 * info[9] = {layout (0 CSR, 1 signed, 2 fp64 values), 0, ELL, slices (ELL:
 * 32-row groups), 0, stored entries incl. padding, nnz, 0, 0}; *bytes = what one application streams
 * from the operator arrays in this layout (the algorithmic count of SURVEY.md
 * 8(d) stays 12 B / nonzero whatever the layout). No reference counterpart. */
int sfeec_dev_layout_info(sfeec_dev* h, int which, int64_t* info, double* bytes);
/* y = A x with a resident operator of the handle: 0 Q_sym, 1 C, 2 C^T, 3 M2, 4 D */
int sfeec_dev_apply(sfeec_dev* h, int which, const double* x, double* y);
/* apply_curl_of_curl (operators.cpp:268-290): y = Q_sym C^T M2 C a with the
 * resident operators (the curl-curl of the Fig. 3 accuracy study); host a[N1],
 * y[N1] */
int sfeec_dev_curl_curl(sfeec_dev* h, const double* a, double* y);
/* make_pattern (spai.cpp:31-72): kind 0 diagonal, 1 S(M1), 2 S(M1^2); the
 * pattern is returned as a CSR with unit values */
int sfeec_make_pattern(const sfeec_csr* m, int kind, sfeec_csr_owned* out);
/* spai_approximate_inverse (spai.cpp:127-286) on pattern `kind`; report[4] =
 * {frobenius_residual, avg_nnz_per_row, max_column_residual, fallback_columns} */
int sfeec_spai(const sfeec_csr* m, int kind, sfeec_csr_owned* q, double* report);
/* operator_from_triplets (sparse.cpp:20-61), int64-safe */
int sfeec_csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int32_t* r,
                            const int32_t* c, const double* v, sfeec_csr_owned* out);
/* symmetric_part (dynamics.cpp:10-25) and transpose (sparse.cpp:75-94) */
int sfeec_csr_symmetric_part(const sfeec_csr* q, sfeec_csr_owned* out);
int sfeec_csr_transpose(const sfeec_csr* a, sfeec_csr_owned* out);

/* ---- multi-rank Kuhn-lattice leapfrog (lattice_slab.cu) ----
 * One process per GPU; rank r owns the whole-mesh vertex planes [P_r, P_{r+1})
 * (P_r = floor(r (nzg + 1) / R)) of the n x n x nzg mesh (spacing 1/n; nzg = n
 * for the unit cube of configs 3 / 5, nzg = n R for a weak-scaling stack of
 * n^3 blocks) and assembles only its slab (planes [P_r - 4, P_{r+1} + 4]) on
 * its device. Ghost planes move after each of the four kernels; the plane
 * sums of energy and CFL are combined in plane order, so every rank count
 * gives bitwise the single-rank numbers. transport: 0 NCCL (comm_id = an
 * ncclUniqueId), 1 CUDA IPC with host-side synchronisation (same node; ranks
 * may share one GPU; comm_id from sfeec_ipc_unique_id). State vectors hold
 * the rank's owned DOFs in whole-mesh order: edges [info[2], info[2] +
 * info[0]), faces [info[3], info[3] + info[1]). info[10] = {owned edges,
 * owned faces, first owned edge / face (whole-mesh id), P_r, P_{r+1}, first /
 * last assembled plane, first owned edge / face (slab-local id)}.
 * energy, cfl_number and curl are collective. No reference counterpart (the
 * reference has no distributed code). */
typedef struct sfeec_lslab sfeec_lslab;
int sfeec_ipc_unique_id(void* out128);
/* Host-only self-check of the IPC transport's shared segment and barrier
 * (ipc_group.hpp): `rounds` barrier-separated all-sums of (rank + round) over
 * the ranks' slots; *out = the last sum. No CUDA call. */
int sfeec_ipc_group_selftest(const void* id128, int rank, int nranks, int rounds, double* out);
int sfeec_lslab_create(int n, int nzg, double jitter, uint64_t seed, double dt, double eps0,
                       double mu0, int split_kind, int rank, int nranks, int transport,
                       const void* comm_id, int device, sfeec_lslab** out, int64_t* info);
void sfeec_lslab_destroy(sfeec_lslab* h);
int sfeec_lslab_set_state(sfeec_lslab* h, const double* b, const double* e, double time);
int sfeec_lslab_get_state(sfeec_lslab* h, double* b, double* e, double* time);
int sfeec_lslab_advance(sfeec_lslab* h, int64_t nsteps);
int sfeec_lslab_energy(sfeec_lslab* h, double* out);
int sfeec_lslab_cfl_number(sfeec_lslab* h, double* out);
int sfeec_lslab_set_dt(sfeec_lslab* h, double dt);
int sfeec_lslab_curl(sfeec_lslab* h, const double* a, double* b);
int sfeec_lslab_stream(sfeec_lslab* h, void** stream);
int64_t sfeec_lslab_last_launches(sfeec_lslab* h);
double sfeec_lslab_step_bytes(sfeec_lslab* h);
/* per-kernel device time (ms[4], launches[4], bytes[4] per launch: 0 K-Q,
 * 1 K-Cb, 2 K-CTe, 3 K-M2) since the last call, then (dis)arm the timing */
int sfeec_lslab_kernel_timing(sfeec_lslab* h, int enable, double* ms, int64_t* launches,
                              double* bytes);

#ifdef __cplusplus
}
#endif
#endif
