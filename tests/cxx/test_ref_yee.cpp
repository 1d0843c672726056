// The drop-in exercised by the reference's own sources: this program is
// compiled together with the UNMODIFIED /root/reference/proj/src/yee.cpp and
// mesh_cubical.cpp, against include/ (this repo's sparse.hpp, dynamics.hpp,
// core.hpp) ahead of the reference's include tree, and linked to
// libsfeec_b200.so -- the reference's SplitScheme, spmv and friends come from
// this repo, its Yee FDTD and cubical mesh from the reference (tests/cxx/
// Makefile, target test_ref_yee).
//
// A cmd_evolve-style run (reference tools/sfeec_main.cpp:151-215) of the
// lumped-mass cubical system that yee_equivalence_check builds
// (yee.cpp:95-135), with the curl assembled from the reference mesh's signed
// boundary (operators.cpp:29-42: sign * |edge| / |face|; derivative_matrix
// itself needs Eigen, absent here): the device SplitScheme must track the
// reference's FDTD grid (yee_fdtd_step, yee_advance_b) to 1e-12
// (test_yee.cpp:157-163), and write the evolve history.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "sfeec/mesh.hpp"  // the reference's header (PeriodicMesh)
#include "sfeec/yee.hpp"   // the reference's header, over this repo's dynamics.hpp
#include "sfeec_b200.h"

using namespace sfeec;

namespace sfeec {  // mesh_cubical.cpp (reference), declared in mesh.hpp
PeriodicMesh generate_cubical_lattice(int nx, int ny, int nz, double dx, double dy, double dz);
}

static SparseOperator cubical_curl(const PeriodicMesh& m) {
  std::vector<Triplet> tri;
  const int nf = m.n_faces(2);
  for (int f = 0; f < nf; ++f) {
    const auto& xs = m.face_coords[2][(size_t)f];
    const double area = (xs[1] - xs[0]).norm() * (xs[3] - xs[0]).norm();
    for (const auto& [edge, sign] : m.boundary[2][(size_t)f]) {
      const auto& es = m.face_coords[1][(size_t)edge];
      tri.push_back({f, edge, (double)sign * ((es[1] - es[0]).norm() / area)});
    }
  }
  return operator_from_triplets(nf, m.n_faces(1), std::move(tri));
}

int main(int argc, char** argv) {
  if (sfeec_device_count() == 0) {
    std::puts("no GPU: skipped");
    return 0;
  }
  const int nx = 6, ny = 5, nz = 7, steps = argc > 1 ? std::atoi(argv[1]) : 40;
  const double dx = 1.0, dy = 0.8, dz = 1.25, dt = 0.2;
  PeriodicMesh mesh = generate_cubical_lattice(nx, ny, nz, dx, dy, dz);
  SparseOperator c = cubical_curl(mesh);
  const double dv = dx * dy * dz;
  const int n1 = c.cols, n2 = c.rows, nc = nx * ny * nz;
  SplitScheme scheme(SplitKind::Strang, dt, scaled_identity(n1, 1.0 / dv), c,
                     scaled_identity(n2, dv), UnitSystem{}, nullptr, false);

  // yee_equivalence_check's shared random start (yee.cpp:107-121)
  Rng rng(2023);
  YeeGrid grid(nx, ny, nz, dx, dy, dz);
  std::vector<double> e0((size_t)n1), b0((size_t)n2);
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < nc; ++i) e0[(size_t)(a * nc + i)] = grid.e[a][(size_t)i] = rng.uniform(-1, 1);
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < nc; ++i) {
      const double v = rng.uniform(-1, 1);
      grid.b[a][(size_t)i] = v;
      b0[(size_t)(a * nc + i)] = v / dv;
    }

  // the evolve loop: one step at a time through the drop-in step(), with a
  // history row every 10 steps (sfeec_main.cpp:193-215)
  FieldState state = make_state(Formulation::BE, b0, e0);
  std::string history = "step,time,energy,gauss_residual\n";
  auto row = [&](int s) {
    char buf[128];
    std::snprintf(buf, sizeof(buf), "%d,%.17g,%.17g,%.17g\n", s, state.time,
                  scheme.energy(state), 0.0);
    history += buf;
  };
  row(0);
  for (int s = 1; s <= steps; ++s) {
    state = scheme.step(state);
    if (s % 10 == 0 || s == steps) row(s);
  }
  FieldState staggered = state;  // b on the half-step points (yee.cpp:126-127)
  scheme.flow_he(staggered, 0.5 * dt);

  yee_advance_b(grid, 0.5 * dt);  // the reference FDTD (yee.cpp:71-74)
  for (int s = 0; s < steps; ++s) yee_fdtd_step(grid, dt);

  double dev = 0;
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < nc; ++i) {
      dev = std::max(dev, std::abs(state.e[(size_t)(a * nc + i)] - grid.e[a][(size_t)i]));
      dev = std::max(dev, std::abs(dv * staggered.first[(size_t)(a * nc + i)] -
                                   grid.b[a][(size_t)i]));
    }
  // the resident multi-step form gives the same state
  FieldState bulk = scheme.advance(make_state(Formulation::BE, b0, e0), steps);
  double dbulk = 0;
  for (int k = 0; k < n1; ++k) dbulk = std::max(dbulk, std::abs(bulk.e[(size_t)k] - state.e[(size_t)k]));
  std::fputs(history.c_str(), stdout);
  std::printf("max deviation vs reference FDTD after %d steps: %.3e (bulk advance %.3e)\n", steps,
              dev, dbulk);
  const bool ok = dev <= 1e-12 && dbulk <= 1e-12 && std::abs(state.time - steps * dt) < 1e-12;
  std::puts(ok ? "reference yee.cpp over the drop-in: passed" : "FAILED");
  return ok ? 0 : 1;
}
