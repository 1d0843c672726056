// The Fig. 3 accuracy pipeline on the device:
// canonical projection of an analytic 1-form onto the Kuhn-tet Whitney
// space, the curl-of-curl Q C^T M2 C a (sfeec_dev_curl_curl), and the
// relative L^2 error of a discrete 1-form against an analytic one
// (reference operators.cpp:181-257 l2_error; convergence.cpp:107-116).
//
// Analytic forms (the PEC cube's TE cavity family, so the PEC-dropped wall
// edges carry no exact tangential field): kind 0 = A_m = sin(m pi y)
// sin(m pi z) dx, kind 1 = curl curl A_m = 2 (m pi)^2 A_m (div A_m = 0).
//
// Quadrature on each tet: the collapsed (Duffy) product of 4-point
// Gauss-Legendre rules, 64 points, exact to degree 5; the reference's
// l2_error sums cell contributions w_q |w_h(x_q) - f(x_q)|^2 |J| the same way.
// Per-tet sums reduce deterministically (fixed grid, fixed combine order).
#include <cmath>
#include <vector>

#include "device_util.cuh"
#include "p2_mesh.hpp"
#include "tet_mesh.hpp"

namespace sfeec_b200 {
namespace {

constexpr double kGLx[4] = {0.06943184420297371, 0.33000947820757187, 0.6699905217924281,
                            0.9305681557970262};
constexpr double kGLw[4] = {0.17392742256872679, 0.3260725774312732, 0.3260725774312732,
                            0.17392742256872679};
__constant__ double cGLx[4] = {0.06943184420297371, 0.33000947820757187, 0.6699905217924281,
                               0.9305681557970262};
__constant__ double cGLw[4] = {0.17392742256872679, 0.3260725774312732, 0.3260725774312732,
                               0.17392742256872679};
__constant__ int cET[7][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0},
                              {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
__constant__ int cPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__constant__ int cLE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

__host__ __device__ inline void analytic(int kind, int mode, const double x[3], double f[3]) {
  const double k = mode * 3.14159265358979323846;
  const double a = sin(k * x[1]) * sin(k * x[2]);
  f[0] = kind == 1 ? 2.0 * k * k * a : a;
  f[1] = 0.0;
  f[2] = 0.0;
}

constexpr int kRT = 256;

__global__ void __launch_bounds__(kRT) k_l2_error(int n, const double* __restrict__ xyz,
                                                  const int32_t* __restrict__ eid,
                                                  const double* __restrict__ w, int kind,
                                                  int mode, double* __restrict__ partials) {
  __shared__ double se[kRT / 32], sx[kRT / 32];
  const int64_t ntets = 6 * (int64_t)n * n * n;
  const int64_t N = n + 1;
  double e2 = 0.0, x2 = 0.0;
  for (int64_t tet = (int64_t)blockIdx.x * kRT + threadIdx.x; tet < ntets;
       tet += (int64_t)gridDim.x * kRT) {
    const int64_t cube = tet / 6;
    const int p = (int)(tet % 6);
    int c[3] = {(int)(cube % n), (int)((cube / n) % n), (int)(cube / ((int64_t)n * n))};
    int64_t vv[4];
    vv[0] = c[0] + N * (c[1] + N * c[2]);
    for (int s = 0; s < 3; ++s) {
      c[cPerm[p][s]] += 1;
      vv[s + 1] = c[0] + N * (c[1] + N * c[2]);
    }
    double X[4][3];
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 3; ++d) X[a][d] = xyz[3 * vv[a] + d];
    double e[3][3], gl[4][3];
    for (int a = 0; a < 3; ++a)
      for (int d = 0; d < 3; ++d) e[a][d] = X[a + 1][d] - X[0][d];
    double c12[3], c20[3], c01[3];
    c12[0] = e[1][1] * e[2][2] - e[1][2] * e[2][1];
    c12[1] = e[1][2] * e[2][0] - e[1][0] * e[2][2];
    c12[2] = e[1][0] * e[2][1] - e[1][1] * e[2][0];
    c20[0] = e[2][1] * e[0][2] - e[2][2] * e[0][1];
    c20[1] = e[2][2] * e[0][0] - e[2][0] * e[0][2];
    c20[2] = e[2][0] * e[0][1] - e[2][1] * e[0][0];
    c01[0] = e[0][1] * e[1][2] - e[0][2] * e[1][1];
    c01[1] = e[0][2] * e[1][0] - e[0][0] * e[1][2];
    c01[2] = e[0][0] * e[1][1] - e[0][1] * e[1][0];
    const double vol6 = e[0][0] * c12[0] + e[0][1] * c12[1] + e[0][2] * c12[2];
    for (int d = 0; d < 3; ++d) {
      gl[1][d] = c12[d] / vol6;
      gl[2][d] = c20[d] / vol6;
      gl[3][d] = c01[d] / vol6;
      gl[0][d] = -((gl[1][d] + gl[2][d]) + gl[3][d]);
    }
    // coefficients of the 6 local edges (ascending local = ascending global)
    double we[6];
    for (int q = 0; q < 6; ++q) {
      const int a = cLE[q][0], b = cLE[q][1];
      int ca[3], cb[3];
      ca[0] = (int)(vv[a] % N);
      ca[1] = (int)((vv[a] / N) % N);
      ca[2] = (int)(vv[a] / (N * N));
      cb[0] = (int)(vv[b] % N);
      cb[1] = (int)((vv[b] / N) % N);
      cb[2] = (int)(vv[b] / (N * N));
      int t = 0;
      for (int u = 0; u < 7; ++u)
        if (cET[u][0] == cb[0] - ca[0] && cET[u][1] == cb[1] - ca[1] && cET[u][2] == cb[2] - ca[2])
          t = u;
      const int32_t id = eid[7 * vv[a] + t];
      we[q] = id >= 0 ? w[id] : 0.0;  // PEC wall edges carry no DOF
    }
    const double jac = fabs(vol6);  // |det J| of the map from the unit tet
    double te = 0.0, tx = 0.0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        for (int k = 0; k < 4; ++k) {
          const double u = cGLx[i], v = cGLx[j], s = cGLx[k];
          const double l1 = u, l2 = v * (1.0 - u), l3 = s * (1.0 - u) * (1.0 - v);
          const double lam[4] = {1.0 - l1 - l2 - l3, l1, l2, l3};
          const double wq = cGLw[i] * cGLw[j] * cGLw[k] * (1.0 - u) * (1.0 - u) * (1.0 - v);
          double x[3], disc[3] = {0.0, 0.0, 0.0}, f[3];
          for (int d = 0; d < 3; ++d)
            x[d] = lam[0] * X[0][d] + lam[1] * X[1][d] + lam[2] * X[2][d] + lam[3] * X[3][d];
          for (int q = 0; q < 6; ++q) {  // Whitney phi_ab = l_a grad l_b - l_b grad l_a
            const int a = cLE[q][0], b = cLE[q][1];
            for (int d = 0; d < 3; ++d)
              disc[d] += we[q] * (lam[a] * gl[b][d] - lam[b] * gl[a][d]);
          }
          analytic(kind, mode, x, f);
          double d2 = 0.0, f2 = 0.0;
          for (int d = 0; d < 3; ++d) {
            const double r = disc[d] - f[d];
            d2 += r * r;
            f2 += f[d] * f[d];
          }
          te += wq * d2;
          tx += wq * f2;
        }
    e2 += te * jac;
    x2 += tx * jac;
  }
  // fixed-order block reduction
  for (int o = 16; o > 0; o >>= 1) {
    e2 += __shfl_down_sync(0xffffffffu, e2, o);
    x2 += __shfl_down_sync(0xffffffffu, x2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = e2;
    sx[threadIdx.x >> 5] = x2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < kRT / 32; ++k) {
      a += se[k];
      b += sx[k];
    }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
  }
}

}  // namespace
}  // namespace sfeec_b200

using namespace sfeec_b200;

extern "C" {

int sfeec_tetmesh_project_cavity(const sfeec_tetmesh* h, int mode, double* out) {
  return guarded([&] {
    require(h && out, "null argument");
    const TetMesh& m = h->m;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m.n_edges; ++e) {
      int64_t v[2];
      m.edge_vertices(e, v);
      double a = 0.0;
      for (int q = 0; q < 4; ++q) {  // int_e A . dx, 4-point Gauss-Legendre
        double x[3], d[3], f[3];
        for (int c = 0; c < 3; ++c) {
          d[c] = m.xyz[(size_t)(3 * v[1] + c)] - m.xyz[(size_t)(3 * v[0] + c)];
          x[c] = m.xyz[(size_t)(3 * v[0] + c)] + kGLx[q] * d[c];
        }
        analytic(0, mode, x, f);
        a += kGLw[q] * ((f[0] * d[0] + f[1] * d[1]) + f[2] * d[2]);
      }
      out[e] = a;
    }
  });
}

int sfeec_tet_l2_error(const sfeec_tetmesh* h, const double* w, int kind, int mode, int device,
                       double* abs_rel) {
  return guarded([&] {
    require(h && w && abs_rel, "null argument");
    require(kind == 0 || kind == 1, "l2_error: kind must be 0 (A_m) or 1 (curl curl A_m)");
    const TetMesh& m = h->m;
    select_device(device);
    Stream st;
    DevBuf<double> dx, dw, part;
    DevBuf<int32_t> deid;
    dx.upload(m.xyz.data(), m.xyz.size(), st.s);
    deid.upload(m.eid.data(), m.eid.size(), st.s);
    dw.upload(w, (size_t)m.n_edges, st.s);
    const int grid = kReduceBlocks;
    part.alloc(2 * (size_t)grid);
    k_l2_error<<<grid, kRT, 0, st.s>>>(m.n, dx.p, deid.p, dw.p, kind, mode, part.p);
    SFEEC_LAUNCH_CHECK();
    std::vector<double> hp(2 * (size_t)grid);
    SFEEC_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * hp.size(),
                               cudaMemcpyDeviceToHost, st.s));
    SFEEC_CUDA(cudaStreamSynchronize(st.s));
    double se = 0.0, sx = 0.0;
    for (int b = 0; b < grid; ++b) {
      se += hp[2 * (size_t)b];
      sx += hp[2 * (size_t)b + 1];
    }
    require(sx > 0.0, "l2_error: exact form has zero norm");
    abs_rel[0] = std::sqrt(se);
    abs_rel[1] = std::sqrt(se) / std::sqrt(sx);
  });
}

}  // extern "C"
