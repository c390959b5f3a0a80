// okg_diag.cuh -- diagnostics and the initial state on the device:
//   total_mass            model.hpp:46-48        -> k_mass
//   integrate_double_well assembly.hpp:220-245   -> k_double_well (closed form)
//   energy                model.hpp:56-86        -> host CG (okg_host.cu) over
//                                                   k_divdiag / k_xpby + the operator kernels
//   initial_state         model.hpp:93-114       -> k_cos_ic + the same CG on M
//
// Double well: the reference integrates (1 - u_h^2)^2 with a degree-4 rule,
// which is exact for this quartic of a linear function, so the closed form
//   int_T u^p = |T| d! p! / (d+p)! h_p(u_0..u_d)   (h_p: complete homogeneous
//   symmetric polynomial of the vertex values)
// gives the same integral up to rounding:  int_T (1-u^2)^2 = |T| (1 - 2 c2 h2 + c4 h4)
// with c2 = 2 d!/(d+2)!, c4 = 24 d!/(d+4)!.  Each grid cell (square / cube) is
// owned by its lowest corner, so a slab owns the cells whose lowest plane it owns.
#pragma once
#include "okg_kernels.cuh"

namespace okg {

// u0 = m + cos(2 pi x) cos(2 pi y) cos(2 pi z) / 50 at the mesh vertices (x = i h)
template <int DIM>
__global__ void __launch_bounds__(BS) k_cos_ic(Grid g, double h, double m, double* __restrict__ u) {
  PDL_ENTRY();
  const uint32_t idx = g.lo + blockIdx.x * BS + threadIdx.x;
  if (idx >= g.hi) return;
  const Node<DIM> nd = locate<DIM>(g, idx);
  constexpr double kPi = 3.14159265358979323846;
  const double x = nd.i * h, y = nd.j * h, z = DIM == 3 ? nd.k * h : 0.0;
  u[idx] = m + cos(2.0 * kPi * x) * cos(2.0 * kPi * y) * cos(2.0 * kPi * z) / 50.0;
}

// z = r / diag(A)  (make_jacobi_preconditioner, operator.hpp:53-64)
template <int DIM>
__global__ void __launch_bounds__(BS) k_divdiag(Grid g, Op<DIM> op, const double* __restrict__ r,
                                                double* __restrict__ z) {
  PDL_ENTRY();
  const uint32_t idx = g.lo + blockIdx.x * BS + threadIdx.x;
  if (idx >= g.hi) return;
  const Node<DIM> nd = locate<DIM>(g, idx);
  constexpr int C = Traits<DIM>::CENTER, NO = Traits<DIM>::NOFF;
  const double d = nd.cls == Traits<DIM>::INTERIOR ? op.w[C] : __ldg(op.tab + nd.cls * (NO + 1) + C);
  z[idx] = r[idx] / d;
}

// p = z + beta p  (krylov.hpp:475)
__global__ void __launch_bounds__(BS) k_xpby(const double* __restrict__ z, double beta, double* __restrict__ p,
                                             size_t n) {
  PDL_ENTRY();
  for (size_t i = (size_t)blockIdx.x * BS + threadIdx.x; i < n; i += (size_t)gridDim.x * BS)
    p[i] = z[i] + beta * p[i];
}

__global__ void __launch_bounds__(BS) k_fill(double v, double* __restrict__ x, size_t n) {
  PDL_ENTRY();
  for (size_t i = (size_t)blockIdx.x * BS + threadIdx.x; i < n; i += (size_t)gridDim.x * BS) x[i] = v;
}

// y = x + a * b_load  (axpy(a, ops.b, y) with the per-class load vector)
template <int DIM>
__global__ void __launch_bounds__(BS) k_add_load(Grid g, const double* __restrict__ btab, double a,
                                                 const double* __restrict__ x, double* __restrict__ y) {
  PDL_ENTRY();
  const uint32_t idx = g.lo + blockIdx.x * BS + threadIdx.x;
  if (idx >= g.hi) return;
  const Node<DIM> nd = locate<DIM>(g, idx);
  y[idx] = x[idx] + a * __ldg(btab + nd.cls);
}

// b^T u over the owned vertices
template <int DIM>
__global__ void __launch_bounds__(BS) k_mass(Grid g, const double* __restrict__ btab, const double* __restrict__ u,
                                             Reduce red) {
  PDL_ENTRY();
  double acc[1] = {0.0};
  for (uint32_t idx = g.lo + blockIdx.x * BS + threadIdx.x; idx < g.hi; idx += gridDim.x * BS) {
    const Node<DIM> nd = locate<DIM>(g, idx);
    acc[0] = fma(__ldg(btab + nd.cls), u[idx], acc[0]);
  }
  grid_reduce<1>(acc, red);
}

// complete homogeneous symmetric polynomials h2, h4 of NV values
template <int NV>
__device__ __forceinline__ void h24(const double (&x)[NV], double& h2, double& h4) {
  double H1 = 0.0, H2 = 0.0, H3 = 0.0, H4 = 0.0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {  // h_p(x_1..x_k) = h_p(x_1..x_{k-1}) + x_k h_{p-1}(x_1..x_k)
    H1 = H1 + x[v];
    H2 = fma(x[v], H1, H2);
    H3 = fma(x[v], H2, H3);
    H4 = fma(x[v], H3, H4);
  }
  h2 = H2;
  h4 = H4;
}

// integral of (1 - u_h^2)^2 over the owned cells (cells whose lowest corner plane is owned)
template <int DIM>
__global__ void __launch_bounds__(BS) k_double_well(Grid g, double cell_vol, const double* __restrict__ u,
                                                    Reduce red) {
  PDL_ENTRY();
  const int n = g.n;
  const int c0 = g.ilo, c1 = min(g.ihi, n);  // owned cell planes
  const uint64_t per = DIM == 3 ? (uint64_t)n * n : (uint64_t)n;
  const uint64_t total = c1 > c0 ? (uint64_t)(c1 - c0) * per : 0;
  constexpr double c2 = DIM == 2 ? 1.0 / 6.0 : 1.0 / 10.0;   // 2 d!/(d+2)!
  constexpr double c4 = DIM == 2 ? 1.0 / 15.0 : 1.0 / 35.0;  // 24 d!/(d+4)!
  double acc[1] = {0.0};
  for (uint64_t t = (uint64_t)blockIdx.x * BS + threadIdx.x; t < total; t += (uint64_t)gridDim.x * BS) {
    const int i = c0 + (int)(t / per);
    const uint32_t r = (uint32_t)(t % per);
    double cell = 0.0;
    if (DIM == 2) {
      const int j = (int)r;
      const uint32_t a = (uint32_t)i * g.s + j;
      const double ua = u[a], ub = u[a + g.s], uc = u[a + g.s + 1], ud = u[a + 1];
      // cells {a,b,c}, {a,c,d} (mesh.hpp:106-114)
      const double t1[3] = {ua, ub, uc}, t2[3] = {ua, uc, ud};
      double h2, h4;
      h24<3>(t1, h2, h4);
      cell += 1.0 - 2.0 * c2 * h2 + c4 * h4;
      h24<3>(t2, h2, h4);
      cell += 1.0 - 2.0 * c2 * h2 + c4 * h4;
    } else {
      const int j = (int)(r / (uint32_t)n), k = (int)(r % (uint32_t)n);
      const uint32_t a = (uint32_t)i * g.ps + (uint32_t)j * g.s + k;
      double cv[8];  // corner (dx,dy,dz) -> index dx*4+dy*2+dz
#pragma unroll
      for (int q = 0; q < 8; ++q) cv[q] = u[a + ((q >> 2) & 1) * g.ps + ((q >> 1) & 1) * g.s + (q & 1)];
      // Kuhn paths 0 -> e_p -> e_p + e_q -> (1,1,1), (p,q) over the 6 axis orders (mesh.hpp:124-148)
      const int bit[3] = {4, 2, 1};
      const int perm[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
#pragma unroll
      for (int pp = 0; pp < 6; ++pp) {
        const int q1 = bit[perm[pp][0]], q2 = q1 | bit[perm[pp][1]];
        const double tv[4] = {cv[0], cv[q1], cv[q2], cv[7]};
        double h2, h4;
        h24<4>(tv, h2, h4);
        cell += 1.0 - 2.0 * c2 * h2 + c4 * h4;
      }
    }
    acc[0] = fma(cell, cell_vol, acc[0]);
  }
  grid_reduce<1>(acc, red);
}

}  // namespace okg
