// okg_ssor.cuh -- SSOR sweeps on the device (cheby_precond = "ssor",
// krylov.hpp:322-418, precond.hpp:156-161):
//   forward   (D/w + L) x = r      x_i = (r_i - sum_{j<i} a_ij x_j) w / d_i
//   backward  (D/w + U) x = r      x_i = (r_i - sum_{j>i} a_ij x_j) w / d_i
// Both are sequential in the natural order, but on the structured mesh every
// lower (upper) neighbour of a vertex lies on a smaller (larger) hyperplane
// l = i + j (+ k): the hyperplanes are visited in order and the vertices of one
// hyperplane are independent.  One thread-block cluster (one thread per mesh
// column, cluster barrier between hyperplanes -- ~0.2 us, and the acquire makes
// the previous hyperplane's global writes visible) runs a whole sweep.
// Per vertex the arithmetic is the reference's: the CSR row in column order,
// s -= a_ij x_j with separate rounding (no FMA contraction), x = (s w) / d.
// Results are bit-identical to the reference's SsorSweeps.
#pragma once
#include "okg_common.cuh"

namespace okg {

constexpr int SSOR_NT = 1024;

__device__ __forceinline__ int cdig_c(int v, int n) { return v == 0 ? 0 : (v == n ? 2 : 1); }

template <int DIM, bool FWD>
__global__ void __launch_bounds__(SSOR_NT, 1) k_ssor_sweep(Grid g, Op<DIM> op, double omega,
                                                           const double* __restrict__ r, double* x) {
  PDL_ENTRY();
  constexpr int NO = Traits<DIM>::NOFF, C = Traits<DIM>::CENTER;
  unsigned rank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int n = g.n, s = g.s;
  const int ncol = DIM == 3 ? s * s : s;  // columns (i, j) in 3D, rows i in 2D
  const int T = (int)csize * SSOR_NT, t0 = (int)rank * SSOR_NT + threadIdx.x;
  const int L = DIM * n;  // hyperplanes 0 .. L
  for (int step = 0; step <= L; ++step) {
    const int l = FWD ? step : L - step;
    for (int col = t0; col < ncol; col += T) {
      const int i = DIM == 3 ? col / s : col;
      const int j = DIM == 3 ? col - i * s : 0;
      const int kk = l - i - j;  // fastest coordinate of the vertex on this hyperplane
      if (kk < 0 || kk > n) continue;
      const int cls = DIM == 3 ? cdig_c(i, n) * 9 + cdig_c(j, n) * 3 + cdig_c(kk, n) : cdig_c(i, n) * 3 + cdig_c(kk, n);
      const uint32_t v = DIM == 3 ? ((uint32_t)i * s + j) * s + kk : (uint32_t)i * s + kk;
      const double* w = op.tab + cls * (NO + 1);
      double acc = r[v];
      if (FWD) {
#pragma unroll
        for (int o = 0; o < C; ++o) {  // lower neighbours, ascending column
          const int ni = i + off_comp(DIM, o, 0);
          const int nj = DIM == 3 ? j + off_comp(DIM, o, 1) : 0;
          const int nk = kk + off_comp(DIM, o, DIM - 1);
          if (ni < 0 || nk < 0 || (DIM == 3 && nj < 0) || nk > n || (DIM == 3 && nj > n)) continue;
          acc = __dsub_rn(acc, __dmul_rn(__ldg(w + o), x[(int)v + g.off[o]]));
        }
      } else {
#pragma unroll
        for (int o = NO - 1; o > C; --o) {  // upper neighbours, descending column
          const int ni = i + off_comp(DIM, o, 0);
          const int nj = DIM == 3 ? j + off_comp(DIM, o, 1) : 0;
          const int nk = kk + off_comp(DIM, o, DIM - 1);
          if (ni > n || nk > n || (DIM == 3 && nj > n) || nk < 0 || (DIM == 3 && nj < 0)) continue;
          acc = __dsub_rn(acc, __dmul_rn(__ldg(w + o), x[(int)v + g.off[o]]));
        }
      }
      x[v] = __ddiv_rn(__dmul_rn(acc, omega), __ldg(w + C));
    }
    if (csize > 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
  }
}

// y = x * (a * f(d_i)), f(d) = d (SSOR middle factor, g = (2-w)/w) or sqrt(d)
// (spectrum probe E^T / E scaling), d = the row's diagonal
template <int DIM, bool SQRT>
__global__ void __launch_bounds__(256) k_diag_scale(Grid g, Op<DIM> op, double a, const double* x, double* y) {
  PDL_ENTRY();
  const uint32_t idx = g.lo + blockIdx.x * 256 + threadIdx.x;
  if (idx >= g.hi) return;
  const Node<DIM> nd = locate<DIM>(g, idx);
  const double d = __ldg(op.tab + nd.cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::CENTER);
  const double f = SQRT ? sqrt(d) : d;
  y[idx] = x[idx] * __dmul_rn(a, f);
}

// d = c1 d + c2 z with separate roundings (krylov.hpp:197-198)
__global__ void __launch_bounds__(256) k_lincomb(double c1, double* __restrict__ d, double c2,
                                                 const double* __restrict__ z, size_t n) {
  PDL_ENTRY();
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256)
    d[i] = __dadd_rn(__dmul_rn(c1, d[i]), __dmul_rn(c2, z[i]));
}

}  // namespace okg
