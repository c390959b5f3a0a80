// okg_tail.cuh -- the bottom of the V-cycle in ONE single-CTA launch.
//
// Below ~5000 vertices a multigrid level is pure launch latency: six kernels
// per level per V-cycle, each a few microseconds of ramp-up for a few
// microseconds of work, times 20 V-cycles per GMRES iteration.  Here one CTA
// runs mg_cycle (multigrid.hpp:97-117) on every level from `lt` down to the
// coarsest -- smoothing, residual, restriction, the coarsest solve with the
// explicit inverse, prolongation and post-smoothing -- separated by
// __syncthreads() only.  The level vectors are tiny and stay L1/L2 resident.
#pragma once
#include "okg_common.cuh"
#include "okg_tiled.cuh"

namespace okg {

constexpr int TAIL_NT = 1024;
constexpr int TAIL_MAXL = 8;

template <int DIM>
struct TailLevel {
  Grid g;
  Op<DIM> op;
  double *b, *x, *ea, *eb, *res;
};

template <int DIM>
struct TailArgs {
  TailLevel<DIM> L[TAIL_MAXL];
  int nl;            // levels in the tail (last one is the coarsest)
  int pre, post;
  double omega;
  const double* rhs;  // rhs of the first tail level
  double* out;        // result of the first tail level
  const double* Ainv;
  int nc;
};

// generic per-vertex row of a constant operator with a staged-value functor
template <int DIM, class SV>
__device__ __forceinline__ double tail_row(const TailLevel<DIM>& L, uint32_t idx, const Node<DIM>& nd,
                                           double& own, SV&& sv) {
  constexpr int NO = Traits<DIM>::NOFF;
  const double* w = L.op.tab + nd.cls * (NO + 1);
  double As = 0.0;
  const int fj = DIM == 3 ? nd.j : 0, fk = DIM == 3 ? nd.k : nd.j;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const int ni = nd.i + off_comp(DIM, o, 0);
    const int nj = DIM == 3 ? fj + off_comp(DIM, o, 1) : 0;
    const int nk = fk + off_comp(DIM, o, DIM - 1);
    if (ni < 0 || ni > L.g.n || nk < 0 || nk > L.g.n || (DIM == 3 && (nj < 0 || nj > L.g.n))) continue;
    const double v = sv((uint32_t)((int)idx + L.g.off[o]), ni, nj, nk);
    if (o == Traits<DIM>::CENTER) own = v;
    const double wo = w[o];
    if (wo != 0.0) As = fma(wo, v, As);
  }
  return As;
}

template <int DIM>
__global__ void __launch_bounds__(TAIL_NT, 1) k_vcycle_tail(const TailArgs<DIM> Ap) {
  PDL_ENTRY();
  constexpr int NO = Traits<DIM>::NOFF;
  const int tid = threadIdx.x;
  __shared__ TailArgs<DIM> A;
  __shared__ double* cur[TAIL_MAXL];
  __shared__ double* oth[TAIL_MAXL];
  {  // word-wise copy of the level descriptors into shared memory
    static_assert(sizeof(TailArgs<DIM>) % 8 == 0, "TailArgs must be 8-byte sized");
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&Ap);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&A);
    for (int w = tid; w < (int)(sizeof(TailArgs<DIM>) / 8); w += TAIL_NT) dst[w] = src[w];
  }
  __syncthreads();
  const double om = A.omega;
  // down sweep: cur[l] holds the pre-smoothed iterate of level l
  for (int l = 0; l < A.nl - 1; ++l) {
    const TailLevel<DIM>& L = A.L[l];
    const double* rhs = l == 0 ? A.rhs : L.b;
    double* c = L.ea;
    double* o = L.eb;
    if (A.pre == 0) {
      for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) c[i] = 0.0;
    } else {
      // sweep 1 from zero: e = w D^-1 b
      for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) {
        const Node<DIM> nd = locate<DIM>(L.g, i);
        c[i] = om * L.op.tab[nd.cls * (NO + 1) + NO] * rhs[i];
      }
      for (int s = 1; s < A.pre; ++s) {
        __syncthreads();
        for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) {
          const Node<DIM> nd = locate<DIM>(L.g, i);
          double own = 0.0;
          const double As = tail_row<DIM>(L, i, nd, own, [&](uint32_t v, int, int, int) { return c[v]; });
          o[i] = fma(om * L.op.tab[nd.cls * (NO + 1) + NO], rhs[i] - As, own);
        }
        double* t = c;
        c = o;
        o = t;
      }
    }
    __syncthreads();
    // residual
    for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) {
      const Node<DIM> nd = locate<DIM>(L.g, i);
      double own = 0.0;
      const double As = tail_row<DIM>(L, i, nd, own, [&](uint32_t v, int, int, int) { return c[v]; });
      L.res[i] = rhs[i] - As;
    }
    __syncthreads();
    // restriction to level l+1 (spmv_transpose order, sparse.hpp:159-169)
    const TailLevel<DIM>& C = A.L[l + 1];
    for (uint32_t i = tid; i < C.g.N; i += TAIL_NT) {
      const Node<DIM> nc = locate<DIM>(C.g, i);
      const uint32_t F = DIM == 3 ? (uint32_t)(2 * nc.i) * L.g.ps + (uint32_t)(2 * nc.j) * L.g.s + 2 * nc.k
                                  : (uint32_t)(2 * nc.i) * L.g.s + 2 * nc.j;
      double s = 0.0;
      const int ci = nc.i, cj = DIM == 3 ? nc.j : 0, ck = DIM == 3 ? nc.k : nc.j;
#pragma unroll
      for (int o2 = 0; o2 < NO; ++o2) {
        const int fi = 2 * ci + off_comp(DIM, o2, 0);
        const int fj = DIM == 3 ? 2 * cj + off_comp(DIM, o2, 1) : 0;
        const int fk = 2 * ck + off_comp(DIM, o2, DIM - 1);
        if (fi < 0 || fi > L.g.n || fk < 0 || fk > L.g.n || (DIM == 3 && (fj < 0 || fj > L.g.n))) continue;
        s += (o2 == Traits<DIM>::CENTER ? 1.0 : 0.5) * L.res[(int)F + L.g.off[o2]];
      }
      C.b[i] = s;
    }
    if (tid == 0) {
      cur[l] = c;
      oth[l] = o;
    }
    __syncthreads();
  }
  // coarsest: x = A_c^{-1} b (warp per row)
  {
    const TailLevel<DIM>& C = A.L[A.nl - 1];
    const double* rhs = A.nl == 1 ? A.rhs : C.b;
    double* dst = A.nl == 1 ? A.out : C.x;
    const int lane = tid & 31, warp = tid >> 5;
    for (int row = warp; row < A.nc; row += TAIL_NT / 32) {
      double s = 0.0;
      const double* a = A.Ainv + (size_t)row * A.nc;
      for (int j = lane; j < A.nc; j += 32) s = fma(__ldg(a + j), rhs[j], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) dst[row] = s;
    }
    __syncthreads();
  }
  // up sweep: prolongate + post-smooth
  for (int l = A.nl - 2; l >= 0; --l) {
    const TailLevel<DIM>& L = A.L[l];
    const TailLevel<DIM>& C = A.L[l + 1];
    const double* rhs = l == 0 ? A.rhs : L.b;
    double* dst = l == 0 ? A.out : L.x;
    double* c = cur[l];
    double* o = oth[l];
    for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) {
      const Node<DIM> nd = locate<DIM>(L.g, i);
      const int fj = DIM == 3 ? nd.j : 0, fk = DIM == 3 ? nd.k : nd.j;
      c[i] = c[i] + prolong_at<DIM>(C.g, C.x, nd.i, fj, fk);
    }
    for (int s = 0; s < A.post; ++s) {
      __syncthreads();
      double* to = (s == A.post - 1) ? dst : o;
      for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) {
        const Node<DIM> nd = locate<DIM>(L.g, i);
        double own = 0.0;
        const double As = tail_row<DIM>(L, i, nd, own, [&](uint32_t v, int, int, int) { return c[v]; });
        to[i] = fma(om * L.op.tab[nd.cls * (NO + 1) + NO], rhs[i] - As, own);
      }
      double* t = c;
      c = o;
      o = t;
    }
    if (A.post == 0)
      for (uint32_t i = tid; i < L.g.N; i += TAIL_NT) dst[i] = c[i];
    __syncthreads();
  }
}

}  // namespace okg
