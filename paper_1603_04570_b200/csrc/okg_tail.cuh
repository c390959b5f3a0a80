// okg_tail.cuh -- the bottom of the V-cycle in ONE launch, in shared memory.
//
// Below ~5000 vertices a multigrid level is pure latency: every level costs
// two launches per V-cycle (k_mg_down / k_mg_up, ~7-10 us each, mostly
// dependent global-memory round trips), the coarsest a third, and there are 20
// V-cycles per GMRES iteration.  Here one CTA of 1024 threads runs mg_cycle
// V(2,2) (multigrid.hpp:97-117) on every level from the tail's first level
// (3D n <= 16, 2D n <= 64) down to the coarsest with all level vectors in
// shared memory (<= 160 KB) and compile-time level sizes, phases separated by
// __syncthreads only.
//
// The dense coarsest solve (x = A_c^{-1} b, up to 289^2 doubles in 2D) is the
// one piece worth spreading over SMs: the kernel is launched as a thread-block
// cluster of C CTAs that all run the same smem V-cycle redundantly, each
// computes 1/C of the coarse rows and reads the others' rows through
// distributed shared memory (DSMEM); only rank 0 writes the result.
//
// Every phase uses the unfused kernels' per-vertex expressions in the same
// order (k_pre2, k_op<EPI_RESID / EPI_JACOBI*>, k_restrict, k_prolong_add,
// k_coarse_solve): results are bit-identical to the multi-launch path.
#pragma once
#include <cooperative_groups.h>

#include "okg_common.cuh"

namespace okg {

constexpr int TAIL_NT = 1024;
constexpr int TAIL_MAXL = 6;

template <int DIM>
struct TailArgs {
  const double* tabs;   // [TAIL_MAXL][NCLS][NOFF+1] level tables + [NCLS][NOFF] restriction weights
  int nl;               // tail levels; the last one is the coarsest
  double omega;
  const double* rhs;    // rhs of the tail's first level (global)
  double* out;          // its V-cycle result (global)
  const double* Ainv;   // dense inverse of the coarsest operator
  int nc;
};

__device__ __forceinline__ void cpa8(double* dst, const double* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory"); }

// largest first-level n the tail supports (shared-memory budget)
template <int DIM>
constexpr int tail_max_n() { return DIM == 3 ? 16 : 64; }

template <int DIM, int n>
struct TL {
  static constexpr int s = n + 1;
  static constexpr int ps = DIM == 3 ? s * s : s;
  static constexpr int N = DIM == 3 ? s * s * s : s * s;
  static constexpr int G = ps + s + 1;  // guard band >= the largest |stencil offset|
  template <int o>
  static constexpr int off() {
    return DIM == 3 ? off_comp(3, o, 0) * ps + off_comp(3, o, 1) * s + off_comp(3, o, 2)
                    : off_comp(2, o, 0) * s + off_comp(2, o, 1);
  }
  static __device__ __forceinline__ int cd(int x) { return x == 0 ? 0 : (x == n ? 2 : 1); }
};

// Shared-memory layout.  Level Q of the tail (n = N0 >> Q) holds K arrays of N
// doubles (level 0: P, A, B; deeper: b, P, A, B, x), each surrounded by zeroed
// guard bands of G doubles: [G][X0][G][X1]...[G].  A stencil tap of a boundary
// vertex whose neighbour does not exist has weight 0 in the class table and
// reads a finite value (guard or another vertex), so every vertex runs the same
// branch-free loop.  Tables: per level [NCLS][NOFF+1] weights (+1/diag), and one
// [NCLS][NOFF] restriction table (1, 1/2 or 0).
template <int DIM, int n, int Q>
struct TLev {
  using T = TL<DIM, n>;
  static constexpr int K = Q == 0 ? 3 : 5;
  static constexpr int SIZE = T::G + K * (T::N + T::G);
  static __device__ __forceinline__ double* arr(double* base, int a) { return base + T::G + a * (T::N + T::G); }
};
template <int DIM, int n, int Q>
constexpr int tail_levels_doubles() {
  if constexpr (n >= 2) return TLev<DIM, n, Q>::SIZE + tail_levels_doubles<DIM, n / 2, Q + 1>();
  else return TLev<DIM, n, Q>::SIZE;
}
template <int DIM>
constexpr int tail_table_doubles() {
  return TAIL_MAXL * Traits<DIM>::NCLS * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NCLS * Traits<DIM>::NOFF;
}
template <int DIM, int N0>
constexpr int tail_smem_doubles() {
  return tail_table_doubles<DIM>() + tail_levels_doubles<DIM, N0, 0>();
}

// zero the guard bands of every level
template <int DIM, int n, int Q>
__device__ __forceinline__ void tail_zero_guards(double* base) {
  using L = TLev<DIM, n, Q>;
  using T = TL<DIM, n>;
  for (int a = 0; a <= L::K; ++a) {
    double* g = base + a * (T::N + T::G);
    for (int t = threadIdx.x; t < T::G; t += TAIL_NT) g[t] = 0.0;
  }
  if constexpr (n >= 2) tail_zero_guards<DIM, n / 2, Q + 1>(base + L::SIZE);
}

// f(v, i, j, k, cls) for every vertex of a level with compile-time n (2D: j is the fast
// coordinate, k = 0, matching Node<2>)
template <int DIM, int n, class F>
__device__ __forceinline__ void tail_each(F&& f) {
  using T = TL<DIM, n>;
  for (int v = threadIdx.x; v < T::N; v += TAIL_NT) {
    int i, j, k;
    if (DIM == 3) {
      i = v / T::ps;
      const int r = v - i * T::ps;
      j = r / T::s;
      k = r - j * T::s;
    } else {
      i = v / T::s;
      j = v - i * T::s;
      k = 0;
    }
    const int cls = DIM == 3 ? T::cd(i) * 9 + T::cd(j) * 3 + T::cd(k) : T::cd(i) * 3 + T::cd(j);
    f(v, i, j, k, cls);
  }
}

// A x at vertex v: all NOFF slots with the class row (missing neighbours weigh 0 --
// the unfused kernels skip those slots, which differs at most in the sign of a zero)
template <int DIM, int n>
__device__ __forceinline__ double tail_row(const double* W, const double* x, int v) {
  using T = TL<DIM, n>;
  double s = 0.0;
  static_for<Traits<DIM>::NOFF>([&](auto o) { s = fma(W[o], x[v + T::template off<o>()], s); });
  return s;
}

// one level of the tail: V(2,2) from zero with rhs `rb` (loader), result into `out`
// (shared memory, or global for level 0 on cluster rank 0)
template <int DIM, int N0, int Q, class RB>
__device__ void tail_level(const TailArgs<DIM>& A, const double* tabs, double* base, const double* ainv, RB&& rb,
                           double* out, bool write_out) {
  constexpr int n = N0 >> Q;
  constexpr int NO = Traits<DIM>::NOFF;
  using T = TL<DIM, n>;
  using L = TLev<DIM, n, Q>;
  const double* Wq = tabs + Q * Traits<DIM>::NCLS * (NO + 1);  // [cls][NOFF+1]
  const double om = A.omega;
  double* P = L::arr(base, Q == 0 ? 0 : 1);
  double* Ab = L::arr(base, Q == 0 ? 1 : 2);
  double* Bb = L::arr(base, Q == 0 ? 2 : 3);
  if (Q == A.nl - 1) {
    // ---- coarsest: x = A_c^{-1} b (k_coarse_solve), rows split over the cluster ----
    namespace cg = cooperative_groups;
    const unsigned C = cg::this_cluster().num_blocks(), rk = cg::this_cluster().block_rank();
    const int nc = A.nc;
    const int r0 = (int)(rk * nc / C), r1 = (int)((rk + 1) * nc / C);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int row = r0 + warp; row < r1; row += TAIL_NT / 32) {
      double s = 0.0;
      const double* a = ainv + (size_t)(row - r0) * nc;
      for (int j = lane; j < nc; j += 32) s = fma(a[j], rb(j), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) out[row] = s;
    }
    if (C > 1) {  // gather the other CTAs' rows through DSMEM
      cg::this_cluster().sync();
      for (unsigned o = 0; o < C; ++o) {
        if (o == rk) continue;
        const double* ro = cg::this_cluster().map_shared_rank(out, o);
        for (int row = (int)(o * nc / C) + (int)threadIdx.x; row < (int)((o + 1) * nc / C); row += TAIL_NT)
          out[row] = ro[row];
      }
    }
    __syncthreads();
    return;
  }
  if constexpr (n >= 2) {
    constexpr int nc = n / 2;
    using TC = TL<DIM, nc>;
    using LC = TLev<DIM, nc, Q + 1>;
    double* cbase = base + L::SIZE;
    double* bc = LC::arr(cbase, 0);
    double* xc = LC::arr(cbase, 4);
    // ---- pre-smoothing from zero (k_pre2): e1 = w D^-1 b -> B, then e2 -> P ----
    tail_each<DIM, n>([&](int v, int, int, int, int cls) {
      Bb[v] = __dmul_rn(om * Wq[cls * (NO + 1) + NO], rb(v));
    });
    __syncthreads();
    tail_each<DIM, n>([&](int v, int, int, int, int cls) {
      const double* W = Wq + cls * (NO + 1);
      const double s = tail_row<DIM, n>(W, Bb, v);
      P[v] = fma(om * W[NO], rb(v) - s, Bb[v]);
    });
    __syncthreads();
    // ---- residual (k_op<EPI_RESID>) -> A ----
    tail_each<DIM, n>([&](int v, int, int, int, int cls) {
      Ab[v] = rb(v) - tail_row<DIM, n>(Wq + cls * (NO + 1), P, v);
    });
    __syncthreads();
    // ---- restriction (k_restrict) -> b of the coarser level ----
    const double* RW = tabs + TAIL_MAXL * Traits<DIM>::NCLS * (NO + 1);  // [cls][NOFF]
    tail_each<DIM, nc>([&](int G, int i, int j, int k, int ccls) {
      const int F = DIM == 3 ? (2 * i) * T::ps + (2 * j) * T::s + 2 * k : (2 * i) * T::s + 2 * j;
      const double* R = RW + ccls * NO;
      double s = 0.0;
      static_for<NO>([&](auto o) { s += R[o] * Ab[F + T::template off<o>()]; });
      bc[G] = s;
    });
    __syncthreads();
    // ---- coarse-grid correction ----
    tail_level<DIM, N0, Q + 1>(A, tabs, cbase, ainv, [&](int u) { return bc[u]; }, xc, true);
    // ---- P += P_l x_c (k_prolong_add) ----
    tail_each<DIM, n>([&](int v, int i, int j, int k, int) {
      const int li = i >> 1, lj = j >> 1, lk = k >> 1;
      const int hi = (i + 1) >> 1, hj = (j + 1) >> 1, hk = (k + 1) >> 1;
      const int lo = DIM == 3 ? li * TC::ps + lj * TC::s + lk : li * TC::s + lj;
      const int up = DIM == 3 ? hi * TC::ps + hj * TC::s + hk : hi * TC::s + hj;
      double t;
      if (lo == up) t = xc[lo];
      else t = fma(0.5, xc[up], 0.5 * xc[lo]);
      P[v] = P[v] + t;
    });
    __syncthreads();
    // ---- two post-sweeps (k_op<EPI_JACOBI>, then EPI_JACOBI_SET) ----
    tail_each<DIM, n>([&](int v, int, int, int, int cls) {
      const double* W = Wq + cls * (NO + 1);
      Bb[v] = fma(om * W[NO], rb(v) - tail_row<DIM, n>(W, P, v), P[v]);
    });
    __syncthreads();
    if (write_out)
      tail_each<DIM, n>([&](int v, int, int, int, int cls) {
        const double* W = Wq + cls * (NO + 1);
        out[v] = fma(om * W[NO], rb(v) - tail_row<DIM, n>(W, Bb, v), Bb[v]);
      });
    __syncthreads();
  }
}

// rows of A_c^{-1} a cluster rank computes
__host__ __device__ inline int tail_rows(int nc, int C, int rk) { return (rk + 1) * nc / C - rk * nc / C; }

template <int DIM, int N0>
__global__ void __launch_bounds__(TAIL_NT, 1) k_vcycle_tail(const TailArgs<DIM> A) {
  extern __shared__ double sm[];
  namespace cg = cooperative_groups;
  const unsigned C = cg::this_cluster().num_blocks(), rk = cg::this_cluster().block_rank();
  constexpr int NTAB = tail_table_doubles<DIM>();
  constexpr int N0V = TL<DIM, N0>::N;
  double* tabs = sm;
  double* rhs0 = tabs + NTAB;
  double* base = rhs0 + N0V;
  double* ainv = base + tail_levels_doubles<DIM, N0, 0>();
  // constants first -- tables (group 0) and this rank's rows of A_c^{-1} (group 1) do
  // not depend on the predecessor kernel, so they are issued before
  // griddepcontrol.wait and overlap its tail; then the rhs (group 2)
  for (int e = threadIdx.x; e < NTAB; e += TAIL_NT) cpa8(tabs + e, A.tabs + e);
  cpa_commit();
  {
    const int r0 = (int)(rk * A.nc / C);
    const int cnt = tail_rows(A.nc, (int)C, (int)rk) * A.nc;
    const double* src = A.Ainv + (size_t)r0 * A.nc;
    for (int e = threadIdx.x; e < cnt; e += TAIL_NT) cpa8(ainv + e, src + e);
  }
  cpa_commit();
  tail_zero_guards<DIM, N0, 0>(base);
  PDL_ENTRY();
  for (int e = threadIdx.x; e < N0V; e += TAIL_NT) cpa8(rhs0 + e, A.rhs + e);
  cpa_commit();
  cpa_wait<0>();  // (the coarse inverse is small enough to wait for here)
  __syncthreads();
  tail_level<DIM, N0, 0>(A, tabs, base, ainv, [&](int u) { return rhs0[u]; }, A.out, rk == 0);
  // no CTA may exit while another still reads its shared memory (coarse rows)
  if (C > 1) cg::this_cluster().sync();
}

}  // namespace okg
