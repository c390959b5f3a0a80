// okg_rr.cuh -- residual and restriction of a tiled multigrid level in ONE launch:
//   b_c = P^T (b - A x)          (multigrid.hpp:106-109, sparse.hpp:159-169)
// The separate kernels write the fine residual r (8 B/vertex), read it again in
// k_restrict, and cost one more dependent launch per level and V-cycle -- at 128^3
// the three k_restrict launches are 10 % of a V-cycle, most of it launch latency.
//
// A CTA owns a block of CI x CJ x CK coarse vertices (one thread each).  The coarse
// vertex (I,J,K) sits on fine vertex (2I,2J,2K) and P^T gathers the fine residual of
// its 1-ring, so the CTA needs r on the (2CI+1) x (2CJ+1) x (2CK+1) fine vertices
// around its block and x one vertex further out:
//   1. the x region is staged in shared memory (cp.async, zero-fill outside the box);
//   2. r = b - A x of every fine vertex of the r region goes to shared memory --
//      interior vertices with the weights in the parameter bank, boundary vertices
//      with their class row, each row summed slot by slot exactly like
//      k_tiled<T_RESID> / boundary_vertex, so r has the same bits;
//   3. every thread sums its coarse vertex's row of P^T in k_restrict's order.
// The r planes/rows/columns shared by neighbouring blocks are computed by both (9/8 per
// axis); nothing is accumulated across CTAs, so the sum order is fixed and b_c is
// bit-identical to k_restrict of the separately computed residual.
#pragma once
#include "okg_tiled.cuh"

namespace okg {

template <int DIM>
struct RRCfg;
template <>
struct RRCfg<3> {
  static constexpr int CI = 4, CJ = 4, CK = 16;
};
template <>
struct RRCfg<2> {
  static constexpr int CI = 4, CJ = 1, CK = 64;
};

template <int DIM>
struct RRGeom {
  using C = RRCfg<DIM>;
  static constexpr int NT = C::CI * C::CJ * C::CK;
  // r region (fine vertices 2*I0-1 ...) and x region (one further out)
  static constexpr int RI = 2 * C::CI + 1, RJ = DIM == 3 ? 2 * C::CJ + 1 : 1, RK = 2 * C::CK + 1;
  static constexpr int XI = RI + 2, XJ = DIM == 3 ? RJ + 2 : 1, XK = RK + 2;
  static constexpr int RSZ = RI * RJ * RK, XSZ = XI * XJ * XK;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(RSZ + XSZ);
};

// number of coarse blocks per axis / in total
template <int DIM>
__host__ __device__ inline int rr_blocks_axis(int nc, int per) {
  return (nc + 1 + per - 1) / per;
}
template <int DIM>
inline unsigned rr_grid(const Grid& gc) {
  using C = RRCfg<DIM>;
  const unsigned bi = rr_blocks_axis<DIM>(gc.n, C::CI), bk = rr_blocks_axis<DIM>(gc.n, C::CK);
  const unsigned bj = DIM == 3 ? rr_blocks_axis<DIM>(gc.n, C::CJ) : 1u;
  return bi * bj * bk;
}

template <int DIM>
__global__ void __launch_bounds__(RRGeom<DIM>::NT) k_resid_restrict(Grid gf, Grid gc, Op<DIM> op,
                                                                    const double* __restrict__ x,
                                                                    const double* __restrict__ b,
                                                                    double* __restrict__ bc) {
  pdl_wait();
  using C = RRCfg<DIM>;
  using G = RRGeom<DIM>;
  constexpr int NO = Traits<DIM>::NOFF;
  extern __shared__ double rr_sm[];
  double* xs = rr_sm;           // [XI][XJ][XK]
  double* rs = rr_sm + G::XSZ;  // [RI][RJ][RK]
  const int tid = threadIdx.x;
  // block -> first coarse vertex (I0, J0, K0)
  int blk = (int)blockIdx.x;
  const int bk = rr_blocks_axis<DIM>(gc.n, C::CK);
  const int bj = DIM == 3 ? rr_blocks_axis<DIM>(gc.n, C::CJ) : 1;
  const int K0 = (blk % bk) * C::CK;
  blk /= bk;
  const int J0 = DIM == 3 ? (blk % bj) * C::CJ : 0;
  const int I0 = (DIM == 3 ? blk / bj : blk) * C::CI;
  // fine coordinates of the x region's origin
  const int xi0 = 2 * I0 - 2, xj0 = DIM == 3 ? 2 * J0 - 2 : 0, xk0 = 2 * K0 - 2;
  // ---- 1. stage x (zero outside the box)
  for (int e = tid; e < G::XSZ; e += G::NT) {
    const int hk = e % G::XK, t = e / G::XK;
    const int hj = DIM == 3 ? t % G::XJ : 0, hi = DIM == 3 ? t / G::XJ : t;
    const int fi = xi0 + hi, fj = xj0 + hj, fk = xk0 + hk;
    const bool in = fi >= 0 && fi <= gf.n && fk >= 0 && fk <= gf.n && (DIM == 2 || (fj >= 0 && fj <= gf.n));
    const uint32_t lin = DIM == 3 ? (uint32_t)fi * gf.ps + (uint32_t)fj * gf.s + fk : (uint32_t)fi * gf.s + fk;
    cp_async8(xs + e, x + (in ? lin : 0u), in);
  }
  cp_commit();
  // the rhs of this thread's r-region vertices, in flight together with the x tile
  constexpr int M = (G::RSZ + G::NT - 1) / G::NT;
  double bv[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int e = tid + m * G::NT;
    const int pk = e % G::RK, t = e / G::RK;
    const int pj = DIM == 3 ? t % G::RJ : 0, pi = DIM == 3 ? t / G::RJ : t;
    const int fi = xi0 + 1 + pi, fj = DIM == 3 ? xj0 + 1 + pj : 0, fk = xk0 + 1 + pk;
    const bool in = e < G::RSZ && fi >= 0 && fi <= gf.n && fk >= 0 && fk <= gf.n && (DIM == 2 || (fj >= 0 && fj <= gf.n));
    const uint32_t lin = DIM == 3 ? (uint32_t)fi * gf.ps + (uint32_t)fj * gf.s + fk : (uint32_t)fi * gf.s + fk;
    bv[m] = in ? b[lin] : 0.0;
  }
  cp_wait<0>();
  __syncthreads();
  pdl_trigger();
  // ---- 2. r = b - A x on the r region (0 outside the box)
  constexpr int XPS = G::XJ * G::XK;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int e = tid + m * G::NT;
    if (e >= G::RSZ) break;
    const int pk = e % G::RK, t = e / G::RK;
    const int pj = DIM == 3 ? t % G::RJ : 0, pi = DIM == 3 ? t / G::RJ : t;
    const int fi = xi0 + 1 + pi, fj = DIM == 3 ? xj0 + 1 + pj : 0, fk = xk0 + 1 + pk;
    const bool in = fi >= 0 && fi <= gf.n && fk >= 0 && fk <= gf.n && (DIM == 2 || (fj >= 0 && fj <= gf.n));
    double r = 0.0;
    if (in) {
      const int cls = class_of<DIM>(gf, fi, fj, fk);
      const double* xc = xs + (pi + 1) * XPS + (DIM == 3 ? (pj + 1) * G::XK : 0) + pk + 1;
      double As = 0.0;
      if (cls == Traits<DIM>::INTERIOR) {
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
          As = fma(op.w[o], xc[di * XPS + dj * G::XK + dk], As);
        }
      } else {
        // class row; a missing neighbour has weight 0 and reads a staged zero
        const double* w = op.tab + cls * (NO + 1);
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
          As = fma(__ldg(w + o), xc[di * XPS + dj * G::XK + dk], As);
        }
      }
      r = bv[m] - As;
    }
    rs[e] = r;
  }
  __syncthreads();
  // ---- 3. this thread's coarse vertex: row of P^T in slot order (k_restrict)
  const int ck = tid % C::CK, t2 = tid / C::CK;
  const int cj = DIM == 3 ? t2 % C::CJ : 0, ci = DIM == 3 ? t2 / C::CJ : t2;
  const int I = I0 + ci, J = J0 + cj, K = K0 + ck;
  if (I > gc.n || K > gc.n || (DIM == 3 && J > gc.n)) return;
  const int cls = class_of<DIM>(gc, I, J, K);
  constexpr int RPS = G::RJ * G::RK;
  const double* rc = rs + (2 * ci + 1) * RPS + (DIM == 3 ? (2 * cj + 1) * G::RK : 0) + 2 * ck + 1;
  double s = 0.0;
  if (cls == Traits<DIM>::INTERIOR) {
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
      s += (o == Traits<DIM>::CENTER ? 1.0 : 0.5) * rc[di * RPS + dj * G::RK + dk];
    }
  } else {
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
      // (a missing slot reads the zero stored for the vertex outside the box)
      s += (slot_ok<DIM>(cls, o) ? (o == Traits<DIM>::CENTER ? 1.0 : 0.5) : 0.0) * rc[di * RPS + dj * G::RK + dk];
    }
  }
  const uint32_t cidx = DIM == 3 ? (uint32_t)I * gc.ps + (uint32_t)J * gc.s + K : (uint32_t)I * gc.s + K;
  bc[cidx] = s;
}

}  // namespace okg
