// okg_cluster.cuh -- the middle of the V-cycle in ONE thread-block-cluster launch.
//
// Below the tiled levels (3D: 33^3 and 17^3 at 128^3; 2D: 257^2 ... 65^2 at
// 2048^2) a multigrid level is latency-bound: k_mg_down + k_mg_up cost 7-11 us
// per level for 0.04-0.3 MB of data, and the collapsed bottom (k_coarse_sym +
// k_coarse_sym_sum) another ~8 us -- ~40 us of every V-cycle at 128^3, 20
// V-cycles per GMRES iteration.  Here a cluster of MC_C = 16 CTAs (one per SM,
// 1024 threads each) keeps those levels in distributed shared memory and runs
// mg_cycle V(2,2) (multigrid.hpp:97-117) on them with barrier.cluster between
// phases instead of kernel boundaries:
//
//  * every level is split into x-plane ranges, one per CTA; the coarser level
//    takes the coarse planes G with 2G in the finer range, so restriction and
//    prolongation need only the +-1 ghost planes every CTA holds;
//  * a phase computes its CTA's planes into local shared memory and stores the
//    first / last plane straight into the ghost planes of the CTAs that need
//    them (st.shared::cluster, fire and forget), then one cluster barrier
//    (release / acquire) publishes them;
//  * pointwise steps (e1 = w D^-1 b, e = e2 + P e_c) are also computed on the
//    ghost planes, so they need no exchange at all;
//  * the bottom is the collapsed operator (okg_params.mg_collapse): the packed
//    symmetric blocks are split over the CTAs, each block's row/column partial
//    products are pushed to the CTA that owns the row block, which adds them in
//    k_coarse_sym_sum's order and broadcasts the rows to every CTA.
//
// Every vertex uses the expressions of the unfused kernels in the same order
// (k_pre2 / k_op<EPI_*> / k_restrict / k_prolong_add, k_coarse_sym +
// k_coarse_sym_sum), so the result is bit-identical to the multi-launch path.
#pragma once
#include <cooperative_groups.h>

#include "okg_kernels.cuh"
#include "okg_tail.cuh"

namespace okg {

constexpr int MC_C = 16;     // CTAs per cluster (non-portable size, opted in at setup)
#ifndef OKG_MC_NT
#define OKG_MC_NT 512
#endif
#ifndef OKG_MC_UMAX
#define OKG_MC_UMAX 2
#endif
constexpr int MC_NT = OKG_MC_NT;  // threads per CTA (512: 92 registers, no spills)
constexpr int MC_MAXL = 4;   // distributed levels at most
constexpr int MC_CB = 64;    // block size of the packed collapsed operator (== CB)
constexpr int MC_TPG = 256;  // threads per block product (k_coarse_sym's CTA)
constexpr int MC_GROUPS = MC_NT / MC_TPG;

// first owned x-plane of cluster rank r on level q (r = MC_C: the plane count)
__host__ __device__ constexpr int mc_lo(int s0, int q, int r) {
  int lo = r * s0 / MC_C;
  for (int t = 0; t < q; ++t) lo = (lo + 1) / 2;
  return lo;
}
__host__ __device__ constexpr int mc_maxown(int s0, int q) {
  int m = 0;
  for (int r = 0; r < MC_C; ++r) {
    const int c = mc_lo(s0, q, r + 1) - mc_lo(s0, q, r);
    if (c > m) m = c;
  }
  return m;
}

// level Q of a cluster run starting at n = N0: three arrays (B = rhs, X1, X2), each
// [guard][ghost plane][owned planes...][ghost plane][guard], the same layout (and
// the same shared-memory offsets) in every CTA of the cluster
template <int DIM, int N0, int Q>
struct MLev {
  static constexpr int n = N0 >> Q;
  using T = TL<DIM, n>;
  static constexpr int G = DIM == 3 ? T::s + 1 : 1;  // reach of a tap beyond the ghost planes
  static constexpr int NP = mc_maxown(N0 + 1, Q) + 2;
  static constexpr int LEN = 2 * G + NP * T::ps;
  static constexpr int SIZE = 3 * LEN;
};
template <int DIM, int N0, int Q, int NL>
constexpr int mc_levels_doubles() {
  if constexpr (Q < NL) return MLev<DIM, N0, Q>::SIZE + mc_levels_doubles<DIM, N0, Q + 1, NL>();
  else return 0;
}

// the collapsed bottom (level NL): full rhs and result on every CTA, the row blocks
// a CTA sums (I = rank, rank + C, ...) with one 64-slot per block term, and the
// column partials of the block products in flight
template <int DIM, int N0, int NL>
struct MBot {
  static constexpr int NB = TL<DIM, (N0 >> NL)>::N;
  static constexpr int nb = (NB + MC_CB - 1) / MC_CB;
  static constexpr int ROWBLK = (nb + MC_C - 1) / MC_C;  // row blocks per CTA
  static constexpr int RECV = ROWBLK * nb * MC_CB;
  static constexpr int CPART = MC_GROUPS * 8 * MC_CB;
  static constexpr int SIZE = 2 * NB + RECV + CPART;
};

template <int DIM>
constexpr int mc_table_doubles(int nl) {
  return nl * Traits<DIM>::NCLS * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NCLS * Traits<DIM>::NOFF;
}

template <int DIM, int N0, int NL>
constexpr size_t mc_smem_bytes() {
  return sizeof(double) *
             ((size_t)mc_table_doubles<DIM>(NL) + mc_levels_doubles<DIM, N0, 0, NL>() + MBot<DIM, N0, NL>::SIZE) +
         sizeof(int) * (MC_MAXL + 1) * (MC_C + 1);
}

template <int DIM>
struct MCArgs {
  const double* tabs;  // [NL][NCLS][NOFF+1] level class rows, then [NCLS][NOFF] restriction weights
  double omega;
  const double* rhs;   // rhs of the first level (global, whole level)
  double* out;         // its V-cycle result (global)
  const double* colA;  // collapsed bottom: packed lower block triangle (k_coarse_pack)
};

namespace mcd {

__device__ __forceinline__ void st_remote(double* local_addr, unsigned rank, double v) {
  namespace cg = cooperative_groups;
  double* r = cg::this_cluster().map_shared_rank(local_addr, rank);
  *r = v;
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// f(local index, i, j, k, rem, cls) over global planes [p0, p1) of level (DIM, n); the
// level's own range starts at `lo` (2D: k is the fast coordinate, j = 0)
template <int DIM, int N0, int Q, class F>
__device__ __forceinline__ void each(int p0, int p1, int lo, F&& f) {
  using L = MLev<DIM, N0, Q>;
  using T = typename L::T;
  const int cnt = (p1 - p0) * (int)T::ps;
  for (int e = threadIdx.x; e < cnt; e += MC_NT) {
    const int a = e / T::ps;
    const int rem = e - a * T::ps;
    const int i = p0 + a;
    int j, k, cls;
    if (DIM == 3) {
      j = rem / T::s;
      k = rem - j * T::s;
      cls = T::cd(i) * 9 + T::cd(j) * 3 + T::cd(k);
    } else {
      j = 0;
      k = rem;
      cls = T::cd(i) * 3 + T::cd(k);
    }
    f(L::G + (i - lo + 1) * T::ps + rem, i, j, k, rem, cls);
  }
}

// A x at local index v (all NOFF taps with the class row, as okg_tail.cuh)
template <int DIM, int n>
__device__ __forceinline__ double row(const double* W, const double* x, int v) {
  using T = TL<DIM, n>;
  double s = 0.0;
  static_for<Traits<DIM>::NOFF>([&](auto o) { s = fma(W[o], x[v + T::template off<o>()], s); });
  return s;
}

enum { SW_JACOBI = 0, SW_RESID = 1, SW_OUT = 2 };

// One smoothing / residual pass over the own planes [lo, hi) of level Q:
//   SW_JACOBI: y = x + w D^-1 (b - A x)  (k_op<EPI_JACOBI>)      -> dst
//   SW_RESID:  y = b - A x               (k_op<EPI_RESID>)       -> dst
//   SW_OUT:    SW_JACOBI written to the global result (level 0 only)
// U vertices per thread with their FMA chains interleaved (the chain of one vertex is
// sequential: 15 dependent DFMAs in 3D).  The first own plane is also stored into
// the high ghost plane of rank-1 (rlo) and the last into the low ghost plane of
// rank+1 (rhi); null at the grid boundary.
template <int DIM, int N0, int Q, int MODE, int U>
__device__ __forceinline__ void sweep(const double* __restrict__ Wq, double om, const double* B, const double* src,
                                      double* dst, double* rlo, double* rhi, int lo, int hi, double* gout) {
  using L = MLev<DIM, N0, Q>;
  using T = typename L::T;
  constexpr int NO = Traits<DIM>::NOFF;
  const int cnt = (hi - lo) * (int)T::ps;
  const int last = (hi - lo - 1) * (int)T::ps;  // first e of the last own plane
  for (int base = threadIdx.x; base < cnt; base += U * MC_NT) {
    int vv[U], cc[U], ee[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e0 = base + u * MC_NT;
      ee[u] = e0;
      const int e = e0 < cnt ? e0 : base;
      const int a = e / T::ps;
      const int rem = e - a * T::ps;
      const int i = lo + a;
      int cls;
      if (DIM == 3) {
        const int j = rem / T::s, k = rem - j * (int)T::s;
        cls = T::cd(i) * 9 + T::cd(j) * 3 + T::cd(k);
      } else {
        cls = T::cd(i) * 3 + T::cd(rem);
      }
      vv[u] = L::G + T::ps + e;
      cc[u] = cls * (NO + 1);
    }
    double sum[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sum[u] = 0.0;
    static_for<NO>([&](auto o) {
#pragma unroll
      for (int u = 0; u < U; ++u) sum[u] = fma(Wq[cc[u] + o], src[vv[u] + T::template off<o>()], sum[u]);
    });
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = ee[u];
      if (e >= cnt) break;
      const double bv = B[vv[u]];
      const double y = MODE == SW_RESID ? bv - sum[u] : fma(om * Wq[cc[u] + NO], bv - sum[u], src[vv[u]]);
      if (MODE == SW_OUT) {
        gout[lo * (int)T::ps + e] = y;
      } else {
        dst[vv[u]] = y;
        if (rlo && e < (int)T::ps) rlo[e] = y;
        if (rhi && e >= last) rhi[e - last] = y;
      }
    }
  }
}

// every CTA owns at least one plane of every distributed level, so a CTA's ghost
// planes are exactly its neighbours' edge planes
template <int N0, int NL>
constexpr bool mc_nonempty() {
  for (int q = 0; q <= NL; ++q)
    for (int r = 0; r < MC_C; ++r)
      if (mc_lo(N0 + 1, q, r + 1) <= mc_lo(N0 + 1, q, r)) return q == NL;  // (the bottom is whole)
  return true;
}

// vertices per thread of one sweep pass (<= 2: more interleaved chains spill at 64
// registers)
template <int DIM, int N0, int Q>
constexpr int mc_unroll() {
  const int v = mc_maxown(N0 + 1, Q) * TL<DIM, (N0 >> Q)>::ps;
  const int u = (v + MC_NT - 1) / MC_NT;
  return u > OKG_MC_UMAX ? OKG_MC_UMAX : (u < 1 ? 1 : u);
}

}  // namespace mcd

template <int DIM, int N0, int NL>
__device__ void mc_bottom(const MCArgs<DIM>& A, double* bot, unsigned rk);

// One level of the cluster V-cycle: V(2,2) from zero.  Level Q's B holds the rhs on
// the own and ghost planes when this is called; the result x is left in X2 (own and
// ghost planes), or for Q == 0 written to A.out.
template <int DIM, int N0, int Q, int NL>
__device__ void mc_level(const MCArgs<DIM>& A, const double* tabs, double* base, double* bot, const int* los,
                         unsigned rk) {
  using L = MLev<DIM, N0, Q>;
  using T = typename L::T;
  constexpr int n = L::n;
  constexpr int NO = Traits<DIM>::NOFF;
  constexpr int NCL = Traits<DIM>::NCLS;
  const double* Wq = tabs + Q * NCL * (NO + 1);
  const double om = A.omega;
  double* B = base;
  double* X1 = base + L::LEN;
  double* X2 = base + 2 * L::LEN;
  const int* lo_q = los + Q * (MC_C + 1);
  const int lo = lo_q[rk], hi = lo_q[rk + 1];
  const int glo = lo > 0 ? lo - 1 : 0, ghi = hi < T::s ? hi + 1 : T::s;  // own + existing ghosts
  constexpr int U = mcd::mc_unroll<DIM, N0, Q>();
  // the neighbours' ghost planes of each array: rank-1's high ghost, rank+1's low ghost
  namespace cg = cooperative_groups;
  const int slot_hi_lo = rk > 0 ? lo - lo_q[rk - 1] + 1 : 0;  // rank-1 owns [lo_q[rk-1], lo)
  auto nb_lo = [&](double* arr) -> double* {
    return rk > 0 ? cg::this_cluster().map_shared_rank(arr + L::G + slot_hi_lo * T::ps, rk - 1) : nullptr;
  };
  auto nb_hi = [&](double* arr) -> double* {
    return rk + 1 < MC_C ? cg::this_cluster().map_shared_rank(arr + L::G, rk + 1) : nullptr;
  };
  // ---- pre-smoothing from zero (k_pre2): e1 = w D^-1 b on own + ghost planes (local) ----
  mcd::each<DIM, N0, Q>(glo, ghi, lo, [&](int v, int, int, int, int, int cls) {
    X1[v] = __dmul_rn(om * Wq[cls * (NO + 1) + NO], B[v]);
  });
  __syncthreads();
  // e2 = e1 + w D^-1 (b - A e1) -> X2
  mcd::sweep<DIM, N0, Q, mcd::SW_JACOBI, U>(Wq, om, B, X1, X2, nb_lo(X2), nb_hi(X2), lo, hi, nullptr);
  mcd::cluster_barrier();
  // ---- residual (k_op<EPI_RESID>) -> X1 ----
  mcd::sweep<DIM, N0, Q, mcd::SW_RESID, U>(Wq, om, B, X2, X1, nb_lo(X1), nb_hi(X1), lo, hi, nullptr);
  mcd::cluster_barrier();
  // ---- restriction (k_restrict) -> rhs of level Q+1 (own + ghost coarse planes of the
  // CTAs that hold them), or the full rhs of the collapsed bottom on every CTA ----
  {
    constexpr int nc = n / 2;
    using TC = TL<DIM, nc>;
    const double* RW = tabs + NL * NCL * (NO + 1);  // [cls][NOFF]
    const int* lo_c = los + (Q + 1) * (MC_C + 1);
    const int clo = lo_c[rk], chi = lo_c[rk + 1];
    double* Bc = nullptr;
    if constexpr (Q + 1 < NL) Bc = base + L::SIZE;  // next level's B
    const int cnt = (chi - clo) * (int)TC::ps;
    for (int e = threadIdx.x; e < cnt; e += MC_NT) {
      const int a = e / TC::ps;
      const int rem = e - a * TC::ps;
      const int Gi = clo + a;
      int Gj, Gk, ccls;
      if (DIM == 3) {
        Gj = rem / TC::s;
        Gk = rem - Gj * TC::s;
        ccls = TC::cd(Gi) * 9 + TC::cd(Gj) * 3 + TC::cd(Gk);
      } else {
        Gj = 0;
        Gk = rem;
        ccls = TC::cd(Gi) * 3 + TC::cd(Gk);
      }
      const int F = L::G + (2 * Gi - lo + 1) * T::ps + (DIM == 3 ? 2 * Gj * T::s + 2 * Gk : 2 * Gk);
      const double* R = RW + ccls * NO;
      double s = 0.0;
      static_for<NO>([&](auto o) { s += R[o] * X1[F + T::template off<o>()]; });
      if constexpr (Q + 1 < NL) {
        using LC = MLev<DIM, N0, Q + 1>;
        Bc[LC::G + (Gi - clo + 1) * TC::ps + rem] = s;
        if (Gi == clo && rk > 0)  // rank-1's high ghost plane
          cg::this_cluster().map_shared_rank(Bc + LC::G + (clo - lo_c[rk - 1] + 1) * TC::ps + rem, rk - 1)[0] = s;
        if (Gi == chi - 1 && rk + 1 < MC_C)  // rank+1's low ghost plane
          cg::this_cluster().map_shared_rank(Bc + LC::G + rem, rk + 1)[0] = s;
      } else {
        const int g = Gi * TC::ps + rem;  // global index on the bottom level
        bot[g] = s;
#pragma unroll 1
        for (int t = 0; t < MC_C; ++t)
          if (t != (int)rk) mcd::st_remote(bot + g, t, s);
      }
    }
  }
  mcd::cluster_barrier();
  // ---- coarse-grid correction ----
  if constexpr (Q + 1 < NL) mc_level<DIM, N0, Q + 1, NL>(A, tabs, base + L::SIZE, bot, los, rk);
  else mc_bottom<DIM, N0, NL>(A, bot, rk);
  // ---- e = e2 + P x_c (k_prolong_add) on own + ghost planes (local) -> X2 ----
  {
    constexpr int nc = n / 2;
    using TC = TL<DIM, nc>;
    const double* xc;
    int cbase;  // local index of coarse plane 0 in xc
    if constexpr (Q + 1 < NL) {
      using LC = MLev<DIM, N0, Q + 1>;
      const int clo = los[(Q + 1) * (MC_C + 1) + rk];
      xc = base + L::SIZE + 2 * LC::LEN;  // next level's X2
      cbase = LC::G + (1 - clo) * TC::ps;
    } else {
      xc = bot + MBot<DIM, N0, NL>::NB;  // full result of the bottom
      cbase = 0;
    }
    mcd::each<DIM, N0, Q>(glo, ghi, lo, [&](int v, int i, int j, int k, int, int) {
        const int li = i >> 1, lj = j >> 1, lk = k >> 1;
        const int hi2 = (i + 1) >> 1, hj = (j + 1) >> 1, hk = (k + 1) >> 1;
        const int clo_i = DIM == 3 ? li * TC::ps + lj * TC::s + lk : li * TC::s + lk;
        const int cup_i = DIM == 3 ? hi2 * TC::ps + hj * TC::s + hk : hi2 * TC::s + hk;
        double t;
        if (clo_i == cup_i) t = xc[cbase + clo_i];
        else t = fma(0.5, xc[cbase + cup_i], 0.5 * xc[cbase + clo_i]);
        X2[v] = X2[v] + t;
      });
  }
  __syncthreads();
  // ---- two post-sweeps (k_op<EPI_JACOBI>, then EPI_JACOBI_SET) ----
  mcd::sweep<DIM, N0, Q, mcd::SW_JACOBI, U>(Wq, om, B, X2, X1, nb_lo(X1), nb_hi(X1), lo, hi, nullptr);
  mcd::cluster_barrier();
  if constexpr (Q == 0) {
    mcd::sweep<DIM, N0, Q, mcd::SW_OUT, U>(Wq, om, B, X1, nullptr, nullptr, nullptr, lo, hi, A.out);
  } else {
    mcd::sweep<DIM, N0, Q, mcd::SW_JACOBI, U>(Wq, om, B, X1, X2, nb_lo(X2), nb_hi(X2), lo, hi, nullptr);
    mcd::cluster_barrier();
  }
}

// The collapsed bottom: y = F b with F the packed symmetric operator.  Block products
// exactly as k_coarse_sym (R = A_IJ x_J by warp rows, C = A_IJ^T x_I by lane columns),
// pushed into the receive slots of the CTA owning row block I (R) or J (C); that CTA
// sums every row in k_coarse_sym_sum's order and broadcasts it.
template <int DIM, int N0, int NL>
__device__ void mc_bottom(const MCArgs<DIM>& A, double* bot, unsigned rk) {
  using Bt = MBot<DIM, N0, NL>;
  constexpr int NB = Bt::NB, nb = Bt::nb, CBk = MC_CB;
  const double* x = bot;        // full rhs
  double* y = bot + NB;         // full result
  double* recv = bot + 2 * NB;  // [ROWBLK][nb][64]
  double* cpart = recv + Bt::RECV;
  const int tid = threadIdx.x, grp = tid / MC_TPG, gt = tid % MC_TPG, lane = gt & 31, w = gt >> 5;
  double* cp = cpart + grp * 8 * CBk;
  constexpr int NBLK = nb * (nb + 1) / 2;
  // slot of the term of block (I, J) (J <= I) in row block I's sum: q = J; in row block
  // J's sum (C part, I > J): q = I
  for (int t0 = (int)rk * MC_GROUPS; t0 < NBLK; t0 += MC_C * MC_GROUPS) {
    const int b = t0 + grp;  // blocks b, b+1, .. b+3 on this CTA's groups in this round
    int I = 0, J = 0;
    if (b < NBLK) tri_index(b, I, J);
    double2 a[CBk / 8];
    if (b < NBLK) {
      const double2* blk = reinterpret_cast<const double2*>(A.colA + (size_t)b * CBk * CBk);
#pragma unroll
      for (int q = 0; q < CBk / 8; ++q) a[q] = __ldg(blk + (size_t)(w + 8 * q) * (CBk / 2) + lane);
    }
    double c0 = 0.0, c1 = 0.0;
    if (b < NBLK) {
      const int cj0 = J * CBk + 2 * lane;
      const double xj0 = cj0 < NB ? x[cj0] : 0.0, xj1 = cj0 + 1 < NB ? x[cj0 + 1] : 0.0;
      const int ownI = I % MC_C, slotI = I / MC_C;
#pragma unroll
      for (int q = 0; q < CBk / 8; ++q) {
        const int r = w + 8 * q;
        double s = fma(a[q].y, xj1, a[q].x * xj0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          double* dst = recv + ((size_t)slotI * nb + J) * CBk + r;
          if (ownI == (int)rk) *dst = s;
          else mcd::st_remote(dst, ownI, s);
        }
        const int ri = I * CBk + r;
        const double xr = ri < NB ? x[ri] : 0.0;
        c0 = fma(a[q].x, xr, c0);
        c1 = fma(a[q].y, xr, c1);
      }
    }
    const bool offd = b < NBLK && I != J;
    if (offd) {
      cp[w * CBk + 2 * lane] = c0;
      cp[w * CBk + 2 * lane + 1] = c1;
    }
    __syncthreads();
    if (offd && gt < CBk) {
      double c = cp[gt];
#pragma unroll
      for (int q = 1; q < 8; ++q) c += cp[q * CBk + gt];
      const int ownJ = J % MC_C, slotJ = J / MC_C;
      double* dst = recv + ((size_t)slotJ * nb + I) * CBk + gt;
      if (ownJ == (int)rk) *dst = c;
      else mcd::st_remote(dst, ownJ, c);
    }
    __syncthreads();
  }
  mcd::cluster_barrier();
  // row sums of the own row blocks (k_coarse_sym_sum: 4 segments in order), broadcast
  constexpr int CSEGk = 4;
  constexpr int per = (nb + CSEGk - 1) / CSEGk;
  for (int e = tid; e < Bt::ROWBLK * CBk; e += MC_NT) {
    const int slot = e / CBk, t = e % CBk;
    const int I = slot * MC_C + (int)rk;
    if (I >= nb) continue;
    const double* rv = recv + (size_t)slot * nb * CBk + t;
    double r = 0.0;
#pragma unroll
    for (int sg = 0; sg < CSEGk; ++sg) {
      const int q0 = sg * per, q1 = min(nb, q0 + per);
      double s = 0.0;
      for (int q = q0; q < q1; ++q) s += rv[(size_t)q * CBk];
      if (sg == 0) r = s;
      else r += s;
    }
    const int row = I * CBk + t;
    if (row < NB) {
      y[row] = r;
#pragma unroll 1
      for (int o = 0; o < MC_C; ++o)
        if (o != (int)rk) mcd::st_remote(y + row, o, r);
    }
  }
  mcd::cluster_barrier();
}

template <int DIM, int N0, int NL>
__global__ void __launch_bounds__(MC_NT, 1) k_mg_cluster(const MCArgs<DIM> A) {
  static_assert(mcd::mc_nonempty<N0, NL>(), "every CTA must own planes of every cluster level");
  extern __shared__ double sm[];
  namespace cg = cooperative_groups;
  const unsigned rk = cg::this_cluster().block_rank();
  constexpr int NTAB = mc_table_doubles<DIM>(NL);
  constexpr int NLEV = mc_levels_doubles<DIM, N0, 0, NL>();
  constexpr int NBOT = MBot<DIM, N0, NL>::SIZE;
  double* tabs = sm;
  double* base = tabs + NTAB;
  double* bot = base + NLEV;
  int* los = reinterpret_cast<int*>(bot + NBOT);  // [NL + 1][MC_C + 1]
  // constants (tables) before griddepcontrol.wait: they overlap the predecessor's tail
  for (int e = threadIdx.x; e < NTAB; e += MC_NT) cpa8(tabs + e, A.tabs + e);
  cpa_commit();
  // zero the level arrays (ghost planes outside the grid and guards are read with
  // weight 0 and must be finite) and the bottom
  for (int e = threadIdx.x; e < NLEV + NBOT; e += MC_NT) base[e] = 0.0;
  for (int e = threadIdx.x; e < (NL + 1) * (MC_C + 1); e += MC_NT)
    los[e] = mc_lo(N0 + 1, e / (MC_C + 1), e % (MC_C + 1));
  __syncthreads();
  // every CTA's zeroing must be done before any CTA stores into its ghost planes
  mcd::cluster_barrier();
  PDL_ENTRY();
  {  // the first level's rhs on own + ghost planes, straight from global
    using L = MLev<DIM, N0, 0>;
    using T = typename L::T;
    const int lo = los[rk], hi = los[rk + 1];
    const int glo = lo > 0 ? lo - 1 : 0, ghi = hi < T::s ? hi + 1 : T::s;
    const int cnt = (ghi - glo) * (int)T::ps;
    for (int e = threadIdx.x; e < cnt; e += MC_NT) {
      const int g = glo * T::ps + e;
      cpa8(base + L::G + (glo - lo + 1) * T::ps + e, A.rhs + g);
    }
    cpa_commit();
  }
  cpa_wait<0>();
  __syncthreads();
  mc_level<DIM, N0, 0, NL>(A, tabs, base, bot, los, rk);
}

}  // namespace okg
