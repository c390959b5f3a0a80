// okg_vcycle.cuh -- temporally blocked multigrid level kernels.
//
// mg_cycle (multigrid.hpp:97-117) with V(2,2) visits every level twice:
//   down:  e1 = w D^-1 b ; e2 = e1 + w D^-1 (b - A e1) ; r = b - A e2 ; b_c = P^T r
//   up:    e = e2 + P e_c ; e' = e + w D^-1 (b - A e) ; x = e' + w D^-1 (b - A e')
// Done naively that is 5-6 kernels per level, each a full pass over the level
// and, below ~10^5 vertices, pure launch/latency cost.  Here each direction is
// ONE kernel: a CTA owns a fine box F of the level (aligned to the coarse
// grid), stages its operand with a halo of 3 (down) or 2 (up) vertices in
// shared memory and computes the successive sweeps on shrinking regions, so
// e1, r and e' never touch global memory.  Boundary vertices use the per-class
// weight table; out-of-box neighbours never occur (the regions nest).
// The arithmetic of every vertex is the same expression, in the same order,
// as the unfused kernels (okg_kernels.cuh / okg_tiled.cuh): results are
// bit-identical to them.
#pragma once
#include "okg_tiled.cuh"

namespace okg {

// fine box per CTA (even extents, aligned to the coarse grid); BX = 1 is the
// larger box used on big levels (less halo redundancy, fewer CTAs)
template <int DIM, int BX = 0>
struct MgBox;
#ifndef OKG_MG3_FI  // (-D overrides: box-shape experiments)
#define OKG_MG3_FI 2
#define OKG_MG3_FJ 2
#define OKG_MG3_FK 8
#define OKG_MG3_NT 512
#endif
#ifndef OKG_MG3_FUSE_N  // 3D / 2D levels with n <= this use the fused kernels (okg_host.cu build)
#define OKG_MG3_FUSE_N 16
#endif
#ifndef OKG_MG2_FUSE_N
#define OKG_MG2_FUSE_N 512
#endif
template <>
struct MgBox<3, 0> {
  static constexpr int FI = OKG_MG3_FI, FJ = OKG_MG3_FJ, FK = OKG_MG3_FK, NT = OKG_MG3_NT;
};
template <>
struct MgBox<3, 1> {
  static constexpr int FI = 4, FJ = 8, FK = 32, NT = 256;
};
#ifndef OKG_MG2_FI
#define OKG_MG2_FI 8
#define OKG_MG2_FK 16
#define OKG_MG2_NT 256
#endif
template <>
struct MgBox<2, 0> {
  static constexpr int FI = OKG_MG2_FI, FJ = 1, FK = OKG_MG2_FK, NT = OKG_MG2_NT;
};
template <>
struct MgBox<2, 1> {
  static constexpr int FI = 8, FJ = 1, FK = 128, NT = 256;
};

// a box region [o_i, o_i+NI) x [o_j, o_j+NJ) x [o_k, o_k+NK) of the level grid,
// extents known at compile time: the box F grown by HALO (minus LO on the high side)
template <int DIM, int HALO, int LO, int BX = 0>
struct Reg {
  using B = MgBox<DIM, BX>;
  static constexpr int NI = B::FI + 2 * HALO - LO;
  static constexpr int NJ = DIM == 3 ? B::FJ + 2 * HALO - LO : 1;
  static constexpr int NK = B::FK + 2 * HALO - LO;
  static constexpr int SIZE = NI * NJ * NK;
  int oi, oj, ok;
  __device__ Reg(int fi0, int fj0, int fk0) : oi(fi0 - HALO), oj(DIM == 3 ? fj0 - HALO : 0), ok(fk0 - HALO) {}
  // local index e -> global coords (k is the fastest coordinate, also in 2D)
  __device__ __forceinline__ void coords(int e, int& i, int& j, int& k) const {
    const int a = e / NK;
    k = ok + (e - a * NK);
    if (DIM == 3) {
      const int b = a / NJ;
      j = oj + (a - b * NJ);
      i = oi + b;
    } else {
      j = 0;
      i = oi + a;
    }
  }
  __device__ __forceinline__ int index(int i, int j, int k) const {
    return DIM == 3 ? ((i - oi) * NJ + (j - oj)) * NK + (k - ok) : (i - oi) * NK + (k - ok);
  }
  __device__ __forceinline__ bool contains(int i, int j, int k) const {
    return i >= oi && i < oi + NI && k >= ok && k < ok + NK && (DIM == 2 || (j >= oj && j < oj + NJ));
  }
};

template <int DIM>
__device__ __forceinline__ bool in_grid(const Grid& g, int i, int j, int k) {
  return i >= 0 && i <= g.n && k >= 0 && k <= g.n && (DIM == 2 || (j >= 0 && j <= g.n));
}

template <int DIM>
__device__ __forceinline__ uint32_t lin_of(const Grid& g, int i, int j, int k) {
  return DIM == 3 ? (uint32_t)i * g.ps + (uint32_t)j * g.s + k : (uint32_t)i * g.s + k;
}

// A s at vertex (i,j,k) of class cls, s read from region buffer `src` (region rs).
// W = the level's class table in shared memory ([NCLS][NOFF+1], missing slots 0):
// every vertex runs the same NOFF taps (the staged region is zero outside the
// grid); vs the unfused kernels, which skip zero-weight slots of boundary rows,
// only the sign of a zero can differ.
template <int DIM, class RS>
__device__ __forceinline__ double reg_row(const double* W, int cls, const double* src, const RS& rs, int i, int j,
                                          int k, double& own) {
  constexpr int NO = Traits<DIM>::NOFF;
  const int c = rs.index(i, j, k);
  constexpr int sj = DIM == 3 ? RS::NK : 0, si = DIM == 3 ? RS::NJ * RS::NK : RS::NK;
  const double* w = W + cls * (NO + 1);
  double As = 0.0;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
    const double v = src[c + di * si + dj * sj + dk];
    if (o == Traits<DIM>::CENTER) own = v;
    As = fma(w[o], v, As);
  }
  return As;
}

template <int DIM>
__device__ __forceinline__ double cls_invd(const double* W, int cls) {
  return W[cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF];
}

// copy the level's class table into shared memory (caller syncs)
// (cp.async: issued before griddepcontrol.wait -- the table is constant -- so its
// latency overlaps the predecessor kernel; the caller waits with cp.async.wait_all)
template <int DIM, int NT>
__device__ __forceinline__ void load_table(double* W, const Op<DIM>& op) {
  constexpr int T = Traits<DIM>::NCLS * (Traits<DIM>::NOFF + 1);
  for (int e = threadIdx.x; e < T; e += NT) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(W + e);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(op.tab + e) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void table_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int DIM>
constexpr int table_doubles() { return Traits<DIM>::NCLS * (Traits<DIM>::NOFF + 1); }

// box origin of this CTA (fine coordinates)
template <int DIM, int BX>
__device__ __forceinline__ void box_origin(const Grid& g, int& fi0, int& fj0, int& fk0) {
  using B = MgBox<DIM, BX>;
  const int nbk = g.n / B::FK + 1, nbj = DIM == 3 ? g.n / B::FJ + 1 : 1;
  int b = blockIdx.x;
  const int bk = b % nbk;
  b /= nbk;
  const int bj = b % nbj;
  const int bi = b / nbj;
  fi0 = bi * B::FI;
  fj0 = DIM == 3 ? bj * B::FJ : 0;
  fk0 = bk * B::FK;
}

// ---------------------------------------------------------------------------
// DOWN: two pre-sweeps from zero, residual, restriction.  Writes e2 (level l)
// and bc = P^T (b - A e2) (level l+1).
//   S = F+3 : e1 = w D^-1 b          E = F+2 : e2 (and b)
//   R = F+1 (low side) : r           coarse points 2G in F : bc
// Staging loads are batched (U in flight per thread); the later phases read
// shared memory only.
// ---------------------------------------------------------------------------
template <int DIM, int BX>
__global__ void __launch_bounds__(MgBox<DIM, BX>::NT) k_mg_down(Grid g, Grid gc, Op<DIM> op, double omega,
                                                                const double* __restrict__ b, double* __restrict__ e2,
                                                                double* __restrict__ bc) {
  using B = MgBox<DIM, BX>;
  using RS = Reg<DIM, 3, 0, BX>;
  using RE = Reg<DIM, 2, 0, BX>;
  using RR = Reg<DIM, 1, 1, BX>;
  extern __shared__ double sm[];
  int fi0, fj0, fk0;
  box_origin<DIM, BX>(g, fi0, fj0, fk0);
  const RS S(fi0, fj0, fk0);
  const RE E(fi0, fj0, fk0);
  const RR R(fi0, fj0, fk0);
  double* se1 = sm;            // |S|
  double* sb = se1 + RS::SIZE; // |E|
  double* se2 = sb + RE::SIZE; // |E|
  double* sr = se1;            // |R| overlays e1 after phase 2
  double* W = se2 + RE::SIZE;  // class table
  const int tid = threadIdx.x;
  constexpr int U = 8;
  PDL_EARLY();
  load_table<DIM, B::NT>(W, op);
  PDL_ENTRY();
  table_wait();
  __syncthreads();
  // phase 1: e1 on S, b on E (batched loads)
  for (int base = tid; base < RS::SIZE; base += B::NT * U) {
    double bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      int i, j, k;
      S.coords(e, i, j, k);
      bv[u] = (e < RS::SIZE && in_grid<DIM>(g, i, j, k)) ? __ldg(b + lin_of<DIM>(g, i, j, k)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      if (e >= RS::SIZE) break;
      int i, j, k;
      S.coords(e, i, j, k);
      const bool in = in_grid<DIM>(g, i, j, k);
      se1[e] = in ? omega * cls_invd<DIM>(W, class_of<DIM>(g, i, j, k)) * bv[u] : 0.0;
      if (E.contains(i, j, k)) sb[E.index(i, j, k)] = bv[u];
    }
  }
  __syncthreads();
  // phase 2: e2 on E ; write e2 for the box F
  for (int e = tid; e < RE::SIZE; e += B::NT) {
    int i, j, k;
    E.coords(e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(W, cls, se1, S, i, j, k, own);
      v = fma(omega * cls_invd<DIM>(W, cls), sb[e] - As, own);
      const bool inF = i >= fi0 && i < fi0 + B::FI && k >= fk0 && k < fk0 + B::FK &&
                       (DIM == 2 || (j >= fj0 && j < fj0 + B::FJ));
      if (inF) e2[lin_of<DIM>(g, i, j, k)] = v;
    }
    se2[e] = v;
  }
  __syncthreads();
  // phase 3: residual on R
  for (int e = tid; e < RR::SIZE; e += B::NT) {
    int i, j, k;
    R.coords(e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(W, cls, se2, E, i, j, k, own);
      v = sb[E.index(i, j, k)] - As;
    }
    sr[e] = v;
  }
  __syncthreads();
  // phase 4: restriction for coarse vertices G with 2G in F (spmv_transpose order)
  constexpr int CI = B::FI / 2, CJ = DIM == 3 ? B::FJ / 2 : 1, CK = B::FK / 2;
  for (int e = tid; e < CI * CJ * CK; e += B::NT) {
    const int ck = e % CK, t = e / CK;
    const int cj = DIM == 3 ? t % CJ : 0, ci = DIM == 3 ? t / CJ : t;
    const int Gi = fi0 / 2 + ci, Gj = DIM == 3 ? fj0 / 2 + cj : 0, Gk = fk0 / 2 + ck;
    if (!in_grid<DIM>(gc, Gi, Gj, Gk)) continue;
    const int c = R.index(2 * Gi, 2 * Gj, 2 * Gk);
    constexpr int sj = DIM == 3 ? RR::NK : 0, si = DIM == 3 ? RR::NJ * RR::NK : RR::NK;
    double s = 0.0;
#pragma unroll
    for (int o = 0; o < Traits<DIM>::NOFF; ++o) {
      const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
      if (!in_grid<DIM>(g, 2 * Gi + di, 2 * Gj + dj, 2 * Gk + dk)) continue;
      s += (o == Traits<DIM>::CENTER ? 1.0 : 0.5) * sr[c + di * si + dj * sj + dk];
    }
    bc[lin_of<DIM>(gc, Gi, Gj, Gk)] = s;
  }
}

// ---------------------------------------------------------------------------
// UP: coarse correction + two post-sweeps.  out = x (SET) or out += x (ACC).
//   P = F+2 : e = e2 + P e_c        Q = F+1 : e'        F : x
// ---------------------------------------------------------------------------
template <int DIM, int BX, bool ACC>
__global__ void __launch_bounds__(MgBox<DIM, BX>::NT) k_mg_up(Grid g, Grid gc, Op<DIM> op, double omega,
                                                              const double* __restrict__ b, const double* __restrict__ e2,
                                                              const double* __restrict__ ec, double* __restrict__ out) {
  using B = MgBox<DIM, BX>;
  using RP = Reg<DIM, 2, 0, BX>;
  using RQ = Reg<DIM, 1, 0, BX>;
  extern __shared__ double sm[];
  int fi0, fj0, fk0;
  box_origin<DIM, BX>(g, fi0, fj0, fk0);
  const RP P(fi0, fj0, fk0);
  const RQ Q(fi0, fj0, fk0);
  double* sp = sm;
  double* sq = sp + RP::SIZE;
  double* sbq = sq + RQ::SIZE;
  double* W = sbq + RQ::SIZE;  // class table
  const int tid = threadIdx.x;
  constexpr int U = 8;
  PDL_EARLY();
  load_table<DIM, B::NT>(W, op);
  PDL_ENTRY();
  for (int base = tid; base < RP::SIZE; base += B::NT * U) {
    double ev[U], tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      int i, j, k;
      P.coords(e, i, j, k);
      const bool in = e < RP::SIZE && in_grid<DIM>(g, i, j, k);
      ev[u] = in ? __ldg(e2 + lin_of<DIM>(g, i, j, k)) : 0.0;
      tv[u] = in ? prolong_at<DIM>(gc, ec, i, j, k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      if (e < RP::SIZE) sp[e] = ev[u] + tv[u];
    }
  }
  for (int base = tid; base < RQ::SIZE; base += B::NT * U) {
    double bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      int i, j, k;
      Q.coords(e, i, j, k);
      bv[u] = (e < RQ::SIZE && in_grid<DIM>(g, i, j, k)) ? __ldg(b + lin_of<DIM>(g, i, j, k)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * B::NT;
      if (e < RQ::SIZE) sbq[e] = bv[u];
    }
  }
  table_wait();
  __syncthreads();
  for (int e = tid; e < RQ::SIZE; e += B::NT) {
    int i, j, k;
    Q.coords(e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(W, cls, sp, P, i, j, k, own);
      v = fma(omega * cls_invd<DIM>(W, cls), sbq[e] - As, own);
    }
    sq[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < B::FI * B::FJ * B::FK; e += B::NT) {
    const int k = fk0 + e % B::FK, t = e / B::FK;
    const int j = DIM == 3 ? fj0 + t % B::FJ : 0, i = fi0 + (DIM == 3 ? t / B::FJ : t);
    if (!in_grid<DIM>(g, i, j, k)) continue;
    const int cls = class_of<DIM>(g, i, j, k);
    double own = 0.0;
    const double As = reg_row<DIM>(W, cls, sq, Q, i, j, k, own);
    const double x = fma(omega * cls_invd<DIM>(W, cls), sbq[Q.index(i, j, k)] - As, own);
    const uint32_t idx = lin_of<DIM>(g, i, j, k);
    if (ACC) out[idx] = out[idx] + x;
    else out[idx] = x;
  }
}

template <int DIM, int BX>
inline unsigned mg_boxes(const Grid& g) {
  using B = MgBox<DIM, BX>;
  return (unsigned)((g.n / B::FK + 1) * (DIM == 3 ? g.n / B::FJ + 1 : 1) * (g.n / B::FI + 1));
}
template <int DIM, int BX>
inline size_t mg_down_smem() {
  using B = MgBox<DIM, BX>;
  const size_t s = (size_t)(B::FI + 6) * (DIM == 3 ? B::FJ + 6 : 1) * (B::FK + 6);
  const size_t e = (size_t)(B::FI + 4) * (DIM == 3 ? B::FJ + 4 : 1) * (B::FK + 4);
  return (s + 2 * e + table_doubles<DIM>()) * sizeof(double);
}
template <int DIM, int BX>
inline size_t mg_up_smem() {
  using B = MgBox<DIM, BX>;
  const size_t p = (size_t)(B::FI + 4) * (DIM == 3 ? B::FJ + 4 : 1) * (B::FK + 4);
  const size_t q = (size_t)(B::FI + 2) * (DIM == 3 ? B::FJ + 2 : 1) * (B::FK + 2);
  return (p + 2 * q + table_doubles<DIM>()) * sizeof(double);
}

}  // namespace okg
