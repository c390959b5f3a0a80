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

// fine box per CTA (even extents, aligned to the coarse grid)
template <int DIM>
struct MgBox;
template <>
struct MgBox<3> {
  static constexpr int FI = 4, FJ = 4, FK = 16, NT = 256;
};
template <>
struct MgBox<2> {
  static constexpr int FI = 8, FJ = 1, FK = 64, NT = 256;
};

// a box region [o_i, o_i+ni) x [o_j, o_j+nj) x [o_k, o_k+nk) of the level grid
struct Reg {
  int oi, oj, ok;
  int ni, nj, nk;
};

template <int DIM>
__device__ __forceinline__ Reg make_reg(int fi0, int fj0, int fk0, int halo, int lo_extra) {
  // region covering [f0 - halo, f0 + F - 1 + halo - lo_extra]... (see callers)
  using B = MgBox<DIM>;
  Reg r;
  r.oi = fi0 - halo;
  r.oj = DIM == 3 ? fj0 - halo : 0;
  r.ok = fk0 - halo;
  r.ni = B::FI + 2 * halo - lo_extra;
  r.nj = DIM == 3 ? B::FJ + 2 * halo - lo_extra : 1;
  r.nk = B::FK + 2 * halo - lo_extra;
  return r;
}

template <int DIM>
__device__ __forceinline__ int reg_size(const Reg& r) {
  return r.ni * r.nj * r.nk;
}

// local index e -> global coords (i, j, k); k is the fastest coordinate in 2D too
template <int DIM>
__device__ __forceinline__ void reg_coords(const Reg& r, int e, int& i, int& j, int& k) {
  const int a = e / r.nk;
  k = r.ok + (e - a * r.nk);
  if (DIM == 3) {
    const int b = a / r.nj;
    j = r.oj + (a - b * r.nj);
    i = r.oi + b;
  } else {
    j = 0;
    i = r.oi + a;
  }
}

template <int DIM>
__device__ __forceinline__ int reg_index(const Reg& r, int i, int j, int k) {
  return DIM == 3 ? ((i - r.oi) * r.nj + (j - r.oj)) * r.nk + (k - r.ok) : (i - r.oi) * r.nk + (k - r.ok);
}

template <int DIM>
__device__ __forceinline__ bool in_grid(const Grid& g, int i, int j, int k) {
  return i >= 0 && i <= g.n && k >= 0 && k <= g.n && (DIM == 2 || (j >= 0 && j <= g.n));
}

template <int DIM>
__device__ __forceinline__ uint32_t lin_of(const Grid& g, int i, int j, int k) {
  return DIM == 3 ? (uint32_t)i * g.ps + (uint32_t)j * g.s + k : (uint32_t)i * g.s + k;
}

// A s at vertex (i,j,k) of class cls, s read from region buffer `src` (region rs)
template <int DIM>
__device__ __forceinline__ double reg_row(const Op<DIM>& op, int cls, const double* src, const Reg& rs, int i, int j,
                                          int k, double& own) {
  constexpr int NO = Traits<DIM>::NOFF;
  const int c = reg_index<DIM>(rs, i, j, k);
  const int sj = DIM == 3 ? rs.nk : 0, si = DIM == 3 ? rs.nj * rs.nk : rs.nk;
  double As = 0.0;
  if (cls == Traits<DIM>::INTERIOR) {
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
      const double v = src[c + di * si + dj * sj + dk];
      if (o == Traits<DIM>::CENTER) own = v;
      As = fma(op.w[o], v, As);
    }
  } else {
    const double* w = op.tab + cls * (NO + 1);
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      const int di = off_comp(DIM, o, 0), dj = DIM == 3 ? off_comp(DIM, o, 1) : 0, dk = off_comp(DIM, o, DIM - 1);
      const double wo = __ldg(w + o);
      const double v = wo != 0.0 || o == Traits<DIM>::CENTER ? src[c + di * si + dj * sj + dk] : 0.0;
      if (o == Traits<DIM>::CENTER) own = v;
      if (wo != 0.0) As = fma(wo, v, As);
    }
  }
  return As;
}

template <int DIM>
__device__ __forceinline__ double cls_invd(const Op<DIM>& op, int cls) {
  return cls == Traits<DIM>::INTERIOR ? op.invd : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
}

// box origin of this CTA (fine coordinates)
template <int DIM>
__device__ __forceinline__ void box_origin(const Grid& g, int& fi0, int& fj0, int& fk0) {
  using B = MgBox<DIM>;
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
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(MgBox<DIM>::NT) k_mg_down(Grid g, Grid gc, Op<DIM> op, double omega,
                                                            const double* __restrict__ b, double* __restrict__ e2,
                                                            double* __restrict__ bc) {
  PDL_ENTRY();
  using B = MgBox<DIM>;
  extern __shared__ double sm[];
  int fi0, fj0, fk0;
  box_origin<DIM>(g, fi0, fj0, fk0);
  const Reg S = make_reg<DIM>(fi0, fj0, fk0, 3, 0);
  const Reg E = make_reg<DIM>(fi0, fj0, fk0, 2, 0);
  Reg R = make_reg<DIM>(fi0, fj0, fk0, 1, 1);  // [f0-1, f0+F-1]
  double* se1 = sm;                          // |S|
  double* sb = se1 + reg_size<DIM>(S);       // |E|
  double* se2 = sb + reg_size<DIM>(E);       // |E|
  double* sr = se1;                          // |R| overlays e1 after phase 2
  const int tid = threadIdx.x;
  // phase 1: e1 on S, b on E
  for (int e = tid; e < reg_size<DIM>(S); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(S, e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const double bv = __ldg(b + lin_of<DIM>(g, i, j, k));
      v = omega * cls_invd<DIM>(op, class_of<DIM>(g, i, j, k)) * bv;
      const bool inE = i >= E.oi && i < E.oi + E.ni && k >= E.ok && k < E.ok + E.nk &&
                       (DIM == 2 || (j >= E.oj && j < E.oj + E.nj));
      if (inE) sb[reg_index<DIM>(E, i, j, k)] = bv;
    } else {
      const bool inE = i >= E.oi && i < E.oi + E.ni && k >= E.ok && k < E.ok + E.nk &&
                       (DIM == 2 || (j >= E.oj && j < E.oj + E.nj));
      if (inE) sb[reg_index<DIM>(E, i, j, k)] = 0.0;
    }
    se1[e] = v;
  }
  __syncthreads();
  // phase 2: e2 on E ; write e2 for the box F
  for (int e = tid; e < reg_size<DIM>(E); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(E, e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(op, cls, se1, S, i, j, k, own);
      v = own + omega * cls_invd<DIM>(op, cls) * (sb[e] - As);
      const bool inF = i >= fi0 && i < fi0 + B::FI && k >= fk0 && k < fk0 + B::FK &&
                       (DIM == 2 || (j >= fj0 && j < fj0 + B::FJ));
      if (inF) e2[lin_of<DIM>(g, i, j, k)] = v;
    }
    se2[e] = v;
  }
  __syncthreads();
  // phase 3: residual on R
  for (int e = tid; e < reg_size<DIM>(R); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(R, e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(op, cls, se2, E, i, j, k, own);
      v = sb[reg_index<DIM>(E, i, j, k)] - As;
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
    const int c = reg_index<DIM>(R, 2 * Gi, 2 * Gj, 2 * Gk);
    const int sj = DIM == 3 ? R.nk : 0, si = DIM == 3 ? R.nj * R.nk : R.nk;
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
template <int DIM, bool ACC>
__global__ void __launch_bounds__(MgBox<DIM>::NT) k_mg_up(Grid g, Grid gc, Op<DIM> op, double omega,
                                                          const double* __restrict__ b, const double* __restrict__ e2,
                                                          const double* __restrict__ ec, double* __restrict__ out) {
  PDL_ENTRY();
  using B = MgBox<DIM>;
  extern __shared__ double sm[];
  int fi0, fj0, fk0;
  box_origin<DIM>(g, fi0, fj0, fk0);
  const Reg P = make_reg<DIM>(fi0, fj0, fk0, 2, 0);
  const Reg Q = make_reg<DIM>(fi0, fj0, fk0, 1, 0);
  double* sp = sm;
  double* sq = sp + reg_size<DIM>(P);
  double* sbq = sq + reg_size<DIM>(Q);
  const int tid = threadIdx.x;
  for (int e = tid; e < reg_size<DIM>(P); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(P, e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const double t = prolong_at<DIM>(gc, ec, i, j, k);
      v = __ldg(e2 + lin_of<DIM>(g, i, j, k)) + t;
    }
    sp[e] = v;
  }
  for (int e = tid; e < reg_size<DIM>(Q); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(Q, e, i, j, k);
    sbq[e] = in_grid<DIM>(g, i, j, k) ? __ldg(b + lin_of<DIM>(g, i, j, k)) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < reg_size<DIM>(Q); e += B::NT) {
    int i, j, k;
    reg_coords<DIM>(Q, e, i, j, k);
    double v = 0.0;
    if (in_grid<DIM>(g, i, j, k)) {
      const int cls = class_of<DIM>(g, i, j, k);
      double own = 0.0;
      const double As = reg_row<DIM>(op, cls, sp, P, i, j, k, own);
      v = own + omega * cls_invd<DIM>(op, cls) * (sbq[e] - As);
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
    const double As = reg_row<DIM>(op, cls, sq, Q, i, j, k, own);
    const double x = own + omega * cls_invd<DIM>(op, cls) * (sbq[reg_index<DIM>(Q, i, j, k)] - As);
    const uint32_t idx = lin_of<DIM>(g, i, j, k);
    if (ACC) out[idx] = out[idx] + x;
    else out[idx] = x;
  }
}

template <int DIM>
inline unsigned mg_boxes(const Grid& g) {
  using B = MgBox<DIM>;
  return (unsigned)((g.n / B::FK + 1) * (DIM == 3 ? g.n / B::FJ + 1 : 1) * (g.n / B::FI + 1));
}
template <int DIM>
inline size_t mg_down_smem() {
  using B = MgBox<DIM>;
  const size_t s = (size_t)(B::FI + 6) * (DIM == 3 ? B::FJ + 6 : 1) * (B::FK + 6);
  const size_t e = (size_t)(B::FI + 4) * (DIM == 3 ? B::FJ + 4 : 1) * (B::FK + 4);
  return (s + 2 * e) * sizeof(double);
}
template <int DIM>
inline size_t mg_up_smem() {
  using B = MgBox<DIM>;
  const size_t p = (size_t)(B::FI + 4) * (DIM == 3 ? B::FJ + 4 : 1) * (B::FK + 4);
  const size_t q = (size_t)(B::FI + 2) * (DIM == 3 ? B::FJ + 2 : 1) * (B::FK + 2);
  return (p + 2 * q) * sizeof(double);
}

}  // namespace okg
