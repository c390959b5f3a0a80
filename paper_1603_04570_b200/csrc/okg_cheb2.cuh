// okg_cheb2.cuh -- two Chebyshev steps in one pass (2D), chebyshev_semi_iteration
// (krylov.hpp:158-202):
//   step a:  r1 = r - A d ;  d1 = c1a d + c2a D^-1 r1 ;  x1 = x + d1
//   step b:  r2 = r1 - A d1 ; d2 = c1b d1 + c2b D^-1 r2 ; x2 = x1 + d2
// A core tile stages d with a 2-vertex halo and r with a 1-vertex halo, computes
// step a on the tile + 1-vertex ring into shared memory (d1, r1 never reach global
// memory) and step b on the tile: 7.5 instead of 12 N-vector passes per two steps
// (the 2D Chebyshev steps are DRAM-bound: 34 MB vectors at 2048^2).  Boundary
// vertices (0.2% in 2D) are done by extra CTAs that recompute step a on their
// 1-ring.  Every value is the single-step kernels' expression in the same order,
// so results equal two T_CHEB launches (up to the sign of a zero).
#pragma once
#include "okg_tiled.cuh"

namespace okg {

struct Cheb2Args {
  const double* d;   // d_j (halo 2)
  const double* r;   // r_j (halo 1); r_0 = b
  const double* x;   // x_j at the vertex (x_1 = d_0 on the first pair)
  double* d_out;     // d_{j+2}   (unless last)
  double* r_out;     // r_{j+2}   (unless last; never aliases r)
  double* x_out;     // x_{j+2}
  double c1a, c2a, c1b, c2b;
  int32_t last;      // the second step is the iteration's last: only x is written
};

template <int TI>
constexpr size_t cheb2_smem_bytes() {
  constexpr int TK = TileCfg<2>::TK;
  return sizeof(double) * ((size_t)(TI + 4) * (TK + 4) + 2 * (size_t)(TI + 2) * (TK + 2));
}

// class of a 2D vertex and its operator row weight / inverse diagonal
__device__ __forceinline__ int cls2(int i, int k, int n) { return cdig(i, n) * 3 + cdig(k, n); }

template <int TI>
__global__ void __launch_bounds__(TileCfg<2>::NT) k_cheb2(Grid g, Op<2> op, Tiling tl, Cheb2Args a) {
  PDL_ENTRY();
  constexpr int NO = Traits<2>::NOFF, TK = TileCfg<2>::TK, NT = TileCfg<2>::NT;
  const int tid = threadIdx.x;
  const int n = g.n;
  const int nbb = (int)((tl.nbnd + NT - 1) / NT);  // boundary CTAs first (see k_tiled)
  if ((int)blockIdx.x < nbb) {
    // ---- boundary vertex: step a on its 1-ring, then step b ----
    const uint32_t t = blockIdx.x * NT + tid;
    if (t >= tl.nbnd) return;
    const uint32_t idx = __ldg(tl.bnd + t);
    const int vi = (int)(idx / (uint32_t)g.s), vk = (int)(idx - (uint32_t)vi * g.s);
    double d1[NO], r1c = 0.0;
#pragma unroll
    for (int q = 0; q < NO; ++q) {  // the ring point u = v + off_q (step a needs d around u)
      const int ui = vi + off_comp(2, q, 0), uk = vk + off_comp(2, q, 1);
      d1[q] = 0.0;
      if (ui < 0 || ui > n || uk < 0 || uk > n) continue;
      const uint32_t u = (uint32_t)((int)idx + g.off[q]);
      const int cu = cls2(ui, uk, n);
      const double* w = op.tab + cu * (NO + 1);
      double dv[NO], wv[NO];
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const int pi = ui + off_comp(2, o, 0), pk = uk + off_comp(2, o, 1);
        const bool ok = pi >= 0 && pi <= n && pk >= 0 && pk <= n;
        wv[o] = cu == Traits<2>::INTERIOR ? op.w[o] : __ldg(w + o);
        dv[o] = __ldg(a.d + (ok ? (int)u + g.off[o] : (int)u));
      }
      double As = 0.0;
#pragma unroll
      for (int o = 0; o < NO; ++o) As = fma(wv[o], dv[o], As);
      const double invd = cu == Traits<2>::INTERIOR ? op.invd : __ldg(w + NO);
      const double r1 = __ldg(a.r + u) - As;
      d1[q] = fma(a.c1a, dv[Traits<2>::CENTER], a.c2a * (r1 * invd));
      if (q == Traits<2>::CENTER) r1c = r1;
    }
    const int cv = cls2(vi, vk, n);
    const double* wv = op.tab + cv * (NO + 1);
    double As = 0.0;
#pragma unroll
    for (int o = 0; o < NO; ++o) As = fma(__ldg(wv + o), d1[o], As);
    const double r2 = r1c - As;
    const double d2 = fma(a.c1b, d1[Traits<2>::CENTER], a.c2b * (r2 * __ldg(wv + NO)));
    a.x_out[idx] = (a.x[idx] + d1[Traits<2>::CENTER]) + d2;
    if (!a.last) {
      a.d_out[idx] = d2;
      a.r_out[idx] = r2;
    }
    return;
  }
  // ---- core tile: rows [i0, i0+ni), columns [k0, k0+TK) of interior vertices ----
  extern __shared__ double sm[];
  constexpr int SW = TK + 4, QW = TK + 2;
  double* sd = sm;                        // d on rows i0-2 .. i0+ni+1, cols k0-2 .. k0+TK+1
  double* sr;                              // r, then r1, on the 1-ring region (right after d)
  double* s1;                              // d1 on the 1-ring region
  const int cb = (int)blockIdx.x - nbb;
  const int kt = cb % tl.ktiles;
  const int ic = cb / tl.ktiles;
  const int k0 = 1 + kt * TK;
  const int i0 = tl.ci0 + ic * TI;
  const int ni = min(TI, tl.ci1 - i0);
  sr = sd + (ni + 4) * SW;
  s1 = sr + (ni + 2) * QW;
  // stage d (halo 2) and r (halo 1), zero outside the grid; U loads in flight per thread
  constexpr int U = 8;
  const int nd_ = (ni + 4) * SW, nr_ = (ni + 2) * QW, tot = nd_ + nr_;
  for (int base = tid; base < tot; base += NT * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      v[u] = 0.0;
      if (e < tot) {
        const bool isd = e < nd_;
        const int ee = isd ? e : e - nd_;
        const int W = isd ? SW : QW, h = isd ? 2 : 1;
        const int p = ee / W, c = ee - p * W;
        const int gi = i0 - h + p, gk = k0 - h + c;
        if (gi >= 0 && gi <= n && gk >= 0 && gk <= n) v[u] = __ldg((isd ? a.d : a.r) + (uint32_t)gi * g.s + gk);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      if (e < tot) sm[e] = v[u];  // sd and sr are contiguous
    }
  }
  __syncthreads();
  // step a on the 1-ring region (boundary vertices on it use their class rows)
  for (int e = tid; e < (ni + 2) * QW; e += NT) {
    const int p = e / QW, c = e - p * QW;
    const int gi = i0 - 1 + p, gk = k0 - 1 + c;
    double d1 = 0.0, r1 = 0.0;
    if (gi >= 0 && gi <= n && gk >= 0 && gk <= n) {
      const int cu = cls2(gi, gk, n);
      const double* sp = sd + (p + 1) * SW + (c + 1);  // this point in the d tile
      double As = 0.0;
      if (cu == Traits<2>::INTERIOR) {
#pragma unroll
        for (int o = 0; o < NO; ++o) As = fma(op.w[o], sp[off_comp(2, o, 0) * SW + off_comp(2, o, 1)], As);
      } else {
        const double* w = op.tab + cu * (NO + 1);
#pragma unroll
        for (int o = 0; o < NO; ++o) As = fma(__ldg(w + o), sp[off_comp(2, o, 0) * SW + off_comp(2, o, 1)], As);
      }
      const double invd = cu == Traits<2>::INTERIOR ? op.invd : __ldg(op.tab + cu * (NO + 1) + NO);
      r1 = sr[e] - As;
      d1 = fma(a.c1a, sp[0], a.c2a * (r1 * invd));
    }
    sr[e] = r1;
    s1[e] = d1;
  }
  __syncthreads();
  // step b on the tile (interior vertices)
  for (int e = tid; e < ni * TK; e += NT) {
    const int p = e / TK, c = e - p * TK;
    const int gi = i0 + p, gk = k0 + c;
    if (gk > n - 1) continue;
    const int q = (p + 1) * QW + (c + 1);
    double As = 0.0;
#pragma unroll
    for (int o = 0; o < NO; ++o) As = fma(op.w[o], s1[q + off_comp(2, o, 0) * QW + off_comp(2, o, 1)], As);
    const double r2 = sr[q] - As;
    const double d2 = fma(a.c1b, s1[q], a.c2b * (r2 * op.invd));
    const uint32_t idx = (uint32_t)gi * g.s + gk;
    a.x_out[idx] = (a.x[idx] + s1[q]) + d2;
    if (!a.last) {
      a.d_out[idx] = d2;
      a.r_out[idx] = r2;
    }
  }
}

}  // namespace okg
