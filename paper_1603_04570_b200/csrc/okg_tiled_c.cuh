// okg_tiled_c.cuh -- tiled kernels for the u-dependent C = -eps^2 K - M_E(u)
// block: apply_C, r2 - C du, the Schur action and the fused block Jacobian
// (precond.hpp:210-298).  Same tile geometry as okg_tiled.cuh.
#pragma once
#include "okg_tiled.cuh"

namespace okg {

// ---------------------------------------------------------------------------
// Tiled C-block kernels (apply_C / apply_schur / jacobian, precond.hpp:210-298)
// The operands x (C operand) and v (second operand) are staged like above;
// the coefficients of C = -eps^2 K - M_E(u) are read straight from global
// memory: the diagonal and positive slots at the vertex, each negative slot q
// from array q at the single shifted position idx - off_q (coalesced).
// ---------------------------------------------------------------------------
struct CTArgs {
  const double* x;   // C operand
  const double* v;   // second operand (JAC: dw, SCHUR: v)
  const double* b;   // rhs (SUB / SCHUR_RES / JAC_RES: stacked)
  double* y;         // output (JAC: stacked)
  const double* coef;
  size_t ldc;
  size_t n2;         // w-block offset in stacked vectors
  double s1;         // SCHUR: c ; JAC: dt*theta ; ME: eps^2
};

enum TCMode { TC_C = 0, TC_SUB = 1, TC_ME = 2, TC_SCHUR = 3, TC_SCHUR_RES = 4, TC_JAC = 5, TC_JAC_RES = 6 };

template <int MODE>
struct CNeeds {
  static constexpr bool V = MODE == TC_SCHUR || MODE == TC_SCHUR_RES || MODE == TC_JAC || MODE == TC_JAC_RES;
  static constexpr int NOPS = V ? 2 : 1;
  static constexpr bool B = MODE == TC_SUB || MODE == TC_SCHUR_RES || MODE == TC_JAC_RES;
};

// coefficient of C for stencil slot o at vertex idx
template <int DIM>
__device__ __forceinline__ double c_coef(const CTArgs& a, uint32_t idx, int off, int o) {
  constexpr int C = Traits<DIM>::CENTER;
  return o < C ? __ldg(a.coef + (size_t)(C - o) * a.ldc + (uint32_t)((int)idx + off))
               : __ldg(a.coef + (size_t)(o - C) * a.ldc + idx);
}

// y-part of one vertex given the staged rows (xs[o], vs[o]) and slot validity
template <int DIM, int MODE>
__device__ __forceinline__ void c_vertex(const Grid& g, const Op<DIM>& Mop, const Op<DIM>& Kop,
                                         const Op<DIM>& Aop, const CTArgs& a, uint32_t idx, int cls,
                                         const double (&xs)[Traits<DIM>::NOFF], const double (&vs)[Traits<DIM>::NOFF],
                                         double b1, double b2, double& nrm) {
  constexpr int NO = Traits<DIM>::NOFF;
  const bool inter = cls == Traits<DIM>::INTERIOR;
  double cx = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
  // all coefficients first (a missing slot reads the vertex's own array entry; its
  // operand xs/vs is 0), so the loads are not serialised behind the FMA chain
  double cf[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) cf[o] = c_coef<DIM>(a, idx, (inter || slot_ok<DIM>(cls, o)) ? g.off[o] : 0, o);
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    cx = fma(cf[o], xs[o], cx);
    if (MODE == TC_ME) {
      const double kw = inter ? Kop.w[o] : __ldg(Kop.tab + cls * (NO + 1) + o);
      t1 = fma(kw, xs[o], t1);
    }
    if (MODE == TC_SCHUR || MODE == TC_SCHUR_RES) {
      const double mw = inter ? Mop.w[o] : __ldg(Mop.tab + cls * (NO + 1) + o);
      t1 = fma(mw, vs[o], t1);
    }
    if (MODE == TC_JAC || MODE == TC_JAC_RES) {
      const double aw = inter ? Aop.w[o] : __ldg(Aop.tab + cls * (NO + 1) + o);
      const double kw = inter ? Kop.w[o] : __ldg(Kop.tab + cls * (NO + 1) + o);
      const double mw = inter ? Mop.w[o] : __ldg(Mop.tab + cls * (NO + 1) + o);
      t1 = fma(aw, xs[o], t1);
      t2 = fma(kw, vs[o], t2);
      t3 = fma(mw, vs[o], t3);
    }
  }
  if (MODE == TC_C) a.y[idx] = cx;
  else if (MODE == TC_SUB) a.y[idx] = b1 - cx;
  else if (MODE == TC_ME) a.y[idx] = -cx - a.s1 * t1;
  else if (MODE == TC_SCHUR || MODE == TC_SCHUR_RES) {
    const double s = t1 - a.s1 * cx;
    a.y[idx] = MODE == TC_SCHUR ? s : b1 - s;
  } else {
    const double y1 = t1 + a.s1 * t2;
    const double y2 = cx + t3;
    if (MODE == TC_JAC) {
      a.y[idx] = y1;
      a.y[a.n2 + idx] = y2;
    } else {
      const double r1 = b1 - y1, r2 = b2 - y2;
      a.y[idx] = r1;
      a.y[a.n2 + idx] = r2;
      nrm += r1 * r1 + r2 * r2;
    }
  }
}

template <int DIM, int MODE, int TI>
__global__ void __launch_bounds__(TileCfg<DIM>::NT, TileCfg<DIM>::MINB_C) k_tiled_c(Grid g, Op<DIM> Mop, Op<DIM> Kop, Op<DIM> Aop,
                                                              Tiling tl, CTArgs a, Reduce red) {
  pdl_wait();  // (the dependent grid is released below, once the tile is staged)
  using TC = TileCfg<DIM>;
  constexpr int NO = Traits<DIM>::NOFF;
  constexpr int NOPS = CNeeds<MODE>::NOPS;
  const int tid = threadIdx.x;
  double nrm[1] = {0.0};
  extern __shared__ double tile[];
  const int nbb = (int)((tl.nbnd + TC::NT - 1) / TC::NT);  // boundary CTAs first (see k_tiled)
  if ((int)blockIdx.x < nbb) {
    const uint32_t t = blockIdx.x * TC::NT + tid;
    if (t < tl.nbnd) {
      const uint32_t idx = __ldg(tl.bnd + t);
      const Node<DIM> nd = locate<DIM>(g, idx);
      double xs[NO], vs[NO];
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const bool ok = slot_ok<DIM>(nd.cls, o);
        const uint32_t v = (uint32_t)((int)idx + g.off[o]);
        xs[o] = ok ? __ldg(a.x + v) : 0.0;
        vs[o] = (CNeeds<MODE>::V && ok) ? __ldg(a.v + v) : 0.0;
      }
      const double b1 = CNeeds<MODE>::B ? a.b[idx] : 0.0;
      const double b2 = MODE == TC_JAC_RES ? a.b[a.n2 + idx] : 0.0;
      c_vertex<DIM, MODE>(g, Mop, Kop, Aop, a, idx, nd.cls, xs, vs, b1, b2, nrm[0]);
    }
  } else {
    int bb = (int)blockIdx.x - nbb;
    const int kt = bb % tl.ktiles;
    bb /= tl.ktiles;
    const int jt = DIM == 3 ? bb % tl.jtiles : 0;
    const int ic = DIM == 3 ? bb / tl.jtiles : bb;
    const int k0 = 1 + kt * TC::TK;
    const int j0 = DIM == 3 ? 1 + jt * TC::TJ : 0;
    const int i0 = tl.ci0 + ic * TI;
    const int ni = min(TI, tl.ci1 - i0);
    const int tk = tid % TC::TK, tj = tid / TC::TK;
    const int k = k0 + tk, j = j0 + tj;
    const bool active = k <= g.n - 1 && (DIM == 2 || j <= g.n - 1);
    const uint32_t idx0 = DIM == 3 ? (uint32_t)i0 * g.ps + (uint32_t)j * g.s + k : (uint32_t)i0 * g.s + k;
    const uint32_t pstride = DIM == 3 ? g.ps : (uint32_t)g.s;
    double pb1[TI], pb2[TI];
#pragma unroll
    for (int t = 0; t < TI; ++t) {
      const bool ok = active && t < ni;
      const uint32_t idx = idx0 + (uint32_t)t * pstride;
      pb1[t] = (CNeeds<MODE>::B && ok) ? a.b[idx] : 0.0;
      pb2[t] = (MODE == TC_JAC_RES && ok) ? a.b[a.n2 + idx] : 0.0;
    }
    // operand tiles by cp.async (zero-fill outside the box), all copies in flight at once
    const int per = (TI + 2) * TC::PSZ;
    const int tot1 = (ni + 2) * TC::PSZ;
#pragma unroll
    for (int op = 0; op < NOPS; ++op) {
      const double* src = op ? a.v : a.x;
      for (int e = tid; e < tot1; e += TC::NT) {
        const int p = e / TC::PSZ;
        const int r = e - p * TC::PSZ;
        const int hj = DIM == 3 ? r / TC::PW : 0;
        const int hk = DIM == 3 ? r - hj * TC::PW : r;
        const int gj = DIM == 3 ? j0 - 1 + hj : 0;
        const int gk = k0 - 1 + hk;
        const uint32_t lin = (uint32_t)(i0 - 1 + p) * pstride + (DIM == 3 ? (uint32_t)gj * g.s : 0u) + gk;
        cp_async8(tile + op * per + e, src + lin, gk <= g.n && gj <= g.n);
      }
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
#if OKG_PDL_TRIGGER == 2
    pdl_trigger();  // operands staged: the dependent grid may start its prologue
#endif
    if (active) {
#pragma unroll
      for (int t = 0; t < TI; ++t) {
        if (t >= ni) continue;
        double xs[NO], vs[NO];
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          const int di = off_comp(DIM, o, 0);
          const int dj = DIM == 3 ? off_comp(DIM, o, 1) : 0;
          const int dk = off_comp(DIM, o, DIM - 1);
          const int sidx = (t + 1 + di) * TC::PSZ + (DIM == 3 ? (tj + 1 + dj) * TC::PW : 0) + tk + 1 + dk;
          xs[o] = tile[sidx];
          vs[o] = CNeeds<MODE>::V ? tile[per + sidx] : 0.0;
        }
        c_vertex<DIM, MODE>(g, Mop, Kop, Aop, a, idx0 + (uint32_t)t * pstride, Traits<DIM>::INTERIOR, xs, vs,
                            pb1[t], pb2[t], nrm[0]);
      }
    }
  }
  if (MODE == TC_JAC_RES) grid_reduce<1>(nrm, red);
}

}  // namespace okg
