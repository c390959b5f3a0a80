// okg_tiled.cuh -- 2.5D shared-memory tiled stencil kernels for the large
// multigrid levels (the V-cycle is ~80% of a Newton step).
//
// Why: the naive one-thread-per-vertex gather issues 15 (3D) global loads per
// vertex; the L1/L2 traffic is ~7x the DRAM traffic and boundary vertices
// make whole warps diverge.  Here a CTA owns a (TJ x TK) tile of the (y,z)
// plane of *interior* vertices over TI consecutive x-planes (x is the slowest
// index) and stages the whole (TI+2) x (TJ+2) x (TK+2) operand tile in shared
// memory at once (cp.async, zero-fill outside the box), so every operand value
// is read from L2 about once; each thread then computes its TI vertices along
// x.  Boundary vertices (any coordinate 0 or n, ~6/n of the grid) are handled
// by extra CTAs from a precomputed index list with the per-class weight table.
// (A CTA marching along x through a cp.async ring was built first and measured
// slower; so were persistent TMA-fed versions of these tiles.)
//
// The staging ("loader") step can transform the operand on its way into
// shared memory, which is how two passes are fused away:
//   L_JAC0   stages e1 = w D^-1 r   -> first two damped-Jacobi sweeps in one
//                                      pass (multigrid.hpp:103-104)
//   L_PROLONG stages e + P e_c      -> coarse-grid correction fused into the
//                                      first post-smoothing sweep
//                                      (multigrid.hpp:111-115)
//   L_CHEB0  stages d0 = (D^-1 r)/theta -> the Chebyshev start vector fused into
//                                      the first Chebyshev step (krylov.hpp:178-182)
// In 2D the "plane" is a row segment of TK vertices.
#pragma once
#include <type_traits>

#include "okg_common.cuh"

namespace okg {

template <int DIM>
struct TileCfg;
template <>
struct TileCfg<3> {
  static constexpr int TK = 32, TJ = 8, NT = TK * TJ;
  static constexpr int PW = TK + 2, PH = TJ + 2, PSZ = PW * PH;
  static constexpr int MINB = 4;  // CTAs per SM the register budget must allow (k_tiled)
  static constexpr int MINB_C = 3;  // same for the C-block kernels (okg_tiled_c.cuh)
};
template <>
struct TileCfg<2> {
  static constexpr int TK = 256, TJ = 1, NT = TK * TJ;
  static constexpr int PW = TK + 2, PH = 1, PSZ = PW;
  static constexpr int MINB = 4;
  static constexpr int MINB_C = 4;
};

struct Tiling {
  int32_t ncore;    // core CTAs
  int32_t ktiles, jtiles, ichunk;  // tiles along z, y; planes per CTA along x (= TI)
  int32_t ci0, ci1;  // interior planes [ci0, ci1) of this slab handled by core CTAs
  uint32_t nbnd;    // boundary vertices
  uint32_t vend;    // end of a level vector's index range (owned + ghost planes): 16-byte staging clamps there
  const uint32_t* __restrict__ bnd;  // boundary vertex indices
};

enum TLoad { L_PLAIN = 0, L_JAC0 = 1, L_PROLONG = 2, L_CHEB0 = 3 };
#ifndef OKG_PROLONG_NOSEL  // coarse-tile P e_c without the all-even select (k_tiled)
#define OKG_PROLONG_NOSEL 1
#endif
// (compile-time switches of measured choices; -D...=0 rebuilds the older path for an A/B, tools/experiments)
#ifndef OKG_EDGE_FIRST  // pre-sweep kernel: edge / corner tiles (the slow ones) first in the grid order
#define OKG_EDGE_FIRST 1
#endif
#ifndef OKG_PROLONG_PREGATHER  // thin prolongation tiles: P e_c gathered while the fine tile is in flight
#define OKG_PROLONG_PREGATHER 1
#endif
#ifndef OKG_PROLONG_BND_NB  // boundary vertices of the prolongation-staged sweep: branch-free gather
#define OKG_PROLONG_BND_NB 1
#endif
#ifndef OKG_WIDE_CA  // 16-byte staging through L1 (.ca) instead of L2 only (.cg).  Measured (A/B on one
                     // box): .ca is slower -- residual sweep 11.35 vs 10.68 us at 128^3, 289 vs 270 us at
                     // 400^3, steps 43.6 vs 42.8 ms (128^3), 52.3 vs 51.3 ms (2D); the tiles are read once
#define OKG_WIDE_CA 0
#endif
#ifndef OKG_JAC0_FOLD  // inner JAC0 tiles: scale folded into the taps (see k_tiled)
#define OKG_JAC0_FOLD 1
#endif
#ifndef OKG_FOLD_FACES  // ... and tiles that touch the boundary along one axis only
#define OKG_FOLD_FACES 1
#endif
enum TEpi {
  T_APPLY = 0,       // y = A s
  T_RESID = 1,       // y = b - A s
  T_JACOBI = 2,      // y = s + w D^-1 (b - A s)
  T_JACOBI_SET = 3,  // acc = s + w D^-1 (b - A s)
  T_JACOBI_ACC = 4,  // acc += s + w D^-1 (b - A s)
  T_CHEB = 5         // Chebyshev step (see k_cheb_step)
};

// L_PROLONG: the coarse values P e_c needs for a fine tile of TI planes are
// staged first as a small coarse tile [CI][CJ][CK] (fine tile origin odd or even)
template <int DIM, int TI>
struct CoarseTile {
  static constexpr int CI = TI / 2 + 2;
  static constexpr int CJ = DIM == 3 ? TileCfg<DIM>::TJ / 2 + 2 : 1;
  static constexpr int CK = TileCfg<DIM>::TK / 2 + 2;
  static constexpr int SIZE = CI * CJ * CK;
};

// WIDE: tile rows of PW + 2 doubles staged in 16-byte chunks (see k_tiled)
template <int DIM, int LOAD, int TI, int WIDE = 0>
constexpr size_t tiled_smem_bytes() {
  // (TI >= 4 only: on thin tiles the extra pass costs more than the loads it saves)
  return sizeof(double) * ((size_t)(TI + 2) * (TileCfg<DIM>::PSZ / TileCfg<DIM>::PW) * (TileCfg<DIM>::PW + (WIDE ? 2 : 0)) +
                           (LOAD == 2 && TI >= 4 ? CoarseTile<DIM, TI>::SIZE : 0));
}

struct TArgs {
  const double* x;   // staged operand (x, r, d or e)
  const double* b;   // rhs / r_in
  double* y;         // output / r_out
  double* acc;       // accumulation target / x_out
  const double* x2;  // x_in (cheb) / e_c (prolong)
  double* y2;        // d_out (cheb)
  double omega, c1, c2;
  double inv_theta;  // L_CHEB0: 1 / theta of the Chebyshev start vector
  int32_t last;
  int32_t xmode;     // T_CHEB: 0: x' = x + d'; 1: x untouched this step; 2: x' = (x + d) + d' (the step before was 1)
  Grid gc;           // coarse grid (L_PROLONG)
};

// cp.async (LDGSTS) of one double, zero-filled when !valid (nothing is read)
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}
// 16-byte cp.async (LDGSTS.128) to a shared-window address, zero-filled when !valid
__device__ __forceinline__ void cp_async16(unsigned sdst, const double* gmem, bool valid) {
#if OKG_WIDE_CA
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
#endif
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// class digit of a coordinate
__device__ __forceinline__ int cdig(int v, int n) { return v == 0 ? 0 : (v == n ? 2 : 1); }

template <int DIM>
__device__ __forceinline__ int class_of(const Grid& g, int i, int j, int k) {
  return DIM == 3 ? cdig(i, g.n) * 9 + cdig(j, g.n) * 3 + cdig(k, g.n) : cdig(i, g.n) * 3 + cdig(k, g.n);
}

// prolongation value (P e_c) at fine vertex (i, j, k) (mesh.hpp:169-194)
template <int DIM>
__device__ __forceinline__ double prolong_at(const Grid& gc, const double* __restrict__ ec, int i, int j, int k) {
  const int li = i >> 1, lj = j >> 1, lk = k >> 1;
  const int hi = (i + 1) >> 1, hj = (j + 1) >> 1, hk = (k + 1) >> 1;
  const uint32_t lo = DIM == 3 ? (uint32_t)li * gc.ps + (uint32_t)lj * gc.s + lk : (uint32_t)li * gc.s + lk;
  const uint32_t up = DIM == 3 ? (uint32_t)hi * gc.ps + (uint32_t)hj * gc.s + hk : (uint32_t)hi * gc.s + hk;
#if OKG_PROLONG_NOSEL
  // no branch on lo == up (all-even vertex): fma(0.5, x, 0.5 x) == x exactly for every normal x, and a
  // branch here keeps the loads of different vertices from being in flight together
  return fma(0.5, __ldg(ec + up), 0.5 * __ldg(ec + lo));
#else
  if (lo == up) return __ldg(ec + lo);
  return fma(0.5, __ldg(ec + up), 0.5 * __ldg(ec + lo));
#endif
}

// staged value of vertex (i,j,k) (linear index v)
template <int DIM, int LOAD>
__device__ __forceinline__ double stage_val(const Grid& g, const Op<DIM>& op, const TArgs& a, uint32_t v, int i,
                                            int j, int k) {
  if (LOAD == L_PLAIN) return __ldg(a.x + v);
  if (LOAD == L_JAC0) {
    const int cls = class_of<DIM>(g, i, j, k);
    const double invd =
        cls == Traits<DIM>::INTERIOR ? op.invd : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
    return a.omega * invd * __ldg(a.x + v);
  }
  if (LOAD == L_CHEB0) {  // d0 = (r D^-1) / theta, k_cheb_first's rounding
    const int cls = class_of<DIM>(g, i, j, k);
    const double invd =
        cls == Traits<DIM>::INTERIOR ? op.invd : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
    return (__ldg(a.x + v) * invd) * a.inv_theta;
  }
  // L_PROLONG: e + P e_c  (x + t, t rounded first: multigrid.hpp:111-112)
  const double t = prolong_at<DIM>(a.gc, a.x2, i, j, k);
  return __ldg(a.x + v) + t;
}

// pointwise operands each epilogue needs (prefetched before the barrier)
template <int EPI>
struct EpiNeeds {
  static constexpr bool B = EPI != T_APPLY;
  static constexpr bool P2 = EPI == T_JACOBI_ACC || EPI == T_CHEB;  // acc / x_in
};

template <int DIM, int EPI>
__device__ __forceinline__ void epilogue_pre(const TArgs& a, uint32_t idx, double s_own, double As, double invd,
                                             double bv, double pv) {
  if (EPI == T_APPLY) {
    a.y[idx] = As;
  } else if (EPI == T_RESID) {
    a.y[idx] = bv - As;
  } else if (EPI == T_CHEB) {
    const double r = bv - As;
    const double z = r * invd;
    const double dn = fma(a.c1, s_own, a.c2 * z);
    // x_{k+1} = x_k + d_{k+1} (krylov.hpp:196); every other step leaves x alone and the next one
    // adds both directions in the reference's order, (x + d_k) + d_{k+1} -- d_k is this step's
    // staged operand -- the same bits for 16 B/vertex less on the skipped step
    if (a.xmode != 1) a.acc[idx] = (a.xmode == 2 ? pv + s_own : pv) + dn;
    if (!a.last) {
      a.y2[idx] = dn;
      a.y[idx] = r;
    }
  } else {
    const double e = fma(a.omega * invd, bv - As, s_own);
    if (EPI == T_JACOBI) a.y[idx] = e;
    else if (EPI == T_JACOBI_SET) a.acc[idx] = e;
    else a.acc[idx] = pv + e;
  }
}

// Boundary vertex t of the tiling's list: class-table path (used by the boundary
// CTAs of k_tiled and k_stream)
template <int DIM, int LOAD, int EPI>
__device__ __forceinline__ void boundary_vertex(const Grid& g, const Op<DIM>& op, const Tiling& tl, const TArgs& a,
                                                uint32_t t) {
  constexpr int NO = Traits<DIM>::NOFF;
  if (t >= tl.nbnd) return;
  // everything up to the class weights is static data (written at setup): it is read BEFORE
  // the grid dependency is waited for, in the shadow of the predecessor's completion
  const uint32_t idx = __ldg(tl.bnd + t);
  const Node<DIM> nd = locate<DIM>(g, idx);
  const double* w = op.tab + nd.cls * (NO + 1);
  double As = 0.0, s_own = 0.0;
  if constexpr (LOAD == L_PROLONG) {
    pdl_wait();
    // per-slot loop (each staged value needs the coarse correction; the batched
    // form below costs this kernel 16+ registers and a CTA per SM)
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      int ni = nd.i + off_comp(DIM, o, 0);
      int nj = DIM == 3 ? nd.j + off_comp(DIM, o, 1) : 0;
      int nk = (DIM == 3 ? nd.k : nd.j) + off_comp(DIM, o, DIM - 1);  // fastest coordinate
#if OKG_PROLONG_BND_NB
      // branch-free: a missing neighbour reads the vertex itself with the class row's weight 0, so the
      // gathers of all slots can be in flight together (as far as the register budget lets them).
      // Measured: 128^3 step 41.28 -> 40.96 ms (the 33^3 level's sweep 4.35 -> 3.33 us; skipping the
      // missing slots but not testing the weight: no gain), 2D 49.57 -> 49.48 ms, same bits
      const bool ok = !(ni < 0 || ni > g.n || nk < 0 || nk > g.n || (DIM == 3 && (nj < 0 || nj > g.n)));
      uint32_t v = (uint32_t)((int)idx + g.off[o]);
      if (!ok) {
        ni = nd.i;
        nj = DIM == 3 ? nd.j : 0;
        nk = DIM == 3 ? nd.k : nd.j;
        v = idx;
      }
      const double sv = stage_val<DIM, LOAD>(g, op, a, v, ni, nj, nk);
      if (o == Traits<DIM>::CENTER) s_own = sv;
      As = fma(__ldg(w + o), sv, As);
#else
      if (ni < 0 || ni > g.n || nk < 0 || nk > g.n || (DIM == 3 && (nj < 0 || nj > g.n))) continue;
      const double sv = stage_val<DIM, LOAD>(g, op, a, (uint32_t)((int)idx + g.off[o]), ni, nj, nk);
      if (o == Traits<DIM>::CENTER) s_own = sv;
      const double wo = __ldg(w + o);
      if (wo != 0.0) As = fma(wo, sv, As);
#endif
    }
  } else {
    // branch-free gather (see op_row): every slot loads -- a missing neighbour reads
    // the vertex itself -- and is weighted by the class row (0 for missing slots)
    double wv[NO], sv[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) wv[o] = __ldg(w + o);
    pdl_wait();
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      int ni = nd.i + off_comp(DIM, o, 0);
      int nj = DIM == 3 ? nd.j + off_comp(DIM, o, 1) : 0;
      int nk = (DIM == 3 ? nd.k : nd.j) + off_comp(DIM, o, DIM - 1);  // fastest coordinate
      const bool ok = !(ni < 0 || ni > g.n || nk < 0 || nk > g.n || (DIM == 3 && (nj < 0 || nj > g.n)));
      uint32_t v = (uint32_t)((int)idx + g.off[o]);
      if (!ok) {
        ni = nd.i;
        nj = DIM == 3 ? nd.j : 0;
        nk = DIM == 3 ? nd.k : nd.j;
        v = idx;
      }
      sv[o] = stage_val<DIM, LOAD>(g, op, a, v, ni, nj, nk);
    }
    s_own = sv[Traits<DIM>::CENTER];
#pragma unroll
    for (int o = 0; o < NO; ++o) As = fma(wv[o], sv[o], As);
  }
  const double bv = EpiNeeds<EPI>::B ? a.b[idx] : 0.0;
  const double pv = LOAD == L_CHEB0 ? s_own
                    : EPI == T_CHEB ? (a.xmode == 1 ? 0.0 : a.x2[idx])
                                    : (EPI == T_JACOBI_ACC ? a.acc[idx] : 0.0);
  epilogue_pre<DIM, EPI>(a, idx, s_own, As, __ldg(w + NO), bv, pv);
}

// Core CTAs: a (TI+2) x (TJ+2) x (TK+2) tile (3D) or (TI+2) x (TK+2) (2D) of
// staged values is loaded with all global loads in flight at once, then each
// thread computes TI vertices along x.  Extra CTAs take the boundary list.
//
// WIDE (plain loads only; levels with an odd row pitch s, i.e. every level that coarsens):
// the shared-memory side of the 8-byte LDGSTS staging is a quarter of the L1 data-pipe
// wavefronts that bound these kernels.  A tile row is not 16-byte
// aligned in the reference's vertex order (s odd), so each row of PW doubles is fetched as
// PW/2 + 1 16-byte chunks from its address rounded DOWN to 16 bytes into a row of RP = PW + 2
// doubles: element hk of row (p, hj) then sits at row * RP + par + hk with par = the address
// parity of the row start = a00 ^ ((p + hj) & 1) (s and s^2 odd) -- in the unrolled tap loop a
// compile-time choice between two per-thread base pointers, no instruction per tap.  Half the
// copies, half their shared-memory wavefronts, bit-identical results.
template <int DIM, int LOAD, int EPI, int TI, int WIDE = 0>
__global__ void __launch_bounds__(TileCfg<DIM>::NT, TileCfg<DIM>::MINB) k_tiled(Grid g, Op<DIM> op, Tiling tl, TArgs a) {
  // (griddepcontrol.wait comes after the index arithmetic and the static loads, right before the
  // first access to data the predecessor wrote; the dependent grid is released once the tile is staged)
  // (releasing the dependents of a one-wave grid already at entry measured slower: 128^3 step
  // 44.1 ms for grids <= 592 CTAs, 43.2 ms for <= 296, against 42.4 ms)
  using TC = TileCfg<DIM>;
  static_assert(!(WIDE && LOAD == L_PROLONG && TI < 4), "16-byte staging of the prolongation needs the coarse tile");
  static_assert(!(WIDE && LOAD == L_CHEB0), "the Chebyshev steps keep the 8-byte staging");
  static_assert(LOAD != L_CHEB0 || EPI == T_CHEB, "L_CHEB0 is the first Chebyshev step");
  constexpr int NO = Traits<DIM>::NOFF;
  constexpr int PHT = TC::PSZ / TC::PW;             // rows per staged plane (1 in 2D)
  constexpr int RP = WIDE ? TC::PW + 2 : TC::PW;    // shared-memory row pitch
  constexpr int PSZ = PHT * RP;                     // doubles per staged plane
  const int tid = threadIdx.x;
  // boundary CTAs come first: their gathers are the longest path of the kernel,
  // so they should overlap the core tiles instead of forming its tail
  const int nbb = (int)((tl.nbnd + TC::NT - 1) / TC::NT);
  if ((int)blockIdx.x < nbb) {
    // ---- boundary vertices: class-table path ----
    boundary_vertex<DIM, LOAD, EPI>(g, op, tl, a, blockIdx.x * TC::NT + tid);
    return;
  }
  // ---- core tile ----
  extern __shared__ __align__(16) double tile[];
  int b = (int)blockIdx.x - nbb;
  const int kt = b % tl.ktiles;
  b /= tl.ktiles;
  int jt = DIM == 3 ? b % tl.jtiles : 0;
  int ic = DIM == 3 ? b / tl.jtiles : b;
#if OKG_EDGE_FIRST
  // the tiles on an edge or corner of the box run the staging transform (below) and take about twice as
  // long: they go first (x tiles in the order 0, last, 1, 2, ...; y tiles the same), not into the last wave
  if (LOAD == L_JAC0 || LOAD == L_CHEB0) {
    const int nic = (tl.ci1 - tl.ci0 + TI - 1) / TI;
    ic = ic == 0 ? 0 : ic == 1 ? nic - 1 : ic - 1;
    if (DIM == 3) jt = jt == 0 ? 0 : jt == 1 ? tl.jtiles - 1 : jt - 1;
  }
#endif
  const int k0 = 1 + kt * TC::TK;
  const int j0 = DIM == 3 ? 1 + jt * TC::TJ : 0;
  const int i0 = tl.ci0 + ic * TI;
  const int ni = min(TI, tl.ci1 - i0);  // planes computed by this CTA
  const int tk = tid % TC::TK, tj = tid / TC::TK;
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k <= g.n - 1 && (DIM == 2 || j <= g.n - 1);
  const uint32_t idx0 = DIM == 3 ? (uint32_t)i0 * g.ps + (uint32_t)j * g.s + k : (uint32_t)i0 * g.s + k;
  const uint32_t pstride = DIM == 3 ? g.ps : (uint32_t)g.s;
  // JAC0 on a tile whose halo holds no boundary vertex: one constant scale w D^-1,
  // FOLDED into the taps (x' = wd * x rounds exactly like the staging transform, so
  // the bits are the same) -- the tile keeps the raw rhs, which is also the
  // epilogue's b (a.x == a.b): no transform pass and no prefetch of b
  const bool inner = i0 - 1 >= 1 && i0 + ni <= g.n - 1 && k0 - 1 >= 1 && k0 + TC::TK <= g.n - 1 &&
                     (DIM == 2 || (j0 - 1 >= 1 && j0 + TC::TJ <= g.n - 1));
  // (L_CHEB0 the same way: d0 = (r D^-1)/theta with the constant D^-1 of an inner tile is two
  // multiplies per tap; the raw tile value is the step's r_in, the scaled one its x_in)
  // A tile that touches the boundary along ONE axis only folds as well (OKG_FOLD_FACES): the boundary
  // vertices in its halo are then all of one face class per side, reached only by the taps whose offset
  // component along that axis points at the face -- those taps take the face class' scale from a
  // register (s_m / s_p; a compile-time choice per tap in the sweep specialised for the axis), every
  // other tap the interior one.  Same products, same bits; at 128^3 this folds 88 % of the core tiles
  // instead of 38 %, and all levels below get folded tiles at all (64^3: 0 -> 68 %).
  const bool fi = !(i0 - 1 >= 1 && i0 + ni <= g.n - 1);
  const bool fk = !(k0 - 1 >= 1 && k0 + TC::TK <= g.n - 1);
  const bool fj = DIM == 3 && !(j0 - 1 >= 1 && j0 + TC::TJ <= g.n - 1);
  const int fax = OKG_FOLD_FACES ? ((int)fi + (int)fj + (int)fk <= 1 ? (fi ? 1 : fj ? 2 : fk ? 3 : 0) : -1)
                                 : (inner ? 0 : -1);
  const bool fold = OKG_JAC0_FOLD && (LOAD == L_JAC0 || LOAD == L_CHEB0) && fax >= 0 && a.x == a.b;
  // tap scales of a folded tile (1.0 -- exact -- on a JAC0 tile that is not folded); static data
  double sc0 = 1.0, s_m = 1.0, s_p = 1.0;
  if constexpr (LOAD == L_JAC0 || LOAD == L_CHEB0) {
    if (fold) {
      sc0 = LOAD == L_JAC0 ? a.omega * op.invd : op.invd;
      s_m = s_p = sc0;
      if (fax > 0) {
        const int st = DIM == 3 ? (fax == 1 ? 9 : fax == 2 ? 3 : 1) : (fax == 1 ? 3 : 1);  // class digit stride
        const bool lo = fax == 1 ? i0 - 1 == 0 : fax == 2 ? j - 1 == 0 : k - 1 == 0;
        const bool hi = fax == 1 ? i0 + ni == g.n : fax == 2 ? j + 1 == g.n : k + 1 == g.n;
        const double dl = __ldg(op.tab + (Traits<DIM>::INTERIOR - st) * (NO + 1) + NO);
        const double dh = __ldg(op.tab + (Traits<DIM>::INTERIOR + st) * (NO + 1) + NO);
        if (lo) s_m = LOAD == L_JAC0 ? a.omega * dl : dl;
        if (hi) s_p = LOAD == L_JAC0 ? a.omega * dh : dh;
      }
    }
  }
  pdl_wait();
  // prefetch the pointwise operands of this thread's TI vertices
  double pb[TI], pp[TI];
#pragma unroll
  for (int t = 0; t < TI; ++t) {
    const bool ok = active && t < ni;
    const uint32_t idx = idx0 + (uint32_t)t * pstride;
    pb[t] = (EpiNeeds<EPI>::B && ok && !fold) ? a.b[idx] : 0.0;
    pp[t] = (EpiNeeds<EPI>::P2 && ok && LOAD != L_CHEB0 && !(EPI == T_CHEB && a.xmode == 1))
                ? (EPI == T_CHEB ? a.x2[idx] : a.acc[idx])
                : 0.0;
  }
  // L_PROLONG: coarse tile covering the fine planes/rows/columns of the staged tile
  using CT = CoarseTile<DIM, TI>;
  double* ct = tile + (TI + 2) * PSZ;
  const int cbi = (i0 - 1) >> 1, cbj = DIM == 3 ? (j0 - 1) >> 1 : 0, cbk = (k0 - 1) >> 1;
  constexpr bool CSTAGE = LOAD == L_PROLONG && TI >= 4;
  if (CSTAGE) {
    for (int e = tid; e < CT::SIZE; e += TC::NT) {
      const int ck = e % CT::CK, t = e / CT::CK;
      const int cj = DIM == 3 ? t % CT::CJ : 0, ci = DIM == 3 ? t / CT::CJ : t;
      const int gi = cbi + ci, gj = cbj + cj, gk = cbk + ck;
      const bool in = gi <= a.gc.n && gk <= a.gc.n && (DIM == 2 || gj <= a.gc.n);
      const uint32_t lin = DIM == 3 ? (uint32_t)gi * a.gc.ps + (uint32_t)gj * a.gc.s + gk : (uint32_t)gi * a.gc.s + gk;
      cp_async8(ct + e, a.x2 + lin, in);
    }
    cp_commit();  // its own group: published by a barrier while the fine tile is in flight
  }
  // stage planes i0-1 .. i0+ni: every element by cp.async (LDGSTS, zero-fill outside
  // the box), all in flight at once together with the pointwise prefetch above --
  // no register staging (measured at 400^3: 1.6x the register-batched loop).  The
  // transform below visits in-plane element r = tid + q NT of every plane (offsets
  // computed once, no per-element division).
  constexpr int PER = (TC::PSZ + TC::NT - 1) / TC::NT;
  int qoff[PER], qgj[PER], qgk[PER];
  bool qin[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int r = tid + q * TC::NT;
    const int hj = DIM == 3 ? r / TC::PW : 0;
    const int hk = DIM == 3 ? r - hj * TC::PW : r;
    qgj[q] = DIM == 3 ? j0 - 1 + hj : 0;
    qgk[q] = k0 - 1 + hk;
    qin[q] = r < TC::PSZ && qgk[q] <= g.n && qgj[q] <= g.n;
    qoff[q] = DIM == 3 ? qgj[q] * g.s + qgk[q] : qgk[q];
  }
  // issue order (measured, A/B on one box): per plane for the transformed loads and the
  // Chebyshev step, in linear tile order for the plain sweeps (5 % either way)
  constexpr bool PLANE_ISSUE = LOAD != L_PLAIN || EPI == T_CHEB;
  // (WIDE) linear index of staged element (plane i0-1, row j0-1, column k0-1) and its address parity
  const uint32_t lin0 = (uint32_t)(i0 - 1) * pstride + (DIM == 3 ? (uint32_t)(j0 - 1) * g.s : 0u) + (uint32_t)(k0 - 1);
  const int a00 = WIDE ? (int)((reinterpret_cast<uintptr_t>(a.x + lin0) >> 3) & 1u) : 0;
  // (WIDE) walk this thread's 16-byte chunks in linear order: chunk e = tid + m NT is chunk
  // c = e % CH of row r = e / CH = (plane p, row hj) and lives at tile + 2 e (RP = 2 CH);
  // (p, hj, c) advance incrementally (NT = DR CH + DC, DR = DP PHT + DH: at most one carry each)
  // Kernels with a staging transform in 3D walk plane by plane instead (chunk tid of every
  // plane, 180 of 256 threads): row, column and coarse-tile offsets are then loop invariants of
  // the unrolled plane loop, as in the 8-byte path -- the linear walk's per-chunk index
  // arithmetic made those kernels slower (400^3 prolongation sweep 475 vs 435 us).
  constexpr bool PLANE_WALK = WIDE && LOAD != L_PLAIN && DIM == 3;
  auto walk_chunks = [&](auto&& f) {
    constexpr int CH = RP / 2, DR = TC::NT / CH, DC = TC::NT % CH, DP = DR / PHT, DH = DR % PHT;
    static_assert(!WIDE || (RP % 2 == 0 && DH + 1 <= PHT), "one carry per step");
    if constexpr (PLANE_WALK) {
      constexpr int NCHP = PHT * CH;
      static_assert(!PLANE_WALK || NCHP <= TC::NT, "one chunk per thread and plane");
      if (tid < NCHP) {
        const int hj = tid / CH, c = tid - hj * CH;
#pragma unroll
        for (int p = 0; p < TI + 2; ++p)
          if (p < ni + 2) f(p * NCHP + tid, p, hj, c);
      }
      return;
    }
    const int total = (ni + 2) * PHT * CH;
    int r0 = tid / CH, c = tid - r0 * CH;
    int p = DIM == 3 ? r0 / PHT : r0, hj = DIM == 3 ? r0 - p * PHT : 0;
    for (int e = tid; e < total; e += TC::NT) {
      f(e, p, hj, c);
      c += DC;
      int dr = DR;
      if (c >= CH) {
        c -= CH;
        dr += 1;
      }
      if (DIM == 3) {
        hj += dr - DP * PHT;
        p += DP;
        if (hj >= PHT) {
          hj -= PHT;
          p += 1;
        }
      } else {
        p += dr;
      }
    }
  };
  if constexpr (WIDE) {
    const int jmax = DIM == 3 ? g.n - (j0 - 1) : 0;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(tile));
    walk_chunks([&](int e, int p, int hj, int c) {
      const uint32_t lin = lin0 + (uint32_t)p * pstride + (DIM == 3 ? (uint32_t)hj * (uint32_t)g.s : 0u) + 2u * (uint32_t)c;
      const int par = a00 ^ ((p + hj) & 1);
      const bool ok = hj <= jmax && lin < tl.vend + (uint32_t)par;  // chunk start lin - par inside the vector
      // (pointer arithmetic, not index arithmetic: lin - par wraps for the first element of a vector
      // that starts 8 bytes into a 16-byte chunk, e.g. the w half of a stacked [u; w])
      cp_async16(sbase + (unsigned)e * 16u, ok ? (a.x + lin) - par : (a.x + lin0) - a00, ok);
    });
  } else if (PLANE_ISSUE) {
#pragma unroll
    for (int p = 0; p < TI + 2; ++p) {
      if (p < ni + 2) {
        const uint32_t pb0 = (uint32_t)(i0 - 1 + p) * pstride;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (tid + q * TC::NT < TC::PSZ) cp_async8(tile + p * TC::PSZ + tid + q * TC::NT, a.x + pb0 + qoff[q], qin[q]);
      }
    }
  } else {
    // linear tile order, e = tid + m NT: the tile coordinates (p, hj, hk) and the global
    // offset advance incrementally (NT = DJ PW + DK; at most one carry per coordinate),
    // no per-element division
    const int total = (ni + 2) * TC::PSZ;
    constexpr int PH = TC::PSZ / TC::PW;  // rows per staged plane (1 in 2D)
    constexpr int DJ = TC::NT / TC::PW, DK = TC::NT % TC::PW;
    static_assert(DJ + 1 <= PH || PH == 1, "one carry per step");
    const int rs = DIM == 3 ? g.s : 0;  // global stride of a tile row
    int hk = tid % TC::PW, hj = tid / TC::PW;  // tid < PSZ: plane 0
    const int kmax = g.n - (k0 - 1), jmax = DIM == 3 ? g.n - (j0 - 1) : 0;
    uint32_t lin = (uint32_t)(i0 - 1) * pstride + (DIM == 3 ? (uint32_t)(j0 - 1 + hj) * g.s : 0u) + (k0 - 1 + hk);
    const int dlin = DJ * rs + DK, cjk = rs - TC::PW, cpj = (int)pstride - PH * rs;
    for (int e = tid; e < total; e += TC::NT) {
      cp_async8(tile + e, a.x + lin, hk <= kmax && hj <= jmax);
      hk += DK;
      hj += DJ;
      int d = dlin;
      if (hk >= TC::PW) {
        hk -= TC::PW;
        ++hj;
        d += cjk;
      }
      if (hj >= PH) {
        hj -= PH;
        d += cpj;
      }
      lin += (uint32_t)d;
    }
  }
  cp_commit();
  // thin tiles (no coarse tile): the coarse-grid correction P e_c of this thread's own staged elements is
  // gathered from global memory WHILE the fine tile is in flight, not after it has landed (one memory
  // round trip instead of two on the latency-bound levels these tiles are used on)
  constexpr bool PREGATHER = OKG_PROLONG_PREGATHER && LOAD == L_PROLONG && !CSTAGE && !WIDE;
  double tq[PREGATHER ? (TI + 2) * PER : 1];
  if constexpr (PREGATHER) {
#pragma unroll
    for (int p = 0; p < TI + 2; ++p)
#pragma unroll
      for (int q = 0; q < PER; ++q)
        tq[p * PER + q] = (p < ni + 2 && qin[q]) ? prolong_at<DIM>(a.gc, a.x2, i0 - 1 + p, qgj[q], qgk[q]) : 0.0;
  }
  if (CSTAGE) {
    cp_wait<1>();     // this thread's coarse copies landed ...
    __syncthreads();  // ... and everyone's: the coarse tile is visible
  }
  cp_wait<0>();
  if constexpr (WIDE && LOAD != L_PLAIN) {
    // staging transform on this thread's own chunks (two elements each, 16-byte shared-memory
    // accesses), same arithmetic per element as the 8-byte path below
    if (!fold) {
      constexpr int CSI = CT::CJ * CT::CK, CSJ = CT::CK;
      const double wd = a.omega * op.invd;
      walk_chunks([&](int e, int p, int hj, int c) {
        double2* q = reinterpret_cast<double2*>(tile) + e;
        double2 v = *q;
        const int ip = i0 - 1 + p, gj = DIM == 3 ? j0 - 1 + hj : 0;
        const int gk = k0 - 1 + 2 * c - (a00 ^ ((p + hj) & 1));  // column of the chunk's first element
        if (LOAD == L_JAC0) {
          if (inner) {
            v.x = wd * v.x;
            v.y = wd * v.y;
          } else {
            const int cij = DIM == 3 ? cdig(ip, g.n) * 9 + cdig(gj, g.n) * 3 : cdig(ip, g.n) * 3;
            const int c0 = cij + cdig(gk, g.n), c1 = cij + cdig(gk + 1, g.n);
            const bool rowin = DIM == 2 || gj <= g.n;
            const double d0 = (c0 == Traits<DIM>::INTERIOR || !rowin || gk < 0 || gk > g.n)
                                  ? op.invd
                                  : __ldg(op.tab + c0 * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
            const double d1 = (c1 == Traits<DIM>::INTERIOR || !rowin || gk + 1 > g.n)
                                  ? op.invd
                                  : __ldg(op.tab + c1 * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
            v.x = a.omega * d0 * v.x;
            v.y = a.omega * d1 * v.y;
          }
        } else {
          // e -> e + P e_c from the coarse tile (slots outside the box read junk that is never used)
          const int pl = ((ip >> 1) - cbi) * CSI + (DIM == 3 ? ((gj >> 1) - cbj) * CSJ : 0) - cbk;
          const int pu = (((ip + 1) >> 1) - cbi) * CSI + (DIM == 3 ? (((gj + 1) >> 1) - cbj) * CSJ : 0) - cbk;
          const double t0 = fma(0.5, ct[pu + ((gk + 1) >> 1)], 0.5 * ct[pl + (gk >> 1)]);
          const double t1 = fma(0.5, ct[pu + ((gk + 2) >> 1)], 0.5 * ct[pl + ((gk + 1) >> 1)]);
          v.x = v.x + t0;
          v.y = v.y + t1;
        }
        *q = v;
      });
    }
  } else if (LOAD != L_PLAIN) {
    // the transform touches only this thread's own staged elements (the per-plane
    // issue mapping), so no barrier is needed before it; L_PROLONG reads the coarse
    // tile published above, the fallback path (no coarse tile) reads global memory
    // staging transform:  L_JAC0 r -> (w D^-1) r ;
    //                     L_PROLONG e -> e + P e_c  (x + t, multigrid.hpp:111-112)
    constexpr int CSI = CT::CJ * CT::CK, CSJ = CT::CK;
    const double wd = a.omega * op.invd;
    if (fold) {
      // (scale applied in the taps below)
    } else if ((LOAD == L_JAC0 || LOAD == L_CHEB0) && inner) {
      // branch-free: every slot of this thread (out-of-box / unused slots are never read)
#pragma unroll
      for (int p = 0; p < TI + 2; ++p)
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (q + 1 < PER || tid + q * TC::NT < TC::PSZ) {
            double& v = tile[p * TC::PSZ + tid + q * TC::NT];
            v = LOAD == L_CHEB0 ? (v * op.invd) * a.inv_theta : wd * v;
          }
    } else if (CSTAGE) {
      // coarse-tile offsets of this thread's slots, in-plane part (the plane part per p)
      int cl[PER], cu[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int gj = qgj[q], gk = qgk[q];
        cl[q] = (DIM == 3 ? ((gj >> 1) - cbj) * CSJ : 0) + ((gk >> 1) - cbk);
        cu[q] = (DIM == 3 ? (((gj + 1) >> 1) - cbj) * CSJ : 0) + (((gk + 1) >> 1) - cbk);
      }
#pragma unroll
      for (int p = 0; p < TI + 2; ++p) {
        if (p >= ni + 2) break;  // CTA-uniform
        const int ip = i0 - 1 + p;
        const int pl = ((ip >> 1) - cbi) * CSI, pu = (((ip + 1) >> 1) - cbi) * CSI;
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if (q + 1 < PER || tid + q * TC::NT < TC::PSZ) {
            double& v = tile[p * TC::PSZ + tid + q * TC::NT];
            const int lo = pl + cl[q], up = pu + cu[q];
#if OKG_PROLONG_NOSEL
            // lo == up (all-even vertex): fma(0.5, x, 0.5 x) == x exactly for every normal
            // x, so the select of prolong_at is dropped (only a subnormal coarse value
            // could round differently). A/B: 400^3 427 -> 423 us, 2D 2048^2 step
            // 55.32 -> 55.09 ms, outputs bit-identical (tools/ab_bits.py)
            const double t = fma(0.5, ct[up], 0.5 * ct[lo]);
#else
            const double t = lo == up ? ct[lo] : fma(0.5, ct[up], 0.5 * ct[lo]);
#endif
            v = v + t;
          }
      }
    } else {
      // class digits of this thread's slots (j, k part once; the plane part per p)
      int qcjk[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) qcjk[q] = DIM == 3 ? cdig(qgj[q], g.n) * 3 + cdig(qgk[q], g.n) : cdig(qgk[q], g.n);
#pragma unroll
      for (int p = 0; p < TI + 2; ++p) {
        if (p >= ni + 2) continue;
        const int ip = i0 - 1 + p;
        const int cip = cdig(ip, g.n) * (DIM == 3 ? 9 : 3);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (!qin[q]) continue;
          double& v = tile[p * TC::PSZ + tid + q * TC::NT];
          if (LOAD == L_JAC0) {
            const int cls = cip + qcjk[q];
            const double invd = cls == Traits<DIM>::INTERIOR
                                    ? op.invd
                                    : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
            v = a.omega * invd * v;
          } else if (LOAD == L_CHEB0) {
            const int cls = cip + qcjk[q];
            const double invd = cls == Traits<DIM>::INTERIOR
                                    ? op.invd
                                    : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
            v = (v * invd) * a.inv_theta;
          } else if constexpr (PREGATHER) {
            v = v + tq[p * PER + q];
          } else {
            v = v + prolong_at<DIM>(a.gc, a.x2, ip, qgj[q], qgk[q]);
          }
        }
      }
    }
  }
  __syncthreads();
#if OKG_PDL_TRIGGER == 2
  pdl_trigger();  // operands staged: the dependent grid may start its prologue
#endif
  if (!active) return;
  // all TI vertex chains are computed unconditionally (no branch between them, so
  // their dependent FMA chains interleave); only the stores are predicated
  // this thread's centre column in rows whose (plane + row) parity equals / differs from its
  // own row's: one pointer without WIDE, two (shifted by the rows' address parity) with it
  const int q0 = DIM == 3 ? (tj & 1) : 1;
  const double* tE = tile + (DIM == 3 ? (tj + 1) * RP : 0) + tk + 1 + (WIDE ? (a00 ^ q0) : 0);
  const double* tO = tile + (DIM == 3 ? (tj + 1) * RP : 0) + tk + 1 + (WIDE ? (a00 ^ q0 ^ 1) : 0);
  // AX: the axis along which a folded tile touches the boundary (0 none, 1 x, 2 y, 3 fastest)
  auto sweep = [&](auto AXC) {
    constexpr int AX = decltype(AXC)::value;
#pragma unroll
    for (int t = 0; t < TI; ++t) {
      double As = 0.0, s_own = 0.0, raw_own = 0.0;
      const double sp_t = (AX == 1 && t == ni - 1) ? s_p : sc0;  // x face above: the tile's last plane only
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const int di = off_comp(DIM, o, 0);
        const int dj = DIM == 3 ? off_comp(DIM, o, 1) : 0;
        const int dk = off_comp(DIM, o, DIM - 1);
        const double raw = (((t + di + dj) & 1) ? tO : tE)[(t + 1 + di) * PSZ + (DIM == 3 ? dj * RP : 0) + dk];
        const int da = AX == 1 ? di : AX == 2 ? dj : AX == 3 ? dk : 0;
        const double sct = da < 0 ? ((AX != 1 || t == 0) ? s_m : sc0) : da > 0 ? (AX == 1 ? sp_t : s_p) : sc0;
        const double sv = (OKG_JAC0_FOLD && LOAD == L_JAC0) ? sct * raw
                          : (LOAD == L_CHEB0 && fold)       ? (raw * sct) * a.inv_theta
                                                             : raw;
        if (o == Traits<DIM>::CENTER) {
          s_own = sv;
          raw_own = raw;
        }
        As = fma(op.w[o], sv, As);
      }
      if (t < ni)
        epilogue_pre<DIM, EPI>(a, idx0 + (uint32_t)t * pstride, s_own, As, op.invd, fold ? raw_own : pb[t],
                               LOAD == L_CHEB0 ? s_own : pp[t]);
    }
  };
  if constexpr (OKG_FOLD_FACES && (LOAD == L_JAC0 || LOAD == L_CHEB0)) {
    if (fax <= 0) sweep(std::integral_constant<int, 0>{});
    else if (fax == 1) sweep(std::integral_constant<int, 1>{});
    else if (DIM == 3 && fax == 2) sweep(std::integral_constant<int, 2>{});
    else sweep(std::integral_constant<int, 3>{});
  } else {
    sweep(std::integral_constant<int, 0>{});
  }
}

}  // namespace okg

