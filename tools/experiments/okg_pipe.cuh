// okg_pipe.cuh -- persistent, TMA-fed version of the 2.5D tiled stencil kernels
// (okg_tiled.cuh) for the large multigrid levels.
//
// k_tiled spends more than half of its instructions on staging: ~1.66 8-byte
// LDGSTS per vertex, each with its own address/predicate arithmetic, and a grid
// of one-tile CTAs pays the load latency once per tile (2.4 waves at 128^3).
// Here a CTA is persistent (PIPE_CPS per SM, grid = 148 x PIPE_CPS) and walks a
// static round-robin list of work items; the operand tile of the NEXT item is
// in flight (TMA bulk copies into the other shared-memory stage, completion on
// an mbarrier) while the current one is computed, and the pointwise operands of
// the next item are prefetched into registers.
//
// Staging without a tensor map: the reference's vertex order has row pitch
// s = n + 1 doubles (odd for every level that coarsens), which is not a
// multiple of 16 bytes, so cuTensorMapEncodeTiled cannot describe a level
// vector.  Every tile row (PW doubles, 16-byte aligned only for every other
// row) is instead fetched by one 1D bulk copy (cp.async.bulk, SASS UBLKCP) of
// RP = PW + 2 doubles starting at the row's address rounded DOWN to 16 bytes:
// element hk of row (p, hj) then sits at shared offset row * RP + a(p, hj) + hk
// with a(p, hj) = address parity of the row start.  For odd s that parity is a
// checkerboard in (p + hj), so in the unrolled stencil loop it is a compile-time
// choice between two per-thread base pointers -- no extra instruction per tap.
// One thread issues one row (100 rows of a 3D tile, 10 of a 2D one).
//
// Values outside the box are never zero-filled: they only feed vertices that
// are not stored (the tile computes interior vertices 1..n-1, whose 1-ring is
// inside the box), and the bytes a row copy reads past the row end are the next
// row's (clamped at the end of the vector, see row_count).
#pragma once
#include "okg_tiled.cuh"

namespace okg {

#ifndef OKG_PIPE_BULK
#define OKG_PIPE_BULK -1  // -1: by dimension (see PipeCfg), 0: never, 1: always
#endif
#ifndef OKG_PIPE_CA
#define OKG_PIPE_CA 0  // 16-byte cp.async through L1 (.ca) or L2 only (.cg)
#endif
#ifndef OKG_PIPE_NSTAGE
#define OKG_PIPE_NSTAGE 2  // shared-memory stages per CTA (1: no prefetch of the next tile)
#endif
#ifndef OKG_PIPE_CPS
#define OKG_PIPE_CPS 2  // persistent CTAs per SM
#endif

template <int DIM, int TI>
struct PipeCfg {
  using TC = TileCfg<DIM>;
  static constexpr int PH = TC::PSZ / TC::PW;  // rows per staged plane (1 in 2D)
  static constexpr int RP = TC::PW + 2;        // shared row pitch (doubles): room for the parity shift
  static constexpr int ROWS = (TI + 2) * PH;   // rows per stage
  static constexpr int PLANE = PH * RP;        // doubles per staged plane
  static constexpr int FINE = ROWS * RP;       // doubles of the fine tile
  static constexpr int NSTAGE = OKG_PIPE_NSTAGE;
  // rows by one cp.async.bulk each (2D: 2 KB rows run at full TMA rate) or by 16-byte
  // cp.async chunks (3D: 288-byte bulk requests are bound by the TMA unit's request rate,
  // ~33 cycles each per SM -- 2.5 TB/s chip-wide against 6.1 TB/s for LDGSTS.128,
  // tools/tma_bench.cu)
  static constexpr bool BULK = OKG_PIPE_BULK >= 0 ? OKG_PIPE_BULK != 0 : DIM == 2;
  static_assert(ROWS <= TC::NT, "one row copy per thread");
  static_assert((RP * 8) % 16 == 0, "row pitch must keep 16-byte alignment");
};

template <int DIM, int LOAD, int TI>
constexpr size_t pipe_stage_doubles() {
  return (size_t)PipeCfg<DIM, TI>::FINE + (LOAD == L_PROLONG ? (CoarseTile<DIM, TI>::SIZE + 1) / 2 * 2 : 0);
}
template <int DIM, int LOAD, int TI>
constexpr size_t pipe_smem_bytes() {
  return sizeof(double) * PipeCfg<DIM, TI>::NSTAGE * pipe_stage_doubles<DIM, LOAD, TI>();
}

// ---- mbarrier / bulk-copy primitives (PTX, sm_90+) --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once every cp.async this thread issued so far has landed (counts as the thread's arrival)
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 16-byte cp.async (LDGSTS.128), zero-filled when !valid (nothing is read)
__device__ __forceinline__ void cp_async16(uint32_t sdst, const double* gmem, bool valid) {
#if OKG_PIPE_CA
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
#endif
}
// generic-proxy writes to a stage (the staging transforms) ordered before the next bulk copy into it
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One work item of the tile list.
template <int DIM, int TI>
struct PipeTile {
  int i0, j0, k0, ni;
  uint32_t lin0;  // linear index of staged element (plane i0-1, row j0-1, column k0-1)
  __device__ __forceinline__ void decode(const Tiling& tl, const Grid& g, int b) {
    using TC = TileCfg<DIM>;
    const int kt = b % tl.ktiles;
    b /= tl.ktiles;
    const int jt = DIM == 3 ? b % tl.jtiles : 0;
    const int ic = DIM == 3 ? b / tl.jtiles : b;
    k0 = 1 + kt * TC::TK;
    j0 = DIM == 3 ? 1 + jt * TC::TJ : 0;
    i0 = tl.ci0 + ic * TI;
    ni = min(TI, tl.ci1 - i0);
    lin0 = DIM == 3 ? (uint32_t)(i0 - 1) * g.ps + (uint32_t)(j0 - 1) * g.s + (uint32_t)(k0 - 1)
                    : (uint32_t)(i0 - 1) * g.s + (uint32_t)(k0 - 1);
  }
};

// Persistent kernel: items [0, nbb) are chunks of the boundary list (class-table
// gathers, as in k_tiled), items [nbb, nbb + ncore) the core tiles.  CTA c takes
// items c, c + G, c + 2G, ...
template <int DIM, int LOAD, int EPI, int TI>
__global__ void __launch_bounds__(TileCfg<DIM>::NT, OKG_PIPE_CPS) k_pipe(Grid g, Op<DIM> op, Tiling tl, TArgs a) {
  using TC = TileCfg<DIM>;
  using PC = PipeCfg<DIM, TI>;
  using CT = CoarseTile<DIM, TI>;
  constexpr int NO = Traits<DIM>::NOFF;
  constexpr int SD = (int)pipe_stage_doubles<DIM, LOAD, TI>();
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[PC::NSTAGE];
  const int tid = threadIdx.x;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < PC::NSTAGE; ++s) mbar_init(&bar[s], TC::NT);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
#if OKG_PDL_TRIGGER != 0
  if (PC::NSTAGE > 1) pdl_trigger();  // a persistent grid is one wave: its dependents can only take the slots it frees
#endif
  const int G = (int)gridDim.x;
  const int nbb = (int)((tl.nbnd + TC::NT - 1) / TC::NT);
  const int total = nbb + tl.ncore;
  const uint32_t pstride = DIM == 3 ? g.ps : (uint32_t)g.s;
  const int sodd = g.s & 1;
  const int tk = tid % TC::TK, tj = tid / TC::TK;

  // ---- issue the operand tile of item `it` into stage st (every thread arrives once) ----
  auto issue = [&](const PipeTile<DIM, TI>& T, int st) {
    double* fine = sm + st * SD;
    if constexpr (PC::BULK) {
      if (tid < PC::ROWS) {
        const int p = DIM == 3 ? tid / PC::PH : tid;
        const int hj = DIM == 3 ? tid - p * PC::PH : 0;
        const int gj = T.j0 - 1 + hj;
        if (p < T.ni + 2 && gj <= g.n) {
          const uint32_t lin = T.lin0 + (uint32_t)p * pstride + (DIM == 3 ? (uint32_t)hj * (uint32_t)g.s : 0u);
          const double* src = a.x + lin;
          const uint32_t par = (uint32_t)(reinterpret_cast<uintptr_t>(src) >> 3) & 1u;
          // doubles to copy: the whole padded row, clamped at the end of the vector (rounded
          // up to the 16-byte chunk the last element lives in)
          const uint32_t left = tl.vend - (lin - par);
          const uint32_t cnt = min((uint32_t)PC::RP, (left + 1u) & ~1u);
          mbar_expect_tx(&bar[st], cnt * 8u);
          bulk_g2s(fine + tid * PC::RP, src - par, cnt * 8u, &bar[st]);
        }
      }
    } else {
      // 16-byte cp.async (LDGSTS.128): chunk e = tid + m NT of the stage is chunk c = e % CH of
      // row r = e / CH and lands at fine + 2 e (RP = 2 CH); the row/plane coordinates advance
      // incrementally (NT = DR CH + DC, DR = DP PH + DH: at most one carry each)
      constexpr int CH = PC::RP / 2, NCH = PC::ROWS * CH;
      constexpr int DR = TC::NT / CH, DC = TC::NT % CH, DP = DR / PC::PH, DH = DR % PC::PH;
      constexpr int M = (NCH + TC::NT - 1) / TC::NT;
      const int a00 = (int)((reinterpret_cast<uintptr_t>(a.x + T.lin0) >> 3) & 1u);
      int r = tid / CH, c = tid - r * CH;
      int p = DIM == 3 ? r / PC::PH : r, hj = DIM == 3 ? r - p * PC::PH : 0;
      const int jmax = DIM == 3 ? g.n - (T.j0 - 1) : 0, pmax = T.ni + 1;
      const uint32_t sdst = smem_u32(fine) + (uint32_t)tid * 16u;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if (m + 1 < M || tid + m * TC::NT < NCH) {
          const uint32_t lin =
              T.lin0 + (uint32_t)p * pstride + (DIM == 3 ? (uint32_t)hj * (uint32_t)g.s : 0u) + 2u * (uint32_t)c;
          const uint32_t par = (uint32_t)(a00 ^ ((p + hj) & sodd));
          const bool ok = p <= pmax && hj <= jmax && lin < tl.vend + par;  // chunk start lin - par inside the vector
          cp_async16(sdst + (uint32_t)m * (TC::NT * 16u), a.x + (ok ? lin - par : T.lin0 - a00), ok);
        }
        c += DC;
        r = DR;
        if (c >= CH) {
          c -= CH;
          r += 1;
        }
        if (DIM == 3) {
          hj += r - DP * PC::PH;
          p += DP;
          if (hj >= PC::PH) {
            hj -= PC::PH;
            p += 1;
          }
        } else {
          p += r;
        }
      }
    }
    if constexpr (LOAD == L_PROLONG) {
      // coarse tile covering the fine tile's planes/rows/columns (dense, 8-byte cp.async)
      double* ct = fine + PC::FINE;
      const int cbi = (T.i0 - 1) >> 1, cbj = DIM == 3 ? (T.j0 - 1) >> 1 : 0, cbk = (T.k0 - 1) >> 1;
      for (int e = tid; e < CT::SIZE; e += TC::NT) {
        const int ck = e % CT::CK, t = e / CT::CK;
        const int cj = DIM == 3 ? t % CT::CJ : 0, ci = DIM == 3 ? t / CT::CJ : t;
        const int gi = cbi + ci, gj = cbj + cj, gk = cbk + ck;
        const bool in = gi <= a.gc.n && gk <= a.gc.n && (DIM == 2 || gj <= a.gc.n);
        const uint32_t lin = DIM == 3 ? (uint32_t)gi * a.gc.ps + (uint32_t)gj * a.gc.s + gk : (uint32_t)gi * a.gc.s + gk;
        cp_async8(ct + e, a.x2 + lin, in);
      }
      mbar_arrive_cp_async(&bar[st]);
    } else if constexpr (!PC::BULK) {
      mbar_arrive_cp_async(&bar[st]);
    } else {
      mbar_arrive(&bar[st]);
    }
  };

  // pointwise operands of this thread's TI vertices of item `it`
  auto prefetch = [&](const PipeTile<DIM, TI>& T, double (&pb)[TI], double (&pp)[TI]) {
    const int k = T.k0 + tk, j = T.j0 + tj;
    const bool active = k <= g.n - 1 && (DIM == 2 || j <= g.n - 1);
    const uint32_t idx0 = DIM == 3 ? (uint32_t)T.i0 * g.ps + (uint32_t)j * g.s + k : (uint32_t)T.i0 * g.s + k;
    const bool inner = T.i0 - 1 >= 1 && T.i0 + T.ni <= g.n - 1 && T.k0 - 1 >= 1 && T.k0 + TC::TK <= g.n - 1 &&
                       (DIM == 2 || (T.j0 - 1 >= 1 && T.j0 + TC::TJ <= g.n - 1));
    const bool fold = LOAD == L_JAC0 && inner && a.x == a.b;
#pragma unroll
    for (int t = 0; t < TI; ++t) {
      const bool ok = active && t < T.ni;
      const uint32_t idx = idx0 + (uint32_t)t * pstride;
      pb[t] = (EpiNeeds<EPI>::B && ok && !fold) ? a.b[idx] : 0.0;
      pp[t] = (EpiNeeds<EPI>::P2 && ok) ? (EPI == T_CHEB ? a.x2[idx] : a.acc[idx]) : 0.0;
    }
  };

  // ---- one tile: wait for its stage, transform (L_JAC0 / L_PROLONG), stencil, store ----
  auto compute = [&](const PipeTile<DIM, TI>& T, int st, uint32_t parity, const double (&pb)[TI],
                     const double (&pp)[TI]) {
    double* fine = sm + st * SD;
    const int k = T.k0 + tk, j = T.j0 + tj;
    const bool active = k <= g.n - 1 && (DIM == 2 || j <= g.n - 1);
    const uint32_t idx0 = DIM == 3 ? (uint32_t)T.i0 * g.ps + (uint32_t)j * g.s + k : (uint32_t)T.i0 * g.s + k;
    const bool inner = T.i0 - 1 >= 1 && T.i0 + T.ni <= g.n - 1 && T.k0 - 1 >= 1 && T.k0 + TC::TK <= g.n - 1 &&
                       (DIM == 2 || (T.j0 - 1 >= 1 && T.j0 + TC::TJ <= g.n - 1));
    const bool fold = LOAD == L_JAC0 && inner && a.x == a.b;
    // parity of staged row (p, hj): a00 ^ ((p + hj) & sodd)
    const int a00 = (int)((reinterpret_cast<uintptr_t>(a.x + T.lin0) >> 3) & 1u);
    mbar_wait(&bar[st], parity);
#if OKG_PDL_TRIGGER == 2
    if (PC::NSTAGE == 1) pdl_trigger();  // multi-wave grid: release the dependents once the tile is staged
#endif
    if (LOAD != L_PLAIN && !fold) {
      // staging transform in shared memory: this thread's in-plane slots r = tid + q NT of every plane
      constexpr int PER = (TC::PSZ + TC::NT - 1) / TC::NT;
      int qoff[PER], qgj[PER], qgk[PER], qpar[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int r = min(tid + q * TC::NT, TC::PSZ - 1);  // (slots past the plane are skipped below)
        const int hj = DIM == 3 ? r / TC::PW : 0;
        const int hk = DIM == 3 ? r - hj * TC::PW : r;
        qgj[q] = DIM == 3 ? T.j0 - 1 + hj : 0;
        qgk[q] = T.k0 - 1 + hk;
        qpar[q] = hj & sodd;
        qoff[q] = hj * PC::RP + hk;
      }
      if (LOAD == L_JAC0) {
        int qcjk[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q)
          qcjk[q] = DIM == 3 ? cdig(qgj[q], g.n) * 3 + cdig(qgk[q], g.n) : cdig(qgk[q], g.n);
#pragma unroll
        for (int p = 0; p < TI + 2; ++p) {
          if (p >= T.ni + 2) break;  // CTA-uniform
          const int ip = T.i0 - 1 + p;
          const int cip = cdig(ip, g.n) * (DIM == 3 ? 9 : 3);
#pragma unroll
          for (int q = 0; q < PER; ++q) {
            if (tid + q * TC::NT >= TC::PSZ) continue;
            double& v = fine[p * PC::PLANE + qoff[q] + (a00 ^ (qpar[q] ^ (p & sodd)))];
            const int cls = cip + qcjk[q];
            const bool in = qgj[q] <= g.n && qgk[q] <= g.n;
            const double invd = (cls == Traits<DIM>::INTERIOR || !in)
                                    ? op.invd
                                    : __ldg(op.tab + cls * (Traits<DIM>::NOFF + 1) + Traits<DIM>::NOFF);
            v = a.omega * invd * v;
          }
        }
      } else {
        // L_PROLONG: e -> e + P e_c  (x + t, t rounded first: multigrid.hpp:111-112)
        const double* ct = fine + PC::FINE;
        constexpr int CSI = CT::CJ * CT::CK, CSJ = CT::CK;
        const int cbi = (T.i0 - 1) >> 1, cbj = DIM == 3 ? (T.j0 - 1) >> 1 : 0, cbk = (T.k0 - 1) >> 1;
        int cl[PER], cu[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const int gj = qgj[q], gk = qgk[q];
          cl[q] = (DIM == 3 ? ((gj >> 1) - cbj) * CSJ : 0) + ((gk >> 1) - cbk);
          cu[q] = (DIM == 3 ? (((gj + 1) >> 1) - cbj) * CSJ : 0) + (((gk + 1) >> 1) - cbk);
        }
#pragma unroll
        for (int p = 0; p < TI + 2; ++p) {
          if (p >= T.ni + 2) break;  // CTA-uniform
          const int ip = T.i0 - 1 + p;
          const int pl = ((ip >> 1) - cbi) * CSI, pu = (((ip + 1) >> 1) - cbi) * CSI;
#pragma unroll
          for (int q = 0; q < PER; ++q) {
            if (tid + q * TC::NT >= TC::PSZ) continue;
            double& v = fine[p * PC::PLANE + qoff[q] + (a00 ^ (qpar[q] ^ (p & sodd)))];
            // (all-even vertex: fma(0.5, x, 0.5 x) == x for every normal x, as in k_tiled)
            const double t = fma(0.5, ct[pu + cu[q]], 0.5 * ct[pl + cl[q]]);
            v = v + t;
          }
        }
      }
      fence_async_smem();
      __syncthreads();
    }
    // per-thread base pointers of the rows with (p + hj) even / odd relative to this thread's own row
    const int q0 = DIM == 3 ? (tj & 1) : 1;  // parity of (p + hj) at tap (t + di + dj) even
    const int oE = a00 ^ (q0 & sodd), oO = a00 ^ ((q0 ^ 1) & sodd);
    const double* bE = fine + (DIM == 3 ? (tj + 1) * PC::RP : 0) + tk + 1 + oE;
    const double* bO = fine + (DIM == 3 ? (tj + 1) * PC::RP : 0) + tk + 1 + oO;
    const double scl = fold ? a.omega * op.invd : 1.0;
    if (active) {
#pragma unroll
      for (int t = 0; t < TI; ++t) {
        double As = 0.0, s_own = 0.0, raw_own = 0.0;
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          const int di = off_comp(DIM, o, 0);
          const int dj = DIM == 3 ? off_comp(DIM, o, 1) : 0;
          const int dk = off_comp(DIM, o, DIM - 1);
          const int c = (t + di + dj) & 1;
          const double raw = (c ? bO : bE)[(t + 1 + di) * PC::PLANE + dj * PC::RP + dk];
          const double sv = LOAD == L_JAC0 ? scl * raw : raw;
          if (o == Traits<DIM>::CENTER) {
            s_own = sv;
            raw_own = raw;
          }
          As = fma(op.w[o], sv, As);
        }
        if (t < T.ni)
          epilogue_pre<DIM, EPI>(a, idx0 + (uint32_t)t * pstride, s_own, As, op.invd, fold ? raw_own : pb[t], pp[t]);
      }
    }
    __syncthreads();  // everyone is done with this stage: it may be refilled
  };

  // first tile item of this CTA
  int it = (int)blockIdx.x;
  if (it < nbb) it += ((nbb - it + G - 1) / G) * G;
  double pbA[TI], ppA[TI];
  PipeTile<DIM, TI> TA;
  if constexpr (PC::NSTAGE == 1) {
    // one stage: boundary items, then tile after tile without prefetch (with one item per
    // CTA this is k_tiled's schedule with 16-byte staging)
    for (int bi = (int)blockIdx.x; bi < nbb; bi += G)
      boundary_vertex<DIM, LOAD, EPI>(g, op, tl, a, (uint32_t)bi * TC::NT + tid);
    uint32_t ph = 0;
    for (; it < total; it += G) {
      TA.decode(tl, g, it - nbb);
      issue(TA, 0);
      prefetch(TA, pbA, ppA);
      compute(TA, 0, ph, pbA, ppA);
      ph ^= 1;
    }
  } else {
    double pbB[TI], ppB[TI];
    PipeTile<DIM, TI> TB;
    if (it < total) {
      TA.decode(tl, g, it - nbb);
      issue(TA, 0);
      prefetch(TA, pbA, ppA);
    }
    // boundary items first (their gathers overlap the first tile's flight)
    for (int bi = (int)blockIdx.x; bi < nbb; bi += G)
      boundary_vertex<DIM, LOAD, EPI>(g, op, tl, a, (uint32_t)bi * TC::NT + tid);
    // tiles, two per trip (stage 0 / stage 1; tile + register sets A / B)
    uint32_t ph = 0;
    while (it < total) {
      it += G;
      if (it < total) {
        TB.decode(tl, g, it - nbb);
        issue(TB, 1);
        prefetch(TB, pbB, ppB);
      }
      compute(TA, 0, ph, pbA, ppA);
      if (it >= total) break;
      it += G;
      if (it < total) {
        TA.decode(tl, g, it - nbb);
        issue(TA, 0);
        prefetch(TA, pbA, ppA);
      }
      compute(TB, 1, ph, pbB, ppB);
      ph ^= 1;
    }
  }
}

}  // namespace okg
