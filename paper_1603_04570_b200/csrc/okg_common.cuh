// okg_common.cuh -- device-side building blocks shared by every kernel.
//
// The structured simplicial mesh of the reference (mesh.hpp:87-157) is never
// materialised on the GPU.  A vertex is its linear index in the reference's
// order (x slowest, mesh.hpp:40-44); the P1 couplings of a vertex are the
// 1-ring offsets below (7 in 2D, 15 in 3D/Kuhn), listed in ascending linear
// order -- the column order of the reference's CSR rows, so every row sum is
// accumulated in the same order as spmv (sparse.hpp:138-150).
//
// Boundary vertices differ only by which of the 2^d surrounding grid cells
// exist, i.e. by a "class" in {lo, interior, hi}^d (3^d classes).  Constant
// operators (M, K, a*M, Shat_l) therefore reduce to one weight row per class
// (built on the host by element assembly, okg_tables.cpp), and interior
// vertices -- all but O(N^{(d-1)/d}) of them -- use weights passed by value
// in the kernel parameter bank.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace okg {

// Programmatic dependent launch (Hopper/Blackwell): every kernel is launched
// with cudaLaunchAttributeProgrammaticStreamSerialization and waits for its
// predecessor grid's completion (and memory) in griddepcontrol.wait before
// touching global memory, so launch latency and CTA ramp-up overlap the
// predecessor's tail.  Where a CTA lets its dependent grid be scheduled
// (griddepcontrol.launch_dependents) is OKG_PDL_TRIGGER:
//   2 (default): the multi-wave fine-level kernels (k_tiled, k_tiled_c) trigger
//      once their operand tile is staged, every other kernel at exit;
//   1: the other kernels right at entry (k_tiled / k_tiled_c at exit);
//   0: every kernel at exit.
// Measured (per-step, graphs on, one B200; "all at entry" was the old default):
// 3D 128^3 all-at-entry 50.9 / 0: 49.7 / 1: 50.9 / 2: 49.2 ms; 2D 2048^2
// 62.8 / 62.8 / 62.7 / 62.7 ms; 400^3 within 0.5 %.  An early trigger lets the
// dependent grid's CTAs take SM slots (spinning in griddepcontrol.wait) that
// the primary's later waves need.
// griddepcontrol.wait is a no-op for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#ifndef OKG_PDL_TRIGGER
#define OKG_PDL_TRIGGER 2
#endif
// The small kernels of the coarse levels (restriction, fused down/up level kernels, packed
// coarse matvec and its row sums) release their dependents at ENTRY (PDL_EARLY) and wait for
// their own predecessor only after their static prologue (index arithmetic, class table,
// operator block): measured with OKG_PDL_EARLY_SMALL = 0/1 on one box, 2D 2048^2 step
// 51.28 -> 50.33 ms, 3D 128^3 42.47 -> 42.42 ms, 400^3 unchanged; bit-identical.
#ifndef OKG_PDL_EARLY_SMALL
#define OKG_PDL_EARLY_SMALL 1
#endif
#if OKG_PDL_EARLY_SMALL
#define PDL_EARLY() pdl_trigger()
#else
#define PDL_EARLY() ((void)0)
#endif
#if OKG_PDL_TRIGGER == 1
#define PDL_ENTRY() \
  do {              \
    pdl_wait();     \
    pdl_trigger();  \
  } while (0)
#else
#define PDL_ENTRY() pdl_wait()
#endif

template <int DIM>
struct Traits;
template <>
struct Traits<2> {
  static constexpr int NOFF = 7;     // stencil offsets incl. centre
  static constexpr int CENTER = 3;
  static constexpr int NPOS = 3;     // strictly positive offsets
  static constexpr int NCLS = 9;     // boundary classes
  static constexpr int INTERIOR = 4; // class of an interior vertex
  static constexpr int NADJ = 6;     // simplices touching an interior vertex
  static constexpr int VPC = 3;      // vertices per simplex
};
template <>
struct Traits<3> {
  static constexpr int NOFF = 15;
  static constexpr int CENTER = 7;
  static constexpr int NPOS = 7;
  static constexpr int NCLS = 27;
  static constexpr int INTERIOR = 13;
  static constexpr int NADJ = 24;
  static constexpr int VPC = 4;
};

// Offsets (dx,dy[,dz]) in ascending linear order.
//  2D: (-1,-1) (-1,0) (0,-1) (0,0) (0,1) (1,0) (1,1)
//  3D: (-1,-1,-1) (-1,-1,0) (-1,0,-1) (-1,0,0) (0,-1,-1) (0,-1,0) (0,0,-1)
//      (0,0,0) (0,0,1) (0,1,0) (0,1,1) (1,0,0) (1,0,1) (1,1,0) (1,1,1)
// The list is point-symmetric: slot CENTER+q and CENTER-q are negatives.
__host__ __device__ constexpr int off_comp(int dim, int slot, int d) {
  // component d of offset `slot`
  return dim == 2
             ? (slot == 0 ? -1 : slot == 1 ? (d == 0 ? -1 : 0)
                : slot == 2 ? (d == 0 ? 0 : -1) : slot == 3 ? 0
                : slot == 4 ? (d == 0 ? 0 : 1) : slot == 5 ? (d == 0 ? 1 : 0) : 1)
             : (slot == 0 ? -1
                : slot == 1 ? (d == 2 ? 0 : -1)
                : slot == 2 ? (d == 1 ? 0 : -1)
                : slot == 3 ? (d == 0 ? -1 : 0)
                : slot == 4 ? (d == 0 ? 0 : -1)
                : slot == 5 ? (d == 1 ? -1 : 0)
                : slot == 6 ? (d == 2 ? -1 : 0)
                : slot == 7 ? 0
                : slot == 8 ? (d == 2 ? 1 : 0)
                : slot == 9 ? (d == 1 ? 1 : 0)
                : slot == 10 ? (d == 0 ? 0 : 1)
                : slot == 11 ? (d == 0 ? 1 : 0)
                : slot == 12 ? (d == 1 ? 0 : 1)
                : slot == 13 ? (d == 2 ? 0 : 1)
                : 1);
}

// Simplices touching a vertex: (cube code, stencil slots of the simplex's
// vertices).  Cube code bit d (MSB = x) is delta_d, the vertex's position in
// that grid cell; the cell exists iff g_d < n when delta_d = 0 and g_d >= 1
// when delta_d = 1.  2D cells {a,b,c},{a,c,d} (mesh.hpp:106-114); 3D Kuhn
// paths 0 -> e_p -> e_p+e_q -> (1,1,1) (mesh.hpp:124-148).
// {cube code, slots of the simplex's vertices}; usable in constant
// expressions on host and device (template-unrolled loops below).
constexpr int kAdj2[6][4] = {{0, 3, 5, 6}, {0, 3, 6, 4}, {1, 2, 5, 3},
                                 {2, 1, 3, 4}, {3, 0, 2, 3}, {3, 0, 3, 1}};
constexpr int kAdj3[24][5] = {
    {0, 7, 11, 13, 14}, {0, 7, 11, 12, 14}, {0, 7, 9, 13, 14}, {0, 7, 9, 10, 14},
    {0, 7, 8, 12, 14},  {0, 7, 8, 10, 14},  {1, 6, 7, 11, 13}, {1, 6, 7, 9, 13},
    {2, 5, 7, 11, 12},  {2, 5, 7, 8, 12},   {3, 4, 6, 7, 11},  {3, 4, 5, 7, 11},
    {4, 3, 7, 9, 10},   {4, 3, 7, 8, 10},   {5, 2, 6, 7, 9},   {5, 2, 3, 7, 9},
    {6, 1, 5, 7, 8},    {6, 1, 3, 7, 8},    {7, 0, 4, 6, 7},   {7, 0, 4, 5, 7},
    {7, 0, 2, 6, 7},    {7, 0, 2, 3, 7},    {7, 0, 1, 5, 7},   {7, 0, 1, 3, 7}};

// One multigrid level / the fine grid.  Nodes are indexed 0..N-1.
struct Grid {
  int32_t n;    // cells per axis
  int32_t s;    // n + 1
  uint32_t ps;  // plane size s^(dim-1)
  uint32_t N;   // vertices of the whole level
  int32_t ilo, ihi;  // owned x-planes [ilo, ihi) of this slab (whole grid: 0, s)
  uint32_t lo, hi;   // owned linear range [ilo*ps, ihi*ps)
  int32_t off[15];   // linear offsets of the stencil slots
};

// Constant stencil by value: interior row in the parameter bank, boundary
// rows in a per-class table [NCLS][NOFF+1] (last column = 1/diag).
template <int DIM>
struct Op {
  double w[Traits<DIM>::NOFF];
  double invd;
  const double* __restrict__ tab;
};

template <int DIM>
struct Node {
  int i, j, k;
  int cls;
};

template <int DIM>
__device__ __forceinline__ Node<DIM> locate(const Grid& g, uint32_t idx) {
  Node<DIM> nd;
  if (DIM == 3) {
    nd.i = (int)(idx / g.ps);
    const uint32_t r = idx - (uint32_t)nd.i * g.ps;
    nd.j = (int)(r / (uint32_t)g.s);
    nd.k = (int)(r - (uint32_t)nd.j * (uint32_t)g.s);
  } else {
    nd.i = (int)(idx / (uint32_t)g.s);
    nd.j = (int)(idx - (uint32_t)nd.i * (uint32_t)g.s);
    nd.k = 0;
  }
  const int cx = nd.i == 0 ? 0 : (nd.i == g.n ? 2 : 1);
  const int cy = nd.j == 0 ? 0 : (nd.j == g.n ? 2 : 1);
  if (DIM == 3) {
    const int cz = nd.k == 0 ? 0 : (nd.k == g.n ? 2 : 1);
    nd.cls = cx * 9 + cy * 3 + cz;
  } else {
    nd.cls = cx * 3 + cy;
  }
  return nd;
}

// Row of a constant operator at one vertex; `ld(j)` loads the operand.
template <int DIM, class LD>
__device__ __forceinline__ double op_row(const Op<DIM>& op, const Grid& g, uint32_t idx,
                                         int cls, LD&& ld) {
  constexpr int NO = Traits<DIM>::NOFF;
  double s = 0.0;
  if (cls == Traits<DIM>::INTERIOR) {
#pragma unroll
    for (int o = 0; o < NO; ++o) s = fma(op.w[o], ld((uint32_t)((int)idx + g.off[o])), s);
  } else {
    // boundary row: all weights, then all operands (a slot whose neighbour does not
    // exist has weight 0 and reads the vertex itself), then the FMA chain -- two
    // memory round trips instead of one per slot.  fma(0, v, s) == s up to the sign
    // of a zero, so rows equal those that skip the zero slots.
    const double* t = op.tab + cls * (NO + 1);
    double w[NO], v[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) w[o] = __ldg(t + o);
#pragma unroll
    for (int o = 0; o < NO; ++o) v[o] = ld(w[o] != 0.0 ? (uint32_t)((int)idx + g.off[o]) : idx);
#pragma unroll
    for (int o = 0; o < NO; ++o) s = fma(w[o], v[o], s);
  }
  return s;
}

template <int DIM>
__device__ __forceinline__ double op_invd(const Op<DIM>& op, int cls) {
  constexpr int NO = Traits<DIM>::NOFF;
  return cls == Traits<DIM>::INTERIOR ? op.invd : __ldg(op.tab + cls * (NO + 1) + NO);
}

// Does grid cell "cube code" exist around vertex nd?
template <int DIM>
__device__ __forceinline__ bool cell_exists(const Grid& g, const Node<DIM>& nd, int code) {
  const int dx = (code >> (DIM - 1)) & 1;
  const int dy = (code >> (DIM - 2)) & 1;
  bool ok = dx ? nd.i >= 1 : nd.i < g.n;
  ok = ok && (dy ? nd.j >= 1 : nd.j < g.n);
  if (DIM == 3) {
    const int dz = code & 1;
    ok = ok && (dz ? nd.k >= 1 : nd.k < g.n);
  }
  return ok;
}

// Deterministic block reduction of NV values (result valid in thread 0).
template <int NV, int BLOCK>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* smem /* [NV][BLOCK/32] */) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double x = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) smem[q * NW + warp] = x;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = lane < NW ? smem[q * NW + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      v[q] = x;
    }
  }
  __syncthreads();
}

}  // namespace okg
