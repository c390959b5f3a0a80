// jv_bench.cu -- register blocking of the tiled sweep over rows (JV vertices per thread along
// y) and 16-byte staging, against a clone of k_tiled's structure (JV = 1, 8-byte LDGSTS).
//   y = x + w D^-1 (b - A x)  (15-point Kuhn stencil, interior vertices of an (n+1)^3 grid)
// Motivation: the tiled sweeps are bound by the L1/shared data pipe --
// per warp of vertices 16 wavefronts of tap reads (8 LDS.64), 8.4 of LDGSTS shared-memory
// writes, 6.4 of global loads/stores.  A thread that owns JV adjacent rows shares taps between
// them: 3 JV + 4 loads per plane instead of 7 JV (JV = 2: 5 per vertex, JV = 4: 4); 16-byte
// LDGSTS chunks halve the staging wavefronts.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/experiments/jv_bench tools/experiments/jv_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

struct W15 {
  double w[15];
};
constexpr double OMEGA_INVD = 0.123;
__host__ __device__ constexpr int off3(int o, int d) {
  constexpr int T[15][3] = {{-1, -1, -1}, {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 0}, {0, -1, -1},
                            {0, -1, 0},   {0, 0, -1},  {0, 0, 0},   {0, 0, 1},  {0, 1, 0},
                            {0, 1, 1},    {1, 0, 0},   {1, 0, 1},   {1, 1, 0},  {1, 1, 1}};
  return T[o][d];
}
struct G3 {
  int n, s;
  unsigned ps;
};

__global__ void v0_naive(G3 g, W15 cw, const double* __restrict__ x, const double* __restrict__ b,
                         double* __restrict__ y) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned idx = blockIdx.x * 256 + threadIdx.x;
  const unsigned N = g.ps * g.s;
  if (idx >= N) return;
  const int i = idx / g.ps, r = idx - i * g.ps, j = r / g.s, k = r - j * g.s;
  if (i < 1 || i >= g.n || j < 1 || j >= g.n || k < 1 || k >= g.n) return;
  double s = 0.0;
#pragma unroll
  for (int o = 0; o < 15; ++o)
    s = fma(cw.w[o], __ldg(x + (int)idx + off3(o, 0) * (int)g.ps + off3(o, 1) * g.s + off3(o, 2)), s);
  y[idx] = fma(OMEGA_INVD, b[idx] - s, x[idx]);
}

__device__ __forceinline__ void cp8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp16(unsigned sa, const double* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

// TK x (TJT * JV) x TI interior vertices per CTA, TK * TJT threads, JV rows x TI planes per thread.
// WIDE = 0: dense tile [TI+2][PH][TK+2], 8-byte LDGSTS in linear order (k_tiled).
// WIDE = 1: rows of RP = TK + 4 doubles fetched as 16-byte chunks from the row start rounded
//           down to 16 bytes; element hk of row (p, hj) at row * RP + par(p, hj) + hk.
template <int TK, int TJT, int JV, int TI, int WIDE, int MINB>
__global__ void __launch_bounds__(TK* TJT, MINB) v_tile(G3 g, W15 cw, const double* __restrict__ x,
                                                        const double* __restrict__ b, double* __restrict__ y,
                                                        int ktiles, int jtiles) {
  constexpr int NT = TK * TJT, TJ = TJT * JV, PH = TJ + 2, PW = TK + 2;
  constexpr int RP = WIDE ? TK + 4 : PW;  // row pitch in shared memory
  constexpr int PSZ = PH * RP;
  extern __shared__ __align__(16) double tile[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * TI;
  const int ni = min(TI, g.n - i0);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  const int k = k0 + tk, jb = j0 + tj * JV;
  const uint32_t lin0 = (uint32_t)(i0 - 1) * g.ps + (uint32_t)(j0 - 1) * g.s + (uint32_t)(k0 - 1);
  // pointwise operand prefetch
  double pb[TI][JV];
#pragma unroll
  for (int t = 0; t < TI; ++t)
#pragma unroll
    for (int v = 0; v < JV; ++v) {
      const bool ok = k <= g.n - 1 && jb + v <= g.n - 1 && t < ni;
      pb[t][v] = ok ? b[(uint32_t)(i0 + t) * g.ps + (uint32_t)(jb + v) * g.s + k] : 0.0;
    }
  int a00 = 0;
  if (WIDE == 0) {
    const int total = (ni + 2) * PSZ;
    for (int e = tid; e < total; e += NT) {
      const int hk = e % PW, r = e / PW, hj = r % PH, p = r / PH;
      const bool in = k0 - 1 + hk <= g.n && j0 - 1 + hj <= g.n;
      cp8(tile + e, x + lin0 + (uint32_t)p * g.ps + (uint32_t)hj * g.s + hk, in);
    }
  } else {
    constexpr int CH = RP / 2;
    a00 = (int)((reinterpret_cast<uintptr_t>(x + lin0) >> 3) & 1u);
    const int nch = (ni + 2) * PH * CH;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(tile);
    const uint32_t vend = g.ps * (uint32_t)g.s;
    for (int e = tid; e < nch; e += NT) {
      const int c = e % CH, r = e / CH, hj = r % PH, p = r / PH;
      const uint32_t lin = lin0 + (uint32_t)p * g.ps + (uint32_t)hj * g.s + 2u * c;
      const uint32_t par = (uint32_t)(a00 ^ ((p + hj) & 1));
      const bool in = j0 - 1 + hj <= g.n && lin < vend + par;
      cp16(sbase + (unsigned)e * 16u, in ? (x + lin) - par : (x + lin0) - a00, in);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (k > g.n - 1) return;
  // row (p, hj) of the tile starts at (p * PH + hj) * RP + par(p, hj); par = a00 ^ ((p + hj) & 1)
  // (s and ps odd).  This thread's rows: hj = tj * JV + v + 1 + dj, planes p = t + 1 + di.
  const int q0 = WIDE ? ((tj * JV) & 1) : 0;
  const double* bE = tile + (tj * JV + 1) * RP + tk + 1 + (WIDE ? (a00 ^ q0) : 0);
  const double* bO = tile + (tj * JV + 1) * RP + tk + 1 + (WIDE ? (a00 ^ q0 ^ 1) : 0);
#pragma unroll
  for (int t = 0; t < TI; ++t) {
#pragma unroll
    for (int v = 0; v < JV; ++v) {
      double As = 0.0, own = 0.0;
#pragma unroll
      for (int o = 0; o < 15; ++o) {
        const int di = off3(o, 0), dj = off3(o, 1), dk = off3(o, 2);
        const int c = (t + di + v + dj) & 1;  // parity of (p + hj) relative to the thread's first row
        const double val = (c ? bO : bE)[(t + 1 + di) * PSZ + (v + dj) * RP + dk];
        if (o == 7) own = val;
        As = fma(cw.w[o], val, As);
      }
      if (t < ni && jb + v <= g.n - 1)
        y[(uint32_t)(i0 + t) * g.ps + (uint32_t)(jb + v) * g.s + k] = fma(OMEGA_INVD, pb[t][v] - As, own);
    }
  }
}

static float time_it(int reps, void (*f)(int, void*), void* ctx) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int r = 0; r < 3; ++r) f(r, ctx);
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) f(r, ctx);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

struct Ctx {
  G3 g;
  W15 w;
  int nsets;
  double **x, **b, **y;
  int ktiles, jtiles, chunks;
  size_t smem;
};

template <class K, class... A>
static void launch_pdl(K kern, unsigned grid, unsigned block, size_t smem, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <int TK, int TJT, int JV, int TI, int WIDE, int MINB>
static void run_tile(int r, void* p) {
  Ctx* c = (Ctx*)p;
  const int q = r % c->nsets;
  launch_pdl(v_tile<TK, TJT, JV, TI, WIDE, MINB>, (unsigned)(c->ktiles * c->jtiles * c->chunks), TK * TJT, c->smem, c->g,
             c->w, (const double*)c->x[q], (const double*)c->b[q], c->y[q], c->ktiles, c->jtiles);
}
static void run_naive(int r, void* p) {
  Ctx* c = (Ctx*)p;
  const int q = r % c->nsets;
  const unsigned N = c->g.ps * c->g.s;
  launch_pdl(v0_naive, (N + 255) / 256, 256, 0, c->g, c->w, (const double*)c->x[q], (const double*)c->b[q], c->y[q]);
}

template <int TK, int TJT, int JV, int TI, int WIDE, int MINB>
static void variant(Ctx& c, const std::vector<double>& ref, int reps, int carve) {
  constexpr int TJ = TJT * JV, RP = WIDE ? TK + 4 : TK + 2;
  const int n = c.g.n;
  c.ktiles = (n - 1 + TK - 1) / TK;
  c.jtiles = (n - 1 + TJ - 1) / TJ;
  c.chunks = (n - 1 + TI - 1) / TI;
  c.smem = (size_t)(TI + 2) * (TJ + 2) * RP * 8;
  auto kern = v_tile<TK, TJT, JV, TI, WIDE, MINB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TK * TJT, c.smem));
  const size_t N = (size_t)c.g.ps * c.g.s;
  CK(cudaMemset(c.y[0], 0, N * 8));
  run_tile<TK, TJT, JV, TI, WIDE, MINB>(0, &c);
  CK(cudaDeviceSynchronize());
  std::vector<double> out(N);
  CK(cudaMemcpy(out.data(), c.y[0], N * 8, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < N; ++i) bad += std::memcmp(&out[i], &ref[i], 8) != 0;
  const float ms = time_it(reps, run_tile<TK, TJT, JV, TI, WIDE, MINB>, &c);
  printf("  tile %2dx%2dx%d JV=%d NT=%3d %s carve=%3d regs=%3d spill=%3zuB smem=%2zuKB occ=%d ctas=%6d: %8.2f us %6.0f GB/s  mismatches=%zu\n",
         TK, TJ, TI, JV, TK * TJT, WIDE ? "16B" : " 8B", carve, fa.numRegs, (size_t)fa.localSizeBytes, c.smem / 1024, occ,
         c.ktiles * c.jtiles * c.chunks, ms * 1e3, 24.0 * N / ms / 1e6, bad);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 128;
  const int reps = argc > 2 ? atoi(argv[2]) : 50;
  Ctx c;
  c.g.n = n;
  c.g.s = n + 1;
  c.g.ps = (unsigned)c.g.s * c.g.s;
  const size_t N = (size_t)c.g.ps * c.g.s;
  for (int o = 0; o < 15; ++o) c.w.w[o] = o == 7 ? 1.0 : -0.03 - 0.001 * o;
  c.nsets = argc > 3 ? atoi(argv[3]) : std::max(1, std::min(8, (int)(400e6 / (24.0 * N)) + 1));
  c.x = new double*[c.nsets];
  c.b = new double*[c.nsets];
  c.y = new double*[c.nsets];
  std::vector<double> hx(N), hb(N);
  srand(1);
  for (size_t i = 0; i < N; ++i) {
    hx[i] = rand() / (double)RAND_MAX - 0.5;
    hb[i] = rand() / (double)RAND_MAX - 0.5;
  }
  for (int q = 0; q < c.nsets; ++q) {
    CK(cudaMalloc(&c.x[q], N * 8 + 64));
    CK(cudaMalloc(&c.b[q], N * 8 + 64));
    CK(cudaMalloc(&c.y[q], N * 8 + 64));
    CK(cudaMemcpy(c.x[q], hx.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.b[q], hb.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(c.y[q], 0, N * 8));
  }
  run_naive(0, &c);
  CK(cudaDeviceSynchronize());
  std::vector<double> ref(N);
  CK(cudaMemcpy(ref.data(), c.y[0], N * 8, cudaMemcpyDeviceToHost));
  printf("n=%d  N=%zu  sets=%d (rotating; 1 = L2-warm)\n", n, N, c.nsets);
  printf("  naive: %8.2f us\n", time_it(reps, run_naive, &c) * 1e3);
  //        TK TJT JV TI WIDE MINB
  variant<32, 8, 1, 8, 0, 4>(c, ref, reps, 50);   // k_tiled's structure
  variant<32, 8, 1, 8, 1, 4>(c, ref, reps, 50);   // + 16-byte staging
  variant<32, 8, 1, 8, 1, 4>(c, ref, reps, 100);
  variant<32, 4, 2, 8, 0, 4>(c, ref, reps, 50);   // JV = 2, same tile, 128 threads
  variant<32, 4, 2, 8, 1, 4>(c, ref, reps, 50);
  variant<32, 4, 2, 8, 1, 6>(c, ref, reps, 100);
  variant<32, 8, 2, 8, 1, 2>(c, ref, reps, 100);  // JV = 2, 16-row tile, 256 threads
  variant<32, 8, 2, 8, 1, 3>(c, ref, reps, 100);
  variant<32, 8, 2, 4, 0, 4>(c, ref, reps, 50);   // JV = 2, TI = 4
  variant<32, 8, 2, 4, 1, 4>(c, ref, reps, 50);
  variant<32, 8, 2, 4, 1, 4>(c, ref, reps, 100);
  variant<32, 4, 4, 4, 1, 4>(c, ref, reps, 50);   // JV = 4, TI = 4, 128 threads
  variant<32, 4, 4, 4, 1, 6>(c, ref, reps, 100);
  variant<32, 8, 4, 4, 1, 2>(c, ref, reps, 100);  // JV = 4, TI = 4, 32-row tile, 256 threads
  variant<32, 4, 4, 8, 1, 3>(c, ref, reps, 100);  // JV = 4, TI = 8, 128 threads
  return 0;
}
