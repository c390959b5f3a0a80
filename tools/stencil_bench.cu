// stencil_bench.cu -- design exploration for the fine-level damped-Jacobi sweep
//   y = x + w D^-1 (b - A x)   (15-point Kuhn stencil, 3D; 7-point, 2D)
// on the BASELINE grids (3D 129^3, 2D 2049^2).  Interior weights only (the
// kernel variants differ in data movement, not in boundary handling).
// Prints GB/s of 24 algorithmic bytes per vertex.  Not part of the product.
//
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/stencil_bench tools/stencil_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e));      \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__constant__ double cw[15];
constexpr double OMEGA_INVD = 0.123;

// offsets (di,dj,dk) of the 15-point Kuhn stencil, ascending
__host__ __device__ constexpr int OFF3[15][3] = {{-1, -1, -1}, {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 0}, {0, -1, -1},
                                                 {0, -1, 0},   {0, 0, -1},  {0, 0, 0},   {0, 0, 1},  {0, 1, 0},
                                                 {0, 1, 1},    {1, 0, 0},   {1, 0, 1},   {1, 1, 0},  {1, 1, 1}};

struct G3 {
  int n, s;
  unsigned ps;
};

// ---------------- V0: naive, one thread per vertex ----------------
__global__ void v0_naive(G3 g, const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ y) {
  const unsigned idx = blockIdx.x * 256 + threadIdx.x;
  const unsigned N = g.ps * g.s;
  if (idx >= N) return;
  const int i = idx / g.ps, r = idx - i * g.ps, j = r / g.s, k = r - j * g.s;
  if (i < 1 || i >= g.n || j < 1 || j >= g.n || k < 1 || k >= g.n) return;
  double s = 0.0;
#pragma unroll
  for (int o = 0; o < 15; ++o)
    s = fma(cw[o], __ldg(x + (int)idx + OFF3[o][0] * (int)g.ps + OFF3[o][1] * g.s + OFF3[o][2]), s);
  y[idx] = x[idx] + OMEGA_INVD * (b[idx] - s);
}

// ---------------- V1: whole-tile staging, U-batched linear loop ----------------
template <int TK, int TJ, int TI>
__global__ void __launch_bounds__(TK* TJ) v1_tile(G3 g, const double* __restrict__ x, const double* __restrict__ b,
                                                  double* __restrict__ y, int ktiles, int jtiles) {
  constexpr int NT = TK * TJ, PW = TK + 2, PSZ = PW * (TJ + 2);
  extern __shared__ double tile[];
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * TI;
  const int ni = min(TI, g.n - i0);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  const int total = (ni + 2) * PSZ;
  constexpr int U = 8;
  for (int base = tid; base < total; base += NT * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      v[u] = 0.0;
      if (e < total) {
        const int p = e / PSZ, r = e - p * PSZ, hj = r / PW, hk = r - hj * PW;
        const int gj = j0 - 1 + hj, gk = k0 - 1 + hk;
        if (gj <= g.n && gk <= g.n) v[u] = __ldg(x + (unsigned)(i0 - 1 + p) * g.ps + gj * g.s + gk);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      if (e < total) tile[e] = v[u];
    }
  }
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k < g.n && j < g.n;
  double pb[TI], px[TI];
  const unsigned idx0 = (unsigned)i0 * g.ps + j * g.s + k;
#pragma unroll
  for (int t = 0; t < TI; ++t) {
    pb[t] = (active && t < ni) ? b[idx0 + t * g.ps] : 0.0;
  }
  __syncthreads();
  if (!active) return;
#pragma unroll
  for (int t = 0; t < TI; ++t) {
    if (t >= ni) break;
    double s = 0.0, own = 0.0;
#pragma unroll
    for (int o = 0; o < 15; ++o) {
      const double v = tile[(t + 1 + OFF3[o][0]) * PSZ + (tj + 1 + OFF3[o][1]) * PW + tk + 1 + OFF3[o][2]];
      if (o == 7) own = v;
      s = fma(cw[o], v, s);
    }
    y[idx0 + t * g.ps] = own + OMEGA_INVD * (pb[t] - s);
  }
  (void)px;
}

// ---------------- V2: marching with register prefetch (2 planes ahead) ----------------
template <int TK, int TJ, int CH>
__global__ void __launch_bounds__(TK* TJ) v2_march(G3 g, const double* __restrict__ x, const double* __restrict__ b,
                                                   double* __restrict__ y, int ktiles, int jtiles) {
  constexpr int NT = TK * TJ, PW = TK + 2, PSZ = PW * (TJ + 2);
  constexpr int RPT = (PSZ + NT - 1) / NT;  // staged positions per thread
  __shared__ double ring[4][PSZ];
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * CH;
  const int i1 = min(i0 + CH, g.n);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k < g.n && j < g.n;
  unsigned off[RPT];
  bool ok[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT;
    const int hj = r / PW, hk = r - hj * PW;
    const int gj = j0 - 1 + hj, gk = k0 - 1 + hk;
    ok[q] = r < PSZ && gj <= g.n && gk <= g.n;
    off[q] = gj * g.s + gk;
  }
  auto fetch = [&](int ip, double (&v)[RPT]) {
#pragma unroll
    for (int q = 0; q < RPT; ++q) v[q] = ok[q] ? __ldg(x + (unsigned)ip * g.ps + off[q]) : 0.0;
  };
  auto put = [&](int ip, const double (&v)[RPT]) {
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      if (tid + q * NT < PSZ) ring[ip & 3][tid + q * NT] = v[q];
  };
  double va[RPT], vb[RPT];
  fetch(i0 - 1, va);
  put(i0 - 1, va);
  fetch(i0, va);
  put(i0, va);
  fetch(i0 + 1, va);                       // plane i0+1 in flight
  if (i0 + 2 <= g.n) fetch(i0 + 2, vb);    // plane i0+2 in flight
  const unsigned idx0 = (unsigned)j * g.s + k;
  double bnext = active ? b[(unsigned)i0 * g.ps + idx0] : 0.0;
  for (int i = i0; i < i1; ++i) {
    put(i + 1, va);
#pragma unroll
    for (int q = 0; q < RPT; ++q) va[q] = vb[q];
    if (i + 3 <= g.n && i + 3 <= i1 + 1) fetch(i + 3, vb);
    const double bcur = bnext;
    if (active && i + 1 < i1) bnext = b[(unsigned)(i + 1) * g.ps + idx0];
    __syncthreads();
    if (active) {
      double s = 0.0, own = 0.0;
#pragma unroll
      for (int o = 0; o < 15; ++o) {
        const double v = ring[(i + OFF3[o][0]) & 3][(tj + 1 + OFF3[o][1]) * PW + tk + 1 + OFF3[o][2]];
        if (o == 7) own = v;
        s = fma(cw[o], v, s);
      }
      y[(unsigned)i * g.ps + idx0] = own + OMEGA_INVD * (bcur - s);
    }
  }
}

// ---------------- V3: one thread per z-run of R vertices, register reuse ----------------
template <int R>
__global__ void __launch_bounds__(256) v3_zrun(G3 g, const double* __restrict__ x, const double* __restrict__ b,
                                               double* __restrict__ y) {
  // thread -> (i, j, k-run); k-runs of R vertices cover k in [1, n-1]
  const int runs = (g.n - 1 + R - 1) / R;
  const unsigned t = blockIdx.x * 256 + threadIdx.x;
  const unsigned rows = (unsigned)(g.n - 1) * (g.n - 1);
  if (t >= rows * runs) return;
  const int run = t % runs;
  const unsigned row = t / runs;
  const int i = 1 + row / (g.n - 1), j = 1 + row % (g.n - 1);
  const int kb = 1 + run * R;
  const unsigned base = (unsigned)i * g.ps + j * g.s;
  // 7 (di,dj) rows, each needs k in [kb-1, kb+R]
  constexpr int RW = R + 2;
  double rowv[7][RW];
  const int dij[7][2] = {{-1, -1}, {-1, 0}, {0, -1}, {0, 0}, {0, 1}, {1, 0}, {1, 1}};
#pragma unroll
  for (int q = 0; q < 7; ++q)
#pragma unroll
    for (int c = 0; c < RW; ++c) {
      const int kk = kb - 1 + c;
      rowv[q][c] = kk <= g.n ? __ldg(x + (int)base + dij[q][0] * (int)g.ps + dij[q][1] * g.s + kk) : 0.0;
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int k = kb + r;
    if (k >= g.n) break;
    double s = 0.0;
#pragma unroll
    for (int o = 0; o < 15; ++o) {
      int q = 0;
#pragma unroll
      for (int qq = 0; qq < 7; ++qq)
        if (dij[qq][0] == OFF3[o][0] && dij[qq][1] == OFF3[o][1]) q = qq;
      s = fma(cw[o], rowv[q][r + 1 + OFF3[o][2]], s);
    }
    const unsigned idx = base + k;
    y[idx] = rowv[3][r + 1] + OMEGA_INVD * (b[idx] - s);
  }
}


// ---------------- cp.async helpers ----------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = ok ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(ok ? gmem : smem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------- V4: whole-tile staging by cp.async (no register staging) ----------------
template <int TK, int TJ, int TI, int MINB>
__global__ void __launch_bounds__(TK* TJ, MINB) v4_tile_async(G3 g, const double* __restrict__ x,
                                                               const double* __restrict__ b, double* __restrict__ y,
                                                               int ktiles, int jtiles) {
  constexpr int NT = TK * TJ, PW = TK + 2, PSZ = PW * (TJ + 2);
  extern __shared__ double tile[];
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * TI;
  const int ni = min(TI, g.n - i0);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  const int total = (ni + 2) * PSZ;
  for (int e = tid; e < total; e += NT) {
    const int p = e / PSZ, r = e - p * PSZ, hj = r / PW, hk = r - hj * PW;
    const int gj = j0 - 1 + hj, gk = k0 - 1 + hk;
    const bool ok = gj <= g.n && gk <= g.n;
    cp_async8(tile + e, x + (unsigned)(i0 - 1 + p) * g.ps + gj * g.s + gk, ok);
  }
  cp_commit();
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k < g.n && j < g.n;
  double pb[TI];
  const unsigned idx0 = (unsigned)i0 * g.ps + j * g.s + k;
#pragma unroll
  for (int t = 0; t < TI; ++t) pb[t] = (active && t < ni) ? b[idx0 + t * g.ps] : 0.0;
  cp_wait<0>();
  __syncthreads();
  if (!active) return;
#pragma unroll
  for (int t = 0; t < TI; ++t) {
    double s = 0.0, own = 0.0;
#pragma unroll
    for (int o = 0; o < 15; ++o) {
      const double v = tile[(t + 1 + OFF3[o][0]) * PSZ + (tj + 1 + OFF3[o][1]) * PW + tk + 1 + OFF3[o][2]];
      if (o == 7) own = v;
      s = fma(cw[o], v, s);
    }
    if (t < ni) y[idx0 + t * g.ps] = own + OMEGA_INVD * (pb[t] - s);
  }
}

// ---------------- V5: x-marching, cp.async ring of 8 planes, PD planes prefetched ----------------
template <int TK, int TJ, int CH, int PD, int MINB>
__global__ void __launch_bounds__(TK* TJ, MINB) v5_march_async(G3 g, const double* __restrict__ x,
                                                                const double* __restrict__ b, double* __restrict__ y,
                                                                int ktiles, int jtiles) {
  constexpr int NT = TK * TJ, PW = TK + 2, PSZ = PW * (TJ + 2);
  constexpr int RPT = (PSZ + NT - 1) / NT;
  extern __shared__ double sm[];
  double* ring = sm;              // [8][PSZ]
  double* bring = sm + 8 * PSZ;   // [8][NT]
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * CH;
  const int i1 = min(i0 + CH, g.n);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k < g.n && j < g.n;
  unsigned off[RPT];
  bool ok[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * NT;
    const int hj = r / PW, hk = r - hj * PW;
    const int gj = j0 - 1 + hj, gk = k0 - 1 + hk;
    ok[q] = r < PSZ && gj <= g.n && gk <= g.n;
    off[q] = ok[q] ? gj * g.s + gk : 0;
  }
  const unsigned own_off = active ? (unsigned)j * g.s + k : 0;
  auto issue = [&](int ip) {  // plane ip of x (+ b at plane ip when it is computed)
    if (ip <= i1) {
      double* dst = ring + (ip & 7) * PSZ;
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (tid + q * NT < PSZ) cp_async8(dst + tid + q * NT, x + (unsigned)ip * g.ps + off[q], ok[q]);
      if (ip >= i0 && ip < i1) cp_async8(bring + (ip & 7) * NT + tid, b + (unsigned)ip * g.ps + own_off, active);
    }
    cp_commit();  // always commit (empty groups keep the wait count uniform)
  };
  issue(i0 - 1);
  for (int d = 0; d <= PD; ++d) issue(i0 + d);
  for (int i = i0; i < i1; ++i) {
    cp_wait<PD>();  // planes <= i+1 landed
    __syncthreads();
    if (active) {
      double s = 0.0, own = 0.0;
#pragma unroll
      for (int o = 0; o < 15; ++o) {
        const double v = ring[((i + OFF3[o][0]) & 7) * PSZ + (tj + 1 + OFF3[o][1]) * PW + tk + 1 + OFF3[o][2]];
        if (o == 7) own = v;
        s = fma(cw[o], v, s);
      }
      y[(unsigned)i * g.ps + own_off] = own + OMEGA_INVD * (bring[(i & 7) * NT + tid] - s);
    }
    issue(i + PD + 1);
  }
}

__global__ void triad(const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) y[i] = x[i] + 0.5 * b[i];
}

// dependent chain element: optionally waits on the predecessor with PDL
template <bool PDL>
__global__ void chain_tiny(double* p, int n) {
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 0.999 + 1.0;
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
}

template <bool PDL>
__global__ void __launch_bounds__(256) v1_pdl(G3 g, const double* __restrict__ x, const double* __restrict__ b,
                                              double* __restrict__ y, int ktiles, int jtiles) {
  constexpr int TK = 32, TJ = 8, TI = 4, NT = 256, PW = TK + 2, PSZ = PW * (TJ + 2);
  extern __shared__ double tile[];
  int bb = blockIdx.x;
  const int kt = bb % ktiles;
  bb /= ktiles;
  const int jt = bb % jtiles, ic = bb / jtiles;
  const int k0 = 1 + kt * TK, j0 = 1 + jt * TJ, i0 = 1 + ic * TI;
  const int ni = min(TI, g.n - i0);
  const int tid = threadIdx.x, tk = tid % TK, tj = tid / TK;
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int total = (ni + 2) * PSZ;
  constexpr int U = 8;
  for (int base = tid; base < total; base += NT * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      v[u] = 0.0;
      if (e < total) {
        const int p = e / PSZ, r = e - p * PSZ, hj = r / PW, hk = r - hj * PW;
        const int gj = j0 - 1 + hj, gk = k0 - 1 + hk;
        if (gj <= g.n && gk <= g.n) v[u] = __ldg(x + (unsigned)(i0 - 1 + p) * g.ps + gj * g.s + gk);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * NT;
      if (e < total) tile[e] = v[u];
    }
  }
  const int k = k0 + tk, j = j0 + tj;
  const bool active = k < g.n && j < g.n;
  double pb[TI];
  const unsigned idx0 = (unsigned)i0 * g.ps + j * g.s + k;
#pragma unroll
  for (int t = 0; t < TI; ++t) pb[t] = (active && t < ni) ? b[idx0 + t * g.ps] : 0.0;
  __syncthreads();
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  if (!active) return;
#pragma unroll
  for (int t = 0; t < TI; ++t) {
    if (t >= ni) break;
    double s = 0.0, own = 0.0;
#pragma unroll
    for (int o = 0; o < 15; ++o) {
      const double v = tile[(t + 1 + OFF3[o][0]) * PSZ + (tj + 1 + OFF3[o][1]) * PW + tk + 1 + OFF3[o][2]];
      if (o == 7) own = v;
      s = fma(cw[o], v, s);
    }
    y[idx0 + t * g.ps] = own + OMEGA_INVD * (pb[t] - s);
  }
}

template <class K, class... Args>
void launch_pdl(bool pdl, K kernel, dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = 0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

template <class F>
float timeit(F&& f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int run(int n, bool extras) {
  const int s = n + 1;
  G3 g{n, s, (unsigned)(s * s)};
  const size_t N = (size_t)s * s * s;
  double h[15];
  for (int o = 0; o < 15; ++o) h[o] = (o == 7) ? 6.0 : -0.3 - 0.01 * o;
  CK(cudaMemcpyToSymbol(cw, h, sizeof h));
  const int NSET = n <= 128 ? 4 : 2;
  double *x[4], *b[4], *y[4];
  std::vector<double> hx(N);
  for (size_t i = 0; i < N; ++i) hx[i] = (double)(i % 1000) * 1e-3;
  for (int q = 0; q < NSET; ++q) {
    CK(cudaMalloc(&x[q], N * 8));
    CK(cudaMalloc(&b[q], N * 8));
    CK(cudaMalloc(&y[q], N * 8));
    CK(cudaMemcpy(x[q], hx.data(), N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b[q], hx.data(), N * 8, cudaMemcpyHostToDevice));
  }
  printf("=== n = %d (%.1f MB per vector)\n", n, N * 8 / 1e6);
  const double bytes = 24.0 * (double)(n - 1) * (n - 1) * (n - 1);
  int rot = 0;
  auto report = [&](const char* name, float ms) { printf("%-28s %8.2f us  %7.0f GB/s\n", name, ms * 1e3, bytes / ms / 1e6); };
  const int reps = 40;
  {
    float ms = timeit([&] { int q = rot++ % NSET; triad<<<148 * 8, 256>>>(x[q], b[q], y[q], N); }, reps);
    printf("%-28s %8.2f us  %7.0f GB/s (24 B/vertex, all vertices)\n", "triad grid-stride", ms * 1e3, 24.0 * N / ms / 1e6);
    ms = timeit([&] { int q = rot++ % NSET; triad<<<(N + 255) / 256, 256>>>(x[q], b[q], y[q], N); }, reps);
    printf("%-28s %8.2f us  %7.0f GB/s\n", "triad 1 elem/thread", ms * 1e3, 24.0 * N / ms / 1e6);
  }
  {
    float ms = timeit([&] { int q = rot++ % NSET; v0_naive<<<(N + 255) / 256, 256>>>(g, x[q], b[q], y[q]); }, reps);
    report("v0 naive", ms);
  }
#define V1(TK, TJ, TI)                                                                                  \
  {                                                                                                     \
    const int kt = (n - 1 + TK - 1) / TK, jt = (n - 1 + TJ - 1) / TJ, it = (n - 1 + TI - 1) / TI;        \
    const size_t sm = (size_t)(TI + 2) * (TK + 2) * (TJ + 2) * 8;                                        \
    CK(cudaFuncSetAttribute(v1_tile<TK, TJ, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    float ms = timeit(                                                                                  \
        [&] {                                                                                           \
          int q = rot++ % NSET;                                                                         \
          v1_tile<TK, TJ, TI><<<kt * jt * it, TK * TJ, sm>>>(g, x[q], b[q], y[q], kt, jt);              \
        },                                                                                              \
        reps);                                                                                          \
    char nm[64];                                                                                        \
    snprintf(nm, 64, "v1 tile %dx%dx%d", TK, TJ, TI);                                                   \
    report(nm, ms);                                                                                     \
  }
  V1(32, 8, 2) V1(32, 8, 4) V1(32, 8, 8) V1(32, 4, 4) V1(32, 4, 8) V1(64, 4, 4) V1(32, 16, 4) V1(128, 2, 4)
#define V2(TK, TJ, CH)                                                                         \
  {                                                                                            \
    const int kt = (n - 1 + TK - 1) / TK, jt = (n - 1 + TJ - 1) / TJ, it = (n - 1 + CH - 1) / CH; \
    float ms = timeit(                                                                         \
        [&] {                                                                                  \
          int q = rot++ % NSET;                                                                \
          v2_march<TK, TJ, CH><<<kt * jt * it, TK * TJ>>>(g, x[q], b[q], y[q], kt, jt);        \
        },                                                                                     \
        reps);                                                                                 \
    char nm[64];                                                                               \
    snprintf(nm, 64, "v2 march %dx%d ch%d", TK, TJ, CH);                                        \
    report(nm, ms);                                                                            \
  }
  V2(32, 8, 8) V2(32, 8, 16) V2(32, 8, 32) V2(32, 4, 16) V2(64, 4, 16) V2(32, 16, 16) V2(32, 8, 64)
#define V3(R)                                                                                  \
  {                                                                                            \
    const unsigned runs = (n - 1 + R - 1) / R, th = (unsigned)(n - 1) * (n - 1) * runs;       \
    float ms = timeit(                                                                         \
        [&] {                                                                                  \
          int q = rot++ % NSET;                                                                \
          v3_zrun<R><<<(th + 255) / 256, 256>>>(g, x[q], b[q], y[q]);                          \
        },                                                                                     \
        reps);                                                                                 \
    char nm[64];                                                                               \
    snprintf(nm, 64, "v3 zrun R=%d", R);                                                        \
    report(nm, ms);                                                                            \
  }
  V3(2) V3(4) V3(8)
#define V4(TK, TJ, TI, MINB)                                                                                  \
  {                                                                                                          \
    const int kt = (n - 1 + TK - 1) / TK, jt = (n - 1 + TJ - 1) / TJ, it = (n - 1 + TI - 1) / TI;             \
    const size_t sm = (size_t)(TI + 2) * (TK + 2) * (TJ + 2) * 8;                                             \
    CK(cudaFuncSetAttribute(v4_tile_async<TK, TJ, TI, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    float ms = timeit(                                                                                       \
        [&] {                                                                                                \
          int q = rot++ % NSET;                                                                              \
          v4_tile_async<TK, TJ, TI, MINB><<<kt * jt * it, TK * TJ, sm>>>(g, x[q], b[q], y[q], kt, jt);       \
        },                                                                                                   \
        reps);                                                                                               \
    char nm[64];                                                                                             \
    snprintf(nm, 64, "v4 async tile %dx%dx%d m%d", TK, TJ, TI, MINB);                                        \
    report(nm, ms);                                                                                          \
  }
  V4(32, 8, 4, 1) V4(32, 8, 4, 6) V4(32, 8, 8, 4) V4(32, 4, 4, 8) V4(32, 8, 2, 8)
#define V5(TK, TJ, CH, PD, MINB)                                                                              \
  {                                                                                                          \
    const int kt = (n - 1 + TK - 1) / TK, jt = (n - 1 + TJ - 1) / TJ, it = (n - 1 + CH - 1) / CH;             \
    const size_t sm = (size_t)8 * ((TK + 2) * (TJ + 2) + TK * TJ) * 8;                                       \
    CK(cudaFuncSetAttribute(v5_march_async<TK, TJ, CH, PD, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    float ms = timeit(                                                                                       \
        [&] {                                                                                                \
          int q = rot++ % NSET;                                                                              \
          v5_march_async<TK, TJ, CH, PD, MINB><<<kt * jt * it, TK * TJ, sm>>>(g, x[q], b[q], y[q], kt, jt);  \
        },                                                                                                   \
        reps);                                                                                               \
    char nm[64];                                                                                             \
    snprintf(nm, 64, "v5 march async %dx%d ch%d pd%d", TK, TJ, CH, PD);                                     \
    report(nm, ms);                                                                                          \
  }
  V5(32, 8, 8, 2, 4) V5(32, 8, 16, 2, 4) V5(32, 8, 16, 4, 4) V5(32, 8, 32, 4, 4) V5(32, 4, 16, 4, 8)
  V5(32, 4, 32, 4, 8) V5(64, 4, 16, 3, 4) V5(32, 8, 16, 6, 4) V5(32, 4, 8, 3, 8)
  if (extras) {
    // PDL: chains of 200 dependent launches
    const int kt = (n - 1 + 31) / 32, jt = (n - 1 + 7) / 8, it = (n - 1 + 3) / 4;
    const size_t sm = (size_t)6 * 34 * 10 * 8;
    for (int pdl = 0; pdl < 2; ++pdl) {
      float ms = timeit(
          [&] {
            for (int r = 0; r < 5; ++r) {
              int q = rot++ % NSET;
              if (pdl) launch_pdl(true, v1_pdl<true>, dim3(kt * jt * it), dim3(256), sm, g, (const double*)x[q], (const double*)b[q], y[q], kt, jt);
              else launch_pdl(false, v1_pdl<false>, dim3(kt * jt * it), dim3(256), sm, g, (const double*)x[q], (const double*)b[q], y[q], kt, jt);
            }
          },
          8);
      printf("%-28s %8.2f us per kernel\n", pdl ? "v1 32x8x4 chain PDL" : "v1 32x8x4 chain", ms * 1e3 / 5);
    }
    double* p;
    CK(cudaMalloc(&p, 1 << 20));
    for (int pdl = 0; pdl < 2; ++pdl)
      for (int blocks : {1, 20, 148}) {
        float ms = timeit(
            [&] {
              for (int r = 0; r < 50; ++r) {
                if (pdl) launch_pdl(true, chain_tiny<true>, dim3(blocks), dim3(256), 0, p, blocks * 256);
                else launch_pdl(false, chain_tiny<false>, dim3(blocks), dim3(256), 0, p, blocks * 256);
              }
            },
            4);
        printf("tiny chain %3d CTAs %s  %6.2f us per kernel\n", blocks, pdl ? "PDL" : "   ", ms * 1e3 / 50);
      }
    // same chains inside a CUDA graph
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaStream_t st;
      CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      cudaGraph_t gr;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      for (int r = 0; r < 50; ++r) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(20);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (pdl) CK(cudaLaunchKernelEx(&cfg, chain_tiny<true>, p, 20 * 256));
        else CK(cudaLaunchKernelEx(&cfg, chain_tiny<false>, p, 20 * 256));
      }
      CK(cudaStreamEndCapture(st, &gr));
      CK(cudaGraphInstantiate(&ge, gr, 0));
      for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
      cudaEvent_t a, bb;
      cudaEventCreate(&a);
      cudaEventCreate(&bb);
      cudaEventRecord(a, st);
      for (int w = 0; w < 10; ++w) CK(cudaGraphLaunch(ge, st));
      cudaEventRecord(bb, st);
      CK(cudaEventSynchronize(bb));
      float ms;
      cudaEventElapsedTime(&ms, a, bb);
      printf("graph tiny chain 20 CTAs %s %6.2f us per kernel\n", pdl ? "PDL" : "   ", ms * 1e3 / 500);
    }
  }
  for (int q = 0; q < NSET; ++q) {
    cudaFree(x[q]);
    cudaFree(b[q]);
    cudaFree(y[q]);
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    for (int a = 1; a < argc; ++a) run(atoi(argv[a]), false);
    return 0;
  }
  run(128, true);
  run(256, false);
  return 0;
}
