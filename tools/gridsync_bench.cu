// gridsync_bench.cu -- cost of a grid-wide barrier on B200 (design probe for a
// persistent multigrid kernel on the coarse levels).  Not part of the product.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gridsync_bench tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__global__ void k_cg_sync(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    g.sync();
  }
  if (acc == -1.0) sink[0] = acc;
}

// sense-reversing barrier: one atomic per CTA, spin on a generation word
__device__ __forceinline__ void my_sync(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_my_sync(int iters, unsigned* count, unsigned* gen, double* sink) {
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    my_sync(count, gen, gridDim.x);
  }
  if (acc == -1.0) sink[0] = acc;
}

// one "phase": every CTA reads a slice of x (global, written by other CTAs in the
// previous phase), 7-point-ish 1D stencil, writes y; then grid sync; swap
__global__ void k_phases(int iters, double* x, double* y, int n) {
  cg::grid_group g = cg::this_grid();
  for (int it = 0; it < iters; ++it) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const double l = i > 0 ? x[i - 1] : 0.0, r = i + 1 < n ? x[i + 1] : 0.0;
      y[i] = 0.5 * x[i] + 0.25 * (l + r);
    }
    g.sync();
    double* t = x;
    x = y;
    y = t;
  }
}

__global__ void k_phase_single(const double* x, double* y, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double l = i > 0 ? x[i - 1] : 0.0, r = i + 1 < n ? x[i + 1] : 0.0;
    y[i] = 0.5 * x[i] + 0.25 * (l + r);
  }
}

int main() {
  double* sink;
  CK(cudaMalloc(&sink, 64));
  unsigned *cnt, *gen;
  CK(cudaMalloc(&cnt, 4));
  CK(cudaMalloc(&gen, 4));
  CK(cudaMemset(cnt, 0, 4));
  CK(cudaMemset(gen, 0, 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 512, 1024}) {
    for (int per_sm : {1, 2}) {
      if (threads * per_sm > 2048) continue;
      int nb = 148 * per_sm;
      int iters = 2000;
      void* args[] = {&iters, &sink};
      CK(cudaLaunchCooperativeKernel((void*)k_cg_sync, nb, threads, args, 0, 0));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      CK(cudaLaunchCooperativeKernel((void*)k_cg_sync, nb, threads, args, 0, 0));
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cg grid.sync  %4d CTAs x %4d thr: %6.3f us per sync\n", nb, threads, ms * 1e3 / iters);
      void* args2[] = {&iters, &cnt, &gen, &sink};
      CK(cudaLaunchCooperativeKernel((void*)k_my_sync, nb, threads, args2, 0, 0));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      CK(cudaLaunchCooperativeKernel((void*)k_my_sync, nb, threads, args2, 0, 0));
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      printf("custom sync   %4d CTAs x %4d thr: %6.3f us per sync\n", nb, threads, ms * 1e3 / iters);
    }
  }
  // phases over vectors of the coarse-level sizes: persistent+sync vs one launch per phase
  for (int n : {274625, 35937, 4913}) {
    double *x, *y;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&y, n * 8));
    CK(cudaMemset(x, 0, n * 8));
    int iters = 200, nb = 148, threads = 1024;
    void* args[] = {&iters, &x, &y, &n};
    CK(cudaLaunchCooperativeKernel((void*)k_phases, nb, threads, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    CK(cudaLaunchCooperativeKernel((void*)k_phases, nb, threads, args, 0, 0));
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("persistent phases n=%6d: %6.3f us per phase\n", n, ms * 1e3 / iters);
    // graph of single launches
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) {
      const int blocks = (n + 255) / 256;
      k_phase_single<<<blocks, 256, 0, st>>>(i % 2 ? y : x, i % 2 ? x : y, n);
    }
    CK(cudaStreamEndCapture(st, &gr));
    CK(cudaGraphInstantiate(&ge, gr, 0));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    cudaEventRecord(a, st);
    CK(cudaGraphLaunch(ge, st));
    cudaEventRecord(b, st);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("graph launches    n=%6d: %6.3f us per phase\n", n, ms * 1e3 / iters);
    cudaFree(x);
    cudaFree(y);
  }
  return 0;
}
