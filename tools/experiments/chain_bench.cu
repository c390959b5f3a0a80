// chain_bench.cu -- latency of a chain of small DEPENDENT kernels inside a CUDA graph, the
// regime of the multigrid levels below the finest (128^3: ~14 kernels of 4-7 us per V-cycle).
// Each kernel reads its predecessor's output (ping-pong buffers) and writes its own.
//   mode 0: plain stream order (no PDL)
//   mode 1: PDL, griddepcontrol.wait at entry, launch_dependents at exit  (the product's small kernels)
//   mode 2: PDL, wait at entry, launch_dependents at entry
//   mode 3: PDL, launch_dependents at entry, NO hardware wait: the dependency is a device
//           counter the predecessor's CTAs bump after their stores (fence + atomic); the
//           consumer's thread 0 polls it (acquire).  Epoch-based so a graph can be replayed.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/experiments/chain_bench tools/experiments/chain_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__global__ void k_epoch(unsigned* epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(epoch, 1u);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_link(const double* __restrict__ in, double* __restrict__ out, int n,
                                              unsigned* cnt_prev, unsigned* cnt_me, const unsigned* epoch,
                                              unsigned prev_grid, int first, int last) {
  if (MODE == 3) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (first || last) asm volatile("griddepcontrol.wait;" ::: "memory");  // graph entry / exit: hardware order
    if (!first) {
      if (threadIdx.x == 0) {
        const unsigned target = *(volatile const unsigned*)epoch * prev_grid;
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt_prev) : "memory");
          if (v < target) __nanosleep(32);
        } while (v < target);
      }
      __syncthreads();
    }
  } else if (MODE >= 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (MODE == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    // a small stencil-like dependent read: neighbours written by other CTAs of the predecessor
    const int l = i > 0 ? i - 1 : i, r = i + 1 < n ? i + 1 : i;
    out[i] = 0.25 * in[l] + 0.5 * in[i] + 0.25 * in[r] + 1e-3;
  }
  if (MODE == 3) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(cnt_me, 1u);
    }
  } else if (MODE == 1) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}

template <int MODE>
static float run(int ctas, int links, int replays, double* a, double* b, unsigned* cnt, unsigned* epoch,
                 double* check) {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaMemsetAsync(cnt, 0, 4096 * sizeof(unsigned), st));
  CK(cudaMemsetAsync(epoch, 0, sizeof(unsigned), st));
  CK(cudaMemsetAsync(a, 0, (size_t)ctas * 256 * 8, st));
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  auto launch = [&](auto kern, dim3 grid, auto... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = MODE >= 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
  };
  if (MODE == 3) launch(k_epoch, dim3(1), epoch);
  for (int l = 0; l < links; ++l) {
    const double* in = l % 2 ? b : a;
    double* out = l % 2 ? a : b;
    launch(k_link<MODE>, dim3(ctas), in, out, ctas * 256, cnt + (l > 0 ? l - 1 : 0), cnt + l,
           (const unsigned*)epoch, (unsigned)ctas, (int)(l == 0), (int)(l == links - 1));
  }
  CK(cudaStreamEndCapture(st, &gr));
  CK(cudaGraphInstantiate(&ge, gr, 0));
  for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  for (int w = 0; w < replays; ++w) CK(cudaGraphLaunch(ge, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaMemcpy(check, links % 2 ? b : a, 8, cudaMemcpyDeviceToHost));
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(gr));
  CK(cudaStreamDestroy(st));
  return ms * 1e3f / (replays * links);
}

int main() {
  const int links = 60, replays = 20;
  double *a, *b;
  unsigned *cnt, *epoch;
  CK(cudaMalloc(&a, 2048 * 256 * 8));
  CK(cudaMalloc(&b, 2048 * 256 * 8));
  CK(cudaMalloc(&cnt, 4096 * sizeof(unsigned)));
  CK(cudaMalloc(&epoch, sizeof(unsigned)));
  for (int ctas : {20, 89, 148, 433, 592, 1184}) {
    double c0, c1, c2, c3;
    const float t0 = run<0>(ctas, links, replays, a, b, cnt, epoch, &c0);
    const float t1 = run<1>(ctas, links, replays, a, b, cnt, epoch, &c1);
    const float t2 = run<2>(ctas, links, replays, a, b, cnt, epoch, &c2);
    const float t3 = run<3>(ctas, links, replays, a, b, cnt, epoch, &c3);
    printf("%5d CTAs: plain %5.2f  PDL(trigger at exit) %5.2f  PDL(trigger at entry) %5.2f  counter-dependency %5.2f us/kernel"
           "   check %s\n",
           ctas, t0, t1, t2, t3, (c0 == c1 && c1 == c2 && c2 == c3) ? "equal" : "DIFFER");
  }
  return 0;
}
