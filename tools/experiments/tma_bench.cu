// Microbenchmark: throughput of 1D TMA bulk copies (cp.async.bulk global->shared,
// mbarrier complete_tx) per request size, and of 16-byte cp.async (LDGSTS.128) for
// comparison -- to size the row copies of okg_pipe.cuh.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_bench tools/tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: bulk copies issued by one elected lane in a uniform loop
// mode 1: bulk copies, one per lane (waterfall)
// mode 2: LDGSTS.128 by all threads (cp.async 16 B), wait_group
template <int MODE>
__global__ void __launch_bounds__(256) k(const double* __restrict__ src, size_t n_dbl, int req_bytes, int reqs,
                                         int iters, double* sink) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t stride_dbl = (size_t)req_bytes / 8;
  size_t base = ((size_t)blockIdx.x * reqs * iters * stride_dbl) % (n_dbl - (size_t)reqs * stride_dbl * 2);
  base &= ~(size_t)1;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const double* s0 = src + base + (size_t)it * reqs * stride_dbl;
    if (s0 + reqs * stride_dbl > src + n_dbl) s0 = src;
    if (MODE == 0) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(reqs * req_bytes));
        for (int r = 0; r < reqs; ++r)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(sm + r * stride_dbl)),
                       "l"(s0 + r * stride_dbl), "r"(req_bytes), "r"(su32(&bar)));
      }
    } else if (MODE == 1) {
      if (tid < 32) {
        if (tid == 0)
          asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                       "r"(reqs * req_bytes));
        __syncwarp();
        for (int r = tid; r < reqs; r += 32)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(sm + r * stride_dbl)),
                       "l"(s0 + r * stride_dbl), "r"(req_bytes), "r"(su32(&bar)));
      }
    } else {
      const int n16 = reqs * req_bytes / 16;
      for (int e = tid; e < n16; e += 256)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + 2 * e)), "l"(s0 + 2 * e));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (MODE != 2) {
      const uint32_t ph = it & 1;
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
              su32(&bar)),
          "r"(ph)
          : "memory");
    }
    __syncthreads();
    acc += sm[tid];
    __syncthreads();
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const size_t n = (size_t)1 << 28;  // 2 GB of doubles
  double *src, *sink;
  cudaMalloc(&src, n * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 0, n * 8);
  const int sizes[] = {288, 544, 1056, 2080, 4096, 8192};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int sz : sizes) {
      const int tile = 32768;  // bytes per "tile"
      const int reqs = tile / sz;
      const int iters = 64;
      const int ctas = 148 * 2;
      const size_t smem = (size_t)reqs * sz;
      auto kk = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kk<<<ctas, 256, smem>>>(src, n, sz, reqs, 2, sink);
      cudaEventRecord(e0);
      kk<<<ctas, 256, smem>>>(src, n, sz, reqs, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)ctas * iters * reqs * sz;
      printf("mode %d size %5d reqs/tile %4d: %7.1f GB/s  (%.1f B/clk/SM, %.1f clk/req/CTA)  err=%s\n", mode, sz, reqs,
             bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.965e9 / 148, ms * 1e-3 * 1.965e9 / (iters * reqs),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
