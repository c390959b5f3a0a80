// okg_host.cu -- host orchestration of the B200 Newton linear solve and the
// C ABI of include/okg.h.
//
// Mirrors the reference call structure (file:line under
// /root/reference/proj/include/okflow):
//   make_schur_context   precond.hpp:126-181  -> okg_create
//   build_hierarchy      multigrid.hpp:43-86  -> build_levels (rediscretised
//                        Shat_l = M_l + eps*sqrt(c) K_l, equal to the Galerkin
//                        P^T Shat P of the reference for nested P1 spaces)
//   mg_cycle / v_cycle / apply_shat_inv  multigrid.hpp:97-149
//   apply_M_inv/A_inv, apply_schur_tilde_inv, apply_schur, apply_S_inv_approx,
//   apply_C, apply_block, jacobian_operator   precond.hpp:185-298
//   gmres                krylov.hpp:44-152
//   residual, newton_solve  model.hpp:121-215
// Everything runs on one CUDA stream; the Arnoldi operator (block
// preconditioner + Jacobian, ~300 kernels) is captured once into a CUDA
// graph and replayed per GMRES iteration.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/okg.h"
#include "okg_kernels.cuh"
#include "okg_diag.cuh"
#include "okg_ssor.cuh"
#include "okg_nccl.h"
#include "okg_cusolver.h"
#include "okg_tables.h"

namespace okg {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

struct Status {
  int code;
};

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e__ = (call);                                                          \
    if (e__ != cudaSuccess)                                                            \
      throw Status{fail(OKG_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e__),   \
                        __FILE__, __LINE__)};                                          \
  } while (0)

#define THROW(code, ...) throw Status{fail(code, __VA_ARGS__)}

#define NCK(c, call)                                                                   \
  do {                                                                                 \
    ncclResult_t r__ = (call);                                                         \
    if (r__ != ncclSuccess)                                                            \
      throw Status{fail(OKG_ECUDA, "%s: %s", #call, (c)->ncl->GetErrorString(r__))};    \
  } while (0)

struct HostOp {
  double w[15];
  double invd;
  double* tab = nullptr;  // device [ncls][noff+1]
  std::vector<double> htab;
};

template <int DIM>
static Op<DIM> dev_op(const HostOp& h) {
  Op<DIM> o;
  for (int q = 0; q < Traits<DIM>::NOFF; ++q) o.w[q] = h.w[q];
  o.invd = h.invd;
  o.tab = h.tab;
  return o;
}

struct Level {
  Grid g;      // owned planes [g.ilo, g.ihi) of this slab (the whole level when not split)
  int gh = 0;  // ghost planes per side (1 on split levels of a multi-slab context)
  size_t B = 0;     // allocation stride of one level vector (owned + ghost planes)
  bool rep = false; // replicated on every slab (levels too thin to split, the coarsest)
  HostOp shat;
  bool tiled = false;
  bool wide = false;   // tiled kernels stage in 16-byte chunks (k_tiled WIDE; odd row pitch)
  bool wide_xf = false;  // ... also the kernels with a staging transform (L_JAC0; L_PROLONG in 2D)
  bool wide_thin = false;  // ... also on levels whose tiles are 2 or 3 planes thick
  bool fused = false;  // V(2,2) through k_mg_down / k_mg_up (okg_vcycle.cuh)
  Tiling tl{};
  unsigned tl_blocks = 0;
  Tiling tlc{};  // the C-block kernels' tiling (okg_tiled_c.cuh): same tiles, their own x-chunks
  unsigned tlc_blocks = 0;
  double *b = nullptr, *x = nullptr, *ea = nullptr, *eb = nullptr, *res = nullptr;
};

struct Group;

}  // namespace okg

using namespace okg;

struct okg_ctx {
  okg_params p;
  int dim = 0, n = 0;
  uint32_t N = 0;
  size_t N2 = 0;
  double h = 0, c = 0, sqrt_c = 0, a_coeff = 0, dt_theta = 0, shat_scale = 1, eps_sqrt_c = 0;
  double lambda_lo = 0, lambda_hi = 0;
  std::vector<double> cheb_c1, cheb_c2;
  double cheb_inv_theta = 0;
  bool cheb_fuse0 = true;  // first Chebyshev step forms the start vector itself (k_tiled L_CHEB0)
  Grid fine;
  HostOp M, K, A;
  std::vector<Level> lv;
  int nc = 0;
  double* Ainv = nullptr;
  // large coarsest level (nc > 2000): device-factorised inverse, rows [coarse_r0, coarse_r1)
  // of it on this slab (all rows unless the level is split for the solve), row stride coarse_ld
  bool coarse_big = false, coarse_split = false;
  int coarse_r0 = 0, coarse_r1 = 0;
  size_t coarse_ld = 0;
  int coarse_nb = 0;  // > 0: one slab, symmetric packed blocks (k_coarse_sym)
  double *coarse_R = nullptr, *coarse_C = nullptr;
  // collapsed bottom of the V-cycle (okg_params.mg_collapse): level collapse_level and
  // everything below it as one symmetric dense operator, packed like the coarse inverse
  int collapse_level = -1, col_nb = 0;
  double *col_A = nullptr, *col_R = nullptr, *col_C = nullptr;
  int tail_start = -1;  // first level run by the cluster tail kernel (-1: none)
  int tail_cluster = 1;  // CTAs in the tail's thread-block cluster
  double* tail_tab = nullptr;  // tail weight tables (okg_tail.cuh)
  double b_int = 0;
  double* b_tab = nullptr;
  Nonlin nl;
  // linearisation
  double* coef = nullptr;
  bool have_lin = false;
  // Krylov
  int vcap = 0;
  double* V = nullptr;
  double *gb = nullptr, *gx = nullptr, *gr = nullptr, *pin = nullptr, *pz = nullptr, *pw = nullptr,
         *gt = nullptr;
  // preconditioner scratch
  double* cr2 = nullptr;  // scratch of the SSOR-preconditioned Chebyshev
  double* cad = nullptr;  // A d of the SSOR-preconditioned Chebyshev
  bool ssor = false;      // cheby_precond == "ssor" (okg_ssor.cuh)
  int ssor_cluster = 1;   // CTAs of the sweep kernels' cluster
  double *cd0 = nullptr, *cd1 = nullptr, *cr = nullptr, *r2p = nullptr, *sy = nullptr, *st = nullptr,
         *kv = nullptr, *zz = nullptr, *rr = nullptr, *z2 = nullptr, *shr = nullptr;
  // state
  double *u_old = nullptr, *w_old = nullptr, *u = nullptr, *w = nullptr;
  double t = 0;
  int step = 0;
  // reductions
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  double* dred = nullptr;
  double* hred = nullptr;  // pinned
  int* dflag = nullptr;
  size_t max_blocks = 0;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t g_arn = nullptr, g_prec = nullptr;
  int arn_nodes = 0, prec_nodes = 0;
  bool capturing = false;
  int cap_count = 0;
  std::vector<void*> allocs;
  size_t bytes = 0;
  // slab decomposition (see okg_group section below); one slab: rank 0 of 1
  int rank = 0, nslabs = 1;
  okg::Group* group = nullptr;
  size_t B = 0;        // fine-level vector stride (== N without ghost planes)
  ptrdiff_t foff = 0;  // flat pointer of a fine-level vector = global-indexed pointer + foff
  Seg seg{};           // owned entries of a stacked fine vector
  int L_rep = 1 << 30; // first replicated level
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::vector<std::pair<double*, int>> reg;  // exchange registry: (global-indexed pointer, level)
  double *io_a = nullptr, *io_b = nullptr, *io_c = nullptr;  // stacked staging of the host-pointer API
  bool handle = false;  // the user's handle of a multi-slab context (its slabs are group->r)
  // one process per GPU (okg_create_rank): the slab transport is NCCL instead of the group
  ncclComm_t comm = nullptr;
  const NcclApi* ncl = nullptr;
  std::vector<int> rep_lo, rep_hi;  // per slab: planes of the first replicated level it restricts into
};

namespace okg {

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
static double* dalloc(okg_ctx* c, size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(double));
  if (e != cudaSuccess) THROW(OKG_ENOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(double), cudaGetErrorString(e));
  CK(cudaMemsetAsync(p, 0, n * sizeof(double), c->stream));
  c->allocs.push_back(p);
  c->bytes += n * sizeof(double);
  return static_cast<double*>(p);
}

// A level vector: owned planes plus gh ghost planes per side, returned as a
// GLOBAL-INDEXED pointer (p[global vertex index] is valid for planes
// [ilo-gh, ihi+gh)), so every kernel indexes with global vertex numbers.
// nb > 1 allocates nb consecutive blocks of stride L.B (stacked vectors).
static double* lvec(okg_ctx* c, const Level& L, int l, int nb = 1) {
  double* base = dalloc(c, L.B * nb);
  double* g = base + (ptrdiff_t)L.gh * L.g.ps - (ptrdiff_t)L.g.ilo * L.g.ps;
  for (int q = 0; q < nb; ++q) c->reg.push_back({g + (ptrdiff_t)q * L.B, l});
  return g;
}

static void note(okg_ctx* c) {
  if (c->capturing) c->cap_count++;
  else g_launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) THROW(OKG_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
}

// every kernel goes through here: PDL attribute (okg_common.cuh) + launch count
template <class... KArgs, class... Args>
static void launch(okg_ctx* c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = c->p.disable_pdl ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) THROW(OKG_ECUDA, "cudaLaunchKernelEx: %s", cudaGetErrorString(e));
}

// one thread-block cluster of `csize` CTAs (k_vcycle_tail), PDL as above
template <class... KArgs, class... Args>
static void launch_cluster(okg_ctx* c, void (*kernel)(KArgs...), unsigned csize, dim3 block, size_t smem,
                           Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = c->p.disable_pdl ? 0 : 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = csize;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = csize > 1 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) THROW(OKG_ECUDA, "cudaLaunchKernelEx (cluster %u): %s", csize, cudaGetErrorString(e));
}

static unsigned nblk(size_t n) { return static_cast<unsigned>((n + BS - 1) / BS); }
// CTAs for one thread per owned vertex of a grid
static unsigned own(const Grid& g) { return std::max(1u, nblk((size_t)(g.hi - g.lo))); }
static unsigned vblk(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + BS - 1) / BS, 148 * 8)); }

static Reduce red(okg_ctx* c, int off) { return Reduce{c->partials, c->ticket, c->dred + off}; }
// layout of dred
enum { R_H = 0, R_C = 40, R_NRM = 80, R_RES = 90, R_JRES = 95, R_DOT = 100, R_FLAG = 105 };

static void sync_read(okg_ctx* c, int off, int cnt) {
  CK(cudaMemcpyAsync(c->hred + off, c->dred + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// flat pointer (allocation order, incl. ghost planes) of a fine-level vector
static double* F(okg_ctx* c, double* p) { return p + c->foff; }
static const double* F(okg_ctx* c, const double* p) { return p + c->foff; }

static void set_owned(Grid& g, int ilo, int ihi) {
  g.ilo = ilo;
  g.ihi = ihi;
  g.lo = (uint32_t)ilo * g.ps;
  g.hi = (uint32_t)ihi * g.ps;
}

// ---------------------------------------------------------------------------
// Slab group: one host thread + one stream per slab.  Ranks
// exchange one ghost plane per neighbour before every stencil kernel and
// allreduce their partial sums (in rank order: deterministic).  All the
// cross-slab ordering is CUDA events + host barriers; no kernel ever waits on
// another, so several slabs may share one GPU (the 1-GPU emulation the tests
// use) or sit on different GPUs (peer copies over NVLink).
// ---------------------------------------------------------------------------
struct Group {
  int S = 1;
  std::vector<okg_ctx*> r;
  std::atomic<int> count{0};
  std::atomic<long> gen{0};
  std::atomic<bool> abort{false};
  std::vector<double> scratch;  // [S][256] allreduce staging
  // worker threads
  std::vector<std::thread> th;
  std::mutex jm;
  std::condition_variable jcv, dcv;
  std::function<void(int)> job;
  long jgen = 0;
  int done = 0;
  bool stop = false;
  std::vector<int> status;
  std::vector<std::string> msg;
  std::atomic<int> first_err{-1};

  void barrier() {
    const long g = gen.load(std::memory_order_acquire);
    if (count.fetch_add(1, std::memory_order_acq_rel) + 1 == S) {
      count.store(0, std::memory_order_relaxed);
      gen.fetch_add(1, std::memory_order_acq_rel);
    } else {
      int spins = 0;
      while (gen.load(std::memory_order_acquire) == g) {
        if (abort.load(std::memory_order_relaxed)) THROW(OKG_EOTHER, "slab group aborted by another slab's error");
        if (++spins > 64) std::this_thread::yield();
      }
    }
  }
};

static void write_red(okg_ctx* c, int off, int cnt);
static void sync_read(okg_ctx* c, int off, int cnt);

static void allreduce(okg_ctx* c, int off, int cnt) {
  if (c->nslabs == 1) return;
  if (c->comm) {  // one process per GPU: NCCL allreduce of the staged sums (same result on every rank)
    write_red(c, off, cnt);
    NCK(c, c->ncl->AllReduce(c->dred + off, c->dred + off, cnt, ncclDouble, ncclSum, c->comm, c->stream));
    sync_read(c, off, cnt);
    return;
  }
  Group* G = c->group;
  for (int i = 0; i < cnt; ++i) G->scratch[(size_t)c->rank * 256 + i] = c->hred[off + i];
  G->barrier();
  for (int i = 0; i < cnt; ++i) {
    double s = 0.0;
    for (int q = 0; q < G->S; ++q) s += G->scratch[(size_t)q * 256 + i];
    c->hred[off + i] = s;
  }
  G->barrier();
}

// hred -> dred for kernels that consume reduction results on the device
static void write_red(okg_ctx* c, int off, int cnt) {
  CK(cudaMemcpyAsync(c->dred + off, c->hred + off, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
}

// The per-slab partial sums a kernel just left in dred[off .. off+cnt), summed over the slabs:
//  * reduce_to_host: the totals in hred on every slab (the host decides something with them);
//  * reduce_on_device: the totals in dred for the NEXT KERNEL -- with one process per GPU this
//    is one in-stream ncclAllReduce on the device scalars and no host round trip at all (the
//    CGS2 passes of an Arnoldi step chain three of them); the thread transport reduces on the
//    host in rank order (one stream synchronisation per reduction).
static void reduce_to_host(okg_ctx* c, int off, int cnt) {
  if (c->nslabs > 1 && c->comm) {
    NCK(c, c->ncl->AllReduce(c->dred + off, c->dred + off, cnt, ncclDouble, ncclSum, c->comm, c->stream));
    sync_read(c, off, cnt);
    return;
  }
  sync_read(c, off, cnt);
  allreduce(c, off, cnt);
}
static void reduce_on_device(okg_ctx* c, int off, int cnt) {
  if (c->nslabs == 1) return;
  if (c->comm) {
    NCK(c, c->ncl->AllReduce(c->dred + off, c->dred + off, cnt, ncclDouble, ncclSum, c->comm, c->stream));
    return;
  }
  sync_read(c, off, cnt);
  allreduce(c, off, cnt);
  write_red(c, off, cnt);
}

static int reg_index(okg_ctx* c, const double* x, int l) {
  for (size_t q = 0; q < c->reg.size(); ++q)
    if (c->reg[q].first == x && c->reg[q].second == l) return (int)q;
  THROW(OKG_EOTHER, "exchange: vector %p (level %d) is not a registered slab vector", (const void*)x, l);
}

// refresh the ghost planes of level-l vector x from the neighbouring slabs
static void exchange(okg_ctx* c, int l, const double* x) {
  if (c->nslabs == 1) return;
  const Level& L = c->lv[l];
  if (L.gh == 0) return;
  if (c->comm) {  // NCCL: boundary planes out, ghost planes in, both neighbours in one group
    double* v = const_cast<double*>(x);
    const size_t ps = L.g.ps;
    NCK(c, c->ncl->GroupStart());
    if (c->rank > 0) {
      NCK(c, c->ncl->Send(v + (size_t)L.g.ilo * ps, ps, ncclDouble, c->rank - 1, c->comm, c->stream));
      NCK(c, c->ncl->Recv(v + (size_t)(L.g.ilo - 1) * ps, ps, ncclDouble, c->rank - 1, c->comm, c->stream));
    }
    if (c->rank + 1 < c->nslabs) {
      NCK(c, c->ncl->Send(v + (size_t)(L.g.ihi - 1) * ps, ps, ncclDouble, c->rank + 1, c->comm, c->stream));
      NCK(c, c->ncl->Recv(v + (size_t)L.g.ihi * ps, ps, ncclDouble, c->rank + 1, c->comm, c->stream));
    }
    NCK(c, c->ncl->GroupEnd());
    return;
  }
  Group* G = c->group;
  const int q = reg_index(c, x, l);
  const size_t pb = (size_t)L.g.ps * sizeof(double);
  CK(cudaEventRecord(c->ev_a, c->stream));
  G->barrier();
  for (int nb : {c->rank - 1, c->rank + 1}) {
    if (nb < 0 || nb >= G->S) continue;
    okg_ctx* o = G->r[nb];
    CK(cudaStreamWaitEvent(c->stream, o->ev_a, 0));
    const int plane = nb < c->rank ? L.g.ilo - 1 : L.g.ihi;
    double* dst = const_cast<double*>(x) + (ptrdiff_t)plane * L.g.ps;
    const double* src = o->reg[q].first + (ptrdiff_t)plane * L.g.ps;
    CK(cudaMemcpyPeerAsync(dst, c->p.device, src, o->p.device, pb, c->stream));
  }
  CK(cudaEventRecord(c->ev_b, c->stream));
  G->barrier();
  for (int nb : {c->rank - 1, c->rank + 1})
    if (nb >= 0 && nb < G->S) CK(cudaStreamWaitEvent(c->stream, G->r[nb]->ev_b, 0));
}

// replicated level l: every slab computed the planes of its restriction range;
// copy them to all other slabs
static void allgather_planes(okg_ctx* c, int l, double* x) {
  if (c->nslabs == 1) return;
  const Level& L = c->lv[l];
  if (c->comm) {
    const size_t ps = L.g.ps;
    const int a = c->rep_lo[c->rank], b = c->rep_hi[c->rank];
    NCK(c, c->ncl->GroupStart());
    for (int o = 0; o < c->nslabs; ++o) {
      if (o == c->rank) continue;
      if (b > a) NCK(c, c->ncl->Send(x + (size_t)a * ps, (size_t)(b - a) * ps, ncclDouble, o, c->comm, c->stream));
      if (c->rep_hi[o] > c->rep_lo[o])
        NCK(c, c->ncl->Recv(x + (size_t)c->rep_lo[o] * ps, (size_t)(c->rep_hi[o] - c->rep_lo[o]) * ps, ncclDouble, o,
                           c->comm, c->stream));
    }
    NCK(c, c->ncl->GroupEnd());
    return;
  }
  Group* G = c->group;
  const int q = reg_index(c, x, l);
  CK(cudaEventRecord(c->ev_a, c->stream));
  G->barrier();
  for (int o = 0; o < G->S; ++o) {
    if (o == c->rank) continue;
    okg_ctx* oc = G->r[o];
    const Grid& fo = oc->lv[l - 1].g;  // the other slab's finer-level planes
    const int a = (fo.ilo + 1) / 2, b = (fo.ihi + 1) / 2;
    if (b <= a) continue;
    CK(cudaStreamWaitEvent(c->stream, oc->ev_a, 0));
    CK(cudaMemcpyPeerAsync(x + (ptrdiff_t)a * L.g.ps, c->p.device, oc->reg[q].first + (ptrdiff_t)a * L.g.ps,
                           oc->p.device, (size_t)(b - a) * L.g.ps * sizeof(double), c->stream));
  }
  CK(cudaEventRecord(c->ev_b, c->stream));
  G->barrier();
  for (int o = 0; o < G->S; ++o)
    if (o != c->rank) CK(cudaStreamWaitEvent(c->stream, G->r[o]->ev_b, 0));
}

// Slab partition: whole x-planes; boundaries even on the finest
// level, so that coarse ranges nest ((a+1)/2: coarse plane G is owned iff fine
// plane 2G is); from the first level where some slab would keep < 2 planes on
// (and always the coarsest), levels are replicated on every slab.  Writes the
// owned planes [lo[l], hi[l]) of `rank` for every split level and returns the
// first replicated level.  s0 = planes of the finest level, nlev = levels.
// A level is replicated (every slab holds and computes all of it) from the first level
// where some slab would keep fewer than 2 planes, from the first level below the finest
// with at most rep_max vertices in total, and always on the coarsest level.  The vertex
// rule is a cost model: one sweep of a whole level of N vertices costs
// max(4 us, N * 24 B / 5 TB/s) on one B200, a sweep of a 1/S share costs the share's
// time plus ~12 us for the ghost-plane exchange, so replicating wins below ~3 M vertices
// whatever S is.
static int64_t rep_max_default() { return 3000000; }
static int64_t rep_max_of(const okg_params& p) { return p.rep_max_vertices == 0 ? rep_max_default() : p.rep_max_vertices; }
static int slab_partition(int dim, int s0, int nlev, int S, int rank, int64_t rep_max, int* lo, int* hi) {
  auto fine = [&](int r, int& a, int& b) {
    a = 2 * (int)(((long)r * s0) / (2L * S));
    b = r == S - 1 ? s0 : 2 * (int)(((long)(r + 1) * s0) / (2L * S));
  };
  int a, b;
  fine(rank, a, b);
  for (int l = 0; l < nlev; ++l) {
    int minp = 1 << 30;
    for (int r = 0; r < S; ++r) {
      int ra, rb;
      fine(r, ra, rb);
      for (int k = 0; k < l; ++k) {
        ra = (ra + 1) / 2;
        rb = (rb + 1) / 2;
      }
      minp = std::min(minp, rb - ra);
    }
    const int64_t sl = (int64_t)((s0 - 1) >> l) + 1, Nl = dim == 2 ? sl * sl : sl * sl * sl;
    if (l > 0 && rep_max > 0 && Nl <= rep_max) return l;
    if (minp < 2 || l + 1 == nlev) return l;
    lo[l] = a;
    hi[l] = b;
    a = (a + 1) / 2;
    b = (b + 1) / 2;
  }
  return nlev;
}

static Grid make_grid(int dim, int n) {
  Grid g;
  g.n = n;
  g.s = n + 1;
  g.ps = dim == 2 ? (uint32_t)g.s : (uint32_t)g.s * (uint32_t)g.s;
  g.N = dim == 2 ? g.ps * (uint32_t)g.s : g.ps * (uint32_t)g.s;
  g.ilo = 0;
  g.ihi = g.s;
  g.lo = 0;
  g.hi = g.N;
  const int noff = dim == 2 ? 7 : 15;
  for (int o = 0; o < 15; ++o) {
    if (o >= noff) {
      g.off[o] = 0;
      continue;
    }
    if (dim == 2) g.off[o] = off_comp(2, o, 0) * g.s + off_comp(2, o, 1);
    else g.off[o] = off_comp(3, o, 0) * (int)g.ps + off_comp(3, o, 1) * g.s + off_comp(3, o, 2);
  }
  return g;
}

// weights w(cls,o) = a * U1(cls,o) + b * U2(cls,o)  (a*U1 when U2 null)
static HostOp make_op(okg_ctx* c, const UnitTables& ut, const std::vector<double>& U1, double a,
                      const std::vector<double>* U2, double b, bool add_form) {
  HostOp op;
  const int ncls = ut.ncls, noff = ut.noff, center = noff / 2;
  const int interior = ncls / 2;
  op.htab.assign(static_cast<size_t>(ncls) * (noff + 1), 0.0);
  for (int cl = 0; cl < ncls; ++cl) {
    for (int o = 0; o < noff; ++o) {
      const double u1 = U1[static_cast<size_t>(cl) * noff + o];
      double v = u1 * a;
      if (U2) {
        const double u2 = (*U2)[static_cast<size_t>(cl) * noff + o];
        // add(M, alpha, K) (sparse.hpp:183-196): M_ij + alpha*K_ij
        v = add_form ? v + b * u2 : v;
      }
      op.htab[static_cast<size_t>(cl) * (noff + 1) + o] = v;
    }
    const double d = op.htab[static_cast<size_t>(cl) * (noff + 1) + center];
    if (!(d > 0.0)) THROW(OKG_ENUMERICAL, "operator: non-positive diagonal entry");
    op.htab[static_cast<size_t>(cl) * (noff + 1) + noff] = 1.0 / d;
  }
  for (int o = 0; o < 15; ++o) op.w[o] = o < noff ? op.htab[static_cast<size_t>(interior) * (noff + 1) + o] : 0.0;
  op.invd = op.htab[static_cast<size_t>(interior) * (noff + 1) + noff];
  op.tab = dalloc(c, op.htab.size());
  CK(cudaMemcpyAsync(op.tab, op.htab.data(), op.htab.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return op;
}

static double ipow(double h, int k) {
  double r = 1.0;
  for (int i = 0; i < k; ++i) r *= h;
  return r;
}

// ---------------------------------------------------------------------------
// kernel launch wrappers (DIM-templated)
// ---------------------------------------------------------------------------
template <int DIM>
static void op_apply(okg_ctx* c, const Grid& g, const HostOp& op, int epi, const double* x, const double* b,
                     double* y, double* acc, double omega = 0.0) {
  const Op<DIM> o = dev_op<DIM>(op);
  switch (epi) {
    case EPI_APPLY: launch(c, k_op<DIM, EPI_APPLY>, own(g), BS, 0, g, o, x, b, y, acc, omega); break;
    case EPI_RESID: launch(c, k_op<DIM, EPI_RESID>, own(g), BS, 0, g, o, x, b, y, acc, omega); break;
    case EPI_JACOBI: launch(c, k_op<DIM, EPI_JACOBI>, own(g), BS, 0, g, o, x, b, y, acc, omega); break;
    case EPI_JACOBI_SET:
      launch(c, k_op<DIM, EPI_JACOBI_SET>, own(g), BS, 0, g, o, x, b, y, acc, omega);
      break;
    case EPI_JACOBI_ACC:
      launch(c, k_op<DIM, EPI_JACOBI_ACC>, own(g), BS, 0, g, o, x, b, y, acc, omega);
      break;
    case EPI_SCALE_APPLY:
      launch(c, k_op<DIM, EPI_SCALE_APPLY>, own(g), BS, 0, g, o, x, b, y, acc, omega);
      break;
  }
  note(c);
}

// shared-memory carveout (percent) of the tiled stencil kernels
#ifndef OKG_CARVEOUT
#define OKG_CARVEOUT 50
#endif
constexpr int SMEM_CARVEOUT = OKG_CARVEOUT;

template <int DIM, int LOAD, int EPI, int TI, int WIDE>
static void tiled_tw(okg_ctx* c, const Level& L, const HostOp& op, const TArgs& a) {
  static bool attr = false;  // dynamic smem above 48 KB needs an opt-in (per kernel instance)
  const size_t smem = tiled_smem_bytes<DIM, LOAD, TI, WIDE>();
  if (!attr) {
    CK(cudaFuncSetAttribute(k_tiled<DIM, LOAD, EPI, TI, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // half of the unified L1/shared array as shared memory: the tiles of 4 CTAs fit, and
    // the rest stays L1 for the cp.async (.ca) and pointwise loads -- measured at 400^3:
    // carveout 100 -> 430 us, 50 -> 267 us per fine-level sweep (30: 320 us)
    CK(cudaFuncSetAttribute(k_tiled<DIM, LOAD, EPI, TI, WIDE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            SMEM_CARVEOUT));
    attr = true;
  }
  launch(c, k_tiled<DIM, LOAD, EPI, TI, WIDE>, L.tl_blocks, TileCfg<DIM>::NT, smem, L.g, dev_op<DIM>(op), L.tl, a);
  note(c);
}

// 16-byte staging (k_tiled's WIDE) for the plain-load kernels of levels with an odd row pitch
template <int DIM, int LOAD, int EPI, int TI>
static void tiled_ti(okg_ctx* c, const Level& L, const HostOp& op, const TArgs& a) {
  // (the Chebyshev step measured no faster with it: 128^3 18.1 vs 18.5 us, 400^3 546 vs 554 us)
  // and the prolongation-staged sweep in 3D slower: 400^3 467 vs 442 us; pre-sweep kernel 289 vs 303 us,
  // 2D: pre-sweeps 13.9 vs 15.6 us, prolongation sweep 20.1 vs 23.2 us)
  if constexpr (EPI != T_CHEB && !(LOAD == L_PROLONG && (TI < 4 || DIM == 3))) {
    if (L.wide && (LOAD == L_PLAIN || L.wide_xf) && (TI >= 4 || L.wide_thin)) {
      tiled_tw<DIM, LOAD, EPI, TI, 1>(c, L, op, a);
      return;
    }
  }
  tiled_tw<DIM, LOAD, EPI, TI, 0>(c, L, op, a);
}

template <int DIM, int LOAD, int EPI>
static void tiled(okg_ctx* c, const Level& L, const HostOp& op, const TArgs& a) {
  if (L.tl.ichunk == 8) tiled_ti<DIM, LOAD, EPI, 8>(c, L, op, a);
  else if (L.tl.ichunk == 4) tiled_ti<DIM, LOAD, EPI, 4>(c, L, op, a);
  else if (L.tl.ichunk == 3) tiled_ti<DIM, LOAD, EPI, 3>(c, L, op, a);
  else tiled_ti<DIM, LOAD, EPI, 2>(c, L, op, a);
}

static TArgs targs(const double* x, const double* b, double* y, double* acc, double omega) {
  TArgs a;
  std::memset(&a, 0, sizeof a);
  a.x = x;
  a.b = b;
  a.y = y;
  a.acc = acc;
  a.omega = omega;
  return a;
}

// core tiles + boundary list for one grid (okg_tiled.cuh)
template <int DIM>
static void make_tiling(okg_ctx* c, Level& L) {
  const int n = L.g.n;
  using TC = TileCfg<DIM>;
  Tiling& t = L.tl;
  t.ktiles = (n - 1 + TC::TK - 1) / TC::TK;
  t.jtiles = DIM == 3 ? (n - 1 + TC::TJ - 1) / TC::TJ : 1;
  // interior planes of this slab
  t.ci0 = std::max(1, L.g.ilo);
  t.ci1 = std::min(n, L.g.ihi);
  const int nci = std::max(0, t.ci1 - t.ci0);
  const int base = t.ktiles * t.jtiles;
  // C-block kernels (okg_tiled_c.cuh): vertices per thread along x 4 in 3D (register
  // budget), 8 in 2D; smaller when the level is too small to give each SM a few CTAs
  auto chunking = [&](int ichunk, Tiling& tt) {
    while (ichunk > 2 && base * ((nci + ichunk - 1) / ichunk) < 148 * 4) ichunk /= 2;
    tt.ichunk = ichunk;
    tt.ncore = base * ((nci + ichunk - 1) / ichunk);
  };
  std::vector<uint32_t> bnd;
  const int s = n + 1;
  if (DIM == 3) {
    for (int i = L.g.ilo; i < L.g.ihi; ++i)
      for (int j = 0; j < s; ++j)
        for (int k = 0; k < s; ++k)
          if (i == 0 || i == n || j == 0 || j == n || k == 0 || k == n)
            bnd.push_back((uint32_t)((i * s + j) * s + k));
  } else {
    for (int i = L.g.ilo; i < L.g.ihi; ++i)
      for (int k = 0; k < s; ++k)
        if (i == 0 || i == n || k == 0 || k == n) bnd.push_back((uint32_t)(i * s + k));
  }
  t.nbnd = (uint32_t)bnd.size();
  const int nbb = (int)((t.nbnd + TC::NT - 1) / TC::NT);
  {
    // planes per core CTA: the k_tiled grid runs in waves of 148 x 4 CTAs (4 per SM by
    // registers), and a CTA's time grows like TI + 4 (staging halo + fixed cost), so
    // take the TI in {8, 4, 3, 2} with the fewest waves x (TI + 4) (ties: larger TI).
    // Measured against "largest power of two with >= 4 CTAs per SM": 65^3 level TI 2
    // -> 3 (one wave instead of 609 CTAs on 592 slots), 1025^2 TI 4 -> 8 (one wave):
    // 3D 128^3 49.1 -> 48.8 ms, 2D 2048^2 61.1 -> 60.5 ms per step, 400^3 unchanged
    int best = 8;
    long bestc = -1;
    for (int ti : {8, 4, 3, 2}) {
      const long T = (long)base * ((nci + ti - 1) / ti) + nbb;
      const long cost = ((T + 148 * 4 - 1) / (148 * 4)) * (ti + 4);
      if (bestc < 0 || cost < bestc) {
        bestc = cost;
        best = ti;
      }
    }
    t.ichunk = best;
    t.ncore = base * ((nci + best - 1) / best);
  }
  t.vend = (uint32_t)(L.g.ihi + L.gh) * L.g.ps;
  {
    const char* e = std::getenv("OKG_WIDE");  // A/B at okg_create: OKG_WIDE=0 keeps the 8-byte staging
    L.wide = (L.g.s & 1) && !(e && std::atoi(e) == 0);
    L.wide_xf = L.wide && !(e && std::atoi(e) == 1);  // A/B: OKG_WIDE=1 plain-load kernels only
    L.wide_thin = L.wide && !(e && std::atoi(e) == 2);  // A/B: OKG_WIDE=2 tiles of 4 and 8 planes only
  }
  double* d = dalloc(c, (bnd.size() + 1) / 2 + 1);
  CK(cudaMemcpyAsync(d, bnd.data(), bnd.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  t.bnd = reinterpret_cast<const uint32_t*>(d);
  L.tl_blocks = (unsigned)t.ncore + (unsigned)((t.nbnd + TC::NT - 1) / TC::NT);
  L.tlc = t;
  chunking(DIM == 3 ? 4 : 8, L.tlc);
  L.tlc_blocks = (unsigned)L.tlc.ncore + (unsigned)((t.nbnd + TC::NT - 1) / TC::NT);
  L.tiled = true;
}

static void axpy(okg_ctx* c, double a, const double* x, double* y, size_t n) {
  launch(c, k_axpy, vblk(n), BS, 0, a, x, y, n);
  note(c);
}
static void scale(okg_ctx* c, double s, const double* x, double* y, size_t n) {
  launch(c, k_scale, vblk(n), BS, 0, s, x, y, n);
  note(c);
}
static void copy(okg_ctx* c, const double* x, double* y, size_t n) {
  CK(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
}

// y = A x, A symmetric as packed CB-blocks (coarsest inverse / collapsed bottom): every
// block is streamed once and forms both of its products (k_coarse_sym), then the
// partials of a row are summed in a fixed order (k_coarse_sym_sum).  (One launch with a
// last-contributor row sum was bit-identical but slower -- DESIGN section 5 item 10.)
static void coarse_sym_apply(okg_ctx* c, int n, int nb, const double* A, const double* x, double* R, double* C,
                             double* y) {
  const unsigned nblk = (unsigned)(nb * (nb + 1) / 2);
  launch(c, k_coarse_sym, nblk, 256, 0, n, A, x, R, C);
  note(c);
  launch(c, k_coarse_sym_sum, (unsigned)nb, CB * CSEG, 0, n, nb, (const double*)R, (const double*)C, y);
  note(c);
}

// ---- multigrid (multigrid.hpp:97-149) --------------------------------------
static void allgather_planes(okg_ctx* c, int l, double* x);

template <int DIM>
static void coarse_solve(okg_ctx* c, const double* b, double* y) {
  if (!c->coarse_big) {
    launch(c, k_coarse_solve, (c->nc + BS / 32 - 1) / (BS / 32), BS, 0, c->nc, c->Ainv, b, y);
    note(c);
    return;
  }
  // large coarsest level: this slab's rows of the inverse, then (split) the planes of
  // every slab's rows are all-gathered -- the same ranges the restriction gathers
  Level& L = c->lv.back();
  const int last = (int)c->lv.size() - 1;
  if (reinterpret_cast<uintptr_t>(b) % 16 != 0) {
    copy(c, b, L.eb, (size_t)c->nc);
    b = L.eb;
  }
  if (c->coarse_nb > 0) {  // one slab: half the bytes through the symmetric block triangle
    const int nb = c->coarse_nb;
    coarse_sym_apply(c, c->nc, nb, c->Ainv, b, c->coarse_R, c->coarse_C, y);
    return;
  }
  double* tgt = c->coarse_split ? L.ea : y;
  const int rows = c->coarse_r1 - c->coarse_r0;
  launch(c, k_coarse_gemv, (rows + BS / 32 - 1) / (BS / 32), BS, 0, c->nc, c->coarse_r0, c->coarse_r1, c->coarse_ld,
         (const double*)c->Ainv, b, tgt);
  note(c);
  if (c->coarse_split) {
    allgather_planes(c, last, L.ea);
    if (y != L.ea) copy(c, L.ea, y, (size_t)c->nc);
  }
}

template <int DIM>
static void mg_level(okg_ctx* c, int l, const double* rhs, double* out, bool acc);

// see okg_params.mg_collapse: column i of the level-lc cycle operator is the cycle
// applied to e_i; the (numerically symmetric) N x N result is packed as a lower block
// triangle (k_coarse_pack takes its row-major upper triangle)
template <int DIM>
static void collapse_levels(okg_ctx* c, int lc) {
  Level& L = c->lv[lc];
  const int N = (int)L.g.N;
  double* F = nullptr;
  const size_t nn = (size_t)N * N;
  cudaError_t e = cudaMalloc(&F, nn * sizeof(double));
  if (e != cudaSuccess) THROW(OKG_ENOMEM, "cudaMalloc(%zu bytes) for the collapsed cycle: %s", nn * sizeof(double),
                              cudaGetErrorString(e));
  try {
    for (int i = 0; i < N; ++i) {
      k_unit<<<(N + 255) / 256, 256, 0, c->stream>>>(L.b, N, i);
      CK(cudaGetLastError());
      mg_level<DIM>(c, lc, L.b, L.x, false);
      CK(cudaMemcpyAsync(F + (size_t)i * N, L.x, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    const int nb = (N + CB - 1) / CB;
    const size_t nblk = (size_t)nb * (nb + 1) / 2;
    c->col_A = dalloc(c, nblk * CB * CB);
    c->col_R = dalloc(c, nblk * CB);
    c->col_C = dalloc(c, nblk * CB);
    k_coarse_pack<<<148 * 8, 256, 0, c->stream>>>(N, nb, F, c->col_A);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  } catch (...) {
    cudaFree(F);
    throw;
  }
  cudaFree(F);
  c->col_nb = (N + CB - 1) / CB;
  c->collapse_level = lc;
  c->tail_start = -1;  // the tail's levels are inside the collapsed operator
}

// Setup of the large coarsest level (nc > 2000): Cholesky + inverse of the dense
// operator on the device (cuSOLVER potrf/potri, okg_cusolver.h), then rows
// [r0, r1) are written in full (stride ld) to c->Ainv.  The host path
// (dense_spd_inverse) is O(nc^3) on one core: hours at 26^3 = 17,576.
static void coarse_inverse_device(okg_ctx* c, const std::vector<double>& Ad, int nc, int r0, int r1) {
  std::string why;
  const CusolverApi* cs = cusolver_api(&why);
  if (!cs) THROW(OKG_ECUDA, "coarse solve (%d unknowns > 2000): %s", nc, why.c_str());
  const size_t nn = (size_t)nc * nc;
  double* F = nullptr;
  int* info = nullptr;
  double* work = nullptr;
  cusolverDnHandle_t h = nullptr;
  auto cleanup = [&]() {
    if (h) cs->Destroy(h);
    cudaFree(F);
    cudaFree(info);
    cudaFree(work);
  };
  try {
    cudaError_t e = cudaMalloc(&F, nn * sizeof(double));
    if (e != cudaSuccess) THROW(OKG_ENOMEM, "cudaMalloc(%zu bytes) for the coarse factor: %s", nn * sizeof(double),
                                cudaGetErrorString(e));
    CK(cudaMalloc(&info, sizeof(int)));
    CK(cudaMemcpyAsync(F, Ad.data(), nn * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (cs->Create(&h) != CUSOLVER_STATUS_SUCCESS) THROW(OKG_ECUDA, "cusolverDnCreate failed");
    cs->SetStream(h, c->stream);
    int lw1 = 0, lw2 = 0;
    if (cs->PotrfBufferSize(h, CUBLAS_FILL_MODE_LOWER, nc, F, nc, &lw1) != CUSOLVER_STATUS_SUCCESS ||
        cs->PotriBufferSize(h, CUBLAS_FILL_MODE_LOWER, nc, F, nc, &lw2) != CUSOLVER_STATUS_SUCCESS)
      THROW(OKG_ECUDA, "cusolverDn potrf/potri bufferSize failed");
    const int lw = std::max(std::max(lw1, lw2), 1);
    CK(cudaMalloc(&work, (size_t)lw * sizeof(double)));
    int hinfo = 0;
    if (cs->Potrf(h, CUBLAS_FILL_MODE_LOWER, nc, F, nc, work, lw, info) != CUSOLVER_STATUS_SUCCESS)
      THROW(OKG_ECUDA, "cusolverDnDpotrf failed");
    CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hinfo != 0) THROW(OKG_ENUMERICAL, "Cholesky: matrix not positive definite");
    if (cs->Potri(h, CUBLAS_FILL_MODE_LOWER, nc, F, nc, work, lw, info) != CUSOLVER_STATUS_SUCCESS)
      THROW(OKG_ECUDA, "cusolverDnDpotri failed");
    CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hinfo != 0) THROW(OKG_ENUMERICAL, "Cholesky: inverse failed (info %d)", hinfo);
    const size_t ld = (size_t)(nc + 1) & ~(size_t)1;
    if (r0 == 0 && r1 == nc && c->p.coarse_split >= 0) {
      // all rows on this slab: symmetric packed blocks
      const int nb = (nc + CB - 1) / CB;
      const size_t nblk = (size_t)nb * (nb + 1) / 2;
      c->Ainv = dalloc(c, nblk * CB * CB);
      c->coarse_R = dalloc(c, nblk * CB);
      c->coarse_C = dalloc(c, nblk * CB);
      k_coarse_pack<<<148 * 8, 256, 0, c->stream>>>(nc, nb, F, c->Ainv);
      c->coarse_nb = nb;
    } else {
      c->Ainv = dalloc(c, (size_t)(r1 - r0) * ld);
      k_coarse_rows<<<148 * 8, 256, 0, c->stream>>>(nc, r0, r1, ld, F, c->Ainv);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    c->coarse_ld = ld;
    c->coarse_r0 = r0;
    c->coarse_r1 = r1;
    c->coarse_big = true;
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

// levels tail_start..coarsest in one launch (okg_tail.cuh)
template <int DIM, int N0>
static size_t tail_smem(int nc, int csize) {
  const int rows = (nc + csize - 1) / csize;
  return sizeof(double) * ((size_t)tail_smem_doubles<DIM, N0>() + TL<DIM, N0>::N + (size_t)rows * nc);
}

template <int DIM, int N0>
static void tail_launch(okg_ctx* c, const TailArgs<DIM>& A) {
  launch_cluster(c, k_vcycle_tail<DIM, N0>, (unsigned)c->tail_cluster, TAIL_NT, tail_smem<DIM, N0>(c->nc, c->tail_cluster),
                 A);
}

// per instantiation: opt in to the shared memory / cluster size it needs
template <int DIM, int N0>
static void tail_prepare(okg_ctx* c) {
  CK(cudaFuncSetAttribute(k_vcycle_tail<DIM, N0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)tail_smem<DIM, N0>(c->nc, c->tail_cluster)));
  if (c->tail_cluster > 8)
    CK(cudaFuncSetAttribute(k_vcycle_tail<DIM, N0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

template <int DIM, class F>
static void tail_dispatch(int n0, F&& f) {
  switch (n0) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    case 32: if constexpr (DIM == 2) f(std::integral_constant<int, 32>{}); break;
    case 64: if constexpr (DIM == 2) f(std::integral_constant<int, 64>{}); break;
    default: THROW(OKG_EOTHER, "tail: unsupported first level n = %d", n0);
  }
}

template <int DIM>
static void run_tail(okg_ctx* c, int l0, const double* rhs, double* out) {
  TailArgs<DIM> A;
  std::memset(&A, 0, sizeof A);
  A.tabs = c->tail_tab;
  A.nl = static_cast<int>(c->lv.size()) - l0;
  A.omega = c->p.mg_omega;
  A.rhs = rhs;
  A.out = out;
  A.Ainv = c->Ainv;
  A.nc = c->nc;
  tail_dispatch<DIM>(c->lv[l0].g.n, [&](auto N0) { tail_launch<DIM, decltype(N0)::value>(c, A); });
  note(c);
}

template <int DIM>
static void mg_level(okg_ctx* c, int l, const double* rhs, double* out, bool acc);

template <int DIM, int BX>
static void mg_fused(okg_ctx* c, int l, const double* rhs, double* out, bool acc) {
  Level& L = c->lv[l];
  Level& C = c->lv[l + 1];
  const Op<DIM> op = dev_op<DIM>(L.shat);
  const double om = c->p.mg_omega;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_mg_down<DIM, BX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mg_down_smem<DIM, BX>()));
    CK(cudaFuncSetAttribute(k_mg_up<DIM, BX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mg_up_smem<DIM, BX>()));
    CK(cudaFuncSetAttribute(k_mg_up<DIM, BX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mg_up_smem<DIM, BX>()));
    attr = true;
  }
  launch(c, k_mg_down<DIM, BX>, mg_boxes<DIM, BX>(L.g), MgBox<DIM, BX>::NT, mg_down_smem<DIM, BX>(), L.g, C.g, op, om, rhs,
         L.ea, C.b);
  note(c);
  mg_level<DIM>(c, l + 1, C.b, C.x, false);
  if (acc) launch(c, k_mg_up<DIM, BX, true>, mg_boxes<DIM, BX>(L.g), MgBox<DIM, BX>::NT, mg_up_smem<DIM, BX>(), L.g, C.g,
                  op, om, rhs, (const double*)L.ea, (const double*)C.x, out);
  else launch(c, k_mg_up<DIM, BX, false>, mg_boxes<DIM, BX>(L.g), MgBox<DIM, BX>::NT, mg_up_smem<DIM, BX>(), L.g, C.g,
              op, om, rhs, (const double*)L.ea, (const double*)C.x, out);
  note(c);
}

template <int DIM>
static void mg_level(okg_ctx* c, int l, const double* rhs, double* out, bool acc) {
  Level& L = c->lv[l];
  const int last = static_cast<int>(c->lv.size()) - 1;
  if (l == c->collapse_level && !acc) {  // the whole cycle below l in one matvec
    const int nb = c->col_nb;
    coarse_sym_apply(c, (int)L.g.N, nb, c->col_A, rhs, c->col_R, c->col_C, out);
    return;
  }
  if (l == c->tail_start && !acc && l > 0) {
    run_tail<DIM>(c, l, rhs, out);
    return;
  }
  if (l == last) {
    if (!acc) {
      coarse_solve<DIM>(c, rhs, out);
    } else {
      coarse_solve<DIM>(c, rhs, L.ea);
      axpy(c, 1.0, L.ea + L.g.lo, out + L.g.lo, L.g.hi - L.g.lo);
    }
    return;
  }
  const double om = c->p.mg_omega;
  const Op<DIM> op = dev_op<DIM>(L.shat);
  if (L.fused) {  // V(2,2) in two launches (okg_vcycle.cuh)
    // BX = 1 (larger box) measured no better on the big levels; kept for experiments
    mg_fused<DIM, 0>(c, l, rhs, out, acc);
    return;
  }
  double* cur = L.ea;
  double* oth = L.eb;
  const int pre = c->p.mg_pre, post = c->p.mg_post;
  // ---- pre-smoothing from zero (multigrid.hpp:102-104)
  if (pre == 0) {
    CK(cudaMemsetAsync(cur + L.g.lo, 0, (L.g.hi - L.g.lo) * sizeof(double), c->stream));
  } else if (pre >= 2) {
    exchange(c, l, rhs);
    if (L.tiled) tiled<DIM, L_JAC0, T_JACOBI>(c, L, L.shat, targs(rhs, rhs, cur, nullptr, om));
    else {
      launch(c, k_pre2<DIM>, own(L.g), BS, 0, L.g, op, rhs, cur, om);
      note(c);
    }
    for (int s = 2; s < pre; ++s) {
      exchange(c, l, cur);
      if (L.tiled) tiled<DIM, L_PLAIN, T_JACOBI>(c, L, L.shat, targs(cur, rhs, oth, nullptr, om));
      else op_apply<DIM>(c, L.g, L.shat, EPI_JACOBI, cur, rhs, oth, nullptr, om);
      std::swap(cur, oth);
    }
  } else {
    launch(c, k_jacobi0<DIM>, own(L.g), BS, 0, L.g, op, rhs, cur, om);
    note(c);
  }
  // ---- residual, restriction, coarse correction (multigrid.hpp:106-110)
  Level& C = c->lv[l + 1];
  exchange(c, l, cur);
  if (L.tiled) tiled<DIM, L_PLAIN, T_RESID>(c, L, L.shat, targs(cur, rhs, L.res, nullptr, 0.0));
  else op_apply<DIM>(c, L.g, L.shat, EPI_RESID, cur, rhs, L.res, nullptr);
  exchange(c, l, L.res);
  {
    // coarse vertices G with 2G in this slab's planes (all of them when not split)
    Grid gcr = C.g;
    if (C.rep && !L.rep) set_owned(gcr, (L.g.ilo + 1) / 2, (L.g.ihi + 1) / 2);
    launch(c, k_restrict<DIM>, own(gcr), BS, 0, L.g, gcr, (const double*)L.res, C.b);
    note(c);
    if (C.rep && !L.rep) allgather_planes(c, l + 1, C.b);
  }
  mg_level<DIM>(c, l + 1, C.b, C.x, false);
  // ---- prolongation + post-smoothing (multigrid.hpp:111-115)
  exchange(c, l + 1, C.x);
  if (post == 0 || !L.tiled) {
    launch(c, k_prolong_add<DIM>, own(L.g), BS, 0, L.g, C.g, (const double*)C.x, cur);
    note(c);
  }
  for (int s = 0; s < post; ++s) {
    const bool lastsweep = (s == post - 1);
    exchange(c, l, cur);
    if (L.tiled) {
      TArgs a = targs(cur, rhs, lastsweep ? nullptr : oth, lastsweep ? out : nullptr, om);
      if (s == 0) {  // stage e + P e_c: the correction is fused into this sweep
        a.x2 = C.x;
        a.gc = C.g;
        if (!lastsweep) tiled<DIM, L_PROLONG, T_JACOBI>(c, L, L.shat, a);
        else if (acc) tiled<DIM, L_PROLONG, T_JACOBI_ACC>(c, L, L.shat, a);
        else tiled<DIM, L_PROLONG, T_JACOBI_SET>(c, L, L.shat, a);
      } else {
        if (!lastsweep) tiled<DIM, L_PLAIN, T_JACOBI>(c, L, L.shat, a);
        else if (acc) tiled<DIM, L_PLAIN, T_JACOBI_ACC>(c, L, L.shat, a);
        else tiled<DIM, L_PLAIN, T_JACOBI_SET>(c, L, L.shat, a);
      }
    } else if (lastsweep) {
      op_apply<DIM>(c, L.g, L.shat, acc ? EPI_JACOBI_ACC : EPI_JACOBI_SET, cur, rhs, nullptr, out, om);
    } else {
      op_apply<DIM>(c, L.g, L.shat, EPI_JACOBI, cur, rhs, oth, nullptr, om);
    }
    if (!lastsweep) std::swap(cur, oth);
  }
  if (post == 0) {
    if (acc) axpy(c, 1.0, cur + L.g.lo, out + L.g.lo, L.g.hi - L.g.lo);
    else copy(c, cur + L.g.lo, out + L.g.lo, L.g.hi - L.g.lo);
  }
}

// plain apply y = A x on level l (tiled when the level is)
template <int DIM>
static void apply_level(okg_ctx* c, int l, const HostOp& op, const double* x, double* y) {
  const Level& L = c->lv[l];
  exchange(c, l, x);
  if (L.tiled) tiled<DIM, L_PLAIN, T_APPLY>(c, L, op, targs(x, nullptr, y, nullptr, 0.0));
  else op_apply<DIM>(c, L.g, op, EPI_APPLY, x, nullptr, y, nullptr);
}

// apply_shat_inv (multigrid.hpp:133-149): `cycles` V-cycles composed by Richardson
template <int DIM>
static void shat_inv(okg_ctx* c, const double* b, double* x, int cycles) {
  for (int cyc = 0; cyc < cycles; ++cyc) {
    const double* rhs = cyc == 0 ? b : c->shr;
    mg_level<DIM>(c, 0, rhs, x, cyc > 0);
    if (cyc + 1 == cycles) break;
    exchange(c, 0, x);
    if (c->lv[0].tiled) tiled<DIM, L_PLAIN, T_RESID>(c, c->lv[0], c->lv[0].shat, targs(x, b, c->shr, nullptr, 0.0));
    else op_apply<DIM>(c, c->lv[0].g, c->lv[0].shat, EPI_RESID, x, b, c->shr, nullptr);
  }
}

template <int DIM>
static void cheb_ssor(okg_ctx* c, const HostOp& A, const double* b, double* x);

// ---- Chebyshev (krylov.hpp:158-202) ---------------------------------------------
template <int DIM>
static void cheb(okg_ctx* c, const HostOp& A, const double* b, double* x) {
  if (c->ssor) {
    cheb_ssor<DIM>(c, A, b, x);
    return;
  }
  const Grid& g = c->fine;
  const Op<DIM> o = dev_op<DIM>(A);
  const int k = c->p.cheby_iters;
  double* dcur = c->cd0;
  double* dnxt = c->cd1;
  // one slab, tiled finest level: the start vector d0 = (D^-1 r)/theta is formed by the first
  // step's staging transform (k_tiled L_CHEB0, k_cheb_first's rounding): one launch and
  // 32 B/vertex less per Chebyshev solve.  OKG_CHEB0=0 at okg_create keeps the separate kernel.
  const bool fuse0 = k >= 2 && c->lv[0].tiled && c->nslabs == 1 && c->cheb_fuse0;
  if (!fuse0) {
    launch(c, k_cheb_first<DIM>, own(g), BS, 0, g, o, b, dcur, c->cheb_inv_theta);
    note(c);
  }
  if (k == 1) {
    copy(c, dcur + g.lo, x + g.lo, g.hi - g.lo);
    return;
  }
  // (two steps per pass -- a halo-2 tile -- was bit-identical but 0.4 % slower per 2D step
  // and is gone: DESIGN section 5)
  for (int j = 0; j + 1 < k; ++j) {
    const int last = (j == k - 2);
    // x is updated every other step from j = 1 on: an odd step with a successor leaves x alone
    // (mode 1), the even step after it adds both directions in the reference's order (mode 2,
    // bit-identical): 16 of 48 B/vertex less on the skipped steps of an HBM-bound kernel
    const int xmode = j == 0 ? 0 : ((j & 1) ? (last ? 0 : 1) : 2);
    if (j == 0 && fuse0) {
      TArgs a = targs(b, b, c->cr, x, 0.0);
      a.y2 = dnxt;
      a.c1 = c->cheb_c1[0];
      a.c2 = c->cheb_c2[0];
      a.inv_theta = c->cheb_inv_theta;
      a.last = last;
      tiled<DIM, L_CHEB0, T_CHEB>(c, c->lv[0], A, a);
      std::swap(dcur, dnxt);
      continue;
    }
    exchange(c, 0, dcur);
    if (c->lv[0].tiled) {
      TArgs a = targs(dcur, j == 0 ? b : c->cr, c->cr, x, 0.0);
      a.x2 = j == 0 ? dcur : x;
      a.y2 = dnxt;
      a.c1 = c->cheb_c1[j];
      a.c2 = c->cheb_c2[j];
      a.last = last;
      a.xmode = xmode;
      tiled<DIM, L_PLAIN, T_CHEB>(c, c->lv[0], A, a);
    } else {
      launch(c, k_cheb_step<DIM>, own(g), BS, 0, g, o, dcur, j == 0 ? b : c->cr, j == 0 ? dcur : x, dnxt,
                                                        c->cr, x, c->cheb_c1[j], c->cheb_c2[j], last, xmode);
      note(c);
    }
    std::swap(dcur, dnxt);
  }
}

// ---- u-dependent blocks ---------------------------------------------------------
template <int DIM, int MODE, int TI>
static void tiled_c(okg_ctx* c, const CTArgs& t, Reduce rd) {
  static bool attr = false;
  const size_t smem = (size_t)CNeeds<MODE>::NOPS * (TI + 2) * TileCfg<DIM>::PSZ * sizeof(double);
  if (!attr) {
    CK(cudaFuncSetAttribute(k_tiled_c<DIM, MODE, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tiled_c<DIM, MODE, TI>, cudaFuncAttributePreferredSharedMemoryCarveout, SMEM_CARVEOUT));
    attr = true;
  }
  const Level& L0 = c->lv[0];
  launch(c, k_tiled_c<DIM, MODE, TI>, L0.tlc_blocks, TileCfg<DIM>::NT, smem,
      L0.g, dev_op<DIM>(c->M), dev_op<DIM>(c->K), dev_op<DIM>(c->A), L0.tlc, t, rd);
  note(c);
}

template <int DIM, int MODE>
static void capply(okg_ctx* c, const double* x, const double* v, const double* b, double* y, double s1,
                   Reduce rd = Reduce{nullptr, nullptr, nullptr}) {
  CArgs a;
  a.x = x;
  a.v = v;
  a.b = b;
  a.y = y;
  a.coef = c->coef;
  a.ldc = c->B;
  a.n2 = c->B;
  a.s1 = s1;
  a.s2 = 0.0;
  const Level& L0 = c->lv[0];
  exchange(c, 0, x);
  if (v && MODE >= CM_SCHUR) exchange(c, 0, v);
  if (L0.tiled) {
    CTArgs t;
    t.x = x;
    t.v = v;
    t.b = b;
    t.y = y;
    t.coef = c->coef;
    t.ldc = c->B;
    t.n2 = c->B;
    t.s1 = s1;
    if (L0.tlc.ichunk == 8) tiled_c<DIM, MODE, 8>(c, t, rd);
    else if (L0.tlc.ichunk == 4) tiled_c<DIM, MODE, 4>(c, t, rd);
    else tiled_c<DIM, MODE, 2>(c, t, rd);
    return;
  }
  launch(c, k_capply<DIM, MODE>, own(c->fine), BS, 0, c->fine, dev_op<DIM>(c->M), dev_op<DIM>(c->K),
                                                        dev_op<DIM>(c->A), a, rd);
  note(c);
}

// apply_schur_tilde_inv (precond.hpp:199-205)
template <int DIM>
static void schur_tilde_inv(okg_ctx* c, const double* b, double* x) {
  shat_inv<DIM>(c, b, c->sy, c->p.mg_cycles);
  apply_level<DIM>(c, 0, c->M, c->sy, c->st);
  shat_inv<DIM>(c, c->st, x, c->p.mg_cycles);
}

// apply_schur (precond.hpp:210-222); resid: y = b - S v
template <int DIM>
static void apply_schur(okg_ctx* c, const double* v, const double* b, double* y) {
  apply_level<DIM>(c, 0, c->K, v, c->kv);
  cheb<DIM>(c, c->M, c->kv, c->zz);
  if (b) capply<DIM, CM_SCHUR_RES>(c, c->zz, v, b, y, c->c);
  else capply<DIM, CM_SCHUR>(c, c->zz, v, nullptr, y, c->c);
}

// apply_S_inv_approx (precond.hpp:227-241) = richardson (krylov.hpp:225-242)
template <int DIM>
static void s_inv_approx(okg_ctx* c, const double* b, double* x) {
  const int k = c->p.richardson_steps;
  schur_tilde_inv<DIM>(c, b, x);
  for (int j = 1; j < k; ++j) {
    apply_schur<DIM>(c, x, b, c->rr);
    schur_tilde_inv<DIM>(c, c->rr, c->z2);
    axpy(c, 1.0, c->z2 + c->fine.lo, x + c->fine.lo, c->fine.hi - c->fine.lo);
  }
}

// apply_block (precond.hpp:257-271)
template <int DIM>
static void apply_block(okg_ctx* c, const double* p, double* z) {
  cheb<DIM>(c, c->A, p, z);
  capply<DIM, CM_SUB>(c, z, nullptr, p + c->B, c->r2p, 0.0);
  s_inv_approx<DIM>(c, c->r2p, z + c->B);
}

template <int DIM>
static void jacobian(okg_ctx* c, const double* x, double* y) {
  capply<DIM, CM_JAC>(c, x, x + c->B, nullptr, y, c->dt_theta);
}

static void check_lin(okg_ctx* c, const char* what) {
  if (!c->have_lin) THROW(OKG_EINCONSISTENT, "%s: linearized double-well block is not set", what);
}

// ---- graphs ------------------------------------------------------------------------
template <int DIM>
static void capture_graphs(okg_ctx* c) {
  cudaGraph_t g;
  c->capturing = true;
  c->cap_count = 0;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    apply_block<DIM>(c, c->pin, c->pz);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    throw;
  }
  CK(cudaStreamEndCapture(c->stream, &g));
  c->prec_nodes = c->cap_count;
  CK(cudaGraphInstantiate(&c->g_prec, g, 0));
  CK(cudaGraphDestroy(g));
  c->cap_count = 0;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    apply_block<DIM>(c, c->pin, c->pz);
    jacobian<DIM>(c, c->pz, c->pw);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    throw;
  }
  CK(cudaStreamEndCapture(c->stream, &g));
  c->arn_nodes = c->cap_count;
  CK(cudaGraphInstantiate(&c->g_arn, g, 0));
  CK(cudaGraphDestroy(g));
  c->capturing = false;
}

// z = P^{-1} pin  (and w = J z when `with_jac`)
template <int DIM>
static void run_arnoldi_op(okg_ctx* c, bool with_jac) {
  if (c->p.use_graphs) {
    CK(cudaGraphLaunch(with_jac ? c->g_arn : c->g_prec, c->stream));
    g_launches += with_jac ? c->arn_nodes : c->prec_nodes;
  } else {
    apply_block<DIM>(c, c->pin, c->pz);
    if (with_jac) jacobian<DIM>(c, c->pz, c->pw);
  }
}

// ---- residual (model.hpp:121-148) ---------------------------------------------------
template <int DIM>
static double residual(okg_ctx* c, const double* un, const double* wn, const double* uo, const double* wo,
                       double* o1, double* o2, double sign, double* s1out = nullptr) {
  ResArgs a;
  a.un = un;
  a.wn = wn;
  a.uo = uo;
  a.wo = wo;
  a.out1 = o1;
  a.out2 = o2;
  a.sign = sign;
  a.dt_theta = c->p.dt * c->p.theta;
  a.dt_1mtheta = c->p.dt * (1.0 - c->p.theta);
  a.sigma = c->p.sigma;
  a.m = c->p.m;
  a.eps2 = c->p.eps * c->p.eps;
  a.b_int = c->b_int;
  a.b_tab = c->b_tab;
  for (const double* v : {un, wn, uo, wo}) exchange(c, 0, v);
  launch(c, k_residual<DIM>, own(c->fine), BS, 0, c->fine, dev_op<DIM>(c->M), dev_op<DIM>(c->K), c->nl, a,
                                                   red(c, R_RES));
  note(c);
  reduce_to_host(c, R_RES, 2);
  const double na = std::sqrt(c->hred[R_RES]), nb = std::sqrt(c->hred[R_RES + 1]);
  if (s1out) *s1out = c->hred[R_RES] + c->hred[R_RES + 1];
  return std::sqrt(na * na + nb * nb);  // stacked_norm, model.hpp:152-155
}

template <int DIM>
static void linearize(okg_ctx* c, const double* u) {
  exchange(c, 0, u);
  launch(c, k_linearize<DIM>, own(c->fine), BS, 0, c->fine, dev_op<DIM>(c->K), c->nl, c->p.eps * c->p.eps, u,
                                                    c->coef, c->B);
  note(c);
  // the negative stencil slots of C are read at the neighbour (positive arrays q >= 1)
  for (int q = 1; q <= Traits<DIM>::NPOS; ++q) exchange(c, 0, c->coef + (ptrdiff_t)q * c->B);
  c->have_lin = true;
}

// ---- GMRES (krylov.hpp:44-152) ----------------------------------------------------------
static void givens(double cs, double sn, double& a, double& b) {
  const double t = cs * a + sn * b;
  b = -sn * a + cs * b;
  a = t;
}

// CGS2: h = V^T w (+ ||w||^2), w' = w - V h, c = V^T w', w'' = w' - V c, ||w''||^2.
// With several slabs every partial reduction is allreduced before a kernel
// consumes it (the single-slab path reads the sums straight from device memory).
template <int NVB>
static void arnoldi_ortho(okg_ctx* c, int nv) {
  const size_t n2 = c->N2, ne = 2 * c->seg.len;
  double* pw = F(c, c->pw);
  double* gt = F(c, c->gt);
  launch(c, k_arnoldi_dot<NVB>, vblk(ne), BS, 0, nv, (const double*)pw, (const double*)c->V, n2, c->seg, ne,
         red(c, R_H));
  note(c);
  reduce_on_device(c, R_H, NVB + 1);
  launch(c, k_arnoldi_update<NVB, 0>, vblk(ne), BS, 0, nv, (const double*)pw, (const double*)c->V, n2, c->seg, ne,
         (const double*)(c->dred + R_H), gt, red(c, R_C));
  note(c);
  reduce_on_device(c, R_C, NVB);
  launch(c, k_arnoldi_update<NVB, 1>, vblk(ne), BS, 0, nv, (const double*)gt, (const double*)c->V, n2, c->seg, ne,
         (const double*)(c->dred + R_C), pw, red(c, R_NRM));
  note(c);
  reduce_on_device(c, R_NRM, 1);
}

// generic (nv > 32): chunked classical Gram-Schmidt twice
static void arnoldi_ortho_chunked(okg_ctx* c, int nv, std::vector<double>& hsum, double& ww) {
  const size_t n2 = c->N2, ne = 2 * c->seg.len;
  double* pw = F(c, c->pw);
  double* gt = F(c, c->gt);
  hsum.assign(nv, 0.0);
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<double> hh(nv, 0.0);
    for (int q0 = 0; q0 < nv; q0 += 32) {
      const int cnt = std::min(32, nv - q0);
      launch(c, k_arnoldi_dot<32>, vblk(ne), BS, 0, cnt, (const double*)pw, (const double*)(c->V + (size_t)q0 * n2),
             n2, c->seg, ne, red(c, R_H));
      note(c);
      reduce_to_host(c, R_H, 33);
      for (int q = 0; q < cnt; ++q) hh[q0 + q] = c->hred[R_H + q];
      if (pass == 0 && q0 == 0) ww = c->hred[R_H + 32];
    }
    for (int q0 = 0; q0 < nv; q0 += 32) {
      const int cnt = std::min(32, nv - q0);
      CK(cudaMemcpyAsync(c->dred + R_C, hh.data() + q0, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      launch(c, k_arnoldi_update<32, 1>, vblk(ne), BS, 0, cnt, (const double*)pw,
             (const double*)(c->V + (size_t)q0 * n2), n2, c->seg, ne, (const double*)(c->dred + R_C), gt,
             red(c, R_NRM));
      note(c);
      copy(c, gt, pw, n2);
      CK(cudaStreamSynchronize(c->stream));
    }
    for (int q = 0; q < nv; ++q) hsum[q] += hh[q];
  }
  reduce_to_host(c, R_NRM, 1);
  write_red(c, R_NRM, 1);
}

template <int DIM>
static int gmres(okg_ctx* c, const double* b, double* x, double rel_tol, int max_iter, int restart,
                 okg_krylov_stats* st, double norm_b_sq = -1.0) {
  const size_t n2 = c->N2;
  okg_krylov_stats local;
  if (!st) st = &local;
  std::memset(st, 0, sizeof *st);
  auto push = [&](double v) {
    if (st->n_residual_norms < 512) st->residual_norms[st->n_residual_norms] = v;
    st->n_residual_norms++;
  };
  const size_t ne = 2 * c->seg.len;
  CK(cudaMemsetAsync(F(c, x), 0, n2 * sizeof(double), c->stream));
  double nb2 = norm_b_sq;
  if (nb2 < 0.0) {
    launch(c, k_dot, vblk(ne), BS, 0, (const double*)F(c, b), (const double*)F(c, b), c->seg, ne, red(c, R_DOT));
    note(c);
    reduce_to_host(c, R_DOT, 1);
    nb2 = c->hred[R_DOT];
  }
  // require_finite(b) (krylov.hpp:52): any NaN/Inf entry makes the sum of squares non-finite
  if (!std::isfinite(nb2)) THROW(OKG_EINVAL, "gmres rhs: vector contains NaN/Inf");
  const double norm_b = std::sqrt(nb2);
  push(norm_b);
  if (norm_b == 0.0) {
    st->converged = 1;
    return OKG_OK;
  }
  const double target = rel_tol * norm_b;
  const int cycle_len = restart > 0 ? std::min(restart, max_iter) : max_iter;
  if (cycle_len + 1 > c->vcap) THROW(OKG_EINVAL, "gmres: basis capacity %d < %d", c->vcap, cycle_len + 1);
  const double* r = b;  // residual of the current iterate (x = 0)
  double beta = norm_b;
  std::vector<std::vector<double>> H;
  std::vector<double> cs, sn, g, hsum;
  while (st->iterations < max_iter) {
    // V0 = r / beta
    launch(c, k_scale, vblk(n2), BS, 0, 1.0 / beta, (const double*)F(c, r), c->V, n2);
    note(c);
    copy(c, c->V, F(c, c->pin), n2);
    H.clear();
    cs.clear();
    sn.clear();
    g.assign(1, beta);
    int j = 0;
    bool breakdown = false;
    while (j < cycle_len && st->iterations < max_iter) {
      run_arnoldi_op<DIM>(c, true);  // pz = P^-1 V_j ; pw = J pz
      const int nv = j + 1;
      std::vector<double> h(j + 2, 0.0);
      double ww, arnoldi_norm;
      if (nv <= 32) {
        if (nv <= 4) arnoldi_ortho<4>(c, nv);
        else if (nv <= 8) arnoldi_ortho<8>(c, nv);
        else if (nv <= 16) arnoldi_ortho<16>(c, nv);
        else arnoldi_ortho<32>(c, nv);
        // V_{j+1} = w / ||w||  (speculative; unused on exit)
        launch(c, k_normalize, vblk(n2), BS, 0, (const double*)F(c, c->pw), (const double*)(c->dred + R_NRM),
               c->V + (size_t)(j + 1) * n2, F(c, c->pin), n2);
        note(c);
        const int nvb = nv <= 4 ? 4 : nv <= 8 ? 8 : nv <= 16 ? 16 : 32;
        // dred[R_H + nvb] holds ||w||^2 (slot NVB of the first reduction)
        CK(cudaMemcpyAsync(c->hred, c->dred, (R_NRM + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        ww = c->hred[R_H + nvb];
        for (int q = 0; q < nv; ++q) h[q] = c->hred[R_H + q] + c->hred[R_C + q];
        arnoldi_norm = std::sqrt(c->hred[R_NRM]);
      } else {
        arnoldi_ortho_chunked(c, nv, hsum, ww);
        for (int q = 0; q < nv; ++q) h[q] = hsum[q];
        arnoldi_norm = std::sqrt(c->hred[R_NRM]);
        launch(c, k_normalize, vblk(n2), BS, 0, (const double*)F(c, c->pw), (const double*)(c->dred + R_NRM),
               c->V + (size_t)(j + 1) * n2, F(c, c->pin), n2);
        note(c);
      }
      const double w_scale = std::sqrt(ww);
      h[j + 1] = arnoldi_norm;
      for (int i = 0; i < j; ++i) givens(cs[i], sn[i], h[i], h[i + 1]);
      const double denom = std::hypot(h[j], h[j + 1]);
      if (denom == 0.0) {
        breakdown = true;
        break;
      }
      const double cg = h[j] / denom, sg = h[j + 1] / denom;
      h[j] = denom;
      cs.push_back(cg);
      sn.push_back(sg);
      g.push_back(0.0);
      givens(cg, sg, g[j], g[j + 1]);
      H.push_back(std::move(h));
      ++st->iterations;
      ++j;
      const double est = std::abs(g[j]);
      push(est);
      if (est <= target) break;
      if (arnoldi_norm <= 1e-13 * w_scale) {
        breakdown = true;
        break;
      }
    }
    // H y = g, u = sum y_i V_i, x += P^-1 u   (krylov.hpp:124-133)
    std::vector<double> y(j, 0.0);
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < j; ++k) s -= H[k][i] * y[k];
      y[i] = H[i][i] != 0.0 ? s / H[i][i] : 0.0;
    }
    for (int q0 = 0; q0 < std::max(j, 1); q0 += 32) {
      Coeffs32 yc;
      const int cnt = std::min(32, j - q0);
      for (int q = 0; q < 32; ++q) yc.c[q] = q < cnt ? y[q0 + q] : 0.0;
      if (q0 == 0) {
        launch(c, k_combine, vblk(n2), BS, 0, std::max(cnt, 0), yc, (const double*)c->V, n2, n2, F(c, c->pin));
        note(c);
      } else {
        launch(c, k_combine, vblk(n2), BS, 0, cnt, yc, (const double*)(c->V + (size_t)q0 * n2), n2, n2, F(c, c->gt));
        note(c);
        axpy(c, 1.0, F(c, c->gt), F(c, c->pin), n2);
      }
    }
    run_arnoldi_op<DIM>(c, false);  // pz = P^-1 u
    axpy(c, 1.0, F(c, c->pz), F(c, x), n2);
    // r = b - J x, beta = ||r||   (krylov.hpp:135-138)
    capply<DIM, CM_JAC_RES>(c, x, x + c->B, b, c->gr, c->dt_theta, red(c, R_JRES));
    reduce_to_host(c, R_JRES, 1);
    beta = std::sqrt(c->hred[R_JRES]);
    st->final_residual = beta;
    r = c->gr;
    if (beta <= target * (1.0 + 1e-9)) {
      st->converged = 1;
      return OKG_OK;
    }
    if (breakdown) {
      st->stagnated = 1;
      return OKG_OK;
    }
    if (restart <= 0) return OKG_OK;
  }
  return OKG_OK;
}

// ---- Lanczos bounds (krylov.hpp:248-320) ------------------------------------------------
// Same start vector as the reference (std::mt19937(1234), uniform(-1,1) over
// the GLOBAL vertex order; each slab keeps its slice); dots allreduced.
// lanczos_extremes (krylov.hpp:248-289) of `apply_B` (y = B x on level-0 vectors),
// widened x0.9 / x1.1 as the estimate_*_spectrum callers do; `what` names the caller
template <int DIM, class ApplyB>
static void lanczos_bounds(okg_ctx* c, ApplyB&& apply_B, const char* what, double& lo, double& hi) {
  const Level& L0 = c->lv[0];
  const uint64_t Nglob = L0.g.N;
  const size_t nloc = L0.g.hi - L0.g.lo, B = L0.B;
  const int steps = (int)std::min<uint64_t>(30u, Nglob);
  std::mt19937 rng(1234u);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (uint64_t g = 0; g < L0.g.lo; ++g) (void)dist(rng);
  std::vector<double> hv(nloc);
  for (auto& e : hv) e = dist(rng);
  // scratch: steps+1 level-0 blocks, in the Krylov basis when it is large enough
  const size_t need = (size_t)steps + 1;
  double* flat = c->V;
  double* tmp = nullptr;
  if ((size_t)2 * c->vcap < need) {
    CK(cudaMalloc(&tmp, need * B * sizeof(double)));
    CK(cudaMemsetAsync(tmp, 0, need * B * sizeof(double), c->stream));
    flat = tmp;
  }
  const size_t reg0 = c->reg.size();
  auto blk = [&](size_t q) {
    double* g = flat + q * B - c->foff;
    c->reg.push_back({g, 0});
    return g;
  };
  const Seg s1{(size_t)L0.gh * L0.g.ps, nloc, B};
  auto dot = [&](const double* x, const double* y) {
    launch(c, k_dot, vblk(nloc), BS, 0, (const double*)F(c, x), (const double*)F(c, y), s1, nloc, red(c, R_DOT));
    note(c);
    reduce_to_host(c, R_DOT, 1);
    return c->hred[R_DOT];
  };
  std::vector<double*> Vv;
  double* v0 = blk(0);
  CK(cudaMemcpyAsync(v0 + L0.g.lo, hv.data(), nloc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const double nv0 = std::sqrt(dot(v0, v0));
  scale(c, 1.0 / nv0, F(c, v0), F(c, v0), B);
  Vv.push_back(v0);
  double* w = blk(need - 1);
  std::vector<double> alpha, beta;
  for (int j = 0; j < steps; ++j) {
    apply_B(Vv[j], w);
    const double a = dot(w, Vv[j]);
    alpha.push_back(a);
    axpy(c, -a, F(c, Vv[j]), F(c, w), B);
    if (j > 0) axpy(c, -beta[j - 1], F(c, Vv[j - 1]), F(c, w), B);
    for (double* q : Vv) axpy(c, -dot(w, q), F(c, q), F(c, w), B);
    const double nb = std::sqrt(dot(w, w));
    if (nb <= 1e-13 * std::abs(a) + 1e-300) break;
    if (j + 1 < steps) {
      beta.push_back(nb);
      double* nvp = blk(j + 1);
      scale(c, 1.0 / nb, F(c, w), F(c, nvp), B);
      Vv.push_back(nvp);
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  c->reg.resize(reg0);
  if (tmp) cudaFree(tmp);
  else CK(cudaMemsetAsync(c->V, 0, need * B * sizeof(double), c->stream));
  const int m = static_cast<int>(alpha.size());
  std::vector<double> T(static_cast<size_t>(m) * m, 0.0), ev;
  for (int i = 0; i < m; ++i) {
    T[i * m + i] = alpha[i];
    if (i + 1 < m) {
      T[i * m + i + 1] = beta[i];
      T[(i + 1) * m + i] = beta[i];
    }
  }
  if (!symmetric_eigenvalues(T, m, ev)) THROW(OKG_ENUMERICAL, "symmetric eigensolver failed to converge");
  if (ev.front() < 0.0) THROW(OKG_ENUMERICAL, "%s: negative Ritz value, matrix not positive definite", what);
  lo = 0.9 * ev.front();
  hi = 1.1 * ev.back();
}

// estimate_jacobi_spectrum(M) (krylov.hpp:296-320): B = D^-1/2 M D^-1/2
template <int DIM>
static void jacobi_spectrum(okg_ctx* c, double& lo, double& hi) {
  lanczos_bounds<DIM>(
      c,
      [&](double* x, double* y) {
        exchange(c, 0, x);
        op_apply<DIM>(c, c->fine, c->M, EPI_SCALE_APPLY, x, nullptr, y, nullptr);
      },
      "estimate_jacobi_spectrum", lo, hi);
}

// ---- SSOR (cheby_precond = "ssor", okg_ssor.cuh) ---------------------------------
// one sweep over the hyperplanes as one thread-block cluster
template <int DIM, bool FWD>
static void ssor_sweep(okg_ctx* c, const HostOp& A, const double* r, double* x) {
  launch_cluster(c, k_ssor_sweep<DIM, FWD>, (unsigned)c->ssor_cluster, SSOR_NT, 0, c->fine, dev_op<DIM>(A), 1.0, r, x);
  note(c);
}

// z = P_ssor^{-1} r = backward((2-w)/w D forward(r)), w = 1 (krylov.hpp:372-378); t scratch
template <int DIM>
static void ssor_apply(okg_ctx* c, const HostOp& A, const double* r, double* z, double* t) {
  ssor_sweep<DIM, true>(c, A, r, t);
  launch(c, k_diag_scale<DIM, false>, own(c->fine), 256, 0, c->fine, dev_op<DIM>(A), (2.0 - 1.0) / 1.0,
         (const double*)t, t);
  note(c);
  ssor_sweep<DIM, false>(c, A, t, z);
}

// estimate_ssor_spectrum(M) (krylov.hpp:390-418): B = E M E^T, E = g D^1/2 (D/w + L)^-1
template <int DIM>
static void ssor_spectrum(okg_ctx* c, double& lo, double& hi) {
  const double g = std::sqrt((2.0 - 1.0) / 1.0);
  const Op<DIM> m = dev_op<DIM>(c->M);
  lanczos_bounds<DIM>(
      c,
      [&](double* x, double* y) {
        launch(c, k_diag_scale<DIM, true>, own(c->fine), 256, 0, c->fine, m, g, (const double*)x, c->cr2);
        note(c);
        ssor_sweep<DIM, false>(c, c->M, c->cr2, c->cd0);
        apply_level<DIM>(c, 0, c->M, c->cd0, c->cd1);
        ssor_sweep<DIM, true>(c, c->M, c->cd1, y);
        launch(c, k_diag_scale<DIM, true>, own(c->fine), 256, 0, c->fine, m, g, (const double*)y, y);
        note(c);
      },
      "estimate_ssor_spectrum", lo, hi);
}

// chebyshev_semi_iteration with the SSOR preconditioner (krylov.hpp:158-202 via
// cheby_mass_solve, precond.hpp:99-119)
template <int DIM>
static void cheb_ssor(okg_ctx* c, const HostOp& A, const double* b, double* x) {
  const size_t B = c->B;
  const int k = c->p.cheby_iters;
  const double lmin = c->lambda_lo, lmax = c->lambda_hi;
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
  double *r = c->cr, *z = c->cd1, *d = c->cd0, *t = c->cr2, *Ad = c->cad;
  CK(cudaMemsetAsync(F(c, x), 0, B * sizeof(double), c->stream));
  copy(c, F(c, b), F(c, r), B);
  ssor_apply<DIM>(c, A, r, z, t);
  scale(c, 1.0 / theta, F(c, z), F(c, d), B);
  for (int j = 0; j < k; ++j) {
    axpy(c, 1.0, F(c, d), F(c, x), B);
    if (delta > 1e-300 && j + 1 == k) break;  // last correction applied
    apply_level<DIM>(c, 0, A, d, Ad);
    axpy(c, -1.0, F(c, Ad), F(c, r), B);
    ssor_apply<DIM>(c, A, r, z, t);
    if (delta <= 1e-300) {  // point spectrum: plain Richardson steps
      scale(c, 1.0 / theta, F(c, z), F(c, d), B);
    } else {
      launch(c, k_lincomb, vblk(B), 256, 0, c->cheb_c1[j], F(c, d), c->cheb_c2[j], (const double*)F(c, z), B);
      note(c);
    }
  }
}

// ---- diagnostics and initial state (okg_diag.cuh) -------------------------
// dot of two level-0 vectors over the owned vertices, allreduced over the slabs
static double dotv(okg_ctx* c, const double* a, const double* b) {
  const size_t ne = c->seg.len;
  const Seg s1{c->seg.off, ne, c->B};
  launch(c, k_dot, vblk(ne), BS, 0, (const double*)F(c, a), (const double*)F(c, b), s1, ne, red(c, R_DOT));
  note(c);
  reduce_to_host(c, R_DOT, 1);
  return c->hred[R_DOT];
}

// conjugate_gradient (krylov.hpp:424-479) with the Jacobi preconditioner of A
// (operator.hpp:53-64) and an optional unit nullspace vector ns; b, x, ns are
// level-0 vectors; returns the iteration count
template <int DIM>
static int cg(okg_ctx* c, const HostOp& A, const double* b, double* x, double rel_tol, int max_iter,
              const double* ns, bool& converged) {
  const size_t B = c->B;
  double *r = c->cd0, *z = c->cd1, *p = c->cr, *Ap = c->st;
  auto project = [&](double* v) {
    if (ns) axpy(c, -dotv(c, v, ns), F(c, ns), F(c, v), B);
  };
  converged = false;
  CK(cudaMemsetAsync(F(c, x), 0, B * sizeof(double), c->stream));
  copy(c, F(c, b), F(c, r), B);
  {  // require_finite(b, "cg rhs") (krylov.hpp:429): a non-finite entry makes ||b|| non-finite
    const double bb = dotv(c, b, b);
    if (!std::isfinite(bb)) THROW(OKG_EINVAL, "cg rhs: vector contains NaN/Inf");
  }
  project(r);
  const double norm_b = std::sqrt(dotv(c, r, r));
  if (norm_b == 0.0) {
    converged = true;
    return 0;
  }
  const double target = rel_tol * norm_b;
  const Op<DIM> op = dev_op<DIM>(A);
  launch(c, k_divdiag<DIM>, own(c->fine), BS, 0, c->fine, op, (const double*)r, z);
  note(c);
  project(z);
  copy(c, F(c, z), F(c, p), B);
  double rz = dotv(c, r, z);
  int it = 0;
  for (; it < max_iter;) {
    apply_level<DIM>(c, 0, A, p, Ap);
    const double pAp = dotv(c, p, Ap);
    if (pAp <= 0.0) THROW(OKG_ENUMERICAL, "cg: operator not positive definite on iterate");
    const double alpha = rz / pAp;
    axpy(c, alpha, F(c, p), F(c, x), B);
    axpy(c, -alpha, F(c, Ap), F(c, r), B);
    project(r);
    ++it;
    const double rn = std::sqrt(dotv(c, r, r));
    if (rn <= target) {
      converged = true;
      break;
    }
    launch(c, k_divdiag<DIM>, own(c->fine), BS, 0, c->fine, op, (const double*)r, z);
    note(c);
    project(z);
    const double rz_new = dotv(c, r, z);
    const double beta = rz_new / rz;
    rz = rz_new;
    launch(c, k_xpby, vblk(B), BS, 0, (const double*)F(c, z), beta, F(c, p), B);
    note(c);
  }
  return it;
}

// total_mass = b^T u (model.hpp:46-48)
template <int DIM>
static double total_mass_impl(okg_ctx* c, const double* u) {
  launch(c, k_mass<DIM>, vblk(c->fine.hi - c->fine.lo), BS, 0, c->fine, (const double*)c->b_tab, u, red(c, R_DOT));
  note(c);
  reduce_to_host(c, R_DOT, 1);
  return c->hred[R_DOT];
}

// integrate_double_well (assembly.hpp:220-245)
template <int DIM>
static double double_well_impl(okg_ctx* c, const double* u) {
  exchange(c, 0, u);
  const Grid& g = c->fine;
  const size_t cells = (size_t)std::max(0, std::min(g.ihi, g.n) - g.ilo) * (DIM == 3 ? (size_t)g.n * g.n : g.n);
  const double vol = DIM == 2 ? c->h * c->h / 2.0 : c->h * c->h * c->h / 6.0;
  launch(c, k_double_well<DIM>, vblk(cells), BS, 0, g, vol, u, red(c, R_DOT));
  note(c);
  reduce_to_host(c, R_DOT, 1);
  return c->hred[R_DOT];
}

// energy (model.hpp:56-86)
template <int DIM>
static double energy_impl(okg_ctx* c, const double* u, int* cg_iters) {
  const okg_params& p = c->p;
  const size_t B = c->B;
  apply_level<DIM>(c, 0, c->K, u, c->kv);
  const double grad_term = 0.5 * p.eps * p.eps * dotv(c, u, c->kv);
  const double well_term = 0.25 * double_well_impl<DIM>(c, u);
  double nonlocal = 0.0;
  if (cg_iters) *cg_iters = 0;
  if (p.sigma != 0.0) {
    double* rhs = c->r2p;
    apply_level<DIM>(c, 0, c->M, u, rhs);
    launch(c, k_add_load<DIM>, own(c->fine), BS, 0, c->fine, (const double*)c->b_tab, -p.m, (const double*)rhs, rhs);
    note(c);
    // mean of the rhs (compatibility of the pure-Neumann solve)
    launch(c, k_fill, vblk(B), BS, 0, 1.0, F(c, c->zz), B);
    note(c);
    const double mean = dotv(c, rhs, c->zz);
    if (std::abs(mean) > 1e-6)
      THROW(OKG_EINCONSISTENT, "energy: potential right-hand side is not mean-zero (|sum| = %f)", std::abs(mean));
    const double q = 1.0 / std::sqrt((double)c->fine.N);
    launch(c, k_fill, vblk(B), BS, 0, q, F(c, c->zz), B);
    note(c);
    bool conv = false;
    const int its = cg<DIM>(c, c->K, rhs, c->sy, 1e-10, 2000, c->zz, conv);
    if (cg_iters) *cg_iters = its;
    if (!conv) THROW(OKG_ENUMERICAL, "energy: potential solve did not converge");
    nonlocal = 0.5 * p.sigma * dotv(c, c->sy, rhs);
  }
  return grad_term + well_term + nonlocal;
}

// initial_state (model.hpp:93-114): the context's state becomes (u0, w0) at t = 0
template <int DIM>
static void initial_state_impl(okg_ctx* c, int* cg_iters) {
  const okg_params& p = c->p;
  const size_t B = c->B;
  launch(c, k_cos_ic<DIM>, own(c->fine), BS, 0, c->fine, c->h, p.m, c->u_old);
  note(c);
  double* rhs = c->kv;
  apply_level<DIM>(c, 0, c->K, c->u_old, rhs);
  scale(c, p.eps * p.eps, F(c, rhs), F(c, rhs), B);
  launch(c, k_nonlinear<DIM>, own(c->fine), BS, 0, c->fine, c->nl, (const double*)c->u_old, c->rr);
  note(c);
  axpy(c, 1.0, F(c, c->rr), F(c, rhs), B);
  bool conv = false;
  const int its = cg<DIM>(c, c->M, rhs, c->w_old, 1e-12, 1000, nullptr, conv);
  if (cg_iters) *cg_iters = its;
  if (!conv) THROW(OKG_ENUMERICAL, "initial_state: mass solve did not converge");
  CK(cudaStreamSynchronize(c->stream));
  c->t = 0.0;
  c->step = 0;
}

// ---- setup (make_schur_context, precond.hpp:126-181) ---------------------------------------
template <int DIM>
static void build(okg_ctx* c) {
  const okg_params& p = c->p;
  const UnitTables ut = build_unit_tables(DIM);
  const int n = p.n;
  c->h = 1.0 / n;
  const double hd = ipow(c->h, DIM), hk = ipow(c->h, DIM - 2);
  c->fine = make_grid(DIM, n);
  c->N = c->fine.N;
  c->M = make_op(c, ut, ut.M, hd, nullptr, 0.0, false);
  c->K = make_op(c, ut, ut.K, hk, nullptr, 0.0, false);
  {
    // a_mat = scale(M, a_coeff): (M_ij) * a   (precond.hpp:154, sparse.hpp:198-202)
    std::vector<double> Mh(ut.M.size());
    for (size_t i = 0; i < Mh.size(); ++i) Mh[i] = ut.M[i] * hd;
    c->A = make_op(c, ut, Mh, c->a_coeff, nullptr, 0.0, false);
  }
  // load vector per class
  {
    std::vector<double> bt(ut.ncls);
    for (int cl = 0; cl < ut.ncls; ++cl) bt[cl] = ut.load[cl] * hd;
    c->b_int = bt[ut.ncls / 2];
    c->b_tab = dalloc(c, bt.size());
    CK(cudaMemcpyAsync(c->b_tab, bt.data(), bt.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  // closed-form nonlinear constants
  const double fact = DIM == 2 ? 2.0 : 6.0;
  c->nl.vol = hd / fact;
  c->nl.kS = DIM == 2 ? (2.0 * 2.0 / 720.0) : (6.0 * 2.0 / 5040.0);
  c->nl.kM = DIM == 2 ? (2.0 / 24.0) : (6.0 / 120.0);
  c->nl.kT = DIM == 2 ? (2.0 * 6.0 / 720.0) : (6.0 * 6.0 / 5040.0);
  // multigrid levels (build_hierarchy, multigrid.hpp:55-86)
  {
    int ln = n;
    for (;;) {
      Level L;
      L.g = make_grid(DIM, ln);
      const double hl = 1.0 / ln;
      const double hld = ipow(hl, DIM), hlk = ipow(hl, DIM - 2);
      std::vector<double> Ml(ut.M.size()), Kl(ut.K.size());
      for (size_t i = 0; i < Ml.size(); ++i) {
        Ml[i] = ut.M[i] * hld;
        Kl[i] = ut.K[i] * hlk;
      }
      L.shat = make_op(c, ut, Ml, 1.0, &Kl, c->eps_sqrt_c, true);
      c->lv.push_back(L);
      if (!((int64_t)L.g.N > p.min_coarse_size && ln % 2 == 0)) break;
      ln /= 2;
    }
    const int64_t coarsest = c->lv.back().g.N;
    if (coarsest > std::max<int64_t>(p.min_coarse_size, 2000))
      THROW(OKG_ECONFIG,
            "build_hierarchy: coarsest level too large for a direct solve; choose a grid with more factors of two");
    // slab partition, see slab_partition()
    const int S = c->nslabs;
    c->L_rep = (int)c->lv.size();
    if (S > 1) {
      std::vector<int> lo(c->lv.size()), hi(c->lv.size());
      c->L_rep = slab_partition(DIM, c->lv[0].g.s, (int)c->lv.size(), S, c->rank, rep_max_of(p), lo.data(), hi.data());
      if (c->L_rep == 0) THROW(OKG_EINVAL, "slab decomposition: %d slabs leave fewer than 2 planes each", S);
      for (int l = 0; l < c->L_rep; ++l) {
        set_owned(c->lv[l].g, lo[l], hi[l]);
        c->lv[l].gh = 1;
      }
      for (size_t l = c->L_rep; l < c->lv.size(); ++l) c->lv[l].rep = true;
      // every slab's restriction range in the first replicated level (allgather_planes)
      c->rep_lo.assign(S, 0);
      c->rep_hi.assign(S, 0);
      for (int r = 0; r < S; ++r) {
        std::vector<int> rl(c->lv.size()), rh(c->lv.size());
        slab_partition(DIM, c->lv[0].g.s, (int)c->lv.size(), S, r, rep_max_of(p), rl.data(), rh.data());
        c->rep_lo[r] = (rl[c->L_rep - 1] + 1) / 2;
        c->rep_hi[r] = (rh[c->L_rep - 1] + 1) / 2;
      }
    }
    for (size_t l = 0; l < c->lv.size(); ++l) {
      Level& L = c->lv[l];
      L.B = (size_t)(L.g.ihi - L.g.ilo + 2 * L.gh) * L.g.ps;
      if (l > 0) {
        L.b = lvec(c, L, (int)l);
        L.x = lvec(c, L, (int)l);
      }
      L.ea = lvec(c, L, (int)l);
      L.eb = lvec(c, L, (int)l);
      L.res = lvec(c, L, (int)l);
    }
    c->fine = c->lv[0].g;
    c->B = c->lv[0].B;
    c->foff = ((ptrdiff_t)c->fine.ilo - c->lv[0].gh) * c->fine.ps;
    c->seg = Seg{(size_t)c->lv[0].gh * c->fine.ps, (size_t)(c->fine.hi - c->fine.lo), c->B};
    c->N2 = 2 * c->B;
    // shared-memory tail for the small levels (okg_tail.cuh): from the first level
    // with n <= tail_max_n (and at most tail_max_vertices vertices when > 0) down to
    // the coarsest, in one launch; V(2,2) only, not on levels split across slabs
    // default depth: the 9^3 (3D) / 33^2 (2D) level -- measured: one SM beats the
    // multi-CTA level kernels only where a level is a few hundred to ~1000 vertices
    const int64_t tmax = p.tail_max_vertices == 0 ? (DIM == 3 ? 1000 : 1100) : p.tail_max_vertices;
    if (p.tail_max_vertices >= 0 && p.mg_pre == 2 && p.mg_post == 2) {
      const int ncv = (int)c->lv.back().g.N;
      for (size_t l = 1; l + 1 < c->lv.size(); ++l) {
        const Level& L = c->lv[l];
        // (the kernel is instantiated for power-of-two first levels only)
        const bool pow2 = L.g.n >= 2 && (L.g.n & (L.g.n - 1)) == 0;
        if (!(pow2 && L.g.n <= tail_max_n<DIM>() && (int64_t)L.g.N <= tmax && c->lv.size() - l <= (size_t)TAIL_MAXL &&
              (S == 1 || (int)l >= c->L_rep)))
          continue;
        // cluster size: split the coarse inverse so each CTA stages <= 96 KB of it
        int C = 1;
        while (C < 16 && (size_t)((ncv + C - 1) / C) * ncv * sizeof(double) > 96 * 1024) C *= 2;
        C = std::min(std::max(C, p.tail_cluster > 0 ? p.tail_cluster : 1), 16);
        size_t need = 0;
        tail_dispatch<DIM>(L.g.n, [&](auto N0) { need = tail_smem<DIM, decltype(N0)::value>(ncv, C); });
        if (need > 220 * 1024) continue;  // shared-memory budget: try a deeper level
        c->tail_start = (int)l;
        c->tail_cluster = C;
        break;
      }
    }
    if (c->tail_start > 0) {
      // tables: every tail level's class rows, then the restriction weights
      const int NO = Traits<DIM>::NOFF, NCL = Traits<DIM>::NCLS;
      std::vector<double> tt((size_t)tail_table_doubles<DIM>(), 0.0);
      for (size_t q = 0; q + c->tail_start < c->lv.size(); ++q) {
        const std::vector<double>& h = c->lv[c->tail_start + q].shat.htab;
        std::copy(h.begin(), h.end(), tt.begin() + q * NCL * (NO + 1));
      }
      for (int cl = 0; cl < NCL; ++cl)
        for (int o = 0; o < NO; ++o) {
          bool ok = true;
          int cc = cl;
          for (int d = DIM - 1; d >= 0; --d) {
            const int cd = cc % 3, od = off_comp(DIM, o, d);
            cc /= 3;
            ok = ok && !(cd == 0 && od < 0) && !(cd == 2 && od > 0);
          }
          tt[(size_t)TAIL_MAXL * NCL * (NO + 1) + cl * NO + o] = ok ? (o == NO / 2 ? 1.0 : 0.5) : 0.0;
        }
      c->tail_tab = dalloc(c, tt.size());
      CK(cudaMemcpyAsync(c->tail_tab, tt.data(), tt.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      c->nc = (int)c->lv.back().g.N;
      tail_dispatch<DIM>(c->lv[c->tail_start].g.n, [&](auto N0) { tail_prepare<DIM, decltype(N0)::value>(c); });
    }
    // temporally blocked down/up kernels for V(2,2) (okg_vcycle.cuh)
    // default: the coarse levels with n <= 512 in 2D, n <= 16 in 3D; above that the
    // tiled single sweeps are faster (measured per step: 2D 2048^2 61.1 vs 62.4 ms with
    // the 1025^2 level tiled; 3D 128^3 49.1 vs 49.3 ms with the 33^3 level tiled --
    // the halo-3 redundancy of a box outweighs the saved launches on bigger levels)
    // (halo 3 / 2: only on levels that are not split across slabs)
    if (p.mg_pre == 2 && p.mg_post == 2 && p.mg_fuse >= 0)
      for (size_t l = (p.mg_fuse == 1 ? 0 : 1); l + 1 < c->lv.size(); ++l)
        if ((p.mg_fuse >= 1 || c->lv[l].g.n <= (DIM == 2 ? OKG_MG2_FUSE_N : OKG_MG3_FUSE_N)) && c->lv[l].gh == 0 &&
            (c->lv[l].rep || S == 1))
          c->lv[l].fused = true;
    // shared-memory tiled kernels for the large levels (okg_tiled.cuh)
    const int tmin = p.tiled_min_n == 0 ? (DIM == 3 ? 32 : 128) : p.tiled_min_n;
    if (tmin > 0)
      for (Level& L : c->lv)
        if (L.g.n >= std::max(tmin, 2)) make_tiling<DIM>(c, L);
    // coarsest: dense SPD inverse (replaces CholeskyFactor, multigrid.hpp:82-83)
    Level& Lc = c->lv.back();
    const int nc = (int)Lc.g.N;
    std::vector<double> Ad(static_cast<size_t>(nc) * nc, 0.0), Ai;
    const int NO = Traits<DIM>::NOFF;
    for (int i = 0; i < nc; ++i) {
      int gi[3] = {0, 0, 0};
      if (DIM == 2) {
        gi[0] = i / Lc.g.s;
        gi[1] = i % Lc.g.s;
      } else {
        gi[0] = i / (int)Lc.g.ps;
        gi[1] = (i / Lc.g.s) % Lc.g.s;
        gi[2] = i % Lc.g.s;
      }
      int cls = 0;
      for (int d = 0; d < DIM; ++d) cls = cls * 3 + (gi[d] == 0 ? 0 : (gi[d] == Lc.g.n ? 2 : 1));
      for (int o = 0; o < NO; ++o) {
        bool ok = true;
        for (int d = 0; d < DIM; ++d) {
          const int v = gi[d] + off_comp(DIM, o, d);
          ok = ok && v >= 0 && v <= Lc.g.n;
        }
        if (!ok) continue;
        const int j = i + Lc.g.off[o];
        Ad[static_cast<size_t>(i) * nc + j] = Lc.shat.htab[static_cast<size_t>(cls) * (NO + 1) + o];
      }
    }
    c->nc = nc;
    if (nc <= 2000) {
      if (!dense_spd_inverse(Ad, nc, Ai)) THROW(OKG_ENUMERICAL, "Cholesky: matrix not positive definite");
      c->Ainv = dalloc(c, Ai.size());
      CK(cudaMemcpyAsync(c->Ainv, Ai.data(), Ai.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    } else {
      // split the rows over the slabs when the coarsest is the first replicated level
      // (its planes are then gathered with the restriction's ranges, allgather_planes)
      int r0 = 0, r1 = nc;
      c->coarse_split = S > 1 && c->L_rep == (int)c->lv.size() - 1 && p.coarse_split >= 0;
      if (c->coarse_split) {
        r0 = c->rep_lo[c->rank] * (int)Lc.g.ps;
        r1 = c->rep_hi[c->rank] * (int)Lc.g.ps;
      }
      coarse_inverse_device(c, Ad, nc, r0, r1);
    }
  }
  // buffers
  const size_t N2 = c->N2;
  Level& L0 = c->lv[0];
  c->max_blocks = std::max<size_t>(nblk(c->N), 148 * 8) + 1;
  c->partials = dalloc(c, c->max_blocks * 40);
  {
    void* t = nullptr;
    CK(cudaMalloc(&t, 64));
    CK(cudaMemsetAsync(t, 0, 64, c->stream));
    c->allocs.push_back(t);
    c->ticket = static_cast<unsigned*>(t);
    c->dflag = reinterpret_cast<int*>(static_cast<char*>(t) + 32);
  }
  c->dred = dalloc(c, 256);
  CK(cudaMallocHost(&c->hred, 256 * sizeof(double)));
  c->coef = lvec(c, L0, 0, Traits<DIM>::NPOS + 1);
  const int cycle_len = p.gmres_restart > 0 ? std::min(p.gmres_restart, p.gmres_maxit) : p.gmres_maxit;
  c->vcap = cycle_len + 1;
  c->V = dalloc(c, (size_t)c->vcap * N2);
  for (double** b : {&c->gb, &c->gx, &c->gr, &c->pin, &c->pz, &c->pw, &c->gt}) *b = lvec(c, L0, 0, 2);
  for (double** b : {&c->cd0, &c->cd1, &c->cr, &c->cr2, &c->cad, &c->r2p, &c->sy, &c->st, &c->kv, &c->zz, &c->rr, &c->z2,
                     &c->shr, &c->u_old, &c->w_old, &c->u, &c->w})
    *b = lvec(c, L0, 0);
  // Chebyshev bounds and coefficients (precond.hpp:156-166)
  c->ssor = p.cheby_ssor != 0;
  {
    const int ncol = DIM == 3 ? c->fine.s * c->fine.s : c->fine.s;
    c->ssor_cluster = std::min(8, (ncol + SSOR_NT - 1) / SSOR_NT);
  }
  if (c->ssor) {
    if (c->nslabs > 1) THROW(OKG_ECONFIG, "config: cheby_precond = 'ssor' needs one slab (sequential sweeps)");
    ssor_spectrum<DIM>(c, c->lambda_lo, c->lambda_hi);
  } else {
    jacobi_spectrum<DIM>(c, c->lambda_lo, c->lambda_hi);
  }
  {
    const double lmin = c->lambda_lo, lmax = c->lambda_hi;
    if (lmin <= 0.0) THROW(OKG_EINVAL, "chebyshev: lambda_min must be positive");
    if (lmax < lmin) THROW(OKG_EINVAL, "chebyshev: bounds out of order");
    const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
    c->cheb_inv_theta = 1.0 / theta;
    if (const char* e = std::getenv("OKG_CHEB0")) c->cheb_fuse0 = std::atoi(e) != 0;
    c->cheb_c1.assign(std::max(p.cheby_iters, 1), 0.0);
    c->cheb_c2.assign(std::max(p.cheby_iters, 1), 1.0 / theta);
    if (delta > 1e-300) {
      const double sigma1 = theta / delta;
      double rho = 1.0 / sigma1;
      for (int j = 0; j + 1 < p.cheby_iters; ++j) {
        const double rho_next = 1.0 / (2.0 * sigma1 - rho);
        c->cheb_c1[j] = rho_next * rho;
        c->cheb_c2[j] = 2.0 * rho_next / delta;
        rho = rho_next;
      }
    }
  }
  // collapse the bottom of the V-cycle (okg_params.mg_collapse): the first coarse level
  // with at most cmax vertices and every level below it apply a fixed linear map --
  // symmetric for V(v,v) with damped Jacobi (the post-smoother is the pre-smoother's
  // adjoint) -- so it is formed once (columns = that level's cycle on unit vectors,
  // run through the existing kernels) and applied as one packed-symmetric matvec.
  // Only on levels every slab holds whole (no communication below them).
  if (p.mg_collapse >= 0 && p.mg_pre == p.mg_post && !c->coarse_big) {
    const int64_t cmax = p.mg_collapse > 0 ? p.mg_collapse : (DIM == 3 ? 1000 : 1100);
    int lc = -1;
    for (size_t l = 1; l + 1 < c->lv.size(); ++l)
      if ((int64_t)c->lv[l].g.N <= cmax) {
        lc = (int)l;
        break;
      }
    if (lc > 0 && (c->nslabs == 1 || lc >= c->L_rep)) collapse_levels<DIM>(c, lc);
  }
  if (p.use_graphs) capture_graphs<DIM>(c);
  CK(cudaStreamSynchronize(c->stream));
}

}  // namespace okg

// =====================================================================================
// C ABI
// =====================================================================================
#define DISPATCH(c, fn, ...) ((c)->dim == 2 ? fn<2>(__VA_ARGS__) : fn<3>(__VA_ARGS__))

template <class F>
static int guard(okg_ctx* c, F&& f) {
  try {
    if (c) {
      cudaError_t e = cudaSetDevice(c->p.device);
      if (e != cudaSuccess) return fail(OKG_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    }
    f();
    return OKG_OK;
  } catch (const Status& s) {
    return s.code;
  } catch (const std::bad_alloc&) {
    return fail(OKG_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(OKG_EOTHER, "%s", e.what());
  }
}

template <int DIM>
static void newton_step_impl(okg_ctx* c, okg_step_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  const long long l0 = g_launches.load();
  okg_step_stats st;
  std::memset(&st, 0, sizeof st);
  const okg_params& p = c->p;
  const size_t B = c->B;
  copy(c, F(c, c->u_old), F(c, c->u), B);
  copy(c, F(c, c->w_old), F(c, c->w), B);
  double s2 = 0.0;
  // residual(next, old) with next = old; gb = -[R1; R2]  (model.hpp:178, :187-190)
  double rnorm = residual<DIM>(c, c->u, c->w, c->u_old, c->w_old, c->gb, c->gb + B, -1.0, &s2);
  const double ref = std::max(1.0, rnorm);
  bool done = rnorm <= p.newton_tol * ref;
  while (!done && st.newton_iters < p.newton_maxit) {
    linearize<DIM>(c, c->u);  // Me at next.u (model.hpp:184-185)
    okg_krylov_stats ks;
    gmres<DIM>(c, c->gb, c->gx, p.gmres_tol, p.gmres_maxit, p.gmres_restart, &ks, s2);
    if (st.newton_iters < OKG_MAX_NEWTON) st.gmres_iters[st.newton_iters] = ks.iterations;
    // require_finite(lin.x) (model.hpp:196)
    CK(cudaMemsetAsync(c->dflag, 0, sizeof(int), c->stream));
    launch(c, k_check_finite, vblk(2 * c->seg.len), BS, 0, (const double*)F(c, c->gx), c->seg, 2 * c->seg.len,
           c->dflag);
    note(c);
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, c->dflag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->hred[R_FLAG] = flag ? 1.0 : 0.0;
    allreduce(c, R_FLAG, 1);
    if (c->hred[R_FLAG] != 0.0) {
      c->have_lin = false;
      THROW(OKG_EINVAL, "newton update: vector contains NaN/Inf");
    }
    axpy(c, 1.0, F(c, c->gx), F(c, c->u), B);
    axpy(c, 1.0, F(c, c->gx) + B, F(c, c->w), B);
    ++st.newton_iters;
    rnorm = residual<DIM>(c, c->u, c->w, c->u_old, c->w_old, c->gb, c->gb + B, -1.0, &s2);
    done = rnorm <= p.newton_tol * ref;
  }
  c->have_lin = false;  // ctx.Me = nullptr (model.hpp:207)
  CK(cudaStreamSynchronize(c->stream));
  std::swap(c->u, c->u_old);
  std::swap(c->w, c->w_old);
  c->t += p.dt;
  c->step += 1;
  st.step = c->step;
  st.t = c->t;
  st.residual_norm = rnorm;
  st.converged = done ? 1 : 0;
  st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st.kernel_launches = g_launches.load() - l0;
  if (stats) *stats = st;
}

template <int DIM>
static void apply_impl(okg_ctx* c, int kind, int level, const double* x, double* y) {
  const int nlev = static_cast<int>(c->lv.size());
  switch (kind) {
    case OKG_OP_M: apply_level<DIM>(c, 0, c->M, x, y); break;
    case OKG_OP_K: apply_level<DIM>(c, 0, c->K, x, y); break;
    case OKG_OP_A: apply_level<DIM>(c, 0, c->A, x, y); break;
    case OKG_OP_SHAT:
      if (level < 0 || level >= nlev) THROW(OKG_EINVAL, "level out of range");
      apply_level<DIM>(c, level, c->lv[level].shat, x, y);
      break;
    case OKG_OP_PROLONG:
      if (level < 0 || level + 1 >= nlev) THROW(OKG_EINVAL, "level out of range");
      CK(cudaMemsetAsync(y, 0, c->lv[level].g.N * sizeof(double), c->stream));
      launch(c, k_prolong_add<DIM>, nblk(c->lv[level].g.N), BS, 0, c->lv[level].g, c->lv[level + 1].g, x, y);
      note(c);
      break;
    case OKG_OP_RESTRICT:
      if (level < 0 || level + 1 >= nlev) THROW(OKG_EINVAL, "level out of range");
      launch(c, k_restrict<DIM>, nblk(c->lv[level + 1].g.N), BS, 0, c->lv[level].g, c->lv[level + 1].g, x, y);
      note(c);
      break;
    case OKG_OP_VCYCLE:  // mg_cycle on level `level` (v_cycle: level 0, multigrid.hpp:124-129)
      if (level < 0 || level >= nlev || (level > 0 && c->nslabs > 1)) THROW(OKG_EINVAL, "level out of range");
      mg_level<DIM>(c, level, x, y, false);
      break;
    case OKG_OP_SHAT_INV: shat_inv<DIM>(c, x, y, c->p.mg_cycles); break;
    case OKG_OP_CHEB_M: cheb<DIM>(c, c->M, x, y); break;
    case OKG_OP_CHEB_A: cheb<DIM>(c, c->A, x, y); break;
    case OKG_OP_ME:
      check_lin(c, "Me apply");
      capply<DIM, CM_ME>(c, x, nullptr, nullptr, y, c->p.eps * c->p.eps);
      break;
    case OKG_OP_C:
      check_lin(c, "constraint block");
      capply<DIM, CM_C>(c, x, nullptr, nullptr, y, 0.0);
      break;
    case OKG_OP_SCHUR:
      check_lin(c, "schur action");
      apply_schur<DIM>(c, x, nullptr, y);
      break;
    case OKG_OP_SCHUR_TILDE_INV: schur_tilde_inv<DIM>(c, x, y); break;
    case OKG_OP_S_INV_APPROX:
      check_lin(c, "schur action");
      s_inv_approx<DIM>(c, x, y);
      break;
    case OKG_OP_BLOCK:
      check_lin(c, "block preconditioner");
      apply_block<DIM>(c, x, y);
      break;
    case OKG_OP_JACOBIAN:
      check_lin(c, "jacobian apply");
      jacobian<DIM>(c, x, y);
      break;
    case OKG_OP_NONLINEAR:
      exchange(c, 0, x);
      launch(c, k_nonlinear<DIM>, own(c->fine), BS, 0, c->fine, c->nl, x, y);
      note(c);
      break;
    case OKG_OP_COARSE_SOLVE: coarse_solve<DIM>(c, x, y); break;
    case OKG_OP_SSOR_M:
      if (c->nslabs > 1) THROW(OKG_EINVAL, "okg_apply: SSOR sweeps need one slab");
      ssor_apply<DIM>(c, c->M, x, y, c->cr2);
      break;
    default: THROW(OKG_EINVAL, "okg_apply: unknown kind %d", kind);
  }
}

extern "C" {

int okg_default_params(okg_params* p) {
  if (!p) return fail(OKG_EINVAL, "null params");
  std::memset(p, 0, sizeof *p);
  p->dim = 2;
  p->n = 64;
  p->eps = 0.02;
  p->sigma = 100.0;
  p->m = 0.4;
  p->theta = 0.5;
  p->dt = 4.0e-4;
  p->newton_tol = 1e-8;
  p->newton_maxit = 20;
  p->gmres_tol = 1e-6;
  p->gmres_maxit = 200;
  p->gmres_restart = 0;
  p->cheby_iters = 10;
  p->richardson_steps = 2;
  p->mg_cycles = 5;
  p->mg_pre = 2;
  p->mg_post = 2;
  p->mg_omega = 2.0 / 3.0;
  p->min_coarse_size = 500;
  p->shat_perturb = 0.0;
  p->max_dofs = 2000000;
  p->device = 0;
  p->use_graphs = 1;
  return OKG_OK;
}

int okg_validate_params(const okg_params* p) {
  // SolverConfig::validate (params.hpp:68-116), fields present in okg_params
  if (!(p->eps > 0.0)) return fail(OKG_ECONFIG, "config: eps must be positive");
  if (p->sigma < 0.0) return fail(OKG_ECONFIG, "config: sigma must be nonnegative");
  if (!(std::abs(p->m) < 1.0)) return fail(OKG_ECONFIG, "config: mean m must satisfy |m| < 1");
  if (!(p->theta > 0.0) || p->theta > 1.0) return fail(OKG_ECONFIG, "config: theta must lie in (0, 1]");
  if (!(p->dt > 0.0)) return fail(OKG_ECONFIG, "config: dt must be positive");
  if (p->dim != 2 && p->dim != 3) return fail(OKG_ECONFIG, "config: dim must be 2 or 3");
  if (p->n < 1) return fail(OKG_ECONFIG, "config: n must be at least 1");
  if (!(p->newton_tol > 0.0)) return fail(OKG_ECONFIG, "config: newton_tol must be positive");
  if (p->newton_maxit < 1) return fail(OKG_ECONFIG, "config: newton_maxit must be at least 1");
  if (!(p->gmres_tol > 0.0)) return fail(OKG_ECONFIG, "config: gmres_tol must be positive");
  if (p->gmres_maxit < 1) return fail(OKG_ECONFIG, "config: gmres_maxit must be at least 1");
  if (p->gmres_restart < 0) return fail(OKG_ECONFIG, "config: gmres_restart must be nonnegative");
  if (p->cheby_iters < 1) return fail(OKG_ECONFIG, "config: cheby_iters must be at least 1");
  if (p->richardson_steps < 1) return fail(OKG_ECONFIG, "config: richardson_steps must be at least 1");
  if (p->mg_cycles < 1) return fail(OKG_ECONFIG, "config: mg_cycles must be at least 1");
  if (p->mg_pre < 0 || p->mg_post < 0 || p->mg_pre + p->mg_post < 1)
    return fail(OKG_ECONFIG, "config: need at least one smoothing sweep per cycle");
  if (!(p->mg_omega > 0.0) || !(p->mg_omega < 2.0)) return fail(OKG_ECONFIG, "config: mg_omega must lie in (0, 2)");
  if (p->min_coarse_size < 1) return fail(OKG_ECONFIG, "config: min_coarse_size must be at least 1");
  if (p->max_dofs < 1) return fail(OKG_ECONFIG, "config: max_dofs must be at least 1");
  int64_t s = (int64_t)p->n + 1, v = s * s;
  if (p->dim == 3) v *= s;
  if (v > p->max_dofs)
    return fail(OKG_ECONFIG, "config: mesh has %lld vertices, exceeding max_dofs = %lld", (long long)v,
                (long long)p->max_dofs);
  return OKG_OK;
}

int okg_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(g_err.size());
}

}  // extern "C"

// ---- contexts ---------------------------------------------------------------------------
static void destroy_ctx(okg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->p.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->g_arn) cudaGraphExecDestroy(c->g_arn);
  if (c->g_prec) cudaGraphExecDestroy(c->g_prec);
  for (void* p : c->allocs) cudaFree(p);
  if (c->hred) cudaFreeHost(c->hred);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->comm) c->ncl->CommDestroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// argument checks, derived constants, stream, then build (one slab)
static void init_ctx(okg_ctx* c) {
  const okg_params* p = &c->p;
  // argument checks of build_mesh (mesh.hpp:88-90), make_schur_context (precond.hpp:132-147),
  // compute_c (precond.hpp:31-38)
  if (p->dim != 2 && p->dim != 3) THROW(OKG_EINVAL, "build_mesh: dim must be 2 or 3");
  if (p->n < 1) THROW(OKG_EINVAL, "build_mesh: n must be positive");
  if (!(p->eps > 0.0)) THROW(OKG_EINVAL, "schur context: eps must be positive");
  const double scale_factor = 1.0 + p->shat_perturb;
  if (!(scale_factor > 0.0)) THROW(OKG_EINVAL, "schur context: perturbation must keep the shifted operator positive");
  if (!(p->dt > 0.0)) THROW(OKG_EINVAL, "compute_c: dt must be positive");
  if (!(p->theta > 0.0) || p->theta > 1.0) THROW(OKG_EINVAL, "compute_c: theta must lie in (0, 1]");
  if (p->sigma < 0.0) THROW(OKG_EINVAL, "compute_c: sigma must be nonnegative");
  if (p->min_coarse_size < 1) THROW(OKG_EINVAL, "build_hierarchy: min_coarse_size < 1");
  if (p->cheby_iters < 1) THROW(OKG_EINVAL, "chebyshev: need at least one step");
  if (p->richardson_steps < 1) THROW(OKG_EINVAL, "schur solve: need at least one refinement step");
  if (p->mg_cycles < 1 || p->mg_pre < 0 || p->mg_post < 0) THROW(OKG_EINVAL, "multigrid: bad cycle settings");
  if (p->gmres_maxit < 1 || p->gmres_restart < 0) THROW(OKG_EINVAL, "gmres: bad iteration settings");
  const int64_t s = (int64_t)p->n + 1;
  const int64_t nv = p->dim == 2 ? s * s : s * s * s;
  if (nv >= (int64_t)1 << 31) THROW(OKG_EINVAL, "mesh too large for one device (%lld vertices)", (long long)nv);
  c->dim = p->dim;
  c->n = p->n;
  c->c = p->dt * p->theta / (1.0 + p->dt * p->theta * p->sigma);
  c->sqrt_c = std::sqrt(c->c);
  c->a_coeff = 1.0 + p->dt * p->theta * p->sigma;
  c->dt_theta = p->dt * p->theta;
  c->shat_scale = scale_factor;
  c->eps_sqrt_c = c->shat_scale * p->eps * c->sqrt_c;
  CK(cudaSetDevice(p->device));
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (c->nslabs > 1) {
    CK(cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming));
  }
  if (c->dim == 2) build<2>(c);
  else build<3>(c);
}

// ---- slab group runtime: one worker thread per slab ---------------------------------------
static void group_worker(Group* G, int r) {
  long seen = 0;
  for (;;) {
    std::function<void(int)> job;
    {
      std::unique_lock<std::mutex> lk(G->jm);
      G->jcv.wait(lk, [&] { return G->stop || G->jgen != seen; });
      if (G->stop) return;
      seen = G->jgen;
      job = G->job;
    }
    job(r);
    {
      std::lock_guard<std::mutex> lk(G->jm);
      if (++G->done == G->S) G->dcv.notify_all();
    }
  }
}

// run f(slab) on every slab thread and wait; every slab's stream is drained before
// the job counts as done.  Returns the status of the first slab that failed (the
// others abort at their next barrier).
static int run_group(Group* G, const std::function<void(int)>& f) {
  G->count.store(0);
  G->abort.store(false);
  G->first_err.store(-1);
  G->status.assign(G->S, OKG_OK);
  G->msg.assign(G->S, std::string());
  {
    std::lock_guard<std::mutex> lk(G->jm);
    G->job = [G, &f](int r) {
      int st = OKG_OK;
      try {
        if (G->r[r]) CK(cudaSetDevice(G->r[r]->p.device));
        f(r);
        if (G->r[r] && G->r[r]->stream) CK(cudaStreamSynchronize(G->r[r]->stream));
      } catch (const Status& s) {
        st = s.code;
      } catch (const std::bad_alloc&) {
        st = fail(OKG_ENOMEM, "host allocation failed");
      } catch (const std::exception& e) {
        st = fail(OKG_EOTHER, "%s", e.what());
      }
      if (st != OKG_OK) {
        G->status[r] = st;
        G->msg[r] = g_err;
        int expect = -1;
        G->first_err.compare_exchange_strong(expect, r);
        G->abort.store(true);
      }
    };
    G->done = 0;
    ++G->jgen;
  }
  G->jcv.notify_all();
  {
    std::unique_lock<std::mutex> lk(G->jm);
    G->dcv.wait(lk, [&] { return G->done == G->S; });
  }
  const int e = G->first_err.load();
  if (e < 0) return OKG_OK;
  g_err = G->msg[e];
  return G->status[e];
}

static void destroy_handle(okg_ctx* h) {
  if (!h) return;
  if (Group* G = h->group) {
    if (!G->th.empty()) {
      run_group(G, [G](int r) {
        destroy_ctx(G->r[r]);
        G->r[r] = nullptr;
      });
      {
        std::lock_guard<std::mutex> lk(G->jm);
        G->stop = true;
      }
      G->jcv.notify_all();
      for (auto& t : G->th) t.join();
    }
    delete G;
  }
  delete h;
}

// f(slab context) on every slab of c (on c itself for a one-slab context)
template <class Fn>
static int each_slab(okg_ctx* c, Fn&& f) {
  if (!c->handle)
    return guard(c, [&] {
      f(c);
      CK(cudaStreamSynchronize(c->stream));
    });
  Group* G = c->group;
  return run_group(G, [&](int r) { f(G->r[r]); });
}

static okg_ctx* slab0(okg_ctx* c) { return c->handle ? c->group->r[0] : c; }

#define SINGLE_SLAB(c, fn)                                                                                    \
  do {                                                                                                        \
    if ((c)->handle || (c)->nslabs > 1)                                                                       \
      return fail(OKG_EINVAL, "%s: device-pointer entry point on a %d-slab context (use the host-pointer API)", \
                  fn, (c)->nslabs);                                                                           \
  } while (0)

// host N-vector blocks <-> the owned planes of a slab's stacked level-0 vector
static void put_owned(okg_ctx* c, const double* h, double* d, int nb) {
  const size_t lo = c->fine.lo, cnt = c->fine.hi - c->fine.lo;
  for (int q = 0; q < nb; ++q)
    CK(cudaMemcpyAsync(d + (size_t)q * c->B + lo, h + (size_t)q * c->N + lo, cnt * sizeof(double),
                       cudaMemcpyHostToDevice, c->stream));
}
static void get_owned(okg_ctx* c, const double* d, double* h, int nb) {
  const size_t lo = c->fine.lo, cnt = c->fine.hi - c->fine.lo;
  for (int q = 0; q < nb; ++q)
    CK(cudaMemcpyAsync(h + (size_t)q * c->N + lo, d + (size_t)q * c->B + lo, cnt * sizeof(double),
                       cudaMemcpyDeviceToHost, c->stream));
}
static void ensure_io(okg_ctx* c) {
  if (c->io_a) return;  // every slab allocates at the same call: registry indices stay aligned
  c->io_a = lvec(c, c->lv[0], 0, 2);
  c->io_b = lvec(c, c->lv[0], 0, 2);
  c->io_c = lvec(c, c->lv[0], 0, 2);
}

// vector lengths of okg_apply kinds: {input, output} vertex counts
static void apply_sizes(okg_ctx* c, int kind, int level, size_t& nin, size_t& nout) {
  const int nlev = static_cast<int>(c->lv.size());
  nin = nout = c->N;
  switch (kind) {
    case OKG_OP_BLOCK: case OKG_OP_JACOBIAN: nin = nout = 2 * (size_t)c->N; break;
    case OKG_OP_SHAT: case OKG_OP_VCYCLE:
      if (level < 0 || level >= nlev) THROW(OKG_EINVAL, "level out of range");
      nin = nout = c->lv[level].g.N;
      break;
    case OKG_OP_PROLONG:
      if (level < 0 || level + 1 >= nlev) THROW(OKG_EINVAL, "level out of range");
      nin = c->lv[level + 1].g.N;
      nout = c->lv[level].g.N;
      break;
    case OKG_OP_RESTRICT:
      if (level < 0 || level + 1 >= nlev) THROW(OKG_EINVAL, "level out of range");
      nin = c->lv[level].g.N;
      nout = c->lv[level + 1].g.N;
      break;
    case OKG_OP_COARSE_SOLVE: nin = nout = c->lv.back().g.N; break;
    default: break;
  }
}

extern "C" {

int okg_create(const okg_params* p, okg_ctx** out) {
  if (!p || !out) return fail(OKG_EINVAL, "okg_create: null argument");
  *out = nullptr;
  const int S = p->nslabs < 1 ? 1 : p->nslabs;
  if (S > 16) return fail(OKG_EINVAL, "okg_create: at most 16 slabs (nslabs = %d)", S);
  if (S == 1) {
    okg_ctx* c = new okg_ctx();
    c->p = *p;
    c->p.nslabs = 1;
    const int st = guard(nullptr, [&] { init_ctx(c); });
    if (st != OKG_OK) {
      destroy_ctx(c);
      return st;
    }
    *out = c;
    return OKG_OK;
  }
  // several slabs: a handle + one worker thread (own stream, own device buffers) per slab
  okg_ctx* h = new okg_ctx();
  h->p = *p;
  h->handle = true;
  h->nslabs = S;
  h->dim = p->dim;
  h->n = p->n;
  Group* G = new Group();
  G->S = S;
  G->r.assign(S, nullptr);
  G->scratch.assign((size_t)S * 256, 0.0);
  h->group = G;
  for (int r = 0; r < S; ++r) G->th.emplace_back(group_worker, G, r);
  const int st = run_group(G, [&](int r) {
    okg_ctx* c = new okg_ctx();
    c->p = *p;
    c->p.device = p->device + (p->slab_devices ? r : 0);
    c->p.use_graphs = 0;  // cross-slab exchanges are host-ordered: not capturable
    c->rank = r;
    c->nslabs = S;
    c->group = G;
    G->r[r] = c;  // published before the first barrier of build()
    CK(cudaSetDevice(c->p.device));
    if (p->slab_devices)
      for (int q = 0; q < S; ++q) {
        const int dq = p->device + q;
        int ok = 0;
        if (dq == c->p.device || cudaDeviceCanAccessPeer(&ok, c->p.device, dq) != cudaSuccess || !ok) continue;
        const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
        if (e != cudaSuccess) (void)cudaGetLastError();  // already enabled / staged copies still work
      }
    init_ctx(c);
  });
  if (st != OKG_OK) {
    destroy_handle(h);
    return st;
  }
  okg_ctx* c0 = G->r[0];
  h->N = c0->N;
  h->c = c0->c;
  h->sqrt_c = c0->sqrt_c;
  h->a_coeff = c0->a_coeff;
  h->dt_theta = c0->dt_theta;
  h->eps_sqrt_c = c0->eps_sqrt_c;
  *out = h;
  return OKG_OK;
}

int okg_nccl_unique_id(void* id, size_t len) {
  if (!id || len < sizeof(ncclUniqueId)) return fail(OKG_EINVAL, "okg_nccl_unique_id: need %zu bytes", sizeof(ncclUniqueId));
  std::string why;
  const NcclApi* nc = nccl_api(&why);
  if (!nc) return fail(OKG_ECUDA, "%s", why.c_str());
  ncclUniqueId u;
  const ncclResult_t r = nc->GetUniqueId(&u);
  if (r != ncclSuccess) return fail(OKG_ECUDA, "ncclGetUniqueId: %s", nc->GetErrorString(r));
  std::memcpy(id, &u, sizeof u);
  return OKG_OK;
}

int okg_create_rank(const okg_params* p, int32_t rank, int32_t nranks, const void* nccl_id, okg_ctx** out) {
  if (!p || !out) return fail(OKG_EINVAL, "okg_create_rank: null argument");
  *out = nullptr;
  if (nranks < 1 || nranks > 16 || rank < 0 || rank >= nranks)
    return fail(OKG_EINVAL, "okg_create_rank: rank %d of %d", rank, nranks);
  if (nranks > 1 && !nccl_id) return fail(OKG_EINVAL, "okg_create_rank: %d ranks need an NCCL id", nranks);
  okg_ctx* c = new okg_ctx();
  c->p = *p;
  c->p.nslabs = nranks;
  c->rank = rank;
  c->nslabs = nranks;
  if (nranks > 1) c->p.use_graphs = 0;
  const int st = guard(nullptr, [&] {
    CK(cudaSetDevice(p->device));
    if (nccl_id) {
      std::string why;
      c->ncl = nccl_api(&why);
      if (!c->ncl) THROW(OKG_ECUDA, "%s", why.c_str());
      ncclUniqueId u;
      std::memcpy(&u, nccl_id, sizeof u);
      NCK(c, c->ncl->CommInitRank(&c->comm, nranks, u, rank));
    }
    init_ctx(c);
  });
  if (st != OKG_OK) {
    destroy_ctx(c);
    return st;
  }
  *out = c;
  return OKG_OK;
}

int okg_slab_partition(int32_t dim, int32_t n, int32_t min_coarse_size, int32_t nslabs, int32_t rank,
                       int64_t rep_max_vertices, int32_t* levels, int32_t* rep_level, int32_t* lo, int32_t* hi) {
  if ((dim != 2 && dim != 3) || n < 1 || min_coarse_size < 1 || nslabs < 1 || rank < 0 || rank >= nslabs || !levels ||
      !rep_level || !lo || !hi)
    return fail(OKG_EINVAL, "okg_slab_partition: bad argument");
  // build_hierarchy's level count (multigrid.hpp:55-86)
  int nlev = 0;
  for (int ln = n;; ln /= 2) {
    ++nlev;
    const int64_t s = (int64_t)ln + 1, N = dim == 2 ? s * s : s * s * s;
    if (!(N > min_coarse_size && ln % 2 == 0) || nlev == 32) break;
  }
  *levels = nlev;
  std::vector<int> l0(nlev, 0), h0(nlev, 0);
  for (int l = 0; l < nlev; ++l) h0[l] = (n >> l) + 1;  // one slab / replicated level: every plane
  int rep = nlev;
  if (nslabs > 1) {
    rep = slab_partition(dim, n + 1, nlev, nslabs, rank, rep_max_vertices == 0 ? rep_max_default() : rep_max_vertices,
                         l0.data(), h0.data());
    if (rep == 0) return fail(OKG_EINVAL, "slab decomposition: %d slabs leave fewer than 2 planes each", nslabs);
    for (int l = rep; l < nlev; ++l) {
      l0[l] = 0;
      h0[l] = (n >> l) + 1;
    }
  }
  *rep_level = rep;
  for (int l = 0; l < nlev; ++l) {
    lo[l] = l0[l];
    hi[l] = h0[l];
  }
  return OKG_OK;
}

void okg_destroy(okg_ctx* c) {
  if (c && c->handle) destroy_handle(c);
  else destroy_ctx(c);
}

int okg_get_info(okg_ctx* h, okg_info* info) {
  if (!h || !info) return fail(OKG_EINVAL, "null argument");
  okg_ctx* c = slab0(h);
  std::memset(info, 0, sizeof *info);
  info->dim = c->dim;
  info->n = c->n;
  info->num_vertices = c->N;
  info->levels = static_cast<int>(c->lv.size());
  for (size_t l = 0; l < c->lv.size() && l < 32; ++l) {
    info->level_size[l] = c->lv[l].g.N;
    info->level_n[l] = c->lv[l].g.n;
  }
  info->c = c->c;
  info->sqrt_c = c->sqrt_c;
  info->a_coeff = c->a_coeff;
  info->dt_theta = c->dt_theta;
  info->lambda_lo = c->lambda_lo;
  info->lambda_hi = c->lambda_hi;
  info->eps_sqrt_c = c->eps_sqrt_c;
  info->graph_nodes = c->arn_nodes;
  info->tail_start = c->tail_start;
  info->tail_cluster = c->tail_start > 0 ? c->tail_cluster : 0;
  info->coarse_rows = c->coarse_big ? c->coarse_r1 - c->coarse_r0 : c->nc;
  info->collapse_level = c->collapse_level;
  for (size_t l = 0; l < c->lv.size() && l < 31; ++l)
    if (c->lv[l].tiled) info->tiled_mask |= (1 << l);
  info->nslabs = h->handle ? h->nslabs : c->nslabs;
  info->rep_level = std::min<int>(c->L_rep, (int)c->lv.size());
  if (h->handle)
    for (okg_ctx* s : h->group->r) info->device_bytes += static_cast<int64_t>(s->bytes);
  else
    info->device_bytes = static_cast<int64_t>(c->bytes);  // this process's slab
  for (int r = 0; r < info->nslabs; ++r) {
    std::vector<int> lo(c->lv.size()), hi(c->lv.size());
    if (info->nslabs > 1) {
      slab_partition(c->dim, c->lv[0].g.s, (int)c->lv.size(), info->nslabs, r, rep_max_of(c->p), lo.data(), hi.data());
    } else {
      lo[0] = 0;
      hi[0] = c->lv[0].g.s;
    }
    info->slab_ilo[r] = lo[0];
    info->slab_ihi[r] = hi[0];
  }
  return OKG_OK;
}

int okg_mesh(int32_t dim, int32_t n, double* vertices, int32_t* cells) {
  // build_mesh (mesh.hpp:87-157): same vertex order and cell connectivity
  if (dim != 2 && dim != 3) return fail(OKG_EINVAL, "build_mesh: dim must be 2 or 3");
  if (n < 1) return fail(OKG_EINVAL, "build_mesh: n must be positive");
  const double h = 1.0 / n;
  const int s = n + 1;
  auto gi = [&](int i, int j, int k) { return dim == 2 ? i * s + j : (i * s + j) * s + k; };
  size_t p = 0, q = 0;
  if (dim == 2) {
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        vertices[p++] = i * h;
        vertices[p++] = j * h;
      }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const int a = gi(i, j, 0), b = gi(i + 1, j, 0), cc = gi(i + 1, j + 1, 0), d = gi(i, j + 1, 0);
        const int v[6] = {a, b, cc, a, cc, d};
        for (int t = 0; t < 6; ++t) cells[q++] = v[t];
      }
  } else {
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j)
        for (int k = 0; k < s; ++k) {
          vertices[p++] = i * h;
          vertices[p++] = j * h;
          vertices[p++] = k * h;
        }
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const bool odd[6] = {false, true, true, false, false, true};
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k)
          for (int pp = 0; pp < 6; ++pp) {
            int g[3] = {i, j, k};
            int idx[4];
            idx[0] = gi(g[0], g[1], g[2]);
            for (int v = 1; v < 4; ++v) {
              g[perms[pp][v - 1]] += 1;
              idx[v] = gi(g[0], g[1], g[2]);
            }
            if (odd[pp]) std::swap(idx[1], idx[2]);
            for (int t = 0; t < 4; ++t) cells[q++] = idx[t];
          }
  }
  return OKG_OK;
}

int okg_seeded_ic(int64_t nverts, uint64_t seed, double m, double* u) {
  // counter-based splitmix64 keyed by (seed, global vertex id)
  for (int64_t g = 0; g < nverts; ++g) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(g) + 0x632BE59BD9B4E019ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x = x ^ (x >> 31);
    const double U = 2.0 * (static_cast<double>(x >> 11) * 0x1.0p-53) - 1.0;
    u[g] = m + 0.01 * U;
  }
  return OKG_OK;
}

int okg_set_state(okg_ctx* c, const double* u, const double* w, double t, int32_t step) {
  if (!c || !u || !w) return fail(OKG_EINVAL, "okg_set_state: null argument");
  return each_slab(c, [&](okg_ctx* s) {
    put_owned(s, u, s->u_old, 1);
    put_owned(s, w, s->w_old, 1);
    s->t = t;
    s->step = step;
  });
}

int okg_get_state(okg_ctx* c, double* u, double* w, double* t, int32_t* step) {
  if (!c) return fail(OKG_EINVAL, "okg_get_state: null context");
  const int st = each_slab(c, [&](okg_ctx* s) {
    if (u) get_owned(s, s->u_old, u, 1);
    if (w) get_owned(s, s->w_old, w, 1);
  });
  if (st == OKG_OK) {
    if (t) *t = slab0(c)->t;
    if (step) *step = slab0(c)->step;
  }
  return st;
}

// newton_solve on every slab; the statistics are slab 0's (every slab takes the same
// decisions: all scalars are allreduced), launches and seconds cover the whole group
static int newton_all(okg_ctx* c, const double* u_old, const double* w_old, double* u_new, double* w_new,
                      okg_step_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  const long long l0 = g_launches.load();
  okg_step_stats s0;
  std::memset(&s0, 0, sizeof s0);
  const int st = each_slab(c, [&](okg_ctx* s) {
    okg_step_stats ss;
    if (u_old) put_owned(s, u_old, s->u_old, 1);
    if (w_old) put_owned(s, w_old, s->w_old, 1);
    DISPATCH(s, newton_step_impl, s, &ss);
    if (u_new) get_owned(s, s->u_old, u_new, 1);
    if (w_new) get_owned(s, s->w_old, w_new, 1);
    if (s->rank == 0) s0 = ss;
  });
  if (st == OKG_OK && stats) {
    *stats = s0;
    stats->kernel_launches = g_launches.load() - l0;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return st;
}

int okg_newton_step(okg_ctx* c, okg_step_stats* stats) {
  if (!c) return fail(OKG_EINVAL, "okg_newton_step: null context");
  return newton_all(c, nullptr, nullptr, nullptr, nullptr, stats);
}

int okg_newton_step_host(okg_ctx* c, const double* u_old, const double* w_old, double* u_new, double* w_new,
                         okg_step_stats* stats) {
  if (!c || !u_old || !w_old || !u_new || !w_new) return fail(OKG_EINVAL, "okg_newton_step_host: null argument");
  return newton_all(c, u_old, w_old, u_new, w_new, stats);
}

// ---- diagnostics and initial state ------------------------------------------
// u == NULL: the context's current state; else a host array of N doubles
static const double* diag_input(okg_ctx* s, const double* u) {
  if (!u) return s->u_old;
  ensure_io(s);
  put_owned(s, u, s->io_a, 1);
  return s->io_a;
}

int okg_total_mass(okg_ctx* c, const double* u, double* mass) {
  if (!c || !mass) return fail(OKG_EINVAL, "okg_total_mass: null argument");
  double r0 = 0.0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    const double v = DISPATCH(s, total_mass_impl, s, diag_input(s, u));
    if (s->rank == 0) r0 = v;
  });
  if (st == OKG_OK) *mass = r0;
  return st;
}

int okg_double_well(okg_ctx* c, const double* u, double* value) {
  if (!c || !value) return fail(OKG_EINVAL, "okg_double_well: null argument");
  double r0 = 0.0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    const double v = DISPATCH(s, double_well_impl, s, diag_input(s, u));
    if (s->rank == 0) r0 = v;
  });
  if (st == OKG_OK) *value = r0;
  return st;
}

int okg_energy(okg_ctx* c, const double* u, double* energy, int32_t* cg_iters) {
  if (!c || !energy) return fail(OKG_EINVAL, "okg_energy: null argument");
  double r0 = 0.0;
  int it0 = 0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    int its = 0;
    const double v = DISPATCH(s, energy_impl, s, diag_input(s, u), &its);
    if (s->rank == 0) {
      r0 = v;
      it0 = its;
    }
  });
  if (st == OKG_OK) {
    *energy = r0;
    if (cg_iters) *cg_iters = it0;
  }
  return st;
}

int okg_initial_state(okg_ctx* c, int32_t* cg_iters) {
  if (!c) return fail(OKG_EINVAL, "okg_initial_state: null context");
  int it0 = 0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    int its = 0;
    DISPATCH(s, initial_state_impl, s, &its);
    if (s->rank == 0) it0 = its;
  });
  if (st == OKG_OK && cg_iters) *cg_iters = it0;
  return st;
}

int okg_advance(okg_ctx* c, int32_t with_energy, okg_step_stats* stats) {
  if (!c) return fail(OKG_EINVAL, "okg_advance: null context");
  okg_step_stats st0;
  int st = newton_all(c, nullptr, nullptr, nullptr, nullptr, &st0);
  if (st != OKG_OK) return st;
  // advance (model.hpp:218-227): diagnostics of the new state
  double mass = 0.0, en = 0.0;
  st = each_slab(c, [&](okg_ctx* s) {
    const double m = DISPATCH(s, total_mass_impl, s, s->u_old);
    const double e = with_energy ? DISPATCH(s, energy_impl, s, s->u_old, nullptr) : 0.0;
    if (s->rank == 0) {
      mass = m;
      en = e;
    }
  });
  if (st != OKG_OK) return st;
  st0.mass = mass;
  st0.energy = with_energy ? en : NAN;
  if (stats) *stats = st0;
  return OKG_OK;
}

int okg_clear_linearization(okg_ctx* c) {
  if (!c) return fail(OKG_EINVAL, "null context");
  if (c->handle)
    for (okg_ctx* s : c->group->r) s->have_lin = false;
  else
    c->have_lin = false;
  return OKG_OK;
}

// ---- host-pointer entry points (any number of slabs) -------------------------------------
int okg_linearize_host(okg_ctx* c, const double* u) {
  if (!c || !u) return fail(OKG_EINVAL, "okg_linearize_host: null argument");
  return each_slab(c, [&](okg_ctx* s) {
    ensure_io(s);
    put_owned(s, u, s->io_a, 1);
    DISPATCH(s, linearize, s, s->io_a);
  });
}

int okg_apply_host(okg_ctx* c, int32_t kind, int32_t level, const double* x, double* y) {
  if (!c || !x || !y) return fail(OKG_EINVAL, "okg_apply_host: null argument");
  if (kind < OKG_OP_M || kind > OKG_OP_SSOR_M) return fail(OKG_EINVAL, "okg_apply_host: unknown kind %d", kind);
  const bool level0 = !(kind == OKG_OP_PROLONG || kind == OKG_OP_RESTRICT || kind == OKG_OP_COARSE_SOLVE ||
                        ((kind == OKG_OP_SHAT || kind == OKG_OP_VCYCLE) && level != 0));
  if (c->handle && !level0)
    return fail(OKG_EINVAL, "okg_apply_host: kind %d on level %d needs a one-slab context", kind, level);
  return each_slab(c, [&](okg_ctx* s) {
    if (level0) {
      const int nb = (kind == OKG_OP_BLOCK || kind == OKG_OP_JACOBIAN) ? 2 : 1;
      ensure_io(s);
      put_owned(s, x, s->io_a, nb);
      DISPATCH(s, apply_impl, s, kind, level, s->io_a, s->io_b);
      get_owned(s, s->io_b, y, nb);
    } else {
      size_t nin = 0, nout = 0;
      apply_sizes(s, kind, level, nin, nout);
      double* dx = dalloc(s, nin);
      double* dy = dalloc(s, nout);
      CK(cudaMemcpyAsync(dx, x, nin * sizeof(double), cudaMemcpyHostToDevice, s->stream));
      DISPATCH(s, apply_impl, s, kind, level, dx, dy);
      CK(cudaMemcpyAsync(y, dy, nout * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      CK(cudaStreamSynchronize(s->stream));
      for (double* q : {dx, dy}) {
        cudaFree(q);
        s->allocs.erase(std::find(s->allocs.begin(), s->allocs.end(), (void*)q));
      }
      s->bytes -= (nin + nout) * sizeof(double);
    }
  });
}

int okg_residual_host(okg_ctx* c, const double* un, const double* wn, const double* uo, const double* wo, double* r1,
                      double* r2) {
  if (!c || !un || !wn || !uo || !wo || !r1 || !r2) return fail(OKG_EINVAL, "okg_residual_host: null argument");
  return each_slab(c, [&](okg_ctx* s) {
    ensure_io(s);
    put_owned(s, un, s->io_a, 1);
    put_owned(s, wn, s->io_a + s->B, 1);
    put_owned(s, uo, s->io_b, 1);
    put_owned(s, wo, s->io_b + s->B, 1);
    DISPATCH(s, residual, s, s->io_a, s->io_a + s->B, s->io_b, s->io_b + s->B, s->io_c, s->io_c + s->B, 1.0,
             nullptr);
    get_owned(s, s->io_c, r1, 1);
    get_owned(s, s->io_c + s->B, r2, 1);
  });
}

int okg_gmres_host(okg_ctx* c, const double* b, double* x, double rel_tol, int32_t max_iter, int32_t restart,
                   okg_krylov_stats* stats) {
  if (!c || !b || !x) return fail(OKG_EINVAL, "okg_gmres_host: null argument");
  okg_krylov_stats k0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    check_lin(s, "jacobian apply");
    ensure_io(s);
    put_owned(s, b, s->io_a, 2);
    okg_krylov_stats ks;
    DISPATCH(s, gmres, s, s->io_a, s->io_b, rel_tol, max_iter, restart, &ks, -1.0);
    get_owned(s, s->io_b, x, 2);
    if (s->rank == 0) k0 = ks;
  });
  if (st == OKG_OK && stats) *stats = k0;
  return st;
}

// ---- length-checked host-pointer entry points: the caller passes its array lengths and a
// mismatch is std::invalid_argument, as the reference's LinearOperator::apply
// (operator.hpp:22-25), gmres (krylov.hpp:48-51) and residual (model.hpp:126-127) throw
int okg_apply_host_n(okg_ctx* c, int32_t kind, int32_t level, const double* x, int64_t nx, double* y, int64_t ny) {
  if (!c || !x || !y) return fail(OKG_EINVAL, "okg_apply_host_n: null argument");
  size_t nin = 0, nout = 0;
  const int st = guard(c, [&] { apply_sizes(slab0(c), kind, level, nin, nout); });
  if (st != OKG_OK) return st;
  if (nx != (int64_t)nin) return fail(OKG_EINVAL, "operator %d: input dimension mismatch (%lld, expected %zu)", kind, (long long)nx, nin);
  if (ny != (int64_t)nout) return fail(OKG_EINVAL, "operator %d: output dimension mismatch (%lld, expected %zu)", kind, (long long)ny, nout);
  return okg_apply_host(c, kind, level, x, y);
}

int okg_linearize_host_n(okg_ctx* c, const double* u, int64_t n) {
  if (!c || !u) return fail(OKG_EINVAL, "okg_linearize_host_n: null argument");
  if (n != (int64_t)slab0(c)->N) return fail(OKG_EINVAL, "assemble_coefficient_mass: vector length mismatch");
  return okg_linearize_host(c, u);
}

int okg_residual_host_n(okg_ctx* c, const double* un, const double* wn, const double* uo, const double* wo, int64_t n,
                        double* r1, double* r2) {
  if (!c) return fail(OKG_EINVAL, "okg_residual_host_n: null argument");
  if (n != (int64_t)slab0(c)->N) return fail(OKG_EINVAL, "residual: states do not match the mesh");
  return okg_residual_host(c, un, wn, uo, wo, r1, r2);
}

int okg_gmres_host_n(okg_ctx* c, const double* b, double* x, int64_t n, double rel_tol, int32_t max_iter,
                     int32_t restart, okg_krylov_stats* stats) {
  if (!c) return fail(OKG_EINVAL, "okg_gmres_host_n: null argument");
  if (n != 2 * (int64_t)slab0(c)->N) return fail(OKG_EINVAL, "gmres: rhs dimension mismatch");
  return okg_gmres_host(c, b, x, rel_tol, max_iter, restart, stats);
}

// ---- device-pointer entry points (one slab) ------------------------------------------------
int okg_linearize(okg_ctx* c, const double* u_dev) {
  if (!c || !u_dev) return fail(OKG_EINVAL, "okg_linearize: null argument");
  SINGLE_SLAB(c, "okg_linearize");
  return guard(c, [&] {
    DISPATCH(c, linearize, c, u_dev);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int okg_apply(okg_ctx* c, int32_t kind, int32_t level, const double* x, double* y) {
  if (!c || !x || !y) return fail(OKG_EINVAL, "okg_apply: null argument");
  SINGLE_SLAB(c, "okg_apply");
  return guard(c, [&] {
    DISPATCH(c, apply_impl, c, kind, level, x, y);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int okg_residual(okg_ctx* c, const double* un, const double* wn, const double* uo, const double* wo, double* r1,
                 double* r2) {
  if (!c || !un || !wn || !uo || !wo || !r1 || !r2) return fail(OKG_EINVAL, "okg_residual: null argument");
  SINGLE_SLAB(c, "okg_residual");
  return guard(c, [&] { DISPATCH(c, residual, c, un, wn, uo, wo, r1, r2, 1.0, nullptr); });
}

int okg_gmres(okg_ctx* c, const double* b, double* x, double rel_tol, int32_t max_iter, int32_t restart,
              okg_krylov_stats* stats) {
  if (!c || !b || !x) return fail(OKG_EINVAL, "okg_gmres: null argument");
  SINGLE_SLAB(c, "okg_gmres");
  return guard(c, [&] {
    check_lin(c, "jacobian apply");
    DISPATCH(c, gmres, c, b, x, rel_tol, max_iter, restart, stats, -1.0);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int okg_jacobi_spectrum(okg_ctx* c, double* lo, double* hi) {
  if (!c || !lo || !hi) return fail(OKG_EINVAL, "null argument");
  double l0 = 0, h0 = 0;
  const int st = each_slab(c, [&](okg_ctx* s) {
    double a = 0, b = 0;
    DISPATCH(s, jacobi_spectrum, s, a, b);
    if (s->rank == 0) {
      l0 = a;
      h0 = b;
    }
  });
  if (st == OKG_OK) {
    *lo = l0;
    *hi = h0;
  }
  return st;
}

int okg_stream(okg_ctx* c, void** stream) {
  if (!c || !stream) return fail(OKG_EINVAL, "null argument");
  *stream = reinterpret_cast<void*>(slab0(c)->stream);
  return OKG_OK;
}

int okg_slab_stream(okg_ctx* c, int32_t slab, void** stream) {
  if (!c || !stream) return fail(OKG_EINVAL, "null argument");
  const int S = c->handle ? c->nslabs : 1;
  if (slab < 0 || slab >= S) return fail(OKG_EINVAL, "okg_slab_stream: slab %d out of range", slab);
  *stream = reinterpret_cast<void*>((c->handle ? c->group->r[slab] : c)->stream);
  return OKG_OK;
}

}  // extern "C"

template <int DIM>
static void kernel_timing_impl(okg_ctx* c, int which, int reps, int flags, double* avg_ms, double* bytes) {
  Level& L0 = c->lv[0];
  const Grid& g = L0.g;
  const double om = c->p.mg_omega;
  const double N = (double)(g.hi - g.lo);  // owned vertices (the whole level on one slab)
  const double B = 8.0;
  // operands: reuse workspace vectors (contents are finite)
  double *x = c->cd0, *b = c->cd1, *y = c->cr, *z = c->kv;
  auto run_once = [&]() {
    const bool T = L0.tiled;
    switch (which) {
      case OKG_KT_SMOOTH:
        if (T) tiled<DIM, L_PLAIN, T_JACOBI>(c, L0, L0.shat, targs(x, b, y, nullptr, om));
        else op_apply<DIM>(c, g, L0.shat, EPI_JACOBI, x, b, y, nullptr, om);
        break;
      case OKG_KT_RESID:
        if (T) tiled<DIM, L_PLAIN, T_RESID>(c, L0, L0.shat, targs(x, b, y, nullptr, 0.0));
        else op_apply<DIM>(c, g, L0.shat, EPI_RESID, x, b, y, nullptr);
        break;
      case OKG_KT_PRE2:
        if (T) tiled<DIM, L_JAC0, T_JACOBI>(c, L0, L0.shat, targs(b, b, y, nullptr, om));
        else {
          launch(c, k_pre2<DIM>, own(g), BS, 0, g, dev_op<DIM>(L0.shat), b, y, om);
          note(c);
        }
        break;
      case OKG_KT_POST_ACC:
        if (T) tiled<DIM, L_PLAIN, T_JACOBI_ACC>(c, L0, L0.shat, targs(x, b, nullptr, z, om));
        else op_apply<DIM>(c, g, L0.shat, EPI_JACOBI_ACC, x, b, nullptr, z, om);
        break;
      case OKG_KT_CHEB:
        if (T) {
          TArgs a = targs(x, b, y, z, 0.0);
          a.x2 = c->zz;
          a.y2 = c->rr;
          a.c1 = c->cheb_c1[0];
          a.c2 = c->cheb_c2[0];
          tiled<DIM, L_PLAIN, T_CHEB>(c, L0, c->A, a);
        } else {
          launch(c, k_cheb_step<DIM>, own(g), BS, 0, g, dev_op<DIM>(c->A), x, b, y, c->zz, c->rr, z,
                                                            c->cheb_c1[0], c->cheb_c2[0], 0, 0);
          note(c);
        }
        break;
      case OKG_KT_JACOBIAN: jacobian<DIM>(c, c->pz, c->pw); break;
      case OKG_KT_RESTRICT:
        launch(c, k_restrict<DIM>, own(c->lv[1].g), BS, 0, g, c->lv[1].g, x, c->lv[1].b);
        note(c);
        break;
      case OKG_KT_PROLONG:
        if (T) {
          TArgs a = targs(x, b, y, nullptr, om);
          a.x2 = c->lv[1].x;
          a.gc = c->lv[1].g;
          tiled<DIM, L_PROLONG, T_JACOBI>(c, L0, L0.shat, a);
        } else {
          launch(c, k_prolong_add<DIM>, own(g), BS, 0, g, c->lv[1].g, c->lv[1].x, y);
          note(c);
        }
        break;
      default: THROW(OKG_EINVAL, "okg_kernel_timing: unknown kernel %d", which);
    }
  };
  if ((which == OKG_KT_RESTRICT || which == OKG_KT_PROLONG) && c->lv.size() < 2)
    THROW(OKG_EINVAL, "okg_kernel_timing: single-level hierarchy");
  const double Nc = c->lv.size() > 1 ? (double)(c->lv[1].g.hi - c->lv[1].g.lo) : 0.0;
  const double npos = Traits<DIM>::NPOS + 1;
  switch (which) {
    case OKG_KT_SMOOTH: case OKG_KT_RESID: *bytes = 3 * N * B; break;
    case OKG_KT_PRE2: *bytes = 2 * N * B; break;
    case OKG_KT_POST_ACC: *bytes = 4 * N * B; break;
    case OKG_KT_CHEB: *bytes = 6 * N * B; break;
    case OKG_KT_JACOBIAN: *bytes = (4 + npos) * N * B; break;
    case OKG_KT_RESTRICT: *bytes = (N + Nc) * B; break;
    case OKG_KT_PROLONG: *bytes = (L0.tiled ? 3 * N + Nc : 2 * N + Nc) * B; break;
  }
  bool had_lin = c->have_lin;
  const bool saved_pdl = c->p.disable_pdl;
  if (flags & OKG_KT_NO_PDL) c->p.disable_pdl = 1;
  for (int i = 0; i < 3; ++i) run_once();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double total_ms = 0.0;
  if (flags & OKG_KT_COLD) {
    // L2-cold: before every launch, overwrite a scratch buffer of twice the L2 size
    // (126 MB on B200), then bracket the launch alone with events
    int dev = 0, l2 = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const size_t fl = 2 * (size_t)std::max(l2, 64 << 20);
    void* scratch = nullptr;
    CK(cudaMalloc(&scratch, fl));
    for (int i = 0; i < reps; ++i) {
      CK(cudaMemsetAsync(scratch, i & 0xff, fl, c->stream));
      CK(cudaEventRecord(e0, c->stream));
      run_once();
      CK(cudaEventRecord(e1, c->stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      total_ms += ms;
    }
    cudaFree(scratch);
  } else {
    CK(cudaEventRecord(e0, c->stream));
    for (int i = 0; i < reps; ++i) run_once();
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    total_ms = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->p.disable_pdl = saved_pdl;
  *avg_ms = total_ms / reps;
  c->have_lin = had_lin;
}

extern "C" {

int okg_kernel_timing(okg_ctx* c, int32_t which, int32_t reps, double* avg_ms, double* bytes) {
  if (!c || !avg_ms || !bytes || reps < 1) return fail(OKG_EINVAL, "okg_kernel_timing: bad argument");
  if (c->handle) return fail(OKG_EINVAL, "okg_kernel_timing: time one slab (okg_create_rank) instead");
  return guard(c, [&] { DISPATCH(c, kernel_timing_impl, c, which, reps, 0, avg_ms, bytes); });
}

int okg_kernel_timing_ex(okg_ctx* c, int32_t which, int32_t reps, int32_t flags, double* avg_ms, double* bytes) {
  if (!c || !avg_ms || !bytes || reps < 1) return fail(OKG_EINVAL, "okg_kernel_timing_ex: bad argument");
  if (c->handle) return fail(OKG_EINVAL, "okg_kernel_timing_ex: time one slab (okg_create_rank) instead");
  return guard(c, [&] { DISPATCH(c, kernel_timing_impl, c, which, reps, (int)flags, avg_ms, bytes); });
}

int okg_device_alloc(int32_t device, size_t bytes, void** ptr) {
  return guard(nullptr, [&] {
    CK(cudaSetDevice(device));
    CK(cudaMalloc(ptr, bytes));
  });
}
int okg_device_free(void* ptr) {
  return guard(nullptr, [&] { CK(cudaFree(ptr)); });
}
int okg_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return guard(nullptr, [&] { CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); });
}
int okg_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return guard(nullptr, [&] { CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}
int okg_device_synchronize(void) {
  return guard(nullptr, [&] { CK(cudaDeviceSynchronize()); });
}
int64_t okg_kernel_launch_count(void) { return g_launches.load(); }

}  // extern "C"
