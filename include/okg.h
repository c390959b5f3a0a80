/*
 * okg.h -- C ABI of the B200-native Newton linear solver (libokg.so).
 *
 * Drop-in boundary for the reference's Newton-solve path
 * (okflow, /root/reference/proj/include/okflow).  Plain C types only: host or
 * device pointers plus sizes, int64 sizes, negative status codes.  No C++
 * exception crosses this boundary; okg/okflow.hpp maps the codes back onto the
 * reference's exception types (errors.hpp:9-28).
 *
 * Vector convention: an N-vector holds one value per mesh vertex in the
 * reference's global vertex order (x slowest, mesh.hpp:40-44); a stacked
 * 2N-vector is [u-block ; w-block] exactly as precond.hpp:257-298 lays it out.
 *
 * Threading: one okg_ctx per GPU/thread, not re-entrant; every call is
 * synchronous on return (the context's stream is drained).
 */
#ifndef OKG_H
#define OKG_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OKG_ABI_VERSION 1

/* opaque solver context: mesh + operators + SchurContext + Krylov workspace */
typedef struct okg_ctx okg_ctx;

/* ---- status codes: errors.hpp:9-28 + std::invalid_argument -------------- */
enum okg_status {
  OKG_OK = 0,
  OKG_EINVAL = -1,        /* std::invalid_argument                        */
  OKG_ENUMERICAL = -2,    /* okflow::NumericalError                       */
  OKG_ECONFIG = -3,       /* okflow::ConfigError                          */
  OKG_EINCONSISTENT = -4, /* okflow::InconsistentState                    */
  OKG_ECOARSEN = -5,      /* okflow::CannotCoarsen                        */
  OKG_ECUDA = -6,         /* CUDA runtime failure (no reference analogue) */
  OKG_ENOMEM = -7,        /* device allocation failure                    */
  OKG_EOTHER = -9
};

/* ---- okflow::SolverConfig (params.hpp:14-54) + context knobs ---------------- */
typedef struct okg_params {
  int32_t dim;              /* 2 or 3                                   */
  int32_t n;                /* cells per axis                            */
  double eps, sigma, m, theta, dt;
  double newton_tol;
  int32_t newton_maxit;
  double gmres_tol;
  int32_t gmres_maxit;
  int32_t gmres_restart;    /* 0 = full GMRES (krylov.hpp:63)            */
  int32_t cheby_iters;
  int32_t richardson_steps;
  int32_t mg_cycles, mg_pre, mg_post;
  double mg_omega;
  int32_t min_coarse_size;
  double shat_perturb;      /* make_schur_context(..., shat_perturb), precond.hpp:126 */
  int64_t max_dofs;         /* SolverConfig::max_dofs (validate only)    */
  int32_t device;           /* CUDA device ordinal                       */
  int32_t use_graphs;       /* capture the Arnoldi operator in a CUDA graph (default 1) */
  int32_t tiled_min_n;      /* levels with n >= this use the shared-memory tiled stencil
                               kernels; 0 = default (3D: 32, 2D: 128), < 0 = never */
  int32_t tail_max_vertices;/* from the first level (below the finest) with at most this
                               many vertices down to the coarsest, the V-cycle runs as ONE
                               thread-block-cluster kernel (shared-memory resident, 3D
                               n <= 16, 2D n <= 64); 0 = default (3D 1000, 2D 1100),
                               < 0 = never */
  int32_t disable_pdl;      /* 1: launch without programmatic dependent launch */
  int32_t mg_fuse;          /* temporally blocked V(2,2) level kernels (one "down" and one
                               "up" launch per level): 0 = default (2D: levels but the
                               finest with n <= 512; 3D: levels with n <= 16), 1 = every
                               level, 2 = every level but the finest, < 0 = never */
  int32_t nslabs;           /* slab decomposition: split the mesh into this
                               many x-plane slabs, one host thread + CUDA stream each;
                               0/1 = one slab.  Results equal the one-slab solve up to
                               the order of the cross-slab reduction sums. */
  int32_t slab_devices;     /* 0: every slab on `device` (1-GPU emulation); 1: slab r on
                               device `device + r` (peer copies over NVLink) */
  int32_t tail_cluster;     /* CTAs in the tail's cluster (they split the rows of the dense
                               coarse inverse): 0 = default (enough for <= 96 KB each), 1..16 */
  int32_t cheby_ssor;       /* SolverConfig::cheby_precond: 0 = "jacobi", 1 = "ssor" (SSOR
                               sweeps as hyperplane wavefronts, one slab only) */
  int32_t coarse_split;     /* coarsest level above 2000 unknowns (device-factorised inverse):
                               0 = default (each slab multiplies the rows of its own coarse
                               planes, then the planes are all-gathered), < 0 = every slab
                               multiplies all rows */
  int32_t mg_collapse;      /* V(v,v) cycles only: the first coarse level with at most this many
                               vertices, together with every level below it, is replaced at setup
                               by the dense symmetric operator it applies (columns = the V-cycle
                               of that level on unit vectors; packed lower block triangle), so
                               the latency-bound bottom of each V-cycle is one HBM-streaming
                               matvec; 0 = default (3D 1000, 2D 1100: the cluster tail's levels),
                               < 0 = never */
  int64_t rep_max_vertices; /* slab decomposition: levels below the finest with at most this many
                               vertices (in total) are replicated on every slab instead of split --
                               a whole small level is cheaper than a share of it plus a ghost-plane
                               exchange per sweep (cost model in DESIGN.md section 7);
                               0 = default (3,000,000), < 0 = split as deep as 2 planes per slab */
} okg_params;

/* ---- okflow::IterationStats (model.hpp:32-42) -------------------------------- */
#define OKG_MAX_NEWTON 64
typedef struct okg_step_stats {
  int32_t step;
  double t;
  int32_t newton_iters;
  int32_t gmres_iters[OKG_MAX_NEWTON]; /* one per Newton iteration       */
  double residual_norm;                /* final stacked nonlinear residual */
  double seconds;                      /* wall time of newton_solve       */
  int32_t converged;
  int64_t kernel_launches;             /* kernels (incl. graph nodes) launched */
  double mass;                         /* b^T u at the new level (okg_advance) */
  double energy;                       /* energy of the new level (okg_advance with_energy; else NaN) */
} okg_step_stats;

/* ---- okflow::KrylovResult (krylov.hpp:21-28) --------------------------------- */
typedef struct okg_krylov_stats {
  int32_t iterations;
  int32_t converged;
  int32_t stagnated;
  double final_residual;
  int32_t n_residual_norms;
  double residual_norms[512]; /* first 512 recorded norms                 */
} okg_krylov_stats;

/* ---- read-only facts about a context ------------------------------------------ */
typedef struct okg_info {
  int32_t dim, n;
  int64_t num_vertices;       /* N; stacked vectors have 2N entries       */
  int32_t levels;             /* multigrid levels, finest = 0             */
  int64_t level_size[32];
  int32_t level_n[32];
  double c, sqrt_c, a_coeff, dt_theta, lambda_lo, lambda_hi, eps_sqrt_c;
  int64_t device_bytes;       /* device memory held by the context        */
  int32_t graph_nodes;        /* kernels in the captured Arnoldi graph    */
  int32_t tail_start;         /* first level of the cluster tail (-1: none) */
  int32_t tiled_mask;         /* bit l set: level l uses the tiled kernels */
  int32_t nslabs;             /* slabs of the decomposition (1: none)      */
  int32_t rep_level;          /* first level replicated on every slab (levels if none) */
  int32_t slab_ilo[16], slab_ihi[16]; /* owned x-planes [ilo, ihi) of the finest level per slab */
  int32_t tail_cluster;       /* CTAs in the tail's thread-block cluster */
  int32_t coarse_rows;        /* rows of the coarse inverse this slab multiplies */
  int32_t collapse_level;     /* first level applied as one dense operator (-1: none) */
} okg_info;

/* operator kinds for okg_apply (same numbering as the oracle's) */
enum okg_op {
  OKG_OP_M = 0,              /* spmv(M)                         sparse.hpp:138         */
  OKG_OP_K = 1,              /* spmv(K)                                                */
  OKG_OP_A = 2,              /* spmv(a_mat), a_mat=(1+dt*theta*sigma)M  precond.hpp:154 */
  OKG_OP_SHAT = 3,           /* level operator Shat_l            multigrid.hpp:55-66   */
  OKG_OP_PROLONG = 4,        /* P_l : level l+1 -> level l       mesh.hpp:169          */
  OKG_OP_RESTRICT = 5,       /* P_l^T : level l -> level l+1     sparse.hpp:159        */
  OKG_OP_VCYCLE = 6,         /* v_cycle (mg_cycle on `level`)    multigrid.hpp:97-129  */
  OKG_OP_SHAT_INV = 7,       /* apply_shat_inv                   multigrid.hpp:133     */
  OKG_OP_CHEB_M = 8,         /* apply_M_inv                      precond.hpp:185       */
  OKG_OP_CHEB_A = 9,         /* apply_A_inv                      precond.hpp:191       */
  OKG_OP_ME = 10,            /* spmv(Me) at the linearization    assembly.hpp:153      */
  OKG_OP_C = 11,             /* apply_C                          precond.hpp:244       */
  OKG_OP_SCHUR = 12,         /* apply_schur                      precond.hpp:210       */
  OKG_OP_SCHUR_TILDE_INV = 13, /* apply_schur_tilde_inv          precond.hpp:199       */
  OKG_OP_S_INV_APPROX = 14,  /* apply_S_inv_approx               precond.hpp:227       */
  OKG_OP_BLOCK = 15,         /* apply_block  (2N -> 2N)          precond.hpp:257       */
  OKG_OP_JACOBIAN = 16,      /* jacobian_operator (2N -> 2N)     precond.hpp:277       */
  OKG_OP_NONLINEAR = 17,     /* assemble_nonlinear(mesh, x)      assembly.hpp:194      */
  OKG_OP_COARSE_SOLVE = 18,  /* coarsest-level direct solve      dense.hpp:197         */
  OKG_OP_SSOR_M = 19         /* SsorSweeps(M, 1).apply_inv       krylov.hpp:372-378    */
};

/* SolverConfig defaults (params.hpp:29-46) */
int okg_default_params(okg_params* p);
/* SolverConfig::validate (params.hpp:68-116) -> OKG_ECONFIG with message */
int okg_validate_params(const okg_params* p);
/* thread-local message of the last failing call */
int okg_last_error(char* buf, size_t len);

/* build_mesh + assemble_operators + make_schur_context, on `p->device`
 * (replaces mesh.hpp:87, assembly.hpp:140, precond.hpp:126-181) */
int okg_create(const okg_params* p, okg_ctx** ctx);
void okg_destroy(okg_ctx* ctx);
int okg_get_info(okg_ctx* ctx, okg_info* info);

/* ---- one process per GPU ------------------------------------------
 * Rank `rank` of `nranks` processes, each owning the x-plane slab of the mesh the
 * partition below assigns it, on its own GPU `p->device`.  Ghost planes travel by
 * NCCL send/recv between neighbours and the Krylov/Lanczos sums by NCCL allreduce
 * (libnccl.so.2 is loaded at run time).  Rank 0 makes the id with
 * okg_nccl_unique_id; the caller hands it to every rank (e.g. a
 * torch.distributed broadcast).  Host-pointer entry points take full-size arrays
 * and read/write the rank's own planes only; device-pointer ones are refused.
 * nranks = 1 with a null id is an ordinary one-slab context. */
int okg_nccl_unique_id(void* id, size_t len); /* len >= 128 */
int okg_create_rank(const okg_params* p, int32_t rank, int32_t nranks, const void* nccl_id,
                    okg_ctx** ctx);
/* the slab partition (pure host; the same function the contexts use): levels of the
 * hierarchy, first level replicated on every slab, and the owned planes [lo[l], hi[l])
 * of `rank` on every level (all planes on replicated levels); lo/hi hold 32 entries */
int okg_slab_partition(int32_t dim, int32_t n, int32_t min_coarse_size, int32_t nslabs,
                       int32_t rank, int64_t rep_max_vertices /* okg_params' */, int32_t* levels,
                       int32_t* rep_level, int32_t* lo, int32_t* hi);

/* build_mesh arrays, bit-exact (mesh.hpp:87-157); host memory.
 * vertices: N*dim doubles; cells: (2n^2 | 6n^3)*(dim+1) int32 */
int okg_mesh(int32_t dim, int32_t n, double* vertices, int32_t* cells);
/* the builder-defined seeded IC of SURVEY.md 8(d) (host) */
int okg_seeded_ic(int64_t nverts, uint64_t seed, double m, double* u);

/* okflow::State at the old time level (host arrays of N doubles) */
int okg_set_state(okg_ctx* ctx, const double* u, const double* w, double t, int32_t step);
int okg_get_state(okg_ctx* ctx, double* u, double* w, double* t, int32_t* step);
/* newton_solve (model.hpp:165-215) from the current state; on return the
 * context's state is the new time level.  Non-convergence is reported in
 * stats->converged, not as an error (model.hpp:159-164). */
int okg_newton_step(okg_ctx* ctx, okg_step_stats* stats);
/* same, through host buffers: H2D of (u_old, w_old), solve, D2H of (u, w) */
int okg_newton_step_host(okg_ctx* ctx, const double* u_old, const double* w_old,
                         double* u_new, double* w_new, okg_step_stats* stats);

/* ---- diagnostics and initial state -------------------------------
 * u: host array of N doubles, or NULL for the context's current state */
/* total_mass = b^T u (model.hpp:46-48) */
int okg_total_mass(okg_ctx* ctx, const double* u, double* mass);
/* integrate_double_well (assembly.hpp:220-245), closed form of the degree-4 integral */
int okg_double_well(okg_ctx* ctx, const double* u, double* value);
/* energy (model.hpp:56-86): grad + double well + nonlocal term via Jacobi CG on K
 * with the constant nullspace projected out (rtol 1e-10, 2000 iterations);
 * OKG_EINCONSISTENT when the potential rhs is not mean-zero, OKG_ENUMERICAL when
 * the CG does not converge -- exactly the reference's failure modes */
int okg_energy(okg_ctx* ctx, const double* u, double* energy, int32_t* cg_iters);
/* initial_state (model.hpp:93-114): the context's state becomes u0 (cosine bump),
 * w0 (Jacobi CG mass solve, rtol 1e-12), t = 0, step = 0 */
int okg_initial_state(okg_ctx* ctx, int32_t* cg_iters);
/* advance (model.hpp:218-227): okg_newton_step + mass (+ energy) of the new state */
int okg_advance(okg_ctx* ctx, int32_t with_energy, okg_step_stats* stats);

/* ---- per-operator entry points on HOST pointers (any nslabs) ---------------------
 * Same operations as the device-pointer entry points below; the context scatters
 * the inputs over its slabs and gathers the outputs.  With nslabs > 1 okg_apply_host
 * supports the finest-level kinds (every kind except PROLONG, RESTRICT,
 * COARSE_SOLVE and SHAT on a level > 0). */
int okg_linearize_host(okg_ctx* ctx, const double* u);
int okg_apply_host(okg_ctx* ctx, int32_t kind, int32_t level, const double* x, double* y);
int okg_residual_host(okg_ctx* ctx, const double* u_next, const double* w_next,
                      const double* u_old, const double* w_old, double* r1, double* r2);
int okg_gmres_host(okg_ctx* ctx, const double* b, double* x, double rel_tol, int32_t max_iter,
                   int32_t restart, okg_krylov_stats* stats);
/* the same four with the caller's array lengths checked first (OKG_EINVAL on a
 * mismatch, nothing read or written): nx/ny = vertex counts of the kind's input /
 * output (N, 2N for BLOCK/JACOBIAN, a level size for SHAT/VCYCLE/PROLONG/RESTRICT/
 * COARSE_SOLVE), n = N (linearize, residual) or 2N (gmres).  Replaces the reference's
 * dimension checks: LinearOperator::apply (operator.hpp:22-25), gmres
 * (krylov.hpp:48-51), residual (model.hpp:126-127). */
int okg_apply_host_n(okg_ctx* ctx, int32_t kind, int32_t level, const double* x, int64_t nx, double* y,
                     int64_t ny);
int okg_linearize_host_n(okg_ctx* ctx, const double* u, int64_t n);
int okg_residual_host_n(okg_ctx* ctx, const double* u_next, const double* w_next, const double* u_old,
                        const double* w_old, int64_t n, double* r1, double* r2);
int okg_gmres_host_n(okg_ctx* ctx, const double* b, double* x, int64_t n, double rel_tol, int32_t max_iter,
                     int32_t restart, okg_krylov_stats* stats);

/* ---- per-operator entry points on DEVICE pointers (parity + composition) ----
 * single-slab contexts only (OKG_EINVAL when nslabs > 1) */
/* ctx.Me = assemble_coefficient_mass(mesh, u) (model.hpp:184-185); u on device */
int okg_linearize(okg_ctx* ctx, const double* u_dev);
int okg_clear_linearization(okg_ctx* ctx);
int okg_apply(okg_ctx* ctx, int32_t kind, int32_t level, const double* x_dev,
              double* y_dev);
/* residual (model.hpp:121-148) on device arrays */
int okg_residual(okg_ctx* ctx, const double* u_next, const double* w_next,
                 const double* u_old, const double* w_old, double* r1,
                 double* r2);
/* gmres(jacobian_operator, block_preconditioner, b, ...) (krylov.hpp:44) */
int okg_gmres(okg_ctx* ctx, const double* b_dev, double* x_dev, double rel_tol,
              int32_t max_iter, int32_t restart, okg_krylov_stats* stats);
/* estimate_jacobi_spectrum(M) (krylov.hpp:296-320), recomputed on device */
int okg_jacobi_spectrum(okg_ctx* ctx, double* lo, double* hi);

/* ---- measurement hooks (bench.py) ---------------------------------------- */
/* the context's CUDA stream (cudaStream_t) -- for events around a region;
 * with nslabs > 1: slab 0's stream (okg_slab_stream for the others) */
int okg_slab_stream(okg_ctx* ctx, int32_t slab, void** stream);
int okg_stream(okg_ctx* ctx, void** stream);
/* fine-level kernels timed live with CUDA events on the context stream:
 * `which` = OKG_KT_* ; avg_ms = mean launch duration over `reps` launches on
 * the context's buffers ; bytes = algorithmic bytes one launch must move */
enum okg_kernel_id {
  OKG_KT_SMOOTH = 0,     /* damped-Jacobi sweep on Shat_0  (x, b -> y)          */
  OKG_KT_RESID = 1,      /* residual b - Shat_0 x                               */
  OKG_KT_PRE2 = 2,       /* fused two pre-smoothing sweeps from zero (r -> e)   */
  OKG_KT_POST_ACC = 3,   /* last post-smooth fused with x += e                  */
  OKG_KT_CHEB = 4,       /* one Chebyshev step (d, r, x -> d', r', x')          */
  OKG_KT_JACOBIAN = 5,   /* fused block Jacobian apply                          */
  OKG_KT_RESTRICT = 6,   /* P^T on the finest level                             */
  OKG_KT_PROLONG = 7,    /* x += P e_c (tiled levels: fused with the first post-smooth) */
  OKG_KT_COUNT = 8
};
int okg_kernel_timing(okg_ctx* ctx, int32_t which, int32_t reps, double* avg_ms, double* bytes);
/* okg_kernel_timing with flags: OKG_KT_COLD = overwrite a 2 x L2-size scratch
 * buffer before every launch and bracket each launch alone with events (the
 * kernel reads its operands from HBM, as ncu's cold-cache replay does);
 * OKG_KT_NO_PDL = launch without programmatic dependent launch */
enum { OKG_KT_COLD = 1, OKG_KT_NO_PDL = 2 };
int okg_kernel_timing_ex(okg_ctx* ctx, int32_t which, int32_t reps, int32_t flags, double* avg_ms,
                         double* bytes);

/* ---- device memory helpers (so a C/ctypes caller needs no CUDA headers) ---- */
int okg_device_alloc(int32_t device, size_t bytes, void** ptr);
int okg_device_free(void* ptr);
int okg_memcpy_h2d(void* dst_dev, const void* src_host, size_t bytes);
int okg_memcpy_d2h(void* dst_host, const void* src_dev, size_t bytes);
int okg_device_synchronize(void);
/* total kernels this library has launched in this process (graph nodes counted) */
int64_t okg_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
