/*
 * okoracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * One C interface implemented twice:
 *   oracle/ref_driver.cpp  -> oracle/_ref/libokref.so   (the reference okflow headers
 *                             compiled from /root/reference, untouched)
 *   oracle/okport.c        -> oracle/libokport.so       (plain-C restatement of the
 *                             reference algorithm, each function citing file:line)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load these libraries.  The product path
 * (paper_1603_04570_b200/libokg.so) never links or calls them.
 *
 * All vectors are host arrays in the reference's global vertex order
 * (x slowest, /root/reference/proj/include/okflow/mesh.hpp:40-44).
 */
#ifndef OKORACLE_H
#define OKORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct oko_params {
  int dim;
  int n;
  double eps, sigma, m, theta, dt;
  double newton_tol;
  int newton_maxit;
  double gmres_tol;
  int gmres_maxit;
  int gmres_restart;
  int cheby_iters;
  int richardson_steps;
  int mg_cycles;
  int mg_pre;
  int mg_post;
  double mg_omega;
  int min_coarse_size;
  double shat_perturb;
  int cheby_ssor; /* cheby_precond: 0 = "jacobi", 1 = "ssor" (krylov.hpp:322-418) */
} oko_params;

/* operator kinds for oko_apply (level only used by SHAT/PROLONG/RESTRICT) */
enum {
  OKO_M = 0,            /* spmv(M)                         sparse.hpp:138 */
  OKO_K = 1,            /* spmv(K)                                        */
  OKO_A = 2,            /* spmv(a_mat) = (1+dt*theta*sigma) M  precond.hpp:154 */
  OKO_SHAT = 3,         /* spmv(hierarchy.ops[level])      multigrid.hpp:55-66 */
  OKO_PROLONG = 4,      /* spmv(prolong[level])  coarse(level+1) -> fine(level) */
  OKO_RESTRICT = 5,     /* spmv_transpose(prolong[level]) fine -> coarse  */
  OKO_VCYCLE = 6,       /* v_cycle(h, b, pre, post)        multigrid.hpp:124 */
  OKO_SHAT_INV = 7,     /* apply_shat_inv(h, b, cycles)    multigrid.hpp:133 */
  OKO_CHEB_M = 8,       /* apply_M_inv                     precond.hpp:185 */
  OKO_CHEB_A = 9,       /* apply_A_inv                     precond.hpp:191 */
  OKO_ME = 10,          /* spmv(Me)  (needs oko_set_linearization)        */
  OKO_C = 11,           /* apply_C                         precond.hpp:244 */
  OKO_SCHUR = 12,       /* apply_schur                     precond.hpp:210 */
  OKO_SCHUR_TILDE_INV = 13, /* apply_schur_tilde_inv         precond.hpp:199 */
  OKO_S_INV_APPROX = 14,/* apply_S_inv_approx              precond.hpp:227 */
  OKO_BLOCK = 15,       /* apply_block (2N -> 2N)          precond.hpp:257 */
  OKO_JACOBIAN = 16,    /* jacobian_operator (2N -> 2N)    precond.hpp:277 */
  OKO_NONLINEAR = 17,   /* assemble_nonlinear(mesh, x)     assembly.hpp:194 */
  OKO_COARSE_SOLVE = 18, /* coarse_solver->solve (coarsest level)         */
  OKO_SSOR_M = 19        /* SsorSweeps(M, 1).apply_inv  krylov.hpp:372-378 */
};

/* status codes (negative) mirror the reference exception types, errors.hpp:9-28 */
enum {
  OKO_OK = 0,
  OKO_EINVAL = -1,        /* std::invalid_argument */
  OKO_ENUMERICAL = -2,    /* NumericalError */
  OKO_ECONFIG = -3,       /* ConfigError */
  OKO_EINCONSISTENT = -4, /* InconsistentState */
  OKO_ECOARSEN = -5,      /* CannotCoarsen */
  OKO_EOTHER = -9
};

/* fills the reference SolverConfig defaults (params.hpp:14-54) */
void oko_default_params(oko_params* p);
/* context = build_mesh + assemble_operators + make_schur_context */
void* oko_create(const oko_params* p, int* status);
void oko_destroy(void* ctx);
const char* oko_last_error(void);

long oko_num_vertices(void* ctx);
int oko_levels(void* ctx);
long oko_level_size(void* ctx, int level);
/* out[0..6] = c, sqrt_c, a_coeff, dt_theta, lambda_lo, lambda_hi, eps*sqrt_c*shat_scale */
int oko_scalars(void* ctx, double* out);
/* load vector b (assembly.hpp:130) */
int oko_load_vector(void* ctx, double* b);
/* dense copy of hierarchy.ops[level] (row-major, level_size^2) */
int oko_level_dense(void* ctx, int level, double* A);

/* mesh arrays exactly as build_mesh produces them (mesh.hpp:87-157) */
int oko_mesh(int dim, int n, double* vertices, int* cells);

/* ctx.Me = assemble_coefficient_mass(mesh, u) (model.hpp:184-185) */
int oko_set_linearization(void* ctx, const double* u);
int oko_apply(void* ctx, int kind, int level, const double* x, double* y);
int oko_residual(void* ctx, const double* u_next, const double* w_next,
                 const double* u_old, const double* w_old, double* r1,
                 double* r2);
/* gmres(jacobian_operator, block_preconditioner, b, ...) krylov.hpp:44 */
int oko_gmres(void* ctx, const double* b, double* x, double rtol, int maxit,
              int restart, int* iterations, double* final_residual,
              int* converged, int* stagnated, double* residual_norms,
              int residual_norms_cap, int* n_residual_norms);
/* newton_solve (model.hpp:165-215); gmres_iters has room for newton_maxit */
int oko_newton_solve(void* ctx, const double* u_old, const double* w_old,
                     double* u_next, double* w_next, int* newton_iters,
                     int* gmres_iters, double* residual_norm, double* seconds,
                     int* converged);
/* Lanczos bounds on diag(M)^-1 M (krylov.hpp:296-320), standalone */
int oko_jacobi_spectrum(void* ctx, double* lo, double* hi);

/* ---- diagnostics and initial state ---- */
/* total_mass = b^T u (model.hpp:46-48) */
int oko_total_mass(void* ctx, const double* u, double* mass);
/* integrate_double_well (assembly.hpp:220-245), degree-4 rule, Kahan sum */
int oko_double_well(void* ctx, const double* u, double* value);
/* energy (model.hpp:56-86); cg_iters = iterations of the potential solve
 * (-1 when the implementation does not report them, 0 when sigma == 0) */
int oko_energy(void* ctx, const double* u, double* energy, int* cg_iters);
/* initial_state (model.hpp:93-114): u0 (cosine bump), w0 (mass solve) */
int oko_initial_state(void* ctx, double* u, double* w, int* cg_iters);

/* ---- output formats; the compiled reference only ---- */
/* format_g17 (vtk.hpp:17-22) into buf (NUL-terminated) */
int oko_format_g17(double x, char* buf, int len);
/* write_vtk (vtk.hpp:28-66) of a dim/n mesh */
int oko_write_vtk(int dim, int n, const double* u, const double* w, const char* path);

/* parse_config (config.hpp:114-236): dump of the parsed SolverConfig, key=value per line */
int oko_parse_config(const char* path, char* out, int len);

/* builder-defined seeded IC, SURVEY.md section 8(d) (counter-based splitmix64) */
void oko_seeded_ic(long nverts, unsigned long long seed, double m, double* u);

#ifdef __cplusplus
}
#endif
#endif
