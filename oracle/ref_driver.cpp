// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Binds the UNMODIFIED reference library (header-only okflow, included from
// /root/reference/proj/include by the -I path of oracle/Makefile; nothing is
// copied) to the C interface of oracle/okoracle.h, so that the parity tests
// and bench.py's reference arm can call the reference's own code path:
//   build_mesh (mesh.hpp:87), assemble_operators (assembly.hpp:140),
//   make_schur_context (precond.hpp:126), newton_solve (model.hpp:165), ...
// Output: oracle/_ref/libokref.so (git-ignored, travels to the GPU box).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "okflow/assembly.hpp"
#include "okflow/config.hpp"
#include "okflow/vtk.hpp"  // (driver.hpp needs the un-vendored nlohmann json.hpp: not built)
#include "okflow/krylov.hpp"
#include "okflow/mesh.hpp"
#include "okflow/model.hpp"
#include "okflow/multigrid.hpp"
#include "okflow/params.hpp"
#include "okflow/precond.hpp"

#include "okoracle.h"

using namespace okflow;

namespace {

thread_local std::string g_err;

struct RefCtx {
  SolverConfig cfg;
  StructuredMesh mesh;
  OperatorSet ops;
  SchurContext ctx;
  SparseMatrix me;
  bool have_me = false;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return OKO_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return OKO_EINVAL;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return OKO_ENUMERICAL;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return OKO_ECONFIG;
  } catch (const InconsistentState& e) {
    g_err = e.what();
    return OKO_EINCONSISTENT;
  } catch (const CannotCoarsen& e) {
    g_err = e.what();
    return OKO_ECOARSEN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return OKO_EOTHER;
  }
}

SolverConfig to_cfg(const oko_params& p) {
  SolverConfig c;
  c.dim = p.dim;
  c.n = p.n;
  c.eps = p.eps;
  c.sigma = p.sigma;
  c.m = p.m;
  c.theta = p.theta;
  c.dt = p.dt;
  c.newton_tol = p.newton_tol;
  c.newton_maxit = p.newton_maxit;
  c.gmres_tol = p.gmres_tol;
  c.gmres_maxit = p.gmres_maxit;
  c.gmres_restart = p.gmres_restart;
  c.cheby_iters = p.cheby_iters;
  c.richardson_steps = p.richardson_steps;
  c.mg_cycles = p.mg_cycles;
  c.mg_pre = p.mg_pre;
  c.mg_post = p.mg_post;
  c.mg_omega = p.mg_omega;
  c.min_coarse_size = p.min_coarse_size;
  c.cheby_precond = p.cheby_ssor ? "ssor" : "jacobi";
  return c;
}

Vector vec_in(const double* x, long n) { return Vector(x, x + n); }
void vec_out(const Vector& v, double* y) {
  std::memcpy(y, v.data(), v.size() * sizeof(double));
}

}  // namespace

extern "C" {

void oko_default_params(oko_params* p) {
  SolverConfig c;
  p->dim = c.dim;
  p->n = c.n;
  p->eps = c.eps;
  p->sigma = c.sigma;
  p->m = c.m;
  p->theta = c.theta;
  p->dt = c.dt;
  p->newton_tol = c.newton_tol;
  p->newton_maxit = c.newton_maxit;
  p->gmres_tol = c.gmres_tol;
  p->gmres_maxit = c.gmres_maxit;
  p->gmres_restart = c.gmres_restart;
  p->cheby_iters = c.cheby_iters;
  p->richardson_steps = c.richardson_steps;
  p->mg_cycles = c.mg_cycles;
  p->mg_pre = c.mg_pre;
  p->mg_post = c.mg_post;
  p->mg_omega = c.mg_omega;
  p->min_coarse_size = c.min_coarse_size;
  p->shat_perturb = 0.0;
  p->cheby_ssor = c.cheby_precond == "ssor" ? 1 : 0;
}

const char* oko_last_error(void) { return g_err.c_str(); }

void* oko_create(const oko_params* p, int* status) {
  RefCtx* r = nullptr;
  int st = guarded([&] {
    auto rc = std::make_unique<RefCtx>();
    rc->cfg = to_cfg(*p);
    rc->mesh = build_mesh(p->dim, p->n);
    rc->ops = assemble_operators(rc->mesh);
    rc->ops.mesh = &rc->mesh;
    rc->ctx = make_schur_context(rc->mesh, rc->ops.M, rc->ops.K, rc->cfg,
                                 p->shat_perturb);
    r = rc.release();
  });
  if (status) *status = st;
  return r;
}

void oko_destroy(void* ctx) { delete static_cast<RefCtx*>(ctx); }

long oko_num_vertices(void* ctx) {
  return static_cast<RefCtx*>(ctx)->mesh.num_vertices();
}

int oko_levels(void* ctx) {
  return static_cast<RefCtx*>(ctx)->ctx.hierarchy.levels();
}

long oko_level_size(void* ctx, int level) {
  auto* r = static_cast<RefCtx*>(ctx);
  if (level < 0 || level >= r->ctx.hierarchy.levels()) return -1;
  return r->ctx.hierarchy.ops[level].rows();
}

int oko_scalars(void* ctx, double* out) {
  auto* r = static_cast<RefCtx*>(ctx);
  out[0] = r->ctx.c;
  out[1] = r->ctx.sqrt_c;
  out[2] = r->ctx.a_coeff;
  out[3] = r->ctx.dt_theta;
  out[4] = r->ctx.lambda_lo;
  out[5] = r->ctx.lambda_hi;
  out[6] = r->ctx.shat_scale * r->ctx.eps * r->ctx.sqrt_c;
  return OKO_OK;
}

int oko_load_vector(void* ctx, double* b) {
  vec_out(static_cast<RefCtx*>(ctx)->ops.b, b);
  return OKO_OK;
}

int oko_level_dense(void* ctx, int level, double* A) {
  auto* r = static_cast<RefCtx*>(ctx);
  return guarded([&] {
    const SparseMatrix& S = r->ctx.hierarchy.ops.at(level);
    DenseMatrix D = dense_from(S);
    std::memcpy(A, D.data().data(), D.data().size() * sizeof(double));
  });
}

int oko_mesh(int dim, int n, double* vertices, int* cells) {
  return guarded([&] {
    StructuredMesh m = build_mesh(dim, n);
    std::memcpy(vertices, m.vertices.data(), m.vertices.size() * sizeof(double));
    std::memcpy(cells, m.cells.data(), m.cells.size() * sizeof(int));
  });
}

int oko_set_linearization(void* ctx, const double* u) {
  auto* r = static_cast<RefCtx*>(ctx);
  return guarded([&] {
    r->me = assemble_coefficient_mass(r->mesh, vec_in(u, r->mesh.num_vertices()));
    r->ctx.Me = &r->me;
    r->have_me = true;
  });
}

int oko_apply(void* ctx, int kind, int level, const double* x, double* y) {
  auto* r = static_cast<RefCtx*>(ctx);
  const long n = r->mesh.num_vertices();
  const MGHierarchy& h = r->ctx.hierarchy;
  return guarded([&] {
    switch (kind) {
      case OKO_M: vec_out(spmv(r->ops.M, vec_in(x, n)), y); break;
      case OKO_K: vec_out(spmv(r->ops.K, vec_in(x, n)), y); break;
      case OKO_A: vec_out(spmv(*r->ctx.a_mat, vec_in(x, n)), y); break;
      case OKO_SHAT: {
        const SparseMatrix& S = h.ops.at(level);
        vec_out(spmv(S, vec_in(x, S.cols())), y);
        break;
      }
      case OKO_PROLONG: {
        const SparseMatrix& P = h.prolong.at(level);
        vec_out(spmv(P, vec_in(x, P.cols())), y);
        break;
      }
      case OKO_RESTRICT: {
        const SparseMatrix& P = h.prolong.at(level);
        vec_out(spmv_transpose(P, vec_in(x, P.rows())), y);
        break;
      }
      case OKO_VCYCLE:
        vec_out(v_cycle(h, vec_in(x, n), r->ctx.mg_pre, r->ctx.mg_post), y);
        break;
      case OKO_SHAT_INV:
        vec_out(apply_shat_inv(h, vec_in(x, n), r->ctx.mg_cycles, r->ctx.mg_pre,
                               r->ctx.mg_post),
                y);
        break;
      case OKO_CHEB_M: vec_out(apply_M_inv(r->ctx, vec_in(x, n)), y); break;
      case OKO_CHEB_A: vec_out(apply_A_inv(r->ctx, vec_in(x, n)), y); break;
      case OKO_ME:
        if (!r->ctx.Me) throw InconsistentState("Me not set");
        vec_out(spmv(*r->ctx.Me, vec_in(x, n)), y);
        break;
      case OKO_C: vec_out(apply_C(r->ctx, vec_in(x, n)), y); break;
      case OKO_SCHUR: vec_out(apply_schur(r->ctx, vec_in(x, n)), y); break;
      case OKO_SCHUR_TILDE_INV:
        vec_out(apply_schur_tilde_inv(r->ctx, vec_in(x, n)), y);
        break;
      case OKO_S_INV_APPROX:
        vec_out(apply_S_inv_approx(r->ctx, vec_in(x, n)), y);
        break;
      case OKO_BLOCK: vec_out(apply_block(r->ctx, vec_in(x, 2 * n)), y); break;
      case OKO_JACOBIAN: {
        LinearOperator J = jacobian_operator(r->ctx);
        vec_out(J(vec_in(x, 2 * n)), y);
        break;
      }
      case OKO_NONLINEAR:
        vec_out(assemble_nonlinear(r->mesh, vec_in(x, n)), y);
        break;
      case OKO_COARSE_SOLVE: {
        const long nc = h.ops.back().rows();
        vec_out(h.coarse_solver->solve(vec_in(x, nc)), y);
        break;
      }
      case OKO_SSOR_M: {  // SsorSweeps(M, 1).apply_inv (krylov.hpp:372-378)
        const SsorSweeps sw(r->ops.M, 1.0);
        vec_out(sw.apply_inv(vec_in(x, n)), y);
        break;
      }
      default:
        throw std::invalid_argument("oko_apply: unknown kind");
    }
  });
}

int oko_residual(void* ctx, const double* u_next, const double* w_next,
                 const double* u_old, const double* w_old, double* r1,
                 double* r2) {
  auto* r = static_cast<RefCtx*>(ctx);
  const long n = r->mesh.num_vertices();
  return guarded([&] {
    State a, b;
    a.u = vec_in(u_next, n);
    a.w = vec_in(w_next, n);
    b.u = vec_in(u_old, n);
    b.w = vec_in(w_old, n);
    auto res = residual(a, b, r->mesh, r->ops, r->cfg);
    vec_out(res.first, r1);
    vec_out(res.second, r2);
  });
}

int oko_gmres(void* ctx, const double* b, double* x, double rtol, int maxit,
              int restart, int* iterations, double* final_residual,
              int* converged, int* stagnated, double* residual_norms,
              int residual_norms_cap, int* n_residual_norms) {
  auto* r = static_cast<RefCtx*>(ctx);
  const long n = r->mesh.num_vertices();
  return guarded([&] {
    KrylovResult k = gmres(jacobian_operator(r->ctx), block_preconditioner(r->ctx),
                           vec_in(b, 2 * n), rtol, maxit, restart);
    vec_out(k.x, x);
    *iterations = k.iterations;
    *final_residual = k.final_residual;
    *converged = k.converged ? 1 : 0;
    *stagnated = k.stagnated ? 1 : 0;
    int cnt = static_cast<int>(k.residual_norms.size());
    if (n_residual_norms) *n_residual_norms = cnt;
    if (residual_norms)
      for (int i = 0; i < cnt && i < residual_norms_cap; ++i)
        residual_norms[i] = k.residual_norms[i];
  });
}

int oko_newton_solve(void* ctx, const double* u_old, const double* w_old,
                     double* u_next, double* w_next, int* newton_iters,
                     int* gmres_iters, double* residual_norm, double* seconds,
                     int* converged) {
  auto* r = static_cast<RefCtx*>(ctx);
  const long n = r->mesh.num_vertices();
  return guarded([&] {
    State old;
    old.u = vec_in(u_old, n);
    old.w = vec_in(w_old, n);
    auto res = newton_solve(old, r->mesh, r->ops, r->ctx, r->cfg);
    vec_out(res.first.u, u_next);
    vec_out(res.first.w, w_next);
    *newton_iters = res.second.newton_iters;
    for (std::size_t i = 0; i < res.second.gmres_iters.size(); ++i)
      gmres_iters[i] = res.second.gmres_iters[i];
    *residual_norm = res.second.residual_norm;
    *seconds = res.second.seconds;
    *converged = res.second.converged ? 1 : 0;
  });
}

int oko_jacobi_spectrum(void* ctx, double* lo, double* hi) {
  auto* r = static_cast<RefCtx*>(ctx);
  return guarded([&] {
    auto b = estimate_jacobi_spectrum(r->ops.M);
    *lo = b.first;
    *hi = b.second;
  });
}

// counter-based splitmix64 keyed by (seed, global id).
void oko_seeded_ic(long nverts, unsigned long long seed, double m, double* u) {
  for (long g = 0; g < nverts; ++g) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(g) +
                 0x632BE59BD9B4E019ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x = x ^ (x >> 31);
    const double U = 2.0 * (static_cast<double>(x >> 11) * 0x1.0p-53) - 1.0;
    u[g] = m + 0.01 * U;
  }
}

int oko_total_mass(void* ctx, const double* u, double* mass) {
  return guarded([&] {
    auto* c = static_cast<RefCtx*>(ctx);
    *mass = total_mass(c->ops, vec_in(u, c->mesh.num_vertices()));
  });
}

int oko_double_well(void* ctx, const double* u, double* value) {
  return guarded([&] {
    auto* c = static_cast<RefCtx*>(ctx);
    *value = integrate_double_well(c->mesh, vec_in(u, c->mesh.num_vertices()));
  });
}

int oko_energy(void* ctx, const double* u, double* e, int* cg_iters) {
  return guarded([&] {
    auto* c = static_cast<RefCtx*>(ctx);
    *e = energy(c->mesh, c->ops, vec_in(u, c->mesh.num_vertices()), c->cfg);
    if (cg_iters) *cg_iters = -1;  // not exposed by the reference
  });
}

int oko_initial_state(void* ctx, double* u, double* w, int* cg_iters) {
  return guarded([&] {
    auto* c = static_cast<RefCtx*>(ctx);
    const State s = initial_state(c->mesh, c->ops, c->cfg);
    vec_out(s.u, u);
    vec_out(s.w, w);
    if (cg_iters) *cg_iters = -1;
  });
}

int oko_format_g17(double x, char* buf, int len) {
  return guarded([&] {
    const std::string s = format_g17(x);
    std::snprintf(buf, (size_t)len, "%s", s.c_str());
  });
}

int oko_write_vtk(int dim, int n, const double* u, const double* w, const char* path) {
  return guarded([&] {
    const StructuredMesh mesh = build_mesh(dim, n);
    write_vtk(mesh, vec_in(u, mesh.num_vertices()), vec_in(w, mesh.num_vertices()), path);
  });
}

int oko_parse_config(const char* path, char* out, int len) {
  return guarded([&] {
    const RunManifest man = parse_config(path);
    const SolverConfig& c = man.config;
    std::ostringstream os;
    auto d = [&](const char* k, double v) { os << k << '=' << format_g17(v) << '\n'; };
    auto i = [&](const char* k, long v) { os << k << '=' << v << '\n'; };
    d("eps", c.eps); d("sigma", c.sigma); d("m", c.m); d("theta", c.theta); d("dt", c.dt);
    i("n_steps", c.n_steps); i("dim", c.dim); i("n", c.n); d("newton_tol", c.newton_tol);
    i("newton_maxit", c.newton_maxit); d("gmres_tol", c.gmres_tol); i("gmres_maxit", c.gmres_maxit);
    i("gmres_restart", c.gmres_restart); i("cheby_iters", c.cheby_iters);
    os << "cheby_precond=" << c.cheby_precond << '\n';
    i("richardson_steps", c.richardson_steps); i("mg_cycles", c.mg_cycles); i("mg_pre", c.mg_pre);
    i("mg_post", c.mg_post); d("mg_omega", c.mg_omega); i("min_coarse_size", c.min_coarse_size);
    i("threads", c.threads); i("max_dofs", c.max_dofs);
    os << "output_dir=" << c.output_dir << '\n';
    i("snapshot_every", c.snapshot_every);
    os << "mesh_study_n=";
    for (size_t q = 0; q < c.mesh_study_n.size(); ++q) os << (q ? "," : "") << c.mesh_study_n[q];
    os << "\neps_list=";
    for (size_t q = 0; q < c.eps_list.size(); ++q) os << (q ? "," : "") << format_g17(c.eps_list[q]);
    os << '\n';
    std::snprintf(out, (size_t)len, "%s", os.str().c_str());
  });
}

}  // extern "C"
