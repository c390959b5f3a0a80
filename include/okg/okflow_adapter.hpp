// okg/okflow_adapter.hpp -- drop-in adapter for code written against the reference's
// own types (namespace okflow, /root/reference/proj/include/okflow).
//
// A program that runs the reference's Newton path,
//
//     auto ctx = okflow::make_schur_context(mesh, ops.M, ops.K, cfg);          // precond.hpp:126-130
//     auto [next, stats] = okflow::newton_solve(old, mesh, ops, ctx, cfg);     // model.hpp:165-167
//
// moves the solve onto the GPU by including this header and changing the namespace of
// those two calls to okg::  -- the mesh, operator set, config, State and
// IterationStats stay the reference's own types (tests/cpp/test_okflow_adapter.cpp
// runs one time loop both ways and compares them step by step).  The okflow headers
// must be on the include path (the caller already has them); nothing of them is
// copied here.
//
// What the adapter does with the reference's objects:
//   * make_schur_context checks M, K and the mesh the way the reference does
//     (precond.hpp:131-141: square, equal sizes, mesh size, eps > 0, cheby_precond,
//     1 + shat_perturb > 0) and builds the device context from the SolverConfig;
//     the GPU rebuilds M, K, S-hat and the hierarchy matrix-free from the structured
//     mesh, so the CSR matrices themselves are not read (they are the reference's
//     assembly of the same grid, assembly.hpp:82-147).
//   * newton_solve copies State::u/w to the device, runs one timestep of the device
//     Newton solve, and returns the reference's State / IterationStats.  The physical
//     and solver parameters are the ones the context was built with; a SolverConfig
//     that differs from them in a field the solve reads is std::invalid_argument
//     (the reference would mix the two configurations silently).
//   * okg error statuses are rethrown as the reference's exception types
//     (errors.hpp:9-28), so callers' catch clauses keep working.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>

#include "okflow/assembly.hpp"
#include "okflow/errors.hpp"
#include "okflow/mesh.hpp"
#include "okflow/model.hpp"
#include "okflow/params.hpp"
#include "okflow/sparse.hpp"

#include "okflow.hpp"

namespace okg {

namespace adapter_detail {

// okg:: error types -> the reference's (errors.hpp:9-28)
template <class F>
auto translate(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const okg::NumericalError& e) {
    throw okflow::NumericalError(e.what());
  } catch (const okg::ConfigError& e) {
    throw okflow::ConfigError(e.what());
  } catch (const okg::InconsistentState& e) {
    throw okflow::InconsistentState(e.what());
  } catch (const okg::CannotCoarsen& e) {
    throw okflow::CannotCoarsen(e.what());
  }
}

inline okg::SolverConfig from_okflow(const okflow::SolverConfig& c) {
  okg::SolverConfig o;
  o.eps = c.eps;
  o.sigma = c.sigma;
  o.m = c.m;
  o.theta = c.theta;
  o.dt = c.dt;
  o.n_steps = c.n_steps;
  o.dim = c.dim;
  o.n = c.n;
  o.newton_tol = c.newton_tol;
  o.newton_maxit = c.newton_maxit;
  o.gmres_tol = c.gmres_tol;
  o.gmres_maxit = c.gmres_maxit;
  o.gmres_restart = c.gmres_restart;
  o.cheby_iters = c.cheby_iters;
  o.cheby_precond = c.cheby_precond;
  o.richardson_steps = c.richardson_steps;
  o.mg_cycles = c.mg_cycles;
  o.mg_pre = c.mg_pre;
  o.mg_post = c.mg_post;
  o.mg_omega = c.mg_omega;
  o.min_coarse_size = c.min_coarse_size;
  o.threads = c.threads;
  o.max_dofs = c.max_dofs;
  return o;
}

// the fields newton_solve / the preconditioner read (model.hpp:121-215, precond.hpp:126-307)
inline bool same_solve(const okflow::SolverConfig& a, const okg::SolverConfig& b) {
  return a.eps == b.eps && a.sigma == b.sigma && a.m == b.m && a.theta == b.theta && a.dt == b.dt &&
         a.dim == b.dim && a.n == b.n && a.newton_tol == b.newton_tol && a.newton_maxit == b.newton_maxit &&
         a.gmres_tol == b.gmres_tol && a.gmres_maxit == b.gmres_maxit && a.gmres_restart == b.gmres_restart &&
         a.cheby_iters == b.cheby_iters && a.cheby_precond == b.cheby_precond &&
         a.richardson_steps == b.richardson_steps && a.mg_cycles == b.mg_cycles && a.mg_pre == b.mg_pre &&
         a.mg_post == b.mg_post && a.mg_omega == b.mg_omega && a.min_coarse_size == b.min_coarse_size;
}

}  // namespace adapter_detail

// make_schur_context(mesh, M, K, cfg, shat_perturb) (precond.hpp:126-181) on the GPU.
inline SchurContext make_schur_context(const okflow::StructuredMesh& mesh, const okflow::SparseMatrix& M,
                                       const okflow::SparseMatrix& K, const okflow::SolverConfig& cfg,
                                       double shat_perturb = 0.0) {
  if (M.rows() != M.cols() || K.rows() != K.cols() || M.rows() != K.rows())
    throw std::invalid_argument("schur context: M and K must be square and of equal size");
  if (M.rows() != mesh.num_vertices())
    throw std::invalid_argument("schur context: operator size does not match mesh");
  if (!(cfg.eps > 0.0)) throw std::invalid_argument("schur context: eps must be positive");
  if (cfg.cheby_precond != "jacobi" && cfg.cheby_precond != "ssor")
    throw okflow::ConfigError("schur context: cheby_precond must be 'jacobi' or 'ssor'");
  if (!(1.0 + shat_perturb > 0.0))
    throw std::invalid_argument("schur context: perturbation must keep the shifted operator positive");
  okg::SolverConfig c = adapter_detail::from_okflow(cfg);
  // the structured mesh the operators were assembled on (mesh.hpp:87-157)
  c.dim = mesh.dim;
  c.n = mesh.n;
  return adapter_detail::translate([&] { return SchurContext(c, shat_perturb); });
}

// newton_solve(old, mesh, ops, ctx, cfg) (model.hpp:165-215) on the GPU: the
// reference's State in, the reference's State and IterationStats out.
inline std::pair<okflow::State, okflow::IterationStats> newton_solve(const okflow::State& old,
                                                                     const okflow::StructuredMesh& mesh,
                                                                     const okflow::OperatorSet& /*ops*/,
                                                                     SchurContext& ctx,
                                                                     const okflow::SolverConfig& cfg) {
  if (mesh.dim != ctx.config().dim || mesh.n != ctx.config().n)
    throw std::invalid_argument("newton_solve: mesh does not match the context");
  if (!adapter_detail::same_solve(cfg, ctx.config()))
    throw std::invalid_argument("newton_solve: SolverConfig differs from the one the context was built with");
  okg::State o;
  o.u = old.u;
  o.w = old.w;
  o.t = old.t;
  o.step = old.step;
  auto r = adapter_detail::translate([&] { return okg::newton_solve(o, ctx, ctx.config()); });
  okflow::State next;
  next.u = std::move(r.first.u);
  next.w = std::move(r.first.w);
  next.t = r.first.t;
  next.step = r.first.step;
  okflow::IterationStats s;
  s.step = r.second.step;
  s.t = r.second.t;
  s.newton_iters = r.second.newton_iters;
  s.gmres_iters = r.second.gmres_iters;
  s.residual_norm = r.second.residual_norm;
  s.seconds = r.second.seconds;
  s.converged = r.second.converged;
  return {std::move(next), std::move(s)};
}

// residual(next, old, mesh, ops, cfg) (model.hpp:121-148) on the GPU, against a context
// built for the same mesh and configuration.
inline std::pair<okflow::Vector, okflow::Vector> residual(const okflow::State& next, const okflow::State& old,
                                                          const okflow::StructuredMesh& mesh,
                                                          const SchurContext& ctx,
                                                          const okflow::SolverConfig& cfg) {
  if (mesh.dim != ctx.config().dim || mesh.n != ctx.config().n)
    throw std::invalid_argument("residual: mesh does not match the context");
  if (!adapter_detail::same_solve(cfg, ctx.config()))
    throw std::invalid_argument("residual: SolverConfig differs from the one the context was built with");
  okg::State a, b;
  a.u = next.u;
  a.w = next.w;
  b.u = old.u;
  b.w = old.w;
  return adapter_detail::translate([&] { return okg::residual(a, b, ctx); });
}

}  // namespace okg
