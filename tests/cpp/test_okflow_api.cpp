// C++ host-API checks written like the reference's own suites (test_model.cpp,
// test_precond.cpp): drives libokg through include/okg/okflow.hpp on a GPU.
// Exit code 0 iff every check passes.  Built by __graft_entry__.build(),
// run by tests/test_cpp_api.py (marked gpu).
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "okg/okflow.hpp"

static int failures = 0;
#define REQUIRE(cond)                                                  \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  using namespace okg;
  // schur scale factor KATs (test_precond.cpp:103-117)
  REQUIRE(std::abs(compute_c(0.0004, 0.5, 100.0) - 0.00019607843137254902) <= 1e-15 * 2e-4);
  REQUIRE(compute_c(1.0, 0.5, 0.0) == 0.5);
  REQUIRE(throws<std::invalid_argument>([] { compute_c(0.0, 0.5, 100.0); }));
  // config validation (params.hpp:68-116)
  SolverConfig bad;
  bad.mg_omega = 2.0;
  REQUIRE(throws<ConfigError>([&] { bad.validate(); }));

  // constant steady pair is a fixed point with zero Newton cost (test_model.cpp:86-109)
  SolverConfig cfg;
  cfg.dim = 2;
  cfg.n = 8;
  {
    SchurContext ctx = make_schur_context(cfg);
    const size_t n = static_cast<size_t>(ctx.rows());
    State steady{Vector(n, cfg.m), Vector(n, cfg.m * cfg.m * cfg.m - cfg.m), 0.0, 0};
    auto res = newton_solve(steady, ctx, cfg);
    REQUIRE(res.second.converged);
    REQUIRE(res.second.newton_iters == 0);
    REQUIRE(res.second.gmres_iters.empty());
    REQUIRE(res.first.step == 1 && res.first.t == cfg.dt);
    // the constraint block needs a linearization (precond.hpp:245-247)
    REQUIRE(throws<InconsistentState>([&] { jacobian_operator(ctx)(Vector(2 * n, 0.0)); }));
  }
  // one implicit step: convergence, bookkeeping (test_model.cpp:197-223)
  cfg.n = 32;
  {
    SchurContext ctx = make_schur_context(cfg);
    const size_t n = static_cast<size_t>(ctx.rows());
    // advance computes the energy, which needs a mean-consistent field (model.hpp:68-73)
    State bad{Vector(n), Vector(n, 0.0), 0.0, 0};
    for (size_t i = 0; i < n; ++i) bad.u[i] = cfg.m + 0.01 * std::sin(0.37 * static_cast<double>(i));
    REQUIRE(throws<InconsistentState>([&] { advance(bad, ctx, cfg); }));
    const State s0 = initial_state(ctx, cfg);  // model.hpp:93-114
    REQUIRE(s0.step == 0 && s0.t == 0.0 && s0.u.size() == n);
    REQUIRE(std::abs(total_mass(ctx, s0.u) - cfg.m) <= 1e-13);
    auto res = advance(s0, ctx, cfg);
    REQUIRE(std::abs(res.second.mass - cfg.m) <= 1e-13);  // mass is conserved
    REQUIRE(std::isfinite(res.second.energy) && res.second.energy <= energy(ctx, s0.u, cfg) + 1e-12);
    REQUIRE(res.second.converged);
    REQUIRE(res.second.newton_iters >= 1 && res.second.newton_iters <= 8);
    REQUIRE(res.second.gmres_iters.size() == static_cast<size_t>(res.second.newton_iters));
    for (int it : res.second.gmres_iters) REQUIRE(it >= 1 && it <= 30);
    REQUIRE(res.second.seconds > 0.0);
    // residual of the accepted step is below the Newton tolerance
    auto r = residual(res.first, s0, ctx);
    double nn = 0.0;
    for (double v : r.first) nn += v * v;
    for (double v : r.second) nn += v * v;
    REQUIRE(std::sqrt(nn) <= 1e-8);
    // block preconditioner is linear (test_precond.cpp:452-499)
    ctx.set_linearization(res.first.u);
    Vector a(2 * n), b(2 * n), ab(2 * n);
    for (size_t i = 0; i < 2 * n; ++i) {
      a[i] = std::cos(0.1 * static_cast<double>(i));
      b[i] = std::sin(0.2 * static_cast<double>(i));
      ab[i] = 2.0 * a[i] - 3.0 * b[i];
    }
    const Vector pa = apply_block(ctx, a), pb = apply_block(ctx, b), pab = apply_block(ctx, ab);
    double d = 0.0, s = 0.0;
    for (size_t i = 0; i < 2 * n; ++i) {
      d += std::pow(pab[i] - (2.0 * pa[i] - 3.0 * pb[i]), 2);
      s += pab[i] * pab[i];
    }
    REQUIRE(std::sqrt(d) <= 1e-12 * std::sqrt(s));
    // gmres with the built-in operator pair reaches its tolerance (krylov.hpp:44-152)
    KrylovResult k = gmres(ctx, a, 1e-10, 200, 30);
    REQUIRE(k.converged && k.iterations >= 1 && k.iterations <= 30);
    REQUIRE(throws<std::invalid_argument>([&] { apply_block(ctx, Vector(n, 0.0)); }));
  }
  // odd grid: the coarsest level is too large for the direct solve (test_multigrid.cpp:196-202)
  cfg.n = 45;
  REQUIRE(throws<ConfigError>([&] { SchurContext ctx(cfg); }));
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "all C++ host-API checks passed", failures);
  return failures ? 1 : 0;
}
