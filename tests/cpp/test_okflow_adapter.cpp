// The drop-in check for code written against the reference's own types: ONE time
// loop over the reference's API (okflow::build_mesh, assemble_operators,
// make_schur_context, newton_solve -- model.hpp:165-215, precond.hpp:126-130) is
// instantiated twice, once with namespace okflow (the reference, compiled from its
// headers) and once with namespace okg (include/okg/okflow_adapter.hpp: the GPU),
// and the two runs are compared step by step: Newton / GMRES counts (+-1), fields
// (<= 1e-8 relative l2), t / step bookkeeping.
//
// Built by __graft_entry__.build() where the reference headers are present
// (-I/root/reference/proj/include; they are not copied); the binary runs on the GPU
// box (tests/test_cpp_api.py, marked gpu).  Exit code 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "okflow/assembly.hpp"
#include "okflow/mesh.hpp"
#include "okflow/model.hpp"
#include "okflow/params.hpp"
#include "okflow/precond.hpp"

#include "okg/okflow_adapter.hpp"

static int failures = 0;
#define REQUIRE(cond)                                                        \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                            \
    }                                                                        \
  } while (0)

// The caller's time loop, written once.  NS is the only thing that changes.
#define TIME_LOOP(NS, cfg, u0, steps, states, stats)                                   \
  do {                                                                                 \
    okflow::StructuredMesh mesh = okflow::build_mesh(cfg.dim, cfg.n);                  \
    okflow::OperatorSet ops = okflow::assemble_operators(mesh);                        \
    auto ctx = NS::make_schur_context(mesh, ops.M, ops.K, cfg);                        \
    okflow::State s{u0, okflow::Vector(u0.size(), 0.0), 0.0, 0};                      \
    for (int k = 0; k < steps; ++k) {                                                  \
      auto r = NS::newton_solve(s, mesh, ops, ctx, cfg);                               \
      s = std::move(r.first);                                                          \
      states.push_back(s);                                                             \
      stats.push_back(r.second);                                                       \
    }                                                                                  \
  } while (0)

static double relerr(const okflow::Vector& a, const okflow::Vector& b) {
  double d = 0.0, nb = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    nb += b[i] * b[i];
  }
  return std::sqrt(d) / (nb > 0 ? std::sqrt(nb) : 1.0);
}

static void run_case(int dim, int n, double m, unsigned long long seed, int steps) {
  okflow::SolverConfig cfg;  // BASELINE.json settings
  cfg.dim = dim;
  cfg.n = n;
  cfg.eps = 0.02;
  cfg.sigma = 100.0;
  cfg.m = m;
  cfg.theta = 0.5;
  cfg.dt = cfg.eps * cfg.eps;
  cfg.newton_tol = 1e-8;
  cfg.gmres_tol = 1e-10;
  cfg.gmres_restart = 30;
  const long N = cfg.num_vertices();
  okflow::Vector u0(static_cast<size_t>(N));
  okg::check(okg_seeded_ic(N, seed, m, u0.data()));  // SURVEY 8(d) seeded IC

  std::vector<okflow::State> ref_states, gpu_states;
  std::vector<okflow::IterationStats> ref_stats, gpu_stats;
  TIME_LOOP(okflow, cfg, u0, steps, ref_states, ref_stats);
  TIME_LOOP(okg, cfg, u0, steps, gpu_states, gpu_stats);

  for (int k = 0; k < steps; ++k) {
    const auto &a = ref_stats[k], &b = gpu_stats[k];
    REQUIRE(a.converged == b.converged);
    REQUIRE(a.newton_iters == b.newton_iters);
    REQUIRE(a.gmres_iters.size() == b.gmres_iters.size());
    for (size_t i = 0; i < a.gmres_iters.size() && i < b.gmres_iters.size(); ++i)
      REQUIRE(std::abs(a.gmres_iters[i] - b.gmres_iters[i]) <= 1);
    REQUIRE(a.step == b.step && a.t == b.t);
    REQUIRE(ref_states[k].step == gpu_states[k].step && ref_states[k].t == gpu_states[k].t);
    const double eu = relerr(gpu_states[k].u, ref_states[k].u), ew = relerr(gpu_states[k].w, ref_states[k].w);
    REQUIRE(eu <= 1e-8 && ew <= 1e-8);
    std::printf("%dD n=%d step %d: newton %d/%d gmres %d/%d  rel l2 u %.2e w %.2e  (reference %.3f s, gpu %.4f s)\n",
                dim, n, k + 1, a.newton_iters, b.newton_iters, a.gmres_iters.empty() ? -1 : a.gmres_iters[0],
                b.gmres_iters.empty() ? -1 : b.gmres_iters[0], eu, ew, a.seconds, b.seconds);
  }
}

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
  run_case(2, 64, 0.0, 0, 3);   // BASELINE configs[0] (+2 more steps)
  run_case(2, 128, 0.1, 1, 2);
  run_case(3, 16, 0.0, 2, 2);

  // the reference's argument checks and exception types survive the swap
  okflow::SolverConfig cfg;
  cfg.dim = 2;
  cfg.n = 16;
  okflow::StructuredMesh mesh = okflow::build_mesh(2, 16);
  okflow::OperatorSet ops = okflow::assemble_operators(mesh);
  okflow::StructuredMesh other = okflow::build_mesh(2, 8);
  REQUIRE(throws<std::invalid_argument>([&] { okg::make_schur_context(other, ops.M, ops.K, cfg); }));
  REQUIRE(throws<std::invalid_argument>([&] { okg::make_schur_context(mesh, ops.M, ops.K, cfg, -1.0); }));
  okflow::SolverConfig bad = cfg;
  bad.cheby_precond = "ilu";
  REQUIRE(throws<okflow::ConfigError>([&] { okg::make_schur_context(mesh, ops.M, ops.K, bad); }));
  auto ctx = okg::make_schur_context(mesh, ops.M, ops.K, cfg);
  okflow::State s{okflow::Vector(mesh.num_vertices(), cfg.m), okflow::Vector(mesh.num_vertices(), 0.0), 0.0, 0};
  okflow::SolverConfig cfg2 = cfg;
  cfg2.dt *= 2.0;
  REQUIRE(throws<std::invalid_argument>([&] { okg::newton_solve(s, mesh, ops, ctx, cfg2); }));
  okflow::State shortstate{okflow::Vector(3, 0.0), okflow::Vector(3, 0.0), 0.0, 0};
  REQUIRE(throws<std::invalid_argument>([&] { okg::newton_solve(shortstate, mesh, ops, ctx, cfg); }));
  // residual through the adapter equals the reference's (model.hpp:121-148)
  okflow::State nx = s;
  for (size_t i = 0; i < nx.u.size(); ++i) nx.u[i] += 1e-3 * std::sin(0.1 * static_cast<double>(i));
  auto rr = okflow::residual(nx, s, mesh, ops, cfg);
  auto rg = okg::residual(nx, s, mesh, ctx, cfg);
  REQUIRE(relerr(rg.first, rr.first) <= 1e-12 && relerr(rg.second, rr.second) <= 1e-12);

  if (failures) {
    std::printf("%d adapter checks FAILED\n", failures);
    return 1;
  }
  std::printf("all okflow-adapter checks passed\n");
  return 0;
}
