// okg/okflow.hpp -- C++ host API of the B200 Newton linear solve, mirroring the
// reference okflow interface for this path (same names, argument meaning and
// exceptions), implemented over the C ABI of okg.h (libokg.so).
//
//   reference (namespace okflow)                      here (namespace okg)
//   SolverConfig            params.hpp:14-117          SolverConfig
//   State, IterationStats   model.hpp:25-42            State, IterationStats
//   KrylovResult            krylov.hpp:21-28           KrylovResult
//   LinearOperator          operator.hpp:16-37         LinearOperator (host vectors)
//   make_schur_context      precond.hpp:126-181        make_schur_context -> SchurContext
//   apply_block / jacobian_operator / block_preconditioner   precond.hpp:257-307
//   gmres(jac, prec, b,...) krylov.hpp:44-152          gmres(ctx, b, ...)
//   residual                model.hpp:121-148          residual
//   newton_solve            model.hpp:165-215          newton_solve
//   advance (minus energy)  model.hpp:218-227          advance
//   errors.hpp:9-28 exception types                    same names, thrown from status codes
//
// The mesh and the operators M, K are implicit in the structured grid, so the
// context is built from the SolverConfig alone; everything else keeps the
// reference's signatures up to that.
#pragma once

#include <cmath>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../okg.h"

namespace okg {

using Vector = std::vector<double>;

// ---- errors.hpp:9-28 ----------------------------------------------------------
struct CannotCoarsen : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InconsistentState : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == OKG_OK) return;
  char buf[1024];
  okg_last_error(buf, sizeof buf);
  const std::string msg(buf);
  switch (status) {
    case OKG_EINVAL: throw std::invalid_argument(msg);
    case OKG_ENUMERICAL: throw NumericalError(msg);
    case OKG_ECONFIG: throw ConfigError(msg);
    case OKG_EINCONSISTENT: throw InconsistentState(msg);
    case OKG_ECOARSEN: throw CannotCoarsen(msg);
    case OKG_ENOMEM: throw std::bad_alloc();
    default: throw CudaError(msg);
  }
}

// ---- params.hpp:14-117 ---------------------------------------------------------
struct SolverConfig {
  double eps = 0.02, sigma = 100.0, m = 0.4, theta = 0.5;
  double dt = 4.0e-4;
  int n_steps = 25;
  int dim = 2, n = 64;
  double newton_tol = 1e-8;
  int newton_maxit = 20;
  double gmres_tol = 1e-6;
  int gmres_maxit = 200, gmres_restart = 0;
  int cheby_iters = 10;
  std::string cheby_precond = "jacobi";
  int richardson_steps = 2, mg_cycles = 5, mg_pre = 2, mg_post = 2;
  double mg_omega = 2.0 / 3.0;
  int min_coarse_size = 500;
  int threads = 1;
  long max_dofs = 2000000;
  int device = 0;
  std::vector<int> mesh_study_n = {32, 64, 128};  // study sweeps (driver.hpp:130-205)
  std::vector<double> eps_list = {0.02, 0.01};
  std::string output_dir = ".";
  int snapshot_every = 0;  // VTK snapshots every k steps; 0 = never
  int nslabs = 1;          // x-plane slabs; > 1: one host thread + stream each
  bool slab_devices = false;  // slab r on device `device + r` (else all on `device`)

  long num_vertices() const {
    long s = static_cast<long>(n) + 1, v = s * s;
    return dim == 3 ? v * s : v;
  }
  okg_params to_params(double shat_perturb = 0.0) const {
    okg_params p;
    okg_default_params(&p);
    p.dim = dim;
    p.n = n;
    p.eps = eps;
    p.sigma = sigma;
    p.m = m;
    p.theta = theta;
    p.dt = dt;
    p.newton_tol = newton_tol;
    p.newton_maxit = newton_maxit;
    p.gmres_tol = gmres_tol;
    p.gmres_maxit = gmres_maxit;
    p.gmres_restart = gmres_restart;
    p.cheby_iters = cheby_iters;
    p.richardson_steps = richardson_steps;
    p.mg_cycles = mg_cycles;
    p.mg_pre = mg_pre;
    p.mg_post = mg_post;
    p.mg_omega = mg_omega;
    p.min_coarse_size = min_coarse_size;
    p.max_dofs = max_dofs;
    p.shat_perturb = shat_perturb;
    p.device = device;
    p.nslabs = nslabs;
    p.slab_devices = slab_devices ? 1 : 0;
    p.cheby_ssor = cheby_precond == "ssor" ? 1 : 0;
    return p;
  }
  // SolverConfig::validate (params.hpp:67-116): the first violated constraint, in the
  // reference's order and with its message
  void validate() const {
    auto bad = [](const std::string& m) { throw ConfigError("config: " + m); };
    if (!(eps > 0.0)) bad("eps must be positive");
    if (sigma < 0.0) bad("sigma must be nonnegative");
    if (!(std::abs(m) < 1.0)) bad("mean m must satisfy |m| < 1");
    if (!(theta > 0.0) || theta > 1.0) bad("theta must lie in (0, 1]");
    if (!(dt > 0.0)) bad("dt must be positive");
    if (n_steps < 0) bad("n_steps must be nonnegative");
    if (dim != 2 && dim != 3) bad("dim must be 2 or 3");
    if (n < 1) bad("n must be at least 1");
    if (!(newton_tol > 0.0)) bad("newton_tol must be positive");
    if (newton_maxit < 1) bad("newton_maxit must be at least 1");
    if (!(gmres_tol > 0.0)) bad("gmres_tol must be positive");
    if (gmres_maxit < 1) bad("gmres_maxit must be at least 1");
    if (gmres_restart < 0) bad("gmres_restart must be nonnegative");
    if (cheby_iters < 1) bad("cheby_iters must be at least 1");
    if (cheby_precond != "jacobi" && cheby_precond != "ssor") bad("cheby_precond must be 'jacobi' or 'ssor'");
    if (richardson_steps < 1) bad("richardson_steps must be at least 1");
    if (mg_cycles < 1) bad("mg_cycles must be at least 1");
    if (mg_pre < 0 || mg_post < 0 || mg_pre + mg_post < 1) bad("need at least one smoothing sweep per cycle");
    if (!(mg_omega > 0.0) || !(mg_omega < 2.0)) bad("mg_omega must lie in (0, 2)");
    if (min_coarse_size < 1) bad("min_coarse_size must be at least 1");
    for (int sn : mesh_study_n)
      if (sn < 1) bad("mesh_study_n entries must be >= 1");
    for (double se : eps_list)
      if (!(se > 0.0)) bad("eps_list entries must be positive");
    if (threads < 1) bad("threads must be at least 1");
    if (max_dofs < 1) bad("max_dofs must be at least 1");
    if (snapshot_every < 0) bad("snapshot_every must be nonnegative");
    if (num_vertices() > max_dofs)
      bad("mesh has " + std::to_string(num_vertices()) + " vertices, exceeding max_dofs = " + std::to_string(max_dofs));
  }
};

inline double compute_c(double dt, double theta, double sigma) {  // precond.hpp:31-38
  if (!(dt > 0.0)) throw std::invalid_argument("compute_c: dt must be positive");
  if (!(theta > 0.0) || theta > 1.0) throw std::invalid_argument("compute_c: theta must lie in (0, 1]");
  if (sigma < 0.0) throw std::invalid_argument("compute_c: sigma must be nonnegative");
  return dt * theta / (1.0 + dt * theta * sigma);
}

// ---- model.hpp:25-42, krylov.hpp:21-28 ------------------------------------------
struct State {
  Vector u, w;
  double t = 0.0;
  int step = 0;
};

struct IterationStats {
  int step = 0;
  double t = 0.0;
  int newton_iters = 0;
  std::vector<int> gmres_iters;
  double residual_norm = 0.0;
  double mass = 0.0;
  double energy = NAN;  // energy diagnostic: out of scope on the GPU path
  double seconds = 0.0;
  bool converged = true;
};

struct KrylovResult {
  Vector x;
  int iterations = 0;
  std::vector<double> residual_norms;
  bool converged = false;
  bool stagnated = false;
  double final_residual = 0.0;
};

// RAII device buffer (host-API convenience)
class DeviceVector {
 public:
  DeviceVector(size_t n, int device) : n_(n) { check(okg_device_alloc(device, (n ? n : 1) * sizeof(double), &p_)); }
  DeviceVector(const Vector& v, int device) : DeviceVector(v.size(), device) {
    check(okg_memcpy_h2d(p_, v.data(), v.size() * sizeof(double)));
  }
  ~DeviceVector() {
    if (p_) okg_device_free(p_);
  }
  DeviceVector(const DeviceVector&) = delete;
  DeviceVector& operator=(const DeviceVector&) = delete;
  Vector host() const {
    Vector v(n_);
    check(okg_memcpy_d2h(v.data(), p_, n_ * sizeof(double)));
    return v;
  }
  double* get() const { return static_cast<double*>(p_); }

 private:
  size_t n_;
  void* p_ = nullptr;
};

// ---- precond.hpp:56-181: the context (plus the device workspace) ------------------
class SchurContext {
 public:
  explicit SchurContext(const SolverConfig& cfg, double shat_perturb = 0.0) : cfg_(cfg) {
    const okg_params p = cfg.to_params(shat_perturb);
    check(okg_create(&p, &h_));
    check(okg_get_info(h_, &info_));
  }
  ~SchurContext() {
    if (h_) okg_destroy(h_);
  }
  SchurContext(const SchurContext&) = delete;
  SchurContext& operator=(const SchurContext&) = delete;
  SchurContext(SchurContext&& o) noexcept : cfg_(o.cfg_), h_(o.h_), info_(o.info_), me_set_(o.me_set_) {
    o.h_ = nullptr;
  }

  int rows() const { return static_cast<int>(info_.num_vertices); }
  double c() const { return info_.c; }
  double sqrt_c() const { return info_.sqrt_c; }
  double a_coeff() const { return info_.a_coeff; }
  double dt_theta() const { return info_.dt_theta; }
  double lambda_lo() const { return info_.lambda_lo; }
  double lambda_hi() const { return info_.lambda_hi; }
  int levels() const { return info_.levels; }
  const SolverConfig& config() const { return cfg_; }
  okg_ctx* handle() const { return h_; }
  int device() const { return cfg_.device; }

  // ctx.Me = assemble_coefficient_mass(mesh, u)   (model.hpp:184-185)
  void set_linearization(const Vector& u) {
    if (static_cast<long>(u.size()) != info_.num_vertices) throw std::invalid_argument("linearization: size mismatch");
    check(okg_linearize_host_n(h_, u.data(), static_cast<int64_t>(u.size())));
    me_set_ = true;
  }
  void clear_linearization() {
    check(okg_clear_linearization(h_));
    me_set_ = false;
  }
  // one operator (OKG_OP_*) on host vectors; the output length follows from the kind
  // and level, a wrong input length is std::invalid_argument (operator.hpp:22-25)
  Vector apply(int kind, const Vector& x, int level = 0) const {
    Vector y(out_size(kind, level));
    check(okg_apply_host_n(h_, kind, level, x.data(), static_cast<int64_t>(x.size()), y.data(),
                           static_cast<int64_t>(y.size())));
    return y;
  }
  size_t out_size(int kind, int level = 0) const {
    const int nl = info_.levels;
    auto lvl = [&](int l) -> size_t {
      if (l < 0 || l >= nl) throw std::invalid_argument("level out of range");
      return static_cast<size_t>(info_.level_size[l]);
    };
    switch (kind) {
      case OKG_OP_SHAT: case OKG_OP_VCYCLE: case OKG_OP_PROLONG: return lvl(level);
      case OKG_OP_RESTRICT: return lvl(level + 1);
      case OKG_OP_BLOCK: case OKG_OP_JACOBIAN: return 2 * static_cast<size_t>(info_.num_vertices);
      case OKG_OP_COARSE_SOLVE: return lvl(nl - 1);
      default: return static_cast<size_t>(info_.num_vertices);
    }
  }
  int nslabs() const { return info_.nslabs; }

 private:
  SolverConfig cfg_;
  okg_ctx* h_ = nullptr;
  okg_info info_{};
  bool me_set_ = false;
};

inline SchurContext make_schur_context(const SolverConfig& cfg, double shat_perturb = 0.0) {
  return SchurContext(cfg, shat_perturb);
}

// ---- operator.hpp:16-37 ------------------------------------------------------------
struct LinearOperator {
  int n = 0;
  int n_in = 0;
  std::function<void(const Vector&, Vector&)> apply_fn;
  std::string label;
  void apply(const Vector& x, Vector& y) const {
    if (static_cast<int>(x.size()) != cols())
      throw std::invalid_argument("operator '" + label + "': input dimension mismatch");
    apply_fn(x, y);
  }
  Vector operator()(const Vector& x) const {
    Vector y;
    apply(x, y);
    return y;
  }
  int rows() const { return n; }
  int cols() const { return n_in > 0 ? n_in : n; }
};

// ---- precond.hpp:257-307 -------------------------------------------------------------
inline Vector apply_block(const SchurContext& ctx, const Vector& r) {
  const int n = ctx.rows();
  if (static_cast<int>(r.size()) != 2 * n) throw std::invalid_argument("block preconditioner: stacked size mismatch");
  return ctx.apply(OKG_OP_BLOCK, r);
}

inline LinearOperator jacobian_operator(const SchurContext& ctx) {
  const int n = ctx.rows();
  return {2 * n, 2 * n,
          [&ctx](const Vector& x, Vector& y) { y = ctx.apply(OKG_OP_JACOBIAN, x); },
          "coupled-jacobian"};
}

inline LinearOperator block_preconditioner(const SchurContext& ctx) {
  const int n = ctx.rows();
  return {2 * n, 2 * n, [&ctx](const Vector& r, Vector& y) { y = apply_block(ctx, r); }, "block-triangular"};
}

// gmres(jacobian_operator(ctx), block_preconditioner(ctx), b, ...)  (krylov.hpp:44-152),
// run entirely on the device.  Unlike the reference's gmres, which takes any pair of
// LinearOperators (krylov.hpp:44-46), this one is specialised to the Newton path's
// operator pair -- the coupled Jacobian right-preconditioned by the block-triangular
// preconditioner -- because both live on the device as fused kernels; an arbitrary
// host LinearOperator would need a host round trip per Arnoldi step.  Its arguments
// and KrylovResult fields otherwise mean what the reference's do.
inline KrylovResult gmres(const SchurContext& ctx, const Vector& b, double rel_tol, int max_iter, int restart = 0) {
  const int n = ctx.rows();
  if (static_cast<int>(b.size()) != 2 * n) throw std::invalid_argument("gmres: rhs dimension mismatch");
  okg_krylov_stats ks;
  KrylovResult r;
  r.x.resize(b.size());
  check(okg_gmres_host_n(ctx.handle(), b.data(), r.x.data(), static_cast<int64_t>(b.size()), rel_tol, max_iter,
                         restart, &ks));
  r.iterations = ks.iterations;
  r.converged = ks.converged != 0;
  r.stagnated = ks.stagnated != 0;
  r.final_residual = ks.final_residual;
  for (int i = 0; i < ks.n_residual_norms && i < 512; ++i) r.residual_norms.push_back(ks.residual_norms[i]);
  return r;
}

// ---- model.hpp:121-227 ------------------------------------------------------------------
inline std::pair<Vector, Vector> residual(const State& next, const State& old, const SchurContext& ctx) {
  const size_t n = static_cast<size_t>(ctx.rows());
  if (next.u.size() != old.u.size() || next.w.size() != old.w.size() || next.u.size() != n)
    throw std::invalid_argument("residual: states do not match the mesh");
  Vector r1(n), r2(n);
  check(okg_residual_host_n(ctx.handle(), next.u.data(), next.w.data(), old.u.data(), old.w.data(),
                            static_cast<int64_t>(n), r1.data(), r2.data()));
  return {r1, r2};
}

inline std::pair<State, IterationStats> newton_solve(const State& old, SchurContext& ctx,
                                                     const SolverConfig& /*cfg: ctx holds it*/) {
  const size_t n = static_cast<size_t>(ctx.rows());
  if (old.u.size() != n || old.w.size() != n) throw std::invalid_argument("residual: states do not match the mesh");
  State next;
  next.u.resize(n);
  next.w.resize(n);
  check(okg_set_state(ctx.handle(), old.u.data(), old.w.data(), old.t, old.step));
  okg_step_stats st;
  check(okg_newton_step(ctx.handle(), &st));
  check(okg_get_state(ctx.handle(), next.u.data(), next.w.data(), &next.t, &next.step));
  IterationStats s;
  s.step = st.step;
  s.t = st.t;
  s.newton_iters = st.newton_iters;
  for (int i = 0; i < st.newton_iters && i < OKG_MAX_NEWTON; ++i) s.gmres_iters.push_back(st.gmres_iters[i]);
  s.residual_norm = st.residual_norm;
  s.seconds = st.seconds;
  s.converged = st.converged != 0;
  return {std::move(next), std::move(s)};
}

inline IterationStats from_stats(const okg_step_stats& st) {
  IterationStats s;
  s.step = st.step;
  s.t = st.t;
  s.newton_iters = st.newton_iters;
  for (int i = 0; i < st.newton_iters && i < OKG_MAX_NEWTON; ++i) s.gmres_iters.push_back(st.gmres_iters[i]);
  s.residual_norm = st.residual_norm;
  s.seconds = st.seconds;
  s.converged = st.converged != 0;
  s.mass = st.mass;
  s.energy = st.energy;
  return s;
}

// ---- model.hpp:46-114: diagnostics and initial state on the device -------------------------
inline double total_mass(const SchurContext& ctx, const Vector& u) {  // b^T u
  double m = 0.0;
  check(okg_total_mass(ctx.handle(), u.data(), &m));
  return m;
}
inline double integrate_double_well(const SchurContext& ctx, const Vector& u) {
  double v = 0.0;
  check(okg_double_well(ctx.handle(), u.data(), &v));
  return v;
}
inline double energy(const SchurContext& ctx, const Vector& u, const SolverConfig& /*cfg: ctx holds it*/) {
  if (static_cast<long>(u.size()) != ctx.rows()) throw std::invalid_argument("energy: vector length mismatch");
  double e = 0.0;
  check(okg_energy(ctx.handle(), u.data(), &e, nullptr));
  return e;
}
inline State initial_state(SchurContext& ctx, const SolverConfig& /*cfg*/) {
  check(okg_initial_state(ctx.handle(), nullptr));
  State s;
  s.u.resize(static_cast<size_t>(ctx.rows()));
  s.w.resize(s.u.size());
  check(okg_get_state(ctx.handle(), s.u.data(), s.w.data(), &s.t, &s.step));
  return s;
}

// advance (model.hpp:218-227): newton_solve + mass + energy of the new state
inline std::pair<State, IterationStats> advance(const State& state, SchurContext& ctx, const SolverConfig& cfg) {
  const size_t n = static_cast<size_t>(ctx.rows());
  if (state.u.size() != n || state.w.size() != n) throw std::invalid_argument("residual: states do not match the mesh");
  (void)cfg;
  check(okg_set_state(ctx.handle(), state.u.data(), state.w.data(), state.t, state.step));
  okg_step_stats st;
  check(okg_advance(ctx.handle(), 1, &st));
  State next;
  next.u.resize(n);
  next.w.resize(n);
  check(okg_get_state(ctx.handle(), next.u.data(), next.w.data(), &next.t, &next.step));
  return {std::move(next), from_stats(st)};
}

// run_simulation (model.hpp:243-279), device-resident between steps; the state is
// copied to the host only for the on_state observer
struct SimulationResult {
  std::vector<IterationStats> stats;
  State final_state;
};

inline SimulationResult run_simulation(const SolverConfig& cfg, const std::function<void(const State&)>& on_state = {},
                                       double shat_perturb = 0.0,
                                       const std::function<void(const IterationStats&)>& on_stats = {}) {
  cfg.validate();
  SchurContext ctx = make_schur_context(cfg, shat_perturb);
  SimulationResult result;
  State state = initial_state(ctx, cfg);
  IterationStats init;
  init.mass = total_mass(ctx, state.u);
  init.energy = energy(ctx, state.u, cfg);
  result.stats.push_back(init);
  if (on_stats) on_stats(init);
  if (on_state) on_state(state);
  for (int k = 0; k < cfg.n_steps; ++k) {
    okg_step_stats st;
    check(okg_advance(ctx.handle(), 1, &st));
    const IterationStats s = from_stats(st);
    result.stats.push_back(s);
    if (on_stats) on_stats(s);
    if (!s.converged)
      throw NumericalError("run_simulation: nonlinear solve failed at step " + std::to_string(s.step) +
                           " (residual " + std::to_string(s.residual_norm) + ")");
    if (on_state) {
      state.u.resize(static_cast<size_t>(ctx.rows()));
      state.w.resize(state.u.size());
      check(okg_get_state(ctx.handle(), state.u.data(), state.w.data(), &state.t, &state.step));
      on_state(state);
    }
  }
  result.final_state.u.resize(static_cast<size_t>(ctx.rows()));
  result.final_state.w.resize(result.final_state.u.size());
  check(okg_get_state(ctx.handle(), result.final_state.u.data(), result.final_state.w.data(), &result.final_state.t,
                      &result.final_state.step));
  return result;
}

}  // namespace okg
