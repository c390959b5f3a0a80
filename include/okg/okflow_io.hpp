// okg/okflow_io.hpp -- output formats of the reference over the
// B200 solver: locale-independent %.17g numbers, legacy-VTK STRUCTURED_POINTS
// snapshots and the streamed stats.csv of `cmd_run`.
//
//   reference (namespace okflow)            here (namespace okg)
//   format_g17           vtk.hpp:17-22      format_g17
//   write_vtk            vtk.hpp:28-66      write_vtk (same bytes)
//   cmd_run              driver.hpp:79-125  cmd_run (device-resident run; snapshots are
//                                           formatted and written by a background thread
//                                           while the GPU computes the next steps)
#pragma once

#include <filesystem>
#include <fstream>
#include <future>
#include <iomanip>
#include <iostream>
#include <locale>
#include <numeric>
#include <sstream>
#include <string>

#include "okflow.hpp"

namespace okg {

// classic-"C" decimal point, 17 significant digits, shortest form ("0", "0.5")
inline std::string format_g17(double x) {
  std::ostringstream os;
  os.imbue(std::locale::classic());
  os << std::setprecision(17) << x;
  return os.str();
}

// nodal fields u and w as ASCII STRUCTURED_POINTS, point data in the format's
// native order (x fastest, z slowest) -- the reference's grid index is x slowest
inline void write_vtk(int dim, int n, const Vector& u, const Vector& w, const std::string& path) {
  const long s = n + 1;
  const long nv = dim == 3 ? s * s * s : s * s;
  if (static_cast<long>(u.size()) != nv || static_cast<long>(w.size()) != nv)
    throw InconsistentState("write_vtk: field size does not match mesh");
  std::ostringstream os;
  os.imbue(std::locale::classic());
  os << "# vtk DataFile Version 3.0\n";
  os << "okflow state\n";
  os << "ASCII\n";
  os << "DATASET STRUCTURED_POINTS\n";
  os << "DIMENSIONS " << s << " " << s << " " << (dim == 3 ? s : 1) << "\n";
  os << "ORIGIN 0 0 0\n";
  const std::string h = format_g17(1.0 / n);
  os << "SPACING " << h << " " << h << " " << h << "\n";
  os << "POINT_DATA " << nv << "\n";
  auto emit = [&](const char* name, const Vector& f) {
    os << "SCALARS " << name << " double 1\n";
    os << "LOOKUP_TABLE default\n";
    const long nz = dim == 3 ? s : 1;
    for (long k = 0; k < nz; ++k)
      for (long j = 0; j < s; ++j)
        for (long i = 0; i < s; ++i) {
          const long g = dim == 2 ? i * s + j : (i * s + j) * s + k;  // mesh.hpp:40-44
          os << format_g17(f[static_cast<size_t>(g)]) << "\n";
        }
  };
  emit("u", u);
  emit("w", w);
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("write_vtk: cannot open " + path);
  out << os.str();
  if (!out) throw std::runtime_error("write_vtk: write failed for " + path);
}

inline std::string format_short(double x) {
  std::ostringstream os;
  os.imbue(std::locale::classic());
  os << std::setprecision(4) << x;
  return os.str();
}

// cmd_run (driver.hpp:79-125): stats.csv streamed row by row (flushed, so a failed
// step leaves the completed rows), VTK snapshots of the initial state and every
// `snapshot_every` steps; returns 1 on a failed nonlinear solve, like the reference
inline int cmd_run(const SolverConfig& cfg, const std::string& output_dir = ".", int snapshot_every = 0,
                   double shat_perturb = 0.0) {
  const std::filesystem::path dir = output_dir.empty() ? std::filesystem::path(".") : std::filesystem::path(output_dir);
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  if (ec) throw ConfigError("output: cannot create directory '" + dir.string() + "': " + ec.message());
  std::ofstream csv(dir / "stats.csv", std::ios::binary);
  if (!csv) throw std::runtime_error("run: cannot open " + (dir / "stats.csv").string());
  csv << "step,newton_iters,total_gmres,avg_gmres,residual,mass,energy,seconds\n";
  csv.flush();
  long tot_newton = 0, tot_gmres = 0;
  const auto on_stats = [&](const IterationStats& st) {
    if (st.step == 0) return;
    const int total = std::accumulate(st.gmres_iters.begin(), st.gmres_iters.end(), 0);
    const double avg = st.newton_iters > 0 ? static_cast<double>(total) / static_cast<double>(st.newton_iters) : 0.0;
    csv << st.step << ',' << st.newton_iters << ',' << total << ',' << format_g17(avg) << ','
        << format_g17(st.residual_norm) << ',' << format_g17(st.mass) << ',' << format_g17(st.energy) << ','
        << format_g17(st.seconds) << "\n";
    csv.flush();
    tot_newton += st.newton_iters;
    tot_gmres += total;
  };
  std::future<void> pending;  // one snapshot in flight: formatting overlaps the next steps
  const auto on_state = [&](const State& s) {
    const bool due = s.step == 0 || (snapshot_every > 0 && s.step % snapshot_every == 0);
    if (!due) return;
    if (pending.valid()) pending.get();
    const std::string path = (dir / ("state_" + std::to_string(s.step) + ".vtk")).string();
    pending = std::async(std::launch::async, [dim = cfg.dim, n = cfg.n, u = s.u, w = s.w, path] {
      write_vtk(dim, n, u, w, path);
    });
  };
  try {
    run_simulation(cfg, on_state, shat_perturb, on_stats);
  } catch (const NumericalError& e) {
    if (pending.valid()) pending.get();
    std::cerr << "run: " << e.what() << "\n";
    return 1;
  }
  if (pending.valid()) pending.get();
  const double avg = tot_newton > 0 ? static_cast<double>(tot_gmres) / static_cast<double>(tot_newton) : 0.0;
  std::cout << "run: " << cfg.n_steps << " steps, " << cfg.dim << "D n=" << cfg.n
            << ", avg GMRES per Newton = " << format_short(avg) << "\n";
  return 0;
}

}  // namespace okg
