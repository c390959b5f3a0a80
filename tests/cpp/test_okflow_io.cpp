// test_okflow_io.cpp -- the C++ output formats (include/okg/okflow_io.hpp):
//   test_okflow_io fmt IN.bin            one format_g17 line per double
//   test_okflow_io vtk DIM N IN.bin OUT  write_vtk of u, w = the halves of IN.bin
//   test_okflow_io run DIM N STEPS EVERY OUTDIR   cmd_run on the GPU
//   test_okflow_io cfg PATH              parse_config dump (as oracle/_ref/okref_io cfg)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <vector>

#include "okg/okflow_cli.hpp"

static std::vector<double> read_all(const char* path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  const std::streamsize bytes = f.tellg();
  std::vector<double> d(static_cast<size_t>(bytes / 8));
  f.seekg(0);
  f.read(reinterpret_cast<char*>(d.data()), bytes);
  return d;
}

int main(int argc, char** argv) {
  if (argc == 3 && !std::strcmp(argv[1], "fmt")) {
    for (double x : read_all(argv[2])) std::cout << okg::format_g17(x) << "\n";
    return 0;
  }
  if (argc == 6 && !std::strcmp(argv[1], "vtk")) {
    const std::vector<double> d = read_all(argv[4]);
    const size_t h = d.size() / 2;
    okg::write_vtk(std::atoi(argv[2]), std::atoi(argv[3]), okg::Vector(d.begin(), d.begin() + h),
                   okg::Vector(d.begin() + h, d.end()), argv[5]);
    return 0;
  }
  if (argc == 7 && !std::strcmp(argv[1], "run")) {
    okg::SolverConfig cfg;
    cfg.dim = std::atoi(argv[2]);
    cfg.n = std::atoi(argv[3]);
    cfg.n_steps = std::atoi(argv[4]);
    cfg.m = 0.1;
    cfg.gmres_tol = 1e-10;
    cfg.gmres_restart = 30;
    return okg::cmd_run(cfg, argv[6], std::atoi(argv[5]));
  }
  if (argc == 3 && !std::strcmp(argv[1], "cfg")) {
    try {
      const okg::RunManifest man = okg::parse_config(argv[2]);
      const okg::SolverConfig& c = man.config;
      auto d = [&](const char* k, double v) { std::cout << k << '=' << okg::format_g17(v) << '\n'; };
      auto i = [&](const char* k, long v) { std::cout << k << '=' << v << '\n'; };
      d("eps", c.eps); d("sigma", c.sigma); d("m", c.m); d("theta", c.theta); d("dt", c.dt);
      i("n_steps", c.n_steps); i("dim", c.dim); i("n", c.n); d("newton_tol", c.newton_tol);
      i("newton_maxit", c.newton_maxit); d("gmres_tol", c.gmres_tol); i("gmres_maxit", c.gmres_maxit);
      i("gmres_restart", c.gmres_restart); i("cheby_iters", c.cheby_iters);
      std::cout << "cheby_precond=" << c.cheby_precond << '\n';
      i("richardson_steps", c.richardson_steps); i("mg_cycles", c.mg_cycles); i("mg_pre", c.mg_pre);
      i("mg_post", c.mg_post); d("mg_omega", c.mg_omega); i("min_coarse_size", c.min_coarse_size);
      i("threads", c.threads); i("max_dofs", c.max_dofs);
      std::cout << "output_dir=" << c.output_dir << '\n';
      i("snapshot_every", c.snapshot_every);
      std::cout << "mesh_study_n=";
      for (size_t q = 0; q < c.mesh_study_n.size(); ++q) std::cout << (q ? "," : "") << c.mesh_study_n[q];
      std::cout << "\neps_list=";
      for (size_t q = 0; q < c.eps_list.size(); ++q) std::cout << (q ? "," : "") << okg::format_g17(c.eps_list[q]);
      std::cout << '\n';
    } catch (const okg::ConfigError& e) {
      std::cout << "ERR -3: " << e.what() << "\n";
    }
    return 0;
  }
  std::cerr << "usage: test_okflow_io fmt IN | vtk DIM N IN OUT | run DIM N STEPS EVERY OUTDIR\n";
  return 1;
}
