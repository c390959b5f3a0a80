// test_okflow_io.cpp -- the C++ output formats (include/okg/okflow_io.hpp):
//   test_okflow_io fmt IN.bin            one format_g17 line per double
//   test_okflow_io vtk DIM N IN.bin OUT  write_vtk of u, w = the halves of IN.bin
//   test_okflow_io run DIM N STEPS EVERY OUTDIR   cmd_run on the GPU
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <vector>

#include "okg/okflow_io.hpp"

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
  std::cerr << "usage: test_okflow_io fmt IN | vtk DIM N IN OUT | run DIM N STEPS EVERY OUTDIR\n";
  return 1;
}
