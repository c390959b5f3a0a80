// okflow_b200 -- the reference's command line (tools/okflow.cpp) over the B200 solver:
//   okflow_b200 {run|mesh-study|eps-study|verify} --config FILE [--output DIR]
//               [--threads N] [--perturb-shat X]
// Exit codes as the reference: 2 on a configuration error, 1 on any other error.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <iostream>
#include <string>

#include "okg/okflow_cli.hpp"

static int usage() {
  std::cerr << "usage: okflow_b200 {run|mesh-study|eps-study|verify} --config FILE [--output DIR] "
               "[--threads N] [--perturb-shat X]\n";
  return 2;
}

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string kind = argv[1];
  if (kind != "run" && kind != "mesh-study" && kind != "eps-study" && kind != "verify") return usage();
  std::string config_path, output_dir;
  int threads = 0;
  double perturb = 0.0;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (i + 1 >= argc) return usage();
    if (a == "--config") config_path = argv[++i];
    else if (a == "--output") output_dir = argv[++i];
    else if (a == "--threads") threads = std::atoi(argv[++i]);
    else if (a == "--perturb-shat") perturb = std::atof(argv[++i]);
    else return usage();
  }
  if (config_path.empty()) return usage();
  try {
    okg::RunManifest man = okg::parse_config(config_path);
    man.kind = kind;
    man.shat_perturb = perturb;
    if (!output_dir.empty()) man.config.output_dir = output_dir;
    if (threads > 0) man.config.threads = threads;
    man.config.validate();
    return okg::run_manifest(man);
  } catch (const okg::ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
