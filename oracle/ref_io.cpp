// ref_io.cpp — TEST INFRASTRUCTURE: the reference's own io.hpp (text problem
// format, settings JSON) driven from the command line, to pin
// paper_1912_04263_b200/textio.py (tests/test_textio.py).  Built from the
// unmodified reference headers by oracle/Makefile into oracle/_ref/.
//
//   ref_io gen <class 0-6> <scale> <seed> <out> [f32]   generate<T> + save_problem
//   ref_io rt <in> <out> [f32]                          load_problem<T> + save_problem
//   ref_io settings <json>                              load_settings<double>, one field per line
//
// Exceptions print "ERR runtime|invalid <what()>" on stdout and exit 3.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "qpcg/bench/generators.hpp"
#include "qpcg/io.hpp"

namespace qb = qpcg::bench;

template <typename T>
int run(int argc, char** argv) {
  const std::string cmd = argv[1];
  if (cmd == "gen" && argc >= 6) {
    qb::BenchSpec spec;
    spec.problem_class = static_cast<qb::ProblemClass>(std::atoi(argv[2]));
    spec.scale_index = static_cast<qpcg::index_t>(std::atoi(argv[3]));
    spec.seed = std::strtoull(argv[4], nullptr, 10);
    qpcg::save_problem(argv[5], qb::generate<T>(spec));
    return 0;
  }
  if (cmd == "rt" && argc >= 4) {
    qpcg::save_problem(argv[3], qpcg::load_problem<T>(argv[2]));
    return 0;
  }
  if (cmd == "settings" && argc >= 3) {
    const qpcg::Settings<double> s = qpcg::load_settings<double>(argv[2]);
    std::printf("alpha=%.17g\nsigma=%.17g\nrho_bar_init=%.17g\neps_abs=%.17g\neps_rel=%.17g\n"
                "eps_pinf=%.17g\neps_dinf=%.17g\nmax_admm_iter=%u\ncheck_interval=%u\n"
                "rho_update_interval=%u\nlambda_pcg=%.17g\neps_pcg_min=%.17g\n"
                "scaling_enabled=%d\neps_equil=%.17g\nequil_max_passes=%u\n",
                s.alpha, s.sigma, s.rho_bar_init, s.eps_abs, s.eps_rel, s.eps_pinf, s.eps_dinf,
                s.max_admm_iter, s.check_interval, s.rho_update_interval, s.lambda_pcg,
                s.eps_pcg_min, int(s.scaling_enabled), s.eps_equil, s.equil_max_passes);
    return 0;
  }
  std::fprintf(stderr, "usage: ref_io gen|rt|settings ...\n");
  return 2;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const bool f32 = std::strcmp(argv[argc - 1], "f32") == 0;
  try {
    return f32 ? run<float>(argc, argv) : run<double>(argc, argv);
  } catch (const std::invalid_argument& e) {
    std::printf("ERR invalid %s\n", e.what());
  } catch (const std::exception& e) {
    std::printf("ERR runtime %s\n", e.what());
  }
  return 3;
}
