// oracle/adapter_check.cpp — TEST INFRASTRUCTURE.  Proves the drop-in: the
// reference's own types and generators (unmodified headers) call both
// qpcg::solve (reference, CPU) and qpcg::b200::solve (include/qpcg_b200_adapter.hpp,
// B200 engine) on the same instance; prints one line per class.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "qpcg/bench/generators.hpp"
#include "qpcg/solver.hpp"
#include "qpcg_b200_adapter.hpp"

int main(int argc, char** argv) {
  const unsigned scale = argc > 1 ? unsigned(std::atoi(argv[1])) : 3;
  int bad = 0;
  for (auto cls : qpcg::bench::all_classes()) {
    qpcg::bench::BenchSpec spec;
    spec.problem_class = cls;
    spec.scale_index = scale;
    const auto p = qpcg::bench::generate<double>(spec);
    qpcg::Settings<double> s;
    s.lambda_pcg = 0.01;
    const auto r = qpcg::solve(p, s);
    qpcg::SolveDiagnostics<double> d;
    const auto g = qpcg::b200::solve(p, s, nullptr, &d);
    const double rel = std::abs(g.objective - r.objective) / std::max(1.0, std::abs(r.objective));
    const bool ok = g.status == r.status && (rel < 1e-2 || !std::isfinite(r.objective));
    bad += !ok;
    std::printf("%s %s/%u/%llu b200 %s/%u/%llu rel_obj=%.2e pcg_calls=%zu %s\n",
                qpcg::bench::to_string(cls), qpcg::to_string(r.status), r.iterations,
                (unsigned long long)r.pcg_iterations_total, qpcg::to_string(g.status),
                g.iterations, (unsigned long long)g.pcg_iterations_total, rel, d.pcg_calls.size(),
                ok ? "OK" : "MISMATCH");
  }
  // exception mapping: invalid settings -> std::invalid_argument
  try {
    qpcg::Settings<double> s;
    s.alpha = 3.0;
    (void)qpcg::b200::solve(qpcg::bench::generate<double>({}), s);
    std::printf("no exception\n");
    bad++;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  return bad ? 1 : 0;
}
