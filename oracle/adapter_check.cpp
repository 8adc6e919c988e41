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
    // objective and x within 1e-3 (x scaled by max(1, |x|inf));
    // classes whose eps = 1e-3 answer is chaotic are compared again at 1e-5
    auto close = [](const auto& a, const auto& b, double& ro, double& rx) {
      ro = std::abs(a.objective - b.objective) / std::max(1.0, std::abs(b.objective));
      double dx = 0, xm = 1;
      for (size_t i = 0; i < b.x.size(); ++i) {
        dx = std::max(dx, std::abs(a.x[i] - b.x[i]));
        xm = std::max(xm, std::abs(b.x[i]));
      }
      rx = dx / xm;
      return a.status == b.status && (!std::isfinite(b.objective) || (ro <= 1e-3 && rx <= 1e-3));
    };
    double rel = 0, rx = 0;
    bool ok = close(g, r, rel, rx);
    const char* at = "1e-3";
    if (!ok && g.status == r.status) {
      qpcg::Settings<double> s5 = s;
      s5.eps_abs = s5.eps_rel = 1e-5;
      s5.max_admm_iter = 20000;
      ok = close(qpcg::b200::solve(p, s5), qpcg::solve(p, s5), rel, rx);
      at = "1e-5";
    }
    bad += !ok;
    std::printf("%s %s/%u/%llu b200 %s/%u/%llu rel_obj=%.2e rel_x=%.2e (eps %s) pcg_calls=%zu %s\n",
                qpcg::bench::to_string(cls), qpcg::to_string(r.status), r.iterations,
                (unsigned long long)r.pcg_iterations_total, qpcg::to_string(g.status),
                g.iterations, (unsigned long long)g.pcg_iterations_total, rel, rx, at,
                d.pcg_calls.size(), ok ? "OK" : "MISMATCH");
  }
  // SolveDiagnostics::on_iteration (solver.hpp:451-454): called once per ADMM
  // iteration with the scaled iterates, through the engine's host-driven loop
  {
    qpcg::bench::BenchSpec spec;
    spec.problem_class = qpcg::bench::ProblemClass::kLasso;
    spec.scale_index = scale;
    const auto p = qpcg::bench::generate<double>(spec);
    qpcg::Settings<double> s;
    s.lambda_pcg = 0.01;
    // the callback also sees this iteration's PcgCall already appended
    // (solver.hpp:446-454 appends it before calling on_iteration)
    bool calls_in_step = true;
    qpcg::SolveDiagnostics<double>* watched = nullptr;
    auto observe = [&calls_in_step, &watched](std::vector<unsigned>& its, std::vector<double>& xn) {
      return [&its, &xn, &calls_in_step, &watched](const qpcg::IterationView<double>& v) {
        if (watched && (watched->pcg_calls.empty() || watched->pcg_calls.back().admm_iter != v.iter))
          calls_in_step = false;
        its.push_back(v.iter);
        double m = 0;
        for (double e : v.x) m = std::max(m, std::abs(e));
        xn.push_back(m);
      };
    };
    std::vector<unsigned> ri, gi;
    std::vector<double> rx, gx;
    qpcg::SolveDiagnostics<double> dr, dg;
    dr.on_iteration = observe(ri, rx);
    dg.on_iteration = observe(gi, gx);
    watched = &dr;
    const auto r = qpcg::solve(p, s, nullptr, &dr);
    const bool ref_in_step = calls_in_step;
    watched = &dg;
    const auto g = qpcg::b200::solve(p, s, nullptr, &dg);
    const bool b200_in_step = calls_in_step && ref_in_step;
    bool ok = gi.size() == g.iterations && ri.size() == r.iterations && !gi.empty();
    for (size_t i = 0; ok && i < gi.size(); ++i) ok = gi[i] == i + 1;
    double d = 0;
    for (size_t i = 0; ok && i < std::min<size_t>(3, gx.size()); ++i)
      d = std::max(d, std::abs(gx[i] - rx[i]) / std::max(1.0, rx[i]));
    ok = ok && d < 1e-6 && b200_in_step && dg.pcg_calls.size() == g.iterations;
    bad += !ok;
    std::printf("on_iteration: reference %zu calls, b200 %zu calls, first |x|inf rel diff %.1e %s\n",
                ri.size(), gi.size(), d, ok ? "OK" : "MISMATCH");
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
