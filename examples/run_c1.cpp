// Minimal C++ user of the drop-in shim: BASELINE config 1 (the reference's
// own layout, feti-schur), first through the reference's step decomposition
// (interface_rhs -> feti_pcg -> back_substitute, timeloop.hpp:163-176), then
// every step of the run (StepSolver::advance on the device-resident state).  Build (tests/test_gpu_boundary.py does):
//   g++ -std=c++17 -Iinclude examples/run_c1.cpp -Lpaper_2509_06673_b200/_lib -lporofeti_b200
//       -Wl,-rpath,$PWD/paper_2509_06673_b200/_lib -o run_c1
#include <cmath>
#include <cstdio>

#include "porofeti_b200.hpp"

namespace pb = porofeti_b200;

int main() {
  pf_config cfg = pb::default_config();
  try {
    {
      pb::Problem problem(cfg);
      const pb::Vector F = problem.interface_rhs();
      const pb::Vector lambda0(problem.n_lambda(), 0.0);
      const pb::PcgResult res = pb::feti_pcg(problem, F, lambda0, cfg.tol, cfg.max_iter);
      const pb::Vector x = problem.back_substitute(res.lambda);
      double nl = 0.0, nx = 0.0;
      for (double v : res.lambda) nl += v * v;
      for (double v : x) nx += v * v;
      std::printf("pieces step 1 iters %d history %zu delta0 %.17g lambda_norm %.17g x_norm %.17g\n",
                  res.report.iterations, res.residual_history.size(),
                  res.residual_history.empty() ? 0.0 : res.residual_history[0], std::sqrt(nl), std::sqrt(nx));
    }
    pb::Problem problem(cfg);
    for (int n = 0; n < problem.info().N; ++n) {
      const pb::PcgReport r = problem.step();
      const auto [eu, ep] = problem.errors();
      std::printf("step %d iters %d rel %.3e true %.3e err_u %.17g err_p %.17g ms %.3f\n", r.step, r.iterations,
                  r.rel_residual, r.true_residual, eu, ep, r.seconds * 1e3);
    }
    // SolverChoice::monolithic (timeloop.hpp:139-160): the direct interface
    // solve, the same discrete solution without Krylov iterations
    pb::SolveOptions mopts;  // the reference's SolveOptions (timeloop.hpp:123-131)
    mopts.solver = pb::SolverChoice::monolithic, mopts.tol = cfg.tol, mopts.max_iter = cfg.max_iter;
    pb::Problem mono(cfg, mopts);
    pb::StepSolver msolver(mono, mopts);
    (void)msolver;
    for (int n = 0; n < mono.info().N; ++n) {
      const pb::PcgReport r = mono.step();
      const auto [eu, ep] = mono.errors();
      std::printf("%s %d iters %d true %.3e err_u %.17g err_p %.17g ms %.3f\n",
                  pb::solver_name(pb::SolverChoice::monolithic), r.step, r.iterations, r.true_residual, eu, ep,
                  r.seconds * 1e3);
    }
  } catch (const pb::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
