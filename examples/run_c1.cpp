// Minimal C++ user of the drop-in shim: BASELINE config 1, all steps.
//   g++ -std=c++17 -Iinclude examples/run_c1.cpp -Lpaper_2509_06673_b200/_lib -lporofeti_b200 \
//       -Wl,-rpath,$PWD/paper_2509_06673_b200/_lib -o run_c1
#include <cstdio>

#include "porofeti_b200.hpp"

int main() {
  pf_config cfg = porofeti_b200::default_config();
  try {
    porofeti_b200::Problem problem(cfg);
    for (const auto& r : porofeti_b200::run_simulation(problem))
      std::printf("step %d  iters %d  rel %.2e  %.3f ms\n", r.step, r.iterations, r.rel_residual, r.seconds * 1e3);
  } catch (const porofeti_b200::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
