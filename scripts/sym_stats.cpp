// Host-only statistics of the symbolic schedule (supernode / panel sizes per
// level) for a BASELINE config: g++ -O2 -std=c++17 -I. scripts/sym_stats.cpp
#include <cstdio>
#include <map>
#include "paper_2509_06673_b200/csrc/pf_disc.hpp"
#include "paper_2509_06673_b200/csrc/pf_symbolic.hpp"
using namespace pf;
int main(int argc, char** argv) {
  pf_config c{};
  c.mesh_n = argc > 1 ? atoi(argv[1]) : 1024; c.SX = c.SY = argc > 2 ? atoi(argv[2]) : 32; c.order = 2;
  c.E = 1, c.nu = 0.3, c.alpha = 1, c.c0 = 1e-3, c.kperm = 1, c.mu_f = 1, c.dt = 1e-2, c.steps = 1;
  c.scenario = PF_SCEN_MMS_T, c.precond = PF_PREC_DIRICHLET_MORTAR, c.tol = 1e-10, c.max_iter = 500;
  c.seed = 20240901ull, c.logk_mean = -2, c.logk_sd = 1;
  Disc D = build_disc(c, nullptr);
  // most common type
  std::map<int, int> cnt;
  for (auto& s : D.subs) cnt[s.type]++;
  int t = 0, best = 0;
  for (auto& kv : cnt) if (kv.second > best) best = kv.second, t = kv.first;
  const SubType& T = D.types[t];
  SymFactor F = analyse(T.K, T.dof_ic, 16384, 256);
  printf("type %d (x%d): n %d nsn %d nval %lld ntask %d nlevel %d\n", t, best, F.n, F.nsn, F.nval, F.ntask, F.nlevel);
  for (int l = 0; l < F.nlevel; ++l) {
    long long vals = 0, nsn = 0, tasks = 0, maxpanel = 0, maxsn = 0, panels = 0;
    std::map<int, long long> hist;  // panel width -> values
    for (int q = F.level_ptr[l]; q < F.level_ptr[l + 1]; ++q) {
      tasks++;
      for (int k = F.task_sn0[q]; k < F.task_sn1[q]; ++k) {
        const int nc = F.sn_ncol[k], m = F.sn_nrow[k];
        long long v = (long long)nc * (m - 1) - (long long)nc * (nc - 1) / 2;
        vals += v, nsn++, maxsn = std::max(maxsn, v);
        for (int p0 = 0; p0 < nc; p0 += 32) {
          int pw = std::min(32, nc - p0);
          long long pv = 0;
          for (int j = p0; j < p0 + pw; ++j) pv += m - j - 1;
          maxpanel = std::max(maxpanel, pv), panels++;
          hist[pw <= 4 ? 4 : pw <= 8 ? 8 : pw <= 16 ? 16 : 32] += pv;
        }
      }
    }
    printf("level %d: tasks %lld sn %lld vals %lld (%.1f%%) vals/task %.0f vals/sn %.0f max sn %lld max panel %lld panels %lld |", l,
           tasks, nsn, vals, 100.0 * vals / F.nval, (double)vals / tasks, (double)vals / nsn, maxsn, maxpanel, panels);
    for (auto& h : hist) printf(" pw<=%d: %.0f%%", h.first, 100.0 * h.second / vals);
    printf("\n");
  }
}
