// pf_common.hpp — shared host types of the B200 FETI engine: configuration,
// error/status codes (reference core.hpp:32-75 mapped to C-ABI codes), and a
// minimal CSR container.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/porofeti_b200.h"

namespace pf {

enum Status : int {
  kOk = PF_OK,
  kSingular = PF_SINGULAR,        // SingularSubproblemError
  kBreakdown = PF_BREAKDOWN,      // PcgBreakdownError
  kNotConverged = PF_NOT_CONVERGED,  // SolverError
  kInvalid = PF_INVALID,          // AssemblyError / ConfigError / MeshError
  kCuda = PF_CUDA,
  kInternal = PF_INTERNAL,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

struct Csr {
  int nr = 0, nc = 0;
  std::vector<int> ptr{0}, col;
  std::vector<double> val;
  int nnz() const { return (int)col.size(); }
  int find(int r, int c) const {  // position of (r,c) or -1 (columns sorted)
    auto b = col.begin() + ptr[r], e = col.begin() + ptr[r + 1];
    auto it = std::lower_bound(b, e, c);
    return (it != e && *it == c) ? int(it - col.begin()) : -1;
  }
};

/// Build a CSR pattern from (row, col) pairs (sorted, unique).
inline Csr pattern_from_pairs(int nr, int nc, std::vector<std::pair<int, int>>& rc) {
  std::sort(rc.begin(), rc.end());
  rc.erase(std::unique(rc.begin(), rc.end()), rc.end());
  Csr m;
  m.nr = nr;
  m.nc = nc;
  m.ptr.assign(nr + 1, 0);
  m.col.resize(rc.size());
  for (std::size_t k = 0; k < rc.size(); ++k) {
    m.ptr[rc[k].first + 1]++;
    m.col[k] = rc[k].second;
  }
  for (int i = 0; i < nr; ++i) m.ptr[i + 1] += m.ptr[i];
  m.val.assign(rc.size(), 0.0);
  return m;
}

struct Material {
  double lam_P = 0, mu_P = 0, lam_E = 0, mu_E = 0, alpha = 1, c0 = 0, kperm = 1, mu_f = 1;
  double k1 = 0, k2 = 0, k3 = 0;
  double tau = 0, T = 0;
  int N = 0;
};

/// Lame constants with the reference's default "paper" shear modulus
/// mu = E/(1+nu) (model.hpp:17-32) and the kappas of model.hpp:38-42.
inline Material make_material(const pf_config& c) {
  if (!(c.E > 0)) fail(kInvalid, "lame_from_young_poisson: E must be positive");
  if (c.nu < 0 || c.nu >= 0.5) fail(kInvalid, "lame_from_young_poisson: need 0 <= nu < 0.5");
  Material m;
  m.lam_P = m.lam_E = c.E * c.nu / ((1 + c.nu) * (1 - 2 * c.nu));
  m.mu_P = m.mu_E = c.mu_conv == 1 ? c.E / (2 * (1 + c.nu)) : c.E / (1 + c.nu);
  m.alpha = c.alpha;
  m.c0 = c.c0;
  if (!(c.kperm > 0)) fail(kInvalid, "make_params: permeability must be positive");
  if (!(c.mu_f > 0)) fail(kInvalid, "make_params: fluid viscosity must be positive");
  m.kperm = c.kperm;
  m.mu_f = c.mu_f;
  const double den = c.alpha * c.alpha + c.c0 * m.lam_P;
  if (den <= 0) fail(kInvalid, "derived_kappas: alpha^2 + c0*lambda_P must be positive");
  m.k1 = c.alpha / den;
  m.k2 = m.lam_P / den;
  m.k3 = c.c0 / den;
  if (!(c.dt > 0) || c.steps < 1) fail(kInvalid, "need dt > 0 and steps >= 1");
  // time grid (timeloop.hpp:15-33): T = steps*dt, N = max(1, llround(T/dt)), tau = T/N
  m.T = c.dt * c.steps;
  m.N = std::max(1, (int)std::llround(m.T / c.dt));
  m.tau = m.T / m.N;
  return m;
}

/// Portable per-element log-normal permeability for the injection scenario
/// (SURVEY App. C D8): splitmix64 -> Box-Muller (cosine branch), element order
/// e = 2*(J*n + I) + k over the global n x n cell grid.
inline std::vector<double> injection_permeability(int n, uint64_t seed, double mean, double sd) {
  std::vector<double> k(std::size_t(2) * n * n);
  uint64_t s = seed;
  auto next = [&s]() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  auto unif = [&]() { return ((double)(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); };
  const double two_pi = 6.283185307179586476925286766559;
  for (auto& v : k) {
    const double u1 = unif(), u2 = unif();
    v = std::pow(10.0, mean + sd * (std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2)));
  }
  return k;
}

}  // namespace pf
