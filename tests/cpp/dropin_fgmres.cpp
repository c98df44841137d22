// fgmres(LinearMap) and solve_cie through the B200 drop-in (include/emie/cie.hpp):
// the device Krylov solver over a caller-supplied host map, with the flexible
// right preconditioner and the live iteration hook of SolverConfig
// (cie.hpp:53-59), on the reference's small contrast grid (test_toeplitz.cpp:
// 25-55). Checks: the map solve reproduces solve_cie (same iteration count,
// solution to 1e-12); the hook runs live once per iteration with the history
// values; a Jacobi preconditioner converges with A x = b; an exception thrown
// by the map propagates unchanged. Prints "dropin_fgmres ok" on success.
#include <cmath>
#include <complex>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "emie/cie.hpp"
#include "emie/greens.hpp"
#include "emie/toeplitz.hpp"

static int fails = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
      ++fails;                                                     \
    }                                                              \
  } while (0)

static double nrm(const emie::GridVector& v) {
  double s = 0;
  for (const auto& c : v.a) s += std::norm(c);
  return std::sqrt(s);
}

int main() {
  using emie::cdouble;
  emie::LayeredModel m;
  m.tops = {0.0, 400.0};
  m.sigma = {cdouble(0.0), cdouble(0.01), cdouble(0.1)};
  emie::AnomalyGrid grid = emie::make_grid(m, {0.0, 200.0, 400.0, 700.0}, 4, 4, 200.0, 260.0, 0.0, 0.0);
  emie::fill_box(grid, 1, 2, 0, 3, 0, 1, cdouble(1.0));
  emie::fill_box(grid, 0, 0, 0, 0, 2, 2, cdouble(0.001));
  const double omega = 2.0 * emie::pi / 50.0;
  const emie::CompressedGreensOperator cop = emie::assemble_operator(grid, m, omega);
  const emie::SpectralOperator sop = emie::transform_operator(cop);
  const emie::SystemOperator sys = emie::build_system(grid, sop);

  emie::GridVector b(4, 4, 3);
  for (std::size_t i = 0; i < b.a.size(); ++i) b.a[i] = cdouble(std::sin(0.37 * i), std::cos(0.11 * i));

  emie::SolverConfig cfg;
  cfg.tol = 1e-10;
  cfg.restart = 7;  // several restart cycles
  std::vector<std::pair<int, double>> seen;
  cfg.on_iteration = [&](int it, double r) { seen.emplace_back(it, r); };
  emie::SolveReport rep;
  const emie::GridVector xs = emie::solve_cie(grid, m, sop, b, cfg, &rep);
  EXPECT(rep.status == emie::SolveStatus::converged);
  EXPECT(static_cast<int>(seen.size()) == rep.iterations);
  for (std::size_t i = 0; i < seen.size() && i < rep.history.size(); ++i) {
    EXPECT(seen[i].first == static_cast<int>(i) + 1);
    EXPECT(seen[i].second == rep.history[i]);
  }

  int calls = 0;
  const emie::LinearMap A = [&](const emie::GridVector& u) {
    ++calls;
    return emie::apply(sys, u);
  };
  seen.clear();
  emie::FgmresResult fr = emie::fgmres(A, b, cfg);
  EXPECT(fr.report.status == emie::SolveStatus::converged);
  EXPECT(fr.report.iterations == rep.iterations);
  EXPECT(static_cast<int>(seen.size()) == fr.report.iterations);
  // one apply per iteration plus one residual per restart cycle, nothing speculative
  const int cycles = (fr.report.iterations + cfg.restart - 1) / cfg.restart;
  EXPECT(calls == fr.report.iterations + cycles);
  double dx = 0;
  for (std::size_t i = 0; i < xs.a.size(); ++i) dx = std::max(dx, std::abs(xs.a[i] - fr.x.a[i]));
  EXPECT(dx <= 1e-12 * nrm(xs));

  // flexible right preconditioning: z = D^-1 v with D the system's diagonal s
  emie::SolverConfig pc = cfg;
  pc.on_iteration = nullptr;
  pc.right_precond = [&](const emie::GridVector& v) {
    emie::GridVector z = v;
    const std::size_t cells = sys.s.size();
    for (std::size_t i = 0; i < z.a.size(); ++i) z.a[i] /= sys.s[i % cells];
    return z;
  };
  emie::FgmresResult pr = emie::fgmres(A, b, pc);
  EXPECT(pr.report.status == emie::SolveStatus::converged);
  const emie::GridVector ax = emie::apply(sys, pr.x);
  emie::GridVector res = b;
  for (std::size_t i = 0; i < res.a.size(); ++i) res.a[i] -= ax.a[i];
  EXPECT(nrm(res) <= 1e-9 * nrm(b));

  // a map that throws: the exception comes back unchanged
  bool caught = false;
  try {
    emie::fgmres([](const emie::GridVector&) -> emie::GridVector { throw std::domain_error("map failed"); }, b, cfg);
  } catch (const std::domain_error& e) {
    caught = std::string(e.what()) == "map failed";
  }
  EXPECT(caught);
  bool bad = false;
  try {
    emie::SolverConfig z = cfg;
    z.restart = 0;
    emie::fgmres(A, b, z);
  } catch (const std::invalid_argument&) {
    bad = true;
  }
  EXPECT(bad);
  if (fails == 0) std::printf("dropin_fgmres ok (%d iterations, %d map calls)\n", fr.report.iterations, calls);
  return fails ? 1 : 0;
}
