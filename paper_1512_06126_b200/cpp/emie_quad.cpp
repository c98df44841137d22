// emie-b200 drop-in: the host-side test oracles of the reference API --
// bessel_zeros (include/emie/quad.hpp:16) and kernel_output_oracle
// (include/emie/hankel.hpp:57-58: "slow; exists so tests can gate the closed
// forms"). Neither is on the device hot path: the Green's build evaluates the
// closed forms (kernel_output) on the GPU; these exist so the reference's own
// quad and hankel suites compile and run unchanged against the drop-in.
#include <cmath>
#include <stdexcept>
#include <utility>
#include <vector>

#include "emie/hankel.hpp"
#include "emie/quad.hpp"

namespace emie {

namespace {
constexpr double kPi = 3.14159265358979323846;

double bessel_j(int nu, double x) { return std::cyl_bessel_j(static_cast<double>(nu), x); }

// n-point Gauss-Legendre rule on [-1, 1] by Newton on P_n (three-term recurrence)
std::vector<std::pair<double, double>> gauss_legendre(int n) {
  std::vector<std::pair<double, double>> r(n);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(kPi * (i + 0.75) / (n + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-16) break;
    }
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (x * p1 - p0) / (x * x - 1.0);
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    r[i] = {x, w};
    r[n - 1 - i] = {-x, w};
  }
  return r;
}

// composite rule on [a, b]: panels of length <= 4 (under one period of the
// Bessel factor), each with the 30-point Gauss rule -- fixed, so the outer
// adaptive integration sees a smooth, noise-free function of its variable
template <class F>
double composite(double a, double b, F&& f) {
  static const std::vector<std::pair<double, double>> gl = gauss_legendre(30);
  if (b <= a) return 0.0;
  const int panels = 1 + static_cast<int>((b - a) / 4.0);
  const double h = 0.5 * (b - a) / panels;
  double sum = 0.0;
  for (int c = 0; c < panels; ++c) {
    const double m = a + (2 * c + 1) * h;
    double s = 0.0;
    for (const auto& [x, w] : gl) s += w * f(m + h * x);
    sum += h * s;
  }
  return sum;
}

void check_orders(int alpha, int beta) {  // hankel.cpp's order check
  if (alpha < 0 || beta < 0 || alpha > 2 || beta > 2 || alpha + beta > 2)
    throw std::invalid_argument("kernel orders: need alpha, beta >= 0 and alpha + beta <= 2");
}
}  // namespace

std::vector<double> bessel_zeros(int nu, int count) {
  if (nu != 0 && nu != 1) throw std::invalid_argument("bessel_zeros: order must be 0 or 1");
  std::vector<double> z;
  if (count <= 0) return z;
  z.reserve(count);
  const double mu = 4.0 * nu * nu;
  for (int k = 1; k <= count; ++k) {
    // McMahon's expansion as the start, then Newton on J_nu
    const double b = (k + 0.5 * nu - 0.25) * kPi;
    double x = b - (mu - 1.0) / (8.0 * b) - 4.0 * (mu - 1.0) * (7.0 * mu - 31.0) / (3.0 * std::pow(8.0 * b, 3));
    for (int it = 0; it < 50; ++it) {
      const double j = bessel_j(nu, x);
      const double dj = nu == 0 ? -bessel_j(1, x) : bessel_j(0, x) - bessel_j(1, x) / x;
      const double dx = j / dj;
      x -= dx;
      if (std::abs(dx) <= 1e-16 * x) break;
    }
    z.push_back(x);
  }
  return z;
}

// The design pair's output by direct evaluation of its defining convolution
// (the closed forms of kernel_output restated as integrals): in log radius,
//   u(s) = int K(e^{s-t}) e^{-(3-a-b)(s-t)} v(e^{-t}) dt,   v = design_input,
// with K(zeta) the lateral cell-pair integral of J0 at scale zeta -- per axis a
// triangular weight (order 0), a signed pair of boxes (order 1) or the
// three-point stencil (order 2) around the scaled centre offset
// zeta (cos phi + p/2, sin phi + q/2) with half-widths zeta p, zeta q.
double kernel_output_oracle(const PairGeometry& g, int alpha, int beta, double s, double rel_tol) {
  check_orders(alpha, beta);
  const int pw = 3 - alpha - beta;
  // one axis' weight: order 0 triangle (h - |x - c|), order 1 boxes (-1 below c, +1 above)
  auto axis_w = [](int order, double c, double h, double x) {
    return order == 0 ? h - std::abs(x - c) : (x < c ? -1.0 : 1.0);
  };
  auto kernel_k = [&](double zeta) -> double {
    const double cx = zeta * (std::cos(g.phi) + 0.5 * g.p), hx = zeta * g.p;
    const double cy = zeta * (std::sin(g.phi) + 0.5 * g.q), hy = zeta * g.q;
    if (alpha == 2 || beta == 2) {  // stencil along one axis, triangle along the other
      const bool onx = alpha == 2;
      const double cs = onx ? cx : cy, hs = onx ? hx : hy;  // stencil axis
      const double ct = onx ? cy : cx, ht = onx ? hy : hx;  // integrated axis
      const double pt[3] = {cs - hs, cs, cs + hs}, cf[3] = {1.0, -2.0, 1.0};
      double acc = 0.0;
      for (int i = 0; i < 3; ++i) {
        auto f = [&](double t) { return axis_w(0, ct, ht, t) * bessel_j(0, std::hypot(pt[i], t)); };
        acc += cf[i] * (composite(ct - ht, ct, f) + composite(ct, ct + ht, f));
      }
      return acc;
    }
    double acc = 0.0;
    // each axis split at its centre (the weights' kink / sign change)
    const double xs[3] = {cx - hx, cx, cx + hx}, ys[3] = {cy - hy, cy, cy + hy};
    for (int sy = 0; sy < 2; ++sy)
      acc += composite(ys[sy], ys[sy + 1], [&](double y) {
        double in = 0.0;
        for (int sx = 0; sx < 2; ++sx)
          in += composite(xs[sx], xs[sx + 1],
                          [&](double x) { return axis_w(alpha, cx, hx, x) * bessel_j(0, std::hypot(x, y)); });
        return axis_w(beta, cy, hy, y) * in;
      });
    return acc;
  };
  // the input's support: v(e^{-t}) is negligible outside t in [-2.7, 42];
  // samples far below the requested accuracy are not priced
  const double tiny = 1e-3 * rel_tol;
  auto integrand = [&](double t) -> double {
    const double v = design_input(std::exp(-t));
    if (std::abs(v) < tiny) return 0.0;
    const double w = s - t;
    return kernel_k(std::exp(w)) * std::exp(-pw * w) * v;
  };
  return integrate(integrand, -2.7, 42.0, 0.1 * rel_tol, 15);
}

}  // namespace emie
