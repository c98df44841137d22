// Boost.Math shim: Bessel J and its zeros, used only by oracle/test code in
// the reference (/root/reference/proj/src/hankel.cpp:119, quad.cpp:7-16).
// TEST INFRASTRUCTURE ONLY. J via libstdc++'s std::cyl_bessel_j; zeros by
// McMahon's expansion refined with Newton steps.
#pragma once
#include <cmath>

namespace boost { namespace math {

template <class T1, class T2>
inline double cyl_bessel_j(T1 nu, T2 x) {
  const double xx = static_cast<double>(x);
  const double v = static_cast<double>(nu);
  if (xx < 0) {
    // integer orders only are used: J_n(-x) = (-1)^n J_n(x)
    const double r = std::cyl_bessel_j(v, -xx);
    return (static_cast<long>(v) % 2) ? -r : r;
  }
  return std::cyl_bessel_j(v, xx);
}

template <class T>
inline double cyl_bessel_j_zero(T nu, int k) {
  const double v = static_cast<double>(nu);
  const double pi = 3.14159265358979323846;
  const double beta = (k + 0.5 * v - 0.25) * pi;
  const double mu = 4 * v * v;
  double x = beta - (mu - 1) / (8 * beta) -
             4 * (mu - 1) * (7 * mu - 31) / (3 * std::pow(8 * beta, 3));
  for (int it = 0; it < 60; ++it) {
    const double j = std::cyl_bessel_j(v, x);
    // J_v'(x) = J_{v-1}(x) - (v/x) J_v(x); J_0' = -J_1
    const double jp = (v == 0) ? -std::cyl_bessel_j(1.0, x)
                               : std::cyl_bessel_j(v - 1, x) - v / x * j;
    const double dx = j / jp;
    x -= dx;
    if (std::fabs(dx) < 1e-15 * x) break;
  }
  return x;
}

}}  // namespace boost::math
