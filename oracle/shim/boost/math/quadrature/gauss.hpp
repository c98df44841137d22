// Boost.Math shim: Gauss-Legendre rules used by the reference oracles
// (/root/reference/proj/src/hankel.cpp:122-130,
//  /root/reference/proj/tests/support/oracle_greens.hpp:36-45).
// TEST INFRASTRUCTURE ONLY. Nodes/weights by Newton iteration on P_N in long
// double; abscissa()/weights() hold the non-negative half, as Boost does.
#pragma once
#include <array>
#include <cmath>

namespace boost { namespace math { namespace quadrature {

template <class Real, unsigned N>
class gauss {
  struct Tables {
    std::array<Real, (N + 1) / 2> x{}, w{};
    Tables() {
      const long double pi = 3.14159265358979323846264338327950288L;
      for (unsigned i = 0; i < (N + 1) / 2; ++i) {
        // i-th non-negative root, ascending: start from the i-th largest
        // Chebyshev-like guess and keep the ascending order Boost uses
        const unsigned k = (N + 1) / 2 - i;  // k-th root counting from the top
        long double z = std::cos(pi * (k - 0.25L) / (N + 0.5L));
        long double dp = 0;
        for (int it = 0; it < 100; ++it) {
          long double p0 = 1, p1 = z;
          for (unsigned n = 2; n <= N; ++n) {
            long double p2 = ((2 * n - 1) * z * p1 - (n - 1) * p0) / n;
            p0 = p1;
            p1 = p2;
          }
          dp = N * (z * p1 - p0) / (z * z - 1);
          long double dz = p1 / dp;
          z -= dz;
          if (std::fabs(dz) < 1e-30L) break;
        }
        {
          long double p0 = 1, p1 = z;
          for (unsigned n = 2; n <= N; ++n) {
            long double p2 = ((2 * n - 1) * z * p1 - (n - 1) * p0) / n;
            p0 = p1;
            p1 = p2;
          }
          dp = N * (z * p1 - p0) / (z * z - 1);
        }
        if (N % 2 == 1 && i == 0) z = 0;
        x[i] = static_cast<Real>(std::fabs(z));
        w[i] = static_cast<Real>(2 / ((1 - z * z) * dp * dp));
      }
    }
  };
  static const Tables& tab() {
    static const Tables t;
    return t;
  }

 public:
  static const std::array<Real, (N + 1) / 2>& abscissa() { return tab().x; }
  static const std::array<Real, (N + 1) / 2>& weights() { return tab().w; }
};

}}}  // namespace boost::math::quadrature
