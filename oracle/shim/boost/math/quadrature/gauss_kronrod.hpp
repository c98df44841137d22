// Boost.Math shim: adaptive Gauss-Kronrod G7/K15 used by
// /root/reference/proj/include/emie/quad.hpp:19-23 (oracle/test code only).
// TEST INFRASTRUCTURE ONLY. Published QUADPACK qk15 nodes and weights; the
// tolerance is taken relative to the L1 norm of the integrand, as Boost does.
#pragma once
#include <cmath>
#include <complex>
#include <type_traits>

namespace boost { namespace math { namespace quadrature {

template <class Real, unsigned N>
class gauss_kronrod;

template <class Real>
class gauss_kronrod<Real, 15> {
  static constexpr double xgk[8] = {
      0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
      0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
      0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
      0.207784955007898467600689403773245, 0.000000000000000000000000000000000};
  static constexpr double wgk[8] = {
      0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
      0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
      0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
      0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
  static constexpr double wg[4] = {
      0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
      0.381830050505118944950369775488975, 0.417959183673469387755102040816327};

  template <class F, class V>
  static void rule(F& f, Real a, Real b, V& k15, V& g7, Real& l1) {
    const Real c = (a + b) / 2, h = (b - a) / 2;
    const V fc = f(c);
    k15 = fc * static_cast<Real>(wgk[7]);
    g7 = fc * static_cast<Real>(wg[3]);
    l1 = std::abs(fc) * static_cast<Real>(wgk[7]);
    for (int j = 0; j < 7; ++j) {
      const Real dx = h * static_cast<Real>(xgk[j]);
      const V f1 = f(c - dx), f2 = f(c + dx);
      k15 += (f1 + f2) * static_cast<Real>(wgk[j]);
      l1 += (std::abs(f1) + std::abs(f2)) * static_cast<Real>(wgk[j]);
      if (j % 2 == 1) g7 += (f1 + f2) * static_cast<Real>(wg[j / 2]);
    }
    k15 *= h;
    g7 *= h;
    l1 *= std::fabs(h);
  }

  template <class F, class V>
  static V recurse(F& f, Real a, Real b, unsigned levels, Real abs_tol, Real& err) {
    V k15, g7;
    Real l1;
    rule(f, a, b, k15, g7, l1);
    Real e = std::abs(k15 - g7);
    if (levels == 0 || !(e > abs_tol) || !(std::fabs(b - a) > 0)) {
      err = e;
      return k15;
    }
    const Real mid = (a + b) / 2;
    Real e1 = 0, e2 = 0;
    V r = recurse<F, V>(f, a, mid, levels - 1, abs_tol / 2, e1) +
          recurse<F, V>(f, mid, b, levels - 1, abs_tol / 2, e2);
    err = e1 + e2;
    return r;
  }

 public:
  template <class F>
  static auto integrate(F f, Real a, Real b, unsigned max_depth = 15,
                        Real tol = 1.4901161193847656e-08, Real* error = nullptr,
                        Real* pL1 = nullptr) {
    using V = std::decay_t<decltype(f(a))>;
    V k15, g7;
    Real l1;
    rule(f, a, b, k15, g7, l1);
    Real err = std::abs(k15 - g7);
    V res = k15;
    if (max_depth > 0 && err > tol * l1) {
      res = recurse<F, V>(f, a, b, max_depth, tol * l1, err);
    }
    if (error) *error = err;
    if (pL1) *pL1 = l1;
    return res;
  }
};

}}}  // namespace boost::math::quadrature
